# benchmark-suite ladder (reference CSV schema) + config-1 parity with least-squares product decoders
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_benchsuite.py tests/test_fused.py -m gpu -x -q -s -k "ablation or config1 or wide" > gpurun_out/pytest_suite.log 2>&1; echo "pytest rc=$?"
grep -E "^benchmark|^(integrator|cconv|pes),|passed|failed|Error" gpurun_out/pytest_suite.log | head -30
timeout 600 python -m paper_1805_11144_b200.benchsuite --benchmark cconv --dims 8 --steps 500 > gpurun_out/cli_cconv.csv 2>&1; echo "cli rc=$?"; cat gpurun_out/cli_cconv.csv
