# tensor-core DotInc: unit tests, config-3 tolerance test, launch list of a config-3 TF32 run
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tc_dot.py tests/test_baseline_sizes.py tests/test_gpu_engine.py -m gpu -x -q -s -k "tc_dot or config3" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"
grep -E "TFLOP|config3 B=512|passed|failed|Error|assert" gpurun_out/pytest_tc.log | head -40
