# quick iteration on the GPU box: parity tests, then the bench (+ section profile)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused.py tests/test_gpu_engine.py -x -q > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_fused.log
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?"
cat gpurun_out/bench_iter.log | tail -3
NENG_FUSED_PROFILE=1 timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "fused profile|error|Error" | tail -4
