# full GPU test suite + bench line + section profile
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_iter.log | cut -c1-300
NENG_FUSED_PROFILE=1 timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "fused profile|rror" | tail -4
