# full GPU tests, then a bench line with the e2e leg
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/bench_e2e.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_e2e.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e'])"
