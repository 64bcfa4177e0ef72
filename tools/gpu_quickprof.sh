# iteration profile: bench line + one full ncu capture of the fused kernel (config 4, 20 steps)
mkdir -p gpurun_out
TAG=${1:-q}
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'])"
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_run -s 1 -c 1 -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
