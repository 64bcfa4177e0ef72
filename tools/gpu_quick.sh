# quick A/B: config-4 and config-2 bench lines + the fused parity tests
mkdir -p gpurun_out
TAG=${1:-q}
timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/q_${TAG}_c4.log 2>&1; echo "c4 rc=$?"
timeout 300 python bench.py --config 2 --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/q_${TAG}_c2.log 2>&1; echo "c2 rc=$?"
for f in gpurun_out/q_${TAG}_c*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', 'ms/step', round(d['ms_per_step'],4), 'G', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2) if d.get('e2e') else None, 'frac', d.get('roofline',{}).get('frac'), d['clocks'])"; done
timeout 1200 python -m pytest tests/test_fused.py tests/test_baseline_sizes.py tests/test_fused_small.py -m gpu -x -q > gpurun_out/q_${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/q_${TAG}_tests.log
