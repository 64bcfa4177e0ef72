# per-config bench lines (configs 0-3; config 3 strict, tf32, bf16x3) + generic profile of config 0
mkdir -p gpurun_out
for c in 0 1 2; do timeout 600 python bench.py --config $c --steps 200 --warmup 5 > gpurun_out/bench_c$c.log 2>&1; echo "config $c rc=$?"; done
for pr in fp32 tf32 bf16x3; do timeout 600 python bench.py --config 3 --precision $pr --steps 100 --warmup 5 > gpurun_out/bench_c3_$pr.log 2>&1; echo "config 3 $pr rc=$?"; done
NENG_GENERIC_PROFILE=1 timeout 300 python bench.py --config 0 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/prof_c0.log 2>&1; echo "prof c0 rc=$?"
for f in gpurun_out/bench_c*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['config']['workload'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'e2e ms/step', round(d['e2e']['ms_per_step'],4), 'cpu', d.get('cpu_baseline',{}).get('value'), 'val', d['value'])"; done
