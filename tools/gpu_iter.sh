# iteration: fused parity tests + bench line (no CPU baseline) + short profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused.py tests/test_baseline_sizes.py -m gpu -q -s -k "not config1" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|mismatch" gpurun_out/pytest_iter.log | tail -15
timeout 300 python bench.py --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_iter.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'G', d['value']/1e9, 'frac', d['roofline']['frac'], 'e2e G', (d.get('e2e') or {}).get('value',0)/1e9)"
