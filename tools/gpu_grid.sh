# config 2: default grid (one CTA per unit) vs every CTA slot (barrier-free claims run ahead into step t+1)
mkdir -p gpurun_out
for g in 0 296; do
  if [ $g = 0 ]; then unset NENG_FUSED_GRID; else export NENG_FUSED_GRID=$g; fi
  timeout 300 python bench.py --config 2 --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/grid_$g.log 2>&1; echo "grid $g rc=$?"
  tail -1 gpurun_out/grid_$g.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('grid $g ms/step', round(d['ms_per_step'],4), 'G', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2), d['clocks'])"
done
export NENG_FUSED_GRID=296
timeout 600 python -m pytest tests/test_baseline_sizes.py -m gpu -x -q -k config2 > gpurun_out/grid_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/grid_tests.log
