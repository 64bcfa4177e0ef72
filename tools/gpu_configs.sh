# per-config bench lines (BASELINE configs 0-3) into gpurun_out/cfg_*.json
mkdir -p gpurun_out
for c in "0 fp32 1000" "2 fp32 1000" "3 fp32 100" "3 tf32 100" "3 bf16x3 100" "1 fp32 1000"; do
  set -- $c
  timeout 900 python bench.py --config $1 --precision $2 --steps $3 --warmup 5 > gpurun_out/cfg_$1_$2.log 2>&1
  echo "== config $1 $2 rc=$? $(tail -1 gpurun_out/cfg_$1_$2.log | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print("ms/step %.4f value %.3g e2e ms/step %.4f mode %s launches %s frac %.3f cpu %s" % (d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"], d["config"]["mode"], d["gpu_launches"], d["roofline"]["frac"], (d.get("cpu_baseline") or {}).get("value")))
except Exception as e: print("parse error", e)')"
  tail -1 gpurun_out/cfg_$1_$2.log > gpurun_out/cfg_$1_$2.json
done
