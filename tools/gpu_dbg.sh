# debug: small fused network under both schedules, launch-blocking
for df in 0 1; do
  echo "== dataflow=$df"
  NENG_FUSED_DATAFLOW=$df CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_small.py 2>&1 | tail -3
done
