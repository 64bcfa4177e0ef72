for v in ${VARIANTS:-A}; do
  cp dbg/lib$v.so paper_1805_11144_b200/libneng_gpu.so
  for df in 0 1; do for g in 1 0; do
  if [ $g != 0 ]; then export NENG_FUSED_GRID=$g; else unset NENG_FUSED_GRID; fi
  echo "== variant $v df=$df grid=$g"; NENG_FUSED_DATAFLOW=$df CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_small.py 2>&1 | tail -1
  done; done
done
