for v in ${VARIANTS:-A B}; do
  cp dbg/lib$v.so paper_1805_11144_b200/libneng_gpu.so
  echo "== variant $v"; NENG_FUSED_GRID=1 NENG_FUSED_DATAFLOW=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_small.py 2>&1 | tail -1
done
