# A/B: dbg/lib<V>.so variants (VARIANTS env, "product" = the in-tree build) on the config-4 bench,
# then the fused parity tests on the product build
mkdir -p gpurun_out
cp paper_1805_11144_b200/libneng_gpu.so /tmp/libneng_product.so
for v in ${VARIANTS:-product}; do
  if [ "$v" = product ]; then cp /tmp/libneng_product.so paper_1805_11144_b200/libneng_gpu.so; else cp dbg/lib$v.so paper_1805_11144_b200/libneng_gpu.so; fi
  timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.log 2>&1
  echo "== $v $(tail -1 gpurun_out/ab_$v.log | grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|Error.*' | tr '\n' ' ')"
done
cp /tmp/libneng_product.so paper_1805_11144_b200/libneng_gpu.so
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest $TESTS -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
fi
