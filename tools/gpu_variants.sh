# A/B of prebuilt library variants dbg/lib<V>.so on the config-4 bench (experiments)
for v in ${VARIANTS}; do
  cp dbg/lib$v.so paper_1805_11144_b200/libneng_gpu.so
  echo "== $v $(timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|Error.*' )"
done
