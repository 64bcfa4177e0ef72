# A/B of prebuilt product-library variants (dbg/lib*.so) on the config-4 bench: each variant is
# copied over the product library for its run, the original restored at the end
mkdir -p gpurun_out
L=paper_1805_11144_b200/libneng_gpu.so
cp $L /tmp/libneng_gpu.orig.so
for v in orig "$@"; do
  if [ $v = orig ]; then cp /tmp/libneng_gpu.orig.so $L; else cp dbg/lib$v.so $L; fi
  timeout 300 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
cp /tmp/libneng_gpu.orig.so $L
