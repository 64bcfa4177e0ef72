mkdir -p gpurun_out
NENG_FUSED_PROFILE=1 timeout 300 python bench.py --config 2 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c2_prof.log 2>&1; echo "prof rc=$?"
grep -v "^{" gpurun_out/c2_prof.log | tail -20
CMD="python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_run -s 1 -c 1 -o gpurun_out/prof_c2 -f $CMD > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
