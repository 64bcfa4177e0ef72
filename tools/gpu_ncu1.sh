# one ncu --set full capture of the fused kernel (product build) + a plain timing
mkdir -p gpurun_out
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1
echo "== plain $(tail -1 gpurun_out/plain.log | grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|Error.*' | tr '\n' ' ')"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_run -s 1 -c 1 -o gpurun_out/${NCU_NAME:-prof_fused} -f python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
