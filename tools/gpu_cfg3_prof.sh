# config 3 (TF32) launch list + one full capture of the tcgen05 DotInc kernel
mkdir -p gpurun_out
timeout 600 python bench.py --config 3 --precision tf32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg3_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg3_tf32_launches.csv python bench.py --config 3 --precision tf32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg3_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_dot_kernel -s 6 -c 1 -o gpurun_out/prof_tcdot -f python bench.py --config 3 --precision tf32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg3_ncu2.log 2>&1; echo "ncu2 rc=$?"
