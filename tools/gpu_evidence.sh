# round evidence: full bench line, launch list and one full ncu capture of the fused kernel
mkdir -p gpurun_out
TAG=${1:-cur}
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}.log | cut -c1-400
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:fused_run -s 1 -c 1 -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
