# the sharded stepped test under compute-sanitizer (fault location), then ncu counters of the config-4 kernel
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --show-backtrace device python -m pytest tests/test_fused.py -m gpu -x -q -k two_ensemble_shards > gpurun_out/sanit_shard.log 2>&1; echo "sanitizer rc=$?"
grep -B2 -A12 -m3 "Illegal\|illegal\|Invalid\|ERROR" gpurun_out/sanit_shard.log | head -60
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:fused_run -c 1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_counters.log 2>&1; echo "ncu rc=$?"
grep -E "fused_run|duration|bytes|inst_executed|issue_active|sectors|requests|registers|warps_active" gpurun_out/ncu_counters.log | head -20
