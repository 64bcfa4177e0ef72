# sharding parity (two shards on one GPU) + stepped-path bench at N=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused.py tests/test_abi.py tests/test_drop_in.py -m gpu -x -q > gpurun_out/pytest_shard.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_shard.log
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e --shard ensemble > gpurun_out/bench_shard.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench_shard.log | cut -c1-400
