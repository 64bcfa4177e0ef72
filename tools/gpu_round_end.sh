mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/gputest.log
bash tools/gpu_evidence.sh v7
bash tools/gpu_configs.sh
