# timing experiment (results not checked): bench + section profile, optional env assignments as args
for kv in "$@"; do export "$kv"; done
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*'
NENG_FUSED_PROFILE=1 timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "fused profile" | tail -1
