NENG_FUSED_PROFILE=1 timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "fused profile|rror" | tail -4
