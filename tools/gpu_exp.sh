# timing experiment on a prebuilt variant (results not checked)
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-260
NENG_FUSED_PROFILE=1 timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "fused profile" | tail -2
