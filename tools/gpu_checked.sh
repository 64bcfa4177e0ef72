# the fused parity tests on the assert-checked build (dbg/libchecked.so: -DNENG_FUSED_CHECKS — the
# barrier-free schedule's dependency claims, queue bounds, shared-memory carve), then the product build
mkdir -p gpurun_out
cp paper_1805_11144_b200/libneng_gpu.so /tmp/libneng_product.so
cp dbg/libchecked.so paper_1805_11144_b200/libneng_gpu.so
timeout 1500 python -m pytest tests/test_fused.py tests/test_baseline_sizes.py -m gpu -q -k "not full_size and not config3 and not config1" > gpurun_out/checked_tests.log 2>&1; echo "checked-build tests rc=$?"; tail -2 gpurun_out/checked_tests.log
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/checked_bench.log 2>&1; echo "checked-build bench rc=$? $(tail -1 gpurun_out/checked_bench.log | cut -c1-200)"
cp /tmp/libneng_product.so paper_1805_11144_b200/libneng_gpu.so
