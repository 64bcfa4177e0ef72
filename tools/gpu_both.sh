# parity + bench + section profile, then one ncu capture of the fused kernel
bash tools/gpu_iter.sh
bash tools/gpu_ncu.sh ${1:-cur}
