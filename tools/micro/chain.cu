// microbenchmark: one sequential 800-term fp32 sum per warp over shared memory (config 0's decoder rows)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float lds_f32(unsigned a) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v; }
template <int MODE>
__global__ void chain(float* out, long long* cyc, int n) {
    __shared__ float A[12 * 800], x[800];
    for (int i = threadIdx.x; i < 12 * 800; i += blockDim.x) A[i] = 1e-3f * (i % 97);
    for (int i = threadIdx.x; i < 800; i += blockDim.x) x[i] = (i % 3) ? 0.f : 10.f;
    __syncthreads();
    long long t0 = clock64();
    int r = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0 && r < 12) {
        float acc = 0.f;
        const float* arow = A + r * n;
        if (MODE == 0) {
#pragma unroll 8
            for (int k = 0; k < n; ++k) acc = acc + arow[k] * x[k];
        } else {
            unsigned ar = (unsigned)__cvta_generic_to_shared(arow), xr = (unsigned)__cvta_generic_to_shared(x);
            for (int k = 0; k + 8 <= n; k += 8) {
                float av[8], xv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) { av[u] = lds_f32(ar + 4 * (k + u)); xv[u] = lds_f32(xr + 4 * (k + u)); }
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = acc + av[u] * xv[u];
            }
        }
        out[r] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) *cyc = clock64() - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 64 * 4); cudaMalloc(&c, 8);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            if (mode == 0) chain<0><<<1, 1024>>>(o, c, 800); else chain<1><<<1, 1024>>>(o, c, 800);
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("mode %d: %lld cycles for 800 terms (%.1f per term)\n", mode, h, h / 800.0);
        }
    }
    return 0;
}
