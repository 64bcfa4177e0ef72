// tc_dot.cu — dense DotInc on tcgen05 tensor cores (see tc_dot.hpp).
//
// Shared-memory operand layouts (the UMMA canonical forms, 128-byte swizzle,
// 1024-byte aligned atoms of 8 rows x 128 B; TMA writes them swizzled):
//   A, K-major : row m of the stage tile at m*128 B (BK = 128 B of k per stage);
//                SBO = 1024 (next 8 rows); one MMA's k-slice = +32 B in the row.
//   X, MN-major: chunk c (128 B of batch columns) of k-row kr at c*CH + kr*128;
//                LBO = CH (next chunk along N); one MMA's k-slice = +kpm*128 B.
//                bf16: 16-B granules, SBO = 1024 (next 8 k-rows); TF32 (32-bit
//                elements): the 32-B-granule swizzle, SBO = 512 (next 4 k-rows).
// The accumulator is a 128-lane x BN-column fp32 TMEM tile (lane = row).
#include "tc_dot.hpp"

#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

namespace nengb {

namespace {

constexpr int kBM = 128;         // rows per CTA tile (TMEM lanes)
constexpr int kTcThreads = 128;  // 4 warps: TMA producer lane, MMA lane, all four in the epilogue

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count));
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tTC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TC_WAIT_%=;\n\t}" ::"r"(sa(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            sa(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(sa(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tm) : "memory");
}

/// UMMA shared-memory descriptor, version 1.  layout: 2 = 128-byte swizzle
/// (16-B chunks XOR row mod 8, 1024-B atoms), 1 = 128-byte swizzle with 32-B
/// granules (32-B chunks XOR row mod 4, 512-B atoms: the only MN-major layout
/// for 32-bit operands).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return smem_desc(saddr, lbo, sbo, 2);
}

/// Instruction descriptor: fp32 accumulator, A K-major, B MN-major, M = 128, N = bn.
/// fmt: 2 = TF32 (kind::tf32), 1 = BF16 (kind::f16).
__host__ __device__ constexpr uint32_t idesc(uint32_t fmt, int bn) {
    return (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (1u << 16) | (static_cast<uint32_t>(bn >> 3) << 17) |
           (static_cast<uint32_t>(kBM >> 4) << 24);
}

template <int MODE>
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t accumulate) {
    if constexpr (MODE == TC_TF32)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(id), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(id), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

/// 32 consecutive accumulator columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

/// Per-mode tile geometry.
template <int MODE, int BN>
struct Geo {
    static constexpr int kEl = MODE == TC_TF32 ? 4 : 2;        // operand element bytes
    static constexpr int kBK = 128 / kEl;                      // k per stage (one 128-B swizzle row)
    static constexpr int kKpm = MODE == TC_TF32 ? 8 : 16;      // k per MMA
    static constexpr int kChunk = 128 / kEl;                   // batch columns per 128-B chunk
    static constexpr int kChunks = BN / kChunk;
    static constexpr int kABytes = kBM * 128;                  // A tile of one stage (per half)
    static constexpr int kXChunkBytes = kBK * 128;             // one chunk of the X tile
    static constexpr int kXBytes = kChunks * kXChunkBytes;     // X tile of one stage (per half)
    static constexpr int kHalves = MODE == TC_TF32 ? 1 : 2;
    static constexpr int kStageBytes = kHalves * (kABytes + kXBytes);
    // as many stages as fit ~200 KB: the k loop is latency-bound on the TMA round trip at these sizes
    static constexpr int kStages = (200 * 1024 / kStageBytes) < 8 ? (200 * 1024 / kStageBytes) : 8;
    static constexpr size_t kSmem = 1024 + static_cast<size_t>(kStages) * kStageBytes + 256;
    static_assert(BN % kChunk == 0, "BN must be a whole number of 128-byte chunks");
};

template <int MODE, int BN>
__global__ void __launch_bounds__(kTcThreads, 1) tc_dot_kernel(const __grid_constant__ TcDotDesc d) {
    using G = Geo<MODE, BN>;
    extern __shared__ uint8_t tc_smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t{1023});
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::kStages * G::kStageBytes);
    uint64_t* empty = full + G::kStages;
    uint64_t* done = empty + G::kStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
    const int nkb = (d.k + G::kBK - 1) / G::kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < G::kStages; ++s) {
            mb_init(full + s, 1);
            mb_init(empty + s, 1);
        }
        mb_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&d.ta);
        prefetch_tmap(&d.tx);
        if constexpr (MODE == TC_BF16X3) {
            prefetch_tmap(&d.ta_lo);
            prefetch_tmap(&d.tx_lo);
        }
    }
    if (warp == 0) {  // TMEM accumulator: BN columns (a power of two >= 32)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tslot)), "r"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (threadIdx.x == 0) {
        // TMA producer
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % G::kStages;
            if (kb >= G::kStages) mb_wait(empty + s, ((kb / G::kStages) + 1) & 1);
            uint8_t* st = smem + s * G::kStageBytes;
            mb_expect_tx(full + s, G::kStageBytes);
            const int k0 = kb * G::kBK;
            tma_2d(st, &d.ta, k0, m0, full + s);
#pragma unroll
            for (int c = 0; c < G::kChunks; ++c)
                tma_2d(st + G::kABytes + c * G::kXChunkBytes, &d.tx, n0 + c * G::kChunk, k0, full + s);
            if constexpr (MODE == TC_BF16X3) {
                uint8_t* lo = st + G::kABytes + G::kXBytes;
                tma_2d(lo, &d.ta_lo, k0, m0, full + s);
#pragma unroll
                for (int c = 0; c < G::kChunks; ++c)
                    tma_2d(lo + G::kABytes + c * G::kXChunkBytes, &d.tx_lo, n0 + c * G::kChunk, k0, full + s);
            }
        }
    } else if (threadIdx.x == 32) {
        // MMA issuer
        constexpr uint32_t id = idesc(MODE == TC_TF32 ? 2u : 1u, BN);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % G::kStages;
            mb_wait(full + s, (kb / G::kStages) & 1);
            tc_fence_after();
            const uint32_t a_s = sa(smem + s * G::kStageBytes);
            const uint32_t x_s = a_s + G::kABytes;
#pragma unroll
            for (int kk = 0; kk < G::kBK / G::kKpm; ++kk) {
                const uint64_t da = sw128_desc(a_s + kk * 32, 16, 1024);
                // X (MN-major): TF32 in the 32-B-granule layout (4-row atoms, SBO 512), bf16 in the 16-B one
                const uint64_t dx = MODE == TC_TF32 ? smem_desc(x_s + kk * G::kKpm * 128, G::kXChunkBytes, 512, 1)
                                                    : sw128_desc(x_s + kk * G::kKpm * 128, G::kXChunkBytes, 1024);
                const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                mma<MODE>(tmem, da, dx, id, acc);
                if constexpr (MODE == TC_BF16X3) {
                    const uint32_t lo_s = a_s + G::kABytes + G::kXBytes;
                    const uint64_t dal = sw128_desc(lo_s + kk * 32, 16, 1024);
                    const uint64_t dxl = sw128_desc(lo_s + G::kABytes + kk * G::kKpm * 128, G::kXChunkBytes, 1024);
                    mma<MODE>(tmem, da, dxl, id, 1u);   // Ah . Xl
                    mma<MODE>(tmem, dal, dx, id, 1u);   // Al . Xh
                }
            }
            mma_commit(empty + s);  // frees the stage once these MMAs have read it
        }
        mma_commit(done);
    }
    __syncwarp();

    // epilogue: thread = row m0 + threadIdx.x; y = y + acc (the reference's `y[r] += acc`)
    mb_wait(done, 0);
    tc_fence_after();
    const int row = m0 + threadIdx.x;
    float* yr = d.y + static_cast<int64_t>(row) * d.ldy + n0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
        if (row < d.m) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (n0 + c0 + 4 * q < d.n) {
                    float4* p = reinterpret_cast<float4*>(yr + c0 + 4 * q);
                    float4 y = *p;
                    y.x = y.x + v[4 * q];
                    y.y = y.y + v[4 * q + 1];
                    y.z = y.z + v[4 * q + 2];
                    y.w = y.w + v[4 * q + 3];
                    *p = y;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
}

/// BF16X3 split: hi = bf16(v), lo = bf16(v - hi) (both round to nearest even).
__global__ void tc_split_kernel(const float* __restrict__ src, int rows, int cols, int ld, uint16_t* __restrict__ hi,
                                uint16_t* __restrict__ lo, int ldo) {
    const int64_t n = static_cast<int64_t>(rows) * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i - r * cols;
        const float v = src[r * ld + c];
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
        hi[r * ldo + c] = __bfloat16_as_ushort(h);
        lo[r * ldo + c] = __bfloat16_as_ushort(l);
    }
}

// ---- host ---------------------------------------------------------------------

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    });
    return fn;
}

/// 2-D tiled map over a row-major [rows][cols] matrix (row stride ld elements),
/// box {box_cols, box_rows}, 128-byte swizzle, out-of-bounds elements read as 0.
bool make_map(CUtensorMap* m, CUtensorMapDataType ty, int esize, const void* base, int rows, int cols, int ld,
              int box_cols, int box_rows, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeTiled fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * esize};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, ty, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE, int BN>
cudaError_t launch_bn(const TcDotDesc& d, cudaStream_t stream) {
    using G = Geo<MODE, BN>;
    static bool attr = false;  // per instantiation
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(tc_dot_kernel<MODE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(G::kSmem));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const dim3 grid((d.m + kBM - 1) / kBM, (d.n + BN - 1) / BN);
    tc_dot_kernel<MODE, BN><<<grid, kTcThreads, G::kSmem, stream>>>(d);
    return cudaGetLastError();
}

size_t pad16(size_t b) { return (b + 15) & ~size_t{15}; }

}  // namespace

size_t tc_dot_scratch_bytes(int m, int k, int ldx) {
    return 2 * pad16(static_cast<size_t>(m) * k * 2) + 2 * pad16(static_cast<size_t>(k) * ldx * 2);
}

const char* tc_dot_prepare(TcDotDesc* d, const float* a, const float* x, float* y, int m, int k, int n, int ldx,
                           int ldy, int mode, void* scratch) {
    std::memset(d, 0, sizeof(*d));
    if (m < 1 || k < 1 || n < 1) return "empty operand";
    if (!encode_fn()) return "cuTensorMapEncodeTiled unavailable";
    // TMA: 16-B aligned base addresses and row strides; float4 epilogue rows
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (!al16(y) || ldy % 4 || n % 4) return "Y rows not 16-byte aligned";
    d->y = y;
    d->a = a;
    d->x = x;
    d->m = m;
    d->k = k;
    d->n = n;
    d->ldx = ldx;
    d->ldy = ldy;
    d->mode = mode;
    // tile width: the widest that still puts ~a CTA on most SMs (the GEMMs here are small)
    int bn = mode == TC_TF32 ? 256 : 256;
    const int min_bn = mode == TC_TF32 ? 32 : 64;
    const int64_t mt = (m + kBM - 1) / kBM;
    while (bn > min_bn && mt * ((n + bn - 1) / bn) < 120) bn >>= 1;
    if (const char* env = std::getenv("NENG_TC_BN")) {  // experiments: a fixed tile width
        const int f = std::atoi(env);
        if (f >= min_bn && f <= 256 && (f & (f - 1)) == 0) bn = f;
    }
    d->bn = bn;
    if (mode == TC_TF32) {
        if (!al16(a) || k % 4) return "A rows not 16-byte aligned";
        if (!al16(x) || ldx % 4) return "X rows not 16-byte aligned";
        if (!make_map(&d->ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a, m, k, k, 32, kBM)) return "tensor map (A)";
        if (!make_map(&d->tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, k, n, ldx, 32, 32,
                      CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
            return "tensor map (X)";
        return "";
    }
    if (mode != TC_BF16X3) return "unknown mode";
    if (!scratch || !al16(scratch)) return "no split scratch";
    const int ldo = (n + 7) & ~7;  // bf16 rows: 16-B multiples
    uint8_t* s = static_cast<uint8_t*>(scratch);
    const int kp = (k + 7) & ~7;
    d->a_hi = reinterpret_cast<uint16_t*>(s);
    d->a_lo = reinterpret_cast<uint16_t*>(s + pad16(static_cast<size_t>(m) * kp * 2));
    d->x_hi = reinterpret_cast<uint16_t*>(s + 2 * pad16(static_cast<size_t>(m) * kp * 2));
    d->x_lo = reinterpret_cast<uint16_t*>(s + 2 * pad16(static_cast<size_t>(m) * kp * 2) +
                                          pad16(static_cast<size_t>(k) * ldo * 2));
    d->ldx = ldx;
    if (!make_map(&d->ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->a_hi, m, k, kp, 64, kBM) ||
        !make_map(&d->ta_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->a_lo, m, k, kp, 64, kBM))
        return "tensor map (A split)";
    if (!make_map(&d->tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->x_hi, k, n, ldo, 64, 64) ||
        !make_map(&d->tx_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d->x_lo, k, n, ldo, 64, 64))
        return "tensor map (X split)";
    return "";
}

cudaError_t tc_dot_split_a(const TcDotDesc& d, cudaStream_t stream) {
    if (d.mode != TC_BF16X3) return cudaSuccess;
    const int kp = (d.k + 7) & ~7;
    const int64_t n = static_cast<int64_t>(d.m) * d.k;
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
    tc_split_kernel<<<blocks, 256, 0, stream>>>(d.a, d.m, d.k, d.k, d.a_hi, d.a_lo, kp);
    return cudaGetLastError();
}

cudaError_t tc_dot_launch(const TcDotDesc& d, cudaStream_t stream) {
    if (d.mode == TC_BF16X3) {
        const int ldo = (d.n + 7) & ~7;
        const int64_t n = static_cast<int64_t>(d.k) * d.n;
        const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
        tc_split_kernel<<<blocks, 256, 0, stream>>>(d.x, d.k, d.n, d.ldx, d.x_hi, d.x_lo, ldo);
        switch (d.bn) {
            case 64: return launch_bn<TC_BF16X3, 64>(d, stream);
            case 128: return launch_bn<TC_BF16X3, 128>(d, stream);
            case 256: return launch_bn<TC_BF16X3, 256>(d, stream);
        }
        return cudaErrorInvalidValue;
    }
    switch (d.bn) {
        case 32: return launch_bn<TC_TF32, 32>(d, stream);
        case 64: return launch_bn<TC_TF32, 64>(d, stream);
        case 128: return launch_bn<TC_TF32, 128>(d, stream);
        case 256: return launch_bn<TC_TF32, 256>(d, stream);
    }
    return cudaErrorInvalidValue;
}

}  // namespace nengb
