// tc_dot.hpp — dense DotInc on the 5th-generation tensor cores (tcgen05).
//
// A dense DotInc member of a per-batch group (shared row-major weights A[M][K],
// per-batch input X and output Y in the arena's [element][batch] layout):
//     Y[m][b] += sum_k A[m][k] X[k][b]            (exec.cpp:226-240)
// computed as acc = A.X on the tensor pipe (fp32 accumulation in TMEM, the sum
// started from 0 as the reference's `acc`), then y = y + acc in the epilogue —
// the reference's association, with acc's products rounded by the mode:
//   TC_TF32   : one kind::tf32 MMA per k-step, operands read as fp32 and rounded
//               to TF32 by the tensor pipe (10-bit mantissa);
//   TC_BF16X3 : A = Ah + Al, X = Xh + Xl split into bf16 pairs by tc_split_kernel;
//               acc = Ah.Xh + Ah.Xl + Al.Xh, three kind::f16 MMAs per k-step
//               (16-bit effective mantissa, the Al.Xl term dropped).
// Operands reach shared memory by TMA (cp.async.bulk.tensor, 128-byte swizzle):
// A K-major, X MN-major (the batch is the arena's innermost dimension).  One CTA
// per 128-row x BN-column tile: thread 0 produces (TMA), thread 32 issues the
// MMAs, all four warps run the epilogue (tcgen05.ld, y + acc, coalesced rows).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace nengb {

enum { TC_TF32 = 0, TC_BF16X3 = 1 };

struct TcDotDesc {
    CUtensorMap ta, tx;        // A (hi), X (hi): fp32 (TF32) or bf16 (BF16X3)
    CUtensorMap ta_lo, tx_lo;  // BF16X3: the low halves
    float* y;                  // Y[M][ldy]
    const float* a;            // fp32 sources of the BF16X3 split
    const float* x;
    uint16_t *a_hi, *a_lo, *x_hi, *x_lo;  // BF16X3 split buffers: A [M][K], X [K][ldx]
    int32_t m, k, n, ldx, ldy;
    int32_t mode, bn;
};

/// Bytes of scratch (device memory) a BF16X3 member needs for its split buffers.
size_t tc_dot_scratch_bytes(int m, int k, int ldx);

/// Fills d for Y[M][n] += A[M][K] X[K][n] (row strides ldx, ldy in floats).
/// Returns an empty string on success, else why the tensor-core path cannot
/// take the member (alignment, shape) — the caller keeps the SIMT path then.
/// scratch: tc_dot_scratch_bytes() bytes, 16-B aligned (BF16X3 only).
const char* tc_dot_prepare(TcDotDesc* d, const float* a, const float* x, float* y, int m, int k, int n, int ldx,
                           int ldy, int mode, void* scratch);

/// BF16X3: split the weights (once per call: constant during a call).
cudaError_t tc_dot_split_a(const TcDotDesc& d, cudaStream_t stream);
/// BF16X3: split X (every step, before tc_dot_launch) — fused into tc_dot_launch.
cudaError_t tc_dot_launch(const TcDotDesc& d, cudaStream_t stream);

}  // namespace nengb
