"""The tcgen05 tensor-core DotInc (csrc/kernels/tc_dot.cu) against an fp64
reference of the same Y += A.X (exec.cpp:226-240), through the C ABI entry
neng_gpu_tc_dot.

Stated tolerances (per output element, S = sum_k |A[m,k] X[k,n]|):
  TF32   : |Y - Y_ref| <= 2^-8 S   (operands rounded to a 10-bit mantissa: <= 2^-10
                                    relative each, so <= ~2^-9 per product)
  BF16X3 : |Y - Y_ref| <= 2^-14 S  (hi + lo bf16 split: operand residual <= 2^-17,
                                    the dropped lo.lo term <= 2^-18 per product)
both plus the fp32 accumulation term k 2^-23 S."""
import numpy as np
import pytest

from paper_1805_11144_b200.engine import PRECISION_BF16X3, PRECISION_TF32, tc_dot

SHAPES = [
    (1024, 784, 512),  # config 3, layer 1 (K not a multiple of the 32-wide k stage)
    (1024, 1024, 512),  # config 3, layer 2
    (10, 1024, 512),  # config 3, output layer (one partial 128-row tile)
    (130, 40, 96),  # row, k and column tails
    (256, 32, 32),
]
BOUND = {PRECISION_TF32: 2.0 ** -8, PRECISION_BF16X3: 2.0 ** -14}


def _case(m, k, n, seed):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-0.1, 0.1, size=(m, k)).astype(np.float32)
    x = rng.uniform(0.0, 1.0, size=(k, n)).astype(np.float32)
    x[rng.random(size=x.shape) < 0.7] = 0.0  # spike-like sparsity
    x[x > 0.5] = 10.0  # amplitude / dt
    y0 = rng.normal(size=(m, n)).astype(np.float32)
    return a, x, y0


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [PRECISION_TF32, PRECISION_BF16X3], ids=["tf32", "bf16x3"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_tc_dot_within_stated_tolerance(shape, precision):
    m, k, n = shape
    a, x, y0 = _case(m, k, n, seed=m * 7 + k + n)
    got, ms = tc_dot(a, x, y0, precision, reps=20)
    a64, x64 = a.astype(np.float64), x.astype(np.float64)
    want = y0.astype(np.float64) + a64 @ x64
    scale = np.abs(a64) @ np.abs(x64)
    err = np.abs(got.astype(np.float64) - want)
    bound = (BOUND[precision] + k * 2.0 ** -23) * scale + 2.0 ** -23 * np.abs(want)
    worst = float((err / np.maximum(bound, 1e-30)).max())
    flops = 2.0 * m * k * n
    print(f"\n{shape} {'tf32' if precision == PRECISION_TF32 else 'bf16x3'}: {ms * 1e3:.1f} us, "
          f"{flops / (ms * 1e-3) / 1e12:.1f} TFLOP/s, max err / bound {worst:.3f}, "
          f"max rel err {float((err / np.maximum(scale, 1e-30)).max()):.2e}")
    assert worst <= 1.0


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [PRECISION_TF32, PRECISION_BF16X3], ids=["tf32", "bf16x3"])
def test_tc_dot_deterministic_and_exact_on_representable_operands(precision):
    # operands exactly representable in bf16 (and so in TF32), small integers: every
    # product and partial sum is exact in fp32, so the result must equal the fp64 one
    rng = np.random.default_rng(5)
    m, k, n = 256, 128, 64
    a = rng.integers(-8, 9, size=(m, k)).astype(np.float32)
    x = rng.integers(0, 4, size=(k, n)).astype(np.float32)
    y0 = rng.integers(-100, 100, size=(m, n)).astype(np.float32)
    got1, _ = tc_dot(a, x, y0, precision)
    got2, _ = tc_dot(a, x, y0, precision)
    want = (y0.astype(np.float64) + a.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
    assert np.array_equal(got1, want)
    assert np.array_equal(got1.view(np.uint32), got2.view(np.uint32))


@pytest.mark.gpu
def test_tc_dot_rejects_misaligned_rows():
    a = np.zeros((16, 34), np.float32)  # K = 34: rows of A are not 16-byte multiples
    x = np.zeros((34, 32), np.float32)
    with pytest.raises(RuntimeError, match="aligned"):
        tc_dot(a, x, np.zeros((16, 32), np.float32))
