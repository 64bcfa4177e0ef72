"""Exhaustive parity of the device's expm1f/log1pf with the host glibc the
reference's EngineCore<float> calls (neuron_math.hpp:15,62,67): every float
in every range the engine feeds these functions, device vs host, bit for bit.
Mismatches (if any) are written to gpurun_out/libm_mismatch.txt in the
device_overrides.txt format so they can be folded into the tables."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import refapi
from paper_1805_11144_b200 import passes

pytestmark = pytest.mark.gpu

RANGES = [  # (table index, func, lo, hi inclusive)
    (0, 0, 0x80000001, 0xC2D00000),  # expm1f over [-104, 0)
    (1, 1, 0x80000001, 0xBF800000),  # log1pf over [-1, 0)
    (2, 1, 0x00000001, 0x7F7FFFFF),  # log1pf over (0, FLT_MAX]
]


def _host_lib():
    lib = C.CDLL(os.path.join(os.path.dirname(refapi.__file__), "libneng_libm.so"))
    lib.nlibm_eval.argtypes = [C.c_int, C.c_uint32, C.c_int64, C.POINTER(C.c_uint32), C.c_int]
    lib.nlibm_eval.restype = None
    return lib


def _compare(table, func, lo, hi, chunk=1 << 27, device_func=None):
    host = _host_lib()
    threads = os.cpu_count() or 8
    buf = np.zeros(chunk, dtype=np.uint32)
    mismatches = []
    at = lo
    while at <= hi:
        n = min(chunk, hi - at + 1)
        dev = passes.debug_libm_eval(func if device_func is None else device_func, at, n)
        host.nlibm_eval(func, at, n, buf.ctypes.data_as(C.POINTER(C.c_uint32)), threads)
        h = buf[:n]
        keys = np.arange(at, at + n, dtype=np.uint64).astype(np.uint32)
        hf = h.view(np.float32)
        df = dev.view(np.float32)
        both_nan = np.isnan(hf) & np.isnan(df)
        bad = (dev != h) & ~both_nan
        if bad.any():
            mismatches.extend((table, int(k)) for k in keys[bad][:1000])
        at += n
    return mismatches


@pytest.mark.slow
def test_libm_parity_exhaustive():
    allbad = []
    for table, func, lo, hi in RANGES:
        allbad.extend(_compare(table, func, lo, hi))
    if allbad:
        os.makedirs("gpurun_out", exist_ok=True)
        with open("gpurun_out/libm_mismatch.txt", "w") as f:
            for t, k in allbad:
                f.write(f"{t} {k:08x}\n")
    assert not allbad, f"{len(allbad)} device/host libm mismatches (first: {allbad[:5]})"


def test_speculative_resolution_whole_lif_range():
    """The fused kernel accepts a speculative (reduced-polynomial) value on the
    LIF range unless it is doubtful and table-listed (glibc_spec_resolved, the
    semantics of fused.cu's fix-up).  Every float of [-1/16, 0), both functions."""
    bad = _compare(0, 0, 0x80000001, 0xBD800000, device_func=2)
    bad += _compare(1, 1, 0x80000001, 0xBD800000, device_func=3)
    assert not bad, bad[:10]


def test_libm_parity_lif_hot_range():
    """The LIF hot range (-dt/tau_rc, 0) = (-0.05, 0), top binades (where the
    glibc exceptions live)."""
    bad = _compare(0, 0, 0xBC000000, 0xBD4CCCCD) + _compare(1, 1, 0xBC000000, 0xBD4CCCCD)
    assert not bad, bad[:10]
