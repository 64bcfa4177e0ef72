"""GpuEngine — Python face of the B200 executor (libneng_gpu.so, C ABI in
include/neng_gpu.h).  Same surface as the reference's neng::EngineCore<float>
(proj/include/nengine/exec.hpp:18-120): construct from a PlannedModel with a
batch size and unroll factor, then run / reset / read_signal / buffer_storage /
steps_completed.  There is no CPU path: if the native library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import _abi, ir

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libneng_gpu.so")

MODE_AUTO, MODE_GENERIC, MODE_FUSED = 0, 1, 2
PRECISION_STRICT_FP32, PRECISION_TF32, PRECISION_BF16X3 = 0, 1, 2
STEP_FIRST_UPDATE, STEP_EPILOGUE = 1, 2
SCHED_GENERIC, SCHED_FUSED_STEPPED, SCHED_BARRIER_FREE, SCHED_FUSED_SMALL = 1, 2, 4, 8  # neng_gpu_last_schedule bits

_lib = None


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"native library missing: {LIB_PATH} — run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.neng_gpu_create.argtypes = [C.POINTER(_abi.neng_planned_model), C.c_int32, C.c_int32,
                                      C.POINTER(_abi.neng_device_cfg), C.POINTER(P)]
        L.neng_gpu_destroy.argtypes = [P]
        L.neng_gpu_destroy.restype = None
        L.neng_gpu_run.argtypes = [P, C.c_int32, C.c_int32, C.POINTER(_abi.neng_feed), C.POINTER(C.c_double)]
        L.neng_gpu_run_device.argtypes = [P, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), P]
        L.neng_gpu_synchronize.argtypes = [P]
        L.neng_gpu_call_begin.argtypes = [P, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), P]
        L.neng_gpu_call_step.argtypes = [P, C.c_int32, C.c_int32]
        L.neng_gpu_call_end.argtypes = [P]
        L.neng_gpu_shard_layout.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_void_p)]
        L.neng_gpu_set_xhat_buffer.argtypes = [P, P]
        L.neng_gpu_reset.argtypes = [P]
        L.neng_gpu_read_signal.argtypes = [P, C.c_int32, C.c_int32, C.POINTER(C.c_double), C.c_int64,
                                           C.POINTER(C.c_int64)]
        L.neng_gpu_buffer_storage.argtypes = [P, C.c_int32, C.POINTER(C.c_int32)]
        L.neng_gpu_probe_dump_size.argtypes = [P, C.POINTER(C.c_int64)]
        L.neng_gpu_probe_dump.argtypes = [P, C.c_void_p, C.c_int64]
        L.neng_gpu_write_probe_binary.argtypes = [P, C.c_char_p]
        L.neng_gpu_write_probe_csv.argtypes = [P, C.c_char_p, C.c_double]
        for fn in ("neng_gpu_batch", "neng_gpu_unroll", "neng_gpu_steps_completed", "neng_gpu_num_probes",
                   "neng_gpu_mode"):
            getattr(L, fn).argtypes = [P]
            getattr(L, fn).restype = C.c_int32
        L.neng_gpu_last_schedule.argtypes = [P]
        L.neng_gpu_last_schedule.restype = C.c_int32
        L.neng_gpu_last_launch_count.argtypes = [P]
        L.neng_gpu_last_launch_count.restype = C.c_int64
        L.neng_gpu_last_error.argtypes = [P]
        L.neng_gpu_last_error.restype = C.c_char_p
        L.neng_last_error.restype = C.c_char_p
        f32p = C.POINTER(C.c_float)
        L.neng_gpu_tc_dot.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, f32p, f32p, f32p, C.c_int32,
                                      C.POINTER(C.c_double)]
        _lib = L
    return _lib


class GpuEngine:
    """Drop-in for EngineCore<float> on a B200.

    ``mode``: MODE_AUTO picks the fused ensemble pipeline when the model is an
    ensemble network it reproduces exactly, else the generic persistent
    interpreter; MODE_GENERIC / MODE_FUSED force one (MODE_FUSED raises
    BuildError if impossible).
    """

    def __init__(self, planned: ir.PlannedModel, batch: int = 1, unroll: int = 1, *, device: int = 0,
                 mode: int = MODE_AUTO, steps_per_launch: int = 0, shard: Optional[tuple] = None,
                 precision: int = PRECISION_STRICT_FP32):
        L = lib()
        self._planned = planned
        self.model = planned.model
        m = _abi.Marshalled()
        view = _abi.planned_model_view(planned, m)
        cfg = _abi.neng_device_cfg()
        cfg.device, cfg.mode, cfg.steps_per_launch = device, mode, steps_per_launch
        cfg.precision = precision  # PRECISION_TF32: dense DotInc on tensor cores (stated tolerance)
        if shard is not None:  # (rank, count): ensemble sharding, see paper_1805_11144_b200.shard
            cfg.shard_rank, cfg.shard_count = int(shard[0]), int(shard[1])
        h = C.c_void_p()
        st = L.neng_gpu_create(C.byref(view), batch, unroll, C.byref(cfg), C.byref(h))
        if st:
            _abi.raise_for(st, L.neng_last_error().decode())
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.neng_gpu_destroy(h)
            self._h = None

    def _check(self, st):
        if st:
            _abi.raise_for(st, lib().neng_gpu_last_error(self._h).decode())

    # -- EngineCore surface --------------------------------------------------
    def run(self, n_steps: int, feeds: Optional[ir.FeedData] = None) -> ir.ProbeOutput:
        m = _abi.Marshalled()
        nf, fv = _abi.feeds_view(feeds or {}, m)
        total = _abi.probe_total(self.model, self.batch(), max(n_steps, 0))
        out = np.zeros(max(total, 1))
        self._check(lib().neng_gpu_run(self._h, n_steps, nf, fv, out.ctypes.data_as(_abi.f64p)))
        return _abi.split_probes(self.model, out, self.batch(), n_steps)

    def run_device(self, n_steps: int, feed_ptrs, probe_ptrs, stream: int = 0):
        """Device-resident step loop: feed_ptrs / probe_ptrs are lists of raw
        device pointers (ints or None), one per feed slot / probe."""
        nfs = len(self.model.feed_slots)
        fp = (C.c_void_p * max(nfs, 1))(*[C.c_void_p(p) if p else None for p in (feed_ptrs or [None] * nfs)])
        npb = len(self.model.probes)
        pp = (C.c_void_p * max(npb, 1))(*[C.c_void_p(p) if p else None for p in (probe_ptrs or [None] * npb)])
        self._check(lib().neng_gpu_run_device(self._h, n_steps, fp, pp, C.c_void_p(stream) if stream else None))

    # -- stepped calls (ensemble sharding) -------------------------------------
    def _ptrs(self, ptrs, n):
        return (C.c_void_p * max(n, 1))(*[C.c_void_p(q) if q else None for q in (ptrs or [None] * n)])

    def call_begin(self, n_steps: int, feed_ptrs, probe_ptrs, stream: int = 0):
        fp = self._ptrs(feed_ptrs, len(self.model.feed_slots))
        pp = self._ptrs(probe_ptrs, len(self.model.probes))
        self._check(lib().neng_gpu_call_begin(self._h, n_steps, fp, pp, C.c_void_p(stream) if stream else None))

    def call_step(self, k: int, flags: int = 0):
        self._check(lib().neng_gpu_call_step(self._h, k, flags))

    def call_end(self):
        self._check(lib().neng_gpu_call_end(self._h))

    def shard_layout(self):
        """(xbuf_floats, rank_floats, device pointer of the xhat parity buffers)."""
        a, b, q = C.c_int64(), C.c_int64(), C.c_void_p()
        self._check(lib().neng_gpu_shard_layout(self._h, C.byref(a), C.byref(b), C.byref(q)))
        return a.value, b.value, q.value

    def set_xhat_buffer(self, ptr: int):
        self._check(lib().neng_gpu_set_xhat_buffer(self._h, C.c_void_p(ptr)))

    def synchronize(self):
        self._check(lib().neng_gpu_synchronize(self._h))

    def reset(self):
        self._check(lib().neng_gpu_reset(self._h))

    def read_signal(self, sig: int, batch_index: int = 0) -> np.ndarray:
        n = C.c_int64()
        self._check(lib().neng_gpu_read_signal(self._h, sig, batch_index, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1))
        self._check(lib().neng_gpu_read_signal(self._h, sig, batch_index, out.ctypes.data_as(_abi.f64p), n.value,
                                               C.byref(n)))
        return out[:n.value]

    # -- probe export (export.hpp:17-25) of the last run ----------------------
    def probe_dump(self) -> bytes:
        """NENG1 bytes of the last run's traces (write_probe_binary)."""
        n = C.c_int64()
        self._check(lib().neng_gpu_probe_dump_size(self._h, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        self._check(lib().neng_gpu_probe_dump(self._h, buf, n.value))
        return buf.raw[:n.value]

    def write_probe_binary(self, path: str):
        self._check(lib().neng_gpu_write_probe_binary(self._h, os.fsencode(path)))

    def write_probe_csv(self, path: str, dt: float):
        self._check(lib().neng_gpu_write_probe_csv(self._h, os.fsencode(path), float(dt)))

    def buffer_storage(self, buffer: int) -> ir.StorageMode:
        mode = C.c_int32()
        self._check(lib().neng_gpu_buffer_storage(self._h, buffer, C.byref(mode)))
        return ir.StorageMode(mode.value)

    def batch(self) -> int:
        return lib().neng_gpu_batch(self._h)

    def unroll(self) -> int:
        return lib().neng_gpu_unroll(self._h)

    def steps_completed(self) -> int:
        return lib().neng_gpu_steps_completed(self._h)

    def planned(self) -> ir.PlannedModel:
        return self._planned

    # -- extras ---------------------------------------------------------------
    def mode(self) -> int:
        return lib().neng_gpu_mode(self._h)

    def last_launch_count(self) -> int:
        return lib().neng_gpu_last_launch_count(self._h)

    def last_schedule(self) -> int:
        """NENG_SCHED_* bits of the most recent call (SCHED_BARRIER_FREE: the bench's kernel)."""
        return lib().neng_gpu_last_schedule(self._h)


def tc_dot(a, x, y, precision: int = PRECISION_TF32, reps: int = 1):
    """Y + A.X on the tcgen05 tensor-core DotInc (the TF32 / BF16X3 path of dense
    DotInc groups) for host float32 arrays A [m][k], X [k][n], Y [m][n].
    Returns (result, mean ms per launch)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.array(y, dtype=np.float32, order="C", copy=True)
    m, k = a.shape
    k2, n = x.shape
    if k2 != k or out.shape != (m, n):
        raise ValueError("tc_dot: shape mismatch")
    ms = C.c_double(0.0)
    f32p = C.POINTER(C.c_float)
    st = lib().neng_gpu_tc_dot(precision, m, k, n, a.ctypes.data_as(f32p), x.ctypes.data_as(f32p),
                               out.ctypes.data_as(f32p), reps, C.byref(ms))
    if st != 0:
        raise RuntimeError(lib().neng_last_error().decode())
    return out, ms.value
