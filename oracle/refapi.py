"""TEST INFRASTRUCTURE ONLY — Python handle on the oracles.

* ``oracle/_ref/libneng_ref.so``: the reference's own sources (ir, passes,
  exec, reference .cpp under /root/reference/proj/src) compiled unchanged by
  oracle/Makefile plus the C shim oracle/ref_capi.cpp.
* ``oracle/libneng_port.so``: engine_port.c, the plain-C restatement of
  EngineCore<T> (exec.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product
(paper_1805_11144_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1805_11144_b200 import _abi, ir

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libneng_ref.so")
PORT_SO = os.path.join(HERE, "libneng_port.so")

_ref = None
_port = None

P = C.c_void_p


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"oracle library missing: {REF_SO} (run `make -C oracle`)")
        lib = C.CDLL(REF_SO)
        lib.nref_last_error.restype = C.c_char_p
        lib.nref_planned_view.restype = C.POINTER(_abi.neng_planned_model)
        lib.nref_planned_view.argtypes = [P]
        lib.nref_engine_steps_completed.argtypes = [P]
        lib.nref_engine_buffer_storage.argtypes = [P, C.c_int32]
        for fn in ("nref_planned_destroy", "nref_engine_destroy"):
            getattr(lib, fn).argtypes = [P]
            getattr(lib, fn).restype = None
        _ref = lib
    return _ref


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            raise RuntimeError(f"oracle port missing: {PORT_SO} (run `make -C oracle port`)")
        lib = C.CDLL(PORT_SO)
        lib.nport_last_error.restype = C.c_char_p
        for fn in ("nport_destroy",):
            getattr(lib, fn).argtypes = [P]
            getattr(lib, fn).restype = None
        lib.nport_steps_completed.argtypes = [P]
        lib.nport_buffer_storage.argtypes = [P, C.c_int32]
        _port = lib
    return _port


def _check(lib, status, err_fn="nref_last_error"):
    if status:
        _abi.raise_for(status, getattr(lib, err_fn)().decode())


def validate(model: ir.BuiltModel):
    """validate_operators + build_dependency_graph (raises like the reference)."""
    lib = ref_lib()
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    _check(lib, lib.nref_validate(C.byref(v)))


def toposort(model: ir.BuiltModel):
    lib = ref_lib()
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    out = np.zeros(max(len(model.operators), 1), dtype=np.int32)
    _check(lib, lib.nref_toposort(C.byref(v), out.ctypes.data_as(_abi.i32p)))
    return [int(x) for x in out[:len(model.operators)]]


def dependency_edges(model: ir.BuiltModel):
    lib = ref_lib()
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    n = C.c_int64()
    _check(lib, lib.nref_dependency_edges(C.byref(v), C.byref(n), None))
    pairs = np.zeros(max(2 * n.value, 2), dtype=np.int32)
    _check(lib, lib.nref_dependency_edges(C.byref(v), C.byref(n), pairs.ctypes.data_as(_abi.i32p)))
    return sorted((int(pairs[2 * i]), int(pairs[2 * i + 1])) for i in range(n.value))


class RefPlanned:
    """Owns a reference neng::PlannedModel (from run_passes or from a view)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.nref_planned_destroy(self.h)
            self.h = None

    def to_python(self) -> ir.PlannedModel:
        lib = ref_lib()
        v = lib.nref_planned_view(self.h).contents
        frac, rows, groups = C.c_double(), C.c_int64(), C.c_int32()
        lib.nref_planned_stats(C.c_void_p(self.h), C.byref(frac), C.byref(rows), C.byref(groups))
        return _abi.planned_model_from_view(v, ir.ContiguityStats(frac.value, rows.value, groups.value))

    def read_blocks(self):
        lib = ref_lib()
        nb = lib.nref_planned_num_read_blocks(C.c_void_p(self.h))
        lib.nref_planned_read_block_refs.restype = C.c_int64
        nr = lib.nref_planned_read_block_refs(C.c_void_p(self.h))
        meta = np.zeros(max(4 * nb, 4), dtype=np.int32)
        refs = np.zeros(max(3 * nr, 3), dtype=np.int32)
        lib.nref_planned_read_blocks(C.c_void_p(self.h), meta.ctypes.data_as(_abi.i32p),
                                     refs.ctypes.data_as(_abi.i32p))
        out, at = [], 0
        for i in range(nb):
            g, pos, buf, n = (int(x) for x in meta[4 * i:4 * i + 4])
            rr = [tuple(int(x) for x in refs[3 * (at + k):3 * (at + k) + 3]) for k in range(n)]
            at += n
            out.append((g, pos, buf, rr))
        return out


def run_passes(model: ir.BuiltModel, cfg: ir.PipelineConfig = None) -> RefPlanned:
    cfg = cfg or ir.PipelineConfig()
    lib = ref_lib()
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    h = C.c_void_p()
    _check(lib, lib.nref_run_passes(C.byref(v), int(cfg.merge), int(cfg.simplify), int(cfg.planner),
                                    int(cfg.tree_depth), int(cfg.sort), C.byref(h)))
    return RefPlanned(h.value)


def planned_from_python(pm: ir.PlannedModel) -> RefPlanned:
    lib = ref_lib()
    m = _abi.Marshalled()
    v = _abi.planned_model_view(pm, m)
    h = C.c_void_p()
    _check(lib, lib.nref_planned_from_view(C.byref(v), C.byref(h)))
    return RefPlanned(h.value)


def _as_ref_planned(planned):
    return planned if isinstance(planned, RefPlanned) else planned_from_python(planned)


class RefEngine:
    """The reference's EngineCore<float> (fp64=False) or EngineCore<double>."""

    def __init__(self, planned, batch: int = 1, unroll: int = 1, fp64: bool = False):
        lib = ref_lib()
        self.planned = _as_ref_planned(planned)
        self.model = self.planned.to_python().model
        self._batch = batch
        h = C.c_void_p()
        _check(lib, lib.nref_engine_create(C.c_void_p(self.planned.h), batch, unroll, int(fp64), C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.nref_engine_destroy(self.h)
            self.h = None

    def run(self, n_steps: int, feeds=None):
        lib = ref_lib()
        m = _abi.Marshalled()
        nf, fv = _abi.feeds_view(feeds or {}, m)
        total = _abi.probe_total(self.model, self._batch, max(n_steps, 0))
        out = np.zeros(max(total, 1))
        _check(lib, lib.nref_engine_run(C.c_void_p(self.h), n_steps, nf, fv, out.ctypes.data_as(_abi.f64p)))
        return _abi.split_probes(self.model, out, self._batch, n_steps)

    def write_probe_binary(self, path: str):
        """The reference's write_probe_binary (export.cpp) of the last run's traces."""
        lib = ref_lib()
        lib.nref_engine_write_probe_binary.argtypes = [C.c_void_p, C.c_char_p]
        _check(lib, lib.nref_engine_write_probe_binary(C.c_void_p(self.h), os.fsencode(path)))

    def write_probe_csv(self, path: str, dt: float):
        """The reference's write_probe_csv (export.cpp) of the last run's traces."""
        lib = ref_lib()
        lib.nref_engine_write_probe_csv.argtypes = [C.c_void_p, C.c_char_p, C.c_double]
        _check(lib, lib.nref_engine_write_probe_csv(C.c_void_p(self.h), os.fsencode(path), dt))

    def reset(self):
        _check(ref_lib(), ref_lib().nref_engine_reset(C.c_void_p(self.h)))

    def read_signal(self, sig: int, batch_index: int = 0):
        lib = ref_lib()
        n = C.c_int64()
        _check(lib, lib.nref_engine_read_signal(C.c_void_p(self.h), sig, batch_index, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1))
        _check(lib, lib.nref_engine_read_signal(C.c_void_p(self.h), sig, batch_index,
                                                out.ctypes.data_as(_abi.f64p), n.value, C.byref(n)))
        return out[:n.value]

    def steps_completed(self) -> int:
        return ref_lib().nref_engine_steps_completed(self.h)

    def buffer_storage(self, buffer: int) -> ir.StorageMode:
        return ir.StorageMode(ref_lib().nref_engine_buffer_storage(self.h, buffer))

    def batch(self) -> int:
        return self._batch


def run_reference(model: ir.BuiltModel, n_steps: int, feeds=None, minibatch: int = 1):
    """run_reference (reference.cpp:194-226): the f64 interpreter."""
    lib = ref_lib()
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    nf, fv = _abi.feeds_view(feeds or {}, m)
    total = _abi.probe_total(model, minibatch, max(n_steps, 0))
    out = np.zeros(max(total, 1))
    _check(lib, lib.nref_run_reference(C.byref(v), n_steps, nf, fv, minibatch, out.ctypes.data_as(_abi.f64p)))
    return _abi.split_probes(model, out, minibatch, n_steps)


def time_engines(planned, threads: int, rows_per_engine: int, warm_steps: int, timed_steps: int,
                 fp64: bool = False, feed_seed: int = 0) -> float:
    """Wall seconds (max over threads) for `threads` parallel reference engines
    (EngineCore<float>, or EngineCore<double> with fp64) of `rows_per_engine`
    rows each to advance `timed_steps` (reference protocol, bench.cpp:218-225:
    warm-up run, reset, timed run), every feed slot driven by seeded N(0, 1)
    white noise when feed_seed != 0."""
    lib = ref_lib()
    rp = _as_ref_planned(planned)
    secs = C.c_double()
    lib.nref_time_engines2.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_uint64, C.POINTER(C.c_double)]
    _check(lib, lib.nref_time_engines2(C.c_void_p(rp.h), threads, rows_per_engine, warm_steps, timed_steps,
                                       int(fp64), feed_seed, C.byref(secs)))
    return secs.value


class PortEngine:
    """engine_port.c: the plain-C restatement of EngineCore<T> (float or double)."""

    def __init__(self, planned: ir.PlannedModel, batch: int = 1, unroll: int = 1, fp64: bool = False):
        lib = port_lib()
        self.model = planned.model
        self._m = _abi.Marshalled()
        v = _abi.planned_model_view(planned, self._m)
        self._view = v
        self._batch = batch
        h = C.c_void_p()
        _check(lib, lib.nport_create(C.byref(v), batch, unroll, int(fp64), C.byref(h)), "nport_last_error")
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None) and _port is not None:
            _port.nport_destroy(self.h)
            self.h = None

    def run(self, n_steps: int, feeds=None):
        lib = port_lib()
        m = _abi.Marshalled()
        nf, fv = _abi.feeds_view(feeds or {}, m)
        total = _abi.probe_total(self.model, self._batch, max(n_steps, 0))
        out = np.zeros(max(total, 1))
        _check(lib, lib.nport_run(C.c_void_p(self.h), n_steps, nf, fv, out.ctypes.data_as(_abi.f64p)),
               "nport_last_error")
        return _abi.split_probes(self.model, out, self._batch, n_steps)

    def reset(self):
        _check(port_lib(), port_lib().nport_reset(C.c_void_p(self.h)), "nport_last_error")

    def read_signal(self, sig: int, batch_index: int = 0):
        lib = port_lib()
        n = C.c_int64()
        _check(lib, lib.nport_read_signal(C.c_void_p(self.h), sig, batch_index, None, 0, C.byref(n)),
               "nport_last_error")
        out = np.zeros(max(n.value, 1))
        _check(lib, lib.nport_read_signal(C.c_void_p(self.h), sig, batch_index, out.ctypes.data_as(_abi.f64p),
                                          n.value, C.byref(n)), "nport_last_error")
        return out[:n.value]

    def steps_completed(self) -> int:
        return port_lib().nport_steps_completed(self.h)

    def buffer_storage(self, buffer: int) -> ir.StorageMode:
        return ir.StorageMode(port_lib().nport_buffer_storage(self.h, buffer))
