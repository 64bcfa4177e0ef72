"""Model tooling through the native library (include/neng_host.h):
run_passes (the reference's passes.cpp:663-694, restated in C++ with
plan-identical output), structural validation, dependency edges, toposort."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi, ir
from .engine import lib as _lib

_configured = False


def lib():
    global _configured
    L = _lib()
    if not _configured:
        P = C.c_void_p
        L.neng_host_last_error.restype = C.c_char_p
        L.neng_run_passes.argtypes = [C.POINTER(_abi.neng_built_model), C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, C.POINTER(P)]
        L.neng_plan_view.argtypes = [P]
        L.neng_plan_view.restype = C.POINTER(_abi.neng_planned_model)
        L.neng_plan_stats.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.neng_plan_destroy.argtypes = [P]
        L.neng_plan_destroy.restype = None
        L.neng_model_validate.argtypes = [C.POINTER(_abi.neng_built_model)]
        L.neng_model_toposort.argtypes = [C.POINTER(_abi.neng_built_model), C.POINTER(C.c_int32)]
        L.neng_model_dependency_edges.argtypes = [C.POINTER(_abi.neng_built_model), C.POINTER(C.c_int64),
                                                  C.POINTER(C.c_int32)]
        L.neng_debug_libm_eval.argtypes = [C.c_int32, C.c_int32, C.c_uint32, C.c_int64, C.POINTER(C.c_uint32)]
        L.neng_solve_decoders.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                          C.c_int32, C.c_double, C.POINTER(C.c_double)]
        _configured = True
    return L


def _check(st):
    if st:
        _abi.raise_for(st, lib().neng_host_last_error().decode())


def run_passes(model: ir.BuiltModel, cfg: ir.PipelineConfig = None) -> ir.PlannedModel:
    cfg = cfg or ir.PipelineConfig()
    L = lib()
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    h = C.c_void_p()
    _check(L.neng_run_passes(C.byref(v), int(cfg.merge), int(cfg.simplify), int(cfg.planner), int(cfg.tree_depth),
                             int(cfg.sort), C.byref(h)))
    try:
        view = L.neng_plan_view(h).contents
        frac, rows, groups = C.c_double(), C.c_int64(), C.c_int32()
        L.neng_plan_stats(h, C.byref(frac), C.byref(rows), C.byref(groups))
        return _abi.planned_model_from_view(view, ir.ContiguityStats(frac.value, rows.value, groups.value))
    finally:
        L.neng_plan_destroy(h)


def validate(model: ir.BuiltModel):
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    _check(lib().neng_model_validate(C.byref(v)))


def toposort(model: ir.BuiltModel):
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    out = np.zeros(max(len(model.operators), 1), dtype=np.int32)
    _check(lib().neng_model_toposort(C.byref(v), out.ctypes.data_as(_abi.i32p)))
    return [int(x) for x in out[:len(model.operators)]]


def dependency_edges(model: ir.BuiltModel):
    m = _abi.Marshalled()
    v = _abi.built_model_view(model, m)
    n = C.c_int64()
    _check(lib().neng_model_dependency_edges(C.byref(v), C.byref(n), None))
    pairs = np.zeros(max(2 * n.value, 2), dtype=np.int32)
    _check(lib().neng_model_dependency_edges(C.byref(v), C.byref(n), pairs.ctypes.data_as(_abi.i32p)))
    return sorted((int(pairs[2 * i]), int(pairs[2 * i + 1])) for i in range(n.value))


def debug_libm_eval(func: int, lo: int, n: int, device: int = 0) -> np.ndarray:
    out = np.zeros(max(n, 1), dtype=np.uint32)
    _check(lib().neng_debug_libm_eval(device, func, lo, n, out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out[:n]


def solve_decoders(activities: np.ndarray, targets: np.ndarray, reg: float = 0.1) -> np.ndarray:
    """solve_decoders (frontend.cpp:56-76), native and Eigen-free: the
    regularised least-squares decoders D [n][d] with
    (A^T A + m sigma^2 I) D = A^T Y, sigma = reg * max|A|, for activities
    A [m][n] and targets Y [m][d] (a 1-D Y is one target column)."""
    a = np.ascontiguousarray(activities, dtype=np.float64)
    y = np.ascontiguousarray(targets, dtype=np.float64)
    if y.ndim == 1:
        y = y[:, None]
    if a.ndim != 2 or y.ndim != 2 or a.shape[0] != y.shape[0]:
        raise ValueError("solve_decoders: activities [m][n] and targets [m][d] expected")
    m, n = a.shape
    d = y.shape[1]
    out = np.zeros((n, d))
    f64 = C.POINTER(C.c_double)
    _check(lib().neng_solve_decoders(a.ctypes.data_as(f64), m, n, y.ctypes.data_as(f64), d, float(reg),
                                     out.ctypes.data_as(f64)))
    return out
