"""ctypes view of include/neng_gpu.h and marshalling of the Python IR mirror
into it.  Shared by the product bindings (engine.py, passes.py) and, as test
infrastructure, by oracle/refapi.py — both libraries take the same POD views.
"""
from __future__ import annotations

import ctypes as C
from typing import List

import numpy as np

from . import ir

i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class neng_signal(C.Structure):
    _fields_ = [("id", C.c_int32), ("ndim", C.c_int32), ("shape", i32p), ("elem", C.c_int32),
                ("n_initial", C.c_int64), ("initial", f64p), ("constant", C.c_int32),
                ("minibatched", C.c_int32), ("trainable", C.c_int32), ("label", C.c_char_p)]


class neng_ref(C.Structure):
    _fields_ = [("signal", C.c_int32), ("start", C.c_int32), ("stop", C.c_int32)]


class neng_operator(C.Structure):
    _fields_ = [("id", C.c_int32), ("kind", C.c_int32), ("n_operands", C.c_int32),
                ("operands", C.POINTER(neng_ref)), ("n_value", C.c_int64), ("value", f64p),
                ("inc", C.c_int32), ("neuron_kind", C.c_int32), ("tau_rc", C.c_double),
                ("tau_ref", C.c_double), ("amplitude", C.c_double), ("tau", C.c_double),
                ("learning_rate", C.c_double), ("dt", C.c_double)]


class neng_probe(C.Structure):
    _fields_ = [("key", C.c_int32), ("signal", C.c_int32), ("label", C.c_char_p)]


class neng_feed_slot(C.Structure):
    _fields_ = [("node_id", C.c_int32), ("signal", C.c_int32), ("dim", C.c_int32),
                ("has_default", C.c_int32), ("label", C.c_char_p)]


class neng_built_model(C.Structure):
    _fields_ = [("n_signals", C.c_int32), ("signals", C.POINTER(neng_signal)),
                ("n_operators", C.c_int32), ("operators", C.POINTER(neng_operator)),
                ("n_probes", C.c_int32), ("probes", C.POINTER(neng_probe)),
                ("n_feed_slots", C.c_int32), ("feed_slots", C.POINTER(neng_feed_slot)),
                ("dt", C.c_double)]


class neng_buffer_desc(C.Structure):
    _fields_ = [("n_trailing", C.c_int32), ("trailing", i32p), ("elem", C.c_int32),
                ("minibatched", C.c_int32), ("trainable", C.c_int32), ("rows", C.c_int32),
                ("n_order", C.c_int32), ("order", i32p)]


class neng_planned_model(C.Structure):
    _fields_ = [("model", neng_built_model), ("n_groups", C.c_int32), ("group_offsets", i32p),
                ("group_members", i32p), ("buffer_of", i32p), ("row_offset", i32p),
                ("n_buffers", C.c_int32), ("buffers", C.POINTER(neng_buffer_desc))]


class neng_feed(C.Structure):
    _fields_ = [("node_id", C.c_int32), ("batch", C.c_int32), ("steps", C.c_int32),
                ("dim", C.c_int32), ("data", f64p)]


class neng_device_cfg(C.Structure):
    _fields_ = [("device", C.c_int32), ("mode", C.c_int32), ("steps_per_launch", C.c_int32),
                ("shard_rank", C.c_int32), ("shard_count", C.c_int32), ("precision", C.c_int32),
                ("reserved", C.c_int32 * 2)]


STATUS_EXC = {1: ir.StructuralError, 2: ir.BuildError, 3: ir.RunError, 4: ir.CudaError,
              5: MemoryError, 6: ValueError}


def raise_for(status: int, msg: str):
    if status:
        raise STATUS_EXC.get(status, RuntimeError)(msg)


def _i32(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int32))


def _f64(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.float64))


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class Marshalled:
    """Holds a C view plus every buffer it points into (keep it alive while
    the view is in use)."""

    def __init__(self):
        self.keep: List[object] = []

    def hold(self, x):
        self.keep.append(x)
        return x


def built_model_view(model: ir.BuiltModel, m: Marshalled) -> neng_built_model:
    ns = len(model.signals)
    sigs = m.hold((neng_signal * max(ns, 1))())
    for i, s in enumerate(model.signals):
        shape = m.hold(_i32(s.shape))
        d = sigs[i]
        d.id = s.id
        d.ndim = len(s.shape)
        d.shape = _ptr(shape, i32p)
        d.elem = int(s.elem)
        if s.initial is not None and len(s.initial):
            init = m.hold(_f64(s.initial))
            d.n_initial = init.size
            d.initial = _ptr(init, f64p)
        d.constant = int(s.constant)
        d.minibatched = int(s.minibatched)
        d.trainable = int(s.trainable)
        d.label = m.hold(s.label.encode())
    no = len(model.operators)
    ops = m.hold((neng_operator * max(no, 1))())
    for i, o in enumerate(model.operators):
        refs = m.hold((neng_ref * max(len(o.operands), 1))())
        for k, r in enumerate(o.operands):
            refs[k].signal, refs[k].start, refs[k].stop = r.signal, r.start, r.stop
        d = ops[i]
        d.id = o.id
        d.kind = int(o.kind)
        d.n_operands = len(o.operands)
        d.operands = refs
        if o.value is not None and len(o.value):
            val = m.hold(_f64(o.value))
            d.n_value = val.size
            d.value = _ptr(val, f64p)
        d.inc = int(o.inc)
        d.neuron_kind = int(o.neuron.kind)
        d.tau_rc, d.tau_ref, d.amplitude = o.neuron.tau_rc, o.neuron.tau_ref, o.neuron.amplitude
        d.tau, d.learning_rate, d.dt = o.tau, o.learning_rate, o.dt
    npb = len(model.probes)
    probes = m.hold((neng_probe * max(npb, 1))())
    for i, p in enumerate(model.probes):
        probes[i].key, probes[i].signal = p.key, p.signal
        probes[i].label = m.hold(p.label.encode())
    nf = len(model.feed_slots)
    slots = m.hold((neng_feed_slot * max(nf, 1))())
    for i, f in enumerate(model.feed_slots):
        slots[i].node_id, slots[i].signal, slots[i].dim = f.node_id, f.signal, f.dim
        slots[i].has_default = int(f.has_default)
        slots[i].label = m.hold(f.label.encode())
    v = neng_built_model()
    v.n_signals, v.signals = ns, sigs
    v.n_operators, v.operators = no, ops
    v.n_probes, v.probes = npb, probes
    v.n_feed_slots, v.feed_slots = nf, slots
    v.dt = model.dt
    return v


def planned_model_view(pm: ir.PlannedModel, m: Marshalled) -> neng_planned_model:
    v = neng_planned_model()
    v.model = built_model_view(pm.model, m)
    offs = [0]
    mem: List[int] = []
    for g in pm.plan:
        mem.extend(g)
        offs.append(len(mem))
    goff = m.hold(_i32(offs))
    gmem = m.hold(_i32(mem if mem else [0]))
    v.n_groups = len(pm.plan)
    v.group_offsets = _ptr(goff, i32p)
    v.group_members = _ptr(gmem, i32p)
    bof = m.hold(_i32(pm.buffers.buffer_of if pm.buffers.buffer_of else [0]))
    rof = m.hold(_i32(pm.buffers.row_offset if pm.buffers.row_offset else [0]))
    v.buffer_of, v.row_offset = _ptr(bof, i32p), _ptr(rof, i32p)
    nb = len(pm.buffers.buffers)
    bufs = m.hold((neng_buffer_desc * max(nb, 1))())
    for i, b in enumerate(pm.buffers.buffers):
        tr = m.hold(_i32(b.trailing if b.trailing else [0]))
        order = m.hold(_i32(b.order if b.order else [0]))
        bufs[i].n_trailing, bufs[i].trailing = len(b.trailing), _ptr(tr, i32p)
        bufs[i].elem, bufs[i].minibatched, bufs[i].trainable = int(b.elem), int(b.minibatched), int(b.trainable)
        bufs[i].rows = b.rows
        bufs[i].n_order, bufs[i].order = len(b.order), _ptr(order, i32p)
    v.n_buffers, v.buffers = nb, bufs
    return v


def _arr_i32(p, n) -> List[int]:
    return [int(p[i]) for i in range(n)] if n else []


def built_model_from_view(v: neng_built_model) -> ir.BuiltModel:
    model = ir.BuiltModel(dt=v.dt)
    for i in range(v.n_signals):
        s = v.signals[i]
        shape = _arr_i32(s.shape, s.ndim)
        init = None
        if s.n_initial > 0:
            init = np.ctypeslib.as_array(s.initial, shape=(s.n_initial,)).copy()
        model.signals.append(ir.Signal(s.id, (s.label or b"").decode(), shape, ir.Elem(s.elem), init,
                                       bool(s.constant), bool(s.minibatched), bool(s.trainable)))
    for i in range(v.n_operators):
        o = v.operators[i]
        refs = [ir.SignalRef(o.operands[k].signal, o.operands[k].start, o.operands[k].stop)
                for k in range(o.n_operands)]
        val = None
        if o.n_value > 0:
            val = np.ctypeslib.as_array(o.value, shape=(o.n_value,)).copy()
        elif o.kind == ir.OpKind.Reset:
            val = np.zeros(0)
        model.operators.append(ir.Operator(o.id, ir.OpKind(o.kind), refs, val, bool(o.inc),
                                           ir.NeuronModel(ir.NeuronKind(o.neuron_kind), o.tau_rc,
                                                          o.tau_ref, o.amplitude),
                                           o.tau, o.learning_rate, o.dt))
    for i in range(v.n_probes):
        p = v.probes[i]
        model.probes.append(ir.ProbeRegistration(p.key, p.signal, (p.label or b"").decode()))
    for i in range(v.n_feed_slots):
        f = v.feed_slots[i]
        model.feed_slots.append(ir.FeedSlot(f.node_id, f.signal, f.dim, bool(f.has_default),
                                            (f.label or b"").decode()))
    return model


def planned_model_from_view(v: neng_planned_model, stats=None) -> ir.PlannedModel:
    model = built_model_from_view(v.model)
    plan = []
    for g in range(v.n_groups):
        plan.append([int(v.group_members[k]) for k in range(v.group_offsets[g], v.group_offsets[g + 1])])
    ns = v.model.n_signals
    bufs = []
    for b in range(v.n_buffers):
        d = v.buffers[b]
        bufs.append(ir.BufferDesc(_arr_i32(d.trailing, d.n_trailing), ir.Elem(d.elem), bool(d.minibatched),
                                  bool(d.trainable), d.rows, _arr_i32(d.order, d.n_order)))
    ba = ir.BufferAssignment(_arr_i32(v.buffer_of, ns), _arr_i32(v.row_offset, ns), bufs)
    return ir.PlannedModel(model, plan, ba, stats or ir.ContiguityStats())


def feeds_view(feeds, m: Marshalled):
    """FeedData (node id -> float64 [batch, steps, dim]) -> neng_feed array."""
    items = sorted(feeds.items())
    arr = m.hold((neng_feed * max(len(items), 1))())
    for i, (node, t) in enumerate(items):
        t = m.hold(np.ascontiguousarray(t, dtype=np.float64))
        if t.ndim != 3:
            raise ValueError("feed tensors must be [batch, steps, dim]")
        arr[i].node_id = int(node)
        arr[i].batch, arr[i].steps, arr[i].dim = t.shape
        arr[i].data = _ptr(t, f64p)
    return len(items), arr


def split_probes(model: ir.BuiltModel, flat: np.ndarray, batch: int, n_steps: int) -> dict:
    """Inverse of the probes_out packing: per probe (registration order) a
    [batch][n_steps][dim] block.  Mirrors ProbeOutput's map-by-key."""
    out = {}
    at = 0
    for p in model.probes:
        dim = model.signals[p.signal].size()
        n = batch * n_steps * dim
        if p.key not in out:
            out[p.key] = flat[at:at + n].reshape(batch, n_steps, dim)
        at += n
    return out


def probe_total(model: ir.BuiltModel, batch: int, n_steps: int) -> int:
    return sum(batch * n_steps * model.signals[p.signal].size() for p in model.probes)
