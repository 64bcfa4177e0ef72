"""Python mirror of the reference's model types (names, fields and error types
follow proj/include/nengine/{ir,model,passes}.hpp so tests read like the
reference's own).  These are plain containers; all validation, planning and
execution happen in C++/CUDA behind the C ABI (include/neng_gpu.h).

  Signal            ir.hpp:37-58        SignalRef        ir.hpp:61-73
  OpKind            ir.hpp:78-87        NeuronKind       ir.hpp:91
  NeuronModel       ir.hpp:95-103       Operator         ir.hpp:114-137
  ProbeRegistration model.hpp:35-39     FeedSlot         model.hpp:41-47
  BuiltModel        model.hpp:54-60     Tensor3          model.hpp:15-31 (ndarray [batch, steps, dim])
  BufferDesc        passes.hpp:63-70    BufferAssignment passes.hpp:72-76
  PipelineConfig    passes.hpp:122-128  PlannedModel     passes.hpp:131-137
  StructuralError / BuildError / RunError  ir.hpp:15-25
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np


class StructuralError(RuntimeError):
    """neng::StructuralError (ir.hpp:15-17)."""


class BuildError(RuntimeError):
    """neng::BuildError (ir.hpp:19-21)."""


class RunError(RuntimeError):
    """neng::RunError (ir.hpp:23-25)."""


class CudaError(RuntimeError):
    """Device failure reported by the engine (no reference equivalent)."""


class OpKind(enum.IntEnum):
    Reset = 0
    Copy = 1
    ElementwiseInc = 2
    DotInc = 3
    SimNeurons = 4
    SimProcess = 5
    SimPES = 6
    TimeUpdate = 7


class NeuronKind(enum.IntEnum):
    LIF = 0
    LIFRate = 1
    RectifiedLinear = 2


class Elem(enum.IntEnum):
    f32 = 0
    f64 = 1


class StorageMode(enum.IntEnum):
    Shared = 0
    PerBatch = 1


class Planner(enum.IntEnum):
    Greedy = 0
    Tree = 1
    TransitiveClosure = 2


@dataclass
class Signal:
    id: int
    label: str
    shape: List[int]
    elem: Elem = Elem.f64
    initial: Optional[np.ndarray] = None  # flattened row-major float64; None = zeros
    constant: bool = False
    minibatched: bool = False
    trainable: bool = False

    def rows(self) -> int:
        return self.shape[0] if self.shape else 0

    def elems_per_row(self) -> int:
        n = 1
        for d in self.shape[1:]:
            n *= d
        return n

    def size(self) -> int:
        return self.rows() * self.elems_per_row()

    def trailing_shape(self) -> List[int]:
        return list(self.shape[1:])


@dataclass(frozen=True)
class SignalRef:
    signal: int
    start: int
    stop: int

    def rows(self) -> int:
        return self.stop - self.start

    @staticmethod
    def full(s: Signal) -> "SignalRef":
        return SignalRef(s.id, 0, s.rows())

    @staticmethod
    def slice(s: Signal, start: int, stop: int) -> "SignalRef":
        return SignalRef(s.id, start, stop)


@dataclass
class NeuronModel:
    kind: NeuronKind = NeuronKind.LIF
    tau_rc: float = 0.02
    tau_ref: float = 0.002
    amplitude: float = 1.0

    def has_state(self) -> bool:
        return self.kind == NeuronKind.LIF


@dataclass
class Operator:
    id: int
    kind: OpKind
    operands: List[SignalRef]
    value: Optional[np.ndarray] = None  # Reset payload (float64)
    inc: bool = False
    neuron: NeuronModel = field(default_factory=NeuronModel)
    tau: float = 0.0
    learning_rate: float = 0.0
    dt: float = 0.0

    # Factories mirror Operator::reset/copy/... (ir.cpp:39-112)
    @staticmethod
    def reset(id: int, dst: SignalRef, value: Sequence[float]) -> "Operator":
        return Operator(id, OpKind.Reset, [dst], value=np.asarray(value, dtype=np.float64))

    @staticmethod
    def copy(id: int, src: SignalRef, dst: SignalRef, inc: bool) -> "Operator":
        return Operator(id, OpKind.Copy, [src, dst], inc=bool(inc))

    @staticmethod
    def elementwise_inc(id: int, a: SignalRef, x: SignalRef, y: SignalRef) -> "Operator":
        return Operator(id, OpKind.ElementwiseInc, [a, x, y])

    @staticmethod
    def dot_inc(id: int, a: SignalRef, x: SignalRef, y: SignalRef) -> "Operator":
        return Operator(id, OpKind.DotInc, [a, x, y])

    @staticmethod
    def sim_neurons(id: int, model: NeuronModel, j: SignalRef, out: SignalRef,
                    states: Sequence[SignalRef] = ()) -> "Operator":
        return Operator(id, OpKind.SimNeurons, [j, out, *states], neuron=model)

    @staticmethod
    def sim_process(id: int, tau: float, inp: SignalRef, out: SignalRef,
                    state: Optional[SignalRef] = None) -> "Operator":
        ops = [inp, out] + ([state] if state is not None else [])
        return Operator(id, OpKind.SimProcess, ops, tau=float(tau))

    @staticmethod
    def sim_pes(id: int, learning_rate: float, pre: SignalRef, error: SignalRef,
                weights: SignalRef) -> "Operator":
        return Operator(id, OpKind.SimPES, [pre, error, weights], learning_rate=float(learning_rate))

    @staticmethod
    def time_update(id: int, dt: float, step: SignalRef, time: SignalRef) -> "Operator":
        return Operator(id, OpKind.TimeUpdate, [step, time], dt=float(dt))


@dataclass
class ProbeRegistration:
    key: int
    signal: int
    label: str = ""


@dataclass
class FeedSlot:
    node_id: int
    signal: int
    dim: int
    has_default: bool = True
    label: str = ""


@dataclass
class BuiltModel:
    signals: List[Signal] = field(default_factory=list)
    operators: List[Operator] = field(default_factory=list)
    probes: List[ProbeRegistration] = field(default_factory=list)
    feed_slots: List[FeedSlot] = field(default_factory=list)
    dt: float = 0.001

    def add_signal(self, label: str, shape: Sequence[int], initial=None, constant=False,
                   minibatched=False, trainable=False) -> int:
        sid = len(self.signals)
        init = None if initial is None else np.ascontiguousarray(initial, dtype=np.float64).ravel()
        self.signals.append(Signal(sid, label, list(shape), Elem.f64, init, bool(constant),
                                   bool(minibatched), bool(trainable)))
        return sid

    def full(self, sid: int) -> SignalRef:
        return SignalRef.full(self.signals[sid])

    def next_op(self) -> int:
        return len(self.operators)


@dataclass
class BufferDesc:
    trailing: List[int]
    elem: Elem
    minibatched: bool
    trainable: bool
    rows: int
    order: List[int]


@dataclass
class BufferAssignment:
    buffer_of: List[int]
    row_offset: List[int]
    buffers: List[BufferDesc]


@dataclass
class ContiguityStats:
    contiguous_read_fraction: float = 1.0
    gather_row_count: int = 0
    groups_per_step: int = 0


@dataclass
class PipelineConfig:
    merge: bool = True
    simplify: bool = True
    planner: Planner = Planner.Tree
    tree_depth: int = 3
    sort: bool = True


@dataclass
class PlannedModel:
    model: BuiltModel
    plan: List[List[int]]
    buffers: BufferAssignment
    stats: ContiguityStats = field(default_factory=ContiguityStats)


Tensor3 = np.ndarray           # float64 [batch, steps, dim]
FeedData = Dict[int, np.ndarray]
ProbeOutput = Dict[int, np.ndarray]


def compare(a: ProbeOutput, b: ProbeOutput, rel_tol: float, abs_tol: float):
    """neng::compare (reference.cpp:228-258): (max_abs_err, max_rel_err,
    within_tolerance, first_divergence)."""
    if set(a) != set(b):
        raise RunError("compare: probe sets differ")
    max_abs = max_rel = 0.0
    ok = True
    first = None
    for key in sorted(a):
        ta, tb = a[key], b[key]
        if ta.shape != tb.shape:
            raise RunError(f"compare: trace shapes differ for probe {key}")
        err = np.abs(ta - tb)
        mag = np.maximum(np.abs(ta), np.abs(tb))
        with np.errstate(invalid="ignore", divide="ignore"):
            if err.size:
                m = np.nanmax(err) if np.any(~np.isnan(err)) else 0.0
                max_abs = max(max_abs, float(m))
                rel = np.where(mag > 0, err / np.where(mag > 0, mag, 1), 0.0)
                if np.any(~np.isnan(rel)):
                    max_rel = max(max_rel, float(np.nanmax(rel)))
            bad = err > abs_tol + rel_tol * mag
        if np.any(bad):
            ok = False
            if first is None:
                idx = tuple(int(i) for i in np.argwhere(bad)[0])
                first = (key, *idx, float(ta[idx]), float(tb[idx]))
    return max_abs, max_rel, ok, first
