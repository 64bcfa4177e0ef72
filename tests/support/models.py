"""Test fixtures mirroring proj/tests/test_exec.cpp:18-139 and
proj/tests/test_reference.cpp:14-28 (chain/learning models, wave feeds,
batch/step slicing, the hand-built golden models), plus comparison helpers."""
from __future__ import annotations

import math

import numpy as np

from paper_1805_11144_b200 import ir
from paper_1805_11144_b200.ir import NeuronKind, NeuronModel, Operator, SignalRef
from paper_1805_11144_b200.networks import NetBuilder


def pipeline_variants():
    """test_exec.cpp:22-33"""
    full = ir.PipelineConfig()
    greedy = ir.PipelineConfig(planner=ir.Planner.Greedy)
    no_merge = ir.PipelineConfig(merge=False)
    no_sort = ir.PipelineConfig(sort=False)
    no_simplify = ir.PipelineConfig(simplify=False)
    return [full, greedy, no_merge, no_sort, no_simplify]


def _decoders(nb: NetBuilder, n: int, d: int, stream: int, scale: float = 1.0):
    rng = np.random.default_rng(1000 + stream)
    return rng.normal(0.0, scale / math.sqrt(n), size=(d, n))


def chain_model(seed: int = 11, dim: int = 2):
    """feedable input -> filtered connection -> spiking ensemble -> decoded probe
    (test_exec.cpp:42-52)."""
    nb = NetBuilder(seed)
    node, u = nb.feedable_node(dim, np.full(dim, 0.25))
    e = nb.ensemble(40, dim)
    nb.connect(u, e.in_, None, synapse=0.01)
    xhat = nb.decoded(e, _decoders(nb, 40, dim, 1, scale=4.0))
    key = nb.probe(xhat, "value")
    return nb.m, node, key


def learning_model(seed: int = 23, dim: int = 2):
    """Decoders of ens -> out start at zero and learn from err = out - target
    (test_exec.cpp:62-90)."""
    nb = NetBuilder(seed)
    node_u, u = nb.feedable_node(dim, np.full(dim, 0.4))
    e = nb.ensemble(60, dim)
    out = nb.passthrough_node(dim)
    node_t, target = nb.feedable_node(dim, np.zeros(dim))
    err = nb.passthrough_node(dim)
    nb.connect(u, e.in_, None, synapse=0.005)
    c = nb.connect(e.out, out, np.zeros((dim, e.n)), synapse=0.005, learned_rate=5e-4, error=err)
    nb.connect(out, err, None, synapse=0.0, scalar=1.0)
    nb.connect(target, err, None, synapse=0.0, scalar=-1.0)
    key = nb.probe(out, "out")
    return nb.m, node_u, node_t, key, c["weights"]


def wave_feed(batch, steps, dim, base):
    """test_exec.cpp:92-99"""
    b = np.arange(batch)[:, None, None]
    s = np.arange(steps)[None, :, None]
    d = np.arange(dim)[None, None, :]
    return base + 0.2 * b - 0.1 * d + 0.3 * np.sin(0.13 * s + b)


def batch_slice(feeds, b):
    return {k: t[b:b + 1].copy() for k, t in feeds.items()}


def step_slice(feeds, start, count):
    return {k: t[:, start:start + count].copy() for k, t in feeds.items()}


def concat_steps(a, b):
    return {k: np.concatenate([a[k], b[k]], axis=1) for k in a}


def make_signal(sid, label, shape, constant=False, minibatched=False, trainable=False, initial=None):
    init = None if initial is None else np.asarray(initial, dtype=np.float64)
    return ir.Signal(sid, label, list(shape), ir.Elem.f64, init, constant, minibatched, trainable)


def constant_drive_lif(j_value):
    """test_reference.cpp:14-28"""
    m = ir.BuiltModel()
    m.signals = [make_signal(0, "J", [1], constant=True, initial=[j_value]), make_signal(1, "spikes", [1]),
                 make_signal(2, "voltage", [1]), make_signal(3, "refractory", [1])]
    f = SignalRef.full
    m.operators = [Operator.sim_neurons(0, NeuronModel(), f(m.signals[0]), f(m.signals[1]),
                                        [f(m.signals[2]), f(m.signals[3])])]
    m.probes = [ir.ProbeRegistration(0, 1, "spikes"), ir.ProbeRegistration(1, 2, "voltage")]
    return m


def assert_bitexact(a, b, context=""):
    """Probe outputs identical bit for bit (NaN positions must match; NaN
    payloads are not compared — see DESIGN.md)."""
    assert set(a) == set(b), f"{context}: probe sets differ"
    for k in a:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.shape == y.shape, f"{context}: probe {k} shape {x.shape} vs {y.shape}"
        nx, ny = np.isnan(x), np.isnan(y)
        assert np.array_equal(nx, ny), f"{context}: probe {k} NaN positions differ"
        xb, yb = x.view(np.uint64), y.view(np.uint64)
        bad = (xb != yb) & ~nx
        if bad.any():
            idx = tuple(int(i) for i in np.argwhere(bad)[0])
            raise AssertionError(f"{context}: probe {k} differs at {idx}: {x[idx]!r} vs {y[idx]!r} "
                                 f"({int(bad.sum())} of {bad.size} elements)")
