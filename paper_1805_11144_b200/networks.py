"""Seeded synthetic workloads at the IR level.

`NetBuilder` lowers ensembles, nodes, connections and probes to Signals and
Operators following the reference frontend's lowering rules
(proj/src/frontend.cpp: lower_ensemble :305-341, lower_node :343-367,
lower_connection :419-517, lower_probe :519-550, Lowering::run :552-567),
with the decoded-output split of SURVEY §8(d) ("unfolded": per ensemble
Reset(xhat,0) + DotInc(D, out, xhat); per connection DotInc(T, xhat_src, acc)).
Ensemble tuning follows sample_ensemble_parameters / gain_bias
(frontend.cpp:38-54, 78-118).  Decoders are drawn as seeded Gaussians (the
configs specify them that way); the least-squares solve of the reference
frontend needs Eigen and is out of scope — both engines consume the same
BuiltModel, so the choice does not affect parity.

`config0 ... config4` build the five BASELINE.json workloads.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import ir
from .ir import NeuronModel, Operator
from .rng import Rng, derive_seed


def gain_bias_lif(max_rates: np.ndarray, intercepts: np.ndarray, tau_rc=0.02, tau_ref=0.002):
    """gain_bias for LIF (frontend.cpp:38-54), vectorised."""
    z = 1.0 / (1.0 - np.exp((tau_ref - 1.0 / max_rates) / tau_rc))
    gain = (z - 1.0) / (1.0 - intercepts)
    return gain, 1.0 - gain * intercepts


@dataclass
class Ens:
    index: int
    n: int
    d: int
    in_: int
    j: int
    out: int
    v: int
    r: int
    enc: int
    xhat: int = -1


class NetBuilder:
    def __init__(self, seed: int = 1, dt: float = 0.001, clock: bool = True):
        self.seed = seed
        self.m = ir.BuiltModel(dt=dt)
        self.ens: List[Ens] = []
        self.n_nodes = 0
        self.n_conn = 0
        self.n_probes = 0
        if clock:  # Lowering::run (frontend.cpp:552-557)
            step = self.m.add_signal("step", [1])
            time = self.m.add_signal("time", [1])
            self.m.operators.append(Operator.time_update(self.m.next_op(), dt, self.m.full(step), self.m.full(time)))

    # -- helpers ---------------------------------------------------------------
    def _op(self, op: Operator):
        self.m.operators.append(op)

    def sample_tuning(self, n: int, d: int, stream: int, max_rate=(200.0, 400.0), intercept=(-1.0, 1.0)):
        """Unit-sphere encoders, U(max_rate), U(intercept) (frontend.cpp:78-118)."""
        rng = Rng(derive_seed(self.seed, stream))
        enc = rng.gaussian_array(n * d).reshape(n, d)
        norm = np.sqrt(np.sum(enc * enc, axis=1, keepdims=True))
        norm[norm < 1e-12] = 1.0
        enc = enc / norm
        max_rates = rng.uniform_array(n, *max_rate)
        intercepts = rng.uniform_array(n, *intercept)
        gain, bias = gain_bias_lif(max_rates, intercepts)
        return enc, gain, bias

    # -- lowering ----------------------------------------------------------------
    def ensemble(self, n: int, d: int, neuron: NeuronModel = None, radius: float = 1.0,
                 gain=None, bias=None, encoders=None) -> Ens:
        """lower_ensemble (frontend.cpp:305-341)."""
        neuron = neuron or NeuronModel()
        i = len(self.ens)
        if encoders is None:
            enc, g, b = self.sample_tuning(n, d, 2 * i)
            gain = g if gain is None else gain
            bias = b if bias is None else bias
        else:
            enc = np.asarray(encoders, dtype=np.float64).reshape(n, d)
            gain = np.ones(n) if gain is None else np.asarray(gain, dtype=np.float64)
            bias = np.zeros(n) if bias is None else np.asarray(bias, dtype=np.float64)
        base = f"ens{i}"
        in_ = self.m.add_signal(base + ".in", [d], minibatched=True)
        j = self.m.add_signal(base + ".J", [n], minibatched=True)
        out = self.m.add_signal(base + ".out", [n], minibatched=True)
        scaled = enc * (np.asarray(gain) / radius)[:, None]
        E = self.m.add_signal(base + ".encoders", [n, d], scaled.ravel(), constant=True, trainable=True)
        self._op(Operator.reset(self.m.next_op(), self.m.full(in_), np.zeros(d)))
        self._op(Operator.reset(self.m.next_op(), self.m.full(j), np.asarray(bias, dtype=np.float64)))
        self._op(Operator.dot_inc(self.m.next_op(), self.m.full(E), self.m.full(in_), self.m.full(j)))
        v = r = -1
        states = []
        if neuron.has_state():
            v = self.m.add_signal(base + ".voltage", [n], minibatched=True)
            r = self.m.add_signal(base + ".refractory", [n], minibatched=True)
            states = [self.m.full(v), self.m.full(r)]
        self._op(Operator.sim_neurons(self.m.next_op(), neuron, self.m.full(j), self.m.full(out), states))
        e = Ens(i, n, d, in_, j, out, v, r, E)
        self.ens.append(e)
        return e

    def solve_decoders(self, e: Ens, fn=None, fn_dim: Optional[int] = None, eval_points_per_dim: int = 500,
                       radius: float = 1.0, reg: float = 0.1, tau_rc: float = 0.02, tau_ref: float = 0.002,
                       amplitude: float = 1.0) -> np.ndarray:
        """Least-squares decoders of f(x) for LIF ensemble e (Lowering::decode,
        frontend.cpp:376-417): eval points uniform in the radius-ball (seeded
        directions, radius * U^(1/d)), activities = the LIF rate of the
        ensemble's own encoders and biases, and the native Eigen-free solve
        (passes.solve_decoders).  Returns D [fn_dim][n] (the decoded()
        layout); fn maps a [m][d] array of points to [m][fn_dim] (default:
        the identity)."""
        from . import passes
        E = np.asarray(self.m.signals[e.enc].initial).reshape(e.n, e.d)  # gain / radius folded in
        bias = next(np.asarray(op.value) for op in self.m.operators
                    if op.kind == ir.OpKind.Reset and op.operands[0].signal == e.j)
        m = eval_points_per_dim * e.d
        rng = Rng(derive_seed(self.seed, 2 * e.index + 1))
        pts = np.empty((m, e.d))
        for s_ in range(m):  # reference order: d normals then one uniform per point
            x = np.array([rng.gaussian() for _ in range(e.d)])
            r = radius * rng.uniform() ** (1.0 / e.d)
            nsq = float(x @ x)
            pts[s_] = x * (0.0 if nsq < 1e-24 else r / math.sqrt(nsq))
        J = pts @ E.T + bias[None, :]
        with np.errstate(divide="ignore"):
            act = np.where(J > 1.0, amplitude / (tau_ref + tau_rc * np.log1p(1.0 / np.maximum(J - 1.0, 1e-300))), 0.0)
        Y = pts if fn is None else np.asarray(fn(pts), dtype=np.float64).reshape(m, -1)
        if fn_dim is not None and Y.shape[1] != fn_dim:
            raise ValueError(f"function returned {Y.shape[1]} values, expected {fn_dim}")
        return passes.solve_decoders(act, Y, reg).T

    def decoded(self, e: Ens, D: np.ndarray) -> int:
        """Decoded value xhat = D . out (D: d_out x n), SURVEY §8(d) unfolded lowering."""
        D = np.asarray(D, dtype=np.float64)
        dout = D.shape[0]
        base = f"ens{e.index}"
        xhat = self.m.add_signal(base + ".xhat", [dout], minibatched=True)
        W = self.m.add_signal(base + ".decoders", [dout, e.n], D.ravel(), constant=True, trainable=True)
        self._op(Operator.reset(self.m.next_op(), self.m.full(xhat), np.zeros(dout)))
        self._op(Operator.dot_inc(self.m.next_op(), self.m.full(W), self.m.full(e.out), self.m.full(xhat)))
        e.xhat = xhat
        return xhat

    def feedable_node(self, dim: int, default: Optional[np.ndarray] = None) -> Tuple[int, int]:
        """lower_node, Feedable (frontend.cpp:351-357): returns (node_id, signal)."""
        node = self.n_nodes
        self.n_nodes += 1
        has_default = default is not None
        sig = self.m.add_signal(f"node{node}.out", [dim], default, minibatched=True)
        self.m.feed_slots.append(ir.FeedSlot(node, sig, dim, has_default, f"node{node}"))
        return node, sig

    def passthrough_node(self, dim: int) -> int:
        """lower_node, Passthrough (frontend.cpp:358-364)."""
        node = self.n_nodes
        self.n_nodes += 1
        sig = self.m.add_signal(f"node{node}.out", [dim], minibatched=True)
        self._op(Operator.reset(self.m.next_op(), self.m.full(sig), np.zeros(dim)))
        return sig

    def connect(self, src: int, dst: Optional[int], transform=None, synapse: float = 0.005,
                scalar: Optional[float] = None, learned_rate: Optional[float] = None,
                error: Optional[int] = None) -> Dict[str, int]:
        """lower_connection (frontend.cpp:419-517) from a value signal `src`
        into `dst` (an ensemble input or node), or into nothing (probe filter)."""
        c = self.n_conn
        self.n_conn += 1
        base = f"conn{c}"
        sdim = self.m.signals[src].size()
        if transform is not None:
            T = np.asarray(transform, dtype=np.float64)
            ddim = T.shape[0]
        else:
            ddim = sdim
        acc = self.m.add_signal(base + ".accum", [ddim], minibatched=True)
        self._op(Operator.reset(self.m.next_op(), self.m.full(acc), np.zeros(ddim)))
        w = -1
        if scalar is not None:
            sc = self.m.add_signal(base + ".scale", [1], [scalar], constant=True, trainable=True)
            self._op(Operator.elementwise_inc(self.m.next_op(), self.m.full(sc), self.m.full(src), self.m.full(acc)))
        else:
            if transform is None:
                T = np.eye(ddim, sdim)
            w = self.m.add_signal(base + ".weights", [ddim, sdim], T.ravel(), constant=learned_rate is None,
                                  trainable=True)
            self._op(Operator.dot_inc(self.m.next_op(), self.m.full(w), self.m.full(src), self.m.full(acc)))
        out = {"accum": acc, "weights": w}
        copied = acc
        if synapse > 0.0:
            filt = self.m.add_signal(base + ".filtered", [ddim], minibatched=True)
            state = self.m.add_signal(base + ".state", [ddim], minibatched=True)
            self._op(Operator.sim_process(self.m.next_op(), synapse, self.m.full(acc), self.m.full(filt),
                                          self.m.full(state)))
            copied = filt
            out["filtered"], out["state"] = filt, state
        if dst is not None:
            self._op(Operator.copy(self.m.next_op(), self.m.full(copied), self.m.full(dst), True))
        if learned_rate is not None:
            # SimPES on the connection weights (frontend.cpp:511-516); src must be neuron output
            self._op(Operator.sim_pes(self.m.next_op(), learned_rate, self.m.full(src), self.m.full(error),
                                      self.m.full(w)))
        out["value"] = copied
        return out

    def probe(self, sig: int, label: str = "") -> int:
        key = self.n_probes
        self.n_probes += 1
        self.m.probes.append(ir.ProbeRegistration(key, sig, label or f"probe{key}"))
        return key


def algorithmic_bytes_per_step(model: ir.BuiltModel, batch: int) -> int:
    """HBM bytes one timestep must move at minimum:
    4 * [ 4*N*B          LIF v, r read + write
        + N              J bias payload
        + sum n*d        encoders       + sum d*n  decoders
        + sum dd*ds      transforms     + 2*sum dd*B  lowpass state read + write
        + sum dim*B      feeds          + sum dim*B   probes ]
    Transients (J, out, in, xhat, acc) are excluded: a fused kernel keeps them
    on-chip.  Counted from the model's operators, so it holds for any
    ensemble network built by NetBuilder."""
    s = model.signals
    floats = 0
    for op in model.operators:
        k = op.kind
        if k == ir.OpKind.SimNeurons and op.neuron.kind == ir.NeuronKind.LIF:
            floats += 4 * s[op.operands[0].signal].size() * batch
        elif k == ir.OpKind.Reset and s[op.operands[0].signal].label.endswith(".J"):
            floats += s[op.operands[0].signal].size()
        elif k == ir.OpKind.DotInc:
            floats += s[op.operands[0].signal].size()
        elif k == ir.OpKind.SimProcess and op.tau > 0:
            floats += 2 * s[op.operands[0].signal].size() * batch
    floats += sum(f.dim for f in model.feed_slots) * batch
    floats += sum(s[p.signal].size() for p in model.probes) * batch
    return 4 * floats


def neuron_count(model: ir.BuiltModel) -> int:
    return sum(model.signals[op.operands[0].signal].size() for op in model.operators
               if op.kind == ir.OpKind.SimNeurons)


# ---------------------------------------------------------------------------
# BASELINE.json configurations

@dataclass
class Workload:
    name: str
    model: ir.BuiltModel
    batch: int
    steps: int
    feeds: Dict[int, np.ndarray]   # node id -> [batch, steps, dim] f64
    neurons: int
    notes: str = ""


def white_noise(seed: int, batch: int, steps: int, dim: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((batch, steps, dim))


def config0(seed: int = 1, steps: int = 1000) -> Workload:
    """Integrator: 1 x 800 LIF, 16-D, recurrent identity through tau=0.1,
    16-D white-noise input through tau=0.01, probe = decoded output through a
    0.01 s filter; B=1."""
    nb = NetBuilder(seed)
    d, n = 16, 800
    e = nb.ensemble(n, d)
    rng = np.random.default_rng(derive_seed(seed, 1000) % (2 ** 63))
    D = rng.normal(0.0, math.sqrt(1.0 / n), size=(d, n))
    xhat = nb.decoded(e, D)
    node, u = nb.feedable_node(d, np.zeros(d))
    nb.connect(u, e.in_, None, synapse=0.01)
    nb.connect(xhat, e.in_, None, synapse=0.1)
    pc = nb.connect(xhat, None, None, synapse=0.01)
    nb.probe(pc["filtered"], "decoded")
    feeds = {node: white_noise(seed, 1, steps, d)}
    return Workload("config0_integrator", nb.m, 1, steps, feeds, n)


def random_network(seed: int, n_ens: int, n: int, d: int, k_out: int, n_inputs: int, batch: int, steps: int,
                   probes: int = 1, name: str = "random") -> Workload:
    """Random decoded network (configs 2 and 4): each ensemble sends k_out
    decoded connections to distinct random other ensembles (decoders
    N(0,1/n), transforms N(0,1/d)*0.5, tau=0.01); n_inputs d-D white-noise
    feeds each drive one random ensemble through tau=0.01."""
    nb = NetBuilder(seed)
    rng = np.random.default_rng(derive_seed(seed, 7) % (2 ** 63))
    ens = [nb.ensemble(n, d) for _ in range(n_ens)]
    for e in ens:
        nb.decoded(e, rng.normal(0.0, math.sqrt(1.0 / n), size=(d, n)))
    for e in ens:
        others = rng.choice(n_ens - 1, size=min(k_out, n_ens - 1), replace=False)
        for o in others:
            t = int(o) if o < e.index else int(o) + 1
            T = rng.normal(0.0, math.sqrt(1.0 / d), size=(d, d)) * 0.5
            nb.connect(e.xhat, ens[t].in_, T, synapse=0.01)
    feeds = {}
    targets = rng.choice(n_ens, size=n_inputs, replace=n_inputs > n_ens)
    for i, t in enumerate(targets):
        node, u = nb.feedable_node(d, np.zeros(d))
        nb.connect(u, ens[int(t)].in_, None, synapse=0.01)
        feeds[node] = None
    for p in range(min(probes, n_ens)):
        nb.probe(ens[p].xhat, f"ens{p}.xhat")
    rngf = np.random.default_rng(seed + 99)
    for node in feeds:
        feeds[node] = rngf.standard_normal((batch, steps, d))
    return Workload(name, nb.m, batch, steps, feeds, n_ens * n)


def config1(seed: int = 1, steps: int = 1000, batch: int = 64, dims: int = 64, decoders: str = "ls") -> Workload:
    """Circular convolution of two `dims`-D inputs (BASELINE config 1): per batch row
    seeded unit-norm Gaussian vectors A, B, constant over the run.  The real DFT
    (frequencies 0..dims/2) projects A and B into 4*(dims/2+1) two-D product
    ensembles (100 LIF each; inputs [row_a.A, row_b.B] for the re*re, im*im,
    re*im, im*re products of each frequency); the product decoders (BASELINE
    leaves them unspecified) are the least-squares decoders of x0 * x1
    (decoders="ls", NetBuilder.solve_decoders: the frontend's regularised solve
    without Eigen), or seeded N(0, 1/100) with decoders="random"; the
    inverse real DFT maps the products onto `dims` one-D output ensembles (50
    LIF each) as scalar-transform decoded connections.  Every synapse is a
    lowpass with tau = 0.005 s.  Probes: the first four output ensembles'
    decoded values."""
    nb = NetBuilder(seed)
    rng = np.random.default_rng(derive_seed(seed, 11) % (2 ** 63))
    d = dims
    nf = d // 2 + 1
    n_idx = np.arange(d)
    cos = np.array([np.cos(2 * np.pi * k * n_idx / d) for k in range(nf)])   # [nf][d]
    sin = np.array([-np.sin(2 * np.pi * k * n_idx / d) for k in range(nf)])
    node_a, a = nb.feedable_node(d, np.zeros(d))
    node_b, b = nb.feedable_node(d, np.zeros(d))
    prods = []  # (ensemble, frequency, type)
    for k in range(nf):
        for typ, (ra, rb) in enumerate(((cos, cos), (sin, sin), (cos, sin), (sin, cos))):
            e = nb.ensemble(100, 2)
            # (the sine rows of frequencies 0 and d/2 vanish: no connection is built for them)
            if np.any(ra[k] != 0.0):
                nb.connect(a, e.in_, np.vstack([ra[k], np.zeros(d)]), synapse=0.005)
            if np.any(rb[k] != 0.0):
                nb.connect(b, e.in_, np.vstack([np.zeros(d), rb[k]]), synapse=0.005)
            if decoders == "ls":  # the product x0 * x1, least squares over the radius-1.5 ball (covers [-1, 1]^2)
                D = nb.solve_decoders(e, lambda p: p[:, :1] * p[:, 1:2], 1, eval_points_per_dim=100, radius=1.5)
            else:
                D = rng.normal(0.0, math.sqrt(1.0 / 100), size=(1, 100))
            nb.decoded(e, D)
            prods.append((e, k, typ))
    outs = []
    for j in range(d):
        e = nb.ensemble(50, 1)
        nb.decoded(e, rng.normal(0.0, math.sqrt(1.0 / 50), size=(1, 50)))
        outs.append(e)
    # inverse real DFT: c_j = sum_k w_k/d (Re C_k cos - Im C_k sin), Re C = rr - ii, Im C = ri + ir
    for (e, k, typ) in prods:
        wk = (1.0 if k == 0 or (d % 2 == 0 and k == d // 2) else 2.0) / d
        for j, o in enumerate(outs):
            c, s_ = math.cos(2 * math.pi * k * j / d), math.sin(2 * math.pi * k * j / d)
            t = wk * (c if typ == 0 else -c if typ == 1 else -s_)
            if t != 0.0:
                nb.connect(e.xhat, o.in_, np.array([[t]]), synapse=0.005)
    for j in range(min(4, d)):
        nb.probe(outs[j].xhat, f"c{j}")
    rngf = np.random.default_rng(seed + 1000)
    feeds = {}
    for node in (node_a, node_b):
        v = rngf.standard_normal((batch, d))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        feeds[node] = np.repeat(v[:, None, :], steps, axis=1)
    return Workload("config1_cconv", nb.m, batch, steps, feeds, len(prods) * 100 + d * 50)


def config2(seed: int = 1, steps: int = 1000, batch: int = 32) -> Workload:
    return random_network(seed, 256, 1024, 16, 4, 32, batch, steps, name="config2_random_256x1024")


def config4(seed: int = 1, steps: int = 500, batch: int = 256) -> Workload:
    return random_network(seed, 2048, 512, 8, 8, 256, batch, steps, name="config4_random_2048x512")


def config3(seed: int = 1, steps: int = 100, batch: int = 512, gain: float = 4.0) -> Workload:
    """Spiking MLP 784-1024-1024-10: LIF hidden layers (amplitude 0.01, bias 0),
    Glorot-uniform weights, lowpass 0.005 between layers, constant U[0,1]
    inputs fed per sample.  The RectifiedLinear->LIF conversion scales each
    hidden layer's input weights by `gain` (4: with gain 1 the Glorot-scaled
    currents stay below the LIF threshold in the second layer and the output
    is silent)."""
    nb = NetBuilder(seed)
    rng = np.random.default_rng(derive_seed(seed, 3) % (2 ** 63))
    sizes = [784, 1024, 1024, 10]

    def glorot(fan_out, fan_in):
        lim = math.sqrt(6.0 / (fan_in + fan_out))
        return rng.uniform(-lim, lim, size=(fan_out, fan_in))

    node, u = nb.feedable_node(784, None)
    lif = NeuronModel(ir.NeuronKind.LIF, amplitude=0.01)
    m = nb.m
    # layer 1: J1 = 0 + W1 . u
    h = []
    src = u
    for li in (1, 2):
        n = sizes[li]
        j = m.add_signal(f"l{li}.J", [n], minibatched=True)
        out = m.add_signal(f"l{li}.out", [n], minibatched=True)
        v = m.add_signal(f"l{li}.voltage", [n], minibatched=True)
        r = m.add_signal(f"l{li}.refractory", [n], minibatched=True)
        m.operators.append(Operator.reset(m.next_op(), m.full(j), np.zeros(n)))
        if li == 1:
            W = m.add_signal("W1", [n, sizes[0]], (gain * glorot(n, sizes[0])).ravel(), constant=True, trainable=True)
            m.operators.append(Operator.dot_inc(m.next_op(), m.full(W), m.full(src), m.full(j)))
        else:
            nb.connect(src, j, gain * glorot(n, sizes[li - 1]), synapse=0.005)
        m.operators.append(Operator.sim_neurons(m.next_op(), lif, m.full(j), m.full(out), [m.full(v), m.full(r)]))
        h.append(out)
        src = out
    pc = nb.connect(src, None, glorot(10, 1024), synapse=0.005)
    nb.probe(pc["filtered"], "output")
    x = np.random.default_rng(seed + 5).uniform(0.0, 1.0, size=(batch, 1, 784))
    feeds = {node: np.repeat(x, steps, axis=1)}
    return Workload("config3_spiking_mlp", nb.m, batch, steps, feeds, 2048)
