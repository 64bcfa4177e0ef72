"""Seeded generator of structurally valid random models — restates the rules
of the reference fixture proj/tests/support/random_models.hpp (pool of
vector sizes {1,2,3,5,8}, all-ones/all-zeros constants so simplification
has material, tentative commits rejected on validation/ordering failure,
at most one inc writer per target (:106-117), unbatched writers read only
unbatched inputs (:91-104, 199-201, 218-220)).  Commits are checked with
the reference's own validate_operators + build_dependency_graph through the
oracle library."""
from __future__ import annotations

from paper_1805_11144_b200 import ir
from paper_1805_11144_b200.ir import NeuronKind, NeuronModel, Operator, SignalRef
from paper_1805_11144_b200.rng import Rng

from oracle import refapi


class RandomModelBuilder:
    def __init__(self, seed: int):
        self.rng = Rng(seed)
        self.model = ir.BuiltModel()
        self.next_op_id = 0
        self.has_clock = False

    def build(self, target_ops: int) -> ir.BuiltModel:
        self.make_pool()
        attempts = 0
        while len(self.model.operators) < target_ops and attempts < target_ops * 30:
            attempts += 1
            self.try_add_random_op()
        self.add_probes()
        return self.model

    def add_signal(self, shape, constant, minibatched, initial=None):
        sid = len(self.model.signals)
        return self.model.add_signal(f"s{sid}", shape, initial, constant, minibatched, False)

    def random_values(self, n, lo=-1.0, hi=1.0):
        return [self.rng.uniform(lo, hi) for _ in range(n)]

    def pick(self, n):
        return int(self.rng.uniform() * n) % n

    def make_pool(self):
        for size in (1, 2, 3, 5, 8):
            for _ in range(2):
                self.add_signal([size], False, True)
                self.add_signal([size], False, False)
        for size in (1, 3, 5):
            self.add_signal([size], True, False, self.random_values(size))
            self.add_signal([size], True, False, [1.0] * size)
            self.add_signal([size], True, False, [0.0] * size)
        for r, c in ((2, 3), (3, 5), (5, 8), (3, 3)):
            self.add_signal([r, c], True, False, self.random_values(r * c))
            self.add_signal([r, c], False, False, self.random_values(r * c))

    def pick_signal(self, rows, minibatched, allow_constant, vector_only=True):
        fits = [s.id for s in self.model.signals
                if (not vector_only or len(s.shape) == 1) and s.rows() == rows
                and s.minibatched == minibatched and (allow_constant or not s.constant)]
        if not fits:
            return -1
        return fits[self.pick(len(fits))]

    def pick_dst(self, rows):
        mb = self.rng.uniform() < 0.65
        s = self.pick_signal(rows, mb, False)
        if s == -1:
            s = self.pick_signal(rows, not mb, False)
        if s == -1:
            return -1, False
        return s, self.model.signals[s].minibatched

    def inc_target_free(self, sig):
        for op in self.model.operators:
            if op.kind == ir.OpKind.Copy and op.inc and op.operands[1].signal == sig:
                return False
            if op.kind in (ir.OpKind.ElementwiseInc, ir.OpKind.DotInc) and op.operands[2].signal == sig:
                return False
        return True

    def maybe_slice(self, sig):
        s = self.model.signals[sig]
        if s.rows() >= 2 and self.rng.uniform() < 0.25:
            start = self.pick(s.rows())
            stop = start + 1 + self.pick(s.rows() - start)
            return SignalRef.slice(s, start, stop)
        return SignalRef.full(s)

    def try_add_random_op(self):
        oid = self.next_op_id
        self.next_op_id += 1
        roll = self.rng.uniform()
        if roll < 0.18:
            added = self.try_reset(oid)
        elif roll < 0.40:
            added = self.try_copy(oid)
        elif roll < 0.62:
            added = self.try_elementwise(oid)
        elif roll < 0.78:
            added = self.try_dot(oid)
        elif roll < 0.86:
            added = self.try_neurons(oid)
        elif roll < 0.94:
            added = self.try_process(oid)
        elif roll < 0.98:
            added = self.try_pes(oid)
        else:
            added = self.try_time(oid)
        if not added:
            self.next_op_id -= 1

    def commit(self, op):
        self.model.operators.append(op)
        try:
            refapi.validate(self.model)
            return True
        except (ir.StructuralError, ir.BuildError):
            self.model.operators.pop()
            return False

    def try_reset(self, oid):
        sig, _ = self.pick_dst(1 + self.pick(8))
        if sig == -1:
            return False
        ref = self.maybe_slice(sig)
        elems = ref.rows() * self.model.signals[sig].elems_per_row()
        return self.commit(Operator.reset(oid, ref, self.random_values(elems)))

    def try_copy(self, oid):
        dsig, dmb = self.pick_dst(1 + self.pick(8))
        if dsig == -1:
            return False
        dref = self.maybe_slice(dsig)
        src = self.pick_signal(dref.rows(), dmb and self.rng.uniform() < 0.8, self.rng.uniform() < 0.4)
        if src == -1 or (self.model.signals[src].minibatched and not dmb):
            return False
        ss = self.model.signals[src]
        sref = SignalRef.full(ss) if ss.rows() == dref.rows() else SignalRef.slice(ss, 0, dref.rows())
        inc = self.rng.uniform() < 0.5
        if inc and not self.inc_target_free(dsig):
            return False
        return self.commit(Operator.copy(oid, sref, dref, inc))

    def try_elementwise(self, oid):
        dsig, dmb = self.pick_dst(1 + self.pick(8))
        if dsig == -1 or not self.inc_target_free(dsig):
            return False
        y = self.model.signals[dsig]
        x = self.pick_signal(y.rows(), dmb and self.rng.uniform() < 0.7, self.rng.uniform() < 0.3)
        a_rows = 1 if self.rng.uniform() < 0.5 else y.rows()
        a = self.pick_signal(a_rows, False, self.rng.uniform() < 0.8)
        if x == -1 or a == -1:
            return False
        if not dmb and (self.model.signals[x].minibatched or self.model.signals[a].minibatched):
            return False
        s = self.model.signals
        return self.commit(Operator.elementwise_inc(oid, SignalRef.full(s[a]), SignalRef.full(s[x]),
                                                    SignalRef.full(y)))

    def try_dot(self, oid):
        mats = [s.id for s in self.model.signals if len(s.shape) == 2]
        if not mats:
            return False
        a = self.model.signals[mats[self.pick(len(mats))]]
        m, n = a.shape
        y = self.pick_signal(m, self.rng.uniform() < 0.5, False)
        x = self.pick_signal(n, self.rng.uniform() < 0.5, self.rng.uniform() < 0.3)
        if x == -1 or y == -1 or not self.inc_target_free(y):
            return False
        s = self.model.signals
        if not s[y].minibatched and (s[x].minibatched or a.minibatched):
            return False
        return self.commit(Operator.dot_inc(oid, SignalRef.full(a), SignalRef.full(s[x]), SignalRef.full(s[y])))

    def try_neurons(self, oid):
        n = 1 + self.pick(6)
        j = self.pick_signal(n, True, False)
        if j == -1:
            return False
        kind = self.rng.uniform()
        nk = NeuronKind.LIF if kind < 0.5 else (NeuronKind.LIFRate if kind < 0.75 else NeuronKind.RectifiedLinear)
        nm = NeuronModel(nk, amplitude=1.0 if self.rng.uniform() < 0.5 else 2.0)
        out = self.add_signal([n], False, True)
        states = []
        if nm.has_state():
            v = self.add_signal([n], False, True)
            r = self.add_signal([n], False, True)
            states = [SignalRef.full(self.model.signals[v]), SignalRef.full(self.model.signals[r])]
        s = self.model.signals
        return self.commit(Operator.sim_neurons(oid, nm, SignalRef.full(s[j]), SignalRef.full(s[out]), states))

    def try_process(self, oid):
        n = 1 + self.pick(8)
        mb = self.rng.uniform() < 0.7
        inp = self.pick_signal(n, mb, not mb)
        if inp == -1:
            return False
        tau = 0.0 if self.rng.uniform() < 0.25 else self.rng.uniform(0.002, 0.1)
        out = self.add_signal([n], False, mb)
        state = None
        if tau > 0.0:
            st = self.add_signal([n], False, mb)
            state = SignalRef.full(self.model.signals[st])
        s = self.model.signals
        return self.commit(Operator.sim_process(oid, tau, SignalRef.full(s[inp]), SignalRef.full(s[out]), state))

    def try_pes(self, oid):
        n = 1 + self.pick(5)
        r = 1 + self.pick(3)
        pre = self.pick_signal(n, True, False)
        err = self.pick_signal(r, True, False)
        if pre == -1 or err == -1:
            return False
        w = self.add_signal([r, n], False, False, self.random_values(r * n, -0.1, 0.1))
        s = self.model.signals
        return self.commit(Operator.sim_pes(oid, self.rng.uniform(1e-4, 1e-2), SignalRef.full(s[pre]),
                                            SignalRef.full(s[err]), SignalRef.full(s[w])))

    def try_time(self, oid):
        if self.has_clock:
            return False
        step = self.add_signal([1], False, False)
        time = self.add_signal([1], False, False)
        s = self.model.signals
        ok = self.commit(Operator.time_update(oid, self.model.dt, SignalRef.full(s[step]), SignalRef.full(s[time])))
        self.has_clock = ok
        return ok

    def add_probes(self):
        candidates = [s.id for s in self.model.signals if not s.constant]
        want = 2 + self.pick(3)
        for key in range(want):
            if not candidates:
                break
            at = self.pick(len(candidates))
            sig = candidates.pop(at)
            self.model.probes.append(ir.ProbeRegistration(key, sig, f"p{key}"))


def random_model(seed: int, target_ops: int = 40) -> ir.BuiltModel:
    return RandomModelBuilder(seed).build(target_ops)
