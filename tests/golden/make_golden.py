"""Generate the golden fixtures in tests/golden/ from the reference itself.

Each fixture is a planned model (planned by the reference's run_passes), its
feeds, and the probe traces produced by the reference's EngineCore<float>
(oracle/_ref, compiled from the unmodified reference sources).  The fixtures
let the CPU suite pin the C port and the GPU suite pin the device engine on a
box where /root/reference (and even oracle/_ref) is absent.

    python tests/golden/make_golden.py        # rewrites tests/golden/*.npz
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1805_11144_b200 import ir  # noqa: E402


def planned_to_json(pm: ir.PlannedModel) -> str:
    m = pm.model
    return json.dumps({
        "dt": m.dt,
        "signals": [[s.id, s.label, s.shape, int(s.elem), None if s.initial is None else [float(v) for v in s.initial],
                     s.constant, s.minibatched, s.trainable] for s in m.signals],
        "operators": [[o.id, int(o.kind), [[r.signal, r.start, r.stop] for r in o.operands],
                       None if o.value is None else [float(v) for v in o.value], o.inc,
                       [int(o.neuron.kind), o.neuron.tau_rc, o.neuron.tau_ref, o.neuron.amplitude],
                       o.tau, o.learning_rate, o.dt] for o in m.operators],
        "probes": [[p.key, p.signal, p.label] for p in m.probes],
        "feed_slots": [[f.node_id, f.signal, f.dim, f.has_default, f.label] for f in m.feed_slots],
        "plan": pm.plan,
        "buffer_of": pm.buffers.buffer_of, "row_offset": pm.buffers.row_offset,
        "buffers": [[b.trailing, int(b.elem), b.minibatched, b.trainable, b.rows, b.order] for b in pm.buffers.buffers],
    })


def planned_from_json(text: str) -> ir.PlannedModel:
    d = json.loads(text)
    m = ir.BuiltModel(dt=d["dt"])
    for sid, label, shape, elem, init, const, mb, tr in d["signals"]:
        m.signals.append(ir.Signal(sid, label, shape, ir.Elem(elem), None if init is None else np.array(init),
                                   const, mb, tr))
    for oid, kind, refs, value, inc, nm, tau, lr, dt in d["operators"]:
        m.operators.append(ir.Operator(oid, ir.OpKind(kind), [ir.SignalRef(*r) for r in refs],
                                       None if value is None else np.array(value), inc,
                                       ir.NeuronModel(ir.NeuronKind(nm[0]), nm[1], nm[2], nm[3]), tau, lr, dt))
    m.probes = [ir.ProbeRegistration(*p) for p in d["probes"]]
    m.feed_slots = [ir.FeedSlot(*f) for f in d["feed_slots"]]
    bufs = [ir.BufferDesc(t, ir.Elem(e), mb, tr, rows, order) for t, e, mb, tr, rows, order in d["buffers"]]
    return ir.PlannedModel(m, d["plan"], ir.BufferAssignment(d["buffer_of"], d["row_offset"], bufs))


def save_case(path, planned, batch, steps, feeds, probes):
    arrays = {"planned": np.frombuffer(planned_to_json(planned).encode(), dtype=np.uint8),
              "meta": np.array([batch, steps])}
    for k, v in (feeds or {}).items():
        arrays[f"feed_{k}"] = v
    for k, v in probes.items():
        arrays[f"probe_{k}"] = v
    np.savez_compressed(path, **arrays)


def load_case(path):
    z = np.load(path)
    planned = planned_from_json(bytes(z["planned"]).decode())
    batch, steps = (int(x) for x in z["meta"])
    feeds = {int(k[5:]): z[k] for k in z.files if k.startswith("feed_")}
    probes = {int(k[6:]): z[k] for k in z.files if k.startswith("probe_")}
    return planned, batch, steps, feeds, probes


def main():
    from oracle import refapi
    from paper_1805_11144_b200 import networks
    from tests.support.models import chain_model, constant_drive_lif, learning_model, wave_feed
    from tests.support.random_models import random_model

    cases = []
    for seed in (1, 2, 3):
        cases.append((f"random_seed{seed}", random_model(seed, 45), 3, 20, {}))
    cm, node, _ = chain_model()
    cases.append(("chain", cm, 2, 30, {node: wave_feed(2, 30, 2, 0.1)}))
    lm, nu, nt, _, _ = learning_model()
    cases.append(("learning", lm, 2, 25, {nu: wave_feed(2, 25, 2, 0.2), nt: wave_feed(2, 25, 2, -0.3)}))
    cases.append(("lif_drive", constant_drive_lif(2.0), 1, 130, {}))
    w = networks.random_network(5, n_ens=4, n=32, d=4, k_out=2, n_inputs=2, batch=4, steps=20)
    cases.append(("ensemble_network", w.model, w.batch, w.steps, w.feeds))
    for name, model, batch, steps, feeds in cases:
        rp = refapi.run_passes(model)
        pm = rp.to_python()
        probes = refapi.RefEngine(rp, batch).run(steps, feeds)
        save_case(os.path.join(HERE, f"{name}.npz"), pm, batch, steps, feeds, probes)
        print("wrote", name)


if __name__ == "__main__":
    main()
