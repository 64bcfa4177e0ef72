"""Cache the REFERENCE planner's plan for the config-4 network (test / baseline
infrastructure, not product).

The reference's own run_passes (proj/src/passes.cpp:663-694, compiled unchanged
into oracle/_ref/libneng_ref.so) plans the 78,849-operator config-4 graph in
~7 minutes on one core, too long to repeat inside a bench run.  This script runs
it once and stores its output (plan groups, buffer assignment, statistics) in
oracle/plans/config4_ref_plan.npz together with a fingerprint of the model it
planned.  bench.py's reference arm and cpu_baseline load it, so the CPU
baseline runs the reference's EngineCore on the reference's own plan;
tests/test_planner.py checks that the repo's planner produces the same plan.

    python oracle/make_ref_plan.py        (needs /root/reference: builds oracle/_ref)
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PLAN_PATH = os.path.join(ROOT, "oracle", "plans", "config4_ref_plan.npz")


def config4_model():
    from paper_1805_11144_b200 import networks
    return networks.random_network(1, 2048, 512, 8, 8, 256, 1, 1, name="config4_random_2048x512").model


def fingerprint(model) -> str:
    """Hash of the operator graph's structure and values (what the planner sees)."""
    h = hashlib.sha256()
    for s in model.signals:
        h.update(repr((s.id, tuple(s.shape), int(s.elem), s.constant, s.minibatched, s.trainable)).encode())
        if s.initial is not None:
            h.update(np.ascontiguousarray(s.initial, dtype=np.float64).tobytes())
    for op in model.operators:
        h.update(repr((op.id, int(op.kind), [(r.signal, r.start, r.stop) for r in op.operands], op.inc)).encode())
        if op.value is not None and len(op.value):
            h.update(np.ascontiguousarray(op.value, dtype=np.float64).tobytes())
    return h.hexdigest()


def save(pm, model_fp, path=PLAN_PATH, seconds=0.0):
    offs = np.cumsum([0] + [len(g) for g in pm.plan]).astype(np.int64)
    mem = np.array([m for g in pm.plan for m in g], dtype=np.int32)
    bufs = pm.buffers.buffers
    tr_off = np.cumsum([0] + [len(b.trailing) for b in bufs]).astype(np.int64)
    ord_off = np.cumsum([0] + [len(b.order) for b in bufs]).astype(np.int64)
    np.savez_compressed(
        path, fingerprint=np.array(model_fp), plan_offsets=offs, plan_members=mem,
        buffer_of=np.array(pm.buffers.buffer_of, dtype=np.int32),
        row_offset=np.array(pm.buffers.row_offset, dtype=np.int32),
        buf_meta=np.array([[int(b.elem), int(b.minibatched), int(b.trainable), b.rows] for b in bufs], dtype=np.int64),
        buf_trailing=np.array([t for b in bufs for t in b.trailing], dtype=np.int32), buf_trailing_off=tr_off,
        buf_order=np.array([o for b in bufs for o in b.order], dtype=np.int32), buf_order_off=ord_off,
        stats=np.array([pm.stats.contiguous_read_fraction, pm.stats.gather_row_count, pm.stats.groups_per_step]),
        plan_seconds=np.array(seconds))


def load(model, path=PLAN_PATH):
    """The cached reference plan attached to `model` (which must match its fingerprint)."""
    from paper_1805_11144_b200 import ir
    z = np.load(path)
    if str(z["fingerprint"]) != fingerprint(model):
        raise ValueError(f"{path}: planned for a different model")
    offs, mem = z["plan_offsets"], z["plan_members"]
    plan = [mem[offs[i]:offs[i + 1]].tolist() for i in range(len(offs) - 1)]
    bufs = []
    for i, (elem, mb, tr, rows) in enumerate(z["buf_meta"].tolist()):
        trailing = z["buf_trailing"][z["buf_trailing_off"][i]:z["buf_trailing_off"][i + 1]].tolist()
        order = z["buf_order"][z["buf_order_off"][i]:z["buf_order_off"][i + 1]].tolist()
        bufs.append(ir.BufferDesc(trailing, ir.Elem(elem), bool(mb), bool(tr), rows, order))
    ba = ir.BufferAssignment(z["buffer_of"].tolist(), z["row_offset"].tolist(), bufs)
    st = z["stats"].tolist()
    return ir.PlannedModel(model, plan, ba, ir.ContiguityStats(st[0], int(st[1]), int(st[2]))), float(z["plan_seconds"])


def main():
    from oracle import refapi
    model = config4_model()
    t0 = time.time()
    ref = refapi.run_passes(model)  # the reference's planner (simplify, merge, layout)
    secs = time.time() - t0
    pm = ref.to_python()
    # the reference plans the model it is given; its simplify pass leaves this graph unchanged
    if len(pm.model.operators) != len(model.operators) or fingerprint(pm.model) != fingerprint(model):
        raise SystemExit("reference simplify changed the config-4 model; the cache format assumes it does not")
    os.makedirs(os.path.dirname(PLAN_PATH), exist_ok=True)
    save(pm, fingerprint(model), seconds=secs)
    print(f"reference plan: {len(pm.plan)} groups, {len(pm.buffers.buffers)} buffers, {secs:.0f} s -> {PLAN_PATH}")


if __name__ == "__main__":
    main()
