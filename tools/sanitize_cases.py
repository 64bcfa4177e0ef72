"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the fused pipeline under both schedules, the generic
interpreter, and the tcgen05 DotInc (TF32, BF16X3).  Each case is checked
against the reference EngineCore<float> (or the strict path), so a sanitizer
run also re-proves parity on these inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import refapi  # noqa: E402
from paper_1805_11144_b200 import networks, passes  # noqa: E402
from paper_1805_11144_b200.engine import (MODE_FUSED, MODE_GENERIC, PRECISION_BF16X3, PRECISION_TF32,  # noqa: E402
                                          SCHED_BARRIER_FREE, SCHED_FUSED_STEPPED, GpuEngine, tc_dot)


def same(a, b):
    return all(np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)) for k in b)


w = networks.random_network(3, n_ens=8, n=64, d=4, k_out=3, n_inputs=3, batch=40, steps=12)
pm = passes.run_passes(w.model)
ref = refapi.RefEngine(pm, w.batch).run(w.steps, w.feeds)
for df in ("1", "0"):
    os.environ["NENG_FUSED_DATAFLOW"] = df
    g = GpuEngine(pm, w.batch, mode=MODE_FUSED)
    out = g.run(w.steps, w.feeds)
    sched = "barrier-free" if g.last_schedule() & SCHED_BARRIER_FREE else (
        "stepped" if g.last_schedule() & SCHED_FUSED_STEPPED else "?")
    print(f"fused dataflow={df} ({sched}):", "OK" if same(out, ref) else "MISMATCH", flush=True)
os.environ.pop("NENG_FUSED_DATAFLOW")
g = GpuEngine(pm, w.batch, mode=MODE_GENERIC)
print("generic:", "OK" if same(g.run(w.steps, w.feeds), ref) else "MISMATCH", flush=True)

w3 = networks.config3(steps=4, batch=64)
pm3 = passes.run_passes(w3.model)
strict = GpuEngine(pm3, w3.batch).run(w3.steps, w3.feeds)
for prec, name in ((PRECISION_TF32, "tf32"), (PRECISION_BF16X3, "bf16x3")):
    out = GpuEngine(pm3, w3.batch, precision=prec).run(w3.steps, w3.feeds)
    (k,) = list(strict)
    rel = np.linalg.norm(out[k] - strict[k]) / max(np.linalg.norm(strict[k]), 1e-30)
    print(f"config3 {name}: rel L2 vs strict {rel:.2e}", flush=True)
a = np.random.default_rng(1).uniform(-1, 1, (130, 40)).astype(np.float32)
x = np.random.default_rng(2).uniform(0, 1, (40, 96)).astype(np.float32)
y, _ = tc_dot(a, x, np.zeros((130, 96), np.float32), PRECISION_TF32)
print("tc_dot tf32 max err", float(np.abs(y - a.astype(np.float64) @ x).max()), flush=True)
