"""Strict vs TF32 precision on BASELINE config 3 (spiking MLP): speed and output error (GPU tool)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from oracle import refapi
from paper_1805_11144_b200 import networks, passes
from paper_1805_11144_b200.engine import GpuEngine, PRECISION_TF32
for B, steps in ((32, 30), (512, 100)):
    w = networks.config3(steps=steps, batch=B)
    pm = passes.run_passes(w.model)
    strict = GpuEngine(pm, B)
    tc = GpuEngine(pm, B, precision=PRECISION_TF32)
    print("mode", strict.mode(), tc.mode())
    strict.run(steps, w.feeds); tc.run(steps, w.feeds)  # warm-up
    strict.reset(); tc.reset()
    t = time.time(); o_s = strict.run(steps, w.feeds); ts = time.time() - t
    t = time.time(); o_t = tc.run(steps, w.feeds); tt = time.time() - t
    k = list(o_s)[0]
    a, b = o_s[k], o_t[k]
    print(f"B={B} steps={steps}: strict {ts*1e3/steps:.3f} ms/step, tf32 {tt*1e3/steps:.3f} ms/step, launches {tc.last_launch_count()}")
    err = np.abs(a - b); scale = np.abs(a).max()
    print(f"  max |out| {scale:.4g}, max abs err {err.max():.4g}, rel-to-max {err.max()/scale:.4g}, rms rel {np.sqrt((err**2).mean())/np.sqrt((a**2).mean()):.4g}")
    tail = slice(steps // 2, None)
    print(f"  last-half mean per sample: rel L2 err {np.linalg.norm(a[:, tail].mean(1) - b[:, tail].mean(1)) / np.linalg.norm(a[:, tail].mean(1)):.4g}")
    if B == 32:
        ref = refapi.RefEngine(pm, B).run(steps, w.feeds)
        print("  strict == reference:", np.array_equal(ref[k].view(np.uint64), a.view(np.uint64)))
