"""Config 1 (circular convolution, 64 dims, B=64) at full size on the GPU vs the
reference EngineCore<float>: bit-exact probes and sampled full state, plus
steps/s.  (Planning takes minutes, so this is a script, not a test.)"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import refapi  # noqa: E402
from paper_1805_11144_b200 import networks, passes  # noqa: E402
from paper_1805_11144_b200.engine import GpuEngine  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
w = networks.config1(steps=steps, batch=64, dims=64)
t = time.time()
pm = passes.run_passes(w.model)
print(f"config1: {len(w.model.operators)} ops, {len(pm.plan)} groups, planned in {time.time() - t:.1f} s", flush=True)
gpu = GpuEngine(pm, w.batch)
ref = refapi.RefEngine(pm, w.batch)
t = time.time()
out = gpu.run(w.steps, w.feeds)
tg = time.time() - t
t = time.time()
r = ref.run(w.steps, w.feeds)
tr = time.time() - t
same = all(np.array_equal(out[k].view(np.uint64), r[k].view(np.uint64)) for k in r)
bad = 0
for s in pm.model.signals[::37]:
    for b in (0, w.batch - 1):
        bad += not np.array_equal(gpu.read_signal(s.id, b).view(np.uint64), ref.read_signal(s.id, b).view(np.uint64))
print(f"mode {gpu.mode()}: probes bit-exact {same}, sampled signals differing {bad}; "
      f"gpu {tg * 1e3 / steps:.3f} ms/step (host I/O incl.), reference {tr * 1e3 / steps:.1f} ms/step")
