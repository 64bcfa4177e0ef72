"""Config 1 geometry at 32 dims on the generic executor: us/step (GPU tool; NENG_GENERIC_GRID from the caller)."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_1805_11144_b200 import networks, passes  # noqa: E402
from paper_1805_11144_b200.engine import MODE_GENERIC, GpuEngine  # noqa: E402

w = networks.config1(steps=200, batch=64, dims=32)
pm = passes.run_passes(w.model)
g = GpuEngine(pm, w.batch, mode=MODE_GENERIC)
g.run(w.steps, w.feeds)
g.reset()
t = time.time()
g.run(w.steps, w.feeds)
print(os.environ.get("NENG_GENERIC_GRID", "default"), f"{(time.time() - t) / w.steps * 1e6:.1f} us/step", flush=True)
