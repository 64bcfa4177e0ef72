"""Fused vs generic executor on small BASELINE configs (GPU tool)."""
import sys, time
sys.path.insert(0, ".")
from paper_1805_11144_b200 import networks, passes
from paper_1805_11144_b200.engine import GpuEngine, MODE_GENERIC, MODE_FUSED
for w in (networks.config0(steps=1000), networks.config2(steps=200)):
  pm = passes.run_passes(w.model)
  for mode in (MODE_FUSED, MODE_GENERIC):
    g = GpuEngine(pm, w.batch, mode=mode)
    g.run(w.steps, w.feeds); g.reset()
    t = time.time(); g.run(w.steps, w.feeds); dt = (time.time() - t) / w.steps
    print(w.name, "mode", mode, f"{dt*1e6:.1f} us/step")
