"""Config 2 steps/s through neng_gpu_run (GPU tool; env knobs via the caller)."""
import sys, time, os
sys.path.insert(0, ".")
from paper_1805_11144_b200 import networks, passes
from paper_1805_11144_b200.engine import GpuEngine
w = networks.config2(steps=300)
pm = passes.run_passes(w.model)
g = GpuEngine(pm, w.batch)
g.run(w.steps, w.feeds); g.reset()
t = time.time(); g.run(w.steps, w.feeds); dt = (time.time() - t) / w.steps
print(os.environ.get("TAG", ""), f"config2 {dt*1e6:.1f} us/step")
