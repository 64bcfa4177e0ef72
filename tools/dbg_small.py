"""Run the small fused network once (debug aid for compute-sanitizer)."""
import sys
sys.path.insert(0, ".")
from tests.test_fused import small_network
from paper_1805_11144_b200 import passes
from paper_1805_11144_b200.engine import GpuEngine

w = small_network()
pm = passes.run_passes(w.model)
g = GpuEngine(pm, w.batch)
print("mode", g.mode())
out = g.run(w.steps, w.feeds)
print("ok", sum(float(abs(v).sum()) for v in out.values()))
