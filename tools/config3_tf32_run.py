"""Config 3 at B=512 in TF32 mode for profiling: warm-up call, then 10 steps."""
import sys
sys.path.insert(0, ".")
from paper_1805_11144_b200 import networks, passes  # noqa: E402
from paper_1805_11144_b200.engine import GpuEngine, PRECISION_TF32, PRECISION_STRICT_FP32  # noqa: E402
prec = PRECISION_TF32 if (len(sys.argv) < 2 or sys.argv[1] == "tf32") else PRECISION_STRICT_FP32
w = networks.config3(steps=10, batch=512)
pm = passes.run_passes(w.model)
e = GpuEngine(pm, 512, precision=prec)
e.run(10, w.feeds)
e.run(10, w.feeds)
