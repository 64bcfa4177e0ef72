"""Steps/s of BASELINE configs 0, 2 and 4 (one call through neng_gpu_run, host f64 feeds,
after a warm-up call of the same size) next to the reference EngineCore<float> on one
host core for a short window (GPU tool; parity is in tests/)."""
import sys
import time

sys.path.insert(0, ".")
from oracle import refapi  # noqa: E402
from paper_1805_11144_b200 import networks, passes  # noqa: E402
from paper_1805_11144_b200.engine import GpuEngine  # noqa: E402

for name, w, ref_steps in (("config0", networks.config0(steps=1000), 200),
                           ("config2", networks.config2(steps=1000), 10)):
    pm = passes.run_passes(w.model)
    g = GpuEngine(pm, w.batch)
    g.run(w.steps, w.feeds)
    g.reset()
    t = time.time()
    g.run(w.steps, w.feeds)
    tg = (time.time() - t) / w.steps
    r = refapi.RefEngine(pm, w.batch)
    fe = {k: v[:, :ref_steps] for k, v in w.feeds.items()}
    t = time.time()
    r.run(ref_steps, fe)
    tr = (time.time() - t) / ref_steps
    nu = networks.neuron_count(w.model) * w.batch
    print(f"{name}: mode {g.mode()}, B={w.batch}: GPU {tg * 1e6:.1f} us/step ({nu / tg / 1e9:.2f} G n-u/s), "
          f"reference 1 core {tr * 1e3:.2f} ms/step ({nu / tr / 1e9:.4f} G n-u/s)", flush=True)
