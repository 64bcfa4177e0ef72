"""The one-CTA fused step (fused_small_kernel): programs too small to fill the
GPU — config 0's single 800-neuron ensemble at batch 1, small ensemble
networks at batch < 32 — run the whole step on one CTA with lanes over
neurons.  Same bar as the multi-CTA pipeline: every probe and every signal of
every batch row bit-identical to the reference EngineCore<float>."""
import numpy as np
import pytest

from oracle import refapi
from paper_1805_11144_b200 import networks, passes
from paper_1805_11144_b200.engine import MODE_FUSED, SCHED_FUSED_SMALL, GpuEngine
from tests.support.models import assert_bitexact, step_slice
from tests.test_fused import full_state_equal, probe_rich_network, small_network

pytestmark = pytest.mark.gpu


def test_config0_auto_picks_the_one_cta_step():
    w = networks.config0(steps=1000)
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch)
    assert gpu.mode() == MODE_FUSED
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, w.feeds), ref.run(w.steps, w.feeds), "config0 small")
    assert gpu.last_schedule() == SCHED_FUSED_SMALL
    full_state_equal(gpu, ref, pm.model, w.batch, "config0 small")


@pytest.mark.parametrize("batch", [1, 4, 33])
def test_small_networks_full_state(batch, monkeypatch):
    monkeypatch.setenv("NENG_FUSED_SMALL", "1")  # batch 33 would otherwise take the multi-CTA pipeline
    w = small_network(seed=7, batch=batch, steps=25)
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch)
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, w.feeds), ref.run(w.steps, w.feeds), f"small B={batch}")
    assert gpu.last_schedule() == SCHED_FUSED_SMALL
    full_state_equal(gpu, ref, pm.model, w.batch, f"small B={batch}")


def test_calls_launches_and_reset():
    w = small_network(seed=5, batch=3, steps=24)
    pm = passes.run_passes(w.model)
    ref = refapi.RefEngine(pm, w.batch)
    whole = ref.run(24, w.feeds)
    gpu = GpuEngine(pm, w.batch)
    head = gpu.run(10, step_slice(w.feeds, 0, 10))
    tail = gpu.run(14, step_slice(w.feeds, 10, 14))
    for k in whole:
        assert np.array_equal(np.concatenate([head[k], tail[k]], axis=1).view(np.uint64), whole[k].view(np.uint64))
    full_state_equal(gpu, ref, pm.model, w.batch, "two calls")
    gpu.reset()
    assert_bitexact(gpu.run(24, w.feeds), whole, "after reset")
    k3 = GpuEngine(pm, w.batch, steps_per_launch=3)
    assert_bitexact(k3.run(24, w.feeds), whole, "3 steps per launch")


def test_captures_orphans_and_clock(monkeypatch):
    monkeypatch.setenv("NENG_FUSED_SMALL", "1")
    w = probe_rich_network(batch=5)
    pm = passes.run_passes(w.model)
    node2 = max(w.feeds)
    calls = [(11, step_slice(w.feeds, 0, 11)),
             (15, {k: v for k, v in step_slice(w.feeds, 11, 15).items() if k != node2})]
    gpu = GpuEngine(pm, w.batch)
    ref = refapi.RefEngine(pm, w.batch)
    for i, (n, f) in enumerate(calls):
        assert_bitexact(gpu.run(n, f), ref.run(n, f), f"call {i}")
        assert gpu.last_schedule() == SCHED_FUSED_SMALL
        full_state_equal(gpu, ref, pm.model, w.batch, f"call {i}")


def test_neuron_state_probes(monkeypatch):
    monkeypatch.setenv("NENG_FUSED_SMALL", "1")
    w = networks.random_network(13, n_ens=6, n=80, d=4, k_out=2, n_inputs=3, batch=6, steps=19)
    m = w.model
    lab = {s.label: s.id for s in m.signals}
    from tests.support.device import add_probes
    add_probes(m, [(lab["ens1.out"], "spikes"), (lab["ens1.voltage"], "v"), (lab["ens2.refractory"], "r"),
                   (lab["ens3.J"], "J")])
    pm = passes.run_passes(m)
    gpu = GpuEngine(pm, w.batch)
    ref = refapi.RefEngine(pm, w.batch)
    out = gpu.run(w.steps, w.feeds)
    assert_bitexact(out, ref.run(w.steps, w.feeds), "state probes")
    assert np.count_nonzero(out[pm.model.probes[-4].key]) > 0
    full_state_equal(gpu, ref, pm.model, w.batch, "state probes")


def test_wide_fed_connections_projected(monkeypatch):
    # fed-node connections wider than the fused rows are projected ahead of each launch
    # (FProj) and read through an identity transform; a second call takes the defaults
    monkeypatch.setenv("NENG_FUSED_SMALL", "1")
    w = networks.config1(steps=25, batch=3, dims=40)
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch, mode=MODE_FUSED)
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, w.feeds), ref.run(w.steps, w.feeds), "projected feeds")
    assert gpu.last_schedule() == SCHED_FUSED_SMALL
    full_state_equal(gpu, ref, pm.model, w.batch, "projected feeds")
    assert_bitexact(gpu.run(7), ref.run(7), "default node values")
    full_state_equal(gpu, ref, pm.model, w.batch, "default node values")


def test_stepped_calls_match_run_device(monkeypatch):
    # the stepped call (begin / step k / epilogue / end) on the one-CTA step leaves the
    # same probe ring as one run_device call
    monkeypatch.setenv("NENG_FUSED_SMALL", "1")
    import torch
    from paper_1805_11144_b200.engine import STEP_EPILOGUE, STEP_FIRST_UPDATE
    from tests.support.device import device_feeds, device_ring
    dev = torch.device("cuda", 0)
    w = small_network(seed=2, batch=2, steps=12)
    pm = passes.run_passes(w.model)
    n, B = w.steps, w.batch
    ts = torch.cuda.Stream(dev)
    with torch.cuda.stream(ts):
        feeds, fptrs = device_feeds(w, n, dev)
        whole = GpuEngine(pm, B)
        ring_w, rptrs_w, _ = device_ring(pm.model, n, B, dev)
        whole.run_device(n, fptrs, rptrs_w, ts.cuda_stream)
        stepped = GpuEngine(pm, B)
        ring_s, rptrs_s, _ = device_ring(pm.model, n, B, dev)
        stepped.call_begin(n, fptrs, rptrs_s, ts.cuda_stream)
        for k in range(n):
            stepped.call_step(k, STEP_FIRST_UPDATE if k else 0)
        stepped.call_step(n, STEP_EPILOGUE)
        stepped.call_end()
        torch.cuda.synchronize(dev)
    assert stepped.last_schedule() & SCHED_FUSED_SMALL
    assert torch.equal(ring_w.view(torch.int32), ring_s.view(torch.int32))
    ref = refapi.RefEngine(pm, B)
    ref.run(n, w.feeds)
    full_state_equal(stepped, ref, pm.model, B, "stepped")
