"""Fused ensemble pipeline parity: the fused kernel must leave every signal of
every batch row bit-identical to the reference EngineCore<float> after every
run() call (not only the probes), on the BASELINE workloads."""
import numpy as np
import pytest

from oracle import refapi
from paper_1805_11144_b200 import networks, passes
from paper_1805_11144_b200.engine import (MODE_FUSED, MODE_GENERIC, SCHED_BARRIER_FREE, SCHED_FUSED_STEPPED,
                                          GpuEngine)
from tests.support.device import device_feeds, device_ring
from tests.support.models import assert_bitexact, batch_slice, step_slice

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def multi_cta_pipeline(monkeypatch):
    # these tests cover the multi-CTA fused kernel; tests/test_fused_small.py runs the
    # one-CTA step that AUTO picks for programs too small to fill the GPU
    monkeypatch.setenv("NENG_FUSED_SMALL", "0")


def full_state_equal(gpu, ref, model, batch, context):
    for s in model.signals:
        for b in {0, batch - 1}:
            g, r = gpu.read_signal(s.id, b), ref.read_signal(s.id, b)
            if not np.array_equal(g.view(np.uint64), r.view(np.uint64)):
                i = int(np.argmax(g.view(np.uint64) != r.view(np.uint64)))
                raise AssertionError(f"{context}: signal {s.label} row {b} elem {i}: {g[i]!r} vs {r[i]!r}")


def small_network(seed=3, batch=4, steps=30):
    return networks.random_network(seed, n_ens=8, n=64, d=4, k_out=3, n_inputs=3, batch=batch, steps=steps)


def test_small_network_fused_bit_exact_full_state():
    w = small_network()
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch)
    assert gpu.mode() == MODE_FUSED
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, w.feeds), ref.run(w.steps, w.feeds), "small fused")
    full_state_equal(gpu, ref, pm.model, w.batch, "small fused")


def test_fused_matches_generic_and_persists_across_calls():
    w = small_network(seed=5, batch=33, steps=24)  # partial batch tile
    pm = passes.run_passes(w.model)
    fused, generic = GpuEngine(pm, w.batch), GpuEngine(pm, w.batch, mode=MODE_GENERIC)
    assert fused.mode() == MODE_FUSED and generic.mode() == MODE_GENERIC
    head = fused.run(10, step_slice(w.feeds, 0, 10))
    tail = fused.run(14, step_slice(w.feeds, 10, 14))
    whole = generic.run(24, w.feeds)
    for k in whole:
        assert np.array_equal(np.concatenate([head[k], tail[k]], axis=1).view(np.uint64), whole[k].view(np.uint64))
    fused.reset()
    assert_bitexact(fused.run(24, w.feeds), whole, "after reset")
    k3 = GpuEngine(pm, w.batch, steps_per_launch=3)
    assert_bitexact(k3.run(24, w.feeds), whole, "3 steps per launch")


def test_config0_integrator_bit_exact():
    w = networks.config0(steps=1000)
    pm = passes.run_passes(w.model)
    assert GpuEngine(pm, w.batch).mode() == MODE_GENERIC  # one unit per step: AUTO keeps the interpreter
    gpu = GpuEngine(pm, w.batch, mode=MODE_FUSED)
    assert gpu.mode() == MODE_FUSED
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, w.feeds), ref.run(w.steps, w.feeds), "config0")
    full_state_equal(gpu, ref, pm.model, w.batch, "config0")


def test_config2_shape_bit_exact():
    # config 2 geometry (256 x 1024 LIF, d=16, K=4, 32 inputs); batch and steps reduced for the CPU reference
    w = networks.random_network(1, 256, 1024, 16, 4, 32, batch=2, steps=12, name="config2_small")
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch)
    assert gpu.mode() == MODE_FUSED
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, w.feeds), ref.run(w.steps, w.feeds), "config2")
    full_state_equal(gpu, ref, pm.model, w.batch, "config2")


def test_config4_full_batch_sampled_rows_bit_exact():
    # full config-4 geometry and batch (2048 x 512, d=8, K=8, 256 inputs, B=256) on the GPU;
    # batch rows are independent (test_exec.cpp:246-267) so rows 0 and 255 are checked against
    # solo reference engines fed the same row.
    w = networks.config4(steps=6)
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch)
    assert gpu.mode() == MODE_FUSED
    out = gpu.run(w.steps, w.feeds)
    for b in (0, w.batch - 1):
        solo = refapi.RefEngine(pm, 1)
        ref = solo.run(w.steps, batch_slice(w.feeds, b))
        for k in ref:
            assert np.array_equal(out[k][b:b + 1].view(np.uint64), ref[k].view(np.uint64)), f"row {b} probe {k}"
        for s in pm.model.signals[::97]:
            assert np.array_equal(gpu.read_signal(s.id, b).view(np.uint64), solo.read_signal(s.id, 0).view(np.uint64)), \
                f"row {b} signal {s.label}"


def test_two_ensemble_shards_match_the_unsharded_engine():
    # two shards of one network driven on one GPU (their launches never wait on each other;
    # the "all-gather" is a copy of each shard's xhat rows into the other's parity buffer)
    import torch

    dev = torch.device("cuda", 0)
    # probes on every ensemble's xhat, so both shards own some
    w = networks.random_network(11, n_ens=10, n=96, d=6, k_out=3, n_inputs=3, batch=64, steps=16, probes=10)
    pm = passes.run_passes(w.model)
    n, B = w.steps, w.batch
    ts = torch.cuda.Stream(dev)  # a real stream: the engine, the copies and the feeds must be ordered
    with torch.cuda.stream(ts):
        _two_shards_on_one_stream(pm, w, n, B, dev, ts.cuda_stream)


def _two_shards_on_one_stream(pm, w, n, B, dev, stream):
    import torch
    from paper_1805_11144_b200.engine import STEP_EPILOGUE, STEP_FIRST_UPDATE
    from paper_1805_11144_b200.shard import attach_xhat_buffer
    feeds, fptrs = device_feeds(w, n, dev)

    whole = GpuEngine(pm, B)
    ring_w, rptrs_w, offs = device_ring(pm.model, n, B, dev)
    whole.run_device(n, fptrs, rptrs_w, stream)

    shards = [GpuEngine(pm, B, shard=(r, 2)) for r in range(2)]
    xb = [attach_xhat_buffer(s, dev) for s in shards]
    rings = [device_ring(pm.model, n, B, dev) for _ in shards]
    for s, (ring, rptrs, _) in zip(shards, rings):
        s.call_begin(n, fptrs, rptrs, stream)
    rf = xb[0][1]
    half = xb[0][0].numel() // 2
    for k in range(n):
        for s in shards:
            s.call_step(k, STEP_FIRST_UPDATE if k else 0)
        h = (k & 1) * half
        for r in range(2):  # shard r's rows into the other shard's buffer
            src = xb[r][0][h + r * rf:h + (r + 1) * rf]
            xb[1 - r][0][h + r * rf:h + (r + 1) * rf].copy_(src)
    for s in shards:
        s.call_step(n, STEP_EPILOGUE)
    for s in shards:
        s.call_end()
    torch.cuda.synchronize(dev)

    # every probe is produced by exactly one shard: its trace equals the unsharded one
    owned = 0
    for (at, cnt) in offs:
        ref = ring_w[at:at + cnt].cpu().numpy().view(np.uint32)
        got = [rg[0][at:at + cnt].cpu().numpy() for rg in rings]
        mine = [g for g in got if not np.isnan(g).all()]
        assert len(mine) == 1
        assert np.array_equal(mine[0].view(np.uint32), ref)
        owned += 1
    assert owned == len(pm.model.probes)
    # neuron state of each shard's ensembles equals the unsharded engine's
    sig = {s.label: s.id for s in pm.model.signals}
    for e in range(10):
        owner = shards[0 if e < 5 else 1]
        for name in (f"ens{e}.voltage", f"ens{e}.refractory"):
            for b in (0, B - 1):
                assert np.array_equal(owner.read_signal(sig[name], b).view(np.uint64),
                                      whole.read_signal(sig[name], b).view(np.uint64)), (name, b)


def test_hard_driven_network_bit_exact_full_state():
    # inputs x30: most neurons fire at their maximum rate and spike again on the step they leave
    # the refractory period, so warp rows carry many lanes into the doubt queue at once (a pair
    # of rows can push 64 entries: the queue must drain to < 32 before the next pair)
    w = networks.random_network(9, n_ens=8, n=64, d=4, k_out=3, n_inputs=8, batch=64, steps=20)
    feeds = {k: 30.0 * v for k, v in w.feeds.items()}
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch)
    assert gpu.mode() == MODE_FUSED
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, feeds), ref.run(w.steps, feeds), "hard driven")
    full_state_equal(gpu, ref, pm.model, w.batch, "hard driven")


def probe_rich_network(seed=11, batch=40, steps=26):
    """Small ring network with every capture and connection kind the fused
    pipeline owns outside the units: a destination-less connection from an
    ensemble and one from a fed node (filt and state probes), two probes on one
    xhat, a fed-node probe and the clock's step/time probes."""
    nb = networks.NetBuilder(seed)
    rng = np.random.default_rng(seed)
    ens = [nb.ensemble(48, 3) for _ in range(6)]
    xs = [nb.decoded(e, rng.normal(0.0, 0.2, size=(3, 48))) for e in ens]
    for i in range(6):
        for j in (1, 3):
            nb.connect(xs[i], ens[(i + j) % 6].in_, rng.normal(0.0, 0.5, size=(3, 3)), synapse=0.01)
    node, u = nb.feedable_node(3, np.zeros(3))
    nb.connect(u, ens[0].in_, None, synapse=0.01)
    node2, u2 = nb.feedable_node(2, np.full(2, 0.25))
    po = nb.connect(xs[2], None, rng.normal(size=(2, 3)), synapse=0.02)
    pf = nb.connect(u2, None, None, synapse=0.005)
    nb.probe(po["filtered"], "orphan.filt")
    nb.probe(po["state"], "orphan.state")
    nb.probe(pf["filtered"], "fed_orphan.filt")
    nb.probe(xs[4], "x4a")
    nb.probe(xs[4], "x4b")
    nb.probe(u, "feed")
    nb.probe(0, "step")
    nb.probe(1, "time")
    feeds = {node: rng.standard_normal((batch, steps, 3)), node2: rng.standard_normal((batch, steps, 2))}
    return networks.Workload("probe_rich", nb.m, batch, steps, feeds, 6 * 48)


@pytest.mark.parametrize("dataflow", ["1", "0"])
def test_captures_and_orphans_both_schedules(dataflow, monkeypatch):
    # barrier-free stepping (default) and one barrier per step: captures, orphan
    # connections, the clock and call boundaries (second call without node2's feed)
    monkeypatch.setenv("NENG_FUSED_DATAFLOW", dataflow)
    w = probe_rich_network()
    pm = passes.run_passes(w.model)
    node2 = max(w.feeds)
    calls = [(11, step_slice(w.feeds, 0, 11)),
             (15, {k: v for k, v in step_slice(w.feeds, 11, 15).items() if k != node2})]
    for spl in (0, 4):
        gpu = GpuEngine(pm, w.batch, steps_per_launch=spl)
        assert gpu.mode() == MODE_FUSED
        ref = refapi.RefEngine(pm, w.batch)
        for i, (n, f) in enumerate(calls):
            assert_bitexact(gpu.run(n, f), ref.run(n, f), f"dataflow={dataflow} spl={spl} call {i}")
            # fed calls longer than 4 steps stage their feeds in chunks: each chunk keeps the schedule
            assert gpu.last_schedule() == (SCHED_BARRIER_FREE if dataflow == "1" else SCHED_FUSED_STEPPED)
            full_state_equal(gpu, ref, pm.model, w.batch, f"dataflow={dataflow} spl={spl} call {i}")


@pytest.mark.parametrize("mode", [MODE_FUSED, MODE_GENERIC])
def test_config1_cconv_geometry_bit_exact(mode):
    # config 1's circular-convolution structure at 16 dims (the full 64-dim graph's
    # 132-way input fan-in makes the planner the bottleneck, not the engine):
    # 36 two-D product ensembles fed by DFT projections, 16 one-D output ensembles
    # fed through the inverse DFT, constant inputs, batch 4
    w = networks.config1(steps=40, batch=4, dims=16)
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch, mode=mode)
    assert gpu.mode() == mode
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, w.feeds), ref.run(w.steps, w.feeds), "config1")
    full_state_equal(gpu, ref, pm.model, w.batch, "config1")


def test_wide_fed_connections_projected_ahead_of_the_kernel():
    # 40-D inputs: the DFT projections (2 x 40 transforms from fed nodes) exceed the fused
    # rows, so they are computed ahead of each launch and read through an identity
    # transform; a second call without feeds takes the nodes' default values from the arena
    w = networks.config1(steps=25, batch=3, dims=40)
    pm = passes.run_passes(w.model)
    gpu = GpuEngine(pm, w.batch, mode=MODE_FUSED)
    ref = refapi.RefEngine(pm, w.batch)
    assert_bitexact(gpu.run(w.steps, w.feeds), ref.run(w.steps, w.feeds), "projected feeds")
    full_state_equal(gpu, ref, pm.model, w.batch, "projected feeds")
    assert_bitexact(gpu.run(7), ref.run(7), "default node values")
    full_state_equal(gpu, ref, pm.model, w.batch, "default node values")


@pytest.mark.parametrize("dataflow", ["1", "0"])
def test_neuron_state_probes_stay_fused(dataflow, monkeypatch):
    # probes on an ensemble's spikes, voltage, refractory state and input current are
    # captured by the unit that steps it (the fused pipeline keeps the graph)
    monkeypatch.setenv("NENG_FUSED_DATAFLOW", dataflow)
    w = networks.random_network(13, n_ens=6, n=80, d=4, k_out=2, n_inputs=3, batch=40, steps=19)
    m = w.model
    lab = {s.label: s.id for s in m.signals}
    from tests.support.device import add_probes
    add_probes(m, [(lab["ens1.out"], "spikes"), (lab["ens1.voltage"], "v"), (lab["ens2.refractory"], "r"),
                   (lab["ens3.J"], "J"), (lab["ens1.out"], "spikes again")])
    pm = passes.run_passes(m)
    gpu = GpuEngine(pm, w.batch)
    assert gpu.mode() == MODE_FUSED
    ref = refapi.RefEngine(pm, w.batch)
    for i, (a, n) in enumerate(((0, 12), (12, 7))):
        f = step_slice(w.feeds, a, n)
        out = gpu.run(n, f)
        assert_bitexact(out, ref.run(n, f), f"state probes call {i}")
        assert np.count_nonzero(out[pm.model.probes[-5].key]) > 0  # the spike probe saw spikes
    full_state_equal(gpu, ref, pm.model, w.batch, "state probes")
