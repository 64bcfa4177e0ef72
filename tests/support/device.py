"""GPU-side fixtures: device-resident feed blocks and probe rings for
GpuEngine.run_device / call_begin (the layouts neng_gpu.h documents), solo
reference engines for sampled batch rows, and the spike-count comparison the
north star states its tolerance in."""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from paper_1805_11144_b200 import ir
from tests.support.models import batch_slice


def device_feeds(w, steps, dev):
    """w.feeds ([batch][steps][dim] f64 per node) as one packed [slot][step][dim][B] f32 block."""
    import torch
    blocks = []
    for fs in w.model.feed_slots:
        f = w.feeds[fs.node_id][:, :steps, :]
        blocks.append(torch.as_tensor(np.ascontiguousarray(f.transpose(1, 2, 0)), dtype=torch.float32).reshape(-1))
    flat = torch.cat(blocks).to(dev) if blocks else torch.zeros(1, device=dev)
    ptrs, at = [], 0
    for fs in w.model.feed_slots:
        ptrs.append(flat.data_ptr() + 4 * at)
        at += steps * fs.dim * w.batch
    return flat, ptrs


def device_ring(model, steps, batch, dev):
    """A NaN-filled probe ring [probe][step][dim][B] f32; returns (ring, per-probe pointers, (offset, count))."""
    import torch
    dims = [model.signals[p.signal].size() for p in model.probes]
    ring = torch.full((max(sum(dims) * steps * batch, 1),), float("nan"), device=dev)
    ptrs, offs, at = [], [], 0
    for d in dims:
        ptrs.append(ring.data_ptr() + 4 * at)
        offs.append((at, d * steps * batch))
        at += d * steps * batch
    return ring, ptrs, offs


def ring_rows(ring, offs, model, steps, batch, rows):
    """Per probe key: the ring's traces of batch rows `rows` as [len(rows)][steps][dim] f32 (host)."""
    import torch
    idx = torch.as_tensor(list(rows), device=ring.device)
    out = {}
    for p, (at, cnt) in zip(model.probes, offs):
        dim = model.signals[p.signal].size()
        t = ring[at:at + cnt].view(steps, dim, batch).index_select(2, idx)  # [steps][dim][rows]
        out[p.key] = t.permute(2, 0, 1).contiguous().cpu().numpy()
    return out


def add_probes(model: ir.BuiltModel, signals_and_labels):
    """Register extra probes (keys after the existing ones); returns their keys."""
    keys = []
    for sig, label in signals_and_labels:
        key = max([p.key for p in model.probes], default=-1) + 1
        model.probes.append(ir.ProbeRegistration(key, sig, label))
        keys.append(key)
    return keys


def solo_reference_rows(refapi, pm, feeds, rows, steps, signals=(), threads=8):
    """Batch rows are independent (test_exec.cpp:246-267): one single-row
    EngineCore<float> per sampled row, run on host threads.  Returns per row
    (probe dict [1][steps][dim] f64, {signal: final state f64})."""
    planned = refapi.planned_from_python(pm)

    def one(b):
        eng = refapi.RefEngine(planned, 1)
        out = eng.run(steps, batch_slice(feeds, b))
        return out, {s: eng.read_signal(s, 0) for s in signals}

    with ThreadPoolExecutor(max_workers=min(threads, len(rows))) as ex:
        return list(ex.map(one, rows))


def spike_count_mismatch(gpu_spikes: np.ndarray, ref_spikes: np.ndarray) -> float:
    """Fraction of (row, neuron) pairs whose spike counts over the run differ
    (the north star's spike tolerance: <= 1e-4).  Inputs [rows][steps][n]."""
    g = np.count_nonzero(gpu_spikes, axis=1)
    r = np.count_nonzero(ref_spikes, axis=1)
    return float(np.mean(g != r))


def assert_f32_bitexact(gpu: np.ndarray, ref: np.ndarray, context: str):
    """gpu (f32 ring values) vs ref (the reference's f64 widening of its f32 values)."""
    r32 = ref.astype(np.float32)
    assert np.array_equal(r32.astype(np.float64).view(np.uint64), ref.view(np.uint64)), f"{context}: ref not f32"
    gb, rb = np.asarray(gpu, dtype=np.float32).view(np.uint32), r32.view(np.uint32)
    nan = np.isnan(r32)
    assert np.array_equal(np.isnan(gpu), nan), f"{context}: NaN positions differ"
    bad = (gb != rb) & ~nan
    if bad.any():
        idx = tuple(int(i) for i in np.argwhere(bad)[0])
        raise AssertionError(f"{context}: differs at {idx}: {gpu[idx]!r} vs {r32[idx]!r} "
                             f"({int(bad.sum())} of {bad.size})")
