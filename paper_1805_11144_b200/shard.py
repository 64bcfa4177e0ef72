"""Ensemble sharding across GPUs (one process per GPU).

A shard owns a contiguous range of ensembles and the connections into them
(fused pipeline, fused.hpp).  Each timestep every shard computes the decoded
outputs (xhat) of its ensembles into its rows of the step-parity buffer; an
all-gather over NCCL (torch.distributed, NVLink / NVSwitch on one node) then
gives every shard every xhat before the next step's connection updates read
them.  The step loop is the engine's stepped call (neng_gpu_call_*):

    begin; for k: step(k) -> all-gather parity k & 1; step(n, epilogue); end

The arithmetic of every shard is the single-GPU engine's (same plan-order
sums), so each shard's probes and state are bit-identical to an unsharded
engine's for the ensembles and connections it owns.  The collective is
injected (`gather`), which is how the CPU tests drive this loop with gloo.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

from .engine import STEP_EPILOGUE, STEP_FIRST_UPDATE


def run_stepped(engine, n_steps: int, feed_ptrs: Optional[Sequence[int]], probe_ptrs: Optional[Sequence[int]],
                gather: Callable[[int], None], stream: int = 0) -> int:
    """Advance `engine` n_steps with `gather(parity)` after every step's
    launch; returns the number of kernel launches."""
    engine.call_begin(n_steps, feed_ptrs, probe_ptrs, stream)
    try:
        for k in range(n_steps):
            engine.call_step(k, STEP_FIRST_UPDATE if k else 0)
            gather(k & 1)
        engine.call_step(n_steps, STEP_EPILOGUE)
    finally:
        engine.call_end()
    return n_steps + 1


class TorchGather:
    """In-place all-gather of the xhat parity buffers over a torch.distributed
    process group: shard r's rows sit at r * rank_floats of each parity half,
    so all_gather_into_tensor(half, half[r-slice]) needs no staging copy."""

    def __init__(self, xbuf, rank_floats: int, rank: int, world: int, group=None):
        import torch.distributed as dist
        self.dist = dist
        half = xbuf.numel() // 2
        if rank_floats * world != half:
            raise ValueError(f"parity buffer of {half} floats is not {world} shards of {rank_floats}")
        self.halves = [xbuf[:half], xbuf[half:]]
        self.rank, self.rank_floats, self.group = rank, rank_floats, group

    def __call__(self, parity: int):
        h = self.halves[parity]
        mine = h[self.rank * self.rank_floats:(self.rank + 1) * self.rank_floats]
        self.dist.all_gather_into_tensor(h, mine, group=self.group)


def attach_xhat_buffer(engine, device):
    """Allocate the engine's parity buffers as a torch tensor (so a collective
    can write them) and hand them to the engine; returns (tensor, rank_floats)."""
    import torch
    total, rank_floats, _ = engine.shard_layout()
    xbuf = torch.zeros(total, dtype=torch.float32, device=device)
    engine.set_xhat_buffer(xbuf.data_ptr())
    return xbuf, rank_floats
