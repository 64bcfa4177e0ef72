"""CPU (gloo, world_size 2): the ensemble-sharded step loop
(paper_1805_11144_b200/shard.py).  Each rank drives a stand-in engine that
writes its shard's rows of the xhat parity buffer at every step and checks,
at the next step's connection update and at the epilogue, that the in-place
all-gather delivered every shard's rows of the previous step — the ordering
contract the fused kernel relies on (fused.hpp, "Ensemble sharding")."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_11144_b200.engine import STEP_EPILOGUE, STEP_FIRST_UPDATE
from paper_1805_11144_b200.shard import TorchGather, run_stepped


class StandInShard:
    def __init__(self, rank, world, rows, batch):
        self.rank, self.world = rank, world
        self.rank_floats = rows * batch
        self.xbuf = torch.zeros(2 * world * self.rank_floats)
        self.log = []
        self.n = None

    def shard_layout(self):
        return self.xbuf.numel(), self.rank_floats, 0

    def call_begin(self, n, feeds, probes, stream):
        assert self.n is None
        self.n = n

    def _half(self, parity):
        h = self.xbuf.numel() // 2
        return self.xbuf[parity * h:(parity + 1) * h]

    def _expect_step(self, k):
        half = self._half(k & 1)
        for r in range(self.world):
            got = half[r * self.rank_floats:(r + 1) * self.rank_floats]
            assert torch.all(got == 1000 * r + k), f"rank {self.rank}: shard {r} rows of step {k} missing"

    def call_step(self, k, flags):
        self.log.append((k, flags))
        if flags & STEP_FIRST_UPDATE:
            self._expect_step(k - 1)  # connection updates of step k-1 read every shard's xhat(k-1)
        if k < self.n:
            mine = self._half(k & 1)[self.rank * self.rank_floats:(self.rank + 1) * self.rank_floats]
            mine.fill_(1000 * self.rank + k)  # this shard's decode of step k
        else:
            assert flags & STEP_EPILOGUE
            self._expect_step(k - 1)

    def call_end(self):
        self.n = None


def _worker(rank, world, port, n_steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = StandInShard(rank, world, rows=5, batch=3)
        gather = TorchGather(eng.xbuf, eng.rank_floats, rank, world)
        launches = run_stepped(eng, n_steps, None, None, gather)
        assert launches == n_steps + 1
        assert eng.log == [(0, 0)] + [(k, STEP_FIRST_UPDATE) for k in range(1, n_steps)] + [(n_steps, STEP_EPILOGUE)]
        q.put((rank, "ok"))
    except Exception as ex:  # report to the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n_steps", [1, 7])
def test_stepped_loop_gathers_every_shard_before_use(n_steps):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get() for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res


def test_gather_rejects_a_mismatched_layout():
    # the layout is validated before any process group is touched
    with pytest.raises(ValueError):
        TorchGather(torch.zeros(2 * 10), 3, 0, 2)
