"""Host side of the one-process-per-GPU tensor-parallel connect (no GPU): every rank exports
its exchange-block handle, the handles are all-gathered over a world-size-2 gloo group, and
each rank imports the full, rank-ordered list (native.connect_tp_dist)."""

import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


class FakeCtx:
    def __init__(self, rank, size):
        self.tp_rank, self.tp_size = rank, size
        self.imported = None

    def tp_export(self, max_tokens):
        return bytes([self.tp_rank]) * 8 + max_tokens.to_bytes(8, "little")

    def tp_import(self, handles):
        self.imported = list(handles)


def _worker(rank, size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        from paper_2602_16603_b200.native import connect_tp_dist

        ctx = FakeCtx(rank, size)
        connect_tp_dist(ctx, 4096)
        q.put((rank, ctx.imported))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_connect_tp_dist_gloo():
    import random

    size, port = 2, random.randint(20000, 40000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=100) for _ in range(size))
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    want = [bytes([r]) * 8 + (4096).to_bytes(8, "little") for r in range(size)]
    assert got[0] == want and got[1] == want
