"""Multi-instance (data-parallel) path on CPU: round-robin sharding of a trace over
world_size 2 gloo ranks, each running its own scheduler + execution pool with no data-path
collective, outcomes gathered for the metrics."""

from conftest import refsim_or_skip  # noqa: E402
import os

import pytest


def test_round_robin_partition():
    from paper_2602_16603_b200 import dispatch, refsim

    ps = refsim_or_skip()
    tr = ps.load_trace(os.path.join(os.path.dirname(__file__), "golden", "config1_trace.jsonl"))
    parts = dispatch.round_robin(tr, 3)
    assert sum(len(p) for p in parts) == len(tr)
    assert [r.id for r in parts[1].requests] == [r.id for r in tr.requests[1::3]]
    res = [ps.run(p, ps.PolicyConfig(), ps.CostParams(num_layers=4), 0).outcomes for p in parts]
    merged = dispatch.merge_outcomes(res)
    assert [o.id for o in merged] == sorted(r.id for r in tr.requests)
    with pytest.raises(ValueError):
        dispatch.merge_outcomes([res[0], res[0]])


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2602_16603_b200 import dispatch, refsim

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ps = refsim_or_skip()
    tr = ps.load_trace(os.path.join(os.path.dirname(__file__), "golden", "config1_trace.jsonl"))
    mine = dispatch.round_robin(tr, world)[rank]
    local = ps.run(mine, ps.PolicyConfig(), ps.CostParams(num_layers=4), 0).outcomes
    merged = dispatch.gather_outcomes(local)
    if rank == 0:
        q.put([(o.id, o.prefill_end_s) for o in merged])
    dist.destroy_process_group()


def test_gloo_two_instances():
    import multiprocessing as mp
    import socket

    from paper_2602_16603_b200 import dispatch, refsim

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ps = refsim_or_skip()
    tr = ps.load_trace(os.path.join(os.path.dirname(__file__), "golden", "config1_trace.jsonl"))
    expect = dispatch.merge_outcomes(
        [ps.run(p, ps.PolicyConfig(), ps.CostParams(num_layers=4), 0).outcomes
         for p in dispatch.round_robin(tr, 2)])
    assert got == [(o.id, o.prefill_end_s) for o in expect]
