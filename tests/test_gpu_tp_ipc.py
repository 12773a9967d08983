"""One process per rank (the deployment path of config 4): two processes, each a TP=2 rank,
exchange their exchange-block handles over a gloo group (connect_tp_dist), map each other's
blocks through CUDA IPC and run independently -- no lock step, each rank's launch stream is its
own. On the single-GPU test box both processes share the device (time-sliced contexts), which
exercises the same cross-process waits (exchange readiness, rank-0 decision ring) the 8-GPU box
runs over NVLink. Checks: logits vs the fp32 oracle, identical logits on both ranks, a
preemption signalled on rank 0 stops both ranks at the same entry, and the FUSED exchange (the
o_proj / down_proj GEMM flags each tile's partial and folds every rank's tile over peer memory
inside the same kernel) matches the GEMM + tp_allreduce_kernel pair (same rank-order sums; only
the summation order of the next norm's sum of squares differs, so within 1%)."""

import os
import random

import numpy as np
import pytest
import torch.multiprocessing as mp

import parity as P
from oracle import forward as F

pytestmark = pytest.mark.gpu

NAME = "tiny-qwen2-tp"


def _rank_main(rank, size, port, q, fused=True, distinct=False):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      FP_TP_FUSED="1" if fused else "0")
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        from paper_2602_16603_b200.config import SHAPES
        from paper_2602_16603_b200.native import PrefillContext, connect_tp_dist

        shape = F.SHAPES[NAME]
        w = F.make_weights(shape, 4321)
        ctx = PrefillContext(SHAPES[NAME], device=rank if distinct else 0, kv_pages=64, max_pos=4096,
                             tp_rank=rank, tp_size=size)
        connect_tp_dist(ctx, 1024)
        ctx.load_weights(w)
        tokens = F.make_tokens([300, 37], shape.vocab, 11)
        # straight run
        t = ctx.create_task(tokens, None, "operator", 0)
        n = t.n_entries
        t.begin_segment(0)
        t.enqueue(0, n)
        ctx.sync()
        straight = t.logits()
        t.destroy()
        # preempted run: rank 0 raises the signal between the two halves
        t = ctx.create_task(tokens, None, "operator", 1)
        k = n // 2 + 1
        t.begin_segment(0)
        t.enqueue(0, k)
        ctx.sync()
        dist.barrier()
        if rank == 0:
            ctx.signal()
        dist.barrier()
        t.enqueue(k, n)
        ctx.sync()
        st = t.poll()
        stop = (st.state, st.cursor)
        t.begin_segment(st.cursor)
        t.enqueue(st.cursor, n)
        ctx.sync()
        done = t.poll().state
        resumed = t.logits()
        t.destroy()
        q.put((rank, straight, stop, done, resumed, ctx.tp_counters()))
        dist.barrier()
        ctx.close()
    finally:
        dist.destroy_process_group()


def _run_group(fused, distinct=False):
    size, port = 2, random.randint(20000, 40000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, size, port, q, fused, distinct))
             for r in range(size)]
    for p in procs:
        p.start()
    try:
        res = {}
        for _ in range(size):
            r, *rest = q.get(timeout=240)
            res[r] = rest
    finally:
        for p in procs:
            p.join(60)
            if p.is_alive():
                p.kill()
    return res


@pytest.mark.timeout(300)
def test_tp2_two_processes_ipc():
    res = _run_group(fused=True)
    shape = F.SHAPES[NAME]
    w = F.make_weights(shape, 4321)
    ref = F.forward_logits(shape, w, F.make_tokens([300, 37], shape.vocab, 11))
    s0, s1 = res[0][0], res[1][0]
    assert np.array_equal(s0, s1)
    P.logits(f"{NAME} tp=2 two processes (fused exchange)", s0, ref)
    n_entries = 5 * shape.num_layers
    k = n_entries // 2 + 1
    assert res[0][1] == res[1][1] == (2, k)  # both ranks stopped at the same entry
    assert res[0][2] == res[1][2] == 3
    assert np.array_equal(res[0][3], s0) and np.array_equal(res[1][3], s0)
    c0, c1 = res[0][4], res[1][4]
    assert (c0["exchanges"], c0["boundaries"]) == (c1["exchanges"], c1["boundaries"])



@pytest.mark.timeout(300)
def test_tp2_fused_exchange_matches_two_kernel_exchange():
    fused, split = _run_group(fused=True), _run_group(fused=False)
    for r in range(2):
        for i in (0, 3):  # straight, preempted + resumed
            a, b = fused[r][i], split[r][i]
            assert np.abs(a - b).max() / np.abs(b).max() <= 0.01
        assert np.array_equal(fused[r][0], fused[r][3])  # fused: preemption changes no bits
        assert fused[r][4]["exchanges"] == split[r][4]["exchanges"]


@pytest.mark.timeout(300)
def test_tp2_two_devices_ipc():
    """The deployment form of config 4 on real hardware: rank r on GPU r, the exchange blocks
    mapped over CUDA IPC across devices (NVLink peer memory). Skipped on a 1-GPU box."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = _run_group(fused=True, distinct=True)
    shape = F.SHAPES[NAME]
    w = F.make_weights(shape, 4321)
    ref = F.forward_logits(shape, w, F.make_tokens([300, 37], shape.vocab, 11))
    s0, s1 = res[0][0], res[1][0]
    assert np.array_equal(s0, s1)
    P.logits(f"{NAME} tp=2 two devices (fused exchange)", s0, ref)
    k = 5 * shape.num_layers // 2 + 1
    assert res[0][1] == res[1][1] == (2, k)
    assert np.array_equal(res[0][3], s0) and np.array_equal(res[1][3], s0)
