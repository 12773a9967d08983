"""Tensor parallelism (BASELINE config 4): Megatron shards, the peer-memory
all-reduce after o_proj / down_proj, and synchronized operator-boundary preemption.

The ranks of a group run on ONE B200 in lock step (fp_tp_connect_local): the device code --
exchange GEMM + publish, peer-memory all-reduce, rank-0 decision ring -- is the same code a
one-process-per-GPU deployment runs.

Tolerances: logits max-abs <= 3% of max|logit|, KV <= 2% of max|kv| vs the fp32 oracle (as in
test_gpu_forward.py); TP vs TP=1 on the same weights <= 1.5% (the partial sums are rounded to
bf16 before the exchange). Replicated state (logits, residual) is bit-identical across ranks;
preempted vs straight runs are bit-identical.
"""

from conftest import refsim_or_skip  # noqa: E402
import json

import numpy as np
import pytest

import parity as P
from oracle import forward as F

pytestmark = pytest.mark.gpu

LOGIT_ATOL_FRAC = 0.03
KV_ATOL_FRAC = 0.02
NAME = "tiny-qwen2-tp"


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-6))


@pytest.fixture(scope="module")
def weights():
    shape = F.SHAPES[NAME]
    return shape, F.make_weights(shape, 4321)


def make_group(tp, w, max_tokens=1024, kv_pages=256, max_pos=4096):
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import TPGroup

    g = TPGroup(SHAPES[NAME], tp, kv_pages=kv_pages, max_pos=max_pos, max_tokens=max_tokens)
    g.load_weights(w)
    return g


def run_straight(ctx, tokens, chunk=None, gran="operator"):
    t = ctx.create_task(tokens, chunk, gran)
    t.begin_segment(0)
    t.enqueue(0, t.n_entries)
    ctx.sync()
    st = t.poll()
    assert st.state == 3 and st.cursor == t.n_entries
    return t


@pytest.mark.parametrize("tp", [2, 4])
@pytest.mark.parametrize("lens,chunk", [([300, 37, 130], None), ([300, 37, 130], 128)])
def test_tp_logits_kv_vs_oracle(weights, tp, lens, chunk):
    shape, w = weights
    g = make_group(tp, w)
    tokens = F.make_tokens(lens, shape.vocab, 11)
    ot = F.OracleTask(shape, w, tokens, chunk)
    ot.run_all()
    t = run_straight(g, tokens, chunk)
    per_rank = t.rank_logits()
    for r in range(1, tp):  # replicated residual stream => identical logits on every rank
        assert np.array_equal(per_rank[r], per_rank[0]), r
    name = f"{NAME} tp={tp} lens={lens} chunk={chunk}"
    P.logits(name, per_rank[0], ot.logits)
    for r in range(len(lens)):
        for layer in (0, shape.num_layers - 1):
            k, v = t.read_kv(r, layer)  # heads gathered rank-major = the model's head order
            P.kv(f"{name} K[{r}][{layer}]", k, ot.k_cache[r][layer])
            P.kv(f"{name} V[{r}][{layer}]", v, ot.v_cache[r][layer])
    cnt = g.tp_counters()
    assert len({(c["exchanges"], c["boundaries"]) for c in cnt}) == 1, cnt
    n_chunks = t.info()["n_chunks"]
    assert cnt[0]["exchanges"] == 2 * shape.num_layers * n_chunks
    assert cnt[0]["boundaries"] == t.n_entries
    assert all(c["gemm_ticket"] == 0 and c["allreduce_ticket"] == 0 for c in cnt)
    t.destroy()
    g.close()


def test_tp_matches_single_rank(weights):
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape, w = weights
    tokens = F.make_tokens([200, 513], shape.vocab, 3)
    one = PrefillContext(SHAPES[NAME], kv_pages=64, max_pos=4096)
    one.load_weights(w)
    t1 = run_straight(one, tokens)
    l1 = t1.logits()
    t1.destroy()
    one.close()
    g = make_group(2, w)
    t2 = run_straight(g, tokens)
    e = rel_err(t2.logits(), l1)
    print("tp=2 vs tp=1:", e)
    assert e <= 0.015
    t2.destroy()
    g.close()


@pytest.mark.parametrize("tp,gran", [(2, "operator"), (4, "operator"), (2, "layer")])
def test_tp_synchronized_preemption(weights, tp, gran):
    """Signal rank 0 only; every rank stops at the same entry (rank 0's decision ring), the
    stop lands on an eligible boundary, and resuming from the cursor reproduces the straight
    run's bits. Interleaves a second task while the first is preempted (shared exchange
    buffers and counters must survive task switches)."""
    shape, w = weights
    g = make_group(tp, w)
    tokens = F.make_tokens([260, 70], shape.vocab, 21)
    other = F.make_tokens([150], shape.vocab, 22)
    ref = run_straight(g, tokens, None, gran)
    lref = ref.logits()
    ref.destroy()
    ref2 = run_straight(g, other, None, gran)
    lref2 = ref2.logits()
    ref2.destroy()

    t = g.create_task(tokens, None, gran, task_id=1)
    n = t.n_entries
    rng = np.random.default_rng(1)
    cursor, stops = 0, 0
    while True:
        t.begin_segment(cursor)
        run_to = min(n, cursor + int(rng.integers(1, 9)))
        t.enqueue(cursor, run_to)
        g.sync()
        if run_to == n:
            break
        g.signal()
        t.enqueue(run_to, n)
        g.sync()
        lanes = t.poll_all()
        assert len({(s.state, s.cursor) for s in lanes}) == 1, [(s.state, s.cursor) for s in lanes]
        st = lanes[0]
        if st.state != 2:
            assert st.state == 3
            g.clear()
            break
        stops += 1
        assert st.cursor >= run_to
        if gran == "layer":
            assert (st.cursor - 1) % 5 == 4
        assert g.poll().signal == 0
        cursor = st.cursor
        if stops == 1:  # a higher-priority task runs while task 1 is preempted
            t2 = run_straight(g, other, None, gran)
            assert np.array_equal(t2.logits(), lref2)
            t2.destroy()
    assert stops > 0
    assert np.array_equal(t.logits(), lref)
    for lg in t.rank_logits():
        assert np.array_equal(lg, lref)
    cnt = g.tp_counters()
    assert len({(c["exchanges"], c["boundaries"]) for c in cnt}) == 1, cnt
    t.destroy()
    g.close()


def test_tp_capacity_error(weights):
    from paper_2602_16603_b200 import _lib

    shape, w = weights
    g = make_group(2, w, max_tokens=256)
    with pytest.raises(_lib.NativeError, match="capacity"):
        g.create_task(F.make_tokens([300], shape.vocab, 1))
    t = g.create_task(F.make_tokens([300], shape.vocab, 1), chunk_tokens=256)  # chunked fits
    t.destroy()
    g.close()


def test_tp_reference_run_config1(golden_dir):
    """The unmodified reference run() on the config-1 trace with a TP=2 group injected: event
    log byte-identical to the golden, device stops on the reference cursors on both ranks."""
    import os

    from paper_2602_16603_b200 import refsim
    from paper_2602_16603_b200.engine import GpuBinding, run_on_gpu, synthetic_tokens

    ps = refsim_or_skip()
    trace = ps.load_trace(os.path.join(golden_dir, "config1_trace.jsonl"))
    shape = F.SHAPES[NAME]
    w = F.make_weights(shape, 4321)
    g = make_group(2, w, max_tokens=40000, kv_pages=2048, max_pos=40000)
    tok = synthetic_tokens(1234, shape.vocab)
    b = GpuBinding(g, tok)
    res = run_on_gpu(trace, ps.PolicyConfig(), ps.CostParams(num_layers=4), b, record_events=True)
    lines = "".join(json.dumps(ev, sort_keys=True) + "\n" for ev in res.events)
    assert lines == open(os.path.join(golden_dir, "config1_events.jsonl")).read()
    assert res.commands["preempt"] >= 1 and len(b.handshakes) == res.commands["preempt"]
    for tid, ref_cursor, dev_cursor, state in b.handshakes:
        assert dev_cursor == ref_cursor and state == 2
    r = min(trace.requests, key=lambda r: r.num_tokens)
    ol = F.forward_logits(shape, w, [tok(r)])[0]
    P.logits(f"{NAME} tp=2 config-1 run request {r.id}", b.logits[r.id], ol)
    g.close()


@pytest.mark.parametrize("tp", [2, 4])
def test_qwen25_32b_shape_tp_reference_parity(tp):
    """Config-4 shape (Qwen2.5-32B: 64 layers, d=5120, 40/8 heads, ffn 27648, QKV bias) at
    TP=2/4, random-init bf16 weights: the reference run() on a two-request trace with the TP
    group injected produces the same event log as the reference's own CPU run, and every
    device stop lands on the reference cursor on all ranks."""
    from paper_2602_16603_b200 import refsim
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.engine import GpuBinding, run_on_gpu, synthetic_tokens
    from paper_2602_16603_b200.native import TPGroup

    ps = refsim_or_skip()
    shape = SHAPES["qwen2.5-32b"]
    trace = ps.Trace((ps.Request(0, "file", 0.0, 6000, 6.0), ps.Request(1, "text", 0.05, 300, 0.25)))
    params = ps.CostParams(num_layers=64, tp_degree=tp)
    cpu = ps.run(trace, ps.PolicyConfig(), params, record_events=True)
    g = TPGroup(shape, tp, kv_pages=128, max_pos=8192, max_tokens=8192)
    g.init_random(seed=0)
    b = GpuBinding(g, synthetic_tokens(0, shape.vocab))
    res = run_on_gpu(trace, ps.PolicyConfig(), params, b, record_events=True)
    assert res.events == cpu.events
    assert cpu.commands["preempt"] >= 1
    assert [(h[1], h[2]) for h in b.handshakes] == [(h[1], h[1]) for h in b.handshakes]
    for rid in (0, 1):
        assert np.isfinite(b.logits[rid]).all() and np.abs(b.logits[rid]).max() > 0
    g.close()


@pytest.mark.parametrize("tp", [2, 4])
def test_op_tp_allreduce(tp):
    """fp_op_tp_allreduce (the row-parallel exchange as a per-op entry point): every rank's h
    becomes bf16(h + part_0 + ... + part_{tp-1}) with the fp32 sum in rank order -- bit-exact
    against torch, identical on every rank, over consecutive exchanges (both slots)."""
    import ctypes as C

    import torch

    from paper_2602_16603_b200 import _lib
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import TPGroup

    shape = SHAPES[NAME]
    g = TPGroup(shape, tp, kv_pages=8, max_pos=1024, max_tokens=512)
    try:
        ctxs = (C.c_void_p * tp)(*[c.h.value for c in g.ranks])
        gen = torch.Generator(device="cuda").manual_seed(tp)
        for M in (300, 1, 512):
            h0 = torch.randn(M, shape.hidden, device="cuda", generator=gen).to(torch.bfloat16)
            hs = [h0.clone() for _ in range(tp)]
            parts = [torch.randn(M, shape.hidden, device="cuda", generator=gen).to(torch.bfloat16)
                     for _ in range(tp)]
            torch.cuda.synchronize()
            hp = (C.c_void_p * tp)(*[x.data_ptr() for x in hs])
            pp = (C.c_void_p * tp)(*[x.data_ptr() for x in parts])
            _lib.check(g.lib.fp_op_tp_allreduce(ctxs, tp, hp, pp, M), "fp_op_tp_allreduce")
            g.sync()
            acc = h0.float()
            for p in parts:
                acc = acc + p.float()
            ref = acc.to(torch.bfloat16)
            for r in range(tp):
                assert torch.equal(hs[r], ref), r
    finally:
        g.close()


def test_tp_group_has_no_wall_clock_worker(weights):
    """A lock-step TPGroup is parity-mode only: start() (the async worker the live driver
    uses) fails loudly instead of deadlocking the ranks' exchange."""
    shape, w = weights
    g = make_group(2, w)
    t = g.create_task(F.make_tokens([40], shape.vocab, 1))
    with pytest.raises(NotImplementedError):
        t.start(0)
    t.destroy()
    g.close()
