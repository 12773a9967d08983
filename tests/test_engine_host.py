"""Host-side logic of the GPU execution pool on CPU (fake native backend, fp32 oracle numbers):
the reference run() with GpuEngine injected reproduces the reference goldens byte-for-byte,
every timeline entry executes exactly once across preemptions, stops land on the reference
cursor, and preempted+resumed logits equal uninterrupted ones."""

from conftest import refsim_or_skip  # noqa: E402
import json
import os

import numpy as np
import pytest

from fake_native import FakeContext
from oracle import forward as F


def _events(res):
    return "".join(json.dumps(ev, sort_keys=True) + "\n" for ev in res.events)


@pytest.fixture(scope="module")
def ps():
    from paper_2602_16603_b200 import refsim

    return refsim_or_skip()


def test_config1_golden_through_gpu_engine(ps, golden_dir):
    from paper_2602_16603_b200.engine import GpuBinding, run_on_gpu, synthetic_tokens

    trace = ps.load_trace(os.path.join(golden_dir, "config1_trace.jsonl"))
    # keep the CPU test fast: only the 12 shortest requests, same arrival times and SLOs
    keep = sorted(trace.requests, key=lambda r: r.num_tokens)[:12]
    sub = ps.Trace(tuple(sorted(keep, key=lambda r: (r.arrival_time, r.id))))
    ctx = FakeContext("tiny")
    tok = synthetic_tokens(1234, ctx.shape.vocab)
    b = GpuBinding(ctx, tok)
    params = ps.CostParams(num_layers=4)
    res = run_on_gpu(sub, ps.PolicyConfig(), params, b, record_events=True)
    ref = ps.run(sub, ps.PolicyConfig(), params, 0, record_events=True)
    assert _events(res) == _events(ref)
    for t in ctx.tasks:  # work conservation: each entry exactly once
        assert t.executed == list(range(t.n_entries))
        assert t.destroyed
    for tid, ref_cursor, dev_cursor, state in b.handshakes:
        assert dev_cursor == ref_cursor and state == 2
    for r in sub.requests:
        solo = F.forward_logits(ctx.oshape, ctx.weights, [tok(r)])[0]
        np.testing.assert_allclose(b.logits[r.id], solo, rtol=0, atol=2e-4)


def test_two_request_golden_event_log(ps, golden_dir):
    """The reference's golden (ACK at cursor 11 of the 8192-token task, 32 layers) through
    GpuEngine; cursor semantics only (no numbers)."""
    from paper_2602_16603_b200.engine import GpuBinding, run_on_gpu, synthetic_tokens

    golden = open(os.path.join(golden_dir, "two_request_events.jsonl")).read()
    trace = ps.Trace((ps.Request(0, "file", 0.0, 8192, 6.0),
                      ps.Request(1, "text", 0.05, 256, 0.25)))
    ref = ps.run(trace, ps.PolicyConfig(), ps.CostParams(), 0, record_events=True)
    assert _events(ref) == golden
    ctx = FakeContext("tiny", num_layers=32, compute=False)
    b = GpuBinding(ctx, synthetic_tokens(0, ctx.shape.vocab), collect_logits=False)
    res = run_on_gpu(trace, ps.PolicyConfig(), ps.CostParams(), b, record_events=True)
    assert _events(res) == golden
    assert b.handshakes == [(0, 11, 11, 2)]
    assert all(t.executed == list(range(t.n_entries)) for t in ctx.tasks)


@pytest.mark.parametrize("gran", ["operator", "layer", "chunk"])
def test_preempt_resume_equals_straight(ps, gran):
    from paper_2602_16603_b200.engine import GpuBinding, run_on_gpu, synthetic_tokens

    # a long low-priority request interrupted by two short urgent ones
    trace = ps.Trace((ps.Request(0, "file", 0.0, 300, 60.0),
                      ps.Request(1, "text", 0.004, 20, 0.02),
                      ps.Request(2, "text", 0.009, 33, 0.02)))
    params = ps.CostParams(num_layers=2)
    ctx = FakeContext("tiny", num_layers=2)
    tok = synthetic_tokens(7, ctx.shape.vocab)
    pc = ps.PolicyConfig(granularity=ps.PreemptionGranularity(gran),
                         chunk_tokens=128 if gran == "chunk" else None)
    b = GpuBinding(ctx, tok)
    res = run_on_gpu(trace, pc, params, b, record_events=True)
    ref = ps.run(trace, pc, params, 0, record_events=True)
    assert _events(res) == _events(ref)
    assert res.commands["preempt"] >= 1
    for r in trace.requests:
        solo = F.forward_logits(ctx.oshape, ctx.weights, [tok(r)], pc.chunk_tokens)[0]
        np.testing.assert_allclose(b.logits[r.id], solo, rtol=0, atol=2e-4)


def test_moe_arch_through_gpu_engine(ps):
    """arch='moe' (MOE_LAYER_OPS, cost_model.py:46-52): the GPU engine maps entries to gate /
    experts, the event log equals the reference's, and stops between gate and experts resume
    to the uninterrupted oracle logits."""
    from paper_2602_16603_b200.engine import GpuBinding, run_on_gpu, synthetic_tokens

    ctx = FakeContext("tiny-moe")
    params = ps.CostParams(num_layers=ctx.shape.num_layers, arch="moe")
    trace = ps.Trace((ps.Request(0, "file", 0.0, 300, 6.0), ps.Request(1, "text", 0.0004, 40, 0.25),
                      ps.Request(2, "text", 0.0009, 70, 0.25)))
    tok = synthetic_tokens(11, ctx.shape.vocab)
    b = GpuBinding(ctx, tok)
    res = run_on_gpu(trace, ps.PolicyConfig(), params, b, record_events=True)
    ref = ps.run(trace, ps.PolicyConfig(), params, 0, record_events=True)
    assert _events(res) == _events(ref)
    assert res.commands["preempt"] >= 1  # the long request was preempted at least once
    for r in trace.requests:
        want = F.forward_logits(ctx.oshape, ctx.weights, [tok(r)])[0]
        np.testing.assert_allclose(b.logits[r.id], want, rtol=0, atol=1e-5)
    dense = GpuBinding(FakeContext("tiny"), tok)
    with pytest.raises(Exception):  # a dense GPU model refuses an MoE cost model
        run_on_gpu(trace, ps.PolicyConfig(), params, dense)
