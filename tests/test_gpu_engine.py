"""GPU execution pool injected into the UNMODIFIED reference run(): the event log must be
byte-identical to the reference goldens, every device-side stop must land on the reference
cursor, and the logits of every request must match the fp32 oracle (bf16 tolerance)."""

from conftest import refsim_or_skip  # noqa: E402
import json
import os

import numpy as np
import pytest

import parity as P
from oracle import forward as F

pytestmark = pytest.mark.gpu


def _event_lines(res):
    return "".join(json.dumps(ev, sort_keys=True) + "\n" for ev in res.events)


def test_config1_trace_parity(golden_dir):
    from paper_2602_16603_b200 import refsim
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.engine import GpuBinding, run_on_gpu, synthetic_tokens
    from paper_2602_16603_b200.native import PrefillContext

    ps = refsim_or_skip()
    trace = ps.load_trace(os.path.join(golden_dir, "config1_trace.jsonl"))
    shape = F.SHAPES["tiny"]
    w = F.make_weights(shape, 1234)
    ctx = PrefillContext(SHAPES["tiny"], kv_pages=4096, page_size=128, max_pos=40000)
    ctx.load_weights(w)
    tok = synthetic_tokens(1234, shape.vocab)
    b = GpuBinding(ctx, tok)
    res = run_on_gpu(trace, ps.PolicyConfig(), ps.CostParams(num_layers=4), b,
                     record_events=True)
    golden = open(os.path.join(golden_dir, "config1_events.jsonl")).read()
    assert _event_lines(res) == golden
    assert res.commands["preempt"] >= 1 and len(b.handshakes) == res.commands["preempt"]
    for tid, ref_cursor, dev_cursor, state in b.handshakes:
        assert dev_cursor == ref_cursor
    assert len(b.logits) == len(trace)
    # numeric check on the shortest requests (the oracle is fp32 numpy)
    reqs = sorted(trace.requests, key=lambda r: r.num_tokens)[:6]
    for r in reqs:
        ol = F.forward_logits(shape, w, [tok(r)])[0]
        P.logits(f"tiny config-1 run request {r.id} ({r.num_tokens} tokens)", b.logits[r.id], ol)
    assert ctx.free_pages() == 4096  # every task released its KV pages
    ctx.close()


def test_two_request_golden_llama3_8b(golden_dir):
    """The reference's own golden (tests/golden/two_request_events.jsonl, cursor 11 ACK) at
    the Llama-3-8B shape: 32 layers, 8192 + 256 tokens, random-init bf16 weights."""
    from paper_2602_16603_b200 import refsim
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.engine import GpuBinding, run_on_gpu, synthetic_tokens
    from paper_2602_16603_b200.native import PrefillContext

    ps = refsim_or_skip()
    shape = SHAPES["llama3-8b"]
    ctx = PrefillContext(shape, kv_pages=96, page_size=128, max_pos=16384)
    ctx.init_random(seed=0)
    b = GpuBinding(ctx, synthetic_tokens(0, shape.vocab))
    trace = ps.Trace((ps.Request(0, "file", 0.0, 8192, 6.0), ps.Request(1, "text", 0.05, 256, 0.25)))
    res = run_on_gpu(trace, ps.PolicyConfig(), ps.CostParams(), b, record_events=True)
    golden = open(os.path.join(golden_dir, "two_request_events.jsonl")).read()
    assert _event_lines(res) == golden
    assert b.handshakes == [(0, 11, 11, 2)]
    for rid in (0, 1):
        assert np.isfinite(b.logits[rid]).all() and np.abs(b.logits[rid]).max() > 0
    ctx.close()
