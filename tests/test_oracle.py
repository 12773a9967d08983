"""The CPU oracle (test infrastructure) pinned against independent evidence:
HF transformers Llama logits (golden), the reference's own build_timeline / known answers,
and the reference's own run() goldens."""

from conftest import refsim_or_skip  # noqa: E402
import json
import os

import numpy as np
import pytest

from oracle import forward as F


@pytest.fixture(scope="module")
def ps():
    from paper_2602_16603_b200 import refsim

    return refsim_or_skip()


def test_oracle_matches_hf_golden(golden_dir):
    g = np.load(os.path.join(golden_dir, "tiny_hf_logits.npz"))
    shape = F.SHAPES["tiny"]
    w = F.make_weights(shape, int(g["seed"]))
    tokens = F.make_tokens(list(g["lens"]), shape.vocab, int(g["seed"]))
    got = F.forward_logits(shape, w, tokens)
    np.testing.assert_allclose(got, g["logits"], rtol=0, atol=1e-4)


def test_chunked_and_batched_oracle_consistent():
    shape = F.Shape(2, 256, 2, 1, 128, 512, 512, 1e4)
    w = F.make_weights(shape, 3)
    toks = F.make_tokens([50, 7, 90], shape.vocab, 3)
    full = F.forward_logits(shape, w, toks)
    for chunk in (16, 33, 64):
        np.testing.assert_allclose(F.forward_logits(shape, w, toks, chunk), full, atol=2e-5)
    for i, t in enumerate(toks):
        np.testing.assert_allclose(F.forward_logits(shape, w, [t])[0], full[i], atol=2e-5)


def test_oracle_preemption_invariance():
    shape = F.Shape(2, 256, 2, 1, 128, 512, 512, 1e4)
    w = F.make_weights(shape, 4)
    toks = F.make_tokens([40, 70], shape.vocab, 4)
    straight = F.OracleTask(shape, w, toks, 32)
    straight.run_all()
    t = F.OracleTask(shape, w, toks, 32)
    rng = np.random.default_rng(0)
    while t.cursor < len(t):
        t.run(t.cursor, min(len(t), t.cursor + int(rng.integers(1, 7))))
    np.testing.assert_array_equal(t.logits, straight.logits)
    with pytest.raises(ValueError):
        t.run(0, 1)  # completed work is never re-run


@pytest.mark.parametrize("lens,chunk", [([1000], None), ([3000, 500], 1024), ([4, 4], 4),
                                        ([4, 4], 3), ([10], 4), ([7, 5], None),
                                        ([33585], 2048), ([1, 1, 1], 2)])
def test_plan_matches_reference_timeline(ps, lens, chunk):
    """Token-level chunk/segment plan reproduces the reference's per-chunk quad mass, chunk
    count and entry order (cost_model.py:212-242)."""
    attn_only = ps.CostParams(num_layers=1, c_lin={}, c_attn=1.0, c_fix={}, c_chunk=0.0,
                              c_check=0.0)
    tl = ps.build_timeline(lens, chunk, attn_only)
    ref_quad = [e.duration for e in tl.entries if e.kind.value == "attn"]
    plan = F.plan(lens, chunk)
    assert [float(F.quad_mass(c)) for c in plan] == ref_quad
    assert sum(c.new_total for c in plan) == sum(lens)
    p3 = ps.CostParams(num_layers=3)
    tl3 = ps.build_timeline(lens, chunk, p3)
    sh = F.Shape(3, 256, 2, 1, 128, 512, 512, 1e4)
    ot = F.OracleTask(sh, {}, [np.zeros(n, np.int32) for n in lens], chunk)
    assert len(ot) == len(tl3)
    for i, e in enumerate(tl3.entries):
        c, l, o = ot.entry(i)
        assert (c, l, F.OPS[o]) == (e.chunk, e.layer, e.kind.value)


def test_reference_known_answers(ps):
    # pkg/tests/test_cost_model.py:96-109 known answers restated through the oracle plan
    assert [F.quad_mass(c) for c in F.plan([4, 4], 4)] == [16, 16]
    assert [F.quad_mass(c) for c in F.plan([4, 4], 3)] == [9, 8, 8]
    assert len(F.plan([10], 4)) == 3


def test_reference_goldens_reproduce(ps, golden_dir):
    trace = ps.Trace((ps.Request(0, "file", 0.0, 8192, 6.0),
                      ps.Request(1, "text", 0.05, 256, 0.25)))
    res = ps.run(trace, ps.PolicyConfig(), ps.CostParams(), 0, record_events=True)
    lines = "".join(json.dumps(ev, sort_keys=True) + "\n" for ev in res.events)
    assert lines == open(os.path.join(golden_dir, "two_request_events.jsonl")).read()
    tr = ps.load_trace(os.path.join(golden_dir, "config1_trace.jsonl"))
    res = ps.run(tr, ps.PolicyConfig(), ps.CostParams(num_layers=4), 0, record_events=True)
    lines = "".join(json.dumps(ev, sort_keys=True) + "\n" for ev in res.events)
    assert lines == open(os.path.join(golden_dir, "config1_events.jsonl")).read()
    assert res.commands == {"submit": 45, "preempt": 2, "resume": 2}


@pytest.mark.parametrize("name", ["tiny-qwen3", "tiny-qwen2"])
def test_oracle_matches_hf_qwen_goldens(golden_dir, name):
    """q/k-norm (Qwen3) and QKV bias (Qwen2.5) variants pinned to HF Qwen3/Qwen2 models."""
    g = np.load(os.path.join(golden_dir, f"{name}_hf_logits.npz"))
    shape = F.SHAPES[name]
    w = F.make_weights(shape, int(g["seed"]))
    tokens = F.make_tokens(list(g["lens"]), shape.vocab, int(g["seed"]))
    np.testing.assert_allclose(F.forward_logits(shape, w, tokens), g["logits"], rtol=0, atol=1e-4)


def test_oracle_matches_hf_qwen3_moe_golden(golden_dir):
    """MoE layers (router softmax + top-k + renormalised SwiGLU experts, cost_model.py:46-52)
    pinned to HF Qwen3MoeForCausalLM."""
    g = np.load(os.path.join(golden_dir, "tiny-moe_hf_logits.npz"))
    shape = F.SHAPES["tiny-moe"]
    w = F.make_weights(shape, int(g["seed"]))
    tokens = F.make_tokens(list(g["lens"]), shape.vocab, int(g["seed"]))
    np.testing.assert_allclose(F.forward_logits(shape, w, tokens), g["logits"], rtol=0, atol=1e-4)
    # chunked and preempted execution give the same logits (routing is per token)
    np.testing.assert_allclose(F.forward_logits(shape, w, tokens, chunk_size=100), g["logits"],
                               rtol=0, atol=1e-4)


def test_moe_route_ties_and_renorm():
    xn = np.eye(4, dtype=np.float32)
    wr = np.array([[1, 0, 0, 0], [1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 0]], np.float32)
    ids, wts = F.moe_route(xn, wr, 2, True)
    assert ids[0].tolist() == [0, 1]            # tie between experts 0 and 1: lower index first
    np.testing.assert_allclose(wts.sum(-1), 1.0, rtol=1e-6)
