"""GPU parity: the full preemptible forward pass through the C ABI vs the CPU fp32 oracle.

Tolerance (bf16 path vs fp32 oracle; stated per BASELINE north_star, tests/parity.py): logits
max-abs error <= 3% of max|logit| and relative L2 error <= 2%; KV max-abs <= 2% of max|kv| and
relative L2 <= 1%. Both error kinds are printed and recorded for every comparison. GPU-vs-GPU
comparisons (preempted vs straight, repeated runs) are bit-exact.
"""

import numpy as np
import pytest

import parity as P
from oracle import forward as F

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape = F.SHAPES["tiny"]
    w = F.make_weights(shape, 1234)
    ctx = PrefillContext(SHAPES["tiny"], kv_pages=512, page_size=128, max_pos=8192)
    ctx.load_weights(w)
    yield shape, w, ctx
    ctx.close()


def run_straight(ctx, tokens, chunk=None, gran="operator"):
    t = ctx.create_task(tokens, chunk, gran)
    t.begin_segment(0)
    t.enqueue(0, t.n_entries)
    ctx.sync()
    st = t.poll()
    assert st.state == 3 and st.cursor == t.n_entries
    return t


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-6))


def test_golden_hf_logits(tiny, golden_dir):
    shape, w, ctx = tiny
    g = np.load(f"{golden_dir}/tiny_hf_logits.npz")
    tokens = F.make_tokens(list(g["lens"]), shape.vocab, int(g["seed"]))
    t = run_straight(ctx, tokens)
    P.logits("tiny vs HF golden", t.logits(), g["logits"])
    t.destroy()


@pytest.mark.parametrize("lens,chunk", [([300], None), ([37, 130, 64, 201], None),
                                        ([37, 130, 64, 201], 100), ([1000, 5], 256)])
def test_logits_and_kv_vs_oracle(tiny, lens, chunk):
    shape, w, ctx = tiny
    tokens = F.make_tokens(lens, shape.vocab, 77)
    ot = F.OracleTask(shape, w, tokens, chunk)
    ot.run_all()
    t = run_straight(ctx, tokens, chunk)
    name = f"tiny lens={lens} chunk={chunk}"
    P.logits(name, t.logits(), ot.logits)
    for r in range(len(lens)):
        for layer in (0, shape.num_layers - 1):
            k, v = t.read_kv(r, layer)
            P.kv(f"{name} K[{r}][{layer}]", k, ot.k_cache[r][layer])
            P.kv(f"{name} V[{r}][{layer}]", v, ot.v_cache[r][layer])
    t.destroy()


def test_batch_composition(tiny):
    """Default (split-K where it pays): per-request results depend on batch composition only
    through the split-K reduction order -- within 1% of max|logit|; repeated runs are
    bit-exact. Batch-invariant mode (no split-K / stream-K): bit-identical alone or batched."""
    shape, w, ctx = tiny
    tokens = F.make_tokens([200, 90, 333, 1, 17], shape.vocab, 5)
    batched = run_straight(ctx, tokens)
    lb = batched.logits()
    again = run_straight(ctx, tokens)
    assert np.array_equal(again.logits(), lb)  # deterministic (fixed split-K reduction order)
    again.destroy()
    for r in range(len(tokens)):
        alone = run_straight(ctx, [tokens[r]])
        assert rel_err(alone.logits()[0], lb[r]) <= 0.01
        alone.destroy()
    batched.destroy()
    ctx.set_batch_invariant(True)
    try:
        batched = run_straight(ctx, tokens)
        lb = batched.logits()
        kb = [batched.read_kv(r, shape.num_layers - 1) for r in range(len(tokens))]
        batched.destroy()
        pairs = run_straight(ctx, [tokens[4], tokens[0]])  # another composition and order
        lp = pairs.logits()
        pairs.destroy()
        assert np.array_equal(lp[0], lb[4]) and np.array_equal(lp[1], lb[0])
        for r in range(len(tokens)):
            alone = run_straight(ctx, [tokens[r]])
            assert np.array_equal(alone.logits()[0], lb[r]), r
            k, v = alone.read_kv(0, shape.num_layers - 1)
            assert np.array_equal(k, kb[r][0]) and np.array_equal(v, kb[r][1]), r
            alone.destroy()
    finally:
        ctx.set_batch_invariant(False)


@pytest.mark.parametrize("gran", ["operator", "layer", "chunk"])
def test_preemption_bitwise_and_cursor(tiny, gran):
    """Stop at device boundary checks, resume from the published cursor: same bits as a
    straight run, and stops only land on eligible boundaries."""
    shape, w, ctx = tiny
    tokens = F.make_tokens([257, 64], shape.vocab, 9)
    chunk = 128 if gran == "chunk" else None
    ref = run_straight(ctx, tokens, chunk, gran)
    lref = ref.logits()
    ref.destroy()
    t = ctx.create_task(tokens, chunk, gran)
    n = t.n_entries
    rng = np.random.default_rng(0)
    cursor, stops = 0, 0
    while True:
        t.begin_segment(cursor)
        run_to = min(n, cursor + int(rng.integers(1, 12)))
        t.enqueue(cursor, run_to)
        ctx.sync()
        if run_to == n:
            break
        ctx.signal()
        t.enqueue(run_to, n)  # the rest of the task is queued behind the signal
        ctx.sync()
        st = t.poll()
        if st.state != 2:  # no eligible boundary left: the task ran to completion
            assert st.state == 3
            ctx.clear()
            break
        stops += 1
        assert st.cursor >= run_to
        prev = st.cursor - 1  # last executed entry; the boundary after it must be eligible
        if gran == "layer":
            assert prev % 5 == 4
        if gran == "chunk":
            assert prev % (5 * shape.num_layers) == 5 * shape.num_layers - 1
        assert ctx.poll().signal == 0  # the device unset the flag when it stopped
        cursor = st.cursor
    assert stops > 0
    assert t.poll().state == 3
    assert np.array_equal(t.logits(), lref)
    t.destroy()


@pytest.mark.parametrize("policy", [-1, 4])
@pytest.mark.parametrize("name", ["tiny-qwen3", "tiny-qwen2"])
def test_qwen_variants_vs_hf_and_oracle(golden_dir, name, policy):
    """Qwen3 q/k-norm and Qwen2.5 QKV bias in the fused QKV epilogue; vocab 8000 (not a
    multiple of 256: lm_head padded internally). Policy 4 runs every launch (chunks of 96) on
    the swap-AB skinny kernel, whose reduction feeds the same epilogues."""
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape = F.SHAPES[name]
    w = F.make_weights(shape, 1234)
    ctx = PrefillContext(SHAPES[name], kv_pages=64, max_pos=4096)
    ctx.load_weights(w)
    ctx.lib.fp_ctx_set_gemm_policy(ctx.h, policy, 0)
    g = np.load(f"{golden_dir}/{name}_hf_logits.npz")
    tokens = F.make_tokens(list(g["lens"]), shape.vocab, int(g["seed"]))
    t = run_straight(ctx, tokens, 96)
    lg = t.logits()
    assert lg.shape == (len(tokens), 8000)
    P.logits(f"{name} (gemm policy {policy}) vs HF golden", lg, g["logits"])
    ot = F.OracleTask(shape, w, tokens, 96)
    ot.run_all()
    P.logits(f"{name} (gemm policy {policy}) vs oracle", lg, ot.logits)
    for r in range(len(tokens)):
        k, v = t.read_kv(r, 1)
        P.kv(f"{name} (policy {policy}) K[{r}][1]", k, ot.k_cache[r][1])
        P.kv(f"{name} (policy {policy}) V[{r}][1]", v, ot.v_cache[r][1])
    t.destroy()
    ctx.close()


@pytest.mark.parametrize("policy", [2, 0, 3])
def test_forced_gemm_tiling_vs_oracle(tiny, policy):
    """Every GEMM of the forward with narrow 128 x 128 tiles (policy 2: residual and QKV
    epilogues), single-CTA 256-wide tiles (policy 0) or stream-K (policy 3: every epilogue,
    the fused norm applied after the partner partials are folded in): logits and KV within
    tolerance."""
    shape, w, ctx = tiny
    tokens = F.make_tokens([37, 300, 130], shape.vocab, 21)
    ot = F.OracleTask(shape, w, tokens, None)
    ot.run_all()
    try:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, policy, 0)
        t = run_straight(ctx, tokens)
        lg = t.logits()
        kv = [t.read_kv(r, shape.num_layers - 1) for r in range(3)]
        t.destroy()
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    name = f"tiny gemm policy {policy}"
    P.logits(name, lg, ot.logits)
    for r, (k, v) in enumerate(kv):
        P.kv(f"{name} K[{r}]", k, ot.k_cache[r][shape.num_layers - 1])
        P.kv(f"{name} V[{r}]", v, ot.v_cache[r][shape.num_layers - 1])


@pytest.mark.parametrize("chunk", [None, 96, 200])
def test_skinny_gemm_forward_vs_oracle(tiny, chunk):
    """Every GEMM launch of at most 256 rows on the swap-AB skinny kernel (policy 4): with
    chunks of 96 / 200 tokens that is every qkv / o / gate_up / down launch of the forward (fused
    input norm, RoPE + paged KV scatter, SwiGLU, residual + sums of squares through the skinny
    kernel's grid-wide reduction), unchunked only the lm_head; logits and KV within tolerance of
    the oracle, and bit-identical run to run."""
    shape, w, ctx = tiny
    tokens = F.make_tokens([37, 300, 130], shape.vocab, 23)
    ot = F.OracleTask(shape, w, tokens, chunk)
    ot.run_all()
    runs = []
    try:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, 4, 0)
        for _ in range(2):
            t = run_straight(ctx, tokens, chunk)
            runs.append((t.logits(), [t.read_kv(r, shape.num_layers - 1) for r in range(3)]))
            t.destroy()
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    (lg, kv), (lg2, kv2) = runs
    assert np.array_equal(lg, lg2)
    for (k, v), (k2, v2) in zip(kv, kv2):
        assert np.array_equal(k, k2) and np.array_equal(v, v2)
    name = f"tiny skinny gemm chunk {chunk}"
    P.logits(name, lg, ot.logits)
    for r, (k, v) in enumerate(kv):
        P.kv(f"{name} K[{r}]", k, ot.k_cache[r][shape.num_layers - 1])
        P.kv(f"{name} V[{r}]", v, ot.v_cache[r][shape.num_layers - 1])


@pytest.mark.parametrize("splits", [2, 4, 8])
def test_cluster_split_forward_bitexact(tiny, splits):
    """A chunked forward with every GEMM tile split into K-slices (forced): the all-split
    launches reduce inside clusters through distributed shared memory (gemm.cuh MODE 4); a
    context created with FP_SPLIT_DSMEM=0 reduces through the L2 workspace. Logits and KV are
    bit-identical between the two and within tolerance of the oracle."""
    import os

    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape, w, ctx = tiny
    os.environ["FP_SPLIT_DSMEM"] = "0"
    try:
        ctx_l2 = PrefillContext(SHAPES["tiny"], kv_pages=64, page_size=128, max_pos=8192)
    finally:
        del os.environ["FP_SPLIT_DSMEM"]
    tokens = F.make_tokens([37, 300, 130], shape.vocab, 29)
    out = []
    try:
        ctx_l2.load_weights(w)
        for c in (ctx, ctx_l2):
            c.lib.fp_ctx_set_gemm_policy(c.h, 0, splits)
            t = run_straight(c, tokens, 96)
            out.append((t.logits(), [t.read_kv(r, shape.num_layers - 1) for r in range(3)]))
            t.destroy()
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
        ctx_l2.close()
    (lg, kv), (lg2, kv2) = out
    assert np.array_equal(lg, lg2)
    for (k, v), (k2, v2) in zip(kv, kv2):
        assert np.array_equal(k, k2) and np.array_equal(v, v2)
    ot = F.OracleTask(shape, w, tokens, 96)
    ot.run_all()
    name = f"tiny cluster split S={splits}"
    P.logits(name, lg, ot.logits)
    for r, (k, v) in enumerate(kv):
        P.kv(f"{name} K[{r}]", k, ot.k_cache[r][shape.num_layers - 1])
        P.kv(f"{name} V[{r}]", v, ot.v_cache[r][shape.num_layers - 1])


def test_page_pool_exhaustion_is_clean():
    """A task that needs more KV pages than are free fails with the pool untouched, and the
    context keeps working (fp_task_create releases everything it took on any failure)."""
    from paper_2602_16603_b200 import _lib
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape = F.SHAPES["tiny"]
    w = F.make_weights(shape, 3)
    c = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=4096)
    try:
        c.load_weights(w)
        assert c.free_pages() == 8
        with pytest.raises(_lib.NativeError, match="exhausted"):
            c.create_task(F.make_tokens([600, 600], shape.vocab, 1))  # 10 pages
        assert c.free_pages() == 8
        t = run_straight(c, F.make_tokens([900], shape.vocab, 2))
        assert c.free_pages() == 8 - 8
        t.destroy()
        assert c.free_pages() == 8
    finally:
        c.close()


def test_context_creation_failure_releases_memory():
    """A context whose KV pool cannot be allocated fails cleanly: the weights and streams it had
    already created are released, and the next context works."""
    import torch

    from paper_2602_16603_b200 import _lib
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    with pytest.raises(_lib.NativeError):
        PrefillContext(SHAPES["llama3-8b"], kv_pages=4_000_000, max_pos=4096)  # ~2 TB of KV
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < (256 << 20), (free0, free1)  # the 16 GB of weights were freed
    c = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    c.close()
