"""Per-operator GPU checks through the C ABI (fp_op_gemm / fp_op_rmsnorm) vs torch fp32."""

import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    c = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    yield c
    c.close()


@pytest.mark.parametrize("M,N,K", [(1, 256, 64), (128, 256, 64), (300, 512, 512),
                                   (1000, 1024, 4096), (77, 4096, 14336), (4096, 6144, 4096)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm(ctx, M, N, K, epi):
    import torch

    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    B = (torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05)
    ref = A.float() @ B.float().t()
    if epi == 1:
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    else:
        out = torch.randn(M, N, device="cuda", dtype=torch.bfloat16, generator=g)
    r0 = out.float().clone()
    torch.cuda.synchronize()
    from paper_2602_16603_b200 import _lib

    _lib.check(ctx.lib.fp_op_gemm(ctx.h, epi, A.data_ptr(), B.data_ptr(), out.data_ptr(), M, N, K))
    ctx.sync()
    if epi == 2:
        ref = ref + r0
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    tol = 1e-5 * scale * K ** 0.5 if epi == 1 else 2 ** -7 * scale + 1e-3
    assert err <= tol, (err, scale)


@pytest.mark.parametrize("d", [512, 4096, 5120])
def test_rmsnorm(ctx, d):
    import torch

    from paper_2602_16603_b200 import _lib

    x = torch.randn(999, d, device="cuda", dtype=torch.bfloat16)
    gm = (torch.rand(d, device="cuda") + 0.5).to(torch.bfloat16)
    o = torch.empty_like(x)
    torch.cuda.synchronize()
    _lib.check(ctx.lib.fp_op_rmsnorm(ctx.h, x.data_ptr(), gm.data_ptr(), o.data_ptr(), 999, d, 1e-5))
    ctx.sync()
    xf = x.float()
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * gm.float()
    assert (o.float() - ref).abs().max().item() <= 2 ** -7 * ref.abs().max().item()


@pytest.mark.parametrize("M,N,K", [(42, 4096, 4096), (300, 1024, 4096), (77, 512, 14336),
                                   (1, 256, 1024), (2000, 4096, 4096)])
@pytest.mark.parametrize("pair,splits", [(0, 3), (0, 16), (1, 5), (1, 12)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_forced_split(ctx, M, N, K, pair, splits, epi):
    """Forced split-K tiling (fp_ctx_set_gemm_policy): the K-slice CTAs of a tile reduce it
    together; within bf16 tolerance of fp32 and bit-identical run to run (partials are summed
    in split order)."""
    import torch

    from paper_2602_16603_b200 import _lib

    g = torch.Generator(device="cuda").manual_seed(M + N + K + splits + epi)
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    if epi == 1:
        R = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    else:
        R = torch.randn(M, N, device="cuda", dtype=torch.bfloat16, generator=g)
    ref = A.float() @ B.float().t() + (R.float() if epi == 2 else 0.0)
    outs = []
    try:
        _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, pair, splits))
        for _ in range(2):
            out = R.clone()
            torch.cuda.synchronize()
            _lib.check(ctx.lib.fp_op_gemm(ctx.h, epi, A.data_ptr(), B.data_ptr(), out.data_ptr(),
                                          M, N, K))
            ctx.sync()
            outs.append(out)
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    assert torch.equal(outs[0], outs[1])
    err = (outs[0].float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    tol = 1e-5 * scale * K ** 0.5 if epi == 1 else 2 ** -7 * scale + 1e-3
    assert err <= tol, (err, scale)


@pytest.mark.parametrize("M,N,K", [(42, 4096, 4096), (450, 4096, 4096), (1000, 1024, 14336),
                                   (1, 256, 128)])
def test_gemm_narrow_tiles(ctx, M, N, K):
    """128 x 128 tiles (residual epilogue), forced: within bf16 tolerance of fp32."""
    import torch

    from paper_2602_16603_b200 import _lib

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    out = torch.randn(M, N, device="cuda", dtype=torch.bfloat16, generator=g)
    ref = A.float() @ B.float().t() + out.float()
    try:
        _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, 2, 0))
        torch.cuda.synchronize()
        _lib.check(ctx.lib.fp_op_gemm(ctx.h, 2, A.data_ptr(), B.data_ptr(), out.data_ptr(), M, N, K))
        ctx.sync()
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    err = (out.float() - ref).abs().max().item()
    assert err <= 2 ** -7 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("M,N,K", [(1, 256, 1024), (42, 4096, 4096), (300, 1024, 4096),
                                   (77, 4096, 14336), (2000, 4096, 4096), (4096, 6144, 4096),
                                   (5000, 4096, 1024)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_streamk(ctx, M, N, K, epi):
    """Stream-K (policy 3): whole tiles first, then equal contiguous (tile, k-block) ranges per
    CTA; a tile's finishing CTA folds its partners' partials into TMEM. Covers all-stream-K
    launches with up to ~8 partners per tile, one-to-two-wave launches, and whole-tile waves in
    front. Within bf16 tolerance of fp32 and bit-identical run to run."""
    import torch

    from paper_2602_16603_b200 import _lib

    g = torch.Generator(device="cuda").manual_seed(M + N + K + epi + 3)
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    if epi == 1:
        R = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    else:
        R = torch.randn(M, N, device="cuda", dtype=torch.bfloat16, generator=g)
    ref = A.float() @ B.float().t() + (R.float() if epi == 2 else 0.0)
    outs = []
    try:
        _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, 3, 0))
        for _ in range(2):
            out = R.clone()
            torch.cuda.synchronize()
            _lib.check(ctx.lib.fp_op_gemm(ctx.h, epi, A.data_ptr(), B.data_ptr(), out.data_ptr(),
                                          M, N, K))
            ctx.sync()
            outs.append(out)
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    assert torch.equal(outs[0], outs[1])
    err = (outs[0].float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    tol = 1e-5 * scale * K ** 0.5 if epi == 1 else 2 ** -7 * scale + 1e-3
    assert err <= tol, (err, scale)


@pytest.mark.parametrize("M,N,K", [(1, 256, 64), (1, 4096, 4096), (7, 512, 1024),
                                   (42, 4096, 4096), (42, 6144, 4096), (64, 1024, 14336),
                                   (100, 28672, 4096), (163, 4096, 14336), (200, 256, 4096),
                                   (256, 4096, 4096), (33, 128256 // 256 * 256, 512)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_skinny(ctx, M, N, K, epi):
    """Swap-AB skinny GEMM (policy 4; skinny.cuh): weight rows as the MMA M dimension, tokens as
    N, equal (128-row slice, k-block) ranges per CTA, contributor-ordered reduction by each
    256-column block's last contributor. Covers one-CTA launches (tiny U), slices split among
    many CTAs (long K), CTAs spanning several slices (wide N), M = 1 ... 256 (three token-tile
    instantiations). Within bf16 tolerance of fp32 and bit-identical run to run."""
    import torch

    from paper_2602_16603_b200 import _lib

    g = torch.Generator(device="cuda").manual_seed(M * 3 + N + K + epi)
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    if epi == 1:
        R = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    else:
        R = torch.randn(M, N, device="cuda", dtype=torch.bfloat16, generator=g)
    ref = A.float() @ B.float().t() + (R.float() if epi == 2 else 0.0)
    outs = []
    try:
        _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, 4, 0))
        for _ in range(2):
            # output inside a guard band of canary rows (an out-of-bounds write check: the
            # compute-sanitizer is not available on the GPU pool)
            band = torch.full((M + 16, N), 7.0, device="cuda", dtype=R.dtype)
            band[8:8 + M] = R
            out = band[8:8 + M]
            torch.cuda.synchronize()
            _lib.check(ctx.lib.fp_op_gemm(ctx.h, epi, A.data_ptr(), B.data_ptr(), out.data_ptr(),
                                          M, N, K))
            ctx.sync()
            assert bool((band[:8] == 7.0).all()) and bool((band[8 + M:] == 7.0).all())
            outs.append(out.clone())
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    assert torch.equal(outs[0], outs[1])
    err = (outs[0].float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    tol = 1e-5 * scale * K ** 0.5 if epi == 1 else 2 ** -7 * scale + 1e-3
    assert err <= tol, (err, scale)


@pytest.mark.parametrize("M", [1, 42, 163, 256])
def test_gemm_skinny_vs_tiled(ctx, M):
    """The skinny plan and the tiled plans agree within bf16 rounding of one output (their K
    summation orders differ)."""
    import torch

    from paper_2602_16603_b200 import _lib

    N, K = 4096, 4096
    g = torch.Generator(device="cuda").manual_seed(M + 11)
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    R = torch.randn(M, N, device="cuda", dtype=torch.bfloat16, generator=g)
    got = {}
    try:
        for mx in (256, 0):  # forced skinny plan, then tiled plans only
            _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, 4 if mx else -1, 0))
            _lib.check(ctx.lib.fp_ctx_set_skinny_max(ctx.h, mx))
            out = R.clone()
            torch.cuda.synchronize()
            _lib.check(ctx.lib.fp_op_gemm(ctx.h, 2, A.data_ptr(), B.data_ptr(), out.data_ptr(),
                                          M, N, K))
            ctx.sync()
            got[mx] = out.float()
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
        ctx.lib.fp_ctx_set_skinny_max(ctx.h, 128)
    scale = got[0].abs().max().item()
    assert (got[256] - got[0]).abs().max().item() <= 2 ** -7 * scale


@pytest.mark.parametrize("policy", [-1, 3, 4])
@pytest.mark.parametrize("M,F,K", [(1, 128, 64), (300, 512, 512), (4096, 1536, 512),
                                   (77, 14336 // 4, 4096), (386, 14336, 4096), (163, 14336, 4096)])
def test_gate_up_swiglu(ctx, M, F, K, policy):
    """gate_up GEMM + SwiGLU epilogue vs torch fp32: silu(x Wg^T) * (x Wu^T)."""
    import torch

    from paper_2602_16603_b200 import _lib

    g = torch.Generator(device="cuda").manual_seed(M + F + K)
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    wg = torch.randn(F, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    wu = torch.randn(F, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    out = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    try:
        _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, policy, 0))
        _lib.check(ctx.lib.fp_op_gate_up_swiglu(ctx.h, x.data_ptr(), wg.data_ptr(), wu.data_ptr(),
                                                out.data_ptr(), M, F, K))
        ctx.sync()
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    xf = x.float()
    ref = torch.nn.functional.silu(xf @ wg.float().t()) * (xf @ wu.float().t())
    err = (out.float() - ref).abs().max().item()
    assert err <= 2 ** -7 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("policy", [-1, 4])
@pytest.mark.parametrize("M,q_cols,kv_cols,K", [(1, 512, 256, 512), (77, 512, 256, 512),
                                                 (300, 4096, 1024, 1024), (700, 1024, 128, 256),
                                                 (42, 4096, 1024, 4096), (256, 1024, 256, 2048)])
def test_qkv_rope_kv(ctx, M, q_cols, kv_cols, K, policy):
    """qkv_proj with its fused epilogue vs torch fp32: [q|k|v] = x W^T, rotate-half RoPE on q and
    k at arbitrary positions (the context's theta), K/V scattered into the paged layout."""
    import torch

    from paper_2602_16603_b200 import _lib

    ps, theta, n_pages = 128, ctx.shape.rope_theta, 8
    hkv = kv_cols // 128
    g = torch.Generator(device="cuda").manual_seed(M + q_cols + K)
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    w = torch.randn(q_cols + 2 * kv_cols, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    pos = torch.randperm(n_pages * ps, generator=torch.Generator().manual_seed(M))[:M]
    page_of = torch.randperm(n_pages, generator=torch.Generator().manual_seed(K))
    tok_page = page_of[pos // ps]
    pos_d = pos.to(torch.int32).cuda()
    tp_d = tok_page.to(torch.int32).cuda()
    q = torch.empty(M, q_cols, device="cuda", dtype=torch.bfloat16)
    kv = torch.zeros(n_pages, 2, hkv, ps, 128, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    if policy == 4 and M > 256:
        pytest.skip("skinny GEMM covers M <= 256")
    try:
        _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, policy, 0))
        _lib.check(ctx.lib.fp_op_qkv_rope_kv(ctx.h, x.data_ptr(), w.data_ptr(), q.data_ptr(),
                                             kv.data_ptr(), pos_d.data_ptr(), tp_d.data_ptr(), M,
                                             q_cols, kv_cols, K))
        ctx.sync()
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    y = x.float() @ w.float().t()
    inv = theta ** (-torch.arange(64, dtype=torch.float64) * 2 / 128)
    ang = pos.double()[:, None] * inv[None, :]
    cos, sin = ang.cos().float().cuda(), ang.sin().float().cuda()

    def rope(t):  # [M, heads*128], rotate-half per head
        t = t.view(M, -1, 128)
        a, b = t[..., :64], t[..., 64:]
        return torch.cat([a * cos[:, None] - b * sin[:, None], b * cos[:, None] + a * sin[:, None]],
                         -1).view(M, -1)

    q_ref = rope(y[:, :q_cols])
    k_ref = rope(y[:, q_cols:q_cols + kv_cols]).view(M, hkv, 128)
    v_ref = y[:, q_cols + kv_cols:].view(M, hkv, 128)
    k_got = kv[tok_page.cuda(), 0, :, (pos % ps).cuda()].float()
    v_got = kv[tok_page.cuda(), 1, :, (pos % ps).cuda()].float()
    for got, ref in ((q.float(), q_ref), (k_got, k_ref), (v_got, v_ref)):
        err = (got - ref).abs().max().item()
        assert err <= 2 ** -7 * ref.abs().max().item() + 1e-3, err
    written = torch.zeros(n_pages, ps, dtype=torch.bool)
    written[tok_page, pos % ps] = True
    untouched = kv.permute(0, 3, 1, 2, 4)[~written.cuda()]
    assert untouched.abs().max().item() == 0  # nothing outside the tokens' slots


@pytest.mark.parametrize("n_q,kv_len", [(1, 1), (37, 37), (128, 128), (200, 200), (130, 700),
                                        (1000, 1000), (64, 4096), (513, 2049)])
def test_attn_prefill_vs_torch(n_q, kv_len):
    """Causal prefill attention (tcgen05, paged K/V, GQA) vs torch fp32 attention with the
    query rows at positions kv_len - n_q ... kv_len - 1 (a chunk share after its prefix)."""
    import torch

    from paper_2602_16603_b200 import _lib
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape = SHAPES["llama3-8b"]  # 32 query heads, 8 KV heads (GQA group 4)
    c = _attn_ctx(shape)
    hq, hkv = shape.n_heads, shape.n_kv_heads
    g = torch.Generator(device="cuda").manual_seed(n_q * 7 + kv_len)
    q = torch.randn(n_q, hq * 128, device="cuda", dtype=torch.bfloat16, generator=g)
    k = torch.randn(kv_len, hkv * 128, device="cuda", dtype=torch.bfloat16, generator=g)
    v = torch.randn(kv_len, hkv * 128, device="cuda", dtype=torch.bfloat16, generator=g)
    out = torch.empty(n_q, hq * 128, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    _lib.check(c.lib.fp_op_attn_prefill(c.h, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                        out.data_ptr(), n_q, kv_len))
    qf = q.float().view(n_q, hq, 128).transpose(0, 1)
    kf = k.float().view(kv_len, hkv, 128).transpose(0, 1).repeat_interleave(hq // hkv, 0)
    vf = v.float().view(kv_len, hkv, 128).transpose(0, 1).repeat_interleave(hq // hkv, 0)
    pos = torch.arange(kv_len - n_q, kv_len, device="cuda")[:, None]
    mask = torch.arange(kv_len, device="cuda")[None, :] <= pos
    ref = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf, attn_mask=mask)
    ref = ref.transpose(0, 1).reshape(n_q, hq * 128)
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item(), err


_ATTN = {}


def _attn_ctx(shape):
    from paper_2602_16603_b200.native import PrefillContext

    if "c" not in _ATTN:  # one context (weights are never touched by the op)
        _ATTN["c"] = PrefillContext(shape, kv_pages=64, page_size=128, max_pos=8192)
    return _ATTN["c"]


@pytest.mark.parametrize("M,N,K,splits", [(42, 4096, 4096, 8), (42, 6144, 4096, 6),
                                          (163, 4096, 14336, 4), (1, 256, 1024, 2),
                                          (100, 1024, 4096, 8)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_split_cluster_matches_l2(ctx, M, N, K, splits, epi):
    """Split-K with every tile split runs as clusters of the K-slice CTAs reducing through
    distributed shared memory (gemm.cuh MODE 4); a context created with FP_SPLIT_DSMEM=0 reduces
    the same partials through the L2 workspace. Both sum in split order from 0: bit-identical,
    and within bf16 tolerance of fp32."""
    import os

    import torch

    from paper_2602_16603_b200 import _lib
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    os.environ["FP_SPLIT_DSMEM"] = "0"
    try:
        ctx_l2 = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    finally:
        del os.environ["FP_SPLIT_DSMEM"]
    g = torch.Generator(device="cuda").manual_seed(M + N + K + splits + epi + 5)
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * 0.05
    if epi == 1:
        R = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    else:
        R = torch.randn(M, N, device="cuda", dtype=torch.bfloat16, generator=g)
    ref = A.float() @ B.float().t() + (R.float() if epi == 2 else 0.0)
    outs = []
    try:
        for c in (ctx, ctx_l2):
            _lib.check(c.lib.fp_ctx_set_gemm_policy(c.h, 0, splits))
            out = R.clone()
            torch.cuda.synchronize()
            _lib.check(c.lib.fp_op_gemm(c.h, epi, A.data_ptr(), B.data_ptr(), out.data_ptr(),
                                        M, N, K))
            c.sync()
            outs.append(out)
    finally:
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
        ctx_l2.close()
    assert torch.equal(outs[0], outs[1])
    err = (outs[0].float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    tol = 1e-5 * scale * K ** 0.5 if epi == 1 else 2 ** -7 * scale + 1e-3
    assert err <= tol, (err, scale)
