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
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
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
