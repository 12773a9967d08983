"""Scratch GPU check of the tcgen05 GEMM and rmsnorm against torch (temporary)."""
import ctypes as C
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2602_16603_b200 import _lib as L

lib = L.load()
cfg = L.ModelCfg(2, 512, 4, 2, 128, 1536, 8192, 4096, 10000.0, 1e-5)
ctx = C.c_void_p()
L.check(lib.fp_ctx_create(0, C.byref(cfg), 0, 1, None, 64, 128, C.byref(ctx)), "ctx")
s = C.c_void_p()
lib.fp_ctx_stream(ctx, C.byref(s))
torch.manual_seed(0)
for (M, N, K) in [(128, 256, 64), (300, 512, 512), (1000, 1024, 4096), (8192, 6144, 4096), (77, 4096, 14336)]:
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.05
    Cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    Cf = torch.empty(M, N, device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    L.check(lib.fp_op_gemm(ctx, 1, A.data_ptr(), B.data_ptr(), Cf.data_ptr(), M, N, K), "gemm")
    L.check(lib.fp_sync(ctx), "sync")
    ref = A.float() @ B.float().t()
    err = (Cf - ref).abs().max().item()
    print(f"gemm f32 M={M} N={N} K={K}: maxerr {err:.3e} refmax {ref.abs().max().item():.3f}", flush=True)
    L.check(lib.fp_op_gemm(ctx, 0, A.data_ptr(), B.data_ptr(), Cb.data_ptr(), M, N, K), "gemm")
    L.check(lib.fp_sync(ctx), "sync")
    print("   bf16 maxerr", (Cb.float() - ref).abs().max().item(), flush=True)
    R = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
    R0 = R.clone()
    torch.cuda.synchronize()
    L.check(lib.fp_op_gemm(ctx, 2, A.data_ptr(), B.data_ptr(), R.data_ptr(), M, N, K), "gemm")
    L.check(lib.fp_sync(ctx), "sync")
    print("   resid maxerr", (R.float() - (ref + R0.float())).abs().max().item(), flush=True)
# timing
M, N, K = 8192, 6144, 4096
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
Cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.ExternalStream(s.value)
for _ in range(3):
    lib.fp_op_gemm(ctx, 0, A.data_ptr(), B.data_ptr(), Cb.data_ptr(), M, N, K)
lib.fp_sync(ctx)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20):
    lib.fp_op_gemm(ctx, 0, A.data_ptr(), B.data_ptr(), Cb.data_ptr(), M, N, K)
e1.record(st)
lib.fp_sync(ctx)
ms = e0.elapsed_time(e1) / 20
print(f"gemm {M}x{N}x{K}: {ms*1e3:.1f} us, {2*M*N*K/ms/1e9:.1f} TFLOP/s", flush=True)
t0 = time.time()
ref = torch.matmul(A, B.t())
torch.cuda.synchronize()
e0.record();
for _ in range(20): torch.matmul(A, B.t())
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"torch {ms*1e3:.1f} us, {2*M*N*K/ms/1e9:.1f} TFLOP/s")
# rmsnorm
x = torch.randn(1000, 4096, device="cuda", dtype=torch.bfloat16)
g = torch.rand(4096, device="cuda", dtype=torch.bfloat16) + 0.5
o = torch.empty_like(x)
torch.cuda.synchronize()
L.check(lib.fp_op_rmsnorm(ctx, x.data_ptr(), g.data_ptr(), o.data_ptr(), 1000, 4096, 1e-5), "rms")
lib.fp_sync(ctx)
xf = x.float()
ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * g.float()
print("rms maxerr", (o.float() - ref).abs().max().item())
lib.fp_ctx_destroy(ctx)
print("OK")
