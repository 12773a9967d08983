"""Microbenchmark: fp_op_gemm (tcgen05, unguarded) vs torch.matmul (cuBLAS) per shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16603_b200 import _lib  # noqa: E402
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402


def timeit(fn, stream, iters=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    ctx = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    st = torch.cuda.ExternalStream(ctx.stream_ptr)
    shapes = [(N, K) for N, K in [(4096, 4096), (4096, 14336), (28672, 4096), (6144, 4096)]]
    for N, K in shapes:
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        for M in [64, 163, 545, 1024, 1572, 4096, 8192]:
            A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ours = timeit(lambda: ctx.lib.fp_op_gemm(ctx.h, 2, A.data_ptr(), B.data_ptr(),
                                                     C.data_ptr(), M, N, K), st)
            ref = timeit(lambda: torch.matmul(A, B.t(), out=C), torch.cuda.current_stream())
            fl = 2 * M * N * K
            print(f"N={N:6d} K={K:6d} M={M:5d}: ours {ours:8.1f} us {fl / ours / 1e6:7.1f} TF | "
                  f"cublas {ref:8.1f} us {fl / ref / 1e6:7.1f} TF", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
