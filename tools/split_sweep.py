"""Sweep forced split-K / pair settings for small-M shapes (run under different env vars)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402
from tools.gemm_bench import timeit  # noqa: E402


def main():
    ctx = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    st = torch.cuda.ExternalStream(ctx.stream_ptr)
    tag = f"pair={os.environ.get('FP_FORCE_PAIR', 'auto')} S={os.environ.get('FP_FORCE_SPLITS', 'auto')}"
    out = []
    for N, K in [(4096, 4096), (4096, 14336), (28672, 4096), (6144, 4096)]:
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        for M in [163, 545, 1024, 1572]:
            A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            t = timeit(lambda: ctx.lib.fp_op_gemm(ctx.h, 2, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                                                  M, N, K), st)
            out.append(f"{N}x{K} M={M}:{t:7.1f}")
    print(tag, " | ".join(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
