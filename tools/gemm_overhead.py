"""Decompose GEMM launch overhead: one tile per CTA, K sweep (t(K) = fixed + K * rate)."""
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
    for M, N in [(1024, 4096), (128, 256), (4096, 4096)]:
        for K in [64, 256, 1024, 4096, 16384]:
            A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
            B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            for epi in (0, 2):
                t = timeit(lambda: ctx.lib.fp_op_gemm(ctx.h, epi, A.data_ptr(), B.data_ptr(),
                                                      C.data_ptr(), M, N, K), st)
                print(f"M={M} N={N} K={K:6d} epi={epi}: {t:8.2f} us  "
                      f"{2 * M * N * K / t / 1e6:7.1f} TF", flush=True)
            # back-to-back launches of an empty-ish kernel: launch floor
    ctx.close()


if __name__ == "__main__":
    main()
