"""Diagnose the 2-CTA GEMM: single tile, long K, pair vs single-CTA kernels."""
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
    tag = os.environ.get("FP_PAIR_GEMM", "1")
    for M, N, K in [(256, 256, 16384), (256, 512, 16384), (2048, 4096, 4096), (8192, 4096, 4096)]:
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t = timeit(lambda: ctx.lib.fp_op_gemm(ctx.h, 0, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                                              M, N, K), st)
        ref = (A.float() @ B.float().t())
        err = (C.float() - ref).abs().max().item() / ref.abs().max().item()
        print(f"pair={tag} M={M} N={N} K={K}: {t:9.2f} us {2*M*N*K/t/1e6:8.1f} TF err {err:.2e}",
              flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
