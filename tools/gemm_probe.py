"""Launch fp_op_gemm (residual epilogue) once per spec for ncu captures:
python tools/gemm_probe.py M,N,K,pair,splits [...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402


def main():
    ctx = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    for spec in sys.argv[1:]:
        M, N, K, pair, S = (int(x) for x in spec.split(","))
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        torch.cuda.synchronize()
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, pair, S)
        for _ in range(2):
            ctx.lib.fp_op_gemm(ctx.h, 2, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K)
        ctx.sync()
    ctx.close()


if __name__ == "__main__":
    main()
