"""Per-CTA phase timeline of fp_op_gemm launches (FP_GEMM_STAMPS=1), weights streamed from HBM.

    FP_GEMM_STAMPS=1 python tools/gemm_stamps.py M,N,K,pair,splits [...]
Prints, per config, the median / max over CTAs of each phase's offset from the earliest CTA
entry (us)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402

NAMES = ["entry", "prolog", "guard", "tma0", "mma0", "commit", "epi", "stored", "splitbar",
         "items", "exit", "teardown", "it_start", "it_sum", "it_resid", "it_done"]


def main():
    os.environ.setdefault("FP_GEMM_STAMPS", "1")
    ctx = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    buf = (C.c_uint64 * (4096 * 16))()
    for spec in sys.argv[1:]:
        M, N, K, pair, S = (int(x) for x in spec.split(","))
        copies = max(2, int(300e6 // (N * K * 2)) + 1)
        Bs = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(copies)]
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        Cm = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        ctx.lib.fp_ctx_set_gemm_policy(ctx.h, pair, S)
        rows = []
        for it in range(6):
            ctx.lib.fp_op_gemm(ctx.h, 2, A.data_ptr(), Bs[it % copies].data_ptr(), Cm.data_ptr(),
                               M, N, K)
            ctx.lib.fp_debug_gemm_stamps(ctx.h, buf, 4096)
            a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16).astype(np.int64)
            a = a[a[:, 0] > 0]
            if it >= 2:
                rows.append(a)
        a = rows[-1]
        t0 = a[:, 0].min()
        print(f"== M={M} N={N} K={K} pair={pair} splits={S} : {len(a)} CTAs")
        for k, nm in enumerate(NAMES):
            v = a[:, k]
            v = v[v > 0]
            if len(v) == 0:
                continue
            d = (v - t0) / 1e3
            print(f"  {nm:9s} median {np.median(d):7.2f} us  max {d.max():7.2f} us")
        del Bs
    ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
    ctx.close()


if __name__ == "__main__":
    main()
