"""Sweep GEMM tiling (CTA pair vs single, forced split-K count) per shape with the weights
streamed from HBM as inside a prefill step (rotating weight copies larger than L2).

    python tools/split_sweep.py [--out gpurun_out/split_sweep.json]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402

SHAPES_NK = [(4096, 4096), (6144, 4096), (28672, 4096), (4096, 14336)]
EPI = {(28672, 4096): 3}  # gate_up: the SwiGLU epilogue (packed gate/up weights); others residual
MS = [42, 163, 386, 545, 872, 1021, 1572, 2048, 3000]
SPLITS = [1, 2, 3, 4, 6, 8, 12, 16]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/split_sweep.json")
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--shapes", default="", help="N,K;N,K subset (default: all four)")
    a = ap.parse_args()
    ctx = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    st = torch.cuda.ExternalStream(ctx.stream_ptr)
    lib = ctx.lib
    res = []
    shapes = [tuple(int(v) for v in x.split(",")) for x in a.shapes.split(";")] if a.shapes else SHAPES_NK
    for N, K in shapes:
        copies = max(2, int(400e6 // (N * K * 2)) + 1)  # > 3x L2 of weights in rotation
        Bs = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(copies)]
        for M in MS:
            A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
            C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
            for pair, S in [(-1, 0), (2, 0), (3, 0)] + [(pair, S) for pair in (0, 1) for S in SPLITS]:
                if True:
                    lib.fp_ctx_set_gemm_policy(ctx.h, pair, S)
                    i = [0]

                    def call():
                        B = Bs[i[0] % copies]
                        i[0] += 1
                        lib.fp_op_gemm(ctx.h, EPI.get((N, K), 2), A.data_ptr(), B.data_ptr(),
                                       C.data_ptr(), M, N, K)

                    for _ in range(3):
                        call()
                    torch.cuda.synchronize()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    for _ in range(a.iters):
                        call()
                    e1.record(st)
                    torch.cuda.synchronize()
                    us = e0.elapsed_time(e1) / a.iters * 1e3
                    res.append({"N": N, "K": K, "M": M, "pair": pair, "S": S,
                                "us": round(us, 2)})
            lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0)
            best = min((r for r in res if r["N"] == N and r["K"] == K and r["M"] == M),
                       key=lambda r: r["us"])
            auto = next(r for r in res if r["N"] == N and r["K"] == K and r["M"] == M
                        and r["pair"] == -1)
            print(f"N={N} K={K} M={M}: auto {auto['us']} us, best pair={best['pair']} "
                  f"S={best['S']} {best['us']} us ({auto['us'] / best['us']:.2f}x)", flush=True)
        del Bs
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(res, fh)
    ctx.close()


if __name__ == "__main__":
    main()
