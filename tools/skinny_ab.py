"""A/B of the swap-AB skinny GEMM (skinny.cuh) against the tiled plans for short launches.

For each Llama-3-8B projection shape and token count M, times fp_op_gemm (residual epilogue)
with the skinny plan forced (policy 4) and disabled (fp_ctx_set_skinny_max 0), rotating through
enough weight copies (> 2x L2) that every launch streams its weights from HBM, as in a forward
pass. Prints us per launch, the HBM weight-streaming bound, and the achieved GB/s and TFLOP/s."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16603_b200 import _lib  # noqa: E402
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402

SHAPES_NK = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096),
             "down": (4096, 14336), "lm_head": (128256, 4096)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,16,42,64,100,128,163,200,256")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--hbm", type=float, default=7.7e12, help="HBM bytes/s for the bound")
    ap.add_argument("--json", default=None)
    ap.add_argument("--ops", default=",".join(SHAPES_NK), help="subset of " + ",".join(SHAPES_NK))
    a = ap.parse_args()
    ctx = PrefillContext(SHAPES["tiny"], kv_pages=8, max_pos=1024)
    st = torch.cuda.ExternalStream(ctx.stream_ptr)
    rows = []
    for name in a.ops.split(","):
        N, K = SHAPES_NK[name]
        wbytes = N * K * 2
        ncopy = max(2, int(600e6 // wbytes) + 1)
        Bs = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.05 for _ in range(ncopy)]
        for M in [int(x) for x in a.ms.split(",")]:
            if name == "lm_head" and M > 16:
                continue
            A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
            C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
            res = {}
            for mx in (256, 0):  # 256: forced skinny plan (policy 4); 0: tiled plans only
                _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, 4 if mx else -1, 0))
                _lib.check(ctx.lib.fp_ctx_set_skinny_max(ctx.h, mx))
                for i in range(3):
                    ctx.lib.fp_op_gemm(ctx.h, 2, A.data_ptr(), Bs[i % ncopy].data_ptr(),
                                       C.data_ptr(), M, N, K)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(st)
                for i in range(a.iters):
                    ctx.lib.fp_op_gemm(ctx.h, 2, A.data_ptr(), Bs[i % ncopy].data_ptr(),
                                       C.data_ptr(), M, N, K)
                e1.record(st)
                torch.cuda.synchronize()
                res[mx] = e0.elapsed_time(e1) / a.iters * 1e3
            _lib.check(ctx.lib.fp_ctx_set_gemm_policy(ctx.h, -1, 0))
            _lib.check(ctx.lib.fp_ctx_set_skinny_max(ctx.h, 128))
            bound = wbytes / a.hbm * 1e6
            fl = 2.0 * M * N * K
            r = {"op": name, "M": M, "N": N, "K": K, "skinny_us": res[256], "tiled_us": res[0],
                 "bound_us": bound, "skinny_gbs": wbytes / res[256] / 1e3,
                 "skinny_tflops": fl / res[256] / 1e6, "speedup": res[0] / res[256]}
            rows.append(r)
            print(f"{name:8s} M={M:4d}: skinny {res[256]:8.1f} us ({r['skinny_gbs']:6.0f} GB/s, "
                  f"{r['skinny_tflops']:6.1f} TF) | tiled {res[0]:8.1f} us | bound {bound:7.1f} us"
                  f" | x{r['speedup']:.2f} | skinny/bound {res[256] / bound:.2f}", flush=True)
        del Bs
        torch.cuda.empty_cache()
    ctx.close()
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
