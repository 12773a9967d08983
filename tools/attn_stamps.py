"""Phase timeline of the attention kernel (diagnostic build, clock64 stamps): per KV tile of
the first work item of CTAs 0..15, when each head's softmax sees S and releases P, and when the
MMA warp issues P*V and the next Q*K^T. Answers "how long is the softmax critical path per tile
vs the tensor-core time per tile".

    python tools/attn_stamps.py --len 4465 [--reps 3]

Builds a -DFP_GEMM_STAMPS copy of the library under /tmp and loads it through FP_AB_LIB (the
in-tree library is untouched)."""
import argparse
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build_stamps() -> str:
    from paper_2602_16603_b200 import build as B

    out = "/tmp/fp_stamps/libflowprefill.so"
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [os.environ.get("NVCC", "nvcc"), *B.NVCC_FLAGS, "-DFP_GEMM_STAMPS", "-o", out,
           *B.sources()]
    subprocess.run(cmd, check=True, capture_output=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--len", type=int, default=4465)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    os.environ["FP_AB_LIB"] = os.environ.get("FP_STAMPS_LIB") or build_stamps()
    os.environ["FP_GEMM_STAMPS"] = "1"
    import torch

    from paper_2602_16603_b200 import _lib
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape = SHAPES["llama3-8b"]
    n = a.len
    c = PrefillContext(shape, kv_pages=(n + 127) // 128 + 8, page_size=128, max_pos=max(8192, n + 8))
    hq, hkv = shape.n_heads, shape.n_kv_heads
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(n, hq * 128, device="cuda", dtype=torch.bfloat16, generator=g)
    k = torch.randn(n, hkv * 128, device="cuda", dtype=torch.bfloat16, generator=g)
    v = torch.randn(n, hkv * 128, device="cuda", dtype=torch.bfloat16, generator=g)
    out = torch.empty(n, hq * 128, device="cuda", dtype=torch.bfloat16)
    buf = np.zeros((4096, 16), np.uint64)
    for r in range(a.reps):
        c.lib.fp_debug_gemm_stamps(c.h, buf.ctypes.data, 4096)  # sync; zeroed per op launch below
        st = torch.cuda.Event(enable_timing=True)
        en = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        st.record()
        _lib.check(c.lib.fp_op_attn_prefill(c.h, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                            out.data_ptr(), n, n))
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en)
    _lib.check(c.lib.fp_debug_gemm_stamps(c.h, buf.ctypes.data, 4096))
    flops = 4 * hq * 128 * n * (n + 1) / 2
    print(f"len {n}: {ms * 1e3:.1f} us (incl. op overhead), {flops / ms / 1e9:.1f} TFLOP/s")
    s = buf.reshape(-1)[: 16 * 64 * 24].reshape(16, 64, 24).astype(np.int64)
    names = ["h0 S seen", "h0 P out", "h1 S seen", "h1 P out", "PV0 issue", "QK0 issued",
             "PV1 issue", "QK1 issued", "K(j+1) in", "-", "h0 S regs", "h0 max", "h0 P st",
             "h0 sum", "h1 S regs", "h1 max", "h1 P st", "h1 sum"]
    for cta in range(2):
        t = s[cta]
        nt = int((t[:, 0] > 0).sum())
        if nt < 3:
            continue
        t0 = t[0, 0]
        print(f"CTA {cta}: {nt} KV tiles (clock64 cycles relative to h0 S seen of tile 0)")
        print("tile " + " ".join(f"{x:>10s}" for x in names))
        for j in range(min(nt, 12)):
            print(f"{j:4d} " + " ".join(f"{(x - t0) if x else 0:10d}" for x in t[j, :18]))
        mid = slice(1, nt - 1)
        for h in (0, 1):
            b = 10 + 4 * h
            seen = t[mid, 2 * h]
            print(f"  head {h} softmax phases (median cycles): S seen->regs "
                  f"{np.median(t[mid, b] - seen):.0f}, ->max {np.median(t[mid, b + 1] - t[mid, b]):.0f}, "
                  f"->P stored {np.median(t[mid, b + 2] - t[mid, b + 1]):.0f}, ->arrive "
                  f"{np.median(t[mid, 2 * h + 1] - t[mid, b + 2]):.0f}, ->sum {np.median(t[mid, b + 3] - t[mid, 2 * h + 1]):.0f}")
        print(f"  MMA: PV0 issue -> K(j+1) in {np.median(t[mid, 8] - t[mid, 4]):.0f}, K in -> QK0 issued "
              f"{np.median(t[mid, 5] - t[mid, 8]):.0f}")
        sm0 = t[1:nt - 1, 1] - t[1:nt - 1, 0]  # softmax h0 latency (S seen -> P out)
        sm1 = t[1:nt - 1, 3] - t[1:nt - 1, 2]
        per = np.diff(t[1:nt - 1, 0])          # h0 period per tile
        s2s0 = t[2:nt, 0] - t[1:nt - 1, 1]       # h0 P out -> next S seen (TC + wakeup)
        print(f"  median softmax latency h0 {np.median(sm0):.0f} h1 {np.median(sm1):.0f} cycles; "
              f"P->next S h0 {np.median(s2s0):.0f}; period per tile {np.median(per):.0f}; "
              f"ideal TC per tile (2 heads, 8192 flop/clk) {2 * 4 * 128 ** 3 / 8192:.0f}")
    # per work item: where the time between items goes
    it = buf.reshape(-1)[24576: 24576 + 16 * 32 * 8].reshape(16, 32, 8).astype(np.int64)
    gaps = {"item fetch -> first QK issued": [], "first QK -> first S seen": [],
            "last P -> O complete": [], "epilogue": [], "epilogue done -> next item's first S": []}
    spans = []
    for cta in range(16):
        t = it[cta]
        n = int((t[:, 2] > 0).sum())
        for i in range(n):
            if t[i, 1] and t[i, 0]:
                gaps["item fetch -> first QK issued"].append(t[i, 1] - t[i, 0])
            if t[i, 2] and t[i, 1]:
                gaps["first QK -> first S seen"].append(t[i, 2] - t[i, 1])
            if t[i, 4] and t[i, 3]:
                gaps["last P -> O complete"].append(t[i, 4] - t[i, 3])
            if t[i, 5] and t[i, 4]:
                gaps["epilogue"].append(t[i, 5] - t[i, 4])
            if i + 1 < n and t[i + 1, 2] and t[i, 5]:
                gaps["epilogue done -> next item's first S"].append(t[i + 1, 2] - t[i, 5])
        if n and t[0, 6]:
            spans.append((t[n - 1, 5] - t[0, 6], t[0, 2] - t[0, 6], n))
    for k, v in gaps.items():
        if v:
            print(f"  per item: {k:40s} median {np.median(v):7.0f} cycles (n={len(v)})")
    if spans:
        print(f"  CTA span (cycles): median {np.median([s[0] for s in spans]):.0f}; kernel start -> "
              f"first S {np.median([s[1] for s in spans]):.0f}; items per CTA {np.median([s[2] for s in spans]):.0f}")
    c.close()


if __name__ == "__main__":
    main()
