"""A/B of the prefill attention kernel against the library attention kernels on this box
(comparators, not oracles): torch SDPA with the cuDNN / flash / efficient backends, causal, GQA,
bf16, one request of N tokens, Llama-3-8B heads (32 q, 8 kv, head_dim 128).

    python tools/attn_compare.py --len 4465 [--len 8192]

Ours is timed with CUDA events around its launch inside a 2-layer prefill task (the event pair
brackets exactly the attention kernel on the prefill stream); algorithmic FLOPs are
4 * d_q * n (n + 1) / 2 for both."""
import argparse
import os
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def ours(n: int, reps: int) -> float:
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape = replace(SHAPES["llama3-8b"], num_layers=2)
    ctx = PrefillContext(shape, kv_pages=(n + 127) // 128 + 8, max_pos=max(40000, n + 8))
    ctx.init_random(0)
    tok = np.random.default_rng(0).integers(0, shape.vocab, n).astype(np.int32)
    task = ctx.create_task([tok])
    times = []
    for r in range(reps + 2):
        ctx.profile(True)
        ctx.drain_profile()
        task.begin_segment(0)
        task.enqueue(0, task.n_entries)
        ctx.sync()
        recs = [x for x in ctx.drain_profile() if x["kind"] == "attn"]
        if r >= 2:
            times += [x["ms"] for x in recs]
    ctx.profile(False)
    task.destroy()
    ctx.close()
    return float(np.median(times))


def sdpa(n: int, reps: int, backend) -> float:
    import torch
    from torch.nn.attention import sdpa_kernel

    q = torch.randn(1, 32, n, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, 8, n, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(1, 8, n, 128, device="cuda", dtype=torch.bfloat16)
    with sdpa_kernel([backend]):
        f = lambda: torch.nn.functional.scaled_dot_product_attention(  # noqa: E731
            q, k, v, is_causal=True, enable_gqa=True)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def fa4(n: int, reps: int) -> float:
    """FlashAttention-4 (CuTe DSL sm100 kernel shipped with vllm): [b, s, h, d] layout."""
    import torch
    from vllm.vllm_flash_attn.cute.interface import flash_attn_func

    q = torch.randn(1, n, 32, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, n, 8, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(1, n, 8, 128, device="cuda", dtype=torch.bfloat16)
    f = lambda: flash_attn_func(q, k, v, causal=True)  # noqa: E731
    return _time(f, reps)


def flashinfer_prefill(n: int, reps: int) -> float:
    import flashinfer
    import torch

    q = torch.randn(n, 32, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(n, 8, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(n, 8, 128, device="cuda", dtype=torch.bfloat16)
    f = lambda: flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True)  # noqa: E731
    return _time(f, reps)


def _time(f, reps):
    import torch

    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--len", type=int, action="append", default=[])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ours-only", action="store_true")
    a = ap.parse_args()
    from torch.nn.attention import SDPBackend

    for n in a.len or [4465]:
        flops = 4 * 4096 * n * (n + 1) / 2
        rows = [("ours (tcgen05, paged KV)", ours(n, a.reps))]
        if a.ours_only:
            print(f"n={n:6d} ours {rows[0][1] * 1e3:9.1f} us  {flops / rows[0][1] / 1e9:8.1f} TFLOP/s")
            continue
        for name, be in (("torch sdpa cudnn", SDPBackend.CUDNN_ATTENTION),
                         ("torch sdpa flash", SDPBackend.FLASH_ATTENTION),
                         ("torch sdpa efficient", SDPBackend.EFFICIENT_ATTENTION)):
            try:
                rows.append((name, sdpa(n, a.reps, be)))
            except Exception as e:  # backend unavailable for this shape / arch
                print(f"n={n} {name}: unavailable ({str(e).splitlines()[0][:100]})")
        for name, fn in (("flash-attn 4 (cute dsl)", fa4), ("flashinfer prefill", flashinfer_prefill)):
            try:
                rows.append((name, fn(n, a.reps)))
            except Exception as e:
                print(f"n={n} {name}: unavailable ({str(e).splitlines()[0][:100] if str(e) else repr(e)})")
        for name, ms in rows:
            print(f"n={n:6d} {name:26s} {ms * 1e3:9.1f} us  {flops / ms / 1e9:8.1f} TFLOP/s")


if __name__ == "__main__":
    main()
