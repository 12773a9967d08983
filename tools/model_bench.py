"""Prefill throughput of one model shape on one B200 (default: the MoE Qwen3-30B-A3B shape, 48 layers,
128 experts, top-8, expert ffn 768), random bf16 weights, the bench's 16 config-2 request
lengths as separate preemptible tasks (operator-granularity checks armed).

    python tools/model_bench.py [--model qwen3-30b-a3b|qwen3-8b|llama3-8b|...] [--steps 3]

Reports tokens/s (CUDA events on the prefill stream) and the per-kernel-kind time and TFLOP/s
of one profiled step; FLOPs count the router and the top_k active experts only.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LENS = [4465, 163, 3971, 545, 386, 3997, 1572, 504, 42, 438, 451, 1021, 872, 437, 5389, 853]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--model", default="qwen3-30b-a3b")
    ap.add_argument("--out", default="gpurun_out/moe_bench.json")
    a = ap.parse_args()
    import torch

    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape = SHAPES[a.model]
    pages = sum((n + 127) // 128 for n in LENS)
    ctx = PrefillContext(shape, kv_pages=pages + 16, page_size=128, max_pos=8192)
    ctx.init_random(seed=0)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    toks = [np.random.default_rng(1000 + i).integers(0, shape.vocab, n).astype(np.int32)
            for i, n in enumerate(LENS)]
    tasks = [ctx.create_task([t], None, "operator", i) for i, t in enumerate(toks)]

    def step():
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)

    for _ in range(2):
        step()
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    ctx.sync()
    ms = e0.elapsed_time(e1) / a.steps
    ctx.profile(True)
    ctx.drain_profile()
    step()
    ctx.sync()
    prof = ctx.drain_profile()
    ctx.profile(False)
    kinds = {}
    for r in prof:
        k = kinds.setdefault(r["kind"], {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
        k["launches"] += 1
        k["ms"] += r["ms"]
        k["flops"] += r["flops"]
        k["bytes"] += r["bytes"]
    for k in kinds.values():
        k["tflops"] = round(k["flops"] / (k["ms"] * 1e-3) / 1e12, 1) if k["flops"] else None
        k["gbs"] = round(k["bytes"] / (k["ms"] * 1e-3) / 1e9, 1) if k["bytes"] else None
        k["ms"] = round(k["ms"], 3)
        del k["flops"], k["bytes"]
    tokens = sum(LENS)
    out = {
        "metric": "prefill_tokens_per_s",
        "model": a.model,
        "value": tokens / (ms * 1e-3),
        "unit": "tok/s",
        "ms_per_step": round(ms, 3),
        "tokens_per_step": tokens,
        "requests": LENS,
        "active_gemm_flops_per_token": shape.gemm_flops_per_token() * shape.num_layers,
        "kernels": kinds,
        "data": "synthetic (random-init bf16 weights, seeded token ids)",
    }
    print(json.dumps(out))
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    for t in tasks:
        t.destroy()
    ctx.close()


if __name__ == "__main__":
    main()
