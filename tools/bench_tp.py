#!/usr/bin/env python
"""Tensor-parallel prefill measurement (BASELINE config 4: Qwen2.5-32B shape, TP = 1/2/4/8).

    python tools/bench_tp.py [--tp 1 2 4 8] [--steps K] [--warmup W] [--out FILE]
    torchrun --nproc-per-node T tools/bench_tp.py --tp T      (one process per GPU)

One step = prefill of the first 8 requests of the config-2 trace (seed 7), one task each,
operator-granularity checks armed, random-init bf16 weights.

* Under torchrun (WORLD_SIZE == T): each process is one rank on its own GPU, connected through
  CUDA IPC (connect_tp_dist); device time on rank 0's stream, max over ranks.
* In one process (the 1-GPU box): the T ranks run in lock step on ONE device
  (TPGroup / fp_tp_enqueue_lockstep). The step time then serialises the ranks, so the line
  reports it as `emulated_step_ms` next to `per_rank_kernel_ms` (the max over ranks of the
  summed kernel times of one rank = the device work each GPU of a real TP=T group does; the
  all-reduce there reads peers over NVLink instead of local HBM). Nothing here is a TP=T
  multi-GPU throughput claim.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

MODEL = "qwen2.5-32b"
N_REQ = 8


def requests():
    tr = bench.config2_trace(8.0, 300.0)
    return tr.requests[:N_REQ]


def summarize(prof, steps):
    out = {}
    for r in prof:
        k = out.setdefault(r["kind"], {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
        k["launches"] += 1
        k["ms"] += r["ms"] / steps
        k["flops"] += r["flops"] / steps
        k["bytes"] += r["bytes"] / steps
    for k in out.values():
        k["tflops"] = round(k["flops"] / (k["ms"] * 1e-3) / 1e12, 1) if k["flops"] else None
        k["gbs"] = round(k["bytes"] / (k["ms"] * 1e-3) / 1e9, 1) if k["bytes"] else None
        k["ms"] = round(k["ms"], 3)
        del k["flops"], k["bytes"]
    return out


def run_local(tp, steps, warmup):
    import torch

    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext, TPGroup

    shape = SHAPES[MODEL]
    reqs = requests()
    tokens = [np.random.default_rng(1000 + r.id).integers(0, shape.vocab, r.num_tokens)
              .astype(np.int32) for r in reqs]
    n_tok = int(sum(len(t) for t in tokens))
    pages = sum((len(t) + 127) // 128 for t in tokens) + 8
    max_m = max(len(t) for t in tokens)
    if tp == 1:
        g = PrefillContext(shape, kv_pages=pages, max_pos=40000)
    else:
        g = TPGroup(shape, tp, kv_pages=pages, max_pos=40000, max_tokens=max_m)
    g.init_random(seed=0)
    stream = torch.cuda.ExternalStream(g.stream_ptr, device=0)
    tasks = [g.create_task([t], None, "operator", i) for i, t in enumerate(tokens)]

    def step():
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)

    for _ in range(warmup):
        step()
    g.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    g.sync()
    ms = e0.elapsed_time(e1) / steps
    g.profile(True)
    g.drain_profile()
    step()
    prof = g.drain_profile()
    g.profile(False)
    ranks = {}
    for r in prof:
        ranks.setdefault(r.get("rank", 0), []).append(r)
    per_rank_ms = max(sum(x["ms"] for x in v) for v in ranks.values())
    kern = summarize(ranks[0], 1)
    xchg_ms = kern.get("tp_allreduce", {}).get("ms", 0.0)
    for t in tasks:
        t.destroy()
    g.close()
    return {
        "tp": tp, "model": MODEL, "requests": [len(t) for t in tokens], "tokens_per_step": n_tok,
        "mode": "single instance" if tp == 1 else f"{tp} ranks in lock step on one GPU",
        "emulated_step_ms": round(ms, 3),
        "emulated_tokens_per_s": round(n_tok / (ms * 1e-3), 1),
        "per_rank_kernel_ms": round(per_rank_ms, 3),
        "per_rank_allreduce_ms": round(xchg_ms, 3),
        "rank0_kernels": kern,
    }


def run_dist(tp, steps, warmup):
    import torch
    import torch.distributed as dist

    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext, connect_tp_dist

    ws, rank, local = bench.dist_env()
    assert ws == tp, "run one process per rank: WORLD_SIZE must equal --tp"
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shape = SHAPES[MODEL]
    reqs = requests()
    tokens = [np.random.default_rng(1000 + r.id).integers(0, shape.vocab, r.num_tokens)
              .astype(np.int32) for r in reqs]
    n_tok = int(sum(len(t) for t in tokens))
    pages = sum((len(t) + 127) // 128 for t in tokens) + 8
    ctx = PrefillContext(shape, device=local, kv_pages=pages, max_pos=40000, tp_rank=rank,
                         tp_size=tp)
    connect_tp_dist(ctx, max(len(t) for t in tokens))
    ctx.init_random(seed=0)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=local)
    tasks = [ctx.create_task([t], None, "operator", i) for i, t in enumerate(tokens)]

    def step():
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)

    for _ in range(warmup):
        step()
    ctx.sync()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    ctx.sync()
    dist.barrier()
    v = torch.tensor([e0.elapsed_time(e1) / steps], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    ms = float(v.item())
    for t in tasks:
        t.destroy()
    ctx.close()
    dist.destroy_process_group()
    if rank == 0:
        return {"tp": tp, "model": MODEL, "mode": f"{tp} processes, one GPU each (CUDA IPC)",
                "step_ms": round(ms, 3), "tokens_per_s": round(n_tok / (ms * 1e-3), 1),
                "tokens_per_step": n_tok}
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rows = []
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        r = run_dist(args.tp[0], args.steps, args.warmup)
        if r:
            rows.append(r)
    else:
        for tp in args.tp:
            rows.append(run_local(tp, args.steps, args.warmup))
            print(json.dumps(rows[-1]), flush=True)
    if args.out and rows:
        with open(args.out, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
