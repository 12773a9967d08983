"""Run one Llama-3-8B-shape prefill task (for ncu launch lists / full captures).

    python tools/prof_task.py --len 4096 [--len 512 ...] [--reps 2]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--len", type=int, action="append", default=[])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--layers", type=int, default=0, help="override layer count (0 = model)")
    ap.add_argument("--profile", action="store_true", help="print per-kernel event timings")
    a = ap.parse_args()
    lens = a.len or [4096]
    shape = SHAPES[a.model]
    if a.layers:
        from dataclasses import replace
        shape = replace(shape, num_layers=a.layers)
    ctx = PrefillContext(shape, kv_pages=sum((n + 127) // 128 for n in lens) + 8, max_pos=40000)
    ctx.init_random(0)
    toks = [np.random.default_rng(i).integers(0, shape.vocab, n).astype(np.int32)
            for i, n in enumerate(lens)]
    tasks = [ctx.create_task([t]) for t in toks]
    for r in range(a.reps):
        if a.profile and r == a.reps - 1:
            ctx.profile(True)
            ctx.drain_profile()
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)
        ctx.sync()
    if a.profile:
        recs = ctx.drain_profile()
        agg = {}
        for rec in recs:
            k = (rec["kind"], rec["M"])
            v = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
            v[0] += 1; v[1] += rec["ms"]; v[2] += rec["flops"]; v[3] += rec["bytes"]
        for (kind, m), (n, ms, fl, by) in sorted(agg.items()):
            rate = f"{fl / ms / 1e9:8.1f} TFLOP/s" if fl else f"{by / ms / 1e6:8.1f} GB/s"
            print(f"{kind:14s} M={m:6d} n={n:4d} avg {ms / n * 1e3:9.1f} us  {rate}")
    ctx.close()


if __name__ == "__main__":
    main()
