"""Per-request breakdown of the bench step: for every request length of the config-2 step, the
event-timed milliseconds and TFLOP/s of each kernel kind (profiled run: events around every
kernel), to see where short / mid requests lose time against the long ones.

    python tools/step_breakdown.py [--model llama3-8b]
"""
import argparse
import collections
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default=bench.MODEL)
    ap.add_argument("--out", default="gpurun_out/step_breakdown.json")
    args = ap.parse_args()
    shape = SHAPES[args.model]
    reqs = bench.step_requests(1, 0)
    tokens = [np.random.default_rng(1000 + r.id).integers(0, shape.vocab, r.num_tokens)
              .astype(np.int32) for r in reqs]
    pages = sum((len(t) + 127) // 128 for t in tokens)
    ctx = PrefillContext(shape, device=0, kv_pages=pages + 64, page_size=128, max_pos=40000)
    ctx.init_random(seed=0)
    tasks = [ctx.create_task([t], None, "operator", i) for i, t in enumerate(tokens)]
    for _ in range(2):
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)
    ctx.sync()
    ctx.profile(True)
    ctx.drain_profile()
    for t in tasks:
        t.begin_segment(0)
        t.enqueue(0, t.n_entries)
    recs = ctx.drain_profile()
    ctx.profile(False)
    by = collections.defaultdict(lambda: collections.defaultdict(lambda: [0.0, 0.0]))
    for r in recs:
        a = by[r["M"]][r["kind"]]
        a[0] += r["ms"]
        a[1] += r["flops"]
    out = {}
    total = sum(r["ms"] for r in recs)
    print(f"step (profiled) {total:.1f} ms")
    for M in sorted(by):
        row = {k: {"ms": round(v[0], 3), "tflops": round(v[1] / (v[0] * 1e-3) / 1e12, 1) if v[1] else None}
               for k, v in by[M].items()}
        ms = sum(v[0] for v in by[M].values())
        fl = sum(v[1] for v in by[M].values())
        out[M] = {"ms": round(ms, 3), "tflops": round(fl / (ms * 1e-3) / 1e12, 1), "kinds": row}
        print(f"M={M:5d} {ms:7.2f} ms {fl / (ms * 1e-3) / 1e12:7.1f} TF/s  " +
              " ".join(f"{k}:{v['ms']:.2f}/{v['tflops']}" for k, v in row.items()))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump({"model": args.model, "step_ms": total, "by_M": out}, fh, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
