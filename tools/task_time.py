"""Device time of one Llama-3-8B-shape task per request length (events around the whole task,
no per-kernel events: programmatic dependent launch stays on), vs the GEMM-FLOP and weight-
streaming bounds.

    python tools/task_time.py [--len 42 --len 545 ...] [--reps 5]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--len", type=int, action="append", default=[])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--model", default="llama3-8b")
    a = ap.parse_args()
    lens = a.len or [42, 163, 386, 545, 872, 1572, 4465]
    sh = SHAPES[a.model]
    ctx = PrefillContext(sh, kv_pages=sum((n + 127) // 128 for n in lens) + 8, max_pos=40000)
    ctx.init_random(seed=0)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    d, q, kv, f = sh.hidden, sh.n_heads * 128, sh.n_kv_heads * 128, sh.ffn
    w_bytes = sh.num_layers * 2 * d * (q + 2 * kv + q + 3 * f)
    for n in lens:
        t = ctx.create_task([np.arange(n, dtype=np.int32) % sh.vocab], None, "operator", 1)
        for _ in range(2):
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)
        ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.reps):
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)
        e1.record(stream)
        ctx.sync()
        ms = e0.elapsed_time(e1) / a.reps
        flops = sh.num_layers * (2 * n * (d * (q + 2 * kv) + q * d + 3 * d * f) + 2 * q * n * (n + 1))
        print(f"M={n:5d} {ms:7.3f} ms  {flops / ms / 1e9:7.1f} TF/s  weight-stream bound "
              f"{w_bytes / 6.5e12 * 1e3:.2f} ms  flop bound@1300 {flops / 1.3e15 * 1e3:.2f} ms")
        t.destroy()
    ctx.close()


if __name__ == "__main__":
    main()
