"""Device time of the bench step (16 config-2 request lengths, one task each) WITHOUT per-kernel
profiling events, so inter-kernel overlap (programmatic dependent launch) is measured too.

    python tools/step_time.py [--steps 5] [--model llama3-8b]     (FP_AB_LIB selects a build)
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LENS = [4465, 163, 3971, 545, 386, 3997, 1572, 504, 42, 438, 451, 1021, 872, 437, 5389, 853]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--granularity", default="operator",
                    help="none: no boundary is eligible, so no kernel reads the host flag")
    a = ap.parse_args()
    import torch

    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    shape = SHAPES[a.model]
    ctx = PrefillContext(shape, kv_pages=sum((n + 127) // 128 for n in LENS) + 16,
                         page_size=128, max_pos=8192)
    ctx.init_random(seed=0)
    st = torch.cuda.ExternalStream(ctx.stream_ptr)
    tasks = [ctx.create_task([np.random.default_rng(i).integers(0, shape.vocab, n).astype(np.int32)],
                             None, a.granularity)
             for i, n in enumerate(LENS)]

    def step():
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)

    for _ in range(2):
        step()
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        step()
    e1.record(st)
    ctx.sync()
    ms = e0.elapsed_time(e1) / a.steps
    print(f"STEP_MS {ms:.3f} TOKS {sum(LENS) / ms * 1e3:.0f}")
    for t in tasks:
        t.destroy()
    ctx.close()


if __name__ == "__main__":
    main()
