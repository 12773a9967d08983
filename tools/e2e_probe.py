"""Where the e2e time goes: bench.py's e2e loop (config-2 step through the public API with host
buffers, double-buffered) with host-side phase timers and device events per step.

    python tools/e2e_probe.py [--steps 5]
Prints per step: host seconds in create_task / enqueue / logits read / destroy, and the device
time between consecutive step-end events (GPU-side step time incl. any idle)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    shape = SHAPES[bench.MODEL]
    reqs = bench.step_requests(1, 0)
    tokens = [np.random.default_rng(1000 + r.id).integers(0, shape.vocab, r.num_tokens)
              .astype(np.int32) for r in reqs]
    pages = sum((len(t) + 127) // 128 for t in tokens)
    ctx = PrefillContext(shape, device=0, kv_pages=3 * pages + 64, page_size=128, max_pos=40000)
    ctx.init_random(seed=0)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=0)
    T = {"create": 0.0, "enqueue": 0.0, "read": 0.0, "destroy": 0.0}

    def submit():
        live = []
        for i, t in enumerate(tokens):
            a = time.perf_counter()
            task = ctx.create_task([t], None, "operator", 10_000 + i)
            b = time.perf_counter()
            task.begin_segment(0)
            task.enqueue(0, task.n_entries)
            T["create"] += b - a
            T["enqueue"] += time.perf_counter() - b
            live.append(task)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        return live, ev

    for _ in range(2):  # warm-up (allocator pool, tensor maps, code paths)
        live, _ = submit()
        for t in live:
            t.logits()
            t.destroy()
    ctx.sync()
    for k in T:
        T[k] = 0.0
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    pending, evs = submit(), []
    for k in range(args.steps):
        nxt = submit() if k + 1 < args.steps else None
        a = time.perf_counter()
        for task in pending[0]:
            task.logits()
        b = time.perf_counter()
        for task in pending[0]:
            task.destroy()
        T["read"] += b - a
        T["destroy"] += time.perf_counter() - b
        evs.append(pending[1])
        pending = nxt
    ctx.sync()
    wall = time.perf_counter() - t0
    step_tok = sum(len(t) for t in tokens)
    prev, dev = e0, []
    for ev in evs:
        dev.append(prev.elapsed_time(ev))
        prev = ev
    print(f"wall {wall * 1e3:.1f} ms for {args.steps} steps -> {step_tok * args.steps / wall:.0f} tok/s")
    print("device step ms (end-to-end event gaps):", [round(x, 1) for x in dev])
    print("host ms per step:", {k: round(v * 1e3 / args.steps, 1) for k, v in T.items()})
    # device-only reference: the same tasks re-run (no create/destroy)
    tasks = [ctx.create_task([t], None, "operator", i) for i, t in enumerate(tokens)]
    for t in tasks:
        t.begin_segment(0)
        t.enqueue(0, t.n_entries)
    ctx.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)
    b.record(stream)
    ctx.sync()
    ms = a.elapsed_time(b) / args.steps
    print(f"device-only step {ms:.1f} ms -> {step_tok / ms * 1e3:.0f} tok/s")
    ctx.close()


if __name__ == "__main__":
    main()
