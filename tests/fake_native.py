"""CPU stand-in for the native context, used to test the host-side engine logic without a GPU.

It mirrors the C ABI's observable semantics (include/flowprefill.h): entries run in order inside
a segment, the boundary check in front of entry e stops iff a signal is pending and the boundary
after e-1 is eligible under the task's granularity and e is not the segment's first entry; a
stopped generation's queued entries are no-ops. Numbers come from the fp32 oracle (test
infrastructure), so the engine's logits can be compared with uninterrupted oracle runs.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from oracle import forward as F

STOPPED, DONE, RUNNING = 2, 3, 1


class FakeTask:
    def __init__(self, ctx, tokens, chunk, gran, task_id):
        self.ctx = ctx
        self.oracle = F.OracleTask(ctx.oshape, ctx.weights, list(tokens), chunk)
        self.n_entries = len(self.oracle)
        self.gran = gran
        self.task_id = task_id
        self.gen = 0
        self.seg_first = 0
        self.stopped_gen = -1
        self.state = 0
        self.cursor = 0
        self.executed = []  # entry indices actually executed
        self.destroyed = False

    def entry_info(self, i):
        c, l, o = self.oracle.entry(i)
        return c, l, o, self.oracle.chunks[c].new_total

    def info(self):
        return {"n_entries": self.n_entries}

    def _eligible_after(self, i):
        L = self.ctx.oshape.num_layers
        op, layer = i % 5, (i // 5) % L
        last = i == self.n_entries - 1
        if self.gran == "operator":
            return True
        if self.gran == "layer":
            return op == 4 or last
        if self.gran == "chunk":
            return (op == 4 and layer == L - 1) or last
        return False

    def begin_segment(self, first):
        self.gen += 1
        self.seg_first = first
        self.state = RUNNING

    def enqueue(self, first, last):
        for e in range(first, last):
            if self.stopped_gen == self.gen:
                continue
            if e != self.seg_first and self._eligible_after(e - 1) and self.ctx.flag:
                self.ctx.flag = 0
                self.stopped_gen = self.gen
                self.state = STOPPED
                self.cursor = e
                self.ctx.ack_seq += 1
                continue
            assert e == len(self.executed), "entries must execute in order exactly once"
            if self.ctx.compute:
                self.oracle.run(e, e + 1)
            self.executed.append(e)
            self.cursor = e + 1
        if self.cursor == self.n_entries and self.state != STOPPED:
            self.state = DONE

    def poll(self):
        return SimpleNamespace(state=self.state, cursor=self.cursor, generation=self.gen)

    def logits(self):
        return self.oracle.logits.copy()

    def destroy(self):
        self.destroyed = True


class FakeContext:
    def __init__(self, shape_name="tiny", seed=1234, num_layers=None, compute=True):
        self.compute = compute
        base = F.SHAPES[shape_name]
        if num_layers is not None:
            base = F.Shape(num_layers, base.hidden, base.n_heads, base.n_kv_heads, base.head_dim,
                           base.ffn, base.vocab, base.rope_theta, base.rms_eps)
        self.oshape = base
        self.shape = base
        self.weights = F.make_weights(base, seed)
        self.flag = 0
        self.ack_seq = 0
        self.tasks = []

    def create_task(self, tokens, chunk, gran, task_id):
        t = FakeTask(self, tokens, chunk, gran, task_id)
        self.tasks.append(t)
        return t

    def signal(self):
        self.flag = 1

    def clear(self):
        self.flag = 0

    def sync(self):
        pass

    def free_pages(self):
        return 0


class FakeLiveTask:
    """Wall-clock fake of an asynchronously running native task: each entry takes `entry_s`
    seconds; a pending signal stops it at the next eligible boundary."""

    def __init__(self, ctx, tokens, chunk, gran, task_id):
        import time

        self.ctx = ctx
        self.time = time
        lens = [len(t) for t in tokens]
        n_chunks = len(F.plan(lens, chunk))
        self.n_entries = n_chunks * ctx.num_layers * 5
        self.gran = gran
        self.task_id = task_id
        self.state = 0
        self.cursor = 0
        self.seg_first = 0
        self.t_start = None
        self.starts = []
        self.destroyed = False

    def _eligible_after(self, i):
        L = self.ctx.num_layers
        op, layer = i % 5, (i // 5) % L
        last = i == self.n_entries - 1
        return {"operator": True, "layer": op == 4 or last,
                "chunk": (op == 4 and layer == L - 1) or last}.get(self.gran, False)

    def start(self, first):
        assert self.state != RUNNING
        self.seg_first = first
        self.cursor = first
        self.t_start = self.time.perf_counter()
        self.state = RUNNING
        self.starts.append(first)

    def poll(self):
        if self.state == RUNNING:
            done = self.seg_first + int((self.time.perf_counter() - self.t_start) / self.ctx.entry_s)
            while self.cursor < min(done, self.n_entries):
                e = self.cursor
                if e != self.seg_first and self.ctx.flag and self._eligible_after(e - 1):
                    self.ctx.flag = 0
                    self.state = STOPPED
                    break
                self.cursor += 1
            if self.state == RUNNING and self.cursor >= self.n_entries:
                self.state = DONE
        return SimpleNamespace(state=self.state, cursor=self.cursor, generation=0)

    def max_entry_s(self):
        return self.ctx.entry_s

    def destroy(self):
        self.destroyed = True


class FakeLiveContext:
    def __init__(self, num_layers=2, entry_s=50e-6):
        self.num_layers = num_layers
        self.entry_s = entry_s
        self.flag = 0
        self.tasks = []

    def create_task(self, tokens, chunk, gran, task_id):
        t = FakeLiveTask(self, tokens, chunk, gran, task_id)
        self.tasks.append(t)
        return t

    def signal(self):
        self.flag = 1

    def clear(self):
        self.flag = 0
