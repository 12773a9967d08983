"""GPU drop-in for the reference execution pool (virtual-clock parity mode).

``prefillsim.engine.run`` (engine.py:384-545) resolves ``Engine`` (engine.py:504),
``ExecutionTask`` (engine.py:445) and ``build_timeline`` (engine.py:440) as module globals at
call time. ``run_on_gpu`` substitutes ``GpuEngine`` / ``GpuTask`` there -- no reference edit --
so the reference scheduler (``schedule_round``), the event heap, the virtual clock and every
hook run unchanged, while each BOUNDARY event executes that timeline entry's kernels on the
B200 and each ACK is realised by the device-side boundary check:

* ``GpuTask`` = ``ExecutionTask`` + a native task whose entry list is cross-checked against the
  reference timeline (same count, same (chunk, layer, kind) at every index).
* ``GpuEngine.step`` launches entry ``b`` when its live BOUNDARY event pops
  (engine.py:300-305), so completed work is never re-run (work conservation).
* ``GpuEngine._finalize_ack`` sets the pinned preemption flag and launches the next entry; the
  device check in front of it must stop and publish exactly the reference cursor
  ``ack_index + 1`` (engine.py:279-291), else ``SchedulerInvariantError``.
* ``_schedule_segment`` (submit/resume, engine.py:193-238) re-arms the device checks from the
  cursor under a new generation.

Because the clock is the reference's own cost model, event logs are bit-identical by
construction; what this mode proves is that the GPU path follows the same cursor semantics and
produces the logits/KV of an uninterrupted run.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib, refsim
from .native import PrefillContext

ps = refsim.load()
from prefillsim import engine as _ref_engine  # noqa: E402
from prefillsim.engine import (  # noqa: E402
    Engine,
    ExecutionTask,
    SchedulerInvariantError,
    TaskState,
    tp_sync_check,
)

_BOUNDARY = _ref_engine._BOUNDARY
_OP_NAMES = ("qkv_proj", "attn", "o_proj", "gate_up_proj", "down_proj")  # DENSE_LAYER_OPS
_MOE_OP_NAMES = ("qkv_proj", "attn", "o_proj", "gate", "experts")       # MOE_LAYER_OPS


def synthetic_tokens(seed: int, vocab: int) -> Callable:
    """Token ids of a request: default_rng(seed + id).integers(0, vocab, n)."""

    def tokens(req) -> np.ndarray:
        return np.random.default_rng(seed + req.id).integers(0, vocab, req.num_tokens).astype(
            np.int32
        )

    return tokens


@dataclass
class GpuBinding:
    ctx: PrefillContext
    tokens: Callable
    chunk_tokens: Optional[int] = None
    granularity: str = "operator"
    collect_logits: bool = True
    check_timeline: bool = True
    logits: dict = field(default_factory=dict)  # request id -> fp32 logits
    handshakes: list = field(default_factory=list)  # (task, reference cursor, device cursor)
    entries_run: int = 0


class GpuTask(ExecutionTask):
    """ExecutionTask whose timeline entries are GPU kernel groups."""

    __slots__ = ("native", "binding")

    def __init__(self, task_id, members, timeline, *, binding: GpuBinding):
        super().__init__(task_id, members, timeline)
        self.binding = binding
        self.native = binding.ctx.create_task(
            [binding.tokens(r) for r in members],
            binding.chunk_tokens,
            binding.granularity,
            task_id,
        )
        if self.native.n_entries != len(timeline):
            raise SchedulerInvariantError(
                f"native timeline has {self.native.n_entries} entries, reference {len(timeline)}"
            )
        if binding.check_timeline:
            names = _MOE_OP_NAMES if binding.ctx.shape.moe else _OP_NAMES
            for i, e in enumerate(timeline.entries):
                c, l, o, _ = self.native.entry_info(i)
                if (c, l, names[o]) != (e.chunk, e.layer, e.kind.value):
                    raise SchedulerInvariantError(f"entry {i} mismatch: {(c, l, o)} vs {e}")


class GpuEngine(Engine):
    """Engine whose entries execute on the GPU; virtual time stays the reference's."""

    def __init__(self, params, granularity, on_arrival=None, on_completion=None, on_ack=None, *,
                 binding: GpuBinding):
        want = "moe" if binding.ctx.shape.moe else "dense"
        if params.arch != want:
            raise SchedulerInvariantError(
                f"cost model arch {params.arch!r} but the GPU model is {want!r}")
        if params.num_layers != binding.ctx.shape.num_layers:
            raise SchedulerInvariantError(
                f"cost model has {params.num_layers} layers, GPU model "
                f"{binding.ctx.shape.num_layers}"
            )
        super().__init__(params, granularity, on_arrival, on_completion, on_ack)
        self.binding = binding

    def _schedule_segment(self, task, now):
        task.native.begin_segment(task.cursor)
        return super()._schedule_segment(task, now)

    def step(self) -> bool:
        if self._heap:
            _, _, kind, a, b, c = self._heap[0]
            if kind == _BOUNDARY:
                task = self.tasks[a]
                if c == task.generation and task.state is TaskState.RUNNING:
                    task.native.enqueue(b, b + 1)
                    self.binding.entries_run += 1
        return super().step()

    def _finalize_completion(self, task, now):
        if self.binding.collect_logits:
            lg = task.native.logits()
            for j, r in enumerate(task.member_requests):
                self.binding.logits[r.id] = lg[j]
        else:
            self.binding.ctx.sync()
        task.native.destroy()
        super()._finalize_completion(task, now)

    def _finalize_ack(self, task, ack_index, now):
        if task.state is not TaskState.DONE:
            nxt = ack_index + 1
            ctx = self.binding.ctx
            ctx.sync()  # entries <= ack_index (launched asynchronously) have completed
            ctx.signal()
            task.native.enqueue(nxt, nxt + 1)
            ctx.sync()
            if hasattr(task.native, "poll_all"):
                # tensor parallel: every rank must have stopped at the same entry -- the
                # reference's lane gate (tp_sync_check, engine.py:50-57,254-255) over the
                # device cursors of all ranks
                lanes = task.native.poll_all()
                if not tp_sync_check([s.cursor for s in lanes]):
                    raise SchedulerInvariantError(
                        f"TP ranks stopped at different entries: {[s.cursor for s in lanes]}")
            st = task.native.poll()
            self.binding.handshakes.append((task.task_id, nxt, st.cursor, st.state))
            if st.state != _lib.FP_TASK_STOPPED or st.cursor != nxt:
                raise SchedulerInvariantError(
                    f"device boundary check stopped task {task.task_id} at {st.cursor} "
                    f"(state {st.state}); reference cursor {nxt}"
                )
        super()._finalize_ack(task, ack_index, now)


def run_on_gpu(trace, policy_config, cost_params, binding: GpuBinding, seed: int = 0,
               record_events: bool = False):
    """The reference ``run()`` with the GPU execution pool injected (no reference edits)."""
    binding.chunk_tokens = policy_config.chunk_tokens
    binding.granularity = policy_config.granularity.value
    orig_engine, orig_task = _ref_engine.Engine, _ref_engine.ExecutionTask
    _ref_engine.Engine = lambda *a, **k: GpuEngine(*a, binding=binding, **k)
    _ref_engine.ExecutionTask = lambda tid, members, tl: GpuTask(tid, members, tl, binding=binding)
    try:
        return _ref_engine.run(trace, policy_config, cost_params, seed, record_events)
    finally:
        _ref_engine.Engine, _ref_engine.ExecutionTask = orig_engine, orig_task
