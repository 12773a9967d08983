"""Wall-clock driver: the reference scheduler driving the GPU execution pool in real time.

``prefillsim.engine.run`` (engine.py:384-545) advances a virtual clock. Here the same event
semantics run against the wall clock and the real device:

* arrivals are released at ``t0 + request.arrival_time``;
* every arrival and completion triggers one reference ``schedule_round`` (scheduler.py:175);
* a round that starts with ``preempt`` sets the pinned flag (``fp_signal``) and PARKS its
  follow-up submit/resume until the device ACK (engine.py:429-435, 490-495); arrivals and
  completions observed while the ACK is outstanding are buffered and their rounds deferred to
  the ACK instant (engine.py:468-470, 484-486, 496-502);
* an ACK that races the task's natural completion resolves as completion-wins
  (engine.py:279-291);
* the scheduler reads ``task.progress()`` from the device-published cursor.

Outcomes, blocking log, round and command counts have the reference ``RunResult`` shape, so
the reference metrics (``slo_attainment``, ``blocking_stats``) apply unchanged.
"""

from __future__ import annotations

import time
from collections import deque
from typing import Callable, Optional

from . import _lib, refsim
from .native import PrefillContext

ps = refsim.load()
from prefillsim.engine import ExecutionTask, RequestOutcome, RunResult, TaskStats  # noqa: E402
from prefillsim.scheduler import SchedulerState, schedule_round  # noqa: E402


class LiveTask(ExecutionTask):
    """ExecutionTask whose cursor is the device-published progress of its native task."""

    __slots__ = ("native", "submit_t")

    def refresh(self) -> None:
        st = self.native.poll()
        if st.state == _lib.FP_TASK_RUNNING:
            self.cursor = max(self.cursor, min(st.cursor, len(self) - 1))


def run_live(
    trace,
    policy_config,
    cost_params,
    ctx: PrefillContext,
    tokens: Callable,
    predictor=None,
    record_events: bool = False,
    time_scale: float = 1.0,
    max_wall_s: Optional[float] = None,
    round_log: Optional[list] = None,
) -> RunResult:
    """Replay ``trace`` in real time on ``ctx``. ``cost_params`` only shapes the timeline
    bookkeeping (progress weights) and, when ``predictor`` is None, the reference's
    self-calibrated TTFT predictor; pass B200-calibrated params (calibrate.py).

    ``round_log`` (a list) receives one record per scheduling round -- its wall time, the
    arrivals and completions it consumes, the cursor of every live task as the scheduler saw
    it, and the commands it returned -- for ``replay_rounds`` (SURVEY.md §7 hard part 5)."""
    if predictor is None:
        predictor = policy_config.predictor  # as the reference run() does (engine.py:399-406)
    if predictor is None:
        predictor = ps.self_calibrated_poly(
            cost_params, degree=policy_config.predictor_degree,
            chunk_size=policy_config.chunk_tokens)
    state = SchedulerState.create(policy_config, predictor)
    gran = policy_config.granularity.value
    events = [] if record_events else None
    counts = {"submit": 0, "preempt": 0, "resume": 0}
    outcomes: dict = {}
    tasks: dict = {}
    blocking: list = []
    rounds = 0
    followup: list = []
    buffered: deque = deque()
    running: Optional[LiveTask] = None
    pending_signal = False
    signal_t = 0.0
    t0 = time.perf_counter()

    def now() -> float:
        return (time.perf_counter() - t0) * time_scale

    def log(kind, task, t, **detail):
        if events is not None:
            events.append({"t": t, "kind": kind, "task": task, "detail": detail})

    noted: list = []  # completions noted since the last round (note_completion order)

    def note(task_id):
        state.note_completion(task_id)
        noted.append(task_id)

    def do_round(t, arrivals, trigger):
        nonlocal rounds, noted
        rounds += 1
        if running is not None:
            running.refresh()
        if round_log is not None:
            live = [running] if running is not None else []
            live += [x for x in state.q_preempted.values()]
            rec = {"round": rounds, "t": t, "trigger": trigger,
                   "arrivals": [r.id for r in arrivals], "completions": noted,
                   "cursors": {x.task_id: x.cursor for x in live},
                   "running": running.task_id if running is not None else None}
        noted = []
        cmds = schedule_round(state, t, arrivals)
        if round_log is not None:
            rec["commands"] = [command_key(c) for c in cmds]
            round_log.append(rec)
        execute(cmds, t)

    def execute(cmds, t):
        nonlocal followup, pending_signal, signal_t
        if not cmds:
            return
        if cmds[0].kind == "preempt":
            counts["preempt"] += 1
            log("preempt_signal", cmds[0].task_id, t)
            if running is None or running.task_id != cmds[0].task_id:
                raise ps.SchedulerInvariantError("preempt of a task that is not running")
            pending_signal = True
            signal_t = t
            ctx.signal()
            followup = list(cmds[1:])
        else:
            run_now(cmds, t)

    def run_now(cmds, t):
        nonlocal running
        for c in cmds:
            if running is not None:
                raise ps.SchedulerInvariantError(f"{c.kind} at t={t}: pool occupied")
            if c.kind == "submit":
                tl = ps.build_timeline([r.num_tokens for r in c.members],
                                       policy_config.chunk_tokens, cost_params)
                task = LiveTask(c.task_id, c.members, tl)
                task.native = ctx.create_task([tokens(r) for r in c.members],
                                              policy_config.chunk_tokens, gran, c.task_id)
                task.submit_t = t
                tasks[c.task_id] = task
                state.attach_task(task)
                task.state = ps.TaskState.RUNNING
                task.native.start(0)
                running = task
                counts["submit"] += 1
                log("submit", c.task_id, t, members=[r.id for r in c.members],
                    tokens=task.agg_tokens)
            elif c.kind == "resume":
                task = tasks[c.task_id]
                task.state = ps.TaskState.RUNNING
                task.resume_count += 1
                task.native.start(task.cursor)
                running = task
                counts["resume"] += 1
                log("resume", c.task_id, t, cursor=task.cursor)
            else:
                raise ps.SchedulerInvariantError(f"unexpected command {c.kind}")

    def on_arrival(req, t):
        log("arrival", None, t, request=req.id, tokens=req.num_tokens)
        if pending_signal:
            buffered.append(("arrival", req))
        else:
            do_round(t, [req], "arrival")

    def finish(task, t):
        for r in task.member_requests:
            outcomes[r.id] = RequestOutcome(id=r.id, task=r.task, arrival_s=r.arrival_time,
                                            tokens=r.num_tokens, slo_s=r.ttft_slo,
                                            prefill_end_s=t)
        task.cursor = len(task)
        task.state = ps.TaskState.DONE
        log("completion", task.task_id, t, requests=[r.id for r in task.member_requests])
        if round_log is not None:
            # measured longest entry (device stamps): the task's wall-clock blocking bound
            round_log.append({"done": task.task_id, "t": t,
                              "max_entry_s": task.native.max_entry_s()})
        task.native.destroy()

    def on_completion(task, t):
        nonlocal running
        running = None
        finish(task, t)
        if pending_signal:
            buffered.append(("completion", task.task_id))
        else:
            note(task.task_id)
            do_round(t, [], "completion")

    def on_ack(task, cursor, t):
        nonlocal running, pending_signal, followup
        running = None
        pending_signal = False
        task.cursor = cursor
        task.state = ps.TaskState.PREEMPTED
        task.generation += 1
        blocking.append((signal_t, t, task.task_id))
        log("preempt_ack", task.task_id, t, blocking_s=t - signal_t, cursor=cursor)
        if round_log is not None:
            round_log.append({"ack": task.task_id, "t": t, "cursor": cursor})
        pending, followup = followup, []
        run_now(pending, t)
        drain_buffer(t)

    def drain_buffer(t):
        while buffered and not pending_signal:
            kind, payload = buffered.popleft()
            if kind == "arrival":
                do_round(t, [payload], "deferred_arrival")
            else:
                note(payload)
                do_round(t, [], "deferred_completion")

    reqs = list(trace.requests)
    i = 0
    while i < len(reqs) or running is not None or buffered or pending_signal:
        t = now()
        if max_wall_s is not None and t > max_wall_s:
            raise TimeoutError(f"live run exceeded {max_wall_s} s")
        if running is not None:
            st = running.native.poll()
            if st.state == _lib.FP_TASK_DONE:
                task = running
                if pending_signal:
                    # completion wins the race with the ACK (engine.py:280-283)
                    ctx.clear()
                    running = None
                    finish(task, t)
                    pending_signal = False
                    blocking.append((signal_t, t, task.task_id))
                    log("preempt_ack", task.task_id, t, blocking_s=t - signal_t,
                        cursor=len(task))
                    if round_log is not None:
                        round_log.append({"ack": task.task_id, "t": t, "cursor": len(task),
                                          "completed": True})
                    buffered.append(("completion", task.task_id))
                    pending, followup = followup, []
                    run_now(pending, t)
                    drain_buffer(t)
                else:
                    on_completion(task, t)
                continue
            if st.state == _lib.FP_TASK_STOPPED:
                on_ack(running, st.cursor, t)
                continue
        if i < len(reqs) and reqs[i].arrival_time <= t:
            on_arrival(reqs[i], t)
            i += 1
            continue
        if running is None and not buffered and not pending_signal and i < len(reqs):
            # idle: sleep until the next arrival
            dt = reqs[i].arrival_time - now()
            if dt > 2e-3:
                time.sleep(dt - 1e-3)

    stats = [
        TaskStats(task_id=t.task_id, members=tuple(r.id for r in t.member_requests),
                  agg_tokens=t.agg_tokens, n_entries=len(t),
                  total_s=t.timeline.total_duration, executed_s=0.0,
                  max_entry_s=t.timeline.max_entry_duration(), resume_count=t.resume_count)
        for t in tasks.values()
    ]
    return RunResult(
        outcomes=[outcomes[r.id] for r in trace.requests],
        blocking_log=blocking,
        rounds=rounds,
        commands=counts,
        tasks=stats,
        batch_audit=list(state.batch_audit),
        seed=0,
        policy=policy_config.policy.value,
        granularity=policy_config.granularity.value,
        events=events,
    )


def command_key(c) -> list:
    """A scheduler ``Command`` (scheduler.py:118-125) as plain data: kind, task, member ids,
    aggregate tokens."""
    return [c.kind, c.task_id, [r.id for r in c.members], c.agg_tokens]


def replay_rounds(trace, policy_config, cost_params, round_log: list, predictor=None) -> dict:
    """Replay a live run's scheduling rounds through a FRESH reference ``SchedulerState`` and
    ``schedule_round`` (scheduler.py:175-245) and check the live driver's protocol against the
    reference ``run()`` semantics (engine.py:419-502). SURVEY.md §7 hard part 5.

    Every round is re-evaluated at its logged wall time with the logged arrivals, the
    completions noted before it, and each live task's cursor as the scheduler saw it (tasks
    are fresh reference ``ExecutionTask`` objects over ``build_timeline``); the commands must
    be identical. The log must also show: every request arriving exactly once; no round and
    no submit/resume between a preempt signal and its ACK; rounds deferred by an outstanding
    signal running at the ACK instant; every ACK cursor an eligible boundary of the task's
    granularity (engine.py:127-134) at or after the cursor the preempting round saw.
    Returns counts; raises ``AssertionError`` on the first mismatch."""
    if predictor is None:
        predictor = policy_config.predictor
    if predictor is None:
        predictor = ps.self_calibrated_poly(
            cost_params, degree=policy_config.predictor_degree,
            chunk_size=policy_config.chunk_tokens)
    state = SchedulerState.create(policy_config, predictor)
    by_id = {r.id: r for r in trace.requests}
    tasks: dict = {}
    seen: set = set()
    gran = policy_config.granularity
    outstanding = None  # (victim task id, cursor seen by the preempting round)
    last_ack_t = None
    last_t = -1.0
    n_rounds = n_cmds = n_acks = 0
    for rec in round_log:
        assert rec["t"] >= last_t, f"time went backwards at {rec}"
        last_t = rec["t"]
        if "done" in rec:
            continue
        if "ack" in rec:
            assert outstanding is not None and outstanding[0] == rec["ack"], \
                f"ACK without an outstanding signal: {rec}"
            task = tasks[rec["ack"]]
            cur = rec["cursor"]
            if not rec.get("completed"):
                assert 0 < cur < len(task), f"ACK cursor out of range: {rec}"
                assert task.boundary_eligible(cur - 1, gran), \
                    f"ACK at a boundary {gran.value} granularity does not allow: {rec}"
            assert cur >= outstanding[1], f"ACK cursor before the signalled cursor: {rec}"
            task.cursor = cur
            outstanding = None
            last_ack_t = rec["t"]
            n_acks += 1
            continue
        assert outstanding is None, f"round {rec['round']} ran while an ACK was outstanding"
        n_rounds += 1
        assert rec["round"] == n_rounds, f"round numbering gap at {rec['round']}"
        if rec["trigger"].startswith("deferred"):
            assert rec["t"] == last_ack_t, f"deferred round not at the ACK instant: {rec}"
        for tid in rec["completions"]:
            state.note_completion(tid)
        for tid, cur in rec["cursors"].items():
            tasks[int(tid)].cursor = cur
        arrivals = [by_id[i] for i in rec["arrivals"]]
        for i in rec["arrivals"]:
            assert i not in seen, f"request {i} arrived twice"
            seen.add(i)
        cmds = schedule_round(state, rec["t"], arrivals)
        got = [command_key(c) for c in cmds]
        assert got == rec["commands"], \
            f"round {rec['round']} at t={rec['t']}: replay {got} != live {rec['commands']}"
        n_cmds += len(cmds)
        for c in cmds:
            if c.kind == "preempt":
                outstanding = (c.task_id, tasks[c.task_id].cursor)
            elif c.kind == "submit":
                tl = ps.build_timeline([r.num_tokens for r in c.members],
                                       policy_config.chunk_tokens, cost_params)
                task = ExecutionTask(c.task_id, c.members, tl)
                tasks[c.task_id] = task
                state.attach_task(task)
    assert outstanding is None, "run ended with an outstanding preempt signal"
    assert seen == set(by_id), f"requests never arrived: {sorted(set(by_id) - seen)[:10]}"
    return {"rounds": n_rounds, "commands": n_cmds, "acks": n_acks, "tasks": len(tasks)}
