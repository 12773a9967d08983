"""Wall-clock driver logic on CPU (fake asynchronous device): no lost requests, one round per
arrival plus one per task completion (test_properties.py:80-84), every preemption is ACKed and
resumed from the device cursor, blocking is bounded by one entry + polling slack."""

from conftest import refsim_or_skip  # noqa: E402
import os

import numpy as np
import pytest

from fake_native import FakeLiveContext


@pytest.mark.parametrize("gran", ["operator", "layer"])
def test_live_driver_invariants(gran):
    from paper_2602_16603_b200 import refsim
    from paper_2602_16603_b200.live import replay_rounds, run_live

    ps = refsim_or_skip()
    # a long request followed by urgent short ones, replayed in ~0.1 s of wall time
    reqs = [ps.Request(0, "file", 0.0, 4000, 10.0)]
    for i in range(1, 9):
        reqs.append(ps.Request(i, "text", 0.005 * i, 50 + 7 * i, 0.05))
    trace = ps.Trace(tuple(reqs))
    params = ps.CostParams(num_layers=2)
    ctx = FakeLiveContext(num_layers=2, entry_s=2e-3)
    pc = ps.PolicyConfig(granularity=ps.PreemptionGranularity(gran))
    rounds = []
    res = run_live(trace, pc, params, ctx, tokens=lambda r: np.zeros(r.num_tokens, np.int32),
                   record_events=True, max_wall_s=30, round_log=rounds)
    rep = replay_rounds(trace, pc, params, rounds)
    assert rep["rounds"] == res.rounds and rep["acks"] == res.commands["preempt"]
    done = {r["done"]: r["max_entry_s"] for r in rounds if "done" in r}
    assert sorted(done) == sorted(t.task_id for t in res.tasks)
    assert sorted(o.id for o in res.outcomes) == list(range(9))
    assert res.rounds == len(trace) + len(res.tasks)
    assert res.commands["preempt"] >= 1
    raced = sum(1 for r in rounds if r.get("completed"))  # completion won the ACK race
    assert res.commands["resume"] == res.commands["preempt"] - raced
    assert len(res.blocking_log) == res.commands["preempt"]
    for sig, ack, _ in res.blocking_log:
        bound = 2e-3 * (5 if gran == "layer" else 1)
        assert 0 <= ack - sig <= bound + 0.02
    # every resume restarts exactly where the device stopped
    raced_tasks = {r["ack"] for r in rounds if r.get("completed")}
    acks = [e for e in res.events if e["kind"] == "preempt_ack" and e["task"] not in raced_tasks]
    resumes = [e for e in res.events if e["kind"] == "resume"]
    assert sorted(a["detail"]["cursor"] for a in acks) == sorted(r["detail"]["cursor"] for r in resumes)
    for t in ctx.tasks:
        assert t.destroyed
    assert 0.0 <= ps.slo_attainment(res.outcomes) <= 1.0


def test_replay_rejects_a_tampered_log():
    """The replay is a real check: a live log whose commands, cursors or deferral disagree
    with the reference scheduler is rejected."""
    import copy

    from paper_2602_16603_b200.live import replay_rounds, run_live

    ps = refsim_or_skip()
    reqs = [ps.Request(0, "file", 0.0, 4000, 10.0)]
    for i in range(1, 6):
        reqs.append(ps.Request(i, "text", 0.005 * i, 50 + 7 * i, 0.05))
    trace = ps.Trace(tuple(reqs))
    params = ps.CostParams(num_layers=2)
    pc = ps.PolicyConfig()
    rounds = []
    run_live(trace, pc, params, FakeLiveContext(num_layers=2, entry_s=2e-3),
             tokens=lambda r: np.zeros(r.num_tokens, np.int32), max_wall_s=30, round_log=rounds)
    replay_rounds(trace, pc, params, rounds)
    pre = next(i for i, r in enumerate(rounds) if r.get("commands", [[None]])[:1]
               and r["commands"][0][0] == "preempt")
    bad = copy.deepcopy(rounds)
    bad[pre]["commands"] = bad[pre]["commands"][1:]  # drop the preempt
    with pytest.raises(AssertionError):
        replay_rounds(trace, pc, params, bad)
    bad = copy.deepcopy(rounds)
    ack = next(i for i in range(pre, len(bad)) if "ack" in bad[i])
    bad[ack]["t"] += 1e-3  # a deferred round no longer at the ACK instant
    if ack + 1 < len(bad) and bad[ack + 1].get("trigger", "").startswith("deferred"):
        with pytest.raises(AssertionError):
            replay_rounds(trace, pc, params, bad)
    bad = copy.deepcopy(rounds)
    bad.insert(ack, dict(bad[pre], round=bad[pre]["round"] + 1))  # a round during the signal
    with pytest.raises(AssertionError):
        replay_rounds(trace, pc, params, bad)
