"""Multi-instance dispatch: independent per-GPU prefill instances behind a round-robin proxy.

The paper's proxy is "simple round-robin" across prefill instances; the reference
simulates a single instance only. Requests are independent -- no cross-request
attention (cost_model.py:225-233) and private per-task state -- so the path shards by request
with NO collective on the data path: every rank runs its own event-driven scheduler and
execution pool on its sub-trace, and only the outcomes are gathered for the metrics.
"""

from __future__ import annotations

from typing import Sequence

from . import refsim


def round_robin(trace, n_instances: int) -> list:
    """Request i (in arrival order) -> instance i mod n. Ids, arrivals and SLOs unchanged."""
    ps = refsim.load()
    if n_instances < 1:
        raise ValueError("n_instances must be >= 1")
    parts = [[] for _ in range(n_instances)]
    for i, r in enumerate(trace.requests):
        parts[i % n_instances].append(r)
    return [ps.Trace(tuple(p), origin=f"{trace.origin} rr{k}/{n_instances}")
            for k, p in enumerate(parts)]


def merge_outcomes(per_instance: Sequence[Sequence]) -> list:
    """Outcomes of all instances, in request-id order (no loss, no duplicates)."""
    out = [o for part in per_instance for o in part]
    ids = [o.id for o in out]
    if len(ids) != len(set(ids)):
        raise ValueError("duplicate request outcomes across instances")
    return sorted(out, key=lambda o: o.id)


def gather_outcomes(local_outcomes: Sequence, group=None) -> list:
    """All-gather the per-rank outcomes over torch.distributed (gloo or nccl plumbing)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    bucket = [None] * world
    dist.all_gather_object(bucket, list(local_outcomes), group=group)
    return merge_outcomes(bucket)


def attainment(outcomes: Sequence) -> float:
    ps = refsim.load()
    return ps.slo_attainment(outcomes)


# ---------------------------------------------------------------------------------------------
# Multi-instance results in the reference artifact formats
#
# A deployment of n independent prefill instances behind the round-robin proxy produces one
# reference ``RunResult`` per instance (reference ``run()`` with the GPU engine injected, or the
# wall-clock driver ``live.run_live``). ``merge_results`` folds them into ONE RunResult of the
# whole deployment, so the reference's own metrics and writers -- ``slo_attainment``,
# ``blocking_stats``, ``summary_dict``, ``write_run_csv``, ``sweep_row``/``write_sweep_csv``
# (prefillsim/metrics.py:195-267) and its goodput bisection (metrics.py:87-140) -- consume
# B200 multi-instance runs unchanged. At n = 1 every artifact is byte-identical to the
# reference CLI's (cli.py:152-166).


def merge_results(results: Sequence):
    """One RunResult for n instances: outcomes in id order, blocking intervals, rounds and
    command counts summed, task stats / batch audits concatenated in instance order."""
    ps = refsim.load()
    from prefillsim.engine import RunResult

    if not results:
        raise ValueError("no instance results")
    if len(results) == 1:
        return results[0]
    first = results[0]
    for r in results[1:]:
        if (r.policy, r.granularity, r.seed) != (first.policy, first.granularity, first.seed):
            raise ValueError("instances ran different policies / granularities / seeds")
    commands: dict = {}
    for r in results:
        for k, v in r.commands.items():
            commands[k] = commands.get(k, 0) + v
    blocking = sorted((e for r in results for e in r.blocking_log), key=lambda e: (e[0], e[1], e[2]))
    del ps
    return RunResult(
        outcomes=merge_outcomes([r.outcomes for r in results]),
        blocking_log=blocking,
        rounds=sum(r.rounds for r in results),
        commands=commands,
        tasks=[t for r in results for t in r.tasks],
        batch_audit=[b for r in results for b in r.batch_audit],
        seed=first.seed,
        policy=first.policy,
        granularity=first.granularity,
        events=None,
    )


def gather_results(local_result, group=None) -> list:
    """All-gather every rank's RunResult (rank order) over torch.distributed."""
    import torch.distributed as dist

    bucket = [None] * dist.get_world_size(group)
    dist.all_gather_object(bucket, local_result, group=group)
    return bucket


def _reference_run(args):
    tr, pol, par, sd, ev = args
    return refsim.load().run(tr, pol, par, sd, record_events=ev)


def run_instances(trace, n_instances: int, policy, params, seed: int = 0, runner=None,
                  record_events: bool = False, jobs: int = 1) -> list:
    """Round-robin ``trace`` over n instances and run each (``runner(trace, policy, params,
    seed, record_events)``; default: the reference ``run`` with whatever engine is injected).
    ``jobs`` > 1 simulates the instances of the default runner in a process pool (virtual
    clock only; results are identical to the serial run)."""
    parts = round_robin(trace, n_instances)
    if runner is None and jobs > 1 and n_instances > 1:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor

        # spawn: the caller may hold a CUDA context and launch threads (no fork)
        with ProcessPoolExecutor(max_workers=min(jobs, n_instances),
                                 mp_context=mp.get_context("spawn")) as pool:
            return list(pool.map(_reference_run,
                                 [(p, policy, params, seed, record_events) for p in parts]))
    if runner is None:
        return [_reference_run((p, policy, params, seed, record_events)) for p in parts]
    return [runner(part, policy, params, seed, record_events) for part in parts]


def write_run_artifacts(results: Sequence, out_dir: str, config_hash: str | None = None) -> dict:
    """Reference ``cmd_run`` artifacts for a (multi-)instance run: merged ``run.csv`` +
    ``summary.json`` (plus ``instances`` when n > 1) and, for n > 1, the same files and the
    event log (when recorded) of every instance under ``instance<k>/``. Returns the summary."""
    import json
    import os

    ps = refsim.load()
    from prefillsim.files import atomic_write_text
    from prefillsim.metrics import summary_dict, write_run_csv

    def write(result, d, extra):
        os.makedirs(d, exist_ok=True)
        write_run_csv(result, os.path.join(d, "run.csv"))
        summary = summary_dict(result)
        if config_hash is not None:
            summary["config_hash"] = config_hash
        summary.update(extra)
        atomic_write_text(os.path.join(d, "summary.json"),
                          json.dumps(summary, sort_keys=True, indent=2) + "\n")
        if result.events is not None:
            result.write_event_log(os.path.join(d, "events.jsonl"))
        return summary

    del ps
    merged = merge_results(results)
    if len(results) > 1:
        for k, r in enumerate(results):
            write(r, os.path.join(out_dir, f"instance{k}"), {"instance": k})
        return write(merged, out_dir, {"instances": len(results)})
    return write(merged, out_dir, {})


def sweep_instances(trace, n_instances: int, policy, params, rates: Sequence[float],
                    seed: int = 0, runner=None, out_dir: str | None = None) -> list:
    """Reference rate sweep (cli.py:177-245 ``values`` mode) of the whole deployment: per rate,
    rescale the base trace, dispatch it round-robin and merge; rows in ``sweep.csv`` format."""
    import os

    ps = refsim.load()
    from prefillsim.metrics import sweep_row, write_sweep_csv

    rows = []
    base = trace.base_rate()
    for rate in rates:
        tr = ps.scale_rate(trace, float(rate) / base)
        merged = merge_results(run_instances(tr, n_instances, policy, params, seed, runner))
        rows.append(sweep_row("rate", float(rate), merged))
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        write_sweep_csv(rows, os.path.join(out_dir, "sweep.csv"))
    return rows


def goodput_search_instances(trace, run_config, n_instances: int, target: float = 0.9,
                             rate_bounds=(0.25, 16.0), tol: float = 0.05, runner=None,
                             jobs: int = 1):
    """The reference's own goodput bisection (metrics.py:87-140) over the whole n-instance
    deployment: its per-probe ``run`` (resolved as a module global at call time) is swapped
    for round-robin dispatch + merge while the search runs."""
    ps = refsim.load()
    import prefillsim.metrics as M

    orig = M.run

    def deployment_run(tr, policy, params, seed=0, record_events=False):
        return merge_results(run_instances(tr, n_instances, policy, params, seed, runner,
                                           record_events, jobs))

    M.run = deployment_run
    try:
        return ps.goodput_search(trace, run_config, target=target, rate_bounds=rate_bounds,
                                 tol=tol)
    finally:
        M.run = orig
