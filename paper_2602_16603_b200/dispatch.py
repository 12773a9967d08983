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
