"""B200 calibration of the reference cost model from live kernel profiles.

The reference scheduler's slack (Eq. 3) and SLO-aware batching (Alg. 1) are only as good as the
TTFT predictor, which the reference fits to its own cost model (``self_calibrated_poly``,
prefillsim/cost_model.py:322-343). Here the cost model's coefficients are refitted from B200
kernel timings -- ``c_fix + c_lin * new`` per operator, plus ``c_attn * quad_mass`` for attention
(cost_model.py:151-166) -- so the unchanged reference ``run()`` / ``goodput_search`` can predict
and simulate on B200 time.
"""

from __future__ import annotations

from collections import defaultdict
from typing import Sequence

import numpy as np

from . import refsim

_ENTRY_OF_KERNEL = {
    "qkv_gemm": "qkv_proj",
    "attn": "attn",
    "o_gemm": "o_proj",
    "gate_up_gemm": "gate_up_proj",
    "down_gemm": "down_proj",
}


def entry_samples(records: Sequence[dict]) -> dict:
    """Group a profile of straight (unpreempted, unchunked, single-request) task runs into
    per-entry durations: op -> list of (new_tokens, seconds). An rmsnorm record is charged to
    the GEMM entry that follows it; the final norm + lm_head are charged per chunk."""
    out = defaultdict(list)
    chunk_extra = []
    pending = 0.0
    for r in records:
        k = r["kind"]
        if k == "rmsnorm":
            pending += r["ms"]
            continue
        if k in ("final_rmsnorm", "lm_head_gemm"):
            chunk_extra.append(r["ms"] * 1e-3)
            continue
        op = _ENTRY_OF_KERNEL[k]
        out[op].append((r["M"], (r["ms"] + pending) * 1e-3))
        pending = 0.0
    out["_chunk_extra"] = chunk_extra
    return out


def _medians(pts):
    """One point per entry size: the median duration over its launches (a profile holds every
    layer of every request, so one clock dip or preempted neighbour does not steer the fit)."""
    by = defaultdict(list)
    for m, y in pts:
        by[m].append(y)
    return [(m, float(np.median(v))) for m, v in sorted(by.items())]


def fit_cost_params(records: Sequence[dict], num_layers: int, c_check: float = 1e-6):
    """CostParams from profile records (single-request tasks: quad = M^2), least squares on the
    RELATIVE error: the profile spans 40-token to 5K-token entries, and an absolute fit would
    let the long entries set every coefficient (max relative error 39% on the short ones),
    while the scheduler's slack and batching decisions need short requests predicted too."""
    ps = refsim.load()
    OK = ps.OperatorKind
    samples = entry_samples(records)
    c_lin, c_fix = {}, {}
    c_attn = 0.0
    for op in ("qkv_proj", "attn", "o_proj", "gate_up_proj", "down_proj"):
        pts = _medians(samples.get(op, []))
        if not pts:
            raise ValueError(f"no samples for {op}")
        m = np.array([p[0] for p in pts], dtype=np.float64)
        y = np.array([p[1] for p in pts], dtype=np.float64)
        if op == "attn":
            X = np.stack([np.ones_like(m), m, m * m], axis=1)
        else:
            X = np.stack([np.ones_like(m), m], axis=1)
        wgt = 1.0 / np.maximum(y, 1e-9)
        coef, *_ = np.linalg.lstsq(X * wgt[:, None], y * wgt, rcond=None)
        coef = np.maximum(coef, 0.0)  # the reference rejects negative coefficients
        c_fix[OK(op)] = float(coef[0])
        c_lin[OK(op)] = float(coef[1])
        if op == "attn":
            c_attn = float(coef[2])
    extra = samples["_chunk_extra"]
    c_chunk = float(np.mean(extra)) if extra else 0.0
    return ps.CostParams(num_layers=num_layers, c_lin=c_lin, c_fix=c_fix, c_attn=c_attn,
                         c_chunk=c_chunk, c_check=c_check)


def predicted_vs_measured(params, records: Sequence[dict]) -> float:
    """Max relative error of the fitted per-entry model over the profiled entry sizes (median
    duration per size)."""
    ps = refsim.load()
    worst = 0.0
    for op, pts in entry_samples(records).items():
        if op.startswith("_"):
            continue
        for m, y in _medians(pts):
            pred = ps.operator_duration(ps.OperatorKind(op), int(m), 0, params)
            worst = max(worst, abs(pred - y) / max(y, 1e-9))
    return worst


def measure_ttft_samples(ctx, shape, lengths: Sequence[int], reps: int = 2) -> list:
    """Measured single-request prefill latency (tokens, seconds) on the device: one task per
    length, CUDA events around its whole entry list on the prefill stream, median of `reps`
    runs after a warm-up run. The profile the reference's `prefillsim calibrate` consumes
    (cli.py:251-267: a tokens,seconds CSV)."""
    import torch

    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    rng = np.random.default_rng(0)
    out = []
    for n in lengths:
        task = ctx.create_task([rng.integers(0, shape.vocab, int(n)).astype(np.int32)])
        times = []
        for r in range(reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            task.begin_segment(0)
            e0.record(stream)
            task.enqueue(0, task.n_entries)
            e1.record(stream)
            ctx.sync()
            if r:
                times.append(e0.elapsed_time(e1) * 1e-3)
        task.destroy()
        out.append((float(n), float(np.median(times))))
    return out


def fit_ttft_predictor(samples: Sequence, degree: int = 2):
    """The reference's own predictor fit on measured latencies (`fit_ttft_poly`,
    cost_model.py:271-301, as `prefillsim calibrate` runs it) and its `fit_quality`."""
    refsim.load()
    from prefillsim import cost_model as cm

    poly = cm.fit_ttft_poly(list(samples), degree)
    return poly, cm.fit_quality(list(samples), poly)


def ttft_grid(lo: int = 64, hi: int = 32768, points: int = 17) -> list:
    """The reference's log-spaced calibration grid (self_calibrated_poly, cost_model.py:322-343),
    capped at the context's position table."""
    return [int(n) for n in np.unique(np.round(np.geomspace(lo, hi, points)).astype(int))]
