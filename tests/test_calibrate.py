"""B200 calibration of the reference cost model: the fit recovers known
CostParams from profile records in the live-profile format, charges pre-GEMM norms to the
following entry and the final norm + lm_head to the chunk, and its predictions go through the
reference's own operator_duration (cost_model.py:151-166)."""

from conftest import refsim_or_skip  # noqa: E402
import numpy as np

from paper_2602_16603_b200 import refsim
from paper_2602_16603_b200.calibrate import entry_samples, fit_cost_params, predicted_vs_measured

OPS = [("qkv_gemm", "qkv_proj"), ("attn", "attn"), ("o_gemm", "o_proj"),
       ("gate_up_gemm", "gate_up_proj"), ("down_gemm", "down_proj")]
FIX = {"qkv_proj": 20e-6, "attn": 12e-6, "o_proj": 15e-6, "gate_up_proj": 40e-6, "down_proj": 30e-6}
LIN = {"qkv_proj": 3e-8, "attn": 1e-8, "o_proj": 2e-8, "gate_up_proj": 1.5e-7, "down_proj": 7e-8}
C_ATTN = 6e-12


def records(lens, norm_ms=0.004, extra_ms=0.25, noise=0.0, seed=0):
    rng = np.random.default_rng(seed)
    out = []
    for m in lens:
        out.append({"kind": "rmsnorm", "M": m, "ms": norm_ms})
        for kind, op in OPS:
            s = FIX[op] + LIN[op] * m + (C_ATTN * m * m if op == "attn" else 0.0)
            if kind in ("qkv_gemm", "gate_up_gemm") and out[-1]["kind"] == "rmsnorm":
                s -= norm_ms * 1e-3  # the fused-norm record is charged to this entry
            out.append({"kind": kind, "M": m, "ms": s * 1e3 * (1 + noise * rng.standard_normal())})
        out.append({"kind": "final_rmsnorm", "M": 1, "ms": 0.01})
        out.append({"kind": "lm_head_gemm", "M": 1, "ms": extra_ms - 0.01})
    return out


def test_fit_recovers_known_cost_params():
    ps = refsim_or_skip()
    lens = [1, 42, 163, 545, 1572, 4465]
    recs = records(lens)
    samples = entry_samples(recs)
    assert len(samples["qkv_proj"]) == len(lens) and len(samples["_chunk_extra"]) == 2 * len(lens)
    p = fit_cost_params(recs, num_layers=32)
    for op in FIX:
        k = ps.OperatorKind(op)
        assert abs(p.c_fix[k] - FIX[op]) <= 1e-3 * FIX[op], op
        assert abs(p.c_lin[k] - LIN[op]) <= 1e-3 * LIN[op], op
    assert abs(p.c_attn - C_ATTN) <= 1e-3 * C_ATTN
    assert predicted_vs_measured(p, recs) <= 1e-6


def test_fit_is_relative_error_weighted():
    """With noisy long entries, the short entries are still predicted within a few percent
    (an absolute least-squares fit would trade them for the long ones)."""
    ps = refsim_or_skip()
    lens = [40, 80, 160, 320, 640, 1280, 2560, 5120]
    recs = records(lens, noise=0.02, seed=3)
    p = fit_cost_params(recs, num_layers=32)
    assert p.num_layers == 32
    d = ps.operator_duration(ps.OperatorKind("o_proj"), 40, 0, p)
    ref = FIX["o_proj"] + LIN["o_proj"] * 40
    assert abs(d - ref) / ref <= 0.05
    assert predicted_vs_measured(p, recs) <= 0.08


def test_fit_ignores_single_outlier_launches():
    """One slow launch of a short entry (a clock dip) does not move the fit: entries are fitted
    on the median duration per size."""
    lens = [42, 163, 545, 1572, 4465]
    recs = []
    for layer in range(8):
        recs += records(lens)
    for r in recs:
        if r["kind"] == "attn" and r["M"] == 42:
            r["ms"] *= 3.0
            break
    p = fit_cost_params(recs, num_layers=32)
    assert predicted_vs_measured(p, recs) <= 1e-3


def test_ttft_predictor_is_the_reference_fit():
    """The live predictor is the reference's own fit_ttft_poly over (tokens, seconds) samples on
    the reference's log-spaced grid (`prefillsim calibrate`, cli.py:251-267); the wall-clock
    driver takes it through PolicyConfig.predictor like the reference run()."""
    from paper_2602_16603_b200.calibrate import fit_ttft_predictor, ttft_grid

    ps = refsim_or_skip()
    from prefillsim import cost_model as cm

    grid = ttft_grid()
    assert grid[0] == 64 and grid[-1] == 32768 and len(grid) == 17
    samples = [(float(n), 2e-3 + 9e-7 * n + 3e-12 * n * n) for n in grid]
    poly, q = fit_ttft_predictor(samples, 2)
    ref = cm.fit_ttft_poly(samples, 2)
    assert poly.coefficients == ref.coefficients
    assert q["r2"] > 0.999999
    assert isinstance(ps.PolicyConfig(predictor=poly).predictor, type(ref))
