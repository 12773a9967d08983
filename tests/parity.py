"""Shared bf16-vs-fp32 parity check (BASELINE north_star: "Logits and KV must match within a
stated bf16 tolerance (max-abs and relative error reported against the reference's fp32
path)").

Every comparison reports three numbers and asserts the stated tolerance on two of them:

* ``max_abs``      = max |got - ref|                          (reported)
* ``max_abs_frac`` = max |got - ref| / max |ref|              (asserted <= ``atol_frac``)
* ``rel_l2``       = ||got - ref||_2 / ||ref||_2              (asserted <= ``rel_tol``)

The stated tolerances (bf16 activations / KV, fp32 accumulation, against the fp32 oracle):
logits max-abs <= 3% of max|logit| and relative L2 <= 2%; KV max-abs <= 2% of max|kv| and
relative L2 <= 1%. Every check is appended to ``RECORDS``; with ``PARITY_REPORT=<path>`` the
session writes them as JSON (conftest.py), e.g. ``profiles/r2_parity.json``.
"""

from __future__ import annotations

import numpy as np

LOGIT_ATOL_FRAC = 0.03
LOGIT_REL_TOL = 0.02
KV_ATOL_FRAC = 0.02
KV_REL_TOL = 0.01

RECORDS: list = []


def errors(got, ref) -> dict:
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    d = got - ref
    max_abs = float(np.abs(d).max()) if d.size else 0.0
    ref_max = float(np.abs(ref).max()) if ref.size else 0.0
    ref_l2 = float(np.linalg.norm(ref))
    return {
        "max_abs": max_abs,
        "max_abs_frac": max_abs / max(ref_max, 1e-6),
        "rel_l2": float(np.linalg.norm(d)) / max(ref_l2, 1e-12),
        "ref_max_abs": ref_max,
        "n": int(d.size),
    }


def check(name: str, got, ref, atol_frac: float, rel_tol: float) -> dict:
    e = errors(got, ref)
    e.update(name=name, atol_frac=atol_frac, rel_tol=rel_tol,
             ok=e["max_abs_frac"] <= atol_frac and e["rel_l2"] <= rel_tol)
    RECORDS.append(e)
    print(f"{name}: max-abs {e['max_abs']:.4g} ({e['max_abs_frac']:.4g} of max|ref|), "
          f"rel-L2 {e['rel_l2']:.4g}")
    assert e["max_abs_frac"] <= atol_frac, f"{name}: max-abs {e['max_abs_frac']:.4g} > {atol_frac}"
    assert e["rel_l2"] <= rel_tol, f"{name}: relative L2 {e['rel_l2']:.4g} > {rel_tol}"
    return e


def logits(name: str, got, ref, atol_frac: float = LOGIT_ATOL_FRAC,
           rel_tol: float = LOGIT_REL_TOL) -> dict:
    return check(name + " logits", got, ref, atol_frac, rel_tol)


def kv(name: str, got, ref, atol_frac: float = KV_ATOL_FRAC, rel_tol: float = KV_REL_TOL) -> dict:
    return check(name, got, ref, atol_frac, rel_tol)
