"""BASELINE config 5 (HoL stress) on one B200 instance: 32K-token prompts mixed with short
high-priority requests, operator-level preemption (S-EDF) vs fixed chunked prefill (EDF +
512 / 2048-token chunks, the DistServe-CP analogue).

    python tools/hol_stress.py [--duration 30] [--rates 3,6,9] [--out gpurun_out/hol_stress.json]
    python tools/hol_stress.py --resim profiles/r1_hol_stress.json   (CPU: redo step 3 only)

Per-GPU instance of the 8 x B200 setup (requests are independent; the 8-GPU deployment is 8
replicas behind the round-robin proxy, dispatch.py). Steps:
  1. calibrate the reference cost model from live kernel profiles of single requests up to
     32K tokens (calibrate.py), for the scheduler's predictor / slack;
  2. replay `duration` seconds of the config-5 trace (seed 5) in real time with the live driver
     for each policy and rate: attainment overall and per class, p99 signal->ACK blocking;
  3. the reference goodput bisection on the calibrated model for each policy, at one instance
     and for the 8-instance deployment (dispatch.goodput_search_instances).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CLASSES = [("file", 32768.0, 0.0, 32768.0, 0.15, 6.0),
           ("text", 590.0, 652.0, 3040.0, 0.85, 0.25)]


def policies_of(ps):
    return {
        "sedf_operator": ps.PolicyConfig(),
        "edf_chunk512": ps.PolicyConfig(policy=ps.PolicyKind.EDF,
                                        granularity=ps.PreemptionGranularity.CHUNK,
                                        chunk_tokens=512),
        "edf_chunk2048": ps.PolicyConfig(policy=ps.PolicyKind.EDF,
                                         granularity=ps.PreemptionGranularity.CHUNK,
                                         chunk_tokens=2048),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--duration", type=float, default=30.0)
    ap.add_argument("--rates", default="3,6,9")
    ap.add_argument("--out", default="gpurun_out/hol_stress.json")
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--resim", default=None, help="recompute the simulated goodputs of a result")
    a = ap.parse_args()
    if a.resim:
        from paper_2602_16603_b200 import dispatch, refsim

        ps = refsim.load()
        with open(a.resim) as fh:
            res = json.load(fh)
        params = ps.CostParams.from_json_dict(res["calibration"]["cost_params"])
        res["goodput_sim_req_s"] = sim_goodput(ps, dispatch, [ps.TaskClass(*c) for c in CLASSES],
                                               policies_of(ps), params)
        with open(a.resim, "w") as fh:
            json.dump(res, fh, indent=1)
        return

    from paper_2602_16603_b200 import dispatch, refsim
    from paper_2602_16603_b200.calibrate import fit_cost_params, predicted_vs_measured
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.live import replay_rounds, run_live
    from paper_2602_16603_b200.native import PrefillContext

    ps = refsim.load()
    shape = SHAPES[a.model]
    ctx = PrefillContext(shape, kv_pages=3200, page_size=128, max_pos=40000)
    ctx.init_random(seed=0)

    # 1. calibration profile: straight single-request tasks
    cal_lens = [256, 1024, 2048, 4096, 8192, 16384, 32768]
    cal = [ctx.create_task([np.random.default_rng(n).integers(0, shape.vocab, n).astype(np.int32)])
           for n in cal_lens]
    for t in cal:  # warm-up
        t.begin_segment(0)
        t.enqueue(0, t.n_entries)
    ctx.sync()
    ctx.profile(True)
    ctx.drain_profile()
    for t in cal:
        t.begin_segment(0)
        t.enqueue(0, t.n_entries)
    ctx.sync()
    prof = ctx.drain_profile()
    ctx.profile(False)
    for t in cal:
        t.destroy()
    params = fit_cost_params(prof, shape.num_layers)
    fit_err = predicted_vs_measured(params, prof)
    t32k = sum(r["ms"] for r in prof if r["M"] == 32768) * 1e-3

    classes = [ps.TaskClass(*c) for c in CLASSES]
    policies = policies_of(ps)

    def tok(r):
        return np.random.default_rng(9000 + r.id).integers(0, shape.vocab,
                                                          r.num_tokens).astype(np.int32)

    # 2. live replays
    live = {}
    for name, pc in policies.items():
        rows = []
        for rate in [float(x) for x in a.rates.split(",")]:
            tr = ps.generate_trace(classes, rate, a.duration, 5)
            t0 = time.perf_counter()
            rounds: list = []
            res = run_live(tr, pc, params, ctx, tok, max_wall_s=10 * a.duration + 120,
                           round_log=rounds)
            bl = ps.blocking_stats(res.blocking_log)
            try:  # wall-clock scheduling parity: every round through a fresh reference scheduler
                rep = replay_rounds(tr, pc, params, rounds)
                replay = {"rounds": rep["rounds"], "mismatches": 0}
            except AssertionError as e:
                replay = {"mismatch": str(e)[:200]}
            max_entry = {r["done"]: r["max_entry_s"] for r in rounds if "done" in r}
            rows.append({
                "rate_req_s": rate,
                "requests": len(tr),
                "attainment": ps.slo_attainment(res.outcomes),
                "attainment_by_class": {c: ps.slo_attainment(res.outcomes, c)
                                        for c in sorted({o.task for o in res.outcomes})},
                "commands": res.commands,
                "p99_blocking_ms": None if bl["p99_s"] is None else round(bl["p99_s"] * 1e3, 3),
                "max_blocking_ms": None if bl["max_s"] is None else round(bl["max_s"] * 1e3, 3),
                "wall_s": round(time.perf_counter() - t0, 2),
                "replay": replay,
                "longest_entry_ms": round(max(max_entry.values()) * 1e3, 3) if max_entry else None,
            })
            print(name, rows[-1], flush=True)
        live[name] = rows

    # 3. reference goodput bisection on the calibrated model (1 instance and 8 instances)
    sim = sim_goodput(ps, dispatch, classes, policies, params)
    result = {
        "config": "BASELINE configs[4]: HoL stress, file(32768, 0, 32768, 0.15, 6.0) + "
                  "text(590, 652, 3040, 0.85, 0.25), seed 5, per-GPU instance",
        "model": a.model,
        "calibration": {"lengths": cal_lens, "fit_max_rel_err": round(fit_err, 4),
                        "prefill_32k_s": round(t32k, 4),
                        "cost_params": params.to_json_dict()},
        "live": live,
        "goodput_sim_req_s": sim,
        "duration_s": a.duration,
    }
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(result, fh, indent=1)
    ctx.close()


def sim_goodput(ps, dispatch, classes, policies, params):
    """Reference goodput bisection on the calibrated model: one instance (base trace 300 s at
    1 req/s) and the 8-instance round-robin deployment (base trace 300 s at 8 req/s, so every
    instance sees the same request count as the single-instance search)."""
    sim = {}
    for name, pc in policies.items():
        rc = ps.RunConfig(pc, params)
        out = {}
        for n in (1, 8):
            base = ps.generate_trace(classes, 1.0 * n, 300.0, 5)
            try:
                r = dispatch.goodput_search_instances(base, rc, n, target=0.9,
                                                      rate_bounds=(0.05, 64.0 * n), tol=0.05,
                                                      jobs=min(n, os.cpu_count() or 1))
                out[f"instances_{n}"] = {"value": r.value, "saturated": r.saturated}
            except Exception as e:  # infeasible floor etc.
                out[f"instances_{n}"] = {"error": repr(e)[:160]}
        sim[name] = out
        print(name, out, flush=True)
    return sim


if __name__ == "__main__":
    main()
