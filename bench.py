#!/usr/bin/env python
"""Benchmark of the B200-native preemptible prefill forward pass (FlowPrefill hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): Llama-3-8B shape, bf16, random-init weights, on one
B200 per rank. One *step* = prefill of STEP_REQUESTS requests drawn from the config-2 trace
(3 TTFT-SLO classes: text 0.76 @0.25 s, search 0.20 @4.0 s, file 0.04 @6.0 s; the reference's
``generate_trace``, seed 7), each request its own task, every entry's boundary check armed
(operator granularity). Under torchrun each rank runs an independent instance on its own
requests (request i -> rank i mod N, the paper's round-robin proxy): weak scaling, no
collective on the data path; the timed region is bracketed by barriers and the max over
ranks is taken.

Reported (one JSON line from rank 0):
  value        prefill tokens/s, whole job, inputs resident in HBM, CUDA events on the
               prefill stream.
  e2e          the same metric through the public API (PrefillContext.create_task from host
               token ids -> all entries -> logits read back to the host), wall clock.
  roofline     dense GEMMs (dominant kernel class), event-timed inside the timed steps.
  p99_preempt  host-observed signal -> device ACK latency on a long request, async launch
               worker, vs the longest operator of that request.
  goodput      req/s at 90% TTFT-SLO attainment from the reference goodput_search with the
               cost model re-fitted to this run's B200 kernel timings (virtual clock), and a
               live wall-clock replay of the config-2 arrivals on the GPU (live_check).
  cpu_baseline the fp32 numpy restatement (oracle/) on this host's cores, bounded sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STEP_REQUESTS = 16
MODEL = "llama3-8b"
CONFIG2_CLASSES = [  # image merged into text
    ("text", 590.0, 652.0, 3040.0, 0.76, 0.25),
    ("search", 5976.0, 3456.0, 16635.0, 0.20, 4.0),
    ("file", 6833.0, 5186.0, 22390.0, 0.04, 6.0),
]


# ------------------------------------------------------------------------------ helpers
def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def config2_trace(rate: float, duration: float, seed: int = 7):
    from paper_2602_16603_b200 import refsim

    ps = refsim.load()
    classes = [ps.TaskClass(*c) for c in CONFIG2_CLASSES]
    return ps.generate_trace(classes, rate, duration, seed)


STEP_TRACE = os.path.join(ROOT, "tests", "golden", "config2_step_trace.jsonl")


class StepRequest:
    __slots__ = ("id", "task", "arrival_s", "num_tokens", "ttft_slo_s")

    def __init__(self, d):
        for k in self.__slots__:
            setattr(self, k, d[k])


def step_requests(world: int, rank: int):
    """The step's requests: the head of the config-2 trace (reference generate_trace, rate 8,
    300 s, seed 7), read from the committed fixture made by tests/golden/make_golden.py so the
    timed legs never need the reference scheduler. Request i -> rank i mod world."""
    with open(STEP_TRACE) as fh:
        reqs = [StepRequest(json.loads(ln)) for ln in fh if ln.strip()]
    if len(reqs) < STEP_REQUESTS * world:
        raise ValueError(f"{STEP_TRACE} holds {len(reqs)} requests, need {STEP_REQUESTS * world}")
    return [r for i, r in enumerate(reqs[: STEP_REQUESTS * world]) if i % world == rank]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sms = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4)
                          if r[3 + j].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sms)) if sms else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------------------ CPU legs
def cpu_sample(shape_name: str = MODEL, n_tokens: int = 512, reps: int = 1):
    """fp32 numpy restatement (oracle/) of ONE layer on n_tokens, scaled to all layers."""
    from oracle import forward as F

    full = F.SHAPES[shape_name]
    one = F.Shape(1, full.hidden, full.n_heads, full.n_kv_heads, full.head_dim, full.ffn, 256,
                  full.rope_theta, full.rms_eps)
    w = F.make_weights(one, 0)
    toks = F.make_tokens([n_tokens], one.vocab, 0)
    times = []
    for _ in range(reps):
        t = F.OracleTask(one, w, toks)
        t0 = time.perf_counter()
        t.run_all()
        times.append(time.perf_counter() - t0)
    per_layer = min(times)
    tok_s = n_tokens / (per_layer * full.num_layers)
    cores = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_info

        cores = max(i.get("num_threads", 1) for i in threadpool_info()) or cores
    except Exception:
        pass
    return tok_s, cores, f"1 layer x {n_tokens} tokens of {shape_name} (fp32 numpy), x{full.num_layers} layers"


def control_plane_time(duration: float = 60.0, rate: float = 20.0):
    """SURVEY 8(d) CPU timing (1): wall time of the reference's own run() (scheduler + event
    engine, virtual clock, default cost model) on the config-2 trace, one host core."""
    from paper_2602_16603_b200 import refsim

    ps = refsim.load()
    tr = config2_trace(rate=rate, duration=duration)
    t0 = time.perf_counter()
    res = ps.run(tr, ps.PolicyConfig(), ps.CostParams(), 0)
    wall = time.perf_counter() - t0
    return {"requests": len(tr), "rounds": res.rounds, "wall_s": round(wall, 3),
            "us_per_round": round(wall / max(res.rounds, 1) * 1e6, 1),
            "what": f"reference prefillsim.run() on {duration:.0f} s of the config-2 trace at "
                    f"{rate:g} req/s (S-EDF, operator), 1 core"}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample(reps=1)
    vals = []
    t0 = time.perf_counter()
    cores, sample = 1, ""
    for _ in range(args.steps):
        v, cores, sample = cpu_sample(reps=1)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = float(np.mean(vals))
    line = {
        "impl": "reference",
        "metric": "prefill_tokens_per_s",
        "value": value,
        "unit": "tok/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": wall * 1e3 / max(args.steps, 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{MODEL} prefill, fp32 CPU restatement of the reference operator "
                               "timeline (oracle/forward.py); the reference itself computes no "
                               "tensors", "sample": sample},
        "cpu_baseline": {"value": value, "unit": "tok/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch

    from paper_2602_16603_b200 import _lib
    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext

    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local
    shape = SHAPES[MODEL]
    reqs = step_requests(ws, rank)
    lens = [r.num_tokens for r in reqs]
    tokens = [np.random.default_rng(1000 + r.id).integers(0, shape.vocab, r.num_tokens)
              .astype(np.int32) for r in reqs]
    step_tokens = int(sum(lens))
    pages = sum((n + 127) // 128 for n in lens)
    long_len = 8192
    live_pages = 0 if args.skip_live else 3000  # preempted tasks keep their KV pages
    ctx = PrefillContext(shape, device=device, kv_pages=3 * pages + long_len // 128 + 64 + live_pages,
                         page_size=128, max_pos=40000)
    ctx.init_random(seed=0)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=device)
    tasks = [ctx.create_task([t], None, "operator", i) for i, t in enumerate(tokens)]

    def run_step():
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        v = torch.tensor([x], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    def sum_over_ranks(x: int) -> int:
        if dist is None:
            return x
        v = torch.tensor([x], dtype=torch.int64, device=f"cuda:{device}")
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        return int(v.item())

    for _ in range(max(args.warmup, 1)):
        run_step()
    ctx.sync()
    log(f"[rank {rank}] step: {len(tasks)} requests, {step_tokens} tokens; lens={lens}")

    # -------- timed region: device events on the prefill stream
    clocks = ClockSampler(device)
    clocks.start()
    launches0 = ctx.launch_count()
    barrier()
    torch.cuda.synchronize(device)
    ctx.sync()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        run_step()
    e1.record(stream)
    ctx.sync()
    torch.cuda.synchronize(device)
    barrier()
    launches = ctx.launch_count() - launches0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms)
    job_step_tokens = sum_over_ranks(step_tokens)  # ranks hold different requests
    total_tokens = job_step_tokens * args.steps
    value = total_tokens / (ms_max / 1e3)

    # -------- per-kernel CUDA events (same steps again, events around every kernel; the
    # events serialise launches, so the unprofiled timed region above is the headline)
    prof_steps = max(1, min(args.steps, 2))
    ctx.profile(True)
    ctx.drain_profile()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(prof_steps):
        run_step()
    p1.record(stream)
    prof = ctx.drain_profile()
    ctx.profile(False)
    ms_prof = p0.elapsed_time(p1) / prof_steps

    # -------- roofline: the dominant kernel (gate_up GEMM + SwiGLU), from the profiled steps
    peaks, peak_kind = measured_peaks()
    peak = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]

    def rate(kinds):
        rs = [r for r in prof if r["kind"] in kinds]
        fl = sum(r["flops"] for r in rs)
        t = sum(r["ms"] for r in rs)
        return (fl / (t * 1e-3) / 1e12 if t > 0 else 0.0), len(rs), fl
    achieved, n_launch, gu_flops = rate({"gate_up_gemm"})
    all_gemm, _, _ = rate({"qkv_gemm", "o_gemm", "gate_up_gemm", "down_gemm"})
    step_ms_sum = sum(r["ms"] for r in prof)
    kernels = {}
    for r in prof:
        k = kernels.setdefault(r["kind"], {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
        k["launches"] += 1
        k["ms"] += r["ms"]
        k["flops"] += r["flops"]
        k["bytes"] += r["bytes"]
    for k in kernels.values():
        k["share"] = round(k["ms"] / step_ms_sum, 4) if step_ms_sum else None
        k["tflops"] = round(k["flops"] / (k["ms"] * 1e-3) / 1e12, 1) if k["flops"] else None
        k["gbs"] = round(k["bytes"] / (k["ms"] * 1e-3) / 1e9, 1) if k["bytes"] else None
        k["ms"] = round(k["ms"], 3)
        del k["flops"], k["bytes"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                tj = json.load(fh)
            traffic = {"dram_bytes_per_launch": tj.get("dram_bytes_per_launch"),
                       "algorithmic_bytes_per_launch": tj.get("algorithmic_bytes"),
                       "launch_M": tj.get("M"), "source": "profiles/ncu_gemm_traffic.json"}
        except Exception:
            traffic = None

    # -------- e2e through the public API with host buffers. Per step: every request's task is
    # created from host token ids (H2D upload on the context's upload stream), enqueued, and its
    # logits read back to the host (D2H), then destroyed. Tasks of a step are created and
    # enqueued before the first read-back so host work overlaps the GPU, as a serving loop would.
    # Steps are double-buffered like a serving loop: step k+1's requests are submitted before
    # step k's results are read back, each read waiting only for its own request.
    e2e_steps = max(1, args.steps)
    h2d = d2h = 0

    def submit_step():
        nonlocal h2d
        live = []
        for i, t in enumerate(tokens):
            task = ctx.create_task([t], None, "operator", 10_000 + i)
            h2d += task.info()["upload_bytes"]
            task.begin_segment(0)
            task.enqueue(0, task.n_entries)
            live.append(task)
        return live

    barrier()
    ctx.sync()
    t0 = time.perf_counter()
    pending = submit_step()
    for k in range(e2e_steps):
        nxt = submit_step() if k + 1 < e2e_steps else []
        for task in pending:
            lg = task.logits()  # device -> host read of the request's result
            d2h += lg.nbytes
            task.destroy()
        pending = nxt
    ctx.sync()
    h2d //= e2e_steps
    d2h //= e2e_steps
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()
    e2e_value = job_step_tokens * e2e_steps / e2e_s

    # -------- p99 preemption latency on a long request (async launch worker)
    try:
        pre = preemption_latency(ctx, shape, rank)
    except Exception as e:  # keep the bench line; record why the leg failed
        pre = {"error": repr(e)[:300]}

    # -------- the TTFT predictor the scheduler ranks with (S-EDF slack, Alg. 1 admission):
    # fitted by the reference's own fit_ttft_poly to measured B200 single-request latencies on
    # its log-spaced grid (`prefillsim calibrate`)
    ttft = None
    if rank == 0 and not args.skip_goodput:
        try:
            from paper_2602_16603_b200.calibrate import (fit_ttft_predictor, measure_ttft_samples,
                                                         ttft_grid)

            samples = measure_ttft_samples(ctx, shape, ttft_grid())
            poly, quality = fit_ttft_predictor(samples, 2)
            ttft = {"poly": poly, "samples": [[int(n), round(t, 6)] for n, t in samples],
                    "coefficients": list(poly.coefficients), **quality}
        except Exception as e:  # the reference is absent or the fit was rejected
            ttft = {"error": repr(e)[:200]}

    # -------- goodput: reference goodput_search on the B200-calibrated cost model
    good = None
    if rank == 0 and not args.skip_goodput:
        try:
            good = calibrated_goodput(prof, shape, args, ws,
                                      ttft.get("poly") if isinstance(ttft, dict) else None)
        except Exception as e:  # keep the bench line even if the reference is unavailable
            good = {"error": repr(e)[:200]}

    # -------- wall-clock check of the calibrated goodput: replay the config-2 trace in real time
    if (rank == 0 and good is not None and "value" in good and not args.skip_live):
        for t in tasks:
            t.destroy()
        tasks = []
        try:
            good["live_check"] = live_check(ctx, shape, good, args,
                                            ttft.get("poly") if isinstance(ttft, dict) else None)
        except Exception as e:
            good["live_check"] = {"error": repr(e)[:300]}

    cpu = None
    if rank == 0 and ws == 1 and not args.skip_cpu:
        v, cores, sample = cpu_sample()
        cpu = {"value": v, "unit": "tok/s", "cores": cores, "kind": "port", "sample": sample}
        try:
            cpu["control_plane"] = control_plane_time()
        except Exception as e:  # the reference scheduler is absent on this host
            cpu["control_plane"] = {"error": repr(e)[:200]}

    for t in tasks:
        t.destroy()
    if rank == 0:
        line = {
            "metric": "prefill_tokens_per_s",
            "value": value,
            "unit": "tok/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "ms_per_step_profiled": round(ms_prof, 3),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random-init weights, seeded token ids, config-2 trace lengths)",
            "config": {
                "workload": f"{MODEL} prefill, {STEP_REQUESTS} requests/step/GPU from the config-2 "
                            "3-class trace (seed 7), operator-granularity boundary checks armed",
                "model": MODEL,
                "tokens_per_step_per_gpu": step_tokens,
                "request_lens_rank0": lens,
                "parallelism": f"{ws} independent instances" if ws > 1 else "single instance",
                "l2": "inputs larger than L2 (16 GB of weights streamed per step)",
            },
            "roofline": {
                "bound": "tensor",
                "kernel": "gate_up_proj GEMM + SwiGLU epilogue (tcgen05, dominant kernel)",
                "timing": f"CUDA events around every kernel on the prefill stream, {prof_steps} "
                          f"profiled steps of the same workload ({n_launch} launches)",
                "algorithmic_flops_per_step": gu_flops / prof_steps,
                "achieved": round(achieved, 1),
                "peak": peak,
                "peak_source": f"{peak_kind} bf16_tflops_sustained (kernels timed inside a long step)",
                "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4) if peak else None,
                # dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full of the
                # same kernel at M = 4465), and where it came from
                "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                "traffic_detail": traffic,
                "all_dense_gemms_tflops": round(all_gemm, 1),
            },
            "kernels": kernels,
            "e2e": {"value": e2e_value, "unit": "tok/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "clocks": clk,
            "goodput_req_s": (good or {}).get("live_check", {}).get("live_goodput_req_s")
            if isinstance(good, dict) else None,
            "goodput_req_s_calibrated_sim": (good or {}).get("value") if isinstance(good, dict) else None,
            "p99_preempt_latency_ms": pre.get("p99_ms"),
            "preemption": pre,
            "goodput": good,
            "ttft_predictor": ({k: v for k, v in ttft.items() if k != "poly"}
                               if isinstance(ttft, dict) else None),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


def preemption_latency(ctx, shape, rank: int, n_signals: int = 40, length: int = 8192):
    """Signal at random instants while a long request runs through the async launch worker;
    blocking = host-observed signal -> ACK. Bound: that request's longest entry."""
    from paper_2602_16603_b200 import _lib

    rng = np.random.default_rng(rank)
    tok = rng.integers(0, shape.vocab, length).astype(np.int32)
    task = ctx.create_task([tok], None, "operator", 900_000)
    # entry durations of a straight run (the reference's blocking bound, test_properties.py:90-94)
    ctx.profile(True)
    ctx.drain_profile()
    task.begin_segment(0)
    task.enqueue(0, task.n_entries)
    prof = ctx.drain_profile()
    ctx.profile(False)
    entry_ms = []
    acc = 0.0
    for r in prof:  # an entry = its kernels up to and including its GEMM / attention
        acc += r["ms"]
        if r["kind"] in ("rmsnorm", "final_rmsnorm"):
            continue
        if r["kind"] == "lm_head_gemm":
            entry_ms[-1] += acc  # final norm + lm_head run inside the last down_proj entry
        else:
            entry_ms.append(acc)
        acc = 0.0
    max_entry = max(entry_ms) if entry_ms else None
    lat, stops_at = [], []
    cursor = 0
    n = task.n_entries
    while len(lat) < n_signals:
        if cursor >= n:
            cursor = 0
        task.start(cursor)
        dwell = rng.uniform(0.2e-3, 3e-3)
        t_end = time.perf_counter() + dwell
        while time.perf_counter() < t_end:
            pass
        st = task.poll()
        if st.state == _lib.FP_TASK_DONE:
            cursor = 0
            continue
        t0 = time.perf_counter()
        ctx.signal()
        while True:
            st = task.poll()
            if st.state in (_lib.FP_TASK_STOPPED, _lib.FP_TASK_DONE):
                break
        t1 = time.perf_counter()
        if st.state == _lib.FP_TASK_DONE:
            ctx.clear()
            cursor = 0
            continue
        lat.append((t1 - t0) * 1e3)
        stops_at.append(st.cursor)
        cursor = st.cursor
    ctx.sync()
    task.destroy()
    lat_sorted = sorted(lat)
    rank99 = max(math.ceil(0.99 * len(lat_sorted)), 1)  # nearest rank, metrics.py:62-74
    return {
        "count": len(lat),
        "p99_ms": round(lat_sorted[rank99 - 1], 4),
        "mean_ms": round(float(np.mean(lat)), 4),
        "max_ms": round(lat_sorted[-1], 4),
        "bound_max_entry_ms": round(max_entry, 4) if max_entry else None,
        "request_tokens": length,
        "mode": "async launch worker, window 8 entries, host-observed",
    }


def live_run(ctx, shape, params, pc, rate, duration):  # pc.predictor: the measured fit
    from paper_2602_16603_b200 import refsim
    from paper_2602_16603_b200.live import replay_rounds, run_live

    ps = refsim.load()
    base = config2_trace(rate=20.0, duration=duration * rate / 20.0)
    trace = ps.scale_rate(base, rate / base.base_rate())

    def tok(r):
        return np.random.default_rng(5000 + r.id).integers(0, shape.vocab, r.num_tokens).astype(np.int32)

    t0 = time.perf_counter()
    rounds: list = []
    res = run_live(trace, pc, params, ctx, tok, max_wall_s=10 * duration + 60, round_log=rounds)
    wall = time.perf_counter() - t0
    bl = ps.blocking_stats(res.blocking_log)
    # wall-clock scheduling parity: every round replayed through a fresh reference scheduler
    try:
        rep = replay_rounds(trace, pc, params, rounds)
        replay = {"rounds": rep["rounds"], "commands": rep["commands"], "mismatches": 0}
    except AssertionError as e:
        replay = {"mismatch": str(e)[:300]}
    max_entry = {r["done"]: r["max_entry_s"] for r in rounds if "done" in r}
    over = sum(1 for sig, ack, tid in res.blocking_log if ack - sig > max_entry.get(tid, 0.0) + 2e-3)
    return {
        "rate_req_s": round(rate, 3),
        "requests": len(trace),
        "attainment": ps.slo_attainment(res.outcomes),
        "attainment_by_class": {c: ps.slo_attainment(res.outcomes, c)
                                for c in sorted({o.task for o in res.outcomes})},
        "commands": res.commands,
        "rounds": res.rounds,
        "p99_blocking_ms": None if bl["p99_s"] is None else round(bl["p99_s"] * 1e3, 3),
        "max_blocking_ms": None if bl["max_s"] is None else round(bl["max_s"] * 1e3, 3),
        "wall_s": round(wall, 2),
        "replay": replay,
        "blocking_over_max_entry_plus_2ms": over,
    }


def live_check(ctx, shape, good, args, predictor=None):
    """Wall-clock goodput: the live driver replays `live_duration` s of the config-2 trace at
    candidate rates (bisection between 0.5x and 1x the calibrated goodput, 90% target), for
    S-EDF + operator preemption; EDF + 2048-token chunks (DistServe-CP analogue) is replayed at
    the same final rate for comparison."""
    from paper_2602_16603_b200 import refsim

    ps = refsim.load()
    params = ps.CostParams.from_json_dict(good["cost_params"])
    sedf = ps.PolicyConfig(predictor=predictor)
    cp2k = ps.PolicyConfig(policy=ps.PolicyKind.EDF, granularity=ps.PreemptionGranularity.CHUNK,
                           chunk_tokens=2048, predictor=predictor)
    r0 = float(good["value"])
    probes = []
    hi_run = live_run(ctx, shape, params, sedf, r0, args.live_duration)
    probes.append(hi_run)
    if hi_run["attainment"] >= 0.9:
        best, saturated = r0, True
    else:
        saturated = False
        lo, hi = 0.5 * r0, r0
        run = live_run(ctx, shape, params, sedf, lo, args.live_duration)
        probes.append(run)
        best = lo if run["attainment"] >= 0.9 else None
        for _ in range(max(0, args.live_probes - 1) if best is not None else 0):
            mid = 0.5 * (lo + hi)
            run = live_run(ctx, shape, params, sedf, mid, args.live_duration)
            probes.append(run)
            if run["attainment"] >= 0.9:
                best, lo = mid, mid
            else:
                hi = mid
    final = best if best is not None else 0.5 * r0
    cmp = live_run(ctx, shape, params, cp2k, final, args.live_duration)
    return {
        "live_goodput_req_s": best,
        "saturated_at_calibrated_rate": saturated,
        "method": f"live driver, {args.live_duration:.0f} s of config-2 arrivals per probe, "
                  "90% TTFT-SLO target, bisection between 0.5x and 1x the calibrated goodput",
        "probes_sedf_operator": probes,
        "edf_chunk2048_at_same_rate": cmp,
    }


def calibrated_goodput(prof, shape, args, n_instances: int = 1, predictor=None):
    from paper_2602_16603_b200 import refsim
    from paper_2602_16603_b200.calibrate import fit_cost_params, predicted_vs_measured

    ps = refsim.load()
    params = fit_cost_params(prof, shape.num_layers)
    err = predicted_vs_measured(params, prof)
    base = config2_trace(rate=20.0, duration=args.goodput_duration)
    rc = ps.RunConfig(ps.PolicyConfig(predictor=predictor), params)
    t0 = time.perf_counter()
    res = ps.goodput_search(base, rc, target=0.9, rate_bounds=(1.0, 512.0), tol=0.05)
    out = {
        "value": res.value,
        "unit": "req/s",
        "saturated": res.saturated,
        "method": "reference goodput_search (S-EDF, operator preemption, G=4096) on the cost "
                  "model re-fitted to this run's B200 kernel timings (virtual clock)",
        "trace": f"config-2 3-class trace, {args.goodput_duration:.0f} s, seed 7",
        "fit_max_rel_err": round(err, 4),
        "probes": res.num_runs,
        "search_s": round(time.perf_counter() - t0, 2),
        "cost_params": params.to_json_dict(),
    }
    # same search for the chunked-prefill baseline (EDF + 2048-token chunks, DistServe-CP)
    try:
        rc2 = ps.RunConfig(ps.PolicyConfig(policy=ps.PolicyKind.EDF,
                                           granularity=ps.PreemptionGranularity.CHUNK,
                                           chunk_tokens=2048, predictor=predictor), params)
        r2 = ps.goodput_search(base, rc2, target=0.9, rate_bounds=(1.0, 512.0), tol=0.05)
        out["edf_chunk2048_value"] = r2.value
    except Exception as e:
        out["edf_chunk2048_value"] = repr(e)[:120]
    if n_instances > 1:
        # the whole N-GPU deployment: round-robin proxy over N independent instances, the
        # reference bisection over the merged outcomes (dispatch.goodput_search_instances)
        from paper_2602_16603_b200 import dispatch

        base_n = config2_trace(rate=20.0 * n_instances, duration=args.goodput_duration)
        rd = dispatch.goodput_search_instances(base_n, rc, n_instances, target=0.9,
                                               rate_bounds=(1.0, 512.0 * n_instances), tol=0.05,
                                               jobs=min(n_instances, os.cpu_count() or 1))
        out["deployment"] = {"instances": n_instances, "value": rd.value, "unit": "req/s",
                             "saturated": rd.saturated, "probes": rd.num_runs,
                             "method": "round-robin over independent instances, reference "
                                       "goodput_search over the merged outcomes"}
    return out


def run_tp(args):
    """Config 4: Qwen2.5-32B shape, tensor parallel over `--tp N` GPUs, one
    process per GPU. Every rank runs the SAME requests on its Megatron shard; the o_proj /
    down_proj GEMMs are the fused exchange kernels (each tile's partial flagged to the peers and
    folded over peer memory while the next tile's MMAs run), and rank 0 decides every boundary
    for all ranks. value = the step's tokens (counted once, not per rank) / the slowest rank's
    device time: strong scaling. The exchange share per rank is the o_proj + down_proj kernel
    time from the profiled steps (the all-reduce lives inside those kernels)."""
    import torch

    from paper_2602_16603_b200.config import SHAPES
    from paper_2602_16603_b200.native import PrefillContext, connect_tp_dist

    ws, rank, local = dist_env()
    if ws != args.tp:
        raise SystemExit(f"--tp {args.tp} needs {args.tp} ranks (WORLD_SIZE={ws})")
    dist = None
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shape = SHAPES["qwen2.5-32b"]
    reqs = step_requests(1, 0)[: args.tp_requests]
    lens = [r.num_tokens for r in reqs]
    tokens = [np.random.default_rng(1000 + r.id).integers(0, shape.vocab, r.num_tokens)
              .astype(np.int32) for r in reqs]
    step_tokens = int(sum(lens))
    pages = sum((n + 127) // 128 for n in lens)
    ctx = PrefillContext(shape, device=local, kv_pages=2 * pages + 64, page_size=128,
                         max_pos=40000, tp_rank=rank, tp_size=ws)
    if ws > 1:
        connect_tp_dist(ctx, max(lens))
    ctx.init_random(seed=0)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=local)
    tasks = [ctx.create_task([t], None, "operator", i) for i, t in enumerate(tokens)]

    def run_step():
        for t in tasks:
            t.begin_segment(0)
            t.enqueue(0, t.n_entries)

    def reduce(x: float, op) -> float:
        if dist is None:
            return x
        v = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(v, op=op)
        return float(v.item())

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(max(args.warmup, 1)):
        run_step()
    ctx.sync()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launch_count()
    barrier()
    torch.cuda.synchronize(local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        run_step()
    e1.record(stream)
    ctx.sync()
    torch.cuda.synchronize(local)
    barrier()
    launches = ctx.launch_count() - launches0
    clk = clocks.stop()
    ms_max = reduce(e0.elapsed_time(e1), dist.ReduceOp.MAX if dist else None)
    value = step_tokens * args.steps / (ms_max / 1e3)
    # per-kernel profile (one step): exchange share and the dominant GEMM's rate
    ctx.profile(True)
    ctx.drain_profile()
    run_step()
    prof = ctx.drain_profile()
    ctx.profile(False)
    tot = sum(r["ms"] for r in prof)
    xch = sum(r["ms"] for r in prof if r["kind"] in ("o_gemm", "down_gemm", "allreduce"))
    gu = [r for r in prof if r["kind"] == "gate_up_gemm"]
    gu_tf = sum(r["flops"] for r in gu) / (sum(r["ms"] for r in gu) * 1e-3) / 1e12 if gu else 0.0
    share = reduce(xch / tot if tot else 0.0, dist.ReduceOp.MAX if dist else None)
    # e2e: host token ids -> host logits through the public API, copies inside the region
    barrier()
    ctx.sync()
    t0 = time.perf_counter()
    h2d = d2h = 0
    for _ in range(args.steps):
        live = []
        for i, t in enumerate(tokens):
            task = ctx.create_task([t], None, "operator", 10_000 + i)
            h2d += task.info()["upload_bytes"]
            task.begin_segment(0)
            task.enqueue(0, task.n_entries)
            live.append(task)
        for task in live:
            d2h += task.logits().nbytes
            task.destroy()
    ctx.sync()
    e2e_s = reduce(time.perf_counter() - t0, dist.ReduceOp.MAX if dist else None)
    for t in tasks:
        t.destroy()
    if rank == 0:
        peaks, peak_kind = measured_peaks()
        peak = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]
        line = {
            "metric": "prefill_tokens_per_s",
            "value": value,
            "unit": "tok/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random-init weights, seeded token ids, config-2 trace lengths)",
            "config": {"workload": f"qwen2.5-32b prefill, tensor parallel TP={ws}, "
                                   f"{len(reqs)} requests/step of the config-2 trace",
                       "model": "qwen2.5-32b", "tokens_per_step": step_tokens,
                       "request_lens": lens, "parallelism": f"tp{ws}",
                       "l2": "inputs larger than L2 (weights streamed per step)"},
            "roofline": {"bound": "tensor", "kernel": "gate_up_proj GEMM + SwiGLU (per rank)",
                         "achieved": round(gu_tf, 1), "peak": peak, "unit": "TFLOP/s",
                         "frac": round(gu_tf / peak, 4) if peak else None, "traffic": None,
                         "peak_source": peak_kind},
            "exchange_share_per_rank": round(share, 4),
            "e2e": {"value": step_tokens * args.steps / e2e_s, "unit": "tok/s",
                    "h2d_bytes_per_step": int(h2d // args.steps),
                    "d2h_bytes_per_step": int(d2h // args.steps)},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-goodput", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--goodput-duration", type=float, default=60.0)
    ap.add_argument("--skip-live", action="store_true")
    ap.add_argument("--live-duration", type=float, default=10.0)
    ap.add_argument("--live-probes", type=int, default=3)
    ap.add_argument("--tp", type=int, default=0,
                    help="config 4: Qwen2.5-32B tensor parallel over this many GPUs (one rank each)")
    ap.add_argument("--tp-requests", type=int, default=STEP_REQUESTS)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.tp:
        if args.tp > 1 and "WORLD_SIZE" not in os.environ:
            sys.exit(spawn_ranks(args.tp))
        run_tp(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    else:
        run_ours(args)


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch as N ranks (one per GPU) the way the
    driver does, so the line always measures N GPUs and reports n_gpus = N."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.run(cmd).returncode


if __name__ == "__main__":
    main()
