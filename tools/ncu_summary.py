"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/...md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def short(name):
    epi = {"0": "store_bf16", "1": "store_f32(lm_head)", "2": "resid(o/down)", "3": "swiglu(gate_up)", "4": "qkv_rope_kv"}
    m = re.search(r"gemm_bf16_tn_kernel<(?:\(int\))?(\d+), *(?:\(int\))?(\d+), *(?:\(int\))?(\d+)(?:, *(?:\(bool\))?(\w+))?>", name)
    if m:
        mode = {"1": " split-capable", "true": " split-capable", "2": " grouped(MoE)",
                "3": " stream-K", "4": " cluster-split"}.get(m.group(4), "")
        width = "" if m.group(1) == "256" else f" {m.group(1)}-wide"
        return f"gemm {epi.get(m.group(2), m.group(2))} cta_group={m.group(3)}{width}{mode}"
    for k in ("attn_prefill_tc_kernel", "rmsnorm_kernel", "init_normal_kernel"):
        if k in name:
            return k
    return name[:40]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        k = short(r[ki])
        agg[k][0] += 1
        agg[k][1] += v
        total += v
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t / 1e3:.1f} | {t / total:.3f} |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    for r in rows[2:]:
        print({w: r[i] for w, i in idx.items()})


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
