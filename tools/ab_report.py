"""Summarise tools/ab_prof.sh output: per-kernel-kind totals (ms per step) per run, and the
per-length comparison of the last round."""
import collections
import glob
import re


def load(f):
    d = collections.defaultdict(dict)
    for line in open(f):
        m = re.match(r'(\S+)\s+M=\s*(\d+)\s+n=\s*(\d+)\s+avg\s+([\d.]+)', line)
        if m:
            d[int(m.group(2))][m.group(1)] = float(m.group(4)) * int(m.group(3)) / 1000
    return d


ks = ['qkv_gemm', 'attn', 'o_gemm', 'gate_up_gemm', 'down_gemm']
files = sorted(glob.glob('gpurun_out/prof_base*.txt')) + sorted(glob.glob('gpurun_out/prof_new*.txt'))
means = {}
for f in files:
    d = load(f)
    tot = {k: round(sum(d[M].get(k, 0) for M in d), 2) for k in ks}
    print(f.split('/')[-1], tot, round(sum(tot.values()), 2))
    arm = 'base' if 'base' in f else 'new'
    means.setdefault(arm, []).append(tot)
for arm, rows in means.items():
    avg = {k: round(sum(r[k] for r in rows) / len(rows), 2) for k in ks}
    print('MEAN', arm, avg, round(sum(avg.values()), 2))
b = load(sorted(glob.glob('gpurun_out/prof_base*.txt'))[-1])
n = load(sorted(glob.glob('gpurun_out/prof_new*.txt'))[-1])
for M in sorted(b):
    if M > 1:
        print(M, ' '.join(f"{k[:5]} {n[M].get(k, 0):.2f}/{b[M].get(k, 0):.2f}" for k in ks))
