"""Top stalled SASS instructions per kernel from an ncu report:
python tools/ncu_hot.py report.ncu-rep [kernel-index ...] [--top N]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = 18
    args = [a for a in sys.argv[2:]]
    if "--top" in args:
        i = args.index("--top")
        top = int(args[i + 1])
        del args[i:i + 2]
    want = [int(a) for a in args]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name",')[1:]
    for bi, b in enumerate(blocks):
        if want and bi not in want:
            continue
        lines = b.split("\n")
        name = lines[0]
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        h = rows[0]
        si = h.index("Warp Stall Sampling (All Samples)")
        cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        tot = sum(int(r[si]) for r in rows[1:] if len(r) > si and r[si].isdigit())
        print(f"== [{bi}] {name[:90]} samples={tot}")
        rs = sorted((r for r in rows[1:] if len(r) > si and r[si].isdigit()), key=lambda r: -int(r[si]))
        for r in rs[:top]:
            st = sorted(((int(r[h.index(c)]), c[6:]) for c in cols if r[h.index(c)].isdigit()), reverse=True)[:2]
            print(f"  {int(r[si]):6d} {r[1].strip()[:60]:60s} {st}")


if __name__ == "__main__":
    main()
