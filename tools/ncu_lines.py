"""Per-source-line share of executed warp instructions (and stall samples) for one kernel of an ncu report.
    python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kre:
    cmd += ["-k", "regex:" + kre]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
cur, agg, hdr = None, {}, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    try:
        ln = int(r[0])
        v = int(r[hdr.index("Instructions Executed")])
        smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    a = agg.setdefault((cur, ln), [0, 0, r[1][:100]])
    a[0] += v
    a[1] += smp
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot}, stall samples {tots}")
for (f, ln), (v, smp, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v / tot * 100:5.1f}% inst {smp / tots * 100:5.1f}% samp  {f}:{ln}  {s}")
