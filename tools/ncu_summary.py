"""Summarise an ncu report: key metrics per kernel + SASS opcode histogram (per HR pixel)."""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
npx = float(sys.argv[2]) if len(sys.argv) > 2 else 4096 * 4096
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "lts__t_bytes.sum"]
stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    out = {w: r[hdr.index(w)] for w in want if w in hdr}
    print(out["Kernel Name"][:60])
    for w in want[1:]:
        if w in out:
            print(f"  {w:60s} {out[w]}")
    if "smsp__inst_executed.sum" in out:
        print(f"  thread-instr / px = {float(out['smsp__inst_executed.sum']) * 32 / npx:.1f}")
    st = sorted(((float(r[hdr.index(h)] or 0), h) for h in stall), reverse=True)[:8]
    print("  stalls:", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in st))
if "--sass" in sys.argv:
    for k in sys.argv[sys.argv.index("--sass") + 1:]:
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                              f"regex:{k}"], capture_output=True, text=True).stdout
        rr = list(csv.reader(src.splitlines()))
        h = rr[1]
        i_src, i_ex = h.index("Source"), h.index("Instructions Executed")
        ops = collections.Counter()
        tot = 0
        for x in rr[2:]:
            try:
                n = int(x[i_ex])
            except (ValueError, IndexError):
                continue
            m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", x[i_src].strip())
            ops[m.group(2) if m else "?"] += n
            tot += n
        print(k, "opcodes / px:", ", ".join(f"{o}={n * 32 / npx:.1f}" for o, n in ops.most_common(24)))
