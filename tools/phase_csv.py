"""Summarise an ncu --csv --metrics per-kernel list: time, instructions per HR pixel, DRAM bytes."""
import csv
import sys

npx = float(sys.argv[2]) if len(sys.argv) > 2 else 4096 * 4096
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
d = {}
for r in rows[1:]:
    d.setdefault((r[iid], r[ik][:40]), {})[r[im]] = r[iv].replace(",", "")
for k, v in d.items():
    inst = float(v.get("smsp__inst_executed.sum", 0))
    print(k[1], "t=%.1f us" % (float(v["gpu__time_duration.sum"]) / 1000), "instr/px=%.1f" % (inst * 32 / npx),
          "dram r=%.0f MB w=%.0f MB" % (float(v.get("dram__bytes_read.sum", 0)) / 1e6, float(v.get("dram__bytes_write.sum", 0)) / 1e6),
          "issue=%s%%" % v.get("smsp__issue_active.avg.pct_of_peak_sustained_active"), "regs", v.get("launch__registers_per_thread"))
