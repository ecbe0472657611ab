"""profiles/traffic.json from the ncu reports of tools/traffic_capture.sh: DRAM read + write bytes per
launch of each config's persistent loop kernel (the `traffic` of bench.py's roofline block)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(ROOT, "profiles", "traffic.json")
tr = json.load(open(path)) if os.path.exists(path) else {}
for cfg in sys.argv[1:]:
    f = os.path.join(ROOT, "gpurun_out", f"traffic_{cfg}.csv")
    if not os.path.exists(f):
        continue
    lines = [ln for ln in open(f) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h, units, r = rows[0], rows[1], rows[2]

    def val(k):
        v = float(r[h.index(k)].replace(",", ""))
        u = units[h.index(k)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    ent = tr.setdefault(cfg, {})
    ent["scg_loop"] = b
    ent["scg_loop_source"] = (f"round 2: ncu --set full of the first timed launch of {r[h.index('Kernel Name')].split('(')[0]} "
                              f"under `bench.py --config {cfg}` (tools/traffic_capture.sh), dram read + write")
    print(cfg, b / 1e9, "GB per launch")
json.dump(tr, open(path, "w"), indent=1)
