"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel count, total, share."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.reader(lines))
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].replace("flmisr::", "").replace("<unnamed>::", "")
    tot[name] += float(r[iv].replace(",", ""))
    cnt[name] += 1
all_ns = sum(tot.values())
print(f"{'kernel':40s} {'launches':>9s} {'total us':>10s} {'avg us':>9s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} {cnt[k]:9d} {tot[k] / 1e3:10.1f} {tot[k] / cnt[k] / 1e3:9.2f} {100 * tot[k] / all_ns:6.1f}%")
print(f"{'TOTAL':40s} {sum(cnt.values()):9d} {all_ns / 1e3:10.1f}")
