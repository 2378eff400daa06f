"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total and mean device time, share of all launches."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[iu], 1e-6)
    v = float(r[iv].replace(",", "")) * scale
    name = r[ik].split("(")[0]
    tot[name] += v
    cnt[name] += 1
allt = sum(tot.values())
print("%-60s %8s %12s %10s %7s" % ("kernel", "launches", "total_ms", "mean_ms", "share"))
for k, v in tot.most_common():
    print("%-60s %8d %12.3f %10.4f %6.2f%%" % (k[:60], cnt[k], v, v / cnt[k], 100 * v / allt))
