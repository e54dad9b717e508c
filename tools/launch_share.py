"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_share.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
tot, cnt, unit = collections.defaultdict(float), collections.Counter(), "ns"
for r in data:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
    unit = r[ui]
T = sum(tot.values())
print(f"launches {sum(cnt.values())}  total {T / 1e6:.2f} ms (cold-cache, serialised: compare shares)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{100 * v / T:6.2f}%  {cnt[k]:6d} launches  {v / cnt[k] / 1e3:10.2f} us/launch  {k[:100]}")
