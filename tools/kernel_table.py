"""Per-kernel DRAM GB/s from an ncu CSV (--metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum): one row per kernel name,
summed over its launches.  usage: python tools/kernel_table.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
acc = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9, "second": 1.0}
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    try:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    except ValueError:
        continue
    acc[name][r[mi]] += v
    if r[mi] == "gpu__time_duration.sum":
        cnt[name] += 1
print(f"{'kernel':58s} {'launches':>8s} {'ms':>10s} {'DRAM GB':>10s} {'GB/s':>8s} {'of 6549':>8s}")
for name, m in sorted(acc.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    t = m["gpu__time_duration.sum"]
    b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    gbs = b / t / 1e9 if t else 0.0
    print(f"{name[:58]:58s} {cnt[name]:8d} {1e3 * t:10.3f} {b / 1e9:10.3f} {gbs:8.0f} {gbs / 6549.4:8.2f}")
