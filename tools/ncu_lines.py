"""Per-CUDA-source-line instruction counts and stall samples from an ncu
report (--import-source on, -lineinfo build).
usage: ncu_lines.py rep.ncu-rep [kernel-substring] [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, path, hdr, agg = None, None, None, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        fn = r[1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and want in (fn or "") and len(r) > 7 and r[2] == "-":
        key = (fn, path, int(r[0]))
        a = agg.setdefault(key, [r[1].strip(), 0, 0])
        a[1] += int(r[hdr.index("Instructions Executed")] or 0)
        a[2] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
for f in sorted({k[0] for k in agg}):
    rows = [(k, v) for k, v in agg.items() if k[0] == f]
    ti = sum(v[1] for _, v in rows) or 1
    ts = sum(v[2] for _, v in rows) or 1
    print(f"== {f[:70]}  warp-inst {ti:.3e}  samples {ts}")
    order = 2 if "--by-stall" in sys.argv else 1
    for (_, p, ln), (src, ni, ns) in sorted(rows, key=lambda kv: -kv[1][order])[:top]:
        print(f"  {p}:{ln:<5d} inst {100 * ni / ti:5.1f}%  stall {100 * ns / ts:5.1f}%  {src[:80]}")
