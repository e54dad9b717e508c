"""Summarise an ncu report: SOL, occupancy, DRAM bytes, stall reasons and the
top SASS lines by warp-stall samples.  usage: ncu_summary.py rep.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units = raw[0], raw[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
for r in raw[2:]:
    print("==", r[hdr.index("Kernel Name")][:60])
    for k in keys:
        if k in hdr:
            print(f"   {k:70s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join(f"{h} {100 * v / tot:.0f}%" for v, h in sorted(st, reverse=True)[:7]))

rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv"))))
kern, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], []]
        kern.append(cur)
    elif r and r[0] != "Address" and cur:
        cur[1].append(r)
seen = set()
for name, rs in kern:
    if name in seen:
        continue
    seen.add(name)
    tot = sum(int(r[2]) for r in rs) or 1
    print("== source", name[:60], "samples", tot)
    idx = sorted(range(len(rs)), key=lambda i: -int(rs[i][2]))[:top]
    for i in sorted(idx):
        print(f"   {100 * int(rs[i][2]) / tot:5.1f}%  {rs[i][1].strip()[:70]:70s} exec {rs[i][5]}")
