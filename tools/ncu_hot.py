"""Print headline metrics and the hottest SASS lines of an ncu report (local analysis helper).

    python tools/ncu_hot.py <report.ncu-rep> [n]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
for w in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
          "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]:
    if w in h:
        print(f"{w} = {v[h.index(w)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ia = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot = sum(int(r[ia]) for r in data) or 1
ins = sum(int(r[ie]) for r in data)
print(f"warp instructions executed: {ins}")
sc = [x for x in hdr if x.startswith("stall_") and "Not" not in x]
order = sorted(range(len(data)), key=lambda i: -int(data[i][ia]))[:n]
for i in order:
    r = data[i]
    st = sorted(((x, int(r[hdr.index(x)])) for x in sc if int(r[hdr.index(x)]) > 0), key=lambda t: -t[1])[:2]
    print(f"{int(r[ia]) * 100 / tot:5.1f}% {r[1].strip()[:58]:58s} {st} <- {data[i - 1][1].strip()[:45]}")
ops = collections.Counter()
for r in data:
    t = r[1].strip().split()
    if t:
        ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += int(r[ie])
print("top opcodes:", ", ".join(f"{k} {c * 100 / max(ins, 1):.1f}%" for k, c in ops.most_common(12)))
