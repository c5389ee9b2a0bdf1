"""Per CUDA source line: share of warp-stall samples and of executed warp instructions, from an
ncu report captured with -lineinfo and --import-source on (cuda,sass correlation).

    python tools/ncu_lines.py <report.ncu-rep> [n]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
samp = collections.Counter()
inst = collections.Counter()
stall = collections.defaultdict(collections.Counter)
text = {}
fname = None
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit():
        continue
    key = (fname, int(row[0]))
    text[key] = row[1].strip()
    try:
        s = int(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        i = int(row[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    samp[key] += s
    inst[key] += i
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
print(f"samples {ts}, warp instructions {ti}")
for key, s in samp.most_common(n):
    print(f"{100 * s / ts:5.1f}% samp {100 * inst[key] / ti:5.1f}% inst  {key[0]}:{key[1]:<4d} {text[key][:90]}")
