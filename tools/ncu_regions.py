"""Stall samples of one kernel in an ncu report, summed between barrier instructions (SASS order)."""
import csv
import subprocess
import sys

rep, which = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        kernels.append(cur)
        hdr = None
        continue
    if cur is None:
        continue
    if r and r[0] == "Address":
        cur.append(("H", r))
        continue
    cur.append(("D", r))
k = kernels[which]
h = [r for t, r in k if t == "H"][0]
data = [dict(zip(h, r)) for t, r in k if t == "D" and len(r) == len(h)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data)
print("instructions", len(data), "samples", tot)
acc, start = 0, 0
marks = ("BAR.SYNC", "UCGABAR", "BAR.ARV", "EXIT", "BRA")
for i, d in enumerate(data):
    acc += int(d["Warp Stall Sampling (All Samples)"])
    s = d["Source"].strip()
    if any(s.startswith(m) or (" " + m) in s for m in marks[:3]) or i == len(data) - 1:
        print("%5d-%5d %6.1f%%  %s" % (start, i, 100.0 * acc / tot, s[:60]))
        acc, start = 0, i + 1
