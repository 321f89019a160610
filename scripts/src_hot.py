#!/usr/bin/env python3
"""Hot source lines of one kernel from an ncu report (--print-source cuda,sass CSV):
   src_hot.py REPORT.ncu-rep KERNEL_REGEX [N]  -> top-N lines by warp-stall samples and by instructions."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, agg = None, {}
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0, 0, r[1][:110]])
    a[0] += samp
    a[1] += inst
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
print("--- by stall samples")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{100 * v[0] / tot_s:5.1f}% s {100 * v[1] / tot_i:5.1f}% i  {k[0]}:{k[1]}  {v[2]}")
print("--- by instructions")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:N]:
    print(f"{100 * v[0] / tot_s:5.1f}% s {100 * v[1] / tot_i:5.1f}% i  {k[0]}:{k[1]}  {v[2]}")
