#!/usr/bin/env python3
"""Aggregate an ncu report's source view (cuda,sass) per CUDA source line: stall samples and
instructions executed. Usage: ncu_lines.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) == len(hdr):
        d = dict(zip(hdr[2:], r[2:]))
        if r[2] != "-":
            continue  # sass rows (address set) are attributed to their cuda line row already
        try:
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        rows.append((samp, inst, fname, int(r[0]), r[1][:90]))
tot_s = sum(x[0] for x in rows) or 1
tot_i = sum(x[1] for x in rows) or 1
print(f"total samples {tot_s}  total warp-inst {tot_i}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {f}:{ln:<4} {src}")
