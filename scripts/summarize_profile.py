#!/usr/bin/env python3
"""Summarise ncu artefacts from gpurun_out/ into a committed markdown file under profiles/.

  summarize_profile.py OUT.md --launches launches.csv --full prof_k_scan.ncu-rep prof_k_graph.ncu-rep
"""
import argparse
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append((d, dict(zip(hdr, units))))
    return res


def stalls(d):
    st = []
    for n, v in d.items():
        if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
            try:
                st.append((float(v.replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in st) or 1.0
    return [(n, 100 * s / tot) for s, n in sorted(st, reverse=True)[:8]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    md = [f"# {a.title}", ""]
    if a.note:
        md += [a.note, ""]
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hdr = None
        per = defaultdict(list)
        for r in rows:
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    name = d["Kernel Name"].split("(")[0].replace("void ", "")
                    per[name].append(float(d["Metric Value"].replace(",", "")))
        tot = sum(sum(v) for v in per.values()) or 1.0
        md += ["## Launch list (ncu `gpu__time_duration.sum`, `--clock-control none`; cold-cache, serialised)", "",
               "| kernel | launches | mean µs | share of our kernel time |", "|---|---|---|---|"]
        for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{name}` | {len(v)} | {sum(v) / len(v) / 1000:.1f} | {100 * sum(v) / tot:.1f} % |")
        md.append("")
    for rep in a.full:
        for d, u in raw(rep):
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
            md += [f"## `{name}` — `ncu --set full` ({rep.split('/')[-1]})", "", "| metric | value |", "|---|---|"]
            for k in KEEP:
                if k in d:
                    md.append(f"| `{k}` | {d[k]} {u.get(k, '')} |")
            md += ["", "Top stall reasons (pc sampling): " + ", ".join(f"{n} {p:.1f} %" for n, p in stalls(d)), ""]
    open(a.out, "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    sys.exit(main())
