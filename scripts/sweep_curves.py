#!/usr/bin/env python3
"""QPS-recall curves of one bench line's sweep (profiles/*.json): per family (recall policy, f3
threshold) and search width, the (itopk, recall, MQPS) points; and per family the fastest point at
each recall level. Tooling only.

  python scripts/sweep_curves.py profiles/r02ll_bench_yfcc.json [--levels 0.85,0.88,0.90,0.95,0.99]
"""
import argparse
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("line")
    ap.add_argument("--levels", default="0.80,0.85,0.88,0.90,0.95,0.97,0.99")
    a = ap.parse_args()
    j = json.load(open(a.line))
    n = j["config"]["queries_per_step"]
    levels = [float(x) for x in a.levels.split(",")]
    fams = {}
    for s in j["sweep"]:
        fams.setdefault((s["recall_mode"], s["and_scan_threshold"]), []).append(s)
    print("| policy | f3 | " + " | ".join(f"QPS @ {l:.2f}" for l in levels) + " | max recall |")
    print("|---|---|" + "---|" * (len(levels) + 1))
    for (mode, f3), pts in sorted(fams.items(), key=lambda kv: (kv[0][0], kv[0][1])):
        cells = []
        for l in levels:
            ok = [p for p in pts if p["recall_tie_aware"] >= l]
            if ok:
                b = min(ok, key=lambda p: p["ms"])
                cells.append(f"{n / b['ms'] / 1e3:.2f}M (w{b['search_width']}, {b['itopk']})")
            else:
                cells.append("—")
        mx = max(p["recall_tie_aware"] for p in pts)
        print(f"| {mode} | {f3} | " + " | ".join(cells) + f" | {mx:.4f} |")


if __name__ == "__main__":
    main()
