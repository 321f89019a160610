#!/usr/bin/env python3
"""Markdown tables for BASELINE.md §4 from committed bench lines (profiles/*.json). Tooling only.

  python scripts/baseline_tables.py profiles/r02gg_bench_yfcc.json profiles/r02gg_bench_sift.json ...
"""
import json
import sys


def m(x):
    return f"{x / 1e6:.2f}M"


def main():
    lines = [json.load(open(p)) for p in sys.argv[1:]]
    print("| Config | Target | Routing | Operating point | QPS | Recall@10 (single / AND2) | e2e QPS | Oracle QPS (cores) |")
    print("|---|---|---|---|---|---|---|---|")
    for j in lines:
        wl = j["config"]["workload"].split(" (")[0]
        cpu = j.get("cpu_baseline") or {}
        for fam, key in (("best", "at_recall"), ("paper", "at_recall_paper")):
            for t, r in j[key].items():
                if "qps" not in r:
                    if fam == "paper":
                        b = r.get("best") or {}
                        print(f"| {wl} ({j['dtype']}) | {t} | paper only | not reached: best {b.get('recall_tie_aware', 0):.4f} "
                              f"({b.get('recall_mode')}, w {b.get('search_width')}, itopk {b.get('itopk')}) | — | — | — | — |")
                    continue
                if fam == "paper" and j["at_recall"].get(t, {}).get("itopk") == r["itopk"] and \
                        j["at_recall"][t].get("and_scan_threshold") == r["and_scan_threshold"]:
                    continue
                split = r.get("by_class_and_path", {})
                s1 = split.get("single", {}).get("recall_tie_aware")
                s2 = split.get("and2", {}).get("recall_tie_aware")
                cls = f" ({s1:.3f} / {s2:.3f})" if s1 is not None and s2 is not None else ""
                e2e = m(j["e2e"]["value"]) if (t == "0.90" and fam == "best" and j.get("e2e")) else "—"
                oq = f"{cpu['value'] / 1e3:.0f}K ({cpu['cores']})" if (t == "0.90" and fam == "best" and cpu) else "—"
                print(f"| {wl} ({j['dtype']}) | {t} | {'f3' if r['and_scan_threshold'] else 'paper'} | itopk {r['itopk']}, w "
                      f"{r['search_width']}, {r['recall_mode']}, f3 {r['and_scan_threshold']} | **{m(r['qps'])}** | "
                      f"{r['recall_tie_aware']:.4f}{cls} | {e2e} | {oq} |")
    print()
    print("| Config | dominant kernel | algorithmic bytes / launch | kernel ms (phase events) | frac | ncu DRAM bytes / launch | phases ms (route / filter / scan / graph / total) |")
    print("|---|---|---|---|---|---|---|")
    for j in lines:
        wl = j["config"]["workload"].split(" (")[0]
        rf, ph = j["roofline"], j["phases_ms"]
        tr = f"{rf['traffic'] / 1e9:.2f} GB" if rf.get("traffic") else "—"
        print(f"| {wl} ({j['dtype']}) | `{rf['kernel']}` | {rf['algorithmic_bytes_per_launch'] / 1e9:.2f} GB | "
              f"{rf['kernel_ms_per_launch']:.3f} | {rf['frac']:.3f} | {tr} | {ph['route']:.2f} / {ph['filter']:.2f} / "
              f"{ph['scan']:.2f} / {ph['graph']:.2f} / {ph['total']:.2f} |")
    print()
    for j in lines:
        lat = j.get("latency")
        if not lat:
            continue
        wl = j["config"]["workload"].split(" (")[0]
        row = " | ".join(f"{lat[b]['host']['p50_ms']:.3f} / {lat[b]['device']['p50_ms']:.3f}" for b in ("batch1", "batch10", "batch100"))
        sv = lat.get("serve", {})
        print(f"latency {wl}: batch 1 / 10 / 100 p50 ms (host / device): {row}; serve p50 {sv.get('p50_ms', 0):.3f} ms "
              f"p99 {sv.get('p99_ms', 0):.3f} ms, single-batch {sv.get('single_batch_qps', 0) / 1e6:.2f}M QPS")


if __name__ == "__main__":
    main()
