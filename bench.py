#!/usr/bin/env python3
"""bench.py -- QPS at recall@10 >= 0.90 / 0.99 for batched label-filtered top-k search on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config sift|yfcc|tiny] [--impl ours|reference]

A "step" is one vf_search call over the whole query batch of the workload (route -> scan ->
graph -> merge, all §8(a) rows) with queries, labels and outputs resident in HBM. The workload is
BASELINE.json configs[1] (SIFT-like: 1M x 128 fp32 integer-valued vectors, 1K Zipf labels, 10K
single-label queries, k = 10) unless --config says otherwise; see DESIGN.md §3 for the recipe.

Ground truth comes from vf_search in exact mode (T = infinity; parity-tested bit-exact against the
CPU oracle in tests/). The operating point for a recall target is the smallest itopk of the grid
whose mean recall@10 reaches it. L2 is flushed (256 MiB write) before every timed step, outside
the step's CUDA events. Under torchrun (N > 1) the index is label-sharded across the ranks (LPT
over |C_l|; X and the predicate table replicated; items exchanged with NCCL inside vf_search) and
every rank brings its own batch (weak scaling); rank 0 prints the line with value = all ranks'
queries / max-over-ranks time.
The CPU oracle is used ONLY for the cpu_baseline leg and for --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG_INDEX = {"tiny": 0, "sift": 1, "yfcc": 2}
# the 0.90 operating point our arm measured per workload (itopk, search_width, and_scan_threshold,
# scan_threshold);
# the reference arm (the oracle) runs at it so both arms answer the same searches
OP_POINT = {"tiny": (32, 1, 0, 0), "sift": (16, 2, 0, 0), "yfcc": (48, 2, 2000, 0)}
ITOPK_GRID = (16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512)
METRIC = "QPS at recall@10 >=0.90 and >=0.99 (1/2/4/8 B200); p50 latency at batch 1"


def log(*a):
    if int(os.environ.get("RANK", "0")) == 0:
        print("[bench]", *a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- workload
def make_inputs(config: str, device, query_stream: int = 0):
    from workload import gen, graphs
    t0 = time.time()
    w = gen.make_workload(config, query_stream=query_stream)
    c = w.cfg
    log(f"workload {config}: N={c.n_points} D={c.dim} L={c.n_labels} Q={c.n_queries} "
        f"dtype={c.dtype} ({time.time() - t0:.1f}s)")
    t0 = time.time()
    # VF_GRAPH_CACHE=<dir>: reuse the fixture graphs between bench processes of ONE job (profiling
    # runs several); nothing relies on it surviving the job
    cache = os.environ.get("VF_GRAPH_CACHE")
    cpath = os.path.join(cache, f"graphs_{config}.npz") if cache else None
    if cpath and os.path.exists(cpath):
        z = np.load(cpath)
        go, gi = z["go"], z["gi"]
    else:
        go, gi = graphs.build_graphs(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, device=device)
        if cpath:
            os.makedirs(cache, exist_ok=True)
            np.savez(cpath, go=go, gi=gi)
    log(f"fixture graphs: {int((np.diff(go) > 0).sum())} HS labels, {int(go[-1])} rows ({time.time() - t0:.1f}s)")
    return w, go, gi


def recall_vs(ids, d, gt, gd, k):
    """(strict, tie-aware) recall@k against the exact ground truth (reading #24)."""
    strict, tie = [], []
    for i in range(ids.shape[0]):
        g = gt[i][gt[i] >= 0]
        if g.size == 0:
            continue
        a = ids[i][ids[i] >= 0]
        hits = np.intersect1d(a, g).size
        kth = gd[i][g.size - 1]
        extra = int(np.sum((~np.isin(a, g)) & (d[i][:a.size] == kth)))
        den = min(k, g.size)
        strict.append(hits / den)
        tie.append(min(1.0, (hits + extra) / den))
    return float(np.mean(strict)), float(np.mean(tie))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.samples = []
        self.stop = threading.Event()
        self.gpu = gpu_index
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) == 6:
                    self.samples.append(f)
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for s in self.samples for j in range(4) if s[2 + j].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, config):
    """The oracle, as it stands, on the host cores (the reference arm for this tier)."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the fixture graphs are an input of both arms; they are built with torch on the GPU when one is
    # present (input generation only -- the search below is the oracle alone, on the host cores)
    dev = None
    try:
        import torch
        if torch.cuda.is_available():
            dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    except Exception:
        dev = None
    w, go, gi = make_inputs(config, dev)
    c = w.cfg
    o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    n = len(w.Q) if args.ref_sample < 0 and config != "yfcc" else min(len(w.Q), 5000 if args.ref_sample < 0 else args.ref_sample)
    Q, qo, ql = w.Q[:n], w.q_off[:n + 1], w.q_lab[:w.q_off[n]]
    threads = os.cpu_count() or 1
    # our arm's 0.90 operating point for this workload (profiles/r01_bench_*.json)
    itopk, w_, as_, st_ = OP_POINT[config] if args.ref_itopk <= 0 else (args.ref_itopk, 1, 0, 0)
    op = "and" if c.query_mode in ("and2", "mix_and") else ("or" if c.query_mode == "or2" else "single")
    for _ in range(args.warmup):
        o.search(Q[:64], qo[:65], ql[:qo[64]], k=c.k, itopk=itopk, search_width=w_, op=op, nthreads=threads,
                 and_scan_threshold=as_, scan_threshold=st_)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.search(Q, qo, ql, k=c.k, itopk=itopk, search_width=w_, op=op, nthreads=threads, and_scan_threshold=as_,
                 scan_threshold=st_)
        times.append(time.perf_counter() - t0)
    total = float(np.sum(times))
    qps = n * args.steps / total
    line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{config} (BASELINE.json configs[{CFG_INDEX[config]}])",
                                             "n_queries_per_step": n, "itopk": itopk, "search_width": w_,
                                             "and_scan_threshold": as_, "scan_threshold": st_, "k": c.k, "flush": "n/a (CPU)"},
            "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "oracle",
                             "sample": f"first {n} queries of the {config} batch per step, itopk={itopk}, w={w_}"},
            "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="sift", choices=["tiny", "sift", "yfcc"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--targets", default="0.90,0.99")
    ap.add_argument("--widths", default="1,2,4", help="search widths w swept for the operating points")
    ap.add_argument("--lat-calls", type=int, default=1000, help="timed calls per small-batch latency point")
    ap.add_argument("--and-scan", default=None,
                    help="f3 selectivity-aware AND routing thresholds swept (0 = the paper's method)")
    ap.add_argument("--scan-thr", default=None,
                    help="f2 search-time specificity thresholds T' swept (0 = the build's T; labels with "
                         "|C_l| < max(T, T') are scanned exactly)")
    ap.add_argument("--gt-sample", type=int, default=-1,
                    help="queries whose exact ground truth is computed for recall (-1: all; yfcc: 5000)")
    ap.add_argument("--cpu-sample", type=int, default=2000)
    ap.add_argument("--ref-sample", type=int, default=-1, help="queries per reference step (-1: all; yfcc 5000)")
    ap.add_argument("--ref-itopk", type=int, default=0, help="0: our arm's 0.90 operating point")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="cpu_baseline: repeat the oracle over the sample until this much CPU time")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dump-stats", default=None)
    args = ap.parse_args()

    if args.and_scan is None:
        args.and_scan = "0,2000,50000" if args.config == "yfcc" else "0"
    if args.scan_thr is None:
        args.scan_thr = "0,10000" if args.config == "sift" else "0"
    if args.gt_sample < 0:
        args.gt_sample = 5000 if args.config == "yfcc" else 0
    if args.impl == "reference":
        run_reference(args, args.config)
        return

    import torch
    import torch.distributed as dist
    import paper_2506_00812_b200 as vf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    w, go, gi = make_inputs(args.config, dev, query_stream=rank)
    c = w.cfg
    t0 = time.time()
    if world > 1:
        # label sharding (§8(e)): one rank per GPU, labels partitioned by LPT over |C_l|, items
        # exchanged with NCCL over NVLink inside vf_search
        uid = torch.tensor(list(vf.nccl_unique_id()) if rank == 0 else [0] * 128, dtype=torch.uint8, device=dev)
        dist.broadcast(uid, 0)
        ix = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi, device=local,
                      world_size=world, rank=rank, nccl_unique_id=bytes(uid.cpu().tolist()))
    else:
        ix = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi, device=local)
    info = ix.info()
    log(f"vf_build_index: {info['bytes_total'] / 2**30:.2f} GiB on device ({time.time() - t0:.1f}s)")
    op = "and" if c.query_mode in ("and2", "mix_and") else ("or" if c.query_mode == "or2" else "single")
    n = len(w.Q)
    k = c.k
    stream = torch.cuda.current_stream()
    Q = torch.from_numpy(w.Q).to(dev)
    qo = torch.from_numpy(w.q_off).to(dev)
    ql = torch.from_numpy(w.q_lab).to(dev)
    n_ql = int(w.q_off[-1])            # = len(q_lab): lets vf_search skip reading q_off[n] back
    ids = torch.empty((n, k), dtype=torch.int32, device=dev)
    dd = torch.empty((n, k), dtype=torch.float32, device=dev)

    # -- ground truth: exact mode (T = inf), in query chunks
    t0 = time.time()
    # recall sample: the first m queries of the batch (all of them unless --gt-sample says fewer)
    m_gt = n if args.gt_sample <= 0 else min(n, args.gt_sample)
    gt = np.empty((m_gt, k), np.int32)
    gd = np.empty((m_gt, k), np.float32)
    step = 2000
    for s in range(0, m_gt, step):
        e = min(m_gt, s + step)
        Qs, qos, qls = Q[s:e], qo[s:e + 1] - qo[s], ql[int(w.q_off[s]):int(w.q_off[e])]
        ti = torch.empty((e - s, k), dtype=torch.int32, device=dev)
        td = torch.empty((e - s, k), dtype=torch.float32, device=dev)
        ix.search_into(Qs, qos.contiguous(), qls.contiguous(), ti, td, k=k, op=op, exact=True, stream=stream)
        torch.cuda.synchronize()
        gt[s:e], gd[s:e] = ti.cpu().numpy(), td.cpu().numpy()
    log(f"ground truth (exact mode) for {m_gt} queries: {time.time() - t0:.1f}s")

    # -- (search_width, itopk) sweep -> operating points: for each recall target the fastest
    #    configuration whose mean tie-aware recall@10 reaches it (the paper traces QPS-recall curves
    #    by sweeping its search parameters)
    targets = [float(x) for x in args.targets.split(",")]
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)

    def quick_ms(itopk, w_, as_=0, st_=0):
        ms = []
        for _ in range(3):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ix.search_into(Q, qo, ql, ids, dd, k=k, itopk=itopk, search_width=w_, op=op,
                           and_scan_threshold=as_, stream=stream, n_query_labels=n_ql, scan_threshold=st_)
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return float(np.median(ms))

    sweep = []
    and_scans = [int(x) for x in args.and_scan.split(",")] if op == "and" else [0]
    scan_thrs = [int(x) for x in args.scan_thr.split(",")]
    for as_, st_, w_ in [(a_, t_, b_) for a_ in and_scans for t_ in scan_thrs
                         for b_ in (int(x) for x in args.widths.split(","))]:
        for itopk in ITOPK_GRID:
            if itopk < k:
                continue
            ix.search_into(Q, qo, ql, ids, dd, k=k, itopk=itopk, search_width=w_, op=op,
                           and_scan_threshold=as_, stream=stream, n_query_labels=n_ql, scan_threshold=st_)
            torch.cuda.synchronize()
            r_strict, r_tie = recall_vs(ids[:m_gt].cpu().numpy(), dd[:m_gt].cpu().numpy(), gt, gd, k)
            qms = quick_ms(itopk, w_, as_, st_)
            if world > 1:   # every rank takes the same decisions (the searches are collective)
                t = torch.tensor([r_strict, r_tie, qms], dtype=torch.float64, device=dev)
                dist.all_reduce(t)
                r_strict, r_tie, qms = (float(x) / world for x in t.tolist())
            sweep.append((itopk, r_strict, r_tie, w_, qms, as_, st_))
            log(f"and_scan={as_} scan_thr={st_} w={w_} itopk={itopk:4d} recall@{k} strict={r_strict:.4f} tie-aware={r_tie:.4f} "
                f"{n / qms / 1e3:.2f} MQPS")
            if r_tie >= max(targets):
                break
    ops = {}
    for tgt in targets:
        ok = [s for s in sweep if s[2] >= tgt]
        ops[tgt] = min(ok, key=lambda s: s[4]) if ok else None

    ix.set_profiling(True)
    hbm_peak, peak_kind = measured_peaks()

    def timed(itopk, w_, as_, st_):
        """W warm-up + exactly K timed steps; per-step CUDA events around vf_search only."""
        for _ in range(args.warmup):
            ix.search_into(Q, qo, ql, ids, dd, k=k, itopk=itopk, search_width=w_, op=op,
                           and_scan_threshold=as_, stream=stream, n_query_labels=n_ql, scan_threshold=st_)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        stats = []
        barrier()
        torch.cuda.synchronize()
        ix.set_profiling(True)          # phase means are taken over the K timed steps only
        torch.cuda.nvtx.range_push("timed")   # ncu --nvtx --nvtx-include timed/ captures these launches
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            ix.search_into(Q, qo, ql, ids, dd, k=k, itopk=itopk, search_width=w_, op=op,
                           and_scan_threshold=as_, stream=stream, n_query_labels=n_ql, scan_threshold=st_)
            ev[i][1].record(stream)
        # no host sync inside the loop: the host enqueues step i+1 while the device runs step i,
        # so the events time the device work (host-side cost is what `e2e` measures)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        stats.append(ix.last_stats(stream))       # work counters of the last step + phase means of all K
        barrier()
        ms = [a.elapsed_time(b) for a, b in ev]
        return ms, stats

    results = {}
    with ClockSampler(local) as clk:
        for tgt, opnt in ops.items():
            if opnt is None:
                continue
            itopk, w_, as_, st_ = opnt[0], opnt[3], opnt[5], opnt[6]
            ms, stats = timed(itopk, w_, as_, st_)
            tot = float(np.sum(ms))
            if world > 1:
                t = torch.tensor([tot], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                tot = float(t.item())
            results[tgt] = (itopk, opnt, ms, stats, tot)
    clocks = clk.summary()

    # -- end to end through the C-ABI with host (pinned) buffers, copies inside the timed region
    main_tgt = targets[0]
    e2e = None
    if main_tgt in results:
        itopk, w_, as_, st_ = results[main_tgt][0], results[main_tgt][1][3], results[main_tgt][1][5], results[main_tgt][1][6]
        Qh = torch.from_numpy(w.Q).pin_memory()
        qoh = torch.from_numpy(w.q_off).pin_memory()
        qlh = torch.from_numpy(w.q_lab).pin_memory()
        oih = torch.empty((n, k), dtype=torch.int32).pin_memory()
        odh = torch.empty((n, k), dtype=torch.float32).pin_memory()
        for _ in range(args.warmup):
            ix.search_into(Qh, qoh, qlh, oih, odh, k=k, itopk=itopk, search_width=w_, op=op,
                           and_scan_threshold=as_, stream=stream, n_query_labels=n_ql, scan_threshold=st_)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            ix.search_into(Qh, qoh, qlh, oih, odh, k=k, itopk=itopk, search_width=w_, op=op,
                           and_scan_threshold=as_, stream=stream, n_query_labels=n_ql, scan_threshold=st_)
        e1.record(stream)
        torch.cuda.synchronize()
        et = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([et], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        h2d = Qh.numel() * Qh.element_size() + qoh.numel() * 8 + qlh.numel() * 4
        d2h = n * k * 8
        e2e = {"value": n * world * args.steps / (et / 1000.0), "unit": "queries/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # -- small-batch latency (BASELINE.json configs[3]): batch 1 / 10 / 100 at the 0.90 operating
    #    point; end to end through the C-ABI with pinned host buffers (H2D, launches, D2H inside) and
    #    with device-resident buffers; wall clock per blocking call, p50 / p99 over many calls
    latency = None
    if main_tgt in results and world == 1 and args.lat_calls > 0:
        itopk, w_, as_, st_ = results[main_tgt][0], results[main_tgt][1][3], results[main_tgt][1][5], results[main_tgt][1][6]
        latency = {}
        for bsz in (1, 10, 100):
            Qh = torch.from_numpy(w.Q[:bsz].copy()).pin_memory()
            qoh = torch.from_numpy(w.q_off[:bsz + 1].copy()).pin_memory()
            qlh = torch.from_numpy(w.q_lab[:w.q_off[bsz]].copy()).pin_memory()
            oih = torch.empty((bsz, k), dtype=torch.int32).pin_memory()
            odh = torch.empty((bsz, k), dtype=torch.float32).pin_memory()
            Qd, qod, qld = Qh.to(dev), qoh.to(dev), qlh.to(dev)
            oid = torch.empty((bsz, k), dtype=torch.int32, device=dev)
            odd = torch.empty((bsz, k), dtype=torch.float32, device=dev)
            res = {}
            for mode in ("host", "device"):
                ts = []
                for it_ in range(args.lat_calls + 50):
                    t0 = time.perf_counter()
                    if mode == "host":
                        ix.search_into(Qh, qoh, qlh, oih, odh, k=k, itopk=itopk, search_width=w_, op=op,
                                       and_scan_threshold=as_, stream=stream, scan_threshold=st_)
                    else:
                        ix.search_into(Qd, qod, qld, oid, odd, k=k, itopk=itopk, search_width=w_, op=op,
                                       and_scan_threshold=as_, stream=stream, n_query_labels=int(w.q_off[bsz]),
                                       scan_threshold=st_)
                        stream.synchronize()
                    if it_ >= 50:
                        ts.append(time.perf_counter() - t0)
                res[mode] = {"p50_ms": 1e3 * float(np.percentile(ts, 50)),
                             "p99_ms": 1e3 * float(np.percentile(ts, 99))}
            latency[f"batch{bsz}"] = res
        # f1: the persistent serving kernel (vf_serve_*) -- single-query latency (one job
        # in flight, host query in, host result out) and single-batch-mode throughput (every query
        # its own job, up to 1024 in flight), the two E13 measurements
        try:
            labs = [np.ascontiguousarray(w.q_lab[w.q_off[i]:w.q_off[i + 1]]) for i in range(min(n, 20000))]
            Qn = np.ascontiguousarray(w.Q)
            with ix.serve(k=k, itopk=itopk, search_width=w_, op=op, and_scan_threshold=as_, scan_threshold=st_,
                          capacity=4096) as sv:
                oi_, od_ = np.empty(k, np.int32), np.empty(k, np.float32)
                ts = []
                for it_ in range(args.lat_calls + 50):
                    i = it_ % len(labs)
                    t0 = time.perf_counter()
                    sv.wait(sv.submit(Qn[i], labs[i]), oi_, od_)
                    if it_ >= 50:
                        ts.append(time.perf_counter() - t0)
                # the whole batch, each query its own job, from a C client loop (vf_serve_run)
                sv.run(Qn[:1024], w.q_off[:1025], w.q_lab[:w.q_off[1024]], max_in_flight=1024)
                m_q = n
                t0 = time.perf_counter()
                sv.run(Qn, w.q_off, w.q_lab, max_in_flight=1024)
                el = time.perf_counter() - t0
                latency["serve"] = {"device_means_us": sv.stats(),
                                    "p50_ms": 1e3 * float(np.percentile(ts, 50)),
                                    "p99_ms": 1e3 * float(np.percentile(ts, 99)),
                                    "single_batch_qps": m_q / el, "in_flight": 1024,
                                    "workers": sv.info()["n_workers"]}
        except Exception as e:   # reported, not fatal: the batched numbers stand on their own
            latency["serve"] = {"error": str(e)}
        log(f"latency: {latency}")

    # -- CPU baseline: the oracle on this host's cores, bounded sample, rank 0 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and main_tgt in results:
        import oracle
        itopk, w_, as_, st_ = results[main_tgt][0], results[main_tgt][1][3], results[main_tgt][1][5], results[main_tgt][1][6]
        o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
        m = min(n, args.cpu_sample)
        threads = os.cpu_count() or 1
        passes, el = 0, 0.0
        while el < args.cpu_seconds and passes < 1000:
            t0 = time.perf_counter()
            o.search(w.Q[:m], w.q_off[:m + 1], w.q_lab[:w.q_off[m]], k=k, itopk=itopk, search_width=w_, op=op,
                     nthreads=threads, and_scan_threshold=as_, scan_threshold=st_)
            el += time.perf_counter() - t0
            passes += 1
        cpu = {"value": m * passes / el, "unit": "queries/s", "cores": threads, "kind": "oracle",
               "sample": f"first {m} of the {n} queries x {passes} passes, itopk={itopk}, w={w_}, "
                         f"{threads} threads, {el:.1f}s"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    if main_tgt not in results:
        print(json.dumps({"metric": METRIC, "value": None, "error": "recall target not reached",
                          "sweep": sweep}), flush=True)
        return
    itopk, opnt, ms, stats, tot = results[main_tgt]
    K = args.steps
    qps = n * world * K / (tot / 1000.0)
    # roofline of the dominant kernel (graph beam search): algorithmic bytes / kernel time
    s0 = stats[-1]
    rb = s0["row_bytes"]
    R = c.degree_R
    # per graph item V vector rows + E adjacency rows of R (local, global) int32 pairs;
    # per scan tile row: the X_LS row + its global id
    g_bytes = s0["graph_V"] * rb + s0["graph_E"] * R * 8
    g_ms = s0["mean_ms_graph"]
    s_bytes = s0["scan_rows"] * (rb + 4)
    s_ms = s0["mean_ms_scan"]
    # dominant kernel: the longer device-clock span (the phase events overlap when scan and graph
    # run concurrently); phase times if the spans are unavailable
    ga, sa = s0.get("ms_graph_active", 0.0), s0.get("ms_scan_active", 0.0)
    dom = ("graph" if ga >= sa else "scan") if (ga > 0 or sa > 0) else ("graph" if g_ms >= s_ms else "scan")
    bytes_dom, ms_dom = (g_bytes, g_ms) if dom == "graph" else (s_bytes, s_ms)
    achieved = bytes_dom / (ms_dom / 1000.0) / 1e9 if ms_dom > 0 else 0.0
    # measured DRAM traffic of that kernel at this operating point, from a committed ncu capture
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f).get(args.config)
        if tj and f"k_{dom}" in tj and (tj["itopk"], tj["search_width"], tj["and_scan_threshold"],
                                        tj["scan_threshold"]) == (itopk, opnt[3], opnt[5], opnt[6]):
            traffic = int(tj[f"k_{dom}"]["bytes"])
    except (OSError, ValueError, KeyError):
        traffic = None
    # the dominant kernel's own device-clock span in the last timed step (first CTA start -> last
    # CTA end): in an overlapped step the phase events above also count time the launched kernel
    # waited for SMs held by the other phase
    act_ms = s0["ms_graph_active"] if dom == "graph" else s0["ms_scan_active"]
    act_gbs = bytes_dom / (act_ms / 1000.0) / 1e9 if act_ms > 0 else None
    line = {
        "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": tot / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8" if (c.dtype == "u8" or info["bytes_u8_store"] > 0) else "f32",
        "data": "synthetic",
        "config": {"workload": f"{args.config} (BASELINE.json configs[{CFG_INDEX[args.config]}])",
                   "n_points": c.n_points, "dim": c.dim, "n_labels": c.n_labels,
                   "queries_per_step": n, "query_mode": c.query_mode, "k": k, "T": c.threshold_T,
                   "R": R, "itopk": itopk, "search_width": opnt[3], "and_scan_threshold": opnt[5],
                   "scan_threshold": opnt[6],
                   "recall_target": main_tgt,
                   "recall": {"strict": opnt[1], "tie_aware": opnt[2]},
                   "recall_sample": f"first {m_gt} queries (exact-mode ground truth)",
                   "flush": "256 MiB L2 flush before every timed step (outside the step events)",
                   "parallelism": f"label-shard{world}" if world > 1 else "single",
                   "queries": "per rank (weak scaling)" if world > 1 else "batch",
                   "storage": ("u8 rows (lossless store of integer-valued fp32 in [0,255]; fp32 rows kept "
                               "for out-of-range query batches)") if (c.dtype != "u8" and info["bytes_u8_store"] > 0)
                              else c.dtype},
        "at_recall": {f"{t:.2f}": {"itopk": r[0], "search_width": r[1][3], "and_scan_threshold": r[1][5], "scan_threshold": r[1][6], "qps": n * world * K / (r[4] / 1000.0),
                                   "ms_per_step": r[4] / K, "recall_strict": r[1][1],
                                   "recall_tie_aware": r[1][2]} for t, r in results.items()},
        "sweep": [{"and_scan_threshold": s[5], "scan_threshold": s[6], "search_width": s[3], "itopk": s[0], "recall_strict": s[1], "recall_tie_aware": s[2],
                   "ms": s[4]} for s in sweep],
        "roofline": {"kernel": f"k_{dom}", "bound": "hbm", "achieved": achieved, "peak": hbm_peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm_peak,
                     "traffic": traffic, "traffic_source": "profiles/traffic.json (ncu --set full)" if traffic else None,
                     "algorithmic_bytes_per_launch": int(bytes_dom),
                     "kernel_ms_per_launch": ms_dom,
                     "kernel_active_ms": act_ms, "achieved_active": act_gbs,
                     "frac_active": act_gbs / hbm_peak if act_gbs else None,
                     "note": ("kernel_ms_per_launch: CUDA events of the kernel's phase on its stream, mean of the K "
                              "timed steps (scan and graph overlap, so it includes waiting for SMs); "
                              "kernel_active_ms: %globaltimer span of the kernel's CTAs in the last step")},
        "phases_ms": {**{p: s0[f"mean_ms_{p}"] for p in ("route", "scan", "graph", "merge", "copy", "total")},
                      "steps_averaged": s0["n_profiled"]},
        "work": {kk: s0[kk] for kk in ("n_items", "n_scan_items", "n_graph_items", "n_segments",
                                       "scan_rows", "graph_V", "graph_E", "graph_iterations", "graph_V_max")},
        "gpu_launches": int(s0["kernel_launches"] * K),
        "latency": latency,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "index_bytes": info["bytes_total"],
    }
    if args.dump_stats:
        with open(args.dump_stats, "w") as f:
            json.dump({"stats": stats, "ms": ms}, f)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
