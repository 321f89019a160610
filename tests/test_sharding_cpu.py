"""Label-sharding host logic (§8(e)) without a GPU: the LPT ownership is deterministic, balanced,
and identical across processes (world_size-2 gloo group), and the sharded protocol (items to label
owners, answers back, merge at the origin) equals the unsharded search."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


@pytest.fixture(scope="module")
def vf():
    from paper_2506_00812_b200 import build as B
    B.build()
    import paper_2506_00812_b200 as vf
    return vf


def _lpt_reference(sizes, world):
    """Independent restatement of the rule in include/vf.h (greedy LPT, stable ties)."""
    order = sorted(range(len(sizes)), key=lambda l: (-sizes[l], l))
    load = [0] * world
    owner = [0] * len(sizes)
    for l in order:
        r = min(range(world), key=lambda r: (load[r], r))
        owner[l] = r
        load[r] += sizes[l]
    return owner, load


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_matches_rule_and_is_balanced(vf, world):
    from workload import gen
    cfg = gen.config("sift")
    off, _ = gen.gen_postings(cfg)
    sizes = np.diff(off)
    owner = vf.partition_labels(sizes, world)
    ref, load = _lpt_reference(sizes.tolist(), world)
    assert owner.tolist() == ref
    got = np.bincount(owner, weights=sizes, minlength=world)
    assert (got == np.array(load)).all()
    # LPT bound: no rank exceeds the average by more than the largest label
    assert got.max() <= sizes.sum() / world + sizes.max()


def _worker(rank, world, port, sizes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import paper_2506_00812_b200 as vf
    owner = torch.from_numpy(vf.partition_labels(sizes, world).astype(np.int64))
    gathered = [torch.empty_like(owner) for _ in range(world)]
    dist.all_gather(gathered, owner)
    same = all((g == gathered[0]).all().item() for g in gathered)
    # every label owned by exactly one rank; each rank can compute its own share locally
    mine = int((owner == rank).sum())
    tot = torch.tensor([mine])
    dist.all_reduce(tot)
    q.put((rank, same, int(tot.item())))
    dist.destroy_process_group()


def test_partition_identical_across_gloo_ranks(vf):
    from workload import gen
    off, _ = gen.gen_postings(gen.config("tiny"))
    sizes = np.diff(off)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sizes, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(same for _, same, _ in res)
    assert all(tot == len(sizes) for _, _, tot in res)


def _exchange_worker(rank, world, port, q):
    """One rank of the label-sharded protocol (§8(e)) over gloo, with the oracle as each rank's
    search engine: this rank's queries are routed (oracle route), every item is sent to the owner
    of its label (LPT ownership from the library), owners answer their items, results return to the
    origin and are merged (Alg. 2). The GPU path does the same exchange with NCCL inside
    vf_search (tested over its loopback transport in tests/test_gpu_parity.py)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2506_00812_b200 as vf
    from workload import gen, graphs
    w = gen.make_workload("tiny", n_queries=240)
    c = w.cfg
    go, gi = graphs.build_graphs(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R)
    o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    owner = vf.partition_labels(np.diff(w.post_off), world)
    ok = True
    for mode, op in (("or2", "or"), ("and2", "and")):
        qoff, qlab = gen.gen_query_labels(c, w.post_off, w.post_ids, n=240, mode=mode)
        mine = [i for i in range(240) if i % world == rank]
        items, _ = o.route(qoff, qlab, op=op)            # (query, label, path, ...) per item
        out = [[] for _ in range(world)]
        for it in items:
            qi, lab = int(it[0]), int(it[1])
            if qi % world == rank:
                out[owner[lab]].append((qi, lab))
        gathered = [None] * world                        # gloo: the item exchange as objects
        dist.all_gather_object(gathered, out)
        inbox = [gathered[src][rank] for src in range(world)]
        answers = [[] for _ in range(world)]
        for src in range(world):
            for qi, lab in inbox[src]:
                assert owner[lab] == rank
                labs = np.array([lab], np.int32) if op == "or" else qlab[qoff[qi]:qoff[qi + 1]]
                ids, d = o.search(w.Q[qi:qi + 1], np.array([0, len(labs)], np.int64), labs, k=10, itopk=32,
                                  op="single" if op == "or" else "and")
                answers[src].append((qi, ids[0].tolist(), d[0].tolist()))
        back = [None] * world
        dist.all_gather_object(back, answers)
        per_q = {}
        for r in range(world):
            for qi, ids, d in back[r][rank]:
                per_q.setdefault(qi, []).append((ids, d))
        ref_i, ref_d = o.search(w.Q, qoff, qlab, k=10, itopk=32, op=op)
        for qi in mine:
            lists = per_q.get(qi, [])
            if not lists:
                ok &= bool((ref_i[qi] == -1).all())
                continue
            mi, md = oracle.merge([x[0] for x in lists], [x[1] for x in lists], 10)
            ok &= bool((mi == ref_i[qi]).all() and (md == ref_d[qi]).all())
    q.put((rank, ok))
    dist.destroy_process_group()


def test_sharded_protocol_over_gloo_equals_unsharded(vf):
    """world_size-2 gloo: route -> items to label owners -> owners answer -> origin merges equals
    the unsharded search for OR and AND queries."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
