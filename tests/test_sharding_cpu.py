"""Label-sharding host logic (§8(e)) without a GPU: the LPT ownership is deterministic, balanced,
and identical across processes (world_size-2 gloo group)."""
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
