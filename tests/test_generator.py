"""Generator pins: the Zipf label recipe reproduces the statistics the paper prints."""
import numpy as np

from workload import gen


def test_zipf_least_specific_sift_cluster_P_L622():
    """SIFT-1M with 50 Zipf labels and F = 3.17: 'the least specific label cluster contains 14,000
    data points'. With s = 1 the expectation is N c / 50 = 14,091."""
    p = gen.zipf_probabilities(50, 3.17)
    assert abs(1_000_000 * p[-1] - 14_091) < 1
    cfg = gen.config("sift", n_labels=50)
    off, ids = gen.gen_postings(cfg)
    sizes = np.diff(off)
    assert abs(sizes.min() - 14_000) < 700
    assert abs(sizes.sum() / cfg.n_points - 3.17) < 0.01        # mean labels per point (L586)


def test_zipf_mean_labels_and_inversion_roundtrip():
    cfg = gen.config("tiny")
    off, ids = gen.gen_postings(cfg)
    assert abs(np.diff(off).sum() / cfg.n_points - 3.17) < 0.05
    for l in range(cfg.n_labels):                                    # ascending, unique
        a = ids[off[l]:off[l + 1]]
        assert (np.diff(a) > 0).all() and (a >= 0).all() and (a < cfg.n_points).all()
    poff, plab = gen.point_labels(cfg.n_points, off, ids)
    assert plab.size == ids.size                                     # sum |C_l| = sum |L_i|
    back = [[] for _ in range(cfg.n_labels)]
    for i in range(cfg.n_points):
        for l in plab[poff[i]:poff[i + 1]]:
            back[l].append(i)
    for l in range(cfg.n_labels):
        assert back[l] == ids[off[l]:off[l + 1]].tolist()


def test_deterministic_and_variants():
    a = gen.make_workload("tiny")
    b = gen.make_workload("tiny")
    assert (a.X == b.X).all() and (a.q_lab == b.q_lab).all() and (a.Q == b.Q).all()
    u8 = gen.gen_vectors(gen.config("tiny", dtype="u8"))
    assert u8.dtype == np.uint8 and (u8.astype(np.float32) == a.X).all()
    fl = gen.gen_vectors(gen.config("tiny", dtype="f32float"))
    inside = (a.X > 0) & (a.X < 255)                                # unclamped values round
    assert fl.dtype == np.float32 and np.abs(fl * 255 - a.X)[inside].max() <= 0.5 + 1e-4


def test_query_labels_frequency_weighted_and_and2_nonempty():
    cfg = gen.config("tiny")
    off, ids = gen.gen_postings(cfg)
    qoff, qlab = gen.gen_query_labels(cfg, off, ids, n=2000, mode="and2")
    assert (np.diff(qoff) == 2).all()
    poff, plab = gen.point_labels(cfg.n_points, off, ids)
    sets = [set(plab[poff[i]:poff[i + 1]].tolist()) for i in range(cfg.n_points)]
    for i in range(0, 2000, 50):
        a, b = qlab[qoff[i]:qoff[i + 1]]
        assert a != b and any({a, b} <= s for s in sets)             # |AND set| >= 1
