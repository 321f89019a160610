import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench, paper_2506_00812_b200 as vf
w, go, gi = bench.make_inputs("sift", torch.device("cuda", 0))
c = w.cfg
ix = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
print("info u8store", ix.info()["bytes_u8_store"])
gt, gd = ix.search(w.Q, w.q_off, w.q_lab, k=10, exact=True)
print("exact stats", ix.last_stats())
for it in (16, 64):
    a, ad = ix.search(w.Q, w.q_off, w.q_lab, k=10, itopk=it, search_width=2)
    st = ix.last_stats()
    rec = np.mean([np.intersect1d(a[i], gt[i]).size / 10 for i in range(len(a))])
    print("itopk", it, "recall", rec, "row_bytes", st["row_bytes"], "ms", st["ms_total"])
import oracle
o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
m = 300
e, ed = o.exact_knn(w.Q[:m], w.q_off[:m+1], w.q_lab[:w.q_off[m]], k=10)
print("exact-mode vs oracle Def1 (first 300):", (gt[:m] == e).mean(), (gd[:m] == ed.astype(np.float32)).mean())
