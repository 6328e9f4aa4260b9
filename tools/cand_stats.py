"""Where do the top-M re-rank candidates live? Fraction of each query's top-M
in its r-th nearest probed list (diagnostics for the re-rank design)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_16007_b200 as rq  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
s = synth.spec(cfg)
dev = torch.device("cuda", 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)[:nq].contiguous()
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=synth.init_centroids(s, dev))
pr = torch.empty(nq, s.nprobe, dtype=torch.int32, device=dev)
tid = torch.empty(nq, s.M, dtype=torch.int64, device=dev)
tes = torch.empty(nq, s.M, dtype=torch.float32, device=dev)
ids, d = idx.search(Q, s.k, s.nprobe, s.M, debug=dict(probes=pr, topm_ids=tid, topm_est=tes))
torch.cuda.synchronize()
ex = idx.export()
lst = np.empty(s.N, dtype=np.int64)
off = ex["list_off"]
for j in range(s.nlist):
    lst[ex["ids"][off[j]:off[j + 1]]] = j
pr = pr.cpu().numpy()
tid = tid.cpu().numpy()
fr = np.zeros(s.nprobe)
for q in range(nq):
    ok = tid[q] >= 0
    l = lst[tid[q][ok]]
    rank = {int(j): r for r, j in enumerate(pr[q])}
    for j in l:
        fr[rank[int(j)]] += 1
fr /= fr.sum()
print(f"CFG{cfg}: share of top-M candidates by probe rank:", np.round(fr[:8], 3), "cum4", round(fr[:4].sum(), 3))

# dense-tile economics: per nearest list j, queries G_j, list size L_j, candidates
# of those queries inside j (sum) and their union
j0 = pr[:, 0]
sizes = np.diff(off)
tot_c = sum(int((tid[q] >= 0).sum()) for q in range(nq))
rows_dense, pairs_sum, pairs_union, pairs_full = 0, 0, 0, 0
for j in np.unique(j0):
    qs = np.where(j0 == j)[0]
    cj = [set(tid[q][(tid[q] >= 0) & (lst[np.maximum(tid[q], 0)] == j)].tolist()) for q in qs]
    u = set().union(*cj)
    pairs_sum += sum(len(c) for c in cj)
    pairs_union += len(qs) * len(u)
    pairs_full += len(qs) * int(sizes[j])
for thr in (1, 2, 4):
    elig = sizes[j0] <= thr * s.M
    print(f"  queries with nearest list <= {thr}M: {elig.mean():.3f}")
print(f"  candidates in nearest list: {pairs_sum / tot_c:.3f}; dense pairs / needed: union {pairs_union / pairs_sum:.2f}, full list {pairs_full / pairs_sum:.2f}")
