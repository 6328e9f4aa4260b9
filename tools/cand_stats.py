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
