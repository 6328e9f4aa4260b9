import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2605_16007_b200 as rq, synth
s = synth.spec(2, nq=500)
dev = torch.device('cuda', 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True)
i1, d1 = idx.search(Q, s.k, s.nprobe, s.M)
os.environ['RABITQ_DENSE_RERANK'] = '0'
i0, d0 = idx.search(Q, s.k, s.nprobe, s.M)
i1, d1, i0, d0 = [t.cpu().numpy() for t in (i1, d1, i0, d0)]
# exact fp64 for returned ids
Xc = X.double(); Qc = Q.double()
rel = []
for q in range(50):
    ex = ((Xc[torch.from_numpy(i1[q]).to(dev)] - Qc[q]) ** 2).sum(1).cpu().numpy()
    rel.append(np.max(np.abs(d1[q] - ex) / ex))
    ex0 = ((Xc[torch.from_numpy(i0[q]).to(dev)] - Qc[q]) ** 2).sum(1).cpu().numpy()
    rel.append(-np.max(np.abs(d0[q] - ex0) / ex0))
rel = np.array(rel)
print('dense max rel err', rel[0::2].max(), 'gather max rel err', -rel[1::2].min(), 'same ids', np.mean(i1 == i0))
