import sys, time, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2605_16007_b200 as rq, synth
s = synth.spec(3)
dev = torch.device('cuda', 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=synth.init_centroids(s, dev))
Qh = Q.cpu().pin_memory()
ih = torch.empty(s.nq, s.k, dtype=torch.int64).pin_memory()
dh = torch.empty(s.nq, s.k, dtype=torch.float32).pin_memory()
for rep in range(4):
    prof = rq.Profile()
    t0 = time.perf_counter()
    idx.search(Qh, s.k, s.nprobe, s.M, out=(ih, dh), profile=prof)
    t1 = time.perf_counter()
    d = prof.as_dict()
    print(rep, round((t1 - t0) * 1e3, 2), {k: round(v, 3) for k, v in d['stage_ms'].items()}, d['retries'], d['batches'], flush=True)
for rep in range(2):
    prof = rq.Profile()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    idx.search(Q, s.k, s.nprobe, s.M, profile=prof)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    d = prof.as_dict()
    print('dev', rep, round((t1 - t0) * 1e3, 2), {k: round(v, 3) for k, v in d['stage_ms'].items()}, flush=True)
