"""Work statistics of the grouped scan for one config (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_16007_b200 as rq  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = synth.spec(cfg)
dev = torch.device("cuda", 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=synth.init_centroids(s, dev))
pr = torch.empty(s.nq, s.nprobe, dtype=torch.int32, device=dev)
idx.search(Q, s.k, s.nprobe, s.M, debug=dict(probes=pr))
ex = idx.export()
L = np.diff(ex["list_off"])
G = np.bincount(pr.cpu().numpy().ravel(), minlength=s.nlist)
Dp = 32 * s.W
nch = (Dp + 127) // 128
NG = min(256, (128 * 1024 // (nch * 128)) // 32 * 32)
tiles = np.ceil(L / 128)
ngr = np.ceil(G / NG)
items = np.ceil(tiles / 8) * ngr
tile_work = tiles * ngr  # (tile, group) accumulators
cols16 = np.where(G > 0, (np.minimum(G, NG) + 15) // 16 * 16, 0)
pairs = (L * G).sum()
mma_pairs = 0
for j in range(s.nlist):
    if G[j] == 0:
        continue
    full = G[j] // NG
    rem = G[j] % NG
    cols = full * NG + ((rem + 15) // 16 * 16 if rem else 0)
    mma_pairs += tiles[j] * 128 * cols
print(f"CFG{cfg}: D={s.D} NG={NG} nchunks={nch} lists probed={int((G>0).sum())}/{s.nlist}")
print(f" pairs={pairs:.3e} items={items.sum():.0f} tiles(acc)={tile_work.sum():.0f} chunks={tile_work.sum()*nch:.0f}")
print(f" MMA pairs incl. padding={mma_pairs:.3e} efficiency={pairs/mma_pairs:.3f}")
print(f" avg cols per (tile,group)={pairs/ (tile_work.sum()*128):.1f}  L mean={L.mean():.0f} max={L.max()}  G mean={G.mean():.0f} max={G.max()}")
w = L * G
o = np.argsort(-w)
print(" top lists by work: ", [(int(L[j]), int(G[j])) for j in o[:10]])
print(f" share of work in top 1%% lists: {w[o[:max(1,s.nlist//100)]].sum()/w.sum():.3f}")
