"""Distribution of the grouped scan's work at a config: for every probed list
the number of (query, list) pairs G_j and tiles T_j, weighted by pairs
scanned (which unit widths and item sizes the small-K scan sees)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16007_b200 as rq  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = synth.spec(cfg)
dev = torch.device("cuda", 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=synth.init_centroids(s, dev))
probes = torch.empty(s.nq, s.nprobe, dtype=torch.int32, device=dev)
idx.search(Q, s.k, s.nprobe, s.M, debug=dict(probes=probes))
off = idx.export()["list_off"] if s.N <= 10_000_000 else None
info = idx.info()
L = None
if off is None:
    # list sizes without a full export: count assignments via a probe-only export is not exposed;
    # use the probe histogram and the index's list offsets through export of list_off only
    from paper_2605_16007_b200 import Export, lib
    import ctypes
    lo = np.empty(s.nlist + 1, np.int64)
    e = Export(list_off=lo.ctypes.data)
    lib().rabitq_index_export(idx._h, ctypes.byref(e))
    off = lo
L = np.diff(off)
G = np.bincount(probes.cpu().numpy().ravel(), minlength=s.nlist)
T = (L + 127) // 128
pairs = (G * L).astype(np.float64)
print(f"CFG{cfg}: pairs {pairs.sum():.3e}, lists probed {np.count_nonzero(G)}, mean G {G[G>0].mean():.1f}")
w = pairs / pairs.sum()
for lo_, hi_ in [(1, 16), (17, 32), (33, 64), (65, 128), (129, 256), (257, 512), (513, 1 << 30)]:
    m = (G >= lo_) & (G <= hi_)
    print(f"G in [{lo_},{hi_}]: {m.sum():6d} lists, {100 * w[m].sum():5.1f} % of pairs")
units = sum(int(t) * int((g + 63) // 64) for g, t in zip(G, T) if g > 0)
print(f"tiles x 64-col units {units}, pairs per unit {pairs.sum() / units:.0f} (full unit 8192)")
