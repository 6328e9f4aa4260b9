"""Threshold-seeding diagnostics (not a test): per-query tau vs the exact M-th
key (the final top-M), survivors distribution, for the near-list seed and the
uniform-prefix seed (VARIANT_UNIFORM_SEED)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_16007_b200 as rq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--nq", type=int, default=0)
ap.add_argument("--variants", default="[0, 16]")
args = ap.parse_args()
ov = {"nq": args.nq} if args.nq else {}
s = synth.spec(args.config, **ov)
dev = torch.device("cuda", 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=synth.init_centroids(s, dev))
nq, M = Q.shape[0], s.M
for var in json.loads(args.variants):
    dbg = dict(tau=torch.empty(nq, device=dev), survivors=torch.empty(nq, dtype=torch.int32, device=dev),
               retries=torch.zeros(1, dtype=torch.int32, device=dev),
               topm_est=torch.empty(nq, M, device=dev), probes=torch.empty(nq, s.nprobe, dtype=torch.int32, device=dev))
    ids, d = idx.search(Q, s.k, s.nprobe, M, debug=dbg, variant=var)
    torch.cuda.synchronize()
    tau = dbg["tau"].cpu().numpy()
    sv = dbg["survivors"].cpu().numpy()
    mth = dbg["topm_est"].cpu().numpy()[:, M - 1]
    under = np.nonzero(tau < mth)[0]
    print(json.dumps({"variant": var, "retries": int(dbg["retries"].item()), "surv_mean": float(sv.mean()),
                      "surv_pct": [int(np.percentile(sv, p)) for p in (0, 1, 10, 50, 90, 99, 100)],
                      "under_q": int(under.size), "under_first": under[:10].tolist(),
                      "tau_over_mth_pct": [float(np.percentile(tau / mth, p)) for p in (0, 1, 50, 99)]}), flush=True)
    top = np.argsort(-sv)[:6]
    lo = None
    for q in top:
        pr = dbg["probes"][q].cpu().numpy()
        if lo is None:
            lo = idx.export()["list_off"] if args.config <= 3 else None
        sz = (np.diff(lo)[pr].tolist() if lo is not None else [])
        print("  top-surv q", int(q), "surv", int(sv[q]), "tau", float(tau[q]), "Mth", float(mth[q]),
              "sizes", sz[:12], "P", int(sum(sz)) if sz else None, flush=True)
    if under.size:
        ex = idx.export() if var == 0 and args.config <= 3 else None
        lo = idx.info()
        for q in under[:5]:
            pr = dbg["probes"][q, :8].cpu().numpy()
            print("  q", int(q), "tau", float(tau[q]), "Mth", float(mth[q]), "surv", int(sv[q]), "probes", pr.tolist(), flush=True)
