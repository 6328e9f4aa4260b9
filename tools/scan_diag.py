"""Grouped-scan diagnostics: stage times of one config with the kernel's
experiment switches (RABITQ_IMMA_EXPERIMENT: 1 skip epilogue math, 2 skip
UMMAs, 3 both), each over `reps` searches (diagnostics only)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_16007_b200 as rq  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
exps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,3").split(",")]
s = synth.spec(cfg)
dev = torch.device("cuda", 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=synth.init_centroids(s, dev))
st = torch.cuda.Stream(dev)
for ex in exps:
    os.environ["RABITQ_IMMA_EXPERIMENT"] = str(ex)
    for rep in range(3):
        prof = rq.Profile()
        idx.search(Q, s.k, s.nprobe, s.M, stream=st, profile=prof)
        torch.cuda.synchronize()
    pd = prof.as_dict()
    print(json.dumps({"cfg": cfg, "experiment": ex, "stage_ms": {k: round(v, 3) for k, v in pd["stage_ms"].items()}}),
          flush=True)
