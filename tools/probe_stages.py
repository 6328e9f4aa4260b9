"""Stage-time probe for one config: builds the index once, runs the search with
several option sets and prints rabitq_profile per run (diagnostics only)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_16007_b200 as rq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--nq", type=int, default=0)
ap.add_argument("--N", type=int, default=0, help="override the base size (probe/quantize stages do not depend on it)")
ap.add_argument("--runs", default='[{}]', help="JSON list of search kwargs")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--profile-last", action="store_true", help="cudaProfilerStart/Stop around the last rep (ncu --profile-from-start off)")
args = ap.parse_args()
ov = {}
if args.nq:
    ov["nq"] = args.nq
if args.N:
    ov["N"] = args.N
s = synth.spec(args.config, **ov)
dev = torch.device("cuda", 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)
t0 = time.time()
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=synth.init_centroids(s, dev))
torch.cuda.synchronize()
print("build_s", round(time.time() - t0, 2), idx.info(), flush=True)
st = torch.cuda.Stream(dev)
for kw in json.loads(args.runs):
    for rep in range(args.reps):
        last = args.profile_last and rep == args.reps - 1
        if last:
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
        prof = rq.Profile()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ids, d = idx.search(Q, s.k, kw.pop("nprobe", s.nprobe) if False else s.nprobe, s.M, stream=st, profile=prof, **kw)
        e1.record(st)
        torch.cuda.synchronize()
        if last:
            torch.cuda.cudart().cudaProfilerStop()
        pd = prof.as_dict()
        pd["stage_ms"] = {k: round(v, 3) for k, v in pd["stage_ms"].items()}
        print(json.dumps({"kw": kw, "rep": rep, "ms": round(e0.elapsed_time(e1), 3), **pd}), flush=True)
