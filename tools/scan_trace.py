"""Clock trace of the grouped scan's CTA 0 (diagnostics): runs one config's
search with RABITQ_SCAN_TRACE set and writes [16384][16] int64 clock64 stamps
per experiment to <out>_e<k>.bin (see scan_imma.cu RQ_TR for the slots)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_16007_b200 as rq  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace"
exps = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0").split(",")]
s = synth.spec(cfg)
dev = torch.device("cuda", 0)
cen = synth.centres(s, dev)
X = synth.base_rows(s, 0, s.N, dev, cen=cen)
Q = synth.queries(s, dev, cen=cen)
idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=synth.init_centroids(s, dev))
for ex in exps:
    os.environ["RABITQ_IMMA_EXPERIMENT"] = str(ex)
    os.environ.pop("RABITQ_SCAN_TRACE", None)
    idx.search(Q, s.k, s.nprobe, s.M)
    torch.cuda.synchronize()
    os.environ["RABITQ_SCAN_TRACE"] = f"{out}_e{ex}.bin"
    idx.search(Q, s.k, s.nprobe, s.M)
    torch.cuda.synchronize()
    print("wrote", f"{out}_e{ex}.bin", flush=True)
