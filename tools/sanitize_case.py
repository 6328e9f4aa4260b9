"""Small searches through every kernel family of the path, for
compute-sanitizer runs (one tool per gpurun call):
small-K tensor-core scan (main, dense sample, re-scan), generic grouped scan
(d = 960, and d = 128 forced), popc scan, quantizer, probe GEMM + select,
select + re-rank, dense re-rank block, merge, the build (k-means argmin GEMM)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_16007_b200 as rq  # noqa: E402
import synth  # noqa: E402


def data(D, N, nlist, nq):
    s = synth.spec(1, D=D, N=N, ncent=nlist, nlist=nlist, nq=nq, kind="iso", data_seed=3)
    cen = synth.centres(s, "cpu")
    return synth.base_rows(s, 0, N, "cpu", cen=cen).cuda(), synth.queries(s, "cpu", cen=cen).cuda()


def main():
    X, Q = data(128, 20000, 32, 300)
    idx = rq.Index(X, nlist=32, seed=42)
    idx.search(Q, 10, 8, 100, scan_path=rq.SCAN_IMMA)
    idx.search(Q, 10, 8, 100, scan_path=rq.SCAN_IMMA, cap=200, seed_max=100)  # forced re-scans
    idx.search(Q, 10, 8, 100, scan_path=rq.SCAN_IMMA, variant=rq.VARIANT_GENERIC_SCAN)
    idx.search(Q, 10, 8, 100, scan_path=rq.SCAN_POPC)
    idx.search(Q, 10, 8, 100, scan_path=rq.SCAN_IMMA, rank_key=rq.RANK_LOWER_BOUND)
    X2, Q2 = data(960, 6000, 16, 260)
    idx2 = rq.Index(X2, nlist=16, seed=42)
    idx2.search(Q2, 100, 4, 400, scan_path=rq.SCAN_IMMA)
    ids = torch.stack([idx.search(Q, 10, 8, 100)[0] for _ in range(2)])
    d = torch.stack([idx.search(Q, 10, 8, 100)[1] for _ in range(2)])
    rq.merge_topk(ids, d)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
