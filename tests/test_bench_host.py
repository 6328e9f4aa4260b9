"""Host-side pieces of bench.py (CPU): the reference arm's torch-built index (run here on the CPU) matches
the oracle's encode of the same P / centroids / assignment."""
import numpy as np
import torch

import bench
import synth


def test_reference_index_encode_matches_oracle(orc):
    s = synth.spec(1, D=40, N=3000, ncent=12, nlist=12, nq=5)
    cen = synth.centres(s, "cpu")
    X = synth.base_rows(s, 0, s.N, "cpu", cen=cen)
    ex = bench.reference_index(s, X, 3)
    off, ids = ex["list_off"], ex["ids"]
    assign = np.empty(s.N, np.int32)
    for j in range(s.nlist):
        assign[ids[off[j]:off[j + 1]]] = j
    codes, n_o, rho = orc.encode(X.numpy()[ids], ex["rotation"], ex["centroids"], assign[ids])
    mism = (codes != ex["codes"]).sum()
    assert mism <= 2, mism  # fp32 CPU matmul vs fp64: only near-zero residual bits may flip
    assert np.allclose(n_o, ex["n_o"], rtol=1e-4, atol=1e-5)
    # and the oracle searches it end to end
    Q = synth.queries(s, "cpu", cen=cen).numpy()
    oi, od = orc.search(Q, ex["rotation"], ex["centroids"], off, ids, ex["codes"], ex["n_o"], ex["rho"],
                        X.numpy(), 5, 4, 50, 42)
    assert (oi >= 0).all()
