"""Helpers for the GPU-vs-oracle parity tests.

Tolerances (BASELINE.json north_star; R#18, R#27):
  ip       bit-exact given identical quantized queries
  est      |est_gpu - est_oracle| <= 1e-4 * n_q * n_o + 2^-20 * (n_o^2 + n_q^2)
  top-k    identical ids except ties within that tolerance (coarse) or within
           1e-5 * d_k (exact distances, fp32 vs fp64)
"""
from __future__ import annotations

import numpy as np

EST_REL = 1e-4
EST_ABS2 = 2.0 ** -20
D_REL = 1e-5


def est_tol(n_o, nq2):
    return EST_REL * np.sqrt(nq2) * n_o + EST_ABS2 * (n_o * n_o + nq2)


def list_pos_of_items(probes_flat, list_off):
    """For the flattened (pair, 32-slot block) scan items, return arrays
    (pair, list, position-in-list) for every (item, lane) entry."""
    sizes = (list_off[1:] - list_off[:-1])[probes_flat]
    nb = (sizes + 31) // 32
    item_pair = np.repeat(np.arange(probes_flat.size), nb)
    item_off = np.concatenate([[0], np.cumsum(nb)])
    blk = np.arange(item_pair.size) - item_off[item_pair]
    pair = np.repeat(item_pair, 32)
    pos = (np.repeat(blk, 32) * 32 + np.tile(np.arange(32), item_pair.size)).astype(np.int64)
    lst = probes_flat[pair]
    valid = pos < sizes[pair]
    return pair, lst, pos, valid, int(item_pair.size)


def check_probe_lists(gpu_probes, qr, Cr, nprobe):
    """L1: identical probe lists except swaps between centroids whose fp64
    distances differ by <= 1e-5 relative.  Returns the number of tie swaps."""
    swaps = 0
    C64 = Cr.astype(np.float64)
    for q in range(gpu_probes.shape[0]):
        d = ((qr[q].astype(np.float64) - C64) ** 2).sum(1)
        order = np.lexsort((np.arange(d.size), d))
        ref = order[:nprobe]
        g = gpu_probes[q]
        if np.array_equal(g, ref):
            continue
        # same multiset up to near-ties at the boundary, and order up to near-ties
        dk = d[ref[-1]]
        for a, b in zip(g, ref):
            if a != b:
                assert abs(d[a] - d[b]) <= 1e-5 * max(dk, 1e-30), (q, a, b, d[a], d[b])
                swaps += 1
    return swaps


def check_final(gpu_ids, gpu_d, ref_ids, ref_d, k):
    """Final top-k: identical except ties within 1e-5 * d_k.  Returns the number
    of tie-explained differences."""
    diffs = 0
    for q in range(gpu_ids.shape[0]):
        if np.array_equal(gpu_ids[q], ref_ids[q]):
            assert np.allclose(gpu_d[q], ref_d[q], rtol=D_REL, atol=0), q
            continue
        dk = float(np.max(ref_d[q][np.isfinite(ref_d[q])], initial=0.0))
        tol = D_REL * max(dk, 1e-30)
        assert np.allclose(np.sort(gpu_d[q]), np.sort(ref_d[q]), rtol=0, atol=tol), (q, gpu_d[q], ref_d[q])
        for a, da in zip(gpu_ids[q], gpu_d[q]):
            if a not in set(ref_ids[q].tolist()):
                # a GPU id outside the reference set must tie with the reference boundary
                assert abs(da - ref_d[q][-1]) <= tol, (q, a, da, ref_d[q][-1])
                diffs += 1
    return diffs


def recall(ids, gt, k):
    return float(np.mean([len(set(a[:k].tolist()) & set(b[:k].tolist())) / k for a, b in zip(ids, gt)]))
