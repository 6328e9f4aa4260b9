"""Sub-index extraction for running the oracle on sampled queries of a big
index (TEST INFRASTRUCTURE: used by tests/ and bench.py's cpu_baseline only).

Given the GPU index's export (list order) and the lists the sampled queries
probe, keep those lists and the fp32 rows they hold; ids are remapped to a
compact, order-preserving numbering (so every (value, id) tie-break is
unchanged) and mapped back after the search.  The oracle's arithmetic is not
touched: it runs unchanged on the smaller arrays.
"""
from __future__ import annotations

import numpy as np


class SubIndex:
    def __init__(self, ex: dict, lists, X_rows_fn):
        """ex: export dict (rotation, centroids, list_off, ids, codes, n_o, rho);
        lists: iterable of list ids to keep; X_rows_fn(ids) -> fp32 rows of
        those global ids (any device/host source)."""
        lists = np.unique(np.asarray(lists, dtype=np.int64))
        off = ex["list_off"]
        nlist = off.size - 1
        keep = np.zeros(nlist, bool)
        keep[lists] = True
        sizes = np.diff(off) * keep
        segs = [np.arange(off[j], off[j + 1]) for j in lists]
        pos = np.concatenate(segs) if segs else np.zeros(0, np.int64)
        gids = ex["ids"][pos]
        order_ids = np.sort(gids)
        self.global_ids = order_ids  # compact index -> global id (ascending)
        self.list_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        # list order is preserved (lists ascending, ids ascending within a list)
        self.list_ids = np.searchsorted(order_ids, gids).astype(np.int64)
        self.codes = ex["codes"][pos]
        self.n_o = ex["n_o"][pos]
        self.rho = ex["rho"][pos]
        self.P = ex["rotation"]
        self.Cr = ex["centroids"]
        self.X = np.ascontiguousarray(X_rows_fn(order_ids), dtype=np.float32)

    def to_global(self, ids):
        out = np.where(ids >= 0, self.global_ids[np.clip(ids, 0, None)], -1)
        return out.astype(np.int64)

    def search(self, orc, Q, k, nprobe, M, seed, **kw):
        res = orc.search(Q, self.P, self.Cr, self.list_off, self.list_ids, self.codes, self.n_o, self.rho, self.X,
                         k, nprobe, M, seed, **kw)
        ids = self.to_global(res[0])
        if kw.get("debug"):
            return (ids, res[1], res[2], self.to_global(res[3]), res[4])
        return ids, res[1]
