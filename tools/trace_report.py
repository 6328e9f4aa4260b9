"""Summarise a grouped-scan clock trace (tools/scan_trace.py output)."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 16)
n = int((t[:, 0] > 0).sum())
nt = int((t[:, 13] > 0).sum())
c = t[:n].astype(np.float64)
base = c[0, 0]
def stat(name, x):
    x = x[np.isfinite(x)]
    print(f"{name:40s} median {np.median(x):8.0f}  mean {x.mean():8.0f}  p90 {np.percentile(x, 90):8.0f}")
print(f"chunks traced {n}, tiles {nt}, span {c[n-1,4]-base:.0f} cycles, per chunk {(c[n-1,4]-base)/n:.0f}")
stat("prod: wait empty", c[:, 1] - c[:, 0])
stat("prod: expand+STS", c[:, 2] - c[:, 1])
stat("prod: fence", c[:, 3] - c[:, 2])
stat("prod: bar+arrive", c[:, 4] - c[:, 3])
stat("prod: chunk period (0->0)", np.diff(c[:, 0]))
stat("prod g1: wait-empty end vs g0", c[:, 5] - c[:, 1])
m = c[:n]
stat("mma: wait bfull", m[:, 8] - m[:, 7])
stat("mma: wait full", m[:, 9] - m[:, 8])
stat("mma: issue+commit", m[:, 10] - m[:, 9])
stat("mma: chunk period", np.diff(m[:, 9]))
stat("full arrive -> mma sees", m[:, 9] - c[:, 4])
# empty: chunk gc+stages freed -> producer waiting on gc+stages
for S in (5, 10):
    if n > S:
        stat(f"mma commit(gc) -> prod empty done(gc+{S})", c[S:, 1] - m[:-S, 10])
e = t[:nt].astype(np.float64)
stat("epi: wait accf", e[:, 14] - e[:, 13])
stat("epi: tile work", e[:, 15] - e[:, 14])
stat("mma: wait acce (per tile)", e[:, 12] - e[:, 11])
