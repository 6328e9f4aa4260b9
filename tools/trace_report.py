"""Summarise a grouped-scan clock trace (tools/scan_trace.py output).
Slots (scan_imma.cu RQ_TR): producer tid 0 per chunk: 0 before slot wait,
1 after, 2 after TMEM stores, 4 after full arrive; MMA lane 0 per chunk:
7 before waits, 9 after full wait, 10 after issue + commits; per tile: MMA
11/12 around the accumulator-empty wait, epilogue warp 0: 13/14 around the
accumulator-full wait, 15 tile done."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 16).astype(np.float64)
n = int((t[:, 0] > 0).sum())
nt = int((t[:, 13] > 0).sum())
c = t[:n]


def stat(name, x):
    x = x[np.isfinite(x)]
    if len(x):
        print(f"{name:44s} median {np.median(x):8.0f}  mean {x.mean():8.0f}  p90 {np.percentile(x, 90):8.0f}")


print(f"chunks traced {n}, tiles {nt}, span {c[n-1,4]-c[0,0]:.0f} cycles, per chunk {(c[n-1,4]-c[0,0])/n:.0f}")
stat("prod: loop top -> issue done", c[:, 5] - c[:, 3])
stat("prod: cp.async wait + LDS", c[:, 6] - c[:, 5])
stat("prod: previous arrive -> loop top", c[1:, 3] - c[:-1, 4])
stat("prod: wait slot", c[:, 1] - c[:, 0])
stat("prod: expand + tcgen05.st", c[:, 2] - c[:, 1])
stat("prod: bar + arrive", c[:, 4] - c[:, 2])
stat("prod: chunk period", np.diff(c[:, 0]))
stat("mma: waits (bfull + full)", c[:, 9] - c[:, 7])
stat("mma: issue + commit", c[:, 10] - c[:, 9])
stat("mma: chunk period", np.diff(c[:, 9]))
stat("full arrive -> mma sees", c[:, 9] - c[:, 4])
e = t[:nt]
stat("epi: wait accf", e[:, 14] - e[:, 13])
stat("epi: tile work", e[:, 15] - e[:, 14])
stat("mma: wait acce (per tile)", e[:, 12] - e[:, 11])
