"""Timeline of the folded scan's CTA 0 (RABITQ_DIAG build, RABITQ_FOLD_TIMELINE=<file>):
median clock deltas between the pipeline events of a tile / unit."""
import sys

import numpy as np

EV = ["A_issue(t)", "rowf_ok(t)", "X_done(t)", "AX_ready(t)", "acce_ok(u)", "issued(u)", "claim_q0(u)", "accf_ok_q0(u)",
      "rel_q0(u)", "rel_q1(u)", "rel_q2(u)", "rel_q3(u)", "flagged_q0(u)"]


def main(path):
    a = np.fromfile(path, dtype=np.int64).reshape(16, 1024)
    n = int(np.count_nonzero(a[5]))
    print("units stamped", n)
    lo, hi = 64, min(n, 1000)
    t = {k: a[i, lo:hi].astype(np.float64) for i, k in enumerate(EV)}

    def med(x, name):
        x = x[np.isfinite(x)]
        print(f"{name:48s} median {np.median(x):8.0f}  p10 {np.percentile(x, 10):8.0f}  p90 {np.percentile(x, 90):8.0f}")

    med(np.diff(t["issued(u)"]), "issue period (unit)")
    med(t["issued(u)"] - t["acce_ok(u)"], "issue - acce_ok")
    med(t["acce_ok(u)"] - t["AX_ready(t)"], "acce_ok - AX_ready (>0: slot is the last gate)")
    med(t["accf_ok_q0(u)"] - t["issued(u)"], "accf_ok(q0) - issued  (MMA latency + wake)")
    med(t["accf_ok_q0(u)"] - t["claim_q0(u)"], "accf_ok(q0) - claim   (epilogue warp waiting)")
    med(t["rel_q0(u)"] - t["accf_ok_q0(u)"], "release(q0) - accf_ok (fast pass)")
    rel = np.maximum.reduce([t[f"rel_q{q}(u)"] for q in range(4)])
    med(rel - t["rel_q0(u)"], "last quarter's release - q0's")
    med(t["acce_ok(u)"][4:] - rel[:-4], "acce_ok(u+4) - last release(u)  (MMA wake)")
    med(t["issued(u)"][4:] - t["issued(u)"][:-4], "issued(u+4) - issued(u)  (slot loop)")
    med(t["X_done(t)"] - t["rowf_ok(t)"], "X_done - rowf_ok")
    med(t["rowf_ok(t)"] - t["A_issue(t)"], "rowf_ok - A_issue (row-constant latency)")
    med(t["AX_ready(t)"] - t["A_issue(t)"], "AX_ready - A_issue (A stage latency)")
    med(t["AX_ready(t)"][1:] - t["issued(u)"][:-1], "AX_ready(t+1) - issued(t) (>0: A supply is the last gate)")
    fl = a[12, lo:hi] != 0
    print("flagged q0 units", int(fl.sum()), "of", hi - lo)


if __name__ == "__main__":
    main(sys.argv[1])
