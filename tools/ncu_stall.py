"""Per-source-line share of one stall reason from an ncu source export
(`--page source --csv --print-source cuda,sass`).  Usage: ncu_stall.py file reason [top]"""
import csv
import sys


def main(path, reason, top=15):
    hdr, f, agg = None, None, {}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0]:
            continue
        if len(r) >= len(hdr) - 20:
            agg[(f, r[0])] = r
    i = hdr.index(reason)
    agg = {k: v for k, v in agg.items() if len(v) > i}
    tot = sum(float(v[i] or 0) for v in agg.values()) or 1
    print(f"{reason}: {tot:.0f} samples")
    for k, v in sorted(agg.items(), key=lambda kv: -float(kv[1][i] or 0))[:top]:
        print(f"{100 * float(v[i] or 0) / tot:5.1f}%  {k[0]}:{k[1]}  {v[1][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 15)
