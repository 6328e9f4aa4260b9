"""Per-source-line instruction and stall-sample shares from an ncu report
(`ncu -i rep --page source --csv --print-source cuda,sass` output file)."""
import csv
import sys


def main(path, top=40):
    f = None
    agg = {}
    hdr = None
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
        try:
            inst = int(r[7] or 0)
            st = int(r[4] or 0)
        except (ValueError, IndexError):
            continue
        agg[(f, r[0])] = (inst, st, r[1][:100])
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {ti}, stall samples {ts}")
    for (fn, ln), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% samp  {fn}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
