"""Opcode / stall histogram of one kernel's SASS from an ncu source export
(`ncu -i rep --page source --csv --print-source sass`); optional address range."""
import collections
import csv
import sys


def load(path, kernel_idx=0):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and len(r) > 10:
            cur["rows"].append(r)
    return blocks[kernel_idx]


def main(path, kernel_idx=0):
    b = load(path, kernel_idx)
    hdr, data = b["hdr"], b["rows"]
    ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ie]) for r in data) or 1
    tots = sum(int(r[ss]) for r in data) or 1
    print(b["name"][:100], "warp-instructions", tot, "stall samples", tots)
    op, ops = collections.Counter(), collections.Counter()
    for r in data:
        t = r[1].split()
        o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        op[o] += int(r[ie])
        ops[o] += int(r[ss])
    for o, c in op.most_common(45):
        print(f"{o:10s} {100 * c / tot:5.1f}% inst {100 * ops[o] / tots:5.1f}% samp")
    for k in hdr:
        if k.startswith("stall_") and "Not" not in k:
            i = hdr.index(k)
            s = sum(int(r[i]) for r in data)
            if s:
                print(f"{k:24s} {100 * s / tots:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
