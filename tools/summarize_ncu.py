"""Summarise ncu outputs into profiles/ (markdown + json).

  python tools/summarize_ncu.py launches <launches.csv> <out.md> [--after KERNEL_REGEX]
  python tools/summarize_ncu.py full <report.ncu-rep> <out.md> <out.json>
"""
import collections
import csv
import json
import re
import subprocess
import sys


def _ns(v, unit):
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)


def launches(path, out, after=None):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                data.append((d["Kernel Name"], _ns(d["Metric Value"], d["Metric Unit"])))
    if after:
        idx = next((i for i, (k, _) in enumerate(data) if re.search(after, k)), 0)
        # start at the first launch of the search path (the step's first kernel)
        data = data[idx:]
    agg = collections.OrderedDict()
    for k, v in data:
        short = re.sub(r"\(.*", "", k).replace("rabitq::<unnamed>::", "").replace("void ", "")
        agg.setdefault(short, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = ["| share | launches | avg us | total ms | kernel |", "|---:|---:|---:|---:|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {sum(v) / tot * 100:.2f}% | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / 1e6:.3f} | `{k}` |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:25]))


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
]


def full(rep, out_md, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = re.sub(r"\(.*", "", d.get("Kernel Name", "")).replace("rabitq::<unnamed>::", "").replace("void ", "")
        m = {}
        for k in KEYS:
            for h, u in zip(hdr, units):
                if h == k:
                    m[k] = (d.get(h), u)
        res.append((name, m))
    lines = []
    js = {}
    for name, m in res:
        lines.append(f"### `{name}`\n\n| metric | value | unit |\n|---|---:|---|")
        for k, (v, u) in m.items():
            lines.append(f"| {k} | {v} | {u} |")
        lines.append("")
        try:
            rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = rd * scale.get(m["dram__bytes_read.sum"][1], 1) + wr * scale.get(m["dram__bytes_write.sum"][1], 1)
            # the bench's dominant-kernel keys: the main scan launch and the re-rank
            # scan_imma_kernel<LB, dump, retry, dense, tma-A>: the main scan has LB = dump = retry = dense = 0
            main_scan = ("scan_imma_kernel<0, 0, 0, 0" in name) or "scan_popc" in name or "scan_fold_kernel" in name
            key = "scan" if main_scan else ("select_rerank" if "select_rerank" in name else name)
            js.setdefault(key, tot)
        except Exception:
            pass
    open(out_md, "w").write("\n".join(lines) + "\n")
    json.dump(js, open(out_json, "w"), indent=1)
    print("\n".join(lines))
    print(js)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        after = sys.argv[sys.argv.index("--after") + 1] if "--after" in sys.argv else None
        launches(sys.argv[2], sys.argv[3], after)
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4])
