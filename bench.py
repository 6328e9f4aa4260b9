#!/usr/bin/env python
"""bench.py -- the IVF-RaBitQ search hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of the whole hot path (rotate, probe, quantize, scan +
estimator, top-M, exact re-rank; + NCCL top-k merge for N > 1) over one batch
of the config's queries against its index, inputs resident in HBM.  The
default workload is BASELINE.json configs[3] (CFG4: D=128, N=1e8 uint8-valued
vectors, nlist=16384, 10k queries, nprobe=64, k=10, re-rank 100), the largest
configuration that fits one GPU.  Rank 0 prints ONE JSON line.

For N > 1 (torchrun, one process per GPU) the index is sharded by contiguous
id slices, every rank scans its shard for all queries, and the
per-rank top-k are merged by an NCCL all-gather: total work is
fixed, "scaling": "strong".

--impl reference times the oracle (oracle/, plain C fp64) on this box's host
cores on the same config/metric, each step a bounded sample of the queries,
over the lists they probe of an index built with plain torch ops (the oracle's
rotation, torch k-means/assignment; no librabitq kernel); rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "QPS at fixed nprobe/k (coarse-scan GB/s vs HBM peak; recall@k vs exact)"
ALU_OPS_PER_PAIR = 5  # fused estimator + threshold per (query, vector) pair


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML every
    ~5 ms from a thread (nvidia-smi's 100 ms period sees one sample of a
    ~100 ms region), nvidia-smi as the fallback."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device, self.rows, self.proc, self.nvml = device, [], None, None
        self.stop_flag = threading.Event()

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.nvml = (pynvml, h)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        while not self.stop_flag.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.t.join(timeout=2)
            sm = [r[0] for r in self.rows]
            reasons = sorted({n for _, rs in self.rows for n, bit in self.REASONS.items() if rs & bit})
            load = [x for x in sm if x > 500] or sm
            return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": float(self.max_sm),
                    "reasons": reasons, "samples": len(self.rows), "source": "nvml 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 8]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows), "source": "nvidia-smi 100 ms"}


# ------------------------------------------------------------- workload --
def workload(args):
    ov = {}
    if args.nq:
        ov["nq"] = args.nq
    if getattr(args, "nprobe", 0):
        ov["nprobe"] = args.nprobe
    return synth.spec(args.config, **ov)


def build_shard(s, rank, world, dev, rq, proxy=None):
    from paper_2605_16007_b200 import dist as rdist

    """Generate this rank's contiguous id slice on the device and build its
    shard (rank 0 trains P and the centroids, the others reuse them).
    proxy = (r, G): a single process builds shard r of G exactly as rank 0
    of a G-GPU job would build its own (CFG5 does not fit one GPU)."""
    lo, hi = rdist.shard_range(s.N, *(proxy if proxy else (rank, world)))
    cen = synth.centres(s, dev)
    t0 = time.time()
    X = synth.base_rows(s, lo, hi, dev, cen=cen)
    Q = synth.queries(s, dev, cen=cen)
    init = synth.init_centroids(s, dev)
    if world > 1:
        torch.distributed.broadcast(Q, 0)
    tgen = time.time() - t0
    t0 = time.time()
    if world == 1:
        idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=init, id_offset=lo)
    else:
        P = torch.empty(s.D, s.D, device=dev)
        C = torch.empty(s.nlist, s.D, device=dev)
        if rank == 0:
            idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=init, id_offset=lo)
            ex = idx.export()
            P.copy_(torch.from_numpy(ex["rotation"]))
            C.copy_(torch.from_numpy(ex["centroids"]))
        rdist.broadcast_params(P, C)
        if rank != 0:
            idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, id_offset=lo, rotation=P,
                           centroids_rot=C)
    torch.cuda.synchronize()
    log(f"[rank {rank}] data {tgen:.1f}s build {time.time() - t0:.1f}s rows [{lo},{hi}) {idx.info()}")
    return idx, X, Q


def l2_flush(buf):
    buf.add_(1.0)  # writes 256 MiB > 126 MB L2


def run_ours(args):
    import paper_2605_16007_b200 as rq
    from paper_2605_16007_b200 import dist as rdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
    s = workload(args)
    proxy = tuple(int(v) for v in args.shard.split("/")) if args.shard else None
    if proxy and world > 1:
        raise SystemExit("--shard is a single-process proxy")
    idx, X, Q = build_shard(s, rank, world, dev, rq, proxy)
    info = idx.info()
    comm = None
    if world > 1:
        uid = rdist.share_unique_id(rq.Comm.unique_id() if rank == 0 else None)
        comm = rq.Comm(uid, rank, world, local)
    stream = torch.cuda.Stream(dev)  # the library's kernels and the timing events share this stream
    ids = torch.empty(s.nq, s.k, dtype=torch.int64, device=dev)
    dist = torch.empty(s.nq, s.k, dtype=torch.float32, device=dev)
    flush = torch.zeros(64 << 20, dtype=torch.float32, device=dev)

    # query-split probing in the single-GPU shard proxy: this rank probes its
    # ceil(nq / G) queries inside the step; the other ranks' lists (which the
    # all-gather of the real job delivers, 5 MB at CFG5) are precomputed here
    qs_probes, qs_slice = None, None
    if proxy and args.query_split:
        c = (s.nq + proxy[1] - 1) // proxy[1]
        qs_slice = (proxy[0] * c, min(s.nq, (proxy[0] + 1) * c))
        qs_probes = idx.probe(Q, s.nprobe, stream=stream)
        torch.cuda.synchronize()

    def step(prof=None):
        if comm is None and qs_probes is not None:
            idx.probe(Q[qs_slice[0]:qs_slice[1]], s.nprobe, stream=stream)
            idx.search(Q, s.k, s.nprobe, s.M, scan_path=args.scan_path, stream=stream, out=(ids, dist),
                       profile=prof, rerank=args.rerank, query_bits=args.query_bits, probes=qs_probes)
        elif comm is None:
            idx.search(Q, s.k, s.nprobe, s.M, scan_path=args.scan_path, stream=stream, out=(ids, dist),
                       profile=None if args.graph else prof, rerank=args.rerank, query_bits=args.query_bits,
                       graph=args.graph, variant=args.variant)
        else:
            kw = dict(scan_path=args.scan_path, stream=stream.cuda_stream, query_split=args.query_split)
            if prof is not None:
                import ctypes

                kw["profile"] = ctypes.pointer(prof)
            r = comm.search_sharded(idx, Q, s.k, s.nprobe, s.M, **kw)
            ids.copy_(r[0])
            dist.copy_(r[1])

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    clk = ClockSampler(local)
    clk.start()
    times, profs = [], []
    for _ in range(args.steps):
        l2_flush(flush)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        prof = rq.Profile()
        e0.record(stream)
        step(prof)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        profs.append(prof.as_dict())
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    if args.graph and comm is None:  # stage times of the same search on the normal (profiled) path
        prof = rq.Profile()
        idx.search(Q, s.k, s.nprobe, s.M, scan_path=args.scan_path, stream=stream, out=(ids, dist), profile=prof,
                   rerank=args.rerank, query_bits=args.query_bits)
        torch.cuda.synchronize()
        profs = [prof.as_dict()]
    total = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(total, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(total.item())
    ms_per_step = total_ms / args.steps
    qps = s.nq * args.steps / (total_ms / 1e3)

    # ---- NEXT-2: small batches on several streams at once (latency mode), host wall clock ----
    overlapped = None
    if args.graph and args.streams > 1 and comm is None:
        streams = [torch.cuda.Stream(dev) for _ in range(args.streams)]
        outs = [(torch.empty_like(ids), torch.empty_like(dist)) for _ in streams]

        def worker(i, n):
            for _ in range(n):
                idx.search(Q, s.k, s.nprobe, s.M, scan_path=args.scan_path, stream=streams[i], out=outs[i], graph=1)

        for i in range(args.streams):  # capture one graph entry per stream
            worker(i, 2)
        torch.cuda.synchronize()
        nrep = max(20, args.steps)
        ths = [threading.Thread(target=worker, args=(i, nrep)) for i in range(args.streams)]
        t0 = time.perf_counter()
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        overlapped = {"streams": args.streams, "batches": args.streams * nrep, "batch": s.nq,
                      "qps": round(args.streams * nrep * s.nq / wall, 1),
                      "ms_per_batch": round(1e3 * wall / nrep, 4),
                      "timing": "host wall clock over all streams' batches (each call synchronises its stream)"}
        for (a_, b_) in outs:
            assert torch.equal(a_, ids) and torch.equal(b_, dist)

    # ---- e2e: the same search through the C ABI with HOST buffers ----
    Qh = Q.cpu().pin_memory()
    ih = torch.empty(s.nq, s.k, dtype=torch.int64).pin_memory()
    dh = torch.empty(s.nq, s.k, dtype=torch.float32).pin_memory()
    for _ in range(1):
        if comm is None:
            idx.search(Qh, s.k, s.nprobe, s.M, scan_path=args.scan_path, out=(ih, dh), rerank=args.rerank,
                       query_bits=args.query_bits, graph=args.graph)
        else:
            comm.search_sharded(idx, Qh, s.k, s.nprobe, s.M, scan_path=args.scan_path, query_split=args.query_split)
    barrier()
    et = []
    for _ in range(max(3, min(args.steps, 10))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if comm is None:
            idx.search(Qh, s.k, s.nprobe, s.M, scan_path=args.scan_path, out=(ih, dh), rerank=args.rerank,
                       query_bits=args.query_bits, graph=args.graph)
        else:
            r = comm.search_sharded(idx, Qh, s.k, s.nprobe, s.M, scan_path=args.scan_path,
                                    query_split=args.query_split)
        et.append(time.perf_counter() - t0)
    log(f"[rank {rank}] e2e ms per call: {[round(t_ * 1e3, 2) for t_ in et]}")
    e2e_t = torch.tensor([sum(et)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(e2e_t, op=torch.distributed.ReduceOp.MAX)
    e2e_qps = s.nq * len(et) / float(e2e_t.item())

    # ---- roofline of the dominant kernel (stage times measured live with CUDA events) ----
    pk = peaks()
    stage_ms = {k_: float(np.mean([p["stage_ms"][k_] for p in profs])) for k_ in profs[0]["stage_ms"]}
    pairs = float(np.mean([p["pairs"] for p in profs]))
    surv = float(np.mean([p["survivors"] for p in profs]))
    max_surv = int(max(p["max_survivors"] for p in profs))
    retries = int(max(p["retries"] for p in profs))
    imma = profs[0]["scan_path_used"] in (2, 3)
    launches = int(round(np.mean([p["kernel_launches"] for p in profs])))
    W = s.W
    scan_bytes = pairs * (4 * W + 8)  # code words + {n_o^2, f1} per (query, vector) pair
    rerank_bytes = s.nq * s.M * (4 * s.D + 8) + surv * 8
    # with the dense nearest-list block (nq >= 256, slot vectors built: CFG2) the gather kernel moves only
    # the rows the block cannot decide: use the DRAM bytes ncu measured for it (same workload), not
    # M (4D + 8) per query, which would read above the HBM peak
    traffic_all = {}
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{s.cfg}.json")
    if os.path.exists(tpath):
        try:
            traffic_all = json.load(open(tpath))
        except Exception:
            traffic_all = {}
    dense_used = info["bytes_slot_vectors"] > 0 and s.nq >= 256 and s.D % 4 == 0
    if dense_used and traffic_all.get("select_rerank"):
        rr_bytes, rr_src = float(traffic_all["select_rerank"]), f"ncu DRAM bytes per launch ({os.path.basename(tpath)})"
    else:
        rr_bytes, rr_src = rerank_bytes, "algorithmic M (4D + 8) per query + survivor keys"
    int8_peak = 2.0 * pk.get("bf16_tflops", 1590.0)  # dense int8 = 2x bf16 (nominal ratio, B200_PROFILING.md)
    scan_ops = 2.0 * pairs * s.D  # int8 multiply-adds of <b, qbar>, 2 ops each
    # d <= 128 (the small-K scan): a pair is 4 K-steps of one UMMA but ~5 FP32 lane
    # operations of the fused estimator + threshold (int->float, 3 FMA, compare;
    # DESIGN.md sec 6): the FP32 ALU, not the tensor pipe, is the roof
    alu_peak = 148 * 128 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12  # lane-ops/s, T
    alu_ops = ALU_OPS_PER_PAIR * pairs
    scan_tensor = {"bound": "tensor", "achieved": scan_ops / (stage_ms["scan"] * 1e-3) / 1e12, "unit": "TFLOP/s",
                   "peak": int8_peak, "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (int8:bf16 = 2:1 nominal)",
                   "algorithmic": scan_ops}
    scan_alu = {"bound": "alu", "achieved": alu_ops / (stage_ms["scan"] * 1e-3) / 1e12, "unit": "Tops/s",
                "peak": round(alu_peak, 2), "algorithmic": alu_ops,
                "peak_source": "148 SMs x 128 FP32 lanes x sm_max_mhz (MEASURED_PEAKS.json), 1 op per lane-instruction"}
    small_k = imma and s.D <= 128
    fold = small_k and profs[0]["scan_path_used"] == 3  # the folded tensor-core survivor test ran
    if fold:
        # folded small-K scan: the survivor test runs on the tensor cores, so
        # the tensor pipe is the roof.  Algorithmic work = the e4m3 ip contraction, 2 D ops per
        # pair, against the f8 peak (2 x measured bf16, nominal f8:bf16 = 2:1); the executed
        # tensor work also holds K = Dp padding and the K = 16 tf32 factor contraction
        # (4 f8-equivalent ops per tf32 op at the nominal 4.5 : 1.1 PF ratio)
        dp = ((s.D + 31) // 32) * 32
        f8_ops = 2.0 * pairs * s.D
        exec_ops = pairs * (2.0 * dp + 2.0 * 16 * 4)
        scan_tensor = {"bound": "tensor", "achieved": f8_ops / (stage_ms["scan"] * 1e-3) / 1e12, "unit": "TFLOP/s",
                       "peak": int8_peak, "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (f8:bf16 = 2:1 nominal)",
                       "algorithmic": f8_ops,
                       "executed_f8_equiv_frac": round(exec_ops / (stage_ms["scan"] * 1e-3) / 1e12 / int8_peak, 4)}
    rl = {
        "scan": (((scan_tensor if fold else scan_alu) if small_k else scan_tensor) if imma else
                 {"bound": "hbm", "achieved": scan_bytes / (stage_ms["scan"] * 1e-3) / 1e9, "unit": "GB/s",
                  "peak": pk["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json hbm_gbs", "algorithmic": scan_bytes}),
        "select_rerank": {"bound": "hbm", "achieved": rr_bytes / (stage_ms["select_rerank"] * 1e-3) / 1e9,
                          "unit": "GB/s", "peak": pk["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                          "algorithmic": rerank_bytes, "bytes_source": rr_src},
    }
    ms_of = {"scan": stage_ms["scan"], "select_rerank": stage_ms["select_rerank"]}
    dom = max(ms_of, key=ms_of.get)
    traffic = None
    prof_path = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{s.cfg}.json")
    if os.path.exists(prof_path):
        try:
            traffic = json.load(open(prof_path)).get(dom)
        except Exception:
            traffic = None
    r = rl[dom]
    roofline = {"kernel": dom, "bound": r["bound"], "achieved": round(r["achieved"], 1), "peak": r["peak"],
                "peak_source": r["peak_source"], "unit": r["unit"], "frac": round(r["achieved"] / r["peak"], 4),
                "traffic": traffic, "algorithmic_per_launch": r["algorithmic"], "ms": round(ms_of[dom], 4)}
    other = "select_rerank" if dom == "scan" else "scan"
    ro = rl[other]
    roofline_other = {"kernel": other, "bound": ro["bound"], "achieved": round(ro["achieved"], 1), "unit": ro["unit"],
                      "frac": round(ro["achieved"] / ro["peak"], 4), "ms": round(ms_of[other], 4),
                      **({"bytes_source": ro["bytes_source"]} if "bytes_source" in ro else {})}
    scan_roof = {"path": ("tcgen05 e4m3 + tf32 folded test" if fold else "tcgen05 int8") if imma else "popc",
                 "pairs": pairs,
                 "hbm_equiv_gbs": round(scan_bytes / (stage_ms["scan"] * 1e-3) / 1e9, 1),
                 "bytes_per_pair": 4 * W + 8, "ms": round(stage_ms["scan"], 4)}
    if fold:
        # the folded scan reads one f32 accumulator per pair from TMEM: against the read rate
        # tools/ubench/tmem_ld.cu measures (375 B per clock and SM with >= 12 reading warps,
        # profiles/r2c/tmem_ld.txt) -- not the bound, stated so that the bound is named by measurement
        tm_peak = 375.0 * 148 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e9
        scan_roof["tmem_read"] = {"achieved_gbs": round(pairs * 4 / (stage_ms["scan"] * 1e-3) / 1e9, 1),
                                  "peak_gbs": round(tm_peak, 1),
                                  "frac": round(pairs * 4 / (stage_ms["scan"] * 1e-3) / 1e9 / tm_peak, 4)}

    # ---- recall@k vs exact on a query sample (torch brute force, outside the timed region) ----
    rec = None
    gt = None
    if world == 1 and args.recall:
        nsub = min(100 if s.N <= 10_000_000 else 20, s.nq)
        step = max(1, (1 << 28) // (s.D * 4 * 8))  # rows per chunk (~1 GiB of fp32 temporaries)
        gt = []
        nx = X.shape[0]
        lo = rdist.shard_range(s.N, *proxy)[0] if proxy else 0
        for q in range(nsub):
            dd = torch.empty(nx, dtype=torch.float64, device=dev)
            for r0 in range(0, nx, step):
                dd[r0:r0 + step] = (X[r0:r0 + step] - Q[q]).pow(2).sum(1, dtype=torch.float64)
            gt.append(torch.topk(dd, s.k, largest=False).indices.cpu() + lo)
        gt = torch.stack(gt).numpy()
        got = ids[:nsub].cpu().numpy()
        rec = float(np.mean([len(set(a_.tolist()) & set(b_.tolist())) / s.k for a_, b_ in zip(got, gt)]))

    line = {
        "metric": METRIC, "value": round(qps, 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": (("u8 (tcgen05 kind::i8: 0/1 codes x four 6-bit digit rows of the 24-bit fixed-point query)"
                   if args.query_bits == 32 else "u8 (tcgen05 kind::i8: 0/1 codes x 4-bit query)")
                  + " + f32 estimator/re-rank" if imma
                  else "u32 bit-planes (AND+POPC) + f32 estimator/re-rank"),
        "data": "synthetic (synth/ seeded Gaussian mixture, generated on device)",
        "config": {"workload": f"CFG{s.cfg}", "D": s.D, "N": s.N, "nlist": s.nlist, "nq": s.nq, "nprobe": s.nprobe,
                   "k": s.k, "n_rerank": s.M, "kind": s.kind, "parallelism": (f"shard {args.shard} (single-GPU proxy: one rank's share)" if proxy
                                   else f"list-shards x{world}"),
                   "l2": "flushed between steps (256 MiB write)", "scan_path": args.scan_path,
                   **({"probing": "query-split" if args.query_split else "replicated"} if (proxy or world > 1) else {}),
                   **({"mode": "latency (CUDA graph per batch, NEXT-2); stage_ms from one profiled normal-path search"}
                      if args.graph else {}),
                   **({"variant": args.variant} if args.variant else {}),
                   **({"rerank": "bound-driven (NEXT-4)"} if args.rerank else {}),
                   **({"query": "unquantized, 24-bit fixed point digit rows (NEXT-1)"} if args.query_bits == 32
                      else {})},
        "e2e": {"value": round(e2e_qps, 1), "unit": "queries/s", "h2d_bytes_per_step": s.nq * s.D * 4 * world,
                "d2h_bytes_per_step": s.nq * s.k * 12 * world},
        "gpu_launches": launches * args.steps,
        "roofline": roofline, "roofline_other": roofline_other, "scan": scan_roof,
        **({"roofline_tensor": {k_: (round(v, 4) if isinstance(v, float) else v) for k_, v in scan_tensor.items()}
            | {"frac": round(scan_tensor["achieved"] / scan_tensor["peak"], 4)}} if small_k and not fold else {}),
        "index_bytes": {"total": info["bytes_total"], "codes_and_factors": info["bytes_codes"] + info["bytes_factors"],
                        "codes8": info["bytes_codes8"], "slot_vectors": info["bytes_slot_vectors"],
                        "vectors_fp32": s.N * s.D * 4 // max(1, world)},
        "stage_ms": {k_: round(v, 4) for k_, v in stage_ms.items()},
        **({"dense_rerank_block": {"kernel": "tgemm_dist1 (side stream, beside stages 2-5)",
                                   "ms": round(float(np.mean([p["dense_ms"] for p in profs])), 4),
                                   "dram_bytes": traffic_all.get("unnamed>::tgemm_dist1_kernel")}}
           if float(np.mean([p["dense_ms"] for p in profs])) > 0 else {}),
        "survivors_per_query": round(surv / s.nq, 1), "max_survivors": max_surv, "overflow_rescans": retries,
        **({"reranked_per_query": round(float(np.mean([p["reranked"] for p in profs])) / s.nq, 1)}
           if args.rerank else {}),
        "recall_at_k": rec, "clocks": clocks,
        **({"overlapped": overlapped} if overlapped else {}),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(s, idx, X, Q, args, gt=gt, got=ids)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.free()
    if world > 1:
        torch.distributed.destroy_process_group()


# ------------------------------------------------------- CPU (oracle) legs --
def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(s, idx, X, Q, args, budget_s=20.0, gt=None, got=None):
    """The oracle as it stands, on this box's host cores, on a bounded query
    sample (about `budget_s` seconds of CPU work) over a sub-index of the lists
    those queries probe (oracle/subindex.py: the oracle's arithmetic unchanged,
    only the arrays it is handed are smaller)."""
    import oracle as orc
    from oracle.subindex import SubIndex

    orc.build()
    cores = _cores()
    nmax = min(s.nq, 4096)
    probes = torch.empty(nmax, s.nprobe, dtype=torch.int32, device=Q.device)
    idx.search(Q[:nmax], s.k, s.nprobe, s.M, debug=dict(probes=probes))
    ex = idx.export()
    Qh = Q[:nmax].cpu().numpy()
    pr = probes.cpu().numpy()

    last = {}

    def timed(n, threads=cores):
        sub = SubIndex(ex, pr[:n].ravel(), lambda g: X[torch.from_numpy(g).to(X.device)].cpu().numpy())
        t0 = time.perf_counter()
        last["ids"] = sub.search(orc, Qh[:n], s.k, s.nprobe, s.M, s.build_seed, num_threads=threads)[0]
        return time.perf_counter() - t0

    n0 = min(nmax, max(2, cores))
    t = timed(n0)
    n = int(min(nmax, max(n0, n0 * budget_s / max(t, 1e-3))))
    t = timed(n)
    out = {"value": round(n / t, 3), "unit": "queries/s", "cores": cores, "kind": "oracle",
           "sample": f"first {n} of {s.nq} CFG{s.cfg} queries, full oracle path (fp64 rotate/probe, pinned fp32 "
                     f"quantizer, plain-loop ip, fp64 estimator, full sort, fp64 re-rank) over a sub-index of their "
                     f"probed lists, OpenMP {cores} threads, {t:.1f} s"}
    # the oracle's recall on the bench's own recall subset (same exact kNN ground
    # truth as recall_at_k) next to the GPU's, and the oracle at 1 thread (about budget_s / 4 s)
    if gt is not None:
        m = min(len(gt), n)
        oids = np.asarray(last["ids"])[:m]
        gids = got[:m].cpu().numpy()

        def rcl(a):
            return float(np.mean([len(set(x.tolist()) & set(y.tolist())) / s.k for x, y in zip(a, gt[:m])]))

        out["recall_subset"] = {"queries": m, "oracle": round(rcl(oids), 4), "gpu": round(rcl(gids), 4),
                                "identical_queries": round(float(np.mean([np.array_equal(np.sort(x), np.sort(y))
                                                                          for x, y in zip(oids, gids)])), 4)}
    n1 = int(max(1, min(n, n * (budget_s / 4) / max(t, 1e-3) / max(1, cores))))
    t1 = timed(n1, threads=1)
    out["value_1thread"] = round(n1 / t1, 3)
    out["sample_1thread"] = f"first {n1} queries, 1 thread, {t1:.1f} s"
    return out


def reference_index(s, X, seed):
    """Index for the reference arm, built with plain torch ops (no librabitq
    kernel; on the GPU when there is one, chunked, so CFG4's 1e8 rows fit): the
    oracle's Haar P; k-means (10 Lloyd iterations on 32 nlist rows) and
    nearest-centroid assignment; sign codes and factors of the rotated residual.
    Returns the export-format dict (list order) the oracle consumes."""
    import oracle as orc

    dev = X.device
    _, P = orc.haar_rotation(s.D, seed)
    Pt = torch.from_numpy(P).to(dev)
    g = torch.Generator().manual_seed(seed)
    ts = min(s.N, 32 * s.nlist)
    T = X[torch.randperm(s.N, generator=g)[:ts].to(dev)] @ Pt
    C = T[torch.randperm(ts, generator=g)[: s.nlist].to(dev)].clone()
    ch = max(1, (1 << 27) // max(1, s.nlist))  # rows per distance block (~512 MB of fp32)

    def nearest(A):
        out = torch.empty(A.shape[0], dtype=torch.int64, device=dev)
        cn = (C * C).sum(1)
        for r0 in range(0, A.shape[0], ch):
            blk = A[r0:r0 + ch]
            out[r0:r0 + ch] = (cn[None, :] - 2.0 * (blk @ C.T)).argmin(1)
        return out

    for _ in range(10):
        a = nearest(T)
        Cn = torch.zeros_like(C).index_add_(0, a, T)
        cnt = torch.bincount(a, minlength=s.nlist)
        C = torch.where(cnt[:, None] > 0, Cn / cnt.clamp_min(1)[:, None], C)
    W = s.W
    assign = torch.empty(s.N, dtype=torch.int64, device=dev)
    codes = torch.empty(s.N, W, dtype=torch.int64, device=dev)
    n_o = torch.empty(s.N, dtype=torch.float32, device=dev)
    rho = torch.empty(s.N, dtype=torch.float32, device=dev)
    shifts = torch.arange(32, device=dev, dtype=torch.int64)
    for r0 in range(0, s.N, 1 << 20):
        Xr = X[r0:r0 + (1 << 20)] @ Pt
        a = nearest(Xr)
        R = (Xr - C[a]).double()
        bits = torch.zeros(R.shape[0], W * 32, dtype=torch.int64, device=dev)
        bits[:, : s.D] = (R >= 0).long()
        codes[r0:r0 + R.shape[0]] = (bits.view(-1, W, 32) << shifts).sum(-1)
        no = R.norm(dim=1)
        n_o[r0:r0 + R.shape[0]] = no.float()
        rho[r0:r0 + R.shape[0]] = torch.where(no > 0, R.abs().sum(1) / (np.sqrt(s.D) * no), torch.ones_like(no)).float()
        assign[r0:r0 + R.shape[0]] = a
    order = torch.argsort(assign, stable=True)
    off = torch.zeros(s.nlist + 1, dtype=torch.int64)
    off[1:] = torch.cumsum(torch.bincount(assign, minlength=s.nlist).cpu(), 0)
    return dict(rotation=P.astype(np.float32), centroids=C.float().cpu().numpy(), list_off=off.numpy(),
                ids=order.cpu().numpy().astype(np.int64),
                codes=codes[order].cpu().numpy().astype(np.uint32), n_o=n_o[order].cpu().numpy(),
                rho=rho[order].cpu().numpy())


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as orc
    from oracle.subindex import SubIndex

    orc.build()
    s = workload(args)
    t0 = time.time()
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    cen = synth.centres(s, dev)
    X = synth.base_rows(s, 0, s.N, dev, cen=cen)
    Q = synth.queries(s, dev, cen=cen)
    ex = reference_index(s, X, s.build_seed)
    Qh = Q.cpu().numpy()
    log(f"[reference] data + index (torch ops on {dev.type}) {time.time() - t0:.1f}s")
    cores = _cores()

    def sub_for(qs):  # the oracle's own probes of these queries -> the lists it will read
        lists = np.unique(np.concatenate([orc.probe(orc.rotate(Qh[q:q + 1], ex["rotation"])[0].astype(np.float32),
                                                    ex["centroids"], s.nprobe) for q in qs]))
        return SubIndex(ex, lists, lambda gids: X[torch.from_numpy(gids).to(dev)].cpu().numpy())

    def timed(sub, q0, n):
        t = time.perf_counter()
        sub.search(orc, Qh[q0:q0 + n], s.k, s.nprobe, s.M, s.build_seed, qid_base=q0, num_threads=cores)
        return time.perf_counter() - t

    n0 = min(s.nq, max(2, cores))
    t = timed(sub_for(range(n0)), 0, n0)
    per_step_budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    nqs = int(min(s.nq, max(1, n0 * per_step_budget / max(t, 1e-3))))
    pool = min(s.nq, nqs * (args.steps + args.warmup))
    sub = sub_for(range(pool))
    starts = [(i * nqs) % max(1, pool - nqs + 1) for i in range(args.steps + args.warmup)]
    for w in range(args.warmup):
        timed(sub, starts[w], nqs)
    tt = [timed(sub, starts[args.warmup + i], nqs) for i in range(args.steps)]
    qps = nqs * len(tt) / sum(tt)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(qps, 3), "unit": "queries/s", "n_gpus": int(
            os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(tt) / len(tt), 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 (oracle)", "data": "synthetic (synth/, same generator as the GPU arm)",
        "config": {"workload": f"CFG{s.cfg}", "D": s.D, "N": s.N, "nlist": s.nlist, "nq": s.nq, "nprobe": s.nprobe,
                   "k": s.k, "n_rerank": s.M, "queries_per_step": nqs},
        "cpu_baseline": {"value": round(qps, 3), "unit": "queries/s", "cores": cores, "kind": "oracle",
                         "sample": f"{nqs} queries per step of CFG{s.cfg}, the full oracle path (fp64 rotate/probe, "
                                   f"pinned fp32 quantizer, plain-loop ip, fp64 estimator, full sort, fp64 re-rank) "
                                   f"over the lists they probe of an index built with torch ops (no librabitq)"},
        "e2e": {"value": round(qps, 3), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_build(args):
    """NEXT-3: index-build throughput as a second timed workload.
    One build = rabitq_build over the config's N synthetic vectors resident in
    HBM (k-means on the sampled training rows, rotation, assignment, encode,
    list layout, the expanded codes and slot-ordered vectors when they fit).
    The build is synchronous and host-orchestrated, so it is timed by the host
    clock between device synchronizations."""
    import paper_2605_16007_b200 as rq

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    s = workload(args)
    cen = synth.centres(s, dev)
    X = synth.base_rows(s, 0, s.N, dev, cen=cen)
    init = synth.init_centroids(s, dev)
    warm = max(1, min(args.warmup, 1))
    steps = max(1, args.steps)
    times = []
    info = None
    for i in range(warm + steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx = rq.Index(X, nlist=s.nlist, seed=s.build_seed, borrow=True, init_centroids=init)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        info = idx.info()
        del idx
        if i >= warm:
            times.append(dt)
        log(f"build {i}: {dt:.3f} s")
    tb = float(np.mean(times))
    line = {
        "metric": "index build throughput", "value": round(s.N / tb, 1), "unit": "vectors/s", "n_gpus": 1,
        "steps": steps, "warmup": warm, "ms_per_step": round(tb * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (k-means, rotation, assignment GEMMs) + u32 codes",
        "data": "synthetic (synth/ seeded Gaussian mixture, generated on device)",
        "config": {"workload": f"CFG{s.cfg} build", "D": s.D, "N": s.N, "nlist": s.nlist, "kind": s.kind,
                   "kmeans": "25 Lloyd iterations on min(N, 256 nlist) stratified training rows",
                   "timing": "host clock between device synchronizations (synchronous build)"},
        "index_bytes": info["bytes_total"], "codes8_bytes": info["bytes_codes8"],
        "slot_vector_bytes": info["bytes_slot_vectors"],
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4,
                    help="BASELINE.json configs[C-1]; default 4 = the largest single-GPU config (N = 1e8)")
    ap.add_argument("--nq", type=int, default=0, help="override the query count (quick runs)")
    ap.add_argument("--nprobe", type=int, default=0, help="override nprobe (CFG3's sweep: 16/32/64/128)")
    ap.add_argument("--nprobe-sweep", default="", dest="nprobe_sweep",
                    help="comma list, e.g. 16,32,64,128 (CFG3): one JSON line per nprobe from one call, same code")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scan-path", type=int, default=0, dest="scan_path")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-recall", dest="recall", action="store_false")
    ap.add_argument("--query-bits", type=int, default=4, choices=[4, 32], dest="query_bits",
                    help="32: unquantized query (NEXT-1; changes the estimates, opt-in)")
    ap.add_argument("--rerank", type=int, default=0, choices=[0, 1],
                    help="1: bound-driven re-rank set (NEXT-4; changes results, opt-in)")
    ap.add_argument("--workload", choices=["search", "build"], default="search",
                    help="build: time rabitq_build (NEXT-3) instead of the search hot path")
    ap.add_argument("--variant", type=int, default=0,
                    help="rabitq_search_opts.variant bits (result-invariant paths: 2 = codes expanded in the scan "
                         "kernel, no expanded-code copy read; 8 = generic grouped scan)")
    ap.add_argument("--streams", type=int, default=1,
                    help="with --graph 1: also time batches issued from this many host threads / streams at once")
    ap.add_argument("--graph", type=int, default=0, choices=[0, 1],
                    help="1: latency mode (NEXT-2): the batch captured once as a CUDA graph and replayed")
    ap.add_argument("--query-split", type=int, default=1, choices=[0, 1], dest="query_split",
                    help="N > 1 / --shard: 1 = each rank probes nq/G queries, probe lists all-gathered (SURVEY 8(e))")
    ap.add_argument("--shard", default="", help="r/G: time shard r of G on one GPU (per-GPU proxy for configs "
                    "that need G GPUs, e.g. CFG5); the line then reports that shard's QPS")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("note: warmup raised to the contract minimum of 3")
        args.warmup = 3
    if args.workload == "build":
        run_build(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.nprobe_sweep:
        for npb in [int(x) for x in args.nprobe_sweep.split(",") if x]:
            args.nprobe = npb
            run_ours(args)
            torch.cuda.empty_cache()
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
