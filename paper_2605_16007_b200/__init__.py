"""Python binding of librabitq -- the B200-native IVF-RaBitQ search hot path.

Argument marshalling only: every step of the path runs in the CUDA kernels of
``librabitq.so`` (built from ``csrc/`` for sm_100a), reached through the C ABI
declared in ``include/rabitq.h``.  PyTorch is used for device memory, streams
and process groups.  There is no CPU fallback: if the library is missing or no
sm_100 device is present the calls raise.

    idx = Index(X, nlist=1024, seed=42)                 # rabitq_build
    ids, dists = idx.search(Q, k=10, nprobe=64, n_rerank=100)   # rabitq_search
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librabitq.so")

OK, ERR_INVALID_ARGUMENT, ERR_INVALID_DATA, ERR_OUT_OF_MEMORY, ERR_CUDA, ERR_NCCL, ERR_UNSUPPORTED, ERR_INTERNAL = range(8)
SCAN_AUTO, SCAN_POPC, SCAN_IMMA = 0, 1, 2
RANK_EST, RANK_LOWER_BOUND = 0, 1
# rabitq_search_opts.variant bits: alternative execution paths, identical results
VARIANT_RADIX_PROBE, VARIANT_EXPAND_IN_KERNEL, VARIANT_NO_DENSE_RERANK, VARIANT_GENERIC_SCAN = 1, 2, 4, 8
VARIANT_UNIFORM_SEED, VARIANT_NO_FOLD, VARIANT_FOLD_INPLACE = 16, 32, 64
RERANK_FIXED, RERANK_BOUND = 0, 1


class RabitqError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rabitq status {status}: {msg}")
        self.status = status


# ------------------------------------------------------------------ C structs
class BuildOpts(ctypes.Structure):
    _fields_ = [
        ("kmeans_iters", ctypes.c_int32),
        ("train_size", ctypes.c_int64),
        ("init_centroids", ctypes.c_void_p),
        ("borrow_vectors", ctypes.c_int32),
        ("id_offset", ctypes.c_int64),
        ("rotation", ctypes.c_void_p),
        ("centroids_rot", ctypes.c_void_p),
        ("device", ctypes.c_int32),
    ]


class Debug(ctypes.Structure):
    _fields_ = [
        ("qrot", ctypes.c_void_p),
        ("probes", ctypes.c_void_p),
        ("qbar", ctypes.c_void_p),
        ("qscal", ctypes.c_void_p),
        ("topm_ids", ctypes.c_void_p),
        ("topm_est", ctypes.c_void_p),
        ("topm_bound", ctypes.c_void_p),
        ("tau", ctypes.c_void_p),
        ("survivors", ctypes.c_void_p),
        ("retries", ctypes.c_void_p),
        ("scan_ip", ctypes.c_void_p),
        ("scan_est", ctypes.c_void_p),
        ("scan_dump_cap", ctypes.c_int64),
    ]


NSTAGES = 8
STAGES = ["rotate", "probe", "quantize", "plan", "seed", "scan", "rescan", "select_rerank"]


class Profile(ctypes.Structure):
    _fields_ = [
        ("stage_ms", ctypes.c_float * NSTAGES),
        ("pairs", ctypes.c_int64),
        ("survivors", ctypes.c_int64),
        ("max_survivors", ctypes.c_int64),
        ("retries", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("scan_path_used", ctypes.c_int32),
        ("batches", ctypes.c_int32),
        ("reranked", ctypes.c_int64),
        ("dense_ms", ctypes.c_float),
    ]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "stage_ms"}
        d["stage_ms"] = {s: float(self.stage_ms[i]) for i, s in enumerate(STAGES)}
        return d


class SearchOpts(ctypes.Structure):
    _fields_ = [
        ("scan_path", ctypes.c_int32),
        ("rank_key", ctypes.c_int32),
        ("eps0", ctypes.c_float),
        ("query_id_base", ctypes.c_int64),
        ("cap_per_query", ctypes.c_int32),
        ("seed_max", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("debug", ctypes.POINTER(Debug)),
        ("profile", ctypes.POINTER(Profile)),
        ("rerank", ctypes.c_int32),
        ("query_bits", ctypes.c_int32),
        ("variant", ctypes.c_uint32),
        ("probes_in", ctypes.c_void_p),
        ("query_split", ctypes.c_int32),
        ("graph", ctypes.c_int32),
    ]


class IndexInfo(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32), ("W", ctypes.c_int32), ("nlist", ctypes.c_int32), ("device", ctypes.c_int32),
        ("n", ctypes.c_int64), ("id_offset", ctypes.c_int64), ("max_list", ctypes.c_int64),
        ("bytes_codes", ctypes.c_int64), ("bytes_factors", ctypes.c_int64), ("bytes_ids", ctypes.c_int64),
        ("bytes_vectors", ctypes.c_int64), ("bytes_total", ctypes.c_int64),
        ("vectors_borrowed", ctypes.c_int32),
        ("bytes_codes8", ctypes.c_int64), ("bytes_slot_vectors", ctypes.c_int64),
    ]


class Export(ctypes.Structure):
    _fields_ = [
        ("rotation", ctypes.c_void_p), ("centroids", ctypes.c_void_p), ("list_off", ctypes.c_void_p),
        ("ids", ctypes.c_void_p), ("codes", ctypes.c_void_p), ("n_o", ctypes.c_void_p), ("rho", ctypes.c_void_p),
    ]


EXPORTED = [
    "rabitq_build", "rabitq_build_ex", "rabitq_build_opts_default", "rabitq_search", "rabitq_search_ex",
    "rabitq_search_opts_default", "rabitq_index_info", "rabitq_index_export", "rabitq_free",
    "rabitq_last_error", "rabitq_version", "rabitq_comm_unique_id", "rabitq_comm_init", "rabitq_comm_free",
    "rabitq_search_sharded", "rabitq_merge_topk", "rabitq_selftest", "rabitq_probe",
]

_lib = None


def lib() -> ctypes.CDLL:
    """Load librabitq.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        L.rabitq_last_error.restype = ctypes.c_char_p
        L.rabitq_version.restype = ctypes.c_char_p
        for f in EXPORTED:
            getattr(L, f)  # every declared symbol must resolve
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        raise RabitqError(status, lib().rabitq_last_error().decode())


def _torch():
    import torch

    return torch


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _as_f32(x):
    torch = _torch()
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if x.dtype != torch.float32:
        x = x.float()
    return x.contiguous()


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream))


def _call_stream(stream, dev_tensor, temps):
    """The stream a device-side call runs on: the caller's, else torch's
    current stream on the tensor's device (so the library's kernels are
    ordered after the torch work that produced the inputs).  Tensors created
    here for the call (dtype / layout copies, outputs) are recorded on a
    foreign stream so the caching allocator does not reuse them early."""
    torch = _torch()
    if dev_tensor is None or not dev_tensor.is_cuda:
        return _stream_handle(stream)
    if stream is None:
        return torch.cuda.current_stream(dev_tensor.device).cuda_stream
    h = _stream_handle(stream)
    if h != torch.cuda.current_stream(dev_tensor.device).cuda_stream:
        ext = stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.ExternalStream(h, device=dev_tensor.device)
        for t in temps:
            if t is not None and t.is_cuda:
                t.record_stream(ext)
    return h


class Index:
    """An IVF-RaBitQ index on one GPU (``rabitq_build_ex``)."""

    def __init__(self, X, nlist: int, seed: int = 42, *, kmeans_iters: int = 0, train_size: int = 0,
                 init_centroids=None, borrow: bool = False, id_offset: int = 0, rotation=None,
                 centroids_rot=None, device: int = -1):
        X = _as_f32(X)
        n, d = X.shape
        keep = []
        o = BuildOpts()
        lib().rabitq_build_opts_default(ctypes.byref(o))
        o.kmeans_iters = kmeans_iters
        o.train_size = train_size
        if init_centroids is not None:
            ic = _as_f32(init_centroids)
            keep.append(ic)
            o.init_centroids = _ptr(ic)
        if rotation is not None:
            r = _as_f32(rotation)
            keep.append(r)
            o.rotation = _ptr(r)
        if centroids_rot is not None:
            c = _as_f32(centroids_rot)
            keep.append(c)
            o.centroids_rot = _ptr(c)
        o.borrow_vectors = 1 if borrow else 0
        o.id_offset = id_offset
        o.device = device if device >= 0 else (X.device.index if X.is_cuda else -1)
        if X.is_cuda:  # the build runs on its own stream: inputs produced by torch must be complete
            _torch().cuda.current_stream(X.device).synchronize()
        h = ctypes.c_void_p()
        _check(lib().rabitq_build_ex(ctypes.c_void_p(_ptr(X)), ctypes.c_int64(n), ctypes.c_int32(d),
                                     ctypes.c_int32(nlist), ctypes.c_uint64(seed & (2**64 - 1)),
                                     ctypes.byref(o), ctypes.byref(h)))
        self._h = h
        self._X = X if borrow else None  # a borrowed X must outlive the index
        self.d, self.n, self.seed = d, n, seed
        self.nlist = self.info()["nlist"]

    # -- rabitq_search_ex -------------------------------------------------------
    def search(self, Q, k: int, nprobe: int, n_rerank: int, *, scan_path: int = SCAN_AUTO,
               rank_key: int = RANK_EST, eps0: float = 0.0, query_id_base: int = 0, cap: int = 0,
               seed_max: int = 0, stream=None, debug: Optional[dict] = None, out=None,
               profile: Optional[Profile] = None, rerank: int = RERANK_FIXED, query_bits: int = 4,
               variant: int = 0, probes=None, graph: int = 0):
        """Returns (ids int64 [nq, k], dists float32 [nq, k]) on Q's device.
        ``debug`` maps rabitq_debug member names to preallocated tensors.
        Device inputs run on ``stream`` (default: torch's current stream)."""
        torch = _torch()
        Q0 = Q
        Q = _as_f32(Q)
        nq = Q.shape[0]
        temps = [Q if Q is not Q0 else None]
        if out is None:
            ids = torch.empty((nq, k), dtype=torch.int64, device=Q.device)
            dists = torch.empty((nq, k), dtype=torch.float32, device=Q.device)
            temps += [ids, dists]
        else:
            ids, dists = out
        o = SearchOpts()
        lib().rabitq_search_opts_default(ctypes.byref(o))
        o.scan_path, o.rank_key, o.eps0 = scan_path, rank_key, eps0
        o.query_id_base, o.cap_per_query, o.seed_max = query_id_base, cap, seed_max
        o.rerank = rerank
        o.query_bits = query_bits
        o.variant = variant
        o.graph = graph
        if probes is not None:
            probes = probes.contiguous() if hasattr(probes, "contiguous") else np.ascontiguousarray(probes, np.int32)
            o.probes_in = _ptr(probes)
        o.stream = _call_stream(stream, Q, temps)
        dbg = None
        if debug:
            dbg = Debug()
            for name, t in debug.items():
                if name == "scan_dump_cap":
                    dbg.scan_dump_cap = int(t)
                else:
                    setattr(dbg, name, _ptr(t))
            o.debug = ctypes.pointer(dbg)
        if profile is not None:
            o.profile = ctypes.pointer(profile)
        _check(lib().rabitq_search_ex(self._h, ctypes.c_void_p(_ptr(Q)), ctypes.c_int64(nq), ctypes.c_int32(k),
                                      ctypes.c_int32(nprobe), ctypes.c_int32(n_rerank), ctypes.byref(o),
                                      ctypes.c_void_p(_ptr(ids)), ctypes.c_void_p(_ptr(dists))))
        return ids, dists

    # -- rabitq_probe (S1-S3 only) ----------------------------------------------
    def probe(self, Q, nprobe: int, *, stream=None):
        """int32 [nq, nprobe]: each query's nearest lists, ascending (d, list)."""
        torch = _torch()
        Q0 = Q
        Q = _as_f32(Q)
        nq = Q.shape[0]
        out = torch.empty((nq, nprobe), dtype=torch.int32, device=Q.device)
        h = _call_stream(stream, Q, [Q if Q is not Q0 else None, out])
        _check(lib().rabitq_probe(self._h, ctypes.c_void_p(_ptr(Q)), ctypes.c_int64(nq), ctypes.c_int32(nprobe),
                                  ctypes.c_void_p(_ptr(out)), ctypes.c_void_p(h)))
        return out

    def info(self) -> dict:
        i = IndexInfo()
        _check(lib().rabitq_index_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in IndexInfo._fields_}

    def export(self) -> dict:
        """Host numpy copies of the index, arrays in list order."""
        inf = self.info()
        n, d, W, nl = inf["n"], inf["d"], inf["W"], inf["nlist"]
        out = dict(
            rotation=np.empty((d, d), np.float32), centroids=np.empty((nl, d), np.float32),
            list_off=np.empty(nl + 1, np.int64), ids=np.empty(n, np.int64),
            codes=np.empty((n, W), np.uint32), n_o=np.empty(n, np.float32), rho=np.empty(n, np.float32),
        )
        e = Export(**{k: v.ctypes.data for k, v in out.items()})
        _check(lib().rabitq_index_export(self._h, ctypes.byref(e)))
        return out

    def free(self):
        if getattr(self, "_h", None):
            lib().rabitq_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def merge_topk(in_ids, in_d, stream=None):
    """(G, nq, k) device tensors -> global top-k by (dist, id) (rabitq_merge_topk)."""
    torch = _torch()
    G, nq, k = in_ids.shape
    oi = torch.empty((nq, k), dtype=torch.int64, device=in_ids.device)
    od = torch.empty((nq, k), dtype=torch.float32, device=in_ids.device)
    s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream(in_ids.device).cuda_stream
    _check(lib().rabitq_merge_topk(ctypes.c_void_p(_ptr(in_ids.contiguous())), ctypes.c_void_p(_ptr(in_d.contiguous())),
                                   ctypes.c_int32(G), ctypes.c_int64(nq), ctypes.c_int32(k),
                                   ctypes.c_void_p(_ptr(oi)), ctypes.c_void_p(_ptr(od)), ctypes.c_void_p(s)))
    return oi, od


class Comm:
    """NCCL communicator for the sharded search (rabitq_comm_*)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().rabitq_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, rank: int, world: int, device: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check(lib().rabitq_comm_init(buf, ctypes.c_int32(rank), ctypes.c_int32(world), ctypes.c_int32(device),
                                      ctypes.byref(h)))
        self._h = h
        self.rank, self.world, self.device = rank, world, device

    def search_sharded(self, shard: Index, Q, k, nprobe, n_rerank, **kw):
        torch = _torch()
        Q0 = Q
        Q = _as_f32(Q)
        nq = Q.shape[0]
        ids = torch.empty((nq, k), dtype=torch.int64, device=Q.device)
        dists = torch.empty((nq, k), dtype=torch.float32, device=Q.device)
        o = SearchOpts()
        lib().rabitq_search_opts_default(ctypes.byref(o))
        stream = kw.pop("stream", None)
        for key, v in kw.items():
            setattr(o, key, v)
        o.stream = _call_stream(stream, Q, [Q if Q is not Q0 else None, ids, dists])
        _check(lib().rabitq_search_sharded(shard._h, self._h, ctypes.c_void_p(_ptr(Q)), ctypes.c_int64(nq),
                                           ctypes.c_int32(k), ctypes.c_int32(nprobe), ctypes.c_int32(n_rerank),
                                           ctypes.byref(o), ctypes.c_void_p(_ptr(ids)),
                                           ctypes.c_void_p(_ptr(dists))))
        return ids, dists

    def free(self):
        if getattr(self, "_h", None):
            lib().rabitq_comm_free(self._h)
            self._h = None


def version() -> str:
    return lib().rabitq_version().decode()


def selftest(what: int, n: int, seed: int = 0) -> int:
    """rabitq_selftest: number of mismatches of a device arithmetic identity
    (what = 1: the quantizer's reciprocal division vs IEEE division)."""
    out = ctypes.c_uint64(0)
    _check(lib().rabitq_selftest(ctypes.c_int32(what), ctypes.c_uint64(n), ctypes.c_uint64(seed), ctypes.byref(out)))
    return int(out.value)
