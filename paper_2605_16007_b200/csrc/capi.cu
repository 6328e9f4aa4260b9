// capi.cu -- the C ABI of librabitq (include/rabitq.h): argument checking,
// host<->device staging, query batching, export/info and the NCCL
// communicator for the sharded search.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <cstdlib>
#include <vector>

#include "index.cuh"
#include "search.cuh"

using rabitq::Error;

namespace {

thread_local std::string g_err;

rabitq_status set_err(rabitq_status s, const std::string& m) {
    g_err = m;
    return s;
}

#define API_BEGIN try {
#define API_END                                                                        \
    }                                                                                  \
    catch (const Error& e) {                                                           \
        return set_err(e.status, e.what());                                            \
    }                                                                                  \
    catch (const std::bad_alloc&) {                                                    \
        return set_err(RABITQ_ERR_OUT_OF_MEMORY, "host allocation failed");            \
    }                                                                                  \
    catch (const std::exception& e) {                                                  \
        return set_err(RABITQ_ERR_INTERNAL, e.what());                                 \
    }                                                                                  \
    catch (...) {                                                                      \
        return set_err(RABITQ_ERR_INTERNAL, "unknown exception");                      \
    }                                                                                  \
    return RABITQ_OK;

bool on_device(const void* p, int device) {
    if (!p) return false;
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged) {
        if (pa.device != device) throw Error(RABITQ_ERR_INVALID_ARGUMENT, "device pointer on another device");
        return true;
    }
    return false;
}

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        throw Error(RABITQ_ERR_UNSUPPORTED, "no usable CUDA device / driver");
    }
    return dev;
}

void require_sm100(int dev) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw Error(RABITQ_ERR_UNSUPPORTED, "no CUDA device");
    }
    RQ_REQUIRE(dev >= 0 && dev < n, RABITQ_ERR_INVALID_ARGUMENT, "bad device ordinal");
    int major = 0, minor = 0;
    RQ_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    RQ_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    RQ_REQUIRE(major == 10 && minor == 0, RABITQ_ERR_UNSUPPORTED,
               "librabitq is built for sm_100a (B200); device is sm_" + std::to_string(major * 10 + minor));
    static bool pool_set[64] = {};
    if (dev < 64 && !pool_set[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;  // keep freed workspace cached: stream-ordered reuse, no re-allocation
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_set[dev] = true;
    }
}

// one NVTX push/pop range per public call (profilers filter on "rabitq:search" etc.)
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
};

// device staging buffer (stream ordered)
struct Stage {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    Stage() = default;
    Stage(size_t bytes, cudaStream_t s) : st(s) {
        if (bytes) RQ_CUDA(cudaMallocAsync(&p, bytes, s));
    }
    ~Stage() {
        if (p) cudaFreeAsync(p, st);
    }
};

// a debug/output pointer that may be host memory: device view + copy-back
template <typename T>
struct DevView {
    T* user = nullptr;
    T* dev = nullptr;
    size_t count = 0;
    std::unique_ptr<Stage> stage;
    void init(T* u, size_t n, int device, cudaStream_t st) {
        user = u;
        count = n;
        if (!u) return;
        if (on_device(u, device)) {
            dev = u;
        } else {
            stage = std::make_unique<Stage>(n * sizeof(T), st);
            dev = (T*)stage->p;
        }
    }
    void copy_back(cudaStream_t st) {
        if (user && dev != user) RQ_CUDA(cudaMemcpyAsync(user, dev, count * sizeof(T), cudaMemcpyDeviceToHost, st));
    }
};

__global__ void export_kernel(int64_t n, int W, int nlist, const int64_t* __restrict__ list_off,
                              const int64_t* __restrict__ slot_off, const uint32_t* __restrict__ codes,
                              const float* __restrict__ n_o, const float* __restrict__ rho,
                              const uint32_t* __restrict__ rows, int64_t id_offset, uint32_t* __restrict__ o_codes,
                              float* __restrict__ o_no, float* __restrict__ o_rho, int64_t* __restrict__ o_ids) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nlist;  // largest j with list_off[j] <= p
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (list_off[mid] <= p) lo = mid;
            else hi = mid;
        }
        const int64_t slot = slot_off[lo] + (p - list_off[lo]);
        if (o_codes)
            for (int w = 0; w < W; ++w) o_codes[(size_t)p * W + w] = codes[((size_t)(slot >> 5) * W + w) * 32 + (slot & 31)];
        if (o_no) o_no[p] = n_o[slot];
        if (o_rho) o_rho[p] = rho[slot];
        if (o_ids) o_ids[p] = (int64_t)rows[slot] + id_offset;
    }
}

}  // namespace

struct rabitq_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
};

extern "C" {

const char* rabitq_last_error(void) { return g_err.c_str(); }
rabitq_status rabitq_selftest(int32_t what, uint64_t n, uint64_t seed, uint64_t* mismatches) {
    API_BEGIN
    RQ_REQUIRE(mismatches != nullptr, RABITQ_ERR_INVALID_ARGUMENT, "mismatches is NULL");
    RQ_REQUIRE(what == 1, RABITQ_ERR_INVALID_ARGUMENT, "unknown selftest");
    cudaStream_t st = nullptr;
    RQ_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
        *mismatches = rabitq::selftest_div(n, seed, st);
    } catch (...) {
        cudaStreamDestroy(st);
        throw;
    }
    RQ_CUDA(cudaStreamDestroy(st));
    API_END
}

const char* rabitq_version(void) { return "librabitq 0.1 (IVF-RaBitQ search hot path, sm_100a)"; }

void rabitq_build_opts_default(rabitq_build_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->device = -1;
}

void rabitq_search_opts_default(rabitq_search_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
}

rabitq_status rabitq_build(const float* X, int64_t n, int32_t d, int32_t nlist, uint64_t seed, rabitq_index** out) {
    rabitq_build_opts o;
    rabitq_build_opts_default(&o);
    return rabitq_build_ex(X, n, d, nlist, seed, &o, out);
}

rabitq_status rabitq_build_ex(const float* X, int64_t n, int32_t d, int32_t nlist, uint64_t seed,
                              const rabitq_build_opts* opts, rabitq_index** out) {
    API_BEGIN
    RQ_REQUIRE(out != nullptr, RABITQ_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    rabitq_build_opts o;
    rabitq_build_opts_default(&o);
    if (opts) o = *opts;
    RQ_REQUIRE(X != nullptr, RABITQ_ERR_INVALID_ARGUMENT, "X is NULL");
    RQ_REQUIRE(d >= 1 && d <= 4096, RABITQ_ERR_INVALID_ARGUMENT, "d must be in [1, 4096]");
    RQ_REQUIRE(n >= 1 && n < ((int64_t)1 << 31), RABITQ_ERR_INVALID_ARGUMENT, "n must be in [1, 2^31)");
    RQ_REQUIRE(nlist >= 0, RABITQ_ERR_INVALID_ARGUMENT, "nlist < 0");
    if (nlist == 0) nlist = (int)std::ceil(std::sqrt((double)n));  // AUTO
    RQ_REQUIRE(n >= nlist, RABITQ_ERR_INVALID_ARGUMENT, "n < nlist");
    RQ_REQUIRE(nlist <= (1 << 24), RABITQ_ERR_INVALID_ARGUMENT, "nlist too large");
    int dev = o.device;
    if (dev < 0) dev = current_device();
    require_sm100(dev);
    RQ_CUDA(cudaSetDevice(dev));
    std::unique_ptr<rabitq_index> idx(new rabitq_index());
    idx->device = dev;
    RQ_CUDA(cudaStreamCreateWithFlags(&idx->stream, cudaStreamNonBlocking));
    try {
        rabitq::build_index(idx.get(), X, n, d, nlist, seed, o);
        RQ_CUDA(cudaStreamSynchronize(idx->stream));
    } catch (...) {
        cudaStreamSynchronize(idx->stream);
        rabitq::free_index_memory(idx.get());
        cudaStreamDestroy(idx->stream);
        cudaGetLastError();
        throw;
    }
    *out = idx.release();
    API_END
}

static void free_graph_cache(void* p);

void rabitq_free(rabitq_index* idx) {
    if (!idx) return;
    cudaSetDevice(idx->device);
    cudaStreamSynchronize(idx->stream);
    free_graph_cache(idx->graphs);
    idx->graphs = nullptr;
    rabitq::free_index_memory(idx);
    cudaStreamDestroy(idx->stream);
    delete idx;
}

rabitq_status rabitq_search(const rabitq_index* idx, const float* Q, int64_t nq, int32_t k, int32_t nprobe,
                            int32_t n_rerank, int64_t* ids, float* dists) {
    return rabitq_search_ex(idx, Q, nq, k, nprobe, n_rerank, nullptr, ids, dists);
}

// ----------------------------------------------------- NEXT-2 latency mode --
// One batch's whole path captured once as a CUDA graph (latency mode: no host
// synchronisation inside, SearchCfg::latency) and replayed: per call one copy
// of Q into the graph's input buffer, one graph launch, one copy out and one
// synchronisation, at which the batch's overflow / non-finite counters are
// read; a batch whose survivor buffers overflowed is re-run on the normal path
// (results never depend on which path ran).  Keyed by every argument that the
// captured kernels bake in; a small per-index cache.
struct GraphEntry {
    std::mutex busy;  // held while the entry's graph and I/O buffers are in use (one replay at a time)
    int64_t nq = 0, qid_base = 0;
    int k = 0, nprobe = 0, M = 0;
    rabitq::SearchCfg cfg;
    cudaGraphExec_t exec = nullptr;
    float* Qg = nullptr;
    int64_t* ids = nullptr;
    float* d = nullptr;
    int* flags = nullptr;  // host pinned [8]
    ~GraphEntry() {
        if (exec) cudaGraphExecDestroy(exec);
        cudaFree(Qg);
        cudaFree(ids);
        cudaFree(d);
        cudaFreeHost(flags);
    }
};
struct GraphCache {
    std::mutex mu;
    std::vector<std::unique_ptr<GraphEntry>> entries;
};

static void free_graph_cache(void* p) { delete static_cast<GraphCache*>(p); }

static bool same_cfg(const rabitq::SearchCfg& a, const rabitq::SearchCfg& b) {
    return a.scan_path == b.scan_path && a.rank_key == b.rank_key && a.eps0 == b.eps0 && a.cap == b.cap &&
           a.seed_max == b.seed_max && a.refine_rank == b.refine_rank && a.rerank == b.rerank && a.full == b.full &&
           a.variant == b.variant;
}

static void search_graph(const rabitq_index* idx, const float* Qd, int64_t nq, int k, int nprobe, int M,
                         const rabitq::SearchCfg& cfg, int64_t qid_base, int64_t* ids_d, float* d_d, cudaStream_t st) {
    rabitq_index* mi = const_cast<rabitq_index*>(idx);
    if (!mi->graphs) mi->graphs = new GraphCache();
    GraphCache* gc = static_cast<GraphCache*>(mi->graphs);
    // a free entry of this shape (concurrent callers on other streams take other entries, so
    // their batches overlap); a new capture when every matching entry is busy
    std::unique_lock<std::mutex> lock(gc->mu);
    GraphEntry* g = nullptr;
    std::unique_lock<std::mutex> held;
    for (auto& e : gc->entries)
        if (e->nq == nq && e->k == k && e->nprobe == nprobe && e->M == M && e->qid_base == qid_base &&
            same_cfg(e->cfg, cfg)) {
            std::unique_lock<std::mutex> t(e->busy, std::try_to_lock);
            if (t.owns_lock()) {
                g = e.get();
                held = std::move(t);
                break;
            }
        }
    const int D = idx->D;
    if (!g) {
        if (gc->entries.size() >= 8) {  // drop the oldest idle entry
            for (auto it = gc->entries.begin(); it != gc->entries.end(); ++it) {
                std::unique_lock<std::mutex> t((*it)->busy, std::try_to_lock);
                if (t.owns_lock()) {
                    t.unlock();
                    gc->entries.erase(it);
                    break;
                }
            }
        }
        auto e = std::make_unique<GraphEntry>();
        e->nq = nq, e->k = k, e->nprobe = nprobe, e->M = M, e->qid_base = qid_base, e->cfg = cfg;
        RQ_CUDA(cudaMalloc(&e->Qg, (size_t)nq * D * sizeof(float)));
        RQ_CUDA(cudaMalloc(&e->ids, (size_t)nq * k * sizeof(int64_t)));
        RQ_CUDA(cudaMalloc(&e->d, (size_t)nq * k * sizeof(float)));
        RQ_CUDA(cudaMallocHost(&e->flags, 8 * sizeof(int)));
        cudaStream_t cs = nullptr;
        RQ_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        rabitq::SearchCfg c = cfg;
        c.latency = true;
        c.flags_out = e->flags;
        cudaGraph_t graph = nullptr;
        RQ_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        try {
            rabitq::SearchStats stats;
            rabitq::search_batch(idx, e->Qg, nq, k, nprobe, M, c, qid_base, e->ids, e->d, rabitq::DebugOut{}, cs,
                                 &stats);
        } catch (...) {
            cudaStreamEndCapture(cs, &graph);
            if (graph) cudaGraphDestroy(graph);
            cudaStreamDestroy(cs);
            throw;
        }
        RQ_CUDA(cudaStreamEndCapture(cs, &graph));
        cudaStreamDestroy(cs);
        const cudaError_t ie = cudaGraphInstantiate(&e->exec, graph, 0);
        cudaGraphDestroy(graph);
        RQ_CUDA(ie);
        g = e.get();
        held = std::unique_lock<std::mutex>(g->busy);
        gc->entries.push_back(std::move(e));
    }
    lock.unlock();  // replay under the entry's own lock only
    RQ_CUDA(cudaMemcpyAsync(g->Qg, Qd, (size_t)nq * D * sizeof(float), cudaMemcpyDeviceToDevice, st));
    RQ_CUDA(cudaGraphLaunch(g->exec, st));
    RQ_CUDA(cudaMemcpyAsync(ids_d, g->ids, (size_t)nq * k * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    RQ_CUDA(cudaMemcpyAsync(d_d, g->d, (size_t)nq * k * sizeof(float), cudaMemcpyDeviceToDevice, st));
    RQ_CUDA(cudaStreamSynchronize(st));
    RQ_REQUIRE(g->flags[0] == 0, RABITQ_ERR_INVALID_DATA, "Q contains non-finite values");
    if (g->flags[1] != 0) {  // a survivor buffer overflowed / under-filled: the normal path re-scans
        rabitq::SearchStats stats;
        rabitq::search_batch(idx, Qd, nq, k, nprobe, M, cfg, qid_base, ids_d, d_d, rabitq::DebugOut{}, st, &stats);
    }
}

static void search_local(const rabitq_index* idx, const float* Q, int64_t nq, int k, int nprobe, int M,
                         const rabitq_search_opts& o, int64_t* ids_d, float* dists_d, cudaStream_t st,
                         const float* Qd, bool trusted_probes = false) {
    (void)Q;
    rabitq::SearchCfg cfg;
    cfg.scan_path = o.scan_path;
    cfg.rank_key = o.rank_key;
    RQ_REQUIRE(o.rerank == 0 || (o.rerank == 1 && o.rank_key == RABITQ_RANK_EST), RABITQ_ERR_INVALID_ARGUMENT,
               "rerank must be 0 or 1 (1 requires rank_key EST)");
    cfg.rerank = o.rerank;
    RQ_REQUIRE(o.query_bits == 0 || o.query_bits == 4 || o.query_bits == 32, RABITQ_ERR_INVALID_ARGUMENT,
               "query_bits must be 0 (4), 4 or 32");
    cfg.full = o.query_bits == 32 ? 1 : 0;
    RQ_REQUIRE(!cfg.full || (o.scan_path != RABITQ_SCAN_POPC && idx->W <= 32), RABITQ_ERR_UNSUPPORTED,
               "query_bits 32 runs on the grouped tensor-core scan only (d <= 1024)");
    cfg.eps0 = o.eps0 > 0.0f ? o.eps0 : 1.9f;
    cfg.variant = o.variant;
    // the survivor buffer is cheap HBM (8 B/entry): size it so that overflow
    // re-scans are rare even when the seeded threshold is loose
    cfg.cap = o.cap_per_query > 0 ? o.cap_per_query : std::max(8192, 16 * M);
    // re-scans shrink the survivors by ~M/cap per round: keep cap >= 2M
    cfg.cap = std::max(cfg.cap, 2 * M);
    // threshold-seeding sample size: 0 -> auto per query (search.cu seed_kernel)
    cfg.seed_max = o.seed_max > 0 ? std::max(o.seed_max, M) : 0;
    RQ_REQUIRE(cfg.seed_max <= 49152, RABITQ_ERR_INVALID_ARGUMENT, "seed_max too large");
    {
        const char* rr = rabitq::rq_diag_env("RABITQ_REFINE_RANK");  // diagnostics: tensor-core threshold refinement pass
        cfg.refine_rank = rr ? atoi(rr) : 0;
    }

    const int D = idx->D, W = idx->W;
    // batch so that per-batch workspace stays bounded (~3 GiB)
    const int64_t per_q = (int64_t)cfg.cap * 8 + (int64_t)nprobe * (W * 16 + 16 + 8 + 8 + 4) + (int64_t)D * 8 +
                          (o.debug && o.debug->qbar ? (int64_t)nprobe * D : 0) + 64;
    const int64_t qbatch = std::max<int64_t>(1, std::min<int64_t>(nq, ((int64_t)3 << 30) / per_q));

    const rabitq_debug* dg = o.debug;
    DevView<uint8_t> v_qbar;
    DevView<int64_t> v_tids;
    DevView<float> v_test, v_tbnd;
    DevView<int32_t> v_sip;
    DevView<float> v_sest;
    if (dg) {
        v_qbar.init(dg->qbar, (size_t)nq * nprobe * D, idx->device, st);
        v_tids.init(dg->topm_ids, (size_t)nq * M, idx->device, st);
        v_test.init(dg->topm_est, (size_t)nq * M, idx->device, st);
        v_tbnd.init(dg->topm_bound, (size_t)nq * M, idx->device, st);
        if (dg->scan_ip) {
            RQ_REQUIRE(qbatch >= nq, RABITQ_ERR_INVALID_ARGUMENT, "scan dump needs a single internal batch");
            v_sip.init(dg->scan_ip, (size_t)dg->scan_dump_cap, idx->device, st);
            v_sest.init(dg->scan_est, (size_t)dg->scan_dump_cap, idx->device, st);
        }
    }
    // caller's probe lists (query-split probing): staged on the device once
    const bool pin_dev = o.probes_in && on_device(o.probes_in, idx->device);
    Stage sp(o.probes_in && !pin_dev ? (size_t)nq * nprobe * sizeof(int32_t) : 0, st);
    const int32_t* probes_d = o.probes_in;
    if (o.probes_in && !pin_dev) {
        RQ_CUDA(cudaMemcpyAsync(sp.p, o.probes_in, (size_t)nq * nprobe * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        probes_d = (const int32_t*)sp.p;
    }
    if (probes_d && !trusted_probes) rabitq::check_probes(probes_d, (int64_t)nq * nprobe, idx->nlist, st);
    if (o.graph && qbatch >= nq && !dg && !o.profile && o.rerank == 0 && !probes_d) {
        search_graph(idx, Qd, nq, k, nprobe, M, cfg, o.query_id_base, ids_d, dists_d, st);
        return;
    }
    rabitq::SearchStats stats;
    stats.timing = o.profile != nullptr;
    for (int64_t b0 = 0; b0 < nq; b0 += qbatch) {
        cfg.probes_in = probes_d ? probes_d + (size_t)b0 * nprobe : nullptr;
        const int64_t m = std::min(qbatch, nq - b0);
        rabitq::DebugOut dbg;
        if (dg) {
            if (dg->qrot) dbg.qrot = dg->qrot + (size_t)b0 * D;
            if (dg->probes) dbg.probes = dg->probes + (size_t)b0 * nprobe;
            if (v_qbar.dev) dbg.qbar = v_qbar.dev + (size_t)b0 * nprobe * D;
            if (dg->qscal) dbg.qscal = reinterpret_cast<float4*>(dg->qscal) + (size_t)b0 * nprobe;
            if (v_tids.dev) dbg.topm_ids = v_tids.dev + (size_t)b0 * M;
            if (v_test.dev) dbg.topm_est = v_test.dev + (size_t)b0 * M;
            if (v_tbnd.dev) dbg.topm_bound = v_tbnd.dev + (size_t)b0 * M;
            if (dg->tau) dbg.tau = dg->tau + b0;
            if (dg->survivors) dbg.survivors = dg->survivors + b0;
            if (v_sip.dev) {
                dbg.scan_ip = v_sip.dev;
                dbg.scan_est = v_sest.dev;
                dbg.scan_dump_cap = dg->scan_dump_cap;
            }
            if (dbg.topm_ids && !dbg.topm_est) {
                // topm_est is written together with topm_ids
                throw Error(RABITQ_ERR_INVALID_ARGUMENT, "debug.topm_ids requires debug.topm_est");
            }
        }
        rabitq::search_batch(idx, Qd + (size_t)b0 * D, m, k, nprobe, M, cfg, o.query_id_base + b0,
                             ids_d + (size_t)b0 * k, dists_d + (size_t)b0 * k, dbg, st, &stats);
    }
    if (o.profile) {
        rabitq_profile* pf = o.profile;
        std::memset(pf, 0, sizeof(*pf));
        for (int i = 0; i < RABITQ_NSTAGES; ++i) pf->stage_ms[i] = stats.stage_ms[i];
        pf->pairs = stats.pairs;
        pf->survivors = stats.survivors;
        pf->max_survivors = stats.max_survivors;
        pf->retries = stats.retries;
        pf->kernel_launches = stats.launches;
        pf->scan_path_used = stats.used_imma == 2 ? 3 : stats.used_imma ? 2 : 1;
        pf->batches = stats.batches;
        pf->reranked = stats.reranked;
        pf->dense_ms = stats.dense_ms;
    }
    if (dg) {
        v_qbar.copy_back(st);
        v_tids.copy_back(st);
        v_test.copy_back(st);
        v_tbnd.copy_back(st);
        v_sip.copy_back(st);
        v_sest.copy_back(st);
        if (dg->retries) {
            int r = stats.retries;
            RQ_CUDA(cudaMemcpyAsync(dg->retries, &r, sizeof(int), cudaMemcpyDefault, st));
        }
        RQ_CUDA(cudaStreamSynchronize(st));
    }
}

static void check_search_args(const rabitq_index* idx, const float* Q, int64_t nq, int32_t k, int32_t& nprobe,
                              int32_t n_rerank, const void* ids, const void* dists) {
    RQ_REQUIRE(idx != nullptr, RABITQ_ERR_INVALID_ARGUMENT, "index is NULL");
    RQ_REQUIRE(nq >= 0, RABITQ_ERR_INVALID_ARGUMENT, "nq < 0");
    RQ_REQUIRE(k >= 1, RABITQ_ERR_INVALID_ARGUMENT, "k < 1");
    RQ_REQUIRE(n_rerank >= k, RABITQ_ERR_INVALID_ARGUMENT, "n_rerank < k");
    RQ_REQUIRE(n_rerank <= 8192, RABITQ_ERR_INVALID_ARGUMENT, "n_rerank > 8192");
    RQ_REQUIRE(nprobe >= 0, RABITQ_ERR_INVALID_ARGUMENT, "nprobe < 0");
    if (nprobe == 0) nprobe = std::max(1, (int)std::ceil(0.05 * idx->nlist));  // AUTO
    RQ_REQUIRE(nprobe <= idx->nlist, RABITQ_ERR_INVALID_ARGUMENT, "nprobe > nlist");
    RQ_REQUIRE(nprobe <= 8192, RABITQ_ERR_INVALID_ARGUMENT, "nprobe > 8192");
    if (nq > 0) {
        RQ_REQUIRE(Q != nullptr && ids != nullptr && dists != nullptr, RABITQ_ERR_INVALID_ARGUMENT,
                   "Q / ids / dists is NULL");
    }
}

rabitq_status rabitq_search_ex(const rabitq_index* idx, const float* Q, int64_t nq, int32_t k, int32_t nprobe,
                               int32_t n_rerank, const rabitq_search_opts* opts, int64_t* ids, float* dists) {
    API_BEGIN
    NvtxScope nvtx_scope("rabitq:search");
    check_search_args(idx, Q, nq, k, nprobe, n_rerank, ids, dists);
    if (nq == 0) return RABITQ_OK;
    rabitq_search_opts o;
    rabitq_search_opts_default(&o);
    if (opts) o = *opts;
    RQ_CUDA(cudaSetDevice(idx->device));
    cudaStream_t st = o.stream ? (cudaStream_t)o.stream : idx->stream;
    const int D = idx->D;
    const bool q_dev = on_device(Q, idx->device);
    const bool i_dev = on_device(ids, idx->device), d_dev = on_device(dists, idx->device);
    Stage sq(q_dev ? 0 : (size_t)nq * D * sizeof(float), st);
    const float* Qd = Q;
    if (!q_dev) {
        RQ_CUDA(cudaMemcpyAsync(sq.p, Q, (size_t)nq * D * sizeof(float), cudaMemcpyHostToDevice, st));
        Qd = (const float*)sq.p;
    }
    Stage si(i_dev ? 0 : (size_t)nq * k * sizeof(int64_t), st), sd(d_dev ? 0 : (size_t)nq * k * sizeof(float), st);
    int64_t* ids_d = i_dev ? ids : (int64_t*)si.p;
    float* d_d = d_dev ? dists : (float*)sd.p;
    search_local(idx, Q, nq, k, nprobe, n_rerank, o, ids_d, d_d, st, Qd);
    if (!i_dev) RQ_CUDA(cudaMemcpyAsync(ids, ids_d, (size_t)nq * k * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (!d_dev) RQ_CUDA(cudaMemcpyAsync(dists, d_d, (size_t)nq * k * sizeof(float), cudaMemcpyDeviceToHost, st));
    if (!i_dev || !d_dev || !o.stream) RQ_CUDA(cudaStreamSynchronize(st));
    API_END
}

rabitq_status rabitq_index_info(const rabitq_index* idx, rabitq_index_info_t* out) {
    API_BEGIN
    RQ_REQUIRE(idx && out, RABITQ_ERR_INVALID_ARGUMENT, "NULL argument");
    std::memset(out, 0, sizeof(*out));
    out->d = idx->D;
    out->W = idx->W;
    out->nlist = idx->nlist;
    out->device = idx->device;
    out->n = idx->n;
    out->id_offset = idx->id_offset;
    out->max_list = idx->max_list;
    const int64_t slots = idx->nslots + 128;
    out->bytes_codes = slots * idx->W * 4;
    out->bytes_factors = slots * (8 + 4 + 4 + 4);
    out->bytes_ids = slots * 4 + idx->n * 4;
    out->bytes_vectors = idx->borrowed ? 0 : idx->n * idx->D * 4;
    out->bytes_codes8 = idx->codes8 ? slots * idx->W * 32 : 0;
    out->bytes_slot_vectors = idx->Xs ? slots * idx->D * 4 : 0;
    out->bytes_total = out->bytes_codes + out->bytes_factors + out->bytes_ids + out->bytes_vectors +
                       out->bytes_codes8 + out->bytes_slot_vectors +
                       (int64_t)idx->D * idx->D * 4 + (int64_t)idx->nlist * (idx->D + 1) * 4 +
                       (int64_t)(idx->nlist + 1) * 16;
    out->vectors_borrowed = idx->borrowed ? 1 : 0;
    API_END
}

rabitq_status rabitq_index_export(const rabitq_index* idx, rabitq_export_t* out) {
    API_BEGIN
    RQ_REQUIRE(idx && out, RABITQ_ERR_INVALID_ARGUMENT, "NULL argument");
    RQ_CUDA(cudaSetDevice(idx->device));
    cudaStream_t st = idx->stream;
    const int D = idx->D, W = idx->W;
    const int64_t n = idx->n;
    if (out->rotation) RQ_CUDA(cudaMemcpyAsync(out->rotation, idx->P, (size_t)D * D * 4, cudaMemcpyDefault, st));
    if (out->centroids)
        RQ_CUDA(cudaMemcpyAsync(out->centroids, idx->Cr, (size_t)idx->nlist * D * 4, cudaMemcpyDefault, st));
    if (out->list_off)
        RQ_CUDA(cudaMemcpyAsync(out->list_off, idx->list_off, (size_t)(idx->nlist + 1) * 8, cudaMemcpyDefault, st));
    if (out->codes || out->n_o || out->rho || out->ids) {
        Stage c(out->codes ? (size_t)n * W * 4 : 0, st), a(out->n_o ? (size_t)n * 4 : 0, st),
            r(out->rho ? (size_t)n * 4 : 0, st), i(out->ids ? (size_t)n * 8 : 0, st);
        const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
        export_kernel<<<grid, 256, 0, st>>>(n, W, idx->nlist, idx->list_off, idx->slot_off, idx->codes, idx->n_o,
                                            idx->rho, idx->rows, idx->id_offset, (uint32_t*)c.p, (float*)a.p,
                                            (float*)r.p, (int64_t*)i.p);
        RQ_CHECK_LAUNCH();
        if (out->codes) RQ_CUDA(cudaMemcpyAsync(out->codes, c.p, (size_t)n * W * 4, cudaMemcpyDefault, st));
        if (out->n_o) RQ_CUDA(cudaMemcpyAsync(out->n_o, a.p, (size_t)n * 4, cudaMemcpyDefault, st));
        if (out->rho) RQ_CUDA(cudaMemcpyAsync(out->rho, r.p, (size_t)n * 4, cudaMemcpyDefault, st));
        if (out->ids) RQ_CUDA(cudaMemcpyAsync(out->ids, i.p, (size_t)n * 8, cudaMemcpyDefault, st));
    }
    RQ_CUDA(cudaStreamSynchronize(st));
    API_END
}

rabitq_status rabitq_probe(const rabitq_index* idx, const float* Q, int64_t nq, int32_t nprobe, int32_t* probes,
                           void* stream) {
    API_BEGIN
    NvtxScope nvtx_scope("rabitq:probe");
    RQ_REQUIRE(idx != nullptr, RABITQ_ERR_INVALID_ARGUMENT, "index is NULL");
    RQ_REQUIRE(nq >= 0 && nprobe >= 0, RABITQ_ERR_INVALID_ARGUMENT, "nq < 0 or nprobe < 0");
    if (nprobe == 0) nprobe = std::max(1, (int)std::ceil(0.05 * idx->nlist));  // AUTO
    RQ_REQUIRE(nprobe <= idx->nlist, RABITQ_ERR_INVALID_ARGUMENT, "nprobe > nlist");
    if (nq == 0) return RABITQ_OK;
    RQ_REQUIRE(Q && probes, RABITQ_ERR_INVALID_ARGUMENT, "Q / probes is NULL");
    RQ_CUDA(cudaSetDevice(idx->device));
    cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
    const int D = idx->D;
    const bool q_dev = on_device(Q, idx->device), p_dev = on_device(probes, idx->device);
    Stage sq(q_dev ? 0 : (size_t)nq * D * 4, st), sp(p_dev ? 0 : (size_t)nq * nprobe * 4, st);
    const float* Qd = Q;
    if (!q_dev) {
        RQ_CUDA(cudaMemcpyAsync(sq.p, Q, (size_t)nq * D * 4, cudaMemcpyHostToDevice, st));
        Qd = (const float*)sq.p;
    }
    int32_t* pd = p_dev ? probes : (int32_t*)sp.p;
    rabitq::probe_only(idx, Qd, nq, nprobe, 0, pd, st);
    if (!p_dev) {
        RQ_CUDA(cudaMemcpyAsync(probes, pd, (size_t)nq * nprobe * 4, cudaMemcpyDeviceToHost, st));
        RQ_CUDA(cudaStreamSynchronize(st));
    }
    API_END
}

// ------------------------------------------------------------ multi-GPU --
rabitq_status rabitq_comm_unique_id(uint8_t uid[128]) {
    API_BEGIN
    RQ_REQUIRE(uid != nullptr, RABITQ_ERR_INVALID_ARGUMENT, "uid is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    RQ_REQUIRE(r == ncclSuccess, RABITQ_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(uid, &id, 128);
    API_END
}

rabitq_status rabitq_comm_init(const uint8_t uid[128], int32_t rank, int32_t world, int32_t device,
                               rabitq_comm** out) {
    API_BEGIN
    RQ_REQUIRE(uid && out, RABITQ_ERR_INVALID_ARGUMENT, "NULL argument");
    *out = nullptr;
    RQ_REQUIRE(world >= 1 && rank >= 0 && rank < world, RABITQ_ERR_INVALID_ARGUMENT, "bad rank/world");
    require_sm100(device);
    RQ_CUDA(cudaSetDevice(device));
    std::unique_ptr<rabitq_comm> c(new rabitq_comm());
    c->rank = rank;
    c->world = world;
    c->device = device;
    ncclUniqueId id;
    std::memcpy(&id, uid, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    RQ_REQUIRE(r == ncclSuccess, RABITQ_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    *out = c.release();
    API_END
}

void rabitq_comm_free(rabitq_comm* comm) {
    if (!comm) return;
    if (comm->comm) ncclCommDestroy(comm->comm);
    delete comm;
}

rabitq_status rabitq_search_sharded(const rabitq_index* shard, rabitq_comm* comm, const float* Q, int64_t nq,
                                    int32_t k, int32_t nprobe, int32_t n_rerank, const rabitq_search_opts* opts,
                                    int64_t* ids, float* dists) {
    API_BEGIN
    NvtxScope nvtx_scope("rabitq:search_sharded");
    check_search_args(shard, Q, nq, k, nprobe, n_rerank, ids, dists);
    RQ_REQUIRE(comm != nullptr, RABITQ_ERR_INVALID_ARGUMENT, "comm is NULL");
    RQ_REQUIRE(comm->device == shard->device, RABITQ_ERR_INVALID_ARGUMENT, "comm and shard on different devices");
    if (nq == 0) return RABITQ_OK;
    rabitq_search_opts o;
    rabitq_search_opts_default(&o);
    if (opts) o = *opts;
    RQ_CUDA(cudaSetDevice(shard->device));
    cudaStream_t st = o.stream ? (cudaStream_t)o.stream : shard->stream;
    const int D = shard->D, G = comm->world;
    const bool q_dev = on_device(Q, shard->device);
    Stage sq(q_dev ? 0 : (size_t)nq * D * 4, st);
    const float* Qd = Q;
    if (!q_dev) {
        RQ_CUDA(cudaMemcpyAsync(sq.p, Q, (size_t)nq * D * 4, cudaMemcpyHostToDevice, st));
        Qd = (const float*)sq.p;
    }
    const size_t nk = (size_t)nq * k;
    Stage li(nk * 8, st), ld(nk * 4, st), gi(nk * G * 8, st), gd(nk * G * 4, st), oi(nk * 8, st), od(nk * 4, st);
    Stage pr, pg;
    if (o.query_split && G > 1 && !o.probes_in) {
        // query-split probing: rank g probes its c = ceil(nq / G)
        // queries, then one all-gather of the [G c x nprobe] probe lists
        const int64_t c = (nq + G - 1) / G, lo = std::min<int64_t>(nq, (int64_t)comm->rank * c);
        const int64_t m = std::min<int64_t>(c, nq - lo);
        pr = Stage((size_t)c * nprobe * sizeof(int32_t), st);
        pg = Stage((size_t)G * c * nprobe * sizeof(int32_t), st);
        if (m > 0) rabitq::probe_only(shard, Qd + (size_t)lo * D, m, nprobe, o.variant, (int32_t*)pr.p, st);
        ncclResult_t r = ncclAllGather(pr.p, pg.p, (size_t)c * nprobe, ncclInt32, comm->comm, st);
        RQ_REQUIRE(r == ncclSuccess, RABITQ_ERR_NCCL, std::string("ncclAllGather (probes): ") + ncclGetErrorString(r));
        o.probes_in = (const int32_t*)pg.p;
    }
    search_local(shard, Q, nq, k, nprobe, n_rerank, o, (int64_t*)li.p, (float*)ld.p, st, Qd,
                 /*trusted_probes=*/o.query_split && G > 1 && !(opts && opts->probes_in));
    // the one exchange step: all-gather of the per-rank top-k over NVLink
    ncclResult_t r = ncclGroupStart();
    if (r == ncclSuccess) r = ncclAllGather(li.p, gi.p, nk, ncclInt64, comm->comm, st);
    if (r == ncclSuccess) r = ncclAllGather(ld.p, gd.p, nk, ncclFloat32, comm->comm, st);
    if (r == ncclSuccess) r = ncclGroupEnd();
    RQ_REQUIRE(r == ncclSuccess, RABITQ_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    rabitq::merge_topk((const int64_t*)gi.p, (const float*)gd.p, G, nq, k, (int64_t*)oi.p, (float*)od.p, st);
    RQ_CUDA(cudaMemcpyAsync(ids, oi.p, nk * 8, cudaMemcpyDefault, st));
    RQ_CUDA(cudaMemcpyAsync(dists, od.p, nk * 4, cudaMemcpyDefault, st));
    RQ_CUDA(cudaStreamSynchronize(st));
    API_END
}

rabitq_status rabitq_merge_topk(const int64_t* in_ids, const float* in_d, int32_t G, int64_t nq, int32_t k,
                                int64_t* out_ids, float* out_d, void* stream) {
    API_BEGIN
    RQ_REQUIRE(G >= 1 && k >= 1 && nq >= 0, RABITQ_ERR_INVALID_ARGUMENT, "bad sizes");
    if (nq == 0) return RABITQ_OK;
    RQ_REQUIRE(in_ids && in_d && out_ids && out_d, RABITQ_ERR_INVALID_ARGUMENT, "NULL argument");
    const int dev = current_device();
    RQ_REQUIRE(on_device(in_ids, dev) && on_device(in_d, dev) && on_device(out_ids, dev) && on_device(out_d, dev),
               RABITQ_ERR_INVALID_ARGUMENT, "merge_topk takes device pointers");
    rabitq::merge_topk(in_ids, in_d, G, nq, k, out_ids, out_d, (cudaStream_t)stream);
    API_END
}

}  // extern "C"
