// index.cuh -- the in-HBM layout of an IVF-RaBitQ index.
//
//   list j holds the vectors assigned to centroid j, ids
//   ascending.  Its vectors occupy SLOTS [slot_off[j], slot_off[j] + size_j),
//   slot_off[j] a multiple of 32.  Codes are stored in blocks of 32 slots,
//   word-interleaved: word w of slot s is codes[((s / 32) * W + w) * 32 + s % 32],
//   so a warp reading word w of 32 consecutive slots issues one 128-byte
//   coalesced load; a 128-slot tile is 128 * W * 4 contiguous bytes.
//   Pad slots have code 0, factors 0 and row kPadRow.
#pragma once
#include <vector>

#include "common.cuh"

struct rabitq_index {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;   // search: the re-rank ordering + dense block overlap the scan on it
    int D = 0, W = 0, nlist = 0;
    int64_t n = 0, id_offset = 0, nslots = 0, max_list = 0;
    int64_t tiles8_sum = 0;        // sum over lists of ceil(ceil(size / 128) / 8) (grouped-scan item bound)
    uint64_t seed = 0;

    float* P = nullptr;            // [D x D] row-major, x' = P^T x
    float* Pt = nullptr;           // [D x D] P^T row-major (tensor-core rotation operand)
    float* Cr = nullptr;           // [nlist x D] rotated centroids c'
    float* cnorm = nullptr;        // [nlist] ||c'||^2
    int64_t* list_off = nullptr;   // [nlist + 1] list boundaries in list order (rank of vector)
    int64_t* slot_off = nullptr;   // [nlist + 1] 32-aligned slot starts
    uint32_t* codes = nullptr;     // [nslots / 32][W][32]
    bool codes8_f8 = false;        // codes8 bytes are e4m3 {0, -1.0} (D <= 128) rather than s8 {0, -1}
    uint8_t* codes8 = nullptr;     // [nslots + 128][32 W] the codes as s8 {0, -1} in the grouped scan's K
                                   // order (scan_imma.cu expand32), slot-major: its A operand by TMA;
                                   // nullable (built when it fits)
    float2* fac = nullptr;         // [nslots] {n_o^2, 2 n_o / (rho sqrt(D))}
    uint16_t* pcnt = nullptr;      // [nslots] popcount of the code (grouped scan epilogue)
    float* list_amax = nullptr;    // [nlist] max n_o^2 of each list (grouped scan fast-test margin)
    float* g1 = nullptr;           // [nslots] 2 n_o sqrt(1 - rho^2) / (rho sqrt(D - 1))  (bound / (eps0 n_q))
    float* n_o = nullptr;          // [nslots]
    float* rho = nullptr;          // [nslots]
    uint32_t* rows = nullptr;      // [nslots] local row id, kPadRow for pad slots
    uint32_t* slot_of_row = nullptr;  // [n] inverse of rows (debug capture of bounds)
    const float* X = nullptr;      // [n x D] fp32 vectors for the exact re-rank (local rows)
    float* Xs = nullptr;           // [nslots + 128 x D] the same vectors in slot (list) order, minus their
                                   // list centroid (original space), pad slots 0; nullable (built when it
                                   // fits; dense re-rank)
    float* Corig = nullptr;        // [nlist x D] centroids in the original space (c = P c'), with Xs
    float* X_owned = nullptr;
    bool borrowed = false;

    std::vector<int64_t> h_list_off, h_slot_off;
    void* graphs = nullptr;        // capi.cu: cache of captured latency-mode search graphs (NEXT-2)
};

namespace rabitq {
void build_index(rabitq_index* idx, const float* X, int64_t n, int D, int nlist, uint64_t seed,
                 const rabitq_build_opts& o);
void free_index_memory(rabitq_index* idx);
}  // namespace rabitq
