// tgemm.cuh -- 3xTF32 tensor-core GEMM C = A B^T (tgemm.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rabitq {

enum { TG_EPI_STORE = 0, TG_EPI_PROBE = 1, TG_EPI_DIST = 2, TG_EPI_ARGMIN = 3 };

// one output tile of a batched product: A rows [a0, a0 + m), B rows [b0, b0 + n)
// (through a_idx / b_idx when given), output at C + c0 with leading dimension ldc
struct TgTile {
    int64_t a0, b0, c0;
    int32_t m, n, ldc, pad;
};

struct TgParams {
    const float* A;          // rows of K floats, stride lda
    int64_t lda;
    const uint32_t* a_idx;   // nullable: A row of tile row r = a_idx[a0 + r]
    const float* B;
    int64_t ldb;
    const uint32_t* b_idx;   // nullable
    int K;
    const TgTile* tiles;     // nullable: plain M x N tiling (128 x 256 tiles, row-major C)
    int ntiles;
    int64_t M, N;            // plain mode
    float* C;
    int64_t ldc;             // plain mode
    const float* b_norm;     // PROBE / ARGMIN: ||c||^2 per B row; DIST: ||q||^2 per (gathered) B row id
    unsigned long long* amin;  // ARGMIN: [M] running min of (orderable(||c||^2 - 2 a.c) << 32 | B row), plain mode
};

// STORE: C = A B^T (row-major tile); PROBE: C = b_norm[col] - 2 A B^T;
// DIST: C[col * ldc + row] = max(0, ||a_row||^2 + b_norm[b id] - 2 a.b) (column-major tile);
// ARGMIN: amin[row] = min(amin[row], key(b_norm[col] - 2 a.b, col)) over the tile's columns
// (k-means / list assignment: nearest centroid, ties -> lowest id; no distance matrix written)
void tgemm(const TgParams& p, int epi, cudaStream_t st);
// dense re-rank block, 1xTF32 fed by TMA (plain A / B rows, p.tiles):
// C[c0 + col ldc + row] = a_norm[a row]^2 + b_norm[b row] - 2 a.b, |error| <= 2^-8 (a_norm^2 + b_norm)
void tgemm_dist1(const TgParams& p, const float* a_norm, cudaStream_t st);

}  // namespace rabitq
