// haar.cpp -- host-side generation of the random orthogonal rotation P
// ("random orthogonal rotation P"; R#5).
//
// A seeded D x D standard-normal matrix G (Philox4x32-10 + Box-Muller) is
// orthonormalised column by column with modified Gram-Schmidt, applied twice
// per column ("twice is enough"), which yields the QR factor with a positive
// diagonal of R -- the Haar-distributed orthogonal matrix.  fp64 throughout,
// rounded to fp32 once at the end.  Build-time only (D <= a few thousand).
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace rabitq {

void haar_rotation_host(int D, uint64_t seed, float* P) {
    const uint32_t k0 = (uint32_t)seed ^ 0x48414152u /* 'HAAR' */, k1 = (uint32_t)(seed >> 32);
    // column-major G: G[j][i] = entry (row i, column j); pairs of normals per Philox call
    std::vector<double> Q((size_t)D * D);
    const size_t total = (size_t)D * D;
    for (size_t e = 0; e < total; e += 4) {
        U4 w = philox4x32_10(k0, k1, U4{(uint32_t)(e >> 2), (uint32_t)(e >> 34), 0u, 0x524F54u});
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        for (int h = 0; h < 4; h += 2) {
            const double u1 = ((ws[h] >> 8) + 0.5) * (1.0 / 16777216.0);
            const double u2 = ((ws[h + 1] >> 8) + 0.5) * (1.0 / 16777216.0);
            const double rad = std::sqrt(-2.0 * std::log(u1));
            const double z0 = rad * std::cos(6.283185307179586 * u2);
            const double z1 = rad * std::sin(6.283185307179586 * u2);
            if (e + h < total) Q[e + h] = z0;
            if (e + h + 1 < total) Q[e + h + 1] = z1;
        }
    }
    // Q holds columns contiguously: column j = Q[j*D .. j*D + D)
    for (int j = 0; j < D; ++j) {
        double* qj = &Q[(size_t)j * D];
        for (int pass = 0; pass < 2; ++pass) {
            for (int p = 0; p < j; ++p) {
                const double* qp = &Q[(size_t)p * D];
                double dot = 0.0;
                for (int i = 0; i < D; ++i) dot += qp[i] * qj[i];
                for (int i = 0; i < D; ++i) qj[i] -= dot * qp[i];
            }
        }
        double nrm = 0.0;
        for (int i = 0; i < D; ++i) nrm += qj[i] * qj[i];
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) throw Error(RABITQ_ERR_INTERNAL, "haar_rotation: rank-deficient Gaussian draw");
        for (int i = 0; i < D; ++i) qj[i] /= nrm;  // R_jj = nrm > 0
    }
    // P row-major: P[i][j] = column j, row i
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) P[(size_t)i * D + j] = (float)Q[(size_t)j * D + i];
}

}  // namespace rabitq
