// Per-node 3x3 rotation projection (reference rotation.hpp:14-24,
// energy.hpp:47-56) for one thread: one-sided (Hestenes) Jacobi SVD in FP64.
//
// One-sided Jacobi orthogonalises the columns of W = A V by plane rotations;
// on exit sigma_i = |w_i| with high relative accuracy, so the degenerate test
// sigma_min < 1e-12 (energy.hpp:53) sees the true smallest singular value.
// R = u1 v1^T + u2 v2^T + s u3 v3^T with u3 = u1 x u2 and s = det(V): this is
// the reference's U diag(1,1,sign det(U V^T)) V^T written without forming the
// sign-ambiguous third left vector, and always has det R = +1.
#pragma once

#include <cuda_runtime.h>

namespace nrr_b200 {

// a: row-major 3x3 (a[r*3+c]); out_r: row-major rotation
__host__ __device__ inline void project_rotation3(const double a[9], double out_r[9], double* sigma_min) {
    double w[9], v[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
#pragma unroll
    for (int k = 0; k < 9; ++k) w[k] = a[k];
    // columns p,q; up to 12 sweeps (3x3 converges in ~4-6)
    for (int sweep = 0; sweep < 12; ++sweep) {
        bool rotated = false;
#pragma unroll
        for (int pair = 0; pair < 3; ++pair) {
            const int p = pair == 2 ? 1 : 0;
            const int q = pair == 0 ? 1 : 2;
            double al = 0, be = 0, ga = 0;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                al += w[r * 3 + p] * w[r * 3 + p];
                be += w[r * 3 + q] * w[r * 3 + q];
                ga += w[r * 3 + p] * w[r * 3 + q];
            }
            if (ga == 0.0 || fabs(ga) <= 2.2e-16 * sqrt(al * be)) continue;
            rotated = true;
            const double zeta = (be - al) / (2.0 * ga);
            const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const double wp = w[r * 3 + p], wq = w[r * 3 + q];
                w[r * 3 + p] = c * wp - s * wq;
                w[r * 3 + q] = s * wp + c * wq;
                const double vp = v[r * 3 + p], vq = v[r * 3 + q];
                v[r * 3 + p] = c * vp - s * vq;
                v[r * 3 + q] = s * vp + c * vq;
            }
        }
        if (!rotated) break;
    }
    double sg[3];
    int idx[3] = {0, 1, 2};
#pragma unroll
    for (int k = 0; k < 3; ++k) sg[k] = sqrt(w[k] * w[k] + w[3 + k] * w[3 + k] + w[6 + k] * w[6 + k]);
    // sort descending (stable)
    if (sg[idx[1]] > sg[idx[0]]) { const int t = idx[0]; idx[0] = idx[1]; idx[1] = t; }
    if (sg[idx[2]] > sg[idx[1]]) { const int t = idx[1]; idx[1] = idx[2]; idx[2] = t; }
    if (sg[idx[1]] > sg[idx[0]]) { const int t = idx[0]; idx[0] = idx[1]; idx[1] = t; }
    if (sigma_min) *sigma_min = sg[idx[2]];
    double V[3][3], U[3][3];  // V[k] = k-th right vector (sorted)
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int r = 0; r < 3; ++r) V[k][r] = v[r * 3 + idx[k]];
    const double s0 = sg[idx[0]], s1 = sg[idx[1]];
    if (!(s0 > 0.0)) {  // zero matrix: Jacobi leaves V = I, so R = I
#pragma unroll
        for (int k = 0; k < 9; ++k) out_r[k] = (k % 4 == 0) ? 1.0 : 0.0;
        return;
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) U[0][r] = w[r * 3 + idx[0]] / s0;
    if (s1 > 1e-300 && s1 > 1e-15 * s0) {
#pragma unroll
        for (int r = 0; r < 3; ++r) U[1][r] = w[r * 3 + idx[1]] / s1;
        // re-orthogonalise against u1 (rank-deficient inputs)
        const double d = U[1][0] * U[0][0] + U[1][1] * U[0][1] + U[1][2] * U[0][2];
        double nn = 0;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            U[1][r] -= d * U[0][r];
            nn += U[1][r] * U[1][r];
        }
        nn = 1.0 / sqrt(nn);
#pragma unroll
        for (int r = 0; r < 3; ++r) U[1][r] *= nn;
    } else {  // rank 1: any unit vector orthogonal to u1 gives a minimiser
        const int ax = (fabs(U[0][0]) <= fabs(U[0][1]) && fabs(U[0][0]) <= fabs(U[0][2])) ? 0
                       : (fabs(U[0][1]) <= fabs(U[0][2]))                                  ? 1
                                                                                            : 2;
        double e[3] = {0, 0, 0};
        e[ax] = 1.0;
        double c[3] = {U[0][1] * e[2] - U[0][2] * e[1], U[0][2] * e[0] - U[0][0] * e[2], U[0][0] * e[1] - U[0][1] * e[0]};
        const double nn = 1.0 / sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
#pragma unroll
        for (int r = 0; r < 3; ++r) U[1][r] = c[r] * nn;
    }
    U[2][0] = U[0][1] * U[1][2] - U[0][2] * U[1][1];
    U[2][1] = U[0][2] * U[1][0] - U[0][0] * U[1][2];
    U[2][2] = U[0][0] * U[1][1] - U[0][1] * U[1][0];
    const double detv = V[0][0] * (V[1][1] * V[2][2] - V[1][2] * V[2][1]) -
                        V[0][1] * (V[1][0] * V[2][2] - V[1][2] * V[2][0]) +
                        V[0][2] * (V[1][0] * V[2][1] - V[1][1] * V[2][0]);
    const double s = detv < 0 ? -1.0 : 1.0;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            out_r[r * 3 + c] = U[0][r] * V[0][c] + U[1][r] * V[1][c] + s * U[2][r] * V[2][c];
}

}  // namespace nrr_b200
