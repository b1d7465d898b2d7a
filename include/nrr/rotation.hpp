// Rotation projection (reference rotation.hpp:14-24) on the device: one-sided
// Jacobi SVD, R = U diag(1,1,sign det(UV^T)) V^T (csrc/svd3.cuh).
#pragma once

#include "nrr/common.hpp"

namespace nrr {

inline Mat3 project_to_rotation(const Mat3& a, double* sigma_min = nullptr) {
    if (!a.allFinite()) throw NumericalError("project_to_rotation: non-finite input matrix");
    // one node: X rows r<3 hold A^T (column-major 4 x 3)
    double X[12] = {0};
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) X[c * 4 + r] = a(c, r);
    double R[9], smin = 0.0;
    int32_t deg = 0;
    detail::check(nrr_project_rotations_sigma(detail::default_context(), X, 1, R, &smin, &deg));
    Mat3 out;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out(r, c) = R[r * 3 + c];
    if (sigma_min) *sigma_min = smin;  // the smallest singular value (rotation.hpp:21)
    return out;
}

}  // namespace nrr
