// ORACLE — TEST INFRASTRUCTURE ONLY. Nothing in the product path may include,
// link or call anything under oracle/. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg use it, as the checker.
//
// CPU restatement of the dense small-matrix arithmetic the reference takes
// from Eigen (absent in this image, so bit-level agreement with an Eigen build
// is unpinned; parity is pinned by the reference's KATs and properties):
//   * 3x3 two-sided Jacobi SVD        (Eigen::JacobiSVD, rotation.hpp:17)
//   * 3x3 symmetric Jacobi eigen       (SelfAdjointEigenSolver, deformation_graph.hpp:87)
//   * column-pivoted Householder QR    (ColPivHouseholderQR, anderson.hpp:37)
//   * pivoted dense LDLT               (MatrixXd::ldlt, anderson.hpp:43)
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------- errors
// common.hpp:14-26
struct IoError : std::runtime_error {
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};

// ---------------------------------------------------------------- Vec3 / Mat3
struct Vec3 {
    double x = 0, y = 0, z = 0;
    Vec3() = default;
    Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
    double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
    Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
    Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
    Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
    Vec3 operator/(double s) const { return {x / s, y / s, z / s}; }
    Vec3& operator+=(const Vec3& o) { x += o.x; y += o.y; z += o.z; return *this; }
    double squaredNorm() const { return x * x + y * y + z * z; }
    double norm() const { return std::sqrt(squaredNorm()); }
    double dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
    bool finite() const { return std::isfinite(x) && std::isfinite(y) && std::isfinite(z); }
};
inline Vec3 operator*(double s, const Vec3& v) { return v * s; }
inline Vec3 cwiseMin(const Vec3& a, const Vec3& b) {
    return {std::min(a.x, b.x), std::min(a.y, b.y), std::min(a.z, b.z)};
}
inline Vec3 cwiseMax(const Vec3& a, const Vec3& b) {
    return {std::max(a.x, b.x), std::max(a.y, b.y), std::max(a.z, b.z)};
}

// row-major 3x3: m[r*3+c]
struct Mat3 {
    double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    static Mat3 identity() {
        Mat3 a;
        a.m[0] = a.m[4] = a.m[8] = 1.0;
        return a;
    }
    double& operator()(int r, int c) { return m[r * 3 + c]; }
    double operator()(int r, int c) const { return m[r * 3 + c]; }
    Vec3 operator*(const Vec3& v) const {
        return {m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
                m[6] * v.x + m[7] * v.y + m[8] * v.z};
    }
    Mat3 operator*(const Mat3& o) const {
        Mat3 r;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += (*this)(i, k) * o(k, j);
                r(i, j) = s;
            }
        return r;
    }
    Mat3 transpose() const {
        Mat3 r;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) r(i, j) = (*this)(j, i);
        return r;
    }
    double determinant() const {
        return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
               m[2] * (m[3] * m[7] - m[4] * m[6]);
    }
    bool finite() const {
        for (double v : m)
            if (!std::isfinite(v)) return false;
        return true;
    }
};

// ------------------------------------------------------- Jacobi rotations
// Plane rotation J = [c s; -s c] acting like Eigen::JacobiRotation<double>.
struct Rot {
    double c = 1, s = 0;
    Rot transpose() const { return {c, -s}; }
    Rot operator*(const Rot& o) const { return {c * o.c - s * o.s, c * o.s + s * o.c}; }
};

// Symmetric 2x2 diagonalizing rotation of [[x,y],[y,z]] (Eigen makeJacobi).
inline Rot make_jacobi(double x, double y, double z) {
    Rot r;
    const double deno = 2.0 * std::abs(y);
    if (deno < std::numeric_limits<double>::min()) {
        r.c = 1.0;
        r.s = 0.0;
    } else {
        const double tau = (x - z) / deno;
        const double w = std::sqrt(tau * tau + 1.0);
        const double t = tau > 0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
        const double sign_t = t > 0 ? 1.0 : -1.0;
        const double n = 1.0 / std::sqrt(t * t + 1.0);
        r.s = -sign_t * (y / std::abs(y)) * std::abs(t) * n;
        r.c = n;
    }
    return r;
}

// rows p,q of a (n x n, row-major, ld=n): x' = c x + s y ; y' = -s x + c y
inline void apply_left(double* a, int n, int p, int q, const Rot& j) {
    for (int k = 0; k < n; ++k) {
        const double x = a[p * n + k], y = a[q * n + k];
        a[p * n + k] = j.c * x + j.s * y;
        a[q * n + k] = -j.s * x + j.c * y;
    }
}
// columns p,q of a by j^T applied as Eigen's applyOnTheRight(p,q,j)
inline void apply_right(double* a, int n, int p, int q, const Rot& j) {
    const Rot t = j.transpose();
    for (int k = 0; k < n; ++k) {
        const double x = a[k * n + p], y = a[k * n + q];
        a[k * n + p] = t.c * x + t.s * y;
        a[k * n + q] = -t.s * x + t.c * y;
    }
}

// 2x2 real SVD step of the two-sided Jacobi SVD (Eigen real_2x2_jacobi_svd).
inline void real_2x2_jacobi_svd(const double* w, int n, int p, int q, Rot& j_left,
                                Rot& j_right) {
    double m[4] = {w[p * n + p], w[p * n + q], w[q * n + p], w[q * n + q]};
    Rot rot1;
    const double t = m[0] + m[3];
    const double d = m[2] - m[1];
    if (std::abs(d) < std::numeric_limits<double>::min()) {
        rot1.s = 0.0;
        rot1.c = 1.0;
    } else {
        const double u = t / d;
        const double tmp = std::sqrt(1.0 + u * u);
        rot1.s = 1.0 / tmp;
        rot1.c = u / tmp;
    }
    apply_left(m, 2, 0, 1, rot1);
    j_right = make_jacobi(m[0], m[1], m[3]);
    j_left = rot1 * j_right.transpose();
}

/// Full SVD of a 3x3 matrix by two-sided Jacobi sweeps: a = U diag(s) V^T,
/// singular values sorted descending (restates Eigen::JacobiSVD as used at
/// reference rotation.hpp:17).
inline void jacobi_svd3(const Mat3& a, Mat3& u, double s[3], Mat3& v) {
    double scale = 0.0;
    for (double x : a.m) scale = std::max(scale, std::abs(x));
    if (!std::isfinite(scale)) throw NumericalError("jacobi_svd3: non-finite input");
    if (scale == 0.0) scale = 1.0;
    double w[9];
    for (int i = 0; i < 9; ++i) w[i] = a.m[i] / scale;
    double U[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    const double consider_zero = std::numeric_limits<double>::min();
    const double precision = 2.0 * std::numeric_limits<double>::epsilon();
    double max_diag = std::max(std::abs(w[0]), std::max(std::abs(w[4]), std::abs(w[8])));
    bool finished = false;
    int sweeps = 0;
    while (!finished && sweeps < 100) {
        finished = true;
        ++sweeps;
        for (int p = 1; p < 3; ++p) {
            for (int q = 0; q < p; ++q) {
                const double threshold = std::max(consider_zero, precision * max_diag);
                if (std::max(std::abs(w[p * 3 + q]), std::abs(w[q * 3 + p])) > threshold) {
                    finished = false;
                    Rot jl, jr;
                    real_2x2_jacobi_svd(w, 3, p, q, jl, jr);
                    apply_left(w, 3, p, q, jl);
                    apply_right(U, 3, p, q, jl.transpose());
                    apply_right(w, 3, p, q, jr);
                    apply_right(V, 3, p, q, jr);
                    max_diag = std::max(max_diag,
                                        std::max(std::abs(w[p * 3 + p]), std::abs(w[q * 3 + q])));
                }
            }
        }
    }
    double sv[3];
    for (int i = 0; i < 3; ++i) {
        const double d = w[i * 3 + i];
        sv[i] = std::abs(d);
        if (d < 0)
            for (int r = 0; r < 3; ++r) U[r * 3 + i] = -U[r * 3 + i];
    }
    // selection sort descending, swapping columns
    for (int i = 0; i < 3; ++i) {
        int best = i;
        for (int k = i + 1; k < 3; ++k)
            if (sv[k] > sv[best]) best = k;
        if (best != i) {
            std::swap(sv[i], sv[best]);
            for (int r = 0; r < 3; ++r) {
                std::swap(U[r * 3 + i], U[r * 3 + best]);
                std::swap(V[r * 3 + i], V[r * 3 + best]);
            }
        }
    }
    for (int i = 0; i < 9; ++i) {
        u.m[i] = U[i];
        v.m[i] = V[i];
    }
    for (int i = 0; i < 3; ++i) s[i] = sv[i] * scale;
}

/// rotation.hpp:14-24 — R = U diag(1,1,sign det(UV^T)) V^T, sigma_min = s[2].
inline Mat3 project_to_rotation(const Mat3& a, double* sigma_min = nullptr) {
    if (!a.finite()) throw NumericalError("project_to_rotation: non-finite input matrix");
    Mat3 u, v;
    double s[3];
    jacobi_svd3(a, u, s, v);
    if (sigma_min) *sigma_min = s[2];
    double sign3 = 1.0;
    if ((u * v.transpose()).determinant() < 0.0) sign3 = -1.0;
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r(i, j) = u(i, 0) * v(j, 0) + u(i, 1) * v(j, 1) + sign3 * u(i, 2) * v(j, 2);
    return r;
}

/// Symmetric eigen-decomposition of a small dense matrix (n<=4) by cyclic
/// Jacobi; eigenvalues ascending, eigenvectors in the columns of `vecs`
/// (row-major n x n). Stands in for SelfAdjointEigenSolver
/// (deformation_graph.hpp:87, energy.hpp:335).
inline void sym_eigen(const double* a_in, int n, double* evals, double* vecs) {
    double a[16], v[16];
    for (int i = 0; i < n * n; ++i) a[i] = a_in[i];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) v[i * n + j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                (i == j ? diag : off) += a[i * n + j] * a[i * n + j];
        if (off <= 1e-300 || off <= (std::numeric_limits<double>::epsilon() *
                                     std::numeric_limits<double>::epsilon()) * diag * 1e-4)
            break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                if (a[p * n + q] == 0.0) continue;
                const Rot j = make_jacobi(a[p * n + p], a[p * n + q], a[q * n + q]);
                // a <- J^T a J  (Eigen: applyOnTheLeft(p,q,j.adjoint()); applyOnTheRight(p,q,j))
                apply_left(a, n, p, q, j.transpose());
                apply_right(a, n, p, q, j);
                apply_right(v, n, p, q, j);
            }
    }
    int idx[4] = {0, 1, 2, 3};
    std::sort(idx, idx + n, [&](int x, int y) { return a[x * n + x] < a[y * n + y]; });
    for (int k = 0; k < n; ++k) {
        evals[k] = a[idx[k] * n + idx[k]];
        for (int r = 0; r < n; ++r) vecs[r * n + k] = v[r * n + idx[k]];
    }
}

// ------------------------------------------------ column-pivoted Householder QR
/// Restates Eigen::ColPivHouseholderQR on a dense column-major (rows x cols)
/// matrix, as used by anderson.hpp:37-38 (rank test) and :39 (solve).
struct ColPivQR {
    int rows = 0, cols = 0;
    std::vector<double> qr;      // column-major, R in the upper triangle
    std::vector<double> hcoeffs;  // tau per reflector
    std::vector<int> perm;        // column permutation: perm[k] = original column
    int nonzero_pivots = 0;
    double maxpivot = 0.0;

    ColPivQR(const std::vector<double>& a, int r, int c) : rows(r), cols(c), qr(a) {
        const int size = std::min(rows, cols);
        hcoeffs.assign(size, 0.0);
        std::vector<double> norms_upd(cols), norms_dir(cols);
        std::vector<int> transpositions(size);
        for (int k = 0; k < cols; ++k) {
            double s = 0;
            for (int i = 0; i < rows; ++i) s += at(i, k) * at(i, k);
            norms_dir[k] = norms_upd[k] = std::sqrt(s);
        }
        double max_norm = 0;
        for (double x : norms_upd) max_norm = std::max(max_norm, x);
        const double eps = std::numeric_limits<double>::epsilon();
        const double threshold_helper = (max_norm * eps) * (max_norm * eps) / rows;
        const double norm_downdate_threshold = std::sqrt(eps);
        nonzero_pivots = size;
        maxpivot = 0.0;
        for (int k = 0; k < size; ++k) {
            int biggest = k;
            for (int j = k + 1; j < cols; ++j)
                if (norms_upd[j] > norms_upd[biggest]) biggest = j;
            const double biggest_sq = norms_upd[biggest] * norms_upd[biggest];
            if (nonzero_pivots == size && biggest_sq < threshold_helper * (rows - k))
                nonzero_pivots = k;
            transpositions[k] = biggest;
            if (k != biggest) {
                for (int i = 0; i < rows; ++i) std::swap(at(i, k), at(i, biggest));
                std::swap(norms_upd[k], norms_upd[biggest]);
                std::swap(norms_dir[k], norms_dir[biggest]);
            }
            // Householder of column k, rows k..
            double tail_sq = 0;
            for (int i = k + 1; i < rows; ++i) tail_sq += at(i, k) * at(i, k);
            const double c0 = at(k, k);
            double tau, beta;
            if (tail_sq <= std::numeric_limits<double>::min()) {
                tau = 0.0;
                beta = c0;
                for (int i = k + 1; i < rows; ++i) at(i, k) = 0.0;
            } else {
                beta = std::sqrt(c0 * c0 + tail_sq);
                if (c0 >= 0) beta = -beta;
                for (int i = k + 1; i < rows; ++i) at(i, k) /= (c0 - beta);
                tau = (beta - c0) / beta;
            }
            at(k, k) = beta;
            hcoeffs[k] = tau;
            if (std::abs(beta) > maxpivot) maxpivot = std::abs(beta);
            // apply H = I - tau [1;v][1;v]^T to columns k+1..
            for (int j = k + 1; j < cols; ++j) {
                double tmp = at(k, j);
                for (int i = k + 1; i < rows; ++i) tmp += at(i, k) * at(i, j);
                at(k, j) -= tau * tmp;
                for (int i = k + 1; i < rows; ++i) at(i, j) -= tau * at(i, k) * tmp;
            }
            for (int j = k + 1; j < cols; ++j) {
                if (norms_upd[j] != 0.0) {
                    double temp = std::abs(at(k, j)) / norms_upd[j];
                    temp = (1.0 + temp) * (1.0 - temp);
                    temp = temp < 0 ? 0 : temp;
                    const double r = norms_upd[j] / norms_dir[j];
                    const double temp2 = temp * r * r;
                    if (temp2 <= norm_downdate_threshold) {
                        double s = 0;
                        for (int i = k + 1; i < rows; ++i) s += at(i, j) * at(i, j);
                        norms_dir[j] = norms_upd[j] = std::sqrt(s);
                    } else {
                        norms_upd[j] *= std::sqrt(temp);
                    }
                }
            }
        }
        perm.resize(cols);
        for (int k = 0; k < cols; ++k) perm[k] = k;
        for (int k = 0; k < size; ++k) std::swap(perm[k], perm[transpositions[k]]);
    }
    double& at(int i, int j) { return qr[static_cast<size_t>(j) * rows + i]; }
    double at(int i, int j) const { return qr[static_cast<size_t>(j) * rows + i]; }

    int rank() const {
        const double thr = maxpivot * std::numeric_limits<double>::epsilon() *
                           static_cast<double>(std::min(rows, cols));
        int r = 0;
        for (int i = 0; i < nonzero_pivots; ++i) r += std::abs(at(i, i)) > thr ? 1 : 0;
        return r;
    }

    std::vector<double> solve(const std::vector<double>& b) const {
        std::vector<double> c(b);
        const int size = std::min(rows, cols);
        for (int k = 0; k < size; ++k) {  // c <- Q^T c
            const double tau = hcoeffs[k];
            double tmp = c[k];
            for (int i = k + 1; i < rows; ++i) tmp += at(i, k) * c[i];
            c[k] -= tau * tmp;
            for (int i = k + 1; i < rows; ++i) c[i] -= tau * at(i, k) * tmp;
        }
        const int nz = nonzero_pivots;
        std::vector<double> y(nz);
        for (int i = nz - 1; i >= 0; --i) {
            double s = c[i];
            for (int j = i + 1; j < nz; ++j) s -= at(i, j) * y[j];
            y[i] = s / at(i, i);
        }
        std::vector<double> x(cols, 0.0);
        for (int i = 0; i < nz; ++i) x[perm[i]] = y[i];
        return x;
    }
};

/// Dense LDLT with symmetric pivoting (stands in for MatrixXd::ldlt(),
/// anderson.hpp:43); a is row-major n x n symmetric.
inline std::vector<double> ldlt_solve(std::vector<double> a, int n, std::vector<double> b) {
    std::vector<int> p(n);
    for (int i = 0; i < n; ++i) p[i] = i;
    for (int k = 0; k < n; ++k) {
        int best = k;
        for (int i = k + 1; i < n; ++i)
            if (std::abs(a[i * n + i]) > std::abs(a[best * n + best])) best = i;
        if (best != k) {
            for (int j = 0; j < n; ++j) std::swap(a[k * n + j], a[best * n + j]);
            for (int j = 0; j < n; ++j) std::swap(a[j * n + k], a[j * n + best]);
            std::swap(p[k], p[best]);
        }
        const double d = a[k * n + k];
        if (d == 0.0) continue;
        std::vector<double> col(n);
        for (int i = k + 1; i < n; ++i) col[i] = a[i * n + k];
        for (int i = k + 1; i < n; ++i) {
            const double l = col[i] / d;
            for (int j = k + 1; j < n; ++j) a[i * n + j] -= l * col[j];
            a[i * n + k] = l;
            a[k * n + i] = l;
        }
    }
    std::vector<double> y(n);
    for (int i = 0; i < n; ++i) y[i] = b[p[i]];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) y[i] -= a[i * n + j] * y[j];
    for (int i = 0; i < n; ++i) y[i] = a[i * n + i] != 0.0 ? y[i] / a[i * n + i] : 0.0;
    for (int i = n - 1; i >= 0; --i)
        for (int j = i + 1; j < n; ++j) y[i] -= a[j * n + i] * y[j];
    std::vector<double> x(n);
    for (int i = 0; i < n; ++i) x[p[i]] = y[i];
    return x;
}

}  // namespace oracle
