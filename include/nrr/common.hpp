// Drop-in C++ API of the B200 registration hot path (mirrors the reference's
// proj/include/nrr/common.hpp:10-28). Eigen is not available in this image, so
// Vec3 / Mat3 / MatrixX are small value types with the subset of the Eigen
// interface the reference API and its callers use; storage is column-major
// like Eigen's, so NodeTransforms::stacked.data() is exactly the reference
// 4N x 3 layout passed through the C ABI (include/nrr_cuda.h).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "nrr_cuda.h"

namespace nrr {

struct Vec3 {
    double v[3] = {0, 0, 0};
    Vec3() = default;
    Vec3(double x, double y, double z) : v{x, y, z} {}
    static Vec3 Zero() { return {}; }
    static Vec3 UnitX() { return {1, 0, 0}; }
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
    double& operator()(int i) { return v[i]; }
    double operator()(int i) const { return v[i]; }
    double x() const { return v[0]; }
    double y() const { return v[1]; }
    double z() const { return v[2]; }
    Vec3 operator+(const Vec3& o) const { return {v[0] + o.v[0], v[1] + o.v[1], v[2] + o.v[2]}; }
    Vec3 operator-(const Vec3& o) const { return {v[0] - o.v[0], v[1] - o.v[1], v[2] - o.v[2]}; }
    Vec3 operator-() const { return {-v[0], -v[1], -v[2]}; }
    Vec3 operator*(double s) const { return {v[0] * s, v[1] * s, v[2] * s}; }
    Vec3 operator/(double s) const { return {v[0] / s, v[1] / s, v[2] / s}; }
    Vec3& operator+=(const Vec3& o) {
        for (int i = 0; i < 3; ++i) v[i] += o.v[i];
        return *this;
    }
    Vec3& operator-=(const Vec3& o) {
        for (int i = 0; i < 3; ++i) v[i] -= o.v[i];
        return *this;
    }
    double dot(const Vec3& o) const { return v[0] * o.v[0] + v[1] * o.v[1] + v[2] * o.v[2]; }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }
    Vec3 normalized() const { return *this / norm(); }
    Vec3 cwiseMin(const Vec3& o) const { return {std::min(v[0], o.v[0]), std::min(v[1], o.v[1]), std::min(v[2], o.v[2])}; }
    Vec3 cwiseMax(const Vec3& o) const { return {std::max(v[0], o.v[0]), std::max(v[1], o.v[1]), std::max(v[2], o.v[2])}; }
    bool allFinite() const { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }
    bool operator==(const Vec3& o) const { return v[0] == o.v[0] && v[1] == o.v[1] && v[2] == o.v[2]; }
};
inline Vec3 operator*(double s, const Vec3& a) { return a * s; }

// 3x3, column-major storage (Eigen::Matrix3d)
struct Mat3 {
    double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    static Mat3 Zero() { return {}; }
    static Mat3 Identity() {
        Mat3 a;
        a(0, 0) = a(1, 1) = a(2, 2) = 1.0;
        return a;
    }
    double& operator()(int r, int c) { return m[c * 3 + r]; }
    double operator()(int r, int c) const { return m[c * 3 + r]; }
    Vec3 operator*(const Vec3& x) const {
        Vec3 y;
        for (int r = 0; r < 3; ++r) y[r] = (*this)(r, 0) * x[0] + (*this)(r, 1) * x[1] + (*this)(r, 2) * x[2];
        return y;
    }
    Mat3 operator*(const Mat3& o) const {
        Mat3 p;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                for (int k = 0; k < 3; ++k) p(r, c) += (*this)(r, k) * o(k, c);
        return p;
    }
    Mat3 operator*(double s) const {
        Mat3 p = *this;
        for (double& x : p.m) x *= s;
        return p;
    }
    Mat3 operator-(const Mat3& o) const {
        Mat3 p;
        for (int k = 0; k < 9; ++k) p.m[k] = m[k] - o.m[k];
        return p;
    }
    Mat3 transpose() const {
        Mat3 t;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) t(r, c) = (*this)(c, r);
        return t;
    }
    double determinant() const {
        const Mat3& a = *this;
        return a(0, 0) * (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) - a(0, 1) * (a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0)) +
               a(0, 2) * (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0));
    }
    double squaredNorm() const {
        double s = 0;
        for (double x : m) s += x * x;
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    bool allFinite() const {
        for (double x : m)
            if (!std::isfinite(x)) return false;
        return true;
    }
};
inline Mat3 operator*(double s, const Mat3& a) { return a * s; }

// dense column-major matrix (Eigen::MatrixXd subset)
struct MatrixX {
    int r = 0, c = 0;
    std::vector<double> d;
    MatrixX() = default;
    MatrixX(int rows, int cols) : r(rows), c(cols), d(static_cast<size_t>(rows) * cols, 0.0) {}
    void setZero(int rows, int cols) {
        r = rows;
        c = cols;
        d.assign(static_cast<size_t>(rows) * cols, 0.0);
    }
    int rows() const { return r; }
    int cols() const { return c; }
    double& operator()(int i, int j) { return d[static_cast<size_t>(j) * r + i]; }
    double operator()(int i, int j) const { return d[static_cast<size_t>(j) * r + i]; }
    double* data() { return d.data(); }
    const double* data() const { return d.data(); }
    size_t size() const { return d.size(); }
    bool allFinite() const {
        for (double x : d)
            if (!std::isfinite(x)) return false;
        return true;
    }
};
using VectorX = std::vector<double>;

// compressed sparse column matrix (Eigen::SparseMatrix<double> subset the
// reference API and its tests use: rows/cols/nonZeros/coeff, the raw arrays,
// transpose, difference, Frobenius norm, products with dense matrices,
// conversion to dense)
struct SparseMatrix {
    int r = 0, c = 0;
    std::vector<int> outer{0};  // c + 1 column starts
    std::vector<int> inner;     // row indices, ascending per column
    std::vector<double> val;
    SparseMatrix() = default;
    SparseMatrix(int rows, int cols) : r(rows), c(cols), outer(static_cast<size_t>(cols) + 1, 0) {}
    int rows() const { return r; }
    int cols() const { return c; }
    int nonZeros() const { return static_cast<int>(val.size()); }
    double* valuePtr() { return val.data(); }
    const double* valuePtr() const { return val.data(); }
    const int* outerIndexPtr() const { return outer.data(); }
    const int* innerIndexPtr() const { return inner.data(); }
    double coeff(int i, int j) const {
        const auto b = inner.begin() + outer[j], e = inner.begin() + outer[j + 1];
        const auto it = std::lower_bound(b, e, i);
        return it != e && *it == i ? val[static_cast<size_t>(it - inner.begin())] : 0.0;
    }
    SparseMatrix transpose() const {
        SparseMatrix t(c, r);
        t.inner.resize(inner.size());
        t.val.resize(val.size());
        for (int i : inner) ++t.outer[i + 1];
        for (int i = 0; i < r; ++i) t.outer[i + 1] += t.outer[i];
        std::vector<int> pos(t.outer.begin(), t.outer.end() - 1);
        for (int j = 0; j < c; ++j)
            for (int k = outer[j]; k < outer[j + 1]; ++k) {
                const int q = pos[inner[k]]++;
                t.inner[q] = j;
                t.val[q] = val[k];
            }
        return t;
    }
    MatrixX toDense() const {
        MatrixX d(r, c);
        for (int j = 0; j < c; ++j)
            for (int k = outer[j]; k < outer[j + 1]; ++k) d(inner[k], j) = val[k];
        return d;
    }
    SparseMatrix operator-(const SparseMatrix& o) const {  // union pattern, explicit zeros kept
        SparseMatrix d(r, c);
        for (int j = 0; j < c; ++j) {
            int a = outer[j], b = o.outer[j];
            while (a < outer[j + 1] || b < o.outer[j + 1]) {
                const int ia = a < outer[j + 1] ? inner[a] : r, ib = b < o.outer[j + 1] ? o.inner[b] : r;
                const int i = std::min(ia, ib);
                d.inner.push_back(i);
                d.val.push_back((ia == i ? val[a++] : 0.0) - (ib == i ? o.val[b++] : 0.0));
            }
            d.outer[j + 1] = static_cast<int>(d.inner.size());
        }
        return d;
    }
    double norm() const {
        double s = 0.0;
        for (double v : val) s += v * v;
        return std::sqrt(s);
    }
    MatrixX operator*(const MatrixX& x) const {
        MatrixX y(r, x.cols());
        for (int q = 0; q < x.cols(); ++q)
            for (int j = 0; j < c; ++j) {
                const double xj = x(j, q);
                for (int k = outer[j]; k < outer[j + 1]; ++k) y(inner[k], q) += val[k] * xj;
            }
        return y;
    }
};

/// File could not be read or written, or its contents are malformed (common.hpp:14-16).
struct IoError : std::runtime_error {
    explicit IoError(const std::string& msg) : std::runtime_error(msg) {}
};
/// An option or input parameter is outside its documented range (common.hpp:19-21).
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& msg) : std::runtime_error(msg) {}
};
/// A numerical operation failed (common.hpp:24-26).
struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& msg) : std::runtime_error(msg) {}
};
/// The device path failed (no B200, CUDA error). The reference has no device.
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& msg) : std::runtime_error(msg) {}
};

inline bool finite(const Vec3& v) { return v.allFinite(); }

namespace detail {
// C-ABI status -> the reference's exception classes (nrr_cli.cpp:266-278)
inline void check(int rc) {
    if (rc == NRR_OK) return;
    const std::string msg = nrr_last_error();
    switch (rc) {
        case NRR_ERR_IO:
            throw IoError(msg);
        case NRR_ERR_NUMERICAL:
            throw NumericalError(msg);
        case NRR_ERR_CONFIG:
            throw ConfigError(msg);
        default:
            throw DeviceError(msg);
    }
}

// RAII handle of one device context (all buffers of one registration)
class Context {
public:
    explicit Context(int device = 0) { check(nrr_ctx_create(device, &ctx_)); }
    ~Context() {
        if (ctx_) nrr_ctx_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    Context(Context&& o) noexcept : ctx_(o.ctx_) { o.ctx_ = nullptr; }
    nrr_ctx* get() const { return ctx_; }

private:
    nrr_ctx* ctx_ = nullptr;
};

// Setup entry points (knn_edges, build_graph) run on the B200 when one is
// visible (bitwise equal to the host build) and on the host
// otherwise; NRR_SETUP_HOST=1 forces the host build.
inline bool setup_on_device() {
    static const bool on = [] {
        const char* e = std::getenv("NRR_SETUP_HOST");
        if (e && *e == '1') return false;
        int32_t c = 0;
        return nrr_device_count(&c) == NRR_OK && c > 0;
    }();
    return on;
}

// per-thread device context for the stateless free functions (the reference
// functions are pure; the device path keeps one context per host thread)
inline nrr_ctx* default_context() {
    thread_local Context ctx(0);
    return ctx.get();
}

inline std::vector<double> flat(const std::vector<Vec3>& pts) {
    std::vector<double> f(pts.size() * 3);
    for (size_t i = 0; i < pts.size(); ++i)
        for (int k = 0; k < 3; ++k) f[3 * i + k] = pts[i][k];
    return f;
}
inline std::vector<Vec3> unflat(const double* f, size_t n) {
    std::vector<Vec3> pts(n);
    for (size_t i = 0; i < n; ++i) pts[i] = Vec3(f[3 * i], f[3 * i + 1], f[3 * i + 2]);
    return pts;
}
}  // namespace detail

}  // namespace nrr
