// The reference API's energy helpers on caller-held arrays (energy.hpp:77-116
// evaluate_energy, :363-378 alignment_weights / regularization_weights), on
// the device: one thread per point, directed pair or node, and fixed-order
// two-level sums (CTA tree, then one CTA over the CTA partials), so the sums
// are reproducible run to run. Inside register_surfaces the same quantities
// come from terms_kernel on resident data; these entries serve callers that
// use the lower-level API (the reference's tests do).
#include <cmath>
#include <vector>

#include "device_common.cuh"
#include "errors.hpp"
#include "nrr_cuda.h"

namespace nrr_b200 {
namespace {

constexpr int kT = 256, kBlocks = 148;

__device__ __forceinline__ double welsch_sq_d(double x2, double nu) { return 1.0 - exp(-x2 / (2.0 * nu * nu)); }
__device__ __forceinline__ double welsch_w_d(double y2, double nu) {
    const double two_nu2 = 2.0 * nu * nu;
    return exp(-y2 / two_nu2) / two_nu2;
}

struct TermsIn {
    int n = 0, N = 0, P = 0;
    const double *deformed = nullptr, *corr = nullptr, *sqdist = nullptr;
    const double *X = nullptr, *node_pos = nullptr, *reg_w = nullptr, *R = nullptr;
    const int* pairs = nullptr;
    double nu_a = 1, nu_r = 1, alpha = 0;
    double *w_align = nullptr, *w_reg = nullptr;
};

// X is the reference 4N x 3 column-major block: A_j(c, r) = X[(4j+r) + 4N c],
// t_j(c) = X[(4j+3) + 4N c] (deformation_graph.hpp:17-38)
__device__ __forceinline__ double xa(const TermsIn& t, int j, int r, int c) { return t.X[4 * j + r + 4 * t.N * c]; }

// partial[b * 3 + {0,1,2}] = this CTA's sums of the align / reg / rot terms
__global__ void __launch_bounds__(kT) terms_api_kernel(TermsIn t, double* __restrict__ partial) {
    __shared__ double sh[kT / 32];
    double s_align = 0.0, s_reg = 0.0, s_rot = 0.0;
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < t.n; i += stride) {
        if (t.w_align && t.sqdist) t.w_align[i] = welsch_w_d(t.sqdist[i], t.nu_a);  // energy.hpp:363-368
        if (t.deformed) {
            double d2 = 0.0;
            for (int c = 0; c < 3; ++c) {
                const double d = t.deformed[3 * i + c] - t.corr[3 * i + c];
                d2 += d * d;
            }
            s_align += welsch_sq_d(d2, t.nu_a);  // energy.hpp:105
        }
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < t.P; e += stride) {
        // reg_difference (energy.hpp:77-84): c (A_j (p_i - p_j) + p_j + t_j - p_i - t_i)
        const int i = t.pairs[2 * e], j = t.pairs[2 * e + 1];
        const double cw = t.reg_w[e];
        double d[3], d2 = 0.0;
        for (int r = 0; r < 3; ++r) d[r] = t.node_pos[3 * i + r] - t.node_pos[3 * j + r];
        for (int c = 0; c < 3; ++c) {
            double v = 0.0;
            for (int r = 0; r < 3; ++r) v += xa(t, j, r, c) * d[r];
            v = cw * (v + t.node_pos[3 * j + c] + xa(t, j, 3, c) - t.node_pos[3 * i + c] - xa(t, i, 3, c));
            d2 += v * v;
        }
        if (t.w_reg) t.w_reg[e] = t.alpha * welsch_w_d(d2, t.nu_r);  // energy.hpp:371-378
        s_reg += welsch_sq_d(d2, t.nu_r);                             // energy.hpp:106-107
    }
    if (t.R)
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < t.N; j += stride) {
            double s = 0.0;  // |A_j - R_j|_F^2 (energy.hpp:108-110)
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) {
                    const double v = xa(t, j, c, r) - t.R[9 * j + 3 * r + c];
                    s += v * v;
                }
            s_rot += s;
        }
    const double a = block_sum(s_align, sh), b = block_sum(s_reg, sh), c = block_sum(s_rot, sh);
    if (threadIdx.x == 0) {
        partial[3 * blockIdx.x] = a;
        partial[3 * blockIdx.x + 1] = b;
        partial[3 * blockIdx.x + 2] = c;
    }
}

__global__ void terms_final_kernel(const double* __restrict__ partial, int nb, double* __restrict__ out3) {
    __shared__ double sh[kT / 32];
    for (int q = 0; q < 3; ++q) {
        double v = 0.0;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) v += partial[3 * b + q];
        v = block_sum(v, sh);
        if (threadIdx.x == 0) out3[q] = v;
    }
}

template <typename T>
struct Buf {
    T* p = nullptr;
    explicit Buf(size_t n) { NRR_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~Buf() {
        if (p) cudaFree(p);
    }
    T* up(const T* h, size_t n, cudaStream_t s) {
        if (h && n) NRR_CUDA_CHECK(cudaMemcpyAsync(p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
        return h ? p : nullptr;
    }
};

}  // namespace

void energy_terms(cudaStream_t s, const nrr_energy_terms_in* in, double* out_w_align, double* out_w_reg,
                  double* out_sums3) {
    const int n = in->n, N = in->node_count, P = in->pair_count;
    if (n < 0 || N < 0 || P < 0) throw ConfigError("energy terms: negative sizes");
    Buf<double> def(3 * static_cast<size_t>(n)), cor(3 * static_cast<size_t>(n)), sq(n), X(12 * static_cast<size_t>(N)),
        pos(3 * static_cast<size_t>(N)), rw(P), R(9 * static_cast<size_t>(N)), wa(n), wr(P), part(3 * kBlocks), out(3);
    Buf<int> pr(2 * static_cast<size_t>(P));
    TermsIn t;
    t.n = n;
    t.N = N;
    t.P = P;
    t.deformed = def.up(in->deformed, 3 * static_cast<size_t>(n), s);
    t.corr = cor.up(in->corr_points, 3 * static_cast<size_t>(n), s);
    if (t.deformed && !t.corr) throw ConfigError("energy terms: deformed points need correspondences");
    t.sqdist = sq.up(in->corr_sqdist, n, s);
    t.X = X.up(in->X, 12 * static_cast<size_t>(N), s);
    t.node_pos = pos.up(in->node_positions, 3 * static_cast<size_t>(N), s);
    t.reg_w = rw.up(in->reg_weights, P, s);
    t.pairs = pr.up(in->reg_pairs, 2 * static_cast<size_t>(P), s);
    t.R = R.up(in->rotations, 9 * static_cast<size_t>(N), s);
    if (P > 0 && (!t.X || !t.node_pos || !t.reg_w || !t.pairs))
        throw ConfigError("energy terms: pair terms need X, node positions, pairs and weights");
    if (t.R && !t.X) throw ConfigError("energy terms: rotation terms need X");
    t.nu_a = in->nu_a;
    t.nu_r = in->nu_r;
    t.alpha = in->alpha;
    t.w_align = out_w_align ? wa.p : nullptr;
    t.w_reg = out_w_reg ? wr.p : nullptr;
    terms_api_kernel<<<kBlocks, kT, 0, s>>>(t, part.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    terms_final_kernel<<<1, kT, 0, s>>>(part.p, kBlocks, out.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    if (out_w_align) NRR_CUDA_CHECK(cudaMemcpyAsync(out_w_align, wa.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out_w_reg) NRR_CUDA_CHECK(cudaMemcpyAsync(out_w_reg, wr.p, P * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out_sums3) NRR_CUDA_CHECK(cudaMemcpyAsync(out_sums3, out.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace nrr_b200
