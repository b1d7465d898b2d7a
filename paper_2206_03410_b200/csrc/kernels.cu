// Per-iteration kernels of the Welsch-MM hot path on sm_100a (FP64):
//   deform_kernel    deform_points + max displacement   (deformation_graph.hpp:225-245,
//                                                         solver.hpp:274-278)
//   terms_kernel     Welsch weights + energy terms + rotation projection
//                    (energy.hpp:47-56, 92-116, 363-378)
//   energy_reduce    fixed-order final energy sums       (energy.hpp:110)
//   assemble_kernel  K values and B of the fixed pattern (energy.hpp:182-228)
//   aa_*             Anderson acceleration window        (anderson.hpp:22-73)
//
// Determinism (reference README.md:181-182): no floating-point atomics decide
// any value. Energies use fixed-size grids and fixed reduction trees; each K/B
// entry is summed by one lane in contributor (vertex) order.
#include <cmath>
#include <cstdlib>

#include "device_common.cuh"
#include "kernels.cuh"
#include "svd3.cuh"

namespace nrr_b200 {

namespace {

// ---------------------------------------------------------------- deform
__global__ void __launch_bounds__(256) deform_kernel(DevProblem p, const double* __restrict__ x,
                                                     double* __restrict__ out, const double* __restrict__ old,
                                                     double* __restrict__ max_disp, int* __restrict__ nonfinite) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double disp = 0.0;
    bool bad = false;
    if (i < p.n) {
        const double vx = p.src[3 * i], vy = p.src[3 * i + 1], vz = p.src[3 * i + 2];
        double ax = 0, ay = 0, az = 0;
        for (int k = p.infl_off[i]; k < p.infl_off[i + 1]; ++k) {
            const int a = p.infl_node[k];
            const double w = p.infl_w[k];
            const double* pa = p.node_pos + 3 * a;
            const double* xa = x + 12 * a;  // rows r: A(c, r) = xa[3r + c]; t = xa[9..11]
            const double dx = vx - pa[0], dy = vy - pa[1], dz = vz - pa[2];
            // w * (A (v - p) + (p + t))   (deformation_graph.hpp:238-240)
            const double ox = xa[0] * dx + xa[3] * dy + xa[6] * dz + (pa[0] + xa[9]);
            const double oy = xa[1] * dx + xa[4] * dy + xa[7] * dz + (pa[1] + xa[10]);
            const double oz = xa[2] * dx + xa[5] * dy + xa[8] * dz + (pa[2] + xa[11]);
            ax += w * ox;
            ay += w * oy;
            az += w * oz;
        }
        out[3 * i] = ax;
        out[3 * i + 1] = ay;
        out[3 * i + 2] = az;
        bad = !isfinite(ax + ay + az);
        if (old) {
            const double ex = ax - old[3 * i], ey = ay - old[3 * i + 1], ez = az - old[3 * i + 2];
            disp = sqrt(ex * ex + ey * ey + ez * ez);
        }
    }
    // one global atomic per block (max is exact in any order): a per-warp
    // atomic on one address serialised ~31K updates at 1M vertices
    __shared__ double s_max[8];
    if (max_disp) {
        disp = warp_max(disp);
        if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = disp;
    }
    const int any_bad = __syncthreads_or(bad ? 1 : 0);
    if (threadIdx.x == 0) {
        if (max_disp) {
            double m = s_max[0];
            for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, s_max[w]);
            if (m > 0.0) atomic_max_nonneg(max_disp, m);
        }
        if (nonfinite && any_bad) atomicOr(nonfinite, 1);
    }
}

// ---------------------------------------------------------------- terms
// Items [0,n) vertices, [n,n+N) nodes, [n+N,n+N+P) directed pairs.
__global__ void __launch_bounds__(kTermThreads) terms_kernel(DevProblem p, const double* __restrict__ x,
                                                             const double* __restrict__ d2, TermParams tp,
                                                             double* __restrict__ wa, double* __restrict__ wr,
                                                             double* __restrict__ R, double* __restrict__ partials,
                                                             int* __restrict__ degenerate) {
    __shared__ double sh[kTermThreads / 32];
    double e_align = 0.0, e_reg = 0.0, e_rot = 0.0;
    int deg = 0;
    const int total = p.n + p.N + p.P;
    const double two_na2 = 2.0 * tp.nu_a * tp.nu_a;
    const double two_nr2 = 2.0 * tp.nu_r * tp.nu_r;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < total; it += gridDim.x * blockDim.x) {
        if (it < p.n) {
            const double v = d2[it];
            // E_align term: welsch_sq(|v_hat - u|^2, nu_a) (energy.hpp:105)
            e_align += 1.0 - exp(-v / two_na2);
            // weight from corr.squared_distance = sqrt(d2)^2 (kd_tree.hpp:37, energy.hpp:39)
            const double dist = sqrt(v);
            const double sd = dist * dist;
            wa[it] = exp(-sd / two_na2) / two_na2;
        } else if (it < p.n + p.N) {
            const int j = it - p.n;
            const double* xj = x + 12 * j;
            double a[9];  // row-major A(c, r) = X(4j+r, c)
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int r = 0; r < 3; ++r) a[c * 3 + r] = xj[3 * r + c];
            double rot[9], smin = 0.0;
            project_rotation3(a, rot, &smin);
            if (smin < 1e-12) ++deg;
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const double d = a[k] - rot[k];
                s += d * d;
                R[9 * j + k] = rot[k];
            }
            e_rot += s;
        } else {
            const int e = it - p.n - p.N;
            const int i = p.pairs[2 * e], j = p.pairs[2 * e + 1];
            const double c = p.pair_c[e];
            const double* pi = p.node_pos + 3 * i;
            const double* pj = p.node_pos + 3 * j;
            const double* xi = x + 12 * i;
            const double* xj = x + 12 * j;
            const double ux = pi[0] - pj[0], uy = pi[1] - pj[1], uz = pi[2] - pj[2];
            // c (A_j (p_i - p_j) + p_j + t_j - p_i - t_i)   (energy.hpp:77-84)
            double D[3];
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const double ad = xj[cc] * ux + xj[3 + cc] * uy + xj[6 + cc] * uz;
                D[cc] = c * ((((ad + pj[cc]) + xj[9 + cc]) - pi[cc]) - xi[9 + cc]);
            }
            const double dd = D[0] * D[0] + D[1] * D[1] + D[2] * D[2];
            e_reg += 1.0 - exp(-dd / two_nr2);
            wr[e] = tp.alpha * (exp(-dd / two_nr2) / two_nr2);
        }
    }
    e_align = block_sum(e_align, sh);
    e_reg = block_sum(e_reg, sh);
    e_rot = block_sum(e_rot, sh);
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x] = e_align;
        partials[3 * blockIdx.x + 1] = e_reg;
        partials[3 * blockIdx.x + 2] = e_rot;
    }
    if (deg) atomicAdd(degenerate, deg);  // integer: order-independent
}

__global__ void __launch_bounds__(256) energy_reduce_kernel(DevProblem p, const double* __restrict__ partials,
                                                            TermParams tp, const double* __restrict__ vhat,
                                                            PassRecord* __restrict__ rec, int nblocks) {
    __shared__ double sh[8];
    double v[3] = {0, 0, 0};
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
        for (int k = 0; k < 3; ++k) v[k] += partials[3 * b + k];
    for (int k = 0; k < 3; ++k) v[k] = block_sum(v[k], sh);
    if (threadIdx.x == 0) {
        rec->align = v[0];
        rec->reg = v[1];
        rec->rot = v[2];
        rec->total = v[0] + tp.alpha * v[1] + tp.beta * v[2];  // energy.hpp:110
        double lm = 0.0;  // solver.hpp:203-208
        if (tp.lm_weight != 0.0)
            for (int l = 0; l < p.landmarks; ++l) {
                const int i = p.lm_vertex[l];
                const double dx = vhat[3 * i] - p.lm_pos[3 * l], dy = vhat[3 * i + 1] - p.lm_pos[3 * l + 1],
                             dz = vhat[3 * i + 2] - p.lm_pos[3 * l + 2];
                lm += dx * dx + dy * dy + dz * dz;
            }
        rec->landmark = lm;
        if (!isfinite(rec->total + tp.lm_weight * lm)) rec->nonfinite |= 2;
    }
}

__global__ void rotations_kernel(const double* __restrict__ x, int N, double* __restrict__ R, int* degenerate,
                                 double* __restrict__ sigma_min) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const double* xj = x + 12 * j;
    double a[9];
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) a[c * 3 + r] = xj[3 * r + c];
    double rot[9], smin = 0.0;
    project_rotation3(a, rot, &smin);
    for (int k = 0; k < 9; ++k) R[9 * j + k] = rot[k];
    if (sigma_min) sigma_min[j] = smin;
    if (smin < 1e-12) atomicAdd(degenerate, 1);
}

// ---------------------------------------------------------------- assembly
// One warp per upper block. Lanes first gather up to 32 contributors' operands
// into shared memory (coalesced index loads, 32 independent gathers in
// flight), then each output entry is owned by one lane that sums the staged
// products in contributor order. Diagonal warps: lanes 0-15 K_jj, 16-27 B_j.
// Edge warps: lanes 0-15 K_ab (written to (a,b) and mirrored to (b,a), so K
// is bitwise symmetric as the reference's mirrored program makes it).
constexpr int kAsmWarps = 8;

__device__ __forceinline__ double gcomp(const double4& g, int r) { return r == 0 ? g.x : r == 1 ? g.y : r == 2 ? g.z : g.w; }
__device__ __forceinline__ double pair_g(const DevProblem& p, int e, int r) {
    // g_e = c [p_i - p_j; 1]  (energy.hpp:163-173), precomputed per problem
    return gcomp(p.pair_gv[e], r);
}

// Warp transpose-reduce: 32 per-lane values -> lane l holds the warp sum of
// slot l. Every butterfly level halves the vector a lane carries (16 + 8 + 4
// + 2 + 1 shuffles instead of 32 x 5). Fixed order: deterministic.
__device__ __forceinline__ double transpose_reduce32(const double (&v)[32]) {
    const int lane = threadIdx.x & 31;
    double v16[16], v8[8], v4[4], v2[2];
    {
        const bool up = lane & 16;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const double keep = up ? v[i + 16] : v[i], send = up ? v[i] : v[i + 16];
            v16[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
    }
    {
        const bool up = lane & 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double keep = up ? v16[i + 8] : v16[i], send = up ? v16[i] : v16[i + 8];
            v8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
    }
    {
        const bool up = lane & 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double keep = up ? v8[i + 4] : v8[i], send = up ? v8[i] : v8[i + 4];
            v4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
    }
    {
        const bool up = lane & 2;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double keep = up ? v4[i + 2] : v4[i], send = up ? v4[i] : v4[i + 2];
            v2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
    }
    const bool up = lane & 1;
    const double keep = up ? v2[1] : v2[0], send = up ? v2[0] : v2[1];
    return keep + __shfl_xor_sync(0xffffffffu, send, 1);
}

// One warp per upper 4x4 block u of K (diagonal block of node u < N, or the
// (a,b) block of edge u - N) and, for diagonal blocks, the node's 4x3 rows of
// B (energy.hpp:182-228). Lane l accumulates the products of contributors
// l, l+32, ... (and, on diagonal blocks, of the node's directed pair l) into
// 28 slots (K[r][s] at 4r+s, B[r][s] at 16+3r+s); one transpose-reduce then
// leaves slot l's total in lane l. Fixed order: deterministic; both mirrored
// halves of an edge block are written from the same value (K bitwise
// symmetric, robust_energy_tests.cpp:185-196).
__global__ void __launch_bounds__(kAsmWarps * 32) assemble_kernel(DevProblem p, const double* __restrict__ wa,
                                                                  const double* __restrict__ q,
                                                                  const double* __restrict__ wr,
                                                                  const double* __restrict__ R, TermParams tp,
                                                                  double* __restrict__ K, double* __restrict__ B) {
    if (p.skip != nullptr && *p.skip) return;
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int u = blockIdx.x * kAsmWarps + wib;
    if (u >= p.U) return;
    const bool diag = u < p.N;
    const int cb = p.ub_cptr[u], ce = p.ub_cptr[u + 1];
    double v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.0;
    for (int t = cb + lane; t < ce; t += 32) {
        const int vtx = p.c_v[t];
        const double4 fa = p.c_fa[t];
        const double w = wa[vtx];
        const double a4[4] = {fa.x, fa.y, fa.z, fa.w};
        if (diag) {
            const double q3[3] = {q[3 * vtx], q[3 * vtx + 1], q[3 * vtx + 2]};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
#pragma unroll
                for (int c = 0; c < 4; ++c) v[4 * r + c] += w * (a4[r] * a4[c]);
                const double wr_ = w * a4[r];
#pragma unroll
                for (int c = 0; c < 3; ++c) v[16 + 3 * r + c] += wr_ * q3[c];
            }
        } else {
            const double4 fb = p.c_fb[t];
            const double b4[4] = {fb.x, fb.y, fb.z, fb.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) v[4 * r + c] += w * (a4[r] * b4[c]);
        }
    }
    if (diag) {
        // regularisation: the reverse pair (i, j) of each own pair (j, i) adds
        // w g g^T to K_jj and w g y^T (y = g[0:3]) to B_j; the own pair adds
        // w c^2 at (3,3) and -w c g[0:3] to B row 3 (energy.hpp:194-227)
        const int j = u;
        const int pb = p.node_pair_off[j], pe = p.node_pair_off[j + 1];
        for (int eo = pb + lane; eo < pe; eo += 32) {
            const int er = p.pair_rev[eo];
            const double w_r = wr[er], w_o = wr[eo];
            const double4 g = p.pair_gv[er], go = p.pair_gv[eo];
            const double g4[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
#pragma unroll
                for (int c = 0; c < 4; ++c) v[4 * r + c] += w_r * (g4[r] * g4[c]);
                const double wg = w_r * g4[r];
#pragma unroll
                for (int c = 0; c < 3; ++c) v[16 + 3 * r + c] += wg * g4[c];
            }
            v[15] += w_o * (go.w * go.w);
            const double wc = w_o * -go.w;
            v[25] += wc * go.x;
            v[26] += wc * go.y;
            v[27] += wc * go.z;
        }
    }
    double acc = transpose_reduce32(v);
    if (diag) {
        const int j = u;
        if (lane < 16) {
            const int r = lane >> 2, c = lane & 3;
            if (r == c && r < 3) acc += tp.beta;
            K[static_cast<size_t>(p.ub_kpos[u]) * 16 + lane] = acc;
        } else if (lane < 28) {
            const int r = (lane - 16) / 3, c = (lane - 16) % 3;
            if (r < 3) acc += tp.beta * R[9 * j + c * 3 + r];  // B += beta R^T (energy.hpp:216-217)
            B[12 * j + 3 * r + c] = acc;
        }
    } else if (lane < 16) {
        const int r = lane >> 2, c = lane & 3;
        const int ed = u - p.N;
        const int eab = p.edge_pab[ed], eba = p.edge_pba[ed];
        if (r == 3) acc += wr[eab] * (-p.pair_c[eab] * pair_g(p, eab, c));
        if (c == 3) acc += wr[eba] * (pair_g(p, eba, r) * -p.pair_c[eba]);
        K[static_cast<size_t>(p.ub_kpos[u]) * 16 + r * 4 + c] = acc;
        K[static_cast<size_t>(p.ub_kpos_t[u]) * 16 + c * 4 + r] = acc;
    }
}

// landmarks (stage 0 only): sequential, one thread, fixed order
__global__ void landmark_kernel(DevProblem p, TermParams tp, double* __restrict__ K, double* __restrict__ B) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (p.skip != nullptr && *p.skip) return;
    const double lw = tp.lm_weight;
    for (int l = 0; l < p.landmarks; ++l) {
        const int i = p.lm_vertex[l];
        const double qx = p.lm_pos[3 * l] - p.anchor[3 * i], qy = p.lm_pos[3 * l + 1] - p.anchor[3 * i + 1],
                     qz = p.lm_pos[3 * l + 2] - p.anchor[3 * i + 2];
        for (int ea = p.infl_off[i]; ea < p.infl_off[i + 1]; ++ea) {
            const int na = p.infl_node[ea];
            const double4 fa4 = p.infl_f[ea];
            const double fa[4] = {fa4.x, fa4.y, fa4.z, fa4.w};
            for (int eb = p.infl_off[i]; eb < p.infl_off[i + 1]; ++eb) {
                const int nb = p.infl_node[eb];
                const double4 fb4 = p.infl_f[eb];
                const double fb[4] = {fb4.x, fb4.y, fb4.z, fb4.w};
                int blk = -1;
                const int ra = p.node_row[na];
                for (int b = p.row_ptr[ra]; b < p.row_ptr[ra + 1]; ++b)
                    if (p.col[b] == nb) blk = b;
                if (blk < 0) continue;
                for (int r = 0; r < 4; ++r)
                    for (int s = 0; s < 4; ++s) K[static_cast<size_t>(blk) * 16 + r * 4 + s] += lw * (fa[r] * fb[s]);
            }
            const double qq[3] = {qx, qy, qz};
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 3; ++c) B[12 * na + 3 * r + c] += (lw * fa[r]) * qq[c];
        }
    }
}

// ---------------------------------------------------------------- Anderson
// Window push: new difference columns dF, dG into ring slot `slot` and the
// current residual f (solver.hpp:267-268, anderson.hpp:31-34).
__global__ void __launch_bounds__(kTermThreads) aa_update_kernel(AADevice aa, const double* __restrict__ g,
                                                                 const double* __restrict__ x,
                                                                 const double* __restrict__ f_in, int D,
                                                                 int have_prev, int slot) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
        const double gi = g[i];
        const double f = f_in ? f_in[i] : gi - x[i];  // F = G - X
        if (have_prev) {
            aa.df[static_cast<size_t>(slot) * D + i] = f - aa.fprev[i];
            aa.dg[static_cast<size_t>(slot) * D + i] = gi - aa.gprev[i];
        }
        aa.fprev[i] = f;
        aa.gprev[i] = gi;
    }
}

// ---- TSQR of the tall-skinny [dF (newest first) | f] (D x K, K = mk+1) with
// Givens rotations: every thread folds its rows into a K x K upper-triangular
// R held in registers, then the R factors are merged pairwise in a fixed tree
// (warp shuffles, shared memory, then one warp over the CTA partials). The
// result is the R factor of a backward-stable QR of the whole matrix, from
// which the reference's column-pivoted Householder QR (anderson.hpp:37-39) is
// finished on a K x K problem: this keeps the QR's kappa*eps accuracy and
// rank decision instead of the kappa^2*eps of normal equations.
template <int K>
struct Tri {
    double r[K * (K + 1) / 2];  // row-major upper triangle
    __device__ __forceinline__ static int at(int i, int j) { return i * K - i * (i - 1) / 2 + (j - i); }
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int t = 0; t < K * (K + 1) / 2; ++t) r[t] = 0.0;
    }
    // fold the row a[k0..K) (entries before k0 are zero) into R
    __device__ __forceinline__ void add_row(double* a, int k0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (k < k0) continue;
            const double ak = a[k];
            if (ak == 0.0) continue;
            const double rk = r[at(k, k)];
            // one reciprocal square root instead of sqrt + two divisions
            // (the merge chains are latency-bound)
            const double h2 = fma(rk, rk, ak * ak);
            const double inv = rsqrt(h2);
            const double c = rk * inv, s = ak * inv;
            r[at(k, k)] = h2 * inv;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                if (j <= k) continue;
                const double t = r[at(k, j)];
                r[at(k, j)] = c * t + s * a[j];
                a[j] = -s * t + c * a[j];
            }
        }
    }
    __device__ __forceinline__ void merge(const Tri& o) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            double a[K];
#pragma unroll
            for (int j = 0; j < K; ++j) a[j] = j < i ? 0.0 : o.r[at(i, j)];
            add_row(a, i);
        }
    }
    __device__ __forceinline__ void shfl_merge(int src_off) {  // merge lane+src_off's R into this lane's
        Tri o;
#pragma unroll
        for (int t = 0; t < K * (K + 1) / 2; ++t) o.r[t] = __shfl_down_sync(0xffffffffu, r[t], src_off);
        if ((threadIdx.x & (2 * src_off - 1)) == 0) merge(o);
    }
};

template <int K>
__global__ void __launch_bounds__(kTermThreads) aa_tsqr_kernel(AADevice aa, int D, SlotList cols) {
    __shared__ double sR[kTermThreads / 32][K * (K + 1) / 2];
    Tri<K> R;
    R.zero();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
        double a[K];
#pragma unroll
        for (int j = 0; j < K - 1; ++j) a[j] = aa.df[static_cast<size_t>(cols.s[j]) * D + i];
        a[K - 1] = aa.fprev[i];
        R.add_row(a, 0);
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) R.shfl_merge(off);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int t = 0; t < K * (K + 1) / 2; ++t) sR[w][t] = R.r[t];
    __syncthreads();
    // fixed binary tree over the warp factors (log2(nw) merges on the critical path)
    for (int step = 1; step < nw; step <<= 1) {
        if (lane == 0 && (w & (2 * step - 1)) == 0 && w + step < nw) {
            Tri<K> o;
#pragma unroll
            for (int t = 0; t < K * (K + 1) / 2; ++t) o.r[t] = sR[w + step][t];
            R.merge(o);
#pragma unroll
            for (int t = 0; t < K * (K + 1) / 2; ++t) sR[w][t] = R.r[t];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
#pragma unroll
        for (int t = 0; t < K * (K + 1) / 2; ++t) aa.partials[static_cast<size_t>(blockIdx.x) * kTriMax + t] = R.r[t];
}

// Merge the CTA partials (one warp, fixed tree) and finish with the
// reference's ColPivHouseholderQR semantics on the K x K factor: pivot on
// the largest remaining column norm (norms downdated as Eigen does), rank =
// #|R_kk| > |R|max * eps * min(D, mk); full rank -> back-substitution,
// otherwise (dF^T dF + 1e-10 I) theta = dF^T f (anderson.hpp:41-43).
template <int K>
__global__ void aa_solve_kernel(AADevice aa, double D, int nblocks) {
    constexpr int mk = K - 1;
    Tri<K> R;
    R.zero();
    for (int b = threadIdx.x; b < nblocks; b += 32) {  // nblocks <= 32: one load per lane
        Tri<K> o;
#pragma unroll
        for (int t = 0; t < K * (K + 1) / 2; ++t) o.r[t] = aa.partials[static_cast<size_t>(b) * kTriMax + t];
        R.merge(o);
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) R.shfl_merge(off);
    if (threadIdx.x != 0) return;
    // dense copy: A = R[:, :mk] (K x mk), c = R[:, mk]
    double A[K][mk > 0 ? mk : 1], c[K];
    for (int i = 0; i < K; ++i) {
        for (int j = 0; j < mk; ++j) A[i][j] = j >= i ? R.r[Tri<K>::at(i, j)] : 0.0;
        c[i] = R.r[Tri<K>::at(i, mk)];
    }
    const double eps = 2.220446049250313e-16;
    double nu[mk > 0 ? mk : 1], nd[mk > 0 ? mk : 1];
    int perm[mk > 0 ? mk : 1];
    double maxnorm = 0.0;
    for (int j = 0; j < mk; ++j) {
        double s = 0.0;
        for (int i = 0; i < K; ++i) s += A[i][j] * A[i][j];
        nu[j] = nd[j] = sqrt(s);
        maxnorm = fmax(maxnorm, nu[j]);
        perm[j] = j;
    }
    const double thr_helper = (maxnorm * eps) * (maxnorm * eps) / D;
    int nonzero = mk;
    double maxpivot = 0.0;
    for (int k = 0; k < mk; ++k) {
        int best = k;
        for (int j = k + 1; j < mk; ++j)
            if (nu[j] > nu[best]) best = j;
        if (nonzero == mk && nu[best] * nu[best] < thr_helper * (D - k)) nonzero = k;
        if (best != k) {
            for (int i = 0; i < K; ++i) {
                const double t = A[i][k];
                A[i][k] = A[i][best];
                A[i][best] = t;
            }
            double t = nu[k];
            nu[k] = nu[best];
            nu[best] = t;
            t = nd[k];
            nd[k] = nd[best];
            nd[best] = t;
            const int tp = perm[k];
            perm[k] = perm[best];
            perm[best] = tp;
        }
        // Householder on A[k.., k]
        double tail = 0.0;
        for (int i = k + 1; i < K; ++i) tail += A[i][k] * A[i][k];
        const double c0 = A[k][k];
        double tau = 0.0, beta = c0;
        if (tail > 2.2250738585072014e-308) {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0) beta = -beta;
            for (int i = k + 1; i < K; ++i) A[i][k] /= (c0 - beta);
            tau = (beta - c0) / beta;
        } else {
            for (int i = k + 1; i < K; ++i) A[i][k] = 0.0;
        }
        A[k][k] = beta;
        maxpivot = fmax(maxpivot, fabs(beta));
        for (int j = k + 1; j < mk; ++j) {  // apply to remaining columns
            double t = A[k][j];
            for (int i = k + 1; i < K; ++i) t += A[i][k] * A[i][j];
            A[k][j] -= tau * t;
            for (int i = k + 1; i < K; ++i) A[i][j] -= tau * A[i][k] * t;
        }
        {  // and to the rhs
            double t = c[k];
            for (int i = k + 1; i < K; ++i) t += A[i][k] * c[i];
            c[k] -= tau * t;
            for (int i = k + 1; i < K; ++i) c[i] -= tau * A[i][k] * t;
        }
        for (int j = k + 1; j < mk; ++j) {  // Eigen's norm downdate
            if (nu[j] != 0.0) {
                double t = fabs(A[k][j]) / nu[j];
                t = (1.0 + t) * (1.0 - t);
                t = t < 0 ? 0 : t;
                const double rr = nu[j] / nd[j];
                if (t * rr * rr <= sqrt(eps)) {
                    double s = 0.0;
                    for (int i = k + 1; i < K; ++i) s += A[i][j] * A[i][j];
                    nu[j] = nd[j] = sqrt(s);
                } else {
                    nu[j] *= sqrt(t);
                }
            }
        }
    }
    const double thr = maxpivot * eps * fmin(D, static_cast<double>(mk));
    int rank = 0;
    for (int k = 0; k < nonzero; ++k) rank += fabs(A[k][k]) > thr ? 1 : 0;
    double theta[mk > 0 ? mk : 1];
    if (rank == mk) {
        double y[mk > 0 ? mk : 1];
        for (int k = nonzero - 1; k >= 0; --k) {
            double v = c[k];
            for (int j = k + 1; j < nonzero; ++j) v -= A[k][j] * y[j];
            y[k] = v / A[k][k];
        }
        for (int k = 0; k < mk; ++k) theta[k] = 0.0;
        for (int k = 0; k < nonzero; ++k) theta[perm[k]] = y[k];
    } else {
        // normal equations from the unpivoted factor: dF^T dF = Rf^T Rf, dF^T f = Rf^T c
        double G[mk > 0 ? mk : 1][mk > 0 ? mk : 1], b[mk > 0 ? mk : 1];
        for (int a = 0; a < mk; ++a) {
            double sb = 0.0;
            for (int t = 0; t <= a; ++t) sb += R.r[Tri<K>::at(t, a)] * R.r[Tri<K>::at(t, mk)];
            b[a] = sb;
            for (int bb = 0; bb < mk; ++bb) {
                double s = 0.0;
                for (int t = 0; t <= min(a, bb); ++t) s += R.r[Tri<K>::at(t, a)] * R.r[Tri<K>::at(t, bb)];
                G[a][bb] = s + (a == bb ? 1e-10 : 0.0);
            }
        }
        for (int k = 0; k < mk; ++k) {  // Cholesky (SPD)
            double dkk = G[k][k];
            for (int t = 0; t < k; ++t) dkk -= G[k][t] * G[k][t];
            dkk = sqrt(fmax(dkk, 1e-300));
            G[k][k] = dkk;
            for (int i = k + 1; i < mk; ++i) {
                double v = G[i][k];
                for (int t = 0; t < k; ++t) v -= G[i][t] * G[k][t];
                G[i][k] = v / dkk;
            }
        }
        double y[mk > 0 ? mk : 1];
        for (int k = 0; k < mk; ++k) {
            double v = b[k];
            for (int t = 0; t < k; ++t) v -= G[k][t] * y[t];
            y[k] = v / G[k][k];
        }
        for (int k = mk - 1; k >= 0; --k) {
            double v = y[k];
            for (int t = k + 1; t < mk; ++t) v -= G[t][k] * y[t];
            y[k] = v / G[k][k];
        }
        for (int k = 0; k < mk; ++k) theta[k] = y[k];
    }
    for (int k = 0; k < mk; ++k) aa.theta[k] = theta[k];
    *aa.rank = rank;
}

__global__ void __launch_bounds__(256) aa_combine_kernel(AADevice aa, int D, SlotList cols,
                                                         double* __restrict__ x_next, int* __restrict__ nonfinite) {
    __shared__ double th[kMaxAA];
    if (threadIdx.x < cols.n) th[threadIdx.x] = aa.theta[threadIdx.x];
    __syncthreads();
    bool bad = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
        double s = 0.0;  // dG theta, then g - (dG theta)  (anderson.hpp:45)
        for (int k = 0; k < cols.n; ++k) s += aa.dg[static_cast<size_t>(cols.s[k]) * D + i] * th[k];
        const double v = aa.gprev[i] - s;
        x_next[i] = v;
        bad |= !isfinite(v);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------- layout
__global__ void pass_decision_kernel(const PassRecord* __restrict__ rec, double e_prev, int current_is_aa,
                                     double lm_w, int* __restrict__ skip) {
    const double e = __dadd_rn(rec->total, __dmul_rn(lm_w, rec->landmark));
    *skip = (!isfinite(e) || (current_is_aa && e > e_prev)) ? 1 : 0;
}

__global__ void col_to_node_kernel(const double* __restrict__ in, double* __restrict__ out, int N) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 12 * N) return;
    const int j = t / 12, rc = t % 12, r = rc / 3, c = rc % 3;
    out[t] = in[static_cast<size_t>(c) * 4 * N + 4 * j + r];
}
__global__ void node_to_col_kernel(const double* __restrict__ in, double* __restrict__ out, int N) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 12 * N) return;
    const int j = t / 12, rc = t % 12, r = rc / 3, c = rc % 3;
    out[static_cast<size_t>(c) * 4 * N + 4 * j + r] = in[t];
}

}  // namespace

void launch_deform(const DevProblem& p, const double* x, double* out, const double* old, double* max_disp,
                   int* nonfinite, cudaStream_t s) {
    if (p.n == 0) return;
    deform_kernel<<<(p.n + 255) / 256, 256, 0, s>>>(p, x, out, old, max_disp, nonfinite);
    NRR_CUDA_CHECK(cudaGetLastError());
}

void launch_terms(const DevProblem& p, const double* x, const double* d2, const TermParams& tp, double* wa,
                  double* wr, double* R, double* partials, int* degenerate, cudaStream_t s) {
    terms_kernel<<<kTermBlocks, kTermThreads, 0, s>>>(p, x, d2, tp, wa, wr, R, partials, degenerate);
    NRR_CUDA_CHECK(cudaGetLastError());
}

void launch_energy_reduce(const DevProblem& p, const double* partials, const TermParams& tp, const double* vhat,
                          PassRecord* rec, cudaStream_t s) {
    energy_reduce_kernel<<<1, 256, 0, s>>>(p, partials, tp, vhat, rec, kTermBlocks);
    NRR_CUDA_CHECK(cudaGetLastError());
}

void launch_pass_decision(const PassRecord* rec, double e_prev, int current_is_aa, double lm_w, int* skip,
                          cudaStream_t s) {
    pass_decision_kernel<<<1, 1, 0, s>>>(rec, e_prev, current_is_aa, lm_w, skip);
    NRR_CUDA_CHECK(cudaGetLastError());
}

void launch_assemble(const DevProblem& p, const double* wa, const double* q, const double* wr, const double* R,
                     const TermParams& tp, double* K, double* B, cudaStream_t s) {
    if (p.U > 0) {
        assemble_kernel<<<(p.U + kAsmWarps - 1) / kAsmWarps, kAsmWarps * 32, 0, s>>>(p, wa, q, wr, R, tp, K, B);
        NRR_CUDA_CHECK(cudaGetLastError());
    }
    if (tp.lm_weight != 0.0 && p.landmarks > 0) {
        landmark_kernel<<<1, 32, 0, s>>>(p, tp, K, B);
        NRR_CUDA_CHECK(cudaGetLastError());
    }
}

void launch_rotations(const double* x, int N, double* R, int* degenerate, cudaStream_t s, double* sigma_min) {
    if (N == 0) return;
    rotations_kernel<<<(N + 127) / 128, 128, 0, s>>>(x, N, R, degenerate, sigma_min);
    NRR_CUDA_CHECK(cudaGetLastError());
}

void launch_aa_update(const AADevice& aa, const double* g, const double* x, const double* f, int D, int have_prev,
                      int slot, cudaStream_t s) {
    aa_update_kernel<<<kTermBlocks, kTermThreads, 0, s>>>(aa, g, x, f, D, have_prev, slot);
    NRR_CUDA_CHECK(cudaGetLastError());
}

template <int K>
static void aa_solve_k(const AADevice& aa, int D, const SlotList& cols, cudaStream_t s) {
    // kBlocks CTAs x 256 threads: a few rows per thread, then log-depth
    // merges (warp shuffles, CTA tree, one warp over the CTA factors); the
    // CTA count trades the per-thread fold chain against the merge depth
    static const int kBlocks = [] {
        const char* e = std::getenv("NRR_AA_BLOCKS");
        const int b = e ? std::atoi(e) : 32;
        return b >= 1 && b <= 32 ? b : 32;
    }();
    aa_tsqr_kernel<K><<<kBlocks, kTermThreads, 0, s>>>(aa, D, cols);
    aa_solve_kernel<K><<<1, 32, 0, s>>>(aa, static_cast<double>(D), kBlocks);
}

void launch_aa_solve(const AADevice& aa, int D, const SlotList& cols, cudaStream_t s) {
    switch (cols.n + 1) {
#define NRR_AA_CASE(k) \
    case k:            \
        aa_solve_k<k>(aa, D, cols, s); \
        break;
        NRR_AA_CASE(2) NRR_AA_CASE(3) NRR_AA_CASE(4) NRR_AA_CASE(5) NRR_AA_CASE(6) NRR_AA_CASE(7)
        NRR_AA_CASE(8) NRR_AA_CASE(9) NRR_AA_CASE(10) NRR_AA_CASE(11) NRR_AA_CASE(12) NRR_AA_CASE(13)
        NRR_AA_CASE(14) NRR_AA_CASE(15) NRR_AA_CASE(16) NRR_AA_CASE(17)
#undef NRR_AA_CASE
        default:
            throw ConfigError("aa_window above the device limit of 16");
    }
    NRR_CUDA_CHECK(cudaGetLastError());
}

void launch_aa_combine(const AADevice& aa, int D, const SlotList& cols, double* x_next, int* nonfinite,
                       cudaStream_t s) {
    aa_combine_kernel<<<kTermBlocks, 256, 0, s>>>(aa, D, cols, x_next, nonfinite);
    NRR_CUDA_CHECK(cudaGetLastError());
}

void launch_colmajor_to_nodemajor(const double* in, double* out, int N, cudaStream_t s) {
    if (N == 0) return;
    col_to_node_kernel<<<(12 * N + 255) / 256, 256, 0, s>>>(in, out, N);
    NRR_CUDA_CHECK(cudaGetLastError());
}
void launch_nodemajor_to_colmajor(const double* in, double* out, int N, cudaStream_t s) {
    if (N == 0) return;
    node_to_col_kernel<<<(12 * N + 255) / 256, 256, 0, s>>>(in, out, N);
    NRR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace nrr_b200
