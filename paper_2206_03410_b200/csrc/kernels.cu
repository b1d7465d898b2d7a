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
// three CTAs per SM (80 registers instead of 92, 16 B of spills): the kernel is latency-bound at 25%
// occupancy; config 2 46.7 -> 37.4 us, config 4 289 -> 208 us (profiles/r04_occupancy_ab.txt)
#ifndef NRR_ASM_MINB
#define NRR_ASM_MINB 3
#endif
__global__ void __launch_bounds__(kAsmWarps * 32, NRR_ASM_MINB) assemble_kernel(DevProblem p, const double* __restrict__ wa,
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

template <int K>
struct Tri {  // packed row-major upper triangle
    __device__ __forceinline__ static int at(int i, int j) { return i * K - i * (i - 1) / 2 + (j - i); }
};

// ---- Least squares min |f - dF theta| (anderson.hpp:36-44) from the R factor
// of the tall-skinny [dF (newest first) | f] (D x K, K = mk+1), computed by a
// communication-avoiding Householder QR: a warp holds a panel of rows (S per
// lane) and reduces it to a K x K triangle with K reflections whose norms and
// dot products are xor-butterfly sums (every lane gets the same bits, fixed
// order: deterministic); triangles are stacked and reduced again (warp panels
// -> one per CTA -> one). This keeps the QR's kappa*eps accuracy and rank
// decision (normal equations would square kappa), and the critical path is
// 3-4 panel factorisations of ~K butterfly rounds each instead of a 14-deep
// tree of serial Givens merges (62 -> ~15 us per pass on config 2).

// Householder QR of the S*32 rows a warp holds: lane l, slot s is one row;
// row (slot 0, lane k) is the pivot row of column k. Afterwards lane k < K
// holds row k of R in a[0][k..K) (entries left of the diagonal, and every
// other row, are to be taken as zero).
template <int K, int S>
__device__ __forceinline__ void warp_house_qr(double (&a)[S][K]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        // rows of slot 0 in lanes < k are finished rows of R
        const bool live0 = lane > k;  // slot 0 is a non-pivot live row
        double tail = live0 ? a[0][k] * a[0][k] : 0.0;
#pragma unroll
        for (int t = 1; t < S; ++t) tail = fma(a[t][k], a[t][k], tail);
        tail = warp_sum(tail);
        const double x0 = __shfl_sync(0xffffffffu, a[0][k], k);
        if (!(tail > 2.2250738585072014e-308)) continue;  // nothing below the pivot (warp-uniform)
        double beta = sqrt(fma(x0, x0, tail));
        if (x0 >= 0) beta = -beta;
        const double vp = x0 - beta;                    // pivot entry of v = x - beta e_p
        const double d = 1.0 / (beta * (beta - x0));   // 2 / v^T v  (> 0)
        const double v0 = lane == k ? vp : (live0 ? a[0][k] : 0.0);
        double f[K];
#pragma unroll
        for (int j = k + 1; j < K; ++j) {
            double dot = v0 * a[0][j];
#pragma unroll
            for (int t = 1; t < S; ++t) dot = fma(a[t][k], a[t][j], dot);
            f[j] = dot;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int j = k + 1; j < K; ++j) f[j] += __shfl_xor_sync(0xffffffffu, f[j], o);
#pragma unroll
        for (int j = k + 1; j < K; ++j) {
            const double fj = f[j] * d;
            a[0][j] = fma(-v0, fj, a[0][j]);
#pragma unroll
            for (int t = 1; t < S; ++t) a[t][j] = fma(-a[t][k], fj, a[t][j]);
        }
        if (lane == k) a[0][k] = beta;
    }
}

constexpr int kAaWarps = kTermThreads / 32;
// rows of a warp panel per lane besides the carried triangle (registers: (SN+1) K doubles)
template <int K>
struct AaPanel {
    static constexpr int SN = K <= 6 ? 8 : (K <= 9 ? 4 : 2);
    static constexpr int SM = (kAaWarps * K + 31) / 32;  // slots for the CTA's stacked warp triangles
    static constexpr int SS = 4;                         // slots per lane in the final kernel
};

// The CTA's warp triangles (lane k < K of every warp: row k in r0[k..K)) are
// stacked in shared memory and reduced by warp 0; returns (warp 0, lane k < K)
// row k of the CTA's R in r0. sR: kAaWarps * K * K doubles.
template <int K>
__device__ __forceinline__ void block_merge_qr(double (&r0)[K], double* sR) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane < K)
#pragma unroll
        for (int j = 0; j < K; ++j) sR[(w * K + lane) * K + j] = j >= lane ? r0[j] : 0.0;
    __syncthreads();
    if (w != 0) return;
    constexpr int SM = AaPanel<K>::SM;
    double a[SM][K];
#pragma unroll
    for (int t = 0; t < SM; ++t) {
        const int row = t * 32 + lane;
#pragma unroll
        for (int j = 0; j < K; ++j) a[t][j] = row < kAaWarps * K ? sR[row * K + j] : 0.0;
    }
    warp_house_qr<K, SM>(a);
#pragma unroll
    for (int j = 0; j < K; ++j) r0[j] = a[0][j];
}

// Window push (solver.hpp:267-268, anderson.hpp:31-34) fused with the panel
// factorisation: row i's new difference entries go to ring slot `slot`, the
// residual f and g are stored, and the row [dF(cols) | f] joins the warp's
// panel. Writes the CTA's triangle (packed rows) to aa.partials.
template <int K>
__global__ void __launch_bounds__(kTermThreads) aa_push_qr_kernel(AADevice aa, const double* __restrict__ g,
                                                                  const double* __restrict__ x,
                                                                  const double* __restrict__ f_in, int D,
                                                                  int have_prev, int slot, SlotList cols) {
    constexpr int SN = AaPanel<K>::SN;
    __shared__ double sR[kAaWarps * K * K];
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kAaWarps + (threadIdx.x >> 5), nwarps = gridDim.x * kAaWarps;
    const int nchunks = (D + 32 * SN - 1) / (32 * SN);
    double a[SN + 1][K];
#pragma unroll
    for (int j = 0; j < K; ++j) a[0][j] = 0.0;
    for (int chunk = gw; chunk < nchunks; chunk += nwarps) {
        // every load of the panel is issued before the first store (the
        // ring columns may alias for the compiler: interleaved, each slot
        // cost its own DRAM round trip)
        double gi[SN], fv[SN], fp[SN], gp[SN];
#pragma unroll
        for (int t = 1; t <= SN; ++t) {
            const int i = (chunk * SN + (t - 1)) * 32 + lane;
            gi[t - 1] = fv[t - 1] = fp[t - 1] = gp[t - 1] = 0.0;
#pragma unroll
            for (int j = 0; j < K; ++j) a[t][j] = 0.0;
            if (i < D) {
                gi[t - 1] = g[i];
                fv[t - 1] = f_in ? f_in[i] : x[i];
                if (have_prev) {
                    fp[t - 1] = aa.fprev[i];
                    gp[t - 1] = aa.gprev[i];
                }
#pragma unroll
                for (int j = 0; j < K - 1; ++j)
                    if (!(have_prev && cols.s[j] == slot)) a[t][j] = aa.df[static_cast<size_t>(cols.s[j]) * D + i];
            }
        }
#pragma unroll
        for (int t = 1; t <= SN; ++t) {
            const int i = (chunk * SN + (t - 1)) * 32 + lane;
            if (i < D) {
                const double f = f_in ? fv[t - 1] : gi[t - 1] - fv[t - 1];  // F = G - X
                if (have_prev) {
                    const double dfn = f - fp[t - 1];
                    aa.df[static_cast<size_t>(slot) * D + i] = dfn;
                    aa.dg[static_cast<size_t>(slot) * D + i] = gi[t - 1] - gp[t - 1];
#pragma unroll
                    for (int j = 0; j < K - 1; ++j)
                        if (cols.s[j] == slot) a[t][j] = dfn;
                }
                aa.fprev[i] = f;
                aa.gprev[i] = gi[t - 1];
                a[t][K - 1] = f;
            }
        }
        warp_house_qr<K, SN + 1>(a);
        // the carried triangle: row k in lane k, zero left of the diagonal; other lanes' slot 0 is spent
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (lane >= K || j < lane) a[0][j] = 0.0;
    }
    double r0[K];
#pragma unroll
    for (int j = 0; j < K; ++j) r0[j] = a[0][j];
    block_merge_qr<K>(r0, sR);
    if (threadIdx.x < K)
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (j >= lane) aa.partials[static_cast<size_t>(blockIdx.x) * kTriMax + Tri<K>::at(lane, j)] = r0[j];
}

// The reference's ColPivHouseholderQR semantics on the K x K factor, one
// column per lane (lane mk: the right-hand side): pivot on the largest
// remaining column norm (ties: first in the permuted order, norms downdated
// as Eigen does), rank = #|R_kk| > |R|max * eps * min(D, mk); full rank ->
// back-substitution, otherwise (dF^T dF + 1e-10 I) theta = dF^T f from the
// unpivoted factor (anderson.hpp:41-43). r0: lane k < K holds row k of R.
// sm: K*K doubles of shared memory. Called by one full warp.
template <int K>
__device__ __forceinline__ void aa_finish(const double (&r0)[K], AADevice aa, double D, double* sm) {
    constexpr int mk = K - 1;
    constexpr unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    if (lane < K)
#pragma unroll
        for (int j = 0; j < K; ++j) sm[lane * K + j] = j >= lane ? r0[j] : 0.0;
    __syncwarp();
    double col[K];
#pragma unroll
    for (int i = 0; i < K; ++i) col[i] = lane < K ? sm[i * K + lane] : 0.0;
    const bool iscol = lane < mk;
    const double eps = 2.220446049250313e-16;
    double nu, nd;
    {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i) s += col[i] * col[i];
        nu = nd = iscol ? sqrt(s) : -1.0;
    }
    const double maxnorm = warp_max(iscol ? nu : 0.0);
    const double thr_helper = (maxnorm * eps) * (maxnorm * eps) / D;
    int pos = iscol ? lane : 64;  // position of the lane's column in the pivoted order
    int nonzero = mk;
    double maxpivot = 0.0;
#pragma unroll
    for (int k = 0; k < mk; ++k) {
        // largest remaining norm, ties to the smallest position
        double bn = (iscol && pos >= k) ? nu : -1.0;
        int bp = pos;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double on = __shfl_xor_sync(full, bn, o);
            const int op = __shfl_xor_sync(full, bp, o);
            if (on > bn || (on == bn && op < bp)) {
                bn = on;
                bp = op;
            }
        }
        bn = __shfl_sync(full, bn, 0);  // one decision for the warp (NaN norms compare inconsistently)
        bp = __shfl_sync(full, bp, 0);
        if (nonzero == mk && bn * bn < thr_helper * (D - k)) nonzero = k;
        const bool is_piv = iscol && pos == bp;
        if (iscol) {
            if (pos == k)
                pos = bp;
            else if (pos == bp)
                pos = k;
        }
        const unsigned pm = __ballot_sync(full, is_piv);
        const int pl = pm ? __ffs(pm) - 1 : 0;
        // Householder on the pivot column's entries k.. (every lane computes it)
        double tail = 0.0;
#pragma unroll
        for (int i = k + 1; i < K; ++i) tail += col[i] * col[i];
        tail = __shfl_sync(full, tail, pl);
        const double c0 = __shfl_sync(full, col[k], pl);
        double ess[K];
        double tau = 0.0, beta = c0;
        if (tail > 2.2250738585072014e-308) {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0) beta = -beta;
#pragma unroll
            for (int i = k + 1; i < K; ++i) ess[i] = __shfl_sync(full, col[i], pl) / (c0 - beta);
            tau = (beta - c0) / beta;
        } else {
#pragma unroll
            for (int i = k + 1; i < K; ++i) ess[i] = 0.0;
        }
        maxpivot = fmax(maxpivot, fabs(beta));
        if ((iscol && pos > k) || lane == mk) {  // remaining columns and the right-hand side
            double t = col[k];
#pragma unroll
            for (int i = k + 1; i < K; ++i) t += ess[i] * col[i];
            col[k] -= tau * t;
#pragma unroll
            for (int i = k + 1; i < K; ++i) col[i] -= tau * ess[i] * t;
        }
        if (is_piv) col[k] = beta;
        if (iscol && pos > k && nu != 0.0) {  // Eigen's norm downdate
            double t = fabs(col[k]) / nu;
            t = (1.0 + t) * (1.0 - t);
            t = t < 0 ? 0 : t;
            const double rr = nu / nd;
            if (t * rr * rr <= sqrt(eps)) {
                double s = 0.0;
#pragma unroll
                for (int i = k + 1; i < K; ++i) s += col[i] * col[i];
                nu = nd = sqrt(s);
            } else {
                nu *= sqrt(t);
            }
        }
    }
    const double thr = maxpivot * eps * fmin(D, static_cast<double>(mk));
    double mydiag = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i)
        if (i == pos) mydiag = col[i];
    const int rank = __popc(__ballot_sync(full, iscol && pos < nonzero && fabs(mydiag) > thr));
    if (rank == mk) {
        // column-oriented back-substitution on the right-hand side lane
        double theta = 0.0;
#pragma unroll
        for (int k = mk - 1; k >= 0; --k) {
            const unsigned pm = __ballot_sync(full, iscol && pos == k);
            const int pl = pm ? __ffs(pm) - 1 : 0;
            const double y = __shfl_sync(full, col[k], mk) / __shfl_sync(full, col[k], pl);
            if (lane == pl) theta = y;
#pragma unroll
            for (int i = 0; i < k; ++i) {
                const double aik = __shfl_sync(full, col[i], pl);
                if (lane == mk) col[i] -= aik * y;
            }
        }
        if (iscol) aa.theta[lane] = theta;
    } else if (lane == 0) {
        // normal equations from the unpivoted factor: dF^T dF = Rf^T Rf, dF^T f = Rf^T c
        double G[mk > 0 ? mk : 1][mk > 0 ? mk : 1], b[mk > 0 ? mk : 1];
        for (int a = 0; a < mk; ++a) {
            double sb = 0.0;
            for (int t = 0; t <= a; ++t) sb += sm[t * K + a] * sm[t * K + mk];
            b[a] = sb;
            for (int bb = 0; bb < mk; ++bb) {
                double s = 0.0;
                for (int t = 0; t <= min(a, bb); ++t) s += sm[t * K + a] * sm[t * K + bb];
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
        for (int k = 0; k < mk; ++k) aa.theta[k] = y[k];
    }
    if (lane == 0) *aa.rank = rank;
}

// One CTA: the nblocks CTA triangles (nblocks * K stacked rows) are reduced
// to one (a single warp panel when they fit AaPanel::SS slots, otherwise one
// panel per warp and a second level) and the least squares finished.
template <int K>
__global__ void __launch_bounds__(kTermThreads) aa_solve_kernel(AADevice aa, double D, int nblocks) {
    constexpr int SS = AaPanel<K>::SS;
    __shared__ double sR[kAaWarps * K * K];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int rows = nblocks * K;
    const bool single = rows <= 32 * SS;
    if (single && w != 0) return;
    const int per_warp = single ? rows : (rows + kAaWarps - 1) / kAaWarps;  // <= 32 * SS (launch_aa_solve)
    const int row0 = single ? 0 : w * per_warp, row1 = min(rows, row0 + per_warp);
    double a[SS][K];
#pragma unroll
    for (int t = 0; t < SS; ++t) {
        const int row = row0 + t * 32 + lane;
        const int b = row / K, i = row - b * K;
#pragma unroll
        for (int j = 0; j < K; ++j)
            a[t][j] = (row < row1 && j >= i) ? aa.partials[static_cast<size_t>(b) * kTriMax + Tri<K>::at(i, j)] : 0.0;
    }
    warp_house_qr<K, SS>(a);
    double r0[K];
#pragma unroll
    for (int j = 0; j < K; ++j) r0[j] = a[0][j];
    if (!single) {
        block_merge_qr<K>(r0, sR);
        if (w != 0) return;
    }
    aa_finish<K>(r0, aa, D, sR);
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
static void aa_push_solve_k(const AADevice& aa, const double* g, const double* x, const double* f, int D,
                            int have_prev, int slot, const SlotList& cols, cudaStream_t s) {
    // one warp panel of 32 * SN rows per warp and pass; the CTA count is
    // bounded by the SMs and by the final kernel's capacity (kAaWarps panels
    // of 32 * SS stacked triangle rows)
    constexpr int SN = AaPanel<K>::SN;
    const int nchunks = (D + 32 * SN - 1) / (32 * SN);
    static const int kMaxBlocks = [] {
        const char* e = std::getenv("NRR_AA_BLOCKS");
        const int b = e ? std::atoi(e) : 148;
        return b >= 1 && b <= kTermBlocks ? b : 148;
    }();
    const int cap = (kAaWarps * 32 * AaPanel<K>::SS) / K;
    const int blocks = std::max(1, std::min(std::min(kMaxBlocks, cap), (nchunks + kAaWarps - 1) / kAaWarps));
    aa_push_qr_kernel<K><<<blocks, kTermThreads, 0, s>>>(aa, g, x, f, D, have_prev, slot, cols);
    aa_solve_kernel<K><<<1, kTermThreads, 0, s>>>(aa, static_cast<double>(D), blocks);
}

void launch_aa_push_solve(const AADevice& aa, const double* g, const double* x, const double* f, int D, int have_prev,
                          int slot, const SlotList& cols, cudaStream_t s) {
    switch (cols.n + 1) {
#define NRR_AA_CASE(k) \
    case k:            \
        aa_push_solve_k<k>(aa, g, x, f, D, have_prev, slot, cols, s); \
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
