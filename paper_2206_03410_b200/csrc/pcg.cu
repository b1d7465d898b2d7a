// SPD solve K X = B (reference SystemAssembler::solve, energy.hpp:233-254;
// solve_system :393-408) as a two-level preconditioned conjugate gradient in
// FP64 on sm_100a.
//
// Layout. Graph nodes are partitioned into one compact subdomain per CTA (one
// CTA per SM): recursive coordinate bisection whose splits fall on coarse
// aggregate boundaries, then a Lloyd relaxation that rounds the subdomains
// (PcgPlan::build). Each CTA copies its rows' K blocks into shared memory once
// per solve (when they fit), so every SpMV reads K from SMEM. The three
// right-hand sides (output coordinates, energy.hpp:118-121) share every K
// read; a thread owns (node, row r, column c) elements in registers.
//
// Preconditioner M^-1 = sum_k K_kk^-1 (subdomain block Jacobi: exact dense
// inverses of the diagonal blocks of <= 32 consecutive rows, sub_invert_kernel)
// + Psi K0^-1 Psi^T, a coarse correction over aggregates of 4 consecutive
// subdomains. Psi spans, per aggregate, the 4 modes that make the regularizer
// vanish (a global affine map: node j's unknowns [a; a.(p_j - c) + b],
// energy.hpp:77-84), so the graph-Laplacian-like low modes that stall block
// Jacobi are solved exactly on the coarse level. K0 = Psi^T K Psi (<= 160 x
// 160) is assembled from CTA partials in a fixed order and inverted by one
// CTA (Gauss-Jordan, SPD); both parts are reused across solves of a stage.
//
// Iteration: pipelined PCG (Ghysels & Vanroose) with ONE grid barrier; all
// reductions are two-level and fixed-order, so the result is bitwise
// reproducible. Before the barrier every CTA holds r, u = M r, w = K u for
// its rows and publishes the partials of (r,u), (w,u), max|r|, Psi^T w and
// m' = M_sub w; after it one L2 round trip brings the totals and the halo of
// m', the coarse part is completed on own and halo rows, n = K m, and the
// recurrences advance (see the loop in pcg_kernel).
// Exit: the recursive residual reaches pcg_rtol*(1+|B|max); the true residual
// B-KX must then meet the reference bar 1e-8*(1+|B|max) (energy.hpp:245),
// otherwise PCG restarts from it. A 4x4 diagonal block whose Cholesky pivot
// is not positive reports "singular diagonal block at node j"
// (energy.hpp:329-340); p^T K p <= 0 reports an indefinite system.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <vector>
#include <chrono>
#include <mutex>
#include <map>
#include <condition_variable>
#include <thread>

#include "device_common.cuh"
#include "pcg.cuh"

namespace cg = cooperative_groups;

namespace nrr_b200 {

namespace {

constexpr int kQ = kPcgSlots;  // partial slots per CTA and phase
// per-iteration clock64 phase probes (NRR_PROF=1 prints them); compiled out
// unless built with -DNRR_PCG_PROBES=1 (they cost issue slots in the loop)
#ifndef NRR_PCG_PROBES
#define NRR_PCG_PROBES 0
#endif
constexpr bool kPcgProbes = NRR_PCG_PROBES != 0;
// subdomain preconditioner matvec: one thread per output element (see
// precond_sub) when a thread owns several elements (EPT >= 2: config 4
// 7.09 -> 6.39 ms per solve), four threads per scalar row with a butterfly
// for EPT = 1 (config 2: 0.847 vs 0.879 ms); 1 forces the former everywhere
#ifndef NRR_PCG_DIRECT
#define NRR_PCG_DIRECT 0
#endif
constexpr int kCoarseThreads = 512;

// coarse mode k of node a in aggregate g: [e_k; d_k] for k < 3, e_3 for k = 3,
// d = p_a - c_g
__device__ __forceinline__ void node_offset(const PcgArgs& a, int node, double d[3]) {
    const int g = a.node_agg[node];
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = a.node_pos[3 * node + k] - a.agg_center[3 * g + k];
}

// Branch-free FP64 reciprocal / quotient: hardware approximation + two Newton
// steps (full precision for normal operands; deterministic, not IEEE-rounded).
// The PCG scalars need no correctly rounded division, and the library
// routine's special-case branch serialises the three columns.
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ double div_nr(double n, double d) {
    const double r = rcp_nr(d);
    const double q = n * r;
    return fma(r, fma(-d, q, n), q);
}

// ---------------------------------------------------------------- blocked Gauss-Jordan
// In-place inverse of nm SPD matrices held in shared memory (matrix k: n_k x
// n_k with n_k = 4 * blocks_k, leading dimension ld, base A + k * msz), all
// processed together by the whole CTA, 4 pivots (one node block) at a time:
//   P = A_TT^{-1} (4x4, one thread per matrix, reciprocal + Newton; a pivot
//       <= drop * dmax_k drops that mode: zero row and column),
//   R = P A_T:,  C = A_:T,
//   A_ij -= C_i R_j,  A_iT = -C_i P,  A_Tj = R_j,  A_TT = P.
// Three barriers per block step; the element updates are spread over every
// thread of the CTA (row-major flattening over the matrices' rows x ncmax
// columns). Fixed operation order: deterministic. Scratch: pb[nm*16],
// cb[nm*4*ld] (C, s-major), rb[nm*4*ld] (R), blocks[nm], dmax[nm].
__device__ void block_gj_inverse(double* A, int nm, const int* blocks, int ld, size_t msz, double* pb, double* cb,
                                 double* rb, const double* dmax, double drop, long long* prof = nullptr) {
    long long tq = clock64();
    auto gprobe = [&](int slot) {
        if (prof != nullptr && threadIdx.x == 0) {
            const long long t = clock64();
            prof[slot] += t - tq;
            tq = t;
        }
    };
    int nb_max = 0, rows_total = 0;
    for (int k = 0; k < nm; ++k) {
        nb_max = max(nb_max, blocks[k]);
        rows_total += 4 * blocks[k];
    }
    // element (gi, j) of the flattened matrix rows -> matrix k, local row i
    auto locate = [&](int gi, int& k, int& i) {
        int base = 0;
        k = 0;
        while (gi >= base + 4 * blocks[k]) base += 4 * blocks[k++];
        i = gi - base;
    };
    for (int T = 0; T < nb_max; ++T) {
        const int t0 = 4 * T;
        // phase 1: P per matrix (thread k); raw C and row block T into cb / rb
        if (threadIdx.x < nm && T < blocks[threadIdx.x]) {
            const int k = threadIdx.x;
            const double* Ak = A + k * msz;
            double m[4][4], inv[4][4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    m[r][c] = Ak[(t0 + r) * ld + t0 + c];
                    inv[r][c] = r == c ? 1.0 : 0.0;
                }
            bool live[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double piv = m[q][q];
                live[q] = piv > drop * dmax[k];
                const double d = live[q] ? rcp_nr(piv) : 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    m[q][c] *= d;
                    inv[q][c] *= d;
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r == q) continue;
                    const double f = m[r][q];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        m[r][c] -= f * m[q][c];
                        inv[r][c] -= f * inv[q][c];
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) pb[k * 16 + r * 4 + c] = (live[r] && live[c]) ? inv[r][c] : 0.0;
        }
        for (int gi = threadIdx.x; gi < rows_total; gi += blockDim.x) {
            int k, i;
            locate(gi, k, i);
            if (T >= blocks[k]) continue;
            const double* Ai = A + k * msz + static_cast<size_t>(i) * ld;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                cb[k * 4 * ld + s * ld + i] = Ai[t0 + s];                                         // C[i][s]
                rb[k * 4 * ld + s * ld + i] = A[k * msz + static_cast<size_t>(t0 + s) * ld + i];  // row T+s, column i
            }
        }
        gprobe(24);
        __syncthreads();
        gprobe(25);
        // phase 2: R = P * (row block), in place in rb
        for (int gi = threadIdx.x; gi < rows_total; gi += blockDim.x) {
            int k, j;
            locate(gi, k, j);
            if (T >= blocks[k]) continue;
            double* rk = rb + k * 4 * ld;
            const double* P = pb + k * 16;
            const double x0 = rk[j], x1 = rk[ld + j], x2 = rk[2 * ld + j], x3 = rk[3 * ld + j];
#pragma unroll
            for (int r = 0; r < 4; ++r) rk[r * ld + j] = P[r * 4] * x0 + P[r * 4 + 1] * x1 + P[r * 4 + 2] * x2 + P[r * 4 + 3] * x3;
        }
        __syncthreads();
        gprobe(26);
        // phase 3: rank-4 update, one warp per row (matrix and row located
        // once), lanes over columns
        {
            const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
            for (int gi = w; gi < rows_total; gi += nw) {
                int k, i;
                locate(gi, k, i);
                if (T >= blocks[k]) continue;
                const int nk = 4 * blocks[k];
                double* Ai = A + k * msz + static_cast<size_t>(i) * ld;
                const double* ck = cb + k * 4 * ld;
                const double* rk = rb + k * 4 * ld;
                const double* P = pb + k * 16;
                const bool in_t = i >= t0 && i < t0 + 4;
                const double c0 = ck[i], c1 = ck[ld + i], c2 = ck[2 * ld + i], c3 = ck[3 * ld + i];
                for (int j = lane; j < nk; j += 32) {
                    const bool jt = j >= t0 && j < t0 + 4;
                    double v;
                    if (in_t && jt) {
                        v = P[(i - t0) * 4 + (j - t0)];
                    } else if (in_t) {
                        v = rk[(i - t0) * ld + j];
                    } else if (jt) {
                        const int q = j - t0;
                        v = -(c0 * P[q] + c1 * P[4 + q] + c2 * P[8 + q] + c3 * P[12 + q]);
                    } else {
                        v = Ai[j] - (c0 * rk[j] + c1 * rk[ld + j] + c2 * rk[2 * ld + j] + c3 * rk[3 * ld + j]);
                    }
                    Ai[j] = v;
                }
            }
        }
        gprobe(27);
        __syncthreads();
        gprobe(28);
    }
}

// ---------------------------------------------------------------- coarse setup
// CTA c: for each aggregate h its rows' columns touch (touch list t < nt),
// partial[c][t][k*4+l] = sum over the CTA's blocks (a,b) with b in h of
// psi_k(a)^T K_ab psi_l(b). One thread per block forms its 4x4 projection
// (staged in shared memory), then 8 lanes per output sum the blocks of that
// aggregate (lane-strided, butterfly-combined): deterministic, no atomics.
constexpr int kCpChunk = 1024;  // blocks per shared-memory pass (a multiple of 8: same sum order as one pass)
constexpr int kCpRounds = 16;   // 64 touched aggregates x 16 entries / 64 lane groups
__global__ void __launch_bounds__(kCoarseThreads) coarse_partial_kernel(PcgArgs a, double* __restrict__ partial) {
    if (a.skip != nullptr && *a.skip) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int c = blockIdx.x;
    const int r0 = a.row_begin[c], r1 = a.row_begin[c + 1];
    const int kb0 = a.row_ptr[r0], nkb = a.row_ptr[r1] - kb0;
    const int t0 = a.touch_off[c], nt = a.touch_off[c + 1] - t0;
    const int chunk = min(kCpChunk, (a.max_kb + 7) & ~7);                   // shared-memory capacity in blocks
    double* Pb = reinterpret_cast<double*>(smem_raw);                         // chunk*16
    int* tb = reinterpret_cast<int*>(Pb + 16 * static_cast<size_t>(chunk));  // touched index of the column aggregate
    int* rowof = tb + chunk;                                                  // solver row of the block
    __shared__ int s_touch[64];
    for (int t = threadIdx.x; t < nt && t < 64; t += blockDim.x) s_touch[t] = a.touch_agg[t0 + t];
    const int l8 = threadIdx.x & 7, g8 = threadIdx.x >> 3, ngroups = blockDim.x >> 3;
    double acc[kCpRounds];
#pragma unroll
    for (int q = 0; q < kCpRounds; ++q) acc[q] = 0.0;
    for (int cb = 0; cb < nkb; cb += chunk) {  // large subdomains: several passes
        const int ce = min(nkb, cb + chunk);
        __syncthreads();  // the previous chunk's reads are done
        for (int j = r0 + threadIdx.x; j < r1; j += blockDim.x) {
            const int b0 = max(a.row_ptr[j] - kb0, cb), b1 = min(a.row_ptr[j + 1] - kb0, ce);
            for (int b = b0; b < b1; ++b) rowof[b - cb] = j;
        }
        __syncthreads();
        for (int lb = cb + threadIdx.x; lb < ce; lb += blockDim.x) {
            const int x = lb - cb;
            const int na = a.row_node[rowof[x]], nb = a.col[kb0 + lb];
            double d[3], e[3];
            node_offset(a, na, d);
            node_offset(a, nb, e);
            const int hb = a.node_agg[nb];
            int t = 0;
            while (t < nt - 1 && s_touch[t] != hb) ++t;
            tb[x] = t;
            const double* K = a.K + static_cast<size_t>(kb0 + lb) * 16;
            double k4[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) k4[q] = K[q];
            double u[4][4];  // u = K_ab psi(b)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
#pragma unroll
                for (int l = 0; l < 3; ++l) u[r][l] = k4[r * 4 + l] + e[l] * k4[r * 4 + 3];
                u[r][3] = k4[r * 4 + 3];
            }
#pragma unroll
            for (int l = 0; l < 4; ++l) {
#pragma unroll
                for (int k = 0; k < 3; ++k) Pb[x * 16 + k * 4 + l] = u[k][l] + d[k] * u[3][l];
                Pb[x * 16 + 12 + l] = u[3][l];
            }
        }
        __syncthreads();
        // 8 lanes per output entry, lane-strided over the blocks (ascending lb)
#pragma unroll
        for (int q = 0; q < kCpRounds; ++q) {
            const int o = q * ngroups + g8;
            if (o >= nt * 16) continue;
            const int t = o >> 4, kl = o & 15;
            for (int x = l8; x < ce - cb; x += 8)
                if (tb[x] == t) acc[q] += Pb[x * 16 + kl];
        }
    }
#pragma unroll
    for (int q = 0; q < kCpRounds; ++q) {
        if (q * ngroups >= nt * 16) break;  // uniform: full-warp shuffles
        double v = acc[q];
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        const int o = q * ngroups + g8;
        if (l8 == 0 && o < nt * 16) partial[(static_cast<size_t>(c) * a.max_touch + (o >> 4)) * 16 + (o & 15)] = v;
    }
}

// One CTA: K0 (g*4+k, h*4+l) = sum over aggregate g's CTAs (in order) of
// their partial for touched aggregate h; symmetrised and inverted in place by
// block Gauss-Jordan on 4x4 node blocks (SPD; modes with a vanishing pivot are
// dropped). Each thread keeps up to kCiTiles 4x4 tiles of K0 in registers for
// the whole inversion; per pivot step only the pivot row / column blocks go
// through shared memory (double-buffered, two barriers per step; stored
// entry-major, X[q * nb + j], so lanes with consecutive tiles hit distinct
// banks: a 16-double stride put every lane of a warp on one bank), so the
// step costs one 4x4x4 product per tile instead of a shared-memory pass over
// the matrix. Deterministic.
constexpr int kCiThreads = 512;
constexpr int kCiTiles = 3;  // n_agg^2 <= kCiThreads * kCiTiles  (n_agg <= 39: the 37 aggregates of 148 CTAs)
__device__ __forceinline__ void mm4(const double* a, const double* b, double* c) {  // c = a b (row-major 4x4)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q)
            c[r * 4 + q] = a[r * 4] * b[q] + a[r * 4 + 1] * b[4 + q] + a[r * 4 + 2] * b[8 + q] + a[r * 4 + 3] * b[12 + q];
}
__global__ void __launch_bounds__(kCiThreads) coarse_invert_kernel(PcgArgs a, const double* __restrict__ partial,
                                                               double* __restrict__ inv, int grid) {
    if (a.skip != nullptr && *a.skip) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nb = a.n_agg, nc = 4 * nb, mt = a.max_touch;
    double* S = reinterpret_cast<double*>(smem_raw);             // nc*nc (symmetrisation)
    double* rowb = S + static_cast<size_t>(nc) * nc;              // 2 x nb x 16: pivot row blocks A_Tj
    double* colb = rowb + 2 * 16 * nb;                            // 2 x nb x 16: pivot column blocks A_iT
    double* Rb = colb + 2 * 16 * nb;                              // 2 x nb x 16: R_j = P A_Tj
    double* Pb = Rb + 2 * 16 * nb;                                // 2 x 16
    int* touch = reinterpret_cast<int*>(Pb + 32);                 // grid * mt
    __shared__ double s_dmax[kCiThreads / 32];
    long long tq = clock64();
    auto cprobe = [&](int slot) {
        if (a.prof != nullptr && threadIdx.x == 0) {
            const long long t = clock64();
            a.prof[slot] += t - tq;
            tq = t;
        }
    };
    for (int i = threadIdx.x; i < grid * mt; i += blockDim.x) {
        const int c = i / mt, t = i - c * mt;
        const int t0 = a.touch_off[c], nt = a.touch_off[c + 1] - t0;
        touch[i] = t < nt ? a.touch_agg[t0 + t] : -1;
    }
    __syncthreads();
    double A[kCiTiles][16];
    int bi[kCiTiles], bj[kCiTiles];
    // fill: tile (g, h) = sum over g's CTAs (CTA order) of their partial for h
#pragma unroll
    for (int u = 0; u < kCiTiles; ++u) {
        const int tile = threadIdx.x + u * blockDim.x;
        bi[u] = tile < nb * nb ? tile / nb : -1;
        bj[u] = tile < nb * nb ? tile - bi[u] * nb : -1;
#pragma unroll
        for (int q = 0; q < 16; ++q) A[u][q] = 0.0;
        if (bi[u] < 0) continue;
        const int c0 = bi[u] * a.agg_ctas, c1 = min(c0 + a.agg_ctas, grid);
        for (int c = c0; c < c1; ++c) {
            int t = 0;
            while (t < mt && touch[c * mt + t] != bj[u]) ++t;
            if (t == mt) continue;
            const double2* src = reinterpret_cast<const double2*>(partial + (static_cast<size_t>(c) * mt + t) * 16);
            double2 x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = __ldcg(src + q);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                A[u][2 * q] += x[q].x;
                A[u][2 * q + 1] += x[q].y;
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) S[(bi[u] * 4 + r) * nc + bj[u] * 4 + q] = A[u][r * 4 + q];
    }
    __syncthreads();
    cprobe(20);
    double dm = 0.0;
#pragma unroll
    for (int u = 0; u < kCiTiles; ++u) {
        if (bi[u] < 0) continue;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = bi[u] * 4 + r, j = bj[u] * 4 + q;
                A[u][r * 4 + q] = 0.5 * (S[i * nc + j] + S[j * nc + i]);
                if (i == j) dm = fmax(dm, fabs(A[u][r * 4 + q]));
            }
    }
    dm = warp_max(dm);
    if ((threadIdx.x & 31) == 0) s_dmax[threadIdx.x >> 5] = dm;
    __syncthreads();
    double dmax = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) dmax = fmax(dmax, s_dmax[w]);
    const double drop = 1e-12 * dmax;
    cprobe(21);
    for (int T = 0; T < nb; ++T) {
        const int par = T & 1;
        double* rowT = rowb + par * 16 * nb;
        double* colT = colb + par * 16 * nb;
        double* RT = Rb + par * 16 * nb;
        double* PT = Pb + par * 16;
        // phase A: pivot inverse (4x4 Gauss-Jordan, dropped modes zeroed) and
        // the pivot row / column blocks
#pragma unroll
        for (int u = 0; u < kCiTiles; ++u) {
            if (bi[u] == T && bj[u] == T) {
                double m[4][4], iv[4][4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        m[r][c] = A[u][r * 4 + c];
                        iv[r][c] = r == c ? 1.0 : 0.0;
                    }
                bool live[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    live[q] = m[q][q] > drop;
                    const double d = live[q] ? rcp_nr(m[q][q]) : 0.0;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        m[q][c] *= d;
                        iv[q][c] *= d;
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        if (r == q) continue;
                        const double f = m[r][q];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            m[r][c] -= f * m[q][c];
                            iv[r][c] -= f * iv[q][c];
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) PT[r * 4 + c] = (live[r] && live[c]) ? iv[r][c] : 0.0;
            }
            if (bi[u] == T)
#pragma unroll
                for (int q = 0; q < 16; ++q) rowT[q * nb + bj[u]] = A[u][q];
            if (bj[u] == T)
#pragma unroll
                for (int q = 0; q < 16; ++q) colT[q * nb + bi[u]] = A[u][q];
        }
        cprobe(24);
        __syncthreads();
        cprobe(25);
        // phase B: R_j = P A_Tj
        for (int j = threadIdx.x; j < nb; j += blockDim.x) {
            double p[16], r[16], o[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                p[q] = PT[q];
                r[q] = rowT[q * nb + j];
            }
            mm4(p, r, o);
#pragma unroll
            for (int q = 0; q < 16; ++q) RT[q * nb + j] = o[q];
        }
        cprobe(26);
        __syncthreads();
        cprobe(27);
        // phase C: A_ij -= C_i R_j; A_Tj = R_j; A_iT = -C_i P; A_TT = P
#pragma unroll
        for (int u = 0; u < kCiTiles; ++u) {
            if (bi[u] < 0) continue;
            if (bi[u] == T) {
#pragma unroll
                for (int q = 0; q < 16; ++q) A[u][q] = bj[u] == T ? PT[q] : RT[q * nb + bj[u]];
                continue;
            }
            double cm[16], o[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) cm[q] = colT[q * nb + bi[u]];
            if (bj[u] == T) {
                double p[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) p[q] = PT[q];
                mm4(cm, p, o);
#pragma unroll
                for (int q = 0; q < 16; ++q) A[u][q] = -o[q];
            } else {
                double r[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) r[q] = RT[q * nb + bj[u]];
                mm4(cm, r, o);
#pragma unroll
                for (int q = 0; q < 16; ++q) A[u][q] -= o[q];
            }
        }
        cprobe(28);
    }
    cprobe(22);
#pragma unroll
    for (int u = 0; u < kCiTiles; ++u) {
        if (bi[u] < 0) continue;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) inv[static_cast<size_t>(bi[u] * 4 + r) * nc + bj[u] * 4 + q] = A[u][r * 4 + q];
    }
}

// Larger coarse spaces (n_agg^2 > kCiThreads * kCiTiles): K0 assembled in
// shared memory and inverted by the shared-memory blocked Gauss-Jordan.
__global__ void __launch_bounds__(1024) coarse_invert_smem_kernel(PcgArgs a, const double* __restrict__ partial,
                                                                   double* __restrict__ inv, int grid) {
    if (a.skip != nullptr && *a.skip) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nb = a.n_agg, nc = 4 * nb, mt = a.max_touch;
    double* A = reinterpret_cast<double*>(smem_raw);  // nc*nc
    double* colk = A + static_cast<size_t>(nc) * nc;   // 4 * nc
    double* rowk = colk + 4 * nc;                      // 4 * nc
    int* touch = reinterpret_cast<int*>(rowk + 4 * nc);  // grid * mt
    __shared__ double s_dmax, s_pb[16];
    __shared__ int s_blocks;
    for (int i = threadIdx.x; i < grid * mt; i += blockDim.x) {
        const int c = i / mt, t = i - c * mt;
        const int t0 = a.touch_off[c], nt = a.touch_off[c + 1] - t0;
        touch[i] = t < nt ? a.touch_agg[t0 + t] : -1;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < nc * nc; o += blockDim.x) {
        const int i = o / nc, j = o - i * nc;
        const int g = i >> 2, k = i & 3, h = j >> 2, l = j & 3;
        const int c0 = g * a.agg_ctas, c1 = min(c0 + a.agg_ctas, grid);
        double sum = 0.0;
        for (int c = c0; c < c1; ++c) {
            int t = 0;
            while (t < mt && touch[c * mt + t] != h) ++t;
            if (t < mt) sum += __ldcg(partial + (static_cast<size_t>(c) * mt + t) * 16 + k * 4 + l);
        }
        A[o] = sum;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < nc * nc; o += blockDim.x) {
        const int i = o / nc, j = o - i * nc;
        if (j < i) {
            const double v = 0.5 * (A[i * nc + j] + A[j * nc + i]);
            A[i * nc + j] = v;
            A[j * nc + i] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int i = 0; i < nc; ++i) m = fmax(m, fabs(A[i * nc + i]));
        s_dmax = m;
        s_blocks = nb;
    }
    __syncthreads();
    block_gj_inverse(A, 1, &s_blocks, nc, 0, s_pb, colk, rowk, &s_dmax, 1e-12);
    for (int o = threadIdx.x; o < nc * nc; o += blockDim.x) inv[o] = A[o];
}

// ---------------------------------------------------------------- subdomain inverses
// CTA c (same row partition as the PCG grid): the CTA's rows are split into
// chunks of at most sub_rows consecutive (RCB-local) nodes; M_k = exact
// inverse of each chunk's 4s x 4s diagonal block of K (blocked Gauss-Jordan,
// block_gj_inverse), written to out[c][k][4s x sub_ld].
constexpr int kInvThreads = 1024;
__global__ void __launch_bounds__(kInvThreads, 1) sub_invert_kernel(PcgArgs a, double* __restrict__ out) {
    if (a.skip != nullptr && *a.skip) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int cta = blockIdx.x;
    const int r0 = a.row_begin[cta], r1 = a.row_begin[cta + 1], nrows = r1 - r0;
    const int S = a.sub_rows, ld = a.sub_ld, nch = (nrows + S - 1) / S;
    const size_t msz = static_cast<size_t>(4) * S * ld;
    double* A = reinterpret_cast<double*>(smem_raw);          // nch * msz
    double* cb = A + nch * msz;                               // nch * 4 * ld
    double* rb = cb + static_cast<size_t>(nch) * 4 * ld;       // nch * 4 * ld
    double* pb = rb + static_cast<size_t>(nch) * 4 * ld;       // nch * 16
    double* dmax = pb + 16 * nch;                             // nch
    int* cstart = reinterpret_cast<int*>(dmax + nch);         // nch + 1
    int* blocks = cstart + nch + 1;                           // nch
    for (int k = threadIdx.x; k <= nch; k += blockDim.x) cstart[k] = (k * nrows) / nch;
    for (size_t i = threadIdx.x; i < nch * msz; i += blockDim.x) A[i] = 0.0;
    __syncthreads();
    // scatter the own-row K blocks that fall inside the row's chunk
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int lr = w; lr < nrows; lr += nw) {
        int k = 0;
        while (cstart[k + 1] <= lr) ++k;
        const int st = cstart[k], en = cstart[k + 1];
        const int j = r0 + lr;
        for (int t = a.row_ptr[j] * 16 + lane; t < a.row_ptr[j + 1] * 16; t += 32) {
            const int b = t >> 4, e = t & 15;
            const int cl = a.colx[b];  // own rows come first in the CTA operand order
            if (cl >= st && cl < en) A[k * msz + ((lr - st) * 4 + (e >> 2)) * ld + (cl - st) * 4 + (e & 3)] = a.K[t];
        }
    }
    __syncthreads();
    if (threadIdx.x < nch) {
        const int k = threadIdx.x;
        blocks[k] = cstart[k + 1] - cstart[k];
        double m = 0.0;
        for (int q = 0; q < 4 * blocks[k]; ++q) m = fmax(m, fabs(A[k * msz + static_cast<size_t>(q) * ld + q]));
        dmax[k] = m;
    }
    __syncthreads();
    block_gj_inverse(A, nch, blocks, ld, msz, pb, cb, rb, dmax, 1e-13);
    double* o = out + static_cast<size_t>(cta) * a.sub_chunks * msz;
    for (int gi = w; gi < 4 * nrows; gi += nw) {
        int k = 0, base = 0;
        while (gi >= base + 4 * blocks[k]) base += 4 * blocks[k++];
        const int i = gi - base, nk = 4 * blocks[k];
        for (int jj = lane; jj < nk; jj += 32) o[k * msz + static_cast<size_t>(i) * ld + jj] = A[k * msz + static_cast<size_t>(i) * ld + jj];
    }
}

// ---------------------------------------------------------------- PCG
struct Shared {
    double* K;       // nkb*16
    int* col;        // nkb
    double* Minv;    // per subdomain chunk: dense inverse of its 4s x 4s diagonal block (leading dim sub_ld)
    double* zz;      // nrows*12: M_sub v
    int* cstart;     // chunk row ranges [cstart[k], cstart[k+1])
    int* rchunk;     // own row -> chunk
    double* rex;     // nrows*12: M_sub input
    double* offx;    // operand rows x 3: node offset to its aggregate centre
    int* tl;         // operand rows: index of its aggregate in the CTA's touched list
    double* cinv;    // touched aggregates x 4 rows of K0^-1 (nc each)
    double* yt;      // touched aggregates x 12: coarse correction
    double* ptq;     // nc x 3 aggregate sums of Psi^T v (replicated)
    double* red;     // kRedDoubles: reduction scratch
    double* bcast;   // kQ
    double* ext;     // (own rows + halo) x 12: the SpMV operand staged from L2
    int* rp;         // max_rows + 1: block range starts of the own rows, relative to the CTA's first block
    int* rnode;      // max_rows: node id of the own rows
};

__device__ __forceinline__ double op2(bool mx, double a, double b) { return mx ? fmax(a, b) : a + b; }

// Block reduction of the 32 per-thread slots into part[blockIdx*kQ + k]
// (sum, or max for slots in max_mask). Within a warp a transpose-reduce
// halves the vector at every butterfly level (16+8+4+2+1 shuffles instead of
// 32x5) and leaves slot l in lane l; then warps combine the per-warp totals
// of each slot. Fixed order.
__device__ __forceinline__ void block_partials(const double* vals, int nq, double* red, double* part,
                                               unsigned max_mask) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double v16[16], v8[8], v4[4], v2[2], v1;
    int base = 0;
    {
        const bool up = lane & 16;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const double keep = up ? vals[i + 16] : vals[i], send = up ? vals[i] : vals[i + 16];
            const int slot = (up ? 16 : 0) + i;
            v16[i] = op2((max_mask >> slot) & 1u, keep, __shfl_xor_sync(0xffffffffu, send, 16));
        }
        base += up ? 16 : 0;
    }
    {
        const bool up = lane & 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double keep = up ? v16[i + 8] : v16[i], send = up ? v16[i] : v16[i + 8];
            const int slot = base + (up ? 8 : 0) + i;
            v8[i] = op2((max_mask >> slot) & 1u, keep, __shfl_xor_sync(0xffffffffu, send, 8));
        }
        base += up ? 8 : 0;
    }
    {
        const bool up = lane & 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double keep = up ? v8[i + 4] : v8[i], send = up ? v8[i] : v8[i + 4];
            const int slot = base + (up ? 4 : 0) + i;
            v4[i] = op2((max_mask >> slot) & 1u, keep, __shfl_xor_sync(0xffffffffu, send, 4));
        }
        base += up ? 4 : 0;
    }
    {
        const bool up = lane & 2;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double keep = up ? v4[i + 2] : v4[i], send = up ? v4[i] : v4[i + 2];
            const int slot = base + (up ? 2 : 0) + i;
            v2[i] = op2((max_mask >> slot) & 1u, keep, __shfl_xor_sync(0xffffffffu, send, 2));
        }
        base += up ? 2 : 0;
    }
    {
        const bool up = lane & 1;
        const double keep = up ? v2[1] : v2[0], send = up ? v2[0] : v2[1];
        const int slot = base + (up ? 1 : 0);
        v1 = op2((max_mask >> slot) & 1u, keep, __shfl_xor_sync(0xffffffffu, send, 1));
        base = slot;  // == lane
    }
    red[base * 32 + w] = v1;
    __syncthreads();
    for (int q = w; q < nq; q += nw) {
        const bool mx = (max_mask >> q) & 1u;
        double v = lane < nw ? red[q * 32 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = op2(mx, v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) part[blockIdx.x * kQ + q] = v;
    }
    __syncthreads();
}

// grid totals of slots [0, nq) (sum or max per mask) into bcast; one warp per
// slot. All of a lane's partials are loaded before any is combined (the grid
// is at most kMaxGridLoads*32 CTAs), so the reads cost one L2 round trip.
constexpr int kMaxGridLoads = 5;  // 160 CTAs
__device__ __forceinline__ void grid_totals(const double* __restrict__ part, int G, double* bcast, int nq,
                                            unsigned max_mask) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w < nq) {
        const bool mx = (max_mask >> w) & 1u;
        double x[kMaxGridLoads];
#pragma unroll
        for (int i = 0; i < kMaxGridLoads; ++i) {
            const int g = lane + 32 * i;
            x[i] = g < G ? __ldcg(part + g * kQ + w) : 0.0;
        }
        double v = x[0];
#pragma unroll
        for (int i = 1; i < kMaxGridLoads; ++i) v = mx ? fmax(v, x[i]) : v + x[i];
        v = mx ? warp_max(v) : warp_sum(v);
        if (lane == 0) bcast[w] = v;
    }
}

// per-aggregate sums of the 12 Psi^T slots [s0, s0+12) into out[nc x 3]:
// out[(g*4+k)*3 + c] = sum over the aggregate's CTAs of part[cta][s0 + k*3 + c]
// (fixed order). Runs on the warps after the grid_totals warps (w >= 4) so
// both reductions overlap; loads are issued 8 at a time before combining.
__device__ __forceinline__ void aggregate_sums(const PcgArgs& a, const double* __restrict__ part, int G, int s0,
                                               double* out, int first_warp) {
    const int nc = 4 * a.n_agg;
    const int first = first_warp * 32;
    if (static_cast<int>(threadIdx.x) < first) return;
    for (int o = threadIdx.x - first; o < nc * 3; o += blockDim.x - first) {
        const int g = o / 12, kc = o % 12;
        const int c0 = g * a.agg_ctas, c1 = min((g + 1) * a.agg_ctas, G);
        double s = 0.0;
        for (int cb = c0; cb < c1; cb += 8) {
            double x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = cb + i < c1 ? __ldcg(part + (cb + i) * kQ + s0 + kc) : 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) s += x[i];
        }
        out[o] = s;
    }
}

// Per-iteration CTA partials of the 7 per-thread values (gamma, delta, max|r|
// and the 4 Psi^T w mode sums; all of a thread's elements share one column c =
// threadIdx % 3). Each value goes to shared memory grouped by column class,
// then one half-warp per output slot sums its 128 (or, for max|r|, 384)
// entries in a fixed order: 7 shared stores per thread instead of a 32-slot
// shuffle transpose. Slots: 0-2 gamma by column, 3-5 delta, 6 max|r|,
// 7 + 3m + c mode m (as grid_totals / aggregate_sums read them).
constexpr int kClass = kPcgThreads / 3;
// The iteration partials are written kPartReplicas times and each CTA reads
// replica (cta % kPartReplicas): right after the barrier all CTAs read the
// same few KB, and replication spreads those reads over more L2 slices.
constexpr int kPartReplicas = 8;
constexpr int kRedDoubles = 7 * kPcgThreads;
static_assert(kRedDoubles >= 32 * kQ, "reduction scratch");
__device__ __forceinline__ void partials_stage(double g, double dl, double rmx, const double ps[4], double* red) {
    const int t = threadIdx.x, c = t % 3, i = t / 3;
    red[(0 * 3 + c) * kClass + i] = g;
    red[(1 * 3 + c) * kClass + i] = dl;
#pragma unroll
    for (int m = 0; m < 4; ++m) red[((2 + m) * 3 + c) * kClass + i] = ps[m];
    red[18 * kClass + t] = rmx;
}
// after a barrier that follows partials_stage
__device__ __forceinline__ void partials_reduce(int nq, const double* red, double* part) {
    const int t = threadIdx.x;
    const int s = t >> 4, hl = t & 15;
    const bool mx = s == 6;
    double v = 0.0;
    if (s < nq) {
        if (mx) {
            double x[kPcgThreads / 16];
#pragma unroll
            for (int k = 0; k < kPcgThreads / 16; ++k) x[k] = red[18 * kClass + hl + 16 * k];
            v = x[0];
#pragma unroll
            for (int k = 1; k < kPcgThreads / 16; ++k) v = fmax(v, x[k]);
        } else {
            const int blk = s < 6 ? s : s - 1;
            double x[kClass / 16];
#pragma unroll
            for (int k = 0; k < kClass / 16; ++k) x[k] = red[blk * kClass + hl + 16 * k];
            v = x[0];
#pragma unroll
            for (int k = 1; k < kClass / 16; ++k) v += x[k];
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v = op2(mx, v, __shfl_xor_sync(0xffffffffu, v, o));
    if (hl == 0 && s < nq) {
        const size_t rs = static_cast<size_t>(kQ) * ((gridDim.x + 7) & ~7);
#pragma unroll
        for (int r = 0; r < kPartReplicas; ++r) part[r * rs + s * ((gridDim.x + 7) & ~7) + blockIdx.x] = v;
    }
}

// Grid totals of slots 0-6 (warps 0-6, one slot each) and the aggregate sums
// of the Psi^T slots (one output per thread) with every L2 load issued before
// any is combined: one round trip. The partials are slot-major (part[s][cta],
// row length round_up(G, 8)): every CTA reads the same few KB right after the
// barrier, so the number of L2 sector requests, not latency, sets the cost;
// this layout makes a slot's grid total 37 sectors and an aggregate sum two
// 32-byte vector loads; the partials are also replicated (kPartReplicas). Same summation order as grid_totals / aggregate_sums.
__device__ __forceinline__ void iter_totals(const PcgArgs& a, const double* __restrict__ part, int G, double* bcast,
                                            double* ptq) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nc = 4 * a.n_agg, Gp = (G + 7) & ~7;
    part += static_cast<size_t>(blockIdx.x % kPartReplicas) * kQ * Gp;  // this CTA's replica
    const bool tot = w < 7;
    double xt[kMaxGridLoads];
#pragma unroll
    for (int i = 0; i < kMaxGridLoads; ++i) {
        const int g = lane + 32 * i;
        xt[i] = tot && g < G ? __ldcg(part + w * Gp + g) : 0.0;
    }
    double2 xa[4];
    const bool fast = a.use_coarse && a.agg_ctas == 8;
    // 4 CTAs per aggregate: 32-byte aligned, zero padded; a thread's two
    // outputs (o, o + blockDim) are loaded together
    const bool fast4 = a.use_coarse && a.agg_ctas == 4 && nc * 3 <= 2 * static_cast<int>(blockDim.x);
    if (fast4) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int o = threadIdx.x + h * blockDim.x;
            xa[2 * h] = xa[2 * h + 1] = make_double2(0.0, 0.0);
            if (o < nc * 3) {
                const int g = o / 12, kc = o % 12;
                const double2* src = reinterpret_cast<const double2*>(part + (7 + kc) * Gp + 4 * g);
                xa[2 * h] = __ldcg(src);
                xa[2 * h + 1] = __ldcg(src + 1);
            }
        }
    }
    for (int o = threadIdx.x; a.use_coarse && !fast4 && o < nc * 3; o += blockDim.x) {
        const int g = o / 12, kc = o % 12;
        const int c0 = g * a.agg_ctas, c1 = min(c0 + a.agg_ctas, G);
        const double* src = part + (7 + kc) * Gp + c0;
        if (fast && o == static_cast<int>(threadIdx.x)) {  // 8 CTAs, 64-byte aligned, zero padded
#pragma unroll
            for (int i = 0; i < 4; ++i) xa[i] = __ldcg(reinterpret_cast<const double2*>(src) + i);
            continue;
        }
        double s = 0.0;
        for (int cb = c0; cb < c1; cb += 8) {
            double x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = cb + i < c1 ? __ldcg(part + (7 + kc) * Gp + cb + i) : 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) s += x[i];
        }
        ptq[o] = s;
    }
    if (tot) {
        const bool mx = w == 6;
        double v = xt[0];
#pragma unroll
        for (int i = 1; i < kMaxGridLoads; ++i) v = mx ? fmax(v, xt[i]) : v + xt[i];
        v = mx ? warp_max(v) : warp_sum(v);
        if (lane == 0) bcast[w] = v;
    }
    if (fast && static_cast<int>(threadIdx.x) < nc * 3) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            s += xa[i].x;
            s += xa[i].y;
        }
        ptq[threadIdx.x] = s;
    }
    if (fast4) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int o = threadIdx.x + h * blockDim.x;
            if (o < nc * 3) ptq[o] = ((xa[2 * h].x + xa[2 * h].y) + xa[2 * h + 1].x) + xa[2 * h + 1].y;
        }
    }
}

template <int EPT>
__global__ void __launch_bounds__(kPcgThreads, 1) pcg_kernel(PcgArgs a_param) {
    if (a_param.skip != nullptr && *a_param.skip) return;  // every CTA: before any grid barrier
    cg::grid_group grid = cg::this_grid();
    // The arguments are read from shared memory inside the loop: every grid
    // barrier's gpu-scope fence invalidates the SM's caches, and a constant
    // bank reload after it cost ~1.5K cycles per iteration (NRR_PROF probes).
    __shared__ PcgArgs s_args;
    if (threadIdx.x == 0) s_args = a_param;
    __syncthreads();
    const PcgArgs& a = s_args;
    const long long t_entry = clock64();
    long long t_probe = t_entry;
    const bool sprof = a.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    auto probe = [&](int slot) {
        if (sprof) {
            const long long t = clock64();
            a.prof[slot] += t - t_probe;
            t_probe = t;
        }
    };
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int cta = blockIdx.x, G = gridDim.x;
    const int r0 = a.row_begin[cta], r1 = a.row_begin[cta + 1];
    const int nrows = r1 - r0;
    const int kb0 = a.row_ptr[r0], nkb = a.row_ptr[r1] - kb0;
    const int nc = 4 * a.n_agg;
    const int e0 = a.ext_off[cta], n_ext = a.ext_off[cta + 1] - e0;
    const int t0 = a.touch_off[cta], nt = a.touch_off[cta + 1] - t0;
    Shared sh;
    {
        double* p = reinterpret_cast<double*>(smem_raw);
        sh.red = p;
        p += kRedDoubles;
        sh.bcast = p;
        p += kQ;
        sh.Minv = p;  // offset kRedDoubles + kQ doubles: even -> 16-byte aligned
        p += static_cast<size_t>(a.sub_chunks) * 4 * a.sub_rows * a.sub_ld;
        sh.zz = p;
        p += 12 * a.max_rows;
        sh.rex = p;
        p += 12 * a.max_rows;
        sh.offx = p;
        p += 3 * static_cast<size_t>(a.max_ext);
        sh.cinv = p;
        if (a.use_coarse) p += 4 * static_cast<size_t>(a.max_touch) * nc;  // as PcgPlan::size_smem
        sh.yt = p;
        p += 12 * a.max_touch;
        sh.ptq = p;
        p += 3 * kCoarseMax;
        sh.ext = p;
        p += 12 * static_cast<size_t>(a.max_ext);
        sh.cstart = reinterpret_cast<int*>(p);
        p += (a.sub_chunks + 2) / 2;
        sh.rchunk = reinterpret_cast<int*>(p);
        p += (a.max_rows + 1) / 2;
        sh.tl = reinterpret_cast<int*>(p);
        p += (a.max_ext + 1) / 2;
        sh.rp = reinterpret_cast<int*>(p);
        p += (a.max_rows + 2) / 2;
        sh.rnode = reinterpret_cast<int*>(p);
        p += (a.max_rows + 1) / 2;
        if ((p - reinterpret_cast<double*>(smem_raw)) & 1) ++p;  // 16-byte aligned K
        if (a.k_in_smem) {
            sh.K = p;
            p += 16 * static_cast<size_t>(a.max_kb);
            sh.col = reinterpret_cast<int*>(p);
        } else {
            sh.K = const_cast<double*>(a.K) + static_cast<size_t>(kb0) * 16;
            sh.col = const_cast<int*>(a.colx) + kb0;
        }
    }
    if (a.k_in_smem) {
        const double2* src = reinterpret_cast<const double2*>(a.K + static_cast<size_t>(kb0) * 16);
        double2* dst = reinterpret_cast<double2*>(sh.K);
        for (int i = threadIdx.x; i < nkb * 8; i += blockDim.x) dst[i] = src[i];
        for (int i = threadIdx.x; i < nkb; i += blockDim.x) sh.col[i] = a.colx[kb0 + i];
    }
    probe(10);  // K -> smem issued
    // coarse rows of the aggregates this CTA's operand rows touch, and every
    // operand row's offset to its aggregate centre (own rows come first)
    if (a.use_coarse) {
        for (int i = threadIdx.x; i < nt * 4 * nc; i += blockDim.x) {
            const int t = i / (4 * nc), kj = i - t * 4 * nc;
            sh.cinv[i] = a.coarse_inv[static_cast<size_t>(a.touch_agg[t0 + t]) * 4 * nc + kj];
        }
    }
    for (int lr = threadIdx.x; lr <= nrows; lr += blockDim.x) {
        sh.rp[lr] = a.row_ptr[r0 + lr] - kb0;
        if (lr < nrows) sh.rnode[lr] = a.row_node[r0 + lr];
    }
    for (int e = threadIdx.x; e < n_ext; e += blockDim.x) {
        double d3[3];
        node_offset(a, a.ext_node[e0 + e], d3);
        for (int t = 0; t < 3; ++t) sh.offx[e * 3 + t] = d3[t];
        sh.tl[e] = a.ext_tl[e0 + e];
    }
    // ---- 4x4 diagonal blocks must be PD (reference describe_failure)
    for (int lr = threadIdx.x; lr < nrows; lr += blockDim.x) {
        const int j = r0 + lr;
        const int node = a.row_node[j];
        int dpos = -1;
        for (int b = a.row_ptr[j]; b < a.row_ptr[j + 1]; ++b)
            if (a.col[b] == node) dpos = b;
        double k[16], l[16] = {0};
        for (int t = 0; t < 16; ++t) k[t] = a.K[static_cast<size_t>(dpos) * 16 + t];
        double dmax = 0;
        for (int t = 0; t < 4; ++t) dmax = fmax(dmax, fabs(k[t * 5]));
        bool ok = dmax > 0 && isfinite(dmax);
        for (int c = 0; c < 4 && ok; ++c) {
            double s = k[c * 4 + c];
            for (int t = 0; t < c; ++t) s -= l[c * 4 + t] * l[c * 4 + t];
            if (!(s > 0.0)) {  // the block is not PD (reference describe_failure: min eigenvalue <= 0)
                ok = false;
                break;
            }
            const double d = sqrt(s);
            l[c * 4 + c] = d;
            for (int r = c + 1; r < 4; ++r) {
                double v = k[r * 4 + c];
                for (int t = 0; t < c; ++t) v -= l[r * 4 + t] * l[c * 4 + t];
                l[r * 4 + c] = v / d;
            }
        }
        if (!ok) atomicMin(&a.status->fail_node, node);
    }
    probe(11);  // coarse rows + 4x4 checks
    // ---- subdomain block Jacobi: M_k (dense inverses of the CTA's chunk
    // diagonal blocks, sub_invert_kernel) staged into shared memory
    const int sub_ld = a.sub_ld;
    const size_t sub_msz = static_cast<size_t>(4) * a.sub_rows * sub_ld;
    {
        const int S = a.sub_rows;
        const int nch = (nrows + S - 1) / S;
        for (int k = threadIdx.x; k <= nch; k += blockDim.x) sh.cstart[k] = (k * nrows) / nch;
        const double2* src = reinterpret_cast<const double2*>(a.sub_inv + static_cast<size_t>(cta) * a.sub_chunks * sub_msz);
        double2* dst = reinterpret_cast<double2*>(sh.Minv);
        for (size_t i = threadIdx.x; i < nch * sub_msz / 2; i += blockDim.x) dst[i] = __ldcg(src + i);
        __syncthreads();
        for (int lr = threadIdx.x; lr < nrows; lr += blockDim.x) {
            int k = 0;
            while (sh.cstart[k + 1] <= lr) ++k;
            sh.rchunk[lr] = k;
        }
    }
    __syncthreads();

    // Element e = threadIdx.x + k*blockDim (blockDim % 12 == 0): the scalar row
    // r and column c are the same for all of a thread's elements, so every
    // per-thread reduction is a scalar register (no dynamic indexing, no
    // local memory).
    const int nel = nrows * 12;
    const int my_rc = threadIdx.x % 12, my_r = my_rc / 3, my_c = my_rc % 3;
    // kLean (4 or more elements per thread): x and the search direction p only
    // accumulate (nothing else in the iteration reads them), so they live in
    // global memory (X itself and the scratch P) instead of 4 registers per
    // element
    constexpr bool kLean = EPT >= 4;
    constexpr int kXp = kLean ? 1 : EPT;
    double xr[kXp], pr[kXp];
    double rr[EPT], ur[EPT], wr[EPT], sr[EPT], qr[EPT], zv[EPT];  // B is re-read at a restart
    // With 4 or more elements per thread the block ranges and global offsets
    // are looked up in shared memory (rp / rnode) instead of held in
    // registers: 5 registers per element, which pcg_kernel<4> spilled
    constexpr int kIdx = kLean ? 1 : EPT;
    int el_row[EPT], el_b0[kIdx], el_b1[kIdx];  // row, block range in the CTA's K
    size_t el_gr[kIdx];
    auto el_g = [&](int k) -> size_t {
        if constexpr (kLean)
            return static_cast<size_t>(sh.rnode[el_row[k]]) * 12 + my_rc;
        else
            return el_gr[k];
    };
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const int e = threadIdx.x + k * blockDim.x;
        const bool live = e < nel;
        const int lr = live ? e / 12 : 0;
        el_row[k] = live ? lr : -1;
        if constexpr (!kLean) {
            el_b0[k] = a.row_ptr[r0 + lr] - kb0;
            el_b1[k] = live ? a.row_ptr[r0 + lr + 1] - kb0 : el_b0[k];
            el_gr[k] = static_cast<size_t>(a.row_node[r0 + lr]) * 12 + my_rc;
        }
        if constexpr (!kLean) {
            xr[k] = live ? a.X[el_g(k)] : 0.0;
            pr[k] = 0.0;
        }
        rr[k] = ur[k] = wr[k] = sr[k] = qr[k] = zv[k] = 0.0;
    }

    // Parities of the exchanged vector Z and of the iteration partials: every
    // publish (write before a grid barrier, read by other CTAs after it)
    // alternates between two buffers. With one barrier per iteration a CTA
    // that leaves the barrier early can finish the next iteration's local
    // work and publish again while a late CTA is still reading the previous
    // publish; with two buffers that write goes to the other parity, and the
    // next write to this parity needs the late CTA at the next barrier first.
    int zph = 0, pph = 0;
    // the thread's first kHaloRegs halo elements: global offsets resolved once,
    // so a fill is kHaloRegs independent L2 loads (one round trip)
    constexpr int kHaloRegs = 4;
    int hoff[kHaloRegs];
#pragma unroll
    for (int k = 0; k < kHaloRegs; ++k) {
        const int t = nrows * 12 + threadIdx.x + k * blockDim.x;
        hoff[k] = t < n_ext * 12 ? a.ext_node[e0 + t / 12] * 12 + t % 12 : -1;
    }
    // halo rows of v (other CTAs' rows, published before the last grid
    // barrier) -> ext; with `totals`, the iteration's grid totals and
    // aggregate sums are loaded in the same L2 round trip
    auto exchange = [&](const double* __restrict__ v, bool totals) {
        double hv[kHaloRegs];
#pragma unroll
        for (int k = 0; k < kHaloRegs; ++k) hv[k] = hoff[k] >= 0 ? __ldcg(v + hoff[k]) : 0.0;
        if (totals) iter_totals(a, a.part_a + pph * a.part_stride, G, sh.bcast, sh.ptq);
        for (int t = nrows * 12 + threadIdx.x + kHaloRegs * blockDim.x; t < n_ext * 12; t += blockDim.x)
            sh.ext[t] = __ldcg(v + static_cast<size_t>(a.ext_node[e0 + t / 12]) * 12 + t % 12);
#pragma unroll
        for (int k = 0; k < kHaloRegs; ++k)
            if (hoff[k] >= 0) sh.ext[nrows * 12 + threadIdx.x + k * blockDim.x] = hv[k];
        __syncthreads();
    };
    auto spmv = [&](int k) -> double {
        int b0, b1;  // empty range for dead elements
        if constexpr (kLean) {
            const int lr = el_row[k];
            b0 = lr >= 0 ? sh.rp[lr] : 0;
            b1 = lr >= 0 ? sh.rp[lr + 1] : 0;
        } else {
            b0 = el_b0[k];
            b1 = el_b1[k];
        }
        // four independent chains, all of a group's loads issued before its
        // FMAs (K comes from L2 when it does not fit in shared memory)
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        int b = b0;
        for (; b + 3 < b1; b += 4) {
            int cc[4];
            double2 ka[4], kb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                cc[u] = sh.col[b + u];
                const double* kp = sh.K + static_cast<size_t>(b + u) * 16 + my_r * 4;
                ka[u] = *reinterpret_cast<const double2*>(kp);
                kb[u] = *reinterpret_cast<const double2*>(kp + 2);
            }
            double vv[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double* v = sh.ext + cc[u] * 12 + my_c;
                vv[u][0] = v[0];
                vv[u][1] = v[3];
                vv[u][2] = v[6];
                vv[u][3] = v[9];
            }
            acc0 = fma(ka[0].x, vv[0][0], acc0);
            acc1 = fma(ka[1].x, vv[1][0], acc1);
            acc2 = fma(ka[2].x, vv[2][0], acc2);
            acc3 = fma(ka[3].x, vv[3][0], acc3);
            acc0 = fma(ka[0].y, vv[0][1], acc0);
            acc1 = fma(ka[1].y, vv[1][1], acc1);
            acc2 = fma(ka[2].y, vv[2][1], acc2);
            acc3 = fma(ka[3].y, vv[3][1], acc3);
            acc0 = fma(kb[0].x, vv[0][2], acc0);
            acc1 = fma(kb[1].x, vv[1][2], acc1);
            acc2 = fma(kb[2].x, vv[2][2], acc2);
            acc3 = fma(kb[3].x, vv[3][2], acc3);
            acc0 = fma(kb[0].y, vv[0][3], acc0);
            acc1 = fma(kb[1].y, vv[1][3], acc1);
            acc2 = fma(kb[2].y, vv[2][3], acc2);
            acc3 = fma(kb[3].y, vv[3][3], acc3);
        }
        for (; b < b1; ++b) {
            const double* kk = sh.K + static_cast<size_t>(b) * 16 + my_r * 4;
            const double* v = sh.ext + sh.col[b] * 12 + my_c;
            acc0 = fma(kk[0], v[0], acc0);
            acc0 = fma(kk[1], v[3], acc0);
            acc0 = fma(kk[2], v[6], acc0);
            acc0 = fma(kk[3], v[9], acc0);
        }
        acc0 += acc1;
        acc2 += acc3;
        return acc0 + acc2;
    };
    // Psi^T contribution of the thread's elements (own column): 4 mode sums
    auto psi_acc = [&](int k, double v, double ps[4]) {
        const int lr = el_row[k];
        if (lr < 0) return;
        if (my_r < 3) {
            ps[my_r] += v;
        } else {
            ps[0] += sh.offx[lr * 3 + 0] * v;
            ps[1] += sh.offx[lr * 3 + 1] * v;
            ps[2] += sh.offx[lr * 3 + 2] * v;
            ps[3] += v;
        }
    };
    double vals[kQ];
    auto zero_vals = [&]() {
#pragma unroll
        for (int j = 0; j < kQ; ++j) vals[j] = 0.0;
    };
    auto put_psi = [&](int base, const double ps[4]) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int c = 0; c < 3; ++c) vals[base + m * 3 + c] = c == my_c ? ps[m] : 0.0;
    };
    const bool prof = a.prof != nullptr && cta == 0 && threadIdx.x == 0;
    long long tp = clock64(), acc_t[16] = {0};
    const long long t_setup = tp - t_entry;
    auto mark = [&](int slot) {
        if (kPcgProbes && prof) {
            const long long t = clock64();
            acc_t[slot] += t - tp;
            tp = t;
        }
    };
    // m' = M_sub v (the subdomain part of the preconditioner) for the own rows:
    // -> ext own rows and the global exchange buffer Z. 4 threads per scalar
    // row split the chunk's columns, butterfly-combined in a fixed order.
    // with_partials: the iteration partials were staged with the input; their
    // CTA reduction shares this routine's first barrier
    auto precond_sub = [&](const double (&v)[EPT], bool with_partials) {
        if constexpr (NRR_PCG_DIRECT != 0 || EPT >= 2) {
        // every thread forms its own elements' m' = (M_sub v)_e: the input is
        // staged column-major by right-hand side (rexT[c][scalar row], leading
        // dimension = 2 mod 16 doubles so the three columns' 16-byte loads hit
        // distinct banks), M_sub rows and the input are read with 16-byte
        // loads, four independent chains; no partial-sum shuffles, no second
        // staging buffer and no second barrier
        double* rexT = sh.zz;  // zz and rex are contiguous: 24 max_rows doubles
        const int ldr = 4 * a.max_rows + 2;
#pragma unroll
        for (int k = 0; k < EPT; ++k)
            if (el_row[k] >= 0) rexT[my_c * ldr + 4 * el_row[k] + my_r] = v[k];
        __syncthreads();
        if (with_partials) partials_reduce(a.use_coarse ? 19 : 7, sh.red, a.part_a + pph * a.part_stride);
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            if (el_row[k] < 0) continue;
            const int lr = el_row[k];
            const int ch = sh.rchunk[lr], st = sh.cstart[ch];
            const int nk = 4 * (sh.cstart[ch + 1] - st);
            const double2* m = reinterpret_cast<const double2*>(sh.Minv + ch * sub_msz +
                                                                static_cast<size_t>(4 * (lr - st) + my_r) * sub_ld);
            const double2* rv = reinterpret_cast<const double2*>(rexT + my_c * ldr + 4 * st);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 4
            for (int j = 0; j < nk / 2; j += 2) {
                const double2 m01 = m[j], m23 = m[j + 1];
                const double2 r01 = rv[j], r23 = rv[j + 1];
                a0 = fma(m01.x, r01.x, a0);
                a1 = fma(m01.y, r01.y, a1);
                a2 = fma(m23.x, r23.x, a2);
                a3 = fma(m23.y, r23.y, a3);
            }
            const double z = (a0 + a1) + (a2 + a3);
            __stcg(a.Z + zph * a.z_stride + el_g(k), z);
            sh.ext[lr * 12 + my_rc] = z;
        }
        return;
        }
#pragma unroll
        for (int k = 0; k < EPT; ++k)
            if (el_row[k] >= 0) sh.rex[el_row[k] * 12 + my_rc] = v[k];
        __syncthreads();
        if (with_partials) partials_reduce(a.use_coarse ? 19 : 7, sh.red, a.part_a + pph * a.part_stride);
        for (int t = threadIdx.x; t < 16 * nrows; t += blockDim.x) {
            const int i = t >> 2, q = t & 3, lr = i >> 2;
            const int ch = sh.rchunk[lr], st = sh.cstart[ch];
            const int nk = 4 * (sh.cstart[ch + 1] - st);
            const double* m = sh.Minv + ch * sub_msz + static_cast<size_t>(i - 4 * st) * sub_ld;
            const double* rv = sh.rex + 12 * st;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
            int j = q;
            for (; j + 4 < nk; j += 8) {
                const double mj = m[j], mk = m[j + 4];
                a0 = fma(mj, rv[3 * j], a0);
                b0 = fma(mk, rv[3 * j + 12], b0);
                a1 = fma(mj, rv[3 * j + 1], a1);
                b1 = fma(mk, rv[3 * j + 13], b1);
                a2 = fma(mj, rv[3 * j + 2], a2);
                b2 = fma(mk, rv[3 * j + 14], b2);
            }
            if (j < nk) {
                const double mj = m[j];
                a0 = fma(mj, rv[3 * j], a0);
                a1 = fma(mj, rv[3 * j + 1], a1);
                a2 = fma(mj, rv[3 * j + 2], a2);
            }
            a0 += b0;
            a1 += b1;
            a2 += b2;
            const unsigned grp = 0xFu << (threadIdx.x & 28);
            a0 += __shfl_xor_sync(grp, a0, 1);
            a1 += __shfl_xor_sync(grp, a1, 1);
            a2 += __shfl_xor_sync(grp, a2, 1);
            a0 += __shfl_xor_sync(grp, a0, 2);
            a1 += __shfl_xor_sync(grp, a1, 2);
            a2 += __shfl_xor_sync(grp, a2, 2);
            if (q == 0) {
                sh.zz[3 * i] = a0;
                sh.zz[3 * i + 1] = a1;
                sh.zz[3 * i + 2] = a2;
            }
        }
        // staged so that every thread stores its own elements of Z (coalesced):
        // direct scattered stores by the q == 0 lanes (and no barrier here)
        // measured +17% per PCG solve
        __syncthreads();
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            if (el_row[k] < 0) continue;
            const double z = sh.zz[el_row[k] * 12 + my_rc];
            __stcg(a.Z + zph * a.z_stride + el_g(k), z);
            sh.ext[el_row[k] * 12 + my_rc] = z;
        }
    };
    // coarse part of the preconditioner on every operand row (own + halo):
    // ext += Psi y with y = K0^-1 (Psi^T v) for the touched aggregates, from
    // the replicated aggregate sums in ptq. 8 lanes per K0^-1 row.
    auto coarse_add = [&]() {
        if (!a.use_coarse) return;
        const int g8 = threadIdx.x >> 3, l8 = threadIdx.x & 7;
        const int ngroups = blockDim.x >> 3;
        for (int row0 = 0; row0 < 4 * nt; row0 += ngroups) {  // uniform trip count: full-warp shuffles
            const int row = row0 + g8;
            double c0 = 0.0, c1 = 0.0, c2 = 0.0;
            if (row < 4 * nt) {
                const double* ci = sh.cinv + static_cast<size_t>(row) * nc;
#pragma unroll 4
                for (int j = l8; j < nc; j += 8) {
                    const double w = ci[j];
                    c0 = fma(w, sh.ptq[3 * j], c0);
                    c1 = fma(w, sh.ptq[3 * j + 1], c1);
                    c2 = fma(w, sh.ptq[3 * j + 2], c2);
                }
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                c0 += __shfl_xor_sync(0xffffffffu, c0, o);
                c1 += __shfl_xor_sync(0xffffffffu, c1, o);
                c2 += __shfl_xor_sync(0xffffffffu, c2, o);
            }
            if (l8 == 0 && row < 4 * nt) {
                sh.yt[row * 3] = c0;
                sh.yt[row * 3 + 1] = c1;
                sh.yt[row * 3 + 2] = c2;
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < n_ext * 12; t += blockDim.x) {
            const int e = t / 12, rc = t - 12 * e, r = rc / 3, c = rc - 3 * r;
            const double* y = sh.yt + sh.tl[e] * 12;
            const double add = r < 3 ? y[r * 3 + c]
                                     : sh.offx[e * 3] * y[c] + sh.offx[e * 3 + 1] * y[3 + c] +
                                           sh.offx[e * 3 + 2] * y[6 + c] + y[9 + c];
            sh.ext[t] += add;
        }
        __syncthreads();
    };

    probe(13);
    grid.sync();  // fail flags visible
    probe(14);
    if (__ldcg(&a.status->fail_node) != 0x7fffffff) return;

    // Pipelined PCG (Ghysels & Vanroose's recurrences with the two-level
    // preconditioner M = M_sub + Psi K0^-1 Psi^T): one grid barrier per
    // iteration. Before barrier i every CTA has r, u = M r, w = K u for its
    // rows; it publishes the partials of gamma = (r,u), delta = (w,u), max|r|
    // and Psi^T w, and m' = M_sub w. After the barrier one L2 round trip brings
    // the totals and the halo of m'; m = m' + Psi K0^-1 Psi^T w is completed
    // locally on own and halo rows, n = K m, and
    //   beta = gamma/gamma_prev, alpha = gamma/(delta - beta gamma/alpha_prev),
    //   z = n + beta z, q = m + beta q, s = w + beta s, p = u + beta p,
    //   x += alpha p, r -= alpha s, u -= alpha q, w -= alpha z.
    int it = 0, restarts = 0;
    double bmax = 0.0, tol = 0.0, bar = 0.0;
    // 1/gamma and 1/alpha of the previous iteration: one division (alpha) on
    // the critical path
    double gam[3] = {0, 0, 0}, inv_gam[3] = {0, 0, 0}, inv_alp[3] = {1, 1, 1};
    bool first = true;
    bool need_init = true;
    int status_code = 0;  // 1 converged, 2 indefinite, 3 max iter
    // per-CTA work (not waiting) cycles: before the barrier, after it
    const bool cprof = a.cta_prof != nullptr && threadIdx.x == 0;
    long long cw[3] = {0, 0, 0}, ct = 0;
    auto cstart_t = [&]() {
        if (kPcgProbes && cprof) ct = clock64();
    };
    auto cstop_t = [&](int k) {
        if (kPcgProbes && cprof) cw[k] += clock64() - ct;
    };

    while (true) {
        if (need_init) {
            // r = b - K x; u = M r; w = K u (three exchanges)
#pragma unroll
            for (int k = 0; k < EPT; ++k)
                if (el_row[k] >= 0) {
                    if constexpr (kLean) {
                        sh.ext[el_row[k] * 12 + my_rc] = __ldcg(a.X + el_g(k));
                    } else {
                        __stcg(a.X + el_g(k), xr[k]);
                        sh.ext[el_row[k] * 12 + my_rc] = xr[k];
                    }
                }
            grid.sync();
            exchange(a.X, false);
            double rmx = 0.0, bmx = 0.0, ps[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const double bk = el_row[k] >= 0 ? __ldg(a.B + el_g(k)) : 0.0;
                rr[k] = bk - spmv(k);
                if (el_row[k] < 0) continue;
                rmx = fmax(rmx, fabs(rr[k]));
                bmx = fmax(bmx, fabs(bk));
                psi_acc(k, rr[k], ps);
            }
            zero_vals();
            vals[0] = rmx;
            vals[1] = bmx;
            put_psi(2, ps);
            block_partials(vals, 14, sh.red, a.part_b, 0x3u);
            precond_sub(rr, false);
            grid.sync();
            exchange(a.Z + zph * a.z_stride, false);
            zph ^= 1;
            grid_totals(a.part_b, G, sh.bcast, 2, 0x3u);
            if (a.use_coarse) aggregate_sums(a, a.part_b, G, 2, sh.ptq, 4);
            __syncthreads();
            const double rmax0 = sh.bcast[0];
            bmax = sh.bcast[1];
            tol = a.rtol * (1.0 + bmax);
            bar = 1e-8 * (1.0 + bmax);
            if (restarts > 0) {
                if (rmax0 <= bar && (rmax0 <= a.true_factor * tol || restarts >= 3)) {
                    status_code = 1;
                    break;
                }
                if (restarts >= 6) {
                    status_code = 3;
                    break;
                }
            }
            if (rmax0 <= tol) {
                ++restarts;
                continue;  // verify on the true residual (need_init stays set)
            }
            coarse_add();  // ext = u on own and halo rows
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                ur[k] = el_row[k] >= 0 ? sh.ext[el_row[k] * 12 + my_rc] : 0.0;
                wr[k] = spmv(k);
                sr[k] = qr[k] = zv[k] = 0.0;
                if constexpr (kLean) {
                    if (el_row[k] >= 0) __stcg(a.P + el_g(k), 0.0);
                } else {
                    pr[k] = 0.0;
                }
            }
            first = true;
            need_init = false;
            __syncthreads();  // ext reads done before precond_sub rewrites own rows
        }
        mark(7);
        cstart_t();
        // ---- before the barrier: partials of (r,u), (w,u), max|r|, Psi^T w; m' = M_sub w
        {
            double g = 0.0, dl = 0.0, rmx = 0.0, ps[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                if (el_row[k] < 0) continue;
                g = fma(rr[k], ur[k], g);
                dl = fma(wr[k], ur[k], dl);
                rmx = fmax(rmx, fabs(rr[k]));
                psi_acc(k, wr[k], ps);
            }
            partials_stage(g, dl, rmx, ps, sh.red);
        }
        mark(0);
        precond_sub(wr, true);
        cstop_t(0);
        mark(1);
        grid.sync();
        mark(2);
        cstart_t();
        exchange(a.Z + zph * a.z_stride, true);
        zph ^= 1;
        pph ^= 1;
        mark(3);
        const double rmax = sh.bcast[6];
        if (rmax <= tol) {  // recursive residual converged: verify on the true residual
            ++restarts;
            need_init = true;
            continue;
        }
        if (it >= a.max_iter) {
            status_code = 3;
            break;
        }
        mark(10);
        // branch-free scalars for the 3 columns (no dynamic register indexing:
        // al / bt stay in registers)
        double al[3], bt[3];
        bool indefinite = false;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double g = sh.bcast[c], d = sh.bcast[3 + c];
            bt[c] = (first || gam[c] == 0.0) ? 0.0 : g * inv_gam[c];
            const double den = bt[c] == 0.0 ? d : d - bt[c] * g * inv_alp[c];
            const bool bad = g != 0.0 && (!(den > 0.0) || !isfinite(den));
            indefinite |= bad;
            al[c] = (g == 0.0 || bad) ? 0.0 : div_nr(g, den);
            gam[c] = g;
        }
        if (indefinite) {
            status_code = 2;
            break;
        }
        first = false;
        mark(8);
        coarse_add();  // ext = m on own and halo rows
        mark(9);
        {
            const double a_c = my_c == 0 ? al[0] : (my_c == 1 ? al[1] : al[2]);
            const double b_c = my_c == 0 ? bt[0] : (my_c == 1 ? bt[1] : bt[2]);
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                if (el_row[k] < 0) continue;
                const double m = sh.ext[el_row[k] * 12 + my_rc];
                double p_old = 0.0, x_old = 0.0;
                size_t g = 0;
                if constexpr (kLean) {  // in flight during this element's SpMV
                    g = el_g(k);
                    p_old = __ldcg(a.P + g);
                    x_old = __ldcg(a.X + g);
                }
                const double n = spmv(k);
                zv[k] = fma(b_c, zv[k], n);
                qr[k] = fma(b_c, qr[k], m);
                sr[k] = fma(b_c, sr[k], wr[k]);
                if constexpr (kLean) {
                    const double pn = fma(b_c, p_old, ur[k]);
                    __stcg(a.P + g, pn);
                    __stcg(a.X + g, fma(a_c, pn, x_old));
                } else {
                    pr[k] = fma(b_c, pr[k], ur[k]);
                    xr[k] = fma(a_c, pr[k], xr[k]);
                }
                rr[k] = fma(-a_c, sr[k], rr[k]);
                ur[k] = fma(-a_c, qr[k], ur[k]);
                wr[k] = fma(-a_c, zv[k], wr[k]);
            }
        }
        ++it;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            inv_gam[c] = gam[c] != 0.0 ? rcp_nr(gam[c]) : 0.0;
            if (al[c] != 0.0) inv_alp[c] = rcp_nr(al[c]);
        }
        // (no CTA barrier: precond_sub's first barrier orders these ext reads
        // before its own-row writes)
        cstop_t(1);
        mark(4);
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k)
        if constexpr (!kLean)
            if (el_row[k] >= 0) a.X[el_g(k)] = xr[k];
    if (prof)
        for (int k = 0; k < 8; ++k) a.prof[k] += acc_t[k];
    if (prof)
        for (int k = 8; k < 16; ++k) a.prof[8 + k] += acc_t[k];
    if (prof) {
        a.prof[8] += t_setup;
        a.prof[9] += 1;
    }
    if (cprof)
        for (int k = 0; k < 3; ++k) a.cta_prof[cta * 4 + k] += cw[k];
    if (cta == 0 && threadIdx.x == 0) {
        a.status->iterations = it;
        a.status->code = status_code;
        a.status->restarts = restarts;
        a.status->bmax = bmax;
    }
}

// ---------------------------------------------------------------- plan (host)
struct RcbCtx {
    const double* pos;
    const int* weight;
    std::vector<int>* ids;
    std::vector<int>* leaf_begin;
    int align = 1;  // splits of more than `align` leaves fall on a multiple of it: aggregates are subtrees
};

void rcb(RcbCtx& ctx, int lo, int hi, int g0, int g1) {
    std::vector<int>& ids = *ctx.ids;
    if (g1 - g0 == 1) {
        (*ctx.leaf_begin)[g0] = lo;
        return;
    }
    int gm = (g0 + g1) / 2;
    if (ctx.align > 1 && g1 - g0 > ctx.align) {
        // the multiple of `align` nearest the midpoint, strictly inside (g0, g1)
        const int A = ctx.align;
        gm = ((g0 + g1 + A) / (2 * A)) * A;
        gm = std::max(gm, (g0 / A + 1) * A);
        gm = std::min(gm, ((g1 - 1) / A) * A);
    }
    double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
    for (int t = lo; t < hi; ++t)
        for (int c = 0; c < 3; ++c) {
            mn[c] = std::min(mn[c], ctx.pos[3 * ids[t] + c]);
            mx[c] = std::max(mx[c], ctx.pos[3 * ids[t] + c]);
        }
    int axis = 0;
    for (int c = 1; c < 3; ++c)
        if (mx[c] - mn[c] > mx[axis] - mn[axis]) axis = c;
    std::sort(ids.begin() + lo, ids.begin() + hi, [&](int x, int y) {
        const double px = ctx.pos[3 * x + axis], py = ctx.pos[3 * y + axis];
        return px != py ? px < py : x < y;
    });
    double total = 0;
    for (int t = lo; t < hi; ++t) total += ctx.weight[ids[t]];
    const double target = total * static_cast<double>(gm - g0) / (g1 - g0);
    double acc = 0;
    int cut = lo;
    while (cut < hi && acc + ctx.weight[ids[cut]] <= target) acc += ctx.weight[ids[cut++]];
    // keep at least one node per leaf on each side when possible
    cut = std::max(cut, lo + (gm - g0));
    cut = std::min(cut, hi - (g1 - gm));
    // the two halves touch disjoint ranges of ids / leaf_begin: the top levels
    // run on separate host threads (same result as the serial recursion)
    if (hi - lo > 2048 && g1 - g0 >= 16) {
        std::thread left([&] { rcb(ctx, lo, cut, g0, gm); });
        rcb(ctx, cut, hi, gm, g1);
        left.join();
    } else {
        rcb(ctx, lo, cut, g0, gm);
        rcb(ctx, cut, hi, gm, g1);
    }
}

}  // namespace

// Lloyd relaxation of the bisection's subdomains: every node moves to the
// nearest centroid among its own and its graph neighbours' subdomains that
// still has room (at most `cap` nodes each; nodes with the clearest choice
// are placed first), `rounds` times. Rounder subdomains have shorter
// interfaces: on config 2 the block-Jacobi + coarse PCG needs 13-17% fewer
// iterations and the largest halo shrinks from 98 to ~70 operand rows
// (tools/partition_study.py). Subdomain numbers, and so the aggregates of
// consecutive subdomains, are kept. Deterministic: fixed-order sums, index
// tie-breaks. Within a subdomain the rows follow a Morton order of the node
// positions, so consecutive rows (the dense preconditioner chunks) are compact.
void lloyd_refine(const double* pos, const int* adj_off, const int* adj, const int* adj_cnt, int N, int G, int cap,
                  int rounds, std::vector<int>& ids, std::vector<int>& leaf_begin) {
    std::vector<int> label(N), fresh(N), count(G), order(N);
    for (int g = 0; g < G; ++g)
        for (int t = leaf_begin[g]; t < (g + 1 < G ? leaf_begin[g + 1] : N); ++t) label[ids[t]] = g;
    constexpr int kCand = 8;  // candidate subdomains kept per node (own + neighbours'; more than 4-5 is rare)
    std::vector<double> cen(3 * static_cast<size_t>(G)), cand_d(static_cast<size_t>(N) * kCand);
    std::vector<int> cand(static_cast<size_t>(N) * kCand), ncand(N);
    std::vector<int> bucket(1027), bkt(N);
    for (int r = 0; r < rounds; ++r) {
        std::fill(cen.begin(), cen.end(), 0.0);
        std::fill(count.begin(), count.end(), 0);
        for (int j = 0; j < N; ++j) {
            double* cg = &cen[3 * static_cast<size_t>(label[j])];
            cg[0] += pos[3 * j];
            cg[1] += pos[3 * j + 1];
            cg[2] += pos[3 * j + 2];
            ++count[label[j]];
        }
        for (int g = 0; g < G; ++g) {
            const double inv = 1.0 / std::max(1, count[g]);
            for (int c = 0; c < 3; ++c) cen[3 * g + c] *= inv;
        }
        for (int j = 0; j < N; ++j) {
            // candidate subdomains: own and the neighbours', nearest centroid first
            int* cs = &cand[static_cast<size_t>(j) * kCand];
            double* ds = &cand_d[static_cast<size_t>(j) * kCand];
            int nc = 0;
            cs[nc++] = label[j];
            for (int t = adj_off[j], te = adj_off[j] + adj_cnt[j]; t < te; ++t) {
                const int g = label[adj[t]];
                bool seen = false;
                for (int u = 0; u < nc; ++u) seen |= cs[u] == g;
                if (!seen && nc < kCand) cs[nc++] = g;
            }
            const double px = pos[3 * j], py = pos[3 * j + 1], pz = pos[3 * j + 2];
            for (int u = 0; u < nc; ++u) {
                const double* cg = &cen[3 * static_cast<size_t>(cs[u])];
                const double x = px - cg[0], y = py - cg[1], z = pz - cg[2];
                ds[u] = x * x + y * y + z * z;
            }
            for (int u = 1; u < nc; ++u)  // insertion sort by (distance, subdomain)
                for (int v = u; v > 0 && (ds[v] < ds[v - 1] || (ds[v] == ds[v - 1] && cs[v] < cs[v - 1])); --v) {
                    std::swap(ds[v], ds[v - 1]);
                    std::swap(cs[v], cs[v - 1]);
                }
            ncand[j] = nc;
        }
        // placement order: nodes with a single candidate first, then by the
        // ratio of the nearest to the second nearest centroid distance in
        // 1024 buckets (the clearest choices first; index order inside a
        // bucket): a counting sort instead of a comparison sort
        std::fill(bucket.begin(), bucket.end(), 0);
        for (int j = 0; j < N; ++j) {
            int b = 0;
            if (ncand[j] > 1) {
                const double d0 = cand_d[static_cast<size_t>(j) * kCand], d1 = cand_d[static_cast<size_t>(j) * kCand + 1];
                const double ratio = d0 / d1;  // in [0, 1]; anything else (0/0, non-finite positions) goes last
                b = (ratio >= 0.0 && ratio < 1.0) ? 1 + static_cast<int>(ratio * 1024.0) : 1024;
            }
            bkt[j] = b;
            ++bucket[b + 1];
        }
        for (int b = 0; b < 1025; ++b) bucket[b + 1] += bucket[b];
        for (int j = 0; j < N; ++j) order[bucket[bkt[j]]++] = j;
        std::fill(count.begin(), count.end(), 0);
        int moved = 0;
        for (int j : order) {
            int pick = -1;
            const int* cs = &cand[static_cast<size_t>(j) * kCand];
            for (int t = 0; t < ncand[j] && pick < 0; ++t)
                if (count[cs[t]] < cap) pick = cs[t];
            if (pick < 0) {  // every candidate is full: the nearest subdomain with room
                double best = 1e300;
                for (int g = 0; g < G; ++g) {
                    if (count[g] >= cap) continue;
                    double d = 0;
                    for (int c = 0; c < 3; ++c) {
                        const double x = pos[3 * j + c] - cen[3 * g + c];
                        d += x * x;
                    }
                    if (d < best) {
                        best = d;
                        pick = g;
                    }
                }
            }
            fresh[j] = pick;
            moved += pick != label[j];
            ++count[pick];
        }
        bool empty = false;
        for (int g = 0; g < G; ++g) empty |= count[g] == 0;
        if (empty) break;  // keep the previous round's subdomains
        label.swap(fresh);
        if (moved <= N / 256) break;  // converged: the last rounds move a handful of nodes
    }
    // rows: subdomain by subdomain, Morton order inside
    std::fill(count.begin(), count.end(), 0);
    for (int j = 0; j < N; ++j) ++count[label[j]];
    leaf_begin[0] = 0;
    for (int g = 0; g + 1 < G; ++g) leaf_begin[g + 1] = leaf_begin[g] + count[g];
    std::vector<int> fill(leaf_begin.begin(), leaf_begin.begin() + G);
    for (int j = 0; j < N; ++j) ids[fill[label[j]]++] = j;
    std::vector<unsigned> code(N);
    for (int g = 0; g < G; ++g) {
        const int lo = leaf_begin[g], hi = lo + count[g];
        double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
        for (int t = lo; t < hi; ++t)
            for (int c = 0; c < 3; ++c) {
                mn[c] = std::min(mn[c], pos[3 * ids[t] + c]);
                mx[c] = std::max(mx[c], pos[3 * ids[t] + c]);
            }
        const double ext = std::max({mx[0] - mn[0], mx[1] - mn[1], mx[2] - mn[2], 1e-300});
        for (int t = lo; t < hi; ++t) {
            unsigned m = 0;
            for (int c = 0; c < 3; ++c) {
                unsigned q = static_cast<unsigned>(std::min(1023.0, (pos[3 * ids[t] + c] - mn[c]) / ext * 1023.0));
                for (int b = 0; b < 10; ++b) m |= ((q >> b) & 1u) << (3 * b + c);
            }
            code[ids[t]] = m;
        }
        std::sort(ids.begin() + lo, ids.begin() + hi,
                  [&](int x, int y) { return code[x] != code[y] ? code[x] < code[y] : x < y; });
    }
}

void PcgPlan::build(const double* node_pos, const int* row_nnz_by_node, int N, int num_sms, size_t smem_limit,
                    const int* adj_off, const int* adj) {
    nodes = N;
    grid = std::max(1, std::min({num_sms, N, 32 * kMaxGridLoads}));
    const int cap_rows = (kPcgThreads * kMaxEpt) / 12;
    while ((N + grid - 1) / grid > cap_rows * 7 / 8 && grid < std::min(num_sms, 32 * kMaxGridLoads)) ++grid;
    if ((N + grid - 1) / grid > cap_rows)
        throw ConfigError("PCG: deformation graph too large for one cooperative grid (nodes per SM > 256)");
    std::vector<int> ids(N), w(N);
    std::iota(ids.begin(), ids.end(), 0);
    // bisection cost per node: wbase + its block count. With the relaxation on
    // top a near count-balanced bisection is the better start (config 2:
    // 1,170 it/s at 6, 1,208 at 30, 1,232 at 100, profiles/r04_rcb_weight_sweep.txt;
    // 6 had measured best for the bisection alone)
    int wbase = 100;
    if (const char* e = std::getenv("NRR_RCB_W")) wbase = std::atoi(e);
    for (int j = 0; j < N; ++j) w[j] = wbase + row_nnz_by_node[j];
    row_begin.assign(grid + 1, N);
    // CTAs per coarse aggregate, decided before the bisection so that its
    // splits fall on aggregate boundaries (an aggregate is then a subtree: a
    // compact box, instead of 4 or 8 consecutive leaves that straddle
    // subtrees). 4 CTAs per aggregate (37 aggregates on 148 CTAs): with
    // aligned splits and rounded subdomains the offline count drops from 88
    // (8 per aggregate) to 73 (tools/partition_study.py).
    agg_ctas = std::max(4, (4 * grid + 159) / 160);
    if (const char* e = std::getenv("NRR_AGG_CTAS")) agg_ctas = std::max((4 * grid + 159) / 160, std::atoi(e));
    RcbCtx ctx{node_pos, w.data(), &ids, &row_begin};
    ctx.align = std::getenv("NRR_RCB_ALIGN") ? std::atoi(std::getenv("NRR_RCB_ALIGN")) : agg_ctas;
    rcb(ctx, 0, N, 0, grid);
    row_begin[grid] = N;
    {
        // The subdomains are rounded with a size cap that keeps the plan's
        // shape: the elements per thread of the bisection's largest
        // subdomain, and (one element per thread) the 24 rows whose 16 x 24
        // subdomain-matvec tasks still fit one round of the CTA's 384
        // threads: 25 rows cost +9% per PCG iteration on config 2, 10% above
        // the mean (24 rows there) measured best (profiles/r04_lloyd_sweep.txt).
        int rcb_max = 0;
        for (int g = 0; g < grid; ++g) rcb_max = std::max(rcb_max, row_begin[g + 1] - row_begin[g]);
        int rounds = 16, cap_add = 10;
        if (const char* e = std::getenv("NRR_LLOYD")) rounds = std::atoi(e);
        if (const char* e = std::getenv("NRR_LLOYD_CAP")) cap_add = std::atoi(e);  // percent above the mean
        int ept_rcb = 1;
        while (rcb_max * 12 > ept_rcb * kPcgThreads) ept_rcb *= 2;
        int bound = ept_rcb * kPcgThreads / 12;
        if (rcb_max <= kPcgThreads / 16) bound = kPcgThreads / 16;
        if (adj_off != nullptr && rounds > 0 && grid > 1) {
            const int mean = (N + grid - 1) / grid;
            const int cap = std::min(bound, std::max(rcb_max, mean + (mean * cap_add + 99) / 100));
            lloyd_refine(node_pos, adj_off, adj, row_nnz_by_node, N, grid, cap, rounds, ids, row_begin);
            row_begin[grid] = N;
        }
    }
    row_node = ids;
    node_row.assign(N, 0);
    for (int r = 0; r < N; ++r) node_row[row_node[r]] = r;
    max_rows = 0;
    for (int g = 0; g < grid; ++g) max_rows = std::max(max_rows, row_begin[g + 1] - row_begin[g]);
    if (max_rows * 12 > kPcgThreads * kMaxEpt)
        throw ConfigError("PCG: deformation graph too large for one cooperative grid (nodes per SM > 256)");
    ept = 1;
    while (max_rows * 12 > ept * kPcgThreads) ept *= 2;
    // aggregates: consecutive CTAs, coarse dimension 4 * n_agg <= kCoarseMax (160)
    // CTAs per coarse aggregate: 8 measured best on cfg2 (~20 nodes per CTA);
    // with large subdomains (cfg4, ~120 nodes per CTA) 4 (37 aggregates):
    // 298 -> 261 iterations, -8% per pass
    if (const char* e = std::getenv("NRR_COARSE")) use_coarse = std::atoi(e) != 0;
    n_agg = (grid + agg_ctas - 1) / agg_ctas;
    node_agg.assign(N, 0);
    agg_center.assign(3 * static_cast<size_t>(n_agg), 0.0);
    std::vector<int> cnt(n_agg, 0);
    for (int g = 0; g < grid; ++g)
        for (int r = row_begin[g]; r < row_begin[g + 1]; ++r) {
            const int node = row_node[r], ag = g / agg_ctas;
            node_agg[node] = ag;
            for (int c = 0; c < 3; ++c) agg_center[3 * ag + c] += node_pos[3 * node + c];
            ++cnt[ag];
        }
    for (int ag = 0; ag < n_agg; ++ag)
        for (int c = 0; c < 3; ++c) agg_center[3 * ag + c] /= std::max(1, cnt[ag]);
    (void)smem_limit;
}

bool nc_limit_exceeded(int n_agg) { return 4 * n_agg > 160; }

void PcgPlan::size_smem(const int* row_ptr_solver, const int* col, size_t smem_limit) {
    max_kb = 0;
    for (int g = 0; g < grid; ++g)
        max_kb = std::max(max_kb, row_ptr_solver[row_begin[g + 1]] - row_ptr_solver[row_begin[g]]);
    // per-CTA operand rows: own rows (in row order) then the halo nodes
    const int nnzb = row_ptr_solver[nodes];
    colx.assign(nnzb, 0);
    ext_off.assign(grid + 1, 0);
    ext_node.clear();
    max_ext = 0;
    std::vector<int> local(nodes, -1);
    for (int g = 0; g < grid; ++g) {
        const int rb = row_begin[g], re = row_begin[g + 1];
        std::vector<int> nodes_g;
        for (int r = rb; r < re; ++r) {
            local[row_node[r]] = r - rb;
            nodes_g.push_back(row_node[r]);
        }
        for (int b = row_ptr_solver[rb]; b < row_ptr_solver[re]; ++b) {
            const int nb = col[b];
            if (local[nb] < 0) {
                local[nb] = static_cast<int>(nodes_g.size());
                nodes_g.push_back(nb);
            }
            colx[b] = local[nb];
        }
        for (int nb : nodes_g) local[nb] = -1;
        ext_node.insert(ext_node.end(), nodes_g.begin(), nodes_g.end());
        ext_off[g + 1] = static_cast<int>(ext_node.size());
        max_ext = std::max(max_ext, static_cast<int>(nodes_g.size()));
    }
    // aggregates touched by each CTA's operand rows (coarse correction on halo rows)
    touch_off.assign(grid + 1, 0);
    touch_agg.clear();
    ext_tl.assign(ext_node.size(), 0);
    max_touch = 1;
    for (int g = 0; g < grid; ++g) {
        std::vector<int> t;
        for (int e = ext_off[g]; e < ext_off[g + 1]; ++e) t.push_back(node_agg[ext_node[e]]);
        std::sort(t.begin(), t.end());
        t.erase(std::unique(t.begin(), t.end()), t.end());
        for (int e = ext_off[g]; e < ext_off[g + 1]; ++e)
            ext_tl[e] = static_cast<int>(std::lower_bound(t.begin(), t.end(), node_agg[ext_node[e]]) - t.begin());
        touch_agg.insert(touch_agg.end(), t.begin(), t.end());
        touch_off[g + 1] = static_cast<int>(touch_agg.size());
        max_touch = std::max(max_touch, static_cast<int>(t.size()));
    }
    // coarse_partial_kernel's touched-list limit; coarse_invert_kernel's register tiles
    if (max_touch > 64 || nc_limit_exceeded(n_agg)) use_coarse = false;
    const size_t nc = 4 * static_cast<size_t>(n_agg);
    const size_t fixed = kRedDoubles + kQ + 12 * static_cast<size_t>(max_rows) /* zz */ +
                         12 * static_cast<size_t>(max_rows) /* rex */ + 3 * static_cast<size_t>(max_ext) /* offx */ +
                         (use_coarse ? 4 * max_touch * nc : 0) /* cinv */ + 12 * static_cast<size_t>(max_touch) +
                         3 * kCoarseMax /* ptq */ + 12 * static_cast<size_t>(max_ext) /* ext */ +
                         (max_rows + 1) / 2 /* rchunk */ + (max_ext + 1) / 2 /* tl */ + (max_rows + 2) / 2 /* rp */ +
                         (max_rows + 1) / 2 /* rnode */ + 2;
    const size_t kbytes = static_cast<size_t>(max_kb) * (16 * sizeof(double) + sizeof(int));
    // largest subdomain chunk (rows per dense block-Jacobi inverse) that fits
    auto sub_doubles = [&](int S) {
        const int ld = sub_leading_dim(S);
        const size_t ch = (max_rows + S - 1) / S;
        return ch * 4 * static_cast<size_t>(S) * ld + (ch + 2) / 2;
    };
    // K stays in shared memory when it fits beside the smallest (1-node)
    // subdomain plan; otherwise the SpMV reads it from L2
    k_in_smem = sizeof(double) * (fixed + sub_doubles(1)) + kbytes + 64 <= smem_limit;
    int S = std::max(1, std::min(max_rows, kSubRowsMax));  // largest chunk that fits; NRR_SUB_ROWS overrides
    if (const char* e = std::getenv("NRR_SUB_ROWS")) S = std::max(1, std::min(max_rows, std::atoi(e)));
    const size_t kpart = k_in_smem ? kbytes : 0;
    while (S > 1 && (sizeof(double) * (fixed + sub_doubles(S)) + kpart + 64 > smem_limit ||
                     sizeof(double) * ((max_rows + S - 1) / S) * (4 * static_cast<size_t>(S) + 8) * sub_leading_dim(S) +
                             1024 > smem_limit))
        --S;
    sub_rows = S;
    sub_ld = sub_leading_dim(S);
    sub_chunks = (max_rows + S - 1) / S;
    smem_bytes = sizeof(double) * (fixed + sub_doubles(S)) + kpart + 64;
    if (smem_bytes > smem_limit)
        throw ConfigError("PCG: shared-memory plan does not fit (" + std::to_string(smem_bytes) + " > " +
                          std::to_string(smem_limit) + " bytes; fixed " + std::to_string(fixed * sizeof(double)) +
                          ", max_rows " + std::to_string(max_rows) + ", max_ext " + std::to_string(max_ext) + ")");
}

void launch_coarse_setup(const PcgPlan& plan, const PcgArgs& a, const CoarseWork& w, cudaStream_t s) {
    const size_t psmem =
        static_cast<size_t>(std::min((plan.max_kb + 7) & ~7, kCpChunk)) * (16 * sizeof(double) + 2 * sizeof(int)) + 64;
    allow_max_smem(reinterpret_cast<const void*>(coarse_partial_kernel));
    PcgArgs b = a;
    b.max_touch = plan.max_touch;
    b.max_kb = plan.max_kb;
    coarse_partial_kernel<<<plan.grid, kCoarseThreads, psmem, s>>>(b, w.partial);
    NRR_CUDA_CHECK(cudaGetLastError());
    const int nc = 4 * plan.n_agg;
    const size_t smem = sizeof(double) * (static_cast<size_t>(nc) * nc + 6 * 16 * static_cast<size_t>(plan.n_agg) + 32) +
                        sizeof(int) * static_cast<size_t>(plan.grid) * plan.max_touch + 16;
    allow_max_smem(reinterpret_cast<const void*>(coarse_invert_kernel));
    if (plan.n_agg * plan.n_agg <= kCiThreads * kCiTiles) {
        coarse_invert_kernel<<<1, kCiThreads, smem, s>>>(b, w.partial, w.inv, plan.grid);
    } else {
        const size_t smem2 = sizeof(double) * (static_cast<size_t>(nc) * nc + 8 * nc) +
                             sizeof(int) * static_cast<size_t>(plan.grid) * plan.max_touch + 16;
        allow_max_smem(reinterpret_cast<const void*>(coarse_invert_smem_kernel));
        coarse_invert_smem_kernel<<<1, 1024, smem2, s>>>(b, w.partial, w.inv, plan.grid);
    }
    NRR_CUDA_CHECK(cudaGetLastError());
}

void launch_sub_invert(const PcgPlan& plan, const PcgArgs& a, double* out, cudaStream_t s) {
    const size_t ch = plan.sub_chunks;
    const size_t smem = sizeof(double) * (ch * 4 * plan.sub_rows * plan.sub_ld + ch * 8 * plan.sub_ld + 17 * ch) +
                        sizeof(int) * (2 * ch + 2) + 16;
    allow_max_smem(reinterpret_cast<const void*>(sub_invert_kernel));
    PcgArgs b = a;
    b.sub_rows = plan.sub_rows;
    b.sub_ld = plan.sub_ld;
    b.sub_chunks = plan.sub_chunks;
    sub_invert_kernel<<<plan.grid, kInvThreads, smem, s>>>(b, out);
    NRR_CUDA_CHECK(cudaGetLastError());
}

namespace {
// Cooperative grids in flight per device, each with the event recorded after
// its launch (polled: no stream callback on the critical path).
struct CoopBudget {
    std::mutex mu;
    std::map<int, std::vector<std::pair<cudaEvent_t, int>>> inflight;
    // Waits until `ctas` more CTAs fit the device's budget and returns with
    // the mutex held: the caller launches its grid and records `ev` behind
    // it before calling commit(), so no other thread can query `ev` between
    // the budget check and the recording (a query of the event's previous,
    // completed recording would drop a grid that is in flight).
    std::unique_lock<std::mutex> acquire(int dev, int ctas, int sms, cudaEvent_t ev) {
        std::unique_lock<std::mutex> lk(mu);
        auto& v = inflight[dev];
        // the caller's previous grid has completed (the host synchronised
        // its stream since): its entry goes before the event is reused
        for (size_t k = 0; k < v.size(); ++k)
            if (v[k].first == ev) {
                v.erase(v.begin() + static_cast<long>(k));
                break;
            }
        while (true) {
            int used = 0;
            for (size_t k = 0; k < v.size();) {
                if (cudaEventQuery(v[k].first) != cudaErrorNotReady) {
                    v.erase(v.begin() + static_cast<long>(k));
                } else {
                    used += v[k].second;
                    ++k;
                }
            }
            if (used == 0 || used + ctas <= sms) break;
            lk.unlock();
            std::this_thread::sleep_for(std::chrono::microseconds(20));
            lk.lock();
        }
        return lk;
    }
    // with the lock from acquire() still held, after cudaEventRecord(ev)
    void commit(int dev, int ctas, cudaEvent_t ev) { inflight[dev].push_back({ev, ctas}); }
    void forget(cudaEvent_t ev) {
        std::lock_guard<std::mutex> lk(mu);
        for (auto& [d, v] : inflight)
            for (size_t k = 0; k < v.size(); ++k)
                if (v[k].first == ev) {
                    v.erase(v.begin() + static_cast<long>(k));
                    break;
                }
    }
};
CoopBudget& coop_budget() {
    static CoopBudget b;
    return b;
}
}  // namespace

void pcg_forget_event(cudaEvent_t ev) { coop_budget().forget(ev); }

void launch_pcg(const PcgPlan& plan, PcgArgs args, cudaStream_t s, cudaEvent_t done) {
    args.max_rows = plan.max_rows;
    args.sub_rows = plan.sub_rows;
    args.sub_ld = plan.sub_ld;
    args.sub_chunks = plan.sub_chunks;
    args.max_kb = plan.max_kb;
    args.max_ext = plan.max_ext;
    args.k_in_smem = plan.k_in_smem ? 1 : 0;
    args.agg_ctas = plan.agg_ctas;
    args.n_agg = plan.n_agg;
    args.use_coarse = plan.use_coarse ? 1 : 0;
    args.max_touch = plan.max_touch;
    void* kargs[] = {&args};
    const void* fn = plan.ept == 1   ? reinterpret_cast<const void*>(pcg_kernel<1>)
                     : plan.ept == 2 ? reinterpret_cast<const void*>(pcg_kernel<2>)
                     : plan.ept == 4 ? reinterpret_cast<const void*>(pcg_kernel<4>)
                                     : reinterpret_cast<const void*>(pcg_kernel<8>);
    allow_max_smem(reinterpret_cast<const void*>(fn));
    int per_sm = 0;
    NRR_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPcgThreads, plan.smem_bytes));
    if (per_sm < 1) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, fn);
        int per_sm0 = 0, dev = 0, smsm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm0, fn, kPcgThreads, 0);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        throw CudaError("PCG kernel does not fit one SM: blocks/SM without smem " + std::to_string(per_sm0) +
                        ", smem/SM " + std::to_string(smsm) + ", maxThreads " + std::to_string(fa.maxThreadsPerBlock) +
                        ", regs " + std::to_string(fa.numRegs) + ", static smem " +
                        std::to_string(fa.sharedSizeBytes) + ", dynamic smem " + std::to_string(plan.smem_bytes) +
                        ", local " + std::to_string(fa.localSizeBytes));
    }
    // Several contexts may launch their PCG grids side by side (config 3).
    // A grid spins at its barriers, so two partially resident grids could
    // wait on each other's SMs; a per-device budget keeps the sum of the
    // cooperative grids in flight within one CTA per SM. A grid's budget
    // returns when its completion event (recorded right behind it, under the
    // budget's lock) is found complete by a later acquire's poll.
    int dev = 0, sms = 0;
    NRR_CUDA_CHECK(cudaGetDevice(&dev));
    NRR_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    auto& budget = coop_budget();
    auto lk = budget.acquire(dev, plan.grid, sms, done);
    NRR_CUDA_CHECK(cudaLaunchCooperativeKernel(fn, dim3(plan.grid), dim3(kPcgThreads), kargs, plan.smem_bytes, s));
    NRR_CUDA_CHECK(cudaEventRecord(done, s));
    budget.commit(dev, plan.grid, done);
}

}  // namespace nrr_b200
