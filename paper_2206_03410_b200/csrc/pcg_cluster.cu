// Cluster-resident block-Jacobi PCG for the 4N x 4N, 3-RHS normal equations
// (reference SystemAssembler::solve, energy.hpp:233-254), for graphs that fit
// the shared memory of one thread-block cluster (<= 16 SMs).
//
// Why: a grid-wide barrier over 148 CTAs costs ~2 us on B200 (measured,
// tools/sync_bench.cu); two cluster barriers plus a DSMEM read cost ~0.64 us
// (tools/cluster_bench.cu). CG needs two barriers per iteration (the SpMV halo
// and the dot products), so the solve is barrier-bound: one cluster of 16
// CTAs iterates several times faster than the whole GPU, and leaves the other
// 132 SMs free for independent registrations (config 3).
//
// Layout. The graph is split by recursive coordinate bisection into one part
// per CTA (rank). Each rank keeps in shared memory
//   * its K blocks: the diagonal blocks, every intra-rank pair ONCE (read
//     directly by the lower row and transposed by the upper one — K is
//     symmetric, energy.hpp:185-196 guarantees it bitwise), and the
//     cross-rank blocks of its rows; blocks that do not fit stay in L2;
//   * z for its own rows plus a halo copy of the neighbour rows, refreshed
//     once per iteration with one DSMEM load per halo double;
//   * its 4x4 block-Jacobi inverses.
// x, r, p, q, b live in registers (thread = (node, row r, column c)).
// All reductions: fixed-order CTA partials, then one warp per quantity over
// the ranks' partials read through DSMEM — bitwise reproducible.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <unordered_map>

#include "device_common.cuh"
#include "pcg_cluster.cuh"

namespace cg = cooperative_groups;

namespace nrr_b200 {

namespace {

constexpr int kSlots = 8;
constexpr int kExt = 14;  // ext row stride in doubles (12 used; 112 B rows avoid bank conflicts)

__device__ __forceinline__ double op2c(bool mx, double a, double b) { return mx ? fmax(a, b) : a + b; }

// block reduction of 8 per-thread slots -> out[8] (sum, or max per mask):
// transpose-reduce inside each warp (4+2+1 shuffles, then 2 more), then one
// warp per slot over the warps. Fixed order, deterministic.
__device__ __forceinline__ void block_slots(const double* vals, int nq, double* red, double* out, unsigned max_mask) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double v4[4], v2[2], v1;
    int base = 0;
    {
        const bool up = lane & 16;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double keep = up ? vals[i + 4] : vals[i], send = up ? vals[i] : vals[i + 4];
            v4[i] = op2c((max_mask >> ((up ? 4 : 0) + i)) & 1u, keep, __shfl_xor_sync(0xffffffffu, send, 16));
        }
        base += up ? 4 : 0;
    }
    {
        const bool up = lane & 8;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double keep = up ? v4[i + 2] : v4[i], send = up ? v4[i] : v4[i + 2];
            v2[i] = op2c((max_mask >> (base + (up ? 2 : 0) + i)) & 1u, keep, __shfl_xor_sync(0xffffffffu, send, 8));
        }
        base += up ? 2 : 0;
    }
    {
        const bool up = lane & 4;
        const double keep = up ? v2[1] : v2[0], send = up ? v2[0] : v2[1];
        base += up ? 1 : 0;
        v1 = op2c((max_mask >> base) & 1u, keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
    const bool mxb = (max_mask >> base) & 1u;
    v1 = op2c(mxb, v1, __shfl_xor_sync(0xffffffffu, v1, 2));
    v1 = op2c(mxb, v1, __shfl_xor_sync(0xffffffffu, v1, 1));
    if ((lane & 3) == 0) red[base * 32 + w] = v1;
    __syncthreads();
    if (w < nq) {
        const bool mx = (max_mask >> w) & 1u;
        double v = lane < nw ? red[w * 32 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = op2c(mx, v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) out[w] = v;
    }
    __syncthreads();
}

// Thread = node: all 4 scalar rows x 3 right-hand sides (12 values) of one
// graph node. Per K block the thread issues 8 LDS.128 for the block and 6 for
// the neighbour's 12 z values, then 48 independent FMAs into 12 accumulators
// (transposed blocks only swap register operands): high ILP, no shuffles.
__global__ void __launch_bounds__(kClusterThreads, 1) pcg_cluster_kernel(ClusterArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    const int CS = static_cast<int>(cl.num_blocks());
    const ClusterPlanDev& P = a.plan;
    const int r0 = P.rank_rows[rank], r1 = P.rank_rows[rank + 1], nrows = r1 - r0;
    const int s0 = P.store_off[rank], ns = P.store_off[rank + 1] - s0;
    const int h0 = P.halo_off[rank], nh = P.halo_off[rank + 1] - h0;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* Kst = reinterpret_cast<double*>(smem_raw);                 // max_store*16
    double* ext = Kst + 16 * static_cast<size_t>(a.max_store);         // max_ext*kExt (rows padded)
    double* M = ext + kExt * static_cast<size_t>(a.max_ext);           // 16 x max_rows (SoA)
    double* part = M + 16 * static_cast<size_t>(a.max_rows);         // 2 x kSlots (read remotely)
    double* red = part + 2 * kSlots;                                   // 32 x kSlots
    double* bcast = red + 32 * kSlots;                                 // kSlots
    int2* ent_s = reinterpret_cast<int2*>(bcast + kSlots);             // max_ent: own rows' entries
    int* eptr_s = reinterpret_cast<int*>(ent_s + a.max_ent);           // max_rows+1
    int* flags = eptr_s + a.max_rows + 1;                              // [0] fail node of this rank

    // 16-byte chunk t of slot s is stored at chunk (t ^ (s & 7)): threads of a
    // quarter-warp reading chunk t of different blocks then spread over the
    // banks instead of all hitting the same four (blocks are 128 B aligned)
    for (int i = threadIdx.x; i < ns * 8; i += blockDim.x) {
        const int slot = i >> 3, t = i & 7;
        reinterpret_cast<double2*>(Kst)[slot * 8 + (t ^ (slot & 7))] =
            reinterpret_cast<const double2*>(a.K)[static_cast<size_t>(P.store_src[s0 + slot]) * 8 + t];
    }
    {
        const int e0 = P.ent_ptr[r0], ne = P.ent_ptr[r1] - e0;
        for (int i = threadIdx.x; i < ne; i += blockDim.x) ent_s[i] = P.ent[e0 + i];
        for (int i = threadIdx.x; i <= nrows; i += blockDim.x) eptr_s[i] = P.ent_ptr[r0 + i] - e0;
    }
    if (threadIdx.x == 0) flags[0] = 0x7fffffff;
    __syncthreads();
    auto load_block = [&](int x, double k[16]) {
        const int off = (x >> 2) * 16;
        if (!(x & 1)) {
            const int sw = (x >> 2) & 7;
            const double2* kb = reinterpret_cast<const double2*>(Kst + off);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const double2 v = kb[t ^ sw];
                k[2 * t] = v.x;
                k[2 * t + 1] = v.y;
            }
        } else {
            const double2* kb = reinterpret_cast<const double2*>(a.K + off);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const double2 v = __ldg(kb + t);
                k[2 * t] = v.x;
                k[2 * t + 1] = v.y;
            }
        }
    };
    // ---- block Jacobi: M_j = K_jj^{-1} (4x4 Cholesky, one thread per row)
    for (int lr = threadIdx.x; lr < nrows; lr += blockDim.x) {
        const int j = r0 + lr;
        double k[16], l[16] = {0};
        load_block(ent_s[P.diag_ent[j] - P.ent_ptr[r0]].x, k);
        double dmax = 0;
        for (int t = 0; t < 4; ++t) dmax = fmax(dmax, fabs(k[t * 5]));
        bool ok = dmax > 0 && isfinite(dmax);
        for (int c = 0; c < 4 && ok; ++c) {
            double sum = k[c * 4 + c];
            for (int t = 0; t < c; ++t) sum -= l[c * 4 + t] * l[c * 4 + t];
            if (!(sum > 0.0)) {  // not PD (reference describe_failure)
                ok = false;
                break;
            }
            const double d = sqrt(sum);
            l[c * 4 + c] = d;
            for (int r = c + 1; r < 4; ++r) {
                double v = k[r * 4 + c];
                for (int t = 0; t < c; ++t) v -= l[r * 4 + t] * l[c * 4 + t];
                l[r * 4 + c] = v / d;
            }
        }
        double* Mj = M + lr;  // element t at Mj[t * max_rows]
        const int ms = a.max_rows;
        if (!ok) {
            atomicMin(&flags[0], P.row_node[j]);
            for (int t = 0; t < 16; ++t) Mj[t * ms] = 0.0;
            continue;
        }
        for (int e = 0; e < 4; ++e) {
            double y[4];
            for (int r = 0; r < 4; ++r) {
                double v = (r == e) ? 1.0 : 0.0;
                for (int t = 0; t < r; ++t) v -= l[r * 4 + t] * y[t];
                y[r] = v / l[r * 4 + r];
            }
            for (int r = 3; r >= 0; --r) {
                double v = y[r];
                for (int t = r + 1; t < 4; ++t) v -= l[t * 4 + r] * y[t];
                y[r] = v / l[r * 4 + r];
            }
            for (int r = 0; r < 4; ++r) Mj[(r * 4 + e) * ms] = y[r];
        }
    }
    cl.sync();
    {  // any rank failed -> every rank exits (consistent decision)
        int fail = 0x7fffffff;
        if ((threadIdx.x & 31) < CS) fail = *cl.map_shared_rank(flags, static_cast<int>(threadIdx.x & 31));
        for (int o = 16; o > 0; o >>= 1) fail = min(fail, __shfl_xor_sync(0xffffffffu, fail, o));
        if (fail != 0x7fffffff) {
            if (rank == 0 && threadIdx.x == 0) atomicMin(&a.status->fail_node, fail);
            return;
        }
    }

    // thread = (node lr, column c): the 4 scalar rows of one right-hand side
    const int lr = threadIdx.x / 3, col = threadIdx.x % 3;
    const bool live = lr < nrows;
    const size_t gb = live ? static_cast<size_t>(P.row_node[r0 + lr]) * 12 + col : 0;  // + 3r
    double xr[4], rr[4], zr[4], pr[4], qr[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        xr[t] = live ? a.X[gb + 3 * t] : 0.0;
        rr[t] = zr[t] = pr[t] = qr[t] = 0.0;
    }
    const bool prof = a.prof != nullptr && rank == 0 && threadIdx.x == 0;
    long long tp = clock64(), acc_t[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    auto mark = [&](int slot) {
        if (prof) {
            const long long t = clock64();
            acc_t[slot] += t - tp;
            tp = t;
        }
    };
    // publish own values into ext, cluster barrier, copy the halo
    auto exchange = [&](const double* own) {
        if (live)
#pragma unroll
            for (int t = 0; t < 4; ++t) ext[lr * kExt + 3 * t + col] = own[t];
        cl.sync();
        mark(8);
        for (int t = threadIdx.x; t < nh * 6; t += blockDim.x) {
            const int2 src = P.halo_src[h0 + t / 6];
            const double2* remote = reinterpret_cast<const double2*>(cl.map_shared_rank(ext, src.x));
            reinterpret_cast<double2*>(ext)[(nrows + t / 6) * (kExt / 2) + (t % 6)] = remote[src.y * (kExt / 2) + (t % 6)];
        }
        __syncthreads();
    };
    // w[r] = (K v)[r][col] for the own node
    auto spmv = [&](double w[4]) {
        w[0] = w[1] = w[2] = w[3] = 0.0;
        if (!live) return;
        const int e1 = eptr_s[lr + 1];
        for (int e = eptr_s[lr]; e < e1; ++e) {
            const int2 en = ent_s[e];
            double k[16];
            load_block(en.x, k);
            const bool tr = en.x & 2;
            const double* vb = ext + en.y * kExt + col;
            const double v0 = vb[0], v1 = vb[3], v2 = vb[6], v3 = vb[9];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double k0 = tr ? k[r] : k[r * 4], k1 = tr ? k[4 + r] : k[r * 4 + 1];
                const double k2 = tr ? k[8 + r] : k[r * 4 + 2], k3 = tr ? k[12 + r] : k[r * 4 + 3];
                w[r] = fma(k0, v0, fma(k1, v1, fma(k2, v2, fma(k3, v3, w[r]))));
            }
        }
    };
    auto precond = [&]() {
        if (!live) return;
        double m[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) m[t] = M[t * a.max_rows + lr];
#pragma unroll
        for (int r = 0; r < 4; ++r) zr[r] = fma(m[r * 4], rr[0], fma(m[r * 4 + 1], rr[1], fma(m[r * 4 + 2], rr[2], m[r * 4 + 3] * rr[3])));
    };
    auto totals = [&](int buf, int nq, unsigned max_mask) {
        cl.sync();
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (w < nq) {
            const bool mx = (max_mask >> w) & 1u;
            double v = 0.0;
            if (lane < CS) v = cl.map_shared_rank(part, lane)[buf * kSlots + w];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = op2c(mx, v, __shfl_xor_sync(0xffffffffu, v, o));
            if (lane == 0) bcast[w] = v;
        }
        __syncthreads();
    };

    double vals[kSlots];
    int it = 0, restarts = 0, status_code = 0;
    double bmax = 0.0, tol = 0.0, bar = 0.0;
    double rz[3] = {0, 0, 0}, beta[3] = {0, 0, 0};
    bool need_init = true;
    // per-thread slots: sums go to the slot of the own column
    auto put_col = [&](int base, double v) {
#pragma unroll
        for (int c = 0; c < 3; ++c) vals[base + c] += c == col ? v : 0.0;
    };
    while (true) {
        if (need_init) {
            exchange(xr);
#pragma unroll
            for (int q = 0; q < kSlots; ++q) vals[q] = 0.0;
            {
                double w[4];
                spmv(w);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const double bk = live ? a.B[gb + 3 * t] : 0.0;
                    rr[t] = bk - w[t];
                    vals[0] = fmax(vals[0], fabs(rr[t]));
                    vals[1] = fmax(vals[1], fabs(bk));
                }
            }
            precond();
            put_col(2, rr[0] * zr[0] + rr[1] * zr[1] + rr[2] * zr[2] + rr[3] * zr[3]);
            block_slots(vals, 5, red, part + kSlots, 0x3u);
            totals(1, 5, 0x3u);
            const double rmax0 = bcast[0];
            bmax = bcast[1];
            tol = a.rtol * (1.0 + bmax);
            bar = 1e-8 * (1.0 + bmax);
            const double rz3[3] = {bcast[2], bcast[3], bcast[4]};
            __syncthreads();
            if (restarts > 0 && rmax0 <= bar && (rmax0 <= 100.0 * tol || restarts >= 3)) {
                status_code = 1;
                break;
            }
            if (restarts >= 6) {
                status_code = 3;
                break;
            }
            if (rmax0 <= tol) {
                ++restarts;
                cl.sync();  // all ranks done reading ext before it is rewritten
                continue;
            }
            for (int c = 0; c < 3; ++c) {
                rz[c] = rz3[c];
                beta[c] = 0.0;
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) pr[t] = qr[t] = 0.0;
            need_init = false;
            cl.sync();  // halo reads of x finished everywhere before z overwrites ext
        }
        mark(9);
        exchange(zr);
        mark(0);
        // ---- phase A: q = K z + beta q, p = z + beta p; (p,q)
#pragma unroll
        for (int q = 0; q < kSlots; ++q) vals[q] = 0.0;
        {
            double w[4];
            spmv(w);
            const double bt = beta[col];
            double pq = 0.0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                qr[t] = w[t] + bt * qr[t];
                pr[t] = zr[t] + bt * pr[t];
                pq += pr[t] * qr[t];
            }
            put_col(0, pq);
        }
        mark(1);
        block_slots(vals, 3, red, part, 0x0u);
        mark(2);
        totals(0, 3, 0x0u);
        mark(3);
        double alpha[3];
        bool indefinite = false;
        for (int c = 0; c < 3; ++c) {
            const double pq = bcast[c];
            if (rz[c] == 0.0) {
                alpha[c] = 0.0;
            } else if (!(pq > 0.0)) {
                indefinite = true;
                alpha[c] = 0.0;
            } else {
                alpha[c] = rz[c] / pq;
            }
        }
        if (indefinite) {
            status_code = 2;
            break;
        }
        // ---- phase B: x += alpha p, r -= alpha q, z = M r; (r,z), max|r|
        {
            const double al = alpha[col];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                xr[t] = fma(al, pr[t], xr[t]);
                rr[t] = fma(-al, qr[t], rr[t]);
            }
        }
        precond();
#pragma unroll
        for (int q = 0; q < kSlots; ++q) vals[q] = 0.0;
        put_col(0, rr[0] * zr[0] + rr[1] * zr[1] + rr[2] * zr[2] + rr[3] * zr[3]);
        vals[3] = fmax(fmax(fabs(rr[0]), fabs(rr[1])), fmax(fabs(rr[2]), fabs(rr[3])));
        mark(4);
        block_slots(vals, 4, red, part + kSlots, 0x8u);
        mark(5);
        totals(1, 4, 0x8u);
        mark(6);
        const double rzn[3] = {bcast[0], bcast[1], bcast[2]};
        const double rmax = bcast[3];
        __syncthreads();
        ++it;
        for (int c = 0; c < 3; ++c) {
            beta[c] = rz[c] != 0.0 ? rzn[c] / rz[c] : 0.0;
            rz[c] = rzn[c];
        }
        if (!isfinite(rz[0] + rz[1] + rz[2])) {
            status_code = 2;
            break;
        }
        if (rmax <= tol) {
            ++restarts;
            need_init = true;
            continue;
        }
        if (it >= a.max_iter) {
            status_code = 3;
            break;
        }
    }
    if (live)
#pragma unroll
        for (int t = 0; t < 4; ++t) a.X[gb + 3 * t] = xr[t];
    if (prof)
        for (int k = 0; k < 10; ++k) a.prof[k] += acc_t[k];
    if (rank == 0 && threadIdx.x == 0) {
        a.status->iterations = it;
        a.status->code = status_code;
        a.status->restarts = restarts;
        a.status->bmax = bmax;
    }
    cl.sync();  // no rank leaves while others may still read its shared memory
}

// ---- recursive coordinate bisection into `parts` parts (node weights)
void rcb_split(const double* pos, const std::vector<int>& w, std::vector<int>& ids, int lo, int hi, int g0, int g1,
               std::vector<int>& part_begin) {
    if (g1 - g0 == 1) {
        part_begin[g0] = lo;
        return;
    }
    const int gm = (g0 + g1) / 2;
    double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
    for (int t = lo; t < hi; ++t)
        for (int c = 0; c < 3; ++c) {
            mn[c] = std::min(mn[c], pos[3 * ids[t] + c]);
            mx[c] = std::max(mx[c], pos[3 * ids[t] + c]);
        }
    int axis = 0;
    for (int c = 1; c < 3; ++c)
        if (mx[c] - mn[c] > mx[axis] - mn[axis]) axis = c;
    std::sort(ids.begin() + lo, ids.begin() + hi, [&](int x, int y) {
        const double px = pos[3 * x + axis], py = pos[3 * y + axis];
        return px != py ? px < py : x < y;
    });
    double total = 0;
    for (int t = lo; t < hi; ++t) total += w[ids[t]];
    const double target = total * static_cast<double>(gm - g0) / (g1 - g0);
    double acc = 0;
    int cut = lo;
    while (cut < hi && acc + w[ids[cut]] <= target) acc += w[ids[cut++]];
    cut = std::max(cut, lo + (gm - g0));
    cut = std::min(cut, hi - (g1 - gm));
    rcb_split(pos, w, ids, lo, cut, g0, gm, part_begin);
    rcb_split(pos, w, ids, cut, hi, gm, g1, part_begin);
}

}  // namespace

void ClusterPlan::build(const double* node_pos, const int* row_ptr, const int* col, const int* node_row_bsr, int N,
                        size_t smem_limit, int max_cs) {
    ok = false;
    if (N <= 0) return;
    CS = std::max(1, std::min(max_cs, N / 16));
    const int cap_rows = kClusterThreads / 3;  // three threads (columns) per node
    if ((N + CS - 1) / CS > cap_rows * 15 / 16) return;  // too large for one cluster
    std::vector<int> ids(N), w(N);
    std::iota(ids.begin(), ids.end(), 0);
    for (int j = 0; j < N; ++j) w[j] = 2 + (row_ptr[node_row_bsr[j] + 1] - row_ptr[node_row_bsr[j]]);
    rank_rows.assign(CS + 1, N);
    rcb_split(node_pos, w, ids, 0, N, 0, CS, rank_rows);
    rank_rows[CS] = N;
    row_node = ids;
    node_row.assign(N, 0);
    std::vector<int> rank_of(N), local_of(N);
    for (int r = 0; r < CS; ++r)
        for (int j = rank_rows[r]; j < rank_rows[r + 1]; ++j) {
            node_row[row_node[j]] = j;
            rank_of[row_node[j]] = r;
            local_of[row_node[j]] = j - rank_rows[r];
        }
    max_rows = 0;
    for (int r = 0; r < CS; ++r) max_rows = std::max(max_rows, rank_rows[r + 1] - rank_rows[r]);
    if (max_rows > cap_rows) return;
    ept = 1;
    ent_ptr.assign(N + 1, 0);
    ent.clear();
    diag_ent.assign(N, -1);
    store_off.assign(CS + 1, 0);
    store_src.clear();
    halo_off.assign(CS + 1, 0);
    halo_src.clear();
    max_store = 0;
    max_ext = 0;
    // uniform smem layout: rows*(16+12) + ext*12 + store*16 doubles + fixed
    const size_t fixed_bytes = sizeof(double) * (2 * kSlots + 32 * kSlots + kSlots) + 64;
    int max_halo_rows = 0;
    for (int r = 0; r < CS; ++r) {
        std::unordered_map<int, int> tmp;
        for (int j = rank_rows[r]; j < rank_rows[r + 1]; ++j) {
            const int a = row_node[j];
            const int bj = node_row_bsr[a];
            for (int p = row_ptr[bj]; p < row_ptr[bj + 1]; ++p)
                if (rank_of[col[p]] != r) tmp.emplace(col[p], 0);
        }
        max_halo_rows = std::max(max_halo_rows, rank_rows[r + 1] - rank_rows[r] + static_cast<int>(tmp.size()));
    }
    int max_entries = 0;
    for (int r = 0; r < CS; ++r) {
        int ne = 0;
        for (int j = rank_rows[r]; j < rank_rows[r + 1]; ++j) {
            const int bj = node_row_bsr[row_node[j]];
            ne += row_ptr[bj + 1] - row_ptr[bj];
        }
        max_entries = std::max(max_entries, ne);
    }
    max_ent = max_entries;
    const size_t ent_bytes = sizeof(int2) * static_cast<size_t>(max_ent) + sizeof(int) * (max_rows + 2);
    const long long store_budget_bytes = static_cast<long long>(smem_limit) -
        static_cast<long long>(fixed_bytes + ent_bytes + sizeof(double) * (16 * static_cast<size_t>(max_rows) +
                                                                          kExt * static_cast<size_t>(max_halo_rows)));
    const int fit = static_cast<int>(std::max<long long>(0, store_budget_bytes / (16 * sizeof(double))));
    for (int r = 0; r < CS; ++r) {
        const int rb = rank_rows[r], re = rank_rows[r + 1], nrows = re - rb;
        std::unordered_map<int, int> halo_idx;
        std::vector<int2> rank_halo;
        std::unordered_map<long long, int> pair_slot;
        std::vector<int> slots;  // global positions
        // pass 1: slots for diagonal, intra-rank upper pairs and cross blocks
        struct E {
            int row, pos, other;
        };
        for (int j = rb; j < re; ++j) {
            const int a = row_node[j];
            const int bj = node_row_bsr[a];
            for (int p = row_ptr[bj]; p < row_ptr[bj + 1]; ++p) {
                const int b = col[p];
                if (b == a || rank_of[b] != r || a < b) {
                    if (b != a && rank_of[b] == r) pair_slot[static_cast<long long>(a) * N + b] = static_cast<int>(slots.size());
                    slots.push_back(p);
                }
            }
        }
        // the first `fit` slots live in shared memory, the rest are read from L2
        const int nslots_smem = std::min<int>(fit, static_cast<int>(slots.size()));
        std::vector<int> slot_code(slots.size());
        for (size_t s = 0; s < slots.size(); ++s) {
            if (static_cast<int>(s) < nslots_smem) {
                slot_code[s] = (static_cast<int>(store_src.size()) - store_off[r]) << 2;
                store_src.push_back(slots[s]);
            } else {
                slot_code[s] = (slots[s] << 2) | 1;
            }
        }
        store_off[r + 1] = static_cast<int>(store_src.size());
        max_store = std::max(max_store, store_off[r + 1] - store_off[r]);
        // pass 2: entries in BSR column order per row
        int sidx = 0;
        for (int j = rb; j < re; ++j) {
            const int a = row_node[j];
            const int bj = node_row_bsr[a];
            for (int p = row_ptr[bj]; p < row_ptr[bj + 1]; ++p) {
                const int b = col[p];
                int code, extc;
                if (b == a || rank_of[b] != r || a < b) {
                    code = slot_code[sidx++];
                } else {
                    code = slot_code[pair_slot.at(static_cast<long long>(b) * N + a)] | 2;  // transposed
                }
                if (rank_of[b] == r) {
                    extc = local_of[b];
                } else {
                    auto it = halo_idx.find(b);
                    if (it == halo_idx.end()) {
                        it = halo_idx.emplace(b, static_cast<int>(rank_halo.size())).first;
                        rank_halo.push_back(make_int2(rank_of[b], local_of[b]));
                    }
                    extc = nrows + it->second;
                }
                if (b == a) diag_ent[j] = static_cast<int>(ent.size());
                ent.push_back(make_int2(code, extc));
            }
            ent_ptr[j + 1] = static_cast<int>(ent.size());
        }
        halo_off[r + 1] = halo_off[r] + static_cast<int>(rank_halo.size());
        halo_src.insert(halo_src.end(), rank_halo.begin(), rank_halo.end());
        max_ext = std::max(max_ext, nrows + static_cast<int>(rank_halo.size()));
    }
    smem_bytes = sizeof(double) * (16 * static_cast<size_t>(max_store) + kExt * static_cast<size_t>(max_ext) +
                                   16 * static_cast<size_t>(max_rows)) +
                 fixed_bytes + ent_bytes;
    if (smem_bytes > smem_limit) return;
    ok = true;
}

void launch_pcg_cluster(const ClusterPlan& plan, ClusterArgs a, cudaStream_t s) {
    a.max_rows = plan.max_rows;
    a.max_store = plan.max_store;
    a.max_ext = plan.max_ext;
    a.max_ent = plan.max_ent;
    const void* fn = reinterpret_cast<const void*>(pcg_cluster_kernel);
    allow_max_smem(reinterpret_cast<const void*>(fn));
    NRR_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.CS);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = plan.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = plan.CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {&a};
    NRR_CUDA_CHECK(cudaLaunchKernelExC(&cfg, fn, args));
}

}  // namespace nrr_b200
