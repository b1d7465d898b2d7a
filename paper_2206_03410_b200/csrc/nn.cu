// Closest-point correspondence (reference SpatialIndex, kd_tree.hpp:17-107,
// and find_correspondences, energy.hpp:28-42) on sm_100a.
//
// Index: targets sorted by 30-bit Morton code, grouped 8 per leaf, with an
// implicit 8-ary tree of FP32 AABBs above the leaves (level l node k covers
// level l-1 nodes 8k..8k+7). Points are stored once as float4 (x, y, z
// relative to the index centre, w = original index bits) so a leaf is two
// coalesced 128-byte lines.
//
// Query: one 8-lane group per query (4 queries per warp). At an internal node
// the 8 lanes test the 8 child boxes in parallel and push the survivors
// nearest-last onto a per-group shared-memory stack; at a leaf the 8 lanes
// test the 8 points. FP32 distances only prune: a candidate whose FP32
// distance is within the rounding margin `delta` of the FP64 best is re-ranked
// in FP64 from the original coordinates with the reference's tie rule
// (d2 < best or d2 == best and index < best index, kd_tree.hpp:88). Boxes are
// pruned only when their FP32 distance exceeds best + delta, i.e. never when
// an equal-distance point could sit inside (the reference's non-strict prune,
// kd_tree.hpp:99-100). The result is the exact FP64 argmin with the smallest
// index on ties. The previous pass's index seeds the bound (warm start).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include <cub/cub.cuh>

#include "device_common.cuh"
#include "nn.cuh"

namespace nrr_b200 {

namespace {
inline uint32_t spread10(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
}  // namespace

void BvhHost::build(const double* tgt, int m_) {
    m = m_;
    if (m <= 0) throw NumericalError("SpatialIndex: cannot index an empty point set");
    double lo[3] = {tgt[0], tgt[1], tgt[2]}, hi[3] = {tgt[0], tgt[1], tgt[2]};
    for (int i = 1; i < m; ++i)
        for (int c = 0; c < 3; ++c) {
            const double v = tgt[3 * i + c];
            if (!std::isfinite(v)) throw NumericalError("SpatialIndex: non-finite target point");
            lo[c] = std::min(lo[c], v);
            hi[c] = std::max(hi[c], v);
        }
    for (int c = 0; c < 3; ++c) {
        center[c] = 0.5 * (lo[c] + hi[c]);
        this->lo[c] = lo[c];
        this->hi[c] = hi[c];
    }
    double ext = 0;
    for (int c = 0; c < 3; ++c) ext = std::max(ext, hi[c] - lo[c]);
    half_extent = 0;
    std::vector<std::pair<uint32_t, int>> keys(m);
    for (int i = 0; i < m; ++i) {
        uint32_t code = 0;
        for (int c = 0; c < 3; ++c) {
            const double u = ext > 0 ? (tgt[3 * i + c] - lo[c]) / ext : 0.0;
            const uint32_t q = static_cast<uint32_t>(std::min(1023.0, std::max(0.0, u * 1024.0)));
            code |= spread10(q) << c;
            half_extent = std::max(half_extent, std::abs(tgt[3 * i + c] - center[c]));
        }
        keys[i] = {code, i};
    }
    // (code, index) order by a stable LSD radix sort on the 30-bit code (16 + 14
    // bits); the input is already in index order, so ties keep it
    {
        std::vector<std::pair<uint32_t, int>> tmp(m);
        for (int pass = 0; pass < 2; ++pass) {
            const int shift = 16 * pass, bins = 1 << 16;
            std::vector<int> cnt(bins + 1, 0);
            for (int i = 0; i < m; ++i) ++cnt[((keys[i].first >> shift) & 0xFFFFu) + 1];
            for (int b = 0; b < bins; ++b) cnt[b + 1] += cnt[b];
            for (int i = 0; i < m; ++i) tmp[cnt[(keys[i].first >> shift) & 0xFFFFu]++] = keys[i];
            keys.swap(tmp);
        }
    }
    const int mpad = (m + 7) / 8 * 8;
    pts.assign(mpad, make_float4(1e18f, 1e18f, 1e18f, 0.f));
    for (int k = 0; k < mpad; ++k) {
        int idx = -1;
        if (k < m) {
            idx = keys[k].second;
            pts[k].x = static_cast<float>(tgt[3 * idx] - center[0]);
            pts[k].y = static_cast<float>(tgt[3 * idx + 1] - center[1]);
            pts[k].z = static_cast<float>(tgt[3 * idx + 2] - center[2]);
        }
        std::memcpy(&pts[k].w, &idx, 4);
    }
    // level 0 boxes over the leaves, then 8-ary levels until <= 8 nodes
    level_off.clear();
    level_cnt.clear();
    box_lo.clear();
    box_hi.clear();
    int cnt = mpad / 8;
    level_off.push_back(0);
    level_cnt.push_back(cnt);
    for (int k = 0; k < cnt; ++k) {
        float4 l = make_float4(INFINITY, INFINITY, INFINITY, 0), h = make_float4(-INFINITY, -INFINITY, -INFINITY, 0);
        for (int t = 0; t < 8; ++t) {
            const int p = 8 * k + t;
            if (p >= m) break;
            l.x = std::min(l.x, pts[p].x);
            l.y = std::min(l.y, pts[p].y);
            l.z = std::min(l.z, pts[p].z);
            h.x = std::max(h.x, pts[p].x);
            h.y = std::max(h.y, pts[p].y);
            h.z = std::max(h.z, pts[p].z);
        }
        box_lo.push_back(l);
        box_hi.push_back(h);
    }
    while (cnt > 8) {
        const int prev_off = level_off.back(), prev_cnt = cnt;
        cnt = (prev_cnt + 7) / 8;
        level_off.push_back(static_cast<int>(box_lo.size()));
        level_cnt.push_back(cnt);
        for (int k = 0; k < cnt; ++k) {
            float4 l = make_float4(INFINITY, INFINITY, INFINITY, 0), h = make_float4(-INFINITY, -INFINITY, -INFINITY, 0);
            for (int t = 0; t < 8; ++t) {
                const int c = 8 * k + t;
                if (c >= prev_cnt) break;
                const float4 cl = box_lo[prev_off + c], ch = box_hi[prev_off + c];
                l.x = std::min(l.x, cl.x);
                l.y = std::min(l.y, cl.y);
                l.z = std::min(l.z, cl.z);
                h.x = std::max(h.x, ch.x);
                h.y = std::max(h.y, ch.y);
                h.z = std::max(h.z, ch.z);
            }
            box_lo.push_back(l);
            box_hi.push_back(h);
        }
    }
    if (level_cnt.size() > static_cast<size_t>(kMaxLevels - 1))
        throw NumericalError("SpatialIndex: target too large for the BVH level table");
}

namespace {

constexpr int kGroupsPerBlock = 32;  // 256 threads
constexpr int kStack = 96;

__device__ __forceinline__ double exact_d2(const double* t, double qx, double qy, double qz) {
    // (t - q).squaredNorm() as x*x + y*y + z*z without contraction, as the
    // reference / oracle evaluate it
    const double dx = __dsub_rn(t[0], qx), dy = __dsub_rn(t[1], qy), dz = __dsub_rn(t[2], qz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// squared FP32 distance from the query to a box (compared with thr^2: no
// square root on the traversal path)
__device__ __forceinline__ float box_dist2(const float4& l, const float4& h, float qx, float qy, float qz) {
    const float dx = fmaxf(fmaxf(l.x - qx, qx - h.x), 0.f);
    const float dy = fmaxf(fmaxf(l.y - qy, qy - h.y), 0.f);
    const float dz = fmaxf(fmaxf(l.z - qz, qz - h.z), 0.f);
    return dx * dx + dy * dy + dz * dz;
}

// five CTAs per SM (48 registers instead of 54, no spills): config 2 49.2 -> 46.5 us, config 4 538 -> 521 us;
// six spill and lose (profiles/r04_occupancy_ab.txt)
#ifndef NRR_NN_MINB
#define NRR_NN_MINB 5
#endif
__global__ void __launch_bounds__(256, NRR_NN_MINB) nn_kernel(BvhView bv, const double* __restrict__ queries, int nq,
                                                  const int* __restrict__ prev_idx, int* __restrict__ out_idx,
                                                  double* __restrict__ out_d2, double* __restrict__ out_q,
                                                  const double* __restrict__ anchor) {
    __shared__ int st_node[kGroupsPerBlock][kStack];
    __shared__ float st_dist[kGroupsPerBlock][kStack];
    const int lane = threadIdx.x & 7;
    const int gl = threadIdx.x >> 3;
    const int group = blockIdx.x * kGroupsPerBlock + gl;
    if (group >= nq) return;  // whole 8-lane group leaves together
    const unsigned gmask = 0xFFu << (threadIdx.x & 24);
    const int gshift = threadIdx.x & 24;

    const double qx = queries[3 * group], qy = queries[3 * group + 1], qz = queries[3 * group + 2];
    const float fx = static_cast<float>(qx - bv.cx), fy = static_cast<float>(qy - bv.cy),
                fz = static_cast<float>(qz - bv.cz);
    // FP32 rounding margin (|d32 - d64| <= ~5e-7 (S + |q-c|), 8x slack)
    const float qmag = fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz)));
    const float delta = 4e-6f * (bv.half_extent + qmag) + 1e-30f;

    double best_d2 = INFINITY;
    int best_i = 0x7fffffff;
    if (prev_idx) {
        const int p = prev_idx[group];
        if (p >= 0 && p < bv.m) {
            best_d2 = exact_d2(bv.tgt64 + 3 * p, qx, qy, qz);
            best_i = p;
        }
    }
    if (best_d2 == INFINITY && bv.gpts != nullptr) {
        // no seed: any point of the query's own cell (if it has one) gives a
        // bound, usually tight enough for the grid path below
        const int ix = static_cast<int>(floorf((fx - bv.glx) * bv.inv_h));
        const int iy = static_cast<int>(floorf((fy - bv.gly) * bv.inv_h));
        const int iz = static_cast<int>(floorf((fz - bv.glz) * bv.inv_h));
        if (ix >= 0 && ix < bv.gnx && iy >= 0 && iy < bv.gny && iz >= 0 && iz < bv.gnz) {
            const int cell = (ix * bv.gny + iy) * bv.gnz + iz;
            const int p0 = bv.cell_start[cell];
            if (p0 < bv.cell_start[cell + 1]) {
                int idx;
                const float w = bv.gpts[p0].w;
                memcpy(&idx, &w, 4);
                best_d2 = exact_d2(bv.tgt64 + 3 * idx, qx, qy, qz);
                best_i = idx;
            }
        }
    }
    // ---- grid path: a warm-started query whose search ball covers at most
    // kGridCells cells scans those cells (8 lanes round-robin over them);
    // every point within the bound lies in one of them (cells partition space)
    if (bv.gpts != nullptr && best_d2 < INFINITY) {
        const float r = static_cast<float>(sqrt(best_d2)) * 1.000001f + delta;
        const int x0 = max(0, static_cast<int>(floorf((fx - r - bv.glx) * bv.inv_h)));
        const int x1 = min(bv.gnx - 1, static_cast<int>(floorf((fx + r - bv.glx) * bv.inv_h)));
        const int y0 = max(0, static_cast<int>(floorf((fy - r - bv.gly) * bv.inv_h)));
        const int y1 = min(bv.gny - 1, static_cast<int>(floorf((fy + r - bv.gly) * bv.inv_h)));
        const int z0 = max(0, static_cast<int>(floorf((fz - r - bv.glz) * bv.inv_h)));
        const int z1 = min(bv.gnz - 1, static_cast<int>(floorf((fz + r - bv.glz) * bv.inv_h)));
        const int cx = x1 - x0 + 1, cy = y1 - y0 + 1, cz = z1 - z0 + 1;
        if (cx > 0 && cy > 0 && cz > 0 && cx * cy * cz <= bv.gmax_cells) {
            const float r2 = r * r;
            double my_d2 = best_d2;
            int my_i = best_i;
            // The cells of one (x, y) column of the ball are consecutive in
            // the cell-major point array, so a column is one contiguous run
            // [cell_start[first], cell_start[last + 1]): two index loads per
            // column instead of two per cell, and the run's points share
            // sectors. A lane takes columns lane, lane + 8, ...; the ranges of
            // two columns and the points of a run (4 at a time) are loaded
            // before they are used, so the dependent chain is ranges -> points
            // -> (rarely) the FP64 coordinates of a candidate.
            auto scan = [&](int p0, int p1) {
                for (int k = p0; k < p1; k += 4) {
                    float4 pt[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) pt[u] = k + u < p1 ? bv.gpts[k + u] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (k + u >= p1) break;
                        const float dx = pt[u].x - fx, dy = pt[u].y - fy, dz = pt[u].z - fz;
                        if (dx * dx + dy * dy + dz * dz > r2) continue;
                        int idx;
                        memcpy(&idx, &pt[u].w, 4);
                        const double d2 = exact_d2(bv.tgt64 + 3 * idx, qx, qy, qz);
                        if (d2 < my_d2 || (d2 == my_d2 && idx < my_i)) {
                            my_d2 = d2;
                            my_i = idx;
                        }
                    }
                }
            };
            const int ncol = cx * cy;
            for (int c = lane; c < ncol; c += 16) {
                const int iy = c % cy, ix = c / cy;
                const int cell = ((x0 + ix) * bv.gny + (y0 + iy)) * bv.gnz + z0;
                const int p0 = bv.cell_start[cell], p1 = bv.cell_start[cell + cz];
                int q0 = 0, q1 = 0;
                if (c + 8 < ncol) {
                    const int c2 = c + 8, jy = c2 % cy, jx = c2 / cy;
                    const int cell2 = ((x0 + jx) * bv.gny + (y0 + jy)) * bv.gnz + z0;
                    q0 = bv.cell_start[cell2];
                    q1 = bv.cell_start[cell2 + cz];
                }
                scan(p0, p1);
                scan(q0, q1);
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(gmask, my_d2, o, 8);
                const int oi = __shfl_xor_sync(gmask, my_i, o, 8);
                if (od < my_d2 || (od == my_d2 && oi < my_i)) {
                    my_d2 = od;
                    my_i = oi;
                }
            }
            if (bv.stats && lane == 0) atomicAdd(bv.stats + 3, 1ull);
            if (lane == 0) {
                out_idx[group] = my_i;
                out_d2[group] = my_d2;
                if (out_q) {
                    const double* t = bv.tgt64 + 3 * my_i;
                    out_q[3 * group] = t[0] - anchor[3 * group];
                    out_q[3 * group + 1] = t[1] - anchor[3 * group + 1];
                    out_q[3 * group + 2] = t[2] - anchor[3 * group + 2];
                }
            }
            return;
        }
    }
    int* sn = st_node[gl];
    float* sd = st_dist[gl];
    int sp = 0;
    if (lane == 0) {
        sn[0] = ((bv.levels) << 27);  // virtual root above the top level
        sd[0] = 0.f;  // squared box distances on the stack
    }
    sp = 1;
    __syncwarp(gmask);
    // prune radius: FP32 sqrt of the FP64 best, inflated by the rounding
    // margin; refreshed only when the best changes
    float thr = static_cast<float>(sqrt(best_d2)) * 1.000001f + delta;  // inf stays inf
    float thr2 = thr * thr;
    while (sp > 0) {
        --sp;
        const int code = sn[sp];
        const float bdist2 = sd[sp];
        __syncwarp(gmask);
        if (bdist2 > thr2) continue;
        const int L = code >> 27, v = code & ((1 << 27) - 1);
        if (bv.stats && lane == 0) atomicAdd(bv.stats + (L == 0 ? 1 : 0), 1ull);
        if (L == 0) {
            const float4 p = bv.pts[8 * v + lane];
            int idx;
            memcpy(&idx, &p.w, 4);
            const float dx = p.x - fx, dy = p.y - fy, dz = p.z - fz;
            const float d2f = dx * dx + dy * dy + dz * dz;
            const bool cand = idx >= 0 && d2f <= thr2;
            // most leaves reached with the warm-start bound hold no candidate:
            // skip the FP64 re-rank and the group reduction
            if (((__ballot_sync(gmask, cand) >> gshift) & 0xFFu) == 0u) continue;
            if (bv.stats && lane == 0) atomicAdd(bv.stats + 2, 1ull);
            double my_d2 = INFINITY;
            int my_i = 0x7fffffff;
            if (cand) {
                my_d2 = exact_d2(bv.tgt64 + 3 * idx, qx, qy, qz);
                my_i = idx;
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(gmask, my_d2, o, 8);
                const int oi = __shfl_xor_sync(gmask, my_i, o, 8);
                if (od < my_d2 || (od == my_d2 && oi < my_i)) {
                    my_d2 = od;
                    my_i = oi;
                }
            }
            if (my_d2 < best_d2 || (my_d2 == best_d2 && my_i < best_i)) {
                if (my_d2 < best_d2) {
                    thr = static_cast<float>(sqrt(my_d2)) * 1.000001f + delta;
                    thr2 = thr * thr;
                }
                best_d2 = my_d2;
                best_i = my_i;
            }
        } else {
            const int cl = L - 1;
            const int c = 8 * v + lane;
            const bool exists = c < bv.level_cnt[cl];
            float bd = INFINITY;
            if (exists) {
                const int b = bv.level_off[cl] + c;
                bd = box_dist2(bv.box_lo[b], bv.box_hi[b], fx, fy, fz);
            }
            const bool valid = exists && bd <= thr2;
            const unsigned ball = (__ballot_sync(gmask, valid) >> gshift) & 0xFFu;
            const int cnt = __popc(ball);
            // children in Morton order (the warm-start bound is already tight,
            // so nearest-first ordering buys little; exactness does not depend
            // on the order)
            const int rank = __popc(ball & ((1u << lane) - 1u));
            if (valid && sp + rank < kStack) {
                sn[sp + rank] = (cl << 27) | c;
                sd[sp + rank] = bd;
            }
            if (sp + cnt > kStack && lane == 0 && bv.overflow) atomicOr(bv.overflow, 1);  // the host raises
            sp = min(sp + cnt, kStack);
            __syncwarp(gmask);
        }
    }
    if (bv.stats && lane == 0) atomicAdd(bv.stats + 3, 1ull);
    if (lane == 0) {
        out_idx[group] = best_i;
        out_d2[group] = best_d2;
        if (out_q) {
            const double* t = bv.tgt64 + 3 * best_i;
            out_q[3 * group] = t[0] - anchor[3 * group];
            out_q[3 * group + 1] = t[1] - anchor[3 * group + 1];
            out_q[3 * group + 2] = t[2] - anchor[3 * group + 2];
        }
    }
}

}  // namespace

void launch_nn(const BvhView& bv, const double* queries, int nq, const int* prev_idx, int* out_idx, double* out_d2,
               double* out_q, const double* anchor, cudaStream_t s) {
    if (nq <= 0) return;
    const int blocks = (nq + kGroupsPerBlock - 1) / kGroupsPerBlock;
    nn_kernel<<<blocks, kGroupsPerBlock * 8, 0, s>>>(bv, queries, nq, prev_idx, out_idx, out_d2, out_q, anchor);
    NRR_CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- uniform grid
namespace {

__global__ void grid_cell_kernel(const double* __restrict__ t, int m, double cx, double cy, double cz, float lx,
                                 float ly, float lz, float inv_h, int nx, int ny, int nz, int* __restrict__ key,
                                 int* __restrict__ val, int* __restrict__ cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    // the same FP32 quantities the query path uses
    const float px = static_cast<float>(t[3 * i] - cx), py = static_cast<float>(t[3 * i + 1] - cy),
                pz = static_cast<float>(t[3 * i + 2] - cz);
    const int ix = min(nx - 1, max(0, static_cast<int>(floorf((px - lx) * inv_h))));
    const int iy = min(ny - 1, max(0, static_cast<int>(floorf((py - ly) * inv_h))));
    const int iz = min(nz - 1, max(0, static_cast<int>(floorf((pz - lz) * inv_h))));
    const int cell = (ix * ny + iy) * nz + iz;
    key[i] = cell;
    val[i] = i;
    atomicAdd(cnt + cell, 1);
}

__global__ void grid_points_kernel(const double* __restrict__ t, int m, double cx, double cy, double cz,
                                   const int* __restrict__ order, float4* __restrict__ gpts) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int i = order[k];
    float4 p;
    p.x = static_cast<float>(t[3 * i] - cx);
    p.y = static_cast<float>(t[3 * i + 1] - cy);
    p.z = static_cast<float>(t[3 * i + 2] - cz);
    memcpy(&p.w, &i, 4);
    gpts[k] = p;
}

size_t a256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

int bits_for(long long n) {
    int b = 1;
    while ((1LL << b) < n) ++b;
    return b;
}

}  // namespace

GridDims grid_dims(const double lo[3], const double hi[3], int m, double factor) {
    GridDims g;
    double ext[3], vol = 1.0, emax = 0.0;
    for (int c = 0; c < 3; ++c) {
        ext[c] = hi[c] - lo[c];
        emax = std::max(emax, ext[c]);
    }
    if (!(emax > 0.0) || m < 64) return g;
    for (int c = 0; c < 3; ++c) vol *= std::max(ext[c], emax * 1e-3);
    double h = factor * std::cbrt(vol / m);
    for (int pass = 0; pass < 64; ++pass) {
        const long long nx = static_cast<long long>(ext[0] / h) + 1, ny = static_cast<long long>(ext[1] / h) + 1,
                        nz = static_cast<long long>(ext[2] / h) + 1;
        if (nx * ny * nz <= (32LL << 20)) {
            g.nx = static_cast<int>(nx);
            g.ny = static_cast<int>(ny);
            g.nz = static_cast<int>(nz);
            g.h = h;
            return g;
        }
        h *= 1.25;
    }
    return g;
}

size_t grid_scratch_bytes(int m, long long ncells) {
    size_t sort_b = 0, scan_b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_b, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                    static_cast<const int*>(nullptr), static_cast<int*>(nullptr), m, 0,
                                    bits_for(ncells));
    cub::DeviceScan::ExclusiveSum(nullptr, scan_b, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                  static_cast<int>(ncells + 1));
    return 4 * a256(sizeof(int) * static_cast<size_t>(m)) + a256(sizeof(int) * static_cast<size_t>(ncells + 1)) +
           a256(std::max(sort_b, scan_b)) + 256;
}

void build_grid(const double* tgt64, int m, const double center[3], const double lo[3], const GridDims& g,
                float4* gpts, int* cell_start, void* scratch, cudaStream_t s) {
    const long long ncells = static_cast<long long>(g.nx) * g.ny * g.nz;
    char* p = static_cast<char*>(scratch);
    const size_t eb = a256(sizeof(int) * static_cast<size_t>(m));
    int* key = reinterpret_cast<int*>(p);
    int* key2 = reinterpret_cast<int*>(p + eb);
    int* val = reinterpret_cast<int*>(p + 2 * eb);
    int* val2 = reinterpret_cast<int*>(p + 3 * eb);
    int* cnt = reinterpret_cast<int*>(p + 4 * eb);
    void* tmp = p + 4 * eb + a256(sizeof(int) * static_cast<size_t>(ncells + 1));
    size_t tb = grid_scratch_bytes(m, ncells);
    NRR_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int) * static_cast<size_t>(ncells + 1), s));
    const float lx = static_cast<float>(lo[0] - center[0]), ly = static_cast<float>(lo[1] - center[1]),
                lz = static_cast<float>(lo[2] - center[2]);
    const float inv_h = static_cast<float>(1.0 / g.h);
    const int blocks = (m + 255) / 256;
    grid_cell_kernel<<<blocks, 256, 0, s>>>(tgt64, m, center[0], center[1], center[2], lx, ly, lz, inv_h, g.nx, g.ny,
                                            g.nz, key, val, cnt);
    NRR_CUDA_CHECK(cudaGetLastError());
    NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, val, val2, m, 0, bits_for(ncells), s));
    tb = grid_scratch_bytes(m, ncells);
    NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, cell_start, static_cast<int>(ncells + 1), s));
    grid_points_kernel<<<blocks, 256, 0, s>>>(tgt64, m, center[0], center[1], center[2], val2, gpts);
    NRR_CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- device BVH build
// The same index as BvhHost::build (Morton order by a stable radix sort of the
// 30-bit codes, float4 points relative to the centre, 8-point leaves, 8-ary
// FP32 box levels), built on the device: identical bits, no host pass over
// the targets beyond the box reduction's few partials.
namespace {
constexpr int kBvhBlocks = 296;
__device__ __forceinline__ unsigned spread10_bvh(unsigned v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void bvh_bbox_kernel(const double* __restrict__ t, int m, double* __restrict__ part, int* __restrict__ bad) {
    __shared__ double sh[6][256];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    bool nf = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        for (int c = 0; c < 3; ++c) {
            const double v = t[3 * i + c];
            nf |= !isfinite(v);
            lo[c] = fmin(lo[c], v);
            hi[c] = fmax(hi[c], v);
        }
    if (nf) atomicOr(bad, 1);
    for (int c = 0; c < 3; ++c) {
        sh[c][threadIdx.x] = lo[c];
        sh[3 + c][threadIdx.x] = hi[c];
    }
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int c = 0; c < 3; ++c) {
                sh[c][threadIdx.x] = fmin(sh[c][threadIdx.x], sh[c][threadIdx.x + o]);
                sh[3 + c][threadIdx.x] = fmax(sh[3 + c][threadIdx.x], sh[3 + c][threadIdx.x + o]);
            }
        __syncthreads();
    }
    if (threadIdx.x < 6) part[6 * blockIdx.x + threadIdx.x] = sh[threadIdx.x][0];
}

// Morton code (BvhHost::build's arithmetic) and max |t - centre| partials
__global__ void bvh_code_kernel(const double* __restrict__ t, int m, double l0, double l1, double l2, double ext,
                                double c0, double c1, double c2, unsigned* __restrict__ code, int* __restrict__ idx,
                                double* __restrict__ hpart) {
    __shared__ double sh[256];
    double h = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const double v[3] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
        const double lo[3] = {l0, l1, l2}, ct[3] = {c0, c1, c2};
        unsigned k = 0;
        for (int c = 0; c < 3; ++c) {
            const double u = ext > 0 ? (v[c] - lo[c]) / ext : 0.0;
            const unsigned q = static_cast<unsigned>(fmin(1023.0, fmax(0.0, u * 1024.0)));
            k |= spread10_bvh(q) << c;
            h = fmax(h, fabs(v[c] - ct[c]));
        }
        code[i] = k;
        idx[i] = i;
    }
    sh[threadIdx.x] = h;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) hpart[blockIdx.x] = sh[0];
}

__global__ void bvh_points_kernel(const double* __restrict__ t, int m, int mpad, const int* __restrict__ order,
                                  double c0, double c1, double c2, float4* __restrict__ pts) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= mpad) return;
    float4 p = make_float4(1e18f, 1e18f, 1e18f, 0.f);
    int idx = -1;
    if (k < m) {
        idx = order[k];
        p.x = static_cast<float>(t[3 * idx] - c0);
        p.y = static_cast<float>(t[3 * idx + 1] - c1);
        p.z = static_cast<float>(t[3 * idx + 2] - c2);
    }
    memcpy(&p.w, &idx, 4);
    pts[k] = p;
}

// level 0: one box per 8 points (valid points only); level l: per 8 children
__global__ void bvh_leaf_box_kernel(const float4* __restrict__ pts, int m, int cnt, float4* __restrict__ lo,
                                    float4* __restrict__ hi) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    float4 l = make_float4(INFINITY, INFINITY, INFINITY, 0), h = make_float4(-INFINITY, -INFINITY, -INFINITY, 0);
    for (int t = 0; t < 8; ++t) {
        const int p = 8 * k + t;
        if (p >= m) break;
        const float4 q = pts[p];
        l.x = fminf(l.x, q.x);
        l.y = fminf(l.y, q.y);
        l.z = fminf(l.z, q.z);
        h.x = fmaxf(h.x, q.x);
        h.y = fmaxf(h.y, q.y);
        h.z = fmaxf(h.z, q.z);
    }
    lo[k] = l;
    hi[k] = h;
}
__global__ void bvh_level_box_kernel(float4* __restrict__ lo, float4* __restrict__ hi, int prev_off, int prev_cnt,
                                     int off, int cnt) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    float4 l = make_float4(INFINITY, INFINITY, INFINITY, 0), h = make_float4(-INFINITY, -INFINITY, -INFINITY, 0);
    for (int t = 0; t < 8; ++t) {
        const int c = 8 * k + t;
        if (c >= prev_cnt) break;
        const float4 cl = lo[prev_off + c], ch = hi[prev_off + c];
        l.x = fminf(l.x, cl.x);
        l.y = fminf(l.y, cl.y);
        l.z = fminf(l.z, cl.z);
        h.x = fmaxf(h.x, ch.x);
        h.y = fmaxf(h.y, ch.y);
        h.z = fmaxf(h.z, ch.z);
    }
    lo[off + k] = l;
    hi[off + k] = h;
}
}  // namespace

void bvh_layout(int m, std::vector<int>& level_off, std::vector<int>& level_cnt, int& total_boxes) {
    level_off.clear();
    level_cnt.clear();
    int cnt = (m + 7) / 8;
    level_off.push_back(0);
    level_cnt.push_back(cnt);
    total_boxes = cnt;
    while (cnt > 8) {
        cnt = (cnt + 7) / 8;
        level_off.push_back(total_boxes);
        level_cnt.push_back(cnt);
        total_boxes += cnt;
    }
    if (level_cnt.size() > static_cast<size_t>(kMaxLevels - 1))
        throw NumericalError("SpatialIndex: target too large for the BVH level table");
}

size_t bvh_scratch_bytes(int m) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<const unsigned*>(nullptr), static_cast<unsigned*>(nullptr),
                                    static_cast<const int*>(nullptr), static_cast<int*>(nullptr), m, 0, 30);
    return 4 * a256(sizeof(int) * static_cast<size_t>(std::max(m, 1))) + a256(b) +
           a256(sizeof(double) * 6 * kBvhBlocks) + a256(sizeof(double) * kBvhBlocks) + 512;
}

void build_bvh_device(const double* tgt64, int m, BvhHost& meta, float4* pts, float4* box_lo, float4* box_hi,
                      void* scratch, cudaStream_t s) {
    if (m <= 0) throw NumericalError("SpatialIndex: cannot index an empty point set");
    meta.m = m;
    char* p = static_cast<char*>(scratch);
    const size_t eb = a256(sizeof(int) * static_cast<size_t>(m));
    unsigned* code = reinterpret_cast<unsigned*>(p);
    unsigned* code2 = reinterpret_cast<unsigned*>(p + eb);
    int* idx = reinterpret_cast<int*>(p + 2 * eb);
    int* order = reinterpret_cast<int*>(p + 3 * eb);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, code, code2, idx, order, m, 0, 30);
    void* tmp = p + 4 * eb;
    double* part = reinterpret_cast<double*>(p + 4 * eb + a256(tb));
    double* hpart = part + 6 * kBvhBlocks;
    int* bad = reinterpret_cast<int*>(hpart + kBvhBlocks);
    NRR_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), s));
    bvh_bbox_kernel<<<kBvhBlocks, 256, 0, s>>>(tgt64, m, part, bad);
    NRR_CUDA_CHECK(cudaGetLastError());
    std::vector<double> h(6 * kBvhBlocks + 1);
    int hbad = 0;
    NRR_CUDA_CHECK(cudaMemcpyAsync(h.data(), part, sizeof(double) * 6 * kBvhBlocks, cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
    if (hbad) throw NumericalError("SpatialIndex: non-finite target point");
    for (int c = 0; c < 3; ++c) {
        meta.lo[c] = INFINITY;
        meta.hi[c] = -INFINITY;
    }
    for (int b = 0; b < kBvhBlocks; ++b)
        for (int c = 0; c < 3; ++c) {
            meta.lo[c] = std::min(meta.lo[c], h[6 * b + c]);
            meta.hi[c] = std::max(meta.hi[c], h[6 * b + 3 + c]);
        }
    double ext = 0;
    for (int c = 0; c < 3; ++c) {
        meta.center[c] = 0.5 * (meta.lo[c] + meta.hi[c]);
        ext = std::max(ext, meta.hi[c] - meta.lo[c]);
    }
    bvh_code_kernel<<<kBvhBlocks, 256, 0, s>>>(tgt64, m, meta.lo[0], meta.lo[1], meta.lo[2], ext, meta.center[0],
                                               meta.center[1], meta.center[2], code, idx, hpart);
    NRR_CUDA_CHECK(cudaGetLastError());
    NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, code, code2, idx, order, m, 0, 30, s));
    const int mpad = (m + 7) / 8 * 8;
    bvh_points_kernel<<<(mpad + 255) / 256, 256, 0, s>>>(tgt64, m, mpad, order, meta.center[0], meta.center[1],
                                                         meta.center[2], pts);
    NRR_CUDA_CHECK(cudaGetLastError());
    int total = 0;
    bvh_layout(m, meta.level_off, meta.level_cnt, total);
    bvh_leaf_box_kernel<<<(meta.level_cnt[0] + 255) / 256, 256, 0, s>>>(pts, m, meta.level_cnt[0], box_lo, box_hi);
    NRR_CUDA_CHECK(cudaGetLastError());
    for (size_t l = 1; l < meta.level_cnt.size(); ++l) {
        bvh_level_box_kernel<<<(meta.level_cnt[l] + 255) / 256, 256, 0, s>>>(
            box_lo, box_hi, meta.level_off[l - 1], meta.level_cnt[l - 1], meta.level_off[l], meta.level_cnt[l]);
        NRR_CUDA_CHECK(cudaGetLastError());
    }
    std::vector<double> hp(kBvhBlocks);
    NRR_CUDA_CHECK(cudaMemcpyAsync(hp.data(), hpart, sizeof(double) * kBvhBlocks, cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
    meta.half_extent = 0;
    for (double v : hp) meta.half_extent = std::max(meta.half_extent, v);
    meta.pts.clear();  // device-resident
    meta.box_lo.clear();
    meta.box_hi.clear();
}

}  // namespace nrr_b200
