// Device-side graph setup: exact kNN connectivity
// (reference knn_edges, surface.hpp:70-94) and the deformation-graph build
// (build_graph, deformation_graph.hpp:157-210, with pca_order :73-106,
// limited_geodesic geodesic.hpp:22-84, influence weights :111-125 and the
// regularization table :130-148) on the B200, bitwise equal to the host
// restatement (setup.cpp) and the oracle.
//
// Exactness rules. Every floating-point expression that decides membership,
// order or an output value is evaluated with the same operations in the same
// order as the host code, without FMA contraction (__dmul_rn / __dadd_rn /
// __dsub_rn; division and sqrt are IEEE on sm_100a). Sums the reference
// accumulates sequentially (the PCA mean and covariance, the inverse-length
// sum of the regularization table) are accumulated sequentially on the
// device by one thread from shared-memory staged chunks; everything else is
// order-independent (min/max, membership, sorting with explicit tie rules).
//
// kNN. Points are counting-sorted into a uniform grid (the host's cell size
// rule). One thread per query, queries in cell order so a warp scans nearby
// cells: shells of cells around the query's cell are scanned until the k-th
// (squared distance, index) candidate is closer than the unvisited region,
// the reference's lexicographic (d2, index) order. Edges (min, max) of all
// queries are radix-sorted and deduplicated on the device.
//
// Graph. The reference's sweep (a point in PCA order becomes a node unless an
// earlier node's geodesic ball of radius R holds it) is the lexicographically
// first maximal independent set of the relation "q's limited geodesic ball
// contains p". It is computed in rounds (Blelloch-style LFMIS): a point is
// decided once every earlier point within Euclidean distance R (a superset of
// the points whose ball can hold it: ball membership needs the BFS test
// |p - q| < R) is decided; it is then a node unless a node's ball already
// marked it. Each round's new nodes compute their balls, one CTA per node:
// the Euclidean candidates (grid of cell >= R), the BFS component through
// in-ball vertices (sorted list + binary search), then the edge-graph
// distances by Bellman-Ford relaxation to the fixed point. With monotone
// correctly rounded addition that fixed point is bitwise the reference's
// Dijkstra result (every Dijkstra distance is the rounded left-to-right sum
// along a path whose prefixes stay below R, and relaxing from every vertex
// below R reaches exactly the minimum over those paths). Later ball members
// are marked covered at once, so the decided front advances about R per
// round. Node ids follow PCA order; influence lists, graph edges and the
// directed pair table are then built by device sorts in the reference order.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "device_common.cuh"
#include "errors.hpp"
#include "setup.hpp"
#include "setup_graph.hpp"

namespace nrr_b200 {

namespace {

constexpr int kT = 256;

template <typename T>
struct Dev {  // plain device array (setup only: allocated per call)
    T* p = nullptr;
    size_t n = 0;
    Dev() = default;
    explicit Dev(size_t count) { resize(count); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    ~Dev() {
        if (p) cudaFree(p);
    }
    void resize(size_t count) {
        if (count <= n && p) return;
        if (p) NRR_CUDA_CHECK(cudaFree(p));
        p = nullptr;
        n = std::max<size_t>(count, 1);
        NRR_CUDA_CHECK(cudaMalloc(&p, n * sizeof(T)));
    }
};

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { NRR_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() {
        if (s) cudaStreamDestroy(s);
    }
};

inline unsigned grid_for(size_t n, int threads = kT) { return static_cast<unsigned>((n + threads - 1) / threads); }

int bits_for(unsigned long long maxval) {
    int b = 1;
    while (b < 64 && (1ull << b) <= maxval) ++b;
    return b;
}

__device__ __forceinline__ double sqn_rn(double dx, double dy, double dz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// ------------------------------------------------------------------ uniform grid
struct Grid {
    double lox = 0, loy = 0, loz = 0, h = 1;
    int gx = 1, gy = 1, gz = 1;
    const int* start = nullptr;  // ncells + 1
    const int* pid = nullptr;    // n: point ids cell-major, ascending within a cell
    const double* sp = nullptr;  // n * 3: coordinates in pid order
};

__device__ __forceinline__ int cell_coord(double v, double lo, double h, int g) {
    return min(g - 1, max(0, static_cast<int>(__ddiv_rn(__dsub_rn(v, lo), h))));
}

__global__ void bbox_kernel(const double* __restrict__ pts, int n, double* __restrict__ out) {
    __shared__ double sh[6][kT];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int c = 0; c < 3; ++c) {
            lo[c] = fmin(lo[c], pts[3 * i + c]);
            hi[c] = fmax(hi[c], pts[3 * i + c]);
        }
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
    if (threadIdx.x < 6) out[6 * blockIdx.x + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void cell_key_kernel(const double* __restrict__ pts, int n, Grid g, unsigned* __restrict__ key,
                                int* __restrict__ idx, int* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int cx = cell_coord(pts[3 * i], g.lox, g.h, g.gx);
    const int cy = cell_coord(pts[3 * i + 1], g.loy, g.h, g.gy);
    const int cz = cell_coord(pts[3 * i + 2], g.loz, g.h, g.gz);
    const unsigned c = static_cast<unsigned>((cz * g.gy + cy) * g.gx + cx);
    key[i] = c;
    idx[i] = i;
    atomicAdd(count + c, 1);
}

__global__ void gather_coords_kernel(const double* __restrict__ pts, const int* __restrict__ pid, int n,
                                     double* __restrict__ sp) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = pid[t];
    sp[3 * t] = pts[3 * i];
    sp[3 * t + 1] = pts[3 * i + 1];
    sp[3 * t + 2] = pts[3 * i + 2];
}

// Device grid over `pts` (already on the device) with cell size h over the
// box [lo, lo + g*h): counting sort by cell, stable in point index.
struct DeviceGrid {
    Grid g;
    Dev<int> start, pid;
    Dev<double> sp;
    void build(const double* d_pts, int n, const double lo[3], double h, int gx, int gy, int gz, cudaStream_t s) {
        g.lox = lo[0];
        g.loy = lo[1];
        g.loz = lo[2];
        g.h = h;
        g.gx = gx;
        g.gy = gy;
        g.gz = gz;
        const size_t ncells = static_cast<size_t>(gx) * gy * gz;
        Dev<unsigned> key(n), key2(n);
        Dev<int> idx(n);
        start.resize(ncells + 1);
        pid.resize(n);
        sp.resize(3 * static_cast<size_t>(n));
        Dev<int> count(ncells + 1);
        NRR_CUDA_CHECK(cudaMemsetAsync(count.p, 0, (ncells + 1) * sizeof(int), s));
        cell_key_kernel<<<grid_for(n), kT, 0, s>>>(d_pts, n, g, key.p, idx.p, count.p);
        NRR_CUDA_CHECK(cudaGetLastError());
        size_t tmp = 0, tmp2 = 0;
        const int bits = bits_for(ncells);
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, idx.p, pid.p, n, 0, bits, s));
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, count.p, start.p, ncells + 1, s));
        Dev<unsigned char> scratch(std::max(tmp, tmp2));
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(scratch.p, tmp, key.p, key2.p, idx.p, pid.p, n, 0, bits, s));
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scratch.p, tmp2, count.p, start.p, ncells + 1, s));
        gather_coords_kernel<<<grid_for(n), kT, 0, s>>>(d_pts, pid.p, n, sp.p);
        NRR_CUDA_CHECK(cudaGetLastError());
        g.start = start.p;
        g.pid = pid.p;
        g.sp = sp.p;
    }
};

void device_bbox(const double* d_pts, int n, double lo[3], double hi[3], cudaStream_t s) {
    const int blocks = std::min<int>(148, static_cast<int>(grid_for(n)));
    Dev<double> part(6 * static_cast<size_t>(blocks));
    bbox_kernel<<<blocks, kT, 0, s>>>(d_pts, n, part.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    std::vector<double> h(6 * static_cast<size_t>(blocks));
    NRR_CUDA_CHECK(cudaMemcpyAsync(h.data(), part.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
    for (int c = 0; c < 3; ++c) {
        lo[c] = INFINITY;
        hi[c] = -INFINITY;
    }
    for (int b = 0; b < blocks; ++b)
        for (int c = 0; c < 3; ++c) {
            lo[c] = std::min(lo[c], h[6 * b + c]);
            hi[c] = std::max(hi[c], h[6 * b + 3 + c]);
        }
}

// sorted unique 64-bit keys (a << 32 | b) -> host pairs
std::vector<std::pair<int, int>> unique_pairs(unsigned long long* d_keys, size_t cnt, cudaStream_t s) {
    Dev<unsigned long long> sorted(cnt), uniq(cnt);
    Dev<int> nsel(1);
    size_t t1 = 0, t2 = 0;
    NRR_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, t1, d_keys, sorted.p, cnt, 0, 64, s));
    NRR_CUDA_CHECK(cub::DeviceSelect::Unique(nullptr, t2, sorted.p, uniq.p, nsel.p, cnt, s));
    Dev<unsigned char> scratch(std::max(t1, t2));
    NRR_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(scratch.p, t1, d_keys, sorted.p, cnt, 0, 64, s));
    NRR_CUDA_CHECK(cub::DeviceSelect::Unique(scratch.p, t2, sorted.p, uniq.p, nsel.p, cnt, s));
    int m = 0;
    NRR_CUDA_CHECK(cudaMemcpyAsync(&m, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<unsigned long long> h(m);
    NRR_CUDA_CHECK(cudaMemcpyAsync(h.data(), uniq.p, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<std::pair<int, int>> out(m);
    for (int t = 0; t < m; ++t) out[t] = {static_cast<int>(h[t] >> 32), static_cast<int>(h[t] & 0xffffffffu)};
    return out;
}

// ================================================================== kNN (f2)
template <int KMAX>
__global__ void __launch_bounds__(128) knn_kernel(Grid g, int n, int k, unsigned long long* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = g.pid[t];
    const double qx = g.sp[3 * t], qy = g.sp[3 * t + 1], qz = g.sp[3 * t + 2];
    const int cx = cell_coord(qx, g.lox, g.h, g.gx), cy = cell_coord(qy, g.loy, g.h, g.gy),
              cz = cell_coord(qz, g.loz, g.h, g.gz);
    double bd[KMAX];
    int bi[KMAX];
    int cnt = 0;
    const int maxs = max(g.gx, max(g.gy, g.gz));
    for (int s = 0; s <= maxs; ++s) {
        for (int dz = -s; dz <= s; ++dz) {
            const int z = cz + dz;
            if (z < 0 || z >= g.gz) continue;
            for (int dy = -s; dy <= s; ++dy) {
                const int y = cy + dy;
                if (y < 0 || y >= g.gy) continue;
                const bool shell_only = s > 0 && abs(dz) < s && abs(dy) < s;
                for (int dx = -s; dx <= s; dx += shell_only ? 2 * s : 1) {
                    const int x = cx + dx;
                    if (x < 0 || x >= g.gx) continue;
                    const int cell = (z * g.gy + y) * g.gx + x;
                    for (int u = g.start[cell]; u < g.start[cell + 1]; ++u) {
                        const int j = g.pid[u];
                        if (j == i) continue;
                        // (points[i] - points[j]).squaredNorm(), surface.hpp:82
                        const double d = sqn_rn(__dsub_rn(qx, g.sp[3 * u]), __dsub_rn(qy, g.sp[3 * u + 1]),
                                                __dsub_rn(qz, g.sp[3 * u + 2]));
                        int pos;
                        if (cnt < k) {
                            pos = cnt++;
                        } else if (d < bd[k - 1] || (d == bd[k - 1] && j < bi[k - 1])) {
                            pos = k - 1;
                        } else {
                            continue;
                        }
                        while (pos > 0 && (d < bd[pos - 1] || (d == bd[pos - 1] && j < bi[pos - 1]))) {
                            bd[pos] = bd[pos - 1];
                            bi[pos] = bi[pos - 1];
                            --pos;
                        }
                        bd[pos] = d;
                        bi[pos] = j;
                    }
                }
            }
        }
        if (cnt >= k) {  // every unvisited point lies outside the (2s+1)^3 box (setup.cpp grid_knn_edges)
            const double h = g.h;
            const double bx = fmin(__dsub_rn(qx, __dadd_rn(g.lox, __dmul_rn(static_cast<double>(cx - s), h))),
                                   __dsub_rn(__dadd_rn(g.lox, __dmul_rn(static_cast<double>(cx + s + 1), h)), qx));
            const double by = fmin(__dsub_rn(qy, __dadd_rn(g.loy, __dmul_rn(static_cast<double>(cy - s), h))),
                                   __dsub_rn(__dadd_rn(g.loy, __dmul_rn(static_cast<double>(cy + s + 1), h)), qy));
            const double bz = fmin(__dsub_rn(qz, __dadd_rn(g.loz, __dmul_rn(static_cast<double>(cz - s), h))),
                                   __dsub_rn(__dadd_rn(g.loz, __dmul_rn(static_cast<double>(cz + s + 1), h)), qz));
            const double bound = __dmul_rn(fmin(bx, fmin(by, bz)), 1.0 - 1e-12);
            if (bd[k - 1] < __dmul_rn(bound, bound)) break;
        }
    }
    for (int q = 0; q < k; ++q) {
        const unsigned a = static_cast<unsigned>(min(i, bi[q])), b = static_cast<unsigned>(max(i, bi[q]));
        out[static_cast<size_t>(i) * k + q] = (static_cast<unsigned long long>(a) << 32) | b;
    }
}

// ================================================================== graph (f1)
struct GraphArgs {
    int n = 0;
    double R = 0;
    const double* pts = nullptr;
    const int* adj_off = nullptr;  // n + 1
    const int* adj_nb = nullptr;   // sorted (neighbour, length) per vertex
    const double* adj_len = nullptr;
    const int* rank = nullptr;     // PCA rank of each point
    Grid g;                        // cell size >= R
};

// surface adjacency: per edge its length |p_u - p_v| (setup.cpp finalize), both directions
__global__ void adj_emit_kernel(const double* __restrict__ pts, int n, const int* __restrict__ edges, int ne,
                                unsigned long long* __restrict__ key, double* __restrict__ len,
                                int* __restrict__ deg, int* __restrict__ bad) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int u = edges[2 * e], v = edges[2 * e + 1];
    if (u < 0 || v < 0 || u >= n || v >= n || u == v) {
        atomicOr(bad, u == v ? 2 : 1);
        key[2 * e] = key[2 * e + 1] = 0;
        len[2 * e] = len[2 * e + 1] = 0;
        return;
    }
    const double l = sqrt(sqn_rn(__dsub_rn(pts[3 * u], pts[3 * v]), __dsub_rn(pts[3 * u + 1], pts[3 * v + 1]),
                                 __dsub_rn(pts[3 * u + 2], pts[3 * v + 2])));
    key[2 * e] = (static_cast<unsigned long long>(u) << 32) | static_cast<unsigned>(v);
    key[2 * e + 1] = (static_cast<unsigned long long>(v) << 32) | static_cast<unsigned>(u);
    len[2 * e] = len[2 * e + 1] = l;
    atomicAdd(deg + u, 1);
    atomicAdd(deg + v, 1);
}

__global__ void adj_split_kernel(const unsigned long long* __restrict__ key, int m, int* __restrict__ nb) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) nb[t] = static_cast<int>(key[t] & 0xffffffffu);
}

__global__ void project_kernel(const double* __restrict__ pts, int n, double ax, double ay, double az,
                               double* __restrict__ proj, int* __restrict__ idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double p = __dadd_rn(__dadd_rn(__dmul_rn(pts[3 * i], ax), __dmul_rn(pts[3 * i + 1], ay)),
                               __dmul_rn(pts[3 * i + 2], az));
    proj[i] = __dadd_rn(p, 0.0);  // -0.0 -> +0.0: the reference compares projections with ==, a radix sort with bits
    idx[i] = i;
}

__global__ void rank_kernel(const int* __restrict__ order, int n, int* __restrict__ rank) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) rank[order[t]] = t;
}

// state: 0 undecided; round * 4 + 1 node; round * 4 + 2 covered
__device__ __forceinline__ bool decided_before(int st, int round) { return st != 0 && (st >> 2) < round; }

// Round `round` over PCA positions [t0, t1): a point whose earlier Euclidean
// neighbours (|p - q| < R, the BFS test of limited_geodesic) are all decided
// before this round, and that no node's ball has marked, becomes a node.
__global__ void decide_kernel(GraphArgs a, const int* __restrict__ order, int t0, int t1, int round,
                              int* __restrict__ state, int* __restrict__ new_nodes, int* __restrict__ n_new,
                              int* __restrict__ new_count) {
    const int t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= t1) return;
    const int p = order[t];
    if (state[p] != 0) return;
    const double px = a.pts[3 * p], py = a.pts[3 * p + 1], pz = a.pts[3 * p + 2];
    const Grid& g = a.g;
    const int cx = cell_coord(px, g.lox, g.h, g.gx), cy = cell_coord(py, g.loy, g.h, g.gy),
              cz = cell_coord(pz, g.loz, g.h, g.gz);
    int cnt = 0;
    for (int z = max(0, cz - 1); z <= min(g.gz - 1, cz + 1); ++z)
        for (int y = max(0, cy - 1); y <= min(g.gy - 1, cy + 1); ++y)
            for (int x = max(0, cx - 1); x <= min(g.gx - 1, cx + 1); ++x) {
                const int cell = (z * g.gy + y) * g.gx + x;
                for (int u = g.start[cell]; u < g.start[cell + 1]; ++u) {
                    // |w - src| with src = q, w = p (geodesic.hpp:51)
                    const double d = sqrt(sqn_rn(__dsub_rn(px, g.sp[3 * u]), __dsub_rn(py, g.sp[3 * u + 1]),
                                                 __dsub_rn(pz, g.sp[3 * u + 2])));
                    if (!(d < a.R)) continue;
                    ++cnt;
                    const int q = g.pid[u];
                    if (a.rank[q] < t && !decided_before(state[q], round)) return;  // wait for q
                }
            }
    state[p] = round * 4 + 1;
    const int slot = atomicAdd(n_new, 1);
    new_nodes[slot] = p;
    new_count[slot] = cnt;  // its Euclidean candidates (ball_kernel's scratch size)
}

// One CTA per new node q: its limited geodesic ball (geodesic.hpp:22-84) into
// ball storage, and later members marked covered. `cand` is the node's
// scratch slice (capacity cap_k = next pow2 >= its Euclidean count).
constexpr int kBallThreads = 256;
__global__ void __launch_bounds__(kBallThreads) ball_kernel(GraphArgs a, const int* __restrict__ new_nodes,
                                                            const long long* __restrict__ cand_off,
                                                            int* __restrict__ cand, double* __restrict__ cdist,
                                                            int* __restrict__ cflag, int round,
                                                            int* __restrict__ state, int* __restrict__ ball_v,
                                                            double* __restrict__ ball_d, int* __restrict__ ball_off,
                                                            int* __restrict__ ball_len, int* __restrict__ pool_top,
                                                            int pool_cap, int* __restrict__ overflow) {
    const int q = new_nodes[blockIdx.x];
    const long long o0 = cand_off[blockIdx.x];
    const int cap = static_cast<int>(cand_off[blockIdx.x + 1] - o0);
    int* C = cand + o0;
    double* D = cdist + o0;
    int* F = cflag + o0;
    const double R = a.R;
    const double qx = a.pts[3 * q], qy = a.pts[3 * q + 1], qz = a.pts[3 * q + 2];
    const Grid& g = a.g;
    __shared__ int s_cnt, s_changed, s_out;
    __shared__ int s_scan[kBallThreads];
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    // 1. Euclidean candidates |w - q| < R
    const int cx = cell_coord(qx, g.lox, g.h, g.gx), cy = cell_coord(qy, g.loy, g.h, g.gy),
              cz = cell_coord(qz, g.loz, g.h, g.gz);
    for (int c27 = 0; c27 < 27; ++c27) {
        const int x = cx + c27 % 3 - 1, y = cy + (c27 / 3) % 3 - 1, z = cz + c27 / 9 - 1;
        if (x < 0 || y < 0 || z < 0 || x >= g.gx || y >= g.gy || z >= g.gz) continue;
        const int cell = (z * g.gy + y) * g.gx + x;
        for (int u = g.start[cell] + threadIdx.x; u < g.start[cell + 1]; u += blockDim.x) {
            const double d = sqrt(sqn_rn(__dsub_rn(g.sp[3 * u], qx), __dsub_rn(g.sp[3 * u + 1], qy),
                                         __dsub_rn(g.sp[3 * u + 2], qz)));
            if (d < R) {
                const int k = atomicAdd(&s_cnt, 1);
                if (k < cap) C[k] = g.pid[u];
            }
        }
    }
    __syncthreads();
    const int m = s_cnt;
    if (m > cap) {  // cannot happen: cap was counted with the same test
        if (threadIdx.x == 0) atomicOr(overflow, 1);
        return;
    }
    for (int k = m + threadIdx.x; k < cap; k += blockDim.x) C[k] = INT_MAX;
    __syncthreads();
    // 2. bitonic sort of the candidate ids (cap is a power of two)
    for (int size = 2; size <= cap; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int k = threadIdx.x; k < cap; k += blockDim.x) {
                const int l = k ^ stride;
                if (l > k) {
                    const bool up = (k & size) == 0;
                    const int x = C[k], y = C[l];
                    if ((x > y) == up) {
                        C[k] = y;
                        C[l] = x;
                    }
                }
            }
            __syncthreads();
        }
    auto find = [&](int v) {  // position of v among the m sorted candidates, -1 if absent
        int lo = 0, hi = m;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (C[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        return lo < m && C[lo] == v ? lo : -1;
    };
    // 3. BFS component through in-ball vertices (flag 1 = in the component)
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
        F[k] = C[k] == q ? 1 : 0;
        D[k] = C[k] == q ? 0.0 : INFINITY;
    }
    __syncthreads();
    do {
        __syncthreads();
        if (threadIdx.x == 0) s_changed = 0;
        __syncthreads();
        for (int k = threadIdx.x; k < m; k += blockDim.x) {
            if (F[k] != 1) continue;
            const int v = C[k];
            for (int e = a.adj_off[v]; e < a.adj_off[v + 1]; ++e) {
                const int w = find(a.adj_nb[e]);
                if (w >= 0 && atomicCAS(F + w, 0, 1) == 0) s_changed = 1;
            }
        }
        __syncthreads();
    } while (s_changed);
    // 4. edge-graph distances: relax from every component vertex below R to
    //    the fixed point (== the reference's Dijkstra, see the file comment)
    do {
        __syncthreads();
        if (threadIdx.x == 0) s_changed = 0;
        __syncthreads();
        for (int k = threadIdx.x; k < m; k += blockDim.x) {
            if (F[k] != 1) continue;
            const double dv = D[k];
            if (!(dv < R)) continue;
            const int v = C[k];
            for (int e = a.adj_off[v]; e < a.adj_off[v + 1]; ++e) {
                const int w = find(a.adj_nb[e]);
                if (w < 0 || F[w] != 1) continue;
                const double cand_d = __dadd_rn(dv, a.adj_len[e]);
                unsigned long long* addr = reinterpret_cast<unsigned long long*>(D + w);
                const unsigned long long nb = static_cast<unsigned long long>(__double_as_longlong(cand_d));
                if (nb < atomicMin(addr, nb)) s_changed = 1;
            }
        }
        __syncthreads();
    } while (s_changed);
    // 5. members (component, distance < R) in vertex order -> ball storage
    const int per = (m + blockDim.x - 1) / blockDim.x;
    const int k0 = threadIdx.x * per, k1 = min(m, k0 + per);
    int mine = 0;
    for (int k = k0; k < k1; ++k) mine += (F[k] == 1 && D[k] < R) ? 1 : 0;
    s_scan[threadIdx.x] = mine;
    __syncthreads();
    for (int off = 1; off < blockDim.x; off <<= 1) {
        const int v = threadIdx.x >= off ? s_scan[threadIdx.x - off] : 0;
        __syncthreads();
        s_scan[threadIdx.x] += v;
        __syncthreads();
    }
    if (threadIdx.x == blockDim.x - 1) {
        const int tot = s_scan[threadIdx.x];
        const int base = atomicAdd(pool_top, tot);
        s_out = base;
        if (base + tot > pool_cap) atomicOr(overflow, 2);
        ball_off[q] = base;
        ball_len[q] = tot;
    }
    __syncthreads();
    if (s_out + s_scan[blockDim.x - 1] > pool_cap) return;
    int w = s_out + s_scan[threadIdx.x] - mine;
    const int rq = a.rank[q];
    for (int k = k0; k < k1; ++k) {
        if (!(F[k] == 1 && D[k] < R)) continue;
        ball_v[w] = C[k];
        ball_d[w] = D[k];
        ++w;
        if (C[k] != q && a.rank[C[k]] > rq) atomicCAS(state + C[k], 0, round * 4 + 2);
    }
}

// ---- fast sweep: every round on the device, no host synchronisation ----
// Round control in device memory: the window [t0, t1) of PCA positions, the
// first undecided position fu, the round's new nodes and an error word.
struct RoundCtl {
    int t0, t1, fu, n_new, pool_top, err, round, pad;
};

// The 27 cells around (cx, cy, cz) as one flat index space: lanes 0..26 of
// the calling warp load their cell's point range, a warp scan gives each
// cell's offset; returns the number of candidate points. A flat index f then
// maps to point slot start[c] + f - pref[c] (cells_locate), so a warp or CTA
// walks every candidate with independent loads instead of 27 dependent
// cell loops.
__device__ __forceinline__ int cells_27(const Grid& g, int cx, int cy, int cz, int lane, int* s_start, int* s_pref) {
    int st = 0, cnt = 0;
    if (lane < 27) {
        const int x = cx + lane % 3 - 1, y = cy + (lane / 3) % 3 - 1, z = cz + lane / 9 - 1;
        if (x >= 0 && y >= 0 && z >= 0 && x < g.gx && y < g.gy && z < g.gz) {
            const int cell = (z * g.gy + y) * g.gx + x;
            st = g.start[cell];
            cnt = g.start[cell + 1] - st;
        }
    }
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    s_start[lane] = st;
    s_pref[lane] = inc - cnt;
    __syncwarp();
    return __shfl_sync(0xffffffffu, inc, 31);
}
__device__ __forceinline__ int cells_locate(int f, const int* s_start, const int* s_pref) {
    int lo = 0, hi = 26;  // last cell c with pref[c] <= f
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pref[mid] <= f) lo = mid;
        else hi = mid - 1;
    }
    return s_start[lo] + f - s_pref[lo];
}

// one warp: window [fu, upper_bound(proj, proj[fu] + 2R)) by a 32-ary search,
// and a fresh round
__global__ void window_kernel(RoundCtl* __restrict__ ctl, const double* __restrict__ proj, int n, double win) {
    const int lane = threadIdx.x;
    const int fu = ctl->fu;
    if (fu >= n) {
        if (lane == 0) {
            ctl->n_new = 0;
            ctl->t0 = ctl->t1 = fu;
        }
        return;
    }
    const double lim = proj[fu] + win;
    int lo = fu + 1, hi = n;  // the answer (first position with proj > lim) lies in [lo, hi]
    while (hi - lo > 32) {
        const long long span = hi - lo;
        const int probe = lo + static_cast<int>((span * (lane + 1)) / 33);  // increasing, in [lo, hi)
        const int cnt = __popc(__ballot_sync(0xffffffffu, proj[probe] <= lim));
        const int p_lo = __shfl_sync(0xffffffffu, probe, cnt > 0 ? cnt - 1 : 0);
        const int p_hi = __shfl_sync(0xffffffffu, probe, cnt < 32 ? cnt : 31);
        if (cnt > 0) lo = p_lo + 1;
        if (cnt < 32) hi = p_hi;
    }
    const int t = lo + lane;
    lo += __popc(__ballot_sync(0xffffffffu, t < hi && proj[t] <= lim));
    if (lane == 0) {
        ctl->n_new = 0;
        ctl->t0 = fu;
        ctl->t1 = lo;
        ++ctl->round;
    }
}

// decide_kernel with one warp per PCA position (lanes split the candidates)
__global__ void __launch_bounds__(kT) decide_warp_kernel(GraphArgs a, const int* __restrict__ order,
                                                         RoundCtl* __restrict__ ctl, int* __restrict__ state,
                                                         int* __restrict__ new_nodes) {
    __shared__ int s_start[kT / 32][32], s_pref[kT / 32][32];
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int t0 = ctl->t0, t1 = ctl->t1, round = ctl->round;
    const Grid& g = a.g;
    for (int t = t0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < t1; t += warps) {
        const int p = order[t];
        if (state[p] != 0) continue;
        const double px = a.pts[3 * p], py = a.pts[3 * p + 1], pz = a.pts[3 * p + 2];
        const int cx = cell_coord(px, g.lox, g.h, g.gx), cy = cell_coord(py, g.loy, g.h, g.gy),
                  cz = cell_coord(pz, g.loz, g.h, g.gz);
        const int wib = threadIdx.x >> 5;
        const int total = cells_27(g, cx, cy, cz, lane, s_start[wib], s_pref[wib]);
        bool blocked = false;
        for (int fb = 0; fb < total && !blocked; fb += 32) {
            const int f = fb + lane;
            bool mine = false;
            if (f < total) {
                const int u = cells_locate(f, s_start[wib], s_pref[wib]);
                const double d = sqrt(sqn_rn(__dsub_rn(px, g.sp[3 * u]), __dsub_rn(py, g.sp[3 * u + 1]),
                                             __dsub_rn(pz, g.sp[3 * u + 2])));
                if (d < a.R) {
                    const int q = g.pid[u];
                    mine = a.rank[q] < t && !decided_before(state[q], round);
                }
            }
            blocked = __any_sync(0xffffffffu, mine);
        }
        if (!blocked && lane == 0) {
            state[p] = round * 4 + 1;
            new_nodes[atomicAdd(&ctl->n_new, 1)] = p;
        }
    }
}

// Limited geodesic balls of the round's new nodes, one CTA per node (grid-
// strided over ctl->n_new), everything in shared memory: the Euclidean
// candidates with an open-addressing id -> slot map, their adjacency with
// local slots, and Bellman-Ford relaxation (from slots below R, into
// candidates only; the BFS component of the reference is implied: every
// relaxation chain from the source runs through in-ball vertices).
constexpr int kBallCap = 2048, kHashCap = 4096, kAdjCap = 8192;
constexpr size_t kBallSmem = kHashCap * 2 * sizeof(int) + kBallCap * (sizeof(int) + sizeof(double)) +
                             (kBallCap + 1) * sizeof(int) + kAdjCap * (sizeof(int) + sizeof(double));
__device__ __forceinline__ int hash_slot(int v) { return static_cast<int>((static_cast<unsigned>(v) * 2654435761u) >> 20); }

__global__ void __launch_bounds__(kBallThreads) ball_smem_kernel(GraphArgs a, const int* __restrict__ new_nodes,
                                                                 RoundCtl* __restrict__ ctl, int* __restrict__ state,
                                                                 int* __restrict__ ball_v, double* __restrict__ ball_d,
                                                                 int* __restrict__ ball_off, int* __restrict__ ball_len,
                                                                 int pool_cap) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* D = reinterpret_cast<double*>(smem);                          // kBallCap
    double* AL = D + kBallCap;                                            // kAdjCap
    int* hkey = reinterpret_cast<int*>(AL + kAdjCap);                     // kHashCap
    int* hval = hkey + kHashCap;                                          // kHashCap
    int* C = hval + kHashCap;                                             // kBallCap
    int* AO = C + kBallCap;                                               // kBallCap + 1
    int* AN = AO + kBallCap + 1;                                          // kAdjCap
    __shared__ int s_cnt, s_changed, s_out, s_adj, s_total;
    __shared__ int s_scan[kBallThreads];
    __shared__ int s_cstart[32], s_cpref[32];
    const int n_new = ctl->n_new, round = ctl->round;
    const double R = a.R;
    const Grid& g = a.g;
    for (int j = blockIdx.x; j < n_new; j += gridDim.x) {
        const int q = new_nodes[j];
        const double qx = a.pts[3 * q], qy = a.pts[3 * q + 1], qz = a.pts[3 * q + 2];
        for (int k = threadIdx.x; k < kHashCap; k += blockDim.x) hkey[k] = -1;
        if (threadIdx.x == 0) s_cnt = 0;
        const int cx = cell_coord(qx, g.lox, g.h, g.gx), cy = cell_coord(qy, g.loy, g.h, g.gy),
                  cz = cell_coord(qz, g.loz, g.h, g.gz);
        if (threadIdx.x < 32) s_total = cells_27(g, cx, cy, cz, threadIdx.x, s_cstart, s_cpref);
        __syncthreads();
        const int total = s_total;
        for (int f = threadIdx.x; f < total; f += blockDim.x) {
            const int u = cells_locate(f, s_cstart, s_cpref);
            const double d = sqrt(sqn_rn(__dsub_rn(g.sp[3 * u], qx), __dsub_rn(g.sp[3 * u + 1], qy),
                                         __dsub_rn(g.sp[3 * u + 2], qz)));
            if (!(d < R)) continue;
            const int k = atomicAdd(&s_cnt, 1);
            if (k >= kBallCap) continue;
            const int v = g.pid[u];
            C[k] = v;
            int h = hash_slot(v) & (kHashCap - 1);
            while (atomicCAS(hkey + h, -1, v) != -1) h = (h + 1) & (kHashCap - 1);
            hval[h] = k;
        }
        __syncthreads();
        const int m = s_cnt;
        if (m > kBallCap) {  // the host reruns the build on the global-memory path
            if (threadIdx.x == 0) atomicOr(&ctl->err, 1);
            __syncthreads();
            continue;
        }
        auto find = [&](int v) {
            int h = hash_slot(v) & (kHashCap - 1);
            while (true) {
                const int key = hkey[h];
                if (key == v) return hval[h];
                if (key == -1) return -1;
                h = (h + 1) & (kHashCap - 1);
            }
        };
        // local adjacency: degree prefix over the candidates (contiguous chunks per thread)
        const int per = (m + blockDim.x - 1) / blockDim.x;
        const int k0 = min(m, threadIdx.x * per), k1 = min(m, k0 + per);
        int mine = 0;
        for (int k = k0; k < k1; ++k) mine += a.adj_off[C[k] + 1] - a.adj_off[C[k]];
        s_scan[threadIdx.x] = mine;
        __syncthreads();
        for (int off = 1; off < blockDim.x; off <<= 1) {
            const int v = threadIdx.x >= off ? s_scan[threadIdx.x - off] : 0;
            __syncthreads();
            s_scan[threadIdx.x] += v;
            __syncthreads();
        }
        if (threadIdx.x == blockDim.x - 1) s_adj = s_scan[threadIdx.x];
        {
            int o = s_scan[threadIdx.x] - mine;
            for (int k = k0; k < k1; ++k) {
                AO[k] = o;
                o += a.adj_off[C[k] + 1] - a.adj_off[C[k]];
            }
            if (k1 == m && k0 < k1) AO[m] = o;
            if (m == 0 && threadIdx.x == 0) AO[0] = 0;
        }
        __syncthreads();
        if (s_adj > kAdjCap) {
            if (threadIdx.x == 0) atomicOr(&ctl->err, 2);
            __syncthreads();
            continue;
        }
        for (int k = threadIdx.x; k < m; k += blockDim.x) {
            const int v = C[k];
            int o = AO[k];
            for (int e = a.adj_off[v]; e < a.adj_off[v + 1]; ++e, ++o) {
                AN[o] = find(a.adj_nb[e]);
                AL[o] = a.adj_len[e];
            }
            D[k] = v == q ? 0.0 : INFINITY;
        }
        __syncthreads();
        // Bellman-Ford to the fixed point (bitwise the reference's Dijkstra)
        do {
            __syncthreads();
            if (threadIdx.x == 0) s_changed = 0;
            __syncthreads();
            for (int k = threadIdx.x; k < m; k += blockDim.x) {
                const double dv = D[k];
                if (!(dv < R)) continue;
                for (int o = AO[k]; o < AO[k + 1]; ++o) {
                    const int w = AN[o];
                    if (w < 0) continue;
                    const double cd = __dadd_rn(dv, AL[o]);
                    if (cd < D[w]) {
                        unsigned long long* addr = reinterpret_cast<unsigned long long*>(D + w);
                        const unsigned long long nb = static_cast<unsigned long long>(__double_as_longlong(cd));
                        if (nb < atomicMin(addr, nb)) s_changed = 1;
                    }
                }
            }
            __syncthreads();
        } while (s_changed);
        // members (distance < R) -> ball storage (any order: the raw lists are sorted later)
        mine = 0;
        for (int k = k0; k < k1; ++k) mine += D[k] < R ? 1 : 0;
        s_scan[threadIdx.x] = mine;
        __syncthreads();
        for (int off = 1; off < blockDim.x; off <<= 1) {
            const int v = threadIdx.x >= off ? s_scan[threadIdx.x - off] : 0;
            __syncthreads();
            s_scan[threadIdx.x] += v;
            __syncthreads();
        }
        if (threadIdx.x == blockDim.x - 1) {
            const int tot = s_scan[threadIdx.x];
            s_out = atomicAdd(&ctl->pool_top, tot);
            if (s_out + tot > pool_cap) atomicOr(&ctl->err, 4);
            ball_off[q] = s_out;
            ball_len[q] = tot;
        }
        __syncthreads();
        if (s_out + s_scan[blockDim.x - 1] <= pool_cap) {
            int w = s_out + s_scan[threadIdx.x] - mine;
            const int rq = a.rank[q];
            for (int k = k0; k < k1; ++k) {
                if (!(D[k] < R)) continue;
                ball_v[w] = C[k];
                ball_d[w] = D[k];
                ++w;
                if (C[k] != q && a.rank[C[k]] > rq) atomicCAS(state + C[k], 0, round * 4 + 2);
            }
        }
        __syncthreads();
    }
}

// next fu: the first undecided position of the window, else the window's end
__global__ void next_fu_kernel(const int* __restrict__ order, const int* __restrict__ state,
                               RoundCtl* __restrict__ ctl, int* __restrict__ first) {
    const int t0 = ctl->t0, t1 = ctl->t1;
    for (int t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < t1; t += gridDim.x * blockDim.x)
        if (state[order[t]] == 0) atomicMin(first, t);
}
__global__ void commit_fu_kernel(RoundCtl* __restrict__ ctl, int* __restrict__ first, int n) {
    const int f = *first;
    ctl->fu = f < n ? f : ctl->t1;
    *first = n;
}

// first undecided PCA position in [t0, t1)
__global__ void first_undecided_kernel(const int* __restrict__ order, const int* __restrict__ state, int t0, int t1,
                                       int* __restrict__ first) {
    const int t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (t < t1 && state[order[t]] == 0) atomicMin(first, t);
}

__global__ void node_flag_kernel(const int* __restrict__ order, const int* __restrict__ state, int n,
                                 int* __restrict__ flag) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) flag[t] = (state[order[t]] & 3) == 1 ? 1 : 0;
}

__global__ void node_ids_kernel(const int* __restrict__ order, const int* __restrict__ flag,
                                const int* __restrict__ scan, int n, int* __restrict__ node_of,
                                int* __restrict__ node_indices) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n || !flag[t]) return;
    node_of[order[t]] = scan[t];
    node_indices[scan[t]] = order[t];
}

// raw influence entries: (vertex << 32 | node id) -> distance
__global__ void raw_emit_kernel(const int* __restrict__ node_indices, int N, const int* __restrict__ ball_off,
                                const int* __restrict__ ball_len, const int* __restrict__ ball_v,
                                const double* __restrict__ ball_d, const int* __restrict__ out_off,
                                unsigned long long* __restrict__ key, double* __restrict__ val,
                                int* __restrict__ kcount) {
    const int j = blockIdx.x;
    if (j >= N) return;
    const int q = node_indices[j];
    const int b0 = ball_off[q], len = ball_len[q], o0 = out_off[j];
    for (int t = threadIdx.x; t < len; t += blockDim.x) {
        const int v = ball_v[b0 + t];
        key[o0 + t] = (static_cast<unsigned long long>(v) << 32) | static_cast<unsigned>(j);
        val[o0 + t] = ball_d[b0 + t];
        atomicAdd(kcount + v, 1);
    }
}

// per vertex: its node ids / distances, weights (1 - D^2/R^2)^3 normalised
// (influence_weights, deformation_graph.hpp:111-125), pair counts for edges
__global__ void influence_kernel(const unsigned long long* __restrict__ key, const double* __restrict__ dist,
                                 const int* __restrict__ off, int n, double R, int* __restrict__ node,
                                 double* __restrict__ w, long long* __restrict__ npairs, int* __restrict__ bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int k0 = off[i], k1 = off[i + 1];
    if (k0 == k1) atomicOr(bad, 1);
    const double R2 = __dmul_rn(R, R);
    double total = 0.0;
    for (int k = k0; k < k1; ++k) {
        node[k] = static_cast<int>(key[k] & 0xffffffffu);
        const double d = dist[k];
        const double ratio = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(d, d), R2));
        if (!(ratio > 0.0)) atomicOr(bad, 2);
        const double wk = __dmul_rn(__dmul_rn(ratio, ratio), ratio);
        w[k] = wk;
        total = __dadd_rn(total, wk);
    }
    for (int k = k0; k < k1; ++k) w[k] = __ddiv_rn(w[k], total);
    const long long kk = k1 - k0;
    npairs[i] = kk * (kk - 1) / 2;
}

__global__ void edge_emit_kernel(const int* __restrict__ node, const int* __restrict__ off,
                                 const long long* __restrict__ pair_off, int n, unsigned long long* __restrict__ key) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long o = pair_off[i];
    for (int a = off[i]; a < off[i + 1]; ++a)
        for (int b = a + 1; b < off[i + 1]; ++b)
            key[o++] = (static_cast<unsigned long long>(node[a]) << 32) | static_cast<unsigned>(node[b]);
}

__global__ void pair_emit_kernel(const unsigned long long* __restrict__ edges, int E, unsigned long long* __restrict__ key) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const unsigned long long k = edges[e];
    key[2 * e] = k;
    key[2 * e + 1] = (k << 32) | (k >> 32);
}

// reg_weight_table (deformation_graph.hpp:130-148): 1/|p_i - p_j| per
// directed pair in (i, sorted j) order; the host sums them sequentially
__global__ void reg_inv_kernel(const unsigned long long* __restrict__ pairs, int P,
                               const double* __restrict__ node_pos, double* __restrict__ inv, int* __restrict__ bad) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P) return;
    const unsigned long long k = pairs[t];
    const int i = static_cast<int>(k >> 32), j = static_cast<int>(k & 0xffffffffu);
    const double len = sqrt(sqn_rn(__dsub_rn(node_pos[3 * i], node_pos[3 * j]),
                                   __dsub_rn(node_pos[3 * i + 1], node_pos[3 * j + 1]),
                                   __dsub_rn(node_pos[3 * i + 2], node_pos[3 * j + 2])));
    if (!(len > 0.0)) atomicOr(bad, 4);
    inv[t] = __ddiv_rn(1.0, len);
}

__global__ void node_pos_kernel(const double* __restrict__ pts, const int* __restrict__ node_indices, int N,
                                double* __restrict__ pos) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const int q = node_indices[j];
    pos[3 * j] = pts[3 * q];
    pos[3 * j + 1] = pts[3 * q + 1];
    pos[3 * j + 2] = pts[3 * q + 2];
}

template <typename T>
std::vector<T> download(const T* d, size_t n, cudaStream_t s) {
    std::vector<T> h(n);
    if (n) NRR_CUDA_CHECK(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
    return h;
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        NRR_CUDA_CHECK(cudaGetDevice(&prev));
        NRR_CUDA_CHECK(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

// -------------------------------------------------------------------- kNN
std::vector<std::pair<int, int>> knn_edges_gpu(int device, const double* pts, int n, int k) {
    if (k < 1) throw ConfigError("knn_edges: k must be >= 1");
    if (k >= n) throw ConfigError("knn_edges: k must be smaller than the point count");
    if (k > kKnnMaxK) throw ConfigError("knn_edges (device): k > " + std::to_string(kKnnMaxK));
    DeviceGuard dg(device);
    Stream st;
    const cudaStream_t s = st.s;
    Dev<double> d_pts(3 * static_cast<size_t>(n));
    NRR_CUDA_CHECK(cudaMemcpyAsync(d_pts.p, pts, 3 * sizeof(double) * n, cudaMemcpyHostToDevice, s));
    double lo[3], hi[3];
    device_bbox(d_pts.p, n, lo, hi, s);
    // cell size rule of the host grid (setup.cpp grid_knn_edges)
    const double ex = hi[0] - lo[0], ey = hi[1] - lo[1], ez = hi[2] - lo[2];
    const double vol = std::max(ex, 1e-12) * std::max(ey, 1e-12) * std::max(ez, 1e-12);
    double h = std::cbrt(vol * 2.0 / n);
    h = std::max(h, std::max(ex, std::max(ey, ez)) / 512.0);
    if (!(h > 0)) h = 1.0;
    const int gx = std::max(1, static_cast<int>(ex / h) + 1);
    const int gy = std::max(1, static_cast<int>(ey / h) + 1);
    const int gz = std::max(1, static_cast<int>(ez / h) + 1);
    DeviceGrid grid;
    grid.build(d_pts.p, n, lo, h, gx, gy, gz, s);
    Dev<unsigned long long> keys(static_cast<size_t>(n) * k);
    const unsigned blocks = grid_for(n, 128);
    if (k <= 8) knn_kernel<8><<<blocks, 128, 0, s>>>(grid.g, n, k, keys.p);
    else if (k <= 16) knn_kernel<16><<<blocks, 128, 0, s>>>(grid.g, n, k, keys.p);
    else knn_kernel<kKnnMaxK><<<blocks, 128, 0, s>>>(grid.g, n, k, keys.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    return unique_pairs(keys.p, static_cast<size_t>(n) * k, s);
}

// -------------------------------------------------------------------- graph
GraphData build_graph_gpu(int device, const double* pts, int n, const int32_t* sedges, int ne, double radius,
                          GraphBuildStats* stats) {
    if (n == 0) throw ConfigError("build_graph: empty source surface");
    if (!(radius > 0.0)) throw ConfigError("build_graph: radius must be positive");
    const bool prof = std::getenv("NRR_SETUP_PROF") != nullptr;
    const auto tp0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what, cudaStream_t ss) {
        if (!prof) return;
        cudaStreamSynchronize(ss);
        std::fprintf(stderr, "build_graph_gpu %-10s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count());
    };
    DeviceGuard dg(device);
    Stream st;
    const cudaStream_t s = st.s;
    Dev<double> d_pts(3 * static_cast<size_t>(n));
    NRR_CUDA_CHECK(cudaMemcpyAsync(d_pts.p, pts, 3 * sizeof(double) * n, cudaMemcpyHostToDevice, s));

    // PCA moments: two sequential sums over the points (pca_order), the one
    // part of the build with a serial dependence chain. A host thread runs
    // them (~1 ns per point and chain, vs ~40 ns on one GPU thread) while the
    // device builds the adjacency and the grid; same code as setup.cpp.
    double cov[9];
    std::thread moments([&] { pca_moments(pts, n, cov); });
    struct Join {
        std::thread& t;
        ~Join() {
            if (t.joinable()) t.join();
        }
    } join_moments{moments};

    // adjacency (Surface::finalize_edges order: neighbours ascending)
    Dev<int> d_bad(1);
    NRR_CUDA_CHECK(cudaMemsetAsync(d_bad.p, 0, sizeof(int), s));
    Dev<int> adj_off(n + 1), adj_nb(2 * static_cast<size_t>(ne)), deg(n + 1);
    Dev<double> adj_len(2 * static_cast<size_t>(ne));
    NRR_CUDA_CHECK(cudaMemsetAsync(deg.p, 0, (n + 1) * sizeof(int), s));
    if (ne > 0) {
        Dev<int> d_edges(2 * static_cast<size_t>(ne));
        NRR_CUDA_CHECK(cudaMemcpyAsync(d_edges.p, sedges, 2 * sizeof(int) * ne, cudaMemcpyHostToDevice, s));
        Dev<unsigned long long> key(2 * static_cast<size_t>(ne)), key2(2 * static_cast<size_t>(ne));
        Dev<double> len(2 * static_cast<size_t>(ne));
        adj_emit_kernel<<<grid_for(ne), kT, 0, s>>>(d_pts.p, n, d_edges.p, ne, key.p, len.p, deg.p, d_bad.p);
        NRR_CUDA_CHECK(cudaGetLastError());
        size_t tmp = 0;
        const int bits = 32 + bits_for(static_cast<unsigned long long>(n));
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, len.p, adj_len.p, 2 * ne, 0, bits, s));
        Dev<unsigned char> scratch(tmp);
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(scratch.p, tmp, key.p, key2.p, len.p, adj_len.p, 2 * ne, 0, bits, s));
        adj_split_kernel<<<grid_for(2 * ne), kT, 0, s>>>(key2.p, 2 * ne, adj_nb.p);
        NRR_CUDA_CHECK(cudaGetLastError());
    }
    {
        size_t tmp = 0;
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg.p, adj_off.p, n + 1, s));
        Dev<unsigned char> scratch(tmp);
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, deg.p, adj_off.p, n + 1, s));
    }
    int bad = 0;
    NRR_CUDA_CHECK(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));

    // Euclidean grid with cells >= R (capped at 256 cells per axis)
    double lo[3], hi[3];
    device_bbox(d_pts.p, n, lo, hi, s);  // synchronises s (bad is valid)
    if (bad & 1) throw NumericalError("surface edge index out of range");
    if (bad & 2) throw NumericalError("surface edge is a self-loop");
    const double maxe = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
    const double h = std::max(radius, maxe / 256.0) * (1.0 + 1e-12);
    int gdim[3];
    for (int c = 0; c < 3; ++c) gdim[c] = std::max(1, static_cast<int>((hi[c] - lo[c]) / h) + 1);
    DeviceGrid grid;
    grid.build(d_pts.p, n, lo, h, gdim[0], gdim[1], gdim[2], s);

    // PCA order (pca_order, deformation_graph.hpp:73-106)
    moments.join();
    double axis[3];
    pca_axis(cov, axis);  // the host's 3x3 Jacobi (setup.cpp), microseconds
    Dev<double> proj(n), proj2(n);
    Dev<int> idx(n), order(n), rank(n);
    project_kernel<<<grid_for(n), kT, 0, s>>>(d_pts.p, n, axis[0], axis[1], axis[2], proj.p, idx.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    {
        size_t tmp = 0;
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, proj.p, proj2.p, idx.p, order.p, n, 0, 64, s));
        Dev<unsigned char> scratch(tmp);
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(scratch.p, tmp, proj.p, proj2.p, idx.p, order.p, n, 0, 64, s));
    }
    rank_kernel<<<grid_for(n), kT, 0, s>>>(order.p, n, rank.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    const std::vector<double> hproj = download(proj2.p, n, s);

    // the sweep as rounds of the lexicographically first maximal independent set
    GraphArgs ga;
    ga.n = n;
    ga.R = radius;
    ga.pts = d_pts.p;
    ga.adj_off = adj_off.p;
    ga.adj_nb = adj_nb.p;
    ga.adj_len = adj_len.p;
    ga.rank = rank.p;
    ga.g = grid.g;
    const double win = 2.0 * radius;
    Dev<int> state(n), new_count(n), new_nodes(n), ball_off(n), ball_len(n);
    NRR_CUDA_CHECK(cudaMemsetAsync(state.p, 0, n * sizeof(int), s));
    int pool_cap = std::max(1 << 20, 4 * n);
    Dev<int> ball_v(pool_cap);
    Dev<double> ball_d(pool_cap);
    Dev<int> ctr(4);  // 0: new nodes, 1: pool top, 2: overflow, 3: first undecided
    NRR_CUDA_CHECK(cudaMemsetAsync(ctr.p, 0, 4 * sizeof(int), s));
    int* h_ctr = nullptr;
    NRR_CUDA_CHECK(cudaMallocHost(&h_ctr, 4 * sizeof(int)));
    struct HostFree {
        int* p;
        ~HostFree() { cudaFreeHost(p); }
    } hf{h_ctr};
    Dev<long long> cand_off(n + 1);
    Dev<int> cand, cflag;
    Dev<double> cdist;
    std::vector<int> h_cnt;
    std::vector<long long> h_off;
    long long pool_used = 0;  // upper bound of the entries written so far
    mark("prepared", s);
    // fast path: all rounds on the device, batches of rounds between host checks
    int rounds = 0;
    bool fast_ok = false;
    if (!std::getenv("NRR_GRAPH_SLOW_SWEEP")) {
        allow_max_smem(reinterpret_cast<const void*>(ball_smem_kernel));
        int sms = 148, dev = 0;
        NRR_CUDA_CHECK(cudaGetDevice(&dev));
        NRR_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        Dev<RoundCtl> ctl(1);
        Dev<int> first(1);
        RoundCtl init{};
        const int nn_init = n;
        NRR_CUDA_CHECK(cudaMemcpyAsync(ctl.p, &init, sizeof init, cudaMemcpyHostToDevice, s));
        NRR_CUDA_CHECK(cudaMemcpyAsync(first.p, &nn_init, sizeof(int), cudaMemcpyHostToDevice, s));
        RoundCtl* h_ctl = nullptr;
        NRR_CUDA_CHECK(cudaMallocHost(&h_ctl, sizeof(RoundCtl)));
        struct PinFree {
            RoundCtl* p;
            ~PinFree() { cudaFreeHost(p); }
        } pf{h_ctl};
        const int batch = 32;
        while (true) {
            for (int r = 0; r < batch; ++r) {
                window_kernel<<<1, 32, 0, s>>>(ctl.p, proj2.p, n, win);
                decide_warp_kernel<<<8 * sms, kT, 0, s>>>(ga, order.p, ctl.p, state.p, new_nodes.p);
                ball_smem_kernel<<<sms, kBallThreads, kBallSmem, s>>>(ga, new_nodes.p, ctl.p, state.p, ball_v.p,
                                                                      ball_d.p, ball_off.p, ball_len.p, pool_cap);
                next_fu_kernel<<<2 * sms, kT, 0, s>>>(order.p, state.p, ctl.p, first.p);
                commit_fu_kernel<<<1, 1, 0, s>>>(ctl.p, first.p, n);
            }
            NRR_CUDA_CHECK(cudaGetLastError());
            NRR_CUDA_CHECK(cudaMemcpyAsync(h_ctl, ctl.p, sizeof(RoundCtl), cudaMemcpyDeviceToHost, s));
            NRR_CUDA_CHECK(cudaStreamSynchronize(s));
            if (h_ctl->err) break;
            if (h_ctl->fu >= n) {
                fast_ok = true;
                rounds = h_ctl->round;
                break;
            }
        }
        if (!fast_ok) {  // a ball exceeded the shared-memory path: redo on the global-memory path
            NRR_CUDA_CHECK(cudaMemsetAsync(state.p, 0, n * sizeof(int), s));
            const long long need = static_cast<long long>(h_ctl->pool_top) * 2 + 4ll * n;
            if (need > pool_cap && need < INT_MAX) {
                pool_cap = static_cast<int>(need);
                ball_v.resize(pool_cap);
                ball_d.resize(pool_cap);
            }
        }
    }
    int fu = fast_ok ? n : 0;
    while (fu < n) {
        ++rounds;
        const double lim = hproj[fu] + win;
        const int t1 = std::max(fu + 1, static_cast<int>(std::upper_bound(hproj.begin() + fu, hproj.end(), lim) -
                                                         hproj.begin()));
        NRR_CUDA_CHECK(cudaMemsetAsync(ctr.p, 0, sizeof(int), s));
        decide_kernel<<<grid_for(t1 - fu), kT, 0, s>>>(ga, order.p, fu, t1, rounds, state.p, new_nodes.p, ctr.p,
                                                       new_count.p);
        NRR_CUDA_CHECK(cudaGetLastError());
        NRR_CUDA_CHECK(cudaMemcpyAsync(h_ctr, ctr.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        NRR_CUDA_CHECK(cudaStreamSynchronize(s));
        const int nn = h_ctr[0];
        if (nn > 0) {
            h_cnt.resize(nn);
            NRR_CUDA_CHECK(cudaMemcpyAsync(h_cnt.data(), new_count.p, nn * sizeof(int), cudaMemcpyDeviceToHost, s));
            NRR_CUDA_CHECK(cudaStreamSynchronize(s));
            // candidate slices: next power of two of each node's Euclidean count
            h_off.assign(nn + 1, 0);
            long long members = 0;
            for (int q = 0; q < nn; ++q) {
                long long c = 1;
                while (c < h_cnt[q]) c <<= 1;
                h_off[q + 1] = h_off[q] + c;
                members += h_cnt[q];
            }
            if (pool_used + members > pool_cap) {  // grow the ball pool before the round writes it
                const long long ncap = std::max<long long>(2ll * pool_cap, pool_used + members + 4ll * n);
                if (ncap > INT_MAX) throw CudaError("build_graph_gpu: ball pool exceeds 2^31 entries");
                Dev<int> v2(ncap);
                Dev<double> d2(ncap);
                NRR_CUDA_CHECK(cudaMemcpyAsync(v2.p, ball_v.p, pool_used * sizeof(int), cudaMemcpyDeviceToDevice, s));
                NRR_CUDA_CHECK(cudaMemcpyAsync(d2.p, ball_d.p, pool_used * sizeof(double), cudaMemcpyDeviceToDevice, s));
                NRR_CUDA_CHECK(cudaStreamSynchronize(s));
                std::swap(ball_v.p, v2.p);
                std::swap(ball_v.n, v2.n);
                std::swap(ball_d.p, d2.p);
                std::swap(ball_d.n, d2.n);
                pool_cap = static_cast<int>(ncap);
            }
            pool_used += members;
            cand.resize(h_off[nn]);
            cflag.resize(h_off[nn]);
            cdist.resize(h_off[nn]);
            NRR_CUDA_CHECK(cudaMemcpyAsync(cand_off.p, h_off.data(), (nn + 1) * sizeof(long long),
                                           cudaMemcpyHostToDevice, s));
            ball_kernel<<<nn, kBallThreads, 0, s>>>(ga, new_nodes.p, cand_off.p, cand.p, cdist.p, cflag.p, rounds,
                                                    state.p, ball_v.p, ball_d.p, ball_off.p, ball_len.p, ctr.p + 1,
                                                    pool_cap, ctr.p + 2);
            NRR_CUDA_CHECK(cudaGetLastError());
        }
        // next first undecided position
        int first = n;
        for (int a0 = fu; a0 < n && first == n;) {
            const int a1 = std::min(n, a0 + std::max(t1 - fu, 4096));
            h_ctr[3] = n;
            NRR_CUDA_CHECK(cudaMemcpyAsync(ctr.p + 3, h_ctr + 3, sizeof(int), cudaMemcpyHostToDevice, s));
            first_undecided_kernel<<<grid_for(a1 - a0), kT, 0, s>>>(order.p, state.p, a0, a1, ctr.p + 3);
            NRR_CUDA_CHECK(cudaGetLastError());
            NRR_CUDA_CHECK(cudaMemcpyAsync(h_ctr, ctr.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
            NRR_CUDA_CHECK(cudaStreamSynchronize(s));
            if (h_ctr[2]) throw CudaError("build_graph_gpu: ball storage overflow");
            first = h_ctr[3];
            a0 = a1;
        }
        fu = first;
    }

    mark(fast_ok ? "sweep" : "slow sweep", s);
    // node ids in PCA order
    Dev<int> flag(n), scan(n), node_of(n), node_indices(n);
    node_flag_kernel<<<grid_for(n), kT, 0, s>>>(order.p, state.p, n, flag.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    {
        size_t tmp = 0;
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag.p, scan.p, n, s));
        Dev<unsigned char> scratch(tmp);
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, flag.p, scan.p, n, s));
    }
    node_ids_kernel<<<grid_for(n), kT, 0, s>>>(order.p, flag.p, scan.p, n, node_of.p, node_indices.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    const std::vector<int> hflag = download(flag.p, n, s);
    int N = 0;
    for (int f : hflag) N += f;
    GraphData out;
    out.node_indices = download(node_indices.p, N, s);
    // ball sizes per node -> raw entry offsets (node order)
    const std::vector<int> hlen = download(ball_len.p, n, s);
    std::vector<int> roff(N + 1, 0);
    for (int j = 0; j < N; ++j) roff[j + 1] = roff[j] + hlen[out.node_indices[j]];
    const int S = roff[N];
    Dev<int> d_roff(N + 1), kcount(n + 1), infl_off(n + 1);
    NRR_CUDA_CHECK(cudaMemcpyAsync(d_roff.p, roff.data(), (N + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
    NRR_CUDA_CHECK(cudaMemsetAsync(kcount.p, 0, (n + 1) * sizeof(int), s));
    Dev<unsigned long long> rkey(S), rkey2(S);
    Dev<double> rval(S), rval2(S);
    raw_emit_kernel<<<N, 128, 0, s>>>(node_indices.p, N, ball_off.p, ball_len.p, ball_v.p, ball_d.p, d_roff.p,
                                       rkey.p, rval.p, kcount.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    {
        size_t t1 = 0, t2 = 0;
        const int bits = 32 + bits_for(static_cast<unsigned long long>(n));
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, t1, rkey.p, rkey2.p, rval.p, rval2.p, S, 0, bits, s));
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, t2, kcount.p, infl_off.p, n + 1, s));
        Dev<unsigned char> scratch(std::max(t1, t2));
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(scratch.p, t1, rkey.p, rkey2.p, rval.p, rval2.p, S, 0, bits, s));
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scratch.p, t2, kcount.p, infl_off.p, n + 1, s));
    }
    Dev<int> inode(S);
    Dev<double> iw(S);
    Dev<long long> npairs(n + 1), pair_off(n + 1);
    NRR_CUDA_CHECK(cudaMemsetAsync(d_bad.p, 0, sizeof(int), s));
    NRR_CUDA_CHECK(cudaMemsetAsync(npairs.p + n, 0, sizeof(long long), s));
    influence_kernel<<<grid_for(n), kT, 0, s>>>(rkey2.p, rval2.p, infl_off.p, n, radius, inode.p, iw.p, npairs.p,
                                                d_bad.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    {
        size_t tmp = 0;
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, npairs.p, pair_off.p, n + 1, s));
        Dev<unsigned char> scratch(tmp);
        NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, npairs.p, pair_off.p, n + 1, s));
    }
    long long npair_total = 0;
    NRR_CUDA_CHECK(cudaMemcpyAsync(&npair_total, pair_off.p + n, sizeof(long long), cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
    if (bad & 1) throw NumericalError("build_graph: point left without influencing nodes");
    if (bad & 2) throw NumericalError("influence_weights: distance not below radius");
    std::vector<std::pair<int, int>> edges;
    if (npair_total > 0) {
        Dev<unsigned long long> ekey(npair_total);
        edge_emit_kernel<<<grid_for(n), kT, 0, s>>>(inode.p, infl_off.p, pair_off.p, n, ekey.p);
        NRR_CUDA_CHECK(cudaGetLastError());
        edges = unique_pairs(ekey.p, npair_total, s);
    }
    const int E = static_cast<int>(edges.size());
    out.edges = edges;
    out.infl_off = download(infl_off.p, n + 1, s);
    out.infl_node = download(inode.p, S, s);
    out.infl_w = download(iw.p, S, s);
    out.infl_d = download(rval2.p, S, s);
    Dev<double> npos(3 * static_cast<size_t>(std::max(N, 1)));
    node_pos_kernel<<<grid_for(N), kT, 0, s>>>(d_pts.p, node_indices.p, N, npos.p);
    NRR_CUDA_CHECK(cudaGetLastError());
    out.node_positions = download(npos.p, 3 * static_cast<size_t>(N), s);
    if (E > 0) {
        std::vector<unsigned long long> hk(E);
        for (int e = 0; e < E; ++e)
            hk[e] = (static_cast<unsigned long long>(edges[e].first) << 32) | static_cast<unsigned>(edges[e].second);
        Dev<unsigned long long> dk(E), pk(2 * static_cast<size_t>(E)), pk2(2 * static_cast<size_t>(E));
        NRR_CUDA_CHECK(cudaMemcpyAsync(dk.p, hk.data(), E * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
        pair_emit_kernel<<<grid_for(E), kT, 0, s>>>(dk.p, E, pk.p);
        NRR_CUDA_CHECK(cudaGetLastError());
        size_t tmp = 0;
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, pk.p, pk2.p, 2 * E, 0, 64, s));
        Dev<unsigned char> scratch(tmp);
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(scratch.p, tmp, pk.p, pk2.p, 2 * E, 0, 64, s));
        Dev<double> cw(2 * static_cast<size_t>(E));
        NRR_CUDA_CHECK(cudaMemsetAsync(d_bad.p, 0, sizeof(int), s));
        reg_inv_kernel<<<grid_for(2 * E), kT, 0, s>>>(pk2.p, 2 * E, npos.p, cw.p, d_bad.p);
        NRR_CUDA_CHECK(cudaGetLastError());
        const std::vector<unsigned long long> hp = download(pk2.p, 2 * static_cast<size_t>(E), s);
        out.pair_w = download(cw.p, 2 * static_cast<size_t>(E), s);
        NRR_CUDA_CHECK(cudaMemcpy(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (bad & 4) throw NumericalError("reg_weight_table: coincident node positions");
        double inv_sum = 0.0;  // sequential, as the reference
        for (double c : out.pair_w) inv_sum += c;
        const double scale = static_cast<double>(out.pair_w.size()) / inv_sum;
        for (auto& c : out.pair_w) c *= scale;
        out.pairs.resize(4 * static_cast<size_t>(E));
        for (size_t t = 0; t < hp.size(); ++t) {
            out.pairs[2 * t] = static_cast<int>(hp[t] >> 32);
            out.pairs[2 * t + 1] = static_cast<int>(hp[t] & 0xffffffffu);
        }
    }
    mark("done", s);
    if (stats) {
        stats->rounds = rounds;
        stats->nodes = N;
    }
    return out;
}

}  // namespace nrr_b200
