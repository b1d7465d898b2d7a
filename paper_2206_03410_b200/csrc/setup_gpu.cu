// Device-side problem setup (see setup_gpu.cuh).
//
// Contributor lists. The assembly kernel accumulates every upper 4x4 block u
// of K (diagonal block of node a, or the (a,b) block of edge e, a < b) from a
// precomputed list of (vertex i, influence a, influence b) triples in vertex
// order: the reference's program order (energy.hpp:290-310, emit_point
// :313-327), which keeps the fill deterministic without atomics. Each vertex
// i emits k_i (k_i + 1) / 2 triples (its diagonal entries and its a < b
// pairs) at a precomputed offset; a stable LSD radix sort by block key then
// yields every block's list in vertex order, identical to the host build.
#include <cub/cub.cuh>

#include "device_common.cuh"
#include "setup_gpu.cuh"

namespace nrr_b200 {

namespace {

constexpr int kSetupThreads = 256;

// f[k] = w_k [v_i - p_a; 1] and anchor_i = sum_k w_k p_a (energy.hpp:150-161),
// unfused so the bits match the host restatement
__global__ void influence_constants_kernel(SetupGpuIn in, double4* __restrict__ f, double* __restrict__ anchor) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= in.n) return;
    const int k0 = in.infl_off[i], k1 = in.infl_off[i + 1];
    const double v0 = in.src[3 * i], v1 = in.src[3 * i + 1], v2 = in.src[3 * i + 2];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = k0; k < k1; ++k) {
        const int a = in.infl_node[k];
        const double w = in.infl_w[k];
        const double p0 = in.node_pos[3 * a], p1 = in.node_pos[3 * a + 1], p2 = in.node_pos[3 * a + 2];
        f[k] = make_double4(__dmul_rn(w, __dsub_rn(v0, p0)), __dmul_rn(w, __dsub_rn(v1, p1)),
                            __dmul_rn(w, __dsub_rn(v2, p2)), w);
        s0 = __dadd_rn(s0, __dmul_rn(w, p0));
        s1 = __dadd_rn(s1, __dmul_rn(w, p1));
        s2 = __dadd_rn(s2, __dmul_rn(w, p2));
    }
    anchor[3 * i] = s0;
    anchor[3 * i + 1] = s1;
    anchor[3 * i + 2] = s2;
}

__device__ __forceinline__ int find_block(const SetupGpuIn& in, int a, int b) {
    const int r = in.node_row[a];
    int lo = in.row_ptr[r], hi = in.row_ptr[r + 1];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (in.col[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    return lo < in.row_ptr[r + 1] && in.col[lo] == b ? lo : -1;
}

// one thread per vertex: its triples in the host order (ka outer; the
// diagonal entry, then the a < b pairs), keyed by upper block
__global__ void emit_kernel(SetupGpuIn in, int* __restrict__ key, int* __restrict__ val, int* __restrict__ ei,
                            int* __restrict__ ea, int* __restrict__ eb, int* __restrict__ ucnt, int* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= in.n) return;
    const int k0 = in.infl_off[i], k1 = in.infl_off[i + 1];
    long long q = in.pair_off[i];
    for (int ka = k0; ka < k1; ++ka) {
        const int a = in.infl_node[ka];
        key[q] = a;
        val[q] = static_cast<int>(q);
        ei[q] = i;
        ea[q] = ka;
        eb[q] = ka;
        atomicAdd(ucnt + a, 1);
        ++q;
        for (int kb = k0; kb < k1; ++kb) {
            const int b = in.infl_node[kb];
            if (a >= b) continue;
            const int blk = find_block(in, a, b);
            const int e = blk >= 0 ? in.edge_of_blk[blk] : -1;
            if (e < 0) {
                atomicOr(flags, 1);
                key[q] = 0;  // keeps the sort well defined; the host raises the error
            } else {
                key[q] = in.N + e;
                atomicAdd(ucnt + in.N + e, 1);
            }
            val[q] = static_cast<int>(q);
            ei[q] = i;
            ea[q] = ka;
            eb[q] = kb;
            ++q;
        }
    }
}

__global__ void gather_kernel(long long count, const int* __restrict__ order, const int* __restrict__ ei,
                              const int* __restrict__ ea, const int* __restrict__ eb, int* __restrict__ cv,
                              int* __restrict__ cea, int* __restrict__ ceb, const double4* __restrict__ f,
                              double4* __restrict__ cfa, double4* __restrict__ cfb) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= count) return;
    const int q = order[p];
    const int a = ea[q], b = eb[q];
    cv[p] = ei[q];
    cea[p] = a;
    ceb[p] = b;
    cfa[p] = f[a];
    cfb[p] = f[b];
}

int key_bits(int U) {
    int b = 1;
    while ((1LL << b) < U) ++b;
    return b;
}

struct Scratch {
    int *key, *key_out, *val, *val_out, *ei, *ea, *eb, *ucnt;
    void* cub_tmp;
    size_t cub_bytes;
};

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

size_t cub_bytes_needed(long long entries, int U) {
    size_t sort_b = 0, scan_b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_b, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                    static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                    static_cast<int>(entries), 0, key_bits(U));
    cub::DeviceScan::ExclusiveSum(nullptr, scan_b, static_cast<const int*>(nullptr), static_cast<int*>(nullptr), U + 1);
    return std::max(sort_b, scan_b);
}

Scratch carve(void* base, long long entries, int U) {
    char* p = static_cast<char*>(base);
    const size_t eb = align256(sizeof(int) * static_cast<size_t>(std::max<long long>(entries, 1)));
    Scratch s{};
    s.key = reinterpret_cast<int*>(p);
    p += eb;
    s.key_out = reinterpret_cast<int*>(p);
    p += eb;
    s.val = reinterpret_cast<int*>(p);
    p += eb;
    s.val_out = reinterpret_cast<int*>(p);
    p += eb;
    s.ei = reinterpret_cast<int*>(p);
    p += eb;
    s.ea = reinterpret_cast<int*>(p);
    p += eb;
    s.eb = reinterpret_cast<int*>(p);
    p += eb;
    s.ucnt = reinterpret_cast<int*>(p);
    p += align256(sizeof(int) * (static_cast<size_t>(U) + 1));
    s.cub_tmp = p;
    s.cub_bytes = cub_bytes_needed(entries, U);
    return s;
}

}  // namespace

size_t setup_gpu_scratch_bytes(long long entries, int U) {
    const size_t eb = align256(sizeof(int) * static_cast<size_t>(std::max<long long>(entries, 1)));
    return 7 * eb + align256(sizeof(int) * (static_cast<size_t>(U) + 1)) + align256(cub_bytes_needed(entries, U)) + 256;
}

void build_setup_gpu(const SetupGpuIn& in, long long entries, const SetupGpuOut& out, void* scratch, cudaStream_t s) {
    if (in.n == 0) {
        NRR_CUDA_CHECK(cudaMemsetAsync(out.cptr, 0, sizeof(int) * (static_cast<size_t>(in.U) + 1), s));
        NRR_CUDA_CHECK(cudaMemsetAsync(out.flags, 0, sizeof(int), s));
        return;
    }
    const int blocks = (in.n + kSetupThreads - 1) / kSetupThreads;
    influence_constants_kernel<<<blocks, kSetupThreads, 0, s>>>(in, out.infl_f, out.anchor);
    NRR_CUDA_CHECK(cudaGetLastError());
    Scratch sc = carve(scratch, entries, in.U);
    NRR_CUDA_CHECK(cudaMemsetAsync(sc.ucnt, 0, sizeof(int) * (static_cast<size_t>(in.U) + 1), s));
    NRR_CUDA_CHECK(cudaMemsetAsync(out.flags, 0, sizeof(int), s));
    emit_kernel<<<blocks, kSetupThreads, 0, s>>>(in, sc.key, sc.val, sc.ei, sc.ea, sc.eb, sc.ucnt, out.flags);
    NRR_CUDA_CHECK(cudaGetLastError());
    size_t tb = sc.cub_bytes;
    NRR_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(sc.cub_tmp, tb, sc.key, sc.key_out, sc.val, sc.val_out,
                                                   static_cast<int>(entries), 0, key_bits(in.U), s));
    tb = sc.cub_bytes;
    NRR_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(sc.cub_tmp, tb, sc.ucnt, out.cptr, in.U + 1, s));
    const int gb = static_cast<int>((entries + kSetupThreads - 1) / kSetupThreads);
    gather_kernel<<<gb, kSetupThreads, 0, s>>>(entries, sc.val_out, sc.ei, sc.ea, sc.eb, out.cv, out.cea, out.ceb,
                                               out.infl_f, out.cfa, out.cfb);
    NRR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace nrr_b200
