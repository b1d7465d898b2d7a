// Device-side problem setup: the per-influence constants and the assembly
// contributor lists (reference SystemAssembler constructor, energy.hpp:137-179,
// 263-310), built on the GPU instead of the host so the one-shot register
// path does not stream ~12 MB of host-built tables.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace nrr_b200 {

struct SetupGpuIn {
    int n = 0, N = 0, U = 0;          // vertices, nodes, upper blocks (N + E)
    const int* infl_off = nullptr;    // n+1
    const int* infl_node = nullptr;   // sum k
    const double* infl_w = nullptr;   // sum k
    const double* src = nullptr;      // n*3
    const double* node_pos = nullptr; // N*3
    const int* node_row = nullptr;    // N: node -> solver row
    const int* row_ptr = nullptr;     // N+1 BSR over solver rows (sorted columns)
    const int* col = nullptr;         // nnzb node ids
    const int* edge_of_blk = nullptr; // nnzb: edge of an (a<b) block, -1 otherwise
    const long long* pair_off = nullptr;  // n+1: prefix of k_i (k_i + 1) / 2 (entries per vertex)
};

struct SetupGpuOut {
    double4* infl_f = nullptr;  // sum k: w [v - p; 1]
    double* anchor = nullptr;   // n*3: sum_a w_a p_a
    int* cptr = nullptr;        // U+1
    int* cv = nullptr;          // entries: vertex
    int* cea = nullptr;         // entries: influence index a
    int* ceb = nullptr;         // entries: influence index b
    double4* cfa = nullptr;     // entries: infl_f[a] (materialised: the assembly streams it instead of gathering)
    double4* cfb = nullptr;     // entries: infl_f[b]
    int* flags = nullptr;       // 1 int: bit 0 = a co-influencing pair is not a graph edge
};

// Scratch sizes (bytes) for build_contributors_gpu at `entries` entries.
size_t setup_gpu_scratch_bytes(long long entries, int U);

// Enqueue on `s`: influence constants, then the contributor lists per upper
// block in vertex order (a stable radix sort of the per-vertex emission by
// block key). `scratch` must hold setup_gpu_scratch_bytes bytes.
void build_setup_gpu(const SetupGpuIn& in, long long entries, const SetupGpuOut& out, void* scratch, cudaStream_t s);

}  // namespace nrr_b200
