// Cluster-resident block-Jacobi PCG (see pcg_cluster.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "pcg.cuh"

namespace nrr_b200 {

constexpr int kClusterThreads = 640;  // three threads (right-hand sides) per graph node of the rank
constexpr int kClusterMaxEPT = 4;  // rows per thread (x 128 rows per pass)

// Per-rank packed plan (all ranks concatenated, offsets per rank).
struct ClusterPlanDev {
    const int* rank_rows;      // CS+1: solver rows of rank r = [rank_rows[r], rank_rows[r+1])
    const int* row_node;       // N: solver row -> node id
    const int* ent_ptr;        // N+1: entries of solver row j = [ent_ptr[j], ent_ptr[j+1])
    const int2* ent;           // x = src<<2 | transposed<<1 | in_global ; y = ext index
    const int* diag_ent;       // N: entry index of the diagonal block of row j
    const int* store_off;      // CS+1: smem block store range per rank
    const int* store_src;      // global BSR block copied into each store slot
    const int* halo_off;       // CS+1
    const int2* halo_src;      // (owner rank, owner-local row) per halo row
};

struct ClusterArgs {
    ClusterPlanDev plan;
    const double* K;  // global BSR values (16 per block)
    const double* B;  // 12N node-major
    double* X;        // 12N node-major in/out
    PcgStatus* status;
    double rtol;
    int max_iter;
    int max_rows, max_store, max_ext, max_ent;  // smem sizing
    long long* prof;  // optional: clock64 per phase (rank 0), accumulated
};

struct ClusterPlan {
    bool ok = false;
    int CS = 0, ept = 1, max_rows = 0, max_store = 0, max_ext = 0, max_ent = 0;
    size_t smem_bytes = 0;
    std::vector<int> rank_rows, row_node, node_row, ent_ptr, diag_ent, store_off, store_src, halo_off;
    std::vector<int2> ent, halo_src;
    // bsr over nodes: row_ptr/col in *any* row order with a position lookup
    void build(const double* node_pos, const int* row_ptr, const int* col, const int* node_row_bsr, int N,
               size_t smem_limit, int max_cs);
};

void launch_pcg_cluster(const ClusterPlan& plan, ClusterArgs a, cudaStream_t s);

}  // namespace nrr_b200
