// Two-level preconditioned CG for the 4N x 4N, 3-RHS normal equations
// (reference SystemAssembler::solve, energy.hpp:233-254); see pcg.cu.
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace nrr_b200 {

constexpr int kPcgThreads = 384;  // multiple of 12: (row r, column c) fixed per thread; 12 warps leave 168 registers
constexpr int kCoarseMax = 256;
constexpr int kPcgSlots = 32;
constexpr int kMaxEpt = 8;       // elements per thread: up to 256 nodes per CTA   // reduction slots per CTA in part_a / part_b
constexpr int kSubRowsMax = 32;  // nodes per dense subdomain block: one chunk per CTA on cfg2 (measured best once the preconditioner is reused)
// leading dimension of a 4s x 4s subdomain inverse: >= 4s and = 4 (mod 16), so
// the 4 threads x 4 rows of a half-warp hit 16 distinct bank pairs
inline int sub_leading_dim(int s) {
    int ld = 4 * s;
    while (ld % 16 != 4) ++ld;
    return ld;
}  // coarse dimension limit (4 modes per aggregate)

struct PcgStatus {
    int fail_node;   // first node whose 4x4 diagonal block is not PD (INT_MAX = none)
    int code;        // 1 converged, 2 indefinite, 3 iteration cap
    int iterations;  // PCG iterations of this solve
    int restarts;    // true-residual checks
    double bmax;     // max |B|
};

// Solver-side layout (built once per problem by PcgPlan):
//   solver rows are graph nodes permuted by recursive coordinate bisection so
//   that each CTA owns a compact subdomain (rows [row_begin[c], row_begin[c+1]));
//   consecutive groups of `agg_ctas` CTAs form the coarse aggregates.
struct PcgArgs {
    const int* row_ptr;   // N+1 BSR over solver rows
    const int* col;       // nnzb, node ids
    const int* row_node;  // N: solver row -> node id
    const int* colx;      // nnzb: per-CTA operand row of each block's column
    const int* ext_off;   // grid+1
    const int* ext_node;  // operand rows (own rows first, then halo) -> node id
    const int* ext_tl;    // operand rows: index of the row's aggregate in the CTA's touched list
    const int* touch_off; // grid+1
    const int* touch_agg; // per CTA: the aggregates its operand rows touch (ascending)
    const double* K;      // nnzb*16
    const double* B;      // 12N node-major (by node id)
    double* X;            // 12N node-major: in = warm start, out = solution
    double* Z;            // 2 x 12N scratch (preconditioned residual, exchanged), two parities
    double* P;            // 12N scratch: the search direction when a thread owns 4 or more elements (pcg.cu kLean)
    size_t z_stride;      // doubles between the parities of Z (>= 12N)
    const int* row_begin; // grid+1
    const double* node_pos;  // N*3
    const double* agg_center;  // n_agg*3
    const int* node_agg;  // N: aggregate of node
    const double* coarse_inv;  // n_c x n_c
    const double* sub_inv;     // grid x sub_chunks x (4 sub_rows x sub_ld): subdomain inverses
    double* part_a;       // 2 parities x kPartReplicas x kPcgSlots x round_up(grid, 8), slot-major (iteration partials)
    size_t part_stride;   // doubles between the parities of part_a
    double* part_b;       // grid*kPcgSlots
    PcgStatus* status;
    const int* skip;      // nonzero: the pass reverts, setup kernels and the solve return at once
    double rtol;
    double true_factor;  // accept the true residual at true_factor * rtol (1+|B|max)
    int max_iter;
    int max_rows, max_kb, k_in_smem, max_ext;
    int sub_rows, sub_ld, sub_chunks;  // subdomain block-Jacobi plan
    int agg_ctas, n_agg, use_coarse, max_touch;
    long long* prof;  // optional clock64 per phase (CTA 0), accumulated
    long long* cta_prof;  // optional per-CTA work cycles [grid][4] (NRR_PROF)
};

struct PcgPlan {
    int nodes = 0, grid = 0, ept = 1, max_rows = 0, max_kb = 0, max_ext = 0;
    int agg_ctas = 1, n_agg = 1, max_touch = 1;
    int sub_rows = 1, sub_ld = 4, sub_chunks = 1;
    bool k_in_smem = false, use_coarse = true;
    size_t smem_bytes = 0;
    std::vector<int> row_begin;   // grid+1
    std::vector<int> row_node;    // N: solver row -> node
    std::vector<int> node_row;    // N: node -> solver row
    std::vector<int> node_agg;    // N
    std::vector<double> agg_center;  // n_agg*3
    std::vector<int> colx, ext_off, ext_node, ext_tl, touch_off, touch_agg;
    // partition + row order; row_nnz = blocks per node (for balance)
    // adj_off / adj: the node graph (CSR by node id, self included; the first row_nnz_by_node[j] entries of
    // row j are its distinct neighbours), used to round the subdomains after the bisection (pcg.cu)
    void build(const double* node_pos, const int* row_nnz_by_node, int N, int num_sms, size_t smem_limit,
               const int* adj_off = nullptr, const int* adj = nullptr);
    // smem sizing once the BSR (in solver-row order) is known
    void size_smem(const int* row_ptr_solver, const int* col, size_t smem_limit);
};

struct CoarseWork {
    double* partial = nullptr;  // grid * 4 * n_c
    double* inv = nullptr;      // n_c * n_c
};

// K_0 = Psi^T K Psi partials per CTA, then one CTA sums and inverts it.
void launch_coarse_setup(const PcgPlan& plan, const PcgArgs& a, const CoarseWork& w, cudaStream_t s);
// dense inverses of the subdomain diagonal blocks (one CTA per PCG CTA)
void launch_sub_invert(const PcgPlan& plan, const PcgArgs& a, double* out, cudaStream_t s);
// `done` (one per caller, reused): recorded after the launch; cooperative grids
// in flight on the device are kept within one CTA per SM in total
void launch_pcg(const PcgPlan& plan, PcgArgs args, cudaStream_t s, cudaEvent_t done);
void pcg_forget_event(cudaEvent_t done);

}  // namespace nrr_b200
