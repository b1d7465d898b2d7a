// Per-iteration kernels of the Welsch-MM hot path (see kernels.cu) and the
// device-side view of one registration problem.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace nrr_b200 {

constexpr int kMaxAA = 16;  // Anderson window supported on the device

// Read-only device view of the problem (built once in nrr_ctx_set_problem).
// Node transforms live node-major: x[12j + 3r + c] = X(4j+r, c) of the
// reference's 4N x 3 column-major stacking (deformation_graph.hpp:17-35).
struct DevProblem {
    int n = 0, N = 0, E = 0, P = 0, U = 0, nnzb = 0;
    const double* src = nullptr;       // n*3
    const int* infl_off = nullptr;     // n+1
    const int* infl_node = nullptr;    // sum k
    const double* infl_w = nullptr;    // sum k
    const double4* infl_f = nullptr;   // sum k: f = w [v - p; 1] (energy.hpp:150-161)
    const double* anchor = nullptr;    // n*3: sum_a w_a p_a
    const double* node_pos = nullptr;  // N*3
    const int* pairs = nullptr;        // P*2 (i, j)
    const double* pair_c = nullptr;    // P
    const int* pair_rev = nullptr;     // P: index of (j, i)
    const double4* pair_gv = nullptr;  // P: g_e = c [p_i - p_j; 1] (energy.hpp:163-173), fixed per problem
    const int* node_pair_off = nullptr;  // N+1: pairs with i == j, ascending j
    const int* row_ptr = nullptr;      // N+1 BSR over solver rows (pcg.cu order)
    const int* col = nullptr;          // nnzb (node ids)
    const int* node_row = nullptr;     // N: node -> solver row
    // assembly plan: upper blocks u < N diagonal j = u, u >= N graph edge u-N
    const int* ub_cptr = nullptr;      // U+1 contributor ranges
    const int* c_v = nullptr;          // contributor vertex
    const int* c_ea = nullptr;         // contributor influence entry of the row node
    const int* c_eb = nullptr;         // contributor influence entry of the column node
    const double4* c_fa = nullptr;     // infl_f[c_ea] per contributor (streamed, not gathered)
    const double4* c_fb = nullptr;     // infl_f[c_eb] per contributor
    const int* ub_kpos = nullptr;      // BSR block (a, b)
    const int* ub_kpos_t = nullptr;    // BSR block (b, a)
    const int* edges = nullptr;        // E*2
    const int* edge_pab = nullptr;     // E: pair (a -> b)
    const int* edge_pba = nullptr;     // E: pair (b -> a)
    int landmarks = 0;
    const int* lm_vertex = nullptr;
    const double* lm_pos = nullptr;
    // pass-level skip flag (device-side safeguard decision, see
    // launch_pass_decision): nonzero = the pass reverts, assembly and solve
    // are no-ops
    const int* skip = nullptr;
};


// per-pass energy record copied to the host (pinned)
struct PassRecord {
    double align, reg, rot, total, landmark;
    double max_disp;
    int degenerate;
    int nonfinite;  // iterate / energy not finite
    int pcg_iters, pcg_code, pcg_fail_node, pcg_restarts;
    int aa_rank, pad;
};

// Safeguard decision of the current pass on the device (solver.hpp:239):
// skip = !finite(E) || (evaluating an AA iterate && E > E_prev), with
// E = total + lm_w * landmark formed like the host does (no contraction).
void launch_pass_decision(const PassRecord* rec, double e_prev, int current_is_aa, double lm_w, int* skip,
                          cudaStream_t s);

struct TermParams {
    double alpha, beta, nu_a, nu_r, lm_weight;
};

void launch_deform(const DevProblem& p, const double* x, double* out, const double* old, double* max_disp,
                   int* nonfinite, cudaStream_t s);
void launch_terms(const DevProblem& p, const double* x, const double* d2, const TermParams& tp, double* wa,
                  double* wr, double* R, double* partials, int* degenerate, cudaStream_t s);
void launch_energy_reduce(const DevProblem& p, const double* partials, const TermParams& tp, const double* vhat,
                          PassRecord* rec, cudaStream_t s);
void launch_assemble(const DevProblem& p, const double* wa, const double* q, const double* wr, const double* R,
                     const TermParams& tp, double* K, double* B, cudaStream_t s);
void launch_rotations(const double* x, int N, double* R, int* degenerate, cudaStream_t s,
                      double* sigma_min = nullptr);

// Anderson acceleration on device vectors of length D = 12N
constexpr int kTriMax = (kMaxAA + 1) * (kMaxAA + 2) / 2;  // packed R of [dF | f]
struct AADevice {
    double* df = nullptr;        // m*D ring of F differences
    double* dg = nullptr;        // m*D ring of G differences
    double* fprev = nullptr;     // D: newest f
    double* gprev = nullptr;     // D: newest g
    double* theta = nullptr;     // kMaxAA (newest-first column order)
    double* partials = nullptr;  // kTermBlocks * kTriMax
    int* rank = nullptr;
};
struct SlotList {  // ring slots, newest first
    int s[kMaxAA];
    int n;
};
// push (g = xmm, x = current iterate, or f given): new difference columns
// into ring slot `slot` when the window held an entry (anderson.hpp:58-61)
void launch_aa_update(const AADevice& aa, const double* g, const double* x, const double* f, int D, int have_prev,
                      int slot, cudaStream_t s);
// the push fused with the least squares min |f - dF theta| over the columns
// `cols` (anderson.hpp:31-44): theta and rank are left in aa.theta / aa.rank
void launch_aa_push_solve(const AADevice& aa, const double* g, const double* x, const double* f, int D, int have_prev,
                          int slot, const SlotList& cols, cudaStream_t s);
// x_next = g - sum_j theta_j dg_{cols[j]} (anderson.hpp:45)
void launch_aa_combine(const AADevice& aa, int D, const SlotList& cols, double* x_next, int* nonfinite,
                       cudaStream_t s);

// layout conversion: reference column-major 4N x 3 <-> node-major 12N
void launch_colmajor_to_nodemajor(const double* in, double* out, int N, cudaStream_t s);
void launch_nodemajor_to_colmajor(const double* in, double* out, int N, cudaStream_t s);

}  // namespace nrr_b200
