// Block-Jacobi PCG solve of the 4N x 4N, 3-RHS normal equations (see pcg.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace nrr_b200 {

struct PcgStatus {
    int fail_node;   // first node whose 4x4 diagonal block is not PD (INT_MAX = none)
    int code;        // 1 converged, 2 indefinite, 3 iteration cap
    int iterations;  // PCG iterations of this solve
    int restarts;    // true-residual checks
    double bmax;     // max |B|
};

struct PcgArgs {
    const int* row_ptr;   // N+1 (BSR)
    const int* col;       // nnzb
    const double* K;      // nnzb*16
    const double* B;      // 12N node-major
    double* X;            // 12N node-major: in = warm start, out = solution
    double* Z;            // 12N scratch (preconditioned residual, exchanged)
    const int* row_begin; // grid+1 CTA row ranges
    double* part_a;       // grid*8
    double* part_b;       // grid*8
    PcgStatus* status;
    double rtol;
    int max_iter;
    int max_rows, max_kb, k_in_smem;  // filled from the plan
};

struct PcgPlan {
    int nodes = 0, grid = 0, ept = 1, max_rows = 0, max_kb = 0;
    bool k_in_smem = false;
    size_t smem_bytes = 0;
    std::vector<int> row_begin;
    void build(const int* row_ptr_host, int N, int num_sms, size_t smem_limit);
};

void launch_pcg(const PcgPlan& plan, PcgArgs args, cudaStream_t s);

}  // namespace nrr_b200
