/* ORACLE — TEST INFRASTRUCTURE ONLY. C entry points of the CPU restatement
 * (nrr_oracle.hpp) for the Python parity tests and the bench's CPU-baseline
 * leg. The view/record structs have the same layout as the product's
 * include/nrr_cuda.h so one set of host buffers feeds both. */
#ifndef NRR_ORACLE_CAPI_H
#define NRR_ORACLE_CAPI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_problem_view {
    int32_t n;                    /* source points */
    const double* source;         /* n*3 xyz */
    double src_avg_edge_length;   /* Surface::avg_edge_length */
    int32_t m;                    /* target points */
    const double* target;         /* m*3 */
    int32_t node_count;           /* N */
    const double* node_positions; /* N*3 */
    int32_t edge_count;           /* E */
    const int32_t* edges;         /* E*2, first < second */
    const int32_t* infl_offsets;  /* n+1 */
    const int32_t* infl_nodes;    /* sum k */
    const double* infl_weights;   /* sum k */
    int32_t pair_count;           /* P = 2E */
    const int32_t* reg_pairs;     /* P*2 (i, j), i-major */
    const double* reg_weights;    /* P */
} oracle_problem_view;

typedef struct oracle_solver_config {
    double k_alpha, k_beta, eps;
    int32_t i_max, aa_window;
    double nu_a_init, nu_a_min, nu_r_init, nu_r_floor;
    int32_t landmark_count;
    const int32_t* landmark_index;
    const double* landmark_pos;
} oracle_solver_config;

typedef struct oracle_iteration_record {
    double e_total, e_align, e_reg, e_rot, e_landmark, max_disp;
    int32_t aa_accepted, stage;
} oracle_iteration_record;

typedef struct oracle_stage_record {
    double nu_a, nu_r, alpha, beta;
    int32_t reverts, converged, first_iteration, iteration_count;
} oracle_stage_record;

typedef struct oracle_pass_record {
    double e_total;
    int32_t stage, reverted;
} oracle_pass_record;

typedef struct oracle_report_summary {
    int32_t stage_count, total_iterations, degenerate_rotations, alpha_forced_zero;
    int32_t total_passes, linear_iterations;
    double solve_seconds, setup_seconds, loop_seconds;
} oracle_report_summary;

const char* oracle_last_error(void);

/* surface / graph setup (surface.hpp, deformation_graph.hpp) */
int oracle_edges_from_faces(const int32_t* faces, int32_t nf, int32_t n, int32_t* out_edges,
                            int32_t cap, int32_t* out_count);
int oracle_knn_edges(const double* pts, int32_t n, int32_t k, int32_t* out_edges, int32_t cap,
                     int32_t* out_count);
int oracle_avg_edge_length(const double* pts, int32_t n, const int32_t* edges, int32_t ne,
                           double* out);
typedef struct oracle_graph oracle_graph;
int oracle_build_graph(const double* pts, int32_t n, const int32_t* edges, int32_t ne,
                       double radius, oracle_graph** out);
void oracle_graph_counts(const oracle_graph* g, int32_t* N, int32_t* E, int32_t* sumk, int32_t* P);
void oracle_graph_export(const oracle_graph* g, int32_t* node_indices, double* node_positions,
                         int32_t* edges, int32_t* infl_offsets, int32_t* infl_nodes,
                         double* infl_weights, double* infl_dist, int32_t* reg_pairs,
                         double* reg_weights);
void oracle_graph_free(oracle_graph* g);

/* normalize_pair (surface.hpp:125-149), in place; out4 = {scale, cx, cy, cz} */
int oracle_normalize_pair(double* src, int32_t n, double* tgt, int32_t m, double* out4);
/* seeded synthetic inputs of BASELINE configs 0-4 (synth/nrr_synth.hpp, shared
 * with the product's nrr_synth_config): lets the bench's reference arm build
 * its inputs without loading the product library. Sizes first with NULL
 * buffers. */
int oracle_synth_config(int32_t which, uint64_t seed, double scale, int32_t* n, int32_t* nf_src, int32_t* m,
                        double* src, int32_t* src_faces, double* tgt);

/* primitives */
int oracle_nearest(const double* target, int32_t m, const double* queries, int32_t q,
                   int32_t* out_index, double* out_distance);
int oracle_deform(const oracle_problem_view* p, const double* X, double* out_points);
int oracle_project_rotations(const double* X, int32_t N, double* out_R, int32_t* out_degenerate);
int oracle_project_to_rotation(const double* A, double* out_R, double* out_sigma_min);

/* One teacher-forced pass at iterate X (12N col-major, reference layout):
 * correspondences, energy, weights, K/B fill and solve.
 * out_K: BSR values in the fixed pattern (block rows = nodes, sorted
 * columns {j} U neighbors(j)), 16 per block row-major; caller sizes it
 * 16*(N+P). out_B and out_Xmm are 12N col-major. prm = {alpha,beta,nu_a,nu_r}. */
int oracle_step(const oracle_problem_view* p, const double* X, const double* prm,
                double landmark_weight, const oracle_solver_config* cfg_for_landmarks,
                int32_t* out_index, double* out_sqdist, double* out_energy4,
                double* out_K, double* out_B, double* out_Xmm);

/* AA: history of h entries (oldest first), each g and f of length dim */
int oracle_anderson_combine(const double* G, const double* F, int32_t h, int32_t dim, int32_t m,
                            double* out, int32_t* out_rank);

/* 0 = RCM (default), 1 = natural node order for the direct solve */
void oracle_set_ldlt_ordering(int mode);
int oracle_register(const oracle_problem_view* p, const oracle_solver_config* cfg, double* out_X,
                    double* out_deformed, oracle_iteration_record* iters, int32_t iter_cap,
                    oracle_stage_record* stages, int32_t stage_cap, oracle_pass_record* passes,
                    int32_t pass_cap, int32_t* pass_nn_index /* pass_cap*n or NULL */,
                    oracle_report_summary* summary);

/* CPU baseline: wall time of `steps` accepted MM iterations after `warmup`
 * accepted ones, single stage at the given config (fixed-count idiom). */
int oracle_time_iterations(const oracle_problem_view* p, const oracle_solver_config* cfg, int32_t warmup,
                           int32_t steps, double* seconds);

/* init_parameters (solver.hpp:86-106): out6 = {nu_a, nu_r, nu_a_min, alpha, beta, forced_zero} */
int oracle_init_parameters(const oracle_problem_view* p, const oracle_solver_config* cfg,
                           double* out6);

#ifdef __cplusplus
}
#endif
#endif
