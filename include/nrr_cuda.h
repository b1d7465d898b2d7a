/*
 * nrr_cuda.h — C ABI of the B200 (sm_100a) implementation of the per-iteration
 * hot path of the reference's Welsch majorization-minimization non-rigid
 * registration (reference: /root/reference/proj/include/nrr, arXiv 2206.03410).
 *
 * Plain pointers and sizes only; no C++ or torch types. Every host buffer is
 * copied at the call; no caller pointer is retained. Each entry point names
 * the reference interface it replaces (file:line under proj/include/nrr).
 *
 * Layouts (all FP64 unless stated; indices int32):
 *   points      n*3 AoS xyz                       (Surface::points, surface.hpp:18)
 *   X           12N, column-major 4N x 3: X[c*4N + 4j + r] = A_j(c,r) for r<3,
 *               t_j(c) for r=3                    (NodeTransforms, deformation_graph.hpp:17-35,
 *                                                  flatten solver.hpp:146-148)
 *   influence   CSR over source points: offsets[n+1], nodes[sum k], weights[sum k]
 *                                                 (DeformationGraph::influence, :54)
 *   reg pairs   P*2 (i,j) i-major directed pairs + weights[P] (:59-60)
 *   K           BSR values of the fixed pattern (block row j = sorted {j} U N(j)),
 *               16 doubles per 4x4 block, row-major (SystemAssembler, energy.hpp:264-279)
 *   B           12N column-major 4N x 3 (LinearSystem::B, energy.hpp:120)
 *   R           N*9, row-major 3x3 per node (project_rotations, energy.hpp:47-56)
 *
 * Errors: every int-returning call returns NRR_OK (0) or the reference CLI's
 * exit-code class (nrr_cli.cpp:266-278): 2 = IoError, 3 = NumericalError,
 * 4 = ConfigError, 5 = CUDA/internal. nrr_last_error() returns the message of
 * the calling thread's last failure; the exception text matches the
 * reference's ("... not positive definite (singular diagonal block at node j)").
 */
#ifndef NRR_CUDA_H
#define NRR_CUDA_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NRR_OK 0
#define NRR_ERR_IO 2
#define NRR_ERR_NUMERICAL 3
#define NRR_ERR_CONFIG 4
#define NRR_ERR_CUDA 5

/* Source/target/graph of one registration (register_surfaces inputs,
 * solver.hpp:180-183: Surface source, Surface target, DeformationGraph). */
typedef struct nrr_problem_view {
    int32_t n;                    /* source point count */
    const double* source;         /* n*3 */
    double src_avg_edge_length;   /* Surface::avg_edge_length (surface.hpp:21) */
    int32_t m;                    /* target point count */
    const double* target;         /* m*3 */
    int32_t node_count;           /* N */
    const double* node_positions; /* N*3 */
    int32_t edge_count;           /* E, graph_edges first < second, sorted */
    const int32_t* edges;         /* E*2 */
    const int32_t* infl_offsets;  /* n+1 */
    const int32_t* infl_nodes;    /* sum k */
    const double* infl_weights;   /* sum k */
    int32_t pair_count;           /* P = 2E */
    const int32_t* reg_pairs;     /* P*2 */
    const double* reg_weights;    /* P */
} nrr_problem_view;

/* SolverConfig (solver.hpp:16-39); NaN overrides mean "derive from data". */
typedef struct nrr_solver_config {
    double k_alpha, k_beta, eps;
    int32_t i_max, aa_window;
    double nu_a_init, nu_a_min, nu_r_init, nu_r_floor;
    int32_t landmark_count;
    const int32_t* landmark_index; /* landmark_count */
    const double* landmark_pos;    /* landmark_count*3 */
} nrr_solver_config;

/* IterationRecord (solver.hpp:108-116) + the stage it belongs to */
typedef struct nrr_iteration_record {
    double e_total, e_align, e_reg, e_rot, e_landmark, max_disp;
    int32_t aa_accepted, stage;
} nrr_iteration_record;

/* StageRecord (solver.hpp:118-124); iterations are [first, first+count) */
typedef struct nrr_stage_record {
    double nu_a, nu_r, alpha, beta;
    int32_t reverts, converged, first_iteration, iteration_count;
} nrr_stage_record;

/* every evaluated pass, including reverted ones (test instrumentation) */
typedef struct nrr_pass_record {
    double e_total;
    int32_t stage, reverted;
} nrr_pass_record;

/* RegistrationReport (solver.hpp:126-138) + device-side counters */
typedef struct nrr_report_summary {
    int32_t stage_count, total_iterations, degenerate_rotations, alpha_forced_zero;
    int32_t total_passes, linear_iterations; /* PCG iterations over the run */
    double solve_seconds, setup_seconds, loop_seconds;
} nrr_report_summary;

/* Solver knobs of the B200 path (no reference counterpart: the reference
 * solves directly). The PCG stops when max|r| <= pcg_rtol*(1+max|B|) and the
 * true residual meets the reference bar 1e-8*(1+max|B|) (energy.hpp:245). */
typedef struct nrr_solve_options {
    double pcg_rtol;      /* default 1e-13: AA trajectories then track the reference as long as the reference tracks itself under a change of direct-solver ordering */
    int32_t pcg_max_iter; /* default 20000 */
    int32_t record_passes;/* keep per-pass records: 1 = records, 2 = + NN indices, 3 = + pass trace (nrr_ctx_trace) */
    int32_t max_ctas;     /* PCG grid cap, 0 = one CTA per SM; set before nrr_ctx_set_problem. Several contexts
                             driven from several host threads then run side by side (config 3 batches) */
} nrr_solve_options;

typedef struct nrr_ctx nrr_ctx;

const char* nrr_last_error(void);
int nrr_device_info(int device, char* name, int32_t cap, int32_t* sm_count);

/* context = all device buffers of one registration (one stream) */
int nrr_ctx_create(int device, nrr_ctx** out);
void nrr_ctx_destroy(nrr_ctx* ctx);
int nrr_ctx_set_options(nrr_ctx* ctx, const nrr_solve_options* opt);

/* SpatialIndex ctor (kd_tree.hpp:115-122): upload the target and build the
 * device BVH (Morton-ordered implicit 8-ary tree). */
int nrr_ctx_set_target(nrr_ctx* ctx, const double* target, int32_t m);

/* SystemAssembler ctor (energy.hpp:139-176) + deform setup: upload source,
 * graph, influence CSR; build the fixed block pattern and assembly plan. */
int nrr_ctx_set_problem(nrr_ctx* ctx, const nrr_problem_view* p);

/* register_surfaces (solver.hpp:180-304) on the uploaded problem. Outputs are
 * host buffers (may be NULL): out_X 12N col-major, out_deformed n*3. */
int nrr_ctx_register(nrr_ctx* ctx, const nrr_solver_config* cfg, double* out_X,
                     double* out_deformed);

/* The same loop, stepped from the host (used by the bench to time exactly K
 * accepted MM iterations with the inputs resident in HBM):
 *   begin   = validate + init_parameters + identity X + first deform
 *             (solver.hpp:183-199)
 *   iterate = run passes until `max_accepted` more iterations were accepted
 *             or the run finished; *device_ms = CUDA-event time of those
 *             passes on the context stream; flush_l2 writes a 2x-L2 buffer
 *             before every pass, outside the timed interval
 *   finish  = outputs + report (solver.hpp:299-303) */
int nrr_ctx_begin(nrr_ctx* ctx, const nrr_solver_config* cfg);
int nrr_ctx_iterate(nrr_ctx* ctx, int32_t max_accepted, int32_t flush_l2, int32_t* accepted, int32_t* done,
                    double* device_ms);
int nrr_ctx_finish(nrr_ctx* ctx, double* out_X, double* out_deformed);

/* one-shot register_surfaces with host buffers (set_target + set_problem + run) */
int nrr_register(nrr_ctx* ctx, const nrr_problem_view* p, const nrr_solver_config* cfg,
                 double* out_X, double* out_deformed);

/* Vertex-sharded registration over NCCL (config 4): every
 * rank calls nrr_ctx_set_comm with the same 128-byte id (from
 * nrr_comm_unique_id on rank 0, broadcast by the caller), then
 * nrr_ctx_set_shard(n_global) and sets a problem view holding ITS contiguous
 * slice of the source vertices (influence CSR rebased) with the full target
 * and graph. The partial energies, K, B and max displacement are allreduced
 * every pass; the solve and Anderson run replicated. Outputs: X (identical on
 * all ranks) and the rank's slice of the deformed points. */
int nrr_comm_unique_id(void* out128);
int nrr_ctx_set_comm(nrr_ctx* ctx, const void* id128, int32_t nranks, int32_t rank);
/* In-process group of contexts (one process, one host thread per context):
 * the sharded path's collectives rendezvous on the host and reduce in rank
 * order on the device. Lets the product's vertex-sharded path run with
 * several ranks on one GPU (tests); NCCL (nrr_ctx_set_comm) is the multi-GPU
 * path. The group must outlive its contexts' runs. */
typedef struct nrr_local_group nrr_local_group;
int nrr_local_group_create(int32_t nranks, nrr_local_group** out);
void nrr_local_group_destroy(nrr_local_group* group);
int nrr_ctx_set_local_comm(nrr_ctx* ctx, nrr_local_group* group, int32_t rank);
int nrr_ctx_set_shard(nrr_ctx* ctx, int32_t n_global);

/* report of the last run */
int nrr_ctx_report(nrr_ctx* ctx, nrr_report_summary* summary, nrr_stage_record* stages,
                   int32_t stage_cap, nrr_iteration_record* iters, int32_t iter_cap,
                   nrr_pass_record* passes, int32_t pass_cap, int32_t* pass_nn_index);

/* Pass trace (test instrumentation; set nrr_solve_options.record_passes = 3
 * before nrr_ctx_begin): every evaluated pass of the last run in order —
 * reverted ones included — with the iterate it was evaluated at (X, 12N
 * column-major), its correspondences (n target indices), its energies, and,
 * for an accepted pass, the solve's x_mm (12N column-major; NaN otherwise).
 * Lets a caller re-run the reference step at every iterate of the device
 * trajectory (teacher-forced parity of solver.hpp:224-289). */
typedef struct nrr_pass_trace {
    double e_align, e_reg, e_rot, e_total, e_landmark;
    double max_disp;          /* accepted passes: max |v' - v| of the next iterate */
    int32_t stage, reverted;  /* reverted: the safeguard (solver.hpp:239) rejected the iterate */
    int32_t pcg_iterations;   /* accepted passes */
    int32_t accepted_index;   /* index of its IterationRecord, -1 for a reverted pass */
} nrr_pass_trace;
int nrr_ctx_trace_count(nrr_ctx* ctx, int32_t* passes);
int nrr_ctx_trace(nrr_ctx* ctx, int32_t pass, nrr_pass_trace* rec, double* x_eval, double* x_mm,
                  int32_t* nn_index);

/* SpatialIndex::nearest / find_correspondences (kd_tree.hpp:124-129,
 * energy.hpp:28-42) for a batch of host queries; out_distance = sqrt(d2). */
int nrr_nearest(nrr_ctx* ctx, const double* queries, int32_t q, int32_t* out_index,
                double* out_distance);
/* the same with a warm start: prev_index[i] (a valid target index, or -1) seeds
 * query i's bound, as the registration loop seeds each pass with the previous
 * pass's correspondences; the result is the same exact argmin */
int nrr_nearest_from(nrr_ctx* ctx, const double* queries, int32_t q, const int32_t* prev_index,
                     int32_t* out_index, double* out_distance);

/* deform_points (deformation_graph.hpp:225-245) at host X */
int nrr_deform(nrr_ctx* ctx, const double* X, double* out_points);

/* project_rotations (energy.hpp:47-56) of host X (N nodes) */
int nrr_project_rotations(nrr_ctx* ctx, const double* X, int32_t N, double* out_R,
                          int32_t* out_degenerate);
/* the same with each node's smallest singular value (project_to_rotation's
   sigma_min, rotation.hpp:14-24); out_sigma_min may be NULL */
int nrr_project_rotations_sigma(nrr_ctx* ctx, const double* X, int32_t N, double* out_R, double* out_sigma_min,
                                int32_t* out_degenerate);

/* The reference API's energy helpers on caller-held arrays, on the device:
 * alignment_weights (energy.hpp:363-368) from corr_sqdist, regularization_
 * weights (:371-378) and the evaluate_energy sums (:92-116) {align, reg, rot}
 * (reg and rot unweighted; total = align + alpha reg + beta rot is formed by
 * the caller). Any input group may be NULL when its outputs are not wanted;
 * X is the reference 4N x 3 column-major block, rotations N x 9 row-major. */
typedef struct nrr_energy_terms_in {
    int32_t n;
    const double* deformed;     /* n*3 */
    const double* corr_points;  /* n*3 */
    const double* corr_sqdist;  /* n */
    double nu_a;
    int32_t node_count;
    const double* X;               /* 12N */
    const double* node_positions;  /* N*3 */
    int32_t pair_count;
    const int32_t* reg_pairs;      /* P*2 */
    const double* reg_weights;     /* P */
    double nu_r, alpha;
    const double* rotations;       /* N*9 */
} nrr_energy_terms_in;
int nrr_energy_terms(nrr_ctx* ctx, const nrr_energy_terms_in* in, double* out_w_align, double* out_w_reg,
                     double* out_sums3);

/* One teacher-forced pass at host X with prm = {alpha, beta, nu_a, nu_r}:
 * find_correspondences + evaluate_energy (energy.hpp:92-116) + weights
 * (:363-378) + SystemAssembler::fill (:182-228) + solve (:233-254).
 * Any output may be NULL. out_energy4 = {align, reg, rot, total}. */
int nrr_step(nrr_ctx* ctx, const double* X, const double* prm, double landmark_weight,
             const nrr_solver_config* cfg_for_landmarks, int32_t* out_index,
             double* out_sqdist, double* out_energy4, double* out_K, double* out_B,
             double* out_Xmm);

/* SystemAssembler::fill (energy.hpp:182-228) from caller state: corr_points =
 * Correspondences::target_point (n*3), w_align (n) = alignment_weights,
 * w_reg (P) = regularization_weights (already scaled by alpha), rotations
 * (N*9, row-major 3x3 per node). out_K = BSR values in the reference pattern
 * order (node a's blocks, ascending column, 16 row-major doubles per block),
 * out_B = 4N x 3 column-major. The system stays resident for nrr_solve. */
int nrr_assemble(nrr_ctx* ctx, const double* corr_points, const double* w_align, const double* w_reg,
                 const double* rotations, double beta, double landmark_weight,
                 const nrr_solver_config* cfg_for_landmarks, double* out_K, double* out_B);

/* SystemAssembler::solve / solve_system (energy.hpp:233-254, :393-409) by the
 * device PCG. K (reference pattern order) and B (4N x 3) may be NULL to reuse
 * the resident system of the last nrr_assemble/nrr_step; X0 = warm start
 * (NULL = zero). Same failure messages as the reference. */
int nrr_solve(nrr_ctx* ctx, const double* K, const double* B, const double* X0, double* out_X);

/* anderson_combine (anderson.hpp:22-46) on a host history of h entries
 * (oldest first, g and f of length dim each), window m. */
int nrr_anderson_combine(nrr_ctx* ctx, const double* G, const double* F, int32_t h,
                         int32_t dim, int32_t m, double* out, int32_t* out_rank);

/* init_parameters (solver.hpp:86-106) on the uploaded problem:
 * out6 = {nu_a, nu_r, nu_a_min, alpha, beta, alpha_forced_zero} */
int nrr_init_parameters(nrr_ctx* ctx, const nrr_solver_config* cfg, double* out6);

/* device-side counters of the context: kernel launches issued by this
 * library since creation, and per-kernel-class CUDA-event timings (ms) of
 * the last run: [0]=NN, [1]=terms+energy, [2]=assembly, [3]=PCG, [4]=AA,
 * [5]=deform. */
int nrr_ctx_stats(nrr_ctx* ctx, int64_t* launches, double* kernel_ms6, int32_t* pcg_iters);
/* CUDA-event time of the per-pass K/B allreduce of a vertex-sharded context
   (timing on), accumulated like the kernel classes of nrr_ctx_stats */
int nrr_ctx_comm_ms(nrr_ctx* ctx, double* out_ms);
int nrr_ctx_enable_timing(nrr_ctx* ctx, int32_t on);

/* host-only probe of the cluster-resident PCG plan for a problem (no device
 * calls): out8 = {ok, cluster size, max rows per CTA, max smem K blocks,
 * max ext rows, smem bytes, smem K blocks total, row entries read from L2} */
int nrr_debug_solver_plan(const nrr_problem_view* p, int32_t num_sms, int64_t smem_limit, int64_t* out8);
/* host-only probe of the PCG plan's partition (no device calls): the solver
 * row order of the graph nodes and the subdomain (one CTA each) boundaries.
 * out3 = {subdomains, CTAs per coarse aggregate, largest subdomain};
 * row_begin has num_sms + 1 entries (the first out3[0] + 1 are written),
 * row_node node_count entries. */
int nrr_debug_pcg_partition(const nrr_problem_view* p, int32_t num_sms, int32_t* out3, int32_t* row_begin,
                            int32_t* row_node);

/* ---- setup (CPU; out of the hot path, the reference's setup API) ---- */
/* edges_from_faces (surface.hpp:49-65); returns edge count, -1 on error */
int nrr_edges_from_faces(const int32_t* faces, int32_t nf, int32_t n, int32_t* out_edges,
                         int32_t cap, int32_t* out_count);
/* knn_edges (surface.hpp:70-94), exact with (distance, index) order */
int nrr_knn_edges(const double* pts, int32_t n, int32_t k, int32_t* out_edges, int32_t cap,
                  int32_t* out_count);
/* limited_geodesic (geodesic.hpp:22-84): vertices with edge-graph distance
   < radius from `source`, ascending index; out arrays may be NULL (count only) */
int nrr_limited_geodesic(const double* pts, int32_t n, const int32_t* edges, int32_t ne, int32_t source,
                         double radius, int32_t* out_idx, double* out_dist, int32_t cap, int32_t* out_count);
/* Surface::finalize_edges mean edge length (surface.hpp:29-45) */
int nrr_avg_edge_length(const double* pts, int32_t n, const int32_t* edges, int32_t ne,
                        double* out);
/* normalize_pair (surface.hpp:125-149), in place; out4 = {scale, cx, cy, cz} */
int nrr_normalize_pair(double* src, int32_t n, double* tgt, int32_t m, double* out4);
/* build_graph (deformation_graph.hpp:157-210) */
typedef struct nrr_graph nrr_graph;
int nrr_build_graph(const double* pts, int32_t n, const int32_t* edges, int32_t ne,
                    double radius, nrr_graph** out);
/* ---- device setup: the same results as nrr_knn_edges /
   nrr_build_graph, bit for bit, computed on the B200 `device` ---- */
int nrr_device_count(int32_t* count);
/* knn_edges on the device; k <= 32 */
int nrr_knn_edges_gpu(int32_t device, const double* pts, int32_t n, int32_t k, int32_t* out_edges,
                      int32_t cap, int32_t* out_count);
/* build_graph on the device; out_rounds (may be NULL) = rounds of the node sweep */
int nrr_build_graph_gpu(int32_t device, const double* pts, int32_t n, const int32_t* edges, int32_t ne,
                        double radius, nrr_graph** out, int32_t* out_rounds);
void nrr_graph_counts(const nrr_graph* g, int32_t* N, int32_t* E, int32_t* sumk, int32_t* P);
void nrr_graph_export(const nrr_graph* g, int32_t* node_indices, double* node_positions,
                      int32_t* edges, int32_t* infl_offsets, int32_t* infl_nodes,
                      double* infl_weights, double* infl_dist, int32_t* reg_pairs,
                      double* reg_weights);
void nrr_graph_free(nrr_graph* g);

/* seeded synthetic inputs standing in for BASELINE.json configs 0-4
 * (SURVEY.md 8(d)); returns a surface pair. Query sizes first with NULL
 * buffers. which: 0 torus, 1 capsule chain, 2 height field 316^2,
 * 3 torus 20K (pair p: seed 4000+p), 4 height field 1000^2. scale in (0,1]
 * shrinks point counts for tests. */
int nrr_synth_config(int32_t which, uint64_t seed, double scale, int32_t* n, int32_t* nf_src,
                     int32_t* m, double* src, int32_t* src_faces, double* tgt);

#ifdef __cplusplus
}
#endif
#endif /* NRR_CUDA_H */
