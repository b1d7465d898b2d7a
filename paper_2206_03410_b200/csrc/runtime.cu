// Host runtime of the B200 hot path: the device context (nrr_ctx) and the
// register_surfaces state machine (reference solver.hpp:180-304) driving the
// sm_100a kernels, plus the device entry points of the C ABI (nrr_cuda.h).
//
// Per accepted pass (one MM iteration) the stream runs:
//   nn -> terms -> energy_reduce -> [host: accept/revert decision]
//   -> assemble -> pcg (cooperative) -> aa_update -> aa_solve -> aa_combine
//   -> deform(+max_disp) -> [host: record / convergence]
// Two small pinned device->host copies per pass carry the energy record and
// the solve status; all vectors stay resident in HBM.
#include <algorithm>
#include <chrono>
#include <exception>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <unordered_map>
#include <mutex>
#include <map>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "device_common.cuh"
#include "kernels.cuh"
#include "nn.cuh"
#include "nrr_cuda.h"
#include "pcg.cuh"
#include "setup_gpu.cuh"
#include "pcg_cluster.cuh"
#include "comm.hpp"

namespace nrr_b200 {
void energy_terms(cudaStream_t s, const nrr_energy_terms_in* in, double* out_w_align, double* out_w_reg,
                  double* out_sums3);  // api_terms.cu
}

namespace nrr_b200 {

namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }

// Process-wide cache of device blocks (per device, by size): contexts are
// created per registration, and cudaMalloc / cudaFree of their ~50 buffers
// (mapping and synchronising) cost more than the setup itself. Blocks return
// to the cache when a buffer is released; every C-ABI call synchronises its
// stream before returning and a context synchronises before it is destroyed,
// so a cached block is never handed out while queued work still uses it.
class BlockCache {
public:
    void* get(size_t bytes) {
        int dev = 0;
        NRR_CUDA_CHECK(cudaGetDevice(&dev));
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto& m = free_[dev];
            auto it = m.lower_bound(bytes);
            if (it != m.end() && it->first <= 2 * bytes + (1 << 20)) {
                void* ptr = it->second;
                sizes_[ptr] = it->first;
                m.erase(it);
                return ptr;
            }
        }
        void* ptr = nullptr;
        const size_t rounded = (bytes + 511) & ~static_cast<size_t>(511);
        NRR_CUDA_CHECK(cudaMalloc(&ptr, rounded));
        std::lock_guard<std::mutex> lk(mu_);
        sizes_[ptr] = rounded;
        devs_[ptr] = dev;
        return ptr;
    }
    void put(void* ptr) {
        std::lock_guard<std::mutex> lk(mu_);
        free_[devs_[ptr]].emplace(sizes_[ptr], ptr);
    }
    size_t capacity(void* ptr) {
        std::lock_guard<std::mutex> lk(mu_);
        return sizes_[ptr];
    }

private:
    std::mutex mu_;
    std::map<int, std::multimap<size_t, void*>> free_;
    std::unordered_map<void*, size_t> sizes_;
    std::unordered_map<void*, int> devs_;
};
BlockCache& block_cache() {
    static BlockCache* c = new BlockCache();  // never destroyed: blocks live until process exit
    return *c;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) block_cache().put(p);
        p = nullptr;
        n = cap = 0;
    }
    void resize(size_t count) {  // grow-only: a context reused for another problem keeps its buffers
        if (count <= cap && p) {
            n = count;
            return;
        }
        release();
        if (count == 0) return;
        p = static_cast<T*>(block_cache().get(count * sizeof(T)));
        n = count;
        cap = block_cache().capacity(p) / sizeof(T);
    }
    void upload(const T* h, size_t count, cudaStream_t s) {
        resize(count);
        if (count) NRR_CUDA_CHECK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void zero(cudaStream_t s) {
        if (n) NRR_CUDA_CHECK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

template <typename T>
struct Pinned {
    T* p = nullptr;
    Pinned() { NRR_CUDA_CHECK(cudaMallocHost(&p, sizeof(T))); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct Params {  // SolverParams (solver.hpp:42-49)
    double nu_a = 0, nu_r = 0, nu_a_min = 0, alpha = 0, beta = 0;
    bool forced_zero = false;
};

// Sliding window of the reference's AndersonWindow (anderson.hpp:50-73),
// vectors on the device, slot bookkeeping on the host.
struct Window {
    int m = 0;
    int hist = 0;     // entries held (<= m+1)
    int newest = -1;  // ring slot of the newest difference column
    std::vector<int> cols;  // slots, newest first
    void reset() {
        hist = 0;
        newest = m > 0 ? m - 1 : -1;
        cols.clear();
    }
    bool extrapolating() const { return m > 0 && hist > 1; }  // anderson.hpp:64
};

// loop state of one registration, so the run can be stepped from the host
struct RunState {
    bool active = false, done = false, stage_open = false;
    nrr_solver_config cfg{};
    std::vector<int> lm_idx;
    std::vector<double> lm_pos;
    Params prm;
    Window win;
    int si = 0, accepted = 0, passes = 0, degenerate_total = 0;
    nrr_stage_record st{};
    double lm_w = 0.0, e_prev = 0.0;
    bool current_is_aa = false;
    std::chrono::steady_clock::time_point t0, t1;
};

}  // namespace nrr_b200

using namespace nrr_b200;

struct nrr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // vertex sharding (comm.hpp): this rank's problem view is its vertex
    // slice; n_global = all ranks' vertices (term weights, median)
    std::unique_ptr<nrr_b200::Collective> comm;  // NCCL or an in-process group (comm.hpp)
    int nranks = 1, rank = 0, n_global = -1;
    cudaStream_t side = nullptr;  // subdomain inverses run beside the coarse setup
    cudaEvent_t fork = nullptr, join = nullptr;
    // side-by-side mode (opt.max_ctas > 0) with NRR_PCG_PRIORITY set: the
    // cooperative PCG grid runs on a greatest-priority stream so its pending
    // CTAs take SMs ahead of the short kernels of the neighbouring contexts as
    // they free (a mitigation candidate for the config-3 hang, DESIGN.md;
    // ~10% slower on config 3, so off by default)
    cudaStream_t pcg_stream = nullptr;
    cudaEvent_t pcg_fork = nullptr;
    int num_sms = 0;
    size_t smem_optin = 0;
    nrr_solve_options opt{1e-13, 20000, 0, 0};
    int64_t launches = 0;
    bool timing = false;

    // ---- target (SpatialIndex)
    BvhHost bvh;
    DevBuf<float4> d_pts, d_lo, d_hi, d_gpts;
    DevBuf<unsigned char> d_bvh_scratch;
    DevBuf<int> d_cell_start;
    DevBuf<unsigned char> d_grid_scratch;
    DevBuf<double> d_tgt;
    BvhView bv{};
    bool has_target = false;

    // ---- problem
    bool has_problem = false;
    int n = 0, N = 0, E = 0, P = 0;
    double src_avg = 0.0;
    std::vector<int> h_row_ptr, h_col;
    std::vector<double> h_src;
    DevBuf<double> d_src, d_infl_w, d_anchor, d_node_pos, d_pair_c;
    std::vector<double> h_anchor;  // sum_a w_a p_a per vertex (energy.hpp:150-161)
    DevBuf<double4> d_infl_f, d_pair_gv, d_cfa, d_cfb;
    DevBuf<double> d_med_sorted;
    DevBuf<unsigned long long> nn_stats;
    DevBuf<int> nn_overflow;  // BVH traversal-stack overflow flag (nn.cu)
    DevBuf<unsigned char> d_med_tmp;
    DevBuf<int> d_edge_of_blk, d_setup_flags, d_skip;
    const int* pcg_skip = nullptr;  // device skip flag for the next solve (speculative pass)
    bool nn_ready = false;          // the next pass's correspondences were queued at the end of the last one
    int sub_age = -1, coarse_age = -1;  // solves since each preconditioner level was built (-1: none valid)
    bool reuse_precond = false;         // only the registration loop may reuse them (one_pass)
    // preconditioner reuse within a stage (one_pass): rebuilt at a stage
    // start, after `refresh` solves (NRR_SUB_REFRESH / NRR_COARSE_REFRESH), or
    // when a solve needs 25% more PCG iterations than the first one after the
    // last rebuild. Measured on config 2: iterations unchanged, -7% per pass.
    int sub_refresh = 64, coarse_refresh = 64;
    bool last_solve_fresh = false;
    // the ages before the latest queued solve: a pass the device reverts skips
    // its solve (and any preconditioner rebuild it asked for), so the host
    // restores them
    int prev_sub_age = -1, prev_coarse_age = -1;
    bool prev_solve_fresh = false;
    int base_iters = 0;
    cudaEvent_t eval_done = nullptr;
    cudaEvent_t end_done = nullptr;
    cudaEvent_t pcg_done = nullptr;  // after each PCG launch (device budget of cooperative grids)
    // the next pass's evaluation (terms, energies, device decision) is queued
    // before the end-of-pass sync, so the GPU works through the host's
    // end-of-pass processing; invalidated when the stage ends
    bool eval_queued = false, eval_nn_ran = false, nn_time_pending = false;
    bool flush_each_pass = false;                 // run_iterate(flush_l2): flush L2 before each queued evaluation
    std::vector<cudaEvent_t> flush_ev;            // pairs around the in-pass flushes (subtracted from the pass time)
    int flush_used = 0;
    DevBuf<long long> d_pair_off;
    DevBuf<unsigned char> d_setup_scratch;
    DevBuf<int> d_infl_off, d_infl_node, d_pairs, d_pair_rev, d_node_pair_off, d_row_ptr, d_col, d_ub_cptr, d_cv,
        d_cea, d_ceb, d_ub_kpos, d_ub_kpos_t, d_edges, d_edge_pab, d_edge_pba, d_lm_vertex;
    DevBuf<double> d_lm_pos;
    DevProblem dp{};

    // ---- per-iteration state
    DevBuf<double> x, xmm, xmm_spec, xnext, vhat, vhat2, d2, q, wa, wr, R, K, B, Z, term_part, pcg_a, pcg_b;
    DevBuf<int> nn_idx, deg, row_begin, d_row_node, d_node_row, d_node_agg, d_colx, d_ext_off, d_ext_node, d_ext_tl, d_touch_off, d_touch_agg;
    DevBuf<double> d_agg_center, coarse_part, coarse_inv, sub_inv;
    PcgPlan plan;
    ClusterPlan cplan;
    bool use_cluster = false;
    DevBuf<int> c_rank_rows, c_row_node, c_ent_ptr, c_diag_ent, c_store_off, c_store_src, c_halo_off;
    DevBuf<int2> c_ent, c_halo_src;
    DevBuf<long long> prof, cta_prof;
    DevBuf<PcgStatus> d_status;
    DevBuf<PassRecord> d_rec;
    Pinned<PassRecord> h_rec, h_rec_end;
    Pinned<PcgStatus> h_status, h_status_init;  // init: constant {no failure}, copied before every solve
    Pinned<int> h_deg;
    // Anderson
    int aa_m = 0;
    size_t aa_dim = 0;
    DevBuf<double> aa_df, aa_dg, aa_fprev, aa_gprev, aa_theta, aa_part;
    DevBuf<int> aa_rank;
    AADevice aa{};

    // ---- report of the last run
    nrr_report_summary summary{};
    std::vector<nrr_stage_record> stages;
    std::vector<nrr_iteration_record> iters;
    std::vector<nrr_pass_record> passes;
    std::vector<int> pass_nn;
    // pass trace (opt.record_passes >= 3, test instrumentation): per evaluated
    // pass the iterate it was evaluated at, its correspondences and energies,
    // and on an accepted pass the solve's x_mm (node-major 12N each)
    std::vector<nrr_pass_trace> trace;
    std::vector<double> trace_x, trace_xmm;
    std::vector<int> trace_nn;

    // ---- timing (CUDA events per kernel class)
    static constexpr int kClasses = 7;  // nn, terms, assembly, pcg, aa, deform, K/B allreduce
    cudaEvent_t ev[kClasses][2] = {};
    double class_ms[kClasses] = {0};
    int pcg_iters_total = 0;
    cudaEvent_t pass_ev[2] = {};
    RunState run;
    size_t l2_bytes = 0;
    DevBuf<double> flush;

    ~nrr_ctx() {
        for (auto& e : ev)
            for (auto& x : e)
                if (x) cudaEventDestroy(x);
        for (auto& x : pass_ev)
            if (x) cudaEventDestroy(x);
        if (fork) cudaEventDestroy(fork);
        if (join) cudaEventDestroy(join);
        if (eval_done) cudaEventDestroy(eval_done);
        if (end_done) cudaEventDestroy(end_done);
        if (pcg_done) {
            nrr_b200::pcg_forget_event(pcg_done);
            cudaEventDestroy(pcg_done);
        }
        for (auto& x : flush_ev) cudaEventDestroy(x);
        if (pcg_fork) cudaEventDestroy(pcg_fork);
        if (pcg_stream) cudaStreamDestroy(pcg_stream);
        if (side) cudaStreamDestroy(side);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace nrr_b200 {
namespace {

enum Cls { kNN = 0, kTerms = 1, kAsm = 2, kPcg = 3, kAA = 4, kDeform = 5, kComm = 6 };

struct ClassTimer {
    nrr_ctx* c;
    int k;
    ClassTimer(nrr_ctx* ctx, int cls) : c(ctx), k(cls) {
        if (c->timing) NRR_CUDA_CHECK(cudaEventRecord(c->ev[k][0], c->stream));
    }
    ~ClassTimer() {
        if (c->timing) cudaEventRecord(c->ev[k][1], c->stream);
    }
};
// after a stream sync: accumulate the elapsed time of every class that ran
void harvest(nrr_ctx* c, const bool ran[nrr_ctx::kClasses]) {
    if (!c->timing) return;
    for (int k = 0; k < nrr_ctx::kClasses; ++k) {
        if (!ran[k]) continue;
        float ms = 0.f;
        // a class whose events were not recorded (timing switched on between
        // a queued evaluation and its harvest) is skipped, and its error
        // cleared so a later launch check does not report it
        if (cudaEventElapsedTime(&ms, c->ev[k][0], c->ev[k][1]) == cudaSuccess) c->class_ms[k] += ms;
        else (void)cudaGetLastError();
    }
}

void sync(nrr_ctx* c) { NRR_CUDA_CHECK(cudaStreamSynchronize(c->stream)); }

void require_target(nrr_ctx* c) {
    if (!c->has_target) throw ConfigError("no target uploaded (nrr_ctx_set_target)");
}
void require_problem(nrr_ctx* c) {
    if (!c->has_problem) throw ConfigError("no problem uploaded (nrr_ctx_set_problem)");
}

void nn_run(nrr_ctx* c, const double* queries, int nq, const int* prev, int* idx, double* d2, double* q,
            const double* anchor) {
    ClassTimer t(c, kNN);
    launch_nn(c->bv, queries, nq, prev, idx, d2, q, anchor, c->stream);
    ++c->launches;
    c->nn_ready = false;
}

void check_nn_overflow(nrr_ctx* c) {
    if (!c->nn_overflow.p) return;
    int ov = 0;
    NRR_CUDA_CHECK(cudaMemcpyAsync(&ov, c->nn_overflow.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    NRR_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    if (ov) throw CudaError("nearest-neighbour traversal stack overflow (the result would be inexact)");
}

// SpatialIndex ctor: the BVH is built on the device (nn.cu build_bvh_device,
// the same bits as BvhHost::build); NRR_BVH_HOST=1 builds it on the host
void set_target(nrr_ctx* c, const double* tgt, int m) {
    if (m <= 0) throw NumericalError("SpatialIndex: cannot index an empty point set");
    c->d_tgt.upload(tgt, static_cast<size_t>(m) * 3, c->stream);
    if (std::getenv("NRR_BVH_HOST")) {
        c->bvh.build(tgt, m);
        c->d_pts.upload(c->bvh.pts.data(), c->bvh.pts.size(), c->stream);
        c->d_lo.upload(c->bvh.box_lo.data(), c->bvh.box_lo.size(), c->stream);
        c->d_hi.upload(c->bvh.box_hi.data(), c->bvh.box_hi.size(), c->stream);
    } else {
        std::vector<int> off, cnt;
        int total = 0;
        bvh_layout(m, off, cnt, total);
        c->d_pts.resize((m + 7) / 8 * 8);
        c->d_lo.resize(total);
        c->d_hi.resize(total);
        c->d_bvh_scratch.resize(bvh_scratch_bytes(m));
        build_bvh_device(c->d_tgt.p, m, c->bvh, c->d_pts.p, c->d_lo.p, c->d_hi.p, c->d_bvh_scratch.p, c->stream);
        c->launches += 6 + static_cast<int>(cnt.size());
    }
    BvhView& b = c->bv;
    b.pts = c->d_pts.p;
    b.box_lo = c->d_lo.p;
    b.box_hi = c->d_hi.p;
    b.tgt64 = c->d_tgt.p;
    b.m = m;
    b.levels = static_cast<int>(c->bvh.level_cnt.size());
    for (int l = 0; l < kMaxLevels; ++l) {
        b.level_off[l] = l < b.levels ? c->bvh.level_off[l] : 0;
        b.level_cnt[l] = l < b.levels ? c->bvh.level_cnt[l] : 0;
    }
    b.cx = c->bvh.center[0];
    b.cy = c->bvh.center[1];
    b.cz = c->bvh.center[2];
    b.half_extent = static_cast<float>(c->bvh.half_extent);
    b.gpts = nullptr;
    b.cell_start = nullptr;
    {  // uniform grid beside the BVH (warm-started queries with a small ball)
        const char* ge = std::getenv("NRR_NN_GRID");
        const char* gh = std::getenv("NRR_NN_GRID_H");
        const GridDims g = (ge && std::atoi(ge) == 0) ? GridDims{}
                                                      : grid_dims(c->bvh.lo, c->bvh.hi, m, gh ? std::atof(gh) : 0.85);
        if (g.nx > 0) {
            const long long ncells = static_cast<long long>(g.nx) * g.ny * g.nz;
            c->d_gpts.resize(m);
            c->d_cell_start.resize(static_cast<size_t>(ncells + 1));
            c->d_grid_scratch.resize(grid_scratch_bytes(m, ncells));
            build_grid(c->d_tgt.p, m, c->bvh.center, c->bvh.lo, g, c->d_gpts.p, c->d_cell_start.p,
                       c->d_grid_scratch.p, c->stream);
            c->launches += 4;
            b.gpts = c->d_gpts.p;
            b.cell_start = c->d_cell_start.p;
            b.gnx = g.nx;
            b.gny = g.ny;
            b.gnz = g.nz;
            b.glx = static_cast<float>(c->bvh.lo[0] - c->bvh.center[0]);
            b.gly = static_cast<float>(c->bvh.lo[1] - c->bvh.center[1]);
            b.glz = static_cast<float>(c->bvh.lo[2] - c->bvh.center[2]);
            b.inv_h = static_cast<float>(1.0 / g.h);
            const char* gc = std::getenv("NRR_NN_GRID_CELLS");
            // cell size factor 0.85 (with the column-run scan: config 2 NN
            // 49 -> 47 us, config 4 594 -> 547 us against 1.0,
            // profiles/r04_nn_grid_sweep.txt) and <= 500 cells per grid-path
            // query (profiles/r02_sweep_nn_c3_b.txt)
            b.gmax_cells = gc ? std::atoi(gc) : 500;
        }
    }
    c->nn_overflow.resize(1);
    c->nn_overflow.zero(c->stream);
    b.overflow = c->nn_overflow.p;
    b.stats = nullptr;
    if (std::getenv("NRR_NN_STATS")) {
        c->nn_stats.resize(4);
        c->nn_stats.zero(c->stream);
        b.stats = c->nn_stats.p;
    }
    c->has_target = true;
}

// SystemAssembler ctor (energy.hpp:139-176) + the B200 assembly plan
struct SetupClock {  // NRR_PROF_SETUP=1: host setup phase timings on stderr
    bool on = std::getenv("NRR_PROF_SETUP") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void lap(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "setup %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

void set_problem(nrr_ctx* c, const nrr_problem_view* p) {
    SetupClock clk;
    const int n = p->n, N = p->node_count, E = p->edge_count, P = p->pair_count;
    if (n < 0 || N < 0 || E < 0 || P < 0) throw ConfigError("negative problem size");
    if (N == 0 && n > 0) throw ConfigError("deformation graph has no nodes");
    cudaStream_t s = c->stream;
    c->n = n;
    c->N = N;
    c->E = E;
    c->P = P;
    c->src_avg = p->src_avg_edge_length;
    c->h_src.assign(p->source, p->source + 3 * static_cast<size_t>(n));
    const int sumk = n > 0 ? p->infl_offsets[n] : 0;
    if (sumk < 0) throw ConfigError("negative influence count");
    // the caller's arrays go to the device on a helper thread while this one
    // builds the plan (pageable copies block the issuing thread); joined before
    // the device setup that reads them, and on any exception
    struct Joiner {
        std::thread t;
        std::exception_ptr err;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
        void join() {
            if (t.joinable()) t.join();
            if (err) std::rethrow_exception(err);
        }
    } uploader;
    uploader.t = std::thread([c, p, n, N, P, sumk, s, &uploader] {
        try {
            NRR_CUDA_CHECK(cudaSetDevice(c->device));
            c->d_src.upload(p->source, 3 * static_cast<size_t>(n), s);
            c->d_infl_off.upload(p->infl_offsets, n + 1, s);
            c->d_infl_node.upload(p->infl_nodes, sumk, s);
            c->d_infl_w.upload(p->infl_weights, sumk, s);
            c->d_node_pos.upload(p->node_positions, 3 * static_cast<size_t>(N), s);
            c->d_pairs.upload(p->reg_pairs, 2 * static_cast<size_t>(P), s);
            c->d_pair_c.upload(p->reg_weights, P, s);
        } catch (...) {
            uploader.err = std::current_exception();
        }
    });
    // BSR pattern: diagonal + both halves of each edge (energy.hpp:264-279)
    // flat CSR by counting (the node itself + both ends of every edge), then
    // each row sorted and deduplicated
    std::vector<int> coff(static_cast<size_t>(N) + 1, 0);
    for (int j = 0; j < N; ++j) coff[j + 1] = 1;
    for (int e = 0; e < E; ++e) {
        const int a = p->edges[2 * e], b = p->edges[2 * e + 1];
        if (a < 0 || b < 0 || a >= N || b >= N || a == b) throw ConfigError("graph edge index out of range");
        ++coff[a + 1];
        ++coff[b + 1];
    }
    for (int j = 0; j < N; ++j) coff[j + 1] += coff[j];
    std::vector<int> cflat(coff[N]), cfill(coff.begin(), coff.end() - 1);
    for (int j = 0; j < N; ++j) cflat[cfill[j]++] = j;
    for (int e = 0; e < E; ++e) {
        const int a = p->edges[2 * e], b = p->edges[2 * e + 1];
        cflat[cfill[a]++] = b;
        cflat[cfill[b]++] = a;
    }
    std::vector<int> deg(N);
    for (int j = 0; j < N; ++j) {
        int* lo = cflat.data() + coff[j];
        int* hi = cflat.data() + coff[j + 1];
        std::sort(lo, hi);
        deg[j] = static_cast<int>(std::unique(lo, hi) - lo);
    }
    clk.lap("pattern");
    // solver row order: bisection + relaxation, one subdomain per CTA (pcg.cu),
    // on a helper thread beside the influence validation below (it only
    // needs the node graph)
    const int sms = c->opt.max_ctas > 0 ? std::min(c->opt.max_ctas, c->num_sms) : c->num_sms;
    Joiner planner;
    if (N > 0)
        planner.t = std::thread([c, p, N, sms, &deg, &coff, &cflat, &planner] {
            try {
                c->plan.build(p->node_positions, deg.data(), N, sms, c->smem_optin, coff.data(), cflat.data());
            } catch (...) {
                planner.err = std::current_exception();
            }
        });
    // influence validation (the constants w [v - p; 1] and sum w p are built
    // on the device, setup_gpu.cu); entries per vertex for the contributor lists
    std::vector<long long> pair_off(static_cast<size_t>(n) + 1, 0);
    {  // validation and per-vertex entry counts on host threads, then the prefix
        const int T = std::max(1, std::min<int>(8, static_cast<int>(std::thread::hardware_concurrency())));
        std::vector<int> bad(T, 0);
        auto part = [&](int t) {
            const int i0 = static_cast<int>(static_cast<long long>(n) * t / T);
            const int i1 = static_cast<int>(static_cast<long long>(n) * (t + 1) / T);
            for (int i = i0; i < i1; ++i) {
                const int k0 = p->infl_offsets[i], k1 = p->infl_offsets[i + 1];
                if (k1 <= k0) {
                    bad[t] |= 1;
                    continue;
                }
                for (int k = k0; k < k1; ++k)
                    if (p->infl_nodes[k] < 0 || p->infl_nodes[k] >= N) bad[t] |= 2;
                const long long kk = k1 - k0;
                pair_off[i + 1] = kk * (kk + 1) / 2;
            }
        };
        std::vector<std::thread> th;
        for (int t = 1; t < T; ++t) th.emplace_back(part, t);
        part(0);
        for (auto& x : th) x.join();
        int b = 0;
        for (int v : bad) b |= v;
        if (b & 1) throw NumericalError("source point without influencing nodes");
        if (b & 2) throw ConfigError("influence node index out of range");
        for (int i = 0; i < n; ++i) pair_off[i + 1] += pair_off[i];
    }
    const long long entries = pair_off[n];
    if (entries >= (1LL << 31)) throw ConfigError("assembly contributor lists exceed 2^31 entries");
    clk.lap("influence constants");
    planner.join();  // solver row order (started above)
    clk.lap("rcb plan (rest)");
    c->h_row_ptr.assign(N + 1, 0);
    c->h_col.clear();
    for (int r = 0; r < N; ++r) {
        const int j = c->plan.row_node[r];
        c->h_row_ptr[r + 1] = c->h_row_ptr[r] + deg[j];
        c->h_col.insert(c->h_col.end(), cflat.begin() + coff[j], cflat.begin() + coff[j] + deg[j]);
    }
    const int nnzb = c->h_row_ptr[N];
    auto find_blk = [&](int a, int b) -> int {
        const int ra = c->plan.node_row[a];
        const auto lo = c->h_col.begin() + c->h_row_ptr[ra], hi = c->h_col.begin() + c->h_row_ptr[ra + 1];
        const auto it = std::lower_bound(lo, hi, b);
        if (it == hi || *it != b) return -1;
        return static_cast<int>(it - c->h_col.begin());
    };
    // edge index per (a<b) block for the contributor lists
    std::vector<int> edge_of_blk(nnzb, -1);
    for (int e = 0; e < E; ++e) {
        const int a = std::min(p->edges[2 * e], p->edges[2 * e + 1]);
        const int b = std::max(p->edges[2 * e], p->edges[2 * e + 1]);
        edge_of_blk[find_blk(a, b)] = e;
    }
    clk.lap("bsr");
    const int U = N + E;
    clk.lap("contributors");
    std::vector<int> kpos(U), kpos_t(U), eab(E), eba(E);
    for (int j = 0; j < N; ++j) kpos[j] = kpos_t[j] = find_blk(j, j);
    // directed pairs: i-major ranges, reverse index
    std::vector<int> npo(N + 1, 0);
    for (int e = 0; e < P; ++e) {
        const int i = p->reg_pairs[2 * e];
        if (i < 0 || i >= N) throw ConfigError("reg pair index out of range");
        if (e > 0 && p->reg_pairs[2 * (e - 1)] > i) throw ConfigError("reg pairs must be i-major");
        ++npo[i + 1];
    }
    for (int j = 0; j < N; ++j) npo[j + 1] += npo[j];
    std::vector<int> rev(P, -1);
    auto pair_index = [&](int i, int j) -> int {
        for (int e = npo[i]; e < npo[i + 1]; ++e)
            if (p->reg_pairs[2 * e + 1] == j) return e;
        return -1;
    };
    {  // reverse pairs and per-edge positions on host threads (independent entries)
        const int T = std::max(1, std::min<int>(8, static_cast<int>(std::thread::hardware_concurrency())));
        std::vector<int> bad(T, 0);
        auto part = [&](int t) {
            for (int e = static_cast<int>(static_cast<long long>(P) * t / T);
                 e < static_cast<int>(static_cast<long long>(P) * (t + 1) / T); ++e) {
                rev[e] = pair_index(p->reg_pairs[2 * e + 1], p->reg_pairs[2 * e]);
                if (rev[e] < 0) bad[t] |= 1;
            }
            for (int e = static_cast<int>(static_cast<long long>(E) * t / T);
                 e < static_cast<int>(static_cast<long long>(E) * (t + 1) / T); ++e) {
                const int a = p->edges[2 * e], b = p->edges[2 * e + 1];
                kpos[N + e] = find_blk(a, b);
                kpos_t[N + e] = find_blk(b, a);
                eab[e] = pair_index(a, b);
                eba[e] = pair_index(b, a);
                if ((eab[e] < 0 || eba[e] < 0) && P > 0) bad[t] |= 2;
            }
        };
        std::vector<std::thread> th;
        for (int t = 1; t < T; ++t) th.emplace_back(part, t);
        part(0);
        for (auto& x : th) x.join();
        int b = 0;
        for (int v : bad) b |= v;
        if (b & 1) throw ConfigError("reg pairs are not symmetric");
        if (b & 2) throw ConfigError("graph edge without reg pairs");
    }
    if (P == 0 && E > 0) throw ConfigError("graph edges without reg pairs");
    clk.lap("pairs");
    // upload (the caller's arrays: on the helper thread)
    uploader.join();
    c->d_infl_f.resize(std::max(sumk, 1));
    c->d_anchor.resize(std::max<size_t>(3 * static_cast<size_t>(n), 1));
    c->h_anchor.clear();  // downloaded on demand (nrr_assemble)
    c->d_pair_rev.upload(rev.data(), P, s);
    {  // g_e = c [p_i - p_j; 1] per directed pair (energy.hpp:163-173)
        std::vector<double4> gv(std::max(P, 1));
        for (int e = 0; e < P; ++e) {
            const int i = p->reg_pairs[2 * e], j = p->reg_pairs[2 * e + 1];
            const double cc = p->reg_weights[e];
            const double* pi = p->node_positions + 3 * i;
            const double* pj = p->node_positions + 3 * j;
            gv[e] = make_double4(cc * (pi[0] - pj[0]), cc * (pi[1] - pj[1]), cc * (pi[2] - pj[2]), cc);
        }
        c->d_pair_gv.upload(gv.data(), gv.size(), s);
    }
    c->d_node_pair_off.upload(npo.data(), N + 1, s);
    c->d_row_ptr.upload(c->h_row_ptr.data(), N + 1, s);
    c->d_col.upload(c->h_col.data(), nnzb, s);
    {  // contributor lists and influence constants on the device
        c->d_node_row.upload(c->plan.node_row.data(), N, s);
        c->d_edge_of_blk.upload(edge_of_blk.data(), nnzb, s);
        c->d_pair_off.upload(pair_off.data(), pair_off.size(), s);
        c->d_ub_cptr.resize(U + 1);
        for (auto* b : {&c->d_cv, &c->d_cea, &c->d_ceb}) b->resize(std::max<long long>(entries, 1));
        for (auto* b : {&c->d_cfa, &c->d_cfb}) b->resize(std::max<long long>(entries, 1));
        c->d_setup_flags.resize(1);
        c->d_setup_scratch.resize(setup_gpu_scratch_bytes(entries, U));
        SetupGpuIn in;
        in.n = n;
        in.N = N;
        in.U = U;
        in.infl_off = c->d_infl_off.p;
        in.infl_node = c->d_infl_node.p;
        in.infl_w = c->d_infl_w.p;
        in.src = c->d_src.p;
        in.node_pos = c->d_node_pos.p;
        in.node_row = c->d_node_row.p;
        in.row_ptr = c->d_row_ptr.p;
        in.col = c->d_col.p;
        in.edge_of_blk = c->d_edge_of_blk.p;
        in.pair_off = c->d_pair_off.p;
        SetupGpuOut out;
        out.infl_f = c->d_infl_f.p;
        out.anchor = c->d_anchor.p;
        out.cptr = c->d_ub_cptr.p;
        out.cv = c->d_cv.p;
        out.cea = c->d_cea.p;
        out.ceb = c->d_ceb.p;
        out.cfa = c->d_cfa.p;
        out.cfb = c->d_cfb.p;
        out.flags = c->d_setup_flags.p;
        build_setup_gpu(in, entries, out, c->d_setup_scratch.p, s);
        c->launches += 4;
    }
    c->d_ub_kpos.upload(kpos.data(), U, s);
    c->d_ub_kpos_t.upload(kpos_t.data(), U, s);
    c->d_edges.upload(p->edges, 2 * static_cast<size_t>(E), s);
    c->d_edge_pab.upload(eab.data(), E, s);
    c->d_edge_pba.upload(eba.data(), E, s);
    DevProblem& d = c->dp;
    d = DevProblem{};
    d.n = n;
    d.N = N;
    d.E = E;
    d.P = P;
    d.U = U;
    d.nnzb = nnzb;
    d.src = c->d_src.p;
    d.infl_off = c->d_infl_off.p;
    d.infl_node = c->d_infl_node.p;
    d.infl_w = c->d_infl_w.p;
    d.infl_f = c->d_infl_f.p;
    d.anchor = c->d_anchor.p;
    d.node_pos = c->d_node_pos.p;
    d.pairs = c->d_pairs.p;
    d.pair_c = c->d_pair_c.p;
    d.pair_rev = c->d_pair_rev.p;
    d.pair_gv = c->d_pair_gv.p;
    d.node_pair_off = c->d_node_pair_off.p;
    d.row_ptr = c->d_row_ptr.p;
    d.col = c->d_col.p;
    d.ub_cptr = c->d_ub_cptr.p;
    d.c_v = c->d_cv.p;
    d.c_ea = c->d_cea.p;
    d.c_eb = c->d_ceb.p;
    d.c_fa = c->d_cfa.p;
    d.c_fb = c->d_cfb.p;
    d.ub_kpos = c->d_ub_kpos.p;
    d.ub_kpos_t = c->d_ub_kpos_t.p;
    d.edges = c->d_edges.p;
    d.edge_pab = c->d_edge_pab.p;
    d.edge_pba = c->d_edge_pba.p;
    // state buffers
    const size_t D = 12 * static_cast<size_t>(N);
    for (auto* b : {&c->x, &c->xmm, &c->xmm_spec, &c->xnext, &c->B}) b->resize(std::max<size_t>(D, 1));
    c->Z.resize(3 * std::max<size_t>(D, 1));  // + the PCG's search-direction scratch (PcgArgs::P)
    c->Z.zero(s);  // two parities (pcg.cu: exchanged vector, see PcgArgs::z_stride)
    c->d_skip.resize(1);
    for (auto* b : {&c->vhat, &c->vhat2, &c->q}) b->resize(std::max<size_t>(3 * static_cast<size_t>(n), 1));
    c->d2.resize(std::max(n, 1));
    c->wa.resize(std::max(n, 1));
    c->nn_idx.resize(std::max(n, 1));
    c->wr.resize(std::max(P, 1));
    c->R.resize(std::max<size_t>(9 * static_cast<size_t>(N), 1));
    c->K.resize(std::max<size_t>(16 * static_cast<size_t>(nnzb), 1));
    c->term_part.resize(3 * kTermBlocks);
    c->deg.resize(1);
    c->d_rec.resize(1);
    c->d_status.resize(1);
    clk.lap("uploads");
    if (N > 0) {
        // the kernels' static shared memory (<= 1 KB) comes out of the same opt-in budget
        c->plan.size_smem(c->h_row_ptr.data(), c->h_col.data(), c->smem_optin - 1024);
        clk.lap("pcg smem plan");
        if (clk.on) {
            const PcgPlan& pl = c->plan;
            std::fprintf(stderr,
                         "pcg plan: grid %d max_rows %d ept %d sub_rows %d chunks %d n_agg %d max_touch %d max_ext %d "
                         "max_kb %d k_in_smem %d smem %zu coarse %d\n",
                         pl.grid, pl.max_rows, pl.ept, pl.sub_rows, pl.sub_chunks, pl.n_agg, pl.max_touch, pl.max_ext,
                         pl.max_kb, pl.k_in_smem ? 1 : 0, pl.smem_bytes, pl.use_coarse ? 1 : 0);
        }
        c->d_colx.upload(c->plan.colx.data(), c->plan.colx.size(), s);
        c->d_ext_off.upload(c->plan.ext_off.data(), c->plan.ext_off.size(), s);
        c->d_ext_node.upload(c->plan.ext_node.data(), c->plan.ext_node.size(), s);
        c->d_ext_tl.upload(c->plan.ext_tl.data(), c->plan.ext_tl.size(), s);
        c->d_touch_off.upload(c->plan.touch_off.data(), c->plan.touch_off.size(), s);
        c->d_touch_agg.upload(c->plan.touch_agg.data(), c->plan.touch_agg.size(), s);
        c->row_begin.upload(c->plan.row_begin.data(), c->plan.row_begin.size(), s);
        c->d_row_node.upload(c->plan.row_node.data(), N, s);
        c->d_node_agg.upload(c->plan.node_agg.data(), N, s);
        c->d_agg_center.upload(c->plan.agg_center.data(), c->plan.agg_center.size(), s);
        const size_t nc = 4 * static_cast<size_t>(c->plan.n_agg);
        c->coarse_part.resize(static_cast<size_t>(c->plan.grid) * 4 * nc);
        c->coarse_inv.resize(nc * nc);
        c->sub_inv.resize(static_cast<size_t>(c->plan.grid) * c->plan.sub_chunks * 4 * c->plan.sub_rows *
                          c->plan.sub_ld);
        // kPartReplicas copies, two parities (PcgArgs::part_stride)
        c->pcg_a.resize(2 * 8 * kPcgSlots * static_cast<size_t>((c->plan.grid + 7) & ~7));
        c->pcg_a.zero(s);  // slot rows are padded to a multiple of 8 CTAs: the padding stays 0
        c->pcg_b.resize(kPcgSlots * static_cast<size_t>(c->plan.grid));
        d.node_row = c->d_node_row.p;
        // cluster-resident solver (opt-in) when the graph fits one cluster's shared memory
        const char* mode = std::getenv("NRR_PCG");
        c->use_cluster = false;
        if (mode && std::string(mode) == "cluster") {
            c->cplan.build(p->node_positions, c->h_row_ptr.data(), c->h_col.data(), c->plan.node_row.data(), N,
                           c->smem_optin, 16);
            c->use_cluster = c->cplan.ok;
        }
        if (c->use_cluster) {
            const ClusterPlan& cp = c->cplan;
            c->c_rank_rows.upload(cp.rank_rows.data(), cp.rank_rows.size(), s);
            c->c_row_node.upload(cp.row_node.data(), cp.row_node.size(), s);
            c->c_ent_ptr.upload(cp.ent_ptr.data(), cp.ent_ptr.size(), s);
            c->c_ent.upload(cp.ent.data(), cp.ent.size(), s);
            c->c_diag_ent.upload(cp.diag_ent.data(), cp.diag_ent.size(), s);
            c->c_store_off.upload(cp.store_off.data(), cp.store_off.size(), s);
            c->c_store_src.resize(std::max<size_t>(cp.store_src.size(), 1));
            if (!cp.store_src.empty()) c->c_store_src.upload(cp.store_src.data(), cp.store_src.size(), s);
            c->c_halo_off.upload(cp.halo_off.data(), cp.halo_off.size(), s);
            c->c_halo_src.resize(std::max<size_t>(cp.halo_src.size(), 1));
            if (!cp.halo_src.empty()) c->c_halo_src.upload(cp.halo_src.data(), cp.halo_src.size(), s);
        }
    }
    NRR_CUDA_CHECK(cudaStreamSynchronize(s));
    clk.lap("pcg uploads + sync");
    int flags = 0;
    NRR_CUDA_CHECK(cudaMemcpy(&flags, c->d_setup_flags.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (flags & 1) throw NumericalError("assemble: co-influencing node pair is not a graph edge");
    c->has_problem = true;
    c->sub_age = c->coarse_age = -1;
    if (const char* e = std::getenv("NRR_SUB_REFRESH")) c->sub_refresh = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("NRR_COARSE_REFRESH")) c->coarse_refresh = std::max(1, std::atoi(e));
}

void ensure_aa(nrr_ctx* c, int m, size_t D) {
    if (m > kMaxAA) throw ConfigError("aa_window above the device limit of 16");
    const int mm = std::max(m, 1);
    if (c->aa_m != mm || c->aa_dim != D) {
        c->aa_df.resize(mm * D);
        c->aa_dg.resize(mm * D);
        c->aa_fprev.resize(D);
        c->aa_gprev.resize(D);
        c->aa_theta.resize(kMaxAA);
        c->aa_part.resize(static_cast<size_t>(kTriMax) * kTermBlocks);
        c->aa_rank.resize(1);
        c->aa_m = mm;
        c->aa_dim = D;
    }
    c->aa.df = c->aa_df.p;
    c->aa.dg = c->aa_dg.p;
    c->aa.fprev = c->aa_fprev.p;
    c->aa.gprev = c->aa_gprev.p;
    c->aa.theta = c->aa_theta.p;
    c->aa.partials = c->aa_part.p;
    c->aa.rank = c->aa_rank.p;
}

SlotList to_slots(const std::vector<int>& v) {
    SlotList s{};
    s.n = static_cast<int>(v.size());
    for (int k = 0; k < s.n; ++k) s.s[k] = v[k];
    return s;
}

// push (g, f = g - x) and combine into x_next (anderson.hpp:22-46)
void aa_push_combine(nrr_ctx* c, Window& w, const double* g, const double* x, const double* f, double* x_next,
                     int D) {
    ClassTimer t(c, kAA);
    const int have_prev = w.hist >= 1 && w.m > 0;
    int slot = -1;
    if (have_prev) {
        slot = (w.newest + 1) % w.m;
        w.newest = slot;
        w.cols.insert(w.cols.begin(), slot);
        if (static_cast<int>(w.cols.size()) > w.m) w.cols.pop_back();
    }
    w.hist = std::min(w.hist + 1, w.m + 1);
    const SlotList cols = to_slots(w.cols);
    const int mk = std::min(w.hist - 1, w.m);
    if (mk <= 0) {
        launch_aa_update(c->aa, g, x, f, D, have_prev, slot < 0 ? 0 : slot, c->stream);
        ++c->launches;
        NRR_CUDA_CHECK(cudaMemcpyAsync(x_next, g, sizeof(double) * D, cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    launch_aa_push_solve(c->aa, g, x, f, D, have_prev, slot < 0 ? 0 : slot, cols, c->stream);
    launch_aa_combine(c->aa, D, cols, x_next, &c->d_rec.p->nonfinite, c->stream);
    c->launches += 3;
}

void validate(const nrr_solver_config& cfg) {  // solver.hpp:32-38
    if (!(cfg.eps > 0.0)) throw ConfigError("eps must be positive");
    if (cfg.i_max < 1) throw ConfigError("i_max must be at least 1");
    if (cfg.aa_window < 0) throw ConfigError("aa_window must be >= 0");
    if (cfg.k_alpha < 0.0 || cfg.k_beta < 0.0) throw ConfigError("k_alpha and k_beta must be non-negative");
}

// ---- vertex sharding collectives (no-ops on an unsharded context)
int n_total(const nrr_ctx* c) { return c->n_global >= 0 ? c->n_global : c->n; }

void allreduce(nrr_ctx* c, void* buf, size_t count, ncclDataType_t t, ncclRedOp_t op) {
    if (!c->comm) return;
    c->comm->allreduce(buf, count, t, op, c->stream);
}

// after the terms: the node terms (reg, rot) exist on rank 0 only, then the
// five energy sums are added over ranks
void reduce_energies(nrr_ctx* c) {
    if (!c->comm) return;
    if (c->rank > 0) NRR_CUDA_CHECK(cudaMemsetAsync(&c->d_rec.p->reg, 0, 2 * sizeof(double), c->stream));
    allreduce(c, &c->d_rec.p->align, 5, ncclFloat64, ncclSum);
}

// node-level terms (regularisation, rotation, beta) are assembled on rank 0 only
TermParams local_terms(const nrr_ctx* c, TermParams tp) {
    if (c->comm && c->rank > 0) {
        tp.alpha = 0.0;
        tp.beta = 0.0;
    }
    return tp;
}

void update_term_weights(Params& p, int n, int E, int N, const nrr_solver_config& cfg) {  // solver.hpp:68-80
    if (E == 0) {
        p.alpha = 0.0;
        p.forced_zero = true;
    } else {
        p.alpha = cfg.k_alpha * (static_cast<double>(n) / E) * (p.nu_r * p.nu_r) / (p.nu_a * p.nu_a);
    }
    p.beta = cfg.k_beta * (static_cast<double>(n) / N) / (2.0 * p.nu_a * p.nu_a);
}

Params init_parameters(nrr_ctx* c, const nrr_solver_config& cfg) {  // solver.hpp:86-106
    require_target(c);
    require_problem(c);
    const int n = c->n;
    nn_run(c, c->d_src.p, n, nullptr, c->nn_idx.p, c->d2.p, nullptr, nullptr);
    std::vector<double> dist;
    if (c->comm) {  // all ranks' distances: gather padded slices (padding = NaN, dropped)
        int mx = n;
        DevBuf<int> dm;
        dm.upload(&mx, 1, c->stream);
        allreduce(c, dm.p, 1, ncclInt32, ncclMax);
        NRR_CUDA_CHECK(cudaMemcpyAsync(&mx, dm.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        sync(c);
        DevBuf<double> pad, all;
        pad.resize(std::max(mx, 1));
        const double qnan = std::numeric_limits<double>::quiet_NaN();
        std::vector<double> hpad(std::max(mx, 1), qnan);
        NRR_CUDA_CHECK(cudaMemcpyAsync(pad.p, hpad.data(), sizeof(double) * hpad.size(), cudaMemcpyHostToDevice, c->stream));
        NRR_CUDA_CHECK(cudaMemcpyAsync(pad.p, c->d2.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
        all.resize(static_cast<size_t>(std::max(mx, 1)) * c->nranks);
        c->comm->allgather(pad.p, all.p, std::max(mx, 1), ncclFloat64, c->stream);
        std::vector<double> h(all.n);
        NRR_CUDA_CHECK(cudaMemcpyAsync(h.data(), all.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c->stream));
        sync(c);
        dist.clear();
        for (double v : h)
            if (!std::isnan(v)) dist.push_back(v);
        if (static_cast<int>(dist.size()) != n_total(c)) throw ConfigError("sharded vertex counts do not add up");
    }
    double median = 0.0;
    if (c->comm) {
        for (auto& d : dist) d = std::sqrt(d);
        const int n_med = static_cast<int>(dist.size());
        if (n_med > 0) {  // the sorted-order median (solver.hpp:92-100) by selection
            std::nth_element(dist.begin(), dist.begin() + n_med / 2, dist.end());
            const double hi = dist[n_med / 2];
            median = n_med % 2 == 1 ? hi : 0.5 * (*std::max_element(dist.begin(), dist.begin() + n_med / 2) + hi);
        }
    } else if (n > 0) {
        // the same median on the device: radix-sort the squared distances
        // (sqrt is monotone, so the middle elements are the same) and read
        // back the two middle values only
        size_t tb = 0;
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tb, static_cast<const double*>(nullptr),
                                                      static_cast<double*>(nullptr), n));
        c->d_med_sorted.resize(n);
        c->d_med_tmp.resize(tb);
        NRR_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(c->d_med_tmp.p, tb, c->d2.p, c->d_med_sorted.p, n, 0, 64,
                                                      c->stream));
        double mid[2] = {0.0, 0.0};
        const int lo = n % 2 == 1 ? n / 2 : n / 2 - 1;
        NRR_CUDA_CHECK(cudaMemcpyAsync(mid, c->d_med_sorted.p + lo, sizeof(double) * (n % 2 == 1 ? 1 : 2),
                                       cudaMemcpyDeviceToHost, c->stream));
        sync(c);
        median = n % 2 == 1 ? std::sqrt(mid[0]) : 0.5 * (std::sqrt(mid[0]) + std::sqrt(mid[1]));
    }
    Params p;
    const double l_bar = c->src_avg;
    p.nu_a_min = std::isnan(cfg.nu_a_min) ? l_bar / std::sqrt(3.0) : cfg.nu_a_min;
    p.nu_a = std::isnan(cfg.nu_a_init) ? std::max(median, p.nu_a_min) : cfg.nu_a_init;
    p.nu_r = std::isnan(cfg.nu_r_init) ? 3.0 * l_bar : cfg.nu_r_init;
    if (!(p.nu_a > 0.0) || !(p.nu_r > 0.0)) throw NumericalError("init_parameters: Welsch parameters must be positive");
    update_term_weights(p, n_total(c), c->E, c->N, cfg);
    return p;
}

void upload_landmarks(nrr_ctx* c, const nrr_solver_config& cfg) {
    const int L = cfg.landmark_count;
    for (int l = 0; l < L; ++l)
        if (cfg.landmark_index[l] < 0 || cfg.landmark_index[l] >= c->n)
            throw ConfigError("landmark source index out of range");
    c->dp.landmarks = L;
    if (L > 0) {
        c->d_lm_vertex.upload(cfg.landmark_index, L, c->stream);
        c->d_lm_pos.upload(cfg.landmark_pos, 3 * static_cast<size_t>(L), c->stream);
        c->dp.lm_vertex = c->d_lm_vertex.p;
        c->dp.lm_pos = c->d_lm_pos.p;
    }
}

void set_identity(nrr_ctx* c, double* x) {
    std::vector<double> h(12 * static_cast<size_t>(c->N), 0.0);
    for (int j = 0; j < c->N; ++j)
        for (int r = 0; r < 3; ++r) h[12 * j + 3 * r + r] = 1.0;
    NRR_CUDA_CHECK(cudaMemcpyAsync(x, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, c->stream));
    sync(c);  // h is stack memory
}

void deform_run(nrr_ctx* c, const double* x, double* out, const double* old, double* max_disp) {
    ClassTimer t(c, kDeform);
    launch_deform(c->dp, x, out, old, max_disp, &c->d_rec.p->nonfinite, c->stream);
    ++c->launches;
}

// evaluate the pass at (x, vhat): correspondences, weights, energies
void evaluate(nrr_ctx* c, const double* x, const double* vhat, const TermParams& tp, bool warm) {
    if (!(warm && c->nn_ready)) nn_run(c, vhat, c->n, warm ? c->nn_idx.p : nullptr, c->nn_idx.p, c->d2.p, c->q.p, c->d_anchor.p);
    c->nn_ready = false;
    ClassTimer t(c, kTerms);
    NRR_CUDA_CHECK(cudaMemsetAsync(c->deg.p, 0, sizeof(int), c->stream));
    launch_terms(c->dp, x, c->d2.p, tp, c->wa.p, c->wr.p, c->R.p, c->term_part.p, c->deg.p, c->stream);
    launch_energy_reduce(c->dp, c->term_part.p, tp, vhat, c->d_rec.p, c->stream);
    c->launches += 2;
}

void assemble(nrr_ctx* c, const TermParams& tp) {
    ClassTimer t(c, kAsm);
    launch_assemble(c->dp, c->wa.p, c->q.p, c->wr.p, c->R.p, tp, c->K.p, c->B.p, c->stream);
    c->launches += (tp.lm_weight != 0.0 && c->dp.landmarks > 0) ? 2 : 1;
}

// PCG solve of the system in c->K / c->B (solver-row order), warm start x0
void solve(nrr_ctx* c, const double* x0, double* xout) {
    ClassTimer t(c, kPcg);
    if (xout != x0)
        NRR_CUDA_CHECK(cudaMemcpyAsync(xout, x0, sizeof(double) * 12 * c->N, cudaMemcpyDeviceToDevice, c->stream));
    *c->h_status_init.p = PcgStatus{0x7fffffff, 0, 0, 0, 0.0};  // pinned: the copy stays asynchronous
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->d_status.p, c->h_status_init.p, sizeof(PcgStatus), cudaMemcpyHostToDevice,
                                   c->stream));
    PcgArgs a{};
    a.row_ptr = c->d_row_ptr.p;
    a.col = c->d_col.p;
    a.row_node = c->d_row_node.p;
    a.colx = c->d_colx.p;
    a.ext_off = c->d_ext_off.p;
    a.ext_node = c->d_ext_node.p;
    a.ext_tl = c->d_ext_tl.p;
    a.touch_off = c->d_touch_off.p;
    a.touch_agg = c->d_touch_agg.p;
    a.skip = c->pcg_skip;
    a.K = c->K.p;
    a.B = c->B.p;
    a.X = xout;
    a.Z = c->Z.p;
    a.P = c->Z.p + 2 * std::max<size_t>(12 * static_cast<size_t>(c->N), 1);
    a.z_stride = std::max<size_t>(12 * static_cast<size_t>(c->N), 1);
    a.part_stride = 8 * kPcgSlots * static_cast<size_t>((c->plan.grid + 7) & ~7);
    a.row_begin = c->row_begin.p;
    a.node_pos = c->d_node_pos.p;
    a.agg_center = c->d_agg_center.p;
    a.node_agg = c->d_node_agg.p;
    a.coarse_inv = c->coarse_inv.p;
    a.sub_inv = c->sub_inv.p;
    a.part_a = c->pcg_a.p;
    a.part_b = c->pcg_b.p;
    a.status = c->d_status.p;
    a.rtol = c->opt.pcg_rtol;
    {
        const char* tf = std::getenv("NRR_PCG_TRUE_FACTOR");
        a.true_factor = tf ? std::atof(tf) : 100.0;
    }
    a.max_iter = c->opt.pcg_max_iter;
    a.agg_ctas = c->plan.agg_ctas;
    a.n_agg = c->plan.n_agg;
    a.use_coarse = c->plan.use_coarse ? 1 : 0;
    if (c->use_cluster) {
        ClusterArgs ca{};
        ca.plan = ClusterPlanDev{c->c_rank_rows.p, c->c_row_node.p, c->c_ent_ptr.p, c->c_ent.p, c->c_diag_ent.p,
                                 c->c_store_off.p, c->c_store_src.p, c->c_halo_off.p, c->c_halo_src.p};
        ca.K = c->K.p;
        ca.B = c->B.p;
        ca.X = xout;
        ca.status = c->d_status.p;
        ca.rtol = c->opt.pcg_rtol;
        ca.max_iter = c->opt.pcg_max_iter;
        if (std::getenv("NRR_PROF")) {
            if (c->prof.n == 0) {
                c->prof.resize(32);
                c->prof.zero(c->stream);
            }
            ca.prof = c->prof.p;
        }
        launch_pcg_cluster(c->cplan, ca, c->stream);
        ++c->launches;
        return;
    }
    if (std::getenv("NRR_PROF")) {
        if (c->prof.n == 0) {
            c->prof.resize(32);
            c->prof.zero(c->stream);
        }
        a.prof = c->prof.p;
        if (c->cta_prof.n == 0) {
            c->cta_prof.resize(4 * static_cast<size_t>(c->plan.grid));
            c->cta_prof.zero(c->stream);
        }
        a.cta_prof = c->cta_prof.p;
    }
    // the subdomain inverses and the coarse operator both depend on K only:
    // run them side by side (one CTA per SM for the former, one CTA for the
    // latter's inversion). Any SPD M keeps PCG exact, so a solve may reuse the
    // preconditioner built from an earlier K of the same stage
    // (precond_refresh passes; 1 = rebuild every solve)
    const bool fresh_sub = !c->reuse_precond || c->sub_age < 0 || c->sub_age >= c->sub_refresh;
    const bool fresh_coarse = !c->reuse_precond || c->coarse_age < 0 || c->coarse_age >= c->coarse_refresh;
    c->prev_sub_age = c->sub_age;
    c->prev_coarse_age = c->coarse_age;
    c->prev_solve_fresh = c->last_solve_fresh;
    c->sub_age = fresh_sub ? 1 : c->sub_age + 1;
    c->coarse_age = fresh_coarse ? 1 : c->coarse_age + 1;
    c->last_solve_fresh = fresh_sub && fresh_coarse;
    if (fresh_sub) {
        NRR_CUDA_CHECK(cudaEventRecord(c->fork, c->stream));
        NRR_CUDA_CHECK(cudaStreamWaitEvent(c->side, c->fork, 0));
        launch_sub_invert(c->plan, a, c->sub_inv.p, std::getenv("NRR_SERIAL_SETUP") ? c->stream : c->side);
        NRR_CUDA_CHECK(cudaEventRecord(c->join, c->side));
        ++c->launches;
    }
    if (c->plan.use_coarse && fresh_coarse) {
        launch_coarse_setup(c->plan, a, CoarseWork{c->coarse_part.p, c->coarse_inv.p}, c->stream);
        c->launches += 2;
    }
    if (c->opt.max_ctas > 0 && std::getenv("NRR_PCG_PRIORITY")) {
        if (!c->pcg_stream) {
            int lo = 0, hi = 0;
            NRR_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            NRR_CUDA_CHECK(cudaStreamCreateWithPriority(&c->pcg_stream, cudaStreamNonBlocking, hi));
            NRR_CUDA_CHECK(cudaEventCreateWithFlags(&c->pcg_fork, cudaEventDisableTiming));
        }
        NRR_CUDA_CHECK(cudaEventRecord(c->pcg_fork, c->stream));
        NRR_CUDA_CHECK(cudaStreamWaitEvent(c->pcg_stream, c->pcg_fork, 0));
        if (fresh_sub) NRR_CUDA_CHECK(cudaStreamWaitEvent(c->pcg_stream, c->join, 0));
        launch_pcg(c->plan, a, c->pcg_stream, c->pcg_done);
        NRR_CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->pcg_done, 0));
    } else {
        if (fresh_sub) NRR_CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->join, 0));
        launch_pcg(c->plan, a, c->stream, c->pcg_done);
    }
    ++c->launches;
}

void assemble_solve(nrr_ctx* c, const TermParams& tp, const double* x0, double* xout) {
    assemble(c, tp);
    solve(c, x0, xout);
}

void check_pcg(nrr_ctx* c, const PcgStatus& st) {
    if (st.fail_node != 0x7fffffff)
        throw NumericalError("linear system not positive definite (singular diagonal block at node " +
                             std::to_string(st.fail_node) + ")");
    if (st.code == 2)
        throw NumericalError("linear system not positive definite (indefinite coupling between node blocks)");
    if (st.code != 1) throw NumericalError("linear solve residual above tolerance");
}

// ---- resumable register_surfaces state machine (solver.hpp:180-304) ----
void run_begin(nrr_ctx* c, const nrr_solver_config& cfg_in) {
    validate(cfg_in);
    require_target(c);
    require_problem(c);
    if (c->n == 0 || c->bv.m == 0) throw NumericalError("register_surfaces: empty surface");
    RunState& r = c->run;
    r = RunState{};
    c->nn_ready = false;
    c->eval_queued = false;
    r.t0 = std::chrono::steady_clock::now();
    r.cfg = cfg_in;
    r.lm_idx.assign(cfg_in.landmark_index, cfg_in.landmark_index + cfg_in.landmark_count);
    r.lm_pos.assign(cfg_in.landmark_pos, cfg_in.landmark_pos + 3 * cfg_in.landmark_count);
    r.cfg.landmark_index = r.lm_idx.data();
    r.cfg.landmark_pos = r.lm_pos.data();
    for (double& v : c->class_ms) v = 0.0;
    c->pcg_iters_total = 0;
    c->stages.clear();
    c->iters.clear();
    c->passes.clear();
    c->pass_nn.clear();
    c->trace.clear();
    c->trace_x.clear();
    c->trace_xmm.clear();
    c->trace_nn.clear();
    if (c->comm && r.cfg.landmark_count > 0) throw ConfigError("landmarks are not supported on a vertex-sharded run");
    upload_landmarks(c, r.cfg);
    r.prm = init_parameters(c, r.cfg);
    ensure_aa(c, r.cfg.aa_window, 12 * c->N);
    r.win.m = r.cfg.aa_window;
    set_identity(c, c->x.p);
    NRR_CUDA_CHECK(cudaMemsetAsync(c->d_rec.p, 0, sizeof(PassRecord), c->stream));
    deform_run(c, c->x.p, c->vhat.p, nullptr, nullptr);
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->xmm.p, c->x.p, sizeof(double) * 12 * c->N, cudaMemcpyDeviceToDevice, c->stream));
    sync(c);
    r.t1 = std::chrono::steady_clock::now();
    r.active = true;
}

void open_stage(nrr_ctx* c) {
    RunState& r = c->run;
    r.st = nrr_stage_record{r.prm.nu_a, r.prm.nu_r, r.prm.alpha, r.prm.beta, 0, 0,
                            static_cast<int32_t>(c->iters.size()), 0};
    r.lm_w = (r.si == 0 && r.cfg.landmark_count > 0) ? 1.0 : 0.0;
    r.win.reset();
    c->sub_age = c->coarse_age = -1;  // weights change at a stage boundary: rebuild the preconditioner
    r.e_prev = std::numeric_limits<double>::infinity();
    r.accepted = 0;
    r.passes = 0;
    r.stage_open = true;
}

void close_stage(nrr_ctx* c) {
    RunState& r = c->run;
    c->stages.push_back(r.st);
    r.stage_open = false;
    ++r.si;
    if (r.prm.nu_a == r.prm.nu_a_min) {  // anneal (solver.hpp:60-64, 292-293)
        r.done = true;
        return;
    }
    r.prm.nu_a = std::max(r.prm.nu_a / 2.0, r.prm.nu_a_min);
    r.prm.nu_r = std::max(r.prm.nu_r / 2.0, r.cfg.nu_r_floor);
    update_term_weights(r.prm, n_total(c), c->E, c->N, r.cfg);
}

// Evaluation of a pass at (x, vhat): correspondences (unless queued), terms,
// energies, the device-side safeguard decision (solver.hpp:239) and the
// record for the host; eval_done marks its end.
void queue_eval(nrr_ctx* c, const TermParams& tp, const double* x, const double* vhat) {
    RunState& r = c->run;
    NRR_CUDA_CHECK(cudaMemsetAsync(c->d_rec.p, 0, sizeof(PassRecord), c->stream));
    // warm start from the previous pass's correspondences (init NN at the first pass)
    c->eval_nn_ran = !c->nn_ready;
    evaluate(c, x, vhat, tp, true);
    reduce_energies(c);
    // the safeguard decision is also taken on the device, so the assembly and
    // the solve are queued right behind the evaluation and the host's
    // decision latency hides behind them; on a revert they return at once
    launch_pass_decision(c->d_rec.p, r.e_prev, r.current_is_aa ? 1 : 0, r.lm_w, c->d_skip.p, c->stream);
    ++c->launches;
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->h_rec.p, c->d_rec.p, sizeof(PassRecord), cudaMemcpyDeviceToHost, c->stream));
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->h_deg.p, c->deg.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (c->opt.record_passes == 2) {
        c->pass_nn.resize(c->pass_nn.size() + c->n);
        NRR_CUDA_CHECK(cudaMemcpyAsync(c->pass_nn.data() + c->pass_nn.size() - c->n, c->nn_idx.p,
                                       sizeof(int) * c->n, cudaMemcpyDeviceToHost, c->stream));
    }
    NRR_CUDA_CHECK(cudaEventRecord(c->eval_done, c->stream));
    c->eval_queued = true;
}

// L2 flush between passes when the caller times with flushed caches: queued
// right before the next evaluation and timed with its own events, which
// run_iterate subtracts
void in_pass_flush(nrr_ctx* c) {
    if (!c->flush_each_pass) return;
    while (static_cast<int>(c->flush_ev.size()) < 2 * (c->flush_used + 1)) {
        cudaEvent_t e;
        NRR_CUDA_CHECK(cudaEventCreate(&e));
        c->flush_ev.push_back(e);
    }
    NRR_CUDA_CHECK(cudaEventRecord(c->flush_ev[2 * c->flush_used], c->stream));
    NRR_CUDA_CHECK(cudaMemsetAsync(c->flush.p, c->flush_used & 0xff, c->flush.n * sizeof(double), c->stream));
    NRR_CUDA_CHECK(cudaEventRecord(c->flush_ev[2 * c->flush_used + 1], c->stream));
    ++c->flush_used;
}

// ---- pass trace (record_passes >= 3): synchronous copies, test instrumentation only
void trace_eval(nrr_ctx* c, const PassRecord& e, bool revert) {
    const size_t D = 12 * static_cast<size_t>(c->N);
    nrr_pass_trace t{};
    t.e_align = e.align;
    t.e_reg = e.reg;
    t.e_rot = e.rot;
    t.e_total = e.total;
    t.e_landmark = e.landmark;
    t.stage = c->run.si;
    t.reverted = revert ? 1 : 0;
    t.accepted_index = -1;
    c->trace.push_back(t);
    c->trace_x.resize(c->trace.size() * D);
    c->trace_xmm.resize(c->trace.size() * D, std::numeric_limits<double>::quiet_NaN());
    c->trace_nn.resize(c->trace.size() * static_cast<size_t>(c->n));
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->trace_x.data() + (c->trace.size() - 1) * D, c->x.p, sizeof(double) * D,
                                   cudaMemcpyDeviceToHost, c->stream));
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->trace_nn.data() + (c->trace.size() - 1) * c->n, c->nn_idx.p,
                                   sizeof(int) * c->n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
}
void trace_accept(nrr_ctx* c, double max_disp) {
    const size_t D = 12 * static_cast<size_t>(c->N);
    nrr_pass_trace& t = c->trace.back();
    t.max_disp = max_disp;
    t.pcg_iterations = c->h_status.p->iterations;
    t.accepted_index = static_cast<int32_t>(c->iters.size());
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->trace_xmm.data() + (c->trace.size() - 1) * D, c->xmm.p, sizeof(double) * D,
                                   cudaMemcpyDeviceToHost, c->stream));
    sync(c);
}

// One evaluated pass (solver.hpp:225-288). Returns true when an iteration was
// accepted; sets *stage_end when the stage converged or hit i_max.
bool one_pass(nrr_ctx* c, bool* stage_end) {
    RunState& r = c->run;
    const int N = c->N, n = c->n, D = 12 * N;
    *stage_end = false;
    if (++r.passes > 2 * r.cfg.i_max + 4) throw NumericalError("solver stage failed to make progress");
    const TermParams tp = local_terms(c, TermParams{r.prm.alpha, r.prm.beta, r.prm.nu_a, r.prm.nu_r, r.lm_w});
    bool ran[nrr_ctx::kClasses];
    std::fill(ran, ran + nrr_ctx::kClasses, false);
    if (!c->eval_queued) queue_eval(c, tp, c->x.p, c->vhat.p);
    c->eval_queued = false;
    ran[kNN] = c->eval_nn_ran || c->nn_time_pending;  // a queued NN is harvested with its evaluation
    c->nn_time_pending = false;
    ran[kTerms] = true;
    c->dp.skip = c->d_skip.p;
    assemble(c, tp);
    if (c->comm) {  // the replicated solve needs the full K and B (north_star: allreduce before the solve)
        ClassTimer tc(c, kComm);
        allreduce(c, c->K.p, 16 * static_cast<size_t>(c->dp.nnzb), ncclFloat64, ncclSum);
        allreduce(c, c->B.p, 12 * static_cast<size_t>(N), ncclFloat64, ncclSum);
    }
    c->pcg_skip = c->d_skip.p;
    c->reuse_precond = true;
    solve(c, c->x.p, c->xmm_spec.p);  // x_mm = solve(), warm start at x; kept aside until accepted
    c->reuse_precond = false;
    c->pcg_skip = nullptr;
    c->dp.skip = nullptr;
    NRR_CUDA_CHECK(cudaEventSynchronize(c->eval_done));
    harvest(c, ran);
    std::fill(ran, ran + nrr_ctx::kClasses, false);
    const PassRecord e = *c->h_rec.p;
    r.degenerate_total += *c->h_deg.p;
    const double e_accept = e.total + r.lm_w * e.landmark;
    if (!std::isfinite(e_accept)) throw NumericalError("solver aborted: energy is not finite");
    const bool revert = e_accept > r.e_prev && r.current_is_aa;  // solver.hpp:239
    if (c->opt.record_passes) c->passes.push_back({e.total, r.si, revert ? 1 : 0});
    if (c->opt.record_passes >= 3) trace_eval(c, e, revert);
    if (revert) {  // solver.hpp:244-248 (x_mm of the previous pass is untouched)
        // the device skipped this pass's solve and preconditioner rebuilds
        c->sub_age = c->prev_sub_age;
        c->coarse_age = c->prev_coarse_age;
        c->last_solve_fresh = c->prev_solve_fresh;
        NRR_CUDA_CHECK(cudaMemcpyAsync(c->x.p, c->xmm.p, sizeof(double) * D, cudaMemcpyDeviceToDevice, c->stream));
        deform_run(c, c->x.p, c->vhat.p, nullptr, nullptr);
        r.current_is_aa = false;
        ++r.st.reverts;
        in_pass_flush(c);
        queue_eval(c, tp, c->x.p, c->vhat.p);  // the next pass re-evaluates at x_mm
        return false;
    }
    r.e_prev = e_accept;
    nrr_iteration_record rec{e.total, e.align, e.reg, e.rot, e.landmark, 0.0, r.current_is_aa ? 1 : 0, r.si};
    std::swap(c->xmm.p, c->xmm_spec.p);
    ran[kAsm] = ran[kPcg] = true;
    ran[kComm] = c->comm != nullptr;
    aa_push_combine(c, r.win, c->xmm.p, c->x.p, nullptr, c->xnext.p, D);
    ran[kAA] = true;
    r.current_is_aa = r.win.extrapolating();
    NRR_CUDA_CHECK(cudaMemsetAsync(&c->d_rec.p->max_disp, 0, sizeof(double), c->stream));
    deform_run(c, c->xnext.p, c->vhat2.p, c->vhat.p, &c->d_rec.p->max_disp);
    ran[kDeform] = true;
    allreduce(c, &c->d_rec.p->max_disp, 1, ncclFloat64, ncclMax);
    allreduce(c, &c->d_rec.p->nonfinite, 1, ncclInt32, ncclMax);
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->h_rec_end.p, c->d_rec.p, sizeof(PassRecord), cudaMemcpyDeviceToHost, c->stream));
    NRR_CUDA_CHECK(cudaMemcpyAsync(c->h_status.p, c->d_status.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost, c->stream));
    NRR_CUDA_CHECK(cudaEventRecord(c->end_done, c->stream));
    // the next pass's correspondences and evaluation at the new iterate are
    // queued before the end-of-pass sync (a new stage only changes the
    // weights: then the queued evaluation is dropped and redone)
    in_pass_flush(c);
    nn_run(c, c->vhat2.p, c->n, c->nn_idx.p, c->nn_idx.p, c->d2.p, c->q.p, c->d_anchor.p);
    c->nn_ready = true;
    c->nn_time_pending = true;
    queue_eval(c, tp, c->xnext.p, c->vhat2.p);
    NRR_CUDA_CHECK(cudaEventSynchronize(c->end_done));
    harvest(c, ran);
    check_pcg(c, *c->h_status.p);
    c->pcg_iters_total += c->h_status.p->iterations;
    {  // preconditioner staleness (deterministic: depends on iteration counts only)
        const int it = c->h_status.p->iterations;
        if (c->last_solve_fresh) c->base_iters = it;
        else if (it > c->base_iters + c->base_iters / 4 + 2) c->sub_age = c->coarse_age = -1;
    }
    if (c->h_rec_end.p->nonfinite) throw NumericalError("solver aborted: iterate is not finite");
    rec.max_disp = c->h_rec_end.p->max_disp;
    if (c->opt.record_passes >= 3) trace_accept(c, rec.max_disp);
    c->iters.push_back(rec);
    ++r.st.iteration_count;
    std::swap(c->x.p, c->xnext.p);
    std::swap(c->vhat.p, c->vhat2.p);
    ++r.accepted;
    if (rec.max_disp < r.cfg.eps) {
        r.st.converged = 1;
        *stage_end = true;
    } else if (r.accepted >= r.cfg.i_max) {
        *stage_end = true;
    }
    if (*stage_end) {  // the queued evaluation used this stage's weights
        c->eval_queued = false;
        c->nn_ready = true;  // the correspondences at x stay valid
    }
    return true;
}

// Runs passes until `max_accepted` more iterations were accepted or the run
// finished. Device time of the passes (CUDA events on the context stream,
// excluding the optional L2 flush before each pass) is added to *device_ms.
int run_iterate(nrr_ctx* c, int max_accepted, bool flush_l2, double* device_ms) {
    RunState& r = c->run;
    if (!r.active) throw ConfigError("no registration in progress (nrr_ctx_begin)");
    int acc = 0;
    if (flush_l2 && c->flush.n == 0) c->flush.resize(c->l2_bytes * 2 / sizeof(double) + 1);
    c->flush_each_pass = flush_l2;
    c->flush_used = 0;
    // one event interval around all the passes of this call (host gaps
    // included), minus the flushes queued inside it; a flush before the first
    // evaluation (when none is queued) stays outside the interval
    if (flush_l2 && !c->eval_queued)
        NRR_CUDA_CHECK(cudaMemsetAsync(c->flush.p, 0x5a, c->flush.n * sizeof(double), c->stream));
    NRR_CUDA_CHECK(cudaEventRecord(c->pass_ev[0], c->stream));
    while (!r.done && acc < max_accepted) {
        if (!r.stage_open) open_stage(c);
        bool stage_end = false;
        const bool accepted = one_pass(c, &stage_end);
        if (accepted) ++acc;
        if (stage_end) close_stage(c);
    }
    NRR_CUDA_CHECK(cudaEventRecord(c->pass_ev[1], c->stream));
    NRR_CUDA_CHECK(cudaEventSynchronize(c->pass_ev[1]));
    float ms = 0.f;
    NRR_CUDA_CHECK(cudaEventElapsedTime(&ms, c->pass_ev[0], c->pass_ev[1]));
    double total = ms;
    for (int k = 0; k < c->flush_used; ++k) {
        float f = 0.f;
        NRR_CUDA_CHECK(cudaEventElapsedTime(&f, c->flush_ev[2 * k], c->flush_ev[2 * k + 1]));
        total -= f;
    }
    c->flush_each_pass = false;
    if (device_ms) *device_ms += total;
    return acc;
}

void run_finish(nrr_ctx* c, double* out_X, double* out_deformed) {
    RunState& r = c->run;
    c->nn_ready = false;
    c->eval_queued = false;
    if (!r.active) throw ConfigError("no registration in progress (nrr_ctx_begin)");
    if (r.stage_open) close_stage(c);  // stopped early: record the partial stage
    check_nn_overflow(c);
    const auto t2 = std::chrono::steady_clock::now();
    const int N = c->N, n = c->n;
    if (out_X) {
        launch_nodemajor_to_colmajor(c->x.p, c->xnext.p, N, c->stream);
        ++c->launches;
        NRR_CUDA_CHECK(cudaMemcpyAsync(out_X, c->xnext.p, sizeof(double) * 12 * N, cudaMemcpyDeviceToHost, c->stream));
    }
    if (out_deformed)
        NRR_CUDA_CHECK(cudaMemcpyAsync(out_deformed, c->vhat.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    nrr_report_summary& s = c->summary;
    s.stage_count = static_cast<int32_t>(c->stages.size());
    s.total_iterations = static_cast<int32_t>(c->iters.size());
    s.degenerate_rotations = r.degenerate_total;
    s.alpha_forced_zero = r.prm.forced_zero ? 1 : 0;
    s.total_passes = 0;
    for (const auto& stg : c->stages) s.total_passes += stg.iteration_count + stg.reverts;
    s.linear_iterations = c->pcg_iters_total;
    s.setup_seconds = std::chrono::duration<double>(r.t1 - r.t0).count();
    s.loop_seconds = std::chrono::duration<double>(t2 - r.t1).count();
    s.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - r.t0).count();
    r.active = false;
}

void run_register(nrr_ctx* c, const nrr_solver_config& cfg, double* out_X, double* out_deformed) {
    run_begin(c, cfg);
    run_iterate(c, std::numeric_limits<int>::max(), false, nullptr);
    run_finish(c, out_X, out_deformed);
}

}  // namespace
}  // namespace nrr_b200

// ================================================================== C ABI
extern "C" {

const char* nrr_last_error(void) { return nrr_b200::g_last_error.c_str(); }

int nrr_device_info(int device, char* name, int32_t cap, int32_t* sm_count) {
    return guarded([&] {
        cudaDeviceProp prop{};
        NRR_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
        if (name && cap > 0) {
            std::strncpy(name, prop.name, cap - 1);
            name[cap - 1] = 0;
        }
        if (sm_count) *sm_count = prop.multiProcessorCount;
    });
}

int nrr_ctx_create(int device, nrr_ctx** out) {
    return guarded([&] {
        *out = nullptr;
        int count = 0;
        NRR_CUDA_CHECK(cudaGetDeviceCount(&count));
        if (count == 0) throw CudaError("no CUDA device");
        NRR_CUDA_CHECK(cudaSetDevice(device));
        cudaDeviceProp prop{};
        NRR_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) throw CudaError("nrr_b200 needs an sm_100a device (B200)");
        auto c = std::make_unique<nrr_ctx>();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        c->smem_optin = prop.sharedMemPerBlockOptin;
        NRR_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        NRR_CUDA_CHECK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        NRR_CUDA_CHECK(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
        NRR_CUDA_CHECK(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
        NRR_CUDA_CHECK(cudaEventCreateWithFlags(&c->eval_done, cudaEventDisableTiming));
        NRR_CUDA_CHECK(cudaEventCreateWithFlags(&c->end_done, cudaEventDisableTiming));
        NRR_CUDA_CHECK(cudaEventCreateWithFlags(&c->pcg_done, cudaEventDisableTiming));
        c->d_rec.resize(1);
        c->d_status.resize(1);
        c->deg.resize(1);
        for (auto& e : c->ev)
            for (auto& x : e) NRR_CUDA_CHECK(cudaEventCreate(&x));
        for (auto& x : c->pass_ev) NRR_CUDA_CHECK(cudaEventCreate(&x));
        c->l2_bytes = prop.l2CacheSize;
        *out = c.release();
    });
}

void nrr_ctx_destroy(nrr_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);  // buffers go back to the block cache
    if (ctx->side) cudaStreamSynchronize(ctx->side);
    delete ctx;
}

int nrr_ctx_set_options(nrr_ctx* ctx, const nrr_solve_options* opt) {
    return guarded([&] {
        if (!(opt->pcg_rtol > 0.0) || opt->pcg_max_iter < 1 || opt->max_ctas < 0) throw ConfigError("invalid solve options");
        ctx->opt = *opt;
    });
}

int nrr_ctx_enable_timing(nrr_ctx* ctx, int32_t on) {
    ctx->timing = on != 0;
    return 0;
}

int nrr_comm_unique_id(void* out128) {
    return guarded([&] {
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "get unique id");
        std::memcpy(out128, &id, sizeof(id));
    });
}

int nrr_ctx_set_comm(nrr_ctx* ctx, const void* id128, int32_t nranks, int32_t rank) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        if (nranks < 1 || rank < 0 || rank >= nranks) throw ConfigError("set_comm: bad rank / size");
        ctx->comm.reset();
        ctx->nranks = nranks;
        ctx->rank = rank;
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        ctx->comm = make_nccl_collective(id, nranks, rank);
    });
}

struct nrr_local_group {
    std::shared_ptr<nrr_b200::LocalGroup> g;
    int n = 0;
};

int nrr_local_group_create(int32_t nranks, nrr_local_group** out) {
    return guarded([&] {
        auto* h = new nrr_local_group;
        try {
            h->g = make_local_group(nranks);
            h->n = nranks;
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void nrr_local_group_destroy(nrr_local_group* g) { delete g; }

int nrr_ctx_set_local_comm(nrr_ctx* ctx, nrr_local_group* group, int32_t rank) {
    return guarded([&] {
        if (!group || rank < 0 || rank >= group->n) throw ConfigError("set_local_comm: bad rank / group");
        ctx->comm.reset();
        ctx->nranks = group->n;
        ctx->rank = rank;
        ctx->comm = make_local_collective(group->g, rank);
    });
}

int nrr_ctx_set_shard(nrr_ctx* ctx, int32_t n_global) {
    return guarded([&] {
        if (n_global < -1) throw ConfigError("set_shard: bad vertex count");
        ctx->n_global = n_global;
    });
}

int nrr_ctx_set_target(nrr_ctx* ctx, const double* target, int32_t m) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        set_target(ctx, target, m);
        NRR_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int nrr_ctx_set_problem(nrr_ctx* ctx, const nrr_problem_view* p) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        if (p->m > 0 && p->target) set_target(ctx, p->target, p->m);
        set_problem(ctx, p);
    });
}

int nrr_ctx_register(nrr_ctx* ctx, const nrr_solver_config* cfg, double* out_X, double* out_deformed) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        run_register(ctx, *cfg, out_X, out_deformed);
    });
}

int nrr_ctx_begin(nrr_ctx* ctx, const nrr_solver_config* cfg) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        run_begin(ctx, *cfg);
    });
}

int nrr_ctx_iterate(nrr_ctx* ctx, int32_t max_accepted, int32_t flush_l2, int32_t* accepted, int32_t* done,
                    double* device_ms) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        double ms = 0.0;
        const int acc = run_iterate(ctx, max_accepted, flush_l2 != 0, &ms);
        if (accepted) *accepted = acc;
        if (done) *done = ctx->run.done ? 1 : 0;
        if (device_ms) *device_ms = ms;
    });
}

int nrr_ctx_finish(nrr_ctx* ctx, double* out_X, double* out_deformed) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        run_finish(ctx, out_X, out_deformed);
    });
}

int nrr_register(nrr_ctx* ctx, const nrr_problem_view* p, const nrr_solver_config* cfg, double* out_X,
                 double* out_deformed) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        validate(*cfg);
        if (p->n == 0 || p->m == 0) throw NumericalError("register_surfaces: empty surface");
        // the target index is built on the device; its kernels run while the
        // host builds the problem plan
        set_target(ctx, p->target, p->m);
        set_problem(ctx, p);
        run_register(ctx, *cfg, out_X, out_deformed);
    });
}

int nrr_ctx_report(nrr_ctx* ctx, nrr_report_summary* summary, nrr_stage_record* stages, int32_t stage_cap,
                   nrr_iteration_record* iters, int32_t iter_cap, nrr_pass_record* passes, int32_t pass_cap,
                   int32_t* pass_nn_index) {
    return guarded([&] {
        if (summary) *summary = ctx->summary;
        for (int k = 0; stages && k < stage_cap && k < static_cast<int>(ctx->stages.size()); ++k) stages[k] = ctx->stages[k];
        for (int k = 0; iters && k < iter_cap && k < static_cast<int>(ctx->iters.size()); ++k) iters[k] = ctx->iters[k];
        const int np = static_cast<int>(ctx->passes.size());
        for (int k = 0; passes && k < pass_cap && k < np; ++k) passes[k] = ctx->passes[k];
        if (pass_nn_index && !ctx->pass_nn.empty()) {
            const size_t cnt = std::min<size_t>(ctx->pass_nn.size(), static_cast<size_t>(pass_cap) * ctx->n);
            std::memcpy(pass_nn_index, ctx->pass_nn.data(), cnt * sizeof(int));
        }
    });
}

int nrr_ctx_trace_count(nrr_ctx* ctx, int32_t* passes) {
    return guarded([&] { *passes = static_cast<int32_t>(ctx->trace.size()); });
}

int nrr_ctx_trace(nrr_ctx* ctx, int32_t pass, nrr_pass_trace* rec, double* x_eval, double* x_mm, int32_t* nn_index) {
    return guarded([&] {
        if (pass < 0 || pass >= static_cast<int32_t>(ctx->trace.size())) throw ConfigError("trace: pass out of range");
        const int N = ctx->N;
        const size_t D = 12 * static_cast<size_t>(N);
        if (rec) *rec = ctx->trace[pass];
        auto to_col = [&](const double* nm, double* out) {  // x[12j+3r+c] -> X[c*4N + 4j + r]
            for (int j = 0; j < N; ++j)
                for (int r = 0; r < 4; ++r)
                    for (int cc = 0; cc < 3; ++cc)
                        out[static_cast<size_t>(cc) * 4 * N + 4 * j + r] = nm[12 * static_cast<size_t>(j) + 3 * r + cc];
        };
        if (x_eval) to_col(ctx->trace_x.data() + pass * D, x_eval);
        if (x_mm) to_col(ctx->trace_xmm.data() + pass * D, x_mm);
        if (nn_index) std::memcpy(nn_index, ctx->trace_nn.data() + static_cast<size_t>(pass) * ctx->n, sizeof(int) * ctx->n);
    });
}

int nrr_nearest_from(nrr_ctx* ctx, const double* queries, int32_t q, const int32_t* prev_index, int32_t* out_index,
                     double* out_distance) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        require_target(ctx);
        if (q <= 0) return;
        DevBuf<double> dq, dd;
        DevBuf<int> di, dp;
        dq.upload(queries, 3 * static_cast<size_t>(q), ctx->stream);
        dd.resize(q);
        di.resize(q);
        if (prev_index) dp.upload(prev_index, q, ctx->stream);
        nn_run(ctx, dq.p, q, prev_index ? dp.p : nullptr, di.p, dd.p, nullptr, nullptr);
        std::vector<double> d2(q);
        NRR_CUDA_CHECK(cudaMemcpyAsync(out_index, di.p, sizeof(int) * q, cudaMemcpyDeviceToHost, ctx->stream));
        NRR_CUDA_CHECK(cudaMemcpyAsync(d2.data(), dd.p, sizeof(double) * q, cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        check_nn_overflow(ctx);
        for (int i = 0; i < q; ++i) out_distance[i] = std::sqrt(d2[i]);  // kd_tree.hpp:128
    });
}

int nrr_nearest(nrr_ctx* ctx, const double* queries, int32_t q, int32_t* out_index, double* out_distance) {
    return nrr_nearest_from(ctx, queries, q, nullptr, out_index, out_distance);
}

int nrr_deform(nrr_ctx* ctx, const double* X, double* out_points) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        require_problem(ctx);
        const int N = ctx->N;
        DevBuf<double> dx;
        dx.upload(X, 12 * static_cast<size_t>(N), ctx->stream);
        launch_colmajor_to_nodemajor(dx.p, ctx->xnext.p, N, ctx->stream);
        NRR_CUDA_CHECK(cudaMemsetAsync(ctx->d_rec.p, 0, sizeof(PassRecord), ctx->stream));
        deform_run(ctx, ctx->xnext.p, ctx->vhat2.p, nullptr, nullptr);
        ++ctx->launches;
        NRR_CUDA_CHECK(cudaMemcpyAsync(out_points, ctx->vhat2.p, sizeof(double) * 3 * ctx->n, cudaMemcpyDeviceToHost,
                                       ctx->stream));
        sync(ctx);
    });
}

int nrr_energy_terms(nrr_ctx* ctx, const nrr_energy_terms_in* in, double* out_w_align, double* out_w_reg,
                     double* out_sums3) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        energy_terms(ctx->stream, in, out_w_align, out_w_reg, out_sums3);
        ctx->launches += 2;
    });
}

int nrr_project_rotations_sigma(nrr_ctx* ctx, const double* X, int32_t N, double* out_R, double* out_sigma_min,
                                int32_t* out_degenerate) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        for (int64_t k = 0; k < 12 * static_cast<int64_t>(N); ++k)
            if (!std::isfinite(X[k])) throw NumericalError("project_to_rotation: non-finite input matrix");
        DevBuf<double> dx, dn, dr, ds;
        DevBuf<int> dd;
        dx.upload(X, 12 * static_cast<size_t>(N), ctx->stream);
        dn.resize(std::max(12 * N, 1));
        dr.resize(std::max(9 * N, 1));
        if (out_sigma_min) ds.resize(std::max(N, 1));
        dd.resize(1);
        dd.zero(ctx->stream);
        launch_colmajor_to_nodemajor(dx.p, dn.p, N, ctx->stream);
        launch_rotations(dn.p, N, dr.p, dd.p, ctx->stream, out_sigma_min ? ds.p : nullptr);
        ctx->launches += 2;
        NRR_CUDA_CHECK(cudaMemcpyAsync(out_R, dr.p, sizeof(double) * 9 * N, cudaMemcpyDeviceToHost, ctx->stream));
        if (out_sigma_min)
            NRR_CUDA_CHECK(cudaMemcpyAsync(out_sigma_min, ds.p, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
        int deg = 0;
        NRR_CUDA_CHECK(cudaMemcpyAsync(&deg, dd.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        if (out_degenerate) *out_degenerate = deg;
    });
}

int nrr_project_rotations(nrr_ctx* ctx, const double* X, int32_t N, double* out_R, int32_t* out_degenerate) {
    return nrr_project_rotations_sigma(ctx, X, N, out_R, nullptr, out_degenerate);
}

int nrr_step(nrr_ctx* ctx, const double* X, const double* prm, double landmark_weight,
             const nrr_solver_config* cfg_for_landmarks, int32_t* out_index, double* out_sqdist, double* out_energy4,
             double* out_K, double* out_B, double* out_Xmm) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        require_target(ctx);
        require_problem(ctx);
        const int N = ctx->N, n = ctx->n;
        if (cfg_for_landmarks) upload_landmarks(ctx, *cfg_for_landmarks);
        else ctx->dp.landmarks = 0;
        DevBuf<double> dx;
        dx.upload(X, 12 * static_cast<size_t>(N), ctx->stream);
        launch_colmajor_to_nodemajor(dx.p, ctx->x.p, N, ctx->stream);
        ++ctx->launches;
        NRR_CUDA_CHECK(cudaMemsetAsync(ctx->d_rec.p, 0, sizeof(PassRecord), ctx->stream));
        deform_run(ctx, ctx->x.p, ctx->vhat.p, nullptr, nullptr);
        const TermParams tp{prm[0], prm[1], prm[2], prm[3], landmark_weight};
        evaluate(ctx, ctx->x.p, ctx->vhat.p, tp, false);
        NRR_CUDA_CHECK(cudaMemcpyAsync(ctx->h_rec.p, ctx->d_rec.p, sizeof(PassRecord), cudaMemcpyDeviceToHost, ctx->stream));
        if (out_index)
            NRR_CUDA_CHECK(cudaMemcpyAsync(out_index, ctx->nn_idx.p, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
        std::vector<double> d2(n);
        NRR_CUDA_CHECK(cudaMemcpyAsync(d2.data(), ctx->d2.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        if (out_sqdist)
            for (int i = 0; i < n; ++i) {
                const double d = std::sqrt(d2[i]);
                out_sqdist[i] = d * d;  // corr.squared_distance (energy.hpp:39)
            }
        if (out_energy4) {
            out_energy4[0] = ctx->h_rec.p->align;
            out_energy4[1] = ctx->h_rec.p->reg;
            out_energy4[2] = ctx->h_rec.p->rot;
            out_energy4[3] = ctx->h_rec.p->total;
        }
        assemble_solve(ctx, tp, ctx->x.p, ctx->xmm.p);
        NRR_CUDA_CHECK(cudaMemcpyAsync(ctx->h_status.p, ctx->d_status.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost,
                                       ctx->stream));
        std::vector<double> kdev(out_K ? 16 * static_cast<size_t>(ctx->dp.nnzb) : 0);
        if (out_K)
            NRR_CUDA_CHECK(cudaMemcpyAsync(kdev.data(), ctx->K.p, sizeof(double) * kdev.size(), cudaMemcpyDeviceToHost,
                                           ctx->stream));
        if (out_B) {
            launch_nodemajor_to_colmajor(ctx->B.p, ctx->xnext.p, N, ctx->stream);
            NRR_CUDA_CHECK(cudaMemcpyAsync(out_B, ctx->xnext.p, sizeof(double) * 12 * N, cudaMemcpyDeviceToHost, ctx->stream));
            sync(ctx);
        }
        sync(ctx);
        if (out_K) {  // solver-row order -> node order (the reference's pattern order)
            size_t o = 0;
            for (int a = 0; a < N; ++a) {
                const int r = ctx->plan.node_row[a];
                const size_t cnt = 16 * static_cast<size_t>(ctx->h_row_ptr[r + 1] - ctx->h_row_ptr[r]);
                std::memcpy(out_K + o, kdev.data() + 16 * static_cast<size_t>(ctx->h_row_ptr[r]), cnt * sizeof(double));
                o += cnt;
            }
        }
        if (out_Xmm) {
            check_pcg(ctx, *ctx->h_status.p);
            launch_nodemajor_to_colmajor(ctx->xmm.p, ctx->xnext.p, N, ctx->stream);
            NRR_CUDA_CHECK(cudaMemcpyAsync(out_Xmm, ctx->xnext.p, sizeof(double) * 12 * N, cudaMemcpyDeviceToHost,
                                           ctx->stream));
            sync(ctx);
        }
    });
}

namespace {
// K in the reference pattern order (node a's row blocks, ascending columns)
// <-> solver-row order on the device
void k_node_to_rows(const nrr_ctx* c, const double* src, double* dst) {
    size_t o = 0;
    for (int a = 0; a < c->N; ++a) {
        const int r = c->plan.node_row[a];
        const size_t cnt = 16 * static_cast<size_t>(c->h_row_ptr[r + 1] - c->h_row_ptr[r]);
        std::memcpy(dst + 16 * static_cast<size_t>(c->h_row_ptr[r]), src + o, cnt * sizeof(double));
        o += cnt;
    }
}
void k_rows_to_node(const nrr_ctx* c, const double* src, double* dst) {
    size_t o = 0;
    for (int a = 0; a < c->N; ++a) {
        const int r = c->plan.node_row[a];
        const size_t cnt = 16 * static_cast<size_t>(c->h_row_ptr[r + 1] - c->h_row_ptr[r]);
        std::memcpy(dst + o, src + 16 * static_cast<size_t>(c->h_row_ptr[r]), cnt * sizeof(double));
        o += cnt;
    }
}
}  // namespace

int nrr_assemble(nrr_ctx* ctx, const double* corr_points, const double* w_align, const double* w_reg,
                 const double* rotations, double beta, double landmark_weight,
                 const nrr_solver_config* cfg_for_landmarks, double* out_K, double* out_B) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        require_problem(ctx);
        const int N = ctx->N, n = ctx->n, P = ctx->dp.P;
        if (!corr_points || !w_align || (!w_reg && P > 0) || !rotations)
            throw ConfigError("assemble: null input array");
        if (cfg_for_landmarks) upload_landmarks(ctx, *cfg_for_landmarks);
        else ctx->dp.landmarks = 0;
        // the assembly consumes q = u - anchor, as the NN pass writes it
        if (ctx->h_anchor.size() != 3 * static_cast<size_t>(n)) {
            ctx->h_anchor.resize(3 * static_cast<size_t>(n));
            if (n > 0)
                NRR_CUDA_CHECK(cudaMemcpy(ctx->h_anchor.data(), ctx->d_anchor.p, sizeof(double) * 3 * n,
                                          cudaMemcpyDeviceToHost));
        }
        std::vector<double> q(3 * static_cast<size_t>(n));
        for (size_t k = 0; k < q.size(); ++k) q[k] = corr_points[k] - ctx->h_anchor[k];
        NRR_CUDA_CHECK(cudaMemcpyAsync(ctx->q.p, q.data(), sizeof(double) * q.size(), cudaMemcpyHostToDevice, ctx->stream));
        NRR_CUDA_CHECK(cudaMemcpyAsync(ctx->wa.p, w_align, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        if (P > 0)
            NRR_CUDA_CHECK(cudaMemcpyAsync(ctx->wr.p, w_reg, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
        NRR_CUDA_CHECK(cudaMemcpyAsync(ctx->R.p, rotations, sizeof(double) * 9 * N, cudaMemcpyHostToDevice, ctx->stream));
        const TermParams tp{0.0, beta, 1.0, 1.0, landmark_weight};
        assemble(ctx, tp);
        if (out_K) {
            std::vector<double> kdev(16 * static_cast<size_t>(ctx->dp.nnzb));
            NRR_CUDA_CHECK(cudaMemcpyAsync(kdev.data(), ctx->K.p, sizeof(double) * kdev.size(), cudaMemcpyDeviceToHost,
                                           ctx->stream));
            sync(ctx);
            k_rows_to_node(ctx, kdev.data(), out_K);
        }
        if (out_B) {
            launch_nodemajor_to_colmajor(ctx->B.p, ctx->xnext.p, N, ctx->stream);
            ++ctx->launches;
            NRR_CUDA_CHECK(cudaMemcpyAsync(out_B, ctx->xnext.p, sizeof(double) * 12 * N, cudaMemcpyDeviceToHost, ctx->stream));
        }
        sync(ctx);
    });
}

int nrr_solve(nrr_ctx* ctx, const double* K, const double* B, const double* X0, double* out_X) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        require_problem(ctx);
        const int N = ctx->N;
        if (K) {
            std::vector<double> krow(16 * static_cast<size_t>(ctx->dp.nnzb));
            k_node_to_rows(ctx, K, krow.data());
            NRR_CUDA_CHECK(cudaMemcpyAsync(ctx->K.p, krow.data(), sizeof(double) * krow.size(), cudaMemcpyHostToDevice,
                                           ctx->stream));
            sync(ctx);
        }
        if (B) {
            DevBuf<double> db;
            db.upload(B, 12 * static_cast<size_t>(N), ctx->stream);
            launch_colmajor_to_nodemajor(db.p, ctx->B.p, N, ctx->stream);
            ++ctx->launches;
            sync(ctx);
        }
        if (X0) {
            DevBuf<double> dx;
            dx.upload(X0, 12 * static_cast<size_t>(N), ctx->stream);
            launch_colmajor_to_nodemajor(dx.p, ctx->x.p, N, ctx->stream);
            ++ctx->launches;
            sync(ctx);
        } else {
            NRR_CUDA_CHECK(cudaMemsetAsync(ctx->x.p, 0, sizeof(double) * 12 * N, ctx->stream));
        }
        solve(ctx, ctx->x.p, ctx->xmm.p);
        NRR_CUDA_CHECK(cudaMemcpyAsync(ctx->h_status.p, ctx->d_status.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost,
                                       ctx->stream));
        sync(ctx);
        check_pcg(ctx, *ctx->h_status.p);
        if (out_X) {
            launch_nodemajor_to_colmajor(ctx->xmm.p, ctx->xnext.p, N, ctx->stream);
            ++ctx->launches;
            NRR_CUDA_CHECK(cudaMemcpyAsync(out_X, ctx->xnext.p, sizeof(double) * 12 * N, cudaMemcpyDeviceToHost,
                                           ctx->stream));
            sync(ctx);
        }
    });
}

int nrr_anderson_combine(nrr_ctx* ctx, const double* G, const double* F, int32_t h, int32_t dim, int32_t m,
                         double* out, int32_t* out_rank) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        if (h <= 0) throw NumericalError("anderson_combine: empty history");
        if (m < 0) throw ConfigError("AndersonWindow: window must be >= 0");
        const int mk = std::min(h - 1, m);
        if (mk <= 0) {  // plain update (anderson.hpp:29)
            std::memcpy(out, G + static_cast<size_t>(h - 1) * dim, sizeof(double) * dim);
            if (out_rank) *out_rank = 0;
            return;
        }
        ensure_aa(ctx, mk, dim);
        Window w;
        w.m = mk;
        w.reset();
        DevBuf<double> dg, df, dn;
        dn.resize(dim);
        NRR_CUDA_CHECK(cudaMemsetAsync(ctx->d_rec.p, 0, sizeof(PassRecord), ctx->stream));
        for (int k = h - mk - 1; k < h; ++k) {  // the newest mk+1 entries decide the result
            dg.upload(G + static_cast<size_t>(k) * dim, dim, ctx->stream);
            df.upload(F + static_cast<size_t>(k) * dim, dim, ctx->stream);
            aa_push_combine(ctx, w, dg.p, nullptr, df.p, dn.p, dim);
            sync(ctx);
        }
        int rank = 0;
        NRR_CUDA_CHECK(cudaMemcpyAsync(out, dn.p, sizeof(double) * dim, cudaMemcpyDeviceToHost, ctx->stream));
        NRR_CUDA_CHECK(cudaMemcpyAsync(&rank, ctx->aa.rank, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        if (out_rank) *out_rank = rank;
    });
}

int nrr_init_parameters(nrr_ctx* ctx, const nrr_solver_config* cfg, double* out6) {
    return guarded([&] {
        NRR_CUDA_CHECK(cudaSetDevice(ctx->device));
        const Params p = init_parameters(ctx, *cfg);
        out6[0] = p.nu_a;
        out6[1] = p.nu_r;
        out6[2] = p.nu_a_min;
        out6[3] = p.alpha;
        out6[4] = p.beta;
        out6[5] = p.forced_zero ? 1.0 : 0.0;
    });
}

int nrr_debug_pcg_partition(const nrr_problem_view* p, int32_t num_sms, int32_t* out3, int32_t* row_begin,
                            int32_t* row_node) {
    return guarded([&] {
        const int N = p->node_count, E = p->edge_count;
        if (N <= 0 || num_sms <= 0) throw ConfigError("nrr_debug_pcg_partition: empty graph or no SMs");
        // the node graph as set_problem builds it: CSR by node, self first, distinct neighbours in front
        std::vector<int> coff(N + 1, 0);
        for (int j = 0; j < N; ++j) coff[j + 1] = 1;
        for (int e = 0; e < E; ++e) {
            ++coff[p->edges[2 * e] + 1];
            ++coff[p->edges[2 * e + 1] + 1];
        }
        for (int j = 0; j < N; ++j) coff[j + 1] += coff[j];
        std::vector<int> cflat(coff[N]), cfill(coff.begin(), coff.end() - 1), deg(N);
        for (int j = 0; j < N; ++j) cflat[cfill[j]++] = j;
        for (int e = 0; e < E; ++e) {
            const int a = p->edges[2 * e], b = p->edges[2 * e + 1];
            cflat[cfill[a]++] = b;
            cflat[cfill[b]++] = a;
        }
        for (int j = 0; j < N; ++j) {
            int* lo = cflat.data() + coff[j];
            int* hi = cflat.data() + coff[j + 1];
            std::sort(lo, hi);
            deg[j] = static_cast<int>(std::unique(lo, hi) - lo);
        }
        PcgPlan plan;
        plan.build(p->node_positions, deg.data(), N, num_sms, 0, coff.data(), cflat.data());
        out3[0] = plan.grid;
        out3[1] = plan.agg_ctas;
        out3[2] = plan.max_rows;
        for (int g = 0; g <= plan.grid; ++g) row_begin[g] = plan.row_begin[g];
        for (int r = 0; r < N; ++r) row_node[r] = plan.row_node[r];
    });
}

int nrr_debug_solver_plan(const nrr_problem_view* p, int32_t num_sms, int64_t smem_limit, int64_t* out8) {
    return guarded([&] {
        const int N = p->node_count, E = p->edge_count;
        std::vector<std::vector<int>> cols(N);
        for (int j = 0; j < N; ++j) cols[j].push_back(j);
        for (int e = 0; e < E; ++e) {
            cols[p->edges[2 * e]].push_back(p->edges[2 * e + 1]);
            cols[p->edges[2 * e + 1]].push_back(p->edges[2 * e]);
        }
        std::vector<int> deg(N), row_ptr(N + 1, 0), col, node_row(N);
        for (int j = 0; j < N; ++j) {
            std::sort(cols[j].begin(), cols[j].end());
            deg[j] = static_cast<int>(cols[j].size());
            row_ptr[j + 1] = row_ptr[j] + deg[j];
            col.insert(col.end(), cols[j].begin(), cols[j].end());
            node_row[j] = j;
        }
        ClusterPlan cp;
        cp.build(p->node_positions, row_ptr.data(), col.data(), node_row.data(), N, static_cast<size_t>(smem_limit), 16);
        out8[0] = cp.ok;
        out8[1] = cp.CS;
        out8[2] = cp.max_rows;
        out8[3] = cp.max_store;
        out8[4] = cp.max_ext;
        out8[5] = static_cast<int64_t>(cp.smem_bytes);
        out8[6] = static_cast<int64_t>(cp.store_src.size());
        int64_t glob = 0;
        for (const auto& e : cp.ent) glob += e.x & 1;
        out8[7] = glob;
        (void)num_sms;
    });
}

int nrr_ctx_comm_ms(nrr_ctx* ctx, double* out_ms) {
    *out_ms = ctx->class_ms[kComm];
    return 0;
}

int nrr_ctx_stats(nrr_ctx* ctx, int64_t* launches, double* kernel_ms6, int32_t* pcg_iters) {
    if (ctx->prof.n && std::getenv("NRR_PROF")) {
        long long h[32];
        cudaMemcpy(h, ctx->prof.p, sizeof(h), cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "pcg phase cycles: %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n",
                     h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
        std::fprintf(stderr, "pcg setup cycles: %lld %lld %lld %lld %lld %lld\n", h[10], h[11], h[12], h[13], h[14], h[15]);
        std::fprintf(stderr, "pcg fine cycles: %lld %lld %lld %lld %lld %lld %lld %lld\n", h[16], h[17], h[18], h[19],
                     h[20], h[21], h[22], h[23]);
        std::fprintf(stderr, "gj cycles: %lld %lld %lld %lld %lld\n", h[24], h[25], h[26], h[27], h[28]);
        if (ctx->cta_prof.n) {
            std::vector<long long> cp(ctx->cta_prof.n);
            cudaMemcpy(cp.data(), ctx->cta_prof.p, sizeof(long long) * cp.size(), cudaMemcpyDeviceToHost);
            const int G = static_cast<int>(cp.size() / 4);
            for (int k = 0; k < 3; ++k) {
                long long mx = 0, sum = 0;
                int arg = 0;
                for (int g = 0; g < G; ++g) {
                    sum += cp[4 * g + k];
                    if (cp[4 * g + k] > mx) mx = cp[4 * g + k], arg = g;
                }
                std::fprintf(stderr, "cta work %d: mean %lld max %lld (cta %d, rows %d)\n", k, sum / G, mx, arg,
                             ctx->plan.row_begin[arg + 1] - ctx->plan.row_begin[arg]);
            }
        }
    }
    if (ctx->nn_stats.n && std::getenv("NRR_NN_STATS")) {
        unsigned long long h[4];
        cudaMemcpy(h, ctx->nn_stats.p, sizeof(h), cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "nn stats: queries %llu internal visits/query %.2f leaf visits/query %.2f leaf hits/query %.3f\n",
                     h[3], double(h[0]) / h[3], double(h[1]) / h[3], double(h[2]) / h[3]);
    }
    if (launches) *launches = ctx->launches;
    if (kernel_ms6)
        for (int k = 0; k < 6; ++k) kernel_ms6[k] = ctx->class_ms[k];
    if (pcg_iters) *pcg_iters = ctx->pcg_iters_total;
    return 0;
}

}  // extern "C"
