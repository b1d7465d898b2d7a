// Device nearest-neighbour index (see nn.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace nrr_b200 {

constexpr int kMaxLevels = 12;

// host-side build product, uploaded once per target (setup)
struct BvhHost {
    int m = 0;
    double center[3] = {0, 0, 0};
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    double half_extent = 0;
    std::vector<float4> pts;             // Morton order, padded to 8
    std::vector<float4> box_lo, box_hi;  // all levels, level 0 = leaves
    std::vector<int> level_off, level_cnt;
    void build(const double* tgt, int m);
};

// kernel argument (by value)
struct BvhView {
    const float4* pts;
    const float4* box_lo;
    const float4* box_hi;
    const double* tgt64;  // original order, m*3
    int m;
    int levels;  // number of box levels; the virtual root sits at `levels`
    int level_off[kMaxLevels];
    int level_cnt[kMaxLevels];
    double cx, cy, cz;
    float half_extent;
    unsigned long long* stats;  // optional (NRR_NN_STATS): [internal visits, leaf visits, leaf hits, queries]
    int* overflow;              // set when a traversal stack overflowed (children would be dropped: the host raises)
    // uniform grid over the same points (warm-started queries whose search
    // ball covers few cells skip the tree): cells of size h from (glx, gly,
    // glz) relative to the centre, cell-major float4 points, cell_start[ncells+1]
    const float4* gpts;
    const int* cell_start;
    int gnx, gny, gnz, gmax_cells;
    float glx, gly, glz, inv_h;
};

// Grid parameters for m points in the box [lo, hi] (cell ~ half the mean
// spacing of a surface sample; <= 32M cells). Returns false if no grid.
struct GridDims {
    int nx = 0, ny = 0, nz = 0;
    double h = 0;
};
GridDims grid_dims(const double lo[3], const double hi[3], int m, double factor = 1.4);
// Device grid build on `s`: targets tgt64 (m x 3, original order), centre.
// scratch: grid_scratch_bytes(m, ncells) bytes; out: gpts (m), cell_start (ncells+1)
size_t grid_scratch_bytes(int m, long long ncells);
void build_grid(const double* tgt64, int m, const double center[3], const double lo[3], const GridDims& g,
                float4* gpts, int* cell_start, void* scratch, cudaStream_t s);

// out_q (optional) = target point - anchor per query (B's q_i, energy.hpp:204)
void launch_nn(const BvhView& bv, const double* queries, int nq, const int* prev_idx, int* out_idx, double* out_d2,
               double* out_q, const double* anchor, cudaStream_t s);

// The BvhHost index built on the device (bitwise the same): fills the meta
// fields of `meta` (centre, box, half extent, level layout; its host point /
// box vectors stay empty) and the device arrays pts (mpad), box_lo / box_hi
// (bvh_layout's total). scratch: bvh_scratch_bytes(m).
void bvh_layout(int m, std::vector<int>& level_off, std::vector<int>& level_cnt, int& total_boxes);
size_t bvh_scratch_bytes(int m);
void build_bvh_device(const double* tgt64, int m, BvhHost& meta, float4* pts, float4* box_lo, float4* box_hi,
                      void* scratch, cudaStream_t s);

}  // namespace nrr_b200
