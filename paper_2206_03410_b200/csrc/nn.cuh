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
};

// out_q (optional) = target point - anchor per query (B's q_i, energy.hpp:204)
void launch_nn(const BvhView& bv, const double* queries, int nq, const int* prev_idx, int* out_idx, double* out_d2,
               double* out_q, const double* anchor, cudaStream_t s);

}  // namespace nrr_b200
