// Device-side graph setup (see setup_graph.cu): exact kNN connectivity and
// the deformation-graph build on the B200, bitwise equal to setup.cpp.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "setup.hpp"

namespace nrr_b200 {

constexpr int kKnnMaxK = 32;  // largest k of the device kNN (register-resident top-k)

struct GraphBuildStats {
    int rounds = 0;  // LFMIS rounds of the node sweep
    int nodes = 0;
};

// knn_edges (surface.hpp:70-94) on `device`
std::vector<std::pair<int, int>> knn_edges_gpu(int device, const double* pts, int n, int k);
// build_graph (deformation_graph.hpp:157-210) on `device`
GraphData build_graph_gpu(int device, const double* pts, int n, const int32_t* sedges, int ne, double radius,
                          GraphBuildStats* stats = nullptr);

}  // namespace nrr_b200
