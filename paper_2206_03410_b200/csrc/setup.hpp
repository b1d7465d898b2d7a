// Setup side of the drop-in API (CPU; see setup.cpp).
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

namespace nrr_b200 {

// DeformationGraph (deformation_graph.hpp:50-67) as flat arrays
struct GraphData {
    std::vector<int> node_indices;
    std::vector<double> node_positions;  // N*3
    std::vector<std::pair<int, int>> edges;
    std::vector<int> infl_off, infl_node;
    std::vector<double> infl_w, infl_d;
    std::vector<int> pairs;  // P*2
    std::vector<double> pair_w;
};

std::vector<std::pair<int, double>> limited_geodesic_impl(const double* pts, int n, const int32_t* edges, int ne,
                                                          int source, double radius);
void pca_moments(const double* pts, int n, double cov[9]);
void pca_axis(const double cov[9], double out_axis[3]);
GraphData build_graph_impl(const double* pts, int n, const int32_t* sedges, int ne, double radius);
void synth_config(int which, uint64_t seed, double scale, std::vector<double>& src, std::vector<int32_t>& faces,
                  std::vector<double>& tgt);
std::vector<std::pair<int, int>> edges_from_faces(const int32_t* faces, int nf, int n);
std::vector<std::pair<int, int>> knn_edges(const double* pts, int n, int k);
double avg_edge_length(const double* pts, int n, const int32_t* edges, int ne);

}  // namespace nrr_b200
