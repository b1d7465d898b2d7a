// C ABI of the setup side (surface.hpp, deformation_graph.hpp, geodesic.hpp,
// synthetic configs): host implementations in setup.cpp, the device builds
// of kNN connectivity and the deformation graph in
// setup_graph.cu.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "errors.hpp"
#include "nrr_cuda.h"

#include "setup.hpp"
#include "setup_graph.hpp"

#include <cuda_runtime.h>

using namespace nrr_b200;

struct nrr_graph {
    GraphData g;
};

namespace {
void put_edges(const std::vector<std::pair<int, int>>& e, int32_t* out, int32_t cap, int32_t* count) {
    *count = static_cast<int32_t>(e.size());
    if (!out) return;
    if (static_cast<int>(e.size()) > cap) throw ConfigError("edge buffer too small");
    for (size_t i = 0; i < e.size(); ++i) {
        out[2 * i] = e[i].first;
        out[2 * i + 1] = e[i].second;
    }
}
}  // namespace

extern "C" {

int nrr_edges_from_faces(const int32_t* faces, int32_t nf, int32_t n, int32_t* out_edges, int32_t cap,
                         int32_t* out_count) {
    return guarded([&] { put_edges(edges_from_faces(faces, nf, n), out_edges, cap, out_count); });
}

int nrr_knn_edges(const double* pts, int32_t n, int32_t k, int32_t* out_edges, int32_t cap, int32_t* out_count) {
    return guarded([&] { put_edges(knn_edges(pts, n, k), out_edges, cap, out_count); });
}

int nrr_avg_edge_length(const double* pts, int32_t n, const int32_t* edges, int32_t ne, double* out) {
    return guarded([&] { *out = avg_edge_length(pts, n, edges, ne); });
}

int nrr_normalize_pair(double* src, int32_t n, double* tgt, int32_t m, double* out4) {
    return guarded([&] {  // surface.hpp:125-149
        if (n <= 0 || m <= 0) throw NumericalError("normalize_pair: empty surface");
        double lo[3] = {src[0], src[1], src[2]}, hi[3] = {src[0], src[1], src[2]};
        for (const auto& [p, cnt] : {std::pair<double*, int>{src, n}, std::pair<double*, int>{tgt, m}})
            for (int i = 0; i < cnt; ++i)
                for (int c = 0; c < 3; ++c) {
                    lo[c] = std::min(lo[c], p[3 * i + c]);
                    hi[c] = std::max(hi[c], p[3 * i + c]);
                }
        const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        const double diag = std::sqrt(dx * dx + dy * dy + dz * dz);
        if (!(diag > 0.0)) throw NumericalError("normalize_pair: degenerate joint bounding box");
        const double scale = 1.0 / diag;
        double ctr[3];
        for (int c = 0; c < 3; ++c) ctr[c] = (lo[c] + hi[c]) * 0.5;
        for (const auto& [p, cnt] : {std::pair<double*, int>{src, n}, std::pair<double*, int>{tgt, m}})
            for (int i = 0; i < cnt; ++i)
                for (int c = 0; c < 3; ++c) p[3 * i + c] = (p[3 * i + c] - ctr[c]) * scale;
        if (out4) {
            out4[0] = scale;
            out4[1] = ctr[0];
            out4[2] = ctr[1];
            out4[3] = ctr[2];
        }
    });
}

int nrr_build_graph(const double* pts, int32_t n, const int32_t* edges, int32_t ne, double radius, nrr_graph** out) {
    return guarded([&] {
        auto* h = new nrr_graph;
        try {
            h->g = build_graph_impl(pts, n, edges, ne, radius);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int nrr_device_count(int32_t* count) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    *count = c;
    return NRR_OK;
}

int nrr_knn_edges_gpu(int32_t device, const double* pts, int32_t n, int32_t k, int32_t* out_edges, int32_t cap,
                      int32_t* out_count) {
    return guarded([&] { put_edges(knn_edges_gpu(device, pts, n, k), out_edges, cap, out_count); });
}

int nrr_build_graph_gpu(int32_t device, const double* pts, int32_t n, const int32_t* edges, int32_t ne,
                        double radius, nrr_graph** out, int32_t* out_rounds) {
    return guarded([&] {
        auto* h = new nrr_graph;
        try {
            GraphBuildStats st;
            h->g = build_graph_gpu(device, pts, n, edges, ne, radius, &st);
            if (out_rounds) *out_rounds = st.rounds;
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int nrr_limited_geodesic(const double* pts, int32_t n, const int32_t* edges, int32_t ne, int32_t source,
                         double radius, int32_t* out_idx, double* out_dist, int32_t cap, int32_t* out_count) {
    return guarded([&] {
        const auto ball = limited_geodesic_impl(pts, n, edges, ne, source, radius);
        *out_count = static_cast<int32_t>(ball.size());
        if (!out_idx && !out_dist) return;
        if (static_cast<int>(ball.size()) > cap) throw ConfigError("geodesic buffer too small");
        for (size_t t = 0; t < ball.size(); ++t) {
            if (out_idx) out_idx[t] = ball[t].first;
            if (out_dist) out_dist[t] = ball[t].second;
        }
    });
}

void nrr_graph_counts(const nrr_graph* h, int32_t* N, int32_t* E, int32_t* sumk, int32_t* P) {
    *N = static_cast<int32_t>(h->g.node_indices.size());
    *E = static_cast<int32_t>(h->g.edges.size());
    *sumk = static_cast<int32_t>(h->g.infl_node.size());
    *P = static_cast<int32_t>(h->g.pair_w.size());
}

void nrr_graph_export(const nrr_graph* h, int32_t* node_indices, double* node_positions, int32_t* edges,
                      int32_t* infl_offsets, int32_t* infl_nodes, double* infl_weights, double* infl_dist,
                      int32_t* reg_pairs, double* reg_weights) {
    const GraphData& g = h->g;
    if (node_indices) std::memcpy(node_indices, g.node_indices.data(), g.node_indices.size() * sizeof(int));
    if (node_positions) std::memcpy(node_positions, g.node_positions.data(), g.node_positions.size() * sizeof(double));
    if (edges)
        for (size_t e = 0; e < g.edges.size(); ++e) {
            edges[2 * e] = g.edges[e].first;
            edges[2 * e + 1] = g.edges[e].second;
        }
    if (infl_offsets) std::memcpy(infl_offsets, g.infl_off.data(), g.infl_off.size() * sizeof(int));
    if (infl_nodes) std::memcpy(infl_nodes, g.infl_node.data(), g.infl_node.size() * sizeof(int));
    if (infl_weights) std::memcpy(infl_weights, g.infl_w.data(), g.infl_w.size() * sizeof(double));
    if (infl_dist) std::memcpy(infl_dist, g.infl_d.data(), g.infl_d.size() * sizeof(double));
    if (reg_pairs) std::memcpy(reg_pairs, g.pairs.data(), g.pairs.size() * sizeof(int));
    if (reg_weights) std::memcpy(reg_weights, g.pair_w.data(), g.pair_w.size() * sizeof(double));
}

void nrr_graph_free(nrr_graph* g) { delete g; }

int nrr_synth_config(int32_t which, uint64_t seed, double scale, int32_t* n, int32_t* nf_src, int32_t* m, double* src,
                     int32_t* src_faces, double* tgt) {
    return guarded([&] {
        std::vector<double> s, t;
        std::vector<int32_t> f;
        synth_config(which, seed, scale, s, f, t);
        *n = static_cast<int32_t>(s.size() / 3);
        *nf_src = static_cast<int32_t>(f.size() / 3);
        *m = static_cast<int32_t>(t.size() / 3);
        if (src) std::memcpy(src, s.data(), s.size() * sizeof(double));
        if (src_faces) std::memcpy(src_faces, f.data(), f.size() * sizeof(int32_t));
        if (tgt) std::memcpy(tgt, t.data(), t.size() * sizeof(double));
    });
}

}  // extern "C"
