// Anderson acceleration (reference anderson.hpp:12-73) on the device: the
// least-squares coefficients come from a Givens TSQR of [dF | f] finished with
// the reference's column-pivoted Householder QR (csrc/kernels.cu).
#pragma once

#include <deque>
#include <vector>

#include "nrr/common.hpp"

namespace nrr {

struct AndersonEntry {  // anderson.hpp:12-15
    VectorX g;
    VectorX f;
};

/// anderson.hpp:22-46
inline VectorX anderson_combine(const std::deque<AndersonEntry>& history, int m) {
    if (history.empty()) throw NumericalError("anderson_combine: empty history");
    const int h = static_cast<int>(history.size());
    const int dim = static_cast<int>(history.back().g.size());
    std::vector<double> G(static_cast<size_t>(h) * dim), F(static_cast<size_t>(h) * dim);
    for (int k = 0; k < h; ++k)
        for (int i = 0; i < dim; ++i) {
            G[static_cast<size_t>(k) * dim + i] = history[k].g[i];
            F[static_cast<size_t>(k) * dim + i] = history[k].f[i];
        }
    VectorX out(dim);
    int32_t rank = 0;
    detail::check(nrr_anderson_combine(detail::default_context(), G.data(), F.data(), h, dim, m, out.data(), &rank));
    return out;
}

/// anderson.hpp:50-73
class AndersonWindow {
public:
    explicit AndersonWindow(int m) : m_(m) {
        if (m < 0) throw ConfigError("AndersonWindow: window must be >= 0");
    }
    void reset() { history_.clear(); }
    void push(VectorX g, VectorX f) {
        history_.push_back({std::move(g), std::move(f)});
        while (static_cast<int>(history_.size()) > m_ + 1) history_.pop_front();
    }
    bool extrapolating() const { return m_ > 0 && history_.size() > 1; }
    VectorX combine() const { return anderson_combine(history_, m_); }
    int size() const { return static_cast<int>(history_.size()); }

private:
    int m_;
    std::deque<AndersonEntry> history_;
};

}  // namespace nrr
