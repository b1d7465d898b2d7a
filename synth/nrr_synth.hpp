// Seeded synthetic inputs standing in for BASELINE.json configs 0-4
// (SURVEY.md 8(d)): surface pairs only, no registration code. INPUT
// GENERATION, shared by the product's C ABI (nrr_synth_config, csrc/setup.cpp)
// and the CPU oracle (oracle_synth_config), so the reference arm of bench.py
// builds its inputs without loading the product library.
//
// mt19937_64 with explicit transforms (uniform = 53-bit mantissa, Box-Muller)
// instead of the implementation-defined std::*_distribution, so the inputs
// are identical wherever this compiles.
#ifndef NRR_SYNTH_HPP
#define NRR_SYNTH_HPP
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <utility>
#include <vector>

namespace nrr_synth {

struct Rng {  // mt19937_64 with explicit, portable transforms
    uint64_t mt[312];
    int idx = 313;
    explicit Rng(uint64_t seed) {
        mt[0] = seed;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
        idx = 312;
    }
    uint64_t next() {
        if (idx >= 312) {
            for (int i = 0; i < 312; ++i) {
                const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
                uint64_t xa = x >> 1;
                if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
                mt[i] = mt[(i + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    }
    double uni() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
    double uni(double a, double b) { return a + (b - a) * uni(); }
    double gauss() {  // Box-Muller
        double u1 = uni();
        while (u1 <= 0.0) u1 = uni();
        const double u2 = uni();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    }
};

struct Cloud {
    std::vector<double> pts;  // k*3
    std::vector<int32_t> faces;
    void add(double x, double y, double z) {
        pts.push_back(x);
        pts.push_back(y);
        pts.push_back(z);
    }
    int count() const { return static_cast<int>(pts.size() / 3); }
};

inline void rotate_axis_angle(double* p, int n, const double ax[3], double ang, const double ctr[3]) {
    const double c = std::cos(ang), s = std::sin(ang), t = 1 - c;
    const double x = ax[0], y = ax[1], z = ax[2];
    const double R[9] = {t * x * x + c,     t * x * y - s * z, t * x * z + s * y,
                         t * x * y + s * z, t * y * y + c,     t * y * z - s * x,
                         t * x * z - s * y, t * y * z + s * x, t * z * z + c};
    for (int i = 0; i < n; ++i) {
        const double v[3] = {p[3 * i] - ctr[0], p[3 * i + 1] - ctr[1], p[3 * i + 2] - ctr[2]};
        for (int r = 0; r < 3; ++r) p[3 * i + r] = ctr[r] + R[r * 3] * v[0] + R[r * 3 + 1] * v[1] + R[r * 3 + 2] * v[2];
    }
}

inline void random_unit(Rng& rng, double out[3]) {
    double n2 = 0;
    do {
        for (int k = 0; k < 3; ++k) out[k] = rng.gauss();
        n2 = out[0] * out[0] + out[1] * out[1] + out[2] * out[2];
    } while (n2 < 1e-12);
    const double inv = 1.0 / std::sqrt(n2);
    for (int k = 0; k < 3; ++k) out[k] *= inv;
}

// area-uniform torus samples (R, r): rejection on the tube angle
inline void torus_samples(Rng& rng, int count, double R, double r, Cloud& out) {
    while (out.count() < count) {
        const double u = rng.uni(0, 2 * M_PI), v = rng.uni(0, 2 * M_PI);
        if (rng.uni() * (R + r) > R + r * std::cos(v)) continue;
        const double w = R + r * std::cos(v);
        out.add(w * std::cos(u), w * std::sin(u), r * std::sin(v));
    }
}

// Gaussian RBF displacement field: sum_k a_k exp(-|p-c_k|^2 / 2 sigma^2)
inline void rbf_warp(double* p, int n, const std::vector<double>& centers, const std::vector<double>& amps, double sigma) {
    const int K = static_cast<int>(centers.size() / 3);
    for (int i = 0; i < n; ++i) {
        double d[3] = {0, 0, 0};
        for (int k = 0; k < K; ++k) {
            const double dx = p[3 * i] - centers[3 * k], dy = p[3 * i + 1] - centers[3 * k + 1],
                         dz = p[3 * i + 2] - centers[3 * k + 2];
            const double g = std::exp(-(dx * dx + dy * dy + dz * dz) / (2 * sigma * sigma));
            for (int c = 0; c < 3; ++c) d[c] += amps[3 * k + c] * g;
        }
        for (int c = 0; c < 3; ++c) p[3 * i + c] += d[c];
    }
}

inline void add_uniform_outliers(Rng& rng, Cloud& c, int count, double enlarge) {
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = 0; i < c.count(); ++i)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], c.pts[3 * i + k]);
            hi[k] = std::max(hi[k], c.pts[3 * i + k]);
        }
    for (int k = 0; k < 3; ++k) {
        const double mid = 0.5 * (lo[k] + hi[k]), half = 0.5 * (hi[k] - lo[k]) * enlarge;
        lo[k] = mid - half;
        hi[k] = mid + half;
    }
    for (int t = 0; t < count; ++t) c.add(rng.uni(lo[0], hi[0]), rng.uni(lo[1], hi[1]), rng.uni(lo[2], hi[2]));
}

// drop points on the far side of a random plane so that `frac` is removed
inline void halfspace_crop(Rng& rng, Cloud& c, double frac, bool planar_dir) {
    double dir[3];
    random_unit(rng, dir);
    if (planar_dir) {
        dir[2] = 0;
        const double l = std::hypot(dir[0], dir[1]);
        dir[0] /= l;
        dir[1] /= l;
    }
    const int n = c.count();
    std::vector<double> proj(n);
    for (int i = 0; i < n; ++i) proj[i] = c.pts[3 * i] * dir[0] + c.pts[3 * i + 1] * dir[1] + c.pts[3 * i + 2] * dir[2];
    std::vector<double> sorted(proj);
    const int cut = std::min(n - 1, static_cast<int>(frac * n));
    std::nth_element(sorted.begin(), sorted.begin() + cut, sorted.end());
    const double thr = sorted[cut];
    Cloud out;
    for (int i = 0; i < n; ++i)
        if (proj[i] >= thr) out.add(c.pts[3 * i], c.pts[3 * i + 1], c.pts[3 * i + 2]);
    c = std::move(out);
}

struct HeightField {
    double a[6], fx[6], fy[6], ph[6];
    int waves = 6;
    double z(double x, double y) const {
        double s = 0;
        for (int k = 0; k < waves; ++k) s += a[k] * std::sin(2 * M_PI * (fx[k] * x + fy[k] * y) + ph[k]);
        return s;
    }
};

inline HeightField random_height(Rng& rng) {
    HeightField h;
    for (int k = 0; k < 6; ++k) {
        h.a[k] = rng.uni(0.05, 0.2);
        const double f = rng.uni(1.0, 4.0), th = rng.uni(0, 2 * M_PI);
        h.fx[k] = f * std::cos(th);
        h.fy[k] = f * std::sin(th);
        h.ph[k] = rng.uni(0, 2 * M_PI);
    }
    return h;
}

// configs 2 and 4: height field grid source; warped, jittered, holed (or
// cropped) and outlier-polluted target
inline void height_pair(Rng& rng, int side, int holes, double hole_area, double crop_frac, double outlier_frac,
                 Cloud& src, Cloud& tgt) {
    const HeightField hf = random_height(rng);
    const double h = 2.0 / (side - 1);
    for (int j = 0; j < side; ++j)
        for (int i = 0; i < side; ++i) {
            const double x = -1.0 + i * h, y = -1.0 + j * h;
            src.add(x, y, hf.z(x, y));
        }
    for (int j = 0; j + 1 < side; ++j)
        for (int i = 0; i + 1 < side; ++i) {
            const int a = j * side + i, b = a + 1, c = a + side, d = c + 1;
            src.faces.insert(src.faces.end(), {a, b, d, a, d, c});
        }
    // 16-centre RBF warp of the analytic surface, sigma 0.25, |d| = 0.08
    std::vector<double> centers, amps;
    for (int k = 0; k < 16; ++k) {
        const double x = rng.uni(-1, 1), y = rng.uni(-1, 1);
        centers.insert(centers.end(), {x, y, hf.z(x, y)});
        double d[3];
        random_unit(rng, d);
        amps.insert(amps.end(), {0.08 * d[0], 0.08 * d[1], 0.08 * d[2]});
    }
    // elliptical holes totalling hole_area of the [-1,1]^2 domain
    std::vector<std::array<double, 5>> ell;  // cx, cy, a, b, angle
    for (int k = 0; k < holes; ++k) {
        const double area = hole_area * 4.0 / holes, aspect = rng.uni(1.0, 2.0);
        const double b = std::sqrt(area / (M_PI * aspect)), a = aspect * b;
        ell.push_back({rng.uni(-0.7, 0.7), rng.uni(-0.7, 0.7), a, b, rng.uni(0, M_PI)});
    }
    for (int j = 0; j < side; ++j)
        for (int i = 0; i < side; ++i) {
            const double x = -1.0 + (i + rng.uni(-0.5, 0.5)) * h, y = -1.0 + (j + rng.uni(-0.5, 0.5)) * h;
            bool in_hole = false;
            for (const auto& e : ell) {
                const double dx = x - e[0], dy = y - e[1], c = std::cos(e[4]), s = std::sin(e[4]);
                const double u = (c * dx + s * dy) / e[2], v = (-s * dx + c * dy) / e[3];
                if (u * u + v * v < 1.0) in_hole = true;
            }
            if (!in_hole) tgt.add(x, y, hf.z(x, y));
        }
    rbf_warp(tgt.pts.data(), tgt.count(), centers, amps, 0.25);
    if (crop_frac > 0) halfspace_crop(rng, tgt, crop_frac, true);
    add_uniform_outliers(rng, tgt, static_cast<int>(outlier_frac * src.count()), 1.0);
}

// configs 0 and 3: torus pair (R=1, r=0.35) with an 8-centre RBF warp, a
// rotation of at most 15 degrees and N(0, 0.002^2) noise
inline void torus_pair(Rng& rng, int count, Cloud& src, Cloud& tgt) {
    torus_samples(rng, count, 1.0, 0.35, src);
    torus_samples(rng, count, 1.0, 0.35, tgt);
    Cloud ctr;
    torus_samples(rng, 8, 1.0, 0.35, ctr);
    std::vector<double> amps(24);
    for (auto& a : amps) a = 0.1 * rng.gauss();
    rbf_warp(tgt.pts.data(), tgt.count(), ctr.pts, amps, 0.3);
    double ax[3];
    random_unit(rng, ax);
    const double ang = rng.uni(0, 15.0 * M_PI / 180.0), zero[3] = {0, 0, 0};
    rotate_axis_angle(tgt.pts.data(), tgt.count(), ax, ang, zero);
    for (auto& v : tgt.pts) v += 0.002 * rng.gauss();
}

// config 1: chain of 5 capsules (radius 0.15, segment 0.6) along x; target
// bent at each joint by U(-40, 40) degrees, 30% half-space crop, 5% outliers
inline void capsule_pair(Rng& rng, int count, Cloud& src, Cloud& tgt) {
    const int segs = 5;
    const double rad = 0.15, len = 0.6;
    auto sample_chain = [&](Cloud& c, std::vector<int>& seg_of) {
        const double cyl = 2 * M_PI * rad * len, cap = 4 * M_PI * rad * rad;
        while (c.count() < count) {
            const int s = std::min(segs - 1, static_cast<int>(rng.uni() * segs));
            const double x0 = s * len;
            if (rng.uni() * (cyl + cap) < cyl) {
                const double t = rng.uni(0, len), th = rng.uni(0, 2 * M_PI);
                c.add(x0 + t, rad * std::cos(th), rad * std::sin(th));
            } else {
                double d[3];
                random_unit(rng, d);
                const double xe = d[0] < 0 ? x0 : x0 + len;
                c.add(xe + rad * d[0], rad * d[1], rad * d[2]);
            }
            seg_of.push_back(s);
        }
    };
    std::vector<int> ss, ts;
    sample_chain(src, ss);
    sample_chain(tgt, ts);
    // forward kinematics from the tail: joint k (at x = k*len on the straight
    // chain) rotates every segment >= k; applying k = segs-1 .. 1 keeps each
    // joint centre at its original position when it is used
    double angles[segs], axes[segs][3];
    for (int k = 1; k < segs; ++k) {
        angles[k] = rng.uni(-40.0, 40.0) * M_PI / 180.0;
        axes[k][0] = 0;
        axes[k][1] = rng.gauss();
        axes[k][2] = rng.gauss();
        const double l = std::hypot(axes[k][1], axes[k][2]);
        axes[k][1] /= l;
        axes[k][2] /= l;
    }
    for (int k = segs - 1; k >= 1; --k) {
        std::vector<int> ids;
        for (int i = 0; i < tgt.count(); ++i)
            if (ts[i] >= k) ids.push_back(i);
        std::vector<double> moved(ids.size() * 3);
        for (size_t t = 0; t < ids.size(); ++t)
            for (int c = 0; c < 3; ++c) moved[3 * t + c] = tgt.pts[3 * ids[t] + c];
        const double jc[3] = {k * len, 0, 0};
        rotate_axis_angle(moved.data(), static_cast<int>(ids.size()), axes[k], angles[k], jc);
        for (size_t t = 0; t < ids.size(); ++t)
            for (int c = 0; c < 3; ++c) tgt.pts[3 * ids[t] + c] = moved[3 * t + c];
    }
    halfspace_crop(rng, tgt, 0.30, false);
    // replace 5% of the remaining points by uniform outliers in 1.2x the bbox
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = 0; i < tgt.count(); ++i)
        for (int c = 0; c < 3; ++c) {
            lo[c] = std::min(lo[c], tgt.pts[3 * i + c]);
            hi[c] = std::max(hi[c], tgt.pts[3 * i + c]);
        }
    for (int c = 0; c < 3; ++c) {
        const double mid = 0.5 * (lo[c] + hi[c]), half = 0.6 * (hi[c] - lo[c]);
        lo[c] = mid - half;
        hi[c] = mid + half;
    }
    const int cnt = tgt.count(), n_out = static_cast<int>(0.05 * cnt);
    std::vector<int> perm(cnt);
    std::iota(perm.begin(), perm.end(), 0);
    for (int t = 0; t < n_out; ++t) {
        const int j = t + static_cast<int>(rng.uni() * (cnt - t)) % (cnt - t);
        std::swap(perm[t], perm[j]);
        const int i = perm[t];
        for (int c = 0; c < 3; ++c) tgt.pts[3 * i + c] = rng.uni(lo[c], hi[c]);
    }
}
inline void synth_config(int which, uint64_t seed, double scale, std::vector<double>& src, std::vector<int32_t>& faces,
                  std::vector<double>& tgt) {
    if (!(scale > 0.0 && scale <= 1.0)) throw std::invalid_argument("synth: scale must be in (0, 1]");
    Rng rng(seed);
    Cloud s, t;
    switch (which) {
        case 0:
            torus_pair(rng, std::max(64, static_cast<int>(5000 * scale)), s, t);
            break;
        case 1:
            capsule_pair(rng, std::max(64, static_cast<int>(50000 * scale)), s, t);
            break;
        case 2:
            height_pair(rng, std::max(8, static_cast<int>(std::lround(316 * std::sqrt(scale)))), 3, 0.10, 0.0, 0.10, s,
                        t);
            break;
        case 3:
            torus_pair(rng, std::max(64, static_cast<int>(20000 * scale)), s, t);
            break;
        case 4:
            height_pair(rng, std::max(8, static_cast<int>(std::lround(1000 * std::sqrt(scale)))), 0, 0.0, 0.20, 0.08,
                        s, t);
            break;
        default:
            throw std::invalid_argument("synth: config must be 0..4");
    }
    src = std::move(s.pts);
    faces = std::move(s.faces);
    tgt = std::move(t.pts);
}

}  // namespace nrr_synth
#endif
