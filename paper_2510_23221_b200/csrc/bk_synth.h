// Random draws of one synthetic chip (bk_synth.cpp), shared by the host
// generator and the device one (bk_synth_dev.cu). Plain C++.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

#include "blockoa_b200.h"

namespace bk {

// Rng (rng.hpp:14-63) restated bit-exactly: xoshiro256** seeded by splitmix64,
// 53-bit uniforms, cached Box-Muller pairs, rejection-sampled integers.
inline std::uint64_t sm64(std::uint64_t& st) {
    std::uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

class Xoshiro {
public:
    explicit Xoshiro(std::uint64_t seed) {
        std::uint64_t st = seed;
        for (auto& w : s_) w = sm64(st);
    }
    std::uint64_t next() {
        const std::uint64_t out = rotl(s_[1] * 5, 7) * 9;
        const std::uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return out;
    }
    double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + u01() * (hi - lo); }
    // the same draw as the reference build evaluates it where GCC contracts
    // the inlined lo + u * (hi - lo) into one fused multiply-add (chip.cpp,
    // pipeline.cpp call sites; pinned bitwise by tests/test_chip.py)
    double uniform_fma(double lo, double hi) { return std::fma(u01(), hi - lo, lo); }
    double normal() {
        if (have_) {
            have_ = false;
            return spare_;
        }
        const double u1 = 1.0 - u01();
        const double u2 = u01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * 3.141592653589793 * u2;
        spare_ = r * std::sin(th);
        have_ = true;
        return r * std::cos(th);
    }
    std::uint64_t below(std::uint64_t n) {
        const std::uint64_t lim = n * (~std::uint64_t{0} / n);
        std::uint64_t x;
        do {
            x = next();
        } while (x >= lim);
        return x % n;
    }

private:
    static std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    std::uint64_t s_[4];
    double spare_ = 0.0;
    bool have_ = false;
};


struct SynthPlan {
    int config = 0, nx = 0, ny = 0, nz = 0, s = 0;
    std::uint64_t chip_seed = 0;
    // k: configs 1/2 tile values (tx x ty tiles of `tile` cells), 4 per-layer
    // values, 3/5 per-layer values x exp(log_sigma * normals[cell])
    std::vector<double> kvals;
    int tile = 0, tx = 0, ty = 0, cpl = 1;
    bool lognormal = false;
    double log_sigma = 0.0;
    std::vector<double> normals;
    // basis maps: blobs [s][nblobs][cx, cy, 1/(2 sigma^2), amp], rectangles
    // [s][nrects][x0, y0, w, h, pw], on z-planes [power_z0, power_z1)
    int nblobs = 0, nrects = 0;
    double scale = 1.0;
    std::vector<double> blobs, rects;
    int power_z0 = 0, power_z1 = 0;
};

bk_status synth_plan(const bk_synth_spec* sp, bk_grid* grid, double* dz_out, int* has_dz,
                     bk_face bc[6], bool want_normals, SynthPlan& p);
void synth_coef(const bk_synth_spec* sp, std::uint64_t chip_seed, double* C);

}  // namespace bk
