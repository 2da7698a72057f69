// Seeded synthetic inputs for the five BASELINE configs (host side).
//
// The reference has no generators for these configs; the
// pins below are ours and are documented in DESIGN.md §Inputs. All draws go
// through a bit-exact restatement of the reference Rng (xoshiro256** seeded by
// splitmix64, rng.hpp:14-63) and derive_seed (rng.cpp:47-60), so the CPU oracle,
// the reference arm and the GPU path consume identical bytes. Field evaluation
// (exp of the Gaussian blobs, lognormal factors) runs here once per chip; the
// GPU forms B = V q + g itself (rhs_from_power, discretize.cpp:246-256).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "blockoa_b200.h"
#include "bk_synth.h"

namespace {

using bk::Xoshiro;
using bk::sm64;

bk_face adiabatic() { return bk_face{BK_FACE_ADIABATIC, 0.0, 0.0}; }
bk_face robin(double h, double u) { return bk_face{BK_FACE_ROBIN, h, u}; }

// Ambient temperature of every Robin face. Fields are temperature rises over
// ambient (with a non-zero ambient every basis RHS is
// dominated by the shared lift g, the block is numerically rank one and the
// reference block CG stagnates or diverges).
constexpr double kUinf = 0.0;

}  // namespace

namespace bk {

// All random draws of one chip, in the reference Rng order; the host
// generator and the device one (bk_synth_dev.cu) evaluate the same plan.
bk_status synth_plan(const bk_synth_spec* sp, bk_grid* grid, double* dz_out, int* has_dz,
                     bk_face bc[6], bool want_normals, SynthPlan& p) {
    if (!sp || !grid || !has_dz || !bc) return BK_INVALID_CONFIG;
    const int nx = sp->nx, ny = sp->ny, nz = sp->nz, s = sp->s;
    if (nx < 1 || ny < 1 || nz < 1 || s < 1 || sp->N < 0) return BK_INVALID_SPEC;
    p = SynthPlan{};
    p.config = sp->config;
    p.nx = nx;
    p.ny = ny;
    p.nz = nz;
    p.s = s;
    const std::int64_t plane = static_cast<std::int64_t>(nx) * ny;
    const std::int64_t n = plane * nz;
    const std::uint64_t chip = bk_derive_seed(sp->master_seed, "chip", sp->chip_id);
    p.chip_seed = chip;
    *has_dz = 0;
    grid->nx = nx;
    grid->ny = ny;
    grid->nz = nz;
    grid->lx = 10e-3;
    grid->ly = 10e-3;
    grid->dz = nullptr;
    for (int f = 0; f < 6; ++f) bc[f] = adiabatic();
    p.power_z0 = 0;
    p.power_z1 = nz;
    switch (sp->config) {
        case 1:
        case 2: {
            // 2D die: nz=1 z+ Robin sink (Appendix A.2), 16x16-cell k tiles
            // with k ~ U[10,150] drawn tile-row-major (A.3).
            grid->lz = 0.15e-3 * nz;
            bc[5] = robin(1e3, kUinf);
            p.tile = 16;
            p.tx = (nx + p.tile - 1) / p.tile;
            p.ty = (ny + p.tile - 1) / p.tile;
            Xoshiro rk(bk_derive_seed(chip, "k", 0));
            p.kvals.resize(static_cast<std::size_t>(p.tx) * p.ty);
            for (auto& v : p.kvals) v = rk.uniform(10.0, 150.0);
            p.nblobs = sp->config == 1 ? 3 : 5;
            break;
        }
        case 3:
        case 5: {
            // 8-layer stack (A.6), bottom->top: bulk U[1,3], Si 150, TIM 5,
            // Si 150, TIM 5, Si 150, TIM 5, Cu 400; nz/8 cells per layer,
            // 0.1 mm per layer (uniform dz), per-cell lognormal sigma = ln 1.2.
            if (nz % 8 != 0) return BK_INVALID_SPEC;
            p.cpl = nz / 8;
            grid->lz = 0.8e-3;
            bc[4] = robin(1e2, kUinf);
            bc[5] = robin(1e4, kUinf);
            Xoshiro rl(bk_derive_seed(chip, "layers", 0));
            p.kvals = {rl.uniform(1.0, 3.0), 150.0, 5.0, 150.0, 5.0, 150.0, 5.0, 400.0};
            p.lognormal = true;
            p.log_sigma = std::log(1.2);
            if (want_normals) {
                Xoshiro rn(bk_derive_seed(chip, "lognormal", 0));
                p.normals.resize(static_cast<std::size_t>(n));
                for (auto& z : p.normals) z = rn.normal();
            }
            p.power_z0 = p.cpl;
            p.power_z1 = 2 * p.cpl;
            p.nblobs = 3;
            p.nrects = 4;
            p.scale = nx / 128.0;
            break;
        }
        case 4: {
            // Distinct chip per chip_id: dz_l ~ U[50,500] um, k_l ~ U[1,400],
            // h_top, h_bot ~ U[1e2,1e4] (in that draw order), sides adiabatic.
            if (!dz_out) return BK_INVALID_CONFIG;
            Xoshiro rl(bk_derive_seed(chip, "layers", 0));
            double lz = 0.0;
            for (int l = 0; l < nz; ++l) {
                dz_out[l] = rl.uniform(50e-6, 500e-6);
                lz += dz_out[l];
            }
            p.kvals.resize(nz);
            for (int l = 0; l < nz; ++l) p.kvals[l] = rl.uniform(1.0, 400.0);
            const double h_top = rl.uniform(1e2, 1e4);
            const double h_bot = rl.uniform(1e2, 1e4);
            grid->lz = lz;
            grid->dz = dz_out;
            *has_dz = 1;
            bc[4] = robin(h_bot, kUinf);
            bc[5] = robin(h_top, kUinf);
            p.power_z0 = std::min(1, nz - 1);
            p.power_z1 = p.power_z0 + 1;
            p.nblobs = 5;
            p.scale = nx / 128.0;
            break;
        }
        default:
            return BK_INVALID_CONFIG;
    }
    // basis maps: per map the blob (cx, cy, 1/(2 sigma^2), amp) and rectangle
    // (x0, y0, w, h, pw) parameters, drawn in the host generator's order
    p.blobs.resize(static_cast<std::size_t>(s) * p.nblobs * 4);
    p.rects.resize(static_cast<std::size_t>(s) * p.nrects * 5);
    const int wmin = std::max(1, static_cast<int>(4 * p.scale));
    const int wmax = std::max(wmin, static_cast<int>(32 * p.scale));
    for (int t = 0; t < s; ++t) {
        Xoshiro rb(bk_derive_seed(chip, "basis", static_cast<std::uint64_t>(t)));
        for (int b = 0; b < p.nblobs; ++b) {
            double* q = &p.blobs[(static_cast<std::size_t>(t) * p.nblobs + b) * 4];
            q[0] = rb.uniform(0.0, nx);
            q[1] = rb.uniform(0.0, ny);
            const double sig = rb.uniform(2.0, 8.0) * p.scale;
            q[3] = rb.uniform(0.0, 1e6);
            q[2] = 1.0 / (2.0 * sig * sig);
        }
        for (int r = 0; r < p.nrects; ++r) {
            double* q = &p.rects[(static_cast<std::size_t>(t) * p.nrects + r) * 5];
            q[0] = static_cast<double>(rb.below(static_cast<std::uint64_t>(nx)));
            q[1] = static_cast<double>(rb.below(static_cast<std::uint64_t>(ny)));
            q[2] = wmin + static_cast<double>(rb.below(static_cast<std::uint64_t>(wmax - wmin + 1)));
            q[3] = wmin + static_cast<double>(rb.below(static_cast<std::uint64_t>(wmax - wmin + 1)));
            q[4] = rb.uniform(0.0, 2e6);
        }
    }
    return BK_OK;
}

void synth_coef(const bk_synth_spec* sp, std::uint64_t chip_seed, double* C) {
    Xoshiro rc(bk_derive_seed(chip_seed, "coef", 0));
    const std::int64_t cnt = static_cast<std::int64_t>(sp->s) * sp->N;
    for (std::int64_t i = 0; i < cnt; ++i) C[i] = rc.u01();
}

}  // namespace bk

extern "C" {

uint64_t bk_derive_seed(uint64_t seed, const char* tag, uint64_t index) {
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (const unsigned char* c = reinterpret_cast<const unsigned char*>(tag); *c; ++c) {
        h ^= *c;
        h *= 0x100000001b3ULL;
    }
    std::uint64_t st = seed;
    const std::uint64_t mixed = sm64(st) ^ h;
    st = mixed + 0x632be59bd9b4e019ULL * (index + 1);
    return sm64(st);
}

void bk_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
    Xoshiro r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next();
}

void bk_rng_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
    Xoshiro r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}

void bk_rng_normal(uint64_t seed, int64_t n, double* out) {
    Xoshiro r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}

bk_status bk_synth_chip(const bk_synth_spec* sp, bk_grid* grid, double* dz_out, int* has_dz,
                        bk_face bc[6], double* k, double* Q, double* C) {
    bk::SynthPlan p;
    const bk_status st = bk::synth_plan(sp, grid, dz_out, has_dz, bc, k != nullptr, p);
    if (st != BK_OK) return st;
    const int nx = p.nx, ny = p.ny, nz = p.nz, s = p.s;
    const std::int64_t plane = static_cast<std::int64_t>(nx) * ny;
    const std::int64_t n = plane * nz;
    if (k) {
        for (std::int64_t i = 0; i < n; ++i) {
            const int ix = static_cast<int>(i % nx), iy = static_cast<int>((i / nx) % ny);
            const int iz = static_cast<int>(i / plane);
            if (p.config <= 2)
                k[i] = p.kvals[(iy / p.tile) * p.tx + ix / p.tile];
            else if (p.lognormal)
                k[i] = p.kvals[iz / p.cpl] * std::exp(p.log_sigma * p.normals[i]);
            else
                k[i] = p.kvals[iz];
        }
    }
    if (Q) {
        std::memset(Q, 0, static_cast<std::size_t>(n) * s * sizeof(double));
        double* pl = new double[static_cast<std::size_t>(plane)];
        for (int t = 0; t < s; ++t) {
            std::fill(pl, pl + plane, 0.0);
            for (int b = 0; b < p.nblobs; ++b) {
                const double* q = &p.blobs[(static_cast<std::size_t>(t) * p.nblobs + b) * 4];
                for (int iy = 0; iy < ny; ++iy) {
                    const double ddy = iy + 0.5 - q[1];
                    for (int ix = 0; ix < nx; ++ix) {
                        const double ddx = ix + 0.5 - q[0];
                        pl[static_cast<std::size_t>(iy) * nx + ix] +=
                            q[3] * std::exp(-(ddx * ddx + ddy * ddy) * q[2]);
                    }
                }
            }
            for (int r = 0; r < p.nrects; ++r) {
                const double* q = &p.rects[(static_cast<std::size_t>(t) * p.nrects + r) * 5];
                const int x0 = static_cast<int>(q[0]), y0 = static_cast<int>(q[1]);
                const int w = static_cast<int>(q[2]), h = static_cast<int>(q[3]);
                for (int iy = y0; iy < std::min(ny, y0 + h); ++iy)
                    for (int ix = x0; ix < std::min(nx, x0 + w); ++ix)
                        pl[static_cast<std::size_t>(iy) * nx + ix] += q[4];
            }
            for (int iz = p.power_z0; iz < p.power_z1; ++iz)
                for (std::int64_t c = 0; c < plane; ++c) Q[(iz * plane + c) * s + t] = pl[c];
        }
        delete[] pl;
    }
    if (C) bk::synth_coef(sp, p.chip_seed, C);
    return BK_OK;
}

bk_status bk_cg_error_bound(double kappa, int m, double e0, double* out) {
    if (!(kappa >= 1.0)) return BK_INVALID_KAPPA;
    if (m < 0 || !(e0 >= 0.0)) return BK_INVALID_CONFIG;
    const double rk = std::sqrt(kappa);
    *out = 2.0 * std::pow((rk - 1.0) / (rk + 1.0), m) * e0;
    return BK_OK;
}

}  // extern "C"
