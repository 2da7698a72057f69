// Chip floorplan model and sample weights of the reference's own generator
// (host side, plain C++): the inputs of generate_blockoa (pipeline.cpp:365-597)
// for a ChipSpec such as configs/default.json.
//
//   build_floorplans        chip.cpp:180-221 (slot grids :112-120, partial
//                           Fisher-Yates :122-131, blocks :133-154, TSVs :156-178)
//   sample_power            chip.cpp:223-236
//   rasterize_conductivity  chip.cpp:238-274
//   rasterize_power         chip.cpp:276-306
//   draw_weights            pipeline.cpp:136-152, sample_seed_for :88-90
//
// Every draw goes through the bit-exact Rng restatement (bk_synth.h), in the
// reference's order, so floorplans, k fields and power maps are bitwise the
// reference's (tests/test_chip.py pins them against the reference build).
// The fields are small (one k field per group, eta maps per group) and are
// uploaded once per generate call; the per-sample work runs on the GPU.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "blockoa_b200.h"
#include "bk_chip.h"
#include "bk_synth.h"

namespace {

using bk::Xoshiro;

struct Slots {
    int gx = 0, gy = 0;
    double sw = 0.0, sh = 0.0;
};

// disjoint slots of a per-layer virtual grid, ~40 % spare, chip aspect
Slots slots_for(const bk_chip_spec& sp, int count) {
    const double aspect = sp.extent[0] / sp.extent[1];
    const double target = 1.4 * count;
    const int gy = std::max(1, (int)std::ceil(std::sqrt(target / aspect)));
    const int gx = std::max(1, (int)std::ceil(target / gy));
    return {gx, gy, sp.extent[0] / gx, sp.extent[1] / gy};
}

// first `take` entries of a seeded partial Fisher-Yates shuffle of 0..n-1
std::vector<int> pick_distinct(int n, int take, Xoshiro& rng) {
    std::vector<int> idx(static_cast<std::size_t>(n));
    std::iota(idx.begin(), idx.end(), 0);
    for (int i = 0; i < take; ++i) {
        const int j = i + static_cast<int>(rng.below(static_cast<std::uint64_t>(n - i)));
        std::swap(idx[static_cast<std::size_t>(i)], idx[static_cast<std::size_t>(j)]);
    }
    idx.resize(static_cast<std::size_t>(take));
    return idx;
}

bool place_blocks(const bk_chip_spec& sp, int layer, int count, bk::BlockRole role, Xoshiro& rng,
                  std::vector<bk::Block>& out) {
    if (count <= 0) return true;
    const Slots sg = slots_for(sp, count);
    if (static_cast<long>(sg.gx) * sg.gy < count) return false;
    const bk_layer& L = sp.layers[layer];
    for (const int slot : pick_distinct(sg.gx * sg.gy, count, rng)) {
        const int sx = slot % sg.gx, sy = slot / sg.gx;
        const double w = sg.sw * rng.uniform_fma(0.55, 0.9);
        const double h = sg.sh * rng.uniform_fma(0.55, 0.9);
        // GCC contracts the inlined draws and the slot offset (as it does
        // for the power densities, which pin it bitwise)
        const double x0 = std::fma(static_cast<double>(sx), sg.sw, rng.uniform_fma(0.0, sg.sw - w));
        const double y0 = std::fma(static_cast<double>(sy), sg.sh, rng.uniform_fma(0.0, sg.sh - h));
        bk::Block b;
        b.lo[0] = x0;
        b.lo[1] = y0;
        b.lo[2] = L.z_lo;
        b.hi[0] = x0 + w;
        b.hi[1] = y0 + h;
        b.hi[2] = L.z_hi;
        b.layer = layer;
        b.role = role;
        out.push_back(b);
    }
    return true;
}

// TSVs span the outermost non-TIM layers
void place_tsvs(const bk_chip_spec& sp, Xoshiro& rng, std::vector<bk::Region>& out) {
    if (sp.tsv_count <= 0) return;
    double z_lo = sp.extent[2], z_hi = 0.0;
    for (int l = 0; l < sp.n_layers; ++l) {
        if (sp.layers[l].role == BK_LAYER_TIM) continue;
        z_lo = std::min(z_lo, sp.layers[l].z_lo);
        z_hi = std::max(z_hi, sp.layers[l].z_hi);
    }
    if (!(z_hi > z_lo)) return;
    const double w = std::min({sp.tsv_width, sp.extent[0], sp.extent[1]});
    for (int i = 0; i < sp.tsv_count; ++i) {
        const double x0 = rng.uniform_fma(0.0, sp.extent[0] - w);
        const double y0 = rng.uniform_fma(0.0, sp.extent[1] - w);
        out.push_back(bk::Region{{x0, y0, z_lo}, {x0 + w, y0 + w, z_hi}, sp.tsv_k});
    }
}

// cell-centre index range covered by [lo, hi) on one axis
void covered(double lo, double hi, double d, int n, int& first, int& last) {
    first = std::max(static_cast<int>(std::ceil(lo / d - 0.5)), 0);
    last = std::min(static_cast<int>(std::ceil(hi / d - 0.5)) - 1, n - 1);
}

}  // namespace

namespace bk {

bk_status check_chip(const bk_chip_spec& sp) {
    if (!(sp.extent[0] > 0.0) || !(sp.extent[1] > 0.0) || !(sp.extent[2] > 0.0))
        return BK_INVALID_SPEC;
    if (sp.n_layers < 1 || sp.n_layers > BK_MAX_LAYERS) return BK_INVALID_SPEC;
    for (int l = 0; l < sp.n_layers; ++l)
        if (!(sp.layers[l].z_hi > sp.layers[l].z_lo) || !(sp.layers[l].k > 0.0))
            return BK_INVALID_SPEC;
    if (sp.core_blocks < 0 || sp.high_power < 0 || sp.high_power > sp.core_blocks ||
        sp.caches_per_layer < 0 || sp.tsv_count < 0)
        return BK_INVALID_SPEC;
    if (sp.tsv_count > 0 && !(sp.tsv_width > 0.0 && sp.tsv_k > 0.0)) return BK_INVALID_SPEC;
    bool core = false;
    for (int l = 0; l < sp.n_layers; ++l) core = core || sp.layers[l].role == BK_LAYER_CORE;
    if (sp.core_blocks > 0 && !core) return BK_INVALID_SPEC;
    return BK_OK;
}

bk_status build_floorplans(const bk_chip_spec& sp, int n_k, std::uint64_t seed,
                           std::vector<Floorplan>& plans) {
    bk_status st = check_chip(sp);
    if (st != BK_OK) return st;
    if (n_k < 1) return BK_INVALID_SPEC;
    std::vector<int> core, cache;
    for (int l = 0; l < sp.n_layers; ++l) {
        if (sp.layers[l].role == BK_LAYER_CORE) core.push_back(l);
        else if (sp.layers[l].role == BK_LAYER_CACHE) cache.push_back(l);
    }
    plans.assign(static_cast<std::size_t>(n_k), Floorplan{});
    for (int f = 0; f < n_k; ++f) {
        Xoshiro rng(bk_derive_seed(seed, "floorplan", static_cast<std::uint64_t>(f)));
        Floorplan& fp = plans[static_cast<std::size_t>(f)];
        fp.id = static_cast<std::uint64_t>(f);
        // core blocks split as evenly as possible over the core layers
        const int nc = static_cast<int>(core.size());
        for (int c = 0; c < nc; ++c) {
            const int share = sp.core_blocks / nc + (c < sp.core_blocks % nc ? 1 : 0);
            if (!place_blocks(sp, core[static_cast<std::size_t>(c)], share, BlockRole::normal, rng,
                              fp.blocks))
                return BK_INVALID_SPEC;
        }
        for (const int i : pick_distinct(sp.core_blocks, sp.high_power, rng))
            fp.blocks[static_cast<std::size_t>(i)].role = BlockRole::high;
        for (const int l : cache)
            if (!place_blocks(sp, l, sp.caches_per_layer, BlockRole::cache, rng, fp.blocks))
                return BK_INVALID_SPEC;
        place_tsvs(sp, rng, fp.regions);
    }
    return BK_OK;
}

void sample_power(const Floorplan& fp, const bk_chip_spec& sp, std::uint64_t seed,
                  std::vector<double>& dens) {
    Xoshiro rng(bk_derive_seed(seed, "power", fp.id));
    dens.clear();
    for (const Block& b : fp.blocks) {
        const double* r = b.role == BlockRole::high     ? sp.p_high
                          : b.role == BlockRole::normal ? sp.p_normal
                                                        : sp.p_cache;
        dens.push_back(rng.uniform_fma(r[0], r[1]));
    }
}

void rasterize_k(const Floorplan& fp, const bk_chip_spec& sp, int nx, int ny, int nz,
                 double* k) {
    const double dx = sp.extent[0] / nx, dy = sp.extent[1] / ny, dz = sp.extent[2] / nz;
    const std::int64_t plane = static_cast<std::int64_t>(nx) * ny;
    for (int iz = 0; iz < nz; ++iz) {
        // base material: the layer whose [z_lo, z_hi) holds the cell centre
        const double zc = (iz + 0.5) * dz;
        double kl = sp.layers[sp.n_layers - 1].k;
        for (int l = 0; l < sp.n_layers; ++l)
            if (zc >= sp.layers[l].z_lo && zc < sp.layers[l].z_hi) {
                kl = sp.layers[l].k;
                break;
            }
        std::fill(k + iz * plane, k + (iz + 1) * plane, kl);
    }
    // material regions override the base, later ones win (half-open boxes)
    for (const Region& r : fp.regions)
        for (int iz = 0; iz < nz; ++iz)
            for (int iy = 0; iy < ny; ++iy)
                for (int ix = 0; ix < nx; ++ix) {
                    const double c[3] = {(ix + 0.5) * dx, (iy + 0.5) * dy, (iz + 0.5) * dz};
                    bool in = true;
                    for (int a = 0; a < 3; ++a) in = in && c[a] >= r.lo[a] && c[a] < r.hi[a];
                    if (in) k[ix + nx * (iy + static_cast<std::int64_t>(ny) * iz)] = r.k;
                }
}

void rasterize_q(const std::vector<double>& dens, const Floorplan& fp, const bk_chip_spec& sp,
                 int nx, int ny, int nz, double* q) {
    const double dx = sp.extent[0] / nx, dy = sp.extent[1] / ny, dz = sp.extent[2] / nz;
    std::fill(q, q + static_cast<std::int64_t>(nx) * ny * nz, 0.0);
    for (std::size_t bi = 0; bi < fp.blocks.size(); ++bi) {
        const Block& b = fp.blocks[bi];
        const bk_layer& L = sp.layers[b.layer];
        // W/mm^2 -> W/m^3 over the owning layer's thickness
        const double qv = dens[bi] * 1e6 / (L.z_hi - L.z_lo);
        int x0, x1, y0, y1, z0, z1;
        covered(b.lo[0], b.hi[0], dx, nx, x0, x1);
        covered(b.lo[1], b.hi[1], dy, ny, y0, y1);
        covered(b.lo[2], b.hi[2], dz, nz, z0, z1);
        for (int iz = z0; iz <= z1; ++iz)
            for (int iy = y0; iy <= y1; ++iy)
                for (int ix = x0; ix <= x1; ++ix)
                    q[ix + nx * (iy + static_cast<std::int64_t>(ny) * iz)] = qv;
    }
}

// normalised Gaussian weights of sample l (resampled while |sum| < 1e-6)
void draw_weights(int n_basis, std::uint64_t master, std::int64_t l, double* mu) {
    const std::uint64_t sample = bk_derive_seed(master, "sample", static_cast<std::uint64_t>(l + 1));
    Xoshiro rng(bk_derive_seed(sample, "mu", 0));
    double sum;
    do {
        sum = 0.0;
        for (int t = 0; t < n_basis; ++t) {
            mu[t] = rng.normal();
            sum += mu[t];
        }
    } while (std::abs(sum) < 1e-6);
    for (int t = 0; t < n_basis; ++t) mu[t] /= sum;
}

}  // namespace bk

extern "C" {

void bk_default_chip(bk_chip_spec* out) {
    constexpr double mm = 1e-3;
    bk_chip_spec sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.extent[0] = 10.0 * mm;
    sp.extent[1] = 10.0 * mm;
    sp.extent[2] = 0.51 * mm;
    // bottom to top: TIM / cache die / TIM / cache die / TIM / core die
    const double t_tim = 0.02 * mm, t_die = 0.15 * mm;
    const double k_si = 150.0, k_tim = 40.0;
    double z = 0.0;
    auto push = [&](double t, double k, int role) {
        sp.layers[sp.n_layers++] = bk_layer{z, z + t, k, role};
        z += t;
    };
    push(t_tim, k_tim, BK_LAYER_TIM);
    push(t_die, k_si, BK_LAYER_CACHE);
    push(t_tim, k_tim, BK_LAYER_TIM);
    push(t_die, k_si, BK_LAYER_CACHE);
    push(t_tim, k_tim, BK_LAYER_TIM);
    push(t_die, k_si, BK_LAYER_CORE);
    sp.core_blocks = 156;
    sp.high_power = 6;
    sp.caches_per_layer = 2;
    sp.p_high[0] = 3.0;
    sp.p_high[1] = 6.0;
    sp.p_normal[0] = 0.5;
    sp.p_normal[1] = 1.0;
    sp.p_cache[0] = 0.02;
    sp.p_cache[1] = 0.04;
    sp.tsv_count = 12;
    sp.tsv_width = 0.2 * mm;
    sp.tsv_k = 413.0;  // copper
    *out = sp;
}

bk_status bk_chip_fields(const bk_chip_spec* spec, int nx, int ny, int nz, int n_k, int eta,
                         uint64_t seed, double* k, double* q) {
    if (!spec || nx < 1 || ny < 1 || nz < 1 || eta < 0) return BK_INVALID_SPEC;
    std::vector<bk::Floorplan> fps;
    const bk_status st = bk::build_floorplans(*spec, n_k, seed, fps);
    if (st != BK_OK) return st;
    const std::int64_t n = static_cast<std::int64_t>(nx) * ny * nz;
    std::vector<double> dens;
    for (int j = 0; j < n_k; ++j) {
        if (k) bk::rasterize_k(fps[static_cast<std::size_t>(j)], *spec, nx, ny, nz, k + j * n);
        if (!q) continue;
        for (int t = 0; t < eta; ++t) {
            const std::uint64_t ds =
                bk_derive_seed(seed, "basis", static_cast<std::uint64_t>(j) * eta + t);
            bk::sample_power(fps[static_cast<std::size_t>(j)], *spec, ds, dens);
            bk::rasterize_q(dens, fps[static_cast<std::size_t>(j)], *spec, nx, ny, nz,
                            q + (static_cast<std::int64_t>(j) * eta + t) * n);
        }
    }
    return BK_OK;
}

bk_status bk_draw_weights(int n_basis, uint64_t seed, int64_t n_data, double* w) {
    if (n_basis < 1) return BK_EMPTY_BASIS;
    for (int64_t l = 0; l < n_data; ++l) bk::draw_weights(n_basis, seed, l, w + l * n_basis);
    return BK_OK;
}

}  // extern "C"
