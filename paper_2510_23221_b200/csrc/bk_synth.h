// Random draws of one synthetic chip (bk_synth.cpp), shared by the host
// generator and the device one (bk_synth_dev.cu). Plain C++.
#pragma once

#include <cstdint>
#include <vector>

#include "blockoa_b200.h"

namespace bk {

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
