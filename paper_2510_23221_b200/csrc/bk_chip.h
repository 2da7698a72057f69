// Host chip floorplan model (bk_chip.cpp): the reference's Floorplan / Block
// types (chip.hpp:82-110) with materials resolved to conductivities.
#pragma once

#include <cstdint>
#include <vector>

#include "blockoa_b200.h"

namespace bk {

enum class BlockRole { high, normal, cache };

struct Block {
    double lo[3], hi[3];  // half-open box, meters
    int layer = 0;
    BlockRole role = BlockRole::normal;
};

struct Region {  // material override (TSVs)
    double lo[3], hi[3];
    double k;
};

struct Floorplan {
    std::uint64_t id = 0;
    std::vector<Block> blocks;
    std::vector<Region> regions;
};

bk_status check_chip(const bk_chip_spec& sp);
bk_status build_floorplans(const bk_chip_spec& sp, int n_k, std::uint64_t seed,
                           std::vector<Floorplan>& plans);
void sample_power(const Floorplan& fp, const bk_chip_spec& sp, std::uint64_t seed,
                  std::vector<double>& densities);
void rasterize_k(const Floorplan& fp, const bk_chip_spec& sp, int nx, int ny, int nz, double* k);
void rasterize_q(const std::vector<double>& densities, const Floorplan& fp,
                 const bk_chip_spec& sp, int nx, int ny, int nz, double* q);
void draw_weights(int n_basis, std::uint64_t master_seed, std::int64_t l, double* mu);

}  // namespace bk
