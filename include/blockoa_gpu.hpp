// blockoa_gpu.hpp — C++ adapter with the reference's own signatures and types
// over the C ABI (blockoa_b200.h), the drop-in a maintainer adds to the
// reference (/root/reference/proj/core). Header-only; compile with the
// reference's include directory on the path and link libblockoa_b200.so.
//
//   blockoa::gpu::block_cg(ctx, op, b, cfg)   block_cg(const DiscreteOperator&,
//                                             const MultiVector&, const SolverConfig&)
//                                             solvers.hpp:85-88, solvers.cpp:452-665
//   blockoa::gpu::combine_action(ctx, basis, group, weights)
//                                             combine_from_weights + operator_action
//                                             pipeline.hpp:85-97, pipeline.cpp:187-251
//   blockoa::gpu::generate_blockoa(ctx, cfg)  generate_blockoa(const GenerationConfig&)
//                                             pipeline.hpp:108, pipeline.cpp:365-597
//
// Status codes are re-thrown as the reference's exceptions (errors.hpp:9-71).
// Compiled and run against the reference build by tests/cpp/adapter_test.cpp.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "blockoa/discretize.hpp"
#include "blockoa/errors.hpp"
#include "blockoa/pipeline.hpp"
#include "blockoa/solvers.hpp"
#include "blockoa_b200.h"

namespace blockoa::gpu {

inline void check(bk_status st, const bk_ctx* ctx) {
    const std::string m = ctx ? bk_last_error(ctx) : "blockoa_b200";
    switch (st) {
        case BK_OK: return;
        case BK_INVALID_SPEC: throw InvalidSpecError(m);
        case BK_INVALID_CONFIG: throw InvalidConfigError(m);
        case BK_DIMENSION_MISMATCH: throw DimensionMismatchError(m);
        case BK_NONPOSITIVE_K: throw NonPositiveConductivityError(m);
        case BK_NONPOSITIVE_HTC: throw NonPositiveHtcError(m);
        case BK_EMPTY_BASIS: throw EmptyBasisError(m);
        case BK_NOT_CONVERGED: throw NotConvergedError(m);
        case BK_INVALID_KAPPA: throw InvalidKappaError(m);
        default: throw Error(m);
    }
}

// One device context per (host thread, GPU).
class Context {
public:
    explicit Context(int device = 0) { check(bk_create(device, &ctx_), nullptr); }
    ~Context() { bk_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    bk_ctx* get() const { return ctx_; }

private:
    bk_ctx* ctx_ = nullptr;
};

inline bk_face to_face(const FaceCondition& f) {
    if (const auto* d = std::get_if<Dirichlet>(&f)) return {BK_FACE_DIRICHLET, d->u0, 0.0};
    const auto& r = std::get<Robin>(f);
    return {BK_FACE_ROBIN, r.h, r.u_inf};
}

inline bk_grid to_grid(const GridSpec& g) { return {g.nx, g.ny, g.nz, g.lx, g.ly, g.lz, nullptr}; }

inline bk_solver_cfg to_cfg(const SolverConfig& c) {
    return {c.rel_tol, c.max_iter, c.preconditioner == SolverConfig::Precond::jacobi ? 1 : 0};
}

// The reference's assembled operator on the device, bit for bit
// (bk_operator_from_csr: the symmetric 7-point CSR, g and the volumes).
class DeviceOperator {
public:
    DeviceOperator(Context& ctx, const DiscreteOperator& op) : ctx_(ctx) {
        const bk_grid g = to_grid(op.grid);
        check(bk_operator_from_csr(ctx.get(), &g, op.A.row_ptr.data(), op.A.col.data(),
                                   op.A.val.data(), op.g.data(), op.volumes.data(), &op_),
              ctx.get());
    }
    ~DeviceOperator() { bk_operator_free(op_); }
    DeviceOperator(const DeviceOperator&) = delete;
    DeviceOperator& operator=(const DeviceOperator&) = delete;
    bk_operator* get() const { return op_; }

private:
    Context& ctx_;
    bk_operator* op_ = nullptr;
};

// Drop-in for blockoa::block_cg(const DiscreteOperator&, const MultiVector&,
// const SolverConfig&): same result type, per-column report, never throws on
// non-convergence (report.converged), device-timed wall_time.
inline BlockCgResult block_cg(Context& ctx, const DiscreteOperator& op, const MultiVector& b,
                              const SolverConfig& cfg) {
    cfg.validate();
    if (b.n != op.A.n) throw DimensionMismatchError("block_cg: rhs rows != operator size");
    DeviceOperator dop(ctx, op);
    BlockCgResult res;
    res.x = MultiVector(b.n, b.s);
    res.report.final_rel_residual.assign(static_cast<std::size_t>(b.s), 0.0);
    res.report.converged.assign(static_cast<std::size_t>(b.s), 0);
    const bk_solver_cfg c = to_cfg(cfg);
    bk_solve_report rep{0, 0, 0.0, res.report.final_rel_residual.data(),
                        res.report.converged.data()};
    check(bk_block_cg(ctx.get(), dop.get(), b.data.data(), b.s, &c, res.x.data.data(), &rep),
          ctx.get());
    res.report.iterations = rep.iterations;
    res.report.matvec_count = rep.matvec_count;
    res.report.wall_time = rep.wall_time;
    return res;
}

// combine_from_weights(basis, w) followed by operator_action(basis, group, x)
// for several weight vectors at once: weights[j] has the group's eta entries
// (one basis group; columns ascending). Returns (T_j, q_j) per weight vector.
struct Combined {
    std::vector<std::vector<double>> t, q;
    std::vector<double> residual;
};
inline Combined combine_action(Context& ctx, const BasisSet& basis, int group,
                               const std::vector<std::vector<double>>& weights) {
    const BasisGroup& grp = basis.groups.at(static_cast<std::size_t>(group));
    const std::int64_t n = grp.x.n, N = static_cast<std::int64_t>(weights.size());
    const int s = grp.x.s;
    std::vector<double> C(static_cast<std::size_t>(s) * N);
    for (std::int64_t j = 0; j < N; ++j) {
        if (static_cast<int>(weights[j].size()) != s)
            throw DimensionMismatchError("combine_action: weight length != basis width");
        for (int t = 0; t < s; ++t) C[static_cast<std::size_t>(t) * N + j] = weights[j][t];
    }
    DeviceOperator dop(ctx, grp.op);
    std::vector<double> T(static_cast<std::size_t>(N) * n), Q(T.size());
    Combined out;
    out.residual.resize(static_cast<std::size_t>(N));
    check(bk_combine_action(ctx.get(), dop.get(), grp.x.data.data(), s, C.data(), N, T.data(),
                            Q.data(), out.residual.data()),
          ctx.get());
    out.t.resize(static_cast<std::size_t>(N));
    out.q.resize(static_cast<std::size_t>(N));
    for (std::int64_t j = 0; j < N; ++j) {
        out.t[j].assign(T.begin() + j * n, T.begin() + (j + 1) * n);
        out.q[j].assign(Q.begin() + j * n, Q.begin() + (j + 1) * n);
    }
    return out;
}

// Drop-in for blockoa::generate_blockoa(const GenerationConfig&): the whole
// run on the GPU with the reference's semantics (n_k floorplan groups, eta maps
// each, cross-group normalised Gaussian weights, interior noise, sample l in
// group l mod n_k). Limits: n_basis <= 64, eta <= 32. Fills the dataset's
// samples and timings; manifest bookkeeping is left to the caller, as
// generate_blockoa's own caller (run_generate) does.
inline GenerationResult generate_blockoa(Context& ctx, const GenerationConfig& cfg) {
    cfg.validate();
    bk_blockoa_cfg c{};
    c.nx = cfg.grid.nx;
    c.ny = cfg.grid.ny;
    c.nz = cfg.grid.nz;
    for (int f = 0; f < 6; ++f) c.bc[f] = to_face(cfg.bc.faces[f]);
    c.n_data = cfg.n_data;
    c.n_basis = cfg.n_basis;
    c.n_k = cfg.n_k;
    c.master_seed = cfg.master_seed;
    c.noise_kind = cfg.noise.kind == NoiseConfig::Kind::none      ? BK_NOISE_NONE
                   : cfg.noise.kind == NoiseConfig::Kind::uniform ? BK_NOISE_UNIFORM
                                                                  : BK_NOISE_GAUSSIAN;
    c.noise_lo = cfg.noise.lo;
    c.noise_hi = cfg.noise.hi;
    c.noise_sigma = cfg.noise.sigma;
    c.solver = to_cfg(cfg.solver);
    const ChipSpec& sp = cfg.chip;
    for (int a = 0; a < 3; ++a) c.chip.extent[a] = sp.extent[a];
    if (sp.layers.size() > BK_MAX_LAYERS) throw InvalidSpecError("generate_blockoa: too many layers");
    c.chip.n_layers = static_cast<int>(sp.layers.size());
    for (int l = 0; l < c.chip.n_layers; ++l) {
        const Layer& L = sp.layers[static_cast<std::size_t>(l)];
        c.chip.layers[l] = {L.z_lo, L.z_hi, sp.material(L.material).conductivity,
                            L.role == LayerRole::core    ? BK_LAYER_CORE
                            : L.role == LayerRole::cache ? BK_LAYER_CACHE
                                                         : BK_LAYER_TIM};
    }
    c.chip.core_blocks = sp.block_counts.core_blocks;
    c.chip.high_power = sp.block_counts.high_power;
    c.chip.caches_per_layer = sp.block_counts.caches_per_layer;
    for (int e = 0; e < 2; ++e) {
        c.chip.p_high[e] = sp.power_ranges.high[static_cast<std::size_t>(e)];
        c.chip.p_normal[e] = sp.power_ranges.normal[static_cast<std::size_t>(e)];
        c.chip.p_cache[e] = sp.power_ranges.cache[static_cast<std::size_t>(e)];
    }
    if (sp.tsvs) {
        c.chip.tsv_count = sp.tsvs->count;
        c.chip.tsv_width = sp.tsvs->width;
        c.chip.tsv_k = sp.material(sp.tsvs->material).conductivity;
    }
    const std::int64_t n = cfg.grid.cell_count();
    std::vector<double> k(static_cast<std::size_t>(cfg.n_k) * n),
        u(static_cast<std::size_t>(cfg.n_data) * n), q(u.size()), r(static_cast<std::size_t>(cfg.n_data));
    std::vector<std::int64_t> ids(static_cast<std::size_t>(cfg.n_data));
    bk_phase_timings t{};
    check(bk_generate_blockoa(ctx.get(), &c, k.data(), u.data(), q.data(), r.data(), ids.data(),
                              nullptr, &t),
          ctx.get());
    GenerationResult out;
    out.dataset.grid = cfg.grid;
    out.dataset.bc = cfg.bc;
    out.dataset.samples.resize(static_cast<std::size_t>(cfg.n_data));
    for (std::int64_t l = 0; l < cfg.n_data; ++l) {
        Sample& sm = out.dataset.samples[static_cast<std::size_t>(l)];
        const std::int64_t gidx = l % cfg.n_k;
        sm.floorplan_id = static_cast<std::uint64_t>(ids[static_cast<std::size_t>(l)]);
        sm.k = {cfg.grid, Unit::conductivity_w_per_m_k,
                std::vector<double>(k.begin() + gidx * n, k.begin() + (gidx + 1) * n)};
        sm.q = {cfg.grid, Unit::power_density_w_per_m3,
                std::vector<double>(q.begin() + l * n, q.begin() + (l + 1) * n)};
        sm.u = {cfg.grid, Unit::temperature_c,
                std::vector<double>(u.begin() + l * n, u.begin() + (l + 1) * n)};
        sm.provenance = Provenance::blockoa;
        sm.residual = r[static_cast<std::size_t>(l)];
    }
    out.timings.basis_solve_s = t.basis_solve_s;
    out.timings.combine_s = t.combine_action_s;
    out.timings.total_s = t.total_s;
    out.timings.iterations_total = t.iterations_total;
    out.timings.matvecs_total = t.matvecs_total;
    return out;
}

}  // namespace blockoa::gpu
