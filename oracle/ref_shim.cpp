// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" shim over the UNMODIFIED reference core (/root/reference/proj/core),
// compiled by oracle/Makefile into oracle/_ref/libblockoa_ref.so. Only tests/,
// __graft_entry__.smoke() and bench.py's CPU legs (cpu_baseline and
// `--impl reference`) load it, as the checker / the timed reference arm.
//
// Every entry point calls the reference's own public API:
//   assemble               discretize.hpp:76  (discretize.cpp:114-237)
//   CsrMatrix::apply_block discretize.hpp:57  (discretize.cpp:75-95)
//   rhs_from_power         discretize.hpp:82  (discretize.cpp:246-256)
//   power_from_rhs         discretize.hpp:87  (discretize.cpp:258-267)
//   relative_residual      discretize.hpp:91  (discretize.cpp:275-286)
//   cg / block_cg          solvers.hpp:45,85  (solvers.cpp:82-171, 452-665)
//   cg_error_bound         solvers.hpp:92     (solvers.cpp:672-680)
//   combine_from_weights   pipeline.hpp:85    (pipeline.cpp:187-225)
//   operator_action        pipeline.hpp:95    (pipeline.cpp:242-251)
//   Rng / derive_seed      rng.hpp:14-63      (rng.cpp)
//   field_digest           discretize.hpp:99  (discretize.cpp:302-319)
//   build_floorplans / sample_power / rasterize_*  chip.hpp:103-124 (chip.cpp:180-306)
//   generate_blockoa       pipeline.hpp:106   (pipeline.cpp:365-597)
//   write_dataset / read_dataset / validate_dataset
//                          dataset_io.hpp:27-47 (dataset_io.cpp:160-361)
// Exceptions are mapped to the status codes of include/blockoa_b200.h.

#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "blockoa/chip.hpp"
#include "blockoa/dataset.hpp"
#include "blockoa/dataset_io.hpp"
#include "blockoa/discretize.hpp"
#include "blockoa/errors.hpp"
#include "blockoa/parallel.hpp"
#include "blockoa/pipeline.hpp"
#include "blockoa/rng.hpp"
#include "blockoa/solvers.hpp"

using namespace blockoa;

namespace {

thread_local std::string g_err;

int map_exception() {
    try {
        throw;
    } catch (const InvalidSpecError& e) {
        g_err = e.what();
        return 1;
    } catch (const InvalidConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const DimensionMismatchError& e) {
        g_err = e.what();
        return 3;
    } catch (const NonPositiveConductivityError& e) {
        g_err = e.what();
        return 4;
    } catch (const NonPositiveHtcError& e) {
        g_err = e.what();
        return 5;
    } catch (const EmptyBasisError& e) {
        g_err = e.what();
        return 6;
    } catch (const NotConvergedError& e) {
        g_err = e.what();
        return 7;
    } catch (const InvalidKappaError& e) {
        g_err = e.what();
        return 8;
    } catch (const ExistsError& e) {
        g_err = e.what();
        return 10;
    } catch (const CorruptManifestError& e) {
        g_err = e.what();
        return 11;
    } catch (const SizeMismatchError& e) {
        g_err = e.what();
        return 12;
    } catch (const IoError& e) {
        g_err = e.what();
        return 9;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

// Face kinds as in include/blockoa_b200.h: 0 Dirichlet{u0=a}, 1 Robin{h=a,
// u_inf=b}, 2 adiabatic. The reference has no adiabatic face; it is expressed
// as Robin{1e-300, 0}, which leaves diag and g bitwise
// equal to a zero-flux face.
BoundarySpec make_bc(const int* kind, const double* a, const double* b) {
    BoundarySpec bc;
    for (int f = 0; f < 6; ++f) {
        if (kind[f] == 0)
            bc.faces[f] = Dirichlet{a[f]};
        else if (kind[f] == 1)
            bc.faces[f] = Robin{a[f], b[f]};
        else
            bc.faces[f] = Robin{1e-300, 0.0};
    }
    return bc;
}

SolverConfig make_cfg(double tol, int max_iter, int precond) {
    SolverConfig c;
    c.rel_tol = tol;
    c.max_iter = max_iter;
    c.preconditioner = precond ? SolverConfig::Precond::jacobi : SolverConfig::Precond::none;
    return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- operator ---------------------------------------------------------------
int ref_op_create(int nx, int ny, int nz, double lx, double ly, double lz,
                  const double* k, const int* bc_kind, const double* bc_a,
                  const double* bc_b, void** out) {
    try {
        GridSpec grid{nx, ny, nz, lx, ly, lz};
        ScalarField kf{grid, Unit::conductivity_w_per_m_k,
                       std::vector<double>(k, k + grid.cell_count())};
        auto* op = new DiscreteOperator(assemble(kf, grid, make_bc(bc_kind, bc_a, bc_b)));
        *out = op;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

void ref_op_free(void* op) { delete static_cast<DiscreteOperator*>(op); }

long long ref_op_nnz(const void* op) {
    return static_cast<const DiscreteOperator*>(op)->A.nnz();
}

void ref_op_export(const void* vop, long long* row_ptr, int* col, double* val,
                   double* g, double* vol) {
    const auto* op = static_cast<const DiscreteOperator*>(vop);
    const auto& a = op->A;
    for (std::size_t i = 0; i < a.row_ptr.size(); ++i) row_ptr[i] = a.row_ptr[i];
    std::memcpy(col, a.col.data(), a.col.size() * sizeof(int));
    std::memcpy(val, a.val.data(), a.val.size() * sizeof(double));
    std::memcpy(g, op->g.data(), op->g.size() * sizeof(double));
    std::memcpy(vol, op->volumes.data(), op->volumes.size() * sizeof(double));
}

int ref_apply_block(const void* vop, const double* x, int s, double* y) {
    try {
        static_cast<const DiscreteOperator*>(vop)->A.apply_block(x, s, y);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_apply(const void* vop, const double* x, double* y) {
    try {
        const auto* op = static_cast<const DiscreteOperator*>(vop);
        const auto n = static_cast<std::size_t>(op->A.n);
        std::vector<double> r = apply(*op, std::span<const double>(x, n));
        std::memcpy(y, r.data(), n * sizeof(double));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_rhs_from_power(const void* vop, const double* q, double* b) {
    try {
        const auto* op = static_cast<const DiscreteOperator*>(vop);
        ScalarField qf{op->grid, Unit::power_density_w_per_m3,
                       std::vector<double>(q, q + op->A.n)};
        std::vector<double> r = rhs_from_power(*op, qf);
        std::memcpy(b, r.data(), r.size() * sizeof(double));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_power_from_rhs(const void* vop, const double* b, double* q) {
    try {
        const auto* op = static_cast<const DiscreteOperator*>(vop);
        ScalarField qf = power_from_rhs(*op, std::span<const double>(b, op->A.n));
        std::memcpy(q, qf.values.data(), qf.values.size() * sizeof(double));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

double ref_relative_residual(const void* vop, const double* u, const double* q) {
    const auto* op = static_cast<const DiscreteOperator*>(vop);
    ScalarField qf{op->grid, Unit::power_density_w_per_m3,
                   std::vector<double>(q, q + op->A.n)};
    return relative_residual(*op, std::span<const double>(u, op->A.n), qf);
}

// ---- solvers ----------------------------------------------------------------
// B, X row-major n x s (MultiVector layout, solvers.hpp:55-58).
int ref_block_cg(const void* vop, const double* b, int s, double tol, int max_iter,
                 int precond, double* x, int* iterations, long long* matvecs,
                 double* resid, char* conv, double* wall) {
    try {
        const auto* op = static_cast<const DiscreteOperator*>(vop);
        MultiVector mb;
        mb.n = op->A.n;
        mb.s = s;
        mb.data.assign(b, b + static_cast<std::size_t>(op->A.n) * s);
        BlockCgResult r = block_cg(*op, mb, make_cfg(tol, max_iter, precond));
        std::memcpy(x, r.x.data.data(), r.x.data.size() * sizeof(double));
        *iterations = r.report.iterations;
        *matvecs = r.report.matvec_count;
        for (int j = 0; j < s; ++j) {
            resid[j] = r.report.final_rel_residual[j];
            conv[j] = r.report.converged[j];
        }
        *wall = r.report.wall_time;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_cg(const void* vop, const double* b, double tol, int max_iter, int precond,
           double* x, int* iterations, long long* matvecs, double* resid, char* conv) {
    try {
        const auto* op = static_cast<const DiscreteOperator*>(vop);
        CgResult r = cg(*op, std::span<const double>(b, op->A.n),
                        make_cfg(tol, max_iter, precond));
        std::memcpy(x, r.x.data(), r.x.size() * sizeof(double));
        *iterations = r.report.iterations;
        *matvecs = r.report.matvec_count;
        *resid = r.report.final_rel_residual[0];
        *conv = r.report.converged[0];
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Generic CSR block CG on a caller-provided SPD matrix (SPEC 100x100 case).
int ref_block_cg_csr(long long n, const long long* row_ptr, const int* col,
                     const double* val, const double* b, int s, double tol,
                     int max_iter, int precond, double* x, int* iterations,
                     long long* matvecs, double* resid, char* conv) {
    try {
        CsrMatrix a;
        a.n = n;
        a.row_ptr.assign(row_ptr, row_ptr + n + 1);
        a.col.assign(col, col + row_ptr[n]);
        a.val.assign(val, val + row_ptr[n]);
        MultiVector mb;
        mb.n = n;
        mb.s = s;
        mb.data.assign(b, b + static_cast<std::size_t>(n) * s);
        BlockCgResult r = block_cg(a, mb, make_cfg(tol, max_iter, precond));
        std::memcpy(x, r.x.data.data(), r.x.data.size() * sizeof(double));
        *iterations = r.report.iterations;
        *matvecs = r.report.matvec_count;
        for (int j = 0; j < s; ++j) {
            resid[j] = r.report.final_rel_residual[j];
            conv[j] = r.report.converged[j];
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_cg_csr(long long n, const long long* row_ptr, const int* col, const double* val,
               const double* b, double tol, int max_iter, int precond, double* x,
               int* iterations, long long* matvecs, double* resid, char* conv) {
    try {
        CsrMatrix a;
        a.n = n;
        a.row_ptr.assign(row_ptr, row_ptr + n + 1);
        a.col.assign(col, col + row_ptr[n]);
        a.val.assign(val, val + row_ptr[n]);
        CgResult r = cg(a, std::span<const double>(b, n), make_cfg(tol, max_iter, precond));
        std::memcpy(x, r.x.data(), r.x.size() * sizeof(double));
        *iterations = r.report.iterations;
        *matvecs = r.report.matvec_count;
        *resid = r.report.final_rel_residual[0];
        *conv = r.report.converged[0];
        return 0;
    } catch (...) {
        return map_exception();
    }
}

double ref_cg_error_bound(double kappa, int m, double e0, int* status) {
    try {
        *status = 0;
        return cg_error_bound(kappa, m, e0);
    } catch (...) {
        *status = map_exception();
        return 0.0;
    }
}

// ---- combination + operator action (one basis group) --------------------------
// X row-major n x s (the group's solved basis), C row-major s x N (column j =
// sample j's weights). T, Q sample-major N x n; resid per sample is the
// reference relative_residual(op, T_j, Q_j). Samples run in parallel_for
// (parallel.hpp:14-34) over `threads` workers, as generate_blockoa does.
int ref_combine_action(const void* vop, const double* x, int s, const double* c,
                       long long n_samples, double* t_out, double* q_out,
                       double* resid, int threads) {
    try {
        const auto* op = static_cast<const DiscreteOperator*>(vop);
        const std::int64_t n = op->A.n;
        BasisSet basis;
        basis.groups.resize(1);
        BasisGroup& grp = basis.groups[0];
        grp.op = *op;
        grp.x.n = n;
        grp.x.s = s;
        grp.x.data.assign(x, x + static_cast<std::size_t>(n) * s);
        parallel_for(0, n_samples, threads, [&](std::int64_t j) {
            std::vector<double> w(static_cast<std::size_t>(s));
            for (int t = 0; t < s; ++t) w[t] = c[static_cast<std::size_t>(t) * n_samples + j];
            std::vector<double> tj = combine_from_weights(basis, w);
            ScalarField qj = operator_action(basis, 0, tj);
            std::memcpy(t_out + j * n, tj.data(), n * sizeof(double));
            std::memcpy(q_out + j * n, qj.values.data(), n * sizeof(double));
            if (resid) resid[j] = relative_residual(*op, tj, qj);
        });
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// The same per-sample path with the basis group built once (the state
// generate_blockoa holds after generate_basis, pipeline.cpp:92-134), so a timed
// call measures only combine_from_weights + operator_action +
// relative_residual for samples [j0, j1) of C (row-major s x n_samples).
void* ref_basis_create(const void* vop, const double* x, int s) {
    try {
        const auto* op = static_cast<const DiscreteOperator*>(vop);
        auto* basis = new BasisSet;
        basis->groups.resize(1);
        BasisGroup& grp = basis->groups[0];
        grp.op = *op;
        grp.x.n = op->A.n;
        grp.x.s = s;
        grp.x.data.assign(x, x + static_cast<std::size_t>(op->A.n) * s);
        return basis;
    } catch (...) {
        map_exception();
        return nullptr;
    }
}

void ref_basis_free(void* b) { delete static_cast<BasisSet*>(b); }

int ref_basis_combine_action(const void* vb, const double* c, long long n_samples, long long j0,
                             long long j1, double* t_out, double* q_out, double* resid,
                             int threads) {
    try {
        const auto* basis = static_cast<const BasisSet*>(vb);
        const BasisGroup& grp = basis->groups[0];
        const int s = grp.x.s;
        const std::int64_t n = grp.x.n;
        parallel_for(j0, j1, threads, [&](std::int64_t j) {
            std::vector<double> w(static_cast<std::size_t>(s));
            for (int t = 0; t < s; ++t) w[t] = c[static_cast<std::size_t>(t) * n_samples + j];
            std::vector<double> tj = combine_from_weights(*basis, w);
            ScalarField qj = operator_action(*basis, 0, tj);
            if (t_out) std::memcpy(t_out + (j - j0) * n, tj.data(), n * sizeof(double));
            if (q_out) std::memcpy(q_out + (j - j0) * n, qj.values.data(), n * sizeof(double));
            if (resid) resid[j - j0] = relative_residual(grp.op, tj, qj);
        });
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// ---- RNG (rng.hpp) ------------------------------------------------------------
unsigned long long ref_derive_seed(unsigned long long seed, const char* tag,
                                   unsigned long long index) {
    return derive_seed(seed, tag, index);
}

void ref_rng_u64(unsigned long long seed, long long n, unsigned long long* out) {
    Rng r(seed);
    for (long long i = 0; i < n; ++i) out[i] = r.next_u64();
}

void ref_rng_uniform(unsigned long long seed, double lo, double hi, long long n,
                     double* out) {
    Rng r(seed);
    for (long long i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}

void ref_rng_normal(unsigned long long seed, long long n, double* out) {
    Rng r(seed);
    for (long long i = 0; i < n; ++i) out[i] = r.normal();
}

void ref_rng_below(unsigned long long seed, unsigned long long bound, long long n,
                   unsigned long long* out) {
    Rng r(seed);
    for (long long i = 0; i < n; ++i) out[i] = r.below(bound);
}

// ---- dataset I/O (dataset_io.hpp) --------------------------------------------
unsigned long long ref_field_digest(int nx, int ny, int nz, const double* values) {
    GridSpec grid{nx, ny, nz, 1.0, 1.0, 1.0};
    ScalarField f{grid, Unit::conductivity_w_per_m_k,
                  std::vector<double>(values, values + grid.cell_count())};
    return field_digest(f);
}

// Dataset from flat sample-major arrays (n_data x n each); timings =
// {basis_solve_s, combine_s, operator_action_s, solve_s, total_s},
// counters = {iterations_total, matvecs_total}.
int ref_write_dataset(const char* dir, int overwrite, int nx, int ny, int nz, double lx,
                      double ly, double lz, const int* bc_kind, const double* bc_a,
                      const double* bc_b, long long n_data, const double* k, const double* q,
                      const double* u, const unsigned long long* ids, const char* method,
                      unsigned long long master_seed, double tol_claimed,
                      const char* tool_version, int n_dig, const unsigned long long* dig_ids,
                      const unsigned long long* digs, const double* timings,
                      const long long* counters, long long requested, long long dropped) {
    try {
        Dataset ds;
        ds.grid = GridSpec{nx, ny, nz, lx, ly, lz};
        ds.bc = make_bc(bc_kind, bc_a, bc_b);
        const std::int64_t n = ds.grid.cell_count();
        ds.samples.resize(static_cast<std::size_t>(n_data));
        for (long long j = 0; j < n_data; ++j) {
            Sample& s = ds.samples[static_cast<std::size_t>(j)];
            s.floorplan_id = ids[j];
            s.k = ScalarField{ds.grid, Unit::conductivity_w_per_m_k,
                              std::vector<double>(k + j * n, k + (j + 1) * n)};
            s.q = ScalarField{ds.grid, Unit::power_density_w_per_m3,
                              std::vector<double>(q + j * n, q + (j + 1) * n)};
            s.u = ScalarField{ds.grid, Unit::temperature_c,
                              std::vector<double>(u + j * n, u + (j + 1) * n)};
        }
        DatasetManifest& m = ds.manifest;
        m.method = method;
        m.n_data = n_data;
        m.master_seed = master_seed;
        for (long long j = 0; j < n_data; ++j) m.floorplan_ids.push_back(ids[j]);
        for (int d = 0; d < n_dig; ++d) m.floorplan_digests.emplace_back(dig_ids[d], digs[d]);
        m.timings.basis_solve_s = timings[0];
        m.timings.combine_s = timings[1];
        m.timings.operator_action_s = timings[2];
        m.timings.solve_s = timings[3];
        m.timings.total_s = timings[4];
        m.timings.iterations_total = counters[0];
        m.timings.matvecs_total = counters[1];
        m.residual_tol_claimed = tol_claimed;
        m.tool_version = tool_version;
        m.requested_n_data = requested;
        m.dropped_count = dropped;
        WriteOptions opts;
        opts.overwrite = overwrite != 0;
        write_dataset(ds, dir, opts);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// read_dataset: call once with k == nullptr to get *n_data and dims/extent,
// then again with arrays of n_data x n (k, q, u) and n_data ids.
int ref_read_dataset(const char* dir, long long* n_data, int* dims, double* extent, double* k,
                     double* q, double* u, unsigned long long* ids) {
    try {
        const Dataset ds = read_dataset(dir);
        *n_data = static_cast<long long>(ds.samples.size());
        dims[0] = ds.grid.nx;
        dims[1] = ds.grid.ny;
        dims[2] = ds.grid.nz;
        extent[0] = ds.grid.lx;
        extent[1] = ds.grid.ly;
        extent[2] = ds.grid.lz;
        if (!k) return 0;
        const std::int64_t n = ds.grid.cell_count();
        for (std::size_t j = 0; j < ds.samples.size(); ++j) {
            std::memcpy(k + j * n, ds.samples[j].k.values.data(), n * sizeof(double));
            std::memcpy(q + j * n, ds.samples[j].q.values.data(), n * sizeof(double));
            std::memcpy(u + j * n, ds.samples[j].u.values.data(), n * sizeof(double));
            ids[j] = ds.samples[j].floorplan_id;
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_validate_dataset(const char* dir, double tol, double* residuals, long long cap,
                         long long* n_out, long long* pass, long long* fail, double* max_res) {
    try {
        const ValidationReport r = validate_dataset(dir, tol);
        *n_out = static_cast<long long>(r.residuals.size());
        for (std::size_t j = 0; j < r.residuals.size() && static_cast<long long>(j) < cap; ++j)
            residuals[j] = r.residuals[j];
        *pass = r.pass_count;
        *fail = r.fail_count;
        *max_res = r.max_residual;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// ---- chip model and the reference-semantics pipeline (default_chip) ---------
// k fields [n_k][n] of build_floorplans(default_chip, n_k, seed) and the basis
// power maps [n_k * eta][n] exactly as generate_basis draws them
// (pipeline.cpp:92-134).
int ref_chip_fields(int nx, int ny, int nz, int n_k, int eta, unsigned long long seed, double* k,
                    double* q) {
    try {
        const ChipSpec spec = ChipSpec::default_chip();
        const GridSpec grid{nx, ny, nz, spec.extent[0], spec.extent[1], spec.extent[2]};
        const std::int64_t n = grid.cell_count();
        const auto fps = build_floorplans(spec, n_k, seed);
        for (int j = 0; j < n_k; ++j) {
            const ScalarField kf = rasterize_conductivity(fps[j], spec, grid);
            std::memcpy(k + j * n, kf.values.data(), n * sizeof(double));
            for (int t = 0; t < eta; ++t) {
                const std::uint64_t ds = derive_seed(seed, "basis", (std::uint64_t)j * eta + t);
                const ScalarField qf =
                    rasterize_power(sample_power(fps[j], spec, ds), fps[j], spec, grid);
                std::memcpy(q + ((std::int64_t)j * eta + t) * n, qf.values.data(), n * sizeof(double));
            }
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// draw_weights(n_basis, sample_seed_for(seed, l + 1)) for l < n_data -> w[n_data][n_basis]
int ref_draw_weights(int n_basis, unsigned long long seed, long long n_data, double* w) {
    try {
        for (long long l = 0; l < n_data; ++l) {
            const auto mu = draw_weights(n_basis, sample_seed_for(seed, l + 1));
            std::memcpy(w + l * n_basis, mu.data(), n_basis * sizeof(double));
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// generate_blockoa on ChipSpec::default_chip() (pipeline.cpp:365-597).
// noise_kind: 0 none, 1 uniform [lo, hi), 2 gaussian sigma. Outputs: k of each
// group [n_k][n], per sample u/q [n_data][n], residual, floorplan id; basis
// iterations per group; wall seconds (PhaseTimings, dataset.hpp:17-25) of the
// basis solve, the whole call, the combination and the operator action.
int ref_generate_blockoa(int nx, int ny, int nz, long long n_data, int n_basis, int n_k,
                         unsigned long long seed, int noise_kind, double lo, double hi,
                         double sigma, double tol, int max_iter, int threads,
                         const int* bc_kind, const double* bc_a, const double* bc_b, double* k,
                         double* u, double* q, double* resid, long long* fp_id, int* iters,
                         double* seconds) {
    try {
        GenerationConfig cfg;
        cfg.chip = ChipSpec::default_chip();
        cfg.grid = GridSpec{nx, ny, nz, cfg.chip.extent[0], cfg.chip.extent[1], cfg.chip.extent[2]};
        cfg.bc = make_bc(bc_kind, bc_a, bc_b);
        cfg.n_data = n_data;
        cfg.n_basis = n_basis;
        cfg.n_k = n_k;
        cfg.master_seed = seed;
        cfg.noise.kind = noise_kind == 0   ? NoiseConfig::Kind::none
                         : noise_kind == 1 ? NoiseConfig::Kind::uniform
                                           : NoiseConfig::Kind::gaussian;
        cfg.noise.lo = lo;
        cfg.noise.hi = hi;
        cfg.noise.sigma = sigma;
        cfg.solver = make_cfg(tol, max_iter, 1);
        cfg.threads = threads;
        const GenerationResult r = generate_blockoa(cfg);
        const std::int64_t n = cfg.grid.cell_count();
        const auto& ds = r.dataset;
        for (long long l = 0; l < n_data; ++l) {
            const Sample& sm = ds.samples[(std::size_t)l];
            if (u) std::memcpy(u + l * n, sm.u.values.data(), n * sizeof(double));
            if (q) std::memcpy(q + l * n, sm.q.values.data(), n * sizeof(double));
            if (resid) resid[l] = sm.residual;
            if (fp_id) fp_id[l] = (long long)sm.floorplan_id;
            if (k && l < n_k) std::memcpy(k + l * n, sm.k.values.data(), n * sizeof(double));
        }
        if (iters) iters[0] = (int)r.timings.iterations_total;
        if (seconds) {
            seconds[0] = r.timings.basis_solve_s;
            seconds[1] = r.timings.total_s;
            seconds[2] = r.timings.combine_s;
            seconds[3] = r.timings.operator_action_s;
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

}  // extern "C"
