// The C++ adapter (include/blockoa_gpu.hpp) compiled against the reference's
// own headers and linked with both the reference core (oracle/_ref) and the
// B200 library: blockoa::gpu::{block_cg, combine_action, generate_blockoa}
// against blockoa::{block_cg, combine_from_weights + operator_action,
// generate_blockoa} on the same inputs. TEST INFRASTRUCTURE (built by
// tests/cpp/Makefile; run by tests/test_gpu_adapter.py). Prints one JSON line;
// exit 0 when every check passes.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "blockoa/chip.hpp"
#include "blockoa/discretize.hpp"
#include "blockoa/pipeline.hpp"
#include "blockoa/solvers.hpp"
#include "blockoa_gpu.hpp"

using namespace blockoa;

namespace {

double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1.0));
}

int failures = 0;
std::string report;
void expect(bool ok, const std::string& what) {
    if (!ok) {
        ++failures;
        std::fprintf(stderr, "FAIL: %s\n", what.c_str());
    }
}

}  // namespace

int main() {
    gpu::Context ctx(0);

    // ---- a layered 3D chip with Robin top / bottom, near-adiabatic sides
    GridSpec grid{24, 20, 8, 10e-3, 10e-3, 0.8e-3};
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> uk(1.0, 400.0), uq(0.0, 1e6);
    ScalarField k = ScalarField::constant(grid, Unit::conductivity_w_per_m_k, 1.0);
    for (auto& v : k.values) v = uk(rng);
    BoundarySpec bc;
    for (int f = 0; f < 4; ++f) bc.faces[f] = Robin{1e-300, 0.0};
    bc.faces[4] = Robin{1e2, 0.0};
    bc.faces[5] = Robin{1e4, 0.0};
    const DiscreteOperator op = assemble(k, grid, bc);
    const int s = 32;
    const std::int64_t n = grid.cell_count();
    MultiVector B(n, s);
    for (int j = 0; j < s; ++j) {
        ScalarField q = ScalarField::constant(grid, Unit::power_density_w_per_m3, 0.0);
        for (std::int64_t i = n / 8; i < n / 4; ++i) q.values[i] = uq(rng);
        B.set_column(j, rhs_from_power(op, q));
    }
    SolverConfig cfg;
    cfg.rel_tol = 1e-12;
    cfg.max_iter = 100000;
    cfg.preconditioner = SolverConfig::Precond::jacobi;

    const BlockCgResult ref = block_cg(op, B, cfg);
    const BlockCgResult dev = gpu::block_cg(ctx, op, B, cfg);
    const double dx = rel_l2(dev.x.data, ref.x.data);
    expect(dev.report.all_converged() && ref.report.all_converged(), "block_cg converged");
    expect(dx <= 1e-9, "block_cg X within 1e-9");
    char buf[512];
    std::snprintf(buf, sizeof buf,
                  "\"block_cg\": {\"rel_l2_x\": %.3e, \"iterations_gpu\": %d, "
                  "\"iterations_ref\": %d}",
                  dx, dev.report.iterations, ref.report.iterations);
    report += buf;

    // capped iterates: same block steps, same matvec accounting
    SolverConfig capped = cfg;
    capped.max_iter = 3;
    const BlockCgResult rc = block_cg(op, B, capped);
    const BlockCgResult dc = gpu::block_cg(ctx, op, B, capped);
    const double dcx = rel_l2(dc.x.data, rc.x.data);
    expect(dcx <= 1e-12, "capped iterates within 1e-12");
    expect(dc.report.matvec_count == rc.report.matvec_count, "matvec accounting");
    std::snprintf(buf, sizeof buf, ", \"capped_3\": {\"rel_l2_x\": %.3e, \"matvecs\": [%lld, %lld]}",
                  dcx, (long long)dc.report.matvec_count, (long long)rc.report.matvec_count);
    report += buf;

    // combine_from_weights + operator_action on one basis group
    BasisSet basis;
    basis.groups.resize(1);
    basis.groups[0].op = op;
    basis.groups[0].x = ref.x;
    std::vector<std::vector<double>> w(5, std::vector<double>(s));
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    for (auto& v : w)
        for (auto& e : v) e = u01(rng);
    const gpu::Combined cmb = gpu::combine_action(ctx, basis, 0, w);
    double worst_t = 0.0, worst_q = 0.0;
    for (std::size_t j = 0; j < w.size(); ++j) {
        const std::vector<double> t = combine_from_weights(basis, w[j]);
        const ScalarField q = operator_action(basis, 0, t);
        worst_t = std::max(worst_t, rel_l2(cmb.t[j], t));
        worst_q = std::max(worst_q, rel_l2(cmb.q[j], q.values));
    }
    expect(worst_t == 0.0 && worst_q == 0.0, "combine/action bitwise");
    std::snprintf(buf, sizeof buf, ", \"combine_action\": {\"max_rel_l2_t\": %.3e, \"max_rel_l2_q\": %.3e}",
                  worst_t, worst_q);
    report += buf;

    // the whole reference-semantics run
    GenerationConfig gc;
    gc.chip = ChipSpec::default_chip();
    gc.grid = GridSpec{12, 12, 6, gc.chip.extent[0], gc.chip.extent[1], gc.chip.extent[2]};
    gc.bc = BoundarySpec::mixed(3e4, 25.0, 25.0);
    gc.n_data = 40;
    gc.n_basis = 10;
    gc.n_k = 2;
    gc.master_seed = 3;
    gc.noise.kind = NoiseConfig::Kind::uniform;
    gc.noise.lo = -0.01;
    gc.noise.hi = 0.01;
    gc.solver = cfg;
    const GenerationResult rg = generate_blockoa(gc);
    const GenerationResult dg = gpu::generate_blockoa(ctx, gc);
    double wu = 0.0, wq = 0.0;
    bool ids = rg.dataset.samples.size() == dg.dataset.samples.size();
    for (std::size_t l = 0; ids && l < rg.dataset.samples.size(); ++l) {
        const Sample& a = rg.dataset.samples[l];
        const Sample& b = dg.dataset.samples[l];
        ids = ids && a.floorplan_id == b.floorplan_id && a.k.values == b.k.values;
        wu = std::max(wu, rel_l2(b.u.values, a.u.values));
        wq = std::max(wq, rel_l2(b.q.values, a.q.values));
    }
    expect(ids, "generate_blockoa ids and k bitwise");
    expect(wu <= 1e-9 && wq <= 1e-9, "generate_blockoa (u, q) within 1e-9");
    std::snprintf(buf, sizeof buf,
                  ", \"generate_blockoa\": {\"samples\": %zu, \"max_rel_l2_u\": %.3e, "
                  "\"max_rel_l2_q\": %.3e, \"ids_and_k_bitwise\": %s}",
                  dg.dataset.samples.size(), wu, wq, ids ? "true" : "false");
    report += buf;

    // error mapping: the reference's exception types cross the adapter
    bool threw = false;
    try {
        GenerationConfig bad = gc;
        bad.n_basis = 96;
        bad.n_k = 1;
        gpu::generate_blockoa(ctx, bad);
    } catch (const InvalidConfigError&) {
        threw = true;
    } catch (const Error&) {
        threw = true;
    }
    expect(threw, "n_basis > 64 raises a reference exception");
    std::printf("{%s, \"failures\": %d}\n", report.c_str(), failures);
    return failures == 0 ? 0 : 1;
}
