// The C ABI (include/blockoa_b200.h): argument validation with the reference's
// error semantics, host/device pointer staging, and the per-chip pipeline.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <new>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "bk_chip.h"
#include "bk_common.cuh"
#include "bk_synth.h"

namespace bk {

bk_status fail(bk_ctx* ctx, bk_status st, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return st;
}

bk_status workspace(bk_ctx* ctx, int slot, size_t bytes, void** out) {
    if (bytes == 0) bytes = 8;
    if (ctx->ws_bytes[slot] < bytes) {
        if (ctx->ws[slot]) {
            cudaStreamSynchronize(ctx->stream);
            cudaFree(ctx->ws[slot]);
            ctx->ws[slot] = nullptr;
            ctx->ws_bytes[slot] = 0;
        }
        const size_t rounded = (bytes + (1u << 20) - 1) & ~size_t((1u << 20) - 1);
        cudaError_t e = cudaMalloc(&ctx->ws[slot], rounded);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, BK_OOM, std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
        }
        ctx->ws_bytes[slot] = rounded;
    }
    *out = ctx->ws[slot];
    return BK_OK;
}

bk_status read_small(bk_ctx* ctx, void* host_dst, const void* dev_src, size_t bytes) {
    constexpr size_t kMap = 64 << 10, kPiece = 32 << 10;  // the upper half holds post_small's slots
    if (bytes % 4) return fail(ctx, BK_INTERNAL, "read_small: size");
    if (!ctx->hmap) {
        BK_CUDA_TRY(ctx, cudaHostAlloc(&ctx->hmap, kMap, cudaHostAllocMapped));
        BK_CUDA_TRY(ctx, cudaHostGetDevicePointer(&ctx->hmap_dev, ctx->hmap, 0));
    }
    // pieces of at most 32 KiB (the reports of a 64-chip batch are 37 KiB)
    for (size_t off = 0; off < bytes; off += kPiece) {
        const size_t m = std::min(kPiece, bytes - off);
        BK_CUDA_TRY(ctx, launch_copy_words(ctx->stream, (unsigned*)ctx->hmap_dev,
                                           (const unsigned*)((const char*)dev_src + off), m / 4));
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        std::memcpy((char*)host_dst + off, ctx->hmap, m);
    }
    return BK_OK;
}

static constexpr size_t kLookSlot0 = 32 << 10;  // post_small slots: past read_small's words

bk_status post_small(bk_ctx* ctx, int slot, const void* dev_src, size_t bytes) {
    if (bytes > 256 || bytes % 4 || slot < 0 || slot > 1) return fail(ctx, BK_INTERNAL, "post_small: size");
    if (!ctx->hmap) {
        BK_CUDA_TRY(ctx, cudaHostAlloc(&ctx->hmap, 64 << 10, cudaHostAllocMapped));
        BK_CUDA_TRY(ctx, cudaHostGetDevicePointer(&ctx->hmap_dev, ctx->hmap, 0));
    }
    if (!ctx->look_ev[slot]) BK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->look_ev[slot], cudaEventDisableTiming));
    unsigned* dst = (unsigned*)((char*)ctx->hmap_dev + kLookSlot0 + 256 * slot);
    BK_CUDA_TRY(ctx, launch_copy_words(ctx->stream, dst, (const unsigned*)dev_src, bytes / 4));
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaEventRecord(ctx->look_ev[slot], ctx->stream));
    return BK_OK;
}

bk_status wait_small(bk_ctx* ctx, int slot, void* host_dst, size_t bytes) {
    if (bytes > 256 || slot < 0 || slot > 1 || !ctx->look_ev[slot]) return fail(ctx, BK_INTERNAL, "wait_small");
    BK_CUDA_TRY(ctx, cudaEventSynchronize(ctx->look_ev[slot]));
    std::memcpy(host_dst, (const char*)ctx->hmap + kLookSlot0 + 256 * slot, bytes);
    return BK_OK;
}

cudaError_t set_max_smem(const void* f, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> given;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    size_t& g = given[{dev, f}];
    if (bytes <= g) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) g = bytes;
    return e;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace bk

namespace {

using namespace bk;

// A device view of a caller buffer: either the caller's device pointer or a
// workspace slot filled from / drained to host memory.
struct Staged {
    double* dev = nullptr;
    bool host = false;
};

bk_status stage_in(bk_ctx* ctx, int slot, const double* p, size_t count, Staged* out) {
    if (is_device_ptr(p)) {
        out->dev = const_cast<double*>(p);
        out->host = false;
        return BK_OK;
    }
    void* d;
    bk_status st = workspace(ctx, slot, count * sizeof(double), &d);
    if (st != BK_OK) return st;
    if (count)
        BK_CUDA_TRY(ctx, cudaMemcpyAsync(d, p, count * sizeof(double), cudaMemcpyHostToDevice,
                                         ctx->stream));
    out->dev = (double*)d;
    out->host = true;
    return BK_OK;
}

bk_status stage_out(bk_ctx* ctx, int slot, double* p, size_t count, Staged* out) {
    if (!p) {
        out->dev = nullptr;
        out->host = false;
        return BK_OK;
    }
    if (is_device_ptr(p)) {
        out->dev = p;
        out->host = false;
        return BK_OK;
    }
    void* d;
    bk_status st = workspace(ctx, slot, count * sizeof(double), &d);
    if (st != BK_OK) return st;
    out->dev = (double*)d;
    out->host = true;
    return BK_OK;
}

bk_status drain(bk_ctx* ctx, const Staged& s, double* host, size_t count) {
    if (s.host && count)
        BK_CUDA_TRY(ctx, cudaMemcpyAsync(host, s.dev, count * sizeof(double),
                                         cudaMemcpyDeviceToHost, ctx->stream));
    return BK_OK;
}

int kernel_width(int s) { return s <= 8 ? 8 : s <= 16 ? 16 : s <= 32 ? 32 : 64; }

}  // namespace

// shared with bk_stream.cu
namespace bk {

bk_status validate_grid(bk_ctx* ctx, const bk_grid* g) {
    if (!g) return fail(ctx, BK_INVALID_SPEC, "grid: null");
    if (g->nx < 1 || g->ny < 1 || g->nz < 1)
        return fail(ctx, BK_INVALID_SPEC, "grid: cell counts must be >= 1");
    if (!(g->lx > 0.0) || !(g->ly > 0.0) || !(g->lz > 0.0))
        return fail(ctx, BK_INVALID_SPEC, "grid: extents must be positive");
    if (g->dz)
        for (int z = 0; z < g->nz; ++z)
            if (!(g->dz[z] > 0.0))
                return fail(ctx, BK_INVALID_SPEC, "grid: layer thicknesses must be positive");
    return BK_OK;
}

bk_status validate_cfg(bk_ctx* ctx, const bk_solver_cfg* c) {
    if (!c) return fail(ctx, BK_INVALID_CONFIG, "solver: null config");
    if (!(c->rel_tol > 0.0) || !(c->rel_tol < 1.0))
        return fail(ctx, BK_INVALID_CONFIG, "solver: rel_tol must be in (0, 1)");
    if (c->max_iter < 1) return fail(ctx, BK_INVALID_CONFIG, "solver: max_iter must be >= 1");
    return BK_OK;
}

void free_op_buffers(bk_operator* op) {
    cudaFree(op->diag);
    cudaFree(op->cx);
    cudaFree(op->cy);
    cudaFree(op->cz);
    cudaFree(op->g);
    cudaFree(op->dinv);
    cudaFree(op->volz);
    op->diag = op->cx = op->cy = op->cz = op->g = op->dinv = op->volz = nullptr;
    op->volz_cap = 0;
}

// Assemble into `op` (buffers reused when the cell count matches).
bk_status assemble_into(bk_ctx* ctx, const bk_grid* grid, const double* k, const bk_face bc[6],
                        bk_operator* op) {
    bk_status st = validate_grid(ctx, grid);
    if (st != BK_OK) return st;
    for (int f = 0; f < 6; ++f) {
        if (bc[f].kind < 0 || bc[f].kind > 2)
            return fail(ctx, BK_INVALID_SPEC, "boundary: unknown face kind");
        if (bc[f].kind == BK_FACE_ROBIN && !(bc[f].a > 0.0))
            return fail(ctx, BK_NONPOSITIVE_HTC, "boundary: Robin h must be > 0");
    }
    const int64_t n = (int64_t)grid->nx * grid->ny * grid->nz;
    if (n > 2147483647LL)
        return fail(ctx, BK_INVALID_SPEC, "assemble: grid too large for 32-bit column indices");
    if (!k) return fail(ctx, BK_DIMENSION_MISMATCH, "assemble: null conductivity");

    Staged kd;
    if ((st = stage_in(ctx, kSlotK, k, (size_t)n, &kd)) != BK_OK) return st;
    // k > 0 everywhere (discretize.cpp:121-123)
    void* flagp;
    if ((st = workspace(ctx, kSlotFlag, sizeof(int), &flagp)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaMemsetAsync(flagp, 0, sizeof(int), ctx->stream));
    BK_CUDA_TRY(ctx, launch_check_positive(ctx, kd.dev, n, (int*)flagp));

    if (op->n != n || !op->diag) {
        free_op_buffers(op);
        const size_t nb = (size_t)n * sizeof(double);
        BK_CUDA_TRY(ctx, cudaMalloc(&op->diag, nb));
        BK_CUDA_TRY(ctx, cudaMalloc(&op->cx, nb));
        BK_CUDA_TRY(ctx, cudaMalloc(&op->cy, nb));
        BK_CUDA_TRY(ctx, cudaMalloc(&op->cz, nb));
        BK_CUDA_TRY(ctx, cudaMalloc(&op->g, nb));
        BK_CUDA_TRY(ctx, cudaMalloc(&op->dinv, nb));
    }
    if (op->volz_cap < 2 * grid->nz) {
        cudaFree(op->volz);
        op->volz = nullptr;
        op->volz_cap = 0;
        BK_CUDA_TRY(ctx, cudaMalloc(&op->volz, (size_t)grid->nz * 2 * sizeof(double)));
        op->volz_cap = 2 * grid->nz;
    }
    op->device = ctx->device;
    op->nx = grid->nx;
    op->ny = grid->ny;
    op->nz = grid->nz;
    op->n = n;

    // geometry exactly as GridSpec: dx = lx/nx, dy = ly/ny, dz = lz/nz and
    // cell_volume = dx*dy*dz (grid.hpp:25-28)
    const double dx = grid->lx / grid->nx, dy = grid->ly / grid->ny;
    std::vector<double> dzv(grid->nz);
    op->h_volz.assign(grid->nz, 0.0);
    for (int z = 0; z < grid->nz; ++z) {
        dzv[z] = grid->dz ? grid->dz[z] : grid->lz / grid->nz;
        op->h_volz[z] = dx * dy * dzv[z];
    }
    // [volz | dz] in one small upload
    std::vector<double> up(op->h_volz);
    up.insert(up.end(), dzv.begin(), dzv.end());
    BK_CUDA_TRY(ctx, cudaMemcpyAsync(op->volz, up.data(), up.size() * sizeof(double),
                                     cudaMemcpyHostToDevice, ctx->stream));
    BK_CUDA_TRY(ctx, launch_assemble(ctx, op, kd.dev, bc, dx, dy, op->volz + grid->nz));
    int flag = 0;
    if ((st = read_small(ctx, &flag, flagp, sizeof(int))) != BK_OK) return st;
    if (flag) return fail(ctx, BK_NONPOSITIVE_K, "assemble: k must be > 0 everywhere");
    return BK_OK;
}

void fill_report(const CgReport& r, int s, double wall, bk_solve_report* out) {
    if (!out) return;
    out->iterations = r.iterations;
    out->matvec_count = r.matvecs;
    out->wall_time = wall;
    for (int j = 0; j < s; ++j) {
        if (out->final_rel_residual) out->final_rel_residual[j] = r.final_res[j];
        if (out->converged) out->converged[j] = r.converged[j];
    }
}

}  // namespace bk

namespace {

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

// One chip. Host outputs are drained in sample chunks on ctx->copy_stream
// while the next chunk is computed. defer = true (bk_generate_batch) returns
// without waiting for that drain; the device output buffers alternate between
// two parities so chip c+1 computes while chip c drains, and a parity is
// reused only after its previous drain finished.
bk_status generate_chip_impl(bk_ctx* ctx, const bk_grid* grid, const double* k,
                             const bk_face bc[6], const double* Qbasis, int s, const double* C,
                             int64_t N, const bk_solver_cfg* cfg, double* T, double* Q,
                             double* resid, bk_solve_report* report, bk_phase_timings* timings,
                             bool defer, int parity) {
    if (!ctx || !bc) return BK_INVALID_CONFIG;
    bk_status st = validate_cfg(ctx, cfg);
    if (st != BK_OK) return st;
    if (s < 1) return fail(ctx, BK_EMPTY_BASIS, "generate: empty basis");
    if (s > 64) return fail(ctx, BK_INVALID_CONFIG, "generate: s > 64 not supported");
    if (N < 0) return fail(ctx, BK_INVALID_CONFIG, "generate: n_data must be >= 0");
    if ((st = validate_grid(ctx, grid)) != BK_OK) return st;
    cudaSetDevice(ctx->device);
    const int64_t n = (int64_t)grid->nx * grid->ny * grid->nz;
    const int S = kernel_width(s);
    cudaEvent_t* ev = ctx->ev;
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[0], ctx->stream));
    Staged qd, cd;
    if ((st = stage_in(ctx, kSlotQ, Qbasis, (size_t)n * s, &qd)) != BK_OK) return st;
    if ((st = stage_in(ctx, kSlotC, C, (size_t)s * N, &cd)) != BK_OK) return st;
    // k is staged inside assemble
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[1], ctx->stream));

    if (!ctx->scratch) ctx->scratch = new bk_operator;
    bk_operator* scratch = ctx->scratch;
    if ((st = assemble_into(ctx, grid, k, bc, scratch)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[2], ctx->stream));

    void *pb, *px;
    if ((st = workspace(ctx, kSlotIn2, (size_t)n * S * 8, &pb)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotOut2, (size_t)n * S * 8, &px)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, launch_rhs_padded(ctx, scratch, qd.dev, s, (double*)pb, S));
    CgReport rep;
    if ((st = block_cg_device(ctx, scratch, (const double*)pb, S, cfg, (double*)px, &rep)) != BK_OK)
        return st;
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[3], ctx->stream));

    Staged td, qo, rd;
    const size_t out_n = (size_t)n * N;
    // the previous drain of this parity must be done before its buffers are reused
    if (ctx->drain_pending[parity]) {
        BK_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->drain_ev[parity], 0));
        ctx->drain_pending[parity] = false;
    }
    if ((st = stage_out(ctx, parity ? kSlotT1 : kSlotT, T, out_n, &td)) != BK_OK) return st;
    if ((st = stage_out(ctx, parity ? kSlotQo1 : kSlotQo, Q, out_n, &qo)) != BK_OK) return st;
    if ((st = stage_out(ctx, parity ? kSlotRes1 : kSlotRes, resid, (size_t)N, &rd)) != BK_OK)
        return st;
    if (!td.host && !qo.host && !rd.host) {
        if ((st = combine_action_device(ctx, scratch, (const double*)px, S, s, cd.dev, N, N,
                                        td.dev, qo.dev, rd.dev)) != BK_OK)
            return st;
        BK_CUDA_TRY(ctx, cudaEventRecord(ev[4], ctx->stream));
    } else {
        // host outputs: combine in sample chunks (~64 MB of T + q each) and
        // drain each chunk on the copy stream while the next one is computed
        // (D2H of T, q — 16 n bytes per sample over PCIe — is the largest
        // cost of a host-memory call)
        if ((st = ensure_copy_stream(ctx)) != BK_OK) return st;
        const int64_t per = std::max<int64_t>(16, ((int64_t)(64 << 20) / (16 * n)) / 16 * 16);
        const int64_t nch = (N + per - 1) / per;
        while ((int64_t)ctx->chunk_ev.size() < nch) {
            cudaEvent_t e;
            BK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ctx->chunk_ev.push_back(e);
        }
        for (int64_t c = 0; c < nch; ++c) {
            const int64_t j0 = c * per, m = std::min(per, N - j0);
            double* tdev = td.dev ? td.dev + j0 * n : nullptr;
            double* qdev = qo.dev ? qo.dev + j0 * n : nullptr;
            if ((st = combine_action_device(ctx, scratch, (const double*)px, S, s, cd.dev + j0, N,
                                            m, tdev, qdev, rd.dev ? rd.dev + j0 : nullptr)) !=
                BK_OK)
                return st;
            BK_CUDA_TRY(ctx, cudaEventRecord(ctx->chunk_ev[c], ctx->stream));
            BK_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->chunk_ev[c], 0));
            const size_t bytes = (size_t)m * n * sizeof(double);
            if (td.host)
                BK_CUDA_TRY(ctx, cudaMemcpyAsync(T + j0 * n, tdev, bytes, cudaMemcpyDeviceToHost,
                                                 ctx->copy_stream));
            if (qo.host)
                BK_CUDA_TRY(ctx, cudaMemcpyAsync(Q + j0 * n, qdev, bytes, cudaMemcpyDeviceToHost,
                                                 ctx->copy_stream));
        }
        if (rd.host)
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(resid, rd.dev, (size_t)N * sizeof(double),
                                             cudaMemcpyDeviceToHost, ctx->copy_stream));
        BK_CUDA_TRY(ctx, cudaEventRecord(ev[4], ctx->stream));
        BK_CUDA_TRY(ctx, cudaEventRecord(ctx->drain_ev[parity], ctx->copy_stream));
        ctx->drain_pending[parity] = true;
        if (!defer) {  // the call returns with the outputs in host memory
            BK_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->drain_ev[parity], 0));
            ctx->drain_pending[parity] = false;
        }
        td.host = qo.host = rd.host = false;  // drained above
    }
    if ((st = drain(ctx, td, T, out_n)) != BK_OK) return st;
    if ((st = drain(ctx, qo, Q, out_n)) != BK_OK) return st;
    if ((st = drain(ctx, rd, resid, (size_t)N)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[5], ctx->stream));
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));

    const double solve_s = elapsed(ev[2], ev[3]) * 1e-3;
    fill_report(rep, s, solve_s, report);
    if (timings) {
        timings->h2d_s = elapsed(ev[0], ev[1]) * 1e-3;
        timings->assemble_s = elapsed(ev[1], ev[2]) * 1e-3;
        timings->basis_solve_s = solve_s;
        timings->combine_action_s = elapsed(ev[3], ev[4]) * 1e-3;
        timings->d2h_s = elapsed(ev[4], ev[5]) * 1e-3;
        timings->total_s = elapsed(ev[0], ev[5]) * 1e-3;
        timings->iterations_total = rep.iterations;
        timings->matvecs_total = rep.matvecs + N;
    }
    for (int j = 0; j < s; ++j)
        if (!rep.converged[j])
            return fail(ctx, BK_NOT_CONVERGED, "basis solve did not reach tolerance");
    return BK_OK;
}

// Batched pipeline of bk_generate_batch (streams = K > 1): groups of K chips
// of identical dims are assembled into slices of one z-stacked operator (the
// chips' block-diagonal system; boundary face conductances are 0, so no
// coupling), their basis blocks solved by ONE cooperative launch in which
// each chip owns 1/K of the SMs (block_cg_device_multi), then combined per
// chip — all on the context's stream. Persistent solves of several chips thus
// overlap without concurrent cooperative launches (which can starve a
// partially resident grid behind other streams' kernels).
bk_status generate_fused(bk_ctx* ctx, int n_chips, const bk_grid* grids, const double* const* k,
                         const bk_face* bc, const double* const* Qbasis, int s,
                         const double* const* C, int64_t N, const bk_solver_cfg* cfg,
                         double* const* T, double* const* Q, double* const* resid,
                         bk_solve_report* reports, int K, bk_phase_timings* timings) {
    bk_status st = validate_cfg(ctx, cfg);
    if (st != BK_OK) return st;
    if (N < 0) return fail(ctx, BK_INVALID_CONFIG, "generate: n_data must be >= 0");
    const bk_grid& g0 = grids[0];
    const int64_t n = (int64_t)g0.nx * g0.ny * g0.nz;
    const int S = kernel_width(s);
    void *pStack, *pb, *px, *pc;
    if ((st = workspace(ctx, kSlotStackDiag, (size_t)6 * K * n * sizeof(double), &pStack)) != BK_OK)
        return st;
    if ((st = workspace(ctx, kSlotIn2, (size_t)K * n * S * sizeof(double), &pb)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotOut2, (size_t)K * n * S * sizeof(double), &px)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotStackCoef, (size_t)K * s * N * sizeof(double) + 8, &pc)) != BK_OK)
        return st;
    double* const base = (double*)pStack;
    while ((int)ctx->views.size() < K) ctx->views.push_back(new bk_operator);
    cudaEvent_t* ev = ctx->ev;
    float t_asm = 0.f, t_solve = 0.f, t_comb = 0.f;
    int64_t iters = 0, matvecs = 0;
    bool all_conv = true;
    std::vector<CgReport> reps(K);
    for (int c0 = 0; c0 < n_chips; c0 += K) {
        const int Kg = std::min(K, n_chips - c0);
        BK_CUDA_TRY(ctx, cudaEventRecord(ev[0], ctx->stream));
        const double* cdev[64];
        for (int j = 0; j < Kg; ++j) {
            const int c = c0 + j;
            bk_operator* v = ctx->views[j];
            double* arr[6];
            for (int q = 0; q < 6; ++q) arr[q] = base + ((int64_t)q * K + j) * n;
            v->diag = arr[0];
            v->cx = arr[1];
            v->cy = arr[2];
            v->cz = arr[3];
            v->g = arr[4];
            v->dinv = arr[5];
            v->n = n;  // assemble_into fills the slices in place
            if ((st = assemble_into(ctx, &grids[c], k[c], bc + 6 * c, v)) != BK_OK) return st;
            Staged qd;
            if ((st = stage_in(ctx, kSlotQ, Qbasis[c], (size_t)n * s, &qd)) != BK_OK) return st;
            BK_CUDA_TRY(ctx, launch_rhs_padded(ctx, v, qd.dev, s, (double*)pb + (int64_t)j * n * S, S));
            if (is_device_ptr(C[c])) {
                cdev[j] = C[c];
            } else {
                double* dst = (double*)pc + (int64_t)j * s * N;
                BK_CUDA_TRY(ctx, cudaMemcpyAsync(dst, C[c], (size_t)s * N * sizeof(double),
                                                 cudaMemcpyHostToDevice, ctx->stream));
                cdev[j] = dst;
            }
        }
        BK_CUDA_TRY(ctx, cudaEventRecord(ev[1], ctx->stream));
        bk_operator stk = *ctx->views[0];
        stk.nz = g0.nz * Kg;
        stk.n = n * Kg;
        stk.volz = nullptr;
        stk.h_volz.clear();
        if ((st = block_cg_device_multi(ctx, &stk, Kg, (const double*)pb, S, cfg, (double*)px,
                                        reps.data())) != BK_OK)
            return st;
        BK_CUDA_TRY(ctx, cudaEventRecord(ev[2], ctx->stream));
        for (int j = 0; j < Kg; ++j) {
            const int c = c0 + j;
            if ((st = combine_action_device(ctx, ctx->views[j], (const double*)px + (int64_t)j * n * S,
                                            S, s, cdev[j], N, N, T ? T[c] : nullptr,
                                            Q ? Q[c] : nullptr, resid ? resid[c] : nullptr)) != BK_OK)
                return st;
            if (reports) fill_report(reps[j], s, 0.0, &reports[c]);
            iters += reps[j].iterations;
            matvecs += reps[j].matvecs + N;
            for (int q = 0; q < s; ++q) all_conv = all_conv && reps[j].converged[q];
        }
        BK_CUDA_TRY(ctx, cudaEventRecord(ev[3], ctx->stream));
        BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        t_asm += elapsed(ev[0], ev[1]);
        t_solve += elapsed(ev[1], ev[2]);
        t_comb += elapsed(ev[2], ev[3]);
    }
    if (timings) {
        std::memset(timings, 0, sizeof(*timings));
        timings->assemble_s = t_asm * 1e-3;
        timings->basis_solve_s = t_solve * 1e-3;
        timings->combine_action_s = t_comb * 1e-3;
        timings->total_s = (t_asm + t_solve + t_comb) * 1e-3;
        timings->iterations_total = iters;
        timings->matvecs_total = matvecs;
    }
    if (!all_conv) return fail(ctx, BK_NOT_CONVERGED, "basis solve did not reach tolerance");
    return BK_OK;
}


// ---------------------------------------------------------------------------
// generate_blockoa (pipeline.cpp:365-597) with the reference's own semantics
// ---------------------------------------------------------------------------
// all groups' basis columns side by side: Xall[i][j eta + t] = X_j[i][t]
// (groups ascending, columns ascending: combine_tile16's term order), zero
// past n_basis up to the kernel width SB
__global__ void pack_basis_kernel(const double* __restrict__ X, int64_t n, int S, int eta, int nk,
                                  int SB, double* __restrict__ Xall) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n * SB) return;
    const int64_t i = e / SB;
    const int c = (int)(e % SB), j = c / eta, t = c % eta;
    Xall[e] = j < nk ? X[((int64_t)j * n + i) * S + t] : 0.0;
}

// Interior noise of sample l, one thread per sample: its own xoshiro256**
// stream (Rng(derive_seed(sample_seed, "eps")), pipeline.cpp:158-172, 470-503)
// walked over the interior cells in z, y, x order; uniform(lo, hi) evaluated
// as the reference build does (fused lo + u (hi - lo)). Boundary-adjacent
// cells stay zero (the buffer is cleared first).
__global__ void noise_uniform_kernel(const uint64_t* __restrict__ state, int64_t N, int nx, int ny,
                                     int nz, double lo, double hi, double* __restrict__ eps) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= N) return;
    uint64_t s0 = state[4 * l], s1 = state[4 * l + 1], s2 = state[4 * l + 2], s3 = state[4 * l + 3];
    const int64_t n = (int64_t)nx * ny * nz;
    double* e = eps + l * n;
    const double span = hi - lo;
    for (int iz = 1; iz + 1 < nz; ++iz)
        for (int iy = 1; iy + 1 < ny; ++iy)
            for (int ix = 1; ix + 1 < nx; ++ix) {
                const uint64_t x = s1 * 5;
                const uint64_t out = ((x << 7) | (x >> 57)) * 9;
                const uint64_t tt = s1 << 17;
                s2 ^= s0;
                s3 ^= s1;
                s1 ^= s2;
                s0 ^= s3;
                s2 ^= tt;
                s3 = (s3 << 45) | (s3 >> 19);
                const double u = (double)(out >> 11) * 0x1.0p-53;
                e[ix + (int64_t)nx * (iy + (int64_t)ny * iz)] = __fma_rn(u, span, lo);
            }
}

bk_status generate_blockoa_impl(bk_ctx* ctx, const bk_blockoa_cfg* cfg, double* k_out, double* U,
                                double* Q, double* resid, int64_t* fp_out,
                                bk_solve_report* reports, bk_phase_timings* timings) {
    if (!cfg) return fail(ctx, BK_INVALID_CONFIG, "generate_blockoa: null config");
    bk_status st = validate_cfg(ctx, &cfg->solver);
    if (st != BK_OK) return st;
    // GenerationConfig::validate (pipeline.cpp) and the limits of this path
    const int nk = cfg->n_k;
    if (nk < 1 || cfg->n_basis < 1 || cfg->n_basis % nk)
        return fail(ctx, BK_INVALID_CONFIG, "generate_blockoa: n_basis must be a positive multiple of n_k");
    if (cfg->n_data < 0) return fail(ctx, BK_INVALID_CONFIG, "generate_blockoa: n_data must be >= 0");
    const int eta = cfg->n_basis / nk;
    if (cfg->n_basis > 64 || eta > 32 || nk > 64)
        return fail(ctx, BK_INVALID_CONFIG,
                    "generate_blockoa: this path supports n_basis <= 64, eta <= 32, n_k <= 64");
    if (cfg->noise_kind < BK_NOISE_NONE || cfg->noise_kind > BK_NOISE_GAUSSIAN)
        return fail(ctx, BK_INVALID_CONFIG, "noise: unknown kind");
    if (cfg->noise_kind == BK_NOISE_UNIFORM && !(cfg->noise_lo <= cfg->noise_hi))
        return fail(ctx, BK_INVALID_CONFIG, "noise: uniform needs lo <= hi");
    if (cfg->noise_kind == BK_NOISE_GAUSSIAN && !(cfg->noise_sigma >= 0.0))
        return fail(ctx, BK_INVALID_CONFIG, "noise: gaussian needs sigma >= 0");
    const bk_chip_spec& chip = cfg->chip;
    bk_grid grid{cfg->nx, cfg->ny, cfg->nz, chip.extent[0], chip.extent[1], chip.extent[2], nullptr};
    if ((st = validate_grid(ctx, &grid)) != BK_OK) return st;
    const int64_t n = (int64_t)grid.nx * grid.ny * grid.nz, N = cfg->n_data;
    const int S = kernel_width(eta), SB = kernel_width(cfg->n_basis);

    cudaEvent_t* ev = ctx->ev;
    const auto t_host = std::chrono::steady_clock::now();
    // host: floorplans, k fields, basis power maps (chip model, bit-exact)
    std::vector<double> kf((size_t)nk * n), qm((size_t)nk * eta * n), qt((size_t)n * eta);
    if ((st = bk_chip_fields(&chip, grid.nx, grid.ny, grid.nz, nk, eta, cfg->master_seed, kf.data(),
                             qm.data())) != BK_OK)
        return fail(ctx, st, "generate_blockoa: invalid chip spec");
    // weights, group-major columns: group g's samples l = g, g + n_k, ...
    std::vector<int64_t> off(nk + 1, 0);
    for (int g = 0; g < nk; ++g) off[g + 1] = off[g] + (N > g ? (N - g + nk - 1) / nk : 0);
    std::vector<double> w((size_t)cfg->n_basis * std::max<int64_t>(N, 1)), mu(cfg->n_basis);
    for (int64_t l = 0; l < N; ++l) {
        bk::draw_weights(cfg->n_basis, cfg->master_seed, l, mu.data());
        const int64_t col = off[l % nk] + l / nk;
        for (int c = 0; c < cfg->n_basis; ++c) w[(size_t)c * N + col] = mu[c];
    }
    const double host_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_host).count();

    void *pStack, *pb, *px, *pxa, *peps = nullptr, *pw, *pseed;
    if ((st = workspace(ctx, kSlotStackDiag, (size_t)6 * nk * n * sizeof(double), &pStack)) != BK_OK)
        return st;
    if ((st = workspace(ctx, kSlotIn2, (size_t)nk * n * S * sizeof(double), &pb)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotOut2, (size_t)nk * n * S * sizeof(double), &px)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotBoaX, (size_t)n * SB * sizeof(double), &pxa)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotBoaW, w.size() * sizeof(double), &pw)) != BK_OK) return st;
    while ((int)ctx->views.size() < nk) ctx->views.push_back(new bk_operator);

    BK_CUDA_TRY(ctx, cudaEventRecord(ev[0], ctx->stream));
    double* const base = (double*)pStack;
    for (int j = 0; j < nk; ++j) {
        bk_operator* v = ctx->views[j];
        double* arr[6];
        for (int q = 0; q < 6; ++q) arr[q] = base + ((int64_t)q * nk + j) * n;
        v->diag = arr[0];
        v->cx = arr[1];
        v->cy = arr[2];
        v->cz = arr[3];
        v->g = arr[4];
        v->dinv = arr[5];
        v->n = n;
        if ((st = assemble_into(ctx, &grid, kf.data() + j * n, cfg->bc, v)) != BK_OK) return st;
        // maps [t][n] -> cell-major n x eta, then B = V q + g (rhs_from_power)
        for (int64_t i = 0; i < n; ++i)
            for (int t = 0; t < eta; ++t) qt[i * eta + t] = qm[((size_t)j * eta + t) * n + i];
        Staged qd;
        if ((st = stage_in(ctx, kSlotQ, qt.data(), (size_t)n * eta, &qd)) != BK_OK) return st;
        BK_CUDA_TRY(ctx, launch_rhs_padded(ctx, v, qd.dev, eta, (double*)pb + (int64_t)j * n * S, S));
    }
    BK_CUDA_TRY(ctx, cudaMemcpyAsync(pw, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice,
                                     ctx->stream));
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[1], ctx->stream));
    // ONE batched block-CG launch over the n_k groups (z-stacked, per-group CTA
    // shares, barriers, reductions and convergence control)
    std::vector<CgReport> reps(nk);
    bk_operator stk = *ctx->views[0];
    stk.nz = grid.nz * nk;
    stk.n = n * nk;
    stk.volz = nullptr;
    stk.h_volz.clear();
    if ((st = block_cg_device_multi(ctx, &stk, nk, (const double*)pb, S, &cfg->solver, (double*)px,
                                    reps.data())) != BK_OK)
        return st;
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[2], ctx->stream));
    pack_basis_kernel<<<(unsigned)((n * SB + 255) / 256), 256, 0, ctx->stream>>>(
        (const double*)px, n, S, eta, nk, SB, (double*)pxa);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    // noise: device streams (uniform) or host draws (gaussian: libm Box-Muller)
    if (cfg->noise_kind != BK_NOISE_NONE && N > 0) {
        if ((st = workspace(ctx, kSlotBoaEps, (size_t)N * n * sizeof(double), &peps)) != BK_OK)
            return st;
        if (cfg->noise_kind == BK_NOISE_UNIFORM) {
            std::vector<uint64_t> states((size_t)4 * N);
            for (int64_t l = 0; l < N; ++l) {
                uint64_t sd = bk_derive_seed(
                    bk_derive_seed(cfg->master_seed, "sample", (uint64_t)(l + 1)), "eps", 0);
                for (int q = 0; q < 4; ++q) states[4 * l + q] = bk::sm64(sd);
            }
            if ((st = workspace(ctx, kSlotBoaSeed, states.size() * sizeof(uint64_t), &pseed)) != BK_OK)
                return st;
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(pseed, states.data(), states.size() * sizeof(uint64_t),
                                             cudaMemcpyHostToDevice, ctx->stream));
            BK_CUDA_TRY(ctx, cudaMemsetAsync(peps, 0, (size_t)N * n * sizeof(double), ctx->stream));
            noise_uniform_kernel<<<(unsigned)((N + 63) / 64), 64, 0, ctx->stream>>>(
                (const uint64_t*)pseed, N, grid.nx, grid.ny, grid.nz, cfg->noise_lo, cfg->noise_hi,
                (double*)peps);
            ++ctx->launches;
            BK_CUDA_TRY(ctx, cudaGetLastError());
        } else {
            std::vector<double> eps((size_t)N * n, 0.0);
            for (int64_t l = 0; l < N; ++l) {
                bk::Xoshiro rng(bk_derive_seed(
                    bk_derive_seed(cfg->master_seed, "sample", (uint64_t)(l + 1)), "eps", 0));
                for (int iz = 1; iz + 1 < grid.nz; ++iz)
                    for (int iy = 1; iy + 1 < grid.ny; ++iy)
                        for (int ix = 1; ix + 1 < grid.nx; ++ix)
                            eps[l * n + ix + (int64_t)grid.nx * (iy + (int64_t)grid.ny * iz)] =
                                cfg->noise_sigma * rng.normal();
            }
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(peps, eps.data(), eps.size() * sizeof(double),
                                             cudaMemcpyHostToDevice, ctx->stream));
            BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // eps is a local
        }
    }
    Staged ud, qo, rd;
    if ((st = stage_out(ctx, kSlotBoaU, U, (size_t)N * n, &ud)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotBoaQ, Q, (size_t)N * n, &qo)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotBoaRes, resid, (size_t)N, &rd)) != BK_OK) return st;
    // per group: all groups' basis columns, the group's operator, its samples
    // written with row stride n_k n (sample l = g + m n_k)
    for (int g = 0; g < nk; ++g) {
        const int64_t m = off[g + 1] - off[g];
        if (m == 0) continue;
        ActExtra ex;
        ex.ldo = (int64_t)nk * n;
        ex.rstride = nk;
        ex.eps = peps ? (const double*)peps + g * n : nullptr;
        ex.fma = 1;
        if ((st = combine_action_device(ctx, ctx->views[g], (const double*)pxa, SB, cfg->n_basis,
                                        (const double*)pw + off[g], N, m,
                                        ud.dev ? ud.dev + g * n : nullptr,
                                        qo.dev ? qo.dev + g * n : nullptr,
                                        rd.dev ? rd.dev + g : nullptr, ex)) != BK_OK)
            return st;
    }
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[3], ctx->stream));
    if ((st = drain(ctx, ud, U, (size_t)N * n)) != BK_OK) return st;
    if ((st = drain(ctx, qo, Q, (size_t)N * n)) != BK_OK) return st;
    if ((st = drain(ctx, rd, resid, (size_t)N)) != BK_OK) return st;
    if (k_out) {
        BK_CUDA_TRY(ctx, cudaMemcpyAsync(k_out, kf.data(), kf.size() * sizeof(double),
                                         cudaMemcpyDefault, ctx->stream));
    }
    if (fp_out) {
        std::vector<int64_t> ids(N);
        for (int64_t l = 0; l < N; ++l) ids[l] = l % nk;  // floorplan id = group index
        BK_CUDA_TRY(ctx, cudaMemcpyAsync(fp_out, ids.data(), N * sizeof(int64_t), cudaMemcpyDefault,
                                         ctx->stream));
        BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    }
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[4], ctx->stream));
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    bool all_conv = true;
    int64_t iters = 0, matvecs = 0;
    for (int j = 0; j < nk; ++j) {
        if (reports) fill_report(reps[j], eta, elapsed(ev[1], ev[2]) * 1e-3, &reports[j]);
        iters += reps[j].iterations;
        matvecs += reps[j].matvecs;
        for (int t = 0; t < eta; ++t) all_conv = all_conv && reps[j].converged[t];
    }
    if (timings) {
        std::memset(timings, 0, sizeof(*timings));
        timings->assemble_s = elapsed(ev[0], ev[1]) * 1e-3 + host_s;
        timings->basis_solve_s = elapsed(ev[1], ev[2]) * 1e-3;
        timings->combine_action_s = elapsed(ev[2], ev[3]) * 1e-3;
        timings->d2h_s = elapsed(ev[3], ev[4]) * 1e-3;
        timings->total_s = elapsed(ev[0], ev[4]) * 1e-3 + host_s;
        timings->iterations_total = iters;
        timings->matvecs_total = matvecs + N;
    }
    if (!all_conv) return fail(ctx, BK_NOT_CONVERGED, "basis solve did not reach tolerance");
    return BK_OK;
}

}  // namespace

extern "C" {

int bk_abi_version(void) { return BK_ABI_VERSION; }

bk_status bk_create(int device, bk_ctx** out) {
    if (!out) return BK_INVALID_CONFIG;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return BK_NO_DEVICE;
    }
    if (device < 0 || device >= count) return BK_NO_DEVICE;
    if (cudaSetDevice(device) != cudaSuccess) return BK_CUDA_ERROR;
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (major < 10) return BK_NO_DEVICE;  // built for sm_100a only
    bk_ctx* ctx = new (std::nothrow) bk_ctx;
    if (!ctx) return BK_OOM;
    ctx->device = device;
    if (const char* e = getenv("BK_CG_RING")) ctx->knobs.ring = atoi(e) != 0;
    ctx->knobs.no_resident = getenv("BK_CG_NO_RESIDENT") != nullptr;
    ctx->knobs.force_large = getenv("BK_CG_LARGE") != nullptr;
    ctx->knobs.cg_profile = getenv("BK_CG_PROFILE") != nullptr;
    ctx->knobs.no_tma_spmm = getenv("BK_NO_TMA_SPMM") != nullptr;
    ctx->knobs.comb_profile = getenv("BK_COMB_PROFILE") != nullptr;
    ctx->knobs.batch_trace = getenv("BK_BATCH_TRACE") != nullptr;
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return BK_CUDA_ERROR;
    }
    ctx->stream = ctx->own_stream;
    for (auto& e : ctx->ev) cudaEventCreate(&e);
    *out = ctx;
    return BK_OK;
}

bk_status bk_last_solve_phases(const bk_ctx* ctx, double* ms, int64_t* counts) {
    if (!ctx || !ms || !counts) return BK_INVALID_CONFIG;
    for (int k = 0; k < bk_phase_clock::kKinds; ++k) {
        ms[k] = ctx->pclk.ms[k];
        counts[k] = ctx->pclk.count[k];
    }
    return BK_OK;
}

namespace {
// register-operand DMMA chains: 4 independent accumulators per warp
__global__ void __launch_bounds__(1024, 1) k_fp64_peak(double* out, int iters) {
    double d[4][4];
    for (int c = 0; c < 4; ++c)
        for (int e = 0; e < 4; ++e) d[c][e] = threadIdx.x * 1e-3 + c;
    const double a0 = 1.0000001, a1 = 0.9999999, b = 1.0000002;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
                "{%0,%1,%2,%3};"
                : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                : "d"(a0), "d"(a1), "d"(b));
    double s = 0.0;
    for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][3];
    out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

bk_status bk_measure_fp64_peak(bk_ctx* ctx, double seconds, double* burst_tflops,
                               double* sustained_tflops) {
    if (!ctx || !burst_tflops || !sustained_tflops || !(seconds >= 0.0))
        return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    const int blocks = ctx->num_sms, threads = 1024, iters = 4000;
    const double flops = 2.0 * 16 * 8 * 4 * 4 * (double)iters * (threads / 32) * blocks;
    double* out = nullptr;
    BK_CUDA_TRY(ctx, cudaMalloc(&out, (size_t)blocks * threads * sizeof(double)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto done = [&](bk_status st) {
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        return st;
    };
    cudaStream_t s = ctx->stream;
    k_fp64_peak<<<blocks, threads, 0, s>>>(out, 10);
    float best = 0.f, ms = 0.f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0, s);
        k_fp64_peak<<<blocks, threads, 0, s>>>(out, iters);
        cudaEventRecord(e1, s);
        if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess)
            return done(fail(ctx, BK_CUDA_ERROR, "measure_fp64_peak: burst launch failed"));
        if (r == 0 || ms < best) best = ms;
    }
    *burst_tflops = flops / (best * 1e-3) / 1e12;
    // sustained: enough back-to-back launches to fill `seconds` at the burst rate
    const int n = (int)(seconds * 1e3 / best) + 1;
    cudaEventRecord(e0, s);
    for (int r = 0; r < n; ++r) k_fp64_peak<<<blocks, threads, 0, s>>>(out, iters);
    cudaEventRecord(e1, s);
    if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess)
        return done(fail(ctx, BK_CUDA_ERROR, "measure_fp64_peak: sustained run failed"));
    *sustained_tflops = flops * n / (ms * 1e-3) / 1e12;
    return done(BK_OK);
}

const char* bk_last_solver_variant(const bk_ctx* ctx) {
    return ctx ? ctx->last_variant.c_str() : "";
}

bk_status bk_set_option(bk_ctx* ctx, const char* name, int value) {
    if (!ctx || !name) return BK_INVALID_CONFIG;
    const std::string k(name);
    if (k == "ring") ctx->knobs.ring = value < 0 ? -1 : value != 0;
    else if (k == "no_resident") ctx->knobs.no_resident = value != 0;
    else if (k == "force_large") ctx->knobs.force_large = value != 0;
    else if (k == "cg_profile") ctx->knobs.cg_profile = value != 0;
    else if (k == "no_tma_spmm") ctx->knobs.no_tma_spmm = value != 0;
    else if (k == "comb_profile") ctx->knobs.comb_profile = value != 0;
    else if (k == "batch_trace") ctx->knobs.batch_trace = value != 0;
    else if (k == "phase_timing") ctx->knobs.phase_timing = value != 0;
    else if (k == "no_ws_update") ctx->knobs.no_ws_update = value != 0;
    else if (k == "no_ws_spmm") ctx->knobs.no_ws_spmm = value != 0;
    else if (k == "no_defer_x") ctx->knobs.no_defer_x = value != 0;
    else if (k == "no_w_prefetch") ctx->knobs.no_w_prefetch = value != 0;
    else if (k == "graph_loop") ctx->knobs.graph_loop = value != 0;
    else if (k == "no_lookahead") ctx->knobs.no_lookahead = value != 0;
    else if (k == "spmm_teams") ctx->knobs.spmm_teams = value != 0;
    else if (k == "spmm_band") ctx->knobs.spmm_band = value;
    else if (k == "comb_one_role") ctx->knobs.comb_one_role = value != 0;
    else return fail(ctx, BK_INVALID_CONFIG, "bk_set_option: unknown option " + k);
    return BK_OK;
}

void bk_destroy(bk_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->out_ctx) bk_destroy(ctx->out_ctx);
    for (cudaEvent_t e : ctx->pclk.ev) cudaEventDestroy(e);
    for (bk_operator* o : ctx->stream_ops)
        if (o) {
            free_op_buffers(o);
            delete o;
        }
    for (int i = 0; i < bk_ctx::kSlots; ++i) cudaFree(ctx->ws[i]);
    for (auto& e : ctx->ev) cudaEventDestroy(e);
    for (auto& e : ctx->look_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->chunk_ev) cudaEventDestroy(e);
    for (auto& e : ctx->drain_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    if (ctx->scratch) {
        free_op_buffers(ctx->scratch);
        delete ctx->scratch;
    }
    for (bk_operator* v : ctx->views) {  // slices of a workspace: only volz is owned
        cudaFree(v->volz);
        delete v;
    }
    if (ctx->hmap) cudaFreeHost(ctx->hmap);
    for (void* p : ctx->pin)
        if (p) cudaFreeHost(p);
    for (auto& e : ctx->stage_ev)
        if (e) cudaEventDestroy(e);
    cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

const char* bk_last_error(const bk_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

bk_status bk_set_stream(bk_ctx* ctx, void* s) {
    if (!ctx) return BK_INVALID_CONFIG;
    ctx->stream = (cudaStream_t)s;
    return BK_OK;
}

bk_status bk_use_own_stream(bk_ctx* ctx) {
    if (!ctx) return BK_INVALID_CONFIG;
    ctx->stream = ctx->own_stream;
    return BK_OK;
}

bk_status bk_synchronize(bk_ctx* ctx) {
    if (!ctx) return BK_INVALID_CONFIG;
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
}

int64_t bk_launch_count(const bk_ctx* ctx) {
    if (!ctx) return 0;
    return ctx->launches;
}

bk_status bk_assemble(bk_ctx* ctx, const bk_grid* grid, const double* k, const bk_face bc[6],
                      bk_operator** out) {
    if (!ctx || !out || !bc) return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    bk_operator* op = new (std::nothrow) bk_operator;
    if (!op) return fail(ctx, BK_OOM, "assemble: host allocation");
    bk_status st = assemble_into(ctx, grid, k, bc, op);
    if (st != BK_OK) {
        free_op_buffers(op);
        delete op;
        return st;
    }
    *out = op;
    return BK_OK;
}

bk_status bk_assemble_into(bk_ctx* ctx, const bk_grid* grid, const double* k, const bk_face bc[6],
                           bk_operator* op) {
    if (!ctx || !op || !bc) return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    if (op->diag && op->device != ctx->device)
        return fail(ctx, BK_INVALID_CONFIG, "assemble_into: operator lives on another device");
    return assemble_into(ctx, grid, k, bc, op);
}

void bk_operator_free(bk_operator* op) {
    if (!op) return;
    cudaSetDevice(op->device);
    free_op_buffers(op);
    delete op;
}

int64_t bk_operator_n(const bk_operator* op) { return op ? op->n : 0; }

bk_status bk_operator_export_csr(bk_ctx* ctx, const bk_operator* op, int64_t* row_ptr,
                                 int32_t* col, double* val, int64_t* nnz, double* g,
                                 double* vol) {
    if (!ctx || !op || !row_ptr || !nnz) return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    const int64_t n = op->n;
    std::vector<double> d(n), cx(n), cy(n), cz(n), gg(n);
    BK_CUDA_TRY(ctx, cudaMemcpy(d.data(), op->diag, n * 8, cudaMemcpyDeviceToHost));
    BK_CUDA_TRY(ctx, cudaMemcpy(cx.data(), op->cx, n * 8, cudaMemcpyDeviceToHost));
    BK_CUDA_TRY(ctx, cudaMemcpy(cy.data(), op->cy, n * 8, cudaMemcpyDeviceToHost));
    BK_CUDA_TRY(ctx, cudaMemcpy(cz.data(), op->cz, n * 8, cudaMemcpyDeviceToHost));
    BK_CUDA_TRY(ctx, cudaMemcpy(gg.data(), op->g, n * 8, cudaMemcpyDeviceToHost));
    const int nx = op->nx, ny = op->ny, nz = op->nz;
    const int64_t plane = (int64_t)nx * ny;
    int64_t p = 0;
    row_ptr[0] = 0;
    // push order z-, y-, x-, diag, x+, y+, z+ skipping zero off-diagonals
    // (discretize.cpp:218-231); pure copies / negations of the stencil.
    auto push = [&](int64_t c, double v) {
        if (col) col[p] = (int32_t)c;
        if (val) val[p] = v;
        ++p;
    };
    for (int64_t i = 0; i < n; ++i) {
        const int ix = (int)(i % nx), iy = (int)((i / nx) % ny), iz = (int)(i / plane);
        if (iz > 0 && cz[i - plane] != 0.0) push(i - plane, -cz[i - plane]);
        if (iy > 0 && cy[i - nx] != 0.0) push(i - nx, -cy[i - nx]);
        if (ix > 0 && cx[i - 1] != 0.0) push(i - 1, -cx[i - 1]);
        push(i, d[i]);
        if (ix < nx - 1 && cx[i] != 0.0) push(i + 1, -cx[i]);
        if (iy < ny - 1 && cy[i] != 0.0) push(i + nx, -cy[i]);
        if (iz < nz - 1 && cz[i] != 0.0) push(i + plane, -cz[i]);
        row_ptr[i + 1] = p;
        if (g) g[i] = gg[i];
        if (vol) vol[i] = op->h_volz[iz];
    }
    *nnz = p;
    return BK_OK;
}

bk_status bk_operator_from_csr(bk_ctx* ctx, const bk_grid* grid, const int64_t* row_ptr,
                               const int32_t* col, const double* val, const double* g,
                               const double* vol, bk_operator** out) {
    if (!ctx || !out || !row_ptr) return BK_INVALID_CONFIG;
    bk_status st = validate_grid(ctx, grid);
    if (st != BK_OK) return st;
    cudaSetDevice(ctx->device);
    const int nx = grid->nx, ny = grid->ny, nz = grid->nz;
    const int64_t plane = (int64_t)nx * ny, n = plane * nz;
    if (n > 2147483647LL) return fail(ctx, BK_INVALID_SPEC, "from_csr: grid too large");
    if (row_ptr[0] != 0) return fail(ctx, BK_INVALID_SPEC, "from_csr: row_ptr[0] != 0");
    if (row_ptr[n] > 0 && (!col || !val))
        return fail(ctx, BK_INVALID_SPEC, "from_csr: null col / val");
    std::vector<double> d(n, 0.0), cx(n, 0.0), cy(n, 0.0), cz(n, 0.0), dinv(n, 1.0);
    // forward faces from the upper entries; every lower entry must mirror the
    // upper one bitwise (interior_conductance is commutative, so the
    // reference's matrix is exactly symmetric)
    for (int64_t i = 0; i < n; ++i) {
        const int64_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
        if (p1 < p0) return fail(ctx, BK_INVALID_SPEC, "from_csr: row_ptr not monotone");
        const int ix = (int)(i % nx), iy = (int)((i / nx) % ny), iz = (int)(i / plane);
        bool has_diag = false, lo_x = false, lo_y = false, lo_z = false;
        for (int64_t p = p0; p < p1; ++p) {
            const int64_t c = col[p];
            const double v = val[p];
            if (c == i) {
                d[i] = v;
                has_diag = true;
            } else if (c == i + 1 && ix < nx - 1) {
                cx[i] = -v;
            } else if (c == i + nx && iy < ny - 1) {
                cy[i] = -v;
            } else if (c == i + plane && iz < nz - 1) {
                cz[i] = -v;
            } else if (c == i - 1 && ix > 0) {
                lo_x = true;
                if (!(-v == cx[i - 1]) || cx[i - 1] == 0.0)
                    return fail(ctx, BK_INVALID_SPEC, "from_csr: matrix is not symmetric");
            } else if (c == i - nx && iy > 0) {
                lo_y = true;
                if (!(-v == cy[i - nx]) || cy[i - nx] == 0.0)
                    return fail(ctx, BK_INVALID_SPEC, "from_csr: matrix is not symmetric");
            } else if (c == i - plane && iz > 0) {
                lo_z = true;
                if (!(-v == cz[i - plane]) || cz[i - plane] == 0.0)
                    return fail(ctx, BK_INVALID_SPEC, "from_csr: matrix is not symmetric");
            } else {
                return fail(ctx, BK_INVALID_SPEC, "from_csr: not a 7-point stencil on this grid");
            }
        }
        // an upper entry of an earlier row needs its mirror in this row
        if ((ix > 0 && cx[i - 1] != 0.0 && !lo_x) || (iy > 0 && cy[i - nx] != 0.0 && !lo_y) ||
            (iz > 0 && cz[i - plane] != 0.0 && !lo_z))
            return fail(ctx, BK_INVALID_SPEC, "from_csr: matrix is not symmetric");
        if (!has_diag) return fail(ctx, BK_INVALID_SPEC, "from_csr: missing diagonal");
        if (d[i] != 0.0) dinv[i] = 1.0 / d[i];
    }
    std::vector<double> vz(nz, 1.0);
    if (vol)
        for (int z = 0; z < nz; ++z) {
            vz[z] = vol[z * plane];
            for (int64_t c = 0; c < plane; ++c)
                if (vol[z * plane + c] != vz[z])
                    return fail(ctx, BK_INVALID_SPEC, "from_csr: volumes must be uniform per z-layer");
        }
    bk_operator* op = new (std::nothrow) bk_operator;
    if (!op) return fail(ctx, BK_OOM, "from_csr: host allocation");
    auto bail = [&](bk_status e, const char* m) {
        free_op_buffers(op);
        delete op;
        return fail(ctx, e, m);
    };
    const size_t nb = (size_t)n * sizeof(double);
    if (cudaMalloc(&op->diag, nb) != cudaSuccess || cudaMalloc(&op->cx, nb) != cudaSuccess ||
        cudaMalloc(&op->cy, nb) != cudaSuccess || cudaMalloc(&op->cz, nb) != cudaSuccess ||
        cudaMalloc(&op->g, nb) != cudaSuccess || cudaMalloc(&op->dinv, nb) != cudaSuccess ||
        cudaMalloc(&op->volz, (size_t)2 * nz * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return bail(BK_OOM, "from_csr: device allocation");
    }
    op->volz_cap = 2 * nz;
    op->device = ctx->device;
    op->nx = nx;
    op->ny = ny;
    op->nz = nz;
    op->n = n;
    op->h_volz = vz;
    std::vector<double> up(vz);
    for (int z = 0; z < nz; ++z) up.push_back(grid->dz ? grid->dz[z] : grid->lz / nz);
    std::vector<double> gz(n, 0.0);
    if (g) std::memcpy(gz.data(), g, nb);
    const bool ok = cudaMemcpy(op->diag, d.data(), nb, cudaMemcpyHostToDevice) == cudaSuccess &&
                    cudaMemcpy(op->cx, cx.data(), nb, cudaMemcpyHostToDevice) == cudaSuccess &&
                    cudaMemcpy(op->cy, cy.data(), nb, cudaMemcpyHostToDevice) == cudaSuccess &&
                    cudaMemcpy(op->cz, cz.data(), nb, cudaMemcpyHostToDevice) == cudaSuccess &&
                    cudaMemcpy(op->g, gz.data(), nb, cudaMemcpyHostToDevice) == cudaSuccess &&
                    cudaMemcpy(op->dinv, dinv.data(), nb, cudaMemcpyHostToDevice) == cudaSuccess &&
                    cudaMemcpy(op->volz, up.data(), up.size() * sizeof(double),
                               cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        return bail(BK_CUDA_ERROR, "from_csr: upload");
    }
    *out = op;
    return BK_OK;
}

bk_status bk_apply_block(bk_ctx* ctx, const bk_operator* op, const double* X, int s, double* Y) {
    if (!ctx || !op) return BK_INVALID_CONFIG;
    if (s < 1) return fail(ctx, BK_DIMENSION_MISMATCH, "apply_block: s must be >= 1");
    cudaSetDevice(ctx->device);
    const size_t cnt = (size_t)op->n * s;
    Staged xd, yd;
    bk_status st;
    if ((st = stage_in(ctx, kSlotIn0, X, cnt, &xd)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotOut0, Y, cnt, &yd)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, launch_apply_block(ctx, op, xd.dev, s, yd.dev));
    if ((st = drain(ctx, yd, Y, cnt)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
}

bk_status bk_rhs_from_power(bk_ctx* ctx, const bk_operator* op, const double* Q, int s,
                            double* B) {
    if (!ctx || !op) return BK_INVALID_CONFIG;
    if (s < 1) return fail(ctx, BK_DIMENSION_MISMATCH, "rhs_from_power: s must be >= 1");
    cudaSetDevice(ctx->device);
    const size_t cnt = (size_t)op->n * s;
    Staged qd, bd;
    bk_status st;
    if ((st = stage_in(ctx, kSlotIn0, Q, cnt, &qd)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotOut0, B, cnt, &bd)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, launch_rhs_from_power(ctx, op, qd.dev, s, bd.dev));
    if ((st = drain(ctx, bd, B, cnt)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
}

bk_status bk_power_from_rhs(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                            double* Q) {
    if (!ctx || !op) return BK_INVALID_CONFIG;
    if (s < 1) return fail(ctx, BK_DIMENSION_MISMATCH, "power_from_rhs: s must be >= 1");
    cudaSetDevice(ctx->device);
    const size_t cnt = (size_t)op->n * s;
    Staged bd, qd;
    bk_status st;
    if ((st = stage_in(ctx, kSlotIn0, B, cnt, &bd)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotOut0, Q, cnt, &qd)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, launch_power_from_rhs(ctx, op, bd.dev, s, qd.dev));
    if ((st = drain(ctx, qd, Q, cnt)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
}

bk_status bk_block_cg(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                      const bk_solver_cfg* cfg, double* X, bk_solve_report* report) {
    if (!ctx || !op) return BK_INVALID_CONFIG;
    bk_status st = validate_cfg(ctx, cfg);
    if (st != BK_OK) return st;
    if (s < 1) return fail(ctx, BK_DIMENSION_MISMATCH, "block_cg: need at least one column");
    if (s > 64) return fail(ctx, BK_INVALID_CONFIG, "block_cg: s > 64 not supported");
    cudaSetDevice(ctx->device);
    const size_t cnt = (size_t)op->n * s;
    Staged bd, xd;
    if ((st = stage_in(ctx, kSlotIn0, B, cnt, &bd)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotOut0, X, cnt, &xd)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaEventRecord(ctx->ev[0], ctx->stream));
    CgReport rep;
    if ((st = block_cg_device(ctx, op, bd.dev, s, cfg, xd.dev, &rep)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaEventRecord(ctx->ev[1], ctx->stream));
    if ((st = drain(ctx, xd, X, cnt)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    fill_report(rep, s, elapsed(ctx->ev[0], ctx->ev[1]) * 1e-3, report);
    return BK_OK;
}

bk_status bk_combine_action(bk_ctx* ctx, const bk_operator* op, const double* X, int s,
                            const double* C, int64_t N, double* T, double* Q, double* resid) {
    if (!ctx || !op) return BK_INVALID_CONFIG;
    if (s < 1) return fail(ctx, BK_EMPTY_BASIS, "combine: empty basis");
    if (s > 64) return fail(ctx, BK_INVALID_CONFIG, "combine: s > 64 not supported");
    if (N < 0) return fail(ctx, BK_DIMENSION_MISMATCH, "combine: negative sample count");
    cudaSetDevice(ctx->device);
    if (N == 0) return BK_OK;
    const int S = kernel_width(s);
    const size_t xn = (size_t)op->n * s, out_n = (size_t)op->n * N;
    Staged xd, cd, td, qd, rd;
    bk_status st;
    if ((st = stage_in(ctx, kSlotIn0, X, xn, &xd)) != BK_OK) return st;
    if ((st = stage_in(ctx, kSlotIn1, C, (size_t)s * N, &cd)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotOut0, T, out_n, &td)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotOut1, Q, out_n, &qd)) != BK_OK) return st;
    if ((st = stage_out(ctx, kSlotOut2, resid, (size_t)N, &rd)) != BK_OK) return st;
    const double* xk = xd.dev;
    if (S != s) {
        void* p;
        if ((st = workspace(ctx, kSlotCgX, (size_t)op->n * S * 8, &p)) != BK_OK) return st;
        BK_CUDA_TRY(ctx, launch_pad_cols(ctx, xd.dev, s, (double*)p, S, op->n));
        xk = (const double*)p;
    }
    // the kernel reads C rows [0, s) with row stride N
    if ((st = combine_action_device(ctx, op, xk, S, s, cd.dev, N, N, td.dev, qd.dev, rd.dev)) !=
        BK_OK)
        return st;
    if ((st = drain(ctx, td, T, out_n)) != BK_OK) return st;
    if ((st = drain(ctx, qd, Q, out_n)) != BK_OK) return st;
    if ((st = drain(ctx, rd, resid, (size_t)N)) != BK_OK) return st;
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
}

bk_status bk_dd_combine_action(bk_ctx* ctx, const bk_operator* op, int y0, int nyl, int S,
                               const double* Xloc, int s, const double* C, int64_t N,
                               double* Tloc, double* Qloc, double* nd) {
    if (!ctx || !op || !Xloc || !C) return BK_INVALID_CONFIG;
    if (s < 1 || s > S || (S != 8 && S != 16 && S != 32 && S != 64))
        return fail(ctx, BK_INVALID_CONFIG, "dd_combine_action: bad widths");
    if (op->nz < 2) return fail(ctx, BK_INVALID_CONFIG, "dd_combine_action: slabs need nz > 1");
    if (y0 < 0 || nyl < 1 || y0 + nyl > op->ny)
        return fail(ctx, BK_DIMENSION_MISMATCH, "dd_combine_action: slab outside the grid");
    if (N < 0) return fail(ctx, BK_DIMENSION_MISMATCH, "dd_combine_action: negative sample count");
    for (const void* p : {(const void*)Xloc, (const void*)C, (const void*)Tloc, (const void*)Qloc,
                          (const void*)nd})
        if (p && !is_device_ptr(p))
            return fail(ctx, BK_INVALID_CONFIG, "dd_combine_action: device pointers only");
    cudaSetDevice(ctx->device);
    if (N == 0) return BK_OK;
    ActExtra ex;
    ex.slab_y0 = y0;
    ex.slab_ny = nyl;
    ex.nd_out = nd != nullptr;
    return combine_action_device(ctx, op, Xloc, S, s, C, N, N, Tloc, Qloc, nd, ex);
}

bk_status bk_dd_resid_from_nd(bk_ctx* ctx, const double* nd, int64_t N, double* resid) {
    if (!ctx || !nd || !resid) return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    BK_CUDA_TRY(ctx, launch_resid_from_nd(ctx->stream, nd, N, resid));
    ++ctx->launches;
    return BK_OK;
}

bk_status bk_generate_chip(bk_ctx* ctx, const bk_grid* grid, const double* k, const bk_face bc[6],
                           const double* Qbasis, int s, const double* C, int64_t N,
                           const bk_solver_cfg* cfg, double* T, double* Q, double* resid,
                           bk_solve_report* report, bk_phase_timings* timings) {
    return generate_chip_impl(ctx, grid, k, bc, Qbasis, s, C, N, cfg, T, Q, resid, report,
                              timings, false, 0);
}

}  // extern "C"

extern "C" {

bk_status bk_set_cg_sm_budget(bk_ctx* ctx, int max_ctas) {
    if (!ctx || max_ctas < 0) return BK_INVALID_CONFIG;
    ctx->cg_max_ctas = max_ctas;
    return BK_OK;
}

bk_status bk_generate_batch(bk_ctx* ctx, int n_chips, const bk_grid* grids,
                            const double* const* k, const bk_face* bc,
                            const double* const* Qbasis, int s, const double* const* C,
                            int64_t N, const bk_solver_cfg* cfg, double* const* T,
                            double* const* Q, double* const* resid, bk_solve_report* reports,
                            int streams, bk_phase_timings* timings) {
    if (!ctx || n_chips < 0 || !grids || !k || !bc || !Qbasis || !C) return BK_INVALID_CONFIG;
    if (streams < 1) streams = 1;
    if (streams > n_chips && n_chips > 0) streams = n_chips;
    cudaSetDevice(ctx->device);
    // streams > 1: the batched pipeline (one cooperative launch per group of
    // chips) when the chips share dims, fit the persistent solver and write
    // device outputs; otherwise chips run one after another
    if (streams > 1) {
        bool fused = streams <= 64 && s >= 1 && s <= 32;
        const int64_t n0 = (int64_t)grids[0].nx * grids[0].ny * grids[0].nz;
        fused = fused && n0 < ((int64_t)1 << 21) && !ctx->knobs.force_large;
        for (int c = 0; c < n_chips && fused; ++c) {
            fused = grids[c].nx == grids[0].nx && grids[c].ny == grids[0].ny &&
                    grids[c].nz == grids[0].nz;
            for (double* const* out : {T, Q, resid})
                if (out && out[c] && !is_device_ptr(out[c])) fused = false;
        }
        if (fused)
            return generate_fused(ctx, n_chips, grids, k, bc, Qbasis, s, C, N, cfg, T, Q, resid,
                                  reports, streams, timings);
        streams = 1;
    }
    // one chip after another on the caller's context; host outputs of chip c
    // drain over PCIe (copy stream, alternating output parities) while chip
    // c+1 computes
    bk_status first = BK_OK;
    std::string msg;
    bk_phase_timings tot;
    std::memset(&tot, 0, sizeof(tot));
    const auto t0 = std::chrono::steady_clock::now();
    int parity = 0;
    for (int c = 0; c < n_chips; ++c, parity ^= 1) {
        bk_phase_timings pt;
        bk_solve_report* rep = reports ? &reports[c] : nullptr;
        const bk_status r = generate_chip_impl(ctx, &grids[c], k[c], bc + 6 * c, Qbasis[c], s, C[c],
                                               N, cfg, T ? T[c] : nullptr, Q ? Q[c] : nullptr,
                                               resid ? resid[c] : nullptr, rep, &pt, true, parity);
        if (r != BK_OK && first == BK_OK) {
            first = r;
            msg = ctx->err;
            if (r != BK_NOT_CONVERGED) break;
        }
        tot.assemble_s += pt.assemble_s;
        tot.basis_solve_s += pt.basis_solve_s;
        tot.combine_action_s += pt.combine_action_s;
        tot.h2d_s += pt.h2d_s;
        tot.d2h_s += pt.d2h_s;
        tot.iterations_total += pt.iterations_total;
        tot.matvecs_total += pt.matvecs_total;
    }
    // outputs of the last chips are still draining
    if (ctx->copy_stream && cudaStreamSynchronize(ctx->copy_stream) != cudaSuccess && first == BK_OK) {
        first = BK_CUDA_ERROR;
        msg = cudaGetErrorString(cudaGetLastError());
    }
    ctx->drain_pending[0] = ctx->drain_pending[1] = false;
    if (timings) {
        *timings = tot;
        timings->total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (first != BK_OK) return fail(ctx, first, msg);
    return BK_OK;
}

bk_status bk_generate_blockoa(bk_ctx* ctx, const bk_blockoa_cfg* cfg, double* k, double* U,
                              double* Q, double* resid, int64_t* floorplan_id,
                              bk_solve_report* reports, bk_phase_timings* timings) {
    if (!ctx) return BK_INVALID_CONFIG;
    try {  // host-side vectors: no exception may cross the C ABI
        return generate_blockoa_impl(ctx, cfg, k, U, Q, resid, floorplan_id, reports, timings);
    } catch (const std::bad_alloc&) {
        return fail(ctx, BK_OOM, "generate_blockoa: host allocation failed");
    }
}

}  // extern "C"
