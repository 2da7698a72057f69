// Internal declarations shared by the libblockoa_b200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "blockoa_b200.h"

// Every kernel launch goes through BK_LAUNCHED so bk_launch_count() reports the
// number of this library's launches (bench.py's gpu_launches claim).
#define BK_CUDA_TRY(ctx, expr)                                                    \
    do {                                                                          \
        cudaError_t e_ = (expr);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            return bk::fail((ctx), e_ == cudaErrorMemoryAllocation ? BK_OOM       \
                                                                   : BK_CUDA_ERROR, \
                            std::string(#expr) + ": " + cudaGetErrorString(e_));  \
        }                                                                         \
    } while (0)

// Debug / A-B switches of one context: read once from the environment when
// the context is created (BK_CG_RING=0|1, BK_CG_NO_RESIDENT, BK_CG_LARGE,
// BK_CG_PROFILE, BK_NO_TMA_SPMM, BK_COMB_PROFILE, BK_BATCH_TRACE) and
// settable per context through bk_set_option.
struct bk_knobs {
    int ring = -1;             // -1: automatic, 0 / 1: force the row ring off / on
    bool no_resident = false;  // never keep X / R resident in shared memory
    bool force_large = false;  // multi-kernel engine for every solve
    bool cg_profile = false;   // in-kernel phase timestamps (stderr)
    bool no_tma_spmm = false;  // S = 64 phase 1 without TMA
    bool comb_profile = false; // combine/action stage timestamps (stderr)
    bool batch_trace = false;
    bool phase_timing = false; // per-kernel-kind event timing of the multi-kernel solve
    bool no_ws_update = false; // S = 64: the cp.async update sweeps instead of the warp-specialised ones
    bool no_w_prefetch = false;  // persistent block CG: single-buffered W staging in phase 2
    bool no_defer_x = false;   // persistent block CG: X += P alpha in phase 2 even where phase 3 would take it
    bool no_ws_spmm = false;   // S = 64: the per-run TMA stencil sweep instead of the z-marching one
    bool spmm_teams = false;   // S = 64: the two-team stencil sweep instead of the role-split one
    bool comb_one_role = false; // single-plane combine/action: the one-role kernel
    int spmm_band = 0;         // S = 64 stencil sweep: x-runs per y-band (0: default 4)
    bool graph_loop = false;   // multi-kernel solve: device-driven iterations (CUDA graph while-loop)
    bool no_lookahead = false; // multi-kernel solve: the synchronous host loop (one drain per iteration)
};

// Optional per-kernel-kind timing of the multi-kernel solve (option
// "phase_timing"): event pairs around each sweep launch, summed per kind at the
// end of the solve (bk_last_solve_phases). Kinds: 0 stencil-SpMM + Gram,
// 1 R update + S_new, 2 P (+ X) update, 3 other (anchor / verify / restart).
struct bk_phase_clock {
    static constexpr int kKinds = 4;
    std::vector<cudaEvent_t> ev;  // pool, grow-only
    std::vector<int> kind;        // per recorded pair
    size_t used = 0;
    double ms[kKinds] = {};
    int64_t count[kKinds] = {};
};

struct bk_ctx {
    bk_knobs knobs;
    bk_phase_clock pclk;
    std::string last_variant;  // kernel instantiation of the last block-CG solve
    int device = 0;
    int num_sms = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[8] = {};
    std::string err;
    int64_t launches = 0;
    bk_operator* scratch = nullptr;  // operator reused by bk_generate_chip
    int cg_max_ctas = 0;             // 0 = every SM (see bk_set_cg_sm_budget)
    std::vector<bk_operator*> views; // per-chip views into the batched pipeline's stacked operator
    cudaStream_t copy_stream = nullptr;    // D2H of host outputs, overlapped with compute
    std::vector<cudaEvent_t> chunk_ev;     // per-chunk "outputs ready" events
    cudaEvent_t drain_ev[2] = {};          // copy stream done with output parity p
    void* hmap = nullptr;                  // mapped pinned host page for small readbacks
    void* hmap_dev = nullptr;
    cudaEvent_t look_ev[2] = {};          // post_small / wait_small slots
    bool drain_pending[2] = {};
    void* pin[2] = {};                     // pinned staging of the dataset writer / validator
    size_t pin_bytes = 0;
    cudaEvent_t stage_ev[4] = {};
    bk_ctx* out_ctx = nullptr;            // output worker of bk_generate_stream (own streams)
    bk_operator* stream_ops[2] = {};       // per-parity chip operators of bk_generate_stream
    // grow-only device workspace slots
    static constexpr int kSlots = 48;
    void* ws[kSlots] = {};
    size_t ws_bytes[kSlots] = {};
};

// Matrix-free operator: SoA stencil in HBM. cx/cy/cz hold
// the conductance of the face towards +x/+y/+z (0 on the domain boundary);
// the -x/-y/-z conductances are the neighbour's forward faces, bitwise equal
// to what the reference computes for the row (interior_conductance is
// commutative, discretize.cpp:99-105).
struct bk_operator {
    int device = 0;
    int nx = 0, ny = 0, nz = 0;
    int64_t n = 0;
    double* diag = nullptr;
    double* cx = nullptr;
    double* cy = nullptr;
    double* cz = nullptr;
    double* g = nullptr;
    double* dinv = nullptr;  // jacobi_inverse (solvers.cpp:53-66)
    int volz_cap = 0;  // doubles allocated at volz (grown only: no per-call cudaFree,
                       // which would synchronize with in-flight output drains)
    double* volz = nullptr;  // cell volume per z-layer (nz)
    std::vector<double> h_volz;
};

namespace bk {

enum Slot : int {
    kSlotIn0 = 0,   // staged host inputs
    kSlotIn1,
    kSlotIn2,
    kSlotOut0,      // staged outputs
    kSlotOut1,
    kSlotOut2,
    kSlotCgB,       // block CG
    kSlotCgX,
    kSlotCgR,
    kSlotCgP,
    kSlotCgW,
    kSlotCgPart,
    kSlotCgRed,
    kSlotCgCtl,
    kSlotActPart,   // combine/action residual partials
    kSlotK,
    kSlotQ,
    kSlotC,
    kSlotT,         // outputs of bk_generate_chip (parity 0) ...
    kSlotQo,
    kSlotRes,
    kSlotFlag,      // assemble's k > 0 check
    kSlotT1,        // ... and parity 1: a batch drains chip c while chip c+1 computes
    kSlotQo1,
    kSlotRes1,
    kSlotCgBars,    // group barriers of the batched (multi-chip) solve
    kSlotCgFlags,   // phase timestamps of a profiled batched solve
    kSlotStackDiag, // z-stacked operator of the batched pipeline (6 arrays)
    kSlotStackCoef, // per-chip combination coefficients of the batched pipeline
    kSlotValRes,    // per-sample residuals of bk_residuals / bk_validate_samples
    kSlotBoaX,      // bk_generate_blockoa: all groups' basis columns (n x SB)
    kSlotBoaEps,    //   per-sample interior noise (n_data x n)
    kSlotBoaW,      //   weights (n_basis x n_data, group-major columns)
    kSlotBoaSeed,   //   noise stream states
    kSlotBoaU,      //   staged outputs
    kSlotBoaQ,
    kSlotBoaRes,
    kSlotStrX0,     // bk_generate_stream: per-parity basis X and coefficients C
    kSlotStrX1,
    kSlotStrC0,
    kSlotStrC1,
    kSlotCgCoef64,  // S = 64 stencil sweep: coefficients packed per 16-cell run
};

bk_status fail(bk_ctx* ctx, bk_status st, const std::string& msg);

// phase clock (no-ops unless ctx->knobs.phase_timing)
inline void phase_reset(bk_ctx* ctx) {
    ctx->pclk.used = 0;
    ctx->pclk.kind.clear();
    for (int k = 0; k < bk_phase_clock::kKinds; ++k) {
        ctx->pclk.ms[k] = 0.0;
        ctx->pclk.count[k] = 0;
    }
}
inline void phase_mark(bk_ctx* ctx, int kind_or_start) {  // -1: start of a pair
    if (!ctx->knobs.phase_timing) return;
    auto& c = ctx->pclk;
    if (c.used == c.ev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        c.ev.push_back(e);
    }
    cudaEventRecord(c.ev[c.used++], ctx->stream);
    if (kind_or_start >= 0) c.kind.push_back(kind_or_start);
}
inline void phase_collect(bk_ctx* ctx) {
    if (!ctx->knobs.phase_timing) return;
    auto& c = ctx->pclk;
    if (c.used == 0) return;
    cudaEventSynchronize(c.ev[c.used - 1]);
    for (size_t p = 0; p < c.kind.size() && 2 * p + 1 < c.used; ++p) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c.ev[2 * p], c.ev[2 * p + 1]);
        c.ms[c.kind[p]] += ms;
        c.count[c.kind[p]] += 1;
    }
}
// relative_residual for N samples (U, Q: N x n device); resid device, N values
bk_status residuals_device(bk_ctx* ctx, const bk_operator* op, const double* U, const double* Q,
                           int64_t N, double* resid);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when `f` needs more
// than it was already given (once per function and device in steady state):
// the attribute is not rewritten while other streams run the same kernel.
cudaError_t set_max_smem(const void* f, size_t bytes);
// Grow-only workspace; contents are not preserved on growth.
bk_status workspace(bk_ctx* ctx, int slot, size_t bytes, void** out);
bk_status ensure_copy_stream(bk_ctx* ctx);
bool is_device_ptr(const void* p);
// Copy a few bytes device -> host through a kernel writing mapped pinned
// memory (no copy engine: it never queues behind a large in-flight D2H drain)
// and synchronize the stream (in pieces of 32 KiB). bytes a multiple of 4.
bk_status read_small(bk_ctx* ctx, void* host_dst, const void* dev_src, size_t bytes);
// Asynchronous form for the lookahead loop: post_small enqueues the copy into
// slot (0 / 1) of the same mapped page and records an event; wait_small waits
// for that event and copies the words out. bytes <= 256, multiple of 4.
bk_status post_small(bk_ctx* ctx, int slot, const void* dev_src, size_t bytes);
bk_status wait_small(bk_ctx* ctx, int slot, void* host_dst, size_t bytes);
cudaError_t launch_copy_words(cudaStream_t s, unsigned* dst, const unsigned* src, size_t words);

// Kernels' host-side launchers (return cudaError_t of the launch).
cudaError_t launch_assemble(bk_ctx* ctx, const bk_operator* op, const double* k,
                            const bk_face* bc, double dx, double dy, const double* dz_dev);
cudaError_t launch_apply_block(bk_ctx* ctx, const bk_operator* op, const double* x, int s,
                               double* y);
cudaError_t launch_rhs_from_power(bk_ctx* ctx, const bk_operator* op, const double* q, int s,
                                  double* b);
// dst (n x dw) <- src (n x sw): copies min(sw, dw) columns, zero-fills the rest.
cudaError_t launch_pad_cols(bk_ctx* ctx, const double* src, int sw, double* dst, int dw,
                            int64_t n);
// B (n x S) = V Q + g for the first s columns (Q is n x s), zero beyond s.
cudaError_t launch_rhs_padded(bk_ctx* ctx, const bk_operator* op, const double* q, int s,
                              double* b, int S);
// flag = any k <= 0 or NaN
cudaError_t launch_check_positive(bk_ctx* ctx, const double* k, int64_t n, int* flag);
cudaError_t launch_power_from_rhs(bk_ctx* ctx, const bk_operator* op, const double* b, int s,
                                  double* q);

struct CgReport {
    int iterations;
    int64_t matvecs;
    double final_res[64];
    char converged[64];
};

// Device-pointer block CG (X, B are n x s on device). Result report copied to
// host (one small D2H at the end of the solve).
bk_status block_cg_device(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                          const bk_solver_cfg* cfg, double* X, CgReport* rep);
bk_status block_cg_large(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                         const bk_solver_cfg* cfg, double* X, CgReport* rep);


// S = kernel width of X (n x S, zero-padded), s = real basis width (rows of
// C read), C row stride ldc (>= N: a sample sub-range of a wider C).
// K chips of identical dims z-stacked (op: nz = K nz_chip): one cooperative
// launch, chip k on an equal SM share (S = 8, 16, 32). reps: K reports.
bk_status block_cg_device_multi(bk_ctx* ctx, const bk_operator* op, int K, const double* B, int S,
                                const bk_solver_cfg* cfg, double* X, CgReport* reps);
// generate_blockoa's variant of the fused combine + action (bk_generate_blockoa):
// outputs (and eps) with row stride ldo (0: n), resid with stride rstride
// (0: 1), per-sample interior noise eps added to T before the action, and
// apply_block's fused-multiply-add stencil order (fma = 1) instead of the
// scalar apply's multiply + add.
struct ActExtra {
    int64_t ldo = 0;
    int64_t rstride = 0;
    const double* eps = nullptr;
    int fma = 0;
    // y-slab of the decomposition (slab_ny > 0): X in the ghost-row layout,
    // outputs slab-local, `resid` receives per-sample (num, den) partials
    int slab_y0 = 0, slab_ny = 0;
    bool nd_out = false;
};
cudaError_t launch_resid_from_nd(cudaStream_t s, const double* nd, int64_t N, double* resid);
bk_status combine_action_device(bk_ctx* ctx, const bk_operator* op, const double* X, int S,
                                int s, const double* C, int64_t ldc, int64_t N, double* T,
                                double* Q, double* resid, const ActExtra& ex = ActExtra{});

}  // namespace bk
