/*
 * blockoa_b200.h — C ABI of the B200-native BlocKOA data-generation hot path.
 *
 * This is the drop-in boundary for the reference's C++ operator API
 * (/root/reference/proj/core/include/blockoa/*.hpp). Each entry point names the
 * reference function it replaces. Plain pointers and sizes only; no C++ or torch
 * types; no exceptions cross the boundary — reference exceptions map 1:1 to
 * bk_status codes (errors.hpp:9-71), with bk_last_error() carrying the message.
 *
 * Data layout contract (bit-exact with the reference):
 *   - cell flat index  i = ix + nx*(iy + ny*iz)          (grid.hpp:30-33)
 *   - face order       x-, x+, y-, y+, z-, z+             (discretize.hpp:26)
 *   - block vectors    row-major n x s, element (i,j) at i*s + j
 *                                                       (MultiVector, solvers.hpp:55-58)
 *   - coefficients C   row-major s x N, column j = sample j's weights
 *   - outputs T, Q     sample-major N x n (one ScalarField per sample,
 *                      Sample{q,u} dataset.hpp:31-38)
 *
 * Every double* argument may be a host pointer (pageable or pinned) or a device
 * pointer on the context's GPU; the library detects which and stages host
 * buffers through its own device workspace.
 *
 * All compute runs on the GPU (sm_100a kernels in libblockoa_b200.so). There is
 * no CPU fallback: without a usable GPU, bk_create returns BK_NO_DEVICE.
 */
#ifndef BLOCKOA_B200_H
#define BLOCKOA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BK_ABI_VERSION 1

typedef enum {
    BK_OK = 0,
    BK_INVALID_SPEC = 1,         /* InvalidSpecError        errors.hpp:14 */
    BK_INVALID_CONFIG = 2,       /* InvalidConfigError      errors.hpp:19 */
    BK_DIMENSION_MISMATCH = 3,   /* DimensionMismatchError  errors.hpp:24 */
    BK_NONPOSITIVE_K = 4,        /* NonPositiveConductivityError errors.hpp:29 */
    BK_NONPOSITIVE_HTC = 5,      /* NonPositiveHtcError     errors.hpp:34 */
    BK_EMPTY_BASIS = 6,          /* EmptyBasisError         errors.hpp:49 */
    BK_NOT_CONVERGED = 7,        /* NotConvergedError       errors.hpp:39 */
    BK_INVALID_KAPPA = 8,        /* InvalidKappaError       errors.hpp:44 */
    BK_IO_ERROR = 9,             /* IoError                 errors.hpp:54 */
    BK_EXISTS = 10,              /* ExistsError             errors.hpp:59 */
    BK_CORRUPT_MANIFEST = 11,    /* CorruptManifestError    errors.hpp:64 */
    BK_SIZE_MISMATCH = 12,       /* SizeMismatchError       errors.hpp:69 */
    BK_CUDA_ERROR = 20,
    BK_OOM = 21,
    BK_NO_DEVICE = 22,
    BK_INTERNAL = 99
} bk_status;

/* Face conditions (discretize.hpp:14-38). BK_FACE_ADIABATIC is the zero-flux
 * face the BASELINE configs need; the reference expresses it as
 * Robin{h=1e-300, u_inf=0}, which assembles to bitwise the same operator. */
typedef enum { BK_FACE_DIRICHLET = 0, BK_FACE_ROBIN = 1, BK_FACE_ADIABATIC = 2 } bk_face_kind;

typedef struct {
    int kind;  /* bk_face_kind */
    double a;  /* Dirichlet: u0 [degC]; Robin: h [W/(m^2 K)] (> 0) */
    double b;  /* Robin: u_inf [degC] */
} bk_face;

/* GridSpec (grid.hpp:14-53) plus an optional per-layer thickness array for
 * non-uniform stacks (BASELINE config 4). dz == NULL: uniform dz = lz/nz. */
typedef struct {
    int nx, ny, nz;
    double lx, ly, lz; /* extents [m] */
    const double* dz;  /* host pointer, nz entries, or NULL */
} bk_grid;

/* SolverConfig (solvers.hpp:13-21). */
typedef struct {
    double rel_tol; /* in (0, 1) */
    int max_iter;   /* >= 1 */
    int precond;    /* 0 none, 1 Jacobi */
} bk_solver_cfg;

/* SolveReport (solvers.hpp:24-32). The two arrays are caller-provided, length s
 * (may be NULL). */
typedef struct {
    int iterations;
    int64_t matvec_count;
    double wall_time; /* seconds, device-timed */
    double* final_rel_residual;
    char* converged;
} bk_solve_report;

/* PhaseTimings (dataset.hpp:17-25), device-timed with CUDA events. */
typedef struct {
    double assemble_s;
    double basis_solve_s;
    double combine_action_s; /* combine_s + operator_action_s (one fused kernel) */
    double h2d_s;
    double d2h_s;
    double total_s;
    int64_t iterations_total;
    int64_t matvecs_total;
} bk_phase_timings;

typedef struct bk_ctx bk_ctx;
typedef struct bk_operator bk_operator;

int bk_abi_version(void);

/* One context per (host thread, GPU): owns a stream, events and a grow-only
 * device workspace. */
bk_status bk_create(int device, bk_ctx** out);
void bk_destroy(bk_ctx* ctx);
const char* bk_last_error(const bk_ctx* ctx);
/* Run subsequent work on an external cudaStream_t (e.g. torch's current
 * stream); NULL is the legacy default stream. bk_use_own_stream restores the
 * context's own (non-blocking) stream. */
bk_status bk_set_stream(bk_ctx* ctx, void* cuda_stream);
bk_status bk_use_own_stream(bk_ctx* ctx);
bk_status bk_synchronize(bk_ctx* ctx);
/* Number of this library's kernel launches issued on ctx so far. */
int64_t bk_launch_count(const bk_ctx* ctx);

/* ---- discretization (discretize.hpp) ------------------------------------ */

/* assemble(k, grid, bc) -> DiscreteOperator        discretize.hpp:76,
 * discretize.cpp:114-237. Builds the matrix-free SoA stencil in HBM. */
bk_status bk_assemble(bk_ctx* ctx, const bk_grid* grid, const double* k,
                      const bk_face bc[6], bk_operator** out);
/* The same, into an existing operator: its device buffers are reused when the
 * cell count matches (no allocation in a per-chip loop). */
bk_status bk_assemble_into(bk_ctx* ctx, const bk_grid* grid, const double* k,
                           const bk_face bc[6], bk_operator* op);
void bk_operator_free(bk_operator* op);
int64_t bk_operator_n(const bk_operator* op);

/* The stencil as the reference's CSR (row_ptr n+1, col/val nnz <= 7n) plus g
 * and volumes — integer structure bit-exact with discretize.cpp:218-231.
 * Pass col/val/g/vol = NULL to query *nnz only. Host pointers. */
bk_status bk_operator_export_csr(bk_ctx* ctx, const bk_operator* op, int64_t* row_ptr,
                                 int32_t* col, double* val, int64_t* nnz, double* g,
                                 double* vol);

/* The device stencil from an operator the reference assembled: drop-in for
 * block_cg(const CsrMatrix&, ...) / DiscreteOperator{A, g, volumes}
 * (solvers.hpp:85, discretize.hpp:62-69). The CSR must be a symmetric 7-point
 * stencil on `grid` (columns i +- 1, +- nx, +- nx*ny with grid adjacency; the
 * reference omits zero off-diagonals) with volumes uniform per z-layer;
 * otherwise BK_INVALID_SPEC. D^-1 is jacobi_inverse (solvers.cpp:53-66).
 * Bitwise the same operator as bk_assemble on the same inputs. Host pointers;
 * g / vol may be NULL (zero lift / unit volumes). */
bk_status bk_operator_from_csr(bk_ctx* ctx, const bk_grid* grid, const int64_t* row_ptr,
                               const int32_t* col, const double* val, const double* g,
                               const double* vol, bk_operator** out);

/* Y = A X for n x s blocks        CsrMatrix::apply_block discretize.hpp:57,
 * discretize.cpp:75-95 (same per-row FMA accumulation order). */
bk_status bk_apply_block(bk_ctx* ctx, const bk_operator* op, const double* X, int s,
                         double* Y);

/* B = V Q + g per column          rhs_from_power discretize.hpp:82 */
bk_status bk_rhs_from_power(bk_ctx* ctx, const bk_operator* op, const double* Q, int s,
                            double* B);
/* Q = (B - g) / V per column      power_from_rhs discretize.hpp:87 */
bk_status bk_power_from_rhs(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                            double* Q);

/* ---- solvers (solvers.hpp) ------------------------------------------------ */

/* block_cg(op, B, cfg) -> {X, report}     solvers.hpp:85, solvers.cpp:452-665.
 * One persistent sm_100a kernel per solve: fused stencil-SpMM + Gram, fused
 * block updates, on-device pivoted-Cholesky s x s solves, per-column
 * verify/freeze/restart. Never fails on non-convergence (report.converged). */
bk_status bk_block_cg(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                      const bk_solver_cfg* cfg, double* X, bk_solve_report* report);

/* ---- pipeline (pipeline.hpp) ------------------------------------------------ */

/* For each sample j: T_j = sum_t C[t][j] X[:,t]  (combine_from_weights,
 * pipeline.cpp:187-225) and Q_j = (A T_j - g)/V (operator_action,
 * pipeline.cpp:242-251), resid[j] = ||A T_j - (V Q_j + g)|| / ||V Q_j + g||
 * (pipeline.cpp:548-571). One fused kernel; T/Q/resid may be NULL to skip. */
bk_status bk_combine_action(bk_ctx* ctx, const bk_operator* op, const double* X, int s,
                            const double* C, int64_t N, double* T, double* Q,
                            double* resid);

/* Whole per-chip pipeline (generate_blockoa, pipeline.cpp:365-597, for one
 * basis group): assemble -> B = V Qbasis + g -> block CG -> fused combine +
 * operator action. Qbasis row-major n x s power maps [W/m^3]; C row-major
 * s x N. Returns BK_NOT_CONVERGED (after filling outputs) if any basis column
 * missed the tolerance, as generate_basis does (pipeline.cpp:128-132). */
bk_status bk_generate_chip(bk_ctx* ctx, const bk_grid* grid, const double* k,
                           const bk_face bc[6], const double* Qbasis, int s,
                           const double* C, int64_t N, const bk_solver_cfg* cfg,
                           double* T, double* Q, double* resid, bk_solve_report* report,
                           bk_phase_timings* timings);

/* Batched per-chip pipeline for many independent chips (BASELINE config 4;
 * also configs 1-3 run as multi-chip jobs): the per-chip loop of
 * generate_blockoa (pipeline.cpp:365-597). streams = 1: chips one after another
 * (host output buffers drain chip c over PCIe while chip c+1 computes).
 * streams = K > 1 with chips of identical dims, s <= 32 and device outputs:
 * groups of K chips are z-stacked (block-diagonal system) and their basis
 * blocks solved by ONE cooperative launch, chip k on 1/K of the SMs, so the
 * latency-bound solves overlap; each chip's results are bitwise those of
 * bk_generate_chip with a 1/K SM budget (bk_set_cg_sm_budget). Other cases
 * fall back to streams = 1. Per-chip arrays of pointers (host or device);
 * T/Q/resid entries may be NULL. reports may be NULL (else n_chips entries
 * whose residual arrays hold s values each). */
bk_status bk_generate_batch(bk_ctx* ctx, int n_chips, const bk_grid* grids,
                            const double* const* k, const bk_face* bc /* n_chips x 6 */,
                            const double* const* Qbasis, int s, const double* const* C,
                            int64_t N, const bk_solver_cfg* cfg, double* const* T,
                            double* const* Q, double* const* resid, bk_solve_report* reports,
                            int streams, bk_phase_timings* timings);

/* Streaming per-chip pipeline for jobs whose outputs do not fit in memory at
 * once (BASELINE config 5: 335 GB of (T, q) per chip): the per-chip loop of
 * generate_blockoa (pipeline.cpp:365-597) with the samples handed to a host
 * sink chunk by chunk. Chips are solved one after another; each chip's samples
 * are combined + operator-actioned in chunks of `chunk` samples (0 = ~2 GB of
 * T + q per chunk) into a device ring, copied over PCIe into a pinned host
 * ring, and passed to sink(user, chip, j0, m, n, T, Q, resid) — T, Q are m x n
 * sample-major, resid m values, valid only during the call — from a library
 * worker thread while the next chip's basis solve runs. sink may be NULL (the
 * samples are still copied to host memory). A non-zero return from sink
 * aborts with BK_IO_ERROR. Inputs are host or device pointers (per-chip
 * arrays as in bk_generate_batch). reports: n_chips entries or NULL. */
typedef int (*bk_sample_sink)(void* user, int chip, int64_t j0, int64_t m, int64_t n,
                              const double* T, const double* Q, const double* resid);
bk_status bk_generate_stream(bk_ctx* ctx, int n_chips, const bk_grid* grids,
                             const double* const* k, const bk_face* bc /* n_chips x 6 */,
                             const double* const* Qbasis, int s, const double* const* C,
                             int64_t N, const bk_solver_cfg* cfg, int64_t chunk,
                             bk_sample_sink sink, void* user, bk_solve_report* reports,
                             bk_phase_timings* timings);

/* Cap the number of CTAs (and thus SMs) one block-CG solve may use on ctx
 * (0 = all SMs). */
bk_status bk_set_cg_sm_budget(bk_ctx* ctx, int max_ctas);

/* Per-context debug / A-B switches, initialised from the environment when the
 * context is created (BK_CG_RING, BK_CG_NO_RESIDENT, BK_CG_LARGE,
 * BK_CG_PROFILE, BK_NO_TMA_SPMM, BK_COMB_PROFILE, BK_BATCH_TRACE). Names:
 * "ring" (-1 automatic, 0 off, 1 on), "no_resident", "force_large",
 * "cg_profile", "no_tma_spmm", "comb_profile", "batch_trace" (0 / 1);
 * "no_defer_x" = 1 keeps X += P alpha in phase 2 of the persistent block CG
 * (bitwise the deferred form; tests compare the two); "no_w_prefetch" = 1
 * single-buffers phase 2's W staging in the row-ring kernels (A/B).
 * Not part of the reference API; used by the tests to pin kernel variants. */
bk_status bk_set_option(bk_ctx* ctx, const char* name, int value);
/* Kernel instantiation the last block-CG solve on ctx ran, e.g.
 * "block_cg_dmma_kernel<16,0,1,1> ring chips=16" (template arguments S,
 * resident, multi-chip, deferred X update) or "block_cg_large<64> tma". */
const char* bk_last_solver_variant(const bk_ctx* ctx);
/* With option "phase_timing" = 1: device time (ms, CUDA events) and launch
 * count per sweep kind of the last multi-kernel block-CG solve on ctx, 4
 * entries: [0] stencil-SpMM + Gram (W = A P, P^T W), [1] R update + S_new,
 * [2] P update (+ the deferred X update), [3] reserved. */
bk_status bk_last_solve_phases(const bk_ctx* ctx, double* ms, int64_t* counts);
/* Measurement aid (no reference counterpart): the FP64 tensor-core rate of
 * this GPU, TFLOP/s of register-operand mma.sync.m16n8k4.f64 chains on every
 * SM (32 warps per SM, 4 independent accumulator chains per warp).
 * burst = best of 10 launches of ~2 ms each; sustained = launches back to back
 * for `seconds` (the rate the FP64 pipe holds at the board's power limit —
 * the roofline denominator for a kernel timed inside a long FP64 step). */
bk_status bk_measure_fp64_peak(bk_ctx* ctx, double seconds, double* burst_tflops,
                               double* sustained_tflops);

/* ---- y-slab domain decomposition (BASELINE config 5 across GPUs) -----------
 * A rank owns global rows [y0, y0 + nyl) of the grid of `op` (the GLOBAL
 * operator, assembled identically on every rank). Its block vectors use the
 * slab-local layout nx x (nyl + 2) x nz x S with one ghost row on each y side.
 * The caller drives the phases below in lockstep across ranks, summing `red`
 * across ranks after every *_SWEEP step and refreshing the ghost rows of P
 * (before BK_DD_SPMM) and of X (before BK_DD_TRUE_RES / BK_DD_RESTART); see
 * paper_2510_23221_b200/dd.py. All buffers are caller-owned device memory. */
typedef struct {
    double* B;     /* local RHS block */
    double* X;
    double* R;
    double* P;
    double* W;
    double* part;  /* per-CTA partials, nb x (S*S + S) */
    double* red;   /* reduced values, S*S + S (all-reduced by the caller) */
    void* ctl;     /* control state, ctl_bytes */
    int nb;        /* CTAs of the sweep kernels */
} bk_dd_bufs;

typedef enum {
    BK_DD_INIT_SWEEP = 0,    /* X = 0, R = B, P = D^-1 R; red = [R^T Z | b^2]   */
    BK_DD_CTL_INIT = 1,
    BK_DD_SPMM = 2,          /* W = A P; red = P^T W                            */
    BK_DD_CTL_ALPHA = 3,     /* alpha = G^+ S_old                               */
    BK_DD_UPDATE = 4,        /* X += P alpha, R -= W alpha; red = [R^T Z | rr]  */
    BK_DD_CTL_UPDATE = 5,    /* convergence test; beta or verification needed   */
    BK_DD_TRUE_RES = 6,      /* red = ||b - A x||^2 of flagged/active columns   */
    BK_DD_CTL_VERIFY = 7,
    BK_DD_RESTART_SWEEP = 8, /* R = B - A X, P = Z; red = R^T Z                 */
    BK_DD_CTL_RESTART = 9,
    BK_DD_PUPDATE = 10,      /* P = D^-1 R + P beta                             */
    BK_DD_CTL_FINAL = 11,    /* report                                          */
    BK_DD_READ = 12,         /* *cmd, *sa (synchronises the stream)             */
    /* deferred-X flow (the single-GPU engine's, used when bk_dd_deferred_x()
     * is 1 — S = 64 on 16-aligned x — with the warp-specialised sweeps):
     * BK_DD_UPDATE_D replaces BK_DD_UPDATE and leaves X alone; X += P alpha
     * then happens in BK_DD_PUPDATE_X (with the P update) or, before a
     * verification, in BK_DD_APPLY_X (followed by BK_DD_PUPDATE).          */
    BK_DD_UPDATE_D = 13,     /* R -= W alpha; red = [R^T Z | rr]                */
    BK_DD_PUPDATE_X = 14,    /* P = D^-1 R + P beta, X += P_old alpha           */
    BK_DD_APPLY_X = 15,      /* X += P alpha                                    */
    /* *cmd, *sa <- the control word, enqueued without synchronising: cmd and
     * sa must point to pinned host memory that stays valid until the stream
     * passes the copies (the caller waits on an event recorded after it)    */
    BK_DD_READ_ASYNC = 16,
    /* flag OR-ed into SPMM / CTL_ALPHA / UPDATE(_D) / CTL_UPDATE / PUPDATE(_X):
     * the kernels run only while the control word is BK_DD_CMD_PUPDATE, so a
     * host can enqueue iteration m + 1 before reading iteration m's word (a
     * pending verification turns the enqueued iteration into no-ops)       */
    BK_DD_GATED = 0x100
} bk_dd_step_kind;

/* 1 if the slab steps of (op, S) use the deferred-X flow above. */
int bk_dd_deferred_x(const bk_operator* op, int S);

/* BK_DD_READ commands */
#define BK_DD_CMD_PUPDATE 0
#define BK_DD_CMD_VERIFY 1
#define BK_DD_CMD_RESTART 2
#define BK_DD_CMD_DONE 3

bk_status bk_dd_sizes(bk_ctx* ctx, const bk_operator* op, int nyl, int S, int64_t* local_elems,
                      int* nb, int64_t* part_elems, int64_t* red_elems, int64_t* ctl_bytes);
bk_status bk_dd_step(bk_ctx* ctx, const bk_operator* op, int y0, int nyl, int S,
                     const bk_dd_bufs* bufs, const bk_solver_cfg* cfg, int step, int m,
                     int* cmd, int* sa, bk_solve_report* report);
/* global n x S block <-> slab-local block (to_local = 1: glob -> loc, ghost
 * rows untouched; 0: loc -> glob interior rows) */
bk_status bk_dd_pack(bk_ctx* ctx, const bk_operator* op, int y0, int nyl, int S, double* glob,
                     double* loc, int to_local);

/* Slab-local combination + operator action after the decomposed solve: each
 * rank forms T_j = X C_j and q_j = (A T_j - g)/V for ALL samples j on its own
 * rows [y0, y0 + nyl) (pipeline.cpp:187-251), from its slab of X in the
 * ghost-row layout with the ghost rows refreshed once (the neighbours' edge
 * rows: one X-halo exchange instead of gathering X). Tloc / Qloc: N x
 * (nx nyl nz) sample-major, slab-local flat index ix + nx (iyl + nyl iz).
 * nd (N x 2, may be NULL): this rank's per-sample (num, den) partials of the
 * residual of pipeline.cpp:548-571; sum them across ranks and call
 * bk_dd_resid_from_nd. Device pointers; 3D grids (nz > 1). */
bk_status bk_dd_combine_action(bk_ctx* ctx, const bk_operator* op, int y0, int nyl, int S,
                               const double* Xloc, int s, const double* C, int64_t N,
                               double* Tloc, double* Qloc, double* nd);
bk_status bk_dd_resid_from_nd(bk_ctx* ctx, const double* nd, int64_t N, double* resid);

/* cg_error_bound(kappa, m, e0)    solvers.hpp:92, solvers.cpp:672-680 (host). */
bk_status bk_cg_error_bound(double kappa, int m, double e0, double* out);

/* ---- seeded synthetic inputs (host; BASELINE configs) ------ */

/* derive_seed / Rng (rng.hpp:14-63) restated bit-exactly on the host. */
uint64_t bk_derive_seed(uint64_t seed, const char* tag, uint64_t index);
void bk_rng_u64(uint64_t seed, int64_t n, uint64_t* out);
void bk_rng_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out);
void bk_rng_normal(uint64_t seed, int64_t n, double* out);

/* Input synthesis for BASELINE config `cfg` in 1..5 (reduced shapes allowed
 * through the size arguments). Fills k (n), Qbasis (n x s), C (s x N), the
 * boundary faces and, for layered stacks, dz (nz, or left untouched when the
 * config has uniform dz; *has_dz tells which). chip_id selects the chip's
 * seed stream derive_seed(master_seed, "chip", chip_id). */
typedef struct {
    int config; /* 1..5 */
    int nx, ny, nz;
    int s;
    int64_t N;
    uint64_t master_seed;
    uint64_t chip_id;
} bk_synth_spec;

bk_status bk_synth_chip(const bk_synth_spec* spec, bk_grid* grid_out, double* dz_out,
                        int* has_dz, bk_face bc_out[6], double* k, double* Qbasis,
                        double* C);

/* The same chip with its fields evaluated on the device: the
 * random draws stay on the host (identical Rng streams), k (n) and the basis
 * maps Qbasis (n x s, row-major) are written to DEVICE buffers by kernels on
 * the context's stream; C (s x N) may be host or device. k for configs 1, 2, 4
 * and C are bitwise bk_synth_chip's; the maps and the lognormal k of configs
 * 3, 5 differ only through CUDA's exp vs the host libm (a few ulp). */
bk_status bk_synth_chip_device(bk_ctx* ctx, const bk_synth_spec* spec, bk_grid* grid_out,
                               double* dz_out, int* has_dz, bk_face bc_out[6], double* k_dev,
                               double* Qbasis_dev, double* C);

/* ---- reference-semantics generation (chip model + generate_blockoa) -------- */

/* ChipSpec (chip.hpp:55-80) with material names resolved to conductivities.
 * Lengths in meters; layers bottom to top tiling [0, extent[2]); power ranges
 * in W/mm^2 (closed intervals). role: BK_LAYER_CORE / CACHE / TIM. */
typedef enum { BK_LAYER_CORE = 0, BK_LAYER_CACHE = 1, BK_LAYER_TIM = 2 } bk_layer_role;
#define BK_MAX_LAYERS 16
typedef struct {
    double z_lo, z_hi;
    double k; /* conductivity of the layer material, W/(m K) */
    int role; /* bk_layer_role */
} bk_layer;
typedef struct {
    double extent[3];
    int n_layers;
    bk_layer layers[BK_MAX_LAYERS];
    int core_blocks, high_power, caches_per_layer; /* BlockCounts */
    double p_high[2], p_normal[2], p_cache[2];      /* PowerRanges, W/mm^2 */
    int tsv_count;                                  /* 0: no TSVs */
    double tsv_width;                               /* m */
    double tsv_k;                                   /* TSV material conductivity */
} bk_chip_spec;

/* ChipSpec::default_chip()   chip.cpp:74-100 (10 x 10 x 0.51 mm, TIM / cache /
 * TIM / cache / TIM / core, 156 core blocks, 6 high power, 2 caches per layer,
 * 12 copper TSVs). */
void bk_default_chip(bk_chip_spec* out);

/* Host chip model, bit-exact with the reference: build_floorplans(spec, n_k,
 * seed) (chip.cpp:180-221), rasterize_conductivity (chip.cpp:238-274) -> k
 * [n_k][n]; for each group j and basis column t, sample_power(fp_j, spec,
 * derive_seed(seed, "basis", j eta + t)) and rasterize_power (chip.cpp:223-306)
 * -> q [n_k eta][n] (generate_basis, pipeline.cpp:92-134). The grid spans the
 * chip extent. q may be NULL. */
bk_status bk_chip_fields(const bk_chip_spec* spec, int nx, int ny, int nz, int n_k, int eta,
                         uint64_t seed, double* k, double* q);

/* draw_weights(n_basis, sample_seed_for(seed, l + 1)) for l < n_data
 * (pipeline.cpp:88-90, 136-152): normalised Gaussian weights -> w
 * [n_data][n_basis]. Host. */
bk_status bk_draw_weights(int n_basis, uint64_t seed, int64_t n_data, double* w);

typedef enum { BK_NOISE_NONE = 0, BK_NOISE_UNIFORM = 1, BK_NOISE_GAUSSIAN = 2 } bk_noise_kind;

/* GenerationConfig (pipeline.hpp:28-43). The grid spans the chip extent. */
typedef struct {
    int nx, ny, nz;
    bk_face bc[6];
    int64_t n_data;
    int n_basis; /* total basis columns; n_k must divide it (eta = n_basis / n_k) */
    int n_k;     /* floorplan groups */
    uint64_t master_seed;
    int noise_kind; /* bk_noise_kind */
    double noise_lo, noise_hi, noise_sigma;
    bk_solver_cfg solver;
    bk_chip_spec chip;
} bk_blockoa_cfg;

/* generate_blockoa(cfg)   pipeline.hpp:106, pipeline.cpp:365-597, on the GPU:
 * the n_k floorplan groups' operators and eta power maps each (host chip model
 * above), ONE batched block-CG launch for all groups, then per group the fused
 * combine + action kernel over ALL groups' basis columns (groups ascending,
 * columns ascending, normalised Gaussian weights drawn on the host), the
 * interior noise stream of every sample generated on the device (uniform;
 * gaussian noise is drawn on the host), q = (A_g T - g)/V with the group's
 * operator in apply_block's fused-multiply-add order, sample l in group
 * l mod n_k. n_basis <= 64, eta <= 32. Outputs (host or device, NULL to
 * skip): k [n_k][n], U and Q [n_data][n], resid [n_data], floorplan_id
 * [n_data]; reports: n_k entries. BK_NOT_CONVERGED if a basis group missed
 * the tolerance (NotConvergedError, pipeline.cpp:128-132). */
bk_status bk_generate_blockoa(bk_ctx* ctx, const bk_blockoa_cfg* cfg, double* k, double* U,
                              double* Q, double* resid, int64_t* floorplan_id,
                              bk_solve_report* reports, bk_phase_timings* timings);

/* ---- dataset sink and validation (dataset_io.hpp) ---------------------------- */

/* field_digest(f)   discretize.hpp:99, discretize.cpp:302-319: FNV-1a over
 * (nx, ny, nz) then the raw little-endian value bytes. Host pointer. */
uint64_t bk_field_digest(int nx, int ny, int nz, const double* values);

/* write_dataset(ds, dir, {overwrite})   dataset_io.hpp:27, dataset_io.cpp:160-225,
 * as a streaming writer. open stages `<dir>.tmp-<pid>` next to dir (BK_EXISTS if
 * dir already holds a manifest and !overwrite); each append adds n_samples
 * samples: k (n, the chip's field, repeated once per sample), Q and U (n_samples
 * x n, sample-major) to k.bin / q.bin / u.bin. Pointers may be host or device
 * (device ones need ctx; they are drained through pinned buffers, PCIe copy
 * overlapped with the file write). commit writes manifest.json (the caller's
 * JSON text, same keys as dataset_io.cpp:120-142) and renames the staged
 * directory into place. bk_dataset_close frees the writer and discards
 * anything not committed. The writer is returned by open even on failure so
 * bk_dataset_error can be read. */
typedef struct bk_dataset_writer bk_dataset_writer;
bk_status bk_dataset_open(const char* dir, int overwrite, int64_t n_cells,
                          bk_dataset_writer** out);
bk_status bk_dataset_append(bk_dataset_writer* w, bk_ctx* ctx, const double* k,
                            int64_t n_samples, const double* Q, const double* U);
bk_status bk_dataset_commit(bk_dataset_writer* w, const char* manifest_json);
void bk_dataset_close(bk_dataset_writer* w);
const char* bk_dataset_error(const bk_dataset_writer* w);
int64_t bk_dataset_count(const bk_dataset_writer* w);
double bk_dataset_write_seconds(const bk_dataset_writer* w);

/* relative_residual(op, u, q)   discretize.hpp:91, discretize.cpp:275-286, for
 * N samples: resid[j] = ||V Q_j + g - A U_j|| / ||V Q_j + g|| (0 or +inf when
 * the denominator is 0). U, Q: N x n sample-major, host (e.g. a memory-mapped
 * file; streamed through pinned buffers) or device; resid host or device. */
bk_status bk_residuals(bk_ctx* ctx, const bk_operator* op, const double* U, const double* Q,
                       int64_t N, double* resid);

/* ValidationReport (dataset_io.hpp:36-41) */
typedef struct {
    int64_t pass_count;
    int64_t fail_count;
    double max_residual;
} bk_validation;

/* The sample loop of validate_dataset(dir, tol)   dataset_io.cpp:328-361, over
 * a dataset already read (read_dataset is host I/O): K, U, Q are n_data x n
 * (K host; U, Q host or device), ids the per-sample floorplan ids, (decl_ids,
 * decl_digests) the manifest's floorplan_digests. A sample whose k digest
 * contradicts its declared digest gets residual +inf and fails; the others are
 * checked against one operator per distinct k, assembled on the GPU from grid
 * and bc. residuals: n_data host values. */
bk_status bk_validate_samples(bk_ctx* ctx, const bk_grid* grid, const bk_face bc[6],
                              const double* K, const double* U, const double* Q, int64_t n_data,
                              const uint64_t* ids, int n_decl, const uint64_t* decl_ids,
                              const uint64_t* decl_digests, double tol, double* residuals,
                              bk_validation* report);

#ifdef __cplusplus
}
#endif

#endif /* BLOCKOA_B200_H */
