// Block conjugate gradient — DMMA variant (kernel widths S = 8, 16, 32).
//
// The reference algorithm is block_cg (solvers.cpp:452-665), restructured
// around FP64 tensor cores: every dense s x s product runs on mma.sync.m16n8k4.f64 (one
// DMMA issue per ~33 cycles per warp; B200's FP64 pipe, shared with SIMT DFMA,
// peaks at 37 TFLOP/s — profiles/r2_summary.md), with operand fragments
// produced in registers by the sweep that loads them — no shared-memory
// staging except a warp-private transpose for R^T Z.
//
//   phase 1  W = A P (CSR-order FMA chain, bitwise the reference apply_block)
//            and the Gram G = P^T W by DMMA with K = cells, per warp in 16-cell
//            tiles; for single-plane chips outside resident mode the P rows and
//            coefficient rows stream through a 4-slot shared-memory ring filled
//            by TMA bulk copies two rows ahead (phase_spmm_gram_ring).
//   phase 2  R -= W alpha as a DMMA GEMM (M = cells, N = columns, K = s), rr
//            and Z = D^-1 R in the epilogue, S_new = R^T Z by DMMA after a
//            warp-private smem transpose; X += P alpha here too, or (DEF) in
//            phase 3, which reads the same P tile (one P read fewer).
//   phase 3  P = Z + P beta, DMMA with the accumulator initialised to Z.
//
// Grid-wide: one chip on all SMs (cooperative launch, cg::grid.sync, 1.2 us
// measured) or K z-stacked chips with per-chip CTA groups and one-word
// flip-bit group barriers; fixed-order distributed reductions (no
// floating-point atomics: bitwise deterministic); redundant per-CTA s x s
// solves (Gauss-Jordan with the reference's pivoted-Cholesky rank semantics).
#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "bk_common.cuh"
#include "bk_small_solve.cuh"

namespace cg = cooperative_groups;

namespace {

using namespace bkcg;

// CTA size per kernel width: 16 warps for S <= 16 (one CTA per SM), 8 warps
// for S = 32 (one CTA per SM, up to 255 registers per thread).
template <int S>
struct CtaShape {
    static constexpr int BS = S <= 16 ? 512 : 256;
    static constexpr int NW = BS / 32;
};
constexpr int PROF_ITERS = 64;
constexpr int PROF_MARKS = 12;

struct Args {
    int nx, ny, nz;
    int64_t n;
    const double* diag;
    const double* cx;
    const double* cy;
    const double* cz;
    const double* dinv;
    const double* B;
    double* X;
    double* R;
    double* P;
    double* W;
    double* part;
    double* red;
    double tol;
    int max_iter;
    int precond;
    bk::CgReport* rep;
    long long* prof;  // optional phase timestamps (CTA 0), PROF_ITERS x PROF_MARKS
    int ring;         // phase 1 through the row ring (phase_spmm_gram_ring)
    int pre_off;      // byte offset (from the dynamic smem base) of phase 2's W prefetch
                      // buffers, NW x 2 tiles; -1: none (single-buffered staging)
    // several independent chips of identical dims in one launch: chip k owns
    // cells [k nchip, (k+1) nchip) of the z-stacked (block-diagonal) system,
    // CTAs [k cpc, (k+1) cpc), reduction partials part + k cpc (S^2+S),
    // results red + k (S^2+S), report rep + k and barrier bars + 2k
    int nchips;
    int cpc;
    int64_t nchip;
    unsigned* bars;
};

__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Resident mode (S <= 16, at most kResCells cells per CTA: BASELINE configs 1,
// 2 and 4 on 148 SMs): X and R live in shared memory for the whole solve
// (XOR-swizzled rows, conflict-free for the DMMA C-fragment layout), removing
// their L2 round trips from phases 2 and 3; they are published to HBM only for
// the rare true-residual / restart sweeps and at exit.
constexpr int kResCells = 448;

template <int S, bool RES>
struct ResStore {
    static constexpr int kVecs = 0;
};
template <int S>
struct ResStore<S, true> {
    alignas(16) double x[kResCells * S];
    alignas(16) double r[kResCells * S];
    double dinv[kResCells];  // D^-1 of the CTA's cells (1.0 without Jacobi)
};

template <int S>
constexpr bool scratch_aliases_tiles() {
    return S * S <= 16 * Strides<S>::RS;
}

template <int S, bool RES = false>
struct Sm {
    double s_old[S * S];
    double mat[S * S];
    alignas(16) double coef[S * Strides<S>::RS];
    alignas(16) double akeep[S * Strides<S>::RS];  // alpha, for the deferred X update
    alignas(16) double aug[S * Strides<S>::LD + 2 * S];
    // per-warp matrix partials; aliased onto the warp's own transpose tile
    // when it fits (written only after that warp's tile loop)
    double scratch[scratch_aliases_tiles<S>() ? 1 : CtaShape<S>::NW * S * S];
    alignas(16) double tileR[CtaShape<S>::NW][16 * Strides<S>::RS];  // warp-private transposes
    alignas(16) double tileZ[CtaShape<S>::NW][16 * Strides<S>::RS];
    alignas(16) ResStore<S, RES> res;
    double vec[S];
    double bnorm[S];
    double fres[S];
    double dpiv[S];
    int perm[S];
    int act[S];
    int idx[S];
    int vflag[S];
    int conv[S];
    int sa;
    int fail;
    int rank;
};

// ---------------------------------------------------------------------------
// stencil at (cell, col) of a row-major n x S block
// ---------------------------------------------------------------------------
struct Coef {
    double d, xm, xp, ym, yp, zm, zp;  // CSR values (-conductance off the diagonal)
    int64_t oxm, oxp, oym, oyp, ozm, ozp;  // neighbour cell offsets (0 if absent)
    bool hxm, hxp, hym, hyp, hzm, hzp;
};

// zlo / zhi: the z range of the cell's chip. A z-stacked batch couples its
// chips through zero face conductances only; skipping those z terms (as the
// single chip has no z neighbour there) leaves every sum bitwise unchanged and
// saves two P-row loads per cell of a stacked 2D chip.
__device__ __forceinline__ void load_coef_at(const Args& a, int64_t c, int ix, int iy, int iz,
                                             int zlo, int zhi, Coef& k) {
    const int64_t plane = (int64_t)a.nx * a.ny;
    k.hzm = iz > zlo;
    k.hym = iy > 0;
    k.hxm = ix > 0;
    k.hxp = ix < a.nx - 1;
    k.hyp = iy < a.ny - 1;
    k.hzp = iz < zhi;
    k.d = a.diag[c];
    k.zm = k.hzm ? -a.cz[c - plane] : 0.0;
    k.ym = k.hym ? -a.cy[c - a.nx] : 0.0;
    k.xm = k.hxm ? -a.cx[c - 1] : 0.0;
    k.xp = k.hxp ? -a.cx[c] : 0.0;
    k.yp = k.hyp ? -a.cy[c] : 0.0;
    k.zp = k.hzp ? -a.cz[c] : 0.0;
    k.ozm = plane;
    k.oym = a.nx;
}

__device__ __forceinline__ void load_coef(const Args& a, int64_t c, int zlo, int zhi, Coef& k) {
    const int ci = (int)c;
    load_coef_at(a, c, ci % a.nx, (ci / a.nx) % a.ny, ci / (a.nx * a.ny), zlo, zhi, k);
}

// grid coordinates of cell c, then stepped by `d` cells (no division per step)
struct CellXYZ {
    int ix, iy, iz;
    __device__ __forceinline__ void set(const Args& a, int64_t c) {
        const int ci = (int)c;
        ix = ci % a.nx;
        iy = (ci / a.nx) % a.ny;
        iz = ci / (a.nx * a.ny);
    }
    __device__ __forceinline__ void step(const Args& a, int d) {
        ix += d;
        while (ix >= a.nx) {
            ix -= a.nx;
            if (++iy == a.ny) {
                iy = 0;
                ++iz;
            }
        }
    }
};

// CSR-order FMA chain (apply_block_fixed, discretize.cpp:57-71)
template <int S>
__device__ __forceinline__ double st_fma(const Coef& k, const double* __restrict__ V, int64_t c,
                                         int col, double& center) {
    const int64_t e = c * S + col;
    double acc = 0.0;
    if (k.hzm) acc = fma(k.zm, V[e - k.ozm * S], acc);
    if (k.hym) acc = fma(k.ym, V[e - k.oym * S], acc);
    if (k.hxm) acc = fma(k.xm, V[e - S], acc);
    center = V[e];
    acc = fma(k.d, center, acc);
    if (k.hxp) acc = fma(k.xp, V[e + S], acc);
    if (k.hyp) acc = fma(k.yp, V[e + k.oym * S], acc);
    if (k.hzp) acc = fma(k.zp, V[e + k.ozm * S], acc);
    return acc;
}

// separate multiply + add (CsrMatrix::apply, used by true_rel_residual)
template <int S>
__device__ __forceinline__ double st_muladd(const Coef& k, const double* __restrict__ V,
                                            int64_t c, int col) {
    const int64_t e = c * S + col;
    double acc = 0.0;
    if (k.hzm) acc = __dadd_rn(acc, __dmul_rn(k.zm, V[e - k.ozm * S]));
    if (k.hym) acc = __dadd_rn(acc, __dmul_rn(k.ym, V[e - k.oym * S]));
    if (k.hxm) acc = __dadd_rn(acc, __dmul_rn(k.xm, V[e - S]));
    acc = __dadd_rn(acc, __dmul_rn(k.d, V[e]));
    if (k.hxp) acc = __dadd_rn(acc, __dmul_rn(k.xp, V[e + S]));
    if (k.hyp) acc = __dadd_rn(acc, __dmul_rn(k.yp, V[e + k.oym * S]));
    if (k.hzp) acc = __dadd_rn(acc, __dmul_rn(k.zp, V[e + k.ozm * S]));
    return acc;
}

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
// Only the upper triangle of a Gram matrix is ever read (the s x s solves read
// M[min(a,b)][max(a,b)]; the reference also computes the upper part and
// mirrors it, solvers.cpp:336-341), so 16x8 output tiles entirely below the
// diagonal are skipped (their accumulators stay zero).
__host__ __device__ constexpr bool gram_tile_needed(int m, int n) { return 8 * n + 7 >= 16 * m; }

// Gram accumulator in DMMA D-fragment layout: tile (mt, nt) holds
// G[16mt+g][8nt+2t+{0,1}] and G[16mt+g+8][8nt+2t+{0,1}].
template <int S>
struct GramAcc {
    static constexpr int MT = (S + 15) / 16;
    static constexpr int NT = S / 8;
    double d[MT][NT][4];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e) d[m][n][e] = 0.0;
    }
    // write this warp's partial into scratch[warp][S*S] (row-major)
    __device__ __forceinline__ void spill(double* dst, int g, int t) const {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const int r0 = 16 * m + g, c0 = 8 * n + 2 * t;
                dst[r0 * S + c0] = d[m][n][0];
                dst[r0 * S + c0 + 1] = d[m][n][1];
                if (r0 + 8 < S) {
                    dst[(r0 + 8) * S + c0] = d[m][n][2];
                    dst[(r0 + 8) * S + c0 + 1] = d[m][n][3];
                }
            }
    }
};

// sum per-warp matrices in warp order -> out[S*S]
template <int S>
__device__ __forceinline__ void cta_sum_mat(const double* scratch, int stride, double* out) {
    constexpr int BS = CtaShape<S>::BS, NW = CtaShape<S>::NW;
    __syncthreads();
    for (int e = threadIdx.x; e < S * S; e += BS) {
        double s = scratch[e];
#pragma unroll
        for (int w = 1; w < NW; ++w) s += scratch[w * stride + e];
        out[e] = s;
    }
    __syncthreads();
}

// per-lane column partials v[nt][e] for columns 8nt+2t+e -> out[S] (warp order)
template <int S>
__device__ __forceinline__ void cta_sum_vec(double (&v)[S / 8][2], double* scratch, int stride,
                                            double* out, int warp, int lane) {
    constexpr int BS = CtaShape<S>::BS, NW = CtaShape<S>::NW;
#pragma unroll
    for (int n = 0; n < S / 8; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double x = v[n][e];
            x += __shfl_xor_sync(0xffffffffu, x, 4);
            x += __shfl_xor_sync(0xffffffffu, x, 8);
            x += __shfl_xor_sync(0xffffffffu, x, 16);
            if (lane < 4) scratch[warp * stride + 8 * n + 2 * lane + e] = x;
        }
    __syncthreads();
    for (int e = threadIdx.x; e < S; e += BS) {
        double s = scratch[e];
        for (int w = 1; w < NW; ++w) s += scratch[w * stride + e];
        out[e] = s;
    }
    __syncthreads();
}

// Barrier over the NB CTAs of one chip's group, the grid.sync protocol on one
// word per chip: the group's CTA 0 adds 0x80000000 - (NB - 1), every other
// CTA adds 1, so the word's top bit flips exactly when the last CTA arrives;
// each master thread then spins until it sees the flip. One fence and one
// atomic per CTA (the previous count + generation pair cost the last arrival
// a second fence and atomic on the critical path). All CTAs of the launch are
// co-resident (one cooperative launch).
__device__ __forceinline__ void group_barrier(unsigned* bar, unsigned NB, bool first) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned inc = first ? 0x80000000u - (NB - 1) : 1u;
        __threadfence();
        const unsigned old = atomicAdd(bar, inc);
        volatile unsigned* vb = bar;
        while (((old ^ *vb) & 0x80000000u) == 0u) {
        }
        __threadfence();
    }
    __syncthreads();
}

template <bool MULTI>
struct Group {
    int chip, b, NB;
    unsigned* bar;
    bool ring;  // phase 1 reads P through the async proxy (TMA row ring)
    __device__ __forceinline__ void sync(cg::grid_group& grid) const {
        // P (and every other block vector) is written with generic stores and,
        // in ring mode, read back by cp.async.bulk (async proxy) after this
        // barrier, possibly by another CTA: order the writer's generic global
        // stores before the async-proxy reads (PTX memory model, proxy fence
        // on the writing side; the issuing thread fences again before issue)
        if (ring) asm volatile("fence.proxy.async.global;" ::: "memory");
        if constexpr (MULTI)
            group_barrier(bar, (unsigned)NB, b == 0);
        else
            grid.sync();
    }
};

template <int BS, bool MULTI>
__device__ void grid_reduce(const Group<MULTI>& gr, cg::grid_group& grid, double* __restrict__ part,
                            double* __restrict__ redg, const double* src, int E, double* dst) {
    constexpr int NW = BS / 32;
    const int b = gr.b, NB = gr.NB;
    for (int e = threadIdx.x; e < E; e += BS) part[(int64_t)b * E + e] = src[e];
    gr.sync(grid);
    const int e0 = (int)((int64_t)E * b / NB), e1 = (int)((int64_t)E * (b + 1) / NB);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = e0 + warp; e < e1; e += NW) {
        double s = 0.0;
        for (int l = lane; l < NB; l += 32) s += __ldcg(part + (int64_t)l * E + e);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) __stcg(redg + e, s);
    }
    gr.sync(grid);
    for (int e = threadIdx.x; e < E; e += BS) dst[e] = __ldcg(redg + e);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// small solves (identical in every CTA)
// ---------------------------------------------------------------------------
template <int S, bool RES>
__device__ void build_index(Sm<S, RES>& sm) {
    if (threadIdx.x == 0) {
        int k = 0;
        for (int q = 0; q < S; ++q)
            if (sm.act[q]) sm.idx[k++] = q;
        sm.sa = k;
    }
    __syncthreads();
}

// out = M^+ RHS on the active block (zero rows/columns elsewhere), the
// semantics of PivotedCholesky(M).solve(RHS) (solvers.cpp:347-414): diagonal
// pivoting on the largest remaining Schur-complement diagonal, rank cutoff
// max(max_diag * s * eps, DBL_MIN), directions beyond the numerical rank get
// zero coefficients. Computed as Gauss-Jordan on [M | RHS] with that pivot
// sequence (the trailing block of Gauss-Jordan IS the Cholesky Schur
// complement, so pivots and rank decisions coincide): one barrier per pivot,
// the pivot search done redundantly by every warp (no broadcast barrier).
// Pivot loop on 4 warps for S <= 16 (named barrier; measured 10.1k -> 7.0k
// cycles at S = 16, 6.4k -> 3.7k at S = 8), on all 8 warps for S = 32.
template <int S>
constexpr int solve_warps() {
    return S <= 16 ? 4 : CtaShape<S>::NW;
}
template <int S, bool PROF = false, int VAR = 0, bool RES = false>
__device__ __forceinline__ void small_solve(Sm<S, RES>& sm, const double* M, const double* RHS,
                                            double* out) {
    small_solve_t<S, CtaShape<S>::BS, PROF, VAR, solve_warps<S>()>(sm, M, RHS, out);
}

// ---------------------------------------------------------------------------
// phases
// ---------------------------------------------------------------------------
// phase 1: W = A P over the CTA's cells, Gram G += P^T W, in 16-cell tiles.
// Lane (q = lane / (S/2), j = lane % (S/2)) owns columns 2j, 2j+1 of cells
// base + q + (32 / (S/2)) u: every load instruction reads whole 128-byte rows
// (4 L1 tag lookups per LDG.128 at S = 16 instead of 16 with a lane per half
// row). Each element's accumulation follows the reference CSR order
// (apply_block_fixed, discretize.cpp:57-71); W leaves with 128-bit stores, and
// P / W are staged in the warp's smem tiles for the DMMA Gram (K = cells).
template <int S>
__device__ __forceinline__ void phase_spmm_gram(const Args& a, int64_t c0, int64_t c1, int zlo,
                                                int zhi, int warp, int lane, double* tp,
                                                double* tw, GramAcc<S>& G) {
    constexpr int NW = CtaShape<S>::NW;
    constexpr int RS = Strides<S>::RS;
    // columns per lane: 2 (one 16-byte pair) up to S = 16; 4 for S = 32, which
    // halves the cells per lane per tile (U = 4 instead of 8) and with them the
    // dependent load / FMA rounds of the per-tile sweep
    constexpr int CPL = S >= 32 ? 4 : 2;
    constexpr int H = CPL / 2;     // 16-byte column pairs per lane
    constexpr int LPR = S / CPL;   // lanes per row
    constexpr int CPI = 32 / LPR;  // cells per load instruction
    constexpr int U = 16 / CPI;    // cells per lane per tile
    const int q = lane / LPR, col = CPL * (lane % LPR);
    const int g = lane >> 2, t = lane & 3;
    const int64_t plane = (int64_t)a.nx * a.ny;
    for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW) {
        CellXYZ xyz;
        xyz.set(a, base + q);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int lr = q + CPI * u;  // row of the tile
            const int64_t cell = base + lr;
            if (u > 0) xyz.step(a, CPI);
            double2 acc[H], ctr[H];
#pragma unroll
            for (int h = 0; h < H; ++h) acc[h] = ctr[h] = make_double2(0.0, 0.0);
            if (cell < c1) {
                Coef k;
                load_coef_at(a, cell, xyz.ix, xyz.iy, xyz.iz, zlo, zhi, k);
                auto row = [&](int64_t c, double coef, bool has) {
                    if (!has) return;
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        const double2 x = *reinterpret_cast<const double2*>(a.P + c * S + col + 2 * h);
                        acc[h].x = fma(coef, x.x, acc[h].x);
                        acc[h].y = fma(coef, x.y, acc[h].y);
                    }
                };
                row(cell - plane, k.zm, k.hzm);
                row(cell - a.nx, k.ym, k.hym);
                row(cell - 1, k.xm, k.hxm);
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    ctr[h] = *reinterpret_cast<const double2*>(a.P + cell * S + col + 2 * h);
                    acc[h].x = fma(k.d, ctr[h].x, acc[h].x);
                    acc[h].y = fma(k.d, ctr[h].y, acc[h].y);
                }
                row(cell + 1, k.xp, k.hxp);
                row(cell + a.nx, k.yp, k.hyp);
                row(cell + plane, k.zp, k.hzp);
#pragma unroll
                for (int h = 0; h < H; ++h)
                    *reinterpret_cast<double2*>(a.W + cell * S + col + 2 * h) = acc[h];
            }
#pragma unroll
            for (int h = 0; h < H; ++h) {
                *reinterpret_cast<double2*>(tp + lr * RS + col + 2 * h) = ctr[h];
                *reinterpret_cast<double2*>(tw + lr * RS + col + 2 * h) = acc[h];
            }
        }
        __syncwarp();
        // G += P^T W over the tile's 16 cells (K = cells)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const int c4 = 4 * kk + t;
#pragma unroll
            for (int m = 0; m < GramAcc<S>::MT; ++m) {
                const double a0 = tp[c4 * RS + 16 * m + g];
                const double a1 = (16 * m + 8 + g < S) ? tp[c4 * RS + 16 * m + 8 + g] : 0.0;
#pragma unroll
                for (int n = 0; n < GramAcc<S>::NT; ++n)
                    if (gram_tile_needed(m, n)) dmma(G.d[m][n], a0, a1, tw[c4 * RS + 8 * n + g]);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// phase 1 through a shared-memory row ring (single-plane chips outside
// resident mode: the batched C2 solve). The per-tile version above keeps only
// one tile's loads in flight per warp (~2.4 KB): at 16 warps per SM that is
// below the bytes in flight DRAM needs, and the batched sweep ran at 2.9 TB/s.
// Here thread 0 streams whole x-rows — the P row (nx S doubles) and the diag,
// cx, cy rows — into a 4-slot ring by TMA bulk copies (mbarrier completion)
// two rows ahead of the row the warps sweep, so each row's P arrives once and
// the y +- 1 neighbours are read from shared memory. Same per-element FMA
// chain, same 16-cell Gram tiles (in row order): bitwise the per-tile sweep's
// W; the Gram partials are summed in a different tile order.
// ---------------------------------------------------------------------------
constexpr int kRing = 4;
__device__ __forceinline__ unsigned sm_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void ring_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void ring_copy(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(sm_u32(dst)),
        "l"(src), "r"(bytes), "r"(sm_u32(bar))
        : "memory");
}
__device__ __forceinline__ void ring_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tRGW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra RGW_%=;\n\t}" ::"r"(sm_u32(bar)),
        "r"(parity)
        : "memory");
}

struct Ring {
    double* P;                // kRing x nx S
    double* C;                // kRing x 3 nx: diag, cx, cy rows
    unsigned long long* bar;  // kRing "full" (TMA landed), then kRing "empty" (NW warps done)
    unsigned ph;              // parity bits: full slots (all threads), empty slots (thread 0)
};

template <int S>
__device__ void phase_spmm_gram_ring(const Args& a, int64_t c0, int64_t c1, int64_t rlo,
                                     int64_t rhi, int warp, int lane, Ring& rg, double* tw,
                                     GramAcc<S>& G) {
    constexpr int NW = CtaShape<S>::NW;
    constexpr int RS = Strides<S>::RS;
    constexpr int LPR = S / 2, CPI = 32 / LPR, U = 16 / CPI;
    const int nx = a.nx;
    const int q = lane / LPR, col = 2 * (lane % LPR);
    const int g = lane >> 2, t = lane & 3;
    const int64_t r0 = c0 / nx, r1 = (c1 - 1) / nx;
    // rows the sweep reads: r0 - 1 .. r1 + 1, inside the chip
    const int64_t ra = r0 - 1 > rlo ? r0 - 1 : rlo, rb = r1 + 1 < rhi ? r1 + 1 : rhi;
    const unsigned pbytes = (unsigned)nx * S * 8, cbytes = (unsigned)nx * 8;
    auto issue = [&](int64_t r) {  // thread 0
        if (r < ra || r > rb) return;
        const int sl = (int)(r & (kRing - 1));
        ring_expect(&rg.bar[sl], pbytes + 3 * cbytes);
        ring_copy(rg.P + (int64_t)sl * nx * S, a.P + r * nx * S, pbytes, &rg.bar[sl]);
        double* cs = rg.C + (int64_t)sl * 3 * nx;
        ring_copy(cs, a.diag + r * nx, cbytes, &rg.bar[sl]);
        ring_copy(cs + nx, a.cx + r * nx, cbytes, &rg.bar[sl]);
        ring_copy(cs + 2 * nx, a.cy + r * nx, cbytes, &rg.bar[sl]);
    };
    auto wait_row = [&](int64_t r) {  // every thread, once per issued row
        if (r < ra || r > rb) return;
        const int sl = (int)(r & (kRing - 1));
        ring_wait(&rg.bar[sl], (rg.ph >> sl) & 1u);
        rg.ph ^= 1u << sl;
    };
    if (threadIdx.x == 0) {
        // the ring's previous contents were read / written by the generic proxy;
        // P rows of this and neighbouring CTAs were written by generic global
        // stores before the last group barrier
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
        for (int64_t r = ra; r <= r0 + 2; ++r) issue(r);
    }
    wait_row(r0 - 1);
    wait_row(r0);
    for (int64_t r = r0; r <= r1; ++r) {
        wait_row(r + 1);
        const int64_t cs = r * nx > c0 ? r * nx : c0;
        const int64_t ce = (r + 1) * nx < c1 ? (r + 1) * nx : c1;
        const int iy = (int)(r % a.ny);
        const bool hym = iy > 0 && r - 1 >= rlo, hyp = iy < a.ny - 1 && r + 1 <= rhi;
        const double* Pm = rg.P + (int64_t)((r - 1) & (kRing - 1)) * nx * S;
        const double* P0 = rg.P + (int64_t)(r & (kRing - 1)) * nx * S;
        const double* Pp = rg.P + (int64_t)((r + 1) & (kRing - 1)) * nx * S;
        const double* C0 = rg.C + (int64_t)(r & (kRing - 1)) * 3 * nx;
        const double* cym = rg.C + (int64_t)((r - 1) & (kRing - 1)) * 3 * nx + 2 * nx;
        const int ntile = (int)((ce - cs + 15) / 16);
        for (int j = warp; j < ntile; j += NW) {
            const int64_t base = cs + 16 * j;
            const int xb = (int)(base - r * nx);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int lr = q + CPI * u;
                const int x = xb + lr;
                double2 acc = make_double2(0.0, 0.0);
                if (base + lr < ce) {
                    // CSR order y-, x-, diag, x+, y+ (single plane: no z terms)
                    const bool hxm = x > 0, hxp = x < nx - 1;
                    auto row = [&](const double* src, double coef) {
                        const double2 v = *reinterpret_cast<const double2*>(src + col);
                        acc.x = fma(coef, v.x, acc.x);
                        acc.y = fma(coef, v.y, acc.y);
                    };
                    if (hym) row(Pm + x * S, -cym[x]);
                    if (hxm) row(P0 + (x - 1) * S, -C0[nx + x - 1]);
                    row(P0 + x * S, C0[x]);
                    if (hxp) row(P0 + (x + 1) * S, -C0[nx + x]);
                    if (hyp) row(Pp + x * S, -C0[2 * nx + x]);
                    *reinterpret_cast<double2*>(a.W + (base + lr) * S + col) = acc;
                }
                *reinterpret_cast<double2*>(tw + lr * RS + col) = acc;
            }
            __syncwarp();
            // G += P^T W over the tile's 16 cells: P straight from the ring row
            // (rows past the range contribute 0 through W = 0)
            const double* tp = P0 + xb * S;
            const int nv = (int)(ce - base < 16 ? ce - base : 16);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int c4 = 4 * kk + t;
#pragma unroll
                for (int m = 0; m < GramAcc<S>::MT; ++m) {
                    const double a0 = c4 < nv ? tp[c4 * S + 16 * m + g] : 0.0;
                    const double a1 =
                        (c4 < nv && 16 * m + 8 + g < S) ? tp[c4 * S + 16 * m + 8 + g] : 0.0;
#pragma unroll
                    for (int n = 0; n < GramAcc<S>::NT; ++n)
                        if (gram_tile_needed(m, n)) dmma(G.d[m][n], a0, a1, tw[c4 * RS + 8 * n + g]);
                }
            }
            __syncwarp();
        }
        // row r was the last reader of row r - 1's slot: each warp releases it,
        // and the producer refills it once all have (no CTA-wide barrier per
        // row: warps drift, hiding one another's Gram / stencil latency)
        __syncwarp();
        const int fr = (int)((r - 1) & (kRing - 1));
        if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_u32(&rg.bar[kRing + fr]))
                         : "memory");
        if (threadIdx.x == 0) {
            ring_wait(&rg.bar[kRing + fr], (rg.ph >> (kRing + fr)) & 1u);
            rg.ph ^= 1u << (kRing + fr);
            issue(r + 3);
        }
    }
    __syncthreads();  // the coefficient rows (tileR area) are read no more
}

// Rows [base, base + 16) of V (n x S) into the warp tile T[16][RS] by
// cp.async whole-row 16-byte copies (rows past c1 zero-filled). The caller
// commits / waits; __syncwarp before reading.
template <int S>
__device__ __forceinline__ void stage_tile(double* T, const double* __restrict__ V, int64_t base,
                                           int64_t c1, int lane) {
    constexpr int RS = Strides<S>::RS;
    constexpr int LPR = S / 2, CPI = 32 / LPR, U = 16 / CPI;
    const int q = lane / LPR, col = 2 * (lane % LPR);
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int lr = q + CPI * u;
        double* dst = T + lr * RS + col;
        if (base + lr < c1) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
                         "l"(V + (base + lr) * S + col)
                         : "memory");
        } else {
            *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
        }
    }
}

__device__ __forceinline__ void cp_commit_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most N of this thread's committed groups are still in flight
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// A fragments of a staged tile: f[ks][0] = T[g][4ks+t], f[ks][1] = T[g+8][4ks+t]
template <int S>
__device__ __forceinline__ void afrag_smem(const double* T, int g, int t, double (&f)[S / 4][2],
                                           double sign) {
    constexpr int RS = Strides<S>::RS;
#pragma unroll
    for (int ks = 0; ks < S / 4; ++ks) {
        f[ks][0] = sign * T[g * RS + 4 * ks + t];
        f[ks][1] = sign * T[(g + 8) * RS + 4 * ks + t];
    }
}

// A-fragment loads of a 16-cell tile: frag[ks][0] = V[base+g][4ks+t],
// frag[ks][1] = V[base+g+8][4ks+t]; rows beyond c1 read as 0.
template <int S>
__device__ __forceinline__ void load_afrag(const double* __restrict__ V, int64_t base, int64_t c1,
                                           int g, int t, double (&f)[S / 4][2], double sign) {
    const bool v0 = base + g < c1, v1 = base + g + 8 < c1;
#pragma unroll
    for (int ks = 0; ks < S / 4; ++ks) {
        f[ks][0] = v0 ? sign * V[(base + g) * S + 4 * ks + t] : 0.0;
        f[ks][1] = v1 ? sign * V[(base + g + 8) * S + 4 * ks + t] : 0.0;
    }
}

// C-layout tile load/store: c[nt] = {V[r0][8nt+2t], V[r0][..+1], V[r1][8nt+2t], V[r1][..+1]}
template <int S>
__device__ __forceinline__ void load_ctile(const double* __restrict__ V, int64_t base, int64_t c1,
                                           int g, int t, double (&c)[S / 8][4]) {
    const bool v0 = base + g < c1, v1 = base + g + 8 < c1;
#pragma unroll
    for (int n = 0; n < S / 8; ++n) {
        double2 x0 = v0 ? *reinterpret_cast<const double2*>(V + (base + g) * S + 8 * n + 2 * t)
                        : make_double2(0.0, 0.0);
        double2 x1 = v1 ? *reinterpret_cast<const double2*>(V + (base + g + 8) * S + 8 * n + 2 * t)
                        : make_double2(0.0, 0.0);
        c[n][0] = x0.x;
        c[n][1] = x0.y;
        c[n][2] = x1.x;
        c[n][3] = x1.y;
    }
}

template <int S>
__device__ __forceinline__ void store_ctile(double* __restrict__ V, int64_t base, int64_t c1,
                                            int g, int t, const double (&c)[S / 8][4]) {
    const bool v0 = base + g < c1, v1 = base + g + 8 < c1;
#pragma unroll
    for (int n = 0; n < S / 8; ++n) {
        if (v0)
            *reinterpret_cast<double2*>(V + (base + g) * S + 8 * n + 2 * t) =
                make_double2(c[n][0], c[n][1]);
        if (v1)
            *reinterpret_cast<double2*>(V + (base + g + 8) * S + 8 * n + 2 * t) =
                make_double2(c[n][2], c[n][3]);
    }
}

// Gram of two C-layout tiles through a warp-private transpose:
// G += Rt^T Zt over the tile's 16 cells.
template <int S>
__device__ __forceinline__ void tile_gram(double* tr, double* tz, const double (&r)[S / 8][4],
                                          const double (&z)[S / 8][4], int g, int t,
                                          GramAcc<S>& G) {
    constexpr int RS = Strides<S>::RS;
#pragma unroll
    for (int n = 0; n < S / 8; ++n) {
        const int col = 8 * n + 2 * t;
        *reinterpret_cast<double2*>(tr + g * RS + col) = make_double2(r[n][0], r[n][1]);
        *reinterpret_cast<double2*>(tr + (g + 8) * RS + col) = make_double2(r[n][2], r[n][3]);
        *reinterpret_cast<double2*>(tz + g * RS + col) = make_double2(z[n][0], z[n][1]);
        *reinterpret_cast<double2*>(tz + (g + 8) * RS + col) = make_double2(z[n][2], z[n][3]);
    }
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const int cell = 4 * kk + t;
#pragma unroll
        for (int m = 0; m < GramAcc<S>::MT; ++m) {
            const double a0 = tr[cell * RS + 16 * m + g];
            const double a1 = (16 * m + 8 + g < S) ? tr[cell * RS + 16 * m + 8 + g] : 0.0;
#pragma unroll
            for (int n = 0; n < GramAcc<S>::NT; ++n)
                if (gram_tile_needed(m, n)) dmma(G.d[m][n], a0, a1, tz[cell * RS + 8 * n + g]);
        }
    }
    __syncwarp();
}

// resident (smem) C-layout tiles: local cell l, even column c -> swizzled slot
template <int S>
__device__ __forceinline__ int res_idx(int l, int c) {
    const int chunk = c >> 1;
    const int sw = (S / 2 >= 8) ? ((l & 1) << 2) : 0;
    return l * S + ((chunk ^ sw) << 1);
}

template <int S>
__device__ __forceinline__ void load_rtile(const double* v, int lb, int cnt, int g, int t,
                                           double (&c)[S / 8][4]) {
    const bool v0 = lb + g < cnt, v1 = lb + g + 8 < cnt;
#pragma unroll
    for (int n = 0; n < S / 8; ++n) {
        const double2 x0 = v0 ? *reinterpret_cast<const double2*>(v + res_idx<S>(lb + g, 8 * n + 2 * t))
                              : make_double2(0.0, 0.0);
        const double2 x1 = v1 ? *reinterpret_cast<const double2*>(v + res_idx<S>(lb + g + 8, 8 * n + 2 * t))
                              : make_double2(0.0, 0.0);
        c[n][0] = x0.x;
        c[n][1] = x0.y;
        c[n][2] = x1.x;
        c[n][3] = x1.y;
    }
}

template <int S>
__device__ __forceinline__ void store_rtile(double* v, int lb, int cnt, int g, int t,
                                            const double (&c)[S / 8][4]) {
    const bool v0 = lb + g < cnt, v1 = lb + g + 8 < cnt;
#pragma unroll
    for (int n = 0; n < S / 8; ++n) {
        if (v0)
            *reinterpret_cast<double2*>(v + res_idx<S>(lb + g, 8 * n + 2 * t)) =
                make_double2(c[n][0], c[n][1]);
        if (v1)
            *reinterpret_cast<double2*>(v + res_idx<S>(lb + g + 8, 8 * n + 2 * t)) =
                make_double2(c[n][2], c[n][3]);
    }
}

// X or R of a 16-cell tile: shared-memory resident or the HBM block vector
template <int S, bool RES>
struct TileVec {
    double* g;   // global n x S
    double* sm;  // resident (RES) local cells x S
    int64_t c0, c1;
    __device__ __forceinline__ void load(int64_t base, int gg, int t, double (&c)[S / 8][4]) const {
        if (RES)
            load_rtile<S>(sm, (int)(base - c0), (int)(c1 - c0), gg, t, c);
        else
            load_ctile<S>(g, base, c1, gg, t, c);
    }
    __device__ __forceinline__ void store(int64_t base, int gg, int t,
                                          const double (&c)[S / 8][4]) const {
        if (RES)
            store_rtile<S>(sm, (int)(base - c0), (int)(c1 - c0), gg, t, c);
        else
            store_ctile<S>(g, base, c1, gg, t, c);
    }
};

__device__ __forceinline__ double dinv_at(const Args& a, int64_t c, int64_t c1, bool jac) {
    return (jac && c < c1) ? a.dinv[c] : 1.0;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
// DEF: X += P alpha deferred from phase 2 to phase 3 (see below); a
// compile-time choice so the other instantiations keep their registers
template <int S, bool RES, bool MULTI, bool DEF>
__global__ void __launch_bounds__(CtaShape<S>::BS, 1) block_cg_dmma_kernel(Args a) {
    constexpr int BS = CtaShape<S>::BS, NW = CtaShape<S>::NW;
    constexpr int NT = S / 8;
    constexpr int KS = S / 4;
    constexpr int E = S * S + S;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Sm<S, RES>& sm = *reinterpret_cast<Sm<S, RES>*>(smem_raw);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    Group<MULTI> gr;
    if constexpr (MULTI) {
        gr.NB = a.cpc;
        gr.chip = (int)blockIdx.x / gr.NB;
        gr.b = (int)blockIdx.x % gr.NB;
        gr.bar = a.bars + 2 * gr.chip;
    } else {
        gr.NB = (int)gridDim.x;
        gr.chip = 0;
        gr.b = (int)blockIdx.x;
        gr.bar = nullptr;
    }
    gr.ring = a.ring != 0;
    const int NB = gr.NB, b = gr.b;
    constexpr bool kAlias = scratch_aliases_tiles<S>();
    double* const scr = kAlias ? &sm.tileR[0][0] : sm.scratch;
    constexpr int kScrStride = kAlias ? 16 * Strides<S>::RS : S * S;
    // CTA ranges in whole 16-cell tiles of this chip (the last CTA takes the
    // ragged end); per-chip reduction buffers and report
    const int64_t nchip = MULTI ? a.nchip : a.n;
    const int64_t cbase = MULTI ? (int64_t)gr.chip * nchip : 0;
    const int64_t ntiles = (nchip + 15) / 16;
    const int64_t c0 = cbase + 16 * (ntiles * b / NB);
    const int64_t c1 = b == NB - 1 ? cbase + nchip : cbase + 16 * (ntiles * (b + 1) / NB);
    // the chip's z range inside the z-stacked batch (the whole grid otherwise)
    const int nzc = MULTI ? a.nz / a.nchips : a.nz;
    const int zlo = gr.chip * nzc, zhi = zlo + nzc - 1;
    double* const partc = MULTI ? a.part + (int64_t)gr.chip * NB * (S * S + S) : a.part;
    double* const redc = MULTI ? a.red + (int64_t)gr.chip * (S * S + S) : a.red;
    bk::CgReport* const repc = MULTI ? a.rep + gr.chip : a.rep;
    const bool jac = a.precond != 0;
    const bool prof = a.prof != nullptr && gr.chip == 0 && b == 0 && tid == 0;
    double* tr = sm.tileR[warp];
    double* tz = sm.tileZ[warp];
    // row ring of phase 1 (a.ring): coefficient rows in the tileR area (free
    // during phase 1), P rows and the slot barriers past Sm
    Ring rg;
    rg.C = &sm.tileR[0][0];
    rg.P = reinterpret_cast<double*>(smem_raw + (sizeof(Sm<S, RES>) + 15) / 16 * 16);
    rg.bar = reinterpret_cast<unsigned long long*>(rg.P + (int64_t)kRing * a.nx * S);
    rg.ph = 0;
    if (a.ring) {
        if (tid == 0) {
            for (int i = 0; i < kRing; ++i)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(&rg.bar[i])));
            for (int i = kRing; i < 2 * kRing; ++i)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(&rg.bar[i])),
                             "r"(NW));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    const int64_t rlo = cbase / a.nx, rhi = (cbase + nchip) / a.nx - 1;  // the chip's x-rows

    double* xres = nullptr;
    double* rres = nullptr;
    if constexpr (RES) {
        xres = sm.res.x;
        rres = sm.res.r;
    }
    const TileVec<S, RES> Xv{a.X, xres, c0, c1};
    const TileVec<S, RES> Rv{a.R, rres, c0, c1};
    if constexpr (RES) {
        for (int64_t c = c0 + tid; c < c1; c += BS) sm.res.dinv[c - c0] = jac ? a.dinv[c] : 1.0;
        __syncthreads();
    }
    // D^-1 of cell c (1.0 past c1 or without Jacobi): shared-memory resident
    // copy in resident mode
    auto dinv_of = [&](int64_t c) -> double {
        if constexpr (RES)
            return c < c1 ? sm.res.dinv[c - c0] : 1.0;
        else
            return dinv_at(a, c, c1, jac);
    };
    // resident X -> HBM (for the stencil sweeps over X and for the output)
    auto publish_x = [&]() {
        if constexpr (RES) {
            for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW) {
                double x[NT][4];
                Xv.load(base, g, t, x);
                store_ctile<S>(a.X, base, c1, g, t, x);
            }
            gr.sync(grid);
        }
    };

    GramAcc<S> G;
    int64_t matvecs = 0;
    int iters = 0;

    // ---- init: X = 0, R = B, Z = D^-1 R, P = Z, bnorm, S_old = R^T Z
    {
        G.zero();
        double bn[NT][2] = {};
        for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW) {
            double r[NT][4], z[NT][4], zero[NT][4];
            load_ctile<S>(a.B, base, c1, g, t, r);
            const double d0 = dinv_of(base + g), d1 = dinv_of(base + g + 8);
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                z[n][0] = d0 * r[n][0];
                z[n][1] = d0 * r[n][1];
                z[n][2] = d1 * r[n][2];
                z[n][3] = d1 * r[n][3];
                bn[n][0] += r[n][0] * r[n][0] + r[n][2] * r[n][2];
                bn[n][1] += r[n][1] * r[n][1] + r[n][3] * r[n][3];
#pragma unroll
                for (int e = 0; e < 4; ++e) zero[n][e] = 0.0;
            }
            Xv.store(base, g, t, zero);
            Rv.store(base, g, t, r);
            store_ctile<S>(a.P, base, c1, g, t, z);
            tile_gram<S>(tr, tz, r, z, g, t, G);
        }
        G.spill(scr + warp * kScrStride, g, t);
        cta_sum_mat<S>(scr, kScrStride, sm.aug);
        cta_sum_vec<S>(bn, scr, kScrStride, sm.aug + S * S, warp, lane);
        grid_reduce<BS, MULTI>(gr, grid, partc, redc, sm.aug, E, sm.aug + E);
        for (int e = tid; e < S * S; e += BS) sm.s_old[e] = sm.aug[E + e];
        if (tid < S) {
            const double bnv = sqrt(sm.aug[E + S * S + tid]);
            sm.bnorm[tid] = bnv;
            sm.act[tid] = bnv != 0.0;
            sm.conv[tid] = bnv == 0.0;
            sm.fres[tid] = 0.0;
        }
        __syncthreads();
        build_index<S>(sm);
    }

    for (int m = 1; m <= a.max_iter && sm.sa > 0; ++m) {
        long long* pm = (prof && m <= PROF_ITERS) ? a.prof + (m - 1) * PROF_MARKS : nullptr;
        if (pm) pm[0] = gtimer();
        // ---- phase 1: W = A P, G = P^T W
        G.zero();
        if (a.ring)
            phase_spmm_gram_ring<S>(a, c0, c1, rlo, rhi, warp, lane, rg, tz, G);
        else
            phase_spmm_gram<S>(a, c0, c1, zlo, zhi, warp, lane, tr, tz, G);
        if (pm) pm[8] = gtimer();
        G.spill(scr + warp * kScrStride, g, t);
        cta_sum_mat<S>(scr, kScrStride, sm.aug);
        if (pm) pm[1] = gtimer();
        grid_reduce<BS, MULTI>(gr, grid, partc, redc, sm.aug, S * S, sm.mat);
        if (pm) pm[2] = gtimer();
        matvecs += sm.sa;
        small_solve<S>(sm, sm.mat, sm.s_old, sm.coef);  // alpha
        for (int e = tid; e < S * Strides<S>::RS; e += BS) sm.akeep[e] = sm.coef[e];
        // X += P alpha deferred to phase 3 (which reads the same P tile: one P
        // read fewer per iteration). Measured: ring mode (C2 x16) +3.3 %, S = 32
        // (C3 x12) +5 %; the per-tile S = 16 sweep (C4) -4 % (the extra X
        // traffic of phase 3 evicts the P rows phase 1 then re-reads), so off
        // there (the host picks DEF = ring || S >= 32).
        constexpr bool defer = DEF;
        bool xdone = !defer;
        if (pm) pm[3] = gtimer();

        // ---- phase 2: [X += P alpha unless deferred], R -= W alpha, rr, Z,
        // S_new = R^T Z
        G.zero();
        double rr[NT][2] = {};
        // With prefetch buffers (a.pre_off >= 0) the W tile of the warp's NEXT
        // 16 cells is in flight (cp.async) while this tile's DMMA chains, R
        // store and Gram run: the single-buffered form exposed one L2 / HBM
        // round trip per tile and warp (batched C2: phase 2 at 4.9 TB/s against
        // phase 3's 6.7).
        // Compiled only into the row-ring kernels (DEF, S <= 16), whose ring
        // slots hold the buffers: measured on the 3D kernels it cost more
        // (shared memory, spills) than it hid (C3 -0.6 %, C4 -2.3 %; C2 +2.7 %).
        constexpr bool kPre = DEF && S <= 16;
        double* const wpre = (kPre && a.pre_off >= 0)
                                 ? reinterpret_cast<double*>(smem_raw + a.pre_off) +
                                       (int64_t)warp * 2 * 16 * Strides<S>::RS
                                 : nullptr;
        if (wpre && c0 + 16 * warp < c1) {
            stage_tile<S>(wpre, a.W, c0 + 16 * warp, c1, lane);
            cp_commit();
        }
        int tix = 0;
        for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW, ++tix) {
            double pa[KS][2], wa[KS][2], x[NT][4], r[NT][4];
            if (!defer) {
                stage_tile<S>(tr, a.P, base, c1, lane);
                Xv.load(base, g, t, x);
            }
            const double* wt = tz;
            if (wpre) {
                if (!defer) cp_commit();  // this tile's P
                const int64_t nxt = base + 16 * NW;
                wt = wpre + (tix & 1) * 16 * Strides<S>::RS;
                Rv.load(base, g, t, r);
                if (nxt < c1) {
                    stage_tile<S>(wpre + ((tix + 1) & 1) * 16 * Strides<S>::RS, a.W, nxt, c1, lane);
                    cp_commit();
                    cp_wait<1>();  // all but the prefetch: this tile's W (and P) landed
                } else {
                    cp_wait<0>();
                }
            } else {
                stage_tile<S>(tz, a.W, base, c1, lane);
                Rv.load(base, g, t, r);
                cp_commit_wait_all();
            }
            __syncwarp();
            if (!defer) afrag_smem<S>(tr, g, t, pa, 1.0);
            afrag_smem<S>(wt, g, t, wa, -1.0);
            __syncwarp();  // tr / tz are rewritten by tile_gram below
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const double bb = sm.coef[(4 * ks + t) * Strides<S>::RS + 8 * n + g];
                    if (!defer) dmma(x[n], pa[ks][0], pa[ks][1], bb);
                    dmma(r[n], wa[ks][0], wa[ks][1], bb);
                }
            if (!defer) Xv.store(base, g, t, x);
            Rv.store(base, g, t, r);
            const double d0 = dinv_of(base + g), d1 = dinv_of(base + g + 8);
            double z[NT][4];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                rr[n][0] += r[n][0] * r[n][0] + r[n][2] * r[n][2];
                rr[n][1] += r[n][1] * r[n][1] + r[n][3] * r[n][3];
                z[n][0] = d0 * r[n][0];
                z[n][1] = d0 * r[n][1];
                z[n][2] = d1 * r[n][2];
                z[n][3] = d1 * r[n][3];
            }
            tile_gram<S>(tr, tz, r, z, g, t, G);
        }
        if (pm) pm[9] = gtimer();
        G.spill(scr + warp * kScrStride, g, t);
        cta_sum_mat<S>(scr, kScrStride, sm.aug);
        cta_sum_vec<S>(rr, scr, kScrStride, sm.aug + S * S, warp, lane);
        if (pm) pm[4] = gtimer();
        grid_reduce<BS, MULTI>(gr, grid, partc, redc, sm.aug, E, sm.aug + E);
        for (int e = tid; e < S * S; e += BS) sm.mat[e] = sm.aug[E + e];  // S_new
        if (tid < S) sm.vec[tid] = sm.aug[E + S * S + tid];              // rr
        __syncthreads();
        iters = m;
        if (pm) pm[5] = gtimer();

        // ---- convergence control (solvers.cpp:582-634)
        if (tid < S) sm.vflag[tid] = sm.act[tid] && (sqrt(sm.vec[tid]) / sm.bnorm[tid] <= a.tol);
        __syncthreads();
        int nver = 0;
#pragma unroll
        for (int q = 0; q < S; ++q) nver += sm.vflag[q];
        bool restart = false;
        // X += P alpha (deferred from phase 2) for every sweep that reads X
        auto x_update = [&]() {
            for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW) {
                double pa[KS][2], x[NT][4];
                stage_tile<S>(tr, a.P, base, c1, lane);
                Xv.load(base, g, t, x);
                cp_commit_wait_all();
                __syncwarp();
                afrag_smem<S>(tr, g, t, pa, 1.0);
                __syncwarp();
#pragma unroll
                for (int n = 0; n < NT; ++n)
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks)
                        dmma(x[n], pa[ks][0], pa[ks][1],
                             sm.akeep[(4 * ks + t) * Strides<S>::RS + 8 * n + g]);
                Xv.store(base, g, t, x);
            }
            // The sweeps that follow apply the stencil to X and so read the
            // halo cells other CTAs of the group just updated: a group
            // barrier, not a CTA one (resident mode gets it from publish_x).
            // Without it the true residual was formed from a mix of old and
            // new X near CTA boundaries and a borderline column could restart
            // in one run and freeze in the next.
            if constexpr (RES)
                __syncthreads();
            else
                gr.sync(grid);
            xdone = true;
        };
        if (nver > 0) {
            if (!xdone) x_update();
            publish_x();
            double rs[NT][2] = {};
            for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t cell = base + g + 8 * h;
                    if (cell >= c1) continue;
                    Coef k;
                    load_coef(a, cell, zlo, zhi, k);
#pragma unroll
                    for (int n = 0; n < NT; ++n)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int col = 8 * n + 2 * t + e;
                            const double rv = a.B[cell * S + col] - st_muladd<S>(k, a.X, cell, col);
                            rs[n][e] += rv * rv;
                        }
                }
            }
            cta_sum_vec<S>(rs, scr, kScrStride, sm.aug, warp, lane);
            grid_reduce<BS, MULTI>(gr, grid, partc, redc, sm.aug, S, sm.aug + S);
            matvecs += nver;
            if (tid == 0) {
                sm.fail = 0;
                for (int q = 0; q < S; ++q) {
                    if (!sm.vflag[q]) continue;
                    const double rt = sqrt(sm.aug[S + q]) / sm.bnorm[q];
                    if (rt <= a.tol) {
                        sm.act[q] = 0;
                        sm.conv[q] = 1;
                        sm.fres[q] = rt;
                    } else {
                        sm.fail = 2;
                    }
                }
            }
            __syncthreads();
            restart = sm.fail == 2;
            build_index<S>(sm);
            if (sm.sa == 0) break;
        }
        if (restart) {
            // R = B - A X, Z, P = Z, S_old = R^T Z (solvers.cpp:616-634)
            G.zero();
            for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW) {
                double r[NT][4], z[NT][4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t cell = base + g + 8 * h;
                    const bool v = cell < c1;
                    Coef k;
                    if (v) load_coef(a, cell, zlo, zhi, k);
                    const double di = dinv_of(cell);
#pragma unroll
                    for (int n = 0; n < NT; ++n)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int col = 8 * n + 2 * t + e;
                            double dummy;
                            const double rv =
                                v ? a.B[cell * S + col] - st_fma<S>(k, a.X, cell, col, dummy) : 0.0;
                            r[n][2 * h + e] = rv;
                            z[n][2 * h + e] = di * rv;
                        }
                }
                Rv.store(base, g, t, r);
                store_ctile<S>(a.P, base, c1, g, t, z);
                tile_gram<S>(tr, tz, r, z, g, t, G);
            }
            G.spill(scr + warp * kScrStride, g, t);
            cta_sum_mat<S>(scr, kScrStride, sm.aug);
            grid_reduce<BS, MULTI>(gr, grid, partc, redc, sm.aug, S * S, sm.s_old);
            matvecs += sm.sa;
            continue;
        }

        // ---- phase 3: beta = S_old^+ S_new, S_old = S_new, P = Z + P beta
        small_solve<S>(sm, sm.s_old, sm.mat, sm.coef);
        for (int e = tid; e < S * S; e += BS) sm.s_old[e] = sm.mat[e];
        if (pm) pm[6] = gtimer();
        for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW) {
            double pa[KS][2], p[NT][4], x[NT][4];
            stage_tile<S>(tr, a.P, base, c1, lane);
            Rv.load(base, g, t, p);
            if (!xdone) Xv.load(base, g, t, x);
            cp_commit_wait_all();
            __syncwarp();
            afrag_smem<S>(tr, g, t, pa, 1.0);
            __syncwarp();
            if (!xdone) {  // X += P alpha with the same P tile (deferred from phase 2)
#pragma unroll
                for (int n = 0; n < NT; ++n)
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks)
                        dmma(x[n], pa[ks][0], pa[ks][1],
                             sm.akeep[(4 * ks + t) * Strides<S>::RS + 8 * n + g]);
                Xv.store(base, g, t, x);
            }
            const double d0 = dinv_of(base + g), d1 = dinv_of(base + g + 8);
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                p[n][0] *= d0;
                p[n][1] *= d0;
                p[n][2] *= d1;
                p[n][3] *= d1;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
                    dmma(p[n], pa[ks][0], pa[ks][1], sm.coef[(4 * ks + t) * Strides<S>::RS + 8 * n + g]);
            }
            store_ctile<S>(a.P, base, c1, g, t, p);
        }
        gr.sync(grid);
        if (pm) pm[7] = gtimer();
    }

    // ---- exit: honest residuals for still-active columns (:655-661)
    publish_x();
    if (sm.sa > 0) {
        double rs[NT][2] = {};
        for (int64_t base = c0 + 16 * warp; base < c1; base += 16 * NW) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t cell = base + g + 8 * h;
                if (cell >= c1) continue;
                Coef k;
                load_coef(a, cell, zlo, zhi, k);
#pragma unroll
                for (int n = 0; n < NT; ++n)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = 8 * n + 2 * t + e;
                        const double rv = a.B[cell * S + col] - st_muladd<S>(k, a.X, cell, col);
                        rs[n][e] += rv * rv;
                    }
            }
        }
        cta_sum_vec<S>(rs, scr, kScrStride, sm.aug, warp, lane);
        grid_reduce<BS, MULTI>(gr, grid, partc, redc, sm.aug, S, sm.aug + S);
        matvecs += sm.sa;
        if (tid < S && sm.act[tid]) {
            const double rt = sqrt(sm.aug[S + tid]) / sm.bnorm[tid];
            sm.fres[tid] = rt;
            sm.conv[tid] = rt <= a.tol;
        }
        __syncthreads();
    }
    if (b == 0 && tid == 0) {
        repc->iterations = iters;
        repc->matvecs = matvecs;
        for (int q = 0; q < S; ++q) {
            repc->final_res[q] = sm.fres[q];
            repc->converged[q] = (char)sm.conv[q];
        }
    }
}

// Row-ring phase 1 (phase_spmm_gram_ring) for single-plane chips outside
// resident mode when the ring fits; BK_CG_RING=0/1 overrides (A/B).
template <int S>
size_t ring_bytes(int nx) {
    return 16 + (size_t)kRing * nx * S * sizeof(double) + 2 * kRing * sizeof(unsigned long long);
}
template <int S>
bool want_ring(const bk_ctx* ctx, bool resident, int nx, int nz_chip) {
    if (resident || nz_chip != 1 || nx % 16 != 0 || S > 16) return false;
    if ((size_t)3 * kRing * nx > (size_t)CtaShape<S>::NW * 16 * Strides<S>::RS) return false;
    if (sizeof(Sm<S, false>) + ring_bytes<S>(nx) > 232448) return false;
    if (ctx->knobs.ring >= 0) return ctx->knobs.ring != 0;
    return true;
}

// Phase 2's W prefetch buffers (NW warps x 2 tiles of 16 x RS doubles) in the
// dynamic shared memory past Sm, for the row-ring kernels: inside the ring's P
// slots when they are large enough (the ring is idle in phase 2; its mbarriers
// sit past the slots), else past the ring. Returns the byte offset, -1 for
// none, and grows `smem` as needed.
template <int S>
int place_prefetch(bool resident, bool ring, int nx, size_t& smem) {
    if (resident || !ring) return -1;  // row-ring kernels only (see phase 2)
    const size_t base = (sizeof(Sm<S, false>) + 15) / 16 * 16;
    const size_t need = (size_t)CtaShape<S>::NW * 2 * 16 * Strides<S>::RS * sizeof(double);
    if (need <= (size_t)kRing * nx * S * sizeof(double)) return (int)base;
    const size_t off = (base + ring_bytes<S>(nx) + 15) / 16 * 16;
    if (off + need > 232448) return -1;
    if (off + need > smem) smem = off + need;
    return (int)off;
}

template <int S>
std::string variant_name(bool res, bool multi, bool def, bool ring) {
    return "block_cg_dmma_kernel<" + std::to_string(S) + "," + (res ? "1" : "0") + "," +
           (multi ? "1" : "0") + "," + (def ? "1" : "0") + ">" + (ring ? " ring" : "");
}

template <int S>
bk_status run_dmma(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                   const bk_solver_cfg* cfg, double* X, bk::CgReport* rep) {
    using namespace bk;
    const int64_t n = op->n;
    const size_t vec_bytes = (size_t)n * S * sizeof(double);
    constexpr int BS = CtaShape<S>::BS;
    int64_t nb = ctx->num_sms;  // one CTA per SM (see CtaShape)
    if (ctx->cg_max_ctas > 0 && nb > ctx->cg_max_ctas) nb = ctx->cg_max_ctas;
    const int64_t ntiles = (n + 15) / 16;
    const int64_t min_tiles = 2;
    if (nb * min_tiles > ntiles) nb = (ntiles + min_tiles - 1) / min_tiles;
    if (nb < 1) nb = 1;
    // shared-memory-resident X/R when every CTA's range fits (S <= 16)
    const int64_t max_cells = 16 * ((ntiles + nb - 1) / nb);
    const bool resident = S <= 16 && max_cells <= kResCells && !ctx->knobs.no_resident;
    const bool ring = want_ring<S>(ctx, resident, op->nx, op->nz);
    const bool defer = !resident && (ring || S >= 32) && !ctx->knobs.no_defer_x;
    const void* kern = resident ? (const void*)block_cg_dmma_kernel<S, true, false, false>
                       : defer  ? (const void*)block_cg_dmma_kernel<S, false, false, true>
                                : (const void*)block_cg_dmma_kernel<S, false, false, false>;
    size_t smem = (resident ? sizeof(Sm<S, true>) : sizeof(Sm<S, false>)) +
                  (ring ? ring_bytes<S>(op->nx) : 0);
    const int pre_off = ctx->knobs.no_w_prefetch ? -1 : place_prefetch<S>(resident, ring, op->nx, smem);
    ctx->last_variant = variant_name<S>(resident, false, defer, ring);
    BK_CUDA_TRY(ctx, bk::set_max_smem((const void*)kern, smem));
    int occ = 0;
    BK_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BS, smem));
    if (occ < 1) return fail(ctx, BK_INTERNAL, "block_cg: DMMA kernel cannot be resident");
    const int E = S * S + S;

    void *pB, *pX, *pR, *pP, *pW, *pPart, *pRed, *pRep;
    bk_status st;
    const bool padded = s != S;
    if ((st = workspace(ctx, kSlotCgR, vec_bytes, &pR)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgP, vec_bytes, &pP)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgW, vec_bytes, &pW)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgPart, (size_t)nb * E * sizeof(double), &pPart)) != BK_OK)
        return st;
    if ((st = workspace(ctx, kSlotCgRed, (size_t)E * sizeof(double), &pRed)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgCtl,
                        sizeof(CgReport) + PROF_ITERS * PROF_MARKS * sizeof(long long), &pRep)) !=
        BK_OK)
        return st;
    if (padded) {
        if ((st = workspace(ctx, kSlotCgB, vec_bytes, &pB)) != BK_OK) return st;
        if ((st = workspace(ctx, kSlotCgX, vec_bytes, &pX)) != BK_OK) return st;
        BK_CUDA_TRY(ctx, launch_pad_cols(ctx, B, s, (double*)pB, S, n));
    } else {
        pB = const_cast<double*>(B);
        pX = X;
    }
    Args a;
    a.nx = op->nx;
    a.ny = op->ny;
    a.nz = op->nz;
    a.n = n;
    a.diag = op->diag;
    a.cx = op->cx;
    a.cy = op->cy;
    a.cz = op->cz;
    a.dinv = op->dinv;
    a.B = (const double*)pB;
    a.X = (double*)pX;
    a.R = (double*)pR;
    a.P = (double*)pP;
    a.W = (double*)pW;
    a.part = (double*)pPart;
    a.red = (double*)pRed;
    a.tol = cfg->rel_tol;
    a.max_iter = cfg->max_iter;
    a.precond = cfg->precond;
    a.rep = (CgReport*)pRep;
    a.nchips = 1;
    a.cpc = (int)nb;
    a.nchip = n;
    a.bars = nullptr;
    a.ring = ring;
    a.pre_off = pre_off;
    const bool want_prof = ctx->knobs.cg_profile;
    a.prof = want_prof ? (long long*)((char*)pRep + sizeof(CgReport)) : nullptr;
    if (want_prof)
        BK_CUDA_TRY(ctx, cudaMemsetAsync(a.prof, 0, PROF_ITERS * PROF_MARKS * sizeof(long long),
                                         ctx->stream));
    void* args[] = {&a};
    const bool trace = ctx->knobs.batch_trace;
    if (trace) fprintf(stderr, "[trace ctx %p] launch cg nb=%lld\n", (void*)ctx, (long long)nb);
    BK_CUDA_TRY(ctx, cudaLaunchCooperativeKernel(kern, dim3((unsigned)nb), dim3(BS), args, smem,
                                                 ctx->stream));
    if (trace) fprintf(stderr, "[trace ctx %p] launched\n", (void*)ctx);
    ++ctx->launches;
    if (padded) BK_CUDA_TRY(ctx, launch_pad_cols(ctx, (const double*)pX, S, X, s, n));
    {
        const bk_status rs = read_small(ctx, rep, pRep, sizeof(CgReport));
        if (trace) fprintf(stderr, "[trace ctx %p] cg done\n", (void*)ctx);
        if (rs != BK_OK) return rs;
    }
    if (want_prof) {
        std::vector<long long> pr(PROF_ITERS * PROF_MARKS);
        cudaMemcpy(pr.data(), a.prof, pr.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        // mean phase durations over the recorded iterations (ns)
        double acc[PROF_MARKS] = {};
        int cnt = 0;
        double loop1 = 0, loop2 = 0;
        for (int i = 1; i < PROF_ITERS; ++i) {
            const long long* r = pr.data() + i * PROF_MARKS;
            if (!r[0] || !r[7]) continue;
            for (int k = 1; k < 8; ++k) acc[k] += (double)(r[k] - r[k - 1]);
            loop1 += (double)(r[8] - r[0]);
            loop2 += (double)(r[9] - r[3]);
            acc[0] += (double)(pr[(i + 1) * PROF_MARKS] ? pr[(i + 1) * PROF_MARKS] - r[7] : 0);
            ++cnt;
        }
        if (cnt)
            fprintf(stderr,
                    "[bk_cg_profile S=%d nb=%lld res=%d] per-iteration ns: phase1 %.0f | reduceG %.0f | "
                    "solve_a %.0f | phase2 %.0f | reduceS %.0f | control+solve_b %.0f | "
                    "phase3+sync %.0f (over %d iterations); tile loops: phase1 %.0f phase2 %.0f\n",
                    S, (long long)nb, (int)resident, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt,
                    acc[5] / cnt, acc[6] / cnt, acc[7] / cnt, cnt, loop1 / cnt, loop2 / cnt);
    }
    return BK_OK;
}

}  // namespace

namespace bk {

// K independent chips of identical dims, z-stacked into one block-diagonal
// system (op: nz = K nz_chip, n = K n_chip; B, X: K n_chip x S), solved by one
// cooperative launch in which chip k owns an equal share of the SMs.
template <int S>
bk_status run_dmma_multi(bk_ctx* ctx, const bk_operator* op, int K, const double* B,
                         const bk_solver_cfg* cfg, double* X, CgReport* reps) {
    const int64_t n = op->n, nchip = n / K;
    constexpr int BS = CtaShape<S>::BS;
    int cpc = ctx->num_sms / K;
    const int64_t ntiles = (nchip + 15) / 16;
    if ((int64_t)cpc * 2 > ntiles) cpc = (int)((ntiles + 1) / 2);
    if (cpc < 1) return fail(ctx, BK_INVALID_CONFIG, "block_cg: too many chips for the SMs");
    const int64_t nb = (int64_t)K * cpc;
    const int64_t max_cells = 16 * ((ntiles + cpc - 1) / cpc);
    const bool resident = S <= 16 && max_cells <= kResCells && !ctx->knobs.no_resident;
    const bool ring = want_ring<S>(ctx, resident, op->nx, op->nz / K);
    const bool defer = !resident && (ring || S >= 32) && !ctx->knobs.no_defer_x;
    const void* kern = resident ? (const void*)block_cg_dmma_kernel<S, true, true, false>
                       : defer  ? (const void*)block_cg_dmma_kernel<S, false, true, true>
                                : (const void*)block_cg_dmma_kernel<S, false, true, false>;
    size_t smem = (resident ? sizeof(Sm<S, true>) : sizeof(Sm<S, false>)) +
                  (ring ? ring_bytes<S>(op->nx) : 0);
    const int pre_off = ctx->knobs.no_w_prefetch ? -1 : place_prefetch<S>(resident, ring, op->nx, smem);
    ctx->last_variant = variant_name<S>(resident, true, defer, ring) +
                        " chips=" + std::to_string(K);
    BK_CUDA_TRY(ctx, set_max_smem(kern, smem));
    int occ = 0;
    BK_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BS, smem));
    if (occ < 1 || nb > (int64_t)occ * ctx->num_sms)
        return fail(ctx, BK_INTERNAL, "block_cg: batched DMMA kernel cannot be resident");
    constexpr int E = S * S + S;
    const size_t vec_bytes = (size_t)n * S * sizeof(double);
    void *pR, *pP, *pW, *pPart, *pRed, *pRep, *pBar;
    bk_status st;
    if ((st = workspace(ctx, kSlotCgR, vec_bytes, &pR)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgP, vec_bytes, &pP)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgW, vec_bytes, &pW)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgPart, (size_t)nb * E * sizeof(double), &pPart)) != BK_OK)
        return st;
    if ((st = workspace(ctx, kSlotCgRed, (size_t)K * E * sizeof(double), &pRed)) != BK_OK)
        return st;
    if ((st = workspace(ctx, kSlotCgCtl, (size_t)K * sizeof(CgReport), &pRep)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgBars, (size_t)2 * K * sizeof(unsigned), &pBar)) != BK_OK)
        return st;
    BK_CUDA_TRY(ctx, cudaMemsetAsync(pBar, 0, (size_t)2 * K * sizeof(unsigned), ctx->stream));
    Args a;
    a.nx = op->nx;
    a.ny = op->ny;
    a.nz = op->nz;
    a.n = n;
    a.diag = op->diag;
    a.cx = op->cx;
    a.cy = op->cy;
    a.cz = op->cz;
    a.dinv = op->dinv;
    a.B = B;
    a.X = X;
    a.R = (double*)pR;
    a.P = (double*)pP;
    a.W = (double*)pW;
    a.part = (double*)pPart;
    a.red = (double*)pRed;
    a.tol = cfg->rel_tol;
    a.max_iter = cfg->max_iter;
    a.precond = cfg->precond;
    a.rep = (CgReport*)pRep;
    a.prof = nullptr;
    const bool want_prof = ctx->knobs.cg_profile;
    long long* dprof = nullptr;
    if (want_prof) {
        void* pp;
        if ((st = workspace(ctx, kSlotCgFlags, PROF_ITERS * PROF_MARKS * sizeof(long long), &pp)) !=
            BK_OK)
            return st;
        dprof = (long long*)pp;
        BK_CUDA_TRY(ctx, cudaMemsetAsync(dprof, 0, PROF_ITERS * PROF_MARKS * sizeof(long long),
                                         ctx->stream));
        a.prof = dprof;
    }
    a.nchips = K;
    a.cpc = cpc;
    a.nchip = nchip;
    a.bars = (unsigned*)pBar;
    a.ring = ring;
    a.pre_off = pre_off;
    void* args[] = {&a};
    BK_CUDA_TRY(ctx, cudaLaunchCooperativeKernel(kern, dim3((unsigned)nb), dim3(BS), args, smem,
                                                 ctx->stream));
    ++ctx->launches;
    st = read_small(ctx, reps, pRep, (size_t)K * sizeof(CgReport));
    if (st == BK_OK && want_prof) {
        std::vector<long long> pr(PROF_ITERS * PROF_MARKS);
        cudaMemcpy(pr.data(), dprof, pr.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        double acc[8] = {};
        int cnt = 0;
        for (int i = 1; i < PROF_ITERS; ++i) {
            const long long* r = pr.data() + i * PROF_MARKS;
            if (!r[0] || !r[7]) continue;
            for (int k = 1; k < 8; ++k) acc[k] += (double)(r[k] - r[k - 1]);
            ++cnt;
        }
        if (cnt)
            fprintf(stderr,
                    "[bk_cg_profile batched K=%d cpc=%d res=%d chip 0] per-iteration ns: phase1 %.0f | "
                    "reduceG %.0f | solve_a %.0f | phase2 %.0f | reduceS %.0f | control+solve_b %.0f | "
                    "phase3+sync %.0f\n",
                    K, cpc, (int)resident, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt,
                    acc[5] / cnt, acc[6] / cnt, acc[7] / cnt);
    }
    return st;
}

bk_status block_cg_device_multi(bk_ctx* ctx, const bk_operator* op, int K, const double* B, int S,
                                const bk_solver_cfg* cfg, double* X, CgReport* reps) {
    if (K < 1 || op->n % K) return fail(ctx, BK_INTERNAL, "block_cg_multi: bad chip count");
    if (S == 8) return run_dmma_multi<8>(ctx, op, K, B, cfg, X, reps);
    if (S == 16) return run_dmma_multi<16>(ctx, op, K, B, cfg, X, reps);
    if (S == 32) return run_dmma_multi<32>(ctx, op, K, B, cfg, X, reps);
    return fail(ctx, BK_INTERNAL, "block_cg_multi: kernel width must be 8, 16 or 32");
}

bk_status block_cg_device(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                          const bk_solver_cfg* cfg, double* X, CgReport* rep) {
    // wide blocks or large grids: one kernel per phase (HBM-bound phases of
    // milliseconds make launch / host-control costs negligible)
    const bool large = s > 32 || (op->n >= (int64_t)1 << 21 && s > 16);
    if (ctx->knobs.force_large || large) return block_cg_large(ctx, op, B, s, cfg, X, rep);
    if (s <= 8) return run_dmma<8>(ctx, op, B, s, cfg, X, rep);
    if (s <= 16) return run_dmma<16>(ctx, op, B, s, cfg, X, rep);
    return run_dmma<32>(ctx, op, B, s, cfg, X, rep);
}

}  // namespace bk

// ---------------------------------------------------------------------------
// debug harness: cycles of the s x s solve in isolation (scripts/ only)
// ---------------------------------------------------------------------------
namespace {
template <int S>
__global__ void __launch_bounds__(CtaShape<S>::BS, 1) small_solve_bench_kernel(int reps, long long* out,
                                                                             double* res) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Sm<S>& sm = *reinterpret_cast<Sm<S>*>(smem_raw);
    constexpr int BS = CtaShape<S>::BS;
    for (int e = threadIdx.x; e < S * S; e += BS) {
        const int i = e / S, j = e % S;
        // SPD with a wide diagonal scale spread, like G near convergence
        sm.mat[e] = (i == j ? 1.0 : 0.01 / (1 + i + j)) * exp(-0.5 * (i + j));
        sm.s_old[e] = (i == j ? 2.0 : 0.1) * exp(-0.25 * (i + j));
    }
    if (threadIdx.x < S) sm.act[threadIdx.x] = 1;
    __syncthreads();
    build_index<S>(sm);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) small_solve<S>(sm, sm.mat, sm.s_old, sm.coef);
    long long t1 = clock64();
    if (threadIdx.x == 0) g_ss_prof = out + 2;
    __syncthreads();
    if (threadIdx.x == 0) out[2 + 62] = clock64();
    small_solve<S, true>(sm, sm.mat, sm.s_old, sm.coef);
    __syncthreads();
    long long tv[8] = {};
    for (int v = 1; v <= 7; ++v) {
        __syncthreads();
        const long long a0 = clock64();
        for (int r = 0; r < 20; ++r) {
            if (v == 1) small_solve<S, false, 1>(sm, sm.mat, sm.s_old, sm.coef);
            if (v == 2) small_solve<S, false, 2>(sm, sm.mat, sm.s_old, sm.coef);
            if (v == 3) small_solve<S, false, 3>(sm, sm.mat, sm.s_old, sm.coef);
            if (v == 4) small_solve_t<S, BS, false, 0, 1>(sm, sm.mat, sm.s_old, sm.coef);
            if (v == 5) small_solve_t<S, BS, false, 0, 2>(sm, sm.mat, sm.s_old, sm.coef);
            if (v == 6) small_solve_t<S, BS, false, 0, 4>(sm, sm.mat, sm.s_old, sm.coef);
            if (v == 7 && BS >= 256) small_solve_t<S, BS, false, 0, 8>(sm, sm.mat, sm.s_old, sm.coef);
        }
        tv[v] = (clock64() - a0) / 20;
    }
    if (threadIdx.x == 0)
        for (int v = 1; v <= 7; ++v) out[69 + v] = tv[v];
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / reps;
        out[1] = sm.rank;
    }
    for (int e = threadIdx.x; e < S * S; e += BS) res[e] = sm.coef[(e / S) * Strides<S>::RS + e % S];
}
}  // namespace

extern "C" int bk_debug_small_solve_cycles(int s, int reps, long long* cycles, int* rank,
                                           double* coef) {
    long long* d;
    double* r;
    cudaMalloc(&d, 80 * 8);
    cudaMemset(d, 0, 80 * 8);
    cudaMalloc(&r, 64 * 64 * 8);
    int err = 0;
    auto run = [&](auto kern, size_t smem, int bs) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<1, bs, smem>>>(reps, d, r);
        err = (int)cudaDeviceSynchronize();
    };
    if (s == 8) run(small_solve_bench_kernel<8>, sizeof(Sm<8>), CtaShape<8>::BS);
    else if (s == 16) run(small_solve_bench_kernel<16>, sizeof(Sm<16>), CtaShape<16>::BS);
    else run(small_solve_bench_kernel<32>, sizeof(Sm<32>), CtaShape<32>::BS);
    long long h[80] = {0};
    cudaMemcpy(h, d, 80 * 8, cudaMemcpyDeviceToHost);
    fprintf(stderr, "small_solve<%d> stamps (cycles from start): setup %lld, first search %lld;", s,
            h[2] - h[64], h[3] - h[64]);
    for (int k = 1; k <= s; ++k) fprintf(stderr, " %lld", h[4 + k] ? h[4 + k] - h[64] : -1);
    fprintf(stderr, "; end %lld | variants: no-update %lld, fixed-order %lld, no-barrier %lld, "
            "warps 1/2/4/8: %lld %lld %lld %lld\n",
            h[65] - h[64], h[70], h[71], h[72], h[73], h[74], h[75], h[76]);
    cudaMemcpy(coef, r, (size_t)s * s * 8, cudaMemcpyDeviceToHost);
    *cycles = h[0];
    *rank = (int)h[1];
    cudaFree(d);
    cudaFree(r);
    return err;
}
