// Block CG for large slabs — one kernel per phase, host-driven control.
//
// Used for wide blocks (S = 64, BASELINE config 5: 4.2 M cells) where each
// iteration streams ~21.6 GB through HBM, so launch and host round-trip costs
// (~20 us) are noise against the ~4 ms phases, and as the per-rank engine of
// the y-slab domain decomposition (bk_dd_*, halo rows and Gram all-reduces are
// inserted between the phases by the caller's communicator hooks).
//
// Vectors live in a slab-local layout with one ghost row on each y side:
// cell (ix, iyl, iz), iyl in [0, nyl + 2), at l = ix + nx (iyl + (nyl + 2) iz),
// row-major [l][S]; interior rows are iyl = 1 .. nyl (global rows y0 ..
// y0 + nyl - 1). Stencil coefficients are read from the GLOBAL operator by
// global index, so every rank's operator is bitwise the single-GPU one.
//
// Same algorithm as block_cg (solvers.cpp:452-665) and the persistent kernels:
// W = A P and G = P^T W (phase 1), alpha = G^+ S_old, X += P alpha,
// R -= W alpha, rr, S_new = R^T D^-1 R (phase 2), per-column verify / freeze /
// restart, beta = S_old^+ S_new, P = D^-1 R + P beta (phase 3). Dense s x s
// products run on mma.sync.m16n8k4.f64; Gram partials are fixed-order per
// CTA and reduced in CTA order (deterministic).
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "bk_common.cuh"
#include "bk_small_solve.cuh"

namespace {

using namespace bkcg;

constexpr int LBS = 256;      // sweep kernels: 8 warps
constexpr int LNW = LBS / 32;
constexpr int CBS = 512;      // control kernels (s x s solves)

struct Slab {
    int nx, nyl, nz, ny, y0;
    int64_t n_int;
};

__device__ __forceinline__ void dmma_l(double (&d)[4], double a0, double a1, double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b));
}

// interior cell u -> local flat l, global flat gi and the stencil
struct LCell {
    int64_t l, gi;
    double d, xm, xp, ym, yp, zm, zp;  // CSR values (-conductance off the diagonal)
    bool hxm, hxp, hym, hyp, hzm, hzp;
};

struct StencilPtr {
    const double* diag;
    const double* cx;
    const double* cy;
    const double* cz;
    const double* dinv;
};

__device__ __forceinline__ void lcell(const Slab& sl, const StencilPtr& st, int64_t u, LCell& c,
                                      bool coefs) {
    const int ix = (int)(u % sl.nx);
    const int64_t q = u / sl.nx;
    const int iyl = 1 + (int)(q % sl.nyl);
    const int iz = (int)(q / sl.nyl);
    const int iyg = sl.y0 + iyl - 1;
    c.l = ix + (int64_t)sl.nx * (iyl + (int64_t)(sl.nyl + 2) * iz);
    c.gi = ix + (int64_t)sl.nx * (iyg + (int64_t)sl.ny * iz);
    c.hxm = ix > 0;
    c.hxp = ix < sl.nx - 1;
    c.hym = iyg > 0;
    c.hyp = iyg < sl.ny - 1;
    c.hzm = iz > 0;
    c.hzp = iz < sl.nz - 1;
    if (coefs) {
        const int64_t plane = (int64_t)sl.nx * sl.ny;
        c.d = st.diag[c.gi];
        c.zm = c.hzm ? -st.cz[c.gi - plane] : 0.0;
        c.ym = c.hym ? -st.cy[c.gi - sl.nx] : 0.0;
        c.xm = c.hxm ? -st.cx[c.gi - 1] : 0.0;
        c.xp = c.hxp ? -st.cx[c.gi] : 0.0;
        c.yp = c.hyp ? -st.cy[c.gi] : 0.0;
        c.zp = c.hzp ? -st.cz[c.gi] : 0.0;
    }
}

// ---------------------------------------------------------------------------
// sweep geometry
//
// A tile is a run of 16 consecutive x cells at fixed (y, z); tiles are walked
// z-fastest (tile T: iz = T % nz, then x-run, then y), so the z +- 1
// neighbours of a tile are the adjacent tiles processed by the same or the
// neighbouring CTA in the same wave and the stencil reads P from HBM once.
//
// All 8 warps of a CTA work on the same TPB = 8 / (S / 8) tiles: warp w owns
// tile slot ts = w / (S / 8) and the 8-column block cb = w % (S / 8). The
// DMMA B fragments of alpha / beta (column block cb, all K) stay in registers
// for the whole sweep, the A operand rows (P, W of the tile group) are staged
// in shared memory by cp.async one group ahead, and the Gram G = U^T V of the
// group is accumulated by warp-owned 16 x 8 output tiles.
// ---------------------------------------------------------------------------
template <int S>
struct Geo {
    static constexpr int RS = S + 4;           // smem row stride (doubles)
    static constexpr int NWC = S / 8;          // warps per tile
    static constexpr int TPB = LNW / NWC;      // tiles per CTA step
    static constexpr int CELLS = 16 * TPB;
    static constexpr int TILE = CELLS * RS;    // doubles per staged block
    static constexpr int MT = (S + 15) / 16, NT = S / 8, GT = MT * NT;
    static constexpr int PER = (GT + LNW - 1) / LNW;
};

__host__ __device__ __forceinline__ int n_tiles(const Slab& sl) {
    return ((sl.nx + 15) / 16) * sl.nyl * sl.nz;
}

struct TileCells {
    int64_t l0, g0;  // slab-local / global flat index of cell 0 of the run
    int ix0, iyg, iz, nv;
};

__device__ __forceinline__ void tile_cells(const Slab& sl, int T, int ntiles, TileCells& tc) {
    if (T >= ntiles) {
        tc.l0 = tc.g0 = 0;
        tc.ix0 = tc.iyg = tc.iz = 0;
        tc.nv = 0;
        return;
    }
    const int ntx = (sl.nx + 15) / 16;
    tc.iz = T % sl.nz;
    const int q = T / sl.nz;
    tc.ix0 = 16 * (q % ntx);
    const int iyl = 1 + q / ntx;
    tc.iyg = sl.y0 + iyl - 1;
    tc.l0 = tc.ix0 + (int64_t)sl.nx * (iyl + (int64_t)(sl.nyl + 2) * tc.iz);
    tc.g0 = tc.ix0 + (int64_t)sl.nx * (tc.iyg + (int64_t)sl.ny * tc.iz);
    tc.nv = sl.nx - tc.ix0 < 16 ? sl.nx - tc.ix0 : 16;
}

// stencil of cell r of a run (CSR values: -conductance off the diagonal)
__device__ __forceinline__ void run_cell(const Slab& sl, const StencilPtr& st, const TileCells& tc,
                                         int r, LCell& c) {
    const int ix = tc.ix0 + r;
    c.l = tc.l0 + r;
    c.gi = tc.g0 + r;
    c.hxm = ix > 0;
    c.hxp = ix < sl.nx - 1;
    c.hym = tc.iyg > 0;
    c.hyp = tc.iyg < sl.ny - 1;
    c.hzm = tc.iz > 0;
    c.hzp = tc.iz < sl.nz - 1;
    const int64_t plane = (int64_t)sl.nx * sl.ny;
    c.d = st.diag[c.gi];
    c.zm = c.hzm ? -st.cz[c.gi - plane] : 0.0;
    c.ym = c.hym ? -st.cy[c.gi - sl.nx] : 0.0;
    c.xm = c.hxm ? -st.cx[c.gi - 1] : 0.0;
    c.xp = c.hxp ? -st.cx[c.gi] : 0.0;
    c.yp = c.hyp ? -st.cy[c.gi] : 0.0;
    c.zp = c.hzp ? -st.cz[c.gi] : 0.0;
}

__device__ __forceinline__ void cp16(double* smem, const double* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// stage NA row arrays of group `grp` (dst + a * TILE, a = 0 .. NA-1) plus,
// when dinv != nullptr, D^-1 of its cells into dst + NA * TILE; the tile
// geometry is computed once per chunk row and shared by all arrays
template <int S, int NA>
__device__ __forceinline__ void stage_multi(double* dst, const double* const (&src)[NA],
                                            const double* __restrict__ dinv, const Slab& sl,
                                            int grp, int ntiles) {
    using G_ = Geo<S>;
    constexpr int CPR = S / 2;
    constexpr int TOT = G_::CELLS * CPR;
    static_assert(TOT % LBS == 0, "chunk count");
#pragma unroll
    for (int e0 = 0; e0 < TOT; e0 += LBS) {
        const int e = e0 + threadIdx.x;
        const int row = e / CPR, ch = e % CPR, r = row % 16;
        TileCells tc;
        tile_cells(sl, grp * G_::TPB + row / 16, ntiles, tc);
        double* d = dst + row * G_::RS + 2 * ch;
        if (r < tc.nv) {
#pragma unroll
            for (int q = 0; q < NA; ++q) cp16(d + q * G_::TILE, src[q] + (tc.l0 + r) * S + 2 * ch);
            if (dinv && ch == 0) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + NA * G_::TILE + row);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa),
                             "l"(dinv + tc.g0 + r)
                             : "memory");
            }
        } else {
#pragma unroll
            for (int q = 0; q < NA; ++q)
                *reinterpret_cast<double2*>(d + q * G_::TILE) = make_double2(0.0, 0.0);
            if (ch == 0) dst[NA * G_::TILE + row] = 1.0;
        }
    }
}

// CTA Gram over a staged group: warp w owns output tiles w, w + LNW, ... of
// G = U^T V (MT x NT grid of 16 x 8 tiles) and accumulates over all cells
template <int S>
struct OwnedGram {
    using G_ = Geo<S>;
    double d[G_::PER][4];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < G_::PER; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) d[i][e] = 0.0;
    }
    __device__ __forceinline__ void accumulate(const double* U, const double* V, int warp, int g,
                                               int t) {
        constexpr int RS = G_::RS;
#pragma unroll 4
        for (int kk = 0; kk < G_::CELLS / 4; ++kk) {
            const int c4 = 4 * kk + t;
#pragma unroll
            for (int i = 0; i < G_::PER; ++i) {
                const int tile = warp + LNW * i;
                if (tile >= G_::GT) break;
                const int m = tile / G_::NT, n = tile % G_::NT;
                if (8 * n + 7 < 16 * m) continue;  // below the diagonal: never read
                const double a0 = U[c4 * RS + 16 * m + g];
                const double a1 = (16 * m + 8 + g < S) ? U[c4 * RS + 16 * m + 8 + g] : 0.0;
                dmma_l(d[i], a0, a1, V[c4 * RS + 8 * n + g]);
            }
        }
    }
    // this CTA's partial: out[r * S + c]
    __device__ __forceinline__ void write(double* out, int warp, int g, int t) const {
#pragma unroll
        for (int i = 0; i < G_::PER; ++i) {
            const int tile = warp + LNW * i;
            if (tile >= G_::GT) break;
            const int m = tile / G_::NT, n = tile % G_::NT;
            const int r0 = 16 * m + g, c0 = 8 * n + 2 * t;
            out[r0 * S + c0] = d[i][0];
            out[r0 * S + c0 + 1] = d[i][1];
            if (r0 + 8 < S) {
                out[(r0 + 8) * S + c0] = d[i][2];
                out[(r0 + 8) * S + c0 + 1] = d[i][3];
            }
        }
    }
};

struct SweepArgs {
    Slab sl;
    StencilPtr st;
    const double* B;
    double* X;
    double* R;
    double* P;
    double* W;
    double* part;        // [gridDim.x][E]
    const double* coef;  // S x (S + 4) (alpha or beta)
    const double* coef2; // alpha kept for the deferred X update (k_pupdate modes 1, 2)
    const int* act;      // per-column mask for masked sweeps
    const int* gate;     // P updates inside the device-driven loop: run only if *gate == 0
    const double* pcoef; // S = 64 stencil sweep: per-run packed coefficients (k_pack_coef64)
    int precond;
};

// C-fragment rows (cells g, g + 8 of the run; columns col, col + 1)
__device__ __forceinline__ void ld_frag(const double* V, int S, const TileCells& tc, int g,
                                        int col, bool v0, bool v1, double (&o)[4]) {
    const double2 a = v0 ? *reinterpret_cast<const double2*>(V + (tc.l0 + g) * S + col)
                         : make_double2(0.0, 0.0);
    const double2 b = v1 ? *reinterpret_cast<const double2*>(V + (tc.l0 + g + 8) * S + col)
                         : make_double2(0.0, 0.0);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = b.x;
    o[3] = b.y;
}
__device__ __forceinline__ void st_frag(double* V, int S, const TileCells& tc, int g, int col,
                                        bool v0, bool v1, const double (&o)[4]) {
    if (v0) *reinterpret_cast<double2*>(V + (tc.l0 + g) * S + col) = make_double2(o[0], o[1]);
    if (v1) *reinterpret_cast<double2*>(V + (tc.l0 + g + 8) * S + col) = make_double2(o[2], o[3]);
}
__device__ __forceinline__ void stage_frag(double* U, int RS, int row0, int col,
                                           const double (&o)[4]) {
    *reinterpret_cast<double2*>(U + row0 * RS + col) = make_double2(o[0], o[1]);
    *reinterpret_cast<double2*>(U + (row0 + 8) * RS + col) = make_double2(o[2], o[3]);
}

// per-column vector partial (sum over the group slots in order) -> out[S*S + c]
template <int S>
__device__ __forceinline__ void write_colsum(double* out, double* vred, int ts, int cb, int lane,
                                             double s0, double s1) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        double x = e ? s1 : s0;
        x += __shfl_xor_sync(0xffffffffu, x, 4);
        x += __shfl_xor_sync(0xffffffffu, x, 8);
        x += __shfl_xor_sync(0xffffffffu, x, 16);
        if (lane < 4) vred[ts * S + 8 * cb + 2 * lane + e] = x;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < S; c += LBS) {
        double s = 0.0;
        for (int q = 0; q < Geo<S>::TPB; ++q) s += vred[q * S + c];
        out[S * S + c] = s;
    }
}

// stages in flight for the update sweep: 3 (two groups ahead) when two CTAs
// still fit an SM, else 2
// XD: X += P alpha deferred to k_pupdate — the stage holds W, R, D^-1 and a Z
// scratch tile instead of P, W, X, R, D^-1
template <int S, bool XD = false>
struct UpdRing {
    static constexpr size_t stage =
        ((XD ? 3 : 4) * (size_t)Geo<S>::TILE + Geo<S>::CELLS) * sizeof(double);
    static constexpr int NST = (2 * (3 * stage + Geo<S>::TPB * S * 8 + 1024) <= 228 * 1024) ? 3 : 2;
};
template <int S, bool XD = false>
constexpr size_t smem_update() {
    return UpdRing<S, XD>::NST * UpdRing<S, XD>::stage + Geo<S>::TPB * S * sizeof(double);
}
template <int S>
constexpr size_t smem_anchor() {
    return (2 * (size_t)Geo<S>::TILE + Geo<S>::TPB * S) * sizeof(double);
}
template <int S>
constexpr size_t smem_spmm() {
    return 2 * (size_t)Geo<S>::TILE * sizeof(double);
}
// k_pupdate MODE 0: P = Z + P beta; 1: and X += P alpha (deferred); 2: X += P alpha only
template <int S, int MODE = 0>
constexpr size_t smem_pupdate() {
    return 3 * ((MODE == 1 ? 3 : 2) * (size_t)Geo<S>::TILE + Geo<S>::CELLS) * sizeof(double);
}

// ---------------------------------------------------------------------------
// sweeps
// ---------------------------------------------------------------------------
enum Sweep : int { kInit = 0, kRestart = 1 };

// X = 0, R = B (init) or R = B - A X (restart); Z = D^-1 R; P = Z;
// partials [R^T Z | sum r^2]
template <int S, int MODE>
__global__ void __launch_bounds__(LBS, 2) k_anchor(SweepArgs a) {
    using G_ = Geo<S>;
    constexpr int RS = G_::RS;
    extern __shared__ __align__(16) double sm_[];
    double* U = sm_;
    double* V = U + G_::TILE;
    double* vred = V + G_::TILE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ts = warp / G_::NWC, cb = warp % G_::NWC, col = 8 * cb + 2 * t;
    const int ntiles = n_tiles(a.sl);
    const int ngroups = (ntiles + G_::TPB - 1) / G_::TPB;
    const int64_t pz = (int64_t)a.sl.nx * (a.sl.nyl + 2);
    const bool jac = a.precond != 0;
    OwnedGram<S> G;
    G.zero();
    double bn0 = 0.0, bn1 = 0.0;
    for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        TileCells tc;
        tile_cells(a.sl, grp * G_::TPB + ts, ntiles, tc);
        const bool v0 = g < tc.nv, v1 = g + 8 < tc.nv;
        double r[4], z[4];
        ld_frag(a.B, S, tc, g, col, v0, v1, r);
        if (MODE == kRestart) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (!(h ? v1 : v0)) continue;
                LCell c;
                run_cell(a.sl, a.st, tc, g + 8 * h, c);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t ee = c.l * S + col + e;
                    double acc = 0.0;
                    if (c.hzm) acc = fma(c.zm, a.X[ee - pz * S], acc);
                    if (c.hym) acc = fma(c.ym, a.X[ee - (int64_t)a.sl.nx * S], acc);
                    if (c.hxm) acc = fma(c.xm, a.X[ee - S], acc);
                    acc = fma(c.d, a.X[ee], acc);
                    if (c.hxp) acc = fma(c.xp, a.X[ee + S], acc);
                    if (c.hyp) acc = fma(c.yp, a.X[ee + (int64_t)a.sl.nx * S], acc);
                    if (c.hzp) acc = fma(c.zp, a.X[ee + pz * S], acc);
                    r[2 * h + e] -= acc;
                }
            }
        }
        const double d0 = (jac && v0) ? a.st.dinv[tc.g0 + g] : 1.0;
        const double d1 = (jac && v1) ? a.st.dinv[tc.g0 + g + 8] : 1.0;
        z[0] = d0 * r[0];
        z[1] = d0 * r[1];
        z[2] = d1 * r[2];
        z[3] = d1 * r[3];
        bn0 += r[0] * r[0] + r[2] * r[2];
        bn1 += r[1] * r[1] + r[3] * r[3];
        if (MODE == kInit) {
            const double zero[4] = {0.0, 0.0, 0.0, 0.0};
            st_frag(a.X, S, tc, g, col, v0, v1, zero);
        }
        st_frag(a.R, S, tc, g, col, v0, v1, r);
        st_frag(a.P, S, tc, g, col, v0, v1, z);
        stage_frag(U, RS, ts * 16 + g, col, r);
        stage_frag(V, RS, ts * 16 + g, col, z);
        __syncthreads();
        G.accumulate(U, V, warp, g, t);
        __syncthreads();
    }
    double* out = a.part + (int64_t)blockIdx.x * (S * S + S);
    G.write(out, warp, g, t);
    write_colsum<S>(out, vred, ts, cb, lane, bn0, bn1);
}

// phase 1: W = A P (CSR-order FMA chain) over interior cells; partial G = P^T W.
// Lane mapping: LPC lanes per cell, each lane 4 columns as two 16-byte pieces
// half a row apart, so one load instruction reads whole 128-byte lines.
template <int S>
__global__ void __launch_bounds__(LBS, 2) k_spmm_gram(SweepArgs a) {
    if (a.gate && *a.gate != 0) return;  // gated (DD lookahead): this iteration is a no-op
    using G_ = Geo<S>;
    constexpr int RS = G_::RS, LPC = 16 / G_::TPB, CPW = 32 / LPC;
    extern __shared__ __align__(16) double sm_[];
    double* U = sm_;
    double* V = U + G_::TILE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int cell = warp * CPW + lane / LPC, slot = cell / 16, r = cell % 16;
    const int ca = 2 * (lane % LPC), cb2 = ca + S / 2;
    const int ntiles = n_tiles(a.sl);
    const int ngroups = (ntiles + G_::TPB - 1) / G_::TPB;
    const int64_t pz = (int64_t)a.sl.nx * (a.sl.nyl + 2);
    OwnedGram<S> G;
    G.zero();
    for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        TileCells tc;
        tile_cells(a.sl, grp * G_::TPB + slot, ntiles, tc);
        double acc[4] = {0.0, 0.0, 0.0, 0.0}, ctr[4] = {0.0, 0.0, 0.0, 0.0};
        if (r < tc.nv) {
            LCell c;
            run_cell(a.sl, a.st, tc, r, c);
            auto row = [&](int64_t l, double cf, bool has) {
                if (!has) return;
                const double2 x0 = *reinterpret_cast<const double2*>(a.P + l * S + ca);
                const double2 x1 = *reinterpret_cast<const double2*>(a.P + l * S + cb2);
                acc[0] = fma(cf, x0.x, acc[0]);
                acc[1] = fma(cf, x0.y, acc[1]);
                acc[2] = fma(cf, x1.x, acc[2]);
                acc[3] = fma(cf, x1.y, acc[3]);
            };
            row(c.l - pz, c.zm, c.hzm);
            row(c.l - a.sl.nx, c.ym, c.hym);
            row(c.l - 1, c.xm, c.hxm);
            {
                const double2 x0 = *reinterpret_cast<const double2*>(a.P + c.l * S + ca);
                const double2 x1 = *reinterpret_cast<const double2*>(a.P + c.l * S + cb2);
                ctr[0] = x0.x;
                ctr[1] = x0.y;
                ctr[2] = x1.x;
                ctr[3] = x1.y;
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] = fma(c.d, ctr[j], acc[j]);
            }
            row(c.l + 1, c.xp, c.hxp);
            row(c.l + a.sl.nx, c.yp, c.hyp);
            row(c.l + pz, c.zp, c.hzp);
            *reinterpret_cast<double2*>(a.W + c.l * S + ca) = make_double2(acc[0], acc[1]);
            *reinterpret_cast<double2*>(a.W + c.l * S + cb2) = make_double2(acc[2], acc[3]);
        }
        *reinterpret_cast<double2*>(U + cell * RS + ca) = make_double2(ctr[0], ctr[1]);
        *reinterpret_cast<double2*>(U + cell * RS + cb2) = make_double2(ctr[2], ctr[3]);
        *reinterpret_cast<double2*>(V + cell * RS + ca) = make_double2(acc[0], acc[1]);
        *reinterpret_cast<double2*>(V + cell * RS + cb2) = make_double2(acc[2], acc[3]);
        __syncthreads();
        G.accumulate(U, V, warp, g, t);
        __syncthreads();
    }
    G.write(a.part + (int64_t)blockIdx.x * (S * S), warp, g, t);
}

// ---------------------------------------------------------------------------
// phase 1 for S = 64 with TMA bulk copies (even nx): per 16-cell run, one
// thread issues cp.async.bulk copies of the centre run with its x-halo, the
// y-1 / y+1 / z-1 / z+1 runs and the stencil coefficients into a 2-stage
// shared-memory ring (mbarrier completion); the stencil then reads shared
// memory only. A few bulk instructions per group instead of thousands of
// 16-byte copies, and the loads of group g+1 overlap the sweep of group g.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tMBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MBW_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

struct TmaStage64 {
    static constexpr int S = 64;
    static constexpr int ROWS = 82;       // centre (x-halo) 18 + 4 runs x 16
    static constexpr int ROWD = S;        // dense rows
    static constexpr int COEF = 6 * 24;   // 6 coefficient runs (<= 18 values, padded)
    static constexpr int DOUBLES = ROWS * ROWD + COEF;
};

// issue the copies of group `grp` (one tile, TPB = 1) into stage `st`
__device__ __forceinline__ void tma_stage64(double* st, unsigned long long* bar, const SweepArgs& a,
                                            int grp, int ntiles) {
    constexpr int S = 64;
    TileCells tc;
    tile_cells(a.sl, grp, ntiles, tc);
    const int nx = a.sl.nx, nv = tc.nv;
    const int64_t pz = (int64_t)nx * (a.sl.nyl + 2);
    const int64_t plane = (int64_t)nx * a.sl.ny;
    const unsigned rowb = S * 8;
    // centre run with halo: cells max(ix0-1, 0) .. min(ix0+nv, nx-1)
    const int lo = tc.ix0 > 0 ? -1 : 0;
    const int hi = tc.ix0 + nv < nx ? nv : nv - 1;  // inclusive, relative to ix0
    unsigned total = (unsigned)(hi - lo + 1) * rowb + 2 * nv * rowb;
    const bool zm = tc.iz > 0, zp = tc.iz < a.sl.nz - 1;
    if (zm) total += nv * rowb;
    if (zp) total += nv * rowb;
    double* coef = st + TmaStage64::ROWS * TmaStage64::ROWD;
    // coefficient runs (16-byte aligned sources): diag[g0..+16), cx[g0-2..+18),
    // cy[g0-nx..+16), cy[g0..+16), cz[g0-plane..+16), cz[g0..+16)
    const int64_t g0 = tc.g0;
    const bool ym = tc.iyg > 0;
    total += 16 * 8 + 18 * 8 + 16 * 8 + 16 * 8;  // diag, cx, cy(y-) , cy(y+)
    if (zm) total += 16 * 8;
    total += 16 * 8;  // cz(z+) run always readable (last plane: value unused)
    mbar_expect_tx(bar, total);
    bulk_g2s(st + (1 + lo) * S, a.P + (tc.l0 + lo) * S, (unsigned)(hi - lo + 1) * rowb, bar);
    bulk_g2s(st + 18 * S, a.P + (tc.l0 - nx) * S, nv * rowb, bar);
    bulk_g2s(st + 34 * S, a.P + (tc.l0 + nx) * S, nv * rowb, bar);
    if (zm) bulk_g2s(st + 50 * S, a.P + (tc.l0 - pz) * S, nv * rowb, bar);
    if (zp) bulk_g2s(st + 66 * S, a.P + (tc.l0 + pz) * S, nv * rowb, bar);
    bulk_g2s(coef, a.st.diag + g0, 16 * 8, bar);
    bulk_g2s(coef + 24, a.st.cx + g0 - 2 + (tc.ix0 == 0 && g0 < 2 ? 2 : 0), 18 * 8, bar);
    bulk_g2s(coef + 48, a.st.cy + (ym ? g0 - nx : g0), 16 * 8, bar);
    bulk_g2s(coef + 72, a.st.cy + g0, 16 * 8, bar);
    if (zm) bulk_g2s(coef + 96, a.st.cz + g0 - plane, 16 * 8, bar);
    bulk_g2s(coef + 120, a.st.cz + g0, 16 * 8, bar);
}

__global__ void __launch_bounds__(LBS, 2) k_spmm_gram_tma64(SweepArgs a) {
    if (a.gate && *a.gate != 0) return;  // gated (DD lookahead): this iteration is a no-op
    constexpr int S = 64;
    using G_ = Geo<S>;
    constexpr int RS = G_::RS, LPC = 16, CPW = 2;
    extern __shared__ __align__(128) double sm_[];
    __shared__ __align__(8) unsigned long long bars[2];
    double* U = sm_ + 2 * TmaStage64::DOUBLES;
    double* V = U + G_::TILE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int r = warp * CPW + lane / LPC;  // cell of the run
    const int ca = 2 * (lane % LPC), cb2 = ca + S / 2;
    const int ntiles = n_tiles(a.sl);
    const int ngroups = ntiles;  // TPB = 1
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    OwnedGram<S> G;
    G.zero();
    int grp = blockIdx.x;
    if (threadIdx.x == 0 && grp < ngroups) tma_stage64(sm_, &bars[0], a, grp, ntiles);
    for (int it = 0; grp < ngroups; grp += gridDim.x, ++it) {
        const int nxt = grp + gridDim.x;
        if (threadIdx.x == 0 && nxt < ngroups) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_stage64(sm_ + ((it + 1) & 1) * TmaStage64::DOUBLES, &bars[(it + 1) & 1], a, nxt,
                        ntiles);
        }
        TileCells tc;
        tile_cells(a.sl, grp, ntiles, tc);
        mbar_wait(&bars[it & 1], (unsigned)((it >> 1) & 1));
        const double* rows = sm_ + (it & 1) * TmaStage64::DOUBLES;
        const double* cf = rows + TmaStage64::ROWS * TmaStage64::ROWD;
        double acc[4] = {0.0, 0.0, 0.0, 0.0}, ctr[4] = {0.0, 0.0, 0.0, 0.0};
        if (r < tc.nv) {
            const int ix = tc.ix0 + r;
            auto row = [&](int rr, double c, bool has) {
                if (!has) return;
                const double2 x0 = *reinterpret_cast<const double2*>(rows + rr * S + ca);
                const double2 x1 = *reinterpret_cast<const double2*>(rows + rr * S + cb2);
                acc[0] = fma(c, x0.x, acc[0]);
                acc[1] = fma(c, x0.y, acc[1]);
                acc[2] = fma(c, x1.x, acc[2]);
                acc[3] = fma(c, x1.y, acc[3]);
            };
            const int xo = (tc.ix0 == 0 && tc.g0 < 2) ? 2 : 0;  // cx run start shift
            // CSR order z-, y-, x-, diag, x+, y+, z+ (values = -conductance)
            row(50 + r, -cf[96 + r], tc.iz > 0);
            row(18 + r, -cf[48 + r], tc.iyg > 0);
            row(r, -cf[24 + 1 + r - xo], ix > 0);
            {
                const double2 x0 = *reinterpret_cast<const double2*>(rows + (r + 1) * S + ca);
                const double2 x1 = *reinterpret_cast<const double2*>(rows + (r + 1) * S + cb2);
                ctr[0] = x0.x;
                ctr[1] = x0.y;
                ctr[2] = x1.x;
                ctr[3] = x1.y;
                const double d = cf[r];
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] = fma(d, ctr[j], acc[j]);
            }
            row(r + 2, -cf[24 + 2 + r - xo], ix < a.sl.nx - 1);
            row(34 + r, -cf[72 + r], tc.iyg < a.sl.ny - 1);
            row(66 + r, -cf[120 + r], tc.iz < a.sl.nz - 1);
            const int64_t l = tc.l0 + r;
            *reinterpret_cast<double2*>(a.W + l * S + ca) = make_double2(acc[0], acc[1]);
            *reinterpret_cast<double2*>(a.W + l * S + cb2) = make_double2(acc[2], acc[3]);
        }
        *reinterpret_cast<double2*>(U + r * RS + ca) = make_double2(ctr[0], ctr[1]);
        *reinterpret_cast<double2*>(U + r * RS + cb2) = make_double2(ctr[2], ctr[3]);
        *reinterpret_cast<double2*>(V + r * RS + ca) = make_double2(acc[0], acc[1]);
        *reinterpret_cast<double2*>(V + r * RS + cb2) = make_double2(acc[2], acc[3]);
        __syncthreads();
        G.accumulate(U, V, warp, g, t);
        __syncthreads();
    }
    G.write(a.part + (int64_t)blockIdx.x * (S * S), warp, g, t);
}

constexpr size_t smem_spmm_tma64() {
    return (2 * (size_t)TmaStage64::DOUBLES + 2 * (size_t)Geo<64>::TILE) * sizeof(double);
}

__device__ __forceinline__ void frag_from_smem(const double* T, int RS, int row0, int col,
                                               double (&o)[4]) {
    const double2 a = *reinterpret_cast<const double2*>(T + row0 * RS + col);
    const double2 b = *reinterpret_cast<const double2*>(T + (row0 + 8) * RS + col);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = b.x;
    o[3] = b.y;
}

// phase 2: X += P alpha, R -= W alpha (DMMA, M = cells, B = alpha fragments in
// registers), rr, Z = D^-1 R; partials [R^T Z | rr]. Every input row of a
// tile group (P, W, X, R, D^-1) is staged by cp.async one group ahead; the
// updated R and Z overwrite the consumed R / X stage rows and feed the Gram.
template <int S, bool XD = false>
__global__ void __launch_bounds__(LBS, 2) k_update(SweepArgs a) {
    if (a.gate && *a.gate != 0) return;  // gated (DD lookahead): this iteration is a no-op
    using G_ = Geo<S>;
    constexpr int RS = G_::RS, KS = S / 4, TL = G_::TILE;
    // stage layout: P, W, X, R, dinv — or (XD) W, R, dinv, Z scratch
    constexpr int STAGE = (XD ? 3 : 4) * TL + G_::CELLS;
    constexpr int OW = XD ? 0 : TL, OR = XD ? TL : 3 * TL, OD = XD ? 2 * TL : 4 * TL;
    constexpr int OZ = XD ? 2 * TL + G_::CELLS : 2 * TL;
    constexpr int NST = UpdRing<S, XD>::NST;
    extern __shared__ __align__(16) double sm_[];
    double* vred = sm_ + NST * STAGE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ts = warp / G_::NWC, cb = warp % G_::NWC, col = 8 * cb + 2 * t;
    const int ntiles = n_tiles(a.sl);
    const int ngroups = (ntiles + G_::TPB - 1) / G_::TPB;
    const bool jac = a.precond != 0;
    double cf[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) cf[ks] = a.coef[(4 * ks + t) * RS + 8 * cb + g];
    OwnedGram<S> G;
    G.zero();
    double rr0 = 0.0, rr1 = 0.0;
    const double* const srcs4[4] = {a.P, a.W, a.X, a.R};
    const double* const srcs2[2] = {a.W, a.R};
    auto stage = [&](int buf, int gr) {
        if constexpr (XD)
            stage_multi<S, 2>(sm_ + buf * STAGE, srcs2, jac ? a.st.dinv : nullptr, a.sl, gr, ntiles);
        else
            stage_multi<S, 4>(sm_ + buf * STAGE, srcs4, jac ? a.st.dinv : nullptr, a.sl, gr, ntiles);
    };
    int grp = blockIdx.x;
#pragma unroll
    for (int p = 0; p < NST - 1; ++p) {
        if (grp + p * (int)gridDim.x < ngroups) stage(p, grp + p * gridDim.x);
        cp_commit();
    }
    for (int it = 0; grp < ngroups; grp += gridDim.x, ++it) {
        const int nxt = grp + (NST - 1) * gridDim.x;
        if (nxt < ngroups) stage((it + NST - 1) % NST, nxt);
        cp_commit();
        TileCells tc;
        tile_cells(a.sl, grp * G_::TPB + ts, ntiles, tc);
        const bool v0 = g < tc.nv, v1 = g + 8 < tc.nv;
        cp_wait<NST - 1>();
        __syncthreads();
        double* st = sm_ + (it % NST) * STAGE;
        const double* Pt = st + ts * 16 * RS;
        const double* Wt = st + OW + ts * 16 * RS;
        double* Xt = st + OZ;  // X (becomes V = Z after the update), or the Z scratch (XD)
        double* Rt = st + OR;  // becomes U (R)
        double x[4], rv[4];
        if constexpr (!XD) frag_from_smem(Xt, RS, ts * 16 + g, col, x);
        frag_from_smem(Rt, RS, ts * 16 + g, col, rv);
        const double d0 = jac ? st[OD + ts * 16 + g] : 1.0;
        const double d1 = jac ? st[OD + ts * 16 + g + 8] : 1.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int kc = 4 * ks + t;
            if constexpr (!XD) dmma_l(x, Pt[g * RS + kc], Pt[(g + 8) * RS + kc], cf[ks]);
            dmma_l(rv, -Wt[g * RS + kc], -Wt[(g + 8) * RS + kc], cf[ks]);
        }
        if constexpr (!XD) st_frag(a.X, S, tc, g, col, v0, v1, x);
        st_frag(a.R, S, tc, g, col, v0, v1, rv);
        double z[4];
        z[0] = d0 * rv[0];
        z[1] = d0 * rv[1];
        z[2] = d1 * rv[2];
        z[3] = d1 * rv[3];
        rr0 += rv[0] * rv[0] + rv[2] * rv[2];
        rr1 += rv[1] * rv[1] + rv[3] * rv[3];
        __syncthreads();  // all X / R fragments read before they are overwritten
        stage_frag(Rt, RS, ts * 16 + g, col, rv);
        stage_frag(Xt, RS, ts * 16 + g, col, z);
        __syncthreads();
        G.accumulate(Rt, Xt, warp, g, t);
        __syncthreads();
    }
    cp_wait<0>();
    double* out = a.part + (int64_t)blockIdx.x * (S * S + S);
    G.write(out, warp, g, t);
    write_colsum<S>(out, vred, ts, cb, lane, rr0, rr1);
}

// phase 3: P = D^-1 R + P beta (DMMA, accumulator initialised to Z; P, R and
// D^-1 rows of the group staged one group ahead)
template <int S, int MODE = 0>
__global__ void __launch_bounds__(LBS, 2) k_pupdate(SweepArgs a) {
    using G_ = Geo<S>;
    constexpr int RS = G_::RS, KS = S / 4, TL = G_::TILE;
    // MODE 0: P, R, dinv; 1: P, R, X, dinv; 2: P, X
    constexpr int NA = MODE == 1 ? 3 : 2;
    constexpr int STAGE = NA * TL + G_::CELLS;
    constexpr int OX = MODE == 1 ? 2 * TL : TL;
    constexpr int NST = 3;
    extern __shared__ __align__(16) double sm_[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ts = warp / G_::NWC, cb = warp % G_::NWC, col = 8 * cb + 2 * t;
    const int ntiles = n_tiles(a.sl);
    const int ngroups = (ntiles + G_::TPB - 1) / G_::TPB;
    const bool jac = a.precond != 0;
    if (a.gate && *a.gate != 0) return;  // graph loop: this iteration needs a verification
    double cf[KS], ca[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
        if (MODE != 2) cf[ks] = a.coef[(4 * ks + t) * RS + 8 * cb + g];    // beta
        if (MODE != 0) ca[ks] = a.coef2[(4 * ks + t) * RS + 8 * cb + g];   // alpha
    }
    const double* const srcs[2] = {a.P, MODE == 2 ? a.X : a.R};
    const double* const srcs3[3] = {a.P, a.R, a.X};
    auto stage = [&](int buf, int gr) {
        if constexpr (MODE == 1)
            stage_multi<S, 3>(sm_ + buf * STAGE, srcs3, jac ? a.st.dinv : nullptr, a.sl, gr, ntiles);
        else
            stage_multi<S, 2>(sm_ + buf * STAGE, srcs, (MODE == 0 && jac) ? a.st.dinv : nullptr,
                              a.sl, gr, ntiles);
    };
    int grp = blockIdx.x;
#pragma unroll
    for (int p = 0; p < NST - 1; ++p) {
        if (grp + p * (int)gridDim.x < ngroups) stage(p, grp + p * gridDim.x);
        cp_commit();
    }
    for (int it = 0; grp < ngroups; grp += gridDim.x, ++it) {
        const int nxt = grp + (NST - 1) * gridDim.x;
        if (nxt < ngroups) stage((it + NST - 1) % NST, nxt);
        cp_commit();
        TileCells tc;
        tile_cells(a.sl, grp * G_::TPB + ts, ntiles, tc);
        const bool v0 = g < tc.nv, v1 = g + 8 < tc.nv;
        cp_wait<NST - 1>();
        __syncthreads();
        const double* st = sm_ + (it % NST) * STAGE;
        const double* Pt = st + ts * 16 * RS;
        if constexpr (MODE != 0) {
            // X += P alpha (deferred from k_update; the same DMMA chain)
            double x[4];
            frag_from_smem(st + OX, RS, ts * 16 + g, col, x);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int kc = 4 * ks + t;
                dmma_l(x, Pt[g * RS + kc], Pt[(g + 8) * RS + kc], ca[ks]);
            }
            st_frag(a.X, S, tc, g, col, v0, v1, x);
        }
        if constexpr (MODE != 2) {
            double p[4];
            frag_from_smem(st + TL, RS, ts * 16 + g, col, p);
            const double d0 = jac ? st[NA * TL + ts * 16 + g] : 1.0;
            const double d1 = jac ? st[NA * TL + ts * 16 + g + 8] : 1.0;
            p[0] *= d0;
            p[1] *= d0;
            p[2] *= d1;
            p[3] *= d1;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int kc = 4 * ks + t;
                dmma_l(p, Pt[g * RS + kc], Pt[(g + 8) * RS + kc], cf[ks]);
            }
            st_frag(a.P, S, tc, g, col, v0, v1, p);
        }
        __syncthreads();  // buffer it % NST is refilled by the prefetch of the next iteration
    }
    cp_wait<0>();
}

template <int S, bool XD = false>
cudaError_t launch_update(const SweepArgs& a, int nb, cudaStream_t s) {
    const cudaError_t e = bk::set_max_smem((const void*)k_update<S, XD>, smem_update<S, XD>());
    if (e != cudaSuccess) return e;
    k_update<S, XD><<<nb, LBS, smem_update<S, XD>(), s>>>(a);
    return cudaGetLastError();
}

template <int S, int MODE = 0>
cudaError_t launch_pupdate(const SweepArgs& a, int nb, cudaStream_t s) {
    const cudaError_t e = bk::set_max_smem((const void*)k_pupdate<S, MODE>, smem_pupdate<S, MODE>());
    if (e != cudaSuccess) return e;
    k_pupdate<S, MODE><<<nb, LBS, smem_pupdate<S, MODE>(), s>>>(a);
    return cudaGetLastError();
}

#include "bk_sweep64.cuh"

// phase 1 launch: the TMA variant for S = 64 on grids whose x-runs are full
// (nx % 16 == 0), else the cp.async-free direct-load kernel
template <int S>
cudaError_t launch_spmm(const SweepArgs& a, int nb, cudaStream_t s, bool no_tma) {
    if constexpr (S == 64) {
        if (a.sl.nx % 16 == 0 && !no_tma) {
            const cudaError_t e = bk::set_max_smem((const void*)k_spmm_gram_tma64, smem_spmm_tma64());
            if (e != cudaSuccess) return e;
            k_spmm_gram_tma64<<<nb, LBS, smem_spmm_tma64(), s>>>(a);
            return cudaGetLastError();
        }
    }
    const cudaError_t e = bk::set_max_smem((const void*)k_spmm_gram<S>, smem_spmm<S>());
    if (e != cudaSuccess) return e;
    k_spmm_gram<S><<<nb, LBS, smem_spmm<S>(), s>>>(a);
    return cudaGetLastError();
}

// CTAs of the sweep kernels (2 per SM: register-bound), same for the
// single-GPU engine and every rank of the decomposition
constexpr int kSweepCtasPerSm = 2;
inline int sweep_ctas(const bk_ctx* ctx, const Slab& sl, int S) {
    const int tpb = LNW / (S / 8);
    const int groups = (n_tiles(sl) + tpb - 1) / tpb;
    int nb = ctx->num_sms * kSweepCtasPerSm;
    if (ctx->cg_max_ctas > 0 && nb > ctx->cg_max_ctas) nb = ctx->cg_max_ctas;
    if (nb > groups) nb = groups;
    return nb < 1 ? 1 : nb;
}

// true residual ||b - A x||^2 per column (CsrMatrix::apply order: mul, add)
template <int S>
__global__ void __launch_bounds__(LBS) k_true_res(SweepArgs a) {
    __shared__ double vred[LBS / S > 0 ? LBS / S : 1][S];
    const int j = threadIdx.x % S, cg = threadIdx.x / S, ncg = LBS / S;
    const int64_t pz = (int64_t)a.sl.nx * (a.sl.nyl + 2);
    double acc2 = 0.0;
    if (a.act[j]) {
        for (int64_t u = (int64_t)blockIdx.x * ncg + cg; u < a.sl.n_int;
             u += (int64_t)gridDim.x * ncg) {
            LCell c;
            lcell(a.sl, a.st, u, c, true);
            const int64_t e = c.l * S + j;
            double y = 0.0;
            if (c.hzm) y = __dadd_rn(y, __dmul_rn(c.zm, a.X[e - pz * S]));
            if (c.hym) y = __dadd_rn(y, __dmul_rn(c.ym, a.X[e - (int64_t)a.sl.nx * S]));
            if (c.hxm) y = __dadd_rn(y, __dmul_rn(c.xm, a.X[e - S]));
            y = __dadd_rn(y, __dmul_rn(c.d, a.X[e]));
            if (c.hxp) y = __dadd_rn(y, __dmul_rn(c.xp, a.X[e + S]));
            if (c.hyp) y = __dadd_rn(y, __dmul_rn(c.yp, a.X[e + (int64_t)a.sl.nx * S]));
            if (c.hzp) y = __dadd_rn(y, __dmul_rn(c.zp, a.X[e + pz * S]));
            const double rv = a.B[e] - y;
            acc2 += rv * rv;
        }
    }
    vred[cg][j] = acc2;
    __syncthreads();
    if (threadIdx.x < S) {
        double s = 0.0;
        for (int q = 0; q < ncg; ++q) s += vred[q][threadIdx.x];
        a.part[(int64_t)blockIdx.x * S + threadIdx.x] = s;
    }
}

// fixed-order reduction over CTAs: out[e] = sum_b part[b][e]; one warp per
// element (lane-strided partial sums, then a fixed shuffle tree)
__global__ void k_reduce(const double* __restrict__ part, int nb, int E, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int e = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (e >= E) return;
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += part[(int64_t)b * E + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[e] = s;
}

// global [n][S] <-> slab-local layout (interior rows), ghost rows zeroed on pack
template <int S>
__global__ void k_pack(Slab sl, double* __restrict__ glob, double* __restrict__ loc,
                       int to_local) {
    const int64_t total = sl.n_int * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = e / S;
        const int j = (int)(e % S);
        const int ix = (int)(u % sl.nx);
        const int64_t q = u / sl.nx;
        const int iyl = 1 + (int)(q % sl.nyl);
        const int iz = (int)(q / sl.nyl);
        const int64_t l = ix + (int64_t)sl.nx * (iyl + (int64_t)(sl.nyl + 2) * iz);
        const int64_t gi = ix + (int64_t)sl.nx * (sl.y0 + iyl - 1 + (int64_t)sl.ny * iz);
        if (to_local)
            loc[l * S + j] = glob[gi * S + j];
        else
            glob[gi * S + j] = loc[l * S + j];
    }
}

// ---------------------------------------------------------------------------
// control kernels: one CTA, state in device memory (identical logic to the
// persistent kernel's control section, solvers.cpp:468-661)
// ---------------------------------------------------------------------------
enum Cmd : int { kCmdPupdate = 0, kCmdVerify = 1, kCmdRestart = 2, kCmdDone = 3 };

template <int S>
struct Ctl {
    double s_old[S * S];
    double snew[S * S];
    double coef[S * (S + 4)];
    double akeep[S * (S + 4)];  // alpha of the iteration (X += P alpha is deferred to k_pupdate)
    double bnorm[S];
    double fres[S];
    double rr[S];
    int act[S];
    int conv[S];
    int vflag[S];
    int sa;
    int nver;
    int iters;
    int cmd;
    long long matvecs;
    double tol;
};

template <int S>
struct CSm {
    int idx[S];
    int sa;
    int rank;
    int fail;
    alignas(16) double aug[S * Strides<S>::LD + 2 * S];
    alignas(16) double m0[S * S];
    alignas(16) double m1[S * S];
    alignas(16) double out[S * Strides<S>::RS];
};

// compacted indices of the active columns, ascending (one warp: ballot +
// prefix popcount instead of a serial scan of the mask in global memory)
template <int S>
__device__ void ctl_index(Ctl<S>* c, CSm<S>& sm) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int base = 0;
#pragma unroll
        for (int q0 = 0; q0 < S; q0 += 32) {
            const int q = q0 + lane;
            const bool on = q < S && c->act[q];
            const unsigned m = __ballot_sync(0xffffffffu, on);
            if (on) sm.idx[base + __popc(m & ((1u << lane) - 1u))] = q;
            base += __popc(m);
        }
        if (lane == 0) {
            sm.sa = base;
            c->sa = base;
        }
    }
    __syncthreads();
}

// out (coef) = M^+ RHS on the active block
template <int S>
__device__ void ctl_solve(Ctl<S>* c, CSm<S>& sm, const double* M, const double* RHS) {
    for (int e = threadIdx.x; e < S * S; e += CBS) {
        sm.m0[e] = M[e];
        sm.m1[e] = RHS[e];
    }
    __syncthreads();
    if constexpr (S == 64)
        small_solve_reg<S, CBS>(sm, sm.m0, sm.m1, sm.out);
    else
        small_solve_t<S, CBS>(sm, sm.m0, sm.m1, sm.out);
    for (int e = threadIdx.x; e < S * (S + 4); e += CBS) c->coef[e] = sm.out[e];
    __syncthreads();
}

// red = [S_old | b^2]
template <int S>
__global__ void __launch_bounds__(CBS) k_ctl_init(Ctl<S>* c, const double* red, double tol) {
    extern __shared__ __align__(16) unsigned char smraw_[];
    CSm<S>& sm = *reinterpret_cast<CSm<S>*>(smraw_);
    if (threadIdx.x == 0) c->tol = tol;
    for (int e = threadIdx.x; e < S * S; e += CBS) c->s_old[e] = red[e];
    if (threadIdx.x < S) {
        const double bn = sqrt(red[S * S + threadIdx.x]);
        c->bnorm[threadIdx.x] = bn;
        c->act[threadIdx.x] = bn != 0.0;
        c->conv[threadIdx.x] = bn == 0.0;
        c->fres[threadIdx.x] = 0.0;
    }
    if (threadIdx.x == 0) {
        c->iters = 0;
        c->matvecs = 0;
        c->cmd = kCmdPupdate;
    }
    __syncthreads();
    ctl_index(c, sm);
}

// red = G: alpha = G^+ S_old
template <int S>
__global__ void __launch_bounds__(CBS) k_ctl_alpha(Ctl<S>* c, const double* red, int gated) {
    if (gated && c->cmd != kCmdPupdate) return;  // DD lookahead: a verification is pending
    extern __shared__ __align__(16) unsigned char smraw_[];
    CSm<S>& sm = *reinterpret_cast<CSm<S>*>(smraw_);
    ctl_index(c, sm);
    ctl_solve(c, sm, red, c->s_old);
    if (threadIdx.x == 0) c->matvecs += sm.sa;
    __syncthreads();
    for (int e = threadIdx.x; e < S * (S + 4); e += blockDim.x) c->akeep[e] = c->coef[e];
}

// red = [S_new | rr]: per-column recurrence test (solvers.cpp:582-590); beta
// (S_old^+ S_new) right away unless a true-residual verification is needed
template <int S>
// m <= 0: the device-driven loop (iteration = c->iters + 1, and the loop's
// while-condition is set to continue unless a verification is due or the
// iteration cap is reached)
__global__ void __launch_bounds__(CBS) k_ctl_update(Ctl<S>* c, const double* red, int m,
                                                    cudaGraphConditionalHandle loop, int max_iter,
                                                    int gated) {
    // DD lookahead: every thread reads cmd before thread 0 can rewrite it (the
    // write below follows at least one __syncthreads)
    if (gated && c->cmd != kCmdPupdate) return;
    extern __shared__ __align__(16) unsigned char smraw_[];
    CSm<S>& sm = *reinterpret_cast<CSm<S>*>(smraw_);
    __shared__ int nver;
    const bool graph = m <= 0;
    if (graph) m = c->iters + 1;
    for (int e = threadIdx.x; e < S * S; e += CBS) c->snew[e] = red[e];
    if (threadIdx.x < S) {
        const int q = threadIdx.x;
        c->rr[q] = red[S * S + q];
        c->vflag[q] = c->act[q] && (sqrt(red[S * S + q]) / c->bnorm[q] <= c->tol);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int k = 0;
        for (int q = 0; q < S; ++q) k += c->vflag[q];
        nver = k;
        c->nver = k;
        c->iters = m;
    }
    __syncthreads();
    if (nver > 0) {
        if (threadIdx.x == 0) {
            c->cmd = kCmdVerify;
            if (graph) cudaGraphSetConditional(loop, 0);
        }
        return;
    }
    ctl_index(c, sm);
    ctl_solve(c, sm, c->s_old, c->snew);  // beta
    for (int e = threadIdx.x; e < S * S; e += CBS) c->s_old[e] = c->snew[e];
    if (threadIdx.x == 0) {
        c->cmd = kCmdPupdate;
        if (graph) cudaGraphSetConditional(loop, m < max_iter ? 1u : 0u);
    }
}

// red = true ||b - A x||^2 of the flagged columns: freeze converged columns
// (active mask = compaction), restart on drift (solvers.cpp:582-634)
template <int S>
__global__ void __launch_bounds__(CBS) k_ctl_verify(Ctl<S>* c, const double* red) {
    extern __shared__ __align__(16) unsigned char smraw_[];
    CSm<S>& sm = *reinterpret_cast<CSm<S>*>(smraw_);
    __shared__ int restart;
    if (threadIdx.x == 0) {
        restart = 0;
        c->matvecs += c->nver;
        for (int q = 0; q < S; ++q) {
            if (!c->vflag[q]) continue;
            const double rt = sqrt(red[q]) / c->bnorm[q];
            if (rt <= c->tol) {
                c->act[q] = 0;
                c->conv[q] = 1;
                c->fres[q] = rt;
            } else {
                restart = 1;
            }
        }
    }
    __syncthreads();
    ctl_index(c, sm);
    if (sm.sa == 0) {
        if (threadIdx.x == 0) c->cmd = kCmdDone;
        return;
    }
    if (restart) {
        if (threadIdx.x == 0) c->cmd = kCmdRestart;
        return;
    }
    ctl_solve(c, sm, c->s_old, c->snew);  // beta on the compacted block
    for (int e = threadIdx.x; e < S * S; e += CBS) c->s_old[e] = c->snew[e];
    if (threadIdx.x == 0) c->cmd = kCmdPupdate;
}

// red = re-anchored S_old
template <int S>
__global__ void __launch_bounds__(CBS) k_ctl_restart(Ctl<S>* c, const double* red) {
    for (int e = threadIdx.x; e < S * S; e += CBS) c->s_old[e] = red[e];
    if (threadIdx.x == 0) {
        c->matvecs += c->sa;
        c->cmd = kCmdPupdate;
    }
}

// red = honest ||b - A x||^2 of still-active columns (solvers.cpp:655-661)
template <int S>
__global__ void k_ctl_final(Ctl<S>* c, const double* red, bk::CgReport* rep) {
    if (threadIdx.x == 0) {
        if (c->sa > 0) c->matvecs += c->sa;
        for (int q = 0; q < S; ++q)
            if (c->act[q]) {
                const double rt = sqrt(red[q]) / c->bnorm[q];
                c->fres[q] = rt;
                c->conv[q] = rt <= c->tol;
            }
        rep->iterations = c->iters;
        rep->matvecs = c->matvecs;
        for (int q = 0; q < S && q < 64; ++q) {
            rep->final_res[q] = c->fres[q];
            rep->converged[q] = (char)c->conv[q];
        }
    }
}

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
}  // namespace

namespace bk {

// Communication hooks for the slab decomposition (all optional; single-slab
// runs pass nullptr). allreduce: in-place sum of `count` device doubles
// across ranks. halo: refresh the two ghost rows of the slab-local block V.
struct LargeComm {
    void* user;
    void (*allreduce)(void* user, double* dev, int64_t count, cudaStream_t stream);
    void (*halo)(void* user, double* dev_local_block, cudaStream_t stream);
};

template <int S>
bk_status block_cg_large_t(bk_ctx* ctx, const bk_operator* op, int nyl, int y0,
                           const double* Bloc, double* Xloc, double* Rloc, double* Ploc,
                           double* Wloc, const bk_solver_cfg* cfg, CgReport* rep,
                           const LargeComm* comm) {
    Slab sl{op->nx, nyl, op->nz, op->ny, y0, (int64_t)op->nx * nyl * op->nz};
    SweepArgs a{};
    a.sl = sl;
    a.st = StencilPtr{op->diag, op->cx, op->cy, op->cz, op->dinv};
    a.B = Bloc;
    a.X = Xloc;
    a.R = Rloc;
    a.P = Ploc;
    a.W = Wloc;
    a.precond = cfg->precond;
    const int nb = sweep_ctas(ctx, sl, S);
    constexpr int E = S * S + S;
    // warp-specialised TMA update sweep for S = 64 on full 16-cell x-runs
    const bool ws_update = S == 64 && update64_ws_ok(sl) && !ctx->knobs.no_ws_update;
    const bool ws_spmm = S == 64 && update64_ws_ok(sl) && !ctx->knobs.no_ws_spmm;
    const int64_t nloc_ws = (int64_t)sl.nx * (sl.nyl + 2) * sl.nz;
    ctx->last_variant = "block_cg_large<" + std::to_string(S) + ">" +
                        ((S == 64 && sl.nx % 16 == 0 && !ctx->knobs.no_tma_spmm) ? " tma" : "") +
                        (ws_update ? " ws-update" : "") + (ws_spmm ? " ws-spmm" : "");
    void *pPart, *pRed, *pCtl, *pHost;
    bk_status st;
    if (ws_spmm && !ctx->knobs.spmm_teams) {  // packed per-run coefficients of the stencil sweep
        void* pc;
        const size_t runs = (size_t)(sl.nx / 16) * sl.ny * sl.nz;
        if ((st = workspace(ctx, kSlotCgCoef64, runs * sweep64::kPC * 8, &pc)) != BK_OK) return st;
        sweep64::k_pack_coef64<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(sl, a.st, (double*)pc);
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaGetLastError());
        a.pcoef = (const double*)pc;
    }
    if ((st = workspace(ctx, kSlotCgPart, (size_t)nb * E * 8, &pPart)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgRed, (size_t)E * 8, &pRed)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgCtl, sizeof(Ctl<S>) + sizeof(CgReport), &pCtl)) != BK_OK)
        return st;
    Ctl<S>* ctl = (Ctl<S>*)pCtl;
    CgReport* drep = (CgReport*)((char*)pCtl + sizeof(Ctl<S>));
    a.part = (double*)pPart;
    a.coef = ctl->coef;
    a.act = ctl->act;
    double* red = (double*)pRed;
    cudaStream_t s = ctx->stream;
    (void)pHost;
    auto reduce = [&](int e_count, int nparts) {
        k_reduce<<<(e_count + 7) / 8, 256, 0, s>>>(a.part, nparts, e_count, red);
        ++ctx->launches;
        if (comm && comm->allreduce) comm->allreduce(comm->user, red, e_count, s);
    };
    auto halo = [&](double* v) {
        if (comm && comm->halo) comm->halo(comm->user, v, s);
    };
    auto read_cmd = [&](int* cmd, int* sa) -> bk_status {
        static_assert(offsetof(Ctl<S>, cmd) == offsetof(Ctl<S>, sa) + 3 * sizeof(int), "layout");
        int h[4];  // sa, nver, iters, cmd
        const bk_status rs = read_small(ctx, h, &ctl->sa, sizeof(h));
        *sa = h[0];
        *cmd = h[3];
        return rs;
    };
    const int tr_blocks = (int)((sl.n_int + (LBS / S) - 1) / (LBS / S) < 4L * ctx->num_sms
                                    ? (sl.n_int + (LBS / S) - 1) / (LBS / S)
                                    : 4L * ctx->num_sms);
    auto true_res = [&]() {
        k_true_res<S><<<tr_blocks, LBS, 0, s>>>(a);
        ++ctx->launches;
        reduce(S, tr_blocks);
    };

    constexpr size_t swa = smem_anchor<S>(), sws = smem_spmm<S>(), swu = smem_update<S>(),
                     swp = smem_pupdate<S>();
    const size_t cs = sizeof(CSm<S>);
    {
        const auto set = [&](const void* f, size_t b) {
            return bk::set_max_smem(f, b);
        };
        BK_CUDA_TRY(ctx, set((const void*)k_anchor<S, kInit>, swa));
        BK_CUDA_TRY(ctx, set((const void*)k_anchor<S, kRestart>, swa));
        BK_CUDA_TRY(ctx, set((const void*)k_spmm_gram<S>, sws));
        BK_CUDA_TRY(ctx, set((const void*)k_update<S>, swu));
        BK_CUDA_TRY(ctx, set((const void*)k_pupdate<S>, swp));
        BK_CUDA_TRY(ctx, set((const void*)k_ctl_init<S>, cs));
        BK_CUDA_TRY(ctx, set((const void*)k_ctl_alpha<S>, cs));
        BK_CUDA_TRY(ctx, set((const void*)k_ctl_update<S>, cs));
        BK_CUDA_TRY(ctx, set((const void*)k_ctl_verify<S>, cs));
    }
    phase_reset(ctx);
    k_anchor<S, kInit><<<nb, LBS, swa, s>>>(a);
    ++ctx->launches;
    reduce(E, nb);
    k_ctl_init<S><<<1, CBS, cs, s>>>(ctl, red, cfg->rel_tol);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    int cmd = 0, sa = 0;
    if ((st = read_cmd(&cmd, &sa)) != BK_OK) return st;
    // X += P alpha is deferred from the update sweep to the P update, which
    // reads the same P rows (one P read fewer per iteration; bitwise the same
    // X); a verification first applies the pending update (k_pupdate MODE 2)
    a.coef2 = ctl->akeep;
    const bool ws = S == 64 && ws_spmm && ws_update;
    const int nbs = ws_spmm && ctx->num_sms < nb ? ctx->num_sms : nb;
    const int nbu = ws_update && ctx->num_sms < nb ? ctx->num_sms : nb;
    // one iteration's sweeps up to and including the convergence test
    // (m <= 0: inside the device-driven loop, see k_ctl_update)
    int gated = 0;  // lookahead loop: control kernels gated on the control word too
    auto sweeps = [&](int m, cudaGraphConditionalHandle loop) -> bk_status {
        halo(a.P);
        phase_mark(ctx, -1);
        if (ws_spmm) {
            BK_CUDA_TRY(ctx, launch_spmm64_ws(a, nbs, s, ctx->knobs.spmm_teams,
                                              ctx->knobs.spmm_band > 0 ? ctx->knobs.spmm_band : 4));
        } else {
            BK_CUDA_TRY(ctx, launch_spmm<S>(a, nb, s, ctx->knobs.no_tma_spmm));
        }
        phase_mark(ctx, 0);
        ++ctx->launches;
        reduce(S * S, nbs);
        k_ctl_alpha<S><<<1, CBS, cs, s>>>(ctl, red, gated);
        ++ctx->launches;
        phase_mark(ctx, -1);
        if (ws_update) {
            BK_CUDA_TRY(ctx, launch_update64_ws(a, nloc_ws, nbu, s));
        } else {
            BK_CUDA_TRY(ctx, (launch_update<S, true>(a, nb, s)));
        }
        phase_mark(ctx, 1);
        ++ctx->launches;
        reduce(E, nbu);
        k_ctl_update<S><<<1, CBS, cs, s>>>(ctl, red, m, loop, cfg->max_iter, gated);
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaGetLastError());
        return BK_OK;
    };
    // the P update closing an iteration (X += P alpha deferred into it)
    auto pupdate = [&]() -> bk_status {
        phase_mark(ctx, -1);
        if (ws_update)
            BK_CUDA_TRY(ctx, launch_pupdate64_ws(a, nloc_ws, nbu, s));
        else
            BK_CUDA_TRY(ctx, (launch_pupdate<S, 1>(a, nb, s)));
        phase_mark(ctx, 2);
        ++ctx->launches;
        return BK_OK;
    };
    // Device-driven loop (option graph_loop; single slab, no per-sweep event
    // timing): the iteration is a CUDA graph body under a while-node;
    // k_ctl_update clears the condition when a true-residual verification is
    // due or max_iter is reached, and the body's P update is gated on the same
    // control word, so the host only wakes up for verifications
    // (solvers.cpp:582-634). Bitwise the host-driven loop. Not the default: on
    // C5 the host-driven loop already hides its one control read per
    // iteration behind the queued sweeps (5.96 vs 6.07 ms per iteration,
    // scripts/c5_loop_ab.py).
    cudaGraphExec_t gexec = nullptr;
    int launches_per_iter = 0;
    if (!comm && !ctx->knobs.phase_timing && ctx->knobs.graph_loop && sa > 0) {
        cudaGraph_t g = nullptr;
        cudaStream_t cap = nullptr;
        cudaGraphConditionalHandle h;
        cudaGraphNodeParams cp = {};
        cudaGraphNode_t node;
        bool ok = cudaGraphCreate(&g, 0) == cudaSuccess &&
                  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
        if (ok) {
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            ok = cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess &&
                 cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess;
        }
        if (ok) {
            const cudaStream_t keep = s;
            const int64_t l0 = ctx->launches;
            s = cap;
            ok = cudaStreamBeginCaptureToGraph(cap, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                               cudaStreamCaptureModeRelaxed) == cudaSuccess;
            bk_status bs = BK_OK;
            if (ok) {
                a.gate = &ctl->cmd;
                bs = sweeps(0, h);
                if (bs == BK_OK) bs = pupdate();
                a.gate = nullptr;
                cudaGraph_t body = nullptr;
                ok = cudaStreamEndCapture(cap, &body) == cudaSuccess && bs == BK_OK;
            }
            s = keep;
            launches_per_iter = (int)(ctx->launches - l0);
            ctx->launches = l0;
            ok = ok && cudaGraphInstantiate(&gexec, g, 0) == cudaSuccess;
            if (bs != BK_OK) ok = false;
        }
        if (cap) cudaStreamDestroy(cap);
        if (g) cudaGraphDestroy(g);
        if (!ok) {
            if (gexec) cudaGraphExecDestroy(gexec);
            gexec = nullptr;
            cudaGetLastError();
            return fail(ctx, BK_INTERNAL, "block_cg: building the device-driven iteration loop failed");
        }
    }
    struct GraphGuard {
        cudaGraphExec_t& e;
        ~GraphGuard() {
            if (e) cudaGraphExecDestroy(e);
        }
    } gguard{gexec};
    auto read_iters = [&](int* iters) -> bk_status {
        return read_small(ctx, iters, &ctl->iters, sizeof(int));
    };
    // the verification due after iteration m (solvers.cpp:582-634): 1 = go on
    // with iteration m + 1, 0 = solve finished, < 0 = error
    auto verify = [&]() -> int {
        if (launch_pupdate<S, 2>(a, nb, s) != cudaSuccess) return -1;
        ++ctx->launches;
        halo(a.X);
        true_res();
        k_ctl_verify<S><<<1, CBS, cs, s>>>(ctl, red);
        ++ctx->launches;
        if (read_cmd(&cmd, &sa) != BK_OK) return -1;
        if (cmd == kCmdDone) return 0;
        if (cmd == kCmdRestart) {
            k_anchor<S, kRestart><<<nb, LBS, swa, s>>>(a);
            ++ctx->launches;
            reduce(E, nb);
            k_ctl_restart<S><<<1, CBS, 0, s>>>(ctl, red);
            ++ctx->launches;
            return 1;
        }
        phase_mark(ctx, -1);
        if (launch_pupdate<S, 0>(a, nb, s) != cudaSuccess) return -1;
        phase_mark(ctx, 2);
        ++ctx->launches;
        return 1;
    };
    int m = 0;  // iterations done
    // Lookahead loop (default; single slab, no graph loop, no per-sweep event
    // timing): iteration m + 1 is enqueued — every sweep and control kernel
    // gated on the control word — before the host waits for iteration m's
    // word, which is copied asynchronously into mapped pinned memory; the
    // device never drains between iterations. A verification due at m turns
    // the enqueued m + 1 into no-ops; the host verifies and re-issues m + 1.
    // The same kernels run on the same data as the synchronous loop, so the
    // result is bitwise the same.
    if (!gexec && !comm && !ctx->knobs.phase_timing && !ctx->knobs.no_lookahead &&
        m < cfg->max_iter && sa > 0) {
        auto issue = [&](int it) -> bk_status {
            a.gate = &ctl->cmd;
            gated = 1;
            bk_status is = sweeps(it, 0);
            if (is == BK_OK) is = pupdate();
            if (is == BK_OK) is = post_small(ctx, it & 1, &ctl->sa, 4 * sizeof(int));
            a.gate = nullptr;
            gated = 0;
            return is;
        };
        m = 1;
        if ((st = issue(m)) != BK_OK) return st;
        for (;;) {
            const bool ahead = m + 1 <= cfg->max_iter;
            if (ahead && (st = issue(m + 1)) != BK_OK) return st;
            int h[4];  // sa, nver, iters, cmd
            if ((st = wait_small(ctx, m & 1, h, sizeof(h))) != BK_OK) return st;
            if (h[3] == kCmdPupdate) {  // iteration m closed with its P update
                if (!ahead) break;
                ++m;
                continue;
            }
            const int v = verify();  // the enqueued m + 1 ran as no-ops
            if (v < 0) return fail(ctx, BK_CUDA_ERROR, "block_cg: verification");
            if (v == 0) break;
            ++m;
            if (m > cfg->max_iter || sa <= 0) break;
            if ((st = issue(m)) != BK_OK) return st;
        }
        m = cfg->max_iter;  // the synchronous loop below does not run
    }
    while (m < cfg->max_iter && sa > 0) {
        if (gexec) {
            BK_CUDA_TRY(ctx, cudaGraphLaunch(gexec, s));
            int it = 0;
            if ((st = read_cmd(&cmd, &sa)) != BK_OK) return st;
            if ((st = read_iters(&it)) != BK_OK) return st;
            ctx->launches += (int64_t)launches_per_iter * (it - m);
            m = it;
            if (cmd == kCmdPupdate) continue;  // iteration cap: the loop's last P update ran
        } else {
            ++m;
            if ((st = sweeps(m, 0)) != BK_OK) return st;
            if ((st = read_cmd(&cmd, &sa)) != BK_OK) return st;
            if (cmd == kCmdPupdate) {
                if ((st = pupdate()) != BK_OK) return st;
                continue;
            }
        }
        // cmd == kCmdVerify
        const int v = verify();
        if (v < 0) return fail(ctx, BK_CUDA_ERROR, "block_cg: verification");
        if (v == 0) break;
    }
    // honest residuals for still-active columns
    if ((st = read_small(ctx, &sa, &ctl->sa, sizeof(int))) != BK_OK) return st;
    if (sa > 0) {
        halo(a.X);
        true_res();
    }
    k_ctl_final<S><<<1, 32, 0, s>>>(ctl, red, drep);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    phase_collect(ctx);
    return read_small(ctx, rep, drep, sizeof(CgReport));
}

// Single-GPU entry: global [n][S] B/X, slab = the whole grid.
template <int S>
bk_status block_cg_large_single(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                                const bk_solver_cfg* cfg, double* X, CgReport* rep) {
    const int nyl = op->ny;
    const int64_t nloc = (int64_t)op->nx * (nyl + 2) * op->nz;
    const size_t bytes = (size_t)nloc * S * sizeof(double);
    void *pB, *pX, *pR, *pP, *pW, *pG;
    bk_status st;
    if ((st = workspace(ctx, kSlotCgB, bytes, &pB)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgX, bytes, &pX)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgR, bytes, &pR)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgP, bytes, &pP)) != BK_OK) return st;
    if ((st = workspace(ctx, kSlotCgW, bytes, &pW)) != BK_OK) return st;
    Slab sl{op->nx, nyl, op->nz, op->ny, 0, (int64_t)op->nx * nyl * op->nz};
    const double* Bg = B;
    if (s != S) {  // zero-pad the columns (zero RHS = pre-converged, solvers.cpp:478-485)
        if ((st = workspace(ctx, kSlotIn2, (size_t)op->n * S * 8, &pG)) != BK_OK) return st;
        BK_CUDA_TRY(ctx, launch_pad_cols(ctx, B, s, (double*)pG, S, op->n));
        Bg = (const double*)pG;
    }
    // ghost rows stay zero: at the global boundary their coefficients are 0
    BK_CUDA_TRY(ctx, cudaMemsetAsync(pB, 0, bytes, ctx->stream));
    BK_CUDA_TRY(ctx, cudaMemsetAsync(pP, 0, bytes, ctx->stream));
    BK_CUDA_TRY(ctx, cudaMemsetAsync(pX, 0, bytes, ctx->stream));
    const int grid = ctx->num_sms * 8;
    k_pack<S><<<grid, 256, 0, ctx->stream>>>(sl, const_cast<double*>(Bg), (double*)pB, 1);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    st = block_cg_large_t<S>(ctx, op, nyl, 0, (const double*)pB, (double*)pX, (double*)pR,
                             (double*)pP, (double*)pW, cfg, rep, nullptr);
    if (st != BK_OK) return st;
    double* Xg = X;
    if (s != S) Xg = (double*)pG;  // reuse the padded buffer for the output
    k_pack<S><<<grid, 256, 0, ctx->stream>>>(sl, Xg, (double*)pX, 0);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    if (s != S) BK_CUDA_TRY(ctx, launch_pad_cols(ctx, Xg, S, X, s, op->n));
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
}

bk_status block_cg_large(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                         const bk_solver_cfg* cfg, double* X, CgReport* rep) {
    if (s <= 16) return block_cg_large_single<16>(ctx, op, B, s, cfg, X, rep);
    if (s <= 32) return block_cg_large_single<32>(ctx, op, B, s, cfg, X, rep);
    if (s <= 64) return block_cg_large_single<64>(ctx, op, B, s, cfg, X, rep);
    return fail(ctx, BK_INVALID_CONFIG, "block_cg: s > 64 is not supported on device");
}

}  // namespace bk

// ---------------------------------------------------------------------------
// C ABI: per-phase steps for the y-slab decomposition (driven by dd.py)
// ---------------------------------------------------------------------------
namespace {

template <int S>
bk_status dd_step_t(bk_ctx* ctx, const bk_operator* op, int y0, int nyl, const bk_dd_bufs* b,
                    const bk_solver_cfg* cfg, int step, int m, int* cmd, int* sa,
                    bk_solve_report* report) {
    using namespace bk;
    Slab sl{op->nx, nyl, op->nz, op->ny, y0, (int64_t)op->nx * nyl * op->nz};
    SweepArgs a{};
    a.sl = sl;
    a.st = StencilPtr{op->diag, op->cx, op->cy, op->cz, op->dinv};
    a.B = b->B;
    a.X = b->X;
    a.R = b->R;
    a.P = b->P;
    a.W = b->W;
    a.part = b->part;
    a.precond = cfg ? cfg->precond : 1;
    Ctl<S>* ctl = (Ctl<S>*)b->ctl;
    CgReport* drep = (CgReport*)((char*)b->ctl + sizeof(Ctl<S>));
    a.coef = ctl->coef;
    a.coef2 = ctl->akeep;
    a.act = ctl->act;
    constexpr int E = S * S + S;
    const int nb = b->nb;
    cudaStream_t s = ctx->stream;
    // BK_DD_GATED: the sweep and control kernels of an iteration enqueued
    // ahead of the host's read of the previous iteration's control word run
    // only while that word says "P update" (no verification pending)
    const int gated = (step & BK_DD_GATED) ? 1 : 0;
    step &= ~BK_DD_GATED;
    if (gated) a.gate = &ctl->cmd;
    // S = 64 on 16-aligned x: the warp-specialised sweeps of the single-GPU
    // engine (one CTA per SM, deferred X), their partial count and the packed
    // stencil coefficients (built by BK_DD_INIT_SWEEP)
    const bool ws = S == 64 && update64_ws_ok(sl);
    const int nws = ctx->num_sms < nb ? ctx->num_sms : nb;
    const int64_t nloc_ws = (int64_t)sl.nx * (sl.nyl + 2) * sl.nz;
    if (ws) {
        void* pc;
        const size_t runs = (size_t)(sl.nx / 16) * sl.ny * sl.nz;
        bk_status wst = workspace(ctx, kSlotCgCoef64, runs * sweep64::kPC * 8, &pc);
        if (wst != BK_OK) return wst;
        a.pcoef = (const double*)pc;
    }
    constexpr size_t swa = smem_anchor<S>(), sws = smem_spmm<S>(), swu = smem_update<S>(),
                     swp = smem_pupdate<S>();
    const size_t cs = sizeof(CSm<S>);
    auto set = [&](const void* f, size_t bytes) {
        return bk::set_max_smem(f, bytes);
    };
    auto reduce = [&](int e_count, int nparts) {
        k_reduce<<<(e_count + 7) / 8, 256, 0, s>>>(b->part, nparts, e_count, b->red);
        ++ctx->launches;
    };
    const int tr_blocks = (int)((sl.n_int + (LBS / S) - 1) / (LBS / S) < 4L * ctx->num_sms
                                    ? (sl.n_int + (LBS / S) - 1) / (LBS / S)
                                    : 4L * ctx->num_sms);
    switch (step) {
        case BK_DD_INIT_SWEEP:
            if (ws) {
                sweep64::k_pack_coef64<<<ctx->num_sms * 8, 256, 0, s>>>(sl, a.st, (double*)a.pcoef);
                ++ctx->launches;
            }
            BK_CUDA_TRY(ctx, set((const void*)k_anchor<S, kInit>, swa));
            k_anchor<S, kInit><<<nb, LBS, swa, s>>>(a);
            ++ctx->launches;
            reduce(E, nb);
            break;
        case BK_DD_CTL_INIT:
            BK_CUDA_TRY(ctx, set((const void*)k_ctl_init<S>, cs));
            k_ctl_init<S><<<1, CBS, cs, s>>>(ctl, b->red, cfg->rel_tol);
            ++ctx->launches;
            break;
        case BK_DD_SPMM:
            if (ws) {
                BK_CUDA_TRY(ctx, launch_spmm64_ws(a, nws, s, false,
                                                  ctx->knobs.spmm_band > 0 ? ctx->knobs.spmm_band : 4));
                ++ctx->launches;
                reduce(S * S, nws);
            } else {
                BK_CUDA_TRY(ctx, launch_spmm<S>(a, nb, s, ctx->knobs.no_tma_spmm));
                ++ctx->launches;
                reduce(S * S, nb);
            }
            break;
        case BK_DD_UPDATE_D:
            if (ws) {
                BK_CUDA_TRY(ctx, launch_update64_ws(a, nloc_ws, nws, s));
                ++ctx->launches;
                reduce(E, nws);
            } else {
                BK_CUDA_TRY(ctx, (launch_update<S, true>(a, nb, s)));
                ++ctx->launches;
                reduce(E, nb);
            }
            break;
        case BK_DD_PUPDATE_X:
            if (ws) {
                BK_CUDA_TRY(ctx, launch_pupdate64_ws(a, nloc_ws, nws, s));
            } else {
                BK_CUDA_TRY(ctx, (launch_pupdate<S, 1>(a, nb, s)));
            }
            ++ctx->launches;
            break;
        case BK_DD_APPLY_X:
            BK_CUDA_TRY(ctx, (launch_pupdate<S, 2>(a, nb, s)));
            ++ctx->launches;
            break;
        case BK_DD_CTL_ALPHA:
            BK_CUDA_TRY(ctx, set((const void*)k_ctl_alpha<S>, cs));
            k_ctl_alpha<S><<<1, CBS, cs, s>>>(ctl, b->red, gated);
            ++ctx->launches;
            break;
        case BK_DD_UPDATE:
            BK_CUDA_TRY(ctx, set((const void*)k_update<S>, swu));
            BK_CUDA_TRY(ctx, launch_update<S>(a, nb, s));
            ++ctx->launches;
            reduce(E, nb);
            break;
        case BK_DD_CTL_UPDATE:
            BK_CUDA_TRY(ctx, set((const void*)k_ctl_update<S>, cs));
            k_ctl_update<S><<<1, CBS, cs, s>>>(ctl, b->red, m, 0, 0, gated);
            ++ctx->launches;
            break;
        case BK_DD_TRUE_RES:
            k_true_res<S><<<tr_blocks, LBS, 0, s>>>(a);
            ++ctx->launches;
            reduce(S, tr_blocks);
            break;
        case BK_DD_CTL_VERIFY:
            BK_CUDA_TRY(ctx, set((const void*)k_ctl_verify<S>, cs));
            k_ctl_verify<S><<<1, CBS, cs, s>>>(ctl, b->red);
            ++ctx->launches;
            break;
        case BK_DD_RESTART_SWEEP:
            BK_CUDA_TRY(ctx, set((const void*)k_anchor<S, kRestart>, swa));
            k_anchor<S, kRestart><<<nb, LBS, swa, s>>>(a);
            ++ctx->launches;
            reduce(E, nb);
            break;
        case BK_DD_CTL_RESTART:
            k_ctl_restart<S><<<1, CBS, 0, s>>>(ctl, b->red);
            ++ctx->launches;
            break;
        case BK_DD_PUPDATE:
            BK_CUDA_TRY(ctx, set((const void*)k_pupdate<S>, swp));
            BK_CUDA_TRY(ctx, launch_pupdate<S>(a, nb, s));
            ++ctx->launches;
            break;
        case BK_DD_CTL_FINAL: {
            k_ctl_final<S><<<1, 32, 0, s>>>(ctl, b->red, drep);
            ++ctx->launches;
            CgReport rep;
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(&rep, drep, sizeof(rep), cudaMemcpyDeviceToHost, s));
            BK_CUDA_TRY(ctx, cudaStreamSynchronize(s));
            if (report) {
                report->iterations = rep.iterations;
                report->matvec_count = rep.matvecs;
                for (int j = 0; j < S; ++j) {
                    if (report->final_rel_residual) report->final_rel_residual[j] = rep.final_res[j];
                    if (report->converged) report->converged[j] = rep.converged[j];
                }
            }
            break;
        }
        case BK_DD_READ_ASYNC:
            // cmd / sa: pinned host words, valid until the stream passes the copies
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(cmd, &ctl->cmd, sizeof(int), cudaMemcpyDeviceToHost, s));
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(sa, &ctl->sa, sizeof(int), cudaMemcpyDeviceToHost, s));
            break;
        case BK_DD_READ: {
            int h[2];
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(h, &ctl->cmd, sizeof(int), cudaMemcpyDeviceToHost, s));
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(h + 1, &ctl->sa, sizeof(int), cudaMemcpyDeviceToHost, s));
            BK_CUDA_TRY(ctx, cudaStreamSynchronize(s));
            if (cmd) *cmd = h[0];
            if (sa) *sa = h[1];
            break;
        }
        default:
            return fail(ctx, BK_INVALID_CONFIG, "dd_step: unknown step");
    }
    BK_CUDA_TRY(ctx, cudaGetLastError());
    return BK_OK;
}

template <int S>
int64_t ctl_bytes_t() {
    return (int64_t)(sizeof(Ctl<S>) + sizeof(bk::CgReport));
}

}  // namespace

// debug harness (scripts/ only): cycles of the S = 64 control solve in one
// CTA of CBS threads, by the number of warps running the pivot loop
template <int NWS>
__device__ long long ctl_solve_cycles(CSm<64>& sm, const double* M, const double* R, int reps) {
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) small_solve_t<64, CBS, false, 0, NWS>(sm, M, R, sm.out);
    __syncthreads();
    return (clock64() - t0) / reps;
}
// the register solve with all BS = 32 NWR threads in the pivot loop
template <int NWR>
__global__ void __launch_bounds__(NWR * 32) k_ctl_solve_bench_nw(int reps, long long* out) {
    extern __shared__ __align__(16) unsigned char smraw_[];
    CSm<64>& sm = *reinterpret_cast<CSm<64>*>(smraw_);
    constexpr int S = 64, BS = NWR * 32;
    for (int e = threadIdx.x; e < S * S; e += BS) {
        const int i = e / S, j = e % S;
        sm.m0[e] = (i == j ? 1.0 : 0.01 / (1 + i + j)) * exp(-0.05 * (i + j));
        sm.m1[e] = (i == j ? 2.0 : 0.1) * exp(-0.025 * (i + j));
    }
    if (threadIdx.x < S) sm.idx[threadIdx.x] = threadIdx.x;
    if (threadIdx.x == 0) sm.sa = S;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) small_solve_reg<64, BS, 0, NWR>(sm, sm.m0, sm.m1, sm.out);
    __syncthreads();
    if (threadIdx.x == 0) *out = (clock64() - t0) / reps;
}
template <int VAR, int NWR = 16>
__device__ long long reg_cycles(CSm<64>& sm, int reps) {
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) small_solve_reg<64, CBS, VAR, NWR>(sm, sm.m0, sm.m1, sm.out);
    __syncthreads();
    return (clock64() - t0) / reps;
}
__global__ void __launch_bounds__(CBS) k_ctl_solve_bench(int reps, long long* out, double* res, int only_reg) {
    extern __shared__ __align__(16) unsigned char smraw_[];
    CSm<64>& sm = *reinterpret_cast<CSm<64>*>(smraw_);
    constexpr int S = 64;
    for (int e = threadIdx.x; e < S * S; e += CBS) {
        const int i = e / S, j = e % S;
        sm.m0[e] = (i == j ? 1.0 : 0.01 / (1 + i + j)) * exp(-0.05 * (i + j));
        sm.m1[e] = (i == j ? 2.0 : 0.1) * exp(-0.025 * (i + j));
    }
    if (threadIdx.x < S) sm.idx[threadIdx.x] = threadIdx.x;
    if (threadIdx.x == 0) sm.sa = S;
    __syncthreads();
    long long c[5] = {};
    if (!only_reg) {
        c[0] = ctl_solve_cycles<16>(sm, sm.m0, sm.m1, reps);
        c[1] = ctl_solve_cycles<8>(sm, sm.m0, sm.m1, reps);
        c[2] = ctl_solve_cycles<4>(sm, sm.m0, sm.m1, reps);
        c[3] = ctl_solve_cycles<2>(sm, sm.m0, sm.m1, reps);
    }
    for (int e = threadIdx.x; e < S * S; e += CBS) res[e] = sm.out[(e / S) * Strides<S>::RS + e % S];
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) small_solve_reg<64, CBS>(sm, sm.m0, sm.m1, sm.out);
    __syncthreads();
    c[4] = (clock64() - t0) / reps;
    if (threadIdx.x == 0) {
        for (int v = 0; v < 5; ++v) out[v] = c[v];
        out[5] = sm.rank;
    }
    for (int e = threadIdx.x; e < S * S; e += CBS)
        res[S * S + e] = sm.out[(e / S) * Strides<S>::RS + e % S];
    long long cv[4] = {};
    if (!only_reg) {
        cv[0] = reg_cycles<1>(sm, reps);
        cv[3] = reg_cycles<3>(sm, reps);
    }
    if (threadIdx.x == 0)
        for (int v = 0; v < 4; ++v) out[6 + v] = cv[v];
}

extern "C" {

int bk_debug_ctl_solve_cycles(int reps, long long* cycles6, double* coef2, int only_reg) {
    long long* d;
    double* r;
    cudaMalloc(&d, 16 * 8);
    cudaMalloc(&r, 2 * 64 * 64 * 8);
    cudaFuncSetAttribute(k_ctl_solve_bench, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(CSm<64>));
    k_ctl_solve_bench<<<1, CBS, sizeof(CSm<64>)>>>(reps, d, r, only_reg);
    int err = (int)cudaDeviceSynchronize();
    if (!only_reg) {
        cudaFuncSetAttribute(k_ctl_solve_bench_nw<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(CSm<64>));
        cudaFuncSetAttribute(k_ctl_solve_bench_nw<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(CSm<64>));
        k_ctl_solve_bench_nw<8><<<1, 256, sizeof(CSm<64>)>>>(reps, d + 7);
        k_ctl_solve_bench_nw<4><<<1, 128, sizeof(CSm<64>)>>>(reps, d + 8);
        err |= (int)cudaDeviceSynchronize();
    }
    cudaMemcpy(cycles6, d, 10 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(coef2, r, 2 * 64 * 64 * 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(r);
    return err;
}

int bk_dd_deferred_x(const bk_operator* op, int S) {
    return op && S == 64 && op->nx % 16 == 0 ? 1 : 0;
}

bk_status bk_dd_sizes(bk_ctx* ctx, const bk_operator* op, int nyl, int S, int64_t* local_elems,
                      int* nb, int64_t* part_elems, int64_t* red_elems, int64_t* ctl_bytes) {
    if (!ctx || !op || nyl < 1 || nyl > op->ny) return BK_INVALID_CONFIG;
    if (S != 16 && S != 32 && S != 64)
        return bk::fail(ctx, BK_INVALID_CONFIG, "dd: kernel width must be 16, 32 or 64");
    const int64_t n_int = (int64_t)op->nx * nyl * op->nz;
    const Slab sl{op->nx, nyl, op->nz, op->ny, 0, n_int};
    const int b = sweep_ctas(ctx, sl, S);
    const int tr = (int)((n_int + (LBS / S) - 1) / (LBS / S) < 4L * ctx->num_sms
                             ? (n_int + (LBS / S) - 1) / (LBS / S)
                             : 4L * ctx->num_sms);
    const int E = S * S + S;
    if (local_elems) *local_elems = (int64_t)op->nx * (nyl + 2) * op->nz * S;
    if (nb) *nb = b;
    if (part_elems) *part_elems = (int64_t)(b > tr ? b : tr) * E;
    if (red_elems) *red_elems = E;
    if (ctl_bytes) *ctl_bytes = S == 16 ? ctl_bytes_t<16>() : S == 32 ? ctl_bytes_t<32>() : ctl_bytes_t<64>();
    return BK_OK;
}

bk_status bk_dd_step(bk_ctx* ctx, const bk_operator* op, int y0, int nyl, int S,
                     const bk_dd_bufs* bufs, const bk_solver_cfg* cfg, int step, int m,
                     int* cmd, int* sa, bk_solve_report* report) {
    if (!ctx || !op || !bufs) return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    if (S == 16) return dd_step_t<16>(ctx, op, y0, nyl, bufs, cfg, step, m, cmd, sa, report);
    if (S == 32) return dd_step_t<32>(ctx, op, y0, nyl, bufs, cfg, step, m, cmd, sa, report);
    if (S == 64) return dd_step_t<64>(ctx, op, y0, nyl, bufs, cfg, step, m, cmd, sa, report);
    return bk::fail(ctx, BK_INVALID_CONFIG, "dd: kernel width must be 16, 32 or 64");
}

bk_status bk_dd_pack(bk_ctx* ctx, const bk_operator* op, int y0, int nyl, int S, double* glob,
                     double* loc, int to_local) {
    if (!ctx || !op || !glob || !loc) return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    Slab sl{op->nx, nyl, op->nz, op->ny, y0, (int64_t)op->nx * nyl * op->nz};
    const int grid = ctx->num_sms * 8;
    if (S == 16) k_pack<16><<<grid, 256, 0, ctx->stream>>>(sl, glob, loc, to_local);
    else if (S == 32) k_pack<32><<<grid, 256, 0, ctx->stream>>>(sl, glob, loc, to_local);
    else if (S == 64) k_pack<64><<<grid, 256, 0, ctx->stream>>>(sl, glob, loc, to_local);
    else return bk::fail(ctx, BK_INVALID_CONFIG, "dd: kernel width must be 16, 32 or 64");
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    return BK_OK;
}

}  // extern "C"
