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
#include <cstdio>
#include <cstdlib>
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

template <int S>
struct LTile {
    static constexpr int RS = S + 4;
    double u[16 * RS];  // A side of the Gram (rows = cells)
    double v[16 * RS];  // B side
};

// CTA Gram over staged tiles: warp w owns (m, n) tiles w, w + LNW, ... of the
// MT x NT tile grid of G = U^T V and accumulates them over every staged tile.
template <int S>
struct OwnedGram {
    static constexpr int MT = (S + 15) / 16;
    static constexpr int NT = S / 8;
    static constexpr int TILES = MT * NT;
    static constexpr int PER = (TILES + LNW - 1) / LNW;
    double d[PER][4];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < PER; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) d[i][e] = 0.0;
    }
    __device__ __forceinline__ void accumulate(const LTile<S>* tiles, int ntiles, int warp, int g,
                                               int t) {
        constexpr int RS = LTile<S>::RS;
        for (int k = 0; k < ntiles; ++k) {
            const double* U = tiles[k].u;
            const double* V = tiles[k].v;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int c4 = 4 * kk + t;
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int tile = warp + LNW * i;
                    if (tile >= TILES) break;
                    const int m = tile / NT, n = tile % NT;
                    const double a0 = U[c4 * RS + 16 * m + g];
                    const double a1 = (16 * m + 8 + g < S) ? U[c4 * RS + 16 * m + 8 + g] : 0.0;
                    dmma_l(d[i], a0, a1, V[c4 * RS + 8 * n + g]);
                }
            }
        }
    }
    // this CTA's partial: out[r * S + c]
    __device__ __forceinline__ void write(double* out, int warp, int g, int t) const {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int tile = warp + LNW * i;
            if (tile >= TILES) break;
            const int m = tile / NT, n = tile % NT;
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
    const int* act;      // per-column mask for masked sweeps
    int precond;
};

// stage two 16-cell C-layout tiles (rows g, g + 8) into smem tile k
template <int S>
__device__ __forceinline__ void stage_c(LTile<S>& tl, const double (&u)[S / 8][4],
                                        const double (&v)[S / 8][4], int g, int t) {
    constexpr int RS = LTile<S>::RS;
#pragma unroll
    for (int n = 0; n < S / 8; ++n) {
        const int col = 8 * n + 2 * t;
        *reinterpret_cast<double2*>(tl.u + g * RS + col) = make_double2(u[n][0], u[n][1]);
        *reinterpret_cast<double2*>(tl.u + (g + 8) * RS + col) = make_double2(u[n][2], u[n][3]);
        *reinterpret_cast<double2*>(tl.v + g * RS + col) = make_double2(v[n][0], v[n][1]);
        *reinterpret_cast<double2*>(tl.v + (g + 8) * RS + col) = make_double2(v[n][2], v[n][3]);
    }
}

template <int S>
__device__ __forceinline__ void ld_c(const double* V, const LCell& c0, const LCell& c1, bool v0,
                                     bool v1, int t, double (&o)[S / 8][4]) {
#pragma unroll
    for (int n = 0; n < S / 8; ++n) {
        const double2 a = v0 ? *reinterpret_cast<const double2*>(V + c0.l * S + 8 * n + 2 * t)
                             : make_double2(0.0, 0.0);
        const double2 b = v1 ? *reinterpret_cast<const double2*>(V + c1.l * S + 8 * n + 2 * t)
                             : make_double2(0.0, 0.0);
        o[n][0] = a.x;
        o[n][1] = a.y;
        o[n][2] = b.x;
        o[n][3] = b.y;
    }
}

template <int S>
__device__ __forceinline__ void st_c(double* V, const LCell& c0, const LCell& c1, bool v0,
                                     bool v1, int t, const double (&o)[S / 8][4]) {
#pragma unroll
    for (int n = 0; n < S / 8; ++n) {
        if (v0)
            *reinterpret_cast<double2*>(V + c0.l * S + 8 * n + 2 * t) = make_double2(o[n][0], o[n][1]);
        if (v1)
            *reinterpret_cast<double2*>(V + c1.l * S + 8 * n + 2 * t) = make_double2(o[n][2], o[n][3]);
    }
}

// ---------------------------------------------------------------------------
// sweeps (all: 16-cell tiles, one per warp per batch; batch = LNW tiles)
// ---------------------------------------------------------------------------
enum Sweep : int { kInit = 0, kRestart = 1 };

// X = 0, R = B (init) or R = B - A X (restart); Z = D^-1 R; P = Z;
// partials [R^T Z | sum b^2 (init)]
template <int S, int MODE>
__global__ void __launch_bounds__(LBS, 1) k_anchor(SweepArgs a) {
    constexpr int NT = S / 8;
    extern __shared__ __align__(16) unsigned char smraw_[];
    LTile<S>* tiles = reinterpret_cast<LTile<S>*>(smraw_);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t ntiles = (a.sl.n_int + 15) / 16;
    OwnedGram<S> G;
    G.zero();
    double bn[NT][2] = {};
    const bool jac = a.precond != 0;
    for (int64_t b0 = (int64_t)blockIdx.x * LNW; b0 < ntiles; b0 += (int64_t)gridDim.x * LNW) {
        const int64_t tile = b0 + warp;
        const int64_t u0 = tile * 16 + g, u1 = u0 + 8;
        const bool v0 = tile < ntiles && u0 < a.sl.n_int, v1 = tile < ntiles && u1 < a.sl.n_int;
        LCell c0, c1;
        if (v0) lcell(a.sl, a.st, u0, c0, MODE == kRestart);
        if (v1) lcell(a.sl, a.st, u1, c1, MODE == kRestart);
        double r[NT][4], z[NT][4];
        ld_c<S>(a.B, c0, c1, v0, v1, t, r);
        if (MODE == kRestart) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const LCell& c = h ? c1 : c0;
                if (!(h ? v1 : v0)) continue;
                const int64_t pz = (int64_t)a.sl.nx * (a.sl.nyl + 2);
#pragma unroll
                for (int n = 0; n < NT; ++n)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int64_t ee = c.l * S + 8 * n + 2 * t + e;
                        double acc = 0.0;
                        if (c.hzm) acc = fma(c.zm, a.X[ee - pz * S], acc);
                        if (c.hym) acc = fma(c.ym, a.X[ee - (int64_t)a.sl.nx * S], acc);
                        if (c.hxm) acc = fma(c.xm, a.X[ee - S], acc);
                        acc = fma(c.d, a.X[ee], acc);
                        if (c.hxp) acc = fma(c.xp, a.X[ee + S], acc);
                        if (c.hyp) acc = fma(c.yp, a.X[ee + (int64_t)a.sl.nx * S], acc);
                        if (c.hzp) acc = fma(c.zp, a.X[ee + pz * S], acc);
                        r[n][2 * h + e] -= acc;
                    }
            }
        }
        const double d0 = (jac && v0) ? a.st.dinv[c0.gi] : 1.0;
        const double d1 = (jac && v1) ? a.st.dinv[c1.gi] : 1.0;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            z[n][0] = d0 * r[n][0];
            z[n][1] = d0 * r[n][1];
            z[n][2] = d1 * r[n][2];
            z[n][3] = d1 * r[n][3];
            bn[n][0] += r[n][0] * r[n][0] + r[n][2] * r[n][2];
            bn[n][1] += r[n][1] * r[n][1] + r[n][3] * r[n][3];
        }
        if (MODE == kInit) {
            double zero[NT][4] = {};
            st_c<S>(a.X, c0, c1, v0, v1, t, zero);
        }
        st_c<S>(a.R, c0, c1, v0, v1, t, r);
        st_c<S>(a.P, c0, c1, v0, v1, t, z);
        stage_c<S>(tiles[warp], r, z, g, t);
        __syncthreads();
        const int nst = (int)((ntiles - b0) < LNW ? (ntiles - b0) : LNW);
        G.accumulate(tiles, nst, warp, g, t);
        __syncthreads();
    }
    constexpr int E = S * S + S;
    double* out = a.part + (int64_t)blockIdx.x * E;
    G.write(out, warp, g, t);
    // sum of squares of B per column (init): warp shuffle over g, then warps in order
    double (*vred)[S] = reinterpret_cast<double (*)[S]>(smraw_ + sizeof(LTile<S>) * LNW);
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double x = bn[n][e];
            x += __shfl_xor_sync(0xffffffffu, x, 4);
            x += __shfl_xor_sync(0xffffffffu, x, 8);
            x += __shfl_xor_sync(0xffffffffu, x, 16);
            if (lane < 4) vred[warp][8 * n + 2 * lane + e] = x;
        }
    __syncthreads();
    for (int c = threadIdx.x; c < S; c += LBS) {
        double s = 0.0;
        for (int w = 0; w < LNW; ++w) s += vred[w][c];
        out[S * S + c] = s;
    }
}

// phase 1: W = A P (CSR-order FMA chain) over interior cells; partial G = P^T W
template <int S>
__global__ void __launch_bounds__(LBS, 1) k_spmm_gram(SweepArgs a) {
    constexpr int RS = LTile<S>::RS;
    constexpr int CW = S / 2 < 8 ? S / 2 : 8;
    constexpr int PASSES = S / (2 * CW);
    extern __shared__ __align__(16) unsigned char smraw_[];
    LTile<S>* tiles = reinterpret_cast<LTile<S>*>(smraw_);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int r = lane >> 1, h = lane & 1;
    const int64_t ntiles = (a.sl.n_int + 15) / 16;
    const int64_t pz = (int64_t)a.sl.nx * (a.sl.nyl + 2);
    OwnedGram<S> G;
    G.zero();
    for (int64_t b0 = (int64_t)blockIdx.x * LNW; b0 < ntiles; b0 += (int64_t)gridDim.x * LNW) {
        const int64_t tile = b0 + warp;
        const int64_t u = tile * 16 + r;
        const bool v = tile < ntiles && u < a.sl.n_int;
        LCell c;
        if (v) lcell(a.sl, a.st, u, c, true);
#pragma unroll
        for (int ps = 0; ps < PASSES; ++ps) {
            const int col = ps * 2 * CW + h * CW;
            double acc[CW], ctr[CW];
#pragma unroll
            for (int j = 0; j < CW; ++j) acc[j] = ctr[j] = 0.0;
            if (v) {
                auto row = [&](int64_t l, double cf, bool has) {
                    if (!has) return;
                    const double2* src = reinterpret_cast<const double2*>(a.P + l * S + col);
#pragma unroll
                    for (int j = 0; j < CW / 2; ++j) {
                        const double2 x = src[j];
                        acc[2 * j] = fma(cf, x.x, acc[2 * j]);
                        acc[2 * j + 1] = fma(cf, x.y, acc[2 * j + 1]);
                    }
                };
                row(c.l - pz, c.zm, c.hzm);
                row(c.l - a.sl.nx, c.ym, c.hym);
                row(c.l - 1, c.xm, c.hxm);
                {
                    const double2* src = reinterpret_cast<const double2*>(a.P + c.l * S + col);
#pragma unroll
                    for (int j = 0; j < CW / 2; ++j) {
                        const double2 x = src[j];
                        ctr[2 * j] = x.x;
                        ctr[2 * j + 1] = x.y;
                        acc[2 * j] = fma(c.d, x.x, acc[2 * j]);
                        acc[2 * j + 1] = fma(c.d, x.y, acc[2 * j + 1]);
                    }
                }
                row(c.l + 1, c.xp, c.hxp);
                row(c.l + a.sl.nx, c.yp, c.hyp);
                row(c.l + pz, c.zp, c.hzp);
                double2* dst = reinterpret_cast<double2*>(a.W + c.l * S + col);
#pragma unroll
                for (int j = 0; j < CW / 2; ++j) dst[j] = make_double2(acc[2 * j], acc[2 * j + 1]);
            }
#pragma unroll
            for (int j = 0; j < CW / 2; ++j) {
                *reinterpret_cast<double2*>(tiles[warp].u + r * RS + col + 2 * j) =
                    make_double2(ctr[2 * j], ctr[2 * j + 1]);
                *reinterpret_cast<double2*>(tiles[warp].v + r * RS + col + 2 * j) =
                    make_double2(acc[2 * j], acc[2 * j + 1]);
            }
        }
        __syncthreads();
        const int nst = (int)((ntiles - b0) < LNW ? (ntiles - b0) : LNW);
        G.accumulate(tiles, nst, warp, g, t);
        __syncthreads();
    }
    G.write(a.part + (int64_t)blockIdx.x * (S * S), warp, g, t);
}

// phase 2: X += P alpha, R -= W alpha (DMMA, M = cells), rr, Z = D^-1 R,
// partials [S_new = R^T Z | rr]
template <int S>
__global__ void __launch_bounds__(LBS, 1) k_update(SweepArgs a) {
    constexpr int NT = S / 8, KS = S / 4, RSC = S + 4;
    extern __shared__ __align__(16) unsigned char smraw_[];
    LTile<S>* tiles = reinterpret_cast<LTile<S>*>(smraw_);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t ntiles = (a.sl.n_int + 15) / 16;
    const bool jac = a.precond != 0;
    OwnedGram<S> G;
    G.zero();
    double rr[NT][2] = {};
    for (int64_t b0 = (int64_t)blockIdx.x * LNW; b0 < ntiles; b0 += (int64_t)gridDim.x * LNW) {
        const int64_t tile = b0 + warp;
        const int64_t u0 = tile * 16 + g, u1 = u0 + 8;
        const bool v0 = tile < ntiles && u0 < a.sl.n_int, v1 = tile < ntiles && u1 < a.sl.n_int;
        LCell c0, c1;
        if (v0) lcell(a.sl, a.st, u0, c0, false);
        if (v1) lcell(a.sl, a.st, u1, c1, false);
        double x[NT][4], rv[NT][4];
        ld_c<S>(a.X, c0, c1, v0, v1, t, x);
        ld_c<S>(a.R, c0, c1, v0, v1, t, rv);
#pragma unroll 4
        for (int ks = 0; ks < KS; ++ks) {
            const int kc = 4 * ks + t;
            const double p0 = v0 ? a.P[c0.l * S + kc] : 0.0, p1 = v1 ? a.P[c1.l * S + kc] : 0.0;
            const double w0 = v0 ? -a.W[c0.l * S + kc] : 0.0, w1 = v1 ? -a.W[c1.l * S + kc] : 0.0;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const double bb = a.coef[kc * RSC + 8 * n + g];
                dmma_l(x[n], p0, p1, bb);
                dmma_l(rv[n], w0, w1, bb);
            }
        }
        st_c<S>(a.X, c0, c1, v0, v1, t, x);
        st_c<S>(a.R, c0, c1, v0, v1, t, rv);
        const double d0 = (jac && v0) ? a.st.dinv[c0.gi] : 1.0;
        const double d1 = (jac && v1) ? a.st.dinv[c1.gi] : 1.0;
        double z[NT][4];
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            rr[n][0] += rv[n][0] * rv[n][0] + rv[n][2] * rv[n][2];
            rr[n][1] += rv[n][1] * rv[n][1] + rv[n][3] * rv[n][3];
            z[n][0] = d0 * rv[n][0];
            z[n][1] = d0 * rv[n][1];
            z[n][2] = d1 * rv[n][2];
            z[n][3] = d1 * rv[n][3];
        }
        stage_c<S>(tiles[warp], rv, z, g, t);
        __syncthreads();
        const int nst = (int)((ntiles - b0) < LNW ? (ntiles - b0) : LNW);
        G.accumulate(tiles, nst, warp, g, t);
        __syncthreads();
    }
    constexpr int E = S * S + S;
    double* out = a.part + (int64_t)blockIdx.x * E;
    G.write(out, warp, g, t);
    double (*vred)[S] = reinterpret_cast<double (*)[S]>(smraw_ + sizeof(LTile<S>) * LNW);
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double xx = rr[n][e];
            xx += __shfl_xor_sync(0xffffffffu, xx, 4);
            xx += __shfl_xor_sync(0xffffffffu, xx, 8);
            xx += __shfl_xor_sync(0xffffffffu, xx, 16);
            if (lane < 4) vred[warp][8 * n + 2 * lane + e] = xx;
        }
    __syncthreads();
    for (int c = threadIdx.x; c < S; c += LBS) {
        double s = 0.0;
        for (int w = 0; w < LNW; ++w) s += vred[w][c];
        out[S * S + c] = s;
    }
}

// phase 3: P = D^-1 R + P beta (DMMA, accumulator initialised to Z)
template <int S>
__global__ void __launch_bounds__(LBS, 1) k_pupdate(SweepArgs a) {
    constexpr int NT = S / 8, KS = S / 4, RSC = S + 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t ntiles = (a.sl.n_int + 15) / 16;
    const bool jac = a.precond != 0;
    for (int64_t tile = (int64_t)blockIdx.x * LNW + warp; tile < ntiles;
         tile += (int64_t)gridDim.x * LNW) {
        const int64_t u0 = tile * 16 + g, u1 = u0 + 8;
        const bool v0 = u0 < a.sl.n_int, v1 = u1 < a.sl.n_int;
        LCell c0, c1;
        if (v0) lcell(a.sl, a.st, u0, c0, false);
        if (v1) lcell(a.sl, a.st, u1, c1, false);
        double p[NT][4];
        ld_c<S>(a.R, c0, c1, v0, v1, t, p);
        const double d0 = (jac && v0) ? a.st.dinv[c0.gi] : 1.0;
        const double d1 = (jac && v1) ? a.st.dinv[c1.gi] : 1.0;
        double pa[KS][2];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            pa[ks][0] = v0 ? a.P[c0.l * S + 4 * ks + t] : 0.0;
            pa[ks][1] = v1 ? a.P[c1.l * S + 4 * ks + t] : 0.0;
        }
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            p[n][0] *= d0;
            p[n][1] *= d0;
            p[n][2] *= d1;
            p[n][3] *= d1;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
                dmma_l(p[n], pa[ks][0], pa[ks][1], a.coef[(4 * ks + t) * RSC + 8 * n + g]);
        }
        st_c<S>(a.P, c0, c1, v0, v1, t, p);
    }
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

// fixed-order reduction over CTAs: out[e] = sum_b part[b][e]
__global__ void k_reduce(const double* __restrict__ part, int nb, int E, double* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += part[(int64_t)b * E + e];
        out[e] = s;
    }
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

template <int S>
__device__ void ctl_index(Ctl<S>* c, CSm<S>& sm) {
    if (threadIdx.x == 0) {
        int k = 0;
        for (int q = 0; q < S; ++q)
            if (c->act[q]) sm.idx[k++] = q;
        sm.sa = k;
        c->sa = k;
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
__global__ void __launch_bounds__(CBS) k_ctl_alpha(Ctl<S>* c, const double* red) {
    extern __shared__ __align__(16) unsigned char smraw_[];
    CSm<S>& sm = *reinterpret_cast<CSm<S>*>(smraw_);
    ctl_index(c, sm);
    ctl_solve(c, sm, red, c->s_old);
    if (threadIdx.x == 0) c->matvecs += sm.sa;
}

// red = [S_new | rr]: per-column recurrence test (solvers.cpp:582-590); beta
// (S_old^+ S_new) right away unless a true-residual verification is needed
template <int S>
__global__ void __launch_bounds__(CBS) k_ctl_update(Ctl<S>* c, const double* red, int m) {
    extern __shared__ __align__(16) unsigned char smraw_[];
    CSm<S>& sm = *reinterpret_cast<CSm<S>*>(smraw_);
    __shared__ int nver;
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
        if (threadIdx.x == 0) c->cmd = kCmdVerify;
        return;
    }
    ctl_index(c, sm);
    ctl_solve(c, sm, c->s_old, c->snew);  // beta
    for (int e = threadIdx.x; e < S * S; e += CBS) c->s_old[e] = c->snew[e];
    if (threadIdx.x == 0) c->cmd = kCmdPupdate;
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
    SweepArgs a;
    a.sl = sl;
    a.st = StencilPtr{op->diag, op->cx, op->cy, op->cz, op->dinv};
    a.B = Bloc;
    a.X = Xloc;
    a.R = Rloc;
    a.P = Ploc;
    a.W = Wloc;
    a.precond = cfg->precond;
    const int64_t ntiles = (sl.n_int + 15) / 16;
    int nb = ctx->num_sms;
    if (ctx->cg_max_ctas > 0 && nb > ctx->cg_max_ctas) nb = ctx->cg_max_ctas;
    if ((int64_t)nb * LNW > ntiles) nb = (int)((ntiles + LNW - 1) / LNW);
    if (nb < 1) nb = 1;
    constexpr int E = S * S + S;
    void *pPart, *pRed, *pCtl, *pHost;
    bk_status st;
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
        k_reduce<<<(e_count + 255) / 256, 256, 0, s>>>(a.part, nparts, e_count, red);
        ++ctx->launches;
        if (comm && comm->allreduce) comm->allreduce(comm->user, red, e_count, s);
    };
    auto halo = [&](double* v) {
        if (comm && comm->halo) comm->halo(comm->user, v, s);
    };
    auto read_cmd = [&](int* cmd, int* sa) -> bk_status {
        int h[2];
        BK_CUDA_TRY(ctx, cudaMemcpyAsync(h, &ctl->cmd, sizeof(int), cudaMemcpyDeviceToHost, s));
        BK_CUDA_TRY(ctx, cudaMemcpyAsync(h + 1, &ctl->sa, sizeof(int), cudaMemcpyDeviceToHost, s));
        BK_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        *cmd = h[0];
        *sa = h[1];
        return BK_OK;
    };
    const int tr_blocks = (int)((sl.n_int + (LBS / S) - 1) / (LBS / S) < 4L * ctx->num_sms
                                    ? (sl.n_int + (LBS / S) - 1) / (LBS / S)
                                    : 4L * ctx->num_sms);
    auto true_res = [&]() {
        k_true_res<S><<<tr_blocks, LBS, 0, s>>>(a);
        ++ctx->launches;
        reduce(S, tr_blocks);
    };

    const size_t sw = sizeof(LTile<S>) * LNW + (size_t)LNW * S * sizeof(double);
    const size_t cs = sizeof(CSm<S>);
    {
        const auto set = [&](const void* f, size_t b) {
            return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
        };
        BK_CUDA_TRY(ctx, set((const void*)k_anchor<S, kInit>, sw));
        BK_CUDA_TRY(ctx, set((const void*)k_anchor<S, kRestart>, sw));
        BK_CUDA_TRY(ctx, set((const void*)k_spmm_gram<S>, sw));
        BK_CUDA_TRY(ctx, set((const void*)k_update<S>, sw));
        BK_CUDA_TRY(ctx, set((const void*)k_ctl_init<S>, cs));
        BK_CUDA_TRY(ctx, set((const void*)k_ctl_alpha<S>, cs));
        BK_CUDA_TRY(ctx, set((const void*)k_ctl_update<S>, cs));
        BK_CUDA_TRY(ctx, set((const void*)k_ctl_verify<S>, cs));
    }
    k_anchor<S, kInit><<<nb, LBS, sw, s>>>(a);
    ++ctx->launches;
    reduce(E, nb);
    k_ctl_init<S><<<1, CBS, cs, s>>>(ctl, red, cfg->rel_tol);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    int cmd = 0, sa = 0;
    if ((st = read_cmd(&cmd, &sa)) != BK_OK) return st;
    for (int m = 1; m <= cfg->max_iter && sa > 0; ++m) {
        halo(a.P);
        k_spmm_gram<S><<<nb, LBS, sw, s>>>(a);
        ++ctx->launches;
        reduce(S * S, nb);
        k_ctl_alpha<S><<<1, CBS, cs, s>>>(ctl, red);
        ++ctx->launches;
        k_update<S><<<nb, LBS, sw, s>>>(a);
        ++ctx->launches;
        reduce(E, nb);
        k_ctl_update<S><<<1, CBS, cs, s>>>(ctl, red, m);
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaGetLastError());
        if ((st = read_cmd(&cmd, &sa)) != BK_OK) return st;
        if (cmd == kCmdVerify) {
            halo(a.X);
            true_res();
            k_ctl_verify<S><<<1, CBS, cs, s>>>(ctl, red);
            ++ctx->launches;
            if ((st = read_cmd(&cmd, &sa)) != BK_OK) return st;
            if (cmd == kCmdDone) break;
            if (cmd == kCmdRestart) {
                k_anchor<S, kRestart><<<nb, LBS, sw, s>>>(a);
                ++ctx->launches;
                reduce(E, nb);
                k_ctl_restart<S><<<1, CBS, 0, s>>>(ctl, red);
                ++ctx->launches;
                continue;
            }
        }
        k_pupdate<S><<<nb, LBS, 0, s>>>(a);
        ++ctx->launches;
    }
    // honest residuals for still-active columns
    BK_CUDA_TRY(ctx, cudaMemcpyAsync(&sa, &ctl->sa, sizeof(int), cudaMemcpyDeviceToHost, s));
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (sa > 0) {
        halo(a.X);
        true_res();
    }
    k_ctl_final<S><<<1, 32, 0, s>>>(ctl, red, drep);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    BK_CUDA_TRY(ctx, cudaMemcpyAsync(rep, drep, sizeof(CgReport), cudaMemcpyDeviceToHost, s));
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    return BK_OK;
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
    SweepArgs a;
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
    a.act = ctl->act;
    constexpr int E = S * S + S;
    const int nb = b->nb;
    cudaStream_t s = ctx->stream;
    const size_t sw = sizeof(LTile<S>) * LNW + (size_t)LNW * S * sizeof(double);
    const size_t cs = sizeof(CSm<S>);
    auto set = [&](const void* f, size_t bytes) {
        return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    };
    auto reduce = [&](int e_count, int nparts) {
        k_reduce<<<(e_count + 255) / 256, 256, 0, s>>>(b->part, nparts, e_count, b->red);
        ++ctx->launches;
    };
    const int tr_blocks = (int)((sl.n_int + (LBS / S) - 1) / (LBS / S) < 4L * ctx->num_sms
                                    ? (sl.n_int + (LBS / S) - 1) / (LBS / S)
                                    : 4L * ctx->num_sms);
    switch (step) {
        case BK_DD_INIT_SWEEP:
            BK_CUDA_TRY(ctx, set((const void*)k_anchor<S, kInit>, sw));
            k_anchor<S, kInit><<<nb, LBS, sw, s>>>(a);
            ++ctx->launches;
            reduce(E, nb);
            break;
        case BK_DD_CTL_INIT:
            BK_CUDA_TRY(ctx, set((const void*)k_ctl_init<S>, cs));
            k_ctl_init<S><<<1, CBS, cs, s>>>(ctl, b->red, cfg->rel_tol);
            ++ctx->launches;
            break;
        case BK_DD_SPMM:
            BK_CUDA_TRY(ctx, set((const void*)k_spmm_gram<S>, sw));
            k_spmm_gram<S><<<nb, LBS, sw, s>>>(a);
            ++ctx->launches;
            reduce(S * S, nb);
            break;
        case BK_DD_CTL_ALPHA:
            BK_CUDA_TRY(ctx, set((const void*)k_ctl_alpha<S>, cs));
            k_ctl_alpha<S><<<1, CBS, cs, s>>>(ctl, b->red);
            ++ctx->launches;
            break;
        case BK_DD_UPDATE:
            BK_CUDA_TRY(ctx, set((const void*)k_update<S>, sw));
            k_update<S><<<nb, LBS, sw, s>>>(a);
            ++ctx->launches;
            reduce(E, nb);
            break;
        case BK_DD_CTL_UPDATE:
            BK_CUDA_TRY(ctx, set((const void*)k_ctl_update<S>, cs));
            k_ctl_update<S><<<1, CBS, cs, s>>>(ctl, b->red, m);
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
            BK_CUDA_TRY(ctx, set((const void*)k_anchor<S, kRestart>, sw));
            k_anchor<S, kRestart><<<nb, LBS, sw, s>>>(a);
            ++ctx->launches;
            reduce(E, nb);
            break;
        case BK_DD_CTL_RESTART:
            k_ctl_restart<S><<<1, CBS, 0, s>>>(ctl, b->red);
            ++ctx->launches;
            break;
        case BK_DD_PUPDATE:
            k_pupdate<S><<<nb, LBS, 0, s>>>(a);
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

extern "C" {

bk_status bk_dd_sizes(bk_ctx* ctx, const bk_operator* op, int nyl, int S, int64_t* local_elems,
                      int* nb, int64_t* part_elems, int64_t* red_elems, int64_t* ctl_bytes) {
    if (!ctx || !op || nyl < 1 || nyl > op->ny) return BK_INVALID_CONFIG;
    if (S != 16 && S != 32 && S != 64)
        return bk::fail(ctx, BK_INVALID_CONFIG, "dd: kernel width must be 16, 32 or 64");
    const int64_t n_int = (int64_t)op->nx * nyl * op->nz;
    const int64_t ntiles = (n_int + 15) / 16;
    int b = ctx->num_sms;
    if ((int64_t)b * LNW > ntiles) b = (int)((ntiles + LNW - 1) / LNW);
    if (b < 1) b = 1;
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
