// Block conjugate gradient as ONE persistent cooperative sm_100a kernel —
// generic SIMT-FP64 variant (any width; the production path for S = 64).
// bk_block_cg_dmma.cu holds the DMMA variant used for S <= 32.
//
// Restates block_cg (solvers.cpp:452-665) without any host round trip per
// iteration. Each CTA owns a contiguous range of cells; block vectors live in
// HBM/L2 in the reference MultiVector layout (row-major n x S). Per iteration:
//
//   phase 1  W = A P (stencil, CSR-order FMA chain) and the CTA's partial of
//            G = P^T W                                  (spmm_gram_fixed :221-242)
//   reduce   fixed-order grid reduction; every CTA then solves alpha = G^+ S_old
//            redundantly (bitwise-identical in all CTAs) (:552)
//   phase 2  X += P alpha, R -= W alpha, rr_j = sum r^2, Z = D^-1 R,
//            partial S_new = R^T Z                      (update_fused_fixed :246-278)
//   reduce   per-column convergence test (:582-600); rare paths: true-residual
//            verification (:521-530), freeze/deflate (:602-614, as an active-column
//            mask instead of memory compaction), restart R = B - A X (:616-634)
//   phase 3  beta = S_old^+ S_new; P = Z + P beta       (p_update_fixed :281-296)
//
// Small s x s solves: Gauss-Jordan on [G | RHS] over the active (compacted)
// block; if any pivot falls near the reference's rank cutoff the exact
// diagonally pivoted Cholesky of solvers.cpp:347-426 runs instead, so
// rank-deficient blocks (duplicate / dependent columns) get zero coefficients
// beyond the numerical rank exactly as in the reference.
//
// Reductions never use floating-point atomics: per-thread sums in cell order,
// CTA sums in thread order, grid sums in CTA order — bitwise run-to-run
// deterministic for a fixed launch shape.
#include <cooperative_groups.h>

#include <cmath>

#include "bk_common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int BS = 256;

struct CgArgs {
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
};

template <int S>
struct Sm {
    double s_old[S * S];
    double mat[S * S];
    double coef[S * S];
    double red[S * S];
    double aug[2 * S * S + 2 * S];
    double vec[S];
    double bnorm[S];
    double fres[S];
    double stP[BS];
    double stW[BS];
    double stR[BS];
    double dpiv[S];
    int perm[S];
    int act[S];   // active flag per column
    int idx[S];   // compacted active index list
    int vflag[S];
    int conv[S];
    int sa;
    int fail;
    int rank;
};

// ---------------------------------------------------------------------------
// stencil helpers: (A V)[c][j] for row-major n x S V.
// ---------------------------------------------------------------------------
template <int S>
struct Geo {
    int nx, ny, nz;
    int64_t plane;
};

// CSR-order FMA chain (apply_block, discretize.cpp:57-71).
template <int S>
__device__ __forceinline__ double stencil_fma(const CgArgs& a, const double* __restrict__ V,
                                              int64_t c, int j, double& center) {
    const int64_t plane = (int64_t)a.nx * a.ny;
    const int ci = (int)c;
    const int ix = ci % a.nx;
    const int iy = (ci / a.nx) % a.ny;
    const int iz = ci / (a.nx * a.ny);
    const int64_t e = c * S + j;
    double acc = 0.0;
    if (iz > 0) acc = fma(-a.cz[c - plane], V[e - plane * S], acc);
    if (iy > 0) acc = fma(-a.cy[c - a.nx], V[e - (int64_t)a.nx * S], acc);
    if (ix > 0) acc = fma(-a.cx[c - 1], V[e - S], acc);
    center = V[e];
    acc = fma(a.diag[c], center, acc);
    if (ix < a.nx - 1) acc = fma(-a.cx[c], V[e + S], acc);
    if (iy < a.ny - 1) acc = fma(-a.cy[c], V[e + (int64_t)a.nx * S], acc);
    if (iz < a.nz - 1) acc = fma(-a.cz[c], V[e + plane * S], acc);
    return acc;
}

// Separate multiply + add (CsrMatrix::apply, discretize.cpp:39-51), used by
// the true-residual verification (true_rel_residual, solvers.cpp:68-78).
template <int S>
__device__ __forceinline__ double stencil_muladd(const CgArgs& a, const double* __restrict__ V,
                                                 int64_t c, int j) {
    const int64_t plane = (int64_t)a.nx * a.ny;
    const int ci = (int)c;
    const int ix = ci % a.nx;
    const int iy = (ci / a.nx) % a.ny;
    const int iz = ci / (a.nx * a.ny);
    const int64_t e = c * S + j;
    double acc = 0.0;
    if (iz > 0) acc = __dadd_rn(acc, __dmul_rn(-a.cz[c - plane], V[e - plane * S]));
    if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(-a.cy[c - a.nx], V[e - (int64_t)a.nx * S]));
    if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(-a.cx[c - 1], V[e - S]));
    acc = __dadd_rn(acc, __dmul_rn(a.diag[c], V[e]));
    if (ix < a.nx - 1) acc = __dadd_rn(acc, __dmul_rn(-a.cx[c], V[e + S]));
    if (iy < a.ny - 1) acc = __dadd_rn(acc, __dmul_rn(-a.cy[c], V[e + (int64_t)a.nx * S]));
    if (iz < a.nz - 1) acc = __dadd_rn(acc, __dmul_rn(-a.cz[c], V[e + plane * S]));
    return acc;
}

// ---------------------------------------------------------------------------
// CTA / grid reductions
// ---------------------------------------------------------------------------

// red[a*S + j] = sum over cell groups (in order) of acc[a] held by thread (j, cg).
template <int S>
__device__ __forceinline__ void cta_reduce_mat(const double (&acc)[S], double* red, int j, int cgi) {
    constexpr int NCG = BS / S;
    for (int r = 0; r < NCG; ++r) {
        if (cgi == r) {
#pragma unroll
            for (int q = 0; q < S; ++q) red[q * S + j] = r == 0 ? acc[q] : red[q * S + j] + acc[q];
        }
        __syncthreads();
    }
}

template <int S>
__device__ __forceinline__ void cta_reduce_vec(double v, double* out, int j, int cgi) {
    constexpr int NCG = BS / S;
    for (int r = 0; r < NCG; ++r) {
        if (cgi == r) out[j] = r == 0 ? v : out[j] + v;
        __syncthreads();
    }
}

// Publish this CTA's E partial values, reduce across CTAs in fixed order, and
// load the E reduced values into dst (smem). Two grid barriers.
__device__ void grid_reduce(cg::grid_group& grid, double* __restrict__ part,
                            double* __restrict__ redg, const double* src, int E, double* dst) {
    const int b = blockIdx.x, NB = gridDim.x;
    for (int e = threadIdx.x; e < E; e += BS) part[(int64_t)b * E + e] = src[e];
    grid.sync();
    const int e0 = (int)((int64_t)E * b / NB), e1 = (int)((int64_t)E * (b + 1) / NB);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = e0 + warp; e < e1; e += BS / 32) {
        double s = 0.0;
        for (int l = lane; l < NB; l += 32) s += __ldcg(part + (int64_t)l * E + e);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) __stcg(redg + e, s);
    }
    grid.sync();
    for (int e = threadIdx.x; e < E; e += BS) dst[e] = __ldcg(redg + e);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// small s x s solves (redundant in every CTA)
// ---------------------------------------------------------------------------

template <int S>
__device__ void build_index(Sm<S>& sm) {
    if (threadIdx.x == 0) {
        int k = 0;
        for (int q = 0; q < S; ++q)
            if (sm.act[q]) sm.idx[k++] = q;
        sm.sa = k;
    }
    __syncthreads();
}

// Reference PivotedCholesky(M).solve(RHS) on the compacted sa x sa block,
// sequential in thread 0 (rare path: rank-deficient blocks). M and RHS are
// symmetric; the upper triangle is read (mirror_upper, solvers.cpp:336-341).
template <int S>
__device__ void pivoted_cholesky_solve(Sm<S>& sm, const double* M, const double* RHS,
                                       double* out) {
    if (threadIdx.x == 0) {
        const int sa = sm.sa;
        double* L = sm.aug;            // sa x sa, stride S
        double* Y = sm.aug + S * S;    // sa x sa, stride S
        double* d = sm.dpiv;
        int* perm = sm.perm;
        auto Mv = [&](int p, int q) {
            const int a = sm.idx[p], b = sm.idx[q];
            return a <= b ? M[a * S + b] : M[b * S + a];
        };
        auto Rv = [&](int p, int q) {
            const int a = sm.idx[p], b = sm.idx[q];
            return a <= b ? RHS[a * S + b] : RHS[b * S + a];
        };
        double maxd = 0.0;
        for (int i = 0; i < sa; ++i) {
            perm[i] = i;
            d[i] = Mv(i, i);
            maxd = fmax(maxd, d[i]);
            for (int t = 0; t < sa; ++t) L[i * S + t] = 0.0;
        }
        const double cutoff = fmax(maxd * sa * 2.220446049250313e-16, 2.2250738585072014e-308);
        int rank = sa;
        for (int k = 0; k < sa; ++k) {
            int piv = k;
            for (int i = k + 1; i < sa; ++i)
                if (d[perm[i]] > d[perm[piv]]) piv = i;
            if (!(d[perm[piv]] > cutoff)) {
                rank = k;
                break;
            }
            const int tp = perm[k];
            perm[k] = perm[piv];
            perm[piv] = tp;
            for (int t = 0; t < k; ++t) {
                const double tv = L[k * S + t];
                L[k * S + t] = L[piv * S + t];
                L[piv * S + t] = tv;
            }
            const int pk = perm[k];
            const double lkk = sqrt(d[pk]);
            L[k * S + k] = lkk;
            for (int i = k + 1; i < sa; ++i) {
                const int pi = perm[i];
                double v = Mv(pi, pk);
                for (int t = 0; t < k; ++t) v -= L[i * S + t] * L[k * S + t];
                const double lik = v / lkk;
                L[i * S + k] = lik;
                d[pi] -= lik * lik;
            }
        }
        // forward L y = P rhs; backward L^T x = y, scattered through perm
        for (int k = 0; k < rank; ++k) {
            const int pk = perm[k];
            for (int q = 0; q < sa; ++q) {
                double v = Rv(pk, q);
                for (int t = 0; t < k; ++t) v -= L[k * S + t] * Y[t * S + q];
                Y[k * S + q] = v / L[k * S + k];
            }
        }
        for (int q = 0; q < S * S; ++q) out[q] = 0.0;
        // x rows in compact index space, then scatter to original columns
        for (int k = rank - 1; k >= 0; --k) {
            const int pk = perm[k];
            for (int q = 0; q < sa; ++q) {
                double v = Y[k * S + q];
                for (int t = k + 1; t < rank; ++t)
                    v -= L[t * S + k] * out[sm.idx[perm[t]] * S + sm.idx[q]];
                out[sm.idx[pk] * S + sm.idx[q]] = v / L[k * S + k];
            }
        }
        sm.rank = rank;
    }
    __syncthreads();
}

// out = M^+ RHS over the active block; zero rows/columns for inactive ones.
template <int S>
__device__ void small_solve(Sm<S>& sm, const double* M, const double* RHS, double* out) {
    const int sa = sm.sa;
    const int W2 = 2 * sa;
    double* aug = sm.aug;  // sa x 2sa, stride 2S
    for (int e = threadIdx.x; e < sa * W2; e += BS) {
        const int p = e / W2, q = e % W2;
        const int a = sm.idx[p];
        double v;
        if (q < sa) {
            const int b = sm.idx[q];
            v = a <= b ? M[a * S + b] : M[b * S + a];
        } else {
            const int b = sm.idx[q - sa];
            v = a <= b ? RHS[a * S + b] : RHS[b * S + a];
        }
        aug[p * 2 * S + q] = v;
    }
    if (threadIdx.x == 0) sm.fail = 0;
    __syncthreads();
    // reference rank cutoff (solvers.cpp:355-359); the fast path bails out
    // 1000x above it so every block it accepts has full numerical rank.
    double maxd = 0.0;
    for (int p = 0; p < sa; ++p) maxd = fmax(maxd, aug[p * 2 * S + p]);
    const double guard =
        1e3 * fmax(maxd * sa * 2.220446049250313e-16, 2.2250738585072014e-308);
    for (int k = 0; k < sa; ++k) {
        const double pk = aug[k * 2 * S + k];
        if (!(pk > guard)) {
            if (threadIdx.x == 0) sm.fail = 1;
            break;  // uniform: every thread reads the same pivot
        }
        const double rinv = 1.0 / pk;
        const int cols = W2 - k - 1;
        const int items = (sa - 1) * cols;
        for (int e = threadIdx.x; e < items; e += BS) {
            int p = e / cols;
            const int q = k + 1 + e % cols;
            p += (p >= k);
            const double f = aug[p * 2 * S + k] * rinv;
            aug[p * 2 * S + q] = fma(-f, aug[k * 2 * S + q], aug[p * 2 * S + q]);
        }
        __syncthreads();
    }
    __syncthreads();
    if (sm.fail) {
        pivoted_cholesky_solve<S>(sm, M, RHS, out);
        return;
    }
    for (int e = threadIdx.x; e < S * S; e += BS) out[e] = 0.0;
    __syncthreads();
    for (int e = threadIdx.x; e < sa * sa; e += BS) {
        const int p = e / sa, q = e % sa;
        out[sm.idx[p] * S + sm.idx[q]] = aug[p * 2 * S + sa + q] / aug[p * 2 * S + p];
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// the persistent kernel
// ---------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(BS, 1) block_cg_kernel(CgArgs a) {
    static_assert(BS % S == 0, "S must divide the CTA size");
    constexpr int NCG = BS / S;
    constexpr int E = S * S + S;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Sm<S>& sm = *reinterpret_cast<Sm<S>*>(smem_raw);

    const int tid = threadIdx.x;
    const int j = tid % S, cgi = tid / S;
    const int NB = gridDim.x, b = blockIdx.x;
    const int64_t c0 = a.n * b / NB, c1 = a.n * (b + 1) / NB;
    const bool jac = a.precond != 0;

    double acc[S];
    int64_t matvecs = 0;
    int iters = 0;

    // ---- init (solvers.cpp:468-519): X = 0, R = B, Z = D^-1 R, P = Z,
    //      bnorm, S_old = R^T Z
    {
#pragma unroll
        for (int q = 0; q < S; ++q) acc[q] = 0.0;
        double bn2 = 0.0;
        for (int64_t base = c0; base < c1; base += NCG) {
            const int64_t c = base + cgi;
            const bool v = c < c1;
            double bv = 0.0, z = 0.0;
            if (v) {
                const int64_t e = c * S + j;
                bv = a.B[e];
                a.X[e] = 0.0;
                a.R[e] = bv;
                z = jac ? a.dinv[c] * bv : bv;
                a.P[e] = z;
                bn2 = fma(bv, bv, bn2);
            }
            sm.stR[cgi * S + j] = bv;
            __syncthreads();
            if (v) {
#pragma unroll
                for (int q = 0; q < S; ++q) acc[q] = fma(sm.stR[cgi * S + q], z, acc[q]);
            }
            __syncthreads();
        }
        cta_reduce_mat<S>(acc, sm.red, j, cgi);
        cta_reduce_vec<S>(bn2, sm.vec, j, cgi);
        // pack [mat | vec] contiguously in aug as the reduction source
        for (int e = tid; e < S * S; e += BS) sm.aug[e] = sm.red[e];
        if (tid < S) sm.aug[S * S + tid] = sm.vec[tid];
        __syncthreads();
        grid_reduce(grid, a.part, a.red, sm.aug, E, sm.aug + E);
        for (int e = tid; e < S * S; e += BS) sm.s_old[e] = sm.aug[E + e];
        if (tid < S) {
            const double bn = sqrt(sm.aug[E + S * S + tid]);
            sm.bnorm[tid] = bn;
            sm.act[tid] = bn != 0.0;   // zero right-hand sides: x = 0 (:478-485)
            sm.conv[tid] = bn == 0.0;
            sm.fres[tid] = 0.0;
        }
        __syncthreads();
        build_index<S>(sm);
    }

    for (int m = 1; m <= a.max_iter && sm.sa > 0; ++m) {
        // ---- phase 1: W = A P, G = P^T W
#pragma unroll
        for (int q = 0; q < S; ++q) acc[q] = 0.0;
        for (int64_t base = c0; base < c1; base += NCG) {
            const int64_t c = base + cgi;
            const bool v = c < c1;
            double w = 0.0, pc = 0.0;
            if (v) {
                w = stencil_fma<S>(a, a.P, c, j, pc);
                a.W[c * S + j] = w;
            }
            sm.stP[cgi * S + j] = pc;
            __syncthreads();
            if (v) {
#pragma unroll
                for (int q = 0; q < S; ++q) acc[q] = fma(sm.stP[cgi * S + q], w, acc[q]);
            }
            __syncthreads();
        }
        cta_reduce_mat<S>(acc, sm.red, j, cgi);
        grid_reduce(grid, a.part, a.red, sm.red, S * S, sm.mat);
        matvecs += sm.sa;
        small_solve<S>(sm, sm.mat, sm.s_old, sm.coef);  // alpha

        // ---- phase 2: X += P alpha, R -= W alpha, rr, Z, S_new
#pragma unroll
        for (int q = 0; q < S; ++q) acc[q] = 0.0;
        double rr = 0.0;
        for (int64_t base = c0; base < c1; base += NCG) {
            const int64_t c = base + cgi;
            const bool v = c < c1;
            const int64_t e = c * S + j;
            sm.stP[cgi * S + j] = v ? a.P[e] : 0.0;
            sm.stW[cgi * S + j] = v ? a.W[e] : 0.0;
            __syncthreads();
            double r = 0.0, z = 0.0;
            if (v) {
                double x = a.X[e];
                r = a.R[e];
#pragma unroll
                for (int t = 0; t < S; ++t) {
                    const double al = sm.coef[t * S + j];
                    x = fma(sm.stP[cgi * S + t], al, x);
                    r = fma(-sm.stW[cgi * S + t], al, r);
                }
                a.X[e] = x;
                a.R[e] = r;
                rr = fma(r, r, rr);
                z = jac ? a.dinv[c] * r : r;
            }
            sm.stR[cgi * S + j] = r;
            __syncthreads();
            if (v) {
#pragma unroll
                for (int q = 0; q < S; ++q) acc[q] = fma(sm.stR[cgi * S + q], z, acc[q]);
            }
        }
        __syncthreads();
        cta_reduce_mat<S>(acc, sm.red, j, cgi);
        cta_reduce_vec<S>(rr, sm.vec, j, cgi);
        for (int e = tid; e < S * S; e += BS) sm.aug[e] = sm.red[e];
        if (tid < S) sm.aug[S * S + tid] = sm.vec[tid];
        __syncthreads();
        grid_reduce(grid, a.part, a.red, sm.aug, E, sm.aug + E);
        for (int e = tid; e < S * S; e += BS) sm.mat[e] = sm.aug[E + e];  // S_new
        if (tid < S) sm.vec[tid] = sm.aug[E + S * S + tid];              // rr
        __syncthreads();
        iters = m;

        // ---- convergence control (solvers.cpp:582-634)
        int nver = 0;
        for (int q = 0; q < S; ++q) {
            const int f = sm.act[q] && (sqrt(sm.vec[q]) / sm.bnorm[q] <= a.tol);
            nver += f;
        }
        bool restart = false;
        if (nver > 0) {
            if (tid < S) sm.vflag[tid] = sm.act[tid] && (sqrt(sm.vec[tid]) / sm.bnorm[tid] <= a.tol);
            __syncthreads();
            // true residual ||b - A x|| for flagged columns (one matvec each)
            double rs = 0.0;
            for (int64_t base = c0; base < c1; base += NCG) {
                const int64_t c = base + cgi;
                if (c < c1) {
                    const double rv = a.B[c * S + j] - stencil_muladd<S>(a, a.X, c, j);
                    rs += rv * rv;
                }
            }
            cta_reduce_vec<S>(rs, sm.red, j, cgi);
            grid_reduce(grid, a.part, a.red, sm.red, S, sm.red + S);
            matvecs += nver;
            if (tid == 0) {
                for (int q = 0; q < S; ++q) {
                    if (!sm.vflag[q]) continue;
                    const double rt = sqrt(sm.red[S + q]) / sm.bnorm[q];
                    if (rt <= a.tol) {
                        sm.act[q] = 0;       // freeze: X column stays as published
                        sm.conv[q] = 1;
                        sm.fres[q] = rt;
                    } else {
                        sm.fail = 2;         // mark restart
                    }
                }
            }
            __syncthreads();
            restart = sm.fail == 2;
            __syncthreads();
            if (tid == 0) sm.fail = 0;
            build_index<S>(sm);
            if (sm.sa == 0) break;
        }
        if (restart) {
            // re-anchor: R = B - A X, P = Z, S_old = R^T Z (:621-633)
#pragma unroll
            for (int q = 0; q < S; ++q) acc[q] = 0.0;
            for (int64_t base = c0; base < c1; base += NCG) {
                const int64_t c = base + cgi;
                const bool v = c < c1;
                double r = 0.0, z = 0.0;
                if (v) {
                    double dummy;
                    const int64_t e = c * S + j;
                    r = a.B[e] - stencil_fma<S>(a, a.X, c, j, dummy);
                    z = jac ? a.dinv[c] * r : r;
                    a.R[e] = r;
                }
                sm.stR[cgi * S + j] = r;
                __syncthreads();
                if (v) {
                    a.P[c * S + j] = z;
#pragma unroll
                    for (int q = 0; q < S; ++q) acc[q] = fma(sm.stR[cgi * S + q], z, acc[q]);
                }
                __syncthreads();
            }
            cta_reduce_mat<S>(acc, sm.red, j, cgi);
            grid_reduce(grid, a.part, a.red, sm.red, S * S, sm.s_old);
            matvecs += sm.sa;
            continue;
        }

        // ---- phase 3: beta = S_old^+ S_new, S_old = S_new, P = Z + P beta
        small_solve<S>(sm, sm.s_old, sm.mat, sm.coef);
        for (int e = tid; e < S * S; e += BS) sm.s_old[e] = sm.mat[e];
        for (int64_t base = c0; base < c1; base += NCG) {
            const int64_t c = base + cgi;
            const bool v = c < c1;
            const int64_t e = c * S + j;
            sm.stP[cgi * S + j] = v ? a.P[e] : 0.0;
            __syncthreads();
            if (v) {
                double p = jac ? a.dinv[c] * a.R[e] : a.R[e];
#pragma unroll
                for (int t = 0; t < S; ++t) p = fma(sm.stP[cgi * S + t], sm.coef[t * S + j], p);
                a.P[e] = p;
            }
            __syncthreads();
        }
        grid.sync();
    }

    // ---- exit: honest residuals for still-active columns (:655-661)
    if (sm.sa > 0) {
        double rs = 0.0;
        for (int64_t base = c0; base < c1; base += NCG) {
            const int64_t c = base + cgi;
            if (c < c1) {
                const double rv = a.B[c * S + j] - stencil_muladd<S>(a, a.X, c, j);
                rs += rv * rv;
            }
        }
        cta_reduce_vec<S>(rs, sm.red, j, cgi);
        grid_reduce(grid, a.part, a.red, sm.red, S, sm.red + S);
        matvecs += sm.sa;
        if (tid < S && sm.act[tid]) {
            const double rt = sqrt(sm.red[S + tid]) / sm.bnorm[tid];
            sm.fres[tid] = rt;
            sm.conv[tid] = rt <= a.tol;
        }
        __syncthreads();
    }
    if (b == 0 && tid == 0) {
        a.rep->iterations = iters;
        a.rep->matvecs = matvecs;
        for (int q = 0; q < S; ++q) {
            a.rep->final_res[q] = sm.fres[q];
            a.rep->converged[q] = (char)sm.conv[q];
        }
    }
}

template <int S>
bk_status run_block_cg(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                       const bk_solver_cfg* cfg, double* X, bk::CgReport* rep) {
    using namespace bk;
    const int64_t n = op->n;
    const size_t vec_bytes = (size_t)n * S * sizeof(double);
    auto kern = block_cg_kernel<S>;
    const size_t smem = sizeof(Sm<S>);
    BK_CUDA_TRY(ctx, bk::set_max_smem((const void*)kern, smem));
    int occ = 0;
    BK_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BS, smem));
    if (occ < 1) return fail(ctx, BK_INTERNAL, "block_cg kernel cannot be resident");
    occ = occ > 4 ? 4 : occ;
    int64_t nb = (int64_t)occ * ctx->num_sms;
    if (ctx->cg_max_ctas > 0 && nb > ctx->cg_max_ctas) nb = ctx->cg_max_ctas;
    const int64_t min_cells = 2 * (BS / S);
    if (nb * min_cells > n) nb = (n + min_cells - 1) / min_cells;
    if (nb < 1) nb = 1;
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
    if ((st = workspace(ctx, kSlotCgCtl, sizeof(CgReport), &pRep)) != BK_OK) return st;
    if (padded) {
        if ((st = workspace(ctx, kSlotCgB, vec_bytes, &pB)) != BK_OK) return st;
        if ((st = workspace(ctx, kSlotCgX, vec_bytes, &pX)) != BK_OK) return st;
        BK_CUDA_TRY(ctx, launch_pad_cols(ctx, B, s, (double*)pB, S, n));
    } else {
        pB = const_cast<double*>(B);
        pX = X;
    }
    CgArgs a;
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
    void* args[] = {&a};
    BK_CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)nb), dim3(BS),
                                                 args, smem, ctx->stream));
    ++ctx->launches;
    if (padded) {
        BK_CUDA_TRY(ctx, launch_pad_cols(ctx, (const double*)pX, S, X, s, n));
    }
    {
        const bk_status rs = read_small(ctx, rep, pRep, sizeof(CgReport));
        if (rs != BK_OK) return rs;
    }
    return BK_OK;
}

}  // namespace

namespace bk {

// Generic (SIMT) path: any kernel width; used for S = 64 and as a cross-check
// of the DMMA path (BK_CG_GENERIC=1).
bk_status block_cg_generic(bk_ctx* ctx, const bk_operator* op, const double* B, int s,
                           const bk_solver_cfg* cfg, double* X, CgReport* rep) {
    if (s <= 8) return run_block_cg<8>(ctx, op, B, s, cfg, X, rep);
    if (s <= 16) return run_block_cg<16>(ctx, op, B, s, cfg, X, rep);
    if (s <= 32) return run_block_cg<32>(ctx, op, B, s, cfg, X, rep);
    if (s <= 64) return run_block_cg<64>(ctx, op, B, s, cfg, X, rep);
    return fail(ctx, BK_INVALID_CONFIG, "block_cg: s > 64 is not supported on device");
}

}  // namespace bk
