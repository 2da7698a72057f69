// Shared s x s solve and shared-memory strides for the block-CG kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bkcg {

static __device__ long long* g_ss_prof = nullptr;  // debug: small-solve step timestamps

// Shared-memory row strides chosen for conflict-free 64-bit fragment access:
// S + 4 makes the DMMA fragment loads [(4k + t) * RS + 8n + g] hit 16 distinct
// 8-byte bank slots per half-warp; the odd 2S + 1 makes the Gauss-Jordan
// column walk aug[i][p] conflict-free.
template <int S>
struct Strides {
    static constexpr int RS = S + 4;      // tile / coefficient rows
    static constexpr int LD = 2 * S + 1;  // augmented [M | RHS] rows
};

// Warp-wide argmax of non-negative doubles through their IEEE bit patterns
// (monotone for x >= 0). The low 6 bits of the pattern are replaced by
// (63 - index), so two integer REDUX steps return both the winner and (up to
// the 2^-46 relative truncation) its value; exact ties keep the lowest index,
// as the reference's strict '>' scan does. key = 0 excludes an entry.
__device__ __forceinline__ unsigned long long pivot_key(double v, int idx) {
    return v > 0.0 ? (((unsigned long long)__double_as_longlong(v) & ~63ull) |
                      (unsigned long long)(63 - idx))
                   : 0ull;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long key) {
    const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
    const unsigned hi = __reduce_max_sync(0xffffffffu, khi);
    const unsigned lo = __reduce_max_sync(0xffffffffu, khi == hi ? klo : 0u);
    return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ unsigned long long pos_bits(double v) {
    return v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
}

// out = M^+ RHS on the active block (zero rows/columns elsewhere), the
// semantics of PivotedCholesky(M).solve(RHS) (solvers.cpp:347-414): diagonal
// pivoting on the largest remaining Schur-complement diagonal, rank cutoff
// max(max_diag * s * eps, DBL_MIN), directions beyond the numerical rank get
// zero coefficients. Computed as Gauss-Jordan on [M | RHS] with that pivot
// sequence (the trailing block of Gauss-Jordan IS the Cholesky Schur
// complement, so pivots and rank decisions coincide). One barrier per pivot;
// every warp redundantly tracks the Schur diagonal in registers and searches
// the next pivot while the block update of the current one is in flight.
// SMT: any shared-memory struct with int sa, rank, idx[S]; double aug[S*LD+2S].
// NWS: warps that run the pivot loop (the others wait at the final barrier);
// fewer warps = a cheaper per-pivot barrier (named barrier 1, or __syncwarp
// for one warp) against more rows per warp.
template <int S, int BS, bool PROF = false, int VAR = 0, int NWS = BS / 32, class SMT>
__device__ void small_solve_t(SMT& sm, const double* M, const double* RHS, double* out) {
    long long* const pr = PROF ? g_ss_prof : nullptr;
    auto stamp = [&](int k) {
        if (PROF && threadIdx.x == 0) pr[k] = clock64();
    };
    constexpr int NWA = BS / 32;  // all warps: fill and output
    static_assert(NWS >= 1 && NWS <= NWA, "participating warps");
    auto wbar = []() {
        if (NWS == NWA)
            __syncthreads();
        else if (NWS == 1)
            __syncwarp();
        else
            asm volatile("bar.sync 1, %0;" ::"n"(NWS * 32) : "memory");
    };
    constexpr int NW = NWS;
    constexpr int LD = Strides<S>::LD;
    constexpr int RS = Strides<S>::RS;
    constexpr int R = (S + 31) / 32;  // diagonal entries per lane (index lane + 32 r)
    static_assert(R <= 2, "S <= 64");
    const int sa = sm.sa;
    double* aug = sm.aug;
    unsigned long long donem = 0ull;  // compacted indices already used as pivots
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // rows by warp, columns by lane: no integer division, conflict-free rows
    for (int i = warp; i < sa; i += NWA) {
        const int a = sm.idx[i];
        for (int q = lane; q < 2 * sa; q += 32) {
            double v;
            if (q < sa) {
                const int b = sm.idx[q];
                v = a <= b ? M[a * S + b] : M[b * S + a];
            } else {
                const int b = sm.idx[q - sa];
                v = a <= b ? RHS[a * S + b] : RHS[b * S + a];
            }
            aug[i * LD + q] = v;
        }
    }
    __syncthreads();
    unsigned long long* const shared_done = reinterpret_cast<unsigned long long*>(aug + S * LD);
    int rank = 0;
    if (warp < NWS) {
    double dg[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        dg[r] = i < sa ? aug[i * LD + i] : 0.0;
    }
    auto search = [&](unsigned long long excl) -> unsigned long long {
        unsigned long long key = 0ull;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = lane + 32 * r;
            const unsigned long long kk = (i < sa && !((excl >> i) & 1ull)) ? pivot_key(dg[r], i) : 0ull;
            key = kk > key ? kk : key;
        }
        return warp_max_u64(key);
    };
    stamp(0);
    unsigned long long best = search(0ull);
    // max_diag of the active block (the reference clamps its scan at 0)
    const int im = best ? 63 - (int)(best & 63ull) : -1;
    const double maxd = im >= 0 ? aug[im * LD + im] : 0.0;
    const double cutoff = fmax(maxd * sa * 2.220446049250313e-16, 2.2250738585072014e-308);
    // exact value of the pivot encoded in `key` (the key is truncated in its
    // low 6 bits), held in lane (p & 31) of dg
    auto pivot_of = [&](unsigned long long key, int& p, double& pv) {
        p = key ? 63 - (int)(key & 63ull) : -1;
        const int src = p < 0 ? 0 : (p & 31);
        pv = __shfl_sync(0xffffffffu, dg[0], src);
        if (R > 1) {
            const double pv1 = __shfl_sync(0xffffffffu, dg[R - 1], src);
            if (p >= 32) pv = pv1;
        }
        if (p < 0) pv = 0.0;
    };
    int p;
    double pv;
    pivot_of(best, p, pv);
    double rinv = __drcp_rn(pv);
    stamp(1);
    constexpr int RPW = (S + NW - 1) / NW;    // rows per warp
    constexpr int CPL = (2 * S + 31) / 32;    // columns per lane
    double* const pivv = aug + S * LD + 1;  // pivot value of each pivoted row
    while (p >= 0 && pv > cutoff) {           // uniform: beyond the rank -> stop
        donem |= 1ull << p;
        if (threadIdx.x == 0) pivv[p] = pv;
        // operands of this pivot's block update and of the Schur-diagonal
        // update (row p and column p are not written by this step)
        double apq[CPL], fi[RPW], aiq[RPW][CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int q = lane + 32 * c;
            apq[c] = q < 2 * sa ? aug[p * LD + q] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int i = warp + NW * r;
            fi[r] = i < sa ? aug[i * LD + p] : 0.0;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const int q = lane + 32 * c;
                aiq[r][c] = (i < sa && q < 2 * sa) ? aug[i * LD + q] : 0.0;
            }
        }
        double colp[R], rowp[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = lane + 32 * r;
            colp[r] = i < sa ? aug[i * LD + p] : 0.0;
            rowp[r] = i < sa ? aug[p * LD + i] : 0.0;
        }
        // block update (issued first so it overlaps the pivot search below);
        // branch-free (predicated stores / selects: divergent `continue`s here
        // compiled to a reconvergence barrier per element)
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int i = warp + NW * r;
            const bool row_ok = i < sa && i != p;
            const double f = fi[r] * rinv;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                // columns of earlier pivots are updated too (they feed only
                // themselves; pivoted rows take their diagonal from pivv), the
                // pivot column itself is not (other threads read it this step)
                const int q = lane + 32 * c;
                const bool ok = row_ok && q < 2 * sa && q != p;
                const double nv = fma(-f, apq[c], aiq[r][c]);
                if (ok) aug[i * LD + q] = nv;
            }
        }
        // Schur diagonal after this pivot (same arithmetic as aug[i][i] above)
        // and the next pivot with its reciprocal, before the barrier
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = lane + 32 * r;
            const double nd = fma(-(colp[r] * rinv), rowp[r], dg[r]);
            dg[r] = (i < sa && !((donem >> i) & 1ull)) ? nd : dg[r];
        }
        unsigned long long nb = search(donem);
        if (VAR == 2) nb = (p + 1 < sa) ? ((1ull << 32) | (unsigned long long)(63 - (p + 1))) : 0ull;
        int pn;
        double pvn;
        pivot_of(nb, pn, pvn);
        const double rn = __drcp_rn(pvn > 0.0 ? pvn : 1.0);
        ++rank;
        if (VAR != 3) wbar();
        stamp(2 + rank);
        p = pn;
        pv = pvn;
        rinv = rn;
    }
    if (NWS < NWA && threadIdx.x == 0) *shared_done = donem;
    }  // warp < NWS
    for (int e = threadIdx.x; e < S * RS; e += BS) out[e] = 0.0;
    __syncthreads();
    if (NWS < NWA) donem = *shared_done;
    for (int i = warp; i < sa; i += NWA) {
        if (!((donem >> i) & 1ull)) continue;
        const double di = __drcp_rn(aug[S * LD + 1 + i]);  // pivv[i] = aug[i][i] at its pivot
        for (int q = lane; q < sa; q += 32) out[sm.idx[i] * RS + sm.idx[q]] = aug[i * LD + sa + q] * di;
    }
    if (threadIdx.x == 0) sm.rank = rank;
    __syncthreads();
    stamp(63);
}


// Register-resident variant for S = 64 and 512 threads (the multi-kernel
// engine's control kernels): the same pivot sequence, rank cutoff and
// per-element arithmetic as small_solve_t (bitwise the same result), but the
// augmented [M | RHS] block lives in registers — warp w holds rows w + 16 a,
// lane l columns l + 32 b (a, b < 4) — so a pivot step moves only the pivot
// row and column through shared memory (published by their owners into a
// double buffer). One barrier per pivot; every warp tracks the Schur diagonal
// and finds the next pivot redundantly, as small_solve_t.
// The block update is unconditional (a predicated update per element made
// the loop issue-bound on integer / select work): entries small_solve_t
// leaves alone are either restored (the pivot row, from the published copy)
// or never read again (columns of earlier pivots feed only themselves; the
// diagonal of a pivoted row is taken from the recorded pivot value, which is
// the same number — the Schur-diagonal recurrence uses aug[i][i]'s arithmetic).
// VAR (timing experiments only): 1 no block update, 2 fixed pivot order,
// 3 no barrier, 4 no reciprocal
// NWR: warps in the pivot loop (warp w < NWR holds rows w + NWR a); the
// others wait at the final barrier. Fewer warps = less replicated pivot
// bookkeeping per pivot against more update work per thread.
template <int S, int BS, int VAR = 0, int NWR = 16, class SMT>
__device__ void small_solve_reg(SMT& sm, const double* M, const double* RHS, double* out) {
    static_assert(S == 64 && BS >= NWR * 32 && (NWR == 4 || NWR == 8 || NWR == 16),
                  "register layout: NWR warps x 64 / NWR rows, 32 lanes x 4 columns");
    constexpr int RS = Strides<S>::RS;
    constexpr int NR = S / NWR, NC = 4;     // rows / columns per thread
    auto wbar = []() {
        if (NWR == BS / 32)
            __syncthreads();
        else
            asm volatile("bar.sync 1, %0;" ::"n"(NWR * 32) : "memory");
    };
    constexpr int BUF = 2 * S + S;          // pivot row (2S) | pivot column (S)
    const int sa = sm.sa;
    double* const pbuf = sm.aug;            // 2 x BUF doubles
    double* const pivv = sm.aug + 2 * BUF;  // pivot value of each pivoted row
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int rank = 0;
    unsigned long long donem = 0ull;
    if (warp < NWR) {
    double v[NR][NC];
#pragma unroll
    for (int a = 0; a < NR; ++a) {
        const int i = warp + NWR * a;
#pragma unroll
        for (int b = 0; b < NC; ++b) {
            const int q = lane + 32 * b;
            double x = 0.0;
            if (i < sa && q < 2 * sa) {
                const int ai = sm.idx[i];
                if (q < sa) {
                    const int bq = sm.idx[q];
                    x = ai <= bq ? M[ai * S + bq] : M[bq * S + ai];
                } else {
                    const int bq = sm.idx[q - sa];
                    x = ai <= bq ? RHS[ai * S + bq] : RHS[bq * S + ai];
                }
            }
            v[a][b] = x;
        }
    }
    double dg[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int i = lane + 32 * r;
        dg[r] = i < sa ? M[sm.idx[i] * S + sm.idx[i]] : 0.0;  // aug[i][i]
    }
    auto search = [&](unsigned long long excl) -> unsigned long long {
        unsigned long long key = 0ull;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int i = lane + 32 * r;
            const unsigned long long kk = (i < sa && !((excl >> i) & 1ull)) ? pivot_key(dg[r], i) : 0ull;
            key = kk > key ? kk : key;
        }
        return warp_max_u64(key);
    };
    auto pivot_of = [&](unsigned long long key, int& p, double& pv) {
        p = key ? 63 - (int)(key & 63ull) : -1;
        const int src = p < 0 ? 0 : (p & 31);
        const double p0 = __shfl_sync(0xffffffffu, dg[0], src);
        const double p1 = __shfl_sync(0xffffffffu, dg[1], src);
        pv = p < 0 ? 0.0 : (p >= 32 ? p1 : p0);
    };
    // owners of row p / column p write them into buffer `buf` (p < 64, so
    // column p is column p & 31 of register block b = p >> 5 <= 1)
    auto publish = [&](int p, int buf) {
        double* rb = pbuf + buf * BUF;
        if (warp == p % NWR) {
            const int ap = p / NWR;
#pragma unroll
            for (int b = 0; b < NC; ++b) {
                double x = v[0][b];
#pragma unroll
                for (int a = 1; a < NR; ++a) x = a == ap ? v[a][b] : x;
                rb[lane + 32 * b] = x;
            }
        }
        if (lane == (p & 31)) {
            const bool hi = p >= 32;
#pragma unroll
            for (int a = 0; a < NR; ++a) rb[2 * S + warp + NWR * a] = hi ? v[a][1] : v[a][0];
        }
    };
    int p;
    double pv;
    const unsigned long long best = search(0ull);
    pivot_of(best, p, pv);
    const double cutoff = fmax(pv * sa * 2.220446049250313e-16, 2.2250738585072014e-308);
    double rinv = __drcp_rn(pv);
    int buf = 0;
    if (p >= 0) publish(p, 0);
    wbar();
    while (p >= 0 && pv > cutoff) {  // uniform
        donem |= 1ull << p;
        if (threadIdx.x == 0) pivv[p] = pv;
        const double* rb = pbuf + buf * BUF;
        double rowp[NC], colp[NR], dgc[2], dgr[2];
#pragma unroll
        for (int b = 0; b < NC; ++b) rowp[b] = rb[lane + 32 * b];
#pragma unroll
        for (int a = 0; a < NR; ++a) colp[a] = rb[2 * S + warp + NWR * a];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            dgc[r] = rb[2 * S + lane + 32 * r];
            dgr[r] = rb[lane + 32 * r];
        }
        if (VAR != 1) {
#pragma unroll
            for (int a = 0; a < NR; ++a) {
                const double f = colp[a] * rinv;
#pragma unroll
                for (int b = 0; b < NC; ++b) v[a][b] = fma(-f, rowp[b], v[a][b]);
            }
            if (warp == p % NWR) {  // the pivot row is not updated
                const int ap = p / NWR;
#pragma unroll
                for (int a = 0; a < NR; ++a)
#pragma unroll
                    for (int b = 0; b < NC; ++b) v[a][b] = a == ap ? rowp[b] : v[a][b];
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int i = lane + 32 * r;
            const double nd = fma(-(dgc[r] * rinv), dgr[r], dg[r]);
            dg[r] = (i < sa && !((donem >> i) & 1ull)) ? nd : dg[r];
        }
        int pn;
        double pvn;
        unsigned long long nk = search(donem);
        if (VAR == 2) nk = (p + 1 < sa) ? ((1ull << 62) | (unsigned long long)(63 - (p + 1))) : 0ull;
        pivot_of(nk, pn, pvn);
        if (VAR == 2) pvn = fmax(pvn, 1.0);
        ++rank;
        buf ^= 1;
        if (pn >= 0 && pvn > cutoff) publish(pn, buf);
        if (VAR != 3) wbar();
        p = pn;
        pv = pvn;
        rinv = VAR == 4 ? pvn : __drcp_rn(pvn > 0.0 ? pvn : 1.0);
    }
    // the RHS block, scaled by the pivoted rows' diagonals, to registers'
    // owners' output rows after the zero fill below
    for (int e = threadIdx.x; e < S * RS; e += NWR * 32) out[e] = 0.0;
    wbar();
#pragma unroll
    for (int a = 0; a < NR; ++a) {
        const int i = warp + NWR * a;  // warp-uniform
        if (i >= sa || !((donem >> i) & 1ull)) continue;
        const double di = __drcp_rn(pivv[i]);  // aug[i][i]
#pragma unroll
        for (int b = 0; b < NC; ++b) {
            const int q = lane + 32 * b - sa;
            if (q >= 0 && q < sa) out[sm.idx[i] * RS + sm.idx[q]] = v[a][b] * di;
        }
    }
    }  // warp < NWR
    if (threadIdx.x == 0) sm.rank = rank;
    __syncthreads();
}
}  // namespace bkcg
