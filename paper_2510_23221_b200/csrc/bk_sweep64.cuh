// Update sweep for S = 64 (BASELINE config 5), warp-specialised.
//
// Included by bk_block_cg_large.cu after its sweep helpers. Phase 2 of
// block_cg (solvers.cpp:557-564; update_fused_fixed :246-278 for s <= 16,
// add_product / gram :199-211, :636-640 above): R -= W alpha, rr_j = sum r^2,
// Z = D^-1 R, S_new = R^T Z — with X += P alpha deferred to the P update.
//
// At S = 64 this sweep is FP64-pipe bound, not HBM bound: per 16-cell run it
// moves 24 KB but issues 128 m16n8k4 DMMAs for R -= W alpha and 80 for the
// upper-triangle Gram (13.3 kflop per cell; the B200 FP64 tensor rate is
// ~37 TFLOP/s, measured, scripts/dmma_tput.cu, shared with SIMT DFMA). The
// design keeps the FP64 pipe fed:
//   * one CTA per SM: 3 teams of 4 warps (12 warps, 3 per SM sub-partition,
//     so up to 168 registers per thread);
//   * each team's leader thread streams the team's next runs (W and R as four
//     16-column panels each, TMA 2D tensor copies with 128-byte swizzle, plus
//     the run's D^-1 by a bulk copy) into the team's ring of stages, one full
//     mbarrier per stage; a stage is refilled right after the team barrier
//     that proves all four warps consumed it — no other loads are issued;
//   * a team owns one run at a time, warp w of the team the output columns
//     16w .. 16w + 15 (two n-tiles; alpha fragments from shared memory);
//     teams synchronise only among their own 128 threads (named barriers), so
//     the teams drift and overlap one another's DMMA, epilogue and wait
//     phases;
//   * after the update the team stages R (same swizzle) and each warp
//     accumulates 5 of the 20 upper 16 x 8 Gram tiles of R^T D^-1 R.
// Fixed group-to-team assignment and a fixed-order sum of the teams' partials:
// run-to-run deterministic.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

namespace sweep64 {

constexpr int kTeams = 3;  // 13 warps: 4 per SMSP at most -> up to 128 registers
constexpr int kTeamWarps = 4;
constexpr int kConsumers = kTeams * kTeamWarps * 32;  // 384
constexpr int kThreads = kConsumers + 32;               // + producer warp
constexpr int kStages = 3;                              // per team
constexpr int kPanelBytes = 16 * 128;                   // 16 rows x 16 doubles
constexpr int kArrBytes = 4 * kPanelBytes;              // one array of a run: 8 KB
constexpr int kStageBytes = 2 * kArrBytes;              // W, R

struct Smem {
    unsigned char stage[kTeams][kStages][kStageBytes];  // 1024-aligned
    unsigned char rstage[kTeams][2][kArrBytes];          // updated R of a run (Gram input)
    double alpha[64 * 64];                               // alpha, swizzled (alpha_at)
    double dinv[kTeams][kStages][16];                    // D^-1 of each stage's run
    unsigned long long full[kTeams][kStages];
};
constexpr size_t smem_bytes() { return sizeof(Smem) + 1024; }

// element (row r, column c) of a 16-row, 64-column array stored as four
// 128B-swizzled 16-column panels: the 16-byte chunk (c % 16) / 2 of row r
// sits at chunk ((c % 16) / 2) ^ (r % 8)
__device__ __forceinline__ int swz(int r, int c) {
    return (c >> 4) * kPanelBytes + r * 128 + ((((c & 15) >> 1) ^ (r & 7)) << 4) + ((c & 1) << 3);
}
// DMMA row g (0..7) of an m-tile <-> cell pi(g) of the run (rows g + 8 <->
// pi(g) + 8): the 3-bit reversal makes the swizzle keys of the 8 lanes of a
// 128-bit access (g = 2j, 2j + 1) differ in bit 2 and those of a half-warp's
// 64-bit access (g = 0..3 or 4..7) all even or all odd — conflict-free reads
// of the swizzled panels (the update is elementwise in the cell dimension,
// so any row order is the same computation)
// alpha[k][c] at k * 64 + (c ^ 4 (k % 4)): the B-fragment loads (lanes g, t
// read row k = 4 ks + t, column c0 + g) hit 16 distinct 8-byte slots per
// half-warp
__device__ __forceinline__ int alpha_at(int k, int c) { return k * 64 + (c ^ ((k & 3) << 2)); }
__device__ __forceinline__ int pi8(int g) { return ((g & 1) << 2) | (g & 2) | (g >> 2); }
// Gram k-step kc, lane t -> cell of the run (all 16 covered once; the 4
// cells of a k-step have swizzle keys of equal parity)
__device__ __forceinline__ int gram_cell(int kc, int t) { return (kc & 1) + 2 * t + 8 * (kc >> 1); }
__device__ __forceinline__ double lds(const unsigned char* base, int r, int c) {
    return *reinterpret_cast<const double*>(base + swz(r, c));
}
__device__ __forceinline__ double2 lds2(const unsigned char* base, int r, int c) {  // c even
    return *reinterpret_cast<const double2*>(base + swz(r, c));
}
__device__ __forceinline__ void sts2(unsigned char* base, int r, int c, double x, double y) {
    *reinterpret_cast<double2*>(base + swz(r, c)) = make_double2(x, y);  // c even
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                       unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void team_sync(int team) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(kTeamWarps * 32) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// the 20 upper-triangle tiles (m 16-row block, n 8-column block) of the 64 x 64
// Gram, 5 per warp of a team (balanced)
__device__ __forceinline__ void gram_tile(int w, int i, int& m, int& n) {
    // tiles in row order: m = 0 -> n 0..7, m = 1 -> n 2..7, m = 2 -> n 4..7, m = 3 -> n 6..7
    const int k = 5 * w + i;
    m = (k >= 8) + (k >= 14) + (k >= 18);
    n = k - (m == 0 ? 0 : m == 1 ? 6 : m == 2 ? 10 : 12);
}

// The same 5 tiles per warp as gram_tile, with the warp's distinct m-blocks
// and n-blocks listed so a k-step loads each A fragment (rows of m-block M[j])
// and each B fragment (columns of n-block N[j]) once: 7-9 fragment loads per
// k-step instead of 15 (the Gram's shared-memory reads halve).
template <int W>
struct GramSet;
template <>
struct GramSet<0> {  // (0,0..4)
    static constexpr int NM = 1, NN = 5, DIAG = 0;
    static __device__ __forceinline__ constexpr int M(int j) { return j == 0 ? 0 : 0; }
    static __device__ __forceinline__ constexpr int N(int j) { return j == 0 ? 0 : j == 1 ? 1 : j == 2 ? 2 : j == 3 ? 3 : 4; }
    static __device__ __forceinline__ constexpr int TM(int j) { return j == 0 ? 0 : j == 1 ? 0 : j == 2 ? 0 : j == 3 ? 0 : 0; }
    static __device__ __forceinline__ constexpr int TN(int j) { return j == 0 ? 0 : j == 1 ? 1 : j == 2 ? 2 : j == 3 ? 3 : 4; }
};
template <>
struct GramSet<1> {  // (0,5..7), (1,2..3)
    static constexpr int NM = 2, NN = 5, DIAG = 3;
    static __device__ __forceinline__ constexpr int M(int j) { return j == 0 ? 0 : 1; }
    static __device__ __forceinline__ constexpr int N(int j) { return j == 0 ? 5 : j == 1 ? 6 : j == 2 ? 7 : j == 3 ? 2 : 3; }
    static __device__ __forceinline__ constexpr int TM(int j) { return j == 0 ? 0 : j == 1 ? 0 : j == 2 ? 0 : j == 3 ? 1 : 1; }
    static __device__ __forceinline__ constexpr int TN(int j) { return j == 0 ? 0 : j == 1 ? 1 : j == 2 ? 2 : j == 3 ? 3 : 4; }
};
template <>
struct GramSet<2> {  // (1,4..7), (2,4)
    static constexpr int NM = 2, NN = 4, DIAG = 4;
    static __device__ __forceinline__ constexpr int M(int j) { return j == 0 ? 1 : 2; }
    static __device__ __forceinline__ constexpr int N(int j) { return j == 0 ? 4 : j == 1 ? 5 : j == 2 ? 6 : j == 3 ? 7 : 0; }
    static __device__ __forceinline__ constexpr int TM(int j) { return j == 0 ? 0 : j == 1 ? 0 : j == 2 ? 0 : j == 3 ? 0 : 1; }
    static __device__ __forceinline__ constexpr int TN(int j) { return j == 0 ? 0 : j == 1 ? 1 : j == 2 ? 2 : j == 3 ? 3 : 0; }
};
template <>
struct GramSet<3> {  // (2,5..7), (3,6..7)
    static constexpr int NM = 2, NN = 3, DIAG = 3;
    static __device__ __forceinline__ constexpr int M(int j) { return j == 0 ? 2 : 3; }
    static __device__ __forceinline__ constexpr int N(int j) { return j == 0 ? 5 : j == 1 ? 6 : j == 2 ? 7 : j == 3 ? 0 : 0; }
    static __device__ __forceinline__ constexpr int TM(int j) { return j == 0 ? 0 : j == 1 ? 0 : j == 2 ? 0 : j == 3 ? 1 : 1; }
    static __device__ __forceinline__ constexpr int TN(int j) { return j == 0 ? 0 : j == 1 ? 1 : j == 2 ? 2 : j == 3 ? 1 : 2; }
};
// Rows 0-7 of a 16 x 8 tile (accumulators d[0], d[1]): one DMMA.8x8x4 instead
// of the m16n8k4's two. Used for each warp's diagonal tile (m, n = 2m), whose
// rows 8-15 lie strictly below the diagonal and are never read (the s x s
// solves read the upper triangle): 18 instead of 20 tile-halves per k-step
// and team, -10 % of the Gram's DMMA work, upper entries bitwise unchanged.
__device__ __forceinline__ void dmma_h(double (&d)[4], double a0, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a0), "d"(b));
}
// one staged 16-cell run into warp W's tiles: A = rows of `At` (m-blocks),
// B = rows of `Bt` (n-blocks) scaled per cell by dg[kc] when SCALE
template <int W, bool SCALE>
__device__ __forceinline__ void gram_run(double (&gacc)[5][4], const unsigned char* At,
                                         const unsigned char* Bt, const double (&dg)[4], int g,
                                         int t) {
    using GS = GramSet<W>;
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
        const int cc = gram_cell(kc, t);
        double a0[GS::NM], a1[GS::NM], b[GS::NN];
#pragma unroll
        for (int j = 0; j < GS::NM; ++j) {
            a0[j] = lds(At, cc, 16 * GS::M(j) + g);
            a1[j] = lds(At, cc, 16 * GS::M(j) + 8 + g);
        }
#pragma unroll
        for (int j = 0; j < GS::NN; ++j) {
            const double x = lds(Bt, cc, 8 * GS::N(j) + g);
            b[j] = SCALE ? dg[kc] * x : x;
        }
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if (i == GS::DIAG)
                dmma_h(gacc[i], a0[GS::TM(i)], b[GS::TN(i)]);
            else
                dmma_l(gacc[i], a0[GS::TM(i)], a1[GS::TM(i)], b[GS::TN(i)]);
        }
    }
}
template <int W>
__device__ __forceinline__ void gram_tile_c(int i, int& m, int& n) {
    m = GramSet<W>::M(GramSet<W>::TM(i));
    n = GramSet<W>::N(GramSet<W>::TN(i));
}

// consumer warp W (0..3) of team q of the update sweep (the Gram tiles and
// output columns of W are compile-time: fragment loads shared across tiles)
template <int W, class Issue>
__device__ __forceinline__ void update64_warp(Smem& sm, const SweepArgs& a, int q, int first,
                                              int ntiles, int nteams, bool jac, bool leader,
                                              Issue& issue) {
    constexpr int S = 64;
    constexpr int w = W;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    // ---- team q, warp w of the team owns columns 16 w .. 16 w + 15.
    // Software-pipelined so that a team needs ONE barrier per run: the update
    // of run i + 1 (independent DMMA work) sits between a warp's write of run
    // i's R into the team's staging buffer and the barrier after which the team
    // reads that buffer for run i's Gram. Staging is double-buffered: a warp
    // that passed the barrier of run i knows every warp finished the Gram of
    // run i - 1, so buffer (i + 1) % 2 is free for run i + 1.
    double gacc[5][4];
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) gacc[i][e] = 0.0;
    double rr[4] = {0.0, 0.0, 0.0, 0.0};  // columns 16w + 8nt + 2t + e

    // R -= W alpha for the run in stage `it`: D (16 cells x 8 columns) per
    // n-tile, K = 64; also fetches D^-1 of the Gram rows kc + 4t (kc = 0..3)
    auto update = [&](int it, double (&d)[2][4], double (&dg)[4], double& d0, double& d1) {
        const int s = it % kStages;
        mbar_wait(&sm.full[q][s], (it / kStages) & 1);
        const unsigned char* Wt = sm.stage[q][s];
        const unsigned char* Rt = Wt + kArrBytes;
        const double* dv = sm.dinv[q][s];
        const int rg = pi8(g);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int c = 16 * w + 8 * nt + 2 * t;
            const double2 lo = lds2(Rt, rg, c), hi = lds2(Rt, rg + 8, c);
            d[nt][0] = lo.x;
            d[nt][1] = lo.y;
            d[nt][2] = hi.x;
            d[nt][3] = hi.y;
        }
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
            const int k = 4 * ks + t;
            const double a0 = -lds(Wt, rg, k), a1 = -lds(Wt, rg + 8, k);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
                dmma_l(d[nt], a0, a1, sm.alpha[alpha_at(k, 16 * w + 8 * nt + g)]);
        }
        d0 = jac ? dv[rg] : 1.0;
        d1 = jac ? dv[rg + 8] : 1.0;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) dg[kc] = jac ? dv[gram_cell(kc, t)] : 1.0;
    };
    // rr, R to HBM, R into staging buffer b (Z = D^-1 R is formed in the Gram)
    auto epilogue = [&](int grp, const double (&d)[2][4], int b) {
        TileCells tc;
        tile_cells(a.sl, grp, ntiles, tc);
        unsigned char* St = sm.rstage[q][b];
        const int rg = pi8(g);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            rr[2 * nt] += d[nt][0] * d[nt][0] + d[nt][2] * d[nt][2];
            rr[2 * nt + 1] += d[nt][1] * d[nt][1] + d[nt][3] * d[nt][3];
            const int c = 16 * w + 8 * nt + 2 * t;
            *reinterpret_cast<double2*>(a.R + (tc.l0 + rg) * S + c) = make_double2(d[nt][0], d[nt][1]);
            *reinterpret_cast<double2*>(a.R + (tc.l0 + rg + 8) * S + c) =
                make_double2(d[nt][2], d[nt][3]);
            sts2(St, rg, c, d[nt][0], d[nt][1]);
            sts2(St, rg + 8, c, d[nt][2], d[nt][3]);
        }
    };
    // S_new += R^T Z over a run's 16 cells (Z = D^-1 R formed from the staged R
    // with each cell's D^-1 — the product the cp.async sweep stores);
    // conflict-free k-step -> cell map, fragments loaded once per k-step
    auto gram = [&](int b, const double (&dg)[4]) {
        const unsigned char* St = sm.rstage[q][b];
        gram_run<W, true>(gacc, St, St, dg, g, t);
    };
    if (first < ntiles) {
        double d[2][4], dg[4], d0, d1;
        update(0, d, dg, d0, d1);
        (void)d0;
        (void)d1;
        epilogue(first, d, 0);
        int it = 0;
        for (int grp = first; grp < ntiles; grp += nteams, ++it) {
            const int nxt = grp + nteams;
            double dn[2][4], dgn[4], e0, e1;
            if (nxt < ntiles) update(it + 1, dn, dgn, e0, e1);
            team_sync(q);  // every warp of the team staged run `it` and consumed run it + 1
            if (leader) {  // refill the stages of runs it and it + 1 (kStages = 3)
                if (it == 0) issue(kStages);
                issue(it + kStages + 1);
            }
            gram(it & 1, dg);
            if (nxt < ntiles) {
                epilogue(nxt, dn, (it + 1) & 1);
#pragma unroll
                for (int kc = 0; kc < 4; ++kc) dg[kc] = dgn[kc];
            }
        }
    }

    // ---- per-CTA partials [S_new (64 x 64) | rr (64)], teams summed in order
    asm volatile("bar.sync %0, %1;" ::"r"(9), "r"(kConsumers) : "memory");
    double* red = reinterpret_cast<double*>(sm.stage[0][0]);  // kTeams x (64*64 + 64) doubles
    static_assert(kTeams * (64 * 64 + 64) * 8 <= sizeof(Smem::stage), "reduction buffer");
    double* mine = red + q * (S * S + S);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        int gm, gn;
        gram_tile_c<W>(i, gm, gn);
        const int r0 = 16 * gm + g, c0 = 8 * gn + 2 * t;
        mine[r0 * S + c0] = gacc[i][0];
        mine[r0 * S + c0 + 1] = gacc[i][1];
        mine[(r0 + 8) * S + c0] = gacc[i][2];
        mine[(r0 + 8) * S + c0 + 1] = gacc[i][3];
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        double x = rr[e];
        x += __shfl_xor_sync(0xffffffffu, x, 4);
        x += __shfl_xor_sync(0xffffffffu, x, 8);
        x += __shfl_xor_sync(0xffffffffu, x, 16);
        if (g == 0) mine[S * S + 16 * w + 8 * (e >> 1) + 2 * t + (e & 1)] = x;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(9), "r"(kConsumers) : "memory");
    double* out = a.part + (int64_t)blockIdx.x * (S * S + S);
    for (int e = threadIdx.x; e < S * S + S; e += kConsumers) {
        if (e < S * S && (e % S) / 8 < 2 * ((e / S) / 16)) {  // below-diagonal tiles
            out[e] = 0.0;
            continue;
        }
        double v = red[e];
        for (int k = 1; k < kTeams; ++k) v += red[k * (S * S + S) + e];
        out[e] = v;
    }
}

// W (a.W) and R (a.R) as 2D tensors (64 columns, nloc rows). No producer
// warp: 12 warps (3 per SM sub-partition, so up to 168 registers — the
// 13-warp form capped them at 128 and spilled inside the run loop); each
// team's leader thread issues its own team's copies: the first kStages runs up
// front, then run it + 4 into the stage of run it + 1 right after the team
// barrier of run it (every warp of the team has consumed runs <= it + 1 by
// then), so two runs are in flight while the team works on a third.
__global__ void __launch_bounds__(kConsumers, 1)
    k_update64_ws(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapR,
                  SweepArgs a) {
    if (a.gate && *a.gate != 0) return;  // gated (DD lookahead): this iteration is a no-op
    constexpr int S = 64;
    extern __shared__ __align__(1024) unsigned char smraw_[];
    // 1024-byte aligned (128B-swizzle atoms); pointer arithmetic on the shared
    // array keeps the state space, so the accesses compile to LDS / STS
    Smem& sm = *reinterpret_cast<Smem*>(smraw_ + ((1024u - (smem_u32(smraw_) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ntiles = n_tiles(a.sl);  // 16-cell runs
    const int nteams = gridDim.x * kTeams;
    const bool jac = a.precond != 0;
    for (int e = threadIdx.x; e < S * S; e += blockDim.x)
        sm.alpha[alpha_at(e / S, e % S)] = a.coef[(e / S) * (S + 4) + e % S];
    const int q = warp / kTeamWarps, w = warp % kTeamWarps;
    const int first = blockIdx.x * kTeams + q;
    const bool leader = w == 0 && lane == 0;
    // run it of this team -> stage it % kStages
    auto issue = [&](int it) {
        const int grp = first + it * nteams;
        if (grp >= ntiles) return;
        const int s = it % kStages;
        TileCells tc;
        tile_cells(a.sl, grp, ntiles, tc);
        unsigned char* st = sm.stage[q][s];
        unsigned long long* bar = &sm.full[q][s];
        mbar_expect_tx(bar, 2 * kArrBytes + (jac ? 128 : 0));
        for (int p = 0; p < 4; ++p) {
            tma_2d(st + p * kPanelBytes, &mapW, 16 * p, (int)tc.l0, bar);
            tma_2d(st + kArrBytes + p * kPanelBytes, &mapR, 16 * p, (int)tc.l0, bar);
        }
        if (jac) bulk_g2s(sm.dinv[q][s], a.st.dinv + tc.g0, 128, bar);
    };
    if (leader) {
        for (int s = 0; s < kStages; ++s) mbar_init(&sm.full[q][s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int it = 0; it < kStages; ++it) issue(it);
    }
    __syncthreads();

    switch (w) {
        case 0: update64_warp<0>(sm, a, q, first, ntiles, nteams, jac, leader, issue); break;
        case 1: update64_warp<1>(sm, a, q, first, ntiles, nteams, jac, leader, issue); break;
        case 2: update64_warp<2>(sm, a, q, first, ntiles, nteams, jac, leader, issue); break;
        default: update64_warp<3>(sm, a, q, first, ntiles, nteams, jac, leader, issue); break;
    }
}

// ---------------------------------------------------------------------------
// P update for S = 64 (the common MODE 1 of k_pupdate): P = D^-1 R + P beta
// and the deferred X += P alpha (solvers.cpp:645-649 and :566-576), both
// GEMMs from the same staged P fragments. Same structure as the update sweep
// (producer warp, per-team TMA ring of P / R / X panels); no reduction, so no
// team barrier at all — each warp owns 16 output columns of P and X, reads
// its accumulator inits (Z, X) and every P row from the stage, releases the
// stage with one arrival and stores its results from registers. Per-element
// DMMA chains in ascending k, as k_pupdate: bitwise the same P and X.
// ---------------------------------------------------------------------------
constexpr int kPStages = 2;
struct SmemP {
    unsigned char stage[kTeams][kPStages][3 * kArrBytes];  // P, R, X panels
    double alpha[64 * 64];                                   // swizzled (alpha_at)
    double beta[64 * 64];
    double dinv[kTeams][kPStages][16];
    unsigned long long full[kTeams][kPStages];
    unsigned long long empty[kTeams][kPStages];
};
constexpr size_t smem_bytes_p() { return sizeof(SmemP) + 1024; }

__global__ void __launch_bounds__(kThreads, 1)
    k_pupdate64_ws(const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapR,
                   const __grid_constant__ CUtensorMap mapX, SweepArgs a) {
    constexpr int S = 64;
    extern __shared__ __align__(1024) unsigned char smraw_[];
    SmemP& sm = *reinterpret_cast<SmemP*>(smraw_ + ((1024u - (smem_u32(smraw_) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ntiles = n_tiles(a.sl);
    const int nteams = gridDim.x * kTeams;
    const bool jac = a.precond != 0;
    if (a.gate && *a.gate != 0) return;  // graph loop: a verification is due
    for (int e = threadIdx.x; e < S * S; e += blockDim.x) {
        sm.beta[alpha_at(e / S, e % S)] = a.coef[(e / S) * (S + 4) + e % S];
        sm.alpha[alpha_at(e / S, e % S)] = a.coef2[(e / S) * (S + 4) + e % S];
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < kTeams; ++q)
            for (int s = 0; s < kPStages; ++s) {
                mbar_init(&sm.full[q][s], 1);
                mbar_init(&sm.empty[q][s], kTeamWarps);
            }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kTeams * kTeamWarps) {  // ---- producer
        if (lane == 0) {
            int it[kTeams] = {};
            bool live = true;
            while (live) {
                live = false;
                for (int q = 0; q < kTeams; ++q) {
                    const int grp = blockIdx.x * kTeams + q + it[q] * nteams;
                    if (grp >= ntiles) continue;
                    live = true;
                    const int s = it[q] % kPStages;
                    if (it[q] >= kPStages) mbar_wait(&sm.empty[q][s], ((it[q] / kPStages) - 1) & 1);
                    TileCells tc;
                    tile_cells(a.sl, grp, ntiles, tc);
                    unsigned char* st = sm.stage[q][s];
                    unsigned long long* bar = &sm.full[q][s];
                    mbar_expect_tx(bar, 3 * kArrBytes + (jac ? 128 : 0));
                    for (int p = 0; p < 4; ++p) {
                        tma_2d(st + p * kPanelBytes, &mapP, 16 * p, (int)tc.l0, bar);
                        tma_2d(st + kArrBytes + p * kPanelBytes, &mapR, 16 * p, (int)tc.l0, bar);
                        tma_2d(st + 2 * kArrBytes + p * kPanelBytes, &mapX, 16 * p, (int)tc.l0, bar);
                    }
                    if (jac) bulk_g2s(sm.dinv[q][s], a.st.dinv + tc.g0, 128, bar);
                    ++it[q];
                }
            }
        }
        return;
    }

    const int q = warp / kTeamWarps, w = warp % kTeamWarps;
    const int rg = pi8(g);
    int it = 0;
    for (int grp = blockIdx.x * kTeams + q; grp < ntiles; grp += nteams, ++it) {
        const int s = it % kPStages;
        mbar_wait(&sm.full[q][s], (it / kPStages) & 1);
        const unsigned char* Pt = sm.stage[q][s];
        const unsigned char* Rt = Pt + kArrBytes;
        const unsigned char* Xt = Pt + 2 * kArrBytes;
        const double d0 = jac ? sm.dinv[q][s][rg] : 1.0, d1 = jac ? sm.dinv[q][s][rg + 8] : 1.0;
        double pv[2][4], xv[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int c = 16 * w + 8 * nt + 2 * t;
            const double2 r0 = lds2(Rt, rg, c), r1 = lds2(Rt, rg + 8, c);
            const double2 x0 = lds2(Xt, rg, c), x1 = lds2(Xt, rg + 8, c);
            pv[nt][0] = r0.x * d0;
            pv[nt][1] = r0.y * d0;
            pv[nt][2] = r1.x * d1;
            pv[nt][3] = r1.y * d1;
            xv[nt][0] = x0.x;
            xv[nt][1] = x0.y;
            xv[nt][2] = x1.x;
            xv[nt][3] = x1.y;
        }
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
            const int k = 4 * ks + t;
            const double a0 = lds(Pt, rg, k), a1 = lds(Pt, rg + 8, k);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int c = alpha_at(k, 16 * w + 8 * nt + g);
                dmma_l(xv[nt], a0, a1, sm.alpha[c]);
                dmma_l(pv[nt], a0, a1, sm.beta[c]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[q][s]);
        TileCells tc;
        tile_cells(a.sl, grp, ntiles, tc);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int c = 16 * w + 8 * nt + 2 * t;
            *reinterpret_cast<double2*>(a.P + (tc.l0 + rg) * S + c) = make_double2(pv[nt][0], pv[nt][1]);
            *reinterpret_cast<double2*>(a.P + (tc.l0 + rg + 8) * S + c) =
                make_double2(pv[nt][2], pv[nt][3]);
            *reinterpret_cast<double2*>(a.X + (tc.l0 + rg) * S + c) = make_double2(xv[nt][0], xv[nt][1]);
            *reinterpret_cast<double2*>(a.X + (tc.l0 + rg + 8) * S + c) =
                make_double2(xv[nt][2], xv[nt][3]);
        }
    }
}

// ---------------------------------------------------------------------------
// Stencil sweep for S = 64: W = A P (CsrMatrix::apply_block order, FMA chain
// z-, y-, x-, diag, x+, y+, z+; discretize.cpp:57-95) and the upper-triangle
// Gram G = P^T W (spmm_gram_fixed, solvers.cpp:221-242), z-marching.
//
// A team (4 warps) owns a pencil — a 16-cell x-run at fixed y — and walks
// it through z, so each P run arrives once from L2 and serves as the centre
// (with its x-halo cells) and as the z -+ 1 neighbour of the adjacent planes
// from a 4-slot ring; per step only the y -+ 1 runs and six coefficient runs
// stream in (a 2-unit ring). The producer warp issues all copies (1D bulk,
// mbarrier completion) two steps ahead; consumers never load from global.
// Per step: each thread forms W for one cell and 8 columns (16-byte shared
// reads of whole rows: conflict-free), stores W, stages P and W (swizzled,
// double-buffered) for the Gram, one team barrier, then each warp
// accumulates 5 of the 20 Gram tiles (conflict-free maps as in the update).
// ---------------------------------------------------------------------------
constexpr int kSTeams = 2;
constexpr int kSWarps = kSTeams * kTeamWarps;   // 8 consumer warps
constexpr int kSThreads = kSWarps * 32 + 32;    // + producer
constexpr int kCRows = 18;                      // centre run with its x-halo cells
constexpr int kCoefLD = 24;                     // doubles per coefficient run
struct SmemS {
    double cring[kSTeams][4][kCRows * 64];      // centre P runs, plane v in slot v % 4
    double yrun[kSTeams][2][2][16 * 64];        // y - 1 / y + 1 runs of a step
    double coef[kSTeams][2][6 * kCoefLD];       // diag, cx (x-halo), cy(y-1), cy, cz(z-1), cz
    unsigned char gst[kSTeams][2][2 * kArrBytes];  // Gram staging P | W (swizzled), 1024-aligned
    unsigned long long full[kSTeams][2], empty[kSTeams][2], pro[kSTeams];
};
constexpr size_t smem_bytes_s() { return sizeof(SmemS) + 1024; }

struct Pencil {
    int ix0, iyl, iyg;
    __device__ int64_t lrow(const Slab& sl, int z) const {  // slab-local row of cell ix0 at plane z
        return ix0 + (int64_t)sl.nx * (iyl + (int64_t)(sl.nyl + 2) * z);
    }
    __device__ int64_t grow(const Slab& sl, int z) const {
        return ix0 + (int64_t)sl.nx * (iyg + (int64_t)sl.ny * z);
    }
};
__device__ __forceinline__ Pencil pencil_of(const Slab& sl, int p) {
    const int ntx = sl.nx / 16;
    Pencil pc;
    pc.ix0 = 16 * (p % ntx);
    pc.iyl = 1 + p / ntx;
    pc.iyg = sl.y0 + pc.iyl - 1;
    return pc;
}

__global__ void __launch_bounds__(kSThreads, 1) k_spmm64_ws(SweepArgs a) {
    if (a.gate && *a.gate != 0) return;  // gated (DD lookahead): this iteration is a no-op
    constexpr int S = 64;
    extern __shared__ __align__(1024) unsigned char smraw_[];
    SmemS& sm = *reinterpret_cast<SmemS*>(smraw_ + ((1024u - (smem_u32(smraw_) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Slab& sl = a.sl;
    const int nz = sl.nz;
    const int npen = (sl.nx / 16) * sl.nyl;
    const int nteams = gridDim.x * kSTeams;
    if (threadIdx.x == 0) {
        for (int q = 0; q < kSTeams; ++q) {
            for (int s = 0; s < 2; ++s) {
                mbar_init(&sm.full[q][s], 1);
                mbar_init(&sm.empty[q][s], kTeamWarps);
            }
            mbar_init(&sm.pro[q], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kSWarps) {  // ---- producer
        if (lane == 0) {
            const int64_t plane = (int64_t)sl.nx * sl.ny;
            const unsigned rowb = S * 8;
            // centre run of plane z of pencil pc into ring slot `slot`
            auto centre = [&](int q, const Pencil& pc, int z, int slot, unsigned long long* bar) {
                const int lo = pc.ix0 > 0 ? -1 : 0, hi = pc.ix0 + 16 < sl.nx ? 16 : 15;
                bulk_g2s(sm.cring[q][slot] + (1 + lo) * S, a.P + (pc.lrow(sl, z) + lo) * S,
                         (unsigned)(hi - lo + 1) * rowb, bar);
            };
            auto centre_bytes = [&](const Pencil& pc) -> unsigned {
                const int lo = pc.ix0 > 0 ? -1 : 0, hi = pc.ix0 + 16 < sl.nx ? 16 : 15;
                return (unsigned)(hi - lo + 1) * rowb;
            };
            int p[kSTeams], z[kSTeams], u[kSTeams], v[kSTeams];
            bool live[kSTeams];
            for (int q = 0; q < kSTeams; ++q) {
                p[q] = blockIdx.x * kSTeams + q;
                z[q] = 0;
                u[q] = 0;
                v[q] = 0;
                live[q] = p[q] < npen;
                if (live[q]) {  // prologue: plane 0 of the first pencil
                    const Pencil pc = pencil_of(sl, p[q]);
                    mbar_expect_tx(&sm.pro[q], centre_bytes(pc));
                    centre(q, pc, 0, 0, &sm.pro[q]);
                }
            }
            bool any = true;
            while (any) {
                any = false;
                for (int q = 0; q < kSTeams; ++q) {
                    if (!live[q]) continue;
                    any = true;
                    const int s = u[q] & 1;
                    if (u[q] >= 2) mbar_wait(&sm.empty[q][s], ((u[q] >> 1) - 1) & 1);
                    const Pencil pc = pencil_of(sl, p[q]);
                    const int64_t g0 = pc.grow(sl, z[q]), l0 = pc.lrow(sl, z[q]);
                    unsigned long long* bar = &sm.full[q][s];
                    // next plane in this team's sequence
                    int pn = p[q], zn = z[q] + 1;
                    if (zn == nz) {
                        pn += nteams;
                        zn = 0;
                    }
                    const bool has_next = pn < npen;
                    Pencil pcn = has_next ? pencil_of(sl, pn) : pc;
                    unsigned bytes = 2 * 16 * rowb + 16 * 8 + 18 * 8 + 16 * 8 * 4;
                    if (has_next) bytes += centre_bytes(pcn);
                    mbar_expect_tx(bar, bytes);
                    bulk_g2s(sm.yrun[q][s][0], a.P + (l0 - sl.nx) * S, 16 * rowb, bar);
                    bulk_g2s(sm.yrun[q][s][1], a.P + (l0 + sl.nx) * S, 16 * rowb, bar);
                    double* cf = sm.coef[q][s];
                    bulk_g2s(cf, a.st.diag + g0, 16 * 8, bar);
                    bulk_g2s(cf + kCoefLD, a.st.cx + (g0 >= 2 ? g0 - 2 : g0), 18 * 8, bar);
                    bulk_g2s(cf + 2 * kCoefLD, a.st.cy + (pc.iyg > 0 ? g0 - sl.nx : g0), 16 * 8, bar);
                    bulk_g2s(cf + 3 * kCoefLD, a.st.cy + g0, 16 * 8, bar);
                    bulk_g2s(cf + 4 * kCoefLD, a.st.cz + (z[q] > 0 ? g0 - plane : g0), 16 * 8, bar);
                    bulk_g2s(cf + 5 * kCoefLD, a.st.cz + g0, 16 * 8, bar);
                    if (has_next) centre(q, pcn, zn, (v[q] + 1) & 3, bar);
                    ++u[q];
                    ++v[q];
                    p[q] = pn;
                    z[q] = zn;
                    live[q] = has_next;
                }
            }
        }
        return;
    }

    // ---- consumers
    const int q = warp / kTeamWarps, w = warp % kTeamWarps;
    const int tt = threadIdx.x & 127;        // thread of the team
    const int r = tt >> 3, cq = tt & 7;      // cell of the run, column quad
    const int g = lane >> 2, t = lane & 3;
    double gacc[5][4];
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) gacc[i][e] = 0.0;
    int gm[5], gn[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) gram_tile(w, i, gm[i], gn[i]);
    const int first = blockIdx.x * kSTeams + q;
    if (first < npen) mbar_wait(&sm.pro[q], 0);
    int u = 0;
    for (int pp = first; pp < npen; pp += nteams) {
        const Pencil pc = pencil_of(sl, pp);
        const int ix = pc.ix0 + r;
        for (int zz = 0; zz < nz; ++zz, ++u) {
            const int xo = (pc.grow(sl, zz) < 2) ? 2 : 0;  // cx run started at g0 (array start)
            const int s = u & 1;
            mbar_wait(&sm.full[q][s], (u >> 1) & 1);
            const double* C0 = sm.cring[q][u & 3];
            const double* Cm = sm.cring[q][(u + 3) & 3];
            const double* Cp = sm.cring[q][(u + 1) & 3];
            const double* Ym = sm.yrun[q][s][0];
            const double* Yp = sm.yrun[q][s][1];
            const double* cf = sm.coef[q][s];
            const bool hzm = zz > 0, hzp = zz < nz - 1, hym = pc.iyg > 0, hyp = pc.iyg < sl.ny - 1;
            const bool hxm = ix > 0, hxp = ix < sl.nx - 1;
            const double czm = -cf[4 * kCoefLD + r], cym = -cf[2 * kCoefLD + r];
            const double cxm = -cf[kCoefLD + r + 1 - xo], dg = cf[r];
            const double cxp = -cf[kCoefLD + r + 2 - xo], cyp = -cf[3 * kCoefLD + r];
            const double czp = -cf[5 * kCoefLD + r];
            double2 acc[4], ctr[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = 2 * cq + 16 * j;
                auto ld = [&](const double* row) {
                    return *reinterpret_cast<const double2*>(row + c);
                };
                double2 x = make_double2(0.0, 0.0);
                auto fm = [&](double cc, double2 v) {
                    x.x = fma(cc, v.x, x.x);
                    x.y = fma(cc, v.y, x.y);
                };
                if (hzm) fm(czm, ld(Cm + (1 + r) * S));
                if (hym) fm(cym, ld(Ym + r * S));
                if (hxm) fm(cxm, ld(C0 + r * S));
                ctr[j] = ld(C0 + (1 + r) * S);
                fm(dg, ctr[j]);
                if (hxp) fm(cxp, ld(C0 + (2 + r) * S));
                if (hyp) fm(cyp, ld(Yp + r * S));
                if (hzp) fm(czp, ld(Cp + (1 + r) * S));
                acc[j] = x;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[q][s]);
            const int64_t l = pc.lrow(sl, zz) + r;
            unsigned char* Ut = sm.gst[q][s];
            unsigned char* Vt = Ut + kArrBytes;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = 2 * cq + 16 * j;
                *reinterpret_cast<double2*>(a.W + l * S + c) = acc[j];
                sts2(Ut, r, c, ctr[j].x, ctr[j].y);
                sts2(Vt, r, c, acc[j].x, acc[j].y);
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(kTeamWarps * 32) : "memory");
#pragma unroll
            for (int kc = 0; kc < 4; ++kc) {
                const int cc = gram_cell(kc, t);
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const double a0 = lds(Ut, cc, 16 * gm[i] + g);
                    const double a1 = lds(Ut, cc, 16 * gm[i] + 8 + g);
                    dmma_l(gacc[i], a0, a1, lds(Vt, cc, 8 * gn[i] + g));
                }
            }
        }
    }

    // ---- per-CTA partial G (64 x 64), teams summed in order
    asm volatile("bar.sync %0, %1;" ::"r"(9), "r"(kSWarps * 32) : "memory");
    double* red = &sm.cring[0][0][0];
    static_assert(kSTeams * 64 * 64 * 8 <= sizeof(SmemS::cring), "reduction buffer");
    double* mine = red + q * (S * S);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int r0 = 16 * gm[i] + g, c0 = 8 * gn[i] + 2 * t;
        mine[r0 * S + c0] = gacc[i][0];
        mine[r0 * S + c0 + 1] = gacc[i][1];
        mine[(r0 + 8) * S + c0] = gacc[i][2];
        mine[(r0 + 8) * S + c0 + 1] = gacc[i][3];
    }
    asm volatile("bar.sync %0, %1;" ::"r"(9), "r"(kSWarps * 32) : "memory");
    double* out = a.part + (int64_t)blockIdx.x * (S * S);
    for (int e = threadIdx.x; e < S * S; e += kSWarps * 32) {
        if ((e % S) / 8 < 2 * ((e / S) / 16)) {
            out[e] = 0.0;
            continue;
        }
        double v = red[e];
        for (int k = 1; k < kSTeams; ++k) v += red[k * (S * S) + e];
        out[e] = v;
    }
}

// ---------------------------------------------------------------------------
// Role-split form of the stencil sweep (the default): one pencil stream per
// CTA, 4 stencil warps + 4 Gram warps + 1 producer warp. The stencil warps
// (one per SM sub-partition) form W for step u + 1 while the Gram warps (one
// per sub-partition) run step u's 80 DMMAs, so every sub-partition always has
// a warp issuing DMMA and the stencil's loads, SIMT FMAs and stores hide
// behind it — in the two-team form a team's stencil, barrier and Gram phases
// ran back to back and the FP64 pipe sat idle ~40 % of the time (ncu).
// Same producer scheme as k_spmm64_ws with a deeper ring (kRS steps ahead);
// the stencil -> Gram hand-off goes through kRG swizzled staging buffers with
// full / empty mbarriers (4 arrivals: one per warp after __syncwarp).
// Each Gram warp owns 5 of the 20 upper tiles for the whole sweep (one
// accumulation chain per tile in step order): run-to-run deterministic.
// ---------------------------------------------------------------------------
// Per-run packed stencil coefficients (one bulk copy per band step instead of
// six 128-byte copies per run: measured 0.2 ms of a 1.3 ms sweep), negated as
// the stencil uses them: [diag 16 | -cx of cells x0 - 1 .. x0 + 15 (17) | -cy
// toward y - 1 (16) | -cy toward y + 1 (16) | -cz toward z - 1 (16) | -cz
// toward z + 1 (16) | pad 3], zero across the domain boundary. The run at
// (x-run xr, row y, plane z) sits at ((xr nz + z) ny + y) kPC, so the runs of
// a y-band at one plane are contiguous.
constexpr int kPC = 100;
constexpr int kPD = 0, kPXM = 16, kPYM = 33, kPYP = 49, kPZM = 65, kPZP = 81;
__global__ void k_pack_coef64(Slab sl, StencilPtr st, double* __restrict__ out) {
    const int ntx = sl.nx / 16;
    const int64_t nrun = (int64_t)ntx * sl.ny * sl.nz;
    const int64_t plane = (int64_t)sl.nx * sl.ny;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nrun * kPC;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t T = e / kPC;
        const int k = (int)(e % kPC);
        const int iy = (int)(T % sl.ny);
        const int64_t q = T / sl.ny;
        const int iz = (int)(q % sl.nz), ix0 = 16 * (int)(q / sl.nz);
        const int64_t g0 = ix0 + (int64_t)sl.nx * (iy + (int64_t)sl.ny * iz);
        double v = 0.0;
        if (k < kPXM) {
            v = st.diag[g0 + k];
        } else if (k < kPYM) {
            const int c = k - kPXM;  // cell x0 - 1 + c
            if (ix0 + c - 1 >= 0) v = -st.cx[g0 + c - 1];
        } else if (k < kPYP) {
            if (iy > 0) v = -st.cy[g0 - sl.nx + (k - kPYM)];
        } else if (k < kPZM) {
            v = -st.cy[g0 + (k - kPYP)];
        } else if (k < kPZP) {
            if (iz > 0) v = -st.cz[g0 - plane + (k - kPZM)];
        } else if (k < kPZP + 16) {
            v = -st.cz[g0 + (k - kPZP)];
        }
        out[e] = v;
    }
}

// ---------------------------------------------------------------------------
// Role-split, y-banded form of the stencil sweep (the default). Work unit: a
// band of B x-runs adjacent in y (same x, rows y0 .. y0 + B - 1), marched
// through z. Per band step the producer brings the B centre runs of the next
// plane (with x-halo cells), the two y-halo runs and the band's packed
// coefficients (B + 3 copies): a run reaches the SM (B + 2) / B times instead
// of 3 times — the sweep was bound by L2 -> SM delivery (ncu: with the Gram
// removed it still took 1.19 of 1.32 ms).
// 4 stencil warps (thread = cell r x column quad cq, looping over the band's
// runs) + 4 Gram warps + 1 producer warp: every SM sub-partition always has a
// Gram warp issuing DMMA while its stencil warp loads / stores. Stencil ->
// Gram hand-off per run through kRG swizzled staging buffers with full /
// empty mbarriers (4 arrivals: one per warp after __syncwarp). Each Gram warp
// owns 5 of the 20 upper tiles for the whole sweep (one accumulation chain per
// tile in run order): run-to-run deterministic.
// ---------------------------------------------------------------------------
template <int B>
struct Band {
    static constexpr int RS = B == 1 ? 6 : B == 2 ? 4 : 2;  // input bundles in flight
    static constexpr int RC = RS + 2;                         // centre-plane slots
};
constexpr int kRG = 2;                          // stencil -> Gram staging buffers
constexpr int kRThreads = 9 * 32;
template <int B>
struct SmemR {
    static constexpr int RS = Band<B>::RS, RC = Band<B>::RC;
    unsigned char gst[kRG][2 * kArrBytes];      // P | W of a run, swizzled (1024-aligned)
    double cring[RC][B][kCRows * 64];           // centre runs with x-halo cells, per plane
    double yrun[RS][2][16 * 64];                // y - 1 / y + B halo runs
    double coef[RS][B * kPC];
    unsigned long long full[RS], empty[RS], gfull[kRG], gempty[kRG], pro;
};
template <int B>
constexpr size_t smem_bytes_r() { return sizeof(SmemR<B>) + 1024; }

// Gram warp W: consumes every staged run, then writes its tiles of the CTA's
// partial G (and zeros in its share of the lower tiles)
template <int W, int B>
__device__ __forceinline__ void spmm_gram_warp(SmemR<B>& sm, const SweepArgs& a, int nruns) {
    constexpr int S = 64;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    double gacc[5][4];
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) gacc[i][e] = 0.0;
    const double one[4] = {1.0, 1.0, 1.0, 1.0};
    for (int v = 0; v < nruns; ++v) {
        const int b = v % kRG;
        mbar_wait(&sm.gfull[b], (v / kRG) & 1);
        const unsigned char* Ut = sm.gst[b];
        gram_run<W, false>(gacc, Ut, Ut + kArrBytes, one, g, t);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.gempty[b]);
    }
    double* out = a.part + (int64_t)blockIdx.x * (S * S);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        int gm, gn;
        gram_tile_c<W>(i, gm, gn);
        const int r0 = 16 * gm + g, c0 = 8 * gn + 2 * t;
        out[r0 * S + c0] = gacc[i][0];
        out[r0 * S + c0 + 1] = gacc[i][1];
        out[(r0 + 8) * S + c0] = gacc[i][2];
        out[(r0 + 8) * S + c0 + 1] = gacc[i][3];
    }
    for (int e = 32 * W + lane; e < S * S; e += 128)
        if ((e % S) / 8 < 2 * ((e / S) / 16)) out[e] = 0.0;
}

template <int B, bool WIN = true>
__global__ void __launch_bounds__(kRThreads, 1) k_spmm64_rs(SweepArgs a) {
    if (a.gate && *a.gate != 0) return;  // gated (DD lookahead): this iteration is a no-op
    constexpr int S = 64;
    constexpr int RS = Band<B>::RS, RC = Band<B>::RC;
    extern __shared__ __align__(1024) unsigned char smraw_[];
    SmemR<B>& sm =
        *reinterpret_cast<SmemR<B>*>(smraw_ + ((1024u - (smem_u32(smraw_) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Slab& sl = a.sl;
    const int nz = sl.nz;
    const int ntx = sl.nx / 16;
    const int nband = ntx * (sl.nyl / B);
    // band -> (x-run, first slab-local row); rows y0 .. y0 + B - 1
    auto band_of = [&](int bd, int& ix0, int& iyl0) {
        ix0 = 16 * (bd % ntx);
        iyl0 = 1 + B * (bd / ntx);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < RS; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kTeamWarps);
        }
        for (int s = 0; s < kRG; ++s) {
            mbar_init(&sm.gfull[s], kTeamWarps);
            mbar_init(&sm.gempty[s], kTeamWarps);
        }
        mbar_init(&sm.pro, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int first = blockIdx.x;
    const int stride = gridDim.x;
    const int64_t nxl = sl.nx, plane_l = (int64_t)sl.nx * (sl.nyl + 2);

    if (warp == 8) {  // ---- producer
        if (lane == 0 && first < nband) {
            const unsigned rowb = S * 8;
            int ix0, iyl0;
            const int lo_x = 0;  // centre rows x0 - 1 .. x0 + 16, clipped to the grid
            (void)lo_x;
            auto cbytes = [&](int x0) -> unsigned {
                const int lo = x0 > 0 ? -1 : 0, hi = x0 + 16 < sl.nx ? 16 : 15;
                return (unsigned)(hi - lo + 1) * rowb * B;
            };
            // the band's B centre runs of plane z into ring slot `slot`
            auto centres = [&](int x0, int y0l, int z, int slot, unsigned long long* bar) {
                const int lo = x0 > 0 ? -1 : 0, hi = x0 + 16 < sl.nx ? 16 : 15;
#pragma unroll 1
                for (int b = 0; b < B; ++b) {
                    const int64_t l = x0 + nxl * (y0l + b) + plane_l * z;
                    bulk_g2s(sm.cring[slot][b] + (1 + lo) * S, a.P + (l + lo) * S,
                             (unsigned)(hi - lo + 1) * rowb, bar);
                }
            };
            int bd = first, z = 0;
            band_of(bd, ix0, iyl0);
            mbar_expect_tx(&sm.pro, cbytes(ix0));
            centres(ix0, iyl0, 0, 0, &sm.pro);
            for (int u = 0;; ++u) {
                const int s = u % RS;
                if (u >= RS) mbar_wait(&sm.empty[s], ((u / RS) - 1) & 1);
                const int64_t l0 = ix0 + nxl * iyl0 + plane_l * z;  // first run of the band
                const int iyg0 = sl.y0 + iyl0 - 1;
                unsigned long long* bar = &sm.full[s];
                int bn = bd, zn = z + 1;
                if (zn == nz) {
                    bn += stride;
                    zn = 0;
                }
                const bool has_next = bn < nband;
                int nx0 = ix0, ny0 = iyl0;
                if (has_next) band_of(bn, nx0, ny0);
                unsigned bytes = 2 * 16 * rowb + B * kPC * 8;
                if (has_next) bytes += cbytes(nx0);
                mbar_expect_tx(bar, bytes);
                bulk_g2s(sm.yrun[s][0], a.P + (l0 - nxl) * S, 16 * rowb, bar);
                bulk_g2s(sm.yrun[s][1], a.P + (l0 + B * nxl) * S, 16 * rowb, bar);
                bulk_g2s(sm.coef[s], a.pcoef + (((int64_t)(ix0 / 16) * nz + z) * sl.ny + iyg0) * kPC,
                         B * kPC * 8, bar);
                if (has_next) centres(nx0, ny0, zn, (u + 1) % RC, bar);
                if (!has_next) break;
                bd = bn;
                z = zn;
                ix0 = nx0;
                iyl0 = ny0;
            }
        }
        return;
    }

    const int nbands = first < nband ? (nband - 1 - first) / stride + 1 : 0;
    if (warp < 4) {  // ---- stencil warps: thread = (cell r, column quad cq) of every run
        const int tt = threadIdx.x;  // 0..127
        const int r = tt >> 3, cq = tt & 7;
        if (nbands) mbar_wait(&sm.pro, 0);
        int u = 0, v = 0;  // band steps, runs
        // this thread's columns of its cell of run b at planes z and z + 1,
        // kept in registers as the band marches (B <= 2; the z - 1 plane is
        // read back from the ring, B = 4 reads all three from the ring)
        constexpr bool ROT = B <= 2;
        double2 pz[ROT ? B : 1][4], pp1[ROT ? B : 1][4];
        // B = 4: the band's y-neighbours come from a register window over the
        // runs (run b - 1 / b / b + 1 at plane z): one centre load per run
        // serves as its own centre and as the y -+ 1 neighbour of the others
        double2 wprv[4], wcur[4], wnxt[4];
        for (int bd = first; bd < nband; bd += stride) {
            int ix0, iyl0;
            band_of(bd, ix0, iyl0);
            const int ix = ix0 + r;
            const int iyg0 = sl.y0 + iyl0 - 1;
            const bool hxm = ix > 0, hxp = ix < sl.nx - 1;
            for (int zz = 0; zz < nz; ++zz, ++u) {
                const int s = u % RS;
                mbar_wait(&sm.full[s], (u / RS) & 1);
                const bool hzm = zz > 0, hzp = zz < nz - 1;
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const double* C0 = sm.cring[u % RC][b];
                    const double* Cm = sm.cring[(u + RC - 1) % RC][b];
                    const double* Cp = sm.cring[(u + 1) % RC][b];
                    const double* Ym = b == 0 ? sm.yrun[s][0] : sm.cring[u % RC][b - 1] + S;
                    const double* Yp = b == B - 1 ? sm.yrun[s][1] : sm.cring[u % RC][b + 1] + S;
                    const double* cf = sm.coef[s] + b * kPC;
                    const bool hym = iyg0 + b > 0, hyp = iyg0 + b < sl.ny - 1;
                    const double czm = cf[kPZM + r], cym = cf[kPYM + r];
                    const double cxm = cf[kPXM + r], dg = cf[kPD + r];
                    const double cxp = cf[kPXM + r + 1], cyp = cf[kPYP + r];
                    const double czp = cf[kPZP + r];
                    double2 acc[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int c = 2 * cq + 16 * j;
                        auto ld = [&](const double* row) {
                            return *reinterpret_cast<const double2*>(row + c);
                        };
                        double2 cz, cp, ym2, yp2;
                        const double2 zero2 = make_double2(0.0, 0.0);
                        if constexpr (ROT) {
                            if (zz == 0)
                                pz[b][j] = ld(C0 + (1 + r) * S);
                            else
                                pz[b][j] = pp1[b][j];
                            pp1[b][j] = hzp ? ld(Cp + (1 + r) * S) : zero2;
                            cz = pz[b][j];
                            cp = pp1[b][j];
                            ym2 = hym ? ld(Ym + r * S) : zero2;
                            yp2 = hyp ? ld(Yp + r * S) : zero2;
                        } else {
                            if (!WIN) {
                                wcur[j] = ld(C0 + (1 + r) * S);
                                wprv[j] = hym ? ld(Ym + r * S) : zero2;
                            } else if (b == 0) {
                                wcur[j] = ld(C0 + (1 + r) * S);
                                wprv[j] = hym ? ld(Ym + r * S) : zero2;
                            } else {
                                wprv[j] = wcur[j];
                                wcur[j] = wnxt[j];
                            }
                            wnxt[j] = (b < B - 1 || hyp) ? ld(Yp + r * S) : zero2;
                            cz = wcur[j];
                            ym2 = wprv[j];
                            yp2 = wnxt[j];
                            cp = hzp ? ld(Cp + (1 + r) * S) : zero2;
                            pz[0][j] = cz;  // staged below
                        }
                        double2 x = make_double2(0.0, 0.0);
                        auto fm = [&](double cc, double2 w2) {
                            x.x = fma(cc, w2.x, x.x);
                            x.y = fma(cc, w2.y, x.y);
                        };
                        if (hzm) fm(czm, ld(Cm + (1 + r) * S));
                        if (hym) fm(cym, ym2);
                        if (hxm) fm(cxm, ld(C0 + r * S));
                        fm(dg, cz);
                        if (hxp) fm(cxp, ld(C0 + (2 + r) * S));
                        if (hyp) fm(cyp, yp2);
                        if (hzp) fm(czp, cp);
                        acc[j] = x;
                    }
                    if (b == B - 1) {  // the bundle is no longer read
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&sm.empty[s]);
                    }
                    const int64_t l = ix0 + nxl * (iyl0 + b) + plane_l * zz + r;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        *reinterpret_cast<double2*>(a.W + l * S + 2 * cq + 16 * j) = acc[j];
                    const int gb = v % kRG;
                    if (v >= kRG) mbar_wait(&sm.gempty[gb], ((v / kRG) - 1) & 1);
                    unsigned char* Ut = sm.gst[gb];
                    unsigned char* Vt = Ut + kArrBytes;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int c = 2 * cq + 16 * j;
                        const double2 pc = pz[ROT ? b : 0][j];
                        sts2(Ut, r, c, pc.x, pc.y);
                        sts2(Vt, r, c, acc[j].x, acc[j].y);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.gfull[gb]);
                    ++v;
                }
            }
        }
        return;
    }

    // ---- Gram warps: G += P^T W, 5 of the 20 upper 16 x 8 tiles each
    const int nruns = nbands * nz * B;
    switch (warp - 4) {
        case 0: spmm_gram_warp<0>(sm, a, nruns); break;
        case 1: spmm_gram_warp<1>(sm, a, nruns); break;
        case 2: spmm_gram_warp<2>(sm, a, nruns); break;
        default: spmm_gram_warp<3>(sm, a, nruns); break;
    }
}

inline PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) !=
                cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// [nrows][64] doubles as a 2D tensor, box 16 columns x 16 rows, 128B swizzle
inline bool make_map(CUtensorMap* m, const double* base, int64_t nrows) {
    auto enc = encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {64, (cuuint64_t)nrows};
    const cuuint64_t strides[1] = {64 * 8};
    const cuuint32_t box[2] = {16, 16};
    const cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace sweep64

// the warp-specialised S = 64 update (XD layout: X is updated by k_pupdate)
inline bool update64_ws_ok(const Slab& sl) { return sl.nx % 16 == 0; }
inline cudaError_t launch_update64_ws(const SweepArgs& a, int64_t nloc, int nsm, cudaStream_t s) {
    CUtensorMap mw, mr;
    if (!sweep64::make_map(&mw, a.W, nloc) || !sweep64::make_map(&mr, a.R, nloc))
        return cudaErrorInvalidValue;
    const size_t smem = sweep64::smem_bytes();
    const cudaError_t e = bk::set_max_smem((const void*)sweep64::k_update64_ws, smem);
    if (e != cudaSuccess) return e;
    sweep64::k_update64_ws<<<nsm, sweep64::kConsumers, smem, s>>>(mw, mr, a);
    return cudaGetLastError();
}

// the warp-specialised S = 64 P update with the deferred X update (MODE 1)
inline cudaError_t launch_pupdate64_ws(const SweepArgs& a, int64_t nloc, int nsm, cudaStream_t s) {
    CUtensorMap mp, mr, mx;
    if (!sweep64::make_map(&mp, a.P, nloc) || !sweep64::make_map(&mr, a.R, nloc) ||
        !sweep64::make_map(&mx, a.X, nloc))
        return cudaErrorInvalidValue;
    const size_t smem = sweep64::smem_bytes_p();
    const cudaError_t e = bk::set_max_smem((const void*)sweep64::k_pupdate64_ws, smem);
    if (e != cudaSuccess) return e;
    sweep64::k_pupdate64_ws<<<nsm, sweep64::kThreads, smem, s>>>(mp, mr, mx, a);
    return cudaGetLastError();
}

// z-marching stencil sweep with the Gram (full 16-cell x-runs, 16-aligned x):
// the role-split kernel, or (teams = true) the two-team form
inline cudaError_t launch_spmm64_ws(const SweepArgs& a, int nsm, cudaStream_t s, bool teams = false,
                                    int band = 2) {
    if (teams) {
        const size_t smem = sweep64::smem_bytes_s();
        const cudaError_t e = bk::set_max_smem((const void*)sweep64::k_spmm64_ws, smem);
        if (e != cudaSuccess) return e;
        sweep64::k_spmm64_ws<<<nsm, sweep64::kSThreads, smem, s>>>(a);
        return cudaGetLastError();
    }
    auto go = [&](auto kern, size_t smem) {
        const cudaError_t e = bk::set_max_smem((const void*)kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<nsm, sweep64::kRThreads, smem, s>>>(a);
        return cudaGetLastError();
    };
    if (band == 4 && a.sl.nyl % 4 == 0) return go(sweep64::k_spmm64_rs<4>, sweep64::smem_bytes_r<4>());
    if (band == 5 && a.sl.nyl % 4 == 0)  // band 4 without the register y-window (A/B)
        return go(sweep64::k_spmm64_rs<4, false>, sweep64::smem_bytes_r<4>());
    if (band >= 2 && a.sl.nyl % 2 == 0) return go(sweep64::k_spmm64_rs<2>, sweep64::smem_bytes_r<2>());
    return go(sweep64::k_spmm64_rs<1>, sweep64::smem_bytes_r<1>());
}
