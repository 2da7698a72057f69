// Fused combination + operator action: one pass writes every (T, q) sample.
//
//   T_j = sum_t C[t][j] X[:,t]        combine_from_weights  pipeline.cpp:187-225
//   q_j = (A T_j - g) / V             operator_action       pipeline.cpp:242-251
//   resid_j = ||A T_j - (V q_j + g)|| / ||V q_j + g||       pipeline.cpp:548-571
//
// Each CTA owns a 32 x 8 x-y tile of cells (all z, marched plane by plane,
// 2.5D blocking) and a chunk of NS samples. A plane of T for the tile plus a
// one-cell x-y halo is formed in shared memory straight from X (L2-resident,
// n x s) and the coefficients; the stencil is then applied to the smem tile and
// T and q leave the SM exactly once, sample-major. A ring of three planes
// supplies the z-1 / z+1 neighbours. No T round trip through HBM, no second
// pass for q.
//
// Bitwise contract: T uses the reference's per-element order (first term a
// product, then one fma per basis column in ascending order — the DMMA's
// accumulation order, verified bitwise); A T uses the
// scalar CsrMatrix::apply order (separate multiply and add, CSR column order);
// q = (y - g) / V is correctly rounded. So given the same X, T and q equal the
// reference's bit for bit (tests/test_gpu_parity.py checks it).
#include <cstdio>
#include <cstdlib>

#include "bk_common.cuh"

namespace {

constexpr int TX = 32, TY = 8, HX = TX + 2, HY = TY + 2, HC = HX * HY;
constexpr int NT = 256;  // = TX * TY: one interior cell per thread in the stencil phase

struct ActArgs {
    int nx, ny, nz;
    int64_t n;
    int64_t N;
    int64_t ldc;  // row stride of C
    const double* diag;
    const double* cx;
    const double* cy;
    const double* cz;
    const double* g;
    const double* volz;
    const double* X;  // n x S
    const double* C;  // S x N
    double* T;        // N x n (nullable)
    double* Q;        // N x n (nullable)
    double* part;     // N x tiles x 2 residual partials (nullable)
    int tiles;
    int s;            // real basis width (<= S)
};

// correctly rounded x / v given r = RN(1/v) (one Newton-style correction).
__device__ __forceinline__ double div_rn(double x, double v, double r) {
    const double q0 = x * r;
    const double e = fma(-q0, v, x);
    return fma(e, r, q0);
}

__device__ __forceinline__ void dmma_c(double (&d)[4], double a0, double a1, double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b));
}

// B-fragment rows of C in shared memory: at most two lanes per 8-byte bank slot
constexpr int CSTRIDE(int NS) { return NS == 8 ? 8 : NS + 4; }

// debug: stage timestamps of CTA (0, 0) when BK_COMB_PROFILE is set
__device__ long long g_comb_prof[64];
__device__ __forceinline__ void comb_mark(int k) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && k < 64) g_comb_prof[k] = clock64();
}

// T for one z-plane of the tile + halo into buf[q * HC + h] (sample-major, so
// the stencil's neighbour reads are bank-conflict free), on FP64 tensor cores:
// T (halo cells x NS samples) = X_rows (cells x S) . C (S x NS) as m16n8k4 DMMA
// with M = cells, N = samples, K = basis columns. The DMMA accumulates in k
// order with one rounding per multiply-add — measured bitwise identical to the
// reference's fma chain (scripts/dmma_bitwise.cu: 0 of 25600 differ) — so T
// stays bitwise the reference's combine_from_weights.
template <int S, int NS>
__device__ __forceinline__ void form_plane(const ActArgs& a, int x0, int y0, int z,
                                           const double* __restrict__ Cs, double* __restrict__ buf) {
    constexpr int CS = CSTRIDE(NS);
    constexpr int MTILES = (HC + 15) / 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t plane = (int64_t)a.nx * a.ny;
    for (int mt = warp; mt < MTILES; mt += NT / 32) {
        const int h0 = 16 * mt + g, h1 = h0 + 8;
        const double* xr[2];
        bool in[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int h = r ? h1 : h0;
            const int gx = x0 - 1 + h % HX, gy = y0 - 1 + h / HX;
            in[r] = h < HC && gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny;
            xr[r] = a.X + (gx + (int64_t)a.nx * gy + plane * z) * S;
        }
        double d[NS / 8][4];
#pragma unroll
        for (int n = 0; n < NS / 8; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) d[n][e] = 0.0;
#pragma unroll 4
        for (int ks = 0; ks < S / 4; ++ks) {
            const double a0 = in[0] ? xr[0][4 * ks + t] : 0.0;
            const double a1 = in[1] ? xr[1][4 * ks + t] : 0.0;
#pragma unroll
            for (int n = 0; n < NS / 8; ++n) dmma_c(d[n], a0, a1, Cs[(4 * ks + t) * CS + 8 * n + g]);
        }
#pragma unroll
        for (int n = 0; n < NS / 8; ++n) {
            const int q = 8 * n + 2 * t;
            if (h0 < HC) {
                buf[q * HC + h0] = d[n][0];
                buf[(q + 1) * HC + h0] = d[n][1];
            }
            if (h1 < HC) {
                buf[q * HC + h1] = d[n][2];
                buf[(q + 1) * HC + h1] = d[n][3];
            }
        }
    }
}

template <int S, int NS>
__global__ void __launch_bounds__(NT, NS == 8 ? 3 : 2) combine_action_kernel(ActArgs a) {
    extern __shared__ __align__(16) double sm[];
    double* Cs = sm;                             // S x (NS + 4)
    double* ring = sm + S * CSTRIDE(NS);         // min(nz,3) x NS x HC
    const int nring = a.nz < 3 ? a.nz : 3;
    // grid: x = sample chunk (fastest), y = cell tile, so the CTAs resident at
    // any moment share one tile's X rows through L2 instead of re-reading X
    // from HBM once per chunk (config 5: X = 2.1 GB)
    const int tilesx = (a.nx + TX - 1) / TX;
    const int tile = blockIdx.y;
    const int x0 = (tile % tilesx) * TX, y0 = (tile / tilesx) * TY;
    const int64_t j0 = (int64_t)blockIdx.x * NS;
    const int tid = threadIdx.x;
    const int64_t plane = (int64_t)a.nx * a.ny;

    comb_mark(0);
    for (int e = tid; e < S * NS; e += NT) {
        const int k = e / NS, q = e % NS;
        Cs[k * CSTRIDE(NS) + q] = (k < a.s && j0 + q < a.N) ? a.C[(int64_t)k * a.ldc + j0 + q] : 0.0;
    }
    __syncthreads();

    const int lx = tid % TX, ly = tid / TX;
    const int gx = x0 + lx, gy = y0 + ly;
    const bool inside = gx < a.nx && gy < a.ny;
    const int h = (ly + 1) * HX + (lx + 1);
    double num[NS], den[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) num[q] = den[q] = 0.0;

    comb_mark(1);
    form_plane<S, NS>(a, x0, y0, 0, Cs, ring);
    if (a.nz > 1) form_plane<S, NS>(a, x0, y0, 1, Cs, ring + HC * NS);
    __syncthreads();
    comb_mark(2);
    for (int z = 0; z < a.nz; ++z) {
        const double* Tm = ring + ((z + nring - 1) % nring) * HC * NS;
        const double* T0 = ring + (z % nring) * HC * NS;
        const double* Tp = ring + ((z + 1) % nring) * HC * NS;
        if (inside) {
            const int64_t i = gx + (int64_t)a.nx * gy + plane * z;
            const double vol = a.volz[z];
            const double rvol = 1.0 / vol;
            const double gi = a.g[i], di = a.diag[i];
            const double czm = z > 0 ? -a.cz[i - plane] : 0.0;
            const double cym = gy > 0 ? -a.cy[i - a.nx] : 0.0;
            const double cxm = gx > 0 ? -a.cx[i - 1] : 0.0;
            const double cxp = gx < a.nx - 1 ? -a.cx[i] : 0.0;
            const double cyp = gy < a.ny - 1 ? -a.cy[i] : 0.0;
            const double czp = z < a.nz - 1 ? -a.cz[i] : 0.0;
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                const int64_t j = j0 + q;
                // y = A T in CSR order z-, y-, x-, diag, x+, y+, z+ (mul, add)
                double y = 0.0;
                if (z > 0) y = __dadd_rn(y, __dmul_rn(czm, Tm[q * HC + h]));
                if (gy > 0) y = __dadd_rn(y, __dmul_rn(cym, T0[q * HC + h - HX]));
                if (gx > 0) y = __dadd_rn(y, __dmul_rn(cxm, T0[q * HC + h - 1]));
                const double tc = T0[q * HC + h];
                y = __dadd_rn(y, __dmul_rn(di, tc));
                if (gx < a.nx - 1) y = __dadd_rn(y, __dmul_rn(cxp, T0[q * HC + h + 1]));
                if (gy < a.ny - 1) y = __dadd_rn(y, __dmul_rn(cyp, T0[q * HC + h + HX]));
                if (z < a.nz - 1) y = __dadd_rn(y, __dmul_rn(czp, Tp[q * HC + h]));
                const double qv = div_rn(__dsub_rn(y, gi), vol, rvol);
                if (j < a.N) {
                    if (a.T) __stcs(a.T + j * a.n + i, tc);
                    if (a.Q) __stcs(a.Q + j * a.n + i, qv);
                    const double bv = fma(vol, qv, gi);
                    const double rv = __dsub_rn(y, bv);
                    num[q] = fma(rv, rv, num[q]);
                    den[q] = fma(bv, bv, den[q]);
                }
            }
        }
        __syncthreads();
        comb_mark(3 + 2 * z);
        if (z + 2 < a.nz) {
            form_plane<S, NS>(a, x0, y0, z + 2, Cs, ring + ((z + 2) % 3) * HC * NS);
            __syncthreads();
        }
        comb_mark(4 + 2 * z);
    }

    if (a.part) {
        // CTA reduction of the residual partials, fixed order. Warp level: a
        // transpose-reduce of the V = 2 NS per-lane sums (V - 1 shuffles, plus
        // one when V = 16); lane L ends with sum L / (32 / V): num of sample k
        // for k < NS, den of sample k - NS otherwise. Then warps in index order.
        // Reuses the ring buffer.
        constexpr int V = 2 * NS;
        static_assert(V == 16 || V == 32, "NS = 8 or 16");
        const int lane = tid & 31, warp = tid >> 5;
        double* red = ring;  // 8 warps x V
        double v[V];
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            v[q] = num[q];
            v[NS + q] = den[q];
        }
#pragma unroll
        for (int o = 16, len = V; o >= 32 / V; o >>= 1, len >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < len / 2; ++i) {
                const double keep = up ? v[len / 2 + i] : v[i];
                const double send = up ? v[i] : v[len / 2 + i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        if (V == 16) v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        if (lane % (32 / V) == 0) red[warp * V + lane / (32 / V)] = v[0];
        __syncthreads();
        if (tid < NS && j0 + tid < a.N) {
            double u = 0.0, w = 0.0;
            for (int k = 0; k < NT / 32; ++k) {
                u += red[k * V + tid];
                w += red[k * V + NS + tid];
            }
            double* pp = a.part + ((j0 + tid) * (int64_t)a.tiles + tile) * 2;
            *reinterpret_cast<double2*>(pp) = make_double2(u, w);
        }
    }
}

// resid_j = sqrt(num / den) over the tiles (one warp per sample: lane-strided
// sums, then a fixed shuffle tree — deterministic); de == 0 handled as
// pipeline.cpp:570-571.
__global__ void resid_finalize(const double* __restrict__ part, int tiles, int64_t N,
                               double* __restrict__ resid) {
    const int lane = threadIdx.x & 31;
    const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (j >= N) return;
    const double2* p = reinterpret_cast<const double2*>(part) + j * tiles;
    double nu = 0.0, de = 0.0;
    for (int t = lane; t < tiles; t += 32) {
        const double2 v = p[t];
        nu += v.x;
        de += v.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nu += __shfl_xor_sync(0xffffffffu, nu, o);
        de += __shfl_xor_sync(0xffffffffu, de, o);
    }
    if (lane == 0) resid[j] = de == 0.0 ? (nu == 0.0 ? 0.0 : 1.0) : sqrt(nu / de);
}

template <int S, int NS>
bk_status run(bk_ctx* ctx, const bk_operator* op, const double* X, int s, const double* C,
              int64_t ldc, int64_t N, double* T, double* Q, double* resid) {
    using namespace bk;
    ActArgs a;
    a.nx = op->nx;
    a.ny = op->ny;
    a.nz = op->nz;
    a.n = op->n;
    a.N = N;
    a.ldc = ldc;
    a.diag = op->diag;
    a.cx = op->cx;
    a.cy = op->cy;
    a.cz = op->cz;
    a.g = op->g;
    a.volz = op->volz;
    a.X = X;
    a.C = C;
    a.T = T;
    a.Q = Q;
    a.s = s;
    const int tilesx = (op->nx + TX - 1) / TX, tilesy = (op->ny + TY - 1) / TY;
    const int tiles = tilesx * tilesy;
    a.part = nullptr;
    a.tiles = tiles;
    if (resid) {
        void* p;
        bk_status st = workspace(ctx, kSlotActPart, (size_t)tiles * N * 2 * sizeof(double), &p);
        if (st != BK_OK) return st;
        a.part = (double*)p;
    }
    const int nring = op->nz < 3 ? op->nz : 3;
    const size_t smem = (size_t)(S * CSTRIDE(NS) + nring * HC * NS) * sizeof(double);
    auto kern = combine_action_kernel<S, NS>;
    BK_CUDA_TRY(ctx, bk::set_max_smem((const void*)kern, smem));
    const int64_t chunks = (N + NS - 1) / NS;
    if (tiles > 65535) return fail(ctx, BK_INVALID_CONFIG, "combine_action: grid too large");
    kern<<<dim3((unsigned)chunks, (unsigned)tiles), NT, smem, ctx->stream>>>(a);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    if (getenv("BK_COMB_PROFILE")) {
        long long h[64];
        cudaStreamSynchronize(ctx->stream);
        cudaMemcpyFromSymbol(h, g_comb_prof, sizeof(h));
        fprintf(stderr, "[bk_comb_profile S=%d nz=%d] cycles: C load %lld, first planes %lld;", S,
                op->nz, h[1] - h[0], h[2] - h[1]);
        for (int z = 0; z < op->nz && 4 + 2 * z < 64; ++z)
            fprintf(stderr, " z%d stencil %lld form %lld;", z, h[3 + 2 * z] - (z ? h[2 + 2 * z] : h[2]),
                    h[4 + 2 * z] - h[3 + 2 * z]);
        fprintf(stderr, "\n");
    }
    if (resid) {
        resid_finalize<<<(unsigned)((N + 7) / 8), 256, 0, ctx->stream>>>(a.part, tiles, N, resid);
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaGetLastError());
    }
    return BK_OK;
}

}  // namespace

namespace bk {

// X is the kernel-width block n x S (zero-padded past the real width s); C is
// s x N with row stride ldc.
bk_status combine_action_device(bk_ctx* ctx, const bk_operator* op, const double* X, int S,
                                int s, const double* C, int64_t ldc, int64_t N, double* T,
                                double* Q, double* resid) {
    if (N == 0) return BK_OK;
    if (s < 1 || s > S || ldc < N) return fail(ctx, BK_INTERNAL, "combine_action: bad widths");
    switch (S) {
        // 16 samples per CTA for a single plane; 8 for 3D grids, whose
        // 3-plane T ring then fits 3 CTAs per SM
        case 8: return op->nz == 1 ? run<8, 16>(ctx, op, X, s, C, ldc, N, T, Q, resid)
                                   : run<8, 8>(ctx, op, X, s, C, ldc, N, T, Q, resid);
        case 16: return op->nz == 1 ? run<16, 16>(ctx, op, X, s, C, ldc, N, T, Q, resid)
                                    : run<16, 8>(ctx, op, X, s, C, ldc, N, T, Q, resid);
        case 32: return op->nz == 1 ? run<32, 16>(ctx, op, X, s, C, ldc, N, T, Q, resid)
                                    : run<32, 8>(ctx, op, X, s, C, ldc, N, T, Q, resid);
        case 64: return op->nz == 1 ? run<64, 16>(ctx, op, X, s, C, ldc, N, T, Q, resid)
                                    : run<64, 8>(ctx, op, X, s, C, ldc, N, T, Q, resid);
        default: return fail(ctx, BK_INTERNAL, "combine_action: unpadded width");
    }
}

}  // namespace bk
