// Fused combination + operator action: one pass writes every (T, q) sample.
//
//   T_j = sum_t C[t][j] X[:,t]        combine_from_weights  pipeline.cpp:187-225
//   q_j = (A T_j - g) / V             operator_action       pipeline.cpp:242-251
//   resid_j = ||A T_j - (V q_j + g)|| / ||V q_j + g||       pipeline.cpp:548-571
//
// Work item = (32 x 8 x-y tile of cells, all z, chunk of NS samples).
// Persistent CTAs (two per SM) walk their items; for each z-plane
// the tile's X rows plus a one-cell x-y halo (34 x 10 cells) arrive by TMA:
// one 4D tensor-map copy per 16-column panel (box 16 x 34 x 10 x 1, 128-byte
// swizzle, out-of-domain halo cells zero-filled by the copy engine) into a
// mbarrier-tracked slot that the producer refills as soon as it is consumed,
// running ahead across planes and items. T for the
// halo plane is formed from the swizzled panels on the FP64 tensor cores
// (m16n8k4 DMMA: M = halo cells, N = samples, K = basis columns) into a ring
// of three T planes; the 7-point stencil is then applied from shared memory
// (2.5D march: the ring supplies z - 1 / z + 1), and T and q leave the SM
// exactly once, sample-major, with streaming stores. No T round trip through
// HBM, no second pass for q.
//
// Why this shape (ncu, profiles/): the previous kernel read the DMMA A
// fragments (8 bytes per lane, 8 rows per instruction) straight from L2; the
// L1 data pipe spent one wavefront per 32-byte sector and ran at 94 % busy,
// 58 % of it on X. TMA moves X without L1 wavefronts; each swizzled fragment
// load is two wavefronts per 256 bytes (conflict free).
//
// Bitwise contract: T uses the reference's per-element order (first term a
// product, then one fma per basis column in ascending order — the DMMA's
// accumulation order, verified bitwise; panels and k-steps are consumed in
// ascending column order); A T uses the scalar CsrMatrix::apply order
// (separate multiply and add, CSR column order); q = (y - g) / V is correctly
// rounded. So given the same X, T and q equal the reference's bit for bit
// (tests/test_gpu_parity.py checks it).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "bk_common.cuh"

namespace {

constexpr int TX = 32, TY = 8, HX = TX + 2, HY = TY + 2, HC = HX * HY;  // 340 halo cells
constexpr int MT = (HC + 15) / 16;     // DMMA m-tiles per halo plane (22)

// Work-item shape: NS samples per item, NT threads. NT = 512 runs one CTA per
// SM (thread = interior cell x 8 samples, two sample halves) with two TMA
// panel slots; NT = 256 runs two CTAs per SM (thread = interior cell x NS
// samples) with one slot each, so one CTA's stencil overlaps the other's DMMA
// chains.
template <int NS, int NT_>
struct Shape {
    static constexpr int NT = NT_;
    static constexpr int NW = NT / 32;
    static constexpr int MPW = (MT + NW - 1) / NW;  // m-tiles per warp
    static constexpr int NB = NS / 8;               // DMMA n-blocks (8 samples each)
    static constexpr int SPT = NS * 256 / NT;       // samples per thread
    static constexpr int NP = NT == 512 ? 2 : 1;    // TMA panel slots
    static constexpr int CSP = NS + 4;              // row stride of C in shared memory
    static constexpr int CTAS = NT == 512 ? 1 : 2;  // CTAs per SM
};

// A panel = PW basis columns of every halo cell of one plane (one TMA box).
template <int S>
struct Panel {
    static constexpr int PW = S >= 16 ? 16 : 8;
    static constexpr int R = S / PW;                        // panels per plane
    static constexpr unsigned BYTES = HC * PW * 8;          // transaction bytes
    static constexpr int SLOT = (BYTES + 1023) / 1024 * 1024;
    static constexpr unsigned SWM = PW == 16 ? 7 : 3;       // 128- / 64-byte swizzle
};

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
    const double* C;  // S x N
    double* T;        // N x n (nullable)
    double* Q;        // N x n (nullable)
    double* part;     // N x tiles x 2 residual partials (nullable)
    int tilesx, tiles;
    int chunks, items;  // items = chunks x tiles < 2^31 (checked on the host)
    int s;            // real basis width (<= S)
    // generate_blockoa extras (bk::ActExtra): output / noise row stride, the
    // per-sample interior noise added to T before the action, and the
    // stencil's rounding order
    int64_t ldo;
    const double* eps;  // N x ldo (nullable)
    int fma;            // 1: apply_block's fused chain, 0: scalar apply's mul + add
    // slab of the y-slab decomposition: local rows 0 .. ny - 1 are global rows
    // cy0 .. cy0 + ny - 1 of a grid with cny rows (coefficients and boundary
    // tests use global rows; outputs are slab-local); X carries one ghost row
    // per side, so the tensor map's y coordinate is shifted by ty = 1
    int cy0, cny, ty;
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
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tCMW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra CMW_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 4D tiled TMA load: box (PW, 34, 10, 1) at (col, x0 - 1, y0 - 1, z)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
        : "memory");
}

// debug: stage timestamps (clock64) of CTA 0's fifth work item when
// BK_COMB_PROFILE is set
__device__ long long g_comb_prof[64];

// the stencil coefficients of one cell (CSR values of its row)
struct Coef {
    double gi, di, zm, ym, xm, xp, yp, zp;
};
__device__ __forceinline__ void load_coef(const ActArgs& a, int gx, int gy, int z, Coef& k) {
    const int gyg = gy + a.cy0;  // global row
    const int64_t plane = (int64_t)a.nx * a.cny;
    const int64_t i = gx + (int64_t)a.nx * gyg + plane * z;
    k.gi = a.g[i];
    k.di = a.diag[i];
    k.zm = z > 0 ? -a.cz[i - plane] : 0.0;
    k.ym = gyg > 0 ? -a.cy[i - a.nx] : 0.0;
    k.xm = gx > 0 ? -a.cx[i - 1] : 0.0;
    k.xp = gx < a.nx - 1 ? -a.cx[i] : 0.0;
    k.yp = gyg < a.cny - 1 ? -a.cy[i] : 0.0;
    k.zp = z < a.nz - 1 ? -a.cz[i] : 0.0;
}

// PL: single-plane grid (nz == 1), compiled without the z-ring logic
template <int S, int NS, int NT_, bool PL>
__global__ void __launch_bounds__(NT_, Shape<NS, NT_>::CTAS)
    combine_action_kernel(const __grid_constant__ CUtensorMap tmx, ActArgs a) {
    using P = Panel<S>;
    using SH = Shape<NS, NT_>;
    constexpr int NT = SH::NT, NW = SH::NW, MPW = SH::MPW, NB = SH::NB, NP = SH::NP, CSP = SH::CSP;
    // Single-plane kernels (PL): thread = (pair of x-adjacent cells, half of the
    // NS samples); the T ring rows are padded to HXR = 36 with the interior
    // starting at an even index, so a pair and its y-neighbour pairs are single
    // 16-byte loads (5 shared loads per pair instead of 7 per cell).
    constexpr int SPT = PL ? NS / 2 : SH::SPT;       // samples per thread
    constexpr int HALVES = PL ? 2 : (NT == 512 ? 2 : 1);
    constexpr int WPH = NW / HALVES;                 // warps per sample half
    constexpr int HXR = PL ? 36 : HX;                // ring row stride
    constexpr int HCR = PL ? HY * 36 + 4 : HC;       // ring sample stride (4 mod 8)
    extern __shared__ unsigned char smraw[];
    unsigned char* panels = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
    const int nz = PL ? 1 : a.nz;
    const int nring = nz < 3 ? nz : 3;
    double* ring = reinterpret_cast<double*>(panels + NP * P::SLOT);  // nring x NS x HCR
    double* Cs = ring + nring * NS * HCR;                               // S x CSP
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(Cs + S * CSP);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int64_t plane = (int64_t)a.nx * a.ny;

    if (tid == 0) {
        for (int p = 0; p < NP; ++p) mbar_init(&bar[p], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // Single plane: each CTA owns a contiguous range of items (sample chunk
    // fastest), so it stays on one tile for many chunks and loads the tile's
    // coefficients and X panel once per tile. 3D: items strided by the grid,
    // so the CTAs resident at once share one tile's X planes through L2
    // (contiguous ranges measured slower there: C3 5.97 -> 6.47 ms).
    const int i_begin = PL ? (int)((int64_t)blockIdx.x * a.items / gridDim.x) : (int)blockIdx.x;
    const int i_end = PL ? (int)((int64_t)(blockIdx.x + 1) * a.items / gridDim.x) : a.items;
    const int i_step = PL ? 1 : (int)gridDim.x;
    constexpr bool KEEP = PL && P::R == 1 && NP == 1;  // panel kept across a tile's items
    // producer (thread 0): walks the panels in consumption order (item, z,
    // column block); slot = panel index mod NP. KEEP: one panel per tile.
    int p_item = i_begin, p_z = 0, p_r = 0, p_slot = 0;
    auto issue = [&]() {
        if (p_item >= i_end) return;
        const int tile = p_item / a.chunks;
        const int x0 = (tile % a.tilesx) * TX, y0 = (tile / a.tilesx) * TY;
        mbar_expect_tx(&bar[p_slot], P::BYTES);
        tma_load_4d(panels + p_slot * P::SLOT, &tmx, p_r * P::PW, x0 - 1, y0 - 1 + a.ty, p_z,
                    &bar[p_slot]);
        p_slot = p_slot + 1 == NP ? 0 : p_slot + 1;
        if (++p_r == P::R) {
            p_r = 0;
            if (++p_z == nz) {
                p_z = 0;
                p_item += i_step;
                if (KEEP)  // next panel: the next tile's
                    while (p_item < i_end && p_item / a.chunks == (p_item - 1) / a.chunks) ++p_item;
            }
        }
    };
    if (tid == 0)
        for (int p = 0; p < NP; ++p) issue();
    unsigned pc = 0;  // panels consumed (uniform across the CTA)
    bool prof = false;
    int pm = 0;
    auto mark = [&]() {
        if (prof && pm < 64) g_comb_prof[pm++] = clock64();
    };

    int ix0 = 0, iy0 = 0;  // current item: tile origin and first sample
    int64_t ij0 = 0;
    bool new_tile = true, last_of_tile = true;  // KEEP: panel / coefficient reuse
    // T + eps at halo cell h of plane z for item sample q (eps is zero outside
    // the domain, where T is zero-filled too): combine_from_weights' noise add
    // (pipeline.cpp:220-223, 470-503)
    auto noisy = [&](double v, int h, int q, int z) {
        const int gx = ix0 - 1 + h % HX, gy = iy0 - 1 + h / HX;
        if (gx < 0 || gx >= a.nx || gy < 0 || gy >= a.ny || ij0 + q >= a.N) return v;
        return __dadd_rn(v, a.eps[(ij0 + q) * a.ldo + gx + (int64_t)a.nx * (gy + (int64_t)a.ny * z)]);
    };
    // DMMA accumulators of m-tile mt (all NB sample blocks) -> T ring plane buf,
    // sample-major [q][h] (conflict-free: HC = 4 mod 8)
    // ring index of halo cell h (box order hy * 34 + hx)
    auto ridx = [&](int hh) { return PL ? (hh / HX) * HXR + hh % HX + 1 : hh; };
    auto store_tile = [&](int mt, const double (&ac)[NB][4], double* buf, int z) {
        const int h0 = 16 * mt + g, h1 = h0 + 8;
        const int r0 = ridx(h0), r1 = ridx(h1);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            const int q = 8 * nb + 2 * t;
            double v[4] = {ac[nb][0], ac[nb][1], ac[nb][2], ac[nb][3]};
            if (a.eps) {
                if (h0 < HC) {
                    v[0] = noisy(v[0], h0, q, z);
                    v[1] = noisy(v[1], h0, q + 1, z);
                }
                if (h1 < HC) {
                    v[2] = noisy(v[2], h1, q, z);
                    v[3] = noisy(v[3], h1, q + 1, z);
                }
            }
            if (h0 < HC) {
                buf[q * HCR + r0] = v[0];
                buf[(q + 1) * HCR + r0] = v[1];
            }
            if (h1 < HC) {
                buf[q * HCR + r1] = v[2];
                buf[(q + 1) * HCR + r1] = v[3];
            }
        }
    };
    // k-steps 0 .. PW/4 of one panel into the accumulators of m-tile mt
    auto mma_tile = [&](const unsigned char* pan, int mt, const double (&bf)[P::PW / 4][NB],
                        double (&ac)[NB][4]) {
        const int h0 = 16 * mt + g;
        // rows h0 and h0 + 8 share the swizzle phase (address bits 7..9)
        const unsigned off0 = (unsigned)h0 * (P::PW * 8);
        const unsigned xr = ((off0 >> 7) & P::SWM) << 4;
        const unsigned char* r0 = pan + off0;
        const bool v0 = h0 < HC, v1 = h0 + 8 < HC;
#pragma unroll
        for (int kk = 0; kk < P::PW / 4; ++kk) {
            const unsigned kx = ((unsigned)(4 * kk + t) * 8u) ^ xr;
            const double a0 = v0 ? *reinterpret_cast<const double*>(r0 + kx) : 0.0;
            const double a1 = v1 ? *reinterpret_cast<const double*>(r0 + 8 * P::PW * 8 + kx) : 0.0;
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) dmma_c(ac[nb], a0, a1, bf[kk][nb]);
        }
    };
    // T of halo plane z (all NS samples) into ring slot z % 3. Panels arrive
    // in ascending column order, so each accumulator sees k ascending.
    auto form = [&](int z) {
        double* buf = ring + (z % 3) * NS * HCR;
        if constexpr (P::R == 1) {
            // one panel per plane: finish and store each m-tile in turn
            const int slot = (int)(pc % NP);
            if (!KEEP || new_tile) mbar_wait(&bar[slot], (pc / NP) & 1u);
            const unsigned char* pan = panels + slot * P::SLOT;
            double bf[P::PW / 4][NB];
#pragma unroll
            for (int kk = 0; kk < P::PW / 4; ++kk)
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) bf[kk][nb] = Cs[(4 * kk + t) * CSP + 8 * nb + g];
            for (int mt = warp; mt < MT; mt += NW) {
                double ac[NB][4];
#pragma unroll
                for (int nb = 0; nb < NB; ++nb)
#pragma unroll
                    for (int e = 0; e < 4; ++e) ac[nb][e] = 0.0;
                mma_tile(pan, mt, bf, ac);
                store_tile(mt, ac, buf, z);
            }
            __syncthreads();  // every warp is done with this slot
            if (!KEEP || last_of_tile) {
                if (tid == 0) issue();
                ++pc;
            }
        } else {
            double acc[MPW][NB][4];
#pragma unroll
            for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
                for (int nb = 0; nb < NB; ++nb)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[mi][nb][e] = 0.0;
            for (int r = 0; r < P::R; ++r) {
                const int slot = (int)(pc % NP);
                mbar_wait(&bar[slot], (pc / NP) & 1u);
                const unsigned char* pan = panels + slot * P::SLOT;
                double bf[P::PW / 4][NB];
#pragma unroll
                for (int kk = 0; kk < P::PW / 4; ++kk)
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb)
                        bf[kk][nb] = Cs[(r * P::PW + 4 * kk + t) * CSP + 8 * nb + g];
#pragma unroll
                for (int mi = 0; mi < MPW; ++mi)
                    if (warp + NW * mi < MT) mma_tile(pan, warp + NW * mi, bf, acc[mi]);
                __syncthreads();  // every warp is done with this slot
                if (tid == 0) issue();
                ++pc;
            }
#pragma unroll
            for (int mi = 0; mi < MPW; ++mi)
                if (warp + NW * mi < MT) store_tile(warp + NW * mi, acc[mi], buf, z);
        }
    };

    // PL: pair p = tid & 127 covers cells (2 (p % 16), p / 16) and its x + 1
    const int cell = PL ? 2 * (tid & 127) : (tid & 255);
    const int qh = PL ? tid >> 7 : (NT == 512 ? tid >> 8 : 0);
    const int lx = cell % TX, ly = cell / TX;
    const int h = (ly + 1) * HX + (lx + 1);

    Coef k{}, k2{};  // k2: the second cell of a planar pair
    int prev_tile = -1;
    for (int item = i_begin; item < i_end; item += i_step) {
        const int chunk = item % a.chunks;
        const int tile = item / a.chunks;
        new_tile = tile != prev_tile;
        last_of_tile = item + i_step >= i_end || (item + i_step) / a.chunks != tile;
        prev_tile = tile;
        const int x0 = (tile % a.tilesx) * TX, y0 = (tile / a.tilesx) * TY;
        const int64_t j0 = (int64_t)chunk * NS;
        ix0 = x0;
        iy0 = y0;
        ij0 = j0;
        prof = blockIdx.x == 0 && tid == 0 && item == i_begin + 4 * i_step;
        pm = 0;
        mark();
        for (int e = tid; e < S * NS; e += NT) {
            const int k = e / NS, q = e % NS;
            Cs[k * CSP + q] = (k < a.s && j0 + q < a.N) ? a.C[(int64_t)k * a.ldc + j0 + q] : 0.0;
        }
        const int gx = x0 + lx, gy = y0 + ly;
        const bool inside = gx < a.nx && gy < a.ny;
        const bool inside2 = PL && gx + 1 < a.nx && gy < a.ny;  // the pair's second cell
        Coef kn{};
        // planar: the pair's coefficients persist across the tile's items
        if (!PL || new_tile) {
            if (inside) load_coef(a, gx, gy, 0, k);
            if (inside2) load_coef(a, gx + 1, gy, 0, k2);
        }
        double num[SPT], den[SPT];
#pragma unroll
        for (int q = 0; q < SPT; ++q) num[q] = den[q] = 0.0;
        __syncthreads();  // Cs ready
        mark();

        form(0);
        if (nz > 1) form(1);
        // one panel per plane: form already ended with a barrier after its
        // T stores; otherwise the stores follow the last panel's barrier
        if (P::R > 1) __syncthreads();
        mark();
        for (int z = 0; z < nz; ++z) {
            if (inside && z + 1 < nz) load_coef(a, gx, gy, z + 1, kn);
            // ring slots of planes z - 1, z, z + 1, offset to this thread's
            // cell and sample half (compile-time offsets below)
            const int sz = z % nring;
            const int sm1 = sz == 0 ? nring - 1 : sz - 1, sp1 = sz + 1 == nring ? 0 : sz + 1;
            const double* b0 = ring + sz * NS * HC + SPT * qh * HC + h;
            const double* bm = ring + sm1 * NS * HC + SPT * qh * HC + h;
            const double* bp = ring + sp1 * NS * HC + SPT * qh * HC + h;
            const bool hzm = z > 0, hzp = z < nz - 1;  // CTA-uniform
            if (PL && inside) {
                // pair (A = x, B = x + 1): 16-byte loads of (A, B) centre and
                // y -+ 1 rows, 8-byte loads of x - 1 and x + 2; each cell's y in
                // CSR order y-, x-, diag, x+, y+ exactly as the scalar path
                const int hb = (ly + 1) * HXR + lx + 2;  // even: 16-byte aligned
                const double* b = ring + SPT * qh * HCR + hb;
                const int64_t i = gx + (int64_t)a.nx * gy;
                const int64_t jb = j0 + SPT * qh;
                double* pt = a.T ? a.T + jb * a.ldo + i : nullptr;
                double* pq = a.Q ? a.Q + jb * a.ldo + i : nullptr;
                const int nv = a.N - jb < SPT ? (int)(a.N - jb) : SPT;
                const double vol = a.volz[0];
                const double rvol = 1.0 / vol;
                const bool vec = inside2 && ((i | a.ldo) & 1) == 0;  // 16-byte stores
#pragma unroll
                for (int qq = 0; qq < SPT; ++qq) {
                    const double2 c2 = *reinterpret_cast<const double2*>(b + qq * HCR);
                    const double2 m2 = *reinterpret_cast<const double2*>(b + qq * HCR - HXR);
                    const double2 p2 = *reinterpret_cast<const double2*>(b + qq * HCR + HXR);
                    const double xl = b[qq * HCR - 1], xr = b[qq * HCR + 2];
                    double ya, yb;
                    // first term added to +0.0 as the scalar path does (a -0
                    // product must not survive as y)
                    if (!a.fma) {
                        ya = __dadd_rn(0.0, __dmul_rn(k.ym, m2.x));
                        ya = __dadd_rn(ya, __dmul_rn(k.xm, xl));
                        ya = __dadd_rn(ya, __dmul_rn(k.di, c2.x));
                        ya = __dadd_rn(ya, __dmul_rn(k.xp, c2.y));
                        ya = __dadd_rn(ya, __dmul_rn(k.yp, p2.x));
                        yb = __dadd_rn(0.0, __dmul_rn(k2.ym, m2.y));
                        yb = __dadd_rn(yb, __dmul_rn(k2.xm, c2.x));
                        yb = __dadd_rn(yb, __dmul_rn(k2.di, c2.y));
                        yb = __dadd_rn(yb, __dmul_rn(k2.xp, xr));
                        yb = __dadd_rn(yb, __dmul_rn(k2.yp, p2.y));
                    } else {
                        ya = __fma_rn(k.ym, m2.x, 0.0);
                        ya = __fma_rn(k.xm, xl, ya);
                        ya = __fma_rn(k.di, c2.x, ya);
                        ya = __fma_rn(k.xp, c2.y, ya);
                        ya = __fma_rn(k.yp, p2.x, ya);
                        yb = __fma_rn(k2.ym, m2.y, 0.0);
                        yb = __fma_rn(k2.xm, c2.x, yb);
                        yb = __fma_rn(k2.di, c2.y, yb);
                        yb = __fma_rn(k2.xp, xr, yb);
                        yb = __fma_rn(k2.yp, p2.y, yb);
                    }
                    const double qa = div_rn(__dsub_rn(ya, k.gi), vol, rvol);
                    const double qb = div_rn(__dsub_rn(yb, k2.gi), vol, rvol);
                    if (qq < nv) {
                        if (vec) {
                            if (pt) __stcs(reinterpret_cast<double2*>(pt), c2);
                            if (pq) __stcs(reinterpret_cast<double2*>(pq), make_double2(qa, qb));
                        } else {
                            if (pt) __stcs(pt, c2.x);
                            if (pq) __stcs(pq, qa);
                            if (inside2 && pt) __stcs(pt + 1, c2.y);
                            if (inside2 && pq) __stcs(pq + 1, qb);
                        }
                        const double ba = fma(vol, qa, k.gi);
                        const double ra = __dsub_rn(ya, ba);
                        num[qq] = fma(ra, ra, num[qq]);
                        den[qq] = fma(ba, ba, den[qq]);
                        if (inside2) {
                            const double bb = fma(vol, qb, k2.gi);
                            const double rb = __dsub_rn(yb, bb);
                            num[qq] = fma(rb, rb, num[qq]);
                            den[qq] = fma(bb, bb, den[qq]);
                        }
                    }
                    pt += a.ldo;
                    pq += a.ldo;
                }
            }
            if (!PL && inside) {
                const int64_t i = gx + (int64_t)a.nx * gy + plane * z;
                const int64_t jb = j0 + SPT * qh;
                double* pt = a.T ? a.T + jb * a.ldo + i : nullptr;
                double* pq = a.Q ? a.Q + jb * a.ldo + i : nullptr;
                const int nv = a.N - jb < SPT ? (int)(a.N - jb) : SPT;  // valid samples
                const double vol = a.volz[z];
                const double rvol = 1.0 / vol;
#pragma unroll
                for (int qq = 0; qq < SPT; ++qq) {
                    // y = A T in CSR order z-, y-, x-, diag, x+, y+, z+ (mul, add).
                    // In-plane neighbours outside the domain have a zero
                    // coefficient and a zero-filled T: adding the +-0 product
                    // leaves y bitwise unchanged (y is never -0), as skipping does
                    double y = 0.0;
                    const double tc = b0[qq * HC];
                    if (!a.fma) {
                        if (hzm) y = __dadd_rn(y, __dmul_rn(k.zm, bm[qq * HC]));
                        y = __dadd_rn(y, __dmul_rn(k.ym, b0[qq * HC - HX]));
                        y = __dadd_rn(y, __dmul_rn(k.xm, b0[qq * HC - 1]));
                        y = __dadd_rn(y, __dmul_rn(k.di, tc));
                        y = __dadd_rn(y, __dmul_rn(k.xp, b0[qq * HC + 1]));
                        y = __dadd_rn(y, __dmul_rn(k.yp, b0[qq * HC + HX]));
                        if (hzp) y = __dadd_rn(y, __dmul_rn(k.zp, bp[qq * HC]));
                    } else {
                        // CsrMatrix::apply_block's chain (discretize.cpp:57-95)
                        if (hzm) y = __fma_rn(k.zm, bm[qq * HC], y);
                        y = __fma_rn(k.ym, b0[qq * HC - HX], y);
                        y = __fma_rn(k.xm, b0[qq * HC - 1], y);
                        y = __fma_rn(k.di, tc, y);
                        y = __fma_rn(k.xp, b0[qq * HC + 1], y);
                        y = __fma_rn(k.yp, b0[qq * HC + HX], y);
                        if (hzp) y = __fma_rn(k.zp, bp[qq * HC], y);
                    }
                    const double qv = div_rn(__dsub_rn(y, k.gi), vol, rvol);
                    if (qq < nv) {
                        if (pt) __stcs(pt, tc);
                        if (pq) __stcs(pq, qv);
                        const double bv = fma(vol, qv, k.gi);
                        const double rv = __dsub_rn(y, bv);
                        num[qq] = fma(rv, rv, num[qq]);
                        den[qq] = fma(bv, bv, den[qq]);
                    }
                    pt += a.ldo;
                    pq += a.ldo;
                }
            }
            if (!PL) k = kn;  // planar: k persists across the tile's items
            __syncthreads();
            mark();
            if (z + 2 < nz) {
                form(z + 2);
                if (P::R > 1) __syncthreads();
            }
            mark();
        }

        if (a.part) {
            // fixed-order reduction of the residual partials over the tile's
            // cells. Warp level: transpose-reduce of the V = 2 SPT per-lane
            // sums (num of the thread's samples, then den); lane L ends with
            // sum L / (32 / V). Then the 8 warps of each sample half in index
            // order. Reuses ring.
            constexpr int V = 2 * SPT;
            static_assert(V == 16 || V == 32, "SPT = 8 or 16");
            double* red = ring;  // NW x V
            double v[V];
#pragma unroll
            for (int q = 0; q < SPT; ++q) {
                v[q] = num[q];
                v[SPT + q] = den[q];
            }
#pragma unroll
            for (int o = 16, len = V; o >= 32 / V; o >>= 1, len >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int e = 0; e < len / 2; ++e) {
                    const double keep = up ? v[len / 2 + e] : v[e];
                    const double send = up ? v[e] : v[len / 2 + e];
                    v[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            if (V == 16) v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
            if (lane % (32 / V) == 0) red[warp * V + lane / (32 / V)] = v[0];
            __syncthreads();
            if (tid < NS && j0 + tid < a.N) {
                const int hq = tid / SPT, qq = tid % SPT;
                double u = 0.0, w = 0.0;
                for (int w2 = 0; w2 < WPH; ++w2) {  // the warps of sample half hq
                    u += red[(WPH * hq + w2) * V + qq];
                    w += red[(WPH * hq + w2) * V + SPT + qq];
                }
                double* pp = a.part + ((j0 + tid) * (int64_t)a.tiles + tile) * 2;
                *reinterpret_cast<double2*>(pp) = make_double2(u, w);
            }
        }
        __syncthreads();  // ring and Cs free for the next item
        mark();
    }
}

// ---------------------------------------------------------------------------
// Single-plane grids with one panel per plane (S <= 16: configs 1 and 2):
// warp-specialised form (C2, 2048 samples: 0.66 ms vs 0.71 ms one-role). 4 former warps build T of a work
// item's halo plane on DMMA into a two-buffer ring while 8 stencil warps apply
// the operator to the previous item and stream T / q out, so the HBM writes,
// the DMMA chains and the stencil's shared-memory loads of different items
// overlap (the one-role kernel ran them back to back: ncu C2, FP64 pipe 21 %,
// 4 CTA barriers per item). Same arithmetic as combine_action_kernel<.., PL>
// (bitwise the same T, q and residual partials): former warp w owns m-tiles
// w, w + 4, ...; the stencil warps map thread = (cell pair, sample half)
// exactly as that kernel's 8 warps do.
// Hand-offs: tfull[b] (NF former arrivals) / tempty[b] (stencil-warp arrivals)
// per ring buffer; the panel (the tile's X halo) is reloaded by TMA when the
// former warps reach a new tile (named barrier 1 among them first); the
// residual reduction needs one named barrier (2) among the stencil warps per
// item, with a two-buffer partial array.
// ---------------------------------------------------------------------------
template <int S, int NS, int NQ, int NF, int NR>
__global__ void __launch_bounds__(32 * NF + 128 * NQ, 1)
    combine_action_pl_ws(const __grid_constant__ CUtensorMap tmx, ActArgs a) {
    using P = Panel<S>;
    static_assert(P::R == 1, "one panel per plane");
    // NQ sample groups of the stencil warps (4 NQ warps, thread = cell pair x
    // sample group of SPT samples): more warps = more independent FP64 chains
    constexpr int NB = NS / 8, SPT = NS / NQ, V = 2 * SPT, NSW = 4 * NQ;
    // ring sample stride 2 mod 8: the former warps' T stores (lanes: 8 halo
    // cells x 4 sample pairs) are conflict-free
    constexpr int HXR = 36, HCR = HY * 36 + 2;
    extern __shared__ unsigned char smraw[];
    unsigned char* panel = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
    double* ring = reinterpret_cast<double*>(panel + P::SLOT);  // 2 x NS x HCR
    double* red = ring + NR * NS * HCR;                          // 2 x NSW warps x V
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(red + 2 * NSW * V);
    unsigned long long* tfull = bar;        // [NR]
    unsigned long long* tempty = bar + NR;  // [NR]
    unsigned long long* pbar = bar + 2 * NR;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    if (tid == 0) {
        for (int b = 0; b < NR; ++b) {
            mbar_init(&tfull[b], NF);
            mbar_init(&tempty[b], NSW);
        }
        mbar_init(pbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int i_begin = (int)((int64_t)blockIdx.x * a.items / gridDim.x);
    const int i_end = (int)((int64_t)(blockIdx.x + 1) * a.items / gridDim.x);
    auto ridx = [&](int hh) { return (hh / HX) * HXR + hh % HX + 1; };

    if (warp < NF) {  // ---- former warps
        int cur_tile = -1;
        unsigned pph = 0;
        // B fragments (coefficients C) of the next item, loaded one item ahead
        // so the global-load latency hides behind this item's DMMA chains
        double bfn[P::PW / 4][NB];
        auto load_bf = [&](int item) {
            const int64_t jn = (int64_t)(item % a.chunks) * NS;
#pragma unroll
            for (int kk = 0; kk < P::PW / 4; ++kk)
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) {
                    const int k = 4 * kk + t;
                    const int64_t q = jn + 8 * nb + g;
                    bfn[kk][nb] =
                        (item < i_end && k < a.s && q < a.N) ? a.C[(int64_t)k * a.ldc + q] : 0.0;
                }
        };
        load_bf(i_begin);
        for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
            const int tile = item / a.chunks, chunk = item % a.chunks;
            const int x0 = (tile % a.tilesx) * TX, y0 = (tile / a.tilesx) * TY;
            const int64_t j0 = (int64_t)chunk * NS;
            const int b = it % NR;
            if (it >= NR) mbar_wait(&tempty[b], ((it / NR) - 1) & 1);
            if (tile != cur_tile) {  // every former warp is done with the old panel
                asm volatile("bar.sync 1, %0;" ::"n"(NF * 32) : "memory");
                if (tid == 0) {
                    mbar_expect_tx(pbar, P::BYTES);
                    tma_load_4d(panel, &tmx, 0, x0 - 1, y0 - 1 + a.ty, 0, pbar);
                }
                mbar_wait(pbar, pph);
                pph ^= 1u;
                cur_tile = tile;
            }
            double bf[P::PW / 4][NB];
#pragma unroll
            for (int kk = 0; kk < P::PW / 4; ++kk)
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) bf[kk][nb] = bfn[kk][nb];
            load_bf(item + 1);
            double* buf = ring + b * NS * HCR;
            for (int mt = warp; mt < MT; mt += NF) {
                double ac[NB][4];
#pragma unroll
                for (int nb = 0; nb < NB; ++nb)
#pragma unroll
                    for (int e = 0; e < 4; ++e) ac[nb][e] = 0.0;
                const int h0 = 16 * mt + g;
                const unsigned off0 = (unsigned)h0 * (P::PW * 8);
                const unsigned xr = ((off0 >> 7) & P::SWM) << 4;
                const unsigned char* r0p = panel + off0;
                const bool v0 = h0 < HC, v1 = h0 + 8 < HC;
#pragma unroll
                for (int kk = 0; kk < P::PW / 4; ++kk) {
                    const unsigned kx = ((unsigned)(4 * kk + t) * 8u) ^ xr;
                    const double a0 = v0 ? *reinterpret_cast<const double*>(r0p + kx) : 0.0;
                    const double a1 =
                        v1 ? *reinterpret_cast<const double*>(r0p + 8 * P::PW * 8 + kx) : 0.0;
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb) dmma_c(ac[nb], a0, a1, bf[kk][nb]);
                }
                const int h1 = h0 + 8;
                const int r0 = ridx(h0), r1 = ridx(h1);
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) {
                    const int q = 8 * nb + 2 * t;
                    double v[4] = {ac[nb][0], ac[nb][1], ac[nb][2], ac[nb][3]};
                    if (a.eps) {  // combine_from_weights' noise add (pipeline.cpp:220-223)
                        auto noisy = [&](double val, int hh, int qq) {
                            const int gx = x0 - 1 + hh % HX, gy = y0 - 1 + hh / HX;
                            if (gx < 0 || gx >= a.nx || gy < 0 || gy >= a.ny || j0 + qq >= a.N)
                                return val;
                            return __dadd_rn(val, a.eps[(j0 + qq) * a.ldo + gx + (int64_t)a.nx * gy]);
                        };
                        if (h0 < HC) {
                            v[0] = noisy(v[0], h0, q);
                            v[1] = noisy(v[1], h0, q + 1);
                        }
                        if (h1 < HC) {
                            v[2] = noisy(v[2], h1, q);
                            v[3] = noisy(v[3], h1, q + 1);
                        }
                    }
                    if (h0 < HC) {
                        buf[q * HCR + r0] = v[0];
                        buf[(q + 1) * HCR + r0] = v[1];
                    }
                    if (h1 < HC) {
                        buf[q * HCR + r1] = v[2];
                        buf[(q + 1) * HCR + r1] = v[3];
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&tfull[b]);
        }
        return;
    }

    // ---- stencil warps: thread = (pair of x-adjacent cells, sample group)
    const int tt = tid - 32 * NF, sw = warp - NF;
    const int cell = 2 * (tt & 127), qh = tt >> 7;
    const int lx = cell % TX, ly = cell / TX;
    Coef k{}, k2{};
    int cur_tile = -1;
    for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
        const int tile = item / a.chunks, chunk = item % a.chunks;
        const int x0 = (tile % a.tilesx) * TX, y0 = (tile / a.tilesx) * TY;
        const int64_t j0 = (int64_t)chunk * NS;
        const int gx = x0 + lx, gy = y0 + ly;
        const bool inside = gx < a.nx && gy < a.ny;
        const bool inside2 = gx + 1 < a.nx && gy < a.ny;
        if (tile != cur_tile) {
            if (inside) load_coef(a, gx, gy, 0, k);
            if (inside2) load_coef(a, gx + 1, gy, 0, k2);
            cur_tile = tile;
        }
        const int b = it % NR;
        mbar_wait(&tfull[b], (it / NR) & 1);
        double num[SPT], den[SPT];
#pragma unroll
        for (int q = 0; q < SPT; ++q) num[q] = den[q] = 0.0;
        if (inside) {
            // pair (A = x, B = x + 1): 16-byte loads of (A, B) centre and
            // y -+ 1 rows, 8-byte loads of x - 1 and x + 2; each cell's y in CSR
            // order y-, x-, diag, x+, y+ exactly as the scalar path
            const int hb = (ly + 1) * HXR + lx + 2;
            const double* bp = ring + b * NS * HCR + SPT * qh * HCR + hb;
            const int64_t i = gx + (int64_t)a.nx * gy;
            const int64_t jb = j0 + SPT * qh;
            double* pt = a.T ? a.T + jb * a.ldo + i : nullptr;
            double* pq = a.Q ? a.Q + jb * a.ldo + i : nullptr;
            const int nv = a.N - jb < SPT ? (int)(a.N - jb) : SPT;
            const double vol = a.volz[0];
            const double rvol = 1.0 / vol;
            const bool vec = inside2 && ((i | a.ldo) & 1) == 0;  // 16-byte stores
#pragma unroll
            for (int qq = 0; qq < SPT; ++qq) {
                const double2 c2 = *reinterpret_cast<const double2*>(bp + qq * HCR);
                const double2 m2 = *reinterpret_cast<const double2*>(bp + qq * HCR - HXR);
                const double2 p2 = *reinterpret_cast<const double2*>(bp + qq * HCR + HXR);
                const double xl = bp[qq * HCR - 1], xr = bp[qq * HCR + 2];
                double ya, yb;
                if (!a.fma) {
                    ya = __dadd_rn(0.0, __dmul_rn(k.ym, m2.x));
                    ya = __dadd_rn(ya, __dmul_rn(k.xm, xl));
                    ya = __dadd_rn(ya, __dmul_rn(k.di, c2.x));
                    ya = __dadd_rn(ya, __dmul_rn(k.xp, c2.y));
                    ya = __dadd_rn(ya, __dmul_rn(k.yp, p2.x));
                    yb = __dadd_rn(0.0, __dmul_rn(k2.ym, m2.y));
                    yb = __dadd_rn(yb, __dmul_rn(k2.xm, c2.x));
                    yb = __dadd_rn(yb, __dmul_rn(k2.di, c2.y));
                    yb = __dadd_rn(yb, __dmul_rn(k2.xp, xr));
                    yb = __dadd_rn(yb, __dmul_rn(k2.yp, p2.y));
                } else {
                    ya = __fma_rn(k.ym, m2.x, 0.0);
                    ya = __fma_rn(k.xm, xl, ya);
                    ya = __fma_rn(k.di, c2.x, ya);
                    ya = __fma_rn(k.xp, c2.y, ya);
                    ya = __fma_rn(k.yp, p2.x, ya);
                    yb = __fma_rn(k2.ym, m2.y, 0.0);
                    yb = __fma_rn(k2.xm, c2.x, yb);
                    yb = __fma_rn(k2.di, c2.y, yb);
                    yb = __fma_rn(k2.xp, xr, yb);
                    yb = __fma_rn(k2.yp, p2.y, yb);
                }
                const double qa = div_rn(__dsub_rn(ya, k.gi), vol, rvol);
                const double qb = div_rn(__dsub_rn(yb, k2.gi), vol, rvol);
                if (qq < nv) {
                    if (vec) {
                        if (pt) __stcs(reinterpret_cast<double2*>(pt), c2);
                        if (pq) __stcs(reinterpret_cast<double2*>(pq), make_double2(qa, qb));
                    } else {
                        if (pt) __stcs(pt, c2.x);
                        if (pq) __stcs(pq, qa);
                        if (inside2 && pt) __stcs(pt + 1, c2.y);
                        if (inside2 && pq) __stcs(pq + 1, qb);
                    }
                    const double ba = fma(vol, qa, k.gi);
                    const double ra = __dsub_rn(ya, ba);
                    num[qq] = fma(ra, ra, num[qq]);
                    den[qq] = fma(ba, ba, den[qq]);
                    if (inside2) {
                        const double bb = fma(vol, qb, k2.gi);
                        const double rb = __dsub_rn(yb, bb);
                        num[qq] = fma(rb, rb, num[qq]);
                        den[qq] = fma(bb, bb, den[qq]);
                    }
                }
                pt += a.ldo;
                pq += a.ldo;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);  // this warp's ring reads are done
        if (a.part) {
            // fixed-order reduction, as combine_action_kernel: warp-level
            // transpose-reduce of the V = 2 SPT per-lane sums, then the 4 warps
            // of each sample half in index order
            double v[V];
#pragma unroll
            for (int q = 0; q < SPT; ++q) {
                v[q] = num[q];
                v[SPT + q] = den[q];
            }
#pragma unroll
            for (int o = 16, len = V; o >= 32 / V; o >>= 1, len >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int e = 0; e < len / 2; ++e) {
                    const double keep = up ? v[len / 2 + e] : v[e];
                    const double send = up ? v[e] : v[len / 2 + e];
                    v[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
#pragma unroll
            for (int o = 32 / V / 2; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
            double* rb = red + (it & 1) * NSW * V;
            if (lane % (32 / V) == 0) rb[sw * V + lane / (32 / V)] = v[0];
            asm volatile("bar.sync 2, %0;" ::"n"(NSW * 32) : "memory");
            if (tt < NS && j0 + tt < a.N) {
                const int hq = tt / SPT, qq = tt % SPT;
                double u = 0.0, w = 0.0;
                for (int w2 = 0; w2 < 4; ++w2) {
                    u += rb[(4 * hq + w2) * V + qq];
                    w += rb[(4 * hq + w2) * V + SPT + qq];
                }
                double* pp = a.part + ((j0 + tt) * (int64_t)a.tiles + tile) * 2;
                *reinterpret_cast<double2*>(pp) = make_double2(u, w);
            }
        }
    }
}

// resid_j = sqrt(num / den) over the tiles (one warp per sample: lane-strided
// sums, then a fixed shuffle tree — deterministic); de == 0 handled as
// pipeline.cpp:570-571.
__global__ void resid_finalize(const double* __restrict__ part, int tiles, int64_t N,
                               double* __restrict__ resid, int64_t rstride) {
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
    if (lane == 0) {
        if (rstride < 0)  // slab partial: (num, den) of this rank, summed across ranks later
            reinterpret_cast<double2*>(resid)[j] = make_double2(nu, de);
        else
            resid[j * rstride] = de == 0.0 ? (nu == 0.0 ? 0.0 : 1.0) : sqrt(nu / de);
    }
}

// resid_j from the (num, den) sums of all ranks (pipeline.cpp:568-571)
__global__ void resid_from_nd(const double2* __restrict__ nd, int64_t N, double* __restrict__ resid) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= N) return;
    const double nu = nd[j].x, de = nd[j].y;
    resid[j] = de == 0.0 ? (nu == 0.0 ? 0.0 : 1.0) : sqrt(nu / de);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    // resolved once; function-local static initialisation is thread-safe
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

template <int S, int NS, int NT, bool PL = false>
bk_status run(bk_ctx* ctx, const bk_operator* op, const double* X, int s, const double* C,
              int64_t ldc, int64_t N, double* T, double* Q, double* resid,
              const bk::ActExtra& ex) {
    using namespace bk;
    using P = Panel<S>;
    using SH = Shape<NS, NT>;
    ActArgs a;
    a.nx = op->nx;
    const bool slab = ex.slab_ny > 0;
    a.ny = slab ? ex.slab_ny : op->ny;
    a.nz = op->nz;
    a.n = (int64_t)a.nx * a.ny * a.nz;
    a.cy0 = slab ? ex.slab_y0 : 0;
    a.cny = op->ny;
    a.ty = slab ? 1 : 0;
    a.N = N;
    a.ldc = ldc;
    a.diag = op->diag;
    a.cx = op->cx;
    a.cy = op->cy;
    a.cz = op->cz;
    a.g = op->g;
    a.volz = op->volz;
    a.C = C;
    a.T = T;
    a.Q = Q;
    a.s = s;
    a.ldo = ex.ldo > 0 ? ex.ldo : a.n;
    a.eps = ex.eps;
    a.fma = ex.fma;
    a.tilesx = (op->nx + TX - 1) / TX;
    a.tiles = a.tilesx * ((a.ny + TY - 1) / TY);
    const int64_t chunks = (N + NS - 1) / NS;
    if (chunks * a.tiles >= (int64_t)1 << 31)
        return fail(ctx, BK_INVALID_CONFIG, "combine_action: too many work items");
    a.chunks = (int)chunks;
    a.items = (int)(chunks * a.tiles);
    a.part = nullptr;
    if (resid) {
        void* p;
        bk_status st = workspace(ctx, kSlotActPart, (size_t)a.tiles * N * 2 * sizeof(double), &p);
        if (st != BK_OK) return st;
        a.part = (double*)p;
    }
    if (reinterpret_cast<uintptr_t>(X) % 16)
        return fail(ctx, BK_INTERNAL, "combine_action: X must be 16-byte aligned");
    // X as a 4D tensor (S, nx, ny, nz): per-axis bounds, so the halo of a
    // boundary tile reads zeros instead of wrapping into the next row
    auto enc = encode_fn();
    if (!enc) return fail(ctx, BK_CUDA_ERROR, "combine_action: cuTensorMapEncodeTiled unavailable");
    CUtensorMap map;
    // (slab: the ghost-row layout nx x (ny + 2) x nz, ghost rows real
    // neighbour data or zero at the physical boundary)
    const int64_t nyt = slab ? a.ny + 2 : a.ny;
    const cuuint64_t dims[4] = {(cuuint64_t)S, (cuuint64_t)op->nx, (cuuint64_t)nyt,
                                (cuuint64_t)op->nz};
    const cuuint64_t strides[3] = {(cuuint64_t)S * 8, (cuuint64_t)S * 8 * op->nx,
                                   (cuuint64_t)S * 8 * op->nx * nyt};
    const cuuint32_t box[4] = {(cuuint32_t)P::PW, (cuuint32_t)HX, (cuuint32_t)HY, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(X), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            P::PW == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS)
        return fail(ctx, BK_CUDA_ERROR, "combine_action: tensor map encode failed (" +
                                            std::to_string((int)cr) + ")");
    const int nring = op->nz < 3 ? op->nz : 3;
    const int hcr = PL ? HY * 36 + 4 : HC;  // the kernel's ring sample stride
    const size_t smem = 1024 + (size_t)SH::NP * P::SLOT +
                        (size_t)(nring * NS * hcr + S * SH::CSP) * sizeof(double) + SH::NP * 8;
    bool done = false;
    if constexpr (PL && P::R == 1 && NS == 16) {
        if (!ctx->knobs.comb_one_role) {
            // measured (C2, 2048 samples): 4 former warps and a two-buffer
            // ring; 8 former warps, 16 stencil warps or three buffers were
            // slower
            constexpr int NQ = 2, NF = 4, NR = 2;
            auto kern = combine_action_pl_ws<S, 16, NQ, NF, NR>;
            const size_t sm2 = 1024 + (size_t)P::SLOT +
                               (size_t)(NR * 16 * (HY * 36 + 2) + 2 * 4 * NQ * 2 * (16 / NQ)) * 8 +
                               (2 * NR + 1) * 8;
            BK_CUDA_TRY(ctx, bk::set_max_smem((const void*)kern, sm2));
            const int grid = a.items < ctx->num_sms ? a.items : ctx->num_sms;
            kern<<<(unsigned)grid, 32 * NF + 128 * NQ, sm2, ctx->stream>>>(map, a);
            done = true;
        }
    }
    if (!done) {
        auto kern = combine_action_kernel<S, NS, NT, PL>;
        BK_CUDA_TRY(ctx, bk::set_max_smem((const void*)kern, smem));
        const int slots = SH::CTAS * ctx->num_sms;
        const int grid = a.items < slots ? a.items : slots;
        kern<<<(unsigned)grid, SH::NT, smem, ctx->stream>>>(map, a);
    }
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    if (ctx->knobs.comb_profile) {
        long long hp[64] = {};
        cudaStreamSynchronize(ctx->stream);
        cudaMemcpyFromSymbol(hp, g_comb_prof, sizeof(hp));
        fprintf(stderr, "[bk_comb_profile S=%d nz=%d] Cs %lld, first planes %lld;", S, op->nz,
                hp[1] - hp[0], hp[2] - hp[1]);
        for (int z = 0; z < op->nz; ++z)
            fprintf(stderr, " z%d stencil %lld form %lld;", z, hp[3 + 2 * z] - hp[2 + 2 * z],
                    hp[4 + 2 * z] - hp[3 + 2 * z]);
        fprintf(stderr, " reduce %lld\n", hp[3 + 2 * op->nz] - hp[2 + 2 * op->nz]);
    }
    if (resid) {
        resid_finalize<<<(unsigned)((N + 7) / 8), 256, 0, ctx->stream>>>(
            a.part, a.tiles, N, resid, ex.nd_out ? -1 : ex.rstride > 0 ? ex.rstride : 1);
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaGetLastError());
    }
    return BK_OK;
}

// Two CTAs of 256 threads per SM, one panel slot each. Single plane: 16
// samples per item (no z-ring, so the T plane fits twice per SM). 3D: 8
// samples per item for the three-plane ring (S = 64: see below). Measured (B200): C2 0.75 ms
// (0.87 with the L2-fragment kernel), C3 5.6 ms (6.6); the one-CTA 512-thread
// NS = 16 shape gave 5.9 ms on C3 (its DMMA chains and stencil do not overlap).
template <int S>
bk_status dispatch(bk_ctx* ctx, const bk_operator* op, const double* X, int s, const double* C,
                   int64_t ldc, int64_t N, double* T, double* Q, double* resid,
                   const bk::ActExtra& ex) {
    if (op->nz == 1) return run<S, 16, 256, true>(ctx, op, X, s, C, ldc, N, T, Q, resid, ex);
    // S = 64: four panels per plane; one 512-thread CTA per SM with two panel
    // slots keeps the next panel in flight (C5: 500 samples 27.9 ms vs 53.9 ms
    // with two one-slot CTAs, whose every panel waited out a full TMA round trip)
    if (S == 64) return run<S, 16, 512>(ctx, op, X, s, C, ldc, N, T, Q, resid, ex);
    return run<S, 8, 256>(ctx, op, X, s, C, ldc, N, T, Q, resid, ex);
}

}  // namespace

namespace bk {

cudaError_t launch_resid_from_nd(cudaStream_t s, const double* nd, int64_t N, double* resid) {
    if (N <= 0) return cudaSuccess;
    resid_from_nd<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const double2*>(nd), N, resid);
    return cudaGetLastError();
}

// X is the kernel-width block n x S (zero-padded past the real width s); C is
// s x N with row stride ldc.
bk_status combine_action_device(bk_ctx* ctx, const bk_operator* op, const double* X, int S,
                                int s, const double* C, int64_t ldc, int64_t N, double* T,
                                double* Q, double* resid, const ActExtra& ex) {
    if (N == 0) return BK_OK;
    if (s < 1 || s > S || ldc < N) return fail(ctx, BK_INTERNAL, "combine_action: bad widths");
    switch (S) {
        case 8: return dispatch<8>(ctx, op, X, s, C, ldc, N, T, Q, resid, ex);
        case 16: return dispatch<16>(ctx, op, X, s, C, ldc, N, T, Q, resid, ex);
        case 32: return dispatch<32>(ctx, op, X, s, C, ldc, N, T, Q, resid, ex);
        case 64: return dispatch<64>(ctx, op, X, s, C, ldc, N, T, Q, resid, ex);
        default: return fail(ctx, BK_INTERNAL, "combine_action: unpadded width");
    }
}

}  // namespace bk
