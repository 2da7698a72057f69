// Stencil assembly and the elementwise/stencil sweeps of discretize.hpp.
//
// assemble_kernel restates discretize.cpp:114-237 for one cell per thread and
// stores the matrix-free SoA stencil. Every expression follows the reference's
// operation order with explicit round-to-nearest intrinsics (no contraction),
// and the one place the reference build contracts (lift += g_face * datum) is an
// explicit fma, so diag/off-diagonals/g are bitwise the reference's values.
#include "bk_common.cuh"

namespace {

__device__ __forceinline__ double harm(double ki, double kj, double area, double delta) {
    // (2.0 * ki * kj / (ki + kj)) * (area / delta)   discretize.cpp:102-105
    const double num = __dmul_rn(__dmul_rn(2.0, ki), kj);
    return __dmul_rn(__ddiv_rn(num, __dadd_rn(ki, kj)), __ddiv_rn(area, delta));
}

// z-face between cells of thicknesses da, db (non-uniform stacks). Equal
// thicknesses take the reference expression, so uniform grids stay bitwise.
__device__ __forceinline__ double zface(double ka, double kb, double da, double db, double area) {
    if (da == db) return harm(ka, kb, area, da);
    const double ra = __ddiv_rn(da, __dmul_rn(2.0, ka));
    const double rb = __ddiv_rn(db, __dmul_rn(2.0, kb));
    return __ddiv_rn(area, __dadd_rn(ra, rb));
}

struct FaceC {
    int kind[6];
    double a[6];
    double b[6];
};

// discretize.cpp:151-165; kind 2 (adiabatic) contributes nothing.
__device__ __forceinline__ void bface(const FaceC& f, int face, double kc, double area,
                                      double delta, double& diag, double& lift) {
    const int kind = f.kind[face];
    if (kind == BK_FACE_DIRICHLET) {
        const double gf = __dmul_rn(__ddiv_rn(__dmul_rn(2.0, kc), delta), area);
        diag = __dadd_rn(diag, gf);
        lift = fma(gf, f.a[face], lift);
    } else if (kind == BK_FACE_ROBIN) {
        const double heff = __ddiv_rn(
            1.0, __dadd_rn(__ddiv_rn(delta, __dmul_rn(2.0, kc)), __ddiv_rn(1.0, f.a[face])));
        const double gf = __dmul_rn(heff, area);
        diag = __dadd_rn(diag, gf);
        lift = fma(gf, f.b[face], lift);
    }
}

__global__ void __launch_bounds__(256) assemble_kernel(
    int nx, int ny, int nz, double dx, double dy, const double* __restrict__ dz,
    const double* __restrict__ k, FaceC bc, double* __restrict__ diag_out,
    double* __restrict__ cx, double* __restrict__ cy, double* __restrict__ cz,
    double* __restrict__ g_out, double* __restrict__ dinv_out) {
    const int64_t plane = (int64_t)nx * ny;
    const int64_t n = plane * nz;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ix = (int)(i % nx);
        const int iy = (int)((i / nx) % ny);
        const int iz = (int)(i / plane);
        const double dzc = dz[iz];
        const double ax = __dmul_rn(dy, dzc), ay = __dmul_rn(dx, dzc), az = __dmul_rn(dx, dy);
        const double kc = k[i];
        double diag = 0.0, lift = 0.0;
        double gzm = 0, gym = 0, gxm = 0, gxp = 0, gyp = 0, gzp = 0;
        // neighbour order z-, y-, x-, x+, y+, z+   (discretize.cpp:175-214)
        if (iz > 0)
            gzm = zface(kc, k[i - plane], dzc, dz[iz - 1], az);
        else
            bface(bc, 4, kc, az, dzc, diag, lift);
        if (iy > 0)
            gym = harm(kc, k[i - nx], ay, dy);
        else
            bface(bc, 2, kc, ay, dy, diag, lift);
        if (ix > 0)
            gxm = harm(kc, k[i - 1], ax, dx);
        else
            bface(bc, 0, kc, ax, dx, diag, lift);
        if (ix < nx - 1)
            gxp = harm(kc, k[i + 1], ax, dx);
        else
            bface(bc, 1, kc, ax, dx, diag, lift);
        if (iy < ny - 1)
            gyp = harm(kc, k[i + nx], ay, dy);
        else
            bface(bc, 3, kc, ay, dy, diag, lift);
        if (iz < nz - 1)
            gzp = zface(kc, k[i + plane], dzc, dz[iz + 1], az);
        else
            bface(bc, 5, kc, az, dzc, diag, lift);
        // diag += g_zm + g_ym + g_xm + g_xp + g_yp + g_zp   (discretize.cpp:216)
        double sum = __dadd_rn(gzm, gym);
        sum = __dadd_rn(sum, gxm);
        sum = __dadd_rn(sum, gxp);
        sum = __dadd_rn(sum, gyp);
        sum = __dadd_rn(sum, gzp);
        diag = __dadd_rn(diag, sum);
        diag_out[i] = diag;
        cx[i] = gxp;
        cy[i] = gyp;
        cz[i] = gzp;
        g_out[i] = lift;
        dinv_out[i] = diag != 0.0 ? __ddiv_rn(1.0, diag) : 1.0;
    }
}

// Y = A X, one thread per (cell, column); CSR-order FMA chain
// (apply_block_fixed, discretize.cpp:57-71): z-, y-, x-, diag, x+, y+, z+.
__global__ void __launch_bounds__(256) apply_block_kernel(
    int nx, int ny, int nz, const double* __restrict__ diag, const double* __restrict__ cx,
    const double* __restrict__ cy, const double* __restrict__ cz,
    const double* __restrict__ x, int s, double* __restrict__ y) {
    const int64_t plane = (int64_t)nx * ny;
    const int64_t n = plane * nz;
    const int64_t total = n * s;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / s;
        const int ix = (int)(i % nx);
        const int iy = (int)((i / nx) % ny);
        const int iz = (int)(i / plane);
        double acc = 0.0;
        if (s != 4) {
            if (iz > 0) acc = fma(-cz[i - plane], x[e - plane * s], acc);
            if (iy > 0) acc = fma(-cy[i - nx], x[e - (int64_t)nx * s], acc);
            if (ix > 0) acc = fma(-cx[i - 1], x[e - s], acc);
            acc = fma(diag[i], x[e], acc);
            if (ix < nx - 1) acc = fma(-cx[i], x[e + s], acc);
            if (iy < ny - 1) acc = fma(-cy[i], x[e + (int64_t)nx * s], acc);
            if (iz < nz - 1) acc = fma(-cz[i], x[e + plane * s], acc);
        } else {
            // the reference build compiles apply_block_fixed<4> without
            // contraction: separate multiply and add per term
            if (iz > 0) acc = __dadd_rn(acc, __dmul_rn(-cz[i - plane], x[e - plane * s]));
            if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(-cy[i - nx], x[e - (int64_t)nx * s]));
            if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(-cx[i - 1], x[e - s]));
            acc = __dadd_rn(acc, __dmul_rn(diag[i], x[e]));
            if (ix < nx - 1) acc = __dadd_rn(acc, __dmul_rn(-cx[i], x[e + s]));
            if (iy < ny - 1) acc = __dadd_rn(acc, __dmul_rn(-cy[i], x[e + (int64_t)nx * s]));
            if (iz < nz - 1) acc = __dadd_rn(acc, __dmul_rn(-cz[i], x[e + plane * s]));
        }
        y[e] = acc;
    }
}

// b = V q + g   (rhs_from_power, discretize.cpp:246-256; contracted to fma in
// the reference build)
__global__ void rhs_kernel(int64_t plane, int64_t n, int s, const double* __restrict__ volz,
                           const double* __restrict__ g, const double* __restrict__ q,
                           double* __restrict__ b) {
    const int64_t total = n * s;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / s;
        b[e] = fma(volz[i / plane], q[e], g[i]);
    }
}

// q = (b - g) / V   (power_from_rhs, discretize.cpp:258-267)
__global__ void power_kernel(int64_t plane, int64_t n, int s, const double* __restrict__ volz,
                             const double* __restrict__ g, const double* __restrict__ b,
                             double* __restrict__ q) {
    const int64_t total = n * s;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / s;
        q[e] = __ddiv_rn(__dsub_rn(b[e], g[i]), volz[i / plane]);
    }
}

__global__ void pad_cols_kernel(const double* __restrict__ src, int sw, double* __restrict__ dst,
                                int dw, int64_t n) {
    const int64_t total = n * dw;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / dw;
        const int q = (int)(e % dw);
        dst[e] = q < sw ? src[i * sw + q] : 0.0;
    }
}

__global__ void rhs_padded_kernel(int64_t plane, int64_t n, int s, int S,
                                  const double* __restrict__ volz, const double* __restrict__ g,
                                  const double* __restrict__ q, double* __restrict__ b) {
    const int64_t total = n * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / S;
        const int c = (int)(e % S);
        b[e] = c < s ? fma(volz[i / plane], q[i * s + c], g[i]) : 0.0;
    }
}

__global__ void check_positive_kernel(const double* __restrict__ k, int64_t n, int* flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!(k[i] > 0.0)) atomicOr(flag, 1);
}

int grid_for(bk_ctx* ctx, int64_t work) {
    int64_t blocks = (work + 255) / 256;
    const int64_t cap = (int64_t)ctx->num_sms * 16;
    return (int)(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

}  // namespace

namespace bk {

cudaError_t launch_assemble(bk_ctx* ctx, const bk_operator* op, const double* k,
                            const bk_face* bc, double dx, double dy, const double* dz_dev) {
    FaceC f;
    for (int i = 0; i < 6; ++i) {
        f.kind[i] = bc[i].kind;
        f.a[i] = bc[i].a;
        f.b[i] = bc[i].b;
    }
    assemble_kernel<<<grid_for(ctx, op->n), 256, 0, ctx->stream>>>(
        op->nx, op->ny, op->nz, dx, dy, dz_dev, k, f, op->diag, op->cx, op->cy, op->cz, op->g,
        op->dinv);
    ++ctx->launches;
    return cudaGetLastError();
}

cudaError_t launch_apply_block(bk_ctx* ctx, const bk_operator* op, const double* x, int s,
                               double* y) {
    apply_block_kernel<<<grid_for(ctx, op->n * s), 256, 0, ctx->stream>>>(
        op->nx, op->ny, op->nz, op->diag, op->cx, op->cy, op->cz, x, s, y);
    ++ctx->launches;
    return cudaGetLastError();
}

cudaError_t launch_rhs_from_power(bk_ctx* ctx, const bk_operator* op, const double* q, int s,
                                  double* b) {
    rhs_kernel<<<grid_for(ctx, op->n * s), 256, 0, ctx->stream>>>(
        (int64_t)op->nx * op->ny, op->n, s, op->volz, op->g, q, b);
    ++ctx->launches;
    return cudaGetLastError();
}

cudaError_t launch_pad_cols(bk_ctx* ctx, const double* src, int sw, double* dst, int dw,
                            int64_t n) {
    pad_cols_kernel<<<grid_for(ctx, n * dw), 256, 0, ctx->stream>>>(src, sw, dst, dw, n);
    ++ctx->launches;
    return cudaGetLastError();
}

cudaError_t launch_rhs_padded(bk_ctx* ctx, const bk_operator* op, const double* q, int s,
                              double* b, int S) {
    rhs_padded_kernel<<<grid_for(ctx, op->n * S), 256, 0, ctx->stream>>>(
        (int64_t)op->nx * op->ny, op->n, s, S, op->volz, op->g, q, b);
    ++ctx->launches;
    return cudaGetLastError();
}

__global__ void copy_words_kernel(unsigned* __restrict__ dst, const unsigned* __restrict__ src,
                                  size_t words) {
    for (size_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    __threadfence_system();
}

cudaError_t launch_copy_words(cudaStream_t s, unsigned* dst, const unsigned* src, size_t words) {
    copy_words_kernel<<<1, 256, 0, s>>>(dst, src, words);
    return cudaGetLastError();
}

cudaError_t launch_check_positive(bk_ctx* ctx, const double* k, int64_t n, int* flag) {
    check_positive_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(k, n, flag);
    ++ctx->launches;
    return cudaGetLastError();
}

cudaError_t launch_power_from_rhs(bk_ctx* ctx, const bk_operator* op, const double* b, int s,
                                  double* q) {
    power_kernel<<<grid_for(ctx, op->n * s), 256, 0, ctx->stream>>>(
        (int64_t)op->nx * op->ny, op->n, s, op->volz, op->g, b, q);
    ++ctx->launches;
    return cudaGetLastError();
}

}  // namespace bk
