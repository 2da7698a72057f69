// Device-side input synthesis: the random draws of a chip
// stay on the host (bk::synth_plan: the reference Rng streams, bit-exact);
// the fields — k and the s basis power maps, the per-cell work dominated by
// exp() — are evaluated here, straight into device buffers the pipeline
// consumes. Same arithmetic order as the host generator (bk_synth.cpp); only
// CUDA's exp differs from the host libm (a few ulp), so k for configs 1, 2, 4
// and all coefficients are bitwise the host's and the maps agree to ~1e-15.
#include <cstring>
#include <vector>

#include "bk_common.cuh"
#include "bk_synth.h"

namespace {

struct KArgs {
    int config, nx, ny, nz, tile, tx, cpl;
    double log_sigma;
    const double* kvals;
    const double* normals;
    double* k;
};

__global__ void synth_k_kernel(KArgs a) {
    const int64_t plane = (int64_t)a.nx * a.ny, n = plane * a.nz;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ix = (int)(i % a.nx), iy = (int)((i / a.nx) % a.ny), iz = (int)(i / plane);
        double v;
        if (a.config <= 2)
            v = a.kvals[(iy / a.tile) * a.tx + ix / a.tile];
        else if (a.normals)
            v = __dmul_rn(a.kvals[iz / a.cpl], exp(__dmul_rn(a.log_sigma, a.normals[i])));
        else
            v = a.kvals[iz];
        a.k[i] = v;
    }
}

struct QArgs {
    int nx, ny, nz, s, nblobs, nrects, z0, z1;
    const double* blobs;  // [s][nblobs][4]
    const double* rects;  // [s][nrects][5]
    double* Q;            // n x s
};

// one thread per (plane cell, map): blobs in order, then rectangles, with the
// host's rounding sequence (separate multiply / add)
__global__ void synth_q_kernel(QArgs a) {
    const int64_t plane = (int64_t)a.nx * a.ny;
    const int64_t total = plane * a.s;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(e % a.s);
        const int64_t c = e / a.s;
        const int ix = (int)(c % a.nx), iy = (int)(c / a.nx);
        double acc = 0.0;
        for (int b = 0; b < a.nblobs; ++b) {
            const double* q = a.blobs + ((int64_t)t * a.nblobs + b) * 4;
            const double ddx = __dsub_rn(__dadd_rn((double)ix, 0.5), q[0]);
            const double ddy = __dsub_rn(__dadd_rn((double)iy, 0.5), q[1]);
            const double r2 = __dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy));
            acc = __dadd_rn(acc, __dmul_rn(q[3], exp(__dmul_rn(-r2, q[2]))));
        }
        for (int r = 0; r < a.nrects; ++r) {
            const double* q = a.rects + ((int64_t)t * a.nrects + r) * 5;
            const int x0 = (int)q[0], y0 = (int)q[1], w = (int)q[2], h = (int)q[3];
            if (ix >= x0 && ix < x0 + w && iy >= y0 && iy < y0 + h) acc = __dadd_rn(acc, q[4]);
        }
        for (int iz = 0; iz < a.nz; ++iz)
            a.Q[(iz * plane + c) * a.s + t] = (iz >= a.z0 && iz < a.z1) ? acc : 0.0;
    }
}

}  // namespace

extern "C" {

bk_status bk_synth_chip_device(bk_ctx* ctx, const bk_synth_spec* sp, bk_grid* grid, double* dz_out,
                               int* has_dz, bk_face bc[6], double* k_dev, double* Q_dev,
                               double* C) {
    using namespace bk;
    if (!ctx) return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    SynthPlan p;
    bk_status st = synth_plan(sp, grid, dz_out, has_dz, bc, k_dev != nullptr, p);
    if (st != BK_OK) return st;
    const int64_t plane = (int64_t)p.nx * p.ny, n = plane * p.nz;
    // parameters -> device (one small staging buffer; normals for 3/5 only)
    const size_t nk = p.kvals.size(), nn = p.normals.size(), nb = p.blobs.size(),
                 nr = p.rects.size();
    void* pw;
    if ((st = workspace(ctx, kSlotIn1, (nk + nn + nb + nr + 4) * sizeof(double), &pw)) != BK_OK)
        return st;
    double* d = (double*)pw;
    std::vector<double> host(nk + nn + nb + nr + 4, 0.0);
    std::memcpy(host.data(), p.kvals.data(), nk * sizeof(double));
    if (nn) std::memcpy(host.data() + nk, p.normals.data(), nn * sizeof(double));
    if (nb) std::memcpy(host.data() + nk + nn, p.blobs.data(), nb * sizeof(double));
    if (nr) std::memcpy(host.data() + nk + nn + nb, p.rects.data(), nr * sizeof(double));
    BK_CUDA_TRY(ctx, cudaMemcpyAsync(d, host.data(), host.size() * sizeof(double),
                                     cudaMemcpyHostToDevice, ctx->stream));
    const int grid_blocks = ctx->num_sms * 8;
    if (k_dev) {
        KArgs ka{p.config, p.nx, p.ny, p.nz, p.tile, p.tx, p.cpl, p.log_sigma, d,
                 nn ? d + nk : nullptr, k_dev};
        synth_k_kernel<<<grid_blocks, 256, 0, ctx->stream>>>(ka);
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaGetLastError());
    }
    if (Q_dev) {
        QArgs qa{p.nx, p.ny, p.nz, p.s, p.nblobs, p.nrects, p.power_z0, p.power_z1,
                 d + nk + nn, d + nk + nn + nb, Q_dev};
        synth_q_kernel<<<grid_blocks, 256, 0, ctx->stream>>>(qa);
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaGetLastError());
    }
    if (C) {
        std::vector<double> ch((size_t)p.s * sp->N);
        synth_coef(sp, p.chip_seed, ch.data());
        if (is_device_ptr(C))
            BK_CUDA_TRY(ctx, cudaMemcpyAsync(C, ch.data(), ch.size() * sizeof(double),
                                             cudaMemcpyHostToDevice, ctx->stream));
        else
            std::memcpy(C, ch.data(), ch.size() * sizeof(double));
    }
    // the staging vector must outlive the async copy
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    (void)n;
    return BK_OK;
}

}  // extern "C"
