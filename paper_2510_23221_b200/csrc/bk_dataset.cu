// Dataset sink and validation:
//
//   * bk_dataset_open / append / commit / abort — write_dataset
//     (dataset_io.hpp:27, dataset_io.cpp:160-225) as a streaming writer: the
//     k.bin / q.bin / u.bin payloads (sample-major little-endian float64) are
//     appended chip by chip, device outputs drained through two pinned
//     buffers so the PCIe copy of chunk c+1 overlaps the file write of chunk
//     c; the directory is staged next to its destination and renamed into
//     place on commit, as the reference does.
//   * bk_residuals — relative_residual (discretize.cpp:275-286) for N samples
//     at once: ||V q + g - A u|| / ||V q + g|| with one stencil kernel that
//     keeps the cell's coefficients in registers across a group of samples.
//   * bk_validate_samples — the sample loop of validate_dataset
//     (dataset_io.cpp:328-361): k digest check against the manifest, one
//     operator per distinct k (assembled on the GPU), per-sample residual.
//   * bk_field_digest — field_digest (discretize.cpp:302-319), FNV-1a over the
//     grid shape and the raw value bytes (byte-serial: host).
#include <fcntl.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <limits>
#include <string>
#include <vector>

#include <math_constants.h>

#include "bk_common.cuh"

namespace fs = std::filesystem;

namespace {

// ---------------------------------------------------------------- residuals
constexpr int kResThreads = 256;
constexpr int kResCellsPerThread = 4;
constexpr int kResTile = kResThreads * kResCellsPerThread;  // cells per CTA
constexpr int kResSamples = 4;                              // samples per CTA (4 beat 1, 2, 8, 16 on B200)

struct ResArgs {
    int nx, ny, nz;
    int64_t n, N;
    int tiles;
    const double *diag, *cx, *cy, *cz, *g, *volz;
    const double* U;  // N x n, sample-major
    const double* Q;
    double* part;     // [N][tiles][2] = (sum r^2, sum b^2)
};

// CTA (tile, sample group): each thread owns kResCellsPerThread cells, loads
// their stencil row once and applies it to kResSamples samples. Per cell the
// arithmetic is the reference build's: b = fma(V, q, g) (rhs_from_power,
// contracted) and A u in CSR order z-, y-, x-, diag, x+, y+, z+ as separate
// multiply and add (CsrMatrix::apply, discretize.cpp:39-51, is not contracted
// by the reference build), so r_i = b_i - (A u)_i is bitwise the reference's.
// This matters: validated samples have residuals ~1e-17 only because A u is
// recomputed exactly as the generator computed it — another summation order
// leaves ~1e-13 of cancellation noise. Only the two norms are reordered (fixed
// tree, deterministic).
__global__ void __launch_bounds__(kResThreads) residual_kernel(ResArgs a) {
    const int tile = blockIdx.x;
    const int64_t j0 = (int64_t)blockIdx.y * kResSamples;
    const int ns = (int)(a.N - j0 < kResSamples ? a.N - j0 : kResSamples);
    const int64_t plane = (int64_t)a.nx * a.ny;
    double nu[kResSamples], de[kResSamples];
#pragma unroll
    for (int j = 0; j < kResSamples; ++j) nu[j] = de[j] = 0.0;
#pragma unroll
    for (int c = 0; c < kResCellsPerThread; ++c) {
        const int64_t i = (int64_t)tile * kResTile + c * kResThreads + threadIdx.x;
        if (i >= a.n) break;
        const int ix = (int)(i % a.nx);
        const int iy = (int)((i / a.nx) % a.ny);
        const int iz = (int)(i / plane);
        const double czm = iz > 0 ? -a.cz[i - plane] : 0.0;
        const double cym = iy > 0 ? -a.cy[i - a.nx] : 0.0;
        const double cxm = ix > 0 ? -a.cx[i - 1] : 0.0;
        const double dg = a.diag[i];
        const double cxp = ix < a.nx - 1 ? -a.cx[i] : 0.0;
        const double cyp = iy < a.ny - 1 ? -a.cy[i] : 0.0;
        const double czp = iz < a.nz - 1 ? -a.cz[i] : 0.0;
        const double gi = a.g[i], vi = a.volz[iz];
#pragma unroll
        for (int j = 0; j < kResSamples; ++j) {
            if (j < ns) {
                const double* u = a.U + (j0 + j) * a.n + i;
                double acc = 0.0;
                if (iz > 0) acc = __dadd_rn(acc, __dmul_rn(czm, u[-plane]));
                if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(cym, u[-a.nx]));
                if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(cxm, u[-1]));
                acc = __dadd_rn(acc, __dmul_rn(dg, u[0]));
                if (ix < a.nx - 1) acc = __dadd_rn(acc, __dmul_rn(cxp, u[1]));
                if (iy < a.ny - 1) acc = __dadd_rn(acc, __dmul_rn(cyp, u[a.nx]));
                if (iz < a.nz - 1) acc = __dadd_rn(acc, __dmul_rn(czp, u[plane]));
                const double b = fma(vi, a.Q[(j0 + j) * a.n + i], gi);
                const double r = b - acc;
                nu[j] = fma(r, r, nu[j]);
                de[j] = fma(b, b, de[j]);
            }
        }
    }
    // CTA reduction: warp trees, then warp 0 folds the 8 warps' values
    __shared__ double red[kResThreads / 32][2 * kResSamples];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < kResSamples; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            nu[j] += __shfl_xor_sync(0xffffffffu, nu[j], o);
            de[j] += __shfl_xor_sync(0xffffffffu, de[j], o);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < kResSamples; ++j) {
            red[warp][2 * j] = nu[j];
            red[warp][2 * j + 1] = de[j];
        }
    }
    __syncthreads();
    if (threadIdx.x < 2 * ns) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < kResThreads / 32; ++w) v += red[w][threadIdx.x];
        const int j = threadIdx.x >> 1;
        a.part[((j0 + j) * a.tiles + tile) * 2 + (threadIdx.x & 1)] = v;
    }
}

// relative_residual's quotient: nr / nb with nb == 0 -> 0 or +inf
// (discretize.cpp:281-285). One warp per sample.
__global__ void residual_finalize(const double* __restrict__ part, int tiles, int64_t N,
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
    if (lane == 0) {
        const double nb = sqrt(de), nr = sqrt(nu);
        resid[j] = nb == 0.0 ? (nr == 0.0 ? 0.0 : CUDART_INF) : nr / nb;
    }
}

// two pinned staging buffers of `bytes` each (grow-only, owned by ctx)
bk_status ensure_pinned(bk_ctx* ctx, size_t bytes) {
    if (ctx->pin_bytes >= bytes) return BK_OK;
    for (auto& p : ctx->pin) {
        if (p) {
            BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->copy_stream));
            cudaFreeHost(p);
            p = nullptr;
        }
    }
    ctx->pin_bytes = 0;
    for (auto& p : ctx->pin) BK_CUDA_TRY(ctx, cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
    ctx->pin_bytes = bytes;
    return BK_OK;
}

constexpr size_t kStageBytes = size_t(128) << 20;  // per pinned buffer

}  // namespace

namespace bk {

// the copy stream and every event that orders work on it (created together:
// the chip drain and the dataset sink both rely on them)
bk_status ensure_copy_stream(bk_ctx* ctx) {
    if (!ctx->copy_stream)
        BK_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->stage_ev)
        if (!e) BK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : ctx->drain_ev)
        if (!e) BK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return BK_OK;
}


// resid (device, N) for device U, Q (N x n each)
bk_status residuals_device(bk_ctx* ctx, const bk_operator* op, const double* U, const double* Q,
                           int64_t N, double* resid) {
    if (N <= 0) return BK_OK;
    const int tiles = (int)((op->n + kResTile - 1) / kResTile);
    void* part;
    bk_status st = workspace(ctx, kSlotActPart, (size_t)N * tiles * 2 * sizeof(double), &part);
    if (st != BK_OK) return st;
    ResArgs a{op->nx, op->ny, op->nz, op->n, N, tiles, op->diag, op->cx, op->cy, op->cz,
              op->g,  op->volz, U, Q, (double*)part};
    const int64_t groups = (N + kResSamples - 1) / kResSamples;
    for (int64_t g0 = 0; g0 < groups; g0 += 65535) {  // grid.y limit
        const int64_t gc = std::min<int64_t>(65535, groups - g0);
        ResArgs b = a;
        b.U = U + g0 * kResSamples * op->n;
        b.Q = Q + g0 * kResSamples * op->n;
        b.N = std::min<int64_t>(N - g0 * kResSamples, gc * kResSamples);
        b.part = (double*)part + g0 * kResSamples * tiles * 2;
        residual_kernel<<<dim3(tiles, (unsigned)gc), kResThreads, 0, ctx->stream>>>(b);
        ++ctx->launches;
        BK_CUDA_TRY(ctx, cudaGetLastError());
    }
    residual_finalize<<<(unsigned)((N + 7) / 8), 256, 0, ctx->stream>>>((double*)part, tiles, N,
                                                                        resid);
    ++ctx->launches;
    BK_CUDA_TRY(ctx, cudaGetLastError());
    return BK_OK;
}

// Residuals of N samples whose U / Q may live on the host (pageable, e.g. a
// memory-mapped dataset file) or the device; resid_host receives N values.
// Host inputs stream through two pinned + two device buffers: the CPU copy of
// chunk c+1 and its H2D overlap the kernels of chunk c.
bk_status residuals_any(bk_ctx* ctx, const bk_operator* op, const double* U, const double* Q,
                        int64_t N, double* resid_host) {
    if (N <= 0) return BK_OK;
    const int64_t n = op->n;
    void* rd;
    bk_status st = workspace(ctx, kSlotValRes, (size_t)N * sizeof(double), &rd);
    if (st != BK_OK) return st;
    const bool du = is_device_ptr(U), dq = is_device_ptr(Q);
    if (du && dq) {
        if ((st = residuals_device(ctx, op, U, Q, N, (double*)rd)) != BK_OK) return st;
    } else {
        if ((st = ensure_copy_stream(ctx)) != BK_OK) return st;
        const int64_t per = std::max<int64_t>(1, (int64_t)(kStageBytes / (2 * n * sizeof(double))));
        const int64_t cs = std::min<int64_t>(per, N);
        const size_t bytes = (size_t)cs * n * 2 * sizeof(double);
        if ((st = ensure_pinned(ctx, bytes)) != BK_OK) return st;
        void* dbuf[2];
        if ((st = workspace(ctx, kSlotIn0, bytes, &dbuf[0])) != BK_OK) return st;
        if ((st = workspace(ctx, kSlotIn1, bytes, &dbuf[1])) != BK_OK) return st;
        cudaEvent_t* h2d = ctx->stage_ev;       // [0], [1]: H2D of buffer p done
        cudaEvent_t* kern = ctx->stage_ev + 2;  // [2], [3]: kernels on buffer p done
        const int64_t chunks = (N + cs - 1) / cs;
        for (int64_t c = 0; c < chunks; ++c) {
            const int p = (int)(c & 1);
            const int64_t j0 = c * cs, m = std::min<int64_t>(cs, N - j0);
            double* hb = (double*)ctx->pin[p];
            double* db = (double*)dbuf[p];
            if (c >= 2) BK_CUDA_TRY(ctx, cudaEventSynchronize(h2d[p]));
            const double* su = U + j0 * n;
            const double* sq = Q + j0 * n;
            const size_t fb = (size_t)m * n * sizeof(double);
            if (c >= 2) BK_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, kern[p], 0));
            if (du) {
                BK_CUDA_TRY(ctx, cudaMemcpyAsync(db, su, fb, cudaMemcpyDeviceToDevice, ctx->copy_stream));
            } else {
                std::memcpy(hb, su, fb);
                BK_CUDA_TRY(ctx, cudaMemcpyAsync(db, hb, fb, cudaMemcpyHostToDevice, ctx->copy_stream));
            }
            if (dq) {
                BK_CUDA_TRY(ctx, cudaMemcpyAsync(db + m * n, sq, fb, cudaMemcpyDeviceToDevice,
                                                 ctx->copy_stream));
            } else {
                std::memcpy(hb + m * n, sq, fb);
                BK_CUDA_TRY(ctx, cudaMemcpyAsync(db + m * n, hb + m * n, fb, cudaMemcpyHostToDevice,
                                                 ctx->copy_stream));
            }
            BK_CUDA_TRY(ctx, cudaEventRecord(h2d[p], ctx->copy_stream));
            BK_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, h2d[p], 0));
            if ((st = residuals_device(ctx, op, db, db + m * n, m, (double*)rd + j0)) != BK_OK)
                return st;
            BK_CUDA_TRY(ctx, cudaEventRecord(kern[p], ctx->stream));
        }
    }
    BK_CUDA_TRY(ctx, cudaMemcpyAsync(resid_host, rd, (size_t)N * sizeof(double),
                                     is_device_ptr(resid_host) ? cudaMemcpyDeviceToDevice
                                                               : cudaMemcpyDeviceToHost,
                                     ctx->stream));
    BK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
}

}  // namespace bk

// ---------------------------------------------------------------- writer
struct bk_dataset_writer {
    std::string dir, staging, err;
    int fd[3] = {-1, -1, -1};
    int64_t n_cells = 0;
    int64_t n_data = 0;
    bool overwrite = false;
    std::vector<double> kbuf;
    double write_s = 0.0;  // time inside write(2)
};

namespace {

constexpr const char* kFieldFiles[3] = {"k.bin", "q.bin", "u.bin"};

bk_status wfail(bk_dataset_writer* w, bk_status st, const std::string& msg) {
    if (w) w->err = msg;
    return st;
}

bk_status write_all(bk_dataset_writer* w, int f, const void* data, size_t bytes) {
    const auto t0 = std::chrono::steady_clock::now();
    const char* p = (const char*)data;
    while (bytes) {
        const ssize_t k = ::write(w->fd[f], p, std::min<size_t>(bytes, size_t(1) << 30));
        if (k < 0) {
            if (errno == EINTR) continue;
            return wfail(w, BK_IO_ERROR, std::string("write_dataset: short write to ") +
                                             kFieldFiles[f] + ": " + std::strerror(errno));
        }
        p += k;
        bytes -= (size_t)k;
    }
    w->write_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return BK_OK;
}

void close_files(bk_dataset_writer* w) {
    for (int& fd : w->fd) {
        if (fd >= 0) ::close(fd);
        fd = -1;
    }
}

// Device field (count doubles) -> file f, through ctx's two pinned buffers on
// the copy stream: D2H of chunk c+1 runs while chunk c is written.
bk_status drain_to_file(bk_dataset_writer* w, bk_ctx* ctx, int f, const double* src,
                        size_t count) {
    using namespace bk;
    bk_status st;
    if ((st = ensure_copy_stream(ctx)) != BK_OK) return st;
    if ((st = ensure_pinned(ctx, kStageBytes)) != BK_OK) return st;
    const size_t chunk = kStageBytes / sizeof(double);
    const size_t chunks = (count + chunk - 1) / chunk;
    cudaEvent_t* ev = ctx->stage_ev;
    // data is produced on ctx->stream
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[2], ctx->stream));
    BK_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ev[2], 0));
    auto issue = [&](size_t c) -> bk_status {
        const size_t off = c * chunk, len = std::min(chunk, count - off);
        BK_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->pin[c & 1], src + off, len * sizeof(double),
                                         cudaMemcpyDeviceToHost, ctx->copy_stream));
        BK_CUDA_TRY(ctx, cudaEventRecord(ev[c & 1], ctx->copy_stream));
        return BK_OK;
    };
    if (chunks && (st = issue(0)) != BK_OK) return st;
    for (size_t c = 0; c < chunks; ++c) {
        if (c + 1 < chunks && (st = issue(c + 1)) != BK_OK) return st;
        BK_CUDA_TRY(ctx, cudaEventSynchronize(ev[c & 1]));
        const size_t len = std::min(chunk, count - c * chunk);
        if ((st = write_all(w, f, ctx->pin[c & 1], len * sizeof(double))) != BK_OK) return st;
    }
    return BK_OK;
}

}  // namespace

extern "C" {

uint64_t bk_field_digest(int nx, int ny, int nz, const double* values) {
    uint64_t h = 0xcbf29ce484222325ULL;
    auto mix = [&h](uint64_t word) {
        for (int byte = 0; byte < 8; ++byte) {
            h ^= (word >> (8 * byte)) & 0xff;
            h *= 0x100000001b3ULL;
        }
    };
    mix((uint64_t)nx);
    mix((uint64_t)ny);
    mix((uint64_t)nz);
    const int64_t n = (int64_t)nx * ny * nz;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t bits;
        std::memcpy(&bits, values + i, sizeof bits);
        mix(bits);
    }
    return h;
}

bk_status bk_dataset_open(const char* dir, int overwrite, int64_t n_cells,
                          bk_dataset_writer** out) {
    if (!dir || !out || n_cells < 1) return BK_INVALID_CONFIG;
    *out = nullptr;
    auto* w = new (std::nothrow) bk_dataset_writer;
    if (!w) return BK_OOM;
    *out = w;  // returned even on failure so bk_dataset_error can be read
    w->dir = dir;
    w->overwrite = overwrite != 0;
    w->n_cells = n_cells;
    const fs::path d(dir);
    std::error_code ec;
    if (fs::exists(d / "manifest.json", ec) && !w->overwrite)
        return wfail(w, BK_EXISTS, "write_dataset: '" + w->dir +
                                       "' already holds a dataset (use overwrite)");
    const fs::path parent = d.has_parent_path() ? d.parent_path() : fs::path(".");
    fs::create_directories(parent, ec);
    const fs::path staging =
        parent / (d.filename().string() + ".tmp-" + std::to_string(::getpid()));
    fs::remove_all(staging, ec);
    if (!fs::create_directories(staging, ec))
        return wfail(w, BK_IO_ERROR, "write_dataset: cannot create staging dir " + staging.string());
    w->staging = staging.string();
    for (int f = 0; f < 3; ++f) {
        w->fd[f] = ::open((staging / kFieldFiles[f]).c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (w->fd[f] < 0) {
            close_files(w);
            fs::remove_all(staging, ec);
            return wfail(w, BK_IO_ERROR, std::string("write_dataset: cannot open ") + kFieldFiles[f]);
        }
    }
    return BK_OK;
}

const char* bk_dataset_error(const bk_dataset_writer* w) { return w ? w->err.c_str() : "null writer"; }

int64_t bk_dataset_count(const bk_dataset_writer* w) { return w ? w->n_data : 0; }

double bk_dataset_write_seconds(const bk_dataset_writer* w) { return w ? w->write_s : 0.0; }

bk_status bk_dataset_append(bk_dataset_writer* w, bk_ctx* ctx, const double* k,
                            int64_t n_samples, const double* Q, const double* U) {
    using namespace bk;
    if (!w || w->fd[0] < 0) return BK_INVALID_CONFIG;
    if (n_samples < 0 || !k || !Q || !U) return wfail(w, BK_INVALID_CONFIG, "append: bad arguments");
    if (n_samples == 0) return BK_OK;
    const int64_t n = w->n_cells;
    const bool dk = is_device_ptr(k), dqp = is_device_ptr(Q), du = is_device_ptr(U);
    if ((dk || dqp || du) && !ctx)
        return wfail(w, BK_INVALID_CONFIG, "append: device outputs need a context");
    if (ctx) cudaSetDevice(ctx->device);
    bk_status st;
    // k: one copy per sample (Sample::k is the group's field, pipeline.cpp:572-577)
    const double* kh = k;
    if (dk) {
        w->kbuf.resize(n);
        cudaError_t e = cudaMemcpyAsync(w->kbuf.data(), k, n * sizeof(double),
                                        cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess)
            return wfail(w, BK_CUDA_ERROR, std::string("append: k readback: ") + cudaGetErrorString(e));
        kh = w->kbuf.data();
    }
    for (int64_t j = 0; j < n_samples; ++j)
        if ((st = write_all(w, 0, kh, n * sizeof(double))) != BK_OK) return st;
    const double* src[2] = {Q, U};
    const bool dev[2] = {dqp, du};
    for (int f = 1; f < 3; ++f) {
        const size_t count = (size_t)n_samples * n;
        if (dev[f - 1]) {
            st = drain_to_file(w, ctx, f, src[f - 1], count);
            if (st != BK_OK) return wfail(w, st, ctx->err.empty() ? w->err : ctx->err);
        } else if ((st = write_all(w, f, src[f - 1], count * sizeof(double))) != BK_OK) {
            return st;
        }
    }
    w->n_data += n_samples;
    return BK_OK;
}

bk_status bk_dataset_commit(bk_dataset_writer* w, const char* manifest_json) {
    if (!w || w->staging.empty() || !manifest_json) return BK_INVALID_CONFIG;
    std::error_code ec;
    const fs::path staging(w->staging), d(w->dir);
    close_files(w);
    {
        const int fd = ::open((staging / "manifest.json").c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (fd < 0) return wfail(w, BK_IO_ERROR, "write_dataset: cannot open manifest.json");
        const size_t len = std::strlen(manifest_json);
        const ssize_t k = ::write(fd, manifest_json, len);
        ::close(fd);
        if (k != (ssize_t)len) return wfail(w, BK_IO_ERROR, "write_dataset: short write to manifest.json");
    }
    // re-check, then swap (dataset_io.cpp:208-220)
    if (fs::exists(d, ec)) {
        if (fs::exists(d / "manifest.json", ec) && !w->overwrite) {
            fs::remove_all(staging, ec);
            w->staging.clear();
            return wfail(w, BK_EXISTS, "write_dataset: '" + w->dir +
                                           "' already holds a dataset (use overwrite)");
        }
        fs::remove_all(d, ec);
    }
    fs::rename(staging, d, ec);
    if (ec) return wfail(w, BK_IO_ERROR, "write_dataset: rename: " + ec.message());
    w->staging.clear();
    return BK_OK;
}

void bk_dataset_close(bk_dataset_writer* w) {
    if (!w) return;
    close_files(w);
    if (!w->staging.empty()) {
        std::error_code ec;
        fs::remove_all(w->staging, ec);  // not committed: discard the staged files
    }
    delete w;
}

bk_status bk_residuals(bk_ctx* ctx, const bk_operator* op, const double* U, const double* Q,
                       int64_t N, double* resid) {
    if (!ctx || !op || N < 0 || (N && (!U || !Q || !resid))) return BK_INVALID_CONFIG;
    cudaSetDevice(ctx->device);
    return bk::residuals_any(ctx, op, U, Q, N, resid);
}

bk_status bk_validate_samples(bk_ctx* ctx, const bk_grid* grid, const bk_face bc[6],
                              const double* K, const double* U, const double* Q, int64_t n_data,
                              const uint64_t* ids, int n_decl, const uint64_t* decl_ids,
                              const uint64_t* decl_digests, double tol, double* residuals,
                              bk_validation* report) {
    using namespace bk;
    if (!ctx || !grid || !bc || n_data < 0 || !report) return BK_INVALID_CONFIG;
    if (n_data && (!K || !U || !Q || !ids || !residuals)) return BK_INVALID_CONFIG;
    if (n_decl && (!decl_ids || !decl_digests)) return BK_INVALID_CONFIG;
    if (is_device_ptr(K)) return fail(ctx, BK_INVALID_CONFIG, "validate: k must be host memory");
    cudaSetDevice(ctx->device);
    const int64_t n = (int64_t)grid->nx * grid->ny * grid->nz;
    report->pass_count = report->fail_count = 0;
    report->max_residual = 0.0;
    // per-sample digest (a k equal to its predecessor's shares its digest)
    std::vector<uint64_t> dig(n_data);
    std::vector<char> bad(n_data, 0);
    for (int64_t j = 0; j < n_data; ++j) {
        const double* kj = K + j * n;
        if (j > 0 && std::memcmp(kj, kj - n, n * sizeof(double)) == 0)
            dig[j] = dig[j - 1];
        else
            dig[j] = bk_field_digest(grid->nx, grid->ny, grid->nz, kj);
        for (int d = 0; d < n_decl; ++d)  // std::map semantics: the last entry for an id wins
            if (decl_ids[d] == ids[j]) bad[j] = decl_digests[d] != dig[j];
    }
    // one operator per run of samples sharing a digest (the reference caches
    // every distinct operator; the residuals do not depend on which copy)
    bk_operator* op = nullptr;
    uint64_t op_digest = 0;
    bk_status st = BK_OK;
    int64_t j = 0;
    while (j < n_data && st == BK_OK) {
        if (bad[j]) {
            residuals[j] = std::numeric_limits<double>::infinity();
            ++j;
            continue;
        }
        int64_t e = j + 1;
        while (e < n_data && !bad[e] && dig[e] == dig[j]) ++e;
        if (!op || op_digest != dig[j]) {
            if (op) bk_operator_free(op);
            op = nullptr;
            if ((st = bk_assemble(ctx, grid, K + j * n, bc, &op)) != BK_OK) break;
            op_digest = dig[j];
        }
        st = residuals_any(ctx, op, U + j * n, Q + j * n, e - j, residuals + j);
        j = e;
    }
    if (op) bk_operator_free(op);
    if (st != BK_OK) return st;
    for (int64_t i = 0; i < n_data; ++i) {
        const double r = residuals[i];
        report->max_residual = std::max(report->max_residual, r);
        if (r <= tol)
            ++report->pass_count;
        else
            ++report->fail_count;
    }
    return BK_OK;
}

}  // extern "C"
