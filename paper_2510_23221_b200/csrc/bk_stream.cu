// Streaming per-chip pipeline with a host sample sink (bk_generate_stream).
//
// The per-chip loop of generate_blockoa (pipeline.cpp:365-597) for jobs whose
// (T, q) do not fit in memory at once — BASELINE config 5 emits 335 GB per
// chip, more than the GPU's HBM and more than a host wants pinned. Chips are
// solved one after another on the context's stream. Each solved chip is handed
// to an output worker (one host thread with a child context: its own compute
// stream and copy stream) that walks the chip's samples in chunks:
//
//   combine + operator action of chunk k   -> device ring slot k % 2
//   D2H of that slot on the copy stream    -> pinned host ring slot k % 2
//   the caller's sink(chunk k - 1)         (pinned buffers valid during the call)
//
// so the PCIe drain of chip c (16 n bytes per sample) overlaps the basis solve
// of chip c + 1 on the main stream. A device slot is refilled only after its
// previous D2H completed (stream wait on the copy event); a pinned slot only
// after the sink returned for its previous chunk (the worker calls the sink
// for chunk k - 1 before it enqueues the D2H of chunk k + 1). Chip c + 2 reuses
// chip c's operator / X / C buffers only after the worker finished chip c.
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>

#include "bk_common.cuh"

namespace bk {
bk_status assemble_into(bk_ctx* ctx, const bk_grid* grid, const double* k, const bk_face bc[6],
                        bk_operator* op);
void free_op_buffers(bk_operator* op);
bk_status validate_grid(bk_ctx* ctx, const bk_grid* g);
bk_status validate_cfg(bk_ctx* ctx, const bk_solver_cfg* c);
void fill_report(const CgReport& r, int s, double wall, bk_solve_report* out);
}  // namespace bk

namespace {

using namespace bk;

int width_of(int s) { return s <= 8 ? 8 : s <= 16 ? 16 : s <= 32 ? 32 : 64; }

// Child context of the output worker: same device, own streams and workspace.
bk_status make_out_ctx(bk_ctx* ctx) {
    if (ctx->out_ctx) return BK_OK;
    bk_ctx* c = new (std::nothrow) bk_ctx;
    if (!c) return fail(ctx, BK_OOM, "generate_stream: output context");
    c->knobs = ctx->knobs;
    c->device = ctx->device;
    c->num_sms = ctx->num_sms;
    if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return fail(ctx, BK_CUDA_ERROR, "generate_stream: output stream");
    }
    c->stream = c->own_stream;
    for (auto& e : c->ev) cudaEventCreate(&e);
    ctx->out_ctx = c;
    return BK_OK;
}

struct Job {
    int chip;
    const bk_operator* op;
    const double* X;  // n x S, device
    const double* C;  // s x N, device
    int S, s;
    int64_t N;
    cudaEvent_t ready;  // basis solve of the chip done (main stream)
};

struct Pipe {
    bk_ctx* out;
    int64_t n, chunk;
    bk_sample_sink sink;
    void* user;
    double* dT[2];
    double* dQ[2];
    double* dR[2];
    double* hT[2];
    double* hQ[2];
    double* hR[2];
    cudaEvent_t comp[2], copied[2];
    std::mutex mu;
    std::condition_variable cv;
    std::deque<Job> jobs;
    bool closed = false;
    int done_chips = 0;   // jobs fully combined and drained
    bk_status err = BK_OK;
    std::string msg;
    int64_t launches = 0;
};

bk_status out_fail(Pipe& p, bk_status st, const std::string& m) {
    std::lock_guard<std::mutex> lk(p.mu);
    if (p.err == BK_OK) {
        p.err = st;
        p.msg = m;
    }
    p.cv.notify_all();
    return st;
}

struct Pending {
    bool live = false;
    int chip, slot;
    int64_t j0, m;
};

// hand a drained chunk to the sink (host thread; waits for its D2H)
bool deliver(Pipe& p, const Pending& d) {
    if (!d.live) return true;
    if (cudaEventSynchronize(p.copied[d.slot]) != cudaSuccess) {
        out_fail(p, BK_CUDA_ERROR, "generate_stream: D2H drain failed");
        return false;
    }
    if (p.sink && p.sink(p.user, d.chip, d.j0, d.m, p.n, p.hT[d.slot], p.hQ[d.slot], p.hR[d.slot])) {
        out_fail(p, BK_IO_ERROR, "generate_stream: sink returned an error");
        return false;
    }
    return true;
}

void worker(Pipe* pp) {
    Pipe& p = *pp;
    bk_ctx* out = p.out;
    cudaSetDevice(out->device);
    Pending prev;
    int64_t k = 0;  // chunk counter across chips
    for (;;) {
        Job job;
        {
            std::unique_lock<std::mutex> lk(p.mu);
            p.cv.wait(lk, [&] { return !p.jobs.empty() || p.closed || p.err != BK_OK; });
            if (p.err != BK_OK) return;
            if (p.jobs.empty()) break;
            job = p.jobs.front();
            p.jobs.pop_front();
        }
        if (cudaStreamWaitEvent(out->stream, job.ready, 0) != cudaSuccess) {
            out_fail(p, BK_CUDA_ERROR, "generate_stream: wait for the solve");
            return;
        }
        for (int64_t j0 = 0; j0 < job.N; j0 += p.chunk, ++k) {
            const int sl = (int)(k & 1);
            const int64_t m = std::min(p.chunk, job.N - j0);
            // the slot's previous D2H must be done before the kernel overwrites it
            if (k >= 2 && cudaStreamWaitEvent(out->stream, p.copied[sl], 0) != cudaSuccess) {
                out_fail(p, BK_CUDA_ERROR, "generate_stream: slot wait");
                return;
            }
            const int64_t l0 = out->launches;
            const bk_status st = combine_action_device(out, job.op, job.X, job.S, job.s, job.C + j0,
                                                       job.N, m, p.dT[sl], p.dQ[sl], p.dR[sl]);
            p.launches += out->launches - l0;
            if (st != BK_OK) {
                out_fail(p, st, out->err);
                return;
            }
            const size_t bytes = (size_t)m * p.n * sizeof(double);
            cudaError_t e = cudaEventRecord(p.comp[sl], out->stream);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(out->copy_stream, p.comp[sl], 0);
            // the pinned slot was released when its previous chunk was
            // delivered (the previous loop turn delivered chunk k - 2)
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(p.hT[sl], p.dT[sl], bytes, cudaMemcpyDeviceToHost,
                                    out->copy_stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(p.hQ[sl], p.dQ[sl], bytes, cudaMemcpyDeviceToHost,
                                    out->copy_stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(p.hR[sl], p.dR[sl], (size_t)m * sizeof(double),
                                    cudaMemcpyDeviceToHost, out->copy_stream);
            if (e == cudaSuccess) e = cudaEventRecord(p.copied[sl], out->copy_stream);
            if (e != cudaSuccess) {
                out_fail(p, BK_CUDA_ERROR, std::string("generate_stream: ") + cudaGetErrorString(e));
                return;
            }
            if (!deliver(p, prev)) return;
            prev = Pending{true, job.chip, sl, j0, m};
        }
        // the chip's last chunk is still in flight; its buffers (op, X, C) are
        // read by kernels already enqueued — release them once those finished
        if (cudaStreamSynchronize(out->stream) != cudaSuccess) {
            out_fail(p, BK_CUDA_ERROR, "generate_stream: output stream failed");
            return;
        }
        {
            std::lock_guard<std::mutex> lk(p.mu);
            ++p.done_chips;
        }
        p.cv.notify_all();
    }
    deliver(p, prev);
}

}  // namespace

extern "C" bk_status bk_generate_stream(bk_ctx* ctx, int n_chips, const bk_grid* grids,
                                        const double* const* k, const bk_face* bc,
                                        const double* const* Qbasis, int s,
                                        const double* const* C, int64_t N,
                                        const bk_solver_cfg* cfg, int64_t chunk,
                                        bk_sample_sink sink, void* user,
                                        bk_solve_report* reports, bk_phase_timings* timings) {
    if (!ctx) return BK_INVALID_CONFIG;
    if (n_chips < 0 || !grids || !k || !bc || !Qbasis || !C)
        return fail(ctx, BK_INVALID_CONFIG, "generate_stream: null argument");
    bk_status st = validate_cfg(ctx, cfg);
    if (st != BK_OK) return st;
    if (s < 1) return fail(ctx, BK_EMPTY_BASIS, "generate_stream: empty basis");
    if (s > 64) return fail(ctx, BK_INVALID_CONFIG, "generate_stream: s > 64 not supported");
    if (N < 0) return fail(ctx, BK_INVALID_CONFIG, "generate_stream: n_data must be >= 0");
    if (n_chips == 0) return BK_OK;
    for (int c = 0; c < n_chips; ++c) {
        if ((st = validate_grid(ctx, &grids[c])) != BK_OK) return st;
        if ((int64_t)grids[c].nx * grids[c].ny * grids[c].nz !=
            (int64_t)grids[0].nx * grids[0].ny * grids[0].nz)
            return fail(ctx, BK_DIMENSION_MISMATCH, "generate_stream: chips must share n");
    }
    cudaSetDevice(ctx->device);
    const int64_t n = (int64_t)grids[0].nx * grids[0].ny * grids[0].nz;
    const int S = width_of(s);
    if (chunk <= 0) chunk = std::max<int64_t>(16, ((int64_t)1 << 31) / (16 * n) / 16 * 16);
    chunk = std::min<int64_t>(chunk, std::max<int64_t>(N, 1));
    if ((st = make_out_ctx(ctx)) != BK_OK) return st;
    bk_ctx* out = ctx->out_ctx;
    out->knobs = ctx->knobs;
    if ((st = ensure_copy_stream(out)) != BK_OK) return fail(ctx, st, out->err);

    // rings: device slots (T, Q, resid per slot) on the output context,
    // pinned host slots [T | Q | resid] grow-only
    Pipe p;
    p.out = out;
    p.n = n;
    p.chunk = chunk;
    p.sink = sink;
    p.user = user;
    const size_t fb = (size_t)chunk * n * sizeof(double);
    const int dslot[2][3] = {{kSlotT, kSlotQo, kSlotRes}, {kSlotT1, kSlotQo1, kSlotRes1}};
    for (int sl = 0; sl < 2; ++sl) {
        void *t, *q, *r;
        if ((st = workspace(out, dslot[sl][0], fb, &t)) != BK_OK ||
            (st = workspace(out, dslot[sl][1], fb, &q)) != BK_OK ||
            (st = workspace(out, dslot[sl][2], (size_t)chunk * sizeof(double), &r)) != BK_OK)
            return fail(ctx, st, out->err);
        p.dT[sl] = (double*)t;
        p.dQ[sl] = (double*)q;
        p.dR[sl] = (double*)r;
    }
    const size_t pb = 2 * fb + (size_t)chunk * sizeof(double);
    if (out->pin_bytes < pb) {
        for (auto& h : out->pin)
            if (h) {
                cudaFreeHost(h);
                h = nullptr;
            }
        out->pin_bytes = 0;
        for (auto& h : out->pin) BK_CUDA_TRY(ctx, cudaHostAlloc(&h, pb, cudaHostAllocDefault));
        out->pin_bytes = pb;
    }
    for (int sl = 0; sl < 2; ++sl) {
        p.hT[sl] = (double*)out->pin[sl];
        p.hQ[sl] = p.hT[sl] + (size_t)chunk * n;
        p.hR[sl] = p.hQ[sl] + (size_t)chunk * n;
        BK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&p.comp[sl], cudaEventDisableTiming));
        BK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&p.copied[sl], cudaEventDisableTiming));
    }

    // per-parity chip state: operator, X, C (chip c + 2 reuses chip c's)
    for (auto& o : ctx->stream_ops)
        if (!o) o = new bk_operator;
    bk_operator* ops[2] = {ctx->stream_ops[0], ctx->stream_ops[1]};
    void *px[2], *pc[2], *pb_;
    cudaEvent_t ready[2];
    for (int q = 0; q < 2; ++q) {
        if ((st = workspace(ctx, q ? kSlotStrX1 : kSlotStrX0, (size_t)n * S * 8, &px[q])) != BK_OK)
            return st;
        if ((st = workspace(ctx, q ? kSlotStrC1 : kSlotStrC0, (size_t)s * std::max<int64_t>(N, 1) * 8,
                            &pc[q])) != BK_OK)
            return st;
        BK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&ready[q], cudaEventDisableTiming));
    }
    if ((st = workspace(ctx, kSlotIn2, (size_t)n * S * 8, &pb_)) != BK_OK) return st;
    cudaEvent_t* ev = ctx->ev;
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[0], ctx->stream));

    std::thread th(worker, &p);
    double solve_s = 0.0;
    int64_t iters = 0, matvecs = 0;
    bool not_conv = false;
    auto finish = [&](bk_status rs) -> bk_status {
        {
            std::lock_guard<std::mutex> lk(p.mu);
            p.closed = true;
            if (rs != BK_OK && p.err == BK_OK) p.err = rs;  // stop the worker
        }
        p.cv.notify_all();
        th.join();
        cudaStreamSynchronize(out->stream);
        cudaStreamSynchronize(out->copy_stream);
        ctx->launches += p.launches;
        for (int q = 0; q < 2; ++q) {
            cudaEventDestroy(ready[q]);
            cudaEventDestroy(p.comp[q]);
            cudaEventDestroy(p.copied[q]);
        }
        if (rs != BK_OK) return rs;
        if (p.err != BK_OK) return fail(ctx, p.err, p.msg);
        return BK_OK;
    };

    // after the worker started, every failure path goes through finish()
#define BK_STR_TRY(expr)                                                                  \
    do {                                                                                  \
        const cudaError_t e_ = (expr);                                                    \
        if (e_ != cudaSuccess)                                                            \
            return finish(fail(ctx, BK_CUDA_ERROR,                                        \
                               std::string(#expr) + ": " + cudaGetErrorString(e_)));      \
    } while (0)
    for (int c = 0; c < n_chips; ++c) {
        const int q = c & 1;
        {  // chip c - 2 (same parity) fully drained before its buffers are reused
            std::unique_lock<std::mutex> lk(p.mu);
            p.cv.wait(lk, [&] { return p.done_chips >= c - 1 || p.err != BK_OK; });
            if (p.err != BK_OK) break;
        }
        const bool cdev = is_device_ptr(C[c]);
        if (cdev)
            BK_STR_TRY(cudaMemcpyAsync(pc[q], C[c], (size_t)s * N * 8,
                                             cudaMemcpyDeviceToDevice, ctx->stream));
        else if (N > 0)
            BK_STR_TRY(cudaMemcpyAsync(pc[q], C[c], (size_t)s * N * 8,
                                             cudaMemcpyHostToDevice, ctx->stream));
        if ((st = assemble_into(ctx, &grids[c], k[c], &bc[6 * c], ops[q])) != BK_OK)
            return finish(st);
        const double* qd = Qbasis[c];
        if (!is_device_ptr(qd)) {
            void* t;
            if ((st = workspace(ctx, kSlotQ, (size_t)n * s * 8, &t)) != BK_OK) return finish(st);
            BK_STR_TRY(cudaMemcpyAsync(t, qd, (size_t)n * s * 8, cudaMemcpyHostToDevice,
                                             ctx->stream));
            qd = (const double*)t;
        }
        BK_STR_TRY(launch_rhs_padded(ctx, ops[q], qd, s, (double*)pb_, S));
        BK_STR_TRY(cudaEventRecord(ev[1], ctx->stream));
        CgReport rep;
        if ((st = block_cg_device(ctx, ops[q], (const double*)pb_, S, cfg, (double*)px[q], &rep)) !=
            BK_OK)
            return finish(st);
        BK_STR_TRY(cudaEventRecord(ev[2], ctx->stream));
        BK_STR_TRY(cudaEventRecord(ready[q], ctx->stream));
        BK_STR_TRY(cudaEventSynchronize(ev[2]));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[1], ev[2]);
        solve_s += ms * 1e-3;
        iters += rep.iterations;
        matvecs += rep.matvecs + N;
        for (int j = 0; j < s; ++j) not_conv = not_conv || !rep.converged[j];
        if (reports) fill_report(rep, s, ms * 1e-3, &reports[c]);
        {
            std::lock_guard<std::mutex> lk(p.mu);
            p.jobs.push_back(Job{c, ops[q], (const double*)px[q], (const double*)pc[q], S, s, N,
                                 ready[q]});
        }
        p.cv.notify_all();
    }
#undef BK_STR_TRY
    st = finish(BK_OK);
    BK_CUDA_TRY(ctx, cudaEventRecord(ev[5], ctx->stream));
    BK_CUDA_TRY(ctx, cudaEventSynchronize(ev[5]));
    if (timings) {
        float tot = 0.f;
        cudaEventElapsedTime(&tot, ev[0], ev[5]);
        *timings = bk_phase_timings{};
        timings->basis_solve_s = solve_s;
        timings->total_s = tot * 1e-3;
        timings->iterations_total = iters;
        timings->matvecs_total = matvecs;
    }
    if (st != BK_OK) return st;
    if (not_conv) return fail(ctx, BK_NOT_CONVERGED, "basis solve did not reach tolerance");
    return BK_OK;
}
