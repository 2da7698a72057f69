// Microbenchmarks for design decisions (not part of the product):
//   1. cooperative grid.sync() cost vs a custom acquire/release barrier
//   2. FP64 DFMA throughput, DMMA (mma.sync m8n8k4 f64) throughput
//   3. L2-resident streaming bandwidth (read+write of a 40 MB working set)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void k_gridsync(int iters, int* out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = iters;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ void my_barrier(unsigned* bar, unsigned nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* count = bar;
        unsigned* gen = bar + 32;
        const unsigned g0 = ld_acquire(gen);
        const unsigned arrived = atom_add_release(count, 1u);
        if (arrived == nb - 1) {
            *count = 0;
            st_release(gen, g0 + 1);
        } else {
            while (ld_acquire(gen) == g0) {
            }
        }
    }
    __syncthreads();
}

__global__ void k_mybar(int iters, unsigned* bar, int* out) {
    for (int i = 0; i < iters; ++i) my_barrier(bar, gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = iters;
}

__global__ void k_dfma(int iters, double* out) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dmma(int iters, double* out) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][2] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c[0][0] + c[1][1] + c[2][0] + c[3][1];
}

__global__ void k_dmma16(int iters, double* out) {
    // m16n8k4: A 16x4 (2 regs), B 4x8 (1 reg), C 16x8 (4 regs)
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                         : "d"(a0), "d"(a1), "d"(b));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c[0][0] + c[1][1] + c[2][2] + c[3][3];
}

__global__ void k_stream(const double2* __restrict__ a, double2* __restrict__ b, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
             i += (size_t)gridDim.x * blockDim.x) {
            double2 v = a[i];
            v.x += 1.0;
            b[i] = v;
        }
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int* d_out;
    cudaMalloc(&d_out, 4);
    unsigned* bar;
    cudaMalloc(&bar, 256);
    cudaMemset(bar, 0, 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int per_sm : {1, 2}) {
        for (int bs : {256, 512}) {
            if (bs * per_sm > 1024) continue;
            int iters = 20000;
            int nb = sms * per_sm;
            void* args[] = {&iters, &d_out};
            cudaLaunchCooperativeKernel((void*)k_gridsync, nb, bs, args, 0, 0);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void*)k_gridsync, nb, bs, args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("grid.sync  blocks=%d bs=%d: %.3f us/sync (%s)\n", nb, bs, ms * 1e3 / iters,
                   cudaGetErrorString(cudaGetLastError()));
            void* args2[] = {&iters, &bar, &d_out};
            cudaLaunchCooperativeKernel((void*)k_mybar, nb, bs, args2, 0, 0);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void*)k_mybar, nb, bs, args2, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("custom bar blocks=%d bs=%d: %.3f us/sync (%s)\n", nb, bs, ms * 1e3 / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    double* dout;
    cudaMalloc(&dout, sizeof(double) * sms * 8 * 1024);
    {
        int iters = 20000;
        k_dfma<<<sms * 4, 512>>>(100, dout);
        cudaEventRecord(e0);
        k_dfma<<<sms * 4, 512>>>(iters, dout);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 64 * iters * (double)sms * 4 * 512;
        printf("DFMA: %.2f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
    }
    {
        int iters = 20000;
        k_dmma<<<sms * 4, 256>>>(100, dout);
        cudaEventRecord(e0);
        k_dmma<<<sms * 4, 256>>>(iters, dout);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 4 * iters * (double)sms * 4 * 8;
        printf("DMMA m8n8k4: %.2f TFLOP/s (%s)\n", flops / (ms * 1e-3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
        k_dmma16<<<sms * 4, 256>>>(100, dout);
        cudaEventRecord(e0);
        k_dmma16<<<sms * 4, 256>>>(iters, dout);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 512 * 4 * iters * (double)sms * 4 * 8;
        printf("DMMA m16n8k4: %.2f TFLOP/s (%s)\n", flops / (ms * 1e-3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (size_t mb : {16, 40, 80, 1024}) {
        size_t n = mb * (1u << 20) / 16;
        double2 *a, *b;
        cudaMalloc(&a, n * 16);
        cudaMalloc(&b, n * 16);
        cudaMemset(a, 0, n * 16);
        int reps = mb <= 80 ? 50 : 5;
        k_stream<<<sms * 8, 512>>>(a, b, n, 1);
        cudaEventRecord(e0);
        k_stream<<<sms * 8, 512>>>(a, b, n, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("stream r+w %zu MB x2: %.0f GB/s\n", mb, 2.0 * n * 16 * reps / (ms * 1e-3) / 1e9);
        cudaFree(a);
        cudaFree(b);
    }
    return 0;
}
