// FP64 tensor-core throughput on the whole GPU: mma.sync m16n8k4 / k8 / k16
// (f64), operands in registers or A fragments loaded from shared memory,
// 4 independent accumulator chains per warp, varying warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_tput dmma_tput.cu
#include <cstdio>

template <int K>
struct Mma;
template <>
struct Mma<4> {
    static __device__ __forceinline__ void run(double (&d)[4], const double* a, const double* b) {
        asm volatile(
            "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
            "{%0,%1,%2,%3};"
            : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
            : "d"(a[0]), "d"(a[1]), "d"(b[0]));
    }
};
template <>
struct Mma<8> {
    static __device__ __forceinline__ void run(double (&d)[4], const double* a, const double* b) {
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
};
template <>
struct Mma<16> {
    static __device__ __forceinline__ void run(double (&d)[4], const double* a, const double* b) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
            "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
            : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
              "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
};

template <int K, int CH, bool SMEM>
__global__ void k_tput(double* out, int n) {
    __shared__ double sa[32 * 64];
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) sa[i] = 1.0 + 1e-9 * i;
    __syncthreads();
    double d[CH][4];
    for (int c = 0; c < CH; ++c)
        for (int e = 0; e < 4; ++e) d[c][e] = threadIdx.x * 1e-3 + c;
    double a[K / 2], b[K / 4];
    for (int i = 0; i < K / 2; ++i) a[i] = 1.0000001 + i * 1e-12;
    for (int i = 0; i < K / 4; ++i) b[i] = 0.9999999 - i * 1e-12;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (SMEM) {
#pragma unroll
                for (int i = 0; i < K / 2; ++i) a[i] = sa[(lane * 2 + i + c * 7 + it) & 2047];
            }
            Mma<K>::run(d[c], a, b);
        }
    }
    double s = 0;
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half the warps run DMMA chains, half DFMA chains (8 independent per
// thread): do the FP64 tensor pipe and the SIMT FP64 pipe run concurrently?
__global__ void k_mixed(double* out, int n, int mode) {
    const int warp = threadIdx.x >> 5;
    const bool do_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
    const bool do_fma = mode == 1 || (mode == 2 && (warp & 1) == 1);
    double d[4][4];
    for (int c = 0; c < 4; ++c)
        for (int e = 0; e < 4; ++e) d[c][e] = threadIdx.x * 1e-3 + c;
    double f[8];
    for (int c = 0; c < 8; ++c) f[c] = threadIdx.x * 1e-3 + c;
    const double a[2] = {1.0000001, 0.9999999}, b[1] = {1.0000002};
    if (do_mma)
        for (int it = 0; it < n; ++it)
#pragma unroll
            for (int c = 0; c < 4; ++c) Mma<4>::run(d[c], a, b);
    if (do_fma)
        for (int it = 0; it < 4 * n; ++it)
#pragma unroll
            for (int c = 0; c < 8; ++c) f[c] = fma(f[c], 1.0000001, 1e-9);
    double s = 0;
    for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][3];
    for (int c = 0; c < 8; ++c) s += f[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

void run_mixed(int mode, double* out) {
    const int n = 2000, blocks = 148 * 2, threads = 512;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_mixed<<<blocks, threads>>>(out, 10, mode);
    cudaEventRecord(e0);
    k_mixed<<<blocks, threads>>>(out, n, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double wm = mode == 0 ? 16 : mode == 2 ? 8 : 0, wf = mode == 1 ? 16 : mode == 2 ? 8 : 0;
    const double mma = 2.0 * 16 * 8 * 4 * 4 * (double)n * wm * blocks;
    const double fmaf = 2.0 * 32 * 8 * 4.0 * n * wf * blocks;
    printf("mixed mode %d (0 dmma, 1 dfma, 2 both): %.2f ms  dmma %.1f + dfma %.1f = %.1f TFLOP/s\n",
           mode, ms, mma / ms / 1e9, fmaf / ms / 1e9, (mma + fmaf) / ms / 1e9);
}

template <int K, int CH, bool SMEM>
void run(int warps, double* out) {
    const int n = 2000;
    const int blocks = 148 * 2;
    const int threads = warps * 32 / 2;  // warps per SM split over 2 CTAs
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_tput<K, CH, SMEM><<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    k_tput<K, CH, SMEM><<<blocks, threads>>>(out, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * K * CH * (double)n * (threads / 32) * blocks;
    printf("m16n8k%-2d chains %d smemA %d warps/SM %2d: %6.1f TFLOP/s\n", K, CH, (int)SMEM, warps,
           flops / ms / 1e9);
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 24);
    for (int w : {4, 8, 16, 32}) {
        run<4, 4, false>(w, out);
        run<8, 4, false>(w, out);
        run<16, 4, false>(w, out);
    }
    for (int w : {8, 16}) {
        run<4, 4, true>(w, out);
        run<8, 4, true>(w, out);
        run<16, 4, true>(w, out);
    }
    run_mixed(0, out);
    run_mixed(1, out);
    run_mixed(2, out);
    run<4, 1, false>(16, out);
    run<4, 2, false>(16, out);
    return 0;
}
