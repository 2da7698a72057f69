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
    run<4, 1, false>(16, out);
    run<4, 2, false>(16, out);
    return 0;
}
