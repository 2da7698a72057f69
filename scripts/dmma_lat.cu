// Latency of dependent FP64 DMMA (mma.sync m16n8k4) and DFMA chains on one warp,
// and DMMA throughput with 1..8 independent chains per warp (cycles, clock64).
#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
}
template <int C>
__global__ void k_dmma(double* out, long long* cyc, int n) {
    double d[C][4];
    for (int c = 0; c < C; ++c) for (int e = 0; e < 4; ++e) d[c][e] = threadIdx.x * 1e-3 + c;
    const double a0 = 1.0000001, a1 = 0.9999999, b = 1.0000002;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) dmma(d[c], a0, a1, b);
    long long t1 = clock64();
    double s = 0; for (int c = 0; c < C; ++c) s += d[c][0] + d[c][3];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma(double* out, long long* cyc, int n) {
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 1.0000001, 1e-9);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
    const int n = 4096; long long h;
    k_dfma<<<1, 32>>>(o, c, n); k_dfma<<<1, 32>>>(o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent chain: %.1f cycles per fma\n", (double)h / n);
#define RUN(C) k_dmma<C><<<1, 32>>>(o, c, n); k_dmma<C><<<1, 32>>>(o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); \
    printf("DMMA m16n8k4, %d chain(s) per warp: %.1f cycles per step (%.1f per mma)\n", C, (double)h / n, (double)h / n / C);
    RUN(1) RUN(2) RUN(4) RUN(8)
    return 0;
}
