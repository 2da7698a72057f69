// Is mma.sync.m16n8k4.f64 accumulation bitwise equal to a k-ordered fma chain?
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void k(const double* A, const double* B, int K, double* D_mma, double* D_fma) {
    // A: 16 x K row-major, B: K x 8 row-major; one warp
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    double d[4] = {0, 0, 0, 0};
    for (int k0 = 0; k0 < K; k0 += 4) {
        double a0 = A[g * K + k0 + t], a1 = A[(g + 8) * K + k0 + t], b = B[(k0 + t) * 8 + g];
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
    }
    const int r0 = g, c0 = 2 * t;
    D_mma[r0 * 8 + c0] = d[0]; D_mma[r0 * 8 + c0 + 1] = d[1];
    D_mma[(r0 + 8) * 8 + c0] = d[2]; D_mma[(r0 + 8) * 8 + c0 + 1] = d[3];
    if (lane < 16) {
        for (int c = 0; c < 8; ++c) {
            double acc = A[lane * K] * B[c];
            for (int kk = 1; kk < K; ++kk) acc = fma(A[lane * K + kk], B[kk * 8 + c], acc);
            D_fma[lane * 8 + c] = acc;
        }
    }
}
int main() {
    const int K = 64;
    double *A, *B, *Dm, *Df;
    cudaMallocManaged(&A, 16 * K * 8); cudaMallocManaged(&B, K * 8 * 8);
    cudaMallocManaged(&Dm, 128 * 8); cudaMallocManaged(&Df, 128 * 8);
    srand(1);
    int total_diff = 0, tot = 0;
    double maxrel = 0;
    for (int trial = 0; trial < 200; ++trial) {
        for (int i = 0; i < 16 * K; ++i) A[i] = (rand() / (double)RAND_MAX) * 50.0 * ((i % 7 == 0) ? -1 : 1);
        for (int i = 0; i < K * 8; ++i) B[i] = rand() / (double)RAND_MAX;
        k<<<1, 32>>>(A, B, K, Dm, Df);
        cudaDeviceSynchronize();
        for (int i = 0; i < 128; ++i) {
            ++tot;
            if (Dm[i] != Df[i]) { ++total_diff; double r = fabs(Dm[i] - Df[i]) / fabs(Df[i]); if (r > maxrel) maxrel = r; }
        }
    }
    printf("DMMA vs fma chain: %d of %d differ, max rel diff %.3e (%s)\n", total_diff, tot, maxrel, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
