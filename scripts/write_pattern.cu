// Write-bandwidth microbenchmark of the combine/action output pattern:
// T and q, sample-major [N][n] (n = 256 x 256), written per work item =
// (TX x TY tile, chunk of 16 samples) by 256 threads (one x-pair each,
// 8 samples per thread half), streaming double2 stores. Items are walked in
// contiguous ranges per CTA (sample chunk fastest), as combine_action_pl_ws.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/write_pattern scripts/write_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int TX, int TY>
__global__ void __launch_bounds__(256) k(double* T, double* Q, int nx, int ny, int N, int order) {
    constexpr int NS = 16;
    const int tilesx = nx / TX, tiles = tilesx * (ny / TY), chunks = N / NS;
    const int items = tiles * chunks;
    const int b0 = (int)((long long)blockIdx.x * items / gridDim.x);
    const int b1 = (int)((long long)(blockIdx.x + 1) * items / gridDim.x);
    const int tt = threadIdx.x;
    const long long n = (long long)nx * ny;
    for (int item = b0; item < b1; ++item) {
        const int tile = order ? item % tiles : item / chunks;
        const int chunk = order ? item / tiles : item % chunks;
        const int x0 = (tile % tilesx) * TX, y0 = (tile / tilesx) * TY;
        for (int p = tt; p < TX * TY / 2; p += 256) {
            const int cell = 2 * p;
            const int gx = x0 + cell % TX, gy = y0 + cell / TX;
            const long long i = gx + (long long)nx * gy;
            for (int q = 0; q < NS; ++q) {
                const long long j = (long long)chunk * NS + q;
                const double2 v = make_double2((double)j, (double)i);
                __stcs(reinterpret_cast<double2*>(T + j * n + i), v);
                __stcs(reinterpret_cast<double2*>(Q + j * n + i), v);
            }
        }
    }
}
template <int TX, int TY>
void run(double* T, double* Q, int order, int grid) {
    const int nx = 256, ny = 256, N = 2048;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k<TX, TY><<<grid, 256>>>(T, Q, nx, ny, N, order);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double bytes = 2.0 * N * nx * ny * 8;
    printf("tile %3dx%-3d order %s grid %4d: %.3f ms  %.0f GB/s\n", TX, TY,
           order ? "tile-fastest " : "chunk-fastest", grid, best, bytes / best / 1e6);
}
int main() {
    double *T, *Q;
    const size_t sz = (size_t)2048 * 65536 * 8;
    cudaMalloc(&T, sz);
    cudaMalloc(&Q, sz);
    for (int grid : {148, 296, 592}) {
        run<32, 8>(T, Q, 0, grid);
        run<32, 8>(T, Q, 1, grid);
        run<64, 4>(T, Q, 0, grid);
        run<128, 2>(T, Q, 0, grid);
        run<256, 1>(T, Q, 0, grid);
        run<256, 1>(T, Q, 1, grid);
    }
    return 0;
}
