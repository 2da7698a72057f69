// Latency microbenchmarks for the s x s solve building blocks (one CTA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/lat scripts/lat_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int reps, long long* out, double* sink) {
    __shared__ double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1.0 + i * 1e-3;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double acc = 0;
    long long t0, t1;
    // 1. barrier only
    t0 = clock64();
    for (int r = 0; r < reps; ++r) __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / reps;
    // 2. REDUX chain (dependent)
    unsigned v = lane * 7 + 3;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) v = __reduce_max_sync(0xffffffffu, v + r) & 0xffff;
    t1 = clock64();
    if (threadIdx.x == 0) out[1] = (t1 - t0) / reps;
    acc += v;
    // 3. double shuffle chain
    double d = lane * 0.5;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) d = __shfl_xor_sync(0xffffffffu, d, 1) + 1.0;
    t1 = clock64();
    if (threadIdx.x == 0) out[2] = (t1 - t0) / reps;
    acc += d;
    // 4. __drcp_rn chain
    d = 1.5 + lane;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) d = __drcp_rn(d) + 1.0;
    t1 = clock64();
    if (threadIdx.x == 0) out[3] = (t1 - t0) / reps;
    acc += d;
    // 5. division chain
    d = 1.5 + lane;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) d = 1.0 / d + 1.0;
    t1 = clock64();
    if (threadIdx.x == 0) out[4] = (t1 - t0) / reps;
    acc += d;
    // 6. DFMA chain
    d = 1.5 + lane;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) d = fma(d, 0.999, 1e-3);
    t1 = clock64();
    if (threadIdx.x == 0) out[5] = (t1 - t0) / reps;
    acc += d;
    // 7. smem load->fma->store chain
    int idx = lane;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double x = sm[idx];
        sm[idx] = fma(x, 0.999, 1e-3);
        idx = (idx + 1) & 1023;
    }
    t1 = clock64();
    if (threadIdx.x == 0) out[6] = (t1 - t0) / reps;
    // 8. DSETP compare chain
    d = 1.5 + lane;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) d = (d > 2.0) ? d - 0.5 : d + 1.0;
    t1 = clock64();
    if (threadIdx.x == 0) out[7] = (t1 - t0) / reps;
    acc += d;
    // 9. smem load latency chain (pointer chasing through smem)
    int j = (int)sm[lane] & 1023;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) j = ((int)sm[j] + r) & 1023;
    t1 = clock64();
    if (threadIdx.x == 0) out[8] = (t1 - t0) / reps;
    acc += j;
    // 10. ballot + ffs chain
    unsigned m = lane;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) m = __ffs(__ballot_sync(0xffffffffu, (lane + m) & 1)) + r;
    t1 = clock64();
    if (threadIdx.x == 0) out[9] = (t1 - t0) / reps;
    acc += m;
    sink[threadIdx.x] = acc;
}

int main() {
    long long* d;
    double* s;
    cudaMalloc(&d, 16 * 8);
    cudaMalloc(&s, 1024 * 8);
    const char* names[] = {"__syncthreads", "REDUX max chain", "double SHFL chain", "__drcp_rn chain",
                           "1.0/x chain", "DFMA chain", "LDS->DFMA->STS chain", "DSETP select chain",
                           "LDS pointer chase", "BALLOT+FFS chain"};
    for (int bs : {32, 128, 256, 512}) {
        k<<<1, bs>>>(1000, d, s);
        cudaDeviceSynchronize();
        long long h[16];
        cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
        printf("block %d threads (%s):\n", bs, cudaGetErrorString(cudaGetLastError()));
        for (int i = 0; i < 10; ++i) printf("  %-24s %lld cycles\n", names[i], h[i]);
    }
    return 0;
}
