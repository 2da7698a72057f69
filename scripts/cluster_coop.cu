// Can a cooperative launch use thread-block clusters on this B200 (one
// ~200 KB CTA per SM), and what do grid.sync / cluster.sync / a DSMEM
// cluster reduction cost? (probe for the block-CG grid reductions)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void probe(long long* out, int iters) {
    extern __shared__ double sm[];
    cg::grid_group grid = cg::this_grid();
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < 512; i += blockDim.x) sm[i] = blockIdx.x + i;
    grid.sync();
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) grid.sync();
    long long t1 = clock64();
    for (int k = 0; k < iters; ++k) cl.sync();
    long long t2 = clock64();
    double acc = 0;
    for (int k = 0; k < iters; ++k) {
        // sum element tid over the cluster's CTAs through DSMEM, then sync
        if (threadIdx.x < 272) {
            double s = 0;
            for (int r = 0; r < (int)cl.num_blocks(); ++r) s += cl.map_shared_rank(sm, r)[threadIdx.x];
            acc += s;
        }
        cl.sync();
    }
    long long t3 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        out[0] = (t1 - t0) / iters;
        out[1] = (t2 - t1) / iters;
        out[2] = (t3 - t2) / iters;
    }
    if (acc == -1.0) out[3] = 1;
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        for (int nb : {nsm, (nsm / cs) * cs, 144, 128}) {
            if (nb % cs) continue;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(nb);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            at[1].id = cudaLaunchAttributeClusterDimension;
            at[1].val.clusterDim.x = cs;
            at[1].val.clusterDim.y = 1;
            at[1].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 2;
            int maxc = -1;
            cudaOccupancyMaxActiveClusters(&maxc, probe, &cfg);
            cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d, 200);
            cudaError_t e2 = cudaDeviceSynchronize();
            long long h[4] = {0};
            cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
            printf("cluster %2d grid %3d: max active clusters %3d launch %s/%s grid.sync %lld cyc, "
                   "cluster.sync %lld cyc, dsmem-reduce+sync %lld cyc\n",
                   cs, nb, maxc, cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[1], h[2]);
            cudaGetLastError();
            break;
        }
    }
    return 0;
}
