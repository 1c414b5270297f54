// dsmem_probe.cu -- cost of the fused step's cluster-histogram steps in isolation:
// 4096-bin merge (every thread, uint4 DSMEM loads) vs one warp reading 64 bins from
// every peer (two rounds), right after a cluster barrier; 512 threads, cluster C.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2508_08256_b200/csrc -Iinclude \
//        -o tools/dsmem_probe tools/dsmem_probe.cu
#include <cstdio>
#include <cooperative_groups.h>
#include "select_radix.cuh"
namespace cg = cooperative_groups;
using namespace fier_cuda;

__global__ void __launch_bounds__(512, 1) probe(long long* out, int mode) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ __align__(16) uint32_t hist[4096];
    __shared__ __align__(16) uint32_t tot[4096];
    __shared__ __align__(16) uint32_t coarse[64];
    for (int i = threadIdx.x; i < 4096; i += 512) hist[i] = (i * 7) & 3;
    if (threadIdx.x < 64) coarse[threadIdx.x] = 100;
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
    long long t0 = clock64();
    const int nct = cl.num_blocks();
    uint32_t x = 0;
    if (mode == 0) {
        t2_merge_hist<4096>(cl, nct, hist, tot);
        __syncthreads();
        x = tot[threadIdx.x];
    } else if (mode == 1) {
        if (threadIdx.x < 32) {
            const uint2 a = rx_cluster_sum2(smem_u32(coarse) + 8u * threadIdx.x, nct);
            const uint2 b = rx_cluster_sum2(smem_u32(hist + 64 * (a.x & 7)) + 8u * threadIdx.x, nct);
            x = a.x + b.y;
        }
        __syncthreads();
    } else {
        asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
    }
    long long t1 = clock64();
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (x == 0xdeadbeef) out[1] = x;
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {2, 4, 8, 16})
        for (int mode = 0; mode < 3; ++mode) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(c * 8, 1, 1);
            cfg.blockDim = dim3(512, 1, 1);
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = c;
            a[0].val.clusterDim.y = 1;
            a[0].val.clusterDim.z = 1;
            cfg.attrs = a;
            cfg.numAttrs = 1;
            long long best = 1LL << 60;
            for (int r = 0; r < 5; ++r) {
                cudaLaunchKernelEx(&cfg, probe, d, mode);
                cudaDeviceSynchronize();
                long long v;
                cudaMemcpy(&v, d, 8, cudaMemcpyDeviceToHost);
                best = v < best ? v : best;
            }
            printf("cluster %2d  %-26s %6lld cycles\n", c,
                   mode == 0 ? "merge 4096 bins (all thr)" : mode == 1 ? "warp: 2 x 64 bins" : "cluster barrier",
                   best);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
