// cluster_probe.cu -- latency of cluster.sync(), __syncthreads() and a DSMEM load on sm_100a
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_probe tools/cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void sync_probe(long long* out, int iters, int mode) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ unsigned buf[1024];
    buf[threadIdx.x % 1024] = threadIdx.x;
    cl.sync();
    long long t0 = clock64();
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) cl.sync();
        else if (mode == 1) __syncthreads();
        else {  // dependent DSMEM load chain from the next CTA
            unsigned* r = cl.map_shared_rank(buf, (cl.block_rank() + 1) % cl.num_blocks());
            acc = r[(acc + threadIdx.x) % 1024];
        }
    }
    long long t1 = clock64();
    cl.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
    if (acc == 0xdeadbeef) out[1] = acc;
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    for (int threads : {512, 1024})
        for (int c : {1, 2, 4, 8, 16}) {
            for (int mode = 0; mode < 3; ++mode) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(c * 16, 1, 1);
                cfg.blockDim = dim3(threads, 1, 1);
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeClusterDimension;
                a[0].val.clusterDim.x = c;
                a[0].val.clusterDim.y = 1;
                a[0].val.clusterDim.z = 1;
                cfg.attrs = a;
                cfg.numAttrs = 1;
                cudaFuncSetAttribute(sync_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaError_t e = cudaLaunchKernelEx(&cfg, sync_probe, d, 200, mode);
                cudaDeviceSynchronize();
                long long v = -1;
                cudaMemcpy(&v, d, 8, cudaMemcpyDeviceToHost);
                printf("threads %4d cluster %2d %-12s %6lld cycles %s\n", threads, c,
                       mode == 0 ? "cluster.sync" : mode == 1 ? "syncthreads" : "dsmem load", v,
                       e ? cudaGetErrorString(e) : "");
            }
        }
    return 0;
}
