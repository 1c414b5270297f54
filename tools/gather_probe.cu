// gather_probe.cu -- achievable HBM bandwidth of the sparse-attention access pattern:
// 256-B K and V rows at sorted random token indices (density p) of a [H][L][128] bf16 cache,
// streamed into shared memory (cp.async 16 B, or one cp.async.bulk per row), no math.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NST, int ROWS>
__global__ void __launch_bounds__(128) gather_cpasync(const uint4* K, const uint4* V, const int* sel, int n, int L,
                                                      int rows_per_warp, float* out, int pitch16) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 4 + warp;
    const int head = gw / ((n + rows_per_warp - 1) / rows_per_warp);
    const int chunk = gw % ((n + rows_per_warp - 1) / rows_per_warp);
    const int r0 = chunk * rows_per_warp, r1 = min(n, r0 + rows_per_warp);
    const int* s = sel + (size_t)head * n;
    const uint4* Kh = K + (size_t)head * L * pitch16;  // pitch16 = 16 (separate K, V) or 32 (interleaved)
    const uint4* Vh = V + (size_t)head * L * pitch16;
    uint8_t* ring = sm + warp * NST * ROWS * 512;
    const int nst = (r1 - r0 + ROWS - 1) / ROWS;
    auto issue = [&](int st) {
        if (st < nst) {
            uint8_t* dst = ring + (st % NST) * ROWS * 512;
            for (int i = lane; i < ROWS * 16; i += 32) {
                const int rr = i / 16, c = i % 16;
                const int r = r0 + st * ROWS + rr;
                if (r < r1) {
                    const int t = __ldg(s + r);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + rr * 512 + c * 16)), "l"(Kh + (size_t)t * pitch16 + c));
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + rr * 512 + 256 + c * 16)), "l"(Vh + (size_t)t * pitch16 + c));
                }
            }
        }
        asm volatile("cp.async.commit_group;");
    };
    for (int st = 0; st < NST - 1; ++st) issue(st);
    float acc = 0;
    for (int st = 0; st < nst; ++st) {
        issue(st + NST - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1));
        __syncwarp();
        acc += reinterpret_cast<const float*>(ring + (st % NST) * ROWS * 512)[lane];
        __syncwarp();
    }
    if (acc == 1.2345f) out[0] = acc;
}

__global__ void read_flush(const uint4* p, size_t n, float* out) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x12345) out[1] = acc;
}

int main() {
    const int H = 32, L = 32768, n = 3604;
    const size_t kv = (size_t)H * L * 256;
    uint4 *K, *V, *KV;
    cudaMalloc(&K, kv);
    cudaMalloc(&V, kv);
    cudaMalloc(&KV, 2 * kv);
    cudaMemset(K, 0, kv);
    cudaMemset(V, 0, kv);
    cudaMemset(KV, 0, 2 * kv);
    char* flush;
    const size_t fl = 512ull << 20;
    cudaMalloc(&flush, fl);
    float* out;
    cudaMalloc(&out, 64);
    std::mt19937 g(1);
    std::vector<int> h((size_t)H * n);
    for (int hh = 0; hh < H; ++hh) {
        std::vector<int> idx(L);
        for (int i = 0; i < L; ++i) idx[i] = i;
        std::shuffle(idx.begin(), idx.end(), g);
        std::sort(idx.begin(), idx.begin() + n);
        std::copy(idx.begin(), idx.begin() + n, h.begin() + (size_t)hh * n);
    }
    int* sel;
    cudaMalloc(&sel, h.size() * 4);
    cudaMemcpy(sel, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    for (int layout = 0; layout < 2; ++layout)
        for (int cfg = 0; cfg < 4; ++cfg) {
            const int rpw = cfg % 2 ? 256 : 112;
            auto kern = cfg < 2 ? gather_cpasync<3, 16> : gather_cpasync<6, 8>;
            const int smem = 4 * (cfg < 2 ? 3 * 16 : 6 * 8) * 512;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int warps = H * ((n + rpw - 1) / rpw);
            const int ctas = (warps + 3) / 4;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float tot = 0;
            const int reps = 10;
            for (int it = 0; it < reps + 2; ++it) {
                read_flush<<<1184, 512>>>((const uint4*)flush, fl / 16, out);  // evict L2 with clean lines
                cudaEventRecord(e0);
                if (layout == 0) kern<<<ctas, 128, smem>>>(K, V, sel, n, L, rpw, out, 16);
                else kern<<<ctas, 128, smem>>>(KV, KV + 16, sel, n, L, rpw, out, 32);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it >= 2) tot += ms;
            }
            const double bytes = (double)H * n * 512;
            printf("%s nst %d rows/warp %3d ctas %5d: cold-L2 %.2f us  %.0f GB/s  %s\n",
                   layout ? "interleaved KV " : "separate K, V  ", cfg < 2 ? 3 : 6, rpw, ctas, tot * 1000 / reps,
                   bytes / (tot * 1e-3 / reps) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
