// gather_tma_probe.cu -- the sparse-attention row gather (K4 / the fused step's phase D):
// 256-B K and V rows at sorted random token indices (C2: 32 heads x 32768 tokens, n = 3604)
// into a per-warp shared-memory ring of 16-row stages, no math, three ways:
//   A  cp.async 16 B per lane (what attn_tc.cuh does)
//   B  one cp.async.bulk per row (256 B, mbarrier completion), lanes 0..15 issue
//   C  TMA tile::gather4: one cp.async.bulk.tensor ... tile::gather4 per 4 rows (a 2D tensor
//     map over the [H*L][128] bf16 cache, box 128 x 1), lanes 0..3 issue
//   D  the same with the layout ldmatrix needs: box 64 x 1 with the 128-byte swizzle, two
//     gather4 per 4 rows (the 256-B rows cannot be swizzled in one box)
// CTAs of 4 warps, 112 rows per warp (the K4 split), ring of NST stages.  In-kernel
// globaltimer first start .. last end (no launch overhead), L2 flushed with clean lines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gather_tma_probe tools/gather_tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

constexpr int H = 32, L = 32768, N = 3604, D = 128, ROWS = 16, RPW = 112;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ bool mbar_wait_bounded(uint32_t bar, uint32_t phase) {
    for (int i = 0; i < (1 << 22); ++i) {
        uint32_t ok;
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(bar), "r"(phase)
            : "memory");
        if (ok) return true;
    }
    return false;  // a wrong expect-tx count: give up instead of hanging the GPU
}

template <int MODE, int NST>
__global__ void __launch_bounds__(128) gather(const uint16_t* K, const uint16_t* V, const int* sel,
                                              const __grid_constant__ CUtensorMap tk,
                                              const __grid_constant__ CUtensorMap tv, unsigned long long* tt,
                                              float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cpw = (N + RPW - 1) / RPW;  // chunks per head
    const int gw = blockIdx.x * 4 + warp;
    const int head = gw / cpw, chunk = gw % cpw;
    uint8_t* ring = sm + warp * NST * ROWS * 512;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 4 * NST * ROWS * 512) + warp * NST;
    float acc = 0.f;
    if (head < H) {
        const int r0 = chunk * RPW, r1 = min(N, r0 + RPW);
        const int* s = sel + (size_t)head * N;
        const int nst = (r1 - r0 + ROWS - 1) / ROWS;
        if (MODE > 0 && lane == 0) {
            for (int i = 0; i < NST; ++i)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bars + i)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        auto issue = [&](int st) {
            if (st >= nst) {
                if (MODE == 0) asm volatile("cp.async.commit_group;");
                return;
            }
            uint8_t* dst = ring + (st % NST) * ROWS * 512;  // K rows [0, 4 KB), V rows [4 KB, 8 KB)
            const int rb = r0 + st * ROWS, nr = min(ROWS, r1 - rb);
            if (MODE == 0) {
                for (int i = lane; i < ROWS * 16; i += 32) {
                    const int rr = i / 16, c = i % 16;
                    const int t = s[rb + min(rr, nr - 1)];
                    const size_t off = ((size_t)head * L + t) * D + c * 8;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + rr * 256 + c * 16)),
                                 "l"(K + off));
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + 4096 + rr * 256 + c * 16)),
                                 "l"(V + off));
                }
                asm volatile("cp.async.commit_group;");
            } else {
                const uint32_t bar = su32(bars + st % NST);
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(ROWS * 512)
                                 : "memory");
                __syncwarp();
                if (MODE == 1 && lane < ROWS) {
                    const int t = s[rb + min(lane, nr - 1)];
                    const size_t off = ((size_t)head * L + t) * D;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                            su32(dst + lane * 256)),
                        "l"(K + off), "r"(bar)
                        : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                            su32(dst + 4096 + lane * 256)),
                        "l"(V + off), "r"(bar)
                        : "memory");
                }
                if (MODE == 3 && lane < ROWS / 4) {
                    int rw[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) rw[j] = head * L + s[rb + min(4 * lane + j, nr - 1)];
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(dst + hh * 2048 + lane * 512)),
                            "l"(&tk), "r"(bar), "r"(64 * hh), "r"(rw[0]), "r"(rw[1]), "r"(rw[2]), "r"(rw[3])
                            : "memory");
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(dst + 4096 + hh * 2048 + lane * 512)),
                            "l"(&tv), "r"(bar), "r"(64 * hh), "r"(rw[0]), "r"(rw[1]), "r"(rw[2]), "r"(rw[3])
                            : "memory");
                    }
                }
                if (MODE == 2 && lane < ROWS / 4) {
                    int rw[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) rw[j] = head * L + s[rb + min(4 * lane + j, nr - 1)];
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(dst + lane * 1024)),
                        "l"(&tk), "r"(bar), "r"(0), "r"(rw[0]), "r"(rw[1]), "r"(rw[2]), "r"(rw[3])
                        : "memory");
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(dst + 4096 + lane * 1024)),
                        "l"(&tv), "r"(bar), "r"(0), "r"(rw[0]), "r"(rw[1]), "r"(rw[2]), "r"(rw[3])
                        : "memory");
                }
            }
        };
        for (int st = 0; st < NST - 1; ++st) issue(st);
        for (int st = 0; st < nst; ++st) {
            issue(st + NST - 1);
            if (MODE == 0) {
                asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1));
            } else if (!mbar_wait_bounded(su32(bars + st % NST), (uint32_t)((st / NST) & 1))) {
                acc = -1e30f;
                break;
            }
            __syncwarp();
            acc += reinterpret_cast<const float*>(ring + (st % NST) * ROWS * 512)[lane];
            __syncwarp();
        }
        if (MODE == 0) asm volatile("cp.async.wait_group 0;");
    }
    if (acc == 1.2345f || acc < -1e29f) out[0] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicMin(tt, t0);
        atomicMax(tt + 1, t1);
    }
}

__global__ void flush(const uint4* p, size_t n, float* out) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc ^= p[i].x;
    if (acc == 0x12345) out[1] = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE, int NST>
void run(const char* name, const uint16_t* K, const uint16_t* V, const int* sel, const CUtensorMap& tk,
         const CUtensorMap& tv, unsigned long long* tt, float* out, const uint4* fl, size_t fn) {
    const int smem = 4 * NST * ROWS * 512 + 4 * NST * 8;
    cudaFuncSetAttribute(gather<MODE, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int warps = H * ((N + RPW - 1) / RPW), ctas = (warps + 3) / 4;
    std::vector<float> ds;
    float hout = 0.f;
    for (int r = 0; r < 9; ++r) {
        flush<<<1184, 512>>>(fl, fn, out);
        unsigned long long init[2] = {~0ull, 0ull};
        cudaMemcpy(tt, init, 16, cudaMemcpyHostToDevice);
        gather<MODE, NST><<<ctas, 128, smem>>>(K, V, sel, tk, tv, tt, out);
        unsigned long long h[2];
        cudaMemcpy(h, tt, 16, cudaMemcpyDeviceToHost);
        cudaMemcpy(&hout, out, 4, cudaMemcpyDeviceToHost);
        ds.push_back((h[1] - h[0]) / 1000.f);
    }
    std::sort(ds.begin(), ds.end());
    const double bytes = (double)H * N * 512;
    printf("%-36s NST %d: %7.2f us  %6.0f GB/s  %s%s\n", name, NST, ds[4], bytes / ds[4] / 1e3,
           cudaGetErrorString(cudaGetLastError()), hout < -1e29f ? "  (TIMED OUT: wrong tx count)" : "");
}

int main() {
    const size_t elems = (size_t)H * L * D;
    uint16_t *K, *V;
    cudaMalloc(&K, elems * 2);
    cudaMalloc(&V, elems * 2);
    cudaMemset(K, 0, elems * 2);
    cudaMemset(V, 0, elems * 2);
    std::mt19937 g(1);
    std::vector<int> h((size_t)H * N);
    for (int hh = 0; hh < H; ++hh) {
        std::vector<int> idx(L);
        for (int i = 0; i < L; ++i) idx[i] = i;
        std::shuffle(idx.begin(), idx.end(), g);
        std::sort(idx.begin(), idx.begin() + N);
        std::copy(idx.begin(), idx.begin() + N, h.begin() + (size_t)hh * N);
    }
    int* sel;
    cudaMalloc(&sel, h.size() * 4);
    cudaMemcpy(sel, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    unsigned long long* tt;
    float* out;
    uint4* fl;
    const size_t fn = (512ull << 20) / 16;
    cudaMalloc(&tt, 16);
    cudaMalloc(&out, 64);
    cudaMemset(out, 0, 64);
    cudaMalloc(&fl, fn * 16);
    cudaMemset(fl, 1, fn * 16);

    EncodeTiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap tk{}, tv{}, tk2{}, tv2{};
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)H * L};
    const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    const cuuint32_t box[2] = {(cuuint32_t)D, 1};
    const cuuint32_t es[2] = {1, 1};
    int ok = enc != nullptr;
    if (ok)
        ok = enc(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                 CUDA_SUCCESS &&
             enc(&tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, V, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                 CUDA_SUCCESS;
    const cuuint32_t box2[2] = {64, 1};
    int ok2 = ok && enc(&tk2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, dims, strides, box2, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
              enc(&tv2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, V, dims, strides, box2, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    printf("tensor maps: %s, swizzled: %s\n", ok ? "ok" : "FAILED", ok2 ? "ok" : "FAILED");
    for (int pass = 0; pass < 2; ++pass) {
        printf("pass %d (C2 selection: %d heads x %d rows of K and V, %.1f MB)\n", pass, H, N, H * N * 512 / 1e6);
        run<0, 2>("A cp.async 16 B", K, V, sel, tk, tv, tt, out, fl, fn);
        run<0, 3>("A cp.async 16 B", K, V, sel, tk, tv, tt, out, fl, fn);
        run<1, 2>("B cp.async.bulk per row", K, V, sel, tk, tv, tt, out, fl, fn);
        run<1, 3>("B cp.async.bulk per row", K, V, sel, tk, tv, tt, out, fl, fn);
        if (ok) {
            run<2, 2>("C TMA tile::gather4", K, V, sel, tk, tv, tt, out, fl, fn);
            run<2, 3>("C TMA tile::gather4", K, V, sel, tk, tv, tt, out, fl, fn);
        }
        if (ok2) {
            run<3, 2>("D TMA gather4, 64-col swizzled boxes", K, V, sel, tk2, tv2, tt, out, fl, fn);
            run<3, 3>("D TMA gather4, 64-col swizzled boxes", K, V, sel, tk2, tv2, tt, out, fl, fn);
        }
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
