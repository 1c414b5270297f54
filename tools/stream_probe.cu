// stream_probe.cu -- what bounds a streaming pass of the wide-grid Top-k (topk_global.cu)?
// C4 shape: 1024 rows x 32768 fp32 scores (134 MB, N(0, 20) values), grid (4, 1024) of 256
// threads, 8192 keys per CTA (8 float4 loads per thread, all in flight).
//   mode 0  loads only (xor-reduced)
//   mode 1  loads + digit-1 histogram, one shared-memory copy (atomics)
//   mode 2  loads + digit-1 histogram, 2 copies (lane & 1)
//   mode 3  1/16 sample: one float4 per 64 scores + one histogram copy
// L2 flushed before every launch; in-kernel globaltimer first start .. last end.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_probe tools/stream_probe.cu
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

constexpr int ROWS = 1024, L = 32768, SLICE = 8192, NT = 256;

__device__ __forceinline__ uint32_t fkey(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float4 ldg4(const float* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w));
}

template <int MODE>
__global__ void __launch_bounds__(NT, 4) probe(const float* s, unsigned long long* tt, uint32_t* sink) {
    __shared__ uint32_t h[(MODE == 2 ? 2 : 1) * 4096];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int tid = threadIdx.x;
    const int copies = MODE == 2 ? 2 : 1;
    if (MODE) {
        for (int i = tid; i < copies * 4096; i += NT) h[i] = 0;
        __syncthreads();
    }
    const float* srow = s + (size_t)blockIdx.y * L;
    uint32_t x = 0;
    if (MODE == 3) {
        if (blockIdx.x == 0) {  // one CTA per row samples the whole row: 512 float4
            float4 v[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) v[u] = ldg4(srow + 64 * (tid + NT * u));
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                atomicAdd(&h[fkey(v[u].x) >> 20], 1u);
                atomicAdd(&h[fkey(v[u].y) >> 20], 1u);
                atomicAdd(&h[fkey(v[u].z) >> 20], 1u);
                atomicAdd(&h[fkey(v[u].w) >> 20], 1u);
            }
        }
    } else {
        const int s0 = blockIdx.x * SLICE;
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ldg4(srow + s0 + u * 4 * NT + 4 * tid);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (MODE == 0) x ^= __float_as_uint(e[j]);
                else atomicAdd(&h[(MODE == 2 ? (tid & 1) * 4096 : 0) + (fkey(e[j]) >> 20)], 1u);
            }
        }
    }
    __syncthreads();
    if (MODE) x ^= h[tid];
    if (x == 0x12345678u) sink[0] = x;
    if (tid == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicMin(tt, t0);
        atomicMax(tt + 1, t1);
    }
}

__global__ void flush(const uint4* p, size_t n, uint32_t* out) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc ^= p[i].x;
    if (acc == 0x12345) out[1] = acc;
}

template <int MODE>
void run(const char* name, const float* s, unsigned long long* tt, uint32_t* sink, const uint4* fl, size_t fn) {
    std::vector<float> ds;
    for (int r = 0; r < 7; ++r) {
        flush<<<1184, 512>>>(fl, fn, sink);
        unsigned long long init[2] = {~0ull, 0ull};
        cudaMemcpy(tt, init, 16, cudaMemcpyHostToDevice);
        probe<MODE><<<dim3(L / SLICE, ROWS), NT>>>(s, tt, sink);
        unsigned long long h[2];
        cudaMemcpy(h, tt, 16, cudaMemcpyDeviceToHost);
        ds.push_back((h[1] - h[0]) / 1000.f);
    }
    std::sort(ds.begin(), ds.end());
    printf("%-44s %8.2f us  %6.0f GB/s (of the full 134 MB)\n", name, ds[3], (double)ROWS * L * 4 / ds[3] / 1e3);
}

int main() {
    const size_t n = (size_t)ROWS * L;
    std::vector<float> hs(n);
    std::mt19937 rng(1);
    std::normal_distribution<float> nd(0.f, 20.f);
    for (auto& v : hs) v = nd(rng);
    float* s;
    unsigned long long* tt;
    uint32_t* sink;
    uint4* fl;
    const size_t fn = (512ull << 20) / 16;
    cudaMalloc(&s, n * 4);
    cudaMalloc(&tt, 16);
    cudaMalloc(&sink, 16);
    cudaMalloc(&fl, fn * 16);
    cudaMemset(fl, 1, fn * 16);
    cudaMemcpy(s, hs.data(), n * 4, cudaMemcpyHostToDevice);
    for (int pass = 0; pass < 2; ++pass) {
        run<0>("mode0 loads only", s, tt, sink, fl, fn);
        run<1>("mode1 loads + histogram (1 copy)", s, tt, sink, fl, fn);
        run<2>("mode2 loads + histogram (2 copies)", s, tt, sink, fl, fn);
        run<3>("mode3 1/16 sample + histogram", s, tt, sink, fl, fn);
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
}
