// mma_probe.cu -- microbenchmarks behind the K2 scorer design.
//  1. exactness of mma.sync m16n8k16 bf16 when A holds single-bit bf16 patterns
//     (2^e, e in {-126,...,1}) and B holds w * 2^-e (the "exponent-bit" unpack)
//  2. legacy mma.sync throughput per SM on sm_100a (independent accumulators)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe tools/mma_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// A: 16x16 bf16 row-major, B: 16x8 bf16 (k-major: B[k][n]), D: 16x8 fp32
__global__ void one_mma(const uint16_t* A, const uint16_t* B, float* D) {
    const int lane = threadIdx.x, r = lane >> 2, c = lane & 3;
    auto pk = [](uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); };
    uint32_t a[4] = {pk(A[r * 16 + 2 * c], A[r * 16 + 2 * c + 1]), pk(A[(r + 8) * 16 + 2 * c], A[(r + 8) * 16 + 2 * c + 1]),
                     pk(A[r * 16 + 2 * c + 8], A[r * 16 + 2 * c + 9]),
                     pk(A[(r + 8) * 16 + 2 * c + 8], A[(r + 8) * 16 + 2 * c + 9])};
    uint32_t b[2] = {pk(B[(2 * c) * 8 + r], B[(2 * c + 1) * 8 + r]), pk(B[(2 * c + 8) * 8 + r], B[(2 * c + 9) * 8 + r])};
    float d[4] = {0, 0, 0, 0};
    mma16816(d, a, b);
    D[r * 8 + 2 * c] = d[0];
    D[r * 8 + 2 * c + 1] = d[1];
    D[(r + 8) * 8 + 2 * c] = d[2];
    D[(r + 8) * 8 + 2 * c + 1] = d[3];
}

template <int NACC>
__global__ void mma_loop(float* out, int iters, uint32_t seed) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i) | 0x3f803f80u;
    b[0] = seed ^ 0x3f803f80u;
    b[1] = seed + 0x3f803f80u;
    float d[NACC][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < NACC; ++j) mma16816(d[j], a, b);
    }
    float s = 0;
    for (int j = 0; j < NACC; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    if (s == 12345.f) out[threadIdx.x] = s;
}

static float bf2f(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}
static uint16_t f2bf(float f) {  // RNE
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7fff + ((u >> 16) & 1);
    return (uint16_t)(u >> 16);
}

int main() {
    // ---- 1. exactness ----
    srand(1);
    const int sigma = 40;
    double worst = 0;
    for (int trial = 0; trial < 2000; ++trial) {
        std::vector<uint16_t> A(256), B(128);
        std::vector<int> e_of_k(16);
        for (int k = 0; k < 16; ++k) e_of_k[k] = (1 << (rand() % 8)) - 127;  // bit q in 7..14 -> 2^(2^(q-7)-127)
        for (int m = 0; m < 16; ++m)
            for (int k = 0; k < 16; ++k) {
                const int q = 0;  (void)q;
                const int ebits = e_of_k[k] + 127;  // exponent field
                A[m * 16 + k] = (rand() & 1) ? (uint16_t)(ebits << 7) : 0;
            }
        for (int k = 0; k < 16; ++k)
            for (int n = 0; n < 8; ++n) {
                const float w = ((rand() / (float)RAND_MAX) * 2 - 1) * 16.f;
                B[k * 8 + n] = f2bf(ldexpf(w, -sigma - e_of_k[k]));
            }
        uint16_t *dA, *dB;
        float* dD;
        cudaMalloc(&dA, 512);
        cudaMalloc(&dB, 256);
        cudaMalloc(&dD, 512);
        cudaMemcpy(dA, A.data(), 512, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), 256, cudaMemcpyHostToDevice);
        one_mma<<<1, 32>>>(dA, dB, dD);
        std::vector<float> D(128);
        cudaMemcpy(D.data(), dD, 512, cudaMemcpyDeviceToHost);
        for (int m = 0; m < 16; ++m)
            for (int n = 0; n < 8; ++n) {
                double ref = 0, mag = 0;
                for (int k = 0; k < 16; ++k) {
                    const double p = (double)bf2f(A[m * 16 + k]) * (double)bf2f(B[k * 8 + n]);
                    ref += p;
                    mag += fabs(p);
                }
                const double err = fabs((double)D[m * 8 + n] - ref) / (mag > 0 ? mag : 1);
                if (err > worst) worst = err;
            }
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dD);
    }
    printf("exactness: worst |D-ref|/sum|terms| = %.3e (fp32 accumulation ~6e-8 expected)\n", worst);

    // ---- 2. throughput ----
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4096);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps = 4; warps <= 16; warps *= 2) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            mma_loop<4><<<sms * 2, warps * 32>>>(out, iters, 7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        int clk = 0;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        const double mmas = (double)sms * 2 * warps * iters * 4;
        const double per_sm_clk = mmas / sms / (ms * 1e-3 * clk * 1e3);
        printf("warps/CTA %2d (2 CTA/SM): %.3f ms, %.1f TFLOP/s, %.3f mma/clk/SM (at %d MHz nominal)\n", warps, ms,
               mmas * 4096 / (ms * 1e-3) / 1e12, per_sm_clk, clk / 1000);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
