#include "topk2_trace.cu"
#include <vector>
#include <algorithm>
#include <random>
namespace fier_cuda {
int fail(int code, const std::string& msg) { printf("fail %s\n", msg.c_str()); return code; }
int check_launch(const char*) { return 0; }
}
int main(int argc, char** argv) {
    int rows = 32, L = 32768, k = 3604;
    if (argc > 1) { rows = atoi(argv[1]); L = atoi(argv[2]); k = atoi(argv[3]); }
    std::vector<float> h((size_t)rows * L);
    std::mt19937 g(1); std::normal_distribution<float> nd(0, 20);
    for (auto& x : h) x = nd(g);
    float* d; int32_t* s; cudaMalloc(&d, h.size() * 4); cudaMalloc(&s, (size_t)rows * k * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    for (int it = 0; it < 5; ++it) fier_cuda::topk2_dispatch(d, rows, L, L, k, s, 0);
    cudaDeviceSynchronize();
    unsigned long long tr[4096][16];
    cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
    // per-phase mean/max over CTAs, relative to the min start
    unsigned long long t0 = ~0ull;
    int n = 0;
    for (int b = 0; b < 4096; ++b) if (tr[b][0]) { t0 = std::min(t0, tr[b][0]); ++n; }
    printf("%d CTAs traced\n", n);
    for (int p = 0; p < 14; ++p) {
        double mean = 0, mx = 0; int c = 0;
        for (int b = 0; b < 4096; ++b) if (tr[b][0] && tr[b][p]) { double v = (tr[b][p] - t0) / 1000.0; mean += v; mx = std::max(mx, v); ++c; }
        printf("phase %d: mean %.2f us  max %.2f us (n=%d)\n", p, c ? mean / c : 0, mx, c);
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int it = 0; it < 50; ++it) fier_cuda::topk2_dispatch(d, rows, L, L, k, s, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("avg %.2f us per launch\n", ms * 1000 / 50);
    return 0;
}
