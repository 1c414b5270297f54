// fier_io.cu -- FIER packed-index and KVD1 cache-dump byte streams straight to/from
// device buffers: persist / replay a prefill index and load real
// captured caches without a host-side (de)serialisation pass.
//
// Formats (reference io.hpp):
//   FIER v1  serialize_packed_keys :197-225 / parse_packed_keys :227-277
//            "FIER" u16 version=1, u32 l, u32 d, u32 g, then channel-major (s, z) binary16
//            pairs [d][ceil(l/g)], then the row-major bit plane, ceil(d/8) bytes per token,
//            LSB-first.
//   KVD1 v1  serialize_cache_dump :110-137 / parse_cache_dump :140-185
//            "KVD1" u16 version=1, u32 l, u32 d, u16 dtype (0 = f16, 1 = f32), u32 nq, then
//            K [l][d], V [l][d], queries [nq][d] in the dtype.
// Device index layout (include/fier_cuda.h): bits [cap][W] u32 (bit i of word w =
// channel 32w + i), params [ceil(cap/g)][d] (s, z) binary16 pairs.  All kernels are
// byte/integer moves, HBM-bound: coalesced 32x32 shared-memory transposes for the
// (s, z) table, one thread per output byte / word for the bit plane.
#include <cuda_fp16.h>

#include <cstring>
#include <string>

#include "common.cuh"

namespace fier_cuda {

constexpr int kFierHdr = 18;
constexpr int kKvdHdr = 20;

__global__ void io_put_header(uint8_t* out, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t w4,
                              int n) {
    // bytes [0, n) of the little-endian words w0..w4 (magic first)
    const int i = threadIdx.x;
    if (i < n) {
        const uint32_t w[5] = {w0, w1, w2, w3, w4};
        out[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
    }
}

// (s, z) table: in[G][d] u32 (s | z << 16) <-> out[d][G] u16 pairs at a 2-byte aligned address.
__global__ void io_sz_to_fier(const uint32_t* __restrict__ in, int G, int d, uint16_t* __restrict__ out) {
    __shared__ uint32_t tile[32][33];
    const int g0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int gi = g0 + r, j = j0 + threadIdx.x;
        if (gi < G && j < d) tile[r][threadIdx.x] = in[(int64_t)gi * d + j];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int j = j0 + r, gi = g0 + threadIdx.x;
        if (gi < G && j < d) {
            const uint32_t v = tile[threadIdx.x][r];
            out[2 * ((int64_t)j * G + gi)] = (uint16_t)v;
            out[2 * ((int64_t)j * G + gi) + 1] = (uint16_t)(v >> 16);
        }
    }
}

__global__ void io_sz_from_fier(const uint16_t* __restrict__ in, int G, int d, uint32_t* __restrict__ out) {
    __shared__ uint32_t tile[32][33];
    const int j0 = blockIdx.y * 32, g0 = blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int j = j0 + r, gi = g0 + threadIdx.x;
        if (gi < G && j < d) {
            const int64_t e = (int64_t)j * G + gi;
            tile[r][threadIdx.x] = (uint32_t)in[2 * e] | ((uint32_t)in[2 * e + 1] << 16);
        }
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int gi = g0 + r, j = j0 + threadIdx.x;
        if (gi < G && j < d) out[(int64_t)gi * d + j] = tile[threadIdx.x][r];
    }
}

// bit plane: byte bb of token t = bits 8bb..8bb+7 of the row (bits past d are zero in the index)
__global__ void io_bits_to_fier(const uint32_t* __restrict__ bits, int64_t l, int W, int row_bytes,
                                uint8_t* __restrict__ out) {
    const int64_t n = l * row_bytes;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / row_bytes;
        const int bb = (int)(i - t * row_bytes);
        out[i] = (uint8_t)(bits[t * W + (bb >> 2)] >> (8 * (bb & 3)));
    }
}

// word w of token t from bytes 4w..4w+3 of its row; channels >= d are dropped (io.hpp:266)
__global__ void io_bits_from_fier(const uint8_t* __restrict__ in, int64_t l, int W, int row_bytes, int d,
                                  uint32_t* __restrict__ bits) {
    const int64_t n = l * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / W;
        const int w = (int)(i - t * W);
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int bb = 4 * w + b;
            if (bb < row_bytes) v |= (uint32_t)in[t * row_bytes + bb] << (8 * b);
        }
        const int valid = d - 32 * w;
        bits[i] = valid >= 32 ? v : (v & ((1u << valid) - 1u));
    }
}

// KVD1 payload <-> fp32 values (binary16 exact in fp32; fp32 -> binary16 round to nearest
// even = double_to_half of the exactly representable value, half.hpp:30-61)
__global__ void io_kvd_decode(const uint8_t* __restrict__ in, int64_t n, int f16, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = f16 ? __half2float(reinterpret_cast<const __half*>(in)[i]) : reinterpret_cast<const float*>(in)[i];
}

__global__ void io_kvd_encode(const float* __restrict__ in, int64_t n, int f16, uint8_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (f16)
            reinterpret_cast<__half*>(out)[i] = __float2half_rn(in[i]);
        else
            reinterpret_cast<float*>(out)[i] = in[i];
    }
}

static int io_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 8 * num_sms())); }

static int launched(const char* what) {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FIER_OK : fail(FIER_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace fier_cuda

using namespace fier_cuda;

extern "C" {

int fier_index_export(const uint32_t* bits, const void* params, int32_t tokens, int32_t dim, int32_t group,
                      uint8_t* out, size_t out_bytes, void* stream) {
    FIER_REQUIRE(tokens >= 1 && dim >= 1 && group >= 1, "serialize_packed_keys: invalid dims");
    const size_t need = kFierHdr + fier_payload_bytes(tokens, dim, group);
    FIER_REQUIRE(bits && params && out && out_bytes >= need, "serialize_packed_keys: output buffer too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int W = (dim + 31) / 32, row_bytes = (dim + 7) / 8;
    const int G = (int)ceil_div(tokens, group);
    // "FIER", version 1, l, d, g (little-endian, 18 bytes)
    io_put_header<<<1, 32, 0, st>>>(out, 0x52454946u, 1u | ((uint32_t)tokens << 16),
                                    ((uint32_t)tokens >> 16) | ((uint32_t)dim << 16),
                                    ((uint32_t)dim >> 16) | ((uint32_t)group << 16), (uint32_t)group >> 16, kFierHdr);
    io_sz_to_fier<<<dim3(ceil_div(dim, 32), ceil_div(G, 32)), dim3(32, 8), 0, st>>>(
        static_cast<const uint32_t*>(params), G, dim, reinterpret_cast<uint16_t*>(out + kFierHdr));
    const int64_t plane = (int64_t)tokens * row_bytes;
    io_bits_to_fier<<<io_grid(plane), 256, 0, st>>>(bits, tokens, W, row_bytes,
                                                    out + kFierHdr + (size_t)4 * dim * G);
    return launched("fier_index_export");
}

int fier_index_import(const uint8_t* in, size_t in_bytes, int32_t* tokens, int32_t* dim, int32_t* group,
                      uint32_t* bits, int64_t bits_words, void* params, int64_t param_pairs, void* stream) {
    FIER_REQUIRE(in != nullptr, "parse_packed_keys: null input");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t hdr[kFierHdr] = {0};
    const size_t nh = in_bytes < (size_t)kFierHdr ? in_bytes : (size_t)kFierHdr;
    if (nh) {
        if (cudaMemcpyAsync(hdr, in, nh, cudaMemcpyDeviceToHost, st) != cudaSuccess || cudaStreamSynchronize(st))
            return fail(FIER_ECUDA, "fier_index_import: header read failed");
    }
    int32_t l = 0, d = 0, g = 0;  // the host parser's checks and diagnostics on (header, length)
    const int rc = fier_fier_to_index(hdr, in_bytes, &l, &d, &g, nullptr, 0, nullptr, 0);
    if (rc != FIER_OK) return rc;
    if (tokens) *tokens = l;
    if (dim) *dim = d;
    if (group) *group = g;
    if (!bits || !params) return FIER_OK;  // size query
    const int W = (d + 31) / 32, row_bytes = (d + 7) / 8;
    const int G = (int)ceil_div(l, g);
    if (bits_words < (int64_t)l * W || param_pairs < (int64_t)G * d)
        return fail(FIER_EINVAL, "parse_packed_keys: output buffers too small");
    io_sz_from_fier<<<dim3(ceil_div(G, 32), ceil_div(d, 32)), dim3(32, 8), 0, st>>>(
        reinterpret_cast<const uint16_t*>(in + kFierHdr), G, d, static_cast<uint32_t*>(params));
    io_bits_from_fier<<<io_grid((int64_t)l * W), 256, 0, st>>>(in + kFierHdr + (size_t)4 * d * G, l, W, row_bytes,
                                                               d, bits);
    return launched("fier_index_import");
}

int fier_kvd1_load(const uint8_t* in, size_t in_bytes, int32_t* tokens, int32_t* dim, int32_t* queries,
                   int32_t* dtype, float* values, int64_t values_cap, void* stream) {
    // Diagnostics follow parse_cache_dump / ByteReader (io.hpp:110-134, 140-185).
    FIER_REQUIRE(in != nullptr, "parse_cache_dump: null input");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t h[kKvdHdr] = {0};
    const size_t nh = in_bytes < (size_t)kKvdHdr ? in_bytes : (size_t)kKvdHdr;
    if (nh) {
        if (cudaMemcpyAsync(h, in, nh, cudaMemcpyDeviceToHost, st) != cudaSuccess || cudaStreamSynchronize(st))
            return fail(FIER_ECUDA, "fier_kvd1_load: header read failed");
    }
    auto u16 = [&](int o) { return (uint32_t)h[o] | ((uint32_t)h[o + 1] << 8); };
    auto u32 = [&](int o) { return u16(o) | (u16(o + 2) << 16); };
    if (in_bytes < 4) return fail(FIER_EDATA, "truncated file while reading magic");
    if (std::memcmp(h, "KVD1", 4) != 0) return fail(FIER_EDATA, "bad magic: expected KVD1");
    if (in_bytes < 6) return fail(FIER_EDATA, "truncated file while reading version");
    if (u16(4) != 1) return fail(FIER_EDATA, "unsupported version: " + std::to_string(u16(4)));
    if (in_bytes < 10) return fail(FIER_EDATA, "truncated file while reading l");
    if (in_bytes < 14) return fail(FIER_EDATA, "truncated file while reading d");
    const uint32_t l = u32(6), d = u32(10);
    if (l == 0) return fail(FIER_EDATA, "invalid l: must be >= 1");
    if (d == 0) return fail(FIER_EDATA, "invalid d: must be >= 1");
    if (in_bytes < 16) return fail(FIER_EDATA, "truncated file while reading dtype");
    const uint32_t dt = u16(14);
    if (dt > 1) return fail(FIER_EDATA, "invalid dtype code: " + std::to_string(dt));
    if (in_bytes < 20) return fail(FIER_EDATA, "truncated file while reading query_count");
    const uint32_t nq = u32(16);
    const size_t vsize = dt == 0 ? 2 : 4;
    const size_t count = (2 * (size_t)l + nq) * (size_t)d;
    if (in_bytes - kKvdHdr != count * vsize)
        return fail(FIER_EDATA, "payload length mismatch: header declares " + std::to_string(count * vsize) +
                                    " bytes, found " + std::to_string(in_bytes - kKvdHdr));
    if (l > 0x7FFFFFFFu || d > 0x7FFFFFFFu || nq > 0x7FFFFFFFu)
        return fail(FIER_EDATA, "cache dump dimensions exceed the device layout");
    if (tokens) *tokens = (int32_t)l;
    if (dim) *dim = (int32_t)d;
    if (queries) *queries = (int32_t)nq;
    if (dtype) *dtype = (int32_t)dt;
    if (!values) return FIER_OK;  // size query
    if (values_cap < (int64_t)count) return fail(FIER_EINVAL, "parse_cache_dump: output buffer too small");
    io_kvd_decode<<<io_grid((int64_t)count), 256, 0, st>>>(in + kKvdHdr, (int64_t)count, dt == 0, values);
    return launched("fier_kvd1_load");
}

int fier_kvd1_store(const float* values, int32_t tokens, int32_t dim, int32_t queries, int32_t dtype, uint8_t* out,
                    size_t out_bytes, void* stream) {
    FIER_REQUIRE(tokens >= 1 && dim >= 1 && queries >= 0 && (dtype == 0 || dtype == 1),
                 "serialize_cache_dump: invalid dims or dtype");
    const size_t count = (2 * (size_t)tokens + (size_t)queries) * (size_t)dim;
    FIER_REQUIRE(values && out && out_bytes >= kKvdHdr + count * (dtype == 0 ? 2 : 4),
                 "serialize_cache_dump: output buffer too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // "KVD1", version 1, l, d, dtype, nq (20 bytes)
    io_put_header<<<1, 32, 0, st>>>(out, 0x3144564Bu, 1u | ((uint32_t)tokens << 16),
                                    ((uint32_t)tokens >> 16) | ((uint32_t)dim << 16),
                                    ((uint32_t)dim >> 16) | ((uint32_t)dtype << 16), (uint32_t)queries, kKvdHdr);
    io_kvd_encode<<<io_grid((int64_t)count), 256, 0, st>>>(values, (int64_t)count, dtype == 0, out + kKvdHdr);
    return launched("fier_kvd1_store");
}

}  // extern "C"
