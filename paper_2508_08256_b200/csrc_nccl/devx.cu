// devx.cu -- the sequence-sharded step's exchange through the NCCL 2.28 device API
// (include/fier_nccl.h).  Replaces the two host-launched ncclAllGather calls of
// shard.DistExchange: each rank's CTA c copies chunk c of its slot into every peer's
// symmetric window with plain (LSA) stores over NVLink, then syncs LSA barrier c with the
// peers' CTA c -- after which every peer's chunk c has landed in this rank's window (the
// barrier orders the peers' stores before this CTA returns), so when the kernel ends the
// whole gathered buffer is complete.  The consumer is the next launch on the same stream.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <climits>
#include <cstring>
#include <string>

#include "../../include/fier_nccl.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

struct Devx {
    ncclComm_t comm = nullptr;
    ncclDevComm dev{};
    ncclWindow_t win = nullptr;
    void* buf = nullptr;
    size_t slot = 0;
    int world = 0, rank = 0, ctas = 0;
    bool have_dev = false;
};

constexpr int kThreads = 512;

__global__ void __launch_bounds__(kThreads) devx_allgather_kernel(ncclDevComm dev, ncclWindow_t win, size_t slot,
                                                                  int rank, int world, const uint4* __restrict__ src,
                                                                  size_t n16) {
    // chunk of this CTA (16-byte words)
    const size_t per = (n16 + gridDim.x - 1) / gridDim.x;
    const size_t w0 = blockIdx.x * per, w1 = w0 + per < n16 ? w0 + per : n16;
    for (int p = 0; p < world; ++p) {
        uint4* dst = reinterpret_cast<uint4*>(ncclGetLsaPointer(win, (size_t)rank * slot, p));
        for (size_t i = w0 + threadIdx.x; i < w1; i += kThreads) dst[i] = src[i];
    }
    // barrier c with the peers' CTA c: their chunk c is in this rank's window after it
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dev, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

// The candidate exchange fused with the candidate construction (fier_shard_candidates):
// element i of row r of this shard's Top-min(n, l) becomes (score, global index) -- or the
// (-inf, -1) padding past k -- and is stored straight into slot `rank` of every peer's window
// ([2][rows][nc] words: score bits, then indices), then LSA barrier c as above.
__global__ void __launch_bounds__(kThreads) devx_candidates_kernel(ncclDevComm dev, ncclWindow_t win, size_t slot,
                                                                   int rank, int world,
                                                                   const float* __restrict__ scores, int64_t ld,
                                                                   const int32_t* __restrict__ sel, int rows, int k,
                                                                   int nc, int start) {
    const int64_t total = (int64_t)rows * nc;
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t e0 = blockIdx.x * per, e1 = e0 + per < total ? e0 + per : total;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
        const int row = (int)(e / nc), i = (int)(e - (int64_t)row * nc);
        float v = -INFINITY;
        int32_t gi = -1;
        if (i < k) {
            const int32_t t = sel[(int64_t)row * k + i];
            v = scores[(int64_t)row * ld + t];
            gi = start + t;
        }
        for (int p = 0; p < world; ++p) {
            uint32_t* dst = reinterpret_cast<uint32_t*>(ncclGetLsaPointer(win, (size_t)rank * slot, p));
            dst[e] = __float_as_uint(v);
            dst[total + e] = (uint32_t)gi;
        }
    }
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dev, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

}  // namespace

extern "C" {

FIER_API int fier_devx_shard_candidates(void* handle, const float* scores, int64_t ld, const int32_t* sel,
                                        int32_t rows, int32_t k, int32_t nc, int64_t start, void* stream,
                                        void** out) {
    Devx* d = static_cast<Devx*>(handle);
    if (!d || !out || rows < 1 || nc < 1 || k < 0 || k > nc || (k > 0 && (!scores || !sel)) ||
        (size_t)rows * nc * 8 > d->slot || start < 0 || start > INT32_MAX)
        return fail(1, "fier_devx_shard_candidates: invalid arguments (rows * nc * 8 bytes must fit the slot)");
    const int64_t total = (int64_t)rows * nc;
    int ctas = (int)((total + kThreads * 4 - 1) / (kThreads * 4));
    if (ctas > d->ctas) ctas = d->ctas;
    if (ctas < 1) ctas = 1;
    devx_candidates_kernel<<<ctas, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        d->dev, d->win, d->slot, d->rank, d->world, scores, ld, sel, rows, k, nc, (int)start);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(3, std::string("fier_devx_shard_candidates: ") + cudaGetErrorString(e));
    *out = d->buf;
    return 0;
}

FIER_API const char* fier_devx_last_error(void) { return g_err.c_str(); }

FIER_API int fier_devx_unique_id(uint8_t* out) {
    if (!out) return fail(1, "fier_devx_unique_id: null buffer");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(3, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, sizeof(id));
    return 0;
}

FIER_API int fier_devx_create(const uint8_t* id, int32_t world, int32_t rank, size_t slot_bytes, int32_t max_ctas,
                              void** handle) {
    if (!id || !handle || world < 1 || rank < 0 || rank >= world || slot_bytes == 0 || slot_bytes % 16 ||
        max_ctas < 1)
        return fail(1, "fier_devx_create: invalid arguments");
    Devx* d = new Devx();
    d->world = world;
    d->rank = rank;
    d->ctas = max_ctas;
    d->slot = (slot_bytes + 4095) / 4096 * 4096;  // NCCL_WIN_REQUIRED_ALIGNMENT per slot
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclResult_t r = ncclCommInitRank(&d->comm, world, uid, rank);
    if (r == ncclSuccess) r = ncclMemAlloc(&d->buf, d->slot * world);
    if (r == ncclSuccess) r = ncclCommWindowRegister(d->comm, d->buf, d->slot * world, &d->win, NCCL_WIN_COLL_SYMMETRIC);
    if (r == ncclSuccess) {
        ncclDevCommRequirements req;
        std::memset(&req, 0, sizeof(req));
        req.lsaBarrierCount = max_ctas;
        r = ncclDevCommCreate(d->comm, &req, &d->dev);
        d->have_dev = r == ncclSuccess;
    }
    if (r != ncclSuccess) {
        const std::string msg = std::string("fier_devx_create: ") + ncclGetErrorString(r);
        fier_devx_destroy(d);
        return fail(3, msg);
    }
    *handle = d;
    return 0;
}

FIER_API int fier_devx_allgather(void* handle, const void* src, size_t bytes, void* stream, void** out) {
    Devx* d = static_cast<Devx*>(handle);
    if (!d || !src || !out || bytes == 0 || bytes % 16 || bytes > d->slot || (reinterpret_cast<uintptr_t>(src) & 15))
        return fail(1, "fier_devx_allgather: invalid arguments (bytes must be a multiple of 16 within the slot)");
    const size_t n16 = bytes / 16;
    int ctas = (int)((n16 + kThreads * 4 - 1) / (kThreads * 4));
    if (ctas > d->ctas) ctas = d->ctas;
    if (ctas < 1) ctas = 1;
    devx_allgather_kernel<<<ctas, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        d->dev, d->win, d->slot, d->rank, d->world, static_cast<const uint4*>(src), n16);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(3, std::string("fier_devx_allgather: ") + cudaGetErrorString(e));
    *out = d->buf;
    return 0;
}

FIER_API int fier_devx_destroy(void* handle) {
    Devx* d = static_cast<Devx*>(handle);
    if (!d) return 0;
    if (d->comm) {
        if (d->have_dev) ncclDevCommDestroy(d->comm, &d->dev);
        if (d->win) ncclCommWindowDeregister(d->comm, d->win);
        if (d->buf) ncclMemFree(d->buf);
        ncclCommDestroy(d->comm);
    }
    delete d;
    return 0;
}

}  // extern "C"
