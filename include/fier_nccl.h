/* fier_nccl.h -- device-initiated exchange of the sequence-sharded decode step:
 * the two all-gathers of paper_2508_08256_b200.shard.sharded_step (per-shard Top-n candidates,
 * per-shard attention partials) done by a kernel that stores each rank's slot straight into
 * every peer's symmetric NCCL window over NVLink (NCCL 2.28 device API: ncclGetLsaPointer)
 * and closes with an LSA barrier -- no host-side collective call.
 *
 * Separate library (libfier_nccl.so, linked to the NCCL that torch ships) so libfier_cuda.so
 * keeps no NCCL dependency.  Status codes as fier_cuda.h (0 ok, 1 invalid argument, 3 CUDA /
 * NCCL error); fier_devx_last_error() returns the message. */
#ifndef FIER_NCCL_H
#define FIER_NCCL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef FIER_API
#define FIER_API __attribute__((visibility("default")))
#endif

/* ncclGetUniqueId into out[128] (rank 0 creates it; every rank receives the same bytes). */
FIER_API int fier_devx_unique_id(uint8_t* out);
/* One communicator + one symmetric window of world * slot_bytes (slot r = rank r's data),
 * device communicator with max_ctas LSA barriers.  The current CUDA device is used. */
FIER_API int fier_devx_create(const uint8_t* id, int32_t world, int32_t rank, size_t slot_bytes,
                              int32_t max_ctas, void** handle);
/* All-gather of `bytes` (<= slot_bytes, multiple of 16) from src into slot `rank` of every
 * rank's window, then an LSA barrier; *out = this rank's window (slot r at r * slot_bytes).
 * Graph-capturable (one kernel launch on `stream`). */
FIER_API int fier_devx_allgather(void* handle, const void* src, size_t bytes, void* stream, void** out);
/* fier_shard_candidates (include/fier_cuda.h) fused with the candidate all-gather: this
 * shard's Top-k (sel [rows][k] local indices into scores [rows][ld]) becomes (score, start +
 * index) pairs padded to nc with (-inf, -1), stored straight into slot `rank` of every peer's
 * window as [2][rows][nc] 32-bit words (score bits, then indices), then the LSA barrier.
 * rows * nc * 8 <= slot_bytes.  *out = this rank's window. */
FIER_API int fier_devx_shard_candidates(void* handle, const float* scores, int64_t ld, const int32_t* sel,
                                        int32_t rows, int32_t k, int32_t nc, int64_t start, void* stream,
                                        void** out);
FIER_API int fier_devx_destroy(void* handle);
FIER_API const char* fier_devx_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
