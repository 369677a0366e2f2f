/*
 * filterkit_b200.h -- C ABI of the B200 (sm_100a) filter kernels.
 *
 * This is the drop-in boundary: each entry point replaces one function of the
 * reference's kernel contract (the module returned by
 * /root/reference/pkg/src/filterkit/_backends.py:29-40, implemented by
 * _ckernels.pyx / _pykernels.py).  The citation above each declaration names
 * the reference function it replaces.
 *
 * Conventions
 *  - Every table/array pointer is a DEVICE pointer owned by the caller
 *    (the Python facades allocate them as torch CUDA tensors).
 *  - Every call is asynchronous on the given stream (cudaStream_t passed as
 *    void*; NULL = legacy default stream) and never throws.
 *  - Return value: 0 on success, a positive filter code where the reference
 *    returns one (GQF_LOAD_CAPACITY=1, GQF_SHIFT_BOUND=2), FK_E_INVARIANT (-9)
 *    for the reference's _INVARIANT, FK_E_ARG (-1000) for bad arguments, or
 *    -(cudaError_t) on a CUDA failure.
 *  - `keys_are_fps`: 0 = inputs are raw 64-bit keys and the kernel hashes
 *    them with `seed` (fused hashing, hashing.py:66-73); 1 = inputs are
 *    already fingerprints exactly as the reference's contract takes them.
 *  - Workspace: callers query fk_*_workspace_bytes() and pass that much
 *    device memory; kernels never allocate.
 */
#ifndef FILTERKIT_B200_H
#define FILTERKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FK_ABI_VERSION 1
#define FK_E_INVARIANT (-9)
#define FK_E_ARG (-1000)

/* Point-TCF geometry.  Mirrors TcfParams (tcf.py:47-92); the host derives
 * cut_slots and backing_slots exactly as the reference does. */
typedef struct fk_tcf_geom {
    int64_t num_blocks;     /* nb */
    int64_t backing_slots;  /* 0 disables the backing table */
    int32_t block_slots;    /* B  (B * 8 * slot_bytes <= 1024) */
    int32_t tag_bits;       /* f  */
    int32_t slot_bytes;     /* w / 8 in {1, 2, 4, 8} */
    int32_t cut_slots;      /* ceil(shortcut_fraction * B) */
    int32_t probe_limit;    /* backing probes */
    int32_t group_width;    /* cooperative-group tile size g in {1,2,4,8,16,32}, g <= B */
    uint64_t seed;
} fk_tcf_geom;

/* Insert modes (the reference has one semantics per call pattern):
 *  FK_ORDERED    -- bit-identical to the sequential reference stream
 *                   (tcf_insert_batch with one caller thread): deterministic
 *                   reservations by input index.
 *  FK_CONCURRENT -- the paper's free-threaded CAS mode (Alg. 1): every key
 *                   runs at once; equivalent to the reference under many
 *                   caller threads (no false negatives, same policy, any
 *                   linearisation). */
#define FK_ORDERED 0
#define FK_CONCURRENT 1

const char *fk_version(void);
int fk_abi_version(void);

/* Device fingerprints (hashing.py:66-73) + TCF/GQF derived streams, for the
 * hashing parity tests.  out5 gets per key: fp, b1, b2, backing start,
 * backing step (nb/bsize = 0 skips the corresponding columns). */
int fk_hash_streams(const uint64_t *keys, int64_t n, uint64_t seed, int bits, uint64_t nb,
                    uint64_t bsize, uint64_t *out5, void *stream);

/* Exact x % d on device through the fast-mod path (tests only). */
int fk_fastmod_check(const uint64_t *x, int64_t n, uint64_t d, uint64_t *out, void *stream);

/* ---- point TCF --------------------------------------------------------- */

size_t fk_tcf_workspace_bytes(const fk_tcf_geom *g, int64_t n, int mode);

/* replaces tcf_insert_batch (_ckernels.pyx:193-238, _pykernels.py:120-149).
 * counters[0] += inserted, counters[1] += backing placements (device int64[3]). */
int fk_tcf_insert(const fk_tcf_geom *g, void *blocks, void *backing, const uint64_t *keys,
                  int keys_are_fps, const uint64_t *values, int64_t n, uint8_t *codes,
                  int64_t *counters, int mode, void *workspace, size_t ws_bytes, void *stream);

/* replaces tcf_query_batch (_ckernels.pyx:252-300, _pykernels.py:161-197).
 * values_out may be NULL; hits (device int64) may be NULL. */
int fk_tcf_query(const fk_tcf_geom *g, const void *blocks, const void *backing,
                 const uint64_t *keys, int keys_are_fps, int64_t n, uint8_t *found,
                 uint64_t *values_out, void *stream);

/* replaces tcf_delete_batch (_ckernels.pyx:303-355, _pykernels.py:200-236).
 * counters[2] += removed. */
int fk_tcf_delete(const fk_tcf_geom *g, void *blocks, void *backing, const uint64_t *keys,
                  int keys_are_fps, int64_t n, uint8_t *removed, int64_t *counters, int mode,
                  void *workspace, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FILTERKIT_B200_H */
