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

/* Per-device setup, called once per device by the facades: sets the L2 fetch
 * granularity hint (cudaLimitMaxL2FetchGranularity) to l2_fetch_bytes (32 by
 * default: every filter probe is a random 32-byte sector); <= 0 leaves it. */
int fk_device_setup(int l2_fetch_bytes);
int fk_device_l2_fetch_bytes(void);

/* Device fingerprints (hashing.py:66-73) + TCF/GQF derived streams, for the
 * hashing parity tests.  out5 gets per key: fp, b1, b2, backing start,
 * backing step (nb/bsize = 0 skips the corresponding columns). */
int fk_hash_streams(const uint64_t *keys, int64_t n, uint64_t seed, int bits, uint64_t nb,
                    uint64_t bsize, uint64_t *out5, void *stream);

/* Measurement kernel (not a reference function): n random 32-byte sector
 * loads over [table, table + table_bytes) with the filters' hash stream; the
 * bench times it on the filter's own table as the random-access ceiling. */
int fk_sector_gather(const void *table, int64_t table_bytes, int64_t n, uint64_t salt, uint32_t *sink,
                     void *stream);

/* Device key generation: out[i] = mix64(mix64(seed ^ tag) + start + i),
 * bit-identical to workloads.counter_stream (fk/workloads.py:23-26) and
 * therefore to the reference CLI's uniform and negative-query key streams
 * (TAG_UNIFORM / TAG_FPR, fk/workloads.py:61-64, :205-208). */
int fk_counter_stream(uint64_t seed, uint64_t tag, uint64_t start, int64_t n, uint64_t *out, void *stream);

/* Measurement kernel (not a reference function): n random 32-byte sector
 * read-modify-writes (load the sector, store one 16-bit word back) over the
 * table -- the insert/delete access pattern; overwrites table contents. */
int fk_sector_rmw(void *table, int64_t table_bytes, int64_t n, uint64_t salt, void *stream);

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

/* Census for Tcf.validate / load_factor (tcf.py:196-249) without copying the
 * table to the host.  Synchronous; out4 (HOST) = live main slots, main slots
 * with a reserved tag, live backing slots, backing slots with a reserved tag. */
int fk_tcf_census(const fk_tcf_geom *g, const void *blocks, const void *backing, int64_t *out4, void *stream);

/* ---- bulk TCF (sorted, front-packed blocks) ----------------------------- */

/* Geometry, derived on the host exactly as BulkTcfParams (tcf_bulk.py:43-77).
 * slot_bytes is the smallest of {1,2,4} holding tag_bits (tcf_bulk.py:80-84);
 * block_slots <= 8192 (one block is staged in shared memory). */
typedef struct fk_btcf_geom {
    int64_t num_blocks;
    int64_t backing_slots;
    int32_t block_slots;
    int32_t tag_bits;
    int32_t slot_bytes;
    int32_t cut_slots;
    int32_t probe_limit;
    int32_t reserved;
    uint64_t seed;
} fk_btcf_geom;

/* Sorted-block invariants of BulkTcf.validate (tcf_bulk.py:354-374) on the
 * device.  Synchronous; out8 (HOST): [0] bitmask (1 fill over capacity,
 * 2 reserved word in a live prefix, 4 unsorted prefix, 8 non-empty tail),
 * [1..4] first offending block per check, [5] sum of fill, [6] live backing
 * slots. */
int fk_btcf_validate(const fk_btcf_geom *g, const void *blocks, const uint32_t *fill, const void *backing,
                     int64_t *out8, void *stream);

/* replaces BulkTcf.insert_batch's kernel sequence (tcf_bulk.py:179-257):
 * _partition_fps + btcf_merge_lists (shortcut) + btcf_route + btcf_merge_lists
 * (dest-grouped) + backing_insert_batch.  `fill` is the device u32[nb] fill
 * array.  failed_keys (device u64[n]) receives the keys the backing table
 * could not take, in the reference's order; *n_failed (device int64) their
 * count.  counters (device int64[3]) += inserts_ok, inserts_backing.
 * status (device u32, caller sets 0xFFFFFFFF) receives 1 + the lowest block a
 * merge would overfill (the reference's AssertionError).  Synchronises the
 * stream twice (batch-dependent sizes); scratch is stream-ordered
 * cudaMallocAsync memory released before return. */
int fk_btcf_insert(const fk_btcf_geom *g, void *blocks, uint32_t *fill, void *backing, const uint64_t *keys,
                   int keys_are_fps, int64_t n, uint64_t *failed_keys, int64_t *n_failed, int64_t *counters,
                   uint32_t *status, void *stream);

/* replaces btcf_query_batch (_ckernels.pyx:552-599); asynchronous. */
int fk_btcf_query(const fk_btcf_geom *g, const void *blocks, const uint32_t *fill, const void *backing,
                  const uint64_t *keys, int keys_are_fps, int64_t n, uint8_t *found, void *stream);

/* replaces BulkTcf.delete_batch (tcf_bulk.py:283-325): btcf_delete_blocklocal
 * over primary then secondary blocks, then backing_delete_batch.  removed
 * (device u8[n]) per input key; counters[2] += removed. */
int fk_btcf_delete(const fk_btcf_geom *g, void *blocks, uint32_t *fill, void *backing, const uint64_t *keys,
                   int keys_are_fps, int64_t n, uint8_t *removed, int64_t *counters, void *stream);

/* replaces _partition_fps (tcf_bulk.py:133-143): sorted_keys[i] =
 * (b1 << tag_bits) | word in stable order, order[i] = input position. */
int fk_btcf_partition(const fk_btcf_geom *g, const uint64_t *keys, int keys_are_fps, int64_t n,
                      uint64_t *sorted_keys, uint32_t *order, void *stream);

/* replaces btcf_merge_lists (_ckernels.pyx:379-405) over all blocks: block b
 * merges words (sorted_keys[i] & tag mask) for i in [seg_lo[b], seg_hi[b]). */
int fk_btcf_merge_lists(const fk_btcf_geom *g, void *blocks, uint32_t *fill, const uint64_t *sorted_keys,
                        const uint32_t *seg_lo, const uint32_t *seg_hi, uint32_t *status, void *stream);

/* ---- bulk-TCF kernel contract, one entry per reference function --------
 * The reference's facade (fk/tcf_bulk.py:145-325) calls these on raw arrays;
 * the fused fk_btcf_insert / fk_btcf_delete above run the same steps without
 * the host round trips.  All synchronous (each returns a host count). */

/* replaces btcf_route (_ckernels.pyx:408-444, _pykernels.py:266-287): the
 * sequential two-choice routing of n items in input order against the
 * committed fill (u32[num_blocks], unchanged); dest (device int64[n]) gets
 * the chosen block or -1.  b1s/b2s are device int64[n]. */
int fk_btcf_route(const uint32_t *fill, int64_t num_blocks, int block_slots, const int64_t *b1s, const int64_t *b2s,
                  int64_t n, int64_t *dest, void *stream);

/* replaces btcf_merge_lists (_ckernels.pyx:379-405, _pykernels.py:244-263):
 * for blocks b in [b_lo, b_hi) in ascending order, merge words[starts[b]:
 * ends[b]] (slot_t, sorted) into the sorted prefix; stops at the first block
 * that would overflow.  *status_out (HOST) = 0, or 1 + that block. */
int fk_btcf_merge_words(const fk_btcf_geom *g, void *blocks, uint32_t *fill, const void *words, int64_t n_words,
                        const int64_t *starts, const int64_t *ends, int64_t b_lo, int64_t b_hi, int64_t *status_out,
                        void *stream);

/* replaces btcf_delete_blocklocal (_ckernels.pyx:482-512, _pykernels.py:
 * 315-337): each sorted item k of block b's segment (b in [b_lo, b_hi))
 * removes one stored copy of words[k] from block b; removed[k] (device u8)
 * flags it; *n_removed (HOST) = the number removed. */
int fk_btcf_delete_blocklocal(const fk_btcf_geom *g, void *blocks, uint32_t *fill, const void *words,
                              int64_t n_words, const int64_t *starts, const int64_t *ends, int64_t b_lo, int64_t b_hi,
                              uint8_t *removed, int64_t *n_removed, void *stream);

/* replaces backing_insert_batch (_ckernels.pyx:447-466, _pykernels.py:
 * 290-301): fingerprints in input order into the backing table; codes
 * (device u8[n]) = P_BACKING (2) or P_FULL (3); *n_fail (HOST) = FULL count. */
int fk_backing_insert_batch(const fk_btcf_geom *g, void *backing, const uint64_t *fps, int64_t n, uint8_t *codes,
                            int64_t *n_fail, void *stream);

/* replaces backing_delete_batch (_ckernels.pyx:515-549, _pykernels.py:
 * 340-363): removed (device u8[n]) per fingerprint, input order;
 * *n_removed (HOST) = the number removed. */
int fk_backing_delete_batch(const fk_btcf_geom *g, void *backing, const uint64_t *fps, int64_t n, uint8_t *removed,
                            int64_t *n_removed, void *stream);

/* ---- GQF (counting quotient filter) ------------------------------------- */

/* Geometry, derived on the host exactly as GqfParams (gqf.py:52-95). */
typedef struct fk_gqf_geom {
    int32_t q, r;              /* 2^q logical slots; r in {8,16,32}; q + r <= 64 */
    int64_t phys;              /* 2^q + min(8192, 2^q) */
    int64_t num_regions;       /* ceil(phys / 8192) */
    int64_t quotient_regions;  /* ceil(2^q / 8192) */
    int64_t max_occupied;      /* int(max_load * 2^q) */
    uint64_t seed;
} fk_gqf_geom;

/* One table image (all device pointers).  slots/occupieds/runends/offsets/
 * stats are bit-identical to the reference's _slots/_occupieds/_runends/
 * _offsets/_stats (gqf.py:111-117); spill (one uint32 per 64 quotients) is a
 * derived run index owned by this library. */
typedef struct fk_gqf_tables {
    void *slots;
    uint64_t *occupieds;
    uint64_t *runends;
    int32_t *offsets;
    int64_t *stats;
    uint32_t *spill;
} fk_gqf_tables;

/* Outcome of a mutation (host struct). */
typedef struct fk_gqf_result {
    int32_t code;        /* 0, GQF_LOAD_CAPACITY=1, GQF_SHIFT_BOUND=2 */
    int32_t swapped;     /* 1: the new image is in `next` (canonical rebuild); 0: `cur` was updated in place */
    int64_t fail_index;  /* point inserts: index of the first failing key (gqf_insert_batch's fail_idx) */
    int64_t fail_region; /* bulk inserts: first failing region in even/odd processing order */
    int64_t shifted;     /* shift-work instrumentation (gqf.py:139-142) */
} fk_gqf_result;

#define FK_GQF_INSERT 0
#define FK_GQF_DELETE 1
#define FK_ORDER_POINT 0 /* items in input order (insert_many / delete_many) */
#define FK_ORDER_BULK 1  /* sorted, even/odd regions, descending deletes (gqf.py:293-353) */

/* replaces gqf_count_batch (_ckernels.pyx:1205-1250); asynchronous. */
int fk_gqf_count(const fk_gqf_geom *g, const fk_gqf_tables *t, const uint64_t *keys, int keys_are_fps,
                 int64_t n, uint64_t *counts, void *stream);

/* replaces gqf_find_run (_ckernels.pyx:754-787): se[2i], se[2i+1] = start, end
 * or -1, -1 when the quotient is unoccupied; asynchronous. */
int fk_gqf_find_run(const fk_gqf_geom *g, const fk_gqf_tables *t, const int64_t *quotients, int64_t n,
                    int64_t *se, void *stream);

/* Device enumeration (replaces the host decode loop of
 * Gqf.enumerate_items, gqf.py:403-409): every stored (fingerprint, count)
 * pair in fingerprint order into device arrays of capacity cap.  Synchronous;
 * *count_out (HOST) = number of items; nothing is written when it exceeds
 * cap (call again with a larger buffer). */
int fk_gqf_enumerate(const fk_gqf_geom *g, const fk_gqf_tables *t, uint64_t *fp_out, uint64_t *cnt_out,
                     int64_t cap, int64_t *count_out, void *stream);

/* Structure validation on the device (replaces the host checks of
 * Gqf.validate, gqf.py:430-492, which decode every run in Python), derived
 * from the bit vectors alone by global rank/select.  Synchronous; out (HOST
 * memory, 24 int64) gets: out[0] = bitmask of failed checks (1<<1 occupieds/
 * runends counts differ, 1<<2 quotient beyond logical table, 1<<3 run past
 * physical table, 1<<5 negative run, 1<<7 region hard bound crossed, 1<<8
 * offset != derived, 1<<11 undecodable run, 1<<12 unsorted groups),
 * out[8 + c] = first offending quotient (region for c = 8), out[1] = used
 * slots, out[2] = decoded total, out[3] = decoded distinct, out[4] = non-zero
 * slots inside runs, out[5] = non-zero slots in the table.  The caller
 * compares out[1..3] with _stats and out[4] with out[5]. */
int fk_gqf_validate(const fk_gqf_geom *g, const fk_gqf_tables *t, int64_t *out, void *stream);

/* Rebuild the derived spill index from occupieds/runends (after the host
 * wrote the image); asynchronous. */
int fk_gqf_rebuild_index(const fk_gqf_geom *g, const fk_gqf_tables *t, void *stream);

/* replaces gqf_insert_batch / gqf_delete_batch (_ckernels.pyx:1147-1202,
 * 1253-1296) together with the facade loops around them (gqf.py:169-216,
 * 293-371).  op = FK_GQF_INSERT / FK_GQF_DELETE; order = FK_ORDER_POINT /
 * FK_ORDER_BULK; deltas NULL = 1 (insert) or 2^63 (delete = all copies);
 * found (deletes) receives per-key flags in input order.  Synchronises the
 * stream (the result is returned to the host); allocates stream-ordered
 * scratch with cudaMallocAsync sized to the batch. */
int fk_gqf_apply(const fk_gqf_geom *g, const fk_gqf_tables *cur, const fk_gqf_tables *next,
                 const uint64_t *keys, int keys_are_fps, const uint64_t *deltas, int64_t n, int op, int order,
                 uint8_t *found, fk_gqf_result *result, void *stream);

/* replaces gqf_insert_batch (_ckernels.pyx:1147-1202, _pykernels.py:772-801)
 * exactly: fingerprints (device u64[n]) with deltas (device u64[n]) applied
 * in input order to the image `t` IN PLACE, stopping at the first capacity
 * failure: *code (HOST) = 0 / GQF_LOAD_CAPACITY / GQF_SHIFT_BOUND,
 * *fail_idx (HOST) = the failing item or -1, *shift_out (HOST) += slots
 * moved.  t->spill is rebuilt from the bit vectors first.  Synchronous. */
int fk_gqf_insert_batch(const fk_gqf_geom *g, const fk_gqf_tables *t, const uint64_t *fps, const uint64_t *deltas,
                        int64_t n, int32_t *code, int64_t *fail_idx, int64_t *shift_out, void *stream);

/* replaces gqf_delete_batch (_ckernels.pyx:1253-1296, _pykernels.py:827-847):
 * input order, in place; found (device u8[n]); *shift_out (HOST) += moved. */
int fk_gqf_delete_batch(const fk_gqf_geom *g, const fk_gqf_tables *t, const uint64_t *fps, const uint64_t *deltas,
                        int64_t n, uint8_t *found, int64_t *shift_out, void *stream);

/* ---- inspection on the device ----------------------------- */

/* Gqf.cluster_stats (gqf.py:416-428): out3 (HOST int64[3]) = {number of
 * maximal contiguous used-slot spans, the longest, their total slots} from a
 * global rank/select over the bit vectors.  Synchronous. */
int fk_gqf_cluster_stats(const fk_gqf_geom *g, const fk_gqf_tables *t, int64_t *out3, void *stream);

/* Tcf.items / BulkTcf.items (tcf.py:196-208, tcf_bulk.py:342-352): idx_out
 * (device int64[n]) gets the positions of the live slots among n slot_bytes
 * words in ascending order, *count (device int64) their number.  A slot is
 * live when its word is > TOMBSTONE, or, with fill (bulk TCF blocks of
 * block_slots), when it lies in its block's filled prefix.  Asynchronous. */
int fk_live_slots(const void *slots, int slot_bytes, int64_t n, const uint32_t *fill, int block_slots,
                  int64_t *idx_out, int64_t *count, void *stream);

/* ---- device key generation -------------------------------- */

/* k-mer windows (workloads.py:147-191): seq (device, n bytes) holds the
 * reads' bases with one non-ACGT separator byte between reads; out (device
 * u64[n]) gets the 2-bit packed value (A=0 C=1 G=2 T=3, first base most
 * significant) of every k-window (1 <= k <= 32) made of ACGT bases only, in
 * position order, *count (device int64) their number.  Asynchronous. */
int fk_kmer_windows(const uint8_t *seq, int64_t n, int k, uint64_t *out, int64_t *count, void *stream);

/* numpy's default_rng streams on the device (workloads.py:61-118): the state
 * and increment are the 128-bit values of Generator.bit_generator.state.
 * fk_pcg64_raw: out[i] = output start + i + 1 (= bit_generator.random_raw).
 * fk_bounded_integers: Generator.integers(low, high, n) for high - low <=
 * 2^32 (int64 out, device); *consumed (HOST) = 64-bit outputs used.
 * fk_zipf_bounded: the ranks of workloads.zipf_bounded(rng, s, universe, n)
 * (int64 out, device) given its h_lo / h_hi / squeeze constants (computed
 * on the host as the reference does); *consumed = doubles drawn.
 * fk_mix_offsets: out[i] = mix64(base + offsets[i]) (the zipf keys).
 * fk_shuffle_u64: a device permutation of n keys by a seeded sort (not
 * numpy's Fisher-Yates order).  The first three synchronise. */
int fk_pcg64_raw(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, uint64_t start, int64_t n,
                 uint64_t *out, void *stream);
int fk_bounded_integers(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t low,
                        int64_t high, int64_t n, int64_t *out, int64_t *consumed, void *stream);
int fk_zipf_bounded(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, double s,
                    int64_t universe, int64_t n, double h_lo, double h_hi, double squeeze, int64_t *ranks,
                    int64_t *consumed, void *stream);
int fk_mix_offsets(uint64_t base, const int64_t *offsets, int64_t n, uint64_t *out, void *stream);
int fk_shuffle_u64(const uint64_t *in, int64_t n, uint64_t seed, uint64_t *out, void *stream);

/* ---- hash-prefix sharding (new in this build) -------------- */

/* Stable partition of a key batch by owner shard, owner = bits
 * [shift, shift + log2_shards) of mix64(key ^ seed) (TCF: shift = 64 -
 * log2_shards, the fingerprint's top bits; GQF: shift = q' + r, the top
 * quotient bits).  keys_out/vals_out get the keys (and optional 64-bit values)
 * grouped by owner in input order, perm[i] the input position of output i,
 * counts (device int64[2^log2_shards]) the group sizes.  Asynchronous. */
int fk_shard_partition(const uint64_t *keys, const uint64_t *vals, int64_t n, uint64_t seed, int shift,
                       int log2_shards, uint64_t *keys_out, uint64_t *vals_out, uint32_t *perm, int64_t *counts,
                       void *stream);

/* dst[perm[i]] = src[i] for 1- or 8-byte elements: per-key results that came
 * back from the owners, restored to input order.  Asynchronous. */
int fk_shard_unpermute(const uint32_t *perm, const void *src, int64_t n, int elem_bytes, void *dst, void *stream);

/* Fused exchange over peer memory (CUDA IPC mappings; NVLink / NVSwitch
 * stores between GPUs) -- the data path of the sharded filters without a
 * collective library.  Pointer arrays are DEVICE arrays of G = 2^log2_shards
 * entries; offset arrays are device int64.  Replaces the all-to-all exchange
 * of SURVEY 8(e).
 *
 * fk_shard_partition with keys_out = NULL computes perm and counts only;
 * fk_shard_dispatch writes key perm[i] of owner o (8 bytes, and its 64-bit
 * value if vals) to peer_keys[o][dst_off[o] + i - seg_start[o]].  Every owner's
 * receive buffer thus holds the sources in rank order, each in its input
 * order, so a key's source and position follow from its offset.
 * fk_shard_combine (owner side): received item j of source s (recv_off[s] <=
 * j < recv_off[s+1], recv_off has G+1 entries) sends its result to
 * peer_back[s][back_off[s] + j - recv_off[s]] -- the key's position in the
 * source's owner-grouped order (one contiguous run per owner); the source
 * restores input order with fk_shard_unpermute.
 * fk_shard_signal: after the stream's prior work, stores epoch into
 * peer_flags[o][rank] for every o (system-scope release);
 * fk_shard_wait: the stream waits until flags[s] >= epoch for all s
 * (acquire), trapping after timeout_s instead of hanging.  All asynchronous. */
int fk_shard_dispatch(const uint64_t *keys, const uint64_t *vals, const uint32_t *perm, int64_t n, uint64_t seed,
                      int shift, int log2_shards, const int64_t *seg_start, const int64_t *dst_off,
                      uint64_t *const *peer_keys, uint64_t *const *peer_vals, void *stream);
int fk_shard_combine(const void *res, int64_t m, int elem_bytes, int log2_shards, const int64_t *recv_off,
                     const int64_t *back_off, void *const *peer_back, void *stream);
int fk_shard_signal(uint32_t *const *peer_flags, int log2_shards, uint32_t rank, uint32_t epoch, void *stream);
int fk_shard_wait(const uint32_t *flags, int log2_shards, uint32_t epoch, double timeout_s, void *stream);

/* Whole-allocation device buffers shareable with the other ranks through
 * CUDA IPC (handles are 64 bytes; open the other ranks' handles, not your own). */
int fk_ipc_alloc(int64_t bytes, void **ptr);
int fk_ipc_free(void *ptr);
int fk_ipc_get_handle(void *ptr, void *handle_out);
int fk_ipc_open(const void *handle, void **ptr);
int fk_ipc_close(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* FILTERKIT_B200_H */
