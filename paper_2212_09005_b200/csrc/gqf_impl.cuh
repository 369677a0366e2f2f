// gqf_impl.cuh -- counting quotient filter (GQF) device code for sm_100a.
//
// Table layout is bit-identical to the reference (gqf.py:111-117): r-bit slot
// words, occupieds/runends bit vectors (u64 words), int32 spill offsets per
// 8192-slot region, int64 stats[3].  On top of it the device keeps one
// derived word per 64 quotients, spill[w] = max(0, end of the last run whose
// quotient < 64w  -  64w + 1), which turns the reference's region-local
// rank/select (popcount of up to 128 occupieds words, _ckernels.pyx:669-683)
// into an O(1) lookup: the run of quotient x ends at the R-th runend after
// 64w + spill[w] - 1, R = rank of x inside its occupieds word.
//
// Mutations: the final table of any insert/delete batch is a pure function of
// the (fingerprint -> count) multiset (runs in quotient order,
// groups sorted by remainder, run start = max(quotient, previous end + 1)), so
// a batch is applied by a canonical rebuild: sort+reduce the batch, decode
// the old table into sorted (fp, count) items, merge, encode, place with a
// max-plus scan, write a fresh table.  Batches that could hit the reference's
// capacity errors (LOAD_CAPACITY / SHIFT_BOUND) run the exact sequential
// algorithm on the device instead (gqf_exact_* below), which reproduces the
// reference's partial application and failure index bit for bit.
#pragma once
#include "../../include/filterkit_b200.h"
#include "fk_common.cuh"

namespace fk {

struct GqfDev {
  void *slots;
  uint64_t *occ;
  uint64_t *run;
  int32_t *offs;
  int64_t *stats;
  uint32_t *spill;  // derived: per 64-quotient word
  int64_t phys;
  int q, r;
  int64_t nregions;
  int64_t max_occ;
};

__device__ __forceinline__ int bit_at(const uint64_t *bv, int64_t i) { return (int)((bv[i >> 6] >> (i & 63)) & 1); }

// k-th set bit strictly after pos (k >= 1), scanning below lim; -2 if none.
__device__ __forceinline__ int64_t select_after_dev(const uint64_t *bv, int64_t pos, int64_t k, int64_t lim) {
  int64_t i = pos + 1 < 0 ? 0 : pos + 1;
  while (i < lim) {
    uint64_t w = bv[i >> 6] >> (i & 63);
    int c = __popcll(w);
    if (c >= k) {
      for (;;) {
        if (--k == 0) return i + __ffsll((long long)w) - 1;
        w &= w - 1;
      }
    }
    k -= c;
    i = (i | 63) + 1;
  }
  return -2;
}

// Run interval of an occupied quotient through the spill index; false if the
// quotient is unoccupied.
__device__ __forceinline__ bool find_run_idx(const GqfDev &T, int64_t quot, int64_t *s, int64_t *e) {
  int64_t w = quot >> 6;
  uint64_t ow = T.occ[w];
  int b = (int)(quot & 63);
  if (!((ow >> b) & 1)) return false;
  int R = __popcll(ow & ((2ull << b) - 1));  // inclusive rank in the word (b=63 -> all bits)
  int64_t E = (w << 6) + (int64_t)T.spill[w] - 1;
  int64_t prev = R == 1 ? E : select_after_dev(T.run, E, R - 1, T.phys);
  int64_t end = select_after_dev(T.run, prev, 1, T.phys);
  *s = quot > prev + 1 ? quot : prev + 1;
  *e = end;
  return end >= 0;
}

// Count group at slot i of a run ending at end (countgroups.py:69-102).
template <typename S>
__device__ __forceinline__ bool parse_group_dev(const S *slots, int64_t i, int64_t end, int r, uint64_t *rem,
                                                uint64_t *cnt, int64_t *nx) {
  uint64_t h = slots[i];
  if (h == 0) {
    int64_t j = i;
    while (j <= end && slots[j] == 0) j++;
    *rem = 0;
    *cnt = (uint64_t)(j - i);
    *nx = j;
    return true;
  }
  if (i == end) { *rem = h; *cnt = 1; *nx = i + 1; return true; }
  uint64_t v = slots[i + 1];
  if (v > h) { *rem = h; *cnt = 1; *nx = i + 1; return true; }
  if (v == h) { *rem = h; *cnt = 2; *nx = i + 2; return true; }
  uint64_t base = (1ull << r) - 1, rest = 0, scale = 1;
  int64_t j = i + 2;
  for (;;) {
    if (j > end) return false;
    uint64_t d = slots[j];
    if (d == h) break;
    rest += scale * (d > h ? d - 1 : d);
    scale *= base;
    j++;
  }
  *rem = h;
  *cnt = v + h * rest + 2;
  *nx = j + 1;
  return true;
}

// countgroups.py:54-66
__host__ __device__ __forceinline__ uint64_t enc_len(uint64_t rem, uint64_t count, int r) {
  if (rem == 0 || count <= 2) return count;
  uint64_t base = (1ull << r) - 1, v = (count - 2) / rem, n = 3;
  while (v) { n++; v /= base; }
  return n;
}

// countgroups.py:28-51 (every slot of the group is written)
template <typename S>
__device__ __forceinline__ void enc_write(S *slots, int64_t pos, uint64_t rem, uint64_t count, int r) {
  if (rem == 0) {
    for (uint64_t i = 0; i < count; i++) slots[pos + (int64_t)i] = 0;
    return;
  }
  slots[pos] = (S)rem;
  if (count == 1) return;
  if (count == 2) { slots[pos + 1] = (S)rem; return; }
  uint64_t v = count - 2, base = (1ull << r) - 1;
  slots[pos + 1] = (S)(v % rem);
  v /= rem;
  int64_t i = pos + 2;
  while (v) {
    uint64_t d = v % base;
    v /= base;
    slots[i++] = (S)(d >= rem ? d + 1 : d);
  }
  slots[i] = (S)rem;
}

// ---------------------------------------------------------------------------
// count query (gqf_count_batch, _ckernels.pyx:1205-1250): pure function
// ---------------------------------------------------------------------------
template <typename S>
__global__ void __launch_bounds__(256) k_gqf_count(GqfDev T, const uint64_t *__restrict__ keys, int keys_are_fps,
                                                   uint64_t seed, int64_t n, uint64_t *__restrict__ counts) {
  const S *slots = reinterpret_cast<const S *>(T.slots);
  uint64_t fmask = (T.q + T.r) >= 64 ? ~0ull : ((1ull << (T.q + T.r)) - 1);
  uint64_t rmask = (1ull << T.r) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t fp = (keys_are_fps ? keys[i] : mix64(keys[i] ^ seed)) & fmask;
    int64_t quot = (int64_t)(fp >> T.r);
    uint64_t rem = fp & rmask;
    uint64_t c = 0;
    int64_t s, e;
    if (find_run_idx(T, quot, &s, &e)) {
      for (int64_t p = s; p <= e;) {
        uint64_t h, cnt;
        int64_t nx;
        if (!parse_group_dev<S>(slots, p, e, T.r, &h, &cnt, &nx)) break;
        if (h == rem) { c = cnt; break; }
        if (h > rem) break;
        p = nx;
      }
    }
    counts[i] = c;
  }
}

__global__ void k_gqf_find_run(GqfDev T, const int64_t *__restrict__ quots, int64_t n, int64_t *__restrict__ se) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = -1, e = -1;
    if (!find_run_idx(T, quots[i], &s, &e)) s = e = -1;
    se[2 * i] = s;
    se[2 * i + 1] = e;
  }
}

// ---------------------------------------------------------------------------
// spill index (re)build from the metadata bit vectors (global rank/select)
// ---------------------------------------------------------------------------
__global__ void k_word_popc(const uint64_t *__restrict__ bv, int64_t nw, int64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __popcll(bv[i]);
}

// rank_occ/rank_run: exclusive prefix sums of per-word popcounts (int64).
// nw: quotient words (spill entries); nrun: runend words over the whole
// physical table -- a run of a quotient near the end can end in the padding
__global__ void k_spill_from_ranks(const uint64_t *__restrict__ run, const int64_t *__restrict__ rank_occ,
                                   const int64_t *__restrict__ rank_run, int64_t nw, int64_t nrun,
                                   uint32_t *__restrict__ spill) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t K = rank_occ[w];  // occupied quotients < 64w
    uint32_t s = 0;
    if (K > 0) {
      // word v holding the K-th runend: last v with rank_run[v] < K
      int64_t lo = 0, hi = nrun - 1;
      while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (rank_run[mid] < K) lo = mid; else hi = mid - 1;
      }
      uint64_t word = run[lo];
      int64_t k = K - rank_run[lo];
      while (--k > 0) word &= word - 1;
      int64_t E = (lo << 6) + __ffsll((long long)word) - 1;
      int64_t sp = E - (w << 6) + 1;
      s = sp > 0 ? (uint32_t)sp : 0u;
    }
    spill[w] = s;
  }
}

// ---------------------------------------------------------------------------
// canonical rebuild pipeline
// ---------------------------------------------------------------------------

__global__ void k_hash_fps(const uint64_t *__restrict__ keys, int keys_are_fps, uint64_t seed, uint64_t fmask,
                           int64_t n, uint64_t *__restrict__ fps, uint32_t *__restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    fps[i] = (keys_are_fps ? keys[i] : mix64(keys[i] ^ seed)) & fmask;
    idx[i] = (uint32_t)i;
  }
}

// fingerprints split into a high byte (bits 32..39, when q + r > 32) and
// the low 32 bits, for the split sort of plain inserts
__global__ void k_hash_split(const uint64_t *__restrict__ keys, int keys_are_fps, uint64_t seed, uint64_t fmask,
                             int64_t n, uint8_t *__restrict__ hi, uint32_t *__restrict__ lo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t fp = (keys_are_fps ? keys[i] : mix64(keys[i] ^ seed)) & fmask;
    if (hi) hi[i] = (uint8_t)(fp >> 32);
    lo[i] = (uint32_t)fp;
  }
}

__global__ void k_widen_split(const uint8_t *__restrict__ hi, const uint32_t *__restrict__ lo, int64_t n,
                              uint64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ((uint64_t)(hi ? hi[i] : 0) << 32) | (uint64_t)lo[i];
}

// bounds[v] = first index of value v in the sorted high bytes (v <= nseg)
__global__ void k_u8_bounds(const uint8_t *__restrict__ hs, int64_t n, int nseg, int64_t *__restrict__ bounds) {
  for (int v = threadIdx.x; v <= nseg; v += blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((int)hs[mid] < v) lo = mid + 1; else hi = mid;
    }
    bounds[v] = lo;
  }
}

// ---- cluster statistics (Gqf.cluster_stats, gqf.py:416-428) ----------------
// Position of the k-th (0-based) set bit of x (k < popc(x)), branch-free.
__device__ __forceinline__ int select64(uint64_t x, int k) {
  int pos = 0, c;
  c = __popc((uint32_t)x);
  if (k >= c) { k -= c; x >>= 32; pos += 32; }
  c = __popc((uint32_t)x & 0xffffu);
  if (k >= c) { k -= c; x >>= 16; pos += 16; }
  c = __popc((uint32_t)x & 0xffu);
  if (k >= c) { k -= c; x >>= 8; pos += 8; }
  c = __popc((uint32_t)x & 0xfu);
  if (k >= c) { k -= c; x >>= 4; pos += 4; }
  c = __popc((uint32_t)x & 0x3u);
  if (k >= c) { k -= c; x >>= 2; pos += 2; }
  c = (int)(x & 1u);
  if (k >= c) pos += 1;
  return pos;
}

// Positions of the set bits of a bit vector, word w's at off[w] onward.
// One warp per 32 consecutive words: a warp prefix sum of their popcounts,
// then rounds of 32 consecutive output ranks, each lane locating its rank's
// word by a 5-step search over the lanes' prefixes -- the stores are
// coalesced (one thread per word would scatter them 30 words apart).
__global__ void k_bit_positions(const uint64_t *__restrict__ bv, int64_t nw, const int64_t *__restrict__ off,
                                int64_t *__restrict__ pos) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (nw + 31) >> 5;
  for (int64_t wp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wp < nwarps;
       wp += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t w0 = wp << 5, w = w0 + lane;
    const uint64_t x = w < nw ? bv[w] : 0ull;
    int incl = __popcll(x);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    const int64_t base = off[w0];
    for (int rb = 0; rb < total; rb += 32) {
      const int r = rb + lane;
      // t = the first lane whose inclusive prefix exceeds r
      int t = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, t + step - 1);
        if (v <= r) t += step;
      }
      const int ex = __shfl_sync(0xffffffffu, incl, t) - __popcll(__shfl_sync(0xffffffffu, x, t));
      const uint64_t xt = __shfl_sync(0xffffffffu, x, t);
      if (r < total) pos[base + r] = ((w0 + t) << 6) + select64(xt, r - ex);
    }
  }
}

// Decode by runs: run k (occupied quotient Q[k], ending at the k-th runend
// bit E[k], starting at max(Q[k], E[k-1] + 1)) is parsed by its own thread;
// mode 0 counts its groups, mode 1 writes them at off[k].
template <typename S>
__global__ void k_decode_runs(GqfDev T, const int64_t *__restrict__ Q, const int64_t *__restrict__ E, int64_t K,
                              int mode, int64_t *__restrict__ gcount, const int64_t *__restrict__ off,
                              uint64_t *__restrict__ it_fp, uint64_t *__restrict__ it_cnt, int *__restrict__ err) {
  const S *slots = reinterpret_cast<const S *>(T.slots);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t quot = Q[k], end = E[k];
    const int64_t prev = k ? E[k - 1] : -1;
    const int64_t st = quot > prev + 1 ? quot : prev + 1;
    int64_t o = mode ? off[k] : 0, g = 0;
    if (end < st) {
      *err = 1;
      continue;
    }
    for (int64_t p = st; p <= end;) {
      uint64_t h, cnt;
      int64_t nx;
      if (!parse_group_dev<S>(slots, p, end, T.r, &h, &cnt, &nx)) {
        *err = 1;
        break;
      }
      if (mode) {
        it_fp[o] = ((uint64_t)quot << T.r) | h;
        it_cnt[o] = cnt;
        o++;
      }
      g++;
      p = nx;
    }
    if (!mode) gcount[k] = g;
  }
}

// Run k = occupied quotient Q[k] ending at E[k] (the k-th runend bit),
// starting at max(Q[k], E[k-1] + 1); a cluster starts where Q[k] > E[k-1] + 1.
// brk[k] = 1 at cluster starts, len[k] = run length.
__global__ void k_run_clusters(const int64_t *__restrict__ Q, const int64_t *__restrict__ E, int64_t K,
                               int64_t *__restrict__ brk, int64_t *__restrict__ len) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pe = k ? E[k - 1] : -2;
    const bool b = k == 0 || Q[k] > pe + 1;
    const int64_t start = b ? Q[k] : pe + 1;
    brk[k] = b ? 1 : 0;
    len[k] = E[k] - start + 1;
  }
}

// ---- partitioned counting of plain counted inserts -------------------------
// Counting the occurrences of a batch (insert of every occurrence, no delta
// array) is a group-by on the fingerprint.  Instead of sorting every
// occurrence on all q + r bits and run-length encoding the result:
//   1. two MSD partition passes (kPartBits each) scatter the hashed
//      occurrences by their top 2 * kPartBits fingerprint bits; a CTA stages a
//      tile in shared memory grouped by digit (unstable ranks: order inside a
//      partition does not matter), reserves one contiguous range per digit
//      with one global atomic, and writes the groups out coalesced;
//   2. one CTA per partition aggregates its low W bits in a shared-memory
//      hash table, sorts only the distinct fingerprints (bitonic), and writes
//      (fingerprint, count) runs; a compaction pass packs the partitions.
// Partitions whose distinct fingerprints overflow the table set a flag and
// the caller recounts the batch on the full-sort path.
constexpr int kPartBits = 9;
constexpr int kPartBins = 1 << kPartBits;
constexpr int kPartThreads = 512;
constexpr int kPartItems = 8;                          // per thread: 4 K occurrences per tile
constexpr int kPartTile = kPartThreads * kPartItems;
constexpr int kAggThreads = 256;
constexpr int kAggSlots = 4096;                        // hash table entries per partition CTA

__device__ __forceinline__ uint64_t part_fp(const uint64_t *keys, int keys_are_fps, uint64_t seed, uint64_t fmask,
                                            int64_t i) {
  const uint64_t k = __ldcs(keys + i);
  return (keys_are_fps ? k : mix64(k ^ seed)) & fmask;
}

// Pass-1 histogram: digit = fingerprint bits [qr - kPartBits, qr).
__global__ void __launch_bounds__(kPartThreads) k_part1_hist(const uint64_t *__restrict__ keys, int keys_are_fps,
                                                             uint64_t seed, uint64_t fmask, int qr, int64_t n,
                                                             unsigned long long *__restrict__ hist) {
  __shared__ unsigned sh[kPartBins];
  for (int i = threadIdx.x; i < kPartBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&sh[part_fp(keys, keys_are_fps, seed, fmask, i) >> (qr - kPartBits)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kPartBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// Tile scatter shared by both passes: every thread holds kPartItems
// (digit, value) pairs; the tile is regrouped by digit in shared memory and
// each digit's group is written to cursor[digit] (reserved with one atomic).
__device__ __forceinline__ void part_scatter_tile(const uint32_t (&dg)[kPartItems], const uint32_t (&val)[kPartItems],
                                                  const bool (&ok)[kPartItems], unsigned long long *cursor,
                                                  uint32_t *out, unsigned *s_cnt, unsigned *s_off,
                                                  unsigned long long *s_base, uint32_t *s_val, uint16_t *s_dg) {
  for (int i = threadIdx.x; i < kPartBins; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  unsigned rk[kPartItems];
#pragma unroll
  for (int j = 0; j < kPartItems; j++) rk[j] = ok[j] ? atomicAdd(&s_cnt[dg[j]], 1u) : 0u;
  __syncthreads();
  // exclusive offsets of the digit groups inside the tile (512 bins, one
  // thread each) and one global reservation per non-empty digit
  {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ unsigned s_w[kPartThreads / 32];
    const unsigned v = threadIdx.x < kPartBins ? s_cnt[threadIdx.x] : 0u;
    unsigned inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if ((int)lane >= o) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    unsigned base = inc - v;
    for (int w = 0; w < (int)warp; w++) base += s_w[w];
    if (threadIdx.x < kPartBins) {
      s_off[threadIdx.x] = base;
      s_base[threadIdx.x] = v ? atomicAdd(&cursor[threadIdx.x], (unsigned long long)v) : 0ull;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kPartItems; j++)
    if (ok[j]) {
      const unsigned pos = s_off[dg[j]] + rk[j];
      s_val[pos] = val[j];
      s_dg[pos] = (uint16_t)dg[j];
    }
  __syncthreads();
  const unsigned tot = s_off[kPartBins - 1] + s_cnt[kPartBins - 1];
  for (unsigned pos = threadIdx.x; pos < tot; pos += blockDim.x) {
    const unsigned d = s_dg[pos];
    out[s_base[d] + (pos - s_off[d])] = s_val[pos];
  }
  __syncthreads();
}

// Pass 1: hash every occurrence, keep its low qr - kPartBits bits (u32) and
// scatter by the top kPartBits.  cursor[d] starts at the digit's offset.
// dynamic shared memory of the scatter kernels: tile values, digits, and the
// per-digit counters / offsets / reserved bases
constexpr size_t kPartSmem = (size_t)kPartTile * 6 + (size_t)kPartBins * 16;
struct PartSmem {
  unsigned long long *base;
  unsigned *cnt, *off;
  uint32_t *val;
  uint16_t *dg;
  __device__ explicit PartSmem(unsigned char *p) {
    base = reinterpret_cast<unsigned long long *>(p);
    cnt = reinterpret_cast<unsigned *>(p + kPartBins * 8);
    off = cnt + kPartBins;
    val = reinterpret_cast<uint32_t *>(p + kPartBins * 16);
    dg = reinterpret_cast<uint16_t *>(p + kPartBins * 16 + (size_t)kPartTile * 4);
  }
};

#ifndef FK_PART_MINB
#define FK_PART_MINB 2
#endif
__global__ void __launch_bounds__(kPartThreads, FK_PART_MINB) k_part1_scatter(const uint64_t *__restrict__ keys,
                                                                              int keys_are_fps, uint64_t seed,
                                                                              uint64_t fmask, int qr, int64_t n,
                                                                              unsigned long long *__restrict__ cursor,
                                                                              uint32_t *__restrict__ out) {
  extern __shared__ __align__(16) unsigned char part_sm[];
  PartSmem P(part_sm);
  const int sh = qr - kPartBits;
  const uint64_t lmask = (1ull << sh) - 1;
  const int64_t step = (int64_t)gridDim.x * kPartTile;
  // the next tile's keys are loaded while this tile is scattered
  uint64_t kr[kPartItems];
#pragma unroll
  for (int j = 0; j < kPartItems; j++) {
    const int64_t i = (int64_t)blockIdx.x * kPartTile + (int64_t)j * kPartThreads + threadIdx.x;
    kr[j] = i < n ? __ldcs(keys + i) : 0ull;
  }
  for (int64_t t0 = (int64_t)blockIdx.x * kPartTile; t0 < n; t0 += step) {
    uint32_t dg[kPartItems], val[kPartItems];
    bool ok[kPartItems];
#pragma unroll
    for (int j = 0; j < kPartItems; j++) {
      const int64_t i = t0 + (int64_t)j * kPartThreads + threadIdx.x;
      ok[j] = i < n;
      const uint64_t fp = (keys_are_fps ? kr[j] : mix64(kr[j] ^ seed)) & fmask;
      dg[j] = (uint32_t)(fp >> sh);
      val[j] = (uint32_t)(fp & lmask);
      const int64_t i2 = i + step;
      kr[j] = i2 < n ? __ldcs(keys + i2) : 0ull;
    }
    part_scatter_tile(dg, val, ok, cursor, out, P.cnt, P.off, P.base, P.val, P.dg);
  }
}

// Pass-2 histogram over the pass-1 output: partition p = (d1 << kPartBits) | d2
// with d1 from the item's position (bounds1) and d2 = bits [sh2, sh2 + kPartBits)
// of the stored value.
// tile t of pass 2 -> its pass-1 digit d1 (tile_start[d1] = d1's first tile)
__device__ __forceinline__ int part_tile_digit(const unsigned long long *tile_start, int64_t t) {
  int lo = 0, hi = kPartBins;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tile_start[mid] <= (unsigned long long)t) lo = mid; else hi = mid;
  }
  return lo;
}

// Pass-2 histogram, per pass-1 digit and tile (the scatter's tiling), so the
// global counters take one atomic per (tile, digit).
__global__ void __launch_bounds__(kPartThreads) k_part2_hist(const uint32_t *__restrict__ in,
                                                             const unsigned long long *__restrict__ bounds1,
                                                             const unsigned long long *__restrict__ tile_start,
                                                             int sh2, int p2, unsigned long long *__restrict__ hist) {
  __shared__ unsigned sh[kPartBins];
  const int64_t ntiles = (int64_t)tile_start[kPartBins];
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < kPartBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int d1 = part_tile_digit(tile_start, t);
    const int64_t a = (int64_t)bounds1[d1] + (t - (int64_t)tile_start[d1]) * kPartTile;
    int64_t e = (int64_t)bounds1[d1 + 1];
    if (e > a + kPartTile) e = a + kPartTile;
    for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&sh[(__ldcs(in + i) >> sh2) & ((1u << p2) - 1)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < (1 << p2); i += blockDim.x)
      if (sh[i]) atomicAdd(&hist[((uint64_t)d1 << p2) | i], (unsigned long long)sh[i]);
    __syncthreads();
  }
}

// bounds1 / cursor1 (exclusive sums of the 512 pass-1 counts) and every
// digit's first pass-2 tile; tile_start[kPartBins] = the number of tiles
__global__ void __launch_bounds__(kPartBins) k_part_plan1(const unsigned long long *__restrict__ hist1,
                                                          unsigned long long *__restrict__ bounds1,
                                                          unsigned long long *__restrict__ cursor1,
                                                          unsigned long long *__restrict__ tile_start) {
  __shared__ unsigned long long sw[kPartBins / 32][2];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long c = hist1[threadIdx.x];
  const unsigned long long nt = (c + kPartTile - 1) / kPartTile;
  unsigned long long ic = c, it = nt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long a = __shfl_up_sync(0xFFFFFFFFu, ic, o), b = __shfl_up_sync(0xFFFFFFFFu, it, o);
    if ((int)lane >= o) {
      ic += a;
      it += b;
    }
  }
  if (lane == 31) {
    sw[warp][0] = ic;
    sw[warp][1] = it;
  }
  __syncthreads();
  unsigned long long bc = ic - c, bt = it - nt;
  for (int w = 0; w < (int)warp; w++) {
    bc += sw[w][0];
    bt += sw[w][1];
  }
  bounds1[threadIdx.x] = bc;
  cursor1[threadIdx.x] = bc;
  tile_start[threadIdx.x] = bt;
  if (threadIdx.x == kPartBins - 1) {
    bounds1[kPartBins] = bc + c;
    tile_start[kPartBins] = bt + nt;
  }
}

// Pass 2: tiles never straddle a pass-1 digit (grid-stride over
// (digit, tile) pairs), so the partition is d1 << kPartBits | d2 and the
// scatter keeps the low sh2 bits.
__global__ void __launch_bounds__(kPartThreads, FK_PART_MINB) k_part2_scatter(const uint32_t *__restrict__ in,
                                                                              const unsigned long long *__restrict__ bounds1,
                                                                              const unsigned long long *__restrict__ tile_start,
                                                                              int sh2, int p2,
                                                                              unsigned long long *__restrict__ cursor,
                                                                              uint32_t *__restrict__ out) {
  extern __shared__ __align__(16) unsigned char part_sm[];
  PartSmem P(part_sm);
  __shared__ unsigned long long s_ts[kPartBins + 1], s_b1[kPartBins + 1];
  for (int i = threadIdx.x; i <= kPartBins; i += blockDim.x) {
    s_ts[i] = tile_start[i];
    s_b1[i] = bounds1[i];
  }
  __syncthreads();
  const uint32_t lmask = sh2 >= 32 ? 0xFFFFFFFFu : ((1u << sh2) - 1u);
  const int64_t ntiles = (int64_t)s_ts[kPartBins];
  // the next tile's values are loaded while this tile is scattered
  int64_t t = blockIdx.x;
  int d1 = t < ntiles ? part_tile_digit(s_ts, t) : 0;
  int64_t a = t < ntiles ? (int64_t)s_b1[d1] + (t - (int64_t)s_ts[d1]) * kPartTile : 0;
  int64_t e = t < ntiles ? (int64_t)s_b1[d1 + 1] : 0;
  uint32_t vr[kPartItems];
#pragma unroll
  for (int j = 0; j < kPartItems; j++) {
    const int64_t i = a + (int64_t)j * kPartThreads + threadIdx.x;
    vr[j] = i < e ? __ldcs(in + i) : 0u;
  }
  for (; t < ntiles; t += gridDim.x) {
    const int64_t t2 = t + gridDim.x;
    const int d1n = t2 < ntiles ? part_tile_digit(s_ts, t2) : 0;
    const int64_t an = t2 < ntiles ? (int64_t)s_b1[d1n] + (t2 - (int64_t)s_ts[d1n]) * kPartTile : 0;
    const int64_t en = t2 < ntiles ? (int64_t)s_b1[d1n + 1] : 0;
    uint32_t dg[kPartItems], val[kPartItems];
    bool ok[kPartItems];
#pragma unroll
    for (int j = 0; j < kPartItems; j++) {
      const int64_t i = a + (int64_t)j * kPartThreads + threadIdx.x;
      ok[j] = i < e;
      const uint32_t v = vr[j];
      dg[j] = (v >> sh2) & ((1u << p2) - 1);
      val[j] = v & lmask;
      const int64_t i2 = an + (int64_t)j * kPartThreads + threadIdx.x;
      vr[j] = i2 < en ? __ldcs(in + i2) : 0u;
    }
    part_scatter_tile(dg, val, ok, cursor + ((uint64_t)d1 << p2), out, P.cnt, P.off, P.base, P.val, P.dg);
    d1 = d1n;
    a = an;
    e = en;
  }
}

// One CTA per partition: hash-aggregate the low W bits, order the distinct
// ones, write (fp, count) at the partition's own offset.
// The hash is order-preserving (home slot = the key's top lg_slots bits) with
// linear probing that never wraps (kAggPad overflow slots), so the table read
// in slot order is sorted except inside clusters of occupied slots: a key's
// home lies in its own cluster and homes grow with the keys.  An in-order
// compaction plus odd-even transposition rounds (a few: clusters are short at
// the ~11 % load of a 3 K-occurrence partition) sort it; more than
// kAggOddEvenMax rounds (skewed keys, dense tables) falls back to a bitonic
// sort.
constexpr int kAggPad = 256;
constexpr int kAggOddEvenMax = 32;
__global__ void __launch_bounds__(kAggThreads) k_part_aggregate(const uint32_t *__restrict__ in,
                                                                const unsigned long long *__restrict__ bounds2,
                                                                int64_t NP, int W, uint64_t *__restrict__ out_fp,
                                                                uint32_t *__restrict__ out_cnt,
                                                                int64_t *__restrict__ ucount,
                                                                unsigned *__restrict__ overflow, int lg_slots) {
  constexpr int kTab = kAggSlots + kAggPad;
  __shared__ uint64_t tab[kTab];  // keys | counts while counting, then ordered (key << 32 | count) words
  __shared__ unsigned s_n, s_bad, s_cnt[kAggThreads / 32];
  uint32_t *hk = reinterpret_cast<uint32_t *>(tab), *hc = hk + kTab;
  constexpr uint32_t kEmpty = 0xFFFFFFFFu;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t p = blockIdx.x; p < NP; p += gridDim.x) {
    const int64_t a = (int64_t)bounds2[p], e = (int64_t)bounds2[p + 1];
    if (a == e) {
      if (threadIdx.x == 0) ucount[p] = 0;
      continue;
    }
    const uint32_t limit = (1u << lg_slots) + kAggPad;  // probe bound (lg_slots < 12 only in overflow tests)
    for (int i = threadIdx.x; i < kTab; i += kAggThreads) {
      hk[i] = kEmpty;
      hc[i] = 0;
    }
    if (threadIdx.x == 0) {
      s_n = 0;
      s_bad = 0;
    }
    __syncthreads();
    for (int64_t i0 = a; i0 < e; i0 += kAggThreads * 8) {
      uint32_t v[8];  // eight loads in flight before the table updates
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int64_t i = i0 + u * kAggThreads + threadIdx.x;
        v[u] = i < e ? __ldcs(in + i) : kEmpty;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t k = v[u];
        if (k == kEmpty) continue;  // (keys have W <= 31 bits)
        uint32_t h = W >= lg_slots ? k >> (W - lg_slots) : k << (lg_slots - W);
        for (;;) {
          // plain read first: most occurrences find their key already there
          // and need one shared-memory atomic, not two
          uint32_t old = *(volatile uint32_t *)&hk[h];
          if (old == kEmpty) old = atomicCAS(&hk[h], kEmpty, k);
          if (old == kEmpty || old == k) {
            atomicAdd(&hc[h], 1u);
            break;
          }
          if (++h == limit) {
            s_bad = 1;
            break;
          }
        }
      }
    }
    __syncthreads();
    if (s_bad) {
      if (threadIdx.x == 0) {
        ucount[p] = -1;
        atomicOr(overflow, 1u);
      }
      __syncthreads();
      continue;
    }
    // in-order compaction: thread t owns slots [t*R, (t+1)*R)
    constexpr int R = (kTab + kAggThreads - 1) / kAggThreads;
    uint64_t mine[R];
    int nm = 0;
#pragma unroll
    for (int j = 0; j < R; j++) {
      const int i = threadIdx.x * R + j;
      if (i < kTab && hk[i] != kEmpty) mine[nm++] = ((uint64_t)hk[i] << 32) | hc[i];
    }
    unsigned inc = nm;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if ((int)lane >= o) inc += t;
    }
    if (lane == 31) s_cnt[warp] = inc;
    __syncthreads();  // (also: every thread has read the table)
    unsigned base = inc - nm;
    for (unsigned w = 0; w < warp; w++) base += s_cnt[w];
    unsigned d = 0;
    for (unsigned w = 0; w < kAggThreads / 32; w++) d += s_cnt[w];
    uint64_t *kv = tab;
    for (int j = 0; j < nm; j++) kv[base + j] = mine[j];
    __syncthreads();
    // odd-even transposition rounds until no pair moves
    bool sorted = false;
    for (int r = 0; r < kAggOddEvenMax; r++) {
      bool moved = false;
      for (unsigned i = 2 * threadIdx.x + (r & 1); i + 1 < d; i += 2 * kAggThreads) {
        const uint64_t x = kv[i], y = kv[i + 1];
        if (x > y) {
          kv[i] = y;
          kv[i + 1] = x;
          moved = true;
        }
      }
      const bool any = __syncthreads_or(moved);
      if (!any && r > 0) {
        sorted = true;
        break;
      }
    }
    if (!sorted) {
      unsigned m2 = 1;
      while (m2 < d) m2 <<= 1;
      for (unsigned i = d + threadIdx.x; i < m2; i += kAggThreads) kv[i] = ~0ull;  // pads sort last
      __syncthreads();
      // bitonic sort; stages whose partner distance is below 64 stay inside a
      // warp's own 64-element chunks (no block barrier), the rest sync the CTA
      constexpr unsigned NW = kAggThreads / 32;
      for (unsigned k2 = 2; k2 <= m2; k2 <<= 1) {
        for (unsigned j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
          const unsigned lj = __ffs(j2) - 1;  // j2 is a power of two: shifts, not divisions
          if (j2 >= 64) {
            for (unsigned q = threadIdx.x; q < m2 / 2; q += kAggThreads) {
              const unsigned i = ((q >> lj) << (lj + 1)) | (q & (j2 - 1)), l = i + j2;
              const uint64_t x = kv[i], y = kv[l];
              if ((x > y) == ((i & k2) == 0)) {
                kv[i] = y;
                kv[l] = x;
              }
            }
            __syncthreads();
          } else {
            const unsigned span = m2 < 64 ? m2 : 64;
            for (unsigned c = warp; c * span < m2; c += NW) {
              if (lane < span / 2) {
                const unsigned i = c * span + (((lane >> lj) << (lj + 1)) | (lane & (j2 - 1))), l = i + j2;
                const uint64_t x = kv[i], y = kv[l];
                if ((x > y) == ((i & k2) == 0)) {
                  kv[i] = y;
                  kv[l] = x;
                }
              }
            }
            __syncwarp();
          }
        }
        __syncthreads();
      }
    }
    for (unsigned j = threadIdx.x; j < d; j += kAggThreads) {
      const uint64_t v = kv[j];
      out_fp[a + j] = ((uint64_t)p << W) | (v >> 32);
      out_cnt[a + j] = (uint32_t)v;
    }
    if (threadIdx.x == 0) ucount[p] = d;
    __syncthreads();
  }
}

// uniq / sums = the partitions' runs, compacted (one warp per partition)
__global__ void k_part_compact(const uint64_t *__restrict__ out_fp, const uint32_t *__restrict__ out_cnt,
                               const unsigned long long *__restrict__ bounds2, const int64_t *__restrict__ ucount,
                               const int64_t *__restrict__ uoff, int64_t NP, uint64_t *__restrict__ uniq,
                               uint64_t *__restrict__ sums) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const unsigned lane = threadIdx.x & 31;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < NP; p += warps) {
    const int64_t s = (int64_t)bounds2[p], d = uoff[p], U = ucount[p];
    for (int64_t j = lane; j < U; j += 32) {
      uniq[d + j] = out_fp[s + j];
      sums[d + j] = out_cnt[s + j];
    }
  }
}

__global__ void k_gather_u64(const uint64_t *__restrict__ src, const uint32_t *__restrict__ idx,
                             uint64_t dflt, int64_t n, uint64_t *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src ? src[idx[i]] : dflt;
}

// new absolute count per unique fp: insert c+sum, delete c-min(c,sum)
__global__ void k_new_counts(const uint64_t *__restrict__ c_old, const uint64_t *__restrict__ sums, int64_t m,
                             int is_delete, uint64_t *__restrict__ c_new) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c = c_old[i], s = sums[i];
    if (is_delete) c_new[i] = c > s ? c - s : 0;
    else { uint64_t t = c + s; c_new[i] = t < c ? ~0ull : t; }
  }
}

// found flags of a duplicate-free delete batch, in sorted order: a key is
// found iff its fingerprint was present
__global__ void k_found_distinct(const uint64_t *__restrict__ c_old, int64_t n, uint8_t *__restrict__ found_s) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    found_s[j] = c_old[j] > 0 ? 1 : 0;
}

// found_s (sorted order) -> found (input order) in passes over input-index
// ranges of 2^shift keys: the pass's byte stores land in a range that stays
// in L2 until its sectors are complete (one random byte store per key
// across the whole array costs a DRAM sector write each)
__global__ void k_found_scatter(const uint8_t *__restrict__ found_s, const uint32_t *__restrict__ idx_s, int64_t n,
                                int shift, int64_t pass, uint8_t *__restrict__ found) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = idx_s[j];
    if ((int64_t)(i >> shift) == pass) found[i] = found_s[j];
  }
}

// 1 where a sorted fingerprint starts a new segment, after the first item
// (so the exclusive sum of heads is the item's segment index)
__global__ void k_seg_heads(const uint64_t *__restrict__ fps_s, int64_t n, int64_t *__restrict__ heads) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    heads[j] = (j + 1 < n && fps_s[j + 1] != fps_s[j]) ? 1 : 0;
}

// Unique fingerprints and saturating delta sums of the sorted batch, one
// thread per fingerprint segment (seg = exclusive sum of k_seg_heads).
__global__ void k_seg_reduce(const uint64_t *__restrict__ fps_s, const uint64_t *__restrict__ del_s,
                             const int64_t *__restrict__ seg, int64_t n, uint64_t *__restrict__ uniq,
                             uint64_t *__restrict__ sums) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t f = fps_s[j];
    if (j > 0 && fps_s[j - 1] == f) continue;  // not a segment head
    uint64_t acc = del_s[j];
    for (int64_t e = j + 1; e < n && fps_s[e] == f; e++) {
      const uint64_t sum = acc + del_s[e];
      acc = sum < acc ? ~0ull : sum;
    }
    const int64_t s = seg[j];
    uniq[s] = f;
    sums[s] = acc;
  }
}

// found flags of a delete batch with repeated fingerprints, one thread per
// fingerprint segment of the sorted batch (segments are short): the copies
// are processed in the facade's order -- input order for point deletes,
// last-input-first for bulk deletes (gqf.py:317-325) -- and copy k finds the
// key iff the deltas of the copies before it leave part of the old count.
// Written in sorted order (k_found_scatter brings them to input order).
__global__ void k_found_walk(const uint64_t *__restrict__ fps_s, const uint64_t *__restrict__ del_s,
                             const int64_t *__restrict__ seg,
                             const uint64_t *__restrict__ c_old, int64_t n, int bulk_order,
                             uint8_t *__restrict__ found_s) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t f = fps_s[j];
    if (j > 0 && fps_s[j - 1] == f) continue;  // not a segment head
    int64_t e = j + 1;
    while (e < n && fps_s[e] == f) e++;
    const uint64_t c = c_old[seg[j]];
    uint64_t pre = 0;
    for (int64_t t = 0; t < e - j; t++) {
      const int64_t k = bulk_order ? e - 1 - t : j + t;
      found_s[k] = pre < c ? 1 : 0;
      const uint64_t d = del_s[k], sum = pre + d;
      pre = sum < pre ? ~0ull : sum;  // saturating, as the reference's counts
    }
  }
}

// First index >= lo with a[index] >= f (a sorted, a[lo - 1] < f): galloping
// steps then a binary search, O(log gap).
__device__ __forceinline__ int64_t gallop_lower(const uint64_t *__restrict__ a, int64_t n, int64_t lo, uint64_t f) {
  int64_t step = 1, hi = lo;
  while (hi < n && a[hi] < f) {
    lo = hi + 1;
    hi += step;
    step <<= 1;
  }
  if (hi > n) hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < f) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// lower_bound of f in a[0..n) by one warp (f warp-uniform): 32-way probes,
// ~log32(n) dependent loads instead of log2(n).
__device__ __forceinline__ int64_t warp_lower_bound(const uint64_t *__restrict__ a, int64_t n, uint64_t f) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int64_t p = lo + (hi - lo) * (lane + 1) / 33;
    const unsigned b = __ballot_sync(0xffffffffu, a[p] < f);
    const int k = __popc(b);
    const int64_t nlo = k ? __shfl_sync(0xffffffffu, p, k - 1) + 1 : lo;
    const int64_t nhi = k < 32 ? __shfl_sync(0xffffffffu, p, k < 32 ? k : 31) : hi;
    lo = nlo;
    hi = nhi;
  }
  const unsigned b = __ballot_sync(0xffffffffu, lo + lane < hi && a[lo + lane] < f);
  return lo + __popc(b);
}

// Join of sorted `probe` (np items) against sorted `a` (na items), one warp
// per chunk of kJoinChunk probes: a warp lower_bound for the chunk's first
// probe, then rounds of 32 consecutive probes against the 32 items of `a`
// after the previous round's last position (coalesced probe reads, window
// reads and result writes); a probe past the window gallops on.
constexpr int kJoinChunk = 1024;
template <typename F>
__device__ __forceinline__ void warp_join(const uint64_t *__restrict__ probe, int64_t np,
                                          const uint64_t *__restrict__ a, int64_t na, F &&emit) {
  const int lane = threadIdx.x & 31;
  const int64_t nch = (np + kJoinChunk - 1) / kJoinChunk;
  for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nch;
       c += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s = c * kJoinChunk, e = s + kJoinChunk < np ? s + kJoinChunk : np;
    int64_t lo = warp_lower_bound(a, na, probe[s]);
    for (int64_t b = s; b < e; b += 32) {
      const int64_t j = b + lane;
      const bool v = j < e;
      const uint64_t f = v ? probe[j] : ~0ull;
      // the next 32 items of a, one coalesced load; each lane's position in
      // that window by a 5-step search over the lanes, galloping on past it
      const uint64_t wa = lo + lane < na ? a[lo + lane] : ~0ull;
      int c = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint64_t at = __shfl_sync(0xffffffffu, wa, c + step - 1);
        if (at < f) c += step;
      }
      if (__shfl_sync(0xffffffffu, wa, 31) < f && c == 31) c = 32;
      int64_t p = lo + c;
      if (v && c == 32) p = gallop_lower(a, na, p, f);
      if (v) emit(j, p, p < na && a[p] == f);
      const int last = (e - b) < 32 ? (int)(e - b) - 1 : 31;
      lo = __shfl_sync(0xffffffffu, p, last);
    }
  }
}

// Old items the batch updates are dropped before the merge.
__global__ void k_keep_old_join(const uint64_t *__restrict__ o_fp, int64_t g_old, const uint64_t *__restrict__ uniq,
                                int64_t m, uint8_t *__restrict__ keep) {
  warp_join(o_fp, g_old, uniq, m, [&](int64_t i, int64_t, bool hit) { keep[i] = hit ? 0 : 1; });
}

// The old count of every batch fingerprint from the decoded table (replaces
// the count query when the whole table is decoded anyway) and its new count
// (as k_new_counts).
__global__ void k_old_counts_join(const uint64_t *__restrict__ uniq, int64_t m, const uint64_t *__restrict__ o_fp,
                                  const uint64_t *__restrict__ o_cnt, int64_t g_old, const uint64_t *__restrict__ sums,
                                  int is_delete, uint64_t *__restrict__ c_old, uint64_t *__restrict__ c_new) {
  warp_join(uniq, m, o_fp, g_old, [&](int64_t j, int64_t p, bool hit) {
    const uint64_t c = hit ? o_cnt[p] : 0, s = sums[j];
    c_old[j] = c;
    if (is_delete) {
      c_new[j] = c > s ? c - s : 0;
    } else {
      const uint64_t t = c + s;
      c_new[j] = t < c ? ~0ull : t;
    }
  });
}

// Decode pass over occupied quotient words: mode 0 counts groups per word,
// mode 1 writes (fp, count) items at off[w].
// Groups of quotient word w (mode 0: their number; mode 1: write them at o).
template <typename S>
__device__ __forceinline__ int64_t decode_word(const GqfDev &T, int64_t w, int mode, int64_t o,
                                               uint64_t *__restrict__ it_fp, uint64_t *__restrict__ it_cnt,
                                               int *__restrict__ err) {
  const S *slots = reinterpret_cast<const S *>(T.slots);
  uint64_t ow = T.occ[w];
  int64_t g = 0;
  if (ow) {
    int64_t prev = (w << 6) + (int64_t)T.spill[w] - 1;
    while (ow) {
      int b = __ffsll((long long)ow) - 1;
      ow &= ow - 1;
      int64_t quot = (w << 6) + b;
      int64_t end = select_after_dev(T.run, prev, 1, T.phys);
      if (end < 0) { *err = 1; break; }
      int64_t s = quot > prev + 1 ? quot : prev + 1;
      for (int64_t p = s; p <= end;) {
        uint64_t h, cnt;
        int64_t nx;
        if (!parse_group_dev<S>(slots, p, end, T.r, &h, &cnt, &nx)) { *err = 1; break; }
        if (mode) {
          it_fp[o] = ((uint64_t)quot << T.r) | h;
          it_cnt[o] = cnt;
          o++;
        }
        g++;
        p = nx;
      }
      prev = end;
    }
  }
  return g;
}

// decode_word over the quotient words of a list of regions (creg[0..K)):
// flat index f -> region creg[f / 128], word f % 128 of it.
template <typename S>
__global__ void k_decode_region_words(GqfDev T, const int64_t *__restrict__ creg, int64_t K, int64_t nqw, int mode,
                                      int64_t *__restrict__ gcount, const int64_t *__restrict__ off,
                                      uint64_t *__restrict__ it_fp, uint64_t *__restrict__ it_cnt,
                                      int *__restrict__ err) {
  constexpr int64_t WPR = kRegionSlots / 64;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < K * WPR; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = creg[f / WPR] * WPR + (f % WPR);
    int64_t g = 0;
    if (w < nqw) g = decode_word<S>(T, w, mode, mode ? off[f] : 0, it_fp, it_cnt, err);
    if (!mode) gcount[f] = g;
  }
}

// zero new counts are dropped before the merge
__global__ void k_nonzero(const uint64_t *__restrict__ c, int64_t m, uint8_t *__restrict__ keep) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
    keep[j] = c[j] > 0 ? 1 : 0;
}

// Max-plus placement: item i maps the end position e of everything before it
// to max(a_i, e + b_i): first item of a run a = quot + L - 1, b = L; later
// items a = -inf, b = L.  The inclusive scan yields each item's last slot.
struct MaxPlus {
  int64_t a, b;
};
constexpr int64_t kNegInf = -(1LL << 60);
// (saturating at kNegInf, so constant maps -- b = kNegInf, the local
// apply's segment resets -- compose without overflow)
struct MaxPlusOp {
  __host__ __device__ __forceinline__ MaxPlus operator()(const MaxPlus &l, const MaxPlus &rr) const {
    MaxPlus o;
    int64_t t = l.a + rr.b;
    o.a = rr.a > t ? rr.a : t;
    o.b = l.b + rr.b;
    if (o.a < kNegInf) o.a = kNegInf;
    if (o.b < kNegInf) o.b = kNegInf;
    return o;
  }
};

__global__ void k_place_terms(const uint64_t *__restrict__ fp, const uint64_t *__restrict__ cnt, int64_t G, int r,
                              MaxPlus *__restrict__ terms, uint64_t *__restrict__ L_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t f = fp[i];
    uint64_t rem = f & ((1ull << r) - 1);
    int64_t quot = (int64_t)(f >> r);
    uint64_t L = enc_len(rem, cnt[i], r);
    int64_t Ls = L > (1ull << 50) ? (1LL << 50) : (int64_t)L;  // clamp: fails the capacity check anyway
    bool first = i == 0 || (fp[i - 1] >> r) != (f >> r);
    MaxPlus m;
    m.a = first ? quot + Ls - 1 : kNegInf;
    m.b = Ls;
    terms[i] = m;
    L_out[i] = (uint64_t)Ls;
  }
}

// Capacity predicates of the fast path (SURVEY H2 / DESIGN.md):
//  flags[0] |= some cluster ends at or beyond min(phys, (region of its first
//              quotient + 2) * 8192)  -> a SHIFT_BOUND is possible
__global__ void k_cluster_check(const uint64_t *__restrict__ fp, const MaxPlus *__restrict__ ends, int64_t G, int r,
                                int64_t phys, int64_t *__restrict__ cfirst, unsigned *__restrict__ flags) {
  // cfirst[i] = quotient of the first run of i's cluster (written for cluster starts, -1 otherwise)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t quot = (int64_t)(fp[i] >> r);
    bool first = i == 0 || (fp[i - 1] >> r) != (fp[i] >> r);
    bool cstart = i == 0 || (first && quot > ends[i - 1].a + 1);
    cfirst[i] = cstart ? quot : -1;
  }
}

__global__ void k_cluster_check2(const MaxPlus *__restrict__ ends, const int64_t *__restrict__ cfirst_scan,
                                 const int64_t *__restrict__ cfirst, int64_t G, int64_t phys,
                                 unsigned *__restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x) {
    bool cend = i == G - 1 || cfirst[i + 1] >= 0;
    if (!cend) continue;
    int64_t g = cfirst_scan[i] >> kRegionBits;
    int64_t hard = (g + 2) << kRegionBits;
    if (hard > phys) hard = phys;
    if (ends[i].a >= hard) atomicOr(&flags[0], 1u);
  }
}

struct MaxI64 {
  __host__ __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

// Write the new table: every item writes its group; run heads set occupieds,
// run tails set runends; region-boundary runs set the next region's offset.
template <typename S>
__global__ void k_write_items(GqfDev T, const uint64_t *__restrict__ fp, const uint64_t *__restrict__ cnt,
                              const MaxPlus *__restrict__ ends, const uint64_t *__restrict__ L, int64_t G) {
  S *slots = reinterpret_cast<S *>(T.slots);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t f = fp[i];
    int64_t quot = (int64_t)(f >> T.r);
    uint64_t rem = f & ((1ull << T.r) - 1);
    int64_t e = ends[i].a;
    int64_t pos = e - (int64_t)L[i] + 1;
    enc_write<S>(slots, pos, rem, cnt[i], T.r);
    bool first = i == 0 || (fp[i - 1] >> T.r) != (f >> T.r);
    bool last = i == G - 1 || (fp[i + 1] >> T.r) != (f >> T.r);
    if (first) atomicOr((unsigned long long *)&T.occ[quot >> 6], 1ull << (quot & 63));
    if (last) {
      atomicOr((unsigned long long *)&T.run[e >> 6], 1ull << (e & 63));
      int64_t g = quot >> kRegionBits;
      int64_t gnext = i == G - 1 ? (1LL << 62) : ((int64_t)(fp[i + 1] >> T.r) >> kRegionBits);
      if (gnext > g && g + 1 < T.nregions) {
        int64_t sp = e - ((g + 1) << kRegionBits) + 1;
        T.offs[g + 1] = sp > 0 ? (int32_t)sp : 0;
      }
    }
  }
}

__global__ void k_stats(const uint64_t *__restrict__ cnt, const uint64_t *__restrict__ L, int64_t G,
                        int64_t *__restrict__ stats) {
  long long a = 0, b = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x) {
    a += (long long)L[i];
    b += (long long)cnt[i];
  }
  cta_add_u64((unsigned long long *)&stats[0], (unsigned long long)a);
  cta_add_u64((unsigned long long *)&stats[1], (unsigned long long)b);
}

// ---- region-parallel placement of the canonical rebuild -----------------------
// The merged items (sorted, canonical counts) are placed region by region:
//   k_region_summary: one CTA per 8192-quotient region composes its items'
//     max-plus terms in order (item i maps the end e of everything before it
//     to max(a_i, e + L_i)), preceded by the clamp e -> max(region start - 1, e);
//   an inclusive scan of the region summaries gives every region's incoming
//   end e_in (the spill of earlier regions' runs);
//   k_region_place: one CTA per region places its items from e_in and writes
//     its whole responsibility range [P_g, P_g+1) of the new image -- slots
//     (zeros between clusters), runend bits (atomics only on the boundary
//     words), its occupieds words, its offset -- so the second image needs
//     no clearing pass; it counts (slot, runend) changes against the old
//     image (the shift metric) and flags the canonical layout as unusable
//     when a cluster would span three regions or pass the table's end (the
//     reference's CLUSTER / SHIFT_BOUND conditions: the exact path runs).
constexpr int kRegThreads = 256;
constexpr int64_t kRegMaxRange = 3 * kRegionSlots;  // a valid region's slot range is < 2 regions

__device__ __forceinline__ MaxPlus mp_id() {
  MaxPlus m;
  m.a = kNegInf;
  m.b = 0;
  return m;
}

__device__ __forceinline__ MaxPlus mp_op(const MaxPlus &l, const MaxPlus &rr) {  // l first, then rr
  return MaxPlusOp()(l, rr);
}

__device__ __forceinline__ MaxPlus item_term(const uint64_t *fp, const uint64_t *cnt, int64_t i, int64_t a, int r,
                                             int64_t *Lout) {
  const uint64_t f = fp[i];
  const uint64_t L = enc_len(f & ((1ull << r) - 1), cnt[i], r);
  const int64_t Ls = L > (1ull << 50) ? (1LL << 50) : (int64_t)L;
  const bool first = i == a || (fp[i - 1] >> r) != (f >> r);
  MaxPlus m;
  m.a = first ? (int64_t)(f >> r) + Ls - 1 : kNegInf;
  m.b = Ls;
  *Lout = Ls;
  return m;
}

// Exclusive (in thread order) max-plus prefix of every thread's value, and
// the block total.  All threads call it.
__device__ __forceinline__ MaxPlus block_excl_mp(MaxPlus v, MaxPlus *sw, MaxPlus *total) {
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  MaxPlus inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    MaxPlus y;
    y.a = __shfl_up_sync(0xFFFFFFFFu, inc.a, o);
    y.b = __shfl_up_sync(0xFFFFFFFFu, inc.b, o);
    if ((int)lane >= o) inc = mp_op(y, inc);
  }
  MaxPlus ex;
  ex.a = __shfl_up_sync(0xFFFFFFFFu, inc.a, 1);
  ex.b = __shfl_up_sync(0xFFFFFFFFu, inc.b, 1);
  if (lane == 0) ex = mp_id();
  if (lane == 31) sw[warp] = inc;
  __syncthreads();
  MaxPlus wp = mp_id();
  for (int w = 0; w < (int)warp; w++) wp = mp_op(wp, sw[w]);
  MaxPlus t = mp_id();
  for (int w = 0; w < kRegThreads / 32; w++) t = mp_op(t, sw[w]);
  *total = t;
  __syncthreads();
  return mp_op(wp, ex);
}

// Regions: creg[0..K) (the local apply's candidate list), or 0..K-1 when
// creg is null.  old_offs (local apply): a region whose predecessor is not
// in the list starts from its old incoming end, base - 1 + old_offs[g]
// (a constant map composed in front of its summary).
__global__ void __launch_bounds__(kRegThreads) k_region_summary(const uint64_t *__restrict__ fp,
                                                                const uint64_t *__restrict__ cnt,
                                                                const int64_t *__restrict__ ib,
                                                                const int64_t *__restrict__ creg, int64_t K,
                                                                const int32_t *__restrict__ old_offs, int r,
                                                                MaxPlus *__restrict__ summ,
                                                                unsigned long long *__restrict__ acc) {
  __shared__ MaxPlus sw[kRegThreads / 32];
  // slot and count sums over every region this CTA composes, added to acc
  // once per CTA at the end (per-warp atomics per region were ~0.5 M
  // same-address atomics at C4)
  unsigned long long ls_all = 0, cs_all = 0;
  for (int64_t li = blockIdx.x; li < K; li += gridDim.x) {
    const int64_t g = creg ? creg[li] : li;
    const int64_t a = ib[g], e = ib[g + 1], n = e - a;
    const int64_t c = (n + kRegThreads - 1) / kRegThreads;
    const int64_t i0 = a + (int64_t)threadIdx.x * c, i1 = min(e, i0 + c);
    MaxPlus v = mp_id();
    unsigned long long ls = 0, cs = 0;
    for (int64_t i = i0; i < i1; i++) {
      int64_t L;
      v = mp_op(v, item_term(fp, cnt, i, a, r, &L));
      ls += (unsigned long long)L;
      cs += cnt[i];
    }
    MaxPlus tot;
    block_excl_mp(v, sw, &tot);
    if (threadIdx.x == 0) {
      MaxPlus clamp;
      clamp.a = (g << kRegionBits) - 1;
      clamp.b = 0;
      MaxPlus el = mp_op(clamp, tot);
      if (old_offs && (li == 0 || creg[li - 1] != g - 1)) {
        MaxPlus reset;
        reset.a = (g << kRegionBits) - 1 + old_offs[g];
        reset.b = kNegInf;
        el = mp_op(reset, el);
      }
      summ[li] = el;
    }
    ls_all += ls;
    cs_all += cs;
  }
  cta_add_u64(&acc[0], ls_all);
  cta_add_u64(&acc[1], cs_all);
}

__device__ __forceinline__ int64_t mp_end(const MaxPlus &m) {  // applied to e = -1
  const int64_t t = m.b - 1;
  return m.a > t ? m.a : t;
}

// Bit j of *chg: slot j of the 64-slot word differs between a and b; of
// *nz: a's slot j is non-zero.  16-byte vector loads (the word is aligned).
template <typename S>
__device__ __forceinline__ void word_slot_masks(const S *a, const S *b, unsigned long long *chg,
                                                unsigned long long *nz) {
  constexpr int PER = 16 / (int)sizeof(S), V = 64 / PER;
  const uint4 *va = reinterpret_cast<const uint4 *>(a), *vb = reinterpret_cast<const uint4 *>(b);
  unsigned long long c = 0, z = 0;
#pragma unroll
  for (int v = 0; v < V; v++) {
    const uint4 x = va[v], y = vb[v];
    const S *xs = reinterpret_cast<const S *>(&x), *ys = reinterpret_cast<const S *>(&y);
#pragma unroll
    for (int j = 0; j < PER; j++) {
      c |= (unsigned long long)(xs[j] != ys[j]) << (v * PER + j);
      z |= (unsigned long long)(xs[j] != 0) << (v * PER + j);
    }
  }
  *chg = c;
  *nz = z;
}

// flags[0] |= 1: the canonical layout breaks the reference's bounds (a
// cluster spans three regions / passes the table end): use the exact path.
// Region list as in k_region_summary.  Global apply (creg null): writes the
// new image T1 (= next) against the old image old_slots / old_run.  Local
// apply (creg, old_offs): T1 is the current image, rewritten in place; a
// first pass with plan_only validates every region (and the old incoming
// ends at the ends of runs of listed regions) and saves each region's old
// window [base, base + kRegMaxRange) to saved_* for the shift metric; the
// second pass writes.
template <typename S>
struct RegionJob {
  const int64_t *creg;
  int64_t K, nqr;
  const int32_t *old_offs;
  int plan_only;
  S *saved_slots;               // [K][kRegMaxRange]
  unsigned long long *saved_run;  // [K][kRegMaxRange / 64 + 1]
};

template <typename S>
__global__ void __launch_bounds__(kRegThreads) k_region_place(GqfDev T1, const S *__restrict__ old_slots,
                                                              const uint64_t *__restrict__ old_run,
                                                              const uint64_t *__restrict__ fp,
                                                              const uint64_t *__restrict__ cnt,
                                                              const int64_t *__restrict__ ib,
                                                              const MaxPlus *__restrict__ cum, RegionJob<S> J,
                                                              const unsigned *__restrict__ not_asc, int bulk_order,
                                                              unsigned *__restrict__ flags,
                                                              unsigned long long *__restrict__ diff) {
  __shared__ MaxPlus sw[kRegThreads / 32];
  __shared__ unsigned long long s_run[kRegMaxRange / 64 + 2];
  __shared__ unsigned long long s_occ[kRegionSlots / 64];
  __shared__ int s_cs, s_bad;
  S *slots = reinterpret_cast<S *>(T1.slots);
  const int r = T1.r;
  const int64_t phys = T1.phys, nqr = J.nqr;
  const bool old_only = bulk_order || !*not_asc;
  const bool local = J.creg != nullptr, plan = J.plan_only != 0;
  constexpr int64_t SW = kRegMaxRange / 64 + 1;  // saved runend words per region
  unsigned long long ndiff = 0;
  for (int64_t li = blockIdx.x; li < J.K; li += gridDim.x) {
    const int64_t g = local ? J.creg[li] : li;
    const int64_t base = g << kRegionBits;
    const bool seg_start = local && (li == 0 || J.creg[li - 1] != g - 1);
    const bool seg_end = local && (li + 1 == J.K || J.creg[li + 1] != g + 1);
    // end of every earlier region's runs (local segment starts: the old one)
    const int64_t e_in = seg_start ? base - 1 + J.old_offs[g] : (li ? mp_end(cum[li - 1]) : -1);
    const int64_t e_out = mp_end(cum[li]);  // >= base - 1 (the summary is clamped)
    const int64_t P0 = e_in + 1 > base ? e_in + 1 : base;
    int64_t P1 = g + 1 < nqr ? (e_out + 1 > base + kRegionSlots ? e_out + 1 : base + kRegionSlots) : phys;
    if (plan) {
      // save the old window for the shift metric (before any region writes)
      S *sv = J.saved_slots + li * kRegMaxRange;
      for (int64_t p = threadIdx.x; p < kRegMaxRange; p += kRegThreads) sv[p] = base + p < phys ? old_slots[base + p] : (S)0;
      for (int64_t w = threadIdx.x; w < SW; w += kRegThreads)
        J.saved_run[li * SW + w] = (base >> 6) + w < (phys >> 6) ? old_run[(base >> 6) + w] : 0ull;
    }
    if (threadIdx.x == 0) {
      s_cs = 0;
      s_bad = 0;
    }
    if (threadIdx.x == 0 && !plan) {
      // the offsets of this region (and of the padding region after the last one)
      T1.offs[g] = (int32_t)(e_in + 1 > base ? e_in + 1 - base : 0);
      if (g + 1 == nqr)
        for (int64_t h = nqr; h < T1.nregions; h++) {
          const int64_t bh = h << kRegionBits;
          T1.offs[h] = (int32_t)(e_out + 1 > bh ? e_out + 1 - bh : 0);
        }
    }
    for (int i = threadIdx.x; i < kRegMaxRange / 64 + 2; i += kRegThreads) s_run[i] = 0;
    for (int i = threadIdx.x; i < kRegionSlots / 64; i += kRegThreads) s_occ[i] = 0;
    __syncthreads();
    bool bad = e_out >= phys || P1 > phys || P1 - base > kRegMaxRange;
    // a run of listed regions must hand the next, unlisted region its old incoming end
    if (seg_end && g + 1 < nqr && e_out > base + kRegionSlots - 1 + J.old_offs[g + 1]) bad = true;
    if (seg_end && g + 1 < nqr && J.old_offs[g + 1] > 0 && e_out != base + kRegionSlots - 1 + J.old_offs[g + 1]) bad = true;
    if (!bad && !plan) {  // zero the range: ragged ends slot by slot, the middle in 16-byte stores
      constexpr int PER = 16 / (int)sizeof(S);
      const int64_t q0 = (P0 + PER - 1) / PER * PER, q1 = P1 / PER * PER;
      if (q0 >= q1) {
        for (int64_t p = P0 + threadIdx.x; p < P1; p += kRegThreads) slots[p] = 0;
      } else {
        for (int64_t p = P0 + threadIdx.x; p < q0; p += kRegThreads) slots[p] = 0;
        for (int64_t p = q1 + threadIdx.x; p < P1; p += kRegThreads) slots[p] = 0;
        uint4 *v = reinterpret_cast<uint4 *>(slots + q0);
        for (int64_t j = threadIdx.x; j < (q1 - q0) / PER; j += kRegThreads) v[j] = make_uint4(0, 0, 0, 0);
      }
    }
    __syncthreads();
    // place: per-thread chunks composed in order, then each item's end
    const int64_t a = ib[g], e = ib[g + 1], n = e - a;
    const int64_t c = (n + kRegThreads - 1) / kRegThreads;
    const int64_t i0 = a + (int64_t)threadIdx.x * c, i1 = min(e, i0 + c);
    MaxPlus v = mp_id();
    for (int64_t i = i0; i < i1; i++) {
      int64_t L;
      v = mp_op(v, item_term(fp, cnt, i, a, r, &L));
    }
    MaxPlus tot;
    const MaxPlus pre = block_excl_mp(v, sw, &tot);
    int64_t run_end = pre.b + e_in > pre.a ? pre.b + e_in : pre.a;  // end of everything before my chunk
    const int64_t w0 = P0 >> 6;
    for (int64_t i = i0; i < i1 && !bad; i++) {
      int64_t L;
      const MaxPlus t = item_term(fp, cnt, i, a, r, &L);
      const int64_t prev = run_end;
      run_end = t.a > prev + L ? t.a : prev + L;
      const uint64_t f = fp[i];
      const int64_t quot = (int64_t)(f >> r);
      const bool first = t.a != kNegInf;
      const bool last = i + 1 == e || (fp[i + 1] >> r) != (f >> r);
      if (first) {
        if (quot > prev + 1) s_cs = 1;  // a cluster starts in this region
        atomicOr(&s_occ[(quot - base) >> 6], 1ull << (quot & 63));
      }
      if (run_end >= P1) {  // (only with a broken layout)
        s_bad = 1;
        break;
      }
      if (!plan) enc_write<S>(slots, run_end - L + 1, f & ((1ull << r) - 1), cnt[i], r);
      if (last) atomicOr(&s_run[(run_end >> 6) - w0], 1ull << (run_end & 63));
    }
    __syncthreads();
    // a spill into the next region must come from a cluster that started here
    if (threadIdx.x == 0 && g + 1 < nqr && e_out >= base + kRegionSlots && !s_cs) s_bad = 1;
    __syncthreads();
    bad = bad || s_bad;
    if (bad) {
      if (threadIdx.x == 0) atomicOr(&flags[0], 1u);
      continue;  // the image is discarded / the local apply does not run
    }
    if (plan) {
      __syncthreads();
      continue;
    }
    // occupieds words of this region's quotients (and the padding's, zero)
    const int64_t nw_own = (phys >> 6) - (base >> 6) < kRegionSlots / 64 ? (phys >> 6) - (base >> 6) : kRegionSlots / 64;
    for (int i = threadIdx.x; i < nw_own; i += kRegThreads) T1.occ[(base >> 6) + i] = s_occ[i];
    if (g + 1 == nqr)
      for (int64_t w = ((base + kRegionSlots) >> 6) + threadIdx.x; w < (phys >> 6); w += kRegThreads) T1.occ[w] = 0;
    // runend words over [P0, P1): boundary words through atomics (neighbours own the other bits)
    const int64_t w1 = (P1 - 1) >> 6;
    for (int64_t w = w0 + threadIdx.x; w <= w1; w += kRegThreads) {
      const int64_t lo = w << 6, hi = lo + 64;
      unsigned long long mask = ~0ull;
      if (P0 > lo) mask &= ~0ull << (P0 - lo);
      if (P1 < hi) mask &= ~0ull >> (hi - P1);
      const unsigned long long bits = s_run[w - w0] & mask;
      if (mask == ~0ull) {
        T1.run[w] = bits;
      } else {
        atomicAnd((unsigned long long *)&T1.run[w], ~mask);
        if (bits) atomicOr((unsigned long long *)&T1.run[w], bits);
      }
      // shift metric: (slot, runend) changes against the old image, 64
      // slots at a time from 16-byte loads
      unsigned long long chg, nz, ob;
      if (local) {
        word_slot_masks<S>(J.saved_slots + li * kRegMaxRange + (lo - base), slots + lo, &chg, &nz);
        ob = J.saved_run[li * SW + (w - (base >> 6))];
      } else {
        word_slot_masks<S>(old_slots + lo, slots + lo, &chg, &nz);
        ob = old_run[w];
      }
      const unsigned long long changed = (chg | (ob ^ bits)) & mask;
      ndiff += __popcll(old_only ? (changed & (nz | ob)) : changed);
    }
    __syncthreads();
  }
  cta_add_u64(diff, (unsigned long long)ndiff);
}

// local apply candidates: regions holding new items, and their successors
__global__ void k_region_candidates(const int64_t *__restrict__ rbu, int64_t nqr, uint8_t *__restrict__ cand) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nqr; g += (int64_t)gridDim.x * blockDim.x) {
    const bool dirty = rbu[g + 1] > rbu[g], prev = g > 0 && rbu[g] > rbu[g - 1];
    cand[g] = (dirty || prev) ? 1 : 0;
  }
}

// slot and count sums of a list of items (the local apply's old items)
__global__ void k_item_sums(const uint64_t *__restrict__ fp, const uint64_t *__restrict__ cnt, int64_t n, int r,
                            unsigned long long *__restrict__ acc) {
  unsigned long long ls = 0, cs = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t L = enc_len(fp[i] & ((1ull << r) - 1), cnt[i], r);
    ls += L;
    cs += cnt[i];
  }
  cta_add_u64(&acc[0], ls);
  cta_add_u64(&acc[1], cs);
}

// stats += new - old (local apply: acc = new sums, old = the replaced items' sums)
__global__ void k_region_stats_delta(const unsigned long long *__restrict__ acc_new,
                                     const unsigned long long *__restrict__ acc_old, int64_t g_new, int64_t g_old,
                                     int64_t *__restrict__ stats) {
  stats[0] += (int64_t)acc_new[0] - (int64_t)acc_old[0];
  stats[1] += (int64_t)acc_new[1] - (int64_t)acc_old[1];
  stats[2] += g_new - g_old;
}

__global__ void k_region_stats(const unsigned long long *__restrict__ acc, int64_t G, int64_t *__restrict__ stats) {
  stats[0] = (int64_t)acc[0];
  stats[1] = (int64_t)acc[1];
  stats[2] = G;
}

// shift instrumentation: slots whose (word, runend bit) changed, optionally
// restricted to positions the old table used
template <typename S>
__global__ void k_diff_count(const S *__restrict__ a, const uint64_t *__restrict__ ra, const S *__restrict__ b,
                             const uint64_t *__restrict__ rb, int64_t phys, int old_only,
                             unsigned long long *__restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < phys; i += (int64_t)gridDim.x * blockDim.x) {
    int ba = bit_at(ra, i), bb = bit_at(rb, i);
    bool used_old = a[i] != 0 || ba;
    if ((a[i] != b[i] || ba != bb) && (!old_only || used_old)) c++;
  }
  cta_add_u64(out, (unsigned long long)c);
}

// *flag = 1 when the batch's fingerprints are NOT non-decreasing in input
// order.  A non-decreasing batch never moves the slots it wrote itself (each
// item lands after every earlier one), so its sequential shift work is made
// of old slots only -- the bulk shift metric.
__global__ void k_not_ascending(const uint64_t *__restrict__ keys, int keys_are_fps, uint64_t seed, uint64_t fmask,
                                int64_t n, unsigned *__restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = keys_are_fps ? keys[i - 1] & fmask : mix64(keys[i - 1] ^ seed) & fmask;
    const uint64_t b = keys_are_fps ? keys[i] & fmask : mix64(keys[i] ^ seed) & fmask;
    if (a > b) *flag = 1u;
  }
}

// ---------------------------------------------------------------------------
// exact sequential path (reference algorithm, _pykernels.py:485-656), used
// only when a batch may hit a capacity error
// ---------------------------------------------------------------------------
template <typename S>
struct SeqGqf {
  S *slots;
  uint64_t *occ, *run;
  int32_t *offs;
  int64_t *stats;
  int64_t phys;
  int r;
  int32_t *scratch;  // GAP_CAP entries for this thread

  static constexpr int64_t kGapCap = 2 * kRegionSlots;

  __device__ int64_t rank_range(const uint64_t *bv, int64_t a, int64_t b) const {
    int64_t n = 0;
    for (int64_t i = a; i < b;) {
      int64_t lo = i & 63, span = 64 - lo;
      if (span > b - i) span = b - i;
      uint64_t w = bv[i >> 6] >> lo;
      if (span < 64) w &= (1ull << span) - 1;
      n += __popcll(w);
      i += span;
    }
    return n;
  }
  __device__ int64_t run_end_local(int64_t x, int64_t hard) const {  // pk:469-482
    int64_t h = x >> kRegionBits, s_h = h << kRegionBits;
    int64_t k = rank_range(occ, s_h, x + 1);
    int64_t base = s_h + offs[h] - 1;
    return k == 0 ? base : select_after_dev(run, base, k, hard);
  }
  __device__ int64_t first_unused(int64_t pos, int64_t hard) const {  // pk:485-495
    for (int64_t x = pos; x < hard;) {
      int64_t e = run_end_local(x, hard);
      if (e == -2) return -2;
      if (e < x) return x;
      x = e + 1;
    }
    return -2;
  }
  __device__ void setb(uint64_t *bv, int64_t i, int v) const {
    uint64_t m = 1ull << (i & 63);
    if (v) bv[i >> 6] |= m; else bv[i >> 6] &= ~m;
  }
  __device__ void move_up(int64_t a, int64_t b, int64_t L) const {  // pk:498-505
    for (int64_t i = b - 1; i >= a; i--) slots[i + L] = slots[i];
    for (int64_t i = b - 1; i >= a; i--) setb(run, i + L, bit_at(run, i));
    int64_t stop = a + L < b + L ? a + L : b + L;
    for (int64_t i = a; i < stop; i++) setb(run, i, 0);
  }
  __device__ int64_t make_room(int64_t pos, int64_t L, int64_t hard, int64_t *far) const {  // pk:508-533
    if (L > kGapCap) return -1;
    int64_t x = pos;
    for (int64_t t = 0; t < L; t++) {
      int64_t e = first_unused(x, hard);
      if (e < 0) return -1;
      scratch[t] = (int32_t)e;
      x = e + 1;
    }
    int64_t moved = 0;
    for (int64_t k = L; k >= 1; k--) {
      int64_t a = (k >= 2 ? (int64_t)scratch[k - 2] : pos - 1) + 1, b = scratch[k - 1];
      if (b > a) { move_up(a, b, L - k + 1); moved += b - a; }
    }
    *far = scratch[L - 1];
    return moved;
  }
  __device__ bool run_interval(int64_t quot, int64_t *s, int64_t *e) const {  // pk:536-549
    int64_t h = quot >> kRegionBits;
    int64_t hard = (h + 2) << kRegionBits;
    if (hard > phys) hard = phys;
    int64_t s_h = h << kRegionBits;
    int64_t k = rank_range(occ, s_h, quot + 1);
    int64_t base = s_h + offs[h] - 1;
    int64_t prev = k == 1 ? base : select_after_dev(run, base, k - 1, hard);
    int64_t end = select_after_dev(run, base, k, hard);
    if (prev == -2 || end == -2) return false;
    *s = quot > prev + 1 ? quot : prev + 1;
    *e = end;
    return true;
  }
  __device__ bool find_group(int64_t st, int64_t en, uint64_t rem, int64_t *gs, int64_t *ge, uint64_t *c,
                             int64_t *sp) const {  // pk:552-566
    *gs = *ge = *sp = -1;
    *c = 0;
    for (int64_t i = st; i <= en;) {
      uint64_t h, cnt;
      int64_t nx;
      if (!parse_group_dev<S>(slots, i, en, r, &h, &cnt, &nx)) return false;
      if (h == rem) { *gs = i; *ge = nx - 1; *c = cnt; return true; }
      if (h > rem) { *sp = i; return true; }
      i = nx;
    }
    *sp = en + 1;
    return true;
  }
  __device__ bool refresh_offset(int64_t h) const {  // pk:569-576
    int64_t b = h << kRegionBits;
    int64_t hard = (h + 1) << kRegionBits;
    if (hard > phys) hard = phys;
    int64_t e = run_end_local(b - 1, hard);
    if (e == -2) return false;
    offs[h] = (int32_t)(e - b + 1 > 0 ? e - b + 1 : 0);
    return true;
  }
  __device__ void add_stats(int64_t a, int64_t b, int64_t c) const {  // fk_atomic_add64 (ck:36)
    if (a) atomicAdd((unsigned long long *)&stats[0], (unsigned long long)a);
    if (b) atomicAdd((unsigned long long *)&stats[1], (unsigned long long)b);
    if (c) atomicAdd((unsigned long long *)&stats[2], (unsigned long long)c);
  }
  // pk:584-656 -> 0 ok, 1 LOAD_CAPACITY, 2 SHIFT_BOUND, -9 invariant
  __device__ int insert_one(int64_t max_occ, uint64_t fp, uint64_t delta, int64_t *moved_out) {
    int64_t quot = (int64_t)(fp >> r);
    uint64_t rem = fp & ((1ull << r) - 1);
    int64_t g = quot >> kRegionBits;
    int64_t hard = (g + 2) << kRegionBits;
    if (hard > phys) hard = phys;
    int64_t moved = 0, far = 0, touched = 0;
    *moved_out = 0;
    if (*(volatile int64_t *)&stats[0] >= max_occ) return 1;
    if (!bit_at(occ, quot)) {
      int64_t e = run_end_local(quot, hard);
      if (e == -2) return 2;
      int64_t pos = quot > e + 1 ? quot : e + 1;
      int64_t L = (int64_t)enc_len(rem, delta, r);
      moved = make_room(pos, L, hard, &far);
      if (moved < 0) return 2;
      enc_write<S>(slots, pos, rem, delta, r);
      setb(occ, quot, 1);
      setb(run, pos + L - 1, 1);
      touched = far + 1;
      add_stats(L, (int64_t)delta, 1);
    } else {
      int64_t s, e, gs, ge, sp;
      uint64_t c;
      if (!run_interval(quot, &s, &e)) return -9;
      if (!find_group(s, e, rem, &gs, &ge, &c, &sp)) return -9;
      if (gs >= 0) {
        int64_t L = (int64_t)enc_len(rem, c + delta, r);
        int64_t diff = L - (ge - gs + 1);
        if (diff > 0) {
          moved = make_room(ge + 1, diff, hard, &far);
          if (moved < 0) return 2;
          if (ge == e) { setb(run, e, 0); setb(run, e + diff, 1); }
          touched = far + 1;
        }
        enc_write<S>(slots, gs, rem, c + delta, r);
        add_stats(diff, (int64_t)delta, 0);
      } else {
        int64_t L = (int64_t)enc_len(rem, delta, r);
        moved = make_room(sp, L, hard, &far);
        if (moved < 0) return 2;
        enc_write<S>(slots, sp, rem, delta, r);
        if (sp == e + 1) { setb(run, e, 0); setb(run, e + L, 1); }
        touched = far + 1;
        add_stats(L, (int64_t)delta, 1);
      }
    }
    int64_t boundary = (g + 1) << kRegionBits;
    if (boundary < phys && touched > boundary)
      if (!refresh_offset(g + 1)) return -9;
    *moved_out = moved;
    return 0;
  }

  // Remove slots [rs, re] of quot's run [start, end], left-compacting the
  // cluster (pk:659-715).  Returns the furthest old slot touched, -1 on an
  // invariant violation; *moved gets the number of slots moved.
  __device__ int64_t remove_slots(int64_t quot, int64_t start, int64_t end, int64_t rs, int64_t re, int64_t hard,
                                  int64_t *moved) const {
    const int64_t L = re - rs + 1;
    const bool emptied = L == end - start + 1;
    int64_t shifted = 0;
    for (int64_t i = 0; i < end - re; i++) slots[rs + i] = slots[re + 1 + i];
    shifted += end - re;
    setb(run, end, 0);
    int64_t wp;
    if (emptied) {
      setb(occ, quot, 0);
      wp = start;
    } else {
      setb(run, end - L, 1);
      wp = end - L + 1;
    }
    int64_t prev_old_end = end, last_old_end = end, nq = quot;
    for (;;) {
      nq = select_after_dev(occ, nq, 1, hard);
      if (nq < 0 || nq > prev_old_end + 1) break;  // a gap: the cluster ends
      const int64_t s2 = prev_old_end + 1;
      const int64_t e2 = select_after_dev(run, s2 - 1, 1, hard);
      if (e2 == -2) return -1;
      const int64_t ns2 = nq > wp ? nq : wp;
      if (ns2 == s2) break;
      for (int64_t i = wp; i < ns2; i++) {  // skipped positions are freed for good
        slots[i] = 0;
        setb(run, i, 0);
      }
      const int64_t n2 = e2 - s2 + 1;
      for (int64_t i = 0; i < n2; i++) slots[ns2 + i] = slots[s2 + i];
      setb(run, e2, 0);
      setb(run, ns2 + n2 - 1, 1);
      shifted += n2;
      wp = ns2 + n2;
      prev_old_end = e2;
      last_old_end = e2;
    }
    for (int64_t i = wp; i <= last_old_end; i++) {
      slots[i] = 0;
      setb(run, i, 0);
    }
    *moved = shifted;
    return last_old_end;
  }

  // pk:718-752 -> found (0/1), -9 on an invariant violation
  __device__ int delete_one(uint64_t fp, uint64_t delta, int64_t *moved_out) {
    const int64_t quot = (int64_t)(fp >> r);
    const uint64_t rem = fp & ((1ull << r) - 1);
    const int64_t g = quot >> kRegionBits;
    int64_t hard = (g + 2) << kRegionBits;
    if (hard > phys) hard = phys;
    *moved_out = 0;
    if (!bit_at(occ, quot)) return 0;
    int64_t st, en, gs, ge, sp;
    uint64_t c;
    if (!run_interval(quot, &st, &en)) return -9;
    if (!find_group(st, en, rem, &gs, &ge, &c, &sp)) return -9;
    if (gs < 0) return 0;
    const uint64_t take = delta < c ? delta : c;
    const uint64_t c2 = c - take;
    int64_t rs, re;
    if (c2 > 0) {
      const int64_t L = (int64_t)enc_len(rem, c2, r);
      const int64_t diff = (ge - gs + 1) - L;
      enc_write<S>(slots, gs, rem, c2, r);
      add_stats(0, -(int64_t)take, 0);
      if (diff == 0) return 1;
      rs = gs + L;
      re = ge;
    } else {
      add_stats(0, -(int64_t)take, -1);
      rs = gs;
      re = ge;
    }
    int64_t moved = 0;
    const int64_t last = remove_slots(quot, st, en, rs, re, hard, &moved);
    if (last < 0) return -9;
    add_stats(-(re - rs + 1), 0, 0);
    const int64_t boundary = (g + 1) << kRegionBits;
    if (boundary < phys && last >= boundary)
      if (!refresh_offset(g + 1)) return -9;
    *moved_out = moved;
    return 1;
  }
};

// insert_many semantics: one thread, input order, stop at the first failure
template <typename S>
__global__ void k_gqf_exact_seq(GqfDev T, const uint64_t *__restrict__ fps, const uint64_t *__restrict__ deltas,
                                int64_t n, int32_t *scratch, int64_t *__restrict__ result) {
  if (blockIdx.x || threadIdx.x) return;
  SeqGqf<S> G{reinterpret_cast<S *>(T.slots), T.occ, T.run, T.offs, T.stats, T.phys, T.r, scratch};
  int64_t moved_total = 0;
  result[0] = 0;
  result[1] = -1;
  for (int64_t k = 0; k < n; k++) {
    int64_t mv;
    int code = G.insert_one(T.max_occ, fps[k], deltas ? deltas[k] : 1, &mv);
    if (code) {
      result[0] = code;
      result[1] = k;
      break;
    }
    moved_total += mv;
  }
  result[2] = moved_total;
}

// bulk_insert semantics: one thread per region of one parity, each applying
// its sorted items in order; a failure stops that region only (gqf.py:293-353)
template <typename S>
__global__ void k_gqf_exact_regions(GqfDev T, const uint64_t *__restrict__ fps_s, const uint64_t *__restrict__ deltas_s,
                                    const int64_t *__restrict__ rb, int64_t nqr, int parity, int32_t *scratch,
                                    int32_t *__restrict__ fail_code, unsigned long long *__restrict__ moved) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t g = parity + 2 * t;
    if (g >= nqr) break;
    int64_t lo = rb[g], hi = rb[g + 1];
    if (lo >= hi) continue;
    int64_t slot = gridDim.x * blockDim.x == 1 ? 0 : t;  // one scratch area per concurrent thread
    SeqGqf<S> G{reinterpret_cast<S *>(T.slots), T.occ, T.run, T.offs, T.stats, T.phys, T.r,
                scratch + (size_t)slot * SeqGqf<S>::kGapCap};
    unsigned long long mv_total = 0;
    for (int64_t k = lo; k < hi; k++) {
      int64_t mv;
      // stats[0] is shared by concurrent regions: the reference's workers race
      // on it the same way (gqf.py:309-315); reads here are atomic snapshots
      int code = G.insert_one(T.max_occ, fps_s[k], deltas_s[k], &mv);
      if (code) {
        fail_code[g] = code;
        break;
      }
      mv_total += (unsigned long long)mv;
    }
    if (mv_total) atomicAdd(moved, mv_total);
  }
}

// Small batches: the reference's region-parallel insert (gqf.py:309-353,
// even regions then odd ones) on the listed regions only, one thread per
// region.  Without a capacity error its result is the canonical table
// (SURVEY H2), at a cost proportional to the batch, not the table.
template <typename S>
__global__ void k_gqf_insert_regions(GqfDev T, const uint64_t *__restrict__ fps_s,
                                     const uint64_t *__restrict__ deltas_s, const int64_t *__restrict__ rb,
                                     const int32_t *__restrict__ list, int64_t nlist, int32_t *scratch,
                                     int32_t *__restrict__ fail_code, unsigned long long *__restrict__ moved) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nlist; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = list[t];
    SeqGqf<S> G{reinterpret_cast<S *>(T.slots), T.occ, T.run, T.offs, T.stats, T.phys, T.r,
                scratch + (size_t)t * SeqGqf<S>::kGapCap};
    unsigned long long mv_total = 0;
    for (int64_t k = rb[g]; k < rb[g + 1]; k++) {
      int64_t mv;
      int code = G.insert_one(T.max_occ, fps_s[k], deltas_s ? deltas_s[k] : 1ull, &mv);
      if (code) {
        fail_code[t] = code;
        break;
      }
      mv_total += (unsigned long long)mv;
    }
    if (mv_total) atomicAdd(moved, mv_total);
  }
}

// Small delete batches: one thread per touched region of one parity,
// applying the region's sorted items in the facade's order -- descending for
// bulk_delete (gqf.py:317-325), ascending (input order) for delete_many --
// and recording each item's found flag at its input position.
template <typename S>
__global__ void k_gqf_delete_regions(GqfDev T, const uint64_t *__restrict__ fps_s, const uint64_t *__restrict__ deltas_s,
                                     const uint32_t *__restrict__ idx_s, const int64_t *__restrict__ rb,
                                     const int32_t *__restrict__ list, int64_t nlist, int descending,
                                     uint8_t *__restrict__ found, int32_t *__restrict__ fail_code,
                                     unsigned long long *__restrict__ moved) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nlist; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = list[t];
    SeqGqf<S> G{reinterpret_cast<S *>(T.slots), T.occ, T.run, T.offs, T.stats, T.phys, T.r, nullptr};
    unsigned long long mv_total = 0;
    const int64_t lo = rb[g], hi = rb[g + 1];
    for (int64_t u = 0; u < hi - lo; u++) {
      const int64_t k = descending ? hi - 1 - u : lo + u;
      int64_t mv;
      const int f = G.delete_one(fps_s[k], deltas_s[k], &mv);
      if (f < 0) {
        fail_code[t] = f;
        break;
      }
      if (found) found[idx_s[k]] = (uint8_t)f;
      mv_total += (unsigned long long)mv;
    }
    if (mv_total) atomicAdd(moved, mv_total);
  }
}

__global__ void k_region_bounds(const uint64_t *__restrict__ fps_s, int64_t n, int shift, int64_t nqr,
                                int64_t *__restrict__ rb) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g <= nqr; g += (int64_t)gridDim.x * blockDim.x) {
    uint64_t mark = (uint64_t)g << shift;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (fps_s[mid] < mark) lo = mid + 1; else hi = mid;
    }
    rb[g] = lo;
  }
}


// ---------------------------------------------------------------------------
// Device-side structure validation (Gqf.validate, gqf.py:430-492), derived
// from the bit vectors alone (global rank/select; the spill index is not
// trusted).  Each failed check sets its code's bit in v[0] and atomicMin's
// the first offending quotient / region / slot into v[8 + code]; v[1..4]
// accumulate used slots, decoded total, decoded distinct, non-zero slots
// inside runs; v[5] = non-zero slots anywhere.
// ---------------------------------------------------------------------------
enum GqfCheck {
  kVRankMismatch = 1, kVQuotBeyond = 2, kVRunPastPhys = 3, kVNegativeRun = 5, kVHardBound = 7,
  kVOffset = 8, kVUndecodable = 11, kVUnsorted = 12
};
constexpr int kValidateWords = 8 + 16;

__device__ __forceinline__ void vfail(int64_t *v, int code, int64_t pos) {
  atomicOr((unsigned long long *)&v[0], 1ull << code);
  atomicMin((long long *)&v[8 + code], (long long)pos);
}

// k-th (0-based) set bit of bv given the exclusive per-word prefix ranks.
__device__ __forceinline__ int64_t select_global(const uint64_t *bv, const int64_t *rank, int64_t nw, int64_t k) {
  int64_t lo = 0, hi = nw;  // last word whose rank <= k
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (rank[mid] <= k) lo = mid; else hi = mid;
  }
  uint64_t w = bv[lo];
  for (int64_t c = k - rank[lo]; c > 0; c--) w &= w - 1;
  return (lo << 6) + __ffsll((long long)w) - 1;
}

template <typename S>
__global__ void k_gqf_validate_runs(GqfDev T, int64_t nw, const int64_t *__restrict__ ro,
                                    const int64_t *__restrict__ rr, int64_t *__restrict__ v) {
  const S *slots = reinterpret_cast<const S *>(T.slots);
  const int64_t logical = 1LL << T.q;
  unsigned long long used = 0, total = 0, distinct = 0, nz = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    uint64_t ow = T.occ[w];
    if (!ow) continue;
    int64_t i = ro[w];  // rank of this word's first occupied quotient
    int64_t prev = i ? select_global(T.run, rr, nw, i - 1) : -1;
    while (ow) {
      int64_t x = (w << 6) + __ffsll((long long)ow) - 1;
      ow &= ow - 1;
      int64_t end = select_after_dev(T.run, prev, 1, T.phys);
      if (end < 0) { vfail(v, kVRankMismatch, x); return; }
      int64_t st = x > prev + 1 ? x : prev + 1;
      if (x >= logical) vfail(v, kVQuotBeyond, x);
      if (end >= T.phys) vfail(v, kVRunPastPhys, x);
      if (st > end) { vfail(v, kVNegativeRun, x); prev = end; continue; }
      if ((end >> kRegionBits) > (x >> kRegionBits) + 1) vfail(v, kVHardBound, x);
      used += (unsigned long long)(end - st + 1);
      int64_t lastrem = -1;
      for (int64_t p = st; p <= end;) {
        uint64_t h, cnt;
        int64_t nx;
        if (!parse_group_dev<S>(slots, p, end, T.r, &h, &cnt, &nx)) { vfail(v, kVUndecodable, x); break; }
        if ((int64_t)h <= lastrem) vfail(v, kVUnsorted, x);
        lastrem = (int64_t)h;
        total += cnt;
        distinct++;
        for (int64_t j = p; j < nx; j++) nz += slots[j] != 0;
        p = nx;
      }
      prev = end;
    }
  }
  if (used) atomicAdd((unsigned long long *)&v[1], used);
  if (total) atomicAdd((unsigned long long *)&v[2], total);
  if (distinct) atomicAdd((unsigned long long *)&v[3], distinct);
  if (nz) atomicAdd((unsigned long long *)&v[4], nz);
}

// derived spill of every region (gqf.py:452-455) against _offsets
__global__ void k_gqf_validate_offsets(GqfDev T, int64_t nw, const int64_t *__restrict__ ro,
                                       const int64_t *__restrict__ rr, int64_t *__restrict__ v) {
  for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < T.nregions;
       h += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = h << kRegionBits;
    int64_t k = (b >> 6) < nw ? ro[b >> 6] : ro[nw - 1] + __popcll(T.occ[nw - 1]);  // occupied quotients < b
    int64_t derived = 0;
    if (k > 0) {
      int64_t e = select_global(T.run, rr, nw, k - 1);
      derived = e - b + 1 > 0 ? e - b + 1 : 0;
    }
    if (derived != (int64_t)T.offs[h]) vfail(v, kVOffset, h);
  }
}

template <typename S>
__global__ void k_count_nonzero(const S *__restrict__ slots, int64_t n, int64_t *__restrict__ v) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += slots[i] != 0;
  cta_add_u64((unsigned long long *)&v[5], (unsigned long long)c);
}

}  // namespace fk
