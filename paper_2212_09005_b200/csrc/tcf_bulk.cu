#include <stdio.h>
#include <stdlib.h>
#include <string.h>
// tcf_bulk.cu -- bulk two-choice filter on sm_100a.
//
// Replaces the bulk half of the reference kernel contract together with the
// numpy orchestration around it (fk/tcf_bulk.py:133-325):
//   partition            _partition_fps            tcf_bulk.py:133-143
//   phase-1 shortcut     btcf_merge_lists          tcf_bulk.py:191-208, ck:379-405
//   two-choice routing   btcf_route                tcf_bulk.py:210-223, ck:408-444
//   dest-grouped merge   btcf_merge_lists          tcf_bulk.py:225-245
//   backing overflow     backing_insert_batch      tcf_bulk.py:247-255, ck:447-466
//   query                btcf_query_batch          ck:552-599
//   3-pass delete        btcf_delete_blocklocal +  tcf_bulk.py:283-325, ck:482-549
//                        backing_delete_batch
//
// Blocks hold B tag words sorted and front-packed (fill[b] live words, the
// tail EMPTY).  Partitioning is a stable CUB radix sort of (block << f | word)
// over exactly the significant bits, so equal keys keep input order as numpy's
// stable argsort does.  Per-block merges/deletes run one warp per block with
// the block staged in shared memory; output positions come from merge-path
// ranks (lower/upper bounds), so a merge is one pass with no serial loop.
// The reference's routing is a sequential greedy pass over the leftovers; it
// is reproduced exactly by windowed deterministic reservations (a leftover
// commits once it holds the minimum pending index on both of its blocks),
// and the ordered backing inserts/deletes likewise by reservations on probe
// positions.  Every result -- table image, fill, failed keys and their order,
// removed flags, counters -- is bit-identical to the reference.
#include <cub/cub.cuh>

#include "../../include/filterkit_b200.h"
#include "fk_common.cuh"
#include "fk_scratch.cuh"

namespace fk {

namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;

struct BDev {
  void *blocks;
  uint32_t *fill;
  void *backing;
  uint64_t nb;
  FastMod nbm;
  uint64_t bsize;
  FastMod bsm;
  int B, f, cut, probe_limit;
  uint64_t fmask;
  uint64_t seed;
  int keys_are_fps;
};

inline int grid_for(int64_t n, int per = 256) {
  int64_t b = (n + per - 1) / per;
  int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

__device__ __forceinline__ uint64_t key_fp(const BDev &P, uint64_t key) {
  return P.keys_are_fps ? key : mix64(key ^ P.seed);  // tcf_bulk.py:115-117
}

// ---------------------------------------------------------------------------
// partition keys: sort key = (block << f) | word, value = position
// ---------------------------------------------------------------------------
// which: 0 = primary block, 1 = secondary block.  idx == nullptr: items are
// keys[0..n); else items are keys[idx[0..n)] (delete passes over pending keys).
__global__ void k_part_keys(BDev P, const uint64_t *__restrict__ keys, const uint32_t *__restrict__ idx, int64_t n,
                            int which, uint64_t *__restrict__ skey, uint32_t *__restrict__ sval) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t src = idx ? idx[i] : (uint32_t)i;
    uint64_t fp = key_fp(P, keys[src]);
    uint64_t word = remap_tag(fp, P.fmask);
    uint64_t b = fmod64(mix64(fp ^ (which ? kBlock2 : kBlock1)), P.nbm);
    skey[i] = (b << P.f) | word;
    sval[i] = src;
  }
}

// seg_lo/seg_hi[s] = [first, last+1) sorted position of segment s = skey >> f
// (arrays pre-zeroed: absent segments stay empty).
__global__ void k_seg_bounds(const uint64_t *__restrict__ skey, int64_t n, int f, uint32_t *__restrict__ seg_lo,
                             uint32_t *__restrict__ seg_hi) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s = skey[p] >> f;
    if (p == 0 || (skey[p - 1] >> f) != s) seg_lo[s] = (uint32_t)p;
    if (p == n - 1 || (skey[p + 1] >> f) != s) seg_hi[s] = (uint32_t)(p + 1);
  }
}

// ---------------------------------------------------------------------------
// per-block merge (btcf_merge_lists, ck:363-405): one warp per block
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ int lower_bound_s(const T *a, int n, uint32_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if ((uint32_t)a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
template <typename T>
__device__ __forceinline__ int upper_bound_s(const T *a, int n, uint32_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if ((uint32_t)a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t lower_bound_g(const uint64_t *a, int64_t lo, int64_t hi, uint64_t v) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t upper_bound_g(const uint64_t *a, int64_t lo, int64_t hi, uint64_t v) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// phase1 = 1: take = min(len, max(0, cut - fill)) and flag the rest of the
// segment as leftovers (tcf_bulk.py:191-213); phase1 = 0: merge everything.
// Segment s of block b is s = b + seg_off (seg_off = 1 for the dest-grouped
// pass, whose segment 0 is the backing list).  Overflow -> atomicMin(status,
// 1 + b) and the block is left untouched (the reference asserts).
template <typename S>
__global__ void __launch_bounds__(256) k_btcf_merge(BDev P, const uint64_t *__restrict__ skey,
                                                    const uint32_t *__restrict__ seg_lo,
                                                    const uint32_t *__restrict__ seg_hi, int seg_off, int phase1,
                                                    uint8_t *__restrict__ left, unsigned *__restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int B = P.B;
  S *E = reinterpret_cast<S *>(smem_raw) + (size_t)wib * 2 * B;
  S *I = E + B;
  S *blocks = reinterpret_cast<S *>(P.blocks);
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; b < (int64_t)P.nb; b += warps) {
    uint32_t lo = seg_lo[b + seg_off], hi = seg_hi[b + seg_off];
    if (hi <= lo) continue;
    uint32_t span = hi - lo;
    int len = span > 0x7FFFFFFFu ? 0x7FFFFFFF : (int)span;
    int cur = (int)P.fill[b];
    int take = len;
    if (phase1) {
      int room = P.cut - cur;
      room = room < 0 ? 0 : room;
      take = len < room ? len : room;
      for (int64_t p = (int64_t)lo + take + lane; p < hi; p += 32) left[p] = 1;
    }
    if (take == 0) continue;
    if (cur + (int64_t)take > B) {
      if (lane == 0) atomicMin(status, (unsigned)(b + 1));
      continue;
    }
    S *blk = blocks + (uint64_t)b * B;
    for (int i = lane; i < cur; i += 32) E[i] = blk[i];
    for (int j = lane; j < take; j += 32) I[j] = (S)(skey[lo + j] & P.fmask);
    __syncwarp();
    // stable merge of [existing, incoming]: existing first on ties
    for (int i = lane; i < cur; i += 32) blk[i + lower_bound_s(I, take, (uint32_t)E[i])] = E[i];
    for (int j = lane; j < take; j += 32) blk[j + upper_bound_s(E, cur, (uint32_t)I[j])] = I[j];
    if (lane == 0) P.fill[b] = (uint32_t)(cur + take);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// per-block delete (btcf_delete_blocklocal, ck:482-512): one warp per block
// ---------------------------------------------------------------------------
// Sequential semantics per block: each sorted item removes one stored copy
// of its word if one is left.  For a word w requested q_w times and stored
// c_w times, the first min(q_w, c_w) requests (in sorted order) hit and
// min(q_w, c_w) copies go; the block is then re-packed.
template <typename S>
__global__ void __launch_bounds__(256) k_btcf_delete(BDev P, const uint64_t *__restrict__ skey,
                                                     const uint32_t *__restrict__ sval,
                                                     const uint32_t *__restrict__ seg_lo,
                                                     const uint32_t *__restrict__ seg_hi, uint8_t *__restrict__ hit,
                                                     uint8_t *__restrict__ removed) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int B = P.B;
  S *E = reinterpret_cast<S *>(smem_raw) + (size_t)wib * B;
  S *blocks = reinterpret_cast<S *>(P.blocks);
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; b < (int64_t)P.nb; b += warps) {
    int64_t lo = seg_lo[b], hi = seg_hi[b];
    if (hi <= lo) continue;
    int cur = (int)P.fill[b];
    if (cur > B) cur = B;
    S *blk = blocks + (uint64_t)b * B;
    for (int i = lane; i < cur; i += 32) E[i] = blk[i];
    __syncwarp();
    const uint64_t bkey = (uint64_t)b << P.f;
    // requests
    for (int64_t k = lo + lane; k < hi; k += 32) {
      uint32_t w = (uint32_t)(skey[k] & P.fmask);
      int64_t r = k - lower_bound_g(skey, lo, k, bkey | w);
      int c = upper_bound_s(E, cur, w) - lower_bound_s(E, cur, w);
      uint8_t h = r < c ? 1 : 0;
      hit[k] = h;
      if (h) removed[sval[k]] = 1;
    }
    // stored copies: drop the first min(q_w, c_w) of each word, re-pack
    int base = 0;
    for (int i0 = 0; i0 < cur; i0 += 32) {
      int i = i0 + lane;
      bool keep = false;
      S w = 0;
      if (i < cur) {
        w = E[i];
        int j = i - lower_bound_s(E, cur, (uint32_t)w);
        int64_t q = upper_bound_g(skey, lo, hi, bkey | (uint32_t)w) - lower_bound_g(skey, lo, hi, bkey | (uint32_t)w);
        keep = (int64_t)j >= q;
      }
      unsigned bal = __ballot_sync(0xFFFFFFFFu, keep);
      if (keep) blk[base + __popc(bal & ((1u << lane) - 1u))] = w;
      base += __popc(bal);
    }
    __syncwarp();
    for (int i = base + lane; i < cur; i += 32) blk[i] = (S)0;
    if (lane == 0) P.fill[b] = (uint32_t)base;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// query (btcf_query_batch, ck:552-599): G lanes per key (btcf_query picks
// G from the block size), each loading its share of the block's 32-byte
// sectors.  The block's sorted prefix is followed by EMPTY (0)
// slots and words are >= 2, so "bisect hit in the prefix" == "some slot of
// the block equals the word".
// ---------------------------------------------------------------------------
template <typename S>
__device__ __forceinline__ bool sector_has(const uint32_t (&r)[8], uint32_t word) {
  if constexpr (sizeof(S) == 2) {
    uint32_t pat = word | (word << 16);
    unsigned m = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) m |= __vcmpeq2(r[i], pat);
    return m != 0;
  } else if constexpr (sizeof(S) == 1) {
    uint32_t pat = word * 0x01010101u;
    unsigned m = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) m |= __vcmpeq4(r[i], pat);
    return m != 0;
  } else {
    bool h = false;
#pragma unroll
    for (int i = 0; i < 8; i++) h |= r[i] == word;
    return h;
  }
}

template <typename S, int G>
__global__ void __launch_bounds__(256) k_btcf_query(BDev P, const uint64_t *__restrict__ keys, int64_t n,
                                                    uint8_t *__restrict__ found) {
  const unsigned lane = threadIdx.x & 31, sub = lane % G, base = lane - sub;
  const unsigned mask = (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u)) << base;
  const S *blocks = reinterpret_cast<const S *>(P.blocks);
  const S *backing = reinterpret_cast<const S *>(P.backing);
  const int64_t bytes = (int64_t)P.B * sizeof(S);
  const bool vec = (bytes % 32) == 0;
  const int sectors = (int)((bytes + 31) / 32);
  const int64_t tiles = (int64_t)gridDim.x * (blockDim.x / G);
  const int64_t first = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  // warp-uniform trip count: every lane of the warp takes part in the ballots
  const int64_t nround = (n + tiles - 1) / tiles;
  for (int64_t it = 0; it < nround; it++) {
    int64_t i = first + it * tiles;
    bool valid = i < n;
    uint64_t fp = valid ? key_fp(P, keys[i]) : 0;
    uint32_t word = (uint32_t)remap_tag(fp, P.fmask);
    bool hit = false;
#pragma unroll 1
    for (int which = 0; which < 2; which++) {
      bool h = false;
      if (valid && !hit) {
        uint64_t b = fmod64(mix64(fp ^ (which ? kBlock2 : kBlock1)), P.nbm);
        const S *blk = blocks + b * (uint64_t)P.B;
        if (vec) {
#pragma unroll 8
          for (int s = (int)sub; s < sectors; s += G) {
            uint32_t r[8];
            load_chunk<32, false>(reinterpret_cast<const char *>(blk) + 32 * s, r);
            h |= sector_has<S>(r, word);
          }
        } else {
          for (int j = (int)sub; j < P.B; j += G) h |= (uint32_t)blk[j] == word;
        }
      }
      hit = hit || (__ballot_sync(0xFFFFFFFFu, h) & mask) != 0;
    }
    if (valid && !hit && P.bsize && sub == 0) {  // backing chain (ck:581-592)
      uint64_t p = fmod64(mix64(fp ^ kBackStart), P.bsm);
      uint64_t step = fmod64(mix64(fp ^ kBackStep) | 1, P.bsm);
      for (int q = 0; q < P.probe_limit; q++) {
        uint64_t w = backing[p];
        if (w == 0) break;
        if (w != 1 && (w & P.fmask) == word) {
          hit = true;
          break;
        }
        p += step;
        p = p >= P.bsize ? p - P.bsize : p;
      }
    }
    if (valid && sub == 0) found[i] = hit ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// sequential two-choice routing (btcf_route, ck:408-444)
// ---------------------------------------------------------------------------
// The reference routes the leftovers one by one in (b1, word) order, each
// decision reading the committed load of both candidate blocks.  Sorted by
// b1, consecutive leftovers share a block, so the dependency chain is long
// (6405 deep for a 0.9-load batch into 2^20 slots) and parallel
// reservations would need thousands of grid-wide rounds.  The walk is
// therefore one warp: the per-block load counters live in shared memory
// (global memory when nb does not fit), leftovers stream in through
// coalesced 32-wide loads, and the next leftover's two counters are fetched
// before the current decision is written back and patched in registers
// (store-to-load forwarding), so the chain costs one short dependent step
// per leftover.
template <bool SMEM>
__global__ void __launch_bounds__(32) k_btcf_route_seq(const uint32_t *__restrict__ lb1,
                                                       const uint32_t *__restrict__ lb2, int64_t m,
                                                       const uint32_t *__restrict__ fill, uint64_t nb,
                                                       uint32_t *__restrict__ gload, uint32_t B,
                                                       int32_t *__restrict__ dest) {
  // Every lane runs the identical walk on broadcast reads and stores the same
  // value, so each lane's next read sees its own store: no cross-lane
  // synchronisation on the chain.  Counters for leftovers j+1 and j+2 are
  // read ahead and patched with the decisions of j (and j+1).
  extern __shared__ uint32_t sload[];
  uint32_t *load = SMEM ? sload : gload;
  const unsigned lane = threadIdx.x;
  if (SMEM) {
    for (uint64_t i = lane; i < nb; i += 32) sload[i] = fill[i];
    __syncwarp();
  }
  if (m <= 0) return;
  uint32_t ca = lane < m ? lb1[lane] : 0, cb = lane < m ? lb2[lane] : 0;
  uint32_t na = 32 + lane < m ? lb1[32 + lane] : 0, nb2 = 32 + lane < m ? lb2[32 + lane] : 0;
  // pipeline registers: (a, b, la, lb) for the current leftover and the next
  uint32_t a0 = __shfl_sync(0xFFFFFFFFu, ca, 0), b0 = __shfl_sync(0xFFFFFFFFu, cb, 0);
  uint32_t l0a = load[a0], l0b = load[b0];
  uint32_t a1 = __shfl_sync(0xFFFFFFFFu, ca, 1 & 31), b1 = __shfl_sync(0xFFFFFFFFu, cb, 1 & 31);
  uint32_t l1a = load[a1], l1b = load[b1];
  int32_t mine = 0;
  // one leftover: decide k, forward the write into the read-ahead slots and
  // read ahead leftover k + 2 (whose blocks are a2/b2)
  // Decision (ck:429-442): pick = b1 if load(b1) <= load(b2) else b2; if the
  // pick is full try the other; both full -> backing.  Since the pick holds
  // the smaller load, "pick full" implies "both full", so the rule is: the
  // smaller-load block (tie -> b1) unless min(load) >= B.  Written branch-free
  // to keep the loop-carried chain short.
  auto step = [&](int j, uint32_t a2, uint32_t b2) {
    uint32_t l2a = load[a2], l2b = load[b2];  // read ahead (a2/b2 are 0 past the end)
    const bool pa = l0a <= l0b;
    const uint32_t lp = pa ? l0a : l0b;
    const uint32_t dsel = pa ? a0 : b0;
    const bool ok = lp < B;
    const uint32_t v = lp + 1;
    if (ok) load[dsel] = v;
    const uint32_t dd = ok ? dsel : 0xFFFFFFFFu;
    l1a = a1 == dd ? v : l1a;
    l1b = b1 == dd ? v : l1b;
    l2a = a2 == dd ? v : l2a;
    l2b = b2 == dd ? v : l2b;
    if ((int)lane == j) mine = ok ? (int32_t)dsel : -1;
    a0 = a1; b0 = b1; l0a = l1a; l0b = l1b;
    a1 = a2; b1 = b2; l1a = l2a; l1b = l2b;
  };
  // one chunk of 32 leftovers: j + 2 < 32 come from the chunk's registers
  // (xa, xb), the last two from the next chunk's (ya, yb)
  auto chunk = [&](int64_t base, uint32_t xa, uint32_t xb, uint32_t ya, uint32_t yb) {
    const int cnt = m - base < 32 ? (int)(m - base) : 32;
    for (int j = 0; j < 30 && j < cnt; j++)
      step(j, __shfl_sync(0xFFFFFFFFu, xa, j + 2), __shfl_sync(0xFFFFFFFFu, xb, j + 2));
    for (int j = 30; j < cnt; j++)
      step(j, __shfl_sync(0xFFFFFFFFu, ya, j - 30), __shfl_sync(0xFFFFFFFFu, yb, j - 30));
    if (base + lane < m) dest[base + lane] = mine;
  };
  // Two chunks per trip with the register sets swapping roles: every
  // leftover load lands in a register first read a whole chunk later (a
  // rotating copy at the loop head would wait for the load just issued).
  for (int64_t base = 0; base < m; base += 64) {
    chunk(base, ca, cb, na, nb2);
    ca = base + 64 + lane < m ? lb1[base + 64 + lane] : 0;
    cb = base + 64 + lane < m ? lb2[base + 64 + lane] : 0;
    if (base + 32 >= m) break;
    chunk(base + 32, na, nb2, ca, cb);
    na = base + 96 + lane < m ? lb1[base + 96 + lane] : 0;
    nb2 = base + 96 + lane < m ? lb2[base + 96 + lane] : 0;
  }
}

// Block-parallel form of the same walk for large tables (bit-identical
// decisions).  One 1024-thread CTA takes the next 1024 leftovers; a leftover
// whose b2 (or b1) meets an earlier leftover's other block inside the window
// ends the window's conflict-free prefix (found with a shared-memory table of
// first touches); inside the prefix the only dependencies left are the b1
// groups (leftovers are sorted by b1), so every b2 counter is read once in
// parallel and each group's head runs the group's one-register scan
// x <- x + [x <= min(y, B - 1)].  Prefixes are ~sqrt(blocks) long, so this
// pays off on large tables only (the caller keeps the warp walk below 2^16
// blocks).
constexpr int kRouteW = 1024, kRouteHT = 4096;
constexpr size_t kRouteSmem = (size_t)kRouteHT * 12 + (size_t)kRouteW * 12 + (size_t)kRouteW * 16;

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__global__ void __launch_bounds__(kRouteW, 1) k_btcf_route_prefix(const uint32_t *__restrict__ lb1,
                                                                  const uint32_t *__restrict__ lb2, int64_t m,
                                                                  uint32_t *__restrict__ load, uint32_t B,
                                                                  int32_t *__restrict__ dest) {
  extern __shared__ uint32_t route_smem[];  // kRouteSmem bytes (dynamic: > 48 KB)
  uint32_t *ht_key = route_smem;
  int *ht_a = reinterpret_cast<int *>(ht_key + kRouteHT), *ht_b = ht_a + kRouteHT;
  uint32_t *s_y = reinterpret_cast<uint32_t *>(ht_b + kRouteHT), *s_a = s_y + kRouteW;
  int32_t *s_d = reinterpret_cast<int32_t *>(s_a + kRouteW);
  // ring of the next 2W leftovers (b1, b2): slot i % 2W holds leftover i;
  // refilled with cp.async a window ahead of use
  uint32_t *ring_a = reinterpret_cast<uint32_t *>(s_d + kRouteW), *ring_b = ring_a + 2 * kRouteW;
  __shared__ int s_first;
  const int k = threadIdx.x;
  constexpr int RM = 2 * kRouteW - 1;
  auto slot = [&](uint32_t blk) {  // insert-or-find in the open-addressed table
    uint32_t h = (blk * 2654435761u) & (kRouteHT - 1);
    for (;;) {
      uint32_t prev = atomicCAS(&ht_key[h], 0xFFFFFFFFu, blk);
      if (prev == 0xFFFFFFFFu || prev == blk) return h;
      h = (h + 1) & (kRouteHT - 1);
    }
  };
  for (int i = k; i < 2 * kRouteW && i < m; i += kRouteW) {
    cp_async4(&ring_a[i], lb1 + i);
    cp_async4(&ring_b[i], lb2 + i);
  }
  cp_async_commit();
  cp_async_commit();  // (an empty group: the loop waits for all but the newest)
  for (int64_t base = 0; base < m;) {
    const int cnt = m - base < kRouteW ? (int)(m - base) : kRouteW;
    cp_async_wait1();
    for (int i = k; i < kRouteHT; i += kRouteW) {
      ht_key[i] = 0xFFFFFFFFu;
      ht_a[i] = ht_b[i] = kRouteW;
    }
    if (k == 0) s_first = cnt;
    __syncthreads();
    const bool live = k < cnt;
    uint32_t a = 0, b = 0, ha = 0, hb = 0, y = 0, x0 = 0;
    if (live) {
      a = ring_a[(base + k) & RM];
      b = ring_b[(base + k) & RM];
      y = load[b];   // issued before the conflict test; valid for prefix members
      x0 = load[a];  // (no prefix leftover but its own group touches either)
      ha = slot(a);
      hb = slot(b);
      atomicMin(&ht_a[ha], k);
      atomicMin(&ht_b[hb], k);
    }
    __syncthreads();
    // conflict: b = an earlier a or b, a = an earlier b, or b = own a
    if (live && (b == a || ht_a[hb] < k || ht_b[hb] < k || ht_b[ha] < k)) atomicMin(&s_first, k);
    __syncthreads();
    const int first = s_first;
    int adv;
    if (first == 0) {  // leftover 0 alone (b1 == b2): the plain rule
      if (k == 0) {
        const uint32_t la = load[a], lbv = load[b];
        const bool pa = la <= lbv;
        const uint32_t lp = pa ? la : lbv, d = pa ? a : b;
        if (lp < B) load[d] = lp + 1;
        dest[base] = lp < B ? (int32_t)d : -1;
      }
      adv = 1;
    } else {
      const bool act = k < first;
      if (act) {
        s_y[k] = y;
        s_a[k] = a;
      }
      __syncthreads();
      // group heads scan their group in order
      if (act && (k == 0 || s_a[k - 1] != a)) {
        uint32_t x = x0;
        for (int j = k; j < first && s_a[j] == a; j++) {
          const uint32_t yj = s_y[j];
          const uint32_t t = yj < B - 1 ? yj : B - 1;
          if (x <= t) {
            s_d[j] = (int32_t)a;
            x++;
          } else {
            s_d[j] = yj < B ? -2 : -1;  // -2: takes its b2 (x > y)
          }
        }
        load[a] = x;
      }
      __syncthreads();
      if (act) {
        int32_t d = s_d[k];
        if (d == -2) {
          load[b] = y + 1;  // b is touched by no other leftover of the prefix
          d = (int32_t)b;
        }
        dest[base + k] = d;
      }
      adv = first;
    }
    // refill the consumed ring slots with leftovers [base + 2W, base + 2W + adv)
    if (k < adv && base + 2 * kRouteW + k < m) {
      const int64_t i = base + 2 * kRouteW + k;
      cp_async4(&ring_a[i & RM], lb1 + i);
      cp_async4(&ring_b[i & RM], lb2 + i);
    }
    cp_async_commit();
    __syncthreads();
    base += adv;
  }
}

// ---------------------------------------------------------------------------
// parallel two-choice routing by fixpoint iteration (btcf_route, ck:408-444)
// ---------------------------------------------------------------------------
// Item k (in the walk's order) decides d_k = rule(L(a_k, k), L(b_k, k)) with
// L(X, k) = fill[X] + #{j < k : d_j = X} and rule = the smaller load (tie ->
// a) unless it is >= B (-> -1).  d_0 depends on fill alone and d_k on
// d_0..d_{k-1} only, so the system has exactly one solution: the sequential
// walk's decisions.  Jacobi sweeps (recompute every d_k from the previous
// iterate's counts) reach it -- after t sweeps at least the first t decisions
// are final -- and in practice the iterate stops changing after ~50 sweeps at
// every table size measured (2^20..2^24 slots): a decision flips only while
// its two loads are within the perturbation of the counts.  A sweep is two
// exclusive prefix sums and one elementwise pass:
//   P1 over the (a, index)-sorted order of c1_j = [d_j == a_j]
//   P2 over the (b, index)-sorted order of c2_j = [d_j == b_j != a_j]
//   L(a_k, k) = fill[a_k] + P1[pos1_k] - P1[s1[a_k]] + P2[qA_k] - P2[s2[a_k]]
//   L(b_k, k) = fill[b_k] + P1[qB_k] - P1[s1[b_k]] + P2[pos2_k] - P2[s2[b_k]]
// where pos1/pos2 place item k in the two orders, s1/s2 start each block's
// segment there, qA_k is the first position of b-order segment a_k holding
// an index >= k, and qB_k likewise in a-order segment b_k.  Stopping rule:
// a sweep that changes no decision has found the fixpoint.  One cooperative
// kernel runs the sweeps (two grid barriers each); if it has not converged
// after kJacobiMax sweeps the caller runs the sequential walk instead.
constexpr int kJT = 256, kJItems = 1, kJTile = kJT * kJItems, kJacobiMax = 4096;
constexpr int kJHeld = 2;  // items a thread keeps in registers across the sweeps
// With few tiles the tile sums live 256 bytes apart: the L2 slice of an
// address is chosen from bit 8 up, so packed counters put every tile's
// atomics on a few slices (measured at 2^20 slots: the decision pass was
// bound by them, 17.8 -> 7.9 us per sweep).  With many tiles they stay
// packed: every tile's offset sums all earlier tile sums (O(T^2) reads),
// which strided counters would turn into one sector each (2^24: 2x slower).
constexpr int kTsStride = 64, kTsStrideMaxTiles = 4096;
// never a decision (decisions are a block index or -1)
constexpr uint32_t kNoB = 0xFFFFFFFEu;

// Per item, everything a sweep reads besides the two prefix arrays is
// static, so it is gathered once: the eight P-array positions of the two
// loads (own position / segment start in each order, for each block) and
// the committed fills.
struct RouteItem {
  uint4 p;  // P1 pos (a), P1 seg start (a), P2 pos (a), P2 seg start (a)
  uint4 q;  // P1 pos (b), P1 seg start (b), P2 pos (b), P2 seg start (b)
  uint4 c;  // a, b, fill[a], fill[b]
};

struct RouteJ {
  const RouteItem *it;        // [m] item order
  const uint32_t *perm1;      // [m] a-order position -> item
  const uint32_t *perm2;      // [m] b-order position -> item
  const uint32_t *a_of1;      // [m] a of the item at a-order position p
  const uint32_t *b_of2;      // [m] b of the item at b-order position p, or kNoB when its a == b
  const uint32_t *pos1, *pos2;  // [m] item -> positions (tile of its flags)
  int32_t *d;                 // [m] decisions (in/out)
  uint32_t *P1, *P2;          // [m + 1] exclusive prefix sums
  uint32_t *ts;               // [2 parities][2 orders][T] tile sums, tss apart
  int tss;                    // tile-sum stride (kTsStride or 1)
  unsigned *ctl;              // [3] sweeps run, [4] converged
  unsigned *chg;              // [gridDim] this CTA's decisions changed in the last sweep
  unsigned long long *clk;    // optional (FK_ROUTE_STATS): globaltimer at each phase end, CTA 0
  int64_t m;
  int T;
  uint32_t B;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int32_t route_rule(uint32_t l1, uint32_t l2, uint32_t a, uint32_t b, uint32_t B) {
  const bool pa = l1 <= l2;
  const uint32_t lp = pa ? l1 : l2;
  return lp < B ? (int32_t)(pa ? a : b) : -1;
}

// tile sums of the flags of decision d (warp-aggregated per tile)
__device__ __forceinline__ void route_tally(const RouteJ &R, uint32_t *tsn, bool live, int32_t d, uint32_t a,
                                            uint32_t b, uint32_t p1, uint32_t p2) {
  const bool c1 = live && d == (int32_t)a, c2 = live && !c1 && d == (int32_t)b;
  const unsigned act = __ballot_sync(0xFFFFFFFFu, c1 || c2);
  if (!(c1 || c2)) return;
  const uint32_t slot = c1 ? p1 / kJTile : (uint32_t)R.T + p2 / kJTile;
  const unsigned peers = __match_any_sync(act, slot);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&tsn[(size_t)slot * R.tss], (unsigned)__popc(peers));
}

__global__ void __launch_bounds__(kJT, 3) k_btcf_route_jacobi(RouteJ R) {
  cg::grid_group grid = cg::this_grid();
  typedef cub::BlockScan<unsigned long long, kJT> Scan;
  typedef cub::BlockReduce<unsigned long long, kJT> Red;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Red::TempStorage red;
  } tmp;
  __shared__ unsigned long long s_off;
  const int64_t m = R.m;
  const int T = R.T;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t mr = (m + 31) & ~(int64_t)31;  // warp-uniform trip counts (ballots below)
  // sweep 0's iterate: the rule on the committed fills alone, with its tile sums
  for (int64_t k = tid; k < mr; k += nth) {
    const bool live = k < m;
    uint4 c = make_uint4(0, 0, 0, 0);
    uint32_t p1 = 0, p2 = 0;
    int32_t d = -1;
    if (live) {
      c = R.it[k].c;
      p1 = R.pos1[k];
      p2 = R.pos2[k];
      d = route_rule(c.z, c.w, c.x, c.y, R.B);
      R.d[k] = d;
    }
    route_tally(R, R.ts, live, d, c.x, c.y, p1, p2);
  }
  grid.sync();
  // items held in registers across the sweeps when every thread has at most
  // kJHeld of them: their static positions and their last decision
  const bool held = m <= kJHeld * nth;
  RouteItem hit[kJHeld];
  int32_t hd[kJHeld];
#pragma unroll
  for (int u = 0; u < kJHeld; u++) {
    const int64_t k = tid + u * nth;
    if (held && k < m) {
      hit[u] = R.it[k];
      hd[u] = __ldcg(&R.d[k]);
    } else {
      hit[u].p = hit[u].q = hit[u].c = make_uint4(0, 0, 0, 0);
      hd[u] = -1;
    }
  }
  if (R.clk && tid == 0) R.clk[0] = gtimer();
  for (unsigned sweep = 0;; sweep++) {
    const int par = sweep & 1;
    uint32_t *ts = R.ts + (size_t)par * 2 * T * R.tss, *tsn = R.ts + (size_t)(par ^ 1) * 2 * T * R.tss;
    // ---- phase S: P1, P2 of the current iterate (tile scans + tile offsets)
    for (int64_t i = tid; i < 2 * (int64_t)T; i += nth) tsn[i * R.tss] = 0;
    unsigned long long off_acc = 0;  // (thread 0) sum of the tile sums before this CTA's current tile
    int done_to = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      // offsets: sums of the tile sums before t, both orders packed (P1 << 32 | P2),
      // accumulated over this CTA's tiles so every tile sum is read once per CTA
      unsigned long long part = 0;
      for (int u = done_to + threadIdx.x; u < t; u += kJT)
        part += ((unsigned long long)__ldcg(&ts[(size_t)u * R.tss]) << 32) | __ldcg(&ts[(size_t)(T + u) * R.tss]);
      const unsigned long long add = Red(tmp.red).Sum(part);
      done_to = t;
      if (threadIdx.x == 0) {
        off_acc += add;
        s_off = off_acc;
      }
      __syncthreads();
      unsigned long long off = s_off;
      unsigned long long v[kJItems];
      const int64_t p0 = (int64_t)t * kJTile + (int64_t)threadIdx.x * kJItems;
      uint32_t i1[kJItems], i2[kJItems];
#pragma unroll
      for (int j = 0; j < kJItems; j++) {
        const int64_t p = p0 + j;
        i1[j] = p < m ? R.perm1[p] : 0;
        i2[j] = p < m ? R.perm2[p] : 0;
      }
#pragma unroll
      for (int j = 0; j < kJItems; j++) {
        const int64_t p = p0 + j;
        unsigned long long c = 0;
        if (p < m) {
          const int32_t d1 = __ldcg(&R.d[i1[j]]), d2 = __ldcg(&R.d[i2[j]]);
          c = ((unsigned long long)(d1 == (int32_t)R.a_of1[p]) << 32) | (unsigned long long)(d2 == (int32_t)R.b_of2[p]);
        }
        v[j] = c;
      }
      unsigned long long tot;
      Scan(tmp.scan).ExclusiveSum(v, v, tot);
#pragma unroll
      for (int j = 0; j < kJItems; j++) {
        const int64_t p = p0 + j;
        if (p < m) {
          const unsigned long long x = v[j] + off;
          R.P1[p] = (uint32_t)(x >> 32);
          R.P2[p] = (uint32_t)x;
        }
      }
      if (t == T - 1 && threadIdx.x == 0) {  // the totals
        const unsigned long long x = tot + off;
        R.P1[m] = (uint32_t)(x >> 32);
        R.P2[m] = (uint32_t)x;
      }
      __syncthreads();
    }
    if (R.clk && tid == 0 && sweep < 64) R.clk[1 + 3 * sweep] = gtimer();
    grid.sync();
    if (R.clk && tid == 0 && sweep < 64) R.clk[2 + 3 * sweep] = gtimer();
    // ---- phase D: every decision from the counts of the current iterate
    unsigned changed = 0;
    if (held) {
      // the thread's items are in registers since sweep 0: the sixteen P
      // reads of its two items go out together (one dependent trip)
      uint32_t v[kJHeld][8];
#pragma unroll
      for (int u = 0; u < kJHeld; u++) {
        if (tid + u * nth < m) {
          v[u][0] = __ldcg(&R.P1[hit[u].p.x]);
          v[u][1] = __ldcg(&R.P1[hit[u].p.y]);
          v[u][2] = __ldcg(&R.P2[hit[u].p.z]);
          v[u][3] = __ldcg(&R.P2[hit[u].p.w]);
          v[u][4] = __ldcg(&R.P1[hit[u].q.x]);
          v[u][5] = __ldcg(&R.P1[hit[u].q.y]);
          v[u][6] = __ldcg(&R.P2[hit[u].q.z]);
          v[u][7] = __ldcg(&R.P2[hit[u].q.w]);
        }
      }
#pragma unroll
      for (int u = 0; u < kJHeld; u++) {
        const int64_t k = tid + u * nth;
        if (k >= mr) break;  // warp-uniform
        const bool live = k < m;
        int32_t d = -1;
        const uint4 c = hit[u].c;
        if (live) {
          const uint32_t l1 = c.z + (v[u][0] - v[u][1]) + (v[u][2] - v[u][3]);
          const uint32_t l2 = c.w + (v[u][4] - v[u][5]) + (v[u][6] - v[u][7]);
          d = route_rule(l1, l2, c.x, c.y, R.B);
          if (d != hd[u]) {
            R.d[k] = d;
            hd[u] = d;
            changed++;
          }
        }
        route_tally(R, tsn, live, d, c.x, c.y, hit[u].p.x, hit[u].q.z);
      }
    }
    // (more items than threads can hold: stream them)
    constexpr int U = 1;
    for (int64_t k0 = held ? mr : tid; k0 < mr; k0 += U * nth) {
      RouteItem it[U];
      int32_t dold[U];
      uint32_t v[U][8];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t k = k0 + u * nth;
        if (k < m) {
          it[u] = R.it[k];
          dold[u] = R.d[k];
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (k0 + u * nth < m) {
          v[u][0] = __ldcg(&R.P1[it[u].p.x]);
          v[u][1] = __ldcg(&R.P1[it[u].p.y]);
          v[u][2] = __ldcg(&R.P2[it[u].p.z]);
          v[u][3] = __ldcg(&R.P2[it[u].p.w]);
          v[u][4] = __ldcg(&R.P1[it[u].q.x]);
          v[u][5] = __ldcg(&R.P1[it[u].q.y]);
          v[u][6] = __ldcg(&R.P2[it[u].q.z]);
          v[u][7] = __ldcg(&R.P2[it[u].q.w]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t k = k0 + u * nth;
        if (k >= mr) break;  // warp-uniform (mr and nth are multiples of 32)
        const bool live = k < m;
        int32_t d = -1;
        uint4 c = make_uint4(0, 0, 0, 0);
        uint32_t p1 = 0, p2 = 0;
        if (live) {
          c = it[u].c;
          p1 = it[u].p.x;
          p2 = it[u].q.z;
          const uint32_t l1 = c.z + (v[u][0] - v[u][1]) + (v[u][2] - v[u][3]);
          const uint32_t l2 = c.w + (v[u][4] - v[u][5]) + (v[u][6] - v[u][7]);
          d = route_rule(l1, l2, c.x, c.y, R.B);
          if (d != dold[u]) {
            R.d[k] = d;
            changed++;
          }
        }
        route_tally(R, tsn, live, d, c.x, c.y, p1, p2);
      }
    }
    // one flag per CTA (a single counter would take ~5K same-address atomics
    // per sweep); each CTA ORs all flags after the barrier.  A CTA rewrites
    // its flag only in the next phase D, after every CTA has read it (they
    // all pass the phase-S barrier in between).
    const int any = __syncthreads_or(changed != 0);
    if (threadIdx.x == 0) R.chg[blockIdx.x] = (unsigned)any;
    if (R.clk && threadIdx.x == 0 && sweep < 64) {
      // slowest CTA's phase-D work (start = CTA 0's post-barrier time)
      const unsigned long long w = gtimer();
      atomicMax(&R.clk[1 + 3 * 64 + sweep], w);
    }
    grid.sync();
    if (R.clk && tid == 0 && sweep < 64) R.clk[3 + 3 * sweep] = gtimer();
    unsigned mine = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) mine |= __ldcg(&R.chg[i]);
    const unsigned cc = (unsigned)__syncthreads_or(mine != 0);
    if (cc == 0 || sweep + 1 >= (unsigned)kJacobiMax) {
      if (tid == 0) {
        R.ctl[3] = sweep + 1;
        R.ctl[4] = cc == 0 ? 1u : 0u;
      }
      return;
    }
  }
}

// ---------------------------------------------------------------------------
// The same fixpoint with the counts kept per block (default router).
// L(X, k) only counts earlier decisions for X among the items that list X:
// block X's a-segment (items with a = X, by index) and b-segment (b = X != a).
// One warp owns block X and, per sweep, (1) recomputes the decision of each
// item in its two segments from the loads the previous sweep left for that
// item -- d_k = rule(LA[k], LB[k]) -- and ballots the flags [d_j == X], then
// (2) writes every segment item's new load on X: fill[X] + the flagged items
// of both segments with a smaller index (own-segment prefix + the other
// segment's prefix at the item's static rank there).  d^t = rule(L(d^{t-1}))
// is the Jacobi iterate of k_btcf_route_jacobi with no global prefix sums and
// one grid barrier per sweep (loads double-buffered by sweep parity); the
// a-owner of an item keeps its decision and flags changes.
#ifndef FK_RB_MINB
#define FK_RB_MINB 4
#endif
constexpr int kRBT = 256, kRBWarps = kRBT / 32, kRBMaxWords = 32;  // segments up to 1024 items
struct RouteBJ {
  const uint4 *st1;           // [m] a-order position: item, b, rank in b-segment a, -
  const uint4 *st2;           // [m] b-order position: item, a, rank in a-segment b, -
  const uint32_t *s1, *e1, *s2, *e2;  // [nb] segment bounds in the two orders
  const uint32_t *fill;       // [nb]
  const uint32_t *a, *b;      // [m]
  uint32_t *LA[2], *LB[2];    // [m] loads of each item on its a / b block, by sweep parity
  int32_t *d;                 // [m] decisions (out; pre-set to a non-decision)
  unsigned *ctl;              // [3] sweeps, [4] converged (2 = segment too long), [5] too-long flag
  unsigned *chg;              // [2][gridDim]
  int64_t m;
  int64_t nb;
  uint32_t B;
};

__device__ __forceinline__ uint32_t seg_prefix(const uint32_t *w, const uint32_t *pre, uint32_t q) {
  return pre[q >> 5] + (uint32_t)__popc(w[q >> 5] & ((1u << (q & 31)) - 1u));
}

// One block's static data: segment bounds, fill, and the first chunk of each
// segment (lane i: entry i) -- a warp keeps this in registers across the
// sweeps for its first kRBHold blocks.
struct RBlk {
  uint32_t x, s1x, nA, s2x, nB, fx;
  uint4 eA0, eB0;
};

__device__ __forceinline__ RBlk rb_load(const RouteBJ &R, int64_t X, int lane) {
  RBlk h;
  const uint4 z4 = make_uint4(0, 0, 0, 0);
  h.x = (uint32_t)X;
  if (X < R.nb) {
    h.s1x = R.s1[X];
    h.nA = R.e1[X] - h.s1x;
    h.s2x = R.s2[X];
    h.nB = R.e2[X] - h.s2x;
    h.fx = R.fill[X];
  } else {
    h.s1x = h.nA = h.s2x = h.nB = h.fx = 0;
  }
  h.eA0 = lane < (int)h.nA ? R.st1[h.s1x + lane] : z4;
  h.eB0 = lane < (int)h.nB ? R.st2[h.s2x + lane] : z4;
  return h;
}

// The previous loads of the first chunks' items (one dependent trip).
struct RBLoads {
  uint32_t la0, lb0, la1, lb1;
  int32_t dold;
};

__device__ __forceinline__ RBLoads rb_fetch(const RouteBJ &R, const RBlk &h, const uint32_t *LAp, const uint32_t *LBp,
                                            int lane) {
  RBLoads v = {0, 0, 0, 0, 0};
  if (lane < (int)h.nA) {
    v.la0 = __ldcg(&LAp[h.eA0.x]);
    v.lb0 = __ldcg(&LBp[h.eA0.x]);
    v.dold = R.d[h.eA0.x];
  }
  if (lane < (int)h.nB && h.eB0.y != h.x) {
    v.la1 = __ldcg(&LAp[h.eB0.x]);
    v.lb1 = __ldcg(&LBp[h.eB0.x]);
  }
  return v;
}

// One sweep's work on one block (see k_btcf_route_blocks).
__device__ __forceinline__ void rb_sweep(const RouteBJ &R, const RBlk &h, const RBLoads &v, const uint32_t *LAp,
                                         const uint32_t *LBp, uint32_t *LAn, uint32_t *LBn, uint32_t *wA,
                                         uint32_t *wB, uint32_t *pA, uint32_t *pB, int lane, unsigned &changed) {
  const uint32_t x = h.x, nA = h.nA, nB = h.nB, s1x = h.s1x, s2x = h.s2x;
  const uint32_t nwA = (nA + 31) >> 5, nwB = (nB + 31) >> 5;
  const bool vA = lane < (int)nA, uB = lane < (int)nB && h.eB0.y != x;  // a == b counts in the a-segment only
  // (1) decisions and flags
  {
    bool fl = false;
    if (vA) {
      const int32_t dk = route_rule(v.la0, v.lb0, x, h.eA0.y, R.B);
      fl = dk == (int32_t)x;
      if (dk != v.dold) {
        R.d[h.eA0.x] = dk;
        changed = 1;
      }
    }
    const unsigned w = __ballot_sync(0xFFFFFFFFu, fl);
    const unsigned wb = __ballot_sync(0xFFFFFFFFu, uB && route_rule(v.la1, v.lb1, h.eB0.y, x, R.B) == (int32_t)x);
    if (lane == 0) {
      wA[0] = w;
      wB[0] = wb;
    }
  }
  for (uint32_t c = 1; c < nwA; c++) {
    const uint32_t i = c * 32 + lane;
    bool fl = false;
    if (i < nA) {
      const uint4 e = R.st1[s1x + i];
      const int32_t dk = route_rule(__ldcg(&LAp[e.x]), __ldcg(&LBp[e.x]), x, e.y, R.B);
      fl = dk == (int32_t)x;
      if (dk != R.d[e.x]) {
        R.d[e.x] = dk;
        changed = 1;
      }
    }
    const unsigned w = __ballot_sync(0xFFFFFFFFu, fl);
    if (lane == 0) wA[c] = w;
  }
  for (uint32_t c = 1; c < nwB; c++) {
    const uint32_t i = c * 32 + lane;
    bool fl = false;
    if (i < nB) {
      const uint4 e = R.st2[s2x + i];
      if (e.y != x) fl = route_rule(__ldcg(&LAp[e.x]), __ldcg(&LBp[e.x]), e.y, x, R.B) == (int32_t)x;
    }
    const unsigned w = __ballot_sync(0xFFFFFFFFu, fl);
    if (lane == 0) wB[c] = w;
  }
  __syncwarp();
  // exclusive prefix popcounts of the flag words (<= 32 words per segment)
  {
    const uint32_t ca = lane < (int)nwA ? (uint32_t)__popc(wA[lane]) : 0u;
    const uint32_t cb = lane < (int)nwB ? (uint32_t)__popc(wB[lane]) : 0u;
    uint32_t ia = ca, ibv = cb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ta = __shfl_up_sync(0xFFFFFFFFu, ia, o), tb = __shfl_up_sync(0xFFFFFFFFu, ibv, o);
      if (lane >= o) {
        ia += ta;
        ibv += tb;
      }
    }
    pA[lane] = ia - ca;
    pB[lane] = ibv - cb;
    if (lane == 31) {
      pA[32] = ia;
      pB[32] = ibv;
    }
    if (lane == 0) {
      if ((nA & 31) == 0) wA[nwA] = 0;  // rank nA = the whole segment
      if ((nB & 31) == 0) wB[nwB] = 0;
    }
  }
  __syncwarp();
  // (2) the items' new loads on X (first chunks from registers)
  if (vA) {
    const uint32_t L = h.fx + seg_prefix(wA, pA, lane) + seg_prefix(wB, pB, h.eA0.z);
    LAn[h.eA0.x] = L;
    if (h.eA0.y == x) LBn[h.eA0.x] = L;
  }
  if (uB) LBn[h.eB0.x] = h.fx + seg_prefix(wB, pB, lane) + seg_prefix(wA, pA, h.eB0.z);
  for (uint32_t c = 1; c < nwA; c++) {
    const uint32_t i = c * 32 + lane;
    if (i < nA) {
      const uint4 e = R.st1[s1x + i];
      const uint32_t L = h.fx + seg_prefix(wA, pA, i) + seg_prefix(wB, pB, e.z);
      LAn[e.x] = L;
      if (e.y == x) LBn[e.x] = L;
    }
  }
  for (uint32_t c = 1; c < nwB; c++) {
    const uint32_t i = c * 32 + lane;
    if (i < nB) {
      const uint4 e = R.st2[s2x + i];
      if (e.y != x) LBn[e.x] = h.fx + seg_prefix(wB, pB, i) + seg_prefix(wA, pA, e.z);
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kRBT, FK_RB_MINB) k_btcf_route_blocks(RouteBJ R) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t sw[kRBWarps][4][kRBMaxWords + 1];  // wA, wB, pA, pB
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t *wA = sw[wib][0], *wB = sw[wib][1], *pA = sw[wib][2], *pB = sw[wib][3];
  // loads before sweep 0 (no earlier decisions): the committed fills
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < R.m; k += (int64_t)gridDim.x * blockDim.x) {
    R.LA[1][k] = R.fill[R.a[k]];
    R.LB[1][k] = R.fill[R.b[k]];
  }
  for (int64_t X = gw; X < R.nb; X += nwarps)
    if (lane == 0 && (R.e1[X] - R.s1[X] > 32u * kRBMaxWords || R.e2[X] - R.s2[X] > 32u * kRBMaxWords))
      atomicOr(&R.ctl[5], 1u);
  // the warp's first two blocks stay in registers across the sweeps
  const RBlk h0 = rb_load(R, gw, lane), h1 = rb_load(R, gw + nwarps, lane);
  grid.sync();
  if (__ldcg(&R.ctl[5])) {
    if (blockIdx.x == 0 && threadIdx.x == 0) R.ctl[4] = 2;
    return;
  }
  for (unsigned sweep = 0;; sweep++) {
    const int cur = sweep & 1, prv = cur ^ 1;
    const uint32_t *LAp = R.LA[prv], *LBp = R.LB[prv];
    uint32_t *LAn = R.LA[cur], *LBn = R.LB[cur];
    unsigned changed = 0;
    // both held blocks' loads go out together: one dependent trip per sweep
    const RBLoads v0 = rb_fetch(R, h0, LAp, LBp, lane), v1 = rb_fetch(R, h1, LAp, LBp, lane);
    if (h0.nA | h0.nB) rb_sweep(R, h0, v0, LAp, LBp, LAn, LBn, wA, wB, pA, pB, lane, changed);
    if (h1.nA | h1.nB) rb_sweep(R, h1, v1, LAp, LBp, LAn, LBn, wA, wB, pA, pB, lane, changed);
    for (int64_t X = gw + 2 * nwarps; X < R.nb; X += nwarps) {
      const RBlk h = rb_load(R, X, lane);
      if (h.nA | h.nB) rb_sweep(R, h, rb_fetch(R, h, LAp, LBp, lane), LAp, LBp, LAn, LBn, wA, wB, pA, pB, lane, changed);
    }
    const int any = __syncthreads_or(changed != 0);
    if (threadIdx.x == 0) R.chg[(size_t)cur * gridDim.x + blockIdx.x] = (unsigned)any;
    grid.sync();
    unsigned mine = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) mine |= __ldcg(&R.chg[(size_t)cur * gridDim.x + i]);
    const unsigned cc = (unsigned)__syncthreads_or(mine != 0);
    if (cc == 0 || sweep + 1 >= (unsigned)kJacobiMax) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        R.ctl[3] = sweep + 1;
        R.ctl[4] = cc == 0 ? 1u : 0u;
      }
      return;
    }
  }
}

// static per-position records of k_btcf_route_blocks
__global__ void k_route_blk_static(const uint32_t *__restrict__ a, const uint32_t *__restrict__ b,
                                   const uint32_t *__restrict__ perm1, const uint32_t *__restrict__ perm2,
                                   const uint32_t *__restrict__ qA, const uint32_t *__restrict__ qB,
                                   const uint32_t *__restrict__ s1, const uint32_t *__restrict__ s2, int64_t m,
                                   uint4 *__restrict__ st1, uint4 *__restrict__ st2) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k1 = perm1[p], k2 = perm2[p];
    st1[p] = make_uint4(k1, b[k1], qA[k1] - s2[a[k1]], 0);
    st2[p] = make_uint4(k2, a[k2], qB[k2] - s1[b[k2]], 0);
  }
}

// the static per-item gather indices of the sweeps (RouteItem)
__global__ void k_route_items(const uint32_t *__restrict__ a, const uint32_t *__restrict__ b,
                              const uint32_t *__restrict__ fill, const uint32_t *__restrict__ pos1,
                              const uint32_t *__restrict__ pos2, const uint32_t *__restrict__ qA,
                              const uint32_t *__restrict__ qB, const uint32_t *__restrict__ s1,
                              const uint32_t *__restrict__ s2, int64_t m, RouteItem *__restrict__ it) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = a[k], y = b[k];
    RouteItem r;
    r.p = make_uint4(pos1[k], s1[x], qA[k], s2[x]);
    r.q = make_uint4(qB[k], s1[y], pos2[k], s2[y]);
    r.c = make_uint4(x, y, fill[x], fill[y]);
    it[k] = r;
  }
}

// a_of1[p] = a of the item at a-order position p; b_of2[p] = b of the item
// at b-order position p, or kNoB when that item's blocks coincide (its
// choice counts as an a choice)
__global__ void k_route_orders(const uint32_t *__restrict__ a, const uint32_t *__restrict__ b,
                               const uint32_t *__restrict__ perm1, const uint32_t *__restrict__ perm2, int64_t m,
                               uint32_t *__restrict__ a_of1, uint32_t *__restrict__ b_of2) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    a_of1[p] = a[perm1[p]];
    const uint32_t i = perm2[p];
    b_of2[p] = a[i] == b[i] ? kNoB : b[i];
  }
}

// segment bounds of a sorted u32 array: s[v] = first position of value v,
// e[v] = one past its last (arrays pre-zeroed: absent values stay empty)
__global__ void k_seg_bounds_u32(const uint32_t *__restrict__ v, int64_t n, uint32_t *__restrict__ s,
                                 uint32_t *__restrict__ e) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = v[p];
    if (p == 0 || v[p - 1] != x) s[x] = (uint32_t)p;
    if (p == n - 1 || v[p + 1] != x) e[x] = (uint32_t)(p + 1);
  }
}

// pos[perm[p]] = p
__global__ void k_invert_perm(const uint32_t *__restrict__ perm, int64_t n, uint32_t *__restrict__ pos) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    pos[perm[p]] = (uint32_t)p;
}

// q[k] = first position p in [s[x_k], e[x_k]) with perm[p] >= k (perm is
// ascending inside a segment), i.e. s[x_k] + #{j < k in segment x_k}
__global__ void k_seg_rank(const uint32_t *__restrict__ x, const uint32_t *__restrict__ perm,
                           const uint32_t *__restrict__ s, const uint32_t *__restrict__ e, int64_t n,
                           uint32_t *__restrict__ q) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = x[k];
    uint32_t lo = s[v], hi = e[v];
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (perm[mid] < (uint32_t)k) lo = mid + 1; else hi = mid;
    }
    q[k] = lo;
  }
}

// leftover positions -> (b1, b2) of each leftover and the words
__global__ void k_left_blocks(BDev P, const uint64_t *__restrict__ keys, const uint32_t *__restrict__ sval,
                              const uint32_t *__restrict__ lpos, int64_t m, uint32_t *__restrict__ lb1,
                              uint32_t *__restrict__ lb2) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t fp = key_fp(P, keys[sval[lpos[k]]]);
    lb1[k] = (uint32_t)fmod64(mix64(fp ^ kBlock1), P.nbm);
    lb2[k] = (uint32_t)fmod64(mix64(fp ^ kBlock2), P.nbm);
  }
}

// second partition: key = ((dest + 1) << f) | word, value = original key index
__global__ void k_dest_keys(BDev P, const uint64_t *__restrict__ skey, const uint32_t *__restrict__ sval,
                            const uint32_t *__restrict__ lpos, const int32_t *__restrict__ dest, int64_t m,
                            uint64_t *__restrict__ skey2, uint32_t *__restrict__ sval2) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t p = lpos[k];
    skey2[k] = ((uint64_t)(dest[k] + 1) << P.f) | (skey[p] & P.fmask);
    sval2[k] = sval[p];
  }
}

// ---------------------------------------------------------------------------
// ordered backing inserts / deletes (backing_insert_batch ck:447-466,
// backing_delete_batch ck:515-549) by reservations on probe positions.
// Item e of `bidx` (priority e) targets, for inserts, its first free probe
// position; for deletes, its first live match before the chain's first
// EMPTY.  Candidates only shrink during a batch, so an item holding its
// target's reservation takes exactly the slot the sequential loop gives it.
// ---------------------------------------------------------------------------
template <typename S, int OP>
__global__ void __launch_bounds__(256) k_backing_ordered(BDev P, const uint64_t *__restrict__ keys,
                                                         const uint32_t *__restrict__ bidx, int64_t m,
                                                         uint32_t *__restrict__ bres, uint8_t *__restrict__ pend,
                                                         uint8_t *__restrict__ out, unsigned *__restrict__ ctl) {
  cg::grid_group grid = cg::this_grid();
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  S *bk = reinterpret_cast<S *>(P.backing);
  unsigned round = 0;
  for (;;) {
    for (int64_t e = tid; e < m; e += nthreads) {
      if (!__ldcg(&pend[e])) continue;
      uint64_t fp = key_fp(P, keys[bidx[e]]);
      uint64_t word = remap_tag(fp, P.fmask);
      uint64_t p = fmod64(mix64(fp ^ kBackStart), P.bsm);
      uint64_t step = fmod64(mix64(fp ^ kBackStep) | 1, P.bsm);
      for (int q = 0; q < P.probe_limit; q++) {
        uint64_t w = load_slot<S, true>(bk + p);
        if (OP == 0) {
          if (!live_word(w)) atomicMin(&bres[p], (uint32_t)e);
        } else {
          if (w == 0) break;
          if (w != 1 && (w & P.fmask) == word) atomicMin(&bres[p], (uint32_t)e);
        }
        p += step;
        p = p >= P.bsize ? p - P.bsize : p;
      }
    }
    grid.sync();
    bool left = false;
    for (int64_t e = tid; e < m; e += nthreads) {
      if (!__ldcg(&pend[e])) continue;
      uint64_t fp = key_fp(P, keys[bidx[e]]);
      uint64_t word = remap_tag(fp, P.fmask);
      uint64_t p0 = fmod64(mix64(fp ^ kBackStart), P.bsm);
      uint64_t step = fmod64(mix64(fp ^ kBackStep) | 1, P.bsm);
      int64_t target = -1;
      uint64_t p = p0;
      for (int q = 0; q < P.probe_limit; q++) {
        uint64_t w = load_slot<S, true>(bk + p);
        if (OP == 0) {
          if (!live_word(w)) { target = (int64_t)p; break; }
        } else {
          if (w == 0) break;
          if (w != 1 && (w & P.fmask) == word) { target = (int64_t)p; break; }
        }
        p += step;
        p = p >= P.bsize ? p - P.bsize : p;
      }
      if (target < 0) {  // nothing claimable now, nor later in this batch
        out[e] = 0;
        pend[e] = 0;
        continue;
      }
      if (__ldcg(&bres[target]) != (uint32_t)e) {
        left = true;
        continue;
      }
      bk[target] = (S)(OP == 0 ? word : 1);
      out[e] = 1;
      pend[e] = 0;
      p = p0;
      for (int q = 0; q < P.probe_limit; q++) {
        atomicCAS(&bres[p], (uint32_t)e, kNone);
        p += step;
        p = p >= P.bsize ? p - P.bsize : p;
      }
    }
    bool any = __syncthreads_or(left ? 1 : 0) != 0;
    if (threadIdx.x == 0) {
      if (any) atomicAdd(&ctl[round & 1], 1u);
      if (blockIdx.x == 0) ctl[(round + 1) & 1] = 0;
    }
    grid.sync();
    unsigned cnt = __ldcg(&ctl[round & 1]);
    round++;
    if (cnt == 0) break;
  }
}

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__global__ void k_iota_u32(uint32_t *__restrict__ a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

__global__ void k_not_u8(const uint8_t *__restrict__ a, int64_t n, uint8_t *__restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i] ? 0 : 1;
}

__global__ void k_gather_keys(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ idx, int64_t n,
                              uint64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = keys[idx[i]];
}

__global__ void k_scatter_ones(const uint32_t *__restrict__ idx, const uint8_t *__restrict__ flag, int64_t n,
                               uint8_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[idx[i]] = 1;
}

// counters[0] += n - fails; counters[1] += n_back - fails (insert);
// counters[2] += sum(removed) (delete)
__global__ void k_count_insert(int64_t n, const int64_t *__restrict__ n_back, const int64_t *__restrict__ n_fail,
                               int64_t *__restrict__ counters) {
  counters[0] += n - *n_fail;
  counters[1] += *n_back - *n_fail;
}

__global__ void k_count_removed(const uint8_t *__restrict__ removed, int64_t n, int64_t *__restrict__ counters) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += removed[i];
  cta_add_u64((unsigned long long *)&counters[2], (unsigned long long)c);
}

__global__ void k_flags_from_codes(const uint8_t *__restrict__ ok, int64_t n, uint8_t *__restrict__ failed,
                                   int64_t *__restrict__ n_fail) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    failed[i] = ok[i] ? 0 : 1;
    c += ok[i] ? 0 : 1;
  }
  cta_add_u64((unsigned long long *)n_fail, (unsigned long long)c);
}

__global__ void k_seg0_len(const uint32_t *__restrict__ seg_lo, const uint32_t *__restrict__ seg_hi,
                           int64_t *__restrict__ out) {
  *out = (int64_t)seg_hi[0] - (int64_t)seg_lo[0];
}

// ---------------------------------------------------------------------------
// contract-shape adapters (the reference's raw-array entry points)
// ---------------------------------------------------------------------------
__global__ void k_i64_to_u32(const int64_t *__restrict__ a, int64_t n, uint32_t *__restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (uint32_t)a[i];
}

__global__ void k_i32_to_i64(const int32_t *__restrict__ a, int64_t n, int64_t *__restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// per-block segments of the contract's (starts, ends) restricted to
// [b_lo, b_hi); every other block gets an empty segment
__global__ void k_contract_segs(const int64_t *__restrict__ starts, const int64_t *__restrict__ ends, int64_t b_lo,
                                int64_t b_hi, uint64_t nb, uint32_t *__restrict__ lo, uint32_t *__restrict__ hi) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < (int64_t)nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const bool in = b >= b_lo && b < b_hi && ends[b] > starts[b];
    lo[b] = in ? (uint32_t)starts[b] : 0u;
    hi[b] = in ? (uint32_t)ends[b] : 0u;
  }
}

// skey[k] = (b << f) | word for every item k of block b's segment (f < 0:
// the word alone -- the merge kernel reads only the word bits)
template <typename S>
__global__ void k_contract_keys(const S *__restrict__ words, const uint32_t *__restrict__ lo,
                                const uint32_t *__restrict__ hi, uint64_t nb, int f, uint64_t *__restrict__ skey) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < (int64_t)nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t bk = f < 0 ? 0 : ((uint64_t)b << f);
    for (uint32_t k = lo[b]; k < hi[b]; k++) skey[k] = bk | (uint64_t)words[k];
  }
}

// the first block (ascending) a merge would overfill: status = 1 + b
__global__ void k_merge_check(const uint32_t *__restrict__ fill, const uint32_t *__restrict__ lo,
                              const uint32_t *__restrict__ hi, uint64_t nb, int B, unsigned *__restrict__ status) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < (int64_t)nb;
       b += (int64_t)gridDim.x * blockDim.x)
    if (hi[b] > lo[b] && (int64_t)fill[b] + (hi[b] - lo[b]) > B) atomicMin(status, (unsigned)(b + 1));
}

// blocks at or past `first` keep their data (the reference's loop stops at
// the first overflow, ck:393-397)
__global__ void k_cut_segs(uint32_t *__restrict__ lo, uint32_t *__restrict__ hi, uint64_t nb,
                           const unsigned *__restrict__ status) {
  const unsigned st = *status;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < (int64_t)nb;
       b += (int64_t)gridDim.x * blockDim.x)
    if (st != kNone && (uint64_t)b >= (uint64_t)(st - 1)) lo[b] = hi[b] = 0;
}

__global__ void k_seg_flag_sum(const uint8_t *__restrict__ flag, const uint32_t *__restrict__ lo,
                               const uint32_t *__restrict__ hi, uint64_t nb, int64_t *__restrict__ out) {
  unsigned long long c = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < (int64_t)nb;
       b += (int64_t)gridDim.x * blockDim.x)
    for (uint32_t k = lo[b]; k < hi[b]; k++) c += flag[k];
  cta_add_u64((unsigned long long *)out, (unsigned long long)c);
}

// backing_insert_batch codes: P_BACKING when placed, P_FULL otherwise
__global__ void k_backing_codes(const uint8_t *__restrict__ ok, int64_t n, uint8_t *__restrict__ codes,
                                int64_t *__restrict__ fails) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    codes[i] = ok[i] ? kBacking : kFull;
    c += ok[i] ? 0 : 1;
  }
  cta_add_u64((unsigned long long *)fails, (unsigned long long)c);
}

__global__ void k_flag_sum(const uint8_t *__restrict__ f, int64_t n, int64_t *__restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += f[i];
  cta_add_u64((unsigned long long *)out, (unsigned long long)c);
}

// ---------------------------------------------------------------------------
// host pipeline pieces
// ---------------------------------------------------------------------------
inline int bits_for(uint64_t v) {  // bits needed to represent v
  int b = 0;
  while (b < 64 && (v >> b)) b++;
  return b;
}

cudaError_t sort_pairs(Scratch &S, const uint64_t *kin, uint64_t *kout, const uint32_t *vin, uint32_t *vout,
                       int64_t n, int end_bit) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, end_bit, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, n, 0, end_bit, S.st);
}

template <typename It>
cudaError_t select_flagged(Scratch &S, It in, const uint8_t *flags, uint32_t *out, int64_t *num, int64_t n) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceSelect::Flagged(nullptr, tb, in, flags, out, num, n, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceSelect::Flagged(tmp, tb, in, flags, out, num, n, S.st);
}

cudaError_t select_keys(Scratch &S, const uint64_t *in, const uint8_t *flags, uint64_t *out, int64_t *num,
                        int64_t n) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceSelect::Flagged(nullptr, tb, in, flags, out, num, n, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceSelect::Flagged(tmp, tb, in, flags, out, num, n, S.st);
}

int64_t read_i64(const int64_t *d, cudaStream_t st, cudaError_t *err) {
  int64_t h = 0;
  *err = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (*err == cudaSuccess) *err = cudaStreamSynchronize(st);
  return h;
}

#define FK_S(expr)                               \
  do {                                           \
    cudaError_t e_ = (expr);                     \
    if (e_ != cudaSuccess) return -(int)e_;      \
  } while (0)
#define FK_P(ptr)                                \
  do {                                           \
    if (!(ptr)) return -(int)S.err;              \
  } while (0)

template <typename S_t>
int per_block_launch_cfg(int B, int per_warp_slots, int *threads, size_t *smem) {
  size_t per_warp = (size_t)per_warp_slots * B * sizeof(S_t);
  int warps = 8;
  while (warps > 1 && per_warp * warps > 48 * 1024) warps >>= 1;
  *threads = 32 * warps;
  *smem = per_warp * warps;
  return *smem <= 200 * 1024 ? 0 : FK_E_ARG;
}

template <typename S_t>
int merge_segments(const BDev &P, const uint64_t *skey, const uint32_t *seg_lo, const uint32_t *seg_hi,
                   int seg_off, int phase1, uint8_t *left, unsigned *status, cudaStream_t st) {
  int threads;
  size_t smem;
  if (per_block_launch_cfg<S_t>(P.B, 2, &threads, &smem)) return FK_E_ARG;
  auto kern = k_btcf_merge<S_t>;
  if (smem > 48 * 1024) FK_S(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t ctas = ((int64_t)P.nb + threads / 32 - 1) / (threads / 32);
  int64_t cap = (int64_t)num_sms() * 32;
  kern<<<(int)(ctas < cap ? ctas : cap), threads, smem, st>>>(P, skey, seg_lo, seg_hi, seg_off, phase1, left,
                                                               status);
  FK_CHECK_LAUNCH();
  return 0;
}

int coop_grid(const void *kern, int threads) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0) != cudaSuccess || per_sm < 1)
    return 0;
  return per_sm * num_sms();
}

template <typename S_t, int OP>
int backing_ordered(const BDev &P, const uint64_t *keys, const uint32_t *bidx, int64_t m, uint8_t *ok, Scratch &S) {
  cudaStream_t st = S.st;
  uint32_t *bres = S.get<uint32_t>(P.bsize);
  FK_P(bres);
  uint8_t *pend = S.get<uint8_t>(m);
  FK_P(pend);
  unsigned *ctl = S.get<unsigned>(4);
  FK_P(ctl);
  FK_S(cudaMemsetAsync(bres, 0xFF, P.bsize * 4, st));
  FK_S(cudaMemsetAsync(pend, 1, m, st));
  FK_S(cudaMemsetAsync(ctl, 0, 16, st));
  auto kern = k_backing_ordered<S_t, OP>;
  int grid = coop_grid((const void *)kern, 256);
  if (!grid) return FK_E_ARG;
  int64_t need = (m + 255) / 256;
  if (need < grid) grid = (int)(need < 1 ? 1 : need);
  void *args[] = {(void *)&P, (void *)&keys, (void *)&bidx, (void *)&m, (void *)&bres, (void *)&pend, (void *)&ok,
                  (void *)&ctl};
  FK_S(cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(256), args, 0, st));
  return 0;
}

cudaError_t sort_pairs_u32(Scratch &S, const uint32_t *kin, uint32_t *kout, const uint32_t *vin, uint32_t *vout,
                           int64_t n, int end_bit) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, end_bit, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, n, 0, end_bit, S.st);
}

// Routing of m items (a = b1s, b = b2s, u32) against the committed fills:
// dest[k] = the sequential walk's decision (block or -1).  a_sorted: items are
// already in ascending a order (the insert pipeline's leftovers), so the
// a-order permutation is the identity and needs no sort.  Tries the
// fixpoint kernel; falls back to the one-warp walk if it did not converge
// (never observed) -- either way the result is the walk's.
int route_items(Scratch &S, const uint32_t *a, const uint32_t *b, int64_t m, const uint32_t *fill, uint64_t nb,
                uint32_t B, bool a_sorted, int32_t *dest) {
  cudaStream_t st = S.st;
  if (m <= 0) return 0;
  const char *force = getenv("FK_ROUTE");  // "seq" | "prefix" | "jacobi" (tests / measurements)
  const bool want_seq = force && !strcmp(force, "seq");
  const bool want_prefix = force && !strcmp(force, "prefix");
  if (!want_seq && !want_prefix) {
    const int kb = bits_for(nb - 1) ? bits_for(nb - 1) : 1;
    uint32_t *iota = S.get<uint32_t>(m), *perm2 = S.get<uint32_t>(m), *pos2 = S.get<uint32_t>(m),
             *qA = S.get<uint32_t>(m), *qB = S.get<uint32_t>(m), *bs = S.get<uint32_t>(m);
    // a-sorted items: the a-order permutation and its inverse are the identity
    uint32_t *perm1 = a_sorted ? iota : S.get<uint32_t>(m), *pos1 = a_sorted ? iota : S.get<uint32_t>(m);
    uint32_t *as = a_sorted ? nullptr : S.get<uint32_t>(m);
    uint32_t *segs = S.get<uint32_t>(4 * nb);
    unsigned *ctl = S.get<unsigned>(8);
    FK_P(perm1); FK_P(perm2); FK_P(pos1); FK_P(pos2); FK_P(qA); FK_P(qB); FK_P(iota); FK_P(bs); FK_P(segs);
    FK_P(ctl);
    if (!a_sorted) FK_P(as);
    uint32_t *s1 = segs, *e1 = segs + nb, *s2 = segs + 2 * nb, *e2 = segs + 3 * nb;
    k_iota_u32<<<grid_for(m), 256, 0, st>>>(iota, m);
    FK_CHECK_LAUNCH();
    FK_S(cudaMemsetAsync(segs, 0, nb * 16, st));
    FK_S(cudaMemsetAsync(ctl, 0, 32, st));
    if (a_sorted) {
      k_seg_bounds_u32<<<grid_for(m), 256, 0, st>>>(a, m, s1, e1);
    } else {
      FK_S(sort_pairs_u32(S, a, as, iota, perm1, m, kb));
      k_invert_perm<<<grid_for(m), 256, 0, st>>>(perm1, m, pos1);
      k_seg_bounds_u32<<<grid_for(m), 256, 0, st>>>(as, m, s1, e1);
    }
    FK_CHECK_LAUNCH();
    FK_S(sort_pairs_u32(S, b, bs, iota, perm2, m, kb));
    k_invert_perm<<<grid_for(m), 256, 0, st>>>(perm2, m, pos2);
    k_seg_bounds_u32<<<grid_for(m), 256, 0, st>>>(bs, m, s2, e2);
    k_seg_rank<<<grid_for(m), 256, 0, st>>>(a, perm2, s2, e2, m, qA);
    k_seg_rank<<<grid_for(m), 256, 0, st>>>(b, perm1, s1, e1, m, qB);
    FK_CHECK_LAUNCH();
    const bool stats = getenv("FK_ROUTE_STATS") != nullptr;
    if (!(force && !strcmp(force, "jacobi"))) {
      // per-block fixpoint (k_btcf_route_blocks); segments over 1024 items
      // take the global-prefix kernel below
      uint4 *st1 = S.get<uint4>(m), *st2 = S.get<uint4>(m);
      uint32_t *L0 = S.get<uint32_t>(4 * m);
      unsigned *chg2 = S.get<unsigned>(2 * 4096);
      FK_P(st1); FK_P(st2); FK_P(L0); FK_P(chg2);
      k_route_blk_static<<<grid_for(m), 256, 0, st>>>(a, b, perm1, perm2, qA, qB, s1, s2, m, st1, st2);
      FK_CHECK_LAUNCH();
      FK_S(cudaMemsetAsync(dest, 0xFE, m * 4, st));  // no decision yet
      RouteBJ RB{st1, st2, s1, e1, s2, e2, fill, a, b, {L0, L0 + m}, {L0 + 2 * m, L0 + 3 * m}, dest, ctl, chg2,
                 m, (int64_t)nb, B};
      int grid = coop_grid((const void *)k_btcf_route_blocks, kRBT);
      if (!grid) return FK_E_ARG;
      if (const char *cps = getenv("FK_RB_CTAS_PER_SM")) {  // measurement knob
        const int g2 = atoi(cps) * num_sms();
        if (g2 > 0 && g2 < grid) grid = g2;
      }
      const int64_t want = ((int64_t)nb + kRBWarps - 1) / kRBWarps;
      if (want < grid) grid = (int)(want < 1 ? 1 : want);
      if (grid > 4096) grid = 4096;
      void *args[] = {(void *)&RB};
      FK_S(cudaLaunchCooperativeKernel((const void *)k_btcf_route_blocks, dim3(grid), dim3(kRBT), args, 0, st));
      unsigned h[2] = {0, 0};
      FK_S(cudaMemcpyAsync(h, ctl + 3, 8, cudaMemcpyDeviceToHost, st));
      FK_S(cudaStreamSynchronize(st));
      if (stats) fprintf(stderr, "fk route (blocks): m=%lld sweeps=%u converged=%u grid=%d\n", (long long)m, h[0], h[1],
                         grid);
      if (h[1] == 1) return 0;
      if (h[1] == 0) goto sequential;
      FK_S(cudaMemsetAsync(ctl, 0, 32, st));  // 2: a segment is too long
    }
    {
    RouteItem *items = S.get<RouteItem>(m);
    uint32_t *a_of1 = S.get<uint32_t>(m), *b_of2 = S.get<uint32_t>(m);
    uint32_t *P1 = S.get<uint32_t>(m + 1), *P2 = S.get<uint32_t>(m + 1);
    const int T = (int)((m + kJTile - 1) / kJTile);
    const int tss = T <= kTsStrideMaxTiles ? kTsStride : 1;
    uint32_t *ts = S.get<uint32_t>((size_t)4 * T * tss);
    unsigned *chg = S.get<unsigned>(4096);
    FK_P(items); FK_P(a_of1); FK_P(b_of2); FK_P(P1); FK_P(P2); FK_P(ts); FK_P(chg);
    FK_S(cudaMemsetAsync(ts, 0, (size_t)16 * T * tss, st));
    k_route_items<<<grid_for(m), 256, 0, st>>>(a, b, fill, pos1, pos2, qA, qB, s1, s2, m, items);
    k_route_orders<<<grid_for(m), 256, 0, st>>>(a, b, perm1, perm2, m, a_of1, b_of2);
    FK_CHECK_LAUNCH();
    unsigned long long *clk = stats ? S.get<unsigned long long>(1 + 4 * 64) : nullptr;
    if (stats) FK_S(cudaMemsetAsync(clk, 0, 8 * (1 + 4 * 64), st));
    RouteJ R{items, perm1, perm2, a_of1, b_of2, pos1, pos2, dest, P1, P2, ts, tss, ctl, chg, clk, m, T, B};
    int grid = coop_grid((const void *)k_btcf_route_jacobi, kJT);
    if (!grid) return FK_E_ARG;
    const int64_t want = (m + kJT - 1) / kJT;
    if (want < grid) grid = (int)(want < T ? T : want);
    if (grid > 4096) grid = 4096;
    void *args[] = {(void *)&R};
    FK_S(cudaLaunchCooperativeKernel((const void *)k_btcf_route_jacobi, dim3(grid), dim3(kJT), args, 0, st));
    unsigned h[2] = {0, 0};
    FK_S(cudaMemcpyAsync(h, ctl + 3, 8, cudaMemcpyDeviceToHost, st));
    FK_S(cudaStreamSynchronize(st));
    if (stats) {
      unsigned long long hc[1 + 4 * 64];
      FK_S(cudaMemcpy(hc, clk, sizeof(hc), cudaMemcpyDeviceToHost));
      double s_work = 0, s_bar = 0, d_all = 0, d_max = 0;
      const unsigned ns = h[0] < 64 ? h[0] : 64;
      for (unsigned i = 0; i < ns; i++) {
        s_work += (double)(hc[1 + 3 * i] - (i ? hc[3 * i] : hc[0]));
        s_bar += (double)(hc[2 + 3 * i] - hc[1 + 3 * i]);
        d_all += (double)(hc[3 + 3 * i] - hc[2 + 3 * i]);
        d_max += (double)(hc[1 + 3 * 64 + i] - hc[2 + 3 * i]);
      }
      fprintf(stderr, "fk route: m=%lld sweeps=%u converged=%u grid=%d  per sweep (us, CTA 0): S work %.2f, S barrier %.2f, D work+barrier %.2f (slowest CTA's D work %.2f)\n",
              (long long)m, h[0], h[1], grid, s_work / ns / 1e3, s_bar / ns / 1e3, d_all / ns / 1e3, d_max / ns / 1e3);
    }
    if (h[1]) return 0;
    // not converged: fall through to the sequential walk
    }
  }
sequential:
  uint32_t *load = S.get<uint32_t>(nb);
  FK_P(load);
  size_t sm = (size_t)nb * 4;
  if (want_prefix) {
    if (!a_sorted) return FK_E_ARG;
    FK_S(cudaMemcpyAsync(load, fill, nb * 4, cudaMemcpyDeviceToDevice, st));
    FK_S(cudaFuncSetAttribute(k_btcf_route_prefix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRouteSmem));
    k_btcf_route_prefix<<<1, kRouteW, kRouteSmem, st>>>(a, b, m, load, B, dest);
  } else if (sm <= 200 * 1024) {
    if (sm > 48 * 1024)
      FK_S(cudaFuncSetAttribute(k_btcf_route_seq<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_btcf_route_seq<true><<<1, 32, sm, st>>>(a, b, m, fill, nb, load, B, dest);
  } else {
    FK_S(cudaMemcpyAsync(load, fill, nb * 4, cudaMemcpyDeviceToDevice, st));
    k_btcf_route_seq<false><<<1, 32, 0, st>>>(a, b, m, fill, nb, load, B, dest);
  }
  FK_CHECK_LAUNCH();
  return 0;
}

// ---- contract entries (host side) ----------------------------------------
template <typename S_t>
int merge_words_t(const BDev &P, const void *words, int64_t n_words, const int64_t *starts, const int64_t *ends,
                  int64_t b_lo, int64_t b_hi, int64_t *status_out, cudaStream_t st) {
  Scratch S(st);
  uint64_t *skey = S.get<uint64_t>(n_words > 0 ? n_words : 1);
  uint32_t *lo = S.get<uint32_t>(P.nb), *hi = S.get<uint32_t>(P.nb);
  unsigned *status = S.get<unsigned>(1);
  FK_P(skey); FK_P(lo); FK_P(hi); FK_P(status);
  FK_S(cudaMemsetAsync(status, 0xFF, 4, st));
  k_contract_segs<<<grid_for(P.nb), 256, 0, st>>>(starts, ends, b_lo, b_hi, P.nb, lo, hi);
  if (n_words > 0) k_contract_keys<S_t><<<grid_for(P.nb), 256, 0, st>>>((const S_t *)words, lo, hi, P.nb, -1, skey);
  k_merge_check<<<grid_for(P.nb), 256, 0, st>>>(P.fill, lo, hi, P.nb, P.B, status);
  k_cut_segs<<<grid_for(P.nb), 256, 0, st>>>(lo, hi, P.nb, status);
  FK_CHECK_LAUNCH();
  int rc = merge_segments<S_t>(P, skey, lo, hi, 0, 0, nullptr, status, st);
  if (rc) return rc;
  unsigned h = kNone;
  FK_S(cudaMemcpyAsync(&h, status, 4, cudaMemcpyDeviceToHost, st));
  FK_S(cudaStreamSynchronize(st));
  *status_out = h == kNone ? 0 : (int64_t)h;
  return 0;
}

template <typename S_t>
int delete_blocklocal_t(const BDev &P, const void *words, int64_t n_words, const int64_t *starts,
                        const int64_t *ends, int64_t b_lo, int64_t b_hi, uint8_t *removed, int64_t *n_out,
                        cudaStream_t st) {
  Scratch S(st);
  const int64_t nw = n_words > 0 ? n_words : 1;
  uint64_t *skey = S.get<uint64_t>(nw);
  uint32_t *sval = S.get<uint32_t>(nw), *lo = S.get<uint32_t>(P.nb), *hi = S.get<uint32_t>(P.nb);
  uint8_t *dummy = S.get<uint8_t>(nw);
  int64_t *cnt = S.get<int64_t>(1);
  FK_P(skey); FK_P(sval); FK_P(lo); FK_P(hi); FK_P(dummy); FK_P(cnt);
  FK_S(cudaMemsetAsync(cnt, 0, 8, st));
  k_iota_u32<<<grid_for(nw), 256, 0, st>>>(sval, nw);
  k_contract_segs<<<grid_for(P.nb), 256, 0, st>>>(starts, ends, b_lo, b_hi, P.nb, lo, hi);
  if (n_words > 0)
    k_contract_keys<S_t><<<grid_for(P.nb), 256, 0, st>>>((const S_t *)words, lo, hi, P.nb, P.f, skey);
  FK_CHECK_LAUNCH();
  int threads;
  size_t smem;
  if (per_block_launch_cfg<S_t>(P.B, 1, &threads, &smem)) return FK_E_ARG;
  auto dkern = k_btcf_delete<S_t>;
  if (smem > 48 * 1024) FK_S(cudaFuncSetAttribute(dkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t ctas = ((int64_t)P.nb + threads / 32 - 1) / (threads / 32);
  int64_t cap = (int64_t)num_sms() * 32;
  // hit[k] (per sorted item) is the contract's removed[k]
  dkern<<<(int)(ctas < cap ? ctas : cap), threads, smem, st>>>(P, skey, sval, lo, hi, removed, dummy);
  k_seg_flag_sum<<<grid_for(P.nb), 256, 0, st>>>(removed, lo, hi, P.nb, cnt);
  FK_CHECK_LAUNCH();
  cudaError_t err;
  *n_out = read_i64(cnt, st, &err);
  FK_S(err);
  return 0;
}

template <typename S_t, int OP>
int backing_batch_t(const BDev &P, const uint64_t *fps, int64_t n, uint8_t *out, int64_t *count_out,
                    cudaStream_t st) {
  Scratch S(st);
  uint32_t *idx = S.get<uint32_t>(n);
  uint8_t *ok = S.get<uint8_t>(n);
  int64_t *cnt = S.get<int64_t>(1);
  FK_P(idx); FK_P(ok); FK_P(cnt);
  FK_S(cudaMemsetAsync(cnt, 0, 8, st));
  if (P.bsize) {
    k_iota_u32<<<grid_for(n), 256, 0, st>>>(idx, n);
    int rc = backing_ordered<S_t, OP>(P, fps, idx, n, ok, S);
    if (rc) return rc;
  } else {
    FK_S(cudaMemsetAsync(ok, 0, n, st));
  }
  if (OP == 0) {
    k_backing_codes<<<grid_for(n), 256, 0, st>>>(ok, n, out, cnt);  // cnt = fails
  } else {
    FK_S(cudaMemcpyAsync(out, ok, n, cudaMemcpyDeviceToDevice, st));
    k_flag_sum<<<grid_for(n), 256, 0, st>>>(ok, n, cnt);
  }
  FK_CHECK_LAUNCH();
  cudaError_t err;
  *count_out = read_i64(cnt, st, &err);
  FK_S(err);
  return 0;
}

// ---- insert_batch (tcf_bulk.py:179-257) ------------------------------------
template <typename S_t>
int btcf_insert(const BDev &P, const uint64_t *keys, int64_t n, uint64_t *failed_keys, int64_t *n_failed,
                int64_t *counters, unsigned *status, cudaStream_t st) {
  Scratch S(st);
  const int end1 = P.f + bits_for(P.nb - 1);
  uint64_t *k0 = S.get<uint64_t>(n), *skey = S.get<uint64_t>(n);
  uint32_t *v0 = S.get<uint32_t>(n), *sval = S.get<uint32_t>(n);
  uint32_t *seg_lo = S.get<uint32_t>(2 * (P.nb + 1)), *seg_hi = seg_lo + P.nb + 1;  // one memset clears both
  uint8_t *left = S.get<uint8_t>(n);
  int64_t *cnt = S.get<int64_t>(4);  // [0] leftovers, [1] backing items, [2] fails
  FK_P(k0); FK_P(skey); FK_P(v0); FK_P(sval); FK_P(seg_lo); FK_P(left); FK_P(cnt);
  FK_S(cudaMemsetAsync(cnt, 0, 32, st));
  FK_S(cudaMemsetAsync(n_failed, 0, 8, st));
  // partition (tcf_bulk.py:133-143): stable sort by (b1, word)
  k_part_keys<<<grid_for(n), 256, 0, st>>>(P, keys, nullptr, n, 0, k0, v0);
  FK_CHECK_LAUNCH();
  FK_S(sort_pairs(S, k0, skey, v0, sval, n, end1));
  FK_S(cudaMemsetAsync(seg_lo, 0, (P.nb + 1) * 8, st));
  k_seg_bounds<<<grid_for(n), 256, 0, st>>>(skey, n, P.f, seg_lo, seg_hi);
  FK_CHECK_LAUNCH();
  // phase 1: shortcut merge up to the cut line, flag leftovers
  FK_S(cudaMemsetAsync(left, 0, n, st));
  int rc = merge_segments<S_t>(P, skey, seg_lo, seg_hi, 0, 1, left, status, st);
  if (rc) return rc;
  // leftovers, in sorted order (tcf_bulk.py:211-213)
  uint32_t *lpos = S.get<uint32_t>(n);
  FK_P(lpos);
  FK_S(select_flagged(S, cub::CountingInputIterator<uint32_t>(0), left, lpos, cnt, n));
  cudaError_t err;
  int64_t m = read_i64(cnt, st, &err);
  FK_S(err);
  if (m > 0) {
    uint32_t *lb1 = S.get<uint32_t>(m), *lb2 = S.get<uint32_t>(m);
    int32_t *dest = S.get<int32_t>(m);
    FK_P(lb1); FK_P(lb2); FK_P(dest);
    k_left_blocks<<<grid_for(m), 256, 0, st>>>(P, keys, sval, lpos, m, lb1, lb2);
    FK_CHECK_LAUNCH();
    // phase 2 routing (tcf_bulk.py:210-223): leftovers are in (b1, word) order
    rc = route_items(S, lb1, lb2, m, P.fill, P.nb, (uint32_t)P.B, true, dest);
    if (rc) return rc;
    // group by destination; segment 0 = backing (tcf_bulk.py:225-234)
    uint64_t *k2 = S.get<uint64_t>(m), *skey2 = S.get<uint64_t>(m);
    uint32_t *v2 = S.get<uint32_t>(m), *sval2 = S.get<uint32_t>(m);
    FK_P(k2); FK_P(skey2); FK_P(v2); FK_P(sval2);
    k_dest_keys<<<grid_for(m), 256, 0, st>>>(P, skey, sval, lpos, dest, m, k2, v2);
    FK_CHECK_LAUNCH();
    FK_S(sort_pairs(S, k2, skey2, v2, sval2, m, P.f + bits_for(P.nb)));
    FK_S(cudaMemsetAsync(seg_lo, 0, (P.nb + 1) * 8, st));
    k_seg_bounds<<<grid_for(m), 256, 0, st>>>(skey2, m, P.f, seg_lo, seg_hi);
    FK_CHECK_LAUNCH();
    rc = merge_segments<S_t>(P, skey2, seg_lo, seg_hi, 1, 0, nullptr, status, st);
    if (rc) return rc;
    // backing overflow, in (word, routing) order (tcf_bulk.py:247-255)
    k_seg0_len<<<1, 1, 0, st>>>(seg_lo, seg_hi, cnt + 1);
    FK_CHECK_LAUNCH();
    int64_t nback = read_i64(cnt + 1, st, &err);
    FK_S(err);
    if (nback > 0) {
      uint8_t *ok = S.get<uint8_t>(nback), *failf = S.get<uint8_t>(nback);
      uint64_t *bkeys = S.get<uint64_t>(nback);
      FK_P(ok); FK_P(failf); FK_P(bkeys);
      if (P.bsize) {
        rc = backing_ordered<S_t, 0>(P, keys, sval2, nback, ok, S);
        if (rc) return rc;
      } else {
        FK_S(cudaMemsetAsync(ok, 0, nback, st));
      }
      k_flags_from_codes<<<grid_for(nback), 256, 0, st>>>(ok, nback, failf, cnt + 2);
      FK_CHECK_LAUNCH();
      k_gather_keys<<<grid_for(nback), 256, 0, st>>>(keys, sval2, nback, bkeys);
      FK_CHECK_LAUNCH();
      FK_S(select_keys(S, bkeys, failf, failed_keys, n_failed, nback));
    }
  }
  k_count_insert<<<1, 1, 0, st>>>(n, cnt + 1, cnt + 2, counters);
  FK_CHECK_LAUNCH();
  return 0;
}

// ---- delete_batch (tcf_bulk.py:283-325) -------------------------------------
template <typename S_t>
int btcf_delete(const BDev &P, const uint64_t *keys, int64_t n, uint8_t *removed, int64_t *counters,
                cudaStream_t st) {
  Scratch S(st);
  const int end1 = P.f + bits_for(P.nb - 1);
  uint32_t *pend = S.get<uint32_t>(n), *pend2 = S.get<uint32_t>(n);
  uint64_t *k0 = S.get<uint64_t>(n), *skey = S.get<uint64_t>(n);
  uint32_t *sval = S.get<uint32_t>(n);
  uint32_t *seg_lo = S.get<uint32_t>(P.nb), *seg_hi = S.get<uint32_t>(P.nb);
  uint8_t *hit = S.get<uint8_t>(n), *miss = S.get<uint8_t>(n);
  int64_t *cnt = S.get<int64_t>(2);
  FK_P(pend); FK_P(pend2); FK_P(k0); FK_P(skey); FK_P(sval); FK_P(seg_lo); FK_P(seg_hi); FK_P(hit); FK_P(miss);
  FK_P(cnt);
  FK_S(cudaMemsetAsync(removed, 0, n, st));
  k_iota_u32<<<grid_for(n), 256, 0, st>>>(pend, n);
  FK_CHECK_LAUNCH();
  int threads;
  size_t smem;
  if (per_block_launch_cfg<S_t>(P.B, 1, &threads, &smem)) return FK_E_ARG;
  auto dkern = k_btcf_delete<S_t>;
  if (smem > 48 * 1024) FK_S(cudaFuncSetAttribute(dkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t ctas = ((int64_t)P.nb + threads / 32 - 1) / (threads / 32);
  int64_t cap = (int64_t)num_sms() * 32;
  int dgrid = (int)(ctas < cap ? ctas : cap);
  int64_t m = n;
  for (int which = 0; which < 2 && m > 0; which++) {
    k_part_keys<<<grid_for(m), 256, 0, st>>>(P, keys, pend, m, which, k0, pend2);
    FK_CHECK_LAUNCH();
    FK_S(sort_pairs(S, k0, skey, pend2, sval, m, end1));
    FK_S(cudaMemsetAsync(seg_lo, 0, P.nb * 4, st));
    FK_S(cudaMemsetAsync(seg_hi, 0, P.nb * 4, st));
    k_seg_bounds<<<grid_for(m), 256, 0, st>>>(skey, m, P.f, seg_lo, seg_hi);
    FK_CHECK_LAUNCH();
    dkern<<<dgrid, threads, smem, st>>>(P, skey, sval, seg_lo, seg_hi, hit, removed);
    FK_CHECK_LAUNCH();
    // misses, in this pass's sorted order (tcf_bulk.py:318)
    k_not_u8<<<grid_for(m), 256, 0, st>>>(hit, m, miss);
    FK_CHECK_LAUNCH();
    FK_S(select_flagged(S, sval, miss, pend, cnt, m));
    cudaError_t err;
    m = read_i64(cnt, st, &err);
    FK_S(err);
  }
  if (m > 0 && P.bsize) {
    uint8_t *ok = S.get<uint8_t>(m);
    FK_P(ok);
    int rc = backing_ordered<S_t, 1>(P, keys, pend, m, ok, S);
    if (rc) return rc;
    k_scatter_ones<<<grid_for(m), 256, 0, st>>>(pend, ok, m, removed);
    FK_CHECK_LAUNCH();
  }
  k_count_removed<<<grid_for(n), 256, 0, st>>>(removed, n, counters);
  FK_CHECK_LAUNCH();
  return 0;
}

template <typename S_t>
int btcf_query(const BDev &P, const uint64_t *keys, int64_t n, uint8_t *found, cudaStream_t st) {
  // lanes per key: one lane per key up to 8 sectors per block (all of a
  // key's sector loads in flight at once; the table is L2-resident at
  // configs[0], so loads in flight, not bytes, bound the query), more lanes
  // for larger blocks.  Measured at configs[0] (2^20 slots, 256-byte
  // blocks): 8 lanes 0.175 / 0.206 ms (pos / neg), 2 lanes 0.140 / 0.106,
  // 1 lane 0.124 / 0.101.  Tunable: FK_BTCF_QUERY_G (1, 2, 4 or 8).
  const int64_t sectors = ((int64_t)P.B * (int64_t)sizeof(S_t) + 31) / 32;
  const char *ge = getenv("FK_BTCF_QUERY_G");
  const int G = ge ? atoi(ge) : (sectors <= 8 ? 1 : (sectors <= 16 ? 2 : (sectors <= 32 ? 4 : 8)));
  int64_t tiles_per_cta = 256 / (G == 1 || G == 2 || G == 4 ? G : 8);
  int64_t need = (n + tiles_per_cta - 1) / tiles_per_cta;
  int64_t cap = (int64_t)num_sms() * 8;
  const int grid = (int)(need < cap ? (need < 1 ? 1 : need) : cap);
  if (G == 1) k_btcf_query<S_t, 1><<<grid, 256, 0, st>>>(P, keys, n, found);
  else if (G == 2) k_btcf_query<S_t, 2><<<grid, 256, 0, st>>>(P, keys, n, found);
  else if (G == 4) k_btcf_query<S_t, 4><<<grid, 256, 0, st>>>(P, keys, n, found);
  else k_btcf_query<S_t, 8><<<grid, 256, 0, st>>>(P, keys, n, found);
  FK_CHECK_LAUNCH();
  return 0;
}

// ---- partition (BulkTcf.partition, tcf_bulk.py:123-143) ---------------------
int btcf_partition(const BDev &P, const uint64_t *keys, int64_t n, uint64_t *sorted_keys, uint32_t *order,
                   cudaStream_t st) {
  Scratch S(st);
  uint64_t *k0 = S.get<uint64_t>(n);
  uint32_t *v0 = S.get<uint32_t>(n);
  FK_P(k0); FK_P(v0);
  k_part_keys<<<grid_for(n), 256, 0, st>>>(P, keys, nullptr, n, 0, k0, v0);
  FK_CHECK_LAUNCH();
  FK_S(sort_pairs(S, k0, sorted_keys, v0, order, n, P.f + bits_for(P.nb - 1)));
  return 0;
}

bool geom_ok(const fk_btcf_geom *g) {
  if (!g || g->num_blocks < 1 || g->num_blocks > 0x7FFFFFF0LL || g->backing_slots < 0) return false;
  if (g->block_slots < 2 || g->block_slots > 8192) return false;
  if (g->slot_bytes != 1 && g->slot_bytes != 2 && g->slot_bytes != 4) return false;
  if (g->tag_bits <= 2 || g->tag_bits > 8 * g->slot_bytes) return false;
  if (g->tag_bits + bits_for((uint64_t)g->num_blocks) > 64) return false;
  return true;
}

BDev make_dev(const fk_btcf_geom *g, void *blocks, uint32_t *fill, void *backing, int keys_are_fps) {
  BDev P;
  P.blocks = blocks;
  P.fill = fill;
  P.backing = backing;
  P.nb = (uint64_t)g->num_blocks;
  P.nbm = make_fastmod(P.nb);
  P.bsize = (uint64_t)g->backing_slots;
  P.bsm = make_fastmod(P.bsize ? P.bsize : 1);
  P.B = g->block_slots;
  P.f = g->tag_bits;
  P.cut = g->cut_slots;
  P.probe_limit = g->probe_limit;
  P.fmask = (1ULL << g->tag_bits) - 1;
  P.seed = g->seed;
  P.keys_are_fps = keys_are_fps;
  return P;
}

}  // namespace

}  // namespace fk

using namespace fk;

namespace fk {
namespace {
// Sorted-block invariants of BulkTcf.validate (tcf_bulk.py:354-374), one
// thread per block: v[0] |= 1 fill over capacity, 2 a reserved word in the
// live prefix, 4 an unsorted prefix, 8 a non-empty tail; v[1 + c] = first
// such block (atomicMin); v[5] = sum of fill; v[6] = live backing slots.
template <typename S>
__global__ void k_btcf_validate(const S *__restrict__ blocks, const uint32_t *__restrict__ fill, int64_t nb, int B,
                                const S *__restrict__ backing, int64_t bsize,
                                unsigned long long *__restrict__ v) {
  unsigned long long sumf = 0, liveb = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t f = fill[b];
    sumf += f;
    unsigned bad = 0;
    if ((int64_t)f > B) bad |= 1;
    const S *blk = blocks + b * (int64_t)B;
    uint64_t prev = 0;
    for (int j = 0; j < B; j++) {
      const uint64_t w = blk[j];
      if ((uint32_t)j < f) {
        if (w < 2) bad |= 2;
        if (j > 0 && w < prev) bad |= 4;
        prev = w;
      } else if (w != 0) {
        bad |= 8;
      }
    }
    for (int c = 0; c < 4; c++)
      if (bad >> c & 1) {
        atomicOr(&v[0], 1ull << c);
        atomicMin(&v[1 + c], (unsigned long long)b);
      }
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < bsize; i += (int64_t)gridDim.x * blockDim.x)
    liveb += (uint64_t)backing[i] > 1;
  if (sumf) atomicAdd(&v[5], sumf);
  if (liveb) atomicAdd(&v[6], liveb);
}

template <typename S>
int btcf_validate_t(const fk_btcf_geom *g, const void *blocks, const uint32_t *fill, const void *backing,
                    int64_t *out8, cudaStream_t st) {
  unsigned long long *d = nullptr;
  FK_TRY(cudaMallocAsync((void **)&d, 8 * sizeof(unsigned long long), st));
  unsigned long long init[8] = {0, ~0ull, ~0ull, ~0ull, ~0ull, 0, 0, 0};
  int rc = 0;
  cudaError_t e = cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    k_btcf_validate<S><<<grid_for(g->num_blocks), 256, 0, st>>>((const S *)blocks, fill, g->num_blocks,
                                                              g->block_slots, (const S *)backing, g->backing_slots,
                                                              d);
    e = cudaGetLastError();
  }
  unsigned long long h[8];
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  if (e != cudaSuccess) return -(int)e;
  for (int i = 0; i < 8; i++) out8[i] = (int64_t)h[i];
  return rc;
}
}  // namespace
}  // namespace fk

extern "C" {

int fk_btcf_validate(const fk_btcf_geom *g, const void *blocks, const uint32_t *fill, const void *backing,
                     int64_t *out8, void *stream) {
  if (!geom_ok(g) || !out8) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return btcf_validate_t<uint8_t>(g, blocks, fill, backing, out8, st);
    case 4: return btcf_validate_t<uint32_t>(g, blocks, fill, backing, out8, st);
    default: return btcf_validate_t<uint16_t>(g, blocks, fill, backing, out8, st);
  }
}

int fk_btcf_insert(const fk_btcf_geom *g, void *blocks, uint32_t *fill, void *backing, const uint64_t *keys,
                   int keys_are_fps, int64_t n, uint64_t *failed_keys, int64_t *n_failed, int64_t *counters,
                   uint32_t *status, void *stream) {
  if (!geom_ok(g) || n < 0 || n > 0xFFFFFFF0LL || !counters || !status || !n_failed) return FK_E_ARG;
  if (n == 0) return 0;
  BDev P = make_dev(g, blocks, fill, backing, keys_are_fps);
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return btcf_insert<uint8_t>(P, keys, n, failed_keys, n_failed, counters, status, st);
    case 4: return btcf_insert<uint32_t>(P, keys, n, failed_keys, n_failed, counters, status, st);
    default: return btcf_insert<uint16_t>(P, keys, n, failed_keys, n_failed, counters, status, st);
  }
}

int fk_btcf_query(const fk_btcf_geom *g, const void *blocks, const uint32_t *fill, const void *backing,
                  const uint64_t *keys, int keys_are_fps, int64_t n, uint8_t *found, void *stream) {
  if (!geom_ok(g) || n < 0) return FK_E_ARG;
  if (n == 0) return 0;
  BDev P = make_dev(g, const_cast<void *>(blocks), const_cast<uint32_t *>(fill), const_cast<void *>(backing),
                    keys_are_fps);
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return btcf_query<uint8_t>(P, keys, n, found, st);
    case 4: return btcf_query<uint32_t>(P, keys, n, found, st);
    default: return btcf_query<uint16_t>(P, keys, n, found, st);
  }
}

int fk_btcf_delete(const fk_btcf_geom *g, void *blocks, uint32_t *fill, void *backing, const uint64_t *keys,
                   int keys_are_fps, int64_t n, uint8_t *removed, int64_t *counters, void *stream) {
  if (!geom_ok(g) || n < 0 || n > 0xFFFFFFF0LL || !counters) return FK_E_ARG;
  if (n == 0) return 0;
  BDev P = make_dev(g, blocks, fill, backing, keys_are_fps);
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return btcf_delete<uint8_t>(P, keys, n, removed, counters, st);
    case 4: return btcf_delete<uint32_t>(P, keys, n, removed, counters, st);
    default: return btcf_delete<uint16_t>(P, keys, n, removed, counters, st);
  }
}

int fk_btcf_partition(const fk_btcf_geom *g, const uint64_t *keys, int keys_are_fps, int64_t n,
                      uint64_t *sorted_keys, uint32_t *order, void *stream) {
  if (!geom_ok(g) || n < 0 || n > 0xFFFFFFF0LL) return FK_E_ARG;
  if (n == 0) return 0;
  BDev P = make_dev(g, nullptr, nullptr, nullptr, keys_are_fps);
  return btcf_partition(P, keys, n, sorted_keys, order, (cudaStream_t)stream);
}

int fk_btcf_merge_lists(const fk_btcf_geom *g, void *blocks, uint32_t *fill, const uint64_t *sorted_keys,
                        const uint32_t *seg_lo, const uint32_t *seg_hi, uint32_t *status, void *stream) {
  if (!geom_ok(g) || !status) return FK_E_ARG;
  BDev P = make_dev(g, blocks, fill, nullptr, 1);
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return merge_segments<uint8_t>(P, sorted_keys, seg_lo, seg_hi, 0, 0, nullptr, status, st);
    case 4: return merge_segments<uint32_t>(P, sorted_keys, seg_lo, seg_hi, 0, 0, nullptr, status, st);
    default: return merge_segments<uint16_t>(P, sorted_keys, seg_lo, seg_hi, 0, 0, nullptr, status, st);
  }
}

// ---- contract-shaped entries (one per reference kernel-contract function) ----

int fk_btcf_route(const uint32_t *fill, int64_t num_blocks, int block_slots, const int64_t *b1s, const int64_t *b2s,
                  int64_t n, int64_t *dest, void *stream) {
  if (!fill || num_blocks < 1 || num_blocks > 0xFFFFFFF0LL || block_slots < 1 || n < 0 || n > 0xFFFFFFF0LL)
    return FK_E_ARG;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch S(st);
  uint32_t *a = S.get<uint32_t>(n), *b = S.get<uint32_t>(n);
  int32_t *d = S.get<int32_t>(n);
  FK_P(a); FK_P(b); FK_P(d);
  k_i64_to_u32<<<grid_for(n), 256, 0, st>>>(b1s, n, a);
  k_i64_to_u32<<<grid_for(n), 256, 0, st>>>(b2s, n, b);
  FK_CHECK_LAUNCH();
  int rc = route_items(S, a, b, n, fill, (uint64_t)num_blocks, (uint32_t)block_slots, false, d);
  if (rc) return rc;
  k_i32_to_i64<<<grid_for(n), 256, 0, st>>>(d, n, dest);
  FK_CHECK_LAUNCH();
  FK_S(cudaStreamSynchronize(st));
  return 0;
}

int fk_btcf_merge_words(const fk_btcf_geom *g, void *blocks, uint32_t *fill, const void *words, int64_t n_words,
                        const int64_t *starts, const int64_t *ends, int64_t b_lo, int64_t b_hi, int64_t *status_out,
                        void *stream) {
  if (!geom_ok(g) || !status_out || n_words < 0 || n_words > 0xFFFFFFF0LL || b_lo < 0 || b_hi > g->num_blocks)
    return FK_E_ARG;
  *status_out = 0;
  if (b_hi <= b_lo) return 0;
  BDev P = make_dev(g, blocks, fill, nullptr, 1);
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return merge_words_t<uint8_t>(P, words, n_words, starts, ends, b_lo, b_hi, status_out, st);
    case 4: return merge_words_t<uint32_t>(P, words, n_words, starts, ends, b_lo, b_hi, status_out, st);
    default: return merge_words_t<uint16_t>(P, words, n_words, starts, ends, b_lo, b_hi, status_out, st);
  }
}

int fk_btcf_delete_blocklocal(const fk_btcf_geom *g, void *blocks, uint32_t *fill, const void *words,
                              int64_t n_words, const int64_t *starts, const int64_t *ends, int64_t b_lo, int64_t b_hi,
                              uint8_t *removed, int64_t *n_removed, void *stream) {
  if (!geom_ok(g) || !n_removed || n_words < 0 || n_words > 0xFFFFFFF0LL || b_lo < 0 || b_hi > g->num_blocks)
    return FK_E_ARG;
  *n_removed = 0;
  if (b_hi <= b_lo || n_words == 0) return 0;
  BDev P = make_dev(g, blocks, fill, nullptr, 1);
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return delete_blocklocal_t<uint8_t>(P, words, n_words, starts, ends, b_lo, b_hi, removed, n_removed, st);
    case 4: return delete_blocklocal_t<uint32_t>(P, words, n_words, starts, ends, b_lo, b_hi, removed, n_removed, st);
    default: return delete_blocklocal_t<uint16_t>(P, words, n_words, starts, ends, b_lo, b_hi, removed, n_removed, st);
  }
}

int fk_backing_insert_batch(const fk_btcf_geom *g, void *backing, const uint64_t *fps, int64_t n, uint8_t *codes,
                            int64_t *n_fail, void *stream) {
  if (!geom_ok(g) || !n_fail || n < 0 || n > 0xFFFFFFF0LL) return FK_E_ARG;
  *n_fail = 0;
  if (n == 0) return 0;
  BDev P = make_dev(g, nullptr, nullptr, backing, 1);
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return backing_batch_t<uint8_t, 0>(P, fps, n, codes, n_fail, st);
    case 4: return backing_batch_t<uint32_t, 0>(P, fps, n, codes, n_fail, st);
    default: return backing_batch_t<uint16_t, 0>(P, fps, n, codes, n_fail, st);
  }
}

int fk_backing_delete_batch(const fk_btcf_geom *g, void *backing, const uint64_t *fps, int64_t n, uint8_t *removed,
                            int64_t *n_removed, void *stream) {
  if (!geom_ok(g) || !n_removed || n < 0 || n > 0xFFFFFFF0LL) return FK_E_ARG;
  *n_removed = 0;
  if (n == 0) return 0;
  BDev P = make_dev(g, nullptr, nullptr, backing, 1);
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->slot_bytes) {
    case 1: return backing_batch_t<uint8_t, 1>(P, fps, n, removed, n_removed, st);
    case 4: return backing_batch_t<uint32_t, 1>(P, fps, n, removed, n_removed, st);
    default: return backing_batch_t<uint16_t, 1>(P, fps, n, removed, n_removed, st);
  }
}

}  // extern "C"
