#pragma once
// tcf_point.cu -- point two-choice filter on sm_100a.
//
// Replaces the reference kernel contract functions tcf_insert_batch,
// tcf_query_batch and tcf_delete_batch (_ckernels.pyx:193-355,
// _pykernels.py:120-236).  One cooperative-group tile of G lanes (1..32)
// serves one key: the tile loads the key's 16-bit-tag block with 128-bit
// vector loads split across its lanes, and votes with warp ballots (the
// paper's Alg. 1).
//
// Two insert/delete semantics:
//   * concurrent (FK_CONCURRENT): every key at once, slot claims by atomicCAS,
//     a lost CAS moves to the next candidate -- the reference's free-threaded
//     semantics.
//   * ordered (FK_ORDERED): bit-identical to one caller thread streaming the
//     batch through the reference.  A persistent cooperative kernel walks the
//     batch in windows; within a window keys take deterministic reservations
//     on both candidate blocks (atomicMin of the input index) and a key
//     commits only when it holds both, i.e. when every earlier key that could
//     change its blocks has already committed.  Backing-table work, which
//     never feeds back into block decisions (ck:228-233), is deferred to a
//     second reservation phase over probe positions.
#include "../../include/filterkit_b200.h"
#include "fk_common.cuh"

namespace fk {

constexpr uint32_t kNoRes = 0xFFFFFFFFu;


struct TcfDev {
  void *blocks;
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

struct KeyInfo {
  uint64_t fp, tag, b1, b2;
};

__device__ __forceinline__ KeyInfo key_info(const TcfDev &P, uint64_t key) {
  KeyInfo k;
  k.fp = P.keys_are_fps ? key : mix64(key ^ P.seed);  // tcf.py:118-120
  k.tag = remap_tag(k.fp, P.fmask);
  k.b1 = fmod64(mix64(k.fp ^ kBlock1), P.nbm);  // hashing.py:92-99
  k.b2 = fmod64(mix64(k.fp ^ kBlock2), P.nbm);
  return k;
}

// G lanes of an aligned warp sub-group serve one key.
template <int G>
struct Tile {
  unsigned lane, base, mask;
  __device__ __forceinline__ Tile() {
    unsigned l = threadIdx.x & 31;
    lane = l % G;
    base = l - lane;
    mask = G == 32 ? 0xFFFFFFFFu : (((1u << G) - 1u) << base);
  }
  __device__ __forceinline__ unsigned ballot(bool p) const {
    if constexpr (G == 1) return p ? 1u : 0u;
    unsigned b = __ballot_sync(mask, p);
    return G == 32 ? b : ((b >> base) & ((1u << G) - 1u));
  }
  template <typename T>
  __device__ __forceinline__ T bcast(T v, int src) const {
    if constexpr (G == 1) return v;
    return __shfl_sync(mask, v, (int)base + src);
  }
  __device__ __forceinline__ int sum(int v) const {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
  }
};

// One lane's contiguous share of a block: slots [lo, lo+cnt).
// BF = compile-time block size (vector loads), 0 = runtime B (scalar loads).
template <typename S, int G, int BF>
struct Chunk {
  static constexpr int MAXB = BF ? BF : (1024 / (8 * (int)sizeof(S)));
  static constexpr int C = (MAXB + G - 1) / G;
  static constexpr int NREG = (C * (int)sizeof(S) + 3) / 4;
  uint32_t r[NREG];
  int lo, cnt;

  template <bool CGL>
  __device__ __forceinline__ void load(const S *blk, int B, unsigned lane) {
    if constexpr (BF != 0) {
      lo = (int)lane * C;
      cnt = C;
      load_chunk<C * (int)sizeof(S), CGL>(blk + lo, r);
    } else {
      int c = (B + G - 1) / G;
      lo = (int)lane * c;
      cnt = B - lo < c ? B - lo : c;
      if (cnt < 0) cnt = 0;
#pragma unroll
      for (int j = 0; j < NREG; j++) r[j] = 0;
#pragma unroll
      for (int j = 0; j < C; j++)
        if (j < cnt) set_reg_slot<S>(r, j, load_slot<S, CGL>(blk + lo + j));
    }
  }
  __device__ __forceinline__ uint64_t at(int j) const { return reg_slot<S>(r, j); }
  __device__ __forceinline__ int used() const {
    int n = 0;
#pragma unroll
    for (int j = 0; j < C; j++) n += (j < cnt && live_word(at(j))) ? 1 : 0;
    return n;
  }
  // first index >= j0 that is free (EMPTY or TOMBSTONE), else -1
  __device__ __forceinline__ int first_free(int j0) const {
#pragma unroll
    for (int j = 0; j < C; j++)
      if (j >= j0 && j < cnt && !live_word(at(j))) return j;
    return -1;
  }
  // Branch-free lowest match for 16-bit slots whose word is the tag itself
  // (tag_bits == 16: no value bits; tags are >= 2, so EMPTY/TOMBSTONE never
  // match): one __vcmpeq2 per register pair of slots.
  __device__ __forceinline__ int first_match_eq16(uint32_t tag) const {
    static_assert(sizeof(S) == 2, "16-bit slots only");
    const uint32_t pat = tag | (tag << 16);
    uint32_t bits = 0;
#pragma unroll
    for (int i = 0; i < NREG; i++) {
      uint32_t m = __vcmpeq2(r[i], pat);
      bits |= ((m & 1u) | ((m >> 15) & 2u)) << (2 * i);
    }
    if (BF == 0) bits &= cnt >= 32 ? 0xFFFFFFFFu : ((1u << cnt) - 1u);
    return bits ? __ffs(bits) - 1 : -1;
  }

  // first index >= j0 holding a live word whose tag bits equal tag, else -1
  __device__ __forceinline__ int first_match(int j0, uint64_t tag, uint64_t fmask) const {
#pragma unroll
    for (int j = 0; j < C; j++) {
      uint64_t w = at(j);
      if (j >= j0 && j < cnt && live_word(w) && (w & fmask) == tag) return j;
    }
    return -1;
  }
};

// ---------------------------------------------------------------------------
// query (pure function of table + keys: bit-exact in every mode)
// ---------------------------------------------------------------------------
template <typename S, int G, int BF>
__global__ void __launch_bounds__(256) k_tcf_query(TcfDev P, const uint64_t *__restrict__ keys, int64_t n,
                                                   uint8_t *__restrict__ found, uint64_t *__restrict__ vals) {
  Tile<G> t;
  const S *blocks = reinterpret_cast<const S *>(P.blocks);
  const S *backing = reinterpret_cast<const S *>(P.backing);
  int64_t tiles = (int64_t)gridDim.x * (blockDim.x / G);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; i < n; i += tiles) {
    KeyInfo k = key_info(P, keys[i]);
    bool hit = false;
    uint64_t val = 0;
    // b1, then b2: first live match in ascending slot order (pk:152-177)
#pragma unroll 1
    for (int which = 0; which < 2 && !hit; which++) {
      uint64_t b = which ? k.b2 : k.b1;
      Chunk<S, G, BF> c;
      c.template load<false>(blocks + b * (uint64_t)P.B, P.B, t.lane);
      int j;
      if constexpr (sizeof(S) == 2 && Chunk<S, G, BF>::C <= 32) {
        j = P.f == 16 ? c.first_match_eq16((uint32_t)k.tag) : c.first_match(0, k.tag, P.fmask);
      } else {
        j = c.first_match(0, k.tag, P.fmask);
      }
      unsigned bal = t.ballot(j >= 0);
      if (bal) {
        int leader = __ffs(bal) - 1;
        uint64_t w = t.bcast(j >= 0 ? c.at(j) : 0ull, leader);
        hit = true;
        val = P.f >= 64 ? 0 : (w >> P.f);
      }
    }
    if (!hit && P.bsize && t.lane == 0) {  // backing chain (pk:178-189)
      uint64_t p = fmod64(mix64(k.fp ^ kBackStart), P.bsm);
      uint64_t step = fmod64(mix64(k.fp ^ kBackStep) | 1, P.bsm);
      for (int q = 0; q < P.probe_limit; q++) {
        uint64_t w = backing[p];
        if (w == 0) break;
        if (w != 1 && (w & P.fmask) == k.tag) {
          hit = true;
          val = P.f >= 64 ? 0 : (w >> P.f);
          break;
        }
        p += step;
        p = p >= P.bsize ? p - P.bsize : p;
      }
    }
    if (t.lane == 0) {
      found[i] = hit ? 1 : 0;
      if (vals) vals[i] = hit ? val : 0;
    }
  }
}

// ---------------------------------------------------------------------------
// Register-resident fast path for the benchmarked geometry (16 x u16 slots =
// one 32-byte sector, G = 1): a block is 8 registers and every decision is a
// 16-bit mask (bit s = slot s), so nothing is ever indexed dynamically and
// the kernels keep no block state in local memory (the generic Chunk path
// does, and a grid barrier's L1 invalidation makes that expensive).
// ---------------------------------------------------------------------------
template <typename S, int G, int BF>
constexpr bool kFast16 = sizeof(S) == 2 && G == 1 && BF == 16;

__device__ __forceinline__ uint32_t live16(const uint32_t (&r)[8]) {  // slot > TOMBSTONE
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    uint32_t g = __vcmpgtu2(r[i], 0x00010001u);
    m |= ((g & 1u) | ((g >> 15) & 2u)) << (2 * i);
  }
  return m;
}

// live slots whose tag bits equal tag (tags are >= 2, so the live test only
// matters when value bits sit above the tag)
__device__ __forceinline__ uint32_t match16(const uint32_t (&r)[8], uint32_t tag, uint32_t fmask) {
  const uint32_t pat = tag | (tag << 16), fm2 = fmask | (fmask << 16);
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    uint32_t g = __vcmpeq2(r[i] & fm2, pat) & __vcmpgtu2(r[i], 0x00010001u);
    m |= ((g & 1u) | ((g >> 15) & 2u)) << (2 * i);
  }
  return m;
}

template <bool CGL>
__device__ __forceinline__ void load16(const uint16_t *blk, uint32_t (&r)[8]) {
  load_chunk<32, CGL>(blk, r);
}

// commit_insert on exclusively reserved blocks, mask form (same policy)
__device__ __forceinline__ uint8_t commit_insert16(const TcfDev &P, uint32_t b1, uint32_t b2, uint16_t word,
                                                   const uint32_t (&r1)[8]) {
  uint16_t *blocks = reinterpret_cast<uint16_t *>(P.blocks);
  uint16_t *blk1 = blocks + (uint64_t)b1 * 16, *blk2 = blocks + (uint64_t)b2 * 16;
  uint32_t l1 = live16(r1);
  int u1 = __popc(l1);
  if (u1 < P.cut) {  // cut <= B, so a free slot exists
    blk1[__ffs(~l1 & 0xFFFFu) - 1] = word;
    return kPrimary;
  }
  uint32_t r2[8];
  load16<true>(blk2, r2);
  uint32_t l2 = live16(r2);
  bool first1 = u1 <= __popc(l2);
  uint32_t fa = ~(first1 ? l1 : l2) & 0xFFFFu, fb = ~(first1 ? l2 : l1) & 0xFFFFu;
  if (fa) {
    (first1 ? blk1 : blk2)[__ffs(fa) - 1] = word;
    return (first1 || b1 == b2) ? kPrimary : kSecondary;
  }
  if (fb) {
    (first1 ? blk2 : blk1)[__ffs(fb) - 1] = word;
    return (!first1 || b1 == b2) ? kPrimary : kSecondary;
  }
  return 4;
}

__device__ __forceinline__ int commit_delete16(const TcfDev &P, uint32_t b1, uint32_t b2, uint32_t tag,
                                               const uint32_t (&r1)[8]) {
  uint16_t *blocks = reinterpret_cast<uint16_t *>(P.blocks);
  const uint32_t fm = (uint32_t)(P.fmask & 0xFFFFu);
  uint32_t m = match16(r1, tag, fm);
  if (m) {
    blocks[(uint64_t)b1 * 16 + __ffs(m) - 1] = 1;
    return 1;
  }
  uint32_t r2[8];
  load16<true>(blocks + (uint64_t)b2 * 16, r2);
  m = match16(r2, tag, fm);
  if (m) {
    blocks[(uint64_t)b2 * 16 + __ffs(m) - 1] = 1;
    return 1;
  }
  return 0;
}


// ---------------------------------------------------------------------------
// concurrent (free-threaded CAS) insert / delete
// ---------------------------------------------------------------------------

// Claim the lowest free slot of a block snapshot by CAS, ascending; a lost CAS
// moves on to the next candidate (ck:150-171).  Returns true on success.
template <typename S, int G, int BF>
__device__ __forceinline__ bool tile_claim_cas(const Tile<G> &t, const Chunk<S, G, BF> &c, S *blk,
                                               uint64_t word) {
  int j0 = 0;
  for (;;) {
    int j = c.first_free(j0);
    unsigned bal = t.ballot(j >= 0);
    if (!bal) return false;
    int leader = __ffs(bal) - 1;
    int ok = 0;
    if ((int)t.lane == leader) {
      ok = cas_slot<S>(blk + c.lo + j, (S)c.at(j), (S)word) ? 1 : 0;
      j0 = j + 1;
    }
    ok = t.bcast(ok, leader);
    if (ok) return true;
  }
}

template <typename S>
__device__ __forceinline__ bool backing_claim_cas(const TcfDev &P, uint64_t fp, uint64_t word) {
  if (!P.bsize) return false;
  S *bk = reinterpret_cast<S *>(P.backing);
  uint64_t p = fmod64(mix64(fp ^ kBackStart), P.bsm);
  uint64_t step = fmod64(mix64(fp ^ kBackStep) | 1, P.bsm);
  for (int q = 0; q < P.probe_limit; q++) {
    uint64_t w = *(volatile S *)(bk + p);
    if (!live_word(w) && cas_slot<S>(bk + p, (S)w, (S)word)) return true;
    p += step;
    p = p >= P.bsize ? p - P.bsize : p;
  }
  return false;
}

template <typename S, int G, int BF>
__global__ void __launch_bounds__(256)
    k_tcf_insert_cas(TcfDev P, const uint64_t *__restrict__ keys, const uint64_t *__restrict__ values, int64_t n,
                     uint8_t *__restrict__ codes, int64_t *__restrict__ counters) {
  Tile<G> t;
  S *blocks = reinterpret_cast<S *>(P.blocks);
  int64_t tiles = (int64_t)gridDim.x * (blockDim.x / G);
  long long n_ok = 0, n_back = 0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; i < n; i += tiles) {
    KeyInfo k = key_info(P, keys[i]);
    uint64_t word = (P.f >= 64 ? 0 : ((values ? values[i] : 0) << P.f)) | k.tag;
    S *blk1 = blocks + k.b1 * (uint64_t)P.B;
    S *blk2 = blocks + k.b2 * (uint64_t)P.B;
    uint8_t code = kFull;
    Chunk<S, G, BF> c1;
    c1.template load<true>(blk1, P.B, t.lane);
    int u1 = t.sum(c1.used());
    if (u1 < P.cut && tile_claim_cas<S, G, BF>(t, c1, blk1, word)) {
      code = kPrimary;  // shortcut (ck:216-218)
    } else {
      c1.template load<true>(blk1, P.B, t.lane);
      Chunk<S, G, BF> c2;
      c2.template load<true>(blk2, P.B, t.lane);
      int o1 = t.sum(c1.used()), o2 = t.sum(c2.used());
      bool first1 = o1 <= o2;  // tie -> primary (ck:222-227)
      if (tile_claim_cas<S, G, BF>(t, first1 ? c1 : c2, first1 ? blk1 : blk2, word)) {
        code = (first1 || k.b1 == k.b2) ? kPrimary : kSecondary;
      } else if (tile_claim_cas<S, G, BF>(t, first1 ? c2 : c1, first1 ? blk2 : blk1, word)) {
        code = (!first1 || k.b1 == k.b2) ? kPrimary : kSecondary;
      } else {
        int ok = 0;
        if (t.lane == 0) ok = backing_claim_cas<S>(P, k.fp, word) ? 1 : 0;
        if (t.bcast(ok, 0)) code = kBacking;
      }
    }
    if (t.lane == 0) {
      codes[i] = code;
      n_ok += code != kFull;
      n_back += code == kBacking;
    }
  }
  cta_add_u64((unsigned long long *)&counters[0], (unsigned long long)n_ok);
  cta_add_u64((unsigned long long *)&counters[1], (unsigned long long)n_back);
}

template <typename S, int G, int BF>
__global__ void __launch_bounds__(256)
    k_tcf_delete_cas(TcfDev P, const uint64_t *__restrict__ keys, int64_t n, uint8_t *__restrict__ removed,
                     int64_t *__restrict__ counters) {
  Tile<G> t;
  S *blocks = reinterpret_cast<S *>(P.blocks);
  int64_t tiles = (int64_t)gridDim.x * (blockDim.x / G);
  long long n_del = 0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; i < n; i += tiles) {
    KeyInfo k = key_info(P, keys[i]);
    bool done = false;
    const bool fast = kFast16<S, G, BF> && P.f == 16;  // slot word == tag: the CAS expects the tag
    if (fast) {
#pragma unroll 1
      for (int which = 0; which < 2 && !done; which++) {
        uint16_t *blk = reinterpret_cast<uint16_t *>(blocks + (which ? k.b2 : k.b1) * (uint64_t)P.B);
        uint32_t r[8];
        load16<true>(blk, r);
        uint32_t m = match16(r, (uint32_t)k.tag, (uint32_t)(P.fmask & 0xFFFFu));
        while (m) {  // first live match, next match on a lost race (ck:328-339)
          int j = __ffs(m) - 1;
          m &= m - 1;
          if (cas_slot<uint16_t>(blk + j, (uint16_t)k.tag, (uint16_t)1)) {
            done = true;
            break;
          }
        }
      }
    }
#pragma unroll 1
    for (int which = 0; which < 2 && !done && !fast; which++) {
      S *blk = blocks + (which ? k.b2 : k.b1) * (uint64_t)P.B;
      Chunk<S, G, BF> c;
      c.template load<true>(blk, P.B, t.lane);
      int j0 = 0;
      for (;;) {  // first live match, CAS to TOMBSTONE, next match on a lost race (ck:328-339)
        int j = c.first_match(j0, k.tag, P.fmask);
        unsigned bal = t.ballot(j >= 0);
        if (!bal) break;
        int leader = __ffs(bal) - 1;
        int ok = 0;
        if ((int)t.lane == leader) {
          ok = cas_slot<S>(blk + c.lo + j, (S)c.at(j), (S)1) ? 1 : 0;
          j0 = j + 1;
        }
        if (t.bcast(ok, leader)) {
          done = true;
          break;
        }
      }
    }
    if (!done && P.bsize && t.lane == 0) {
      S *bk = reinterpret_cast<S *>(P.backing);
      uint64_t p = fmod64(mix64(k.fp ^ kBackStart), P.bsm);
      uint64_t step = fmod64(mix64(k.fp ^ kBackStep) | 1, P.bsm);
      for (int q = 0; q < P.probe_limit; q++) {
        uint64_t w = *(volatile S *)(bk + p);
        if (w == 0) break;
        if (w != 1 && (w & P.fmask) == k.tag && cas_slot<S>(bk + p, (S)w, (S)1)) {
          done = true;
          break;
        }
        p += step;
        p = p >= P.bsize ? p - P.bsize : p;
      }
    }
    if (t.lane == 0) {
      removed[i] = done ? 1 : 0;
      n_del += done;
    }
  }
  cta_add_u64((unsigned long long *)&counters[2], (unsigned long long)n_del);
}

// ---------------------------------------------------------------------------
// ordered (sequential-semantics) insert / delete: persistent cooperative kernel
// ---------------------------------------------------------------------------

struct OrdScratch {
  uint32_t *res;        // per-block reservation word (min pending input index)
  uint32_t *bres;       // per-backing-slot reservation word
  uint32_t *carry[2];   // keys carried to the next round (double-buffered)
  uint32_t *defer_idx;  // input indices deferred to the backing phase (unordered)
  uint8_t *defer_pend;
  unsigned int *ctl;    // [0..1] carry counts, [2] defer count, [3..4] backing-phase round flags,
                        // [5] main rounds, [6] backing rounds, [7] keys carried (sum over rounds)
  int64_t defer_cap;
  int64_t window;       // keys introduced per round
  int res_shift;        // reservation granularity: 2^res_shift blocks per word
  int hints;            // 1: L2 evict_last on reservation words, evict_first on streams
  int ctas_per_sm;      // 0: occupancy limit; else cap (fewer grid-barrier participants)
  int prefetch;         // 1: the reserve pass prefetches each key's b1 block into L2
  uint32_t *res2;       // one-barrier kernel: reservation words of odd rounds
  int slots;            // one-barrier kernel: keys held per thread (<= KB)
  int held_only;        // one-barrier kernel: clear only the words a key holds (no no-op CAS)
};

// A control word every thread needs after a grid barrier, loaded once per
// CTA and broadcast through shared memory: one L2 request per CTA instead of
// one per warp to a single address (measured on the B200: 2^20-slot ordered
// insert 0.66 -> 0.58 ms, 2^24 1.60 -> 1.46 ms).  All threads must call.
__device__ __forceinline__ unsigned cta_ldcg(const unsigned *a) {
  __shared__ unsigned s_v;
  __syncthreads();  // (s_v is reused)
  if (threadIdx.x == 0) s_v = __ldcg(a);
  __syncthreads();
  return s_v;
}

// CTA-wide OR of a predicate (all threads of the CTA must call).
__device__ __forceinline__ bool cta_any(bool p) { return __syncthreads_or(p ? 1 : 0) != 0; }

template <typename S, int G, int BF>
__device__ __forceinline__ int tile_first_free(const Tile<G> &t, const Chunk<S, G, BF> &c, int *slot) {
  int j = c.first_free(0);
  unsigned bal = t.ballot(j >= 0);
  if (!bal) return 0;
  int leader = __ffs(bal) - 1;
  *slot = t.bcast(j >= 0 ? c.lo + j : 0, leader);
  return 1;
}

// True when the b1 block alone decides a key's op (insert: b1 below the cut
// line; delete: the tag is live in b1): the op then touches b1 only, so a key
// holding its b1 reservation may commit without its b2 one (pk:132-134,
// pk:213-218) -- no earlier
// pending key touches b1 (it would hold a smaller bid there).  Tile-collective.
template <typename S, int G, int BF, int OP>
__device__ __forceinline__ bool b1_decides(const TcfDev &P, const Tile<G> &t, const Chunk<S, G, BF> &c1,
                                           uint64_t tag) {
  if (OP == 0) return t.sum(c1.used()) < P.cut;
  return t.ballot(c1.first_match(0, tag, P.fmask) >= 0) != 0;
}

// The sequential insert policy (pk:126-148) on exclusively reserved blocks.
// Returns the placement code, or 4 = "both blocks full, defer to backing".
template <typename S, int G, int BF>
__device__ __forceinline__ uint8_t commit_insert(const TcfDev &P, const Tile<G> &t, uint32_t b1, uint32_t b2,
                                                 uint64_t word, const Chunk<S, G, BF> &c1) {
  S *blocks = reinterpret_cast<S *>(P.blocks);
  S *blk1 = blocks + (uint64_t)b1 * P.B, *blk2 = blocks + (uint64_t)b2 * P.B;
  int u1 = t.sum(c1.used());
  int slot;
  if (u1 < P.cut) {
    tile_first_free<S, G, BF>(t, c1, &slot);  // cut <= B, so a free slot exists
    if (t.lane == 0) blk1[slot] = (S)word;
    return kPrimary;
  }
  Chunk<S, G, BF> c2;
  c2.template load<true>(blk2, P.B, t.lane);
  int u2 = t.sum(c2.used());
  bool first1 = u1 <= u2;
  if (tile_first_free<S, G, BF>(t, first1 ? c1 : c2, &slot)) {
    if (t.lane == 0) (first1 ? blk1 : blk2)[slot] = (S)word;
    return (first1 || b1 == b2) ? kPrimary : kSecondary;
  }
  if (tile_first_free<S, G, BF>(t, first1 ? c2 : c1, &slot)) {
    if (t.lane == 0) (first1 ? blk2 : blk1)[slot] = (S)word;
    return (!first1 || b1 == b2) ? kPrimary : kSecondary;
  }
  return 4;
}

// The sequential delete (pk:207-222) on exclusively reserved blocks:
// tombstone the first live match of b1, else of b2.  1 = done, 0 = defer.
template <typename S, int G, int BF>
__device__ __forceinline__ int commit_delete(const TcfDev &P, const Tile<G> &t, uint32_t b1, uint32_t b2,
                                             uint64_t tag, const Chunk<S, G, BF> &c1) {
  S *blocks = reinterpret_cast<S *>(P.blocks);
#pragma unroll 1
  for (int which = 0; which < 2; which++) {
    S *blk = blocks + (uint64_t)(which ? b2 : b1) * P.B;
    Chunk<S, G, BF> c;
    if (which) c.template load<true>(blk, P.B, t.lane);
    else c = c1;
    int j = c.first_match(0, tag, P.fmask);
    unsigned bal = t.ballot(j >= 0);
    if (bal) {
      int leader = __ffs(bal) - 1;
      if ((int)t.lane == leader) blk[c.lo + j] = (S)1;
      return 1;
    }
  }
  return 0;
}

// Recompute a deferred key's fingerprint and slot word / tag from the inputs.
template <int OP>
__device__ __forceinline__ void deferred_key(const TcfDev &P, const uint64_t *keys, const uint64_t *values,
                                             uint32_t i, uint64_t *fp, uint64_t *word) {
  uint64_t key = keys[i];
  *fp = P.keys_are_fps ? key : mix64(key ^ P.seed);
  uint64_t tag = remap_tag(*fp, P.fmask);
  *word = OP == 0 ? ((P.f >= 64 ? 0 : ((values ? values[i] : 0) << P.f)) | tag) : tag;
}

// Backing phase of the ordered kernels: deferred keys (both blocks full on
// insert / no match on delete) claim backing positions in input-index order
// by reservations over probe positions (pk:104-117, pk:223-233).  Returns
// the round counter after the phase.
template <typename S, int G, int OP>
__device__ __forceinline__ unsigned ordered_backing_phase(const TcfDev &P, const uint64_t *__restrict__ keys,
                                                          const uint64_t *__restrict__ values,
                                                          uint8_t *__restrict__ out, const OrdScratch &X,
                                                          const Tile<G> &t, int64_t tiles, int64_t tid,
                                                          cg::grid_group &grid, unsigned round, long long *n_a,
                                                          long long *n_b) {
  grid.sync();
  int64_t nd = (int64_t)cta_ldcg(&X.ctl[2]);
  if (nd > X.defer_cap) nd = X.defer_cap;
  S *bk = reinterpret_cast<S *>(P.backing);
  if (nd > 0) {
    for (;;) {
      // reserve every position this key could still take: for inserts all
      // free probe positions, for deletes all live matches before the chain
      // ends (pk:104-117, pk:223-233)
      for (int64_t e = tid; e < nd; e += tiles) {
        if (t.lane != 0 || !__ldcg(&X.defer_pend[e])) continue;
        uint32_t idx = __ldcg(&X.defer_idx[e]);
        uint64_t fp, word;
        deferred_key<OP>(P, keys, values, idx, &fp, &word);
        if (!P.bsize) continue;
        uint64_t p = fmod64(mix64(fp ^ kBackStart), P.bsm);
        uint64_t step = fmod64(mix64(fp ^ kBackStep) | 1, P.bsm);
        for (int q = 0; q < P.probe_limit; q++) {
          uint64_t w = load_slot<S, true>(bk + p);
          if (OP == 0) {
            if (!live_word(w)) atomicMin(&X.bres[p], idx);
          } else {
            if (w == 0) break;
            if (w != 1 && (w & P.fmask) == word) atomicMin(&X.bres[p], idx);
          }
          p += step;
          p = p >= P.bsize ? p - P.bsize : p;
        }
      }
      grid.sync();
      bool left = false;
      for (int64_t e = tid; e < nd; e += tiles) {
        if (t.lane != 0 || !__ldcg(&X.defer_pend[e])) continue;
        uint32_t idx = __ldcg(&X.defer_idx[e]);
        int64_t i = idx;
        uint64_t fp, word;
        deferred_key<OP>(P, keys, values, idx, &fp, &word);
        int64_t target = -1;
        if (P.bsize) {
          uint64_t p = fmod64(mix64(fp ^ kBackStart), P.bsm);
          uint64_t step = fmod64(mix64(fp ^ kBackStep) | 1, P.bsm);
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
        }
        if (target < 0) {  // nothing claimable now, nor ever in this batch
          out[i] = OP == 0 ? kFull : 0;
          X.defer_pend[e] = 0;
          continue;
        }
        if (__ldcg(&X.bres[target]) != idx) {
          left = true;
          continue;
        }
        bk[target] = (S)(OP == 0 ? word : 1);
        out[i] = OP == 0 ? kBacking : 1;
        (*n_a)++;
        *n_b += OP == 0;
        X.defer_pend[e] = 0;
        // release every reservation still carrying our index
        uint64_t p = fmod64(mix64(fp ^ kBackStart), P.bsm);
        uint64_t step = fmod64(mix64(fp ^ kBackStep) | 1, P.bsm);
        for (int q = 0; q < P.probe_limit; q++) {
          atomicCAS(&X.bres[p], idx, kNoRes);
          p += step;
          p = p >= P.bsize ? p - P.bsize : p;
        }
      }
      bool any = cta_any(left);
      if (threadIdx.x == 0) {
        if (any) atomicAdd(&X.ctl[3 + (round & 1)], 1u);
        if (blockIdx.x == 0) X.ctl[3 + ((round + 1) & 1)] = 0;
      }
      grid.sync();
      unsigned cnt = cta_ldcg(&X.ctl[3 + (round & 1)]);
      round++;
      if (cnt == 0) break;
    }
  }
  return round;
}

template <typename S, int G, int BF, int KB, int OP>
__global__ void __launch_bounds__(256, 4)
    k_tcf_ordered(TcfDev P, const uint64_t *__restrict__ keys, const uint64_t *__restrict__ values, int64_t n,
                  uint8_t *__restrict__ out, int64_t *__restrict__ counters, OrdScratch X) {
  // Sliding-window deterministic reservations.  Every round introduces the
  // next input indices [F, F+room) (all keys below the frontier F are thus
  // introduced) plus the keys carried over from the previous round; each
  // bids its input index on both blocks (atomicMin), and after a grid
  // barrier a key that holds both commits -- every earlier key that could
  // change those blocks has committed already -- while the others are
  // carried.  The minimum pending index always commits, so the carry is
  // bounded by the window; no round is spent draining a window tail.
  cg::grid_group grid = cg::this_grid();
  Tile<G> t;
  const int64_t tiles = (int64_t)gridDim.x * (blockDim.x / G);
  const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t Wn = X.window;
  long long n_a = 0;  // insert: placed in a block; delete: removed
  int64_t F = 0;
  int64_t nc = 0;
  int cur = 0;
  unsigned round = 0;
  const uint64_t pol_keep = l2_evict_last(), pol_stream = l2_evict_first();

  for (;;) {
    int64_t room = Wn - nc;
    if (room < 0) room = 0;
    int64_t Fend = F + room < n ? F + room : n;
    int64_t total = (Fend - F) + nc;
    const uint32_t *cin = X.carry[cur];
    uint32_t *cout = X.carry[cur ^ 1];

    // ---- reserve --------------------------------------------------------
    // One chunk of KB keys per tile (the host caps the window at tiles*KB):
    // the key's blocks and tag stay in registers for the commit pass.
    uint32_t idx[KB], b1[KB], b2[KB];
    uint64_t tg[KB];
    bool ok[KB], hold[KB];
#pragma unroll
    for (int j = 0; j < KB; j++) {
      int64_t e = tid + (int64_t)j * tiles;
      ok[j] = e < total;
      idx[j] = ok[j] ? (e < nc ? __ldcg(cin + e) : (uint32_t)(F + e - nc)) : 0u;
    }
#pragma unroll
    for (int j = 0; j < KB; j++) {
      b1[j] = b2[j] = 0;
      tg[j] = 0;
      if (!ok[j]) continue;
      KeyInfo ki = key_info(P, X.hints ? ld_stream_u64(keys + idx[j], pol_stream) : keys[idx[j]]);
      b1[j] = (uint32_t)ki.b1;
      b2[j] = (uint32_t)ki.b2;
      tg[j] = ki.tag;
      // the commit pass reads b1 after the barrier: start the DRAM fetch now
      if (X.prefetch && t.lane == 0)
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(reinterpret_cast<const S *>(P.blocks) +
                                                                 (uint64_t)b1[j] * P.B));
    }
    if (t.lane == 0) {
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!ok[j]) continue;
        uint32_t g1 = b1[j] >> X.res_shift, g2 = b2[j] >> X.res_shift;
        if (X.hints) {
          red_min_u32(&X.res[g1], idx[j], pol_keep);
          if (g2 != g1) red_min_u32(&X.res[g2], idx[j], pol_keep);
        } else {
          atomicMin(&X.res[g1], idx[j]);
          if (g2 != g1) atomicMin(&X.res[g2], idx[j]);
        }
      }
    }
    grid.sync();

    // ---- commit ---------------------------------------------------------
    if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[cur] = 0;  // list `cur` is consumed this round
    {
      bool hold2[KB];
#pragma unroll
      for (int j = 0; j < KB; j++) {
        hold[j] = ok[j] && (X.hints ? ld_cg_u32(&X.res[b1[j] >> X.res_shift], pol_keep)
                                    : __ldcg(&X.res[b1[j] >> X.res_shift])) == idx[j];
        hold2[j] = ok[j] && (X.hints ? ld_cg_u32(&X.res[b2[j] >> X.res_shift], pol_keep)
                                     : __ldcg(&X.res[b2[j] >> X.res_shift])) == idx[j];
      }
      constexpr bool fast = kFast16<S, G, BF>;
      constexpr int KC = fast ? 1 : KB;      // generic path: one Chunk per key
      constexpr int KR = fast ? KB : 1;      // fast path: 8 registers per key
      Chunk<S, G, BF> c1[KC];
      uint32_t r1[KR][8];
      S *blocks = reinterpret_cast<S *>(P.blocks);
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!hold[j]) continue;
        if constexpr (fast) load16<true>(reinterpret_cast<uint16_t *>(blocks) + (uint64_t)b1[j] * 16, r1[j]);
        else c1[j].template load<true>(blocks + (uint64_t)b1[j] * P.B, P.B, t.lane);
      }
      // commit with both words, or with the b1 word when b1 decides the op
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!hold[j] || hold2[j]) continue;
        bool d;
        if constexpr (fast) d = OP == 0 ? __popc(live16(r1[j])) < P.cut
                                        : match16(r1[j], (uint32_t)tg[j], (uint32_t)(P.fmask & 0xFFFFu)) != 0;
        else d = b1_decides<S, G, BF, OP>(P, t, c1[j], tg[j]);
        hold[j] = d;
        hold2[j] = false;  // (not ours: leave the b2 word to its holder)
      }

      // carry the losers: one warp-aggregated atomicAdd (every lane joins)
      {
        unsigned mine = 0;
#pragma unroll
        for (int j = 0; j < KB; j++) mine += (ok[j] && !hold[j] && t.lane == 0) ? 1u : 0u;
        unsigned lane = threadIdx.x & 31;
        unsigned incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          unsigned v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if ((int)lane >= o) incl += v;
        }
        unsigned total_w = __shfl_sync(0xFFFFFFFFu, incl, 31);
        unsigned basepos = 0;
        if (lane == 31 && total_w) basepos = atomicAdd(&X.ctl[cur ^ 1], total_w);
        basepos = __shfl_sync(0xFFFFFFFFu, basepos, 31);
        unsigned pos = basepos + incl - mine;
#pragma unroll
        for (int j = 0; j < KB; j++)
          if (ok[j] && !hold[j] && t.lane == 0) cout[pos++] = idx[j];
      }
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!hold[j]) continue;
        bool defer;
        if (OP == 0) {
          uint64_t word = (P.f >= 64 || !values ? 0 : (values[idx[j]] << P.f)) | tg[j];
          uint8_t code;
          if constexpr (fast) code = commit_insert16(P, b1[j], b2[j], (uint16_t)word, r1[j]);
          else code = commit_insert<S, G, BF>(P, t, b1[j], b2[j], word, c1[j]);
          defer = code == 4;
          if (!defer && t.lane == 0) {
            out[idx[j]] = code;
            n_a++;
          }
        } else {
          int done;
          if constexpr (fast) done = commit_delete16(P, b1[j], b2[j], (uint32_t)tg[j], r1[j]);
          else done = commit_delete<S, G, BF>(P, t, b1[j], b2[j], tg[j], c1[j]);
          defer = !done && P.bsize;
          if (!defer && t.lane == 0) {
            out[idx[j]] = done ? 1 : 0;
            n_a += done;
          }
        }
        if (t.lane == 0) {
          if (defer) {
            unsigned slot = atomicAdd(&X.ctl[2], 1u);
            if (slot < X.defer_cap) {
              X.defer_idx[slot] = idx[j];
              X.defer_pend[slot] = 1;
            }
          }
          // only the holder writes these words now
          if (X.hints) {
            st_u32(&X.res[b1[j] >> X.res_shift], kNoRes, pol_keep);
            if (hold2[j]) st_u32(&X.res[b2[j] >> X.res_shift], kNoRes, pol_keep);
          } else {
            X.res[b1[j] >> X.res_shift] = kNoRes;
            if (hold2[j]) X.res[b2[j] >> X.res_shift] = kNoRes;
          }
        }
      }
    }
    grid.sync();
    nc = (int64_t)cta_ldcg(&X.ctl[cur ^ 1]);
    cur ^= 1;
    F = Fend;
    round++;
    if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[7] += (unsigned)nc;
    if (F >= n && nc == 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[5] = round;
  const unsigned main_rounds = round;

  long long n_b = 0;
  round = ordered_backing_phase<S, G, OP>(P, keys, values, out, X, t, tiles, tid, grid, round, &n_a, &n_b);
  if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[6] = round - main_rounds;
  // (only tile leaders count)
  if (OP == 0) {
    cta_add_u64((unsigned long long *)&counters[0], (unsigned long long)n_a);
    cta_add_u64((unsigned long long *)&counters[1], (unsigned long long)n_b);
  } else {
    cta_add_u64((unsigned long long *)&counters[2], (unsigned long long)n_a);
  }
}

// ---------------------------------------------------------------------------
// One-barrier ordered kernel (u16 slots, B = 16, G = 1: the benchmarked
// geometry).  Same deterministic reservations as k_tcf_ordered, restructured
// so a round needs one grid barrier instead of two:
//   * reservation words alternate between two arrays (even / odd rounds);
//   * every thread keeps its pending keys in registers (no carry list): after
//     committing round r it immediately grabs new input indices (a global
//     atomic frontier, so introduced keys always form a prefix of the input)
//     and bids for round r+1 into the other array, then waits at the barrier;
//   * a key that loses a round retracts its own bids (CAS idx -> free) and a
//     holder releases its words, so an array is clean when its next round
//     starts -- that round's bids begin only after the next barrier.
// Correctness is the same argument: a key commits only holding both words of
// its round, i.e. no earlier pending key touches its blocks, and every
// earlier key is either committed (before an earlier barrier) or pending
// (and bid this round).  ctl[8..10] count pending keys per round (mod 3),
// ctl[11] is the frontier.
// ---------------------------------------------------------------------------
template <int KB, int OP>
__global__ void __launch_bounds__(256, 4)
    k_tcf_ordered1(TcfDev P, const uint64_t *__restrict__ keys, const uint64_t *__restrict__ values, int64_t n,
                   uint8_t *__restrict__ out, int64_t *__restrict__ counters, OrdScratch X) {
  cg::grid_group grid = cg::this_grid();
  Tile<1> t;
  const int64_t tiles = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t pol_keep = l2_evict_last(), pol_stream = l2_evict_first();
  uint16_t *blocks = reinterpret_cast<uint16_t *>(P.blocks);
  const int rs = X.res_shift;
  uint32_t idx[KB], b1[KB], b2[KB], tg[KB];
  bool pend[KB];
#pragma unroll
  for (int j = 0; j < KB; j++) {
    pend[j] = false;
    idx[j] = b1[j] = b2[j] = tg[j] = 0;
  }
  long long n_a = 0;
  unsigned losses = 0;
  unsigned r = 0;
  __shared__ unsigned s_warp[32];
  __shared__ unsigned s_base;

  // this lane's first new input index for `need` slots: one frontier atomic
  // per CTA (a single L2 address takes every grab), so the introduced keys
  // always form a prefix of the input
  auto grab = [&](unsigned need) -> unsigned {
    unsigned incl = need;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)lane >= o) incl += v;
    }
    __syncthreads();  // s_warp / s_base are reused
    if (lane == 31) s_warp[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned acc = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
        unsigned v = s_warp[w];
        s_warp[w] = acc;
        acc += v;
      }
      s_base = acc ? atomicAdd(&X.ctl[11], acc) : 0u;
    }
    __syncthreads();
    return s_base + s_warp[threadIdx.x >> 5] + incl - need;
  };

  // round 0's keys
  {
    unsigned nx = grab((unsigned)X.slots);
#pragma unroll
    for (int j = 0; j < KB; j++) {
      if (j < X.slots && (int64_t)nx < n) {
        idx[j] = nx;
        pend[j] = true;
        KeyInfo ki = key_info(P, ld_stream_u64(keys + nx, pol_stream));
        b1[j] = (uint32_t)ki.b1;
        b2[j] = (uint32_t)ki.b2;
        tg[j] = (uint32_t)ki.tag;
      }
      nx += j < X.slots ? 1u : 0u;
    }
  }

  for (;;) {
    // ---- bid for round r ----------------------------------------------------
    {
      uint32_t *R = (r & 1) ? X.res2 : X.res;
      unsigned mine = 0;
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!pend[j]) continue;
        mine++;
        uint32_t g1 = b1[j] >> rs, g2 = b2[j] >> rs;
        red_min_u32(&R[g1], idx[j], pol_keep);
        if (g2 != g1) red_min_u32(&R[g2], idx[j], pol_keep);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xFFFFFFFFu, mine, o);
      __syncthreads();  // s_warp is reused
      if (lane == 0) s_warp[threadIdx.x >> 5] = mine;
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned acc = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) acc += s_warp[w];
        if (acc) atomicAdd(&X.ctl[8 + r % 3], acc);
      }
    }
    grid.sync();
    const unsigned total = cta_ldcg(&X.ctl[8 + r % 3]);

    // ---- commit round r, refill from the frontier for round r+1 -------------
    // A key holding its b1 word commits when it also holds its b2 word, or
    // when its b1 block alone decides the op (insert: b1 below the cut line;
    // delete: the tag is live in b1) -- the op then touches b1 only, and no
    // earlier pending key touches b1 (it would hold a smaller bid there).
    {
      uint32_t *R = (r & 1) ? X.res2 : X.res;
      bool hold[KB], hold2[KB];
      uint32_t rb[KB][8];
#pragma unroll
      for (int j = 0; j < KB; j++) {
        hold[j] = pend[j] && ld_cg_u32(&R[b1[j] >> rs], pol_keep) == idx[j];
        hold2[j] = pend[j] && ld_cg_u32(&R[b2[j] >> rs], pol_keep) == idx[j];
        if (hold[j]) load16<true>(blocks + (uint64_t)b1[j] * 16, rb[j]);
      }
      // (no thread has a pending key when total == 0, so nothing was loaded)
      if (total == 0) break;
      if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[8 + (r + 2) % 3] = 0;
      bool go[KB];
#pragma unroll
      for (int j = 0; j < KB; j++) {
        bool b1_decides = false;
        if (hold[j] && !hold2[j]) {
          if (OP == 0) b1_decides = __popc(live16(rb[j])) < P.cut;
          else b1_decides = match16(rb[j], tg[j], (uint32_t)(P.fmask & 0xFFFFu)) != 0;
        }
        go[j] = hold[j] && (hold2[j] || b1_decides);
      }
      // Refill early: the slots of this round's committers and the empty
      // slots take the next input indices now, so the frontier atomic and the
      // key loads overlap the commits below.
      bool refill[KB];
      unsigned need = 0;
#pragma unroll
      for (int j = 0; j < KB; j++) {
        refill[j] = j < X.slots && (!pend[j] || go[j]);
        need += refill[j] ? 1u : 0u;
      }
      unsigned nx = grab(need);
      uint64_t nk[KB];
      {
        unsigned k = 0;
#pragma unroll
        for (int j = 0; j < KB; j++) {
          nk[j] = 0;
          if (!refill[j]) continue;
          if ((int64_t)(nx + k) < n) nk[j] = ld_stream_u64(keys + nx + k, pol_stream);
          k++;
        }
      }
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!pend[j]) continue;
        uint32_t g1 = b1[j] >> rs, g2 = b2[j] >> rs;
        if (!go[j]) {  // lost: retract our own bids so the array is clean
          if (X.held_only) {
            // a word's minimum bidder always clears it (release or this
            // retraction), so a bid on a word held by another key is gone
            // once that key clears it: only the words we hold need a store
            if (hold[j]) st_u32(&R[g1], kNoRes, pol_keep);
            if (g2 != g1 && hold2[j]) st_u32(&R[g2], kNoRes, pol_keep);
          } else {
            atomicCAS(&R[g1], idx[j], kNoRes);
            if (g2 != g1) atomicCAS(&R[g2], idx[j], kNoRes);
          }
          losses++;
          continue;
        }
        bool defer;
        if (OP == 0) {
          uint64_t word = (P.f >= 64 || !values ? 0 : (values[idx[j]] << P.f)) | tg[j];
          uint8_t code = commit_insert16(P, b1[j], b2[j], (uint16_t)word, rb[j]);
          defer = code == 4;
          if (!defer) {
            out[idx[j]] = code;
            n_a++;
          }
        } else {
          int done = commit_delete16(P, b1[j], b2[j], tg[j], rb[j]);
          defer = !done && P.bsize;
          if (!defer) {
            out[idx[j]] = done ? 1 : 0;
            n_a += done;
          }
        }
        if (defer) {
          unsigned slot = atomicAdd(&X.ctl[2], 1u);
          if (slot < X.defer_cap) {
            X.defer_idx[slot] = idx[j];
            X.defer_pend[slot] = 1;
          }
        }
        // release the b1 word; the b2 word only if we hold it, else retract
        // our bid there (an earlier key holds it)
        st_u32(&R[g1], kNoRes, pol_keep);
        if (g2 != g1) {
          if (hold2[j]) st_u32(&R[g2], kNoRes, pol_keep);
          else if (!X.held_only) atomicCAS(&R[g2], idx[j], kNoRes);
        }
        pend[j] = false;
      }
      // install the new keys (slot order = input order within this lane)
      unsigned k = 0;
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!refill[j]) continue;
        unsigned i = nx + k;
        k++;
        if ((int64_t)i >= n) continue;
        idx[j] = i;
        pend[j] = true;
        KeyInfo ki = key_info(P, nk[j]);
        b1[j] = (uint32_t)ki.b1;
        b2[j] = (uint32_t)ki.b2;
        tg[j] = (uint32_t)ki.tag;
      }
    }
    r++;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[5] = r;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) losses += __shfl_xor_sync(0xFFFFFFFFu, losses, o);
  if (lane == 0 && losses) atomicAdd(&X.ctl[7], losses);

  long long n_b = 0;
  unsigned round = ordered_backing_phase<uint16_t, 1, OP>(P, keys, values, out, X, t, tiles, tid, grid, r, &n_a,
                                                          &n_b);
  if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[6] = round - r;
  if (OP == 0) {
    cta_add_u64((unsigned long long *)&counters[0], (unsigned long long)n_a);
    cta_add_u64((unsigned long long *)&counters[1], (unsigned long long)n_b);
  } else {
    cta_add_u64((unsigned long long *)&counters[2], (unsigned long long)n_a);
  }
}

// Dispatch over (G, compile-time B) for one slot type -------------------------
// BF=16 is the vectorised fast path for the default/benchmarked geometry
// (B=16); BF=32 the CG-32 sweep point (B=32, u16); everything else BF=0.
// keys per tile per round in the ordered kernel: 2 on the register-resident
// G=1 path (4 spills at the 64-register cap of 4 CTAs/SM), 4 otherwise
// ---------------------------------------------------------------------------
// Multi-pass ordered kernel for cooperative groups of G >= 2 lanes.  Same
// rounds and reservations as k_tcf_ordered, but the reserve and commit passes
// each stream the window in chunks of KB keys per tile and the commit pass
// re-derives the key's blocks and tag from the (L2-resident) window keys, so
// the window is not capped at one chunk per tile.  Measured at 2^28 slots
// (profiles/r1g_cg_ordered.txt): G = 2 6.6 G inserts/s vs 4.0 for the
// register-held kernel, G = 8 3.7 vs 2.0; G = 1 is the other way round.
template <typename S, int G, int BF, int KB, int OP>
__global__ void __launch_bounds__(256, 4)
    k_tcf_ordered_mp(TcfDev P, const uint64_t *__restrict__ keys, const uint64_t *__restrict__ values, int64_t n,
                     uint8_t *__restrict__ out, int64_t *__restrict__ counters, OrdScratch X) {
  cg::grid_group grid = cg::this_grid();
  Tile<G> t;
  const int64_t tiles = (int64_t)gridDim.x * (blockDim.x / G);
  const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t Wn = X.window;
  long long n_a = 0;  // insert: placed in a block; delete: removed
  int64_t F = 0;
  int64_t nc = 0;
  int cur = 0;
  unsigned round = 0;
  const uint64_t pol_keep = l2_evict_last(), pol_stream = l2_evict_first();

  for (;;) {
    int64_t room = Wn - nc;
    if (room < 0) room = 0;
    int64_t Fend = F + room < n ? F + room : n;
    int64_t total = (Fend - F) + nc;
    const uint32_t *cin = X.carry[cur];
    uint32_t *cout = X.carry[cur ^ 1];

    // ---- reserve --------------------------------------------------------
    for (int64_t base = tid; base < total; base += tiles * KB) {
      uint32_t idx[KB], b1[KB], b2[KB];
      bool ok[KB];
#pragma unroll
      for (int j = 0; j < KB; j++) {
        int64_t e = base + (int64_t)j * tiles;
        ok[j] = e < total;
        idx[j] = ok[j] ? (e < nc ? __ldcg(cin + e) : (uint32_t)(F + e - nc)) : 0u;
      }
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!ok[j]) continue;
        KeyInfo ki = key_info(P, X.hints ? ld_stream_u64(keys + idx[j], pol_stream) : keys[idx[j]]);
        b1[j] = (uint32_t)ki.b1;
        b2[j] = (uint32_t)ki.b2;
      }
      if (t.lane == 0) {
#pragma unroll
        for (int j = 0; j < KB; j++) {
          if (!ok[j]) continue;
          uint32_t g1 = b1[j] >> X.res_shift, g2 = b2[j] >> X.res_shift;
          if (X.hints) {
            red_min_u32(&X.res[g1], idx[j], pol_keep);
            if (g2 != g1) red_min_u32(&X.res[g2], idx[j], pol_keep);
          } else {
            atomicMin(&X.res[g1], idx[j]);
            if (g2 != g1) atomicMin(&X.res[g2], idx[j]);
          }
        }
      }
    }
    grid.sync();

    // ---- commit ---------------------------------------------------------
    if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[cur] = 0;  // list `cur` is consumed this round
    for (int64_t base = tid;; base += tiles * KB) {
      // warp-uniform trip count: lanes past the end still join the shuffles
      if (!__any_sync(0xFFFFFFFFu, base < total)) break;
      uint32_t idx[KB], b1[KB], b2[KB];
      uint64_t word[KB];
      bool ok[KB], hold[KB], hold2[KB];
#pragma unroll
      for (int j = 0; j < KB; j++) {
        int64_t e = base + (int64_t)j * tiles;
        ok[j] = e < total;
        idx[j] = ok[j] ? (e < nc ? __ldcg(cin + e) : (uint32_t)(F + e - nc)) : 0u;
      }
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!ok[j]) continue;
        KeyInfo ki = key_info(P, X.hints ? ld_stream_u64(keys + idx[j], pol_stream) : keys[idx[j]]);
        b1[j] = (uint32_t)ki.b1;
        b2[j] = (uint32_t)ki.b2;
        word[j] = OP == 0 ? ((P.f >= 64 ? 0 : ((values ? values[idx[j]] : 0) << P.f)) | ki.tag) : ki.tag;
      }
#pragma unroll
      for (int j = 0; j < KB; j++) {
        hold[j] = ok[j] && (X.hints ? ld_cg_u32(&X.res[b1[j] >> X.res_shift], pol_keep)
                                    : __ldcg(&X.res[b1[j] >> X.res_shift])) == idx[j];
        hold2[j] = ok[j] && (X.hints ? ld_cg_u32(&X.res[b2[j] >> X.res_shift], pol_keep)
                                     : __ldcg(&X.res[b2[j] >> X.res_shift])) == idx[j];
      }
      Chunk<S, G, BF> c1[KB];
      S *blocks = reinterpret_cast<S *>(P.blocks);
#pragma unroll
      for (int j = 0; j < KB; j++)
        if (hold[j]) c1[j].template load<true>(blocks + (uint64_t)b1[j] * P.B, P.B, t.lane);
      // commit with both words, or with the b1 word when b1 decides the op
      // (the tag bits of word[] are the tag for either op)
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!hold[j] || hold2[j]) continue;
        hold[j] = b1_decides<S, G, BF, OP>(P, t, c1[j], word[j] & P.fmask);
      }
      // carry the losers: one warp-aggregated atomicAdd per pass
      {
        unsigned mine = 0;
#pragma unroll
        for (int j = 0; j < KB; j++) mine += (ok[j] && !hold[j] && t.lane == 0) ? 1u : 0u;
        unsigned lane = threadIdx.x & 31;
        unsigned incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          unsigned v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if ((int)lane >= o) incl += v;
        }
        unsigned total_w = __shfl_sync(0xFFFFFFFFu, incl, 31);
        unsigned basepos = 0;
        if (lane == 31 && total_w) basepos = atomicAdd(&X.ctl[cur ^ 1], total_w);
        basepos = __shfl_sync(0xFFFFFFFFu, basepos, 31);
        unsigned pos = basepos + incl - mine;
#pragma unroll
        for (int j = 0; j < KB; j++)
          if (ok[j] && !hold[j] && t.lane == 0) cout[pos++] = idx[j];
      }
#pragma unroll
      for (int j = 0; j < KB; j++) {
        if (!ok[j] || !hold[j]) continue;
        bool defer;
        if (OP == 0) {
          uint8_t code = commit_insert<S, G, BF>(P, t, b1[j], b2[j], word[j], c1[j]);
          defer = code == 4;
          if (!defer && t.lane == 0) {
            out[idx[j]] = code;
            n_a++;
          }
        } else {
          int done = commit_delete<S, G, BF>(P, t, b1[j], b2[j], word[j], c1[j]);
          defer = !done && P.bsize;
          if (!defer && t.lane == 0) {
            out[idx[j]] = done ? 1 : 0;
            n_a += done;
          }
        }
        if (t.lane == 0) {
          if (defer) {
            unsigned slot = atomicAdd(&X.ctl[2], 1u);
            if (slot < X.defer_cap) {
              X.defer_idx[slot] = idx[j];
              X.defer_pend[slot] = 1;
            }
          }
          // only the holder writes these words now
          if (X.hints) {
            st_u32(&X.res[b1[j] >> X.res_shift], kNoRes, pol_keep);
            if (hold2[j]) st_u32(&X.res[b2[j] >> X.res_shift], kNoRes, pol_keep);
          } else {
            X.res[b1[j] >> X.res_shift] = kNoRes;
            if (hold2[j]) X.res[b2[j] >> X.res_shift] = kNoRes;
          }
        }
      }
    }
    grid.sync();
    nc = (int64_t)cta_ldcg(&X.ctl[cur ^ 1]);
    cur ^= 1;
    F = Fend;
    round++;
    if (F >= n && nc == 0) break;
  }

  if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[5] = round;
  const unsigned main_rounds = round;

  long long n_b = 0;
  round = ordered_backing_phase<S, G, OP>(P, keys, values, out, X, t, tiles, tid, grid, round, &n_a, &n_b);
  if (blockIdx.x == 0 && threadIdx.x == 0) X.ctl[6] = round - main_rounds;
  // (only tile leaders count)
  if (OP == 0) {
    cta_add_u64((unsigned long long *)&counters[0], (unsigned long long)n_a);
    cta_add_u64((unsigned long long *)&counters[1], (unsigned long long)n_b);
  } else {
    cta_add_u64((unsigned long long *)&counters[2], (unsigned long long)n_a);
  }
}


template <int G>
constexpr int kOrdKB = G == 1 ? 2 : 4;

template <typename S, int G, int BF, int OP>
constexpr auto ord_kernel() {
  if constexpr (G > 1) return k_tcf_ordered_mp<S, G, BF, kOrdKB<G>, OP>;
  else return k_tcf_ordered<S, G, BF, kOrdKB<G>, OP>;
}

template <typename S, int G, int BF, int OP>
static int launch_ordered(const TcfDev &P, const uint64_t *keys, const uint64_t *values, int64_t n, uint8_t *out,
                          int64_t *counters, OrdScratch X, cudaStream_t st) {
  if constexpr (kFast16<S, G, BF>) {
    auto k1 = k_tcf_ordered1<kOrdKB<1>, OP>;
    int per_sm = 0;
    FK_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1, 256, 0));
    if (per_sm < 1) return FK_E_ARG;
    if (X.ctas_per_sm > 0 && X.ctas_per_sm < per_sm) per_sm = X.ctas_per_sm;
    int grid = per_sm * num_sms();
    int64_t thr = (int64_t)grid * 256;
    // one-barrier kernel when the window gives at least every fourth thread
    // a key (its window is grid * 256 * slots, slots = the nearest whole
    // number, >= 1); smaller windows keep the carry-list kernel, whose window
    // is exact (measured, profiles/r1g_ord_tune_small.jsonl: 2^22 slots,
    // window 65 K for 76 K threads, 3.5 vs 2.7 G inserts/s; 2^20, 16 K for
    // 38 K, 1.1-1.3 vs 0.9-1.0)
    // (its 32-bit frontier may overshoot n by a round's grabs: keep clear of 2^32)
    if (X.res2 && 4 * X.window >= thr && n < (int64_t)0xFFFFFFFFLL - 4 * thr * kOrdKB<1>) {
      int slots = (int)((X.window + thr / 2) / thr);  // (clamped to >= 1 below)
      X.slots = slots < 1 ? 1 : (slots > kOrdKB<1> ? kOrdKB<1> : slots);
      void *args[] = {(void *)&P, (void *)&keys, (void *)&values, (void *)&n, (void *)&out, (void *)&counters,
                      (void *)&X};
      FK_TRY(cudaLaunchCooperativeKernel((const void *)k1, dim3(grid), dim3(256), args, 0, st));
      return 0;
    }
  }
  // G >= 2: the multi-pass kernel; G = 1: the register-held kernel, whose
  // window is one chunk of kOrdKB<1> keys per tile and round
  constexpr bool mp = G > 1;
  auto kern = ord_kernel<S, G, BF, OP>();
  int per_sm = 0;
  FK_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
  if (per_sm < 1) return FK_E_ARG;
  if (X.ctas_per_sm > 0 && X.ctas_per_sm < per_sm) per_sm = X.ctas_per_sm;
  int grid = per_sm * num_sms();
  int64_t cap = (int64_t)grid * (256 / G) * kOrdKB<G>;
  if (!mp && X.window > cap) X.window = cap;
  void *args[] = {(void *)&P, (void *)&keys, (void *)&values, (void *)&n, (void *)&out, (void *)&counters, (void *)&X};
  FK_TRY(cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(256), args, 0, st));
  return 0;
}

static inline int grid_for(int64_t n, int G) {
  int64_t tiles_per_cta = 256 / G;
  int64_t need = (n + tiles_per_cta - 1) / tiles_per_cta;
  int64_t cap = (int64_t)num_sms() * 8;
  if (need > cap) need = cap;
  return (int)(need < 1 ? 1 : need);
}

enum TcfOp { kOpQuery = 0, kOpInsCas = 1, kOpDelCas = 2, kOpInsOrd = 3, kOpDelOrd = 4 };

struct TcfCall {
  const uint64_t *keys;
  const uint64_t *values;
  int64_t n;
  uint8_t *out;
  uint64_t *vals_out;
  int64_t *counters;
  OrdScratch X;
};

template <typename S, int G, int BF>
static int tcf_run_gb(int op, const TcfDev &P, const TcfCall &c, cudaStream_t st) {
  int grid = grid_for(c.n, G);
  switch (op) {
    case kOpQuery:
      k_tcf_query<S, G, BF><<<grid, 256, 0, st>>>(P, c.keys, c.n, c.out, c.vals_out);
      break;
    case kOpInsCas:
      k_tcf_insert_cas<S, G, BF><<<grid, 256, 0, st>>>(P, c.keys, c.values, c.n, c.out, c.counters);
      break;
    case kOpDelCas:
      k_tcf_delete_cas<S, G, BF><<<grid, 256, 0, st>>>(P, c.keys, c.n, c.out, c.counters);
      break;
    case kOpInsOrd:
      return launch_ordered<S, G, BF, 0>(P, c.keys, c.values, c.n, c.out, c.counters, c.X, st);
    default:
      return launch_ordered<S, G, BF, 1>(P, c.keys, nullptr, c.n, c.out, c.counters, c.X, st);
  }
  FK_CHECK_LAUNCH();
  return 0;
}

template <typename S, int BF>
static int tcf_run_b(int op, int G, const TcfDev &P, const TcfCall &c, cudaStream_t st) {
  switch (G) {
    case 1: return tcf_run_gb<S, 1, BF>(op, P, c, st);
    case 2: return tcf_run_gb<S, 2, BF>(op, P, c, st);
    case 4: return tcf_run_gb<S, 4, BF>(op, P, c, st);
    case 8: return tcf_run_gb<S, 8, BF>(op, P, c, st);
    case 16: return tcf_run_gb<S, 16, BF>(op, P, c, st);
    default: return tcf_run_gb<S, 32, (BF == 16 ? 0 : BF)>(op, P, c, st);
  }
}

// One explicit instantiation per slot type lives in tcf_point_s{1,2,4,8}.cu so
// the (type x G x B) kernel matrix compiles in parallel.
template <typename S>
int tcf_run(int op, int G, int B, const TcfDev &P, const TcfCall &c, cudaStream_t st) {
  if constexpr (sizeof(S) == 2) {
    if (B == 16) return tcf_run_b<S, 16>(op, G, P, c, st);
    if (B == 32) return tcf_run_b<S, 32>(op, G, P, c, st);
  }
  return tcf_run_b<S, 0>(op, G, P, c, st);
}

}  // namespace fk
