// fk_common.cuh -- shared device helpers for the B200 filter kernels.
//
// Hashing here is bit-identical to the reference's host hashing
// (/root/reference/pkg/src/filterkit/hashing.py:22-154); every derived stream
// (fingerprint, block pair, backing schedule, GQF quotient/remainder, tag
// remap) is computed on the device, fused into the kernel that consumes it.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fk {

namespace cg = cooperative_groups;

// hashing.py:22-25
constexpr uint64_t kBlock1 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kBlock2 = 0xC2B2AE3D27D4EB4FULL;
constexpr uint64_t kBackStart = 0x165667B19E3779F9ULL;
constexpr uint64_t kBackStep = 0x27D4EB2F165667C5ULL;

// Placement codes (tcf.py:31-37) and GQF codes (_pykernels.py:37-40).
constexpr uint8_t kPrimary = 0, kSecondary = 1, kBacking = 2, kFull = 3;
constexpr int kRegionBits = 13;
constexpr int64_t kRegionSlots = 1LL << kRegionBits;

// hashing.py:28-36 (SplitMix64 finalizer)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// Exact x % d for a runtime 64-bit divisor without the ~70-instruction
// software division: q = umulhi(x, floor((2^64-1)/d)) undershoots floor(x/d)
// by at most 2, fixed by two conditional subtracts.  Powers of two take the
// mask path.  (exhaustively checked in tests/test_hashing_gpu.py.)
struct FastMod {
  uint64_t d;
  uint64_t m;     // floor((2^64-1)/d), unused for powers of two
  uint64_t mask;  // d-1 when d is a power of two, else 0
  int pow2;
};

inline FastMod make_fastmod(uint64_t d) {
  FastMod f;
  f.d = d ? d : 1;
  f.pow2 = (f.d & (f.d - 1)) == 0;
  f.mask = f.pow2 ? f.d - 1 : 0;
  f.m = f.pow2 ? 0 : (~0ULL) / f.d;
  return f;
}

__device__ __forceinline__ uint64_t fmod64(uint64_t x, const FastMod &f) {
  if (f.pow2) return x & f.mask;
  uint64_t q = __umul64hi(x, f.m);
  uint64_t r = x - q * f.d;
  r = r >= f.d ? r - f.d : r;
  r = r >= f.d ? r - f.d : r;
  return r;
}

// hashing.py:120-132
__device__ __forceinline__ uint64_t remap_tag(uint64_t fp, uint64_t fmask) {
  uint64_t t = fp & fmask;
  return t < 2 ? (t | 2) : t;
}

__device__ __forceinline__ bool live_word(uint64_t w) { return w > 1; }

// --- atomics on every slot width --------------------------------------------
template <typename S>
__device__ __forceinline__ bool cas_slot(S *p, S expected, S desired);

template <>
__device__ __forceinline__ bool cas_slot<uint8_t>(uint8_t *p, uint8_t e, uint8_t v) {
  // no 8-bit CAS: CAS the aligned 32-bit word, retrying while only the other
  // three bytes change underneath us.
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  unsigned int *w = reinterpret_cast<unsigned int *>(a & ~uintptr_t(3));
  unsigned int sh = (unsigned int)(a & 3) * 8;
  unsigned int old = *(volatile unsigned int *)w;
  for (;;) {
    if (((old >> sh) & 0xFF) != e) return false;
    unsigned int nw = (old & ~(0xFFu << sh)) | ((unsigned int)v << sh);
    unsigned int got = atomicCAS(w, old, nw);
    if (got == old) return true;
    old = got;
  }
}
template <>
__device__ __forceinline__ bool cas_slot<uint16_t>(uint16_t *p, uint16_t e, uint16_t v) {
  return atomicCAS(reinterpret_cast<unsigned short *>(p), (unsigned short)e, (unsigned short)v) == e;
}
template <>
__device__ __forceinline__ bool cas_slot<uint32_t>(uint32_t *p, uint32_t e, uint32_t v) {
  return atomicCAS(reinterpret_cast<unsigned int *>(p), e, v) == e;
}
template <>
__device__ __forceinline__ bool cas_slot<uint64_t>(uint64_t *p, uint64_t e, uint64_t v) {
  return atomicCAS(reinterpret_cast<unsigned long long *>(p), (unsigned long long)e,
                   (unsigned long long)v) == e;
}

// --- raw byte-chunk loads (vectorised when the chunk is naturally aligned) --
// Loads NB bytes at p into regs[] (NB a power of two).  ld.global.nc is NOT
// used for tables that the same kernel mutates.
// CG=true loads through L2 only (ld.global.cg): used by the persistent
// ordered kernels, whose tables are rewritten by other SMs between grid
// barriers, so a stale L1 line must never be read.
template <int NB, bool CG = false>
__device__ __forceinline__ void load_chunk(const void *p, uint32_t *regs) {
  if constexpr (NB % 32 == 0) {
    // one 256-bit LDG per 32-byte sector (sm_100 LDG.E.256): a TCF block of
    // 16 x u16 is exactly one request
#pragma unroll
    for (int i = 0; i < NB / 32; i++) {
      const uint32_t *q = reinterpret_cast<const uint32_t *>(p) + 8 * i;
      uint32_t *r = regs + 8 * i;
      if constexpr (CG) {
        asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                       "=r"(r[7])
                     : "l"(q));
      } else {
        asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                       "=r"(r[7])
                     : "l"(q));
      }
    }
  } else if constexpr (NB >= 16) {
#pragma unroll
    for (int i = 0; i < NB / 16; i++) {
      const uint4 *q = reinterpret_cast<const uint4 *>(p) + i;
      uint4 v = CG ? __ldcg(q) : *q;
      regs[4 * i] = v.x; regs[4 * i + 1] = v.y; regs[4 * i + 2] = v.z; regs[4 * i + 3] = v.w;
    }
  } else if constexpr (NB == 8) {
    const uint2 *q = reinterpret_cast<const uint2 *>(p);
    uint2 v = CG ? __ldcg(q) : *q;
    regs[0] = v.x; regs[1] = v.y;
  } else if constexpr (NB == 4) {
    const unsigned int *q = reinterpret_cast<const unsigned int *>(p);
    regs[0] = CG ? __ldcg(q) : *q;
  } else if constexpr (NB == 2) {
    const unsigned short *q = reinterpret_cast<const unsigned short *>(p);
    regs[0] = CG ? __ldcg(q) : *q;
  } else {
    const unsigned char *q = reinterpret_cast<const unsigned char *>(p);
    regs[0] = CG ? __ldcg(q) : *q;
  }
}

template <typename S, bool CG>
__device__ __forceinline__ uint64_t load_slot(const S *p) {
  if constexpr (sizeof(S) == 8) {
    const unsigned long long *q = reinterpret_cast<const unsigned long long *>(p);
    return CG ? __ldcg(q) : *q;
  } else if constexpr (sizeof(S) == 4) {
    const unsigned int *q = reinterpret_cast<const unsigned int *>(p);
    return CG ? __ldcg(q) : *q;
  } else if constexpr (sizeof(S) == 2) {
    const unsigned short *q = reinterpret_cast<const unsigned short *>(p);
    return CG ? __ldcg(q) : *q;
  } else {
    const unsigned char *q = reinterpret_cast<const unsigned char *>(p);
    return CG ? __ldcg(q) : *q;
  }
}

template <typename S>
__device__ __forceinline__ void set_reg_slot(uint32_t *regs, int i, uint64_t v) {
  if constexpr (sizeof(S) == 8) {
    regs[2 * i] = (uint32_t)v;
    regs[2 * i + 1] = (uint32_t)(v >> 32);
  } else if constexpr (sizeof(S) == 4) {
    regs[i] = (uint32_t)v;
  } else if constexpr (sizeof(S) == 2) {
    int s = (i & 1) * 16;
    regs[i >> 1] = (regs[i >> 1] & ~(0xFFFFu << s)) | ((uint32_t)v << s);
  } else {
    int s = (i & 3) * 8;
    regs[i >> 2] = (regs[i >> 2] & ~(0xFFu << s)) | ((uint32_t)v << s);
  }
}

template <typename S>
__device__ __forceinline__ uint64_t reg_slot(const uint32_t *regs, int i) {
  if constexpr (sizeof(S) == 8) {
    return (uint64_t)regs[2 * i] | ((uint64_t)regs[2 * i + 1] << 32);
  } else if constexpr (sizeof(S) == 4) {
    return regs[i];
  } else if constexpr (sizeof(S) == 2) {
    return (regs[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
  } else {
    return (regs[i >> 2] >> ((i & 3) * 8)) & 0xFFu;
  }
}

// --- L2 cache-policy hints (createpolicy + .L2::cache_hint) -----------------
// Small, hot side structures (reservation words) are kept with evict_last so
// that the stream of random table sectors (evict_first) does not push them
// out of L2.
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void red_min_u32(uint32_t *a, uint32_t v, uint64_t pol) {
  asm volatile("red.relaxed.gpu.global.min.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t *a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_u32(uint32_t *a, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t *a, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}

// Sum of a per-thread count over the CTA, added to *dst with one atomic per
// CTA.  Per-thread or per-warp atomics on one address serialise at its L2
// slice (151 K threads end the C3 ordered kernels).  Every thread of the
// CTA must call (blockDim.x a multiple of 32).
__device__ __forceinline__ void cta_add_u64(unsigned long long *dst, unsigned long long v) {
  __shared__ unsigned long long s_part[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  __syncthreads();  // (s_part is reused)
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_part[w];
    if (t) atomicAdd(dst, t);
  }
}

// Error plumbing for the C ABI: never throw, return a negative cudaError_t.
#define FK_CHECK_LAUNCH()                                 \
  do {                                                    \
    cudaError_t e_ = cudaGetLastError();                  \
    if (e_ != cudaSuccess) return -(int)e_;               \
  } while (0)

#define FK_TRY(expr)                                      \
  do {                                                    \
    cudaError_t e_ = (expr);                              \
    if (e_ != cudaSuccess) return -(int)e_;               \
  } while (0)

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace fk
