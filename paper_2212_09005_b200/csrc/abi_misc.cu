// abi_misc.cu -- version, hashing-parity and inspection entry points of the C ABI.
#include <cub/cub.cuh>

#include "../../include/filterkit_b200.h"
#include "fk_common.cuh"
#include "fk_scratch.cuh"

namespace fk {

// slot i holds a live word (> TOMBSTONE); with fill (sorted bulk blocks):
// i lies in its block's filled prefix
struct LiveSlot {
  const void *slots;
  int bytes;
  const uint32_t *fill;
  int B;
  __device__ bool operator()(int64_t i) const {
    if (fill) return (uint32_t)(i % B) < fill[i / B];
    switch (bytes) {
      case 1: return reinterpret_cast<const uint8_t *>(slots)[i] > 1;
      case 2: return reinterpret_cast<const uint16_t *>(slots)[i] > 1;
      case 4: return reinterpret_cast<const uint32_t *>(slots)[i] > 1;
      default: return reinterpret_cast<const uint64_t *>(slots)[i] > 1;
    }
  }
};

// fp, b1, b2, backing start, backing step per key (hashing.py:66-117).
__global__ void k_hash_streams(const uint64_t *__restrict__ keys, int64_t n, uint64_t seed, uint64_t fpmask,
                               uint64_t nb, FastMod nbm, uint64_t bs, FastMod bsm, uint64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t fp = mix64(keys[i] ^ seed) & fpmask;
    out[5 * i] = fp;
    out[5 * i + 1] = nb ? fmod64(mix64(fp ^ kBlock1), nbm) : 0;
    out[5 * i + 2] = nb ? fmod64(mix64(fp ^ kBlock2), nbm) : 0;
    out[5 * i + 3] = bs ? fmod64(mix64(fp ^ kBackStart), bsm) : 0;
    out[5 * i + 4] = bs ? fmod64(mix64(fp ^ kBackStep) | 1, bsm) : 0;
  }
}

__global__ void k_fastmod(const uint64_t *__restrict__ x, int64_t n, FastMod m, uint64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fmod64(x[i], m);
}

// Random 32-byte sector gather over a table: the random-access ceiling the
// filter kernels are measured against (same hash stream, same sector size,
// same 256-bit loads, run on the filter's own table in the same process).
__global__ void __launch_bounds__(256) k_sector_gather(const uint32_t *__restrict__ table, uint64_t nsec, FastMod m,
                                                       int64_t n, uint64_t salt, uint32_t *__restrict__ sink) {
  uint32_t acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t b = fmod64(mix64((uint64_t)i ^ salt), m);
    uint32_t r[8];
    load_chunk<32, false>(table + 8 * b, r);
#pragma unroll
    for (int j = 0; j < 8; j++) acc ^= r[j];
  }
  if (acc == 0x9E3779B9u) sink[blockIdx.x & 31] = acc;  // keeps the loads live
}

// Random 32-byte sector read-modify-write: load a random sector, bump one
// 16-bit word of it, store it back -- the access pattern of a TCF insert or
// delete that lands in its first block (the measured ceiling for those ops).
__global__ void __launch_bounds__(256) k_sector_rmw(uint32_t *__restrict__ table, uint64_t nsec, FastMod m,
                                                    int64_t n, uint64_t salt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = mix64((uint64_t)i ^ salt);
    uint64_t b = fmod64(h, m);
    uint32_t r[8];
    load_chunk<32, true>(table + 8 * b, r);
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) x += r[j];
    uint16_t *w = reinterpret_cast<uint16_t *>(table + 8 * b) + (h >> 60);
    *w = (uint16_t)(x | 2);
  }
}

// counter_stream (workloads.py:23-26): mix64(mix64(seed ^ tag) + i) for
// i in [start, start + n) -- the uniform key generator, exactly distinct.
// Two keys per thread as one 128-bit store.
__global__ void __launch_bounds__(256) k_counter_stream(uint64_t base, int64_t n, uint64_t *__restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * p < n; p += stride) {
    int64_t i = 2 * p;
    uint64_t a = mix64(base + (uint64_t)i);
    if (i + 1 < n && (((uintptr_t)(out + i)) & 15) == 0) {
      ulonglong2 v;
      v.x = a;
      v.y = mix64(base + (uint64_t)i + 1);
      *reinterpret_cast<ulonglong2 *>(out + i) = v;
    } else {
      out[i] = a;
      if (i + 1 < n) out[i + 1] = mix64(base + (uint64_t)i + 1);
    }
  }
}

}  // namespace fk

using namespace fk;

extern "C" {

const char *fk_version(void) { return "filterkit-b200 0.1.0 (sm_100a)"; }
int fk_abi_version(void) { return FK_ABI_VERSION; }

int fk_device_setup(int l2_fetch_bytes) {
  // Random 32-byte block probes are the whole TCF/GQF access pattern; the
  // default L2 fetch granularity would turn every miss into a 64-128 B DRAM
  // read.  This is a per-context hint (cudaLimitMaxL2FetchGranularity).
  if (l2_fetch_bytes > 0) FK_TRY(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)l2_fetch_bytes));
  // Batch pipelines take their scratch from the device's default memory pool
  // (cudaMallocAsync).  With the default release threshold of 0 the pool
  // hands memory back to the driver at every stream synchronisation and the
  // next batch pays for re-mapping it; keep it cached instead.
  int dev = 0;
  FK_TRY(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  FK_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = ~0ULL;
  FK_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  return 0;
}

int fk_device_l2_fetch_bytes(void) {
  size_t v = 0;
  if (cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity) != cudaSuccess) return -1;
  return (int)v;
}

int fk_hash_streams(const uint64_t *keys, int64_t n, uint64_t seed, int bits, uint64_t nb, uint64_t bsize,
                    uint64_t *out5, void *stream) {
  if (n < 0 || bits < 1 || bits > 64) return FK_E_ARG;
  if (n == 0) return 0;
  uint64_t m = bits >= 64 ? ~0ULL : ((1ULL << bits) - 1);
  int grid = (int)((n + 255) / 256);
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  k_hash_streams<<<grid, 256, 0, (cudaStream_t)stream>>>(keys, n, seed, m, nb, make_fastmod(nb ? nb : 1), bsize,
                                                         make_fastmod(bsize ? bsize : 1), out5);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_counter_stream(uint64_t seed, uint64_t tag, uint64_t start, int64_t n, uint64_t *out, void *stream) {
  if (n < 0 || (n && !out)) return FK_E_ARG;
  if (n == 0) return 0;
  int64_t pairs = (n + 1) / 2;
  int64_t blocks = (pairs + 255) / 256;
  int cap = num_sms() * 8;
  k_counter_stream<<<(int)(blocks < cap ? blocks : cap), 256, 0, (cudaStream_t)stream>>>(mix64(seed ^ tag) + start, n,
                                                                                      out);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_sector_gather(const void *table, int64_t table_bytes, int64_t n, uint64_t salt, uint32_t *sink,
                     void *stream) {
  if (n < 0 || table_bytes < 32 || ((uintptr_t)table & 31)) return FK_E_ARG;
  if (n == 0) return 0;
  uint64_t nsec = (uint64_t)table_bytes / 32;
  int grid = num_sms() * 8;
  k_sector_gather<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint32_t *)table, nsec, make_fastmod(nsec), n, salt,
                                                          sink);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_sector_rmw(void *table, int64_t table_bytes, int64_t n, uint64_t salt, void *stream) {
  if (n < 0 || table_bytes < 32 || ((uintptr_t)table & 31)) return FK_E_ARG;
  if (n == 0) return 0;
  uint64_t nsec = (uint64_t)table_bytes / 32;
  k_sector_rmw<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>((uint32_t *)table, nsec, make_fastmod(nsec), n, salt);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_fastmod_check(const uint64_t *x, int64_t n, uint64_t d, uint64_t *out, void *stream) {
  if (n < 0 || d == 0) return FK_E_ARG;
  if (n == 0) return 0;
  int grid = (int)((n + 255) / 256);
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  k_fastmod<<<grid, 256, 0, (cudaStream_t)stream>>>(x, n, make_fastmod(d), out);
  FK_CHECK_LAUNCH();
  return 0;
}

// k-mer windows (fk/workloads.py:147-191) on the device: seq holds the
// reads' bases, reads separated by a non-ACGT byte, so a window is valid
// iff its k bytes are all ACGT (either case); valid windows are kept in
// position order by the stream compaction.
__device__ __forceinline__ int base_code(uint8_t c) {
  switch (c | 0x20) {  // lowercase
    case 'a': return 0;
    case 'c': return 1;
    case 'g': return 2;
    case 't': return 3;
    default: return -1;
  }
}

__global__ void k_kmer_windows(const uint8_t *__restrict__ seq, int64_t m, int k, uint64_t *__restrict__ val,
                               uint8_t *__restrict__ ok) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t v = 0;
    bool good = true;
    for (int j = 0; j < k; j++) {
      const int c = base_code(seq[i + j]);
      good &= c >= 0;
      v = (v << 2) | (uint64_t)(c & 3);
    }
    val[i] = v;
    ok[i] = good ? 1 : 0;
  }
}

// Tcf.items / BulkTcf.items on the device (fk/tcf.py:196-208,
// fk/tcf_bulk.py:342-352): positions of the live slots, ascending.
int fk_live_slots(const void *slots, int slot_bytes, int64_t n, const uint32_t *fill, int block_slots,
                  int64_t *idx_out, int64_t *count, void *stream) {
  if (n < 0 || !idx_out || !count || (fill && block_slots < 1)) return FK_E_ARG;
  if (slot_bytes != 1 && slot_bytes != 2 && slot_bytes != 4 && slot_bytes != 8) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {
    FK_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    return 0;
  }
  Scratch S(st);
  LiveSlot pred{slots, slot_bytes, fill, block_slots};
  cub::CountingInputIterator<int64_t> it(0);
  size_t tb = 0;
  FK_TRY(cub::DeviceSelect::If(nullptr, tb, it, idx_out, count, n, pred, st));
  void *tmp = S.get<char>(tb);
  if (!tmp) return -(int)S.err;
  FK_TRY(cub::DeviceSelect::If(tmp, tb, it, idx_out, count, n, pred, st));
  return 0;
}

int fk_kmer_windows(const uint8_t *seq, int64_t n, int k, uint64_t *out, int64_t *count, void *stream) {
  if (n < 0 || k < 1 || k > 32 || !out || !count) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t m = n - k + 1;
  if (m <= 0) {
    FK_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    return 0;
  }
  Scratch S(st);
  uint64_t *val = S.get<uint64_t>(m);
  uint8_t *ok = S.get<uint8_t>(m);
  if (S.err) return -(int)S.err;
  int64_t g = (m + 255) / 256, cap = (int64_t)num_sms() * 16;
  k_kmer_windows<<<(int)(g < cap ? g : cap), 256, 0, st>>>(seq, m, k, val, ok);
  FK_CHECK_LAUNCH();
  size_t tb = 0;
  FK_TRY(cub::DeviceSelect::Flagged(nullptr, tb, val, ok, out, count, m, st));
  void *tmp = S.get<char>(tb);
  if (!tmp) return -(int)S.err;
  FK_TRY(cub::DeviceSelect::Flagged(tmp, tb, val, ok, out, count, m, st));
  return 0;
}

}  // extern "C"
