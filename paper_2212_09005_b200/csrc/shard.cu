// shard.cu -- hash-prefix sharding of key batches across GPUs.
//
// The reference is single-process; this is the new build's scale-out path.
// A key's owner is a prefix of its fingerprint: for the TCF the top log2(G)
// bits of mix64(key ^ seed) (b1, b2, tag and backing schedule all come from
// other hash streams, so each shard is an independent Tcf(num_blocks / G));
// for the GQF the top log2(G) quotient bits, i.e. bits [q' + r, q + r) with
// q' = q - log2(G), so the shard's own Gqf(q', r) sees exactly the low
// q' + r fingerprint bits and its counts equal a global Gqf(q, r)'s.
//
// fk_shard_partition stably groups a batch by owner (one-digit CUB radix
// sort of the owner ids, then a gather of keys and optional 64-bit values)
// and counts per owner; the caller exchanges the groups either over peer
// memory (fk_shard_dispatch / fk_shard_combine / fk_shard_signal /
// fk_shard_wait, below) or with one NCCL all-to-all.  fk_shard_unpermute
// scatters the per-key results that come back into input order.
#include <cub/cub.cuh>
#include <string.h>

#include "../../include/filterkit_b200.h"
#include "fk_common.cuh"
#include "fk_scratch.cuh"

namespace fk {
namespace {

inline int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

__global__ void k_owner(const uint64_t *__restrict__ keys, int64_t n, uint64_t seed, int shift, uint32_t gmask,
                        uint8_t *__restrict__ owner, uint32_t *__restrict__ iota,
                        unsigned long long *__restrict__ counts) {
  __shared__ unsigned int hist[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = mix64(keys[i] ^ seed);
    uint32_t o = shift >= 64 ? 0u : (uint32_t)(h >> shift) & gmask;
    owner[i] = (uint8_t)o;
    iota[i] = (uint32_t)i;
    atomicAdd(&hist[o], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= (int)gmask; i += blockDim.x)
    if (hist[i]) atomicAdd(&counts[i], (unsigned long long)hist[i]);
}

__global__ void k_gather2(const uint64_t *__restrict__ keys, const uint64_t *__restrict__ vals,
                          const uint32_t *__restrict__ perm, int64_t n, uint64_t *__restrict__ keys_out,
                          uint64_t *__restrict__ vals_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t p = perm[i];
    keys_out[i] = keys[p];
    if (vals) vals_out[i] = vals[p];
  }
}

template <typename T>
__global__ void k_unpermute(const uint32_t *__restrict__ perm, const T *__restrict__ src, int64_t n,
                            T *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[perm[i]] = src[i];
}

// Fused exchange over peer memory (CUDA IPC mappings of the other ranks'
// buffers; NVLink / NVSwitch stores between GPUs).
//   dispatch: the gather of the stable owner partition writes every key (8 B,
//     plus its value if any) straight into its owner's receive buffer, at this
//     rank's offset there.  The receive layout -- sources in rank order, each
//     source's keys in its input order -- identifies every key's source and
//     position, so no tag travels with it.
//   combine: the owner writes each received key's result straight into its
//     source's return buffer, at the key's position in the source's
//     owner-grouped order: one contiguous run per (owner, source) pair; the
//     source restores its input order locally (fk_shard_unpermute).
//   signal / wait: stream-ordered cross-GPU handoff -- after the exchange
//     kernel, every rank stores an epoch into every peer's flag word for it
//     (system-scope release); the receiving stream spins (acquire) until all
//     sources reached the epoch.  No host synchronisation.
__global__ void k_dispatch(const uint64_t *__restrict__ keys, const uint64_t *__restrict__ vals,
                           const uint32_t *__restrict__ perm, int64_t n, uint64_t seed, int shift, uint32_t gmask,
                           const int64_t *__restrict__ seg_start, const int64_t *__restrict__ dst_off,
                           uint64_t *const *__restrict__ pk, uint64_t *const *__restrict__ pv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[i];
    const uint64_t k = keys[p];
    const uint32_t o = shift >= 64 ? 0u : (uint32_t)(mix64(k ^ seed) >> shift) & gmask;
    const int64_t j = dst_off[o] + (i - seg_start[o]);
    pk[o][j] = k;
    if (vals) pv[o][j] = vals[p];
  }
  __threadfence_system();
}

template <typename T>
__global__ void k_combine(const T *__restrict__ res, int64_t m, int G, const int64_t *__restrict__ recv_off,
                          const int64_t *__restrict__ back_off, T *const *__restrict__ pback) {
  __shared__ int64_t s_off[257], s_back[256];
  for (int s = threadIdx.x; s <= G; s += blockDim.x) {
    s_off[s] = recv_off[s];
    if (s < G) s_back[s] = back_off[s];
  }
  __syncthreads();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    int s = 0;
    while (s + 1 < G && j >= s_off[s + 1]) s++;
    pback[s][s_back[s] + (j - s_off[s])] = res[j];
  }
  __threadfence_system();
}

__global__ void k_signal(uint32_t *const *__restrict__ pflags, int G, uint32_t rank, uint32_t epoch) {
  const int o = threadIdx.x;
  if (o >= G) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pflags[o] + rank), "r"(epoch) : "memory");
}

__global__ void k_wait(const uint32_t *__restrict__ flags, int G, uint32_t epoch, unsigned long long timeout_ns) {
  const int s = threadIdx.x;
  if (s >= G) return;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + s) : "memory");
    if ((int32_t)(v - epoch) >= 0) break;
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) __trap();  // a peer never arrived: fail loudly instead of hanging
  }
}

}  // namespace
}  // namespace fk

using namespace fk;

extern "C" {

int fk_shard_partition(const uint64_t *keys, const uint64_t *vals, int64_t n, uint64_t seed, int shift, int log2_shards,
                       uint64_t *keys_out, uint64_t *vals_out, uint32_t *perm, int64_t *counts, void *stream) {
  if (n < 0 || n > 0xFFFFFFF0LL || log2_shards < 0 || log2_shards > 8 || shift < 0 || !counts) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  int G = 1 << log2_shards;
  FK_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * G, st));
  if (n == 0) return 0;
  Scratch S(st);
  uint8_t *owner = S.get<uint8_t>(n), *owner_s = S.get<uint8_t>(n);
  uint32_t *iota = S.get<uint32_t>(n);
  if (!owner || !owner_s || !iota) return -(int)S.err;
  int sh = log2_shards == 0 ? 64 : shift;
  k_owner<<<grid_for(n), 256, 0, st>>>(keys, n, seed, sh, (uint32_t)(G - 1), owner, iota,
                                       reinterpret_cast<unsigned long long *>(counts));
  FK_CHECK_LAUNCH();
  if (log2_shards == 0) {
    FK_TRY(cudaMemcpyAsync(perm, iota, 4 * (size_t)n, cudaMemcpyDeviceToDevice, st));
  } else {
    size_t tb = 0;
    FK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, owner, owner_s, iota, perm, n, 0, log2_shards, st));
    void *tmp = S.get<char>(tb);
    if (!tmp) return -(int)S.err;
    FK_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, owner, owner_s, iota, perm, n, 0, log2_shards, st));
  }
  if (keys_out) {  // the peer-memory path gathers inside fk_shard_dispatch instead
    k_gather2<<<grid_for(n), 256, 0, st>>>(keys, vals, perm, n, keys_out, vals_out);
    FK_CHECK_LAUNCH();
  }
  return 0;
}

int fk_shard_dispatch(const uint64_t *keys, const uint64_t *vals, const uint32_t *perm, int64_t n, uint64_t seed,
                      int shift, int log2_shards, const int64_t *seg_start, const int64_t *dst_off,
                      uint64_t *const *peer_keys, uint64_t *const *peer_vals, void *stream) {
  if (n < 0 || log2_shards < 0 || log2_shards > 8 || !peer_keys || (vals && !peer_vals)) return FK_E_ARG;
  if (n == 0) return 0;
  const int sh = log2_shards == 0 ? 64 : shift;
  k_dispatch<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(keys, vals, perm, n, seed, sh,
                                                            (uint32_t)((1 << log2_shards) - 1), seg_start, dst_off,
                                                            peer_keys, peer_vals);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_shard_combine(const void *res, int64_t m, int elem_bytes, int log2_shards, const int64_t *recv_off,
                     const int64_t *back_off, void *const *peer_back, void *stream) {
  if (m < 0 || log2_shards < 0 || log2_shards > 8 || !peer_back || !recv_off || !back_off) return FK_E_ARG;
  if (m == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int G = 1 << log2_shards;
  if (elem_bytes == 1)
    k_combine<uint8_t><<<grid_for(m), 256, 0, st>>>((const uint8_t *)res, m, G, recv_off, back_off,
                                                    (uint8_t *const *)peer_back);
  else if (elem_bytes == 8)
    k_combine<uint64_t><<<grid_for(m), 256, 0, st>>>((const uint64_t *)res, m, G, recv_off, back_off,
                                                     (uint64_t *const *)peer_back);
  else
    return FK_E_ARG;
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_shard_signal(uint32_t *const *peer_flags, int log2_shards, uint32_t rank, uint32_t epoch, void *stream) {
  if (!peer_flags || log2_shards < 0 || log2_shards > 8) return FK_E_ARG;
  const int G = 1 << log2_shards;
  k_signal<<<1, G < 32 ? 32 : G, 0, (cudaStream_t)stream>>>(peer_flags, G, rank, epoch);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_shard_wait(const uint32_t *flags, int log2_shards, uint32_t epoch, double timeout_s, void *stream) {
  if (!flags || log2_shards < 0 || log2_shards > 8 || timeout_s <= 0) return FK_E_ARG;
  const int G = 1 << log2_shards;
  k_wait<<<1, G < 32 ? 32 : G, 0, (cudaStream_t)stream>>>(flags, G, epoch, (unsigned long long)(timeout_s * 1e9));
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_ipc_alloc(int64_t bytes, void **ptr) {
  if (bytes <= 0 || !ptr) return FK_E_ARG;
  FK_TRY(cudaMalloc(ptr, (size_t)bytes));
  return 0;
}

int fk_ipc_free(void *ptr) {
  if (ptr) FK_TRY(cudaFree(ptr));
  return 0;
}

int fk_ipc_get_handle(void *ptr, void *handle_out) {
  if (!ptr || !handle_out) return FK_E_ARG;
  FK_TRY(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t *>(handle_out), ptr));
  return 0;
}

int fk_ipc_open(const void *handle, void **ptr) {
  if (!handle || !ptr) return FK_E_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  FK_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int fk_ipc_close(void *ptr) {
  if (ptr) FK_TRY(cudaIpcCloseMemHandle(ptr));
  return 0;
}

int fk_shard_unpermute(const uint32_t *perm, const void *src, int64_t n, int elem_bytes, void *dst, void *stream) {
  if (n < 0) return FK_E_ARG;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  switch (elem_bytes) {
    case 1:
      k_unpermute<uint8_t><<<grid_for(n), 256, 0, st>>>(perm, (const uint8_t *)src, n, (uint8_t *)dst);
      break;
    case 8:
      k_unpermute<uint64_t><<<grid_for(n), 256, 0, st>>>(perm, (const uint64_t *)src, n, (uint64_t *)dst);
      break;
    default:
      return FK_E_ARG;
  }
  FK_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
