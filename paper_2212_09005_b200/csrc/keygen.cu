// keygen.cu -- device key streams bit-identical to the reference's numpy
// generators (fk/workloads.py:61-118):
//   * PCG64, numpy's default_rng bit generator: 128-bit LCG (multiplier
//     0x2360ED051FC65DA44385DF649FCCF645, odd increment), step then XSL-RR
//     output, with jump-ahead so every thread starts at its own position;
//   * Generator.integers(low, high) for high - low <= 2^32: Lemire's bounded
//     method on the buffered 32-bit halves of the 64-bit outputs (low half
//     first); a draw is rejected iff (v * range) mod 2^32 < (2^32 - range) %
//     range, a property of the draw alone, so the accepted draws are selected
//     in order by a stream compaction;
//   * Generator.random doubles ((raw >> 11) * 2^-53) and the bounded-Zipf
//     rejection-inversion sampler of fk/workloads.py:81-118, pass by pass
//     (each pass draws one double per remaining rank, in order), with every
//     add / multiply / divide rounded separately (no FMA contraction) as
//     numpy evaluates them.
// Generator.shuffle (the ur_count stream's order) is a sequential
// Fisher-Yates with masked rejection and is not reproduced here.
#include <cub/cub.cuh>

#include "../../include/filterkit_b200.h"
#include "fk_common.cuh"
#include "fk_scratch.cuh"

namespace fk {
namespace {

struct U128 {
  uint64_t lo, hi;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

__device__ __forceinline__ U128 pcg_mult() {
  U128 m;
  m.hi = 0x2360ED051FC65DA4ULL;
  m.lo = 0x4385DF649FCCF645ULL;
  return m;
}

__device__ __forceinline__ uint64_t pcg_out(U128 s) {  // XSL-RR
  const unsigned rot = (unsigned)(s.hi >> 58);
  const uint64_t x = s.hi ^ s.lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}

// the state after `delta` steps (affine map composition, O(log delta))
__device__ U128 pcg_advance(U128 state, U128 inc, uint64_t delta) {
  U128 acc_mult{1, 0}, acc_plus{0, 0}, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{1, 0}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, state), acc_plus);
}

constexpr int kChunk = 64;  // outputs per thread (one jump, then plain steps)

// out[i] = output number start + i + 1 of the generator (numpy's random_raw)
__global__ void k_pcg64_raw(U128 st, U128 inc, uint64_t start, int64_t n, uint64_t *__restrict__ out) {
  const int64_t chunks = (n + kChunk - 1) / kChunk;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < chunks; c += (int64_t)gridDim.x * blockDim.x) {
    U128 s = pcg_advance(st, inc, start + (uint64_t)c * kChunk);
    const U128 m = pcg_mult();
    const int64_t e = (c + 1) * kChunk < n ? (c + 1) * kChunk : n;
    for (int64_t i = c * kChunk; i < e; i++) {
      s = add128(mul128(s, m), inc);
      out[i] = pcg_out(s);
    }
  }
}

// 32-bit draw j of the buffered stream: the low half of output j / 2 first
struct LemireAccept {
  const uint64_t *raw;
  uint32_t range, threshold;
  __device__ bool operator()(int64_t j) const {
    const uint64_t r = raw[j >> 1];
    const uint32_t v = (j & 1) ? (uint32_t)(r >> 32) : (uint32_t)r;
    return (uint32_t)((uint64_t)v * range) >= threshold;
  }
};

// full: the range is all of 2^32 (numpy returns the draw itself)
__global__ void k_lemire_values(const uint64_t *__restrict__ raw, const int64_t *__restrict__ sel, int64_t n,
                                uint32_t range, int full, int64_t low, int64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = sel[i];
    const uint64_t r = raw[j >> 1];
    const uint32_t v = (j & 1) ? (uint32_t)(r >> 32) : (uint32_t)r;
    out[i] = low + (int64_t)(full ? (uint64_t)v : (((uint64_t)v * range) >> 32));
  }
}

__global__ void k_fill_i64(int64_t *__restrict__ out, int64_t n, int64_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

// fk/workloads.py:84-99, operation by operation as numpy evaluates it
__device__ __forceinline__ double h_integral(double x, double s) {
  const double lx = log(x);
  const double z = __dmul_rn(__dadd_rn(1.0, -s), lx);
  const bool tiny = fabs(z) < 1e-8;
  const double safe = z == 0.0 ? 1.0 : z;
  const double ratio = tiny ? __dadd_rn(1.0, __ddiv_rn(z, 2.0)) : __ddiv_rn(expm1(z), safe);
  return __dmul_rn(ratio, lx);
}

__device__ __forceinline__ double h_integral_inverse(double y, double s) {
  double z = __dmul_rn(y, __dadd_rn(1.0, -s));
  z = z < -1.0 ? -1.0 : z;
  const bool tiny = fabs(z) < 1e-8;
  const double safe = z == 0.0 ? 1.0 : z;
  const double ratio = tiny ? __dadd_rn(1.0, -__ddiv_rn(z, 2.0)) : __ddiv_rn(log1p(z), safe);
  return exp(__dmul_rn(ratio, y));
}

// One rejection-inversion pass over the m remaining ranks (todo[i], in
// order), drawing doubles at generator positions pos .. pos + m - 1.
__global__ void k_zipf_pass(U128 st, U128 inc, uint64_t pos, const int64_t *__restrict__ todo, int64_t m, double s,
                            int64_t universe, double h_lo, double h_hi, double squeeze, int64_t *__restrict__ ranks,
                            uint8_t *__restrict__ again) {
  const int64_t chunks = (m + kChunk - 1) / kChunk;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < chunks; c += (int64_t)gridDim.x * blockDim.x) {
    U128 st_c = pcg_advance(st, inc, pos + (uint64_t)c * kChunk);
    const U128 mlt = pcg_mult();
    const int64_t e = (c + 1) * kChunk < m ? (c + 1) * kChunk : m;
    for (int64_t i = c * kChunk; i < e; i++) {
      st_c = add128(mul128(st_c, mlt), inc);
      const double d = __dmul_rn((double)(pcg_out(st_c) >> 11), 1.0 / 9007199254740992.0);
      const double u = __dadd_rn(h_hi, __dmul_rn(d, __dadd_rn(h_lo, -h_hi)));
      const double x = h_integral_inverse(u, s);
      int64_t k = (int64_t)floor(__dadd_rn(x, 0.5));
      k = k < 1 ? 1 : (k > universe ? universe : k);
      const double kd = (double)k;
      const bool ok = __dadd_rn(kd, -x) <= squeeze ||
                      u >= __dadd_rn(h_integral(__dadd_rn(kd, 0.5), s), -pow(kd, -s));
      if (ok) ranks[todo ? todo[i] : i] = k;
      again[i] = ok ? 0 : 1;
    }
  }
}

__global__ void k_iota_i64(int64_t *__restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

// key = mix64(base + rank) (fk/workloads.py:74-77)
__global__ void k_mix_offsets(uint64_t base, const int64_t *__restrict__ r, int64_t n, uint64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mix64(base + (uint64_t)r[i]);
}

__global__ void k_shuffle_keys(uint64_t seed, int64_t n, uint64_t *__restrict__ key, uint32_t *__restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = mix64((uint64_t)i ^ seed);
    idx[i] = (uint32_t)i;
  }
}

__global__ void k_gather_keys(const uint64_t *__restrict__ in, const uint32_t *__restrict__ perm, int64_t n,
                              uint64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[perm[i]];
}

inline int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256, cap = (int64_t)num_sms() * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

U128 u128(uint64_t hi, uint64_t lo) { return U128{lo, hi}; }

}  // namespace
}  // namespace fk

using namespace fk;

extern "C" {

int fk_pcg64_raw(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, uint64_t start, int64_t n,
                 uint64_t *out, void *stream) {
  if (n < 0 || !out) return FK_E_ARG;
  if (n == 0) return 0;
  k_pcg64_raw<<<grid_for((n + kChunk - 1) / kChunk), 256, 0, (cudaStream_t)stream>>>(
      u128(state_hi, state_lo), u128(inc_hi, inc_lo), start, n, out);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_bounded_integers(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t low,
                        int64_t high, int64_t n, int64_t *out, int64_t *consumed, void *stream) {
  if (n < 0 || !out || !consumed || high <= low || high - low > (1LL << 32)) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  *consumed = 0;
  if (n == 0) return 0;
  const uint64_t rng = (uint64_t)(high - low - 1);
  if (rng == 0) {  // numpy draws nothing
    k_fill_i64<<<grid_for(n), 256, 0, st>>>(out, n, low);
    FK_CHECK_LAUNCH();
    return 0;
  }
  const uint32_t range = (uint32_t)(rng + 1);  // 0 when rng == 2^32 - 1: every draw is accepted as is
  const uint32_t threshold = range ? (uint32_t)((0x100000000ULL - range) % range) : 0u;
  for (int64_t slack = 64 + n / 1024;; slack *= 4) {
    Scratch S(st);
    const int64_t draws = n + slack, outs = (draws + 1) / 2;
    uint64_t *raw = S.get<uint64_t>(outs);
    int64_t *sel = S.get<int64_t>(draws), *cnt = S.get<int64_t>(1);
    if (S.err) return -(int)S.err;
    k_pcg64_raw<<<grid_for((outs + kChunk - 1) / kChunk), 256, 0, st>>>(u128(state_hi, state_lo),
                                                                        u128(inc_hi, inc_lo), 0, outs, raw);
    LemireAccept pred{raw, range ? range : 1u, range ? threshold : 0u};
    cub::CountingInputIterator<int64_t> it(0);
    size_t tb = 0;
    FK_TRY(cub::DeviceSelect::If(nullptr, tb, it, sel, cnt, draws, pred, st));
    void *tmp = S.get<char>(tb);
    if (!tmp) return -(int)S.err;
    FK_TRY(cub::DeviceSelect::If(tmp, tb, it, sel, cnt, draws, pred, st));
    int64_t h = 0;
    FK_TRY(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    FK_TRY(cudaStreamSynchronize(st));
    if (h < n) continue;  // more rejections than slack: draw further
    k_lemire_values<<<grid_for(n), 256, 0, st>>>(raw, sel, n, range, range ? 0 : 1, low, out);
    FK_CHECK_LAUNCH();
    int64_t last = 0;
    FK_TRY(cudaMemcpyAsync(&last, sel + n - 1, sizeof(last), cudaMemcpyDeviceToHost, st));
    FK_TRY(cudaStreamSynchronize(st));
    *consumed = last / 2 + 1;  // 64-bit outputs used (the unused high half is dropped, as numpy does)
    return 0;
  }
}

int fk_zipf_bounded(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, double s,
                    int64_t universe, int64_t n, double h_lo, double h_hi, double squeeze, int64_t *ranks,
                    int64_t *consumed, void *stream) {
  if (n < 0 || !ranks || !consumed || universe < 1 || !(s > 0)) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  *consumed = 0;
  if (n == 0) return 0;
  Scratch S(st);
  int64_t *todo = S.get<int64_t>(n), *todo2 = S.get<int64_t>(n), *cnt = S.get<int64_t>(1);
  uint8_t *again = S.get<uint8_t>(n);
  if (S.err) return -(int)S.err;
  uint64_t pos = 0;
  int64_t m = n;
  const int64_t *cur = nullptr;  // first pass: todo = 0..n-1
  for (;;) {
    k_zipf_pass<<<grid_for((m + kChunk - 1) / kChunk), 256, 0, st>>>(u128(state_hi, state_lo), u128(inc_hi, inc_lo),
                                                                     pos, cur, m, s, universe, h_lo, h_hi, squeeze,
                                                                     ranks, again);
    FK_CHECK_LAUNCH();
    pos += (uint64_t)m;
    if (!cur) {
      k_iota_i64<<<grid_for(m), 256, 0, st>>>(todo, m);
      cur = todo;
    }
    size_t tb = 0;
    FK_TRY(cub::DeviceSelect::Flagged(nullptr, tb, cur, again, todo2, cnt, m, st));
    void *tmp = S.get<char>(tb);
    if (!tmp) return -(int)S.err;
    FK_TRY(cub::DeviceSelect::Flagged(tmp, tb, cur, again, todo2, cnt, m, st));
    int64_t h = 0;
    FK_TRY(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    FK_TRY(cudaStreamSynchronize(st));
    if (h == 0) break;
    FK_TRY(cudaMemcpyAsync(todo, todo2, h * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    cur = todo;
    m = h;
  }
  *consumed = (int64_t)pos;
  return 0;
}

int fk_mix_offsets(uint64_t base, const int64_t *offsets, int64_t n, uint64_t *out, void *stream) {
  if (n < 0 || (n && (!offsets || !out))) return FK_E_ARG;
  if (n == 0) return 0;
  k_mix_offsets<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(base, offsets, n, out);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_shuffle_u64(const uint64_t *in, int64_t n, uint64_t seed, uint64_t *out, void *stream) {
  if (n < 0 || n > 0xFFFFFFF0LL || (n && (!in || !out))) return FK_E_ARG;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch S(st);
  uint64_t *k = S.get<uint64_t>(n), *ks = S.get<uint64_t>(n);
  uint32_t *idx = S.get<uint32_t>(n), *perm = S.get<uint32_t>(n);
  if (S.err) return -(int)S.err;
  k_shuffle_keys<<<grid_for(n), 256, 0, st>>>(seed, n, k, idx);
  size_t tb = 0;
  FK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, k, ks, idx, perm, n, 0, 64, st));
  void *tmp = S.get<char>(tb);
  if (!tmp) return -(int)S.err;
  FK_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, k, ks, idx, perm, n, 0, 64, st));
  k_gather_keys<<<grid_for(n), 256, 0, st>>>(in, perm, n, out);
  FK_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
