// tcf_point.cu -- C-ABI entry points of the point two-choice filter.
// Kernels: tcf_point_impl.cuh (instantiated per slot width in tcf_point_s*.cu).
#include <stdlib.h>

#include "tcf_point_impl.cuh"

namespace fk {
extern template int tcf_run<uint8_t>(int, int, int, const TcfDev &, const TcfCall &, cudaStream_t);
extern template int tcf_run<uint16_t>(int, int, int, const TcfDev &, const TcfCall &, cudaStream_t);
extern template int tcf_run<uint32_t>(int, int, int, const TcfDev &, const TcfCall &, cudaStream_t);
extern template int tcf_run<uint64_t>(int, int, int, const TcfDev &, const TcfCall &, cudaStream_t);

static int geom_ok(const fk_tcf_geom *g) {
  if (!g || g->num_blocks < 1 || g->num_blocks > 0xFFFFFFF0LL) return 0;
  if (g->block_slots < 1 || g->backing_slots < 0) return 0;
  int w = g->slot_bytes;
  if (w != 1 && w != 2 && w != 4 && w != 8) return 0;
  if (g->tag_bits <= 2 || g->tag_bits > 8 * w) return 0;
  if (g->block_slots * 8 * w > 1024) return 0;
  int G = g->group_width;
  if (G != 1 && G != 2 && G != 4 && G != 8 && G != 16 && G != 32) return 0;
  if (G > g->block_slots) return 0;
  return 1;
}

static TcfDev make_dev(const fk_tcf_geom *g, const void *blocks, const void *backing, int keys_are_fps) {
  TcfDev P;
  P.blocks = const_cast<void *>(blocks);
  P.backing = const_cast<void *>(backing);
  P.nb = (uint64_t)g->num_blocks;
  P.nbm = make_fastmod(P.nb);
  P.bsize = (uint64_t)g->backing_slots;
  P.bsm = make_fastmod(P.bsize ? P.bsize : 1);
  P.B = g->block_slots;
  P.f = g->tag_bits;
  P.cut = g->cut_slots;
  P.probe_limit = g->probe_limit;
  P.fmask = g->tag_bits >= 64 ? ~0ULL : ((1ULL << g->tag_bits) - 1);
  P.seed = g->seed;
  P.keys_are_fps = keys_are_fps;
  return P;
}

static int run(const fk_tcf_geom *g, int op, const TcfDev &P, const TcfCall &c, cudaStream_t st) {
  switch (g->slot_bytes) {
    case 1: return tcf_run<uint8_t>(op, g->group_width, g->block_slots, P, c, st);
    case 4: return tcf_run<uint32_t>(op, g->group_width, g->block_slots, P, c, st);
    case 8: return tcf_run<uint64_t>(op, g->group_width, g->block_slots, P, c, st);
    default: return tcf_run<uint16_t>(op, g->group_width, g->block_slots, P, c, st);
  }
}

// Reservation granularity: 2^rs blocks per word, keeping the word array at
// <= 2^22 words (16 MiB, L2-resident next to the streamed keys); measured
// best at C3 (nb = 2^24 -> rs = 2).  Tunable: FK_ORD_RES_SHIFT.
static int ord_res_shift(int64_t nb) {
  int rs = 0;
  while ((nb >> rs) > (1LL << 22)) rs++;
  if (const char *e = getenv("FK_ORD_RES_SHIFT")) rs = atoi(e);
  return rs < 0 ? 0 : (rs > 16 ? 16 : rs);
}

// Keys introduced per round, as a fraction of the reservation words: 1/4 up
// to 2^18 words, 1/8 up to 2^20, else 1/16, capped at 2^18 (measured on the
// B200, profiles/r1c_ord_tune.jsonl: small tables are bound by the fixed
// per-round cost of ~9-12 us, so a wide window wins despite more lost bids;
// C3 (2^22 words) is best at 2^18).
// Tunable: FK_ORD_WINDOW.
static int64_t ord_window(int64_t nb, int64_t n) {
  int64_t ng = nb >> ord_res_shift(nb);
  int64_t w = ng <= (1 << 18) ? ng / 4 : (ng <= (1 << 20) ? ng / 8 : ng / 16);
  w = w < 4096 ? 4096 : (w > (1 << 18) ? (1 << 18) : w);
  if (const char *e = getenv("FK_ORD_WINDOW")) {
    long long v = atoll(e);
    if (v > 0) w = v;
  }
  return w < n ? w : (n < 1 ? 1 : n);
}

static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

static int ord_hints() {
  const char *e = getenv("FK_ORD_HINTS");
  return e ? atoi(e) != 0 : 1;
}

// the one-barrier ordered kernel (u16 slots, B = 16, G = 1) keeps a second
// reservation array (tunable: FK_ORD_ONEBAR=0 selects the carry-list kernel)
static int ord_onebar(const fk_tcf_geom *g) {
  return g->slot_bytes == 2 && g->block_slots == 16 && g->group_width == 1 && env_int("FK_ORD_ONEBAR", 1);
}

static size_t ord_ws_layout(const fk_tcf_geom *g, int64_t n, size_t *off) {
  // off[]: res, bres, defer_idx, defer_pend, ctl, carry0, carry1, res2
  size_t a = 0;
  auto take = [&](size_t bytes) { size_t o = a; a += (bytes + 255) & ~(size_t)255; return o; };
  int64_t cap = n < 1 ? 1 : n;
  int64_t w = ord_window(g->num_blocks, n);
  off[0] = take((size_t)((g->num_blocks >> ord_res_shift(g->num_blocks)) + 1) * 4);
  off[1] = take((size_t)(g->backing_slots ? g->backing_slots : 1) * 4);
  off[2] = take((size_t)cap * 4);
  off[3] = take((size_t)cap);
  off[4] = take(64);
  off[5] = take((size_t)w * 4);
  off[6] = take((size_t)w * 4);
  off[7] = ord_onebar(g) ? take((size_t)((g->num_blocks >> ord_res_shift(g->num_blocks)) + 1) * 4) : 0;
  return a;
}

static int prep_ordered(const fk_tcf_geom *g, int64_t n, void *ws, size_t ws_bytes, OrdScratch *X,
                        cudaStream_t st) {
  size_t off[8];
  size_t need = ord_ws_layout(g, n, off);
  if (!ws || ws_bytes < need) return FK_E_ARG;
  char *b = (char *)ws;
  X->res = (uint32_t *)(b + off[0]);
  X->bres = (uint32_t *)(b + off[1]);
  X->defer_idx = (uint32_t *)(b + off[2]);
  X->defer_pend = (uint8_t *)(b + off[3]);
  X->ctl = (unsigned int *)(b + off[4]);
  X->carry[0] = (uint32_t *)(b + off[5]);
  X->carry[1] = (uint32_t *)(b + off[6]);
  X->defer_cap = n < 1 ? 1 : n;
  X->window = ord_window(g->num_blocks, n);
  X->res_shift = ord_res_shift(g->num_blocks);
  X->hints = ord_hints();
  // fewer grid-barrier participants when a round holds few keys (measured)
  X->prefetch = env_int("FK_ORD_PREFETCH", 0);  // measured slower (8.1 vs 8.7 G/s at C3)
  X->ctas_per_sm = env_int("FK_ORD_CTAS_PER_SM", g->num_blocks <= (1 << 17) ? 1 : (g->num_blocks <= (1 << 20) ? 2 : 0));
  FK_TRY(cudaMemsetAsync(X->res, 0xFF, (size_t)((g->num_blocks >> X->res_shift) + 1) * 4, st));
  X->res2 = nullptr;
  if (ord_onebar(g)) {
    X->res2 = (uint32_t *)(b + off[7]);
    FK_TRY(cudaMemsetAsync(X->res2, 0xFF, (size_t)((g->num_blocks >> X->res_shift) + 1) * 4, st));
  }
  X->slots = 1;
  X->held_only = env_int("FK_ORD_HELD_ONLY", 1);
  FK_TRY(cudaMemsetAsync(X->bres, 0xFF, (size_t)(g->backing_slots ? g->backing_slots : 1) * 4, st));
  FK_TRY(cudaMemsetAsync(X->ctl, 0, 64, st));
  return 0;
}

// Census of a slot array for validate() / load_factor() (tcf.py:196-249):
// live slots (word > TOMBSTONE) and live slots whose tag bits are reserved
// (tag < 2).  Grid-stride, warp-reduced, one atomic per warp.
template <typename S>
__global__ void k_tcf_census(const S *__restrict__ slots, int64_t n, uint64_t fmask,
                             unsigned long long *__restrict__ out) {
  unsigned long long live = 0, bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t w = slots[i];
    if (w > 1) {
      live++;
      bad += (w & fmask) < 2;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    live += __shfl_xor_sync(0xFFFFFFFFu, live, o);
    bad += __shfl_xor_sync(0xFFFFFFFFu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (live) atomicAdd(&out[0], live);
    if (bad) atomicAdd(&out[1], bad);
  }
}

template <typename S>
static int census_t(const void *p, int64_t n, uint64_t fmask, unsigned long long *d, cudaStream_t st) {
  if (n <= 0) return 0;
  int64_t blocks = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 8;
  k_tcf_census<S><<<(int)(blocks < cap ? blocks : cap), 256, 0, st>>>((const S *)p, n, fmask, d);
  FK_CHECK_LAUNCH();
  return 0;
}

static int census(int wbytes, const void *p, int64_t n, uint64_t fmask, unsigned long long *d, cudaStream_t st) {
  switch (wbytes) {
    case 1: return census_t<uint8_t>(p, n, fmask, d, st);
    case 4: return census_t<uint32_t>(p, n, fmask, d, st);
    case 8: return census_t<uint64_t>(p, n, fmask, d, st);
    default: return census_t<uint16_t>(p, n, fmask, d, st);
  }
}

}  // namespace fk

using namespace fk;

extern "C" {

size_t fk_tcf_workspace_bytes(const fk_tcf_geom *g, int64_t n, int mode) {
  if (!g || mode != FK_ORDERED) return 0;
  size_t off[8];
  return ord_ws_layout(g, n, off);
}

int fk_tcf_insert(const fk_tcf_geom *g, void *blocks, void *backing, const uint64_t *keys, int keys_are_fps,
                  const uint64_t *values, int64_t n, uint8_t *codes, int64_t *counters, int mode, void *ws,
                  size_t ws_bytes, void *stream) {
  if (!geom_ok(g) || n < 0 || !counters) return FK_E_ARG;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  TcfDev P = make_dev(g, blocks, backing, keys_are_fps);
  TcfCall c = {keys, values, n, codes, nullptr, counters, OrdScratch{}};
  if (mode == FK_CONCURRENT) return run(g, kOpInsCas, P, c, st);
  if (n > 0xFFFFFFF0LL) return FK_E_ARG;
  int rc = prep_ordered(g, n, ws, ws_bytes, &c.X, st);
  return rc ? rc : run(g, kOpInsOrd, P, c, st);
}

int fk_tcf_query(const fk_tcf_geom *g, const void *blocks, const void *backing, const uint64_t *keys,
                 int keys_are_fps, int64_t n, uint8_t *found, uint64_t *values_out, void *stream) {
  if (!geom_ok(g) || n < 0) return FK_E_ARG;
  if (n == 0) return 0;
  TcfDev P = make_dev(g, blocks, backing, keys_are_fps);
  TcfCall c = {keys, nullptr, n, found, values_out, nullptr, OrdScratch{}};
  return run(g, kOpQuery, P, c, (cudaStream_t)stream);
}

int fk_tcf_delete(const fk_tcf_geom *g, void *blocks, void *backing, const uint64_t *keys, int keys_are_fps,
                  int64_t n, uint8_t *removed, int64_t *counters, int mode, void *ws, size_t ws_bytes,
                  void *stream) {
  if (!geom_ok(g) || n < 0 || !counters) return FK_E_ARG;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  TcfDev P = make_dev(g, blocks, backing, keys_are_fps);
  TcfCall c = {keys, nullptr, n, removed, nullptr, counters, OrdScratch{}};
  if (mode == FK_CONCURRENT) return run(g, kOpDelCas, P, c, st);
  if (n > 0xFFFFFFF0LL) return FK_E_ARG;
  int rc = prep_ordered(g, n, ws, ws_bytes, &c.X, st);
  return rc ? rc : run(g, kOpDelOrd, P, c, st);
}

int fk_tcf_census(const fk_tcf_geom *g, const void *blocks, const void *backing, int64_t *out4, void *stream) {
  if (!geom_ok(g) || !out4) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *d = nullptr;
  FK_TRY(cudaMallocAsync((void **)&d, 4 * sizeof(unsigned long long), st));
  FK_TRY(cudaMemsetAsync(d, 0, 4 * sizeof(unsigned long long), st));
  const uint64_t fm = g->tag_bits >= 64 ? ~0ULL : ((1ULL << g->tag_bits) - 1);
  int rc = census(g->slot_bytes, blocks, g->num_blocks * (int64_t)g->block_slots, fm, d, st);
  if (!rc) rc = census(g->slot_bytes, backing, g->backing_slots, fm, d + 2, st);
  unsigned long long h[4] = {0, 0, 0, 0};
  if (!rc) {
    cudaError_t e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = -(int)e;
  }
  cudaFreeAsync(d, st);
  for (int i = 0; i < 4; i++) out4[i] = (int64_t)h[i];
  return rc;
}

}  // extern "C"
