// gqf.cu -- host side of the GQF C ABI: count / find_run / index rebuild /
// insert+delete batches (canonical rebuild, exact sequential fallback).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "fk_scratch.cuh"
#include "gqf_impl.cuh"

namespace fk {

namespace {

inline int blocks_for(int64_t n, int per = 256) {
  int64_t b = (n + per - 1) / per;
  int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

GqfDev make_dev(const fk_gqf_geom *g, const fk_gqf_tables *t) {
  GqfDev T;
  T.slots = t->slots;
  T.occ = t->occupieds;
  T.run = t->runends;
  T.offs = t->offsets;
  T.stats = t->stats;
  T.spill = t->spill;
  T.phys = g->phys;
  T.q = g->q;
  T.r = g->r;
  T.nregions = g->num_regions;
  T.max_occ = g->max_occupied;
  return T;
}

bool geom_ok(const fk_gqf_geom *g) {
  if (!g || g->q < 6 || g->q > 40) return false;
  if (g->r != 8 && g->r != 16 && g->r != 32) return false;
  if (g->q + g->r > 64) return false;
  int64_t logical = 1LL << g->q;
  int64_t pad = logical < kRegionSlots ? logical : kRegionSlots;
  return g->phys == logical + pad && g->num_regions == (g->phys + kRegionSlots - 1) / kRegionSlots;
}

// ---- CUB helpers (type-independent, instantiated once) ---------------------
cudaError_t cub_sort_pairs(Scratch &S, const uint64_t *kin, uint64_t *kout, const uint32_t *vin, uint32_t *vout,
                           int64_t n, int end_bit) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, end_bit, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, n, 0, end_bit, S.st);
}

cudaError_t cub_sort_keys(Scratch &S, const uint64_t *kin, uint64_t *kout, int64_t n, int end_bit) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, tb, kin, kout, n, 0, end_bit, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRadixSort::SortKeys(tmp, tb, kin, kout, n, 0, end_bit, S.st);
}

cudaError_t cub_sort_keys_u32(Scratch &S, const uint32_t *kin, uint32_t *kout, int64_t n, int end_bit) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, tb, kin, kout, n, 0, end_bit, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRadixSort::SortKeys(tmp, tb, kin, kout, n, 0, end_bit, S.st);
}

cudaError_t cub_sort_keys_u32_bits(Scratch &S, const uint32_t *kin, uint32_t *kout, int64_t n, int begin_bit,
                                   int end_bit) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, tb, kin, kout, n, begin_bit, end_bit, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRadixSort::SortKeys(tmp, tb, kin, kout, n, begin_bit, end_bit, S.st);
}

cudaError_t cub_sort_pairs_u8_u32(Scratch &S, const uint8_t *kin, uint8_t *kout, const uint32_t *vin, uint32_t *vout,
                                  int64_t n, int end_bit) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, end_bit, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, n, 0, end_bit, S.st);
}

// fingerprint i of a split sort: (high byte << 32) | low word
struct WidenSplit {
  const uint8_t *hi;
  const uint32_t *lo;
  __host__ __device__ uint64_t operator()(int64_t i) const {
    return ((uint64_t)(hi ? hi[i] : 0) << 32) | (uint64_t)lo[i];
  }
};

cudaError_t cub_rle_counts_split(Scratch &S, const uint8_t *hi, const uint32_t *lo, uint64_t *uniq, uint64_t *counts,
                                 int64_t *num, int64_t n) {
  auto it = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), WidenSplit{hi, lo});
  size_t tb = 0;
  cudaError_t e = cub::DeviceRunLengthEncode::Encode(nullptr, tb, it, uniq, counts, num, n, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRunLengthEncode::Encode(tmp, tb, it, uniq, counts, num, n, S.st);
}

cudaError_t cub_rle_counts(Scratch &S, const uint64_t *keys, uint64_t *uniq, uint64_t *counts, int64_t *num,
                           int64_t n) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceRunLengthEncode::Encode(nullptr, tb, keys, uniq, counts, num, n, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceRunLengthEncode::Encode(tmp, tb, keys, uniq, counts, num, n, S.st);
}

cudaError_t cub_excl_sum_i64(Scratch &S, const int64_t *in, int64_t *out, int64_t n) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, n, S.st);
}

cudaError_t cub_merge(Scratch &S, const uint64_t *k1, const uint64_t *v1, int64_t n1, const uint64_t *k2,
                      const uint64_t *v2, int64_t n2, uint64_t *ko, uint64_t *vo) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceMerge::MergePairs(nullptr, tb, k1, v1, n1, k2, v2, n2, ko, vo, cuda::std::less<>(), S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceMerge::MergePairs(tmp, tb, k1, v1, n1, k2, v2, n2, ko, vo, cuda::std::less<>(), S.st);
}

cudaError_t cub_select_flagged(Scratch &S, const uint64_t *in, const uint8_t *flags, uint64_t *out, int64_t *num,
                               int64_t n) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceSelect::Flagged(nullptr, tb, in, flags, out, num, n, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceSelect::Flagged(tmp, tb, in, flags, out, num, n, S.st);
}

cudaError_t cub_maxplus_scan(Scratch &S, const MaxPlus *in, MaxPlus *out, int64_t n) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::InclusiveScan(nullptr, tb, in, out, MaxPlusOp(), n, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceScan::InclusiveScan(tmp, tb, in, out, MaxPlusOp(), n, S.st);
}

cudaError_t cub_max_scan_i64(Scratch &S, const int64_t *in, int64_t *out, int64_t n) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::InclusiveScan(nullptr, tb, in, out, MaxI64(), n, S.st);
  if (e) return e;
  void *tmp = S.get<char>(tb);
  if (!tmp) return S.err;
  return cub::DeviceScan::InclusiveScan(tmp, tb, in, out, MaxI64(), n, S.st);
}

#define FK_CU(expr)                              \
  do {                                           \
    cudaError_t e_ = (expr);                     \
    if (e_ != cudaSuccess) return -(int)e_;      \
  } while (0)

int rebuild_index(const fk_gqf_geom *g, const fk_gqf_tables *t, cudaStream_t st) {
  Scratch S(st);
  int64_t nw = g->phys >> 6;
  int64_t nqw = ((1LL << g->q) + 63) >> 6;
  int64_t *po = S.get<int64_t>(nw), *pr = S.get<int64_t>(nw), *ro = S.get<int64_t>(nw), *rr = S.get<int64_t>(nw);
  if (S.err) return -(int)S.err;
  k_word_popc<<<blocks_for(nw), 256, 0, st>>>(t->occupieds, nw, po);
  k_word_popc<<<blocks_for(nw), 256, 0, st>>>(t->runends, nw, pr);
  FK_CU(cub_excl_sum_i64(S, po, ro, nw));
  FK_CU(cub_excl_sum_i64(S, pr, rr, nw));
  k_spill_from_ranks<<<blocks_for(nqw), 256, 0, st>>>(t->runends, ro, rr, nqw, nw, t->spill);
  FK_CHECK_LAUNCH();
  return 0;
}

template <typename S_t>
int validate_t(const fk_gqf_geom *g, const fk_gqf_tables *t, int64_t *out, cudaStream_t st) {
  Scratch S(st);
  GqfDev T = make_dev(g, t);
  int64_t nw = g->phys >> 6;
  int64_t *po = S.get<int64_t>(nw), *pr = S.get<int64_t>(nw), *ro = S.get<int64_t>(nw), *rr = S.get<int64_t>(nw);
  int64_t *v = S.get<int64_t>(kValidateWords);
  if (S.err) return -(int)S.err;
  int64_t init[kValidateWords];
  for (int i = 0; i < kValidateWords; i++) init[i] = i < 8 ? 0 : INT64_MAX;
  FK_CU(cudaMemcpyAsync(v, init, sizeof(init), cudaMemcpyHostToDevice, st));
  k_word_popc<<<blocks_for(nw), 256, 0, st>>>(t->occupieds, nw, po);
  k_word_popc<<<blocks_for(nw), 256, 0, st>>>(t->runends, nw, pr);
  FK_CU(cub_excl_sum_i64(S, po, ro, nw));
  FK_CU(cub_excl_sum_i64(S, pr, rr, nw));
  int64_t tails[4];
  FK_CU(cudaMemcpyAsync(&tails[0], ro + nw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_CU(cudaMemcpyAsync(&tails[1], po + nw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_CU(cudaMemcpyAsync(&tails[2], rr + nw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_CU(cudaMemcpyAsync(&tails[3], pr + nw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_CU(cudaStreamSynchronize(st));
  if (tails[0] + tails[1] != tails[2] + tails[3]) {  // _derive_structure's first check
    for (int i = 0; i < kValidateWords; i++) out[i] = init[i];
    out[0] = 1LL << kVRankMismatch;
    out[8 + kVRankMismatch] = 0;
    return 0;
  }
  k_gqf_validate_runs<S_t><<<blocks_for(nw), 256, 0, st>>>(T, nw, ro, rr, v);
  k_gqf_validate_offsets<<<blocks_for(g->num_regions), 256, 0, st>>>(T, nw, ro, rr, v);
  k_count_nonzero<S_t><<<blocks_for(g->phys), 256, 0, st>>>(reinterpret_cast<const S_t *>(t->slots), g->phys, v);
  FK_CHECK_LAUNCH();
  FK_CU(cudaMemcpyAsync(out, v, sizeof(init), cudaMemcpyDeviceToHost, st));
  FK_CU(cudaStreamSynchronize(st));
  return 0;
}

// a batch touching at most this many distinct fingerprints takes the
// region-local path (tunable: FK_GQF_SMALL; 0 disables)
// Partition counting (k_part_*) of plain counted inserts: two kPartBits MSD
// passes then shared-memory aggregation of the low W = qr - 2 kPartBits bits.
// Used from 2^22 occurrences (smaller batches keep the CUB sort; tunable:
// FK_GQF_PART=0 disables, FK_GQF_PART_MIN sets the threshold).
// Pass 2 uses p2 <= kPartBits bits, so partitions average ~3 K occurrences.
inline bool part_plan(int64_t n, int qr, int *W, int *p2) {
  const char *e = getenv("FK_GQF_PART");
  if (e && atoi(e) == 0) return false;
  const char *m = getenv("FK_GQF_PART_MIN");
  const int64_t nmin = m ? atoll(m) : (1LL << 22);
  int b = 1;
  while (b < kPartBits && (n >> (kPartBits + b)) > 3072) b++;
  const int w = qr - kPartBits - b;
  if (n < nmin || w < 4 || qr - kPartBits > 32) return false;
  *W = w;
  *p2 = b;
  return true;
}

// m = the number of segments (the last item's segment id + 1; 0 when n = 0)
__global__ void k_seg_count(const int64_t *__restrict__ seg, int64_t n, int64_t *__restrict__ m) {
  *m = n > 0 ? seg[n - 1] + 1 : 0;
}

__global__ void k_part_total(const int64_t *__restrict__ uoff, const int64_t *__restrict__ ucount, int64_t NP,
                             const unsigned *__restrict__ overflow, int64_t *__restrict__ out) {
  out[0] = uoff[NP - 1] + ucount[NP - 1];
  out[1] = *overflow;
}

// Count a plain insert batch by partitions: uniq / sums / *d_num like the
// sort + run-length path.  Returns 0, 1 when a partition overflowed its
// shared-memory table (nothing usable; recount on the sort path), or < 0.
int part_count(Scratch &S, const uint64_t *keys, int keys_are_fps, uint64_t seed, uint64_t fmask, int qr, int W,
               int p2, int64_t n, uint64_t *uniq, uint64_t *sums, int64_t *d_num) {
  cudaStream_t st = S.st;
  const int64_t NP = 1LL << (kPartBits + p2);
  unsigned long long *hist1 = S.get<unsigned long long>(kPartBins), *bounds1 = S.get<unsigned long long>(kPartBins + 1),
                     *cursor1 = S.get<unsigned long long>(kPartBins),
                     *tstart = S.get<unsigned long long>(kPartBins + 1);
  unsigned long long *hist2 = S.get<unsigned long long>(NP + 1), *bounds2 = S.get<unsigned long long>(NP + 1);
  int64_t *ucount = S.get<int64_t>(NP), *uoff = S.get<int64_t>(NP);
  uint32_t *buf1 = S.get<uint32_t>(n), *buf2 = S.get<uint32_t>(n);
  uint64_t *out_fp = S.get<uint64_t>(n);
  unsigned *ovf = S.get<unsigned>(1);
  if (S.err) return -(int)S.err;
  FK_TRY(cudaMemsetAsync(hist1, 0, kPartBins * sizeof(unsigned long long), st));
  FK_TRY(cudaMemsetAsync(hist2, 0, (NP + 1) * sizeof(unsigned long long), st));
  FK_TRY(cudaMemsetAsync(ovf, 0, sizeof(unsigned), st));
  static bool attr = false;
  if (!attr) {
    FK_TRY(cudaFuncSetAttribute(k_part1_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPartSmem));
    FK_TRY(cudaFuncSetAttribute(k_part2_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPartSmem));
    attr = true;
  }
  const int sms = num_sms();
  k_part1_hist<<<sms * 4, kPartThreads, 0, st>>>(keys, keys_are_fps, seed, fmask, qr, n, hist1);
  k_part_plan1<<<1, kPartBins, 0, st>>>(hist1, bounds1, cursor1, tstart);
  k_part1_scatter<<<sms * 4, kPartThreads, kPartSmem, st>>>(keys, keys_are_fps, seed, fmask, qr, n, cursor1, buf1);
  k_part2_hist<<<sms * 4, kPartThreads, 0, st>>>(buf1, bounds1, tstart, W, p2, hist2);
  {
    size_t tb = 0;
    FK_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, hist2, bounds2, NP + 1, st));
    void *tmp = S.get<char>(tb);
    if (!tmp) return -(int)S.err;
    FK_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, hist2, bounds2, NP + 1, st));
  }
  FK_TRY(cudaMemcpyAsync(hist2, bounds2, NP * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));  // cursors
  k_part2_scatter<<<sms * 4, kPartThreads, kPartSmem, st>>>(buf1, bounds1, tstart, W, p2, hist2, buf2);
  uint32_t *out_cnt = buf1;  // pass-1 output is dead now
  int lg = 12;  // log2(kAggSlots); FK_GQF_PART_SLOTS (a power of two below it) exercises the overflow path
  if (const char *e = getenv("FK_GQF_PART_SLOTS"))
    while (lg > 1 && (1 << lg) > atoi(e)) lg--;
  k_part_aggregate<<<sms * 6, kAggThreads, 0, st>>>(buf2, bounds2, NP, W, out_fp, out_cnt, ucount, ovf, lg);
  FK_TRY(cub_excl_sum_i64(S, ucount, uoff, NP));
  k_part_total<<<1, 1, 0, st>>>(uoff, ucount, NP, ovf, d_num + 2);
  int64_t h2[2];
  FK_TRY(cudaMemcpyAsync(h2, d_num + 2, sizeof(h2), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  if (h2[1]) return 1;
  k_part_compact<<<blocks_for(NP * 32), 256, 0, st>>>(out_fp, out_cnt, bounds2, ucount, uoff, NP, uniq, sums);
  FK_TRY(cudaMemcpyAsync(d_num, d_num + 2, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  FK_CHECK_LAUNCH();
  return 0;
}

// region-parallel placement of the canonical rebuild (k_region_*); FK_GQF_REGION_PLACE=0
// keeps the global max-plus scan and item-parallel writes
inline bool region_place_enabled() {
  const char *e = getenv("FK_GQF_REGION_PLACE");
  return !e || atoi(e) != 0;
}

// region-local in-place apply of mid-size batches (apply_local_t); FK_GQF_LOCAL=0 disables
inline bool local_apply_enabled() {
  const char *e = getenv("FK_GQF_LOCAL");
  return !e || atoi(e) != 0;
}

inline int64_t small_batch_limit(const fk_gqf_geom *g) {
  const char *e = getenv("FK_GQF_SMALL");
  if (e) return atoll(e);
  int64_t lim = g->quotient_regions * 2;
  return lim < (1 << 16) ? lim : (1 << 16);
}

// Region-local insert of a sorted batch into a copy of `cur` written to
// `nxt`.  Returns 0 when applied (tables swapped), 1 when a region reported
// a capacity failure (nothing applied; the caller runs the full path), or a
// negative error.
template <typename S_t>
int apply_small_t(const fk_gqf_geom *g, const fk_gqf_tables *cur, const fk_gqf_tables *nxt, const uint64_t *fps_s,
                  const uint64_t *del_s, int64_t n, fk_gqf_result *res, cudaStream_t st) {
  Scratch S(st);
  const int64_t nqr = g->quotient_regions;
  int64_t *rb = S.get<int64_t>(nqr + 1);
  if (S.err) return -(int)S.err;
  k_region_bounds<<<blocks_for(nqr + 1), 256, 0, st>>>(fps_s, n, g->r + kRegionBits, nqr, rb);
  std::vector<int64_t> hrb(nqr + 1);
  FK_CU(cudaMemcpyAsync(hrb.data(), rb, (nqr + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  // the copy the regions are applied to
  FK_CU(cudaMemcpyAsync(nxt->slots, cur->slots, (size_t)g->phys * sizeof(S_t), cudaMemcpyDeviceToDevice, st));
  FK_CU(cudaMemcpyAsync(nxt->occupieds, cur->occupieds, (size_t)(g->phys >> 6) * 8, cudaMemcpyDeviceToDevice, st));
  FK_CU(cudaMemcpyAsync(nxt->runends, cur->runends, (size_t)(g->phys >> 6) * 8, cudaMemcpyDeviceToDevice, st));
  FK_CU(cudaMemcpyAsync(nxt->offsets, cur->offsets, (size_t)g->num_regions * 4, cudaMemcpyDeviceToDevice, st));
  FK_CU(cudaMemcpyAsync(nxt->stats, cur->stats, 3 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  FK_CU(cudaStreamSynchronize(st));
  std::vector<int32_t> lists[2];
  for (int64_t r = 0; r < nqr; r++)
    if (hrb[r + 1] > hrb[r]) lists[r & 1].push_back((int32_t)r);
  const size_t most = lists[0].size() > lists[1].size() ? lists[0].size() : lists[1].size();
  int32_t *dlist = S.get<int32_t>(most), *fail = S.get<int32_t>(most);
  int32_t *scr = S.get<int32_t>(most * SeqGqf<S_t>::kGapCap);
  unsigned long long *moved = S.get<unsigned long long>(1);
  if (S.err) return -(int)S.err;
  FK_CU(cudaMemsetAsync(moved, 0, sizeof(unsigned long long), st));
  GqfDev T1 = make_dev(g, nxt);
  for (int parity = 0; parity < 2; parity++) {
    const std::vector<int32_t> &L = lists[parity];
    if (L.empty()) continue;
    FK_CU(cudaMemcpyAsync(dlist, L.data(), L.size() * 4, cudaMemcpyHostToDevice, st));
    FK_CU(cudaMemsetAsync(fail, 0, L.size() * 4, st));
    k_gqf_insert_regions<S_t><<<blocks_for((int64_t)L.size(), 64), 64, 0, st>>>(T1, fps_s, del_s, rb, dlist,
                                                                            (int64_t)L.size(), scr, fail, moved);
    FK_CHECK_LAUNCH();
    std::vector<int32_t> hf(L.size());
    FK_CU(cudaMemcpyAsync(hf.data(), fail, L.size() * 4, cudaMemcpyDeviceToHost, st));
    FK_CU(cudaStreamSynchronize(st));
    for (int32_t f : hf)
      if (f) return f < 0 ? FK_E_INVARIANT : 1;
  }
  // The regions ran in sorted order and in parallel, each reading the shared
  // occupancy racily, so their load checks prove nothing.  The reference
  // checks occupancy before each insert (pk:592-593), so if the final
  // occupancy is below max_occupied, no order could have failed.  Otherwise
  // discard the copy and let the full path decide in input order.
  int64_t h_occ = 0;
  FK_CU(cudaMemcpyAsync(&h_occ, nxt->stats, sizeof(h_occ), cudaMemcpyDeviceToHost, st));
  FK_CU(cudaStreamSynchronize(st));
  if (h_occ >= g->max_occupied) return 1;
  unsigned long long hm = 0;
  FK_CU(cudaMemcpyAsync(&hm, moved, sizeof(hm), cudaMemcpyDeviceToHost, st));
  int rc = rebuild_index(g, nxt, st);
  if (rc) return rc;
  FK_CU(cudaStreamSynchronize(st));
  res->swapped = 1;
  res->shifted = (int64_t)hm;
  return 0;
}

// Region-local delete of a sorted batch, in place on `cur` (deletes raise
// no capacity errors); found flags at the items' input positions.
template <typename S_t>
int apply_small_delete_t(const fk_gqf_geom *g, const fk_gqf_tables *cur, const uint64_t *fps_s,
                         const uint64_t *del_s, const uint32_t *idx_s, int64_t n, int order, uint8_t *found,
                         fk_gqf_result *res, cudaStream_t st) {
  Scratch S(st);
  const int64_t nqr = g->quotient_regions;
  int64_t *rb = S.get<int64_t>(nqr + 1);
  if (S.err) return -(int)S.err;
  k_region_bounds<<<blocks_for(nqr + 1), 256, 0, st>>>(fps_s, n, g->r + kRegionBits, nqr, rb);
  std::vector<int64_t> hrb(nqr + 1);
  FK_CU(cudaMemcpyAsync(hrb.data(), rb, (nqr + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_CU(cudaStreamSynchronize(st));
  std::vector<int32_t> lists[2];
  for (int64_t r = 0; r < nqr; r++)
    if (hrb[r + 1] > hrb[r]) lists[r & 1].push_back((int32_t)r);
  const size_t most = lists[0].size() > lists[1].size() ? lists[0].size() : lists[1].size();
  int32_t *dlist = S.get<int32_t>(most), *fail = S.get<int32_t>(most);
  unsigned long long *moved = S.get<unsigned long long>(1);
  if (S.err) return -(int)S.err;
  FK_CU(cudaMemsetAsync(moved, 0, sizeof(unsigned long long), st));
  GqfDev T0 = make_dev(g, cur);
  for (int parity = 0; parity < 2; parity++) {
    const std::vector<int32_t> &L = lists[parity];
    if (L.empty()) continue;
    FK_CU(cudaMemcpyAsync(dlist, L.data(), L.size() * 4, cudaMemcpyHostToDevice, st));
    FK_CU(cudaMemsetAsync(fail, 0, L.size() * 4, st));
    k_gqf_delete_regions<S_t><<<blocks_for((int64_t)L.size(), 64), 64, 0, st>>>(
        T0, fps_s, del_s, idx_s, rb, dlist, (int64_t)L.size(), order == FK_ORDER_BULK ? 1 : 0, found, fail, moved);
    FK_CHECK_LAUNCH();
    std::vector<int32_t> hf(L.size());
    FK_CU(cudaMemcpyAsync(hf.data(), fail, L.size() * 4, cudaMemcpyDeviceToHost, st));
    FK_CU(cudaStreamSynchronize(st));
    for (int32_t f : hf)
      if (f) return FK_E_INVARIANT;
  }
  unsigned long long hm = 0;
  FK_CU(cudaMemcpyAsync(&hm, moved, sizeof(hm), cudaMemcpyDeviceToHost, st));
  int rc = rebuild_index(g, cur, st);
  if (rc) return rc;
  FK_CU(cudaStreamSynchronize(st));
  res->shifted = (int64_t)hm;
  return 0;
}

// Decode of the whole table by runs (k_decode_runs): the k-th occupied
// quotient and the k-th runend from a global rank/select of the two bit
// vectors, then one thread per run -- pass 0 counts each run's groups,
// pass 1 writes them at the scanned offsets.  Scratch stays in S.
// threads for a warp_join over n probes (one warp per kJoinChunk)
inline int64_t join_threads(int64_t n) { return (n + kJoinChunk - 1) / kJoinChunk * 32; }

struct RunDecode {
  int64_t K = 0, items = 0;
  int64_t *Q = nullptr, *E = nullptr, *gcount = nullptr, *goff = nullptr;
  int *err = nullptr;
};

template <typename S_t>
int decode_runs_count(Scratch &S, const fk_gqf_geom *g, const fk_gqf_tables *t, const GqfDev &T, RunDecode *D,
                      cudaStream_t st) {
  const int64_t nbw = g->phys >> 6;
  int64_t *pops = S.get<int64_t>(2 * nbw), *poff = S.get<int64_t>(2 * nbw);
  D->err = S.get<int>(4);
  if (S.err) return -(int)S.err;
  int64_t hk[4] = {0, 0, 0, 0};
  FK_CU(cudaMemsetAsync(D->err, 0, 4 * sizeof(int), st));
  k_word_popc<<<blocks_for(nbw), 256, 0, st>>>(t->occupieds, nbw, pops);
  k_word_popc<<<blocks_for(nbw), 256, 0, st>>>(t->runends, nbw, pops + nbw);
  FK_CU(cub_excl_sum_i64(S, pops, poff, nbw));
  FK_CU(cub_excl_sum_i64(S, pops + nbw, poff + nbw, nbw));
  FK_CU(cudaMemcpyAsync(&hk[0], poff + nbw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_CU(cudaMemcpyAsync(&hk[1], pops + nbw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_CU(cudaMemcpyAsync(&hk[2], poff + 2 * nbw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_CU(cudaMemcpyAsync(&hk[3], pops + 2 * nbw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_CU(cudaStreamSynchronize(st));
  D->K = hk[0] + hk[1];
  if (D->K != hk[2] + hk[3]) return FK_E_INVARIANT;  // occupieds / runends set-bit counts differ
  D->Q = S.get<int64_t>(D->K);
  D->E = S.get<int64_t>(D->K);
  D->gcount = S.get<int64_t>(D->K);
  D->goff = S.get<int64_t>(D->K);
  if (S.err) return -(int)S.err;
  D->items = 0;
  if (D->K == 0) return 0;
  k_bit_positions<<<blocks_for(nbw), 256, 0, st>>>(t->occupieds, nbw, poff, D->Q);
  k_bit_positions<<<blocks_for(nbw), 256, 0, st>>>(t->runends, nbw, poff + nbw, D->E);
  k_decode_runs<S_t><<<blocks_for(D->K), 256, 0, st>>>(T, D->Q, D->E, D->K, 0, D->gcount, nullptr, nullptr, nullptr,
                                                      D->err);
  FK_CU(cub_excl_sum_i64(S, D->gcount, D->goff, D->K));
  int64_t tail[2] = {0, 0};
  int h_err = 0;
  FK_CU(cudaMemcpyAsync(&tail[0], D->goff + D->K - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_CU(cudaMemcpyAsync(&tail[1], D->gcount + D->K - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_CU(cudaMemcpyAsync(&h_err, D->err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FK_CU(cudaStreamSynchronize(st));
  if (h_err) return FK_E_INVARIANT;
  D->items = tail[0] + tail[1];
  return 0;
}

template <typename S_t>
int decode_runs_write(const GqfDev &T, const RunDecode &D, uint64_t *fp_out, uint64_t *cnt_out, cudaStream_t st) {
  if (D.K == 0) return 0;
  k_decode_runs<S_t><<<blocks_for(D.K), 256, 0, st>>>(T, D.Q, D.E, D.K, 1, nullptr, D.goff, fp_out, cnt_out, D.err);
  FK_CHECK_LAUNCH();
  return 0;
}

// (fingerprint, count) items of the whole table in fingerprint order, by
// the run decode the rebuild uses.  *count_out = the number of items;
// nothing is written when it exceeds cap.
template <typename S_t>
int enumerate_t(const fk_gqf_geom *g, const fk_gqf_tables *t, uint64_t *fp_out, uint64_t *cnt_out, int64_t cap,
                int64_t *count_out, cudaStream_t st) {
  Scratch S(st);
  GqfDev T = make_dev(g, t);
  RunDecode D;
  int rc = decode_runs_count<S_t>(S, g, t, T, &D, st);
  if (rc) return rc;
  *count_out = D.items;
  if (*count_out > cap) return 0;
  rc = decode_runs_write<S_t>(T, D, fp_out, cnt_out, st);
  if (rc) return rc;
  FK_CU(cudaStreamSynchronize(st));
  return 0;
}

template <typename S_t>
int count_t(const fk_gqf_geom *g, const fk_gqf_tables *t, const uint64_t *keys, int keys_are_fps, int64_t n,
            uint64_t *counts, cudaStream_t st) {
  GqfDev T = make_dev(g, t);
  k_gqf_count<S_t><<<blocks_for(n), 256, 0, st>>>(T, keys, keys_are_fps, g->seed, n, counts);
  FK_CHECK_LAUNCH();
  return 0;
}

// Region-local apply in place (batches touching at most a quarter of the
// regions): only the regions holding new items and their successors are
// decoded, merged, placed and rewritten; every other region -- its slots,
// bits and offset -- stays as it is.  The placement scan restarts at each run
// of listed regions from the old incoming end (old offsets), a plan pass
// validates every listed region and checks that each run hands the next,
// unlisted region its old incoming end (else the layout change would reach
// it: the global path runs instead), and only then does the write pass
// touch the table.  Returns 0 (applied, or dry run answered), 1 (not
// applicable: the caller continues with the global path), 2 (the exact
// path is needed; *load_possible set), or < 0.
constexpr int kApplyDryFlag = 1;
// Regions the batch's fingerprints touch (creg[0..K)); K = -1 for tables too
// small to split.
int local_regions(Scratch &S, const fk_gqf_geom *g, const uint64_t *uniq, int64_t m, int64_t **creg_out,
                  int64_t *K_out) {
  cudaStream_t st = S.st;
  const int64_t nqr = g->quotient_regions;
  *K_out = -1;
  if (m <= 0 || nqr < 8) return 0;
  int64_t *rbu = S.get<int64_t>(nqr + 1), *creg = S.get<int64_t>(nqr), *d_k = S.get<int64_t>(1);
  uint8_t *cand = S.get<uint8_t>(nqr);
  if (S.err) return -(int)S.err;
  k_region_bounds<<<blocks_for(nqr + 1), 256, 0, st>>>(uniq, m, g->r + kRegionBits, nqr, rbu);
  k_region_candidates<<<blocks_for(nqr), 256, 0, st>>>(rbu, nqr, cand);
  {
    cub::CountingInputIterator<int64_t> it(0);
    size_t tb = 0;
    FK_TRY(cub::DeviceSelect::Flagged(nullptr, tb, it, cand, creg, d_k, nqr, st));
    void *tmp = S.get<char>(tb);
    if (!tmp) return -(int)S.err;
    FK_TRY(cub::DeviceSelect::Flagged(tmp, tb, it, cand, creg, d_k, nqr, st));
  }
  int64_t K = 0;
  FK_TRY(cudaMemcpyAsync(&K, d_k, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  if (getenv("FK_GQF_TRACE"))
    fprintf(stderr, "fk gqf local: m=%lld listed regions %lld of %lld\n", (long long)m, (long long)K,
            (long long)nqr);
  *creg_out = creg;
  *K_out = K;
  return 0;
}

// Regions listed by local_regions: K > 0 and at most a quarter of them.
inline bool local_applicable(const fk_gqf_geom *g, int64_t K) { return K > 0 && 4 * K <= g->quotient_regions; }

template <typename S_t>
int apply_local_t(Scratch &S, const fk_gqf_geom *g, const fk_gqf_tables *cur, const int64_t *creg, int64_t K,
                  const uint64_t *keys, int keys_are_fps, uint64_t fmask, int64_t n, const uint64_t *uniq,
                  const uint64_t *c_new, int64_t m, bool is_del, int order, int flags, fk_gqf_result *res,
                  bool *load_possible) {
  cudaStream_t st = S.st;
  const int64_t nqr = g->quotient_regions;
  if (!local_applicable(g, K)) return 1;
  const bool trace = getenv("FK_GQF_TRACE") != nullptr;
  GqfDev T0 = make_dev(g, cur);
  // old items of the listed regions
  const int64_t nqw = ((1LL << g->q) + 63) >> 6, nw = K * (kRegionSlots / 64);
  int64_t *gcount = S.get<int64_t>(nw), *goff = S.get<int64_t>(nw);
  int *d_err = S.get<int>(1);
  int64_t *d_num = S.get<int64_t>(4);
  if (S.err) return -(int)S.err;
  FK_TRY(cudaMemsetAsync(d_err, 0, sizeof(int), st));
  k_decode_region_words<S_t><<<blocks_for(nw), 256, 0, st>>>(T0, creg, K, nqw, 0, gcount, nullptr, nullptr, nullptr,
                                                              d_err);
  FK_TRY(cub_excl_sum_i64(S, gcount, goff, nw));
  int64_t tail[2];
  int h_err = 0;
  FK_TRY(cudaMemcpyAsync(&tail[0], goff + nw - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaMemcpyAsync(&tail[1], gcount + nw - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  if (h_err) return FK_E_INVARIANT;
  const int64_t g_old = tail[0] + tail[1];
  uint64_t *o_fp = S.get<uint64_t>(g_old), *o_cnt = S.get<uint64_t>(g_old);
  if (S.err) return -(int)S.err;
  k_decode_region_words<S_t><<<blocks_for(nw), 256, 0, st>>>(T0, creg, K, nqw, 1, nullptr, goff, o_fp, o_cnt, d_err);
  // merge with the batch's fingerprints (all inside listed regions)
  uint8_t *keep_o = S.get<uint8_t>(g_old), *keep_u = S.get<uint8_t>(m);
  uint64_t *o2_fp = S.get<uint64_t>(g_old), *o2_cnt = S.get<uint64_t>(g_old);
  uint64_t *u2_fp = S.get<uint64_t>(m), *u2_cnt = S.get<uint64_t>(m);
  if (S.err) return -(int)S.err;
  k_keep_old_join<<<blocks_for(join_threads(g_old)), 256, 0, st>>>(o_fp, g_old, uniq, m, keep_o);
  k_nonzero<<<blocks_for(m), 256, 0, st>>>(c_new, m, keep_u);
  FK_TRY(cub_select_flagged(S, o_fp, keep_o, o2_fp, d_num, g_old));
  FK_TRY(cub_select_flagged(S, o_cnt, keep_o, o2_cnt, d_num + 1, g_old));
  FK_TRY(cub_select_flagged(S, uniq, keep_u, u2_fp, d_num + 2, m));
  FK_TRY(cub_select_flagged(S, c_new, keep_u, u2_cnt, d_num + 3, m));
  int64_t hn[4];
  FK_TRY(cudaMemcpyAsync(hn, d_num, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  const int64_t G = hn[0] + hn[2];
  uint64_t *it_fp = S.get<uint64_t>(G), *it_cnt = S.get<uint64_t>(G);
  if (S.err) return -(int)S.err;
  if (G > 0) FK_TRY(cub_merge(S, o2_fp, o2_cnt, hn[0], u2_fp, u2_cnt, hn[2], it_fp, it_cnt));
  // summaries of the listed regions, restarted from the old incoming end at each run of them
  int64_t *ib = S.get<int64_t>(nqr + 1);
  MaxPlus *summ = S.get<MaxPlus>(K), *cum = S.get<MaxPlus>(K);
  unsigned long long *acc = S.get<unsigned long long>(4), *acc_old = S.get<unsigned long long>(2);
  unsigned *rflags = S.get<unsigned>(2);
  constexpr int64_t SW = kRegMaxRange / 64 + 1;
  S_t *saved = S.get<S_t>((size_t)K * kRegMaxRange);
  unsigned long long *saved_run = S.get<unsigned long long>((size_t)K * SW);
  if (S.err) return -(int)S.err;
  FK_TRY(cudaMemsetAsync(acc, 0, 4 * sizeof(unsigned long long), st));
  FK_TRY(cudaMemsetAsync(acc_old, 0, 2 * sizeof(unsigned long long), st));
  FK_TRY(cudaMemsetAsync(rflags, 0, 2 * sizeof(unsigned), st));
  if (G > 0) k_region_bounds<<<blocks_for(nqr + 1), 256, 0, st>>>(it_fp, G, g->r + kRegionBits, nqr, ib);
  else FK_TRY(cudaMemsetAsync(ib, 0, (nqr + 1) * sizeof(int64_t), st));
  const int rgrid = (int)(K < (int64_t)num_sms() * 8 ? K : (int64_t)num_sms() * 8);
  k_region_summary<<<rgrid, kRegThreads, 0, st>>>(it_fp, it_cnt, ib, creg, K, cur->offsets, g->r, summ, acc);
  FK_TRY(cub_maxplus_scan(S, summ, cum, K));
  k_item_sums<<<blocks_for(g_old), 256, 0, st>>>(o_fp, o_cnt, g_old, g->r, acc_old);
  if (order == FK_ORDER_POINT)
    k_not_ascending<<<blocks_for(n), 256, 0, st>>>(keys, keys_are_fps, g->seed, fmask, n, rflags + 1);
  // plan pass: validate, save the old windows (nothing written)
  RegionJob<S_t> job{creg, K, nqr, cur->offsets, 1, saved, saved_run};
  const S_t *cs = reinterpret_cast<const S_t *>(cur->slots);
  k_region_place<S_t><<<rgrid, kRegThreads, 0, st>>>(T0, cs, cur->runends, it_fp, it_cnt, ib, cum, job, rflags + 1,
                                                     order == FK_ORDER_BULK ? 1 : 0, rflags, acc + 2);
  unsigned long long ha[2], ho[2];
  unsigned hfl = 0;
  int64_t hst0 = 0;
  FK_TRY(cudaMemcpyAsync(ha, acc, sizeof(ha), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaMemcpyAsync(ho, acc_old, sizeof(ho), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaMemcpyAsync(&hfl, rflags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaMemcpyAsync(&hst0, cur->stats, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  FK_CHECK_LAUNCH();
  const int64_t h_occ = hst0 + (int64_t)ha[0] - (int64_t)ho[0];
  if (trace) fprintf(stderr, "fk gqf local: plan flags %u, occupancy %lld / %lld\n", hfl, (long long)h_occ,
                     (long long)g->max_occupied);
  bool exact = false;
  if (!is_del) {
    exact = hfl != 0 || h_occ >= g->max_occupied;
    *load_possible = h_occ >= g->max_occupied;
  }
  if (flags & kApplyDryFlag) {
    if (!exact && hfl) return 1;  // (a delete whose change reaches an unlisted region: let the global path answer)
    res->code = exact ? 1 : 0;
    return 0;
  }
  if (exact) return 2;
  if (hfl) return 1;
  // write pass, in place
  job.plan_only = 0;
  FK_TRY(cudaMemsetAsync(acc + 2, 0, sizeof(unsigned long long), st));
  k_region_place<S_t><<<rgrid, kRegThreads, 0, st>>>(T0, cs, cur->runends, it_fp, it_cnt, ib, cum, job, rflags + 1,
                                                     order == FK_ORDER_BULK ? 1 : 0, rflags, acc + 2);
  k_region_stats_delta<<<1, 1, 0, st>>>(acc, acc_old, G, g_old, cur->stats);
  int rc = rebuild_index(g, cur, st);
  if (rc) return rc;
  unsigned long long hd = 0;
  FK_TRY(cudaMemcpyAsync(&hd, acc + 2, sizeof(hd), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  FK_CHECK_LAUNCH();
  res->shifted = (int64_t)hd;
  res->swapped = 0;
  return 0;
}

// apply_t flags: dry run (steps 1-12 only; res->code = 1 if the batch would
// need the exact sequential path), or go straight to the exact path.
constexpr int kApplyDry = 1, kApplyForceExact = 2;
// Point-order batches longer than this that may hit a capacity error first
// apply their longest provably safe prefix canonically (found by binary
// search over dry runs) and run only the rest through the one-thread
// sequential kernel.
constexpr int64_t kExactSeqDirect = 2048;

template <typename S_t>
int apply_t(const fk_gqf_geom *g, const fk_gqf_tables *cur, const fk_gqf_tables *nxt, const uint64_t *keys,
            int keys_are_fps, const uint64_t *deltas, int64_t n, int op, int order, uint8_t *found,
            fk_gqf_result *res, cudaStream_t st, int flags = 0) {
  Scratch S(st);
  const int qr = g->q + g->r;
  const uint64_t fmask = qr >= 64 ? ~0ull : ((1ull << qr) - 1);
  const bool is_del = op == FK_GQF_DELETE;
  GqfDev T0 = make_dev(g, cur);
  res->code = 0;
  res->swapped = 0;
  res->fail_index = -1;
  res->fail_region = -1;
  res->shifted = 0;

  // 1-3. hash, stable sort by fingerprint, deltas in sorted order
  // Plain counted inserts (no deltas: every occurrence adds one) need
  // neither the input permutation nor delta sums.  Their fingerprints
  // (q + r <= 40 bits) are sorted as u32 low words, after one pass that
  // buckets them by the <= 8 high bits: 42 instead of 80 bytes moved per
  // occurrence for q + r = 36; run-length counts then read (high, low) pairs.
  const bool plain_ins = !is_del && deltas == nullptr;
  const bool split = plain_ins && qr <= 40;
  uint64_t *fps = nullptr, *fps_s = nullptr, *del_s = nullptr;
  int64_t *seg_heads = nullptr, *seg_ids = nullptr;
  uint32_t *idx = nullptr, *idx_s = nullptr;
  uint8_t *hi_s = nullptr;
  uint32_t *lo_s = nullptr;
  uint64_t *uniq = S.get<uint64_t>(n), *sums = S.get<uint64_t>(n);
  int64_t *d_num = S.get<int64_t>(4);
  if (S.err) return -(int)S.err;
  // the split sort of the occurrences (hi_s, lo_s sorted by fingerprint)
  auto split_sort = [&]() -> int {
    uint32_t *lo = S.get<uint32_t>(n);
    lo_s = S.get<uint32_t>(n);
    uint8_t *hi = nullptr;
    if (qr > 32) {
      hi = S.get<uint8_t>(n);
      hi_s = S.get<uint8_t>(n);
    }
    if (S.err) return -(int)S.err;
    k_hash_split<<<blocks_for(n), 256, 0, st>>>(keys, keys_are_fps, g->seed, fmask, n, hi, lo);
    if (qr <= 32) {
      FK_TRY(cub_sort_keys_u32(S, lo, lo_s, n, qr));
    } else {
      uint32_t *lo_p = S.get<uint32_t>(n);
      const int nseg = 1 << (qr - 32);
      int64_t *bounds = S.get<int64_t>(nseg + 1);
      if (S.err) return -(int)S.err;
      FK_TRY(cub_sort_pairs_u8_u32(S, hi, hi_s, lo, lo_p, n, qr - 32));
      k_u8_bounds<<<1, 256, 0, st>>>(hi_s, n, nseg, bounds);
      std::vector<int64_t> hb(nseg + 1);
      FK_TRY(cudaMemcpyAsync(hb.data(), bounds, (nseg + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      FK_TRY(cudaStreamSynchronize(st));
      for (int sgi = 0; sgi < nseg; sgi++)
        if (hb[sgi + 1] > hb[sgi]) FK_TRY(cub_sort_keys_u32(S, lo_p + hb[sgi], lo_s + hb[sgi], hb[sgi + 1] - hb[sgi], 32));
    }
    return 0;
  };
  if (split) {
    int W = 0, p2 = 0, rc = 1;
    if (part_plan(n, qr, &W, &p2))
      rc = part_count(S, keys, keys_are_fps, g->seed, fmask, qr, W, p2, n, uniq, sums, d_num);
    if (rc < 0) return rc;
    if (rc == 1) {  // the sort + run-length path
      int rs = split_sort();
      if (rs) return rs;
      FK_CU(cub_rle_counts_split(S, hi_s, lo_s, uniq, sums, d_num, n));
    }
  } else {
    fps_s = S.get<uint64_t>(n);
    del_s = S.get<uint64_t>(n);
    idx_s = S.get<uint32_t>(n);
    if (S.err) return -(int)S.err;
    fps = S.get<uint64_t>(n);
    idx = S.get<uint32_t>(n);
    if (S.err) return -(int)S.err;
    k_hash_fps<<<blocks_for(n), 256, 0, st>>>(keys, keys_are_fps, g->seed, fmask, n, fps, idx);
    if (plain_ins) {
      FK_CU(cub_sort_keys(S, fps, fps_s, n, qr));
      FK_CU(cub_rle_counts(S, fps_s, uniq, sums, d_num, n));
    } else {
      FK_CU(cub_sort_pairs(S, fps, fps_s, idx, idx_s, n, qr));
      const uint64_t dflt = is_del ? (1ull << 63) : 1ull;
      k_gather_u64<<<blocks_for(n), 256, 0, st>>>(deltas, idx_s, dflt, n, del_s);
      // 4. unique fingerprints with saturating delta sums: segment ids by a
      // scan of the segment ends (kept for the found flags), then one thread
      // per segment
      seg_heads = S.get<int64_t>(n);
      seg_ids = S.get<int64_t>(n);
      if (S.err) return -(int)S.err;
      k_seg_heads<<<blocks_for(n), 256, 0, st>>>(fps_s, n, seg_heads);
      FK_CU(cub_excl_sum_i64(S, seg_heads, seg_ids, n));
      k_seg_reduce<<<blocks_for(n), 256, 0, st>>>(fps_s, del_s, seg_ids, n, uniq, sums);
      k_seg_count<<<1, 1, 0, st>>>(seg_ids, n, d_num);
    }
  }
  int64_t m = 0;
  FK_CU(cudaMemcpyAsync(&m, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_CU(cudaStreamSynchronize(st));

  // 4'. small insert batches: region-local sequential inserts on a copy of
  // the table (the canonical result whenever nothing overflows); any
  // capacity failure discards the copy and falls through to the full path
  if (!is_del && !(flags & (kApplyDry | kApplyForceExact)) && m > 0 && m <= small_batch_limit(g)) {
    int rc = apply_small_t<S_t>(g, cur, nxt, uniq, sums, m, res, st);  // one insert per fingerprint
    if (rc <= 0) return rc;  // done (0) or an error (< 0); 1 = fall through
  }

  if (is_del && !(flags & (kApplyDry | kApplyForceExact)) && n <= small_batch_limit(g))
    return apply_small_delete_t<S_t>(g, cur, fps_s, del_s, idx_s, n, order, found, res, st);

  // Regions the batch touches: a batch within a quarter of them is applied
  // region-locally in place (8'); otherwise the whole table is decoded (8)
  // and the old counts come from joining the two sorted lists.
  bool exact = (flags & kApplyForceExact) != 0, load_possible = exact;
  const bool try_local = !exact && region_place_enabled() && local_apply_enabled();
  int64_t *creg = nullptr, Kreg = -1;
  if (try_local) {
    int lrc = local_regions(S, g, uniq, m, &creg, &Kreg);
    if (lrc) return lrc;
  }
  const bool go_local = try_local && local_applicable(g, Kreg);
  uint64_t *c_old = S.get<uint64_t>(m), *c_new = S.get<uint64_t>(m);
  if (S.err) return -(int)S.err;
  // 8. (global path) decode the old table into sorted (fp, count) items
  // (one thread per run)
  int64_t g_old = 0;
  uint64_t *o_fp = nullptr, *o_cnt = nullptr;
  if (!go_local) {
    RunDecode D;
    int drc = decode_runs_count<S_t>(S, g, cur, T0, &D, st);
    if (drc) return drc;
    g_old = D.items;
    o_fp = S.get<uint64_t>(g_old);
    o_cnt = S.get<uint64_t>(g_old);
    if (S.err) return -(int)S.err;
    drc = decode_runs_write<S_t>(T0, D, o_fp, o_cnt, st);
    if (drc) return drc;
  }

  // 5-6. old counts (the pure count query, or the join with the decoded
  // items), new absolute counts
  // An insert into an empty table (the bench's and a fresh filter's case):
  // the new counts are the batch sums and the merged items are the batch.
  const bool fresh_insert = !go_local && g_old == 0 && plain_ins;  // (explicit deltas may be 0)
  if (go_local) {
    k_gqf_count<S_t><<<blocks_for(m), 256, 0, st>>>(T0, uniq, 1, 0, m, c_old);
    k_new_counts<<<blocks_for(m), 256, 0, st>>>(c_old, sums, m, is_del ? 1 : 0, c_new);
  } else if (fresh_insert) {
    c_new = sums;
  } else {
    k_old_counts_join<<<blocks_for(join_threads(m)), 256, 0, st>>>(uniq, m, o_fp, o_cnt, g_old, sums, is_del ? 1 : 0,
                                                                   c_old, c_new);
  }

  // 7. delete found flags: sequential semantics via a segmented prefix sum,
  // computed in sorted order, then scattered to input order
  if (is_del && found) {
    uint8_t *found_s = S.get<uint8_t>(n);
    if (S.err) return -(int)S.err;
    if (m == n) {
      // no fingerprint repeats in the batch: a key is found iff its
      // fingerprint was present
      k_found_distinct<<<blocks_for(n), 256, 0, st>>>(c_old, n, found_s);
    } else {
      // one thread per segment walks its copies in the facade's order
      // (bulk: each region descending, gqf.py:317-325)
      k_found_walk<<<blocks_for(n), 256, 0, st>>>(fps_s, del_s, seg_ids, c_old, n, order == FK_ORDER_BULK ? 1 : 0,
                                                  found_s);
    }
    constexpr int kScatterShift = 25;  // 32 MiB of found bytes per pass
    for (int64_t p = 0; p <= ((n - 1) >> kScatterShift); p++)
      k_found_scatter<<<blocks_for(n), 256, 0, st>>>(found_s, idx_s, n, kScatterShift, p, found);
  }

  // 8'. region-local apply in place (mid-size batches; apply_local_t)
  bool region_done = false;
  unsigned long long region_shift = 0;
  MaxPlus *ends = nullptr;
  uint64_t *L = nullptr;
  int64_t G = 0;
  uint64_t *it_fp = nullptr, *it_cnt = nullptr;
  bool local_exact = false;
  if (go_local) {
    bool lp = false;
    const int lr = apply_local_t<S_t>(S, g, cur, creg, Kreg, keys, keys_are_fps, fmask, n, uniq, c_new, m, is_del,
                                      order, flags, res, &lp);
    if (lr <= 0) return lr;  // applied (or dry run answered), or an error
    if (lr == 2) {
      local_exact = exact = true;
      load_possible = lp;
    }
  }
  if (!local_exact) {
    if (go_local) {  // the local path declined: decode the whole table after all
      RunDecode D;
      int drc = decode_runs_count<S_t>(S, g, cur, T0, &D, st);
      if (drc) return drc;
      g_old = D.items;
      o_fp = S.get<uint64_t>(g_old);
      o_cnt = S.get<uint64_t>(g_old);
      if (S.err) return -(int)S.err;
      drc = decode_runs_write<S_t>(T0, D, o_fp, o_cnt, st);
      if (drc) return drc;
    }

    // 9-10. drop old items the batch updates and zero counts, then merge the
    // two duplicate-free sorted lists
    if (fresh_insert) {
      G = m;  // counts are positive sums
      it_fp = uniq;
      it_cnt = sums;
    } else {
    uint8_t *keep_o = S.get<uint8_t>(g_old), *keep_u = S.get<uint8_t>(m);
    uint64_t *o2_fp = S.get<uint64_t>(g_old), *o2_cnt = S.get<uint64_t>(g_old);
    uint64_t *u2_fp = S.get<uint64_t>(m), *u2_cnt = S.get<uint64_t>(m);
    if (S.err) return -(int)S.err;
    k_keep_old_join<<<blocks_for(join_threads(g_old)), 256, 0, st>>>(o_fp, g_old, uniq, m, keep_o);
    k_nonzero<<<blocks_for(m), 256, 0, st>>>(c_new, m, keep_u);
    FK_CU(cub_select_flagged(S, o_fp, keep_o, o2_fp, d_num, g_old));
    FK_CU(cub_select_flagged(S, o_cnt, keep_o, o2_cnt, d_num + 1, g_old));
    FK_CU(cub_select_flagged(S, uniq, keep_u, u2_fp, d_num + 2, m));
    FK_CU(cub_select_flagged(S, c_new, keep_u, u2_cnt, d_num + 3, m));
    int64_t hn[4];
    FK_CU(cudaMemcpyAsync(hn, d_num, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FK_CU(cudaStreamSynchronize(st));
    G = hn[0] + hn[2];
    it_fp = S.get<uint64_t>(G);
    it_cnt = S.get<uint64_t>(G);
    if (S.err) return -(int)S.err;
    if (G > 0) FK_CU(cub_merge(S, o2_fp, o2_cnt, hn[0], u2_fp, u2_cnt, hn[2], it_fp, it_cnt));
    }

    // 11-12. placement and the capacity predicates.  Region placement
    // (default): per-region max-plus summaries, a scan over the regions, then
    // one CTA per region writes its whole slot range of `next` and reports a
    // broken layout; the result is used unless the batch needs the exact path.
    if (!exact && region_place_enabled()) {
      const int64_t nqr = g->quotient_regions;
      int64_t *ib = S.get<int64_t>(nqr + 1);
      MaxPlus *summ = S.get<MaxPlus>(nqr), *cum = S.get<MaxPlus>(nqr);
      unsigned long long *acc = S.get<unsigned long long>(4);  // [0] slots, [1] counts, [2] shift
      unsigned *rflags = S.get<unsigned>(2);                   // [0] broken layout, [1] not ascending
      if (S.err) return -(int)S.err;
      FK_CU(cudaMemsetAsync(acc, 0, 4 * sizeof(unsigned long long), st));
      FK_CU(cudaMemsetAsync(rflags, 0, 2 * sizeof(unsigned), st));
      if (G > 0) k_region_bounds<<<blocks_for(nqr + 1), 256, 0, st>>>(it_fp, G, g->r + kRegionBits, nqr, ib);
      else FK_CU(cudaMemsetAsync(ib, 0, (nqr + 1) * sizeof(int64_t), st));
      const int rgrid = (int)(nqr < (int64_t)num_sms() * 8 ? nqr : (int64_t)num_sms() * 8);
      k_region_summary<<<rgrid, kRegThreads, 0, st>>>(it_fp, it_cnt, ib, nullptr, nqr, nullptr, g->r, summ, acc);
      FK_CU(cub_maxplus_scan(S, summ, cum, nqr));
      if (order == FK_ORDER_POINT)  // point order: the shift metric counts the batch's own slots unless ascending
        k_not_ascending<<<blocks_for(n), 256, 0, st>>>(keys, keys_are_fps, g->seed, fmask, n, rflags + 1);
      RegionJob<S_t> job{nullptr, nqr, nqr, nullptr, 0, nullptr, nullptr};
      k_region_place<S_t><<<rgrid, kRegThreads, 0, st>>>(make_dev(g, nxt), reinterpret_cast<const S_t *>(cur->slots),
                                                         cur->runends, it_fp, it_cnt, ib, cum, job, rflags + 1,
                                                         order == FK_ORDER_BULK ? 1 : 0, rflags, acc + 2);
      k_region_stats<<<1, 1, 0, st>>>(acc, G, nxt->stats);
      unsigned long long hacc[3];
      unsigned hfl = 0;
      FK_CU(cudaMemcpyAsync(hacc, acc, sizeof(hacc), cudaMemcpyDeviceToHost, st));
      FK_CU(cudaMemcpyAsync(&hfl, rflags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
      FK_CU(cudaStreamSynchronize(st));
      FK_CHECK_LAUNCH();
      const int64_t h_occ = (int64_t)hacc[0];
      if (!is_del) {
        // every item's pre-insert occupancy is <= the final one, so a final
        // occupancy below the ceiling rules LOAD_CAPACITY out for any order
        exact = hfl != 0 || h_occ >= g->max_occupied;
        load_possible = h_occ >= g->max_occupied;
      }
      region_done = hfl == 0;  // (a delete never breaks the layout of a valid table)
      region_shift = hacc[2];
    }
    if (!region_done && !exact) {
      // global placement: max-plus scan over every item
      MaxPlus *terms = S.get<MaxPlus>(G);
      ends = S.get<MaxPlus>(G);
      L = S.get<uint64_t>(G);
      if (S.err) return -(int)S.err;
      if (G > 0) {
        k_place_terms<<<blocks_for(G), 256, 0, st>>>(it_fp, it_cnt, G, g->r, terms, L);
        FK_CU(cub_maxplus_scan(S, terms, ends, G));
      }
      // would the sequential reference have raised?  (inserts only)
      if (!is_del && G > 0) {
        int64_t *cfirst = S.get<int64_t>(G), *cfs = S.get<int64_t>(G);
        unsigned *cflags = S.get<unsigned>(4);
        if (S.err) return -(int)S.err;
        FK_CU(cudaMemsetAsync(cflags, 0, 4 * sizeof(unsigned), st));
        k_cluster_check<<<blocks_for(G), 256, 0, st>>>(it_fp, ends, G, g->r, g->phys, cfirst, cflags);
        FK_CU(cub_max_scan_i64(S, cfirst, cfs, G));
        k_cluster_check2<<<blocks_for(G), 256, 0, st>>>(ends, cfs, cfirst, G, g->phys, cflags);
        int64_t *occ_sum = S.get<int64_t>(4);
        if (S.err) return -(int)S.err;
        FK_CU(cudaMemsetAsync(occ_sum, 0, 4 * sizeof(int64_t), st));
        k_stats<<<blocks_for(G), 256, 0, st>>>(it_cnt, L, G, occ_sum);
        unsigned h_flags = 0;
        int64_t h_occ = 0;
        FK_CU(cudaMemcpyAsync(&h_flags, cflags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        FK_CU(cudaMemcpyAsync(&h_occ, occ_sum, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        FK_CU(cudaStreamSynchronize(st));
        exact = h_flags != 0 || h_occ >= g->max_occupied;
        load_possible = h_occ >= g->max_occupied;
      }
    }
  }

  if (flags & kApplyDry) {
    res->code = exact ? 1 : 0;
    return 0;
  }
  if (exact && order == FK_ORDER_POINT && !(flags & kApplyForceExact) && n > kExactSeqDirect) {
    // 13''. the reference fails at the first key whose insertion overflows;
    // "the canonical layout of a prefix is safe" is monotone in the prefix
    // length (inserts only grow clusters and occupancy) and implies that the
    // reference raised nothing on it, so the longest safe prefix is applied
    // canonically and only the keys after it run sequentially.
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      int64_t mid = lo + (hi - lo) / 2;
      fk_gqf_result r2{};
      int rc = apply_t<S_t>(g, cur, nxt, keys, keys_are_fps, deltas, mid, op, order, nullptr, &r2, st, kApplyDry);
      if (rc) return rc;
      if (r2.code == 0) lo = mid; else hi = mid;
    }
    const fk_gqf_tables *c2 = cur, *n2 = nxt;
    if (lo > 0) {
      fk_gqf_result r3{};
      int rc = apply_t<S_t>(g, cur, nxt, keys, keys_are_fps, deltas, lo, op, order, nullptr, &r3, st);
      if (rc) return rc;
      if (r3.code) return FK_E_INVARIANT;  // a safe prefix cannot fail
      res->shifted += r3.shifted;
      if (r3.swapped) {
        res->swapped = 1;
        c2 = nxt;
        n2 = cur;
      }
    }
    fk_gqf_result r4{};
    int rc = apply_t<S_t>(g, c2, n2, keys + lo, keys_are_fps, deltas ? deltas + lo : nullptr, n - lo, op, order,
                          nullptr, &r4, st, kApplyForceExact);
    if (rc) return rc;
    res->code = r4.code;
    res->fail_index = r4.fail_index >= 0 ? r4.fail_index + lo : -1;
    res->shifted += r4.shifted;
    return 0;
  }

  if (exact) {
    // 13'. exact sequential application in place on `cur`
    if (order == FK_ORDER_POINT) {
      int32_t *scr = S.get<int32_t>(SeqGqf<S_t>::kGapCap);
      int64_t *out3 = S.get<int64_t>(4);
      if (S.err) return -(int)S.err;
      if (!fps) {  // the split sort never materialised the input-order fingerprints
        fps = S.get<uint64_t>(n);
        idx = S.get<uint32_t>(n);
        if (S.err) return -(int)S.err;
        k_hash_fps<<<blocks_for(n), 256, 0, st>>>(keys, keys_are_fps, g->seed, fmask, n, fps, idx);
      }
      k_gqf_exact_seq<S_t><<<1, 1, 0, st>>>(T0, fps, deltas, n, scr, out3);
      int64_t h3[3];
      FK_CU(cudaMemcpyAsync(h3, out3, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      FK_CU(cudaStreamSynchronize(st));
      if (h3[0] < 0) return FK_E_INVARIANT;
      res->code = (int32_t)h3[0];
      res->fail_index = h3[1];
      res->shifted = h3[2];
    } else {
      int64_t nqr = g->quotient_regions;
      int64_t *rb = S.get<int64_t>(nqr + 1);
      int32_t *fail = S.get<int32_t>(nqr);
      unsigned long long *moved = S.get<unsigned long long>(1);
      int64_t half = (nqr + 1) / 2;
      int32_t *scr = S.get<int32_t>((size_t)half * SeqGqf<S_t>::kGapCap);
      if (S.err) return -(int)S.err;
      FK_CU(cudaMemsetAsync(fail, 0, nqr * sizeof(int32_t), st));
      FK_CU(cudaMemsetAsync(moved, 0, sizeof(unsigned long long), st));
      if (plain_ins) {
        if (!fps_s) {  // sorted occurrences from the split sort
          fps_s = S.get<uint64_t>(n);
          if (S.err) return -(int)S.err;
          if (!lo_s) {  // counted by partitions: sort the occurrences now
            int rs = split_sort();
            if (rs) return rs;
          }
          k_widen_split<<<blocks_for(n), 256, 0, st>>>(hi_s, lo_s, n, fps_s);
        }
        if (!del_s) del_s = S.get<uint64_t>(n);
        if (S.err) return -(int)S.err;
        k_gather_u64<<<blocks_for(n), 256, 0, st>>>(nullptr, nullptr, 1ull, n, del_s);  // all ones
      }
      k_region_bounds<<<blocks_for(nqr + 1), 256, 0, st>>>(fps_s, n, g->r + kRegionBits, nqr, rb);
      // the ceiling check reads the shared occupancy counter, so when it can
      // trigger, regions run one after another in the reference's workers=1
      // order (even ascending, then odd); otherwise a parity's regions are
      // independent (disjoint [g, g+2) windows) and run in parallel
      for (int parity = 0; parity < 2; parity++) {
        if (load_possible)
          k_gqf_exact_regions<S_t><<<1, 1, 0, st>>>(T0, fps_s, del_s, rb, nqr, parity, scr, fail, moved);
        else
          k_gqf_exact_regions<S_t><<<blocks_for(half, 64), 64, 0, st>>>(T0, fps_s, del_s, rb, nqr, parity, scr,
                                                                         fail, moved);
      }
      std::vector<int32_t> hf(nqr);
      unsigned long long hm = 0;
      FK_CU(cudaMemcpyAsync(hf.data(), fail, nqr * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      FK_CU(cudaMemcpyAsync(&hm, moved, sizeof(hm), cudaMemcpyDeviceToHost, st));
      FK_CU(cudaStreamSynchronize(st));
      for (int parity = 0; parity < 2 && res->code == 0; parity++)
        for (int64_t gg = parity; gg < nqr; gg += 2)
          if (hf[gg]) {
            if (hf[gg] < 0) return FK_E_INVARIANT;
            res->code = hf[gg];
            res->fail_region = gg;
            break;
          }
      res->shifted = (int64_t)hm;
    }
    int rc = rebuild_index(g, cur, st);
    if (rc) return rc;
    FK_CU(cudaStreamSynchronize(st));
    return 0;
  }

  // 13. canonical rebuild into `next`
  if (region_done) {  // already written region by region
    int rc = rebuild_index(g, nxt, st);
    if (rc) return rc;
    res->shifted = (int64_t)region_shift;
    res->swapped = 1;
    FK_CHECK_LAUNCH();
    return 0;
  }
  GqfDev T1 = make_dev(g, nxt);
  FK_CU(cudaMemsetAsync(nxt->slots, 0, (size_t)g->phys * sizeof(S_t), st));
  FK_CU(cudaMemsetAsync(nxt->occupieds, 0, (size_t)(g->phys >> 6) * 8, st));
  FK_CU(cudaMemsetAsync(nxt->runends, 0, (size_t)(g->phys >> 6) * 8, st));
  FK_CU(cudaMemsetAsync(nxt->offsets, 0, (size_t)g->num_regions * 4, st));
  FK_CU(cudaMemsetAsync(nxt->stats, 0, 3 * sizeof(int64_t), st));
  if (G > 0) {
    k_write_items<S_t><<<blocks_for(G), 256, 0, st>>>(T1, it_fp, it_cnt, ends, L, G);
    k_stats<<<blocks_for(G), 256, 0, st>>>(it_cnt, L, G, nxt->stats);
    FK_CU(cudaMemcpyAsync(nxt->stats + 2, &G, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  }
  int rc = rebuild_index(g, nxt, st);
  if (rc) return rc;
  // shift instrumentation: bulk = old slots that moved; point = every slot
  // the batch wrote or moved
  unsigned long long *dc = S.get<unsigned long long>(1);
  if (S.err) return -(int)S.err;
  FK_CU(cudaMemsetAsync(dc, 0, sizeof(unsigned long long), st));
  // point order counts the batch's own slots too (a later item can move an
  // earlier one's), unless the batch is non-decreasing (k_not_ascending)
  unsigned *nasc = S.get<unsigned>(1);
  if (S.err) return -(int)S.err;
  unsigned h_nasc = 1;
  if (order == FK_ORDER_POINT) {
    FK_CU(cudaMemsetAsync(nasc, 0, sizeof(unsigned), st));
    k_not_ascending<<<blocks_for(n), 256, 0, st>>>(keys, keys_are_fps, g->seed, fmask, n, nasc);
    FK_CU(cudaMemcpyAsync(&h_nasc, nasc, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    FK_CU(cudaStreamSynchronize(st));
  }
  k_diff_count<S_t><<<blocks_for(g->phys), 256, 0, st>>>(
      reinterpret_cast<const S_t *>(cur->slots), cur->runends, reinterpret_cast<const S_t *>(nxt->slots),
      nxt->runends, g->phys, (order == FK_ORDER_BULK || !h_nasc) ? 1 : 0, dc);
  unsigned long long hdc = 0;
  FK_CU(cudaMemcpyAsync(&hdc, dc, sizeof(hdc), cudaMemcpyDeviceToHost, st));
  FK_CU(cudaStreamSynchronize(st));
  res->shifted = (int64_t)hdc;
  res->swapped = 1;
  FK_CHECK_LAUNCH();
  return 0;
}

}  // namespace

}  // namespace fk

using namespace fk;

extern "C" {

int fk_gqf_count(const fk_gqf_geom *g, const fk_gqf_tables *t, const uint64_t *keys, int keys_are_fps, int64_t n,
                 uint64_t *counts, void *stream) {
  if (!geom_ok(g) || !t || n < 0) return FK_E_ARG;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->r) {
    case 8: return count_t<uint8_t>(g, t, keys, keys_are_fps, n, counts, st);
    case 16: return count_t<uint16_t>(g, t, keys, keys_are_fps, n, counts, st);
    default: return count_t<uint32_t>(g, t, keys, keys_are_fps, n, counts, st);
  }
}

int fk_gqf_find_run(const fk_gqf_geom *g, const fk_gqf_tables *t, const int64_t *quotients, int64_t n, int64_t *se,
                    void *stream) {
  if (!geom_ok(g) || !t || n < 0) return FK_E_ARG;
  if (n == 0) return 0;
  GqfDev T = make_dev(g, t);
  k_gqf_find_run<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(T, quotients, n, se);
  FK_CHECK_LAUNCH();
  return 0;
}

int fk_gqf_enumerate(const fk_gqf_geom *g, const fk_gqf_tables *t, uint64_t *fp_out, uint64_t *cnt_out, int64_t cap,
                     int64_t *count_out, void *stream) {
  if (!geom_ok(g) || !t || !count_out || cap < 0) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->r) {
    case 8: return enumerate_t<uint8_t>(g, t, fp_out, cnt_out, cap, count_out, st);
    case 16: return enumerate_t<uint16_t>(g, t, fp_out, cnt_out, cap, count_out, st);
    default: return enumerate_t<uint32_t>(g, t, fp_out, cnt_out, cap, count_out, st);
  }
}

int fk_gqf_validate(const fk_gqf_geom *g, const fk_gqf_tables *t, int64_t *out, void *stream) {
  if (!geom_ok(g) || !t || !out) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->r) {
    case 8: return validate_t<uint8_t>(g, t, out, st);
    case 16: return validate_t<uint16_t>(g, t, out, st);
    default: return validate_t<uint32_t>(g, t, out, st);
  }
}

int fk_gqf_cluster_stats(const fk_gqf_geom *g, const fk_gqf_tables *t, int64_t *out3, void *stream) {
  if (!geom_ok(g) || !t || !out3) return FK_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch S(st);
  const int64_t nw = g->phys >> 6;
  int64_t *po = S.get<int64_t>(nw), *pr = S.get<int64_t>(nw), *oo = S.get<int64_t>(nw), *orr = S.get<int64_t>(nw);
  if (S.err) return -(int)S.err;
  k_word_popc<<<blocks_for(nw), 256, 0, st>>>(t->occupieds, nw, po);
  k_word_popc<<<blocks_for(nw), 256, 0, st>>>(t->runends, nw, pr);
  FK_TRY(cub_excl_sum_i64(S, po, oo, nw));
  FK_TRY(cub_excl_sum_i64(S, pr, orr, nw));
  int64_t h[4];
  FK_TRY(cudaMemcpyAsync(&h[0], oo + nw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaMemcpyAsync(&h[1], po + nw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaMemcpyAsync(&h[2], orr + nw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaMemcpyAsync(&h[3], pr + nw - 1, 8, cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  const int64_t K = h[0] + h[1];
  if (K != h[2] + h[3]) return FK_E_INVARIANT;  // occupieds / runends set-bit counts differ
  out3[0] = out3[1] = out3[2] = 0;
  if (K == 0) return 0;
  int64_t *Q = S.get<int64_t>(K), *E = S.get<int64_t>(K), *brk = S.get<int64_t>(K), *len = S.get<int64_t>(K);
  int64_t *cid = S.get<int64_t>(K), *ukey = S.get<int64_t>(K), *clen = S.get<int64_t>(K), *d3 = S.get<int64_t>(4);
  if (S.err) return -(int)S.err;
  k_bit_positions<<<blocks_for(nw), 256, 0, st>>>(t->occupieds, nw, oo, Q);
  k_bit_positions<<<blocks_for(nw), 256, 0, st>>>(t->runends, nw, orr, E);
  k_run_clusters<<<blocks_for(K), 256, 0, st>>>(Q, E, K, brk, len);
  size_t tb = 0;
  FK_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb, brk, cid, K, st));
  void *tmp = S.get<char>(tb);
  if (!tmp) return -(int)S.err;
  FK_TRY(cub::DeviceScan::InclusiveSum(tmp, tb, brk, cid, K, st));
  // per-cluster lengths (sum of its runs' lengths: runs of a cluster are contiguous)
  tb = 0;
  FK_TRY(cub::DeviceReduce::ReduceByKey(nullptr, tb, cid, ukey, len, clen, d3, cuda::std::plus<>(), K, st));
  tmp = S.get<char>(tb);
  if (!tmp) return -(int)S.err;
  FK_TRY(cub::DeviceReduce::ReduceByKey(tmp, tb, cid, ukey, len, clen, d3, cuda::std::plus<>(), K, st));
  int64_t nc = 0;
  FK_TRY(cudaMemcpyAsync(&nc, d3, 8, cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  tb = 0;
  FK_TRY(cub::DeviceReduce::Max(nullptr, tb, clen, d3 + 1, nc, st));
  tmp = S.get<char>(tb);
  if (!tmp) return -(int)S.err;
  FK_TRY(cub::DeviceReduce::Max(tmp, tb, clen, d3 + 1, nc, st));
  tb = 0;
  FK_TRY(cub::DeviceReduce::Sum(nullptr, tb, clen, d3 + 2, nc, st));
  tmp = S.get<char>(tb);
  if (!tmp) return -(int)S.err;
  FK_TRY(cub::DeviceReduce::Sum(tmp, tb, clen, d3 + 2, nc, st));
  FK_TRY(cudaMemcpyAsync(out3, d3, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FK_TRY(cudaStreamSynchronize(st));
  return 0;
}

int fk_gqf_rebuild_index(const fk_gqf_geom *g, const fk_gqf_tables *t, void *stream) {
  if (!geom_ok(g) || !t) return FK_E_ARG;
  return rebuild_index(g, t, (cudaStream_t)stream);
}

int fk_gqf_apply(const fk_gqf_geom *g, const fk_gqf_tables *cur, const fk_gqf_tables *next, const uint64_t *keys,
                 int keys_are_fps, const uint64_t *deltas, int64_t n, int op, int order, uint8_t *found,
                 fk_gqf_result *result, void *stream) {
  if (!geom_ok(g) || !cur || !next || !result || n < 0 || n > 0xFFFFFFF0LL) return FK_E_ARG;
  if (op != FK_GQF_INSERT && op != FK_GQF_DELETE) return FK_E_ARG;
  result->code = 0;
  result->swapped = 0;
  result->fail_index = -1;
  result->fail_region = -1;
  result->shifted = 0;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  switch (g->r) {
    case 8: return apply_t<uint8_t>(g, cur, next, keys, keys_are_fps, deltas, n, op, order, found, result, st);
    case 16: return apply_t<uint16_t>(g, cur, next, keys, keys_are_fps, deltas, n, op, order, found, result, st);
    default: return apply_t<uint32_t>(g, cur, next, keys, keys_are_fps, deltas, n, op, order, found, result, st);
  }
}

// ---- contract-shaped entries (the reference's raw-array kernel contract) ----
//
// gqf_insert_batch / gqf_delete_batch (_ckernels.pyx:1147-1202, :1253-1296)
// mutate ONE table image in place and process the fingerprints in input
// order.  fk_gqf_apply may leave its result in a second image (canonical
// rebuild); these wrappers give it stream-ordered scratch for that image and
// copy the result back, so the caller sees the contract's in-place update.
// The derived run index (t->spill) is rebuilt from the bit vectors first:
// a contract caller hands in raw arrays it may have written itself.
static int contract_apply(const fk_gqf_geom *g, const fk_gqf_tables *t, const uint64_t *fps, const uint64_t *deltas,
                          int64_t n, int op, uint8_t *found, fk_gqf_result *res, cudaStream_t st) {
  int rc = rebuild_index(g, t, st);
  if (rc) return rc;
  const size_t sb = g->r / 8;
  const size_t words = (size_t)(g->phys >> 6);
  const size_t spill = (size_t)((1LL << g->q) >> 6) > 0 ? (size_t)((1LL << g->q) >> 6) : 1;
  Scratch S(st);
  fk_gqf_tables nx;
  nx.slots = S.get<char>((size_t)g->phys * sb);
  nx.occupieds = S.get<uint64_t>(words);
  nx.runends = S.get<uint64_t>(words);
  nx.offsets = S.get<int32_t>((size_t)g->num_regions);
  nx.stats = S.get<int64_t>(3);
  nx.spill = S.get<uint32_t>(spill);
  if (S.err) return -(int)S.err;
  rc = fk_gqf_apply(g, t, &nx, fps, 1, deltas, n, op, FK_ORDER_POINT, found, res, st);
  if (rc) return rc;
  if (res->swapped) {
    FK_CU(cudaMemcpyAsync(t->slots, nx.slots, (size_t)g->phys * sb, cudaMemcpyDeviceToDevice, st));
    FK_CU(cudaMemcpyAsync(t->occupieds, nx.occupieds, words * 8, cudaMemcpyDeviceToDevice, st));
    FK_CU(cudaMemcpyAsync(t->runends, nx.runends, words * 8, cudaMemcpyDeviceToDevice, st));
    FK_CU(cudaMemcpyAsync(t->offsets, nx.offsets, (size_t)g->num_regions * 4, cudaMemcpyDeviceToDevice, st));
    FK_CU(cudaMemcpyAsync(t->stats, nx.stats, 3 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    FK_CU(cudaMemcpyAsync(t->spill, nx.spill, spill * 4, cudaMemcpyDeviceToDevice, st));
    res->swapped = 0;
  }
  FK_CU(cudaStreamSynchronize(st));
  return 0;
}

int fk_gqf_insert_batch(const fk_gqf_geom *g, const fk_gqf_tables *t, const uint64_t *fps, const uint64_t *deltas,
                        int64_t n, int32_t *code, int64_t *fail_idx, int64_t *shift_out, void *stream) {
  if (!geom_ok(g) || !t || !code || !fail_idx || !deltas || n < 0 || n > 0xFFFFFFF0LL) return FK_E_ARG;
  *code = 0;
  *fail_idx = -1;
  if (n == 0) return 0;
  fk_gqf_result res{};
  int rc = contract_apply(g, t, fps, deltas, n, FK_GQF_INSERT, nullptr, &res, (cudaStream_t)stream);
  if (rc) return rc;
  *code = res.code;
  *fail_idx = res.code ? res.fail_index : -1;
  if (shift_out) *shift_out += res.shifted;
  return 0;
}

int fk_gqf_delete_batch(const fk_gqf_geom *g, const fk_gqf_tables *t, const uint64_t *fps, const uint64_t *deltas,
                        int64_t n, uint8_t *found, int64_t *shift_out, void *stream) {
  if (!geom_ok(g) || !t || !found || !deltas || n < 0 || n > 0xFFFFFFF0LL) return FK_E_ARG;
  if (n == 0) return 0;
  fk_gqf_result res{};
  int rc = contract_apply(g, t, fps, deltas, n, FK_GQF_DELETE, found, &res, (cudaStream_t)stream);
  if (rc) return rc;
  if (shift_out) *shift_out += res.shifted;
  return 0;
}

}  // extern "C"
