/*
 * oracle/fk_oracle.c -- CPU restatement of the filterkit kernel contract.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
 * paper_2212_09005_b200/) may link, load or call this file.  It is the checker
 * that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg compare
 * the CUDA path against.
 *
 * Every function restates one reference function; the citation is in the
 * comment above it ("ck" = /root/reference/pkg/src/filterkit/_ckernels.pyx,
 * "pk" = .../_pykernels.py, which is the normative readable twin).  Parity is
 * pinned by tests/golden/ fixtures generated from the reference itself
 * (tests/golden/make_golden.py) and by tests/test_oracle_vs_ref.py when the
 * reference build in oracle/_ref is present.
 *
 * Slot arrays are passed as (void *, wbytes) with wbytes in {1,2,4,8}; the
 * reference fuses the same functions over slot_t in {u8,u16,u32,u64}
 * (ck:92-96).  Everything is sequential: this is the "one thread calls
 * insert_many" semantics the GPU ordered modes must reproduce bit-exactly.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EMPTY_W 0u
#define TOMB_W 1u
#define REG_BITS 13
#define REG_SLOTS (1LL << REG_BITS)
#define GAP_CAP (2 * REG_SLOTS) /* ck:84 */
#define RC_INVARIANT (-9)       /* ck:77 */

/* hashing.py:22-25 */
#define K_BLOCK1 0x9E3779B97F4A7C15ULL
#define K_BLOCK2 0xC2B2AE3D27D4EB4FULL
#define K_BSTART 0x165667B19E3779F9ULL
#define K_BSTEP 0x27D4EB2F165667C5ULL

/* hashing.py:28-36 (SplitMix64 finalizer) */
uint64_t orc_mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

static inline uint64_t getw(const void *a, int wb, int64_t i) {
    switch (wb) {
    case 1: return ((const uint8_t *)a)[i];
    case 2: return ((const uint16_t *)a)[i];
    case 4: return ((const uint32_t *)a)[i];
    default: return ((const uint64_t *)a)[i];
    }
}
static inline void putw(void *a, int wb, int64_t i, uint64_t v) {
    switch (wb) {
    case 1: ((uint8_t *)a)[i] = (uint8_t)v; break;
    case 2: ((uint16_t *)a)[i] = (uint16_t)v; break;
    case 4: ((uint32_t *)a)[i] = (uint32_t)v; break;
    default: ((uint64_t *)a)[i] = v; break;
    }
}
static inline int live(uint64_t w) { return w != EMPTY_W && w != TOMB_W; }

/* hashing.py:120-132, pk:63-65 */
static inline uint64_t tag_word(uint64_t fp, int f) {
    uint64_t t = f >= 64 ? fp : (fp & ((1ULL << f) - 1));
    return t < 2 ? (t | 2) : t;
}
static inline uint64_t fmask_of(int f) { return f >= 64 ? ~0ULL : ((1ULL << f) - 1); }

/* hashing.py:66-73 */
void orc_fingerprint_many(const uint64_t *keys, int64_t n, uint64_t seed, int bits, uint64_t *out) {
    uint64_t m = bits >= 64 ? ~0ULL : ((1ULL << bits) - 1);
    for (int64_t i = 0; i < n; i++) out[i] = orc_mix64(keys[i] ^ seed) & m;
}

/* ------------------------------------------------------------------ */
/* point TCF                                                           */
/* ------------------------------------------------------------------ */

/* pk:77-83 */
static int64_t used_in_block(const void *blk, int wb, int64_t base, int B) {
    int64_t n = 0;
    for (int i = 0; i < B; i++) n += live(getw(blk, wb, base + i));
    return n;
}

/* pk:86-101: group width only strides the scan; claim order is ascending. */
static int claim_first_free(void *blk, int wb, int64_t base, int B, uint64_t word) {
    for (int i = 0; i < B; i++) {
        if (!live(getw(blk, wb, base + i))) {
            putw(blk, wb, base + i, word);
            return 1;
        }
    }
    return 0;
}

/* pk:104-117 */
static int backing_claim(void *bk, int wb, int64_t size, int probe_limit, uint64_t fp, uint64_t word) {
    if (size <= 0) return 0;
    uint64_t idx = orc_mix64(fp ^ K_BSTART) % (uint64_t)size;
    uint64_t step = (orc_mix64(fp ^ K_BSTEP) | 1) % (uint64_t)size;
    for (int t = 0; t < probe_limit; t++) {
        if (!live(getw(bk, wb, (int64_t)idx))) {
            putw(bk, wb, (int64_t)idx, word);
            return 1;
        }
        idx = (idx + step) % (uint64_t)size;
    }
    return 0;
}

/* pk:120-149 / ck:193-238.  Returns n_ok; *n_back_out gets backing placements. */
int64_t orc_tcf_insert_batch(void *blocks, int wb, int64_t nblocks, void *backing, int64_t bsize,
                             int B, int f, int cut, int probe_limit, const uint64_t *fps,
                             const uint64_t *values, int64_t n, uint8_t *codes, int64_t *n_back_out) {
    int64_t n_ok = 0, n_back = 0;
    for (int64_t k = 0; k < n; k++) {
        uint64_t fp = fps[k];
        uint64_t word = ((values ? values[k] : 0) << f) | tag_word(fp, f);
        if (f >= 64) word = tag_word(fp, f);
        int64_t b1 = (int64_t)(orc_mix64(fp ^ K_BLOCK1) % (uint64_t)nblocks);
        int64_t b2 = (int64_t)(orc_mix64(fp ^ K_BLOCK2) % (uint64_t)nblocks);
        int code = 3;
        if (used_in_block(blocks, wb, b1 * B, B) < cut && claim_first_free(blocks, wb, b1 * B, B, word)) {
            code = 0;
        } else {
            int64_t o1 = used_in_block(blocks, wb, b1 * B, B);
            int64_t o2 = used_in_block(blocks, wb, b2 * B, B);
            int64_t first = o1 <= o2 ? b1 : b2, second = o1 <= o2 ? b2 : b1;
            if (claim_first_free(blocks, wb, first * B, B, word)) code = first == b1 ? 0 : 1;
            else if (claim_first_free(blocks, wb, second * B, B, word)) code = second == b1 ? 0 : 1;
            else if (backing_claim(backing, wb, bsize, probe_limit, fp, word)) { code = 2; n_back++; }
        }
        if (code != 3) n_ok++;
        codes[k] = (uint8_t)code;
    }
    if (n_back_out) *n_back_out = n_back;
    return n_ok;
}

/* pk:152-158 */
static int64_t find_tag(const void *blk, int wb, int64_t base, int B, uint64_t tag, uint64_t fm) {
    for (int i = 0; i < B; i++) {
        uint64_t w = getw(blk, wb, base + i);
        if (live(w) && (w & fm) == tag) return base + i;
    }
    return -1;
}

/* pk:161-197 */
int64_t orc_tcf_query_batch(const void *blocks, int wb, int64_t nblocks, const void *backing, int64_t bsize,
                            int B, int f, int probe_limit, const uint64_t *fps, int64_t n,
                            uint8_t *found, uint64_t *values_out) {
    uint64_t fm = fmask_of(f);
    int64_t hits = 0;
    for (int64_t k = 0; k < n; k++) {
        uint64_t fp = fps[k], tag = tag_word(fp, f);
        int64_t b1 = (int64_t)(orc_mix64(fp ^ K_BLOCK1) % (uint64_t)nblocks);
        int64_t b2 = (int64_t)(orc_mix64(fp ^ K_BLOCK2) % (uint64_t)nblocks);
        int64_t at = find_tag(blocks, wb, b1 * B, B, tag, fm);
        if (at < 0) at = find_tag(blocks, wb, b2 * B, B, tag, fm);
        int hit = at >= 0;
        uint64_t val = hit ? (f >= 64 ? 0 : getw(blocks, wb, at) >> f) : 0;
        if (!hit && bsize > 0) {
            uint64_t p = orc_mix64(fp ^ K_BSTART) % (uint64_t)bsize;
            uint64_t step = (orc_mix64(fp ^ K_BSTEP) | 1) % (uint64_t)bsize;
            for (int t = 0; t < probe_limit; t++) {
                uint64_t w = getw(backing, wb, (int64_t)p);
                if (w == EMPTY_W) break;
                if (w != TOMB_W && (w & fm) == tag) {
                    hit = 1;
                    val = f >= 64 ? 0 : w >> f;
                    break;
                }
                p = (p + step) % (uint64_t)bsize;
            }
        }
        found[k] = (uint8_t)hit;
        if (values_out) values_out[k] = hit ? val : 0;
        hits += hit;
    }
    return hits;
}

/* pk:200-236 */
int64_t orc_tcf_delete_batch(void *blocks, int wb, int64_t nblocks, void *backing, int64_t bsize,
                             int B, int f, int probe_limit, const uint64_t *fps, int64_t n, uint8_t *removed) {
    uint64_t fm = fmask_of(f);
    int64_t cnt = 0;
    for (int64_t k = 0; k < n; k++) {
        uint64_t fp = fps[k], tag = tag_word(fp, f);
        int64_t b1 = (int64_t)(orc_mix64(fp ^ K_BLOCK1) % (uint64_t)nblocks);
        int64_t b2 = (int64_t)(orc_mix64(fp ^ K_BLOCK2) % (uint64_t)nblocks);
        int64_t at = find_tag(blocks, wb, b1 * B, B, tag, fm);
        if (at < 0) at = find_tag(blocks, wb, b2 * B, B, tag, fm);
        int done = 0;
        if (at >= 0) {
            putw(blocks, wb, at, TOMB_W);
            done = 1;
        } else if (bsize > 0) {
            uint64_t p = orc_mix64(fp ^ K_BSTART) % (uint64_t)bsize;
            uint64_t step = (orc_mix64(fp ^ K_BSTEP) | 1) % (uint64_t)bsize;
            for (int t = 0; t < probe_limit; t++) {
                uint64_t w = getw(backing, wb, (int64_t)p);
                if (w == EMPTY_W) break;
                if (w != TOMB_W && (w & fm) == tag) {
                    putw(backing, wb, (int64_t)p, TOMB_W);
                    done = 1;
                    break;
                }
                p = (p + step) % (uint64_t)bsize;
            }
        }
        removed[k] = (uint8_t)done;
        cnt += done;
    }
    return cnt;
}

/* ------------------------------------------------------------------ */
/* bulk TCF                                                            */
/* ------------------------------------------------------------------ */

/* pk:244-263 / ck:363-405: merge sorted words[lo:hi) into block b's sorted prefix. */
int64_t orc_btcf_merge_lists(void *blocks, int wb, uint32_t *fill, int B, const void *words,
                             const int64_t *starts, const int64_t *ends, int64_t b_lo, int64_t b_hi) {
    for (int64_t b = b_lo; b < b_hi; b++) {
        int64_t lo = starts[b], hi = ends[b];
        if (lo >= hi) continue;
        int64_t m = hi - lo, cur = fill[b], base = b * (int64_t)B;
        if (cur + m > B) return 1 + b;
        int64_t i = cur - 1, j = hi - 1, o = cur + m - 1;
        while (j >= lo) {
            if (i >= 0 && getw(blocks, wb, base + i) > getw(words, wb, j)) {
                putw(blocks, wb, base + o, getw(blocks, wb, base + i));
                i--;
            } else {
                putw(blocks, wb, base + o, getw(words, wb, j));
                j--;
            }
            o--;
        }
        fill[b] = (uint32_t)(cur + m);
    }
    return 0;
}

/* pk:266-287 / ck:408-444: sequential greedy two-choice routing. */
int orc_btcf_route(const uint32_t *fill, int64_t nb, int B, const int64_t *b1s, const int64_t *b2s,
                   int64_t n, int64_t *dest) {
    int64_t *pend = (int64_t *)calloc((size_t)(nb > 0 ? nb : 1), sizeof(int64_t));
    if (!pend) return -1;
    for (int64_t k = 0; k < n; k++) {
        int64_t x = b1s[k], y = b2s[k];
        int64_t lx = (int64_t)fill[x] + pend[x], ly = (int64_t)fill[y] + pend[y];
        int64_t pick = lx <= ly ? x : y, other = lx <= ly ? y : x;
        if ((int64_t)fill[pick] + pend[pick] >= B) {
            pick = other;
            if ((int64_t)fill[pick] + pend[pick] >= B) {
                dest[k] = -1;
                continue;
            }
        }
        pend[pick]++;
        dest[k] = pick;
    }
    free(pend);
    return 0;
}

/* pk:290-301 */
int64_t orc_backing_insert_batch(void *backing, int wb, int64_t bsize, int probe_limit, int f,
                                 const uint64_t *fps, int64_t n, uint8_t *codes) {
    int64_t fails = 0;
    for (int64_t k = 0; k < n; k++) {
        if (backing_claim(backing, wb, bsize, probe_limit, fps[k], tag_word(fps[k], f))) codes[k] = 2;
        else { codes[k] = 3; fails++; }
    }
    return fails;
}

/* pk:366-375 */
static int64_t bisect_block(const void *blk, int wb, int64_t base, int64_t n, uint64_t word) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (getw(blk, wb, base + mid) < word) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/* pk:315-337 */
int64_t orc_btcf_delete_blocklocal(void *blocks, int wb, uint32_t *fill, int B, const void *words,
                                   const int64_t *starts, const int64_t *ends, int64_t b_lo, int64_t b_hi,
                                   uint8_t *removed) {
    int64_t cnt = 0;
    for (int64_t b = b_lo; b < b_hi; b++) {
        int64_t base = b * (int64_t)B;
        for (int64_t k = starts[b]; k < ends[b]; k++) {
            uint64_t word = getw(words, wb, k);
            int64_t cur = fill[b];
            int64_t i = bisect_block(blocks, wb, base, cur, word);
            if (i < cur && getw(blocks, wb, base + i) == word) {
                for (int64_t t = i; t < cur - 1; t++) putw(blocks, wb, base + t, getw(blocks, wb, base + t + 1));
                putw(blocks, wb, base + cur - 1, EMPTY_W);
                fill[b] = (uint32_t)(cur - 1);
                removed[k] = 1;
                cnt++;
            } else {
                removed[k] = 0;
            }
        }
    }
    return cnt;
}

/* pk:340-363 */
int64_t orc_backing_delete_batch(void *backing, int wb, int64_t bsize, int probe_limit, int f,
                                 const uint64_t *fps, int64_t n, uint8_t *removed) {
    uint64_t fm = fmask_of(f);
    int64_t cnt = 0;
    for (int64_t k = 0; k < n; k++) {
        uint64_t fp = fps[k], word = tag_word(fp, f);
        int done = 0;
        if (bsize > 0) {
            uint64_t p = orc_mix64(fp ^ K_BSTART) % (uint64_t)bsize;
            uint64_t step = (orc_mix64(fp ^ K_BSTEP) | 1) % (uint64_t)bsize;
            for (int t = 0; t < probe_limit; t++) {
                uint64_t w = getw(backing, wb, (int64_t)p);
                if (w == EMPTY_W) break;
                if (w != TOMB_W && (w & fm) == word) {
                    putw(backing, wb, (int64_t)p, TOMB_W);
                    done = 1;
                    break;
                }
                p = (p + step) % (uint64_t)bsize;
            }
        }
        removed[k] = (uint8_t)done;
        cnt += done;
    }
    return cnt;
}

/* pk:378-411 */
int64_t orc_btcf_query_batch(const void *blocks, int wb, const uint32_t *fill, int64_t nblocks,
                             const void *backing, int64_t bsize, int B, int f, int probe_limit,
                             const uint64_t *fps, int64_t n, uint8_t *found) {
    uint64_t fm = fmask_of(f);
    int64_t hits = 0;
    for (int64_t k = 0; k < n; k++) {
        uint64_t fp = fps[k], word = tag_word(fp, f);
        int hit = 0;
        for (int which = 0; which < 2 && !hit; which++) {
            int64_t b = (int64_t)(orc_mix64(fp ^ (which ? K_BLOCK2 : K_BLOCK1)) % (uint64_t)nblocks);
            int64_t base = b * (int64_t)B, cur = fill[b];
            int64_t i = bisect_block(blocks, wb, base, cur, word);
            if (i < cur && getw(blocks, wb, base + i) == word) hit = 1;
        }
        if (!hit && bsize > 0) {
            uint64_t p = orc_mix64(fp ^ K_BSTART) % (uint64_t)bsize;
            uint64_t step = (orc_mix64(fp ^ K_BSTEP) | 1) % (uint64_t)bsize;
            for (int t = 0; t < probe_limit; t++) {
                uint64_t w = getw(backing, wb, (int64_t)p);
                if (w == EMPTY_W) break;
                if (w != TOMB_W && (w & fm) == word) { hit = 1; break; }
                p = (p + step) % (uint64_t)bsize;
            }
        }
        found[k] = (uint8_t)hit;
        hits += hit;
    }
    return hits;
}

/* ------------------------------------------------------------------ */
/* GQF                                                                 */
/* ------------------------------------------------------------------ */

typedef struct {
    void *slots;
    int wb;
    uint64_t *occ, *run;
    int32_t *offs;
    int64_t *stats;
    int64_t phys;
    int q, r;
    int64_t *scratch; /* GAP_CAP entries */
} gqf_t;

static inline int bit_get(const uint64_t *bv, int64_t i) { return (int)((bv[i >> 6] >> (i & 63)) & 1); }
static inline void bit_put(uint64_t *bv, int64_t i, int v) {
    uint64_t m = 1ULL << (i & 63);
    if (v) bv[i >> 6] |= m;
    else bv[i >> 6] &= ~m;
}

/* pk:429-442: set bits in [a, b) */
static int64_t rank_range(const uint64_t *bv, int64_t a, int64_t b) {
    if (a >= b) return 0;
    int64_t n = 0;
    for (int64_t i = a; i < b;) {
        int64_t wi = i >> 6, lo = i & 63;
        int64_t span = 64 - lo;
        if (span > b - i) span = b - i;
        uint64_t w = bv[wi] >> lo;
        if (span < 64) w &= (1ULL << span) - 1;
        n += __builtin_popcountll(w);
        i += span;
    }
    return n;
}

/* pk:445-466: k-th set bit strictly after pos, below hard; -2 if none. */
static int64_t select_after(const uint64_t *bv, int64_t pos, int64_t k, int64_t hard) {
    int64_t i = pos + 1 < 0 ? 0 : pos + 1;
    while (i < hard) {
        uint64_t w = bv[i >> 6] >> (i & 63);
        int64_t c = __builtin_popcountll(w);
        if (c >= k) {
            for (;;) {
                if (--k == 0) return i + __builtin_ctzll(w);
                w &= w - 1;
            }
        }
        k -= c;
        i = (i | 63) + 1;
    }
    return -2;
}

/* pk:469-482 */
static int64_t run_end_local(gqf_t *G, int64_t x, int64_t hard) {
    int64_t h = x >> REG_BITS, s_h = h << REG_BITS;
    int64_t k = rank_range(G->occ, s_h, x + 1);
    int64_t base = s_h + G->offs[h] - 1;
    return k == 0 ? base : select_after(G->run, base, k, hard);
}

/* pk:485-495 */
static int64_t first_unused(gqf_t *G, int64_t pos, int64_t hard) {
    for (int64_t x = pos; x < hard;) {
        int64_t e = run_end_local(G, x, hard);
        if (e == -2) return -2;
        if (e < x) return x;
        x = e + 1;
    }
    return -2;
}

/* pk:498-505 */
static void move_up(gqf_t *G, int64_t a, int64_t b, int64_t L) {
    for (int64_t i = b - 1; i >= a; i--) putw(G->slots, G->wb, i + L, getw(G->slots, G->wb, i));
    for (int64_t i = b - 1; i >= a; i--) bit_put(G->run, i + L, bit_get(G->run, i));
    int64_t stop = a + L < b + L ? a + L : b + L;
    for (int64_t i = a; i < stop; i++) bit_put(G->run, i, 0);
}

/* pk:508-533: returns slots moved (>=0) and *far, or -1 when no room below hard. */
static int64_t make_room(gqf_t *G, int64_t pos, int64_t L, int64_t hard, int64_t *far) {
    if (L > GAP_CAP) return -1;
    int64_t x = pos;
    for (int64_t t = 0; t < L; t++) {
        int64_t e = first_unused(G, x, hard);
        if (e < 0) return -1;
        G->scratch[t] = e;
        x = e + 1;
    }
    int64_t moved = 0;
    for (int64_t k = L; k >= 1; k--) {
        int64_t a = (k >= 2 ? G->scratch[k - 2] : pos - 1) + 1, b = G->scratch[k - 1];
        if (b > a) {
            move_up(G, a, b, L - k + 1);
            moved += b - a;
        }
    }
    *far = G->scratch[L - 1];
    return moved;
}

/* pk:536-549 */
static int run_interval(gqf_t *G, int64_t quot, int64_t *s, int64_t *e) {
    int64_t h = quot >> REG_BITS;
    int64_t hard = (h + 2) << REG_BITS;
    if (hard > G->phys) hard = G->phys;
    if (!bit_get(G->occ, quot)) { *s = *e = -1; return 0; }
    int64_t s_h = h << REG_BITS;
    int64_t k = rank_range(G->occ, s_h, quot + 1);
    int64_t base = s_h + G->offs[h] - 1;
    int64_t prev = k == 1 ? base : select_after(G->run, base, k - 1, hard);
    int64_t end = select_after(G->run, base, k, hard);
    if (prev == -2 || end == -2) return RC_INVARIANT;
    *s = quot > prev + 1 ? quot : prev + 1;
    *e = end;
    return 0;
}

/* countgroups.py:69-102 */
static int group_at(gqf_t *G, int64_t i, int64_t end, uint64_t *rem, uint64_t *cnt, int64_t *nx) {
    uint64_t h = getw(G->slots, G->wb, i);
    if (h == 0) {
        int64_t j = i;
        while (j <= end && getw(G->slots, G->wb, j) == 0) j++;
        *rem = 0; *cnt = (uint64_t)(j - i); *nx = j;
        return 0;
    }
    if (i == end) { *rem = h; *cnt = 1; *nx = i + 1; return 0; }
    uint64_t v = getw(G->slots, G->wb, i + 1);
    if (v > h) { *rem = h; *cnt = 1; *nx = i + 1; return 0; }
    if (v == h) { *rem = h; *cnt = 2; *nx = i + 2; return 0; }
    uint64_t base = G->r >= 64 ? ~0ULL : ((1ULL << G->r) - 1);
    uint64_t rest = 0, scale = 1;
    int64_t j = i + 2;
    for (;;) {
        if (j > end) return RC_INVARIANT;
        uint64_t d = getw(G->slots, G->wb, j);
        if (d == h) break;
        rest += scale * (d > h ? d - 1 : d);
        scale *= base;
        j++;
    }
    *rem = h; *cnt = v + h * rest + 2; *nx = j + 1;
    return 0;
}

/* pk:552-566 */
static int find_group(gqf_t *G, int64_t start, int64_t end, uint64_t rem, int64_t *gs, int64_t *ge,
                      uint64_t *c, int64_t *sp) {
    *gs = *ge = *sp = -1;
    *c = 0;
    for (int64_t i = start; i <= end;) {
        uint64_t h, cnt;
        int64_t nx;
        if (group_at(G, i, end, &h, &cnt, &nx)) return RC_INVARIANT;
        if (h == rem) { *gs = i; *ge = nx - 1; *c = cnt; return 0; }
        if (h > rem) { *sp = i; return 0; }
        i = nx;
    }
    *sp = end + 1;
    return 0;
}

/* pk:569-576 */
static int refresh_offset(gqf_t *G, int64_t h) {
    int64_t b = h << REG_BITS;
    int64_t hard = (h + 1) << REG_BITS;
    if (hard > G->phys) hard = G->phys;
    int64_t e = run_end_local(G, b - 1, hard);
    if (e == -2) return RC_INVARIANT;
    G->offs[h] = (int32_t)(e - b + 1 > 0 ? e - b + 1 : 0);
    return 0;
}

/* countgroups.py:54-66 */
int64_t orc_encoded_length(uint64_t rem, uint64_t count, int r) {
    if (rem == 0) return (int64_t)count;
    if (count <= 2) return (int64_t)count;
    uint64_t base = r >= 64 ? ~0ULL : ((1ULL << r) - 1);
    uint64_t v = (count - 2) / rem;
    int64_t n = 3;
    while (v) { n++; v /= base; }
    return n;
}

/* countgroups.py:28-51 */
static void write_group(gqf_t *G, int64_t pos, uint64_t rem, uint64_t count) {
    if (rem == 0) {
        for (uint64_t i = 0; i < count; i++) putw(G->slots, G->wb, pos + (int64_t)i, 0);
        return;
    }
    putw(G->slots, G->wb, pos, rem);
    if (count == 1) return;
    if (count == 2) { putw(G->slots, G->wb, pos + 1, rem); return; }
    uint64_t v = count - 2, base = G->r >= 64 ? ~0ULL : ((1ULL << G->r) - 1);
    putw(G->slots, G->wb, pos + 1, v % rem);
    v /= rem;
    int64_t i = pos + 2;
    while (v) {
        uint64_t d = v % base;
        v /= base;
        putw(G->slots, G->wb, i++, d >= rem ? d + 1 : d);
    }
    putw(G->slots, G->wb, i, rem);
}

/* pk:584-656: returns 0 / 1 (LOAD) / 2 (SHIFT) / -9. */
static int insert_one(gqf_t *G, int64_t max_occ, uint64_t fp, uint64_t delta, int64_t *moved_out) {
    uint64_t rmask = G->r >= 64 ? ~0ULL : ((1ULL << G->r) - 1);
    int64_t quot = (int64_t)(G->r >= 64 ? 0 : fp >> G->r);
    uint64_t rem = fp & rmask;
    int64_t g = quot >> REG_BITS;
    int64_t hard = (g + 2) << REG_BITS;
    if (hard > G->phys) hard = G->phys;
    int64_t moved = 0, far = 0, touched = 0;
    *moved_out = 0;
    if (G->stats[0] >= max_occ) return 1;
    if (!bit_get(G->occ, quot)) {
        int64_t e = run_end_local(G, quot, hard);
        if (e == -2) return 2;
        int64_t pos = quot > e + 1 ? quot : e + 1;
        int64_t L = orc_encoded_length(rem, delta, G->r);
        moved = make_room(G, pos, L, hard, &far);
        if (moved < 0) return 2;
        write_group(G, pos, rem, delta);
        bit_put(G->occ, quot, 1);
        bit_put(G->run, pos + L - 1, 1);
        touched = far + 1;
        G->stats[0] += L; G->stats[1] += (int64_t)delta; G->stats[2] += 1;
    } else {
        int64_t s, e, gs, ge, sp;
        uint64_t c;
        if (run_interval(G, quot, &s, &e)) return RC_INVARIANT;
        if (find_group(G, s, e, rem, &gs, &ge, &c, &sp)) return RC_INVARIANT;
        if (gs >= 0) {
            int64_t L = orc_encoded_length(rem, c + delta, G->r);
            int64_t diff = L - (ge - gs + 1);
            if (diff > 0) {
                moved = make_room(G, ge + 1, diff, hard, &far);
                if (moved < 0) return 2;
                if (ge == e) { bit_put(G->run, e, 0); bit_put(G->run, e + diff, 1); }
                touched = far + 1;
            }
            write_group(G, gs, rem, c + delta);
            G->stats[0] += diff; G->stats[1] += (int64_t)delta;
        } else {
            int64_t L = orc_encoded_length(rem, delta, G->r);
            moved = make_room(G, sp, L, hard, &far);
            if (moved < 0) return 2;
            write_group(G, sp, rem, delta);
            if (sp == e + 1) { bit_put(G->run, e, 0); bit_put(G->run, e + L, 1); }
            touched = far + 1;
            G->stats[0] += L; G->stats[1] += (int64_t)delta; G->stats[2] += 1;
        }
    }
    int64_t boundary = (g + 1) << REG_BITS;
    if (boundary < G->phys && touched > boundary)
        if (refresh_offset(G, g + 1)) return RC_INVARIANT;
    *moved_out = moved;
    return 0;
}

/* pk:659-715: delete [rs, re] from quot's run and left-compact the cluster. */
static int drop_slots(gqf_t *G, int64_t quot, int64_t start, int64_t end, int64_t rs, int64_t re,
                      int64_t hard, int64_t *moved_out, int64_t *last_out) {
    int64_t L = re - rs + 1;
    int emptied = L == end - start + 1;
    int64_t moved = 0, tail = end - re;
    for (int64_t i = 0; i < tail; i++) putw(G->slots, G->wb, rs + i, getw(G->slots, G->wb, re + 1 + i));
    moved += tail;
    bit_put(G->run, end, 0);
    int64_t wpos;
    if (emptied) { bit_put(G->occ, quot, 0); wpos = start; }
    else { bit_put(G->run, end - L, 1); wpos = end - L + 1; }
    int64_t prev_old_end = end, last_old_end = end, nq = quot;
    for (;;) {
        nq = select_after(G->occ, nq, 1, hard);
        if (nq < 0 || nq > prev_old_end + 1) break;
        int64_t s2 = prev_old_end + 1;
        int64_t e2 = select_after(G->run, s2 - 1, 1, hard);
        if (e2 == -2) return RC_INVARIANT;
        int64_t ns2 = nq > wpos ? nq : wpos;
        if (ns2 == s2) break;
        for (int64_t i = wpos; i < ns2; i++) { putw(G->slots, G->wb, i, 0); bit_put(G->run, i, 0); }
        int64_t n2 = e2 - s2 + 1;
        for (int64_t i = 0; i < n2; i++) putw(G->slots, G->wb, ns2 + i, getw(G->slots, G->wb, s2 + i));
        bit_put(G->run, e2, 0);
        bit_put(G->run, ns2 + n2 - 1, 1);
        moved += n2;
        wpos = ns2 + n2;
        prev_old_end = e2;
        last_old_end = e2;
    }
    for (int64_t i = wpos; i <= last_old_end; i++) { putw(G->slots, G->wb, i, 0); bit_put(G->run, i, 0); }
    *moved_out = moved;
    *last_out = last_old_end;
    return 0;
}

/* pk:718-755 */
static int delete_one(gqf_t *G, uint64_t fp, uint64_t delta, int *found, int64_t *moved_out) {
    uint64_t rmask = G->r >= 64 ? ~0ULL : ((1ULL << G->r) - 1);
    int64_t quot = (int64_t)(G->r >= 64 ? 0 : fp >> G->r);
    uint64_t rem = fp & rmask;
    int64_t g = quot >> REG_BITS;
    int64_t hard = (g + 2) << REG_BITS;
    if (hard > G->phys) hard = G->phys;
    *found = 0;
    *moved_out = 0;
    if (!bit_get(G->occ, quot)) return 0;
    int64_t s, e, gs, ge, sp, rs, re;
    uint64_t c;
    if (run_interval(G, quot, &s, &e)) return RC_INVARIANT;
    if (find_group(G, s, e, rem, &gs, &ge, &c, &sp)) return RC_INVARIANT;
    if (gs < 0) return 0;
    uint64_t take = delta < c ? delta : c, c2 = c - take;
    if (c2 > 0) {
        int64_t L2 = orc_encoded_length(rem, c2, G->r);
        int64_t diff = (ge - gs + 1) - L2;
        write_group(G, gs, rem, c2);
        G->stats[1] -= (int64_t)take;
        if (diff == 0) { *found = 1; return 0; }
        rs = gs + L2;
        re = ge;
    } else {
        G->stats[1] -= (int64_t)take;
        G->stats[2] -= 1;
        rs = gs;
        re = ge;
    }
    int64_t moved, last;
    if (drop_slots(G, quot, s, e, rs, re, hard, &moved, &last)) return RC_INVARIANT;
    G->stats[0] -= re - rs + 1;
    int64_t boundary = (g + 1) << REG_BITS;
    if (boundary < G->phys && last >= boundary)
        if (refresh_offset(G, g + 1)) return RC_INVARIANT;
    *found = 1;
    *moved_out = moved;
    return 0;
}

static int gqf_open(gqf_t *G, void *slots, int wb, uint64_t *occ, uint64_t *run, int32_t *offs,
                    int64_t *stats, int64_t phys, int q, int r) {
    G->slots = slots; G->wb = wb; G->occ = occ; G->run = run; G->offs = offs; G->stats = stats;
    G->phys = phys; G->q = q; G->r = r;
    G->scratch = (int64_t *)malloc(GAP_CAP * sizeof(int64_t));
    return G->scratch ? 0 : -1;
}

/* pk:772-801.  Returns code; *fail_idx = first failing index or -1. */
int orc_gqf_insert_batch(void *slots, int wb, uint64_t *occ, uint64_t *run, int32_t *offs, int64_t *stats,
                         int64_t phys, int q, int r, int64_t max_occ, const uint64_t *fps,
                         const uint64_t *deltas, int64_t n, int64_t *shift_out, int64_t *fail_idx) {
    gqf_t G;
    if (gqf_open(&G, slots, wb, occ, run, offs, stats, phys, q, r)) return -1;
    int64_t total = 0;
    int code = 0;
    *fail_idx = -1;
    for (int64_t k = 0; k < n; k++) {
        int64_t mv;
        code = insert_one(&G, max_occ, fps[k], deltas ? deltas[k] : 1, &mv);
        if (code) { *fail_idx = k; break; }
        total += mv;
    }
    free(G.scratch);
    if (shift_out) *shift_out += total;
    return code;
}

/* pk:804-824 */
int orc_gqf_count_batch(void *slots, int wb, uint64_t *occ, uint64_t *run, int32_t *offs, int64_t phys,
                        int q, int r, const uint64_t *fps, int64_t n, uint64_t *counts) {
    gqf_t G;
    G.slots = slots; G.wb = wb; G.occ = occ; G.run = run; G.offs = offs; G.stats = NULL;
    G.phys = phys; G.q = q; G.r = r; G.scratch = NULL;
    uint64_t rmask = r >= 64 ? ~0ULL : ((1ULL << r) - 1);
    for (int64_t k = 0; k < n; k++) {
        int64_t quot = (int64_t)(fps[k] >> r);
        counts[k] = 0;
        if (!bit_get(occ, quot)) continue;
        int64_t s, e, gs, ge, sp;
        uint64_t c;
        if (run_interval(&G, quot, &s, &e)) return RC_INVARIANT;
        if (find_group(&G, s, e, fps[k] & rmask, &gs, &ge, &c, &sp)) return RC_INVARIANT;
        counts[k] = gs >= 0 ? c : 0;
    }
    return 0;
}

/* pk:827-847 */
int orc_gqf_delete_batch(void *slots, int wb, uint64_t *occ, uint64_t *run, int32_t *offs, int64_t *stats,
                         int64_t phys, int q, int r, const uint64_t *fps, const uint64_t *deltas, int64_t n,
                         uint8_t *found, int64_t *shift_out) {
    gqf_t G;
    if (gqf_open(&G, slots, wb, occ, run, offs, stats, phys, q, r)) return -1;
    int64_t total = 0;
    int code = 0;
    for (int64_t k = 0; k < n; k++) {
        int ok;
        int64_t mv;
        code = delete_one(&G, fps[k], deltas ? deltas[k] : (1ULL << 63), &ok, &mv);
        if (code) break;
        found[k] = (uint8_t)ok;
        total += mv;
    }
    free(G.scratch);
    if (shift_out) *shift_out += total;
    return code;
}

/* pk:536-549 */
int orc_gqf_find_run(uint64_t *occ, uint64_t *run, int32_t *offs, int64_t phys, int64_t quot,
                     int64_t *s, int64_t *e) {
    gqf_t G;
    G.occ = occ; G.run = run; G.offs = offs; G.phys = phys;
    return run_interval(&G, quot, s, e);
}
