/* lshbeam_oracle.c -- plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see lshbeam_oracle.h). Each function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj. Floating-point order is reproduced deliberately:
 * compile with -ffp-contract=off and without -ffast-math (oracle/Makefile).
 */
#define _GNU_SOURCE
#include "lshbeam_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define LSO_OK 0
#define LSO_EINVAL 1
#define LSO_ERUNTIME 2

static const uint32_t kEmptyCode = 0x7FFFFFFFu; /* include/lshbeam/wta_hash.hpp:13 */
static const uint64_t kGamma = 0x9E3779B97F4A7C15ull;

/* ------------------------------------------------------------------ RNG */

/* SplitMix64::next, include/lshbeam/rng.hpp:15-20 */
uint64_t lso_sm64_next(uint64_t* s) {
  uint64_t z = (*s += kGamma);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* SplitMix64::bounded, rng.hpp:24-29 (rejection below the largest multiple) */
uint64_t lso_sm64_bounded(uint64_t* s, uint64_t bound) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t x = lso_sm64_next(s);
  while (x >= limit) x = lso_sm64_next(s);
  return x % bound;
}

/* SplitMix64::gaussian, rng.hpp:36-40: Box-Muller cosine branch, two draws */
double lso_sm64_gaussian(uint64_t* s) {
  const double u1 = (double)((lso_sm64_next(s) >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(lso_sm64_next(s) >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* mix_seed, rng.hpp:49-52 */
uint64_t lso_mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t s = seed ^ (0xBF58476D1CE4E5B9ull * (stream + 1));
  return lso_sm64_next(&s);
}

/* fill_gaussian, src/model_provider.cpp:15-19. The state after k draws is
 * seed + k*gamma, so chunks can start anywhere in the stream. */
void lso_gaussian_fill(uint64_t seed, uint64_t skip_gauss, float* out, size_t n,
                       float scale) {
  const size_t chunk = 1u << 16;
  const int64_t nchunks = (int64_t)((n + chunk - 1) / chunk);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nchunks; ++c) {
    const size_t lo = (size_t)c * chunk;
    const size_t hi = lo + chunk < n ? lo + chunk : n;
    uint64_t s = seed + 2ull * (skip_gauss + lo) * kGamma;
    for (size_t i = lo; i < hi; ++i) out[i] = (float)lso_sm64_gaussian(&s) * scale;
  }
}

/* ------------------------------------------------------------- WTA hash */

/* WtaParams::bits_for, src/wta_hash.cpp:12-16 */
int lso_bits_for(int K) {
  int bits = 0;
  while ((1 << bits) < K) ++bits;
  return bits;
}

/* WtaParams ctor validation, src/wta_hash.cpp:18-29 */
int lso_wta_params_check(int K, int u, int W) {
  if (K < 2 || u < 1 || W < 1) return LSO_EINVAL;
  if (u * lso_bits_for(K) >= 31) return LSO_EINVAL;
  return LSO_OK;
}

/* PermutationSet::generate, src/wta_hash.cpp:31-55: per row a fresh iota of
 * [0,d), K Fisher-Yates steps from ONE stream, keep the prefix. */
int lso_generate_perms(int d, int P, int K, uint64_t seed, uint32_t* out) {
  if (K < 1 || d < K) return LSO_EINVAL;
  uint32_t* scratch = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)d);
  uint64_t s = seed;
  for (int p = 0; p < P; ++p) {
    for (int i = 0; i < d; ++i) scratch[i] = (uint32_t)i;
    for (int k = 0; k < K; ++k) {
      const uint64_t j = (uint64_t)k + lso_sm64_bounded(&s, (uint64_t)(d - k));
      const uint32_t t = scratch[k];
      scratch[k] = scratch[j];
      scratch[j] = t;
      out[(size_t)p * K + k] = scratch[k];
    }
  }
  free(scratch);
  return LSO_OK;
}

/* hash_matrix = NaN scan + hash_into + pack_into, src/wta_hash.cpp:75-116,
 * :147-171. argmax uses strict '>' so ties go to the smallest k (:85). */
int lso_hash_matrix(const float* M, int64_t n, int d, const uint32_t* perms, int K,
                    int u, int W, uint32_t* out) {
  if (lso_wta_params_check(K, u, W)) return LSO_EINVAL;
  const int bits = lso_bits_for(K);
  int nan_seen = 0;
#pragma omp parallel for schedule(static) reduction(| : nan_seen)
  for (int64_t i = 0; i < n; ++i) {
    const float* v = M + i * (int64_t)d;
    int bad = 0;
    for (int c = 0; c < d; ++c) bad |= isnan(v[c]) ? 1 : 0;
    if (bad) {
      nan_seen = 1;
      continue;
    }
    for (int w = 0; w < W; ++w) {
      uint32_t code = 0;
      for (int b = 0; b < u; ++b) {
        const uint32_t* row = perms + (size_t)(w * u + b) * K;
        uint32_t best = 0;
        float best_val = v[row[0]];
        for (int k = 1; k < K; ++k) {
          const float val = v[row[k]];
          if (val > best_val) {
            best_val = val;
            best = (uint32_t)k;
          }
        }
        code |= best << (b * bits);
      }
      out[i * W + w] = code;
    }
  }
  return nan_seen ? LSO_EINVAL : LSO_OK;
}

/* ------------------------------------------------------- cuckoo + bands */

/* next_pow2_log, src/band_index.cpp:14-18 */
static uint32_t next_pow2_log(size_t n) {
  uint32_t lg = 0;
  while (((size_t)1 << lg) < n) ++lg;
  return lg;
}

uint32_t lso_lg_max(uint32_t V) {
  const uint32_t lg = next_pow2_log(V);
  return lg < 1 ? 1 : lg;
}

/* CuckooTable::slot_of, include/lshbeam/band_index.hpp:61-64 */
static inline uint32_t slot_of(uint64_t mul, uint32_t lg, uint32_t key) {
  return (uint32_t)((mul * (uint64_t)key) >> (64 - lg));
}

/* CuckooTable::build, src/band_index.cpp:32-71: lg = max(1, ceil log2 n);
 * attempts 0..kMaxRebuilds(8) draw (next|1, next|1) from SplitMix64(seed);
 * each insert starts in table 0, swaps, evictee flips table, <=128 hops. */
int lso_cuckoo_build(const uint32_t* keys, const uint32_t* starts, const uint32_t* lens,
                     size_t n, uint64_t seed, uint32_t* lg_out, uint64_t* mul2,
                     uint32_t* slots) {
  for (size_t i = 0; i < n; ++i)
    if (keys[i] >= kEmptyCode) return LSO_EINVAL;
  uint32_t lg = next_pow2_log(n);
  if (lg < 1) lg = 1;
  const uint32_t cap = 1u << lg;
  uint64_t g = seed;
  for (int attempt = 0; attempt <= 8; ++attempt) {
    mul2[0] = lso_sm64_next(&g) | 1;
    mul2[1] = lso_sm64_next(&g) | 1;
    for (uint32_t s = 0; s < 2 * cap; ++s) {
      slots[3 * s] = kEmptyCode;
      slots[3 * s + 1] = 0;
      slots[3 * s + 2] = 0;
    }
    int ok = 1;
    for (size_t e = 0; e < n && ok; ++e) {
      uint32_t cur[3] = {keys[e], starts[e], lens[e]};
      int table = 0, placed = 0;
      for (int hop = 0; hop < 128; ++hop) {
        uint32_t* s = slots + 3 * ((size_t)table * cap + slot_of(mul2[table], lg, cur[0]));
        for (int f = 0; f < 3; ++f) {
          const uint32_t t = s[f];
          s[f] = cur[f];
          cur[f] = t;
        }
        if (cur[0] == kEmptyCode) {
          placed = 1;
          break;
        }
        table = 1 - table;
      }
      ok = placed;
    }
    if (ok) {
      *lg_out = lg;
      return LSO_OK;
    }
  }
  return LSO_ERUNTIME;
}

/* CuckooTable::find_counted, src/band_index.cpp:73-83 */
int lso_cuckoo_find(uint32_t lg, const uint64_t* mul2, const uint32_t* slots,
                    uint32_t key, uint32_t* start, uint32_t* len, int* probes) {
  const uint32_t cap = 1u << lg;
  const uint32_t* s0 = slots + 3 * (size_t)slot_of(mul2[0], lg, key);
  *probes = 1;
  if (s0[0] == key) {
    *start = s0[1];
    *len = s0[2];
    return 1;
  }
  const uint32_t* s1 = slots + 3 * ((size_t)cap + slot_of(mul2[1], lg, key));
  *probes = 2;
  if (s1[0] == key) {
    *start = s1[1];
    *len = s1[2];
    return 1;
  }
  return 0;
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* BandIndex::build, src/band_index.cpp:90-132: per band sort (code<<32|id),
 * word ids band-major, one span per distinct code, table seed mix_seed(seed,w). */
int lso_band_index_build(const uint32_t* codes, uint32_t V, int W, uint64_t seed,
                         uint32_t* word_ids, uint32_t* lg, uint64_t* mul,
                         uint32_t* slots, size_t slot_stride_u32) {
  int failed = 0, bad = 0;
#pragma omp parallel
  {
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (V ? V : 1));
    uint32_t* ek = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
    uint32_t* es = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
    uint32_t* el = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
#pragma omp for schedule(dynamic)
    for (int w = 0; w < W; ++w) {
      for (uint32_t j = 0; j < V; ++j)
        keys[j] = ((uint64_t)codes[(size_t)j * W + w] << 32) | j;
      qsort(keys, V, sizeof(uint64_t), cmp_u64);
      uint32_t* ids = word_ids + (size_t)w * V;
      size_t ne = 0;
      for (uint32_t pos = 0; pos < V; ++pos) {
        const uint32_t code = (uint32_t)(keys[pos] >> 32);
        ids[pos] = (uint32_t)keys[pos];
        if (pos == 0 || code != (uint32_t)(keys[pos - 1] >> 32)) {
          ek[ne] = code;
          es[ne] = pos;
          el[ne] = 1;
          ++ne;
        } else {
          el[ne - 1]++;
        }
      }
      const int rc = lso_cuckoo_build(ek, es, el, ne, lso_mix_seed(seed, (uint64_t)w),
                                      lg + w, mul + 2 * w, slots + (size_t)w * slot_stride_u32);
      if (rc == LSO_ERUNTIME) {
#pragma omp atomic write
        failed = 1;
      } else if (rc) {
#pragma omp atomic write
        bad = 1;
      }
    }
    free(keys);
    free(ek);
    free(es);
    free(el);
  }
  if (bad) return LSO_EINVAL;
  return failed ? LSO_ERUNTIME : LSO_OK;
}

/* BandIndex::lookup_hits_into, src/band_index.cpp:134-162 */
int lso_lookup_hits(const uint32_t* word_ids, uint32_t V, int W, const uint32_t* lg,
                    const uint64_t* mul, const uint32_t* slots, size_t slot_stride_u32,
                    const uint32_t* q, int B, int32_t* L) {
  memset(L, 0, sizeof(int32_t) * (size_t)B * V);
  for (int i = 0; i < B; ++i) {
    int32_t* row = L + (size_t)i * V;
    for (int w = 0; w < W; ++w) {
      uint32_t start, len;
      int probes;
      if (!lso_cuckoo_find(lg[w], mul + 2 * w, slots + (size_t)w * slot_stride_u32,
                           q[(size_t)i * W + w], &start, &len, &probes))
        continue;
      const uint32_t* ids = word_ids + (size_t)w * V + start;
      for (uint32_t k = 0; k < len; ++k) row[ids[k]]++;
    }
  }
  return LSO_OK;
}

/* ref::lookup_hits, src/ref_kernels.cpp:19-36 (index-free brute force) */
int lso_lookup_hits_bruteforce(const uint32_t* vocab_codes, uint32_t V,
                               const uint32_t* q, int B, int W, int32_t* L) {
  for (int i = 0; i < B; ++i)
    for (uint32_t j = 0; j < V; ++j) {
      int32_t h = 0;
      for (int w = 0; w < W; ++w) h += q[(size_t)i * W + w] == vocab_codes[(size_t)j * W + w];
      L[(size_t)i * V + j] = h;
    }
  return LSO_OK;
}

/* ----------------------------------------------------------- candidates */

/* select_candidates, src/candidate_selector.cpp:14-55 */
int lso_select_candidates(const int32_t* L, int B, uint32_t V, int t, uint32_t* ids,
                          uint32_t* n, uint32_t* from_threshold) {
  if (t < 0) return LSO_EINVAL;
  uint32_t cnt = 0;
  for (uint32_t j = 0; j < V; ++j) {
    int keep = t == 0;
    for (int i = 0; i < B && !keep; ++i) keep = L[(size_t)i * V + j] >= t;
    if (keep) ids[cnt++] = j;
  }
  *n = cnt;
  *from_threshold = cnt;
  return LSO_OK;
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

/* merge_top_frequent, src/candidate_selector.cpp:57-103 (loop restated
 * literally, including the provenance counters). prov = {thr, top, specials}. */
int lso_merge_top_frequent(const uint32_t* ids, uint32_t n, uint32_t from_thr,
                           uint32_t T, const uint32_t* specials, uint32_t nspec,
                           uint32_t V, uint32_t* out, uint32_t* nout, uint32_t* prov) {
  if (T > V) return LSO_EINVAL;
  uint32_t* extra = (uint32_t*)malloc(sizeof(uint32_t) * (nspec ? nspec : 1));
  memcpy(extra, specials, sizeof(uint32_t) * nspec);
  qsort(extra, nspec, sizeof(uint32_t), cmp_u32);
  uint32_t ne = 0;
  for (uint32_t i = 0; i < nspec; ++i)
    if (ne == 0 || extra[ne - 1] != extra[i]) extra[ne++] = extra[i];
  for (uint32_t i = 0; i < ne; ++i)
    if (extra[i] >= V) {
      free(extra);
      return LSO_EINVAL;
    }
  uint32_t m = 0, ci = 0, seen_below = 0, from_specials = 0;
  for (; ci < n && ids[ci] < T; ++ci) ++seen_below;
  for (uint32_t id = 0; id < T; ++id) out[m++] = id;
  uint32_t si = 0;
  while (si < ne && extra[si] < T) ++si;
  while (ci < n || si < ne) {
    uint32_t next;
    int from_special = 0;
    if (si == ne || (ci < n && ids[ci] <= extra[si])) {
      next = ids[ci];
      if (si < ne && extra[si] == next) ++si;
      ++ci;
    } else {
      next = extra[si++];
      from_special = 1;
    }
    if (m > 0 && out[m - 1] == next) continue;
    out[m++] = next;
    if (from_special) ++from_specials;
  }
  *nout = m;
  prov[0] = from_thr;
  prov[1] = T - seen_below;
  prov[2] = from_specials;
  free(extra);
  return LSO_OK;
}

/* gather_embeddings, src/candidate_selector.cpp:105-119 */
void lso_gather(const float* E, int d, const uint32_t* ids, uint32_t n, float* out) {
  for (uint32_t r = 0; r < n; ++r)
    memcpy(out + (size_t)r * d, E + (size_t)ids[r] * d, sizeof(float) * (size_t)d);
}

/* ------------------------------------------------------ reduced softmax */

/* The dot product exactly as GCC 13 -O3 (x86-64 baseline, SSE, no FMA)
 * compiles the `omp simd reduction(+:acc)` loop of compute_logits
 * (src/beam_decoder.cpp:34-42): four lane accumulators, lane k sums
 * fl(h[c]*e[c]) for c = k mod 4 in ascending c over the first 4*floor(d/4)
 * columns; the d mod 4 tail is added into lane 0 in order; the result is
 * (((0 + l0) + l1) + l2) + l3. Pinned bit-exact against oracle/_ref. */
float lso_dot_ref_order(const float* h, const float* e, int64_t d) {
  volatile float lane[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  float l0 = 0.0f, l1 = 0.0f, l2 = 0.0f, l3 = 0.0f;
  const int64_t d4 = d >= 4 ? (d & ~(int64_t)3) : 0;
  for (int64_t c = 0; c < d4; c += 4) {
    l0 = l0 + h[c] * e[c];
    l1 = l1 + h[c + 1] * e[c + 1];
    l2 = l2 + h[c + 2] * e[c + 2];
    l3 = l3 + h[c + 3] * e[c + 3];
  }
  for (int64_t c = d4; c < d; ++c) l0 = h[c] * e[c] + l0;
  lane[0] = l0;
  lane[1] = l1;
  lane[2] = l2;
  lane[3] = l3;
  float acc = 0.0f;
  acc = acc + lane[0];
  acc = acc + lane[1];
  acc = acc + lane[2];
  acc = acc + lane[3];
  return acc;
}

/* compute_logits, src/beam_decoder.cpp:23-44 */
void lso_compute_logits(const float* H, int rows, const float* Esub, int64_t n,
                        int64_t d, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t ir = 0; ir < (int64_t)rows * n; ++ir)
    out[ir] = lso_dot_ref_order(H + (ir / n) * d, Esub + (ir % n) * d, d);
}

/* compute_logits over E[ids] plus the bias add of decode()
 * (src/beam_decoder.cpp:237-247): logit = dot + bias[id] in float. */
void lso_compute_logits_ids(const float* H, int rows, const float* E, const uint32_t* ids,
                            int64_t n, int64_t d, const float* bias, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t ir = 0; ir < (int64_t)rows * n; ++ir) {
    const uint32_t id = ids ? ids[ir % n] : (uint32_t)(ir % n);
    float v = lso_dot_ref_order(H + (ir / n) * d, E + (size_t)id * d, d);
    if (bias) v = v + bias[id];
    out[ir] = v;
  }
}

/* softmax_rows, src/beam_decoder.cpp:46-74: float max, exp in double,
 * sequential double denominator, float(1/denom) multiply. */
int lso_softmax_rows(const float* logits, int rows, int64_t n, float* out) {
  int empty_row = 0;
#pragma omp parallel for schedule(static) reduction(| : empty_row)
  for (int i = 0; i < rows; ++i) {
    const float* in = logits + (int64_t)i * n;
    float* o = out + (int64_t)i * n;
    float mx = -INFINITY;
    for (int64_t j = 0; j < n; ++j) mx = (mx < in[j]) ? in[j] : mx;
    if (n == 0 || (isinf(mx) && mx < 0)) {
      empty_row = 1;
      continue;
    }
    double denom = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const double e = exp((double)in[j] - (double)mx);
      o[j] = (float)e;
      denom += e;
    }
    const float inv = (float)(1.0 / denom);
    for (int64_t j = 0; j < n; ++j) o[j] = o[j] * inv;
  }
  return empty_row ? LSO_EINVAL : LSO_OK;
}

typedef struct {
  double score;
  uint32_t beam;
  int64_t word;
} lso_choice;

/* expand_beams comparator, src/beam_decoder.cpp:102-106 */
static int better_first(const void* a, const void* b) {
  const lso_choice* x = (const lso_choice*)a;
  const lso_choice* y = (const lso_choice*)b;
  if (x->score != y->score) return x->score > y->score ? -1 : 1;
  if (x->beam != y->beam) return x->beam < y->beam ? -1 : 1;
  return x->word < y->word ? -1 : (x->word > y->word);
}

/* expand_beams, src/beam_decoder.cpp:76-111. The comparator is a total
 * order on distinct (beam, word) pairs, so sorting the whole pool yields
 * the same top-B as partial_sort. */
int lso_expand_beams(const float* probs, int rows, int64_t n, const double* cum,
                     const uint32_t* live, const double* fz_score,
                     const uint32_t* fz_beam, int nfrozen, int B,
                     const uint32_t* id_map, double* out_score, uint32_t* out_beam,
                     int64_t* out_word, int* nout) {
  const size_t total = (size_t)rows * n + nfrozen;
  lso_choice* pool = (lso_choice*)malloc(sizeof(lso_choice) * (total ? total : 1));
  size_t m = 0;
  for (int f = 0; f < nfrozen; ++f) pool[m++] = (lso_choice){fz_score[f], fz_beam[f], -1};
  for (int i = 0; i < rows; ++i)
    for (int64_t r = 0; r < n; ++r)
      pool[m++] = (lso_choice){cum[i] + log((double)probs[(int64_t)i * n + r]), live[i],
                               id_map ? (int64_t)id_map[r] : r};
  qsort(pool, m, sizeof(lso_choice), better_first);
  const size_t keep = (size_t)B < m ? (size_t)B : m;
  for (size_t k = 0; k < keep; ++k) {
    out_score[k] = pool[k].score;
    out_beam[k] = pool[k].beam;
    out_word[k] = pool[k].word;
  }
  *nout = (int)keep;
  free(pool);
  return LSO_OK;
}

/* --------------------------------------------------------------- model */

/* synth_model + finish_model, src/model_provider.cpp:21-65: one stream,
 * E (V*d), then w_hidden, w_embed (scaled), h0 = tanhf(gauss), then the
 * mean-centred Zipf bias computed in double. Any output may be NULL (its
 * draws are still skipped). */
int lso_synth_model(uint32_t V, int d, uint64_t seed, float bias_strength, float* E,
                    float* wh, float* we, float* h0, float* fbias) {
  if (V < 2 || d < 1) return LSO_EINVAL;
  const uint64_t nE = (uint64_t)V * d, nW = (uint64_t)d * d;
  const float scale = 1.0f / sqrtf((float)d);
  if (E) lso_gaussian_fill(seed, 0, E, nE, 1.0f);
  if (wh) lso_gaussian_fill(seed, nE, wh, nW, scale);
  if (we) lso_gaussian_fill(seed, nE + nW, we, nW, 0.02f * scale);
  if (h0) {
    uint64_t s = seed + 2ull * (nE + 2 * nW) * kGamma;
    for (int i = 0; i < d; ++i) h0[i] = tanhf((float)lso_sm64_gaussian(&s));
  }
  if (fbias) {
    double sum = 0.0;
    for (uint32_t j = 0; j < V; ++j) sum += 1.0 / (1.0 + j);
    const double mean = sum / V;
    for (uint32_t j = 0; j < V; ++j)
      fbias[j] = (float)((double)bias_strength * (1.0 / (1.0 + j) - mean));
  }
  return LSO_OK;
}

/* step_hidden, src/model_provider.cpp:83-102, with the same 4-lane no-FMA
 * order as compute_logits; lane term fl(fl(wh*h) + fl(we*emb)). */
int lso_step_hidden(const float* E, const float* wh, const float* we, uint32_t V, int d,
                    const float* h, uint32_t token, float* out) {
  if (token >= V) return LSO_EINVAL;
  const float* emb = E + (size_t)token * d;
  const int d4 = d >= 4 ? (d & ~3) : 0;
  for (int r = 0; r < d; ++r) {
    const float* a = wh + (size_t)r * d;
    const float* b = we + (size_t)r * d;
    float l[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int c = 0; c < d4; c += 4)
      for (int k = 0; k < 4; ++k) {
        const float t = a[c + k] * h[c + k] + b[c + k] * emb[c + k];
        l[k] = l[k] + t;
      }
    for (int c = d4; c < d; ++c) {
      const float t = a[c] * h[c] + b[c] * emb[c];
      l[0] = t + l[0];
    }
    float acc = 0.0f;
    acc = acc + l[0];
    acc = acc + l[1];
    acc = acc + l[2];
    acc = acc + l[3];
    out[r] = tanhf(acc);
  }
  return LSO_OK;
}

/* --------------------------------------------------------- eval oracle */

static int topb_cmp(const void* a, const void* b, void* ctx) {
  const float* row = (const float*)ctx;
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  if (row[x] != row[y]) return row[x] > row[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}

/* exact_topb_logits, src/eval_oracle.cpp:11-40: value desc, smaller id */
int lso_exact_topb_logits(const float* logits, int rows, int64_t n, int b,
                          uint32_t* ids, float* vals) {
  if (b < 0 || b > n) return LSO_EINVAL;
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (int i = 0; i < rows; ++i) {
    const float* row = logits + (int64_t)i * n;
    for (int64_t j = 0; j < n; ++j) order[j] = (uint32_t)j;
    qsort_r(order, n, sizeof(uint32_t), topb_cmp, (void*)row);
    for (int k = 0; k < b; ++k) {
      ids[(size_t)i * b + k] = order[k];
      vals[(size_t)i * b + k] = row[order[k]];
    }
  }
  free(order);
  return LSO_OK;
}

/* recall_at_b, src/eval_oracle.cpp:46-63 (mean over rows of hit fraction) */
double lso_recall_at_b(const uint32_t* cands, uint32_t ncand, const uint32_t* exact_ids,
                       int rows, int b) {
  if (rows == 0) return 0.0;
  double total = 0.0;
  for (int i = 0; i < rows; ++i) {
    size_t hit = 0;
    for (int k = 0; k < b; ++k)
      if (bsearch(&exact_ids[(size_t)i * b + k], cands, ncand, sizeof(uint32_t), cmp_u32))
        ++hit;
    total += b == 0 ? 0.0 : (double)hit / b;
  }
  return total / rows;
}
