/* lshbeam_oracle.h -- plain-C restatement of the reference LSH beam-search
 * hot path (arXiv 1806.00588 artifact, /root/reference/proj).
 *
 * TEST INFRASTRUCTURE ONLY: the checker that tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg compare the CUDA product against. The
 * product (paper_1806_00588_b200/) never links or calls it.
 *
 * Parity is pinned two ways (tests/test_oracle_pinning.py):
 *   1. against the reference's own known-answer tests (tests/golden/), and
 *   2. against the real reference compiled in place (oracle/_ref).
 *
 * Status codes: 0 ok, 1 invalid argument (reference: std::invalid_argument),
 * 2 runtime error (reference: std::runtime_error).
 */
#ifndef LSHBEAM_ORACLE_H
#define LSHBEAM_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (include/lshbeam/rng.hpp:11-52) ---- */
uint64_t lso_sm64_next(uint64_t* state);
uint64_t lso_sm64_bounded(uint64_t* state, uint64_t bound);
double lso_sm64_gaussian(uint64_t* state);
uint64_t lso_mix_seed(uint64_t seed, uint64_t stream);
/* Gaussian floats of the stream SplitMix64(seed) starting after `skip_gauss`
 * gaussians (each consumes exactly two draws), times `scale`. Parallel via
 * jump-ahead; identical to the sequential stream. */
void lso_gaussian_fill(uint64_t seed, uint64_t skip_gauss, float* out, size_t n, float scale);

/* ---- WTA hash (src/wta_hash.cpp) ---- */
int lso_bits_for(int K);
int lso_wta_params_check(int K, int u, int W);
int lso_generate_perms(int d, int P, int K, uint64_t seed, uint32_t* out);
int lso_hash_matrix(const float* M, int64_t n, int d, const uint32_t* perms, int K,
                    int u, int W, uint32_t* out);

/* ---- Band index + cuckoo (src/band_index.cpp) ----
 * slots: per band, 2*2^lg (key,start,len) triples, band w at
 * slots + w*slot_stride_u32. */
uint32_t lso_lg_max(uint32_t V);
int lso_cuckoo_build(const uint32_t* keys, const uint32_t* starts, const uint32_t* lens,
                     size_t n, uint64_t seed, uint32_t* lg, uint64_t* mul2,
                     uint32_t* slots);
int lso_cuckoo_find(uint32_t lg, const uint64_t* mul2, const uint32_t* slots,
                    uint32_t key, uint32_t* start, uint32_t* len, int* probes);
int lso_band_index_build(const uint32_t* codes, uint32_t V, int W, uint64_t seed,
                         uint32_t* word_ids, uint32_t* lg, uint64_t* mul,
                         uint32_t* slots, size_t slot_stride_u32);
int lso_lookup_hits(const uint32_t* word_ids, uint32_t V, int W, const uint32_t* lg,
                    const uint64_t* mul, const uint32_t* slots, size_t slot_stride_u32,
                    const uint32_t* q, int B, int32_t* L);
int lso_lookup_hits_bruteforce(const uint32_t* vocab_codes, uint32_t V,
                               const uint32_t* q, int B, int W, int32_t* L);

/* ---- Candidates (src/candidate_selector.cpp) ---- */
int lso_select_candidates(const int32_t* L, int B, uint32_t V, int t, uint32_t* ids,
                          uint32_t* n, uint32_t* from_threshold);
int lso_merge_top_frequent(const uint32_t* ids, uint32_t n, uint32_t from_thr,
                           uint32_t T, const uint32_t* specials, uint32_t nspec,
                           uint32_t V, uint32_t* out, uint32_t* nout, uint32_t* prov);
void lso_gather(const float* E, int d, const uint32_t* ids, uint32_t n, float* out);

/* ---- Reduced softmax + expansion (src/beam_decoder.cpp) ---- */
float lso_dot_ref_order(const float* h, const float* e, int64_t d);
void lso_compute_logits(const float* H, int rows, const float* Esub, int64_t n,
                        int64_t d, float* out);
void lso_compute_logits_ids(const float* H, int rows, const float* E, const uint32_t* ids,
                            int64_t n, int64_t d, const float* bias, float* out);
int lso_softmax_rows(const float* logits, int rows, int64_t n, float* out);
int lso_expand_beams(const float* probs, int rows, int64_t n, const double* cum,
                     const uint32_t* live, const double* fz_score,
                     const uint32_t* fz_beam, int nfrozen, int B,
                     const uint32_t* id_map, double* out_score, uint32_t* out_beam,
                     int64_t* out_word, int* nout);

/* ---- Model + oracle metrics (src/model_provider.cpp, src/eval_oracle.cpp) ---- */
int lso_synth_model(uint32_t V, int d, uint64_t seed, float bias_strength, float* E,
                    float* wh, float* we, float* h0, float* fbias);
int lso_step_hidden(const float* E, const float* wh, const float* we, uint32_t V, int d,
                    const float* h, uint32_t token, float* out);
int lso_exact_topb_logits(const float* logits, int rows, int64_t n, int b,
                          uint32_t* ids, float* vals);
double lso_recall_at_b(const uint32_t* cands, uint32_t ncand, const uint32_t* exact_ids,
                       int rows, int b);

#ifdef __cplusplus
}
#endif
#endif
