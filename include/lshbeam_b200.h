/* lshbeam_b200.h -- C ABI of the B200-native LSH beam-search hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch
 * types. Each entry point names the reference interface it replaces
 * (paths under /root/reference/proj). The C++ drop-in API in
 * include/lshbeam/*.hpp (namespace lshbeam) is a thin layer over these
 * calls, and INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Conventions
 *  - Every call returns an lsb_status; lsb_last_error() gives a
 *    thread-local message for the last failure on this thread.
 *  - "_host" buffers are host memory (pageable or pinned); "_dev" buffers are
 *    device pointers on the context's device. Stage entry points (section 3)
 *    take host buffers and synchronise, like the reference's by-value API.
 *    The fused step (section 4) is device-resident and asynchronous.
 *  - Errors map to the reference's exceptions: LSB_EINVAL ~
 *    std::invalid_argument, LSB_ERUNTIME ~ std::runtime_error.
 *  - Matrices are dense row-major, as lshbeam::Mat<T>
 *    (include/lshbeam/matrix.hpp:11-41); E is |V| x d
 *    (include/lshbeam/model_provider.hpp:27).
 */
#ifndef LSHBEAM_B200_H
#define LSHBEAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSB_ABI_VERSION 1

typedef enum lsb_status {
  LSB_OK = 0,
  LSB_EINVAL = 1,   /* bad shape / parameter / NaN input / sentinel key / T > V */
  LSB_ERUNTIME = 2, /* cuckoo rebuild budget exhausted, empty candidate set */
  LSB_ECUDA = 3,    /* CUDA runtime / launch failure */
  LSB_ENOMEM = 4    /* device or pinned allocation failed */
} lsb_status;

/* Reduced-softmax arithmetic.
 *  PARITY: FP32 multiplies and adds in the reference's exact order (4 SSE
 *          lanes, no FMA; src/beam_decoder.cpp:34-42 as compiled by GCC -O3),
 *          so logits, probabilities and chosen ids are bit-identical to the
 *          CPU reference.
 *  FAST:   tcgen05 tensor cores (3xTF32, fp32 accumulation) for the dense
 *          part -- the top-T block shared by >= 256 rows, or the whole
 *          vocabulary -- and paired FP32 FFMA for the rest;
 *          |dlogit| <= 1e-4 (1+|l|), ids exact except at near-ties. */
typedef enum lsb_mode { LSB_MODE_PARITY = 0, LSB_MODE_FAST = 1 } lsb_mode;

/* One beam continuation, layout-compatible with lshbeam::BeamChoice
 * (include/lshbeam/beam_decoder.hpp:22-26): score, source hypothesis, word
 * (-1 = frozen hypothesis carried over). */
typedef struct lsb_choice {
  double score;
  uint32_t beam;
  uint32_t _pad;
  int64_t word;
} lsb_choice;

typedef struct lsb_ctx lsb_ctx;     /* device + CUDA stream + error word  */
typedef struct lsb_model lsb_model; /* device E (|V| x d fp32) + logit bias */
typedef struct lsb_index lsb_index; /* device WTA perms + band index       */
typedef struct lsb_batch lsb_batch; /* per-step scratch for S sentences   */

/* ------------------------------------------------------------ 1. context */
const char* lsb_last_error(void);
int lsb_abi_version(void);
/* stream: a cudaStream_t on `device`, LSB_STREAM_LEGACY for the legacy
 * default stream (cudaStreamLegacy), or NULL to create a private
 * non-blocking stream (which does NOT synchronise with the default stream). */
#define LSB_STREAM_LEGACY ((void*)0x1)
lsb_status lsb_ctx_create(int device, void* stream, lsb_ctx** out);
lsb_status lsb_ctx_destroy(lsb_ctx* ctx);
lsb_status lsb_ctx_sync(lsb_ctx* ctx);       /* sync + surface device errors */
void* lsb_ctx_stream(lsb_ctx* ctx);          /* the cudaStream_t in use      */
int lsb_ctx_device(lsb_ctx* ctx);
int lsb_ctx_sm_count(lsb_ctx* ctx);
/* Number of kernels this context has launched (for launch accounting). */
uint64_t lsb_ctx_launch_count(lsb_ctx* ctx);

/* -------------------------------------------------------------- 2. model
 * Replaces holding SynthModel::embeddings / freq_bias in host memory
 * (include/lshbeam/model_provider.hpp:21-32). E_host/bias_host are copied;
 * bias_host may be NULL (all zero). */
lsb_status lsb_model_create(lsb_ctx* ctx, const float* E_host, uint32_t vocab, int dim,
                            const float* bias_host, lsb_model** out);
/* Same, from device memory already on the context's device (copied). */
lsb_status lsb_model_create_dev(lsb_ctx* ctx, const float* E_dev, uint32_t vocab, int dim,
                                const float* bias_dev, lsb_model** out);
lsb_status lsb_model_destroy(lsb_model* m);
const float* lsb_model_embeddings_dev(const lsb_model* m);
uint32_t lsb_model_vocab(const lsb_model* m);
int lsb_model_dim(const lsb_model* m);

/* -------------------------------------------------------------- 3. index */

/* Replaces build_lsh_index(E, WtaParams{K,u,W,perm_seed}, index_seed)
 * (src/band_index.cpp:189-196): permutations on the host (bit-exact
 * SplitMix64 Fisher-Yates, src/wta_hash.cpp:31-55), WTA hash of E (K1), then
 * per band the stable (code, id) sort, spans and the parallel cuckoo build
 * (K2-build). LSB_EINVAL on bad {K,u,W} or NaN in E; LSB_ERUNTIME if a
 * band's cuckoo build exhausts the rebuild budget. */
lsb_status lsb_index_build(lsb_ctx* ctx, const lsb_model* model, int K, int u, int W,
                           uint64_t perm_seed, uint64_t index_seed, lsb_index** out);
/* Replaces BandIndex::build(band_codes, seed) (src/band_index.cpp:90-132) for a
 * host |V| x W code matrix (no permutations attached: step calls need an
 * index from lsb_index_build). */
lsb_status lsb_index_build_codes(lsb_ctx* ctx, const uint32_t* codes_host, uint32_t vocab,
                                 int W, uint64_t index_seed, lsb_index** out);
lsb_status lsb_index_destroy(lsb_index* idx);

typedef struct lsb_index_info {
  uint32_t vocab;
  int W, K, u, bits_per_index, dim;
  uint64_t perm_seed, index_seed;
  uint32_t max_span;      /* BandIndex::max_span_length (band_index.cpp:177-183) */
  uint32_t build_attempts;/* cuckoo attempts used by the worst band (1 = first) */
} lsb_index_info;
lsb_status lsb_index_info_get(const lsb_index* idx, lsb_index_info* out);
/* Band w as the reference exposes it: band_words(w) (V ids), the table's
 * log2 capacity, multipliers and 2*2^lg slots as (key, start, length)
 * triples (BandIndex::band_words / CuckooTable::slots). Any output may be
 * NULL; *lg is always written. Slot placement is the GPU build's; spans are
 * identical to the reference's. */
lsb_status lsb_index_band(const lsb_index* idx, int w, uint32_t* word_ids_host,
                          uint32_t* lg, uint64_t* mul2, uint32_t* slots_host);
/* CuckooTable::find for a batch of (band, key) queries, on the device:
 * found[i] = 1 and (start,len) on a hit (band_index.cpp:73-88). */
lsb_status lsb_index_find(lsb_ctx* ctx, const lsb_index* idx, const int32_t* bands_host,
                          const uint32_t* keys_host, size_t n, uint32_t* start_host,
                          uint32_t* len_host, uint8_t* found_host);
/* Permutation prefixes (u*W x K) of the index, as generated. */
lsb_status lsb_index_perms(const lsb_index* idx, uint32_t* perms_host);

/* -------------------------------------------- 4. stage entry points (host)
 * Each mirrors one reference function; used by the C++ drop-in layer and
 * the per-stage parity tests. Synchronous. */

/* hash_matrix(M, perms, params) (src/wta_hash.cpp:147-171): n x d rows ->
 * n x W band codes; perms_host is (u*W) x K prefixes. NaN -> LSB_EINVAL. */
lsb_status lsb_wta_hash(lsb_ctx* ctx, const float* M_host, int64_t n, int d,
                        const uint32_t* perms_host, int K, int u, int W,
                        uint32_t* codes_host);
/* BandIndex::lookup_hits_into(query_codes, L) (src/band_index.cpp:134-162):
 * dense B x V int32 hit counts. */
lsb_status lsb_lookup_hits(lsb_ctx* ctx, const lsb_index* idx, const uint32_t* q_host,
                           int B, int32_t* L_host);
/* select_candidates(L, t) (src/candidate_selector.cpp:14-55). ids_host has
 * room for V ids. */
lsb_status lsb_select_candidates(lsb_ctx* ctx, const int32_t* L_host, int B, uint32_t V,
                                 int t, uint32_t* ids_host, uint32_t* n_out,
                                 uint32_t* from_threshold);
/* merge_top_frequent(cands, T, specials, V) (src/candidate_selector.cpp:57-103).
 * out_host has room for n + T + nspec ids; prov = {from_threshold,
 * from_top, from_specials}. */
lsb_status lsb_merge_top_frequent(lsb_ctx* ctx, const uint32_t* ids_host, uint32_t n,
                                  uint32_t from_threshold, uint32_t T,
                                  const uint32_t* specials_host, uint32_t nspec, uint32_t V,
                                  uint32_t* out_host, uint32_t* n_out, uint32_t* prov);
/* gather_embeddings(E, cands) (src/candidate_selector.cpp:105-119). */
lsb_status lsb_gather_embeddings(lsb_ctx* ctx, const lsb_model* model,
                                 const uint32_t* ids_host, uint32_t n, float* out_host);
/* compute_logits(H, E_sub) (src/beam_decoder.cpp:23-44): rows x n logits. */
lsb_status lsb_compute_logits(lsb_ctx* ctx, const float* H_host, int rows,
                              const float* Esub_host, int64_t n, int d, lsb_mode mode,
                              float* out_host);
/* softmax_rows(logits) (src/beam_decoder.cpp:46-74). A row with no finite
 * entry (or n == 0) -> LSB_EINVAL. */
lsb_status lsb_softmax_rows(lsb_ctx* ctx, const float* logits_host, int rows, int64_t n,
                            float* out_host);
/* expand_beams(probs, cum, live, frozen, B, id_map) (src/beam_decoder.cpp:76-111).
 * id_map_host may be NULL (identity). frozen entries use word = -1.
 * out_host has room for B choices. */
lsb_status lsb_expand_beams(lsb_ctx* ctx, const float* probs_host, int rows, int64_t n,
                            const double* cum_host, const uint32_t* live_host,
                            const lsb_choice* frozen_host, int nfrozen, int B,
                            const uint32_t* id_map_host, lsb_choice* out_host, int* n_out);

/* --------------------------------------- 5. fused per-step pipeline (device)
 * One decode step of S independent sentences, each holding up to B
 * hypotheses: the kLsh branch of decode() plus expansion
 * (src/beam_decoder.cpp:166-289), batched. Per sentence s the state mirrors
 * decode()'s `hyps` vector: hypotheses 0..n_hyp[s]-1 with cumulative score,
 * finished flag and hidden vector; live = unfinished (in index order),
 * frozen = finished (they compete with their carried score).
 *
 * K1+K2 (hash + cuckoo probe + hit count, vocab-tiled smem counters) ->
 * K3 (threshold bitmap U top-T U specials, ascending compaction) ->
 * K4 (H . E_LSH^T + bias, shared top-T block + per-sentence survivors) ->
 * K5 (row softmax, per-row top-B, per-sentence top-B merge, hidden reorder).
 * No host synchronisation; errors surface at the next lsb_ctx_sync. */
typedef struct lsb_step_config {
  int S;                    /* sentences per batch                        */
  int B;                    /* beam width (hypothesis slots per sentence) */
  uint32_t top_merge;       /* T                                          */
  int threshold;            /* t (0 = whole vocabulary)                   */
  const uint32_t* specials; /* host ids always kept (decode adds EOS)     */
  int nspec;
  lsb_mode mode;
  int full_vocab;           /* 1 = kFull: score all of V, no LSH stages   */
  int top_only;             /* 1 = kTopOnly: [0,T) U specials, no index   */
} lsb_step_config;

/* Validates like DecodeConfig::validate (src/candidate_selector.cpp:121-132). */
lsb_status lsb_batch_create(lsb_ctx* ctx, const lsb_model* model, const lsb_index* idx,
                            const lsb_step_config* cfg, lsb_batch** out);
lsb_status lsb_batch_destroy(lsb_batch* b);

typedef struct lsb_state_dev {
  const float* hidden;      /* [S][B][d]  hypothesis hidden vectors */
  const double* scores;     /* [S][B]     cumulative log-prob       */
  const uint8_t* finished;  /* [S][B]     1 = frozen                */
  const int32_t* n_hyp;     /* [S]        live+frozen hypotheses    */
} lsb_state_dev;

typedef struct lsb_out_dev {
  lsb_choice* choices;      /* [S][B]                                   */
  int32_t* n_choices;       /* [S]                                      */
  float* hidden_out;        /* [S][B][d] parent rows (reorder) or NULL  */
} lsb_out_dev;

lsb_status lsb_step(lsb_batch* b, const lsb_state_dev* in, const lsb_out_dev* out);

/* End-to-end variant for host-resident state (pinned or pageable): copies
 * the state in, runs lsb_step, copies choices/n_choices (and hidden_out if
 * non-NULL) back, synchronises and surfaces errors. */
typedef struct lsb_state_host {
  const float* hidden;
  const double* scores;
  const uint8_t* finished;
  const int32_t* n_hyp;
} lsb_state_host;
lsb_status lsb_step_host(lsb_batch* b, const lsb_state_host* in, lsb_choice* choices_host,
                         int32_t* n_choices_host, float* hidden_out_host);

/* Pipelined form of lsb_step_host for a stream of steps: enqueues the
 * uploads on internal copy streams (three staging slots, so step k+1's
 * upload overlaps step k's kernels), the step, and the read-back of the
 * choices into the caller's (pinned) buffers; does not synchronise. The
 * host buffers must stay valid until lsb_batch_wait returns. */
lsb_status lsb_step_host_async(lsb_batch* b, const lsb_state_host* in, lsb_choice* choices_host,
                               int32_t* n_choices_host);
lsb_status lsb_batch_wait(lsb_batch* b);   /* drain + surface device errors */
/* lsb_step recorded once as a CUDA graph on these fixed device buffers, then
 * replayed with one launch per step (the decode loop rewrites the buffers in
 * place). The context must own a created stream (not the legacy default). */
lsb_status lsb_batch_graph_capture(lsb_batch* b, const lsb_state_dev* in, const lsb_out_dev* out);
lsb_status lsb_batch_graph_launch(lsb_batch* b);

/* Per-sentence views of the last step (device -> host copies, synchronous):
 * candidate ids (|V_LSH| of them, ascending), provenance
 * {from_threshold, from_top, from_specials}, query band codes
 * ([B][W], live rows only), and probabilities over the candidates for each
 * live row ([n_live][n_cand]). */
lsb_status lsb_batch_candidates(lsb_batch* b, int s, uint32_t* ids_host, uint32_t* n_cand,
                                uint32_t* prov3);
lsb_status lsb_batch_query_codes(lsb_batch* b, int s, uint32_t* codes_host);
lsb_status lsb_batch_probs(lsb_batch* b, int s, float* probs_host, int* n_live);
/* Device pointer to the last step's per-sentence candidate counts [S]. */
const uint32_t* lsb_batch_n_cand_dev(lsb_batch* b);
/* Keep probabilities of every live row after a step (default off: the step
 * then writes only what the top-B selection needs). */
lsb_status lsb_batch_keep_probs(lsb_batch* b, int on);

/* Per-kernel device time, milliseconds, measured with CUDA events recorded
 * on the context stream between the step's kernels when profiling is on
 * (lsb_batch_profile(b, n): n = 1 every step, n > 1 every n-th step, 0 off):
 * [probe_count, compact, logits, softmax_topb, expand]. stage_ms: last step;
 * stage_totals: sum over the steps since the previous call (<= 1024). */
lsb_status lsb_batch_profile(lsb_batch* b, int on);
lsb_status lsb_batch_stage_ms(lsb_batch* b, float* ms5);
lsb_status lsb_batch_stage_totals(lsb_batch* b, float* ms5, int* nsteps);

/* ------------------------------------------------ 6. device memory helpers
 * So callers (the C++ drop-in layer, cgo/JNI bindings) never need their own
 * CUDA runtime: allocations on the context's device and copies ordered on
 * its stream. lsb_copy_to_host synchronises the stream and surfaces device
 * errors like lsb_ctx_sync. */
lsb_status lsb_device_alloc(lsb_ctx* ctx, size_t bytes, void** out);
lsb_status lsb_device_free(lsb_ctx* ctx, void* p);
lsb_status lsb_copy_to_device(lsb_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);
lsb_status lsb_copy_to_host(lsb_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);

/* ----------------------------------- 7. drop-in support (C++ layer, I/O)
 * Entry points the C++ drop-in API (include/lshbeam/*.hpp) needs besides the
 * per-step path. */

/* Cuckoo slot placement for index builds on this context. 0 (default):
 * REFERENCE placement -- per band the entries are inserted in the reference's
 * order with its swap-and-flip eviction chain, so slots, multipliers and
 * rebuild counts equal CuckooTable::build's (src/band_index.cpp:32-71;
 * deterministic, WTAIDX1 bytes match). 1: PARALLEL placement -- one thread
 * per entry with 64-bit atomicExch eviction chains (same lookups, different
 * slot order). */
lsb_status lsb_ctx_set_parallel_cuckoo(lsb_ctx* ctx, int on);
/* log2 of the per-array capacity for n entries: max(1, ceil(log2 n))
 * (src/band_index.cpp:39). */
uint32_t lsb_cuckoo_log2_capacity(size_t n_entries);
/* CuckooTable::build(entries, seed) (src/band_index.cpp:32-71) on the device:
 * n distinct keys with their spans -> lg, the two multipliers and
 * 2*2^lg slots as (key, start, length) triples (kEmptyCode = empty).
 * LSB_EINVAL for a sentinel key, LSB_ERUNTIME when the rebuild budget runs out. */
lsb_status lsb_cuckoo_build(lsb_ctx* ctx, const uint32_t* keys, const uint32_t* starts,
                            const uint32_t* lens, uint32_t n, uint64_t seed, uint32_t* lg_out,
                            uint64_t* mul2_out, uint32_t* slots_out, uint32_t* attempts_out);
/* wta_hash_vector over n rows (src/wta_hash.cpp:75-92, :119-125): the
 * P = num_perms raw argmax indices per row, unpacked (K >= 1). */
lsb_status lsb_wta_indices(lsb_ctx* ctx, const float* M_host, int64_t n, int d,
                           const uint32_t* perms_host, int P, int K, uint32_t* idx_host);
/* Uploads a host-described index: the raw-state constructors
 * CuckooTable(lg, mul0, mul1, slots) / BandIndex(vocab, W, word_ids, tables)
 * (include/lshbeam/band_index.hpp) and load_lsh_index (src/band_index.cpp:245-289).
 * word_ids_host: W x vocab (may be NULL: spans then index zeros); lg_host[W];
 * mul_host[2W]; slots_host: per band 2*2^lg (key,start,length) triples,
 * bands back to back. perms_host (u*W x K, may be NULL) attaches the WTA
 * permutations so the index can serve lsb_step. */
lsb_status lsb_index_import(lsb_ctx* ctx, uint32_t vocab, int W, const uint32_t* word_ids_host,
                            const uint32_t* lg_host, const uint64_t* mul_host,
                            const uint32_t* slots_host, const uint32_t* perms_host, int K, int u,
                            int dim, uint64_t perm_seed, lsb_index** out);

/* The recurrence of the synthetic scorer, h' = tanh(W_h h + W_e E[token])
 * (src/model_provider.cpp:83-102), on the device: FP32 in the reference's
 * 4-lane order without FMA, then glibc's tanhf algorithm restated with
 * explicitly rounded single-precision operations (bit-identical to the
 * reference's std::tanh(float); checked over all 2^32 inputs). */
typedef struct lsb_recurrent lsb_recurrent;  /* device W_h, W_e (d x d)  */
lsb_status lsb_recurrent_create(lsb_ctx* ctx, const float* wh_host, const float* we_host, int d,
                                lsb_recurrent** out);
lsb_status lsb_recurrent_destroy(lsb_recurrent* r);
/* n hypotheses, device buffers: tokens[k] < 0 copies hidden_in[k] (a frozen
 * hypothesis is carried unchanged). Asynchronous. */
lsb_status lsb_recurrence(lsb_ctx* ctx, const lsb_model* model, const lsb_recurrent* rec,
                          const float* hidden_in_dev, const int64_t* tokens_dev, int n,
                          float* hidden_out_dev);
/* step_hidden(model, h, token) with host vectors (synchronous). */
lsb_status lsb_step_hidden(lsb_ctx* ctx, const lsb_model* model, const lsb_recurrent* rec,
                           const float* h_host, uint32_t token, float* out_host);

/* exact_topb_logits(H . E^T (+ bias), b) (src/eval_oracle.cpp:11-44): per row
 * the b largest full-vocabulary logits, ties to the smaller id; rows x b ids
 * and values to host buffers. H is a device pointer when H_on_device. */
lsb_status lsb_exact_topb(lsb_ctx* ctx, const lsb_model* model, const float* H, int rows,
                          int H_on_device, int b, int add_bias, uint32_t* ids_host,
                          float* values_host);

/* Measured peak of the paired FP32 pipe (lane-ops/s, 2 per FMUL+FADD MAC as
 * K4 PARITY issues them); bench.py's roofline denominator for K4. */
lsb_status lsb_measure_fp32x2_peak(lsb_ctx* ctx, double* lane_ops_per_s);

/* Self-test: out_dev[k] = log((double) p_dev[k]) by the device function the
 * beam expansion scores with (glibc's log, bit for bit; the reference's
 * cum + log(p) in src/beam_decoder.cpp is evaluated by the host libm).
 * Device pointers; synchronises the context stream. */
lsb_status lsb_selftest_log(lsb_ctx* ctx, const float* p_dev, double* out_dev, size_t n);
/* Self-test: out_dev[k] = exp(x_dev[k]) by the device function the softmax
 * uses (glibc's exp, bit for bit; src/beam_decoder.cpp:46-74 evaluates
 * exp((double) l - mx) with the host libm). */
lsb_status lsb_selftest_exp(lsb_ctx* ctx, const double* x_dev, double* out_dev, size_t n);

/* ---------------------------------- 8. vocabulary-sharded step (cfg 4)
 * One rank's share of a decode step when E is split by contiguous vocabulary
 * slices across ranks (the reference has no multi-device path; SURVEY
 * §8(e)). The rank's lsb_batch is built over its slice (lsb_model of
 * E[v0:v0+n], an index over the slice with the global permutation seed,
 * T_local = clamp(T - v0, 0, n), specials shifted by -v0). Between the phases
 * the caller all-gathers, in rank order, the S*B row maxima (float) and then
 * the S*B row sums (double) and the S*B x lsb_shard_width() top entries.
 * Every rank ends with identical choices and hidden_out; results equal the
 * unsharded step (PARITY: bit-exact unless > 4 entries of one rank tie in p
 * with the B-th winner). */
typedef struct lsb_shard_top {
  float e;        /* float(exp(l - global max)); < 0 marks an empty entry */
  uint32_t word;  /* global word id */
} lsb_shard_top;
int lsb_shard_width(const lsb_batch* b); /* B' = B + 4 entries per row */
lsb_status lsb_shard_phase1(lsb_batch* b, const lsb_state_dev* in, float* rowmax_dev);
lsb_status lsb_shard_phase2(lsb_batch* b, const lsb_state_dev* in, const float* allmax_dev, int G,
                            uint32_t word_base, double* rowsum_dev, lsb_shard_top* top_dev);
lsb_status lsb_shard_phase3(lsb_batch* b, const lsb_state_dev* in, const double* allsum_dev,
                            const lsb_shard_top* alltop_dev, int G, const lsb_out_dev* out);
/* The same with ONE gather after phase 2: each rank passes rowsum_dev = P
 * and top_dev = (lsb_shard_top*)(P + S*B) of one buffer P of
 * S*B*(1 + lsb_shard_width()) 8-byte words, and the ranks' buffers are
 * gathered back to back (rank order) into packed_dev. */
lsb_status lsb_shard_phase3_packed(lsb_batch* b, const lsb_state_dev* in, const void* packed_dev,
                                   int G, const lsb_out_dev* out);

/* The same step with the exchange over PEER MEMORY instead of collectives
 * (NVLink / NVSwitch between the GPUs of a node, CUDA IPC between processes):
 * each rank creates an exchange area, publishes its 64-byte IPC handle, opens
 * every peer's (or, for ranks in one process, attaches their areas with
 * lsb_shard_xchg_set_peer), then lsb_shard_step_peer runs phase 1, pushes its
 * row maxima into every peer's area and waits on per-rank sequence flags on
 * the device, runs phase 2, pushes the packed sums + lists, waits, and runs
 * phase 3 -- no host synchronisation and no collective call per step. The
 * ranks' streams must be able to run concurrently (one process per GPU, or
 * separate streams of one GPU); ranks that share ONE process must use eager
 * CUDA module loading (CUDA_MODULE_LOADING=EAGER), since a lazy kernel load
 * on the host thread would wait for that process's spinning flag wait. */
typedef struct lsb_shard_xchg lsb_shard_xchg;
lsb_status lsb_shard_xchg_create(lsb_batch* b, int G, int rank, lsb_shard_xchg** out);
lsb_status lsb_shard_xchg_destroy(lsb_shard_xchg* x);
void* lsb_shard_xchg_area(lsb_shard_xchg* x);
lsb_status lsb_shard_xchg_ipc_handle(lsb_shard_xchg* x, void* handle64);
lsb_status lsb_shard_xchg_open_ipc(lsb_shard_xchg* x, int peer, const void* handle64);
lsb_status lsb_shard_xchg_set_peer(lsb_shard_xchg* x, int peer, void* area_dev);
lsb_status lsb_shard_step_peer(lsb_batch* b, lsb_shard_xchg* x, const lsb_state_dev* in,
                               uint32_t word_base, const lsb_out_dev* out);

#ifdef __cplusplus
}
#endif
#endif /* LSHBEAM_B200_H */
