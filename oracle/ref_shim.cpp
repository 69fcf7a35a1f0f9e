// ref_shim.cpp -- extern "C" wrapper over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. This file is compiled against the reference's
// public headers (/root/reference/proj/include/lshbeam/*.hpp) and linked with
// the reference's own sources into oracle/_ref/libref_lshbeam.so (see
// oracle/Makefile). It lets the Python tests and bench.py's reference arm call
// the reference's real code path through ctypes. Nothing under
// paper_1806_00588_b200/ links or loads it.
//
// Every entry point returns 0 on success, 1 on std::invalid_argument,
// 2 on std::runtime_error, 3 on anything else (message via ref_last_error()),
// mirroring the exception classes the reference throws.

#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lshbeam/band_index.hpp"
#include "lshbeam/beam_decoder.hpp"
#include "lshbeam/candidate_selector.hpp"
#include "lshbeam/eval_oracle.hpp"
#include "lshbeam/model_provider.hpp"
#include "lshbeam/ref_kernels.hpp"
#include "lshbeam/rng.hpp"
#include "lshbeam/wta_hash.hpp"

using namespace lshbeam;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

MatF to_mat(const float* p, size_t rows, size_t cols) {
  MatF m(rows, cols);
  if (rows * cols) std::memcpy(m.data(), p, rows * cols * sizeof(float));
  return m;
}

MatU32 to_matu(const uint32_t* p, size_t rows, size_t cols) {
  MatU32 m(rows, cols);
  if (rows * cols) std::memcpy(m.data(), p, rows * cols * sizeof(uint32_t));
  return m;
}

struct RefIndex {
  std::unique_ptr<LshIndex> lsh;      // when built from embeddings
  std::unique_ptr<BandIndex> bands;   // when built from codes only
  const BandIndex& b() const { return lsh ? lsh->bands : *bands; }
};

// Model-side state for the per-step reference pipeline: E as a MatF plus the
// logit bias, as decode() holds them in SynthModel.
struct RefCtx {
  MatF E;
  std::vector<float> bias;
};

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads(void) { return omp_get_max_threads(); }

uint64_t ref_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

// SplitMix64(seed) gaussian stream, cast to float and scaled, as fill_gaussian
// (src/model_provider.cpp:15-19).
void ref_gaussian_fill(uint64_t seed, float* out, size_t n, float scale) {
  SplitMix64 g(seed);
  for (size_t i = 0; i < n; ++i) out[i] = static_cast<float>(g.gaussian()) * scale;
}

void ref_splitmix_next(uint64_t seed, uint64_t* out, size_t n) {
  SplitMix64 g(seed);
  for (size_t i = 0; i < n; ++i) out[i] = g.next();
}

void ref_splitmix_bounded(uint64_t seed, uint64_t bound, uint64_t* out, size_t n) {
  SplitMix64 g(seed);
  for (size_t i = 0; i < n; ++i) out[i] = g.bounded(bound);
}

int ref_wta_params_check(int K, int u, int W) {
  return guarded([&] { WtaParams p(K, u, W, 0); (void)p; });
}

int ref_generate_perms(int d, int P, int K, uint64_t seed, uint32_t* out) {
  return guarded([&] {
    const auto perms = PermutationSet::generate(d, P, K, seed);
    for (int p = 0; p < P; ++p) {
      auto r = perms.row(p);
      std::memcpy(out + static_cast<size_t>(p) * K, r.data(), K * sizeof(uint32_t));
    }
  });
}

// hash_matrix with permutations regenerated from (d, params) exactly as
// build_lsh_index does.
int ref_hash_matrix(const float* M, int64_t n, int d, int K, int u, int W,
                    uint64_t seed, uint32_t* out) {
  return guarded([&] {
    const WtaParams params(K, u, W, seed);
    const auto perms = generate_permutations(d, params);
    const MatU32 codes = hash_matrix(to_mat(M, n, d), perms, params);
    if (n) std::memcpy(out, codes.data(), n * W * sizeof(uint32_t));
  });
}

// hash_matrix over explicit permutation prefixes (P = u*W rows of K).
int ref_hash_matrix_perms(const float* M, int64_t n, int d, int K, int u, int W,
                          const uint32_t* prefixes, uint32_t* out) {
  return guarded([&] {
    const WtaParams params(K, u, W, 0);
    const PermutationSet perms(
        d, K, std::vector<uint32_t>(prefixes, prefixes + static_cast<size_t>(u) * W * K));
    const MatU32 codes = hash_matrix(to_mat(M, n, d), perms, params);
    if (n) std::memcpy(out, codes.data(), n * W * sizeof(uint32_t));
  });
}

int ref_pack_bands(const uint32_t* indices, int K, int u, int W, uint32_t* out) {
  return guarded([&] {
    const WtaParams params(K, u, W, 0);
    const auto b = pack_bands(std::span<const uint32_t>(indices, static_cast<size_t>(u) * W), params);
    std::memcpy(out, b.data(), W * sizeof(uint32_t));
  });
}

void* ref_index_from_codes(const uint32_t* codes, uint32_t V, int W, uint64_t seed) {
  auto* h = new RefIndex;
  const int rc = guarded([&] {
    h->bands = std::make_unique<BandIndex>(BandIndex::build(to_matu(codes, V, W), seed));
  });
  if (rc) { delete h; return nullptr; }
  return h;
}

void* ref_index_from_embeddings(const float* E, uint32_t V, int d, int K, int u,
                                int W, uint64_t perm_seed, uint64_t index_seed) {
  auto* h = new RefIndex;
  const int rc = guarded([&] {
    h->lsh = std::make_unique<LshIndex>(
        build_lsh_index(to_mat(E, V, d), WtaParams(K, u, W, perm_seed), index_seed));
  });
  if (rc) { delete h; return nullptr; }
  return h;
}

void ref_index_free(void* h) { delete static_cast<RefIndex*>(h); }

// WTAIDX1 / WTAEMB1 files (src/band_index.cpp:198-289,
// src/model_provider.cpp:116-154): save an index built from embeddings, load
// one back (the LshIndex round trip), save / load an embedding matrix.
int ref_index_save(void* h, const char* path) {
  return guarded([&] { save_lsh_index(*static_cast<RefIndex*>(h)->lsh, path); });
}
void* ref_index_load(const char* path) {
  auto* h = new RefIndex;
  const int rc = guarded([&] { h->lsh = std::make_unique<LshIndex>(load_lsh_index(path)); });
  if (rc) { delete h; return nullptr; }
  return h;
}
int ref_embeddings_save(const float* E, uint32_t V, int d, const char* path) {
  return guarded([&] { save_embeddings(to_mat(E, V, d), path); });
}
int ref_embeddings_load(const char* path, float* E, uint64_t cap, uint32_t* V, int* d) {
  return guarded([&] {
    const MatF M = load_embeddings(path);
    *V = static_cast<uint32_t>(M.rows());
    *d = static_cast<int>(M.cols());
    if (E && cap >= M.rows() * M.cols())
      for (size_t i = 0; i < M.rows(); ++i)
        std::memcpy(E + i * M.cols(), M.row(i).data(), M.cols() * sizeof(float));
  });
}

int ref_index_band_words(void* h, int w, uint32_t* out) {
  const auto& b = static_cast<RefIndex*>(h)->b();
  auto s = b.band_words(w);
  std::memcpy(out, s.data(), s.size() * sizeof(uint32_t));
  return 0;
}

// Table w: lg, multipliers, and (if slots != NULL) 2*2^lg slots as
// (key, start, length) u32 triples.
int ref_index_table(void* h, int w, uint32_t* lg, uint64_t* mul0, uint64_t* mul1,
                    uint32_t* slots) {
  const auto& t = static_cast<RefIndex*>(h)->b().table(w);
  *lg = t.log2_capacity();
  *mul0 = t.multiplier(0);
  *mul1 = t.multiplier(1);
  if (slots) {
    size_t i = 0;
    for (const auto& s : t.slots()) {
      slots[i++] = s.key;
      slots[i++] = s.start;
      slots[i++] = s.length;
    }
  }
  return 0;
}

int ref_index_find(void* h, int w, uint32_t key, uint32_t* start, uint32_t* len,
                   int* probes) {
  const auto& t = static_cast<RefIndex*>(h)->b().table(w);
  const auto r = t.find_counted(key, *probes);
  if (!r) return 0;
  *start = r->start;
  *len = r->length;
  return 1;
}

int ref_index_lookup_hits(void* h, const uint32_t* q, int B, int32_t* L) {
  return guarded([&] {
    const auto& b = static_cast<RefIndex*>(h)->b();
    HitMatrix out;
    b.lookup_hits_into(to_matu(q, B, b.num_bands()), out);
    if (out.rows() * out.cols())
      std::memcpy(L, out.data(), out.rows() * out.cols() * sizeof(int32_t));
  });
}

int ref_lookup_hits_bruteforce(const uint32_t* vocab_codes, uint32_t V,
                               const uint32_t* q, int B, int W, int32_t* L) {
  return guarded([&] {
    const HitMatrix out = ref::lookup_hits(to_matu(vocab_codes, V, W), to_matu(q, B, W));
    if (out.rows() * out.cols())
      std::memcpy(L, out.data(), out.rows() * out.cols() * sizeof(int32_t));
  });
}

// Cuckoo table built standalone (CuckooTable::build) from (key,start,len)
// entries; returns lg/mul and slots like ref_index_table.
int ref_cuckoo_build(const uint32_t* keys, const uint32_t* starts, const uint32_t* lens,
                     size_t n, uint64_t seed, uint32_t* lg, uint64_t* mul0,
                     uint64_t* mul1, uint32_t* slots, size_t slots_cap) {
  return guarded([&] {
    std::vector<std::pair<uint32_t, CuckooTable::Span>> entries;
    for (size_t i = 0; i < n; ++i) entries.push_back({keys[i], {starts[i], lens[i]}});
    const CuckooTable t = CuckooTable::build(entries, seed);
    *lg = t.log2_capacity();
    *mul0 = t.multiplier(0);
    *mul1 = t.multiplier(1);
    if (slots) {
      if (t.slots().size() * 3 > slots_cap) throw std::runtime_error("slot buffer too small");
      size_t i = 0;
      for (const auto& s : t.slots()) {
        slots[i++] = s.key;
        slots[i++] = s.start;
        slots[i++] = s.length;
      }
    }
  });
}

int ref_select_candidates(const int32_t* L, int B, uint32_t V, int t, uint32_t* ids,
                          uint32_t* n, uint32_t* from_threshold) {
  return guarded([&] {
    MatI32 m(B, V);
    if (static_cast<size_t>(B) * V) std::memcpy(m.data(), L, sizeof(int32_t) * B * V);
    const CandidateSet c = select_candidates(m, t);
    std::memcpy(ids, c.word_ids.data(), c.word_ids.size() * sizeof(uint32_t));
    *n = static_cast<uint32_t>(c.word_ids.size());
    *from_threshold = c.from_threshold;
  });
}

int ref_merge_top_frequent(const uint32_t* ids, uint32_t n, uint32_t from_thr,
                           uint32_t T, const uint32_t* specials, uint32_t nspec,
                           uint32_t V, uint32_t* out, uint32_t* nout, uint32_t* prov) {
  return guarded([&] {
    CandidateSet c;
    c.word_ids.assign(ids, ids + n);
    c.from_threshold = from_thr;
    const CandidateSet m = merge_top_frequent(
        std::move(c), T, std::span<const uint32_t>(specials, nspec), V);
    std::memcpy(out, m.word_ids.data(), m.word_ids.size() * sizeof(uint32_t));
    *nout = static_cast<uint32_t>(m.word_ids.size());
    prov[0] = m.from_threshold;
    prov[1] = m.from_top;
    prov[2] = m.from_specials;
  });
}

int ref_gather(const float* E, uint32_t V, int d, const uint32_t* ids, uint32_t n,
               float* out) {
  return guarded([&] {
    CandidateSet c;
    c.word_ids.assign(ids, ids + n);
    const auto g = gather_embeddings(to_mat(E, V, d), c);
    if (n) std::memcpy(out, g.rows.data(), sizeof(float) * n * d);
  });
}

int ref_compute_logits(const float* H, int rows, const float* Esub, int64_t n, int d,
                       float* out) {
  return guarded([&] {
    const MatF L = compute_logits(to_mat(H, rows, d), to_mat(Esub, n, d));
    if (rows * n) std::memcpy(out, L.data(), sizeof(float) * rows * n);
  });
}

int ref_softmax_rows(const float* logits, int rows, int64_t n, float* out) {
  return guarded([&] {
    const MatF P = softmax_rows(to_mat(logits, rows, n));
    if (rows * n) std::memcpy(out, P.data(), sizeof(float) * rows * n);
  });
}

int ref_serial_compute_logits(const float* H, int rows, const float* Esub, int64_t n,
                              int d, float* out) {
  return guarded([&] {
    const MatF L = ref::compute_logits(to_mat(H, rows, d), to_mat(Esub, n, d));
    if (rows * n) std::memcpy(out, L.data(), sizeof(float) * rows * n);
  });
}

int ref_expand_beams(const float* probs, int rows, int64_t n, const double* cum,
                     const uint32_t* live, const double* fz_score,
                     const uint32_t* fz_beam, int nfrozen, int B,
                     const uint32_t* id_map, double* out_score, uint32_t* out_beam,
                     int64_t* out_word, int* nout) {
  return guarded([&] {
    std::vector<BeamChoice> frozen;
    for (int i = 0; i < nfrozen; ++i) frozen.push_back({fz_score[i], fz_beam[i], -1});
    const auto c = expand_beams(
        to_mat(probs, rows, n), std::span<const double>(cum, rows),
        std::span<const uint32_t>(live, rows), frozen, B,
        id_map ? std::span<const uint32_t>(id_map, n) : std::span<const uint32_t>{});
    for (size_t k = 0; k < c.size(); ++k) {
      out_score[k] = c[k].score;
      out_beam[k] = c[k].beam;
      out_word[k] = c[k].word;
    }
    *nout = static_cast<int>(c.size());
  });
}

int ref_exact_topb_logits(const float* logits, int rows, int64_t n, int b,
                          uint32_t* ids, float* vals) {
  return guarded([&] {
    const TopB t = exact_topb_logits(to_mat(logits, rows, n), b);
    if (rows * b) {
      std::memcpy(ids, t.ids.data(), sizeof(uint32_t) * rows * b);
      std::memcpy(vals, t.values.data(), sizeof(float) * rows * b);
    }
  });
}

// ---------------------------------------------------------------- model
void* ref_synth_model(uint32_t V, int d, uint64_t seed, float bias) {
  SynthModel* m = nullptr;
  const int rc = guarded([&] { m = new SynthModel(synth_model(V, d, seed, bias)); });
  return rc ? nullptr : m;
}
void ref_model_free(void* m) { delete static_cast<SynthModel*>(m); }

// Copies any non-NULL field out: E (V*d), w_hidden (d*d), w_embed (d*d),
// h0 (d), freq_bias (V).
void ref_model_get(void* mp, float* E, float* wh, float* we, float* h0, float* bias) {
  const auto& m = *static_cast<SynthModel*>(mp);
  const size_t V = m.vocab, d = m.dim;
  if (E) std::memcpy(E, m.embeddings.data(), V * d * sizeof(float));
  if (wh) std::memcpy(wh, m.w_hidden.data(), d * d * sizeof(float));
  if (we) std::memcpy(we, m.w_embed.data(), d * d * sizeof(float));
  if (h0) std::memcpy(h0, m.h0.data(), d * sizeof(float));
  if (bias) std::memcpy(bias, m.freq_bias.data(), V * sizeof(float));
}

void ref_model_set(void* mp, const float* h0, const float* bias) {
  auto& m = *static_cast<SynthModel*>(mp);
  if (h0) m.h0.assign(h0, h0 + m.dim);
  if (bias) m.freq_bias.assign(bias, bias + m.vocab);
}

int ref_step_hidden(void* mp, const float* h, uint32_t token, float* out) {
  return guarded([&] {
    const auto& m = *static_cast<SynthModel*>(mp);
    step_hidden(m, std::span<const float>(h, m.dim), token, std::span<float>(out, m.dim));
  });
}

// ---------------------------------------------------------------- decode
struct RefDecode {
  DecodeResult r;
};

void* ref_decode(void* mp, int beam, uint32_t T, int t, int max_len,
                 const uint32_t* specials, int nspec, int mode, void* index,
                 int with_oracle, int* status) {
  auto* out = new RefDecode;
  *status = guarded([&] {
    DecodeConfig cfg;
    cfg.beam = beam;
    cfg.top_merge = T;
    cfg.threshold = t;
    cfg.max_len = max_len;
    cfg.specials.assign(specials, specials + nspec);
    const LshIndex* lsh = index ? static_cast<RefIndex*>(index)->lsh.get() : nullptr;
    out->r = decode(*static_cast<SynthModel*>(mp), cfg, static_cast<DecodeMode>(mode), lsh,
                    with_oracle != 0);
  });
  if (*status) { delete out; return nullptr; }
  return out;
}
void ref_decode_free(void* h) { delete static_cast<RefDecode*>(h); }

// Summary: [n_hyp, steps, n_vlsh, n_recall]; counters [thr, top, specials];
// stage ms [wta, cuckoo, cand, elsh, mm, norm, expand, recurrence, oracle].
void ref_decode_info(void* h, int* info, uint64_t* prov, double* stages) {
  const auto& r = static_cast<RefDecode*>(h)->r;
  info[0] = static_cast<int>(r.hypotheses.size());
  info[1] = r.steps;
  info[2] = static_cast<int>(r.per_step_vlsh.size());
  info[3] = static_cast<int>(r.per_step_recall.size());
  prov[0] = r.threshold_survivors;
  prov[1] = r.top_added;
  prov[2] = r.specials_added;
  const auto& s = r.stages;
  const double v[9] = {s.wta_hash, s.cuckoo_lookup, s.construct_candidate_list,
                       s.construct_e_lsh, s.matrix_multiply, s.normalization,
                       s.beam_expansion, s.recurrence, s.oracle};
  std::memcpy(stages, v, sizeof(v));
}

// Hypothesis k: number of tokens, score, finished; tokens copied if non-NULL.
int ref_decode_hyp(void* h, int k, uint32_t* tokens, double* score, int* finished) {
  const auto& hy = static_cast<RefDecode*>(h)->r.hypotheses[k];
  if (tokens) std::memcpy(tokens, hy.tokens.data(), hy.tokens.size() * sizeof(uint32_t));
  *score = hy.score;
  *finished = hy.finished ? 1 : 0;
  return static_cast<int>(hy.tokens.size());
}

void ref_decode_steps(void* h, uint32_t* vlsh, double* recall) {
  const auto& r = static_cast<RefDecode*>(h)->r;
  if (vlsh) std::memcpy(vlsh, r.per_step_vlsh.data(), r.per_step_vlsh.size() * sizeof(uint32_t));
  if (recall)
    std::memcpy(recall, r.per_step_recall.data(), r.per_step_recall.size() * sizeof(double));
}

// ------------------------------------------------- one LSH step, reference
// The body of decode()'s kLsh branch plus expansion
// (src/beam_decoder.cpp:200-289), driven with an externally supplied H so the
// CPU baseline times exactly the reference's per-step hot path. stage_ms gets
// [wta, cuckoo, cand, elsh, mm(+bias), norm, expand]. mode 0 = lsh, 1 = full.
void* ref_ctx_create(const float* E, uint32_t V, int d, const float* bias) {
  auto* c = new RefCtx;
  c->E = to_mat(E, V, d);
  c->bias.assign(bias, bias + V);
  return c;
}
void ref_ctx_free(void* c) { delete static_cast<RefCtx*>(c); }

int ref_step(void* ctxp, void* indexp, int mode, const float* H, int rows,
             const double* cum, const uint32_t* live, int B, uint32_t T, int t,
             const uint32_t* specials, int nspec, double* out_score,
             uint32_t* out_beam, int64_t* out_word, int* nout, uint32_t* n_cand,
             double* stage_ms) {
  return guarded([&] {
    const RefCtx& ctx = *static_cast<RefCtx*>(ctxp);
    const uint32_t V = static_cast<uint32_t>(ctx.E.rows());
    const int d = static_cast<int>(ctx.E.cols());
    MatF Hm = to_mat(H, rows, d);
    for (int i = 0; i < 7; ++i) stage_ms[i] = 0.0;
    CandidateSet cands;
    GatheredEmbeddings gathered;
    const MatF* e_sub = &ctx.E;
    const bool full = mode == 1;
    if (!full) {
      const LshIndex& lsh = *static_cast<RefIndex*>(indexp)->lsh;
      thread_local HitMatrix L;
      auto t0 = Clock::now();
      const MatU32 q = hash_matrix(Hm, lsh.perms, lsh.params);
      stage_ms[0] = ms_since(t0);
      t0 = Clock::now();
      lsh.bands.lookup_hits_into(q, L);
      stage_ms[1] = ms_since(t0);
      t0 = Clock::now();
      cands = select_candidates(L, t);
      cands = merge_top_frequent(std::move(cands), T,
                                 std::span<const uint32_t>(specials, nspec), V);
      stage_ms[2] = ms_since(t0);
      t0 = Clock::now();
      gathered = gather_embeddings(ctx.E, cands);
      stage_ms[3] = ms_since(t0);
      e_sub = &gathered.rows;
    }
    auto t0 = Clock::now();
    MatF logits = compute_logits(Hm, *e_sub);
    {
      const int64_t r = static_cast<int64_t>(logits.rows());
      const int64_t n = static_cast<int64_t>(logits.cols());
      const uint32_t* ids = full ? nullptr : gathered.id_map.data();
      const float* bias = ctx.bias.data();
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < r; ++i) {
        float* row = logits.row(i).data();
        for (int64_t c = 0; c < n; ++c) row[c] += bias[ids ? ids[c] : c];
      }
    }
    stage_ms[4] = ms_since(t0);
    t0 = Clock::now();
    const MatF probs = softmax_rows(logits);
    stage_ms[5] = ms_since(t0);
    t0 = Clock::now();
    const auto chosen = expand_beams(
        probs, std::span<const double>(cum, rows), std::span<const uint32_t>(live, rows),
        {}, B, full ? std::span<const uint32_t>{} : std::span<const uint32_t>(gathered.id_map));
    stage_ms[6] = ms_since(t0);
    for (size_t k = 0; k < chosen.size(); ++k) {
      out_score[k] = chosen[k].score;
      out_beam[k] = chosen[k].beam;
      out_word[k] = chosen[k].word;
    }
    *nout = static_cast<int>(chosen.size());
    *n_cand = full ? V : static_cast<uint32_t>(cands.size());
  });
}

}  // extern "C"
