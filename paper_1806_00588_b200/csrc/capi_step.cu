// capi_step.cu -- the fused per-step pipeline (lsb_batch / lsb_step).
//
// One call = one decode step of S sentences: decode()'s kLsh branch plus
// expand_beams (src/beam_decoder.cpp:200-289), batched over sentences, all on
// the context stream with no host synchronisation:
//   K1+K2 k_probe_count -> K3 k_compact -> K4 k_logits -> K5a k_softmax_topb
//   -> K5b k_expand.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "batch.cuh"

using namespace lsb;

static constexpr int kRing = 1024;

namespace {

template <class T>
cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T));
}

lsb_status free_batch(lsb_batch* b) {
  if (!b) return LSB_OK;
  void* ptrs[] = {b->specials, b->qcodes,   b->bitmap,     b->ids,          b->n_cand,
                  b->prov,     b->logits,   b->top,        b->top_n,        b->h_hidden,
                  b->h_scores, b->h_finished, b->h_nhyp,   b->h_choices,    b->h_nchoices,
                  b->h_hidden_out, b->sh_top, b->sh_topn, b->tc_A, b->tc_H, b->arrive,
                  b->seg_max, b->seg_sum, b->seg_c, b->seg_b, b->seg_top, b->seg_n,
                  b->seg_count, b->seg_e,
                  b->seg_inv,
                  b->split_cnt, b->split_arrive};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (b->fused_stamps) cudaFreeHost(b->fused_stamps);
  for (auto& sl : b->slot) {
    void* sp[] = {sl.hidden, sl.scores, sl.finished, sl.n_hyp, sl.choices, sl.n_choices};
    for (void* p : sp)
      if (p) cudaFree(p);
    if (sl.uploaded) cudaEventDestroy(sl.uploaded);
    if (sl.consumed) cudaEventDestroy(sl.consumed);
    if (sl.computed) cudaEventDestroy(sl.computed);
    if (sl.uploaded2) cudaEventDestroy(sl.uploaded2);
  }
  if (b->graph_exec) cudaGraphExecDestroy(b->graph_exec);
  if (b->graph) cudaGraphDestroy(b->graph);
  if (b->copy_stream) cudaStreamDestroy(b->copy_stream);
  if (b->copy_stream2) cudaStreamDestroy(b->copy_stream2);
  if (b->down_stream) cudaStreamDestroy(b->down_stream);
  for (auto& e : b->ring)
    if (e) cudaEventDestroy(e);
  delete b;
  return LSB_OK;
}

}  // namespace

ProbeArgs lsb::probe_args(const lsb_batch* b, const lsb_state_dev* in) {
  ProbeArgs pa{};
  pa.ix = b->idx->view();
  pa.hidden = in->hidden;
  pa.finished = in->finished;
  pa.n_hyp = in->n_hyp;
  pa.S = b->S;
  pa.B = b->B;
  pa.t = b->t;
  pa.slice_len = b->slice_len;
  pa.counter_bytes = b->counter_bytes;
  pa.levels = b->levels;
  pa.qcodes = b->qcodes;
  pa.bitmap = b->bitmap;
  pa.nwords = b->nwords;
  pa.err = b->ctx->err_dev;
  return pa;
}

CompactArgs lsb::compact_args(const lsb_batch* b, const lsb_state_dev* in, int empty_is_error) {
  CompactArgs ca{};
  ca.bitmap_in = b->bitmap;
  ca.bitmap_clear = b->bitmap;
  ca.nwords = b->nwords;
  ca.V = b->V;
  ca.T = b->T;
  ca.mode = b->cmode;
  ca.specials = b->specials;
  ca.nspec = b->nspec;
  ca.ids = b->ids;
  ca.ncap = b->ncap;
  ca.n_cand = b->n_cand;
  ca.prov = b->prov;
  ca.empty_is_error = empty_is_error;
  ca.n_hyp = in->n_hyp;
  ca.finished = in->finished;
  ca.B = b->B;
  ca.err = b->ctx->err_dev;
  return ca;
}

LogitsArgs lsb::logits_args(const lsb_batch* b, const lsb_state_dev* in) {
  LogitsArgs la{};
  la.H = in->hidden;
  la.d = b->d;
  la.R_total = b->S * b->B;
  la.Bsent = b->B;
  la.E = b->model->E;
  la.bias = b->model->bias;
  la.n_shared = b->n_shared;
  la.ids = b->cmode == 0 ? b->ids : nullptr;
  la.ncap = b->ncap;
  la.n_cand = b->n_cand;
  la.S = b->S;
  la.out = b->logits;
  la.ldo = b->ncap;
  la.tc_A = b->tc_A;
  la.tc_H = b->tc_H;
  la.tc_N = b->tc_N;
  return la;
}

SoftmaxArgs lsb::softmax_args(const lsb_batch* b, const lsb_state_dev* in) {
  SoftmaxArgs sa{};
  sa.logits = b->logits;
  sa.ldl = b->ncap;
  sa.R_total = b->S * b->B;
  sa.Bsent = b->B;
  sa.topB = b->B;
  sa.n_cand = b->n_cand;
  sa.finished = in->finished;
  sa.n_hyp = in->n_hyp;
  sa.keep_probs = b->keep_probs;
  sa.top = b->top;
  sa.top_n = b->top_n;
  sa.err = b->ctx->err_dev;
  sa.seq_denominator = b->seq_denom;
  return sa;
}

ExpandArgs lsb::expand_args(const lsb_batch* b, const lsb_state_dev* in, const lsb_out_dev* out) {
  ExpandArgs ea{};
  ea.S = b->S;
  ea.Bsent = b->B;
  ea.topB = b->B;
  ea.top = b->top;
  ea.top_n = b->top_n;
  ea.scores = in->scores;
  ea.finished = in->finished;
  ea.n_hyp = in->n_hyp;
  ea.ids = b->cmode == 0 ? b->ids : nullptr;
  ea.ncap = b->ncap;
  ea.n_shared = b->n_shared;
  ea.hidden = in->hidden;
  ea.d = b->d;
  ea.hidden_out = out->hidden_out;
  ea.choices = out->choices;
  ea.n_choices = out->n_choices;
  return ea;
}

lsb_status lsb::step_front(lsb_batch* b, const lsb_state_dev* in, int empty_is_error) {
  lsb_ctx* ctx = b->ctx;
  cudaStream_t st = ctx->stream;
  lsb_status rc;
  b->rec = b->profile && (b->step_count++ % static_cast<uint64_t>(b->profile_every)) == 0;
  if (b->rec) {
    b->ev = &b->ring[static_cast<size_t>(b->ring_next) * 6];
    b->ring_next = (b->ring_next + 1) % kRing;
    b->ring_used = std::min(b->ring_used + 1, kRing);
    LSB_CUDA(cudaEventRecord(b->ev[0], st));
  }
  // K1 + K2 (kTopOnly has no index: the bitmap stays empty)
  if (b->cmode != 2 && b->idx) {
    const ProbeArgs pa = probe_args(b, in);
    if ((rc = b->probe_G > 0 ? launch_probe_split(ctx, pa, b->probe_G, b->split_cnt,
                                                  b->split_words, b->split_arrive)
                             : launch_probe(ctx, pa)))
      return rc;
  }
  if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[1], st));
  // K3
  if ((rc = launch_compact(ctx, compact_args(b, in, empty_is_error), b->S))) return rc;
  if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[2], st));
  // K4
  if ((rc = launch_logits(ctx, logits_args(b, in), b->mode, ctx->sm_count * 8))) return rc;
  if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[3], st));
  return LSB_OK;
}

extern "C" {

lsb_status lsb_batch_create(lsb_ctx* ctx, const lsb_model* model, const lsb_index* idx,
                            const lsb_step_config* cfg, lsb_batch** out) {
  if (!ctx || !model || !cfg || !out) return set_error("lsb_batch_create: null argument"), LSB_EINVAL;
  *out = nullptr;
  const uint32_t V = model->V;
  // DecodeConfig::validate (src/candidate_selector.cpp:121-132)
  if (cfg->B < 1) return set_error("config: beam must be >= 1"), LSB_EINVAL;
  if (cfg->B > 64) return set_error("config: beam above 64 is not supported by the fused step"), LSB_EINVAL;
  if (cfg->S < 1) return set_error("config: at least one sentence"), LSB_EINVAL;
  // the gather kernels address E rows by 32-bit element offsets (bit 31 marks
  // a padding column)
  if (static_cast<uint64_t>(V) * model->d >= (1ull << 31))
    return set_error("lsb_batch_create: |V| x d must stay below 2^31 elements"), LSB_EINVAL;
  if (cfg->top_merge > V) return set_error("config: T exceeds vocabulary size"), LSB_EINVAL;
  if (!cfg->full_vocab && !cfg->top_only) {
    if (!idx || !idx->has_perms)
      return set_error("decode: lsh mode requires an index"), LSB_EINVAL;
    if (idx->V != V || idx->dim != model->d)
      return set_error("decode: index does not match the model"), LSB_EINVAL;
    if (cfg->threshold < 0 || cfg->threshold > idx->W)
      return set_error("config: t must be in [0, W]"), LSB_EINVAL;
  }
  std::vector<uint32_t> spec(cfg->specials, cfg->specials + std::max(0, cfg->nspec));
  for (uint32_t id : spec)
    if (id >= V) return set_error("config: special id out of range"), LSB_EINVAL;
  std::sort(spec.begin(), spec.end());
  spec.erase(std::unique(spec.begin(), spec.end()), spec.end());
  LSB_CUDA(cudaSetDevice(ctx->device));

  auto* b = new lsb_batch;
  b->ctx = ctx;
  b->model = model;
  b->idx = (cfg->full_vocab || cfg->top_only) ? nullptr : idx;
  b->S = cfg->S;
  b->B = cfg->B;
  b->d = model->d;
  b->V = V;
  b->T = cfg->top_merge;
  b->t = cfg->threshold;
  b->mode = cfg->mode;
  // kTopOnly ignores t and scores [0,T) U specials (src/beam_decoder.cpp:189-199)
  b->cmode = cfg->full_vocab ? 2 : (!cfg->top_only && cfg->threshold == 0 ? 1 : 0);
  {
    const char* sd = getenv("LSB_SEQ_DENOM");
    b->seq_denom = sd && atoi(sd) == 1;  // always the sequential sum
  }
  b->n_shared = b->cmode ? V : b->T;
  b->ncap = (static_cast<size_t>(V) + 3) & ~size_t(3);
  b->nwords = (V + 31) / 32;
  b->nspec = static_cast<int>(spec.size());
  if (b->idx) {
    b->counter_bytes = b->idx->W < 256 ? 1 : 2;
    if (b->t >= 1 && b->t <= 8) {
      // t bit planes of the slice (t-1 levels + the marked set), <= 32 KB
      b->levels = b->t - 1;
      // (cfg 4, V=200k -> 2 slices per row: 32 KB of planes measured best,
      // 16 / 64 / 96 KB: probe 47.6 / 36.4 / 37.4 vs 33.3 us)
      const uint32_t budget = 32 * 1024 * 8 / b->t;  // words per slice
      const uint32_t nslices = (V + budget - 1) / budget;
      b->slice_len = ((V + nslices - 1) / nslices + 127) & ~127u;  // planes of 16-B multiples
    } else {
      const uint32_t budget = 96 * 1024 / b->counter_bytes;
      const uint32_t nslices = (V + budget - 1) / budget;
      b->slice_len = ((V + nslices - 1) / nslices + 63) & ~63u;
    }
  }
  const size_t SB = static_cast<size_t>(b->S) * b->B;
  cudaError_t e = dalloc(&b->specials, spec.size());
  if (e == cudaSuccess && !spec.empty())
    e = cudaMemcpy(b->specials, spec.data(), spec.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = dalloc(&b->qcodes, SB * (b->idx ? b->idx->W : 1));
  // rows that are frozen or past n_hyp are never hashed; keep their codes defined
  if (e == cudaSuccess) e = cudaMemset(b->qcodes, 0, SB * (b->idx ? b->idx->W : 1) * 4);
  if (e == cudaSuccess) e = dalloc(&b->bitmap, static_cast<size_t>(b->S) * b->nwords);
  if (e == cudaSuccess)
    e = cudaMemset(b->bitmap, 0, std::max<size_t>(1, static_cast<size_t>(b->S) * b->nwords) * 4);
  if (e == cudaSuccess) e = dalloc(&b->ids, static_cast<size_t>(b->S) * b->ncap);
  if (e == cudaSuccess) e = dalloc(&b->n_cand, b->S);
  if (e == cudaSuccess) e = dalloc(&b->prov, 3 * b->S);
  if (e == cudaSuccess) e = dalloc(&b->logits, SB * b->ncap);
  if (e == cudaSuccess) e = dalloc(&b->top, SB * b->B);
  if (e == cudaSuccess) e = dalloc(&b->top_n, SB);
  if (e == cudaSuccess) e = dalloc(&b->arrive, b->S);
  if (e == cudaSuccess) e = cudaMemset(b->arrive, 0, b->S * sizeof(uint32_t));
  // Few rows with many bands (a one-sentence decode at W > 64): k_probe_count
  // would run S*B CTAs on a 148-SM GPU, each walking every band's span; split
  // each row's bands over G CTAs (k_probe_split) so the grid covers ~2 CTAs
  // per SM. Measured at S=1, V=50k, W=500: K=8 (98-word spans) 100 -> 29 us;
  // with short spans (K=16: 12 words) and at W=16 (cfg 1: 16.7 vs 10.8 us,
  // global-counter atomics vs shared-memory ones) k_probe_count stays faster.
  // LSB_PROBE_SPLIT=0 turns it off, =G forces G.
  if (e == cudaSuccess && b->idx && b->t > 0) {
    static const int split_env = getenv("LSB_PROBE_SPLIT") ? atoi(getenv("LSB_PROBE_SPLIT")) : -1;
    const uint32_t nslices = b->slice_len ? (V + b->slice_len - 1) / b->slice_len : 1;
    const int R = static_cast<int>(SB);
    int G = 0;
    if (split_env > 0) G = split_env;
    else if (split_env < 0 && b->idx->W > 64 && b->idx->W <= 65535 &&  // 16-bit counts <= W
             static_cast<long>(R) * nslices < ctx->sm_count &&
             // long spans only: with ~12-word spans (K=16, u=3: 12-bit codes)
             // k_probe_count is faster (26 vs 33 us at S=1, V=50k, W=500)
             (b->idx->u * b->idx->bits >= 32 ||
              (static_cast<uint64_t>(V) >> (b->idx->u * b->idx->bits)) >= 32))
      G = (2 * ctx->sm_count + R - 1) / R;
    G = std::min(G, b->idx->W);
    const uint32_t words = ((V + 1) / 2 + 3) & ~3u;
    if (G > 1 && SB * words * 4 <= (64ull << 20)) {
      b->probe_G = G;
      b->split_words = words;
      e = dalloc(&b->split_cnt, SB * words);
      if (e == cudaSuccess) e = cudaMemset(b->split_cnt, 0, SB * words * 4);
      if (e == cudaSuccess) e = dalloc(&b->split_arrive, SB);
      if (e == cudaSuccess) e = cudaMemset(b->split_arrive, 0, SB * 4);
    }
  }
  // every row scores all V words (full vocabulary, t = 0): rows that long
  // take the segmented K5a (one CTA per row segment)
  static const bool seg_off = getenv("LSB_NO_SEG") != nullptr;
  if (e == cudaSuccess && b->cmode != 0 && V >= 8192 && !seg_off) {
    b->seg_P = seg_count(ctx, static_cast<int>(SB), V, b->B);
    const size_t np = SB * b->seg_P;
    e = dalloc(&b->seg_max, np);
    if (e == cudaSuccess) e = dalloc(&b->seg_sum, np);
    if (e == cudaSuccess) e = dalloc(&b->seg_c, np);
    if (e == cudaSuccess) e = dalloc(&b->seg_b, np);
    if (e == cudaSuccess) e = dalloc(&b->seg_top, np * b->B);
    if (e == cudaSuccess) e = dalloc(&b->seg_n, np);
    if (e == cudaSuccess) e = dalloc(&b->seg_count, SB);
    if (e == cudaSuccess) e = cudaMemset(b->seg_count, 0, SB * sizeof(uint32_t));
    if (e == cudaSuccess) e = dalloc(&b->seg_e, SB * b->ncap);
    if (e == cudaSuccess) e = dalloc(&b->seg_inv, SB);
  }
  // FAST: the rows sharing [0, n_shared) form a dense contraction for the
  // tensor cores; E's block is split into 3xTF32 and tiled once, here
  const int R = b->S * b->B;
  if (e == cudaSuccess && b->mode == LSB_MODE_FAST && R >= kTcMinRows && b->n_shared > 0 &&
      (b->d & 3) == 0 && (reinterpret_cast<uintptr_t>(model->E) & 15) == 0) {
    b->tc_N = tc_rows_per_tile(ctx, R, b->n_shared);
    e = dalloc(&b->tc_A, tf32_tiled_floats(static_cast<int>(b->n_shared), b->d, 128));
    if (e == cudaSuccess) e = dalloc(&b->tc_H, tf32_tiled_floats(R, b->d, b->tc_N));
    if (e == cudaSuccess &&
        launch_tf32_tile(ctx, model->E, static_cast<int>(b->n_shared), b->d, 128, b->tc_A) != LSB_OK)
      e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    free_batch(b);
    return cuda_status(e, "lsb_batch_create");
  }
  *out = b;
  return LSB_OK;
}

lsb_status lsb_batch_destroy(lsb_batch* b) {
  if (b && b->ctx) cudaStreamSynchronize(b->ctx->stream);
  return free_batch(b);
}

lsb_status lsb_batch_keep_probs(lsb_batch* b, int on) {
  if (!b) return LSB_EINVAL;
  b->keep_probs = on ? 1 : 0;
  return LSB_OK;
}

lsb_status lsb_batch_profile(lsb_batch* b, int on) {
  if (!b) return LSB_EINVAL;
  // on > 1: sample every on-th step (stage events break programmatic
  // dependent launch between the kernels they separate)
  b->profile_every = on > 1 ? on : 1;
  b->step_count = 0;
  if (on && b->ring.empty()) {
    b->ring.assign(kRing * 6, nullptr);
    for (auto& e : b->ring) LSB_CUDA(cudaEventCreate(&e));
  }
  b->profile = on != 0;
  b->ring_next = b->ring_used = 0;
  return LSB_OK;
}

// Sums the per-stage device time of the steps recorded since the last call
// (at most the last kRing steps) and restarts the ring.
lsb_status lsb_batch_stage_totals(lsb_batch* b, float* ms5, int* nsteps) {
  if (!b || !ms5) return LSB_EINVAL;
  if (!b->profile) return set_error("profiling is off"), LSB_EINVAL;
  for (int k = 0; k < 5; ++k) ms5[k] = 0.0f;
  const int n = std::min(b->ring_used, kRing);
  for (int i = 0; i < n; ++i) {
    cudaEvent_t* ev = &b->ring[static_cast<size_t>(i) * 6];
    LSB_CUDA(cudaEventSynchronize(ev[5]));
    for (int k = 0; k < 5; ++k) {
      float ms = 0.0f;
      LSB_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
      ms5[k] += ms;
    }
  }
  if (nsteps) *nsteps = n;
  b->ring_next = b->ring_used = 0;
  return LSB_OK;
}

lsb_status lsb_batch_stage_ms(lsb_batch* b, float* ms5) {
  if (!b || !ms5) return LSB_EINVAL;
  if (!b->profile || !b->ring_used) return set_error("profiling is off"), LSB_EINVAL;
  const int last = (b->ring_next + kRing - 1) % kRing;
  cudaEvent_t* ev = &b->ring[static_cast<size_t>(last) * 6];
  LSB_CUDA(cudaEventSynchronize(ev[5]));
  for (int k = 0; k < 5; ++k) LSB_CUDA(cudaEventElapsedTime(&ms5[k], ev[k], ev[k + 1]));
  return LSB_OK;
}

lsb_status lsb_step(lsb_batch* b, const lsb_state_dev* in, const lsb_out_dev* out) {
  if (!b || !in || !out || !in->hidden || !in->scores || !out->choices || !out->n_choices)
    return set_error("lsb_step: null argument"), LSB_EINVAL;
  lsb_ctx* ctx = b->ctx;
  cudaStream_t st = ctx->stream;
  // small batches: the whole step in one cooperative launch (k_step_fused.cu)
  bool fused = false;
  lsb_status rc = launch_step_fused(b, in, out, &fused);
  if (rc) return rc;
  if (fused) {
    b->last = *in;
    b->has_last = true;
    return LSB_OK;
  }
  rc = step_front(b, in, 1);
  if (rc) return rc;
  // K5a + K5b
  const SoftmaxArgs sa = softmax_args(b, in);
  const ExpandArgs ea = expand_args(b, in, out);
  // K5 variant (LSB_K5): 0 = CTA-per-row softmax + per-sentence expansion
  // (default; measured fastest with the K5b reorder batched), 1 = warp-per-row
  // softmax + expansion, 2 = one fused launch per sentence. All three are
  // bit-identical (tests/test_gpu_step.py runs under each).
  static const int k5 = [] {
    const char* e = getenv("LSB_K5");
    return e ? atoi(e) : 0;
  }();
  if (b->cmode == 0 && k5 == 2 && select_fused_applies(sa, ea)) {
    // one launch: CTA per sentence, warp per row, then the expansion
    if ((rc = launch_select_fused(ctx, sa, ea, static_cast<uint32_t>(b->ncap), b->arrive))) return rc;
    if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[4], st));
  } else if (b->cmode == 0 && k5 == 1) {
    // warp per row over the whole GPU, then the per-sentence expansion
    if ((rc = launch_softmax_warp(ctx, sa, static_cast<uint32_t>(b->ncap)))) return rc;
    if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[4], st));
    if ((rc = launch_expand(ctx, ea))) return rc;
  } else if (b->seg_P > 0) {
    SegArgs g{};
    g.sa = sa;
    g.P = b->seg_P;
    g.seglen = static_cast<uint32_t>((b->V + b->seg_P - 1) / b->seg_P);
    g.part_max = b->seg_max;
    g.part_sum = b->seg_sum;
    g.part_c = b->seg_c;
    g.part_b = b->seg_b;
    g.seg_top = b->seg_top;
    g.seg_n = b->seg_n;
    g.count = b->seg_count;
    g.e_out = b->seg_e;
    g.inv = b->seg_inv;
    if ((rc = launch_softmax_seg(ctx, g))) return rc;
    if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[4], st));
    if ((rc = launch_expand(ctx, ea))) return rc;
  } else {
    if ((rc = launch_softmax(ctx, sa))) return rc;
    if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[4], st));
    if ((rc = launch_expand(ctx, ea))) return rc;
  }
  if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[5], st));
  b->last = *in;
  b->has_last = true;
  return LSB_OK;
}

lsb_status lsb_step_host(lsb_batch* b, const lsb_state_host* in, lsb_choice* choices_host,
                         int32_t* n_choices_host, float* hidden_out_host) {
  if (!b || !in || !in->hidden || !in->scores || !choices_host || !n_choices_host)
    return set_error("lsb_step_host: null argument"), LSB_EINVAL;
  const size_t SB = static_cast<size_t>(b->S) * b->B;
  const size_t HD = SB * b->d;
  cudaStream_t st = b->ctx->stream;
  if (!b->h_hidden) {
    LSB_CUDA(dalloc(&b->h_hidden, HD));
    LSB_CUDA(dalloc(&b->h_scores, SB));
    LSB_CUDA(dalloc(&b->h_finished, SB));
    LSB_CUDA(dalloc(&b->h_nhyp, b->S));
    LSB_CUDA(dalloc(&b->h_choices, SB));
    LSB_CUDA(dalloc(&b->h_nchoices, b->S));
    // rows past n_choices[s] are never written; zero them once so the
    // whole-buffer read-back copies defined bytes
    LSB_CUDA(cudaMemsetAsync(b->h_choices, 0, SB * sizeof(lsb_choice), st));
  }
  if (hidden_out_host && !b->h_hidden_out) {
    LSB_CUDA(dalloc(&b->h_hidden_out, HD));
    // rows past n_choices[s] are not written by the reorder (see h_choices)
    LSB_CUDA(cudaMemsetAsync(b->h_hidden_out, 0, HD * 4, st));
  }
  LSB_CUDA(cudaMemcpyAsync(b->h_hidden, in->hidden, HD * 4, cudaMemcpyHostToDevice, st));
  LSB_CUDA(cudaMemcpyAsync(b->h_scores, in->scores, SB * 8, cudaMemcpyHostToDevice, st));
  lsb_state_dev d{};
  d.hidden = b->h_hidden;
  d.scores = b->h_scores;
  if (in->finished) {
    LSB_CUDA(cudaMemcpyAsync(b->h_finished, in->finished, SB, cudaMemcpyHostToDevice, st));
    d.finished = b->h_finished;
  }
  if (in->n_hyp) {
    LSB_CUDA(cudaMemcpyAsync(b->h_nhyp, in->n_hyp, b->S * 4, cudaMemcpyHostToDevice, st));
    d.n_hyp = b->h_nhyp;
  }
  lsb_out_dev o{};
  o.choices = b->h_choices;
  o.n_choices = b->h_nchoices;
  o.hidden_out = hidden_out_host ? b->h_hidden_out : nullptr;
  lsb_status rc = lsb_step(b, &d, &o);
  if (rc) return rc;
  LSB_CUDA(cudaMemcpyAsync(choices_host, b->h_choices, SB * sizeof(lsb_choice),
                           cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaMemcpyAsync(n_choices_host, b->h_nchoices, b->S * 4, cudaMemcpyDeviceToHost, st));
  if (hidden_out_host)
    LSB_CUDA(cudaMemcpyAsync(hidden_out_host, b->h_hidden_out, HD * 4, cudaMemcpyDeviceToHost, st));
  return lsb_ctx_sync(b->ctx);
}

// Pipelined variant of lsb_step_host: uploads go to an upload stream into
// one of three staging slots while the previous step's kernels run; the step
// waits for its upload; its choices are read back on a third stream, so the
// step stream runs kernels only.
// Nothing synchronises the host; lsb_batch_wait drains the pipeline.
lsb_status lsb_step_host_async(lsb_batch* b, const lsb_state_host* in, lsb_choice* choices_host,
                               int32_t* n_choices_host) {
  if (!b || !in || !in->hidden || !in->scores || !choices_host || !n_choices_host)
    return set_error("lsb_step_host_async: null argument"), LSB_EINVAL;
  const size_t SB = static_cast<size_t>(b->S) * b->B;
  const size_t HD = SB * b->d;
  cudaStream_t st = b->ctx->stream;
  if (!b->copy_stream) {
    LSB_CUDA(cudaStreamCreateWithFlags(&b->copy_stream, cudaStreamNonBlocking));
    LSB_CUDA(cudaStreamCreateWithFlags(&b->copy_stream2, cudaStreamNonBlocking));
    LSB_CUDA(cudaStreamCreateWithFlags(&b->down_stream, cudaStreamNonBlocking));
    for (auto& sl : b->slot) {
      LSB_CUDA(dalloc(&sl.hidden, HD));
      LSB_CUDA(dalloc(&sl.scores, SB));
      LSB_CUDA(dalloc(&sl.finished, SB));
      LSB_CUDA(dalloc(&sl.n_hyp, b->S));
      LSB_CUDA(dalloc(&sl.choices, SB));
      LSB_CUDA(dalloc(&sl.n_choices, b->S));
      LSB_CUDA(cudaMemset(sl.choices, 0, SB * sizeof(lsb_choice)));
      LSB_CUDA(cudaEventCreateWithFlags(&sl.uploaded, cudaEventDisableTiming));
      LSB_CUDA(cudaEventCreateWithFlags(&sl.consumed, cudaEventDisableTiming));
      LSB_CUDA(cudaEventCreateWithFlags(&sl.computed, cudaEventDisableTiming));
      LSB_CUDA(cudaEventCreateWithFlags(&sl.uploaded2, cudaEventDisableTiming));
    }
  }
  auto& sl = b->slot[b->next_slot];
  b->next_slot = (b->next_slot + 1) % lsb_batch::kSlots;
  cudaStream_t cs = b->copy_stream;
  // the step that used this slot three calls ago must be done reading it
  cudaStream_t cs2 = b->copy_stream2;
  if (sl.used) {
    LSB_CUDA(cudaStreamWaitEvent(cs, sl.consumed, 0));
    LSB_CUDA(cudaStreamWaitEvent(cs2, sl.consumed, 0));
  }
  // the hidden states (the bulk: S*B*d floats) go up in two halves on two
  // streams, i.e. two copy engines (one 3 MB pinned copy measured 30-45 GB/s
  // on B200 boxes, two halves in parallel 48-49 GB/s)
  const size_t half = (HD / 2) & ~size_t(3);
  LSB_CUDA(cudaMemcpyAsync(sl.hidden + half, in->hidden + half, (HD - half) * 4,
                           cudaMemcpyHostToDevice, cs2));
  LSB_CUDA(cudaEventRecord(sl.uploaded2, cs2));
  LSB_CUDA(cudaMemcpyAsync(sl.hidden, in->hidden, half * 4, cudaMemcpyHostToDevice, cs));
  LSB_CUDA(cudaMemcpyAsync(sl.scores, in->scores, SB * 8, cudaMemcpyHostToDevice, cs));
  lsb_state_dev d{};
  d.hidden = sl.hidden;
  d.scores = sl.scores;
  if (in->finished) {
    LSB_CUDA(cudaMemcpyAsync(sl.finished, in->finished, SB, cudaMemcpyHostToDevice, cs));
    d.finished = sl.finished;
  }
  if (in->n_hyp) {
    LSB_CUDA(cudaMemcpyAsync(sl.n_hyp, in->n_hyp, b->S * 4, cudaMemcpyHostToDevice, cs));
    d.n_hyp = sl.n_hyp;
  }
  LSB_CUDA(cudaEventRecord(sl.uploaded, cs));
  LSB_CUDA(cudaStreamWaitEvent(st, sl.uploaded, 0));
  LSB_CUDA(cudaStreamWaitEvent(st, sl.uploaded2, 0));
  lsb_out_dev o{};
  o.choices = sl.choices;
  o.n_choices = sl.n_choices;
  lsb_status rc = lsb_step(b, &d, &o);
  if (rc) return rc;
  // read-back on the copy stream, so the step stream goes straight on to the
  // next step; `consumed` then covers both the kernels' reads of the staged
  // inputs and the read-back of the staged outputs
  cudaStream_t ds = b->down_stream;
  LSB_CUDA(cudaEventRecord(sl.computed, st));
  LSB_CUDA(cudaStreamWaitEvent(ds, sl.computed, 0));
  LSB_CUDA(cudaMemcpyAsync(choices_host, sl.choices, SB * sizeof(lsb_choice),
                           cudaMemcpyDeviceToHost, ds));
  LSB_CUDA(cudaMemcpyAsync(n_choices_host, sl.n_choices, b->S * 4, cudaMemcpyDeviceToHost, ds));
  LSB_CUDA(cudaEventRecord(sl.consumed, ds));
  sl.used = true;
  return LSB_OK;
}

lsb_status lsb_batch_wait(lsb_batch* b) {
  if (!b) return set_error("lsb_batch_wait: null"), LSB_EINVAL;
  if (b->copy_stream) LSB_CUDA(cudaStreamSynchronize(b->copy_stream));
  if (b->copy_stream2) LSB_CUDA(cudaStreamSynchronize(b->copy_stream2));
  if (b->down_stream) LSB_CUDA(cudaStreamSynchronize(b->down_stream));
  return lsb_ctx_sync(b->ctx);
}

lsb_status lsb_batch_candidates(lsb_batch* b, int s, uint32_t* ids_host, uint32_t* n_cand,
                                uint32_t* prov3) {
  if (!b || s < 0 || s >= b->S || !n_cand) return set_error("lsb_batch_candidates: bad sentence"), LSB_EINVAL;
  cudaStream_t st = b->ctx->stream;
  uint32_t prov[3];
  LSB_CUDA(cudaMemcpyAsync(n_cand, b->n_cand + s, 4, cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaMemcpyAsync(prov, b->prov + 3 * s, 12, cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaStreamSynchronize(st));
  if (prov3) std::memcpy(prov3, prov, 12);
  if (ids_host) {
    if (b->cmode == 0) {
      LSB_CUDA(cudaMemcpy(ids_host, b->ids + static_cast<size_t>(s) * b->ncap, *n_cand * 4ull,
                          cudaMemcpyDeviceToHost));
    } else {
      for (uint32_t r = 0; r < *n_cand; ++r) ids_host[r] = r;
    }
  }
  return LSB_OK;
}

lsb_status lsb_batch_query_codes(lsb_batch* b, int s, uint32_t* codes_host) {
  if (!b || !b->idx || s < 0 || s >= b->S) return set_error("lsb_batch_query_codes: bad sentence"), LSB_EINVAL;
  const size_t n = static_cast<size_t>(b->B) * b->idx->W;
  LSB_CUDA(cudaMemcpy(codes_host, b->qcodes + s * n, n * 4, cudaMemcpyDeviceToHost));
  return LSB_OK;
}

lsb_status lsb_batch_probs(lsb_batch* b, int s, float* probs_host, int* n_live) {
  if (!b || s < 0 || s >= b->S || !b->has_last) return set_error("lsb_batch_probs: no step"), LSB_EINVAL;
  if (!b->keep_probs) return set_error("lsb_batch_probs: enable lsb_batch_keep_probs first"), LSB_EINVAL;
  cudaStream_t st = b->ctx->stream;
  LSB_CUDA(cudaStreamSynchronize(st));
  uint32_t n = 0;
  int32_t nh = b->B;
  std::vector<uint8_t> fin(b->B, 0);
  LSB_CUDA(cudaMemcpy(&n, b->n_cand + s, 4, cudaMemcpyDeviceToHost));
  if (b->last.n_hyp) LSB_CUDA(cudaMemcpy(&nh, b->last.n_hyp + s, 4, cudaMemcpyDeviceToHost));
  if (b->last.finished)
    LSB_CUDA(cudaMemcpy(fin.data(), b->last.finished + static_cast<size_t>(s) * b->B, b->B,
                        cudaMemcpyDeviceToHost));
  int live = 0;
  for (int i = 0; i < nh; ++i) {
    if (fin[i]) continue;
    if (probs_host)
      LSB_CUDA(cudaMemcpy(probs_host + static_cast<size_t>(live) * n,
                          b->logits + (static_cast<size_t>(s) * b->B + i) * b->ncap, n * 4ull,
                          cudaMemcpyDeviceToHost));
    ++live;
  }
  if (n_live) *n_live = live;
  return LSB_OK;
}

const uint32_t* lsb_batch_n_cand_dev(lsb_batch* b) { return b ? b->n_cand : nullptr; }

// One lsb_step recorded as a CUDA graph on the context stream (the PDL
// launch attributes become programmatic edges), replayed with one
// cudaGraphLaunch per step: the decode loop updates the same device buffers
// in place every step, so their addresses are fixed. Replaces the five
// per-kernel host launches of a small batch by one.
lsb_status lsb_batch_graph_capture(lsb_batch* b, const lsb_state_dev* in, const lsb_out_dev* out) {
  if (!b || !in || !out) return set_error("lsb_batch_graph_capture: null argument"), LSB_EINVAL;
  lsb_ctx* ctx = b->ctx;
  if (ctx->stream == nullptr || ctx->stream == cudaStreamLegacy || ctx->stream == cudaStreamPerThread)
    return set_error("lsb_batch_graph_capture: needs a created (non-default) stream"), LSB_EINVAL;
  if (b->graph_exec) cudaGraphExecDestroy(b->graph_exec);
  if (b->graph) cudaGraphDestroy(b->graph);
  b->graph_exec = nullptr;
  b->graph = nullptr;
  // one eager step first: kernel attributes (shared-memory limits) and lazily
  // created side streams are set up outside the capture
  lsb_status rc = lsb_step(b, in, out);
  if (rc) return rc;
  LSB_CUDA(cudaStreamSynchronize(ctx->stream));
  const bool prof = b->profile;
  b->profile = false;  // no stage events inside the graph
  const uint64_t before = ctx->launches;
  LSB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  rc = lsb_step(b, in, out);
  cudaGraph_t g = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(ctx->stream, &g);
  b->profile = prof;
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  LSB_CUDA(ee);
  b->graph_kernels = ctx->launches - before;
  ctx->launches = before;
  b->graph = g;
  LSB_CUDA(cudaGraphInstantiate(&b->graph_exec, g, 0));
  return LSB_OK;
}

lsb_status lsb_batch_graph_launch(lsb_batch* b) {
  if (!b || !b->graph_exec) return set_error("lsb_batch_graph_launch: no captured graph"), LSB_EINVAL;
  LSB_CUDA(cudaGraphLaunch(b->graph_exec, b->ctx->stream));
  b->ctx->launches += b->graph_kernels;
  return LSB_OK;
}

}  // extern "C"
