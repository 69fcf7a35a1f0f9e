// capi_stages.cu -- stage-by-stage entry points with host buffers, each the
// device replacement of one reference function. They reuse the fused step's
// kernels (K3/K4/K5) with a one-sentence configuration and synchronise, as
// the reference's by-value API does.
#include <algorithm>
#include <cstring>
#include <vector>

#include <cstdlib>

#include "k_step.cuh"

using namespace lsb;

namespace {

template <class T>
struct Buf {
  T* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)); }
};

#define TRY_ALLOC(buf, n) LSB_CUDA((buf).alloc(n))

}  // namespace

extern "C" {

lsb_status lsb_select_candidates(lsb_ctx* ctx, const int32_t* L_host, int B, uint32_t V, int t,
                                 uint32_t* ids_host, uint32_t* n_out, uint32_t* from_threshold) {
  if (!ctx || B < 0 || !n_out || !from_threshold) return set_error("select_candidates: bad arguments"), LSB_EINVAL;
  if (t < 0) return set_error("select_candidates: negative threshold"), LSB_EINVAL;
  cudaStream_t st = ctx->stream;
  const uint32_t nwords = (V + 31) / 32;
  Buf<int32_t> L;
  Buf<uint32_t> bm, ids, n, prov;
  TRY_ALLOC(L, static_cast<size_t>(B) * V);
  TRY_ALLOC(bm, nwords);
  TRY_ALLOC(ids, V);
  TRY_ALLOC(n, 1);
  TRY_ALLOC(prov, 3);
  if (static_cast<size_t>(B) * V)
    LSB_CUDA(cudaMemcpyAsync(L.p, L_host, static_cast<size_t>(B) * V * 4, cudaMemcpyHostToDevice, st));
  LSB_CUDA(cudaMemsetAsync(bm.p, 0, std::max<uint32_t>(nwords, 1) * 4, st));
  lsb_status rc;
  if (t > 0 && (rc = launch_bitmap_from_dense(ctx, L.p, B, V, t, bm.p))) return rc;
  CompactArgs ca{};
  ca.bitmap_in = bm.p;
  ca.nwords = nwords;
  ca.V = V;
  ca.T = 0;
  ca.mode = t == 0 ? 1 : 0;  // t == 0 keeps every word (src/candidate_selector.cpp:21-27)
  ca.ids = ids.p;
  ca.ncap = V;
  ca.n_cand = n.p;
  ca.prov = prov.p;
  ca.err = ctx->err_dev;
  if ((rc = launch_compact(ctx, ca, 1))) return rc;
  LSB_CUDA(cudaMemcpyAsync(n_out, n.p, 4, cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaStreamSynchronize(st));
  *from_threshold = *n_out;
  if (ids_host && *n_out) {
    if (t == 0) {
      for (uint32_t j = 0; j < V; ++j) ids_host[j] = j;
    } else {
      LSB_CUDA(cudaMemcpy(ids_host, ids.p, *n_out * 4ull, cudaMemcpyDeviceToHost));
    }
  }
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_merge_top_frequent(lsb_ctx* ctx, const uint32_t* ids_host, uint32_t n,
                                  uint32_t from_threshold, uint32_t T,
                                  const uint32_t* specials_host, uint32_t nspec, uint32_t V,
                                  uint32_t* out_host, uint32_t* n_out, uint32_t* prov) {
  if (!ctx || !n_out || !prov) return set_error("merge_top_frequent: bad arguments"), LSB_EINVAL;
  if (T > V) return set_error("merge_top_frequent: T exceeds vocabulary"), LSB_EINVAL;
  std::vector<uint32_t> spec(specials_host, specials_host + nspec);
  std::sort(spec.begin(), spec.end());
  spec.erase(std::unique(spec.begin(), spec.end()), spec.end());
  for (uint32_t id : spec)
    if (id >= V)
      return set_error("merge_top_frequent: special id " + std::to_string(id) + " out of range"),
             LSB_EINVAL;
  for (uint32_t k = 0; k < n; ++k)
    if (ids_host[k] >= V) return set_error("merge_top_frequent: candidate id out of range"), LSB_EINVAL;
  cudaStream_t st = ctx->stream;
  const uint32_t nwords = (V + 31) / 32;
  Buf<uint32_t> in, bm, ids, cnt, pv, sp;
  TRY_ALLOC(in, n);
  TRY_ALLOC(bm, nwords);
  TRY_ALLOC(ids, V);
  TRY_ALLOC(cnt, 1);
  TRY_ALLOC(pv, 3);
  TRY_ALLOC(sp, spec.size());
  if (n) LSB_CUDA(cudaMemcpyAsync(in.p, ids_host, n * 4ull, cudaMemcpyHostToDevice, st));
  if (!spec.empty())
    LSB_CUDA(cudaMemcpyAsync(sp.p, spec.data(), spec.size() * 4, cudaMemcpyHostToDevice, st));
  LSB_CUDA(cudaMemsetAsync(bm.p, 0, std::max<uint32_t>(nwords, 1) * 4, st));
  lsb_status rc;
  if ((rc = launch_bitmap_from_ids(ctx, in.p, n, bm.p))) return rc;
  CompactArgs ca{};
  ca.bitmap_in = bm.p;
  ca.nwords = nwords;
  ca.V = V;
  ca.T = T;
  ca.mode = 0;
  ca.specials = sp.p;
  ca.nspec = static_cast<int>(spec.size());
  ca.ids = ids.p;
  ca.ncap = V;
  ca.n_cand = cnt.p;
  ca.prov = pv.p;
  ca.err = ctx->err_dev;
  if ((rc = launch_compact(ctx, ca, 1))) return rc;
  LSB_CUDA(cudaMemcpyAsync(n_out, cnt.p, 4, cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaMemcpyAsync(prov, pv.p, 12, cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaStreamSynchronize(st));
  prov[0] = from_threshold;  // carried through (src/candidate_selector.cpp:73)
  if (out_host && *n_out) LSB_CUDA(cudaMemcpy(out_host, ids.p, *n_out * 4ull, cudaMemcpyDeviceToHost));
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_gather_embeddings(lsb_ctx* ctx, const lsb_model* model, const uint32_t* ids_host,
                                 uint32_t n, float* out_host) {
  if (!ctx || !model) return set_error("gather_embeddings: bad arguments"), LSB_EINVAL;
  for (uint32_t k = 0; k < n; ++k)
    if (ids_host[k] >= model->V) return set_error("gather_embeddings: id out of range"), LSB_EINVAL;
  if (!n) return LSB_OK;
  cudaStream_t st = ctx->stream;
  Buf<uint32_t> ids;
  Buf<float> out;
  TRY_ALLOC(ids, n);
  TRY_ALLOC(out, static_cast<size_t>(n) * model->d);
  LSB_CUDA(cudaMemcpyAsync(ids.p, ids_host, n * 4ull, cudaMemcpyHostToDevice, st));
  lsb_status rc = launch_gather(ctx, model->E, model->d, ids.p, n, out.p);
  if (rc) return rc;
  LSB_CUDA(cudaMemcpyAsync(out_host, out.p, static_cast<size_t>(n) * model->d * 4,
                           cudaMemcpyDeviceToHost, st));
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_compute_logits(lsb_ctx* ctx, const float* H_host, int rows, const float* Esub_host,
                              int64_t n, int d, lsb_mode mode, float* out_host) {
  if (!ctx || rows < 0 || n < 0 || d < 0) return set_error("compute_logits: bad arguments"), LSB_EINVAL;
  if (rows == 0 || n == 0) return LSB_OK;
  cudaStream_t st = ctx->stream;
  Buf<float> H, E, out;
  TRY_ALLOC(H, static_cast<size_t>(rows) * d);
  TRY_ALLOC(E, static_cast<size_t>(n) * d);
  TRY_ALLOC(out, static_cast<size_t>(rows) * n);
  if (d) {
    LSB_CUDA(cudaMemcpyAsync(H.p, H_host, static_cast<size_t>(rows) * d * 4, cudaMemcpyHostToDevice, st));
    LSB_CUDA(cudaMemcpyAsync(E.p, Esub_host, static_cast<size_t>(n) * d * 4, cudaMemcpyHostToDevice, st));
  }
  if (d == 0) {
    LSB_CUDA(cudaMemsetAsync(out.p, 0, static_cast<size_t>(rows) * n * 4, st));
  } else {
    LogitsArgs la{};
    la.H = H.p;
    la.d = d;
    la.R_total = rows;
    la.Bsent = std::min(rows, 16);
    la.E = E.p;
    la.n_shared = static_cast<uint32_t>(n);
    la.S = 0;
    la.out = out.p;
    la.ldo = static_cast<size_t>(n);
    lsb_status rc = launch_logits(ctx, la, mode, ctx->sm_count * 8);
    if (rc) return rc;
  }
  LSB_CUDA(cudaMemcpyAsync(out_host, out.p, static_cast<size_t>(rows) * n * 4, cudaMemcpyDeviceToHost, st));
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_softmax_rows(lsb_ctx* ctx, const float* logits_host, int rows, int64_t n,
                            float* out_host) {
  if (!ctx || rows < 0 || n < 0) return set_error("softmax_rows: bad arguments"), LSB_EINVAL;
  if (rows == 0) return LSB_OK;
  if (n == 0) return set_error("softmax_rows: row without finite entries"), LSB_EINVAL;
  cudaStream_t st = ctx->stream;
  Buf<float> L;
  Buf<TopEntry> top;
  Buf<int32_t> topn;
  TRY_ALLOC(L, static_cast<size_t>(rows) * n);
  TRY_ALLOC(top, rows);
  TRY_ALLOC(topn, rows);
  LSB_CUDA(cudaMemcpyAsync(L.p, logits_host, static_cast<size_t>(rows) * n * 4, cudaMemcpyHostToDevice, st));
  SoftmaxArgs sa{};
  sa.logits = L.p;
  sa.ldl = static_cast<size_t>(n);
  sa.R_total = rows;
  sa.Bsent = 1;
  sa.topB = 1;
  sa.n_const = static_cast<uint32_t>(n);
  sa.keep_probs = 1;
  sa.top = top.p;
  sa.top_n = topn.p;
  sa.err = ctx->err_dev;
  sa.seq_denominator = getenv("LSB_SEQ_DENOM") && atoi(getenv("LSB_SEQ_DENOM")) == 1;
  lsb_status rc = launch_softmax(ctx, sa);
  if (rc) return rc;
  LSB_CUDA(cudaMemcpyAsync(out_host, L.p, static_cast<size_t>(rows) * n * 4, cudaMemcpyDeviceToHost, st));
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_expand_beams(lsb_ctx* ctx, const float* probs_host, int rows, int64_t n,
                            const double* cum_host, const uint32_t* live_host,
                            const lsb_choice* frozen_host, int nfrozen, int B,
                            const uint32_t* id_map_host, lsb_choice* out_host, int* n_out) {
  if (!ctx || rows < 0 || n < 0 || nfrozen < 0 || !n_out) return set_error("expand_beams: bad arguments"), LSB_EINVAL;
  if (B < 0) return set_error("expand_beams: negative beam"), LSB_EINVAL;
  if (B > 256) return set_error("expand_beams: beam above 256 is not supported"), LSB_EINVAL;
  cudaStream_t st = ctx->stream;
  const int R = std::max(rows, 1);
  Buf<float> P;
  Buf<double> cum, fzs;
  Buf<uint32_t> live, fzb, idm;
  Buf<TopEntry> top;
  Buf<int32_t> topn, nc;
  Buf<lsb_choice> ch;
  TRY_ALLOC(P, static_cast<size_t>(R) * std::max<int64_t>(n, 1));
  TRY_ALLOC(cum, R);
  TRY_ALLOC(live, R);
  TRY_ALLOC(fzs, nfrozen);
  TRY_ALLOC(fzb, nfrozen);
  TRY_ALLOC(idm, n);
  TRY_ALLOC(top, static_cast<size_t>(R) * std::max(B, 1));
  TRY_ALLOC(topn, R);
  TRY_ALLOC(nc, 1);
  TRY_ALLOC(ch, std::max(B, 1));
  if (rows && n)
    LSB_CUDA(cudaMemcpyAsync(P.p, probs_host, static_cast<size_t>(rows) * n * 4, cudaMemcpyHostToDevice, st));
  if (rows) {
    LSB_CUDA(cudaMemcpyAsync(cum.p, cum_host, rows * 8ull, cudaMemcpyHostToDevice, st));
    LSB_CUDA(cudaMemcpyAsync(live.p, live_host, rows * 4ull, cudaMemcpyHostToDevice, st));
  }
  std::vector<double> fs(nfrozen);
  std::vector<uint32_t> fb(nfrozen);
  for (int f = 0; f < nfrozen; ++f) {
    fs[f] = frozen_host[f].score;
    fb[f] = frozen_host[f].beam;
  }
  if (nfrozen) {
    LSB_CUDA(cudaMemcpyAsync(fzs.p, fs.data(), nfrozen * 8ull, cudaMemcpyHostToDevice, st));
    LSB_CUDA(cudaMemcpyAsync(fzb.p, fb.data(), nfrozen * 4ull, cudaMemcpyHostToDevice, st));
  }
  if (id_map_host && n)
    LSB_CUDA(cudaMemcpyAsync(idm.p, id_map_host, n * 4ull, cudaMemcpyHostToDevice, st));
  lsb_status rc;
  SoftmaxArgs sa{};
  sa.logits = P.p;
  sa.ldl = static_cast<size_t>(n);
  sa.R_total = rows;
  sa.Bsent = R;
  sa.topB = B;
  sa.n_const = static_cast<uint32_t>(n);
  sa.probs_in = 1;
  sa.top = top.p;
  sa.top_n = topn.p;
  sa.err = ctx->err_dev;
  if (rows && (rc = launch_softmax(ctx, sa))) return rc;
  ExpandArgs ea{};
  ea.S = 1;
  ea.Bsent = rows;
  ea.topB = B;
  ea.top = top.p;
  ea.top_n = topn.p;
  ea.scores = cum.p;
  ea.live_ids = live.p;
  ea.n_shared = static_cast<uint32_t>(n);
  ea.id_map = id_map_host && n ? idm.p : nullptr;
  ea.choices = ch.p;
  ea.n_choices = nc.p;
  ea.frozen_mode = 1;
  ea.fz_score = fzs.p;
  ea.fz_beam = fzb.p;
  ea.nfrozen = nfrozen;
  if ((rc = launch_expand(ctx, ea))) return rc;
  int32_t cnt = 0;
  LSB_CUDA(cudaMemcpyAsync(&cnt, nc.p, 4, cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaStreamSynchronize(st));
  *n_out = cnt;
  if (cnt) LSB_CUDA(cudaMemcpy(out_host, ch.p, cnt * sizeof(lsb_choice), cudaMemcpyDeviceToHost));
  return lsb_ctx_sync(ctx);
}

}  // extern "C"
