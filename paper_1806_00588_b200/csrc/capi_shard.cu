// capi_shard.cu -- one rank's share of a VOCABULARY-SHARDED decode step
// (BASELINE cfg 4). Rank g owns the contiguous vocabulary
// slice [v_g, v_g + n_g) of E with its own band index over the slice (same
// permutations: a word's codes, hence its hit counts, do not depend on the
// other words). The row softmax and the beam expansion need the whole row,
// so a step is three device phases separated by two small all-gathers:
//
//   phase 1  K1+K2 -> K3 -> K4 on the slice; per row the local max m_g.
//   [all-gather m_g]                                   S*B floats per rank
//   phase 2  global m = max_g m_g; e = exp((double)l - m) kept as float(e)
//            (exactly the reference's values, src/beam_decoder.cpp:56-64);
//            local sum s_g (double); local top-B' by (e desc, word asc).
//   [all-gather s_g, top-B' lists]                     S*B*(8 + 8*B') bytes
//   phase 3  denominator = sum_g s_g in fixed rank order; p = e * float(1/denom);
//            per row top-B by (p desc, word asc) over the gathered lists; then
//            the reference expansion (K5b) and the hidden reorder, identically
//            on every rank (hidden states are replicated).
//
// B' = B + kShardSlack: selecting by e and re-ranking by p is exact unless
// more than kShardSlack entries of one rank tie in p with the B-th winner.
#include <algorithm>
#include <cfloat>

#include "batch.cuh"
#include "glibc_log.cuh"

namespace lsb {

constexpr int kShardSlack = 4;
constexpr int kShT = 128;

__global__ void __launch_bounds__(kShT) k_shard_rowmax(const float* __restrict__ logits, size_t ldl,
                                                       const uint32_t* __restrict__ n_cand, int Bsent,
                                                       const uint8_t* finished, const int32_t* n_hyp,
                                                       float* __restrict__ rowmax) {
  __shared__ float red[kShT / 32];
  const int row = blockIdx.x, s = row / Bsent, i = row % Bsent;
  const bool live = !(n_hyp && i >= n_hyp[s]) && !(finished && finished[row]);
  const uint32_t n = live ? n_cand[s] : 0;
  const float* L = logits + static_cast<size_t>(row) * ldl;
  float mx = -INFINITY;
  for (uint32_t r = threadIdx.x; r < n; r += kShT) {
    const float v = L[r];
    mx = (mx < v) ? v : mx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (mx < y) ? y : mx;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kShT / 32; ++w) mx = (mx < red[w]) ? red[w] : mx;
    rowmax[row] = red[0] < mx ? mx : red[0];
  }
}

__global__ void __launch_bounds__(kShT) k_shard_exp(float* __restrict__ logits, size_t ldl,
                                                    const uint32_t* __restrict__ n_cand, int Bsent,
                                                    int R, const uint8_t* finished,
                                                    const int32_t* n_hyp,
                                                    const float* __restrict__ allmax, int G,
                                                    double* __restrict__ rowsum) {
  __shared__ double red[kShT / 32];
  __shared__ unsigned long long exptab[256];
  stage_exp_table(exptab);
  __syncthreads();
  const int row = blockIdx.x, s = row / Bsent, i = row % Bsent;
  const bool live = !(n_hyp && i >= n_hyp[s]) && !(finished && finished[row]);
  const uint32_t n = live ? n_cand[s] : 0;
  float m = -INFINITY;
  for (int g = 0; g < G; ++g) {
    const float v = allmax[static_cast<size_t>(g) * R + row];
    m = (m < v) ? v : m;
  }
  float* L = logits + static_cast<size_t>(row) * ldl;
  double sum = 0.0;
  if (!(isinf(m) && m < 0)) {
    const double dm = static_cast<double>(m);
    for (uint32_t r = threadIdx.x; r < n; r += kShT) {
      const double e = glibc_exp_smem(static_cast<double>(L[r]) - dm, exptab);
      L[r] = static_cast<float>(e);
      sum += e;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kShT / 32; ++w) t += red[w];
    rowsum[row] = t;
  }
}

// TopEntry{e, column} -> lsb_shard_top{e, global word}; unused slots e = -1.
__global__ void k_shard_pack(const TopEntry* __restrict__ top, const int32_t* __restrict__ top_n,
                             int R, int Bp, int Bsent, const uint32_t* __restrict__ ids,
                             size_t ncap, uint32_t n_shared, int identity, uint32_t word_base,
                             lsb_shard_top* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= R * Bp) return;
  const int row = q / Bp, k = q % Bp;
  lsb_shard_top o{-1.0f, 0xFFFFFFFFu};
  if (k < top_n[row]) {
    const TopEntry t = top[q];
    const int s = row / Bsent;
    const uint32_t local = (identity || t.r < n_shared) ? t.r : ids[static_cast<size_t>(s) * ncap + t.r];
    o.e = t.p;
    o.word = word_base + local;
  }
  out[q] = o;
}

// Phase 3 selection: per row, p = fl(e * inv) for the G*B' gathered entries,
// top-B by (p desc, word asc) via ranks (entries are distinct words).
// Rank g's sums start at allsum + g * rank_stride and its lists at
// alltop + g * rank_stride (strides in 8-byte words: separate gathers use
// R and R * Bp; the packed layout R + R * Bp for both).
__global__ void __launch_bounds__(kShT) k_shard_combine(const double* __restrict__ allsum,
                                                        const lsb_shard_top* __restrict__ alltop,
                                                        size_t sum_stride, size_t top_stride,
                                                        int G, int R, int Bp, int B, int Bsent,
                                                        const uint8_t* finished, const int32_t* n_hyp,
                                                        TopEntry* __restrict__ top,
                                                        int32_t* __restrict__ top_n, uint32_t* err) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* sp = reinterpret_cast<float*>(smem);
  uint32_t* sw = reinterpret_cast<uint32_t*>(sp + G * Bp);
  __shared__ int s_cnt;
  const int row = blockIdx.x, s = row / Bsent, i = row % Bsent;
  const bool live = !(n_hyp && i >= n_hyp[s]) && !(finished && finished[row]);
  if (!live) {
    if (threadIdx.x == 0) top_n[row] = 0;
    return;
  }
  double denom = 0.0;
  for (int g = 0; g < G; ++g) denom += allsum[g * sum_stride + row];  // rank order
  if (!(denom > 0.0)) {
    if (threadIdx.x == 0) {
      atomicOr(err, kErrEmptyRow);
      top_n[row] = 0;
    }
    return;
  }
  const float inv = static_cast<float>(1.0 / denom);
  const int n = G * Bp;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < n; q += kShT) {
    const lsb_shard_top t = alltop[(q / Bp) * top_stride + static_cast<size_t>(row) * Bp + q % Bp];
    const bool ok = t.e >= 0.0f;
    sp[q] = ok ? __fmul_rn(t.e, inv) : -1.0f;
    sw[q] = t.word;
    if (ok) atomicAdd(&s_cnt, 1);
  }
  __syncthreads();
  const int keep = min(B, s_cnt);
  for (int q = threadIdx.x; q < n; q += kShT) {
    const float p = sp[q];
    if (p < 0.0f) continue;
    const uint32_t w = sw[q];
    int rank = 0;
    for (int j = 0; j < n && rank < keep; ++j) {
      const float pj = sp[j];
      rank += (pj > p) || (pj == p && sw[j] < w);
    }
    if (rank < keep) top[static_cast<size_t>(row) * B + rank] = TopEntry{p, w};
  }
  if (threadIdx.x == 0) top_n[row] = keep;
}

}  // namespace lsb

using namespace lsb;

// Allocates the phase-2 scratch of a shard batch (first phase-2 call, or
// up front: the peer exchange must not allocate -- cudaMalloc synchronises the
// device while a flag-wait kernel may be spinning on another rank's push).
lsb_status lsb::ensure_shard_scratch(lsb_batch* b, int G) {
  const size_t R = static_cast<size_t>(b->S) * b->B;
  const int Bp = b->B + kShardSlack;
  if (!b->sh_top) {
    LSB_CUDA(cudaMalloc(&b->sh_top, R * Bp * sizeof(TopEntry)));
    LSB_CUDA(cudaMalloc(&b->sh_topn, R * sizeof(int32_t)));
  }
  (void)G;
  return LSB_OK;
}

namespace {

bool live_args(const lsb_batch* b, const lsb_state_dev* in) {
  return b && in && in->hidden && in->scores;
}

}  // namespace

extern "C" {

int lsb_shard_width(const lsb_batch* b) { return b ? b->B + kShardSlack : 0; }

lsb_status lsb_shard_phase1(lsb_batch* b, const lsb_state_dev* in, float* rowmax_dev) {
  if (!live_args(b, in) || !rowmax_dev) return set_error("lsb_shard_phase1: bad arguments"), LSB_EINVAL;
  if (b->cmode == 2) return set_error("lsb_shard_phase1: use a slice model, not kFull"), LSB_EINVAL;
  lsb_status rc = step_front(b, in, /*empty_is_error=*/0);
  if (rc) return rc;
  const int R = b->S * b->B;
  k_shard_rowmax<<<R, kShT, 0, b->ctx->stream>>>(b->logits, b->ncap, b->n_cand, b->B, in->finished,
                                                  in->n_hyp, rowmax_dev);
  LSB_LAUNCHED(b->ctx, "k_shard_rowmax");
  b->last = *in;
  b->has_last = true;
  return LSB_OK;
}

lsb_status lsb_shard_phase2(lsb_batch* b, const lsb_state_dev* in, const float* allmax_dev, int G,
                            uint32_t word_base, double* rowsum_dev, lsb_shard_top* top_dev) {
  if (!live_args(b, in) || !allmax_dev || G < 1 || !rowsum_dev || !top_dev)
    return set_error("lsb_shard_phase2: bad arguments"), LSB_EINVAL;
  lsb_status rc = ensure_shard_scratch(b, G);
  if (rc) return rc;
  lsb_ctx* ctx = b->ctx;
  const int R = b->S * b->B;
  const int Bp = b->B + kShardSlack;
  k_shard_exp<<<R, kShT, 0, ctx->stream>>>(b->logits, b->ncap, b->n_cand, b->B, R, in->finished,
                                            in->n_hyp, allmax_dev, G, rowsum_dev);
  LSB_LAUNCHED(ctx, "k_shard_exp");
  // local top-B' by (e desc, column asc) = (e desc, word asc): K5a in
  // selection-only mode over the exponentials
  SoftmaxArgs sa{};
  sa.logits = b->logits;
  sa.ldl = b->ncap;
  sa.R_total = R;
  sa.Bsent = b->B;
  sa.topB = Bp;
  sa.n_cand = b->n_cand;
  sa.probs_in = 1;
  sa.finished = in->finished;
  sa.n_hyp = in->n_hyp;
  sa.top = b->sh_top;
  sa.top_n = b->sh_topn;
  sa.err = ctx->err_dev;
  if ((rc = launch_softmax(ctx, sa))) return rc;
  const int total = R * Bp;
  k_shard_pack<<<(total + 255) / 256, 256, 0, ctx->stream>>>(
      b->sh_top, b->sh_topn, R, Bp, b->B, b->ids, b->ncap, b->n_shared, b->cmode != 0 ? 1 : 0,
      word_base, top_dev);
  LSB_LAUNCHED(ctx, "k_shard_pack");
  return LSB_OK;
}

static lsb_status shard_phase3(lsb_batch* b, const lsb_state_dev* in, const double* allsum_dev,
                               const lsb_shard_top* alltop_dev, size_t sum_stride,
                               size_t top_stride, int G, const lsb_out_dev* out) {
  lsb_ctx* ctx = b->ctx;
  const int R = b->S * b->B;
  const int Bp = b->B + kShardSlack;
  const size_t smem = static_cast<size_t>(G) * Bp * 8;
  if (smem > ctx->smem_optin) return set_error("lsb_shard_phase3: too many shards"), LSB_EINVAL;
  if (lsb_status rc = ensure_smem(ctx, k_shard_combine, smem)) return rc;
  k_shard_combine<<<R, kShT, smem, ctx->stream>>>(allsum_dev, alltop_dev, sum_stride, top_stride,
                                                   G, R, Bp, b->B, b->B, in->finished, in->n_hyp,
                                                   b->top, b->top_n, ctx->err_dev);
  LSB_LAUNCHED(ctx, "k_shard_combine");
  // profiled steps: phase 1 recorded stage events 0..3 (step_front); the
  // softmax stage spans phase 2 + the exchange + the combine
  if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[4], ctx->stream));
  ExpandArgs ea{};
  ea.S = b->S;
  ea.Bsent = b->B;
  ea.topB = b->B;
  ea.top = b->top;
  ea.top_n = b->top_n;
  ea.scores = in->scores;
  ea.finished = in->finished;
  ea.n_hyp = in->n_hyp;
  ea.ids = nullptr;  // entries already carry global word ids
  ea.n_shared = 0xFFFFFFFFu;
  ea.hidden = in->hidden;
  ea.d = b->d;
  ea.hidden_out = out->hidden_out;
  ea.choices = out->choices;
  ea.n_choices = out->n_choices;
  lsb_status rc = launch_expand(ctx, ea);
  if (rc) return rc;
  if (b->rec) LSB_CUDA(cudaEventRecord(b->ev[5], ctx->stream));
  return LSB_OK;
}

lsb_status lsb_shard_phase3(lsb_batch* b, const lsb_state_dev* in, const double* allsum_dev,
                            const lsb_shard_top* alltop_dev, int G, const lsb_out_dev* out) {
  if (!live_args(b, in) || !allsum_dev || !alltop_dev || G < 1 || !out || !out->choices ||
      !out->n_choices)
    return set_error("lsb_shard_phase3: bad arguments"), LSB_EINVAL;
  const size_t R = static_cast<size_t>(b->S) * b->B;
  return shard_phase3(b, in, allsum_dev, alltop_dev, R, R * (b->B + kShardSlack), G, out);
}

lsb_status lsb_shard_phase3_packed(lsb_batch* b, const lsb_state_dev* in, const void* packed_dev,
                                   int G, const lsb_out_dev* out) {
  if (!live_args(b, in) || !packed_dev || G < 1 || !out || !out->choices || !out->n_choices)
    return set_error("lsb_shard_phase3_packed: bad arguments"), LSB_EINVAL;
  const size_t R = static_cast<size_t>(b->S) * b->B;
  const size_t stride = R + R * (b->B + kShardSlack);  // 8-byte words per rank
  const double* sums = static_cast<const double*>(packed_dev);
  return shard_phase3(b, in, sums, reinterpret_cast<const lsb_shard_top*>(sums + R), stride,
                      stride, G, out);
}

}  // extern "C"
