// k_select.cu -- K5: reduced softmax normalisation, per-row top-B and the
// per-sentence beam expansion with the hidden-state reorder.
//
//  K5a k_softmax_topb : one 128-thread CTA per hypothesis row. softmax_rows
//      (src/beam_decoder.cpp:46-74): float max; e = exp((double)l - mx) kept
//      as float(e); double denominator (a tree, certified equal to the
//      reference's sequential sum or redone sequentially: softmax_denom.cuh);
//      p = float(e) * float(1/denom). Then the row's top-B by (p desc, column
//      asc): per-thread sorted lists (columns ascend within a thread, so equal
//      p never displaces an earlier column) merged by B rounds of a block-wide
//      arg-max; the owner of a winning column is column % 128.
//  K5b k_expand       : one CTA per sentence. expand_beams
//      (src/beam_decoder.cpp:76-111): the candidates are the per-row top-B
//      lists (score = cum + log((double)p), sorted by the reference
//      comparator score desc, beam asc, word asc) plus the frozen hypotheses.
//      Every candidate's global rank is its position in its own list plus,
//      per other list, a binary search for how many of that list's entries
//      beat it; ranks < B are written in place. No serial tournament. Then
//      each chosen child copies its parent's hidden vector (the paper's
//      hidden-state reorder), replacing the D2H copy + CPU
//      heapsort of the paper's pipeline.
//      k_expand_tournament keeps a B-round warp tournament for stage-API
//      calls with more lists than the rank kernel holds in shared memory.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "glibc_log.cuh"
#include "k_step.cuh"
#include "softmax_denom.cuh"

namespace lsb {

constexpr int kSelT = 128;  // threads per row CTA

__device__ __forceinline__ bool top_better(float pa, uint32_t ra, float pb, uint32_t rb) {
  return pa > pb || (pa == pb && ra < rb);
}

// Block-wide reduction through red[kSelT / 32]. FIRST: red is used for the
// first time in this CTA, so no barrier is needed before overwriting it.
template <class T, class Op, bool FIRST = false>
__device__ __forceinline__ T block_reduce(T v, T* red, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if constexpr (!FIRST) __syncthreads();  // red[] may still be read from a previous reduction
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = red[0];
#pragma unroll
  for (int w = 1; w < kSelT / 32; ++w) v = op(v, red[w]);
  return v;
}

struct FMaxOp {
  __device__ float operator()(float x, float y) const { return (x < y) ? y : x; }
};
struct DSumOp {
  __device__ double operator()(double x, double y) const { return x + y; }
};
// log((double) p) of a row probability as the reference's host libm
// computes it (glibc_log.cuh: bit for bit; CUDA's log() is within 1 ulp and
// differed on one score of a test step); the score is then
// __dadd_rn(cum, log_p(p)), never contracted.
static __device__ __forceinline__ double log_p(float p) { return glibc_log(static_cast<double>(p)); }

static __device__ constexpr FMaxOp fmax_op{};
static __device__ constexpr DSumOp dsum_op{};

// The K-th largest of the CTA's kSelT per-thread values x (-1 = none): each
// warp sorts its 32 with a shuffle bitonic network, every lane ranks its value
// against the other warps' sorted lists in (value desc, position asc) order.
// K lanes hold an entry >= the result, so it bounds the row's K-th largest
// from below. Returns -1 when K > kSelT. Contains barriers (whole CTA); call
// it at most once per CTA (its shared scratch is not protected for reuse).
__device__ __forceinline__ float kth_lane_max(float x, int K) {
  __shared__ float s_lm[kSelT];
  __shared__ float s_tau;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1)  // bitonic sort, descending
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const float y = __shfl_xor_sync(0xffffffffu, x, stride);
      const bool up = ((lane & size) == 0) == ((lane & stride) == 0);
      x = up ? fmaxf(x, y) : fminf(x, y);
    }
  if (K <= 32) {
    // cheaper, looser bound: each warp's K-th largest (K lanes of that warp
    // hold an entry >= it), maximised over the warps
    const float kw = __shfl_sync(0xffffffffu, x, K - 1);
    if (lane == 0) s_lm[warp] = kw;
    __syncthreads();
    float t = s_lm[0];
#pragma unroll
    for (int w = 1; w < kSelT / 32; ++w) t = fmaxf(t, s_lm[w]);
    return t;
  }
  s_lm[tid] = x;
  if (tid == 0) s_tau = -1.0f;
  __syncthreads();
  if (K <= kSelT) {
    int rank = lane;
#pragma unroll
    for (int w = 0; w < kSelT / 32; ++w) {
      if (w == warp) continue;
      const float* l = s_lm + w * 32;
      int lo = 0, hi = 32;  // entries of l before me: > x, or >= x for earlier warps
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const bool before = w < warp ? l[mid] >= x : l[mid] > x;
        if (before) lo = mid + 1;
        else hi = mid;
      }
      rank += lo;
    }
    if (rank == K - 1) s_tau = x;
  }
  __syncthreads();
  return s_tau;
}


// The reference's softmax denominator: softmax_denom.cuh.

// Rows of at most kSelT * kSelReg candidates (the LSH step's): the row lives
// in registers, kSelReg values per thread -- one global read, no exp/prob
// round trips through L2 -- and the top-B is B rounds of a block-wide
// arg-max by (p desc, column asc) in which only the owner of the winning
// column rescans its registers. Same arithmetic as the general path.
constexpr int kSelReg = 24;
constexpr int kSelCand = 256;  // threshold survivors ranked directly

template <int REG>
__device__ __forceinline__ void row_registers(const SoftmaxArgs& a, int row, float* L, uint32_t n,
                                              float* red_f, double* red_d,
                                              const unsigned long long* exptab) {
  __shared__ float win_p[2][kSelT / 32];
  __shared__ uint32_t win_r[2][kSelT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = a.topB;
  float v[REG];
  float mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < REG; ++k) {
    const uint32_t c = tid + kSelT * k;
    v[k] = c < n ? L[c] : -INFINITY;
    mx = (mx < v[k]) ? v[k] : mx;
  }
  mx = block_reduce<float, decltype(fmax_op), true>(mx, red_f, fmax_op);
  if (n == 0 || (isinf(mx) && mx < 0)) {
    if (tid == 0) {
      atomicOr(a.err, kErrEmptyRow);
      a.top_n[row] = 0;
    }
    return;
  }
  const double dmx = static_cast<double>(mx);
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < REG; ++k) {
    if (tid + kSelT * k < n) {
      const double e = glibc_exp_smem(static_cast<double>(v[k]) - dmx, exptab);
      v[k] = static_cast<float>(e);
      sum += e;
    }
  }
  sum = block_reduce<double, decltype(dsum_op), true>(sum, red_d, dsum_op);
  const float inv = reference_inv_cta<kSelT>(sum, n, L, dmx, a.seq_denominator);
#pragma unroll
  for (int k = 0; k < REG; ++k) {
    const uint32_t c = tid + kSelT * k;
    if (c < n) {
      v[k] = __fmul_rn(v[k], inv);
      if (a.keep_probs) L[c] = v[k];
    } else {
      v[k] = -1.0f;
    }
  }
  // Threshold filter: only entries >= tau (the B-th largest lane maximum,
  // kth_lane_max) can be in the top-B. Usually a few dozen survive; all
  // threads rank them exactly by (p desc, column asc).
  {
    __shared__ int s_nc;
    __shared__ float c_p[kSelCand];
    __shared__ uint32_t c_c[kSelCand];
    float x = -1.0f;
#pragma unroll
    for (int k = 0; k < REG; ++k) x = fmaxf(x, v[k]);
    if (tid == 0) s_nc = 0;  // published by kth_lane_max's barriers
    const float tau_k = kth_lane_max(x, B);
    const float tau = fmaxf(tau_k, 0.0f);  // valid entries are >= 0, padding -1
#pragma unroll
    for (int k = 0; k < REG; ++k)
      if (v[k] >= tau) {
        const int at = atomicAdd(&s_nc, 1);
        if (at < kSelCand) {
          c_p[at] = v[k];
          c_c[at] = tid + kSelT * k;
        }
      }
    __syncthreads();
    pdl_trigger();
    const int nc = s_nc;
    const int keep = static_cast<int>(min(static_cast<uint32_t>(B), n));
    if (nc <= kSelCand) {
      TopEntry* out = a.top + static_cast<size_t>(row) * B;
      for (int q = tid; q < nc; q += kSelT) {
        const float p = c_p[q];
        const uint32_t c = c_c[q];
        int rank = 0;
        for (int j = 0; j < nc; ++j) rank += top_better(c_p[j], c_c[j], p, c);
        if (rank < keep) out[rank] = TopEntry{p, c};
      }
      if (tid == 0) a.top_n[row] = keep;
      return;
    }
    // (many ties at the threshold: fall through to the round-based merge)
  }
  float bp = -1.0f;
  int bk = 0;
#pragma unroll
  for (int k = 0; k < REG; ++k)
    if (v[k] > bp) {
      bp = v[k];
      bk = k;
    }
  TopEntry* out = a.top + static_cast<size_t>(row) * B;
  const int keep = static_cast<int>(min(static_cast<uint32_t>(B), n));
  for (int r = 0; r < keep; ++r) {
    float p = bp;
    uint32_t c = bp >= 0.0f ? tid + kSelT * static_cast<uint32_t>(bk) : 0xFFFFFFFFu;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float yp = __shfl_xor_sync(0xffffffffu, p, o);
      const uint32_t yc = __shfl_xor_sync(0xffffffffu, c, o);
      if (top_better(yp, yc, p, c)) {
        p = yp;
        c = yc;
      }
    }
    const int buf = r & 1;  // double-buffered winners: one barrier per round
    if (lane == 0) {
      win_p[buf][warp] = p;
      win_r[buf][warp] = c;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kSelT / 32; ++w)
      if (top_better(win_p[buf][w], win_r[buf][w], p, c)) {
        p = win_p[buf][w];
        c = win_r[buf][w];
      }
    if (tid == 0) out[r] = TopEntry{p, c};
    if (c % kSelT == static_cast<uint32_t>(tid)) {  // the owner drops it and rescans
#pragma unroll
      for (int k = 0; k < REG; ++k)
        if (k == bk) v[k] = -1.0f;
      bp = -1.0f;
      bk = 0;
#pragma unroll
      for (int k = 0; k < REG; ++k)
        if (v[k] > bp) {
          bp = v[k];
          bk = k;
        }
    }
  }
  if (tid == 0) a.top_n[row] = keep;
}

// ===================================================================== K5a
// One row's softmax + top-B by a 128-thread CTA (k_softmax_topb: a CTA per
// row; the fused small-batch step calls it from persistent CTAs).
static __device__ void softmax_row(const SoftmaxArgs& a, int row) {
  __shared__ float red_f[kSelT / 32];
  __shared__ double red_d[kSelT / 32];
  __shared__ float win_p[kSelT / 32];
  __shared__ uint32_t win_r[kSelT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = row / a.Bsent, i = row % a.Bsent;
  const bool live = !(a.n_hyp && i >= a.n_hyp[s]) && !(a.finished && a.finished[row]);
  if (!live) {
    if (tid == 0) a.top_n[row] = 0;
    return;
  }
  const int B = a.topB;
  const uint32_t n = a.n_cand ? a.n_cand[s] : a.n_const;
  float* L = a.logits + static_cast<size_t>(row) * a.ldl;
  // exp's 2^(i/128) table in shared memory (published by the max reduction's
  // barrier before the first exp)
  __shared__ unsigned long long s_exptab[256];
  stage_exp_table(s_exptab);
  if (!a.probs_in && n <= kSelT * kSelReg && B > 0) {
    if (n <= kSelT * 16) row_registers<16>(a, row, L, n, red_f, red_d, s_exptab);
    else row_registers<kSelReg>(a, row, L, n, red_f, red_d, s_exptab);
    return;
  }
  float inv = 1.0f;
  if (!a.probs_in) {
    // float max, as std::max over the row (src/beam_decoder.cpp:55)
    float mx = -INFINITY;
    for (uint32_t r = tid; r < n; r += kSelT) {
      const float v = L[r];
      mx = (mx < v) ? v : mx;
    }
    mx = block_reduce<float, decltype(fmax_op), true>(mx, red_f, fmax_op);
    if (n == 0 || (isinf(mx) && mx < 0)) {
      if (tid == 0) {
        atomicOr(a.err, kErrEmptyRow);
        a.top_n[row] = 0;
      }
      return;
    }
    const double dmx = static_cast<double>(mx);
    double sum = 0.0;
    for (uint32_t r = tid; r < n; r += kSelT)
      sum += glibc_exp_smem(static_cast<double>(L[r]) - dmx, s_exptab);
    sum = block_reduce<double, decltype(dsum_op), true>(sum, red_d, dsum_op);
    inv = reference_inv_cta<kSelT>(sum, n, L, dmx, a.seq_denominator);
    // (the logits are needed until inv is known: float(e) replaces them now)
    for (uint32_t r = tid; r < n; r += kSelT)
      L[r] = static_cast<float>(glibc_exp_smem(static_cast<double>(L[r]) - dmx, s_exptab));
  }
  if (B <= 0) {
    if (tid == 0) a.top_n[row] = 0;
    return;
  }
  // Rows longer than the register path (or probabilities given): the same
  // threshold selection over global memory. Pass 1 forms p (written back when
  // requested) and each thread's maximum; tau = the B-th largest of those
  // maxima bounds the row's B-th largest p from below.
  const bool pw = a.probs_in || a.keep_probs;  // L holds p after pass 1
  auto p_at = [&](uint32_t r) { return pw ? L[r] : __fmul_rn(L[r], inv); };
  float x = -1.0f;
  for (uint32_t r = tid; r < n; r += kSelT) {
    const float p = a.probs_in ? L[r] : __fmul_rn(L[r], inv);
    if (a.keep_probs && !a.probs_in) L[r] = p;
    x = fmaxf(x, p);
  }
  __shared__ int s_nc;
  __shared__ float c_p[kSelCand];
  __shared__ uint32_t c_c[kSelCand];
  if (tid == 0) s_nc = 0;  // published by kth_lane_max's barriers
  const float tau = kth_lane_max(x, B);
  const int keep = static_cast<int>(min(static_cast<uint32_t>(B), n));
  TopEntry* out = a.top + static_cast<size_t>(row) * B;
  // pass 2: survivors p >= tau (tau > 0), or every positive p (tau <= 0:
  // fewer than B threads saw a positive p; zeros then fill by column)
  for (uint32_t r = tid; r < n; r += kSelT) {
    const float p = p_at(r);
    if (tau > 0.0f ? p >= tau : p > 0.0f) {
      const int at = atomicAdd(&s_nc, 1);
      if (at < kSelCand) {
        c_p[at] = p;
        c_c[at] = r;
      }
    }
  }
  __syncthreads();
  const int nc = s_nc;
  if (nc <= kSelCand) {
    for (int q = tid; q < nc; q += kSelT) {
      const float p = c_p[q];
      const uint32_t c = c_c[q];
      int rank = 0;
      for (int j = 0; j < nc; ++j) rank += top_better(c_p[j], c_c[j], p, c);
      if (rank < keep) out[rank] = TopEntry{p, c};
    }
    // zeros, by ascending column, after every positive p
    int filled = min(nc, keep);
    for (uint32_t base = 0; filled < keep && base < n; base += kSelT) {
      const uint32_t r = base + tid;
      const bool z = r < n && !(p_at(r) > 0.0f);
      const unsigned bal = __ballot_sync(0xffffffffu, z);
      if (lane == 0) win_r[warp] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kSelT / 32; ++w) {
        before += w < warp ? static_cast<int>(win_r[w]) : 0;
        total += static_cast<int>(win_r[w]);
      }
      const int pos = filled + before + __popc(bal & ((1u << lane) - 1u));
      if (z && pos < keep) out[pos] = TopEntry{p_at(r), r};
      filled += total;
      __syncthreads();
    }
    if (tid == 0) a.top_n[row] = keep;
    return;
  }
  // many ties at tau: keep rounds of a block-wide arg-max below the last key
  float lp = INFINITY;
  uint32_t lc = 0;
  for (int k = 0; k < keep; ++k) {
    float bp = -1.0f;
    uint32_t br = 0xFFFFFFFFu;
    for (uint32_t r = tid; r < n; r += kSelT) {
      const float p = p_at(r);
      if (top_better(lp, lc, p, r) && top_better(p, r, bp, br)) {
        bp = p;
        br = r;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float yp = __shfl_xor_sync(0xffffffffu, bp, o);
      const uint32_t yr = __shfl_xor_sync(0xffffffffu, br, o);
      if (top_better(yp, yr, bp, br)) {
        bp = yp;
        br = yr;
      }
    }
    if (lane == 0) {
      win_p[warp] = bp;
      win_r[warp] = br;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kSelT / 32; ++w)
      if (top_better(win_p[w], win_r[w], bp, br)) {
        bp = win_p[w];
        br = win_r[w];
      }
    if (tid == 0) out[k] = TopEntry{bp, br};
    lp = bp;
    lc = br;
    __syncthreads();
  }
  if (tid == 0) a.top_n[row] = keep;
}

#ifndef LSB_BODIES_ONLY  // (k_step_fused.cu includes this file for its device functions)
__global__ void __launch_bounds__(kSelT) k_softmax_topb(const __grid_constant__ SoftmaxArgs a) {
  pdl_wait();
  softmax_row(a, blockIdx.x);
}

lsb_status launch_softmax(lsb_ctx* ctx, const SoftmaxArgs& a) {
  if (a.R_total == 0) return LSB_OK;
  LSB_CUDA(launch_pdl(ctx, k_softmax_topb, dim3(a.R_total), dim3(kSelT), 0, a));
  LSB_LAUNCHED(ctx, "k_softmax_topb");
  return LSB_OK;
}
#endif  // LSB_BODIES_ONLY

// ===================================================================== K5b
struct Cand {
  double score;
  uint32_t beam;
  long long word;
};

__device__ __forceinline__ bool cand_better(const Cand& x, const Cand& y) {
  if (x.score != y.score) return x.score > y.score;
  if (x.beam != y.beam) return x.beam < y.beam;
  return x.word < y.word;
}

// Word id of candidate column r of sentence s.
__device__ __forceinline__ long long word_of(const ExpandArgs& a, const uint32_t* ids,
                                             uint32_t r) {
  if (a.id_map) return a.id_map[r];
  return (r < a.n_shared || !ids) ? static_cast<long long>(r) : static_cast<long long>(ids[r]);
}

// Hidden-state reorder: child k of sentence s starts from its parent's vector.
// One flat (child, float4) index space; each thread keeps 8 loads in flight
// before storing (a load->store chain per element would serialise on
// latency: the store could alias the next load).
static __device__ void reorder_hidden(const ExpandArgs& a, int s, int count, const uint32_t* beams,
                                      int part = 0, int nparts = 1) {
  const int d = a.d;
  const size_t rbase = static_cast<size_t>(s) * a.Bsent;
  const size_t obase = static_cast<size_t>(s) * a.topB;
  constexpr int U = 8;
  if ((d & 3) == 0) {
    const int d4 = d >> 2;
    // this CTA's slice [q_lo, total) of the (child, float4) space
    const int all = count * d4;
    const int q_lo = static_cast<int>(static_cast<long long>(all) * part / nparts);
    const int total = static_cast<int>(static_cast<long long>(all) * (part + 1) / nparts);
    for (int q0 = q_lo + threadIdx.x; q0 < total; q0 += U * blockDim.x) {
      float4 t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < total) {
          const int k = q / d4, c = q - k * d4;
          t[u] = __ldg(reinterpret_cast<const float4*>(a.hidden + (rbase + beams[k]) * d) + c);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < total) {
          const int k = q / d4, c = q - k * d4;
          reinterpret_cast<float4*>(a.hidden_out + (obase + k) * d)[c] = t[u];
        }
      }
    }
  } else {
    const int all = count * d;
    const int q_lo = static_cast<int>(static_cast<long long>(all) * part / nparts);
    const int total = static_cast<int>(static_cast<long long>(all) * (part + 1) / nparts);
    for (int q0 = q_lo + threadIdx.x; q0 < total; q0 += U * blockDim.x) {
      float t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < total) {
          const int k = q / d, c = q - k * d;
          t[u] = __ldg(a.hidden + (rbase + beams[k]) * d + c);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < total) {
          const int k = q / d, c = q - k * d;
          a.hidden_out[(obase + k) * d + c] = t[u];
        }
      }
    }
  }
}

// Rank selection. Lists: [0, nfz) explicit frozen singletons, then one list
// per hypothesis row (a finished row is a singleton carrying its score).
// Shared memory: per list off/len (ints), then per candidate score, beam, word.
constexpr int kRankMaxLists = 128;

// One sentence's expansion by the whole CTA (any blockDim); smem holds the
// candidates (expand_smem_bytes). k_expand runs nparts CTAs per sentence: each
// ranks the candidates (the same bits), part 0 writes the choices, and each
// copies its 1/nparts of the hidden-state reorder.
static __device__ void expand_sentence(const ExpandArgs& a, int s, unsigned char* smem,
                                       int part = 0, int nparts = 1) {
  __shared__ int s_off[kRankMaxLists + 1];
  __shared__ uint32_t s_beams[64];
  __shared__ int s_count;
  const int R = a.Bsent;
  const int nfz = a.frozen_mode ? a.nfrozen : 0;
  const int nl = nfz + R;
  const int nhyp = a.n_hyp ? a.n_hyp[s] : R;
  const size_t rbase = static_cast<size_t>(s) * R;
  const uint32_t* ids = a.ids ? a.ids + static_cast<size_t>(s) * a.ncap : nullptr;
  const int cap = nl * a.topB;
  double* cs = reinterpret_cast<double*>(smem);
  long long* cw = reinterpret_cast<long long*>(cs + cap);
  uint32_t* cb = reinterpret_cast<uint32_t*>(cw + cap);
  int* co = reinterpret_cast<int*>(cb + cap);  // own list of each candidate
  int* cr = co + cap;                          // rank accumulators
  int* surv = cr + cap;                        // candidates left after pruning
  __shared__ int s_heads[kRankMaxLists];       // list heads, best first
  __shared__ int s_nh, s_nsurv;

  // list lengths -> offsets (nl <= kRankMaxLists: one warp scans)
  if (threadIdx.x < 32) {
    int carry = 0;
    for (int l0 = 0; l0 < nl; l0 += 32) {
      const int l = l0 + threadIdx.x;
      int len = 0;
      if (l < nl) {
        if (l < nfz) {
          len = 1;
        } else {
          const int row = l - nfz;
          if (row < nhyp) len = (a.finished && a.finished[rbase + row]) ? 1 : a.top_n[rbase + row];
        }
      }
      int x = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) >= o) x += y;
      }
      if (l < nl) s_off[l + 1] = carry + x;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (threadIdx.x == 0) s_off[0] = 0;
  }
  __syncthreads();
  const int total = s_off[nl];
  // materialise every candidate (score, beam, word)
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int lo = 0, hi = nl - 1;  // list of e: last l with s_off[l] <= e
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    const int l = lo, j = e - s_off[l];
    double sc;
    uint32_t beam;
    long long wd;
    if (l < nfz) {
      sc = a.fz_score[l];
      beam = a.fz_beam[l];
      wd = -1;
    } else {
      const int row = l - nfz;
      beam = a.live_ids ? a.live_ids[rbase + row] : static_cast<uint32_t>(row);
      if (a.finished && a.finished[rbase + row]) {
        sc = a.scores[rbase + row];
        wd = -1;
      } else {
        const TopEntry t = a.top[(rbase + row) * a.topB + j];
        sc = __dadd_rn(a.scores[rbase + row], log_p(t.p));
        wd = word_of(a, ids, t.r);
      }
    }
    cs[e] = sc;
    cb[e] = beam;
    cw[e] = wd;
    co[e] = l;
    cr[e] = j;  // position in its own list
  }
  __syncthreads();
  // Pruning (large beams): a candidate at position j of its list is beaten
  // by its j predecessors and by every other list's head that beats it, so
  // j + #(better foreign heads) >= B rules it out of the top-B without its
  // nl binary searches; heads are ranked once (nl <= kRankMaxLists).
  const int B = a.topB;
  int nsurv = total;
  const bool prune = B > 16;
  if (prune) {
    if (threadIdx.x == 0) {
      s_nh = 0;
      s_nsurv = 0;
    }
    __syncthreads();
    if (threadIdx.x < nl && s_off[threadIdx.x] < s_off[threadIdx.x + 1]) {
      const int eh = s_off[threadIdx.x];
      const Cand me{cs[eh], cb[eh], cw[eh]};
      int rank = 0;
      for (int l = 0; l < nl; ++l) {
        const int o = s_off[l];
        if (l != static_cast<int>(threadIdx.x) && o < s_off[l + 1] &&
            cand_better(Cand{cs[o], cb[o], cw[o]}, me))
          ++rank;
      }
      s_heads[rank] = eh;
      atomicAdd(&s_nh, 1);
    }
    __syncthreads();
    const int nh = s_nh;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const Cand me{cs[e], cb[e], cw[e]};
      int lo = 0, hi = nh;  // heads better than me (includes my own when j > 0)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int h = s_heads[mid];
        if (cand_better(Cand{cs[h], cb[h], cw[h]}, me)) lo = mid + 1;
        else hi = mid;
      }
      const int j = cr[e];
      if (j + lo - (j > 0 ? 1 : 0) < B) surv[atomicAdd(&s_nsurv, 1)] = e;
      else cr[e] = 0x3FFFFFFF;  // rank >= B: never written out
    }
    __syncthreads();
    nsurv = s_nsurv;
  }
  // rank = own position + per other list the count of better entries; one
  // (candidate, list) pair per thread so the binary searches run in parallel
  for (int q = threadIdx.x; q < nsurv * nl; q += blockDim.x) {
    const int qe = q / nl, l = q - qe * nl;
    const int e = prune ? surv[qe] : qe;
    if (l == co[e] || s_off[l] == s_off[l + 1]) continue;
    const Cand me{cs[e], cb[e], cw[e]};
    int b0 = s_off[l], b1 = s_off[l + 1];  // first entry of l not better than me
    while (b0 < b1) {
      const int mid = (b0 + b1) >> 1;
      if (cand_better(Cand{cs[mid], cb[mid], cw[mid]}, me)) b0 = mid + 1;
      else b1 = mid;
    }
    if (b0 > s_off[l]) atomicAdd(cr + e, b0 - s_off[l]);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int rank = cr[e];
    const Cand me{cs[e], cb[e], cw[e]};
    if (rank < B) {
      if (part == 0)
        a.choices[static_cast<size_t>(s) * B + rank] =
            lsb_choice{me.score, me.beam, 0u, static_cast<int64_t>(me.word)};
      if (rank < 64) s_beams[rank] = me.beam;
    }
  }
  const int count = min(B, total);
  if (threadIdx.x == 0) {
    if (part == 0) a.n_choices[s] = count;
    s_count = count;
  }
  __syncthreads();
  pdl_trigger();
  if (a.hidden_out && a.hidden) reorder_hidden(a, s, min(s_count, 64), s_beams, part, nparts);
}

#ifndef LSB_BODIES_ONLY
template <int NT>
__global__ void __launch_bounds__(NT) k_expand(const __grid_constant__ ExpandArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  pdl_wait();
  expand_sentence(a, blockIdx.x, smem, blockIdx.y, gridDim.y);
}

size_t expand_smem_bytes(const ExpandArgs& a) {
  const int nl = (a.frozen_mode ? a.nfrozen : 0) + a.Bsent;
  return static_cast<size_t>(nl) * std::max(a.topB, 1) * (8 + 8 + 4 + 4 + 4 + 4);
}

// B-round warp tournament over list heads (any number of lists).
__global__ void k_expand_tournament(ExpandArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int s = blockIdx.x;
  const int R = a.Bsent;
  const int nfz = a.frozen_mode ? a.nfrozen : 0;
  const int nl = nfz + R;
  double* hscore = reinterpret_cast<double*>(smem);
  long long* hword = reinterpret_cast<long long*>(hscore + nl);
  int* hpos = reinterpret_cast<int*>(hword + nl);
  int* hlen = hpos + nl;
  uint32_t* hbeam = reinterpret_cast<uint32_t*>(hlen + nl);
  __shared__ int s_count;
  __shared__ uint32_t s_beams[64];
  const int lane = threadIdx.x & 31;
  const int nhyp = a.n_hyp ? a.n_hyp[s] : R;
  const size_t rbase = static_cast<size_t>(s) * R;
  const uint32_t* ids = a.ids ? a.ids + static_cast<size_t>(s) * a.ncap : nullptr;
  auto live_score = [&](int row, int pos, double& sc, long long& wd) {
    const TopEntry e = a.top[(rbase + row) * a.topB + pos];
    sc = __dadd_rn(a.scores[rbase + row], log_p(e.p));
    wd = word_of(a, ids, e.r);
  };
  if (threadIdx.x < 32) {
    for (int l = lane; l < nl; l += 32) {
      int len = 0;
      double sc = -INFINITY;
      long long wd = 0;
      uint32_t beam = 0;
      if (l < nfz) {
        len = 1;
        sc = a.fz_score[l];
        wd = -1;
        beam = a.fz_beam[l];
      } else {
        const int row = l - nfz;
        beam = a.live_ids ? a.live_ids[rbase + row] : static_cast<uint32_t>(row);
        if (row < nhyp) {
          if (a.finished && a.finished[rbase + row]) {
            len = 1;
            sc = a.scores[rbase + row];
            wd = -1;
          } else {
            len = a.top_n[rbase + row];
            if (len > 0) live_score(row, 0, sc, wd);
          }
        }
      }
      hscore[l] = sc;
      hword[l] = wd;
      hpos[l] = 0;
      hlen[l] = len;
      hbeam[l] = beam;
    }
    __syncwarp();
    int count = 0;
    for (int k = 0; k < a.topB; ++k) {
      Cand best{-INFINITY, 0xFFFFFFFFu, 0x7FFFFFFFFFFFFFFFll};
      int bl = -1;
      for (int l = lane; l < nl; l += 32) {
        if (hpos[l] >= hlen[l]) continue;
        const Cand c{hscore[l], hbeam[l], hword[l]};
        if (bl < 0 || cand_better(c, best)) {
          best = c;
          bl = l;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        Cand y;
        y.score = __shfl_xor_sync(0xffffffffu, best.score, o);
        y.beam = __shfl_xor_sync(0xffffffffu, best.beam, o);
        y.word = __shfl_xor_sync(0xffffffffu, best.word, o);
        const int yl = __shfl_xor_sync(0xffffffffu, bl, o);
        if (yl >= 0 && (bl < 0 || cand_better(y, best))) {
          best = y;
          bl = yl;
        }
      }
      if (bl < 0) break;
      if (lane == 0) {
        a.choices[static_cast<size_t>(s) * a.topB + k] =
            lsb_choice{best.score, best.beam, 0u, static_cast<int64_t>(best.word)};
        if (k < 64) s_beams[k] = best.beam;
      }
      if ((bl & 31) == lane) {
        const int np = ++hpos[bl];
        if (np < hlen[bl]) {
          double sc;
          long long wd;
          live_score(bl - nfz, np, sc, wd);
          hscore[bl] = sc;
          hword[bl] = wd;
        }
      }
      __syncwarp();
      ++count;
    }
    if (lane == 0) {
      a.n_choices[s] = count;
      s_count = count;
    }
  }
  __syncthreads();
  if (a.hidden_out && a.hidden) reorder_hidden(a, s, min(s_count, 64), s_beams);
}

// ============================================================ fused K5a+K5b
// The LSH step's rows are short (|V_LSH| ~ 1-2k), so one WARP per row keeps
// the row in registers (KMAX floats per lane): float max, double exp/sum,
// p = float(e) * float(1/denom), then B rounds of a warp arg-max by
// (p desc, column asc) -- the lane that owns the winner drops it and
// rescans its registers. One CTA per sentence: after a barrier the CTA runs
// the sentence's expansion (rank selection, as k_expand) and the hidden
// reorder, so K5 is one launch with no top-list round trip through HBM.
constexpr int kFusedMaxB = 16;

// Row softmax + top-B with the row in registers (n <= 32*KMAX).
template <int KMAX>
__device__ __forceinline__ void fused_row_registers(const SoftmaxArgs& sa, int row, float* L,
                                                    uint32_t n, TopEntry* out, int lane) {
  const int B = sa.topB;
  float v[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const uint32_t c = lane + 32u * k;
    v[k] = c < n ? L[c] : -INFINITY;
  }
  float mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) mx = (mx < v[k]) ? v[k] : mx;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (mx < y) ? y : mx;
  }
  if (n == 0 || (isinf(mx) && mx < 0)) {
    if (lane == 0) {
      atomicOr(sa.err, kErrEmptyRow);
      sa.top_n[row] = 0;
    }
    return;
  }
  const double dmx = static_cast<double>(mx);
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (lane + 32u * k < n) {
      const double e = glibc_exp(static_cast<double>(v[k]) - dmx);
      v[k] = static_cast<float>(e);
      sum += e;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = reference_inv_warp(sum, n, L, dmx, lane, sa.seq_denominator);
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const uint32_t c = lane + 32u * k;
    if (c < n) {
      v[k] = __fmul_rn(v[k], inv);
      if (sa.keep_probs) L[c] = v[k];
    } else {
      v[k] = -1.0f;  // below every probability
    }
  }
  // lane-local best: strict '>' in ascending k keeps the smallest column
  float bp = -1.0f;
  int bk = 0;
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
    if (v[k] > bp) {
      bp = v[k];
      bk = k;
    }
  const int keep = static_cast<int>(min(static_cast<uint32_t>(B), n));
  for (int r = 0; r < keep; ++r) {
    float p = bp;
    uint32_t col = lane + 32u * bk;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float yp = __shfl_xor_sync(0xffffffffu, p, o);
      const uint32_t yc = __shfl_xor_sync(0xffffffffu, col, o);
      if (top_better(yp, yc, p, col)) {
        p = yp;
        col = yc;
      }
    }
    if (lane == 0) out[r] = TopEntry{p, col};
    if ((col & 31u) == static_cast<uint32_t>(lane)) {  // the owner drops it, rescans
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k == bk) v[k] = -1.0f;
      bp = -1.0f;
      bk = 0;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (v[k] > bp) {
          bp = v[k];
          bk = k;
        }
    }
  }
  if (lane == 0) sa.top_n[row] = keep;
}

// Same for rows too long for registers: the row stays in global memory and
// round r takes the best entry strictly below round r-1's winner.
__device__ void fused_row_global(const SoftmaxArgs& sa, int row, float* L, uint32_t n,
                                 TopEntry* out, int lane) {
  const int B = sa.topB;
  float mx = -INFINITY;
  for (uint32_t c = lane; c < n; c += 32) mx = (mx < L[c]) ? L[c] : mx;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (mx < y) ? y : mx;
  }
  if (n == 0 || (isinf(mx) && mx < 0)) {
    if (lane == 0) {
      atomicOr(sa.err, kErrEmptyRow);
      sa.top_n[row] = 0;
    }
    return;
  }
  const double dmx = static_cast<double>(mx);
  double sum = 0.0;
  for (uint32_t c = lane; c < n; c += 32) sum += glibc_exp(static_cast<double>(L[c]) - dmx);
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = reference_inv_warp(sum, n, L, dmx, lane, sa.seq_denominator);
  __syncwarp();
  for (uint32_t c = lane; c < n; c += 32)  // probabilities
    L[c] = __fmul_rn(static_cast<float>(glibc_exp(static_cast<double>(L[c]) - dmx)), inv);
  const int keep = static_cast<int>(min(static_cast<uint32_t>(B), n));
  float pp = INFINITY;
  uint32_t pc = 0xFFFFFFFFu;
  for (int r = 0; r < keep; ++r) {
    float bp = -1.0f;
    uint32_t bc = 0xFFFFFFFFu;
    for (uint32_t c = lane; c < n; c += 32) {
      const float p = L[c];
      if (top_better(pp, pc, p, c) && top_better(p, c, bp, bc)) {
        bp = p;
        bc = c;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float yp = __shfl_xor_sync(0xffffffffu, bp, o);
      const uint32_t yc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (top_better(yp, yc, bp, bc)) {
        bp = yp;
        bc = yc;
      }
    }
    if (lane == 0) out[r] = TopEntry{bp, bc};
    pp = bp;
    pc = bc;
  }
  if (lane == 0) sa.top_n[row] = keep;
}

// One CTA per sentence, one warp per hypothesis row (B <= 16 warps): every
// row's softmax/top-B, then (after one barrier) the sentence's expansion by
// rank selection and the hidden reorder by the whole CTA.
template <int KMAX>
__global__ void __launch_bounds__(kFusedMaxB * 32) k_select_fused(SoftmaxArgs sa, ExpandArgs ea) {
  __shared__ double s_score[kFusedMaxB * kFusedMaxB];
  __shared__ long long s_word[kFusedMaxB * kFusedMaxB];
  __shared__ uint32_t s_beam[kFusedMaxB * kFusedMaxB];
  __shared__ int s_off[kFusedMaxB + 1];
  __shared__ uint32_t s_pick[kFusedMaxB];
  __shared__ int s_count;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s = blockIdx.x;
  const int Bs = sa.Bsent, B = sa.topB;
  const size_t rbase = static_cast<size_t>(s) * Bs;
  const int nhyp = sa.n_hyp ? sa.n_hyp[s] : Bs;
  if (w < Bs) {
    const int row = static_cast<int>(rbase) + w;
    const bool live = w < nhyp && !(sa.finished && sa.finished[row]);
    TopEntry* out = sa.top + static_cast<size_t>(row) * B;
    if (live) {
      const uint32_t n = sa.n_cand[s];
      float* L = sa.logits + static_cast<size_t>(row) * sa.ldl;
      if (n <= 32u * KMAX) fused_row_registers<KMAX>(sa, row, L, n, out, lane);
      else fused_row_global(sa, row, L, n, out, lane);
    } else if (lane == 0) {
      sa.top_n[row] = 0;
    }
  }
  __syncthreads();
  const uint32_t* ids = ea.ids ? ea.ids + static_cast<size_t>(s) * ea.ncap : nullptr;
  if (w == 0) {
    int len = 0;
    if (lane < Bs && lane < nhyp)
      len = (ea.finished && ea.finished[rbase + lane]) ? 1 : ea.top_n[rbase + lane];
    int x = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane < Bs) s_off[lane + 1] = x;
    if (lane == 0) s_off[0] = 0;
  }
  __syncthreads();
  const int total = s_off[Bs];
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int l = 0;
    while (l + 1 < Bs && s_off[l + 1] <= e) ++l;
    const int j = e - s_off[l];
    double sc;
    long long wd;
    if (ea.finished && ea.finished[rbase + l]) {
      sc = ea.scores[rbase + l];
      wd = -1;
    } else {
      const TopEntry t = ea.top[(rbase + l) * B + j];
      sc = __dadd_rn(ea.scores[rbase + l], log_p(t.p));
      wd = word_of(ea, ids, t.r);
    }
    s_score[e] = sc;
    s_word[e] = wd;
    s_beam[e] = static_cast<uint32_t>(l);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int own = 0;
    while (own + 1 < Bs && s_off[own + 1] <= e) ++own;
    const Cand me{s_score[e], s_beam[e], s_word[e]};
    int rank = e - s_off[own];
    for (int l = 0; l < Bs && rank < B; ++l) {
      if (l == own) continue;
      int b0 = s_off[l], b1 = s_off[l + 1];
      while (b0 < b1) {
        const int mid = (b0 + b1) >> 1;
        if (cand_better(Cand{s_score[mid], s_beam[mid], s_word[mid]}, me)) b0 = mid + 1;
        else b1 = mid;
      }
      rank += b0 - s_off[l];
    }
    if (rank < B) {
      ea.choices[static_cast<size_t>(s) * B + rank] =
          lsb_choice{me.score, me.beam, 0u, static_cast<int64_t>(me.word)};
      s_pick[rank] = me.beam;
    }
  }
  if (threadIdx.x == 0) {
    s_count = min(B, total);
    ea.n_choices[s] = s_count;
  }
  __syncthreads();
  if (ea.hidden_out && ea.hidden) reorder_hidden(ea, s, s_count, s_pick);
}

// K5a alone, one warp per row over the whole GPU (4 rows per CTA).
template <int KMAX>
__global__ void __launch_bounds__(128) k_softmax_topb_warp(SoftmaxArgs sa) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (row >= sa.R_total) return;
  const int s = row / sa.Bsent, i = row % sa.Bsent;
  const bool live = !(sa.n_hyp && i >= sa.n_hyp[s]) && !(sa.finished && sa.finished[row]);
  if (!live) {
    if (lane == 0) sa.top_n[row] = 0;
    return;
  }
  const uint32_t n = sa.n_cand[s];
  float* L = sa.logits + static_cast<size_t>(row) * sa.ldl;
  TopEntry* out = sa.top + static_cast<size_t>(row) * sa.topB;
  if (n <= 32u * KMAX) fused_row_registers<KMAX>(sa, row, L, n, out, lane);
  else fused_row_global(sa, row, L, n, out, lane);
}

lsb_status launch_softmax_warp(lsb_ctx* ctx, const SoftmaxArgs& sa, uint32_t max_n) {
  const int grid = (sa.R_total + 3) / 4;
  if (max_n <= 32u * 32u) k_softmax_topb_warp<32><<<grid, 128, 0, ctx->stream>>>(sa);
  else k_softmax_topb_warp<48><<<grid, 128, 0, ctx->stream>>>(sa);
  LSB_LAUNCHED(ctx, "k_softmax_topb_warp");
  return LSB_OK;
}

// Fused K5 for the batched step: B <= 16 hypotheses per sentence. Rows up
// to 32*KMAX candidates stay in registers (KMAX from the largest possible
// row, ncap), longer ones take the global-memory path. `arrive` holds S
// zeroed counters; the kernel leaves them zeroed.
bool select_fused_applies(const SoftmaxArgs& sa, const ExpandArgs& ea) {
  return sa.topB <= kFusedMaxB && sa.Bsent == sa.topB && !ea.frozen_mode && !ea.live_ids &&
         !ea.id_map && !sa.probs_in && sa.n_cand;
}

lsb_status launch_select_fused(lsb_ctx* ctx, const SoftmaxArgs& sa, const ExpandArgs& ea,
                               uint32_t max_n, uint32_t* arrive) {
  (void)arrive;
  const int S = sa.R_total / sa.Bsent;
  const int threads = sa.Bsent * 32;
  if (max_n <= 32u * 32u)
    k_select_fused<32><<<S, threads, 0, ctx->stream>>>(sa, ea);
  else
    k_select_fused<48><<<S, threads, 0, ctx->stream>>>(sa, ea);
  LSB_LAUNCHED(ctx, "k_select_fused");
  return LSB_OK;
}

lsb_status launch_expand(lsb_ctx* ctx, const ExpandArgs& a) {
  if (a.S == 0) return LSB_OK;
  const int nl = (a.frozen_mode ? a.nfrozen : 0) + a.Bsent;
  const size_t rank_smem = static_cast<size_t>(nl) * std::max(a.topB, 1) * (8 + 8 + 4 + 4 + 4 + 4);
  if (nl <= kRankMaxLists && rank_smem <= ctx->smem_optin) {
    // 1024 threads for small beams (cfg 2: 132.5 -> 131.3 us/step), 512 for
    // large ones (cfg 3, B=50: 49 vs 61 us)
    const bool wide = a.topB <= 16;
    auto* kern = wide ? k_expand<1024> : k_expand<512>;
    if (lsb_status rc = ensure_smem(ctx, kern, rank_smem)) return rc;
    // few sentences: several CTAs per sentence share the hidden reorder
    // (each re-ranks the same candidates). Measured (B200, cfg 2 S=64: 1 / 2 /
    // 4 / 8 parts 13.6 / 12.4 / 18.5 / 28.6 us; cfg 1 S=1: 37.7 -> 36.9 us per
    // step at 8): the ranking, not the copy, bounds K5b, so only mildly.
    static const int parts_env = getenv("LSB_K5B_PARTS") ? atoi(getenv("LSB_K5B_PARTS")) : 0;
    const int parts = parts_env > 0                  ? parts_env
                      : 16 * a.S <= ctx->sm_count    ? 8
                      : 2 * a.S <= ctx->sm_count     ? 2
                                                     : 1;
    LSB_CUDA(launch_pdl(ctx, kern, dim3(a.S, parts), dim3(wide ? 1024 : 512), rank_smem, a));
    LSB_LAUNCHED(ctx, "k_expand");
    return LSB_OK;
  }
  const size_t smem = static_cast<size_t>(nl) * (8 + 8 + 4 + 4 + 4) + 16;
  if (smem > ctx->smem_optin) return set_error("expand: too many rows"), LSB_EINVAL;
  if (lsb_status rc = ensure_smem(ctx, k_expand_tournament, smem)) return rc;
  k_expand_tournament<<<a.S, 256, smem, ctx->stream>>>(a);
  LSB_LAUNCHED(ctx, "k_expand_tournament");
  return LSB_OK;
}

#endif  // LSB_BODIES_ONLY

}  // namespace lsb
