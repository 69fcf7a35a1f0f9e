// k_softmax_seg.cu -- K5a for long rows (the full-vocabulary step): each row
// is split into P segments of `seglen` columns, one CTA per (row, segment),
// so the 12 rows of a one-sentence full-vocabulary step spread over the whole
// GPU instead of 12 CTAs (S=1, V=40k: 150 us in k_softmax_topb).
//
// softmax_rows (src/beam_decoder.cpp:46-74) in four launches:
//   k_seg_max    : segment float max -> part_max[row][p]
//   k_seg_exp    : row max = max over the P partials (float max is exact in
//                  any order); e = exp((double)l - mx) (glibc's exp), stored
//                  as float(e) in a separate buffer (the logits stay intact);
//                  segment compensated sum (hi, c) and the bound
//                  sum min(e, 2^-52) -> part_sum / part_c / part_b[row][p]
//   k_seg_denom  : one CTA per row: the exact row sum and the bound give an
//                  interval holding the reference's sequential sum; its
//                  float(1/x) if both ends agree, else the sequential sum
//                  redone from the logits (softmax_denom.cuh) -> inv[row]
//   k_seg_select : p = float(e) * inv (written back into the logits when
//                  kept); segment top-B by (p desc, column asc) with the
//                  threshold selection of k_softmax_topb; the row's last
//                  segment CTA to finish merges the P sorted lists into the
//                  row's top-B.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "glibc_log.cuh"
#include "k_step.cuh"
#include "softmax_denom.cuh"

namespace lsb {

namespace {

constexpr int kSegT = 128;
constexpr int kSegCand = 256;   // threshold survivors ranked directly
constexpr int kSegMerge = 512;  // P * B entries merged by the last CTA

__device__ __forceinline__ bool seg_better(float pa, uint32_t ra, float pb, uint32_t rb) {
  return pa > pb || (pa == pb && ra < rb);
}

template <class T, class Op>
__device__ __forceinline__ T seg_reduce(T v, T* red, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = red[0];
#pragma unroll
  for (int w = 1; w < kSegT / 32; ++w) v = op(v, red[w]);
  return v;
}

struct SegFMax {
  __device__ float operator()(float x, float y) const { return (x < y) ? y : x; }
};

// The row's (segment's) coordinates; false for rows that are not scored.
__device__ __forceinline__ bool seg_row(const SegArgs& g, int& row, int& p, uint32_t& c0,
                                        uint32_t& c1, uint32_t& n) {
  const SoftmaxArgs& a = g.sa;
  row = blockIdx.x / g.P;
  p = blockIdx.x % g.P;
  const int s = row / a.Bsent, i = row % a.Bsent;
  if ((a.n_hyp && i >= a.n_hyp[s]) || (a.finished && a.finished[row])) return false;
  n = a.n_cand ? a.n_cand[s] : a.n_const;
  c0 = min(n, static_cast<uint32_t>(p) * g.seglen);
  c1 = min(n, c0 + g.seglen);
  return true;
}

// A lower bound for the K-th largest of the CTA's per-thread maxima x (-1 =
// none): each warp sorts its 32 with a shuffle bitonic network; for K <= 32
// the max over warps of each warp's K-th largest (K lanes of that warp hold an
// entry >= it), else the exact K-th by ranking in shared memory.
__device__ float seg_kth(float x, int K, float* s_lm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float s_tau;
  if (K <= 32) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1)  // bitonic sort, descending
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const float y = __shfl_xor_sync(0xffffffffu, x, stride);
        const bool up = ((lane & size) == 0) == ((lane & stride) == 0);
        x = up ? fmaxf(x, y) : fminf(x, y);
      }
    const float kw = __shfl_sync(0xffffffffu, x, K - 1);
    if (lane == 0) s_lm[warp] = kw;
    __syncthreads();
    float t = s_lm[0];
#pragma unroll
    for (int w = 1; w < kSegT / 32; ++w) t = fmaxf(t, s_lm[w]);
    return t;
  }
  s_lm[tid] = x;
  if (tid == 0) s_tau = -1.0f;
  __syncthreads();
  if (K <= kSegT) {
    int rank = 0;
    for (int j = 0; j < kSegT; ++j) {
      const float y = s_lm[j];
      rank += (y > x) || (y == x && j < tid);
    }
    if (rank == K - 1) s_tau = x;
  }
  __syncthreads();
  return s_tau;
}

// The row max over the P segment partials (float max: exact in any order);
// thread q loads partial q (one round trip, not P dependent ones).
__device__ __forceinline__ float seg_row_max(const SegArgs& g, int row, float* red) {
  float v = -INFINITY;
  for (int q = threadIdx.x; q < g.P; q += kSegT) {
    const float y = g.part_max[row * g.P + q];
    v = (v < y) ? y : v;
  }
  return seg_reduce(v, red, SegFMax{});
}

}  // namespace

__global__ void __launch_bounds__(kSegT) k_seg_max(SegArgs g) {
  __shared__ float red[kSegT / 32];
  pdl_wait();
  int row, p;
  uint32_t c0, c1, n;
  if (!seg_row(g, row, p, c0, c1, n)) return;
  const float* L = g.sa.logits + static_cast<size_t>(row) * g.sa.ldl;
  float mx = -INFINITY;
  for (uint32_t c = c0 + threadIdx.x; c < c1; c += kSegT) {
    const float v = L[c];
    mx = (mx < v) ? v : mx;
  }
  mx = seg_reduce(mx, red, SegFMax{});
  pdl_trigger();
  if (threadIdx.x == 0) g.part_max[blockIdx.x] = mx;
}

__global__ void __launch_bounds__(kSegT) k_seg_exp(SegArgs g) {
  __shared__ float redf[kSegT / 32];
  __shared__ unsigned long long exptab[256];  // published by seg_row_max's barriers
  stage_exp_table(exptab);
  pdl_wait();
  int row, p;
  uint32_t c0, c1, n;
  if (!seg_row(g, row, p, c0, c1, n)) return;
  const float mx = seg_row_max(g, row, redf);
  if (n == 0 || (isinf(mx) && mx < 0)) {  // src/beam_decoder.cpp:72
    if (threadIdx.x == 0 && p == 0) atomicOr(g.sa.err, kErrEmptyRow);
    return;
  }
  const float* L = g.sa.logits + static_cast<size_t>(row) * g.sa.ldl;
  float* Eo = g.e_out + static_cast<size_t>(row) * g.sa.ldl;
  const double dmx = static_cast<double>(mx);
  // compensated sum (hi + c exact) and the sequential-error bound b
  double hi = 0.0, cc = 0.0, bnd = 0.0;
  // four independent loads / exps in flight per thread
  uint32_t c = c0 + threadIdx.x;
  for (; c + 3 * kSegT < c1; c += 4 * kSegT) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = L[c + k * kSegT];
    double e[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) e[k] = glibc_exp_smem(static_cast<double>(v[k]) - dmx, exptab);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      Eo[c + k * kSegT] = static_cast<float>(e[k]);
      dd_add(hi, cc, e[k]);
      bnd = __dadd_rn(bnd, fmin(e[k], 0x1p-52));
    }
  }
  for (; c < c1; c += kSegT) {
    const double e = glibc_exp_smem(static_cast<double>(L[c]) - dmx, exptab);
    Eo[c] = static_cast<float>(e);
    dd_add(hi, cc, e);
    bnd = __dadd_rn(bnd, fmin(e, 0x1p-52));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    const double c2 = __shfl_xor_sync(0xffffffffu, cc, o);
    dd_merge(hi, cc, h2, c2);
    bnd = __dadd_rn(bnd, __shfl_xor_sync(0xffffffffu, bnd, o));
  }
  __shared__ double s_hi[kSegT / 32], s_c[kSegT / 32], s_b[kSegT / 32];
  if ((threadIdx.x & 31) == 0) {
    s_hi[threadIdx.x >> 5] = hi;
    s_c[threadIdx.x >> 5] = cc;
    s_b[threadIdx.x >> 5] = bnd;
  }
  __syncthreads();
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kSegT / 32; ++w) {
      dd_merge(hi, cc, s_hi[w], s_c[w]);
      bnd = __dadd_rn(bnd, s_b[w]);
    }
    g.part_sum[blockIdx.x] = hi;
    g.part_c[blockIdx.x] = cc;
    g.part_b[blockIdx.x] = bnd;
  }
}

// One CTA per row: the row's exact sum from the P compensated segment
// partials and the sequential-error bound (softmax_denom.cuh), certified
// float(1/denom) or the sequential sum from the intact logits; inv[row] for
// k_seg_select.
__global__ void __launch_bounds__(kSegT) k_seg_denom(SegArgs g) {
  __shared__ float redf[kSegT / 32];
  __shared__ double s_part[kSegMaxP], s_pc[kSegMaxP], s_pb[kSegMaxP];
  const SoftmaxArgs& a = g.sa;
  pdl_wait();
  const int row = blockIdx.x;
  const int s = row / a.Bsent, i = row % a.Bsent;
  if ((a.n_hyp && i >= a.n_hyp[s]) || (a.finished && a.finished[row])) return;
  const uint32_t n = a.n_cand ? a.n_cand[s] : a.n_const;
  const float mx = seg_row_max(g, row, redf);
  if (n == 0 || (isinf(mx) && mx < 0)) return;
  for (int q = threadIdx.x; q < g.P; q += kSegT) {
    s_part[q] = g.part_sum[row * g.P + q];
    s_pc[q] = g.part_c[row * g.P + q];
    s_pb[q] = g.part_b[row * g.P + q];
  }
  __syncthreads();
  double hi = 0.0, cc = 0.0, bnd = 0.0;
  for (int q = 0; q < g.P; ++q) {
    dd_merge(hi, cc, s_part[q], s_pc[q]);
    bnd = __dadd_rn(bnd, s_pb[q]);
  }
  float inv;
  if (a.seq_denominator == 1 || !inv_from_exact(hi, cc, bnd, &inv))
    inv = sequential_inv_cta<kSegT>(n, a.logits + static_cast<size_t>(row) * a.ldl,
                                    static_cast<double>(mx));
  pdl_trigger();
  if (threadIdx.x == 0) g.inv[row] = inv;
}

__global__ void __launch_bounds__(kSegT) k_seg_select(SegArgs g) {
  __shared__ float s_lm[kSegT];
  __shared__ int s_nc;
  __shared__ float c_p[kSegMerge];
  __shared__ uint32_t c_c[kSegMerge];
  __shared__ float win_p[kSegT / 32];
  __shared__ uint32_t win_r[kSegT / 32];
  __shared__ bool s_last;
  __shared__ float redf[kSegT / 32];
  __shared__ int s_off[kSegMaxP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SoftmaxArgs& a = g.sa;
  pdl_wait();
  int row, p;
  uint32_t c0, c1, n;
  const int B = a.topB;
  if (!seg_row(g, row, p, c0, c1, n)) {
    if (tid == 0 && p == 0) a.top_n[row] = 0;
    return;
  }
  // an empty row (error raised in k_seg_exp) or no selection
  const float mx = seg_row_max(g, row, redf);
  if (n == 0 || (isinf(mx) && mx < 0) || B <= 0) {
    if (tid == 0 && p == 0) a.top_n[row] = 0;
    return;
  }
  // float(1/denom): k_seg_denom's (certified or sequential)
  const float inv = g.inv[row];
  float* L = a.logits + static_cast<size_t>(row) * a.ldl;
  const float* Eo = g.e_out + static_cast<size_t>(row) * a.ldl;
  const uint32_t m = c1 - c0;
  // pass 1: p (kept when asked) and each thread's maximum
  float x = -1.0f;
  for (uint32_t c = c0 + tid; c < c1; c += kSegT) {
    const float pv = __fmul_rn(Eo[c], inv);
    if (a.keep_probs) L[c] = pv;
    x = fmaxf(x, pv);
  }
  auto p_at = [&](uint32_t c) { return a.keep_probs ? L[c] : __fmul_rn(Eo[c], inv); };
  if (tid == 0) s_nc = 0;
  const float tau = seg_kth(x, B, s_lm);
  const int keep = static_cast<int>(min(static_cast<uint32_t>(B), m));
  TopEntry* out = g.seg_top + static_cast<size_t>(blockIdx.x) * B;
  // pass 2: survivors p >= tau (tau > 0), else every positive p
  for (uint32_t c = c0 + tid; c < c1; c += kSegT) {
    const float pv = p_at(c);
    if (tau > 0.0f ? pv >= tau : pv > 0.0f) {
      const int at = atomicAdd(&s_nc, 1);
      if (at < kSegCand) {
        c_p[at] = pv;
        c_c[at] = c;
      }
    }
  }
  __syncthreads();
  const int nc = s_nc;
  if (nc <= kSegCand) {
    for (int q = tid; q < nc; q += kSegT) {
      const float pv = c_p[q];
      const uint32_t c = c_c[q];
      int rank = 0;
      for (int j = 0; j < nc; ++j) rank += seg_better(c_p[j], c_c[j], pv, c);
      if (rank < keep) out[rank] = TopEntry{pv, c};
    }
    // zeros, by ascending column, after every positive p
    int filled = min(nc, keep);
    for (uint32_t base = c0; filled < keep && base < c1; base += kSegT) {
      const uint32_t c = base + tid;
      const bool z = c < c1 && !(p_at(c) > 0.0f);
      const unsigned bal = __ballot_sync(0xffffffffu, z);
      if (lane == 0) win_r[warp] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kSegT / 32; ++w) {
        before += w < warp ? static_cast<int>(win_r[w]) : 0;
        total += static_cast<int>(win_r[w]);
      }
      const int pos = filled + before + __popc(bal & ((1u << lane) - 1u));
      if (z && pos < keep) out[pos] = TopEntry{p_at(c), c};
      filled += total;
      __syncthreads();
    }
  } else {
    // many ties at tau: rounds of a block-wide arg-max below the last key
    float lp = INFINITY;
    uint32_t lc = 0;
    for (int k = 0; k < keep; ++k) {
      float bp = -1.0f;
      uint32_t br = 0xFFFFFFFFu;
      for (uint32_t c = c0 + tid; c < c1; c += kSegT) {
        const float pv = p_at(c);
        if (seg_better(lp, lc, pv, c) && seg_better(pv, c, bp, br)) {
          bp = pv;
          br = c;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float yp = __shfl_xor_sync(0xffffffffu, bp, o);
        const uint32_t yr = __shfl_xor_sync(0xffffffffu, br, o);
        if (seg_better(yp, yr, bp, br)) {
          bp = yp;
          br = yr;
        }
      }
      __syncthreads();
      if (lane == 0) {
        win_p[warp] = bp;
        win_r[warp] = br;
      }
      __syncthreads();
#pragma unroll
      for (int w = 0; w < kSegT / 32; ++w)
        if (seg_better(win_p[w], win_r[w], bp, br)) {
          bp = win_p[w];
          br = win_r[w];
        }
      if (tid == 0) out[k] = TopEntry{bp, br};
      lp = bp;
      lc = br;
    }
  }
  if (tid == 0) g.seg_n[blockIdx.x] = keep;
  // the row's last segment to finish merges the P lists
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&g.count[row], 1u) == static_cast<uint32_t>(g.P - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  pdl_trigger();
  // Merge. Every list is sorted by (p desc, column asc), so the row's B-th
  // best is no worse than the B-th best list head (tau_h): only entries at
  // least as good as tau_h can be in the top-B. Rank the heads, collect the
  // entries >= tau_h, rank those.
  __shared__ float h_p[kSegMaxP];
  __shared__ uint32_t h_c[kSegMaxP];
  __shared__ int s_cnt;
  __shared__ float s_tp;
  __shared__ uint32_t s_tc;
  if (tid < g.P) {
    const int k = __ldcg(g.seg_n + row * g.P + tid);
    const TopEntry* src = g.seg_top + static_cast<size_t>(row * g.P + tid) * B;
    h_p[tid] = k > 0 ? __ldcg(&src->p) : -2.0f;  // empty list: worse than any p
    h_c[tid] = k > 0 ? __ldcg(&src->r) : 0xFFFFFFFFu;
    s_off[tid] = k;
  }
  if (tid == 0) {
    s_cnt = 0;
    s_tp = -2.0f;  // fewer than B heads: keep everything
    s_tc = 0xFFFFFFFFu;
  }
  __syncthreads();
  if (tid < g.P && h_p[tid] > -2.0f) {
    int rank = 0;
    for (int q = 0; q < g.P; ++q) rank += seg_better(h_p[q], h_c[q], h_p[tid], h_c[tid]);
    if (rank == B - 1) {
      s_tp = h_p[tid];
      s_tc = h_c[tid];
    }
  }
  __syncthreads();
  const float tp = s_tp;
  const uint32_t tc = s_tc;
  for (int e = tid; e < g.P * B; e += kSegT) {
    const int q = e / B, k = e % B;
    if (k < s_off[q]) {
      const TopEntry* src = g.seg_top + static_cast<size_t>(row * g.P + q) * B + k;
      const float pv = __ldcg(&src->p);
      const uint32_t c = __ldcg(&src->r);
      if (!seg_better(tp, tc, pv, c)) {  // (pv, c) at least as good as tau_h
        const int at = atomicAdd(&s_cnt, 1);
        c_p[at] = pv;
        c_c[at] = c;
      }
    }
  }
  __syncthreads();
  const int total = s_cnt;
  const int kr = min(B, total);
  TopEntry* ro = a.top + static_cast<size_t>(row) * B;
  for (int q = tid; q < total; q += kSegT) {
    const float pv = c_p[q];
    const uint32_t c = c_c[q];
    int rank = 0;
    for (int j = 0; j < total; ++j) rank += seg_better(c_p[j], c_c[j], pv, c);
    if (rank < kr) ro[rank] = TopEntry{pv, c};
  }
  if (tid == 0) {
    a.top_n[row] = kr;
    g.count[row] = 0;  // self-resetting for the next step
  }
}

// Segments per row: enough CTAs for ~4 per SM, segments of >= 1024 columns,
// and P * B entries for the merge's shared memory.
int seg_count(lsb_ctx* ctx, int R, uint32_t n, int B) {
  // (and segments of <= 8192 columns: the exp pass is latency-bound per CTA)
  const int want = std::max((4 * ctx->sm_count + std::max(R, 1) - 1) / std::max(R, 1),
                            static_cast<int>((n + 8191) / 8192));
  const int by_len = static_cast<int>((n + 1023) / 1024);
  const int by_merge = kSegMerge / std::max(B, 1);
  return std::max(1, std::min({want, by_len, by_merge, kSegMaxP}));
}

lsb_status launch_softmax_seg(lsb_ctx* ctx, const SegArgs& g) {
  if (g.sa.R_total == 0) return LSB_OK;
  const dim3 grid(g.sa.R_total * g.P);
  LSB_CUDA(launch_pdl(ctx, k_seg_max, grid, dim3(kSegT), 0, g));
  LSB_LAUNCHED(ctx, "k_seg_max");
  LSB_CUDA(launch_pdl(ctx, k_seg_exp, grid, dim3(kSegT), 0, g));
  LSB_LAUNCHED(ctx, "k_seg_exp");
  LSB_CUDA(launch_pdl(ctx, k_seg_denom, dim3(g.sa.R_total), dim3(kSegT), 0, g));
  LSB_LAUNCHED(ctx, "k_seg_denom");
  LSB_CUDA(launch_pdl(ctx, k_seg_select, grid, dim3(kSegT), 0, g));
  LSB_LAUNCHED(ctx, "k_seg_select");
  return LSB_OK;
}

}  // namespace lsb
