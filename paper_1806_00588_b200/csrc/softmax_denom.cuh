// softmax_denom.cuh -- the reference's softmax denominator on the device
// (shared by K5a in k_select.cu and the segmented K5a in k_softmax_seg.cu).
//
// src/beam_decoder.cpp:46-74 sums e_j = exp(l_j - mx) in double SEQUENTIALLY
// in column order, then inv = float(1 / denom). f(x) = float(fl64(1 / x)) is
// monotone in x, so whenever an interval known to hold the sequential sum has
// the same f at both ends, that value IS the reference's inv.
//  * K5a (rows up to 8k columns): the tree sum (per-thread runs, then a block
//    reduction) with the worst-case bound -- the sequential sum is within
//    (n - 1) u S of the exact S and the tree within depth * u S (u = 2^-53),
//    so tol = (n + 64) 2^-52 * tree. It fails for about n 2^-28 of rows
//    (1e-5 at 1-2k candidates).
//  * The segmented K5a (the full vocabulary): the exact sum S* by compensated
//    (TwoSum) accumulation, and the bound sum_k min(e_k, 2^-52) on the
//    sequential sum's error -- each sequential addition moves the running sum
//    by less than e_k and rounds at half the sum's ulp. That interval is set
//    by the few terms above ulp(S): it fails for ~1e-6 of rows.
//  * Otherwise: the sequential sum itself, e_j recomputed from the (still
//    unmodified) logits, one running sum added in column order.
#pragma once
#include <cstdint>

#include "glibc_log.cuh"
// (the sequential sums call glibc_exp_special -- the out-of-line full-domain
// exp, the same bits as glibc_exp -- so they add no register pressure to the
// kernels that inline glibc_exp in their hot loops)

namespace lsb {

// force_seq (test hook, LSB_SEQ_DENOM=1): always the sequential sum
__device__ __forceinline__ bool inv_certified(double tree, uint32_t n, int force_seq, float* inv) {
  const double tol = static_cast<double>(n + 64) * 0x1p-52 * tree;
  const float lo = static_cast<float>(1.0 / (tree + tol));
  const float hi = static_cast<float>(1.0 / (tree - tol));
  *inv = lo;
  return lo == hi && !force_seq;
}

// The sequential sum by an NT-thread CTA: e_j recomputed NT at a time into
// shared memory, thread 0 adding them in column order. Out of line: rare.
template <int NT>
static __device__ __noinline__ float sequential_inv_cta(uint32_t n, const float* L, double dmx) {
  // rounds of U*NT terms: every thread computes U of them (loads in flight),
  // then thread 0 adds the round in column order (U small: the kernel's
  // static shared memory, i.e. K5a's occupancy, carries this buffer)
  constexpr int U = 1;
  __shared__ double s_e[U * NT];
  __shared__ float s_inv;
  double seq = 0.0;
  for (uint32_t c0 = 0; c0 < n; c0 += U * NT) {
    __syncthreads();  // the previous round's s_e has been added
    float l[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t c = c0 + u * NT + threadIdx.x;
      l[u] = c < n ? L[c] : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s_e[u * NT + threadIdx.x] = glibc_exp_special(static_cast<double>(l[u]) - dmx);
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t m = min(static_cast<uint32_t>(U * NT), n - c0);
      for (uint32_t k = 0; k < m; ++k) seq = __dadd_rn(seq, s_e[k]);
    }
  }
  if (threadIdx.x == 0) s_inv = static_cast<float>(1.0 / seq);
  __syncthreads();
  return s_inv;
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& err) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// (hi, c) pairs: hi + c tracks an exact sum (c accumulates the TwoSum
// errors; its own roundings stay below n^2 u^2 S)
__device__ __forceinline__ void dd_add(double& hi, double& c, double e) {
  double err;
  two_sum(hi, e, hi, err);
  c = __dadd_rn(c, err);
}
__device__ __forceinline__ void dd_merge(double& hi, double& c, double hi2, double c2) {
  double err;
  two_sum(hi, hi2, hi, err);
  c = __dadd_rn(c, __dadd_rn(c2, err));
}

// The interval test for an exact sum hi + c and b = sum_k min(e_k, 2^-52):
// true and the reference's inv, or false. Every sequential partial sum lies
// below 2^ex (S_seq < x (1 + 2^-20)), where one addition errs by at most
// min(e_k, 2^(ex-53)) <= max(1, 2^(ex-1)) min(e_k, 2^-52).
__device__ __forceinline__ bool inv_from_exact(double hi, double c, double b, float* inv) {
  const double x = __dadd_rn(hi, c);
  int ex;
  frexp(__dmul_rn(x, 1.0 + 0x1p-20), &ex);  // x (1 + 2^-20) in [2^(ex-1), 2^ex)
  const double scale = ex > 1 ? ldexp(1.0, ex - 1) : 1.0;
  // b: a double sum of non-negative terms (relative error < 2^-30); hi + c:
  // exact to 2^-60 S; x within ulp(x)/2 of it; the endpoints round once more
  const double r = __dadd_rn(__dmul_rn(__dmul_rn(b, scale), 1.0 + 0x1p-30), __dmul_rn(x, 0x1p-50));
  const double lo_end = __dsub_rn(x, r), hi_end = __dadd_rn(x, r);
  const float f_lo = static_cast<float>(1.0 / hi_end), f_hi = static_cast<float>(1.0 / lo_end);
  *inv = f_lo;
  return lo_end > 0.0 && f_lo == f_hi;
}

template <int NT>
__device__ __forceinline__ float reference_inv_cta(double tree, uint32_t n, const float* L,
                                                   double dmx, int force_seq) {
  float inv;
  if (inv_certified(tree, n, force_seq, &inv)) return inv;
  return sequential_inv_cta<NT>(n, L, dmx);
}

// Warp-wide (the fused K5's warp per row): every lane adds the same shuffled
// terms, so every lane ends with the reference's sum.
static __device__ __noinline__ float sequential_inv_warp(uint32_t n, const float* L, double dmx,
                                                         int lane) {
  double seq = 0.0;
  for (uint32_t c0 = 0; c0 < n; c0 += 32) {
    const uint32_t c = c0 + lane;
    const double e = c < n ? glibc_exp_special(static_cast<double>(L[c]) - dmx) : 0.0;
    const int m = static_cast<int>(min(32u, n - c0));
    for (int k = 0; k < m; ++k) seq = __dadd_rn(seq, __shfl_sync(0xffffffffu, e, k));
  }
  return static_cast<float>(1.0 / seq);
}
__device__ __forceinline__ float reference_inv_warp(double tree, uint32_t n, const float* L,
                                                    double dmx, int lane, int force_seq) {
  float inv;
  if (inv_certified(tree, n, force_seq, &inv)) return inv;
  return sequential_inv_warp(n, L, dmx, lane);
}

}  // namespace lsb
