// softmax_denom.cuh -- the reference's softmax denominator on the device
// (shared by K5a in k_select.cu and the segmented K5a in k_softmax_seg.cu).
//
// src/beam_decoder.cpp:46-74 sums e_j = exp(l_j - mx) in double SEQUENTIALLY
// in column order, then inv = float(1 / denom). The device sums the same e_j
// in a tree (per-thread runs, then a warp / block reduction, or per-segment
// partials added in segment order). f(x) = float(fl64(1 / x)) is monotone in
// x, so whenever an interval known to hold the sequential sum has the same f
// at both ends, that value IS the reference's inv. Three tiers:
//  1. the tree sum with the worst-case bound: the sequential sum is within
//     (n - 1) u S of the exact S and the tree within depth * u S (u = 2^-53),
//     tol = (n + 64) 2^-52 * tree. Fails for about (n 2^-52) / 2^-24 of rows
//     (1e-5 at 1-2k candidates, 2e-4 at 40k);
//  2. (rare; long rows only) a tight interval from one parallel pass over the row: the exact
//     sum S* by compensated (TwoSum) accumulation, and since each sequential
//     addition errs by at most min(e_k, ulp(S)/2) (it moves the running sum
//     by less than e_k, and rounds at the sum's ulp), the sequential sum lies
//     in S* +- sum_k min(e_k, ulp(S)/2) -- a bound set by the few terms above
//     ulp(S), orders of magnitude tighter than tier 1;
//  3. (far rarer) the sequential sum itself: e_j recomputed from the (still
//     unmodified) logits, one running sum added in column order.
#pragma once
#include <cstdint>

#include "glibc_log.cuh"
// (the rare tiers call glibc_exp_special -- the out-of-line full-domain exp,
// the same bits as glibc_exp -- so they add no register pressure to the
// kernels that inline glibc_exp in their hot loops)

namespace lsb {

// force_seq (test hook, LSB_SEQ_DENOM): 1 = skip tiers 1-2 (always the
// sequential sum), 2 = skip tier 1 (tier 2, then the sequential sum)
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

// Tier 2 by an NT-thread CTA (uniform arguments); returns true and the
// certified inv, or false. Out of line: rare.
template <int NT>
static __device__ __noinline__ bool tight_inv_cta(double tree, uint32_t n, const float* L,
                                                  double dmx, float* inv_out) {
  __shared__ double s_hi[NT / 32], s_c[NT / 32], s_b[NT / 32];
  // h >= ulp(S)/2 for every partial sum: S <= tree (1 + 2^-30) < 2 tree
  int ex;
  frexp(tree, &ex);                      // tree in [2^(ex-1), 2^ex)
  const double h = ldexp(1.0, ex - 52);  // ulp of [2^ex, 2^(ex+1)) / 2
  // any order: U loads in flight per thread
  constexpr int U = 4;
  double hi = 0.0, c = 0.0, b = 0.0;
  for (uint32_t k0 = threadIdx.x; k0 < n; k0 += U * NT) {
    float l[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = k0 + u * NT;
      l[u] = k < n ? L[k] : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double e = glibc_exp_special(static_cast<double>(l[u]) - dmx);  // 0 past n
      double err;
      two_sum(hi, e, hi, err);
      c = __dadd_rn(c, err);
      b = __dadd_rn(b, fmin(e, h));
    }
  }
  // (hi, c) pairs combine exactly up to c's roundings: warp shuffles, then
  // thread 0 over the warps
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
    const double c2 = __shfl_xor_sync(0xffffffffu, c, o);
    const double b2 = __shfl_xor_sync(0xffffffffu, b, o);
    double err;
    two_sum(hi, hi2, hi, err);
    c = __dadd_rn(c, __dadd_rn(c2, err));
    b = __dadd_rn(b, b2);
  }
  if ((threadIdx.x & 31) == 0) {
    s_hi[threadIdx.x >> 5] = hi;
    s_c[threadIdx.x >> 5] = c;
    s_b[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  __shared__ bool s_ok;
  __shared__ float s_inv;
  if (threadIdx.x == 0) {
    hi = 0.0;
    c = 0.0;
    b = 0.0;
    for (int t = 0; t < NT / 32; ++t) {
      double err;
      two_sum(hi, s_hi[t], hi, err);
      c = __dadd_rn(c, __dadd_rn(s_c[t], err));
      b = __dadd_rn(b, s_b[t]);
    }
    // S* = hi + c up to n^2 u^2 S (the compensations' own roundings) <=
    // 2^-60 S for n < 2^22; x = fl(hi + c) is within ulp(x)/2 of hi + c; the
    // bound b is a double sum of non-negative terms (relative error <= n u)
    const double x = __dadd_rn(hi, c);
    const double r = __dadd_rn(__dmul_rn(b, 1.0 + 0x1p-30), __dmul_rn(fabs(x), 0x1p-51));
    const double lo_end = __dsub_rn(x, r), hi_end = __dadd_rn(x, r);
    const float f_lo = static_cast<float>(1.0 / hi_end), f_hi = static_cast<float>(1.0 / lo_end);
    s_ok = lo_end > 0.0 && f_lo == f_hi;
    s_inv = f_lo;
  }
  __syncthreads();
  *inv_out = s_inv;
  return s_ok;
}

// extra_depth: additions beyond n in the tree (segment partials). TIER2: try
// the tight interval before the sequential sum -- for long rows (the
// full vocabulary: tier 1 fails for ~2e-4 of 40k-column rows and the
// sequential sum costs ~250 us); K5a's rows (<= 8k columns) go straight to
// the sequential sum (tier 2's registers would cost K5a occupancy: 64 -> 72+)
template <int NT, bool TIER2 = false>
__device__ __forceinline__ float reference_inv_cta(double tree, uint32_t n, const float* L,
                                                   double dmx, int force_seq,
                                                   uint32_t extra_depth = 0) {
  float inv;
  if (inv_certified(tree, n + extra_depth, force_seq, &inv)) return inv;
  if constexpr (TIER2)
    if (force_seq != 1 && tight_inv_cta<NT>(tree, n, L, dmx, &inv)) return inv;
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
