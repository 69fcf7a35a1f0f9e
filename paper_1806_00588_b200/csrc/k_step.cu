// k_step.cu -- the per-step hot path kernels.
//
//  K1+K2  k_probe_count   hash a hypothesis row (K1), probe the W cuckoo
//                         tables one warp per band (lanes 0/1 probe both
//                         tables) and walk each span coalesced, counting hits
//                         in shared-memory counters over a vocabulary slice.
//                         A word whose count reaches t sets its bit in the
//                         sentence's threshold bitmap (HBM/L2, atomicOr), so
//                         the dense B x |V| hit matrix of the reference
//                         (src/band_index.cpp:134-162) is never materialised.
//  K3     k_compact       bitmap U [0,T) U specials, provenance counters, and
//                         an ascending compaction: every 32-bit bitmap word is
//                         one warp ballot; per-word popcounts are prefix-summed
//                         across the CTA (src/candidate_selector.cpp:14-103).
//  K4     k_logits        logits = H . E[ids]^T + bias[ids]. PARITY mode keeps
//                         four lane accumulators per output and adds
//                         fl(h*e) in the reference's SSE order without FMA
//                         (src/beam_decoder.cpp:34-42), bit-identical logits.
//                         FAST mode uses one FFMA chain.
//  K5a    k_softmax_topb  one warp per row: float max, double exp / sum,
//                         float(1/denom) scale (src/beam_decoder.cpp:46-74) and
//                         a per-row top-B by (p desc, column asc).
//  K5b    k_expand        per sentence: B-round tournament over the per-row
//                         lists and frozen hypotheses by (score desc, beam asc,
//                         word asc), score = cum + log((double)p)
//                         (src/beam_decoder.cpp:76-111), then the parent-row
//                         gather of the hidden state (the paper's "hidden-state
//                         reorder"), replacing its D2H copy + CPU heapsort.
#include <algorithm>
#include <cfloat>

#include "k_step.cuh"

namespace lsb {

// =================================================================== K1+K2
__global__ void __launch_bounds__(512) k_probe_count(ProbeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const IndexView& ix = a.ix;
  const int row = blockIdx.x;
  const int s = row / a.B, i = row % a.B;
  if (a.n_hyp && i >= a.n_hyp[s]) return;
  if (a.finished && a.finished[row]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const uint32_t lo = blockIdx.y * a.slice_len;
  const uint32_t hi = min(ix.V, lo + a.slice_len);
  const bool count = a.t > 0;
  const size_t cbytes = count ? ((static_cast<size_t>(a.slice_len) * a.counter_bytes + 15) & ~size_t(15)) : 0;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
  float* h = reinterpret_cast<float*>(smem + cbytes);
  const int dpad = (ix.d + 3) & ~3;
  uint32_t* codes = reinterpret_cast<uint32_t*>(h + dpad);
  uint8_t* idx = reinterpret_cast<uint8_t*>(codes + ix.W);

  for (size_t k = threadIdx.x; k < cbytes / 16; k += blockDim.x)
    reinterpret_cast<uint4*>(cnt)[k] = make_uint4(0, 0, 0, 0);
  const float* src = a.hidden + static_cast<size_t>(row) * ix.d;
  int nan = 0;
  if ((ix.d & 3) == 0) {
    for (int c = threadIdx.x; c < (ix.d >> 2); c += blockDim.x) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(src) + c);
      nan |= isnan(v.x) | isnan(v.y) | isnan(v.z) | isnan(v.w);
      reinterpret_cast<float4*>(h)[c] = v;
    }
  } else {
    for (int c = threadIdx.x; c < ix.d; c += blockDim.x) {
      const float v = __ldg(src + c);
      nan |= isnan(v);
      h[c] = v;
    }
  }
  if (__syncthreads_or(nan)) {
    if (threadIdx.x == 0) atomicOr(a.err, kErrNaN);
    return;
  }
  // K1: windowed argmax per permutation, ties to the smallest k.
  for (int p = threadIdx.x; p < ix.P; p += blockDim.x) {
    const uint32_t* pr = ix.perms + static_cast<size_t>(p) * ix.K;
    uint32_t best = 0;
    float bv = h[__ldg(pr)];
    for (int k = 1; k < ix.K; ++k) {
      const float v = h[__ldg(pr + k)];
      if (v > bv) {
        bv = v;
        best = k;
      }
    }
    idx[p] = static_cast<uint8_t>(best);
  }
  __syncthreads();
  for (int w = threadIdx.x; w < ix.W; w += blockDim.x) {
    uint32_t code = 0;
    for (int b = 0; b < ix.u; ++b) code |= static_cast<uint32_t>(idx[w * ix.u + b]) << (b * ix.bits);
    codes[w] = code;
    if (blockIdx.y == 0) a.qcodes[static_cast<size_t>(row) * ix.W + w] = code;
  }
  __syncthreads();
  if (!count) return;
  // K2: one warp per band; walk the span, count hits in the slice.
  uint32_t* bm = a.bitmap + static_cast<size_t>(s) * a.nwords;
  const uint32_t t = static_cast<uint32_t>(a.t);
  for (int w = warp; w < ix.W; w += nwarp) {
    uint32_t start, len;
    if (!warp_probe(ix, w, codes[w], start, len)) continue;
    const uint32_t* ids = ix.word_ids + static_cast<size_t>(w) * ix.V + start;
    for (uint32_t k = lane; k < len; k += 32) {
      const uint32_t id = __ldg(ids + k);
      if (id < lo || id >= hi) continue;
      const uint32_t local = id - lo;
      uint32_t c;
      if (a.counter_bytes == 1) {
        const uint32_t sh = (local & 3) * 8;
        c = (atomicAdd(cnt + (local >> 2), 1u << sh) >> sh) & 0xFFu;
      } else {
        const uint32_t sh = (local & 1) * 16;
        c = (atomicAdd(cnt + (local >> 1), 1u << sh) >> sh) & 0xFFFFu;
      }
      if (c + 1 == t) atomicOr(bm + (id >> 5), 1u << (id & 31));
    }
  }
}

lsb_status launch_probe(lsb_ctx* ctx, const ProbeArgs& a) {
  const IndexView& ix = a.ix;
  const uint32_t nslices = a.t > 0 ? (ix.V + a.slice_len - 1) / a.slice_len : 1;
  const size_t cbytes =
      a.t > 0 ? ((static_cast<size_t>(a.slice_len) * a.counter_bytes + 15) & ~size_t(15)) : 0;
  const size_t smem = cbytes + ((ix.d + 3) & ~3) * 4 + ix.W * 4 + ix.P + 16;
  if (smem > ctx->smem_optin) {
    set_error("probe: shared memory budget exceeded");
    return LSB_EINVAL;
  }
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    LSB_CUDA(cudaFuncSetAttribute(k_probe_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  dim3 grid(a.S * a.B, std::max(1u, nslices));
  k_probe_count<<<grid, 512, smem, ctx->stream>>>(a);
  LSB_LAUNCHED(ctx, "k_probe_count");
  return LSB_OK;
}

// ====================================================================== K3
__device__ __forceinline__ uint32_t below_mask(uint32_t word, uint32_t T) {
  // bits of ids < T inside bitmap word `word`
  const uint32_t base = word * 32;
  if (T >= base + 32) return 0xFFFFFFFFu;
  if (T <= base) return 0u;
  return (1u << (T - base)) - 1u;
}

__device__ __forceinline__ uint32_t valid_mask(uint32_t word, uint32_t V) {
  return below_mask(word, V);
}

__device__ uint32_t block_scan_excl(uint32_t v, uint32_t* wsum, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarp = (blockDim.x + 31) >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t z = lane < nwarp ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < nwarp) wsum[lane] = z;
    if (lane == 31) wsum[32] = z;
  }
  __syncthreads();
  const uint32_t r = (warp ? wsum[warp - 1] : 0) + x - v;
  if (total) *total = wsum[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) k_compact(CompactArgs a) {
  extern __shared__ uint32_t bm[];  // nwords
  __shared__ uint32_t wsum[33];
  __shared__ uint32_t s_thr, s_below, s_spec;
  const int s = blockIdx.x;
  uint32_t* ids = a.ids + static_cast<size_t>(s) * a.ncap;
  if (a.mode != 0) {
    // t == 0 (every word survives, src/candidate_selector.cpp:21-27) or
    // full vocabulary: the candidate list is the identity; ids are implicit.
    if (threadIdx.x == 0) {
      a.n_cand[s] = a.V;
      a.prov[3 * s] = a.mode == 1 ? a.V : 0;
      a.prov[3 * s + 1] = 0;
      a.prov[3 * s + 2] = 0;
    }
    return;
  }
  const uint32_t nw = a.nwords;
  if (threadIdx.x == 0) {
    s_thr = 0;
    s_below = 0;
    s_spec = 0;
  }
  uint32_t thr = 0, below = 0;
  for (uint32_t w = threadIdx.x; w < nw; w += blockDim.x) {
    uint32_t m = a.bitmap_in ? a.bitmap_in[static_cast<size_t>(s) * nw + w] : 0u;
    if (a.bitmap_clear) a.bitmap_clear[static_cast<size_t>(s) * nw + w] = 0u;
    m &= valid_mask(w, a.V);
    bm[w] = m;
    thr += __popc(m);
    below += __popc(m & below_mask(w, a.T));
  }
  __syncthreads();
  atomicAdd(&s_thr, thr);
  atomicAdd(&s_below, below);
  // specials >= T that are not threshold survivors are new
  // (src/candidate_selector.cpp:85-101); specials < T are inside [0,T).
  for (int k = threadIdx.x; k < a.nspec; k += blockDim.x) {
    const uint32_t id = a.specials[k];
    if (id >= a.T) {
      const uint32_t bit = 1u << (id & 31);
      const uint32_t old = atomicOr(&bm[id >> 5], bit);
      if (!(old & bit)) atomicAdd(&s_spec, 1u);
    }
  }
  __syncthreads();
  // [0, T) prefix, then per-thread contiguous word ranges for the ordered emit
  const uint32_t per = (nw + blockDim.x - 1) / blockDim.x;
  const uint32_t w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
  uint32_t cnt = 0;
  for (uint32_t w = w0; w < w1; ++w) {
    const uint32_t m = bm[w] | below_mask(w, a.T);
    bm[w] = m;
    cnt += __popc(m);
  }
  uint32_t total;
  uint32_t base = block_scan_excl(cnt, wsum, &total);
  for (uint32_t w = w0; w < w1; ++w) {
    uint32_t m = bm[w];
    while (m) {
      const int b = __ffs(m) - 1;
      ids[base++] = w * 32 + b;
      m &= m - 1;
    }
  }
  if (threadIdx.x == 0) {
    a.n_cand[s] = total;
    a.prov[3 * s] = s_thr;
    a.prov[3 * s + 1] = a.T - s_below;
    a.prov[3 * s + 2] = s_spec;
    if (total == 0 && a.empty_is_error) {
      bool live = true;
      if (a.n_hyp) {
        live = false;
        for (int i = 0; i < a.n_hyp[s]; ++i)
          live |= !(a.finished && a.finished[static_cast<size_t>(s) * a.B + i]);
      }
      if (live) atomicOr(a.err, kErrEmptyCands);
    }
  }
}

lsb_status launch_compact(lsb_ctx* ctx, const CompactArgs& a, int S) {
  const size_t smem = static_cast<size_t>(a.nwords) * 4;
  if (smem > ctx->smem_optin) return set_error("compact: vocabulary too large"), LSB_EINVAL;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    LSB_CUDA(cudaFuncSetAttribute(k_compact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  k_compact<<<S, 1024, smem, ctx->stream>>>(a);
  LSB_LAUNCHED(ctx, "k_compact");
  return LSB_OK;
}

__global__ void k_bitmap_from_dense(const int32_t* __restrict__ L, int B, uint32_t V, int t,
                                    uint32_t* __restrict__ bitmap) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  bool keep = false;
  if (j < V)
    for (int i = 0; i < B && !keep; ++i) keep = L[static_cast<size_t>(i) * V + j] >= t;
  const unsigned ballot = __ballot_sync(0xffffffffu, keep);
  if ((threadIdx.x & 31) == 0 && j < V) bitmap[j >> 5] = ballot;
}

__global__ void k_bitmap_from_ids(const uint32_t* __restrict__ ids, uint32_t n,
                                  uint32_t* __restrict__ bitmap) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) atomicOr(bitmap + (ids[k] >> 5), 1u << (ids[k] & 31));
}

lsb_status launch_bitmap_from_dense(lsb_ctx* ctx, const int32_t* L, int B, uint32_t V, int t,
                                    uint32_t* bitmap) {
  const uint32_t blocks = (V + 255) / 256;
  if (!blocks) return LSB_OK;
  k_bitmap_from_dense<<<blocks, 256, 0, ctx->stream>>>(L, B, V, t, bitmap);
  LSB_LAUNCHED(ctx, "k_bitmap_from_dense");
  return LSB_OK;
}

lsb_status launch_bitmap_from_ids(lsb_ctx* ctx, const uint32_t* ids, uint32_t n,
                                  uint32_t* bitmap) {
  if (!n) return LSB_OK;
  k_bitmap_from_ids<<<(n + 255) / 256, 256, 0, ctx->stream>>>(ids, n, bitmap);
  LSB_LAUNCHED(ctx, "k_bitmap_from_ids");
  return LSB_OK;
}

__global__ void k_gather(const float* __restrict__ E, int d, const uint32_t* __restrict__ ids,
                         uint32_t n, float* __restrict__ out) {
  const uint32_t r = blockIdx.x;
  if (r >= n) return;
  const float* src = E + static_cast<size_t>(ids[r]) * d;
  float* dst = out + static_cast<size_t>(r) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) dst[c] = __ldg(src + c);
}

lsb_status launch_gather(lsb_ctx* ctx, const float* E, int d, const uint32_t* ids, uint32_t n,
                         float* out) {
  if (!n) return LSB_OK;
  k_gather<<<n, 256, 0, ctx->stream>>>(E, d, ids, n, out);
  LSB_LAUNCHED(ctx, "k_gather");
  return LSB_OK;
}

// ====================================================================== K4
constexpr int kLogitThreads = 128;
constexpr int kDC = 256;  // columns of H staged per chunk

template <int RB, int CB, bool PARITY, bool VEC>
__global__ void __launch_bounds__(kLogitThreads) k_logits(LogitsArgs a) {
  __shared__ __align__(16) float hs[RB][kDC];
  constexpr int CT = kLogitThreads * CB;
  const int d = a.d;
  const int d4 = d >= 4 ? (d & ~3) : 0;

  int row0, rowlim, ncols;
  uint32_t col0;
  const uint32_t* cid = nullptr;  // null: identity ids starting at col0
  int tile_first, tile_step;
  int s = 0;
  if (static_cast<int>(blockIdx.x) < a.jobs_shared) {
    const int rg = blockIdx.x / a.ctiles_shared, ct = blockIdx.x % a.ctiles_shared;
    row0 = rg * RB;
    rowlim = a.R_total;
    col0 = ct * CT;
    ncols = static_cast<int>(min(static_cast<uint32_t>(CT), a.n_shared - col0));
    tile_first = 0;
    tile_step = 1;
  } else {
    const int e = blockIdx.x - a.jobs_shared;
    s = e / (a.G * a.X);
    const int g = (e / a.X) % a.G;
    row0 = s * a.Bsent + g * RB;
    rowlim = s * a.Bsent + a.Bsent;
    tile_first = e % a.X;
    tile_step = a.X;
    col0 = 0;
    ncols = 0;
  }
  const bool shared_job = static_cast<int>(blockIdx.x) < a.jobs_shared;
  const uint32_t m = shared_job ? 0u
                                : (a.n_cand[s] > a.n_shared ? a.n_cand[s] - a.n_shared : 0u);
  for (int tile = tile_first;; tile += tile_step) {
    if (!shared_job) {
      if (static_cast<uint32_t>(tile) * CT >= m) break;
      col0 = a.n_shared + tile * CT;
      ncols = static_cast<int>(min(static_cast<uint32_t>(CT), m - tile * CT));
      cid = a.ids + static_cast<size_t>(s) * a.ncap + col0;
    } else if (tile > 0) {
      break;
    }
    uint32_t id[CB];
    bool cv[CB];
    const float* er[CB];
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      const int c = threadIdx.x + kLogitThreads * cb;
      cv[cb] = c < ncols;
      id[cb] = cv[cb] ? (cid ? __ldg(cid + c) : col0 + c) : (cid ? __ldg(cid) : col0);
      er[cb] = a.E + static_cast<size_t>(id[cb]) * d;
    }
    float acc[RB][CB][PARITY ? 4 : 1];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
      for (int cb = 0; cb < CB; ++cb)
#pragma unroll
        for (int k = 0; k < (PARITY ? 4 : 1); ++k) acc[rb][cb][k] = 0.0f;

    for (int c0 = 0; c0 < d; c0 += kDC) {
      const int kw = min(kDC, d - c0);
      __syncthreads();
      for (int q = threadIdx.x; q < RB * kDC; q += kLogitThreads) {
        const int rb = q / kDC, k = q % kDC;
        const int r = row0 + rb;
        hs[rb][k] = (k < kw && r < rowlim) ? __ldg(a.H + static_cast<size_t>(r) * d + c0 + k) : 0.0f;
      }
      __syncthreads();
      const int kv = max(0, min(kw, d4 - c0));  // columns in full 4-lane groups
      if (ncols > 0) {
#pragma unroll 2
        for (int k = 0; k < kv; k += 4) {
          float4 e[CB];
#pragma unroll
          for (int cb = 0; cb < CB; ++cb) {
            if (VEC) {
              e[cb] = __ldg(reinterpret_cast<const float4*>(er[cb] + c0 + k));
            } else {
              e[cb].x = __ldg(er[cb] + c0 + k);
              e[cb].y = __ldg(er[cb] + c0 + k + 1);
              e[cb].z = __ldg(er[cb] + c0 + k + 2);
              e[cb].w = __ldg(er[cb] + c0 + k + 3);
            }
          }
#pragma unroll
          for (int rb = 0; rb < RB; ++rb) {
            const float4 hv = *reinterpret_cast<const float4*>(&hs[rb][k]);
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) {
              if (PARITY) {
                acc[rb][cb][0] = __fadd_rn(acc[rb][cb][0], __fmul_rn(hv.x, e[cb].x));
                acc[rb][cb][1] = __fadd_rn(acc[rb][cb][1], __fmul_rn(hv.y, e[cb].y));
                acc[rb][cb][2] = __fadd_rn(acc[rb][cb][2], __fmul_rn(hv.z, e[cb].z));
                acc[rb][cb][3] = __fadd_rn(acc[rb][cb][3], __fmul_rn(hv.w, e[cb].w));
              } else {
                float x = acc[rb][cb][0];
                x = fmaf(hv.x, e[cb].x, x);
                x = fmaf(hv.y, e[cb].y, x);
                x = fmaf(hv.z, e[cb].z, x);
                x = fmaf(hv.w, e[cb].w, x);
                acc[rb][cb][0] = x;
              }
            }
          }
        }
        // tail columns (d mod 4 when d >= 4, or all of d < 4) go to lane 0
        for (int k = kv; k < kw; ++k) {
          float ev[CB];
#pragma unroll
          for (int cb = 0; cb < CB; ++cb) ev[cb] = __ldg(er[cb] + c0 + k);
#pragma unroll
          for (int rb = 0; rb < RB; ++rb)
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) {
              if (PARITY)
                acc[rb][cb][0] = __fadd_rn(__fmul_rn(hs[rb][k], ev[cb]), acc[rb][cb][0]);
              else
                acc[rb][cb][0] = fmaf(hs[rb][k], ev[cb], acc[rb][cb][0]);
            }
        }
      }
    }
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      if (!cv[cb]) continue;
      const float bias = a.bias ? __ldg(a.bias + id[cb]) : 0.0f;
      const uint32_t col = col0 + threadIdx.x + kLogitThreads * cb;
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        const int r = row0 + rb;
        if (r >= rowlim) continue;
        float v;
        if (PARITY) {
          v = __fadd_rn(0.0f, acc[rb][cb][0]);
          v = __fadd_rn(v, acc[rb][cb][1]);
          v = __fadd_rn(v, acc[rb][cb][2]);
          v = __fadd_rn(v, acc[rb][cb][3]);
        } else {
          v = acc[rb][cb][0];
        }
        if (a.bias) v = __fadd_rn(v, bias);
        a.out[static_cast<size_t>(r) * a.ldo + col] = v;
      }
    }
  }
}

int choose_rb(int B) {
  static const int opts[] = {16, 12, 10, 8, 6, 4, 2, 1};
  int best = 1, best_pad = 1 << 30;
  for (int rb : opts) {
    if (rb > B && rb != 1) continue;
    const int pad = ((B + rb - 1) / rb) * rb - B;
    const int groups = (B + rb - 1) / rb;
    // fewest groups first (fewest H re-reads), then least padding
    const int cost = groups * 64 + pad;
    if (cost < best_pad) {
      best_pad = cost;
      best = rb;
    }
  }
  return best;
}

template <int RB, int CB>
static lsb_status launch_logits_rb(lsb_ctx* ctx, LogitsArgs a, lsb_mode mode, int target) {
  constexpr int CT = kLogitThreads * CB;
  const int rgroups = (a.R_total + RB - 1) / RB;
  a.ctiles_shared = static_cast<int>((a.n_shared + CT - 1) / CT);
  a.jobs_shared = a.n_shared ? rgroups * a.ctiles_shared : 0;
  a.G = (a.Bsent + RB - 1) / RB;
  if (a.ids && a.S > 0) {
    const int want = std::max(1, (target - a.jobs_shared) / std::max(1, a.S * a.G));
    a.X = std::min(want, 64);
  } else {
    a.X = 0;
  }
  const int grid = a.jobs_shared + a.S * a.G * a.X;
  if (grid == 0) return LSB_OK;
  const bool vec = (a.d & 3) == 0 && (reinterpret_cast<uintptr_t>(a.E) & 15) == 0;
  if (mode == LSB_MODE_PARITY) {
    if (vec) k_logits<RB, CB, true, true><<<grid, kLogitThreads, 0, ctx->stream>>>(a);
    else k_logits<RB, CB, true, false><<<grid, kLogitThreads, 0, ctx->stream>>>(a);
  } else {
    if (vec) k_logits<RB, CB, false, true><<<grid, kLogitThreads, 0, ctx->stream>>>(a);
    else k_logits<RB, CB, false, false><<<grid, kLogitThreads, 0, ctx->stream>>>(a);
  }
  LSB_LAUNCHED(ctx, "k_logits");
  return LSB_OK;
}

lsb_status launch_logits(lsb_ctx* ctx, LogitsArgs a, lsb_mode mode, int target_ctas) {
  switch (choose_rb(a.Bsent)) {
    case 16: return launch_logits_rb<16, 1>(ctx, a, mode, target_ctas);
    case 12: return launch_logits_rb<12, 2>(ctx, a, mode, target_ctas);
    case 10: return launch_logits_rb<10, 2>(ctx, a, mode, target_ctas);
    case 8: return launch_logits_rb<8, 2>(ctx, a, mode, target_ctas);
    case 6: return launch_logits_rb<6, 2>(ctx, a, mode, target_ctas);
    case 4: return launch_logits_rb<4, 2>(ctx, a, mode, target_ctas);
    case 2: return launch_logits_rb<2, 2>(ctx, a, mode, target_ctas);
    default: return launch_logits_rb<1, 2>(ctx, a, mode, target_ctas);
  }
}

// ===================================================================== K5a
__device__ __forceinline__ bool top_better(float pa, uint32_t ra, float pb, uint32_t rb) {
  return pa > pb || (pa == pb && ra < rb);
}

__device__ void select_topb(const SoftmaxArgs& a, int row, float* L, uint32_t n, float inv,
                            float* lp, uint32_t* lr, bool given);

__global__ void k_softmax_topb(SoftmaxArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int row = blockIdx.x * wpb + warp;
  if (row >= a.R_total) return;
  const int s = row / a.Bsent, i = row % a.Bsent;
  const bool live = !(a.n_hyp && i >= a.n_hyp[s]) && !(a.finished && a.finished[row]);
  if (!live) {
    if (lane == 0) a.top_n[row] = 0;
    return;
  }
  const int B = a.topB;
  float* lp = reinterpret_cast<float*>(smem) + static_cast<size_t>(warp) * B * 64;
  uint32_t* lr = reinterpret_cast<uint32_t*>(lp + B * 32);
  const uint32_t n = a.n_cand ? a.n_cand[s] : a.n_const;
  float* L = a.logits + static_cast<size_t>(row) * a.ldl;
  if (a.probs_in) {  // expand_beams over given probabilities: selection only
    select_topb(a, row, L, n, 1.0f, lp, lr, true);
    return;
  }
  // float max, as std::max over the row (src/beam_decoder.cpp:55)
  float mx = -INFINITY;
  for (uint32_t r = lane; r < n; r += 32) {
    const float v = L[r];
    mx = (mx < v) ? v : mx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (mx < y) ? y : mx;
  }
  if (n == 0 || (isinf(mx) && mx < 0)) {
    if (lane == 0) {
      atomicOr(a.err, kErrEmptyRow);
      a.top_n[row] = 0;
    }
    return;
  }
  // e = exp((double)l - mx) in double; float(e) kept; denominator in double
  double sum = 0.0;
  const double dmx = static_cast<double>(mx);
  for (uint32_t r = lane; r < n; r += 32) {
    const double e = exp(static_cast<double>(L[r]) - dmx);
    L[r] = static_cast<float>(e);
    sum += e;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = static_cast<float>(1.0 / sum);
  select_topb(a, row, L, n, inv, lp, lr, false);
}

// Per-lane sorted top-B lists (columns ascend per lane, so an equal p never
// displaces an earlier column), then a 32-way warp merge.
__device__ void select_topb(const SoftmaxArgs& a, int row, float* L, uint32_t n, float inv,
                            float* lp, uint32_t* lr, bool given) {
  const int lane = threadIdx.x & 31;
  const int B = a.topB;
  if (B <= 0) {
    if (lane == 0) a.top_n[row] = 0;
    return;
  }
  int cnt = 0;
  for (uint32_t r = lane; r < n; r += 32) {
    const float p = given ? L[r] : __fmul_rn(L[r], inv);
    if (a.keep_probs && !given) L[r] = p;
    if (cnt == B && !(p > lp[(B - 1) * 32 + lane])) continue;
    int j = cnt < B ? cnt++ : B - 1;
    while (j > 0 && lp[(j - 1) * 32 + lane] < p) {
      lp[j * 32 + lane] = lp[(j - 1) * 32 + lane];
      lr[j * 32 + lane] = lr[(j - 1) * 32 + lane];
      --j;
    }
    lp[j * 32 + lane] = p;
    lr[j * 32 + lane] = r;
  }
  // 32-way merge of the lane lists
  const int keep = static_cast<int>(min(static_cast<uint32_t>(B), n));
  int head = 0;
  TopEntry* out = a.top + static_cast<size_t>(row) * B;
  for (int k = 0; k < keep; ++k) {
    float bp = head < cnt ? lp[head * 32 + lane] : -1.0f;
    uint32_t br = head < cnt ? lr[head * 32 + lane] : 0xFFFFFFFFu;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float yp = __shfl_xor_sync(0xffffffffu, bp, o);
      const uint32_t yr = __shfl_xor_sync(0xffffffffu, br, o);
      if (top_better(yp, yr, bp, br)) {
        bp = yp;
        br = yr;
      }
    }
    if ((br & 31) == static_cast<uint32_t>(lane)) ++head;
    if (lane == 0) out[k] = TopEntry{bp, br};
  }
  if (lane == 0) a.top_n[row] = keep;
}

lsb_status launch_softmax(lsb_ctx* ctx, const SoftmaxArgs& a) {
  if (a.R_total == 0) return LSB_OK;
  const size_t per_warp = static_cast<size_t>(a.topB) * 64 * 4;
  int wpb = static_cast<int>(std::max<size_t>(1, std::min<size_t>(4, (96 * 1024) / per_warp)));
  const size_t smem = per_warp * wpb;
  if (smem > ctx->smem_optin) return set_error("softmax: beam too large"), LSB_EINVAL;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    LSB_CUDA(cudaFuncSetAttribute(k_softmax_topb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  k_softmax_topb<<<(a.R_total + wpb - 1) / wpb, wpb * 32, smem, ctx->stream>>>(a);
  LSB_LAUNCHED(ctx, "k_softmax_topb");
  return LSB_OK;
}

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

// Lists: [0, nfz) frozen singletons, then one list per live row.
__global__ void k_expand(ExpandArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int s = blockIdx.x;
  const int R = a.Bsent;
  const int nfz_explicit = a.frozen_mode ? a.nfrozen : 0;
  const int nl = nfz_explicit + R;
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
    const double cum = a.scores[rbase + row];
    sc = cum + log(static_cast<double>(e.p));
    if (a.id_map) wd = a.id_map[e.r];
    else wd = (e.r < a.n_shared || !ids) ? static_cast<long long>(e.r) : static_cast<long long>(ids[e.r]);
  };
  if (threadIdx.x < 32) {
    for (int l = lane; l < nl; l += 32) {
      int len = 0;
      double sc = -INFINITY;
      long long wd = 0;
      uint32_t beam = 0;
      if (l < nfz_explicit) {
        len = 1;
        sc = a.fz_score[l];
        wd = -1;
        beam = a.fz_beam[l];
      } else {
        const int row = l - nfz_explicit;
        beam = a.live_ids ? a.live_ids[rbase + row] : static_cast<uint32_t>(row);
        if (row < nhyp) {
          const bool fin = a.finished && a.finished[rbase + row];
          if (fin) {  // frozen hypothesis competes with its carried score
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
        a.choices[static_cast<size_t>(s) * a.topB + k] = lsb_choice{best.score, best.beam, 0u,
                                                                   static_cast<int64_t>(best.word)};
        if (k < 64) s_beams[k] = best.beam;
      }
      if ((bl & 31) == lane) {  // owner advances its list head
        const int np = ++hpos[bl];
        if (np < hlen[bl]) {
          double sc;
          long long wd;
          live_score(bl - nfz_explicit, np, sc, wd);
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
  if (!a.hidden_out || !a.hidden) return;
  // hidden-state reorder: child k starts from its parent's hidden vector
  const int count = min(s_count, 64);
  const int d = a.d;
  for (int k = 0; k < count; ++k) {
    const float* src = a.hidden + (rbase + s_beams[k]) * d;
    float* dst = a.hidden_out + (static_cast<size_t>(s) * a.topB + k) * d;
    if ((d & 3) == 0) {
      for (int c = threadIdx.x; c < (d >> 2); c += blockDim.x)
        reinterpret_cast<float4*>(dst)[c] = __ldg(reinterpret_cast<const float4*>(src) + c);
    } else {
      for (int c = threadIdx.x; c < d; c += blockDim.x) dst[c] = __ldg(src + c);
    }
  }
}

lsb_status launch_expand(lsb_ctx* ctx, const ExpandArgs& a) {
  if (a.S == 0) return LSB_OK;
  const int nl = (a.frozen_mode ? a.nfrozen : 0) + a.Bsent;
  const size_t smem = static_cast<size_t>(nl) * (8 + 8 + 4 + 4 + 4) + 16;
  if (smem > ctx->smem_optin) return set_error("expand: too many rows"), LSB_EINVAL;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    LSB_CUDA(cudaFuncSetAttribute(k_expand, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  k_expand<<<a.S, 256, smem, ctx->stream>>>(a);
  LSB_LAUNCHED(ctx, "k_expand");
  return LSB_OK;
}

}  // namespace lsb
