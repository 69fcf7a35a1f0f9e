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
//  K4 (k_logits.cu) and K5 (k_select.cu) live in their own files.
#include <algorithm>
#include <cfloat>

#include "k_step.cuh"

namespace lsb {

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

static __device__ uint32_t block_scan_excl(uint32_t v, uint32_t* wsum, uint32_t* total) {
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

// One sentence's K3 by the whole CTA (any blockDim <= 1024): bm = nwords
// words of shared memory. k_compact runs a CTA per sentence; the fused
// small-batch step (k_step_fused.cu) calls it from a persistent CTA.
static __device__ void compact_sentence(const CompactArgs& a, int s, uint32_t* bm) {
  __shared__ uint32_t wsum[33];
  __shared__ uint32_t s_thr, s_below, s_spec;
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
    // L2 read: in the fused step the bits were set by other CTAs' atomics
    uint32_t m = a.bitmap_in ? __ldcg(a.bitmap_in + static_cast<size_t>(s) * nw + w) : 0u;
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
  // Every id < T is a candidate (the top-T merge), so positions [0, T) hold
  // 0..T-1 -- written coalesced by all threads -- and an id >= T sits at
  // T + its rank among the set bits >= T: per-thread contiguous word ranges,
  // one block scan, ordered emit of the (few) bits above the prefix.
  pdl_trigger();
  for (uint32_t i = threadIdx.x; i < a.T; i += blockDim.x) ids[i] = i;
  const uint32_t per = (nw + blockDim.x - 1) / blockDim.x;
  const uint32_t w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
  uint32_t cnt = 0;
  for (uint32_t w = w0; w < w1; ++w) cnt += __popc(bm[w] & ~below_mask(w, a.T));
  uint32_t total;
  uint32_t base = a.T + block_scan_excl(cnt, wsum, &total);
  total += a.T;
  for (uint32_t w = w0; w < w1; ++w) {
    uint32_t m = bm[w] & ~below_mask(w, a.T);
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

#ifndef LSB_BODIES_ONLY  // (k_step_fused.cu includes this file for its device functions)
__global__ void __launch_bounds__(1024) k_compact(const __grid_constant__ CompactArgs a) {
  extern __shared__ uint32_t bm_dyn[];  // nwords
  pdl_wait();
  compact_sentence(a, blockIdx.x, bm_dyn);
}
#endif

// =================================================================== K1+K2
constexpr int kWarpBands = 64;  // up to this many bands: a warp per band
#ifndef LSB_FLAT_LOADS
#define LSB_FLAT_LOADS 4
#endif
constexpr int kFlatLoads = LSB_FLAT_LOADS;  // many-band span walk: id loads in flight per lane

// One CTA's K1+K2 for hypothesis row `row` and vocabulary slice `slice`
// (any blockDim <= 1024); returns uniformly per CTA.
static __device__ void probe_row(const ProbeArgs& a, unsigned char* smem, int row, int slice) {
  const IndexView& ix = a.ix;
  const int s = row / a.B, i = row % a.B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const uint32_t lo = static_cast<uint32_t>(slice) * a.slice_len;
  const uint32_t hi = min(ix.V, lo + a.slice_len);
  const bool count = a.t > 0;
  const bool bits = a.levels >= 0;  // bit-sliced counting (t <= 8)
  const size_t cbytes =
      !count ? 0
      : bits ? static_cast<size_t>(a.levels + 1) * (a.slice_len / 8)
             : ((static_cast<size_t>(a.slice_len) * a.counter_bytes + 15) & ~size_t(15));
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
  float* h = reinterpret_cast<float*>(smem + cbytes);
  const int dpad = (ix.d + 3) & ~3;
  uint32_t* codes = reinterpret_cast<uint32_t*>(h + dpad);
  uint32_t* sp_start = codes + ix.W;    // per band: span start (hit) ...
  uint32_t* sp_pre = sp_start + ix.W;   // ... and exclusive prefix of span lengths [W + 1]
  uint16_t* idx = reinterpret_cast<uint16_t*>(sp_pre + ix.W + 1);  // K <= 65536

  __shared__ BandMeta s_bands[kWarpBands];  // few-band path: probe metadata
  if (ix.W <= kWarpBands)
    for (int w = threadIdx.x; w < ix.W; w += blockDim.x) s_bands[w] = ix.bands[w];
  for (size_t k = threadIdx.x; k < cbytes / 16; k += blockDim.x)
    reinterpret_cast<uint4*>(cnt)[k] = make_uint4(0, 0, 0, 0);
  // this thread's permutation row, fetched while the hidden row is in flight
  constexpr int kMaxKReg = 16;
  uint32_t pk[kMaxKReg];
  const int p_own = threadIdx.x;
  if (p_own < ix.P && ix.K <= kMaxKReg) {
    const uint32_t* pr = ix.perms + static_cast<size_t>(p_own) * ix.K;
#pragma unroll
    for (int k = 0; k < kMaxKReg; ++k) pk[k] = k < ix.K ? __ldg(pr + k) : 0u;
  }
  // everything above reads only the index (static); the step inputs below
  // may come from the previous kernel
  pdl_wait();
  const bool dead = (a.n_hyp && i >= a.n_hyp[s]) || (a.finished && a.finished[row]);
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
  if (dead) return;  // uniform per CTA
  if (__syncthreads_or(nan)) {
    if (threadIdx.x == 0) atomicOr(a.err, kErrNaN);
    return;
  }
  // K1: windowed argmax per permutation, ties to the smallest k.
  if (ix.K <= kMaxKReg && ix.P <= static_cast<int>(blockDim.x)) {
    if (p_own < ix.P) {
      uint32_t best = 0;
      float bv = h[pk[0]];
#pragma unroll
      for (int k = 1; k < kMaxKReg; ++k) {
        if (k < ix.K) {
          const float v = h[pk[k]];
          if (v > bv) {
            bv = v;
            best = k;
          }
        }
      }
      idx[p_own] = static_cast<uint16_t>(best);
    }
  } else if (ix.K <= kMaxKReg) {
    // more permutations than threads (large W): each thread's permutation
    // rows are fetched whole (K loads in flight), not one load per step
    for (int p = threadIdx.x; p < ix.P; p += blockDim.x) {
      uint32_t q[kMaxKReg];
      if (ix.perms16) {  // 8 uint16 indices per 16-byte load (2 loads at K = 16, not 16)
        const uint4* pr = reinterpret_cast<const uint4*>(ix.perms16 + static_cast<size_t>(p) * ix.K16);
#pragma unroll
        for (int c = 0; c < kMaxKReg / 8; ++c) {
          const uint4 v = c * 8 < ix.K ? __ldg(pr + c) : make_uint4(0, 0, 0, 0);
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int h2 = 0; h2 < 4; ++h2) {
            q[c * 8 + 2 * h2] = w[h2] & 0xFFFFu;
            q[c * 8 + 2 * h2 + 1] = w[h2] >> 16;
          }
        }
      } else {
        const uint32_t* pr = ix.perms + static_cast<size_t>(p) * ix.K;
#pragma unroll
        for (int k = 0; k < kMaxKReg; ++k) q[k] = k < ix.K ? __ldg(pr + k) : 0u;
      }
      uint32_t best = 0;
      float bv = h[q[0]];
#pragma unroll
      for (int k = 1; k < kMaxKReg; ++k) {
        if (k < ix.K) {
          const float v = h[q[k]];
          if (v > bv) {
            bv = v;
            best = k;
          }
        }
      }
      idx[p] = static_cast<uint16_t>(best);
    }
  } else {
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
      idx[p] = static_cast<uint16_t>(best);
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < ix.W; w += blockDim.x) {
    uint32_t code = 0;
    for (int b = 0; b < ix.u; ++b) code |= static_cast<uint32_t>(idx[w * ix.u + b]) << (b * ix.bits);
    codes[w] = code;
    if (slice == 0) a.qcodes[static_cast<size_t>(row) * ix.W + w] = code;
  }
  __syncthreads();
  if (!count) return;
  uint32_t* bm = a.bitmap + static_cast<size_t>(s) * a.nwords;
  const uint32_t t = static_cast<uint32_t>(a.t);
  auto count_id = [&](uint32_t id) {
    if (id < lo || id >= hi) return;
    const uint32_t local = id - lo;
    if (bits) {
      // level k holds "seen more than k times"; a visit climbs one level,
      // the one after level t-2 marks the word (count == t)
      const uint32_t wd = local >> 5, bit = 1u << (local & 31);
      const uint32_t nw = a.slice_len >> 5;
      int lvl = 0;
      for (; lvl < a.levels; ++lvl)
        if (!(atomicOr(cnt + lvl * nw + wd, bit) & bit)) break;
      if (lvl == a.levels) atomicOr(cnt + a.levels * nw + wd, bit);
      return;
    }
    uint32_t c;
    if (a.counter_bytes == 1) {
      const uint32_t sh = (local & 3) * 8;
      c = (atomicAdd(cnt + (local >> 2), 1u << sh) >> sh) & 0xFFu;
    } else {
      const uint32_t sh = (local & 1) * 16;
      c = (atomicAdd(cnt + (local >> 1), 1u << sh) >> sh) & 0xFFFFu;
    }
    if (c + 1 == t) atomicOr(bm + (id >> 5), 1u << (id & 31));
  };
  constexpr int U = 4;  // id loads in flight per thread
  if (ix.W <= kWarpBands) {
    // K2, few bands (long spans): one warp per band. A warp's bands (at most
    // 16) are probed in one round trip -- lanes 2j / 2j+1 probe tables 0 / 1
    // of band j, metadata from shared memory -- then each span is walked
    // coalesced, U loads in flight per lane.
    const int nb = warp < ix.W ? (ix.W - warp + nwarp - 1) / nwarp : 0;
    const int j = lane >> 1;
    uint4 sl = make_uint4(0, 0, 0, 0);
    bool hit = false;
    if (j < nb) {
      const int w = warp + j * nwarp;
      const BandMeta m = s_bands[w];
      const uint32_t key = codes[w];
      const uint32_t pos = m.slot_off + ((lane & 1) ? (1u << m.lg) + slot_of(m.mul1, m.lg, key)
                                                    : slot_of(m.mul0, m.lg, key));
      sl = __ldg(ix.slots + pos);
      hit = sl.x == key;
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, hit);
    for (int jj = 0; jj < nb; ++jj) {
      const unsigned two = (ballot >> (2 * jj)) & 3u;
      if (!two) continue;
      const int src = 2 * jj + ((two & 1u) ? 0 : 1);  // table 0 wins (probed first)
      const uint32_t start = __shfl_sync(0xffffffffu, sl.y, src);
      const uint32_t len = __shfl_sync(0xffffffffu, sl.z, src);
      const int w = warp + jj * nwarp;
      const uint32_t* ids = ix.word_ids + static_cast<size_t>(w) * ix.V + start;
      for (uint32_t k0 = lane; k0 < len; k0 += 32 * U) {
        uint32_t idu[U];
#pragma unroll
        for (int u = 0; u < U; ++u) idu[u] = k0 + 32 * u < len ? __ldg(ids + k0 + 32 * u) : 0xFFFFFFFFu;
#pragma unroll
        for (int u = 0; u < U; ++u) count_id(idu[u]);
      }
    }
  } else {
    // K2, many bands (short spans) in three block-wide phases, so the
    // dependent global round trips are paid once per row rather than once
    // per band: (A) a thread per band probes both cuckoo tables; (B)
    // exclusive scan of the span lengths; (C) the concatenated spans are
    // walked flat, U id loads in flight per thread.
    for (int w = threadIdx.x; w < ix.W; w += blockDim.x) {
      const BandMeta m = ix.bands[w];
      const uint32_t key = codes[w];
      const uint32_t cap = 1u << m.lg;
      const uint4 s0 = __ldg(ix.slots + m.slot_off + slot_of(m.mul0, m.lg, key));
      const uint4 s1 = __ldg(ix.slots + m.slot_off + cap + slot_of(m.mul1, m.lg, key));
      uint32_t st = 0, ln = 0;
      if (s0.x == key) {  // table 0 wins (the reference probes it first)
        st = s0.y;
        ln = s0.z;
      } else if (s1.x == key) {
        st = s1.y;
        ln = s1.z;
      }
      sp_start[w] = st;
      sp_pre[w] = ln;
    }
    __syncthreads();
    {  // exclusive scan of sp_pre[0..W) in place; sp_pre[W] = total
      const int per = (ix.W + blockDim.x - 1) / blockDim.x;
      const int b0 = min(ix.W, static_cast<int>(threadIdx.x) * per), b1 = min(ix.W, b0 + per);
      uint32_t sum = 0;
      for (int w = b0; w < b1; ++w) sum += sp_pre[w];
      uint32_t x = sum;  // inclusive warp scan of the chunk sums
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      __shared__ uint32_t wsum[32];
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      uint32_t off = 0, tot = 0;
      for (int q = 0; q < nwarp; ++q) {
        off += q < warp ? wsum[q] : 0u;
        tot += wsum[q];
      }
      uint32_t run = off + x - sum;
      for (int w = b0; w < b1; ++w) {
        const uint32_t l = sp_pre[w];
        sp_pre[w] = run;
        run += l;
      }
      if (threadIdx.x == 0) sp_pre[ix.W] = tot;
    }
    __syncthreads();
    const uint32_t total = sp_pre[ix.W];
    // each warp walks one contiguous chunk of the concatenated spans, lanes on
    // consecutive positions (coalesced id loads); a lane finds its band once
    // by binary search and then advances it across span boundaries (~1 smem
    // read per id instead of a log2(W)-step search per id: at W=500 the
    // search was ~90 % of this kernel's instructions)
    const uint32_t chunk = (total + nwarp - 1) / nwarp;
    const uint32_t p0 = min(total, static_cast<uint32_t>(warp) * chunk);
    const uint32_t p1 = min(total, p0 + chunk);
    int band = 0;
    {
      const uint32_t q = min(p0 + lane, total > 0 ? total - 1 : 0u);
      int bl = 0, bh = ix.W - 1;  // last w with sp_pre[w] <= q
      while (bl < bh) {
        const int mid = (bl + bh + 1) >> 1;
        if (sp_pre[mid] <= q) bl = mid;
        else bh = mid - 1;
      }
      band = bl;
    }
    constexpr int UF = kFlatLoads;  // id loads in flight per lane
    for (uint32_t pb = p0; pb < p1; pb += 32 * UF) {
      uint32_t idu[UF];
#pragma unroll
      for (int u = 0; u < UF; ++u) {
        const uint32_t q = pb + 32 * u + lane;
        idu[u] = 0xFFFFFFFFu;
        if (q < p1) {
          while (sp_pre[band + 1] <= q) ++band;
          idu[u] = __ldg(ix.word_ids + static_cast<size_t>(band) * ix.V + sp_start[band] +
                         (q - sp_pre[band]));
        }
      }
#pragma unroll
      for (int u = 0; u < UF; ++u) count_id(idu[u]);
    }
  }
  pdl_trigger();
  if (bits) {  // OR this slice's marked words into the sentence bitmap
    __syncthreads();
    const uint32_t nw = a.slice_len >> 5;
    const uint32_t* fin = cnt + a.levels * nw;
    const uint32_t w0 = lo >> 5, wend = min(nw, a.nwords - w0);
    for (uint32_t w = threadIdx.x; w < wend; w += blockDim.x)
      if (fin[w]) atomicOr(bm + w0 + w, fin[w]);
  }
}

#ifndef LSB_BODIES_ONLY
template <int NT>
__global__ void __launch_bounds__(NT, NT == 1024 ? 1 : 1536 / NT) k_probe_count(const __grid_constant__ ProbeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  probe_row(a, smem, blockIdx.x, blockIdx.y);
}

size_t probe_smem_bytes(const ProbeArgs& a) {
  const IndexView& ix = a.ix;
  const size_t cbytes =
      a.t <= 0 ? 0
      : a.levels >= 0 ? static_cast<size_t>(a.levels + 1) * (a.slice_len / 8)
                      : ((static_cast<size_t>(a.slice_len) * a.counter_bytes + 15) & ~size_t(15));
  return cbytes + ((ix.d + 3) & ~3) * 4 + (3 * ix.W + 1) * 4 + 2 * ix.P + 16;
}

lsb_status launch_probe(lsb_ctx* ctx, const ProbeArgs& a) {
  const IndexView& ix = a.ix;
  const uint32_t nslices = a.t > 0 ? (ix.V + a.slice_len - 1) / a.slice_len : 1;
  const size_t cbytes =
      a.t <= 0 ? 0
      : a.levels >= 0 ? static_cast<size_t>(a.levels + 1) * (a.slice_len / 8)
                      : ((static_cast<size_t>(a.slice_len) * a.counter_bytes + 15) & ~size_t(15));
  const size_t smem = cbytes + ((ix.d + 3) & ~3) * 4 + (3 * ix.W + 1) * 4 + 2 * ix.P + 16;
  if (smem > ctx->smem_optin) {
    set_error("probe: shared memory budget exceeded");
    return LSB_EINVAL;
  }
  dim3 grid0(a.S * a.B, std::max(1u, nslices));
  const int threads = static_cast<int>(grid0.x * grid0.y) < ctx->sm_count ? 1024
                      : a.levels >= 0                                       ? 256
                                                                            : 512;
  auto* kern = threads == 1024 ? k_probe_count<1024>
               : threads == 512 ? k_probe_count<512>
                                : k_probe_count<256>;
  if (lsb_status rc = ensure_smem(ctx, kern, smem)) return rc;
  // bit-sliced counters need little shared memory: 256-thread CTAs, 6 per SM,
  // so a 768-row step runs in one wave; a grid smaller than the GPU gets
  // 1024-thread CTAs (more loads in flight per row)
  LSB_CUDA(launch_pdl(ctx, kern, grid0, dim3(threads), smem, a));
  LSB_LAUNCHED(ctx, "k_probe_count");
  return LSB_OK;
}

// ================================================= K1+K2, band-split variant
// For steps with few hypothesis rows (a one-sentence decode: 12 rows, so
// k_probe_count would run 12 CTAs on 148 SMs) the row's bands are split
// over G CTAs: CTA (row, g) hashes and probes bands [W g / G, W (g+1) / G)
// and walks their spans one warp per band, coalesced, U id loads in flight.
// Hit counts per (row, word) are 16-bit counters in global memory (L2); the
// visit that lifts a count to t sets the word's bit in the sentence bitmap
// (atomicAdd returns the old count, so exactly once). The row's last CTA to
// finish (arrival counter) zeroes its counters and the counter for the next
// step -- self-cleaning, so the kernel also replays inside a CUDA graph.
template <int NT>
__global__ void __launch_bounds__(NT) k_probe_split(ProbeArgs a, int G, uint32_t* cnt,
                                                    uint32_t cnt_words, uint32_t* arrive) {
  extern __shared__ __align__(16) unsigned char smem[];
  const IndexView& ix = a.ix;
  const int row = blockIdx.x, g = blockIdx.y;
  const int s = row / a.B, i = row % a.B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nwarp = NT / 32;
  const int w0 = static_cast<int>((static_cast<long long>(ix.W) * g) / G);
  const int w1 = static_cast<int>((static_cast<long long>(ix.W) * (g + 1)) / G);
  const int nb = w1 - w0;
  const int np = nb * ix.u;  // permutations of these bands
  float* h = reinterpret_cast<float*>(smem);
  const int dpad = (ix.d + 3) & ~3;
  uint32_t* sp_start = reinterpret_cast<uint32_t*>(h + dpad);
  uint32_t* sp_len = sp_start + nb;
  uint16_t* idx = reinterpret_cast<uint16_t*>(sp_len + nb);
  constexpr int kMaxKReg = 16;
  uint32_t pk[kMaxKReg];
  const int p_own = threadIdx.x;
  const bool kreg = ix.K <= kMaxKReg;
  if (p_own < np && kreg) {
    const uint32_t* pr = ix.perms + static_cast<size_t>(w0 * ix.u + p_own) * ix.K;
#pragma unroll
    for (int k = 0; k < kMaxKReg; ++k) pk[k] = k < ix.K ? __ldg(pr + k) : 0u;
  }
  pdl_wait();
  const bool dead = (a.n_hyp && i >= a.n_hyp[s]) || (a.finished && a.finished[row]);
  if (dead) return;  // uniform over the row's CTAs: no counting, nothing to clear
  const float* src = a.hidden + static_cast<size_t>(row) * ix.d;
  int nan = 0;
  if ((ix.d & 3) == 0) {
    for (int c = threadIdx.x; c < (ix.d >> 2); c += NT) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(src) + c);
      nan |= isnan(v.x) | isnan(v.y) | isnan(v.z) | isnan(v.w);
      reinterpret_cast<float4*>(h)[c] = v;
    }
  } else {
    for (int c = threadIdx.x; c < ix.d; c += NT) {
      const float v = __ldg(src + c);
      nan |= isnan(v);
      h[c] = v;
    }
  }
  if (__syncthreads_or(nan)) {
    if (threadIdx.x == 0 && g == 0) atomicOr(a.err, kErrNaN);
    return;  // uniform over the row's CTAs (same row)
  }
  // K1 for this CTA's permutations (ties to the smallest k)
  for (int p = threadIdx.x; p < np; p += NT) {
    const uint32_t* pr = ix.perms + static_cast<size_t>(w0 * ix.u + p) * ix.K;
    uint32_t best = 0;
    if (kreg && p == p_own) {
      float bv = h[pk[0]];
#pragma unroll
      for (int k = 1; k < kMaxKReg; ++k)
        if (k < ix.K) {
          const float v = h[pk[k]];
          if (v > bv) {
            bv = v;
            best = k;
          }
        }
    } else {
      float bv = h[__ldg(pr)];
      for (int k = 1; k < ix.K; ++k) {
        const float v = h[__ldg(pr + k)];
        if (v > bv) {
          bv = v;
          best = k;
        }
      }
    }
    idx[p] = static_cast<uint16_t>(best);
  }
  __syncthreads();
  // codes + cuckoo probe, a thread per band
  for (int j = threadIdx.x; j < nb; j += NT) {
    const int w = w0 + j;
    uint32_t code = 0;
    for (int b = 0; b < ix.u; ++b) code |= static_cast<uint32_t>(idx[j * ix.u + b]) << (b * ix.bits);
    a.qcodes[static_cast<size_t>(row) * ix.W + w] = code;
    const BandMeta m = ix.bands[w];
    const uint32_t cap = 1u << m.lg;
    const uint4 s0 = __ldg(ix.slots + m.slot_off + slot_of(m.mul0, m.lg, code));
    const uint4 s1 = __ldg(ix.slots + m.slot_off + cap + slot_of(m.mul1, m.lg, code));
    uint32_t st = 0, ln = 0;
    if (s0.x == code) {  // table 0 wins (the reference probes it first)
      st = s0.y;
      ln = s0.z;
    } else if (s1.x == code) {
      st = s1.y;
      ln = s1.z;
    }
    sp_start[j] = st;
    sp_len[j] = ln;
  }
  __syncthreads();
  if (a.t > 0) {
    uint32_t* bm = a.bitmap + static_cast<size_t>(s) * a.nwords;
    uint32_t* rc = cnt + static_cast<size_t>(row) * cnt_words;
    const uint32_t t = static_cast<uint32_t>(a.t);
    constexpr int U = 4;
    for (int j = warp; j < nb; j += nwarp) {
      const uint32_t st = sp_start[j], ln = sp_len[j];
      const uint32_t* ids = ix.word_ids + static_cast<size_t>(w0 + j) * ix.V + st;
      for (uint32_t k0 = lane; k0 < ln; k0 += 32 * U) {
        uint32_t idu[U];
#pragma unroll
        for (int u = 0; u < U; ++u) idu[u] = k0 + 32 * u < ln ? __ldg(ids + k0 + 32 * u) : 0xFFFFFFFFu;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t id = idu[u];
          if (id == 0xFFFFFFFFu) continue;
          const uint32_t sh = (id & 1) * 16;
          const uint32_t c = (atomicAdd(rc + (id >> 1), 1u << sh) >> sh) & 0xFFFFu;
          if (c + 1 == t) atomicOr(bm + (id >> 5), 1u << (id & 31));
        }
      }
    }
  }
  pdl_trigger();
  if (a.t <= 0) return;
  // the row's last CTA clears its counters for the next step
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(arrive + row, 1u) == static_cast<uint32_t>(G - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  uint4* rc4 = reinterpret_cast<uint4*>(cnt + static_cast<size_t>(row) * cnt_words);
  for (uint32_t k = threadIdx.x; k < cnt_words / 4; k += NT) rc4[k] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) arrive[row] = 0;
}

lsb_status launch_probe_split(lsb_ctx* ctx, const ProbeArgs& a, int G, uint32_t* cnt,
                              uint32_t cnt_words, uint32_t* arrive) {
  const IndexView& ix = a.ix;
  const int nbmax = (ix.W + G - 1) / G;
  constexpr int NT = 256;
  if (nbmax * ix.u > NT * 8) return set_error("probe_split: too many bands per CTA"), LSB_EINVAL;
  const size_t smem = ((ix.d + 3) & ~3) * 4 + 2 * nbmax * 4 + 2 * nbmax * ix.u + 16;
  if (smem > ctx->smem_optin) return set_error("probe_split: shared memory budget"), LSB_EINVAL;
  auto* kern = k_probe_split<NT>;
  if (lsb_status rc = ensure_smem(ctx, kern, smem)) return rc;
  LSB_CUDA(launch_pdl(ctx, kern, dim3(a.S * a.B, G), dim3(NT), smem, a, G, cnt, cnt_words, arrive));
  LSB_LAUNCHED(ctx, "k_probe_split");
  return LSB_OK;
}

lsb_status launch_compact(lsb_ctx* ctx, const CompactArgs& a, int S) {
  const size_t smem = static_cast<size_t>(a.nwords) * 4;
  if (smem > ctx->smem_optin) return set_error("compact: vocabulary too large"), LSB_EINVAL;
  if (lsb_status rc = ensure_smem(ctx, k_compact, smem)) return rc;
  LSB_CUDA(launch_pdl(ctx, k_compact, dim3(S), dim3(1024), smem, a));
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

#endif  // LSB_BODIES_ONLY

}  // namespace lsb
