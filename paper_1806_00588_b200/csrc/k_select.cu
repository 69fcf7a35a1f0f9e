// k_select.cu -- K5: reduced softmax normalisation, per-row top-B and the
// per-sentence beam expansion with the hidden-state reorder.
//
//  K5a k_softmax_topb : one 128-thread CTA per hypothesis row. softmax_rows
//      (src/beam_decoder.cpp:46-74): float max; e = exp((double)l - mx) kept
//      as float(e); double denominator (a fixed-shape tree, so deterministic);
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

#include "k_step.cuh"

namespace lsb {

constexpr int kSelT = 128;  // threads per row CTA

__device__ __forceinline__ bool top_better(float pa, uint32_t ra, float pb, uint32_t rb) {
  return pa > pb || (pa == pb && ra < rb);
}

template <class T, class Op>
__device__ __forceinline__ T block_reduce(T v, T* red, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();  // red[] may still be read from a previous reduction
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = red[0];
#pragma unroll
  for (int w = 1; w < kSelT / 32; ++w) v = op(v, red[w]);
  return v;
}

// ===================================================================== K5a
__global__ void __launch_bounds__(kSelT) k_softmax_topb(SoftmaxArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ float red_f[kSelT / 32];
  __shared__ double red_d[kSelT / 32];
  __shared__ float win_p[kSelT / 32];
  __shared__ uint32_t win_r[kSelT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = blockIdx.x;
  const int s = row / a.Bsent, i = row % a.Bsent;
  const bool live = !(a.n_hyp && i >= a.n_hyp[s]) && !(a.finished && a.finished[row]);
  if (!live) {
    if (tid == 0) a.top_n[row] = 0;
    return;
  }
  const int B = a.topB;
  const uint32_t n = a.n_cand ? a.n_cand[s] : a.n_const;
  float* L = a.logits + static_cast<size_t>(row) * a.ldl;
  float inv = 1.0f;
  if (!a.probs_in) {
    // float max, as std::max over the row (src/beam_decoder.cpp:55)
    float mx = -INFINITY;
    for (uint32_t r = tid; r < n; r += kSelT) {
      const float v = L[r];
      mx = (mx < v) ? v : mx;
    }
    mx = block_reduce(mx, red_f, [](float x, float y) { return (x < y) ? y : x; });
    if (n == 0 || (isinf(mx) && mx < 0)) {
      if (tid == 0) {
        atomicOr(a.err, kErrEmptyRow);
        a.top_n[row] = 0;
      }
      return;
    }
    const double dmx = static_cast<double>(mx);
    double sum = 0.0;
    for (uint32_t r = tid; r < n; r += kSelT) {
      const double e = exp(static_cast<double>(L[r]) - dmx);
      L[r] = static_cast<float>(e);
      sum += e;
    }
    sum = block_reduce(sum, red_d, [](double x, double y) { return x + y; });
    inv = static_cast<float>(1.0 / sum);
  }
  if (B <= 0) {
    if (tid == 0) a.top_n[row] = 0;
    return;
  }
  // per-thread sorted lists, entry j of thread t at [j * kSelT + t]
  float* lp = reinterpret_cast<float*>(smem);
  uint32_t* lr = reinterpret_cast<uint32_t*>(lp + B * kSelT);
  int cnt = 0;
  for (uint32_t r = tid; r < n; r += kSelT) {
    const float p = a.probs_in ? L[r] : __fmul_rn(L[r], inv);
    if (a.keep_probs && !a.probs_in) L[r] = p;
    if (cnt == B && !(p > lp[(B - 1) * kSelT + tid])) continue;
    int j = cnt < B ? cnt++ : B - 1;
    while (j > 0 && lp[(j - 1) * kSelT + tid] < p) {
      lp[j * kSelT + tid] = lp[(j - 1) * kSelT + tid];
      lr[j * kSelT + tid] = lr[(j - 1) * kSelT + tid];
      --j;
    }
    lp[j * kSelT + tid] = p;
    lr[j * kSelT + tid] = r;
  }
  const int keep = static_cast<int>(min(static_cast<uint32_t>(B), n));
  TopEntry* out = a.top + static_cast<size_t>(row) * B;
  int head = 0;
  for (int k = 0; k < keep; ++k) {
    float bp = head < cnt ? lp[head * kSelT + tid] : -INFINITY;
    uint32_t br = head < cnt ? lr[head * kSelT + tid] : 0xFFFFFFFFu;
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
    if ((br % kSelT) == static_cast<uint32_t>(tid)) ++head;
    if (tid == 0) out[k] = TopEntry{bp, br};
    __syncthreads();
  }
  if (tid == 0) a.top_n[row] = keep;
}

lsb_status launch_softmax(lsb_ctx* ctx, const SoftmaxArgs& a) {
  if (a.R_total == 0) return LSB_OK;
  const size_t smem = static_cast<size_t>(std::max(a.topB, 1)) * kSelT * 8;
  if (smem > ctx->smem_optin) return set_error("softmax: beam too large"), LSB_EINVAL;
  static size_t configured = 0;
  if (smem > configured) {
    LSB_CUDA(cudaFuncSetAttribute(k_softmax_topb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  k_softmax_topb<<<a.R_total, kSelT, smem, ctx->stream>>>(a);
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

// Word id of candidate column r of sentence s.
__device__ __forceinline__ long long word_of(const ExpandArgs& a, const uint32_t* ids,
                                             uint32_t r) {
  if (a.id_map) return a.id_map[r];
  return (r < a.n_shared || !ids) ? static_cast<long long>(r) : static_cast<long long>(ids[r]);
}

// Hidden-state reorder: child k of sentence s starts from its parent's vector.
__device__ void reorder_hidden(const ExpandArgs& a, int s, int count, const uint32_t* beams) {
  // one flat index space over (child, column) so every load is independent
  const int d = a.d;
  const size_t rbase = static_cast<size_t>(s) * a.Bsent;
  const size_t obase = static_cast<size_t>(s) * a.topB;
  if ((d & 3) == 0) {
    const int d4 = d >> 2;
    for (int q = threadIdx.x; q < count * d4; q += blockDim.x) {
      const int k = q / d4, c = q - k * d4;
      reinterpret_cast<float4*>(a.hidden_out + (obase + k) * d)[c] =
          __ldg(reinterpret_cast<const float4*>(a.hidden + (rbase + beams[k]) * d) + c);
    }
  } else {
    for (int q = threadIdx.x; q < count * d; q += blockDim.x) {
      const int k = q / d, c = q - k * d;
      a.hidden_out[(obase + k) * d + c] = __ldg(a.hidden + (rbase + beams[k]) * d + c);
    }
  }
}

// Rank selection. Lists: [0, nfz) explicit frozen singletons, then one list
// per hypothesis row (a finished row is a singleton carrying its score).
// Shared memory: per list off/len (ints), then per candidate score, beam, word.
constexpr int kExpT = 256;
constexpr int kRankMaxLists = 128;

__global__ void __launch_bounds__(kExpT) k_expand(ExpandArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_off[kRankMaxLists + 1];
  __shared__ uint32_t s_beams[64];
  __shared__ int s_count;
  const int s = blockIdx.x;
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
        sc = a.scores[rbase + row] + log(static_cast<double>(t.p));
        wd = word_of(a, ids, t.r);
      }
    }
    cs[e] = sc;
    cb[e] = beam;
    cw[e] = wd;
  }
  __syncthreads();
  // rank = own position + per other list the count of better entries
  const int B = a.topB;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int lo = 0, hi = nl - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    const int own = lo;
    const Cand me{cs[e], cb[e], cw[e]};
    int rank = e - s_off[own];
    for (int l = 0; l < nl && rank < B; ++l) {
      if (l == own) continue;
      int b0 = s_off[l], b1 = s_off[l + 1];  // first entry of l not better than me
      while (b0 < b1) {
        const int mid = (b0 + b1) >> 1;
        if (cand_better(Cand{cs[mid], cb[mid], cw[mid]}, me)) b0 = mid + 1;
        else b1 = mid;
      }
      rank += b0 - s_off[l];
    }
    if (rank < B) {
      a.choices[static_cast<size_t>(s) * B + rank] =
          lsb_choice{me.score, me.beam, 0u, static_cast<int64_t>(me.word)};
      if (rank < 64) s_beams[rank] = me.beam;
    }
  }
  const int count = min(B, total);
  if (threadIdx.x == 0) {
    a.n_choices[s] = count;
    s_count = count;
  }
  __syncthreads();
  if (a.hidden_out && a.hidden) reorder_hidden(a, s, min(s_count, 64), s_beams);
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
    sc = a.scores[rbase + row] + log(static_cast<double>(e.p));
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

lsb_status launch_expand(lsb_ctx* ctx, const ExpandArgs& a) {
  if (a.S == 0) return LSB_OK;
  const int nl = (a.frozen_mode ? a.nfrozen : 0) + a.Bsent;
  const size_t rank_smem = static_cast<size_t>(nl) * std::max(a.topB, 1) * (8 + 8 + 4);
  if (nl <= kRankMaxLists && rank_smem <= ctx->smem_optin) {
    static size_t configured = 0;
    if (rank_smem > configured) {
      LSB_CUDA(cudaFuncSetAttribute(k_expand, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(rank_smem)));
      configured = rank_smem;
    }
    k_expand<<<a.S, kExpT, rank_smem, ctx->stream>>>(a);
    LSB_LAUNCHED(ctx, "k_expand");
    return LSB_OK;
  }
  const size_t smem = static_cast<size_t>(nl) * (8 + 8 + 4 + 4 + 4) + 16;
  if (smem > ctx->smem_optin) return set_error("expand: too many rows"), LSB_EINVAL;
  static size_t configured = 0;
  if (smem > configured) {
    LSB_CUDA(cudaFuncSetAttribute(k_expand_tournament,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  k_expand_tournament<<<a.S, 256, smem, ctx->stream>>>(a);
  LSB_LAUNCHED(ctx, "k_expand_tournament");
  return LSB_OK;
}

}  // namespace lsb
