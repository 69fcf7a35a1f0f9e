// capi_dropin.cu -- C-ABI entry points that the C++ drop-in layer
// (include/lshbeam/*.hpp) needs beyond the per-step path:
//  * standalone cuckoo tables (CuckooTable::build, src/band_index.cpp:32-71),
//  * importing a host-described index (raw-state constructors and the WTAIDX1
//    loader, src/band_index.cpp:245-289),
//  * the recurrence h' = tanh(W_h h + W_e emb(token)) on the device
//    (src/model_provider.cpp:83-102),
//  * the exact full-vocabulary top-b used for recall@B
//    (src/eval_oracle.cpp:11-40, decode's oracle branch
//    src/beam_decoder.cpp:255-272).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "glibc_tanhf.cuh"
#include "k_step.cuh"

namespace lsb {

lsb_status launch_wta_hash(lsb_ctx* ctx, const float* M, long long n, int d,
                           const uint32_t* perms, int K, int u, int W, uint32_t* out);
lsb_status build_cuckoo_band(lsb_ctx* ctx, const uint32_t* keys, const uint32_t* starts,
                             const uint32_t* lens, uint32_t n, uint64_t seed, uint32_t lg,
                             uint4* slots_dev, BandMeta* meta_dev, uint32_t* attempts_dev);

// ------------------------------------------------------------ recurrence
// out[k] = tanh(W_h h_k + W_e E[tok_k]) for tok_k >= 0, else a copy of h_k
// (a finished hypothesis is carried unchanged, src/beam_decoder.cpp:303-305).
// One warp per output element r of one hypothesis; the reference's 4-lane
// SSE order without FMA: lane j accumulates fl(fl(wh*h) + fl(we*emb)) for
// c = j mod 4 ascending, the d mod 4 tail into lane 0, final ((l0+l1)+l2)+l3.
// Each lane owns columns 4*lane.. (a 128-column stripe per warp pass), so the
// 4 partial sums of one stripe are reduced in stripe order by lane 0.
__global__ void k_recurrence(const float* __restrict__ wh, const float* __restrict__ we,
                             const float* __restrict__ E, uint32_t V, int d,
                             const float* __restrict__ hin, const int64_t* __restrict__ tok,
                             int n, float* __restrict__ hout, uint32_t* err) {
  extern __shared__ __align__(16) float sh[];  // h then emb of this hypothesis
  const int k = blockIdx.y;
  const int64_t t = tok[k];
  const float* h = hin + static_cast<size_t>(k) * d;
  float* o = hout + static_cast<size_t>(k) * d;
  if (t < 0) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d; c += gridDim.x * blockDim.x)
      o[c] = h[c];
    return;
  }
  if (t >= static_cast<int64_t>(V)) {
    if (threadIdx.x == 0) atomicOr(err, kErrNaN);
    return;
  }
  float* hs = sh;
  float* es = sh + d;
  const float* emb = E + static_cast<size_t>(t) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    hs[c] = h[c];
    es[c] = emb[c];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int d4 = d >= 4 ? (d & ~3) : 0;
  for (int r = blockIdx.x * nwarp + warp; r < d; r += gridDim.x * nwarp) {
    const float* a = wh + static_cast<size_t>(r) * d;
    const float* b = we + static_cast<size_t>(r) * d;
    // per lane: partial lane sums over its groups, kept per group for the
    // ordered combine (each group of 4 columns belongs to one lane)
    float l0 = 0.f, l1 = 0.f, l2 = 0.f, l3 = 0.f;
    for (int g0 = 0; g0 < d4; g0 += 128) {
      float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
      const int c = g0 + 4 * lane;
      const bool ok = c < d4;
      if (ok) {
        t0 = __fadd_rn(__fmul_rn(a[c], hs[c]), __fmul_rn(b[c], es[c]));
        t1 = __fadd_rn(__fmul_rn(a[c + 1], hs[c + 1]), __fmul_rn(b[c + 1], es[c + 1]));
        t2 = __fadd_rn(__fmul_rn(a[c + 2], hs[c + 2]), __fmul_rn(b[c + 2], es[c + 2]));
        t3 = __fadd_rn(__fmul_rn(a[c + 3], hs[c + 3]), __fmul_rn(b[c + 3], es[c + 3]));
      }
      // sequential accumulation in column order: lane 0's group first
      for (int src = 0; src < 32; ++src) {
        const float u0 = __shfl_sync(0xffffffffu, t0, src);
        const float u1 = __shfl_sync(0xffffffffu, t1, src);
        const float u2 = __shfl_sync(0xffffffffu, t2, src);
        const float u3 = __shfl_sync(0xffffffffu, t3, src);
        if (g0 + 4 * src < d4) {
          l0 = __fadd_rn(l0, u0);
          l1 = __fadd_rn(l1, u1);
          l2 = __fadd_rn(l2, u2);
          l3 = __fadd_rn(l3, u3);
        }
      }
    }
    if (lane == 0) {
      for (int c = d4; c < d; ++c)
        l0 = __fadd_rn(__fadd_rn(__fmul_rn(a[c], hs[c]), __fmul_rn(b[c], es[c])), l0);
      float acc = __fadd_rn(0.0f, l0);
      acc = __fadd_rn(acc, l1);
      acc = __fadd_rn(acc, l2);
      acc = __fadd_rn(acc, l3);
      o[r] = lsb_tanhf::tanhf(acc);  // glibc tanhf, bit for bit (glibc_tanhf.cuh)
    }
  }
}


// ------------------------------------------------------- exact top-b
// Order-preserving unsigned key of a float: larger float -> larger key; -0 and
// +0 share a key (the reference compares with !=, so they tie and the smaller
// id wins, src/eval_oracle.cpp:29-32).
__device__ __forceinline__ uint32_t ordered_key(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7fffffffu) == 0) u = 0;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// One CTA per row: radix select of the b-th largest key (4 passes of 8-bit
// digits over the row, which stays in L2), then the entries above it plus the
// smallest-index entries equal to it, ranked by (value desc, index asc).
// Works for any sign (exact_topb runs on raw logits).
constexpr int kTopbThreads = 512;
__global__ void __launch_bounds__(kTopbThreads) k_exact_topb(const float* __restrict__ L,
                                                             size_t ld, uint32_t n, int b,
                                                             uint32_t* __restrict__ ids,
                                                             float* __restrict__ vals) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_prefix, s_mask, s_above, s_need;
  __shared__ uint32_t wsum[33];
  __shared__ uint32_t sel_key[64], sel_col[64];
  __shared__ uint32_t s_nsel;
  const float* row = L + static_cast<size_t>(blockIdx.x) * ld;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_prefix = 0;
    s_mask = 0;
    s_above = 0;  // entries known to be above the selected prefix
    s_need = b;   // rank (1-based) still to locate inside the prefix bucket
    s_nsel = 0;
  }
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int k = tid; k < 256; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix, mask = s_mask;
    for (uint32_t c = tid; c < n; c += blockDim.x) {
      const uint32_t key = ordered_key(__ldg(row + c));
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      // walk digits from the top until the need-th largest is inside
      uint32_t need = s_need, acc = 0;
      int dg = 255;
      for (; dg > 0; --dg) {
        if (acc + hist[dg] >= need) break;
        acc += hist[dg];
      }
      s_need = need - acc;
      s_above += acc;
      s_prefix = prefix | (static_cast<uint32_t>(dg) << shift);
      s_mask = mask | (255u << shift);
    }
    __syncthreads();
  }
  const uint32_t tau = s_prefix;     // the b-th largest key
  const uint32_t take_eq = s_need;   // how many entries equal to tau are kept
  // entries above tau (fewer than b of them, any order)
  for (uint32_t c = tid; c < n; c += blockDim.x) {
    const uint32_t key = ordered_key(__ldg(row + c));
    if (key > tau) {
      const uint32_t at = atomicAdd(&s_nsel, 1u);
      sel_key[at] = key;
      sel_col[at] = c;
    }
  }
  // entries equal to tau: the take_eq smallest columns, by a block scan over
  // contiguous per-thread column ranges
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t c0 = min(n, tid * per), c1 = min(n, c0 + per);
  uint32_t eq = 0;
  for (uint32_t c = c0; c < c1; ++c) eq += ordered_key(__ldg(row + c)) == tau;
  __syncthreads();
  const uint32_t base_sel = s_nsel;
  // block exclusive scan of eq (per-thread column ranges are in thread order)
  const int lane = tid & 31, warp = tid >> 5;
  uint32_t incl = eq;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t w = lane < nw ? wsum[lane] : 0u, wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    if (lane < nw) wsum[lane] = wi - w;
  }
  __syncthreads();
  uint32_t ex = wsum[warp] + incl - eq;
  for (uint32_t c = c0; c < c1 && ex < take_eq; ++c) {
    if (ordered_key(__ldg(row + c)) == tau) {
      sel_key[base_sel + ex] = tau;
      sel_col[base_sel + ex] = c;
      ++ex;
    }
  }
  __syncthreads();
  // rank the b selected entries: key desc, column asc
  if (tid < b) {
    const uint32_t k = sel_key[tid], c = sel_col[tid];
    int rank = 0;
    for (int j = 0; j < b; ++j) {
      const uint32_t kj = sel_key[j], cj = sel_col[j];
      rank += (kj > k) || (kj == k && cj < c);
    }
    ids[static_cast<size_t>(blockIdx.x) * b + rank] = c;
    vals[static_cast<size_t>(blockIdx.x) * b + rank] = __ldg(row + c);
  }
}

}  // namespace lsb

using namespace lsb;

struct lsb_recurrent {
  float* wh = nullptr;
  float* we = nullptr;
};

namespace {

template <class T>
struct Dev {
  T* p = nullptr;
  ~Dev() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)); }
};

uint32_t table_lg(size_t n) {
  uint32_t lg = 0;
  while ((size_t{1} << lg) < n) ++lg;
  return std::max(1u, lg);  // src/band_index.cpp:39
}

}  // namespace

extern "C" {

lsb_status lsb_device_alloc(lsb_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || !out) return set_error("lsb_device_alloc: null"), LSB_EINVAL;
  LSB_CUDA(cudaSetDevice(ctx->device));
  const cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
  if (e != cudaSuccess) return set_error("device allocation failed"), LSB_ENOMEM;
  return LSB_OK;
}

lsb_status lsb_device_free(lsb_ctx* ctx, void* p) {
  if (!ctx) return set_error("lsb_device_free: null"), LSB_EINVAL;
  if (p) LSB_CUDA(cudaFree(p));
  return LSB_OK;
}

lsb_status lsb_copy_to_device(lsb_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx || (bytes && (!dst || !src))) return set_error("lsb_copy_to_device: null"), LSB_EINVAL;
  if (bytes) LSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return LSB_OK;
}

lsb_status lsb_copy_to_host(lsb_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx || (bytes && (!dst || !src))) return set_error("lsb_copy_to_host: null"), LSB_EINVAL;
  if (bytes) LSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_ctx_set_parallel_cuckoo(lsb_ctx* ctx, int on) {
  if (!ctx) return set_error("lsb_ctx_set_parallel_cuckoo: null"), LSB_EINVAL;
  ctx->cuckoo_parallel = on ? 1 : 0;
  return LSB_OK;
}

uint32_t lsb_cuckoo_log2_capacity(size_t n_entries) { return table_lg(n_entries); }

lsb_status lsb_cuckoo_build(lsb_ctx* ctx, const uint32_t* keys, const uint32_t* starts,
                            const uint32_t* lens, uint32_t n, uint64_t seed, uint32_t* lg_out,
                            uint64_t* mul2_out, uint32_t* slots_out, uint32_t* attempts_out) {
  if (!ctx || !lg_out || (n && (!keys || !starts || !lens)))
    return set_error("lsb_cuckoo_build: bad arguments"), LSB_EINVAL;
  for (uint32_t i = 0; i < n; ++i)
    if (keys[i] >= kEmptyCode)  // src/band_index.cpp:35-36
      return set_error("CuckooTable: key collides with sentinel"), LSB_EINVAL;
  const uint32_t lg = table_lg(n);
  *lg_out = lg;
  const uint32_t nslots = 2u << lg;
  Dev<uint32_t> k, s, l, att;
  Dev<uint4> slots;
  Dev<BandMeta> meta;
  LSB_CUDA(k.alloc(n));
  LSB_CUDA(s.alloc(n));
  LSB_CUDA(l.alloc(n));
  LSB_CUDA(att.alloc(1));
  LSB_CUDA(slots.alloc(nslots));
  LSB_CUDA(meta.alloc(1));
  cudaStream_t st = ctx->stream;
  if (n) {
    LSB_CUDA(cudaMemcpyAsync(k.p, keys, n * 4ull, cudaMemcpyHostToDevice, st));
    LSB_CUDA(cudaMemcpyAsync(s.p, starts, n * 4ull, cudaMemcpyHostToDevice, st));
    LSB_CUDA(cudaMemcpyAsync(l.p, lens, n * 4ull, cudaMemcpyHostToDevice, st));
  }
  lsb_status rc = build_cuckoo_band(ctx, k.p, s.p, l.p, n, seed, lg, slots.p, meta.p, att.p);
  if (rc) return rc;
  BandMeta m{};
  std::vector<uint4> tmp(nslots);
  uint32_t attempts = 0;
  LSB_CUDA(cudaMemcpyAsync(&m, meta.p, sizeof(m), cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaMemcpyAsync(tmp.data(), slots.p, nslots * sizeof(uint4), cudaMemcpyDeviceToHost, st));
  LSB_CUDA(cudaMemcpyAsync(&attempts, att.p, 4, cudaMemcpyDeviceToHost, st));
  rc = lsb_ctx_sync(ctx);
  if (rc) return rc;
  if (mul2_out) {
    mul2_out[0] = m.mul0;
    mul2_out[1] = m.mul1;
  }
  if (slots_out)
    for (uint32_t i = 0; i < nslots; ++i) {
      slots_out[3 * i] = tmp[i].x;
      slots_out[3 * i + 1] = tmp[i].y;
      slots_out[3 * i + 2] = tmp[i].z;
    }
  if (attempts_out) *attempts_out = attempts;
  return LSB_OK;
}

lsb_status lsb_wta_indices(lsb_ctx* ctx, const float* M_host, int64_t n, int d,
                           const uint32_t* perms_host, int P, int K, uint32_t* idx_host) {
  if (!ctx || n < 0 || d < 1 || P < 1 || K < 1 || K > 65536)
    return set_error("wta_hash_vector: bad arguments"), LSB_EINVAL;
  if (d < K) return set_error("PermutationSet: dimension smaller than window"), LSB_EINVAL;
  for (size_t i = 0; i < static_cast<size_t>(P) * K; ++i)
    if (perms_host[i] >= static_cast<uint32_t>(d))
      return set_error("PermutationSet: index out of range"), LSB_EINVAL;
  if (n == 0) return LSB_OK;
  Dev<float> M;
  Dev<uint32_t> p, out;
  LSB_CUDA(M.alloc(static_cast<size_t>(n) * d));
  LSB_CUDA(p.alloc(static_cast<size_t>(P) * K));
  LSB_CUDA(out.alloc(static_cast<size_t>(n) * P));
  cudaStream_t st = ctx->stream;
  LSB_CUDA(cudaMemcpyAsync(M.p, M_host, static_cast<size_t>(n) * d * 4, cudaMemcpyHostToDevice, st));
  LSB_CUDA(cudaMemcpyAsync(p.p, perms_host, static_cast<size_t>(P) * K * 4, cudaMemcpyHostToDevice, st));
  // u = 1, W = P: every "band" is one raw index (no packing shift)
  lsb_status rc = launch_wta_hash(ctx, M.p, n, d, p.p, K, 1, P, out.p);
  if (rc) return rc;
  LSB_CUDA(cudaMemcpyAsync(idx_host, out.p, static_cast<size_t>(n) * P * 4, cudaMemcpyDeviceToHost, st));
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_index_import(lsb_ctx* ctx, uint32_t vocab, int W, const uint32_t* word_ids_host,
                            const uint32_t* lg_host, const uint64_t* mul_host,
                            const uint32_t* slots_host, const uint32_t* perms_host, int K, int u,
                            int dim, uint64_t perm_seed, lsb_index** out) {
  if (!ctx || !out || W < 1 || !lg_host || !mul_host || !slots_host)
    return set_error("lsb_index_import: bad arguments"), LSB_EINVAL;
  *out = nullptr;
  LSB_CUDA(cudaSetDevice(ctx->device));
  auto* idx = new lsb_index;
  idx->ctx = ctx;
  idx->V = vocab;
  idx->W = W;
  idx->dim = dim;
  idx->perm_seed = perm_seed;
  idx->attempts = 0;
  idx->bands_host.resize(W);
  uint32_t total = 0;
  for (int w = 0; w < W; ++w) {
    if (lg_host[w] < 1 || lg_host[w] > 30) {
      lsb_index_destroy(idx);
      return set_error("lsb_index_import: table size out of range"), LSB_EINVAL;
    }
    idx->bands_host[w] = BandMeta{mul_host[2 * w], mul_host[2 * w + 1], lg_host[w], total};
    total += 2u << lg_host[w];
  }
  idx->total_slots = total;
  std::vector<uint4> slots(total);
  uint32_t max_span = 0;
  for (uint32_t i = 0; i < total; ++i) {
    slots[i] = make_uint4(slots_host[3 * i], slots_host[3 * i + 1], slots_host[3 * i + 2], 0);
    if (slots[i].x != kEmptyCode) {
      max_span = std::max(max_span, slots[i].z);
      if (word_ids_host && static_cast<uint64_t>(slots[i].y) + slots[i].z > vocab) {
        lsb_index_destroy(idx);
        return set_error("lsb_index_import: span exceeds the vocabulary"), LSB_EINVAL;
      }
    }
  }
  idx->max_span = max_span;
  const size_t VW = static_cast<size_t>(vocab) * W;
  auto fail = [&](cudaError_t e, const char* what) {
    lsb_index_destroy(idx);
    return cuda_status(e, what);
  };
  cudaError_t e = cudaMalloc(&idx->word_ids, std::max<size_t>(VW, 1) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&idx->slots, std::max<size_t>(total, 1) * sizeof(uint4));
  if (e == cudaSuccess) e = cudaMalloc(&idx->bands, W * sizeof(BandMeta));
  if (e != cudaSuccess) return fail(e, "lsb_index_import alloc");
  cudaStream_t st = ctx->stream;
  if (VW && word_ids_host)
    e = cudaMemcpyAsync(idx->word_ids, word_ids_host, VW * 4, cudaMemcpyHostToDevice, st);
  else if (VW)
    e = cudaMemsetAsync(idx->word_ids, 0, VW * 4, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(idx->slots, slots.data(), total * sizeof(uint4), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(idx->bands, idx->bands_host.data(), W * sizeof(BandMeta),
                        cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return fail(e, "lsb_index_import upload");
  if (perms_host) {
    if (K < 2 || u < 1 || dim < K) {
      lsb_index_destroy(idx);
      return set_error("lsb_index_import: bad permutation parameters"), LSB_EINVAL;
    }
    idx->K = K;
    idx->u = u;
    int bits = 0;
    while ((1 << bits) < K) ++bits;
    idx->bits = bits;
    idx->P = u * W;
    idx->perms_host.assign(perms_host, perms_host + static_cast<size_t>(idx->P) * K);
    for (uint32_t p : idx->perms_host)
      if (p >= static_cast<uint32_t>(dim)) {
        lsb_index_destroy(idx);
        return set_error("PermutationSet: index out of range"), LSB_EINVAL;
      }
    e = cudaMalloc(&idx->perms, idx->perms_host.size() * 4);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(idx->perms, idx->perms_host.data(), idx->perms_host.size() * 4,
                          cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = upload_perms16(idx, st);
    if (e != cudaSuccess) return fail(e, "lsb_index_import perms");
    idx->has_perms = true;
  }
  lsb_status rc = lsb_ctx_sync(ctx);
  if (rc) {
    lsb_index_destroy(idx);
    return rc;
  }
  *out = idx;
  return LSB_OK;
}

lsb_status lsb_recurrent_create(lsb_ctx* ctx, const float* wh_host, const float* we_host, int d,
                                lsb_recurrent** out) {
  if (!ctx || !wh_host || !we_host || d < 1 || !out)
    return set_error("lsb_recurrent_create: bad arguments"), LSB_EINVAL;
  LSB_CUDA(cudaSetDevice(ctx->device));
  auto* r = new lsb_recurrent;
  const size_t dd = static_cast<size_t>(d) * d;
  cudaError_t e = cudaMalloc(&r->wh, dd * 4);
  if (e == cudaSuccess) e = cudaMalloc(&r->we, dd * 4);
  if (e == cudaSuccess) e = cudaMemcpyAsync(r->wh, wh_host, dd * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(r->we, we_host, dd * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    if (r->wh) cudaFree(r->wh);
    if (r->we) cudaFree(r->we);
    delete r;
    return cuda_status(e, "lsb_recurrent_create");
  }
  *out = r;
  return LSB_OK;
}

lsb_status lsb_recurrent_destroy(lsb_recurrent* r) {
  if (!r) return LSB_OK;
  if (r->wh) cudaFree(r->wh);
  if (r->we) cudaFree(r->we);
  delete r;
  return LSB_OK;
}

lsb_status lsb_recurrence(lsb_ctx* ctx, const lsb_model* model, const lsb_recurrent* rec,
                          const float* hidden_in_dev, const int64_t* tokens_dev, int n,
                          float* hidden_out_dev) {
  if (!ctx || !model || !rec || n < 0) return set_error("lsb_recurrence: bad arguments"), LSB_EINVAL;
  if (n == 0) return LSB_OK;
  const int d = model->d;
  const size_t smem = static_cast<size_t>(d) * 8;
  if (smem > ctx->smem_optin) return set_error("lsb_recurrence: dimension too large"), LSB_EINVAL;
  if (lsb_status rc = ensure_smem(ctx, k_recurrence, smem)) return rc;
  const int threads = 256;
  const int gx = std::max(1, std::min((d + 7) / 8, 64));
  k_recurrence<<<dim3(gx, n), threads, smem, ctx->stream>>>(rec->wh, rec->we, model->E, model->V,
                                                             d, hidden_in_dev, tokens_dev, n,
                                                             hidden_out_dev, ctx->err_dev);
  LSB_LAUNCHED(ctx, "k_recurrence");
  return LSB_OK;
}

lsb_status lsb_step_hidden(lsb_ctx* ctx, const lsb_model* model, const lsb_recurrent* rec,
                           const float* h_host, uint32_t token, float* out_host) {
  if (!ctx || !model || !rec || !h_host || !out_host)
    return set_error("step_hidden: bad arguments"), LSB_EINVAL;
  if (token >= model->V)
    return set_error("step_hidden: token " + std::to_string(token) + " out of range"), LSB_EINVAL;
  const int d = model->d;
  Dev<float> h, o;
  Dev<int64_t> t;
  LSB_CUDA(h.alloc(d));
  LSB_CUDA(o.alloc(d));
  LSB_CUDA(t.alloc(1));
  const int64_t tok = token;
  cudaStream_t st = ctx->stream;
  LSB_CUDA(cudaMemcpyAsync(h.p, h_host, d * 4ull, cudaMemcpyHostToDevice, st));
  LSB_CUDA(cudaMemcpyAsync(t.p, &tok, 8, cudaMemcpyHostToDevice, st));
  lsb_status rc = lsb_recurrence(ctx, model, rec, h.p, t.p, 1, o.p);
  if (rc) return rc;
  LSB_CUDA(cudaMemcpyAsync(out_host, o.p, d * 4ull, cudaMemcpyDeviceToHost, st));
  return lsb_ctx_sync(ctx);
}

// exact_topb_logits(H . E^T + bias, b): per row the b largest logits, ties
// to the smaller id (src/eval_oracle.cpp:11-40). PARITY logits (K4 over the
// whole vocabulary), then k_exact_topb on the signed values.
lsb_status lsb_exact_topb(lsb_ctx* ctx, const lsb_model* model, const float* H, int rows,
                          int H_on_device, int b, int add_bias, uint32_t* ids_host,
                          float* values_host) {
  if (!ctx || !model || rows < 0 || b < 0) return set_error("exact_topb: bad arguments"), LSB_EINVAL;
  if (static_cast<uint32_t>(b) > model->V)
    return set_error("exact_topb: b_out exceeds column count"), LSB_EINVAL;
  if (rows == 0 || b == 0) return LSB_OK;
  if (b > 64) return set_error("exact_topb: b above 64 is not supported"), LSB_EINVAL;
  const int d = model->d;
  const uint32_t V = model->V;
  cudaStream_t st = ctx->stream;
  Dev<float> Hd, L, vals;
  Dev<uint32_t> ids;
  const float* Hp = H;
  if (!H_on_device) {
    LSB_CUDA(Hd.alloc(static_cast<size_t>(rows) * d));
    LSB_CUDA(cudaMemcpyAsync(Hd.p, H, static_cast<size_t>(rows) * d * 4, cudaMemcpyHostToDevice, st));
    Hp = Hd.p;
  }
  LSB_CUDA(L.alloc(static_cast<size_t>(rows) * V));
  LSB_CUDA(ids.alloc(static_cast<size_t>(rows) * b));
  LSB_CUDA(vals.alloc(static_cast<size_t>(rows) * b));
  LogitsArgs la{};
  la.H = Hp;
  la.d = d;
  la.R_total = rows;
  la.Bsent = std::min(rows, 16);
  la.E = model->E;
  la.bias = add_bias ? model->bias : nullptr;
  la.n_shared = V;
  la.out = L.p;
  la.ldo = V;
  lsb_status rc = launch_logits(ctx, la, LSB_MODE_PARITY, ctx->sm_count * 8);
  if (rc) return rc;
  k_exact_topb<<<rows, kTopbThreads, 0, st>>>(L.p, V, V, b, ids.p, vals.p);
  LSB_LAUNCHED(ctx, "k_exact_topb");
  if (ids_host)
    LSB_CUDA(cudaMemcpyAsync(ids_host, ids.p, static_cast<size_t>(rows) * b * 4,
                             cudaMemcpyDeviceToHost, st));
  if (values_host)
    LSB_CUDA(cudaMemcpyAsync(values_host, vals.p, static_cast<size_t>(rows) * b * 4,
                             cudaMemcpyDeviceToHost, st));
  return lsb_ctx_sync(ctx);
}

}  // extern "C"
