// k_index.cu -- K1 (WTA hash) and K2-build (band index + parallel cuckoo).
//
// K1  k_wta_hash_rows : one warp per row; the row is staged in shared memory
//     with 16-byte coalesced loads, each lane evaluates permutations
//     p = lane, lane+32, ... (argmax over K permuted entries, strict '>' so
//     ties go to the smallest k: src/wta_hash.cpp:79-91) and the band codes
//     are packed u indices at a time, first index in the low bits
//     (src/wta_hash.cpp:106-116). Bit-exact by construction (comparisons only).
// K2  k_band_sort     : one CTA per band: stable LSD radix sort of (code, id)
//     on the code bits only (ids enter in ascending order, so the result is
//     the reference's sort of (code<<32 | id), src/band_index.cpp:103-108),
//     then the span table (code -> start, length).
//     k_cuckoo_build  : one CTA per band. REFERENCE placement (default): one
//     thread inserts the band's entries in the reference's order with its
//     swap-and-flip eviction chain, so slots, multipliers and rebuild count
//     are identical to CuckooTable::build (deterministic; WTAIDX1 bytes
//     match). PARALLEL placement: one thread per entry, 64-bit atomicExch
//     eviction chains (lookups are placement-independent). Both cap chains at
//     kMaxDisplacements hops and, on failure, retry with the next multiplier
//     pair of SplitMix64(mix_seed(seed, w)) (src/band_index.cpp:44-70).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lsb_internal.cuh"

namespace lsb {

constexpr unsigned long long kEmpty64 = ~0ull;

// ------------------------------------------------------------------ K1
__global__ void k_wta_hash_rows(const float* __restrict__ M, long long n, int d,
                                const uint32_t* __restrict__ perms, int K, int u, int W,
                                int bits, uint32_t* __restrict__ out, uint32_t* err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int P = u * W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  const int dpad = (d + 3) & ~3;
  const size_t per_warp = (static_cast<size_t>(dpad) * 4 + 2 * P + 15) & ~size_t(15);
  float* row = reinterpret_cast<float*>(smem + warp * per_warp);
  uint16_t* idx = reinterpret_cast<uint16_t*>(row + dpad);  // K <= 65536
  const bool vec = (d & 3) == 0;
  for (long long r = static_cast<long long>(blockIdx.x) * nwarp + warp; r < n;
       r += static_cast<long long>(gridDim.x) * nwarp) {
    const float* src = M + r * d;
    bool nan = false;
    if (vec) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* r4 = reinterpret_cast<float4*>(row);
      for (int c = lane; c < (d >> 2); c += 32) {
        const float4 v = __ldg(s4 + c);
        nan |= isnan(v.x) | isnan(v.y) | isnan(v.z) | isnan(v.w);
        r4[c] = v;
      }
    } else {
      for (int c = lane; c < d; c += 32) {
        const float v = __ldg(src + c);
        nan |= isnan(v);
        row[c] = v;
      }
    }
    if (__any_sync(0xffffffffu, nan)) {
      if (lane == 0) atomicOr(err, kErrNaN);
      continue;
    }
    __syncwarp();
    for (int p = lane; p < P; p += 32) {
      const uint32_t* pr = perms + static_cast<size_t>(p) * K;
      uint32_t best = 0;
      float bv = row[__ldg(pr)];
      for (int k = 1; k < K; ++k) {
        const float v = row[__ldg(pr + k)];
        if (v > bv) {
          bv = v;
          best = k;
        }
      }
      idx[p] = static_cast<uint16_t>(best);
    }
    __syncwarp();
    for (int w = lane; w < W; w += 32) {
      uint32_t code = 0;
      for (int i = 0; i < u; ++i) code |= static_cast<uint32_t>(idx[w * u + i]) << (i * bits);
      out[r * W + w] = code;
    }
    __syncwarp();
  }
}

// Exclusive scan of one value per thread over the CTA (blockDim <= 1024).
// Returns the exclusive prefix; *total receives the sum. Uses 33 words of smem.
__device__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* wsum, uint32_t* total) {
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
    uint32_t s = lane < nwarp ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nwarp) wsum[lane] = s;  // inclusive warp totals
    if (lane == 31) wsum[32] = s;
  }
  __syncthreads();
  const uint32_t base = warp ? wsum[warp - 1] : 0;
  const uint32_t res = base + x - v;
  if (total) *total = wsum[32];
  __syncthreads();
  return res;
}

// ------------------------------------------------------------- K2 sort
// Sorts band w's (code, id) pairs by code, stably. codes: V x W row-major
// (column w is this band). Ping-pong buffers ka/ia, kb/ib hold V entries per
// band. Output: word_ids[w][pos], entries (key,start,len) and their count.
__global__ void __launch_bounds__(1024) k_band_sort(
    const uint32_t* __restrict__ codes, uint32_t V, int W, int nbits, uint32_t* ka,
    uint32_t* ia, uint32_t* kb, uint32_t* ib, uint32_t* __restrict__ word_ids,
    uint32_t* __restrict__ ekey, uint32_t* __restrict__ estart, uint32_t* __restrict__ elen,
    uint32_t* __restrict__ n_entries, uint32_t* __restrict__ max_span) {
  extern __shared__ uint32_t hist[];  // 1 << digit bits
  __shared__ uint32_t wsum[33];
  __shared__ uint32_t carry;
  const int w = blockIdx.x;
  const size_t off = static_cast<size_t>(w) * V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  const int passes = nbits <= 0 ? 0 : (nbits + 11) / 12;
  const int dbits = passes ? (nbits + passes - 1) / passes : 0;
  const uint32_t nbins = 1u << dbits;

  uint32_t *sk = ka + off, *si = ia + off, *dk = kb + off, *di = ib + off;
  for (uint32_t j = threadIdx.x; j < V; j += blockDim.x) {
    sk[j] = codes[static_cast<size_t>(j) * W + w];
    si[j] = j;
  }
  __syncthreads();
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = pass * dbits;
    const uint32_t mask = nbins - 1;
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < V; j += blockDim.x)
      atomicAdd(&hist[(sk[j] >> shift) & mask], 1u);
    __syncthreads();
    // exclusive scan of the histogram, bins distributed contiguously
    const uint32_t per = (nbins + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per;
    uint32_t local = 0;
    for (uint32_t b = b0; b < b0 + per && b < nbins; ++b) local += hist[b];
    uint32_t run = block_exclusive_scan(local, wsum, nullptr);
    for (uint32_t b = b0; b < b0 + per && b < nbins; ++b) {
      const uint32_t c = hist[b];
      hist[b] = run;
      run += c;
    }
    __syncthreads();
    // ordered scatter: tiles of blockDim elements, warps take turns in order
    for (uint32_t base = 0; base < V; base += blockDim.x) {
      const uint32_t j = base + threadIdx.x;
      const bool valid = j < V;
      const uint32_t key = valid ? sk[j] : 0;
      const uint32_t id = valid ? si[j] : 0;
      const uint32_t dig = valid ? ((key >> shift) & mask) : 0xFFFFFFFFu;
      const unsigned peers = __match_any_sync(0xffffffffu, dig);
      const unsigned lt = (1u << lane) - 1;
      const uint32_t rank = __popc(peers & lt);
      const bool leader = (peers & lt) == 0;
      for (int tw = 0; tw < nwarp; ++tw) {
        if (warp == tw && valid) {
          const uint32_t pos = hist[dig] + rank;
          dk[pos] = key;
          di[pos] = id;
        }
        __syncwarp();
        if (warp == tw && valid && leader) hist[dig] += __popc(peers);
        __syncthreads();
      }
    }
    __syncthreads();
    uint32_t* t;
    t = sk; sk = dk; dk = t;
    t = si; si = di; di = t;
  }
  // word ids + spans
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  uint32_t* ids_out = word_ids + off;
  uint32_t span_max = 0;
  for (uint32_t base = 0; base < V; base += blockDim.x) {
    const uint32_t j = base + threadIdx.x;
    uint32_t flag = 0, key = 0;
    if (j < V) {
      key = sk[j];
      ids_out[j] = si[j];
      flag = (j == 0 || key != sk[j - 1]) ? 1u : 0u;
    }
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan(flag, wsum, &tot);
    if (flag) {
      ekey[off + carry + ex] = key;
      estart[off + carry + ex] = j;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  const uint32_t ne = carry;
  // lengths from consecutive starts
  for (uint32_t e = threadIdx.x; e < ne; e += blockDim.x) {
    const uint32_t s = estart[off + e];
    const uint32_t nx = e + 1 < ne ? estart[off + e + 1] : V;
    elen[off + e] = nx - s;
    span_max = max(span_max, nx - s);
  }
  if (span_max) atomicMax(max_span, span_max);
  if (threadIdx.x == 0) n_entries[w] = ne;
}

// ----------------------------------------------------------- K2 cuckoo
__global__ void __launch_bounds__(1024) k_cuckoo_build(
    const uint32_t* __restrict__ ekey, const uint32_t* __restrict__ estart,
    const uint32_t* __restrict__ elen, const uint32_t* __restrict__ n_entries, uint32_t V,
    unsigned long long index_seed, BandMeta* __restrict__ bands,
    unsigned long long* __restrict__ tmp, uint4* __restrict__ slots,
    uint32_t* __restrict__ attempts_out, uint32_t* err, int sequential, int smem_cap,
    int raw_seed) {
  __shared__ unsigned long long mul[2];
  __shared__ int fail;
  extern __shared__ __align__(16) unsigned long long sm_tab[];
  const int w = blockIdx.x;
  const size_t off = static_cast<size_t>(w) * V;
  const uint32_t ne = n_entries[w];
  BandMeta m = bands[w];
  const uint32_t cap = 1u << m.lg;
  // The band's two tables (and its keys) live in shared memory when they fit
  // (smem_cap >= cap): the reference-order insertion is one thread's serial
  // eviction chain, so its per-hop latency is the build time (global-memory
  // atomics: 772 us at cfg 2, shared memory: see DESIGN §4).
  const bool in_smem = cap <= static_cast<uint32_t>(smem_cap);
  unsigned long long* t = in_smem ? sm_tab : tmp + m.slot_off;
  const uint32_t* keys = ekey + off;
  if (in_smem) {
    uint32_t* sk = reinterpret_cast<uint32_t*>(sm_tab + 2 * cap);
    for (uint32_t e = threadIdx.x; e < ne; e += blockDim.x) sk[e] = ekey[off + e];
    keys = sk;
  }
  // BandIndex::build seeds band w's table with mix_seed(seed, w)
  // (src/band_index.cpp:90-132); a standalone CuckooTable::build(entries,
  // seed) draws its multipliers from SplitMix64(seed) itself (:42-45)
  unsigned long long g = raw_seed ? index_seed
                                  : mix_seed_dev(index_seed, static_cast<unsigned long long>(w));
  for (int attempt = 0; attempt <= kMaxRebuilds; ++attempt) {
    if (threadIdx.x == 0) {
      mul[0] = sm64_next(g) | 1ull;
      mul[1] = sm64_next(g) | 1ull;
      fail = 0;
    }
    for (uint32_t s = threadIdx.x; s < 2 * cap; s += blockDim.x) t[s] = kEmpty64;
    __syncthreads();
    const unsigned long long m0 = mul[0], m1 = mul[1];
    const uint32_t e0 = sequential ? (threadIdx.x == 0 ? 0u : ne) : threadIdx.x;
    const uint32_t estep = sequential ? 1u : blockDim.x;
    for (uint32_t e = e0; e < ne; e += estep) {
      unsigned long long cur = (static_cast<unsigned long long>(keys[e]) << 32) | e;
      int table = 0;
      bool placed = false;
      for (int hop = 0; hop < kMaxDisplacements; ++hop) {
        const uint32_t key = static_cast<uint32_t>(cur >> 32);
        const uint32_t pos = table ? cap + slot_of(m1, m.lg, key) : slot_of(m0, m.lg, key);
        if (sequential) {  // one thread: plain swap (shared-memory 64-bit atomics are slow)
          const unsigned long long prev = t[pos];
          t[pos] = cur;
          cur = prev;
        } else {
          cur = atomicExch(t + pos, cur);
        }
        if (cur == kEmpty64) {
          placed = true;
          break;
        }
        table = 1 - table;  // the evictee moves to its other table
      }
      if (!placed) {
        fail = 1;
        if (sequential) break;  // the reference abandons the attempt here
      }
    }
    __syncthreads();
    if (!fail) {
      for (uint32_t s = threadIdx.x; s < 2 * cap; s += blockDim.x) {
        const unsigned long long v = t[s];
        uint4 o = make_uint4(kEmptyCode, 0, 0, 0);
        if (v != kEmpty64) {
          const uint32_t e = static_cast<uint32_t>(v);
          o = make_uint4(static_cast<uint32_t>(v >> 32), estart[off + e], elen[off + e], 0);
        }
        slots[m.slot_off + s] = o;
      }
      if (threadIdx.x == 0) {
        m.mul0 = m0;
        m.mul1 = m1;
        bands[w] = m;
        atomicMax(attempts_out, static_cast<uint32_t>(attempt + 1));
      }
      return;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicOr(err, kErrCuckoo);
}

// ------------------------------------------------- K2-lookup (dense stage)
// BandIndex::lookup_hits_into: one CTA per query row, one warp per band
// (lanes 0/1 probe both tables, then the warp walks the span coalesced).
__global__ void k_lookup_dense(IndexView ix, const uint32_t* __restrict__ q, int B,
                               int32_t* __restrict__ L) {
  const int row = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  int32_t* Lr = L + static_cast<size_t>(row) * ix.V;
  for (int w = warp; w < ix.W; w += nwarp) {
    uint32_t start, len;
    if (!warp_probe(ix, w, q[static_cast<size_t>(row) * ix.W + w], start, len)) continue;
    const uint32_t* ids = ix.word_ids + static_cast<size_t>(w) * ix.V + start;
    for (uint32_t k = lane; k < len; k += 32) atomicAdd(Lr + __ldg(ids + k), 1);
  }
}

__global__ void k_find_batch(IndexView ix, const int32_t* __restrict__ bands,
                             const uint32_t* __restrict__ keys, size_t n,
                             uint32_t* __restrict__ start, uint32_t* __restrict__ len,
                             uint8_t* __restrict__ found) {
  const size_t qi = static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (qi >= n) return;
  uint32_t s = 0, l = 0;
  const bool hit = warp_probe(ix, bands[qi], keys[qi], s, l);
  if ((threadIdx.x & 31) == 0) {
    found[qi] = hit;
    start[qi] = hit ? s : 0;
    len[qi] = hit ? l : 0;
  }
}

// ------------------------------------------------------------ host side
// PermutationSet::generate, src/wta_hash.cpp:31-55 (host, bit-exact).
cudaError_t upload_perms16(lsb_index* idx, cudaStream_t st) {
  if (idx->dim > 65535 || idx->K < 1 || idx->perms_host.empty()) return cudaSuccess;
  const int K16 = (idx->K + 7) & ~7;
  std::vector<uint16_t> h(static_cast<size_t>(idx->P) * K16, 0);
  for (int p = 0; p < idx->P; ++p)
    for (int k = 0; k < idx->K; ++k)
      h[static_cast<size_t>(p) * K16 + k] =
          static_cast<uint16_t>(idx->perms_host[static_cast<size_t>(p) * idx->K + k]);
  cudaError_t e = cudaMalloc(&idx->perms16, h.size() * sizeof(uint16_t));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(idx->perms16, h.data(), h.size() * sizeof(uint16_t),
                        cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // h is a stack temporary
  if (e == cudaSuccess) idx->K16 = K16;
  return e;
}

static void generate_perms_host(int d, int P, int K, uint64_t seed, std::vector<uint32_t>& out) {
  out.assign(static_cast<size_t>(P) * K, 0);
  std::vector<uint32_t> scratch(d);
  uint64_t s = seed;
  auto next = [&s]() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  for (int p = 0; p < P; ++p) {
    for (int i = 0; i < d; ++i) scratch[i] = static_cast<uint32_t>(i);
    for (int k = 0; k < K; ++k) {
      const uint64_t bound = static_cast<uint64_t>(d - k);
      const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
      uint64_t x = next();
      while (x >= limit) x = next();
      const uint64_t j = k + x % bound;
      std::swap(scratch[k], scratch[j]);
      out[static_cast<size_t>(p) * K + k] = scratch[k];
    }
  }
}

int bits_for(int K) {
  int b = 0;
  while ((1 << b) < K) ++b;
  return b;
}

// WtaParams ctor, src/wta_hash.cpp:18-29
lsb_status check_wta_params(int K, int u, int W) {
  if (K < 2) return set_error("WtaParams: K must be >= 2"), LSB_EINVAL;
  if (u < 1) return set_error("WtaParams: u must be >= 1"), LSB_EINVAL;
  if (W < 1) return set_error("WtaParams: W must be >= 1"), LSB_EINVAL;
  // the device keeps argmax indices in 16 bits (K <= d in practice)
  if (K > 65536) return set_error("WtaParams: K above 65536 is not supported"), LSB_EINVAL;
  if (u * bits_for(K) >= 31)
    return set_error("WtaParams: packing overflow, u*ceil(log2(K)) = " +
                     std::to_string(u * bits_for(K)) +
                     " bits does not fit a 31-bit band code"),
           LSB_EINVAL;
  return LSB_OK;
}

// Launch K1 over n device rows.
lsb_status launch_wta_hash(lsb_ctx* ctx, const float* M, long long n, int d,
                           const uint32_t* perms, int K, int u, int W, uint32_t* out) {
  if (n == 0) return LSB_OK;
  const int P = u * W;
  const int dpad = (d + 3) & ~3;
  const size_t per_warp = (static_cast<size_t>(dpad) * 4 + 2 * P + 15) & ~size_t(15);
  const size_t budget = 96 * 1024;
  int warps = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, budget / per_warp)));
  const size_t smem = per_warp * warps;
  if (smem > ctx->smem_optin) {
    set_error("wta_hash: row of dimension " + std::to_string(d) + " exceeds shared memory");
    return LSB_EINVAL;
  }
  if (lsb_status rc = ensure_smem(ctx, k_wta_hash_rows, smem)) return rc;
  const long long blocks_needed = (n + warps - 1) / warps;
  const int grid = static_cast<int>(std::min<long long>(blocks_needed, ctx->sm_count * 16LL));
  k_wta_hash_rows<<<grid, warps * 32, smem, ctx->stream>>>(M, n, d, perms, K, u, W, bits_for(K),
                                                          out, ctx->err_dev);
  LSB_LAUNCHED(ctx, "k_wta_hash_rows");
  return LSB_OK;
}

// Device buffer that frees itself.
template <class T>
struct DevBuf {
  // stream-ordered scratch (cudaMallocAsync / cudaFreeAsync on the context
  // stream): the build's dozen temporaries cost no device-wide allocator
  // synchronisation (cudaMalloc + cudaFree: ~5 ms of a 6 ms cfg-2 build)
  T* p = nullptr;
  cudaStream_t st = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(size_t n, cudaStream_t stream) {
    st = stream;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), st);
  }
};

// Largest table capacity (2^lg slots per table) whose two tables (8 B per
// slot) and keys (4 B per entry, <= 2^lg) fit the device's shared memory;
// 0 = none (global tables).
static int cuckoo_smem_cap(const lsb_ctx* ctx, uint32_t lg_max) {
  static const bool off = getenv("LSB_CUCKOO_GLOBAL") != nullptr;
  if (off || lg_max > 16) return 0;
  const size_t need = (static_cast<size_t>(1) << lg_max) * 20;
  return need + 64 <= ctx->smem_optin ? (1 << lg_max) : 0;
}

// Builds the band tables of `idx` from device codes (V x W).
static lsb_status build_bands(lsb_ctx* ctx, lsb_index* idx, const uint32_t* codes_dev,
                              int nbits) {
  const uint32_t V = idx->V;
  const int W = idx->W;
  const size_t VW = static_cast<size_t>(V) * W;
  DevBuf<uint32_t> ka, ia, kb, ib, ekey, estart, elen, nent, maxspan, attempts;
  LSB_CUDA(ka.alloc(VW, ctx->stream));
  LSB_CUDA(ia.alloc(VW, ctx->stream));
  LSB_CUDA(kb.alloc(VW, ctx->stream));
  LSB_CUDA(ib.alloc(VW, ctx->stream));
  LSB_CUDA(ekey.alloc(VW, ctx->stream));
  LSB_CUDA(estart.alloc(VW, ctx->stream));
  LSB_CUDA(elen.alloc(VW, ctx->stream));
  LSB_CUDA(nent.alloc(W, ctx->stream));
  LSB_CUDA(maxspan.alloc(1, ctx->stream));
  LSB_CUDA(attempts.alloc(1, ctx->stream));
  LSB_CUDA(cudaMalloc(&idx->word_ids, std::max<size_t>(VW, 1) * sizeof(uint32_t)));
  LSB_CUDA(cudaMemsetAsync(maxspan.p, 0, 4, ctx->stream));
  LSB_CUDA(cudaMemsetAsync(attempts.p, 0, 4, ctx->stream));
  const int passes = nbits <= 0 ? 0 : (nbits + 11) / 12;
  const int dbits = passes ? (nbits + passes - 1) / passes : 0;
  const size_t hsmem = sizeof(uint32_t) << dbits;
  k_band_sort<<<W, 1024, hsmem, ctx->stream>>>(codes_dev, V, W, nbits, ka.p, ia.p, kb.p, ib.p,
                                               idx->word_ids, ekey.p, estart.p, elen.p, nent.p,
                                               maxspan.p);
  LSB_LAUNCHED(ctx, "k_band_sort");
  std::vector<uint32_t> ne(W);
  LSB_CUDA(cudaMemcpyAsync(ne.data(), nent.p, W * 4, cudaMemcpyDeviceToHost, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(&idx->max_span, maxspan.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  LSB_CUDA(cudaStreamSynchronize(ctx->stream));
  // Table sizes: lg = max(1, ceil log2 #entries) (src/band_index.cpp:39).
  idx->bands_host.resize(W);
  uint32_t total = 0;
  for (int w = 0; w < W; ++w) {
    uint32_t lg = 0;
    while ((1ull << lg) < ne[w]) ++lg;
    lg = std::max(1u, lg);
    idx->bands_host[w] = BandMeta{1ull, 1ull, lg, total};
    total += 2u << lg;
  }
  idx->total_slots = total;
  DevBuf<unsigned long long> tmp;
  LSB_CUDA(tmp.alloc(total, ctx->stream));
  LSB_CUDA(cudaMalloc(&idx->slots, std::max<size_t>(total, 1) * sizeof(uint4)));
  LSB_CUDA(cudaMalloc(&idx->bands, W * sizeof(BandMeta)));
  LSB_CUDA(cudaMemcpyAsync(idx->bands, idx->bands_host.data(), W * sizeof(BandMeta),
                           cudaMemcpyHostToDevice, ctx->stream));
  uint32_t lg_max = 1;
  for (int w = 0; w < W; ++w) lg_max = std::max(lg_max, idx->bands_host[w].lg);
  const int smem_cap = cuckoo_smem_cap(ctx, lg_max);
  const size_t csmem = smem_cap ? static_cast<size_t>(smem_cap) * 20 : 0;
  if (csmem) LSB_CUDA(cudaFuncSetAttribute(k_cuckoo_build, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(csmem)));
  k_cuckoo_build<<<W, 1024, csmem, ctx->stream>>>(ekey.p, estart.p, elen.p, nent.p, V,
                                                  idx->index_seed, idx->bands, tmp.p, idx->slots,
                                                  attempts.p, ctx->err_dev,
                                                  ctx->cuckoo_parallel ? 0 : 1, smem_cap, 0);
  LSB_LAUNCHED(ctx, "k_cuckoo_build");
  LSB_CUDA(cudaMemcpyAsync(idx->bands_host.data(), idx->bands, W * sizeof(BandMeta),
                           cudaMemcpyDeviceToHost, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(&idx->attempts, attempts.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  return lsb_ctx_sync(ctx);
}

// One standalone table (CuckooTable::build): entries already on the device.
lsb_status build_cuckoo_band(lsb_ctx* ctx, const uint32_t* keys, const uint32_t* starts,
                             const uint32_t* lens, uint32_t n, uint64_t seed, uint32_t lg,
                             uint4* slots_dev, BandMeta* meta_dev, uint32_t* attempts_dev) {
  DevBuf<unsigned long long> tmp;
  DevBuf<uint32_t> ne;
  LSB_CUDA(tmp.alloc(2u << lg, ctx->stream));
  LSB_CUDA(ne.alloc(1, ctx->stream));
  const BandMeta m{1ull, 1ull, lg, 0};
  LSB_CUDA(cudaMemcpyAsync(ne.p, &n, 4, cudaMemcpyHostToDevice, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(meta_dev, &m, sizeof(m), cudaMemcpyHostToDevice, ctx->stream));
  LSB_CUDA(cudaMemsetAsync(attempts_dev, 0, 4, ctx->stream));
  const int smem_cap = cuckoo_smem_cap(ctx, lg);
  const size_t csmem = smem_cap ? static_cast<size_t>(smem_cap) * 20 : 0;
  if (csmem) LSB_CUDA(cudaFuncSetAttribute(k_cuckoo_build, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(csmem)));
  k_cuckoo_build<<<1, 1024, csmem, ctx->stream>>>(keys, starts, lens, ne.p, n, seed, meta_dev, tmp.p,
                                                 slots_dev, attempts_dev, ctx->err_dev,
                                                 ctx->cuckoo_parallel ? 0 : 1, smem_cap, 1);
  LSB_LAUNCHED(ctx, "k_cuckoo_build");
  return lsb_ctx_sync(ctx);
}

}  // namespace lsb

using namespace lsb;

extern "C" {

lsb_status lsb_index_destroy(lsb_index* idx) {
  if (!idx) return LSB_OK;
  if (idx->perms) cudaFree(idx->perms);
  if (idx->perms16) cudaFree(idx->perms16);
  if (idx->word_ids) cudaFree(idx->word_ids);
  if (idx->slots) cudaFree(idx->slots);
  if (idx->bands) cudaFree(idx->bands);
  delete idx;
  return LSB_OK;
}

lsb_status lsb_index_build(lsb_ctx* ctx, const lsb_model* model, int K, int u, int W,
                           uint64_t perm_seed, uint64_t index_seed, lsb_index** out) {
  if (!ctx || !model || !out) return set_error("lsb_index_build: null argument"), LSB_EINVAL;
  *out = nullptr;
  lsb_status st = check_wta_params(K, u, W);
  if (st) return st;
  if (model->d < K)
    return set_error("PermutationSet: dimension " + std::to_string(model->d) +
                     " smaller than window " + std::to_string(K)),
           LSB_EINVAL;
  LSB_CUDA(cudaSetDevice(ctx->device));
  auto* idx = new lsb_index;
  idx->ctx = ctx;
  idx->V = model->V;
  idx->W = W;
  idx->K = K;
  idx->u = u;
  idx->bits = bits_for(K);
  idx->P = u * W;
  idx->dim = model->d;
  idx->perm_seed = perm_seed;
  idx->index_seed = index_seed;
  idx->has_perms = true;
  generate_perms_host(model->d, idx->P, K, perm_seed, idx->perms_host);
  auto fail = [&](lsb_status s) {
    lsb_index_destroy(idx);
    return s;
  };
  cudaError_t e = cudaMalloc(&idx->perms, idx->perms_host.size() * sizeof(uint32_t));
  if (e != cudaSuccess) return fail(cuda_status(e, "cudaMalloc perms"));
  e = cudaMemcpyAsync(idx->perms, idx->perms_host.data(), idx->perms_host.size() * 4,
                      cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) return fail(cuda_status(e, "upload perms"));
  e = upload_perms16(idx, ctx->stream);
  if (e != cudaSuccess) return fail(cuda_status(e, "upload perms16"));
  DevBuf<uint32_t> codes;
  e = codes.alloc(static_cast<size_t>(model->V) * W, ctx->stream);
  if (e != cudaSuccess) return fail(cuda_status(e, "cudaMalloc codes"));
  st = launch_wta_hash(ctx, model->E, model->V, model->d, idx->perms, K, u, W, codes.p);
  if (st) return fail(st);
  st = lsb_ctx_sync(ctx);  // NaN in E -> EINVAL before building tables
  if (st) return fail(st);
  st = build_bands(ctx, idx, codes.p, u * idx->bits);
  if (st) return fail(st);
  *out = idx;
  return LSB_OK;
}

lsb_status lsb_index_build_codes(lsb_ctx* ctx, const uint32_t* codes_host, uint32_t vocab,
                                 int W, uint64_t index_seed, lsb_index** out) {
  if (!ctx || !out || (!codes_host && vocab) || W < 1)
    return set_error("lsb_index_build_codes: bad arguments"), LSB_EINVAL;
  *out = nullptr;
  const size_t VW = static_cast<size_t>(vocab) * W;
  uint32_t maxc = 0;
  for (size_t i = 0; i < VW; ++i) maxc = std::max(maxc, codes_host[i]);
  if (VW && maxc >= kEmptyCode)  // CuckooTable::build, src/band_index.cpp:35-36
    return set_error("CuckooTable: key collides with sentinel"), LSB_EINVAL;
  LSB_CUDA(cudaSetDevice(ctx->device));
  auto* idx = new lsb_index;
  idx->ctx = ctx;
  idx->V = vocab;
  idx->W = W;
  idx->index_seed = index_seed;
  int nbits = 0;
  while (nbits < 32 && (maxc >> nbits)) ++nbits;
  DevBuf<uint32_t> codes;
  cudaError_t e = codes.alloc(VW, ctx->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(codes.p, codes_host, VW * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) {
    lsb_index_destroy(idx);
    return cuda_status(e, "upload codes");
  }
  lsb_status st = build_bands(ctx, idx, codes.p, nbits);
  if (st) {
    lsb_index_destroy(idx);
    return st;
  }
  *out = idx;
  return LSB_OK;
}

lsb_status lsb_index_info_get(const lsb_index* idx, lsb_index_info* o) {
  if (!idx || !o) return set_error("lsb_index_info_get: null"), LSB_EINVAL;
  o->vocab = idx->V;
  o->W = idx->W;
  o->K = idx->K;
  o->u = idx->u;
  o->bits_per_index = idx->bits;
  o->dim = idx->dim;
  o->perm_seed = idx->perm_seed;
  o->index_seed = idx->index_seed;
  o->max_span = idx->max_span;
  o->build_attempts = idx->attempts;
  return LSB_OK;
}

lsb_status lsb_index_band(const lsb_index* idx, int w, uint32_t* word_ids_host, uint32_t* lg,
                          uint64_t* mul2, uint32_t* slots_host) {
  if (!idx || w < 0 || w >= idx->W || !lg) return set_error("lsb_index_band: bad band"), LSB_EINVAL;
  const BandMeta& m = idx->bands_host[w];
  *lg = m.lg;
  if (mul2) {
    mul2[0] = m.mul0;
    mul2[1] = m.mul1;
  }
  cudaStream_t s = idx->ctx->stream;
  if (word_ids_host && idx->V)
    LSB_CUDA(cudaMemcpyAsync(word_ids_host, idx->word_ids + static_cast<size_t>(w) * idx->V,
                             idx->V * 4ull, cudaMemcpyDeviceToHost, s));
  std::vector<uint4> tmp;
  if (slots_host) {
    tmp.resize(2u << m.lg);
    LSB_CUDA(cudaMemcpyAsync(tmp.data(), idx->slots + m.slot_off, tmp.size() * sizeof(uint4),
                             cudaMemcpyDeviceToHost, s));
  }
  LSB_CUDA(cudaStreamSynchronize(s));
  for (size_t i = 0; i < tmp.size(); ++i) {
    slots_host[3 * i] = tmp[i].x;
    slots_host[3 * i + 1] = tmp[i].y;
    slots_host[3 * i + 2] = tmp[i].z;
  }
  return LSB_OK;
}

lsb_status lsb_index_perms(const lsb_index* idx, uint32_t* perms_host) {
  if (!idx || !perms_host || !idx->has_perms)
    return set_error("lsb_index_perms: index has no permutations"), LSB_EINVAL;
  std::memcpy(perms_host, idx->perms_host.data(), idx->perms_host.size() * 4);
  return LSB_OK;
}

lsb_status lsb_index_find(lsb_ctx* ctx, const lsb_index* idx, const int32_t* bands_host,
                          const uint32_t* keys_host, size_t n, uint32_t* start_host,
                          uint32_t* len_host, uint8_t* found_host) {
  if (!ctx || !idx) return set_error("lsb_index_find: null"), LSB_EINVAL;
  if (n == 0) return LSB_OK;
  for (size_t i = 0; i < n; ++i)
    if (bands_host[i] < 0 || bands_host[i] >= idx->W)
      return set_error("lsb_index_find: band out of range"), LSB_EINVAL;
  DevBuf<int32_t> b;
  DevBuf<uint32_t> k, s, l;
  DevBuf<uint8_t> f;
  LSB_CUDA(b.alloc(n, ctx->stream));
  LSB_CUDA(k.alloc(n, ctx->stream));
  LSB_CUDA(s.alloc(n, ctx->stream));
  LSB_CUDA(l.alloc(n, ctx->stream));
  LSB_CUDA(f.alloc(n, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(b.p, bands_host, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(k.p, keys_host, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  const int wpb = 8;
  k_find_batch<<<static_cast<unsigned>((n + wpb - 1) / wpb), wpb * 32, 0, ctx->stream>>>(
      idx->view(), b.p, k.p, n, s.p, l.p, f.p);
  LSB_LAUNCHED(ctx, "k_find_batch");
  LSB_CUDA(cudaMemcpyAsync(start_host, s.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(len_host, l.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(found_host, f.p, n, cudaMemcpyDeviceToHost, ctx->stream));
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_wta_hash(lsb_ctx* ctx, const float* M_host, int64_t n, int d,
                        const uint32_t* perms_host, int K, int u, int W,
                        uint32_t* codes_host) {
  if (!ctx || n < 0 || d < 1) return set_error("lsb_wta_hash: bad arguments"), LSB_EINVAL;
  lsb_status st = check_wta_params(K, u, W);
  if (st) return st;
  const size_t P = static_cast<size_t>(u) * W;
  for (size_t i = 0; i < P * K; ++i)
    if (perms_host[i] >= static_cast<uint32_t>(d))
      return set_error("PermutationSet: index out of range"), LSB_EINVAL;
  if (n == 0) return LSB_OK;
  DevBuf<float> M;
  DevBuf<uint32_t> p, out;
  LSB_CUDA(M.alloc(static_cast<size_t>(n) * d, ctx->stream));
  LSB_CUDA(p.alloc(P * K, ctx->stream));
  LSB_CUDA(out.alloc(static_cast<size_t>(n) * W, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(M.p, M_host, static_cast<size_t>(n) * d * 4, cudaMemcpyHostToDevice,
                           ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(p.p, perms_host, P * K * 4, cudaMemcpyHostToDevice, ctx->stream));
  st = launch_wta_hash(ctx, M.p, n, d, p.p, K, u, W, out.p);
  if (st) return st;
  // a NaN row raises (invalid_argument) before anything is copied back, so
  // codes_host is left untouched as by the reference's throw
  if ((st = lsb_ctx_sync(ctx))) return st;
  LSB_CUDA(cudaMemcpyAsync(codes_host, out.p, static_cast<size_t>(n) * W * 4,
                           cudaMemcpyDeviceToHost, ctx->stream));
  return lsb_ctx_sync(ctx);
}

lsb_status lsb_lookup_hits(lsb_ctx* ctx, const lsb_index* idx, const uint32_t* q_host, int B,
                           int32_t* L_host) {
  if (!ctx || !idx || B < 0) return set_error("lsb_lookup_hits: bad arguments"), LSB_EINVAL;
  if (B == 0 || idx->V == 0) return LSB_OK;
  const size_t BV = static_cast<size_t>(B) * idx->V;
  DevBuf<uint32_t> q;
  DevBuf<int32_t> L;
  LSB_CUDA(q.alloc(static_cast<size_t>(B) * idx->W, ctx->stream));
  LSB_CUDA(L.alloc(BV, ctx->stream));
  LSB_CUDA(cudaMemcpyAsync(q.p, q_host, static_cast<size_t>(B) * idx->W * 4,
                           cudaMemcpyHostToDevice, ctx->stream));
  LSB_CUDA(cudaMemsetAsync(L.p, 0, BV * 4, ctx->stream));
  k_lookup_dense<<<B, 256, 0, ctx->stream>>>(idx->view(), q.p, B, L.p);
  LSB_LAUNCHED(ctx, "k_lookup_dense");
  LSB_CUDA(cudaMemcpyAsync(L_host, L.p, BV * 4, cudaMemcpyDeviceToHost, ctx->stream));
  return lsb_ctx_sync(ctx);
}

}  // extern "C"
