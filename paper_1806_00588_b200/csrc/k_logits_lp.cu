// k_logits_lp.cu -- K4 PARITY with the reference's four accumulation lanes
// split over two threads ("lane pairs").
//
// Same job as k_logits (logits = H . E[ids]^T + bias[ids], gathered E rows,
// shared top-T block + per-sentence survivors; src/candidate_selector.cpp:
// 105-119, src/beam_decoder.cpp:23-44, :237-247) and the same bits: lane j of
// an output sums fl(h[c] * e[c]) for c = j mod 4 in ascending c, the d mod 4
// tail goes into lane 0, and the result is ((0 + l0) + l1 + l2) + l3 + bias.
//
// Why a second PARITY kernel: the 4-lanes-per-thread tile of k_logits needs a
// 16-byte H load per row and per column per d-quad, and a 16-byte shared-memory
// load costs 4 wavefronts on sm_100 whatever the broadcast pattern, so it is
// shared-memory bound (ncu r01h: 28 wavefronts per 48 FFMA2 per warp, LSU ~117%
// of the FP32 pipe's demand). Here a thread owns ONE lane pair (reference
// lanes 2p, 2p+1) of RB rows x 4 columns: per d-quad it loads one 8-byte H
// pair per row and one 8-byte E pair per column (2 wavefronts each) for
// 2 x RB x 4 FFMA2 -- at RB = 12 that is 32 wavefronts per 96 FFMA2 per warp,
// ~67% of the FP32 pipe, so the kernel is FP32-issue bound. The two halves of
// each output meet in the epilogue through one shuffle.
//
// Warp layout: lane = 2 * cl + p (cl = 0..15 column slot, p = lane pair); a
// thread's columns are warp * 64 + cl + 16 j (j = 0..3). With a shared-memory
// row pitch of 20 floats (KC = 16), the 8-byte loads of a half-warp hit 16
// distinct bank pairs (8 columns x 2 lane pairs).
//
// Exactness of the paired ops (as in k_logits' mac4_x2): fma(h, e, -0) is
// fl(h*e) and fma(acc, 1, prod) is fl(acc + prod), signed zeros included; the
// -0 and 1 operands are runtime values so ptxas cannot re-contract the pair
// into a single-rounding FFMA2.
#include <algorithm>
#include <cstdlib>

#include "k_step.cuh"

namespace lsb {

namespace {

constexpr int kLpKC = 16;              // d floats per staged chunk
constexpr int kLpKS = kLpKC + 4;       // smem row pitch (floats)
constexpr int kLpColsPerWarp = 64;

__device__ __forceinline__ void lp_cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void lp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void lp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ unsigned long long lp_f2fma(unsigned long long a, unsigned long long b,
                                                       unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float lo_f(unsigned long long v) {
  return __uint_as_float(static_cast<uint32_t>(v));
}
__device__ __forceinline__ float hi_f(unsigned long long v) {
  return __uint_as_float(static_cast<uint32_t>(v >> 32));
}

}  // namespace

template <int RB, int NW, int NS>
constexpr size_t lp_smem_bytes() {
  return static_cast<size_t>(NS) * (NW * kLpColsPerWarp + RB) * kLpKS * 4 +
         NW * kLpColsPerWarp * 4;
}

// RB rows (even) x NW*64 columns per CTA tile, NS-stage cp.async ring.
template <int RB, int NW, int NS>
__global__ void __launch_bounds__(NW * 32, 12 / NW) k_logits_lp(LogitsArgs a) {
  static_assert(RB % 2 == 0 && RB <= 12, "RB even, <= 12");
  constexpr int NT = NW * 32;
  constexpr int CT = NW * kLpColsPerWarp;
  constexpr int STAGE = (CT + RB) * kLpKS;
  constexpr int kPieces = kLpKC / 4;           // 16-byte pieces per staged row
  constexpr int HALF = RB / 2;
  extern __shared__ __align__(16) float sm[];
  uint32_t* sid = reinterpret_cast<uint32_t*>(sm + NS * STAGE);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = lane & 1, cl = lane >> 1;
  const int cbase = warp * kLpColsPerWarp + cl;   // + 16 j
  const int d = a.d;
  const int d4 = d & ~3;
  const int nchunks = (d + kLpKC - 1) / kLpKC;
  const unsigned long long negz = a.x2_negzero, one = a.x2_one;

  pdl_wait();
  const bool shared_job = static_cast<int>(blockIdx.x) < a.jobs_shared;
  int row0, rowlim, tile_first, tile_step, s = 0;
  uint32_t m = 0;
  if (shared_job) {
    const int rg = blockIdx.x / a.ctiles_shared;
    row0 = rg * RB;
    rowlim = a.R_total;
    tile_first = blockIdx.x % a.ctiles_shared;
    tile_step = a.ctiles_shared;
    m = a.n_shared;
  } else {
    const int e = blockIdx.x - a.jobs_shared;
    s = e / (a.G * a.X);
    const int g = (e / a.X) % a.G;
    row0 = s * a.Bsent + g * RB;
    rowlim = s * a.Bsent + a.Bsent;
    tile_first = e % a.X;
    tile_step = a.X;
    m = a.n_cand[s] > a.n_shared ? a.n_cand[s] - a.n_shared : 0u;
  }
  const uint32_t* list = shared_job ? nullptr : a.ids + static_cast<size_t>(s) * a.ncap + a.n_shared;
  const int ntiles = static_cast<int>((m + CT - 1) / CT);

  for (int tile = tile_first; tile < ntiles; tile += tile_step) {
    const uint32_t t0 = static_cast<uint32_t>(tile) * CT;
    const int ncols = static_cast<int>(min(static_cast<uint32_t>(CT), m - t0));
    const uint32_t col0 = (shared_job ? 0u : a.n_shared) + t0;
    __syncthreads();  // the previous tile's readers are done with sid / stages
    for (int c = tid; c < CT; c += NT)
      sid[c] = c < ncols ? (list ? __ldg(list + t0 + c) : t0 + c) * static_cast<uint32_t>(d)
                         : 0x80000000u;
    __syncthreads();
    const int part = tid % kPieces;
    const int hrow = tid / kPieces;
    const uint32_t hoff = (hrow < RB && row0 + hrow < rowlim)
                              ? static_cast<uint32_t>(row0 + hrow) * d + part * 4
                              : 0x80000000u;
    auto load_chunk = [&](int stage, int kc) {
      float* Es = sm + stage * STAGE;
      float* Hs = Es + CT * kLpKS;
      const int c0 = kc * kLpKC;
      const bool kin = c0 + part * 4 < d;
#pragma unroll
      for (int i = 0; i < CT * kPieces / NT; ++i) {
        const int col = tid / kPieces + (NT / kPieces) * i;
        const uint32_t off = sid[col];
        const bool ok = kin && !(off & 0x80000000u);
        lp_cp_async16(Es + col * kLpKS + part * 4, a.E + (ok ? off + part * 4 + c0 : 0),
                      ok ? 16 : 0);
      }
      if (hrow < RB) {
        const bool ok = kin && !(hoff & 0x80000000u);
        lp_cp_async16(Hs + hrow * kLpKS + part * 4, a.H + (ok ? hoff + c0 : 0), ok ? 16 : 0);
      }
    };

    unsigned long long acc[RB][4];
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[r][j] = 0ull;

#pragma unroll
    for (int st = 0; st < NS - 1; ++st) {
      if (st < nchunks) load_chunk(st, st);
      lp_commit();
    }
    const bool warp_live = warp * kLpColsPerWarp < ncols;
    for (int kc = 0; kc < nchunks; ++kc) {
      lp_wait<NS - 2>();
      __syncthreads();
      {
        const int nk = kc + NS - 1;
        if (nk < nchunks) load_chunk(nk % NS, nk);
        lp_commit();
      }
      const float* Es = sm + (kc % NS) * STAGE;
      const float* Hs = Es + CT * kLpKS;
      const int kv = max(0, min(kLpKC, d4 - kc * kLpKC)) >> 2;  // full 4-lane groups
      if (warp_live) {
        auto quad = [&](int q) {
          unsigned long long e[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            e[j] = *reinterpret_cast<const unsigned long long*>(Es + (cbase + 16 * j) * kLpKS +
                                                                4 * q + 2 * p);
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            const unsigned long long h =
                *reinterpret_cast<const unsigned long long*>(Hs + r * kLpKS + 4 * q + 2 * p);
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[r][j] = lp_f2fma(acc[r][j], one, lp_f2fma(h, e[j], negz));
          }
        };
        if (kv == kLpKC / 4) {
#pragma unroll
          for (int q = 0; q < kLpKC / 4; ++q) quad(q);
        } else {
          for (int q = 0; q < kv; ++q) quad(q);
        }
      }
    }
    lp_wait<0>();
    pdl_trigger();
    // the d mod 4 tail (all of d when d < 4) sits in the last chunk: lane 0,
    // i.e. the low half of lane pair 0
    if (d4 < d && warp_live && p == 0) {
      const int cbeg = (nchunks - 1) * kLpKC;
      const float* Es = sm + ((nchunks - 1) % NS) * STAGE;
      const float* Hs = Es + CT * kLpKS;
      for (int k = d4; k < d; ++k) {
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const float h = Hs[r * kLpKS + k - cbeg];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float e = Es[(cbase + 16 * j) * kLpKS + k - cbeg];
            const float l0 = __fadd_rn(__fmul_rn(h, e), lo_f(acc[r][j]));
            acc[r][j] = (acc[r][j] & 0xFFFFFFFF00000000ull) | __float_as_uint(l0);
          }
        }
      }
    }
    // epilogue: thread p = 0 finishes rows [0, RB/2), p = 1 rows [RB/2, RB);
    // each receives the other lane pair of its outputs from its neighbour
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = cbase + 16 * j;
      const bool col_ok = c < ncols;
      const uint32_t wid = col_ok ? sid[c] / static_cast<uint32_t>(d) : 0u;
      const float bias = (a.bias && col_ok) ? __ldg(a.bias + wid) : 0.0f;
      const size_t col = col0 + c;
#pragma unroll
      for (int rl = 0; rl < HALF; ++rl) {
        const unsigned long long a0 = acc[rl][j], a1 = acc[rl + HALF][j];
        const unsigned long long send = p ? a0 : a1;
        const unsigned long long mine = p ? a1 : a0;
        const unsigned long long recv = __shfl_xor_sync(0xffffffffu, send, 1);
        const unsigned long long l01 = p ? recv : mine;  // reference lanes 0, 1
        const unsigned long long l23 = p ? mine : recv;  // reference lanes 2, 3
        float v = __fadd_rn(0.0f, lo_f(l01));
        v = __fadd_rn(v, hi_f(l01));
        v = __fadd_rn(v, lo_f(l23));
        v = __fadd_rn(v, hi_f(l23));
        if (a.bias) v = __fadd_rn(v, bias);
        const int r = row0 + rl + (p ? HALF : 0);
        if (col_ok && r < rowlim && warp_live) a.out[static_cast<size_t>(r) * a.ldo + col] = v;
      }
    }
  }
}

static const int kLpMinSurvivorCtas =
    getenv("LSB_K4_MIN_SURV") ? atoi(getenv("LSB_K4_MIN_SURV")) : 4;

template <int RB, int NW, int NS>
static lsb_status launch_lp(lsb_ctx* ctx, LogitsArgs a, int target) {
  constexpr int CT = NW * kLpColsPerWarp;
  const int rgroups = (a.R_total + RB - 1) / RB;
  a.ctiles_shared = static_cast<int>((a.n_shared + CT - 1) / CT);
  a.jobs_shared = (a.n_shared && !a.skip_shared) ? rgroups * a.ctiles_shared : 0;
  a.G = (a.Bsent + RB - 1) / RB;
  if (a.ids && a.S > 0) {
    const size_t max_tiles = (a.ncap > a.n_shared ? a.ncap - a.n_shared : 0) / CT + 1;
    const int want =
        std::max(kLpMinSurvivorCtas, (target - a.jobs_shared) / std::max(1, a.S * a.G));
    a.X = static_cast<int>(std::min<size_t>({static_cast<size_t>(want), size_t(512), max_tiles}));
  } else {
    a.X = 0;
  }
  const int grid = a.jobs_shared + a.S * a.G * a.X;
  if (grid == 0) return LSB_OK;
  constexpr size_t smem = lp_smem_bytes<RB, NW, NS>();
  auto* kern = k_logits_lp<RB, NW, NS>;
  if (lsb_status rc = ensure_smem(ctx, kern, smem)) return rc;
  LSB_CUDA(launch_pdl(ctx, kern, dim3(grid), dim3(NW * 32), smem, a));
  LSB_LAUNCHED(ctx, "k_logits_lp");
  return LSB_OK;
}

// True when the lane-pair kernel takes this PARITY launch (16-byte aligned
// rows); it then also picks its row-group size.
bool logits_lp_applies(const LogitsArgs& a) {
  static const bool off = getenv("LSB_K4_LP_OFF") != nullptr;
  return !off && (a.d & 3) == 0 && (reinterpret_cast<uintptr_t>(a.E) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(a.H) & 15) == 0;
}

// Row-group size for B rows per sentence: the even RB <= 12 with the fewest
// padded rows, ties to the larger tile.
static int lp_choose_rb(int B) {
  int best = 12, best_rows = 1 << 30;
  for (int rb : {12, 10, 8, 6, 4, 2}) {
    const int rows = ((B + rb - 1) / rb) * rb;
    if (rows < best_rows) {
      best_rows = rows;
      best = rb;
    }
  }
  return best;
}

lsb_status launch_logits_lp(lsb_ctx* ctx, const LogitsArgs& a, int target_ctas) {
  switch (lp_choose_rb(a.Bsent)) {
    case 12: return launch_lp<12, 4, 3>(ctx, a, target_ctas);
    case 10: return launch_lp<10, 4, 3>(ctx, a, target_ctas);
    case 8: return launch_lp<8, 4, 3>(ctx, a, target_ctas);
    case 6: return launch_lp<6, 4, 3>(ctx, a, target_ctas);
    case 4: return launch_lp<4, 4, 3>(ctx, a, target_ctas);
    default: return launch_lp<2, 4, 3>(ctx, a, target_ctas);
  }
}

}  // namespace lsb
