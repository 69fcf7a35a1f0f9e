// k_logits_ln.cu -- K4 PARITY, one reference accumulation lane per thread.
//
// Same job and the same bits as k_logits (logits = H . E[ids]^T + bias[ids],
// gathered E rows, shared top-T block + per-sentence survivors;
// src/candidate_selector.cpp:105-119, src/beam_decoder.cpp:23-44, :237-247):
// lane j of an output sums fl(h[c] * e[c]) for c = j mod 4 in ascending c and
// the result is ((0 + l0) + l1 + l2) + l3 + bias. This kernel takes d % 4 == 0
// (no tail lane), which is every BASELINE shape.
//
// Why: FFMA2 issues at 2 cycles per SMSP (128 FP32 lane-ops / SM / clock,
// scripts/micro/fp32x2_tput.cu measured 121 on B200), so PARITY's
// FMUL + FADD per MAC is FP32-bound only if shared memory delivers the
// operands at <= 0.5 wavefronts per FFMA2 per warp. k_logits' 4-lanes-per-
// thread 3 x 4 tile needs 28 wavefronts per 48 FFMA2 (0.58, LSU-bound). Here
// a thread owns ONE lane j of RT rows x 4 columns: per lane element it loads
// RT/2 row pairs {h_r, h_r+1} (8-byte loads from a pair-interleaved H stage)
// and 4 scalar E values, and issues RT/2 x 4 mul + RT/2 x 4 add FFMA2 with the
// E scalar as FFMA2's broadcast (.F32) operand -- RT + 4 wavefronts (+ the
// cp.async writes) per 4 RT FFMA2: 0.42 at RT = 12 with 48 accumulator
// registers (the lane-pair variant needed 96 and lost occupancy).
//
// Warp: lane = 4 cg + j (cg = column group 0..7, j = reference lane), columns
// cg + 8 i (i = 0..3) of the warp's 32. The four lanes of an output meet in
// the epilogue through three xor shuffles; thread j finishes column 8 j + cg
// for all RT rows, so each row's 32 outputs leave as one 128-byte store.
//
// CTA = NW warps. Shared-block jobs (identity columns, scored once for all
// S*B rows) arrange them WRS rows x NW/WRS columns of warp tiles, so an E chunk
// in shared memory serves WRS * RT rows; survivor jobs (one sentence's RT
// rows) put all NW warps side by side.
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

constexpr int kLnKC = 32;          // d floats per staged chunk
constexpr int kLnKS = kLnKC + 4;   // E row pitch: 36 = 4 mod 32 banks

__device__ __forceinline__ void ln_cp16(void* dst, const void* src, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void ln_cp4(void* dst, const void* src, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void ln_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void ln_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ unsigned long long ln_f2fma(unsigned long long a, unsigned long long b,
                                                       unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
// {x, x}: ptxas folds it into FFMA2's scalar-broadcast operand (no MOV)
__device__ __forceinline__ unsigned long long ln_dup(float x) {
  unsigned long long d;
  asm("mov.b64 %0, {%1, %1};" : "=l"(d) : "f"(x));
  return d;
}
__device__ __forceinline__ float ln_sel4(const float (&v)[4], int k) {
  return k == 0 ? v[0] : k == 1 ? v[1] : k == 2 ? v[2] : v[3];
}

}  // namespace

template <int RT, int NW, int WRS, int NS>
constexpr size_t ln_smem_bytes() {
  return static_cast<size_t>(NS) * (NW * 32 * kLnKS + WRS * RT * kLnKC) * 4 + NW * 32 * 8;
}

// H stage layout: rows in quads {h_4a, h_4a+1, h_4a+2, h_4a+3}[k] (one 16-byte
// load feeds two FFMA2 row pairs); an RT % 4 == 2 tile ends in a row pair.
__device__ __forceinline__ int ln_hslot(int r, int k, int RT) {
  const int w = r / RT, rr = r % RT;  // warp-row block, row within it
  const int q4 = (RT / 4) * 4;
  // floats per warp-row block: RT * KC; quads first, then the trailing pair
  const int base = w * RT * kLnKC;
  return rr < q4 ? base + (rr >> 2) * 4 * kLnKC + k * 4 + (rr & 3)
                 : base + q4 * kLnKC + k * 2 + (rr & 1);
}

// One job's column tiles with a compile-time CTA shape: WR x WC warp tiles of
// RT rows x 32 columns (RTT = WR RT rows, CTT = 32 WC columns per CTA tile).
// Staging: thread tid copies E pieces (column tid/8 + NT/8 i, floats 4 (tid%8)..)
// and H elements (row tid/32 + 4 i, float tid%32) of every chunk. Columns past
// the tile end and rows past the row limit copy a valid column / row instead
// (their outputs are never stored and every output is independent), so the
// only predicate is the d tail of the last chunk.
template <int RT, int WR, int WC, int NS, int STAGE_E, int STAGE>
__device__ __forceinline__ void ln_job(const LogitsArgs& a, float* sm, uint32_t* soff,
                                       uint32_t* swid, int row0, int rowlim, int tile_first,
                                       int tile_step, uint32_t m, const uint32_t* list,
                                       uint32_t colbase) {
  constexpr int NT = WR * WC * 32;
  constexpr int RTT = WR * RT, CTT = WC * 32;
  constexpr int NQ = RT / 4;        // row quads per thread
  constexpr int NP = (RT % 4) / 2;  // + a trailing row pair
  constexpr int NPE = CTT * (kLnKC / 4) / NT;  // E pieces per thread per chunk
  constexpr int ECS = NT / (kLnKC / 4);        // columns covered per pass
  constexpr int HRS = NT / kLnKC;              // H rows covered per pass
  constexpr int NPH = (RTT + HRS - 1) / HRS;   // H elements per thread per chunk
  static_assert(NPE * NT == CTT * (kLnKC / 4), "whole pieces");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = lane & 3, cg = lane >> 2;
  const int wr = warp % WR, wc = warp / WR;
  const int d = a.d;
  const int nchunks = (d + kLnKC - 1) / kLnKC;
  const unsigned long long negz = a.x2_negzero, one = a.x2_one;
  const int ntiles = static_cast<int>((m + CTT - 1) / CTT);
  const int wcol = wc * 32;
  const int epart = tid & 7, ecol0 = tid >> 3;
  // H: with 128 threads a warp writes rows 4 i + (lane & 3) x 8 consecutive k
  // -> 32 consecutive floats of the quad layout (conflict-free)
  const int hk = tid / HRS, hr0 = tid % HRS;
  // H sources (rows clamped into [row0, rowlim)) and smem slots: fixed per job
  // (32-bit element offsets: the chunk's base pointer is uniform)
  uint32_t hsrc[NPH];
  int hdst[NPH];
#pragma unroll
  for (int i = 0; i < NPH; ++i) {
    const int r = hr0 + HRS * i;
    hsrc[i] = static_cast<uint32_t>(min(row0 + r, rowlim - 1)) * d + hk;
    hdst[i] = r < RTT ? ln_hslot(r, hk, RT) : -1;
  }

  for (int tile = tile_first; tile < ntiles; tile += tile_step) {
    const uint32_t t0 = static_cast<uint32_t>(tile) * CTT;
    const int ncols = static_cast<int>(min(static_cast<uint32_t>(CTT), m - t0));
    __syncthreads();  // the previous tile's readers are done with soff / stages
    for (int c = tid; c < CTT; c += NT) {
      const int cc = min(c, ncols - 1);  // past the end: a copy of the last column
      const uint32_t w = list ? __ldg(list + t0 + cc) : t0 + cc;
      swid[c] = w;
      soff[c] = w * static_cast<uint32_t>(d);  // element offset of the row
    }
    __syncthreads();
    // wide tiles re-read their piece offsets from shared memory (registers)
    constexpr bool EREG = NPE <= 4;
    uint32_t esrc[EREG ? NPE : 1];
    if constexpr (EREG) {
#pragma unroll
      for (int i = 0; i < NPE; ++i) esrc[i] = soff[ecol0 + ECS * i] + epart * 4;
    }
    auto eoff = [&](int i) -> uint32_t {
      if constexpr (EREG) return esrc[i];
      else return soff[ecol0 + ECS * i] + epart * 4;
    };

    auto load_chunk = [&](int stage, int kc) {
      float* Es = sm + stage * STAGE + ecol0 * kLnKS + epart * 4;
      float* Hs = sm + stage * STAGE + STAGE_E;
      const int c0 = kc * kLnKC;
      const float* Ec = a.E + c0;
      const float* Hc = a.H + c0;
      if (c0 + kLnKC <= d) {
#pragma unroll
        for (int i = 0; i < NPE; ++i) ln_cp16(Es + ECS * i * kLnKS, Ec + eoff(i), 16);
#pragma unroll
        for (int i = 0; i < NPH; ++i)
          if (NPH * HRS == RTT || hdst[i] >= 0) ln_cp4(Hs + hdst[i], Hc + hsrc[i], 4);
      } else {  // the d tail (d % 4 == 0: a piece is all in or out)
        const bool ein = c0 + epart * 4 < d, hin = c0 + hk < d;
#pragma unroll
        for (int i = 0; i < NPE; ++i)
          ln_cp16(Es + ECS * i * kLnKS, ein ? Ec + eoff(i) : a.E, ein ? 16 : 0);
#pragma unroll
        for (int i = 0; i < NPH; ++i)
          if (NPH * HRS == RTT || hdst[i] >= 0)
            ln_cp4(Hs + hdst[i], hin ? Hc + hsrc[i] : a.H, hin ? 4 : 0);
      }
    };

    unsigned long long acc[RT / 2][4];
#pragma unroll
    for (int hp = 0; hp < RT / 2; ++hp)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[hp][i] = 0ull;

#pragma unroll
    for (int st = 0; st < NS - 1; ++st) {
      if (st < nchunks) load_chunk(st, st);
      ln_commit();
    }
    const bool warp_live = wcol < ncols;
    for (int kc = 0; kc < nchunks; ++kc) {
      ln_wait<NS - 2>();
      __syncthreads();
      {
        const int nk = kc + NS - 1;
        if (nk < nchunks) load_chunk(nk % NS, nk);
        ln_commit();
      }
      const float* Es = sm + (kc % NS) * STAGE;
      const float* Hs = Es + STAGE_E + wr * RT * kLnKC + 4 * j;
      const float* Ecol = Es + (wcol + cg) * kLnKS + j;
      const int nq = min(kLnKC, d - kc * kLnKC) >> 2;
      if (warp_live) {
        auto step = [&](int q) {
          float e[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) e[i] = Ecol[i * 8 * kLnKS + 4 * q];
#pragma unroll
          for (int hq = 0; hq < NQ; ++hq) {
            const ulonglong2 h4 =
                *reinterpret_cast<const ulonglong2*>(Hs + (hq * kLnKC + 4 * q) * 4);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              acc[2 * hq][i] = ln_f2fma(acc[2 * hq][i], one, ln_f2fma(h4.x, ln_dup(e[i]), negz));
              acc[2 * hq + 1][i] =
                  ln_f2fma(acc[2 * hq + 1][i], one, ln_f2fma(h4.y, ln_dup(e[i]), negz));
            }
          }
          if constexpr (NP) {
            const unsigned long long h2 = *reinterpret_cast<const unsigned long long*>(
                Hs + NQ * 4 * kLnKC + (4 * q) * 2 - 2 * j);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              acc[2 * NQ][i] = ln_f2fma(acc[2 * NQ][i], one, ln_f2fma(h2, ln_dup(e[i]), negz));
          }
        };
        if (nq == kLnKC / 4) {
#pragma unroll
          for (int q = 0; q < kLnKC / 4; ++q) step(q);
        } else {
          for (int q = 0; q < nq; ++q) step(q);
        }
      }
    }
    ln_wait<0>();
    pdl_trigger();
    // epilogue: thread j collects the four lanes of column 8 j + cg
    const int cme = wcol + cg + 8 * j;  // tile column this thread finishes
    const bool col_ok = warp_live && cme < ncols;
    const float bias = (a.bias && col_ok) ? __ldg(a.bias + swid[cme]) : 0.0f;
    const size_t ocol = colbase + t0 + cme;
#pragma unroll
    for (int hp = 0; hp < RT / 2; ++hp) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float mine[4];  // my lane j for the 4 columns i
#pragma unroll
        for (int i = 0; i < 4; ++i)
          mine[i] = __uint_as_float(static_cast<uint32_t>(acc[hp][i] >> (32 * half)));
        float got[4];  // got[k] = lane (j ^ k) of my column
        got[0] = ln_sel4(mine, j);
#pragma unroll
        for (int k = 1; k < 4; ++k)
          got[k] = __shfl_xor_sync(0xffffffffu, ln_sel4(mine, j ^ k), k);
        float v = 0.0f;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) v = __fadd_rn(v, ln_sel4(got, jj ^ j));
        if (a.bias) v = __fadd_rn(v, bias);
        const int r = row0 + wr * RT + 2 * hp + half;
        if (col_ok && r < rowlim) a.out[static_cast<size_t>(r) * a.ldo + ocol] = v;
      }
    }
  }
}

template <int RT, int NW, int WRS, int NS>
__global__ void __launch_bounds__(NW * 32, (RT == 12 ? 16 : 20) / NW) k_logits_ln(LogitsArgs a) {
  static_assert(RT % 2 == 0 && RT <= 12, "RT even, <= 12");
  static_assert(NW % WRS == 0, "whole warp columns");
  constexpr int CTMAX = NW * 32;
  constexpr int RTMAX = WRS * RT;
  constexpr int STAGE_E = CTMAX * kLnKS;
  constexpr int STAGE = STAGE_E + RTMAX * kLnKC;
  extern __shared__ __align__(16) float sm[];
  uint32_t* soff = reinterpret_cast<uint32_t*>(sm + NS * STAGE);  // element offset id*d
  uint32_t* swid = soff + CTMAX;                                    // word id

  pdl_wait();
  const int bid = blockIdx.x;
  if (bid < a.jobs_shared) {
    // shared block: identity columns [0, n_shared) for all S*B rows
    // column-tile-major order: the row groups that share one E tile run
    // back to back, so a block larger than L2 (the full vocabulary: 160 MB)
    // streams from HBM once instead of once per row group (5.0 GB at S=64)
    const int rgroups = a.jobs_shared / a.ctiles_shared;
    const int rg = bid % rgroups;
    ln_job<RT, WRS, NW / WRS, NS, STAGE_E, STAGE>(a, sm, soff, swid, rg * RTMAX, a.R_total,
                                                  bid / rgroups, a.ctiles_shared, a.n_shared,
                                                  nullptr, 0u);
  } else {
    // survivors: one sentence's RT rows over its candidates past n_shared
    const int e = bid - a.jobs_shared;
    const int s = e / (a.G * a.X);
    const int g = (e / a.X) % a.G;
    const uint32_t n = a.n_cand[s];
    ln_job<RT, 1, NW, NS, STAGE_E, STAGE>(
        a, sm, soff, swid, s * a.Bsent + g * RT, s * a.Bsent + a.Bsent, e % a.X, a.X,
        n > a.n_shared ? n - a.n_shared : 0u, a.ids + static_cast<size_t>(s) * a.ncap + a.n_shared,
        a.n_shared);
  }
}

static const int kLnMinSurvivorCtas =
    getenv("LSB_K4_MIN_SURV") ? atoi(getenv("LSB_K4_MIN_SURV")) : 4;

template <int RT, int NW, int WRS, int NS>
static lsb_status launch_ln(lsb_ctx* ctx, LogitsArgs a, int target) {
  constexpr int RTS = WRS * RT, CTS = (NW / WRS) * 32, CTV = NW * 32;
  a.ctiles_shared = static_cast<int>((a.n_shared + CTS - 1) / CTS);
  a.jobs_shared =
      (a.n_shared && !a.skip_shared) ? ((a.R_total + RTS - 1) / RTS) * a.ctiles_shared : 0;
  a.G = (a.Bsent + RT - 1) / RT;
  if (a.ids && a.S > 0) {
    const size_t max_tiles = (a.ncap > a.n_shared ? a.ncap - a.n_shared : 0) / CTV + 1;
    const int want =
        std::max(kLnMinSurvivorCtas, (target - a.jobs_shared) / std::max(1, a.S * a.G));
    a.X = static_cast<int>(std::min<size_t>({static_cast<size_t>(want), size_t(512), max_tiles}));
  } else {
    a.X = 0;
  }
  const int grid = a.jobs_shared + a.S * a.G * a.X;
  if (grid == 0) return LSB_OK;
  constexpr size_t smem = ln_smem_bytes<RT, NW, WRS, NS>();
  auto* kern = k_logits_ln<RT, NW, WRS, NS>;
  if (lsb_status rc = ensure_smem(ctx, kern, smem)) return rc;
  LSB_CUDA(launch_pdl(ctx, kern, dim3(grid), dim3(NW * 32), smem, a));
  LSB_LAUNCHED(ctx, "k_logits_ln");
  return LSB_OK;
}

bool logits_ln_applies(const LogitsArgs& a) {
  return (a.d & 3) == 0 && (reinterpret_cast<uintptr_t>(a.E) & 15) == 0;
}

// Rows per thread for B rows per sentence: the even RT <= 12 with the fewest
// padded rows, ties to the larger tile.
static int ln_choose_rt(int B) {
  int best = 12, best_rows = 1 << 30;
  for (int rt : {12, 10, 8, 6, 4, 2}) {
    const int rows = ((B + rt - 1) / rt) * rt;
    if (rows < best_rows) {
      best_rows = rows;
      best = rt;
    }
  }
  return best;
}

template <int RT>
static lsb_status launch_ln_rt(lsb_ctx* ctx, const LogitsArgs& a, int target) {
  static const int wrs_env = getenv("LSB_K4_LN_WRS") ? atoi(getenv("LSB_K4_LN_WRS")) : 0;
  // rows sharing the identity block: stack two warp rows once there are more
  // rows than one warp tile holds (E chunk reused by 2 RT rows)
  const int wrs = wrs_env ? wrs_env : (a.R_total > RT ? 2 : 1);
  // (one row group over a long identity block -- a one-sentence full-
  // vocabulary step -- in 64-column CTAs with a 4-deep ring measured 70.7 us
  // vs 67.6 for k_logits' 128-column tiles: FP-latency, not bytes in flight)
  return wrs >= 2 ? launch_ln<RT, 4, 2, 2>(ctx, a, target) : launch_ln<RT, 4, 1, 2>(ctx, a, target);
}

lsb_status launch_logits_ln(lsb_ctx* ctx, const LogitsArgs& a, int target_ctas) {
  switch (ln_choose_rt(a.Bsent)) {
    case 12: return launch_ln_rt<12>(ctx, a, target_ctas);
    case 10: return launch_ln_rt<10>(ctx, a, target_ctas);
    case 8: return launch_ln_rt<8>(ctx, a, target_ctas);
    case 6: return launch_ln_rt<6>(ctx, a, target_ctas);
    case 4: return launch_ln_rt<4>(ctx, a, target_ctas);
    default: return launch_ln_rt<2>(ctx, a, target_ctas);
  }
}

}  // namespace lsb
