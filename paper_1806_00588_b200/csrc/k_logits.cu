// k_logits.cu -- K4: logits = H . E[ids]^T + bias[ids] over the candidate set.
//
// Replaces gather_embeddings + compute_logits + the bias loop of decode()
// (src/candidate_selector.cpp:105-119, src/beam_decoder.cpp:23-44, :237-247).
// E_LSH is never materialised: each CTA owns RB hypothesis rows x 128*CB
// candidate columns and streams the candidates' embedding rows straight from
// E (row gather by id) into shared memory with cp.async, d in chunks of 32
// floats through a 2-stage ring (5 CTAs per SM), so the inner loop reads only shared memory:
// the H row chunk as a warp-wide broadcast and each thread's own E row with
// conflict-free 16-byte loads (row pitch 36 floats = 4 mod 32 banks).
//
// Jobs (one CTA each):
//  * shared block: candidate positions [0, n_shared) are ids 0..T-1 for every
//    sentence (the top-T prefix, src/candidate_selector.cpp:57-103), so they
//    are scored once for all S*B rows in groups of RB rows;
//  * survivors: per (sentence, row group), X CTAs stride over that
//    sentence's remaining candidate positions [n_shared, n_cand[s]).
//
// PARITY keeps four lane accumulators per output and adds fl(h*e) with
// separate FMUL/FADD in the reference's SSE order (lane j takes columns
// c = j mod 4 ascending; the d mod 4 tail goes to lane 0; final
// ((l0+l1)+l2)+l3), which GCC -O3 emits for the omp-simd reduction at
// src/beam_decoder.cpp:34-42 -> bit-identical logits. FAST uses one FFMA
// chain per output.
#include <algorithm>
#include <cstdlib>

#include "k_step.cuh"

namespace lsb {

constexpr int kLT = 128;        // threads per CTA
// d is staged in chunks of KC floats (32, or 16 for 2-column tiles); the
// shared-memory row pitch KC + 4 floats is 4 mod 32 words for KC = 32 and
// 20 for KC = 16 -- both conflict-free for 16-byte loads by 8-thread phases.

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// columns per CTA tile: CB per thread, one per thread-column (1-D: 128
// threads) or 8 per warp (2-D: 4 warps)
template <int CB, bool TWO_D>
constexpr int tile_cols() {
  return TWO_D ? 32 * CB : kLT * CB;
}

template <int RB, int CB, int NS, int KC, bool TWO_D = false>
constexpr size_t logits_smem_bytes() {
  constexpr int CT = tile_cols<CB, TWO_D>();
  return static_cast<size_t>(NS) * (CT + RB) * (KC + 4) * 4 + CT * 4;
}

// One 4-wide step of d for RB rows x CB columns: float4 of H (smem
// broadcast) times float4 of each column's E row.
template <int RB, int CB, bool PARITY, int KS>
__device__ __forceinline__ void mac4(float (&acc)[RB][CB][PARITY ? 4 : 1], const float* Es,
                                     const float* Hs, int rbase, int cbase, int cstride, int k4) {
  float4 e[CB];
#pragma unroll
  for (int cb = 0; cb < CB; ++cb)
    e[cb] = *reinterpret_cast<const float4*>(Es + (cbase + cb * cstride) * KS + k4 * 4);
#pragma unroll
  for (int rb = 0; rb < RB; ++rb) {
    const float4 h = *reinterpret_cast<const float4*>(Hs + (rbase + rb) * KS + k4 * 4);
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      if constexpr (PARITY) {
        acc[rb][cb][0] = __fadd_rn(acc[rb][cb][0], __fmul_rn(h.x, e[cb].x));
        acc[rb][cb][1] = __fadd_rn(acc[rb][cb][1], __fmul_rn(h.y, e[cb].y));
        acc[rb][cb][2] = __fadd_rn(acc[rb][cb][2], __fmul_rn(h.z, e[cb].z));
        acc[rb][cb][3] = __fadd_rn(acc[rb][cb][3], __fmul_rn(h.w, e[cb].w));
      } else {
        float x = acc[rb][cb][0];
        x = fmaf(h.x, e[cb].x, x);
        x = fmaf(h.y, e[cb].y, x);
        x = fmaf(h.z, e[cb].z, x);
        x = fmaf(h.w, e[cb].w, x);
        acc[rb][cb][0] = x;
      }
    }
  }
}

// PARITY with Blackwell's paired FP32 pipe (FFMA2 on f32x2 register pairs):
// lanes (0,1) and (2,3) of the reference's 4-lane accumulation advance
// together. Exactness: fma(h, e, -0) == fl(h*e) and fma(acc, 1, p) ==
// fl(acc + p) (a single rounding each, the same signed zeros), so the pair
// ops reproduce FMUL/FADD bit for bit. The -0 / 1.0 operands come from
// kernel arguments: were they compile-time constants, ptxas would turn the
// pair back into mul + add and contract it into one FFMA2, which rounds once
// instead of twice.
__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// FAST with paired FP32: each output keeps two partial FFMA chains (even /
// odd d) in one f32x2 register pair, one FFMA2 per two MACs; summed in the
// epilogue (FAST's tolerance, not the reference order).
template <int RB, int CB, int KS>
__device__ __forceinline__ void mac4_f2(unsigned long long (&acc)[RB][CB], const float* Es,
                                        const float* Hs, int rbase, int cbase, int cstride,
                                        int k4) {
  ulonglong2 e[CB];
#pragma unroll
  for (int cb = 0; cb < CB; ++cb)
    e[cb] = *reinterpret_cast<const ulonglong2*>(Es + (cbase + cb * cstride) * KS + k4 * 4);
#pragma unroll
  for (int rb = 0; rb < RB; ++rb) {
    const ulonglong2 h = *reinterpret_cast<const ulonglong2*>(Hs + (rbase + rb) * KS + k4 * 4);
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      acc[rb][cb] = f2fma(h.x, e[cb].x, acc[rb][cb]);
      acc[rb][cb] = f2fma(h.y, e[cb].y, acc[rb][cb]);
    }
  }
}

template <int RB, int CB, int KS>
__device__ __forceinline__ void mac4_x2(unsigned long long (&acc)[RB][CB][2], const float* Es,
                                        const float* Hs, int rbase, int cbase, int cstride, int k4,
                                        unsigned long long negz, unsigned long long one) {
  ulonglong2 e[CB];
#pragma unroll
  for (int cb = 0; cb < CB; ++cb)
    e[cb] = *reinterpret_cast<const ulonglong2*>(Es + (cbase + cb * cstride) * KS + k4 * 4);
#pragma unroll
  for (int rb = 0; rb < RB; ++rb) {
    const ulonglong2 h = *reinterpret_cast<const ulonglong2*>(Hs + (rbase + rb) * KS + k4 * 4);
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      acc[rb][cb][0] = f2fma(acc[rb][cb][0], one, f2fma(h.x, e[cb].x, negz));
      acc[rb][cb][1] = f2fma(acc[rb][cb][1], one, f2fma(h.y, e[cb].y, negz));
    }
  }
}

// TWO_D: a warp owns all RB rows x 8 TC columns as a 4 x 8 lane grid, each
// lane RB/4 rows x TC columns (stride 8): its H loads are shared by the 8
// lanes of a row group and its E loads by the 4 of a column group, so one
// 16-byte LDS is a single wavefront (vs 4 for 32 distinct E rows) and a
// thread issues RB/4 + TC loads per 4-step instead of RB + 1.
// One K4 job (a shared-block tile or a sentence row group's survivor tiles)
// by a 128-thread CTA; `bid` is the job index. k_logits runs a CTA per job;
// the fused small-batch step (k_step_fused.cu) loops its persistent CTAs over
// the jobs.
// Survivor ids: read-only for k_logits; written by K3 in the same launch in
// the fused step (k_step_fused.cu), which must not use the read-only path.
#ifdef LSB_BODIES_ONLY
#define LSB_LD_IDS(p) __ldcg(p)
#else
#define LSB_LD_IDS(p) __ldg(p)
#endif
template <int RB, int CB, bool PARITY, bool VEC, int kStages, int KC, bool TWO_D = false>
__device__ __forceinline__ void logits_job(const LogitsArgs& a, int bid, float* sm) {
  constexpr int kKC = KC;
  constexpr int kKS = KC + 4;
  constexpr int kParts = KC / 4;           // 16-byte pieces per row chunk
  constexpr int kRowStep = kLT / kParts;   // rows covered by one pass of the CTA
  constexpr int CT = tile_cols<CB, TWO_D>();
  constexpr int STAGE = (CT + RB) * kKS;
  constexpr int NA = PARITY ? 4 : 1;
  uint32_t* sid = reinterpret_cast<uint32_t*>(sm + kStages * STAGE);
  const int tid = threadIdx.x, warp = tid >> 5;
  static_assert(!TWO_D || RB % 4 == 0, "2-D tile: RB = 4 TR");
  static_assert(CT % (kLT / (KC / 4)) == 0, "whole 16-byte pieces per loader thread");
  constexpr int TR = TWO_D ? RB / 4 : RB;  // rows per thread
  constexpr int TC = CB;                   // columns per thread
  const int rbase = TWO_D ? ((tid & 31) >> 3) * TR : 0;
  const int cbase = TWO_D ? warp * (8 * TC) + (tid & 7) : tid;
  constexpr int cstride = TWO_D ? 8 : kLT;
  const int d = a.d;
  const int d4 = d & ~3;
  const int nchunks = (d + kKC - 1) / kKC;

  pdl_wait();  // (no-op unless launched as a PDL dependent)
  const bool shared_job = bid < a.jobs_shared;
  int row0, rowlim, tile_first, tile_step, s = 0;
  uint32_t m = 0;
  if (shared_job) {
    const int rg = bid / a.ctiles_shared;
    row0 = rg * RB;
    rowlim = a.R_total;
    tile_first = bid % a.ctiles_shared;
    tile_step = a.ctiles_shared;  // exactly one tile
    m = a.n_shared;
  } else {
    const int e = bid - a.jobs_shared;
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
    __syncthreads();  // previous tile's readers are done with sid / stages
    for (int c = tid; c < CT; c += kLT)
      sid[c] = c < ncols ? (list ? LSB_LD_IDS(list + t0 + c) : t0 + c) : 0u;
    __syncthreads();

    // per-tile source offsets (elements) of this thread's 16-byte pieces:
    // piece i covers column (tid >> 3) + 16 i, floats [4 (tid & 7), +4) of
    // every chunk; invalid columns / rows carry bit 31 and are zero-filled
    const int part = tid % kParts;
    // sid[] now holds each column's element offset sid*d (bit 31 = invalid),
    // re-read per chunk instead of pinning 8 registers per thread
    if constexpr (VEC) {
      __syncthreads();
      for (int c = tid; c < CT; c += kLT)
        sid[c] = c < ncols ? sid[c] * static_cast<uint32_t>(d) : 0x80000000u;
      __syncthreads();
    }
    const int hrow = tid / kParts;
    const uint32_t hoff = (tid < RB * kParts && row0 + hrow < rowlim)
                              ? static_cast<uint32_t>(row0 + hrow) * d + part * 4
                              : 0x80000000u;

    auto load_chunk = [&](int stage, int kc) {
      float* Es = sm + stage * STAGE;
      float* Hs = Es + CT * kKS;
      const int c0 = kc * kKC;
      if constexpr (VEC) {
        const bool kin = c0 + part * 4 < d;
#pragma unroll
        for (int i = 0; i < CT / kRowStep; ++i) {
          const int col = tid / kParts + kRowStep * i;
          const uint32_t off = sid[col];
          const bool ok = kin && !(off & 0x80000000u);
          cp_async16(Es + col * kKS + part * 4, a.E + (ok ? off + part * 4 + c0 : 0), ok ? 16 : 0);
        }
        if (tid < RB * kParts) {
          const bool ok = kin && !(hoff & 0x80000000u);
          cp_async16(Hs + hrow * kKS + part * 4, a.H + (ok ? hoff + c0 : 0), ok ? 16 : 0);
        }
      } else {
        for (int q = tid; q < CT * kKC; q += kLT) {
          const int col = q / kKC, kk = q % kKC;
          const bool ok = col < ncols && c0 + kk < d;
          const float* src = ok ? a.E + static_cast<size_t>(sid[col]) * d + c0 + kk : a.E;
          cp_async4(Es + col * kKS + kk, src, ok ? 4 : 0);
        }
        for (int q = tid; q < RB * kKC; q += kLT) {
          const int rb = q / kKC, kk = q % kKC;
          const bool ok = row0 + rb < rowlim && c0 + kk < d;
          const float* src = ok ? a.H + static_cast<size_t>(row0 + rb) * d + c0 + kk : a.H;
          cp_async4(Hs + rb * kKS + kk, src, ok ? 4 : 0);
        }
      }
    };

    float acc[TR][TC][NA];
#pragma unroll
    for (int rb = 0; rb < TR; ++rb)
#pragma unroll
      for (int cb = 0; cb < TC; ++cb)
#pragma unroll
        for (int k = 0; k < NA; ++k) acc[rb][cb][k] = 0.0f;
    constexpr bool X2 = PARITY && VEC;   // paired FP32 path (see mac4_x2)
    constexpr bool F2 = !PARITY && VEC;  // FAST paired path (see mac4_f2)
    unsigned long long acc2[X2 ? TR : 1][X2 ? TC : 1][2];
    unsigned long long accf[F2 ? TR : 1][F2 ? TC : 1];
    if constexpr (X2) {
#pragma unroll
      for (int rb = 0; rb < TR; ++rb)
#pragma unroll
        for (int cb = 0; cb < TC; ++cb) acc2[rb][cb][0] = acc2[rb][cb][1] = 0ull;
    }
    if constexpr (F2) {
#pragma unroll
      for (int rb = 0; rb < TR; ++rb)
#pragma unroll
        for (int cb = 0; cb < TC; ++cb) accf[rb][cb] = 0ull;
    }

#pragma unroll
    for (int st = 0; st < kStages - 1; ++st) {
      if (st < nchunks) load_chunk(st, st);
      cp_async_commit();
    }
    // a warp whose 32 columns are all past the tile end skips the math
    const bool warp_live = (TWO_D ? warp * 8 * TC : warp * 32) < ncols;
    for (int kc = 0; kc < nchunks; ++kc) {
      cp_async_wait<kStages - 2>();
      __syncthreads();
      {
        const int nk = kc + kStages - 1;
        if (nk < nchunks) load_chunk(nk % kStages, nk);
        cp_async_commit();
      }
      const float* Es = sm + (kc % kStages) * STAGE;
      const float* Hs = Es + CT * kKS;
      const int kv = max(0, min(kKC, d4 - kc * kKC)) >> 2;  // full 4-lane groups
      if (warp_live) {
        if constexpr (X2) {
          if (kv == kKC / 4) {
#pragma unroll
            for (int k4 = 0; k4 < kKC / 4; ++k4)
              mac4_x2<TR, TC, kKS>(acc2, Es, Hs, rbase, cbase, cstride, k4, a.x2_negzero,
                                   a.x2_one);
          } else {
            for (int k4 = 0; k4 < kv; ++k4)
              mac4_x2<TR, TC, kKS>(acc2, Es, Hs, rbase, cbase, cstride, k4, a.x2_negzero,
                                   a.x2_one);
          }
        } else if constexpr (F2) {
          if (kv == kKC / 4) {
#pragma unroll
            for (int k4 = 0; k4 < kKC / 4; ++k4)
              mac4_f2<TR, TC, kKS>(accf, Es, Hs, rbase, cbase, cstride, k4);
          } else {
            for (int k4 = 0; k4 < kv; ++k4)
              mac4_f2<TR, TC, kKS>(accf, Es, Hs, rbase, cbase, cstride, k4);
          }
        } else {
          if (kv == kKC / 4) {
#pragma unroll
            for (int k4 = 0; k4 < kKC / 4; ++k4)
              mac4<TR, TC, PARITY, kKS>(acc, Es, Hs, rbase, cbase, cstride, k4);
          } else {
            for (int k4 = 0; k4 < kv; ++k4)
              mac4<TR, TC, PARITY, kKS>(acc, Es, Hs, rbase, cbase, cstride, k4);
          }
        }
      }
    }
    cp_async_wait<0>();
    if constexpr (F2) {  // the two partial chains of each output
#pragma unroll
      for (int rb = 0; rb < TR; ++rb)
#pragma unroll
        for (int cb = 0; cb < TC; ++cb)
          acc[rb][cb][0] = __uint_as_float(static_cast<uint32_t>(accf[rb][cb])) +
                           __uint_as_float(static_cast<uint32_t>(accf[rb][cb] >> 32));
    }
    if constexpr (X2) {  // unpack the pairs into the four reference lanes
#pragma unroll
      for (int rb = 0; rb < TR; ++rb)
#pragma unroll
        for (int cb = 0; cb < TC; ++cb) {
          acc[rb][cb][0] = __uint_as_float(static_cast<uint32_t>(acc2[rb][cb][0]));
          acc[rb][cb][1] = __uint_as_float(static_cast<uint32_t>(acc2[rb][cb][0] >> 32));
          acc[rb][cb][2] = __uint_as_float(static_cast<uint32_t>(acc2[rb][cb][1]));
          acc[rb][cb][3] = __uint_as_float(static_cast<uint32_t>(acc2[rb][cb][1] >> 32));
        }
    }
    pdl_trigger();
    // the d mod 4 tail (all of d when d < 4) sits in the last chunk: lane 0
    if (d4 < d && warp_live) {
      const int cl = (nchunks - 1) * kKC;
      const float* Es = sm + ((nchunks - 1) % kStages) * STAGE;
      const float* Hs = Es + CT * kKS;
      for (int k = d4; k < d; ++k) {
#pragma unroll
        for (int rb = 0; rb < TR; ++rb) {
          const float h = Hs[(rbase + rb) * kKS + k - cl];
#pragma unroll
          for (int cb = 0; cb < TC; ++cb) {
            const float e = Es[(cbase + cb * cstride) * kKS + k - cl];
            if (PARITY) acc[rb][cb][0] = __fadd_rn(__fmul_rn(h, e), acc[rb][cb][0]);
            else acc[rb][cb][0] = fmaf(h, e, acc[rb][cb][0]);
          }
        }
      }
    }
#pragma unroll
    for (int cb = 0; cb < TC; ++cb) {
      const int c = cbase + cstride * cb;
      if (c >= ncols) continue;
      const uint32_t wid = VEC ? sid[c] / static_cast<uint32_t>(d) : sid[c];  // VEC: sid = id*d
      const float bias = a.bias ? __ldg(a.bias + wid) : 0.0f;
      const size_t col = col0 + c;
#pragma unroll
      for (int rb = 0; rb < TR; ++rb) {
        const int r = row0 + rbase + rb;
        if (r >= rowlim) continue;
        float v;
        if constexpr (PARITY) {
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

#ifndef LSB_BODIES_ONLY  // (k_step_fused.cu includes this file for logits_job)
template <int RB, int CB, bool PARITY, bool VEC, int kStages, int KC, bool TWO_D = false>
__global__ void __launch_bounds__(kLT, kStages == 2 ? 5 : 3) k_logits(const __grid_constant__ LogitsArgs a) {
  extern __shared__ __align__(16) float sm[];
  logits_job<RB, CB, PARITY, VEC, kStages, KC, TWO_D>(a, blockIdx.x, sm);
}

// Rows per CTA for beam B: minimise the padded rows a sentence costs,
// weighted by the measured relative throughput of each tile (2-D 3x4 lanes
// at RB = 12 is the fastest; RB = 16 spills at 96 registers).
int choose_rb(int B) {
  struct Opt {
    int rb;
    float eff;
  };
  static const Opt opts[] = {{12, 1.0f}, {8, 0.9f}, {10, 0.8f}, {16, 0.75f},
                             {6, 0.7f},  {4, 0.6f}, {2, 0.4f},  {1, 0.3f}};
  int best = 1;
  float best_cost = 1e30f;
  for (const Opt& o : opts) {
    const int groups = (B + o.rb - 1) / o.rb;
    const float cost = static_cast<float>(groups * o.rb) / o.eff;
    if (cost < best_cost) {
      best_cost = cost;
      best = o.rb;
    }
  }
  return best;
}

template <int RB, int CB, bool PARITY, bool VEC, int NS, int KC = 32, bool TWO_D = false>
static lsb_status launch_variant(lsb_ctx* ctx, const LogitsArgs& a, int grid) {
  constexpr size_t smem = logits_smem_bytes<RB, CB, NS, KC, TWO_D>();
  auto* kern = k_logits<RB, CB, PARITY, VEC, NS, KC, TWO_D>;
  if (lsb_status rc = ensure_smem(ctx, kern, smem)) return rc;
  LSB_CUDA(launch_pdl(ctx, kern, dim3(grid), dim3(kLT), smem, a));
  LSB_LAUNCHED(ctx, "k_logits");
  return LSB_OK;
}

static const int kMinSurvivorCtas =
    getenv("LSB_K4_MIN_SURV") ? atoi(getenv("LSB_K4_MIN_SURV")) : 4;

template <int RB, int CB, bool PARITY, int KC = 32, bool TWO_D = false, int NSO = 0>
static lsb_status launch_logits_rb(lsb_ctx* ctx, LogitsArgs a, int target) {
  constexpr int CT = tile_cols<CB, TWO_D>();
  const int rgroups = (a.R_total + RB - 1) / RB;
  a.ctiles_shared = static_cast<int>((a.n_shared + CT - 1) / CT);
  a.jobs_shared = (a.n_shared && !a.skip_shared) ? rgroups * a.ctiles_shared : 0;
  a.G = (a.Bsent + RB - 1) / RB;
  if (a.ids && a.S > 0) {
    const size_t max_tiles = (a.ncap > a.n_shared ? a.ncap - a.n_shared : 0) / CT + 1;
    // at least 4 CTAs per row group: a large shared block must not leave each
    // sentence's ~3 survivor tiles to one CTA in series (S=128: 283 -> see DESIGN)
    const int want = std::max(kMinSurvivorCtas, (target - a.jobs_shared) / std::max(1, a.S * a.G));
    a.X = static_cast<int>(std::min<size_t>({static_cast<size_t>(want), size_t(512), max_tiles}));
  } else {
    a.X = 0;
  }
  const int grid = a.jobs_shared + a.S * a.G * a.X;
  if (grid == 0) return LSB_OK;
  const bool vec = (a.d & 3) == 0 && (reinterpret_cast<uintptr_t>(a.E) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(a.H) & 15) == 0;
  if constexpr (NSO > 0)  // explicit ring depth (small batches: latency-bound)
    return vec ? launch_variant<RB, CB, PARITY, true, NSO, KC, TWO_D>(ctx, a, grid)
               : launch_variant<RB, CB, PARITY, false, NSO, KC, TWO_D>(ctx, a, grid);
  // Survivor-only launches (the shared block went to the tensor cores) have
  // no other CTAs to hide their L2 latency behind: 3-stage ring instead of 2.
  if (a.skip_shared)
    return vec ? launch_variant<RB, CB, PARITY, true, 3, KC, TWO_D>(ctx, a, grid)
               : launch_variant<RB, CB, PARITY, false, 3, KC, TWO_D>(ctx, a, grid);
  return vec ? launch_variant<RB, CB, PARITY, true, 2, KC, TWO_D>(ctx, a, grid)
             : launch_variant<RB, CB, PARITY, false, 2, KC, TWO_D>(ctx, a, grid);
}

static lsb_status launch_logits_survivors(lsb_ctx* ctx, LogitsArgs a, lsb_mode mode,
                                          int target_ctas);

// One column per thread, RB rows: 8 FP instructions (PARITY) or 4 FFMA
// (FAST) per 16-byte E load; 5 CTAs per SM.
lsb_status launch_logits(lsb_ctx* ctx, LogitsArgs a, lsb_mode mode, int target_ctas) {
  const bool fast = mode == LSB_MODE_FAST;
  a.x2_negzero = 0x8000000080000000ull;  // runtime operands of the paired FP32 path
  a.x2_one = 0x3F8000003F800000ull;
  // FAST + enough rows sharing the identity columns [0, n_shared): a dense
  // contraction -> tcgen05 tensor cores; the per-sentence survivors stay on
  // the FFMA kernel below.
  static const bool tc_off = getenv("LSB_NO_TC") != nullptr;
  // (The tensor-core block pays off for large dense blocks -- the full
  // vocabulary; for a T = 1000 shared block the paired-FFMA tile was faster:
  // 92 vs 97 us at cfg 2, before FAST used FFMA2.)
  static const int tc_min_cols = getenv("LSB_TC_MIN_COLS") ? atoi(getenv("LSB_TC_MIN_COLS")) : 1;
  if (fast && !tc_off && a.n_shared >= static_cast<uint32_t>(std::max(1, tc_min_cols)) &&
      a.R_total >= (a.ids ? 4 * kTcMinRows : kTcMinRows) && (a.d & 3) == 0 &&
      (reinterpret_cast<uintptr_t>(a.E) & 15) == 0 && (reinterpret_cast<uintptr_t>(a.H) & 15) == 0) {
    // With survivors to score, the tensor-core block goes to a side stream
    // (fork / join events) so it overlaps the survivor tiles on this one.
    const bool overlap = a.ids && a.S > 0;
    cudaStream_t main_stream = ctx->stream;
    if (overlap) {
      if (!ctx->side) {
        LSB_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        LSB_CUDA(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming));
        LSB_CUDA(cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming));
      }
      LSB_CUDA(cudaEventRecord(ctx->fork, main_stream));
      LSB_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork, 0));
      ctx->stream = ctx->side;
    }
    lsb_status rc;
    if (a.tc_A && a.tc_H) {
      rc = launch_tf32_tile(ctx, a.H, a.R_total, a.d, a.tc_N, a.tc_H);
      if (!rc)
        rc = launch_tc_logits_tiled(ctx, a.tc_A, a.tc_H, a.tc_N, a.R_total, a.d, a.bias, 0,
                                    a.n_shared, a.out, a.ldo, 0);
    } else {
      rc = launch_tc_logits(ctx, a.H, a.R_total, a.E, a.bias, a.d, 0, a.n_shared, a.out, a.ldo, 0);
    }
    ctx->stream = main_stream;
    if (rc) return rc;
    a.skip_shared = 1;
    if (!overlap) return LSB_OK;
    LSB_CUDA(cudaEventRecord(ctx->join, ctx->side));
    lsb_status rs = launch_logits_survivors(ctx, a, mode, target_ctas);
    LSB_CUDA(cudaStreamWaitEvent(main_stream, ctx->join, 0));
    return rs;
  }
  return launch_logits_survivors(ctx, a, mode, target_ctas);
}

// The FFMA tiles: the whole candidate set, or (skip_shared) the survivors.
static lsb_status launch_logits_survivors(lsb_ctx* ctx, LogitsArgs a, lsb_mode mode,
                                          int target_ctas) {
  const bool fast = mode == LSB_MODE_FAST;
  // PARITY over a large identity block shared by >= 2 row groups (the full
  // vocabulary): the one-lane-per-thread kernel of k_logits_ln.cu (same bits;
  // B200 cfg-2 shapes, S = 16 / 64 / 128: 588 / 2265 / 4606 us vs 633 / 2696 /
  // 5328 us here). With per-sentence survivors it measured slower (108-125 vs
  // 100 us at cfg 2), and so did the cfg-2 shared block alone on it beside
  // the survivor tiles on a second stream (119 vs 102 us: 512 CTAs, under one
  // wave, no steady state), so the LSH step keeps the tiles below. (Also
  // measured: the top-T block started on a side stream at the step's start,
  // overlapping K1-K3: 500 k vs 508 k sentence-steps/s -- the FP-bound block
  // takes the SM slots the latency-bound probe needs.)
  // (On the LSH step it wins only with many survivors per sentence: d = 256
  // and ~2470 survivors, S = 64: 75.8 vs 100.4 us; with the operating point's
  // ~400 candidates it lost, 0.146 vs 0.132 ms per step: survivor counts are
  // only known on the device, so the LSH step keeps the tiles below.)
  static const int ln_mode = getenv("LSB_K4_LN") ? atoi(getenv("LSB_K4_LN")) : 1;
  if (!fast && ln_mode && logits_ln_applies(a) &&
      (ln_mode == 2 || (!a.ids && a.R_total > 12 && a.n_shared >= 4096)))
    return launch_logits_ln(ctx, a, target_ctas);
#define LSB_RB(R)                                                        \
  case R:                                                                \
    return fast ? launch_logits_rb<R, 1, false>(ctx, a, target_ctas)     \
                : launch_logits_rb<R, 1, true>(ctx, a, target_ctas);
  // Measured at cfg 2 (PARITY, B200): 1-D 12x1 tile 119 us; 2-D 3x4 per
  // lane 100 us; 2-D 3x3 106 us; 2-D with 64- or 256-thread CTAs 115 / 165
  // us; 1-D 6x2 with 16-float chunks 151 us; 4 CTAs/SM at 128 registers
  // 116 us; TMA bulk row copies 129 us (the per-lane operands serialise);
  // shared block in 16-row 4x4 tiles at 4 CTAs/SM 141 us; 3x2 lanes at 8
  // CTAs/SM 150 us; output halves (reference lanes 0-1 / 2-3) in neighbouring
  // lanes, 3x8 half-outputs per lane with 8-byte loads (22 instead of 28
  // wavefronts per 48 FFMA2, bit-exact) 105 us; 3x2 lanes (64-column tiles) at
  // 5 CTAs/SM 125 us; 16-float chunks in a 4-deep ring at 5 CTAs/SM 113 us.
  // (Also measured: the whole per-sentence candidate list -- the identity
  // block [0, T) is its prefix -- as survivor tiles only, 128 columns, so no
  // part-filled block/survivor tile boundary: cfg 2 K4 102.1 vs 102.5 us but
  // 502 vs 504 k sentence-steps/s, and S=128 231 vs 186 us.)
  // Small batches (a few sentences) fill a fraction of the GPU and each CTA
  // waits on its chunk loads: 32-column tiles (4x the CTAs) and an 8-deep ring.
  // (Measured, cfg 2 shapes: S=1 36 -> 18 us, S=8 49 -> 29, S=16 66 -> 49,
  // S=32 equal.) "Small" = the 128-column tiling would give at most two CTAs
  // per SM; without a shared block assume ~10 survivor tiles per row group.
  static const bool no_small = getenv("LSB_K4_NO_SMALL") != nullptr;
  const int rb = choose_rb(a.Bsent);
  const long est = static_cast<long>((a.R_total + rb - 1) / rb) *
                   (a.n_shared ? static_cast<long>((a.n_shared + 127) / 128) : 10L);
  // survivor-only launches (the shared block went to the tensor cores):
  // assume ~3 column tiles of 128 per row group; small ones use 64-column
  // tiles and a 4-deep ring (FAST cfg 2: 96.5 -> 89.2 us/step vs 32-column,
  // 8-deep; 128-column 93.8)
  const long est_surv = static_cast<long>(a.S) * ((a.Bsent + rb - 1) / rb) * 3L;
  const bool small = !no_small && (a.skip_shared ? est_surv <= 2L * ctx->sm_count
                                                 : est <= 2L * ctx->sm_count);
#define LSB_RB2(R)                                                                   \
  case R:                                                                            \
    if (small && a.skip_shared) /* survivors beside the TC block */                  \
      return fast ? launch_logits_rb<R, 2, false, 32, true, 4>(ctx, a, target_ctas)  \
                  : launch_logits_rb<R, 2, true, 32, true, 4>(ctx, a, target_ctas);  \
    if (small)                                                                       \
      return fast ? launch_logits_rb<R, 1, false, 32, true, 8>(ctx, a, target_ctas)  \
                  : launch_logits_rb<R, 1, true, 32, true, 8>(ctx, a, target_ctas);  \
    return fast ? launch_logits_rb<R, 4, false, 32, true>(ctx, a, target_ctas)       \
                : launch_logits_rb<R, 4, true, 32, true>(ctx, a, target_ctas);
  switch (rb) {
    LSB_RB2(16)
    LSB_RB2(12)
    LSB_RB(10)
    LSB_RB2(8)
    LSB_RB(6)
    LSB_RB(4)
    LSB_RB(2)
    default:
      return fast ? launch_logits_rb<1, 1, false>(ctx, a, target_ctas)
                  : launch_logits_rb<1, 1, true>(ctx, a, target_ctas);
  }
#undef LSB_RB
#undef LSB_RB2
}

#endif  // LSB_BODIES_ONLY

}  // namespace lsb
