// k_tc_logits.cu -- K4 on the 5th-generation tensor cores (FAST mode only).
//
// When S*B rows share the same candidate columns -- the top-T prefix of the
// LSH step (ids 0..T-1 for every sentence) and the whole vocabulary of the
// kFull baseline -- the logits are a real dense contraction
// logits[r][c] = sum_k H[r][k] * E[c0 + c][k], and run as a tcgen05 GEMM:
//
//  * operands are split once into 3xTF32 pairs (hi = rna_tf32(x),
//    lo = rna_tf32(x - hi)) and PRE-TILED in global memory in the canonical
//    no-swizzle K-major UMMA layout (k_tf32_tile): for every tile of R rows
//    and every 32-wide chunk of d, [plane hi|lo][8 core columns of 4 tf32]
//    [R rows] x 16 B is one contiguous block of R * 256 bytes. E's top-T
//    block is tiled once per batch, H once per step.
//  * CTA tile: M = 128 candidate columns (operand A = E) x N in {32, 64, 128}
//    hypothesis rows (operand B = H). One thread streams each chunk's A and B
//    blocks into a 3-4 stage shared-memory ring with cp.async.bulk (TMA bulk
//    copies completing on "full" mbarriers) and issues 4 K-steps x 3
//    tcgen05.mma.kind::tf32 (A_lo.B_hi + A_hi.B_lo + A_hi.B_hi) per chunk;
//    tcgen05.commit on the stage's "empty" mbarrier releases the slot.
//  * promotion: every kTcPromote chunks accumulate into their own TMEM
//    accumulator (two, ping-pong, 128 lanes x N fp32 columns); while the
//    next chunks' MMAs run, all threads drain the finished one (tcgen05.ld 32x32b: warp w owns
//    TMEM lanes 32w..32w+31 = candidate columns) and add it into fp32
//    registers with round-to-nearest FADDs. Measured on B200 at d = 1000:
//    accumulating all 125 K-steps inside the tensor core gave 3.5e-4
//    relative error (its internal adds keep fewer bits), promotion gives
//    ~2e-5 -- inside FAST's 1e-4 (1+|l|) and at the FFMA path's level.
//  * epilogue: + bias, coalesced stores of the [row][col] logits.
#include <algorithm>
#include <cstdlib>

#include "async_copy.cuh"
#include "k_step.cuh"

namespace lsb {

namespace tc {

constexpr int kM = 128;        // candidate columns per CTA (UMMA M)
constexpr int kKC = 32;        // d per chunk
constexpr int kThreads = 128;

// Canonical K-major, no-swizzle UMMA shared-memory descriptor: 8-row x 16-B
// core matrices, rows 16 B apart; the next 8 rows SBO bytes away, the next
// 16 B of K (4 tf32) LBO bytes away (cute::UMMA::SmemDescriptor layout,
// version 1 for sm_100).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // version
  return d;         // base offset 0, legacy LBO mode, layout SWIZZLE_NONE
}

// kind::tf32 instruction descriptor: F32 accumulate, A/B TF32, both K-major.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(mbar)));
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

}  // namespace tc

// Chunks (of 32 along d) summed inside one TMEM accumulator before the fp32
// promotion: 2 keeps the error at the FFMA level (see the header comment)
// and halves the drains.
constexpr int kTcPromote = 2;

// ------------------------------------------------------- operand pre-tiling
// out[((tile * nchunks + c) * 2 + plane) * 8 + k4][r] (16-B units) holds
// rows tile*R + r, floats c*32 + 4*k4 .. +4 of src, split into tf32 hi / lo
// planes; rows >= nrows and floats >= d are zero.
__global__ void k_tf32_tile(const float* __restrict__ src, int nrows, int d, int R, int nchunks,
                            int ntiles, float4* __restrict__ out) {
  const long long total = static_cast<long long>(ntiles) * nchunks * 8 * R;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(q % R);
    long long t = q / R;
    const int k4 = static_cast<int>(t % 8);
    t /= 8;
    const int c = static_cast<int>(t % nchunks);
    const int tile = static_cast<int>(t / nchunks);
    const int row = tile * R + r;
    const int k = c * tc::kKC + k4 * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < nrows && k < d) {
      const float* p = src + static_cast<size_t>(row) * d + k;
      if (k + 4 <= d && (d & 3) == 0) {
        v = __ldg(reinterpret_cast<const float4*>(p));
      } else {
        v.x = p[0];
        if (k + 1 < d) v.y = p[1];
        if (k + 2 < d) v.z = p[2];
        if (k + 3 < d) v.w = p[3];
      }
    }
    float4 hi, lo;
    hi.x = tc::tf32_rna(v.x); lo.x = tc::tf32_rna(v.x - hi.x);
    hi.y = tc::tf32_rna(v.y); lo.y = tc::tf32_rna(v.y - hi.y);
    hi.z = tc::tf32_rna(v.z); lo.z = tc::tf32_rna(v.z - hi.z);
    hi.w = tc::tf32_rna(v.w); lo.w = tc::tf32_rna(v.w - hi.w);
    const size_t base = ((static_cast<size_t>(tile) * nchunks + c) * 2) * 8;
    out[(base + k4) * R + r] = hi;
    out[(base + 8 + k4) * R + r] = lo;
  }
}

size_t tf32_tiled_floats(int nrows, int d, int R) {
  const size_t ntiles = (static_cast<size_t>(nrows) + R - 1) / R;
  const size_t nchunks = (static_cast<size_t>(d) + tc::kKC - 1) / tc::kKC;
  return ntiles * nchunks * 2 * 8 * R * 4;
}

lsb_status launch_tf32_tile(lsb_ctx* ctx, const float* src, int nrows, int d, int R, float* out) {
  if (nrows <= 0) return LSB_OK;
  const int ntiles = (nrows + R - 1) / R;
  const int nchunks = (d + tc::kKC - 1) / tc::kKC;
  const long long total = static_cast<long long>(ntiles) * nchunks * 8 * R;
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, ctx->sm_count * 16LL));
  k_tf32_tile<<<grid, 256, 0, ctx->stream>>>(src, nrows, d, R, nchunks, ntiles,
                                             reinterpret_cast<float4*>(out));
  LSB_LAUNCHED(ctx, "k_tf32_tile");
  return LSB_OK;
}

// ------------------------------------------------------------------ GEMM
struct TcLogitsArgs {
  const float* A;     // tiled E block (R = 128)
  const float* Bm;    // tiled H (R = N)
  const float* bias;  // indexed by col0 + c, or null
  int nchunks;
  int rows;           // hypothesis rows
  uint32_t col0, ncols;  // candidate columns [col0, col0 + ncols)
  float* out;         // out[r * ldo + out_col0 + c]
  size_t ldo;
  uint32_t out_col0;
};

// N hypothesis rows per tile, S pipeline stages, P chunks per promotion.
template <int N, int S, int P>
__global__ void __launch_bounds__(tc::kThreads, 1) k_tc_logits(TcLogitsArgs a) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr uint32_t kABytes = kM * 256;  // one chunk of A: hi + lo planes
  constexpr uint32_t kBBytes = N * 256;
  constexpr uint32_t kStage = kABytes + kBBytes;
  __shared__ __align__(8) uint64_t full[S], empty[S];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * N;        // first hypothesis row (x: launched fastest)
  const uint32_t m0 = blockIdx.y * kM;  // first candidate column
  const int nchunks = a.nchunks;
  const char* gA = reinterpret_cast<const char*>(a.A) + static_cast<size_t>(blockIdx.y) * nchunks * kABytes;
  const char* gB = reinterpret_cast<const char*>(a.Bm) + static_cast<size_t>(blockIdx.x) * nchunks * kBBytes;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "n"(2 * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base_s;
  constexpr uint32_t idesc = make_idesc(kM, N);

  auto load = [&](int kc) {  // thread 0 only
    const int s = kc % S;
    unsigned char* dst = smem + s * kStage;
    mbar_expect_tx(&full[s], kStage);
    bulk_g2s(dst, gA + static_cast<size_t>(kc) * kABytes, kABytes, &full[s]);
    bulk_g2s(dst + kABytes, gB + static_cast<size_t>(kc) * kBBytes, kBBytes, &full[s]);
  };
  if (tid == 0)
    for (int kc = 0; kc < S && kc < nchunks; ++kc) load(kc);

  float sum[N];
#pragma unroll
  for (int j = 0; j < N; ++j) sum[j] = 0.0f;
  auto drain = [&](int acc) {
#pragma unroll
    for (int c = 0; c < N; c += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + acc * N + c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) sum[c + j] = __fadd_rn(sum[c + j], __uint_as_float(v[j]));
    }
  };

  for (int kc = 0; kc < nchunks; ++kc) {
    const int s = kc % S;
    if (tid == 0) {
      mbar_wait(&full[s], (kc / S) & 1);  // chunk kc landed
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t ab = smem_u32(smem + s * kStage);
      const uint32_t ahi = ab, alo = ab + kM * 128;
      const uint32_t bhi = ab + kABytes, blo = ab + kABytes + N * 128;
      const uint32_t dacc = tmem + ((kc / P) & 1) * N;
      const bool fresh = kc % P == 0;
#pragma unroll
      for (int j = 0; j < kKC / 8; ++j) {  // UMMA K = 8 tf32 = two 16-B core columns
        const uint32_t oa = j * 2 * kM * 16, ob = j * 2 * N * 16;
        const uint64_t dah = make_desc(ahi + oa, kM * 16, 128);
        const uint64_t dal = make_desc(alo + oa, kM * 16, 128);
        const uint64_t dbh = make_desc(bhi + ob, N * 16, 128);
        const uint64_t dbl = make_desc(blo + ob, N * 16, 128);
        mma_tf32(dacc, dal, dbh, idesc, (fresh && j == 0) ? 0u : 1u);  // small terms first
        mma_tf32(dacc, dah, dbl, idesc, 1u);
        mma_tf32(dacc, dah, dbh, idesc, 1u);
      }
      mma_commit(&empty[s]);
      // refill the slot of chunk kc-1 once its MMAs have read it
      if (kc >= 1 && kc - 1 + S < nchunks) {
        mbar_wait(&empty[(kc - 1) % S], ((kc - 1) / S) & 1);
        load(kc - 1 + S);
      }
    }
    // chunk kc-1 closed a promotion block: drain that accumulator while
    // chunk kc's MMAs run (only here do the threads synchronise)
    if (kc >= 1 && kc % P == 0) {
      mbar_wait(&empty[(kc - 1) % S], ((kc - 1) / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      drain(((kc - 1) / P) & 1);
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      __syncthreads();
    }
  }
  {
    const int kc = nchunks - 1;
    mbar_wait(&empty[kc % S], (kc / S) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    drain((kc / P) & 1);
  }

  const uint32_t col = m0 + warp * 32 + lane;
  if (col < a.ncols) {
    const float bias = a.bias ? __ldg(a.bias + a.col0 + col) : 0.0f;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int r = n0 + j;
      if (r < a.rows)
        a.out[static_cast<size_t>(r) * a.ldo + a.out_col0 + col] = __fadd_rn(sum[j], bias);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(2 * N));
}

template <int N, int S, int P = kTcPromote>
static lsb_status launch_tc_n(lsb_ctx* ctx, const TcLogitsArgs& a) {
  constexpr size_t smem = static_cast<size_t>(S) * (tc::kM * 256 + N * 256);
  if (lsb_status rc = ensure_smem(ctx, k_tc_logits<N, S, P>, smem)) return rc;
  // x = hypothesis-row tiles (launched fastest), y = candidate-column tiles:
  // the CTAs that share one E tile run back to back and hit it in L2
  dim3 grid((a.rows + N - 1) / N, (a.ncols + tc::kM - 1) / tc::kM);
  k_tc_logits<N, S, P><<<grid, tc::kThreads, smem, ctx->stream>>>(a);
  LSB_LAUNCHED(ctx, "k_tc_logits");
  return LSB_OK;
}

// Widest tile that still gives every SM work (narrower tiles re-read E more).
int tc_rows_per_tile(lsb_ctx* ctx, int rows, uint32_t ncols) {
  static const int force = getenv("LSB_TC_N") ? atoi(getenv("LSB_TC_N")) : 0;
  if (force == 64 || force == 128) return force;
  const long long mt = (ncols + tc::kM - 1) / tc::kM;
  if (mt * ((rows + 127) / 128) >= 2 * ctx->sm_count) return 128;
  return 64;  // N = 32 measured slower: TMA latency exposed with 2 stages
}

lsb_status launch_tc_logits_tiled(lsb_ctx* ctx, const float* A_tiled, const float* H_tiled,
                                  int N, int rows, int d, const float* bias, uint32_t col0,
                                  uint32_t ncols, float* out, size_t ldo, uint32_t out_col0) {
  if (rows <= 0 || ncols == 0) return LSB_OK;
  TcLogitsArgs a{A_tiled, H_tiled, bias, (d + tc::kKC - 1) / tc::kKC, rows, col0, ncols,
                 out, ldo, out_col0};
  if (N == 128) return launch_tc_n<128, 3>(ctx, a);
  if (N == 64) return launch_tc_n<64, 4>(ctx, a);
  return launch_tc_n<32, 2>(ctx, a);  // 80 KB: two CTAs per SM
}

// One-off calls: tiles both operands into stream-ordered temporaries.
lsb_status launch_tc_logits(lsb_ctx* ctx, const float* H, int rows, const float* E,
                            const float* bias, int d, uint32_t col0, uint32_t ncols, float* out,
                            size_t ldo, uint32_t out_col0) {
  if (rows <= 0 || ncols == 0) return LSB_OK;
  const int N = tc_rows_per_tile(ctx, rows, ncols);
  float *At = nullptr, *Ht = nullptr;
  LSB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&At), tf32_tiled_floats(ncols, d, tc::kM) * 4,
                           ctx->stream));
  LSB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&Ht), tf32_tiled_floats(rows, d, N) * 4,
                           ctx->stream));
  lsb_status rc = launch_tf32_tile(ctx, E + static_cast<size_t>(col0) * d, ncols, d, tc::kM, At);
  if (!rc) rc = launch_tf32_tile(ctx, H, rows, d, N, Ht);
  if (!rc)
    rc = launch_tc_logits_tiled(ctx, At, Ht, N, rows, d, bias, col0, ncols, out, ldo, out_col0);
  cudaFreeAsync(At, ctx->stream);
  cudaFreeAsync(Ht, ctx->stream);
  return rc;
}

}  // namespace lsb
