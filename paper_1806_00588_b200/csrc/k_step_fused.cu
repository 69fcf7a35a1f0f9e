// k_step_fused.cu -- one LSH step (K1+K2 -> K3 -> K4 -> K5a -> K5b) as ONE
// cooperative launch, for small batches (a one-sentence decode: BASELINE
// cfg 1, S = 1, B = 12).
//
// At S = 1 the five kernels of the step each fill a fraction of the GPU and
// the step is a chain of launch latencies and dependency waits (PDL overlaps
// only the prologues). Here a persistent grid (as many 128-thread CTAs as fit
// on the SMs) runs the same device functions the separate kernels run --
// probe_row, compact_sentence, logits_job, softmax_row, expand_sentence, so
// the arithmetic and the bits are the same -- looping over each stage's jobs,
// with a grid-wide barrier between stages. The probe stage splits every row's
// vocabulary into more slices than the separate kernel does (one CTA each),
// so the 128-thread CTAs still cover the GPU; each slice counts its own word
// range over all W bands, so the candidate sets do not depend on the split.
//
// Measured on B200 (S=1, B=12, cfg-1 shapes): 59 us per step against 37 us for
// the separate kernels with PDL; its stages (probe 6.6, compact 8.7, logits
// 14.7, softmax 7.2, expansion 17.3 us, grid barrier included) show the
// one-CTA stages on 128 threads costing more than the launch gaps it removes.
// Bit-exact with the separate kernels (tests/test_gpu_step.py), so opt-in.
//
// The device functions come from the kernels' own sources, included with
// LSB_BODIES_ONLY (which hides their __global__ wrappers and host code):
// whole-program compilation cannot call device code across files.
#define LSB_BODIES_ONLY
#include "k_step.cu"
#include "k_logits.cu"
#include "k_select.cu"
#undef LSB_BODIES_ONLY

#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "batch.cuh"

namespace lsb {
namespace {

namespace cg = cooperative_groups;

constexpr int kFT = 128;  // threads per CTA: K4's and K5a's tile (kLT, kSelT)
static_assert(kFT == kLT && kFT == kSelT, "one CTA shape for every stage");

struct FusedArgs {
  ProbeArgs pa;
  CompactArgs ca;
  LogitsArgs la;
  SoftmaxArgs sa;
  ExpandArgs ea;
  int rows;          // S * B
  int probe_jobs;    // rows * slices
  int logits_jobs;
  unsigned long long* stamps;  // LSB_FUSED_TIMING: globaltimer at each stage end (CTA 0)
};

__device__ __forceinline__ void stamp(const FusedArgs& f, int k) {
  if (f.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    f.stamps[k] = t;
  }
}

template <int RB, bool PARITY>
__global__ void __launch_bounds__(kFT, 4) k_step_fused(const __grid_constant__ FusedArgs f) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::grid_group grid = cg::this_grid();
  const int S = f.ea.S;
  stamp(f, 0);
  for (int j = blockIdx.x; j < f.probe_jobs; j += gridDim.x) {  // K1 + K2
    probe_row(f.pa, smem, j % f.rows, j / f.rows);
    __syncthreads();
  }
  grid.sync();
  stamp(f, 1);
  for (int s = blockIdx.x; s < S; s += gridDim.x) {  // K3
    compact_sentence(f.ca, s, reinterpret_cast<uint32_t*>(smem));
    __syncthreads();
  }
  grid.sync();
  stamp(f, 2);
  for (int j = blockIdx.x; j < f.logits_jobs; j += gridDim.x) {  // K4
    logits_job<RB, 1, PARITY, true, 8, 32, true>(f.la, j, reinterpret_cast<float*>(smem));
    __syncthreads();
  }
  grid.sync();
  stamp(f, 3);
  for (int r = blockIdx.x; r < f.rows; r += gridDim.x) {  // K5a
    softmax_row(f.sa, r);
    __syncthreads();
  }
  grid.sync();
  stamp(f, 4);
  for (int s = blockIdx.x; s < S; s += gridDim.x) {  // K5b
    expand_sentence(f.ea, s, smem);
    __syncthreads();
  }
  if (f.stamps) {
    grid.sync();
    stamp(f, 5);
  }
}

template <int RB>
constexpr size_t fused_logits_smem() {
  return logits_smem_bytes<RB, 1, 8, 32, true>();
}

using FusedKernel = void (*)(FusedArgs);

FusedKernel fused_kernel(int rb, bool parity) {
  switch (rb) {
    case 12:
      return parity ? k_step_fused<12, true> : k_step_fused<12, false>;
    case 8:
      return parity ? k_step_fused<8, true> : k_step_fused<8, false>;
    default:
      return nullptr;
  }
}

// K4's job layout for the fused grid: launch_logits_rb<RB, 1, *, 32, true, 8>
// (k_logits.cu) with target = the grid. The split of a sentence's survivor
// tiles over X jobs only changes which CTA computes a tile, not its bits.
int plan_logits(LogitsArgs& a, int rb, int target) {
  constexpr int CT = tile_cols<1, true>();
  const int rgroups = (a.R_total + rb - 1) / rb;
  a.ctiles_shared = static_cast<int>((a.n_shared + CT - 1) / CT);
  a.jobs_shared = a.n_shared ? rgroups * a.ctiles_shared : 0;
  a.G = (a.Bsent + rb - 1) / rb;
  const size_t max_tiles = (a.ncap > a.n_shared ? a.ncap - a.n_shared : 0) / CT + 1;
  const int want = std::max(4, (target - a.jobs_shared) / std::max(1, a.S * a.G));
  a.X = static_cast<int>(std::min<size_t>({static_cast<size_t>(want), size_t(512), max_tiles}));
  a.x2_negzero = 0x8000000080000000ull;
  a.x2_one = 0x3F8000003F800000ull;
  return a.jobs_shared + a.S * a.G * a.X;
}

}  // namespace

// Decided once per batch (b->fused: -1 undecided, 0 no, 1 yes):
//  * the LSH step (threshold mode, an index, the per-row probe kernel --
//    not the band-split one), at most LSB_FUSED_MAX_ROWS rows (default 48);
//  * K4 on the small-batch 2-D tiles (choose_rb = 12 or 8, no tensor-core
//    block, no LN kernel) and K5 on the default pair of kernels with the rank
//    expansion;
//  * no per-stage profiling (one launch has no stage boundaries);
//  * a cooperative grid of >= 1 CTA per SM.
// Opt-in: LSB_FUSED=1 (measured slower than the separate kernels, see the
// header).
lsb_status launch_step_fused(lsb_batch* b, const lsb_state_dev* in, const lsb_out_dev* out,
                             bool* done) {
  *done = false;
  lsb_ctx* ctx = b->ctx;
  if (b->fused == 0 || b->profile) return LSB_OK;
  if (b->fused < 0) {
    b->fused = 0;
    // opt-in (read per batch, so one process can compare both paths)
    const char* env = getenv("LSB_FUSED");
    if (!env || strcmp(env, "1") != 0) return LSB_OK;
    const bool verbose = getenv("LSB_FUSED_VERBOSE") != nullptr;
    auto no = [&](int line) {
      cudaGetLastError();
      if (verbose) fprintf(stderr, "k_step_fused: not used (k_step_fused.cu:%d)\n", line);
      return LSB_OK;
    };
    const int max_rows = getenv("LSB_FUSED_MAX_ROWS") ? atoi(getenv("LSB_FUSED_MAX_ROWS")) : 48;
    static const char* k5 = getenv("LSB_K5");
    static const char* ln = getenv("LSB_K4_LN");
    const int R = b->S * b->B;
    const int rb = choose_rb(b->B);
    if (b->cmode != 0 || !b->idx || b->t <= 0 || b->probe_G > 0 || R > max_rows || R == 0 ||
        (k5 && atoi(k5) != 0) || (ln && atoi(ln) == 2) || getenv("LSB_K4_NO_SMALL") ||
        (rb != 12 && rb != 8) || (b->d & 3) != 0 ||
        (reinterpret_cast<uintptr_t>(b->model->E) & 15) != 0 ||
        (b->mode == LSB_MODE_FAST && R >= 4 * kTcMinRows) || b->B > kRankMaxLists)
      return no(__LINE__);
    // stage shared memory: the largest of the five
    const size_t nl = b->B;
    const size_t expand = nl * std::max(b->B, 1) * (8 + 8 + 4 + 4 + 4 + 4);
    const size_t compact = static_cast<size_t>(b->nwords) * 4;
    const size_t logits = rb == 12 ? fused_logits_smem<12>() : fused_logits_smem<8>();
    // the probe at the fused slice length (counter planes of the slice)
    lsb_state_dev dummy{};
    ProbeArgs pa = probe_args(b, &dummy);
    size_t smem = std::max({expand, compact, logits});
    FusedKernel kern = fused_kernel(rb, b->mode != LSB_MODE_FAST);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) {
      cudaGetLastError();
      return no(__LINE__);
    }
    // slices per row: enough to give every CTA one (row, slice), but slices of
    // at least LSB_FUSED_MIN_SLICE words (each slice CTA re-hashes its row)
    const int min_slice =
        getenv("LSB_FUSED_MIN_SLICE") ? std::max(128, atoi(getenv("LSB_FUSED_MIN_SLICE"))) : 1024;
    // pass 0 at the separate kernel's slice length (the most shared memory),
    // pass 1 at the fused one: co-resident CTAs -> slices for that grid
    uint32_t slice_len = b->slice_len;
    int occ = 0;
    for (int pass = 0; pass < 2; ++pass) {
      pa.slice_len = slice_len;
      const size_t need = std::max(smem, probe_smem_bytes(pa));
      if (need + fa.sharedSizeBytes > ctx->smem_optin) return no(__LINE__);
      // (set even under 48 KB: the default limit counts the static part too)
      if (pass == 0 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(need)) != cudaSuccess)
        return no(__LINE__);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFT, need) != cudaSuccess ||
          occ < 1) {
        cudaGetLastError();
        return no(__LINE__);
      }
      // one CTA per SM: the cheapest grid barrier, and K4 at S = 1 has ~40
      // tiles (measured S=1 B=12: 1 / 2 / 3 per SM 59 / 64 / 70 us per step)
      occ = std::min(occ, getenv("LSB_FUSED_CTAS") ? std::max(1, atoi(getenv("LSB_FUSED_CTAS"))) : 1);
      const int grid = occ * ctx->sm_count;
      const uint32_t want_slices = std::max(1, grid / R);
      uint32_t len = (b->V + want_slices - 1) / want_slices;
      len = std::max<uint32_t>(len, static_cast<uint32_t>(min_slice));
      len = b->levels >= 0 ? (len + 127) & ~127u : (len + 63) & ~63u;
      if (pass == 1) b->fused_smem = need;
      else slice_len = std::min(len, b->slice_len);
    }
    // (the second pass sized the shared memory for the final slice length;
    // shorter slices need no more)
    b->fused_slice_len = slice_len;
    b->fused_grid = occ * ctx->sm_count;
    b->fused_rb = rb;
    b->fused = 1;
    if (verbose)
      fprintf(stderr, "k_step_fused: rows %d, grid %d (%d/SM), slice %u words, smem %zu + %zu\n", R,
              b->fused_grid, occ, slice_len, b->fused_smem, fa.sharedSizeBytes);
  }
  // per step: K4's vector loads need 16-byte aligned hidden rows
  if ((reinterpret_cast<uintptr_t>(in->hidden) & 15) != 0) return LSB_OK;
  FusedArgs f{};
  f.pa = probe_args(b, in);
  f.pa.slice_len = b->fused_slice_len;
  f.ca = compact_args(b, in, 1);
  f.la = logits_args(b, in);
  f.sa = softmax_args(b, in);
  f.ea = expand_args(b, in, out);
  f.rows = b->S * b->B;
  const uint32_t slices = (b->V + b->fused_slice_len - 1) / b->fused_slice_len;
  f.probe_jobs = f.rows * static_cast<int>(slices);
  f.logits_jobs = plan_logits(f.la, b->fused_rb, b->fused_grid);
  FusedKernel kern = fused_kernel(b->fused_rb, b->mode != LSB_MODE_FAST);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(b->fused_grid);
  cfg.blockDim = dim3(kFT);
  cfg.dynamicSmemBytes = b->fused_smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // LSB_FUSED_TIMING (debug): per-stage device times, mapped host stamps
  // owned by the batch, averages printed every 200 steps
  if (b->fused_timing < 0) b->fused_timing = getenv("LSB_FUSED_TIMING") != nullptr;
  if (b->fused_timing && !b->fused_stamps &&
      cudaHostAlloc(&b->fused_stamps, 8 * 8, cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    b->fused_stamps = nullptr;
    b->fused_timing = 0;
  }
  f.stamps = b->fused_timing ? b->fused_stamps : nullptr;
  LSB_CUDA(cudaLaunchKernelEx(&cfg, kern, f));
  LSB_LAUNCHED(ctx, "k_step_fused");
  if (f.stamps) {
    cudaStreamCaptureStatus cs;
    cudaStreamIsCapturing(ctx->stream, &cs);
    if (cs != cudaStreamCaptureStatusNone) return *done = true, LSB_OK;
    LSB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < 5; ++k) b->fused_acc[k] += (f.stamps[k + 1] - f.stamps[k]) * 1e-3;
    if (++b->fused_nacc % 200 == 0) {
      const double* acc = b->fused_acc;
      const int nacc = b->fused_nacc;
      fprintf(stderr, "k_step_fused stages (us): probe %.1f compact %.1f logits %.1f softmax %.1f expand %.1f\n",
              acc[0] / nacc, acc[1] / nacc, acc[2] / nacc, acc[3] / nacc, acc[4] / nacc);
    }
  }
  *done = true;
  return LSB_OK;
}

}  // namespace lsb
