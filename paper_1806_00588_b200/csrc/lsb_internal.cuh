// lsb_internal.cuh -- shared types and device helpers of the B200 LSH
// beam-search library. Host handles (lsb_ctx, lsb_model, lsb_index,
// lsb_batch) are defined here so every translation unit sees one layout.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "lshbeam_b200.h"

struct lsb_ctx;

namespace lsb {

// ------------------------------------------------------------- constants
constexpr uint32_t kEmptyCode = 0x7FFFFFFFu;  // include/lshbeam/wta_hash.hpp:13
constexpr int kMaxDisplacements = 128;        // include/lshbeam/band_index.hpp:56
constexpr int kMaxRebuilds = 8;               // include/lshbeam/band_index.hpp:57

// Device error word bits, surfaced by lsb_ctx_sync / synchronous calls.
enum : uint32_t {
  kErrNaN = 1u,         // NaN in a hashed row  -> LSB_EINVAL (wta_hash.cpp:169)
  kErrEmptyRow = 2u,    // softmax row without finite entries -> LSB_EINVAL
  kErrEmptyCands = 4u,  // empty candidate set -> LSB_ERUNTIME (beam_decoder.cpp:250)
  kErrCuckoo = 8u,      // rebuild budget exhausted -> LSB_ERUNTIME
};

// Per-band cuckoo metadata. Slots of band w live at slots[slot_off ..
// slot_off + 2*2^lg): table 0 then table 1, each slot {key,start,len,0}.
struct BandMeta {
  unsigned long long mul0, mul1;
  uint32_t lg, slot_off;
};

// Read-only device view of an index, passed by value to kernels.
struct IndexView {
  const uint32_t* perms;     // P x K prefixes
  const uint32_t* word_ids;  // W x V, band-major
  const uint4* slots;        // all bands' tables
  const BandMeta* bands;     // W
  uint32_t V;
  int W, K, u, bits, P, d;
  const uint16_t* perms16;   // P x K16 (K padded to a multiple of 8), or null
  int K16;
};

// ----------------------------------------------------------- host state
void set_error(const std::string& msg);
// Uploads idx->perms_host as the uint16 copy the probe kernels read with
// 16-byte loads (perms16, row stride K16 = K rounded up to 8); no-op for d > 65535.
cudaError_t upload_perms16(lsb_index* idx, cudaStream_t st);
lsb_status cuda_status(cudaError_t e, const char* what);
// Raises `func`'s dynamic shared-memory limit to at least `bytes` on the
// context's device. cudaFuncSetAttribute is per device, so the configured size
// is remembered per (kernel, device) under a lock (thread-safe, multi-GPU).
lsb_status ensure_smem(const lsb_ctx* ctx, const void* func, size_t bytes);
template <class F>
lsb_status ensure_smem(const lsb_ctx* ctx, F* func, size_t bytes) {
  return ensure_smem(ctx, reinterpret_cast<const void*>(func), bytes);
}

}  // namespace lsb

struct lsb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 148;
  size_t smem_optin = 0;
  uint32_t* err_dev = nullptr;   // device error word
  uint32_t* err_host = nullptr;  // pinned mirror
  uint64_t launches = 0;
  int cuckoo_parallel = 0;        // 0: reference slot placement
  int pdl = 1;                    // programmatic dependent launch between step kernels
  // FAST: the tensor-core shared block runs on a side stream concurrently
  // with the survivor tiles (created on first use)
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

struct lsb_model {
  lsb_ctx* ctx = nullptr;
  uint32_t V = 0;
  int d = 0;
  float* E = nullptr;     // V x d
  float* bias = nullptr;  // V
};

struct lsb_index {
  lsb_ctx* ctx = nullptr;
  uint32_t V = 0;
  int W = 0, K = 0, u = 0, bits = 0, P = 0, dim = 0;
  bool has_perms = false;
  uint64_t perm_seed = 0, index_seed = 0;
  uint32_t* perms = nullptr;     // P x K (device)
  uint16_t* perms16 = nullptr;   // P x K16 (device, d <= 65535): 16-byte loads of 8 indices
  int K16 = 0;
  uint32_t* word_ids = nullptr;  // W x V (device)
  uint4* slots = nullptr;        // total_slots (device)
  lsb::BandMeta* bands = nullptr;  // W (device)
  std::vector<lsb::BandMeta> bands_host;
  std::vector<uint32_t> perms_host;
  uint32_t total_slots = 0;
  uint32_t max_span = 0;
  uint32_t attempts = 0;

  lsb::IndexView view() const {
    return lsb::IndexView{perms, word_ids, slots, bands, V, W, K, u, bits, P, dim, perms16, K16};
  }
};

// ------------------------------------------------------------- macros
#define LSB_CUDA(expr)                                           \
  do {                                                           \
    cudaError_t _e = (expr);                                     \
    if (_e != cudaSuccess) return lsb::cuda_status(_e, #expr);   \
  } while (0)

#define LSB_LAUNCHED(ctx, what)                                        \
  do {                                                                 \
    (ctx)->launches++;                                                 \
    cudaError_t _e = cudaGetLastError();                               \
    if (_e != cudaSuccess) return lsb::cuda_status(_e, what);          \
  } while (0)

// ------------------------------------------------------ device helpers
namespace lsb {

// Programmatic dependent launch: a step kernel launched with
// launch_pdl() may start (launch, set up shared memory, compute addresses)
// while its predecessor on the stream drains; pdl_wait() blocks until the
// predecessor's results are visible and must precede every read of them.
// Without the launch attribute it returns immediately.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Lets the next kernel on the stream launch once every CTA of this grid has
// called it (or exited); that kernel still waits for this grid's completion
// in pdl_wait(), so placement only affects overlap, never correctness.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(lsb_ctx* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx->pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ uint32_t slot_of(unsigned long long mul, uint32_t lg,
                                            uint32_t key) {
  // CuckooTable::slot_of, include/lshbeam/band_index.hpp:61-64
  return static_cast<uint32_t>((mul * static_cast<unsigned long long>(key)) >> (64 - lg));
}

__device__ __forceinline__ unsigned long long sm64_next(unsigned long long& s) {
  // SplitMix64::next, include/lshbeam/rng.hpp:15-20
  unsigned long long z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long mix_seed_dev(unsigned long long seed,
                                                           unsigned long long stream) {
  unsigned long long s = seed ^ (0xBF58476D1CE4E5B9ull * (stream + 1));
  return sm64_next(s);
}

// Probe band w's two cuckoo slots for `key` with lanes 0 and 1 of the
// calling warp in parallel (the lookup is <= 2 compares, band_index.cpp:73-83);
// all lanes receive (found, start, len).
// Cuckoo lookup of `key` in band w by a group of GS lanes (GS divides 32):
// the group's lanes 0 / 1 probe tables 0 / 1, the hit is broadcast to the
// group. Every lane of the warp must call it (warp-wide ballot / shuffles);
// lanes of a group pass the same (w, key); `active` false = no probe.
template <int GS>
__device__ __forceinline__ bool group_probe(const IndexView& ix, int w, uint32_t key, bool active,
                                            uint32_t& start, uint32_t& len) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (GS - 1), gbase = lane & ~(GS - 1);
  bool hit = false;
  uint4 s = make_uint4(0, 0, 0, 0);
  if (active && gl < 2) {
    const BandMeta m = ix.bands[w];
    const uint32_t cap = 1u << m.lg;
    const uint32_t pos = m.slot_off + (gl ? cap + slot_of(m.mul1, m.lg, key)
                                          : slot_of(m.mul0, m.lg, key));
    s = __ldg(ix.slots + pos);
    hit = s.x == key;
  }
  const unsigned ballot = __ballot_sync(0xffffffffu, hit);
  const unsigned mine = (ballot >> gbase) & 3u;
  const int src = gbase + ((mine & 1u) ? 0 : 1);  // table 0 wins (it is probed first)
  start = __shfl_sync(0xffffffffu, s.y, src);
  len = __shfl_sync(0xffffffffu, s.z, src);
  return mine != 0;
}

__device__ __forceinline__ bool warp_probe(const IndexView& ix, int w, uint32_t key,
                                           uint32_t& start, uint32_t& len) {
  return group_probe<32>(ix, w, key, true, start, len);
}

}  // namespace lsb
