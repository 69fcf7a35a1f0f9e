// capi_xchg.cu -- the vocabulary-sharded step's exchange over PEER MEMORY
// instead of collectives (BASELINE cfg 4).
//
// Every rank owns one exchange area in device memory, shared with the other
// ranks through CUDA IPC handles (NVLink / NVSwitch peer memory between the
// GPUs of one node; plain device memory when ranks share a GPU):
//
//   flags  [2][G] u32            per phase, the step sequence number each
//                                source rank last delivered (256-B aligned)
//   max    [G][R] f32            gathered row maxima (phase 1 -> 2)
//   pack   [G][R (1 + B')] u64   gathered row sums + top-B' lists (2 -> 3),
//                                the layout lsb_shard_phase3_packed reads
//
// lsb_shard_step_peer runs phase 1 writing its maxima straight into its own
// slot, then k_xchg_push stores that slot into every peer's area (one CTA per
// destination, 4- / 8-byte stores, a system-scope fence, then the sequence flag
// with release semantics) and k_xchg_wait spins (acquire) until every peer's
// flag for this step has arrived; the same for phase 2's packed slot, then
// phase 3 reads the gathered area in rank order. No host synchronisation and
// no collective call per step: two pushes of ~3 KB and ~105 KB and two flag
// waits (S=64, B=12) instead of two NCCL all-gathers.
//
// Reuse is safe without double buffering: a peer can overwrite my max slot
// for step k+1 only after finishing step k, which needed my phase-2 push of
// step k, issued after my phase 2 consumed the maxima; likewise for pack.
#include <cstring>

#include "batch.cuh"

namespace lsb {
namespace {

constexpr int kXchgMaxG = 64;

// T = the widest store the slot's alignment allows (u32 for the maxima, u64
// for the packed slot: slots are contiguous in rank order, as phase 2 / 3 read them)
template <class T>
__global__ void __launch_bounds__(1024) k_xchg_push(const T* __restrict__ src, size_t n,
                                                   char* const* peer_area, size_t dst_off,
                                                   size_t flag_off, int rank, uint32_t seq) {
  const int peer = blockIdx.x;
  if (peer == rank) return;  // my own slot already holds the data
  char* base = peer_area[peer];
  T* dst = reinterpret_cast<T*>(base + dst_off);
  for (size_t k = threadIdx.x; k < n; k += blockDim.x) dst[k] = src[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // the data before the flag, as seen from any GPU
    uint32_t* flag = reinterpret_cast<uint32_t*>(base + flag_off) + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(flag), "r"(seq) : "memory");
  }
}

__global__ void k_xchg_wait(const uint32_t* flags, int G, int rank, uint32_t seq) {
  const int g = threadIdx.x;
  if (g < G && g != rank) {
    uint32_t v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flags + g) : "memory");
      if (static_cast<int32_t>(v - seq) >= 0) break;  // delivered this step (wrap-safe)
      __nanosleep(64);
    }
  }
  __syncthreads();
}

}  // namespace
}  // namespace lsb

using namespace lsb;

struct lsb_shard_xchg {
  lsb_batch* b = nullptr;
  int G = 0, rank = 0, R = 0, Bp = 0;
  size_t flags_bytes = 0, max_off = 0, pack_off = 0, pack_slot = 0, bytes = 0;
  char* area = nullptr;                   // own exchange area (cudaMalloc: IPC-exportable)
  char* peer[kXchgMaxG] = {};             // every rank's area (own included)
  bool ipc_opened[kXchgMaxG] = {};
  char** d_peer = nullptr;                // device copy of peer[]
  bool dirty = true;                      // peer[] changed since the last upload
  uint32_t seq = 0;
};

extern "C" {

lsb_status lsb_shard_xchg_create(lsb_batch* b, int G, int rank, lsb_shard_xchg** out) {
  if (!b || !out || G < 1 || G > kXchgMaxG || rank < 0 || rank >= G)
    return set_error("lsb_shard_xchg_create: bad arguments"), LSB_EINVAL;
  *out = nullptr;
  LSB_CUDA(cudaSetDevice(b->ctx->device));
  auto* x = new lsb_shard_xchg;
  x->b = b;
  x->G = G;
  x->rank = rank;
  x->R = b->S * b->B;
  x->Bp = lsb_shard_width(b);
  x->flags_bytes = 256;  // 2 x G u32 (G <= 32 fits; padded for alignment)
  if (2 * G * 4 > 256) x->flags_bytes = ((2 * G * 4 + 255) / 256) * 256;
  x->max_off = x->flags_bytes;
  const size_t max_bytes = ((static_cast<size_t>(G) * x->R * 4 + 255) / 256) * 256;
  x->pack_off = x->max_off + max_bytes;
  x->pack_slot = static_cast<size_t>(x->R) * (1 + x->Bp) * 8;
  x->bytes = x->pack_off + static_cast<size_t>(G) * x->pack_slot;
  // every allocation of the step happens here, never inside a step: a
  // cudaMalloc there would synchronise the device while a flag wait spins
  if (lsb_status rc = ensure_shard_scratch(b, G)) {
    delete x;
    return rc;
  }
  cudaError_t e = cudaMalloc(&x->area, x->bytes);
  if (e == cudaSuccess) e = cudaMemset(x->area, 0, x->bytes);
  if (e == cudaSuccess) e = cudaMalloc(&x->d_peer, G * sizeof(char*));
  if (e != cudaSuccess) {
    if (x->area) cudaFree(x->area);
    if (x->d_peer) cudaFree(x->d_peer);
    delete x;
    return cuda_status(e, "lsb_shard_xchg_create");
  }
  x->peer[rank] = x->area;
  *out = x;
  return LSB_OK;
}

lsb_status lsb_shard_xchg_destroy(lsb_shard_xchg* x) {
  if (!x) return LSB_OK;
  cudaSetDevice(x->b->ctx->device);
  cudaStreamSynchronize(x->b->ctx->stream);
  for (int g = 0; g < x->G; ++g)
    if (x->ipc_opened[g]) cudaIpcCloseMemHandle(x->peer[g]);
  if (x->d_peer) cudaFree(x->d_peer);
  if (x->area) cudaFree(x->area);
  delete x;
  return LSB_OK;
}

void* lsb_shard_xchg_area(lsb_shard_xchg* x) { return x ? x->area : nullptr; }

lsb_status lsb_shard_xchg_ipc_handle(lsb_shard_xchg* x, void* handle64) {
  if (!x || !handle64) return set_error("lsb_shard_xchg_ipc_handle: null"), LSB_EINVAL;
  cudaIpcMemHandle_t h;
  LSB_CUDA(cudaIpcGetMemHandle(&h, x->area));
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  std::memcpy(handle64, &h, sizeof(h));
  return LSB_OK;
}

lsb_status lsb_shard_xchg_open_ipc(lsb_shard_xchg* x, int peer, const void* handle64) {
  if (!x || !handle64 || peer < 0 || peer >= x->G || peer == x->rank)
    return set_error("lsb_shard_xchg_open_ipc: bad arguments"), LSB_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* p = nullptr;
  LSB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  x->peer[peer] = static_cast<char*>(p);
  x->ipc_opened[peer] = true;
  x->dirty = true;
  return LSB_OK;
}

lsb_status lsb_shard_xchg_set_peer(lsb_shard_xchg* x, int peer, void* area_dev) {
  if (!x || !area_dev || peer < 0 || peer >= x->G || peer == x->rank)
    return set_error("lsb_shard_xchg_set_peer: bad arguments"), LSB_EINVAL;
  x->peer[peer] = static_cast<char*>(area_dev);
  x->dirty = true;
  return LSB_OK;
}

lsb_status lsb_shard_step_peer(lsb_batch* b, lsb_shard_xchg* x, const lsb_state_dev* in,
                               uint32_t word_base, const lsb_out_dev* out) {
  if (!b || !x || x->b != b || !in || !out)
    return set_error("lsb_shard_step_peer: bad arguments"), LSB_EINVAL;
  for (int g = 0; g < x->G; ++g)
    if (!x->peer[g]) return set_error("lsb_shard_step_peer: peer area not attached"), LSB_EINVAL;
  lsb_ctx* ctx = b->ctx;
  cudaStream_t st = ctx->stream;
  if (x->dirty) {
    LSB_CUDA(cudaMemcpyAsync(x->d_peer, x->peer, x->G * sizeof(char*), cudaMemcpyHostToDevice, st));
    x->dirty = false;
  }
  const uint32_t seq = ++x->seq;
  const int R = x->R;
  uint32_t* flags = reinterpret_cast<uint32_t*>(x->area);
  // phase 1: maxima into my slot, pushed to every peer, wait for theirs
  float* my_max = reinterpret_cast<float*>(x->area + x->max_off) + static_cast<size_t>(x->rank) * R;
  lsb_status rc = lsb_shard_phase1(b, in, my_max);
  if (rc) return rc;
  k_xchg_push<uint32_t><<<x->G, 1024, 0, st>>>(reinterpret_cast<const uint32_t*>(my_max),
                                               static_cast<size_t>(R), x->d_peer,
                                     x->max_off + static_cast<size_t>(x->rank) * R * 4, 0, x->rank,
                                     seq);
  LSB_LAUNCHED(ctx, "k_xchg_push");
  k_xchg_wait<<<1, kXchgMaxG, 0, st>>>(flags, x->G, x->rank, seq);
  LSB_LAUNCHED(ctx, "k_xchg_wait");
  // phase 2: sums + lists into my packed slot, pushed, wait
  char* my_pack = x->area + x->pack_off + static_cast<size_t>(x->rank) * x->pack_slot;
  rc = lsb_shard_phase2(b, in, reinterpret_cast<const float*>(x->area + x->max_off), x->G,
                        word_base, reinterpret_cast<double*>(my_pack),
                        reinterpret_cast<lsb_shard_top*>(my_pack + static_cast<size_t>(R) * 8));
  if (rc) return rc;
  k_xchg_push<unsigned long long><<<x->G, 1024, 0, st>>>(
      reinterpret_cast<const unsigned long long*>(my_pack), x->pack_slot / 8, x->d_peer,
                                     x->pack_off + static_cast<size_t>(x->rank) * x->pack_slot,
                                     static_cast<size_t>(x->G) * 4, x->rank, seq);
  LSB_LAUNCHED(ctx, "k_xchg_push");
  k_xchg_wait<<<1, kXchgMaxG, 0, st>>>(flags + x->G, x->G, x->rank, seq);
  LSB_LAUNCHED(ctx, "k_xchg_wait");
  // phase 3 over the gathered slots (rank order)
  return lsb_shard_phase3_packed(b, in, x->area + x->pack_off, x->G, out);
}

}  // extern "C"
