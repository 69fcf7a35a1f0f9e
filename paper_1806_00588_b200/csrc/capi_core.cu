// capi_core.cu -- error plumbing, context and model handles of the C ABI.
#include <cstdio>
#include <cstring>
#include <string>

#include <cstdlib>
#include <map>
#include <mutex>

#include "lsb_internal.cuh"

namespace lsb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

lsb_status cuda_status(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? LSB_ENOMEM : LSB_ECUDA;
}

lsb_status ensure_smem(const lsb_ctx* ctx, const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return LSB_OK;  // the default limit
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> configured;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = configured[{func, ctx->device}];
  if (bytes <= have) return LSB_OK;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != ctx->device) LSB_CUDA(cudaSetDevice(ctx->device));
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(bytes));
  if (cur >= 0 && cur != ctx->device) cudaSetDevice(cur);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(max dynamic smem)");
  have = bytes;
  return LSB_OK;
}

}  // namespace lsb

using namespace lsb;

extern "C" {

const char* lsb_last_error(void) { return g_last_error.c_str(); }
int lsb_abi_version(void) { return LSB_ABI_VERSION; }

lsb_status lsb_ctx_create(int device, void* stream, lsb_ctx** out) {
  if (!out) {
    set_error("lsb_ctx_create: null out");
    return LSB_EINVAL;
  }
  *out = nullptr;
  int ndev = 0;
  LSB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    set_error("lsb_ctx_create: no such device");
    return LSB_EINVAL;
  }
  LSB_CUDA(cudaSetDevice(device));
  const bool pdl = getenv("LSB_NO_PDL") == nullptr;  // A/B switch for measurements
  cudaDeviceProp prop;
  LSB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("lsb_ctx_create: this build targets sm_100a (B200); device is sm_" +
              std::to_string(prop.major * 10 + prop.minor));
    return LSB_ECUDA;
  }
  auto* c = new lsb_ctx;
  c->pdl = pdl ? 1 : 0;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  {
    // stream-ordered scratch (index builds, stage calls): keep up to 512 MB
    // of freed blocks in the device's default pool instead of unmapping them
    // at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = 512ull << 20;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      return cuda_status(e, "cudaStreamCreate");
    }
    c->own_stream = true;
  }
  cudaError_t e = cudaMalloc(&c->err_dev, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMallocHost(&c->err_host, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(c->err_dev, 0, sizeof(uint32_t), c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    lsb_ctx_destroy(c);
    return cuda_status(e, "lsb_ctx_create");
  }
  *out = c;
  return LSB_OK;
}

lsb_status lsb_ctx_destroy(lsb_ctx* c) {
  if (!c) return LSB_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->join) cudaEventDestroy(c->join);
  if (c->err_dev) cudaFree(c->err_dev);
  if (c->err_host) cudaFreeHost(c->err_host);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return LSB_OK;
}

// Synchronise the context stream and translate the device error word into
// the reference's exception classes. The word is cleared afterwards.
lsb_status lsb_ctx_sync(lsb_ctx* c) {
  if (!c) return LSB_EINVAL;
  LSB_CUDA(cudaMemcpyAsync(c->err_host, c->err_dev, sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, c->stream));
  LSB_CUDA(cudaStreamSynchronize(c->stream));
  const uint32_t err = *c->err_host;
  if (!err) return LSB_OK;
  LSB_CUDA(cudaMemsetAsync(c->err_dev, 0, sizeof(uint32_t), c->stream));
  LSB_CUDA(cudaStreamSynchronize(c->stream));
  if (err & kErrNaN) {
    set_error("hash_matrix: NaN input");
    return LSB_EINVAL;
  }
  if (err & kErrEmptyRow) {
    set_error("softmax_rows: row without finite entries");
    return LSB_EINVAL;
  }
  if (err & kErrEmptyCands) {
    set_error("decode: empty candidate set");
    return LSB_ERUNTIME;
  }
  if (err & kErrCuckoo) {
    set_error("BandIndex: cuckoo build failed");
    return LSB_ERUNTIME;
  }
  set_error("device error word " + std::to_string(err));
  return LSB_ERUNTIME;
}

void* lsb_ctx_stream(lsb_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }
int lsb_ctx_device(lsb_ctx* c) { return c ? c->device : -1; }
int lsb_ctx_sm_count(lsb_ctx* c) { return c ? c->sm_count : 0; }
uint64_t lsb_ctx_launch_count(lsb_ctx* c) { return c ? c->launches : 0; }

static lsb_status model_create_impl(lsb_ctx* ctx, const float* E, uint32_t V, int d,
                                    const float* bias, bool on_dev, lsb_model** out) {
  if (!ctx || !out || !E || d < 1 || V < 1) {
    set_error("lsb_model_create: bad arguments");
    return LSB_EINVAL;
  }
  *out = nullptr;
  LSB_CUDA(cudaSetDevice(ctx->device));
  auto* m = new lsb_model;
  m->ctx = ctx;
  m->V = V;
  m->d = d;
  const size_t nE = static_cast<size_t>(V) * d;
  const cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  cudaError_t e = cudaMalloc(&m->E, nE * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&m->bias, V * sizeof(float));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(m->E, E, nE * sizeof(float), kind, ctx->stream);
  if (e == cudaSuccess)
    e = bias ? cudaMemcpyAsync(m->bias, bias, V * sizeof(float), kind, ctx->stream)
             : cudaMemsetAsync(m->bias, 0, V * sizeof(float), ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    lsb_model_destroy(m);
    return cuda_status(e, "lsb_model_create");
  }
  *out = m;
  return LSB_OK;
}

lsb_status lsb_model_create(lsb_ctx* ctx, const float* E_host, uint32_t vocab, int dim,
                            const float* bias_host, lsb_model** out) {
  return model_create_impl(ctx, E_host, vocab, dim, bias_host, false, out);
}

lsb_status lsb_model_create_dev(lsb_ctx* ctx, const float* E_dev, uint32_t vocab, int dim,
                                const float* bias_dev, lsb_model** out) {
  return model_create_impl(ctx, E_dev, vocab, dim, bias_dev, true, out);
}

lsb_status lsb_model_destroy(lsb_model* m) {
  if (!m) return LSB_OK;
  if (m->E) cudaFree(m->E);
  if (m->bias) cudaFree(m->bias);
  delete m;
  return LSB_OK;
}

const float* lsb_model_embeddings_dev(const lsb_model* m) { return m ? m->E : nullptr; }
uint32_t lsb_model_vocab(const lsb_model* m) { return m ? m->V : 0; }
int lsb_model_dim(const lsb_model* m) { return m ? m->d : 0; }

}  // extern "C"
