// dropin_runtime.hpp -- shared plumbing of the C++ drop-in layer: the
// process-wide device context the reference-shaped free functions run on,
// status -> exception mapping (LSB_EINVAL -> std::invalid_argument, like the
// reference; everything else -> std::runtime_error) and RAII owners of the C
// handles. Internal: not installed with include/lshbeam.
#pragma once

#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "lshbeam_b200.h"

namespace lshbeam::detail {

// Device context (device = $LSHBEAM_DEVICE, default 0), created on first use.
lsb_ctx* ctx();
// Serialises drop-in calls on the shared context stream.
std::recursive_mutex& api_mutex();
using Guard = std::lock_guard<std::recursive_mutex>;

[[noreturn]] void raise(lsb_status st, const char* what);
inline void check(lsb_status st, const char* what) {
  if (st != LSB_OK) raise(st, what);
}

struct ModelDeleter {
  void operator()(lsb_model* m) const { lsb_model_destroy(m); }
};
struct IndexDeleter {
  void operator()(lsb_index* i) const { lsb_index_destroy(i); }
};
struct BatchDeleter {
  void operator()(lsb_batch* b) const { lsb_batch_destroy(b); }
};
struct RecurrentDeleter {
  void operator()(lsb_recurrent* r) const { lsb_recurrent_destroy(r); }
};
using ModelPtr = std::unique_ptr<lsb_model, ModelDeleter>;
using BatchPtr = std::unique_ptr<lsb_batch, BatchDeleter>;
using RecurrentPtr = std::unique_ptr<lsb_recurrent, RecurrentDeleter>;

inline std::shared_ptr<lsb_index> share(lsb_index* i) {
  return std::shared_ptr<lsb_index>(i, IndexDeleter{});
}

// Device copy of E (+ optional bias).
ModelPtr upload_model(const float* E, uint32_t vocab, int dim, const float* bias);

// Cached device copies for the per-call reference functions (gather_embeddings,
// step_hidden, decode, build_lsh_index): the reference passes host matrices by
// reference on every call, so the device copy is kept keyed by (host pointer,
// shape) and a content fingerprint (every element up to 1 MB, else 64 Ki
// evenly spaced samples plus the first and last rows), and re-uploaded when
// either changes. A few entries, least recently used first out.
std::shared_ptr<lsb_model> cached_model(const float* E, uint32_t vocab, int dim,
                                        const float* bias);
std::shared_ptr<lsb_recurrent> cached_recurrent(const float* wh, const float* we, int dim);

// Device buffer owner.
struct DevMem {
  void* p = nullptr;
  DevMem() = default;
  explicit DevMem(size_t bytes);
  ~DevMem();
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};
void h2d(void* dst, const void* src, size_t bytes);
void d2h(void* dst, const void* src, size_t bytes);

}  // namespace lshbeam::detail
