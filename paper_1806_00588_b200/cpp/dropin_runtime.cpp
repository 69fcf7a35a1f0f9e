// dropin_runtime.cpp -- see dropin_runtime.hpp.
#include "dropin_runtime.hpp"

#include <cstdlib>

namespace lshbeam::detail {

// C++ callers (the reference's CLI, tests, bench) time individual decode
// steps: with CUDA's default lazy module loading the first launch of every
// kernel variant pays a module load inside the timed region (the CLI's
// softmax path read 16.9 ms instead of 2.1 ms over 30 steps). Ask for eager
// loading unless the process chose otherwise; this runs when the library is
// loaded, before the CUDA runtime initialises.
namespace {
struct EagerModuleLoading {
  EagerModuleLoading() { setenv("CUDA_MODULE_LOADING", "EAGER", 0); }
} eager_module_loading;
}  // namespace

namespace {
struct CtxHolder {
  lsb_ctx* c = nullptr;
  ~CtxHolder() {
    if (c) lsb_ctx_destroy(c);
  }
};
}  // namespace

std::recursive_mutex& api_mutex() {
  static std::recursive_mutex m;
  return m;
}

lsb_ctx* ctx() {
  static CtxHolder holder;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("LSHBEAM_DEVICE");
    const int dev = env ? std::atoi(env) : 0;
    lsb_ctx* c = nullptr;
    check(lsb_ctx_create(dev, nullptr, &c), "lshbeam: device context");
    holder.c = c;
  });
  if (!holder.c) throw std::runtime_error("lshbeam: no device context");
  return holder.c;
}

void raise(lsb_status st, const char* what) {
  const char* msg = lsb_last_error();
  std::string m = msg && *msg ? std::string(msg) : std::string(what);
  if (st == LSB_EINVAL) throw std::invalid_argument(m);
  throw std::runtime_error(m);
}

ModelPtr upload_model(const float* E, uint32_t vocab, int dim, const float* bias) {
  lsb_model* m = nullptr;
  check(lsb_model_create(ctx(), E, vocab, dim, bias, &m), "model upload");
  return ModelPtr(m);
}

DevMem::DevMem(size_t bytes) { check(lsb_device_alloc(ctx(), bytes, &p), "device allocation"); }
DevMem::~DevMem() {
  if (p) lsb_device_free(ctx(), p);
}

void h2d(void* dst, const void* src, size_t bytes) {
  check(lsb_copy_to_device(ctx(), dst, src, bytes), "host-to-device copy");
}
void d2h(void* dst, const void* src, size_t bytes) {
  check(lsb_copy_to_host(ctx(), dst, src, bytes), "device-to-host copy");
}

}  // namespace lshbeam::detail
