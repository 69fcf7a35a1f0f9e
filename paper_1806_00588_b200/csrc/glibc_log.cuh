// glibc_log.cuh -- glibc's double log() and exp() on the device, bit for bit
// (glibc_log_impl.h, glibc_exp_impl.h). The reference evaluates its softmax
// exp((double) l - mx) and its beam score cum + log((double) p) with the host
// libm (src/beam_decoder.cpp:46-111); CUDA's own log() / exp() are within
// 1 ulp of them, and log() differed on real inputs (tests/test_gpu_step.py,
// one score of 8).
#pragma once
#include <cstdint>

namespace lsb {
namespace glibc_log_detail {
#define LSB_LOG_CONST static __device__ const
#include "glibc_log_data.h"
#include "glibc_exp_data.h"
#undef LSB_LOG_CONST
}  // namespace glibc_log_detail

#define LSB_LOG_FN static __device__ __forceinline__ double glibc_log(double x)
#define LSB_EXP_FN static __device__ __forceinline__ double glibc_exp(double x)
#define LSB_EXP_SPECIAL_FN static __device__ __noinline__ double glibc_exp_special(double x)
#define LSB_EXP_SPECIAL_NAME glibc_exp_special
#define LSB_FMA(a, b, c) __fma_rn((a), (b), (c))
#define LSB_MUL(a, b) __dmul_rn((a), (b))
#define LSB_ADD(a, b) __dadd_rn((a), (b))
#define LSB_SUB(a, b) __dsub_rn((a), (b))
#define LSB_AS_U64(x) static_cast<uint64_t>(__double_as_longlong(x))
#define LSB_AS_F64(u) __longlong_as_double(static_cast<long long>(u))
#define LSB_LOAD(t, i) __ldg(&glibc_log_detail::t[(i)])
#define LSB_CONST(t, i) (glibc_log_detail::t[(i)])  // constant index: folded
#define LSB_EXP_TAB(i) LSB_LOAD(kExpTab, i)
#define static_cast_u32(x) static_cast<uint32_t>(x)
#define static_cast_int(x) static_cast<int>(x)
#define static_cast_i64(x) static_cast<int64_t>(x)
#define static_cast_f64(x) static_cast<double>(x)
#include "glibc_log_impl.h"
#include "glibc_exp_impl.h"
// exp with kExpTab staged in shared memory (stage_exp_table) by the kernels
// that evaluate it per logit
#undef LSB_EXP_FN
#undef LSB_EXP_SPECIAL_FN
#undef LSB_EXP_TAB
#define LSB_EXP_FN                                                                   \
  static __device__ __forceinline__ double glibc_exp_smem(double x,                   \
                                                           const unsigned long long* tab)
#define LSB_EXP_TAB(i) tab[(i)]
#include "glibc_exp_impl.h"
#undef LSB_EXP_TAB
#undef LSB_LOG_FN
#undef LSB_EXP_FN
#undef LSB_EXP_SPECIAL_FN
#undef LSB_EXP_SPECIAL_NAME
#undef LSB_FMA
#undef LSB_MUL
#undef LSB_ADD
#undef LSB_SUB
#undef LSB_AS_U64
#undef LSB_AS_F64
#undef LSB_LOAD
#undef LSB_CONST
#undef static_cast_u32
#undef static_cast_int
#undef static_cast_i64
#undef static_cast_f64
// Copies kExpTab (2 KB) into a CTA's shared memory; call before a barrier.
__device__ __forceinline__ void stage_exp_table(unsigned long long* tab) {
  for (int k = threadIdx.x; k < 256; k += blockDim.x) tab[k] = __ldg(&glibc_log_detail::kExpTab[k]);
}
}  // namespace lsb
