// glibc_log.cuh -- glibc's double log() on the device, bit for bit (see
// glibc_log_impl.h). The beam score is cum + log((double) p) as the
// reference evaluates it with the host libm (src/beam_decoder.cpp's
// expansion); CUDA's own log() is within 1 ulp of it and differed on real
// inputs (tests/test_gpu_step.py, one score of 8).
#pragma once
#include <cstdint>

namespace lsb {
namespace glibc_log_detail {
#define LSB_LOG_CONST static __device__ const
#include "glibc_log_data.h"
#undef LSB_LOG_CONST
}  // namespace glibc_log_detail

#define LSB_LOG_FN static __device__ __forceinline__ double glibc_log(double x)
#define LSB_FMA(a, b, c) __fma_rn((a), (b), (c))
#define LSB_MUL(a, b) __dmul_rn((a), (b))
#define LSB_ADD(a, b) __dadd_rn((a), (b))
#define LSB_SUB(a, b) __dsub_rn((a), (b))
#define LSB_AS_U64(x) static_cast<uint64_t>(__double_as_longlong(x))
#define LSB_AS_F64(u) __longlong_as_double(static_cast<long long>(u))
#define LSB_LOAD(t, i) __ldg(&glibc_log_detail::t[(i)])
#define static_cast_u32(x) static_cast<uint32_t>(x)
#define static_cast_int(x) static_cast<int>(x)
#define static_cast_i64(x) static_cast<int64_t>(x)
#define static_cast_f64(x) static_cast<double>(x)
#include "glibc_log_impl.h"
#undef LSB_LOG_FN
#undef LSB_FMA
#undef LSB_MUL
#undef LSB_ADD
#undef LSB_SUB
#undef LSB_AS_U64
#undef LSB_AS_F64
#undef LSB_LOAD
#undef static_cast_u32
#undef static_cast_int
#undef static_cast_i64
#undef static_cast_f64
}  // namespace lsb
