// capi_calib.cu -- live peak of the FP32 pipe that bounds K4 PARITY.
//
// K4 PARITY issues one FMUL + one FADD per MAC in the reference's order as
// paired FP32 ops (fma.rn.f32x2 with -0 / 1.0 operands). This calibration
// kernel runs the same instruction pair on register-resident operands (16
// independent chains per thread, the h operand from shared memory as in K4)
// with 16 CTAs of 128 threads per SM and reports lane-ops per second
// (2 per MAC): the denominator bench.py uses for K4's fp32 roofline, measured
// on the same GPU in the same run (scripts/micro/fp32x2_tput.cu is the
// standalone version; 35.2 T lane-ops/s = 121 per SM per clock on B200).
#include "glibc_log.cuh"
#include "lsb_internal.cuh"

namespace {

__global__ void k_selftest_log(const float* __restrict__ p, double* __restrict__ out, size_t n) {
  for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[k] = lsb::glibc_log(static_cast<double>(p[k]));
}

__global__ void k_selftest_exp(const double* __restrict__ x, double* __restrict__ out, size_t n) {
  for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[k] = lsb::glibc_exp(x[k]);
}

constexpr int kCalChains = 16, kCalIters = 2048;

__global__ void __launch_bounds__(128) k_fp32x2_peak(unsigned long long* out,
                                                     unsigned long long h0,
                                                     unsigned long long negz,
                                                     unsigned long long one) {
  unsigned long long acc[kCalChains], e[kCalChains];
  __shared__ unsigned long long hs[64];
  if (threadIdx.x < 64) hs[threadIdx.x] = h0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kCalChains; ++i) {
    acc[i] = 0;
    e[i] = h0 * (threadIdx.x + i + 1);
  }
  __syncthreads();
  for (int it = 0; it < kCalIters; ++it) {
    const unsigned long long h = hs[it & 63];
#pragma unroll
    for (int i = 0; i < kCalChains; ++i) {
      unsigned long long p, r;
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(h), "l"(e[i]), "l"(negz));
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(acc[i]), "l"(one), "l"(p));
      acc[i] = r;
    }
  }
  unsigned long long s = 0;
#pragma unroll
  for (int i = 0; i < kCalChains; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

extern "C" lsb_status lsb_measure_fp32x2_peak(lsb_ctx* ctx, double* lane_ops_per_s) {
  if (!ctx || !lane_ops_per_s) return lsb::set_error("lsb_measure_fp32x2_peak: null"), LSB_EINVAL;
  LSB_CUDA(cudaSetDevice(ctx->device));
  const int grid = ctx->sm_count * 16;
  unsigned long long* out = nullptr;
  LSB_CUDA(cudaMalloc(&out, static_cast<size_t>(grid) * 128 * 8));
  cudaEvent_t a, b;
  LSB_CUDA(cudaEventCreate(&a));
  LSB_CUDA(cudaEventCreate(&b));
  const unsigned long long h0 = 0x3f8000013f800001ull, negz = 0x8000000080000000ull,
                           one = 0x3F8000003F800000ull;
  k_fp32x2_peak<<<grid, 128, 0, ctx->stream>>>(out, h0, negz, one);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    LSB_CUDA(cudaEventRecord(a, ctx->stream));
    k_fp32x2_peak<<<grid, 128, 0, ctx->stream>>>(out, h0, negz, one);
    LSB_CUDA(cudaEventRecord(b, ctx->stream));
    LSB_CUDA(cudaEventSynchronize(b));
    float ms = 0.0f;
    LSB_CUDA(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  LSB_CUDA(cudaGetLastError());
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  // 2 FFMA2 per chain step = 2 MACs' FMUL + FADD = 4 lane-ops per thread
  const double lane_ops = static_cast<double>(grid) * 128 * kCalIters * kCalChains * 4;
  *lane_ops_per_s = lane_ops / (best * 1e-3);
  return LSB_OK;
}

// Self-test of the device log the beam score uses (glibc_log.cuh): out[k] =
// log((double) p[k]) for n floats in device memory, on the context stream
// (synchronised). tests/test_gpu_glibc_log.py compares it with the host libm.
extern "C" lsb_status lsb_selftest_log(lsb_ctx* ctx, const float* p_dev, double* out_dev,
                                       size_t n) {
  if (!ctx || (n && (!p_dev || !out_dev))) return lsb::set_error("lsb_selftest_log: null"), LSB_EINVAL;
  if (n == 0) return LSB_OK;
  LSB_CUDA(cudaSetDevice(ctx->device));
  k_selftest_log<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(p_dev, out_dev, n);
  LSB_LAUNCHED(ctx, "k_selftest_log");
  LSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return LSB_OK;
}

// Self-test of the device exp the softmax uses (glibc_log.cuh: glibc_exp):
// out[k] = exp(x[k]) for n doubles in device memory (synchronised).
extern "C" lsb_status lsb_selftest_exp(lsb_ctx* ctx, const double* x_dev, double* out_dev,
                                       size_t n) {
  if (!ctx || (n && (!x_dev || !out_dev))) return lsb::set_error("lsb_selftest_exp: null"), LSB_EINVAL;
  if (n == 0) return LSB_OK;
  LSB_CUDA(cudaSetDevice(ctx->device));
  k_selftest_exp<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(x_dev, out_dev, n);
  LSB_LAUNCHED(ctx, "k_selftest_exp");
  LSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return LSB_OK;
}
