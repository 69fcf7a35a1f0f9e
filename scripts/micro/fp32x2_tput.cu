// Microbenchmark: issue rate of the FP32 forms K4 PARITY can use on sm_100a.
//   0: acc = fma2(acc, ONE, fma2(h, e, NEGZ)), ONE/NEGZ kernel params (uniform regs)
//   1: same with ONE/NEGZ forced into regular registers
//   2: scalar FMUL + FADD per lane (two lanes)
//   3: plain FFMA2 chain acc = fma2(h, e, acc) (FAST; 1 instr per 2 MACs)
// Every accumulator has its own e, h comes from shared memory each iteration.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

constexpr int NACC = 16, ITERS = 4096;
template <int MODE>
__global__ void __launch_bounds__(128) k(u64* out, u64 h0, u64 negz, u64 one) {
  u64 acc[NACC], e[NACC];
  __shared__ u64 hs[64];
  if (threadIdx.x < 64) hs[threadIdx.x] = h0 + threadIdx.x;
  for (int i = 0; i < NACC; ++i) { acc[i] = 0; e[i] = h0 * (threadIdx.x + i + 1); }
  if (MODE == 1) {  // launder into regular registers
    asm volatile("mov.b64 %0, %0;" : "+l"(negz));
    asm volatile("mov.b64 %0, %0;" : "+l"(one));
    negz += threadIdx.x >> 10; one += threadIdx.x >> 10;
  }
  __syncthreads();
  for (int it = 0; it < ITERS; ++it) {
    u64 h = hs[it & 63];
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      if (MODE <= 1) acc[i] = f2fma(acc[i], one, f2fma(h, e[i], negz));
      else if (MODE == 3) acc[i] = f2fma(h, e[i], acc[i]);
      else {
        float a0 = __uint_as_float((unsigned)acc[i]), a1 = __uint_as_float((unsigned)(acc[i] >> 32));
        float h0f = __uint_as_float((unsigned)h), h1f = __uint_as_float((unsigned)(h >> 32));
        float e0 = __uint_as_float((unsigned)e[i]), e1 = __uint_as_float((unsigned)(e[i] >> 32));
        a0 = __fadd_rn(a0, __fmul_rn(h0f, e0)); a1 = __fadd_rn(a1, __fmul_rn(h1f, e1));
        acc[i] = (u64)__float_as_uint(a0) | ((u64)__float_as_uint(a1) << 32);
      }
    }
  }
  u64 s = 0;
  for (int i = 0; i < NACC; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  u64* out; cudaMalloc(&out, 148 * 16 * 128 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    for (int ctas = 4; ctas <= 16; ctas *= 2) {
      auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
      int grid = sms * ctas;
      kern<<<grid, 128>>>(out, 0x3f8000013f800001ull, 0x8000000080000000ull, 0x3F8000003F800000ull);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) kern<<<grid, 128>>>(out, 0x3f8000013f800001ull, 0x8000000080000000ull, 0x3F8000003F800000ull);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
      double macs = (double)grid * 128 * ITERS * NACC * 2;
      double lane_ops = macs * (mode == 3 ? 1 : 2);
      printf("mode %d ctas/SM %2d: %.3f ms  %.2f T lane-ops/s  (%.1f lane-ops/SM/clk at 1965 MHz)\n", mode, ctas, ms,
             lane_ops / ms / 1e9, lane_ops / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
