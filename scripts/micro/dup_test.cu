typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 dup(float x) { u64 d; asm("mov.b64 %0, {%1, %1};" : "=l"(d) : "f"(x)); return d; }
__global__ void k(const float* __restrict__ E, const u64* __restrict__ H, u64* out, u64 negz, u64 one, int n) {
  extern __shared__ float sm[];
  u64 acc[6][4] = {};
  for (int it = 0; it < n; ++it) {
    u64 e2[4];
    for (int j = 0; j < 4; ++j) e2[j] = dup(sm[threadIdx.x + 33 * j + it * 128]);
    for (int r = 0; r < 6; ++r) {
      u64 h = reinterpret_cast<const u64*>(sm + 4096)[r * 4 + (threadIdx.x & 3) + it * 24];
      for (int j = 0; j < 4; ++j) acc[r][j] = f2fma(acc[r][j], one, f2fma(h, e2[j], negz));
    }
  }
  u64 s = 0; for (int r = 0; r < 6; ++r) for (int j = 0; j < 4; ++j) s ^= acc[r][j];
  out[threadIdx.x] = s;
}
