/* glibc_log_check.c -- CPU check of the device log (csrc/glibc_log_impl.h,
 * the same source, explicit FMAs; compiled with -ffp-contract=off) against
 * the host libm's log() itself, bit for bit.  Test infrastructure
 * (tests/test_glibc_log.py):
 *
 *   glibc_log_check all      every positive float <= 1 (the domain of the
 *                            beam score's log(p)) + a sweep of doubles
 *   libm_log_array(...)      (shared-library use) libm log of n floats, for
 *                            the GPU test's comparison
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "glibc_log_data.h"

static inline uint64_t as_u64(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double as_f64(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

#define LSB_LOG_FN static double restated_log(double x)
#define LSB_FMA(a, b, c) fma((a), (b), (c))
#define LSB_MUL(a, b) ((a) * (b))
#define LSB_ADD(a, b) ((a) + (b))
#define LSB_SUB(a, b) ((a) - (b))
#define LSB_AS_U64(x) as_u64(x)
#define LSB_AS_F64(u) as_f64(u)
#define LSB_LOAD(t, i) (t)[(i)]
#define static_cast_u32(x) ((uint32_t)(x))
#define static_cast_int(x) ((int)(x))
#define static_cast_i64(x) ((int64_t)(x))
#define static_cast_f64(x) ((double)(x))
#include "glibc_log_impl.h"

void libm_log_array(const float* p, double* out, long n) {
  for (long k = 0; k < n; ++k) out[k] = log((double)p[k]);
}

long restated_log_array(const float* p, double* out, long n) {
  for (long k = 0; k < n; ++k) out[k] = restated_log((double)p[k]);
  return n;
}

int main(void) {
  long bad = 0, n = 0, bad2 = 0;
#pragma omp parallel for reduction(+ : bad, n) schedule(static)
  for (long u = 0; u <= 0x3f800000L; ++u) {
    float f;
    uint32_t w = (uint32_t)u;
    memcpy(&f, &w, 4);
    ++n;
    if (as_u64(restated_log((double)f)) != as_u64(log((double)f))) ++bad;
  }
  const uint64_t lo = 1, hi = 0x7ff0000000000000ull, steps = 50000000ull;
#pragma omp parallel for reduction(+ : bad2) schedule(static)
  for (long j = 0; j < (long)steps; ++j) {
    const double x = as_f64(lo + (uint64_t)j * ((hi - lo) / steps));
    const double a = restated_log(x), b = log(x);
    if (as_u64(a) != as_u64(b) && !(isnan(a) && isnan(b))) ++bad2;
  }
  printf("floats %ld mismatches %ld; double sweep %llu mismatches %ld\n", n, bad,
         (unsigned long long)steps, bad2);
  return (bad || bad2) ? 1 : 0;
}
