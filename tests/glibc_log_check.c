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

#include "glibc_exp_data.h"
#include "glibc_log_data.h"

static inline uint64_t as_u64(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double as_f64(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

#define LSB_LOG_FN static double restated_log(double x)
#define LSB_EXP_FN static double restated_exp(double x)
#define LSB_EXP_SPECIAL_FN static double restated_exp_special(double x)
#define LSB_EXP_SPECIAL_NAME restated_exp_special
#define LSB_FMA(a, b, c) fma((a), (b), (c))
#define LSB_MUL(a, b) ((a) * (b))
#define LSB_ADD(a, b) ((a) + (b))
#define LSB_SUB(a, b) ((a) - (b))
#define LSB_AS_U64(x) as_u64(x)
#define LSB_AS_F64(u) as_f64(u)
#define LSB_LOAD(t, i) (t)[(i)]
#define LSB_CONST(t, i) (t)[(i)]
#define LSB_EXP_TAB(i) kExpTab[(i)]
#define static_cast_u32(x) ((uint32_t)(x))
#define static_cast_int(x) ((int)(x))
#define static_cast_i64(x) ((int64_t)(x))
#define static_cast_f64(x) ((double)(x))
#include "glibc_log_impl.h"
#include "glibc_exp_impl.h"

void libm_log_array(const float* p, double* out, long n) {
  for (long k = 0; k < n; ++k) out[k] = log((double)p[k]);
}

long restated_log_array(const float* p, double* out, long n) {
  for (long k = 0; k < n; ++k) out[k] = restated_log((double)p[k]);
  return n;
}

void libm_exp_array(const double* x, double* out, long n) {
  for (long k = 0; k < n; ++k) out[k] = exp(x[k]);
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
  /* exp over the softmax's domain x = (double) l - (double) mx <= 0: every
   * difference of two floats is a double; sweep negative doubles uniformly in
   * value over [-800, 0] and uniformly in bits from -2^-60 to -800, plus a
   * uniform sweep of [-1100, 720] (overflow, subnormal results, specials) */
  long ebad = 0, ebad2 = 0;
  const long M = 100000000L;
#pragma omp parallel for reduction(+ : ebad) schedule(static)
  for (long j = 0; j < M; ++j) {
    const double x = (j & 1) ? -800.0 * (double)(j >> 1) / (double)(M / 2)
                             : -as_f64(0x3c30000000000000ull +
                                       (uint64_t)(j >> 1) *
                                           ((0x4089000000000000ull - 0x3c30000000000000ull) / (M / 2)));
    if (as_u64(restated_exp(x)) != as_u64(exp(x))) ++ebad;
  }
#pragma omp parallel for reduction(+ : ebad2) schedule(static)
  for (long j = 0; j < M; ++j) {
    const double x = -1100.0 + 1820.0 * (double)j / (double)M;
    if (as_u64(restated_exp(x)) != as_u64(exp(x))) ++ebad2;
  }
  const double sp[] = {0.0, -0.0, 1e-300, -1e-300, 0x1p-54, -0x1p-55, 709.7, 709.8, -745.1, -745.2,
                       -708.4, -1000.0, 1.0 / 0.0, -1.0 / 0.0};
  for (unsigned k = 0; k < sizeof sp / sizeof sp[0]; ++k)
    if (as_u64(restated_exp(sp[k])) != as_u64(exp(sp[k]))) ++ebad2;
  printf("exp sweeps %ld + %ld mismatches %ld + %ld\n", M, M, ebad, ebad2);
  return (bad || bad2 || ebad || ebad2) ? 1 : 0;
}
