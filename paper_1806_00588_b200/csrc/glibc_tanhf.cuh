// glibc_tanhf.cuh -- tanhf bit-identical to the host libm the reference links.
//
// The reference's recurrence calls std::tanh(float)
// (/root/reference/proj/src/model_provider.cpp:99), i.e. glibc's tanhf. In
// glibc 2.39 (this image) tanhf and expm1f are the generic fdlibm-derived
// single-precision routines (sysdeps/ieee754/flt-32/s_tanhf.c, s_expm1f.c; no
// ifunc variants: `nm -D libm.so.6` lists both as plain symbols), so their
// results depend only on IEEE single-precision +, -, *, / with
// round-to-nearest. This header restates that published algorithm with every
// operation explicitly rounded (__fadd_rn & co. on the device, so nvcc cannot
// contract a*b+c into an FMA). The same source compiles on the host with
// -ffp-contract=off, where tests/test_tanhf.py compares it with libm's tanhf
// over every float (all 2^32 bit patterns).
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define LSB_HD __host__ __device__ __forceinline__
#else
#define LSB_HD static inline
#endif

namespace lsb_tanhf {

#if defined(__CUDA_ARCH__)
LSB_HD float add(float a, float b) { return __fadd_rn(a, b); }
LSB_HD float sub(float a, float b) { return __fsub_rn(a, b); }
LSB_HD float mul(float a, float b) { return __fmul_rn(a, b); }
LSB_HD float div(float a, float b) { return __fdiv_rn(a, b); }
LSB_HD uint32_t bits(float x) { return __float_as_uint(x); }
LSB_HD float from_bits(uint32_t u) { return __uint_as_float(u); }
#else
LSB_HD float add(float a, float b) { return a + b; }
LSB_HD float sub(float a, float b) { return a - b; }
LSB_HD float mul(float a, float b) { return a * b; }
LSB_HD float div(float a, float b) { return a / b; }
LSB_HD uint32_t bits(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  return u;
}
LSB_HD float from_bits(uint32_t u) {
  float x;
  memcpy(&x, &u, 4);
  return x;
}
#endif

// expm1f for the arguments tanhf passes (|x| < 44, finite): Cody-Waite
// reduction x = k ln2 + r (ln2 split hi/lo), a rational approximation of
// expm1 on the primary range with the scaled coefficients Q1..Q5, then the
// k-dependent reconstruction.
LSB_HD float expm1f(float x) {
  const float ln2_hi = from_bits(0x3f317180u), ln2_lo = from_bits(0x3717f7d1u);
  const float invln2 = from_bits(0x3fb8aa3bu);
  const float Q1 = from_bits(0xbd088889u), Q2 = from_bits(0x3ad00d01u),
              Q3 = from_bits(0xb8a670cdu), Q4 = from_bits(0x36867e54u),
              Q5 = from_bits(0xb457edbbu);
  const float one = 1.0f, tiny = 1.0e-30f;
  uint32_t hx = bits(x);
  const uint32_t xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  if (hx >= 0x4195b844u) {         // |x| >= 27 ln2
    if (hx >= 0x42b17218u) {       // |x| >= 88.72: tanhf never passes these
      if (hx > 0x7f800000u) return add(x, x);
      if (hx == 0x7f800000u) return xsb == 0 ? x : -1.0f;
      if (xsb == 0) return from_bits(0x7f800000u);
    }
    if (xsb != 0) return sub(tiny, one);  // x < -27 ln2: -1
  }
  float hi, lo, c = 0.0f;
  int32_t k;
  if (hx > 0x3eb17218u) {          // |x| > 0.5 ln2
    if (hx < 0x3F851592u) {        // and |x| < 1.5 ln2
      if (xsb == 0) {
        hi = sub(x, ln2_hi);
        lo = ln2_lo;
        k = 1;
      } else {
        hi = add(x, ln2_hi);
        lo = -ln2_lo;
        k = -1;
      }
    } else {
      k = static_cast<int32_t>(add(mul(invln2, x), xsb == 0 ? 0.5f : -0.5f));
      const float t = static_cast<float>(k);
      hi = sub(x, mul(t, ln2_hi));  // t*ln2_hi is exact here
      lo = mul(t, ln2_lo);
    }
    x = sub(hi, lo);
    c = sub(sub(hi, x), lo);
  } else if (hx < 0x33000000u) {   // |x| < 2^-25: x
    const float huge = 1.0e30f;
    const float t = add(huge, x);
    return sub(x, sub(t, add(huge, x)));
  } else {
    k = 0;
  }
  // x is now in the primary range
  const float hfx = mul(0.5f, x);
  const float hxs = mul(x, hfx);
  const float r1 =
      add(one, mul(hxs, add(Q1, mul(hxs, add(Q2, mul(hxs, add(Q3, mul(hxs, add(Q4, mul(hxs, Q5))))))))));
  float t = sub(3.0f, mul(r1, hfx));
  float e = mul(hxs, div(sub(r1, t), sub(6.0f, mul(x, t))));
  if (k == 0) return sub(x, sub(mul(x, e), hxs));  // c is 0
  e = sub(mul(x, sub(e, c)), c);
  e = sub(e, hxs);
  if (k == -1) return sub(mul(0.5f, sub(x, e)), 0.5f);
  if (k == 1) {
    if (x < -0.25f) return mul(-2.0f, sub(e, add(x, 0.5f)));
    return add(one, mul(2.0f, sub(x, e)));
  }
  float y;
  if (k <= -2 || k > 56) {         // exp(x) - 1 directly
    y = sub(one, sub(e, x));
    if (k == 128) {
      y = mul(mul(y, 2.0f), from_bits(0x7f000000u));  // 0x1p127
    } else {
      y = from_bits(bits(y) + (static_cast<uint32_t>(k) << 23));
    }
    return sub(y, one);
  }
  if (k < 23) {
    t = from_bits(0x3f800000u - (0x1000000u >> k));  // 1 - 2^-k
    y = sub(t, sub(e, x));
    y = from_bits(bits(y) + (static_cast<uint32_t>(k) << 23));
  } else {
    t = from_bits(static_cast<uint32_t>(0x7f - k) << 23);  // 2^-k
    y = sub(x, add(e, t));
    y = add(y, one);
    y = from_bits(bits(y) + (static_cast<uint32_t>(k) << 23));
  }
  return y;
}

// tanhf: |x| >= 22 -> +-1; |x| >= 1: 1 - 2/(expm1(2|x|) + 2);
// else -t/(t + 2) with t = expm1(-2|x|); tiny |x| -> x(1 + x).
LSB_HD float tanhf(float x) {
  const float one = 1.0f, two = 2.0f, tiny = 1.0e-30f;
  const uint32_t jx = bits(x);
  const uint32_t ix = jx & 0x7fffffffu;
  if (ix >= 0x7f800000u) {         // inf or NaN
    if (!(jx & 0x80000000u)) return add(div(one, x), one);
    return sub(div(one, x), one);
  }
  float z;
  if (ix < 0x41b00000u) {          // |x| < 22
    if (ix == 0) return x;
    if (ix < 0x24000000u) return mul(x, add(one, x));  // |x| < 2^-55
    const float ax = from_bits(ix);
    if (ix >= 0x3f800000u) {       // |x| >= 1
      const float t = expm1f(mul(two, ax));
      z = sub(one, div(two, add(t, two)));
    } else {
      const float t = expm1f(mul(-two, ax));
      z = div(-t, add(t, two));
    }
  } else {
    z = sub(one, tiny);            // +-1 (inexact)
  }
  return (jx & 0x80000000u) ? -z : z;
}

}  // namespace lsb_tanhf

#undef LSB_HD
