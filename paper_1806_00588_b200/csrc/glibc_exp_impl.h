// glibc_exp_impl.h -- the body of glibc's double exp() (>= 2.28, x86-64 FMA
// build: sysdeps/ieee754/dbl-64/e_exp.c from ARM's optimized-routines, as
// GCC contracts it with -mfma), restated with EXPLICIT fused multiply-adds and
// separately rounded products and sums (the LSB_* macros of
// glibc_log_impl.h). Constants: glibc_exp_data.h (kExpHead = 128/ln2, the
// rounding shift 1.5*2^52, -ln2/128 hi/lo, C2..C5; kExpTab = per i < 128 the
// tail and the scale bits of 2^(i/128)).
//
// Two functions: LSB_EXP_SPECIAL_FN (every input, incl. |x| < 2^-54 and
// |x| >= 512: overflow, subnormal results) and LSB_EXP_FN, the common path
// inline, calling the former outside it (kept out of line on the device).
// LSB_EXP_TAB(i) reads kExpTab (global memory, or a shared-memory copy: the
// header may be included again with only LSB_EXP_FN defined).

// x = k ln2/128 + r, |r| <= ln2/256: exp(x) = 2^(k/128) exp(r) ~ scale (1 + tmp);
// sets ki, sbits, tmp
#define LSB_EXP_CORE(x)                                                                  \
  const double shift_ = LSB_CONST(kExpHead, 1);                                           \
  double kd_ = LSB_FMA((x), LSB_CONST(kExpHead, 0), shift_);                              \
  const uint64_t ki = LSB_AS_U64(kd_);                                                   \
  kd_ = LSB_SUB(kd_, shift_);                                                            \
  const double r_ =                                                                      \
      LSB_FMA(kd_, LSB_CONST(kExpHead, 3), LSB_FMA(kd_, LSB_CONST(kExpHead, 2), (x)));     \
  const int idx_ = static_cast_int(2 * (ki % 128));                                      \
  const double tail_ = LSB_AS_F64(LSB_EXP_TAB(idx_));                              \
  uint64_t sbits = LSB_EXP_TAB(idx_ + 1) + (ki << 45);                             \
  const double r2_ = LSB_MUL(r_, r_);                                                    \
  const double p23_ = LSB_FMA(r_, LSB_CONST(kExpHead, 5), LSB_CONST(kExpHead, 4));         \
  const double p45_ = LSB_FMA(r_, LSB_CONST(kExpHead, 7), LSB_CONST(kExpHead, 6));         \
  const double tmp = LSB_FMA(p45_, LSB_MUL(r2_, r2_), LSB_FMA(p23_, r2_, LSB_ADD(r_, tail_)));

#ifdef LSB_EXP_SPECIAL_FN
LSB_EXP_SPECIAL_FN {
  const uint64_t ux = LSB_AS_U64(x);
  const uint32_t abstop = static_cast_u32(ux >> 52) & 0x7ffu;
  if (abstop < 0x3c9u) return LSB_ADD(1.0, x);  // |x| < 2^-54 (and 0): 1 + x
  if (abstop >= 0x409u) {                       // |x| >= 1024, inf, nan
    if (ux == 0xfff0000000000000ull) return 0.0;
    if (abstop >= 0x7ffu) return LSB_ADD(1.0, x);
    return (ux >> 63) ? 0.0 : 1.0 / 0.0;  // underflow to +0 / overflow
  }
  LSB_EXP_CORE(x)
  if (abstop < 0x408u) {  // 2^-54 <= |x| < 512: the common path
    const double scale = LSB_AS_F64(sbits);
    return LSB_FMA(scale, tmp, scale);
  }
  // 512 <= |x| < 1024
  if ((ki & 0x80000000ull) == 0) {  // k > 0: the scale's exponent may overflow
    sbits -= 1009ull << 52;
    const double scale = LSB_AS_F64(sbits);
    return LSB_MUL(LSB_FMA(scale, tmp, scale), 0x1p1009);
  }
  // k < 0: round once before scaling into the subnormal range
  sbits += 1022ull << 52;
  const double scale = LSB_AS_F64(sbits);
  const double st = LSB_MUL(scale, tmp);
  double y = LSB_ADD(scale, st);
  if (y < 1.0) {
    const double hi = LSB_ADD(y, 1.0);
    const double lo = LSB_ADD(LSB_SUB(scale, y), st);
    y = LSB_SUB(LSB_ADD(LSB_ADD(LSB_ADD(LSB_SUB(1.0, hi), y), lo), hi), 1.0);
    if (y == 0.0) return 0.0;
  }
  return LSB_MUL(y, 0x1p-1022);
}
#endif  // LSB_EXP_SPECIAL_FN

LSB_EXP_FN {
  const uint32_t abstop = static_cast_u32(LSB_AS_U64(x) >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) return LSB_EXP_SPECIAL_NAME(x);
  LSB_EXP_CORE(x)
  const double scale = LSB_AS_F64(sbits);
  return LSB_FMA(scale, tmp, scale);
}
#undef LSB_EXP_CORE
