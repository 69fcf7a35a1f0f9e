// glibc_log_impl.h -- the body of glibc's double log() (>= 2.28, x86-64 FMA
// build: sysdeps/ieee754/dbl-64/e_log.c from ARM's optimized-routines, as
// GCC contracts it with -mfma), restated with EXPLICIT fused multiply-adds
// and separately rounded products and sums, so no compiler contraction can
// change a bit. The constants are glibc_log_data.h.
//
// The includer defines LSB_LOG_FN (the function head), LSB_FMA(a, b, c) =
// a * b + c rounded once, LSB_MUL / LSB_ADD / LSB_SUB rounded, LSB_AS_U64 /
// LSB_AS_F64 bit casts, LSB_CONST(array, i) for constant indices and
// LSB_LOAD(table, i) for data-dependent ones. One source for the device
// function (glibc_log.cuh) and the CPU check against libm itself
// (tests/glibc_log_check.c: every positive float <= 1, bit for bit).
LSB_LOG_FN {
  uint64_t ix = LSB_AS_U64(x);
  // |x - 1| small: log1p polynomial with an exact split of r^2 / 2
  if (ix - LSB_AS_U64(1.0 - 0x1p-4) < LSB_AS_U64(1.0 + 0x1.09p-4) - LSB_AS_U64(1.0 - 0x1p-4)) {
    if (ix == LSB_AS_U64(1.0)) return 0.0;
    const double r = LSB_SUB(x, 1.0);
    const double r2 = LSB_MUL(r, r), r3 = LSB_MUL(r, r2);
    const double t1 = LSB_FMA(r2, LSB_CONST(kLogPoly1, 3), LSB_FMA(r, LSB_CONST(kLogPoly1, 2), LSB_CONST(kLogPoly1, 1)));
    const double t2 = LSB_FMA(r2, LSB_CONST(kLogPoly1, 6), LSB_FMA(r, LSB_CONST(kLogPoly1, 5), LSB_CONST(kLogPoly1, 4)));
    const double t3 = LSB_FMA(r3, LSB_CONST(kLogPoly1, 10),
                              LSB_FMA(r2, LSB_CONST(kLogPoly1, 9), LSB_FMA(r, LSB_CONST(kLogPoly1, 8), LSB_CONST(kLogPoly1, 7))));
    const double p = LSB_FMA(LSB_FMA(t3, r3, t2), r3, t1);
    const double b0 = LSB_CONST(kLogPoly1, 0);
    const double rhi = LSB_FMA(-r, 0x1p27, LSB_FMA(r, 0x1p27, r));
    const double rlo = LSB_SUB(r, rhi);
    const double rhi2 = LSB_MUL(rhi, rhi);
    const double hi = LSB_FMA(rhi2, b0, r);
    double lo = LSB_FMA(rhi2, b0, LSB_SUB(r, hi));
    lo = LSB_FMA(LSB_ADD(r, rhi), LSB_MUL(rlo, b0), lo);
    return LSB_ADD(hi, LSB_FMA(p, r3, lo));
  }
  const uint32_t top = static_cast_u32(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if ((ix << 1) == 0) return -1.0 / 0.0;                    // +-0
    if (ix == 0x7ff0000000000000ull) return x;                // +inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return (x - x) / (x - x);  // < 0, nan
    ix = LSB_AS_U64(LSB_MUL(x, 0x1p52)) - (52ull << 52);      // subnormal: normalise
  }
  // x = 2^k z, z in [0x1.6p-1, 0x1.6p0); log x = k ln2 + log c + log1p(z/c - 1)
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = static_cast_int((tmp >> 45) % 128);
  const int k = static_cast_int(static_cast_i64(tmp) >> 52);
  const double z = LSB_AS_F64(ix - (tmp & (0xfffull << 52)));
  const double invc = LSB_LOAD(kLogTab, 2 * i), logc = LSB_LOAD(kLogTab, 2 * i + 1);
  const double r = LSB_FMA(z, invc, -1.0);
  const double kd = static_cast_f64(k);
  const double w = LSB_FMA(kd, LSB_CONST(kLogLn2, 0), logc);
  const double r2 = LSB_MUL(r, r);
  const double hi = LSB_ADD(w, r);
  const double lo = LSB_FMA(kd, LSB_CONST(kLogLn2, 1), LSB_ADD(LSB_SUB(w, hi), r));
  const double r3 = LSB_MUL(r, r2);
  const double q = LSB_FMA(r2, LSB_FMA(r, LSB_CONST(kLogPoly, 4), LSB_CONST(kLogPoly, 3)),
                           LSB_FMA(r, LSB_CONST(kLogPoly, 2), LSB_CONST(kLogPoly, 1)));
  return LSB_ADD(LSB_FMA(q, r3, LSB_FMA(r2, LSB_CONST(kLogPoly, 0), lo)), hi);
}
