// log1p with the exact rounding of the host's libm, for the ziggurat tail of
// the device Gaussian draw (numpy's `random_standard_normal` calls libm log1p,
// numpy/random/src/distributions/distributions.c).
//
// x86-64 glibc 2.39 resolves log1p (an IFUNC) to its FMA build of the fdlibm
// algorithm (sysdeps/ieee754/dbl-64/s_log1p.c: argument reduction to
// 1+f in [sqrt(2)/2, sqrt(2)], s = f/(2+f), degree-14 odd polynomial in s
// evaluated in Estrin form).  The sequence below states every rounding of that
// build explicitly -- which products the compiler fused (.FMA / .FMS / .FNMA)
// and which it rounded -- so the device result is bit-identical.  nvcc must
// not contract anything here, hence the _rn intrinsics throughout.  Validated
// against the host libm on 2e7 random u in [0, 1) (tools/check_log1p.cu) and
// on the GPU against numpy by tests/test_gpu_rng.py.
#pragma once
#include <stdint.h>

namespace rs {

#ifdef __CUDA_ARCH__
#define RS_L1P_FMA(a, b, c) __fma_rn(a, b, c)
#define RS_L1P_MUL(a, b) __dmul_rn(a, b)
#define RS_L1P_ADD(a, b) __dadd_rn(a, b)
#define RS_L1P_SUB(a, b) __dsub_rn(a, b)
#define RS_L1P_DIV(a, b) __ddiv_rn(a, b)
#define RS_L1P_HI(x) ((int32_t)(__double_as_longlong(x) >> 32))
#define RS_L1P_BITS(x) ((uint64_t)__double_as_longlong(x))
#define RS_L1P_FROM(b) __longlong_as_double((long long)(b))
#else
#define RS_L1P_FMA(a, b, c) __builtin_fma(a, b, c)
#define RS_L1P_MUL(a, b) rs_l1p_mul(a, b)
#define RS_L1P_ADD(a, b) rs_l1p_add(a, b)
#define RS_L1P_SUB(a, b) rs_l1p_sub(a, b)
#define RS_L1P_DIV(a, b) rs_l1p_div(a, b)
#define RS_L1P_HI(x) ((int32_t)(rs_l1p_bits(x) >> 32))
#define RS_L1P_BITS(x) rs_l1p_bits(x)
#define RS_L1P_FROM(b) rs_l1p_from(b)
// out-of-line-ish helpers so the host compiler cannot contract a*b+c
static inline double rs_l1p_mul(double a, double b) { volatile double r = a * b; return r; }
static inline double rs_l1p_add(double a, double b) { volatile double r = a + b; return r; }
static inline double rs_l1p_sub(double a, double b) { volatile double r = a - b; return r; }
static inline double rs_l1p_div(double a, double b) { volatile double r = a / b; return r; }
static inline uint64_t rs_l1p_bits(double x) { uint64_t b; __builtin_memcpy(&b, &x, 8); return b; }
static inline double rs_l1p_from(uint64_t b) { double x; __builtin_memcpy(&x, &b, 8); return x; }
#endif

__host__ __device__ inline double libm_log1p(double x) {
  const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
  const double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2, Lp3 = 0x1.2492494229359p-2,
               Lp4 = 0x1.c71c51d8e78afp-3, Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3,
               Lp7 = 0x1.2f112df3e5244p-3;
  const int32_t hx = RS_L1P_HI(x);
  const int32_t ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0, hfsq;
  if (hx < 0x3FDA827A) {               // x < 0.41422
    if (ax >= 0x3ff00000) {            // x <= -1
      return x == -1.0 ? -__builtin_inf() : __builtin_nan("");
    }
    if (ax < 0x3e200000) {             // |x| < 2^-29
      if (ax < 0x3c900000) return x;   // |x| < 2^-54
      return RS_L1P_FMA(-RS_L1P_MUL(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return RS_L1P_ADD(x, x);
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = RS_L1P_ADD(x, 1.0);
      hu = RS_L1P_HI(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? RS_L1P_SUB(1.0, RS_L1P_SUB(u, x)) : RS_L1P_SUB(x, RS_L1P_SUB(u, 1.0));
      c = RS_L1P_DIV(c, u);
    } else {
      u = x;
      hu = RS_L1P_HI(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    const uint64_t lo = RS_L1P_BITS(u) & 0xffffffffull;
    if (hu < 0x6a09e) {                // normalise u
      u = RS_L1P_FROM(((uint64_t)(uint32_t)(hu | 0x3ff00000) << 32) | lo);
    } else {                           // normalise u/2
      k += 1;
      u = RS_L1P_FROM(((uint64_t)(uint32_t)(hu | 0x3fe00000) << 32) | lo);
      hu = (0x00100000 - hu) >> 2;
    }
    f = RS_L1P_SUB(u, 1.0);
  }
  hfsq = RS_L1P_MUL(RS_L1P_MUL(f, 0.5), f);
  const double dk = (double)k;
  if (hu == 0) {                       // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = RS_L1P_FMA(dk, ln2_lo, c);
      return RS_L1P_FMA(dk, ln2_hi, c);
    }
    const double R = RS_L1P_MUL(RS_L1P_FMA(-f, 0x1.5555555555555p-1, 1.0), hfsq);
    if (k == 0) return RS_L1P_SUB(f, R);
    const double t = RS_L1P_SUB(RS_L1P_SUB(R, RS_L1P_FMA(dk, ln2_lo, c)), f);
    return RS_L1P_FMA(dk, ln2_hi, -t);
  }
  const double s = RS_L1P_DIV(f, RS_L1P_ADD(f, 2.0));
  const double z = RS_L1P_MUL(s, s);
  const double z2 = RS_L1P_MUL(z, z);
  const double R2 = RS_L1P_FMA(z, Lp3, Lp2);
  const double z4 = RS_L1P_MUL(z2, z2);
  const double R3 = RS_L1P_FMA(z, Lp5, Lp4);
  const double z6 = RS_L1P_MUL(z2, z4);
  const double R4 = RS_L1P_FMA(z, Lp7, Lp6);
  double R = RS_L1P_FMA(z, Lp1, RS_L1P_MUL(z2, R2));
  R = RS_L1P_FMA(z4, R3, R);
  R = RS_L1P_FMA(z6, R4, R);
  const double sr = RS_L1P_MUL(s, RS_L1P_ADD(R, hfsq));
  if (k == 0) return RS_L1P_SUB(f, RS_L1P_SUB(hfsq, sr));
  const double t = RS_L1P_SUB(RS_L1P_SUB(hfsq, RS_L1P_ADD(RS_L1P_FMA(dk, ln2_lo, c), sr)), f);
  return RS_L1P_FMA(dk, ln2_hi, -t);
}

}  // namespace rs
