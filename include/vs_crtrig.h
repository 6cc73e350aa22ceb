/*
 * vs_crtrig.h — correctly rounded double sin/cos, identical on host and device.
 *
 * Why: the reference materialises torsions with Eigen::AngleAxisd, i.e. glibc
 * std::sin/std::cos of the torsion angle (transform.cpp:64, Appendix A item 7
 * of SURVEY.md).  CUDA's sin/cos are not glibc's, so the device needs ONE
 * routine that both the device kernels and the oracle's "device-trig" mode
 * can evaluate bit-identically.  This one returns the correctly rounded
 * (round-to-nearest) result: Cody–Waite reduction by pi/2 in double-double
 * (|x| < 2^20; our torsion angles stay below ~100 rad), then Taylor series in
 * double-double (relative error < 2^-100), rounded once.  glibc 2.39 itself
 * differs from the correctly rounded value on ~0.3% of random inputs
 * (measured, tests/test_crtrig.py), which is the one known source of
 * non-bit-exactness between the GPU path and the glibc-faithful oracle.
 *
 * Only IEEE double add/mul and fma() are used, written in an explicit order,
 * so host code compiled with -ffp-contract=off and device code compiled with
 * -fmad=false produce identical bits.
 */
#ifndef VS_CRTRIG_H
#define VS_CRTRIG_H

#if defined(__CUDACC__)
#define VS_HD __host__ __device__ __forceinline__
#else
#include <cmath>
#define VS_HD inline
#endif

namespace vs_crtrig {

struct dd { double hi, lo; };

VS_HD dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
VS_HD dd fast_two_sum(double a, double b) {
  const double s = a + b;
  const double e = b - (s - a);
  return {s, e};
}
VS_HD dd two_prod(double a, double b) {
  const double p = a * b;
  const double e = fma(a, b, -p);
  return {p, e};
}
VS_HD dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  const double cross = a.hi * b.lo + a.lo * b.hi;
  return fast_two_sum(p.hi, p.lo + cross);
}
VS_HD dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s = fast_two_sum(s.hi, s.lo + t.hi);
  return fast_two_sum(s.hi, s.lo + t.lo);
}

/* (-1)^n/(2n+1)! and (-1)^n/(2n)! as double-double (generated with mpmath,
 * 300-bit precision). */
#define VS_SIN_TERMS 15
#define VS_COS_TERMS 16

#define VS_SIN_TABLE \
  {0x1.0000000000000p+0, 0x0.0p+0}, \
  {-0x1.5555555555555p-3, -0x1.5555555555555p-57}, \
  {0x1.1111111111111p-7, 0x1.1111111111111p-63}, \
  {-0x1.a01a01a01a01ap-13, -0x1.a01a01a01a01ap-73}, \
  {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73}, \
  {-0x1.ae64567f544e4p-26, 0x1.c062e06d1f209p-80}, \
  {0x1.6124613a86d09p-33, 0x1.f28e0cc748ebep-87}, \
  {-0x1.ae7f3e733b81fp-41, -0x1.1d8656b0ee8cbp-97}, \
  {0x1.952c77030ad4ap-49, 0x1.ac981465ddc6cp-103}, \
  {-0x1.2f49b46814157p-57, -0x1.2650f61dbdcb4p-112}, \
  {0x1.71b8ef6dcf572p-66, -0x1.d043ae40c4647p-120}, \
  {-0x1.761b41316381ap-75, 0x1.3423c7d91404fp-130}, \
  {0x1.3f3ccdd165fa9p-84, -0x1.58ddadf344487p-139}, \
  {-0x1.d1ab1c2dccea3p-94, -0x1.054d0c78aea14p-149}, \
  {0x1.259f98b4358adp-103, 0x1.eaf8c39dd9bc5p-157},
#define VS_COS_TABLE \
  {0x1.0000000000000p+0, 0x0.0p+0}, \
  {-0x1.0000000000000p-1, 0x0.0p+0}, \
  {0x1.5555555555555p-5, 0x1.5555555555555p-59}, \
  {-0x1.6c16c16c16c17p-10, 0x1.f49f49f49f49fp-65}, \
  {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76}, \
  {-0x1.27e4fb7789f5cp-22, -0x1.cbbc05b4fa99ap-76}, \
  {0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83}, \
  {-0x1.93974a8c07c9dp-37, -0x1.05d6f8a2efd1fp-92}, \
  {0x1.ae7f3e733b81fp-45, 0x1.1d8656b0ee8cbp-101}, \
  {-0x1.6827863b97d97p-53, -0x1.eec01221a8b0bp-107}, \
  {0x1.e542ba4020225p-62, 0x1.ea72b4afe3c2fp-120}, \
  {-0x1.0ce396db7f853p-70, 0x1.aebcdbd20331cp-124}, \
  {0x1.f2cf01972f578p-80, -0x1.9ada5fcc1ab14p-135}, \
  {-0x1.88e85fc6a4e5ap-89, 0x1.71c37ebd16540p-143}, \
  {0x1.0a18a2635085dp-98, 0x1.b9e2e28e1aa54p-153}, \
  {-0x1.3932c5047d60ep-108, -0x1.832b7b530a627p-162},

/* Coefficient tables: constant memory on the device (uniform index, no
 * branches), plain static arrays on the host; same literals. */
#if defined(__CUDACC__)
static __constant__ double vs_sin_tab_d[VS_SIN_TERMS][2] = {VS_SIN_TABLE};
static __constant__ double vs_cos_tab_d[VS_COS_TERMS][2] = {VS_COS_TABLE};
#endif
static const double vs_sin_tab_h[VS_SIN_TERMS][2] = {VS_SIN_TABLE};
static const double vs_cos_tab_h[VS_COS_TERMS][2] = {VS_COS_TABLE};

VS_HD dd sin_coeff(int n) {
#if defined(__CUDA_ARCH__)
  return {vs_sin_tab_d[n][0], vs_sin_tab_d[n][1]};
#else
  return {vs_sin_tab_h[n][0], vs_sin_tab_h[n][1]};
#endif
}
VS_HD dd cos_coeff(int n) {
#if defined(__CUDA_ARCH__)
  return {vs_cos_tab_d[n][0], vs_cos_tab_d[n][1]};
#else
  return {vs_cos_tab_h[n][0], vs_cos_tab_h[n][1]};
#endif
}

VS_HD dd dd_neg(dd a) { return {-a.hi, -a.lo}; }

/* Taylor series of sin(r), cos(r) in double-double, |r| <= pi/4.  Loops
 * kept rolled: this routine is cold on the device and must not bloat the
 * search kernel's code.  The two Horner recurrences are independent; one loop
 * runs both so their dependency chains overlap (same operations, same order
 * per polynomial). */
VS_HD void sincos_poly(dd r, dd r2, dd *s_out, dd *c_out) {
  dd ps = sin_coeff(VS_SIN_TERMS - 1);
  dd pc = dd_add(dd_mul(cos_coeff(VS_COS_TERMS - 1), r2), cos_coeff(VS_COS_TERMS - 2));
#if defined(__CUDACC__)
#pragma unroll 1
#endif
  for (int n = VS_SIN_TERMS - 2; n >= 0; --n) {
    ps = dd_add(dd_mul(ps, r2), sin_coeff(n));
    pc = dd_add(dd_mul(pc, r2), cos_coeff(n));
  }
  *s_out = dd_mul(ps, r);
  *c_out = pc;
}

/* sin(x) and cos(x) as normalised double-double (relative error < 2^-100);
 * the hi parts are the correctly rounded values. */
VS_HD void sincos_dd(double x, dd *s_out, dd *c_out) {
  if (x == 0.0) {  /* keeps the sign of zero, as sin does */
    *s_out = dd{x, 0.0};
    *c_out = dd{1.0, 0.0};
    return;
  }
  if (!(x - x == 0.0)) {  /* inf or nan */
    *s_out = dd{x - x, 0.0};
    *c_out = dd{x - x, 0.0};
    return;
  }
  /* k = nearest integer to x*2/pi; r = x - k*pi/2 in double-double.
   * pi/2 = P1 + P2 + P3 + P3t, P1..P3 carry 33 significant bits so k*Pi is
   * exact for |k| < 2^20. */
  const double two_over_pi = 0x1.45f306dc9c883p-1;
  const double P1 = 0x1.921fb54400000p+0;
  const double P2 = 0x1.0b4611a600000p-34;
  const double P3 = 0x1.3198a2e000000p-69;
  const double P3t = 0x1.b839a252049c1p-104;
  const double kd = rint(x * two_over_pi);
  const double a = x - kd * P1; /* exact */
  dd r = two_sum(a, -(kd * P2));
  r = dd_add(r, dd{-(kd * P3), 0.0});
  r = dd_add(r, dd{-(kd * P3t), 0.0});
  const dd r2 = dd_mul(r, r);

  dd sr, pc;
  if (fabs(r.hi) < 0x1p-30) {
    /* tiny reduced argument (x next to a multiple of pi/2, as sums of
     * lattice angles and torsion steps often are): the next Taylor terms are
     * below 2^-120 relative */
    sr = dd_add(r, dd_neg(dd_mul(dd_mul(r2, r), dd{0x1.5555555555555p-3, 0x1.5555555555555p-57})));
    pc = dd_add(dd{1.0, 0.0}, dd{-0.5 * r2.hi, -0.5 * r2.lo});
  } else {
    sincos_poly(r, r2, &sr, &pc);
  }
  const long long q = ((long long)kd) & 3;
  if (q == 0) { *s_out = sr; *c_out = pc; }
  else if (q == 1) { *s_out = pc; *c_out = dd_neg(sr); }
  else if (q == 2) { *s_out = dd_neg(sr); *c_out = dd_neg(pc); }
  else { *s_out = dd_neg(pc); *c_out = sr; }
}

/* Correctly rounded sin(x) and cos(x): hi parts of sincos_dd (fast_two_sum
 * normalisation makes hi = RN(hi + lo)). */
VS_HD void sincos_cr(double x, double *s_out, double *c_out) {
  dd s, c;
  sincos_dd(x, &s, &c);
  *s_out = s.hi;
  *c_out = c.hi;
}

/* The search's torsion moves: a' = RN(a + d) and sin/cos(a') as double-
 * double from the double-double sin/cos of a and of d (angle addition, then
 * the exact rounding offset delta = a' - (a + d) to second order).  Relative
 * error ~2^-103 per call (it accumulates slowly along a chain of moves), so
 * the hi parts are the correctly rounded sin/cos of a' except within that
 * distance of a rounding midpoint; tests/test_crtrig.py checks the hi parts
 * against sincos_cr along random move chains.  Returns false when sin or
 * cos of a' is below 2^-8 in magnitude (cancellation): then the caller
 * evaluates sincos_dd(*a_out). */
VS_HD bool sincos_shift(double a, dd sa, dd ca, double d, dd sd, dd cd, double *a_out, dd *s_out, dd *c_out) {
  const dd sum = two_sum(a, d); /* a + d = sum.hi + sum.lo exactly */
  const double del = -sum.lo;   /* a' = (a + d) + del */
  const dd ss = dd_add(dd_mul(sa, cd), dd_mul(ca, sd));         /* sin(a + d) */
  const dd cs = dd_add(dd_mul(ca, cd), dd_neg(dd_mul(sa, sd))); /* cos(a + d) */
  const double h = 0.5 * (del * del);
  /* sin(a') = ss + cs*del - h*ss ; cos(a') = cs - ss*del - h*cs */
  const dd sp = two_prod(cs.hi, del);
  const dd cp = two_prod(ss.hi, del);
  dd sn = dd_add(ss, sp);
  sn = dd_add(sn, dd{cs.lo * del - h * ss.hi, 0.0});
  dd cn = dd_add(cs, dd_neg(cp));
  cn = dd_add(cn, dd{-(ss.lo * del) - h * cs.hi, 0.0});
  *a_out = sum.hi;
  *s_out = sn;
  *c_out = cn;
  /* next to a zero of sin or cos the angle addition cancels: the caller
   * must use sincos_dd(*a_out) instead */
  return !(fabs(sn.hi) < 0x1p-8 || fabs(cn.hi) < 0x1p-8);
}

}  // namespace vs_crtrig

#endif /* VS_CRTRIG_H */
