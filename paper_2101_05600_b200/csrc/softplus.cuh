// softplus.cuh — branch-free fp64 log_add for the device recursions.
//
// The reference's log_add (logmath.hpp:19-23) is a + log1p(exp(b - a)) with
// the libm exp/log1p. libdevice's versions cost ~576 cycles of latency per
// call on sm_100a and their special-case branches keep the three chains of
// the CTC recursion from interleaving. This is a straight-line replacement:
// softplus(d) = log1p(exp(d)) for d <= 0 from two 64-entry tables and short
// polynomials (~25 fp64 instructions, no data-dependent branches), accurate
// to ~1 ulp, and a log_add with the reference's exact zero semantics.
// Host-compilable so tests can check it against high-precision values.
#pragma once
#include <cstdint>
#include <cstring>

#include "softplus_tables.h"

#ifndef __CUDACC__
#include <cmath>
#define SP_HD inline
#else
#define SP_HD __host__ __device__ __forceinline__
#endif


// fp64 constants of the polynomials: in device code they are read from a
// __constant__ block, so every DFMA/DADD takes its constant straight from the
// constant bank instead of materialising 64-bit immediates with register
// moves inside the serial chains (that was ~40 of ~146 instructions per chain
// step). Host builds use the literals.
struct SpConsts {
  double k64ln2, ln2_64_hi, ln2_64_lo, ln2_hi, ln2_lo, half, one, c24, c6, c720, c120, c3, mhalf, c5, m4, c7, m6, c9, m8, m10, mone;
};
#if defined(__CUDACC__)
static __constant__ SpConsts c_spk = {SP_64_OVER_LN2, SP_LN2_64_HI, SP_LN2_64_LO, SP_LN2_HI, SP_LN2_LO, 0.5, 1.0, 1.0 / 24.0, 1.0 / 6.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 3.0, -0.5, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 7.0, -1.0 / 6.0, 1.0 / 9.0, -1.0 / 8.0, -1.0 / 10.0, -1.0};
#endif
#ifdef __CUDA_ARCH__
#define SPK(f, lit) (c_spk.f)
#else
#define SPK(f, lit) (lit)
#endif

namespace bl {

struct SpTables {
  double thi[64], tlo[64], inv[64], lh[64], ll[64];
};

SP_HD double sp_bits_to_double(long long b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(b);
#else
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
#endif
}
SP_HD long long sp_double_to_bits(double d) {
#ifdef __CUDA_ARCH__
  return __double_as_longlong(d);
#else
  long long b;
  std::memcpy(&b, &d, sizeof b);
  return b;
#endif
}
SP_HD double sp_pow2(int k) {  // 2^k, 0 below the normal range
  return k < -1022 ? 0.0 : sp_bits_to_double((long long)(k + 1023) << 52);
}
// rint(x) for |x| < 2^51 and the same value as an int, by the 1.5*2^52
// shifter (x + 1.5*2^52 rounds to an integer, round-half-even like rint; its
// low word is the integer): two DADDs instead of FRND + F2I conversions.
SP_HD double sp_rint_int(double x, int* ni) {
  const double t = x + 6755399441055744.0;
  *ni = (int)(unsigned)(sp_double_to_bits(t) & 0xffffffffLL);
  return t - 6755399441055744.0;
}

// log1p(exp(d)) for d <= 0 (any d; very negative d returns ~exp(d) or 0).
// Polynomials are evaluated in Estrin form to shorten the dependent chain.
SP_HD double softplus_neg(double d, const SpTables& tb) {
  // exp(d) = 2^k * 2^(j/64) * exp(r)
  const double dd = fmax(d, -800.0);
  int ni;
  const double n = sp_rint_int(dd * SPK(k64ln2, SP_64_OVER_LN2), &ni);
  double r = fma(-n, SPK(ln2_64_hi, SP_LN2_64_HI), dd);
  r = fma(-n, SPK(ln2_64_lo, SP_LN2_64_LO), r);
  const int j = ni & 63;
  const int k = ni >> 6;  // floor division (arithmetic shift)
  const double th = tb.thi[j];
  const double tl = tb.tlo[j];
  // q = exp(r) - 1 = r + r^2/2 + ... + r^6/720  (Estrin)
  const double r2 = r * r;
  const double a01 = fma(r, SPK(half, 0.5), SPK(one, 1.0));                 // 1 + r/2
  const double a23 = fma(r, SPK(c24, 1.0 / 24.0), SPK(c6, 1.0 / 6.0));    // 1/6 + r/24
  const double a45 = fma(r, SPK(c720, 1.0 / 720.0), SPK(c120, 1.0 / 120.0)); // 1/120 + r/720
  const double r4 = r2 * r2;
  const double lo4 = fma(r2, a23, a01);
  const double q = r * fma(r4, a45, lo4);
  const double e = (th + fma(th, q, tl)) * sp_pow2(k);
  // log1p(e), e in [0, 1]
  const double u = SPK(one, 1.0) + e;
  const double c = e - (u - 1.0);  // rounding error of 1 + e (exact)
  const long long bits = sp_double_to_bits(u);
  const int E = (int)(bits >> 52) - 1023;  // 0 or 1
  const int jj = (int)((bits >> 46) & 63);
  const double m = sp_bits_to_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double iv = tb.inv[jj];
  const double lh = tb.lh[jj], ll = tb.ll[jj];
  const double rr = fma(m, iv, SPK(mone, -1.0));
  // log1p(rr) = rr - rr^2/2 + rr^3/3 - ... - rr^10/10  (Estrin in rr)
  const double s2 = rr * rr;
  const double b0 = fma(rr, SPK(c3, 1.0 / 3.0), SPK(mhalf, -0.5));          // -1/2 + rr/3
  const double b1 = fma(rr, SPK(c5, 1.0 / 5.0), SPK(m4, -1.0 / 4.0));    // -1/4 + rr/5
  const double b2 = fma(rr, SPK(c7, 1.0 / 7.0), -SPK(c6, 1.0 / 6.0));
  const double b3 = fma(rr, SPK(c9, 1.0 / 9.0), SPK(m8, -1.0 / 8.0));
  const double s4 = s2 * s2;
  const double c0 = fma(s2, b1, b0);
  const double c1 = fma(s2, SPK(m10, -1.0 / 10.0), b3);
  const double c2 = fma(s4, fma(s2, c1, b2), c0);       // b0 + s2 b1 + s4 (b2 + s2 b3 + s4 (-1/10))
  const double pl = fma(s2, c2, rr);                    // log1p(rr)
  const double Ed = E ? 1.0 : 0.0;  // E is 0 or 1 here
  const double corr = c * iv * (E ? 0.5 : 1.0);  // c / u
  const double hi = fma(Ed, SPK(ln2_hi, SP_LN2_HI), lh);
  const double lo = fma(Ed, SPK(ln2_lo, SP_LN2_LO), ll) + pl + corr;
  return hi + lo;
}

// exp(d) for d <= 0 (the first half of softplus_neg; 0 below ~-745).
SP_HD double exp_neg(double d, const SpTables& tb) {
  const double dd = fmax(d, -800.0);
  int ni;
  const double n = sp_rint_int(dd * SPK(k64ln2, SP_64_OVER_LN2), &ni);
  double r = fma(-n, SPK(ln2_64_hi, SP_LN2_64_HI), dd);
  r = fma(-n, SPK(ln2_64_lo, SP_LN2_64_LO), r);
  const double th = tb.thi[ni & 63];
  const double tl = tb.tlo[ni & 63];
  const double r2 = r * r;
  const double a01 = fma(r, SPK(half, 0.5), SPK(one, 1.0));
  const double a23 = fma(r, SPK(c24, 1.0 / 24.0), SPK(c6, 1.0 / 6.0));
  const double a45 = fma(r, SPK(c720, 1.0 / 720.0), SPK(c120, 1.0 / 120.0));
  const double r4 = r2 * r2;
  const double q = r * fma(r4, a45, fma(r2, a23, a01));
  return (th + fma(th, q, tl)) * sp_pow2(ni >> 6);
}

// log(x) for a positive normal x (the second half of softplus_neg).
SP_HD double log_pos(double x, const SpTables& tb) {
  const long long bits = sp_double_to_bits(x);
  const int E = (int)(bits >> 52) - 1023;
  const int jj = (int)((bits >> 46) & 63);
  const double m = sp_bits_to_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double iv = tb.inv[jj];
  const double rr = fma(m, iv, SPK(mone, -1.0));
  const double s2 = rr * rr;
  const double b0 = fma(rr, SPK(c3, 1.0 / 3.0), SPK(mhalf, -0.5));
  const double b1 = fma(rr, SPK(c5, 1.0 / 5.0), SPK(m4, -1.0 / 4.0));
  const double b2 = fma(rr, SPK(c7, 1.0 / 7.0), -SPK(c6, 1.0 / 6.0));
  const double b3 = fma(rr, SPK(c9, 1.0 / 9.0), SPK(m8, -1.0 / 8.0));
  const double s4 = s2 * s2;
  const double c0 = fma(s2, b1, b0);
  const double c1 = fma(s2, SPK(m10, -1.0 / 10.0), b3);
  const double c2 = fma(s4, fma(s2, c1, b2), c0);
  const double pl = fma(s2, c2, rr);
  const double hi = fma((double)E, SPK(ln2_hi, SP_LN2_HI), tb.lh[jj]);
  const double lo = fma((double)E, SPK(ln2_lo, SP_LN2_LO), tb.ll[jj]) + pl;
  return hi + lo;
}

// log_add (logmath.hpp:19-23) with the reference's exact zero semantics:
// a zero operand returns the other operand bit-exactly, two zeros return
// kLogZero exactly.
SP_HD double log_add_fast(double a, double b, const SpTables& tb) {
  const double mx = a < b ? b : a;
  const double mn = a < b ? a : b;
  const double s = mx + softplus_neg(mn - mx, tb);
  const double r = mn <= -1e29 ? mx : s;
  return mx <= -1e29 ? -1e30 : r;
}

}  // namespace bl

namespace bl {
// Two independent log_adds with their instruction streams interleaved at the
// source level, so the two serial chains of the CTC recursion overlap.
SP_HD void log_add2(double a1, double b1, double a2, double b2, const SpTables& tb,
                    double* o1, double* o2) {
  const double mx1 = a1 < b1 ? b1 : a1, mn1 = a1 < b1 ? a1 : b1;
  const double mx2 = a2 < b2 ? b2 : a2, mn2 = a2 < b2 ? a2 : b2;
  const double dd1 = fmax(mn1 - mx1, -800.0), dd2 = fmax(mn2 - mx2, -800.0);
  int ni1, ni2;
  const double n1 = sp_rint_int(dd1 * SPK(k64ln2, SP_64_OVER_LN2), &ni1);
  const double n2 = sp_rint_int(dd2 * SPK(k64ln2, SP_64_OVER_LN2), &ni2);
  double r1 = fma(-n1, SPK(ln2_64_hi, SP_LN2_64_HI), dd1), r2 = fma(-n2, SPK(ln2_64_hi, SP_LN2_64_HI), dd2);
  r1 = fma(-n1, SPK(ln2_64_lo, SP_LN2_64_LO), r1);
  r2 = fma(-n2, SPK(ln2_64_lo, SP_LN2_64_LO), r2);
  const double th1 = tb.thi[ni1 & 63], th2 = tb.thi[ni2 & 63];
  const double tl1 = tb.tlo[ni1 & 63], tl2 = tb.tlo[ni2 & 63];
  const double p1 = sp_pow2(ni1 >> 6), p2 = sp_pow2(ni2 >> 6);
  const double q21 = r1 * r1, q22 = r2 * r2;
  const double a011 = fma(r1, SPK(half, 0.5), SPK(one, 1.0)), a012 = fma(r2, SPK(half, 0.5), SPK(one, 1.0));
  const double a231 = fma(r1, SPK(c24, 1.0 / 24.0), SPK(c6, 1.0 / 6.0)), a232 = fma(r2, SPK(c24, 1.0 / 24.0), SPK(c6, 1.0 / 6.0));
  const double a451 = fma(r1, SPK(c720, 1.0 / 720.0), SPK(c120, 1.0 / 120.0)), a452 = fma(r2, SPK(c720, 1.0 / 720.0), SPK(c120, 1.0 / 120.0));
  const double q41 = q21 * q21, q42 = q22 * q22;
  const double lo41 = fma(q21, a231, a011), lo42 = fma(q22, a232, a012);
  const double q1 = r1 * fma(q41, a451, lo41), q2 = r2 * fma(q42, a452, lo42);
  const double e1 = (th1 + fma(th1, q1, tl1)) * p1, e2 = (th2 + fma(th2, q2, tl2)) * p2;
  const double u1 = 1.0 + e1, u2 = SPK(one, 1.0) + e2;
  const double c1 = e1 - (u1 - 1.0), c2 = e2 - (u2 - 1.0);
  const long long bt1 = sp_double_to_bits(u1), bt2 = sp_double_to_bits(u2);
  const int E1 = (int)(bt1 >> 52) - 1023, E2 = (int)(bt2 >> 52) - 1023;
  const int j1 = (int)((bt1 >> 46) & 63), j2 = (int)((bt2 >> 46) & 63);
  const double m1 = sp_bits_to_double((bt1 & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double m2 = sp_bits_to_double((bt2 & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double iv1 = tb.inv[j1], iv2 = tb.inv[j2];
  const double lh1 = tb.lh[j1], lh2 = tb.lh[j2];
  const double ll1 = tb.ll[j1], ll2 = tb.ll[j2];
  const double rr1 = fma(m1, iv1, SPK(mone, -1.0)), rr2 = fma(m2, iv2, SPK(mone, -1.0));
  const double s21 = rr1 * rr1, s22 = rr2 * rr2;
  const double b01 = fma(rr1, SPK(c3, 1.0 / 3.0), SPK(mhalf, -0.5)), b02 = fma(rr2, SPK(c3, 1.0 / 3.0), SPK(mhalf, -0.5));
  const double b11 = fma(rr1, SPK(c5, 1.0 / 5.0), SPK(m4, -1.0 / 4.0)), b12 = fma(rr2, SPK(c5, 1.0 / 5.0), SPK(m4, -1.0 / 4.0));
  const double b21 = fma(rr1, SPK(c7, 1.0 / 7.0), -SPK(c6, 1.0 / 6.0)), b22 = fma(rr2, SPK(c7, 1.0 / 7.0), -SPK(c6, 1.0 / 6.0));
  const double b31 = fma(rr1, SPK(c9, 1.0 / 9.0), SPK(m8, -1.0 / 8.0)), b32 = fma(rr2, SPK(c9, 1.0 / 9.0), SPK(m8, -1.0 / 8.0));
  const double s41 = s21 * s21, s42 = s22 * s22;
  const double c01 = fma(s21, b11, b01), c02 = fma(s22, b12, b02);
  const double c11 = fma(s21, SPK(m10, -1.0 / 10.0), b31), c12 = fma(s22, SPK(m10, -1.0 / 10.0), b32);
  const double d21 = fma(s41, fma(s21, c11, b21), c01), d22 = fma(s42, fma(s22, c12, b22), c02);
  const double pl1 = fma(s21, d21, rr1), pl2 = fma(s22, d22, rr2);
  const double cr1 = c1 * iv1 * (E1 ? 0.5 : 1.0), cr2 = c2 * iv2 * (E2 ? 0.5 : 1.0);
  const double Ed1 = E1 ? 1.0 : 0.0, Ed2 = E2 ? 1.0 : 0.0;  // 0 or 1
  const double h1 = fma(Ed1, SPK(ln2_hi, SP_LN2_HI), lh1), h2 = fma(Ed2, SPK(ln2_hi, SP_LN2_HI), lh2);
  const double l1 = fma(Ed1, SPK(ln2_lo, SP_LN2_LO), ll1) + pl1 + cr1;
  const double l2 = fma(Ed2, SPK(ln2_lo, SP_LN2_LO), ll2) + pl2 + cr2;
  const double s1 = mx1 + (h1 + l1), s2 = mx2 + (h2 + l2);
  const double z1 = mn1 <= -1e29 ? mx1 : s1, z2 = mn2 <= -1e29 ? mx2 : s2;
  *o1 = mx1 <= -1e29 ? -1e30 : z1;
  *o2 = mx2 <= -1e29 ? -1e30 : z2;
}
}  // namespace bl
