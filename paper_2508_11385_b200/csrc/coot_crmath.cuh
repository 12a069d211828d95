// Correctly rounded EXP and LOG for the fused path (reading R6).
//
// Every node of an expression is rounded to eT (R5), and the oracle's EXP /
// LOG are correctly rounded (f32 via f64 exp / long double log, f64 via
// binary128; pinned in tests/).  So that a composed program stays bit-identical
// to the oracle — later nodes may amplify a 1-ulp difference without bound —
// the device's EXP / LOG return the correctly rounded eT value too.  Ziv's
// strategy, two phases:
//
//  * fast phase: an approximation y = hi + lo with a proven relative error
//    bound eps (f32: one double, eps < 2^-50; f64: a double-double, eps <
//    2^-65).  A rounding test checks that every value within eps |y| rounds to
//    the same eT number; if so that number is the correctly rounded result.
//  * accurate phase (__noinline__, taken with probability ~2^-12 for f64 and
//    ~2^-23 for f32): a double-double evaluation with relative error < 2^-100,
//    rounded once.  For f32 that decides every input (checked exhaustively
//    against the oracle, tests/test_gpu_transcendental.py); for f64 it decides
//    all but inputs whose result lies within 2^-100 of a rounding midpoint —
//    the worst cases of the Lefevre tables, which the oracle's binary128
//    reference cannot decide either (SURVEY §8(c) "parity unpinned").
//
// exp: x = k ln2/128 + r (k = 128 m + j, |r| <= ln2/256), e^x = 2^m 2^(j/128)
// e^r; log: x = 2^e m (m in [0.75, 1.5)), m c_j - 1 = r exactly (|r| < 2^-7.4),
// log x = e ln2 - log c_j + log1p(r).  Tables and split constants:
// tools/gen_crmath_tables.py (mpmath, 400 bits) -> crmath_tables.inc.
//
// The functions are __host__ __device__ so that the same code can be checked
// on the host; device code reads the tables through the read-only path.  The
// build uses -fmad=false: every + - * below rounds on its own, FMAs are
// explicit.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define CRM_HD __host__ __device__ __forceinline__
#define CRM_SLOW static __host__ __device__ __noinline__
#else
#define CRM_HD static inline
#define CRM_SLOW static
#endif

namespace coot {
namespace crm {

#define CRM_CONST static constexpr
#if defined(__CUDACC__)
namespace dev {
#define CRM_TABLE static __device__ const
#include "crmath_tables.inc"
static __device__ const double kExp2Tab[128] = {
#include "exp2_table.inc"
};
#undef CRM_TABLE
}  // namespace dev
#endif
namespace host {
#define CRM_TABLE static const
#include "crmath_tables.inc"
static const double kExp2Tab[128] = {
#include "exp2_table.inc"
};
#undef CRM_TABLE
}  // namespace host
using host::kExpL1;
using host::kExpL2;
using host::kExpL3;
using host::kExpInvL;
using host::kLn2Hi;
using host::kLn2Mid;
using host::kLn2Lo;

#if defined(__CUDA_ARCH__)
#define CRM_TAB(name, i) __ldg(&dev::name[(i)])
#else
#define CRM_TAB(name, i) (host::name[(i)])
#endif

CRM_HD uint64_t bits_of(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
}
CRM_HD double double_of(uint64_t u) {
  double x;
  memcpy(&x, &u, 8);
  return x;
}
CRM_HD double pow2i(int e) {  // 2^e for e in [-1022, 1023]
  return double_of((uint64_t)(e + 1023) << 52);
}

// ---- double-double arithmetic -------------------------------------------------
struct dd {
  double hi, lo;
};
CRM_HD dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
CRM_HD dd fast_two_sum(double a, double b) {  // |a| >= |b| (or a == 0)
  const double s = a + b;
  return {s, b - (s - a)};
}
CRM_HD dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
CRM_HD dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  const dd t = two_sum(x.lo, y.lo);
  s.lo += t.hi;
  s = fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return fast_two_sum(s.hi, s.lo);
}
CRM_HD dd dd_mul(dd x, dd y) {
  dd p = two_prod(x.hi, y.hi);
  p.lo += x.hi * y.lo + x.lo * y.hi;
  return fast_two_sum(p.hi, p.lo);
}
CRM_HD dd dd_mul_d(dd x, double d) {
  dd p = two_prod(x.hi, d);
  p.lo += x.lo * d;
  return fast_two_sum(p.hi, p.lo);
}

// Rounding tests.  (hi, lo) normalised (hi = RN(hi + lo)); the exact value is
// within eps |hi| of hi + lo.  hi is the correctly rounded double iff no
// rounding midpoint lies between: |lo| + eps |hi| < ulp(hi)/2.  With |hi| <
// 2^54 ulp(hi)/2 that holds when hi + lo * (1 + 2^54 eps) rounds back to hi
// (CRlibm's test).  kRoundC64 covers eps = 2^-65 (measured fast-phase error:
// < 2^-68.9 for exp and log over 10^7 random inputs, tools/crmath_check.py).
constexpr double kRoundC64 = 1.0 + 0x1p-11;
CRM_HD bool f64_decided(dd y, double c) { return y.hi + y.lo * c == y.hi; }

// f32 rounding of a double y known to within `margin` double ulps: decided
// unless y lies within margin ulps of an f32 rounding midpoint (the low 29
// mantissa bits 1000...0), or 0 < |y| < 2^-126 (below the f32 normal range
// the f32 grid is coarser than bit 29).  0, inf and the canonical NaN have
// zero low bits and are decided.  Integer-only, branch-free (it runs once per
// element on the hot path).
CRM_HD bool f32_mid_clear(double y, uint32_t margin) {
  const uint32_t lo = (uint32_t)bits_of(y) & 0x1fffffffu;
  return ((lo + (0x10000000u + margin)) & 0x1fffffffu) > 2 * margin;
}
CRM_HD bool f32_decided(double y, uint32_t margin) {
  const uint64_t u = bits_of(y);
  const uint32_t hi = (uint32_t)(u >> 32) & 0x7fffffffu;
  const uint32_t lo = (uint32_t)u & 0x1fffffffu;
  const bool clear = ((lo + (0x10000000u + margin)) & 0x1fffffffu) > 2 * margin;
  return clear && (hi - 1u >= 0x380fffffu);  // hi == 0 (zero) or |y| >= 2^-126
}

// f32 RN(hi + lo) for a normalised double-double: RN(hi) unless hi is itself
// an f32 rounding midpoint, in which case lo's sign breaks the tie.
CRM_HD float f32_of_dd(dd y) {
  const float f = (float)y.hi;
  if (y.lo == 0) return f;
  const double back = (double)f;
  if (back == y.hi) return f;  // hi is an f32 number: lo < ulp/2 cannot move it
  // neighbours of hi in f32 and the midpoint between them
  const float g = (back < y.hi) ? nextafterf(f, INFINITY) : nextafterf(f, -INFINITY);
  const double mid = 0.5 * ((double)f + (double)g);
  if (mid != y.hi) return f;
  // hi is exactly the midpoint: the sign of lo decides (towards g if lo moves
  // the value to g's side)
  return ((g > f) == (y.lo > 0)) ? g : f;
}

// ---- exp -----------------------------------------------------------------------
// Fast phase: e^x = 2^m (hi + lo), relative error < 2^-67 (degree-6 Taylor on
// |r| <= 2^-8.5: truncation < 2^-71.8; r to < 2^-78 (k ln2/128 to 2^-82,
// Fast2Sum of s - t exact unless |s| < |t| < 2^-26, then off by < 2^-79); the
// rest are double roundings of terms below 2^-17 relative).  ~30 FP64 ops.
CRM_HD dd exp_fast(double x, int* m) {
  const double kShift = 0x1.8p52;  // rint trick: k in the low bits of ks
  const double ks = fma(x, kExpInvL, kShift);
  const double kd = ks - kShift;
  const int k = (int)(bits_of(ks) & 0xffffffffu);
  const double s = fma(-kd, kExpL1, x);  // exact: kd * L1 fits 53 bits, s in [2^-43, 2^-8]
  const double t = kd * kExpL2;          // |t| < 2^-26; rounding < 2^-79 (kd L3 < 2^-82: dropped)
  const double rh = s - t;
  const double rl = (s - rh) - t;
  double P = fma(rh, 1.0 / 720, 1.0 / 120);
  P = fma(P, rh, 1.0 / 24);
  P = fma(P, rh, 1.0 / 6);
  P = fma(P, rh, 0.5);
  // e^r - 1 = rh + qlo, qlo = rl + rh rl + rh^2 P(rh)
  const double qlo = fma(rh * rh, P, fma(rh, rl, rl));
  const int j = k & 127;
  const double Th = CRM_TAB(kExpT, 2 * j), Tl = CRM_TAB(kExpT, 2 * j + 1);
  // T (1 + q) = Th + Th rh + (Th qlo + Tl + Tl rh)
  const dd p = two_prod(Th, rh);
  dd y = fast_two_sum(Th, p.hi);
  y.lo += p.lo + fma(Th, qlo, fma(Tl, rh, Tl));
  *m = k >> 7;
  return fast_two_sum(y.hi, y.lo);
}

// v * 2^m by an add to the exponent field (v normal, the result normal)
CRM_HD double scale_exp(double v, int m) {
  const uint64_t u = bits_of(v);
  return double_of(((uint64_t)((uint32_t)(u >> 32) + ((uint32_t)m << 20)) << 32) |
                   (u & 0xffffffffu));
}

// Accurate phase: relative error < 2^-100 (dd Taylor to degree 10 on |r| <=
// 2^-8.5: truncation < 2^-118; ~2^-104 per dd operation).
CRM_SLOW dd exp_accurate(double x, int* m) {
  const double kd = rint(x * kExpInvL);
  const int k = (int)kd;
  const double s = x - kd * kExpL1;
  const dd p2 = two_prod(kd, kExpL2);
  dd r = two_sum(s, -p2.hi);
  r.lo = (r.lo - p2.lo) - kd * kExpL3;
  r = fast_two_sum(r.hi, r.lo);
  dd p = {CRM_TAB(kExpInvFact, 20), CRM_TAB(kExpInvFact, 21)};
  for (int i = 9; i >= 0; --i) {
    p = dd_mul(p, r);
    p = dd_add(p, dd{CRM_TAB(kExpInvFact, 2 * i), CRM_TAB(kExpInvFact, 2 * i + 1)});
  }
  const int j = k & 127;
  *m = k >> 7;
  return dd_mul(dd{CRM_TAB(kExpT, 2 * j), CRM_TAB(kExpT, 2 * j + 1)}, p);
}

// hi * 2^m for a result in the normal range (m in [-1022, 1025])
CRM_HD double scale_normal(double hi, int m) {
  return m > 1000 ? (hi * pow2i(m - 4)) * 16.0 : hi * pow2i(m);
}

// Results below 2^-1021 share the grid 2^-1074 (subnormals and the lowest
// binade): round (hi + lo) 2^(m + 1074) to an integer, ties broken by lo.
CRM_SLOW double exp_tiny(double x) {
  int m;
  const dd y = exp_accurate(x, &m);
  const double q = pow2i(m + 1074 - 60) * 0x1p60;  // m + 1074 in [-2, 60]
  const double qh = y.hi * q, ql = y.lo * q;       // exact scalings
  double n = rint(qh);  // nearest, ties to even
  // a tie in qh alone: the true value lies on lo's side of it
  if (fabs(qh - n) == 0.5 && ql != 0) n = ql > 0 ? qh + 0.5 : qh - 0.5;
  return n * 0x1p-1074;  // exact
}

// RN(a + b + c) for a = RN(a + b) (|b| <= ulp(a)/2) and |c| <= ulp(b)/2:
// a, unless b is exactly half the gap to a's neighbour on b's side — then the
// sign of c breaks the tie (c == 0: the even one).
CRM_HD double round3(double a, double b, double c) {
  if (b == 0) return a;
  const double n = nextafter(a, b > 0 ? INFINITY : -INFINITY);
  if (b != 0.5 * (n - a)) return a;
  if (c == 0) return (bits_of(a) & 1) ? n : a;
  return ((c > 0) == (b > 0)) ? n : a;
}

// 2^-54 < |x| < 2^-26: e^x = 1 + x + x^2/2 + x^3/6 + x^4/24 (+ < 2^-137),
// summed (nearly) exactly so that the hard cases next to 1 (e.g. x = 2^-53:
// e^x = 1 + 2^-53 + 2^-107 + ...) round correctly.
CRM_SLOW double exp_small(double x) {
  const dd s = two_sum(1.0, x);
  dd q = two_prod(x, x);
  q.hi *= 0.5;  // x^2/2 exactly
  q.lo *= 0.5;
  const double c3 = (q.hi * x) * (1.0 / 3);  // x^3/6, |.| < 2^-79, rel. error < 2^-51
  const double c4 = (q.hi * q.hi) * (1.0 / 6);  // x^4/24 < 2^-106
  const dd t = two_sum(s.lo, q.hi);
  const double e2 = ((q.lo + c3) + c4) + t.lo;  // < 2^-78: error < 2^-130
  const dd ab = two_sum(s.hi, t.hi);
  const dd bc = two_sum(ab.lo, e2);
  const dd a = fast_two_sum(ab.hi, bc.hi);
  return round3(a.hi, a.lo, bc.lo);
}

CRM_SLOW double exp_f64_slow(double x) {
  int m;
  const dd y = exp_accurate(x, &m);
  return scale_normal(y.hi, m);
}

// Vectorisable fast phase of cr_exp: straight-line code for any x (clamped
// into the ordinary range); `ok` is false when x needs a special path (NaN,
// |x| < 2^-26, results outside [2^-1021, 2^1024)) or the rounding test fails
// — then cr_exp(x) (the slow, branchy version) must be used.
CRM_HD double exp_fast_ok(double x, bool& ok) {
  const double xc = fmin(fmax(x, -708.0), 709.0);
  int m;
  const dd y = exp_fast(xc, &m);  // y.hi in [0.99, 2), m in [-1022, 1023]
  const double ax = fabs(x);
  const bool one = ax <= 0x1p-54;  // e^x rounds to 1 (zeros included)
  ok = one || ((x >= -708.0) && (x <= 709.0) && (ax >= 0x1p-26) && f64_decided(y, kRoundC64));
  return one ? 1.0 : scale_exp(y.hi, m);
}

// Correctly rounded e^x, binary64.
CRM_HD double cr_exp(double x) {
  if (x != x) return x + x;
  if (x > 709.79) return INFINITY;                     // e^x > 2^1024
  if (x < -745.14) return 0.0;                         // e^x < 2^-1075: rounds to +0
  if (fabs(x) <= 0x1p-54) return 1.0;                  // e^x in (1 - 2^-54, 1 + 2^-54)
  if (fabs(x) < 0x1p-26) return exp_small(x);
  if (x < -708.0) return exp_tiny(x);                  // e^x < 2^-1021
  int m;
  const dd y = exp_fast(x, &m);
  if (f64_decided(y, kRoundC64)) return scale_normal(y.hi, m);
  return exp_f64_slow(x);
}

CRM_SLOW double cr_exp_slow(double x) { return cr_exp(x); }

// ---- f32 exp: one double with error < 2^-49, rounded once (R6) ---------------
// e^x = 2^m * 2^(j/128) * e^r with k = rint(x 128/ln2) = 128 m + j and r = x -
// k ln2/128 (ln2/128 = C1 + C2 by two FMAs: |error| < 2^-60), |r| <= ln2/256 =
// 2^-8.5: e^r - 1 by a degree-4 Taylor polynomial (truncation r^5/120 <
// 2^-49.4 relative), 2^(j/128) correctly rounded: relative error < 2^-49,
// i.e. < 16 ulps of the double — the f32 rounding test uses a 32-ulp margin
// (kF32Margin), so an undecided element (probability ~2^-23) takes the
// double-double accurate phase.  About 10 FP64 operations per element.
// The evaluation for x in [-104, 89] (as a double; any other x gives a
// meaningless but finite-or-NaN value: callers range-check).
CRM_HD double exp_f64_of_f32_core(double x) {
  const double kShift = 0x1.8p52;  // 1.5 * 2^52: rint trick
  const double ks = fma(x, 0x1.71547652b82fep+7, kShift);  // x 128/ln2 + shift
  const double k = ks - kShift;
  const int ki = (int)(bits_of(ks) & 0xffffffffu);
  const double r = fma(-k, 0x1.62e42fefa39efp-8, x);    // C1 = RN(ln2/128)
  const double rr = fma(-k, 0x1.abc9e3b39803fp-63, r);  // C2 = RN(ln2/128 - C1)
  double p = fma(rr, 1.0 / 24.0, 1.0 / 6.0);
  p = fma(p, rr, 0.5);
  p = fma(p, rr, 1.0);
  p = p * rr;  // e^r - 1
  const double t = CRM_TAB(kExp2Tab, ki & 127);
  const double y = fma(t, p, t);  // in [2^-1/256.., 2): scaling by 2^m touches the high word only
  const uint64_t u = bits_of(y);
  return double_of(((uint64_t)((uint32_t)(u >> 32) + ((uint32_t)(ki >> 7) << 20)) << 32) |
                   (u & 0xffffffffu));
}

CRM_HD double exp_f64_of_f32_raw(float xf) {
  const float xc = fminf(fmaxf(xf, -104.0f), 89.0f);  // e^-104 < 2^-150 -> 0; e^89 -> inf
  return exp_f64_of_f32_core((double)xc);  // a NaN input is clamped: the caller handles NaN
}

// Inputs whose f32 e^x is a normal number (e^-87.33 > 2^-126, e^88.72 <
// FLT_MAX): there the fast value's f32 rounding test on its low bits applies.
CRM_HD bool expf_fast_range(float x) { return x >= -87.33f && x <= 88.72f; }

CRM_HD double exp_f64_of_f32(float xf) {
  const double y = exp_f64_of_f32_raw(xf);
  return (xf != xf) ? (double)xf : y;  // NaN passes through
}

CRM_SLOW float exp_f32_slow(float x) {
  if (x < -104.0f) return 0.0f;
  if (x > 89.0f) return INFINITY;
  int m;
  const dd y = exp_accurate((double)x, &m);
  // the scalings are exact (results of f32 inputs stay far from the double
  // range ends)
  const double s = pow2i(m);
  return f32_of_dd(fast_two_sum(y.hi * s, y.lo * s));
}

constexpr uint32_t kF32Margin = 32;  // double ulps (the fast value is within 2^-49: 16 ulps)

// Correctly rounded e^x, binary32.
CRM_HD float cr_expf(float x) {
  if (x != x) return x + x;
  const double y = exp_f64_of_f32_raw(x);
  if (f32_decided(y, kF32Margin)) return (float)y;
  return exp_f32_slow(x);
}

// ---- log -----------------------------------------------------------------------
struct LogRed {
  double ed, r;  // log x = ed ln2 + T[j] + log1p(r), r exact
  int j;
};
// x finite, > 0 (kSub: subnormal x possible; without it x must be normal —
// any other bit pattern gives a meaningless reduction with an in-range table
// index, for callers that range-check)
template <bool kSub = true>
CRM_HD LogRed log_reduce(double x) {
  uint64_t u = bits_of(x);
  int e = (int)(u >> 52) - 1023;
  if (kSub && e == -1023) {  // subnormal: scale into the normal range
    u = bits_of(x * 0x1p54);
    e = (int)(u >> 52) - 1023 - 54;
  }
  double m = double_of((u & 0x000fffffffffffffull) | 0x3ff0000000000000ull);  // [1, 2)
  if (m >= 1.5) {
    m *= 0.5;
    e += 1;
  }
  LogRed red;
  red.j = (int)((m - 0.75) * 256.0);  // m - 0.75 exact (Sterbenz); 0..191
  red.r = fma(m, CRM_TAB(kLogC, red.j), -1.0);  // exact: bits in [2^-60, 2^-8]
  red.ed = (double)e;
  return red;
}

// Fast phase: relative error < 2^-66 (degree 9 in r: truncation < 2^-78
// absolute; e ln2 and T as double-doubles; only terms below 2^-22 are
// summed in plain double).
CRM_HD dd log_fast(double x) {
  const LogRed red = log_reduce(x);
  const double r = red.r;
  const double Th = CRM_TAB(kLogT, 2 * red.j), Tl = CRM_TAB(kLogT, 2 * red.j + 1);
  // ed * Ln2Hi is exact (11 x 42 bits) and, when not 0, larger than |Th| <=
  // 0.41: Fast2Sum is exact
  const dd a = fast_two_sum(red.ed * kLn2Hi, Th);
  const double alo = a.lo + fma(red.ed, kLn2Mid, Tl);
  const dd b = two_sum(a.hi, r);
  const dd sq = two_prod(r, r);
  // |b.hi| >= 2^-8.1 or b.hi = r (e = 0, T = 0) dominates r^2/2: Fast2Sum
  const dd c = fast_two_sum(b.hi, -0.5 * sq.hi);
  double Q = fma(r, 1.0 / 9, -1.0 / 8);
  Q = fma(Q, r, 1.0 / 7);
  Q = fma(Q, r, -1.0 / 6);
  Q = fma(Q, r, 1.0 / 5);
  Q = fma(Q, r, -0.25);
  Q = fma(Q, r, 1.0 / 3);
  const double tail = ((alo + b.lo) + c.lo) + fma(sq.hi * r, Q, -0.5 * sq.lo);
  return fast_two_sum(c.hi, tail);
}

// Accurate phase: relative error < 2^-98 (dd log1p series to r^13, |r| <
// 2^-7.4: truncation < 2^-104 relative).
CRM_SLOW dd log_accurate(double x) {
  const LogRed red = log_reduce(x);
  const double r = red.r;
  dd p = {CRM_TAB(kLogInv, 2 * 12), CRM_TAB(kLogInv, 2 * 12 + 1)};  // 1/13
  for (int k = 11; k >= 0; --k) {
    p = dd_mul_d(p, r);
    p = dd_add(p, dd{CRM_TAB(kLogInv, 2 * k), CRM_TAB(kLogInv, 2 * k + 1)});
  }
  p = dd_mul_d(p, r);  // log1p(r)
  dd L = dd_add(two_prod(red.ed, kLn2Hi), two_prod(red.ed, kLn2Mid));
  L.lo += red.ed * kLn2Lo;
  L = fast_two_sum(L.hi, L.lo);
  const dd T = {CRM_TAB(kLogT, 2 * red.j), CRM_TAB(kLogT, 2 * red.j + 1)};
  return dd_add(dd_add(L, T), p);
}

CRM_SLOW double log_f64_slow(double x) { return log_accurate(x).hi; }

// Vectorisable fast phase of cr_log (see exp_fast_ok): x outside the normal
// positive range (<= 0, subnormal, inf, NaN) is evaluated at 1 and flagged.
CRM_HD double log_fast_ok(double x, bool& ok) {
  const bool normal = (x >= 0x1p-1022) && (x < INFINITY);
  const dd y = log_fast(normal ? x : 1.0);
  ok = normal && f64_decided(y, kRoundC64);
  return y.hi;
}

// Correctly rounded log x, binary64.
CRM_HD double cr_log(double x) {
  if (!(x > 0) || x == INFINITY) {
    if (x == 0) return -INFINITY;
    return (x == INFINITY) ? x : (x - x) / (x - x);  // x < 0 or NaN -> NaN
  }
  const dd y = log_fast(x);
  if (f64_decided(y, kRoundC64)) return y.hi;
  return log_f64_slow(x);
}

CRM_SLOW double cr_log_slow(double x) { return cr_log(x); }

CRM_SLOW float log_f32_slow(float x) { return f32_of_dd(log_accurate((double)x)); }

// f32 log as a double within 2^-51 (within a few double ulps): CUDA's log on
// the device (<= 1 ulp), libm's on the host.  0 -> -inf, < 0 / NaN -> NaN,
// inf -> inf, all exact.
CRM_HD double log_f64_of_f32(float x) { return log((double)x); }

// The hot-path f32 log for x a positive finite f32 (callers range-check):
// log x = e ln2 + T[j] + log1p(r) with the exact reduction of log_reduce (an
// f32 x is a normal double) and log1p(r) = r - r^2/2 + ... - r^8/8 by Horner
// in double (|r| < 2^-7.48: truncation < 2^-67 absolute and < 2^-58 relative
// to r), T[j] and e ln2 rounded: relative error < 2^-49 (16 ulps), the same
// 32-ulp margin as f32 EXP.  ~12 FP64 operations.
CRM_HD double logf_fast_core(float xf) {
  const LogRed red = log_reduce<false>((double)xf);
  const double r = red.r;
  double q = fma(r, -1.0 / 8, 1.0 / 7);
  q = fma(q, r, -1.0 / 6);
  q = fma(q, r, 1.0 / 5);
  q = fma(q, r, -0.25);
  q = fma(q, r, 1.0 / 3);
  q = fma(q, r, -0.5);
  const double l1p = fma(r * r, q, r);  // log1p(r)
  const double th = CRM_TAB(kLogT, 2 * red.j);
  return fma(red.ed, kLn2Hi, th) + fma(red.ed, kLn2Mid, l1p);
}
// positive, finite, and not 1 (log 1 = +0 exactly; the sum above returns it
// too, but 1 sits on the rounding test's edge): the fast phase applies
CRM_HD bool logf_fast_range(float x) { return x > 0.0f && x < INFINITY; }

// Correctly rounded log x, binary32: the double log (within 1 ulp) rounded
// once when the rounding test decides it, else the double-double phase.
CRM_HD float cr_logf(float x) {
  const double y = log_f64_of_f32(x);
  if (f32_decided(y, kF32Margin)) return (float)y;
  return log_f32_slow(x);
}

}  // namespace crm
}  // namespace coot
