/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the fused
 * element-wise expression + reduction path computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path under paper_2508_11385_b200/csrc/.
 *
 * What it follows (PAPER.md = /root/reference/PAPER.md):
 *  - Eager evaluation (§3, "standard eager evaluation"): every
 *    node of the expression produces a full temporary array, computed element
 *    by element in the element type eT.  The delayed/fused GPU path must reach
 *    the same values (reading R5: every node rounded to eT).
 *  - eOp (element-wise unary incl. "multiplying matrix by scalar") and
 *    eGlue (element-wise binary on objects of the same dimensions).
 *  - `sum` of all elements (P:168 `float result = sum(A)`, P:517 task 1):
 *    the exact sum, rounded once to eT (reading R10).  Accumulated with
 *    long-double Neumaier compensation in index order, final add in
 *    __float128 then one rounding to eT.
 *  - sum(X,0) / sum(X,1): Armadillo convention (API compatibility P:144-152;
 *    reading R3): dim 0 -> column sums (1 x n_cols), dim 1 -> row sums
 *    (n_rows x 1); column-major storage (reading R2).
 *  - min / max / norm2 / dot: readings R11-R13 in DESIGN.md.
 *  - Input generator: SplitMix64 finaliser over (seed, stream, index)
 *    (DESIGN.md "Input recipe"); fill::randu is uniform [0,1).
 *
 * Pins: every function here is pinned by tests/test_oracle_*.py.
 * Parity unpinned (corners, R6 / R13): f64 EXP / LOG inputs whose
 * result lies within 2^-98 of a rounding midpoint (binary128 cannot decide
 * all of them); f64 VAR / STDDEV whose squared deviations leave the f64 range
 * (the device's shifted f64 squares overflow / flush there, the oracle's
 * long-double ones do not); MIN / MAX with NaN inputs and the sign of a zero
 * extreme.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared (x86-64 SSE2,
 * FLT_EVAL_METHOD == 0) -lquadmath -lm.  See oracle/build.py.
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- element types and opcodes (the oracle's own numbering) ------------ */
/* BF16 / F16 (reading R24): 16-bit storage, every node rounded to the storage
 * format; the roadmap's low-precision types. */
/* E4M3 / E5M2 (reading R25): 8-bit STORAGE types — the expression is evaluated
 * in f32 (every node an f32 node) and each element's value is rounded once to
 * the 8-bit format; reductions consume those 8-bit values and return f32. */
enum { ORC_F32 = 0, ORC_F64 = 1, ORC_U32 = 2, ORC_S64 = 3, ORC_BF16 = 4, ORC_F16 = 5,
       ORC_E4M3 = 6, ORC_E5M2 = 7 };

enum {
  ORC_LOAD = 0, ORC_SCALAR = 1,
  ORC_NEG = 2, ORC_ABS = 3, ORC_SQUARE = 4, ORC_SQRT = 5, ORC_EXP = 6, ORC_LOG = 7,
  ORC_ADD = 8, ORC_SUB = 9, ORC_MUL = 10, ORC_DIV = 11, ORC_MIN = 12, ORC_MAX = 13
};

enum { ORC_ACCU = 0, ORC_RMIN = 1, ORC_RMAX = 2, ORC_MINMAX = 3, ORC_NORM2 = 4 };

enum {
  ORC_E_OK = 0, ORC_E_TYPE = -1, ORC_E_PROGRAM = -2, ORC_E_NOMEM = -3,
  ORC_E_EMPTY = -4, ORC_E_KIND = -5, ORC_E_SHAPE = -6
};

static size_t esize(int type) {
  switch (type) {
    case ORC_F32: return 4;
    case ORC_F64: return 8;
    case ORC_U32: return 4;
    case ORC_S64: return 8;
    case ORC_BF16: return 2;
    case ORC_F16: return 2;
    case ORC_E4M3: return 1;
    case ORC_E5M2: return 1;
  }
  return 0;
}

static int is_half(int type) { return type == ORC_BF16 || type == ORC_F16; }
static int is_fp8(int type) { return type == ORC_E4M3 || type == ORC_E5M2; }
static int is_flt(int type) {
  return type == ORC_F32 || type == ORC_F64 || is_half(type) || is_fp8(type);
}

/* ---- 16-bit float formats ------------------------------------------------
 * bf16: 1 sign, 8 exponent, 7 mantissa bits (bias 127);
 * f16 (IEEE binary16): 1 sign, 5 exponent, 10 mantissa bits (bias 15).
 * half_decode is exact; half_round rounds an exact __float128 value to the
 * format with round-half-to-even (subnormals, overflow to inf), written out
 * with integer arithmetic on the scaled significand. */
static void fmt_of(int type, int* ebits, int* mbits) {
  *ebits = type == ORC_BF16 ? 8 : 5;
  *mbits = type == ORC_BF16 ? 7 : 10;
}

static double half_decode(int type, uint16_t b) {
  int ebits, mbits;
  fmt_of(type, &ebits, &mbits);
  const int bias = (1 << (ebits - 1)) - 1;
  const int sign = b >> 15;
  const int e = (b >> mbits) & ((1 << ebits) - 1);
  const int m = b & ((1 << mbits) - 1);
  double v;
  if (e == (1 << ebits) - 1) v = m ? NAN : INFINITY;
  else if (e == 0) v = ldexp((double)m, 1 - bias - mbits);
  else v = ldexp((double)(m | (1 << mbits)), e - bias - mbits);
  return sign ? -v : v;
}

static uint16_t half_round(int type, __float128 x) {
  int ebits, mbits;
  fmt_of(type, &ebits, &mbits);
  const int bias = (1 << (ebits - 1)) - 1;
  const uint16_t emask = (uint16_t)(((1 << ebits) - 1) << mbits);
  if (isnanq(x)) return (uint16_t)(emask | (1u << (mbits - 1)));
  const uint16_t sign = signbitq(x) ? 0x8000 : 0;
  __float128 a = fabsq(x);
  if (isinfq(a)) return (uint16_t)(sign | emask);
  if (a == 0) return sign;
  int k;
  frexpq(a, &k);               /* a = f * 2^k, f in [0.5, 1) */
  int E = k - 1;               /* 2^E <= a < 2^(E+1) */
  const int emin = 1 - bias;
  const int qe = (E < emin ? emin : E) - mbits;  /* exponent of one ulp */
  const __float128 scaled = ldexpq(a, -qe);       /* exact */
  uint64_t n = (uint64_t)floorq(scaled);
  const __float128 rem = scaled - (__float128)n;
  if (rem > 0.5Q || (rem == 0.5Q && (n & 1))) ++n;
  /* n * 2^qe is the rounded magnitude */
  int field;
  uint64_t mant;
  if (n < (1ull << mbits)) {   /* subnormal (or rounded up to the smallest normal below) */
    field = 0;
    mant = n;
  } else {
    int eq = qe;
    if (n == (2ull << mbits)) { n >>= 1; ++eq; }
    field = eq + mbits + bias;
    mant = n - (1ull << mbits);
    if (field >= (1 << ebits) - 1) return (uint16_t)(sign | emask);  /* overflow */
  }
  return (uint16_t)(sign | ((uint16_t)field << mbits) | (uint16_t)mant);
}

uint16_t orc_half_from_double(int type, double x) { return half_round(type, (__float128)x); }

/* ---- 8-bit float formats (OCP 8-bit floating point) ------------------------
 * E4M3 ("fn"): 1 sign, 4 exponent, 3 mantissa bits, bias 7, NO infinities:
 *   exponent field 15 with mantissa 7 is NaN, so the largest finite is
 *   1.75 * 2^8 = 448; subnormals m * 2^-9.
 * E5M2: 1 sign, 5 exponent, 2 mantissa bits, bias 15, IEEE-style: field 31
 *   is inf (m = 0) / NaN; largest finite 1.75 * 2^15 = 57344; subnormals
 *   m * 2^-16.
 * fp8_round: round-to-nearest-even of the exact value, SATURATING to the
 * largest finite magnitude on overflow and for +-inf (reading R25: the
 * hardware conversion to these formats is the saturating one); NaN -> 0x7f. */
static void fmt8_of(int type, int* ebits, int* mbits) {
  *ebits = type == ORC_E4M3 ? 4 : 5;
  *mbits = type == ORC_E4M3 ? 3 : 2;
}

static double fp8_decode(int type, uint8_t b) {
  int ebits, mbits;
  fmt8_of(type, &ebits, &mbits);
  const int bias = (1 << (ebits - 1)) - 1;
  const int sign = b >> 7;
  const int e = (b >> mbits) & ((1 << ebits) - 1);
  const int m = b & ((1 << mbits) - 1);
  double v;
  if (type == ORC_E4M3 && e == 15 && m == 7) v = NAN;
  else if (type == ORC_E5M2 && e == 31) v = m ? NAN : INFINITY;
  else if (e == 0) v = ldexp((double)m, 1 - bias - mbits);
  else v = ldexp((double)(m | (1 << mbits)), e - bias - mbits);
  return sign ? -v : v;
}

static uint8_t fp8_round(int type, __float128 x) {
  int ebits, mbits;
  fmt8_of(type, &ebits, &mbits);
  const int bias = (1 << (ebits - 1)) - 1;
  /* largest finite: E4M3 0x7e (field 15, m 6), E5M2 0x7b (field 30, m 3) */
  const uint8_t maxfin = type == ORC_E4M3 ? 0x7e : 0x7b;
  if (isnanq(x)) return 0x7f;
  const uint8_t sign = signbitq(x) ? 0x80 : 0;
  __float128 a = fabsq(x);
  if (isinfq(a)) return (uint8_t)(sign | maxfin);
  if (a == 0) return sign;
  int k;
  frexpq(a, &k);
  const int E = k - 1;                            /* 2^E <= a < 2^(E+1) */
  const int emin = 1 - bias;
  const int qe = (E < emin ? emin : E) - mbits;   /* exponent of one ulp */
  const __float128 scaled = ldexpq(a, -qe);
  uint64_t n = (uint64_t)floorq(scaled);
  const __float128 rem = scaled - (__float128)n;
  if (rem > 0.5Q || (rem == 0.5Q && (n & 1))) ++n;
  if (n < (1ull << mbits)) return (uint8_t)(sign | n);   /* subnormal */
  int eq = qe;
  if (n == (2ull << mbits)) { n >>= 1; ++eq; }
  const int field = eq + mbits + bias;
  const uint8_t code = (uint8_t)((field << mbits) | (int)(n - (1ull << mbits)));
  /* beyond the largest finite (incl. E4M3's NaN slot / E5M2's inf field) */
  if (field > (1 << ebits) - 1 || code > maxfin) return (uint8_t)(sign | maxfin);
  return (uint8_t)(sign | code);
}

uint8_t orc_fp8_from_double(int type, double x) { return fp8_round(type, (__float128)x); }
double orc_fp8_to_double(int type, uint8_t b) { return fp8_decode(type, b); }

/* ---- input generator ----------------------------------------------------
 * mix(z): SplitMix64 finaliser (Vigna, splitmix64.c).
 * key = seed ^ (stream * 0xD1B54A32D192ED03)
 * h(i) = mix(key + (i+1) * 0x9E3779B97F4A7C15)   (wrapping uint64)
 * With seed = stream = 0, h(0), h(1), ... is Vigna's splitmix64 sequence from
 * state 0 (pinned in tests/golden/splitmix64_vigna.txt). */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_hash(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t key = seed ^ (stream * 0xD1B54A32D192ED03ULL);
  return mix64(key + (i + 1) * 0x9E3779B97F4A7C15ULL);
}

/* Fill kinds (structured variants for closed forms, DESIGN.md input recipe) */
enum { ORC_FILL_RANDU = 0, ORC_FILL_ONES = 1, ORC_FILL_IOTA = 2, ORC_FILL_MODK = 3,
       ORC_FILL_COLIDX = 4, ORC_FILL_ROWIDX = 5, ORC_FILL_ZEROS = 6 };

/* Element g (global linear index) of a matrix with n_rows rows.  */
static void fill_one(int type, int kind, uint64_t seed, uint64_t stream,
                     uint64_t g, uint64_t n_rows, uint64_t k, void* out, uint64_t idx) {
  uint64_t h = 0, iv = 0;
  switch (kind) {
    case ORC_FILL_RANDU: h = orc_hash(seed, stream, g); break;
    case ORC_FILL_ONES: iv = 1; break;
    case ORC_FILL_IOTA: iv = g; break;
    case ORC_FILL_MODK: iv = g % k; break;
    case ORC_FILL_COLIDX: iv = g / n_rows; break;
    case ORC_FILL_ROWIDX: iv = g % n_rows; break;
    case ORC_FILL_ZEROS: iv = 0; break;
  }
  if (kind == ORC_FILL_RANDU) {
    switch (type) {
      case ORC_F32: ((float*)out)[idx] = (float)(h >> 40) * 0x1p-24f; break;
      case ORC_F64: ((double*)out)[idx] = (double)(h >> 11) * 0x1p-53; break;
      case ORC_U32: ((uint32_t*)out)[idx] = (uint32_t)(h >> 32); break;
      case ORC_S64: ((int64_t*)out)[idx] = (int64_t)h; break;
      /* uniform [0,1) on the format's significand grid (exactly representable) */
      case ORC_BF16: ((uint16_t*)out)[idx] = half_round(type, (__float128)(h >> 56) * 0x1p-8Q); break;
      case ORC_F16: ((uint16_t*)out)[idx] = half_round(type, (__float128)(h >> 53) * 0x1p-11Q); break;
      case ORC_E4M3: ((uint8_t*)out)[idx] = fp8_round(type, (__float128)(h >> 60) * 0x1p-4Q); break;
      case ORC_E5M2: ((uint8_t*)out)[idx] = fp8_round(type, (__float128)(h >> 61) * 0x1p-3Q); break;
    }
  } else {
    switch (type) {
      case ORC_F32: ((float*)out)[idx] = (float)iv; break;
      case ORC_F64: ((double*)out)[idx] = (double)iv; break;
      case ORC_U32: ((uint32_t*)out)[idx] = (uint32_t)iv; break;
      case ORC_S64: ((int64_t*)out)[idx] = (int64_t)iv; break;
      case ORC_BF16:
      case ORC_F16: ((uint16_t*)out)[idx] = half_round(type, (__float128)iv); break;
      case ORC_E4M3:
      case ORC_E5M2: ((uint8_t*)out)[idx] = fp8_round(type, (__float128)iv); break;
    }
  }
}

int orc_fill(int type, int kind, uint64_t seed, uint64_t stream, uint64_t start,
             uint64_t count, uint64_t n_rows, uint64_t k, void* out) {
  if (esize(type) == 0) return ORC_E_TYPE;
  if (n_rows == 0) n_rows = 1;
  if (k == 0) k = 1;
  for (uint64_t i = 0; i < count; ++i)
    fill_one(type, kind, seed, stream, start + i, n_rows, k, out, i);
  return ORC_E_OK;
}

/* ---- per-element semantics (readings R5-R9) -------------------
 * Floating point: IEEE-754 binary32/binary64 round-to-nearest-even, each op
 * computed in eT (compiled with -ffp-contract=off; SSE2, no x87 excess
 * precision).  EXP/LOG are correctly rounded:
 *   f32 exp: (float)exp((double)x)      f32 log: (float)logl((long double)x)
 *   f64 exp: (double)expq((__float128)x) f64 log: (double)logq((__float128)x)
 * (pinned against mpmath in tests/test_oracle_elementwise.py).
 * MIN(a,b) = (b < a) ? b : a ; MAX(a,b) = (a < b) ? b : a   (reading R13).
 * u32: arithmetic mod 2^32.  s64: two's complement mod 2^64, computed in
 * uint64_t (reading R8).  Integer DIV/SQRT/EXP/LOG are rejected (R9). */

static float f32_un(int op, float a) {
  switch (op) {
    case ORC_NEG: return -a;
    case ORC_ABS: return fabsf(a);
    case ORC_SQUARE: return a * a;
    case ORC_SQRT: return sqrtf(a);
    case ORC_EXP: return (float)exp((double)a);
    case ORC_LOG: return (float)logl((long double)a);
  }
  return 0.0f;
}

static double f64_un(int op, double a) {
  switch (op) {
    case ORC_NEG: return -a;
    case ORC_ABS: return fabs(a);
    case ORC_SQUARE: return a * a;
    case ORC_SQRT: return sqrt(a);
    case ORC_EXP: return (double)expq((__float128)a);
    case ORC_LOG: return (double)logq((__float128)a);
  }
  return 0.0;
}

static uint32_t u32_un(int op, uint32_t a) {
  switch (op) {
    case ORC_NEG: return (uint32_t)(0u - a);
    case ORC_ABS: return a;
    case ORC_SQUARE: return (uint32_t)(a * a);
  }
  return 0;
}

static uint64_t s64_un(int op, uint64_t a) {
  switch (op) {
    case ORC_NEG: return 0ULL - a;
    case ORC_ABS: return ((int64_t)a < 0) ? 0ULL - a : a;
    case ORC_SQUARE: return a * a;
  }
  return 0;
}

static float f32_bin(int op, float a, float b) {
  switch (op) {
    case ORC_ADD: return a + b;
    case ORC_SUB: return a - b;
    case ORC_MUL: return a * b;
    case ORC_DIV: return a / b;
    case ORC_MIN: return (b < a) ? b : a;
    case ORC_MAX: return (a < b) ? b : a;
  }
  return 0.0f;
}

static double f64_bin(int op, double a, double b) {
  switch (op) {
    case ORC_ADD: return a + b;
    case ORC_SUB: return a - b;
    case ORC_MUL: return a * b;
    case ORC_DIV: return a / b;
    case ORC_MIN: return (b < a) ? b : a;
    case ORC_MAX: return (a < b) ? b : a;
  }
  return 0.0;
}

static uint32_t u32_bin(int op, uint32_t a, uint32_t b) {
  switch (op) {
    case ORC_ADD: return (uint32_t)(a + b);
    case ORC_SUB: return (uint32_t)(a - b);
    case ORC_MUL: return (uint32_t)(a * b);
    case ORC_MIN: return (b < a) ? b : a;
    case ORC_MAX: return (a < b) ? b : a;
  }
  return 0;
}

static uint64_t s64_bin(int op, uint64_t a, uint64_t b) {
  switch (op) {
    case ORC_ADD: return a + b;
    case ORC_SUB: return a - b;
    case ORC_MUL: return a * b;
    case ORC_MIN: return ((int64_t)b < (int64_t)a) ? b : a;
    case ORC_MAX: return ((int64_t)a < (int64_t)b) ? b : a;
  }
  return 0;
}

/* bf16 / f16 (reading R24): the exact value of the node, rounded once to the
 * 16-bit format.  + - * / sqrt are computed in binary64 — exact or correctly
 * rounded there, and 53 >= 2p + 2 for p = 8 (bf16) and p = 11 (f16), so the
 * second rounding to the format is still the correctly rounded result
 * (Figueroa's double-rounding theorem); exp/log in binary128.  NEG / ABS flip
 * or clear the sign bit; MIN / MAX return one of the inputs. */
static uint16_t h_un(int type, int op, uint16_t a) {
  const double x = half_decode(type, a);
  switch (op) {
    case ORC_NEG: return (uint16_t)(a ^ 0x8000);
    case ORC_ABS: return (uint16_t)(a & 0x7fff);
    case ORC_SQUARE: return half_round(type, (__float128)(x * x));
    case ORC_SQRT: return half_round(type, (__float128)sqrt(x));
    case ORC_EXP: return half_round(type, expq((__float128)x));
    case ORC_LOG: return half_round(type, logq((__float128)x));
  }
  return 0;
}

static uint16_t h_bin(int type, int op, uint16_t a, uint16_t b) {
  const double x = half_decode(type, a), y = half_decode(type, b);
  switch (op) {
    case ORC_ADD: return half_round(type, (__float128)(x + y));
    case ORC_SUB: return half_round(type, (__float128)(x - y));
    case ORC_MUL: return half_round(type, (__float128)(x * y));
    case ORC_DIV: return half_round(type, (__float128)(x / y));
    case ORC_MIN: return (y < x) ? b : a;
    case ORC_MAX: return (x < y) ? b : a;
  }
  return 0;
}

static int is_unary(int op) { return op >= ORC_NEG && op <= ORC_LOG; }
static int is_binary(int op) { return op >= ORC_ADD && op <= ORC_MAX; }
static int legal_for(int type, int op) {
  if (type == ORC_U32 || type == ORC_S64)
    return !(op == ORC_SQRT || op == ORC_EXP || op == ORC_LOG || op == ORC_DIV);
  return 1;
}

/* Unary op over a whole temporary: dst[i] = f(a[i]). */
static void apply_unary(int type, int op, uint64_t n, const void* a, void* dst) {
  for (uint64_t i = 0; i < n; ++i) {
    switch (type) {
      case ORC_F32: ((float*)dst)[i] = f32_un(op, ((const float*)a)[i]); break;
      case ORC_F64: ((double*)dst)[i] = f64_un(op, ((const double*)a)[i]); break;
      case ORC_U32: ((uint32_t*)dst)[i] = u32_un(op, ((const uint32_t*)a)[i]); break;
      case ORC_S64: ((uint64_t*)dst)[i] = s64_un(op, ((const uint64_t*)a)[i]); break;
      case ORC_BF16:
      case ORC_F16: ((uint16_t*)dst)[i] = h_un(type, op, ((const uint16_t*)a)[i]); break;
    }
  }
}

/* Binary op over whole temporaries: dst[i] = f(a[i], b[i]). */
static void apply_binary(int type, int op, uint64_t n, const void* a, const void* b, void* dst) {
  for (uint64_t i = 0; i < n; ++i) {
    switch (type) {
      case ORC_F32:
        ((float*)dst)[i] = f32_bin(op, ((const float*)a)[i], ((const float*)b)[i]);
        break;
      case ORC_F64:
        ((double*)dst)[i] = f64_bin(op, ((const double*)a)[i], ((const double*)b)[i]);
        break;
      case ORC_U32:
        ((uint32_t*)dst)[i] = u32_bin(op, ((const uint32_t*)a)[i], ((const uint32_t*)b)[i]);
        break;
      case ORC_S64:
        ((uint64_t*)dst)[i] = s64_bin(op, ((const uint64_t*)a)[i], ((const uint64_t*)b)[i]);
        break;
      case ORC_BF16:
      case ORC_F16:
        ((uint16_t*)dst)[i] = h_bin(type, op, ((const uint16_t*)a)[i], ((const uint16_t*)b)[i]);
        break;
    }
  }
}

/* ---- eager evaluation of a postfix program ------------------------------
 * Postfix semantics: LOAD k pushes operand k; SCALAR k pushes scalar k
 * (broadcast, materialised as a full temporary); a unary op pops a and pushes
 * f(a); a binary op pops b (top) then a and pushes a OP b.  Every step
 * allocates a NEW full temporary (the eager evaluation of P:366-367).  The
 * program must leave exactly one entry, which is copied to `out`.
 * `scalars` is an array of n_scalars values of eT. */
#define ORC_MAX_STACK 64

int orc_eval(int type, uint64_t n, const void* const* operands, int n_operands,
             const void* scalars, int n_scalars, const int* ops, const int* args,
             int n_instr, void* out);

/* 8-bit storage types (reading R25): decode every operand exactly to f32,
 * evaluate the program as an f32 program (scalars are f32), round each
 * element's final value once to the 8-bit format. */
static int eval_fp8(int type, uint64_t n, const void* const* operands, int n_operands,
                    const void* scalars, int n_scalars, const int* ops, const int* args,
                    int n_instr, void* out) {
  if (n_operands < 0 || n_operands > ORC_MAX_STACK) return ORC_E_PROGRAM;
  size_t fb = (size_t)(n ? n : 1) * sizeof(float);
  float* dec[ORC_MAX_STACK] = {0};
  const void* cdec[ORC_MAX_STACK] = {0};
  float* res = (float*)malloc(fb);
  int rc = res ? ORC_E_OK : ORC_E_NOMEM;
  int made = 0;
  for (; rc == ORC_E_OK && made < n_operands; ++made) {
    dec[made] = (float*)malloc(fb);
    if (!dec[made]) { rc = ORC_E_NOMEM; break; }
    for (uint64_t i = 0; i < n; ++i)
      dec[made][i] = (float)fp8_decode(type, ((const uint8_t*)operands[made])[i]);
    cdec[made] = dec[made];
  }
  if (rc == ORC_E_OK)
    rc = orc_eval(ORC_F32, n, cdec, n_operands, scalars, n_scalars, ops, args, n_instr, res);
  if (rc == ORC_E_OK)
    for (uint64_t i = 0; i < n; ++i) ((uint8_t*)out)[i] = fp8_round(type, (__float128)res[i]);
  for (int k = 0; k < made; ++k) free(dec[k]);
  free(res);
  return rc;
}

int orc_eval(int type, uint64_t n, const void* const* operands, int n_operands,
             const void* scalars, int n_scalars, const int* ops, const int* args,
             int n_instr, void* out) {
  size_t es = esize(type);
  if (es == 0) return ORC_E_TYPE;
  if (is_fp8(type))
    return eval_fp8(type, n, operands, n_operands, scalars, n_scalars, ops, args, n_instr, out);
  void* stack[ORC_MAX_STACK];
  int sp = 0;
  int rc = ORC_E_OK;
  size_t bytes = (size_t)n * es;
  size_t alloc = bytes ? bytes : 1;
  for (int pc = 0; pc < n_instr; ++pc) {
    int op = ops[pc], arg = args[pc];
    if (!legal_for(type, op)) { rc = ORC_E_PROGRAM; goto fail; }
    if (op == ORC_LOAD) {
      if (arg < 0 || arg >= n_operands || sp >= ORC_MAX_STACK) { rc = ORC_E_PROGRAM; goto fail; }
      void* t = malloc(alloc);
      if (!t) { rc = ORC_E_NOMEM; goto fail; }
      if (bytes) memcpy(t, operands[arg], bytes);
      stack[sp++] = t;
    } else if (op == ORC_SCALAR) {
      if (arg < 0 || arg >= n_scalars || sp >= ORC_MAX_STACK) { rc = ORC_E_PROGRAM; goto fail; }
      void* t = malloc(alloc);
      if (!t) { rc = ORC_E_NOMEM; goto fail; }
      for (uint64_t i = 0; i < n; ++i)
        memcpy((char*)t + i * es, (const char*)scalars + (size_t)arg * es, es);
      stack[sp++] = t;
    } else if (is_unary(op)) {
      if (sp < 1) { rc = ORC_E_PROGRAM; goto fail; }
      void* t = malloc(alloc);
      if (!t) { rc = ORC_E_NOMEM; goto fail; }
      apply_unary(type, op, n, stack[sp - 1], t);
      free(stack[sp - 1]);
      stack[sp - 1] = t;
    } else if (is_binary(op)) {
      if (sp < 2) { rc = ORC_E_PROGRAM; goto fail; }
      void* t = malloc(alloc);
      if (!t) { rc = ORC_E_NOMEM; goto fail; }
      apply_binary(type, op, n, stack[sp - 2], stack[sp - 1], t);
      free(stack[sp - 1]);
      free(stack[sp - 2]);
      sp -= 2;
      stack[sp++] = t;
    } else {
      rc = ORC_E_PROGRAM;
      goto fail;
    }
  }
  if (sp != 1) { rc = ORC_E_PROGRAM; goto fail; }
  if (bytes) memcpy(out, stack[0], bytes);
  free(stack[0]);
  return ORC_E_OK;
fail:
  while (sp > 0) free(stack[--sp]);
  return rc;
}

/* Many programs over the same operands: program p is ops/args[offs[p] ..
 * offs[p+1]) and its element-wise result goes to out + p*n*es.  Plumbing for
 * the brute-force program tests (one C call for 10^5 programs instead of one
 * ctypes round trip each); each program is exactly one orc_eval. */
int orc_eval_batch(int type, uint64_t n, const void* const* operands, int n_operands,
                   const void* scalars, int n_scalars, const int* ops, const int* args,
                   const int64_t* offs, int64_t n_progs, void* out) {
  size_t es = esize(type);
  if (es == 0) return ORC_E_TYPE;
  for (int64_t p = 0; p < n_progs; ++p) {
    int rc = orc_eval(type, n, operands, n_operands, scalars, n_scalars, ops + offs[p],
                      args + offs[p], (int)(offs[p + 1] - offs[p]),
                      (char*)out + (size_t)p * (size_t)n * es);
    if (rc) return rc;
  }
  return ORC_E_OK;
}

/* ---- reductions ---------------------------------------------------------
 * Accumulator state so that a reduction can be fed chunk by chunk (the
 * chunked mode is bit-identical to one call over the whole array: same
 * operations in the same index order). */
typedef struct {
  int type, kind;
  long double s, c;      /* Neumaier sum and compensation (floats)          */
  uint64_t isum;         /* modular integer sum                              */
  uint64_t count;
  double fmin, fmax;     /* running min/max for floats (f32 values exact)   */
  uint64_t umin, umax;   /* running min/max for ints (bits)                  */
} orc_acc;

size_t orc_acc_size(void) { return sizeof(orc_acc); }

int orc_acc_init(orc_acc* a, int type, int kind) {
  if (esize(type) == 0) return ORC_E_TYPE;
  if (kind < ORC_ACCU || kind > ORC_NORM2) return ORC_E_KIND;
  if (kind == ORC_NORM2 && (type == ORC_U32 || type == ORC_S64)) return ORC_E_KIND;
  memset(a, 0, sizeof(*a));
  a->type = type;
  a->kind = kind;
  return ORC_E_OK;
}

/* Neumaier (improved Kahan-Babuska) step in long double. */
static void neumaier(long double* s, long double* c, long double x) {
  long double t = *s + x;
  if (fabsl(*s) >= fabsl(x))
    *c += (*s - t) + x;
  else
    *c += (x - t) + *s;
  *s = t;
}

static long double elem_as_ld(int type, const void* v, uint64_t i) {
  if (type == ORC_F32) return (long double)((const float*)v)[i];
  if (is_half(type)) return (long double)half_decode(type, ((const uint16_t*)v)[i]);
  if (is_fp8(type)) return (long double)fp8_decode(type, ((const uint8_t*)v)[i]);
  return (long double)((const double*)v)[i];
}

/* Size of one reduction result: eT, except f32 for the 8-bit storage types
 * (R25: their sums, norms and statistics are returned in f32). */
static size_t rsize(int type) { return is_fp8(type) ? 4 : esize(type); }

/* Round an exact-ish binary128 value once to the result type and store it. */
static void store_flt(int type, void* out, size_t idx, __float128 r) {
  switch (type) {
    case ORC_F32:
    case ORC_E4M3:
    case ORC_E5M2: ((float*)out)[idx] = (float)r; break;
    case ORC_F64: ((double*)out)[idx] = (double)r; break;
    default: ((uint16_t*)out)[idx] = half_round(type, r); break;
  }
}

static uint64_t elem_as_u64(int type, const void* v, uint64_t i) {
  if (type == ORC_U32) return (uint64_t)((const uint32_t*)v)[i];
  return ((const uint64_t*)v)[i];
}

static int int_less(int type, uint64_t a, uint64_t b) {
  if (type == ORC_S64) return (int64_t)a < (int64_t)b;
  return a < b;
}

int orc_acc_add(orc_acc* a, uint64_t n, const void* v) {
  int type = a->type;
  for (uint64_t i = 0; i < n; ++i) {
    if (is_flt(type)) {
      long double x = elem_as_ld(type, v, i);
      switch (a->kind) {
        case ORC_ACCU: neumaier(&a->s, &a->c, x); break;
        case ORC_NORM2: neumaier(&a->s, &a->c, x * x); break;
        default: {
          double d = (double)x;
          if (a->count == 0) { a->fmin = d; a->fmax = d; }
          else {
            if (d < a->fmin) a->fmin = d;
            if (a->fmax < d) a->fmax = d;
          }
        }
      }
    } else {
      uint64_t x = elem_as_u64(type, v, i);
      if (a->kind == ORC_ACCU) {
        a->isum += x;
      } else {
        if (a->count == 0) { a->umin = x; a->umax = x; }
        else {
          if (int_less(type, x, a->umin)) a->umin = x;
          if (int_less(type, a->umax, x)) a->umax = x;
        }
      }
    }
    a->count++;
  }
  return ORC_E_OK;
}

/* Exact value of the Neumaier state rounded once: s + c is formed in
 * __float128 (113-bit significand) and rounded to eT. */
static __float128 acc_total(const orc_acc* a) {
  return (__float128)a->s + (__float128)a->c;
}

/* result: 1 eT (ACCU/MIN/MAX/NORM2) or 2 eT (MINMAX: [min, max]). */
int orc_acc_final(const orc_acc* a, void* result) {
  int type = a->type;
  if ((a->kind == ORC_RMIN || a->kind == ORC_RMAX || a->kind == ORC_MINMAX) && a->count == 0)
    return ORC_E_EMPTY;
  if (is_flt(type)) {
    switch (a->kind) {
      case ORC_ACCU: store_flt(type, result, 0, acc_total(a)); return ORC_E_OK;
      case ORC_NORM2: store_flt(type, result, 0, sqrtq(acc_total(a))); return ORC_E_OK;
      case ORC_RMIN: store_flt(type, result, 0, (__float128)a->fmin); return ORC_E_OK;
      case ORC_RMAX: store_flt(type, result, 0, (__float128)a->fmax); return ORC_E_OK;
      case ORC_MINMAX:  /* extremes are elements: exactly representable */
        store_flt(type, result, 0, (__float128)a->fmin);
        store_flt(type, result, 1, (__float128)a->fmax);
        return ORC_E_OK;
    }
    return ORC_E_KIND;
  }
  uint64_t r0 = 0, r1 = 0;
  int two = 0;
  switch (a->kind) {
    case ORC_ACCU: r0 = a->isum; break;
    case ORC_RMIN: r0 = a->umin; break;
    case ORC_RMAX: r0 = a->umax; break;
    case ORC_MINMAX: r0 = a->umin; r1 = a->umax; two = 1; break;
  }
  if (type == ORC_U32) {
    ((uint32_t*)result)[0] = (uint32_t)r0;
    if (two) ((uint32_t*)result)[1] = (uint32_t)r1;
  } else {
    ((uint64_t*)result)[0] = r0;
    if (two) ((uint64_t*)result)[1] = r1;
  }
  return ORC_E_OK;
}

/* One-shot full reduction of v[0..n). */
int orc_reduce(int type, int kind, uint64_t n, const void* v, void* result) {
  orc_acc a;
  int rc = orc_acc_init(&a, type, kind);
  if (rc) return rc;
  orc_acc_add(&a, n, v);
  return orc_acc_final(&a, result);
}

/* ---- statistics ("mean, variance"; reading R22) --------------------
 * Floats only.  mean = (sum v) / n ; var = sum (v - mean)^2 / (n - 1) with
 * n == 1 -> 0 (Armadillo's default normalisation); stddev = sqrt(var); each
 * rounded once to eT.  The textbook two-pass definition: pass 1 the exact-ish
 * mean (Neumaier in long double, divided in __float128), pass 2 the Neumaier
 * sum of squared deviations from that mean in long double.
 * index_min / index_max: linear scan, strict comparison, so the FIRST index
 * of the extreme value is returned (as uint64). */
enum { ORC_MEAN = 0, ORC_VAR = 1, ORC_STDDEV = 2, ORC_IMIN = 3, ORC_IMAX = 4 };

int orc_stats(int type, int kind, uint64_t n, const void* v, void* result) {
  if (esize(type) == 0) return ORC_E_TYPE;
  if (kind == ORC_IMIN || kind == ORC_IMAX) {
    if (n == 0) return ORC_E_EMPTY;
    uint64_t best = 0;
    for (uint64_t i = 1; i < n; ++i) {
      int better;
      switch (type) {
        case ORC_F32: {
          float a = ((const float*)v)[i], b = ((const float*)v)[best];
          better = kind == ORC_IMIN ? (a < b) : (a > b);
          break;
        }
        case ORC_F64: {
          double a = ((const double*)v)[i], b = ((const double*)v)[best];
          better = kind == ORC_IMIN ? (a < b) : (a > b);
          break;
        }
        case ORC_U32: {
          uint32_t a = ((const uint32_t*)v)[i], b = ((const uint32_t*)v)[best];
          better = kind == ORC_IMIN ? (a < b) : (a > b);
          break;
        }
        case ORC_BF16:
        case ORC_F16:
        case ORC_E4M3:
        case ORC_E5M2: {
          double a = (double)elem_as_ld(type, v, i), b = (double)elem_as_ld(type, v, best);
          better = kind == ORC_IMIN ? (a < b) : (a > b);
          break;
        }
        default: {
          int64_t a = ((const int64_t*)v)[i], b = ((const int64_t*)v)[best];
          better = kind == ORC_IMIN ? (a < b) : (a > b);
          break;
        }
      }
      if (better) best = i;
    }
    *(uint64_t*)result = best;
    return ORC_E_OK;
  }
  if (!is_flt(type)) return ORC_E_KIND;
  if (kind < ORC_MEAN || kind > ORC_STDDEV) return ORC_E_KIND;
  if (n == 0) return ORC_E_EMPTY;
  long double s = 0, c = 0;
  for (uint64_t i = 0; i < n; ++i) neumaier(&s, &c, elem_as_ld(type, v, i));
  const __float128 mean_q = ((__float128)s + (__float128)c) / (__float128)n;
  __float128 r;
  if (kind == ORC_MEAN) {
    r = mean_q;
  } else {
    const long double mean = (long double)mean_q;
    long double s2 = 0, c2 = 0;
    for (uint64_t i = 0; i < n; ++i) {
      const long double d = elem_as_ld(type, v, i) - mean;
      neumaier(&s2, &c2, d * d);
    }
    r = n > 1 ? ((__float128)s2 + (__float128)c2) / (__float128)(n - 1) : (__float128)0;
    if (kind == ORC_STDDEV) r = sqrtq(r);
  }
  store_flt(type, result, 0, r);
  return ORC_E_OK;
}

typedef struct orc_rows_s orc_rows;
orc_rows* orc_rows_new(int type, uint64_t m);
void orc_rows_free(orc_rows* r);
int orc_rows_add(orc_rows* r, uint64_t i0, uint64_t rows, uint64_t ncols, uint64_t ld,
                 const void* X);
int orc_rows_final(const orc_rows* r, void* out);

/* ---- dimension sums (reading R3) ----------------------------------------
 * X is column-major m x n (element (i,j) at X[i + j*m]).
 * dim 0: out[j] = sum_{i=0..m-1} X(i,j)   (n_cols results, a Row)
 * dim 1: out[i] = sum_{j=0..n-1} X(i,j)   (n_rows results, a Col)
 * Each output is its own exact-then-rounded sum (Neumaier over the stated
 * index order).  For dim 1 the loop nest visits j outer / i inner so memory
 * is read contiguously; every row's own summation order is still j = 0..n-1,
 * so the arithmetic is exactly that of the plain per-row loop. */
int orc_sum_dim(int type, int dim, uint64_t m, uint64_t n, const void* X, void* out) {
  size_t es = esize(type);
  if (es == 0) return ORC_E_TYPE;
  if (dim == 0) {
    for (uint64_t j = 0; j < n; ++j) {
      orc_acc a;
      orc_acc_init(&a, type, ORC_ACCU);
      orc_acc_add(&a, m, (const char*)X + (size_t)(j * m) * es);
      orc_acc_final(&a, (char*)out + (size_t)j * rsize(type));
    }
    return ORC_E_OK;
  }
  if (dim != 1) return ORC_E_KIND;
  orc_rows* r = orc_rows_new(type, m);
  if (!r) return ORC_E_NOMEM;
  orc_rows_add(r, 0, m, n, m, X);
  orc_rows_final(r, out);
  orc_rows_free(r);
  return ORC_E_OK;
}

/* ---- dim-1 sums fed column block by column block -------------------------
 * The per-row state of orc_sum_dim's dim-1 loop (Neumaier s, c per row for
 * floats, a modular u64 per row for integers), kept between calls so a
 * matrix too large for host RAM can be fed a block of columns at a time, in
 * column order: orc_rows_add(r, i0, rows, ncols, ld, X) adds columns
 * X(:, 0..ncols-1) of rows i0..i0+rows-1 (element (i, j) at X[i + j*ld]) to
 * rows i0.. of the state.  Each row still sums j = 0..n-1 in order, so any
 * split into column blocks, and any split of the rows between callers, gives
 * exactly orc_sum_dim's arithmetic (tested). */
struct orc_rows_s {
  int type;
  uint64_t m;
  long double* s;
  long double* c;
  uint64_t* u;
};

orc_rows* orc_rows_new(int type, uint64_t m) {
  if (esize(type) == 0) return NULL;
  orc_rows* r = (orc_rows*)calloc(1, sizeof(orc_rows));
  if (!r) return NULL;
  size_t mm = m ? m : 1;
  r->type = type;
  r->m = m;
  if (is_flt(type)) {
    r->s = (long double*)calloc(mm, sizeof(long double));
    r->c = (long double*)calloc(mm, sizeof(long double));
  } else {
    r->u = (uint64_t*)calloc(mm, sizeof(uint64_t));
  }
  if (is_flt(type) ? (!r->s || !r->c) : !r->u) {
    orc_rows_free(r);
    return NULL;
  }
  return r;
}

void orc_rows_free(orc_rows* r) {
  if (!r) return;
  free(r->s);
  free(r->c);
  free(r->u);
  free(r);
}

int orc_rows_add(orc_rows* r, uint64_t i0, uint64_t rows, uint64_t ncols, uint64_t ld,
                 const void* X) {
  if (i0 + rows > r->m || (ncols > 0 && rows > ld)) return ORC_E_SHAPE;
  size_t es = esize(r->type);
  for (uint64_t j = 0; j < ncols; ++j) {
    const char* col = (const char*)X + (size_t)(j * ld) * es;
    for (uint64_t i = 0; i < rows; ++i) {
      if (r->s) neumaier(&r->s[i0 + i], &r->c[i0 + i], elem_as_ld(r->type, col, i));
      else r->u[i0 + i] += elem_as_u64(r->type, col, i);
    }
  }
  return ORC_E_OK;
}

/* out: m results (eT; f32 for the fp8 storage types), each row's exact-ish
 * Neumaier state rounded once. */
int orc_rows_final(const orc_rows* r, void* out) {
  for (uint64_t i = 0; i < r->m; ++i) {
    switch (r->type) {
      case ORC_U32: ((uint32_t*)out)[i] = (uint32_t)r->u[i]; break;
      case ORC_S64: ((uint64_t*)out)[i] = r->u[i]; break;
      default: store_flt(r->type, out, i, (__float128)r->s[i] + (__float128)r->c[i]); break;
    }
  }
  return ORC_E_OK;
}

/* ---- chunked mode --------------------------------------------------------
 * Evaluate a program over global indices [start, start+count) whose operands
 * are regenerated chunk by chunk from (seed, stream = operand index, global
 * index) with per-operand fill kinds, feeding the reduction accumulator `acc`
 * (may be NULL) and optionally writing the element-wise result to `out`
 * (count elements, may be NULL).  Because every step is the same element-wise
 * arithmetic and the accumulator consumes elements in index order, this is
 * bit-identical to generating everything and calling orc_eval + orc_reduce
 * once (tested).  Lets 2^32-element configurations fit in host RAM. */
int orc_run_chunked(int type, uint64_t start, uint64_t count, uint64_t n_rows,
                    int n_operands, const int* fill_kinds, uint64_t seed, uint64_t modk,
                    const void* scalars, int n_scalars, const int* ops, const int* args,
                    int n_instr, uint64_t chunk, orc_acc* acc, void* out) {
  size_t es = esize(type);
  if (es == 0) return ORC_E_TYPE;
  if (n_operands < 0 || n_operands > 16) return ORC_E_PROGRAM;
  if (chunk == 0) chunk = (uint64_t)1 << 24;
  void* bufs[16];
  const void* cops[16];
  void* res = malloc((size_t)chunk * es);
  if (!res) return ORC_E_NOMEM;
  for (int k = 0; k < n_operands; ++k) {
    bufs[k] = malloc((size_t)chunk * es);
    if (!bufs[k]) {
      for (int q = 0; q < k; ++q) free(bufs[q]);
      free(res);
      return ORC_E_NOMEM;
    }
    cops[k] = bufs[k];
  }
  int rc = ORC_E_OK;
  for (uint64_t off = 0; off < count; off += chunk) {
    uint64_t len = count - off < chunk ? count - off : chunk;
    for (int k = 0; k < n_operands; ++k)
      orc_fill(type, fill_kinds[k], seed, (uint64_t)k, start + off, len, n_rows, modk, bufs[k]);
    rc = orc_eval(type, len, cops, n_operands, scalars, n_scalars, ops, args, n_instr, res);
    if (rc) break;
    if (acc) orc_acc_add(acc, len, res);
    if (out) memcpy((char*)out + (size_t)off * es, res, (size_t)len * es);
  }
  for (int k = 0; k < n_operands; ++k) free(bufs[k]);
  free(res);
  return rc;
}
