// Device-side building blocks shared by every libcoot kernel (sm_100a):
// element semantics per opcode and type, 16-byte streaming loads/stores,
// per-thread accumulators and the fixed-order (deterministic) block and
// final reductions.
//
// Numerics (readings R5-R10):
//  * every node rounds to eT, no FMA contraction: explicit __f*_rn / __d*_rn
//    intrinsics (and the build uses -fmad=false, no FTZ, IEEE div/sqrt), so
//    + - * / sqrt are bit-identical to the eager oracle;
//  * EXP/LOG are correctly rounded in every float type (coot_crmath.cuh: a
//    fast phase with a rounding test, a double-double accurate phase);
//  * f32 reductions: 16-byte unit (4 elements) summed pairwise in f32, then
//    accumulated in f64; the final value is rounded once to eT;
//  * integers: modular (u64 accumulator, truncated at the end).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/coot.h"
#include "coot_crmath.cuh"

namespace coot {

typedef long long s64;
typedef unsigned long long u64;

// 16-bit float storage types (R24): a value is its bit pattern; every op
// widens to f32 (exact), computes with IEEE round-to-nearest and rounds once
// back (correctly rounded: 24 >= 2p + 2 for p = 8 and 11).  T(0) is +0.
struct bf16 {
  uint16_t bits;
  __host__ __device__ constexpr bf16() : bits(0) {}
  __host__ __device__ constexpr explicit bf16(int) : bits(0) {}
  __host__ __device__ constexpr bf16(unsigned short b, bool) : bits(b) {}
};
struct f16 {
  uint16_t bits;
  __host__ __device__ constexpr f16() : bits(0) {}
  __host__ __device__ constexpr explicit f16(int) : bits(0) {}
  __host__ __device__ constexpr f16(unsigned short b, bool) : bits(b) {}
};
// 8-bit float STORAGE types (R25, OCP E4M3 "fn" / E5M2): elements are decoded
// exactly to f32, the program runs as an f32 program, and the element's final
// value is rounded once (RNE, saturating: cvt.rn.satfinite) to the format.
// Reductions consume those 8-bit values and return f32.
struct e4m3 {
  uint8_t bits;
  __host__ __device__ constexpr e4m3() : bits(0) {}
  __host__ __device__ constexpr explicit e4m3(int) : bits(0) {}
  __host__ __device__ constexpr e4m3(unsigned char b, bool) : bits(b) {}
};
struct e5m2 {
  uint8_t bits;
  __host__ __device__ constexpr e5m2() : bits(0) {}
  __host__ __device__ constexpr explicit e5m2(int) : bits(0) {}
  __host__ __device__ constexpr e5m2(unsigned char b, bool) : bits(b) {}
};
// arithmetic type of an expression over T (f32 for the 8-bit storage types)
template <class T>
struct ComputeT {
  typedef T type;
};
template <>
struct ComputeT<e4m3> {
  typedef float type;
};
template <>
struct ComputeT<e5m2> {
  typedef float type;
};
// type of a reduction / dim-sum result (eT; f32 for the 8-bit storage types)
template <class T>
struct ResultT {
  typedef T type;
};
template <>
struct ResultT<e4m3> {
  typedef float type;
};
template <>
struct ResultT<e5m2> {
  typedef float type;
};

enum AccKind {
  ACC_NONE = 0, ACC_SUM = 1, ACC_SUMSQ = 2, ACC_MINMAX = 3,
  ACC_VAR = 4, ACC_IMIN = 5, ACC_IMAX = 6
};
enum FinalMode { FINAL_ROUND = 0, FINAL_PARTIAL = 1, FINAL_EXCHANGE = 2 };

// In-kernel exchange (FINAL_EXCHANGE): mailbox of rank p at mbox[p] (this
// process's mapping): records slot[0..P) then u64 flags[0..P).
struct Exchange {
  unsigned long long mbox[COOT_MAX_RANKS];
  unsigned long long epoch;
  uint32_t nranks, rank;
};

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// One reduction partial record (COOT_PARTIAL_BYTES = 32).
struct __align__(16) Rec {
  u64 a, b, count, pad;
};

// Kernel arguments for the fused element-wise pass (passed as a
// __grid_constant__ parameter; < 1 KB).
struct FusedArgs {
  const void* in[COOT_MAX_OPERANDS];
  void* out;          // element-wise result or nullptr
  u64 n;              // elements
  u64 head;           // scalar elements before the 16-byte aligned body
  u64 nunits;         // 16-byte units in the body
  u64 tail_begin;     // = head + nunits * W
  u64 scalars[COOT_MAX_SCALARS];  // eT bits
  Rec* partials;      // per-block records (ctx scratch)
  unsigned* ticket;   // self-resetting arrival counter (ctx scratch)
  void* result;       // eT result(s) or a Rec (FINAL_PARTIAL)
  u64 count;          // element count recorded in a partial
  uint32_t final_mode;
  uint32_t kind;      // coot_reduce_kind
  uint32_t n_operands;
  uint32_t n_instr;
  uint32_t tile_units;  // TMA driver: 16-byte units per tile (multiple of 256)
  uint32_t stages;      // TMA driver: smem pipeline depth
  uint32_t producer_sleep;  // TMA drivers: the producer sleeps while the ring is full
  // strided (view) path: element (i, j) of operand k at in[k][i*inc[k] + j*ld[k]]
  u64 m;                // rows of the expression
  u64 ld[COOT_MAX_OPERANDS], inc[COOT_MAX_OPERANDS];
  u64 out_ld, out_inc;
  // column-segmented view path: pieces = (column, segment of seg_len rows)
  u64 ncols, seg_len;
  uint32_t nseg;
  // interpreter instruction: dispatch index (op * 9 + depth) | argument << 16
  // (one 32-bit word: the constant-bank load lands in a register as is)
  uint32_t code[COOT_MAX_INSTR];
  Exchange ex;  // FINAL_EXCHANGE only
};

template <class T>
struct Unit {
  static constexpr int W = 16 / sizeof(T);
};

// ---- scalar slot decoding -------------------------------------------------
template <class T>
__device__ __forceinline__ T scalar_as(u64 bits);
template <>
__device__ __forceinline__ float scalar_as<float>(u64 bits) {
  return __uint_as_float((unsigned)bits);
}
template <>
__device__ __forceinline__ double scalar_as<double>(u64 bits) {
  return __longlong_as_double((long long)bits);
}
template <>
__device__ __forceinline__ uint32_t scalar_as<uint32_t>(u64 bits) {
  return (uint32_t)bits;
}
template <>
__device__ __forceinline__ s64 scalar_as<s64>(u64 bits) {
  return (s64)bits;
}
template <>
__device__ __forceinline__ bf16 scalar_as<bf16>(u64 bits) {
  return bf16((unsigned short)bits, true);
}
template <>
__device__ __forceinline__ f16 scalar_as<f16>(u64 bits) {
  return f16((unsigned short)bits, true);
}
// (8-bit types: only partial records carry their bits; program scalars are f32)
template <>
__device__ __forceinline__ e4m3 scalar_as<e4m3>(u64 bits) {
  return e4m3((unsigned char)bits, true);
}
template <>
__device__ __forceinline__ e5m2 scalar_as<e5m2>(u64 bits) {
  return e5m2((unsigned char)bits, true);
}

template <class T>
__device__ __forceinline__ u64 to_bits(T v);
template <>
__device__ __forceinline__ u64 to_bits<float>(float v) {
  return (u64)__float_as_uint(v);
}
template <>
__device__ __forceinline__ u64 to_bits<double>(double v) {
  return (u64)__double_as_longlong(v);
}
template <>
__device__ __forceinline__ u64 to_bits<uint32_t>(uint32_t v) {
  return (u64)v;
}
template <>
__device__ __forceinline__ u64 to_bits<s64>(s64 v) {
  return (u64)v;
}
template <>
__device__ __forceinline__ u64 to_bits<bf16>(bf16 v) {
  return (u64)v.bits;
}
template <>
__device__ __forceinline__ u64 to_bits<f16>(f16 v) {
  return (u64)v.bits;
}
template <>
__device__ __forceinline__ u64 to_bits<e4m3>(e4m3 v) {
  return (u64)v.bits;
}
template <>
__device__ __forceinline__ u64 to_bits<e5m2>(e5m2 v) {
  return (u64)v.bits;
}

template <class T>
struct FloatTrait {
  static constexpr bool value = false;
  static constexpr bool half = false;
};
template <>
struct FloatTrait<float> {
  static constexpr bool value = true;
  static constexpr bool half = false;
};
template <>
struct FloatTrait<double> {
  static constexpr bool value = true;
  static constexpr bool half = false;
};
template <>
struct FloatTrait<bf16> {
  static constexpr bool value = true;
  static constexpr bool half = true;
};
template <>
struct FloatTrait<f16> {
  static constexpr bool value = true;
  static constexpr bool half = true;
};
template <>
struct FloatTrait<e4m3> {
  static constexpr bool value = true;
  static constexpr bool half = false;
};
template <>
struct FloatTrait<e5m2> {
  static constexpr bool value = true;
  static constexpr bool half = false;
};
template <class T>
__host__ __device__ constexpr bool is_float() {
  return FloatTrait<T>::value;
}
template <class T>
__host__ __device__ constexpr bool is_half() {
  return FloatTrait<T>::half;
}
template <class T>
__host__ __device__ constexpr bool is_fp8() {
  return std::is_same<T, e4m3>::value || std::is_same<T, e5m2>::value;
}
// bit-pattern storage types whose values are handled widened to f32
template <class T>
__host__ __device__ constexpr bool is_narrow() {
  return is_half<T>() || is_fp8<T>();
}

// ---- 16-bit conversions: widening is exact; narrowing rounds once (RNE) --------
__device__ __forceinline__ float to_f32(bf16 v) { return __uint_as_float((unsigned)v.bits << 16); }
__device__ __forceinline__ float to_f32(f16 v) { return __half2float(__ushort_as_half(v.bits)); }
template <class H>
__device__ __forceinline__ H half_from_f32(float x);
template <>
__device__ __forceinline__ bf16 half_from_f32<bf16>(float x) {
  return bf16(__bfloat16_as_ushort(__float2bfloat16_rn(x)), true);
}
template <>
__device__ __forceinline__ f16 half_from_f32<f16>(float x) {
  return f16(__half_as_ushort(__float2half_rn(x)), true);
}
template <class H>
__device__ __forceinline__ H half_from_f64(double x);
template <>
__device__ __forceinline__ bf16 half_from_f64<bf16>(double x) {
  return bf16(__bfloat16_as_ushort(__double2bfloat16(x)), true);  // F2F.BF16.F64
}
template <>
__device__ __forceinline__ f16 half_from_f64<f16>(double x) {
  return f16(__half_as_ushort(__double2half(x)), true);  // F2F.F16.F64
}
// ---- 8-bit conversions: decoding is exact (every E4M3 / E5M2 value is an f16
// value); encoding is cvt.rn.satfinite (nearest-even, overflow and +-inf to the
// largest finite magnitude, NaN to NaN) ----------------------------------------
__device__ __forceinline__ float to_f32(e4m3 v) {
  unsigned h2;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"((unsigned short)v.bits));
  return __half2float(__ushort_as_half((unsigned short)(h2 & 0xffffu)));
}
__device__ __forceinline__ float to_f32(e5m2 v) {  // E5M2 = the top byte of an f16
  return __half2float(__ushort_as_half((unsigned short)((unsigned)v.bits << 8)));
}
template <class H>
__device__ __forceinline__ H fp8_from_f32(float x) {
  unsigned short p;
  if constexpr (std::is_same<H, e4m3>::value)
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(0.0f), "f"(x));
  else
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(p) : "f"(0.0f), "f"(x));
  return H((unsigned char)(p & 0xffu), true);
}
// exact value of any element type as f64 (floats only are used)
__device__ __forceinline__ double as_double(float v) { return (double)v; }
__device__ __forceinline__ double as_double(double v) { return v; }
__device__ __forceinline__ double as_double(bf16 v) { return (double)to_f32(v); }
__device__ __forceinline__ double as_double(f16 v) { return (double)to_f32(v); }
__device__ __forceinline__ double as_double(e4m3 v) { return (double)to_f32(v); }
__device__ __forceinline__ double as_double(e5m2 v) { return (double)to_f32(v); }
__device__ __forceinline__ double as_double(uint32_t v) { return (double)v; }
__device__ __forceinline__ double as_double(s64 v) { return (double)v; }
// exact value of an f32 / 16-bit / 8-bit element as f32
__device__ __forceinline__ float as_float(float v) { return v; }
__device__ __forceinline__ float as_float(bf16 v) { return to_f32(v); }
__device__ __forceinline__ float as_float(f16 v) { return to_f32(v); }
__device__ __forceinline__ float as_float(e4m3 v) { return to_f32(v); }
__device__ __forceinline__ float as_float(e5m2 v) { return to_f32(v); }
// ordering (IEEE semantics for floats)
template <class T>
__device__ __forceinline__ bool lt(T a, T b) {
  if constexpr (is_narrow<T>()) return to_f32(a) < to_f32(b);
  else return a < b;
}
// element loads bypassing L1 (operands may alias the output exactly)
template <class T>
__device__ __forceinline__ T ldcg_elem(const T* p) {
  if constexpr (is_half<T>()) return T(__ldcg(reinterpret_cast<const unsigned short*>(p)), true);
  else if constexpr (is_fp8<T>()) return T(__ldcg(reinterpret_cast<const unsigned char*>(p)), true);
  else return __ldcg(p);
}

// Two 8-bit values -> two f32, exactly: one cvt.rn.f16x2.{e4m3x2,e5m2x2}
// (E5M2 is a byte permute) and a paired f16 -> f32 widening.
template <class T>
__device__ __forceinline__ float2 fp8x2_to_f32x2(T lo, T hi) {
  const unsigned short pk = (unsigned short)(lo.bits | ((unsigned)hi.bits << 8));
  unsigned h2;
  if constexpr (std::is_same<T, e4m3>::value) {
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(pk));
  } else {
    h2 = __byte_perm((unsigned)pk, 0u, 0x1404);  // bytes -> the high byte of each f16
  }
  __half2 h;
  memcpy(&h, &h2, 4);
  return __half22float2(h);
}

// Exact f32 values of W f32 / 16-bit / 8-bit elements (8-bit: pairwise).
template <class T, int W>
__device__ __forceinline__ void widen_f32(const T (&v)[W], float (&x)[W]) {
  if constexpr (is_fp8<T>()) {
#pragma unroll
    for (int w = 0; w + 1 < W; w += 2) {
      const float2 f = fp8x2_to_f32x2(v[w], v[w + 1]);
      x[w] = f.x;
      x[w + 1] = f.y;
    }
    if constexpr (W & 1) x[W - 1] = to_f32(v[W - 1]);
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) x[w] = as_float(v[w]);
  }
}

// ---- storage <-> arithmetic type (identity except for the 8-bit types) ------
template <class T, int W>
__device__ __forceinline__ void widen_vec(const T (&v)[W], typename ComputeT<T>::type (&c)[W]) {
  if constexpr (is_fp8<T>()) {
    widen_f32<T, W>(v, c);
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) c[w] = v[w];
  }
}
// f32 -> 8-bit, two at a time (cvt.rn.satfinite.{e4m3x2,e5m2x2}.f32)
template <class T, int W>
__device__ __forceinline__ void narrow_vec(const typename ComputeT<T>::type (&c)[W], T (&v)[W]) {
  if constexpr (is_fp8<T>()) {
#pragma unroll
    for (int w = 0; w + 1 < W; w += 2) {
      unsigned short p;
      if constexpr (std::is_same<T, e4m3>::value)
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(c[w + 1]), "f"(c[w]));
      else
        asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(p) : "f"(c[w + 1]), "f"(c[w]));
      v[w] = T((unsigned char)(p & 0xffu), true);
      v[w + 1] = T((unsigned char)(p >> 8), true);
    }
    if constexpr (W & 1) v[W - 1] = fp8_from_f32<T>(c[W - 1]);
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = c[w];
  }
}

// ---- op legality (R9) -----------------------------------------------------
template <class T>
__host__ __device__ constexpr bool op_legal(int op) {
  return is_float<T>() ? true
                       : !(op == COOT_OP_SQRT || op == COOT_OP_EXP || op == COOT_OP_LOG ||
                           op == COOT_OP_DIV);
}

// ---- EXP / LOG (R6): correctly rounded, coot_crmath.cuh ----------------------
using crm::exp_f64_of_f32;  // f32 e^x as a double within 2^-51 (the 16-bit types' fallback)

// ---- element semantics ------------------------------------------------------
template <int OP>
__device__ __forceinline__ float un(float a) {
  if constexpr (OP == COOT_OP_NEG) return -a;
  else if constexpr (OP == COOT_OP_ABS) return fabsf(a);
  else if constexpr (OP == COOT_OP_SQUARE) return __fmul_rn(a, a);
  else if constexpr (OP == COOT_OP_SQRT) return __fsqrt_rn(a);
  // f32 EXP/LOG are correctly rounded (R6, coot_crmath.cuh): evaluated in
  // f64 and rounded once when that provably decides the f32 result, else by
  // the double-double accurate phase.  This keeps composed expressions
  // bit-identical to the correctly rounded oracle, where expf/logf (<= 2 / 1
  // ulp) would let later nodes amplify the difference.
  else if constexpr (OP == COOT_OP_EXP) return crm::cr_expf(a);
  else if constexpr (OP == COOT_OP_LOG) return crm::cr_logf(a);
  else return a;
}
template <int OP>
__device__ __forceinline__ double un(double a) {
  if constexpr (OP == COOT_OP_NEG) return -a;
  else if constexpr (OP == COOT_OP_ABS) return fabs(a);
  else if constexpr (OP == COOT_OP_SQUARE) return __dmul_rn(a, a);
  else if constexpr (OP == COOT_OP_SQRT) return __dsqrt_rn(a);
  else if constexpr (OP == COOT_OP_EXP) return crm::cr_exp(a);  // correctly rounded (R6)
  else if constexpr (OP == COOT_OP_LOG) return crm::cr_log(a);
  else return a;
}
// bf16 / f16 EXP / LOG (R24): the f32 expf / logf result (CUDA math library:
// <= 2 / <= 1 ulp) already decides the correctly rounded 16-bit value unless
// it lies within a few f32 ulps of a rounding midpoint of the format (the
// bits below the format's last place are 100...0 +- margin), or outside the
// format's normal range, or is not finite.  Those rare elements (~2^-12 of
// bf16, ~2^-9 of f16 results) take the f64 path, so every element still gets
// the correctly rounded result while the common case stays in FP32/MUFU.
//
// half_mid_dist(y) = (bits below the last place - midpoint + margin) mod 2^b:
// the rounding is undecided iff it is <= 2 * margin.  bf16 shares f32's
// exponent range, so the last place is bit 16 for every f32 (subnormal
// included) and inf / 0 / NaN round the same from y as from the true value
// (an f32 result beyond FLT_MAX is far past bf16's overflow midpoint).  f16's
// last place is bit 13 only in its normal range; results below 2^-14 go to
// the fallback, results past 65520 round to inf either way.
constexpr unsigned kHalfMargin = 8;  // f32 ulps (4x the library's bound)
template <class H>
__device__ __forceinline__ unsigned half_mid_dist(float y) {
  const unsigned u = __float_as_uint(y);
  if constexpr (std::is_same<H, bf16>::value) {
    return (u + (0x8000u + kHalfMargin)) & 0xffffu;
  } else {
    const unsigned d = (u + (0x1000u + kHalfMargin)) & 0x1fffu;
    return fabsf(y) < 0x1p-14f ? 0u : d;
  }
}
template <class H>
__device__ __forceinline__ bool half_round_decided(float y) {
  return half_mid_dist<H>(y) > 2 * kHalfMargin;
}

// bf16 / f16 (R24): widen exactly, compute (f32 for + - * / sqrt, f32 with an
// f64 fallback for exp / log), round once to the format.
template <int OP, class H>
__device__ __forceinline__ H half_un(H a) {
  if constexpr (OP == COOT_OP_NEG) return H((unsigned short)(a.bits ^ 0x8000u), true);
  else if constexpr (OP == COOT_OP_ABS) return H((unsigned short)(a.bits & 0x7fffu), true);
  else {
    const float x = to_f32(a);
    if constexpr (OP == COOT_OP_SQUARE) return half_from_f32<H>(__fmul_rn(x, x));
    else if constexpr (OP == COOT_OP_SQRT) return half_from_f32<H>(__fsqrt_rn(x));
    else if constexpr (OP == COOT_OP_EXP) {
      const float y = expf(x);
      if (__builtin_expect(half_round_decided<H>(y), 1)) return half_from_f32<H>(y);
      return half_from_f64<H>(exp_f64_of_f32(x));
    } else if constexpr (OP == COOT_OP_LOG) {
      const float y = logf(x);
      if (__builtin_expect(half_round_decided<H>(y), 1)) return half_from_f32<H>(y);
      return half_from_f64<H>(log((double)x));
    } else return a;
  }
}
template <int OP>
__device__ __forceinline__ bf16 un(bf16 a) {
  return half_un<OP, bf16>(a);
}
template <int OP>
__device__ __forceinline__ f16 un(f16 a) {
  return half_un<OP, f16>(a);
}
// A unary node over the W elements one dispatch holds.  For bf16/f16 EXP/LOG
// the fast f32 results of all W elements are formed first and the rare f64
// fix-up runs after them under one branch, so the W dependency chains stay
// independent (interleavable) instead of being split by a branch per element.
// (defined after every un<> overload below)
template <int OP, class H>
__device__ __forceinline__ H half_bin(H a, H b) {
  const float x = to_f32(a), y = to_f32(b);
  if constexpr (OP == COOT_OP_ADD) return half_from_f32<H>(__fadd_rn(x, y));
  else if constexpr (OP == COOT_OP_SUB) return half_from_f32<H>(__fsub_rn(x, y));
  else if constexpr (OP == COOT_OP_MUL) return half_from_f32<H>(__fmul_rn(x, y));
  else if constexpr (OP == COOT_OP_DIV) return half_from_f32<H>(__fdiv_rn(x, y));
  else if constexpr (OP == COOT_OP_MIN) return (y < x) ? b : a;
  else if constexpr (OP == COOT_OP_MAX) return (x < y) ? b : a;
  else return a;
}
template <int OP>
__device__ __forceinline__ bf16 bin(bf16 a, bf16 b) {
  return half_bin<OP, bf16>(a, b);
}
template <int OP>
__device__ __forceinline__ f16 bin(f16 a, f16 b) {
  return half_bin<OP, f16>(a, b);
}
// 8-bit storage types: only MIN / MAX are applied to stored values (by the
// min/max accumulators); every other op runs on the f32 arithmetic type.
template <int OP>
__device__ __forceinline__ e4m3 bin(e4m3 a, e4m3 b) {
  static_assert(OP == COOT_OP_MIN || OP == COOT_OP_MAX, "8-bit values are only compared");
  return OP == COOT_OP_MIN ? (lt(b, a) ? b : a) : (lt(a, b) ? b : a);
}
template <int OP>
__device__ __forceinline__ e5m2 bin(e5m2 a, e5m2 b) {
  static_assert(OP == COOT_OP_MIN || OP == COOT_OP_MAX, "8-bit values are only compared");
  return OP == COOT_OP_MIN ? (lt(b, a) ? b : a) : (lt(a, b) ? b : a);
}
template <int OP>
__device__ __forceinline__ uint32_t un(uint32_t a) {
  if constexpr (OP == COOT_OP_NEG) return 0u - a;
  else if constexpr (OP == COOT_OP_SQUARE) return a * a;
  else return a;  // ABS of unsigned is the identity; illegal ops never reach here
}
template <int OP>
__device__ __forceinline__ s64 un(s64 a) {
  const u64 x = (u64)a;
  if constexpr (OP == COOT_OP_NEG) return (s64)(0ull - x);
  else if constexpr (OP == COOT_OP_ABS) return a < 0 ? (s64)(0ull - x) : a;
  else if constexpr (OP == COOT_OP_SQUARE) return (s64)(x * x);
  else return a;
}

template <int OP>
__device__ __forceinline__ float bin(float a, float b) {
  if constexpr (OP == COOT_OP_ADD) return __fadd_rn(a, b);
  else if constexpr (OP == COOT_OP_SUB) return __fsub_rn(a, b);
  else if constexpr (OP == COOT_OP_MUL) return __fmul_rn(a, b);
  else if constexpr (OP == COOT_OP_DIV) return __fdiv_rn(a, b);
  else if constexpr (OP == COOT_OP_MIN) return (b < a) ? b : a;
  else if constexpr (OP == COOT_OP_MAX) return (a < b) ? b : a;
  else return a;
}
template <int OP>
__device__ __forceinline__ double bin(double a, double b) {
  if constexpr (OP == COOT_OP_ADD) return __dadd_rn(a, b);
  else if constexpr (OP == COOT_OP_SUB) return __dsub_rn(a, b);
  else if constexpr (OP == COOT_OP_MUL) return __dmul_rn(a, b);
  else if constexpr (OP == COOT_OP_DIV) return __ddiv_rn(a, b);
  else if constexpr (OP == COOT_OP_MIN) return (b < a) ? b : a;
  else if constexpr (OP == COOT_OP_MAX) return (a < b) ? b : a;
  else return a;
}
template <int OP>
__device__ __forceinline__ uint32_t bin(uint32_t a, uint32_t b) {
  if constexpr (OP == COOT_OP_ADD) return a + b;
  else if constexpr (OP == COOT_OP_SUB) return a - b;
  else if constexpr (OP == COOT_OP_MUL) return a * b;
  else if constexpr (OP == COOT_OP_MIN) return (b < a) ? b : a;
  else if constexpr (OP == COOT_OP_MAX) return (a < b) ? b : a;
  else return a;
}
template <int OP>
__device__ __forceinline__ s64 bin(s64 a, s64 b) {
  const u64 x = (u64)a, y = (u64)b;
  if constexpr (OP == COOT_OP_ADD) return (s64)(x + y);
  else if constexpr (OP == COOT_OP_SUB) return (s64)(x - y);
  else if constexpr (OP == COOT_OP_MUL) return (s64)(x * y);
  else if constexpr (OP == COOT_OP_MIN) return (b < a) ? b : a;
  else if constexpr (OP == COOT_OP_MAX) return (a < b) ? b : a;
  else return a;
}

// Round W f32 values to a 16-bit format two at a time: cvt.rn.{bf16x2,f16x2}.f32
// (F2FP.PACK_AB, one instruction per pair, not on the quarter-rate XU pipe that
// the single-value F2F conversion occupies).  Same RNE result per element.
template <class H, int W>
__device__ __forceinline__ void half_round_vec(const float (&y)[W], H (&v)[W]) {
#pragma unroll
  for (int w = 0; w + 1 < W; w += 2) {
    unsigned p;
    if constexpr (std::is_same<H, bf16>::value) {
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(y[w + 1]), "f"(y[w]));
    } else {
      asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(y[w + 1]), "f"(y[w]));
    }
    memcpy(&v[w], &p, 4);  // the pair as one 32-bit register (no repacking)
  }
  if constexpr (W & 1) v[W - 1] = half_from_f32<H>(y[W - 1]);
}

// + - * on 16-bit pairs with the packed instructions ({add,sub,mul}.rn.{bf16x2,
// f16x2}: one HADD2/HMUL2/HFMA2 per pair instead of widen x4, two f32 ops and a
// narrowing).  Same bits as the f32 route: each returns the exact result
// rounded once (RNE, subnormals kept — no .ftz), and the f32 route's double
// rounding is innocuous (R24: 24 >= 2p + 2), so both equal RNE16(exact).
// `.rn` is explicit, so ptxas may not contract a MUL into a following ADD.
template <int OP, class H>
__device__ __forceinline__ uint32_t half2_op(uint32_t x, uint32_t y) {
  uint32_t d;
  if constexpr (std::is_same<H, bf16>::value) {
    if constexpr (OP == COOT_OP_ADD) asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (OP == COOT_OP_SUB) asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
  } else {
    if constexpr (OP == COOT_OP_ADD) asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (OP == COOT_OP_SUB) asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
  }
  return d;
}
template <int OP, class H, int W>
__device__ __forceinline__ void half2_vec(H (&a)[W], const H (&b)[W]) {
#pragma unroll
  for (int w = 0; w + 1 < W; w += 2) {
    // (a[w], a[w+1]) read / written as one 32-bit register: element w in the
    // low half, as loaded from memory — a shift-and-or repack here made ptxas
    // emit two byte permutes per pair that it could not fold away
    uint32_t x, y;
    memcpy(&x, &a[w], 4);
    memcpy(&y, &b[w], 4);
    const uint32_t d = half2_op<OP, H>(x, y);
    memcpy(&a[w], &d, 4);
  }
  if constexpr (W & 1) a[W - 1] = half_bin<OP, H>(a[W - 1], b[W - 1]);
}

template <int OP, class T, int W>
__device__ __forceinline__ void bin_vec(T (&a)[W], const T (&b)[W]) {
  if constexpr (is_half<T>() && (OP == COOT_OP_ADD || OP == COOT_OP_SUB || OP == COOT_OP_MUL)) {
    half2_vec<OP, T, W>(a, b);
  } else if constexpr (is_half<T>() && OP == COOT_OP_DIV) {
    float y[W];
#pragma unroll
    for (int w = 0; w < W; ++w) y[w] = bin<OP>(to_f32(a[w]), to_f32(b[w]));
    half_round_vec<T, W>(y, a);
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) a[w] = bin<OP>(a[w], b[w]);
  }
}

// The rare accurate phase of a W-element EXP / LOG: the undecided elements
// go one by one through ONE call site (a local copy of the W inputs /
// results; the hot path keeps its registers).
// The rare accurate phase of a W-element EXP / LOG: every element of the
// group is recomputed by the scalar correctly rounded function (the same
// result for the ones the fast phase already decided) through ONE call site
// with a local copy of the inputs / results, so the hot path keeps its
// registers and stays straight-line.
template <int OP, class T, int W>
__device__ __noinline__ void slow_fix_call(const T (&x)[W], T (&v)[W]) {
#pragma unroll 1
  for (int w = 0; w < W; ++w) {
    if constexpr (std::is_same<T, float>::value)
      v[w] = (OP == COOT_OP_EXP) ? crm::cr_expf(x[w]) : crm::cr_logf(x[w]);
    else
      v[w] = (OP == COOT_OP_EXP) ? crm::cr_exp_slow(x[w]) : crm::cr_log_slow(x[w]);
  }
}
template <int OP, class T, int W>
__device__ __forceinline__ void slow_fix(const T (&x)[W], T (&v)[W]) {
  T xs[W], vs[W];
#pragma unroll
  for (int w = 0; w < W; ++w) xs[w] = x[w];
  slow_fix_call<OP, T, W>(xs, vs);
#pragma unroll
  for (int w = 0; w < W; ++w) v[w] = vs[w];
}

// EXP / LOG group size: the catalog kernels take 8 elements at a time (all
// of a 2-unit dispatch: the most interleaving); the interpreter 4 (it holds
// its register stack next to them).
#ifndef COOT_EXP_GROUP
#define COOT_EXP_GROUP 8
#endif
template <int OP, int GMAX = COOT_EXP_GROUP, class T, int W>
__device__ __forceinline__ void un_vec(T (&v)[W]) {
  if constexpr (is_half<T>() && OP == COOT_OP_SQUARE) {
    half2_vec<COOT_OP_MUL, T, W>(v, v);
  } else if constexpr (is_half<T>() && OP == COOT_OP_SQRT) {
    float y[W];
#pragma unroll
    for (int w = 0; w < W; ++w) y[w] = un<OP>(to_f32(v[w]));
    half_round_vec<T, W>(y, v);
  } else if constexpr ((std::is_same<T, float>::value || std::is_same<T, double>::value) &&
                       (OP == COOT_OP_EXP || OP == COOT_OP_LOG)) {
    // correctly rounded EXP / LOG (R6), in groups of up to 4 elements: the
    // fast phase of the group first (straight-line, its chains interleave),
    // then ONE rare branch if the rounding test left any element undecided.
    // Groups of 4 bound the live registers (the interpreter evaluates 16
    // elements per dispatch next to its register stack).
    constexpr int G = W < GMAX ? W : GMAX;
    static_assert(W % G == 0, "group size");
#ifdef COOT_EXPERIMENT_EXPF  // A/B experiment only (not correctly rounded): the cost of CR
    if constexpr (std::is_same<T, float>::value) {
#pragma unroll
      for (int w = 0; w < W; ++w) v[w] = (OP == COOT_OP_EXP) ? expf(v[w]) : logf(v[w]);
      return;
    }
#endif
#pragma unroll
    for (int g = 0; g < W; g += G) {
      T x[G];
      bool all = true;
#pragma unroll
      for (int w = 0; w < G; ++w) {
        x[w] = v[g + w];
        if constexpr (std::is_same<T, float>::value) {
          // outside the fast range (non-normal results, NaN, <= 0 for LOG)
          // the fast value is meaningless and the slow path decides
          const bool in = (OP == COOT_OP_EXP) ? crm::expf_fast_range(x[w]) : crm::logf_fast_range(x[w]);
          const double y = (OP == COOT_OP_EXP) ? crm::exp_f64_of_f32_core((double)x[w])
                                               : crm::logf_fast_core(x[w]);
          all = all && in && crm::f32_mid_clear(y, crm::kF32Margin);
          v[g + w] = (float)y;
        } else {
          bool ok;
          v[g + w] = (OP == COOT_OP_EXP) ? crm::exp_fast_ok(x[w], ok) : crm::log_fast_ok(x[w], ok);
          all = all && ok;
        }
      }
      if (__builtin_expect(!all, 0)) {
        T r[G];
        slow_fix<OP, T, G>(x, r);
#pragma unroll
        for (int w = 0; w < G; ++w) v[g + w] = r[w];
      }
    }
  } else if constexpr (is_half<T>() && (OP == COOT_OP_EXP || OP == COOT_OP_LOG)) {
    float x[W], y[W];
    unsigned closest = 0xffffffffu;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      x[w] = to_f32(v[w]);
      y[w] = (OP == COOT_OP_EXP) ? expf(x[w]) : logf(x[w]);
      closest = min(closest, half_mid_dist<T>(y[w]));
    }
    half_round_vec<T, W>(y, v);
    if (__builtin_expect(closest <= 2 * kHalfMargin, 0)) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (!half_round_decided<T>(y[w]))
          v[w] = half_from_f64<T>((OP == COOT_OP_EXP) ? exp_f64_of_f32(x[w]) : log((double)x[w]));
      }
    }
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = un<OP>(v[w]);
  }
}

// ---- 16-byte streaming memory access --------------------------------------
// Coherent loads (an operand may alias `out` exactly), no L1 allocation
// (each byte is touched once); the element-wise output is stored with the
// evict-first (.cs) hint.
__device__ __forceinline__ uint4 ld16(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st16(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

template <class T>
__device__ __forceinline__ void load_unit(const T* p, T (&v)[Unit<T>::W]) {
  uint4 r = ld16(p);
  static_assert(sizeof(v) == 16, "unit is 16 bytes");
  memcpy(&v[0], &r, 16);
}
template <class T>
__device__ __forceinline__ void store_unit(T* p, const T (&v)[Unit<T>::W]) {
  uint4 r;
  memcpy(&r, &v[0], 16);
  st16(p, r);
}

// ---- mbarrier + 1-D TMA bulk copies (cp.async.bulk) -------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Block until the phase with the given parity has completed.
// Wait for an mbarrier phase.  SLEEP: the thread is suspended until the phase
// completes or a 100 us hint runs out (else the short system limit applies and
// the thread re-polls).  Used for the producer's wait for a free stage when the
// program is compute-heavy (FusedArgs::producer_sleep): there a re-polling
// producer warp takes issue slots from the consumers (bf16 / f16 / E4M3 c2
// +2-3 %); memory-bound programs keep polling (prompt re-issue of the ring).
template <bool SLEEP = false>
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done;
  do {
    if constexpr (SLEEP) {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(addr), "r"(parity), "n"(100000)
          : "memory");
    } else {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(addr), "r"(parity)
          : "memory");
    }
  } while (!done);
}
__device__ __forceinline__ void producer_wait(uint64_t* bar, uint32_t parity, uint32_t sleep) {
  if (sleep) mbar_wait<true>(bar, parity);
  else mbar_wait<false>(bar, parity);
}
// L2 policy for data that is streamed exactly once.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// global -> shared 1-D bulk copy completing `bytes` of transaction on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint4 lds16(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}

// ---- warp shuffles for 64-bit values ---------------------------------------
__device__ __forceinline__ double shfl_xor(double v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
__device__ __forceinline__ u64 shfl_xor(u64 v, int m) {
  return (u64)__shfl_xor_sync(0xffffffffu, (long long)v, m);
}
__device__ __forceinline__ float shfl_xor(float v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
__device__ __forceinline__ uint32_t shfl_xor(uint32_t v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
__device__ __forceinline__ s64 shfl_xor(s64 v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
__device__ __forceinline__ bf16 shfl_xor(bf16 v, int m) {
  return bf16((unsigned short)__shfl_xor_sync(0xffffffffu, (unsigned)v.bits, m), true);
}
__device__ __forceinline__ f16 shfl_xor(f16 v, int m) {
  return f16((unsigned short)__shfl_xor_sync(0xffffffffu, (unsigned)v.bits, m), true);
}
__device__ __forceinline__ e4m3 shfl_xor(e4m3 v, int m) {
  return e4m3((unsigned char)__shfl_xor_sync(0xffffffffu, (unsigned)v.bits, m), true);
}
__device__ __forceinline__ e5m2 shfl_xor(e5m2 v, int m) {
  return e5m2((unsigned char)__shfl_xor_sync(0xffffffffu, (unsigned)v.bits, m), true);
}

// ---- per-thread accumulators -------------------------------------------------
template <class T>
struct MinMaxId;
template <>
struct MinMaxId<float> {
  __device__ static float lo() { return __int_as_float(0x7f800000); }   // +inf
  __device__ static float hi() { return __int_as_float((int)0xff800000u); }  // -inf
};
template <>
struct MinMaxId<double> {
  __device__ static double lo() { return __longlong_as_double(0x7ff0000000000000ll); }
  __device__ static double hi() { return __longlong_as_double((long long)0xfff0000000000000ull); }
};
template <>
struct MinMaxId<uint32_t> {
  __device__ static uint32_t lo() { return 0xffffffffu; }
  __device__ static uint32_t hi() { return 0u; }
};
template <>
struct MinMaxId<s64> {
  __device__ static s64 lo() { return 0x7fffffffffffffffll; }
  __device__ static s64 hi() { return (s64)0x8000000000000000ull; }
};
template <>
struct MinMaxId<bf16> {
  __device__ static bf16 lo() { return bf16(0x7f80, true); }  // +inf
  __device__ static bf16 hi() { return bf16(0xff80, true); }  // -inf
};
template <>
struct MinMaxId<f16> {
  __device__ static f16 lo() { return f16(0x7c00, true); }
  __device__ static f16 hi() { return f16(0xfc00, true); }
};
template <>
struct MinMaxId<e4m3> {  // no infinities: the largest finite magnitudes (+-448)
  __device__ static e4m3 lo() { return e4m3(0x7e, true); }
  __device__ static e4m3 hi() { return e4m3(0xfe, true); }
};
template <>
struct MinMaxId<e5m2> {  // +-inf
  __device__ static e5m2 lo() { return e5m2(0x7c, true); }
  __device__ static e5m2 hi() { return e5m2(0xfc, true); }
};

// Sum type: f64 for floats, u64 (modular) for integers.
template <class T>
struct SumT {
  typedef double type;
};
template <>
struct SumT<uint32_t> {
  typedef u64 type;
};
template <>
struct SumT<s64> {
  typedef u64 type;
};

template <class S>
__device__ __forceinline__ S sum_add(S a, S b);
template <>
__device__ __forceinline__ double sum_add<double>(double a, double b) {
  return __dadd_rn(a, b);
}
template <>
__device__ __forceinline__ u64 sum_add<u64>(u64 a, u64 b) {
  return a + b;
}

// Pairwise sum of a unit (or one element) in eT, then widened.  For f32 the
// unit of 4 is ((v0+v1)+(v2+v3)) in f32 — one f32->f64 conversion per unit.
// Pairwise f32 sum of W (power of two) f32 values.
template <int W>
__device__ __forceinline__ float pairwise_f32(const float (&x)[W]) {
  if constexpr (W == 1) {
    return x[0];
  } else {
    float h[W / 2];
#pragma unroll
    for (int w = 0; w < W / 2; ++w) h[w] = __fadd_rn(x[2 * w], x[2 * w + 1]);
    return pairwise_f32<W / 2>(h);
  }
}

// ---- 16-bit views of narrow elements and the mixed-precision add ------------
// Every bf16 / f16 / E4M3 / E5M2 value is exactly a 16-bit value: bf16 itself,
// the others f16 (8-bit types decoded two per cvt).  add.rn.f32.{f16,bf16}
// (sm_100 FHADD) adds such a value to an f32 and rounds once — exactly
// RN(widen(a) + c), one instruction instead of a widening plus an FADD.
template <class T>
__device__ __forceinline__ void to_h16(const T (&v)[2], unsigned short (&h)[2]) {
  if constexpr (is_half<T>()) {
    h[0] = v[0].bits;
    h[1] = v[1].bits;
  } else {
    const unsigned short pk = (unsigned short)(v[0].bits | ((unsigned)v[1].bits << 8));
    unsigned h2;
    if constexpr (std::is_same<T, e4m3>::value)
      asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(pk));
    else
      h2 = __byte_perm((unsigned)pk, 0u, 0x1404);
    h[0] = (unsigned short)(h2 & 0xffffu);
    h[1] = (unsigned short)(h2 >> 16);
  }
}
template <class T>
__device__ __forceinline__ float h16_to_f32(unsigned short h) {
  if constexpr (std::is_same<T, bf16>::value) return __uint_as_float((unsigned)h << 16);
  else return __half2float(__ushort_as_half(h));
}
template <class T>
__device__ __forceinline__ float add_f32_h16(float c, unsigned short h) {
  float d;
  if constexpr (std::is_same<T, bf16>::value)
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(d) : "h"(h), "f"(c));
  else
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(d) : "h"(h), "f"(c));
  return d;
}
// widen(a) + widen(b), rounded once to f32, from the 16-bit views
template <class T>
__device__ __forceinline__ float pair_sum_h16(unsigned short a, unsigned short b) {
  return add_f32_h16<T>(h16_to_f32<T>(a), b);
}

template <class T, int W>
__device__ __forceinline__ typename SumT<T>::type unit_sum(const T (&v)[W]) {
  if constexpr (is_narrow<T>() && W >= 2) {
    // pairwise sum in f32 of the exact values (error ~2^-24, far below the
    // format's 2^-9 / 2^-12 rounding; E4M3 unit sums are exact), the first
    // level as mixed-precision adds; one conversion to f64 per unit
    float x[W / 2];
#pragma unroll
    for (int w = 0; w < W / 2; ++w) {
      unsigned short h[2];
      to_h16<T>({v[2 * w], v[2 * w + 1]}, h);
      x[w] = pair_sum_h16<T>(h[0], h[1]);
    }
    return (double)pairwise_f32<W / 2>(x);
  } else if constexpr (is_narrow<T>()) {
    return (double)as_float(v[0]);
  } else if constexpr (is_float<T>()) {
    if constexpr (W == 1) {
      return (double)v[0];
    } else if constexpr (W == 2) {
      return (double)bin<COOT_OP_ADD>(v[0], v[1]);
    } else {
      static_assert(W == 4, "unit");
      return (double)bin<COOT_OP_ADD>(bin<COOT_OP_ADD>(v[0], v[1]), bin<COOT_OP_ADD>(v[2], v[3]));
    }
  } else {
    u64 s = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) s += (u64)v[w];
    return s;
  }
}

// Sums of squares inside a unit in f32 (norm2, var): trusted when the f32 sum
// u is a normal number >= 2^-100 — then no square overflowed (u would be inf)
// and squares that fell below 2^-126 are < 2^-26 of u.  Anything else (inf,
// NaN, tiny, 0) sends the unit to f64.  Only bf16 and f32 values can leave the
// range (f16 / E4M3 / E5M2 squares are exact normal f32 values or 0).
template <class T>
__host__ __device__ constexpr bool sq_range_checked() {
  return std::is_same<T, float>::value || std::is_same<T, bf16>::value;
}
__device__ __forceinline__ bool sq_sum_ok(float u) {
  return u >= 0x1p-100f && u <= 3.40282347e38f;
}
// sum of exact f64 squares of W f32 values, in element order
template <int W>
__device__ __forceinline__ double sumsq_f64(const float (&x)[W]) {
  double r = 0.0;
#pragma unroll
  for (int w = 0; w < W; ++w) r = __fma_rn((double)x[w], (double)x[w], r);
  return r;
}

// f64 sums of squares over the whole f64 range (norm2, R12): value = s * 2^es
// (es even).  Units whose squares are normal numbers well inside the range add
// to s directly while es == 0 (the common case: one compare more than a plain
// sum); any other unit (a square outside [2^-900, 2^900], huge or tiny values,
// subnormals, non-finite) is squared after an exact power-of-two scaling by its
// largest exponent and merged with exponent alignment, and a merged s above
// 2^900 is renormalised — so neither a square nor the sum overflows or flushes
// (an f64 norm2 of 1e200-sized data was inf; of 1e-200-sized data 0).
__device__ __forceinline__ void sq_merge_scaled(double& s, int& es, double o, int eo) {
  if (o == 0.0) return;
  if (s == 0.0) {
    s = o;
    es = eo;
  } else if (eo > es) {
    s = __dadd_rn(scalbn(s, es - eo), o);
    es = eo;
  } else {
    s = __dadd_rn(s, scalbn(o, eo - es));
  }
  if (s > 0x1p900 && s <= 1.7976931348623157e308) {  // keep the sum far from overflow
    s = scalbn(s, -400);
    es += 400;
  }
}
// The scaled add of one f64 unit (W <= 2 values: v1 unused when w2 is false).
// Arguments and result by value: a noinline callee taking the accumulator by
// reference pins it to local memory in the hot loop (f64 norm2 7.2 -> 4.7 TB/s).
struct SqAcc {
  double s;
  int es;
};
static __device__ __noinline__ SqAcc sq_add_scaled(double s, int es, double v0, double v1, bool w2) {
  SqAcc r{s, es};
  const double a0 = fabs(v0), a1 = w2 ? fabs(v1) : 0.0;
  const double kMax = 1.7976931348623157e308;
  if (!(a0 <= kMax) || !(a1 <= kMax)) {  // inf / NaN propagate: inf^2 = inf, NaN stays NaN
    r.s = __dadd_rn(r.s, __fma_rn(v0, v0, w2 ? __dmul_rn(v1, v1) : 0.0));
    return r;
  }
  int m = -2000;
  if (a0 != 0.0) m = ilogb(a0) + 1;
  if (a1 != 0.0) m = max(m, ilogb(a1) + 1);
  if (m == -2000) return r;  // all zeros
  // the unit's squares scaled by 2^-2m (the largest lies in [1/4, 1))
  const double x0 = scalbn(v0, -m), x1 = w2 ? scalbn(v1, -m) : 0.0;
  sq_merge_scaled(r.s, r.es, __fma_rn(x1, x1, __dmul_rn(x0, x0)), 2 * m);
  return r;
}

// Per-thread / per-block / per-rank accumulator for every reduction kind.
//  ACC_SUM, ACC_SUMSQ: s (f64 for floats, u64 modular for ints)
//  ACC_MINMAX:         mn, mx
//  ACC_VAR:            n elements, shift c, s1 = sum(x - c), s2 = sum(x - c)^2 in
//                      f64 (c = the thread's first element, so the shifted sums
//                      do not cancel); merged with Chan et al.'s pairwise update,
//                      after which c is the mean, s1 = 0 and s2 = M2
//  ACC_IMIN, ACC_IMAX: best value + its (first) global index
template <class T, int ACC>
struct Accum {
  typedef typename SumT<T>::type S;
  S s;
  T mn, mx;
  u64 n, idx;
  double c, s1, s2;
  float cf;  // VAR on f32 / 16-bit / 8-bit: the shift c as f32 (exact: c is an element)
  bool has;  // IMIN / IMAX: an element has been seen (hot-loop copy of idx != ~0)
  int es;    // SUMSQ on f64: the sum is s * 2^es (sq_add_scaled)
  __device__ __forceinline__ void init() {
    s = S(0);
    es = 0;
    mn = MinMaxId<T>::lo();
    mx = MinMaxId<T>::hi();
    n = 0;
    idx = ~0ull;
    c = s1 = s2 = 0.0;
    cf = 0.f;
    has = false;
  }
  // Accumulate W consecutive elements whose first element has global index
  // `base` (only the index-returning kinds use it).
  template <int W>
  __device__ __forceinline__ void add_at(const T (&v)[W], u64 base) {
    if constexpr (ACC == ACC_IMIN || ACC == ACC_IMAX) {
      // best of the unit first (strict comparisons: the first occurrence wins,
      // indices increase within a thread), then one comparison with the
      // running best; the sentinel idx admits the very first element
      T bv = v[0];
      int bw = 0;
#pragma unroll
      for (int w = 1; w < W; ++w) {
        const bool better = (ACC == ACC_IMIN) ? lt(v[w], bv) : lt(bv, v[w]);
        bv = better ? v[w] : bv;
        bw = better ? w : bw;
      }
      const bool better = (ACC == ACC_IMIN) ? lt(bv, mn) : lt(mx, bv);
      if (!has || better) {
        if constexpr (ACC == ACC_IMIN) mn = bv;
        else mx = bv;
        idx = base + (u64)bw;
        has = true;
      }
    } else {
      add<W>(v);
    }
  }
  template <int W>
  __device__ __forceinline__ void add(const T (&v)[W]) {
    if constexpr (ACC == ACC_VAR) {
      if (n == 0) {  // the shift: the thread's first element
        c = as_double(v[0]);
        if constexpr (!std::is_same<T, double>::value && is_float<T>()) cf = as_float(v[0]);
      }
      if constexpr (std::is_same<T, double>::value || !is_float<T>()) {
        double a1 = 0.0, a2 = 0.0;  // the unit's shifted sums, then one update each
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const double d = __dsub_rn(as_double(v[w]), c);
          a1 = __dadd_rn(a1, d);
          a2 = __fma_rn(d, d, a2);
        }
        s1 = __dadd_rn(s1, a1);
        s2 = __dadd_rn(s2, a2);
      } else {
        // f32 / 16-bit: the unit's shifted sums in f32 (the shift is an element,
        // so exact in f32; x - c is exact when x is near c), widened to f64 once
        // per unit — relative error ~W * 2^-24, far inside the 1e-5 bar
        float a1 = 0.f, a2 = 0.f;
        if constexpr (is_narrow<T>() && W >= 2) {
          // d = RN(x - c) straight from the 16-bit view (add.rn.f32.{bf16,f16}
          // of -c: one FHADD instead of a widening and an FSUB, same bits)
#pragma unroll
          for (int w = 0; w + 1 < W; w += 2) {
            unsigned short h[2];
            to_h16<T>({v[w], v[w + 1]}, h);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const float d = add_f32_h16<T>(-cf, h[k]);
              a1 = __fadd_rn(a1, d);
              a2 = __fmaf_rn(d, d, a2);
            }
          }
        } else {
          float x[W];
          widen_f32<T, W>(v, x);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const float d = __fsub_rn(x[w], cf);
            a1 = __fadd_rn(a1, d);
            a2 = __fmaf_rn(d, d, a2);
          }
        }
        if (__builtin_expect(!sq_range_checked<T>() || sq_sum_ok(a2), 1)) {
          s1 = __dadd_rn(s1, (double)a1);
          s2 = __dadd_rn(s2, (double)a2);
        } else {
          // squared deviations left f32's range (x - c or a square overflowed,
          // or all are tiny), or the unit equals the shift: shifted sums in f64
          float x[W];
          widen_f32<T, W>(v, x);
          double b1 = 0.0, b2 = 0.0;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const double e = __dsub_rn((double)x[w], c);
            b1 = __dadd_rn(b1, e);
            b2 = __fma_rn(e, e, b2);
          }
          s1 = __dadd_rn(s1, b1);
          s2 = __dadd_rn(s2, b2);
        }
      }
      n += W;
    } else if constexpr (ACC == ACC_SUM) {
      s = sum_add<S>(s, unit_sum<T, W>(v));
    } else if constexpr (ACC == ACC_SUMSQ) {
      if constexpr (is_narrow<T>() || std::is_same<T, float>::value) {
        // squares in f32 (exact for 16/8-bit values), summed pairwise in f32.
        // bf16 / f32 only: a unit whose f32 sum is not a normal number >= 2^-100
        // (a square overflowed, or every square is tiny and may have lost its
        // bits, or the unit is zero / non-finite) is redone in f64 — so norm2
        // is accurate over the whole range at one compare per unit
        float q[W];
        widen_f32<T, W>(v, q);
        float qq[W];
#pragma unroll
        for (int w = 0; w < W; ++w) qq[w] = __fmul_rn(q[w], q[w]);
        const float u = pairwise_f32<W>(qq);
        if (__builtin_expect(!sq_range_checked<T>() || sq_sum_ok(u), 1))
          s = sum_add<S>(s, (double)u);
        else
          s = sum_add<S>(s, sumsq_f64<W>(q));
      } else if constexpr (std::is_same<T, double>::value) {
        T q[W];
#pragma unroll
        for (int w = 0; w < W; ++w) q[w] = bin<COOT_OP_MUL>(v[w], v[w]);
        const double u = unit_sum<T, W>(q);
        bool zero = true;  // u == 0 from squares that flushed is not a zero unit
#pragma unroll
        for (int w = 0; w < W; ++w) zero = zero && (v[w] == 0.0);
        // (a thread adds far fewer than 2^100 units of <= 2^901 each: s cannot
        // overflow here; merges renormalise — no test on the s chain per unit)
        if (__builtin_expect(es == 0 && ((u >= 0x1p-900 && u <= 0x1p900) || zero), 1)) {
          s = __dadd_rn(s, u);
        } else {
          static_assert(W <= 2, "f64 units hold at most 2 elements");
          const SqAcc r = sq_add_scaled(s, es, v[0], W > 1 ? v[W - 1] : 0.0, W > 1);
          s = r.s;
          es = r.es;
        }
      } else {
        T q[W];
#pragma unroll
        for (int w = 0; w < W; ++w) q[w] = bin<COOT_OP_MUL>(v[w], v[w]);
        s = sum_add<S>(s, unit_sum<T, W>(q));
      }
    } else if constexpr (ACC == ACC_MINMAX) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        mn = bin<COOT_OP_MIN>(mn, v[w]);
        mx = bin<COOT_OP_MAX>(mx, v[w]);
      }
    }
  }
  // Fixed xor-butterfly (a deterministic tree per lane).
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      if constexpr (ACC == ACC_SUMSQ && std::is_same<T, double>::value) {
        const double o = shfl_xor(s, m);
        const int eo = __shfl_xor_sync(0xffffffffu, es, m);
        sq_merge_scaled(s, es, o, eo);
      } else if constexpr (ACC == ACC_SUM || ACC == ACC_SUMSQ) {
        s = sum_add<S>(s, shfl_xor(s, m));
      } else if constexpr (ACC == ACC_MINMAX) {
        mn = bin<COOT_OP_MIN>(mn, shfl_xor(mn, m));
        mx = bin<COOT_OP_MAX>(mx, shfl_xor(mx, m));
      } else if constexpr (ACC != ACC_NONE) {
        Accum o = *this;
        o.n = shfl_xor((u64)n, m);
        o.idx = shfl_xor((u64)idx, m);
        o.c = shfl_xor(c, m);
        o.s1 = shfl_xor(s1, m);
        o.s2 = shfl_xor(s2, m);
        o.mn = shfl_xor(mn, m);
        o.mx = shfl_xor(mx, m);
        merge(o);
      }
    }
  }
  __device__ __forceinline__ void merge(const Accum& o) {
    if constexpr (ACC == ACC_SUMSQ && std::is_same<T, double>::value) {
      sq_merge_scaled(s, es, o.s, o.es);
    } else if constexpr (ACC == ACC_SUM || ACC == ACC_SUMSQ) {
      s = sum_add<S>(s, o.s);
    } else if constexpr (ACC == ACC_MINMAX) {
      mn = bin<COOT_OP_MIN>(mn, o.mn);
      mx = bin<COOT_OP_MAX>(mx, o.mx);
    } else if constexpr (ACC == ACC_VAR) {
      if (o.n == 0) return;
      if (n == 0) {
        *this = o;
        return;
      }
      // (n, mean, M2) of both sides, then Chan's pairwise combination
      const double na = (double)n, nb = (double)o.n, nab = (double)(n + o.n);
      const double ma = __dadd_rn(c, __ddiv_rn(s1, na));
      const double mb = __dadd_rn(o.c, __ddiv_rn(o.s1, nb));
      const double m2a = __dsub_rn(s2, __ddiv_rn(__dmul_rn(s1, s1), na));
      const double m2b = __dsub_rn(o.s2, __ddiv_rn(__dmul_rn(o.s1, o.s1), nb));
      const double delta = __dsub_rn(mb, ma);
      c = __dadd_rn(ma, __ddiv_rn(__dmul_rn(delta, nb), nab));
      s2 = __dadd_rn(__dadd_rn(m2a, m2b),
                     __ddiv_rn(__dmul_rn(__dmul_rn(delta, delta), __dmul_rn(na, nb)), nab));
      s1 = 0.0;
      n += o.n;
    } else if constexpr (ACC == ACC_IMIN || ACC == ACC_IMAX) {
      if (o.idx == ~0ull) return;
      const T ov = ACC == ACC_IMIN ? o.mn : o.mx, v = ACC == ACC_IMIN ? mn : mx;
      const bool better = ACC == ACC_IMIN ? lt(ov, v) : lt(v, ov);
      if (idx == ~0ull || better || (!lt(v, ov) && !lt(ov, v) && o.idx < idx)) {
        mn = o.mn;
        mx = o.mx;
        idx = o.idx;
      }
    }
  }
  __device__ __forceinline__ Rec to_rec(u64 count) const {
    Rec r;
    r.count = count;
    r.pad = 0;
    if constexpr (ACC == ACC_MINMAX) {
      r.a = to_bits<T>(mn);
      r.b = to_bits<T>(mx);
    } else if constexpr (ACC == ACC_VAR) {
      // (mean, M2, n): the merged form of the shifted sums
      const double mean = n ? __dadd_rn(c, __ddiv_rn(s1, (double)n)) : 0.0;
      const double m2 = n ? __dsub_rn(s2, __ddiv_rn(__dmul_rn(s1, s1), (double)n)) : 0.0;
      r.a = (u64)__double_as_longlong(mean);
      r.b = (u64)__double_as_longlong(m2);
      r.count = n;
    } else if constexpr (ACC == ACC_IMIN || ACC == ACC_IMAX) {
      r.a = to_bits<T>(ACC == ACC_IMIN ? mn : mx);
      r.b = idx;
    } else if constexpr (is_float<T>()) {
      r.a = (u64)__double_as_longlong((double)s);
      r.b = (u64)(long long)es;  // 0 except for f64 SUMSQ (the scale exponent)
    } else {
      r.a = (u64)s;
      r.b = 0;
    }
    return r;
  }
  __device__ __forceinline__ void from_rec(const Rec& r) {
    init();
    if constexpr (ACC == ACC_MINMAX) {
      // empty producers publish the identities (+inf/-inf, UINT_MAX/0, ...)
      mn = scalar_as<T>(r.a);
      mx = scalar_as<T>(r.b);
    } else if constexpr (ACC == ACC_VAR) {
      c = __longlong_as_double((long long)r.a);
      s2 = __longlong_as_double((long long)r.b);
      s1 = 0.0;
      n = r.count;
    } else if constexpr (ACC == ACC_IMIN || ACC == ACC_IMAX) {
      mn = mx = scalar_as<T>(r.a);
      idx = r.b;
    } else if constexpr (is_float<T>()) {
      s = __longlong_as_double((long long)r.a);
      if constexpr (ACC == ACC_SUMSQ && std::is_same<T, double>::value) es = (int)(long long)r.b;
    } else {
      s = r.a;
    }
  }
};

// Programmatic dependent launch (coot_launch.cuh launch_k).  pdl_wait() is the
// first statement of every kernel launched that way: it blocks until the
// previous grid on the stream has completed and its writes are visible.
// pdl_trigger() — issued by the fused kernels once their streaming loop is
// done — lets the next kernel's CTAs be scheduled during this one's final
// reduction (without it they launch when this grid completes).  Triggering
// at kernel start instead measured 10-20 % slower on low-register kernels
// (var / index_min / norm2): the early CTAs sat on the SMs for the whole run.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Load a record written by another block of this grid (bypass L1).
__device__ __forceinline__ Rec load_rec_cg(const Rec* p) {
  Rec r;
  r.a = __ldcg(&p->a);
  r.b = __ldcg(&p->b);
  r.count = __ldcg(&p->count);
  r.pad = 0;
  return r;
}

template <class T>
__device__ __forceinline__ T round_to(double x) {
  if constexpr (is_half<T>()) return half_from_f64<T>(x);
  else if constexpr (sizeof(T) == 4 && is_float<T>()) return __double2float_rn(x);
  else return (T)x;
}

// the result-type value of an element (exact: the 8-bit types widen to f32)
template <class T>
__device__ __forceinline__ typename ResultT<T>::type as_result(T v) {
  if constexpr (is_fp8<T>()) return to_f32(v);
  else return v;
}

// Round the combined accumulator into the user-visible result (ResultT<eT>,
// or a u64 index).  `count` = number of elements reduced (MEAN's divisor).
template <class T, int ACC>
__device__ __forceinline__ void write_final(const Accum<T, ACC>& acc, uint32_t kind, void* result,
                                            u64 count) {
  typedef typename ResultT<T>::type R;
  R* out = reinterpret_cast<R*>(result);
  if constexpr (ACC == ACC_VAR) {
    const double var = acc.n > 1 ? __ddiv_rn(acc.s2 - __ddiv_rn(__dmul_rn(acc.s1, acc.s1),
                                                                (double)acc.n),
                                             (double)(acc.n - 1))
                                 : 0.0;
    const double v = var > 0.0 ? var : 0.0;
    out[0] = round_to<R>(kind == COOT_RED_STDDEV ? __dsqrt_rn(v) : v);
  } else if constexpr (ACC == ACC_IMIN || ACC == ACC_IMAX) {
    *reinterpret_cast<u64*>(result) = acc.idx;
  } else if constexpr (ACC == ACC_SUM && is_float<T>()) {
    if (kind == COOT_RED_MEAN) out[0] = round_to<R>(__ddiv_rn(acc.s, (double)count));
    else out[0] = round_to<R>(acc.s);
  } else if constexpr (ACC == ACC_MINMAX) {
    if (kind == COOT_RED_MIN) out[0] = as_result(acc.mn);
    else if (kind == COOT_RED_MAX) out[0] = as_result(acc.mx);
    else {
      out[0] = as_result(acc.mn);
      out[1] = as_result(acc.mx);
    }
  } else if constexpr (ACC == ACC_SUMSQ) {
    if constexpr (std::is_same<T, double>::value)
      out[0] = scalbn(__dsqrt_rn(acc.s), acc.es / 2);  // es is even: exact scaling
    else
      out[0] = round_to<R>(__dsqrt_rn(acc.s));
  } else if constexpr (ACC == ACC_SUM) {
    if constexpr (is_float<T>()) {
      out[0] = round_to<R>(acc.s);
    } else {
      out[0] = (T)acc.s;  // modular truncation for u32
    }
  }
}

// Block-level fixed-order reduction of per-thread accumulators; returns the
// block total in thread 0 (other threads: unspecified).
template <class T, int ACC>
__device__ __forceinline__ Accum<T, ACC> block_reduce(Accum<T, ACC> acc) {
  __shared__ Accum<T, ACC> ws[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (int)(blockDim.x >> 5);
  acc.warp_reduce();
  if (lane == 0) ws[warp] = acc;
  __syncthreads();
  Accum<T, ACC> r;
  r.init();
  if (warp == 0) {
    if (lane < nwarps) r = ws[lane];
    r.warp_reduce();
  }
  __syncthreads();
  return r;
}

// Merge partial records of consecutive shards in rank order 0..nparts-1 and
// round once into `result` (index reductions: shard-local index + the element
// count of the shards before it).  Shared by coot_combine and the exchange.
template <class T, int ACC, class LoadRec>
__device__ __forceinline__ void combine_in_order(uint32_t nparts, LoadRec load, uint32_t kind,
                                                 void* result) {
  Accum<T, ACC> acc;
  acc.init();
  u64 before = 0;
  for (uint32_t p = 0; p < nparts; ++p) {
    const Rec r = load(p);
    Accum<T, ACC> o;
    o.from_rec(r);
    if constexpr (ACC == ACC_IMIN || ACC == ACC_IMAX) {
      if (o.idx != ~0ull) o.idx += before;  // shard-local -> global index
    }
    acc.merge(o);
    before += r.count;
  }
  write_final<T, ACC>(acc, kind, result, before);
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// FINAL_EXCHANGE, one thread.  Mailbox layout: records slot[2][MAX_RANKS]
// (double-buffered by epoch parity), then u64 flag[MAX_RANKS].  Publish this
// rank's record into slot[epoch & 1][rank] of every peer's mailbox (remote
// stores over NVLink / peer memory), then raise flag[rank] = epoch there
// (system-scope release: the record is visible before the flag); wait until
// every flag of the OWN mailbox reaches epoch (acquire) and combine
// slot[epoch & 1][0..P) in rank order.  Parity buffering: a fast rank's record
// for epoch e+1 lands in the other half, and it cannot reach e+2 before this
// rank has raised its e+1 flags, i.e. finished reading epoch e.  A peer that
// never arrives -> trap after ~20 s (the host sees a device fault).
template <class T, int ACC>
__device__ void exchange_finish(const Rec& mine, const Exchange& ex, uint32_t kind, void* result) {
  const uint32_t P = ex.nranks;
  const unsigned long long half = (ex.epoch & 1ull) * COOT_MAX_RANKS;
  const unsigned long long flag_off = 2ull * COOT_MAX_RANKS * sizeof(Rec);
  for (uint32_t p = 0; p < P; ++p) {
    Rec* slot = reinterpret_cast<Rec*>(ex.mbox[p]) + half + ex.rank;
    __stcg(&slot->a, mine.a);
    __stcg(&slot->b, mine.b);
    __stcg(&slot->count, mine.count);
    __stcg(&slot->pad, ex.epoch);  // which call this record belongs to
  }
  __threadfence_system();
  for (uint32_t p = 0; p < P; ++p)
    st_release_sys(reinterpret_cast<unsigned long long*>(ex.mbox[p] + flag_off) + ex.rank,
                   ex.epoch);
  const unsigned long long* own =
      reinterpret_cast<const unsigned long long*>(ex.mbox[ex.rank] + flag_off);
  const unsigned long long t0 = globaltimer_ns();
  for (uint32_t q = 0; q < P; ++q) {
    while (ld_acquire_sys(own + q) < ex.epoch) {
      __nanosleep(256);
      if (globaltimer_ns() - t0 > 20000000000ull) __trap();  // a rank never arrived
    }
  }
  const Rec* slots = reinterpret_cast<const Rec*>(ex.mbox[ex.rank]) + half;
  // every record must be this call's: a peer whose flag passed `epoch` without
  // writing epoch's record (it skipped a call) is a protocol fault, not data
  for (uint32_t q = 0; q < P; ++q)
    if (__ldcg(&slots[q].pad) != ex.epoch) __trap();
  combine_in_order<T, ACC>(P, [&](uint32_t q) { return load_rec_cg(slots + q); }, kind, result);
}

// Deterministic single-launch finish: every block publishes a record; the
// last block to arrive (ticket) combines ALL records in a fixed order (a
// function of the grid and block size only: block-strided per thread, then
// block_reduce's fixed tree) and rounds once.  The ticket
// self-resets so the next launch on the stream can reuse it.
template <class T, int ACC>
__device__ __forceinline__ void grid_finish(const Accum<T, ACC>& block_total, Rec* partials,
                                            unsigned* ticket, uint32_t final_mode,
                                            uint32_t kind, void* result, u64 count,
                                            const Exchange& ex) {
  __shared__ bool am_last;
  if (gridDim.x == 1) {
    // a one-CTA grid (n of one tile or less): the same arithmetic as the last-
    // block path below — its one record merged into an empty accumulator, then
    // a block tree — without the record store, the ticket atomic and the
    // record load (three dependent L2 round trips)
    Accum<T, ACC> acc;
    acc.init();
    if (threadIdx.x == 0) {
      Accum<T, ACC> o;
      o.from_rec(block_total.to_rec(0));
      acc.merge(o);
    }
    const Accum<T, ACC> tot = block_reduce<T, ACC>(acc);
    if (threadIdx.x == 0) {
      if (final_mode == FINAL_PARTIAL) {
        *reinterpret_cast<Rec*>(result) = tot.to_rec(count);
      } else if (final_mode == FINAL_EXCHANGE) {
        exchange_finish<T, ACC>(tot.to_rec(count), ex, kind, result);
      } else {
        write_final<T, ACC>(tot, kind, result, count);
      }
    }
    return;
  }
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = block_total.to_rec(0);
    // acq_rel: releases this block's record, and (for the last arrival)
    // acquires every other block's — no separate membar.gl on either side
    const unsigned t = atom_add_acq_rel_gpu(ticket, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();  // extends thread 0's acquire to the whole block
  if (!am_last) return;
  // the last block loads the records with all its threads (one L2 round trip
  // for grids <= blockDim), then reduces them in a fixed tree: thread t merges
  // records t, t + blockDim, ... in order, then block_reduce
  Accum<T, ACC> acc;
  acc.init();
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    Accum<T, ACC> o;
    o.from_rec(load_rec_cg(&partials[b]));
    acc.merge(o);
  }
  const Accum<T, ACC> tot = block_reduce<T, ACC>(acc);
  if (threadIdx.x == 0) {
    *ticket = 0u;
    if (final_mode == FINAL_PARTIAL) {
      *reinterpret_cast<Rec*>(result) = tot.to_rec(count);
    } else if (final_mode == FINAL_EXCHANGE) {
      exchange_finish<T, ACC>(tot.to_rec(count), ex, kind, result);
    } else {
      write_final<T, ACC>(tot, kind, result, count);
    }
  }
}

}  // namespace coot
