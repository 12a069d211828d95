// K1 (templated catalog) and K2 (warp-uniform register interpreter) fused
// element-wise + terminal-reduction kernels.
//
// Both evaluators run inside the SAME driver loop (fused_tma_kernel by
// default, fused_kernel as the register-pipelined alternative), so the element
// -> thread map and the accumulation order are identical: for the same
// expression and grid, K1 and K2 produce bit-identical results.
//
// Element semantics live in coot_device.cuh; operands reach an evaluator
// through a "source": RegSrc (values already in registers) or SmemSrc (a
// 16-byte unit in the TMA-staged shared-memory tile, read on LOAD).
#pragma once
#include "coot_catalog.h"
#include "coot_device.cuh"

// Minimum resident CTAs per SM requested from ptxas for catalog kernels of the
// LDG driver (bounds registers at 65536 / (256 * MINB)).
#ifndef COOT_CAT_MINB
#define COOT_CAT_MINB 2
#endif

namespace coot {

__host__ __device__ constexpr int ins_op(int c) { return c >> 4; }
__host__ __device__ constexpr int ins_arg(int c) { return c & 15; }
__host__ __device__ constexpr bool is_unary_op(int op) {
  return op >= COOT_OP_NEG && op <= COOT_OP_LOG;
}

// ---- operand sources -----------------------------------------------------------
template <class T, int K, int W>
struct RegSrc {
  const T (&in)[K][W];
  template <int k>
  __device__ __forceinline__ void get_c(T (&v)[W]) const {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = in[k][w];
  }
  __device__ __forceinline__ void get(int k, T (&v)[W]) const {
    switch (k) {
#define COOT_RS(c)                             \
  case c:                                      \
    if constexpr ((c) < K) get_c<(c) < K ? (c) : 0>(v); \
    break;
      COOT_RS(0) COOT_RS(1) COOT_RS(2) COOT_RS(3) COOT_RS(4) COOT_RS(5) COOT_RS(6) COOT_RS(7)
#undef COOT_RS
      default:
        break;
    }
  }
};

// UD 16-byte units of operand k: stage + k * stride + (i + j * 256) * 16.
template <class T, int UD>
struct SmemSrc {
  static constexpr int WU = Unit<T>::W;
  const unsigned char* p;  // = stage base + i * 16
  uint32_t stride;         // bytes between operands in the stage
  template <int k>
  __device__ __forceinline__ void get_c(T (&v)[UD * WU]) const {
    get(k, v);
  }
  __device__ __forceinline__ void get(int k, T (&v)[UD * WU]) const {
#pragma unroll
    for (int j = 0; j < UD; ++j) {
      const uint4 r = lds16(p + (size_t)k * stride + (size_t)j * 256 * 16);
      memcpy(&v[j * WU], &r, 16);
    }
  }
};

// ---- K1: compile-time program ------------------------------------------------
template <int... Code>
struct StaticProg {
  static constexpr int n_instr = sizeof...(Code);
  static constexpr int codes[sizeof...(Code)] = {Code...};
  static constexpr int n_ops() {
    int k = 0;
    for (int i = 0; i < n_instr; ++i)
      if (ins_op(codes[i]) == COOT_OP_LOAD && ins_arg(codes[i]) + 1 > k) k = ins_arg(codes[i]) + 1;
    return k;
  }
  template <class T>
  static constexpr bool legal() {
    for (int i = 0; i < n_instr; ++i)
      if (!op_legal<T>(ins_op(codes[i]))) return false;
    return true;
  }
};

// LOAD into the arithmetic-type stack (a plain copy unless T is an 8-bit
// storage type, which is decoded to f32).
template <class T, int W, class Src>
__device__ __forceinline__ void load_to(const Src& src, int k,
                                        typename ComputeT<T>::type (&dst)[W]) {
  if constexpr (std::is_same<typename ComputeT<T>::type, T>::value) {
    src.get(k, dst);
  } else {
    T raw[W];
    src.get(k, raw);
    widen_vec<T, W>(raw, dst);
  }
}

// The stack holds ComputeT<T> (T itself except for the 8-bit storage types,
// whose programs run in f32); results are narrowed back to T at the end.
template <class T, int W, int SP, int C, int... Rest>
struct StaticStep {
  typedef typename ComputeT<T>::type CT;
  template <class Src>
  __device__ __forceinline__ static void run(CT (&st)[COOT_MAX_STACK][W], const Src& src,
                                             const FusedArgs& a) {
    constexpr int op = ins_op(C), arg = ins_arg(C);
    constexpr int nsp = (op == COOT_OP_LOAD || op == COOT_OP_SCALAR) ? SP + 1
                        : is_unary_op(op)                            ? SP
                                                                     : SP - 1;
    if constexpr (op == COOT_OP_LOAD) {
      load_to<T, W>(src, arg, st[SP]);
    } else if constexpr (op == COOT_OP_SCALAR) {
      const CT s = scalar_as<CT>(a.scalars[arg]);
#pragma unroll
      for (int w = 0; w < W; ++w) st[SP][w] = s;
    } else if constexpr (is_unary_op(op)) {
      un_vec<op>(st[SP - 1]);
    } else {
      bin_vec<op>(st[SP - 2], st[SP - 1]);
    }
    if constexpr (sizeof...(Rest) > 0) StaticStep<T, W, nsp, Rest...>::run(st, src, a);
  }
};

// ---- fp8 storage, catalog c2 (exp(A % B) + s*C): cheap EXP, verified ------
// R25 makes an fp8 program an f32 program whose FINAL value is rounded once
// to the 8-bit format.  For c2 the device may therefore evaluate EXP with the
// cheap CUDA expf (<= 2 ulp) instead of the correctly rounded f32 EXP (R6) as
// long as the final 8-bit result provably cannot differ.  With E = RN32(e^x)
// (the exact program's node) and E' = expf(x): |E' - E| <= 2.5 ulp(E'), and
// the exact z = RN32(E + t), the fast z' = RN32(E' + t) (t = RN32(s C), any
// sign) differ by at most D0 = |E' - E| + 2 ulp(z') <= |E'| 2^-21 + |z'| 2^-22.
// The test brackets z' by lo = RN32(z' - D), hi = RN32(z' + D) with D = 2 D0
// (covers the half-ulp rounding of lo / hi) and narrows both: RN8 (saturating)
// is monotone, so if RN8(lo) == RN8(hi) (same byte), RN8(z) is that byte.
// x = A % B = 0 gives E' = E = 1 exactly: D = 0.  Undecided (a bracket that
// straddles an 8-bit rounding boundary, or a non-finite E'): the whole
// dispatch is recomputed with the exact program.
// the exact program over the whole dispatch (the rare undecided case):
// operands reloaded from the source, the correctly rounded f32 EXP (R6)
template <class T, int W, class Src>
__device__ __noinline__ void fp8_c2_exact(const Src& src, float sc, float (&z)[W]) {
  float y[W];
  load_to<T, W>(src, 0, z);
  load_to<T, W>(src, 1, y);
#pragma unroll 1
  for (int w = 0; w < W; ++w) z[w] = crm::cr_expf(bin<COOT_OP_MUL>(z[w], y[w]));
  load_to<T, W>(src, 2, y);
#pragma unroll 1
  for (int w = 0; w < W; ++w) z[w] = bin<COOT_OP_ADD>(z[w], bin<COOT_OP_MUL>(sc, y[w]));
}
template <int... Code>
struct IsC2 {
  static constexpr bool value = false;
};
template <>
struct IsC2<COOT_OP_LOAD << 4, (COOT_OP_LOAD << 4) | 1, COOT_OP_MUL << 4, COOT_OP_EXP << 4,
            COOT_OP_SCALAR << 4, (COOT_OP_LOAD << 4) | 2, COOT_OP_MUL << 4, COOT_OP_ADD << 4> {
  static constexpr bool value = true;
};
template <int... Code>
constexpr bool is_c2_prog() {
  return IsC2<Code...>::value;
}
#ifndef COOT_FP8_FAST_EXP
#define COOT_FP8_FAST_EXP 1
#endif

template <class Prog>
struct CatalogEval;
template <int... Code>
struct CatalogEval<StaticProg<Code...>> {
  static constexpr int K = StaticProg<Code...>::n_ops();
  static constexpr int kStack = COOT_MAX_STACK;
  static constexpr bool kInterp = false;
  // the program is the plain matrix [L0]
  static constexpr bool kIdentity = sizeof...(Code) == 1 && StaticProg<Code...>::codes[0] == 0;
  template <class T, int W, class Src>
  __device__ __forceinline__ static void eval_src(const Src& src, const FusedArgs& a, T (&out)[W]) {
    if constexpr (COOT_FP8_FAST_EXP && is_fp8<T>() && is_c2_prog<Code...>()) {
      float z[W], y[W];
      load_to<T, W>(src, 0, z);
      load_to<T, W>(src, 1, y);
#pragma unroll
      for (int w = 0; w < W; ++w) z[w] = bin<COOT_OP_MUL>(z[w], y[w]);
      load_to<T, W>(src, 2, y);
      const float sc = scalar_as<float>(a.scalars[0]);
      float lo[W], hi[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const float e0 = expf(z[w]);
        // x == 0: E' = 1 exactly and D = 0; else D = 2 (|E'| 2^-21 + |z'| 2^-22).
        // Selects in PTX: ptxas otherwise branches around the expf.
        const float x = z[w];
        float e, D;
        asm("{ .reg .pred p; setp.eq.f32 p, %2, 0f00000000; selp.f32 %0, 0f3F800000, %1, p; }"
            : "=f"(e) : "f"(e0), "f"(x));
        z[w] = bin<COOT_OP_ADD>(e, bin<COOT_OP_MUL>(sc, y[w]));
        const float Dv = __fmaf_rn(fabsf(e0), 0x1p-20f, fabsf(z[w]) * 0x1p-21f);
        asm("{ .reg .pred p; setp.eq.f32 p, %2, 0f00000000; selp.f32 %0, 0f00000000, %1, p; }"
            : "=f"(D) : "f"(Dv), "f"(x));
        lo[w] = __fsub_rn(z[w], D);
        hi[w] = __fadd_rn(z[w], D);
      }
      T nlo[W], nhi[W];
      narrow_vec<T, W>(lo, nlo);
      narrow_vec<T, W>(hi, nhi);
      uint32_t diff = 0;
#pragma unroll
      for (int w = 0; w + 3 < W; w += 4) {
        uint32_t a4, b4;
        memcpy(&a4, &nlo[w], 4);
        memcpy(&b4, &nhi[w], 4);
        diff |= a4 ^ b4;
      }
#pragma unroll
      for (int w = W & ~3; w < W; ++w) diff |= (uint32_t)(nlo[w].bits ^ nhi[w].bits);
      const bool ok = diff == 0;
      if (__builtin_expect(!ok, 0)) {
        float r[W];  // a local copy: only the rare branch touches memory
        fp8_c2_exact<T, W>(src, sc, r);
        narrow_vec<T, W>(r, nlo);
      }
#pragma unroll
      for (int w = 0; w < W; ++w) out[w] = nlo[w];
    } else {
      typename ComputeT<T>::type st[COOT_MAX_STACK][W];
      StaticStep<T, W, 0, Code...>::run(st, src, a);
      narrow_vec<T, W>(st[0], out);
    }
  }
  template <class T, int W>
  __device__ __forceinline__ static void eval(const T (&in)[K][W], const FusedArgs& a, T (&out)[W]) {
    eval_src<T, W>(RegSrc<T, K, W>{in}, a, out);
  }
};

// ---- K2: warp-uniform register interpreter --------------------------------
// The host precomputes a key = op * 9 + depth for every instruction (depth =
// stack size before it, 0..8).  Keys live in the kernel's parameter bank and
// are uniform across the grid, so each `switch` is a uniform branch (ptxas
// lowers it to a shallow compare tree; a gap-free key layout did not make it
// emit a BRX jump table); every case touches stack registers with
// compile-time indices.  LOAD takes its operand index at run time from the
// source (a shared-memory address under the TMA driver).  One dispatch
// evaluates UD whole 16-byte units.
// EXP / LOG group size inside the interpreter (coot_device.cuh un_vec)
#ifndef COOT_INTERP_EXP_GROUP
#define COOT_INTERP_EXP_GROUP 4
#endif
#define COOT_KEY(op, d) ((op) * 9 + (d))
// Fused-operand dispatch ops (host peephole, runtime.cu fill_program): an ADD,
// SUB or MUL whose right operand is an operand load or a scalar, "L k OP" -> OP_L k and
// "S k OP" -> OP_S k (and "S k L j OP" -> "L j" OP_S k for the commutative ADD /
// MUL), so the loaded / broadcast value never takes a stack slot or a dispatch
// of its own.  Same arithmetic, same operand order (a OP b, b = the fused
// operand) as the unfused sequence.  c2: 8 dispatches -> 6, axpy 5 -> 3.
#define COOT_XOP_L(op) (14 + (op) - COOT_OP_ADD)  // ADD, SUB, MUL -> 14..16
#define COOT_XOP_S(op) (17 + (op) - COOT_OP_ADD)  // ADD, SUB, MUL -> 17..19

template <int KMAX, int SMAX>
struct InterpEval {
  static constexpr int K = KMAX;
  static constexpr int kStack = SMAX;
  static constexpr bool kInterp = true;
  static constexpr bool kIdentity = false;

  template <class T, int W, class Src>
  __device__ __forceinline__ static void eval_src(const Src& src, const FusedArgs& a, T (&out)[W]) {
    typedef typename ComputeT<T>::type CT;
    CT st[SMAX][W];  // every slot is written (LOAD/SCALAR) before it is read

#define COOT_LOAD_CASE(d)                                                  \
  case COOT_KEY(COOT_OP_LOAD, d):                                          \
    if constexpr ((d) < SMAX) load_to<T, W>(src, (int)arg, st[(d) < SMAX ? (d) : 0]); \
    break;
#define COOT_SCALAR_CASE(d)                                                \
  case COOT_KEY(COOT_OP_SCALAR, d):                                        \
    if constexpr ((d) < SMAX) {                                            \
      const CT s = scalar_as<CT>(a.scalars[arg]);                          \
      _Pragma("unroll") for (int w = 0; w < W; ++w) st[d][w] = s;          \
    }                                                                      \
    break;
#define COOT_UN_CASE(OP, d)                                                \
  case COOT_KEY(COOT_OP_##OP, d):                                          \
    if constexpr ((d) >= 1 && (d) <= SMAX && op_legal<T>(COOT_OP_##OP)) {  \
      un_vec<COOT_OP_##OP, COOT_INTERP_EXP_GROUP>(st[(d) >= 1 ? (d) - 1 : 0]);   \
    } else if constexpr ((d) >= 1 && (d) <= SMAX) {                        \
      __trap(); /* op illegal for T: rejected on the host (R9) */          \
    }                                                                      \
    break;
#define COOT_BIN_CASE(OP, d)                                               \
  case COOT_KEY(COOT_OP_##OP, d):                                          \
    if constexpr ((d) >= 2 && (d) <= SMAX && op_legal<T>(COOT_OP_##OP)) {  \
      bin_vec<COOT_OP_##OP>(st[(d) >= 2 ? (d) - 2 : 0], st[(d) >= 2 ? (d) - 1 : 0]); \
    } else if constexpr ((d) >= 2 && (d) <= SMAX) {                        \
      __trap(); /* op illegal for T: rejected on the host (R9) */          \
    }                                                                      \
    break;
#define COOT_BINL_CASE(OP, d)                                              \
  case COOT_KEY(COOT_XOP_L(COOT_OP_##OP), d):                              \
    if constexpr ((d) >= 1 && (d) <= SMAX && op_legal<T>(COOT_OP_##OP)) {  \
      CT t[W];                                                             \
      load_to<T, W>(src, (int)arg, t);                                     \
      bin_vec<COOT_OP_##OP>(st[(d) >= 1 ? (d) - 1 : 0], t);                \
    } else if constexpr ((d) >= 1 && (d) <= SMAX) {                        \
      __trap();                                                            \
    }                                                                      \
    break;
#define COOT_BINS_CASE(OP, d)                                              \
  case COOT_KEY(COOT_XOP_S(COOT_OP_##OP), d):                              \
    if constexpr ((d) >= 1 && (d) <= SMAX && op_legal<T>(COOT_OP_##OP)) {  \
      const CT s = scalar_as<CT>(a.scalars[arg]);                          \
      CT t[W];                                                             \
      _Pragma("unroll") for (int w = 0; w < W; ++w) t[w] = s;              \
      bin_vec<COOT_OP_##OP>(st[(d) >= 1 ? (d) - 1 : 0], t);                \
    } else if constexpr ((d) >= 1 && (d) <= SMAX) {                        \
      __trap();                                                            \
    }                                                                      \
    break;
#define COOT_D(M, ...) M(__VA_ARGS__ 0) M(__VA_ARGS__ 1) M(__VA_ARGS__ 2) M(__VA_ARGS__ 3) \
  M(__VA_ARGS__ 4) M(__VA_ARGS__ 5) M(__VA_ARGS__ 6) M(__VA_ARGS__ 7) M(__VA_ARGS__ 8)

    // the next instruction is fetched before this one is dispatched, so its
    // constant-bank latency overlaps the case body
    uint32_t next = a.code[0];
#pragma unroll 1
    for (uint32_t i = 0; i < a.n_instr; ++i) {
      const uint32_t key = next & 0xffffu, arg = next >> 16;
      next = a.code[i + 1 < COOT_MAX_INSTR ? i + 1 : i];
      switch (key) {
        COOT_D(COOT_LOAD_CASE)
        COOT_D(COOT_SCALAR_CASE)
        COOT_D(COOT_UN_CASE, NEG,)
        COOT_D(COOT_UN_CASE, ABS,)
        COOT_D(COOT_UN_CASE, SQUARE,)
        COOT_D(COOT_UN_CASE, SQRT,)
        COOT_D(COOT_UN_CASE, EXP,)
        COOT_D(COOT_UN_CASE, LOG,)
        COOT_D(COOT_BIN_CASE, ADD,)
        COOT_D(COOT_BIN_CASE, SUB,)
        COOT_D(COOT_BIN_CASE, MUL,)
        COOT_D(COOT_BIN_CASE, DIV,)
        COOT_D(COOT_BIN_CASE, MIN,)
        COOT_D(COOT_BIN_CASE, MAX,)
        COOT_D(COOT_BINL_CASE, ADD,)
        COOT_D(COOT_BINL_CASE, SUB,)
        COOT_D(COOT_BINL_CASE, MUL,)
        COOT_D(COOT_BINS_CASE, ADD,)
        COOT_D(COOT_BINS_CASE, SUB,)
        COOT_D(COOT_BINS_CASE, MUL,)
        default:
          break;
      }
    }
#undef COOT_D
#undef COOT_BINS_CASE
#undef COOT_BINL_CASE
#undef COOT_BIN_CASE
#undef COOT_UN_CASE
#undef COOT_SCALAR_CASE
#undef COOT_LOAD_CASE
    narrow_vec<T, W>(st[0], out);
  }
  template <class T, int W>
  __device__ __forceinline__ static void eval(const T (&in)[K][W], const FusedArgs& a, T (&out)[W]) {
    eval_src<T, W>(RegSrc<T, K, W>{in}, a, out);
  }
};

// ---- operand loading (register drivers) -------------------------------------
template <class T, class EV>
__device__ __forceinline__ void load_units(const FusedArgs& a, u64 e,
                                           T (&in)[EV::K][Unit<T>::W]) {
#pragma unroll
  for (int k = 0; k < EV::K; ++k) {
    if (!EV::kInterp || k < (int)a.n_operands)
      load_unit<T>(reinterpret_cast<const T*>(a.in[k]) + e, in[k]);
  }
}
template <class T, class EV>
__device__ __forceinline__ void load_units_p(const FusedArgs& a, u64 boff, uint32_t u,
                                             T (&in)[EV::K][Unit<T>::W]) {
#pragma unroll
  for (int k = 0; k < EV::K; ++k) {
    if (!EV::kInterp || k < (int)a.n_operands) {
      uint4 r = ld16(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(a.in[k]) + boff) + u);
      memcpy(&in[k][0], &r, 16);
    }
  }
}
template <class T, class EV>
__device__ __forceinline__ void load_elem(const FusedArgs& a, u64 e, T (&in)[EV::K][1]) {
#pragma unroll
  for (int k = 0; k < EV::K; ++k) {
    if (!EV::kInterp || k < (int)a.n_operands)
      in[k][0] = ldcg_elem(reinterpret_cast<const T*>(a.in[k]) + e);
    else
      in[k][0] = T(0);
  }
}

// ---- LDG driver (register-pipelined; COOT_DRIVER=0) ---------------------------
// Element -> thread map: head [0, head) and tail [tail_begin, n) scalars by
// global thread index; body 16-byte unit u -> thread u mod N (N = grid*256),
// each thread walking its units in increasing order.  The loads of the NEXT U
// units are issued before the current ones are evaluated.  The body is walked
// in segments of SEG units (SEG = 0 mod N, < 2^31) so the loop index is 32-bit.
template <class T, int ACC, class EV, int U>
__global__ void __launch_bounds__(kThreads, EV::kInterp ? 1 : COOT_CAT_MINB)
    fused_kernel(const __grid_constant__ FusedArgs a) {
  pdl_wait();
  constexpr int W = Unit<T>::W;
  constexpr int K = EV::K;
  Accum<T, ACC> acc;
  acc.init();
  const u64 tid = (u64)blockIdx.x * kThreads + threadIdx.x;
  const u64 nthr = (u64)gridDim.x * kThreads;
  T* out = reinterpret_cast<T*>(a.out);

  for (u64 e = tid; e < a.head; e += nthr) {
    T in[K][1], v[1];
    load_elem<T, EV>(a, e, in);
    EV::template eval<T, 1>(in, a, v);
    if (out) out[e] = v[0];
    acc.template add_at<1>(v, e);
  }
  {
    const uint32_t nthr32 = (uint32_t)nthr, tid32 = (uint32_t)tid;
    const u64 SEG = (u64)(0x7fffffffu / nthr32) * nthr32;
    for (u64 s0 = 0; s0 < a.nunits; s0 += SEG) {
      const uint32_t nloc = (uint32_t)((a.nunits - s0) < SEG ? (a.nunits - s0) : SEG);
      const u64 boff = a.head * sizeof(T) + s0 * 16;
      uint4* po = out ? reinterpret_cast<uint4*>(reinterpret_cast<char*>(out) + boff) : nullptr;
      uint32_t u = tid32;
      T cur[U][K][W];
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (u + j * nthr32 < nloc) load_units_p<T, EV>(a, boff, u + j * nthr32, cur[j]);
      while (u < nloc) {
        const uint32_t un = u + U * nthr32;
        T nxt[U][K][W];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (un + j * nthr32 < nloc) load_units_p<T, EV>(a, boff, un + j * nthr32, nxt[j]);
#pragma unroll
        for (int j = 0; j < U; ++j) {
          if (u + j * nthr32 < nloc) {
            T v[W];
            EV::template eval<T, W>(cur[j], a, v);
            if (po) {
              uint4 r;
              memcpy(&r, &v[0], 16);
              st16(po + u + j * nthr32, r);
            }
            acc.template add_at<W>(v, a.head + (s0 + u + (u64)j * nthr32) * W);
          }
        }
#pragma unroll
        for (int j = 0; j < U; ++j)
#pragma unroll
          for (int k = 0; k < K; ++k)
#pragma unroll
            for (int w = 0; w < W; ++w) cur[j][k][w] = nxt[j][k][w];
        u = un;
      }
    }
  }
  for (u64 e = a.tail_begin + tid; e < a.n; e += nthr) {
    T in[K][1], v[1];
    load_elem<T, EV>(a, e, in);
    EV::template eval<T, 1>(in, a, v);
    if (out) out[e] = v[0];
    acc.template add_at<1>(v, e);
  }

  pdl_trigger();  // streaming done: the next kernel may start launching
  if constexpr (ACC != ACC_NONE) {
    Accum<T, ACC> bt = block_reduce<T, ACC>(acc);
    grid_finish<T, ACC>(bt, a.partials, a.ticket, a.final_mode, a.kind, a.result, a.count, a.ex);
  }
}

// ---- strided driver (views: diag / submatrix / row) -------------
// Element e of the m x n expression -> (i, j) = (e mod m, e / m); operand k
// is read at in[k][i*inc[k] + j*ld[k]] and the result written to
// out[i*out_inc + j*out_ld].  Thread t walks e = t, t + N, ... (N threads);
// (i, j) advance incrementally, no division in the loop.  Always driven by the
// interpreter (one kernel per type/reduction), so results do not depend on
// catalog matching.
template <class T, int ACC, class EV>
__global__ void __launch_bounds__(kThreads) fused_strided_kernel(const __grid_constant__ FusedArgs a) {
  pdl_wait();
  constexpr int K = EV::K;
  Accum<T, ACC> acc;
  acc.init();
  const u64 tid = (u64)blockIdx.x * kThreads + threadIdx.x;
  const u64 nthr = (u64)gridDim.x * kThreads;
  const u64 m = a.m;
  u64 i = tid % m, j = tid / m;
  const u64 di = nthr % m, dj = nthr / m;
  T* out = reinterpret_cast<T*>(a.out);
  for (u64 e = tid; e < a.n; e += nthr) {
    T in[K][1], v[1];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!EV::kInterp || k < (int)a.n_operands)
        in[k][0] = ldcg_elem(reinterpret_cast<const T*>(a.in[k]) + i * a.inc[k] + j * a.ld[k]);
      else
        in[k][0] = T(0);
    }
    EV::template eval<T, 1>(in, a, v);
    if (out) out[i * a.out_inc + j * a.out_ld] = v[0];
    acc.template add_at<1>(v, e);
    i += di;
    j += dj;
    if (i >= m) {
      i -= m;
      ++j;
    }
  }
  pdl_trigger();  // streaming done: the next kernel may start launching
  if constexpr (ACC != ACC_NONE) {
    Accum<T, ACC> bt = block_reduce<T, ACC>(acc);
    grid_finish<T, ACC>(bt, a.partials, a.ticket, a.final_mode, a.kind, a.result, a.count, a.ex);
  }
}

// ---- the TMA-staged driver (default on B200) ---------------------------------
// One producer warp streams tiles of every operand into a `stages`-deep shared
// memory ring with 1-D bulk copies (cp.async.bulk + mbarrier complete_tx,
// L2 evict-first); 8 consumer warps evaluate the program out of shared memory,
// store the element-wise result and accumulate.  Memory-level parallelism
// (stages x operands x tile bytes in flight per CTA) does not depend on
// registers or occupancy, so compute-heavy programs (f64-evaluated EXP) and
// the interpreter keep HBM busy.
//
// Element -> thread map: tile t (tile_units 16-byte units) -> CTA t mod G;
// unit i of a tile -> consumer thread i mod 256; each thread walks its units
// tile by tile in increasing order; head/tail scalars -> global consumer
// thread index.  Depends only on (n, operands, SM count) and is shared by K1
// and K2, which therefore agree bit for bit.
constexpr int kConsumerWarps = 8;
constexpr int kTmaThreads = (kConsumerWarps + 1) * 32;
// Units evaluated per dispatch: 2 (more ILP, half the interpreter dispatch
// cost) except for the 8-operand interpreter, whose stack would not fit.
#ifndef COOT_UD
#define COOT_UD 2
#endif
constexpr int kTileUnits = 2 * kConsumerWarps * 32;  // 512 units = 8 KB per operand
// 16-byte units per evaluator dispatch: COOT_UD, except 1 for the 8-operand
// interpreter and for 8-bit types (16 elements per unit already; their f32
// stack of 2 units would not fit the register budget).
template <class T, class EV>
constexpr int units_per_dispatch() {
  return ((EV::kInterp && EV::K > 4) || sizeof(T) == 1) ? 1 : COOT_UD;
}
#ifndef COOT_INTERP4_MINB
#define COOT_INTERP4_MINB 2
#endif
#ifndef COOT_INTERP4_UD
#define COOT_INTERP4_UD 2
#endif
#ifndef COOT_INTERP2_UD
#define COOT_INTERP2_UD 4
#endif
// fused_tma_kernel: the small interpreter on 4-byte types takes 4 units (16
// elements) per dispatch — halving the per-element cost of its uniform
// instruction dispatch; the host sizes those tiles at 4 * 256 units.
template <class T, class EV>
constexpr int tma_units_per_dispatch() {
  return (EV::kInterp && EV::K <= 4 && sizeof(T) == 4)
             ? (EV::kStack <= 2 ? COOT_INTERP2_UD : COOT_INTERP4_UD)
             : units_per_dispatch<T, EV>();
}
// Resident CTAs per SM the register budget is sized for: 2 (<= 96 registers),
// except the 8-operand interpreter, which gets the whole register file.
template <class EV>
constexpr int tma_min_ctas() {
  return (EV::kInterp && EV::K > 4) ? 1 : (EV::kInterp ? COOT_INTERP4_MINB : 2);
}

// In-band producer for the small interpreter: the CTA is the 8 consumer warps
// only (256 threads) and consumer thread 0 issues the bulk copies — the first
// S tiles up front, then the refill of each stage as soon as all 8 warps have
// released it.  Two 256-thread CTAs per SM get 128 registers per thread (a
// 288-thread CTA is allocated registers for 10 warps: 96), which is what the
// interpreter's register stack of 4 units x 4 slots needs without spilling.
#ifndef COOT_INTERP_INBAND
#define COOT_INTERP_INBAND 1
#endif
template <class EV>
constexpr bool tma_inband() {
  return COOT_INTERP_INBAND && EV::kInterp && EV::K <= 4;
}
template <class EV>
constexpr int tma_threads() {
  return tma_inband<EV>() ? kConsumerWarps * 32 : kTmaThreads;
}

template <class T, int ACC, class EV>
__global__ void __launch_bounds__(tma_threads<EV>(), tma_min_ctas<EV>())
    fused_tma_kernel(const __grid_constant__ FusedArgs a) {
  constexpr bool kInband = tma_inband<EV>();
  pdl_wait();
  constexpr int W = Unit<T>::W;
  constexpr int K = EV::K;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t nk = EV::kInterp ? a.n_operands : (uint32_t)K;
  const uint32_t S = a.stages, TU = a.tile_units;
  const uint32_t tile_bytes = TU * 16u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * nk * tile_bytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  Accum<T, ACC> acc;
  acc.init();
  const u64 ntiles = (a.nunits + TU - 1) / TU;
  const u64 boff = a.head * sizeof(T);  // body starts 16-byte aligned here
  // the bulk copies of this CTA's j-th tile into stage j % S
  auto issue = [&](u64 t, uint32_t st, uint64_t pol) {
    const u64 u0 = t * TU;
    const uint32_t nu = (uint32_t)((a.nunits - u0) < TU ? (a.nunits - u0) : TU);
    mbar_expect_tx(&full[st], nu * 16u * nk);
    for (uint32_t k = 0; k < nk; ++k)
      bulk_g2s(smem + ((size_t)st * nk + k) * tile_bytes,
               reinterpret_cast<const char*>(a.in[k]) + boff + u0 * 16, nu * 16u, &full[st], pol);
  };
  if constexpr (kInband) {
    if (threadIdx.x == 0) {
      const uint64_t pol = policy_evict_first();
      u64 t = blockIdx.x;
      for (uint32_t st = 0; st < S && t < ntiles; ++st, t += gridDim.x) issue(t, st, pol);
    }
  }

  if (!kInband && warp == kConsumerWarps) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t s = 0, ph = 0;
      u64 i = 0;
      for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        if (i >= S) producer_wait(&empty[s], ph ^ 1u, a.producer_sleep);
        const u64 u0 = t * TU;
        const uint32_t nu = (uint32_t)((a.nunits - u0) < TU ? (a.nunits - u0) : TU);
        mbar_expect_tx(&full[s], nu * 16u * nk);
        for (uint32_t k = 0; k < nk; ++k)
          bulk_g2s(smem + ((size_t)s * nk + k) * tile_bytes,
                   reinterpret_cast<const char*>(a.in[k]) + boff + u0 * 16, nu * 16u, &full[s],
                   pol);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    // ---------------- consumers ----------------
    const u64 ctid = (u64)blockIdx.x * (kConsumerWarps * 32) + threadIdx.x;
    const u64 cthr = (u64)gridDim.x * (kConsumerWarps * 32);
    T* out = reinterpret_cast<T*>(a.out);
    for (u64 e = ctid; e < a.head; e += cthr) {
      T in[K][1], v[1];
      load_elem<T, EV>(a, e, in);
      EV::template eval<T, 1>(in, a, v);
      if (out) out[e] = v[0];
      acc.template add_at<1>(v, e);
    }
    uint4* po = out ? reinterpret_cast<uint4*>(reinterpret_cast<char*>(out) + boff) : nullptr;
    uint32_t s = 0, ph = 0;
    for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const u64 u0 = t * TU;
      const uint32_t nu = (uint32_t)((a.nunits - u0) < TU ? (a.nunits - u0) : TU);
      mbar_wait(&full[s], ph);
      const unsigned char* stg = smem + (size_t)s * nk * tile_bytes;
      // each dispatch evaluates UD units (i, i + 256, ...) of the tile together;
      // units are stored / accumulated in increasing order (TU >= UD * 256, so
      // units past nu are read from the stage buffer and discarded)
      constexpr int UD = tma_units_per_dispatch<T, EV>();
      for (uint32_t i = threadIdx.x; i < nu; i += UD * kConsumerWarps * 32) {
        T v[UD * W];
        EV::template eval_src<T, UD * W>(SmemSrc<T, UD>{stg + (size_t)i * 16, tile_bytes}, a, v);
#pragma unroll
        for (int j = 0; j < UD; ++j) {
          const uint32_t ij = i + j * kConsumerWarps * 32;
          if (j == 0 || ij < nu) {
            T vj[W];
#pragma unroll
            for (int w = 0; w < W; ++w) vj[w] = v[j * W + w];
            if (po) {
              uint4 r;
              memcpy(&r, &vj[0], 16);
              st16(po + u0 + ij, r);
            }
            acc.template add_at<W>(vj, a.head + (u0 + ij) * W);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if constexpr (kInband) {
        // refill this stage with the tile S rounds ahead once every warp has
        // released it (thread 0 waits for the slowest warp of the CTA)
        const u64 tn = t + (u64)S * gridDim.x;
        if (threadIdx.x == 0 && tn < ntiles) {
          producer_wait(&empty[s], ph, a.producer_sleep);
          issue(tn, s, policy_evict_first());
        }
      }
      if (++s == S) {
        s = 0;
        ph ^= 1u;
      }
    }
    for (u64 e = a.tail_begin + ctid; e < a.n; e += cthr) {
      T in[K][1], v[1];
      load_elem<T, EV>(a, e, in);
      EV::template eval<T, 1>(in, a, v);
      if (out) out[e] = v[0];
      acc.template add_at<1>(v, e);
    }
  }

  pdl_trigger();  // streaming done: the next kernel may start launching
  if constexpr (ACC != ACC_NONE) {
    Accum<T, ACC> bt = block_reduce<T, ACC>(acc);
    grid_finish<T, ACC>(bt, a.partials, a.ticket, a.final_mode, a.kind, a.result, a.count, a.ex);
  } else {
    __syncthreads();  // the producer stays resident until every staged tile is consumed
  }
}

// ---- views with contiguous columns (submatrix / column / row-block views) ------
// When every operand and the destination have inc == 1 and their column starts
// share one 16-byte misalignment (ld * sizeof(T) % 16 == 0, equal base
// misalignment), each column of the view is a contiguous run: the same
// producer / consumer TMA ring as fused_tma_kernel streams it, piece by piece
// (piece = (column j, segment s) of seg_len rows), with scalar head / tail
// elements per piece.  Interpreter evaluators only (views never use the
// catalog), element index for index reductions = j * m + i.
template <class T, int ACC, class EV>
__global__ void __launch_bounds__(kTmaThreads, tma_min_ctas<EV>())
    fused_cols_tma_kernel(const __grid_constant__ FusedArgs a) {
  pdl_wait();
  constexpr int W = Unit<T>::W;
  constexpr int K = EV::K;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t nk = a.n_operands;
  const uint32_t S = a.stages, TU = a.tile_units;
  const uint32_t tile_bytes = TU * 16u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * nk * tile_bytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  Accum<T, ACC> acc;
  acc.init();
  const u64 npieces = a.ncols * a.nseg, m = a.m;
  const uintptr_t base0 = reinterpret_cast<uintptr_t>(a.in[0]);
  // geometry of piece p (identical on producer and consumers)
  auto piece = [&](u64 p, u64& j, u64& r0, u64& len, u64& head, u64& nun) {
    j = p / a.nseg;
    r0 = (p % a.nseg) * a.seg_len;
    len = (m - r0) < a.seg_len ? (m - r0) : a.seg_len;
    const uintptr_t mis = (base0 + (j * a.ld[0] + r0) * sizeof(T)) & 15;
    head = ((16 - mis) & 15) / sizeof(T);
    if (head > len) head = len;
    nun = (len - head) / W;
  };
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t s = 0, ph = 0;
      u64 i = 0;
      for (u64 p = blockIdx.x; p < npieces; p += gridDim.x) {
        u64 j, r0, len, head, nun;
        piece(p, j, r0, len, head, nun);
        for (u64 u0 = 0; u0 < nun; u0 += TU, ++i) {
          if (i >= S) producer_wait(&empty[s], ph ^ 1u, a.producer_sleep);
          const uint32_t nu = (uint32_t)((nun - u0) < TU ? (nun - u0) : TU);
          mbar_expect_tx(&full[s], nu * 16u * nk);
          for (uint32_t k = 0; k < nk; ++k)
            bulk_g2s(smem + ((size_t)s * nk + k) * tile_bytes,
                     reinterpret_cast<const char*>(a.in[k]) +
                         (j * a.ld[k] + r0 + head) * sizeof(T) + u0 * 16,
                     nu * 16u, &full[s], pol);
          if (++s == S) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else {
    T* out = reinterpret_cast<T*>(a.out);
    uint32_t s = 0, ph = 0;
    constexpr int UD = units_per_dispatch<T, EV>();
    for (u64 p = blockIdx.x; p < npieces; p += gridDim.x) {
      u64 j, r0, len, head, nun;
      piece(p, j, r0, len, head, nun);
      const u64 e0 = j * m + r0;  // linear index of the piece's first element
      auto scalar_elem = [&](u64 i) {
        T in[K][1], v[1];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (k < (int)nk)
            in[k][0] = ldcg_elem(reinterpret_cast<const T*>(a.in[k]) + j * a.ld[k] + r0 + i);
          else
            in[k][0] = T(0);
        }
        EV::template eval<T, 1>(in, a, v);
        if (out) out[j * a.out_ld + r0 + i] = v[0];
        acc.template add_at<1>(v, e0 + i);
      };
      for (u64 i = threadIdx.x; i < head; i += kConsumerWarps * 32) scalar_elem(i);
      uint4* po = out ? reinterpret_cast<uint4*>(out + j * a.out_ld + r0 + head) : nullptr;
      for (u64 u0 = 0; u0 < nun; u0 += TU) {
        const uint32_t nu = (uint32_t)((nun - u0) < TU ? (nun - u0) : TU);
        mbar_wait(&full[s], ph);
        const unsigned char* stg = smem + (size_t)s * nk * tile_bytes;
        for (uint32_t i = threadIdx.x; i < nu; i += UD * kConsumerWarps * 32) {
          T v[UD * W];
          EV::template eval_src<T, UD * W>(SmemSrc<T, UD>{stg + (size_t)i * 16, tile_bytes}, a, v);
#pragma unroll
          for (int q = 0; q < UD; ++q) {
            const uint32_t iq = i + q * kConsumerWarps * 32;
            if (q == 0 || iq < nu) {
              T vq[W];
#pragma unroll
              for (int w = 0; w < W; ++w) vq[w] = v[q * W + w];
              if (po) {
                uint4 r;
                memcpy(&r, &vq[0], 16);
                st16(po + u0 + iq, r);
              }
              acc.template add_at<W>(vq, e0 + head + (u0 + iq) * W);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
      for (u64 i = head + nun * W + threadIdx.x; i < len; i += kConsumerWarps * 32) scalar_elem(i);
    }
  }
  pdl_trigger();  // streaming done: the next kernel may start launching
  if constexpr (ACC != ACC_NONE) {
    Accum<T, ACC> bt = block_reduce<T, ACC>(acc);
    grid_finish<T, ACC>(bt, a.partials, a.ticket, a.final_mode, a.kind, a.result, a.count, a.ex);
  } else {
    __syncthreads();  // the producer stays resident until every staged tile is consumed
  }
}

}  // namespace coot
