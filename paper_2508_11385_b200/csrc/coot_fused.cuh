// K1 (templated catalog) and K2 (warp-uniform register interpreter) fused
// element-wise + terminal-reduction kernels.  Both share ONE driver loop
// (fused_kernel) so the element -> thread map and the accumulation order are
// identical: for the same grid, K1 and K2 produce bit-identical results.
//
// Element -> thread map (deterministic, R14): the n elements are split into
//   head   [0, head)                    scalar elements up to 16-B alignment
//   body   [head, head + nunits*W)      16-byte units, unit u -> thread u mod N
//   tail   [tail_begin, n)              scalar elements
// N = gridDim.x * 256 threads; each thread walks its units in increasing order
// (U units per iteration, loads issued together for memory-level parallelism;
// U does not change the order).  The grid depends only on (n, SM count).
#pragma once
#include "coot_catalog.h"
#include "coot_device.cuh"

namespace coot {

__host__ __device__ constexpr int ins_op(int c) { return c >> 4; }
__host__ __device__ constexpr int ins_arg(int c) { return c & 15; }
__host__ __device__ constexpr bool is_unary_op(int op) {
  return op >= COOT_OP_NEG && op <= COOT_OP_LOG;
}

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

template <class T, int W, int SP, int C, int... Rest>
struct StaticStep {
  template <int K>
  __device__ __forceinline__ static void run(T (&st)[COOT_MAX_STACK][W], const T (&in)[K][W],
                                             const FusedArgs& a) {
    constexpr int op = ins_op(C), arg = ins_arg(C);
    constexpr int nsp = (op == COOT_OP_LOAD || op == COOT_OP_SCALAR) ? SP + 1
                        : is_unary_op(op)                            ? SP
                                                                     : SP - 1;
    if constexpr (op == COOT_OP_LOAD) {
#pragma unroll
      for (int w = 0; w < W; ++w) st[SP][w] = in[arg][w];
    } else if constexpr (op == COOT_OP_SCALAR) {
      const T s = scalar_as<T>(a.scalars[arg]);
#pragma unroll
      for (int w = 0; w < W; ++w) st[SP][w] = s;
    } else if constexpr (is_unary_op(op)) {
#pragma unroll
      for (int w = 0; w < W; ++w) st[SP - 1][w] = un<op>(st[SP - 1][w]);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) st[SP - 2][w] = bin<op>(st[SP - 2][w], st[SP - 1][w]);
    }
    if constexpr (sizeof...(Rest) > 0) StaticStep<T, W, nsp, Rest...>::template run<K>(st, in, a);
  }
};

template <class Prog>
struct CatalogEval;
template <int... Code>
struct CatalogEval<StaticProg<Code...>> {
  static constexpr int K = StaticProg<Code...>::n_ops();
  static constexpr bool kInterp = false;
  template <class T, int W>
  __device__ __forceinline__ static void eval(const T (&in)[K][W], const FusedArgs& a,
                                              T (&out)[W]) {
    T st[COOT_MAX_STACK][W];
    StaticStep<T, W, 0, Code...>::template run<K>(st, in, a);
#pragma unroll
    for (int w = 0; w < W; ++w) out[w] = st[0][w];
  }
};

// ---- K2: warp-uniform register interpreter --------------------------------
// The host precomputes key = (op << 8) | (depth << 4) | arg for every
// instruction (depth = stack size before it).  The key lives in the kernel's
// parameter bank and is uniform across the grid, so each `switch` is a
// uniform branch; every case touches stack registers with compile-time
// indices (no local memory).  One dispatch handles a whole 16-byte unit.
#define COOT_KEY(op, d, a) (((op) << 8) | ((d) << 4) | (a))

template <int KMAX, int SMAX>
struct InterpEval {
  static constexpr int K = KMAX;
  static constexpr bool kInterp = true;

  template <class T, int W>
  __device__ __forceinline__ static void eval(const T (&in)[K][W], const FusedArgs& a,
                                              T (&out)[W]) {
    T st[SMAX][W];  // every slot is written (LOAD/SCALAR) before it is read

#define COOT_LOAD_CASE(d, k)                                               \
  case COOT_KEY(COOT_OP_LOAD, d, k):                                       \
    if constexpr ((d) < SMAX && (k) < K) {                                 \
      _Pragma("unroll") for (int w = 0; w < W; ++w) st[d][w] = in[k][w];   \
    }                                                                      \
    break;
#define COOT_SCALAR_CASE(d)                                                \
  case COOT_KEY(COOT_OP_SCALAR, d, 0):                                     \
    if constexpr ((d) < SMAX) {                                            \
      const T s = scalar_as<T>(a.scalars[a.arg[i]]);                       \
      _Pragma("unroll") for (int w = 0; w < W; ++w) st[d][w] = s;          \
    }                                                                      \
    break;
#define COOT_UN_CASE(OP, d)                                                \
  case COOT_KEY(COOT_OP_##OP, d, 0):                                       \
    if constexpr ((d) >= 1 && (d) <= SMAX && op_legal<T>(COOT_OP_##OP)) {  \
      _Pragma("unroll") for (int w = 0; w < W; ++w)                        \
          st[(d) - 1][w] = un<COOT_OP_##OP>(st[(d) - 1][w]);                \
    }                                                                      \
    break;
#define COOT_BIN_CASE(OP, d)                                               \
  case COOT_KEY(COOT_OP_##OP, d, 0):                                       \
    if constexpr ((d) >= 2 && (d) <= SMAX && op_legal<T>(COOT_OP_##OP)) {  \
      _Pragma("unroll") for (int w = 0; w < W; ++w)                        \
          st[(d) - 2][w] = bin<COOT_OP_##OP>(st[(d) - 2][w], st[(d) - 1][w]); \
    }                                                                      \
    break;
#define COOT_CASES_AT(d)                                                             \
  COOT_LOAD_CASE(d, 0) COOT_LOAD_CASE(d, 1) COOT_LOAD_CASE(d, 2) COOT_LOAD_CASE(d, 3) \
  COOT_LOAD_CASE(d, 4) COOT_LOAD_CASE(d, 5) COOT_LOAD_CASE(d, 6) COOT_LOAD_CASE(d, 7) \
  COOT_SCALAR_CASE(d)                                                                \
  COOT_UN_CASE(NEG, d) COOT_UN_CASE(ABS, d) COOT_UN_CASE(SQUARE, d)                  \
  COOT_UN_CASE(SQRT, d) COOT_UN_CASE(EXP, d) COOT_UN_CASE(LOG, d)                    \
  COOT_BIN_CASE(ADD, d) COOT_BIN_CASE(SUB, d) COOT_BIN_CASE(MUL, d)                  \
  COOT_BIN_CASE(DIV, d) COOT_BIN_CASE(MIN, d) COOT_BIN_CASE(MAX, d)

#pragma unroll 1
    for (uint32_t i = 0; i < a.n_instr; ++i) {
      switch (a.key[i]) {
        COOT_CASES_AT(0)
        COOT_CASES_AT(1)
        COOT_CASES_AT(2)
        COOT_CASES_AT(3)
        COOT_CASES_AT(4)
        COOT_CASES_AT(5)
        COOT_CASES_AT(6)
        COOT_CASES_AT(7)
        COOT_CASES_AT(8)
        default:
          break;
      }
    }
#undef COOT_CASES_AT
#undef COOT_BIN_CASE
#undef COOT_UN_CASE
#undef COOT_SCALAR_CASE
#undef COOT_LOAD_CASE
#pragma unroll
    for (int w = 0; w < W; ++w) out[w] = st[0][w];
  }
};

// ---- operand loading ------------------------------------------------------
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
__device__ __forceinline__ void load_elem(const FusedArgs& a, u64 e, T (&in)[EV::K][1]) {
#pragma unroll
  for (int k = 0; k < EV::K; ++k) {
    if (!EV::kInterp || k < (int)a.n_operands)
      in[k][0] = __ldcg(reinterpret_cast<const T*>(a.in[k]) + e);
    else
      in[k][0] = T(0);
  }
}

// ---- the shared driver --------------------------------------------------
template <class T, int ACC, class EV, int U>
__global__ void __launch_bounds__(kThreads) fused_kernel(const __grid_constant__ FusedArgs a) {
  constexpr int W = Unit<T>::W;
  constexpr int K = EV::K;
  Accum<T, ACC> acc;
  acc.init();
  const u64 tid = (u64)blockIdx.x * kThreads + threadIdx.x;
  const u64 nthr = (u64)gridDim.x * kThreads;
  T* out = reinterpret_cast<T*>(a.out);

  // head (scalar)
  for (u64 e = tid; e < a.head; e += nthr) {
    T in[K][1], v[1];
    load_elem<T, EV>(a, e, in);
    EV::template eval<T, 1>(in, a, v);
    if (out) out[e] = v[0];
    acc.template add<1>(v);
  }
  // body: 16-byte units
  u64 u = tid;
  if constexpr (U > 1) {
    for (; u + (U - 1) * nthr < a.nunits; u += U * nthr) {
      T in[U][K][W];
#pragma unroll
      for (int j = 0; j < U; ++j) load_units<T, EV>(a, a.head + (u + j * nthr) * W, in[j]);
#pragma unroll
      for (int j = 0; j < U; ++j) {
        T v[W];
        EV::template eval<T, W>(in[j], a, v);
        if (out) store_unit<T>(out + a.head + (u + j * nthr) * W, v);
        acc.template add<W>(v);
      }
    }
  }
  for (; u < a.nunits; u += nthr) {
    T in[K][W], v[W];
    load_units<T, EV>(a, a.head + u * W, in);
    EV::template eval<T, W>(in, a, v);
    if (out) store_unit<T>(out + a.head + u * W, v);
    acc.template add<W>(v);
  }
  // tail (scalar)
  for (u64 e = a.tail_begin + tid; e < a.n; e += nthr) {
    T in[K][1], v[1];
    load_elem<T, EV>(a, e, in);
    EV::template eval<T, 1>(in, a, v);
    if (out) out[e] = v[0];
    acc.template add<1>(v);
  }

  if constexpr (ACC != ACC_NONE) {
    Accum<T, ACC> bt = block_reduce<T, ACC>(acc);
    grid_finish<T, ACC>(bt, a.partials, a.ticket, a.final_mode, a.kind, a.result, a.count);
  }
}

}  // namespace coot
