// Kernel tables and launchers, instantiated once per element type in
// kernels_<type>.cu (so the four type families compile in parallel).
#pragma once
#include <mutex>
#include <type_traits>
#include <unordered_set>

#include "coot_dim.cuh"
#include "coot_dim_tma.cuh"
#include "coot_internal.h"

namespace coot {

typedef void (*FusedFn)(const FusedArgs);
typedef void (*DimFn)(const DimArgs);

// LDG driver: U units per thread per iteration (prefetched one iteration
// ahead) so every thread keeps >= 64 bytes of loads in flight.
constexpr int unroll_for(int k) { return k <= 1 ? 4 : (k == 2 ? 2 : 1); }

// driver: 0 = LDG, 1 = TMA-staged, 2 = strided views (interpreter only),
// 3 = contiguous-column views
template <class T, int ACC, class EV, int U>
FusedFn driver_kernel(int driver) {
  if constexpr (EV::kInterp) {
    if (driver == 2) return &fused_strided_kernel<T, ACC, EV>;
  }
  // contiguous-column views: the catalog programs get their own instances (the
  // interpreter at 96 registers spilled and ran submatrix axpy at 0.57 of dense)
  if (driver == 3) return &fused_cols_tma_kernel<T, ACC, EV>;
  if constexpr (is_narrow<T>()) {
    // 16/8-bit types: TMA driver only (the host never plans driver 0 for them)
    return driver == 1 ? &fused_tma_kernel<T, ACC, EV> : nullptr;
  } else {
    if (driver == 1) return &fused_tma_kernel<T, ACC, EV>;
    return &fused_kernel<T, ACC, EV, U>;
  }
}

template <class T, int ACC, int... Code>
FusedFn catalog_kernel(int driver) {
  typedef StaticProg<Code...> P;
  if (driver == 2) return nullptr;  // element-strided views run on the interpreter
  if constexpr (P::template legal<T>()) {
    return driver_kernel<T, ACC, CatalogEval<P>, unroll_for(P::n_ops())>(driver);
  } else {
    return nullptr;
  }
}

// The statistics / index reductions (ACC_VAR, ACC_IMIN, ACC_IMAX) are
// instantiated for the plain-matrix program [L0] and the interpreter only (the
// host routes other catalog shapes to the interpreter for them).
template <class T, int ACC>
FusedFn pick_fused_acc(int catalog, int interp_large, int driver) {
  if constexpr ((ACC == ACC_SUMSQ || ACC == ACC_VAR) && !is_float<T>()) {
    return nullptr;
  } else {
    if constexpr (ACC >= ACC_VAR) {
      if (catalog == 0) return catalog_kernel<T, ACC, CL(0)>(driver);
    } else {
      switch (catalog) {
#define COOT_X(id, ...) \
  case id:              \
    return catalog_kernel<T, ACC, __VA_ARGS__>(driver);
        COOT_CATALOG(COOT_X)
#undef COOT_X
        default:
          break;
      }
    }
    if (interp_large == 1) return driver_kernel<T, ACC, InterpEval<8, 8>, 1>(driver);
    // shallow programs (fused stack depth <= 2) on the TMA driver: a 2-slot
    // stack leaves the registers for 4 units (16 elements) per dispatch
    if (interp_large == 2 && driver == 1) return &fused_tma_kernel<T, ACC, InterpEval<4, 2>>;
    return driver_kernel<T, ACC, InterpEval<4, 4>, 1>(driver);
  }
}

template <class T>
FusedFn pick_fused(const FusedPlan& p) {
  switch (p.acc) {
    case ACC_NONE: return pick_fused_acc<T, ACC_NONE>(p.catalog, p.interp_large, p.driver);
    case ACC_SUM: return pick_fused_acc<T, ACC_SUM>(p.catalog, p.interp_large, p.driver);
    case ACC_SUMSQ: return pick_fused_acc<T, ACC_SUMSQ>(p.catalog, p.interp_large, p.driver);
    case ACC_MINMAX: return pick_fused_acc<T, ACC_MINMAX>(p.catalog, p.interp_large, p.driver);
    case ACC_VAR: return pick_fused_acc<T, ACC_VAR>(p.catalog, p.interp_large, p.driver);
    case ACC_IMIN: return pick_fused_acc<T, ACC_IMIN>(p.catalog, p.interp_large, p.driver);
    case ACC_IMAX: return pick_fused_acc<T, ACC_IMAX>(p.catalog, p.interp_large, p.driver);
  }
  return nullptr;
}

// Opt every TMA-driver kernel into > 48 KB of dynamic shared memory once.
inline cudaError_t allow_smem(const void* fn, unsigned bytes) {
  static std::mutex mu;
  static std::unordered_set<const void*> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(fn)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e == cudaSuccess) done.insert(fn);
  (void)bytes;
  return e;
}

// Programmatic dependent launch: the kernel may be scheduled while the previous
// kernel on the stream is still finishing (once every CTA of that grid has
// executed pdl_trigger() or exited); every kernel launched this way begins
// with pdl_wait(), which blocks until the previous grid has completed and its
// memory is visible — so only the launch latency overlaps, never the data.
template <class Args>
cudaError_t launch_k(void (*k)(const Args), unsigned grid, unsigned block, unsigned smem,
                     cudaStream_t s, const Args& a, int pdl) {
  if (!pdl) {
    k<<<grid, block, smem, s>>>(a);
    return cudaGetLastError();
  }
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

template <class T>
cudaError_t launch_fused_t(const FusedPlan& p, const FusedArgs& a, cudaStream_t s) {
  FusedFn k = pick_fused<T>(p);
  if (!k) return cudaErrorInvalidDeviceFunction;
  if (p.driver == 1 || p.driver == 3) {
    cudaError_t e = allow_smem(reinterpret_cast<const void*>(k), p.smem);
    if (e != cudaSuccess) return e;
    // fused_tma_kernel with the small interpreter: in-band producer, 8 warps
    const bool inband = COOT_INTERP_INBAND && p.driver == 1 && p.catalog < 0 && p.interp_large != 1;
    return launch_k(k, p.grid, inband ? (unsigned)kConsumerWarps * 32 : (unsigned)kTmaThreads,
                    p.smem, s, a, p.pdl);
  }
  return launch_k(k, p.grid, kThreads, 0, s, a, p.pdl);
}

// Dimension sums: catalog [L0] (plain matrix) or the interpreter.
template <class T, template <class, class> class KER>
DimFn pick_dim_ev(const DimPlan& p) {
  if (p.catalog == 0) return KER<T, CatalogEval<StaticProg<CL(0)>>>::run;
  if (p.interp_large == 1) return KER<T, InterpEval<8, 8>>::run;
  return KER<T, InterpEval<4, 4>>::run;
}

template <class T, class EV>
struct Dim0Block {
  static constexpr DimFn run = &dim0_block_kernel<T, EV>;
};
template <class T, class EV>
struct Dim0Warp {
  static constexpr DimFn run = &dim0_warp_kernel<T, EV>;
};
// dim1_kernel_b8 only for catalog programs: capped at 85 registers the
// interpreter spills 400-700 B per thread (252-255 registers uncapped)
template <class EV>
struct IsInterp : std::false_type {};
template <int S, int I>
struct IsInterp<InterpEval<S, I>> : std::true_type {};
// (a specialisation, not ?: — taking both addresses instantiated both kernels)
template <class T, class EV, bool B8>
struct Dim1Pick {
  static constexpr DimFn run = &dim1_kernel<T, EV>;
};
template <class T, class EV>
struct Dim1Pick<T, EV, true> {
  static constexpr DimFn run = &dim1_kernel_b8<T, EV>;
};
template <class T, class EV>
struct Dim1 : Dim1Pick<T, EV, sizeof(T) == 1 && !IsInterp<EV>::value> {};
template <class T, class EV>
struct DimStrided {
  static constexpr DimFn run = &dim_strided_kernel<T, EV>;
};
template <class T, class EV>
struct Dim0Tma {
  static constexpr DimFn run = &dim0_tma_kernel<T, EV>;
};
template <class T, class EV>
struct Dim1Tma {
  static constexpr DimFn run = &dim1_tma_kernel<T, EV>;
};

template <class T>
cudaError_t launch_dim_t(const DimPlan& p, const DimArgs& a, cudaStream_t s) {
  DimFn k = nullptr;
  bool tma = false;
  switch (p.kernel) {
    case DIMK_DIM0_BLOCK: k = pick_dim_ev<T, Dim0Block>(p); break;
    case DIMK_DIM0_WARP: k = pick_dim_ev<T, Dim0Warp>(p); break;
    case DIMK_DIM1: k = pick_dim_ev<T, Dim1>(p); break;
    case DIMK_DIM0_TMA: k = pick_dim_ev<T, Dim0Tma>(p); tma = true; break;
    case DIMK_DIM1_TMA: k = pick_dim_ev<T, Dim1Tma>(p); tma = true; break;
    case DIMK_STRIDED: k = pick_dim_ev<T, DimStrided>(p); break;
  }
  if (!k) return cudaErrorInvalidDeviceFunction;
  if (tma) {
    cudaError_t e = allow_smem(reinterpret_cast<const void*>(k), p.smem);
    if (e != cudaSuccess) return e;
    return launch_k(k, p.grid, kTmaThreads, p.smem, s, a, p.pdl);
  }
  return launch_k(k, p.grid, kThreads, 0, s, a, p.pdl);
}

// ---- multi-GPU combine (K6) and partial bookkeeping -------------------------
// Scalar partial records are merged strictly in part order 0..nparts-1.
template <class T, int ACC>
__global__ void combine_rec_kernel(const Rec* parts, uint32_t nparts, uint32_t kind,
                                   void* result) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  combine_in_order<T, ACC>(nparts, [&](uint32_t p) { return parts[p]; }, kind, result);
}

// Vector partials (SUM_DIM*): result[i] = round(sum_p parts[p][i]), p in order.
template <class T>
__global__ void combine_vec_kernel(const typename SumT<T>::type* parts, uint32_t nparts, u64 len,
                                   typename ResultT<T>::type* result) {
  typedef typename SumT<T>::type S;
  typedef typename ResultT<T>::type R;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (u64)gridDim.x * blockDim.x) {
    S s = S(0);
    for (uint32_t p = 0; p < nparts; ++p) s = sum_add<S>(s, parts[(u64)p * len + i]);
    if constexpr (is_float<T>()) result[i] = round_to<R>(s);
    else result[i] = (R)s;
  }
}

// Identity record for an empty shard (no elements => no kernel to publish it):
// written to `out`, or (exchange mode) published to the peers' mailboxes and
// combined into the result `out`.
template <class T, int ACC>
__global__ void empty_rec_kernel(Rec* out, const Exchange ex, uint32_t kind, int exchange) {
  Accum<T, ACC> acc;
  acc.init();
  if (exchange) exchange_finish<T, ACC>(acc.to_rec(0), ex, kind, out);
  else *out = acc.to_rec(0);
}

template <class T>
cudaError_t launch_combine_t(uint32_t kind, int acc, const void* parts, uint32_t nparts, u64 len,
                             void* result, unsigned grid, cudaStream_t s) {
  if (kind == COOT_RED_SUM_DIM0 || kind == COOT_RED_SUM_DIM1) {
    combine_vec_kernel<T><<<grid, kThreads, 0, s>>>(
        reinterpret_cast<const typename SumT<T>::type*>(parts), nparts, len,
        reinterpret_cast<typename ResultT<T>::type*>(result));
    return cudaGetLastError();
  }
  const Rec* r = reinterpret_cast<const Rec*>(parts);
  switch (acc) {
    case ACC_SUM: combine_rec_kernel<T, ACC_SUM><<<1, 32, 0, s>>>(r, nparts, kind, result); break;
    case ACC_SUMSQ:
      if constexpr (is_float<T>()) {
        combine_rec_kernel<T, ACC_SUMSQ><<<1, 32, 0, s>>>(r, nparts, kind, result);
        break;
      } else {
        return cudaErrorInvalidValue;
      }
    case ACC_MINMAX:
      combine_rec_kernel<T, ACC_MINMAX><<<1, 32, 0, s>>>(r, nparts, kind, result);
      break;
    case ACC_VAR:
      if constexpr (is_float<T>()) {
        combine_rec_kernel<T, ACC_VAR><<<1, 32, 0, s>>>(r, nparts, kind, result);
        break;
      } else {
        return cudaErrorInvalidValue;
      }
    case ACC_IMIN: combine_rec_kernel<T, ACC_IMIN><<<1, 32, 0, s>>>(r, nparts, kind, result); break;
    case ACC_IMAX: combine_rec_kernel<T, ACC_IMAX><<<1, 32, 0, s>>>(r, nparts, kind, result); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_empty_rec_t(int acc, void* out, cudaStream_t s, const Exchange* ex,
                               uint32_t kind) {
  Rec* r = reinterpret_cast<Rec*>(out);
  const Exchange e = ex ? *ex : Exchange{};
  const int x = ex != nullptr;
  switch (acc) {
    case ACC_SUM: empty_rec_kernel<T, ACC_SUM><<<1, 1, 0, s>>>(r, e, kind, x); break;
    case ACC_SUMSQ:
      if constexpr (is_float<T>()) {
        empty_rec_kernel<T, ACC_SUMSQ><<<1, 1, 0, s>>>(r, e, kind, x);
        break;
      } else {
        return cudaErrorInvalidValue;
      }
    case ACC_MINMAX: empty_rec_kernel<T, ACC_MINMAX><<<1, 1, 0, s>>>(r, e, kind, x); break;
    case ACC_VAR:
      if constexpr (is_float<T>()) {
        empty_rec_kernel<T, ACC_VAR><<<1, 1, 0, s>>>(r, e, kind, x);
        break;
      } else {
        return cudaErrorInvalidValue;
      }
    case ACC_IMIN: empty_rec_kernel<T, ACC_IMIN><<<1, 1, 0, s>>>(r, e, kind, x); break;
    case ACC_IMAX: empty_rec_kernel<T, ACC_IMAX><<<1, 1, 0, s>>>(r, e, kind, x); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ---- synthetic input generator (harness) ---------
__device__ __forceinline__ u64 splitmix_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <class T>
__global__ void fill_kernel(uint32_t kind, u64 seed, u64 stream, u64 start, u64 count,
                            u64 n_rows, u64 k, T* out) {
  const u64 key = seed ^ (stream * 0xD1B54A32D192ED03ull);
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (u64)gridDim.x * blockDim.x) {
    const u64 g = start + i;
    T v;
    if (kind == 0) {
      const u64 h = splitmix_mix(key + (g + 1) * 0x9E3779B97F4A7C15ull);
      if constexpr (std::is_same<T, bf16>::value) v = half_from_f32<bf16>((float)(h >> 56) * 0x1p-8f);
      else if constexpr (std::is_same<T, f16>::value) v = half_from_f32<f16>((float)(h >> 53) * 0x1p-11f);
      else if constexpr (std::is_same<T, e4m3>::value) v = fp8_from_f32<e4m3>((float)(h >> 60) * 0x1p-4f);
      else if constexpr (std::is_same<T, e5m2>::value) v = fp8_from_f32<e5m2>((float)(h >> 61) * 0x1p-3f);
      else if constexpr (sizeof(T) == 4 && is_float<T>()) v = (float)(h >> 40) * 0x1p-24f;
      else if constexpr (is_float<T>()) v = (double)(h >> 11) * 0x1p-53;
      else if constexpr (sizeof(T) == 4) v = (T)(h >> 32);
      else v = (T)h;
    } else {
      u64 iv = 0;
      switch (kind) {
        case 1: iv = 1; break;
        case 2: iv = g; break;
        case 3: iv = g % k; break;
        case 4: iv = g / n_rows; break;
        case 5: iv = g % n_rows; break;
        default: iv = 0; break;
      }
      if constexpr (is_half<T>()) v = half_from_f64<T>((double)iv);
      else if constexpr (is_fp8<T>()) v = fp8_from_f32<T>((float)iv);  // exact below 2^24; saturates far sooner
      else v = (T)iv;
    }
    out[i] = v;
  }
}

template <class T>
cudaError_t launch_fill_t(uint32_t kind, u64 seed, u64 stream, u64 start, u64 count, u64 n_rows,
                          u64 k, void* out, unsigned grid, cudaStream_t s) {
  fill_kernel<T><<<grid, kThreads, 0, s>>>(kind, seed, stream, start, count, n_rows ? n_rows : 1,
                                           k ? k : 1, reinterpret_cast<T*>(out));
  return cudaGetLastError();
}

// Each type's fused kernels are instantiated per reduction kind in their own
// translation unit (kernels_<type>_acc<k>.cu) so the build parallelises; the
// type's main unit sees them as extern templates.
#define COOT_EXTERN_ACC(T)                                                  \
  extern template FusedFn pick_fused_acc<T, ACC_NONE>(int, int, int);       \
  extern template FusedFn pick_fused_acc<T, ACC_SUM>(int, int, int);        \
  extern template FusedFn pick_fused_acc<T, ACC_SUMSQ>(int, int, int);      \
  extern template FusedFn pick_fused_acc<T, ACC_MINMAX>(int, int, int);     \
  extern template FusedFn pick_fused_acc<T, ACC_VAR>(int, int, int);        \
  extern template FusedFn pick_fused_acc<T, ACC_IMIN>(int, int, int);       \
  extern template FusedFn pick_fused_acc<T, ACC_IMAX>(int, int, int);

#define COOT_INSTANTIATE_ACC(T, ACC) template FusedFn pick_fused_acc<T, ACC>(int, int, int);

#define COOT_INSTANTIATE(T)                                                                     \
  template cudaError_t launch_fused_t<T>(const FusedPlan&, const FusedArgs&, cudaStream_t);   \
  template cudaError_t launch_dim_t<T>(const DimPlan&, const DimArgs&, cudaStream_t);         \
  template cudaError_t launch_combine_t<T>(uint32_t, int, const void*, uint32_t, u64, void*,  \
                                           unsigned, cudaStream_t);                           \
  template cudaError_t launch_empty_rec_t<T>(int, void*, cudaStream_t, const Exchange*,       \
                                             uint32_t);                                       \
  template cudaError_t launch_fill_t<T>(uint32_t, u64, u64, u64, u64, u64, u64, void*,        \
                                        unsigned, cudaStream_t);

}  // namespace coot
