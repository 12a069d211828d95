// K4 sum(X,0) and K5 sum(X,1) over a column-major m x n expression X
// (Armadillo convention, R3: dim 0 -> column sums, a Row of n; dim 1 -> row
// sums, a Col of m).  X may itself be a fused element-wise expression: every
// element is produced by the same evaluators as the fused pass (K1 [L0] or
// K2), so nothing is materialised.
//
// Both kernels are single-launch and deterministic: the split of the work
// into (column, segment) / (row tile, column chunk) pieces depends only on
// (m, n, SM count); split pieces publish unrounded partials that the LAST
// arriving block (per column / per row tile, via a self-resetting ticket)
// combines in fixed piece order before rounding once to eT.
#pragma once
#include "coot_fused.cuh"

namespace coot {

struct DimArgs {
  FusedArgs f;          // operands, scalars, program (f.n unused)
  u64 m, n;             // rows, cols
  void* result;         // eT out (FINAL_ROUND) or S partial vector (FINAL_PARTIAL)
  void* part;           // scratch: S partials of split pieces
  unsigned* tickets;    // scratch: per column (dim0) / per row tile (dim1)
  u64 seg_len;          // dim0: rows per segment (multiple of 4)
  uint32_t nseg;        // dim0: segments per column (1 = no split)
  uint32_t vec_ok;      // all operand columns 16-byte aligned alike
  uint32_t final_mode;
  uint32_t tpr;         // dim1: threads per row tile (32..256, power of two)
  u64 ccols;            // dim1: columns per chunk
  uint32_t nchunks;     // dim1: column chunks (1 = no split)
  uint32_t nrt;         // dim1: row tiles
  uint32_t cg;          // dim1 TMA: columns per pipeline stage
  uint32_t dim;         // strided kernel: 0 or 1
  u64 vcap;             // FINAL_EXCHANGE (sum(X,1) over column shards): rows per
                        // vector-mailbox slot; the mailboxes are f.ex.mbox[]
};

// ---- in-kernel exchange of sum(X,1) partial vectors (FINAL_EXCHANGE) -------
// Column shards of a Mat: every rank holds all n_rows of some columns, so each
// rank's row sums are partials of the global ones.  Vector mailbox of a rank
// (coot_vec_mailbox_create): u64 flag[MAX_RANKS] at 0, u64 tag[2][MAX_RANKS]
// at 64 (epoch of each slot), S data[2][MAX_RANKS][vcap] at 256; half =
// epoch & 1 (double-buffered like the record mailboxes, §7).
//  1. every finisher of a row tile (the CTA that rounds its rows in the
//     single-GPU kernel) instead stores its rows' unrounded S partials into
//     data[half][rank][row] of EVERY rank's mailbox (NVLink P2P stores);
//  2. it then adds its row count to a ticket; the CTA completing the m rows
//     of this rank (all tiles published) tags and flags every mailbox and waits
//     for every rank's flag in its own — nothing else of this rank is still
//     running, so the wait cannot hold up this rank's own work;
//  3. that CTA combines the P vectors in rank order 0..P-1 (the same S sum as
//     coot_combine's combine_vec_kernel) and rounds once: identical bits on
//     every rank and to the host-staged partial -> all-gather -> combine path.
constexpr u64 kVecMboxHeader = 256;
template <class T>
__device__ __forceinline__ void publish_dim_value(const DimArgs& d, u64 idx,
                                                  typename SumT<T>::type s) {
  typedef typename SumT<T>::type S;
  const Exchange& ex = d.f.ex;
  const u64 off = ((ex.epoch & 1ull) * COOT_MAX_RANKS + ex.rank) * d.vcap + idx;
  for (uint32_t p = 0; p < ex.nranks; ++p)
    __stcg(reinterpret_cast<S*>(ex.mbox[p] + kVecMboxHeader) + off, s);
}

// The last of this rank's finishers (all m rows published): flags, wait,
// rank-order combine of all rows by the NT threads of the calling group.
template <class T, class Sync>
__device__ void vec_exchange_finish(const DimArgs& d, uint32_t tid, uint32_t NT, Sync sync) {
  typedef typename SumT<T>::type S;
  typedef typename ResultT<T>::type R;
  const Exchange& ex = d.f.ex;
  const uint32_t P = ex.nranks;
  const u64 half = (ex.epoch & 1ull) * COOT_MAX_RANKS;
  if (tid == 0) {
    __threadfence_system();  // this CTA's data stores (the others fenced before their ticket)
    for (uint32_t p = 0; p < P; ++p)
      __stcg(reinterpret_cast<unsigned long long*>(ex.mbox[p] + 64) + half + ex.rank, ex.epoch);
    __threadfence_system();
    for (uint32_t p = 0; p < P; ++p)
      st_release_sys(reinterpret_cast<unsigned long long*>(ex.mbox[p]) + ex.rank, ex.epoch);
    const unsigned long long* own = reinterpret_cast<const unsigned long long*>(ex.mbox[ex.rank]);
    const unsigned long long t0 = globaltimer_ns();
    for (uint32_t q = 0; q < P; ++q) {
      while (ld_acquire_sys(own + q) < ex.epoch) {
        __nanosleep(256);
        if (globaltimer_ns() - t0 > 20000000000ull) __trap();  // a rank never arrived
      }
    }
    for (uint32_t q = 0; q < P; ++q)  // every slot must hold this call's vector
      if (__ldcg(own + 8 + half + q) != ex.epoch) __trap();
    d.tickets[d.nrt] = 0u;  // self-reset for the next call
  }
  sync();
  const S* data = reinterpret_cast<const S*>(ex.mbox[ex.rank] + kVecMboxHeader) + half * d.vcap;
  // one CTA combines all m rows, 8 rows per thread at a time so that their
  // loads are in flight together (a rolled loop paid an L2 round trip per
  // row); each row still sums q = 0..P-1 in order, as combine_vec_kernel
  for (u64 r0 = tid; r0 < d.m; r0 += 8ull * NT) {
    S tot[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) tot[k] = S(0);
    for (uint32_t q = 0; q < P; ++q) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const u64 r = r0 + (u64)k * NT;
        if (r < d.m) tot[k] = sum_add<S>(tot[k], __ldcg(data + (u64)q * d.vcap + r));
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const u64 r = r0 + (u64)k * NT;
      if (r < d.m) {
        R v;
        if constexpr (is_float<T>()) v = round_to<R>(tot[k]);
        else v = (R)tot[k];
        reinterpret_cast<R*>(d.result)[r] = v;
      }
    }
  }
}

// A finisher's rows are published: count them; the group completing the m
// rows runs the exchange.  Called by every thread of the group (NT threads,
// synchronised by `sync`); `flag` is a shared word of the group.
template <class T, class Sync>
__device__ __forceinline__ void vec_exchange_arrive(const DimArgs& d, u64 rows, uint32_t tid,
                                                    uint32_t NT, bool* flag, Sync sync) {
  __threadfence_system();  // this thread's remote stores before the ticket
  sync();
  if (tid == 0) {
    const unsigned old = atomicAdd(&d.tickets[d.nrt], (unsigned)rows);
    *flag = (u64)old + rows == d.m;
  }
  sync();
  if (*flag) vec_exchange_finish<T>(d, tid, NT, sync);
  sync();  // *flag is rewritten by the group's next call
}

template <class T>
__device__ __forceinline__ void publish_dim_value(const DimArgs& d, u64 idx,
                                                  typename SumT<T>::type s);
template <class T>
__device__ __forceinline__ void store_dim_value(const DimArgs& d, u64 idx,
                                                typename SumT<T>::type s) {
  typedef typename SumT<T>::type S;
  if (d.final_mode == FINAL_EXCHANGE) {
    publish_dim_value<T>(d, idx, s);
  } else if (d.final_mode == FINAL_PARTIAL) {
    reinterpret_cast<S*>(d.result)[idx] = s;
  } else {
    typedef typename ResultT<T>::type R;  // f32 for the 8-bit storage types
    R v;
    if constexpr (is_float<T>()) v = round_to<R>(s);
    else v = (R)s;
    reinterpret_cast<R*>(d.result)[idx] = v;
  }
}

// sum(X, dim) never stores element values.  For the plain-matrix program on
// E4M3 the f32 round trip of a value (exact decode, saturating re-encode, R25)
// is the identity except for the sign of a NaN, which a sum propagates as NaN
// either way — so the raw bytes go straight to the accumulation.  (Not E5M2:
// its +-inf saturate to +-57344 on re-encoding.)
template <class T, class EV, int W, class In>
__device__ __forceinline__ void dim_eval(const In& in, const FusedArgs& f, T (&v)[W]) {
  if constexpr (EV::kIdentity && std::is_same<T, e4m3>::value) {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = in[0][w];
  } else {
    EV::template eval<T, W>(in, f, v);
  }
}

// ---- K4a: block per (column, segment) — tall columns ------------------------
template <class T, class EV>
__global__ void __launch_bounds__(kThreads) dim0_block_kernel(const __grid_constant__ DimArgs d) {
  pdl_wait();
  constexpr int W = Unit<T>::W;
  constexpr int K = EV::K;
  typedef typename SumT<T>::type S;
  const u64 npieces = d.n * d.nseg;
  for (u64 p = blockIdx.x; p < npieces; p += gridDim.x) {
    const u64 j = p / d.nseg, s = p % d.nseg;
    const u64 r0 = s * d.seg_len;
    const u64 len = (d.m - r0) < d.seg_len ? (d.m - r0) : d.seg_len;
    const u64 e0 = j * d.m + r0;
    u64 head = len, nun = 0;
    if (d.vec_ok) {
      const uintptr_t addr = reinterpret_cast<uintptr_t>(d.f.in[0]) + e0 * sizeof(T);
      head = ((16 - (addr & 15)) & 15) / sizeof(T);
      if (head > len) head = len;
      nun = (len - head) / W;
    }
    const u64 tb = head + nun * W;
    Accum<T, ACC_SUM> acc;
    acc.init();
    for (u64 i = threadIdx.x; i < head; i += kThreads) {
      T in[K][1], v[1];
      load_elem<T, EV>(d.f, e0 + i, in);
      dim_eval<T, EV, 1>(in, d.f, v);
      acc.template add<1>(v);
    }
    u64 u = threadIdx.x;
    constexpr int UL = EV::kInterp ? 1 : 4;  // units whose loads are issued together
    if constexpr (UL > 1) {
      for (; u + (UL - 1) * kThreads < nun; u += UL * kThreads) {
        T in[UL][K][W];
#pragma unroll
        for (int q = 0; q < UL; ++q)
          load_units<T, EV>(d.f, e0 + head + (u + q * kThreads) * W, in[q]);
#pragma unroll
        for (int q = 0; q < UL; ++q) {
          T v[W];
          dim_eval<T, EV, W>(in[q], d.f, v);
          acc.template add<W>(v);
        }
      }
    }
    for (; u < nun; u += kThreads) {
      T in[K][W], v[W];
      load_units<T, EV>(d.f, e0 + head + u * W, in);
      dim_eval<T, EV, W>(in, d.f, v);
      acc.template add<W>(v);
    }
    for (u64 i = tb + threadIdx.x; i < len; i += kThreads) {
      T in[K][1], v[1];
      load_elem<T, EV>(d.f, e0 + i, in);
      dim_eval<T, EV, 1>(in, d.f, v);
      acc.template add<1>(v);
    }
    Accum<T, ACC_SUM> bt = block_reduce<T, ACC_SUM>(acc);
    if (d.nseg == 1) {
      if (threadIdx.x == 0) store_dim_value<T>(d, j, bt.s);
    } else {
      __shared__ bool last;
      if (threadIdx.x == 0) {
        reinterpret_cast<S*>(d.part)[p] = bt.s;
        __threadfence();
        const unsigned t = atomicAdd(&d.tickets[j], 1u);
        last = (t == d.nseg - 1);
        if (last) {
          __threadfence();
          S tot = S(0);
          for (uint32_t q = 0; q < d.nseg; ++q)
            tot = sum_add<S>(tot, __ldcg(reinterpret_cast<const S*>(d.part) + j * d.nseg + q));
          store_dim_value<T>(d, j, tot);
          d.tickets[j] = 0u;
        }
      }
      __syncthreads();
    }
  }
}

// ---- K4b: warp per column — short columns (m < 2048) ------------------------
template <class T, class EV>
__global__ void __launch_bounds__(kThreads) dim0_warp_kernel(const __grid_constant__ DimArgs d) {
  pdl_wait();
  constexpr int K = EV::K;
  const int lane = threadIdx.x & 31;
  const u64 warp = ((u64)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * kThreads) >> 5;
  for (u64 j = warp; j < d.n; j += nwarps) {
    Accum<T, ACC_SUM> acc;
    acc.init();
    const u64 e0 = j * d.m;
    for (u64 i = lane; i < d.m; i += 32) {
      T in[K][1], v[1];
      load_elem<T, EV>(d.f, e0 + i, in);
      dim_eval<T, EV, 1>(in, d.f, v);
      acc.template add<1>(v);
    }
    acc.warp_reduce();
    if (lane == 0) store_dim_value<T>(d, j, acc.s);
  }
}

// ---- strided views: sum(view, 0) warp per column, sum(view, 1) thread per row --
// Operand k element (i, j) at in[k][i*inc[k] + j*ld[k]] (d.f.ld / d.f.inc).
template <class T, class EV>
__device__ __forceinline__ void load_elem_strided(const FusedArgs& a, u64 i, u64 j,
                                                  T (&in)[EV::K][1]) {
#pragma unroll
  for (int k = 0; k < EV::K; ++k) {
    if (!EV::kInterp || k < (int)a.n_operands)
      in[k][0] = ldcg_elem(reinterpret_cast<const T*>(a.in[k]) + i * a.inc[k] + j * a.ld[k]);
    else
      in[k][0] = T(0);
  }
}

template <class T, class EV>
__global__ void __launch_bounds__(kThreads) dim_strided_kernel(const __grid_constant__ DimArgs d) {
  pdl_wait();
  if (d.dim == 0) {
    const int lane = threadIdx.x & 31;
    const u64 warp = ((u64)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const u64 nwarps = ((u64)gridDim.x * kThreads) >> 5;
    for (u64 j = warp; j < d.n; j += nwarps) {
      Accum<T, ACC_SUM> acc;
      acc.init();
      for (u64 i = lane; i < d.m; i += 32) {
        T in[EV::K][1], v[1];
        load_elem_strided<T, EV>(d.f, i, j, in);
        dim_eval<T, EV, 1>(in, d.f, v);
        acc.template add<1>(v);
      }
      acc.warp_reduce();
      if (lane == 0) store_dim_value<T>(d, j, acc.s);
    }
  } else {
    for (u64 i = (u64)blockIdx.x * kThreads + threadIdx.x; i < d.m;
         i += (u64)gridDim.x * kThreads) {
      Accum<T, ACC_SUM> acc;
      acc.init();
      for (u64 j = 0; j < d.n; ++j) {
        T in[EV::K][1], v[1];
        load_elem_strided<T, EV>(d.f, i, j, in);
        dim_eval<T, EV, 1>(in, d.f, v);
        acc.template add<1>(v);
      }
      store_dim_value<T>(d, i, acc.s);
    }
  }
}

// ---- K5: row sums — row tile x column chunk ---------------------------------
// Block b -> row tile rt = b mod nrt, column chunk cc = b / nrt.  Threads form
// G = 256/tpr groups; group g walks columns c0+g, c0+g+G, ... of the chunk and
// each thread owns W consecutive rows (one 16-byte unit per column) of the
// tile (vec path) or rows r0+q, r0+q+tpr, ... (scalar path).  Groups are
// combined in g order through shared memory; chunks in cc order by the last
// block of the row tile.
template <class T, class EV>
__device__ __forceinline__ void dim1_body(const DimArgs& d) {
  pdl_wait();
  constexpr int W = Unit<T>::W;
  constexpr int K = EV::K;
  typedef typename SumT<T>::type S;
  __shared__ S red[kThreads * W];
  __shared__ bool last;
  const uint32_t tpr = d.tpr, G = kThreads / tpr;
  const uint32_t g = threadIdx.x / tpr, q = threadIdx.x % tpr;
  const u64 rt = blockIdx.x % d.nrt, cc = blockIdx.x / d.nrt;
  const u64 R = (u64)tpr * W;
  const u64 r0 = rt * R;
  const u64 c0 = cc * d.ccols;
  const u64 c1 = (c0 + d.ccols < d.n) ? c0 + d.ccols : d.n;
  S acc[W];
#pragma unroll
  for (int w = 0; w < W; ++w) acc[w] = S(0);

  // Uniform per block: a full tile uses the unit map, a ragged last tile the
  // scalar map (both cover rows [r0, r0 + R) exactly once).
  const bool vec_rows = d.vec_ok && (r0 + R <= d.m);
  if (vec_rows) {
    const u64 rbase = r0 + (u64)q * W;
    u64 j = c0 + g;
    for (; j + 3 * G < c1; j += 4 * G) {
      T v[4][W];
      if constexpr (!EV::kInterp) {
        T in[4][K][W];
#pragma unroll
        for (int c = 0; c < 4; ++c) load_units<T, EV>(d.f, (j + c * G) * d.m + rbase, in[c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) dim_eval<T, EV, W>(in[c], d.f, v[c]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          T in[K][W];
          load_units<T, EV>(d.f, (j + c * G) * d.m + rbase, in);
          dim_eval<T, EV, W>(in, d.f, v[c]);
        }
      }
      if constexpr (is_narrow<T>()) {
        // widen each column's unit on its own (adjacent-byte pairs decode
        // without repacking), then the same f32 pairwise sum of the 4 columns
        // as unit_sum<T, 4> — bit-identical to it
        float x[4][W];
#pragma unroll
        for (int c = 0; c < 4; ++c) widen_f32<T, W>(v[c], x[c]);
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const float c4[4] = {x[0][w], x[1][w], x[2][w], x[3][w]};
          acc[w] = sum_add<S>(acc[w], (S)pairwise_f32<4>(c4));
        }
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          T col4[4] = {v[0][w], v[1][w], v[2][w], v[3][w]};
          if constexpr (is_float<T>()) {
            acc[w] = sum_add<S>(acc[w], unit_sum<T, 4>(col4));
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[w] = sum_add<S>(acc[w], (S)col4[c]);
          }
        }
      }
    }
    for (; j < c1; j += G) {
      T in[K][W], v[W];
      load_units<T, EV>(d.f, j * d.m + rbase, in);
      dim_eval<T, EV, W>(in, d.f, v);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        T one[1] = {v[w]};
        acc[w] = sum_add<S>(acc[w], unit_sum<T, 1>(one));
      }
    }
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const u64 r = r0 + q + (u64)w * tpr;
      if (r < d.m) {
        for (u64 j = c0 + g; j < c1; j += G) {
          T in[K][1], v[1];
          load_elem<T, EV>(d.f, j * d.m + r, in);
          dim_eval<T, EV, 1>(in, d.f, v);
          acc[w] = sum_add<S>(acc[w], unit_sum<T, 1>(v));
        }
      }
    }
  }
  // combine column groups in g order
#pragma unroll
  for (int w = 0; w < W; ++w) red[threadIdx.x * W + w] = acc[w];
  __syncthreads();
  if (g == 0) {
    for (uint32_t h = 1; h < G; ++h) {
#pragma unroll
      for (int w = 0; w < W; ++w) acc[w] = sum_add<S>(acc[w], red[(h * tpr + q) * W + w]);
    }
  }
  // row index owned by (q, w)
  auto row_of = [&](int w) -> u64 {
    return vec_rows ? r0 + (u64)q * W + w : r0 + q + (u64)w * tpr;
  };
  auto block_sync = [] { __syncthreads(); };
  const u64 tile_rows = (d.m - r0) < R ? (d.m - r0) : R;
  if (d.nchunks == 1) {
    if (g == 0) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const u64 r = row_of(w);
        if (r < d.m) store_dim_value<T>(d, r, acc[w]);
      }
    }
    if (d.final_mode == FINAL_EXCHANGE)
      vec_exchange_arrive<T>(d, tile_rows, threadIdx.x, kThreads, &last, block_sync);
    return;
  }
  S* part = reinterpret_cast<S*>(d.part);
  if (g == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const u64 r = row_of(w);
      if (r < d.m) part[cc * d.m + r] = acc[w];
    }
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(&d.tickets[rt], 1u);
    last = (t == d.nchunks - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (g == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const u64 r = row_of(w);
      if (r < d.m) {
        S tot = S(0);
        for (uint32_t c = 0; c < d.nchunks; ++c) tot = sum_add<S>(tot, __ldcg(part + c * d.m + r));
        store_dim_value<T>(d, r, tot);
      }
    }
  }
  if (threadIdx.x == 0) d.tickets[rt] = 0u;
  if (d.final_mode == FINAL_EXCHANGE)
    vec_exchange_arrive<T>(d, tile_rows, threadIdx.x, kThreads, &last, block_sync);
}

template <class T, class EV>
__global__ void __launch_bounds__(kThreads) dim1_kernel(const __grid_constant__ DimArgs d) {
  dim1_body<T, EV>(d);
}
// 8-bit types: <= 85 registers so 3 CTAs fit per SM (86 registers allowed only
// 2, and the host's 4-per-SM grid ran in two waves: E4M3 sum(X,1) at 50 % of
// DRAM bandwidth, long-scoreboard bound with 16 warps per SM)
// (a separate kernel: an explicit minBlocks = 1 on the others changed their
// register allocation and cost bf16 sum(X,1) 17 %)
template <class T, class EV>
__global__ void __launch_bounds__(kThreads, 3) dim1_kernel_b8(const __grid_constant__ DimArgs d) {
  dim1_body<T, EV>(d);
}

}  // namespace coot
