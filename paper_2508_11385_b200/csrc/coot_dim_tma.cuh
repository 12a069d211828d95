// TMA-staged sum(X,0) / sum(X,1) (K4/K5 default path; R3).
//
// Same producer/consumer structure as fused_tma_kernel: one producer warp
// streams contiguous column segments of every operand into a shared-memory
// ring with 1-D bulk copies (cp.async.bulk + mbarrier complete_tx, L2
// evict-first); 8 consumer warps evaluate the (fused) expression out of shared
// memory and accumulate.  The ring runs continuously across the pieces a CTA
// owns, so piece boundaries (block reductions, partial write-backs) overlap
// the next piece's copies.
//
// dim 0 (column sums, a Row): piece = (column j, segment s); a column is a
//   contiguous run of m elements, streamed as tiles of 512 units.  Segment
//   partials are merged in segment order by the last-arriving CTA.
// dim 1 (row sums, a Col): piece = (row tile rt, column chunk cc); a stage
//   holds `cg` column segments of R = 256 * W rows; consumer thread t owns
//   the 16-byte unit t (W rows) of every column.  Chunk partials are merged in
//   chunk order by the last CTA of the row tile.
// Both need every operand column 16-byte aligned (m * sizeof(T) % 16 == 0,
// same base misalignment); otherwise the LDG kernels of coot_dim.cuh run.
#pragma once
#include "coot_dim.cuh"

namespace coot {

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}

// Fixed-order sum over the 256 consumer threads; result valid in thread 0.
template <class S>
__device__ __forceinline__ S consumer_reduce_sum(S v, S* ws) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = sum_add<S>(v, shfl_xor(v, m));
  if (lane == 0) ws[warp] = v;
  consumer_sync();
  S r = S(0);
  if (warp == 0) {
    r = lane < kConsumerWarps ? ws[lane] : S(0);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) r = sum_add<S>(r, shfl_xor(r, m));
  }
  consumer_sync();  // ws may be reused by the next piece
  return r;
}

// ---- dim 0 -------------------------------------------------------------------
template <class T, class EV>
__global__ void __launch_bounds__(kTmaThreads, tma_min_ctas<EV>()) dim0_tma_kernel(const __grid_constant__ DimArgs d) {
  pdl_wait();
  constexpr int W = Unit<T>::W;
  constexpr int K = EV::K;
  typedef typename SumT<T>::type S;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ S ws[kConsumerWarps];
  const FusedArgs& a = d.f;
  const uint32_t nk = EV::kInterp ? a.n_operands : (uint32_t)K;
  const uint32_t NS = a.stages, TU = a.tile_units;
  const uint32_t tile_bytes = TU * 16u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * nk * tile_bytes);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const u64 npieces = d.n * d.nseg;
  const uintptr_t base0 = reinterpret_cast<uintptr_t>(a.in[0]);

  if (warp == kConsumerWarps) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t s = 0, ph = 0;
      u64 i = 0;
      for (u64 p = blockIdx.x; p < npieces; p += gridDim.x) {
        const u64 j = p / d.nseg, r0 = (p % d.nseg) * d.seg_len;
        const u64 len = (d.m - r0) < d.seg_len ? (d.m - r0) : d.seg_len;
        const u64 e0 = j * d.m + r0;
        const u64 head = (((16 - ((base0 + e0 * sizeof(T)) & 15)) & 15) / sizeof(T)) < len
                             ? ((16 - ((base0 + e0 * sizeof(T)) & 15)) & 15) / sizeof(T)
                             : len;
        const u64 nun = (len - head) / W;
        for (u64 u0 = 0; u0 < nun; u0 += TU, ++i) {
          if (i >= NS) mbar_wait(&empty[s], ph ^ 1u);
          const uint32_t nu = (uint32_t)((nun - u0) < TU ? (nun - u0) : TU);
          mbar_expect_tx(&full[s], nu * 16u * nk);
          for (uint32_t k = 0; k < nk; ++k)
            bulk_g2s(smem + ((size_t)s * nk + k) * tile_bytes,
                     reinterpret_cast<const char*>(a.in[k]) + (e0 + head) * sizeof(T) + u0 * 16,
                     nu * 16u, &full[s], pol);
          if (++s == NS) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else {
  // consumers (named barrier 1 synchronises the 256 consumer threads only)
  constexpr int UD = units_per_dispatch<T, EV>();
  uint32_t s = 0, ph = 0;
  for (u64 p = blockIdx.x; p < npieces; p += gridDim.x) {
    const u64 j = p / d.nseg, r0 = (p % d.nseg) * d.seg_len;
    const u64 len = (d.m - r0) < d.seg_len ? (d.m - r0) : d.seg_len;
    const u64 e0 = j * d.m + r0;
    const u64 head = (((16 - ((base0 + e0 * sizeof(T)) & 15)) & 15) / sizeof(T)) < len
                         ? ((16 - ((base0 + e0 * sizeof(T)) & 15)) & 15) / sizeof(T)
                         : len;
    const u64 nun = (len - head) / W;
    Accum<T, ACC_SUM> acc;
    acc.init();
    for (u64 i = threadIdx.x; i < head; i += kConsumerWarps * 32) {
      T in[K][1], v[1];
      load_elem<T, EV>(a, e0 + i, in);
      EV::template eval<T, 1>(in, a, v);
      acc.template add<1>(v);
    }
    for (u64 u0 = 0; u0 < nun; u0 += TU) {
      const uint32_t nu = (uint32_t)((nun - u0) < TU ? (nun - u0) : TU);
      mbar_wait(&full[s], ph);
      const unsigned char* stg = smem + (size_t)s * nk * tile_bytes;
      for (uint32_t i = threadIdx.x; i < nu; i += UD * kConsumerWarps * 32) {
        T v[UD * W];
        EV::template eval_src<T, UD * W>(SmemSrc<T, UD>{stg + (size_t)i * 16, tile_bytes}, a, v);
#pragma unroll
        for (int q = 0; q < UD; ++q) {
          if (q == 0 || i + q * kConsumerWarps * 32 < nu) {
            T vq[W];
#pragma unroll
            for (int w = 0; w < W; ++w) vq[w] = v[q * W + w];
            acc.template add<W>(vq);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
    }
    for (u64 i = head + nun * W + threadIdx.x; i < len; i += kConsumerWarps * 32) {
      T in[K][1], v[1];
      load_elem<T, EV>(a, e0 + i, in);
      EV::template eval<T, 1>(in, a, v);
      acc.template add<1>(v);
    }
    const S tot = consumer_reduce_sum<S>(acc.s, ws);
    if (threadIdx.x == 0) {
      if (d.nseg == 1) {
        store_dim_value<T>(d, j, tot);
      } else {
        reinterpret_cast<S*>(d.part)[p] = tot;
        __threadfence();
        const unsigned t = atomicAdd(&d.tickets[j], 1u);
        if (t == d.nseg - 1) {
          __threadfence();
          S sum = S(0);
          for (uint32_t q = 0; q < d.nseg; ++q)
            sum = sum_add<S>(sum, __ldcg(reinterpret_cast<const S*>(d.part) + j * d.nseg + q));
          store_dim_value<T>(d, j, sum);
          d.tickets[j] = 0u;
        }
      }
    }
  }
  }
  __syncthreads();  // the producer stays resident until every staged tile is consumed
}

// ---- dim 1 -------------------------------------------------------------------
template <class T, class EV>
__global__ void __launch_bounds__(kTmaThreads, tma_min_ctas<EV>()) dim1_tma_kernel(const __grid_constant__ DimArgs d) {
  pdl_wait();
  constexpr int W = Unit<T>::W;
  typedef typename SumT<T>::type S;
  constexpr u64 R = (u64)kConsumerWarps * 32 * W;  // rows per tile
  constexpr uint32_t seg_bytes = (uint32_t)(R * sizeof(T));
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ bool last;
  const FusedArgs& a = d.f;
  const uint32_t nk = EV::kInterp ? a.n_operands : (uint32_t)EV::K;
  const uint32_t NS = a.stages, CG = d.cg;
  const uint32_t stage_bytes = nk * CG * seg_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * stage_bytes);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const u64 npieces = (u64)d.nrt * d.nchunks;

  if (warp == kConsumerWarps) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t s = 0, ph = 0;
      u64 i = 0;
      for (u64 p = blockIdx.x; p < npieces; p += gridDim.x) {
        const u64 rt = p % d.nrt, cc = p / d.nrt;
        const u64 r0 = rt * R;
        const u64 nrows = (d.m - r0) < R ? (d.m - r0) : R;
        const u64 c0 = cc * d.ccols, c1 = (c0 + d.ccols < d.n) ? c0 + d.ccols : d.n;
        for (u64 j = c0; j < c1; j += CG, ++i) {
          const uint32_t ncg = (uint32_t)((c1 - j) < CG ? (c1 - j) : CG);
          if (i >= NS) mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], (uint32_t)(nk * ncg * nrows * sizeof(T)));
          for (uint32_t k = 0; k < nk; ++k)
            for (uint32_t c = 0; c < ncg; ++c)
              bulk_g2s(smem + (size_t)s * stage_bytes + ((size_t)k * CG + c) * seg_bytes,
                       reinterpret_cast<const char*>(a.in[k]) + ((j + c) * d.m + r0) * sizeof(T),
                       (uint32_t)(nrows * sizeof(T)), &full[s], pol);
          if (++s == NS) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else {
  uint32_t s = 0, ph = 0;
  const uint32_t t = threadIdx.x;
  for (u64 p = blockIdx.x; p < npieces; p += gridDim.x) {
    const u64 rt = p % d.nrt, cc = p / d.nrt;
    const u64 r0 = rt * R;
    const u64 nrows = (d.m - r0) < R ? (d.m - r0) : R;
    const u64 c0 = cc * d.ccols, c1 = (c0 + d.ccols < d.n) ? c0 + d.ccols : d.n;
    const bool valid = (u64)t * W < nrows;  // nrows is a multiple of W (vec path)
    S acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = S(0);
    for (u64 j = c0; j < c1; j += CG) {
      const uint32_t ncg = (uint32_t)((c1 - j) < CG ? (c1 - j) : CG);
      mbar_wait(&full[s], ph);
      if (valid) {
        const unsigned char* stg = smem + (size_t)s * stage_bytes + (size_t)t * 16;
        if (ncg == 4) {
          T v[4][W];
#pragma unroll
          for (int c = 0; c < 4; ++c)
            EV::template eval_src<T, W>(SmemSrc<T, 1>{stg + (size_t)c * seg_bytes, CG * seg_bytes},
                                        a, v[c]);
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
        } else {
          for (uint32_t c = 0; c < ncg; ++c) {
            T v[W];
            EV::template eval_src<T, W>(SmemSrc<T, 1>{stg + (size_t)c * seg_bytes, CG * seg_bytes},
                                        a, v);
#pragma unroll
            for (int w = 0; w < W; ++w) {
              T one[1] = {v[w]};
              acc[w] = sum_add<S>(acc[w], unit_sum<T, 1>(one));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
    }
    if (d.nchunks == 1) {
      if (valid) {
#pragma unroll
        for (int w = 0; w < W; ++w) store_dim_value<T>(d, r0 + (u64)t * W + w, acc[w]);
      }
      if (d.final_mode == FINAL_EXCHANGE)
        vec_exchange_arrive<T>(d, nrows, t, kConsumerWarps * 32, &last, consumer_sync);
      continue;
    }
    S* part = reinterpret_cast<S*>(d.part);
    if (valid) {
#pragma unroll
      for (int w = 0; w < W; ++w) part[cc * d.m + r0 + (u64)t * W + w] = acc[w];
    }
    __threadfence();
    consumer_sync();
    if (t == 0) last = (atomicAdd(&d.tickets[rt], 1u) == d.nchunks - 1);
    consumer_sync();
    if (last) {
      __threadfence();
      if (valid) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const u64 r = r0 + (u64)t * W + w;
          S tot = S(0);
          for (uint32_t c = 0; c < d.nchunks; ++c) tot = sum_add<S>(tot, __ldcg(part + (u64)c * d.m + r));
          store_dim_value<T>(d, r, tot);
        }
      }
      if (t == 0) d.tickets[rt] = 0u;
      if (d.final_mode == FINAL_EXCHANGE) {
        consumer_sync();  // every thread has read `last` before the arrive rewrites it
        vec_exchange_arrive<T>(d, nrows, t, kConsumerWarps * 32, &last, consumer_sync);
      }
    }
    consumer_sync();  // `last` is rewritten by the next piece
  }
  }
  __syncthreads();  // the producer stays resident until every staged tile is consumed
}

}  // namespace coot
