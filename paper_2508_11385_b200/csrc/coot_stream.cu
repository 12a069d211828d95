// Stream microbenchmark kernels: the achievable HBM bandwidth for each
// read:write mix (SURVEY §8(d) "Same-run stream microbenchmarks"), measured in
// the same process as the fused kernels so that every config's roofline
// fraction is taken against the mix it actually streams (1R: accu / norm2 /
// dim sums; 2R: dot; 3R: c2 / c4 reduce-only; 1R1W copy; 2R1W axpy; 3R1W c2
// with Z stored).  Trivial by design: out[i] = sum_k in_k[i] over f32 in
// 16-byte units, 4 units in flight per thread per array, grid = SMs x 8 CTAs of
// 256 threads (grid-stride); read-only mixes fold into one value per thread
// written to `sink` so the loads are live.
#include <cuda_runtime.h>
#include <stdint.h>

#include "coot_internal.h"

namespace coot {
namespace {

constexpr int kStreamThreads = 256;
constexpr int kStreamUnroll = 4;

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w));
}

template <int R, int W>
__global__ void __launch_bounds__(kStreamThreads) stream_mix_kernel(
    const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
    float4* __restrict__ o, unsigned long long units, float* sink) {
  const unsigned long long stride = (unsigned long long)gridDim.x * kStreamThreads;
  unsigned long long i = (unsigned long long)blockIdx.x * kStreamThreads + threadIdx.x;
  float acc = 0.f;
  for (; i + (kStreamUnroll - 1) * stride < units; i += kStreamUnroll * stride) {
    float4 v[kStreamUnroll];
#pragma unroll
    for (int u = 0; u < kStreamUnroll; ++u) {
      const unsigned long long e = i + u * stride;
      v[u] = R >= 1 ? ld_stream(a + e) : make_float4(1.f, 1.f, 1.f, 1.f);
      if (R >= 2) {
        const float4 t = ld_stream(b + e);
        v[u].x += t.x; v[u].y += t.y; v[u].z += t.z; v[u].w += t.w;
      }
      if (R >= 3) {
        const float4 t = ld_stream(c + e);
        v[u].x += t.x; v[u].y += t.y; v[u].z += t.z; v[u].w += t.w;
      }
    }
#pragma unroll
    for (int u = 0; u < kStreamUnroll; ++u) {
      if (W) st_stream(o + i + u * stride, v[u]);
      else acc += (v[u].x + v[u].y) + (v[u].z + v[u].w);
    }
  }
  for (; i < units; i += stride) {
    float4 v = R >= 1 ? ld_stream(a + i) : make_float4(1.f, 1.f, 1.f, 1.f);
    if (R >= 2) { const float4 t = ld_stream(b + i); v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w; }
    if (R >= 3) { const float4 t = ld_stream(c + i); v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w; }
    if (W) st_stream(o + i, v);
    else acc += (v.x + v.y) + (v.z + v.w);
  }
  if (!W && acc == 1.2345e-38f) *sink = acc;  // keeps the loads live; practically never taken
}

}  // namespace

cudaError_t launch_stream_mix(uint32_t n_read, uint32_t n_write, unsigned long long units,
                              const void* const* in, void* out, void* sink, int sm_count,
                              cudaStream_t s) {
  const unsigned long long want = (units + kStreamThreads * kStreamUnroll - 1) /
                                  (kStreamThreads * kStreamUnroll);
  const unsigned grid = (unsigned)(want < (unsigned long long)sm_count * 8 ? (want ? want : 1)
                                                                          : (unsigned long long)sm_count * 8);
  const float4* a = n_read >= 1 ? static_cast<const float4*>(in[0]) : nullptr;
  const float4* b = n_read >= 2 ? static_cast<const float4*>(in[1]) : nullptr;
  const float4* c = n_read >= 3 ? static_cast<const float4*>(in[2]) : nullptr;
  float4* o = static_cast<float4*>(out);
  float* k = static_cast<float*>(sink);
#define COOT_MIX(R, W) \
  if (n_read == R && n_write == W) stream_mix_kernel<R, W><<<grid, kStreamThreads, 0, s>>>(a, b, c, o, units, k);
  COOT_MIX(1, 0) else COOT_MIX(2, 0) else COOT_MIX(3, 0) else COOT_MIX(0, 1) else COOT_MIX(1, 1)
  else COOT_MIX(2, 1) else COOT_MIX(3, 1) else return cudaErrorInvalidValue;
#undef COOT_MIX
  return cudaGetLastError();
}

}  // namespace coot
