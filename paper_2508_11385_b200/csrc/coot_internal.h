// Internal interface between the host runtime (runtime.cu) and the per-type
// kernel translation units (kernels_<type>.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace coot {

struct FusedArgs;
struct DimArgs;
struct Exchange;

struct FusedPlan {
  int catalog;       // >= 0 catalog id, -1 interpreter
  int interp_large;  // interpreter size class: 0 = <=4 operands / depth 4, 1 = <=8 / 8
  int acc;           // AccKind
  unsigned grid;
  int driver;        // 0 = register-pipelined LDG driver, 1 = TMA-staged driver
  unsigned smem;     // dynamic shared memory (TMA driver)
  int pdl = 1;       // launch as a programmatic dependent of the previous kernel
};

enum DimKernel {
  DIMK_DIM0_BLOCK = 0, DIMK_DIM0_WARP = 1, DIMK_DIM1 = 2,  // LDG kernels
  DIMK_DIM0_TMA = 3, DIMK_DIM1_TMA = 4,                    // TMA-staged kernels
  DIMK_STRIDED = 5                                         // strided views
};

struct DimPlan {
  int kernel;        // DimKernel
  int catalog;       // 0 = plain [L0] matrix, -1 interpreter
  int interp_large;
  unsigned grid;
  unsigned smem;     // dynamic shared memory (TMA kernels)
  int pdl = 1;       // launch as a programmatic dependent of the previous kernel
};

template <class T>
cudaError_t launch_fused_t(const FusedPlan& p, const FusedArgs& a, cudaStream_t s);
template <class T>
cudaError_t launch_dim_t(const DimPlan& p, const DimArgs& a, cudaStream_t s);
template <class T>
cudaError_t launch_combine_t(uint32_t kind, int acc, const void* parts, uint32_t nparts,
                             unsigned long long len, void* result, unsigned grid, cudaStream_t s);
// identity record of an empty shard into `out`; with ex != nullptr the record
// is exchanged instead and `out` receives the combined result
template <class T>
cudaError_t launch_empty_rec_t(int acc, void* out, cudaStream_t s, const Exchange* ex,
                               uint32_t kind);
template <class T>
cudaError_t launch_fill_t(uint32_t kind, unsigned long long seed, unsigned long long stream,
                          unsigned long long start, unsigned long long count,
                          unsigned long long n_rows, unsigned long long k, void* out,
                          unsigned grid, cudaStream_t s);

// stream microbenchmark (coot_stream.cu): units of 16 bytes (4 x f32)
cudaError_t launch_stream_mix(uint32_t n_read, uint32_t n_write, unsigned long long units,
                              const void* const* in, void* out, void* sink, int sm_count,
                              cudaStream_t s);

}  // namespace coot
