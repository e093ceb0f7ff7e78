// Shared helpers for the blockmm B200 kernels: error state, launch counting,
// int64 block reductions.  Every C-ABI entry point returns 0 or a negative
// BMM_E* code and records a message retrievable with bmm_last_error().
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <cuda_runtime.h>

#include "../../include/blockmm_b200.h"

namespace bmm {

void set_error(const char* fmt, ...);
void count_launch(int n = 1);

#define BMM_CHECK_LAUNCH(what)                                                        \
  do {                                                                                \
    cudaError_t _e = cudaGetLastError();                                              \
    if (_e != cudaSuccess) {                                                          \
      ::bmm::set_error("%s: launch failed: %s", what, cudaGetErrorString(_e));        \
      return BMM_E_CUDA;                                                              \
    }                                                                                 \
    ::bmm::count_launch();                                                            \
  } while (0)

#define BMM_REQUIRE(cond, code, ...)                                                  \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      ::bmm::set_error(__VA_ARGS__);                                                  \
      return code;                                                                    \
    }                                                                                 \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grid size for a grid-stride kernel: enough CTAs to cover `work` threads,
// capped at `waves` full waves of 148 SMs x `per_sm` resident CTAs.
inline unsigned grid_for(int64_t work, int threads, int per_sm = 8, int waves = 8) {
  int64_t g = ceil_div(work, threads);
  int64_t cap = 148LL * per_sm * waves;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// ---------------------------------------------------------------- device side

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_or(int v) { return __any_sync(0xffffffffu, v); }

// Block-wide int64 sum; `red` must hold >= 32 entries. All threads get the total.
__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  v = warp_sum_i64(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int64_t t = 0;
  for (int i = 0; i < nwarps; ++i) t += red[i];
  __syncthreads();
  return t;
}

}  // namespace bmm
