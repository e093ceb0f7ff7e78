// K1 -- the norm pass (bandwidth-bound, one read of M and N).
//
// Reference: column_norms / row_norms (pkg/src/blockmm/matrix.py:107-114),
// reached through _index_scores (plan.py:165-167) by every allocator.
//
// colsq: one thread owns VEC adjacent columns (one 16-byte load per row) and
//        walks the rows in order, so the float64 chain is exactly NumPy's
//        sequential add.reduce(M*M, axis=0).  R rows of loads are issued
//        before they are consumed, which keeps R*16 bytes in flight per thread.
// rowsq: one thread owns one row of N and evaluates NumPy's pairwise tree with
//        8-wide vector steps (leaf starts are multiples of 8, so a leaf streams
//        32/64-byte aligned vectors).
#include "common.cuh"
#include "pairwise.cuh"

namespace bmm {

template <typename T> struct Vec16;
template <> struct Vec16<double> { using V = double2; static constexpr int N = 2; };
template <> struct Vec16<float> { using V = float4; static constexpr int N = 4; };

__device__ __forceinline__ void unpack(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
__device__ __forceinline__ void unpack(const float4& v, double* o) {
  o[0] = (double)v.x; o[1] = (double)v.y; o[2] = (double)v.z; o[3] = (double)v.w;
}

template <typename T, int R>
__global__ void __launch_bounds__(256) colsq_vec_kernel(const T* __restrict__ M, int64_t m, int64_t n,
                                                        int64_t ldm, int64_t strideM, int64_t batch,
                                                        int accumulate, double* __restrict__ colsq) {
  using V = typename Vec16<T>::V;
  constexpr int W = Vec16<T>::N;
  const int64_t groups = n / W;
  const int64_t total = groups * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / groups, c0 = (g - b * groups) * W;
    const T* base = M + b * strideM + c0;
    double* out = colsq + b * n + c0;
    double acc[W];
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] = accumulate ? out[j] : 0.0;
    int64_t h = 0;
    for (; h + R <= m; h += R) {
      V v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = __ldcs(reinterpret_cast<const V*>(base + (h + r) * ldm));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double x[W];
        unpack(v[r], x);
#pragma unroll
        for (int j = 0; j < W; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(x[j], x[j]));
      }
    }
    for (; h < m; ++h) {
      V v = __ldcs(reinterpret_cast<const V*>(base + h * ldm));
      double x[W];
      unpack(v, x);
#pragma unroll
      for (int j = 0; j < W; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(x[j], x[j]));
    }
#pragma unroll
    for (int j = 0; j < W; ++j) out[j] = acc[j];
  }
}

// Scalar path: unaligned layouts and the n % W tail columns [c_begin, n).
template <typename T, int R>
__global__ void __launch_bounds__(256) colsq_scalar_kernel(const T* __restrict__ M, int64_t m, int64_t n,
                                                           int64_t c_begin, int64_t ldm, int64_t strideM,
                                                           int64_t batch, int accumulate,
                                                           double* __restrict__ colsq) {
  const int64_t cols = n - c_begin;
  const int64_t total = cols * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / cols, c = c_begin + (g - b * cols);
    const T* base = M + b * strideM + c;
    double acc = accumulate ? colsq[b * n + c] : 0.0;
    int64_t h = 0;
    for (; h + R <= m; h += R) {
      double v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = (double)base[(h + r) * ldm];
#pragma unroll
      for (int r = 0; r < R; ++r) acc = __dadd_rn(acc, __dmul_rn(v[r], v[r]));
    }
    for (; h < m; ++h) { double x = (double)base[h * ldm]; acc = __dadd_rn(acc, __dmul_rn(x, x)); }
    colsq[b * n + c] = acc;
  }
}

template <typename T>
__global__ void __launch_bounds__(128) rowsq_kernel(const T* __restrict__ N, int64_t n, int64_t p,
                                                    int64_t ldn, int64_t strideN, int64_t batch,
                                                    double* __restrict__ rowsq) {
  const int64_t total = n * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / n, i = g - b * n;
    const T* row = N + b * strideN + i * ldn;
    SrcSq<T> src{row, (reinterpret_cast<uintptr_t>(row) & 15) == 0};
    // NumPy: add.reduce starts from the identity 0 and adds the pairwise sum.
    rowsq[g] = __dadd_rn(0.0, pw_sum(src, 0, p));
  }
}

// Few, wide rows: one warp per row (warp_pw_sum), so a row's loads are all in
// flight at once; same tree, same bits as rowsq_kernel.
constexpr int kRowWarps = 8;

template <typename T>
__global__ void __launch_bounds__(32 * kRowWarps) rowsq_warp_kernel(const T* __restrict__ N, int64_t n,
                                                                    int64_t p, int64_t ldn, int64_t strideN,
                                                                    int64_t batch, double* __restrict__ rowsq) {
  __shared__ WarpPwScratch scratch[kRowWarps];
  WarpPwScratch* scr = &scratch[threadIdx.x >> 5];
  const int64_t total = n * batch;
  for (int64_t g = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5); g < total;
       g += (int64_t)gridDim.x * kRowWarps) {
    const int64_t b = g / n, i = g - b * n;
    const T* row = N + b * strideN + i * ldn;
    SrcSq<T> src{row, false};
    const double v = __dadd_rn(0.0, warp_pw_sum(src, 0, p, scr));
    if ((threadIdx.x & 31) == 0) rowsq[g] = v;
  }
}

template <typename T>
int launch_norms(const T* M, int64_t m, int64_t n, int64_t ldm, int64_t strideM, const T* N,
                 int64_t p, int64_t ldn, int64_t strideN, int64_t batch, int accumulate,
                 double* colsq, double* rowsq, cudaStream_t st) {
  constexpr int W = Vec16<T>::N;
  if (M != nullptr) {
    BMM_REQUIRE(colsq != nullptr, BMM_E_ARG, "bmm_norms: colsq is NULL");
    // Few columns (e.g. config 2: 20000): one column per thread in 64-thread CTAs
    // spreads the chains over every SM and keeps 32 row loads in flight each.
    const bool narrow = (n / W) * batch < 148LL * 256;
    const bool vec_ok = !narrow && (reinterpret_cast<uintptr_t>(M) % 16 == 0) && (ldm % W == 0) &&
                        (strideM % W == 0) && n >= W;
    int64_t c_tail = 0;
    if (vec_ok) {
      const int64_t groups = n / W;
      c_tail = groups * W;
      colsq_vec_kernel<T, 16><<<grid_for(groups * batch, 256, 8, 64), 256, 0, st>>>(
          M, m, n, ldm, strideM, batch, accumulate, colsq);
      BMM_CHECK_LAUNCH("colsq_vec_kernel");
    }
    if (c_tail < n) {
      if (narrow) {
        colsq_scalar_kernel<T, 32><<<grid_for((n - c_tail) * batch, 64, 32, 64), 64, 0, st>>>(
            M, m, n, c_tail, ldm, strideM, batch, accumulate, colsq);
      } else {
        colsq_scalar_kernel<T, 16><<<grid_for((n - c_tail) * batch, 256, 8, 64), 256, 0, st>>>(
            M, m, n, c_tail, ldm, strideM, batch, accumulate, colsq);
      }
      BMM_CHECK_LAUNCH("colsq_scalar_kernel");
    }
  }
  if (N != nullptr) {
    BMM_REQUIRE(rowsq != nullptr, BMM_E_ARG, "bmm_norms: rowsq is NULL");
    const int64_t rows = n * batch;
    if (rows < 148LL * 512 && p > 128) {
      const int64_t blocks = std::min<int64_t>(ceil_div(rows, kRowWarps), 148LL * 8 * 64);
      rowsq_warp_kernel<T><<<(unsigned)blocks, 32 * kRowWarps, 0, st>>>(N, n, p, ldn, strideN, batch, rowsq);
      BMM_CHECK_LAUNCH("rowsq_warp_kernel");
    } else {
      rowsq_kernel<T><<<grid_for(rows, 128, 16, 64), 128, 0, st>>>(N, n, p, ldn, strideN, batch, rowsq);
      BMM_CHECK_LAUNCH("rowsq_kernel");
    }
  }
  return BMM_OK;
}

}  // namespace bmm

extern "C" int bmm_norms(int dtype, const void* M, int64_t m, int64_t n, int64_t ldm,
                         int64_t strideM, const void* N, int64_t p, int64_t ldn, int64_t strideN,
                         int64_t batch, int accumulate, double* colsq, double* rowsq,
                         void* stream) {
  using namespace bmm;
  BMM_REQUIRE(m >= 0 && n >= 0 && p >= 0 && batch >= 1, BMM_E_ARG, "bmm_norms: bad shape");
  if (n == 0) return BMM_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == BMM_F64)
    return launch_norms<double>((const double*)M, m, n, ldm, strideM, (const double*)N, p, ldn,
                                strideN, batch, accumulate, colsq, rowsq, st);
  if (dtype == BMM_F32)
    return launch_norms<float>((const float*)M, m, n, ldm, strideM, (const float*)N, p, ldn,
                               strideN, batch, accumulate, colsq, rowsq, st);
  set_error("bmm_norms: unknown dtype %d", dtype);
  return BMM_E_ARG;
}
