// K7'' -- segmented square sums of a sketch with few columns per segment, by Gram matrices.
//
//   gsq[b, j] = || C_j D_j ||_F^2 = sum_{a, a'} (C_j^T C_j)[a, a'] (D_j D_j^T)[a, a']
//
// for the sketch C = M[:, column] * scale, D = N[column, :] * scale and segment
// j = sketch positions [seg[j], seg[j+1]).  The two-step pilot norms
// ||C0_k D0_k||_F^2 (plan.py:457-464) contract c0/K pilot draws per block
// (config 3: 5): the explicit product costs 2 m p L flops per segment, the two
// L x L Gram matrices 2 (m + p) L^2 / 2 -- 100x fewer at L = 5, m = p = 1000,
// and the work becomes two streaming passes over the gathered columns.
//
// CTA per (segment, problem).  Pairs (a, a') are handled in 8 x 8 tiles (a
// tile pair at a time, 64 accumulators per thread); the C side walks the m
// rows, the D side the p columns (coalesced rows of N); partial sums are
// reduced across the CTA in a fixed order (deterministic).  Float64 with FMA:
// the reference's value comes from BLAS in its own order, so parity is to
// rounding (~1e-15 relative), as for the DMMA kernel it replaces.
#include "common.cuh"

namespace bmm {

constexpr int GR_T = 8;         // Gram tile (sketch positions)
constexpr int GR_THREADS = 256;

template <typename T>
__device__ __forceinline__ double gr_ld(const T* p) { return (double)__ldg(p); }

// CTA-wide fixed-order sum of acc[0..63] into out[0..63] (thread 0 holds the result in shared memory)
__device__ __forceinline__ void gr_reduce64(double (&acc)[GR_T * GR_T], double* red /* [8 warps][64] */,
                                            double* out /* [64] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < GR_T * GR_T; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp * GR_T * GR_T + q] = v;
  }
  __syncthreads();
  if (threadIdx.x < GR_T * GR_T) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < GR_THREADS / 32; ++w) v += red[w * GR_T * GR_T + threadIdx.x];
    out[threadIdx.x] = v;
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(GR_THREADS) segsq_gram_kernel(const T* __restrict__ M, int64_t ldm, int64_t strideM,
                                                                const T* __restrict__ N, int64_t ldn, int64_t strideN,
                                                                int64_t m, int64_t p,
                                                                const int64_t* __restrict__ column,
                                                                const double* __restrict__ scale, int64_t w_stride,
                                                                const int64_t* __restrict__ seg, int64_t nseg,
                                                                int64_t seg_stride, double* __restrict__ gsq) {
  __shared__ double red[(GR_THREADS / 32) * GR_T * GR_T];
  __shared__ double gc[GR_T * GR_T], gd[GR_T * GR_T];
  __shared__ int64_t cols[2][GR_T];
  __shared__ double scs[2][GR_T];
  __shared__ int nv[2];
  const int64_t j = blockIdx.x, b = blockIdx.y;
  const int64_t s0 = seg[b * seg_stride + j], L = seg[b * seg_stride + j + 1] - s0;
  const T* Mb = M + b * strideM;
  const T* Nb = N + b * strideN;
  const int64_t* colb = column + b * w_stride + s0;
  const double* scb = scale + b * w_stride + s0;
  const int nt = (int)((L + GR_T - 1) / GR_T);
  double total = 0.0;  // thread 0
  for (int ta = 0; ta < nt; ++ta) {
    for (int tb = ta; tb < nt; ++tb) {
      if (threadIdx.x < 2 * GR_T) {
        const int side = threadIdx.x / GR_T, a = threadIdx.x % GR_T;
        const int64_t pos = (int64_t)(side == 0 ? ta : tb) * GR_T + a;
        cols[side][a] = pos < L ? colb[pos] : 0;
        scs[side][a] = pos < L ? scb[pos] : 0.0;  // zero scale: the padding contributes nothing
        if (a == 0) nv[side] = (int)min((int64_t)GR_T, L - (int64_t)(side == 0 ? ta : tb) * GR_T);
      }
      __syncthreads();
      double acc[GR_T * GR_T];
      // C side: (C^T C)[a, a'] = sum_h C[h, a] C[h, a']
#pragma unroll
      for (int q = 0; q < GR_T * GR_T; ++q) acc[q] = 0.0;
      for (int64_t h = threadIdx.x; h < m; h += GR_THREADS) {
        const T* row = Mb + h * ldm;
        double va[GR_T], vb[GR_T];
#pragma unroll
        for (int a = 0; a < GR_T; ++a) va[a] = a < nv[0] ? __dmul_rn(gr_ld(row + cols[0][a]), scs[0][a]) : 0.0;
#pragma unroll
        for (int a = 0; a < GR_T; ++a) vb[a] = a < nv[1] ? __dmul_rn(gr_ld(row + cols[1][a]), scs[1][a]) : 0.0;
#pragma unroll
        for (int a = 0; a < GR_T; ++a)
#pragma unroll
          for (int c = 0; c < GR_T; ++c) acc[a * GR_T + c] = fma(va[a], vb[c], acc[a * GR_T + c]);
      }
      gr_reduce64(acc, red, gc);
      // D side: (D D^T)[a, a'] = sum_f D[a, f] D[a', f]
#pragma unroll
      for (int q = 0; q < GR_T * GR_T; ++q) acc[q] = 0.0;
      for (int64_t f = threadIdx.x; f < p; f += GR_THREADS) {
        double va[GR_T], vb[GR_T];
#pragma unroll
        for (int a = 0; a < GR_T; ++a) va[a] = a < nv[0] ? __dmul_rn(gr_ld(Nb + cols[0][a] * ldn + f), scs[0][a]) : 0.0;
#pragma unroll
        for (int a = 0; a < GR_T; ++a) vb[a] = a < nv[1] ? __dmul_rn(gr_ld(Nb + cols[1][a] * ldn + f), scs[1][a]) : 0.0;
#pragma unroll
        for (int a = 0; a < GR_T; ++a)
#pragma unroll
          for (int c = 0; c < GR_T; ++c) acc[a * GR_T + c] = fma(va[a], vb[c], acc[a * GR_T + c]);
      }
      gr_reduce64(acc, red, gd);
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < GR_T * GR_T; ++q) t = fma(gc[q], gd[q], t);
        total += (ta == tb) ? t : 2.0 * t;  // the (tb, ta) block is the transpose: same contribution
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) gsq[b * nseg + j] = total;
}

}  // namespace bmm

using namespace bmm;

extern "C" int bmm_segsq_gram_gather(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                     int64_t ldn, int64_t strideN, int64_t m, int64_t nc, const int64_t* column,
                                     const double* scale, int64_t w_stride, const int64_t* seg, int64_t nseg,
                                     int64_t seg_stride, int64_t batch, double* gsq, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && nseg >= 1 && batch >= 1, BMM_E_ARG, "bmm_segsq_gram_gather: bad shape");
  BMM_REQUIRE(M != nullptr && N != nullptr && column != nullptr && scale != nullptr && seg != nullptr &&
                  gsq != nullptr,
              BMM_E_ARG, "bmm_segsq_gram_gather: null pointer");
  BMM_REQUIRE(nseg < (1LL << 31) && batch <= 65535, BMM_E_UNSUPPORTED, "bmm_segsq_gram_gather: grid too large");
  dim3 grid((unsigned)nseg, (unsigned)batch);
  cudaStream_t st = as_stream(stream);
  if (dtype == BMM_F64) {
    segsq_gram_kernel<double><<<grid, GR_THREADS, 0, st>>>((const double*)M, ldm, strideM, (const double*)N, ldn,
                                                           strideN, m, nc, column, scale, w_stride, seg, nseg,
                                                           seg_stride, gsq);
  } else if (dtype == BMM_F32) {
    segsq_gram_kernel<float><<<grid, GR_THREADS, 0, st>>>((const float*)M, ldm, strideM, (const float*)N, ldn,
                                                          strideN, m, nc, column, scale, w_stride, seg, nseg,
                                                          seg_stride, gsq);
  } else {
    set_error("bmm_segsq_gram_gather: unknown dtype %d", dtype);
    return BMM_E_ARG;
  }
  BMM_CHECK_LAUNCH("segsq_gram_kernel");
  return BMM_OK;
}
