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
// tile pair at a time: 36 accumulators per thread on the diagonal, where the
// tile is symmetric, 64 off it); the C side walks the m rows, the D side the p
// columns (coalesced rows of N); partial sums are reduced across the CTA
// through shared memory in a fixed order (deterministic).  Float64 with FMA:
// the reference's value comes from BLAS in its own order, so parity is to
// rounding (~1e-15 relative), as for the DMMA kernel it replaces.
#include "common.cuh"

namespace bmm {

constexpr int GR_T = 8;         // Gram tile (sketch positions)
constexpr int GR_THREADS = 128;
constexpr int GR_NDIAG = GR_T * (GR_T + 1) / 2;

template <typename T>
__device__ __forceinline__ double gr_ld(const T* p) { return (double)__ldg(p); }

// CTA-wide fixed-order sums of acc[0..NA), 32 at a time: each thread stores its
// partials in a column of red[32][GR_THREADS + 1], thread q < 32 adds row q in
// index order (four fixed interleaved chains).
constexpr int GR_RED = 32;
template <int NA>
__device__ __forceinline__ void gr_reduce(const double (&acc)[NA], double* red, double* out) {
#pragma unroll
  for (int q0 = 0; q0 < NA; q0 += GR_RED) {
#pragma unroll
    for (int q = 0; q < GR_RED; ++q)
      if (q0 + q < NA) red[q * (GR_THREADS + 1) + threadIdx.x] = acc[q0 + q];
    __syncthreads();
    if (threadIdx.x < GR_RED && q0 + (int)threadIdx.x < NA) {
      const double* r = red + threadIdx.x * (GR_THREADS + 1);
      double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
      for (int i = 0; i < GR_THREADS; i += 4) {
        v0 += r[i];
        v1 += r[i + 1];
        v2 += r[i + 2];
        v3 += r[i + 3];
      }
      out[q0 + threadIdx.x] = (v0 + v1) + (v2 + v3);
    }
    __syncthreads();
  }
}

// One side's Gram tile: sum over `len` positions x of u_a(x) v_c(x), where
// u_a(x) = src[x, cols0[a]] * sc0[a] (C side: x = row h of M, value at column col)
// or src[cols0[a], x] * sc0[a] (D side: x = column f of N).  DIAG: the tile is
// symmetric (same positions), only a <= c is accumulated.
template <typename T, bool DIAG, bool CSIDE>
__device__ __forceinline__ void gr_tile(const T* __restrict__ base, int64_t ld, int64_t len, const int64_t* cols0,
                                        const double* sc0, int n0, const int64_t* cols1, const double* sc1, int n1,
                                        double* red, double* out) {
  constexpr int NA = DIAG ? GR_NDIAG : GR_T * GR_T;
  double acc[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) acc[q] = 0.0;
#pragma unroll 2
  for (int64_t x = threadIdx.x; x < len; x += GR_THREADS) {
    double va[GR_T], vb[GR_T];
#pragma unroll
    for (int a = 0; a < GR_T; ++a) {
      const T* ptr = CSIDE ? base + x * ld + cols0[a] : base + cols0[a] * ld + x;
      va[a] = a < n0 ? __dmul_rn(gr_ld(ptr), sc0[a]) : 0.0;
    }
    if constexpr (!DIAG) {
#pragma unroll
      for (int a = 0; a < GR_T; ++a) {
        const T* ptr = CSIDE ? base + x * ld + cols1[a] : base + cols1[a] * ld + x;
        vb[a] = a < n1 ? __dmul_rn(gr_ld(ptr), sc1[a]) : 0.0;
      }
    }
    int q = 0;
#pragma unroll
    for (int a = 0; a < GR_T; ++a)
#pragma unroll
      for (int c = DIAG ? a : 0; c < GR_T; ++c, ++q) acc[q] = fma(va[a], DIAG ? va[c] : vb[c], acc[q]);
  }
  gr_reduce<NA>(acc, red, out);
}

// SINGLE: every segment has at most GR_T positions -- one symmetric tile, 36
// accumulators (fewer registers, more CTAs per SM)
template <typename T, bool SINGLE>
__global__ void __launch_bounds__(GR_THREADS) segsq_gram_kernel(const T* __restrict__ M, int64_t ldm, int64_t strideM,
                                                                const T* __restrict__ N, int64_t ldn, int64_t strideN,
                                                                int64_t m, int64_t p,
                                                                const int64_t* __restrict__ column,
                                                                const double* __restrict__ scale, int64_t w_stride,
                                                                const int64_t* __restrict__ seg, int64_t nseg,
                                                                int64_t seg_stride, double* __restrict__ gsq) {
  __shared__ double red[GR_RED * (GR_THREADS + 1)];
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
  const int nt = SINGLE ? (L > 0 ? 1 : 0) : (int)((L + GR_T - 1) / GR_T);
  double total = 0.0;  // thread 0
  for (int ta = 0; ta < nt; ++ta) {
    for (int tb = ta; tb < nt; ++tb) {
      if (threadIdx.x < 2 * GR_T) {
        const int side = threadIdx.x / GR_T, a = threadIdx.x % GR_T;
        const int64_t pos = (int64_t)(side == 0 ? ta : tb) * GR_T + a;
        cols[side][a] = pos < L ? colb[pos] : 0;
        scs[side][a] = pos < L ? scb[pos] : 0.0;
        if (a == 0) nv[side] = (int)min((int64_t)GR_T, L - (int64_t)(side == 0 ? ta : tb) * GR_T);
      }
      __syncthreads();
      double t = 0.0;
      if (SINGLE || ta == tb) {
        gr_tile<T, true, true>(Mb, ldm, m, cols[0], scs[0], nv[0], cols[0], scs[0], nv[0], red, gc);
        gr_tile<T, true, false>(Nb, ldn, p, cols[0], scs[0], nv[0], cols[0], scs[0], nv[0], red, gd);
        if (threadIdx.x == 0) {
          int q = 0;
          for (int a = 0; a < GR_T; ++a)
            for (int c = a; c < GR_T; ++c, ++q) t = fma(a == c ? gc[q] : 2.0 * gc[q], gd[q], t);
        }
      } else if constexpr (!SINGLE) {
        gr_tile<T, false, true>(Mb, ldm, m, cols[0], scs[0], nv[0], cols[1], scs[1], nv[1], red, gc);
        gr_tile<T, false, false>(Nb, ldn, p, cols[0], scs[0], nv[0], cols[1], scs[1], nv[1], red, gd);
        if (threadIdx.x == 0) {
          for (int q = 0; q < GR_T * GR_T; ++q) t = fma(gc[q], gd[q], t);
          t *= 2.0;  // the (tb, ta) block is the transpose: same contribution
        }
      }
      if (threadIdx.x == 0) total += t;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) gsq[b * nseg + j] = total;
}

}  // namespace bmm

using namespace bmm;

template <typename T>
static void gram_launch(dim3 grid, cudaStream_t st, bool single, const T* M, int64_t ldm, int64_t strideM, const T* N,
                        int64_t ldn, int64_t strideN, int64_t m, int64_t nc, const int64_t* column,
                        const double* scale, int64_t w_stride, const int64_t* seg, int64_t nseg, int64_t seg_stride,
                        double* gsq) {
  if (single)
    segsq_gram_kernel<T, true><<<grid, GR_THREADS, 0, st>>>(M, ldm, strideM, N, ldn, strideN, m, nc, column, scale,
                                                            w_stride, seg, nseg, seg_stride, gsq);
  else
    segsq_gram_kernel<T, false><<<grid, GR_THREADS, 0, st>>>(M, ldm, strideM, N, ldn, strideN, m, nc, column, scale,
                                                             w_stride, seg, nseg, seg_stride, gsq);
}

extern "C" int bmm_segsq_gram_gather(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                     int64_t ldn, int64_t strideN, int64_t m, int64_t nc, const int64_t* column,
                                     const double* scale, int64_t w_stride, const int64_t* seg, int64_t nseg,
                                     int64_t seg_stride, int64_t max_len, int64_t batch, double* gsq, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && nseg >= 1 && batch >= 1 && max_len >= 0, BMM_E_ARG,
              "bmm_segsq_gram_gather: bad shape");
  BMM_REQUIRE(M != nullptr && N != nullptr && column != nullptr && scale != nullptr && seg != nullptr &&
                  gsq != nullptr,
              BMM_E_ARG, "bmm_segsq_gram_gather: null pointer");
  BMM_REQUIRE(nseg < (1LL << 31) && batch <= 65535, BMM_E_UNSUPPORTED, "bmm_segsq_gram_gather: grid too large");
  dim3 grid((unsigned)nseg, (unsigned)batch);
  cudaStream_t st = as_stream(stream);
  const bool single = max_len <= GR_T;
  if (dtype == BMM_F64) {
    gram_launch<double>(grid, st, single, (const double*)M, ldm, strideM, (const double*)N, ldn, strideN, m, nc,
                        column, scale, w_stride, seg, nseg, seg_stride, gsq);
  } else if (dtype == BMM_F32) {
    gram_launch<float>(grid, st, single, (const float*)M, ldm, strideM, (const float*)N, ldn, strideN, m, nc, column,
                       scale, w_stride, seg, nseg, seg_stride, gsq);
  } else {
    set_error("bmm_segsq_gram_gather: unknown dtype %d", dtype);
    return BMM_E_ARG;
  }
  BMM_CHECK_LAUNCH("segsq_gram_kernel");
  return BMM_OK;
}
