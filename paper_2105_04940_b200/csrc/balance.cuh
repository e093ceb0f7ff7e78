// Balanced exponents and the problem's shift for the fp16 split (K6): shared by
// f16_balance_kernel (gemm_tf32.cu) and the fused small-problem plan (plan.cu).
#pragma once
#include <cstdint>

namespace bmm {

// kexp[t] = round(log2(||N_i|| / ||M_i||) / 2) (i = column[t]), *gshift such that every
// scaled operand |C[h,t]| 2^(kexp - G), |D[t,f]| 2^(-kexp - G) < 2^15 -- bounded by
// the column / row norms from the norm pass times the sketch scale.  One CTA per
// problem (at most 1024 threads); all pointers are the problem's own.
__device__ __forceinline__ void f16_balance_body(const double* __restrict__ colsq, const double* __restrict__ rowsq,
                                                 const int64_t* column, const double* scale, int64_t w, int64_t kd,
                                                 int32_t* kexp, int32_t* gshift) {
  __shared__ int red[32];
  int emax = -100000;
#pragma unroll 4
  for (int64_t t = threadIdx.x; t < w; t += blockDim.x) {
    int32_t e = 0;
    if (t < kd) {
      const int64_t i = column[t];
      const double c = colsq[i], r = rowsq[i], sc = fabs(scale[t]);
      if (c > 0.0 && r > 0.0 && sc > 0.0 && c < 1e300 && r < 1e300 && sc < 1e300) {
        const int d = ilogb(r) - ilogb(c);
        e = (int32_t)((d >= 0 ? d + 2 : d - 2) / 4);
        e = max(-60, min(60, e));
        const double bc = ldexp(sqrt(c) * sc, e), bd = ldexp(sqrt(r) * sc, -e);
        emax = max(emax, ilogb(fmax(bc, bd)) + 1);
      }
    }
    kexp[t] = e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    int v = red[0];
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j) v = max(v, red[j]);
    *gshift = v <= -100000 ? 0 : max(-60, min(60, v - 15));
  }
}

}  // namespace bmm
