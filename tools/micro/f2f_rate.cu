// Throughput of F2F.F64.F32 (float -> double conversion) against an integer-built widening, and
// of the norm chain step acc = fma(x, x, acc) with each: the config-4 column sums convert every
// element once.   nvcc -arch=sm_100a -O3 f2f_rate.cu -o f2f_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// exact float -> double for finite normal inputs and zero by integer ops; denormals, inf and
// nan (rare) through the conversion unit
__device__ __forceinline__ double widen_int(float x) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t a = u & 0x7fffffffu;
  if (a - 0x00800000u >= 0x7f000000u && a != 0u) return (double)x;  // denormal, inf, nan
  const uint32_t hi = (u & 0x80000000u) | ((a >> 3) + (a ? 0x38000000u : 0u));
  const uint32_t lo = u << 29;
  return __hiloint2double((int)hi, (int)lo);
}

template <int MODE>
__global__ void chain_kernel(const float* __restrict__ in, double* out, int iters) {
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = 0.0;
  float x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = in[(threadIdx.x + c * 32) & 1023];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double d = MODE == 0 ? (double)x[c] : widen_int(x[c]);
      acc[c] = fma(d, d, acc[c]);
      x[c] = __uint_as_float(__float_as_uint(x[c]) + 3u);  // a new value every step: the conversion stays in the loop
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount;
  float* in;
  double* out;
  cudaMalloc(&in, 4096);
  cudaMemset(in, 0x3f, 4096);
  cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  const int iters = 20000;
  for (int mode = 0; mode < 2; ++mode) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) chain_kernel<0><<<sms * 8, 256>>>(in, out, iters);
      else chain_kernel<1><<<sms * 8, 256>>>(in, out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double el = 8.0 * iters * (double)sms * 8 * 256;
    printf("%s: %.1f G elements/s = %.1f per clk per SM (nominal %d MHz)\n",
           mode == 0 ? "F2F.F64.F32 + DFMA" : "integer widening + DFMA", el / ms / 1e6,
           el / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
  }
  return 0;
}
