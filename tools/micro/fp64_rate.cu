// Non-tensor float64 throughput and latency on this GPU: independent DFMA chains per thread
// (throughput), one dependent chain per thread at one warp per SM sub-partition (latency),
// and the same for __dsqrt_rn / __ddiv_rn.   nvcc -arch=sm_100a -O3 fp64_rate.cu -o fp64_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP, int CHAINS>
__global__ void slow_kernel(double* out, int iters, double a) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = 1.0 + threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = OP == 0 ? __dsqrt_rn(x[c]) + a : __ddiv_rn(a, x[c]) + a;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
float time_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  const int iters = 20000;
  {
    float ms = time_ms([&] { dfma_kernel<8><<<sms * 8, 256>>>(out, iters, 1.0000001, 1e-9); });
    double fl = 2.0 * 8 * iters * (double)sms * 8 * 256;
    printf("DFMA throughput (8 chains, 8x256 threads/SM): %.2f TF/s = %.1f DFMA/clk/SM at %d MHz nominal\n",
           fl / ms / 1e9, fl / 2 / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
  }
  {
    float ms = time_ms([&] { dfma_kernel<1><<<sms, 128>>>(out, iters, 1.0000001, 1e-9); });
    printf("DFMA dependent latency (1 warp per sub-partition): %.1f clk\n", ms * 1e-3 * clk_khz * 1e3 / iters);
  }
  {
    float ms = time_ms([&] { dfma_kernel<1><<<sms * 4, 128>>>(out, iters, 1.0000001, 1e-9); });
    printf("DFMA dependent chain, 4 warps per sub-partition: %.1f clk per step\n", ms * 1e-3 * clk_khz * 1e3 / iters);
  }
  const int it2 = 2000;
  {
    float ms = time_ms([&] { slow_kernel<0, 4><<<sms * 8, 256>>>(out, it2, 1.5); });
    double ops = 4.0 * it2 * (double)sms * 8 * 256;
    printf("dsqrt_rn throughput: %.2f G/s = %.2f per clk per SM\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk_khz * 1e3));
    ms = time_ms([&] { slow_kernel<0, 1><<<sms, 128>>>(out, it2, 1.5); });
    printf("dsqrt_rn dependent latency: %.0f clk\n", ms * 1e-3 * clk_khz * 1e3 / it2);
  }
  {
    float ms = time_ms([&] { slow_kernel<1, 4><<<sms * 8, 256>>>(out, it2, 1.5); });
    double ops = 4.0 * it2 * (double)sms * 8 * 256;
    printf("ddiv_rn throughput: %.2f G/s = %.2f per clk per SM\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk_khz * 1e3));
    ms = time_ms([&] { slow_kernel<1, 1><<<sms, 128>>>(out, it2, 1.5); });
    printf("ddiv_rn dependent latency: %.0f clk\n", ms * 1e-3 * clk_khz * 1e3 / it2);
  }
  return 0;
}
