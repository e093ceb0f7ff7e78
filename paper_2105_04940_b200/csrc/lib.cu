// Library-level state of the C ABI: thread-local error text and the launch
// counter that bench.py reports as gpu_launches.
#include <atomic>
#include <cstring>
#include "common.cuh"

namespace bmm {

static thread_local char g_err[512] = {0};
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace bmm

extern "C" int bmm_version(void) { return 1; }
extern "C" const char* bmm_last_error(void) { return bmm::g_err; }
extern "C" int64_t bmm_launch_count(void) { return bmm::g_launches.load(std::memory_order_relaxed); }

// Strided host<->device copy for the streamed end-to-end path (column slabs of
// a row-major host matrix): cudaMemcpy2DAsync, capturable in a CUDA graph.
extern "C" int bmm_copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
                          int64_t height, int kind, void* stream) {
  cudaMemcpyKind k;
  switch (kind) {
    case 1: k = cudaMemcpyHostToDevice; break;
    case 2: k = cudaMemcpyDeviceToHost; break;
    case 3: k = cudaMemcpyDeviceToDevice; break;
    default: bmm::set_error("bmm_copy2d: unknown kind %d", kind); return BMM_E_ARG;
  }
  if (width_bytes <= 0 || height <= 0) return BMM_OK;
  const cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width_bytes,
                                          (size_t)height, k, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    bmm::set_error("bmm_copy2d: %s", cudaGetErrorString(e));
    return BMM_E_CUDA;
  }
  return BMM_OK;
}

// Device clock stamp (%globaltimer, ns) into out[0]: a one-thread kernel that
// tools/timeline.py records after every stage of a captured pipeline group, to see
// when each branch's kernels finish inside one graph replay.
__global__ void stamp_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  out[0] = t;
}

extern "C" int bmm_timestamp(unsigned long long* out, void* stream) {
  stamp_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    bmm::set_error("bmm_timestamp: %s", cudaGetErrorString(e));
    return BMM_E_CUDA;
  }
  return BMM_OK;
}
