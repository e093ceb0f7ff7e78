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
