// C1-C3 of the sharded product (SURVEY.md §8(b2) "optional ncclComm_t variants
// that enqueue C1-C3 on the same stream", §8(e1)) as C-ABI calls on an NCCL
// communicator: the all-gather that every exchange of distributed.py is built
// from, and the rank-ordered sum of K- or n-length float64 partials
// (all-gather + a fixed-order reduction kernel, so every rank holds the same
// bits whatever algorithm NCCL picks -- an all-reduce would not).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, preferring the copy
// the process already has loaded, e.g. torch's), so the library still loads
// on hosts without NCCL; the calls then fail with BMM_E_UNSUPPORTED.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace bmm {
namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
  bool ok = false;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) return;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.get_version = reinterpret_cast<decltype(a.get_version)>(dlsym(h, "ncclGetVersion"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_gather && a.error_string &&
           a.get_version;
  });
  return a;
}

#define BMM_NCCL(call, what)                                                                 \
  do {                                                                                       \
    ncclResult_t _r = (call);                                                                \
    if (_r != ncclSuccess) {                                                                 \
      set_error("%s: %s", what, api().error_string ? api().error_string(_r) : "nccl error"); \
      return BMM_E_CUDA;                                                                     \
    }                                                                                        \
  } while (0)

#define BMM_NCCL_API()                                                                               \
  BMM_REQUIRE(api().ok, BMM_E_UNSUPPORTED, "NCCL is not available in this process (libnccl.so.2)")

// out[i] = ((parts[0][i] + parts[1][i]) + parts[2][i]) + ...  (rank order, as exchange_sum)
__global__ void __launch_bounds__(256) ordered_sum_kernel(const double* __restrict__ parts, int nranks, int64_t len,
                                                          double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = parts[i];
    for (int r = 1; r < nranks; ++r) acc = __dadd_rn(acc, parts[(int64_t)r * len + i]);
    out[i] = acc;
  }
}

}  // namespace
}  // namespace bmm

using namespace bmm;

extern "C" int bmm_nccl_version(void) {
  if (!api().ok) return 0;
  int v = 0;
  return api().get_version(&v) == ncclSuccess ? v : 0;
}

extern "C" int bmm_nccl_unique_id(void* id_out) {
  BMM_REQUIRE(id_out != nullptr, BMM_E_ARG, "bmm_nccl_unique_id: id_out is NULL");
  BMM_NCCL_API();
  ncclUniqueId id;
  BMM_NCCL(api().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof(id));
  return BMM_OK;
}

extern "C" int bmm_nccl_comm_init(void** comm_out, int nranks, const void* id, int rank) {
  BMM_REQUIRE(comm_out != nullptr && id != nullptr && nranks >= 1 && rank >= 0 && rank < nranks, BMM_E_ARG,
              "bmm_nccl_comm_init: bad arguments");
  BMM_NCCL_API();
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  BMM_NCCL(api().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
  *comm_out = c;
  return BMM_OK;
}

extern "C" int bmm_nccl_comm_destroy(void* comm) {
  if (comm == nullptr) return BMM_OK;
  BMM_NCCL_API();
  BMM_NCCL(api().comm_destroy(reinterpret_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  return BMM_OK;
}

extern "C" int bmm_all_gather_f64_nccl(void* comm, const double* src, int64_t len, double* dst, void* stream) {
  BMM_REQUIRE(comm != nullptr && len >= 0, BMM_E_ARG, "bmm_all_gather_f64_nccl: bad arguments");
  BMM_NCCL_API();
  if (len == 0) return BMM_OK;
  BMM_NCCL(api().all_gather(src, dst, (size_t)len, ncclFloat64, reinterpret_cast<ncclComm_t>(comm),
                            as_stream(stream)),
           "ncclAllGather");
  return BMM_OK;
}

extern "C" int bmm_exchange_sum_nccl(void* comm, int nranks, const double* partial, int64_t len, double* ws,
                                     double* out, void* stream) {
  BMM_REQUIRE(comm != nullptr && nranks >= 1 && len >= 0 && (len == 0 || (partial && ws && out)), BMM_E_ARG,
              "bmm_exchange_sum_nccl: bad arguments");
  if (len == 0) return BMM_OK;
  int rc = bmm_all_gather_f64_nccl(comm, partial, len, ws, stream);
  if (rc != BMM_OK) return rc;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(len, 256), 148LL * 8);
  ordered_sum_kernel<<<grid, 256, 0, as_stream(stream)>>>(ws, nranks, len, out);
  BMM_CHECK_LAUNCH("ordered_sum_kernel");
  return BMM_OK;
}
