// K3 sampler and K4 gather.
//
// Reference: _draw_indices (estimators.py:34-44), sketch_columns (55-81),
// estimate_product (125-175), estimate_product_block_sampling (221-253).
//
// One warp per block: lane L serves draws L, L+32, ... of the block's child
// stream; lane L jumps its PCG64 state L+1 steps ahead, then 32 steps per
// draw, so the warp consumes exactly the uniform sequence rng.random(c_k)
// would produce.  The CDF is the sequential np.cumsum of the block
// probabilities; the draw is upper_bound (searchsorted side="right") clamped
// onto the last positive-probability index.
#include "common.cuh"
#include "rng.cuh"
#include "pairwise.cuh"

namespace bmm {

constexpr int kCdfWarps = 4;

// One warp per block: sequential np.cumsum (warp_cumsum) and the last index
// with p > 0.
__global__ void __launch_bounds__(32 * kCdfWarps) block_cdf_kernel(
    const double* __restrict__ probs, const int64_t* __restrict__ offsets, int64_t K, int64_t batch, int64_t n,
    double* __restrict__ cum, int64_t* __restrict__ last) {
  const int64_t total = K * batch;
  for (int64_t g = blockIdx.x * (int64_t)kCdfWarps + (threadIdx.x >> 5); g < total;
       g += (int64_t)gridDim.x * kCdfWarps) {
    const int64_t b = g / K, k = g - b * K;
    const int64_t o = offsets[k], len = offsets[k + 1] - o;
    const int64_t lst = warp_cumsum(probs + b * n + o, cum + b * n + o, len);
    if ((threadIdx.x & 31) == 0) last[g] = lst;
  }
}

__global__ void seed_streams_kernel(const uint32_t* __restrict__ words, int64_t nw,
                                    const int64_t* __restrict__ first_child, int64_t count,
                                    int64_t batch, uint64_t* __restrict__ states) {
  const int64_t total = count * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / count, j = g - b * count;
    U128 st, inc;
    seed_pcg64(words + b * nw, nw, (uint64_t)(first_child[b] + j), st, inc);
    uint64_t* o = states + 4 * g;
    o[0] = st.hi;
    o[1] = st.lo;
    o[2] = inc.hi;
    o[3] = inc.lo;
  }
}

constexpr int kSampleWarps = 4;

// One warp per block.  SMEM: the block's CDF is staged in shared memory
// (max_len doubles per warp) so the binary searches stay on chip.
constexpr int64_t kSampleChunk = 128;  // draws per warp work item

// SHARED: one plan (probs, cum, last, budgets, col_off) for every problem b --
// Monte Carlo replications; only the streams and outputs are per problem.
template <bool SMEM, bool SHARED = false>
__global__ void __launch_bounds__(32 * kSampleWarps) sample_kernel(
    const double* __restrict__ probs, const double* __restrict__ cum,
    const int64_t* __restrict__ last, const int64_t* __restrict__ offsets, int64_t K, int64_t batch,
    int64_t n, const int64_t* __restrict__ budgets, const int64_t* __restrict__ col_off,
    int64_t w_stride, const uint64_t* __restrict__ states, int64_t* __restrict__ column,
    double* __restrict__ prob, double* __restrict__ scale, int64_t max_len, int wpb) {
  extern __shared__ double scum_all[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  if (w >= wpb) return;
  double* scum = scum_all + (SMEM ? 2 * w * max_len : 0);
  double* sprob = scum + max_len;
  // work slots: (draw chunk, problem, block), chunk-major so that the first
  // chunks of every block come first and empty slots (chunk beyond the budget)
  // cluster at the end; a chunk is kSampleChunk consecutive draws of one block
  const int64_t cmax = (w_stride + kSampleChunk - 1) / kSampleChunk;
  const int64_t warps_total = K * batch * cmax;
  for (int64_t g = blockIdx.x * (int64_t)wpb + w; g < warps_total; g += (int64_t)gridDim.x * wpb) {
    const int64_t ch = g / (K * batch), r = g - ch * (K * batch);
    const int64_t b = r / K, k = r - b * K;
    const int64_t pb_ = SHARED ? 0 : b;  // plan index
    const int64_t gp = pb_ * K + k;
    const int64_t ck = budgets[gp];
    const int64_t c0 = ch * kSampleChunk;
    if (c0 >= ck) continue;
    const int64_t c1 = min(ck, c0 + kSampleChunk);
    const int64_t o = offsets[k], len = offsets[k + 1] - o;
    const double* cb = cum + pb_ * n + o;
    const double* pb = probs + pb_ * n + o;
    if (SMEM) {
      __syncwarp();
      for (int64_t i = lane; i < len; i += 32) {
        scum[i] = cb[i];
        sprob[i] = pb[i];
      }
      __syncwarp();
      cb = scum;
      pb = sprob;
    }
    const int64_t lst = last[gp];
    const uint64_t* sp = states + 4 * (b * K + k);
    U128 st{sp[0], sp[1]}, inc{sp[2], sp[3]};
    U128 m1, p1, m32, p32;
    pcg_jump((uint64_t)(c0 + lane) + 1, inc, m1, p1);
    pcg_jump(32, inc, m32, p32);
    st = add128(mul128(m1, st), p1);
    const double dck = (double)ck;
    const int64_t t0 = col_off[pb_ * (K + 1) + k];
    for (int64_t j = c0 + lane; j < c1; j += 32) {
      const double u = u53(pcg_output(st));
      // first index with cum > u  (searchsorted side="right")
      int64_t lo = 0, hi = len;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cb[mid] > u) hi = mid; else lo = mid + 1;
      }
      // lst < 0 only for an all-zero (or NaN) block, which a valid plan never samples;
      // clamp anyway so a failed plan (status != OK) cannot index outside the block
      const int64_t idx = max((int64_t)0, lo < lst ? lo : lst);
      const double pr = pb[idx];
      const double sc = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(dck, pr)));
      const int64_t t = b * w_stride + t0 + j;
      column[t] = o + idx;
      prob[t] = pr;
      scale[t] = sc;
      st = add128(mul128(m32, st), p32);
    }
  }
}

__device__ __forceinline__ int64_t ceil_div_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- K4 gather

__device__ __forceinline__ double load_as_double(const double* p) { return __ldg(p); }
__device__ __forceinline__ double load_as_double(const float* p) { return (double)__ldg(p); }
__device__ __forceinline__ void store_val(double* p, double v) { *p = v; }
__device__ __forceinline__ void store_val(float* p, double v) { *p = (float)v; }

// C[h, t] = M[h, column[t]] * scale[t]: thread per sketch column t (index and
// scale loaded once), GC_ROWS rows per CTA, coalesced stores along t; columns
// past the device count of a compressed sketch exit at once
constexpr int GC_ROWS = 16;
template <typename T, typename TO>
__global__ void __launch_bounds__(256) gather_c_kernel(const T* __restrict__ M, int64_t ldm, int64_t strideM,
                                                       int64_t m, const int64_t* __restrict__ column,
                                                       const double* __restrict__ scale, int64_t W,
                                                       int64_t w_stride, int64_t batch, TO* __restrict__ C,
                                                       int64_t ldc, int64_t strideC,
                                                       const int64_t* __restrict__ wdev) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t h0 = (int64_t)blockIdx.y * GC_ROWS;
  for (int64_t b = blockIdx.z; b < batch; b += gridDim.z) {
    if (t >= W || (wdev != nullptr && t >= wdev[b])) continue;  // compressed sketch: unused columns
    const int64_t col = column[b * w_stride + t];
    const double s = scale[b * w_stride + t];
    const T* src = M + b * strideM + col;
    TO* dst = C + b * strideC + t;
    const int64_t h1 = min(m, h0 + GC_ROWS);
#pragma unroll 8
    for (int64_t h = h0; h < h1; ++h) store_val(dst + h * ldc, __dmul_rn(load_as_double(src + h * ldm), s));
  }
}

// D[t, f] = N[column[t], f] * scale[t]: CTA per GD_ROWS sketch rows, threads
// along the contiguous row of N
constexpr int GD_ROWS = 4;
template <typename T, typename TO>
__global__ void __launch_bounds__(128) gather_d_kernel(const T* __restrict__ N, int64_t ldn, int64_t strideN,
                                                       int64_t p, const int64_t* __restrict__ column,
                                                       const double* __restrict__ scale, int64_t W,
                                                       int64_t w_stride, int64_t batch, TO* __restrict__ D,
                                                       int64_t ldd, int64_t strideD,
                                                       const int64_t* __restrict__ wdev) {
  for (int64_t b = blockIdx.y; b < batch; b += gridDim.y) {
    const int64_t wend = wdev != nullptr ? min(W, wdev[b]) : W;
#pragma unroll
    for (int r = 0; r < GD_ROWS; ++r) {
      const int64_t t = (int64_t)blockIdx.x * GD_ROWS + r;
      if (t >= wend) break;
      const int64_t row = column[b * w_stride + t];
      const double s = scale[b * w_stride + t];
      const T* src = N + b * strideN + row * ldn;
      TO* dst = D + b * strideD + t * ldd;
      for (int64_t f = threadIdx.x; f < p; f += 128) store_val(dst + f, __dmul_rn(load_as_double(src + f), s));
    }
  }
}

// SSM: sketch column j belongs to draw t with sk_off[t] <= j < sk_off[t+1]
template <typename T>
__global__ void gather_blocks_kernel(const T* __restrict__ M, int64_t ldm, const T* __restrict__ N,
                                     int64_t ldn, int64_t m, int64_t p,
                                     const int64_t* __restrict__ offsets,
                                     const int64_t* __restrict__ blocks,
                                     const double* __restrict__ scale,
                                     const int64_t* __restrict__ sk_off, int64_t draws, int64_t W,
                                     T* __restrict__ C, int64_t ldc, T* __restrict__ D, int64_t ldd) {
  const int64_t totC = C ? m * W : 0;
  const int64_t totD = D ? W * p : 0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < totC + totD;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t j, h = 0, f = 0;
    if (g < totC) { h = g / W; j = g - h * W; }
    else { const int64_t r = g - totC; j = r / p; f = r - j * p; }
    int64_t lo = 0, hi = draws;  // last t with sk_off[t] <= j
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (sk_off[mid] <= j) lo = mid; else hi = mid;
    }
    const int64_t t = lo;
    const int64_t src = offsets[blocks[t]] + (j - sk_off[t]);
    const double s = scale[t];
    if (g < totC) store_val(C + h * ldc + j, __dmul_rn(s, load_as_double(M + h * ldm + src)));
    else store_val(D + j * ldd + f, __dmul_rn(s, load_as_double(N + src * ldn + f)));
  }
}

template <typename T, typename TO>
int launch_gather(const T* M, int64_t ldm, int64_t strideM, const T* N, int64_t ldn, int64_t strideN,
                  int64_t m, int64_t p, const int64_t* column, const double* scale, int64_t W,
                  int64_t w_stride, int64_t batch, TO* C, int64_t ldc, int64_t strideC, TO* D,
                  int64_t ldd, int64_t strideD, cudaStream_t st, const int64_t* wdev = nullptr) {
  if (C != nullptr && m > 0) {
    BMM_REQUIRE(ceil_div(W, 256) < (1LL << 31) && ceil_div(m, GC_ROWS) <= 65535, BMM_E_UNSUPPORTED,
                "gather: sketch too large");
    dim3 g((unsigned)ceil_div(W, 256), (unsigned)ceil_div(m, GC_ROWS), (unsigned)std::min<int64_t>(batch, 65535));
    gather_c_kernel<T, TO><<<g, 256, 0, st>>>(M, ldm, strideM, m, column, scale, W, w_stride, batch, C, ldc, strideC,
                                              wdev);
    BMM_CHECK_LAUNCH("gather_c_kernel");
  }
  if (D != nullptr && p > 0) {
    BMM_REQUIRE(ceil_div(W, GD_ROWS) < (1LL << 31), BMM_E_UNSUPPORTED, "gather: sketch too large");
    dim3 g((unsigned)ceil_div(W, GD_ROWS), (unsigned)std::min<int64_t>(batch, 65535));
    gather_d_kernel<T, TO><<<g, 128, 0, st>>>(N, ldn, strideN, p, column, scale, W, w_stride, batch, D, ldd, strideD,
                                              wdev);
    BMM_CHECK_LAUNCH("gather_d_kernel");
  }
  return BMM_OK;
}

}  // namespace bmm

using namespace bmm;

extern "C" int bmm_block_cdf(const double* probs, const int64_t* offsets, int64_t K, int64_t batch,
                             int64_t n, double* cum, int64_t* last_support, void* stream) {
  BMM_REQUIRE(K >= 1 && batch >= 1, BMM_E_ARG, "bmm_block_cdf: bad shape");
  const int64_t blocks = std::min<int64_t>(ceil_div(K * batch, kCdfWarps), 148LL * 16 * 64);
  block_cdf_kernel<<<(unsigned)blocks, 32 * kCdfWarps, 0, as_stream(stream)>>>(probs, offsets, K, batch, n, cum,
                                                                              last_support);
  BMM_CHECK_LAUNCH("block_cdf_kernel");
  return BMM_OK;
}

extern "C" int bmm_seed_streams(const uint32_t* words, int64_t n_words, const int64_t* first_child,
                                int64_t count, int64_t batch, uint64_t* states, void* stream) {
  BMM_REQUIRE(n_words >= 4 && count >= 0 && batch >= 1, BMM_E_ARG,
              "bmm_seed_streams: need >= 4 entropy words (padded run entropy)");
  if (count == 0) return BMM_OK;
  seed_streams_kernel<<<grid_for(count * batch, 128), 128, 0, as_stream(stream)>>>(words, n_words, first_child,
                                                                                  count, batch, states);
  BMM_CHECK_LAUNCH("seed_streams_kernel");
  return BMM_OK;
}

// Many small blocks (config 5): one THREAD per (problem, block) draws the block's
// budget sequentially -- one PCG64 step per draw, binary search of the block's CDF
// (64 entries, L1-resident) -- instead of a warp whose lanes jump ahead 32 steps
// and, with ~16 draws per block, sit half idle.  Same draws, same order.
template <bool SHARED>
__global__ void __launch_bounds__(128) sample_thread_kernel(
    const double* __restrict__ probs, const double* __restrict__ cum, const int64_t* __restrict__ last,
    const int64_t* __restrict__ offsets, int64_t K, int64_t batch, int64_t n, const int64_t* __restrict__ budgets,
    const int64_t* __restrict__ col_off, int64_t w_stride, const uint64_t* __restrict__ states,
    int64_t* __restrict__ column, double* __restrict__ prob, double* __restrict__ scale) {
  const int64_t total = K * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / K, k = g - b * K;
    const int64_t pb_ = SHARED ? 0 : b;
    const int64_t gp = pb_ * K + k;
    const int64_t ck = budgets[gp];
    if (ck <= 0) continue;
    const int64_t o = offsets[k], len = offsets[k + 1] - o;
    const double* cb = cum + pb_ * n + o;
    const double* pb = probs + pb_ * n + o;
    const int64_t lst = last[gp];
    const uint64_t* sp = states + 4 * (b * K + k);
    U128 st{sp[0], sp[1]};
    const U128 inc{sp[2], sp[3]};
    const double dck = (double)ck;
    const int64_t t0 = b * w_stride + col_off[pb_ * (K + 1) + k];
    for (int64_t j = 0; j < ck; ++j) {
      st = pcg_step(st, inc);
      const double u = u53(pcg_output(st));
      int64_t lo = 0, hi = len;  // first index with cum > u (searchsorted side="right")
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cb[mid] > u) hi = mid; else lo = mid + 1;
      }
      const int64_t idx = max((int64_t)0, lo < lst ? lo : lst);
      const double pr = pb[idx];
      column[t0 + j] = o + idx;
      prob[t0 + j] = pr;
      scale[t0 + j] = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(dck, pr)));
    }
  }
}

template <bool SHARED>
static int sample_impl(const double* probs, const double* cum, const int64_t* last_support, const int64_t* offsets,
                       int64_t K, int64_t batch, int64_t n, int64_t max_len, const int64_t* budgets,
                       const int64_t* col_off, int64_t w_stride, const uint64_t* states, int64_t* column,
                       double* prob, double* scale, cudaStream_t st) {
  BMM_REQUIRE(K >= 1 && batch >= 1 && max_len >= 1, BMM_E_ARG, "bmm_sample: bad shape");
  static const int thread_mode = [] {
    const char* e = getenv("BMM_SAMPLE_THREAD");  // A/B switch: 0 keeps the warp kernel for small blocks
    return e ? atoi(e) : 1;
  }();
  if (thread_mode != 0 && max_len <= 128 && K * batch >= 16384) {
    sample_thread_kernel<SHARED><<<(unsigned)std::min<int64_t>(ceil_div(K * batch, 128), 148LL * 16 * 64), 128, 0,
                                   st>>>(probs, cum, last_support, offsets, K, batch, n, budgets, col_off, w_stride,
                                         states, column, prob, scale);
    BMM_CHECK_LAUNCH("sample_thread_kernel");
    return BMM_OK;
  }
  const int64_t warps = K * batch * ((w_stride + kSampleChunk - 1) / kSampleChunk);
  const int64_t per_warp = 2 * max_len * 8;  // CDF and probabilities
  int wpb = kSampleWarps;
  bool smem = true;
  if (per_warp * kSampleWarps > 96 * 1024) wpb = 1;
  if (per_warp > 200 * 1024) smem = false;
  const int64_t blocks = std::min<int64_t>(ceil_div(warps, wpb), 148LL * 16 * 64);
  if (smem) {
    const int bytes = (int)(per_warp * wpb);
    static int attr = 0;
    if (bytes > 48 * 1024 && bytes > attr) {
      cudaFuncSetAttribute(sample_kernel<true, SHARED>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = 200 * 1024;
    }
    sample_kernel<true, SHARED><<<(unsigned)blocks, 32 * kSampleWarps, bytes, st>>>(
        probs, cum, last_support, offsets, K, batch, n, budgets, col_off, w_stride, states, column, prob, scale,
        max_len, wpb);
  } else {
    sample_kernel<false, SHARED><<<(unsigned)blocks, 32 * kSampleWarps, 0, st>>>(
        probs, cum, last_support, offsets, K, batch, n, budgets, col_off, w_stride, states, column, prob, scale,
        max_len, wpb);
  }
  BMM_CHECK_LAUNCH("sample_kernel");
  return BMM_OK;
}

extern "C" int bmm_sample(const double* probs, const double* cum, const int64_t* last_support,
                          const int64_t* offsets, int64_t K, int64_t batch, int64_t n, int64_t max_len,
                          const int64_t* budgets, const int64_t* col_off, int64_t w_stride,
                          const uint64_t* states, int64_t* column, double* prob, double* scale,
                          void* stream) {
  return sample_impl<false>(probs, cum, last_support, offsets, K, batch, n, max_len, budgets, col_off, w_stride,
                            states, column, prob, scale, as_stream(stream));
}

extern "C" int bmm_sample_reps(const double* probs, const double* cum, const int64_t* last_support,
                               const int64_t* offsets, int64_t K, int64_t reps, int64_t n, int64_t max_len,
                               const int64_t* budgets, const int64_t* col_off, int64_t w_stride,
                               const uint64_t* states, int64_t* column, double* prob, double* scale,
                               void* stream) {
  return sample_impl<true>(probs, cum, last_support, offsets, K, reps, n, max_len, budgets, col_off, w_stride,
                           states, column, prob, scale, as_stream(stream));
}

static int gather_impl(int dtype, int out_dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                       int64_t ldn, int64_t strideN, int64_t m, int64_t p, const int64_t* column,
                       const double* scale, int64_t W, int64_t w_stride, const int64_t* w_dev, int64_t batch, void* C,
                       int64_t ldc, int64_t strideC, void* D, int64_t ldd, int64_t strideD, cudaStream_t st) {
  BMM_REQUIRE(W >= 0 && batch >= 1, BMM_E_ARG, "bmm_gather: bad shape");
  if (W == 0) return BMM_OK;
#define BMM_GATHER_CASE(TI, TO)                                                                       \
  return launch_gather<TI, TO>((const TI*)M, ldm, strideM, (const TI*)N, ldn, strideN, m, p, column, \
                               scale, W, w_stride, batch, (TO*)C, ldc, strideC, (TO*)D, ldd, strideD, st, w_dev)
  if (dtype == BMM_F64 && out_dtype == BMM_F64) BMM_GATHER_CASE(double, double);
  if (dtype == BMM_F32 && out_dtype == BMM_F64) BMM_GATHER_CASE(float, double);
  if (dtype == BMM_F32 && out_dtype == BMM_F32) BMM_GATHER_CASE(float, float);
  if (dtype == BMM_F64 && out_dtype == BMM_F32) BMM_GATHER_CASE(double, float);
#undef BMM_GATHER_CASE
  set_error("bmm_gather: unknown dtype %d/%d", dtype, out_dtype);
  return BMM_E_ARG;
}

extern "C" int bmm_gather(int dtype, int out_dtype, const void* M, int64_t ldm, int64_t strideM,
                          const void* N, int64_t ldn, int64_t strideN, int64_t m, int64_t p,
                          const int64_t* column, const double* scale, int64_t W, int64_t w_stride,
                          int64_t batch, void* C, int64_t ldc, int64_t strideC, void* D, int64_t ldd,
                          int64_t strideD, void* stream) {
  return gather_impl(dtype, out_dtype, M, ldm, strideM, N, ldn, strideN, m, p, column, scale, W, w_stride, nullptr,
                     batch, C, ldc, strideC, D, ldd, strideD, as_stream(stream));
}

extern "C" int bmm_gather_dk(int dtype, int out_dtype, const void* M, int64_t ldm, int64_t strideM,
                             const void* N, int64_t ldn, int64_t strideN, int64_t m, int64_t p,
                             const int64_t* column, const double* scale, int64_t W, int64_t w_stride,
                             const int64_t* w_dev, int64_t batch, void* C, int64_t ldc, int64_t strideC, void* D,
                             int64_t ldd, int64_t strideD, void* stream) {
  BMM_REQUIRE(w_dev != nullptr, BMM_E_ARG, "bmm_gather_dk: w_dev is NULL");
  return gather_impl(dtype, out_dtype, M, ldm, strideM, N, ldn, strideN, m, p, column, scale, W, w_stride, w_dev,
                     batch, C, ldc, strideC, D, ldd, strideD, as_stream(stream));
}

extern "C" int bmm_gather_blocks(int dtype, const void* M, int64_t ldm, const void* N, int64_t ldn,
                                 int64_t m, int64_t p, const int64_t* offsets, const int64_t* blocks,
                                 const double* scale, const int64_t* sk_off, int64_t draws, int64_t W,
                                 void* C, int64_t ldc, void* D, int64_t ldd, void* stream) {
  BMM_REQUIRE(draws >= 1 && W >= 1, BMM_E_ARG, "bmm_gather_blocks: bad shape");
  cudaStream_t st = as_stream(stream);
  const int64_t work = (C ? m * W : 0) + (D ? W * p : 0);
  if (work == 0) return BMM_OK;
  if (dtype == BMM_F64) {
    gather_blocks_kernel<double><<<grid_for(work, 256), 256, 0, st>>>(
        (const double*)M, ldm, (const double*)N, ldn, m, p, offsets, blocks, scale, sk_off, draws, W,
        (double*)C, ldc, (double*)D, ldd);
  } else if (dtype == BMM_F32) {
    gather_blocks_kernel<float><<<grid_for(work, 256), 256, 0, st>>>(
        (const float*)M, ldm, (const float*)N, ldn, m, p, offsets, blocks, scale, sk_off, draws, W,
        (float*)C, ldc, (float*)D, ldd);
  } else {
    set_error("bmm_gather_blocks: unknown dtype %d", dtype);
    return BMM_E_ARG;
  }
  BMM_CHECK_LAUNCH("gather_blocks_kernel");
  return BMM_OK;
}

// ---- sketch compression (K4 prologue): all draws of a column i share the
// scale s_i = 1/sqrt(c_k p_i), so its c_i duplicates contribute
// c_i s_i^2 M[:, i] N[i, :] to C @ D.  The GEMM then runs over the distinct
// columns (in column order) with scale s_i sqrt(c_i): the same product up to
// rounding, and only as many rank-1 terms as distinct draws.  Counts are
// integers (atomics are order-free), so the result is deterministic.
__global__ void sketch_count_kernel(const int64_t* __restrict__ column, const double* __restrict__ scale, int64_t W,
                                    int64_t w_stride, int64_t n, int64_t batch, int32_t* __restrict__ cnt,
                                    double* __restrict__ sval) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < W * batch;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / W, t = g - b * W;
    const int64_t j = column[b * w_stride + t];
    atomicAdd(&cnt[b * n + j], 1);
    sval[b * n + j] = scale[b * w_stride + t];  // every draw of column j carries the same scale
  }
}

constexpr int kCompactThreads = 1024;

// One CTA per problem; warp w owns a contiguous range of columns (a multiple of
// 32), walked 32 columns at a time with coalesced loads: pass 1 counts the
// drawn columns by ballot, a prefix over the warps gives each warp its output
// base, pass 2 writes the distinct columns in column order.
__global__ void __launch_bounds__(kCompactThreads) sketch_compact_kernel(
    const int32_t* __restrict__ cnt, const double* __restrict__ sval, int64_t n, int64_t W, int64_t w_stride,
    int64_t* __restrict__ out_col, double* __restrict__ out_scale, int64_t* __restrict__ out_count) {
  __shared__ int64_t warp_base[kCompactThreads / 32 + 1];
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t per = ((ceil_div_dev(n, kCompactThreads / 32) + 31) / 32) * 32;
  const int64_t lo = min(n, w * per), hi = min(n, lo + per);
  const int32_t* cb = cnt + b * n;
  int64_t mine = 0;
#pragma unroll 4
  for (int64_t j0 = lo; j0 < hi; j0 += 32) {
    const int64_t j = j0 + lane;
    mine += __popc(__ballot_sync(0xffffffffu, j < hi && cb[j] > 0));
  }
  if (lane == 0) warp_base[w + 1] = mine;
  __syncthreads();
  if (tid == 0) {
    warp_base[0] = 0;
    for (int i = 1; i <= kCompactThreads / 32; ++i) warp_base[i] += warp_base[i - 1];
  }
  __syncthreads();
  int64_t pos = warp_base[w];
  const int64_t total = warp_base[kCompactThreads / 32];
  int64_t* oc = out_col + b * w_stride;
  double* os = out_scale + b * w_stride;
  const unsigned below = (1u << lane) - 1u;
  for (int64_t j0 = lo; j0 < hi; j0 += 32) {
    const int64_t j = j0 + lane;
    const int32_t c = j < hi ? cb[j] : 0;
    const unsigned mk = __ballot_sync(0xffffffffu, c > 0);
    if (c > 0) {
      const int64_t q = pos + __popc(mk & below);
      oc[q] = j;
      os[q] = __dmul_rn(sval[b * n + j], __dsqrt_rn((double)c));
    }
    pos += __popc(mk);
  }
  // zero padding up to the next multiple of 64 (the float32 contractions' K steps: 32, 64)
  const int64_t pad_end = min(W, ((total + 63) / 64) * 64);
  for (int64_t u = total + tid; u < pad_end; u += kCompactThreads) {
    oc[u] = 0;
    os[u] = 0.0;
  }
  if (tid == 0) out_count[b] = total;
}

extern "C" int64_t bmm_compress_workspace(int64_t n, int64_t batch) { return batch * n * (4 + 8); }

extern "C" int bmm_compress_sketch(const int64_t* column, const double* scale, int64_t W, int64_t w_stride,
                                   int64_t n, int64_t batch, void* ws, int64_t ws_bytes, int64_t* out_column,
                                   double* out_scale, int64_t* out_count, void* stream) {
  BMM_REQUIRE(W >= 1 && n >= 1 && batch >= 1 && w_stride >= W, BMM_E_ARG, "bmm_compress_sketch: bad shape");
  BMM_REQUIRE(ws != nullptr && ws_bytes >= batch * n * 12, BMM_E_ARG, "bmm_compress_sketch: workspace too small");
  BMM_REQUIRE(batch <= 65535, BMM_E_UNSUPPORTED, "bmm_compress_sketch: batch too large");
  cudaStream_t st = as_stream(stream);
  double* sval = reinterpret_cast<double*>(ws);
  int32_t* cnt = reinterpret_cast<int32_t*>(sval + batch * n);
  if (cudaMemsetAsync(cnt, 0, (size_t)(batch * n) * sizeof(int32_t), st) != cudaSuccess) {
    set_error("bmm_compress_sketch: memset failed");
    return BMM_E_CUDA;
  }
  sketch_count_kernel<<<grid_for(W * batch, 256), 256, 0, st>>>(column, scale, W, w_stride, n, batch, cnt, sval);
  BMM_CHECK_LAUNCH("sketch_count_kernel");
  sketch_compact_kernel<<<(unsigned)batch, kCompactThreads, 0, st>>>(cnt, sval, n, W, w_stride, out_column,
                                                                     out_scale, out_count);
  BMM_CHECK_LAUNCH("sketch_compact_kernel");
  return BMM_OK;
}

// ---- SSM whole-block draws as sketch columns (estimators.py:244-249): draw t
// of problem b copies block blocks[b, t] (equal blocks of block_len columns)
// scaled by scale[b, t]; column[b, t * block_len + j] = offsets[blocks] + j.
// The compress / gather / contraction stages then run unchanged, so the SSM
// baseline shares the float32 tcgen05 and float64 DMMA contractions.
__global__ void expand_blocks_kernel(const int64_t* __restrict__ blocks, const double* __restrict__ scale,
                                     int64_t draws, int64_t d_stride, const int64_t* __restrict__ offsets,
                                     int64_t block_len, int64_t batch, int64_t* __restrict__ column,
                                     double* __restrict__ col_scale, int64_t w_stride) {
  const int64_t per = draws * block_len, total = per * batch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / per, r = i - b * per, t = r / block_len, j = r - t * block_len;
    const int64_t k = blocks[b * d_stride + t];
    column[b * w_stride + r] = offsets[k] + j;
    col_scale[b * w_stride + r] = scale[b * d_stride + t];
  }
}

extern "C" int bmm_expand_blocks(const int64_t* blocks, const double* scale, int64_t draws, int64_t d_stride,
                                 const int64_t* offsets, int64_t block_len, int64_t batch, int64_t* column,
                                 double* col_scale, int64_t w_stride, void* stream) {
  BMM_REQUIRE(draws >= 1 && block_len >= 1 && batch >= 1 && d_stride >= draws && w_stride >= draws * block_len,
              BMM_E_ARG, "bmm_expand_blocks: bad shape");
  BMM_REQUIRE(blocks && scale && offsets && column && col_scale, BMM_E_ARG, "bmm_expand_blocks: null pointer");
  expand_blocks_kernel<<<grid_for(draws * block_len * batch, 256), 256, 0, as_stream(stream)>>>(
      blocks, scale, draws, d_stride, offsets, block_len, batch, column, col_scale, w_stride);
  BMM_CHECK_LAUNCH("expand_blocks_kernel");
  return BMM_OK;
}
