// K2 -- probabilities, score sums and integer budgets, on device.
//
// Reference: pkg/src/blockmm/plan.py
//   _index_scores 165-167, score_sums 170-173, optimal_probabilities 192-206,
//   block_norm_probabilities 483-496, integerize 242-347,
//   optimal_size_weights 350-361, _cap_array 373-380, allocate_* 383-480.
// All float64 arithmetic follows NumPy's evaluation order (pairwise.cuh) so
// probabilities, score sums and budgets are bit-identical to the reference
// given bit-identical norms.
#include "common.cuh"
#include "pairwise.cuh"
#include "rng.cuh"
#include "balance.cuh"

namespace bmm {

// sc[i] = sqrt(colsq[i]) * sqrt(rowsq[i])   (plan.py:167: column_norms * row_norms)
struct SrcScore {
  const double* cs;
  const double* rs;
  __device__ double operator()(int64_t i) const { return __dmul_rn(__dsqrt_rn(cs[i]), __dsqrt_rn(rs[i])); }
  __device__ void load8(int64_t i, double* v) const {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (*this)(i + j);
  }
};

constexpr int kProbWarps = 4;

// One warp per (problem, block).  Elementwise steps are lane-parallel
// (coalesced); the NumPy sums are warp_pw_sum; the optional CDF is the
// sequential np.cumsum (warp_cumsum, estimators.py:37-38) so the sampler can
// start from it directly.  SMEM: the block's scores are staged in a per-warp
// shared-memory slice (max_len doubles), so the three sums, two divisions and
// the cumsum run on chip; only the score loads and the final stores touch HBM.
template <bool SMEM>
__global__ void __launch_bounds__(32 * kProbWarps) block_probs_kernel(
    const double* __restrict__ colsq, const double* __restrict__ rowsq, int64_t n,
    const int64_t* __restrict__ offsets, int64_t K, int64_t batch, double* __restrict__ probs,
    double* __restrict__ s, double* __restrict__ fnorm, double* __restrict__ cum,
    int64_t* __restrict__ last, int64_t max_len) {
  __shared__ WarpPwScratch scratch[kProbWarps];
  extern __shared__ double dyn[];
  WarpPwScratch* scr = &scratch[threadIdx.x >> 5];
  double* sbuf = dyn + (SMEM ? (threadIdx.x >> 5) * max_len : 0);
  const int lane = threadIdx.x & 31;
  const int64_t total = K * batch;
  for (int64_t g = blockIdx.x * (int64_t)kProbWarps + (threadIdx.x >> 5); g < total;
       g += (int64_t)gridDim.x * kProbWarps) {
    const int64_t b = g / K, k = g - b * K;
    const int64_t o = offsets[k], nk = offsets[k + 1] - o;
    const double* cs = colsq + b * n;
    const double* rs = rowsq + b * n;
    SrcScore sc{cs, rs};
    if (probs != nullptr) {
      double* pb = probs + b * n + o;
      double* wb = SMEM ? sbuf : pb;
      // stage the scores, then normalise in place
#pragma unroll 4
      for (int64_t i = lane; i < nk; i += 32) wb[i] = sc(o + i);
      __syncwarp();
      const SrcF64 sp{wb};
      // total = sk.sum(); p = sk / total; p / p.sum()      plan.py:199-205
      const double tot = __dadd_rn(0.0, warp_pw_sum(sp, 0, nk, scr));
      if (s != nullptr) {
        // np.add.reduceat: first element, then the pairwise sum of the rest   plan.py:173
        const double rest = warp_pw_sum(sp, 1, nk - 1, scr);
        if (lane == 0) s[g] = __dadd_rn(wb[0], rest);
      }
      __syncwarp();
      if (tot == 0.0) {
        for (int64_t i = lane; i < nk; i += 32) wb[i] = 0.0;
      } else {
        for (int64_t i = lane; i < nk; i += 32) wb[i] = __ddiv_rn(wb[i], tot);
        __syncwarp();
        const double tot2 = __dadd_rn(0.0, warp_pw_sum(sp, 0, nk, scr));
        for (int64_t i = lane; i < nk; i += 32) wb[i] = __ddiv_rn(wb[i], tot2);
      }
      __syncwarp();
      if (SMEM)
        for (int64_t i = lane; i < nk; i += 32) pb[i] = wb[i];
      if (cum != nullptr) {
        const int64_t lst = warp_cumsum(wb, cum + b * n + o, nk);
        if (lane == 0) last[g] = lst;
      }
      __syncwarp();
    } else if (s != nullptr) {
      const double rest = warp_pw_sum(sc, o + 1, nk - 1, scr);
      if (lane == 0) s[g] = __dadd_rn(sc(o), rest);
    }
    if (fnorm != nullptr) {
      // ||M^k||_F * ||N_k||_F (plan.py:489).  The reference takes each factor
      // from a BLAS ddot, whose order is not reproducible; tolerance-level.
      const double fm = __dsqrt_rn(__dadd_rn(0.0, warp_pw_sum(SrcF64{cs}, o, nk, scr)));
      const double fn = __dsqrt_rn(__dadd_rn(0.0, warp_pw_sum(SrcF64{rs}, o, nk, scr)));
      if (lane == 0) fnorm[g] = __dmul_rn(fm, fn);
    }
  }
}

// Many small blocks (config 5: 4096 problems x 64 blocks of 64): one THREAD per
// (problem, block).  The warp version keeps 32 lanes busy on 64-element sums,
// shuffles and a 64-step sequential cumsum and ran issue-bound (0.56 ms at
// config 5); here each thread walks its block with NumPy's scalar pairwise
// sum (pw_sum) and the sequential cumsum out of a thread-local buffer (local
// memory is interleaved across the warp's threads, so the buffer accesses are
// coalesced).  Same operations in the same order: bit-identical results.
template <int MAXL>
__global__ void __launch_bounds__(128) block_probs_thread_kernel(
    const double* __restrict__ colsq, const double* __restrict__ rowsq, int64_t n,
    const int64_t* __restrict__ offsets, int64_t K, int64_t batch, double* __restrict__ probs,
    double* __restrict__ s, double* __restrict__ fnorm, double* __restrict__ cum, int64_t* __restrict__ last) {
  const int64_t total = K * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / K, k = g - b * K;
    const int64_t o = offsets[k], nk = offsets[k + 1] - o;
    const double* cs = colsq + b * n + o;
    const double* rs = rowsq + b * n + o;
    double buf[MAXL];
    for (int64_t i = 0; i < nk; ++i) buf[i] = __dmul_rn(__dsqrt_rn(cs[i]), __dsqrt_rn(rs[i]));
    const SrcF64 sp{buf};
    if (s != nullptr) s[g] = __dadd_rn(buf[0], pw_sum(sp, 1, nk - 1));  // np.add.reduceat   plan.py:173
    if (probs != nullptr) {
      const double tot = __dadd_rn(0.0, pw_sum(sp, 0, nk));             // plan.py:199-205
      if (tot == 0.0) {
        for (int64_t i = 0; i < nk; ++i) buf[i] = 0.0;
      } else {
        for (int64_t i = 0; i < nk; ++i) buf[i] = __ddiv_rn(buf[i], tot);
        const double tot2 = __dadd_rn(0.0, pw_sum(sp, 0, nk));
        for (int64_t i = 0; i < nk; ++i) buf[i] = __ddiv_rn(buf[i], tot2);
      }
      double* pb = probs + b * n + o;
      for (int64_t i = 0; i < nk; ++i) pb[i] = buf[i];
      if (cum != nullptr) {  // np.cumsum, sequential   estimators.py:37-38
        double acc = 0.0;
        int64_t lst = -1;
        double* cb = cum + b * n + o;
        for (int64_t i = 0; i < nk; ++i) {
          acc = __dadd_rn(acc, buf[i]);
          cb[i] = acc;
          if (buf[i] > 0.0) lst = i;
        }
        last[g] = lst;
      }
    }
    if (fnorm != nullptr) {  // ||M^k||_F * ||N_k||_F (plan.py:489), the warp kernel's order
      const double fm = __dsqrt_rn(__dadd_rn(0.0, pw_sum(SrcF64{cs}, 0, nk)));
      const double fn = __dsqrt_rn(__dadd_rn(0.0, pw_sum(SrcF64{rs}, 0, nk)));
      fnorm[g] = __dmul_rn(fm, fn);
    }
  }
}

// Large blocks (max_len > 256): one 256-thread CTA per block.  The elementwise
// scores and the two divisions use every thread; warp 0 runs the NumPy sums
// and the sequential cumsum from the shared-memory copy.  Same arithmetic and
// order as block_probs_kernel, so the results are bit-identical.
constexpr int kProbCtaThreads = 256;

__global__ void __launch_bounds__(kProbCtaThreads) block_probs_cta_kernel(
    const double* __restrict__ colsq, const double* __restrict__ rowsq, int64_t n,
    const int64_t* __restrict__ offsets, int64_t K, double* __restrict__ probs, double* __restrict__ s,
    double* __restrict__ cum, int64_t* __restrict__ last) {
  __shared__ WarpPwScratch scr, scr1;
  __shared__ double sh_tot[2];
  extern __shared__ double wb[];
  const int64_t g = blockIdx.x;
  const int64_t b = g / K, k = g - b * K;
  const int64_t o = offsets[k], nk = offsets[k + 1] - o;
  const double* cs = colsq + b * n;
  const double* rs = rowsq + b * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  SrcScore sc{cs, rs};
  double* pb = probs + b * n + o;
#pragma unroll 4
  for (int64_t i = tid; i < nk; i += kProbCtaThreads) wb[i] = sc(o + i);
  __syncthreads();
  const SrcF64 sp{wb};
  // the block total and the score sum's reduceat tail are independent trees: two warps
  if (warp == 0) {
    const double tot = __dadd_rn(0.0, warp_pw_sum(sp, 0, nk, &scr));
    if (lane == 0) sh_tot[0] = tot;
  } else if (warp == 1 && s != nullptr) {
    const double rest = warp_pw_sum(sp, 1, nk - 1, &scr1);
    if (lane == 0) s[g] = __dadd_rn(wb[0], rest);
  }
  __syncthreads();
  const double tot = sh_tot[0];
  if (tot == 0.0) {
    for (int64_t i = tid; i < nk; i += kProbCtaThreads) wb[i] = 0.0;
  } else {
    for (int64_t i = tid; i < nk; i += kProbCtaThreads) wb[i] = __ddiv_rn(wb[i], tot);
    __syncthreads();
    if (warp == 0) {
      const double tot2 = __dadd_rn(0.0, warp_pw_sum(sp, 0, nk, &scr));
      if (lane == 0) sh_tot[1] = tot2;
    }
    __syncthreads();
    const double tot2 = sh_tot[1];
    for (int64_t i = tid; i < nk; i += kProbCtaThreads) wb[i] = __ddiv_rn(wb[i], tot2);
  }
  __syncthreads();
  for (int64_t i = tid; i < nk; i += kProbCtaThreads) pb[i] = wb[i];
  if (cum != nullptr) {
    // np.cumsum: one thread runs the chain out of shared memory (independent
    // loads, one dependent add per element), then the CTA stores it
    double* wc = wb + nk;
    if (tid == 0) {
      // batches of 8: the loads of a batch are independent of its stores, so one
      // shared-memory latency per 8 elements instead of one per element
      const double* __restrict__ src = wb;
      double* __restrict__ dst = wc;
      double acc = 0.0;  // 0 + p[0] == p[0]: probabilities are never -0
      int64_t i = 0;
      for (; i + 8 <= nk; i += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = src[i + j];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc = __dadd_rn(acc, v[j]);
          dst[i + j] = acc;
        }
      }
      for (; i < nk; ++i) {
        acc = __dadd_rn(acc, src[i]);
        dst[i] = acc;
      }
    }
    // last index with p > 0 (the support clamp of _draw_indices, estimators.py:38-44)
    int64_t lst = -1;
    for (int64_t i = tid; i < nk; i += kProbCtaThreads)
      if (wb[i] > 0.0) lst = i;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const int64_t v = __shfl_xor_sync(0xffffffffu, lst, off);
      lst = v > lst ? v : lst;
    }
    __shared__ int64_t wl[kProbCtaThreads / 32];
    if (lane == 0) wl[warp] = lst;
    __syncthreads();
    double* cb = cum + b * n + o;
    for (int64_t i = tid; i < nk; i += kProbCtaThreads) cb[i] = wc[i];
    if (tid == 0) {
      int64_t m = -1;
      for (int w = 0; w < kProbCtaThreads / 32; ++w) m = wl[w] > m ? wl[w] : m;
      last[g] = m;
    }
  }
}

// q = f / f.sum()   (plan.py:493-496)
__global__ void normalize_kernel(const double* __restrict__ f, int64_t K, int64_t batch, double* q,
                                 int32_t* status) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch;
       b += (int64_t)gridDim.x * blockDim.x) {
    const double tot = __dadd_rn(0.0, pw_sum(SrcF64{f + b * K}, 0, K));
    // non-finite norms: q is NaN and _draw_indices finds no support   estimators.py:39-40
    if (status) status[b] = (tot == 0.0) ? BMM_ST_ZERO_SCORE : (isfinite(tot) ? BMM_ST_OK : BMM_ST_EMPTY_SUPPORT);
    for (int64_t k = 0; k < K; ++k) q[b * K + k] = (tot == 0.0) ? 0.0 : __ddiv_rn(f[b * K + k], tot);
  }
}

__global__ void pairwise_sum_kernel(const double* __restrict__ x, int64_t len, int64_t stride,
                                    int64_t batch, double* out) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch;
       b += (int64_t)gridDim.x * blockDim.x)
    out[b] = __dadd_rn(0.0, pw_sum(SrcF64{x + b * stride}, 0, len));
}

// ---------------------------------------------------------------- integerize

constexpr int kBudgetThreads = 256;

struct BudgetWs {
  double* w;        // K   weights
  double* wa;       // K   compacted active weights
  double* r;        // K   real shares of the active set
  int64_t* maxs;    // K
  int64_t* base;    // K   floor(r) of the active set
  int32_t* idx;     // K   compacted active block indices
  uint8_t* mins;    // K
  uint8_t* capped;  // K
  uint8_t* floored; // K
  uint64_t* key;    // P2  sort keys (descending remainder)
  int32_t* kpos;    // P2  sort payload (position in the active list)
};

__host__ __device__ inline int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline int64_t budget_ws_bytes(int64_t K) {
  const int64_t P2 = next_pow2(K);
  int64_t b = 0;
  b += 3 * align_up(8 * K, 256);        // w, wa, r
  b += 2 * align_up(8 * K, 256);        // maxs, base
  b += align_up(4 * K, 256);            // idx
  b += 3 * align_up(K, 256);            // mins, capped, floored
  b += align_up(8 * P2, 256);           // key
  b += align_up(4 * P2, 256);           // kpos
  return b;
}

__device__ inline BudgetWs carve_ws(char* p, int64_t K) {
  const int64_t P2 = next_pow2(K);
  BudgetWs ws;
  auto take = [&](int64_t bytes) { char* q = p; p += align_up(bytes, 256); return q; };
  ws.w = (double*)take(8 * K);
  ws.wa = (double*)take(8 * K);
  ws.r = (double*)take(8 * K);
  ws.maxs = (int64_t*)take(8 * K);
  ws.base = (int64_t*)take(8 * K);
  ws.idx = (int32_t*)take(4 * K);
  ws.mins = (uint8_t*)take(K);
  ws.capped = (uint8_t*)take(K);
  ws.floored = (uint8_t*)take(K);
  ws.key = (uint64_t*)take(8 * P2);
  ws.kpos = (int32_t*)take(4 * P2);
  return ws;
}

// Block-wide exclusive scan of per-thread int64 counts (thread order).
__device__ int64_t block_exclusive_scan(int64_t v, int64_t* red, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[warp] = x;
  __syncthreads();
  int64_t before = 0, all = 0;
  for (int i = 0; i < nwarps; ++i) {
    if (i < warp) before += red[i];
    all += red[i];
  }
  __syncthreads();
  *total = all;
  return before + x - v;
}

__device__ inline bool key_less(uint64_t ka, int32_t pa, uint64_t kb, int32_t pb) {
  return ka < kb || (ka == kb && pa < pb);
}

// Bitonic sort of (key, pos) pairs ascending; n is a power of two.
__device__ void bitonic_sort(uint64_t* key, int32_t* pos, int64_t n) {
  for (int64_t size = 2; size <= n; size <<= 1) {
    for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int64_t t = threadIdx.x; t < n / 2; t += blockDim.x) {
        const int64_t i = 2 * t - (t & (stride - 1));
        const int64_t j = i + stride;
        const bool up = ((i & size) == 0);
        uint64_t ki = key[i], kj = key[j];
        int32_t pi = pos[i], pj = pos[j];
        const bool swap = up ? key_less(kj, pj, ki, pi) : key_less(ki, pi, kj, pj);
        if (swap) { key[i] = kj; key[j] = ki; pos[i] = pj; pos[j] = pi; }
      }
    }
  }
  __syncthreads();
}

// integerize + the allocators' weights for ONE problem, run by every thread of the CTA
// (budgets_kernel: one CTA per problem; plan_small_kernel: a stage of the fused plan).
// sb / ab: the problem's K score sums / auxiliary values (global or shared memory).
__device__ void budgets_body(int rule, const double* sb, const double* ab, const int64_t* __restrict__ sizes,
                             const int64_t* caps_b, const uint8_t* floors_b, int64_t K, int64_t c, int cap,
                             int64_t* budgets_b, int64_t* col_off_b, int32_t* status_b, int64_t* diag_b,
                             int32_t* notes_b, BudgetWs ws) {
  __shared__ int64_t red[32];
  __shared__ int64_t sh_scalar[4];
  __shared__ double sh_S;
  const int tid = threadIdx.x;
  const int NT = blockDim.x;
  // chunked ownership keeps compaction in ascending block order
  const int64_t per = (K + NT - 1) / NT;
  const int64_t k_lo = tid * per, k_hi = min(K, k_lo + per);
  if (rule == BMM_RULE_PILOT) {
    // floor(c0/K) pilot draws for every block whose pilot distribution is nonzero
    int64_t run = 0;
    for (int64_t k = k_lo; k < k_hi; ++k) {
      const int64_t v = (sb == nullptr || sb[k] > 0.0) ? c : 0;
      budgets_b[k] = v;
      run += v;
    }
    if (col_off_b != nullptr) {
      int64_t tot = 0;
      int64_t before = block_exclusive_scan(run, red, &tot);
      for (int64_t k = k_lo; k < k_hi; ++k) {
        col_off_b[k] = before;
        before += budgets_b[k];
      }
      if (tid == 0) col_off_b[K] = tot;
    }
    if (tid == 0) {
      if (status_b) *status_b = BMM_ST_OK;
      if (diag_b) *diag_b = 0;
      if (notes_b) *notes_b = 0;
    }
    return;
  }

  int local_err = 0;  // reference error raised by this thread's blocks
  int64_t any_pos_s = 0;
  int64_t first_nonfinite = K;  // first block whose score sum (so its probabilities) is not finite
  // ---- allocator weights, caps and floors (plan.py:373-421, 465-470)
  for (int64_t k = k_lo; k < k_hi; ++k) {
    double w = 0.0;
    int64_t capk = c;
    uint8_t mn = 0;
    const double sk = sb ? sb[k] : 0.0;
    if (rule == BMM_RULE_UU) {
      w = 1.0;
      capk = cap ? sizes[k] : c;
      mn = 1;
    } else if (rule == BMM_RULE_EXPLICIT) {
      w = ab[k];
      capk = caps_b ? caps_b[k] : c;
      mn = floors_b ? (floors_b[k] != 0) : (w > 0.0);
      if (!(isfinite(w)) || w < 0.0) local_err = max(local_err, 100 + BMM_ST_BAD_WEIGHT);
    } else {
      if (sk > 0.0) any_pos_s = 1;
      // NaN/Inf in M or N: the reference's BlockProbabilities raises for the first such
      // block before any size rule runs                               plan.py:68-69
      if (!isfinite(sk)) first_nonfinite = min(first_nonfinite, k);
      if (rule == BMM_RULE_ONC) {
        w = sk;
      } else if (rule == BMM_RULE_OPL) {
        const double g = __dsqrt_rn(ab[k]);  // g_k = ||M^k N_k||_F, then squared again
        // BlockScores Cauchy-Schwarz check                              plan.py:119-120
        if (g > __dadd_rn(__dmul_rn(sk, 1.0 + 1e-9), 1e-300)) local_err = max(local_err, 100 + BMM_ST_CAUCHY_SCHWARZ);
        const double s2 = __dmul_rn(sk, sk);
        const double rad = __dsub_rn(s2, __dmul_rn(g, g));
        if (rad < __dmul_rn(-1e-9, s2)) local_err = max(local_err, 50 + BMM_ST_RADICAND);
        w = __dsqrt_rn(fmax(rad, 0.0));
      } else {  // BMM_RULE_TWO_STEP
        const double pn = __dsqrt_rn(ab[k]);  // pilot norm ||C0 D0||_F
        w = __dsqrt_rn(fabs(__dsub_rn(__dmul_rn(sk, sk), __dmul_rn(pn, pn))));
      }
      capk = (cap ? sizes[k] : c);
      if (!(sk > 0.0)) capk = 0;
      mn = (sk > 0.0);
      if (!isfinite(w)) local_err = max(local_err, 100 + BMM_ST_BAD_WEIGHT);  // integerize, plan.py:265-266
    }
    ws.w[k] = w;
    ws.maxs[k] = min(capk, c);
    ws.mins[k] = mn;
    ws.capped[k] = 0;
  }
  // reduce: error flags, positive-score existence, positive weights
  int64_t any_w = 0, err_max = local_err;
  for (int64_t k = k_lo; k < k_hi; ++k) any_w |= (ws.w[k] > 0.0);
  __syncthreads();
  {
    // pack three small values into one reduction round each
    int64_t v0 = block_sum_i64(any_pos_s, red);
    int64_t v1 = block_sum_i64(any_w, red);
    int64_t fn = first_nonfinite;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fn = min(fn, (int64_t)__shfl_xor_sync(0xffffffffu, fn, o));
    if ((tid & 31) == 0) red[tid >> 5] = fn;
    __syncthreads();
    first_nonfinite = K;
    for (int i = 0; i < (NT >> 5); ++i) first_nonfinite = min(first_nonfinite, (int64_t)red[i]);
    __syncthreads();
    // max via per-warp max then smem
    int e = (int)err_max;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
    if ((tid & 31) == 0) red[tid >> 5] = e;
    __syncthreads();
    int emax = 0;
    for (int i = 0; i < (NT >> 5); ++i) emax = max(emax, (int)red[i]);
    __syncthreads();
    any_pos_s = v0;
    any_w = v1;
    err_max = emax;
  }
  int32_t st = BMM_ST_OK;
  int64_t dg = 0;
  int32_t note = 0;
  const bool scored = (rule == BMM_RULE_ONC || rule == BMM_RULE_OPL || rule == BMM_RULE_TWO_STEP);
  // (allocate_two_step validates the optimal probabilities only after integerize, so a
  // two-step plan on NaN/Inf input raises integerize's BAD_WEIGHT, plan.py:465-479)
  if (scored && rule != BMM_RULE_TWO_STEP && first_nonfinite < K) { st = BMM_ST_BAD_PROBS; dg = first_nonfinite; }
  else if (scored && any_pos_s == 0) st = BMM_ST_ZERO_SCORE;                  // plan.py:390,410,453
  else if (err_max > 100) st = (int32_t)(err_max - 100);                       // CS / bad weight
  else if (err_max > 50) st = (int32_t)(err_max - 50);                         // radicand
  if (st == BMM_ST_OK && (rule == BMM_RULE_OPL || rule == BMM_RULE_TWO_STEP) && any_w == 0) {
    // fall back to the score-sum split                       plan.py:395-398, 467-469
    for (int64_t k = k_lo; k < k_hi; ++k) ws.w[k] = sb[k];
    note = 1;
    any_w = any_pos_s;
  }
  __syncthreads();
  if (st == BMM_ST_OK && any_w == 0) st = BMM_ST_ALL_ZERO_WEIGHT;              // plan.py:267
  if (st == BMM_ST_OK) {
    int64_t bad = 0, smin = 0, smax = 0;
    for (int64_t k = k_lo; k < k_hi; ++k) {
      bad |= (ws.maxs[k] < (int64_t)ws.mins[k]);
      smin += ws.mins[k];
      smax += ws.maxs[k];
    }
    bad = block_sum_i64(bad, red);
    smin = block_sum_i64(smin, red);
    smax = block_sum_i64(smax, red);
    if (bad) st = BMM_ST_CAP_BELOW_FLOOR;                                       // plan.py:285
    else if (smin > c) { st = BMM_ST_BELOW_FLOORS; dg = smin; }                 // plan.py:287
    else if (smax < c) { st = BMM_ST_ABOVE_CAPS; dg = smax; }                   // plan.py:289
  }

  // ---- two-level fixpoint (plan.py:296-347)
  bool done = (st != BMM_ST_OK);
  for (int64_t outer = 0; outer < K + 1 && !done; ++outer) {
    for (int64_t k = k_lo; k < k_hi; ++k) ws.floored[k] = 0;
    __syncthreads();
    bool restart = false;
    while (!done && !restart) {
      // active set, budget, compaction
      int64_t cnt_local = 0, pinned = 0;
      for (int64_t k = k_lo; k < k_hi; ++k) {
        if (ws.capped[k]) pinned += ws.maxs[k];
        else if (ws.floored[k]) pinned += ws.mins[k];
        else ++cnt_local;
      }
      const int64_t budget = c - block_sum_i64(pinned, red);
      int64_t cnt = 0;
      int64_t pos = block_exclusive_scan(cnt_local, red, &cnt);
      for (int64_t k = k_lo; k < k_hi; ++k) {
        if (!ws.capped[k] && !ws.floored[k]) { ws.idx[pos] = (int32_t)k; ws.wa[pos] = ws.w[k]; ++pos; }
      }
      __syncthreads();
      if (cnt == 0) {
        if (budget != 0) st = BMM_ST_NO_CONVERGE;                               // plan.py:305-306
        done = true;
        break;
      }
      if (tid == 0) sh_S = pw_sum(SrcF64{ws.wa}, 0, cnt);
      __syncthreads();
      const double S = sh_S;  // wa.sum() (0 + pairwise; 0 + x == x for x >= 0)
      if (S == 0.0) {
        // zero-weight leftovers: hand out the budget in index order   plan.py:311-322
        if (tid == 0) {
          int64_t left = budget;
          for (int64_t j = 0; j < cnt; ++j) {
            const int64_t i = ws.idx[j];
            const int64_t take = min(left, ws.maxs[i]);
            ws.base[j] = take;
            left -= take;
          }
          sh_scalar[0] = left;
        }
        __syncthreads();
        if (sh_scalar[0] != 0) st = BMM_ST_NO_CONVERGE;
        done = true;
        break;
      }
      // r = budget * wa / wa.sum()                                   plan.py:323
      const double bud = (double)budget;
      int64_t above = 0, below = 0;
      for (int64_t j = tid; j < cnt; j += NT) {
        const double r = __ddiv_rn(__dmul_rn(bud, ws.wa[j]), S);
        ws.r[j] = r;
        const int32_t i = ws.idx[j];
        above |= (r > __dadd_rn((double)ws.maxs[i], 1e-12));
        below |= (r < (double)ws.mins[i]);
      }
      above = __syncthreads_or((int)above);
      if (above) {
        for (int64_t j = tid; j < cnt; j += NT) {
          const int32_t i = ws.idx[j];
          if (ws.r[j] > __dadd_rn((double)ws.maxs[i], 1e-12)) ws.capped[i] = 1;
        }
        __syncthreads();
        restart = true;                                                          // plan.py:325-327
        break;
      }
      below = __syncthreads_or((int)below);
      if (below) {
        for (int64_t j = tid; j < cnt; j += NT) {
          const int32_t i = ws.idx[j];
          if (ws.r[j] < (double)ws.mins[i]) ws.floored[i] = 1;
        }
        __syncthreads();
        continue;                                                                // plan.py:328-331
      }
      // largest remainders                                            plan.py:332-340
      const int64_t P2 = next_pow2(cnt);
      int64_t bsum = 0;
      for (int64_t j = tid; j < P2; j += NT) {
        if (j < cnt) {
          const double r = ws.r[j];
          const double fl = floor(r);
          const int64_t bj = (int64_t)fl;
          ws.base[j] = bj;
          bsum += bj;
          const double frac = __dsub_rn(r, (double)bj);  // exact
          // ascending key == descending remainder; ties keep list order (stable argsort)
          ws.key[j] = 0x3FF0000000000000ULL - (uint64_t)__double_as_longlong(frac);
          ws.kpos[j] = (int32_t)j;
        } else {
          ws.key[j] = ~0ULL;
          ws.kpos[j] = 0x7fffffff;
        }
      }
      const int64_t deficit = budget - block_sum_i64(bsum, red);
      if (deficit < 0) { st = BMM_ST_NOT_PLACED; done = true; break; }
      if (deficit > 0) {
        bitonic_sort(ws.key, ws.kpos, P2);
        // rank eligible entries (base < max) in sorted order; the first `deficit` get +1
        const int64_t per2 = (cnt + NT - 1) / NT;
        const int64_t q_lo = tid * per2, q_hi = min(cnt, q_lo + per2);
        int64_t elig = 0;
        for (int64_t q = q_lo; q < q_hi; ++q) {
          const int32_t j = ws.kpos[q];
          elig += (ws.base[j] < ws.maxs[ws.idx[j]]);
        }
        int64_t tot_elig = 0;
        int64_t rank = block_exclusive_scan(elig, red, &tot_elig);
        for (int64_t q = q_lo; q < q_hi; ++q) {
          const int32_t j = ws.kpos[q];
          if (ws.base[j] < ws.maxs[ws.idx[j]]) {
            if (rank < deficit) ws.base[j] += 1;
            ++rank;
          }
        }
        if (tot_elig < deficit) st = BMM_ST_NOT_PLACED;                          // plan.py:341-342
      }
      __syncthreads();
      done = true;
    }
    if (done) break;
  }
  if (!done && st == BMM_ST_OK) st = BMM_ST_NO_CONVERGE;                         // plan.py:347
  __syncthreads();
  // ---- outputs
  int64_t cnt_local = 0;
  for (int64_t k = k_lo; k < k_hi; ++k) cnt_local += (!ws.capped[k] && !ws.floored[k]);
  int64_t cnt_total = 0;
  int64_t pos = block_exclusive_scan(cnt_local, red, &cnt_total);
  int64_t run = 0;
  int64_t first_bad = K;  // SamplingPlan check: budget 0 <=> zero-probability block
  for (int64_t k = k_lo; k < k_hi; ++k) {
    int64_t v;
    if (st != BMM_ST_OK) v = 0;
    else if (ws.capped[k]) v = ws.maxs[k];
    else if (ws.floored[k]) v = ws.mins[k];
    else v = ws.base[pos++];
    budgets_b[k] = v;
    ws.maxs[k] = v;  // reuse for the prefix below
    run += v;
    if (scored && (v == 0) != !(sb[k] > 0.0)) first_bad = min(first_bad, k);
  }
  if (st == BMM_ST_OK && scored) {
    // the zero-weight hand-out (plan.py:311-322) ignores floors, so a scored
    // block can end at 0; the reference's SamplingPlan then raises  plan.py:146-152
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first_bad = min(first_bad, (int64_t)__shfl_xor_sync(0xffffffffu, first_bad, o));
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = first_bad;
    __syncthreads();
    int64_t fb = K;
    for (int i = 0; i < (NT >> 5); ++i) fb = min(fb, red[i]);
    __syncthreads();
    if (fb < K) { st = BMM_ST_PLAN_MISMATCH; dg = fb; }
  }
  if (col_off_b != nullptr) {
    int64_t tot = 0;
    int64_t before = block_exclusive_scan(run, red, &tot);
    for (int64_t k = k_lo; k < k_hi; ++k) {
      col_off_b[k] = before;
      before += ws.maxs[k];
    }
    if (tid == 0) col_off_b[K] = tot;
  }
  if (tid == 0) {
    if (status_b) *status_b = st;
    if (diag_b) *diag_b = dg;
    if (notes_b) *notes_b = note;
  }
}


__global__ void __launch_bounds__(kBudgetThreads) budgets_kernel(
    int rule, const double* __restrict__ s, const double* __restrict__ aux,
    const int64_t* __restrict__ sizes, const int64_t* __restrict__ caps_in,
    const uint8_t* __restrict__ floors_in, int64_t K, const int64_t* __restrict__ c_arr, int cap,
    int64_t* budgets, int64_t* col_off, int32_t* status, int64_t* diag, int32_t* notes,
    char* ws_base, int use_smem) {
  // working set in shared memory when it fits (every fixpoint phase then
  // costs shared- rather than L2-latency round trips); global otherwise
  extern __shared__ __align__(16) char dyn_ws[];
  const int64_t b = blockIdx.x;
  BudgetWs ws = carve_ws(use_smem ? dyn_ws : ws_base + b * budget_ws_bytes(K), K);
  budgets_body(rule, s ? s + b * K : nullptr, aux ? aux + b * K : nullptr, sizes, caps_in ? caps_in + b * K : nullptr,
               floors_in ? floors_in + b * K : nullptr, K, c_arr[b], cap, budgets + b * K,
               col_off ? col_off + b * (K + 1) : nullptr, status ? status + b : nullptr, diag ? diag + b : nullptr,
               notes ? notes + b : nullptr, ws);
}


// ---- K2 + K3 for many small problems (config 5: 4096 problems of n = 4096, K = 64): the
// whole plan of ONE problem in ONE CTA -- scores, block probabilities, score sums, CDF
// (plan.py:165-206, estimators.py:37-38), budgets (budgets_body), child streams
// (estimators.py:141), the draws (estimators.py:34-44,78), the compressed sketch
// (bmm_compress_sketch) and the fp16 split's balanced exponents (bmm_balance_f16) -- with the
// probabilities and the CDF held in shared memory instead of making a round trip through HBM
// between seven launches.  Every value comes from the same device functions in the same
// order as the separate kernels, so budgets, draws and scales are bit-identical to them
// (tests/test_gpu_pipeline.py::test_plan_small_matches_separate_kernels).
struct PlanSmallArgs {
  int rule, cap;
  const double* colsq;
  const double* rowsq;
  int64_t n;
  const int64_t* offsets;
  const int64_t* sizes;
  int64_t K;
  const double* aux;  // OPL: g_k^2 (batch x K)
  const int64_t* c_arr;
  const uint32_t* words;
  int64_t n_words;
  const int64_t* first_child;
  int64_t W;  // sketch width (= row stride of the draw arrays)
  double* probs;
  double* s;
  double* cum;     // optional
  int64_t* last;   // optional
  int64_t* budgets;
  int64_t* col_off;
  int32_t* status;
  int64_t* diag;
  int32_t* notes;
  uint64_t* states;  // optional
  int64_t* column;
  double* prob;
  double* scale;
  int64_t* k_column;
  double* k_scale;
  int64_t* k_count;
  int32_t* kexp;    // optional (with gshift): balanced exponents of the compressed sketch
  int32_t* gshift;
  long long* dbg;   // optional: 16 clock64 stamps per problem (tools/plan_small_probe.py)
};

constexpr int kPlanThreads = 128;

__host__ __device__ inline int64_t plan_small_smem(int64_t n, int64_t K, int64_t W) {
  int64_t b = 0;
  b += align_up(8 * (n + K), 16);          // padded scores -> probabilities -> CDF (in place)
  b += align_up(8 * K, 16);                // score sums
  b += 2 * align_up(8 * (K + 1), 16);      // offsets, first sketch column of each block
  b += 2 * align_up(8 * K, 16);            // budgets, last support index
  b += align_up(32 * K, 16);               // child PCG64 states
  b += align_up(4 * ((n + 1) / 2), 16);    // draw counts per column (16-bit fields)
  b += align_up(2 * W, 16);                // drawn column of every sketch slot, then the distinct list
  b += 256 + budget_ws_bytes(K);           // integerize working set
  return b;
}

// NumPy's pairwise sum of buf[start, start + n) for n <= 128 (one leaf, pairwise.cuh) by an
// aligned group of 8 lanes: lane j runs accumulator r_j, the xor butterfly combines them as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), the group's first lane adds the n % 8 tail; every lane
// of the group gets the sum.  `gmask` = the group's 8 lanes (other groups may diverge).
__device__ __forceinline__ double group8_pw_sum(const double* buf, int64_t start, int64_t n, int j, unsigned gmask,
                                                int lane0) {
  double r = 0.0;
  if (n < 8) {
    if (j == 0)
      for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, buf[start + i]);
  } else {
    r = warp_leaf8(SrcF64{buf}, start, n, j);
    r = __dadd_rn(r, __shfl_xor_sync(gmask, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(gmask, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(gmask, r, 4));
    if (j == 0)
      for (int64_t i = n - (n % 8); i < n; ++i) r = __dadd_rn(r, buf[start + i]);
  }
  return __shfl_sync(gmask, r, lane0);
}

// buf[i] /= d for this lane's elements i = j, j + 8, ...; 4 independent divisions per step
__device__ __forceinline__ void group8_divide(double* buf, int64_t nk, int j, double d) {
  for (int64_t i0 = j; i0 < nk; i0 += 32) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (i0 + 8 * u < nk) ? buf[i0 + 8 * u] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ddiv_rn(v[u], d);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + 8 * u < nk) buf[i0 + 8 * u] = v[u];
  }
}

__global__ void __launch_bounds__(kPlanThreads, 4) plan_small_kernel(const PlanSmallArgs a) {
  extern __shared__ __align__(16) char dyn_plan[];
  __shared__ int64_t red[32];
  const int64_t b = blockIdx.x, n = a.n, K = a.K, W = a.W;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  char* q = dyn_plan;
  auto take = [&](int64_t bytes) { char* r = q; q += align_up(bytes, 16); return r; };
  // block k's scores, then probabilities, then CDF at sc[offsets[k] + k ...] (the pad spreads the banks)
  double* sc = (double*)take(8 * (n + K));
  double* ss = (double*)take(8 * K);
  int64_t* s_off = (int64_t*)take(8 * (K + 1));
  int64_t* s_col = (int64_t*)take(8 * (K + 1));
  int64_t* s_bud = (int64_t*)take(8 * K);
  int64_t* s_last = (int64_t*)take(8 * K);
  uint64_t* s_state = (uint64_t*)take(32 * K);
  uint32_t* cnt = (uint32_t*)take(4 * ((n + 1) / 2));
  uint16_t* s_draw = (uint16_t*)take(2 * W);
  q = (char*)(((uintptr_t)q + 255) & ~(uintptr_t)255);
  BudgetWs ws = carve_ws(q, K);
  auto stamp = [&](int i) {
    if (a.dbg != nullptr && tid == 0) a.dbg[b * 16 + i] = clock64();
  };
  stamp(0);
  for (int64_t k = tid; k <= K; k += NT) s_off[k] = a.offsets[k];
  for (int64_t j = tid; j < (n + 1) / 2; j += NT) cnt[j] = 0u;
  __syncthreads();
  const double* cs = a.colsq + b * n;
  const double* rs = a.rowsq + b * n;
  double* probs_b = a.probs + b * n;
  // ---- a group of 8 lanes per block: scores (plan.py:167), score sum (:173), the two
  // normalisations (:199-205), then the CDF in place (np.cumsum, estimators.py:37-38)
  {
    const int j = lane & 7, grp = tid >> 3, ngrp = NT >> 3;
    const unsigned gmask = 0xffu << (lane & 24);
    const int lane0 = lane & 24;
    for (int64_t k = grp; k < K; k += ngrp) {
      const int64_t o = s_off[k], nk = s_off[k + 1] - o;
      double* buf = sc + o + k;
      // 4 elements per step, loads first: independent square roots overlap their latencies
      for (int64_t i0 = j; i0 < nk; i0 += 32) {
        double c4[4], r4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = i0 + 8 * u;
          c4[u] = i < nk ? cs[o + i] : 0.0;
          r4[u] = i < nk ? rs[o + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) c4[u] = __dmul_rn(__dsqrt_rn(c4[u]), __dsqrt_rn(r4[u]));
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + 8 * u < nk) buf[i0 + 8 * u] = c4[u];
      }
      __syncwarp(gmask);
      if (k == 0) stamp(8);
      const double rest = group8_pw_sum(buf, 1, nk - 1, j, gmask, lane0);
      const double tot = __dadd_rn(0.0, group8_pw_sum(buf, 0, nk, j, gmask, lane0));
      if (j == 0) {
        const double sk = __dadd_rn(buf[0], rest);
        ss[k] = sk;
        a.s[b * K + k] = sk;
      }
      __syncwarp(gmask);
      if (k == 0) stamp(9);
      if (tot == 0.0) {
        for (int64_t i = j; i < nk; i += 8) buf[i] = 0.0;
      } else {
        group8_divide(buf, nk, j, tot);
        __syncwarp(gmask);
        const double tot2 = __dadd_rn(0.0, group8_pw_sum(buf, 0, nk, j, gmask, lane0));
        __syncwarp(gmask);
        group8_divide(buf, nk, j, tot2);
      }
      __syncwarp(gmask);
      if (k == 0) stamp(10);
      for (int64_t i = j; i < nk; i += 8) probs_b[o + i] = buf[i];
      __syncwarp(gmask);
      if (k == 0) stamp(11);
    }
    if (tid == 0) stamp(12);
  }
  __syncthreads();
  // the CDF in place, one lane per block: np.cumsum is a sequential chain (estimators.py:37-38)
  for (int64_t k = tid; k < K; k += NT) {
    const int64_t o = s_off[k], nk = s_off[k + 1] - o;
    double* buf = sc + o + k;
    double acc = 0.0;
    int64_t lst = -1;
    for (int64_t i = 0; i < nk; ++i) {
      const double x = buf[i];
      acc = __dadd_rn(acc, x);
      buf[i] = acc;
      if (x > 0.0) lst = i;
    }
    s_last[k] = lst;
    if (a.last != nullptr) a.last[b * K + k] = lst;
  }
  if (tid == 0) stamp(13);
  __syncthreads();
  stamp(1);
  if (a.cum != nullptr) {
    for (int64_t k = warp; k < K; k += nwarps) {
      const int64_t o = s_off[k], nk = s_off[k + 1] - o;
      for (int64_t i = lane; i < nk; i += 32) a.cum[b * n + o + i] = sc[o + k + i];
    }
  }
  stamp(2);
  // ---- budgets                                                     plan.py:242-421
  budgets_body(a.rule, ss, a.aux ? a.aux + b * K : nullptr, a.sizes, nullptr, nullptr, K, a.c_arr[b], a.cap,
               a.budgets + b * K, a.col_off + b * (K + 1), a.status + b, a.diag ? a.diag + b : nullptr,
               a.notes ? a.notes + b : nullptr, ws);
  __syncthreads();
  stamp(3);
  for (int64_t k = tid; k <= K; k += NT) {
    s_col[k] = a.col_off[b * (K + 1) + k];
    if (k < K) s_bud[k] = a.budgets[b * K + k];
  }
  // ---- child streams                                               estimators.py:141
  for (int64_t k = tid; k < K; k += NT) {
    U128 st, inc;
    seed_pcg64(a.words + b * a.n_words, a.n_words, (uint64_t)(a.first_child[b] + k), st, inc);
    s_state[4 * k] = st.hi;
    s_state[4 * k + 1] = st.lo;
    s_state[4 * k + 2] = inc.hi;
    s_state[4 * k + 3] = inc.lo;
    if (a.states != nullptr) {
      uint64_t* o = a.states + 4 * (b * K + k);
      o[0] = st.hi; o[1] = st.lo; o[2] = inc.hi; o[3] = inc.lo;
    }
  }
  __syncthreads();
  stamp(4);
  // ---- draws, flat over the sketch slots: slot t is draw j = t - s_col[k] of block k; its
  // stream state is j + 1 steps ahead of the child's seed (pcg_ahead: two 128-bit multiplies
  // from the jump table), inverse CDF by binary search, scale 1 / sqrt(c_k p_i)
  // (estimators.py:34-44, 78).  Four slots per step: their searches, probability loads (L2)
  // and square roots overlap.
  {
    auto block_of_slot = [&](int64_t t) {  // the last k with s_col[k] <= t (empty blocks skipped)
      int64_t lo = 0, hi = K;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (s_col[mid] <= t) lo = mid; else hi = mid;
      }
      return lo;
    };
    const int64_t drawn = s_col[K];
    for (int64_t t0 = tid; t0 < drawn; t0 += 4 * NT) {
      int64_t col[4];
      double dck[4], pr[4], sv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t t = t0 + u * NT;
        col[u] = 0;
        dck[u] = 1.0;
        if (t < drawn) {
          const int64_t k = block_of_slot(t);
          const int64_t o = s_off[k], len = s_off[k + 1] - o, lst = s_last[k];
          const double* cb = sc + o + k;
          const U128 st = pcg_ahead(U128{s_state[4 * k], s_state[4 * k + 1]},
                                    U128{s_state[4 * k + 2], s_state[4 * k + 3]}, (uint64_t)(t - s_col[k] + 1));
          const double uu = u53(pcg_output(st));
          int64_t lo = 0, hi = len;  // first index with cum > u (searchsorted side="right")
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (cb[mid] > uu) hi = mid; else lo = mid + 1;
          }
          const int64_t idx = max((int64_t)0, lo < lst ? lo : lst);
          col[u] = o + idx;
          dck[u] = (double)s_bud[k];
          atomicAdd(&cnt[col[u] >> 1], 1u << (16 * (int)(col[u] & 1)));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) pr[u] = (t0 + u * NT < drawn) ? probs_b[col[u]] : 1.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) sv[u] = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(dck[u], pr[u])));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t t = t0 + u * NT;
        if (t < drawn) {
          a.column[b * W + t] = col[u];
          a.prob[b * W + t] = pr[u];
          a.scale[b * W + t] = sv[u];
        }
      }
    }
  }
  __syncthreads();
  stamp(5);
  // ---- compressed sketch: the distinct drawn columns in column order with scale
  // s_i sqrt(c_i) (sketch_count_kernel + sketch_compact_kernel): warp w owns a contiguous
  // range of columns, 32 at a time; ballots count and place the drawn ones
  int64_t total = 0;
  {
    const int64_t per = (((n + nwarps - 1) / nwarps + 31) / 32) * 32;
    const int64_t lo = min(n, (int64_t)warp * per), hi = min(n, lo + per);
    auto count_of = [&](int64_t j) { return (cnt[j >> 1] >> (16 * (int)(j & 1))) & 0xffffu; };
    int64_t mine = 0;
    for (int64_t j0 = lo; j0 < hi; j0 += 32) {
      const int64_t j = j0 + lane;
      mine += __popc(__ballot_sync(0xffffffffu, j < hi && count_of(j) != 0u));
    }
    if (lane == 0) red[warp] = mine;
    __syncthreads();
    int64_t pos = 0;
    for (int w = 0; w < nwarps; ++w) {
      if (w < warp) pos += red[w];
      total += red[w];
    }
    int64_t* oc = a.k_column + b * W;
    double* os = a.k_scale + b * W;
    const unsigned below = (1u << lane) - 1u;
    __syncthreads();  // s_draw: every slot's column has been read above; now the distinct list
    for (int64_t j0 = lo; j0 < hi; j0 += 32) {
      const int64_t j = j0 + lane;
      const unsigned mk = __ballot_sync(0xffffffffu, j < hi && count_of(j) != 0u);
      if ((mk >> lane) & 1u) {
        const int64_t qpos = pos + __popc(mk & below);
        oc[qpos] = j;
        s_draw[qpos] = (uint16_t)j;
      }
      pos += __popc(mk);
    }
    __syncthreads();
    // scales s_i sqrt(c_i), four distinct columns per step
    for (int64_t q0 = tid; q0 < total; q0 += 4 * NT) {
      double pr[4], dck[4], dc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t qq = q0 + u * NT;
        const int64_t j = qq < total ? (int64_t)s_draw[qq] : 0;
        pr[u] = qq < total ? probs_b[j] : 1.0;
        int64_t kl = 0, kh = K;  // block of column j: the last k with offsets[k] <= j
        while (kh - kl > 1) {
          const int64_t mid = (kl + kh) >> 1;
          if (s_off[mid] <= j) kl = mid; else kh = mid;
        }
        dck[u] = qq < total ? (double)s_bud[kl] : 1.0;
        dc[u] = qq < total ? (double)count_of(j) : 1.0;
      }
      double sv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        sv[u] = __dmul_rn(__ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(dck[u], pr[u]))), __dsqrt_rn(dc[u]));
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + u * NT < total) os[q0 + u * NT] = sv[u];
    }
    // zero padding up to the next multiple of 64 (the float32 contractions' K steps)
    const int64_t pad_end = min(W, ((total + 63) / 64) * 64);
    for (int64_t u = total + tid; u < pad_end; u += NT) {
      oc[u] = 0;
      os[u] = 0.0;
    }
    if (tid == 0) a.k_count[b] = total;
  }
  stamp(6);
  if (a.kexp != nullptr) {
    __syncthreads();  // the compressed sketch of this CTA, written above
    f16_balance_body(cs, rs, a.k_column + b * W, a.k_scale + b * W, W, min(total, W), a.kexp + b * W, a.gshift + b);
  }
  stamp(7);
}

}  // namespace bmm

using namespace bmm;

extern "C" int bmm_block_probs(const double* colsq, const double* rowsq, int64_t n,
                               const int64_t* offsets, int64_t K, int64_t batch, int64_t max_len,
                               double* probs, double* s, double* fnorm, double* cum, int64_t* last_support,
                               void* stream) {
  BMM_REQUIRE(K >= 1 && batch >= 1 && n >= 1 && max_len >= 1, BMM_E_ARG, "bmm_block_probs: bad shape");
  BMM_REQUIRE(cum == nullptr || (probs != nullptr && last_support != nullptr), BMM_E_ARG,
              "bmm_block_probs: cum needs probs and last_support");
  const int64_t warps = K * batch;
  unsigned grid = (unsigned)std::min<int64_t>(ceil_div(warps, kProbWarps), 148LL * 16 * 64);
  const int64_t smem = max_len * 8 * kProbWarps;
  cudaStream_t st = as_stream(stream);
  static const int thread_mode = [] {
    const char* e = getenv("BMM_PROBS_THREAD");  // A/B switch: 0 keeps the warp kernel for small blocks
    return e ? atoi(e) : 1;
  }();
  if (thread_mode != 0 && max_len <= 64 && K * batch >= 16384) {
    block_probs_thread_kernel<64><<<(unsigned)std::min<int64_t>(ceil_div(K * batch, 128), 148LL * 16 * 64), 128,
                                    0, st>>>(colsq, rowsq, n, offsets, K, batch, probs, s, fnorm, cum, last_support);
  } else if (probs != nullptr && fnorm == nullptr && max_len > 256 && max_len * 16 <= 160 * 1024 &&
      K * batch < (1LL << 31)) {
    static bool attr_c = false;
    if (!attr_c) {
      cudaFuncSetAttribute(block_probs_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      attr_c = true;
    }
    block_probs_cta_kernel<<<(unsigned)(K * batch), kProbCtaThreads, (size_t)(max_len * 16), st>>>(
        colsq, rowsq, n, offsets, K, probs, s, cum, last_support);
  } else if (smem <= 160 * 1024) {
    static int64_t attr = 0;
    if (smem > 48 * 1024 && attr == 0) {
      cudaFuncSetAttribute(block_probs_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      attr = 1;
    }
    block_probs_kernel<true><<<grid, 32 * kProbWarps, (size_t)smem, st>>>(colsq, rowsq, n, offsets, K, batch, probs,
                                                                          s, fnorm, cum, last_support, max_len);
  } else {
    block_probs_kernel<false><<<grid, 32 * kProbWarps, 0, st>>>(colsq, rowsq, n, offsets, K, batch, probs, s, fnorm,
                                                               cum, last_support, max_len);
  }
  BMM_CHECK_LAUNCH("block_probs_kernel");
  return BMM_OK;
}

extern "C" int bmm_normalize(const double* f, int64_t K, int64_t batch, double* q, int32_t* status,
                             void* stream) {
  BMM_REQUIRE(K >= 1 && batch >= 1, BMM_E_ARG, "bmm_normalize: bad shape");
  normalize_kernel<<<grid_for(batch, 64), 64, 0, as_stream(stream)>>>(f, K, batch, q, status);
  BMM_CHECK_LAUNCH("normalize_kernel");
  return BMM_OK;
}

extern "C" int bmm_pairwise_sum(const double* x, int64_t len, int64_t stride, int64_t batch,
                                double* out, void* stream) {
  BMM_REQUIRE(len >= 0 && batch >= 1, BMM_E_ARG, "bmm_pairwise_sum: bad shape");
  pairwise_sum_kernel<<<grid_for(batch, 64), 64, 0, as_stream(stream)>>>(x, len, stride, batch, out);
  BMM_CHECK_LAUNCH("pairwise_sum_kernel");
  return BMM_OK;
}

extern "C" int64_t bmm_budgets_workspace(int64_t K) { return budget_ws_bytes(K); }

extern "C" int bmm_budgets(int rule, const double* s, const double* aux, const int64_t* sizes,
                           const int64_t* caps, const uint8_t* floors, int64_t K, int64_t batch,
                           const int64_t* c, int cap, int64_t* budgets, int64_t* col_off,
                           int32_t* status, int64_t* diag, int32_t* notes, void* ws,
                           void* stream) {
  BMM_REQUIRE(K >= 1 && batch >= 1, BMM_E_ARG, "bmm_budgets: bad shape");
  BMM_REQUIRE(K < (1LL << 30), BMM_E_UNSUPPORTED, "bmm_budgets: K too large");
  BMM_REQUIRE(rule >= BMM_RULE_EXPLICIT && rule <= BMM_RULE_PILOT, BMM_E_ARG, "bmm_budgets: bad rule");
  BMM_REQUIRE(rule == BMM_RULE_UU || rule == BMM_RULE_EXPLICIT || rule == BMM_RULE_PILOT || s != nullptr, BMM_E_ARG,
              "bmm_budgets: score sums required");
  BMM_REQUIRE(!(rule == BMM_RULE_OPL || rule == BMM_RULE_TWO_STEP || rule == BMM_RULE_EXPLICIT) ||
                  aux != nullptr, BMM_E_ARG, "bmm_budgets: aux required");
  BMM_REQUIRE(rule == BMM_RULE_EXPLICIT || rule == BMM_RULE_PILOT || sizes != nullptr, BMM_E_ARG, "bmm_budgets: sizes required");
  BMM_REQUIRE(budgets != nullptr && ws != nullptr && c != nullptr, BMM_E_ARG, "bmm_budgets: null output");
  const int64_t bytes = budget_ws_bytes(K);
  const bool smem = bytes <= 160 * 1024;
  if (smem && bytes > 48 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(budgets_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      attr = true;
    }
  }
  // few blocks: fewer threads, so the fixpoint's block-wide reductions and barriers are cheap
  const int nt = K <= 64 ? 64 : (K <= 128 ? 128 : kBudgetThreads);
  budgets_kernel<<<(unsigned)batch, nt, smem ? (size_t)bytes : 0, as_stream(stream)>>>(
      rule, s, aux, sizes, caps, floors, K, c, cap, budgets, col_off, status, diag, notes, (char*)ws, smem ? 1 : 0);
  BMM_CHECK_LAUNCH("budgets_kernel");
  return BMM_OK;
}

extern "C" int64_t bmm_plan_small_smem(int64_t n, int64_t K, int64_t W) { return plan_small_smem(n, K, W); }

static long long* g_plan_dbg = nullptr;
// diagnostics: 16 SM-clock stamps per problem (stage boundaries) written by the next launches
extern "C" int bmm_plan_small_debug(long long* stamps) {
  g_plan_dbg = stamps;
  return BMM_OK;
}

extern "C" int bmm_plan_small(int rule, const double* colsq, const double* rowsq, int64_t n, const int64_t* offsets,
                              const int64_t* sizes, int64_t K, int64_t batch, int64_t max_len, const double* aux,
                              const int64_t* c,
                              int cap, const uint32_t* words, int64_t n_words, const int64_t* first_child, int64_t W,
                              double* probs, double* s, double* cum, int64_t* last_support, int64_t* budgets,
                              int64_t* col_off, int32_t* status, int64_t* diag, int32_t* notes, uint64_t* states,
                              int64_t* column, double* prob, double* scale, int64_t* k_column, double* k_scale,
                              int64_t* k_count, int32_t* kexp, int32_t* gshift, void* stream) {
  BMM_REQUIRE(n >= 1 && K >= 1 && K <= n && batch >= 1 && W >= 1 && max_len >= 1, BMM_E_ARG,
              "bmm_plan_small: bad shape");
  BMM_REQUIRE(max_len <= 128, BMM_E_UNSUPPORTED,
              "bmm_plan_small: blocks of at most 128 columns (one leaf of NumPy's pairwise sum per block)");
  BMM_REQUIRE(rule == BMM_RULE_ONC || rule == BMM_RULE_OPL, BMM_E_UNSUPPORTED,
              "bmm_plan_small: score-sum (ONC) and optimal (OPL) sizes only");
  BMM_REQUIRE(rule != BMM_RULE_OPL || aux != nullptr, BMM_E_ARG, "bmm_plan_small: OPL needs g_k^2");
  BMM_REQUIRE(W < 65536 && n < 65536, BMM_E_UNSUPPORTED,
              "bmm_plan_small: W and n must be below 65536 (16-bit draw counts and column lists)");
  BMM_REQUIRE(colsq && rowsq && offsets && sizes && c && words && first_child && probs && s && budgets && col_off && status &&
                  column && prob && scale && k_column && k_scale && k_count,
              BMM_E_ARG, "bmm_plan_small: null pointer");
  BMM_REQUIRE((kexp == nullptr) == (gshift == nullptr), BMM_E_ARG, "bmm_plan_small: kexp and gshift go together");
  BMM_REQUIRE(n_words >= 4, BMM_E_ARG, "bmm_plan_small: need >= 4 entropy words (padded run entropy)");
  const int64_t smem = plan_small_smem(n, K, W);
  BMM_REQUIRE(smem <= 200 * 1024, BMM_E_UNSUPPORTED, "bmm_plan_small: problem too large for one CTA (%lld bytes)",
              (long long)smem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(plan_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  PlanSmallArgs a{rule, cap, colsq, rowsq, n, offsets, sizes, K, aux, c, words, n_words, first_child, W,
                  probs, s, cum, last_support, budgets, col_off, status, diag, notes, states, column, prob, scale,
                  k_column, k_scale, k_count, kexp, gshift, g_plan_dbg};
  plan_small_kernel<<<(unsigned)batch, kPlanThreads, (size_t)smem, as_stream(stream)>>>(a);
  BMM_CHECK_LAUNCH("plan_small_kernel");
  return BMM_OK;
}
