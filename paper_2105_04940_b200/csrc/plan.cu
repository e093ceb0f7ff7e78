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
