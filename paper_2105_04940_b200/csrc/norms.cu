// K1 -- the norm pass (bandwidth-bound, one read of M and N).
//
// Reference: column_norms / row_norms (pkg/src/blockmm/matrix.py:107-114),
// reached through _index_scores (plan.py:165-167) by every allocator.
//
// colsq: one thread owns VEC adjacent columns (one 16-byte load per row) and
//        walks the rows in order, so the float64 chain is exactly NumPy's
//        sequential add.reduce(M*M, axis=0).  R rows of loads are issued
//        before they are consumed, which keeps R*16 bytes in flight per thread.
// rowsq (NumPy's pairwise tree per row), by input size and shape:
//   * rowsq_tma_kernel   p = 128 * 2^k, contiguous: the tree is perfect, the
//                        matrix is a [leaves x 128] array streamed by TMA with
//                        SWIZZLE_128B, lane per leaf, butterfly tree (cfg4/cfg5:
//                        79-92% of HBM, tools/norms_sweep.py)
//   * rowsq_leaf_kernel  other widths <= 16384: lane per leaf from global memory,
//                        tree from a per-CTA plan of NumPy's split (60%)
//   * rowsq_warp_kernel / rowsq_kernel: small inputs and odd layouts
//   BMM_ROWSQ_VARIANT=1 skips the TMA kernel, =2 uses only the small-input kernels
//   (A/B timing in tools/norms_sweep.py).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "pairwise.cuh"

namespace bmm {

template <typename T> struct Vec16;
template <> struct Vec16<double> { using V = double2; static constexpr int N = 2; };
template <> struct Vec16<float> { using V = float4; static constexpr int N = 4; };

__device__ __forceinline__ void unpack(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
__device__ __forceinline__ void unpack(const float4& v, double* o) {
  o[0] = (double)v.x; o[1] = (double)v.y; o[2] = (double)v.z; o[3] = (double)v.w;
}

// acc + x*x with NumPy's rounding: float64 data rounds the square, then the sum
// (dmul, dadd); float32 data (x exactly representable, x*x exact in 48 bits) has
// ONE rounding either way, so a fused multiply-add gives the same bits with one
// float64 instruction fewer per element.
template <typename T>
__device__ __forceinline__ double add_sq(double acc, double x) {
  if constexpr (sizeof(T) == 4) return __fma_rn(x, x, acc);
  else return __dadd_rn(acc, __dmul_rn(x, x));
}

template <typename T, int R>
__global__ void __launch_bounds__(256) colsq_vec_kernel(const T* __restrict__ M, int64_t m, int64_t n,
                                                        int64_t ldm, int64_t strideM, int64_t batch,
                                                        int accumulate, double* __restrict__ colsq) {
  using V = typename Vec16<T>::V;
  constexpr int W = Vec16<T>::N;
  const int64_t groups = n / W;
  const int64_t total = groups * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / groups, c0 = (g - b * groups) * W;
    const T* base = M + b * strideM + c0;
    double* out = colsq + b * n + c0;
    double acc[W];
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] = accumulate ? out[j] : 0.0;
    int64_t h = 0;
    for (; h + R <= m; h += R) {
      V v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = __ldcs(reinterpret_cast<const V*>(base + (h + r) * ldm));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double x[W];
        unpack(v[r], x);
#pragma unroll
        for (int j = 0; j < W; ++j) acc[j] = add_sq<T>(acc[j], x[j]);
      }
    }
    for (; h < m; ++h) {
      V v = __ldcs(reinterpret_cast<const V*>(base + h * ldm));
      double x[W];
      unpack(v, x);
#pragma unroll
      for (int j = 0; j < W; ++j) acc[j] = add_sq<T>(acc[j], x[j]);
    }
#pragma unroll
    for (int j = 0; j < W; ++j) out[j] = acc[j];
  }
}

// Scalar path: unaligned layouts and the n % W tail columns [c_begin, n).
template <typename T, int R>
__global__ void __launch_bounds__(256) colsq_scalar_kernel(const T* __restrict__ M, int64_t m, int64_t n,
                                                           int64_t c_begin, int64_t ldm, int64_t strideM,
                                                           int64_t batch, int accumulate,
                                                           double* __restrict__ colsq) {
  const int64_t cols = n - c_begin;
  const int64_t total = cols * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / cols, c = c_begin + (g - b * cols);
    const T* base = M + b * strideM + c;
    double acc = accumulate ? colsq[b * n + c] : 0.0;
    int64_t h = 0;
    for (; h + R <= m; h += R) {
      double v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = (double)base[(h + r) * ldm];
#pragma unroll
      for (int r = 0; r < R; ++r) acc = add_sq<T>(acc, v[r]);
    }
    for (; h < m; ++h) { double x = (double)base[h * ldm]; acc = add_sq<T>(acc, x); }
    colsq[b * n + c] = acc;
  }
}

template <typename T>
__global__ void __launch_bounds__(128) rowsq_kernel(const T* __restrict__ N, int64_t n, int64_t p,
                                                    int64_t ldn, int64_t strideN, int64_t batch,
                                                    double* __restrict__ rowsq) {
  const int64_t total = n * batch;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / n, i = g - b * n;
    const T* row = N + b * strideN + i * ldn;
    SrcSq<T> src{row, (reinterpret_cast<uintptr_t>(row) & 15) == 0};
    // NumPy: add.reduce starts from the identity 0 and adds the pairwise sum.
    rowsq[g] = __dadd_rn(0.0, pw_sum(src, 0, p));
  }
}

// Few, wide rows: one warp per row (warp_pw_sum), so a row's loads are all in
// flight at once; same tree, same bits as rowsq_kernel.
constexpr int kRowWarps = 8;

template <typename T>
__global__ void __launch_bounds__(32 * kRowWarps) rowsq_warp_kernel(const T* __restrict__ N, int64_t n,
                                                                    int64_t p, int64_t ldn, int64_t strideN,
                                                                    int64_t batch, double* __restrict__ rowsq) {
  __shared__ WarpPwScratch scratch[kRowWarps];
  WarpPwScratch* scr = &scratch[threadIdx.x >> 5];
  const int64_t total = n * batch;
  for (int64_t g = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5); g < total;
       g += (int64_t)gridDim.x * kRowWarps) {
    const int64_t b = g / n, i = g - b * n;
    const T* row = N + b * strideN + i * ldn;
    SrcSq<T> src{row, false};
    const double v = __dadd_rn(0.0, warp_pw_sum(src, 0, p, scr));
    if ((threadIdx.x & 31) == 0) rowsq[g] = v;
  }
}

// ---- tree rowsq: one warp per row (or 2-4 short rows per warp), leaves read
// straight from global memory by 8-lane groups (lane j = accumulator r_j, as
// warp_pw_sum), NumPy's split tree for width p built ONCE per CTA in shared
// memory and evaluated level by level with __syncwarp only (node = left +
// right, so the evaluation order cannot change the bits).  No serial per-row
// tree walks, no block barriers in the main loop.
constexpr int kMaxLeaves = 128;  // p <= 16384

struct PwPlan {
  int32_t leaf_start[kMaxLeaves];
  int16_t leaf_len[kMaxLeaves];
  int16_t left[kMaxLeaves], right[kMaxLeaves];  // children of internal node k: >= 0 leaf, < 0 internal ~c
  int16_t order[kMaxLeaves];                    // internal nodes by height
  int16_t level_end[16];
  int32_t leaves, internal, levels, root;       // root: leaf id or ~internal
};

__device__ void build_pw_plan(int64_t p, PwPlan* P, int8_t* height) {
  // post-order walk of the split tree (as pw_tree), creating nodes instead of sums
  int64_t fs[40], fl[40];
  int16_t fleft[40];
  int8_t hleft[40];
  int fstage[40];
  int sp = 0, leaves = 0, internal = 0;
  fs[0] = 0; fl[0] = p; fstage[0] = 0;
  int16_t ret = 0;
  int8_t hret = 0;
  for (;;) {
    const int64_t len = fl[sp];
    if (len > 128) {
      int64_t n2 = len / 2;
      n2 -= n2 % 8;
      fstage[sp] = 0;
      ++sp;
      fs[sp] = fs[sp - 1];
      fl[sp] = n2;
      continue;
    }
    P->leaf_start[leaves] = (int32_t)fs[sp];
    P->leaf_len[leaves] = (int16_t)len;
    ret = (int16_t)leaves++;
    hret = 0;
    bool done = false;
    for (;;) {
      if (sp == 0) { done = true; break; }
      --sp;
      const int64_t plen = fl[sp];
      int64_t n2 = plen / 2;
      n2 -= n2 % 8;
      if (fstage[sp] == 0) {
        fleft[sp] = ret;
        hleft[sp] = hret;
        fstage[sp] = 1;
        ++sp;
        fs[sp] = fs[sp - 1] + n2;
        fl[sp] = plen - n2;
        fstage[sp] = 0;
        break;
      }
      const int k = internal++;
      P->left[k] = fleft[sp];
      P->right[k] = ret;
      height[k] = (int8_t)(1 + (hleft[sp] > hret ? hleft[sp] : hret));
      ret = (int16_t)~k;
      hret = height[k];
    }
    if (done) break;
  }
  P->leaves = leaves;
  P->internal = internal;
  P->root = ret;
  int levels = 0;
  for (int k = 0; k < internal; ++k) levels = height[k] > levels ? height[k] : levels;
  int pos = 0;
  for (int h = 1; h <= levels; ++h) {
    for (int k = 0; k < internal; ++k)
      if (height[k] == h) P->order[pos++] = (int16_t)k;
    P->level_end[h - 1] = (int16_t)pos;
  }
  P->levels = levels;
}

__device__ __forceinline__ double sq_of(double x) { return __dmul_rn(x, x); }
__device__ __forceinline__ double sq_of(float x) { const double d = (double)x; return __dmul_rn(d, d); }

// Rows wider than a leaf: lane-per-leaf.  Each LANE evaluates one whole leaf
// straight from global memory -- its 8 accumulators r_0..r_7 are independent
// chains (ILP 8) fed by 16-byte loads issued a 128-byte line at a time (the line
// is fetched once, the rest of its loads hit L1) -- then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and the tail, exactly pw_leaf.  A warp
// takes 32 leaves per pass: 32/L whole rows when a row has L <= 32 leaves, else
// one row over several passes.  Row base pointers are formed once per row and
// shuffled to the lanes.  NumPy's split tree for width p is built once per CTA
// (PwPlan) and evaluated level by level by the warp (node = left + right, so
// the evaluation order cannot change the bits).
constexpr int kLeafWarps = 8;

template <typename T> struct LeafLoad;
template <> struct LeafLoad<float> {
  static constexpr int CH = 4;  // steps of 8 elements per 128-byte line
  __device__ static void line(const float* x, double (&r)[8]) {
    float4 q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = __ldg(reinterpret_cast<const float4*>(x) + k);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const float f[8] = {q[2 * s].x, q[2 * s].y, q[2 * s].z, q[2 * s].w,
                          q[2 * s + 1].x, q[2 * s + 1].y, q[2 * s + 1].z, q[2 * s + 1].w};
#pragma unroll
      for (int k = 0; k < 8; ++k) { const double d = (double)f[k]; r[k] = __dadd_rn(r[k], __dmul_rn(d, d)); }
    }
  }
  __device__ static void step(const float* x, double (&r)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(x)), b = __ldg(reinterpret_cast<const float4*>(x) + 1);
    const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) { const double d = (double)f[k]; r[k] = __dadd_rn(r[k], __dmul_rn(d, d)); }
  }
};
template <> struct LeafLoad<double> {
  static constexpr int CH = 2;
  __device__ static void line(const double* x, double (&r)[8]) {
    double2 q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = __ldg(reinterpret_cast<const double2*>(x) + k);
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 t = q[4 * s + k];
        r[2 * k] = __dadd_rn(r[2 * k], __dmul_rn(t.x, t.x));
        r[2 * k + 1] = __dadd_rn(r[2 * k + 1], __dmul_rn(t.y, t.y));
      }
  }
  __device__ static void step(const double* x, double (&r)[8]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(x) + k);
      r[2 * k] = __dadd_rn(r[2 * k], __dmul_rn(t.x, t.x));
      r[2 * k + 1] = __dadd_rn(r[2 * k + 1], __dmul_rn(t.y, t.y));
    }
  }
};

template <typename T>
__device__ __forceinline__ double leaf_sum(const T* x, int len) {
  if (len < 8) {
    double acc = 0.0;
    for (int t = 0; t < len; ++t) acc = __dadd_rn(acc, sq_of(x[t]));
    return acc;
  }
  double r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  LeafLoad<T>::step(x, r);  // 0 + x_j^2 == x_j^2: initialises the accumulators as pw_leaf
  const int steps = len >> 3;
  constexpr int CH = LeafLoad<T>::CH;
  int s = 1;
  for (; s < steps && (s % CH) != 0; ++s) LeafLoad<T>::step(x + 8 * s, r);
  for (; s + CH <= steps; s += CH) LeafLoad<T>::line(x + 8 * s, r);
  for (; s < steps; ++s) LeafLoad<T>::step(x + 8 * s, r);
  double acc = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (int t = len & ~7; t < len; ++t) acc = __dadd_rn(acc, sq_of(x[t]));
  return acc;
}

template <typename T>
__global__ void __launch_bounds__(32 * kLeafWarps) rowsq_leaf_kernel(const T* __restrict__ N, int64_t n, int64_t p,
                                                                     int64_t ldn, int64_t strideN, int64_t batch,
                                                                     double* __restrict__ rowsq) {
  __shared__ PwPlan P;
  __shared__ int8_t hs[kMaxLeaves];
  __shared__ double vals[kLeafWarps][2 * kMaxLeaves];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) build_pw_plan(p, &P, hs);
  __syncthreads();
  double* v = vals[w];
  const int L = P.leaves, nodes = L + P.internal, levels = P.levels;
  const int root = P.root >= 0 ? P.root : L + ~P.root;
  const bool packed = L <= 32;
  const int RG = packed ? 32 / L : 1;
  const int U = packed ? 1 : (L + 31) / 32;
  // this lane's leaf within a pass (fixed for packed rows)
  const int my_r = packed ? lane / L : 0;
  const int64_t total_rows = n * batch;
  const int64_t groups = (total_rows + RG - 1) / RG;
  for (int64_t gi = (int64_t)blockIdx.x * kLeafWarps + w; gi < groups; gi += (int64_t)gridDim.x * kLeafWarps) {
    const int64_t row0 = gi * RG;
    const int rows = (int)min((int64_t)RG, total_rows - row0);
    const T* rowp = N;
    if (lane < rows) {
      const int64_t g = row0 + lane, b = g / n, i = g - b * n;
      rowp = N + b * strideN + i * ldn;
    }
    const T* myrow = reinterpret_cast<const T*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(rowp), my_r));
    for (int u = 0; u < U; ++u) {
      const int la = packed ? 0 : u * 32;
      const int nitems = packed ? rows * L : min(L, la + 32) - la;
      if (lane < nitems) {
        const int q = packed ? lane - my_r * L : la + lane;
        v[my_r * nodes + q] = leaf_sum(myrow + P.leaf_start[q], (int)P.leaf_len[q]);
      }
    }
    __syncwarp();
    for (int h = 0; h < levels; ++h) {
      const int beg = h ? P.level_end[h - 1] : 0, cnt = P.level_end[h] - beg;
      for (int t = lane; t < rows * cnt; t += 32) {
        const int sub = t / cnt;
        const int k = P.order[beg + t - sub * cnt];
        const int a = P.left[k] >= 0 ? P.left[k] : L + ~P.left[k];
        const int c = P.right[k] >= 0 ? P.right[k] : L + ~P.right[k];
        v[sub * nodes + L + k] = __dadd_rn(v[sub * nodes + a], v[sub * nodes + c]);
      }
      __syncwarp();
    }
    if (lane < rows) rowsq[row0 + lane] = __dadd_rn(0.0, v[lane * nodes + root]);
    __syncwarp();
  }
}

template <typename T>
static bool launch_rowsq_leaf(const T* N, int64_t n, int64_t p, int64_t ldn, int64_t strideN, int64_t batch,
                              double* rowsq, cudaStream_t st) {
  constexpr int64_t sz = sizeof(T);
  if (p < 32 || p > 128LL * kMaxLeaves || (ldn * sz) % 16 || (strideN * sz) % 16 ||
      reinterpret_cast<uintptr_t>(N) % 16)
    return false;
  const int64_t leaves = p <= 128 ? 1 : p / 64;
  const int64_t rg = leaves <= 32 ? std::max<int64_t>(1, 32 / leaves) : 1;
  const int64_t groups = ceil_div(n * batch, rg);
  const int64_t blocks = std::min<int64_t>(ceil_div(groups, kLeafWarps), 148LL * 8);
  rowsq_leaf_kernel<T><<<(unsigned)blocks, 32 * kLeafWarps, 0, st>>>(N, n, p, ldn, strideN, batch, rowsq);
  return true;
}

// Uniform leaves (p = 128 * 2^k, contiguous problems): NumPy's tree for width p is
// then perfect -- every leaf is 128 elements and nodes pair in order -- so the
// matrix IS a [total_leaves x 128] array.  Each warp streams 32 leaves per
// stage with TMA (SWIZZLE_128B boxes of 32 leaves x 128 bytes, 3-stage ring per
// warp on its own mbarriers), each LANE evaluates one leaf (8 independent
// accumulator chains, conflict-free 16-byte swizzled loads), and the tree is
// butterfly shuffles over the lanes (xor 1, 2, 4, ... pairs leaves in order),
// then, for rows wider than 32 leaves, an in-order pairwise combine of the
// per-stage subtrees.
constexpr int kTmaWarps = 4, kTmaStages = 3;

template <typename T>
constexpr int tma_box_elems() { return 128 / (int)sizeof(T); }  // one 128-byte swizzle row
template <typename T>
constexpr int tma_boxes() { return 128 / tma_box_elems<T>(); }   // boxes per 128-element leaf
constexpr int kTmaBoxBytes = 32 * 128;                            // 32 leaves x 128 bytes
template <typename T>
constexpr int tma_stage_bytes() { return tma_boxes<T>() * kTmaBoxBytes; }
template <typename T>
constexpr int tma_smem() { return kTmaWarps * kTmaStages * tma_stage_bytes<T>() + 1024; }

__device__ __forceinline__ uint32_t sm_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte chunk `k` of leaf row `q` inside a swizzled 32 x 128-byte box
__device__ __forceinline__ const unsigned char* swz(const unsigned char* box, int q, int k) {
  return box + q * 128 + ((k ^ (q & 7)) << 4);
}

// WARPS warps per CTA (one CTA per SM), each with its own 3-stage ring; a stage
// holds NBS of the NB boxes of a 32-leaf unit (P = NB / NBS stages per unit): the
// lane's 8 accumulator chains continue across the P stages of its leaf.  Smaller
// stages let more warps share the SM's shared memory -- with 4 warps and whole
// units per stage each SM sub-partition ran one dependent chain at a time.
template <typename T, int WARPS, int NBS>
__global__ void __launch_bounds__(32 * WARPS) rowsq_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                               int64_t total_rows, int L, int log2L,
                                                               double* __restrict__ rowsq) {
  constexpr int NB = tma_boxes<T>(), SB = NBS * kTmaBoxBytes, P = NB / NBS;
  static_assert(NB % NBS == 0, "boxes per stage must divide the boxes of a leaf");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[WARPS][kTmaStages];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* ring = smem + (int64_t)w * kTmaStages * SB;
  if (lane == 0) {
    for (int s = 0; s < kTmaStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm_addr(&bars[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const bool packed = L <= 32;
  const int U = packed ? 1 : L / 32;              // 32-leaf units per row
  const int RG = packed ? 32 / L : 1;             // rows per unit
  const int64_t units = packed ? (total_rows + RG - 1) / RG : total_rows;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + w, Wt = (int64_t)gridDim.x * WARPS;
  const int64_t nseq = gw < units ? ((units - 1 - gw) / Wt + 1) * U * P : 0;
  auto issue = [&](int64_t sq) {
    if (lane == 0 && sq < nseq) {
      const int64_t su = sq / P;  // unit-stage index (as without the split)
      const int part = (int)(sq % P);
      const int64_t unit = gw + (su / U) * Wt;
      const int64_t leaf0 = packed ? unit * 32 : unit * L + (su % U) * 32;
      uint64_t* bar = &bars[w][sq % kTmaStages];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm_addr(bar)), "r"(SB)
                   : "memory");
      unsigned char* dst = ring + (int64_t)(sq % kTmaStages) * SB;
#pragma unroll
      for (int c = 0; c < NBS; ++c)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
                sm_addr(dst + c * kTmaBoxBytes)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(sm_addr(bar)), "r"((part * NBS + c) * tma_box_elems<T>()),
            "r"((int)leaf0)
            : "memory");
    }
  };
  for (int s = 0; s < kTmaStages; ++s) issue(s);
  double part_sum[4];
  double r[8];
  for (int64_t sq = 0; sq < nseq; ++sq) {
    const int st = (int)(sq % kTmaStages);
    const int part = (int)(sq % P);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(sm_addr(&bars[w][st])),
        "r"((uint32_t)((sq / kTmaStages) & 1))
        : "memory");
    const unsigned char* stage = ring + (int64_t)st * SB;
    if (part == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = 0.0;
    }
    // this lane's leaf, elements [part * 128 / P, +128 / P): steps of 8
#pragma unroll
    for (int s8 = 0; s8 < 16 / P; ++s8) {
      constexpr int CPS = 8 * (int)sizeof(T) / 16;  // 16-byte chunks per step
      const int e0 = 8 * s8;                        // first element of the step within the stage
      const unsigned char* box = stage + (e0 / tma_box_elems<T>()) * kTmaBoxBytes;
      const int k0 = (e0 % tma_box_elems<T>()) * (int)sizeof(T) / 16;
#pragma unroll
      for (int h = 0; h < CPS; ++h) {
        const unsigned char* p = swz(box, lane, k0 + h);
        if constexpr (sizeof(T) == 4) {
          const float4 a = *reinterpret_cast<const float4*>(p);
          const float f[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double d = (double)f[k];
            r[4 * h + k] = add_sq<T>(r[4 * h + k], d);
          }
        } else {
          const double2 a = *reinterpret_cast<const double2*>(p);
          r[2 * h] = __dadd_rn(r[2 * h], __dmul_rn(a.x, a.x));
          r[2 * h + 1] = __dadd_rn(r[2 * h + 1], __dmul_rn(a.y, a.y));
        }
      }
    }
    __syncwarp();
    issue(sq + kTmaStages);  // stage st is consumed (all lanes past their loads)
    if (part != P - 1) continue;
    double t = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    // perfect tree over the 32 leaves: xor 1, 2, 4, ... (stops at the row width when packed)
    const int lim = packed ? L : 32;
    for (int o = 1; o < lim; o <<= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
    const int64_t su = sq / P;
    if (packed) {
      const int64_t row0 = (gw + (su / U) * Wt) * RG;
      const int sub = lane >> log2L;
      if ((lane & (L - 1)) == 0 && row0 + sub < total_rows) rowsq[row0 + sub] = __dadd_rn(0.0, t);
    } else {
      const int u = (int)(su % U);
      part_sum[u & 3] = t;
      if (u == U - 1) {
        double rt;
        if (U == 2) rt = __dadd_rn(part_sum[0], part_sum[1]);
        else rt = __dadd_rn(__dadd_rn(part_sum[0], part_sum[1]), __dadd_rn(part_sum[2], part_sum[3]));
        if (lane == 0) rowsq[gw + (su / U) * Wt] = __dadd_rn(0.0, rt);
      }
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <typename T>
static bool launch_rowsq_tma(const T* N, int64_t n, int64_t p, int64_t ldn, int64_t strideN, int64_t batch,
                             double* rowsq, cudaStream_t st) {
  if (p < 128 || p > 16384 || (p & (p - 1)) != 0 || ldn != p || (batch > 1 && strideN != n * p) ||
      reinterpret_cast<uintptr_t>(N) % 16 != 0)
    return false;
  const int64_t total_rows = n * batch;
  const int L = (int)(p / 128);
  const int64_t leaves = total_rows * L;
  if (leaves >= (1LL << 31)) return false;
  auto enc = tma_encode_fn();
  if (enc == nullptr) return false;
  CUtensorMap map;
  cuuint64_t dims[2] = {128, (cuuint64_t)leaves};
  cuuint64_t strides[1] = {128 * sizeof(T)};
  cuuint32_t box[2] = {(cuuint32_t)tma_box_elems<T>(), 32};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  if (enc(&map, dt, 2, const_cast<T*>(N), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return false;
  int log2L = 0;
  while ((1 << log2L) < L) ++log2L;
  const int64_t units = L <= 32 ? ceil_div(total_rows, 32 / L) : total_rows;
  static const int rcfg = [] {
    const char* e = getenv("BMM_ROWSQ_TMA_CFG");  // A/B switch (tools/cfg4_norms_probe.py)
    return e ? atoi(e) : -1;
  }();
  // default: float32 8 warps x 3 stages of half units (8 KB); float64 8 warps x quarter units
  const int cfgsel = rcfg >= 0 ? rcfg : 1;
  auto go = [&](auto kern, int warps, int nbs) {
    const int smem = warps * kTmaStages * nbs * kTmaBoxBytes + 1024;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return false;
    const int64_t blocks = std::min<int64_t>(ceil_div(units, warps), 148);
    kern<<<(unsigned)blocks, 32 * warps, smem, st>>>(map, total_rows, L, log2L, rowsq);
    return true;
  };
  if constexpr (sizeof(T) == 4) {
    switch (cfgsel) {
      case 0: return go(rowsq_tma_kernel<T, 4, 4>, 4, 4);   // round-1 shape: whole units per stage
      case 2: return go(rowsq_tma_kernel<T, 16, 1>, 16, 1);
      default: return go(rowsq_tma_kernel<T, 8, 2>, 8, 2);
    }
  } else {
    if (cfgsel == 2) return go(rowsq_tma_kernel<T, 16, 1>, 16, 1);
    return go(rowsq_tma_kernel<T, 8, 2>, 8, 2);
  }
}

// ---- Any width (e.g. config 2: p = 500, config 3: p = 1000): lane = ROW.  A
// warp owns 32 consecutive rows and streams them left to right in column
// stages (NBOX SWIZZLE_128B boxes of 32 rows x 128 bytes each) through its own
// TMA ring.  NumPy's split tree for width p is the same for every row, so it is
// compiled once per CTA into one op per 8-element group (start a leaf, add to
// its 8 accumulators, close the leaf body with ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
// add a tail element, push the leaf and fold `combines` pairs of a post-order
// stack) and every lane executes the same op stream on its own row: no
// divergence, no per-row tree walks, conflict-free 16-byte swizzled loads.
enum : uint16_t { kOpStart = 1, kOpEndMain = 2, kOpTail = 4, kOpPush = 8 };
constexpr int kRsStack = 16;

// ops[g] for the 8-element group g of a row of width p (p >= 8): bits 0-3 flags,
// bits 4-6 tail count, bits 8-11 post-order combines after the push.
__device__ void build_row_ops(int64_t p, uint16_t* ops) {
  int64_t fs[40], fl[40];
  int fstage[40];
  int sp = 0, last_leaf_group = -1;
  fs[0] = 0; fl[0] = p; fstage[0] = 0;
  for (;;) {
    const int64_t len = fl[sp];
    if (len > 128) {
      int64_t n2 = len / 2;
      n2 -= n2 % 8;
      fstage[sp] = 0;
      ++sp;
      fs[sp] = fs[sp - 1];
      fl[sp] = n2;
      continue;
    }
    // leaf [fs, fs + len): fs is a multiple of 8, only the row's last leaf has a tail
    const int g0 = (int)(fs[sp] / 8), full = (int)(len / 8), tail = (int)(len % 8);
    for (int j = 0; j < full; ++j) ops[g0 + j] = (uint16_t)((j == 0 ? kOpStart : 0) | (j == full - 1 ? kOpEndMain : 0));
    if (tail) ops[g0 + full] = (uint16_t)(kOpTail | (tail << 4));
    last_leaf_group = tail ? g0 + full : g0 + full - 1;
    ops[last_leaf_group] |= kOpPush;
    bool done = false;
    for (;;) {
      if (sp == 0) { done = true; break; }
      --sp;
      const int64_t plen = fl[sp];
      int64_t n2 = plen / 2;
      n2 -= n2 % 8;
      if (fstage[sp] == 0) {
        fstage[sp] = 1;
        ++sp;
        fs[sp] = fs[sp - 1] + n2;
        fl[sp] = plen - n2;
        fstage[sp] = 0;
        break;
      }
      ops[last_leaf_group] += (uint16_t)(1 << 8);  // node = left + right, right after its last leaf
    }
    if (done) break;
  }
}

template <typename T, int WARPS, int STAGES, int NBOX>
__global__ void __launch_bounds__(32 * WARPS) rowsq_stream_kernel(const __grid_constant__ CUtensorMap map,
                                                                  int64_t total_rows, int64_t p,
                                                                  double* __restrict__ rowsq) {
  constexpr int BOXC = tma_box_elems<T>(), SC = NBOX * BOXC, GPS = SC / 8, SB = NBOX * kTmaBoxBytes;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[WARPS][STAGES];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = (int)((p + 7) / 8), U = (int)((p + SC - 1) / SC);
  uint16_t* ops = reinterpret_cast<uint16_t*>(smem + (int64_t)WARPS * STAGES * SB);
  unsigned char* ring = smem + (int64_t)w * STAGES * SB;
  if (threadIdx.x == 0) build_row_ops(p, ops);
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm_addr(&bars[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t units = (total_rows + 31) / 32;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + w, Wt = (int64_t)gridDim.x * WARPS;
  const int64_t nseq = gw < units ? ((units - 1 - gw) / Wt + 1) * U : 0;
  auto issue = [&](int64_t sq) {
    if (lane == 0 && sq < nseq) {
      const int64_t unit = gw + (sq / U) * Wt;
      const int64_t c0 = (sq % U) * SC;
      const int nb = (int)min((int64_t)NBOX, (p - c0 + BOXC - 1) / BOXC);  // boxes that start inside the row
      uint64_t* bar = &bars[w][sq % STAGES];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm_addr(bar)),
                   "r"(nb * kTmaBoxBytes)
                   : "memory");
      unsigned char* dst = ring + (int64_t)(sq % STAGES) * SB;
      for (int c = 0; c < nb; ++c)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
                sm_addr(dst + c * kTmaBoxBytes)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(sm_addr(bar)), "r"((int)(c0 + c * BOXC)), "r"((int)(unit * 32))
            : "memory");
    }
  };
  for (int s = 0; s < STAGES; ++s) issue(s);
  double stk[kRsStack];
  int sp = 0;
  double r[8], acc = 0.0;
  for (int64_t sq = 0; sq < nseq; ++sq) {
    const int st = (int)(sq % STAGES);
    const int u = (int)(sq % U);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(sm_addr(&bars[w][st])),
        "r"((uint32_t)((sq / STAGES) & 1))
        : "memory");
    const unsigned char* stage = ring + (int64_t)st * SB;
    const int gend = min(GPS, G - u * GPS);
#pragma unroll
    for (int j = 0; j < GPS; ++j) {
      if (j < gend) {
        const uint16_t op = ops[u * GPS + j];
        double q[8];
        const unsigned char* box = stage + ((8 * j) / BOXC) * kTmaBoxBytes;
        const int k0 = ((8 * j) % BOXC) * (int)sizeof(T) / 16;
        if constexpr (sizeof(T) == 4) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 a = *reinterpret_cast<const float4*>(swz(box, lane, k0 + h));
            q[4 * h] = sq_of(a.x); q[4 * h + 1] = sq_of(a.y); q[4 * h + 2] = sq_of(a.z); q[4 * h + 3] = sq_of(a.w);
          }
        } else {
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const double2 a = *reinterpret_cast<const double2*>(swz(box, lane, k0 + h));
            q[2 * h] = sq_of(a.x); q[2 * h + 1] = sq_of(a.y);
          }
        }
        if (op & kOpTail) {
          const int t = (op >> 4) & 7;
#pragma unroll
          for (int k = 0; k < 7; ++k)
            if (k < t) acc = __dadd_rn(acc, q[k]);
        } else {
          if (op & kOpStart) {
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = q[k];
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], q[k]);
          }
          if (op & kOpEndMain)
            acc = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        }
        if (op & kOpPush) {
          stk[sp++] = acc;
          for (int c = op >> 8; c > 0; --c) {
            const double b = stk[--sp];
            stk[sp - 1] = __dadd_rn(stk[sp - 1], b);
          }
        }
      }
    }
    __syncwarp();
    issue(sq + STAGES);  // stage st consumed by every lane
    if (u == U - 1) {
      const int64_t row = (gw + (sq / U) * Wt) * 32 + lane;
      if (row < total_rows) rowsq[row] = __dadd_rn(0.0, stk[0]);
      sp = 0;
    }
  }
}

template <typename T, int WARPS, int STAGES, int NBOX>
static bool launch_rowsq_stream_cfg(const CUtensorMap& map, int64_t total_rows, int64_t p, double* rowsq,
                                    cudaStream_t st) {
  auto kern = rowsq_stream_kernel<T, WARPS, STAGES, NBOX>;
  const int smem = WARPS * STAGES * NBOX * kTmaBoxBytes + 1024 + (int)(2 * ((p + 7) / 8) + 16);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return false;
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * WARPS, smem) != cudaSuccess || occ < 1) occ = 1;
  const int64_t units = (total_rows + 31) / 32;
  const int64_t blocks = std::min<int64_t>(ceil_div(units, WARPS), 148LL * occ);
  kern<<<(unsigned)blocks, 32 * WARPS, smem, st>>>(map, total_rows, p, rowsq);
  return true;
}

template <typename T>
static bool launch_rowsq_stream(const T* N, int64_t n, int64_t p, int64_t ldn, int64_t strideN, int64_t batch,
                                double* rowsq, int cfg, cudaStream_t st) {
  const int64_t total_rows = n * batch;
  // op-stream stack: depth <= 2 + log2(p / 64)
  if (p < 32 || p > 16384 || (ldn * (int64_t)sizeof(T)) % 16 != 0 || (batch > 1 && strideN != n * ldn) ||
      reinterpret_cast<uintptr_t>(N) % 16 != 0 || total_rows >= (1LL << 31))
    return false;
  auto enc = tma_encode_fn();
  if (enc == nullptr) return false;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)p, (cuuint64_t)total_rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ldn * sizeof(T))};
  cuuint32_t box[2] = {(cuuint32_t)tma_box_elems<T>(), 32};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  if (enc(&map, dt, 2, const_cast<T*>(N), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return false;
  // auto: few 32-row units (config 2: 625) -> one warp per CTA so all of them are
  // resident at once, 8 KB stages; many (config 3: 3125) -> 4 warps, 4 KB stages
  if (cfg == 0) cfg = (total_rows + 31) / 32 < 148LL * 8 ? 1 : 3;
  switch (cfg) {
    case 1: return launch_rowsq_stream_cfg<T, 1, 4, 2>(map, total_rows, p, rowsq, st);
    case 2: return launch_rowsq_stream_cfg<T, 2, 3, 4>(map, total_rows, p, rowsq, st);
    case 3: return launch_rowsq_stream_cfg<T, 4, 4, 1>(map, total_rows, p, rowsq, st);
    default: return launch_rowsq_stream_cfg<T, 2, 4, 2>(map, total_rows, p, rowsq, st);
  }
}

// ---- TMA-staged column sums for few columns (e.g. config 2: 20000 columns,
// 500 rows): a warp owns a strip of 32 columns, its lane j the chain of column
// j.  Row slabs (32 rows x 32 columns, 4-8 KB) stream into a per-warp ring by
// TMA, so many slabs are in flight without registers while each lane walks its
// chain out of shared memory (adjacent lanes read adjacent columns: conflict
// free).  Persistent warps take strips round robin.  Default shape (measured,
// tools/norms_sweep.py): the CTA-wide variant below with 2 warps sharing 64-column
// slabs of 16 rows, 6 stages (config 2: 36.9 -> 22.7 us with the old scalar
// kernel as baseline); BMM_COLSQ_VARIANT=2..9 selects the other shapes.
template <typename T, int kCsWarps, int kCsStages, int kCsRows>
__global__ void __launch_bounds__(32 * kCsWarps) colsq_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                                  int64_t m, int64_t n, int64_t batch,
                                                                  int accumulate, double* __restrict__ colsq) {
  constexpr int SLAB = kCsRows * 32 * (int)sizeof(T);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[kCsWarps][kCsStages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const T* ring = reinterpret_cast<const T*>(smem + (int64_t)w * kCsStages * SLAB);
  if (lane == 0) {
    for (int s = 0; s < kCsStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm_addr(&bars[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const int64_t strips_per_b = (n + 31) / 32;
  const int64_t strips = strips_per_b * batch;
  const int64_t slabs = (m + kCsRows - 1) / kCsRows;
  const int64_t gw = (int64_t)blockIdx.x * kCsWarps + w, Wt = (int64_t)gridDim.x * kCsWarps;
  int64_t it = 0;  // slab counter across this warp's strips (ring position and phase)
  for (int64_t sid = gw; sid < strips; sid += Wt) {
    const int64_t b = sid / strips_per_b, c0 = (sid - b * strips_per_b) * 32;
    const int64_t row0 = b * m;  // rows of problem b in the [batch * m, n] view
    auto issue = [&](int64_t q) {  // slab q of this strip into ring slot (it + q) % S
      if (lane == 0 && q < slabs) {
        const int64_t pos = it + q;
        uint64_t* bar = &bars[w][pos % kCsStages];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm_addr(bar)), "r"(SLAB)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
                sm_addr(ring + (pos % kCsStages) * (SLAB / (int)sizeof(T)))),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(sm_addr(bar)), "r"((int)c0), "r"((int)(row0 + q * kCsRows))
            : "memory");
      }
    };
    for (int64_t q = 0; q < kCsStages - 1; ++q) issue(q);
    const int64_t col = c0 + lane;
    double acc = (accumulate && col < n) ? colsq[b * n + col] : 0.0;
    for (int64_t q = 0; q < slabs; ++q) {
      issue(q + kCsStages - 1);
      const int64_t pos = it + q;
      asm volatile(
          "{\n"
          ".reg .pred P1;\n"
          "WAIT_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra WAIT_%=;\n"
          "}\n" ::"r"(sm_addr(&bars[w][pos % kCsStages])),
          "r"((uint32_t)((pos / kCsStages) & 1))
          : "memory");
      const T* slab = ring + (pos % kCsStages) * (SLAB / (int)sizeof(T));
      const int rows = (int)min((int64_t)kCsRows, m - q * kCsRows);  // rows past m belong to the next problem
      double v[kCsRows];
#pragma unroll
      for (int r = 0; r < kCsRows; ++r) v[r] = r < rows ? (double)slab[r * 32 + lane] : 0.0;
#pragma unroll
      for (int r = 0; r < kCsRows; ++r)
        if (r < rows) acc = add_sq<T>(acc, v[r]);
      __syncwarp();  // slot is refilled by the issue of a later iteration
    }
    if (col < n) colsq[b * n + col] = acc;
    it += slabs;
  }
}

// CTA-wide variant: the CTA's warps share one slab of 32*WARPS columns, so
// each TMA row segment is 32*WARPS*sizeof(T) contiguous bytes.
template <typename T, int WARPS, int STAGES, int ROWS>
__global__ void __launch_bounds__(32 * WARPS) colsq_tma_cta_kernel(const __grid_constant__ CUtensorMap map, int64_t m,
                                                                   int64_t n, int64_t batch, int accumulate,
                                                                   double* __restrict__ colsq) {
  constexpr int COLS = 32 * WARPS, SLAB = ROWS * COLS * (int)sizeof(T);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[STAGES];
  const T* ring = reinterpret_cast<const T*>(smem);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm_addr(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t strips_per_b = (n + COLS - 1) / COLS;
  const int64_t strips = strips_per_b * batch;
  const int64_t slabs = (m + ROWS - 1) / ROWS;
  int64_t it = 0;
  for (int64_t sid = blockIdx.x; sid < strips; sid += gridDim.x) {
    const int64_t b = sid / strips_per_b, c0 = (sid - b * strips_per_b) * COLS;
    const int64_t row0 = b * m;
    auto issue = [&](int64_t q) {
      if (threadIdx.x == 0 && q < slabs) {
        const int64_t pos = it + q;
        uint64_t* bar = &bars[pos % STAGES];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm_addr(bar)), "r"(SLAB)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
                sm_addr(ring + (pos % STAGES) * (SLAB / (int)sizeof(T)))),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(sm_addr(bar)), "r"((int)c0), "r"((int)(row0 + q * ROWS))
            : "memory");
      }
    };
    for (int64_t q = 0; q < STAGES - 1; ++q) issue(q);
    const int64_t col = c0 + threadIdx.x;
    double acc = (accumulate && col < n) ? colsq[b * n + col] : 0.0;
    for (int64_t q = 0; q < slabs; ++q) {
      issue(q + STAGES - 1);
      const int64_t pos = it + q;
      asm volatile(
          "{\n"
          ".reg .pred P1;\n"
          "WAIT_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra WAIT_%=;\n"
          "}\n" ::"r"(sm_addr(&bars[pos % STAGES])),
          "r"((uint32_t)((pos / STAGES) & 1))
          : "memory");
      const T* slab = ring + (pos % STAGES) * (SLAB / (int)sizeof(T));
      const int rows = (int)min((int64_t)ROWS, m - q * ROWS);
      double v[ROWS];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) v[r] = r < rows ? (double)slab[r * COLS + threadIdx.x] : 0.0;
#pragma unroll
      for (int r = 0; r < ROWS; ++r)
        if (r < rows) acc = add_sq<T>(acc, v[r]);
      __syncthreads();  // every warp is done with the slot before it is refilled
    }
    if (col < n) colsq[b * n + col] = acc;
    it += slabs;
  }
}

template <typename T, int WARPS, int STAGES, int ROWS>
static bool launch_colsq_tma_cta(const CUtensorMap& map, int64_t m, int64_t n, int64_t batch, int accumulate,
                                 double* colsq, cudaStream_t st) {
  auto kern = colsq_tma_cta_kernel<T, WARPS, STAGES, ROWS>;
  constexpr int smem = STAGES * ROWS * 32 * WARPS * (int)sizeof(T);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return false;
    attr = true;
  }
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * WARPS, smem) != cudaSuccess || occ < 1) occ = 1;
  const int64_t strips = ((n + 32 * WARPS - 1) / (32 * WARPS)) * batch;
  const int64_t blocks = std::min<int64_t>(strips, 148LL * occ);
  kern<<<(unsigned)blocks, 32 * WARPS, smem, st>>>(map, m, n, batch, accumulate, colsq);
  return true;
}

template <typename T, int kCsWarps, int kCsStages, int kCsRows>
static bool launch_colsq_tma_cfg(const CUtensorMap& map, int64_t m, int64_t n, int64_t batch, int accumulate,
                                 double* colsq, cudaStream_t st) {
  auto kern = colsq_tma_kernel<T, kCsWarps, kCsStages, kCsRows>;
  constexpr int smem = kCsWarps * kCsStages * kCsRows * 32 * (int)sizeof(T);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return false;
    attr = true;
  }
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kCsWarps, smem) != cudaSuccess || occ < 1)
    occ = 1;
  const int64_t strips = ((n + 31) / 32) * batch;
  const int64_t blocks = std::min<int64_t>(ceil_div(strips, kCsWarps), 148LL * occ);
  kern<<<(unsigned)blocks, 32 * kCsWarps, smem, st>>>(map, m, n, batch, accumulate, colsq);
  return true;
}

template <typename T>
static bool launch_colsq_tma(const T* M, int64_t m, int64_t n, int64_t ldm, int64_t strideM, int64_t batch,
                             int accumulate, double* colsq, int variant, cudaStream_t st) {
  if (ldm != n || (batch > 1 && strideM != m * n) || (n * (int64_t)sizeof(T)) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(M) % 16 != 0 || batch * m >= (1LL << 31) || n >= (1LL << 31))
    return false;
  auto enc = tma_encode_fn();
  if (enc == nullptr) return false;
  const int rows = (variant == 2 || variant == 5 || variant == 8) ? 32 : 16;
  const int bcols = variant == 6 || variant == 8 ? 128 : variant == 7 ? 64 : 32;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)(batch * m)};
  cuuint64_t strides[1] = {(cuuint64_t)(n * sizeof(T))};
  cuuint32_t box[2] = {(cuuint32_t)bcols, (cuuint32_t)rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  if (enc(&map, dt, 2, const_cast<T*>(M), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return false;
  switch (variant) {
    case 2: return launch_colsq_tma_cfg<T, 1, 4, 32>(map, m, n, batch, accumulate, colsq, st);
    case 3: return launch_colsq_tma_cfg<T, 2, 6, 16>(map, m, n, batch, accumulate, colsq, st);
    case 4: return launch_colsq_tma_cfg<T, 1, 3, 16>(map, m, n, batch, accumulate, colsq, st);
    case 5: return launch_colsq_tma_cfg<T, 4, 6, 32>(map, m, n, batch, accumulate, colsq, st);
    case 6: return launch_colsq_tma_cta<T, 4, 6, 16>(map, m, n, batch, accumulate, colsq, st);
    case 7: return launch_colsq_tma_cta<T, 2, 6, 16>(map, m, n, batch, accumulate, colsq, st);
    case 8: return launch_colsq_tma_cta<T, 4, 4, 32>(map, m, n, batch, accumulate, colsq, st);
    case 9: return launch_colsq_tma_cfg<T, 4, 4, 16>(map, m, n, batch, accumulate, colsq, st);
    // default: per-warp rings (variant 3).  The CTA-wide ring with 6 stages of 16 rows
    // (variants 0 and 6, the round-1 default) gave wrong column sums for a warp's 32
    // columns in ~1 of 2 replays of the cfg2 graph whenever the int8 g_k chain ran
    // concurrently (tools/stress_group.py, tests/test_gpu_stress.py); variants 2, 3, 8
    // and 9 never did in 80 replays each, and 3 is as fast at cfg2 (22.6 us)
    case 0: return launch_colsq_tma_cfg<T, 2, 6, 16>(map, m, n, batch, accumulate, colsq, st);
    default: return launch_colsq_tma_cta<T, 2, 6, 16>(map, m, n, batch, accumulate, colsq, st);
  }
}

// ---- Wide column sums (config 4: M 16384 x 262144 f32; config 3: 1000 x 100000
// f64).  The direct-load kernel (colsq_vec) stalls at ~55% of HBM on config 4:
// ptxas sinks its row loads next to their uses, so few bytes are in flight per
// thread.  Here TMA does the loads: the n columns are cut into 32-column units
// and each CTA owns an equal contiguous run of units (at most kWideUnits; two
// CTAs per SM, so every unit is resident in ONE wave -- no tail of half-empty
// waves), one consumer warp per unit (lane = column: the exact sequential
// chain of NumPy's add.reduce over rows) and one producer warp that streams
// RB-row slabs of every unit of the CTA into a STAGES-deep ring (full/empty
// mbarriers).  Rows past m inside the last slab are TMA zero-fill and skipped.
constexpr int kWideWarps = 28;  // consumer warps per CTA (at most)

// QB units (32-column strips) per TMA box: a box is 32*QB columns x RB rows, so the
// single producer thread issues 1/QB as many bulk copies (measured: the copy issue
// rate, not HBM, bounded the 1-unit boxes at ~4.9 TB/s).  Consumer warp w owns
// unit w (lane = column): box w / QB, columns 32 * (w % QB) + lane.
template <typename T, int RB, int STAGES, int QB>
__global__ void __launch_bounds__(32 * (kWideWarps + 1), 2) colsq_wide_kernel(const __grid_constant__ CUtensorMap map,
                                                                             int64_t m, int64_t n, int64_t groups,
                                                                             int accumulate, double* __restrict__ colsq) {
  constexpr int BOX = 32 * QB * RB * (int)sizeof(T);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = (int)(blockDim.x >> 5) - 1;  // consumer warps; warp nw produces
  // this CTA's boxes: groups [g0, g1) of 32*QB columns
  const int64_t g0 = (int64_t)blockIdx.x * groups / gridDim.x, g1 = (int64_t)(blockIdx.x + 1) * groups / gridDim.x;
  const int G = (int)(g1 - g0);
  const int64_t c_end = min(n, g1 * 32 * QB);                       // columns this CTA owns
  const int U = (int)((c_end - g0 * 32 * QB + 31) / 32);            // its units (<= G * QB)
  const int64_t slabs = (m + RB - 1) / RB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm_addr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sm_addr(&empty[s])), "r"(U));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == nw) {
    if (lane == 0) {
      for (int64_t q = 0; q < slabs; ++q) {
        const int st = (int)(q % STAGES);
        if (q >= STAGES) {
          const uint32_t par = (uint32_t)(((q / STAGES) - 1) & 1);
          asm volatile(
              "{\n"
              ".reg .pred P1;\n"
              "WAIT_%=:\n"
              "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
              "@!P1 bra WAIT_%=;\n"
              "}\n" ::"r"(sm_addr(&empty[st])),
              "r"(par)
              : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm_addr(&full[st])),
                     "r"(G * BOX)
                     : "memory");
        for (int g = 0; g < G; ++g)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
                  sm_addr(smem + (int64_t)(st * G + g) * BOX)),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(sm_addr(&full[st])), "r"((int)((g0 + g) * 32 * QB)),
              "r"((int)(q * RB))
              : "memory");
      }
    }
    return;
  }
  if (warp >= U) return;
  const int64_t col = g0 * 32 * QB + warp * 32 + lane;
  double acc = (accumulate && col < n) ? colsq[col] : 0.0;
  const int bx = warp / QB, sub = (warp % QB) * 32 + lane;
  for (int64_t q = 0; q < slabs; ++q) {
    const int st = (int)(q % STAGES);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(sm_addr(&full[st])),
        "r"((uint32_t)((q / STAGES) & 1))
        : "memory");
    const T* slab = reinterpret_cast<const T*>(smem + (int64_t)(st * G + bx) * BOX);
    const int rows = (int)min((int64_t)RB, m - q * RB);
    double v[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) v[r] = (double)slab[r * 32 * QB + sub];
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (r < rows) acc = add_sq<T>(acc, v[r]);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sm_addr(&empty[st])) : "memory");
  }
  if (col < n) colsq[col] = acc;
}

template <typename T, int RB, int STAGES, int QB>
static bool launch_colsq_wide_cfg(const T* M, int64_t m, int64_t n, int64_t ldm, int accumulate, double* colsq,
                                  cudaStream_t st) {
  auto enc = tma_encode_fn();
  if (enc == nullptr) return false;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
  cuuint64_t strides[1] = {(cuuint64_t)(ldm * sizeof(T))};
  cuuint32_t box[2] = {(cuuint32_t)(32 * QB), (cuuint32_t)RB};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  if (enc(&map, dt, 2, const_cast<T*>(M), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return false;
  const int64_t groups = (n + 32 * QB - 1) / (32 * QB);
  // two CTAs per SM; every group in ONE wave while groups <= 296 * (kWideWarps / QB)
  int64_t ctas = std::max<int64_t>(296, ceil_div(groups, (int64_t)(kWideWarps / QB)));
  ctas = std::min<int64_t>(ctas, groups);
  const int gmax = (int)ceil_div(groups, ctas);
  auto kern = colsq_wide_kernel<T, RB, STAGES, QB>;
  const int smem = STAGES * gmax * 32 * QB * RB * (int)sizeof(T) + 1024;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return false;
  kern<<<(unsigned)ctas, 32 * (gmax * QB + 1), smem, st>>>(map, m, n, groups, accumulate, colsq);
  return true;
}

template <typename T>
static bool launch_colsq_wide(const T* M, int64_t m, int64_t n, int64_t ldm, int accumulate, double* colsq,
                              cudaStream_t st) {
  if ((ldm * (int64_t)sizeof(T)) % 16 != 0 || ldm < n || reinterpret_cast<uintptr_t>(M) % 16 != 0 ||
      m >= (1LL << 31) || n >= (1LL << 31))
    return false;
  static const int cfg = [] {
    const char* e = getenv("BMM_COLSQ_WIDE_CFG");  // A/B switch (tools/cfg4_norms_probe.py)
    return e ? atoi(e) : 0;
  }();
  if constexpr (sizeof(T) == 8) {
    if (cfg == 1) return launch_colsq_wide_cfg<T, 8, 2, 1>(M, m, n, ldm, accumulate, colsq, st);
    return launch_colsq_wide_cfg<T, 8, 2, 4>(M, m, n, ldm, accumulate, colsq, st);
  } else {
    switch (cfg) {
      case 1: return launch_colsq_wide_cfg<T, 8, 3, 1>(M, m, n, ldm, accumulate, colsq, st);
      case 2: return launch_colsq_wide_cfg<T, 16, 2, 2>(M, m, n, ldm, accumulate, colsq, st);
      case 3: return launch_colsq_wide_cfg<T, 4, 6, 4>(M, m, n, ldm, accumulate, colsq, st);
      default: return launch_colsq_wide_cfg<T, 8, 3, 4>(M, m, n, ldm, accumulate, colsq, st);
    }
  }
}

template <typename T>
int launch_norms(const T* M, int64_t m, int64_t n, int64_t ldm, int64_t strideM, const T* N,
                 int64_t p, int64_t ldn, int64_t strideN, int64_t batch, int accumulate,
                 double* colsq, double* rowsq, cudaStream_t st) {
  constexpr int W = Vec16<T>::N;
  if (M != nullptr) {
    BMM_REQUIRE(colsq != nullptr, BMM_E_ARG, "bmm_norms: colsq is NULL");
    // Few columns (e.g. config 2: 20000): one column per thread in 64-thread CTAs
    // spreads the chains over every SM and keeps 32 row loads in flight each.
    const bool narrow = (n / W) * batch < 148LL * 256;
    static const int cs_variant = [] {
      const char* e = getenv("BMM_COLSQ_VARIANT");  // A/B switch: 1 disables the TMA-staged kernel, 2-5 pick its shape
      return e ? atoi(e) : 0;
    }();
    static const int wide_mode = [] {
      const char* e = getenv("BMM_COLSQ_WIDE");  // A/B switch: 0 keeps the direct-load kernel for wide M
      return e ? atoi(e) : 1;
    }();
    // wide, long single matrices (>= 256 MB): the TMA-streamed one-wave kernel
    // (BMM_COLSQ_WIDE=2 forces it for any single matrix: sanitizer runs on small inputs)
    const bool wide = batch == 1 && ((wide_mode == 2 && n >= 32) ||
                                     (!narrow && wide_mode != 0 && m >= 64 && m * n * (int64_t)sizeof(T) >= (256LL << 20)));
    bool done = wide && launch_colsq_wide<T>(M, m, n, ldm, accumulate, colsq, st);
    if (done) BMM_CHECK_LAUNCH("colsq_wide_kernel");
    done = done || (narrow && cs_variant != 1 &&
                    launch_colsq_tma<T>(M, m, n, ldm, strideM, batch, accumulate, colsq, cs_variant, st));
    if (done) BMM_CHECK_LAUNCH("colsq_tma_kernel");
    const bool vec_ok = !done && !narrow && (reinterpret_cast<uintptr_t>(M) % 16 == 0) && (ldm % W == 0) &&
                        (strideM % W == 0) && n >= W;
    int64_t c_tail = 0;
    if (vec_ok) {
      const int64_t groups = n / W;
      c_tail = groups * W;
      // few column groups (< 8 warps per SM): twice the rows in flight per thread
      static const int rdeep = [] {
        const char* e = getenv("BMM_COLSQ_R");  // A/B switch (16 or 32)
        return e ? atoi(e) : 0;
      }();
      const bool deep = rdeep == 32 || (rdeep == 0 && groups * batch < 148LL * 256 * 2);
      if (deep)
        colsq_vec_kernel<T, 32><<<grid_for(groups * batch, 256, 8, 64), 256, 0, st>>>(
            M, m, n, ldm, strideM, batch, accumulate, colsq);
      else
        colsq_vec_kernel<T, 16><<<grid_for(groups * batch, 256, 8, 64), 256, 0, st>>>(
            M, m, n, ldm, strideM, batch, accumulate, colsq);
      BMM_CHECK_LAUNCH("colsq_vec_kernel");
    }
    if (!done && c_tail < n) {
      if (narrow) {
        colsq_scalar_kernel<T, 32><<<grid_for((n - c_tail) * batch, 64, 32, 64), 64, 0, st>>>(
            M, m, n, c_tail, ldm, strideM, batch, accumulate, colsq);
      } else {
        colsq_scalar_kernel<T, 16><<<grid_for((n - c_tail) * batch, 256, 8, 64), 256, 0, st>>>(
            M, m, n, c_tail, ldm, strideM, batch, accumulate, colsq);
      }
      BMM_CHECK_LAUNCH("colsq_scalar_kernel");
    }
  }
  if (N != nullptr) {
    BMM_REQUIRE(rowsq != nullptr, BMM_E_ARG, "bmm_norms: rowsq is NULL");
    const int64_t rows = n * batch;
    static const int variant = [] {
      // A/B switch for tools/norms_sweep.py: 1 skips the TMA kernels, 2 uses the small-row kernels only
      const char* e = getenv("BMM_ROWSQ_VARIANT");
      return e ? atoi(e) : 0;
    }();
    const bool big = rows * p * (int64_t)sizeof(T) >= (8LL << 20);
    static const int scfg = [] {
      const char* e = getenv("BMM_ROWSQ_STREAM");  // A/B: shape of the streamed kernel
      return e ? atoi(e) : 0;
    }();
    if (variant == 0 && big && launch_rowsq_tma<T>(N, n, p, ldn, strideN, batch, rowsq, st)) {
      BMM_CHECK_LAUNCH("rowsq_tma_kernel");
    } else if (variant == 0 && big && launch_rowsq_stream<T>(N, n, p, ldn, strideN, batch, rowsq, scfg, st)) {
      BMM_CHECK_LAUNCH("rowsq_stream_kernel");
    } else if (variant <= 1 && big && launch_rowsq_leaf<T>(N, n, p, ldn, strideN, batch, rowsq, st)) {
      BMM_CHECK_LAUNCH("rowsq_leaf_kernel");
    } else if (rows < 148LL * 512 && p > 128) {
      const int64_t blocks = std::min<int64_t>(ceil_div(rows, kRowWarps), 148LL * 8 * 64);
      rowsq_warp_kernel<T><<<(unsigned)blocks, 32 * kRowWarps, 0, st>>>(N, n, p, ldn, strideN, batch, rowsq);
      BMM_CHECK_LAUNCH("rowsq_warp_kernel");
    } else {
      rowsq_kernel<T><<<grid_for(rows, 128, 16, 64), 128, 0, st>>>(N, n, p, ldn, strideN, batch, rowsq);
      BMM_CHECK_LAUNCH("rowsq_kernel");
    }
  }
  return BMM_OK;
}

}  // namespace bmm

extern "C" int bmm_norms(int dtype, const void* M, int64_t m, int64_t n, int64_t ldm,
                         int64_t strideM, const void* N, int64_t p, int64_t ldn, int64_t strideN,
                         int64_t batch, int accumulate, double* colsq, double* rowsq,
                         void* stream) {
  using namespace bmm;
  BMM_REQUIRE(m >= 0 && n >= 0 && p >= 0 && batch >= 1, BMM_E_ARG, "bmm_norms: bad shape");
  if (n == 0) return BMM_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == BMM_F64)
    return launch_norms<double>((const double*)M, m, n, ldm, strideM, (const double*)N, p, ldn,
                                strideN, batch, accumulate, colsq, rowsq, st);
  if (dtype == BMM_F32)
    return launch_norms<float>((const float*)M, m, n, ldm, strideM, (const float*)N, p, ldn,
                               strideN, batch, accumulate, colsq, rowsq, st);
  set_error("bmm_norms: unknown dtype %d", dtype);
  return BMM_E_ARG;
}
