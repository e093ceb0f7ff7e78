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
        for (int j = 0; j < W; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(x[j], x[j]));
      }
    }
    for (; h < m; ++h) {
      V v = __ldcs(reinterpret_cast<const V*>(base + h * ldm));
      double x[W];
      unpack(v, x);
#pragma unroll
      for (int j = 0; j < W; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(x[j], x[j]));
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
      for (int r = 0; r < R; ++r) acc = __dadd_rn(acc, __dmul_rn(v[r], v[r]));
    }
    for (; h < m; ++h) { double x = (double)base[h * ldm]; acc = __dadd_rn(acc, __dmul_rn(x, x)); }
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

template <typename T>
__global__ void __launch_bounds__(32 * kTmaWarps) rowsq_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                                   int64_t total_rows, int L, int log2L,
                                                                   double* __restrict__ rowsq) {
  constexpr int NB = tma_boxes<T>(), SB = tma_stage_bytes<T>();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[kTmaWarps][kTmaStages];
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
  const int U = packed ? 1 : L / 32;              // stages per row
  const int RG = packed ? 32 / L : 1;             // rows per stage
  const int64_t units = packed ? (total_rows + RG - 1) / RG : total_rows;
  const int64_t gw = (int64_t)blockIdx.x * kTmaWarps + w, Wt = (int64_t)gridDim.x * kTmaWarps;
  const int64_t nseq = gw < units ? ((units - 1 - gw) / Wt + 1) * U : 0;
  auto issue = [&](int64_t sq) {
    if (lane == 0 && sq < nseq) {
      const int64_t unit = gw + (sq / U) * Wt;
      const int64_t leaf0 = packed ? unit * 32 : unit * L + (sq % U) * 32;
      uint64_t* bar = &bars[w][sq % kTmaStages];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm_addr(bar)), "r"(SB)
                   : "memory");
      unsigned char* dst = ring + (int64_t)(sq % kTmaStages) * SB;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
                sm_addr(dst + c * kTmaBoxBytes)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(sm_addr(bar)), "r"(c * tma_box_elems<T>()), "r"((int)leaf0)
            : "memory");
    }
  };
  for (int s = 0; s < kTmaStages; ++s) issue(s);
  double part[4];
  for (int64_t sq = 0; sq < nseq; ++sq) {
    const int st = (int)(sq % kTmaStages);
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
    // this lane's leaf: 16 steps of 8 elements
    double r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int s8 = 0; s8 < 16; ++s8) {
      constexpr int CPS = 8 * (int)sizeof(T) / 16;  // 16-byte chunks per step
      const int e0 = 8 * s8;                        // first element of the step
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
            r[4 * h + k] = __dadd_rn(r[4 * h + k], __dmul_rn(d, d));
          }
        } else {
          const double2 a = *reinterpret_cast<const double2*>(p);
          r[2 * h] = __dadd_rn(r[2 * h], __dmul_rn(a.x, a.x));
          r[2 * h + 1] = __dadd_rn(r[2 * h + 1], __dmul_rn(a.y, a.y));
        }
      }
    }
    double t = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    __syncwarp();
    issue(sq + kTmaStages);  // stage st is consumed (all lanes past their loads)
    // perfect tree over the 32 leaves: xor 1, 2, 4, ... (stops at the row width when packed)
    const int lim = packed ? L : 32;
    for (int o = 1; o < lim; o <<= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (packed) {
      const int64_t row0 = (gw + (sq / U) * Wt) * RG;
      const int sub = lane >> log2L;
      if ((lane & (L - 1)) == 0 && row0 + sub < total_rows) rowsq[row0 + sub] = __dadd_rn(0.0, t);
    } else {
      const int u = (int)(sq % U);
      part[u & 3] = t;
      if (u == U - 1) {
        double rt;
        if (U == 2) rt = __dadd_rn(part[0], part[1]);
        else rt = __dadd_rn(__dadd_rn(part[0], part[1]), __dadd_rn(part[2], part[3]));
        if (lane == 0) rowsq[gw + (sq / U) * Wt] = __dadd_rn(0.0, rt);
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
  constexpr int smem = tma_smem<T>();
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(rowsq_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return false;
    attr = true;
  }
  int log2L = 0;
  while ((1 << log2L) < L) ++log2L;
  const int64_t units = L <= 32 ? ceil_div(total_rows, 32 / L) : total_rows;
  const int64_t blocks = std::min<int64_t>(ceil_div(units, kTmaWarps), 148);
  rowsq_tma_kernel<T><<<(unsigned)blocks, 32 * kTmaWarps, smem, st>>>(map, total_rows, L, log2L, rowsq);
  return true;
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
    const bool vec_ok = !narrow && (reinterpret_cast<uintptr_t>(M) % 16 == 0) && (ldm % W == 0) &&
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
    if (c_tail < n) {
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
      const char* e = getenv("BMM_ROWSQ_VARIANT");  // A/B switch for tools/norms_sweep.py
      return e ? atoi(e) : 0;
    }();
    const bool big = rows * p * (int64_t)sizeof(T) >= (8LL << 20);
    if (variant == 0 && big && launch_rowsq_tma<T>(N, n, p, ldn, strideN, batch, rowsq, st)) {
      BMM_CHECK_LAUNCH("rowsq_tma_kernel");
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
