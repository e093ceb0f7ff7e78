// K7 (Gram form) -- OPL block-product norms through the Gram identity.
//
//   g_j^2 = || M[:, seg_j] N[seg_j, :] ||_F^2 = < G_M^j , G_N^j >_F
//   G_M^j = M[:, seg_j]^T M[:, seg_j]   (L x L, contraction over the m rows)
//   G_N^j = N[seg_j, :] N[seg_j, :]^T   (L x L, contraction over the p columns)
//
// The reference multiplies out every block, K dgemms of m x n_k x p followed by
// a ddot (block_scores, pkg/src/blockmm/plan.py:176-189): 2 m p n flops.  The
// Gram form costs 2 (m + p) n L flops and reads M and N exactly once -- 128x
// fewer flops at config 4 (n_k = 64, m = p = 16384), 4x at config 5
// (m = p = 256); it wins whenever L < m p / (m + p).
//
// sm_100a has no tcgen05 float64 kind, so the Gram tiles run on the DMMA pipe
// (mma.sync.m8n8k4.f64): a 64 x 64 Gram is 8 x 8 tiles of 8 x 8, of which the
// 36 with t <= u are computed (symmetry).  A and B fragments of X^T X come from
// the SAME staged tile (thread lane holds X[x0 + lane%4][8t + lane/4] for both
// operands), so one k-step is 8 shared loads feeding 36 DMMAs.
//
// CTA per (segment, problem), 4 warps.  The M side streams m x L row pieces
// (256 B per row at L = 64, float32) through a 4-stage cp.async ring, the N
// side L x p (coalesced rows of N); float32 inputs are widened to float64 on
// the fragment load (exact).  Warp w takes k-steps w, w+4 of every 32-position
// stage; the four warps' partial Grams are summed in a fixed order through
// shared memory (deterministic), and warp 0 forms < G_M, G_N > with a fixed
// shuffle tree.  Parity with the reference is to rounding (~1e-15 relative,
// as for the DMMA / int8 segmented GEMMs it replaces); g^2 is clamped at 0 (the
// reference's norm is >= 0 by construction).
#include <cstdlib>

#include "common.cuh"

namespace bmm {

namespace gb {

constexpr int L = 64;          // longest segment (one 64 x 64 Gram panel)
constexpr int WARPS = 4, THREADS = 32 * WARPS;
constexpr int KX = 32;         // contraction positions per stage (8 DMMA k-steps)
constexpr int STAGES = 4;
constexpr int NT = L / 8;      // 8 x 8 tiles per side
constexpr int NTILE = NT * (NT + 1) / 2;   // 36 tiles with t <= u
// M side stage: X[x][a] (x = row of M, a = segment column), row stride SM.
// Fragment (x = 4s + lane%4, a = 8t + lane/4): 4 rows x 8 consecutive elements;
// SM = 72 elements puts the 4 rows on disjoint banks for 4- and 8-byte elements.
constexpr int SM = L + 8;
// N side stage: Y[a][x] (a = segment row of N, x = column of N), row stride SN.
// Fragment (a = 8t + lane/4, x = 4s + lane%4): 8 rows x 4 consecutive; SN = 36.
constexpr int SN = KX + 4;
template <typename T>
constexpr int stage_elems() { return (KX * SM > L * SN) ? KX * SM : L * SN; }
template <typename T>
constexpr int ring_bytes() { return STAGES * stage_elems<T>() * (int)sizeof(T); }
constexpr int GM_BYTES = NTILE * 64 * 8;   // G_M tiles in fragment order
constexpr int RED_BYTES = 2 * NTILE * 64 * 8;  // two warps' partial Grams
template <typename T>
constexpr int smem_bytes() {
  return (ring_bytes<T>() > RED_BYTES ? ring_bytes<T>() : RED_BYTES) + GM_BYTES;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp8(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp4(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename T>
__device__ __forceinline__ void cp_elem(uint32_t dst, const T* src, int bytes) {
  if constexpr (sizeof(T) == 8) cp8(dst, src, bytes);
  else cp4(dst, src, bytes);
}

// Stage `st` of one side: positions x0 .. x0+KX-1 of the contraction.
//   MSIDE: X[x][a] = M[(x0 + x) * ld + col0 + a], x < len, a < Lj
//   else : Y[a][x] = N[(col0 + a) * ld + x0 + x]
// Out-of-range elements are zero-filled (cp.async src-size 0).  `vec`: rows
// are 16-byte aligned at col0 (M) / x0 (N): 16-byte copies, else per element.
template <typename T, bool MSIDE>
__device__ __forceinline__ void load_stage(T* stage, const T* __restrict__ base, int64_t ld, int64_t col0, int Lj,
                                           int64_t x0, int64_t len, bool vec) {
  constexpr int VE = 16 / (int)sizeof(T);  // elements per 16-byte chunk
  const int tid = threadIdx.x;
  if (MSIDE) {
    if (vec) {
      constexpr int CPR = L / VE;  // chunks per row
      for (int q = tid; q < KX * CPR; q += THREADS) {
        const int x = q / CPR, a = (q % CPR) * VE;
        const int64_t gx = x0 + x;
        const int nv = (gx < len) ? max(0, min(VE, Lj - a)) : 0;
        const T* src = nv ? base + gx * ld + col0 + a : base;
        cp16(smem_u32(stage + x * SM + a), src, nv * (int)sizeof(T));
      }
    } else {
      for (int q = tid; q < KX * L; q += THREADS) {
        const int x = q / L, a = q % L;
        const int64_t gx = x0 + x;
        const bool ok = gx < len && a < Lj;
        cp_elem<T>(smem_u32(stage + x * SM + a), ok ? base + gx * ld + col0 + a : base, ok ? (int)sizeof(T) : 0);
      }
    }
  } else {
    if (vec) {
      constexpr int CPR = KX / VE;
      for (int q = tid; q < L * CPR; q += THREADS) {
        const int a = q / CPR, x = (q % CPR) * VE;
        const int64_t gx = x0 + x;
        const int nv = (a < Lj) ? (int)max((int64_t)0, min((int64_t)VE, len - gx)) : 0;
        const T* src = nv ? base + (col0 + a) * ld + gx : base;
        cp16(smem_u32(stage + a * SN + x), src, nv * (int)sizeof(T));
      }
    } else {
      for (int q = tid; q < L * KX; q += THREADS) {
        const int a = q / KX, x = q % KX;
        const int64_t gx = x0 + x;
        const bool ok = a < Lj && gx < len;
        cp_elem<T>(smem_u32(stage + a * SN + x), ok ? base + (col0 + a) * ld + gx : base, ok ? (int)sizeof(T) : 0);
      }
    }
  }
}

// acc + x*x with NumPy's rounding (as norms.cu add_sq: one rounding for float32
// data, where the square is exact; the square then the sum for float64)
template <typename T>
__device__ __forceinline__ double gb_add_sq(double acc, double x) {
  if constexpr (sizeof(T) == 4) return __fma_rn(x, x, acc);
  else return __dadd_rn(acc, __dmul_rn(x, x));
}

// The norm pass fused into the Gram's stream (NORMS): the CTA already reads its
// block's m x L columns of M and L x p rows of N once, in order, so thread a < L
// also runs
//   M side: column a's sequential chain over the rows (NumPy's column_norms,
//           matrix.py:107-109), 32 rows per stage;
//   N side: row a's pairwise tree (matrix.py:112-114) for p = 128 * 2^k: NumPy's
//           leaves are the 128-element runs (8 interleaved accumulators, then
//           ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))), 4 stages each, and the leaves
//           pair in order (a binary counter of pending subtrees).
// Same operations in the same order as norms.cu: bit-identical colsq / rowsq.
constexpr int TREE_LEVELS = 24;

template <typename T>
struct RowTree {
  double r[8];
  double pend[TREE_LEVELS];
  int64_t leaves = 0;
  __device__ __forceinline__ void stage(const T* row, int x0) {  // 32 elements of the row, x0 = stage start
    if ((x0 & 127) == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = 0.0;
    }
#pragma unroll
    for (int x = 0; x < KX; ++x) r[x & 7] = gb_add_sq<T>(r[x & 7], (double)row[x]);
    if ((x0 & 127) == 96) {  // the leaf is complete
      double v = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      int l = 0;
      for (; (leaves >> l) & 1; ++l) v = __dadd_rn(pend[l], v);  // left sibling + right
      pend[l] = v;
      ++leaves;
    }
  }
  __device__ __forceinline__ double root() const {  // leaves = 2^k: one pending subtree
    int l = 0;
    while (!((leaves >> l) & 1)) ++l;
    return pend[l];
  }
};

// One side's Gram (36 upper tiles) over `len` contraction positions, summed
// over the CTA's warps in a fixed order; the result is left in warp 0's acc.
// NORMS: also the side's squared norms of the block (see RowTree) into nrm[0..Lj).
template <typename T, bool MSIDE, bool NORMS = false>
__device__ __forceinline__ void gram_side(double (&acc)[NTILE][2], T* ring, double* red, const T* __restrict__ base,
                                          int64_t ld, int64_t col0, int Lj, int64_t len, bool vec,
                                          double* __restrict__ nrm = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double chain = 0.0;     // M side: column threadIdx.x's sequential sum
  RowTree<T> tree;        // N side: row threadIdx.x's pairwise tree
  const bool owner = NORMS && (int)threadIdx.x < Lj;
#pragma unroll
  for (int q = 0; q < NTILE; ++q) acc[q][0] = acc[q][1] = 0.0;
  const int64_t nst = (len + KX - 1) / KX;
  constexpr int SE = stage_elems<T>();
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nst) load_stage<T, MSIDE>(ring + s * SE, base, ld, col0, Lj, (int64_t)s * KX, len, vec);
    commit();
  }
  for (int64_t i = 0; i < nst; ++i) {
    wait_group<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nx = i + STAGES - 1;
      if (nx < nst) load_stage<T, MSIDE>(ring + (nx % STAGES) * SE, base, ld, col0, Lj, nx * KX, len, vec);
      commit();
    }
    const T* stg = ring + (i % STAGES) * SE;
    if (owner) {
      if (MSIDE) {
#pragma unroll
        for (int x = 0; x < KX; ++x) chain = gb_add_sq<T>(chain, (double)stg[x * SM + threadIdx.x]);
      } else {
        tree.stage(stg + threadIdx.x * SN, (int)(i * KX));
      }
    }
#pragma unroll
    for (int kk = 0; kk < KX / 4 / WARPS; ++kk) {
      const int s = warp + kk * WARPS;  // k-step within the stage
      double f[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int x = 4 * s + (lane & 3), a = 8 * t + (lane >> 2);
        f[t] = (double)(MSIDE ? stg[x * SM + a] : stg[a * SN + x]);
      }
      int q = 0;
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int u = t; u < NT; ++u, ++q) dmma(acc[q], f[t], f[u]);
    }
  }
  if (owner) nrm[threadIdx.x] = MSIDE ? chain : tree.root();
  wait_group<0>();
  __syncthreads();  // the ring is free: reuse it (red) for the cross-warp sum
  // fixed order: (w0 + w2) + (w1 + w3)
  if (warp >= 2) {
    double* r = red + (warp - 2) * NTILE * 64;
#pragma unroll
    for (int q = 0; q < NTILE; ++q) {
      r[q * 64 + 2 * lane] = acc[q][0];
      r[q * 64 + 2 * lane + 1] = acc[q][1];
    }
  }
  __syncthreads();
  if (warp < 2) {
    const double* r = red + warp * NTILE * 64;
#pragma unroll
    for (int q = 0; q < NTILE; ++q) {
      acc[q][0] += r[q * 64 + 2 * lane];
      acc[q][1] += r[q * 64 + 2 * lane + 1];
    }
  }
  __syncthreads();
  if (warp == 1) {
#pragma unroll
    for (int q = 0; q < NTILE; ++q) {
      red[q * 64 + 2 * lane] = acc[q][0];
      red[q * 64 + 2 * lane + 1] = acc[q][1];
    }
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NTILE; ++q) {
      acc[q][0] += red[q * 64 + 2 * lane];
      acc[q][1] += red[q * 64 + 2 * lane + 1];
    }
  }
  __syncthreads();
}

template <typename T, int SIDES>
__global__ void __launch_bounds__(THREADS, 2)
    block_gram_kernel(const T* __restrict__ M, int64_t ldm, int64_t strideM, const T* __restrict__ N, int64_t ldn,
                      int64_t strideN, int64_t m, int64_t p, const int64_t* __restrict__ seg, int64_t nseg,
                      int64_t seg_stride, double* __restrict__ gsq, double* __restrict__ colsq,
                      double* __restrict__ rowsq, int64_t n_stride) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* ring = reinterpret_cast<T*>(smem);
  double* red = reinterpret_cast<double*>(smem);
  double* gm = reinterpret_cast<double*>(smem + (ring_bytes<T>() > RED_BYTES ? ring_bytes<T>() : RED_BYTES));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = blockIdx.x, b = blockIdx.y;
  const int64_t o = seg[b * seg_stride + j];
  const int64_t Lj64 = seg[b * seg_stride + j + 1] - o;
  if (Lj64 <= 0 || Lj64 > L) {  // empty segment: 0; too long: NaN (host guards the engine choice)
    if (threadIdx.x == 0) gsq[b * nseg + j] = Lj64 == 0 ? 0.0 : __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  const int Lj = (int)Lj64;
  const T* Mb = M + b * strideM;
  const T* Nb = N + b * strideN;
  constexpr int VE = 16 / (int)sizeof(T);
  const bool vecM = ((reinterpret_cast<uintptr_t>(Mb) & 15) == 0) && (ldm % VE == 0) && (o % VE == 0);
  const bool vecN = ((reinterpret_cast<uintptr_t>(Nb) & 15) == 0) && (ldn % VE == 0);
  double acc[NTILE][2];
  gram_side<T, true, (SIDES & 1) != 0>(acc, ring, red, Mb, ldm, o, Lj, m, vecM,
                                       (SIDES & 1) ? colsq + b * n_stride + o : nullptr);
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NTILE; ++q) {
      gm[q * 64 + 2 * lane] = acc[q][0];
      gm[q * 64 + 2 * lane + 1] = acc[q][1];
    }
  }
  // (gram_side begins with cp.async into the ring only; gm is a separate region)
  gram_side<T, false, (SIDES & 2) != 0>(acc, ring, red, Nb, ldn, o, Lj, p, vecN,
                                        (SIDES & 2) ? rowsq + b * n_stride + o : nullptr);
  if (warp == 0) {
    double t = 0.0;
    int q = 0;
#pragma unroll
    for (int ta = 0; ta < NT; ++ta)
#pragma unroll
      for (int u = ta; u < NT; ++u, ++q) {
        const double w = (ta == u) ? 1.0 : 2.0;  // an off-diagonal tile stands for its transpose too
        const double v = __dmul_rn(gm[q * 64 + 2 * lane], acc[q][0]) + __dmul_rn(gm[q * 64 + 2 * lane + 1], acc[q][1]);
        t = fma(w, v, t);
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0) gsq[b * nseg + j] = t > 0.0 ? t : 0.0;
  }
}

}  // namespace gb

}  // namespace bmm

using namespace bmm;

template <typename T, int SIDES>
static int block_gram_launch(const void* M, int64_t ldm, int64_t strideM, const void* N, int64_t ldn,
                             int64_t strideN, int64_t m, int64_t nc, const int64_t* seg, int64_t nseg,
                             int64_t seg_stride, int64_t batch, double* gsq, double* colsq, double* rowsq,
                             int64_t n_stride, cudaStream_t st) {
  constexpr int smem = gb::smem_bytes<T>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gb::block_gram_kernel<T, SIDES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((unsigned)nseg, (unsigned)batch);
  gb::block_gram_kernel<T, SIDES><<<grid, gb::THREADS, smem, st>>>(
      (const T*)M, ldm, strideM, (const T*)N, ldn, strideN, m, nc, seg, nseg, seg_stride, gsq, colsq, rowsq, n_stride);
  BMM_CHECK_LAUNCH("block_gram_kernel");
  return BMM_OK;
}

extern "C" int64_t bmm_segsq_gram_max_len(void) { return gb::L; }

extern "C" int bmm_segsq_gram(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N, int64_t ldn,
                              int64_t strideN, int64_t m, int64_t nc, const int64_t* seg, int64_t nseg,
                              int64_t seg_stride, int64_t batch, double* gsq, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && nseg >= 1 && batch >= 1, BMM_E_ARG, "bmm_segsq_gram: bad shape");
  BMM_REQUIRE(M != nullptr && N != nullptr && seg != nullptr && gsq != nullptr, BMM_E_ARG,
              "bmm_segsq_gram: null pointer");
  BMM_REQUIRE(nseg < (1LL << 31) && batch <= 65535, BMM_E_UNSUPPORTED, "bmm_segsq_gram: grid too large");
  cudaStream_t st = as_stream(stream);
  if (dtype == BMM_F64)
    return block_gram_launch<double, 0>(M, ldm, strideM, N, ldn, strideN, m, nc, seg, nseg, seg_stride, batch,
                                            gsq, nullptr, nullptr, 0, st);
  if (dtype == BMM_F32)
    return block_gram_launch<float, 0>(M, ldm, strideM, N, ldn, strideN, m, nc, seg, nseg, seg_stride, batch,
                                           gsq, nullptr, nullptr, 0, st);
  set_error("bmm_segsq_gram: unknown dtype %d", dtype);
  return BMM_E_ARG;
}

extern "C" int bmm_segsq_gram_norms(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                    int64_t ldn, int64_t strideN, int64_t m, int64_t nc, const int64_t* seg,
                                    int64_t nseg, int64_t seg_stride, int64_t batch, double* gsq, double* colsq,
                                    double* rowsq, int64_t n_stride, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && nseg >= 1 && batch >= 1, BMM_E_ARG, "bmm_segsq_gram_norms: bad shape");
  BMM_REQUIRE(M != nullptr && N != nullptr && seg != nullptr && gsq != nullptr && colsq != nullptr &&
                  rowsq != nullptr, BMM_E_ARG, "bmm_segsq_gram_norms: null pointer");
  BMM_REQUIRE(nseg < (1LL << 31) && batch <= 65535, BMM_E_UNSUPPORTED, "bmm_segsq_gram_norms: grid too large");
  BMM_REQUIRE(nc >= 128 && (nc & (nc - 1)) == 0, BMM_E_UNSUPPORTED,
              "bmm_segsq_gram_norms: p must be 128 * 2^k (NumPy's row tree is then perfect)");
  cudaStream_t st = as_stream(stream);
  // A/B (tools/gram_norms_probe.py): BMM_GRAM_NORMS_SIDES=1 fuses only colsq (rowsq untouched)
  static const int sides = [] {
    const char* e = getenv("BMM_GRAM_NORMS_SIDES");
    return e ? atoi(e) : 3;
  }();
#define BMM_GN(TT, S) \
  return block_gram_launch<TT, S>(M, ldm, strideM, N, ldn, strideN, m, nc, seg, nseg, seg_stride, batch, gsq, colsq, \
                                  rowsq, n_stride, st)
  if (dtype == BMM_F64) {
    if (sides == 1) BMM_GN(double, 1);
    BMM_GN(double, 3);
  }
  if (dtype == BMM_F32) {
    if (sides == 1) BMM_GN(float, 1);
    BMM_GN(float, 3);
  }
#undef BMM_GN
  set_error("bmm_segsq_gram_norms: unknown dtype %d", dtype);
  return BMM_E_ARG;
}
