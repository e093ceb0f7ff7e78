// K5 / K7 / K8 / K9 -- float64 contractions on the DMMA tensor pipe.
//
// sm_100a has no tcgen05 float64 kind, so float64 GEMMs use the warp-level
// DMMA path (mma.sync.m8n8k4.f64 -> DMMA.8x8x4).  CTA tile 64x64x16, four
// warps of 32x32, a 4-stage cp.async ring, padded shared-memory rows so the
// A/B fragment loads are bank-conflict free per half-warp.
//
// Reference call sites replaced:
//   C @ D                     estimators.py:175, 253
//   M @ N (exact product)     matrix.py:98-104
//   ||M^k @ N_k||_F^2         plan.py:183-188   (segmented square-sum mode)
//   ||C0 @ D0||_F^2 (pilot)   plan.py:463-464   (segmented square-sum mode)
//   ||exact - approx||_F^2    analysis.py:318-325 (bmm_sqdiff)
// Split-K partials and per-tile square-sums are reduced in a fixed order, so
// every result is run-to-run deterministic.
#include "common.cuh"

namespace bmm {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// CTA tile BM x BN x 16, warp tile WM x WN (FM x FN DMMA 8x8 fragments),
// STAGES-deep cp.async ring.  Shared rows are padded by 4 doubles so the
// fragment loads (row g / column t patterns) are conflict-free per half-warp.
template <int BM_, int BN_, int WM_, int WN_, int STAGES_>
struct DCfg {
  static constexpr int BM = BM_, BN = BN_, BK = 16, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int WARPS_N = BN / WN, WARPS = (BM / WM) * WARPS_N, THREADS = 32 * WARPS;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int A_STR = BK + 4, B_STR = BN + 4;
  static constexpr int A_TILE = BM * A_STR, B_TILE = BK * B_STR;
  static constexpr int SMEM = STAGES * (A_TILE + B_TILE) * 8;
  static_assert((BM * BK / 2) % THREADS == 0 && (BK * BN / 2) % THREADS == 0, "loader split");
};

struct TileArgs {
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  int64_t m, nc;      // rows of A, columns of B
  int64_t m0, n0;     // tile origin
  // gather mode (G): the inner index k is a sketch column t; A[h, t] is read as
  // M[h, col[t]], B[t, f] as N[col[t], f], and each product is scaled by
  // scale[t]^2 -- C @ D without materialising the sketch.
  const int64_t* col = nullptr;
  const double* scale = nullptr;
  // squared mode (SQ): A and B elements are squared and B row k is weighted
  // by wk[k] -- sum_k A[h,k]^2 B[k,f]^2 w_k (elementwise variance, term 1)
  const double* wk = nullptr;
};

// Stage one BK slice [k0, k0+BK) of the A and B tiles; inner indices outside [klo, kend) are zero
// (k0 may start one below klo so that 16-byte copies stay aligned at odd segment starts).
template <class C, bool V16, bool G = false>
__device__ __forceinline__ void load_stage(const TileArgs& ta, int64_t k0, int64_t klo, int64_t kend, double* as,
                                           double* bs) {
  const int tid = threadIdx.x;
  if constexpr (G) {
    // A: one gathered element per 8-byte copy; B: rows of N picked by col[t]
#pragma unroll
    for (int q = 0; q < C::BM * C::BK / C::THREADS; ++q) {
      const int c = tid + C::THREADS * q;
      const int row = c / C::BK, kk = c % C::BK;
      const int64_t gr = ta.m0 + row, gk = k0 + kk;
      const bool ok = gr < ta.m && gk < kend;
      cp_async8(smem_u32(as + row * C::A_STR + kk), ok ? ta.A + gr * ta.lda + ta.col[gk] : ta.A, ok ? 8 : 0);
    }
    if constexpr (V16) {
#pragma unroll
      for (int q = 0; q < C::BK * C::BN / 2 / C::THREADS; ++q) {
        const int c = tid + C::THREADS * q;
        const int row = c / (C::BN / 2), nc2 = (c % (C::BN / 2)) * 2;
        const int64_t gk = k0 + row, gn = ta.n0 + nc2;
        int64_t nv = ta.nc - gn;
        nv = nv < 0 ? 0 : (nv > 2 ? 2 : nv);
        if (gk >= kend || gk < klo) nv = 0;
        const double* src = nv ? ta.B + ta.col[gk] * ta.ldb + gn : ta.B;
        cp_async16(smem_u32(bs + row * C::B_STR + nc2), src, (int)(nv * 8));
      }
    } else {
#pragma unroll
      for (int q = 0; q < C::BK * C::BN / C::THREADS; ++q) {
        const int c = tid + C::THREADS * q;
        const int row = c / C::BN, nn = c % C::BN;
        const int64_t gk = k0 + row, gn = ta.n0 + nn;
        const bool ok = gk < kend && gn < ta.nc;
        cp_async8(smem_u32(bs + row * C::B_STR + nn), ok ? ta.B + ta.col[gk] * ta.ldb + gn : ta.B, ok ? 8 : 0);
      }
    }
  } else if constexpr (V16) {
#pragma unroll
    for (int q = 0; q < C::BM * C::BK / 2 / C::THREADS; ++q) {
      const int c = tid + C::THREADS * q;
      const int row = c >> 3, kc = (c & 7) * 2;
      const int64_t gr = ta.m0 + row, gk = k0 + kc;
      int64_t nv = kend - gk;
      nv = nv < 0 ? 0 : (nv > 2 ? 2 : nv);
      if (gr >= ta.m) nv = 0;
      const double* src = nv ? ta.A + gr * ta.lda + gk : ta.A;
      if (gk < klo) {
        // the pair straddling an odd segment start: zero, then the element at klo
        cp_async8(smem_u32(as + row * C::A_STR + kc), ta.A, 0);
        cp_async8(smem_u32(as + row * C::A_STR + kc + 1), nv == 2 ? src + 1 : ta.A, nv == 2 ? 8 : 0);
      } else {
        cp_async16(smem_u32(as + row * C::A_STR + kc), src, (int)(nv * 8));
      }
    }
#pragma unroll
    for (int q = 0; q < C::BK * C::BN / 2 / C::THREADS; ++q) {
      const int c = tid + C::THREADS * q;
      const int row = c / (C::BN / 2), nc2 = (c % (C::BN / 2)) * 2;
      const int64_t gk = k0 + row, gn = ta.n0 + nc2;
      int64_t nv = ta.nc - gn;
      nv = nv < 0 ? 0 : (nv > 2 ? 2 : nv);
      if (gk >= kend || gk < klo) nv = 0;
      const double* src = nv ? ta.B + gk * ta.ldb + gn : ta.B;
      cp_async16(smem_u32(bs + row * C::B_STR + nc2), src, (int)(nv * 8));
    }
  } else {
#pragma unroll
    for (int q = 0; q < C::BM * C::BK / C::THREADS; ++q) {
      const int c = tid + C::THREADS * q;
      const int row = c / C::BK, kk = c % C::BK;
      const int64_t gr = ta.m0 + row, gk = k0 + kk;
      const bool ok = gr < ta.m && gk < kend && gk >= klo;
      cp_async8(smem_u32(as + row * C::A_STR + kk), ok ? ta.A + gr * ta.lda + gk : ta.A, ok ? 8 : 0);
    }
#pragma unroll
    for (int q = 0; q < C::BK * C::BN / C::THREADS; ++q) {
      const int c = tid + C::THREADS * q;
      const int row = c / C::BN, nn = c % C::BN;
      const int64_t gk = k0 + row, gn = ta.n0 + nn;
      const bool ok = gk < kend && gk >= klo && gn < ta.nc;
      cp_async8(smem_u32(bs + row * C::B_STR + nn), ok ? ta.B + gk * ta.ldb + gn : ta.B, ok ? 8 : 0);
    }
  }
}

// acc += A[m0:+BM, kbeg:kend] @ B[kbeg:kend, n0:+BN]
template <class C, bool V16, bool G = false, bool SQ = false>
__device__ __forceinline__ void mainloop(const TileArgs& ta, int64_t kbeg, int64_t kend, double* smem,
                                         double (&acc)[C::FM][C::FN][2]) {
  double* As = smem;
  double* Bs = smem + C::STAGES * C::A_TILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  // 16-byte A copies need an even start: begin one early at odd kbeg (masked to zero)
  const int64_t kbase = (V16 && !G) ? (kbeg & ~int64_t(1)) : kbeg;
  const int64_t ktiles = (kend - kbase + C::BK - 1) / C::BK;
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < ktiles)
      load_stage<C, V16, G>(ta, kbase + s * C::BK, kbeg, kend, As + s * C::A_TILE, Bs + s * C::B_TILE);
    cp_async_commit();
  }
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    const int64_t nt = kt + C::STAGES - 1;
    if (nt < ktiles) {
      const int ns = (int)(nt % C::STAGES);
      load_stage<C, V16, G>(ta, kbase + nt * C::BK, kbeg, kend, As + ns * C::A_TILE, Bs + ns * C::B_TILE);
    }
    cp_async_commit();
    const int cs = (int)(kt % C::STAGES);
    const double* as = As + cs * C::A_TILE + (wm * C::WM + g) * C::A_STR + t;
    const double* bs = Bs + cs * C::B_TILE + t * C::B_STR + wn * C::WN + g;
#pragma unroll
    for (int kk = 0; kk < C::BK; kk += 4) {
      double a[C::FM], b[C::FN];
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi) a[mi] = as[mi * 8 * C::A_STR + kk];
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) b[ni] = bs[kk * C::B_STR + ni * 8];
      if constexpr (G) {
        // this lane's B fragment row is sketch column t = k + kk + t_lane: scale it by s_t^2
        const int64_t gk = kbase + kt * C::BK + kk + t;
        const double sv = gk < kend ? ta.scale[gk] : 0.0;
        const double s2 = __dmul_rn(sv, sv);
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) b[ni] = __dmul_rn(b[ni], s2);
      }
      if constexpr (SQ) {
        const int64_t gk = kbase + kt * C::BK + kk + t;
        const double wv = (gk >= kbeg && gk < kend) ? ta.wk[gk] : 0.0;
#pragma unroll
        for (int mi = 0; mi < C::FM; ++mi) a[mi] = __dmul_rn(a[mi], a[mi]);
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) b[ni] = __dmul_rn(__dmul_rn(b[ni], b[ni]), wv);
      }
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// K9 -- fused error epilogue (SURVEY.md §8 b2 `err_sq_out_opt`; relative_error,
// analysis.py:318-325): with a reference product `ref` (the exact M @ N) the tile's
// sum of (ref - acc)^2 is taken straight from the accumulator registers (or, under
// split-K, in the ordered split reduction) and written as one partial per tile; the
// product itself need not be stored.  Fixed thread / warp / tile order: deterministic.
struct ErrEpi {
  const double* ref = nullptr;  // batch stride strideR (0: one reference for every problem)
  int64_t ldr = 0, strideR = 0;
  double* part = nullptr;       // batch x parts partial sums
  int write_out = 1;
};

// split-K plan for an inner length known only on the device (compressed sketch):
// the host rule of plan_split (>= 4 k-tiles per split) capped at the launched splits
__device__ __forceinline__ void device_split(int64_t k, int64_t smax, int bk, int64_t& splits, int64_t& kchunk) {
  int64_t s = (k + 4 * bk - 1) / (4 * bk);
  s = s > smax ? smax : (s < 1 ? 1 : s);
  kchunk = (((k + s - 1) / s) + bk - 1) / bk * bk;
  if (kchunk < bk) kchunk = bk;
  splits = (k + kchunk - 1) / kchunk;
  if (splits < 1) splits = 1;
}

template <class C, bool V16, bool G = false, bool SQ = false>
__global__ void __launch_bounds__(C::THREADS) gemm_f64_kernel(const double* __restrict__ A, int64_t lda,
                                                              int64_t strideA, const double* __restrict__ B,
                                                              int64_t ldb, int64_t strideB, int64_t m, int64_t nc,
                                                              int64_t k, int64_t splits, int64_t kchunk,
                                                              double* __restrict__ out, int64_t ldo,
                                                              int64_t strideO, double* __restrict__ part,
                                                              const int64_t* __restrict__ col,
                                                              const double* __restrict__ scale, int64_t w_stride,
                                                              const int64_t* __restrict__ kdev = nullptr,
                                                              const ErrEpi err = ErrEpi{}) {
  extern __shared__ __align__(16) double smem[];
  const int64_t z = blockIdx.z;
  const int64_t b = z / splits, sp = z - b * splits;
  if (kdev != nullptr) {  // inner length from the device: re-plan the split, idle CTAs leave
    k = kdev[b];
    int64_t se;
    device_split(k, splits, C::BK, se, kchunk);
    if (sp >= se) return;
  }
  TileArgs ta{A + b * strideA, lda, B + b * strideB, ldb, m, nc, (int64_t)blockIdx.y * C::BM,
              (int64_t)blockIdx.x * C::BN};
  if constexpr (G) {
    ta.col = col + b * w_stride;
    ta.scale = scale + b * w_stride;
  }
  if constexpr (SQ) ta.wk = scale + b * w_stride;
  const int64_t kbeg = sp * kchunk;
  const int64_t kend = min(k, kbeg + kchunk);
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
    for (int ni = 0; ni < C::FN; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  if (kbeg < kend) mainloop<C, V16, G, SQ>(ta, kbeg, kend, smem, acc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N, g = lane >> 2, t = lane & 3;
  if constexpr (!G && !SQ) {
    if (err.ref != nullptr && splits == 1) {
      // sum of (ref - acc)^2 over the tile: thread order, warp butterfly, warps in order
      const double* rb = err.ref + b * err.strideR;
      double se = 0.0;
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi) {
        const int64_t r = ta.m0 + wm * C::WM + mi * 8 + g;
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) {
          const int64_t c0 = ta.n0 + wn * C::WN + ni * 8 + 2 * t;
          if (r < m && c0 < nc) { const double d = rb[r * err.ldr + c0] - acc[mi][ni][0]; se = fma(d, d, se); }
          if (r < m && c0 + 1 < nc) { const double d = rb[r * err.ldr + c0 + 1] - acc[mi][ni][1]; se = fma(d, d, se); }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      if (lane == 0) smem[warp] = se;  // the mainloop's stages are drained (its closing barrier)
      __syncthreads();
      if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < C::THREADS / 32; ++w) a += smem[w];
        const int64_t tiles = (int64_t)gridDim.x * gridDim.y;
        err.part[b * tiles + (int64_t)blockIdx.y * gridDim.x + blockIdx.x] = a;
      }
      if (!err.write_out) return;
    }
  }
  double* dst;
  int64_t ld;
  if (splits == 1) { dst = out + b * strideO; ld = ldo; }
  else { dst = part + z * m * nc; ld = nc; }
#pragma unroll
  for (int mi = 0; mi < C::FM; ++mi) {
    const int64_t r = ta.m0 + wm * C::WM + mi * 8 + g;
    if (r >= m) continue;
#pragma unroll
    for (int ni = 0; ni < C::FN; ++ni) {
      const int64_t c0 = ta.n0 + wn * C::WN + ni * 8 + 2 * t;
      if (c0 < nc) dst[r * ld + c0] = acc[mi][ni][0];
      if (c0 + 1 < nc) dst[r * ld + c0 + 1] = acc[mi][ni][1];
    }
  }
}

// split-K form of the error epilogue: CTA c of problem b sums its chunk of elements over the
// splits in split order, squares the difference to the reference and writes one partial
constexpr int ERR_THREADS = 256;
__global__ void __launch_bounds__(ERR_THREADS) splitk_reduce_err_kernel(
    const double* __restrict__ part, int64_t splits, int64_t m, int64_t nc, int64_t parts, double* __restrict__ out,
    int64_t ldo, int64_t strideO, const ErrEpi err) {
  __shared__ double red[ERR_THREADS / 32];
  const int64_t b = blockIdx.y, c = blockIdx.x;
  const int64_t per = m * nc;
  const int64_t chunk = (per + parts - 1) / parts;
  const int64_t e0 = c * chunk, e1 = min(per, e0 + chunk);
  const double* rb = err.ref + b * err.strideR;
  double se = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += ERR_THREADS) {
    const double* p = part + b * splits * per + e;
    double acc = p[0];
    for (int64_t s = 1; s < splits; ++s) acc = __dadd_rn(acc, p[s * per]);
    const int64_t r = e / nc, col = e - r * nc;
    if (err.write_out) out[b * strideO + r * ldo + col] = acc;
    const double d = rb[r * err.ldr + col] - acc;
    se = fma(d, d, se);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = se;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < ERR_THREADS / 32; ++w) a += red[w];
    err.part[b * parts + c] = a;
  }
}

__global__ void err_final_kernel(const double* __restrict__ part, int64_t parts, int64_t batch,
                                 double* __restrict__ err_sq) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch;
       b += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int64_t c = 0; c < parts; ++c) a += part[b * parts + c];
    err_sq[b] = a;
  }
}

__global__ void splitk_reduce_kernel(const double* __restrict__ part, int64_t splits, int64_t m, int64_t nc,
                                     int64_t batch, double* __restrict__ out, int64_t ldo, int64_t strideO,
                                     const int64_t* __restrict__ kdev = nullptr, int bk = 16) {
  const int64_t per = m * nc;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < per * batch;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / per, e = g - b * per;
    const double* p = part + b * splits * per + e;
    int64_t se = splits;
    if (kdev != nullptr) {
      int64_t kc;
      device_split(kdev[b], splits, bk, se, kc);
    }
    double acc = p[0];
    for (int64_t s = 1; s < se; ++s) acc = __dadd_rn(acc, p[s * per]);
    const int64_t r = e / nc, c = e - r * nc;
    out[b * strideO + r * ldo + c] = acc;
  }
}

// ---- segmented square sums
template <class C, bool V16, bool G = false>
__global__ void __launch_bounds__(C::THREADS) segsq_f64_kernel(const double* __restrict__ A, int64_t lda,
                                                               int64_t strideA, const double* __restrict__ B,
                                                               int64_t ldb, int64_t strideB, int64_t m,
                                                               int64_t nc, const int64_t* __restrict__ seg,
                                                               int64_t nseg, int64_t seg_stride,
                                                               int64_t chunks, double* __restrict__ part,
                                                               const int64_t* __restrict__ col,
                                                               const double* __restrict__ scale, int64_t w_stride) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double red[C::WARPS];
  const int64_t z = blockIdx.z;
  const int64_t b = z / chunks, ch = z - b * chunks;
  const int64_t per = (nseg + chunks - 1) / chunks;
  const int64_t j0 = ch * per, j1 = min(nseg, j0 + per);
  TileArgs ta{A + b * strideA, lda, B + b * strideB, ldb, m, nc, (int64_t)blockIdx.y * C::BM,
              (int64_t)blockIdx.x * C::BN};
  if constexpr (G) {
    ta.col = col + b * w_stride;
    ta.scale = scale + b * w_stride;
  }
  const int64_t tiles = (int64_t)gridDim.x * gridDim.y;
  const int64_t tile = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  // one segment per CTA (few, unequal segments): longest first, so the tail of
  // the grid is short segments (rank = # longer segments, ties by index)
  __shared__ int64_t lpt_j;
  const bool lpt = (chunks == nseg) && nseg <= 128;
  if (lpt) {
    const int64_t* sb = seg + b * seg_stride;
    if (threadIdx.x == 0) lpt_j = -1;
    __syncthreads();
    for (int64_t jj = threadIdx.x; jj < nseg; jj += C::THREADS) {
      const int64_t lj = sb[jj + 1] - sb[jj];
      int64_t rank = 0;
      for (int64_t i = 0; i < nseg; ++i) {
        const int64_t li = sb[i + 1] - sb[i];
        rank += (li > lj) || (li == lj && i < jj);
      }
      if (rank == ch) lpt_j = jj;
    }
    __syncthreads();
  }
  for (int64_t jl = j0; jl < j1; ++jl) {
    const int64_t j = lpt ? lpt_j : jl;
    const int64_t kbeg = seg[b * seg_stride + j], kend = seg[b * seg_stride + j + 1];
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    if (kbeg < kend) mainloop<C, V16, G>(ta, kbeg, kend, smem, acc);
    double sq = 0.0;
#pragma unroll
    for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) {
        sq = fma(acc[mi][ni][0], acc[mi][ni][0], sq);
        sq = fma(acc[mi][ni][1], acc[mi][ni][1], sq);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = red[0];
      for (int w = 1; w < C::WARPS; ++w) tot += red[w];
      part[(b * nseg + j) * tiles + tile] = tot;
    }
    __syncthreads();
  }
}

__global__ void segsq_reduce_kernel(const double* __restrict__ part, int64_t tiles, int64_t total,
                                    double* __restrict__ gsq) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const double* p = part + g * tiles;
    double acc = 0.0;
    for (int64_t i = 0; i < tiles; ++i) acc += p[i];
    gsq[g] = acc;
  }
}

// ---- segmented weighted squares into a matrix: part[ch] = sum_{j in chunk ch} w_j (A_j B_j)^2
// (elementwise variance, term 2: sum_k (M^k N_k)^2 / c_k;  analysis.py:82-89)
template <class C, bool V16>
__global__ void __launch_bounds__(C::THREADS) segsq_mat_kernel(const double* __restrict__ A, int64_t lda,
                                                               const double* __restrict__ B, int64_t ldb, int64_t m,
                                                               int64_t nc, const int64_t* __restrict__ seg,
                                                               int64_t nseg, const double* __restrict__ wseg,
                                                               int64_t chunks, double* __restrict__ part) {
  extern __shared__ __align__(16) double smem[];
  const int64_t ch = blockIdx.z;
  const int64_t per = (nseg + chunks - 1) / chunks;
  const int64_t j0 = ch * per, j1 = min(nseg, j0 + per);
  TileArgs ta{A, lda, B, ldb, m, nc, (int64_t)blockIdx.y * C::BM, (int64_t)blockIdx.x * C::BN};
  double sq[C::FM][C::FN][2];
#pragma unroll
  for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
    for (int ni = 0; ni < C::FN; ++ni) sq[mi][ni][0] = sq[mi][ni][1] = 0.0;
  for (int64_t j = j0; j < j1; ++j) {
    const double w = wseg[j];
    const int64_t kbeg = seg[j], kend = seg[j + 1];
    if (w == 0.0 || kbeg >= kend) continue;
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    mainloop<C, V16>(ta, kbeg, kend, smem, acc);
#pragma unroll
    for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) {
        sq[mi][ni][0] = fma(w, acc[mi][ni][0] * acc[mi][ni][0], sq[mi][ni][0]);
        sq[mi][ni][1] = fma(w, acc[mi][ni][1] * acc[mi][ni][1], sq[mi][ni][1]);
      }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N, g = lane >> 2, t = lane & 3;
  double* dst = part + ch * m * nc;
#pragma unroll
  for (int mi = 0; mi < C::FM; ++mi) {
    const int64_t r = ta.m0 + wm * C::WM + mi * 8 + g;
    if (r >= m) continue;
#pragma unroll
    for (int ni = 0; ni < C::FN; ++ni) {
      const int64_t c0 = ta.n0 + wn * C::WN + ni * 8 + 2 * t;
      if (c0 < nc) dst[r * nc + c0] = sq[mi][ni][0];
      if (c0 + 1 < nc) dst[r * nc + c0 + 1] = sq[mi][ni][1];
    }
  }
}

// out[r, c] -= sum over chunks of part[ch][r, c], chunks in order
__global__ void sub_chunks_kernel(const double* __restrict__ part, int64_t chunks, int64_t m, int64_t nc,
                                  double* __restrict__ out, int64_t ldo) {
  const int64_t per = m * nc;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.x * blockDim.x) {
    double acc = part[e];
    for (int64_t c = 1; c < chunks; ++c) acc = __dadd_rn(acc, part[c * per + e]);
    const int64_t r = e / nc, c = e - r * nc;
    out[r * ldo + c] = __dsub_rn(out[r * ldo + c], acc);
  }
}

// variance weights: w_col[i] = 1 / (c_k p_i) where p_i > 0 and c_k > 0 (else 0),
// w_blk[k] = 1 / c_k (else 0); bad[0] = first block with a contributing column
// (sqrt(colsq) sqrt(rowsq) > 0) of zero probability, as K - k (0: none)   analysis.py:77-79
__global__ void variance_weights_kernel(const double* __restrict__ probs, const double* __restrict__ colsq,
                                        const double* __restrict__ rowsq, const int64_t* __restrict__ offsets,
                                        int64_t K, const double* __restrict__ budgets, double* __restrict__ w_col,
                                        double* __restrict__ w_blk, int64_t* __restrict__ bad) {
  const int64_t n = offsets[K];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = K;  // block k with offsets[k] <= i < offsets[k+1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (offsets[mid] <= i) lo = mid; else hi = mid;
    }
    const double p = probs[i], ck = budgets[lo];
    w_col[i] = (p > 0.0 && ck > 0.0) ? __ddiv_rn(1.0, __dmul_rn(ck, p)) : 0.0;
    if (!(p > 0.0) && __dmul_rn(__dsqrt_rn(colsq[i]), __dsqrt_rn(rowsq[i])) > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)(K - lo));  // K - first block
    if (i == offsets[lo]) w_blk[lo] = ck > 0.0 ? __ddiv_rn(1.0, ck) : 0.0;
  }
}

// per block sum over p_i > 0 of sc_i^2 / p_i  (expected_sq_error term 1,
// analysis.py:109); warp per block, fixed lane order
__global__ void block_term1_kernel(const double* __restrict__ probs, const double* __restrict__ colsq,
                                   const double* __restrict__ rowsq, const int64_t* __restrict__ offsets, int64_t K,
                                   double* __restrict__ out, int64_t* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < K;
       k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double acc = 0.0;
    for (int64_t i = offsets[k] + lane; i < offsets[k + 1]; i += 32) {
      const double p = probs[i];
      const double sc = __dmul_rn(__dsqrt_rn(colsq[i]), __dsqrt_rn(rowsq[i]));
      if (p > 0.0) acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(sc, sc), p));
      else if (sc > 0.0) atomicMax(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)(K - k));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) out[k] = acc;
  }
}

// ---- squared difference / squared norm (error evaluation)
constexpr int SQ_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(SQ_THREADS) sqdiff_kernel(const T* __restrict__ X, int64_t ldx, int64_t strideX,
                                                            const T* __restrict__ Y, int64_t ldy, int64_t strideY,
                                                            int64_t m, int64_t nc, int64_t parts,
                                                            double* __restrict__ part) {
  __shared__ double red[2][SQ_THREADS / 32];
  const int64_t b = blockIdx.y, c = blockIdx.x;
  const int64_t total = m * nc;
  const int64_t chunk = (total + parts - 1) / parts;
  const int64_t e0 = c * chunk, e1 = min(total, e0 + chunk);
  const T* xb = X + b * strideX;
  const T* yb = Y ? Y + b * strideY : nullptr;
  double se = 0.0, sr = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += SQ_THREADS) {
    const int64_t r = e / nc, col = e - r * nc;
    const double x = (double)xb[r * ldx + col];
    const double y = yb ? (double)yb[r * ldy + col] : 0.0;
    const double d = x - y;
    se = fma(d, d, se);
    sr = fma(x, x, sr);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    se += __shfl_xor_sync(0xffffffffu, se, o);
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = se; red[1][threadIdx.x >> 5] = sr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, r = 0.0;
    for (int w = 0; w < SQ_THREADS / 32; ++w) { a += red[0][w]; r += red[1][w]; }
    part[(b * parts + c) * 2] = a;
    part[(b * parts + c) * 2 + 1] = r;
  }
}

__global__ void sqdiff_final_kernel(const double* __restrict__ part, int64_t parts, int64_t batch,
                                    double* __restrict__ err) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch;
       b += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0, r = 0.0;
    for (int64_t c = 0; c < parts; ++c) { a += part[(b * parts + c) * 2]; r += part[(b * parts + c) * 2 + 1]; }
    err[2 * b] = a;
    err[2 * b + 1] = r;
  }
}

inline int64_t sq_parts(int64_t m, int64_t nc, int64_t batch) {
  int64_t parts = ceil_div(m * nc, 4096);
  int64_t target = ceil_div(148 * 8, batch);
  if (parts > target) parts = target;
  if (parts > 1024) parts = 1024;
  if (parts < 1) parts = 1;
  return parts;
}

struct SplitPlan {
  int64_t splits, kchunk;
};

// ---- tile-configuration variants (selected once; bmm_gemm_f64_set_variant for tuning)
using DV0 = DCfg<64, 64, 32, 32, 3>;
using DV1 = DCfg<64, 128, 32, 64, 3>;
using DV2 = DCfg<128, 64, 64, 32, 3>;
using DV3 = DCfg<128, 128, 64, 32, 3>;
using DV4 = DCfg<128, 128, 32, 64, 3>;
using DV5 = DCfg<64, 64, 32, 32, 4>;
using DV6 = DCfg<128, 64, 32, 32, 3>;
using DV7 = DCfg<40, 40, 40, 40, 3>;  // one warp, 5x5 fragments: small outputs (200 = 5 x 40, no padding)
constexpr int kVariants = 8;
static int g_variant = 2;      // C.D / exact-product tiles: 128x64, 4 warps of 64x32 (tools/tune_dmma.py)
static int g_seg_variant = 5;  // segmented square sums: 64x64, 4 warps of 32x32, 4 stages (tools/tune_dmma.py)

struct VariantInfo {
  int BM, BN, BK, threads, smem, occ;
};

template <class C>
static VariantInfo info_of() {
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(gemm_f64_kernel<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(gemm_f64_kernel<C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(segsq_f64_kernel<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(segsq_f64_kernel<C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, gemm_f64_kernel<C, true>, C::THREADS, C::SMEM) !=
            cudaSuccess || o < 1)
      o = 1;
    occ = o;
  }
  return VariantInfo{C::BM, C::BN, C::BK, C::THREADS, C::SMEM, occ};
}

static VariantInfo variant_info(int v) {
  switch (v) {
    case 1: return info_of<DV1>();
    case 2: return info_of<DV2>();
    case 3: return info_of<DV3>();
    case 4: return info_of<DV4>();
    case 5: return info_of<DV5>();
    case 6: return info_of<DV6>();
    case 7: return info_of<DV7>();
    default: return info_of<DV0>();
  }
}

inline SplitPlan plan_split(const VariantInfo& vi, int64_t m, int64_t nc, int64_t k, int64_t batch) {
  const int64_t tiles = ceil_div(m, vi.BM) * ceil_div(nc, vi.BN) * batch;
  int64_t splits = ((int64_t)vi.occ * 148) / tiles;  // fill one wave without spilling into a second
  const int64_t max_splits = ceil_div(k, 4 * vi.BK);        // at least 64 of k per split
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  if (batch * splits > 65535) splits = 65535 / batch;
  int64_t kchunk = ceil_div(ceil_div(k, splits), vi.BK) * vi.BK;
  splits = ceil_div(k, kchunk);
  if (splits < 1) splits = 1;
  return {splits, kchunk};
}

inline int64_t segsq_chunks(const VariantInfo& vi, int64_t m, int64_t nc, int64_t nseg, int64_t batch) {
  const int64_t tiles = ceil_div(m, vi.BM) * ceil_div(nc, vi.BN) * batch;
  int64_t ch = ((int64_t)vi.occ * 148) / tiles;
  if (ch > nseg) ch = nseg;
  if (ch < 1) ch = 1;
  if (batch * ch > 65535) ch = 65535 / batch;
  return ch;
}

template <class C>
static void launch_gemm(bool v16, dim3 grid, cudaStream_t st, const double* A, int64_t lda, int64_t strideA,
                        const double* B, int64_t ldb, int64_t strideB, int64_t m, int64_t nc, int64_t k,
                        const SplitPlan& sp, double* out, int64_t ldo, int64_t strideO, double* part,
                        const int64_t* col = nullptr, const double* scale = nullptr, int64_t w_stride = 0,
                        const int64_t* kdev = nullptr, const ErrEpi err = ErrEpi{}) {
  if (col != nullptr) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_f64_kernel<C, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      cudaFuncSetAttribute(gemm_f64_kernel<C, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      attr = true;
    }
    if (v16)
      gemm_f64_kernel<C, true, true><<<grid, C::THREADS, C::SMEM, st>>>(A, lda, strideA, B, ldb, strideB, m, nc, k,
                                                                       sp.splits, sp.kchunk, out, ldo, strideO, part,
                                                                       col, scale, w_stride);
    else
      gemm_f64_kernel<C, false, true><<<grid, C::THREADS, C::SMEM, st>>>(A, lda, strideA, B, ldb, strideB, m, nc, k,
                                                                        sp.splits, sp.kchunk, out, ldo, strideO, part,
                                                                        col, scale, w_stride);
    return;
  }
  if (v16)
    gemm_f64_kernel<C, true><<<grid, C::THREADS, C::SMEM, st>>>(A, lda, strideA, B, ldb, strideB, m, nc, k, sp.splits,
                                                               sp.kchunk, out, ldo, strideO, part, nullptr, nullptr, 0,
                                                               kdev, err);
  else
    gemm_f64_kernel<C, false><<<grid, C::THREADS, C::SMEM, st>>>(A, lda, strideA, B, ldb, strideB, m, nc, k, sp.splits,
                                                                sp.kchunk, out, ldo, strideO, part, nullptr, nullptr, 0,
                                                                kdev, err);
}

template <class C>
static void launch_segsq(bool v16, dim3 grid, cudaStream_t st, const double* A, int64_t lda, int64_t strideA,
                         const double* B, int64_t ldb, int64_t strideB, int64_t m, int64_t nc, const int64_t* seg,
                         int64_t nseg, int64_t seg_stride, int64_t chunks, double* part, const int64_t* col = nullptr,
                         const double* scale = nullptr, int64_t w_stride = 0) {
  if (col != nullptr) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(segsq_f64_kernel<C, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      cudaFuncSetAttribute(segsq_f64_kernel<C, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      attr = true;
    }
    if (v16)
      segsq_f64_kernel<C, true, true><<<grid, C::THREADS, C::SMEM, st>>>(A, lda, strideA, B, ldb, strideB, m, nc, seg,
                                                                        nseg, seg_stride, chunks, part, col, scale,
                                                                        w_stride);
    else
      segsq_f64_kernel<C, false, true><<<grid, C::THREADS, C::SMEM, st>>>(A, lda, strideA, B, ldb, strideB, m, nc,
                                                                         seg, nseg, seg_stride, chunks, part, col,
                                                                         scale, w_stride);
    return;
  }
  if (v16)
    segsq_f64_kernel<C, true><<<grid, C::THREADS, C::SMEM, st>>>(A, lda, strideA, B, ldb, strideB, m, nc, seg, nseg,
                                                                seg_stride, chunks, part, nullptr, nullptr, 0);
  else
    segsq_f64_kernel<C, false><<<grid, C::THREADS, C::SMEM, st>>>(A, lda, strideA, B, ldb, strideB, m, nc, seg, nseg,
                                                                 seg_stride, chunks, part, nullptr, nullptr, 0);
}

}  // namespace bmm

using namespace bmm;

extern "C" int bmm_gemm_f64_set_variant(int gemm_variant, int segsq_variant) {
  BMM_REQUIRE(gemm_variant >= 0 && gemm_variant < kVariants && segsq_variant >= 0 && segsq_variant < kVariants,
              BMM_E_ARG, "bmm_gemm_f64_set_variant: unknown variant %d/%d", gemm_variant, segsq_variant);
  g_variant = gemm_variant;
  g_seg_variant = segsq_variant;
  return BMM_OK;
}

// Small outputs (e.g. the Monte Carlo engine's 200 x 200 products): the
// 40 x 40 single-warp tiles when they waste much less padding than the default
static int pick_variant(int64_t m, int64_t nc) {
  if (g_variant != 2 || m > 256 || nc > 256) return g_variant;
  const int64_t a40 = ceil_div(m, 40) * 40 * ceil_div(nc, 40) * 40;
  const int64_t a2 = ceil_div(m, 128) * 128 * ceil_div(nc, 64) * 64;
  return 5 * a40 < 4 * a2 ? 7 : g_variant;
}

extern "C" int64_t bmm_gemm_f64_workspace(int64_t m, int64_t nc, int64_t k, int64_t batch) {
  SplitPlan sp = plan_split(variant_info(pick_variant(m, nc)), m, nc, k, batch);
  return sp.splits > 1 ? sp.splits * batch * m * nc * 8 : 0;
}

static int gemm_impl(const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb, int64_t strideB,
                     int64_t m, int64_t nc, int64_t k, int64_t batch, double* out, int64_t ldo, int64_t strideO,
                     void* ws, int64_t ws_bytes, cudaStream_t st, const int64_t* col, const double* scale,
                     int64_t w_stride, const int64_t* kdev = nullptr, ErrEpi err = ErrEpi{},
                     double* err_sq = nullptr) {
  if (m == 0 || nc == 0) return BMM_OK;
  if (k == 0) {
    for (int64_t b = 0; b < batch; ++b)
      if (cudaMemset2DAsync(out + b * strideO, ldo * 8, 0, nc * 8, m, st) != cudaSuccess) {
        set_error("bmm_gemm_f64: memset failed");
        return BMM_E_CUDA;
      }
    return BMM_OK;
  }
  const int variant = pick_variant(m, nc);
  const VariantInfo vi = variant_info(variant);
  SplitPlan sp = plan_split(vi, m, nc, k, batch);
  int64_t need = sp.splits > 1 ? sp.splits * batch * m * nc * 8 : 0;
  int64_t err_parts = 0;
  if (err.ref != nullptr) {
    // one partial per tile (fused epilogue) or per reduction CTA (split-K), after the split partials
    err_parts = sp.splits > 1 ? sq_parts(m, nc, batch) : ceil_div(m, vi.BM) * ceil_div(nc, vi.BN);
    err.part = (double*)((char*)ws + need);
    need += batch * err_parts * 8;
  }
  BMM_REQUIRE(ws_bytes >= need && (need == 0 || ws != nullptr), BMM_E_ARG,
              "bmm_gemm_f64: workspace too small (%lld < %lld)", (long long)ws_bytes, (long long)need);
  BMM_REQUIRE(ceil_div(m, vi.BM) <= 65535, BMM_E_UNSUPPORTED, "bmm_gemm_f64: m too large");
  // 16-byte copies need aligned rows; in gather mode only B's rows are copied in 16-byte chunks
  const bool v16 = (col != nullptr || ((reinterpret_cast<uintptr_t>(A) % 16 == 0) && lda % 2 == 0 && strideA % 2 == 0)) &&
                   (reinterpret_cast<uintptr_t>(B) % 16 == 0) && ldb % 2 == 0 && strideB % 2 == 0;
  dim3 grid((unsigned)ceil_div(nc, vi.BN), (unsigned)ceil_div(m, vi.BM), (unsigned)(batch * sp.splits));
  double* part = (double*)ws;
#define BMM_GEMM_CASE(V)                                                                                       \
  launch_gemm<V>(v16, grid, st, A, lda, strideA, B, ldb, strideB, m, nc, k, sp, out, ldo, strideO, part, col, \
                 scale, w_stride, kdev, err)
  switch (variant) {
    case 1: BMM_GEMM_CASE(DV1); break;
    case 2: BMM_GEMM_CASE(DV2); break;
    case 3: BMM_GEMM_CASE(DV3); break;
    case 4: BMM_GEMM_CASE(DV4); break;
    case 5: BMM_GEMM_CASE(DV5); break;
    case 6: BMM_GEMM_CASE(DV6); break;
    case 7: BMM_GEMM_CASE(DV7); break;
    default: BMM_GEMM_CASE(DV0);
  }
#undef BMM_GEMM_CASE
  BMM_CHECK_LAUNCH("gemm_f64_kernel");
  if (sp.splits > 1 && err.ref != nullptr) {
    dim3 rgrid((unsigned)err_parts, (unsigned)batch);
    splitk_reduce_err_kernel<<<rgrid, ERR_THREADS, 0, st>>>((const double*)ws, sp.splits, m, nc, err_parts, out, ldo,
                                                            strideO, err);
    BMM_CHECK_LAUNCH("splitk_reduce_err_kernel");
  } else if (sp.splits > 1) {
    splitk_reduce_kernel<<<grid_for(m * nc * batch, 256), 256, 0, st>>>((const double*)ws, sp.splits, m, nc,
                                                                        batch, out, ldo, strideO, kdev, vi.BK);
    BMM_CHECK_LAUNCH("splitk_reduce_kernel");
  }
  if (err.ref != nullptr) {
    err_final_kernel<<<grid_for(batch, 128), 128, 0, st>>>(err.part, err_parts, batch, err_sq);
    BMM_CHECK_LAUNCH("err_final_kernel");
  }
  return BMM_OK;
}

extern "C" int64_t bmm_gemm_f64_err_workspace(int64_t m, int64_t nc, int64_t k, int64_t batch) {
  const VariantInfo vi = variant_info(pick_variant(m, nc));
  SplitPlan sp = plan_split(vi, m, nc, k, batch);
  const int64_t parts = sp.splits > 1 ? sq_parts(m, nc, batch) : ceil_div(m, vi.BM) * ceil_div(nc, vi.BN);
  return (sp.splits > 1 ? sp.splits * batch * m * nc * 8 : 0) + batch * parts * 8 + 256;
}

extern "C" int bmm_gemm_f64_err(const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                                int64_t strideB, int64_t m, int64_t nc, int64_t k, int64_t batch, const double* ref,
                                int64_t ldr, int64_t strideR, double* out_opt, int64_t ldo, int64_t strideO,
                                double* err_sq, void* ws, int64_t ws_bytes, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && k >= 1 && batch >= 1, BMM_E_ARG, "bmm_gemm_f64_err: bad shape");
  BMM_REQUIRE(ref != nullptr && err_sq != nullptr && ldr >= nc, BMM_E_ARG, "bmm_gemm_f64_err: reference and output required");
  ErrEpi err;
  err.ref = ref;
  err.ldr = ldr;
  err.strideR = strideR;
  err.write_out = out_opt != nullptr ? 1 : 0;
  return gemm_impl(A, lda, strideA, B, ldb, strideB, m, nc, k, batch, out_opt, ldo, strideO, ws, ws_bytes,
                   as_stream(stream), nullptr, nullptr, 0, nullptr, err, err_sq);
}

extern "C" int bmm_gemm_f64(const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                            int64_t strideB, int64_t m, int64_t nc, int64_t k, int64_t batch, double* out,
                            int64_t ldo, int64_t strideO, void* ws, int64_t ws_bytes, void* stream) {
  BMM_REQUIRE(m >= 0 && nc >= 0 && k >= 0 && batch >= 1, BMM_E_ARG, "bmm_gemm_f64: bad shape");
  return gemm_impl(A, lda, strideA, B, ldb, strideB, m, nc, k, batch, out, ldo, strideO, ws, ws_bytes,
                   as_stream(stream), nullptr, nullptr, 0);
}

extern "C" int bmm_gemm_f64_dk(const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                               int64_t strideB, int64_t m, int64_t nc, int64_t k_max, const int64_t* k_dev,
                               int64_t batch, double* out, int64_t ldo, int64_t strideO, void* ws, int64_t ws_bytes,
                               void* stream) {
  BMM_REQUIRE(m >= 0 && nc >= 0 && k_max >= 1 && batch >= 1 && k_dev != nullptr, BMM_E_ARG,
              "bmm_gemm_f64_dk: bad shape");
  return gemm_impl(A, lda, strideA, B, ldb, strideB, m, nc, k_max, batch, out, ldo, strideO, ws, ws_bytes,
                   as_stream(stream), nullptr, nullptr, 0, k_dev);
}

extern "C" int bmm_gemm_f64_gather(const double* M, int64_t ldm, int64_t strideM, const double* N, int64_t ldn,
                                   int64_t strideN, int64_t m, int64_t nc, const int64_t* column,
                                   const double* scale, int64_t W, int64_t w_stride, int64_t batch, double* out,
                                   int64_t ldo, int64_t strideO, void* ws, int64_t ws_bytes, void* stream) {
  BMM_REQUIRE(m >= 0 && nc >= 0 && W >= 0 && batch >= 1 && column != nullptr && scale != nullptr, BMM_E_ARG,
              "bmm_gemm_f64_gather: bad arguments");
  return gemm_impl(M, ldm, strideM, N, ldn, strideN, m, nc, W, batch, out, ldo, strideO, ws, ws_bytes,
                   as_stream(stream), column, scale, w_stride);
}

extern "C" int64_t bmm_segsq_f64_workspace(int64_t m, int64_t nc, int64_t nseg, int64_t batch) {
  const VariantInfo vi = variant_info(g_seg_variant);
  return ceil_div(m, vi.BM) * ceil_div(nc, vi.BN) * nseg * batch * 8;
}

static int segsq_impl(const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb, int64_t strideB,
                      int64_t m, int64_t nc, const int64_t* seg, int64_t nseg, int64_t seg_stride, int64_t batch,
                      double* gsq, void* ws, int64_t ws_bytes, cudaStream_t st, const int64_t* col,
                      const double* scale, int64_t w_stride) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && nseg >= 1 && batch >= 1, BMM_E_ARG, "bmm_segsq_f64: bad shape");
  const VariantInfo vi = variant_info(g_seg_variant);
  const int64_t tiles = ceil_div(m, vi.BM) * ceil_div(nc, vi.BN);
  const int64_t need = tiles * nseg * batch * 8;
  BMM_REQUIRE(ws_bytes >= need && ws != nullptr, BMM_E_ARG, "bmm_segsq_f64: workspace too small");
  BMM_REQUIRE(ceil_div(m, vi.BM) <= 65535, BMM_E_UNSUPPORTED, "bmm_segsq_f64: m too large");
  // partition blocks (no gather): one segment per CTA, the block scheduler balances unequal
  // segments; gathered pilot segments are short, so a CTA walks several
  int64_t chunks = col == nullptr ? nseg : segsq_chunks(vi, m, nc, nseg, batch);
  if (batch * chunks > 65535) chunks = 65535 / batch;
  const bool v16 = (col != nullptr || ((reinterpret_cast<uintptr_t>(A) % 16 == 0) && lda % 2 == 0 && strideA % 2 == 0)) &&
                   (reinterpret_cast<uintptr_t>(B) % 16 == 0) && ldb % 2 == 0 && strideB % 2 == 0;
  dim3 grid((unsigned)ceil_div(nc, vi.BN), (unsigned)ceil_div(m, vi.BM), (unsigned)(batch * chunks));
  double* part = (double*)ws;
#define BMM_SEG_CASE(V)                                                                                             \
  launch_segsq<V>(v16, grid, st, A, lda, strideA, B, ldb, strideB, m, nc, seg, nseg, seg_stride, chunks, part, col, \
                  scale, w_stride)
  switch (g_seg_variant) {
    case 1: BMM_SEG_CASE(DV1); break;
    case 2: BMM_SEG_CASE(DV2); break;
    case 3: BMM_SEG_CASE(DV3); break;
    case 4: BMM_SEG_CASE(DV4); break;
    case 5: BMM_SEG_CASE(DV5); break;
    case 6: BMM_SEG_CASE(DV6); break;
    default: BMM_SEG_CASE(DV0);
  }
#undef BMM_SEG_CASE
  BMM_CHECK_LAUNCH("segsq_f64_kernel");
  segsq_reduce_kernel<<<grid_for(nseg * batch, 128), 128, 0, st>>>((const double*)ws, tiles, nseg * batch, gsq);
  BMM_CHECK_LAUNCH("segsq_reduce_kernel");
  return BMM_OK;
}

extern "C" int bmm_segsq_f64(const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                             int64_t strideB, int64_t m, int64_t nc, const int64_t* seg, int64_t nseg,
                             int64_t seg_stride, int64_t batch, double* gsq, void* ws, int64_t ws_bytes,
                             void* stream) {
  return segsq_impl(A, lda, strideA, B, ldb, strideB, m, nc, seg, nseg, seg_stride, batch, gsq, ws, ws_bytes,
                    as_stream(stream), nullptr, nullptr, 0);
}

extern "C" int bmm_segsq_f64_gather(const double* M, int64_t ldm, int64_t strideM, const double* N, int64_t ldn,
                                    int64_t strideN, int64_t m, int64_t nc, const int64_t* column,
                                    const double* scale, int64_t w_stride, const int64_t* seg, int64_t nseg,
                                    int64_t seg_stride, int64_t batch, double* gsq, void* ws, int64_t ws_bytes,
                                    void* stream) {
  BMM_REQUIRE(column != nullptr && scale != nullptr, BMM_E_ARG, "bmm_segsq_f64_gather: bad arguments");
  return segsq_impl(M, ldm, strideM, N, ldn, strideN, m, nc, seg, nseg, seg_stride, batch, gsq, ws, ws_bytes,
                    as_stream(stream), column, scale, w_stride);
}

extern "C" int64_t bmm_sqdiff_workspace(int64_t m, int64_t nc, int64_t batch) {
  return sq_parts(m, nc, batch) * batch * 2 * 8;
}

extern "C" int bmm_sqdiff(int dtype, const void* X, int64_t ldx, int64_t strideX, const void* Y, int64_t ldy,
                          int64_t strideY, int64_t m, int64_t nc, int64_t batch, double* err, void* ws,
                          int64_t ws_bytes, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && batch >= 1 && batch <= 65535, BMM_E_ARG, "bmm_sqdiff: bad shape");
  const int64_t parts = sq_parts(m, nc, batch);
  BMM_REQUIRE(ws_bytes >= parts * batch * 16 && ws != nullptr, BMM_E_ARG, "bmm_sqdiff: workspace too small");
  cudaStream_t st = as_stream(stream);
  dim3 grid((unsigned)parts, (unsigned)batch);
  if (dtype == BMM_F64)
    sqdiff_kernel<double><<<grid, SQ_THREADS, 0, st>>>((const double*)X, ldx, strideX, (const double*)Y, ldy,
                                                       strideY, m, nc, parts, (double*)ws);
  else if (dtype == BMM_F32)
    sqdiff_kernel<float><<<grid, SQ_THREADS, 0, st>>>((const float*)X, ldx, strideX, (const float*)Y, ldy,
                                                      strideY, m, nc, parts, (double*)ws);
  else {
    set_error("bmm_sqdiff: unknown dtype %d", dtype);
    return BMM_E_ARG;
  }
  BMM_CHECK_LAUNCH("sqdiff_kernel");
  sqdiff_final_kernel<<<grid_for(batch, 64), 64, 0, st>>>((const double*)ws, parts, batch, err);
  BMM_CHECK_LAUNCH("sqdiff_final_kernel");
  return BMM_OK;
}

// ---- exact variance analytics: analysis.py:57-116
namespace bmm {
using VarCfg = DV2;     // term 1 GEMM tiles
using VarSegCfg = DV0;  // term 2: the square accumulators double the register tile, so 32x32 warp tiles

inline int64_t var_chunks(int64_t m, int64_t p, int64_t K) {
  const VariantInfo vi = variant_info(0);
  const int64_t tiles = ceil_div(m, vi.BM) * ceil_div(p, vi.BN);
  int64_t ch = ((int64_t)vi.occ * 148) / tiles;
  if (ch > K) ch = K;
  if (ch > 64) ch = 64;
  if (ch < 1) ch = 1;
  return ch;
}

inline int64_t var_ws_head(int64_t n, int64_t K) { return ceil_div(8 * (n + K), 256) * 256; }
}  // namespace bmm

extern "C" int64_t bmm_variance_workspace(int64_t m, int64_t p, int64_t n, int64_t K) {
  const SplitPlan sp = plan_split(variant_info(2), m, p, n, 1);
  const int64_t gemm_need = sp.splits > 1 ? sp.splits * m * p * 8 : 0;
  const int64_t seg_need = var_chunks(m, p, K) * m * p * 8;
  return var_ws_head(n, K) + std::max(gemm_need, seg_need);
}

extern "C" int bmm_elementwise_variance(const double* M, int64_t ldm, const double* N, int64_t ldn, int64_t m,
                                        int64_t n, int64_t p, const int64_t* offsets, int64_t K,
                                        const double* probs, const double* colsq, const double* rowsq,
                                        const double* budgets, double* var, int64_t ldv, int64_t* bad, void* ws,
                                        int64_t ws_bytes, void* stream) {
  BMM_REQUIRE(m >= 1 && n >= 1 && p >= 1 && K >= 1 && var != nullptr && bad != nullptr, BMM_E_ARG,
              "bmm_elementwise_variance: bad arguments");
  const int64_t need = bmm_variance_workspace(m, p, n, K);
  BMM_REQUIRE(ws != nullptr && ws_bytes >= need, BMM_E_ARG, "bmm_elementwise_variance: workspace too small");
  cudaStream_t st = as_stream(stream);
  double* w_col = (double*)ws;
  double* w_blk = w_col + n;
  double* part = (double*)((char*)ws + var_ws_head(n, K));
  if (cudaMemsetAsync(bad, 0, sizeof(int64_t), st) != cudaSuccess) {
    set_error("bmm_elementwise_variance: memset failed");
    return BMM_E_CUDA;
  }
  variance_weights_kernel<<<grid_for(n, 256), 256, 0, st>>>(probs, colsq, rowsq, offsets, K, budgets, w_col, w_blk,
                                                            bad);
  BMM_CHECK_LAUNCH("variance_weights_kernel");
  // term 1: sum_i M_hi^2 N_if^2 / (c_k p_i)  (one squared-mode GEMM over the whole inner dimension)
  const VariantInfo vi = variant_info(2);
  const SplitPlan sp = plan_split(vi, m, p, n, 1);
  const bool v16 = (reinterpret_cast<uintptr_t>(M) % 16 == 0) && ldm % 2 == 0 &&
                   (reinterpret_cast<uintptr_t>(N) % 16 == 0) && ldn % 2 == 0;
  {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_f64_kernel<VarCfg, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           VarCfg::SMEM);
      cudaFuncSetAttribute(gemm_f64_kernel<VarCfg, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           VarCfg::SMEM);
      cudaFuncSetAttribute(segsq_mat_kernel<VarSegCfg, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           VarSegCfg::SMEM);
      cudaFuncSetAttribute(segsq_mat_kernel<VarSegCfg, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           VarSegCfg::SMEM);
      attr = true;
    }
  }
  dim3 grid((unsigned)ceil_div(p, vi.BN), (unsigned)ceil_div(m, vi.BM), (unsigned)sp.splits);
  if (v16)
    gemm_f64_kernel<VarCfg, true, false, true><<<grid, VarCfg::THREADS, VarCfg::SMEM, st>>>(
        M, ldm, 0, N, ldn, 0, m, p, n, sp.splits, sp.kchunk, var, ldv, 0, part, nullptr, w_col, 0);
  else
    gemm_f64_kernel<VarCfg, false, false, true><<<grid, VarCfg::THREADS, VarCfg::SMEM, st>>>(
        M, ldm, 0, N, ldn, 0, m, p, n, sp.splits, sp.kchunk, var, ldv, 0, part, nullptr, w_col, 0);
  BMM_CHECK_LAUNCH("gemm_f64_kernel(sq)");
  if (sp.splits > 1) {
    splitk_reduce_kernel<<<grid_for(m * p, 256), 256, 0, st>>>(part, sp.splits, m, p, 1, var, ldv, 0);
    BMM_CHECK_LAUNCH("splitk_reduce_kernel");
  }
  // term 2: sum_k (M^k N_k)^2 / c_k, subtracted in chunk order
  const int64_t chunks = var_chunks(m, p, K);
  dim3 g2((unsigned)ceil_div(p, VarSegCfg::BN), (unsigned)ceil_div(m, VarSegCfg::BM), (unsigned)chunks);
  if (v16)
    segsq_mat_kernel<VarSegCfg, true><<<g2, VarSegCfg::THREADS, VarSegCfg::SMEM, st>>>(M, ldm, N, ldn, m, p, offsets,
                                                                                       K, w_blk, chunks, part);
  else
    segsq_mat_kernel<VarSegCfg, false><<<g2, VarSegCfg::THREADS, VarSegCfg::SMEM, st>>>(M, ldm, N, ldn, m, p,
                                                                                        offsets, K, w_blk, chunks,
                                                                                        part);
  BMM_CHECK_LAUNCH("segsq_mat_kernel");
  sub_chunks_kernel<<<grid_for(m * p, 256), 256, 0, st>>>(part, chunks, m, p, var, ldv);
  BMM_CHECK_LAUNCH("sub_chunks_kernel");
  return BMM_OK;
}

extern "C" int bmm_block_term1(const double* probs, const double* colsq, const double* rowsq, const int64_t* offsets,
                               int64_t K, double* out, int64_t* bad, void* stream) {
  BMM_REQUIRE(K >= 1 && out != nullptr && bad != nullptr, BMM_E_ARG, "bmm_block_term1: bad arguments");
  cudaStream_t st = as_stream(stream);
  if (cudaMemsetAsync(bad, 0, sizeof(int64_t), st) != cudaSuccess) {
    set_error("bmm_block_term1: memset failed");
    return BMM_E_CUDA;
  }
  block_term1_kernel<<<grid_for(K * 32, 256), 256, 0, st>>>(probs, colsq, rowsq, offsets, K, out, bad);
  BMM_CHECK_LAUNCH("block_term1_kernel");
  return BMM_OK;
}
