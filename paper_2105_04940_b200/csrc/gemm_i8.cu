// K7' -- float64 segmented square sums on the int8 tensor cores (Ozaki scheme).
//
//   gsq[b, j] = || A[:, seg_j] @ B[seg_j, :] ||_F^2        (plan.py:183-188, OPL g_k^2)
//
// sm_100a runs float64 only on the DMMA pipe (~36 TF/s measured), while its
// tcgen05 int8 path is two orders of magnitude faster.  Every float64 value is
// therefore split EXACTLY into int8 digits and the contraction runs as integer
// MMAs with exact int32 accumulation:
//
//   * scale: each row h of A^k (one block's columns of M) gets sigma = 2^e with
//     max_i |A[h,i]| < 2^e; each column f of B_k likewise (tau = 2^e').
//   * digits: F = rint(|x| 2^(55-e)) < 2^55 (exact for |x| >= 2^(e-2); one
//     rounding below), written in balanced base 128 as S = 8 digits
//     d_0..d_7 in [-64, 64] (d_0 most significant) and the sign applied, so
//     x = sigma 2^-55 sum_t d_t 128^(7-t) up to 2^-56 sigma.
//   * products: A B = sigma tau 2^-12 sum_d 2^-7d acc_d with
//     acc_d = sum_{t+u=d} D_t E_u (d = 0..7; levels d >= 8 weigh < 2^-56 and are
//     dropped).  |acc_d| <= 8 * 64 * 64 * K < 2^31 for K <= 65504: int32 exact.
//   * epilogue: hi = sum_{d<4} acc_d 128^(3-d), lo = sum_{d>=4} acc_d 128^(7-d)
//     (exact int64, < 2^53), v = hi 2^-21 + lo 2^-49 (one rounding), and the
//     per-tile partial sum of (sigma tau 2^-12 v)^2, reduced in a fixed order.
//
// The result agrees with a float64 GEMM to ~1e-16 relative (the split is exact
// to 55 bits per row/column scale, the integer sums are exact), deterministic.
//
// Kernels: oz_prep (segment padding to 32, longest-first order), oz_split_rows
// (A: warp per row segment, digits written K-major), oz_split_cols (B: CTA per
// segment x 64 columns, transposed through shared memory), oz_segsq (persistent
// tcgen05 kernel: TMA SWIZZLE_32B ring of S digit planes per operand, one
// elected thread issues kind::i8 MMAs M=128 into 8 level accumulators
// occupying all 512 TMEM columns -- A plane t times the B planes 0..7-t in
// ONE MMA of N = 64 (8-t) (<= 256 per instruction), landing in levels t..7 --
// and four epilogue warps drain the levels), oz_reduce.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>

#include "common.cuh"
#include "tcgen05.cuh"

namespace bmm {

constexpr int OZ_S = 8;            // digit planes per operand
constexpr int OZ_BM = 128;         // output rows per tile (UMMA M)
constexpr int OZ_BN = 64;          // output columns per tile (one level = 64 TMEM columns)
constexpr int OZ_BK = 32;          // K per stage = one kind::i8 MMA = one 32-byte swizzle row
constexpr int OZ_KMAX = 65504;     // segment length bound for exact int32 levels
constexpr int OZ_A_PLANE = OZ_BM * OZ_BK;            // 4 KB
constexpr int OZ_B_PLANE = OZ_BN * OZ_BK;            // 2 KB
constexpr int OZ_STAGE = OZ_S * (OZ_A_PLANE + OZ_B_PLANE);  // 48 KB
constexpr int OZ_STAGES = 4;
constexpr int OZ_SMEM = OZ_STAGES * OZ_STAGE + 1024 + 1024;
constexpr int OZ_THREADS = 192;    // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int OZ_TMEM_COLS = 512;

// balanced base-128 offset: 64 in every digit position (F + C has fields f_t,
// F = sum (f_t - 64) 128^t)
constexpr uint64_t OZ_C = 0x0081020408102040ull;  // sum_{t=0..7} 64 * 128^t

// ---------------------------------------------------------------- digits

// The two packed words of one value: byte t of w0 = digit t (t = 0..3, most
// significant first), byte t of w1 = digit 4 + t.  e = the row/column scale.
__device__ __forceinline__ void oz_digits(double x, double s1, double s2, uint32_t& w0, uint32_t& w1) {
  const double y = (fabs(x) * s1) * s2;  // exact: powers of two, y < 2^55
  const uint64_t F = __double2ull_rn(y);
  const uint64_t G = F + OZ_C;
  const uint32_t hi = (uint32_t)(G >> 28);           // fields 3,2,1 (7 bits) and 0 (8 bits)
  const uint32_t lo = (uint32_t)G & 0x0FFFFFFFu;     // fields 7,6,5,4
  w0 = ((hi >> 21) & 0xFFu) | (((hi >> 14) & 127u) << 8) | (((hi >> 7) & 127u) << 16) | ((hi & 127u) << 24);
  w1 = ((lo >> 21) & 127u) | (((lo >> 14) & 127u) << 8) | (((lo >> 7) & 127u) << 16) | ((lo & 127u) << 24);
  w0 = __vsub4(w0, 0x40404040u);
  w1 = __vsub4(w1, 0x40404040u);
  if (x < 0.0) {
    w0 = __vneg4(w0);
    w1 = __vneg4(w1);
  }
}

// scale factors for exponent e: x * 2^(55-e) as two exact multiplies
__device__ __forceinline__ void oz_scales(int e, double& s1, double& s2) {
  const int k = 55 - e;
  const int k1 = k / 2;
  s1 = ldexp(1.0, k1);
  s2 = ldexp(1.0, k - k1);
}

__device__ __forceinline__ int oz_exponent(double mx) {
  if (!(mx > 0.0)) return 0;  // all-zero row/column: digits are all zero
  int e;
  frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): every |x| <= mx < 2^e
  return e;
}

template <typename T>
__device__ __forceinline__ double oz_ld(const T* p) { return (double)__ldg(p); }

// byte `u` of each of a[0..3] packed into one word
__device__ __forceinline__ uint32_t oz_gather_byte(const uint32_t (&a)[4], int u) {
  const uint32_t p01 = __byte_perm(a[0], a[1], (uint32_t)(u | ((u + 4) << 4)));
  const uint32_t p23 = __byte_perm(a[2], a[3], (uint32_t)(u | ((u + 4) << 4)));
  return __byte_perm(p01, p23, 0x5410);
}

// ---------------------------------------------------------------- prep
// Per problem: padded lengths L_j = ceil32(len_j), padded offsets po_j
// (exclusive scan), longest-first order (nseg <= 4096), and a status flag:
// 1 = a segment is negative or longer than OZ_KMAX, 2 = padded extent > cap.
__global__ void __launch_bounds__(1024) oz_prep_kernel(const int64_t* __restrict__ seg, int64_t nseg,
                                                       int64_t seg_stride, int64_t cap, int64_t* __restrict__ po,
                                                       int32_t* __restrict__ L, int32_t* __restrict__ perm,
                                                       int32_t* __restrict__ flag) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t base_s;
  __shared__ int flag_s;
  const int64_t b = blockIdx.x;
  const int64_t* s = seg + b * seg_stride;
  int32_t* Lb = L + b * nseg;
  int64_t* pob = po + b * nseg;
  int32_t* pb = perm + b * nseg;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    base_s = 0;
    flag_s = 0;
  }
  __syncthreads();
  for (int64_t j0 = 0; j0 < nseg; j0 += 1024) {
    const int64_t j = j0 + threadIdx.x;
    int64_t l = 0;
    if (j < nseg) {
      const int64_t len = s[j + 1] - s[j];
      if (len < 0 || len > OZ_KMAX) {
        atomicOr(&flag_s, 1);
      } else {
        l = (len + 31) & ~int64_t(31);
      }
      Lb[j] = (int32_t)l;
    }
    // block exclusive scan of l
    int64_t v = l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int64_t w = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const int64_t excl = base_s + (warp > 0 ? wsum[warp - 1] : 0) + v - l;
    if (j < nseg) pob[j] = excl;
    __syncthreads();
    if (threadIdx.x == 0) base_s += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0 && base_s > cap) flag_s |= 2;
  __syncthreads();
  // longest first (ties by index): rank by counting
  for (int64_t j = threadIdx.x; j < nseg; j += 1024) {
    if (nseg > 4096) {
      pb[j] = (int32_t)j;
      continue;
    }
    const int32_t lj = Lb[j];
    int64_t r = 0;
    for (int64_t i = 0; i < nseg; ++i) {
      const int32_t li = Lb[i];
      r += (li > lj) || (li == lj && i < j);
    }
    pb[r] = (int32_t)j;
  }
  if (threadIdx.x == 0) flag[b] = flag_s;
}

// ---------------------------------------------------------------- split of A
// Warp per (row h, segment j): row maximum, exponent, then the 8 digit planes
// of the row segment (zero-padded to L_j), 4 consecutive values per lane so
// each plane store is one coalesced 128-byte row piece.
template <typename T>
__global__ void __launch_bounds__(256) oz_split_rows_kernel(const T* __restrict__ A, int64_t lda, int64_t strideA,
                                                            int64_t m, const int64_t* __restrict__ seg,
                                                            int64_t nseg, int64_t seg_stride,
                                                            const int64_t* __restrict__ po,
                                                            const int32_t* __restrict__ L, int64_t P,
                                                            uint8_t* __restrict__ planes, int32_t* __restrict__ ex,
                                                            const int32_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t h = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t j = blockIdx.y, b = blockIdx.z;
  if (h >= m || flag[b] != 0) return;  // bad segments: no writes (the result is NaN)
  const int64_t Lj = L[b * nseg + j];
  if (Lj == 0) return;
  const int64_t s0 = seg[b * seg_stride + j];
  const int64_t len = seg[b * seg_stride + j + 1] - s0;
  const T* row = A + b * strideA + h * lda + s0;
  double mx = 0.0;
  for (int64_t i0 = 4 * lane; i0 < len; i0 += 128) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + q < len) mx = fmax(mx, fabs(oz_ld(row + i0 + q)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int e = oz_exponent(mx);
  if (lane == 0) ex[(b * nseg + j) * m + h] = e;
  double s1, s2;
  oz_scales(e, s1, s2);
  const int64_t pob = po[b * nseg + j];
  uint8_t* out = planes + ((b * OZ_S) * m + h) * P + pob;
  const int64_t plane = m * P;
  for (int64_t i0 = 4 * lane; i0 < Lj; i0 += 128) {
    uint32_t w0[4], w1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double x = i0 + q < len ? oz_ld(row + i0 + q) : 0.0;
      oz_digits(x, s1, s2, w0[q], w1[q]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      *reinterpret_cast<uint32_t*>(out + u * plane + i0) = oz_gather_byte(w0, u);
      *reinterpret_cast<uint32_t*>(out + (4 + u) * plane + i0) = oz_gather_byte(w1, u);
    }
  }
}

// ---------------------------------------------------------------- split of B
// CTA per (segment j, 64 columns): column maxima over the segment's rows, then
// 32-row chunks: thread (g, c) converts rows 8g..8g+7 of column c, the digit
// bytes are transposed into a [plane][column][32] shared tile and written as
// 16-byte pieces of the K-major planes B^T.
template <typename T>
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const T* __restrict__ B, int64_t ldb, int64_t strideB,
                                                            int64_t nc, const int64_t* __restrict__ seg,
                                                            int64_t nseg, int64_t seg_stride,
                                                            const int64_t* __restrict__ po,
                                                            const int32_t* __restrict__ L, int64_t P,
                                                            uint8_t* __restrict__ planes, int32_t* __restrict__ ex,
                                                            const int32_t* __restrict__ flag) {
  __shared__ double red[4][64];
  __shared__ __align__(16) uint8_t tile[OZ_S][64][32];
  const int64_t j = blockIdx.y, b = blockIdx.z;
  const int64_t Lj = L[b * nseg + j];
  if (Lj == 0 || flag[b] != 0) return;
  const int g = threadIdx.x >> 6, c = threadIdx.x & 63;
  const int64_t f0 = (int64_t)blockIdx.x * 64;
  const int64_t f = f0 + c;
  const bool fv = f < nc;
  const int64_t s0 = seg[b * seg_stride + j];
  const int64_t len = seg[b * seg_stride + j + 1] - s0;
  const T* col = B + b * strideB + s0 * ldb + f;
  double mx = 0.0;
  if (fv)
    for (int64_t i = g; i < len; i += 4) mx = fmax(mx, fabs(oz_ld(col + i * ldb)));
  red[g][c] = mx;
  __syncthreads();
  mx = fmax(fmax(red[0][c], red[1][c]), fmax(red[2][c], red[3][c]));
  const int e = oz_exponent(mx);
  if (g == 0 && fv) ex[(b * nseg + j) * nc + f] = e;
  double s1, s2;
  oz_scales(e, s1, s2);
  const int64_t pob = po[b * nseg + j];
  const int64_t plane = nc * P;
  uint8_t* out = planes + (b * OZ_S) * plane + pob;
  for (int64_t i0 = 0; i0 < Lj; i0 += 32) {
    uint32_t w0[8], w1[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int64_t i = i0 + 8 * g + r;
      const double x = (fv && i < len) ? oz_ld(col + i * ldb) : 0.0;
      oz_digits(x, s1, s2, w0[r], w1[r]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t a0[4] = {w0[0], w0[1], w0[2], w0[3]}, a1[4] = {w0[4], w0[5], w0[6], w0[7]};
      const uint32_t b0[4] = {w1[0], w1[1], w1[2], w1[3]}, b1[4] = {w1[4], w1[5], w1[6], w1[7]};
      *reinterpret_cast<uint2*>(&tile[u][c][8 * g]) = make_uint2(oz_gather_byte(a0, u), oz_gather_byte(a1, u));
      *reinterpret_cast<uint2*>(&tile[4 + u][c][8 * g]) = make_uint2(oz_gather_byte(b0, u), oz_gather_byte(b1, u));
    }
    __syncthreads();
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const int q = threadIdx.x + 256 * z;  // 1024 pieces of 16 bytes
      const int u = q >> 7, cc = (q >> 1) & 63, half = q & 1;
      if (f0 + cc < nc)
        *reinterpret_cast<uint4*>(out + u * plane + (f0 + cc) * P + i0 + 16 * half) =
            *reinterpret_cast<const uint4*>(&tile[u][cc][16 * half]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- tcgen05 kernel

// UMMA shared-memory descriptor: K-major, SWIZZLE_32B (32-byte rows, 8-row
// groups 256 B apart)
__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // leading byte offset (unused: K fits one swizzle row)
  d |= (uint64_t)(256 >> 4) << 32;     // stride byte offset: 8 rows x 32 B
  d |= (uint64_t)1 << 46;              // Blackwell descriptor version
  d |= (uint64_t)6 << 61;              // SWIZZLE_32B
  return d;
}

// kind::i8: S32 accumulate, signed int8 A and B, K-major, M = 128, N = n
__device__ __forceinline__ uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(OZ_BM >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

struct OzItem {
  int64_t b, j, tm, tn;
  int64_t k0;   // padded offset of the segment
  int ktiles;   // stages (32 K each)
};

struct OzGeom {
  int64_t m, nc, nseg, TM, TN, items;
};

__device__ __forceinline__ OzItem oz_item(const OzGeom& g, int64_t it, const int32_t* __restrict__ perm,
                                          const int64_t* __restrict__ po, const int32_t* __restrict__ L) {
  OzItem r;
  const int64_t tiles = g.TM * g.TN;
  const int64_t tile = it % tiles;
  const int64_t rest = it / tiles;
  const int64_t rank = rest % g.nseg;
  r.b = rest / g.nseg;
  r.j = perm[r.b * g.nseg + rank];
  r.tn = tile % g.TN;
  r.tm = tile / g.TN;
  r.k0 = po[r.b * g.nseg + r.j];
  r.ktiles = L[r.b * g.nseg + r.j] / OZ_BK;
  return r;
}

// Persistent: CTA c takes items c, c + G, ... of the longest-first item list.
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_segsq_kernel(const __grid_constant__ CUtensorMap tm_a,
                                                                 const __grid_constant__ CUtensorMap tm_b, OzGeom geo,
                                                                 const int32_t* __restrict__ perm,
                                                                 const int64_t* __restrict__ po,
                                                                 const int32_t* __restrict__ L,
                                                                 const int32_t* __restrict__ exA,
                                                                 const int32_t* __restrict__ exB,
                                                                 double* __restrict__ part) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZ_STAGES * OZ_STAGE);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* acc_full = empty + OZ_STAGES;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  double* wcol = reinterpret_cast<double*>(smem + OZ_STAGES * OZ_STAGE + 256);  // [2][64]
  double* red = wcol + 128;                                                     // [4]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_b)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(OZ_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer: the S digit planes of A and B for every stage
      uint32_t it = 0;
      for (int64_t w = blockIdx.x; w < geo.items; w += gridDim.x) {
        const OzItem I = oz_item(geo, w, perm, po, L);
        const int arow = (int)(I.b * OZ_S * geo.m + I.tm * OZ_BM);
        const int brow = (int)(I.b * OZ_S * geo.nc + I.tn * OZ_BN);
        for (int kt = 0; kt < I.ktiles; ++kt, ++it) {
          const int s = it % OZ_STAGES;
          if (it >= OZ_STAGES) mbar_wait(&empty[s], ((it / OZ_STAGES) - 1) & 1);
          uint8_t* st = smem + s * OZ_STAGE;
          mbar_expect_tx(&full[s], OZ_STAGE);
          const int kc = (int)(I.k0 + kt * OZ_BK);
#pragma unroll
          for (int t = 0; t < OZ_S; ++t) tma_load_2d(st + t * OZ_A_PLANE, &tm_a, &full[s], kc, arow + t * (int)geo.m);
#pragma unroll
          for (int u = 0; u < OZ_S; ++u)
            tma_load_2d(st + OZ_S * OZ_A_PLANE + u * OZ_B_PLANE, &tm_b, &full[s], kc, brow + u * (int)geo.nc);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: per stage, A plane t x B planes 0..S-1-t into levels t..S-1
      uint32_t it = 0, n_items = 0;
      for (int64_t w = blockIdx.x; w < geo.items; w += gridDim.x) {
        const OzItem I = oz_item(geo, w, perm, po, L);
        if (I.ktiles == 0) continue;
        if (n_items > 0) mbar_wait(acc_empty, (n_items - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        for (int kt = 0; kt < I.ktiles; ++kt, ++it) {
          const int s = it % OZ_STAGES;
          mbar_wait(&full[s], (it / OZ_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t base = su32(smem + s * OZ_STAGE);
#pragma unroll
          for (int t = 0; t < OZ_S; ++t) {
            const uint64_t adesc = umma_desc_sw32(base + t * OZ_A_PLANE);
#pragma unroll
            for (int u0 = 0; u0 < OZ_S - t; u0 += 4) {
              const int nu = (OZ_S - t - u0) < 4 ? (OZ_S - t - u0) : 4;
              const uint64_t bdesc = umma_desc_sw32(base + OZ_S * OZ_A_PLANE + u0 * OZ_B_PLANE);
              umma_i8(tmem + (uint32_t)((t + u0) * OZ_BN), adesc, bdesc, idesc_i8(nu * OZ_BN),
                      (kt > 0 || t > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[s]);
        }
        umma_commit(acc_full);
        ++n_items;
      }
    }
  } else {
    // ---- epilogue: drain the 8 levels, square-sum the tile
    const int e_id = threadIdx.x - 64;  // 0..127
    const int quarter = warp & 3;
    uint32_t n_items = 0;
    for (int64_t w = blockIdx.x; w < geo.items; w += gridDim.x) {
      const OzItem I = oz_item(geo, w, perm, po, L);
      double* prow = part + ((I.b * geo.nseg + I.j) * geo.TM + I.tm) * geo.TN + I.tn;
      if (I.ktiles == 0) {
        if (e_id == 0) *prow = 0.0;
        continue;
      }
      double* wc = wcol + 64 * (n_items & 1);
      if (e_id < 64) {
        const int64_t f = I.tn * OZ_BN + e_id;
        wc[e_id] = f < geo.nc ? ldexp(1.0, exB[(I.b * geo.nseg + I.j) * geo.nc + f] - 12) : 0.0;
      }
      named_sync(1, 128);
      mbar_wait(acc_full, n_items & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int64_t row = I.tm * OZ_BM + quarter * 32 + lane;
      double R = 0.0;
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < OZ_BN; c0 += 16) {
        uint32_t v[OZ_S][16];
#pragma unroll
        for (int d = 0; d < OZ_S; ++d) tmem_ld16(tbase + (uint32_t)(d * OZ_BN + c0), v[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (c0 + 16 == OZ_BN) {
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t hi = ((((int64_t)(int32_t)v[0][q] * 128 + (int32_t)v[1][q]) * 128 + (int32_t)v[2][q]) * 128) +
                             (int32_t)v[3][q];
          const int64_t lo = ((((int64_t)(int32_t)v[4][q] * 128 + (int32_t)v[5][q]) * 128 + (int32_t)v[6][q]) * 128) +
                             (int32_t)v[7][q];
          const double x = fma((double)lo, 0x1p-49, (double)hi * 0x1p-21) * wc[c0 + q];
          R = fma(x, x, R);
        }
      }
      if (row < geo.m) {
        const double sr = ldexp(1.0, exA[(I.b * geo.nseg + I.j) * geo.m + row]);
        R = (R * sr) * sr;
      } else {
        R = 0.0;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) R += __shfl_xor_sync(0xffffffffu, R, o);
      if (lane == 0) red[quarter] = R;
      named_sync(1, 128);
      if (e_id == 0) *prow = (red[0] + red[1]) + (red[2] + red[3]);
      ++n_items;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(OZ_TMEM_COLS));
  }
}

__global__ void oz_reduce_kernel(const double* __restrict__ part, int64_t tiles, int64_t nseg, int64_t total,
                                 const int32_t* __restrict__ flag, double* __restrict__ gsq) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    if (flag[g / nseg] != 0) {
      gsq[g] = __longlong_as_double(0x7ff8000000000000ll);  // NaN: bad segments (status in the workspace)
      continue;
    }
    const double* p = part + g * tiles;
    double acc = 0.0;
    for (int64_t i = 0; i < tiles; ++i) acc += p[i];
    gsq[g] = acc;
  }
}

// ---------------------------------------------------------------- host side

struct OzLayout {
  int64_t P;                 // padded inner extent (row pitch of the planes)
  int64_t off_a, off_b, off_exa, off_exb, off_po, off_L, off_perm, off_flag, off_part, total;
};

static inline int64_t al256(int64_t x) { return (x + 255) & ~int64_t(255); }

static OzLayout oz_layout(int64_t m, int64_t nc, int64_t n_inner, int64_t nseg, int64_t batch) {
  OzLayout l;
  l.P = ((n_inner + 31) / 32) * 32 + 32 * nseg;
  const int64_t TM = ceil_div(m, OZ_BM), TN = ceil_div(nc, OZ_BN);
  int64_t o = 0;
  l.off_a = o;    o = al256(o + batch * OZ_S * m * l.P);
  l.off_b = o;    o = al256(o + batch * OZ_S * nc * l.P);
  l.off_exa = o;  o = al256(o + batch * nseg * m * 4);
  l.off_exb = o;  o = al256(o + batch * nseg * nc * 4);
  l.off_po = o;   o = al256(o + batch * nseg * 8);
  l.off_L = o;    o = al256(o + batch * nseg * 4);
  l.off_perm = o; o = al256(o + batch * nseg * 4);
  l.off_flag = o; o = al256(o + batch * 4);
  l.off_part = o; o = al256(o + batch * nseg * TM * TN * 8);
  l.total = o;
  return l;
}

static int oz_map(CUtensorMap* map, const uint8_t* base, int64_t rows, int64_t P, int box_rows) {
  auto enc = get_encode();
  BMM_REQUIRE(enc != nullptr, BMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)P};
  cuuint32_t box[2] = {(cuuint32_t)OZ_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BMM_REQUIRE(r == CUDA_SUCCESS, BMM_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BMM_OK;
}

}  // namespace bmm

using namespace bmm;

extern "C" int64_t bmm_segsq_i8_workspace(int64_t m, int64_t nc, int64_t n_inner, int64_t nseg, int64_t batch) {
  if (m < 1 || nc < 1 || n_inner < 0 || nseg < 1 || batch < 1) return 0;
  return oz_layout(m, nc, n_inner, nseg, batch).total;
}

extern "C" int bmm_segsq_i8(int dtype, const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                            int64_t strideB, int64_t m, int64_t nc, int64_t n_inner, const int64_t* seg, int64_t nseg,
                            int64_t seg_stride, int64_t batch, double* gsq, void* ws, int64_t ws_bytes,
                            void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && n_inner >= 0 && nseg >= 1 && batch >= 1, BMM_E_ARG, "bmm_segsq_i8: bad shape");
  BMM_REQUIRE(A != nullptr && B != nullptr && seg != nullptr && gsq != nullptr, BMM_E_ARG,
              "bmm_segsq_i8: null pointer");
  BMM_REQUIRE(dtype == BMM_F64 || dtype == BMM_F32, BMM_E_ARG, "bmm_segsq_i8: unknown dtype %d", dtype);
  const OzLayout l = oz_layout(m, nc, n_inner, nseg, batch);
  BMM_REQUIRE(ws != nullptr && ws_bytes >= l.total, BMM_E_ARG, "bmm_segsq_i8: workspace too small (%lld < %lld)",
              (long long)ws_bytes, (long long)l.total);
  BMM_REQUIRE(batch * OZ_S * (m > nc ? m : nc) < (1LL << 31) && l.P < (1LL << 31), BMM_E_UNSUPPORTED,
              "bmm_segsq_i8: problem too large for 32-bit TMA coordinates");
  BMM_REQUIRE(nseg <= 65535 && batch <= 65535 && ceil_div(m, 8) <= (1LL << 31) - 1, BMM_E_UNSUPPORTED,
              "bmm_segsq_i8: grid too large");
  uint8_t* w = (uint8_t*)ws;
  uint8_t* pa = w + l.off_a;
  uint8_t* pb = w + l.off_b;
  int32_t* exa = (int32_t*)(w + l.off_exa);
  int32_t* exb = (int32_t*)(w + l.off_exb);
  int64_t* po = (int64_t*)(w + l.off_po);
  int32_t* L = (int32_t*)(w + l.off_L);
  int32_t* perm = (int32_t*)(w + l.off_perm);
  int32_t* flag = (int32_t*)(w + l.off_flag);
  double* part = (double*)(w + l.off_part);
  cudaStream_t st = as_stream(stream);

  oz_prep_kernel<<<(unsigned)batch, 1024, 0, st>>>(seg, nseg, seg_stride, l.P, po, L, perm, flag);
  BMM_CHECK_LAUNCH("oz_prep_kernel");
  dim3 ga((unsigned)ceil_div(m, 8), (unsigned)nseg, (unsigned)batch);
  dim3 gb((unsigned)ceil_div(nc, 64), (unsigned)nseg, (unsigned)batch);
  if (dtype == BMM_F64) {
    oz_split_rows_kernel<double><<<ga, 256, 0, st>>>((const double*)A, lda, strideA, m, seg, nseg, seg_stride, po, L,
                                                     l.P, pa, exa, flag);
    BMM_CHECK_LAUNCH("oz_split_rows_kernel");
    oz_split_cols_kernel<double><<<gb, 256, 0, st>>>((const double*)B, ldb, strideB, nc, seg, nseg, seg_stride, po, L,
                                                     l.P, pb, exb, flag);
  } else {
    oz_split_rows_kernel<float><<<ga, 256, 0, st>>>((const float*)A, lda, strideA, m, seg, nseg, seg_stride, po, L,
                                                    l.P, pa, exa, flag);
    BMM_CHECK_LAUNCH("oz_split_rows_kernel");
    oz_split_cols_kernel<float><<<gb, 256, 0, st>>>((const float*)B, ldb, strideB, nc, seg, nseg, seg_stride, po, L,
                                                    l.P, pb, exb, flag);
  }
  BMM_CHECK_LAUNCH("oz_split_cols_kernel");

  CUtensorMap ma, mb;
  int rc;
  if ((rc = oz_map(&ma, pa, batch * OZ_S * m, l.P, OZ_BM)) != BMM_OK) return rc;
  if ((rc = oz_map(&mb, pb, batch * OZ_S * nc, l.P, OZ_BN)) != BMM_OK) return rc;
  OzGeom geo;
  geo.m = m;
  geo.nc = nc;
  geo.nseg = nseg;
  geo.TM = ceil_div(m, OZ_BM);
  geo.TN = ceil_div(nc, OZ_BN);
  geo.items = batch * nseg * geo.TM * geo.TN;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(oz_segsq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
    attr = true;
  }
  static int nsm = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const unsigned grid = (unsigned)(geo.items < nsm ? geo.items : nsm);
  oz_segsq_kernel<<<grid, OZ_THREADS, OZ_SMEM, st>>>(ma, mb, geo, perm, po, L, exa, exb, part);
  BMM_CHECK_LAUNCH("oz_segsq_kernel");
  oz_reduce_kernel<<<grid_for(batch * nseg, 128), 128, 0, st>>>(part, geo.TM * geo.TN, nseg, batch * nseg, flag, gsq);
  BMM_CHECK_LAUNCH("oz_reduce_kernel");
  return BMM_OK;
}
