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
//   * digits: F = rint(x 2^(54-e)), |F| < 2^54 (exact for |x| >= 2^(e-1); one
//     rounding below), written in balanced base 128 as S = 8 digits
//     d_0..d_7 in [-64, 63] (d_0 most significant), so
//     x = sigma 2^-54 sum_t d_t 128^(7-t) up to 2^-55 sigma.
//   * products: A B = sigma tau 2^-10 sum_d 2^-7d acc_d with
//     acc_d = sum_{t+u=d} D_t E_u (d = 0..7; levels d >= 8 weigh < 2^-55 and are
//     dropped).  |acc_d| <= 8 * 64 * 64 * K < 2^31 for K <= 32768: int32 exact.
//   * epilogue: hi = sum_{d<4} acc_d 128^(3-d), lo = sum_{d>=4} acc_d 128^(7-d)
//     (exact int64, < 2^51), v = hi 2^-21 + lo 2^-49 (one rounding), and the
//     per-tile partial sum of (sigma tau 2^-10 v)^2, reduced in a fixed order.
//
// The result agrees with a float64 GEMM to ~1e-16 relative (the split is exact
// to 54 bits per row/column scale, the integer sums are exact), deterministic.
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
#include <cstdlib>

#include "common.cuh"
#include "tcgen05.cuh"

namespace bmm {

constexpr int OZ_S = 8;            // digit planes per operand
constexpr int OZ_BM = 128;         // output rows per tile (UMMA M)
constexpr int OZ_BN = 64;          // output columns per tile (one level = 64 TMEM columns)
constexpr int OZ_BK = 32;          // K per stage = one kind::i8 MMA = one 32-byte swizzle row
constexpr int OZ_KMAX = 32768;     // segment length bound: exact int32 levels, |hi|, |lo| < 2^51
constexpr int OZ_A_PLANE = OZ_BM * OZ_BK;            // 4 KB
constexpr int OZ_B_PLANE = OZ_BN * OZ_BK;            // 2 KB
constexpr int OZ_STAGE = OZ_S * (OZ_A_PLANE + OZ_B_PLANE);  // 48 KB
constexpr int OZ_STAGES = 4;
// stages (1024-aligned inside the allocation: up to 1023 bytes of padding), then the
// barriers (256 B), wcol [2][64] and red[] doubles: 1344 bytes past the stages.  (Round 2:
// this was + 1024 + 1024, so with an unaligned base the epilogue's red[] landed past the
// CTA's allocation -- in a co-resident CTA's shared memory: the colsq ring of a concurrent
// norm pass got corrupted; tools/stress_group.py found it.)
constexpr int OZ_SMEM = OZ_STAGES * OZ_STAGE + 1024 + 2048;
constexpr int OZ_EPI_WARPS = 8;    // two per TMEM lane quarter, 32 columns each
constexpr int OZ_EPI_COLS = OZ_BN / (OZ_EPI_WARPS / 4);
constexpr int OZ_THREADS = 64 + 32 * OZ_EPI_WARPS;  // warp 0 TMA, warp 1 MMA, then the epilogue warps
constexpr int OZ_TMEM_COLS = 512;

// balanced base-128 offset: 64 in every digit position (F + C has fields f_t,
// F = sum (f_t - 64) 128^t)
constexpr uint64_t OZ_C = 0x0081020408102040ull;  // sum_{t=0..7} 64 * 128^t

// ---------------------------------------------------------------- digits

// 7-bit fields f (bits 21, 14, 7, 0 of a 28-bit value, most significant first)
// spread into bytes 0..3 as f - 64 (two's complement; per-byte, no carries:
// ((b | 0x80) - 0x40) ^ 0x80 = b - 64 mod 256 for b < 128)
__device__ __forceinline__ uint32_t oz_spread(uint32_t v) {
  const uint32_t w = (v >> 21) | ((v >> 6) & 0x7F00u) | ((v << 9) & 0x7F0000u) | ((v << 24) & 0x7F000000u);
  return ((w | 0x80808080u) - 0x40404040u) ^ 0x80808080u;
}

// The two packed words of one value: byte t of w0 = digit t (t = 0..3, most
// significant first), byte t of w1 = digit 4 + t.  s1 s2 = 2^(54-e).
// Fs = rint(x 2^(54-e)) in (-2^54, 2^54); G = Fs + C has eight 7-bit fields
// f_t (C > 2^54 keeps G positive, the top field in [32, 96]) and
// Fs = sum_t (f_t - 64) 128^(7-t): balanced digits in [-64, 63].
__device__ __forceinline__ void oz_digits(double x, double s1, double s2, uint32_t& w0, uint32_t& w1) {
  const long long Fs = __double2ll_rn((x * s1) * s2);  // the scaling is exact (powers of two)
  const uint64_t G = (uint64_t)(Fs + (long long)OZ_C);
  w0 = oz_spread((uint32_t)(G >> 28));
  w1 = oz_spread((uint32_t)G & 0x0FFFFFFFu);
}

__device__ __forceinline__ double oz_pow2(int k) {  // k in [-1022, 1023]
  return __longlong_as_double((long long)(k + 1023) << 52);
}

// scale factors for exponent e: x * 2^(54-e) as two exact multiplies
__device__ __forceinline__ void oz_scales(int e, double& s1, double& s2) {
  const int k = 54 - e;
  const int k1 = k / 2;
  s1 = oz_pow2(k1);
  s2 = oz_pow2(k - k1);
}

// biased float64 exponent field of x (the scale only needs the largest one:
// integer max instead of fmax and its NaN handling)
__device__ __forceinline__ uint32_t oz_ebits(double x) { return ((uint32_t)__double2hiint(x) >> 20) & 0x7FFu; }

// e with every |x| < 2^e from the largest biased exponent field: a normal x
// is below 2^(field - 1022); subnormals (field 0) are below 2^-1022
__device__ __forceinline__ int oz_exponent_from_bits(uint32_t eb) { return (int)(eb > 1u ? eb : 1u) - 1022; }

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
                                                       int32_t* __restrict__ flag, int4* __restrict__ cmap) {
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
  // chunk map over the padded inner extent: chunk c (32 padded positions) ->
  // (segment, first original row, real rows in the chunk); -1 past the end
  const int64_t nch = cap / 32;
  int4* cm = cmap + b * nch;
  const int64_t used = flag_s ? 0 : base_s / 32;
  for (int64_t j = threadIdx.x; j < nseg && !flag_s; j += 1024) {
    const int64_t len = s[j + 1] - s[j];
    const int64_t c0 = pob[j] / 32, nc = Lb[j] / 32;
    for (int64_t c = 0; c < nc; ++c) {
      const int64_t k = s[j] + 32 * c;  // < 2^31: checked on the host
      cm[c0 + c] = make_int4((int)j, (int)k, (int)min((int64_t)32, len - 32 * c), 0);
    }
  }
  for (int64_t c = used + threadIdx.x; c < nch; c += 1024) cm[c] = make_int4(-1, 0, 0, 0);
}

// ---------------------------------------------------------------- split of A
// Warp per (row h, segment j): row maximum, exponent, then the 8 digit planes
// of the row segment (zero-padded to L_j), 4 consecutive values per lane so
// each plane store is one coalesced 128-byte row piece (the second read of the
// row segment hits L1).
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
  const int Lj = L[b * nseg + j];
  if (Lj == 0) return;
  const int64_t s0 = seg[b * seg_stride + j];
  const int len = (int)(seg[b * seg_stride + j + 1] - s0);
  const T* row = A + b * strideA + h * lda + s0;
  uint32_t eb = 0;
  for (int i0 = 4 * lane; i0 < len; i0 += 128) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = i0 + q < len ? oz_ld(row + i0 + q) : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) eb = max(eb, oz_ebits(v[q]));
  }
  eb = __reduce_max_sync(0xffffffffu, eb);
  const int e = oz_exponent_from_bits(eb);
  if (lane == 0) ex[(b * nseg + j) * m + h] = e;
  double s1, s2;
  oz_scales(e, s1, s2);
  uint8_t* out = planes + ((b * OZ_S) * m + h) * P + po[b * nseg + j];
  const int64_t plane = m * P;
  for (int i0 = 4 * lane; i0 < Lj; i0 += 128) {
    uint32_t w0[4], w1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double x = i0 + q < len ? oz_ld(row + i0 + q) : 0.0;
      oz_digits(x, s1, s2, w0[q], w1[q]);
    }
    uint8_t* o = out + i0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      *reinterpret_cast<uint32_t*>(o + u * plane) = oz_gather_byte(w0, u);
      *reinterpret_cast<uint32_t*>(o + (4 + u) * plane) = oz_gather_byte(w1, u);
    }
  }
}

// ---------------------------------------------------------------- split of B
// Chunk-parallel over the padded inner extent (32 rows of N per chunk, each
// inside one segment): (1) column maxima as biased exponent fields, atomicMax
// into the segment's per-column slot; (2) digits: CTA per (chunk, 64 columns),
// thread (g, c) converts rows 8g..8g+7 of column c, the digit bytes are
// transposed into a [plane][column][32] shared tile and written as 16-byte
// pieces of the K-major planes B^T.
template <typename T>
__global__ void __launch_bounds__(256) oz_seg_colmax_kernel(const T* __restrict__ B, int64_t ldb, int64_t strideB,
                                                            int64_t nc, int64_t nseg, int64_t nch,
                                                            const int4* __restrict__ cmap,
                                                            uint32_t* __restrict__ ex) {
  const int64_t c = blockIdx.x, b = blockIdx.z;
  const int4 cm = cmap[b * nch + c];
  const int64_t f = (int64_t)blockIdx.y * 256 + threadIdx.x;
  if (cm.x < 0 || f >= nc) return;
  const T* p = B + b * strideB + (int64_t)cm.y * ldb + f;
  uint32_t eb = 0;
  int r = 0;
  for (; r + 8 <= cm.z; r += 8) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = oz_ld(p + (int64_t)(r + q) * ldb);
#pragma unroll
    for (int q = 0; q < 8; ++q) eb = max(eb, oz_ebits(v[q]));
  }
  for (; r < cm.z; ++r) eb = max(eb, oz_ebits(oz_ld(p + (int64_t)r * ldb)));
  if (eb != 0) atomicMax(&ex[(b * nseg + cm.x) * nc + f], eb);
}

// Column digit kernels: CTA per (128 padded rows, 32 columns).  Thread (g, c)
// converts rows 16g..16g+15 of column c; the digit bytes go to a
// [plane][column][128] shared tile, written out as full 128-byte rows of the
// K-major planes B^T.
constexpr int OZ_CD_ROWS = 128, OZ_CD_COLS = 32;

// 8 values' digit bytes of plane u -> tile[u][c][16g + 8hh .. +7]
__device__ __forceinline__ void oz_cd_stash8(uint8_t (*tile)[OZ_CD_COLS][OZ_CD_ROWS], int g, int c, int hh,
                                             const uint32_t (&w0)[8], const uint32_t (&w1)[8]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t a0[4] = {w0[0], w0[1], w0[2], w0[3]}, a1[4] = {w0[4], w0[5], w0[6], w0[7]};
    const uint32_t b0[4] = {w1[0], w1[1], w1[2], w1[3]}, b1[4] = {w1[4], w1[5], w1[6], w1[7]};
    // 16-byte chunks of a tile row XOR-swizzled by the column: lanes (columns) 128 B
    // apart would otherwise all hit the same banks
    const int off = 16 * (g ^ (c & 7)) + 8 * hh;
    *reinterpret_cast<uint2*>(&tile[u][c][off]) = make_uint2(oz_gather_byte(a0, u), oz_gather_byte(a1, u));
    *reinterpret_cast<uint2*>(&tile[4 + u][c][off]) = make_uint2(oz_gather_byte(b0, u), oz_gather_byte(b1, u));
  }
}

// tile -> planes: 8 x 32 rows of 128 bytes (rows >= valid_rows of the block skipped)
__device__ __forceinline__ void oz_cd_store(const uint8_t (*tile)[OZ_CD_COLS][OZ_CD_ROWS], uint8_t* out,
                                            int64_t plane, int64_t P, int64_t f0, int64_t nc, int bytes) {
#pragma unroll
  for (int z = 0; z < 8; ++z) {
    const int q = threadIdx.x + 256 * z;  // 2048 pieces of 16 bytes
    const int u = q >> 8, c = (q >> 3) & 31, piece = q & 7;
    if (f0 + c < nc && 16 * piece < bytes)
      *reinterpret_cast<uint4*>(out + u * plane + (f0 + c) * P + 16 * piece) =
          *reinterpret_cast<const uint4*>(&tile[u][c][16 * (piece ^ (c & 7))]);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) oz_seg_coldigits_kernel(const T* __restrict__ B, int64_t ldb, int64_t strideB,
                                                               int64_t nc, int64_t nseg, int64_t nch,
                                                               const int4* __restrict__ cmap,
                                                               const uint32_t* __restrict__ ex, int64_t P,
                                                               uint8_t* __restrict__ planes) {
  __shared__ __align__(16) uint8_t tile[OZ_S][OZ_CD_COLS][OZ_CD_ROWS];
  const int64_t b = blockIdx.z;
  const int64_t ch0 = (int64_t)blockIdx.x * (OZ_CD_ROWS / 32);
  if (cmap[b * nch + ch0].x < 0) return;  // the block starts past the used extent
  const int g = threadIdx.x >> 5, c = threadIdx.x & 31;
  const int64_t f0 = (int64_t)blockIdx.y * OZ_CD_COLS, f = f0 + c;
  const bool fv = f < nc;
  const int4 cm = ch0 + g / 2 < nch ? cmap[b * nch + ch0 + g / 2] : make_int4(-1, 0, 0, 0);
  const int r0 = 16 * (g & 1);  // first row of this thread inside its 32-row chunk
  double s1 = 0.0, s2 = 0.0;
  if (fv && cm.x >= 0) oz_scales(oz_exponent_from_bits(ex[(b * nseg + cm.x) * nc + f]), s1, s2);
  const T* p = B + b * strideB + (int64_t)cm.y * ldb + f;
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int rr = r0 + 8 * hh + r;
      x[r] = (fv && cm.x >= 0 && rr < cm.z) ? oz_ld(p + (int64_t)rr * ldb) : 0.0;
    }
    uint32_t w0[8], w1[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) oz_digits(x[r], s1, s2, w0[r], w1[r]);
    oz_cd_stash8(tile, g, c, hh, w0, w1);
  }
  __syncthreads();
  // chunks past the used extent have no planes to fill (the tensor maps never read them)
  int used = 0;
  for (int q = 0; q < OZ_CD_ROWS / 32; ++q)
    if (ch0 + q < nch && cmap[b * nch + ch0 + q].x >= 0) used = q + 1;
  oz_cd_store(tile, planes + (b * OZ_S) * (nc * P) + 32 * ch0, nc * P, P, f0, nc, 32 * used);
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

// one box of all S digit planes: {32 bytes of K, rows, S planes}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

struct OzItem {
  int64_t b, j, tm, tn;
  int64_t k0;   // first K column of the planes (segment start / split start)
  int ktiles;   // stages (32 K each)
};

struct OzGeom {
  int64_t m, nc, nseg, TM, TN, items;
  // product mode (EPI_OUT): nseg = K splits, kinfo[2b] = inner length, kinfo[2b+1] = split chunk
  const int64_t* kinfo;
  double* out;
  int64_t ldo, strideO;
};

enum { EPI_SEG = 0, EPI_OUT = 1 };

// MC = 2: items are column-tile PAIRS (tn = 2 tnp + rank) computed by a CTA pair
template <int EPI, int MC = 1>
__device__ __forceinline__ OzItem oz_item(const OzGeom& g, int64_t it, const int32_t* __restrict__ perm,
                                          const int64_t* __restrict__ po, const int32_t* __restrict__ L,
                                          int rank = 0) {
  OzItem r;
  const int64_t TNI = (g.TN + MC - 1) / MC;  // column tiles (or pairs) per row of tiles
  const int64_t tiles = g.TM * TNI;
  if constexpr (EPI == EPI_SEG) {
    const int64_t tile = it % tiles;
    const int64_t rest = it / tiles;
    const int64_t rank_ = rest % g.nseg;
    r.b = rest / g.nseg;
    r.j = perm[r.b * g.nseg + rank_];
    r.tn = (tile % TNI) * MC + rank;
    r.tm = tile / TNI;
    r.k0 = po[r.b * g.nseg + r.j];
    r.ktiles = L[r.b * g.nseg + r.j] / OZ_BK;
  } else {
    // every tile of one K split before the next split: the co-resident CTAs share
    // that split's digit planes through L2
    const int64_t tile = it % tiles;
    r.j = (it / tiles) % g.nseg;  // K split
    r.b = it / (g.nseg * tiles);
    r.tn = (tile % TNI) * MC + rank;
    r.tm = tile / TNI;
    const int64_t kd = g.kinfo[2 * r.b], chunk = g.kinfo[2 * r.b + 1];
    r.k0 = r.j * chunk;
    const int64_t k1 = min(kd, r.k0 + chunk);
    r.ktiles = k1 > r.k0 ? (int)((k1 - r.k0 + OZ_BK - 1) / OZ_BK) : 0;
  }
  return r;
}

// Persistent: CTA c takes items c, c + G, ... of the item list (segments
// longest first).  EPI_SEG: per-tile square sums of the product into part;
// EPI_OUT: the product tile itself (float64) into out, or into the split-K
// partials part[b][split] when nseg > 1.  Exponents: EPI_SEG int e per
// (segment, row/column); EPI_OUT biased exponent fields (oz_exponent_from_bits).
// MC = 2: a cluster of two CTAs computes two adjacent column tiles of the same
// rows; each loads one 64-row half of every A digit plane and multicasts it to
// both (A read from L2 once per pair: a third less operand traffic), and a
// stage is refilled only after both CTAs' MMAs have read it.
template <int EPI, int MC = 1>
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_mma_kernel(const __grid_constant__ CUtensorMap tm_a,
                                                                 const __grid_constant__ CUtensorMap tm_b,
                                                                 const __grid_constant__ CUtensorMap tm_a2, OzGeom geo,
                                                                 const int32_t* __restrict__ perm,
                                                                 const int64_t* __restrict__ po,
                                                                 const int32_t* __restrict__ L,
                                                                 const int32_t* __restrict__ exA,
                                                                 const int32_t* __restrict__ exB,
                                                                 double* __restrict__ part, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZ_STAGES * OZ_STAGE);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* acc_full = empty + OZ_STAGES;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  double* wcol = reinterpret_cast<double*>(smem + OZ_STAGES * OZ_STAGE + 256);  // [2][64]
  double* red = wcol + 128;                                                     // [OZ_EPI_WARPS]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t crank = 0;
  if constexpr (MC > 1) asm("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
  const int64_t first = blockIdx.x / MC, step = gridDim.x / MC;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);  // every CTA of the pair commits its reads of the stage
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, OZ_EPI_WARPS);
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
  if constexpr (MC > 1) cluster_sync_all();  // the peer's barriers exist before any multicast lands
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer: the S digit planes of A and B for every stage
      uint32_t it = 0;
      for (int64_t w = first; w < geo.items; w += step) {
        const OzItem I = oz_item<EPI, MC>(geo, w, perm, po, L, (int)crank);
        const int arow = (int)(I.tm * OZ_BM), brow = (int)(I.tn * OZ_BN), plane0 = (int)(I.b * OZ_S);
        for (int kt = 0; kt < I.ktiles; ++kt, ++it) {
          const int s = it % OZ_STAGES;
          if (it >= OZ_STAGES) mbar_wait(&empty[s], ((it / OZ_STAGES) - 1) & 1);
          uint8_t* st = smem + s * OZ_STAGE;
          if (mode == 2) {  // timing experiment: no operand loads
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_expect_tx(&full[s], OZ_STAGE);
          const int kc = (int)(I.k0 + kt * OZ_BK);
          // rows past m / nc are zero-filled by the tensor map bounds
          if constexpr (MC > 1) {
            // this CTA's 64-row half of every A plane, to both CTAs (2-D map over the
            // stacked planes: rows past m belong to the next plane, masked in the epilogue)
#pragma unroll
            for (int t = 0; t < OZ_S; ++t)
              tma_load_2d_mc(st + t * OZ_A_PLANE + crank * (OZ_A_PLANE / 2), &tm_a2, &full[s], kc,
                             (int)((I.b * OZ_S + t) * geo.m) + arow + (int)crank * 64, 0x3);
          } else {
            tma_load_3d(st, &tm_a, &full[s], kc, arow, plane0);
          }
          tma_load_3d(st + OZ_S * OZ_A_PLANE, &tm_b, &full[s], kc, brow, plane0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: per stage, A plane t x B planes 0..S-1-t into levels t..S-1
      uint32_t it = 0, n_items = 0;
      for (int64_t w = first; w < geo.items; w += step) {
        const OzItem I = oz_item<EPI, MC>(geo, w, perm, po, L, (int)crank);
        if (I.ktiles == 0) continue;
        if (n_items > 0) mbar_wait(acc_empty, (n_items - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        for (int kt = 0; kt < I.ktiles; ++kt, ++it) {
          const int s = it % OZ_STAGES;
          mbar_wait(&full[s], (it / OZ_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t base = su32(smem + s * OZ_STAGE);
          if (mode >= 3) {  // timing experiment: the same MACs as 9 (mode 3) or 18 (mode 4) uniform MMAs
            const int nn = mode == 3 ? 256 : 128;
            for (int i = 0; i < (mode == 3 ? 9 : 18); ++i)
              umma_i8(tmem + (uint32_t)((i & 1) * 256), umma_desc_sw32(base + (i & 7) * OZ_A_PLANE),
                      umma_desc_sw32(base + OZ_S * OZ_A_PLANE), idesc_i8(nn), (kt > 0 || i > 1) ? 1u : 0u);
            umma_commit(&empty[s]);
            continue;
          }
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
          if constexpr (MC > 1) umma_commit_mc(&empty[s], 0x3);  // both CTAs may refill after both read
          else umma_commit(&empty[s]);
        }
        umma_commit(acc_full);
        ++n_items;
      }
    }
  } else {
    // ---- epilogue: drain the 8 levels, square-sum the tile
    const int e_id = threadIdx.x - 64;  // 0 .. 32 * OZ_EPI_WARPS - 1
    const int quarter = warp & 3;       // TMEM lanes this warp may read
    const int cpart = (warp - 2) / 4;   // which OZ_EPI_COLS columns of the tile
    constexpr int EPI_T = 32 * OZ_EPI_WARPS;
    uint32_t n_items = 0;
    for (int64_t w = first; w < geo.items; w += step) {
      const OzItem I = oz_item<EPI, MC>(geo, w, perm, po, L, (int)crank);
      double* prow = part + ((I.b * geo.nseg + I.j) * geo.TM + I.tm) * geo.TN + I.tn;
      const int64_t row = I.tm * OZ_BM + quarter * 32 + lane;
      const int64_t col0 = I.tn * OZ_BN;
      double* orow = nullptr;  // EPI_OUT: this thread's output row (64 columns from col0)
      if constexpr (EPI == EPI_OUT) {
        orow = geo.nseg > 1 ? part + ((I.b * geo.nseg + I.j) * geo.m + row) * geo.nc
                            : geo.out + I.b * geo.strideO + row * geo.ldo;
      }
      if (I.ktiles == 0) {
        if constexpr (EPI == EPI_SEG) {
          if (e_id == 0 && I.tn < geo.TN) *prow = 0.0;
        } else if (row < geo.m) {
          for (int q = 0; q < OZ_BN; ++q)
            if (col0 + q < geo.nc) orow[col0 + q] = 0.0;
        }
        continue;
      }
      double* wc = wcol + 64 * (n_items & 1);
      if (e_id < 64) {
        const int64_t f = col0 + e_id;
        if constexpr (EPI == EPI_SEG)
          wc[e_id] = f < geo.nc
                         ? ldexp(1.0, oz_exponent_from_bits((uint32_t)exB[(I.b * geo.nseg + I.j) * geo.nc + f]) - 10)
                         : 0.0;
        else
          wc[e_id] = f < geo.nc ? ldexp(1.0, oz_exponent_from_bits((uint32_t)exB[I.b * geo.nc + f]) - 10) : 0.0;
      }
      named_sync(1, EPI_T);
      mbar_wait(acc_full, n_items & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (mode == 1) {  // timing experiment: release the accumulators at once
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
        ++n_items;
        continue;
      }
      double R = 0.0;
      double sr = 0.0;  // row scale 2^e_h
      if (row < geo.m) {
        if constexpr (EPI == EPI_SEG)
          sr = ldexp(1.0, exA[(I.b * geo.nseg + I.j) * geo.m + row]);
        else
          sr = ldexp(1.0, oz_exponent_from_bits((uint32_t)exA[I.b * geo.m + row]));
      }
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
      for (int c0 = cpart * OZ_EPI_COLS; c0 < (cpart + 1) * OZ_EPI_COLS; c0 += 16) {
        uint32_t v[OZ_S][16];
#pragma unroll
        for (int d = 0; d < OZ_S; ++d) tmem_ld16(tbase + (uint32_t)(d * OZ_BN + c0), v[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (c0 + 16 == (cpart + 1) * OZ_EPI_COLS) {
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t hi = ((int64_t)(int32_t)v[0][q] << 21) + ((int64_t)(int32_t)v[1][q] << 14) +
                             ((int64_t)(int32_t)v[2][q] << 7) + (int64_t)(int32_t)v[3][q];
          const int64_t lo = ((int64_t)(int32_t)v[4][q] << 21) + ((int64_t)(int32_t)v[5][q] << 14) +
                             ((int64_t)(int32_t)v[6][q] << 7) + (int64_t)(int32_t)v[7][q];
          // exact int64 -> double for |x| < 2^51 without the conversion unit
          const double hd = __longlong_as_double(hi + 0x4338000000000000ll) - 6755399441055744.0;
          const double ld = __longlong_as_double(lo + 0x4338000000000000ll) - 6755399441055744.0;
          const double x = fma(ld, 0x1p-49, hd * 0x1p-21) * wc[c0 + q];
          if constexpr (EPI == EPI_SEG) {
            R = fma(x, x, R);
          } else {
            if (row < geo.m && col0 + c0 + q < geo.nc) orow[col0 + c0 + q] = x * sr;
          }
        }
      }
      if constexpr (EPI == EPI_SEG) {
        R = (R * sr) * sr;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) R += __shfl_xor_sync(0xffffffffu, R, o);
        if (lane == 0) red[warp - 2] = R;
        named_sync(1, EPI_T);
        if (e_id == 0 && I.tn < geo.TN) {  // (a pair's phantom tile past the last column has no slot)
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < OZ_EPI_WARPS; ++q) t += red[q];
          *prow = t;
        }
      }
      ++n_items;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(OZ_TMEM_COLS));
  }
  // the peer's last multicast loads and MMA commits target this CTA's shared memory
  if constexpr (MC > 1) cluster_sync_all();
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

// ---------------------------------------------------------------- product mode
// out[b] = A[b] (m x k) @ B[b] (k x nc) in float64 through the same digit planes:
// one scale per row of A / column of B over the whole inner length (biased
// exponent fields, atomicMax over K chunks), digits written chunk-parallel,
// K split across CTAs when the output has few tiles, partials reduced in a
// fixed order.  Gathered operands (the sampled sketch, estimators.py:78-81):
// A[h, t] = M[h, col[t]] * scale[t], B[t, f] = N[col[t], f] * scale[t], one
// float64 rounding as in the reference, then split.

// Optional balance exponents kx[k]: A[:, k] 2^kx[k] and B[k, :] 2^-kx[k] (exact;
// the product is unchanged) so the per-row / per-column digit scales are set
// by the terms that dominate the product rather than by one operand's range.
template <typename T, bool G>
struct OzRows {  // A[h, k]
  const T* base; int64_t ld; const int64_t* col; const double* sc; const int32_t* kx;
  __device__ __forceinline__ double at(int64_t h, int64_t k) const {
    double v;
    if constexpr (G) v = __dmul_rn(oz_ld(base + h * ld + col[k]), sc[k]);
    else v = oz_ld(base + h * ld + k);
    return kx != nullptr ? v * oz_pow2(kx[k]) : v;
  }
};

template <typename T, bool G>
struct OzCols {  // B[k, f]
  const T* base; int64_t ld; const int64_t* col; const double* sc; const int32_t* kx;
  __device__ __forceinline__ double at(int64_t k, int64_t f) const {
    double v;
    if constexpr (G) v = __dmul_rn(oz_ld(base + col[k] * ld + f), sc[k]);
    else v = oz_ld(base + k * ld + f);
    return kx != nullptr ? v * oz_pow2(-kx[k]) : v;
  }
};

// kexp[t] = round(log2(||N_i|| / ||M_i||) / 2), i = column[t] (or t): the sketch
// columns of C and rows of D both scaled to ~sqrt(||M_i|| ||N_i||) s_t
__global__ void oz_balance_kernel(const double* __restrict__ colsq, const double* __restrict__ rowsq,
                                  int64_t n_stride, const int64_t* __restrict__ column, int64_t w, int64_t w_stride,
                                  const int64_t* __restrict__ kdev, int32_t* __restrict__ kexp) {
  const int64_t b = blockIdx.y;
  const int64_t kd = kdev != nullptr ? min(kdev[b], w) : w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < w; t += (int64_t)gridDim.x * blockDim.x) {
    int32_t e = 0;
    if (t < kd) {
      const int64_t i = column != nullptr ? column[b * w_stride + t] : t;
      const double c = colsq[b * n_stride + i], r = rowsq[b * n_stride + i];
      if (c > 0.0 && r > 0.0 && c < 1e300 && r < 1e300) {
        const int d = ilogb(r) - ilogb(c);  // log2(||N_i||^2 / ||M_i||^2)
        e = (int32_t)((d >= 0 ? d + 2 : d - 2) / 4);
        e = max(-200, min(200, e));
      }
    }
    kexp[b * w_stride + t] = e;
  }
}

// per problem: inner length, split chunk; zero the exponent maxima
__global__ void oz_gemm_prep_kernel(const int64_t* __restrict__ kdev, int64_t kmax, int64_t splits, int64_t m,
                                    int64_t nc, int64_t* __restrict__ kinfo, uint32_t* __restrict__ exA,
                                    uint32_t* __restrict__ exB) {
  const int64_t b = blockIdx.x;
  if (threadIdx.x == 0) {
    int64_t kd = kdev != nullptr ? kdev[b] : kmax;
    kd = kd < 0 ? 0 : (kd > kmax ? kmax : kd);
    int64_t chunk = (kd + splits - 1) / splits;
    chunk = ((chunk + OZ_BK - 1) / OZ_BK) * OZ_BK;
    kinfo[2 * b] = kd;
    kinfo[2 * b + 1] = chunk < OZ_BK ? OZ_BK : chunk;
  }
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) exA[b * m + i] = 0u;
  for (int64_t i = threadIdx.x; i < nc; i += blockDim.x) exB[b * nc + i] = 0u;
}

// row maxima of A: warp per (row, OZ_RM_SPAN columns), all loads in flight
constexpr int OZ_RM_SPAN = 512;
template <typename T, bool G>
__global__ void __launch_bounds__(256) oz_rowmax_kernel(OzRows<T, G> A, int64_t strideA, int64_t w_stride, int64_t m,
                                                        const int64_t* __restrict__ kinfo, uint32_t* __restrict__ exA) {
  const int lane = threadIdx.x & 31;
  const int64_t h = (int64_t)blockIdx.y * 8 + (threadIdx.x >> 5), b = blockIdx.z;
  const int64_t kd = kinfo[2 * b];
  const int64_t base = (int64_t)blockIdx.x * OZ_RM_SPAN;
  if (h >= m || base >= kd) return;
  OzRows<T, G> a = A;
  a.base += b * strideA;
  if constexpr (G) { a.col += b * w_stride; a.sc += b * w_stride; }
  if (a.kx != nullptr) a.kx += b * w_stride;
  double v[OZ_RM_SPAN / 32];
#pragma unroll
  for (int it = 0; it < OZ_RM_SPAN / 128; ++it)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = base + 128 * it + 4 * lane + q;
      v[4 * it + q] = i < kd ? a.at(h, i) : 0.0;
    }
  uint32_t eb = 0;
#pragma unroll
  for (int q = 0; q < OZ_RM_SPAN / 32; ++q) eb = max(eb, oz_ebits(v[q]));
  eb = __reduce_max_sync(0xffffffffu, eb);
  if (lane == 0 && eb != 0) atomicMax(&exA[b * m + h], eb);
}

// column maxima of B: thread per column, 32 rows
template <typename T, bool G>
__global__ void __launch_bounds__(256) oz_colmax_kernel(OzCols<T, G> B, int64_t strideB, int64_t w_stride, int64_t nc,
                                                        const int64_t* __restrict__ kinfo, uint32_t* __restrict__ exB) {
  const int64_t f = (int64_t)blockIdx.y * 256 + threadIdx.x, b = blockIdx.z;
  const int64_t kd = kinfo[2 * b];
  const int64_t k0 = (int64_t)blockIdx.x * 32;
  if (f >= nc || k0 >= kd) return;
  OzCols<T, G> a = B;
  a.base += b * strideB;
  if constexpr (G) { a.col += b * w_stride; a.sc += b * w_stride; }
  if (a.kx != nullptr) a.kx += b * w_stride;
  const int64_t k1 = min(kd, k0 + 32);
  uint32_t eb = 0;
  int64_t k = k0;
  for (; k + 8 <= k1; k += 8) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = a.at(k + r, f);
#pragma unroll
    for (int r = 0; r < 8; ++r) eb = max(eb, oz_ebits(v[r]));
  }
  for (; k < k1; ++k) eb = max(eb, oz_ebits(a.at(k, f)));
  if (eb != 0) atomicMax(&exB[b * nc + f], eb);
}

// digit planes of A: warp per (row, OZ_RD_SPAN columns), zero past the inner length
constexpr int OZ_RD_SPAN = 256;
template <typename T, bool G>
__global__ void __launch_bounds__(256) oz_rowdigits_kernel(OzRows<T, G> A, int64_t strideA, int64_t w_stride, int64_t m,
                                                           const int64_t* __restrict__ kinfo,
                                                           const uint32_t* __restrict__ exA, int64_t P,
                                                           uint8_t* __restrict__ planes) {
  const int lane = threadIdx.x & 31;
  const int64_t h = (int64_t)blockIdx.y * 8 + (threadIdx.x >> 5), b = blockIdx.z;
  const int64_t kd = kinfo[2 * b];
  const int64_t kpad = ((kd + OZ_BK - 1) / OZ_BK) * OZ_BK;
  const int64_t base = (int64_t)blockIdx.x * OZ_RD_SPAN;
  if (h >= m || base >= kpad) return;
  OzRows<T, G> a = A;
  a.base += b * strideA;
  if constexpr (G) { a.col += b * w_stride; a.sc += b * w_stride; }
  if (a.kx != nullptr) a.kx += b * w_stride;
  double s1, s2;
  oz_scales(oz_exponent_from_bits(exA[b * m + h]), s1, s2);
  double x[OZ_RD_SPAN / 32];
#pragma unroll
  for (int it = 0; it < OZ_RD_SPAN / 128; ++it)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = base + 128 * it + 4 * lane + q;
      x[4 * it + q] = i < kd ? a.at(h, i) : 0.0;
    }
  const int64_t plane = m * P;
#pragma unroll
  for (int it = 0; it < OZ_RD_SPAN / 128; ++it) {
    const int64_t i0 = base + 128 * it + 4 * lane;
    if (i0 >= kpad) break;
    uint32_t w0[4], w1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) oz_digits(x[4 * it + q], s1, s2, w0[q], w1[q]);
    uint8_t* o = planes + ((b * OZ_S) * m + h) * P + i0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      *reinterpret_cast<uint32_t*>(o + u * plane) = oz_gather_byte(w0, u);
      *reinterpret_cast<uint32_t*>(o + (4 + u) * plane) = oz_gather_byte(w1, u);
    }
  }
}

// digit planes of B^T: CTA per (128 rows, 32 columns), transposed in shared memory
template <typename T, bool G>
__global__ void __launch_bounds__(256) oz_coldigits_kernel(OzCols<T, G> B, int64_t strideB, int64_t w_stride,
                                                           int64_t nc, const int64_t* __restrict__ kinfo,
                                                           const uint32_t* __restrict__ exB, int64_t P,
                                                           uint8_t* __restrict__ planes) {
  __shared__ __align__(16) uint8_t tile[OZ_S][OZ_CD_COLS][OZ_CD_ROWS];
  const int64_t b = blockIdx.z;
  const int64_t kd = kinfo[2 * b];
  const int64_t kpad = ((kd + OZ_BK - 1) / OZ_BK) * OZ_BK;
  const int64_t k0 = (int64_t)blockIdx.x * OZ_CD_ROWS;
  if (k0 >= kpad) return;
  const int g = threadIdx.x >> 5, c = threadIdx.x & 31;
  const int64_t f0 = (int64_t)blockIdx.y * OZ_CD_COLS, f = f0 + c;
  const bool fv = f < nc;
  OzCols<T, G> a = B;
  a.base += b * strideB;
  if constexpr (G) { a.col += b * w_stride; a.sc += b * w_stride; }
  if (a.kx != nullptr) a.kx += b * w_stride;
  double s1 = 0.0, s2 = 0.0;
  if (fv) oz_scales(oz_exponent_from_bits(exB[b * nc + f]), s1, s2);
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int64_t k = k0 + 16 * g + 8 * hh + r;
      x[r] = (fv && k < kd) ? a.at(k, f) : 0.0;
    }
    uint32_t w0[8], w1[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) oz_digits(x[r], s1, s2, w0[r], w1[r]);
    oz_cd_stash8(tile, g, c, hh, w0, w1);
  }
  __syncthreads();
  oz_cd_store(tile, planes + (b * OZ_S) * (nc * P) + k0, nc * P, P, f0, nc,
              (int)(kpad - k0 < OZ_CD_ROWS ? kpad - k0 : OZ_CD_ROWS));
}

// out[b] = sum over splits (fixed order) of part[b][split]
__global__ void oz_splitk_reduce_kernel(const double* __restrict__ part, int64_t splits, int64_t m, int64_t nc,
                                        int64_t batch, double* __restrict__ out, int64_t ldo, int64_t strideO) {
  const int64_t total = batch * m * nc;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g / (m * nc), r = g % (m * nc);
    const int64_t h = r / nc, f = r % nc;
    const double* p = part + (b * splits) * m * nc + r;
    double acc = p[0];
    for (int64_t s = 1; s < splits; ++s) acc += p[s * m * nc];
    out[b * strideO + h * ldo + f] = acc;
  }
}

// ---------------------------------------------------------------- host side

struct OzLayout {
  int64_t P;                 // padded inner extent (row pitch of the planes)
  int64_t off_a, off_b, off_exa, off_exb, off_po, off_L, off_perm, off_flag, off_part, off_cmap, total;
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
  l.off_cmap = o; o = al256(o + batch * (l.P / 32) * 16);
  l.total = o;
  return l;
}

// digit planes [plane][rows][P] as a 3-D tensor; box = all S planes of one
// 32-byte K slice of `box_rows` rows (SWIZZLE_32B)
static int oz_map(CUtensorMap* map, const uint8_t* base, int64_t rows, int64_t planes, int64_t P, int box_rows) {
  auto enc = get_encode();
  BMM_REQUIRE(enc != nullptr, BMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)P, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)P, (cuuint64_t)(P * rows)};
  cuuint32_t box[3] = {(cuuint32_t)OZ_BK, (cuuint32_t)box_rows, (cuuint32_t)OZ_S};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BMM_REQUIRE(r == CUDA_SUCCESS, BMM_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BMM_OK;
}

// 2-D view of the stacked digit planes ([planes * rows] x P) with 64-row boxes:
// the halves a CTA pair multicasts
static int oz_map2d(CUtensorMap* map, const uint8_t* base, int64_t rows, int64_t P) {
  auto enc = get_encode();
  BMM_REQUIRE(enc != nullptr, BMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)P};
  cuuint32_t box[2] = {(cuuint32_t)OZ_BK, 64u};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BMM_REQUIRE(r == CUDA_SUCCESS, BMM_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BMM_OK;
}

static int oz_nsm_count() {
  static int nsm = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    // BMM_OZ_CTAS: persistent CTAs of the g_k contraction (fewer leave SMs to concurrent graph branches)
    const char* e = getenv("BMM_OZ_CTAS");
    if (e != nullptr && atoi(e) >= 2 && atoi(e) < n) n = atoi(e) & ~1;
    return n;
  }();
  return nsm;
}

// Launch the persistent MMA kernel: CTA pairs sharing the A planes by multicast
// when there are at least two column tiles (BMM_OZ_PAIR=0 disables), else
// single CTAs.  geo.items is set here from the per-row item count `rows_items`
// (items with one column tile each = rows_items * TN).
template <int EPI>
static int oz_launch_mma(const CUtensorMap& ma, const CUtensorMap& mb, const uint8_t* planes_a, int64_t a_rows,
                         int64_t P, OzGeom geo, int64_t rows_items, const int32_t* perm, const int64_t* po,
                         const int32_t* L, const int32_t* exa, const int32_t* exb, double* part, int mode,
                         cudaStream_t st) {
  static const int pair_env = [] {
    const char* e = getenv("BMM_OZ_PAIR");
    return e ? atoi(e) : 1;
  }();
  const bool pair = pair_env != 0 && geo.TN >= 2 && mode == 0;
  static bool attr1 = false, attr2 = false;
  const int nsm = oz_nsm_count();
  if (!pair) {
    if (!attr1) {
      cudaFuncSetAttribute(oz_mma_kernel<EPI, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
      attr1 = true;
    }
    geo.items = rows_items * geo.TN;
    const unsigned grid = (unsigned)(geo.items < nsm ? geo.items : nsm);
    oz_mma_kernel<EPI, 1><<<grid, OZ_THREADS, OZ_SMEM, st>>>(ma, mb, ma, geo, perm, po, L, exa, exb, part, mode);
    BMM_CHECK_LAUNCH("oz_mma_kernel");
    return BMM_OK;
  }
  if (!attr2) {
    cudaFuncSetAttribute(oz_mma_kernel<EPI, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
    attr2 = true;
  }
  CUtensorMap ma2;
  int rc;
  if ((rc = oz_map2d(&ma2, planes_a, a_rows, P)) != BMM_OK) return rc;
  geo.items = rows_items * ((geo.TN + 1) / 2);
  const int64_t clusters = geo.items < nsm / 2 ? geo.items : nsm / 2;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(2 * clusters), 1, 1);
  lc.blockDim = dim3(OZ_THREADS, 1, 1);
  lc.dynamicSmemBytes = OZ_SMEM;
  lc.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = 2;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  lc.attrs = la;
  lc.numAttrs = 1;
  if (cudaLaunchKernelEx(&lc, oz_mma_kernel<EPI, 2>, ma, mb, ma2, geo, perm, po, L, exa, exb, part, mode) !=
      cudaSuccess) {
    set_error("oz_mma_kernel: cluster launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return BMM_E_CUDA;
  }
  count_launch();
  return BMM_OK;
}

}  // namespace bmm

using namespace bmm;

extern "C" int64_t bmm_segsq_i8_workspace(int64_t m, int64_t nc, int64_t n_inner, int64_t nseg, int64_t batch) {
  if (m < 1 || nc < 1 || n_inner < 0 || nseg < 1 || batch < 1) return 0;
  return oz_layout(m, nc, n_inner, nseg, batch).total;
}

static int segsq_i8_impl(int dtype, const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                         int64_t strideB, int64_t m, int64_t nc, int64_t n_inner, const int64_t* seg, int64_t nseg,
                         int64_t seg_stride, int64_t batch, double* gsq, void* ws, int64_t ws_bytes, void* stream,
                         cudaEvent_t* ev) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && n_inner >= 0 && nseg >= 1 && batch >= 1, BMM_E_ARG, "bmm_segsq_i8: bad shape");
  BMM_REQUIRE(A != nullptr && B != nullptr && seg != nullptr && gsq != nullptr, BMM_E_ARG,
              "bmm_segsq_i8: null pointer");
  BMM_REQUIRE(dtype == BMM_F64 || dtype == BMM_F32, BMM_E_ARG, "bmm_segsq_i8: unknown dtype %d", dtype);
  const OzLayout l = oz_layout(m, nc, n_inner, nseg, batch);
  BMM_REQUIRE(ws != nullptr && ws_bytes >= l.total, BMM_E_ARG, "bmm_segsq_i8: workspace too small (%lld < %lld)",
              (long long)ws_bytes, (long long)l.total);
  BMM_REQUIRE(batch * OZ_S * (m > nc ? m : nc) < (1LL << 31) && l.P < (1LL << 31), BMM_E_UNSUPPORTED,
              "bmm_segsq_i8: problem too large for 32-bit TMA coordinates");
  BMM_REQUIRE(nseg <= 65535 && batch <= 65535 && l.P / 32 < (1LL << 31) && ceil_div(m, 8) <= (1LL << 31) - 1 &&
                  ceil_div(nc, 64) <= 65535,
              BMM_E_UNSUPPORTED,
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

  if (ev) cudaEventRecord(ev[0], st);
  int4* cmap = (int4*)(w + l.off_cmap);
  const int64_t nch = l.P / 32;
  oz_prep_kernel<<<(unsigned)batch, 1024, 0, st>>>(seg, nseg, seg_stride, l.P, po, L, perm, flag, cmap);
  BMM_CHECK_LAUNCH("oz_prep_kernel");
  cudaMemsetAsync(exb, 0, (size_t)batch * nseg * nc * 4, st);
  dim3 ga((unsigned)ceil_div(m, 8), (unsigned)nseg, (unsigned)batch);
  dim3 gm((unsigned)nch, (unsigned)ceil_div(nc, 256), (unsigned)batch);
  dim3 gd((unsigned)ceil_div(nch, OZ_CD_ROWS / 32), (unsigned)ceil_div(nc, OZ_CD_COLS), (unsigned)batch);
  if (dtype == BMM_F64) {
    oz_split_rows_kernel<double><<<ga, 256, 0, st>>>((const double*)A, lda, strideA, m, seg, nseg, seg_stride, po, L,
                                                     l.P, pa, exa, flag);
    oz_seg_colmax_kernel<double><<<gm, 256, 0, st>>>((const double*)B, ldb, strideB, nc, nseg, nch, cmap,
                                                     (uint32_t*)exb);
    oz_seg_coldigits_kernel<double><<<gd, 256, 0, st>>>((const double*)B, ldb, strideB, nc, nseg, nch, cmap,
                                                        (const uint32_t*)exb, l.P, pb);
  } else {
    oz_split_rows_kernel<float><<<ga, 256, 0, st>>>((const float*)A, lda, strideA, m, seg, nseg, seg_stride, po, L,
                                                    l.P, pa, exa, flag);
    oz_seg_colmax_kernel<float><<<gm, 256, 0, st>>>((const float*)B, ldb, strideB, nc, nseg, nch, cmap,
                                                    (uint32_t*)exb);
    oz_seg_coldigits_kernel<float><<<gd, 256, 0, st>>>((const float*)B, ldb, strideB, nc, nseg, nch, cmap,
                                                       (const uint32_t*)exb, l.P, pb);
  }
  count_launch(2);
  BMM_CHECK_LAUNCH("oz_split_kernels");

  CUtensorMap ma, mb;
  int rc;
  if ((rc = oz_map(&ma, pa, m, batch * OZ_S, l.P, OZ_BM)) != BMM_OK) return rc;
  if ((rc = oz_map(&mb, pb, nc, batch * OZ_S, l.P, OZ_BN)) != BMM_OK) return rc;
  OzGeom geo;
  geo.m = m;
  geo.nc = nc;
  geo.nseg = nseg;
  geo.TM = ceil_div(m, OZ_BM);
  geo.TN = ceil_div(nc, OZ_BN);
  geo.kinfo = nullptr;
  geo.out = nullptr;
  geo.ldo = geo.strideO = 0;
  static const int mode = [] {
    const char* e = getenv("BMM_OZ_MODE");  // timing experiments only (1: no epilogue, 2: no loads)
    return e ? atoi(e) : 0;
  }();
  if (ev) cudaEventRecord(ev[1], st);
  if ((rc = oz_launch_mma<EPI_SEG>(ma, mb, pa, batch * OZ_S * m, l.P, geo, batch * nseg * geo.TM, perm, po, L, exa,
                                   exb, part, mode, st)) != BMM_OK)
    return rc;
  if (ev) cudaEventRecord(ev[2], st);
  oz_reduce_kernel<<<grid_for(batch * nseg, 128), 128, 0, st>>>(part, geo.TM * geo.TN, nseg, batch * nseg, flag, gsq);
  BMM_CHECK_LAUNCH("oz_reduce_kernel");
  if (ev) cudaEventRecord(ev[3], st);
  return BMM_OK;
}

extern "C" int bmm_segsq_i8(int dtype, const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                            int64_t strideB, int64_t m, int64_t nc, int64_t n_inner, const int64_t* seg, int64_t nseg,
                            int64_t seg_stride, int64_t batch, double* gsq, void* ws, int64_t ws_bytes,
                            void* stream) {
  return segsq_i8_impl(dtype, A, lda, strideA, B, ldb, strideB, m, nc, n_inner, seg, nseg, seg_stride, batch, gsq, ws,
                       ws_bytes, stream, nullptr);
}

extern "C" int bmm_segsq_i8_timed(int dtype, const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                                  int64_t strideB, int64_t m, int64_t nc, int64_t n_inner, const int64_t* seg,
                                  int64_t nseg, int64_t seg_stride, int64_t batch, double* gsq, void* ws,
                                  int64_t ws_bytes, void* stream, float* ms) {
  BMM_REQUIRE(ms != nullptr, BMM_E_ARG, "bmm_segsq_i8_timed: ms is NULL");
  cudaEvent_t ev[4];
  for (auto& e : ev) cudaEventCreate(&e);
  int rc = segsq_i8_impl(dtype, A, lda, strideA, B, ldb, strideB, m, nc, n_inner, seg, nseg, seg_stride, batch, gsq,
                         ws, ws_bytes, stream, ev);
  if (rc == BMM_OK) {
    cudaEventSynchronize(ev[3]);
    cudaEventElapsedTime(&ms[0], ev[0], ev[1]);
    cudaEventElapsedTime(&ms[1], ev[1], ev[2]);
    cudaEventElapsedTime(&ms[2], ev[2], ev[3]);
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

// ---------------------------------------------------------------- product mode host side
namespace bmm {
struct OzGemmLayout {
  int64_t P, splits;
  int64_t off_a, off_b, off_exa, off_exb, off_kinfo, off_part, total;
};

static int oz_nsm() {
  static int nsm = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return nsm;
}

// K splits: minimise waves x (stages per item + epilogue allowance), at least 8 stages per item
static int64_t oz_splits(int64_t tiles, int64_t k_max) {
  const int64_t kt = (k_max + OZ_BK - 1) / OZ_BK;
  const int64_t nsm = oz_nsm();
  const int64_t s_min = ceil_div(k_max, OZ_KMAX);  // exact int32 levels per split
  int64_t best = s_min;
  double best_cost = 1e300;
  for (int64_t s = s_min; s <= 16; ++s) {
    if (s > s_min && ceil_div(kt, s) < 8) break;
    const double cost = (double)ceil_div(tiles * s, nsm) * (double)(ceil_div(kt, s) + 3);
    if (cost < best_cost * 0.97) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

static OzGemmLayout oz_gemm_layout(int64_t m, int64_t nc, int64_t k_max, int64_t batch) {
  OzGemmLayout l;
  l.P = ((k_max + OZ_BK - 1) / OZ_BK) * OZ_BK;
  l.splits = oz_splits(batch * ceil_div(m, OZ_BM) * ceil_div(nc, OZ_BN), k_max);
  int64_t o = 0;
  l.off_a = o;     o = al256(o + batch * OZ_S * m * l.P);
  l.off_b = o;     o = al256(o + batch * OZ_S * nc * l.P);
  l.off_exa = o;   o = al256(o + batch * m * 4);
  l.off_exb = o;   o = al256(o + batch * nc * 4);
  l.off_kinfo = o; o = al256(o + batch * 16);
  l.off_part = o;  o = al256(o + (l.splits > 1 ? batch * l.splits * m * nc * 8 : 0));
  l.total = o;
  return l;
}
}  // namespace bmm

extern "C" int64_t bmm_gemm_i8_workspace(int64_t m, int64_t nc, int64_t k_max, int64_t batch) {
  if (m < 1 || nc < 1 || k_max < 1 || batch < 1) return 0;
  return oz_gemm_layout(m, nc, k_max, batch).total;
}

template <typename T, bool G>
static void oz_gemm_split_launch(const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                                 int64_t strideB, const int64_t* col, const double* scale, const int32_t* kexp,
                                 int64_t w_stride, int64_t m, int64_t nc, int64_t batch, const OzGemmLayout& l,
                                 uint8_t* w, cudaStream_t st) {
  const int64_t* kinfo = (const int64_t*)(w + l.off_kinfo);
  uint32_t* exa = (uint32_t*)(w + l.off_exa);
  uint32_t* exb = (uint32_t*)(w + l.off_exb);
  OzRows<T, G> ra{(const T*)A, lda, col, scale, kexp};
  OzCols<T, G> cb{(const T*)B, ldb, col, scale, kexp};
  dim3 grm((unsigned)ceil_div(l.P, OZ_RM_SPAN), (unsigned)ceil_div(m, 8), (unsigned)batch);
  dim3 grd((unsigned)ceil_div(l.P, OZ_RD_SPAN), (unsigned)ceil_div(m, 8), (unsigned)batch);
  dim3 gc((unsigned)ceil_div(l.P, 32), (unsigned)ceil_div(nc, 256), (unsigned)batch);
  dim3 gd((unsigned)ceil_div(l.P, OZ_CD_ROWS), (unsigned)ceil_div(nc, OZ_CD_COLS), (unsigned)batch);
  oz_rowmax_kernel<T, G><<<grm, 256, 0, st>>>(ra, strideA, w_stride, m, kinfo, exa);
  oz_colmax_kernel<T, G><<<gc, 256, 0, st>>>(cb, strideB, w_stride, nc, kinfo, exb);
  oz_rowdigits_kernel<T, G><<<grd, 256, 0, st>>>(ra, strideA, w_stride, m, kinfo, exa, l.P, w + l.off_a);
  oz_coldigits_kernel<T, G><<<gd, 256, 0, st>>>(cb, strideB, w_stride, nc, kinfo, exb, l.P, w + l.off_b);
  count_launch(3);
}

static int gemm_i8_impl(int dtype, const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                        int64_t strideB, const int64_t* col, const double* scale, const int32_t* kexp,
                        int64_t w_stride, int64_t m,
                        int64_t nc, int64_t k_max, const int64_t* k_dev, int64_t batch, double* out, int64_t ldo,
                        int64_t strideO, void* ws, int64_t ws_bytes, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && k_max >= 1 && batch >= 1, BMM_E_ARG, "bmm_gemm_i8: bad shape");
  BMM_REQUIRE(A != nullptr && B != nullptr && out != nullptr, BMM_E_ARG, "bmm_gemm_i8: null pointer");
  BMM_REQUIRE(dtype == BMM_F64 || dtype == BMM_F32, BMM_E_ARG, "bmm_gemm_i8: unknown dtype %d", dtype);
  BMM_REQUIRE(k_max <= OZ_KMAX * 16, BMM_E_UNSUPPORTED, "bmm_gemm_i8: k_max > %d", OZ_KMAX * 16);
  const OzGemmLayout l = oz_gemm_layout(m, nc, k_max, batch);
  BMM_REQUIRE(ceil_div(k_max, l.splits) <= OZ_KMAX, BMM_E_UNSUPPORTED, "bmm_gemm_i8: split longer than %d",
              OZ_KMAX);
  BMM_REQUIRE(ws != nullptr && ws_bytes >= l.total, BMM_E_ARG, "bmm_gemm_i8: workspace too small (%lld < %lld)",
              (long long)ws_bytes, (long long)l.total);
  BMM_REQUIRE(batch * OZ_S <= 65535 && batch <= 65535 && l.P < (1LL << 31) && m < (1LL << 31) && nc < (1LL << 31),
              BMM_E_UNSUPPORTED, "bmm_gemm_i8: problem too large");
  uint8_t* w = (uint8_t*)ws;
  cudaStream_t st = as_stream(stream);
  int64_t* kinfo = (int64_t*)(w + l.off_kinfo);
  oz_gemm_prep_kernel<<<(unsigned)batch, 256, 0, st>>>(k_dev, k_max, l.splits, m, nc, kinfo,
                                                       (uint32_t*)(w + l.off_exa), (uint32_t*)(w + l.off_exb));
  BMM_CHECK_LAUNCH("oz_gemm_prep_kernel");
  const bool g = col != nullptr;
  if (dtype == BMM_F64) {
    if (g) oz_gemm_split_launch<double, true>(A, lda, strideA, B, ldb, strideB, col, scale, kexp, w_stride, m, nc, batch, l, w, st);
    else oz_gemm_split_launch<double, false>(A, lda, strideA, B, ldb, strideB, col, scale, kexp, w_stride, m, nc, batch, l, w, st);
  } else {
    if (g) oz_gemm_split_launch<float, true>(A, lda, strideA, B, ldb, strideB, col, scale, kexp, w_stride, m, nc, batch, l, w, st);
    else oz_gemm_split_launch<float, false>(A, lda, strideA, B, ldb, strideB, col, scale, kexp, w_stride, m, nc, batch, l, w, st);
  }
  BMM_CHECK_LAUNCH("oz_digits_kernel");
  CUtensorMap ma, mb;
  int rc;
  if ((rc = oz_map(&ma, w + l.off_a, m, batch * OZ_S, l.P, OZ_BM)) != BMM_OK) return rc;
  if ((rc = oz_map(&mb, w + l.off_b, nc, batch * OZ_S, l.P, OZ_BN)) != BMM_OK) return rc;
  OzGeom geo;
  geo.m = m;
  geo.nc = nc;
  geo.nseg = l.splits;
  geo.TM = ceil_div(m, OZ_BM);
  geo.TN = ceil_div(nc, OZ_BN);
  geo.kinfo = kinfo;
  geo.out = out;
  geo.ldo = ldo;
  geo.strideO = strideO;
  double* part = (double*)(w + l.off_part);
  if ((rc = oz_launch_mma<EPI_OUT>(ma, mb, w + l.off_a, batch * OZ_S * m, l.P, geo, batch * l.splits * geo.TM,
                                   nullptr, nullptr, nullptr, (const int32_t*)(w + l.off_exa),
                                   (const int32_t*)(w + l.off_exb), part, 0, st)) != BMM_OK)
    return rc;
  if (l.splits > 1) {
    oz_splitk_reduce_kernel<<<grid_for(batch * m * nc, 256), 256, 0, st>>>(part, l.splits, m, nc, batch, out, ldo,
                                                                          strideO);
    BMM_CHECK_LAUNCH("oz_splitk_reduce_kernel");
  }
  return BMM_OK;
}

extern "C" int bmm_gemm_i8(int dtype, const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                           int64_t strideB, int64_t m, int64_t nc, int64_t k_max, const int64_t* k_dev,
                           const int32_t* kexp, int64_t batch, double* out, int64_t ldo, int64_t strideO, void* ws,
                           int64_t ws_bytes, void* stream) {
  return gemm_i8_impl(dtype, A, lda, strideA, B, ldb, strideB, nullptr, nullptr, kexp, k_max, m, nc, k_max, k_dev,
                      batch, out, ldo, strideO, ws, ws_bytes, stream);
}

extern "C" int bmm_gemm_i8_gather(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                  int64_t ldn, int64_t strideN, const int64_t* column, const double* scale,
                                  const int32_t* kexp, int64_t w_stride, int64_t m, int64_t nc, int64_t k_max,
                                  const int64_t* k_dev, int64_t batch, double* out, int64_t ldo, int64_t strideO,
                                  void* ws, int64_t ws_bytes, void* stream) {
  BMM_REQUIRE(column != nullptr && scale != nullptr, BMM_E_ARG, "bmm_gemm_i8_gather: column/scale is NULL");
  return gemm_i8_impl(dtype, M, ldm, strideM, N, ldn, strideN, column, scale, kexp, w_stride, m, nc, k_max, k_dev,
                      batch, out, ldo, strideO, ws, ws_bytes, stream);
}

extern "C" int bmm_balance_exponents(const double* colsq, const double* rowsq, int64_t n_stride,
                                     const int64_t* column, int64_t w, int64_t w_stride, const int64_t* k_dev,
                                     int64_t batch, int32_t* kexp, void* stream) {
  BMM_REQUIRE(colsq != nullptr && rowsq != nullptr && kexp != nullptr && w >= 1 && batch >= 1 && batch <= 65535,
              BMM_E_ARG, "bmm_balance_exponents: bad arguments");
  dim3 grid((unsigned)ceil_div(w, 256) < 1024u ? (unsigned)ceil_div(w, 256) : 1024u, (unsigned)batch);
  oz_balance_kernel<<<grid, 256, 0, as_stream(stream)>>>(colsq, rowsq, n_stride, column, w, w_stride, k_dev, kexp);
  BMM_CHECK_LAUNCH("oz_balance_kernel");
  return BMM_OK;
}
