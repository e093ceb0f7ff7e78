// K6 -- float32 sampled contraction on the 5th-generation tensor cores.
//
// C (m x W) @ D (W x p) for float32 inputs (configs 4 and 5), where the
// reference computes in float64 (estimators.py:143-144,175).  1xTF32 misses
// the 1e-5 tolerance at W = 32768, so every sketch value is split once,
// x = h + l with h = tf32_rna(x) and l = x - h, and
//     x.y ~= h_x.h_y            (kind::tf32, exact products)
//          + [h_x | l_x].[l_y | h_y]   (kind::f16 on bf16 pairs: both cross
//                                       terms in ONE K=16 MMA)
// accumulated into one float32 TMEM accumulator: two tensor instructions per
// 8 K-elements instead of three for 3xTF32, error ~2^-19 per product.
//
//   * bmm_gather_f32split: the K4 gather writes the operands K-major:
//       a_hi[b*m + h, t]   = h(M[h, column[t]] * scale[t])          (float32 / tf32)
//       a_x [b*m + h, t']  = bf16 pairs [h_x(8) | l_x(8)] per 8-column group
//       b_hi[b*p + f, t], b_x: the same for D^T with pairs [l_y(8) | h_y(8)]
//   * bmm_gemm_f32split: one CTA per 128x128 output tile; warp 0 drives TMA
//     (SWIZZLE_128B, 128-byte x 128-row boxes) into a 3-stage mbarrier ring,
//     one thread of warp 1 issues tcgen05.mma (M=128, N=128) into two TMEM
//     accumulators alternated every 128 K-elements, and four drain warps
//     promote each finished chunk into round-to-nearest float32 registers.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "tcgen05.cuh"
#include "balance.cuh"

namespace bmm {

constexpr int T_BM = 128, T_BK = 32;
constexpr int T_TILE_BYTES = T_BM * T_BK * 4;                // 16 KB: one A operand tile (128 rows)

// Tile configurations: 128x128 (3-stage ring, 4 drain warps) or 128x256 (one
// UMMA of N=256 per step: twice the flops per byte of A staged, 2-stage ring,
// the full 512-column TMEM for the two chunk accumulators, 8 drain warps)
template <int BN>
struct TCfg {
  static constexpr int STAGES = BN == 128 ? 3 : 2;
  static constexpr int B_TILE = BN * T_BK * 4;
  static constexpr int STAGE = 2 * T_TILE_BYTES + 2 * B_TILE;  // A_hi, A_x, B_hi, B_x
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr int DRAIN = BN / 32;  // drain warps: 32 TMEM lanes x 128 columns each
  static constexpr int WARPS = 2 + DRAIN;
  static constexpr int TMEM_COLS = 2 * BN;
};

// Instruction descriptor: F32 accumulate, TF32 A/B, both K-major, M=128, N=BN.
template <int BN>
constexpr uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(T_BM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// kind::f16 with BF16 A/B, F32 accumulate, K-major, M=128, N=BN (K = 16 per MMA).
template <int BN>
constexpr uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(T_BM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Warp roles: 0 = TMA producer, 1 = MMA issuer, 2..5 = accumulator drain /
// epilogue (warp w reads TMEM lanes 32*(w%4) .. +31, the quarter it may access).
//
// Chunked accumulation: the tensor core's float32 accumulate truncates, so
// its error grows linearly with K (measured ~6e-9 per K element).  Every
// T_CHUNK stages the MMA issuer switches between two TMEM accumulators
// (accumulate=0 at the chunk start) and the drain warps add the finished
// chunk into round-to-nearest float32 registers; the error then stays at one
// chunk's worth (~1e-6) for any W.
constexpr int T_CHUNK = 4;           // stages per accumulation chunk (128 K elements)

// MC = 2: CTA pairs (a cluster along the column-tile axis) compute two adjacent
// 128-column tiles of the same 128 rows; each CTA loads one 64-row half of the
// shared A tiles and multicasts it to both, so A is read from L2 once per pair
// (a quarter less operand traffic per flop).  A stage may be refilled only when
// both CTAs' MMAs have read it: the MMA commits arrive on both CTAs' `empty`
// barriers (count 2).
template <int BN, int MC = 1>
__global__ void __launch_bounds__(32 * TCfg<BN>::WARPS, 1) gemm_f32split_kernel(
    const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_ax,
    const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_bx, int64_t m, int64_t nc,
    int64_t k, float* __restrict__ out, int64_t ldo, int64_t strideO, const int64_t* __restrict__ kdev) {
  using Cfg = TCfg<BN>;
  constexpr int T_STAGES = Cfg::STAGES, T_STAGE_BYTES = Cfg::STAGE, T_BN = BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + T_STAGES * T_STAGE_BYTES);
  uint64_t* empty = full + T_STAGES;
  uint64_t* acc_full = empty + T_STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.z;
  uint32_t rank = 0;
  if constexpr (MC > 1) asm("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  // Grouped rasterisation: consecutive CTAs (clusters) sweep GROUP_M row tiles
  // before moving to the next column tile, so the ~148 co-resident CTAs share
  // both their A row blocks and their B column blocks through L2 (row-major
  // launch order would re-stream all of B from HBM once per row block).
  constexpr int GROUP_M = 16;
  int tile_m, tile_n;
  {
    const int tm = gridDim.y, tn = gridDim.x / MC;
    const int lin = blockIdx.y * tn + blockIdx.x / MC;
    const int group = lin / (GROUP_M * tn);
    const int first_m = group * GROUP_M;
    const int gsz = min(tm - first_m, GROUP_M);
    tile_m = first_m + (lin % (GROUP_M * tn)) % gsz;
    tile_n = ((lin % (GROUP_M * tn)) / gsz) * MC + (int)rank;
  }
  if (kdev != nullptr) {  // compressed sketch: contract the first ceil32(count) columns (zero-padded)
    const int64_t kd = ((kdev[b] + T_BK - 1) / T_BK) * T_BK;
    k = kd < k ? kd : k;
  }
  const int a_row0 = (int)(b * m + (int64_t)tile_m * T_BM);
  const int b_row0 = (int)(b * nc + (int64_t)tile_n * T_BN);
  const int ktiles = (int)((k + T_BK - 1) / T_BK);
  const int nchunks = (ktiles + T_CHUNK - 1) / T_CHUNK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < T_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);  // every CTA of the pair commits its reads of the stage
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&acc_full[q], 1);
      mbar_init(&acc_empty[q], Cfg::DRAIN);  // one arrive per drain warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_ax)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_bx)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if constexpr (MC > 1) cluster_sync_all();  // peers' barriers exist before any multicast lands
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % T_STAGES;
        if (kt >= T_STAGES) mbar_wait(&empty[s], ((kt / T_STAGES) - 1) & 1);
        uint8_t* st = smem + s * T_STAGE_BYTES;
        mbar_expect_tx(&full[s], T_STAGE_BYTES);
        const int kc = kt * T_BK;
        if constexpr (MC > 1) {
          // this CTA's 64-row half of the shared A tiles, to both CTAs
          const uint32_t half = rank * (T_TILE_BYTES / 2);
          tma_load_2d_mc(st + 0 * T_TILE_BYTES + half, &tm_ahi, &full[s], kc, a_row0 + (int)rank * 64, 0x3);
          tma_load_2d_mc(st + 1 * T_TILE_BYTES + half, &tm_ax, &full[s], kc, a_row0 + (int)rank * 64, 0x3);
        } else {
          tma_load_2d(st + 0 * T_TILE_BYTES, &tm_ahi, &full[s], kc, a_row0);
          tma_load_2d(st + 1 * T_TILE_BYTES, &tm_ax, &full[s], kc, a_row0);
        }
        tma_load_2d(st + 2 * T_TILE_BYTES, &tm_bhi, &full[s], kc, b_row0);
        tma_load_2d(st + 2 * T_TILE_BYTES + Cfg::B_TILE, &tm_bx, &full[s], kc, b_row0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % T_STAGES;
        const int chunk = kt / T_CHUNK, q = chunk & 1;
        const bool first = (kt % T_CHUNK) == 0;
        if (first && chunk >= 2) mbar_wait(&acc_empty[q], ((chunk >> 1) - 1) & 1);
        mbar_wait(&full[s], (kt / T_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t base = su32(smem + s * T_STAGE_BYTES);
        const uint32_t acc = tmem + (uint32_t)(q * T_BN);
#pragma unroll
        for (int kk = 0; kk < T_BK / 8; ++kk) {
          // 8 K-elements = 32 bytes of the 128-byte swizzle row: 8 tf32 values,
          // or the 16 bf16 of one cross-term pair group
          const uint32_t off = kk * 32;
          const uint64_t ahi = umma_desc_sw128(base + 0 * T_TILE_BYTES + off);
          const uint64_t ax = umma_desc_sw128(base + 1 * T_TILE_BYTES + off);
          const uint64_t bhi = umma_desc_sw128(base + 2 * T_TILE_BYTES + off);
          const uint64_t bx = umma_desc_sw128(base + 2 * T_TILE_BYTES + Cfg::B_TILE + off);
          umma_bf16(acc, ax, bx, idesc_bf16<BN>(), !(first && kk == 0));  // h_x.l_y + l_x.h_y
          umma_tf32(acc, ahi, bhi, idesc_tf32<BN>(), 1);                  // h_x.h_y
        }
        if constexpr (MC > 1) umma_commit_mc(&empty[s], 0x3);  // both CTAs may refill after both read
        else umma_commit(&empty[s]);  // stage s free once these MMAs have read it
        if ((kt % T_CHUNK) == T_CHUNK - 1 || kt == ktiles - 1) umma_commit(&acc_full[q]);
      }
    }
  } else {
    // ---- drain: add each finished chunk into float32 registers, then store.
    // Warp w may read TMEM lanes 32*(w%4)..; with 8 drain warps the second four
    // take the upper 128 accumulator columns.
    constexpr int DC = 128;  // columns per drain warp
    const int quarter = warp & 3;
    const int half = (warp - 2) / 4;
    float sum[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) sum[c] = 0.f;
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      const int q = chunk & 1;
      mbar_wait(&acc_full[q], (chunk >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int c = 0; c < DC; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(q * T_BN + half * DC + c), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[c + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[q]);
    }
    const int64_t row = (int64_t)tile_m * T_BM + quarter * 32 + lane;
    if (row < m) {
      float* orow = out + b * strideO + row * ldo;
      const int64_t col0 = (int64_t)tile_n * T_BN + half * DC;
      const bool vec = (col0 + DC <= nc) && (ldo % 4) == 0 && ((reinterpret_cast<uintptr_t>(orow + col0) & 15) == 0);
      if (vec) {
        float4* o4 = reinterpret_cast<float4*>(orow + col0);
#pragma unroll
        for (int j = 0; j < DC / 4; ++j)
          o4[j] = make_float4(sum[4 * j], sum[4 * j + 1], sum[4 * j + 2], sum[4 * j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < DC; ++j)
          if (col0 + j < nc) orow[col0 + j] = sum[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(Cfg::TMEM_COLS));
  }
  // the peer's last MMA commits arrive on this CTA's barriers: leave together
  if constexpr (MC > 1) cluster_sync_all();
}

// ---- cta_group::2: one 256 x 256 output tile per CTA pair (a 2-CTA cluster on
// one TPC).  Each CTA stages 128 rows of A and 128 rows of B^T (its halves, 64 KB
// per stage as above); the leader issues tcgen05.mma.cta_group::2 with M = 256,
// N = 256, so each MMA reads A and B from BOTH CTAs' shared memory and writes
// each CTA's 128 rows x 256 columns of the accumulator into its own TMEM.  Per
// SM that is twice the outputs of the 128 x 128 kernel for the same shared
// memory, L2 and HBM operand bytes: half the operand traffic per flop.
//   * TMA: both CTAs load their halves with .cta_group::2, completing bytes on
//     the LEADER's full[s] barrier (expect_tx of both halves);
//   * MMA commits go to both CTAs' empty[s] (each refills its own stage) and,
//     at a chunk end, to both CTAs' acc_full[q];
//   * the 8 drain warps of each CTA promote their TMEM rows into float32
//     registers (as above) and arrive on the leader's acc_empty[q] (16 arrivals).
constexpr int P_STAGES = 3;
constexpr int P_STAGE = 4 * T_TILE_BYTES;           // A_hi, A_x, B_hi, B_x halves: 64 KB
constexpr int P_SMEM = P_STAGES * P_STAGE + 1024 + 256;
constexpr int P_DRAIN = 8;                           // 32 TMEM lanes x 128 columns each
constexpr int P_WARPS = 2 + P_DRAIN;

template <int M_, int N_>
constexpr uint32_t idesc_tf32_mn() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N_ >> 3) << 17) | ((uint32_t)(M_ >> 4) << 24);
}
template <int M_, int N_>
constexpr uint32_t idesc_bf16_mn() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N_ >> 3) << 17) | ((uint32_t)(M_ >> 4) << 24);
}

__device__ __forceinline__ uint32_t cluster_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(su32(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void umma2_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma2_bf16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma2_commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          su32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__global__ void __launch_bounds__(32 * P_WARPS, 1) gemm_f32split_2sm_kernel(
    const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_ax,
    const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_bx, int64_t m, int64_t nc,
    int64_t k, float* __restrict__ out, int64_t ldo, int64_t strideO, const int64_t* __restrict__ kdev) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE);
  uint64_t* empty = full + P_STAGES;
  uint64_t* acc_full = empty + P_STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.z;
  uint32_t rank;
  asm("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  constexpr int GROUP_M = 8;  // grouped rasterisation over 256 x 256 pair tiles
  int tile_m, tile_n;
  {
    const int tm = gridDim.y, tn = gridDim.x / 2;
    const int lin = blockIdx.y * tn + blockIdx.x / 2;
    const int group = lin / (GROUP_M * tn);
    const int first_m = group * GROUP_M;
    const int gsz = min(tm - first_m, GROUP_M);
    tile_m = first_m + (lin % (GROUP_M * tn)) % gsz;
    tile_n = (lin % (GROUP_M * tn)) / gsz;
  }
  if (kdev != nullptr) {
    const int64_t kd = ((kdev[b] + T_BK - 1) / T_BK) * T_BK;
    k = kd < k ? kd : k;
  }
  // this CTA's halves: A rows and B^T rows (= output columns) [128 * rank, +128) of the pair tile
  const int a_row0 = (int)(b * m + (int64_t)tile_m * 256 + 128 * rank);
  const int b_row0 = (int)(b * nc + (int64_t)tile_n * 256 + 128 * rank);
  const int ktiles = (int)((k + T_BK - 1) / T_BK);
  const int nchunks = (ktiles + T_CHUNK - 1) / T_CHUNK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full[s], 1);   // the leader's producer arrives (with both halves' bytes)
      mbar_init(&empty[s], 1);  // the leader's MMA commit, multicast to both CTAs
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&acc_full[q], 1);
      mbar_init(&acc_empty[q], 2 * P_DRAIN);  // both CTAs' drain warps (leader's barrier is used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_ax)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_bx)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers and TMEM exist before any cross-CTA signal
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t full0 = cluster_addr(&full[0], 0);  // the leader's full[] (same layout in both CTAs)

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): this CTA's halves into its own stage
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % P_STAGES;
        if (kt >= P_STAGES) mbar_wait(&empty[s], ((kt / P_STAGES) - 1) & 1);
        uint8_t* st = smem + s * P_STAGE;
        if (rank == 0) mbar_expect_tx(&full[s], 2 * P_STAGE);
        const uint32_t fb = full0 + (uint32_t)(s * sizeof(uint64_t));
        const int kc = kt * T_BK;
        tma_load_2d_2sm(st + 0 * T_TILE_BYTES, &tm_ahi, fb, kc, a_row0);
        tma_load_2d_2sm(st + 1 * T_TILE_BYTES, &tm_ax, fb, kc, a_row0);
        tma_load_2d_2sm(st + 2 * T_TILE_BYTES, &tm_bhi, fb, kc, b_row0);
        tma_load_2d_2sm(st + 3 * T_TILE_BYTES, &tm_bx, fb, kc, b_row0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---- MMA issuer (leader only): M = 256 (both CTAs' A halves), N = 256 (both B halves)
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % P_STAGES;
        const int chunk = kt / T_CHUNK, q = chunk & 1;
        const bool first = (kt % T_CHUNK) == 0;
        if (first && chunk >= 2) mbar_wait(&acc_empty[q], ((chunk >> 1) - 1) & 1);
        mbar_wait(&full[s], (kt / P_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t base = su32(smem + s * P_STAGE);
        const uint32_t acc = tmem + (uint32_t)(q * 256);
#pragma unroll
        for (int kk = 0; kk < T_BK / 8; ++kk) {
          const uint32_t off = kk * 32;
          const uint64_t ahi = umma_desc_sw128(base + 0 * T_TILE_BYTES + off);
          const uint64_t ax = umma_desc_sw128(base + 1 * T_TILE_BYTES + off);
          const uint64_t bhi = umma_desc_sw128(base + 2 * T_TILE_BYTES + off);
          const uint64_t bx = umma_desc_sw128(base + 3 * T_TILE_BYTES + off);
          umma2_bf16(acc, ax, bx, idesc_bf16_mn<256, 256>(), !(first && kk == 0));  // h_x.l_y + l_x.h_y
          umma2_tf32(acc, ahi, bhi, idesc_tf32_mn<256, 256>(), 1);                  // h_x.h_y
        }
        umma2_commit_mc(&empty[s]);  // both CTAs may refill stage s once these MMAs have read it
        if ((kt % T_CHUNK) == T_CHUNK - 1 || kt == ktiles - 1) umma2_commit_mc(&acc_full[q]);
      }
    }
  } else {
    // ---- drain (both CTAs): warp w reads TMEM lanes 32*(w%4).. of this CTA's 128 rows,
    // columns half*128 .. +128 of the 256
    constexpr int DC = 128;
    const int quarter = warp & 3;
    const int half = (warp - 2) / 4;
    const uint32_t ae0 = cluster_addr(&acc_empty[0], 0);
    float sum[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) sum[c] = 0.f;
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      const int q = chunk & 1;
      mbar_wait(&acc_full[q], (chunk >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int c = 0; c < DC; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(q * 256 + half * DC + c), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[c + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(
                         ae0 + (uint32_t)(q * sizeof(uint64_t)))
                     : "memory");
    }
    const int64_t row = (int64_t)tile_m * 256 + 128 * rank + quarter * 32 + lane;
    if (row < m) {
      float* orow = out + b * strideO + row * ldo;
      const int64_t col0 = (int64_t)tile_n * 256 + half * DC;
      const bool vec = (col0 + DC <= nc) && (ldo % 4) == 0 && ((reinterpret_cast<uintptr_t>(orow + col0) & 15) == 0);
      if (vec) {
        float4* o4 = reinterpret_cast<float4*>(orow + col0);
#pragma unroll
        for (int j = 0; j < DC / 4; ++j)
          o4[j] = make_float4(sum[4 * j], sum[4 * j + 1], sum[4 * j + 2], sum[4 * j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < DC; ++j)
          if (col0 + j < nc) orow[col0 + j] = sum[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs and arrivals target this CTA: leave together
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

// ---- F16 split, CTA pairs (round 2): C = h + l (two fp16 arrays) . D^T = h' + l',
// operands scaled by the balanced exponents and the problem's shift
// (bmm_balance_f16).  Per 16 K-elements three kind::f16 MMAs, h.h' + h.l' + l.h'
// (the TF32 form needs four tensor instructions) on 4 operand bytes per element
// (8 there; 6 in the first version, which kept the cross terms as [h|l].[l|h]
// pair tiles).  Stage = 64 K: A_h, A_l, B_h, B_l, one SWIZZLE_128B tile of 128 rows
// x 64 fp16 each: 64 KB per CTA, 3 stages; accumulators promoted every 128 K.
// power of two 2^k as a float (|k| <= 126)
__device__ __forceinline__ float pow2f(int k) { return __int_as_float((127 + k) << 23); }

constexpr int H_BK = 64;
constexpr int H_TILE = 128 * 128;  // 16 KB
constexpr int H_STAGES = 3;
constexpr int H_STAGE = 4 * H_TILE;  // A_h, A_l, B_h, B_l
constexpr int H_SMEM = H_STAGES * H_STAGE + 1024 + 256;
constexpr int H_CHUNK_DEFAULT = 2;  // stages per promotion chunk (128 K)

template <int M_, int N_>
constexpr uint32_t idesc_f16_mn() {  // kind::f16, A/B F16, D F32, K-major
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N_ >> 3) << 17) | ((uint32_t)(M_ >> 4) << 24);
}

template <int H_CHUNK>
__global__ void __launch_bounds__(32 * P_WARPS, 1) gemm_f16split_2sm_kernel(
    const __grid_constant__ CUtensorMap tm_ah, const __grid_constant__ CUtensorMap tm_ax,
    const __grid_constant__ CUtensorMap tm_bh, const __grid_constant__ CUtensorMap tm_bx, int64_t m, int64_t nc,
    int64_t k, float* __restrict__ out, int64_t ldo, int64_t strideO, const int64_t* __restrict__ kdev,
    const int32_t* __restrict__ gshift, int group_m) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + H_STAGES * H_STAGE);
  uint64_t* empty = full + H_STAGES;
  uint64_t* acc_full = empty + H_STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.z;
  uint32_t rank;
  asm("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const int GROUP_M = group_m;  // grouped rasterisation over 256 x 256 pair tiles (default 8)
  int tile_m, tile_n;
  {
    const int tm = gridDim.y, tn = gridDim.x / 2;
    const int lin = blockIdx.y * tn + blockIdx.x / 2;
    const int group = lin / (GROUP_M * tn);
    const int first_m = group * GROUP_M;
    const int gsz = min(tm - first_m, GROUP_M);
    tile_m = first_m + (lin % (GROUP_M * tn)) % gsz;
    tile_n = (lin % (GROUP_M * tn)) / gsz;
  }
  if (kdev != nullptr) {
    const int64_t kd = ((kdev[b] + H_BK - 1) / H_BK) * H_BK;
    k = kd < k ? kd : k;
  }
  const int a_row0 = (int)(b * m + (int64_t)tile_m * 256 + 128 * rank);
  const int b_row0 = (int)(b * nc + (int64_t)tile_n * 256 + 128 * rank);
  const int ktiles = (int)((k + H_BK - 1) / H_BK);
  const int nchunks = (ktiles + H_CHUNK - 1) / H_CHUNK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < H_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&acc_full[q], 1);
      mbar_init(&acc_empty[q], 2 * P_DRAIN);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_ah)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_ax)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_bh)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_bx)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t full0 = cluster_addr(&full[0], 0);

  if (warp == 0) {
    if (lane == 0) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % H_STAGES;
        if (kt >= H_STAGES) mbar_wait(&empty[s], ((kt / H_STAGES) - 1) & 1);
        uint8_t* st = smem + s * H_STAGE;
        if (rank == 0) mbar_expect_tx(&full[s], 2 * H_STAGE);
        const uint32_t fb = full0 + (uint32_t)(s * sizeof(uint64_t));
        const int kc = kt * H_BK;
        tma_load_2d_2sm(st + 0 * H_TILE, &tm_ah, fb, kc, a_row0);
        tma_load_2d_2sm(st + 1 * H_TILE, &tm_ax, fb, kc, a_row0);  // A_l
        tma_load_2d_2sm(st + 2 * H_TILE, &tm_bh, fb, kc, b_row0);
        tma_load_2d_2sm(st + 3 * H_TILE, &tm_bx, fb, kc, b_row0);  // B_l
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_f16_mn<256, 256>();
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % H_STAGES;
        const int chunk = kt / H_CHUNK, q = chunk & 1;
        const bool first = (kt % H_CHUNK) == 0;
        if (first && chunk >= 2) mbar_wait(&acc_empty[q], ((chunk >> 1) - 1) & 1);
        mbar_wait(&full[s], (kt / H_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t base = su32(smem + s * H_STAGE);
        const uint32_t acc = tmem + (uint32_t)(q * 256);
#pragma unroll
        for (int kk = 0; kk < H_BK / 16; ++kk) {
          // elements 16kk .. 16kk+15 (32 bytes of the 128-byte swizzle row): h.h' + h.l' + l.h'
          const uint64_t dah = umma_desc_sw128(base + 0 * H_TILE + kk * 32);
          const uint64_t dal = umma_desc_sw128(base + 1 * H_TILE + kk * 32);
          const uint64_t dbh = umma_desc_sw128(base + 2 * H_TILE + kk * 32);
          const uint64_t dbl = umma_desc_sw128(base + 3 * H_TILE + kk * 32);
          umma2_bf16(acc, dah, dbh, idesc, !(first && kk == 0));
          umma2_bf16(acc, dah, dbl, idesc, 1);
          umma2_bf16(acc, dal, dbh, idesc, 1);
        }
        umma2_commit_mc(&empty[s]);
        if ((kt % H_CHUNK) == H_CHUNK - 1 || kt == ktiles - 1) umma2_commit_mc(&acc_full[q]);
      }
    }
  } else {
    constexpr int DC = 128;
    const int quarter = warp & 3;
    const int half = (warp - 2) / 4;
    const uint32_t ae0 = cluster_addr(&acc_empty[0], 0);
    float sum[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) sum[c] = 0.f;
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      const int q = chunk & 1;
      mbar_wait(&acc_full[q], (chunk >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int c = 0; c < DC; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(q * 256 + half * DC + c), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[c + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(
                         ae0 + (uint32_t)(q * sizeof(uint64_t)))
                     : "memory");
    }
    const float unscale = pow2f(2 * gshift[b]);  // undo 2^-G on both operands (exact)
    const int64_t row = (int64_t)tile_m * 256 + 128 * rank + quarter * 32 + lane;
    if (row < m) {
      float* orow = out + b * strideO + row * ldo;
      const int64_t col0 = (int64_t)tile_n * 256 + half * DC;
      const bool vec = (col0 + DC <= nc) && (ldo % 4) == 0 && ((reinterpret_cast<uintptr_t>(orow + col0) & 15) == 0);
      if (vec) {
        float4* o4 = reinterpret_cast<float4*>(orow + col0);
#pragma unroll
        for (int j = 0; j < DC / 4; ++j)
          o4[j] = make_float4(sum[4 * j] * unscale, sum[4 * j + 1] * unscale, sum[4 * j + 2] * unscale,
                              sum[4 * j + 3] * unscale);
      } else {
#pragma unroll
        for (int j = 0; j < DC; ++j)
          if (col0 + j < nc) orow[col0 + j] = sum[j] * unscale;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

// balanced exponents and the problem's shift for the F16 split (balance.cuh)
__global__ void __launch_bounds__(256) f16_balance_kernel(const double* __restrict__ colsq,
                                                          const double* __restrict__ rowsq, int64_t n_stride,
                                                          const int64_t* __restrict__ column,
                                                          const double* __restrict__ scale, int64_t w,
                                                          int64_t w_stride, const int64_t* __restrict__ kdev,
                                                          int32_t* __restrict__ kexp, int32_t* __restrict__ gshift) {
  const int64_t b = blockIdx.x;
  const int64_t kd = kdev != nullptr ? min(kdev[b], w) : w;
  f16_balance_body(colsq + b * n_stride, rowsq + b * n_stride, column + b * w_stride, scale + b * w_stride, w, kd,
                   kexp + b * w_stride, gshift + b);
}

// ---- split gather (K4 for the float32 path)

// position of element t inside its row of bf16 pairs: group t/8 holds 16 bf16
__device__ __forceinline__ int64_t pair_pos(int64_t t) { return 2 * (t & ~int64_t(7)) + (t & 7); }

__device__ __forceinline__ void split_tf32(double x, float& hi, float& lo) {
  const float xf = (float)x;
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(xf));
  hi = __uint_as_float(h);
  lo = (float)(x - (double)hi);
}

template <typename T>
__device__ __forceinline__ double ld_d(const T* p) { return (double)__ldg(p); }

// x = hi + lo, hi = x rounded to tf32 (nearest, ties away: cvt.rna.tf32), lo exact;
// float32 arithmetic only (the float32 inputs' sketch values are scaled in float32)
__device__ __forceinline__ void split_rna(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
  lo = x - hi;
}

// a_hi / a_x for rows of C = M[:, column] * scale.  A CTA owns 256 sketch
// columns of one problem and walks A_ROWS rows: the column index and scale
// are loaded once per thread, and every row's stores are coalesced.
constexpr int A_ROWS = 32;

// F16 (round 2, the CTA-pair contraction): x = h + l with h = fp16_rn(y),
// l = fp16_rn(y - h), y = x * 2^(kexp[t] - gshift) -- the sketch column scaled by the
// norm-balanced exponent (C column up, D row down by the same power of two) and the
// problem's shift that keeps |y| < 2^15 (bmm_balance_f16); both exact.  Two fp16
// halves carry 22 bits (the tf32 + bf16 form: 21) and one kind::f16 MMA of K = 16
// does the work of two kind::tf32 MMAs of K = 8 for the leading products.
__device__ __forceinline__ void split_f16(float y, float& hi, float& lo) {
  const __half h = __float2half_rn(y);
  hi = __half2float(h);
  lo = __half2float(__float2half_rn(y - hi));
}

template <typename T, bool F16 = false>
__global__ void __launch_bounds__(256) gather_a_split_kernel(const T* __restrict__ M, int64_t ldm, int64_t strideM,
                                                             int64_t m, const int64_t* __restrict__ column,
                                                             const double* __restrict__ scale, int64_t W,
                                                             int64_t w_stride, float* __restrict__ ahi,
                                                             __nv_bfloat16* __restrict__ ax,
                                                             const int64_t* __restrict__ wdev,
                                                             const int32_t* __restrict__ kexp = nullptr,
                                                             const int32_t* __restrict__ gshift = nullptr) {
  constexpr int KPAD = F16 ? 64 : 32;  // the contraction's K step
  const int64_t b = blockIdx.z;
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t h0 = (int64_t)blockIdx.y * A_ROWS;
  if (t >= W) return;
  if (wdev != nullptr && t >= ((wdev[b] + KPAD - 1) / KPAD) * KPAD) return;  // past the GEMM's K
  const int64_t col = column[b * w_stride + t];
  const double sc = scale[b * w_stride + t];
  const T* src = M + b * strideM + col;
  const int64_t h1 = min(m, h0 + A_ROWS);
  const float scf = (float)sc;
  if constexpr (F16) {
    const float f2 = pow2f(kexp[b * w_stride + t] - gshift[b]);
    __half* oh = reinterpret_cast<__half*>(ahi) + (b * m) * W + t;
    __half* ol = reinterpret_cast<__half*>(ax) + (b * m) * W + t;  // the low halves, same layout
#pragma unroll 8
    for (int64_t h = h0; h < h1; ++h) {
      float x;
      if constexpr (sizeof(T) == 4) x = __fmul_rn(__ldg(src + h * ldm), scf);
      else x = (float)__dmul_rn(ld_d(src + h * ldm), sc);
      float hi, lo;
      split_f16(__fmul_rn(x, f2), hi, lo);
      oh[h * W] = __float2half_rn(hi);
      ol[h * W] = __float2half_rn(lo);
    }
  } else {
    float* oh = ahi + (b * m) * W + t;
    __nv_bfloat16* ox = ax + (b * m) * 2 * W + pair_pos(t);
#pragma unroll 8
    for (int64_t h = h0; h < h1; ++h) {
      float hi, lo;
      if constexpr (sizeof(T) == 4) {
        split_rna(__fmul_rn(__ldg(src + h * ldm), scf), hi, lo);  // float32 inputs: no float64 conversions
      } else {
        split_tf32(__dmul_rn(ld_d(src + h * ldm), sc), hi, lo);
      }
      oh[h * W] = hi;
      ox[h * 2 * W] = __float2bfloat16_rn(hi);      // [h_x | l_x]
      ox[h * 2 * W + 8] = __float2bfloat16_rn(lo);
    }
  }
}

// b_hi / b_x for rows of D^T (D = N[column, :] * scale[:, None]): a CTA stages
// a 32 (t) x 128 (f) tile through shared memory -- 512-byte coalesced row
// reads of N, coalesced writes of the transposed operand.
template <typename T, bool F16 = false>
__global__ void __launch_bounds__(256) gather_bt_split_kernel(const T* __restrict__ N, int64_t ldn, int64_t strideN,
                                                              int64_t p, const int64_t* __restrict__ column,
                                                              const double* __restrict__ scale, int64_t W,
                                                              int64_t w_stride, float* __restrict__ bhi,
                                                              __nv_bfloat16* __restrict__ bx,
                                                              const int64_t* __restrict__ wdev,
                                                              const int32_t* __restrict__ kexp = nullptr,
                                                              const int32_t* __restrict__ gshift = nullptr) {
  constexpr int KPAD = F16 ? 64 : 32;
  __shared__ float sh[32][129], sl[32][129];
  __shared__ int64_t scol[32];
  __shared__ double sscale[32];
  __shared__ float sf2[32];
  const int64_t b = blockIdx.z;
  const int64_t t0 = (int64_t)blockIdx.x * 32, f0 = (int64_t)blockIdx.y * 128;
  if (wdev != nullptr && t0 >= ((wdev[b] + KPAD - 1) / KPAD) * KPAD) return;  // whole CTA past the compressed K
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int64_t t = t0 + tid;
    scol[tid] = t < W ? column[b * w_stride + t] : 0;
    sscale[tid] = t < W ? scale[b * w_stride + t] : 0.0;
    if constexpr (F16) sf2[tid] = t < W ? pow2f(-kexp[b * w_stride + t] - gshift[b]) : 0.f;
  }
  __syncthreads();
  // reads: 32 lanes x 4 consecutive f per row (16-byte loads when the rows allow),
  // 8 rows per pass, all 4 passes' loads issued before any is used
  const int fq = (tid & 31) * 4, ty = tid >> 5;  // 32 x 8
  const bool vec = (sizeof(T) == 4) && (ldn % 4 == 0) && (strideN % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(N) & 15) == 0) && (f0 + 128 <= p);
  using VT = typename std::conditional<sizeof(T) == 4, float, double>::type;
  VT v[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = ty + 8 * r;
    const int64_t t = t0 + i;
    const T* src = N + b * strideN + scol[i] * ldn + f0 + fq;
    if (t < W && vec) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(src));
      v[r][0] = q.x; v[r][1] = q.y; v[r][2] = q.z; v[r][3] = q.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[r][e] = (t < W && f0 + fq + e < p) ? (VT)__ldg(src + e) : (VT)0;
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = ty + 8 * r;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float hi = 0.f, lo = 0.f;
      if (t0 + i < W && f0 + fq + e < p) {
        if constexpr (F16) {
          const float x = sizeof(T) == 4 ? __fmul_rn((float)v[r][e], (float)sscale[i])
                                         : (float)__dmul_rn((double)v[r][e], sscale[i]);
          split_f16(__fmul_rn(x, sf2[i]), hi, lo);
        } else if constexpr (sizeof(T) == 4) {
          split_rna(__fmul_rn((float)v[r][e], (float)sscale[i]), hi, lo);
        } else {
          split_tf32(__dmul_rn(v[r][e], sscale[i]), hi, lo);
        }
      }
      sh[i][fq + e] = hi;
      sl[i][fq + e] = lo;
    }
  }
  __syncthreads();
  // writes: per f row a warp stores 32 hi floats (128 B) and the 64 bf16 of the
  // pair groups [l_y(8) | h_y(8)] x 4 as 32 packed bf16x2 words (128 B)
  const int tx = tid & 31, fy = tid >> 5;  // 32 x 8
  const int64_t t = t0 + tx;
  const int q = (2 * tx) & 15, tl = 8 * (tx >> 3) + (q & 7);  // this lane's bf16 pair
  const bool is_h = q >= 8;
#pragma unroll 4
  for (int i = fy; i < 128; i += 8) {
    const int64_t f = f0 + i;
    if (f < p) {
      const int64_t row = b * p + f;
      if constexpr (F16) {
        if (t < W) {
          reinterpret_cast<__half*>(bhi)[row * W + t] = __float2half_rn(sh[tx][i]);
          reinterpret_cast<__half*>(bx)[row * W + t] = __float2half_rn(sl[tx][i]);  // the low halves
        }
        continue;
      } else {
        if (t < W) bhi[row * W + t] = sh[tx][i];
      }
      if (t0 + tl < W) {
        const float a = is_h ? sh[tl][i] : sl[tl][i];
        const float c = is_h ? sh[tl + 1][i] : sl[tl + 1][i];
        if constexpr (F16)
          *reinterpret_cast<__half2*>(reinterpret_cast<__half*>(bx) + row * 2 * W + 2 * t0 + 2 * tx) =
              __halves2half2(__float2half_rn(a), __float2half_rn(c));
        else
          *reinterpret_cast<__nv_bfloat162*>(bx + row * 2 * W + 2 * t0 + 2 * tx) =
              __halves2bfloat162(__float2bfloat16_rn(a), __float2bfloat16_rn(c));
      }
    }
  }
}

// ---- fused split gather + contraction (float32 inputs, compressed sketches)
//
// The split operands of the two kernels above cost a write and a read of
// 8 bytes per sketch element and problem (config 5: ~23 GB per step, more than
// the gather's own reads of M).  Here the producer warps gather the sketch
// straight into the swizzled shared-memory stages the MMA reads, so the split
// operands never reach HBM:
//   warp 0       tcgen05.mma issuer (as gemm_f32split_kernel<128>)
//   warps 1-4    A = C tile: lane = sketch column t (the compressed columns are
//                in ascending order, so a warp's 32 loads of one row of M share
//                sectors), 32 rows per warp; hi and the [h|l] bf16 pair words
//                are 4-byte shared stores, conflict-free under the swizzle
//   warps 5-8    B = D^T tile: lane = output column f (each load of a row of N
//                is one coalesced 128-byte line), 8 t per 16-byte chunk
//   warps 9-12   drain: one warp per TMEM lane quarter (128 running sums each)
// Scaling and the split run in float32 (x = M * float(s); hi = rna_tf32(x),
// lo = x - hi exactly): no float64 conversions on the producer path.  Output
// tiles are 128 x 128, so A is gathered once per column tile and B once per row
// tile (the sibling CTAs of a problem are adjacent in launch order: their
// second reads hit L2).
// Measured (tools/fused_probe.py, sketches of 680 sorted distinct columns of
// 4096): single-tile outputs (128 x 128, 2048 problems) 1.34 ms vs 1.76 ms for
// the two kernels; 256 x 256 outputs (512 problems) 1.27 vs 0.90 ms -- the
// producers, one CTA per SM, process every element twice there.  A 2 x 2
// cluster variant that gathered each element once and stored it into the
// sibling CTAs through distributed shared memory was slower still (1.47 ms):
// its cluster-scope proxy fences and release/acquire barriers compile to
// MEMBAR.ALL.GPU / CCTL.IVALL per stage.  So plan.f32_fused picks this kernel
// for single-tile outputs only.
constexpr int FG_PA = 4, FG_PB = 4, FG_DRAIN = 4;
constexpr int FG_WARPS = 1 + FG_PA + FG_PB + FG_DRAIN;
constexpr int FG_STAGES = 2;                // MMA operand ring
constexpr int FG_STAGE = 4 * T_TILE_BYTES;  // A_hi, A_x, B_hi, B_x (128 rows x 128 B each)
constexpr int FG_SDEPTH = 3;                // cp.async staging ring: 32 floats per producer thread
constexpr int FG_STAGING = FG_SDEPTH * 32 * 256 * 4;
constexpr int FG_SMEM = FG_STAGES * FG_STAGE + FG_STAGING + 1024 + 256;
constexpr int FG_PRODUCERS = 32 * (FG_PA + FG_PB);

// byte offset of (row r, byte c of its 128-byte K row) in a SWIZZLE_128B tile
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((c >> 4) ^ (r & 7)) << 4) | (c & 15)));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo_addr, float hi_addr) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo_addr, hi_addr);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// 4-byte cp.async (zero-filled when !ok; src must still be a valid address)
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}

__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32s(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts128s(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

__device__ __forceinline__ void sts32(uint8_t* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }
__device__ __forceinline__ void sts128(uint8_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  *reinterpret_cast<uint4*>(p) = make_uint4(a, b, c, d);
}

__global__ void __launch_bounds__(32 * FG_WARPS, 1) gemm_f32split_gather_kernel(
    const float* __restrict__ M, int64_t ldm, int64_t strideM, const float* __restrict__ N, int64_t ldn,
    int64_t strideN, int64_t m, int64_t nc, const int64_t* __restrict__ column, const double* __restrict__ scale,
    int64_t W, int64_t w_stride, const int64_t* __restrict__ count, float* __restrict__ out, int64_t ldo,
    int64_t strideO) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FG_STAGES * FG_STAGE + FG_STAGING);
  uint64_t* empty = full + FG_STAGES;
  uint64_t* acc_full = empty + FG_STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.z;
  const int tile_n = blockIdx.x, tile_m = blockIdx.y;
  int64_t cnt = W;
  if (count != nullptr) cnt = count[b] < W ? count[b] : W;
  const int ktiles = (int)((cnt + T_BK - 1) / T_BK);
  const int nchunks = (ktiles + T_CHUNK - 1) / T_CHUNK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < FG_STAGES; ++s) {
      mbar_init(&full[s], FG_PRODUCERS);  // every producer thread arrives after its stores
      mbar_init(&empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&acc_full[q], 1);
      mbar_init(&acc_empty[q], FG_DRAIN);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(2 * 128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- MMA issuer (gemm_f32split_kernel<128>)
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % FG_STAGES;
        const int chunk = kt / T_CHUNK, q = chunk & 1;
        const bool first = (kt % T_CHUNK) == 0;
        if (first && chunk >= 2) mbar_wait(&acc_empty[q], ((chunk >> 1) - 1) & 1);
        mbar_wait(&full[s], (kt / FG_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t base = su32(smem + s * FG_STAGE);
        const uint32_t acc = tmem + (uint32_t)(q * 128);
#pragma unroll
        for (int kk = 0; kk < T_BK / 8; ++kk) {
          const uint32_t off = kk * 32;
          const uint64_t ahi = umma_desc_sw128(base + 0 * T_TILE_BYTES + off);
          const uint64_t ax = umma_desc_sw128(base + 1 * T_TILE_BYTES + off);
          const uint64_t bhi = umma_desc_sw128(base + 2 * T_TILE_BYTES + off);
          const uint64_t bx = umma_desc_sw128(base + 3 * T_TILE_BYTES + off);
          umma_bf16(acc, ax, bx, idesc_bf16<128>(), !(first && kk == 0));
          umma_tf32(acc, ahi, bhi, idesc_tf32<128>(), 1);
        }
        umma_commit(&empty[s]);
        if ((kt % T_CHUNK) == T_CHUNK - 1 || kt == ktiles - 1) umma_commit(&acc_full[q]);
      }
    }
  } else if (warp <= FG_PA + FG_PB) {
    // ---- producers.  The gathers go through cp.async into a per-thread staging
    // ring (FG_SDEPTH stages of 32 values, [value][thread] so every access is
    // conflict-free): two stages of loads are in flight while a thread splits
    // and stores the third, without holding them in registers.  Sketch indices
    // are fetched one stage before their loads are issued.
    const int ptid = threadIdx.x - 32;  // 0..255
    const bool is_a = warp <= FG_PA;
    const int pw = is_a ? warp - 1 : warp - 1 - FG_PA;
    const int64_t* colp = column + b * w_stride;
    const double* scp = scale + b * w_stride;
    const int r0 = pw * 32;  // A: first tile row of this warp
    const int64_t f = (int64_t)tile_n * 128 + pw * 32 + lane;  // B: this lane's output column
    const bool fvalid = f < nc;
    const int64_t rleft = m - ((int64_t)tile_m * 128 + r0);
    const int rows = rleft < 32 ? (int)rleft : 32;  // A rows of this warp inside M (may be <= 0)
    const float* Mb = M + b * strideM + ((int64_t)tile_m * 128 + (rows > 0 ? r0 : 0)) * ldm;
    const float* Nb = N + b * strideN + (fvalid ? f : 0);
    const uint32_t stg = su32(smem + FG_STAGES * FG_STAGE) + 4u * ptid;  // + (buf*32 + j) * 1024
    // A: lane t's column of M; B: lane t's row offset into N (shuffled to the f lanes); -1 = none
    auto index = [&](int kt, int64_t& ci, float& si) {
      const int64_t t = (int64_t)kt * T_BK + lane;
      const bool tv = kt < ktiles && t < cnt;
      const int64_t c = tv ? __ldg(colp + t) : (int64_t)-1;
      ci = (is_a || c < 0) ? c : c * ldn;
      si = tv ? (float)__ldg(scp + t) : 0.f;
    };
    auto issue = [&](int kt, int64_t ci) {
      const uint32_t dst = stg + (uint32_t)((kt % FG_SDEPTH) * 32) * 1024u;
      if (is_a) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const bool ok = ci >= 0 && j < rows;
          cp_async4(dst + j * 1024u, ok ? (const void*)(Mb + ci + (int64_t)j * ldm) : (const void*)M, ok);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int64_t o = __shfl_sync(0xffffffffu, ci, j);
          const bool ok = fvalid && o >= 0;
          cp_async4(dst + j * 1024u, ok ? (const void*)(Nb + o) : (const void*)N, ok);
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int64_t c0, c1, c2;
    float s0, s1, s2;
    index(0, c0, s0);
    index(1, c1, s1);
    issue(0, c0);
    issue(1, c1);
    index(2, c2, s2);
    const int g = lane >> 3, e = lane & 7;
    const int xb = (lane & 1) ? g * 32 + 16 + (e - 1) * 2 : g * 32 + e * 2;  // A: this lane's pair word
    const int fr = pw * 32 + lane;                                           // B: this lane's tile row
    const uint32_t svs = stg;  // staging: + (buf * 32 + j) * 1024
    const uint32_t sbase = su32(smem);
    uint32_t offh[8], offx[8], offb[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      offh[q] = (uint32_t)((((lane >> 2) ^ q) << 4) | ((lane & 3) << 2));          // A hi: byte 4t of row (q)
      offx[q] = (uint32_t)((((xb >> 4) ^ q) << 4) | (xb & 15));                   // A pair word of row (q)
      offb[q] = sw128(fr, 16 * q);                                                  // B row fr: chunk q
    }
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % FG_STAGES;
      issue(kt + 2, c2);  // staging buffer (kt+2) % 3 held stage kt-1: already consumed
      int64_t c3;
      float s3;
      index(kt + 3, c3, s3);
      asm volatile("cp.async.wait_group 2;\n" ::: "memory");  // this thread's stage-kt values landed
      const uint32_t v = svs + (uint32_t)((kt % FG_SDEPTH) * 32) * 1024u;  // this thread's staged values
      if (kt >= FG_STAGES) mbar_wait(&empty[s], ((kt / FG_STAGES) - 1) & 1);
      const uint32_t st = sbase + (uint32_t)(s * FG_STAGE);
      if (is_a) {
        // tile rows r0 + j: (r >> 3) * 1024 + (r & 7) * 128 are immediates, the swizzled
        // 16-byte chunk depends on j & 7 only (precomputed per lane)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float hi, lo;
          split_rna(lds_f32(v + j * 1024u) * s0, hi, lo);
          const uint32_t row = st + (uint32_t)(r0 * 128 + (j >> 3) * 1024 + (j & 7) * 128);
          sts32s(row + offh[j & 7], __float_as_uint(hi));
          // pair words: even lanes (h_t, h_t+1), odd lanes (l_t-1, l_t)
          const float recv = __shfl_xor_sync(0xffffffffu, (lane & 1) ? hi : lo, 1);
          sts32s(row + T_TILE_BYTES + offx[j & 7], (lane & 1) ? pack_bf16(recv, lo) : pack_bf16(hi, recv));
        }
      } else {
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
          float h[8], l[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            split_rna(lds_f32(v + (8 * gg + j) * 1024u) * __shfl_sync(0xffffffffu, s0, 8 * gg + j), h[j], l[j]);
          const uint32_t bh = st + 2 * T_TILE_BYTES, bx = st + 3 * T_TILE_BYTES;
          sts128s(bh + offb[2 * gg], __float_as_uint(h[0]), __float_as_uint(h[1]), __float_as_uint(h[2]),
                  __float_as_uint(h[3]));
          sts128s(bh + offb[2 * gg + 1], __float_as_uint(h[4]), __float_as_uint(h[5]), __float_as_uint(h[6]),
                  __float_as_uint(h[7]));
          // B pairs: [l(8) | h(8)]
          sts128s(bx + offb[2 * gg], pack_bf16(l[0], l[1]), pack_bf16(l[2], l[3]), pack_bf16(l[4], l[5]),
                  pack_bf16(l[6], l[7]));
          sts128s(bx + offb[2 * gg + 1], pack_bf16(h[0], h[1]), pack_bf16(h[2], h[3]), pack_bf16(h[4], h[5]),
                  pack_bf16(h[6], h[7]));
        }
      }
      // generic-proxy stores -> visible to the tensor core's async proxy, then arrive
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive(&full[s]);
      c2 = c3;
      s0 = s1;
      s1 = s2;
      s2 = s3;
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  } else {
    // ---- drain: warp w reads TMEM lanes 32*(w%4), all 128 columns
    const int quarter = warp & 3;
    float sum[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) sum[c] = 0.f;
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      const int q = chunk & 1;
      mbar_wait(&acc_full[q], (chunk >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int c = 0; c < 128; c += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(q * 128 + c), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) sum[c + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[q]);
    }
    const int64_t row = (int64_t)tile_m * 128 + quarter * 32 + lane;
    if (row < m) {
      float* orow = out + b * strideO + row * ldo;
      const int64_t col0 = (int64_t)tile_n * 128;
      const bool vec = (col0 + 128 <= nc) && ((reinterpret_cast<uintptr_t>(orow + col0) & 15) == 0);
      if (vec) {
        float4* o4 = reinterpret_cast<float4*>(orow + col0);
#pragma unroll
        for (int j = 0; j < 32; ++j) o4[j] = make_float4(sum[4 * j], sum[4 * j + 1], sum[4 * j + 2], sum[4 * j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 128; ++j)
          if (col0 + j < nc) orow[col0 + j] = sum[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * 128));
  }
}

// ---- fused fp16-split gather + contraction, one CTA per 256 x 256 output tile
// (round 2, config 5: 4096 problems of 256 x 4096 x 256)
//
// The two-kernel form writes the split operands (6 bytes per sketch element)
// and reads them back: at config 5 that is ~18 GB of the step's ~75 GB of HBM
// traffic.  Here the sketch is gathered straight into the shared-memory stages
// the tensor core reads, and one CTA owns a whole 256 x 256 output, so every
// element of C and D is gathered exactly once (the round-1 fused kernel used
// 128 x 128 tiles: four CTAs per config-5 problem, each element gathered twice).
//
// All global reads are TMA, so the bytes in flight are bounded by shared memory,
// not registers (per-thread loads of the drawn columns of M, one stage ahead in
// registers, made a first version long-scoreboard bound at 7.7 ms; 3.5 ms now):
//   * C: M is streamed in SWIZZLE_64B slabs of 256 rows x 16 columns, only the
//     slabs that hold a drawn column (680 distinct of 4096 at config 5 touch
//     ~95% of them -- what per-element gathers fetch from DRAM anyway), 5 deep;
//   * D: each drawn row of N (256 output columns, 1 KB) is one TMA box, 3
//     stages of 16 rows deep.
//   warp 0       tcgen05.mma issuer: per stage (16 K) and row half, h.h, h.l and
//                l.h (three kind::f16 MMAs, M=128, N=256) into that half's TMEM
//                accumulator (2 x 256 columns: the whole TMEM)
//   warps 1-8    C converters: thread = tile row; each drawn column is picked
//                out of its slab, scaled by scale * 2^(kexp - G), split into
//                fp16 h + l, stored as the row's [h(16) | l(16)] SWIZZLE_64B
//                operand line; then the drain (TMEM -> 2^(2G) -> global)
//   warps 9-16   D^T converters: thread = output column; the stage's 16 rows of
//                N are read across (conflict-free), scaled, split, stored as the
//                column's operand line (the transpose happens here)
//   warp 17      TMA issuer for the slabs of M (a ballot over 32 sketch columns
//                finds where a new slab starts)
//   warp 18      TMA issuer for the drawn rows of N
// Accumulation is not promoted (the TMEM holds no second accumulator pair):
// the tensor core's truncating float32 accumulate adds ~4.5e-9 relative error
// per K element in this form, so plan.f16_fused selects the kernel for sketch
// widths W <= 1024 only (<= 5e-6; config 5 measures 2.4e-6, the bar is 1e-5).
constexpr int GF_BK = 16;                            // sketch columns per operand stage
constexpr int GF_TILE = 256 * 64;                    // 16 KB: 256 operand rows x 64 B ([h(16) | l(16)] fp16)
constexpr int GF_STAGE = 2 * GF_TILE;                // A, B
constexpr int GF_STAGES = 3;
constexpr int GF_SLAB_COLS = 16;
constexpr int GF_SLAB = 256 * GF_SLAB_COLS * 4;      // 16 KB: 256 rows x 64 B of M (SWIZZLE_64B)
constexpr int GF_SLABS = 5;
constexpr int GF_BROW = 256 * 4;                     // one row of N: 256 output columns, float32
constexpr int GF_BRAW = GF_BK * GF_BROW;             // 16 KB: a stage's 16 rows of N
constexpr int GF_BRAWS = 3;
constexpr int GF_WARPS = 19;
constexpr int GF_SMEM = GF_STAGES * GF_STAGE + GF_SLABS * GF_SLAB + GF_BRAWS * GF_BRAW + 1024 + 256;

// UMMA shared-memory descriptor: K-major, SWIZZLE_64B (64-byte rows, 8-row groups 512 B apart)
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;           // leading byte offset (unused: K fits one swizzle row)
  d |= (uint64_t)(512 >> 4) << 32;  // stride byte offset: 8 rows x 64 B
  d |= (uint64_t)1 << 46;           // Blackwell descriptor version
  d |= (uint64_t)4 << 61;           // SWIZZLE_64B
  return d;
}

// byte offset of 16-byte chunk q (0..3) of row r in a SWIZZLE_64B tile of 64-byte rows
__device__ __forceinline__ uint32_t sw64(int r, int q) {
  return (uint32_t)(r * 64 + ((q ^ ((r >> 1) & 3)) << 4));
}

__device__ __forceinline__ void split_pair(float y0, float y1, uint32_t& hw, uint32_t& lw) {
  const __half2 h = __floats2half2_rn(y0, y1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(y0 - hf.x, y1 - hf.y);
  hw = *reinterpret_cast<const uint32_t*>(&h);
  lw = *reinterpret_cast<const uint32_t*>(&l);
}

__device__ __forceinline__ void tma_load_3d_gf(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
      ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__global__ void __launch_bounds__(32 * GF_WARPS, 1) gemm_f16split_gather_kernel(
    const __grid_constant__ CUtensorMap tm_M, const __grid_constant__ CUtensorMap tm_N, int64_t m, int64_t nc,
    const int64_t* __restrict__ column, const double* __restrict__ scale, const int32_t* __restrict__ kexp,
    const int32_t* __restrict__ gshift, int64_t W, int64_t w_stride, const int64_t* __restrict__ count,
    float* __restrict__ out, int64_t ldo, int64_t strideO) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* slabs = smem + GF_STAGES * GF_STAGE;
  uint8_t* braw = slabs + GF_SLABS * GF_SLAB;
  uint64_t* full = reinterpret_cast<uint64_t*>(braw + GF_BRAWS * GF_BRAW);
  uint64_t* empty = full + GF_STAGES;
  uint64_t* slab_full = empty + GF_STAGES;
  uint64_t* slab_empty = slab_full + GF_SLABS;
  uint64_t* braw_full = slab_empty + GF_SLABS;
  uint64_t* braw_empty = braw_full + GF_BRAWS;
  uint64_t* acc_full = braw_empty + GF_BRAWS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.z;
  const int64_t row0 = (int64_t)blockIdx.y * 256, col0 = (int64_t)blockIdx.x * 256;
  int64_t cnt = W;
  if (count != nullptr) cnt = count[b] < W ? count[b] : W;
  const int ktiles = (int)((cnt + GF_BK - 1) / GF_BK);
  const int G = gshift[b];
  const int64_t* colp = column + b * w_stride;
  const double* scp = scale + b * w_stride;
  const int32_t* kxp = kexp + b * w_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < GF_STAGES; ++s) {
      mbar_init(&full[s], 16);  // one arrive per converter warp (8 C + 8 D^T), after its stores
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < GF_SLABS; ++s) {
      mbar_init(&slab_full[s], 1);
      mbar_init(&slab_empty[s], 8);
    }
    for (int s = 0; s < GF_BRAWS; ++s) {
      mbar_init(&braw_full[s], 1);
      mbar_init(&braw_empty[s], 8);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_M)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_N)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- MMA issuer: per stage (16 K) and row half: h.h, h.l, l.h
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_mn<128, 256>();
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % GF_STAGES;
        mbar_wait(&full[s], (kt / GF_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t a = su32(smem + s * GF_STAGE), bb = a + GF_TILE;
        const uint64_t bh = umma_desc_sw64(bb), bl = umma_desc_sw64(bb + 32);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t ah = a + h * (GF_TILE / 2);
          const uint32_t acc = tmem + (uint32_t)(h * 256);
          umma_bf16(acc, umma_desc_sw64(ah), bh, idesc, kt > 0);
          umma_bf16(acc, umma_desc_sw64(ah), bl, idesc, 1);
          umma_bf16(acc, umma_desc_sw64(ah + 32), bh, idesc, 1);
        }
        umma_commit(&empty[s]);
      }
      if (ktiles > 0) umma_commit(acc_full);
    }
  } else if (warp == 17) {
    // ---- TMA issuer for C: the slabs of M (16 columns x 256 rows) holding a drawn
    // column, in order; 32 sketch columns scanned at a time (ballot of slab changes)
    int64_t prev = -1;
    int j = 0;
    for (int64_t g = 0; g < cnt; g += 32) {
      const int64_t t = g + lane;
      const int64_t slab = t < cnt ? (__ldg(colp + t) >> 4) : (int64_t)-1;
      int64_t before = __shfl_up_sync(0xffffffffu, slab, 1);
      if (lane == 0) before = prev;
      uint32_t fresh = __ballot_sync(0xffffffffu, t < cnt && slab != before);
      prev = __shfl_sync(0xffffffffu, slab, 31);
      while (fresh) {
        const int src = __ffs(fresh) - 1;
        fresh &= fresh - 1;
        const int64_t c = __shfl_sync(0xffffffffu, slab, src);
        if (lane == 0) {
          const int s = j % GF_SLABS;
          if (j >= GF_SLABS) mbar_wait(&slab_empty[s], ((j / GF_SLABS) - 1) & 1);
          mbar_expect_tx(&slab_full[s], GF_SLAB);
          tma_load_3d_gf(slabs + s * GF_SLAB, &tm_M, &slab_full[s], (int)(c * GF_SLAB_COLS), (int)row0, (int)b);
        }
        ++j;
      }
    }
  } else if (warp == 18) {
    // ---- TMA issuer for D: each stage's 16 drawn rows of N (256 output columns each)
    if (lane == 0) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % GF_BRAWS;
        if (kt >= GF_BRAWS) mbar_wait(&braw_empty[s], ((kt / GF_BRAWS) - 1) & 1);
        const int nval = (int)min((int64_t)GF_BK, cnt - (int64_t)kt * GF_BK);
        mbar_expect_tx(&braw_full[s], nval * GF_BROW);
        for (int i = 0; i < nval; ++i)
          tma_load_3d_gf(braw + s * GF_BRAW + i * GF_BROW, &tm_N, &braw_full[s], (int)col0,
                         (int)__ldg(colp + (int64_t)kt * GF_BK + i), (int)b);
      }
    }
  } else if (warp <= 8) {
    // ---- C converters: thread = tile row r, one stage (16 sketch columns) per iteration,
    // unrolled.  Lane i < 16 holds sketch column 16 kt + i: its byte in an unswizzled slab
    // row and its factor scale * 2^(kexp - G) (exact: a power of two); a ballot marks where
    // a new slab starts.  Pairs of columns are split with one packed conversion each way;
    // a stage's row goes out as four 16-byte stores ([h(8)] [h(8)] [l(8)] [l(8)]).
    const int r = (warp - 1) * 32 + lane;
    const uint32_t sbase = su32(smem);
    const uint32_t rslab = su32(slabs) + (uint32_t)(r * 64);
    const uint32_t rsw16 = (uint32_t)(((r >> 1) & 3) << 4);  // SWIZZLE_64B: chunk ^= (r >> 1) & 3
    int j = -1;
    uint32_t sl = 0;
    int64_t carry = -1;  // the slab of the previous stage's last column
    auto meta = [&](int kt, int64_t& c_, float& f_) {  // lane's sketch column of stage kt (lanes < 16)
      const int64_t t = (int64_t)kt * GF_BK + lane;
      const bool ok = lane < GF_BK && t < cnt;
      c_ = ok ? __ldg(colp + t) : (int64_t)-1;
      f_ = ok ? __fmul_rn((float)__ldg(scp + t), pow2f(__ldg(kxp + t) - G)) : 0.f;
    };
    int64_t ncol;
    float nfac;
    meta(0, ncol, nfac);
    for (int kt = 0; kt < ktiles; ++kt) {
      const int64_t t = (int64_t)kt * GF_BK + lane;
      const bool ok = lane < GF_BK && t < cnt;
      const int64_t col = ncol;
      const float fac = nfac;
      meta(kt + 1, ncol, nfac);  // one stage ahead
      const int64_t slab = col >> 4;
      int64_t before = __shfl_up_sync(0xffffffffu, slab, 1);
      if (lane == 0) before = carry;
      const uint32_t fresh = __ballot_sync(0xffffffffu, ok && slab != before);
      const int nval = (int)min((int64_t)GF_BK, cnt - (int64_t)kt * GF_BK);
      carry = __shfl_sync(0xffffffffu, slab, nval - 1);
      const uint32_t q4 = (uint32_t)(col & 15) * 4;
      if (kt >= GF_STAGES) mbar_wait(&empty[kt % GF_STAGES], ((kt / GF_STAGES) - 1) & 1);
      const uint32_t st = sbase + (uint32_t)((kt % GF_STAGES) * GF_STAGE);
      uint32_t hw[8], lw[8];
#pragma unroll
      for (int i = 0; i < GF_BK; i += 2) {
        float y[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int tt = i + u;
          if ((fresh >> tt) & 1u) {  // warp-uniform: the next slab
            if (j >= 0) {
              __syncwarp();
              if (lane == 0) mbar_arrive(&slab_empty[j % GF_SLABS]);
            }
            ++j;
            mbar_wait(&slab_full[j % GF_SLABS], (j / GF_SLABS) & 1);
            sl = rslab + (uint32_t)((j % GF_SLABS) * GF_SLAB);
          }
          const uint32_t o = __shfl_sync(0xffffffffu, q4, tt) ^ rsw16;
          const float f = __shfl_sync(0xffffffffu, fac, tt);
          y[u] = tt < nval ? __fmul_rn(lds_f32(sl + o), f) : 0.f;
        }
        split_pair(y[0], y[1], hw[i >> 1], lw[i >> 1]);
      }
      sts128s(st + sw64(r, 0), hw[0], hw[1], hw[2], hw[3]);
      sts128s(st + sw64(r, 1), hw[4], hw[5], hw[6], hw[7]);
      sts128s(st + sw64(r, 2), lw[0], lw[1], lw[2], lw[3]);
      sts128s(st + sw64(r, 3), lw[4], lw[5], lw[6], lw[7]);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[kt % GF_STAGES]);
    }
    if (j >= 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&slab_empty[j % GF_SLABS]);
    }
    // ---- drain: warp w reads TMEM lanes 32 (w % 4), row half (w - 1) / 4, all 256 columns
    const int quarter = warp & 3, half = (warp - 1) >> 2;
    if (ktiles > 0) {
      mbar_wait(acc_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    const float unscale = pow2f(2 * G);
    const int64_t row = row0 + half * 128 + quarter * 32 + lane;
    float* orow = out + b * strideO + (row < m ? row : 0) * ldo;
    const bool vec = (col0 + 256 <= nc) && (ldo % 4) == 0 && ((reinterpret_cast<uintptr_t>(orow + col0) & 15) == 0);
#pragma unroll 1
    for (int cc = 0; cc < 256; cc += 32) {
      uint32_t v[32];
      if (ktiles > 0) {
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(half * 256 + cc), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      } else {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) v[jj] = 0u;
      }
      if (row < m) {
        if (vec) {
          float4* o4 = reinterpret_cast<float4*>(orow + col0 + cc);
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            o4[jj] = make_float4(__uint_as_float(v[4 * jj]) * unscale, __uint_as_float(v[4 * jj + 1]) * unscale,
                                 __uint_as_float(v[4 * jj + 2]) * unscale, __uint_as_float(v[4 * jj + 3]) * unscale);
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            if (col0 + cc + jj < nc) orow[col0 + cc + jj] = __uint_as_float(v[jj]) * unscale;
        }
      }
    }
  } else {
    // ---- D^T converters (warps 9-16): thread = output column f of the tile; the stage's
    // 16 rows of N arrive by TMA (a 1 KB row each), are scaled, split and stored as the
    // thread's operand row [h(16) | l(16)]
    const int fl = (warp - 9) * 32 + lane;
    const uint32_t sbase = su32(smem);
    auto meta = [&](int kt) {  // lane's factor scale * 2^(-kexp - G) of stage kt (lanes < 16)
      const int64_t t = (int64_t)kt * GF_BK + lane;
      const bool ok = lane < GF_BK && t < cnt;
      return ok ? __fmul_rn((float)__ldg(scp + t), pow2f(-__ldg(kxp + t) - G)) : 0.f;
    };
    float nfac = meta(0);
    for (int kt = 0; kt < ktiles; ++kt) {
      const float fac = nfac;
      nfac = meta(kt + 1);  // one stage ahead
      const int nval = (int)min((int64_t)GF_BK, cnt - (int64_t)kt * GF_BK);
      const int sr = kt % GF_BRAWS;
      mbar_wait(&braw_full[sr], (kt / GF_BRAWS) & 1);
      const uint32_t raw = su32(braw + sr * GF_BRAW) + 4u * fl;
      float y[GF_BK];
#pragma unroll
      for (int i = 0; i < GF_BK; ++i)
        y[i] = i < nval ? __fmul_rn(lds_f32(raw + i * GF_BROW), __shfl_sync(0xffffffffu, fac, i)) : 0.f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&braw_empty[sr]);
      uint32_t hw[8], lw[8];
#pragma unroll
      for (int i = 0; i < GF_BK; i += 2) split_pair(y[i], y[i + 1], hw[i >> 1], lw[i >> 1]);
      if (kt >= GF_STAGES) mbar_wait(&empty[kt % GF_STAGES], ((kt / GF_STAGES) - 1) & 1);
      const uint32_t bt = sbase + (uint32_t)((kt % GF_STAGES) * GF_STAGE) + GF_TILE;
      sts128s(bt + sw64(fl, 0), hw[0], hw[1], hw[2], hw[3]);
      sts128s(bt + sw64(fl, 1), hw[4], hw[5], hw[6], hw[7]);
      sts128s(bt + sw64(fl, 2), lw[0], lw[1], lw[2], lw[3]);
      sts128s(bt + sw64(fl, 3), lw[4], lw[5], lw[6], lw[7]);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[kt % GF_STAGES]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

// ---- host side

static int make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int box_rows = T_BM) {
  auto enc = get_encode();
  BMM_REQUIRE(enc != nullptr, BMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)T_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BMM_REQUIRE(r == CUDA_SUCCESS, BMM_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BMM_OK;
}

}  // namespace bmm

using namespace bmm;

static int gather_split_impl(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N, int64_t ldn,
                             int64_t strideN, int64_t m, int64_t p, const int64_t* column, const double* scale,
                             int64_t W, int64_t w_stride, const int64_t* w_dev, int64_t batch, float* a_hi, void* a_x,
                             float* b_hi, void* b_x, cudaStream_t st) {
  BMM_REQUIRE(m >= 1 && p >= 1 && W >= 1 && batch >= 1, BMM_E_ARG, "bmm_gather_f32split: bad shape");
  BMM_REQUIRE(W % 8 == 0, BMM_E_UNSUPPORTED, "bmm_gather_f32split: W must be a multiple of 8");
  __nv_bfloat16* ax = (__nv_bfloat16*)a_x;
  __nv_bfloat16* bx = (__nv_bfloat16*)b_x;
  BMM_REQUIRE(batch <= 65535 && ceil_div(m, A_ROWS) <= 65535, BMM_E_UNSUPPORTED, "bmm_gather_f32split: grid too large");
  dim3 agrid((unsigned)ceil_div(W, 256), (unsigned)ceil_div(m, A_ROWS), (unsigned)batch);
  dim3 tgrid((unsigned)ceil_div(W, 32), (unsigned)ceil_div(p, 128), (unsigned)batch);
  if (dtype == BMM_F32) {
    gather_a_split_kernel<float><<<agrid, 256, 0, st>>>((const float*)M, ldm, strideM, m, column, scale, W, w_stride,
                                                        a_hi, ax, w_dev);
    BMM_CHECK_LAUNCH("gather_a_split_kernel");
    gather_bt_split_kernel<float><<<tgrid, 256, 0, st>>>((const float*)N, ldn, strideN, p, column, scale, W,
                                                         w_stride, b_hi, bx, w_dev);
  } else if (dtype == BMM_F64) {
    gather_a_split_kernel<double><<<agrid, 256, 0, st>>>((const double*)M, ldm, strideM, m, column, scale, W,
                                                         w_stride, a_hi, ax, w_dev);
    BMM_CHECK_LAUNCH("gather_a_split_kernel");
    gather_bt_split_kernel<double><<<tgrid, 256, 0, st>>>((const double*)N, ldn, strideN, p, column, scale, W,
                                                          w_stride, b_hi, bx, w_dev);
  } else {
    set_error("bmm_gather_f32split: unknown dtype %d", dtype);
    return BMM_E_ARG;
  }
  BMM_CHECK_LAUNCH("gather_bt_split_kernel");
  return BMM_OK;
}

extern "C" int bmm_gather_f32split(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                   int64_t ldn, int64_t strideN, int64_t m, int64_t p, const int64_t* column,
                                   const double* scale, int64_t W, int64_t w_stride, int64_t batch, float* a_hi,
                                   void* a_x, float* b_hi, void* b_x, void* stream) {
  return gather_split_impl(dtype, M, ldm, strideM, N, ldn, strideN, m, p, column, scale, W, w_stride, nullptr, batch,
                           a_hi, a_x, b_hi, b_x, as_stream(stream));
}

extern "C" int bmm_gather_f32split_dk(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                      int64_t ldn, int64_t strideN, int64_t m, int64_t p, const int64_t* column,
                                      const double* scale, int64_t W, int64_t w_stride, const int64_t* w_dev,
                                      int64_t batch, float* a_hi, void* a_x, float* b_hi, void* b_x, void* stream) {
  BMM_REQUIRE(w_dev != nullptr, BMM_E_ARG, "bmm_gather_f32split_dk: w_dev is NULL");
  return gather_split_impl(dtype, M, ldm, strideM, N, ldn, strideN, m, p, column, scale, W, w_stride, w_dev, batch,
                           a_hi, a_x, b_hi, b_x, as_stream(stream));
}

static int gemm_split_impl(const float* a_hi, const void* a_x, const float* b_hi, const void* b_x, int64_t m,
                           int64_t nc, int64_t k, const int64_t* k_dev, int64_t batch, float* out, int64_t ldo,
                           int64_t strideO, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && k >= 1 && batch >= 1, BMM_E_ARG, "bmm_gemm_f32split: bad shape");
  BMM_REQUIRE(k % 8 == 0, BMM_E_UNSUPPORTED, "bmm_gemm_f32split: k must be a multiple of 8");
  const float* a_lo = (const float*)a_x;  // bf16 pairs: the same bytes per row as k floats
  const float* b_lo = (const float*)b_x;
  BMM_REQUIRE(batch * m < (1LL << 31) && batch * nc < (1LL << 31) && batch <= 65535, BMM_E_UNSUPPORTED,
              "bmm_gemm_f32split: problem too large for 32-bit TMA coordinates");
  // 128x256 tiles when one column tile then covers the output (A streamed once per
  // problem: the batched config 5, 256 wide); large outputs keep 128x128 -- its
  // 3-stage ring measured ~8% more tensor work per clock at config 4 (64.1 ms at
  // 1.51 GHz vs 63.3 ms at 1.65 GHz for 128x256)
  static const int tile_env = [] {
    const char* e = getenv("BMM_TF32_BN");  // A/B switch for timing (128 or 256)
    return e ? atoi(e) : 0;
  }();
  const int bn = tile_env == 128 || tile_env == 256 ? tile_env : (nc > 128 && nc <= 256 ? 256 : 128);
  // CTA pairs sharing A by TMA multicast (BMM_TF32_PAIR=1): 3.6% more tensor work per
  // clock at config 4, but the power-capped clock fell further (65.2 ms at 1.46 GHz vs
  // 64.3 ms at 1.53 GHz), so single CTAs stay the default
  static const int pair_env = [] {
    const char* e = getenv("BMM_TF32_PAIR");
    return e ? atoi(e) : 0;
  }();
  const bool pair = bn == 128 && pair_env != 0 && nc > 256;
  // cta_group::2 (256 x 256 per CTA pair): large outputs (BMM_TF32_2SM=0 disables)
  static const int sm2_env = [] {
    const char* e = getenv("BMM_TF32_2SM");
    return e ? atoi(e) : 1;
  }();
  const bool two_sm = sm2_env != 0 && tile_env == 0 && pair_env == 0 && m >= 256 && nc >= 512;
  CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
  int rc;
  if ((rc = make_map(&ma_hi, a_hi, batch * m, k)) != BMM_OK) return rc;
  if ((rc = make_map(&ma_lo, a_lo, batch * m, k)) != BMM_OK) return rc;
  if ((rc = make_map(&mb_hi, b_hi, batch * nc, k, bn)) != BMM_OK) return rc;
  if ((rc = make_map(&mb_lo, b_lo, batch * nc, k, bn)) != BMM_OK) return rc;
  cudaStream_t st = as_stream(stream);
  if (two_sm) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_f32split_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM);
      attr = true;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(2 * ceil_div(nc, 256)), (unsigned)ceil_div(m, 256), (unsigned)batch);
    lc.blockDim = dim3(32 * P_WARPS, 1, 1);
    lc.dynamicSmemBytes = P_SMEM;
    lc.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = 2;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    lc.attrs = la;
    lc.numAttrs = 1;
    if (cudaLaunchKernelEx(&lc, gemm_f32split_2sm_kernel, ma_hi, ma_lo, mb_hi, mb_lo, m, nc, k, out, ldo, strideO,
                           k_dev) != cudaSuccess) {
      set_error("bmm_gemm_f32split: 2-SM cluster launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      return BMM_E_CUDA;
    }
  } else if (bn == 256) {
    using Cfg = TCfg<256>;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_f32split_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
      attr = true;
    }
    dim3 grid((unsigned)ceil_div(nc, 256), (unsigned)ceil_div(m, T_BM), (unsigned)batch);
    gemm_f32split_kernel<256><<<grid, 32 * Cfg::WARPS, Cfg::SMEM, st>>>(ma_hi, ma_lo, mb_hi, mb_lo, m, nc, k, out,
                                                                         ldo, strideO, k_dev);
  } else if (pair) {
    // CTA pairs sharing A through TMA multicast (cluster 2 x 1 x 1 along the column tiles)
    using Cfg = TCfg<128>;
    CUtensorMap pa_hi, pa_lo;
    if ((rc = make_map(&pa_hi, a_hi, batch * m, k, 64)) != BMM_OK) return rc;
    if ((rc = make_map(&pa_lo, a_lo, batch * m, k, 64)) != BMM_OK) return rc;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_f32split_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
      attr = true;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(2 * ceil_div(ceil_div(nc, 128), 2)), (unsigned)ceil_div(m, T_BM), (unsigned)batch);
    lc.blockDim = dim3(32 * Cfg::WARPS, 1, 1);
    lc.dynamicSmemBytes = Cfg::SMEM;
    lc.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = 2;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    lc.attrs = la;
    lc.numAttrs = 1;
    if (cudaLaunchKernelEx(&lc, gemm_f32split_kernel<128, 2>, pa_hi, pa_lo, mb_hi, mb_lo, m, nc, k, out, ldo,
                           strideO, k_dev) != cudaSuccess) {
      set_error("bmm_gemm_f32split: cluster launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      return BMM_E_CUDA;
    }
  } else {
    using Cfg = TCfg<128>;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_f32split_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
      attr = true;
    }
    dim3 grid((unsigned)ceil_div(nc, 128), (unsigned)ceil_div(m, T_BM), (unsigned)batch);
    gemm_f32split_kernel<128><<<grid, 32 * Cfg::WARPS, Cfg::SMEM, st>>>(ma_hi, ma_lo, mb_hi, mb_lo, m, nc, k, out,
                                                                         ldo, strideO, k_dev);
  }
  BMM_CHECK_LAUNCH("gemm_f32split_kernel");
  return BMM_OK;
}

static int make_map_f16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols) {
  auto enc = get_encode();
  BMM_REQUIRE(enc != nullptr, BMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)H_BK, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BMM_REQUIRE(r == CUDA_SUCCESS, BMM_E_CUDA, "cuTensorMapEncodeTiled (f16) failed (%d)", (int)r);
  return BMM_OK;
}

extern "C" int bmm_balance_f16(const double* colsq, const double* rowsq, int64_t n_stride, const int64_t* column,
                               const double* scale, int64_t w, int64_t w_stride, const int64_t* k_dev, int64_t batch,
                               int32_t* kexp, int32_t* gshift, void* stream) {
  BMM_REQUIRE(colsq && rowsq && column && scale && kexp && gshift && w >= 1 && batch >= 1 && w_stride >= w,
              BMM_E_ARG, "bmm_balance_f16: bad arguments");
  f16_balance_kernel<<<(unsigned)batch, 256, 0, as_stream(stream)>>>(colsq, rowsq, n_stride, column, scale, w,
                                                                      w_stride, k_dev, kexp, gshift);
  BMM_CHECK_LAUNCH("f16_balance_kernel");
  return BMM_OK;
}

extern "C" int bmm_gather_f16split_dk(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                      int64_t ldn, int64_t strideN, int64_t m, int64_t p, const int64_t* column,
                                      const double* scale, const int32_t* kexp, const int32_t* gshift, int64_t W,
                                      int64_t w_stride, const int64_t* w_dev, int64_t batch, void* a_h, void* a_x,
                                      void* b_h, void* b_x, void* stream) {
  BMM_REQUIRE(m >= 1 && p >= 1 && W >= 1 && batch >= 1, BMM_E_ARG, "bmm_gather_f16split_dk: bad shape");
  BMM_REQUIRE(W % 8 == 0, BMM_E_UNSUPPORTED, "bmm_gather_f16split_dk: W must be a multiple of 8");
  BMM_REQUIRE(kexp && gshift && column && scale, BMM_E_ARG, "bmm_gather_f16split_dk: null pointer");
  BMM_REQUIRE(batch <= 65535 && ceil_div(m, A_ROWS) <= 65535, BMM_E_UNSUPPORTED,
              "bmm_gather_f16split_dk: grid too large");
  cudaStream_t st = as_stream(stream);
  dim3 agrid((unsigned)ceil_div(W, 256), (unsigned)ceil_div(m, A_ROWS), (unsigned)batch);
  dim3 tgrid((unsigned)ceil_div(W, 32), (unsigned)ceil_div(p, 128), (unsigned)batch);
  float* ah = (float*)a_h;
  float* bh = (float*)b_h;
  __nv_bfloat16* ax = (__nv_bfloat16*)a_x;
  __nv_bfloat16* bx = (__nv_bfloat16*)b_x;
  if (dtype == BMM_F32) {
    gather_a_split_kernel<float, true><<<agrid, 256, 0, st>>>((const float*)M, ldm, strideM, m, column, scale, W,
                                                              w_stride, ah, ax, w_dev, kexp, gshift);
    BMM_CHECK_LAUNCH("gather_a_split_kernel<f16>");
    gather_bt_split_kernel<float, true><<<tgrid, 256, 0, st>>>((const float*)N, ldn, strideN, p, column, scale, W,
                                                               w_stride, bh, bx, w_dev, kexp, gshift);
  } else if (dtype == BMM_F64) {
    gather_a_split_kernel<double, true><<<agrid, 256, 0, st>>>((const double*)M, ldm, strideM, m, column, scale, W,
                                                               w_stride, ah, ax, w_dev, kexp, gshift);
    BMM_CHECK_LAUNCH("gather_a_split_kernel<f16>");
    gather_bt_split_kernel<double, true><<<tgrid, 256, 0, st>>>((const double*)N, ldn, strideN, p, column, scale,
                                                                W, w_stride, bh, bx, w_dev, kexp, gshift);
  } else {
    set_error("bmm_gather_f16split_dk: unknown dtype %d", dtype);
    return BMM_E_ARG;
  }
  BMM_CHECK_LAUNCH("gather_bt_split_kernel<f16>");
  return BMM_OK;
}

extern "C" int bmm_gemm_f16split_dk(const void* a_h, const void* a_x, const void* b_h, const void* b_x, int64_t m,
                                    int64_t nc, int64_t k_max, const int64_t* k_dev, const int32_t* gshift,
                                    int64_t batch, float* out, int64_t ldo, int64_t strideO, void* stream) {
  BMM_REQUIRE(m >= 1 && nc >= 1 && k_max >= 1 && batch >= 1 && gshift != nullptr, BMM_E_ARG,
              "bmm_gemm_f16split_dk: bad shape");
  BMM_REQUIRE(k_max % 8 == 0, BMM_E_UNSUPPORTED, "bmm_gemm_f16split_dk: k must be a multiple of 8");
  BMM_REQUIRE(batch * m < (1LL << 31) && batch * nc < (1LL << 31) && batch <= 65535, BMM_E_UNSUPPORTED,
              "bmm_gemm_f16split_dk: problem too large for 32-bit TMA coordinates");
  CUtensorMap ma_h, ma_x, mb_h, mb_x;
  int rc;
  if ((rc = make_map_f16(&ma_h, a_h, batch * m, k_max)) != BMM_OK) return rc;
  if ((rc = make_map_f16(&ma_x, a_x, batch * m, k_max)) != BMM_OK) return rc;
  if ((rc = make_map_f16(&mb_h, b_h, batch * nc, k_max)) != BMM_OK) return rc;
  if ((rc = make_map_f16(&mb_x, b_x, batch * nc, k_max)) != BMM_OK) return rc;
  // promotion chunk: 256 K (default: half the TMEM drain traffic) or 128 K (BMM_F16_CHUNK=2)
  static const int chunk = [] {
    const char* e = getenv("BMM_F16_CHUNK");
    return e ? atoi(e) : 4;  // 256 K per promotion: 35.0 vs 36.2 ms at config 4, error 1.0e-6 vs 6.1e-7
  }();
  auto kern = chunk == 4 ? gemm_f16split_2sm_kernel<4> : gemm_f16split_2sm_kernel<H_CHUNK_DEFAULT>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_f16split_2sm_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, H_SMEM);
    cudaFuncSetAttribute(gemm_f16split_2sm_kernel<H_CHUNK_DEFAULT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         H_SMEM);
    attr = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(2 * ceil_div(nc, 256)), (unsigned)ceil_div(m, 256), (unsigned)batch);
  lc.blockDim = dim3(32 * P_WARPS, 1, 1);
  lc.dynamicSmemBytes = H_SMEM;
  lc.stream = as_stream(stream);
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = 2;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  lc.attrs = la;
  lc.numAttrs = 1;
  static const int group_m = [] {
    const char* e = getenv("BMM_F16_GROUP_M");  // A/B switch: pair-tile rows per raster group
    const int v = e ? atoi(e) : 4;  // config 4 (profiles/r2bj_gemm_sweep.txt): 4 -> 36.2 ms, 8 -> 39, 16 -> 41
    return v >= 1 ? v : 4;
  }();
  if (cudaLaunchKernelEx(&lc, kern, ma_h, ma_x, mb_h, mb_x, m, nc, k_max, out, ldo, strideO, k_dev, gshift,
                         group_m) != cudaSuccess) {
    set_error("bmm_gemm_f16split_dk: cluster launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return BMM_E_CUDA;
  }
  BMM_CHECK_LAUNCH("gemm_f16split_2sm_kernel");
  return BMM_OK;
}

extern "C" int bmm_gemm_f32split(const float* a_hi, const void* a_x, const float* b_hi, const void* b_x,
                                 int64_t m, int64_t nc, int64_t k, int64_t batch, float* out, int64_t ldo,
                                 int64_t strideO, void* stream) {
  return gemm_split_impl(a_hi, a_x, b_hi, b_x, m, nc, k, nullptr, batch, out, ldo, strideO, stream);
}

extern "C" int bmm_gemm_f32split_dk(const float* a_hi, const void* a_x, const float* b_hi, const void* b_x,
                                    int64_t m, int64_t nc, int64_t k_max, const int64_t* k_dev, int64_t batch,
                                    float* out, int64_t ldo, int64_t strideO, void* stream) {
  BMM_REQUIRE(k_dev != nullptr, BMM_E_ARG, "bmm_gemm_f32split_dk: k_dev is NULL");
  return gemm_split_impl(a_hi, a_x, b_hi, b_x, m, nc, k_max, k_dev, batch, out, ldo, strideO, stream);
}

extern "C" int bmm_gemm_f32split_gather(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                        int64_t ldn, int64_t strideN, int64_t m, int64_t p, const int64_t* column,
                                        const double* scale, int64_t W, int64_t w_stride, const int64_t* w_dev,
                                        int64_t batch, float* out, int64_t ldo, int64_t strideO, void* stream) {
  BMM_REQUIRE(m >= 1 && p >= 1 && W >= 1 && batch >= 1, BMM_E_ARG, "bmm_gemm_f32split_gather: bad shape");
  BMM_REQUIRE(dtype == BMM_F32, BMM_E_UNSUPPORTED, "bmm_gemm_f32split_gather: float32 inputs only");
  BMM_REQUIRE(batch <= 65535 && ceil_div(m, 128) <= 65535, BMM_E_UNSUPPORTED,
              "bmm_gemm_f32split_gather: grid too large");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_f32split_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FG_SMEM);
    attr = true;
  }
  dim3 grid((unsigned)ceil_div(p, 128), (unsigned)ceil_div(m, 128), (unsigned)batch);
  gemm_f32split_gather_kernel<<<grid, 32 * FG_WARPS, FG_SMEM, as_stream(stream)>>>(
      (const float*)M, ldm, strideM, (const float*)N, ldn, strideN, m, p, column, scale, W, w_stride, w_dev, out, ldo,
      strideO);
  BMM_CHECK_LAUNCH("gemm_f32split_gather_kernel");
  return BMM_OK;
}

extern "C" int bmm_gemm_f16split_gather(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                                        int64_t ldn, int64_t strideN, int64_t m, int64_t n, int64_t p,
                                        const int64_t* column, const double* scale, const int32_t* kexp,
                                        const int32_t* gshift, int64_t W, int64_t w_stride, const int64_t* w_dev,
                                        int64_t batch, float* out, int64_t ldo, int64_t strideO, void* stream) {
  BMM_REQUIRE(m >= 1 && n >= 1 && p >= 1 && W >= 1 && batch >= 1, BMM_E_ARG, "bmm_gemm_f16split_gather: bad shape");
  BMM_REQUIRE(kexp != nullptr && gshift != nullptr, BMM_E_ARG, "bmm_gemm_f16split_gather: kexp / gshift is NULL");
  BMM_REQUIRE(dtype == BMM_F32, BMM_E_UNSUPPORTED, "bmm_gemm_f16split_gather: float32 inputs only");
  BMM_REQUIRE(batch <= 65535 && ceil_div(m, 256) <= 65535 && n < (1LL << 31), BMM_E_UNSUPPORTED,
              "bmm_gemm_f16split_gather: grid too large");
  BMM_REQUIRE(ldm % 4 == 0 && (batch == 1 || strideM % 4 == 0) && (reinterpret_cast<uintptr_t>(M) & 15) == 0,
              BMM_E_UNSUPPORTED, "bmm_gemm_f16split_gather: M rows must be 16-byte aligned (TMA)");
  auto enc = get_encode();
  BMM_REQUIRE(enc != nullptr, BMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  // M as [batch][m][n] float32: boxes of 16 columns x 256 rows of one problem, SWIZZLE_64B
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)m, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)ldm * 4, (cuuint64_t)(batch == 1 ? ldm * m : strideM) * 4};
  cuuint32_t box[3] = {(cuuint32_t)GF_SLAB_COLS, 256, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(M), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BMM_REQUIRE(r == CUDA_SUCCESS, BMM_E_CUDA, "bmm_gemm_f16split_gather: cuTensorMapEncodeTiled failed (%d)", (int)r);
  BMM_REQUIRE(ldn % 4 == 0 && (batch == 1 || strideN % 4 == 0) && (reinterpret_cast<uintptr_t>(N) & 15) == 0,
              BMM_E_UNSUPPORTED, "bmm_gemm_f16split_gather: N rows must be 16-byte aligned (TMA)");
  // N as [batch][n][p] float32: one drawn row (256 output columns of the tile) per box
  CUtensorMap tn;
  cuuint64_t ndims[3] = {(cuuint64_t)p, (cuuint64_t)n, (cuuint64_t)batch};
  cuuint64_t nstrides[2] = {(cuuint64_t)ldn * 4, (cuuint64_t)(batch == 1 ? ldn * n : strideN) * 4};
  cuuint32_t nbox[3] = {256, 1, 1};
  r = enc(&tn, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(N), ndims, nstrides, nbox, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BMM_REQUIRE(r == CUDA_SUCCESS, BMM_E_CUDA, "bmm_gemm_f16split_gather: cuTensorMapEncodeTiled (N) failed (%d)", (int)r);
  static const cudaError_t attr =
      cudaFuncSetAttribute(gemm_f16split_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GF_SMEM);
  BMM_REQUIRE(attr == cudaSuccess, BMM_E_CUDA, "bmm_gemm_f16split_gather: %d bytes of shared memory: %s", GF_SMEM,
              cudaGetErrorString(attr));
  dim3 grid((unsigned)ceil_div(p, 256), (unsigned)ceil_div(m, 256), (unsigned)batch);
  gemm_f16split_gather_kernel<<<grid, 32 * GF_WARPS, GF_SMEM, as_stream(stream)>>>(
      tm, tn, m, p, column, scale, kexp, gshift, W, w_stride, w_dev, out, ldo, strideO);
  {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFuncAttributes fa = {};
      cudaFuncGetAttributes(&fa, gemm_f16split_gather_kernel);
      set_error("gemm_f16split_gather_kernel: launch failed: %s (regs %d, max threads %d, static smem %zu, "
                "max dynamic %d, requested %d x %d threads)", cudaGetErrorString(e), fa.numRegs,
                fa.maxThreadsPerBlock, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, GF_SMEM, 32 * GF_WARPS);
      return BMM_E_CUDA;
    }
    count_launch();
  }
  return BMM_OK;
}
