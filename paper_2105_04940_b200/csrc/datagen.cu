// On-device synthetic instances -- the reference's
// gen_normal_instance / gen_heavy_tail_instance (pkg/src/blockmm/datagen.py:55-110).
//
// The reference draws Z ~ N(0,1) on the host and forms L @ Z with the Cholesky
// factor L of an AR(1) covariance (scale * rho^|i-j|, datagen.py:38-42).  For
// that covariance the product is the AR(1) recursion
//     x_0 = sqrt(s) z_0,   x_i = rho x_{i-1} + sqrt(s (1 - rho^2)) z_i,
// so every sample vector costs O(dim) instead of O(dim^2) and is generated
// where it is stored: M's columns (dimension m) by one thread each walking the
// rows (coalesced stores across threads), N's rows (dimension p) by one lane
// each, staged through a 32 x 32 shared tile so the warp stores whole rows.
// The heavy-tailed variant divides each vector by sqrt(w), w = z'^2 ~ chi^2(1)
// (redrawn if 0) and adds the location (datagen.py:82-110).
//
// Randomness: vector j of side `tag` has its own PCG64 stream, seeded by the
// SeedSequence hash (rng.cuh) of (entropy words, tag) with child index j;
// normals by Box-Muller on (1 - u, u') with both outputs used.  The streams are
// NOT numpy's ziggurat normals: instances are distribution-identical and
// deterministic per seed, not bit-identical to the reference's.
#include "common.cuh"
#include "rng.cuh"

namespace bmm {

struct NormalStream {
  U128 st, inc;
  double spare;
  bool has_spare;
  __device__ void init(const uint32_t* words, int64_t nw, uint64_t child) {
    seed_pcg64(words, nw, child, st, inc);
    has_spare = false;
  }
  __device__ __forceinline__ double uniform() {
    st = pcg_step(st, inc);
    return u53(pcg_output(st));
  }
  __device__ __forceinline__ double next() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = 1.0 - uniform();  // (0, 1]
    const double u2 = uniform();
    const double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    spare = r * sn;
    has_spare = true;
    return r * cs;
  }
};

__device__ __forceinline__ void put(double* p, double v) { *p = v; }
__device__ __forceinline__ void put(float* p, double v) { *p = (float)v; }

__device__ __forceinline__ void make_words(uint64_t hi, uint64_t lo, uint32_t tag, uint32_t* w) {
  w[0] = (uint32_t)lo;
  w[1] = (uint32_t)(lo >> 32);
  w[2] = (uint32_t)hi;
  w[3] = (uint32_t)(hi >> 32);
  w[4] = tag;
}

// inverse chi-square(1) square root for the heavy-tailed variant
__device__ __forceinline__ double inv_sqrt_chi2(NormalStream& g) {
  double w = 0.0;
  while (w == 0.0) {
    const double z = g.next();
    w = z * z;
  }
  return 1.0 / sqrt(w);
}

// M (m x n): column j = AR(1) vector of dimension m
template <typename T>
__global__ void __launch_bounds__(256) gen_cols_kernel(T* __restrict__ M, int64_t m, int64_t n, int64_t ld,
                                                       uint64_t seed_hi, uint64_t seed_lo, double sqrt_s,
                                                       double rho, double innov, int heavy, double loc) {
  uint32_t words[5];
  make_words(seed_hi, seed_lo, heavy ? 3u : 1u, words);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    NormalStream g;
    g.init(words, 5, (uint64_t)j);
    const double scale = heavy ? inv_sqrt_chi2(g) : 1.0;
    double x = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      const double z = g.next();
      x = (i == 0) ? sqrt_s * z : fma(rho, x, innov * z);
      put(M + i * ld + j, heavy ? loc + x * scale : x);
    }
  }
}

// N (n x p): row j = AR(1) vector of dimension p; lane = row, 32-wide f chunks
// staged through shared memory so the stores are row-contiguous
template <typename T>
__global__ void __launch_bounds__(128) gen_rows_kernel(T* __restrict__ N, int64_t n, int64_t p, int64_t ld,
                                                       uint64_t seed_hi, uint64_t seed_lo, double sqrt_s,
                                                       double rho, double innov, int heavy, double loc) {
  __shared__ double tile[4][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t words[5];
  make_words(seed_hi, seed_lo, heavy ? 4u : 2u, words);
  for (int64_t row0 = ((int64_t)blockIdx.x * 4 + w) * 32; row0 < n; row0 += (int64_t)gridDim.x * 4 * 32) {
    const int64_t j = row0 + lane;
    NormalStream g;
    g.init(words, 5, (uint64_t)(j < n ? j : 0));
    const double scale = heavy ? inv_sqrt_chi2(g) : 1.0;
    double x = 0.0;
    for (int64_t f0 = 0; f0 < p; f0 += 32) {
      const int cnt = (int)min((int64_t)32, p - f0);
      for (int f = 0; f < cnt; ++f) {
        const double z = g.next();
        x = (f0 + f == 0) ? sqrt_s * z : fma(rho, x, innov * z);
        tile[w][lane][f] = heavy ? loc + x * scale : x;
      }
      __syncwarp();
      for (int r = 0; r < 32 && row0 + r < n; ++r)
        if (lane < cnt) put(N + (row0 + r) * ld + f0 + lane, tile[w][r][lane]);
      __syncwarp();
    }
  }
}

template <typename T>
static int gen_impl(int heavy, int64_t m, int64_t n, int64_t p, uint64_t seed_hi, uint64_t seed_lo, double sL,
                    double rhoL, double sR, double rhoR, double loc, T* M, int64_t ldm, T* N, int64_t ldn,
                    cudaStream_t st) {
  if (M != nullptr) {
    gen_cols_kernel<T><<<grid_for(n, 256, 8, 4), 256, 0, st>>>(M, m, n, ldm, seed_hi, seed_lo, sqrt(sL), rhoL,
                                                              sqrt(sL * (1.0 - rhoL * rhoL)), heavy, loc);
    BMM_CHECK_LAUNCH("gen_cols_kernel");
  }
  if (N != nullptr) {
    gen_rows_kernel<T><<<grid_for(ceil_div(n, 32) * 32, 128, 8, 4), 128, 0, st>>>(
        N, n, p, ldn, seed_hi, seed_lo, sqrt(sR), rhoR, sqrt(sR * (1.0 - rhoR * rhoR)), heavy, loc);
    BMM_CHECK_LAUNCH("gen_rows_kernel");
  }
  return BMM_OK;
}


// ---- the reference's own variates (datagen.py:70-71, 104-106) -------------------------------
// Z (dim x count, row-major float64) holds rng.standard_normal((dim, count)) exactly as the
// reference draws it; vector j is column j of Z.  out = L @ Z by the AR(1) recursion (no
// transpose: out[i, j], M's layout) or its transpose (out[j, i], N's layout: the reference's
// ascontiguousarray((L @ Z).T)).  w != NULL: the heavy-tailed form loc + x / sqrt(w[j]) with
// the reference's operation order (a division by the square root, then the location).
template <typename T>
__global__ void __launch_bounds__(256) ar1_cols_kernel(const double* __restrict__ Z, int64_t dim, int64_t count,
                                                       int64_t ldz, double sqrt_s, double rho, double innov,
                                                       const double* __restrict__ w, double loc,
                                                       T* __restrict__ out, int64_t ldo) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double sw = w ? sqrt(w[j]) : 1.0;
    double x = 0.0;
    for (int64_t i = 0; i < dim; ++i) {
      const double z = Z[i * ldz + j];
      x = (i == 0) ? sqrt_s * z : fma(rho, x, innov * z);
      put(out + i * ldo + j, w ? loc + x / sw : x);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(128) ar1_rows_kernel(const double* __restrict__ Z, int64_t dim, int64_t count,
                                                       int64_t ldz, double sqrt_s, double rho, double innov,
                                                       const double* __restrict__ w, double loc,
                                                       T* __restrict__ out, int64_t ldo) {
  __shared__ double tile[4][32][33];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int64_t row0 = ((int64_t)blockIdx.x * 4 + wp) * 32; row0 < count; row0 += (int64_t)gridDim.x * 4 * 32) {
    const int64_t j = row0 + lane;
    const bool live = j < count;
    const double sw = (w && live) ? sqrt(w[j]) : 1.0;
    double x = 0.0;
    for (int64_t f0 = 0; f0 < dim; f0 += 32) {
      const int cnt = (int)min((int64_t)32, dim - f0);
      for (int f = 0; f < cnt; ++f) {
        const double z = live ? Z[(f0 + f) * ldz + j] : 0.0;
        x = (f0 + f == 0) ? sqrt_s * z : fma(rho, x, innov * z);
        tile[wp][lane][f] = w ? loc + x / sw : x;
      }
      __syncwarp();
      for (int r = 0; r < 32 && row0 + r < count; ++r)
        if (lane < cnt) put(out + (row0 + r) * ldo + f0 + lane, tile[wp][r][lane]);
      __syncwarp();
    }
  }
}

template <typename T>
static int ar1_impl(const double* Z, int64_t dim, int64_t count, int64_t ldz, int transpose_out, double scale,
                    double rho, const double* w, double loc, T* out, int64_t ldo, cudaStream_t st) {
  const double sqrt_s = sqrt(scale), innov = sqrt(scale * (1.0 - rho * rho));
  if (!transpose_out) {
    ar1_cols_kernel<T><<<grid_for(count, 256, 8, 4), 256, 0, st>>>(Z, dim, count, ldz, sqrt_s, rho, innov, w, loc,
                                                                  out, ldo);
    BMM_CHECK_LAUNCH("ar1_cols_kernel");
  } else {
    ar1_rows_kernel<T><<<grid_for(ceil_div(count, 32) * 32, 128, 8, 4), 128, 0, st>>>(Z, dim, count, ldz, sqrt_s,
                                                                                      rho, innov, w, loc, out, ldo);
    BMM_CHECK_LAUNCH("ar1_rows_kernel");
  }
  return BMM_OK;
}

}  // namespace bmm

using namespace bmm;

extern "C" int bmm_gen_instance(int heavy, int dtype, int64_t m, int64_t n, int64_t p, uint64_t seed_hi,
                                uint64_t seed_lo, double scale_left, double rho_left, double scale_right,
                                double rho_right, double location, void* M, int64_t ldm, void* N, int64_t ldn,
                                void* stream) {
  BMM_REQUIRE(m >= 1 && n >= 1 && p >= 1, BMM_E_ARG, "bmm_gen_instance: dimensions must be >= 1");
  BMM_REQUIRE(scale_left > 0 && scale_right > 0 && rho_left > -1 && rho_left < 1 && rho_right > -1 && rho_right < 1,
              BMM_E_ARG, "bmm_gen_instance: bad covariance parameters");
  cudaStream_t st = as_stream(stream);
  if (dtype == BMM_F64)
    return gen_impl<double>(heavy, m, n, p, seed_hi, seed_lo, scale_left, rho_left, scale_right, rho_right, location,
                            (double*)M, ldm, (double*)N, ldn, st);
  if (dtype == BMM_F32)
    return gen_impl<float>(heavy, m, n, p, seed_hi, seed_lo, scale_left, rho_left, scale_right, rho_right, location,
                           (float*)M, ldm, (float*)N, ldn, st);
  set_error("bmm_gen_instance: unknown dtype %d", dtype);
  return BMM_E_ARG;
}

extern "C" int bmm_ar1_transform(int dtype, const double* Z, int64_t dim, int64_t count, int64_t ldz,
                                 int transpose_out, double scale, double rho, const double* w_opt, double location,
                                 void* out, int64_t ldo, void* stream) {
  BMM_REQUIRE(dim >= 1 && count >= 1 && ldz >= count, BMM_E_ARG, "bmm_ar1_transform: bad dimensions");
  BMM_REQUIRE(ldo >= (transpose_out ? dim : count), BMM_E_ARG, "bmm_ar1_transform: bad output stride");
  BMM_REQUIRE(scale > 0 && rho > -1 && rho < 1, BMM_E_ARG, "bmm_ar1_transform: bad covariance parameters");
  cudaStream_t st = as_stream(stream);
  if (dtype == BMM_F64)
    return ar1_impl<double>(Z, dim, count, ldz, transpose_out, scale, rho, w_opt, location, (double*)out, ldo, st);
  if (dtype == BMM_F32)
    return ar1_impl<float>(Z, dim, count, ldz, transpose_out, scale, rho, w_opt, location, (float*)out, ldo, st);
  set_error("bmm_ar1_transform: unknown dtype %d", dtype);
  return BMM_E_ARG;
}
