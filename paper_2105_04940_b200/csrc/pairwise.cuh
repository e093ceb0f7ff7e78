// numpy's float64 summation orders, restated for one device thread.
//
// The reference reduces with numpy (third-party, numpy 2.3.5 in this image):
//   * ``x.sum()`` / ``add.reduce`` over a contiguous axis is 0 + pairwise(x)
//     (plan.py:200,205; integerize plan.py:267,311,323; row_norms matrix.py:114)
//   * ``np.add.reduceat(x, starts)`` is x[o] + pairwise(x[o+1:e])  (plan.py:173)
//   * ``np.cumsum`` is strictly sequential                           (estimators.py:37)
// pairwise(n):  n < 8    -> ((0 + a0) + a1) + ...
//               n <= 128 -> 8 strided accumulators r0..r7, combined as
//                           ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8
//                           tail added sequentially
//               else     -> n2 = n/2 - (n/2)%8;  pairwise(a[:n2]) + pairwise(a[n2:])
// Verified bit-for-bit against numpy in tests/test_oracle_orders.py.
//
// `Src` supplies element values as doubles: src(i) for one element and
// src.load8(i, v) for 8 consecutive elements starting at i (i % 8 == 0 within
// the summed range) so that a leaf streams 32/64-byte vectors per step.
#pragma once
#include <cstdint>

namespace bmm {

template <class Src>
__device__ __forceinline__ double pw_leaf(const Src& src, int64_t s, int64_t len) {
  if (len < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < len; ++i) r = __dadd_rn(r, src(s + i));
    return r;
  }
  double r[8];
  src.load8(s, r);
  const int64_t body = len - (len % 8);
  int64_t i = 8;
#pragma unroll 4
  for (; i < body; i += 8) {
    double v[8];
    src.load8(s + i, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < len; ++i) res = __dadd_rn(res, src(s + i));
  return res;
}

// Post-order walk of NumPy's pairwise split tree over [start, start+n),
// calling leaf(s, len) for the <=128-element leaves left to right and
// combining left + right exactly as the recursion does (depth <=
// log2(n/64) + 1, so 40 frames cover any int64 n).
template <class LeafFn>
__device__ double pw_tree(int64_t start, int64_t n, LeafFn&& leaf) {
  if (n <= 128) return leaf(start, n);
  int64_t fs[40], fl[40];
  double fleft[40];
  int fstage[40];
  int sp = 0;
  fs[0] = start; fl[0] = n; fstage[0] = 0;
  for (;;) {
    int64_t len = fl[sp];
    if (len > 128) {
      // descend into the left child
      int64_t n2 = len / 2;
      n2 -= n2 % 8;
      fstage[sp] = 0;
      ++sp;
      fs[sp] = fs[sp - 1];
      fl[sp] = n2;
      continue;
    }
    double ret = leaf(fs[sp], len);
    // unwind: combine with finished left siblings, or descend into a right child
    for (;;) {
      if (sp == 0) return ret;
      --sp;
      int64_t plen = fl[sp];
      int64_t n2 = plen / 2;
      n2 -= n2 % 8;
      if (fstage[sp] == 0) {
        fleft[sp] = ret;
        fstage[sp] = 1;
        ++sp;
        fs[sp] = fs[sp - 1] + n2;
        fl[sp] = plen - n2;
        fstage[sp] = 0;
        break;
      }
      ret = __dadd_rn(fleft[sp], ret);
    }
  }
}

// numpy pairwise sum of src(start .. start+n), one thread.
template <class Src>
__device__ double pw_sum(const Src& src, int64_t start, int64_t n) {
  return pw_tree(start, n, [&](int64_t s, int64_t len) { return pw_leaf(src, s, len); });
}

// np.cumsum of p[0..len) into cum (strictly sequential float64 chain,
// cum[0] = p[0]) by one warp: lanes load 32 values at a time, every lane runs
// the same 32-step chain over the shuffled values and keeps its own prefix,
// so loads and stores are coalesced while the adds stay in NumPy's order.
// Returns (to every lane) the last index with p > 0, or -1.
__device__ __forceinline__ int64_t warp_cumsum(const double* __restrict__ p, double* __restrict__ cum,
                                               int64_t len) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  int64_t last = -1;
  for (int64_t base = 0; base < len; base += 32) {
    const int64_t i = base + lane;
    const double x = (i < len) ? p[i] : 0.0;
    const unsigned pos = __ballot_sync(0xffffffffu, x > 0.0);
    if (pos) last = base + 31 - __clz(pos);
    double mine = 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const double v = __shfl_sync(0xffffffffu, x, q);
      acc = __dadd_rn(acc, v);  // 0 + p[0] == p[0]: probabilities are never -0
      if (lane == q) mine = acc;
    }
    if (i < len) cum[i] = mine;
  }
  return last;
}

// ---- warp-cooperative version --------------------------------------------
// The same tree, with leaves evaluated in parallel: lane group g = lane/8
// takes leaf 4q+g, lane j = lane%8 runs accumulator r_j (elements j, j+8, ...),
// the 8 accumulators combine through an xor butterfly (commutative adds, so
// every lane ends with ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))), lane j=0 adds
// the tail, and lane 0 walks the tree over the stored leaf values.
// scratch: per-warp shared memory for kWarpLeaves leaves.
constexpr int kWarpLeaves = 128;

struct WarpPwScratch {
  double val[kWarpLeaves];
  int64_t start[kWarpLeaves];
  int32_t len[kWarpLeaves];
};

template <class Src>
__device__ __forceinline__ double warp_leaf8(const Src& src, int64_t s, int64_t len, int j) {
  // accumulator j of a leaf with 8 <= len <= 128: at most 16 strided elements,
  // all loaded before the (ordered) adds so the whole leaf is in flight at once
  const int steps = (int)(len / 8);
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = (q < steps) ? src(s + 8 * q + j) : 0.0;
  double r = v[0];
#pragma unroll
  for (int q = 1; q < 16; ++q)
    if (q < steps) r = __dadd_rn(r, v[q]);
  return r;
}

__device__ __forceinline__ double group8_reduce(double r) {
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
  return r;
}

// All 32 lanes must call; every lane receives the sum.
template <class Src>
__device__ double warp_pw_sum(const Src& src, int64_t start, int64_t n, WarpPwScratch* scr) {
  const int lane = threadIdx.x & 31;
  const int j = lane & 7, grp = lane >> 3;
  if (n < 8) {
    double r = 0.0;
    if (lane == 0)
      for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, src(start + i));
    return __shfl_sync(0xffffffffu, r, 0);
  }
  if (n <= 128) {
    double r = (grp == 0) ? warp_leaf8(src, start, n, j) : 0.0;
    r = group8_reduce(r);
    if (lane == 0)
      for (int64_t i = n - (n % 8); i < n; ++i) r = __dadd_rn(r, src(start + i));
    return __shfl_sync(0xffffffffu, r, 0);
  }
  // enumerate leaves (lane 0) in left-to-right order
  int count = 0;
  if (lane == 0) {
    pw_tree(start, n, [&](int64_t s, int64_t len) {
      if (count < kWarpLeaves) { scr->start[count] = s; scr->len[count] = (int32_t)len; }
      ++count;
      return 0.0;
    });
  }
  count = __shfl_sync(0xffffffffu, count, 0);
  __syncwarp();
  if (count > kWarpLeaves) {  // very long range: single-lane walk
    double r = 0.0;
    if (lane == 0) r = pw_sum(src, start, n);
    return __shfl_sync(0xffffffffu, r, 0);
  }
  for (int base = 0; base < count; base += 4) {
    const int q = base + grp;
    const bool on = q < count;
    int64_t s = 0, len = 0;
    double r = 0.0;
    if (on) {
      s = scr->start[q];
      len = scr->len[q];
      r = warp_leaf8(src, s, len, j);
    }
    r = group8_reduce(r);
    if (on && j == 0) {
      for (int64_t i = len - (len % 8); i < len; ++i) r = __dadd_rn(r, src(s + i));
      scr->val[q] = r;
    }
  }
  __syncwarp();
  double res = 0.0;
  if (lane == 0) {
    int idx = 0;
    res = pw_tree(start, n, [&](int64_t, int64_t) { return scr->val[idx++]; });
  }
  res = __shfl_sync(0xffffffffu, res, 0);
  __syncwarp();
  return res;
}

// ---- element sources -------------------------------------------------------

// Plain contiguous float64 array.
struct SrcF64 {
  const double* a;
  __device__ double operator()(int64_t i) const { return a[i]; }
  __device__ void load8(int64_t i, double* v) const {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = a[i + j];
  }
};

// Squares of a contiguous row (float64 or float32 upcast); vectorised loads
// when the row base is 16-byte aligned.
template <class T>
struct SrcSq;

template <>
struct SrcSq<double> {
  const double* a;
  bool aligned;
  __device__ double operator()(int64_t i) const { double x = a[i]; return __dmul_rn(x, x); }
  __device__ void load8(int64_t i, double* v) const {
    if (aligned) {
      const double2* p = reinterpret_cast<const double2*>(a + i);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double2 t = __ldg(p + j);
        v[2 * j] = __dmul_rn(t.x, t.x);
        v[2 * j + 1] = __dmul_rn(t.y, t.y);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) { double x = a[i + j]; v[j] = __dmul_rn(x, x); }
    }
  }
};

template <>
struct SrcSq<float> {
  const float* a;
  bool aligned;
  __device__ double operator()(int64_t i) const { double x = (double)a[i]; return __dmul_rn(x, x); }
  __device__ void load8(int64_t i, double* v) const {
    if (aligned) {
      const float4* p = reinterpret_cast<const float4*>(a + i);
      float4 t0 = __ldg(p), t1 = __ldg(p + 1);
      float f[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) { double x = (double)f[j]; v[j] = __dmul_rn(x, x); }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) { double x = (double)a[i + j]; v[j] = __dmul_rn(x, x); }
    }
  }
};

}  // namespace bmm
