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
#pragma unroll 2
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

// numpy pairwise sum of src(start .. start+n).  Iterative post-order walk of
// the split tree (depth <= log2(n/64) + 1, so 40 frames cover any int64 n).
template <class Src>
__device__ double pw_sum(const Src& src, int64_t start, int64_t n) {
  if (n <= 128) return pw_leaf(src, start, n);
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
    double ret = pw_leaf(src, fs[sp], len);
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
