// numpy-compatible random streams on device: SeedSequence pool hashing and
// PCG64 (XSL-RR 128/64, "set-seq" seeding), plus O(log n) jump-ahead so the
// 32 lanes of a warp draw consecutive uniforms of one stream in parallel.
//
// The reference draws with numpy.random.Generator(PCG64): rng.spawn(K)
// (estimators.py:141,207; plan.py:456) and rng.random(count)
// (estimators.py:41).  numpy is a third-party dependency (numpy 2.3.5 here);
// the published algorithms are restated in oracle/numpy_rng.py and pinned
// against live numpy vectors (tests/test_oracle_rng.py).
#pragma once
#include <cstdint>

namespace bmm {

struct U128 {
  uint64_t hi, lo;
};

__host__ __device__ __forceinline__ U128 u128(uint64_t hi, uint64_t lo) { return U128{hi, lo}; }

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ULL : 0ULL);
  return r;
}

// PCG_DEFAULT_MULTIPLIER_128 = 0x2360ED051FC65DA44385DF649FCCF645
__device__ __forceinline__ U128 pcg_mult() { return U128{0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL}; }

__device__ __forceinline__ U128 pcg_step(U128 state, U128 inc) { return add128(mul128(state, pcg_mult()), inc); }

// XSL-RR output of a 128-bit state
__device__ __forceinline__ uint64_t pcg_output(U128 s) {
  const unsigned rot = (unsigned)(s.hi >> 58);
  const uint64_t x = s.hi ^ s.lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// next_double: (next64 >> 11) * 2^-53
__device__ __forceinline__ double u53(uint64_t x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }

// Affine map (mult, plus) advancing an LCG state by `delta` steps.
__device__ __forceinline__ void pcg_jump(uint64_t delta, U128 inc, U128& am, U128& ap) {
  U128 acc_m{0, 1}, acc_p{0, 0}, cur_m = pcg_mult(), cur_p = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_m = mul128(acc_m, cur_m);
      acc_p = add128(mul128(acc_p, cur_m), cur_p);
    }
    cur_p = mul128(add128(cur_m, U128{0, 1}), cur_p);
    cur_m = mul128(cur_m, cur_m);
    delta >>= 1;
  }
  am = acc_m;
  ap = acc_p;
}

// ---- PCG64 jump table: the state i steps ahead is a^i * s + inc * S_i (mod 2^128) with
// S_i = 1 + a + ... + a^(i-1) independent of the stream, so a draw's state costs two 128-bit
// multiplies instead of pcg_jump's O(log i) loop.  Constant-initialised at compile time.
struct U128c {
  uint64_t hi, lo;
};

constexpr U128c mul128c(U128c a, U128c b) {
  const uint64_t a0 = a.lo & 0xffffffffULL, a1 = a.lo >> 32, b0 = b.lo & 0xffffffffULL, b1 = b.lo >> 32;
  const uint64_t p00 = a0 * b0, p01 = a0 * b1, p10 = a1 * b0, p11 = a1 * b1;
  const uint64_t mid = (p00 >> 32) + (p01 & 0xffffffffULL) + (p10 & 0xffffffffULL);
  const uint64_t lo = (p00 & 0xffffffffULL) | (mid << 32);
  const uint64_t hi = p11 + (p01 >> 32) + (p10 >> 32) + (mid >> 32) + a.lo * b.hi + a.hi * b.lo;
  return U128c{hi, lo};
}

constexpr int kPcgTable = 1024;

struct PcgTable {
  uint64_t v[kPcgTable + 1][4];  // a^i (hi, lo), S_i (hi, lo)
  constexpr PcgTable() : v{} {
    const U128c a{0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL};
    U128c am{0, 1}, S{0, 0};
    for (int i = 0; i <= kPcgTable; ++i) {
      v[i][0] = am.hi;
      v[i][1] = am.lo;
      v[i][2] = S.hi;
      v[i][3] = S.lo;
      S = mul128c(S, a);
      S.lo += 1;
      if (S.lo == 0) S.hi += 1;
      am = mul128c(am, a);
    }
  }
};

__device__ constexpr PcgTable kPcgAhead{};

// the state `steps` >= 0 ahead of `state` on the stream with increment `inc`
__device__ __forceinline__ U128 pcg_ahead(U128 state, U128 inc, uint64_t steps) {
  if (steps <= (uint64_t)kPcgTable) {
    const uint64_t* e = kPcgAhead.v[steps];
    return add128(mul128(state, U128{e[0], e[1]}), mul128(inc, U128{e[2], e[3]}));
  }
  U128 am, ap;
  pcg_jump(steps, inc, am, ap);
  return add128(mul128(state, am), ap);
}

// ---- SeedSequence (pool_size 4)
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

__device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= kMultA;
  v *= hc;
  v ^= v >> 16;
  return v;
}

__device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

// Entropy = words[0..nw) followed by the 32-bit words of `child` (1 or 2).
// Returns the PCG64 (state, inc) numpy derives from that SeedSequence.
__device__ inline void seed_pcg64(const uint32_t* words, int64_t nw, uint64_t child, U128& state,
                                  U128& inc) {
  const int64_t nchild = (child >> 32) ? 2 : 1;
  const int64_t L = nw + nchild;
  auto ent = [&](int64_t i) -> uint32_t {
    if (i < nw) return words[i];
    return (i == nw) ? (uint32_t)(child & 0xffffffffu) : (uint32_t)(child >> 32);
  };
  uint32_t hc = kInitA;
  uint32_t pool[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < L ? ent(i) : 0u, hc);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int64_t s = 4; s < L; ++s) {
    const uint32_t e = ent(s);
#pragma unroll
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(e, hc));
  }
  // generate_state(4, uint64)
  uint32_t w[8];
  uint32_t hb = kInitB;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  const uint64_t s0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  const uint64_t s1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
  const uint64_t s2 = (uint64_t)w[4] | ((uint64_t)w[5] << 32);
  const uint64_t s3 = (uint64_t)w[6] | ((uint64_t)w[7] << 32);
  // pcg_setseq_128_srandom_r(initstate = s0:s1, initseq = s2:s3)
  inc = U128{(s2 << 1) | (s3 >> 63), (s3 << 1) | 1ULL};
  U128 st{0, 0};
  st = pcg_step(st, inc);
  st = add128(st, U128{s0, s1});
  st = pcg_step(st, inc);
  state = st;
}

}  // namespace bmm
