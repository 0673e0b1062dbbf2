// hjmc_rng.cuh — counter-based Gaussian sampling in registers (SURVEY §8(a) rows a2–a3).
//
// Philox4x32-10 (Salmon et al., SC'11) and the Box–Muller transform exactly as frozen in
// include/hjmc.h "RANDOM NUMBERS" (reading R19). No sample ever touches memory: every normal is
// regenerated from (sample index, quad, iterate, horizon, query id, tag) when it is needed.
//
// Paper passages: samples y_i ~ N(0, I_n) i.i.d. (Cor. logsumexp; Thm 1).
#pragma once
#include <cstdint>

namespace hjmc {

// ---- MUFU-backed approximations (sm_100a). All are within ~2 ulp-equivalents of the exact
// functions on the ranges used here (DESIGN.md §5 lists the error budget). -----------------
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sin_approx(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cos_approx(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Hide a value's provenance from the optimiser so a loop-invariant stays in a register instead of
// being re-derived inside the sample loop (e.g. a double→float conversion on the XU pipe).
__device__ __forceinline__ float opaque(float v) {
  float r;
  asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// ---- Philox4x32-10 ---------------------------------------------------------------------------
// The 10 round keys (k0 + r·0x9E3779B9, k1 + r·0xBB67AE85) are the same for every sample, so
// the host precomputes them into the kernel parameters: the XOR reads them straight from the
// constant bank and the loop carries no key-schedule arithmetic.
struct RoundKeys {
  uint32_t k0[10], k1[10];
};

inline void make_round_keys(uint64_t seed, RoundKeys* rk) {
  uint32_t k0 = (uint32_t)(seed & 0xFFFFFFFFull), k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    rk->k0[r] = k0;
    rk->k1[r] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// 32×32→64 multiply as one IMAD.WIDE.U32 (4 FMA-heavy cycles per warp); left to itself ptxas
// sometimes splits it into IMAD + IMAD.HI (2 + 4 cycles).
__device__ __forceinline__ void mul_wide(uint32_t a, uint32_t m, uint32_t& hi, uint32_t& lo) {
  asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}"
      : "=r"(lo), "=r"(hi)
      : "r"(a), "r"(m));
}

// ---- the high word of a Philox product on the FP64 pipe -----------------------------------------
// IMAD.WIDE.U32 occupies the FMA-heavy pipe for 4 cycles per warp, and that pipe is one of the
// three co-limits of the sample loop. The same product can be split: the low word
// by IMAD (2 cycles, FMA-heavy) and the high word by ONE DFMA on the separate FP64 pipe, exactly.
// Carry a 32-bit word c as the double whose bit pattern is {lo = c, hi = 0x43300000}, i.e.
// a = 2^52 + c. With b = M·2^-32 and K = 2^52 − 2^20·M (both exact: M and 2^32 − M are 32-bit
// integers scaled by powers of two),
//   fma.rm(a, b, K) = 2^52 + c·M·2^-32 rounded down = 2^52 + floor(c·M / 2^32),
// because c·M·2^-32 < 2^32 keeps the sum in [2^52, 2^53) where one ulp is 1. So the result's low
// word IS mulhi(c, M) and its high word is again 0x43300000 — the pattern the next round's input
// needs, since the round's XOR rewrites only the low word. Exact integer arithmetic: bit-identical
// to IMAD.WIDE by construction.
// Which of the 20 products take the FP64 path: bit 2r = round r's c0·M0 product, bit 2r + 1 =
// round r's c2·M1 product. 0 = IMAD.WIDE everywhere.
#ifndef HJMC_PHILOX_DFMA_MASK
#define HJMC_PHILOX_DFMA_MASK 0u
#endif
constexpr uint64_t kPairHi = 0x4330000000000000ull;  // {lo = c, hi = 0x43300000} = 2^52 + c

template <uint32_t kM>
__device__ __forceinline__ uint64_t mulhi_dfma(uint64_t pair) {
  constexpr double kB = (double)kM * (1.0 / 4294967296.0);
  constexpr double kK = 4503599627370496.0 - 1048576.0 * (double)kM;  // 2^52 − 2^20·M
  double r;
  asm("fma.rm.f64 %0, %1, %2, %3;" : "=d"(r) : "d"(__longlong_as_double((long long)pair)),
      "d"(kB), "d"(kK));
  return (uint64_t)__double_as_longlong(r);
}

template <uint32_t kMask>
__device__ __forceinline__ uint4 philox4x32_10_mixed(uint32_t c0, uint32_t c1, uint32_t c2,
                                                     uint32_t c3, const RoundKeys& rk) {
  constexpr uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;
  // p0 / p2: c0 / c2 carried as {word, 0x43300000}; the XOR below touches only the low word
  uint64_t p0 = kPairHi | c0, p2 = kPairHi | c2;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const bool d0 = (kMask >> (2 * r)) & 1u, d1 = (kMask >> (2 * r + 1)) & 1u;
    const uint32_t w0 = (uint32_t)p0, w2 = (uint32_t)p2;
    uint64_t h0, h1;  // {mulhi, 0x43300000}
    uint32_t lo0, lo1;
    if (d0) {
      h0 = mulhi_dfma<kMul0>(p0);
      lo0 = w0 * kMul0;
    } else {
      uint32_t hi;
      mul_wide(w0, kMul0, hi, lo0);
      h0 = kPairHi | hi;
    }
    if (d1) {
      h1 = mulhi_dfma<kMul1>(p2);
      lo1 = w2 * kMul1;
    } else {
      uint32_t hi;
      mul_wide(w2, kMul1, hi, lo1);
      h1 = kPairHi | hi;
    }
    p0 = h1 ^ (uint64_t)(c1 ^ rk.k0[r]);
    p2 = h0 ^ (uint64_t)(c3 ^ rk.k1[r]);
    c1 = lo1;
    c3 = lo0;
  }
  return make_uint4((uint32_t)p0, c1, (uint32_t)p2, c3);
}

__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               const RoundKeys& rk) {
  if constexpr (HJMC_PHILOX_DFMA_MASK != 0u)
    return philox4x32_10_mixed<HJMC_PHILOX_DFMA_MASK>(c0, c1, c2, c3, rk);
  constexpr uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mul_wide(c0, kMul0, hi0, lo0);
    mul_wide(c2, kMul1, hi1, lo1);
    const uint32_t n0 = hi1 ^ c1 ^ rk.k0[r];
    const uint32_t n2 = hi0 ^ c3 ^ rk.k1[r];
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}

// m = w >> 9 (high 23 bits). 0x3F800000 + m is the float 1 + m·2^-23 = 1 + a(w) (one LEA.HI):
//   u(w) = (2m+1)·2^-24 = (1 + m·2^-23) − (1 − 2^-24)   exact (both operands in [0.5, 2))
__device__ __forceinline__ float mantissa_float(uint32_t w) {
  return __uint_as_float((w >> 9) + 0x3F800000u);
}
__device__ __forceinline__ float unif_open(uint32_t w) {
  return mantissa_float(w) - 0.99999994039535522f;  // 1 − 2^-24
}

// Box–Muller scaled by 1/C, C = sqrt(2 ln 2): returns ẑ with z = C·ẑ, i.e.
//   ẑ_cos = sqrt(−log2 u)·cos(2π(1 + a)),  ẑ_sin = sqrt(−log2 u)·sin(2π(1 + a)),
// since r = sqrt(−2 ln u) = C·sqrt(−log2 u) and sin/cos are 2π-periodic, so the angle is
// formed straight from the mantissa float 1 + a (no centring add); MUFU.SIN/COS take their
// argument in revolutions, so 2π(1+a)·(1/2π) ∈ [1, 2) keeps the full 2^-23 angle resolution.
// The caller folds C into σ (y = x + (σC)·ẑ) and into the moment epilogue, which saves one
// multiply per pair. kNeedSin = false skips the sin (odd n: last normal of the quad unused).
constexpr float kBMScale = 1.1774100225154747f;  // sqrt(2 ln 2)

template <bool kNeedSin = true>
__device__ __forceinline__ void box_muller_hat(uint32_t w_r, uint32_t w_a, float& zc, float& zs) {
  constexpr float kTwoPi = 6.2831853071795865f;
  // log2 u < 0 for every u < 1; |·| guards the MUFU rounding sign near u = 1 (free modifier)
  const float rh = sqrt_approx(fabsf(lg2_approx(unif_open(w_r))));
  const float th = kTwoPi * mantissa_float(w_a);
  zc = rh * cos_approx(th);
  if (kNeedSin) zs = rh * sin_approx(th);
}

// The same transform left in polar form: ẑ_cos = rh·c, ẑ_sin = rh·s. The lane-group kernel keeps
// (rh, c, s) and never forms the products: the sample position comes from one FFMA per
// coordinate in σ-scaled coordinates, the moments from the pair's w·rh (hjmc_solve_impl.cuh).
__device__ __forceinline__ void box_muller_polar(uint32_t w_r, uint32_t w_a, float& rh, float& c,
                                                 float& s) {
  constexpr float kTwoPi = 6.2831853071795865f;
  rh = sqrt_approx(fabsf(lg2_approx(unif_open(w_r))));
  const float th = kTwoPi * mantissa_float(w_a);
  c = cos_approx(th);
  s = sin_approx(th);
}

// Counter word 1 for quad b: b | kw << 8 | jw << 16.
__device__ __forceinline__ uint32_t ctr_word1(uint32_t b, uint32_t kw, uint32_t jw) {
  return b | (kw << 8) | (jw << 16);
}

// ---- draw layout (R19) -----------------------------------------------------------------------
// G = 4/gcd(n,4) consecutive draws share one flat stream of G·n normals (Q = G·n/4 Philox
// blocks) when G·n ≤ 16; otherwise G = 1 and a draw owns Q = ceil(n/4) blocks. Block b of
// draw group g has counter (g, b | kw<<8 | jw<<16, qid, tag): for n = 2, 3, 6 no normal of a
// Philox call is wasted, and since c0 = g is common to the group's blocks while c1 differs only
// by the compile-time b, the first Philox rounds are shared across them (their multiplies are
// per group or warp-uniform).
template <int NDIM>
struct DrawLayout {
  static constexpr int G0 = (NDIM % 4 == 0) ? 1 : ((NDIM % 2 == 0) ? 2 : 4);
  static constexpr int G = (G0 * NDIM <= 16) ? G0 : 1;
  static constexpr int Q = (G == 1) ? (NDIM + 3) / 4 : G * NDIM / 4;
  static constexpr int L = G * NDIM;  // normals produced per group
};

// The G·n normals ẑ of draw group g (sample r of the group: zz[r·n .. r·n + n − 1]).
template <int NDIM>
__device__ __forceinline__ void group_normals_hat(float (&zz)[DrawLayout<NDIM>::L], uint32_t g,
                                                  uint32_t w1base, uint32_t qid, uint32_t tag,
                                                  const RoundKeys& rk) {
  using L = DrawLayout<NDIM>;
#pragma unroll
  for (int b = 0; b < L::Q; ++b) {
    const uint4 w = philox4x32_10(g, w1base | (uint32_t)b, qid, tag, rk);
    constexpr int kLen = L::L;
    const int e = 4 * b;
    float t0, t1, t2, t3;
    if (e < kLen) {
      if (e + 1 < kLen) box_muller_hat<true>(w.x, w.y, t0, t1);
      else box_muller_hat<false>(w.x, w.y, t0, t1);
      zz[e] = t0;
      if (e + 1 < kLen) zz[e + 1] = t1;
    }
    if (e + 2 < kLen) {
      if (e + 3 < kLen) box_muller_hat<true>(w.z, w.w, t2, t3);
      else box_muller_hat<false>(w.z, w.w, t2, t3);
      zz[e + 2] = t2;
      if (e + 3 < kLen) zz[e + 3] = t3;
    }
  }
}

// The same G·n normals in polar form: ẑ_e = rr[e]·tt[e], rr[e] = rr[e ^ 1] the pair's radius
// (duplicated per normal so a sample's coordinates index it directly; after unrolling the copies
// are the same register).
template <int NDIM>
__device__ __forceinline__ void group_normals_polar(float (&tt)[DrawLayout<NDIM>::L],
                                                    float (&rr)[DrawLayout<NDIM>::L], uint32_t g,
                                                    uint32_t w1base, uint32_t qid, uint32_t tag,
                                                    const RoundKeys& rk) {
  using L = DrawLayout<NDIM>;
  constexpr int kLen = L::L;
#pragma unroll
  for (int b = 0; b < L::Q; ++b) {
    const uint4 w = philox4x32_10(g, w1base | (uint32_t)b, qid, tag, rk);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = 4 * b + 2 * h;
      if (e < kLen) {
        constexpr float kTwoPi = 6.2831853071795865f;
        const float rh = sqrt_approx(fabsf(lg2_approx(unif_open(h ? w.z : w.x))));
        const float th = kTwoPi * mantissa_float(h ? w.w : w.y);
        rr[e] = rh;
        tt[e] = cos_approx(th);
        if (e + 1 < kLen) {
          rr[e + 1] = rh;
          tt[e + 1] = sin_approx(th);
        }
      }
    }
  }
}

}  // namespace hjmc
