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

__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               const RoundKeys& rk) {
  constexpr uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(kMul0, c0), lo0 = kMul0 * c0;
    const uint32_t hi1 = __umulhi(kMul1, c2), lo1 = kMul1 * c2;
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

// Counter word 1 for quad b: b | kw << 8 | jw << 16.
__device__ __forceinline__ uint32_t ctr_word1(uint32_t b, uint32_t kw, uint32_t jw) {
  return b | (kw << 8) | (jw << 16);
}

// ẑ of quads B.. of a sample from their Philox words (compile-time recursion over quads).
template <int NDIM, int B = 0>
__device__ __forceinline__ void normals_from_words(float (&z)[NDIM],
                                                   const uint4 (&w)[(NDIM + 3) / 4]) {
  constexpr int d = 4 * B;
  float t0, t1, t2, t3;
  box_muller_hat<(d + 1 < NDIM)>(w[B].x, w[B].y, t0, t1);
  z[d] = t0;
  if constexpr (d + 1 < NDIM) z[d + 1] = t1;
  if constexpr (d + 2 < NDIM) {
    box_muller_hat<(d + 3 < NDIM)>(w[B].z, w[B].w, t2, t3);
    z[d + 2] = t2;
    if constexpr (d + 3 < NDIM) z[d + 3] = t3;
  }
  if constexpr (B + 1 < (NDIM + 3) / 4) normals_from_words<NDIM, B + 1>(z, w);
}

// ẑ of one quad from its Philox words (the first min(NDIM, 4) coordinates).
template <int NDIM>
__device__ __forceinline__ void quad_normals_hat(float (&z)[NDIM], uint4 w) {
  float t0, t1, t2, t3;
  box_muller_hat<(NDIM >= 2)>(w.x, w.y, t0, t1);
  z[0] = t0;
  if constexpr (NDIM >= 2) z[1] = t1;
  if constexpr (NDIM >= 3) {
    box_muller_hat<(NDIM >= 4)>(w.z, w.w, t2, t3);
    z[2] = t2;
    if constexpr (NDIM >= 4) z[3] = t3;
  }
}

// ẑ (= z / C) of draw `draw` (= sample index, or index >> 1 under antithetic sampling).
template <int NDIM>
__device__ __forceinline__ void sample_normals_hat(float (&z)[NDIM], uint32_t draw, uint32_t w1base,
                                                   uint32_t qid, uint32_t tag, const RoundKeys& rk) {
  constexpr int kQuads = (NDIM + 3) / 4;
#pragma unroll
  for (int b = 0; b < kQuads; ++b) {
    const uint4 w = philox4x32_10(draw, w1base | (uint32_t)b, qid, tag, rk);
    float t0, t1, t2, t3;
    box_muller_hat<true>(w.x, w.y, t0, t1);
    if (4 * b + 0 < NDIM) z[4 * b + 0] = t0;
    if (4 * b + 1 < NDIM) z[4 * b + 1] = t1;
    if (4 * b + 2 < NDIM) {
      if (4 * b + 3 < NDIM) {
        box_muller_hat<true>(w.z, w.w, t2, t3);
        z[4 * b + 2] = t2;
        z[4 * b + 3] = t3;
      } else {
        box_muller_hat<false>(w.z, w.w, t2, t3);
        z[4 * b + 2] = t2;
      }
    }
  }
}

}  // namespace hjmc
