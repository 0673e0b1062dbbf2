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
struct Key {
  uint32_t k0, k1;
};

__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               Key key) {
  constexpr uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;
  constexpr uint32_t kWeyl0 = 0x9E3779B9u, kWeyl1 = 0xBB67AE85u;
  uint32_t k0 = key.k0, k1 = key.k1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(kMul0, c0), lo0 = kMul0 * c0;
    const uint32_t hi1 = __umulhi(kMul1, c2), lo1 = kMul1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += kWeyl0;
    k1 += kWeyl1;
  }
  return make_uint4(c0, c1, c2, c3);
}

// u(w) = (2m+1)·2^-24 with m = w & 0x7FFFFF, built exactly from the mantissa bits:
// 1 + m·2^-23 − (1 − 2^-24) = (2m+1)·2^-24 (both operands in [0.5, 2): exact subtraction).
__device__ __forceinline__ float unif_open(uint32_t w) {
  return __int_as_float((w & 0x007FFFFFu) | 0x3F800000u) - 0.99999994039535522f;  // 1 − 2^-24
}
// a(w) − 1/2 = m·2^-23 − 1/2 ∈ [−1/2, 1/2), exact.
__device__ __forceinline__ float unif_angle_centered(uint32_t w) {
  return __int_as_float((w & 0x007FFFFFu) | 0x3F800000u) - 1.5f;
}

// One Box–Muller pair from words (w_r, w_a): (r cos 2πa, r sin 2πa).
// cos(2πa) = −cos(2π(a − ½)), sin(2πa) = −sin(2π(a − ½)); the centred angle keeps the MUFU
// sin/cos argument in [−π, π) where their error is smallest. kNeedSin = false skips the sin
// (odd dimension: the last normal of the quad is not used).
template <bool kNeedSin = true>
__device__ __forceinline__ void box_muller(uint32_t w_r, uint32_t w_a, float& z_cos, float& z_sin) {
  constexpr float kMinus2Ln2 = -1.3862943611198906f;  // −2 ln 2: −2 ln u = −2 ln2 · log2 u
  constexpr float kTwoPi = 6.2831853071795865f;
  const float nr = -sqrt_approx(kMinus2Ln2 * lg2_approx(unif_open(w_r)));  // −r
  const float th = kTwoPi * unif_angle_centered(w_a);
  z_cos = nr * cos_approx(th);
  if (kNeedSin) z_sin = nr * sin_approx(th);
}

// Counter word 1 for quad b: b | kw << 8 | jw << 16.
__device__ __forceinline__ uint32_t ctr_word1(uint32_t b, uint32_t kw, uint32_t jw) {
  return b | (kw << 8) | (jw << 16);
}

// The NDIM normals of draw `draw` (= sample index, or index >> 1 under antithetic sampling).
template <int NDIM>
__device__ __forceinline__ void sample_normals(float (&z)[NDIM], uint32_t draw, uint32_t w1base,
                                               uint32_t qid, uint32_t tag, Key key) {
  constexpr int kQuads = (NDIM + 3) / 4;
#pragma unroll
  for (int b = 0; b < kQuads; ++b) {
    const uint4 w = philox4x32_10(draw, w1base | (uint32_t)b, qid, tag, key);
    float t0, t1, t2, t3;
    box_muller<true>(w.x, w.y, t0, t1);
    if (4 * b + 0 < NDIM) z[4 * b + 0] = t0;
    if (4 * b + 1 < NDIM) z[4 * b + 1] = t1;
    if (4 * b + 2 < NDIM) {
      if (4 * b + 3 < NDIM) {
        box_muller<true>(w.z, w.w, t2, t3);
        z[4 * b + 2] = t2;
        z[4 * b + 3] = t3;
      } else {
        box_muller<false>(w.z, w.w, t2, t3);
        z[4 * b + 2] = t2;
      }
    }
  }
}

}  // namespace hjmc
