// hjmc_solve_impl.cuh — the fused Monte-Carlo Picard kernel (SURVEY §8(a) rows a1–a11).
//
// A group of threads — one warp, four warps or the whole CTA, chosen from N (launch_solve) —
// owns one work unit = (query m, horizon j) and runs the whole Picard loop of that horizon
// (Algorithm 1) without leaving the SM: queries and horizons are mutually
// independent (R5, R9), so no grid-wide synchronisation or inter-CTA traffic exists.
// Per Picard iterate (one Φ pass):
//   every thread walks a strided subset of the N samples; per sample it regenerates its
//   normals from Philox in registers (no sample array in memory), forms y = x + σz, evaluates
//   g, and accumulates w = 2^(A·core + B) and w·z (A = −c log2 e; B a guaranteed-safe shift,
//   hjmc_targets.cuh) — one FFMA + one MUFU.EX2 per weight, no per-sample max or rescale;
//   then a warp-shuffle butterfly and a shared-memory merge across the group's warps give the
//   unit's sums, and the group's thread 0 forms v, Dv and the next frozen coefficient
//   c = Γ(x, Dv) in double. For n = 37–48 pair-min targets a sample is spread over a lane
//   group instead (lg_pass), and under CRN a pass at an already-used c is not re-sampled
//   (HJMC_FLAG_REUSE_PASSES).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "hjmc_kernels.cuh"

namespace hjmc {

#ifndef HJMC_UNROLL
#define HJMC_UNROLL 2
#endif
#ifndef HJMC_LG_UNROLL
#define HJMC_LG_UNROLL 2
#endif
#ifndef HJMC_GROUP_UNROLL
#define HJMC_GROUP_UNROLL 2
#endif

namespace {

constexpr int kSampleUnroll = HJMC_UNROLL;
constexpr int kLgUnroll = HJMC_LG_UNROLL;
constexpr int kGroupUnroll = HJMC_GROUP_UNROLL;  // draw groups per trip when G > 1
constexpr double kLog2e = 1.4426950408889634074;
constexpr double kLn2 = 0.69314718055994530942;
// Two-pass fallback threshold, scaled with N. ex2.approx.ftz flushes every weight below 2^-126
// to 0, so a pass may drop up to N·2^-126 of weight mass; falling back whenever the shifted sum
// S < N·2^-102 keeps that loss below 2^-24 of S (one fp32 ulp) for every N (R24).
__device__ __forceinline__ double underflow_floor(uint32_t N) { return (double)N * 0x1p-102; }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Accumulate the weighted sums of one Φ pass over this thread's samples.
//   S += w,  Mz[d] += w ẑ_d,  w = 2^(A core(y) + B)
// Samples are walked in draw groups (R19, DrawLayout): a thread generates the group's normal
// stream (Q Philox blocks) and then runs its G samples; groups are strided over the CTA.
// kTilt (Laplace proposal, R28): the log2 weight gains the likelihood-ratio term sgn·(tz·ẑ).
// Speculative second weight (HJMC_FLAG_SPECULATE_CLAMPS): the same sample's sums at another
// frozen coefficient c' — w' = 2^(A'·core + B') — accumulated alongside (same core, same order).
template <int NDIM>
struct SpecSums {
  float A, B, S, Mz[NDIM];
};

template <class Tgt, int NDIM, bool kTilt, bool kSpec = false>
__device__ __forceinline__ void accumulate_sample(const Tgt& tgt, const float (&xs)[NDIM],
                                                  float sigma, float A, float B,
                                                  const float (&tz)[NDIM], const float* zg,
                                                  float sgn, float& S, float (&Mz)[NDIM],
                                                  SpecSums<NDIM>* sp = nullptr) {
  float z[NDIM];
#pragma unroll
  for (int d = 0; d < NDIM; ++d) z[d] = zg[d];
  const float core_v = tgt.core(xs, sgn * sigma, z);
  float a = fmaf(A, core_v, B);
  if constexpr (kSpec) {
    const float w2 = ex2_approx(fmaf(sp->A, core_v, sp->B));
    sp->S += w2;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) sp->Mz[d] = fmaf(w2, z[d], sp->Mz[d]);
  }
  if constexpr (kTilt) {
    float t = 0.f;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) t = fmaf(tz[d], z[d], t);
    a = fmaf(sgn, t, a);
  }
  const float w = ex2_approx(a);
  S += w;
  const float sw = sgn * w;
#pragma unroll
  for (int d = 0; d < NDIM; ++d) Mz[d] = fmaf(sw, z[d], Mz[d]);
}

// Polar variant for homogeneous targets (distances; Tgt::kHomog) with the plain proposal: the
// pass runs in σ-scaled coordinates — xs = x/σ', A = fl(A·σ') (the kernel undoes A/σ' in the
// epilogue) — so a coordinate is one FFMA x'_d + (±r̂)·trig_d from the polar draw and the
// moments take (±w·r̂)·trig_d, with no r̂·trig products ("σ-scaled coordinates").
template <class Tgt, int NDIM, bool kSpec = false>
__device__ __forceinline__ void accumulate_sample_polar(const Tgt& tgt, const float (&xs)[NDIM],
                                                        float A, float B, const float* tg,
                                                        const float* rg, float sgn, float& S,
                                                        float (&Mz)[NDIM],
                                                        SpecSums<NDIM>* sp = nullptr) {
  float t[NDIM], r[NDIM];
#pragma unroll
  for (int d = 0; d < NDIM; ++d) {
    t[d] = tg[d];
    r[d] = sgn * rg[d];
  }
  const float core_v = tgt.core_polar(xs, r, t);
  if constexpr (kSpec) {
    const float w2 = ex2_approx(fmaf(sp->A, core_v, sp->B));
    sp->S += w2;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) sp->Mz[d] = fmaf(w2 * rg[d], t[d], sp->Mz[d]);
  }
  const float w = ex2_approx(fmaf(A, core_v, B));
  S += w;
  const float sw = sgn * w;
#pragma unroll
  for (int d = 0; d < NDIM; ++d) Mz[d] = fmaf(sw * rg[d], t[d], Mz[d]);
}

// NT here is the size of the thread group that shares one unit (the CTA, or one warp in the
// warp-per-unit kernel) and tid the thread's index in it.
template <class Tgt, int NDIM, int NT, bool kTilt = false, bool kSpec = false>
__device__ __forceinline__ void mc_accumulate(const Tgt& tgt, const float (&xs)[NDIM],
                                                   float sigma, float A, float B, uint32_t N,
                                                   int antithetic, uint32_t w1base, uint32_t qid,
                                                   uint32_t tag, const RoundKeys& rk, float& S,
                                                   float (&Mz)[NDIM], const float (&tz)[NDIM],
                                                   uint32_t tid, SpecSums<NDIM>* sp = nullptr) {
  static_assert(!(kSpec && kTilt), "speculation only for the plain proposal");
  using L = DrawLayout<NDIM>;
  S = 0.f;
#pragma unroll
  for (int d = 0; d < NDIM; ++d) Mz[d] = 0.f;
  const uint32_t draws = antithetic ? (N >> 1) + (N & 1u) : N;
  const uint32_t groups = (draws + L::G - 1) / L::G;
  if constexpr (Tgt::kHomog && !kTilt) {  // σ-scaled polar pass (xs = x/σ', A = A·σ')
    const uint32_t full = antithetic ? 0u : N / L::G;
#pragma unroll(L::G == 1 ? kSampleUnroll : kGroupUnroll)
    for (uint32_t g = tid; g < full; g += NT) {
      float tt[L::L], rr[L::L];
      group_normals_polar<NDIM>(tt, rr, g, w1base, qid, tag, rk);
#pragma unroll
      for (int r = 0; r < L::G; ++r)
        accumulate_sample_polar<Tgt, NDIM, kSpec>(tgt, xs, A, B, tt + r * NDIM, rr + r * NDIM,
                                                  1.f, S, Mz, sp);
    }
    for (uint32_t g = full + tid; g < groups; g += NT) {  // ragged tail group / antithetic
      float tt[L::L], rr[L::L];
      group_normals_polar<NDIM>(tt, rr, g, w1base, qid, tag, rk);
#pragma unroll
      for (int r = 0; r < L::G; ++r) {
        const uint32_t q = g * L::G + r;
        if (antithetic) {
          if (L::G == 1 || q < draws) {
            accumulate_sample_polar<Tgt, NDIM>(tgt, xs, A, B, tt + r * NDIM, rr + r * NDIM, 1.f,
                                               S, Mz);
            if (2 * q + 1 < N)
              accumulate_sample_polar<Tgt, NDIM>(tgt, xs, A, B, tt + r * NDIM, rr + r * NDIM,
                                                 -1.f, S, Mz);
          }
        } else if (q < N) {
          accumulate_sample_polar<Tgt, NDIM, kSpec>(tgt, xs, A, B, tt + r * NDIM, rr + r * NDIM,
                                                    1.f, S, Mz, sp);
        }
      }
    }
    return;
  }
  if (!antithetic) {
    const uint32_t full = N / L::G;  // groups whose G samples all exist: no per-sample guard
#pragma unroll(L::G == 1 ? kSampleUnroll : kGroupUnroll)
    for (uint32_t g = tid; g < full; g += NT) {
      float zz[L::L];
      group_normals_hat<NDIM>(zz, g, w1base, qid, tag, rk);
#pragma unroll
      for (int r = 0; r < L::G; ++r)
        accumulate_sample<Tgt, NDIM, kTilt, kSpec>(tgt, xs, sigma, A, B, tz, zz + r * NDIM, 1.f, S,
                                                   Mz, sp);
    }
    for (uint32_t g = full + tid; g < groups; g += NT) {  // ragged tail group
      float zz[L::L];
      group_normals_hat<NDIM>(zz, g, w1base, qid, tag, rk);
#pragma unroll
      for (int r = 0; r < L::G; ++r)
        if (g * L::G + r < N)
          accumulate_sample<Tgt, NDIM, kTilt, kSpec>(tgt, xs, sigma, A, B, tz, zz + r * NDIM, 1.f,
                                                     S, Mz, sp);
    }
  } else {
    for (uint32_t g = tid; g < groups; g += NT) {
      float zz[L::L];
      group_normals_hat<NDIM>(zz, g, w1base, qid, tag, rk);
#pragma unroll
      for (int r = 0; r < L::G; ++r) {
        const uint32_t q = g * L::G + r;
        if (L::G == 1 || q < draws) {
          accumulate_sample<Tgt, NDIM, kTilt>(tgt, xs, sigma, A, B, tz, zz + r * NDIM, 1.f, S, Mz);
          if (2 * q + 1 < N)
            accumulate_sample<Tgt, NDIM, kTilt>(tgt, xs, sigma, A, B, tz, zz + r * NDIM, -1.f, S, Mz);
        }
      }
    }
  }
}

// Largest exponent A·core(y_i) over this thread's samples (fallback shift; rarely used).
// kPolar: the σ-scaled polar form of mc_accumulate (same core values as that pass).
template <class Tgt, int NDIM, int NT, bool kPolar = false>
__device__ float mc_max_exponent(const Tgt& tgt, const float (&xs)[NDIM], float sigma, float A,
                                 uint32_t N, int antithetic, uint32_t w1base, uint32_t qid,
                                 uint32_t tag, const RoundKeys& rk, const float (&tz)[NDIM],
                                 uint32_t tid) {
  using L = DrawLayout<NDIM>;
  float amax = -3.0e38f;
  const uint32_t draws = antithetic ? (N >> 1) + (N & 1u) : N;
  const uint32_t groups = (draws + L::G - 1) / L::G;
  if constexpr (kPolar) {
    for (uint32_t g = tid; g < groups; g += NT) {
      float tt[L::L], rr[L::L];
      group_normals_polar<NDIM>(tt, rr, g, w1base, qid, tag, rk);
#pragma unroll
      for (int r = 0; r < L::G; ++r) {
        const uint32_t q = g * L::G + r;
        if (q >= draws) continue;
        float t[NDIM], rp[NDIM], rn[NDIM];
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
          t[d] = tt[r * NDIM + d];
          rp[d] = rr[r * NDIM + d];
          rn[d] = -rp[d];
        }
        amax = fmaxf(amax, A * tgt.core_polar(xs, rp, t));
        if (antithetic && 2 * q + 1 < N) amax = fmaxf(amax, A * tgt.core_polar(xs, rn, t));
      }
    }
  } else {
    for (uint32_t g = tid; g < groups; g += NT) {
      float zz[L::L];
      group_normals_hat<NDIM>(zz, g, w1base, qid, tag, rk);
#pragma unroll
      for (int r = 0; r < L::G; ++r) {
        const uint32_t q = g * L::G + r;
        if (q >= draws) continue;
        float z[NDIM];
#pragma unroll
        for (int d = 0; d < NDIM; ++d) z[d] = zz[r * NDIM + d];
        float t = 0.f;  // tilt term (zero for the plain proposal)
#pragma unroll
        for (int d = 0; d < NDIM; ++d) t = fmaf(tz[d], z[d], t);
        amax = fmaxf(amax, fmaf(A, tgt.core(xs, sigma, z), t));
        if (antithetic && 2 * q + 1 < N) amax = fmaxf(amax, fmaf(A, tgt.core(xs, -sigma, z), -t));
      }
    }
  }
  return amax;
}

// Pass memo (HJMC_FLAG_REUSE_PASSES): under CRN a Φ pass of one (query, horizon) is a pure
// function of its frozen coefficient c (same samples, and A, B, the proposal centre and the
// fallback shift all follow from c), so a pass at a c already seen by this unit returns the
// stored CTA sums instead of re-sampling. The C2 trajectories cycle between the two clamps
// (e.g. c_min, c_max, c_min, …; R8), which the stationary skip alone cannot shortcut.
constexpr int kMemo = 8;

template <int NDIM, int NT>
struct SolveSmem {
  float part[NT / 32][NDIM + 1];
  double sum[NDIM + 1];
  double sum2[NDIM + 1];  // speculative pass sums (HJMC_FLAG_SPECULATE_CLAMPS)
  double memo_sum[kMemo][NDIM + 1];
  double memo_c[kMemo];
  float memo_B[kMemo];
  int n_memo;
  float xs[NDIM];   // lane-group kernel: x (+ bτ) staged once; thread 0 derives the pass shift
  float lg_B, lg_B2;
  double dg[NDIM];  // Dg(x + bτ) for the Laplace proposal (R28)
  float fmax_part[NT / 32];
  double c_next;
  float shift;
};

// Barrier over the GS threads that share a unit in a CTA of CTA threads: the CTA barrier, the
// warp, or named barrier 1 + group index (bar.sync id, GS).
template <int GS, int CTA>
__device__ __forceinline__ void group_sync() {
  if constexpr (GS == CTA) __syncthreads();
  else if constexpr (GS == 32) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / GS)), "r"(GS) : "memory");
}

// Group-wide merge of (S, Mz[NDIM]) into sm.sum (double), deterministic order. NT = group
// size: the CTA or a part of it (shared-memory merge across its warps) or one warp (shuffles).
template <int NDIM, int NT, int CTA = NT>
__device__ __forceinline__ void cta_reduce(SolveSmem<NDIM, NT>& sm, float S, float (&Mz)[NDIM],
                                           uint32_t tid, double* dst = nullptr) {
  double* out = dst ? dst : sm.sum;
  const int lane = tid & 31, warp = tid >> 5;
  S = warp_sum(S);
#pragma unroll
  for (int d = 0; d < NDIM; ++d) Mz[d] = warp_sum(Mz[d]);
  if constexpr (NT == 32) {
    if (lane == 0) {
      out[0] = (double)S;
#pragma unroll
      for (int d = 0; d < NDIM; ++d) out[1 + d] = (double)Mz[d];
    }
    __syncwarp();
    return;
  }
  if (lane == 0) {
    sm.part[warp][0] = S;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) sm.part[warp][1 + d] = Mz[d];
  }
  group_sync<NT, CTA>();
  for (int col = tid; col < NDIM + 1; col += NT) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) acc += (double)sm.part[w][col];
    out[col] = acc;
  }
  group_sync<NT, CTA>();
}

// ---- lane-group layout for the K-pair union at n = 39..48 (C5: n = 45) -----------------------
// One sample is spread over 4 consecutive lanes; lane ℓ owns coordinates [12ℓ, 12ℓ + 12): its
// Philox blocks b = 3ℓ..3ℓ+2 (12 = lcm(3, 4), so neither a block nor a (x, y) pair straddles
// lanes), its pairs' partial min of |pos|², and its 12 moment accumulators. Two shuffles give
// the group min, every lane forms the same weight, lane ℓ = 0's S is the one reduced. A lane
// keeps 12 + 12 + 12 live floats instead of 45 + 45 + 45, so 4 CTAs fit per SM (255 → ≤ 64
// registers). Same samples, same counters, same arithmetic as the generic path.
// Targets whose core is a min over (x, y) pairs of 3-coordinate blocks: the K-pair union and the
// paper's pursuit-min, where every lane also needs the evader's sampled position — it
// lives in one lane and reaches the others by two shuffles.
#ifndef HJMC_NO_LANE_GROUPS
#define HJMC_NO_LANE_GROUPS 0   // build variant: the per-thread layout at n = 37–48 too
#endif
template <class Tgt, int NDIM>
struct UseLaneGroups {
  static constexpr bool kPursuit = std::is_same<Tgt, PursuitMin<NDIM>>::value;
  static constexpr bool value =
      (std::is_same<Tgt, PairUnion<NDIM>>::value || kPursuit) && NDIM >= 37 && NDIM <= 48 &&
      !HJMC_NO_LANE_GROUPS;
};

#ifndef HJMC_LG_LANES
#define HJMC_LG_LANES 4
#endif
// Lanes per sample (4 or 2) and what each lane owns: kLgSpan = 48 / lanes coordinates
// (a multiple of lcm(3, 4) = 12), i.e. kLgSpan / 4 Philox blocks and kLgSpan / 3 (x, y, θ) pairs.
constexpr int kLgLanes = HJMC_LG_LANES;
#ifndef HJMC_LG_DUAL
#define HJMC_LG_DUAL 1
#endif
#ifndef HJMC_LG_DUAL_UNROLL
#define HJMC_LG_DUAL_UNROLL 2
#endif
constexpr bool kLgDual = HJMC_LG_DUAL != 0;  // two samples per lane-group trip (lg_pass)
constexpr int kLgDualUnroll = HJMC_LG_DUAL_UNROLL;
#ifndef HJMC_LG_CHAIN
#define HJMC_LG_CHAIN 1
#endif
#ifndef HJMC_LG_CHAIN_AT
#define HJMC_LG_CHAIN_AT 0
#endif

constexpr int kLgSpan = 48 / kLgLanes;
static_assert(kLgLanes == 2 || kLgLanes == 4, "lane groups of 2 or 4");

// Speculative sums of the lane-group pass (HJMC_FLAG_SPECULATE_CLAMPS): the same samples at a
// second coefficient, weight 2^(A·core + B).
struct LgSpec {
  float A, B, S, S1, Mb[kLgSpan];
};

// σ-scaled coordinates (round 2). The pass works on y/σ' (σ' = σC, the transform scale):
// x' = x/σ' once per unit, so a sample coordinate is x' + ẑ = x' + rh·trig — ONE FFMA from the
// polar Box–Muller output (rh, cos, sin), with no rh·trig product; the moments take the pair's
// w·rh (one FMUL per pair instead of one per coordinate). The pair-union core is homogeneous,
// core(y) = σ'·core(y/σ'), so the caller passes A' = fl(A·σ') and the epilogue undoes A'/σ'
// (kernel: A_eff). Per lane and sample this removes 6 FP32 multiplies of ~210 instructions.
// x' carries one extra rounding, |x|·2^-24 absolute in position (the unscaled fma rounds once
// at |y|), far inside R20. Coordinates past n get x' = 1e18 (a sentinel whose |pos|² = 2e36
// never wins the min), so the pair-union partial min needs no per-lane guard.
template <int NDIM, int NT, bool kMaxMode, bool kPursuit = false, bool kSpec = false>
__device__ __forceinline__ void lg_pass(const SolveParams& P, int64_t m, float tau, float sigma_s,
                                        float A, float B, uint32_t w1base, uint32_t qid,
                                        float& S, float (&Mb)[kLgSpan], float& amax,
                                        LgSpec* sp = nullptr) {
  constexpr int kBlocks = kLgSpan / 4, kTriples = kLgSpan / 3, kPairs = kLgSpan / 2;
  const int lane = threadIdx.x & 31, l = lane & (kLgLanes - 1);
  const uint32_t slot = (threadIdx.x >> 5) * (32 / kLgLanes) + (lane / kLgLanes);  // sample slot
  constexpr uint32_t kStride = NT / kLgLanes;
  float xb[kLgSpan];  // x' = x / σ'
#pragma unroll
  for (int c = 0; c < kLgSpan; ++c) {
    const int d = kLgSpan * l + c;
    float xv = kPursuit ? 0.f : 1.0e18f;
    if (d < NDIM) {
      xv = P.x[m * NDIM + d];
      if (P.drift) xv = __fadd_rn(xv, __fmul_rn(P.drift[m * NDIM + d], tau));
      xv = __fdiv_rn(xv, sigma_s);
    }
    xb[c] = xv;
  }
  S = 0.f;
  amax = -3.0e38f;
#pragma unroll
  for (int c = 0; c < kLgSpan; ++c) Mb[c] = 0.f;
  const uint32_t N = P.N;
  // this lane's share of sample i in polar form: ẑ_c = r[c/2]·t[c] (its Philox blocks
  // kBlocks·l .. kBlocks·l + kBlocks − 1; pair p = normals 2p, 2p + 1)
  struct Draw {
    float t[kLgSpan], r[kPairs];
  };
  auto draw = [&](uint32_t i, Draw& z) {
#pragma unroll
    for (int qd = 0; qd < kBlocks; ++qd) {
      const uint4 w = philox4x32_10(i, w1base | (uint32_t)(kBlocks * l + qd), qid, P.tag, P.rk);
      box_muller_polar(w.x, w.y, z.r[2 * qd], z.t[4 * qd], z.t[4 * qd + 1]);
      box_muller_polar(w.z, w.w, z.r[2 * qd + 1], z.t[4 * qd + 2], z.t[4 * qd + 3]);
    }
  };
  const uint32_t rzero = (uint32_t)(P.M >> 62);  // a runtime zero (M < 2^62)
  auto coord = [&](const Draw& z, int c) { return fmaf(z.r[c / 2], z.t[c], xb[c]); };

  // min over this lane's (x, y) pairs of |pos'|² (pursuit: |pursuer − evader|²), pos' = y/σ'
  auto partial_min = [&](const Draw& z) -> float {
    float best = 3.0e38f;
    if constexpr (kPursuit) {
      // the evader (last agent, coordinates kE, kE + 1) is owned by lane kE / kLgSpan
      constexpr int kE = NDIM - 3, kLaneE = kE / kLgSpan, kCE = kE % kLgSpan;
      const int src = (lane & ~(kLgLanes - 1)) | kLaneE;
      const float ex = __shfl_sync(0xffffffffu, coord(z, kCE), src);
      const float ey = __shfl_sync(0xffffffffu, coord(z, kCE + 1), src);
#pragma unroll
      for (int pq = 0; pq < kTriples; ++pq) {
        const float a = coord(z, 3 * pq) - ex;
        const float b = coord(z, 3 * pq + 1) - ey;
        const float r2 = fmaf(a, a, b * b);
        best = (kLgSpan * l + 3 * pq < kE) ? fminf(best, r2) : best;   // pursuers only
      }
    } else {
#pragma unroll
      for (int pq = 0; pq < kTriples; ++pq) {
        const float a = coord(z, 3 * pq);
        const float b = coord(z, 3 * pq + 1);
        best = fminf(best, fmaf(a, a, b * b));  // coordinates past n: the 1e18 sentinel
      }
    }
    return best;
  };
  // Mb[c] += w·ẑ_c as (w·rh_p)·trig_c
  auto moments = [&](float (&acc)[kLgSpan], float w, const Draw& z) {
#pragma unroll
    for (int p = 0; p < kPairs; ++p) {
      const float wr = w * z.r[p];
      acc[2 * p] = fmaf(wr, z.t[2 * p], acc[2 * p]);
      acc[2 * p + 1] = fmaf(wr, z.t[2 * p + 1], acc[2 * p + 1]);
    }
  };
  // One sample per lane group per trip; trips where every slot's sample exists run without
  // the i < N guard (C5: N = 2^20, all of them), the ragged last trip with it.
  // The weight sum is split by trip parity into two fp32 accumulators (S for even trips, S1 for
  // odd ones, added at the end): a lane group sums N/64 = 16,384 weights per pass at C5, and at
  // c = c_min (weights ≈ 1) one accumulator's rounding walk reaches ~5e-6 relative, which
  // v = −log(S/N)/c amplifies by 1/c = 20 (R20 allows 5e-5 absolute near v = 0). Two halves cut
  // that by 2√2 at no cost in the loop; every path (one- or two-sample trips, speculative sums)
  // uses the same split, so a speculative pass still equals a real one bit for bit.
  float S1 = 0.f;
  auto trip = [&](uint32_t i, bool guard, bool odd) {
    Draw z;
    draw(i, z);
    float best = partial_min(z);
#pragma unroll
    for (int o = 1; o < kLgLanes; o <<= 1) best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
    const float core = sqrt_approx(best);
    if (!guard || i < N) {
      if (kMaxMode) {
        amax = fmaxf(amax, A * core);
      } else {
        const float wt = ex2_approx(fmaf(A, core, B));
        if (odd) S1 += wt;
        else S += wt;
        moments(Mb, wt, z);
        if constexpr (kSpec) {
          const float w2 = ex2_approx(fmaf(sp->A, core, sp->B));
          if (odd) sp->S1 += w2;
          else sp->S += w2;
          moments(sp->Mb, w2, z);
        }
      }
    }
  };
  const uint32_t full = N / kStride;
  uint32_t t0 = 0;
  if constexpr (kLgDual && kLgLanes == 4 && !kMaxMode && !kSpec) {
    // Two samples in flight per trip (trips t, t + 1 of the slot): their 24 Philox blocks are
    // independent instruction streams the scheduler interleaves, and the weight work is split
    // across the group — lanes 0–1 form sample t's weight, lanes 2–3 sample t + 1's, one
    // shuffle swaps them — so each lane runs one SQRT + EX2 per two samples instead of two.
    // The min is exact and each weight is formed from the same fp32 values by the same MUFU
    // ops, and S, Mb accumulate w_t then w_{t+1} as the one-sample loop does: bit-identical.
    const bool lo = l < 2;
#pragma unroll(kLgDualUnroll)
    for (; t0 + 1 < full; t0 += 2) {
      Draw z0, z1;
      draw(t0 * kStride + slot, z0);
      // a pure scheduling tie: sample t + 1's counter is XORed with (one of sample t's Box–Muller
      // radii AND a runtime zero), so ptxas starts t + 1's Philox chains after that point and
      // interleaves them with t's MUFU work instead of front-loading all 24 blocks' integer
      // work (values unchanged; with the loop unrolled ×2: 4379 → 4330 ms on the C5 queries)
      uint32_t i1 = (t0 + 1) * kStride + slot;
      if (HJMC_LG_CHAIN) i1 ^= __float_as_uint(z0.r[HJMC_LG_CHAIN_AT]) & rzero;
      draw(i1, z1);
      const float b0 = partial_min(z0), b1 = partial_min(z1);
      float mine = lo ? b0 : b1;
      const float other = lo ? b1 : b0;
      mine = fminf(mine, __shfl_xor_sync(0xffffffffu, other, 2));  // partner's part of my sample
      mine = fminf(mine, __shfl_xor_sync(0xffffffffu, mine, 1));   // lanes l, l^1: same sample
      const float wm = ex2_approx(fmaf(A, sqrt_approx(mine), B));
      const float wo = __shfl_xor_sync(0xffffffffu, wm, 2);
      const float w0 = lo ? wm : wo, w1 = lo ? wo : wm;
      S += w0;                                                     // t0 even
      moments(Mb, w0, z0);
      S1 += w1;                                                    // t0 + 1 odd
      moments(Mb, w1, z1);
    }
  }
#pragma unroll(kLgUnroll)
  for (uint32_t t = t0; t < full; ++t) trip(t * kStride + slot, false, t & 1u);
  if (full * kStride < N) trip(full * kStride + slot, true, full & 1u);
  S += S1;
  if constexpr (kSpec) sp->S += sp->S1;
}

// Merge the lane-group sums into sm.sum (double), deterministic order.
template <int NDIM, int NT>
__device__ __forceinline__ void lg_reduce(SolveSmem<NDIM, NT>& sm, float S, float (&Mb)[kLgSpan],
                                          double* dst = nullptr) {
  double* out = dst ? dst : sm.sum;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, l = lane & (kLgLanes - 1);
#pragma unroll
  for (int o = kLgLanes; o < 32; o <<= 1) {      // sum over the warp's lane groups
    S += __shfl_xor_sync(0xffffffffu, S, o);
#pragma unroll
    for (int c = 0; c < kLgSpan; ++c) Mb[c] += __shfl_xor_sync(0xffffffffu, Mb[c], o);
  }
  if (lane < kLgLanes) {
    if (l == 0) sm.part[warp][0] = S;
#pragma unroll
    for (int c = 0; c < kLgSpan; ++c)
      if (kLgSpan * l + c < NDIM) sm.part[warp][1 + kLgSpan * l + c] = Mb[c];
  }
  __syncthreads();
  for (int col = threadIdx.x; col < NDIM + 1; col += NT) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) acc += (double)sm.part[w][col];
    out[col] = acc;
  }
  __syncthreads();
}

// Thread 0's per-iterate epilogue (a9–a10), double precision: v and Dv from the CTA sums,
// outputs, and the next frozen coefficient Γ(x, Dv) (returned; solve mode only).
// Exact-stationarity skip (HJMC_FLAG_SKIP_STATIONARY, needs CRN): when Γ returns the same c,
// the next pass has bit-identical inputs (same samples, same c), hence bit-identical outputs;
// the remaining iterates are copied instead of recomputed and *done is set.
// dshift (Laplace proposal only, else null): (μ − x)/σ of the pass; the likelihood ratio
// contributes −|μ − x|²/(2σ²) to the log-mean and (μ − x)/σ to E_W[(y − x)/σ] (R28).
template <class Tgt, int NDIM>
__device__ __noinline__ double pass_epilogue(const SolveParams& P, const Tgt& tgt, int64_t m, int j,
                                             int k, uint32_t id, double c, double sigma_d,
                                             double A, float B, float core_ref, const double* sum,
                                             const double* dshift, bool* done) {
  const double A_d = -c * kLog2e;
  const double Ssum = sum[0];
  double tilt_log2 = 0.0;
  if (dshift)
    for (int d = 0; d < NDIM; ++d) tilt_log2 -= 0.5 * dshift[d] * dshift[d] * kLog2e;
  // log2 of (1/N) Σ exp(−c g_i)·LR_i: undo the shift B and the fp32 rounding of A
  const double log2mean = log2(Ssum) - log2((double)P.N) - (double)B + A_d * (double)tgt.off +
                          (A_d - A) * (double)core_ref + tilt_log2;
  const double v = -(kLn2 / c) * log2mean;                           // Cor. logsumexp
  double dv[NDIM];
  bool finite = isfinite(v);
  for (int d = 0; d < NDIM; ++d) {
    // Cor. mc_gradient; the sums hold ẑ = z/C (hjmc_rng.cuh), so E_w[z] = C·M̂/S
    dv[d] = -((double)kBMScale * sum[1 + d] / Ssum + (dshift ? dshift[d] : 0.0)) / (c * sigma_d);
    finite = finite && isfinite(dv[d]);
  }
  if (!finite && P.err) {
    atomicOr(P.err, 1);
    atomicMin(P.bad, (unsigned long long)id);
  }
  const bool last = (k == P.Kp - 1);
  if (P.mode == kModePass) {  // stepwise Picard: [K][M] outputs, state update
    const size_t o = (size_t)(j - 1) * (size_t)P.M + (size_t)m;
    if (P.v) P.v[o] = (float)v;
    if (P.dv)
      for (int d = 0; d < NDIM; ++d) P.dv[o * NDIM + d] = (float)dv[d];
    double xd[NDIM];
    for (int d = 0; d < NDIM; ++d) xd[d] = (double)P.x[m * NDIM + d];
    const double c_next = gamma_update(P.sp, P.gp, xd, dv);
    P.c_state[o] = c_next;
    if (P.c_out) P.c_out[o] = (float)c_next;
    *done = true;
    return c_next;
  }
  if (P.mode != kModeSolve) {
    if (P.v) P.v[m] = (float)v;
    if (P.dv)
      for (int d = 0; d < NDIM; ++d) P.dv[m * NDIM + d] = (float)dv[d];
    return c;
  }
  const size_t hi = ((size_t)(j - 1) * (size_t)P.Kp + (size_t)k) * (size_t)P.M + (size_t)m;
  if (P.vhist) P.vhist[hi] = (float)v;
  if (P.chist) P.chist[hi] = (float)c;
  double xd[NDIM];
  for (int d = 0; d < NDIM; ++d) xd[d] = (double)P.x[m * NDIM + d];
  const double c_next = gamma_update(P.sp, P.gp, xd, dv);           // Γ; dv → p̃
  const bool stationary = P.skip_stationary && P.crn && !last && c_next == c;
  if (stationary) {
    for (int kk = k + 1; kk < P.Kp; ++kk) {
      const size_t h2 = ((size_t)(j - 1) * (size_t)P.Kp + (size_t)kk) * (size_t)P.M + (size_t)m;
      if (P.vhist) P.vhist[h2] = (float)v;
      if (P.chist) P.chist[h2] = (float)c;
    }
  }
  *done = last || stationary;
  if (last || stationary) {
    if (P.vfinal) P.vfinal[(size_t)(j - 1) * (size_t)P.M + (size_t)m] = (float)v;
    if (j == P.K) {
      if (P.v) P.v[m] = (float)v;
      if (P.dv)
        for (int d = 0; d < NDIM; ++d)
          P.dv[m * NDIM + d] = (float)(-((double)kBMScale * sum[1 + d] / Ssum +
                                         (dshift ? dshift[d] : 0.0)) / (c * sigma_d));
      if (P.c_out) P.c_out[m] = (float)c_next;
    }
  }
  return c_next;
}

// Thread 0's prologue: g(x) output, τ = 0 point-mass case, and c^(0) = Γ(x, Dg(x))
// (Algorithm 1 init) or the caller's frozen c (value_grad). Returns c (0 when
// the unit is complete because σ = 0; the caller flags that case).
template <class Tgt, int NDIM>
__device__ __noinline__ double unit_prologue(const SolveParams& P, const Tgt& tgt, int64_t m, int j,
                                             double sigma_d, const float* xs, double* dg_out) {
  double xd[NDIM], p[NDIM];
  if (P.proposal) {
    for (int d = 0; d < NDIM; ++d) xd[d] = (double)xs[d];
    tgt.dg(xd, dg_out);
  }
  for (int d = 0; d < NDIM; ++d) xd[d] = (double)P.x[m * NDIM + d];
  if (P.mode == kModeSolve && j == 1 && P.g0) P.g0[m] = (float)tgt.g_host(xd);
  if (sigma_d == 0.0) {  // τ = 0: point mass, v = g(x), Dv = Dg(x)
    for (int d = 0; d < NDIM; ++d) xd[d] = (double)xs[d];
    if (P.v) P.v[m] = (float)tgt.g_host(xd);
    tgt.dg(xd, p);
    if (P.dv)
      for (int d = 0; d < NDIM; ++d) P.dv[m * NDIM + d] = (float)p[d];
    return 0.0;
  }
  if (P.mode == kModePass) return P.c_state[(size_t)(j - 1) * (size_t)P.M + (size_t)m];
  if (P.mode != kModeSolve) return (double)P.c_in[m];
  tgt.dg(xd, p);
  return gamma_update(P.sp, P.gp, xd, p);
}

#ifndef HJMC_NT
#define HJMC_NT 256
#endif
// Resident CTAs per SM requested from ptxas (caps registers: 4 → 64, 3 → 80 at 256 threads).
// Measured on B200: C2 (n = 3) 4/SM beats 3/SM by 2% and 1/SM by 7%. C4 (n = 15): with the
// proposal compiled out of the plain kernel (kProp) 3/SM (80 regs, no spill) runs 2% faster
// than 4/SM (64 regs, spill loads in the sample loop) and 4.7% faster than 2/SM. Above n = 16
// the generic path needs z[n] and the moments in registers (1/SM).
#ifndef HJMC_MINB
#define HJMC_MINB 0
#endif
template <int NDIM, bool kLG, bool kSpec = false>
#ifndef HJMC_LG_SPEC_MINB
#define HJMC_LG_SPEC_MINB 2
#endif
constexpr int min_blocks() {
  if (HJMC_MINB > 0) return HJMC_MINB;
  // + 12 speculative moments per lane; with the σ-scaled pass (polar draws, 18 live floats per
  // sample) 2 CTAs/SM beat 3 (C5 fastpath 479 vs 502 ms; 3 CTAs spill inside the loop)
  if (kLG && kSpec) return kLgLanes == 4 ? HJMC_LG_SPEC_MINB : 2;
  // two samples in flight (kLgDual) need 128 registers: 2 CTAs/SM, measured 1.9 % faster on C5
  // than one sample at 4 CTAs/SM; 2-lane groups hold 24 + 24 + 16 floats
  if (kLG) return (kLgLanes == 4 && !kLgDual) ? 4 : 2;
  if (kSpec && NDIM > 6) return 2;                 // + n + 1 speculative sums (n ≤ 16)
  return NDIM <= 6 ? 4 : (NDIM <= 16 ? 3 : 1);
}

// kLG: the lane-group instantiation (non-antithetic passes of UseLaneGroups targets); it does
// not contain the generic per-thread path, so its register budget is the lane layout's.
// kProp: the Laplace-tilted proposal (R28) is compiled into its own instantiation, so the plain
// kernels carry no proposal centre / tilt arrays (register pressure at n = 15).
// GS: threads per unit — the whole CTA (GS = NT), or one warp (GS = 32: the warp-per-unit
// kernel for small N, where a CTA-wide unit would spend most of its time in the per-pass
// reduction, barriers and thread-0 epilogue; with one unit per warp those latencies of one
// unit overlap the sampling of the CTA's other seven, and no __syncthreads exists).
// kSpec (HJMC_FLAG_SPECULATE_CLAMPS, plain passes, n ≤ 6): while sampling at c, also
// accumulate the sums at the opposite clamp (c_max ↔ c_min) and memoize them, so a Picard
// 2-cycle between the clamps costs one sampling pass instead of two.
template <class Tgt, int NDIM, int NT, bool kLG = false, bool kProp = false, int GS = NT,
          bool kSpec = false>
__global__ void __launch_bounds__(NT, min_blocks<NDIM, kLG, kSpec>()) solve_kernel(const __grid_constant__ SolveParams P) {
  static_assert(GS == NT || (!kLG && GS >= 32 && NT % GS == 0 && GS % 32 == 0),
                "thread groups smaller than the CTA only for the generic kernel");
  __shared__ SolveSmem<NDIM, GS> smv[NT / GS];
  SolveSmem<NDIM, GS>& sm = smv[threadIdx.x / GS];
  constexpr bool kPolarG = !kLG && Tgt::kHomog && !kProp;  // σ-scaled generic passes
  const uint32_t tid = threadIdx.x % GS;
  auto gsync = [] { group_sync<GS, NT>(); };
  const int64_t unit = (int64_t)blockIdx.x * (NT / GS) + threadIdx.x / GS;
  if constexpr (GS != NT) {
    const int64_t units = (P.mode == kModeSolve)  ? P.M * (int64_t)P.K
                          : (P.mode == kModePass) ? P.M * (int64_t)P.n_active
                                                  : P.M;
    if (unit >= units) return;  // whole warp: the last CTA's spare warps
  }
  int64_t m;
  int j;
  if (P.mode == kModeSolve) {
    m = unit / P.K;
    j = (int)(unit % P.K) + 1;
  } else if (P.mode == kModePass) {
    m = unit / P.n_active;
    j = P.active_j[unit % P.n_active];
    if (P.active_mask && !P.active_mask[j - 1]) return;  // retired horizon (whole group)
  } else {
    m = unit;
    j = 1;
  }
  const Tgt tgt(P.tp);

  // a1: query staging (uniform across the CTA; served from L1 after the first warp)
  const uint32_t id = P.qid ? P.qid[m] : P.qid_base + (uint32_t)m;
  const double tau = (P.mode != kModeValueGrad) ? (double)j * P.T / (double)P.K : P.tau_vg;
  const double sigma_d = sqrt(P.gp.delta_eff * tau);
  const float sigma = (float)sigma_d;
  const float sigma_s = opaque((float)(sigma_d * (double)kBMScale));  // y = x + σz = x + (σC)ẑ
  // generic kernel: every thread keeps x in registers (the sample loop reads it); lane-group
  // kernel: each lane loads its own 12 coordinates inside lg_pass, so x is staged once in
  // shared memory for thread 0's per-pass shift and epilogue (no 3 × n register arrays to spill)
  float xs[kLG ? 1 : NDIM];
  if constexpr (kLG) {
    for (int d = threadIdx.x; d < NDIM; d += NT) {
      const float xv = P.x[m * NDIM + d];
      sm.xs[d] = P.drift ? __fadd_rn(xv, __fmul_rn(P.drift[m * NDIM + d], (float)tau)) : xv;
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int d = 0; d < NDIM; ++d) {
      const float xv = P.x[m * NDIM + d];
      xs[d] = P.drift ? __fadd_rn(xv, __fmul_rn(P.drift[m * NDIM + d], (float)tau)) : xv;
    }
  }

  if (tid == 0) {
    sm.c_next = unit_prologue<Tgt, NDIM>(P, tgt, m, j, sigma_d, kLG ? sm.xs : xs, sm.dg);
    sm.shift = (sigma_d == 0.0) ? 1.f : 0.f;
    sm.n_memo = 0;
  }
  gsync();
  double c = sm.c_next;
  if (sm.shift != 0.f) return;  // σ = 0: handled by the prologue (uniform branch)
  gsync();

  const uint32_t jw = (P.mode != kModeValueGrad) ? (uint32_t)j : P.jtag;
  unsigned passes = 0;  // Φ passes this unit executed (thread 0)
  const bool memo_on = P.reuse_passes && P.crn && P.mode == kModeSolve;

  for (int k = 0; k < P.Kp; ++k) {
    const uint32_t kw = (P.mode == kModeSolve)  ? (P.crn ? 0u : (uint32_t)k)
                        : (P.mode == kModePass) ? (P.crn ? 0u
                                                   : (uint32_t)(P.kiter_dev ? *P.kiter_dev
                                                                            : P.kiter))
                                                : P.ktag;
    const uint32_t w1base = (kw << 8) | (jw << 16);
    const float A = opaque((float)(-c * kLog2e));
    // lane-group passes and the generic passes of homogeneous targets with the plain proposal
    // run in σ-scaled coordinates (lg_pass, accumulate_sample_polar): A' = fl(A·σ'), and the
    // epilogue takes the effective A'/σ' in place of A
    constexpr bool kScaled = kLG || kPolarG;
    const float A_lg = kScaled ? opaque(A * sigma_s) : A;
    const double A_eff = kScaled ? (double)A_lg / (double)sigma_s : (double)A;
    // Proposal centre (R28): plain → x + bτ; Laplace → μ = x + bτ − cσ²·Dg(x + bτ) (fp32, every
    // thread computes the same values in double); tz = log2-domain tilt per ẑ coordinate.
    // The lane-group kernel (plain proposal only) has thread 0 derive B and core_ref from the
    // staged x and broadcast B.
    float ctr[kLG ? 1 : NDIM], tz[kLG ? 1 : NDIM];
    float core_ref = 0.f, B;
    if constexpr (kLG) {
      if (tid == 0) {
        float z0[NDIM];
#pragma unroll
        for (int d = 0; d < NDIM; ++d) z0[d] = 0.f;
        core_ref = tgt.core(sm.xs, 0.f, z0);
        sm.lg_B = -A * tgt.core_lower(sm.xs, sigma);   // every a_i = A core_i + B ≤ 0
      }
      __syncthreads();
      B = opaque(sm.lg_B);
    } else {
      float tilt_max = 0.f;
#pragma unroll
      for (int d = 0; d < NDIM; ++d) {
        ctr[d] = xs[d];
        tz[d] = 0.f;
      }
      if constexpr (kProp) {
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
          ctr[d] = (float)((double)xs[d] - c * sigma_d * sigma_d * sm.dg[d]);
          const double dsh = ((double)ctr[d] - (double)xs[d]) / sigma_d;
          tz[d] = opaque((float)(-kLog2e * (double)kBMScale * dsh));
          tilt_max += fabsf(tz[d]);
        }
        tilt_max *= kZmax / kBMScale;  // |ẑ_d| ≤ kZmax / C
      }
      {
        float z0[NDIM];
#pragma unroll
        for (int d = 0; d < NDIM; ++d) z0[d] = 0.f;
        core_ref = tgt.core(ctr, 0.f, z0);
      }
      // every a_i = A core_i + B (+ tilt) ≤ 0: no weight can overflow
      B = opaque(-A * tgt.core_lower(ctr, sigma) - tilt_max);
      if constexpr (kPolarG) {
#pragma unroll
        for (int d = 0; d < NDIM; ++d) ctr[d] = __fdiv_rn(ctr[d], sigma_s);  // x' = x/σ'
      }
    }

    int hit = -1;  // CTA-uniform: every thread reads the same memo after the last barrier
    if (memo_on)
      for (int e = 0; e < sm.n_memo; ++e)
        if (sm.memo_c[e] == c) {
          hit = e;
          break;
        }
    // speculation target: the opposite clamp, if not memoized yet and the memo has room for both
    double c_spec = 0.0;
    float B_spec = 0.f;
    bool do_spec = false;
    if constexpr (kSpec) {
      if (memo_on && hit < 0) {
        c_spec = (c == P.gp.c_max) ? P.gp.c_min : ((c == P.gp.c_min) ? P.gp.c_max : 0.0);
        do_spec = c_spec != 0.0 && sm.n_memo + 2 <= kMemo;
        for (int e = 0; e < sm.n_memo; ++e)
          if (sm.memo_c[e] == c_spec) do_spec = false;
      }
    }
    if (hit < 0) {
      if constexpr (kLG) {
        float S, Mb[kLgSpan], amax;
        bool plain_lg = true;
        if constexpr (kSpec) {
          if (do_spec) {
            LgSpec sp;
            const float A_spec = opaque((float)(-c_spec * kLog2e));
            sp.A = opaque(A_spec * sigma_s);  // exactly the A' a pass at c_spec would use
            if (tid == 0) sm.lg_B2 = -A_spec * tgt.core_lower(sm.xs, sigma);  // as a pass at c_spec
            __syncthreads();
            sp.B = opaque(sm.lg_B2);
            sp.S = 0.f;
            sp.S1 = 0.f;
#pragma unroll
            for (int c2 = 0; c2 < kLgSpan; ++c2) sp.Mb[c2] = 0.f;
            lg_pass<NDIM, NT, false, UseLaneGroups<Tgt, NDIM>::kPursuit, true>(
                P, m, (float)tau, sigma_s, A_lg, B, w1base, id, S, Mb, amax, &sp);
            lg_reduce<NDIM, NT>(sm, S, Mb);
            lg_reduce<NDIM, NT>(sm, sp.S, sp.Mb, sm.sum2);
            B_spec = sp.B;
            plain_lg = false;
          }
        }
        if (plain_lg) {
          lg_pass<NDIM, NT, false, UseLaneGroups<Tgt, NDIM>::kPursuit>(P, m, (float)tau, sigma_s,
                                                                       A_lg, B, w1base, id, S, Mb,
                                                                       amax);
          lg_reduce<NDIM, NT>(sm, S, Mb);
        }
      } else {
        float S, Mz[NDIM];
        bool plain = true;
        if constexpr (kSpec) {
          if (do_spec) {
            // exactly the A and B a pass at c_spec would use (tilt 0: plain proposal)
            SpecSums<NDIM> sp;
            const float A_spec = opaque((float)(-c_spec * kLog2e));
            sp.A = kPolarG ? opaque(A_spec * sigma_s) : A_spec;  // as a pass at c_spec
            sp.B = opaque(-A_spec * tgt.core_lower(xs, sigma) - 0.f);  // plain: centre = x
            sp.S = 0.f;
#pragma unroll
            for (int d = 0; d < NDIM; ++d) sp.Mz[d] = 0.f;
            mc_accumulate<Tgt, NDIM, GS, false, true>(tgt, ctr, sigma_s, A_lg, B, P.N, 0, w1base, id,
                                                      P.tag, P.rk, S, Mz, tz, tid, &sp);
            cta_reduce<NDIM, GS, NT>(sm, S, Mz, tid);
            cta_reduce<NDIM, GS, NT>(sm, sp.S, sp.Mz, tid, sm.sum2);
            B_spec = sp.B;
            plain = false;
          }
        }
        if (plain) {
          mc_accumulate<Tgt, NDIM, GS, kProp>(tgt, ctr, sigma_s, A_lg, B, P.N, P.antithetic, w1base,
                                              id, P.tag, P.rk, S, Mz, tz, tid);
          cta_reduce<NDIM, GS, NT>(sm, S, Mz, tid);
        }
      }
      if (!(sm.sum[0] >= underflow_floor(P.N))) {
        // The bound-based shift left every weight tiny (or g was non-finite): redo the pass with
        // the exact maximum exponent, the plain two-pass log-sum-exp.
        float amax_t;
        if constexpr (kLG) {
          float S, Mb[kLgSpan];
          lg_pass<NDIM, NT, true, UseLaneGroups<Tgt, NDIM>::kPursuit>(P, m, (float)tau, sigma_s, A_lg, B, w1base, id, S, Mb, amax_t);
        } else {
          amax_t = mc_max_exponent<Tgt, NDIM, GS, kPolarG>(tgt, ctr, sigma_s, A_lg, P.N, P.antithetic, w1base,
                                                  id, P.tag, P.rk, tz, tid);
        }
        const float amax = warp_max(amax_t);
        if ((tid & 31) == 0) sm.fmax_part[tid >> 5] = amax;
        gsync();
        if (tid == 0) {
          float mx = sm.fmax_part[0];
          for (int w = 1; w < GS / 32; ++w) mx = fmaxf(mx, sm.fmax_part[w]);
          sm.shift = mx;
        }
        gsync();
        B = -sm.shift;
        if constexpr (kLG) {
          float S, Mb[kLgSpan], am;
          lg_pass<NDIM, NT, false, UseLaneGroups<Tgt, NDIM>::kPursuit>(P, m, (float)tau, sigma_s, A_lg, B, w1base, id, S, Mb, am);
          lg_reduce<NDIM, NT>(sm, S, Mb);
        } else {
          float S, Mz[NDIM];
          mc_accumulate<Tgt, NDIM, GS, kProp>(tgt, ctr, sigma_s, A_lg, B, P.N, P.antithetic, w1base,
                                              id, P.tag, P.rk, S, Mz, tz, tid);
          cta_reduce<NDIM, GS, NT>(sm, S, Mz, tid);
        }
      }
    }  // hit < 0
    if (tid == 0) {
      const double* sums = sm.sum;
      if (hit >= 0) {
        sums = sm.memo_sum[hit];
        B = sm.memo_B[hit];
      } else {
        ++passes;
        if (memo_on && sm.n_memo < kMemo) {
          const int e = sm.n_memo;
          sm.memo_c[e] = c;
          sm.memo_B[e] = B;
          for (int d = 0; d <= NDIM; ++d) sm.memo_sum[e][d] = sm.sum[d];
          sm.n_memo = e + 1;
        }
        // a speculative sum is kept only when a real pass at c_spec would not have needed the
        // two-pass fallback (same S, same threshold): then it equals that pass bit for bit
        if (do_spec && sm.sum2[0] >= underflow_floor(P.N) && sm.n_memo < kMemo) {
          const int e = sm.n_memo;
          sm.memo_c[e] = c_spec;
          sm.memo_B[e] = B_spec;
          for (int d = 0; d <= NDIM; ++d) sm.memo_sum[e][d] = sm.sum2[d];
          sm.n_memo = e + 1;
        }
      }
      bool done = false;
      double dsh[NDIM];
      if constexpr (kProp) {
        for (int d = 0; d < NDIM; ++d) dsh[d] = ((double)ctr[d] - (double)xs[d]) / sigma_d;
      }
      sm.c_next = pass_epilogue<Tgt, NDIM>(P, tgt, m, j, k, id, c, sigma_d, A_eff, B, core_ref, sums,
                                           kProp ? dsh : nullptr, &done);
      sm.shift = done ? 1.f : 0.f;
    }
    gsync();
    c = sm.c_next;
    const bool done = sm.shift != 0.f;
    gsync();
    if (done) break;
  }
  if (tid == 0 && P.passes) atomicAdd(P.passes, (unsigned long long)passes);
}

// Plain passes with at most this many samples run one unit per warp (GS = 32), up to
// HJMC_QUAD_WARP_MAX_N one unit per 4 warps (GS = 128), above that one unit per CTA.
#ifndef HJMC_WARP_UNIT_MAX_N
#define HJMC_WARP_UNIT_MAX_N 4096
#endif
constexpr uint32_t kWarpUnitMaxN = HJMC_WARP_UNIT_MAX_N;

// Threads per unit of the plain kernel above HJMC_QUAD_WARP_MAX_N (the CTA by default; a
// build variant may set 64 or 128: 4 or 2 units per CTA, synchronised by named barriers).
#ifndef HJMC_CTA_GROUP
#define HJMC_CTA_GROUP HJMC_NT
#endif
constexpr int kCtaGroup = HJMC_CTA_GROUP;
// Plain passes with N ≤ this many samples (and above the warp switch) run 2 units per CTA
// (GS = 128, named barriers per unit).
#ifndef HJMC_QUAD_WARP_MAX_N
#define HJMC_QUAD_WARP_MAX_N 65536
#endif
constexpr uint32_t kQuadWarpMaxN = HJMC_QUAD_WARP_MAX_N;

template <class Tgt, int NDIM, int NT>
cudaError_t launch_solve(const SolveParams& p, int64_t units, cudaStream_t s) {
  if (units <= 0) return cudaSuccess;
  if (units > 0x7FFFFFFFLL) return cudaErrorInvalidValue;
  if constexpr (UseLaneGroups<Tgt, NDIM>::value) {
    if (!p.antithetic && !p.proposal) {
      if (p.speculate && p.reuse_passes && p.crn && p.mode == kModeSolve)
        solve_kernel<Tgt, NDIM, NT, true, false, NT, true><<<(unsigned)units, NT, 0, s>>>(p);
      else
        solve_kernel<Tgt, NDIM, NT, true, false><<<(unsigned)units, NT, 0, s>>>(p);
      return cudaGetLastError();
    }
  }
  if (p.proposal) {
    solve_kernel<Tgt, NDIM, NT, false, true><<<(unsigned)units, NT, 0, s>>>(p);
    return cudaGetLastError();
  }
  // Threads per unit for plain passes, from N alone (measured): one warp up to
  // N = 4,096, four warps up to N = 65,536, the CTA above. N is part of the configuration, so
  // every shard of a slice, every subset of horizons of a stepwise pass and the fused solve run
  // the same kernel with the same reduction order: results stay bit-identical across splits.
  auto launch_group = [&](auto gs_tag) {
    constexpr int GS = decltype(gs_tag)::value;
    constexpr int kPerCta = NT / GS;
    solve_kernel<Tgt, NDIM, NT, false, false, GS>
        <<<(unsigned)((units + kPerCta - 1) / kPerCta), NT, 0, s>>>(p);
  };
  // (the bowl, linear and constant targets never cycle between clamps: no speculative variant)
  constexpr bool kSpecTarget = !std::is_same<Tgt, QuadBowl<NDIM>>::value &&
                               !std::is_same<Tgt, Linear<NDIM>>::value &&
                               !std::is_same<Tgt, Const<NDIM>>::value;
  if constexpr (NDIM <= 16 && kSpecTarget) {
    if (p.speculate && p.reuse_passes && p.crn && p.mode == kModeSolve && !p.antithetic) {
      auto launch_spec = [&](auto gs_tag) {
        constexpr int GS = decltype(gs_tag)::value;
        constexpr int kPerCta = NT / GS;
        solve_kernel<Tgt, NDIM, NT, false, false, GS, true>
            <<<(unsigned)((units + kPerCta - 1) / kPerCta), NT, 0, s>>>(p);
      };
      if (p.N <= kWarpUnitMaxN)
        launch_spec(std::integral_constant<int, 32>{});
      else if (p.N <= kQuadWarpMaxN)
        launch_spec(std::integral_constant<int, 128>{});
      else
        launch_spec(std::integral_constant<int, kCtaGroup>{});
      return cudaGetLastError();
    }
  }
  if (p.N <= kWarpUnitMaxN)
    launch_group(std::integral_constant<int, 32>{});
  else if (p.N <= kQuadWarpMaxN)
    launch_group(std::integral_constant<int, 128>{});
  else
    launch_group(std::integral_constant<int, kCtaGroup>{});
  return cudaGetLastError();
}

// ---- small kernels ---------------------------------------------------------------------------
template <class Tgt, int NDIM>
__global__ void eval_target_kernel(const EvalParams P) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= P.M) return;
  const Tgt tgt(P.tp);
  double x[NDIM], dg[NDIM];
  for (int d = 0; d < NDIM; ++d) x[d] = (double)P.x[m * NDIM + d];
  if (P.g) P.g[m] = (float)tgt.g_host(x);
  if (P.dg) {
    tgt.dg(x, dg);
    for (int d = 0; d < NDIM; ++d) P.dg[m * NDIM + d] = (float)dg[d];
  }
}

template <class Tgt, int NDIM>
cudaError_t launch_eval_target(const EvalParams& p, cudaStream_t s) {
  if (p.M <= 0) return cudaSuccess;
  const int bs = 128;
  eval_target_kernel<Tgt, NDIM><<<(unsigned)((p.M + bs - 1) / bs), bs, 0, s>>>(p);
  return cudaGetLastError();
}

// Stepwise Picard initialisation (Algorithm 1): v^(0) = g(x), c^(0) = Γ(x, Dg(x)),
// identical for every horizon.
template <class Tgt, int NDIM>
__global__ void picard_init_kernel(const __grid_constant__ PicardInitParams P) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= P.M) return;
  const Tgt tgt(P.tp);
  double xd[NDIM], p[NDIM];
  for (int d = 0; d < NDIM; ++d) xd[d] = (double)P.x[m * NDIM + d];
  const float g = (float)tgt.g_host(xd);
  if (P.g0) P.g0[m] = g;
  tgt.dg(xd, p);
  const double c0 = gamma_update(P.sp, P.gp, xd, p);
  for (int j = 0; j < P.K; ++j) {
    P.c_state[(size_t)j * (size_t)P.M + (size_t)m] = c0;
    P.v_prev[(size_t)j * (size_t)P.M + (size_t)m] = g;
  }
}

template <class Tgt, int NDIM>
cudaError_t launch_picard_init(const PicardInitParams& p, cudaStream_t s) {
  if (p.M <= 0) return cudaSuccess;
  picard_init_kernel<Tgt, NDIM><<<(unsigned)((p.M + 127) / 128), 128, 0, s>>>(p);
  return cudaGetLastError();
}

// One instantiation set per (target, n): the fused solve kernel and the g/Dg evaluator.
template <template <int> class T, int NDIM>
KernelSet make_set() {
  constexpr int kThreads = HJMC_NT;
  KernelSet k;
  k.solve = &launch_solve<T<NDIM>, NDIM, kThreads>;
  k.eval_target = &launch_eval_target<T<NDIM>, NDIM>;
  k.picard_init = &launch_picard_init<T<NDIM>, NDIM>;
  k.threads = kThreads;
  return k;
}

}  // namespace

#define HJMC_CASE(TGT_ID, TMPL, NN) \
  if (target == TGT_ID && n == NN) { \
    *out = make_set<TMPL, NN>();     \
    return true;                     \
  }

}  // namespace hjmc
