// hjmc_targets.cuh — terminal costs g(y) as device functors.
//
// Each functor splits g = core(y) + off so the hot loop forms the log2-domain weight exponent
// with a single FFMA, a = A·core + B, A = −c·log2(e). It also supplies
//   core_lower(xs, σ): a guaranteed lower bound of core(xs + σz) over every z the sampler can
//                      emit (|z_d| ≤ ZMAX, include/hjmc.h), which fixes a safe exponent shift
//                      (no weight can exceed 2^0);
//   g_host/dg:         g(x) and the analytic Dg(x) in double for c^(0) (R7);
//   kHomog, core_polar: the pair union and pursuit-min (distances, homogeneous of degree 1
//                      in the position) also evaluate core(y)/σ' from σ-scaled coordinates x/σ'
//                      and the polar Box–Muller output, coordinate d = x'_d + rr_d·t_d (one FFMA;
//                      no r̂·cos / r̂·sin products — hjmc_solve_impl.cuh).
// Definitions follow include/hjmc.h TARGETS (R15, R16).
#pragma once
#include <cstdint>

#include "hjmc_rng.cuh"

namespace hjmc {

constexpr float kZmax = 5.7684f;         // sqrt(48 ln 2) = 5.76829…, plus MUFU slack
constexpr float kZmax2 = 8.1578f;        // bound of the norm of any two coordinates

struct TargetParams {
  float p[72];
  int np;
};

// ---------------------------------------------------------------------------------------------
template <int NDIM>
struct QuadBowl {  // g = |y|²/2 − α0
  static constexpr bool kHomog = false;
  float off;
  __device__ explicit QuadBowl(const TargetParams& t) : off(-(t.np > 0 ? t.p[0] : 0.25f)) {}
  __device__ __forceinline__ float core(const float (&xs)[NDIM], float sigma,
                                        const float (&z)[NDIM]) const {
    float s = 0.f;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) {
      const float y = fmaf(sigma, z[d], xs[d]);
      s = fmaf(y, y, s);
    }
    return 0.5f * s;
  }
  __device__ float core_lower(const float (&xs)[NDIM], float sigma) const {
    float r2 = 0.f;
    for (int d = 0; d < NDIM; ++d) r2 = fmaf(xs[d], xs[d], r2);
    const float lo = fmaxf(0.f, sqrtf(r2) - sigma * kZmax * sqrtf((float)NDIM));
    return 0.5f * lo * lo * 0.9999f;
  }
  __device__ double g_host(const double* x) const {
    double s = 0.0;
    for (int d = 0; d < NDIM; ++d) s += x[d] * x[d];
    return 0.5 * s + (double)off;
  }
  __device__ void dg(const double* x, double* g) const {
    for (int d = 0; d < NDIM; ++d) g[d] = x[d];
  }
};

// ---------------------------------------------------------------------------------------------
template <int NDIM>
struct Disk {  // g = sqrt(y0² + y1²) − r
  static_assert(NDIM >= 2, "DISK needs n >= 2");
  // a distance too, but kept on the unscaled path: measured −2.6 % on C2 with the polar pass,
  // yet the changed rounding flips one more non-contractive C2 trajectory unit (query 500, R27)
  // than the capped parity sample allows
  static constexpr bool kHomog = false;
  float off;
  __device__ explicit Disk(const TargetParams& t) : off(-(t.np > 0 ? t.p[0] : 5.0f)) {}
  __device__ __forceinline__ float core(const float (&xs)[NDIM], float sigma,
                                        const float (&z)[NDIM]) const {
    const float y0 = fmaf(sigma, z[0], xs[0]);
    const float y1 = fmaf(sigma, z[1], xs[1]);
    return sqrt_approx(fmaf(y0, y0, y1 * y1));
  }
  __device__ float core_lower(const float (&xs)[NDIM], float sigma) const {
    return fmaxf(0.f, sqrtf(xs[0] * xs[0] + xs[1] * xs[1]) - sigma * kZmax2) * 0.9999f;
  }
  __device__ double g_host(const double* x) const {
    return sqrt(x[0] * x[0] + x[1] * x[1]) + (double)off;
  }
  __device__ void dg(const double* x, double* g) const {
    for (int d = 0; d < NDIM; ++d) g[d] = 0.0;
    const double rho = sqrt(x[0] * x[0] + x[1] * x[1]);
    if (rho > 0.0) {
      g[0] = x[0] / rho;
      g[1] = x[1] / rho;
    } else {
      g[0] = 1.0;
    }
  }
};

// ---------------------------------------------------------------------------------------------
template <int NDIM>
struct RelDisk6 {  // g = ‖(y0 − y3, y1 − y4)‖ − r  (n = 6)
  static_assert(NDIM == 6, "REL_DISK6 needs n == 6");
  // unscaled path: the polar pass measured a tie on C3 (the relative coordinates cost an FFMA
  // more each)
  static constexpr bool kHomog = false;
  float off;
  __device__ explicit RelDisk6(const TargetParams& t) : off(-(t.np > 0 ? t.p[0] : 1.5f)) {}
  __device__ __forceinline__ float core(const float (&xs)[NDIM], float sigma,
                                        const float (&z)[NDIM]) const {
    // (x0 − x3) + σ(z0 − z3): the x difference is loop-invariant (hoisted by the compiler),
    // leaving one FADD + one FFMA per relative coordinate
    const float dx = fmaf(sigma, z[0] - z[3], xs[0] - xs[3]);
    const float dz = fmaf(sigma, z[1] - z[4], xs[1] - xs[4]);
    return sqrt_approx(fmaf(dx, dx, dz * dz));
  }
  __device__ float core_lower(const float (&xs)[NDIM], float sigma) const {
    const float dx = xs[0] - xs[3], dz = xs[1] - xs[4];
    return fmaxf(0.f, sqrtf(dx * dx + dz * dz) - 2.f * sigma * kZmax2) * 0.9999f;
  }
  __device__ double g_host(const double* x) const {
    const double dx = x[0] - x[3], dz = x[1] - x[4];
    return sqrt(dx * dx + dz * dz) + (double)off;
  }
  __device__ void dg(const double* x, double* g) const {
    for (int d = 0; d < NDIM; ++d) g[d] = 0.0;
    const double dx = x[0] - x[3], dz = x[1] - x[4];
    const double rho = sqrt(dx * dx + dz * dz);
    if (rho > 0.0) {
      g[0] = dx / rho;
      g[1] = dz / rho;
      g[3] = -dx / rho;
      g[4] = -dz / rho;
    } else {
      g[0] = 1.0;
    }
  }
};

// ---------------------------------------------------------------------------------------------
template <int NDIM>
struct PairUnion {  // g = sqrt(min_q (y_{3q}² + y_{3q+1}²)) − r  (n = 3K)
  static_assert(NDIM % 3 == 0, "PAIR_UNION needs n = 3K");
  static constexpr int kPairs = NDIM / 3;
  static constexpr bool kHomog = true;
  float off;
  __device__ explicit PairUnion(const TargetParams& t) : off(-(t.np > 0 ? t.p[0] : 1.0f)) {}
  __device__ __forceinline__ float core_polar(const float (&xs)[NDIM], const float (&rr)[NDIM],
                                              const float (&t)[NDIM]) const {
    float best = 3.0e38f;
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      const float a = fmaf(rr[3 * q], t[3 * q], xs[3 * q]);
      const float b = fmaf(rr[3 * q + 1], t[3 * q + 1], xs[3 * q + 1]);
      best = fminf(best, fmaf(a, a, b * b));
    }
    return sqrt_approx(best);
  }
  __device__ __forceinline__ float core(const float (&xs)[NDIM], float sigma,
                                        const float (&z)[NDIM]) const {
    float best = 3.0e38f;
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      const float a = fmaf(sigma, z[3 * q], xs[3 * q]);
      const float b = fmaf(sigma, z[3 * q + 1], xs[3 * q + 1]);
      best = fminf(best, fmaf(a, a, b * b));
    }
    return sqrt_approx(best);
  }
  __device__ float core_lower(const float (&xs)[NDIM], float sigma) const {
    float best = 3.0e38f;
    for (int q = 0; q < kPairs; ++q)
      best = fminf(best, xs[3 * q] * xs[3 * q] + xs[3 * q + 1] * xs[3 * q + 1]);
    return fmaxf(0.f, sqrtf(best) - sigma * kZmax2) * 0.9999f;
  }
  __device__ double g_host(const double* x) const {
    double best = 1e300;
    for (int q = 0; q < kPairs; ++q) {
      const double d = sqrt(x[3 * q] * x[3 * q] + x[3 * q + 1] * x[3 * q + 1]);
      best = d < best ? d : best;
    }
    return best + (double)off;
  }
  __device__ void dg(const double* x, double* g) const {
    for (int d = 0; d < NDIM; ++d) g[d] = 0.0;
    double best = 1e300;
    int arg = 0;
    for (int q = 0; q < kPairs; ++q) {
      const double d = sqrt(x[3 * q] * x[3 * q] + x[3 * q + 1] * x[3 * q + 1]);
      if (d < best) {  // first minimiser on ties
        best = d;
        arg = q;
      }
    }
    if (best > 0.0) {
      g[3 * arg] = x[3 * arg] / best;
      g[3 * arg + 1] = x[3 * arg + 1] / best;
    } else {
      g[0] = 1.0;
    }
  }
};

// ---------------------------------------------------------------------------------------------
template <int NDIM>
struct PursuitMin {  // g = min_{i < A−1} ‖pos_i − pos_{A−1}‖ − r  (n = 3A)
  static_assert(NDIM % 3 == 0 && NDIM >= 6, "PURSUIT_MIN needs n = 3A, A >= 2");
  static constexpr int kAgents = NDIM / 3;
  static constexpr int kE = 3 * (kAgents - 1);  // evader's first coordinate
  static constexpr bool kHomog = true;
  float off;
  __device__ explicit PursuitMin(const TargetParams& t) : off(-(t.np > 0 ? t.p[0] : 1.5f)) {}
  __device__ __forceinline__ float core_polar(const float (&xs)[NDIM], const float (&rr)[NDIM],
                                              const float (&t)[NDIM]) const {
    const float ex = fmaf(rr[kE], t[kE], xs[kE]);
    const float ey = fmaf(rr[kE + 1], t[kE + 1], xs[kE + 1]);
    float best = 3.0e38f;
#pragma unroll
    for (int i = 0; i < kAgents - 1; ++i) {
      const float dx = fmaf(rr[3 * i], t[3 * i], xs[3 * i]) - ex;
      const float dy = fmaf(rr[3 * i + 1], t[3 * i + 1], xs[3 * i + 1]) - ey;
      best = fminf(best, fmaf(dx, dx, dy * dy));
    }
    return sqrt_approx(best);
  }
  __device__ __forceinline__ float core(const float (&xs)[NDIM], float sigma,
                                        const float (&z)[NDIM]) const {
    const float ex = fmaf(sigma, z[kE], xs[kE]);
    const float ey = fmaf(sigma, z[kE + 1], xs[kE + 1]);
    float best = 3.0e38f;
#pragma unroll
    for (int i = 0; i < kAgents - 1; ++i) {
      const float dx = fmaf(sigma, z[3 * i], xs[3 * i]) - ex;
      const float dy = fmaf(sigma, z[3 * i + 1], xs[3 * i + 1]) - ey;
      best = fminf(best, fmaf(dx, dx, dy * dy));
    }
    return sqrt_approx(best);
  }
  __device__ float core_lower(const float (&xs)[NDIM], float sigma) const {
    float best = 3.0e38f;
    for (int i = 0; i < kAgents - 1; ++i) {
      const float dx = xs[3 * i] - xs[kE], dy = xs[3 * i + 1] - xs[kE + 1];
      best = fminf(best, dx * dx + dy * dy);
    }
    return fmaxf(0.f, sqrtf(best) - 2.f * sigma * kZmax2) * 0.9999f;
  }
  __device__ double g_host(const double* x) const {
    double best = 1e300;
    for (int i = 0; i < kAgents - 1; ++i) {
      const double dx = x[3 * i] - x[kE], dy = x[3 * i + 1] - x[kE + 1];
      const double d = sqrt(dx * dx + dy * dy);
      best = d < best ? d : best;
    }
    return best + (double)off;
  }
  __device__ void dg(const double* x, double* g) const {
    for (int d = 0; d < NDIM; ++d) g[d] = 0.0;
    double best = 1e300;
    int arg = 0;
    for (int i = 0; i < kAgents - 1; ++i) {
      const double dx = x[3 * i] - x[kE], dy = x[3 * i + 1] - x[kE + 1];
      const double d = sqrt(dx * dx + dy * dy);
      if (d < best) {  // first minimiser on ties
        best = d;
        arg = i;
      }
    }
    if (best > 0.0) {
      const double ux = (x[3 * arg] - x[kE]) / best, uy = (x[3 * arg + 1] - x[kE + 1]) / best;
      g[3 * arg] = ux;
      g[3 * arg + 1] = uy;
      g[kE] = -ux;
      g[kE + 1] = -uy;
    } else {
      g[0] = 1.0;
    }
  }
};

// ---------------------------------------------------------------------------------------------
template <int NDIM>
struct Linear {  // g = a·y + b (test target; Gaussian-tilt identities)
  static constexpr bool kHomog = false;
  float a[NDIM];
  float off;
  __device__ explicit Linear(const TargetParams& t) {
    for (int d = 0; d < NDIM; ++d) a[d] = t.p[d];
    off = t.p[NDIM];
  }
  __device__ __forceinline__ float core(const float (&xs)[NDIM], float sigma,
                                        const float (&z)[NDIM]) const {
    float s = 0.f;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) s = fmaf(a[d], fmaf(sigma, z[d], xs[d]), s);
    return s;
  }
  __device__ float core_lower(const float (&xs)[NDIM], float sigma) const {
    float s = 0.f, l1 = 0.f;
    for (int d = 0; d < NDIM; ++d) {
      s = fmaf(a[d], xs[d], s);
      l1 += fabsf(a[d]);
    }
    const float lo = s - sigma * kZmax * l1;
    return lo - 1e-4f * fabsf(lo) - 1e-6f;
  }
  __device__ double g_host(const double* x) const {
    double s = (double)off;
    for (int d = 0; d < NDIM; ++d) s += (double)a[d] * x[d];
    return s;
  }
  __device__ void dg(const double* x, double* g) const {
    for (int d = 0; d < NDIM; ++d) g[d] = (double)a[d];
  }
};

// ---------------------------------------------------------------------------------------------
template <int NDIM>
struct Const {  // g = k (test target)
  static constexpr bool kHomog = false;
  float off;
  __device__ explicit Const(const TargetParams& t) : off(t.np > 0 ? t.p[0] : 0.f) {}
  __device__ __forceinline__ float core(const float (&)[NDIM], float, const float (&)[NDIM]) const {
    return 0.f;
  }
  __device__ float core_lower(const float (&)[NDIM], float) const { return 0.f; }
  __device__ double g_host(const double*) const { return (double)off; }
  __device__ void dg(const double*, double* g) const {
    for (int d = 0; d < NDIM; ++d) g[d] = 0.0;
  }
};

}  // namespace hjmc
