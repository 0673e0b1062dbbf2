// hjmc_systems.cuh — Hamiltonians H(x, p) and the frozen-coefficient map Γ.
//
// Evaluated once per query per Picard iterate (reading R5: c is frozen per query, so H never
// enters the per-sample loop), in double precision: it is off the hot loop and the extra
// precision keeps the Picard feedback (|·| kinks, clamps, 1/|p|²) close to the oracle's.
// Definitions: include/hjmc.h SYSTEMS (R13; R15; R16).
#pragma once
#include <cstdint>

namespace hjmc {

enum : int {
  kSysQuadratic = 0, kSysDubinsRel = 1, kSysRocket6 = 2, kSysDubinsPairs = 3, kSysRocket3 = 4,
  kSysDoubleIntegrator = 5, kSysMultiAgent = 6
};

struct SystemParams {
  int id;
  int n;
  float p[8];
  int np;
};

__device__ __forceinline__ double sys_param(const SystemParams& s, int i, double dflt) {
  return s.np > i ? (double)s.p[i] : dflt;
}

// Eq. dubins_ham_general verbatim.
__device__ __forceinline__ double dubins_rel_H(double vp, double ve, double w, const double* x,
                                               const double* p) {
  double sn, cs;
  sincos(x[2], &sn, &cs);
  return p[0] * (vp * cs - ve) - p[1] * (vp * sn) + w * fabs(p[0] * x[1] - p[1] * x[0] - p[2]) -
         w * fabs(p[2]);
}

__device__ inline double hamiltonian(const SystemParams& s, const double* x, const double* p) {
  const int n = s.n;
  switch (s.id) {
    case kSysQuadratic: {  // H = |p|²/2
      double a = 0.0;
      for (int d = 0; d < n; ++d) a += p[d] * p[d];
      return 0.5 * a;
    }
    case kSysDubinsRel:
      return dubins_rel_H(sys_param(s, 0, 5.0), sys_param(s, 1, 5.0), sys_param(s, 2, 1.0), x, p);
    case kSysRocket6: {  // R15
      const double a = sys_param(s, 0, 64.0), grav = sys_param(s, 1, 32.0),
                   dmax = sys_param(s, 2, 1.0);
      double h = 0.0;
      for (int v = 0; v < 2; ++v) {
        double sn, cs;
        sincos(x[3 * v + 2], &sn, &cs);
        h += a * (p[3 * v] * cs + p[3 * v + 1] * sn) - grav * p[3 * v + 1];
      }
      return h - fabs(p[2]) + fabs(p[5]) + dmax * sqrt(p[3] * p[3] + p[4] * p[4]);
    }
    case kSysRocket3: {  // Eq. rocket_ham_simplified verbatim (R14)
      const double a = sys_param(s, 0, 64.0), grav = sys_param(s, 1, 32.0);
      double sn, cs;
      sincos(x[2], &sn, &cs);
      return -(a * p[0] * cs + p[1] * (a + a * sn - grav) - fabs(p[0] * x[0] + p[2]) -
               fabs(p[1] * x[0] - p[2]));
    }
    case kSysDoubleIntegrator:  // Eq. dint_ham, u = −sign(p2)
      return p[0] * x[1] - fabs(p[1]);
    case kSysMultiAgent: {  // last agent evades (+|p_θ|), the others pursue (−|p_θ|)
      const int A = n / 3;
      const double ap = sys_param(s, 0, 1.0), ae = sys_param(s, 1, 1.0);
      double h = 0.0;
      for (int i = 0; i < A; ++i) {
        double sn, cs;
        sincos(x[3 * i + 2], &sn, &cs);
        const double a = (i == A - 1) ? ae : ap;
        h += a * (p[3 * i] * cs + p[3 * i + 1] * sn);
        h += (i == A - 1) ? fabs(p[3 * i + 2]) : -fabs(p[3 * i + 2]);
      }
      return h;
    }
    case kSysDubinsPairs: {  // R16: decoupled relative Dubins pairs
      const double vp = sys_param(s, 0, 5.0), ve = sys_param(s, 1, 5.0), w = sys_param(s, 2, 1.0);
      double h = 0.0;
      for (int q = 0; q < n / 3; ++q) h += dubins_rel_H(vp, ve, w, x + 3 * q, p + 3 * q);
      return h;
    }
  }
  return __longlong_as_double(0x7FF8000000000000LL);  // NaN: unknown system
}

struct GammaParams {
  double delta_eff, m0, c_min, c_max;
};

// Γ(x, p) = clamp(2 H(x, p̃) / (δ_eff |p̃|²), c_min, c_max), p̃ = p·max(1, m0/|p|), p̃ = m0 e1
// at p = 0. `p` is overwritten with p̃. Returns NaN if H is NaN.
__device__ inline double gamma_update(const SystemParams& s, const GammaParams& g, const double* x,
                               double* p) {
  const int n = s.n;
  double nrm2 = 0.0;
  for (int d = 0; d < n; ++d) nrm2 += p[d] * p[d];
  const double nrm = sqrt(nrm2);
  if (nrm == 0.0) {
    p[0] = g.m0;
  } else if (nrm < g.m0) {
    const double sc = g.m0 / nrm;
    for (int d = 0; d < n; ++d) p[d] *= sc;
  }
  double pt2 = 0.0;
  for (int d = 0; d < n; ++d) pt2 += p[d] * p[d];
  const double H = hamiltonian(s, x, p);
  const double c = 2.0 * H / (g.delta_eff * pt2);
  if (c != c) return c;
  return c < g.c_min ? g.c_min : (c > g.c_max ? g.c_max : c);
}

}  // namespace hjmc
