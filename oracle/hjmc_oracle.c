/*
 * hjmc_oracle.c — TEST INFRASTRUCTURE ONLY. Not part of the product; the product path never
 * loads this file's library (see hjmc_oracle.h for who may, and for each function's pins).
 *
 * A plain, slow, obviously-correct CPU implementation, in double precision, of what the
 * B200 path computes: the Monte-Carlo Picard evaluation of the viscous HJ value v^δ and its
 * gradient Dv^δ (arxiv/paper_2605_18566). Every function follows the paper's formulas in the
 * paper's order; citations are PAPER.md line numbers (P:…), SPEC.md lines (S:…) and the
 * readings R# listed in DESIGN.md §3. No blocking, fusion or reordering: the estimator
 * stores the exponents, takes their maximum, and sums in sample order (two passes).
 */
#include "hjmc_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------------------------
 * Random numbers (R19). Philox4x32-10 as published by Salmon, Moraes, Dror & Shaw (SC'11):
 * a 10-round Feistel-like bijection of a 128-bit counter under a 64-bit key.
 * ---------------------------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)x0;  /* multiplier M0 on word 0 */
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)x2;  /* multiplier M1 on word 2 */
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t y0 = hi1 ^ x1 ^ k0;
    uint32_t y1 = lo1;
    uint32_t y2 = hi0 ^ x3 ^ k1;
    uint32_t y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    /* Weyl key schedule: bump the key between rounds */
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* u(w) = (2m+1)/2^24 in (0,1) and a(w) = m/2^23 in [0,1), m = high 23 bits of w (R19). */
static double unif_open(uint32_t w) { return (2.0 * (double)(w >> 9) + 1.0) / 16777216.0; }
static double unif_angle(uint32_t w) { return (double)(w >> 9) / 8388608.0; }

/* Grouping of draws (R19): G = 4/gcd(n,4) consecutive draws share one flat stream of
 * G*n normals (G*n/4 Philox blocks) when G*n <= 16, else G = 1 and each draw takes
 * ceil(n/4) blocks of its own. */
static int draw_group(int n) {
  int g = (n % 4 == 0) ? 1 : ((n % 2 == 0) ? 2 : 4);
  return (g * n <= 16) ? g : 1;
}

/* One Philox block -> its four normals: Box-Muller on word pairs (0,1) and (2,3). */
static void block_normals(const orc_problem* P, uint32_t group, uint32_t b, uint32_t qid,
                          uint32_t jw, uint32_t kw, double zz[4], uint32_t w[4]) {
  const double two_pi = 6.283185307179586476925286766559;
  uint32_t key[2] = {(uint32_t)(P->seed & 0xFFFFFFFFu), (uint32_t)(P->seed >> 32)};
  uint32_t ctr[4] = {group, b | (kw << 8) | (jw << 16), qid, P->tag};
  orc_philox4x32_10(ctr, key, w);
  double r01 = sqrt(-2.0 * log(unif_open(w[0])));
  double r23 = sqrt(-2.0 * log(unif_open(w[2])));
  zz[0] = r01 * cos(two_pi * unif_angle(w[1]));
  zz[1] = r01 * sin(two_pi * unif_angle(w[1]));
  zz[2] = r23 * cos(two_pi * unif_angle(w[3]));
  zz[3] = r23 * sin(two_pi * unif_angle(w[3]));
}

/* The n standard normals z_{i,0..n-1} of sample i ("y_i ~ N(0, I_n)"): draw
 * q = i (antithetic: i >> 1, odd i negated), group g = q / G, r = q mod G; the group's Q
 * blocks (Q = ceil(n/4) for G = 1, G*n/4 otherwise) b = 0..Q-1 have counter
 * (g, b | kw << 8 | jw << 16, qid, tag) and their Box-Muller outputs form one stream; normal
 * d is element l = r*n + d (G = 1: l = d), i.e. word l % 4 of block l / 4 (R19). raw (may be
 * NULL) receives the 4 words of every block the sample touches, in order. */
void orc_sample_normals(const orc_problem* P, uint32_t qid, uint32_t jw, uint32_t kw, uint32_t i,
                        double* z, uint32_t* raw) {
  int n = P->n;
  uint32_t draw = P->antithetic ? (i >> 1) : i;
  double sign = (P->antithetic && (i & 1u)) ? -1.0 : 1.0;
  int G = draw_group(n);
  uint32_t g = draw / (uint32_t)G;
  int r = (int)(draw % (uint32_t)G);
  int first = (G == 1) ? 0 : r * n;                 /* position of normal 0 in the stream */
  int64_t cur = -1;
  double zz[4];
  uint32_t w[4];
  int nraw = 0;
  for (int d = 0; d < n; ++d) {
    int l = first + d;
    int64_t blk = l / 4;
    if (blk != cur) {
      block_normals(P, g, (uint32_t)blk, qid, jw, kw, zz, w);
      if (raw) { for (int t = 0; t < 4; ++t) raw[4 * nraw + t] = w[t]; }
      ++nraw;
      cur = blk;
    }
    z[d] = sign * zz[l % 4];
  }
}

/* ------------------------------------------------------------------------------------------
 * Targets g (terminal costs; signed distances minus a radius; R15, R16).
 * ---------------------------------------------------------------------------------------- */
static double tparam(const orc_problem* P, int idx, double dflt) {
  return (P->n_tgt_params > idx) ? P->tgt_params[idx] : dflt;
}

double orc_target_g(const orc_problem* P, const double* y) {
  int n = P->n;
  switch (P->target) {
    case ORC_TGT_QUAD_BOWL: { /* g = |y|^2/2 - alpha0 (config 1; P:107 exact case) */
      double s = 0.0;
      for (int d = 0; d < n; ++d) s += y[d] * y[d];
      return 0.5 * s - tparam(P, 0, 0.25);
    }
    case ORC_TGT_DISK: /* cylinder x1^2 + x2^2 <= r^2 as signed distance */
      return sqrt(y[0] * y[0] + y[1] * y[1]) - tparam(P, 0, 5.0);
    case ORC_TGT_REL_DISK6: { /* ||(xP - xE, zP - zE)|| - r (R15) */
      double dx = y[0] - y[3], dz = y[1] - y[4];
      return sqrt(dx * dx + dz * dz) - tparam(P, 0, 1.5);
    }
    case ORC_TGT_PAIR_UNION: { /* min over pairs of ||pos_q|| - r (R16) */
      double best = INFINITY;
      for (int q = 0; q < n / 3; ++q) {
        double dq = sqrt(y[3 * q] * y[3 * q] + y[3 * q + 1] * y[3 * q + 1]);
        if (dq < best) best = dq;
      }
      return best - tparam(P, 0, 1.0);
    }
    case ORC_TGT_LINEAR: { /* g = a.y + b */
      double s = tparam(P, n, 0.0);
      for (int d = 0; d < n; ++d) s += tparam(P, d, 0.0) * y[d];
      return s;
    }
    case ORC_TGT_CONST:
      return tparam(P, 0, 0.0);
    case ORC_TGT_PURSUIT_MIN: { /* min over pursuers i of ||pos_i - pos_evader|| - r */
      int A = n / 3;
      const double* e = y + 3 * (A - 1);
      double best = INFINITY;
      for (int i = 0; i < A - 1; ++i) {
        double dx = y[3 * i] - e[0], dy = y[3 * i + 1] - e[1];
        double d = sqrt(dx * dx + dy * dy);
        if (d < best) best = d;
      }
      return best - tparam(P, 0, 1.5);
    }
  }
  return NAN;
}

/* BRAT avoid function l(x): positive inside the obstacle; the tube is
 * clamped to max(tube, l(x)) so states inside the avoid set are excluded from the BRAT. */
double orc_avoid_l(const orc_problem* P, const double* x) {
  if (P->avoid == ORC_AVOID_DISK) {
    double dx = x[0] - P->avoid_params[0], dy = x[1] - P->avoid_params[1];
    return P->avoid_params[2] - sqrt(dx * dx + dy * dy);
  }
  return -INFINITY;
}

/* Analytic Dg for c^(0) (R7: e1 at the singular point of a distance). */
void orc_target_dg(const orc_problem* P, const double* x, double* dg) {
  int n = P->n;
  for (int d = 0; d < n; ++d) dg[d] = 0.0;
  switch (P->target) {
    case ORC_TGT_QUAD_BOWL:
      for (int d = 0; d < n; ++d) dg[d] = x[d];
      return;
    case ORC_TGT_DISK: {
      double rho = sqrt(x[0] * x[0] + x[1] * x[1]);
      if (rho > 0.0) { dg[0] = x[0] / rho; dg[1] = x[1] / rho; } else { dg[0] = 1.0; }
      return;
    }
    case ORC_TGT_REL_DISK6: {
      double dx = x[0] - x[3], dz = x[1] - x[4];
      double rho = sqrt(dx * dx + dz * dz);
      if (rho > 0.0) {
        dg[0] = dx / rho; dg[1] = dz / rho; dg[3] = -dx / rho; dg[4] = -dz / rho;
      } else {
        dg[0] = 1.0;
      }
      return;
    }
    case ORC_TGT_PAIR_UNION: {
      int arg = 0;
      double best = INFINITY;
      for (int q = 0; q < n / 3; ++q) {
        double dq = sqrt(x[3 * q] * x[3 * q] + x[3 * q + 1] * x[3 * q + 1]);
        if (dq < best) { best = dq; arg = q; }   /* first minimiser on ties */
      }
      if (best > 0.0) { dg[3 * arg] = x[3 * arg] / best; dg[3 * arg + 1] = x[3 * arg + 1] / best; }
      else { dg[0] = 1.0; }
      return;
    }
    case ORC_TGT_LINEAR:
      for (int d = 0; d < n; ++d) dg[d] = tparam(P, d, 0.0);
      return;
    case ORC_TGT_CONST:
      return;
    case ORC_TGT_PURSUIT_MIN: {
      int A = n / 3, arg = 0;
      const double* e = x + 3 * (A - 1);
      double best = INFINITY;
      for (int i = 0; i < A - 1; ++i) {
        double dx = x[3 * i] - e[0], dy = x[3 * i + 1] - e[1];
        double d = sqrt(dx * dx + dy * dy);
        if (d < best) { best = d; arg = i; }   /* first minimiser on ties */
      }
      if (best > 0.0) {
        double dx = (x[3 * arg] - e[0]) / best, dy = (x[3 * arg + 1] - e[1]) / best;
        dg[3 * arg] = dx; dg[3 * arg + 1] = dy;
        dg[3 * (A - 1)] = -dx; dg[3 * (A - 1) + 1] = -dy;
      } else {
        dg[0] = 1.0;
      }
      return;
    }
  }
}

/* ------------------------------------------------------------------------------------------
 * Hamiltonians H(x, p) (sign box P:89–100: H = max_u min_w <p, f>).
 * ---------------------------------------------------------------------------------------- */
static double sparam(const orc_problem* P, int idx, double dflt) {
  return (P->n_sys_params > idx) ? P->sys_params[idx] : dflt;
}

/* Eq. dubins_ham_general, verbatim (R13). State (x1, x2, x3). */
static double dubins_H(double vp, double ve, double w, const double* x, const double* p) {
  return p[0] * (vp * cos(x[2]) - ve) - p[1] * (vp * sin(x[2])) +
         w * fabs(p[0] * x[1] - p[1] * x[0] - p[2]) - w * fabs(p[2]);
}

double orc_hamiltonian(const orc_problem* P, const double* x, const double* p) {
  int n = P->n;
  switch (P->system) {
    case ORC_SYS_QUADRATIC: { /* H = |p|^2 / 2 */
      double s = 0.0;
      for (int d = 0; d < n; ++d) s += p[d] * p[d];
      return 0.5 * s;
    }
    case ORC_SYS_DUBINS_REL:
      return dubins_H(sparam(P, 0, 5.0), sparam(P, 1, 5.0), sparam(P, 2, 1.0), x, p);
    case ORC_SYS_ROCKET6: { /* R15: two vehicles (x, z, theta) each, thrust a, gravity, disturbance */
      double a = sparam(P, 0, 64.0), grav = sparam(P, 1, 32.0), dmax = sparam(P, 2, 1.0);
      double h = 0.0;
      for (int v = 0; v < 2; ++v) {
        const double* xv = x + 3 * v;
        const double* pv = p + 3 * v;
        h += a * (pv[0] * cos(xv[2]) + pv[1] * sin(xv[2])) - grav * pv[1];
      }
      h += -fabs(p[2]) + fabs(p[5]) + dmax * sqrt(p[3] * p[3] + p[4] * p[4]);
      return h;
    }
    case ORC_SYS_ROCKET3: { /* Eq. rocket_ham_simplified, verbatim (R14) */
      double a = sparam(P, 0, 64.0), grav = sparam(P, 1, 32.0);
      return -(a * p[0] * cos(x[2]) + p[1] * (a + a * sin(x[2]) - grav) -
               fabs(p[0] * x[0] + p[2]) - fabs(p[1] * x[0] - p[2]));
    }
    case ORC_SYS_DOUBLE_INTEGRATOR: /* Eq. dint_ham P:1300–1303 with u = -sign(p2) */
      return p[0] * x[1] - fabs(p[1]);
    case ORC_SYS_MULTIAGENT: { /* agents (x, y, theta), speed a_i, |u_i| <= 1; last =
                                  evader (maximises), others pursuers (minimise) */
      int A = n / 3;
      double ap = sparam(P, 0, 1.0), ae = sparam(P, 1, 1.0);
      double h = 0.0;
      for (int i = 0; i < A; ++i) {
        double a = (i == A - 1) ? ae : ap;
        h += a * (p[3 * i] * cos(x[3 * i + 2]) + p[3 * i + 1] * sin(x[3 * i + 2]));
        h += (i == A - 1) ? fabs(p[3 * i + 2]) : -fabs(p[3 * i + 2]);
      }
      return h;
    }
    case ORC_SYS_DUBINS_PAIRS: { /* R16: sum of independent relative Dubins pairs */
      double h = 0.0;
      for (int q = 0; q < n / 3; ++q)
        h += dubins_H(sparam(P, 0, 5.0), sparam(P, 1, 5.0), sparam(P, 2, 1.0), x + 3 * q, p + 3 * q);
      return h;
    }
  }
  return NAN;
}

static double delta_eff(const orc_problem* P) { return P->full_laplacian ? 2.0 * P->delta : P->delta; }

/* Coefficient update Γ (Algorithm 1 step 4; P:336 map Γ), with the floor |p| >= m0
 * and the clamp [c_min, c_max] of Assumption 1 item 2 (R8). */
double orc_gamma(const orc_problem* P, const double* x, const double* p) {
  int n = P->n;
  double pt[ORC_MAX_N];
  double norm2 = 0.0;
  for (int d = 0; d < n; ++d) norm2 += p[d] * p[d];
  double norm = sqrt(norm2);
  if (norm == 0.0) {
    for (int d = 0; d < n; ++d) pt[d] = 0.0;
    pt[0] = P->m0;                               /* p~ = m0 e1 */
  } else {
    double s = (norm < P->m0) ? P->m0 / norm : 1.0; /* p~ = p max(1, m0/|p|) */
    for (int d = 0; d < n; ++d) pt[d] = p[d] * s;
  }
  double pt2 = 0.0;
  for (int d = 0; d < n; ++d) pt2 += pt[d] * pt[d];
  double H = orc_hamiltonian(P, x, pt);
  double c = 2.0 * H / (delta_eff(P) * pt2);     /* Eq. coeff_frozen */
  if (c < P->c_min) c = P->c_min;
  if (c > P->c_max) c = P->c_max;
  return c;
}

/* ------------------------------------------------------------------------------------------
 * One Φ pass (Thm 2's map Φ) by the Monte-Carlo estimators of Cor. logsumexp
 * and Cor. mc_gradient:
 *   v  = -(1/c) log( (1/N) sum_i exp(-c g(x + sigma y_i)) ),  sigma = sqrt(delta (T - t))
 *   Dv = (1/(c sigma^2)) (x - sum_i s_i w_i / sum_i w_i)  =  -(sum_i w_i z_i / sum_i w_i)/(c sigma)
 * (R2: the prefactor is the sampling variance sigma^2 = delta_eff tau; R23: the z-form is the
 * same number). Log-sum-exp "for numerical stability": A = max_i a_i, two passes.
 * diag (may be NULL): [min_i g_i, mean_i g_i, ESS = (sum w)^2 / sum w^2, SE_v, A, log sum w].
 * se_dv (may be NULL): delta-method standard error of each Dv component.
 * ---------------------------------------------------------------------------------------- */
int orc_phi(const orc_problem* P, const double* x, const double* drift, uint32_t qid, double c,
            double tau, uint32_t jw, uint32_t kw, double* v, double* dv, double* diag,
            double* se_dv) {
  int n = P->n;
  uint32_t N = P->N;
  double xs[ORC_MAX_N], z[ORC_MAX_N], y[ORC_MAX_N], mu[ORC_MAX_N], ze[ORC_MAX_N];
  for (int d = 0; d < n; ++d) xs[d] = x[d] + (drift ? drift[d] * tau : 0.0);
  if (tau <= 0.0) { /* sigma = 0: the kernel is a point mass, v = g(x) and Dv = Dg */
    *v = orc_target_g(P, xs);
    if (dv) orc_target_dg(P, xs, dv);
    if (diag) { diag[0] = diag[1] = *v; diag[2] = N; diag[3] = 0.0; diag[4] = -c * *v; diag[5] = 0.0; }
    if (se_dv) for (int d = 0; d < n; ++d) se_dv[d] = 0.0;
    return isfinite(*v) ? 0 : 2;
  }
  double sigma = sqrt(delta_eff(P) * tau);
  /* Proposal (R28). Plain: y ~ N(xs, sigma^2 I) as in Cor. logsumexp. Laplace-tilted:
   * y ~ N(mu, sigma^2 I), mu = xs - c sigma^2 Dg(xs) (one step toward the mode of
   * e^{-c g(y)} phi_sigma(y - xs)), each sample weighted by the likelihood ratio
   * phi_sigma(y - xs) / phi_sigma(y - mu), so E_q[e^{-cg} LR] = E_p[e^{-cg}] (same v, Dv). */
  if (P->proposal == 1) {
    double dg[ORC_MAX_N];
    orc_target_dg(P, xs, dg);
    for (int d = 0; d < n; ++d) mu[d] = xs[d] - c * sigma * sigma * dg[d];
  } else {
    for (int d = 0; d < n; ++d) mu[d] = xs[d];
  }
  double* a = (double*)malloc(sizeof(double) * (size_t)N);
  if (!a) return 1;
  /* pass 1: exponents a_i = -c g(y_i) + log LR_i */
  double gmin = INFINITY, gsum = 0.0, A = -INFINITY;
  for (uint32_t i = 0; i < N; ++i) {
    orc_sample_normals(P, qid, jw, kw, i, z, NULL);
    double r2x = 0.0, r2m = 0.0;
    for (int d = 0; d < n; ++d) {
      y[d] = mu[d] + sigma * z[d];
      r2x += (y[d] - xs[d]) * (y[d] - xs[d]);
      r2m += (y[d] - mu[d]) * (y[d] - mu[d]);
    }
    double g = orc_target_g(P, y);
    if (g < gmin) gmin = g;
    gsum += g;
    a[i] = -c * g - (r2x - r2m) / (2.0 * sigma * sigma);
    if (a[i] > A) A = a[i];
  }
  /* pass 2: S = sum exp(a_i - A), M = sum exp(a_i - A) (y_i - xs)/sigma */
  double S = 0.0, S2 = 0.0;
  double Mz[ORC_MAX_N], Mzz[ORC_MAX_N], Mz2[ORC_MAX_N];
  for (int d = 0; d < n; ++d) Mz[d] = Mzz[d] = Mz2[d] = 0.0;
  for (uint32_t i = 0; i < N; ++i) {
    orc_sample_normals(P, qid, jw, kw, i, z, NULL);
    for (int d = 0; d < n; ++d) ze[d] = z[d] + (mu[d] - xs[d]) / sigma;  /* (y_i - xs)/sigma */
    double w = exp(a[i] - A);
    S += w;
    S2 += w * w;
    for (int d = 0; d < n; ++d) {
      Mz[d] += w * ze[d];
      Mz2[d] += w * w * ze[d];
      Mzz[d] += w * w * ze[d] * ze[d];
    }
  }
  free(a);
  *v = -(A + log(S / (double)N)) / c;
  for (int d = 0; d < n; ++d) {
    double mu = Mz[d] / S;                       /* self-normalised E_w[z_d] */
    if (dv) dv[d] = -mu / (c * sigma);
    if (se_dv) {
      /* Var(sum w (z - mu) / sum w) ~ sum w^2 (z - mu)^2 / (sum w)^2 */
      double var = (Mzz[d] - 2.0 * mu * Mz2[d] + mu * mu * S2) / (S * S);
      se_dv[d] = sqrt(fmax(var, 0.0)) / (c * sigma);
    }
  }
  if (diag) {
    double ess = S * S / S2;
    double cv2 = (double)N * S2 / (S * S) - 1.0; /* Var(Z)/E[Z]^2 estimate */
    diag[0] = gmin;
    diag[1] = gsum / (double)N;
    diag[2] = ess;
    diag[3] = sqrt(fmax(cv2, 0.0) / (double)N) / c;
    diag[4] = A;
    diag[5] = log(S);
  }
  int ok = isfinite(*v);
  if (dv) for (int d = 0; d < n; ++d) ok = ok && isfinite(dv[d]);
  return ok ? 0 : 2;
}

/* Phi at a list of independent items (one per (query, horizon, frozen c)): item i evaluates
 * orc_phi at x[xi[i]] with global id qid[i], coefficient c[i], time-to-go tau[i] and counter
 * tags (jw[i], kw[i]); outputs v[i] and dv[i][n] (dv may be NULL). A plain loop over orc_phi
 * (OpenMP over items) — the teacher-forced parity tests use it to evaluate Phi at the oracle's
 * own coefficient history. Returns the last nonzero orc_phi status, else 0. */
int orc_phi_batch(const orc_problem* P, const float* x, const int64_t* xi, const uint32_t* qid,
                  const double* c, const double* tau, const uint32_t* jw, const uint32_t* kw,
                  int64_t count, double* v, double* dv, int32_t nthreads) {
  int status = 0;
  const int n = P->n;
#ifdef _OPENMP
  const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
  for (int64_t i = 0; i < count; ++i) {
    double xm[ORC_MAX_N];
    for (int d = 0; d < n; ++d) xm[d] = (double)x[xi[i] * n + d];
    int st = orc_phi(P, xm, NULL, qid[i], c[i], tau[i], jw[i], kw[i], &v[i],
                     dv ? dv + (size_t)i * (size_t)n : NULL, NULL, NULL);
    if (st) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
      status = st;
    }
  }
  return status;
}

/* ------------------------------------------------------------------------------------------
 * Algorithm 1 per query and horizon, then the running-min tube (R9).
 *   tau_j = j T / K (R9); v^(0) = g; c^(0) = Gamma(x, Dg);
 *   for k: freeze c^(k); (v^(k+1), Dv^(k+1)) = Phi(c^(k)); c^(k+1) = Gamma(x, Dv^(k+1)).
 * Outputs (each may be NULL): v, dv, c at tau_K after the last iterate (c = Gamma of the last
 * Dv); tube = min(g(x), min_j v_j); vhist/chist [K][Kp][M]; g0 [M]; dvhist [K][Kp][M][n] (the
 * Dv of every iterate, a diagnostic output for the tests).
 * Queries x arrive as the same fp32 array the GPU receives, converted to double (R22).
 * ---------------------------------------------------------------------------------------- */
int orc_solve_slice(const orc_problem* P, const float* x, const float* drift, const uint32_t* qid,
                    uint32_t qid_base, int64_t M, double* v, double* dv, double* c, double* tube,
                    double* vhist, double* chist, double* g0, double* dvhist, int32_t nthreads) {
  int n = P->n, K = P->K, Kp = P->Kp;
  double* vfinal = (double*)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1) * (size_t)(M > 0 ? M : 1));
  if (!vfinal) return 1;
  int status = 0;
  int64_t units = M * (int64_t)K;
#ifdef _OPENMP
  const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();  /* per call, not global */
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
  for (int64_t u = 0; u < units; ++u) {
    int64_t m = u / K;
    int j = (int)(u % K) + 1;
    double xm[ORC_MAX_N], bm[ORC_MAX_N], dgm[ORC_MAX_N], dvm[ORC_MAX_N];
    for (int d = 0; d < n; ++d) {
      xm[d] = (double)x[m * n + d];
      bm[d] = drift ? (double)drift[m * n + d] : 0.0;
    }
    uint32_t id = qid ? qid[m] : qid_base + (uint32_t)m;
    double tau = (double)j * P->T / (double)K;
    orc_target_dg(P, xm, dgm);
    double ck = orc_gamma(P, xm, dgm);
    double vk = 0.0;
    for (int k = 0; k < Kp; ++k) {
      uint32_t kw = P->crn ? 0u : (uint32_t)k;
      int st = orc_phi(P, xm, drift ? bm : NULL, id, ck, tau, (uint32_t)j, kw, &vk, dvm, NULL, NULL);
      if (st) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
        status = st;
      }
      size_t hi = ((size_t)(j - 1) * (size_t)Kp + (size_t)k) * (size_t)M + (size_t)m;
      if (vhist) vhist[hi] = vk;
      if (chist) chist[hi] = ck;
      if (dvhist) for (int d = 0; d < n; ++d) dvhist[hi * (size_t)n + d] = dvm[d];
      ck = orc_gamma(P, xm, dvm);
    }
    vfinal[(size_t)(j - 1) * (size_t)M + (size_t)m] = vk;
    if (j == K) {
      if (v) v[m] = vk;
      if (dv) for (int d = 0; d < n; ++d) dv[m * n + d] = dvm[d];
      if (c) c[m] = ck;
    }
  }
  for (int64_t m = 0; m < M; ++m) {
    double xm[ORC_MAX_N];
    for (int d = 0; d < n; ++d) xm[d] = (double)x[m * n + d];
    double gm = orc_target_g(P, xm);
    if (g0) g0[m] = gm;
    double t = gm;                                   /* running min incl. g */
    for (int j = 0; j < K; ++j) {
      double vj = vfinal[(size_t)j * (size_t)M + (size_t)m];
      if (vj < t) t = vj;
    }
    double l = orc_avoid_l(P, xm);                   /* BRAT clamp: max(tube, l) */
    if (l > t) t = l;
    if (tube) tube[m] = t;
  }
  free(vfinal);
  return status;
}

/* Algorithm 1 WITH its convergence test (step 5): for each horizon j, v^(0) = g,
 * c^(0) = Gamma(x, Dg); repeat for all queries: Phi at frozen c, then
 * eps = ||v^(k+1) - v^(k)||_2 / ||v^(k)||_2 over the M queries (R11), c <- Gamma(x, Dv);
 * stop when eps < tol or after max_iter passes. Outputs (caller-sized): v [K][M] (final
 * iterate), iters [K], eps and dsup [K][max_iter] (NAN after the stop; dsup = sup-norm of the
 * difference, Theorem 2's quantity). */
int orc_picard_adaptive(const orc_problem* P, const float* x, const uint32_t* qid,
                        uint32_t qid_base, int64_t M, double tol, int32_t max_iter, double* v_out,
                        double* iters, double* eps, double* dsup, int32_t nthreads) {
  int n = P->n, K = P->K;
  double* vprev = (double*)malloc(sizeof(double) * (size_t)M);
  double* vcur = (double*)malloc(sizeof(double) * (size_t)M);
  double* c = (double*)malloc(sizeof(double) * (size_t)M);
  if (!vprev || !vcur || !c) { free(vprev); free(vcur); free(c); return 1; }
  int status = 0;
#ifdef _OPENMP
  const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();  /* per call, not global */
#endif
  for (int j = 1; j <= K; ++j) {
    double tau = (double)j * P->T / (double)K;
    for (int64_t m = 0; m < M; ++m) {         /* v^(0) = g, c^(0) = Gamma(x, Dg) */
      double xm[ORC_MAX_N], dg[ORC_MAX_N];
      for (int d = 0; d < n; ++d) xm[d] = (double)x[m * n + d];
      vprev[m] = orc_target_g(P, xm);
      orc_target_dg(P, xm, dg);
      c[m] = orc_gamma(P, xm, dg);
    }
    for (int k = 0; k < max_iter; ++k) {
      eps[(size_t)(j - 1) * max_iter + k] = NAN;
      dsup[(size_t)(j - 1) * max_iter + k] = NAN;
    }
    int k;
    for (k = 0; k < max_iter; ++k) {
      uint32_t kw = P->crn ? 0u : (uint32_t)k;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
      for (int64_t m = 0; m < M; ++m) {
        double xm[ORC_MAX_N], dvm[ORC_MAX_N];
        for (int d = 0; d < n; ++d) xm[d] = (double)x[m * n + d];
        uint32_t id = qid ? qid[m] : qid_base + (uint32_t)m;
        int st = orc_phi(P, xm, NULL, id, c[m], tau, (uint32_t)j, kw, &vcur[m], dvm, NULL, NULL);
        if (st) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
          status = st;
        }
        c[m] = orc_gamma(P, xm, dvm);
      }
      double num = 0.0, den = 0.0, mx = 0.0;
      for (int64_t m = 0; m < M; ++m) {
        double d = vcur[m] - vprev[m];
        num += d * d;
        den += vprev[m] * vprev[m];
        if (fabs(d) > mx) mx = fabs(d);
        vprev[m] = vcur[m];
      }
      double e = sqrt(num / den);
      eps[(size_t)(j - 1) * max_iter + k] = e;
      dsup[(size_t)(j - 1) * max_iter + k] = mx;
      if (e < tol) { ++k; break; }
    }
    iters[j - 1] = (double)k;
    for (int64_t m = 0; m < M; ++m) v_out[(size_t)(j - 1) * M + m] = vprev[m];
  }
  free(vprev); free(vcur); free(c);
  return status;
}

/* Running-min reach tube of per-horizon final iterates with the BRAT clamp (
 * S:345): tube[m] = max( min( g(x_m), min_j vfinal[j][m] ), l(x_m) ), l = -inf
 * without an obstacle. x is the fp32 query array (converted to double), vfinal [K][M]. */
void orc_tube(const orc_problem* P, const float* x, int64_t M, const double* vfinal, double* tube) {
  int n = P->n, K = P->K;
  for (int64_t m = 0; m < M; ++m) {
    double xm[ORC_MAX_N];
    for (int d = 0; d < n; ++d) xm[d] = (double)x[m * n + d];
    double t = orc_target_g(P, xm);
    for (int j = 0; j < K; ++j) {
      double vj = vfinal[(size_t)j * (size_t)M + (size_t)m];
      if (vj < t) t = vj;
    }
    double l = orc_avoid_l(P, xm);
    if (l > t) t = l;
    tube[m] = t;
  }
}

/* Picard residual partial sums (relative L2 over the slice, R11), v^(0) = g. */
void orc_residual_partials(const double* vhist, const double* g0, int32_t K, int32_t Kp,
                           int64_t M, double* out) {
  for (int j = 0; j < K; ++j) {
    for (int k = 0; k < Kp; ++k) {
      double num = 0.0, den = 0.0;
      for (int64_t m = 0; m < M; ++m) {
        double prev = (k == 0) ? g0[m] : vhist[((size_t)j * Kp + (k - 1)) * M + m];
        double cur = vhist[((size_t)j * Kp + k) * M + m];
        num += (cur - prev) * (cur - prev);
        den += prev * prev;
      }
      out[((size_t)j * Kp + k) * 2 + 0] = num;
      out[((size_t)j * Kp + k) * 2 + 1] = den;
    }
  }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
