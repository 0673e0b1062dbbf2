/*
 * hjmc_oracle.h — TEST INFRASTRUCTURE ONLY. Not part of the product.
 *
 * The plain, slow, double-precision CPU oracle for the Monte-Carlo frozen-coefficient
 * Cole–Hopf path of arxiv/paper_2605_18566. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. It shares no code, header,
 * constant or helper with the CUDA path (paper_2605_18566_b200/csrc, include/hjmc.h).
 *
 * Parity status per function (DESIGN.md §4 lists the pins):
 *   orc_philox4x32_10   pinned: bit-exact vs CUDA toolkit curand_Philox4x32_10 (library routine)
 *   orc_sample_normals  pinned: N(0,1) moments / KS vs scipy.stats.norm; antithetic exact; |z| bound
 *   orc_target_g/dg     pinned: closed-form values (distance, bowl), FD of g for Dg
 *   orc_hamiltonian     pinned: SPEC worked cases, 1-homogeneity, reductions
 *   orc_gamma           pinned: quadratic c = 1/δ_eff, clamp/floor cases
 *   orc_phi             pinned: constant/linear/quadratic closed forms, Gauss–Hermite and
 *                       noncentral-χ² quadrature, Jensen bounds, shift/translation identities
 *   orc_phi_batch       a plain OpenMP loop of orc_phi over independent items
 *   orc_solve_slice     pinned: quadratic CRN stationarity, tube ≤ g and ≤ every v_j,
 *                       per-sample BRT band bound; every step is orc_phi + orc_gamma; the MC
 *                       Picard reproduces a Gauss–Hermite-quadrature Picard on clamped queries
 *   orc_tube            pinned: tube ≤ g, ≤ every v_j, = max(·, ℓ) with an obstacle (same as solve_slice's)
 *   orc_avoid_l         pinned: BRAT clamp identities (disk obstacle)
 *   orc_picard_adaptive pinned: equals the fixed schedule at tol = 0, stops at the first
 *                       ε < tol (Algorithm 1 step 5); SPEC's contraction example
 *   orc_residual_partials  pinned: hand-computable small arrays
 *   (Laplace proposal mode of orc_phi) pinned: zero variance on linear g, closed form and ESS
 *                       gain on the quadratic bowl, agreement with the plain estimator
 * Parity unpinned: end-to-end BRT accuracy against the true inviscid value (needs grid
 * reference solutions the paper used, P:469 — not available).
 */
#ifndef HJMC_ORACLE_H_
#define HJMC_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Oracle-side identifiers (the tests map them to the library's). */
enum { ORC_SYS_QUADRATIC = 0, ORC_SYS_DUBINS_REL = 1, ORC_SYS_ROCKET6 = 2, ORC_SYS_DUBINS_PAIRS = 3,
       ORC_SYS_ROCKET3 = 4, ORC_SYS_DOUBLE_INTEGRATOR = 5, ORC_SYS_MULTIAGENT = 6 };
enum { ORC_TGT_QUAD_BOWL = 0, ORC_TGT_DISK = 1, ORC_TGT_REL_DISK6 = 2, ORC_TGT_PAIR_UNION = 3,
       ORC_TGT_LINEAR = 4, ORC_TGT_CONST = 5, ORC_TGT_PURSUIT_MIN = 6 };
enum { ORC_AVOID_NONE = 0, ORC_AVOID_DISK = 1 };

#define ORC_MAX_N 64
#define ORC_MAX_PARAMS 72

typedef struct orc_problem {
  int32_t n;
  double delta;
  double T;
  int32_t K;
  int32_t Kp;
  uint32_t N;
  uint64_t seed;
  int32_t full_laplacian;   /* 0: paper (δ/2)Δ, δ_eff = δ; 1: δΔ, δ_eff = 2δ */
  int32_t crn;
  int32_t antithetic;
  double m0;
  double c_min;
  double c_max;
  uint32_t tag;
  int32_t system;
  int32_t n_sys_params;
  double sys_params[8];
  int32_t target;
  int32_t n_tgt_params;
  double tgt_params[ORC_MAX_PARAMS];
  int32_t avoid;            /* BRAT obstacle: ORC_AVOID_* */
  double avoid_params[3];   /* disk: centre (x0, x1) and radius */
  int32_t proposal;         /* 0: plain N(x, sigma^2 I); 1: Laplace-tilted (R28) */
} orc_problem;

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void orc_sample_normals(const orc_problem* P, uint32_t qid, uint32_t jw, uint32_t kw, uint32_t i,
                        double* z, uint32_t* raw);
double orc_target_g(const orc_problem* P, const double* y);
double orc_avoid_l(const orc_problem* P, const double* x);
void orc_target_dg(const orc_problem* P, const double* x, double* dg);
double orc_hamiltonian(const orc_problem* P, const double* x, const double* p);
double orc_gamma(const orc_problem* P, const double* x, const double* p);
int orc_phi(const orc_problem* P, const double* x, const double* drift, uint32_t qid, double c,
            double tau, uint32_t jw, uint32_t kw, double* v, double* dv, double* diag,
            double* se_dv);
int orc_phi_batch(const orc_problem* P, const float* x, const int64_t* xi, const uint32_t* qid,
                  const double* c, const double* tau, const uint32_t* jw, const uint32_t* kw,
                  int64_t count, double* v, double* dv, int32_t nthreads);
int orc_solve_slice(const orc_problem* P, const float* x, const float* drift, const uint32_t* qid,
                    uint32_t qid_base, int64_t M, double* v, double* dv, double* c, double* tube,
                    double* vhist, double* chist, double* g0, double* dvhist, int32_t nthreads);
int orc_picard_adaptive(const orc_problem* P, const float* x, const uint32_t* qid,
                        uint32_t qid_base, int64_t M, double tol, int32_t max_iter, double* v_out,
                        double* iters, double* eps, double* dsup, int32_t nthreads);
void orc_tube(const orc_problem* P, const float* x, int64_t M, const double* vfinal, double* tube);
void orc_residual_partials(const double* vhist, const double* g0, int32_t K, int32_t Kp,
                           int64_t M, double* out);
int orc_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
