/*
 * hjmc.h — C-ABI of libhjmc: the B200 (sm_100a) hot path of arxiv/paper_2605_18566,
 * "Monte-Carlo frozen-coefficient Cole–Hopf solver for viscous HJ(I) reachability".
 *
 * Citation format: P:123 = /root/reference/PAPER.md line 123 (+ section / equation name).
 *                  S:45  = SPEC.md line 45 (interfaces / readings only).
 *                  R#    = reading # in DESIGN.md §3 (where the paper is silent or garbled).
 *
 * ----------------------------------------------------------------------------------------
 * WHAT THE LIBRARY COMPUTES (the contract both the CUDA path and the independent CPU oracle
 * implement; neither shares code with the other — this header is the CUDA side's only)
 * ----------------------------------------------------------------------------------------
 * Viscous HJ PDE  v_t + H(x, Dv) = (δ/2) Δv,  v(0,x) = g(x)                (Eq. HJ-Visc)
 * Frozen coefficient  c(x) = 2 H(x, Dv) / (δ |Dv|²)                        (Eq. coeff_frozen)
 * With c frozen per query, ω = exp(−c v) solves the heat equation, whose Gaussian solution
 * gives, for a query x, horizon-to-go τ and σ = sqrt(δ_eff τ):               (Prop. 1, Lemmas 2–3)
 *
 *   Φ pass (one Monte-Carlo evaluation at frozen c, Cor. logsumexp / mc_gradient):
 *     y_i = x + b τ + σ z_i,  z_i ~ N(0, I_n),  i = 0..N−1                  (b = optional drift, default 0; R4)
 *     v   = −(1/c) · log( (1/N) Σ_i exp(−c g(y_i)) )                        (Eq. logsumexp; R12 keeps 1/N)
 *     Dv  = −( Σ_i w_i z_i / Σ_i w_i ) / (c σ),  w_i = exp(−c g(y_i))       (Eq. mc_grad, rewritten; R2, R23)
 *   The GPU evaluates the log-sum-exp with a guaranteed-safe exponent shift;
 *   the result is the same number in exact arithmetic (R24).
 *
 *   Coefficient update Γ (Algorithm 1 step 4; P:336 map Γ; floors/clamps S:205–213, R8):
 *     p̃ = p · max(1, m0/|p|)  if p ≠ 0,   p̃ = m0 · e1  if p = 0
 *     c = clamp( 2 H(x, p̃) / (δ_eff |p̃|²), c_min, c_max )
 *
 *   Picard / horizon loop for one query (Algorithm 1; R9, R10):
 *     for j = 1..K:  τ_j = j T / K
 *       c ← Γ(x, Dg(x))                    (c^(0) from the analytic target gradient, R7)
 *       for k = 0..Kp−1:  (v, Dv) ← Φ_j(c);  vhist[j−1][k] = v;  chist[j−1][k] = c;  c ← Γ(x, Dv)
 *     tube = min( g(x), min_j vhist[j−1][Kp−1] )                           (running-min BRT, R9)
 *   Every query is independent of every other query (Γ and Φ are pointwise in m).
 *
 *   δ_eff = δ        for HJMC_VISC_PAPER_HALF_LAPLACIAN (the paper's (δ/2)Δ, canonical; R1)
 *   δ_eff = 2 δ      for HJMC_VISC_FULL_LAPLACIAN      (north_star's δΔ convention)
 *
 * ----------------------------------------------------------------------------------------
 * RANDOM NUMBERS (frozen bit-exactly; R19). Both sides generate them independently.
 * ----------------------------------------------------------------------------------------
 *  Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), identical to the CUDA toolkit's
 *  curand_Philox4x32_10(uint4 ctr, uint2 key):
 *    key   (k0, k1) = (seed & 0xffffffff, seed >> 32)
 *    round (c0,c1,c2,c3) → ( hi(M1·c2) ^ c1 ^ k0,  lo(M1·c2),  hi(M0·c0) ^ c3 ^ k1,  lo(M0·c0) )
 *          M0 = 0xD2511F53, M1 = 0xCD9E8D57; after each of the first 9 rounds
 *          k0 += 0x9E3779B9, k1 += 0xBB67AE85; the output (x0,x1,x2,x3) is the 10th round's.
 *  Draw layout (which Philox block feeds which normal): draw q = i (antithetic: q = i >> 1,
 *  odd i use −z). Let G = 4/gcd(n, 4) if G·n ≤ 16, else G = 1; Q = G·n/4 (G > 1) or ceil(n/4)
 *  (G = 1). Draw group γ = q / G has blocks b = 0..Q−1 whose Box–Muller outputs form one flat
 *  stream; draw q's normal d is stream element (q mod G)·n + d (G = 1: element d). Block b of
 *  group γ is Philox with counter
 *    c0 = γ,   c1 = b | (kw << 8) | (jw << 16),   c2 = global query id,   c3 = tag
 *         solve_slice: jw = j (1..K), kw = crn ? 0 : k (0..Kp−1);  value_grad: caller's tags
 *  (n = 2, 3, 6 thus use every normal a Philox call makes; the Q blocks of a group share the
 *  first Philox rounds, which depend on c0 but not on b.)
 *  Uniforms from a 32-bit word w:  m = w >> 9 (its high 23 bits);
 *    u(w) = (2m + 1) · 2^−24  ∈ (0, 1)       (radius argument, never 0 or 1)
 *    a(w) = m · 2^−23          ∈ [0, 1)       (angle fraction)
 *  Box–Muller, per block output (x0, x1, x2, x3) → stream elements 4t .. 4t+3 of the block's slot t:
 *    r = sqrt(−2 ln u(x0)):  ζ_{4t}   = r cos(2π a(x1)),  ζ_{4t+1} = r sin(2π a(x1))
 *    r'= sqrt(−2 ln u(x2)):  ζ_{4t+2} = r'cos(2π a(x3)),  ζ_{4t+3} = r'sin(2π a(x3))
 *  Hence |z_d| ≤ sqrt(48 ln 2) = 5.7683 for every coordinate.
 *
 * ----------------------------------------------------------------------------------------
 * SYSTEMS (H) AND TARGETS (g). Parameters are float arrays; np = 0 selects the defaults.
 * ----------------------------------------------------------------------------------------
 *  HJMC_SYS_QUADRATIC     any n    H = |p|²/2                                    (§2.1)
 *  HJMC_SYS_DUBINS_REL    n = 3    params {v_p, v_e, w} = {5, 5, 1}              (R13)
 *        H = p1 (v_p cos x3 − v_e) − p2 v_p sin x3 + w |p1 x2 − p2 x1 − p3| − w |p3|
 *  HJMC_SYS_ROCKET6       n = 6    params {a, g_grav, d_max} = {64, 32, 1}       (R15; a, g from P:1371)
 *        state (xP, zP, θP, xE, zE, θE);
 *        H = Σ_{v∈{P,E}} [ a (p_xv cos θv + p_zv sin θv) − g_grav p_zv ] − |p_θP| + |p_θE|
 *            + d_max · ‖(p_xE, p_zE)‖
 *  HJMC_SYS_DUBINS_PAIRS  n = 3K   params {v_p, v_e, w} = {5, 5, 1}              (R16)
 *        H = Σ_{q<K} H_DUBINS_REL(x[3q..3q+2], p[3q..3q+2])
 *  HJMC_SYS_ROCKET3       n = 3    params {a, g_grav} = {64, 32}        (R14)
 *        state (x, z, θ);  H = −[ a p1 cos θ + p2 (a + a sin θ − g) − |p1 x + p3| − |p2 x − p3| ]
 *  HJMC_SYS_DOUBLE_INTEGRATOR n = 2  no params
 *        H = p1 x2 − |p2|   (ẋ1 = x2, ẋ2 = u, |u| ≤ 1, u = −sign(p2))
 *  HJMC_SYS_MULTIAGENT    n = 3A   params {a_pursuer, a_evader} = {1, 1}
 *        agents (x_i, y_i, θ_i), ẋ = a cos θ, ẏ = a sin θ, θ̇ = u_i ∈ [−1, 1]; the last agent evades:
 *        H = Σ_i a_i (p_xi cos θ_i + p_yi sin θ_i) + |p_θ,A−1| − Σ_{i<A−1} |p_θi|
 *
 *  HJMC_TGT_QUAD_BOWL     any n    params {α0} = {0.25}:   g = |y|²/2 − α0        (config 1)
 *        Dg = x
 *  HJMC_TGT_DISK          n ≥ 2    params {r} = {5}:       g = sqrt(y0² + y1²) − r
 *        Dg = (x0, x1, 0..)/ρ, ρ = sqrt(x0² + x1²);  Dg = e1 at ρ = 0 (R7)
 *  HJMC_TGT_REL_DISK6     n = 6    params {r} = {1.5}:     g = sqrt((y0−y3)² + (y1−y4)²) − r  (R15)
 *        Dg = (Δx, Δz, 0, −Δx, −Δz, 0)/ρ;  e1 at ρ = 0
 *  HJMC_TGT_PAIR_UNION    n = 3K   params {r} = {1}:       g = sqrt(min_q (y_{3q}² + y_{3q+1}²)) − r  (R16)
 *        Dg = unit vector of the first minimising pair's position;  e1 at ρ = 0
 *  HJMC_TGT_PURSUIT_MIN   n = 3A   params {r} = {1.5}:  g = min_{i<A−1} ‖pos_i − pos_{A−1}‖ − r
 *        Dg = ±unit vector of the first minimising pursuer–evader pair;  e1 at ρ = 0
 *  HJMC_TGT_LINEAR        any n    params {a_0..a_{n−1}, b}: g = a·y + b,  Dg = a     (test target)
 *  HJMC_TGT_CONST         any n    params {k}:             g = k,  Dg = 0              (test target)
 *
 * Supported (target, n) kernel instantiations are listed by hjmc_supported(); any other
 * combination returns HJMC_EUNSUPPORTED from hjmc_set_target.
 *
 * ----------------------------------------------------------------------------------------
 * CONVENTIONS
 * ----------------------------------------------------------------------------------------
 *  * Every array argument is caller-owned; the library never frees or retains it beyond the
 *    call's stream order. "dev" pointers are CUDA device pointers on cfg.device; "host"
 *    pointers are ordinary host memory. Layouts are row-major, fp32 unless stated:
 *      x[M][n], dv[M][n], drift[M][n], v[M], c[M], tube[M], vhist[K][Kp][M], chist[K][Kp][M].
 *  * Device entry points are asynchronous on the given cudaStream_t (NULL = legacy default
 *    stream); they return only argument and launch errors. Numerical failures (a non-finite
 *    v or Dv) are recorded on the device and reported by hjmc_check(), which synchronises.
 *    With cfg.flags & HJMC_FLAG_SYNC_CHECK every device entry point synchronises and returns
 *    HJMC_ENUMERIC itself.
 *  * Results are a pure function of (config, system, target, x, drift, global query ids):
 *    independent of M, of how queries are split across calls or GPUs, and of the grid shape —
 *    bit for bit: the kernel variant (threads per (query, horizon) unit, hence the reduction
 *    order) is chosen from the configuration (N, n, target, antithetic, proposal) only.
 *  * A handle is not thread-safe; use one per host thread / stream. No C++ exception crosses
 *    the ABI. hjmc_last_error() returns a human-readable message for the last failure.
 */
#ifndef HJMC_H_
#define HJMC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define HJMC_API __attribute__((visibility("default")))
#else
#define HJMC_API
#endif

#define HJMC_VERSION_MAJOR 0
#define HJMC_VERSION_MINOR 2

/* Error codes (S:540 maps config errors to exit 2 and numeric errors to exit 3). */
#define HJMC_OK 0
#define HJMC_EINVAL 1          /* invalid argument or configuration                        */
#define HJMC_ENUMERIC 2        /* non-finite v or Dv at some query (see hjmc_last_bad_query) */
#define HJMC_ECUDA 3           /* CUDA runtime / launch failure                            */
#define HJMC_EUNSUPPORTED 4    /* (target, n) combination without a compiled kernel        */
#define HJMC_ENOMEM 5          /* device allocation of handle scratch failed               */

/* Viscosity convention (R1). */
#define HJMC_VISC_PAPER_HALF_LAPLACIAN 0
#define HJMC_VISC_FULL_LAPLACIAN 1

/* Config flags. */
#define HJMC_FLAG_SYNC_CHECK 1u
/* With crn = 1: when Γ returns exactly the coefficient just used, every remaining Picard iterate
 * of that (query, horizon) has bit-identical inputs and therefore bit-identical outputs; they
 * are copied instead of recomputed (Algorithm 1's convergence test at ε = 0, per query).
 * Outputs are identical with and without the flag; hjmc_pass_count() reports the work done. */
#define HJMC_FLAG_SKIP_STATIONARY 2u
/* With crn = 1: a Φ pass is a pure function of its frozen coefficient c (same samples; the
 * log-sum-exp shift and the proposal follow from c), so a pass whose c equals, bit for bit,
 * the c of an earlier pass of the same (query, horizon) reuses that pass's sums instead of
 * re-sampling (up to 8 distinct c per unit are kept). This shortcuts the Picard 2-cycles
 * between the clamps c_min ↔ c_max that dominate the game slices (R8, R27). Outputs are
 * identical with and without the flag; hjmc_pass_count() reports the sample passes run. */
#define HJMC_FLAG_REUSE_PASSES 4u
/* With HJMC_FLAG_REUSE_PASSES and crn = 1, for the game targets with n ≤ 16 or the n = 37–48
 * lane-group kernels, plain proposal, no antithetic
 * sampling: a pass whose frozen c sits on a clamp (c_min or c_max) also accumulates, from the
 * same samples, the sums at the opposite clamp and memoizes them (when they need no two-pass
 * fallback), so a c_min ↔ c_max Picard 2-cycle costs one sampling pass (C2 −16 %, C4 −22 %,
 * C5 −43 %); where units are stationary after one pass the extra sums go unused (≈ +4 %).
 * Outputs are identical with and without the flag; ignored where it does not apply. */
#define HJMC_FLAG_SPECULATE_CLAMPS 8u

/* Sampling proposal of a Φ pass (reading R28).
 *  PLAIN:   y_i = x + bτ + σ z_i — the estimator of Cor. logsumexp / mc_gradient.
 *  LAPLACE: y_i = μ + σ z_i with μ = x + bτ − c σ² Dg(x + bτ) (one step toward the mode of
 *           e^{−c g(y)} φ_σ(y − x − bτ)); each sample carries the likelihood ratio
 *           φ_σ(y − x − bτ)/φ_σ(y − μ), so v and Dv estimate the same quantities with lower
 *           variance where the weights concentrate (c‖g‖ ≫ 1). Exactly zero-variance
 *           for linear g. Dv = −E_W[(y − x − bτ)/σ]/(cσ). */
#define HJMC_PROPOSAL_PLAIN 0
#define HJMC_PROPOSAL_LAPLACE 1

/* Systems (Hamiltonians). */
#define HJMC_SYS_QUADRATIC 0
#define HJMC_SYS_DUBINS_REL 1
#define HJMC_SYS_ROCKET6 2
#define HJMC_SYS_DUBINS_PAIRS 3
#define HJMC_SYS_ROCKET3 4
#define HJMC_SYS_DOUBLE_INTEGRATOR 5
#define HJMC_SYS_MULTIAGENT 6

/* Targets (terminal costs g). */
#define HJMC_TGT_QUAD_BOWL 0
#define HJMC_TGT_DISK 1
#define HJMC_TGT_REL_DISK6 2
#define HJMC_TGT_PAIR_UNION 3
#define HJMC_TGT_LINEAR 4
#define HJMC_TGT_CONST 5
#define HJMC_TGT_PURSUIT_MIN 6

/* BRAT avoid sets. */
#define HJMC_AVOID_NONE 0
#define HJMC_AVOID_DISK 1

#define HJMC_MAX_N 64            /* state dimension limit of this build                    */
#define HJMC_MAX_PARAMS 72       /* max float parameters of a system or target             */

typedef struct hjmc_config {
  int32_t n;          /* state dimension, 1..HJMC_MAX_N                                       */
  float delta;        /* viscosity δ > 0                                               */
  float T;            /* horizon T > 0; τ_j = j T / K                                         */
  int32_t K;          /* horizons, 1..65535 (R9)                                              */
  int32_t Kp;         /* Picard iterates per horizon, ≥ 1 (≤ 256 when crn = 0)                */
  uint32_t N;         /* samples per query per Φ pass, 1..2^32−1 ("i.i.d. samples")     */
  uint64_t seed;      /* Philox key                                                           */
  int32_t visc;       /* HJMC_VISC_*                                                          */
  int32_t crn;        /* 1 = common random numbers across Picard iterates (R10, default)      */
  int32_t antithetic; /* 1 = samples in (z, −z) pairs                                  */
  float m0;           /* gradient floor, ≥ 0 (Assumption 1; S:248 default 1e−3)   */
  float c_min;        /* coefficient clamp, 0 < c_min ≤ c_max (S:248 defaults 0.05, 20)       */
  float c_max;
  uint32_t tag;       /* Philox counter word c3 (independent stream family)                   */
  int32_t device;     /* CUDA device ordinal                                                  */
  uint32_t flags;     /* HJMC_FLAG_*                                                          */
  int32_t proposal;   /* HJMC_PROPOSAL_* (default PLAIN)                                      */
} hjmc_config;

/* Outputs of hjmc_solve_slice. Every pointer may be NULL (= do not write). */
typedef struct hjmc_result {
  float* v;      /* [M]        v at τ_K after the last Picard iterate                         */
  float* dv;     /* [M][n]     Dv at τ_K after the last Picard iterate                        */
  float* c;      /* [M]        Γ(x, Dv) at τ_K: the coefficient the next iterate would freeze */
  float* tube;   /* [M]        min(g(x), min_j vhist[j][Kp−1])                                 */
  float* vhist;  /* [K][Kp][M] every Picard iterate's v                                       */
  float* chist;  /* [K][Kp][M] the frozen coefficient of every Picard iterate                 */
  float* g0;     /* [M]        g(x)                                                           */
} hjmc_result;

typedef struct hjmc_handle hjmc_handle;

/* Fill *cfg with the defaults: n=2, δ=0.05, T=0.5, K=1, Kp=1, N=4096, seed=0x5EED000000000001,
 * paper convention, crn=1, antithetic=0, m0=1e−3, c_min=0.05, c_max=20, tag=0, device=0, flags=0. */
HJMC_API void hjmc_config_defaults(hjmc_config* cfg);

/* Validate cfg (δ>0, T>0, 1≤n≤HJMC_MAX_N, K in 1..65535, Kp≥1 (≤256 if !crn), N≥1,
 * m0≥0, 0<c_min≤c_max, visc∈{0,1}) and create a handle on cfg->device.
 * Returns HJMC_EINVAL (no handle) or HJMC_ECUDA; *out is NULL on failure. */
HJMC_API int hjmc_create(const hjmc_config* cfg, hjmc_handle** out);

/* Release the handle's device scratch. Safe on NULL. Synchronises the device. */
HJMC_API void hjmc_destroy(hjmc_handle* h);

/* Select the Hamiltonian H (see SYSTEMS above). params: host pointer to np floats (np=0 →
 * defaults). HJMC_EINVAL if the id is unknown, np is wrong or n is incompatible. */
HJMC_API int hjmc_set_dynamics(hjmc_handle* h, int32_t system_id, const float* params, int32_t np);

/* Select the terminal cost g (see TARGETS above). HJMC_EUNSUPPORTED if no kernel exists for
 * (target, n); HJMC_EINVAL for a bad id / np / n. */
HJMC_API int hjmc_set_target(hjmc_handle* h, int32_t target_id, const float* params, int32_t np);

/* Reach–avoid (BRAT, Eq. HJI-RCBRAT-Visc): avoid function ℓ(x) > 0 inside the
 * obstacle; the tube becomes max(tube, ℓ(x)). HJMC_AVOID_DISK params
 * {c0, c1, r}: ℓ(x) = r − ‖(x0 − c0, x1 − c1)‖. HJMC_AVOID_NONE (default) restores the BRT. */
HJMC_API int hjmc_set_avoid(hjmc_handle* h, int32_t avoid_id, const float* params, int32_t np);

/* 1 if a kernel for (target_id, n) is compiled in, else 0. */
HJMC_API int hjmc_supported(int32_t target_id, int32_t n);

/* One Φ pass at frozen per-query coefficients (Thm 2's map Φ).
 *   x      dev [M][n]   query states
 *   c      dev [M]      frozen coefficients (> 0; used as given, not clamped)
 *   qid    dev [M] global query ids, or NULL → qid_base + m
 *   tau    horizon-to-go τ ≥ 0; τ = 0 returns v = g(x), Dv = Dg(x)
 *   j_tag  counter jw (≤ 65535), k_tag counter kw (≤ 255)
 *   drift  dev [M][n] or NULL (R4)
 *   v      dev [M] out;  dv dev [M][n] out or NULL
 * M = 0 is a no-op. Asynchronous on stream. */
HJMC_API int hjmc_value_grad(hjmc_handle* h, const float* x, const float* c, const uint32_t* qid,
                    uint32_t qid_base, int64_t M, float tau, uint32_t j_tag, uint32_t k_tag,
                    const float* drift, float* v, float* dv, void* stream);

/* The whole slice solve (a1–a11 of SURVEY §8(a)): K horizons × Kp Picard iterates and the
 * running-min tube, for M queries, in one fused kernel plus a tube epilogue kernel.
 *   x dev [M][n]; qid / qid_base as in hjmc_value_grad; drift dev [M][n] or NULL.
 *   out: device pointers (each may be NULL). M = 0 is a no-op. Asynchronous on stream. */
HJMC_API int hjmc_solve_slice(hjmc_handle* h, const float* x, const uint32_t* qid, uint32_t qid_base,
                     int64_t M, const float* drift, const hjmc_result* out, void* stream);

/* End-to-end convenience: the same solve with HOST buffers. Copies x (and qid, drift) to
 * handle-owned device scratch, solves, copies the requested outputs back to the HOST pointers in
 * *out_host, and synchronises. qid_host [M] (may be NULL → qid_base + m) gives explicit global
 * query ids, as in hjmc_solve_slice. Returns HJMC_ENUMERIC on a numerical failure. */
HJMC_API int hjmc_solve_slice_host(hjmc_handle* h, const float* x_host, const uint32_t* qid_host,
                          uint32_t qid_base, int64_t M, const float* drift_host,
                          const hjmc_result* out_host);

/* ---- Stepwise Picard: Algorithm 1 with its convergence test (step 5) ------------
 * The fused solve runs a fixed Kp. Algorithm 1 instead stops when
 *   ε_j(k) = ‖v^(k+1) − v^(k)‖₂ / ‖v^(k)‖₂ < ε     (norms over the slice's queries, R11),
 * a slice-wide (and, sharded, cross-GPU) quantity. The caller drives it:
 *   hjmc_picard_begin  — v^(0) = g(x), c^(0) = Γ(x, Dg(x)) for every horizon (handle state);
 *                        x / qid / drift must stay valid until the last pass.
 *   hjmc_picard_pass   — one Φ pass (iterate k) for every horizon with active[j] != 0 (NULL =
 *                        all): v (dev [K][M]), dv (dev [K][M][n]) and c (dev [K][M], the
 *                        updated Γ(x, Dv)) are written for active rows (each may be NULL);
 *                        partials (HOST [K][3]) receives per horizon (Σ(v^(k+1)−v^(k))²,
 *                        Σ(v^(k))², max|v^(k+1)−v^(k)|) over this handle's queries, zeros for
 *                        inactive horizons. Synchronises the stream. Sum the first two and take
 *                        the max of the third across shards, then ε_j(k) = sqrt(num/den) and
 *                        Theorem 2's sup-norm differences. Iterates run with the
 *                        same counters as hjmc_solve_slice, so with every horizon active for
 *                        Kp passes the v rows equal vhist[·][k] bit for bit. */
HJMC_API int hjmc_picard_begin(hjmc_handle* h, const float* x, const uint32_t* qid,
                               uint32_t qid_base, int64_t M, const float* drift, void* stream);
HJMC_API int hjmc_picard_pass(hjmc_handle* h, int32_t k, const uint8_t* active, float* v,
                              float* dv, float* c, double* partials, void* stream);

/* Algorithm 1's stopping test (step 5) on residual partials that the caller has already
 * combined across shards (HOST partials [K][3]: Σ(v^(k+1)−v^(k))², Σ(v^(k))² summed, max
 * |v^(k+1)−v^(k)| maxed — one all-reduce): for every horizon j with active[j] != 0,
 *   ε_j = sqrt(Σ(v^(k+1)−v^(k))² / max(Σ(v^(k))², 1e-300))   (relative L2, R11)
 * is written to eps[j] and the sup-norm difference to dsup[j] (Theorem 2's d_k, P:346–360;
 * NaN for inactive horizons; either may be NULL), and horizon j is retired (active[j] = 0)
 * when ε_j < tol. *n_active (may be NULL) receives the horizons still active. The same double
 * expression as the decision kernel of hjmc_picard_solve, so a host-driven (e.g. sharded) loop
 * takes identical decisions. Host-only, no handle; EINVAL for K < 1, tol < 0 or NULL
 * partials / active. */
HJMC_API int hjmc_picard_decide(const double* partials, int32_t K, double tol, uint8_t* active,
                                double* eps, double* dsup, int32_t* n_active);

/* Algorithm 1 with its stopping test for a SHARDED slice, device-resident (no host round trip
 * per iterate): the caller enqueues, on one stream, hjmc_picard_dev_begin once and then
 * max_iter times { hjmc_picard_dev_pass; an all-reduce of `reduced` across the shards — rows 0–1
 * summed, row 2 maxed (e.g. NCCL through torch.distributed, or nothing for one process);
 * hjmc_picard_dev_decide } — the sequence can be captured into one CUDA graph.
 *   dev_begin  — v^(0) = g, c^(0) = Γ(x, Dg) for every horizon, all horizons active, k = 0,
 *                iters [K] = 0, eps / dsup [K][max_iter] = NaN (device outputs). x / qid /
 *                drift must stay valid until the last call.
 *   dev_pass   — one Φ pass of every still-active horizon (retired horizons' units exit at
 *                once), v (dev [K][M], required), dv ([K][M][n]) and c ([K][M]) as
 *                hjmc_picard_pass writes them, and reduced (dev double [3][K]) = this
 *                handle's (Σ(v^(k+1)−v^(k))², Σ(v^(k))², max|v^(k+1)−v^(k)|) per horizon,
 *                zeros for retired ones. No synchronisation, no allocation (capturable).
 *   dev_decide — Algorithm 1 step 5 on the (all-reduced) reduced partials, the same
 *                double expression as hjmc_picard_solve's decision kernel: records ε_j(k), the
 *                sup-norm difference and the iterate count of every active horizon, retires it
 *                when ε_j(k) < tol, advances k; a no-op past max_iter. Capturable.
 * With one process (no all-reduce) the results equal hjmc_picard_solve bit for bit. */
HJMC_API int hjmc_picard_dev_begin(hjmc_handle* h, const float* x, const uint32_t* qid,
                                   uint32_t qid_base, int64_t M, const float* drift,
                                   int32_t max_iter, int32_t* iters, double* eps, double* dsup,
                                   void* stream);
HJMC_API int hjmc_picard_dev_pass(hjmc_handle* h, float* v, float* dv, float* c, double* reduced,
                                  void* stream);
HJMC_API int hjmc_picard_dev_decide(hjmc_handle* h, const double* reduced, double tol,
                                    int32_t* iters, double* eps, double* dsup, void* stream);

/* Theorem 2's contraction constant (Eq. contraction_const; R18 reads 2G/c_min):
 *   q = (2G/c_min) · (2 L_D/δ) · (L_H/m0² + 2 H_star P_star / m0⁴).  Host-only, no handle. */
HJMC_API double hjmc_contraction_constant(double G, double c_min, double L_D, double delta, double L_H,
                                          double m0, double H_star, double P_star);

/* Theorem 2 diagnostics from the sup-norm Picard differences d[0..count−1]
 * (d_k = ‖v^(k+1) − v^(k)‖∞, e.g. hjmc_picard_solve's dsup row): q_hat[k] = d[k+1]/d[k] for
 * k < count − 1 (IEEE division: 0/0 = NaN, x/0 = ±inf); when 0 ≤ q < 1 the a-posteriori bound
 * apost[k] = q/(1−q)·d[k] on ‖v^(k+1) − v*‖∞ (Eq. aposteriori-error) is written
 * and 1 is returned (certified), else apost is untouched and 0 is returned. q_hat / apost may
 * be NULL; −1 (EINVAL-like) for count < 0 or NULL d with count > 0. Host-only. */
HJMC_API int hjmc_contraction_report(const double* d, int64_t count, double q, double* q_hat,
                                     double* apost);

/* Post-hoc residuals (a12; R11) from summed partials (HOST [count][2] = (num, den), e.g.
 * hjmc_residual_partials all-reduced over shards): eps[i] = sqrt(num / max(den, 1e-300)). */
HJMC_API int hjmc_residual_eps(const double* partials, int64_t count, double* eps);

/* The running-min reach tube of per-horizon final iterates, with the BRAT clamp when
 * hjmc_set_avoid installed an obstacle:
 *   tube[m] = max( min( g(x_m), min_j vfinal[j][m] ), ℓ(x_m) )
 * x [M][n], vfinal [K][M] (e.g. the v output of hjmc_picard_pass / hjmc_picard_solve), tube [M]:
 * device pointers, stream-ordered. g(x) goes through handle scratch. */
HJMC_API int hjmc_tube(hjmc_handle* h, const float* x, int64_t M, const float* vfinal, float* tube,
                       void* stream);

/* Algorithm 1 with its stopping test (iterate until ε_j(k) < tol, step 5), for every
 * horizon, entirely on the device: hjmc_picard_begin, then one CUDA graph whose conditional
 * 'while' node repeats {Φ pass of the still-active horizons, residual partials, decision} —
 * the decision kernel computes ε_j(k) = sqrt(Σ(v^(k+1)−v^(k))² / Σ(v^(k))²) over this handle's
 * queries (R11; single process — sharded slices use hjmc_picard_pass and an all-reduce),
 * retires horizon j when ε_j(k) < tol, and stops the loop when none is left or after max_iter
 * passes. Outputs (device): v [K][M], dv [K][M][n] (may be NULL), c [K][M] (may be NULL) of each
 * horizon's final iterate; iters [K] (int32) passes run per horizon; eps, dsup [K][max_iter]
 * (double) ε_j(k) and max_m |v^(k+1) − v^(k)|, NaN past the stop; tube [M] (may be NULL) the
 * running-min tube over the horizons' final iterates with the BRAT clamp, exactly hjmc_tube's
 * (P:194–210), formed inside the same graph after the loop. Same kernels, counters and
 * reduction order as hjmc_picard_pass driven from the host: identical results. Stream-ordered
 * (asynchronous): one graph launch on stream; the instantiated graph is cached in the handle and
 * reused while the arguments and the handle's dynamics / target / avoid set are unchanged.
 * x, qid, drift and the outputs must stay valid until the stream reaches the launch.
 * EINVAL for M < 1, max_iter < 1, tol < 0 or missing outputs. */
HJMC_API int hjmc_picard_solve(hjmc_handle* h, const float* x, const uint32_t* qid,
                               uint32_t qid_base, int64_t M, const float* drift, double tol,
                               int32_t max_iter, float* v, float* dv, float* c, int32_t* iters,
                               double* eps, double* dsup, float* tube, void* stream);

/* g(x) and the analytic Dg(x) used for c^(0) (dev pointers; dg may be NULL). */
HJMC_API int hjmc_eval_target(hjmc_handle* h, const float* x, int64_t M, float* g, float* dg,
                     void* stream);

/* H(x, p) and Γ(x, p) per query (dev pointers; either output may be NULL). */
HJMC_API int hjmc_eval_hamiltonian(hjmc_handle* h, const float* x, const float* p, int64_t M,
                          float* H, float* c, void* stream);

/* The sampled normals exactly as the kernels generate them, for RNG parity tests:
 * z[s][n] (dev) for samples i = i0 .. i0+count−1 of query qid with counter tags (jw, kw);
 * raw[s][4·(ceil(n/4)+1)] (dev, may be NULL) receives the words of every Philox block the
 * sample touches, in order (unused tail entries untouched). Antithetic sign applies. */
HJMC_API int hjmc_debug_normals(hjmc_handle* h, uint32_t qid, uint32_t jw, uint32_t kw, uint32_t i0,
                       uint32_t count, float* z, uint32_t* raw, void* stream);

/* Synchronise stream, then return HJMC_ENUMERIC if any earlier call on this handle produced
 * a non-finite value (clearing the flag), else HJMC_OK. */
HJMC_API int hjmc_check(hjmc_handle* h, void* stream);

/* Number of Φ passes (each N samples of one query) the device executed since the previous call
 * (synchronises stream). Without HJMC_FLAG_SKIP_STATIONARY / HJMC_FLAG_REUSE_PASSES a
 * solve_slice executes M·K·Kp. */
HJMC_API int hjmc_pass_count(hjmc_handle* h, void* stream, uint64_t* passes);

/* Smallest global query id that failed numerically since the last hjmc_check, or −1. */
HJMC_API int64_t hjmc_last_bad_query(const hjmc_handle* h);

/* Message of the last failure on this handle (or of the last failed hjmc_create if h is NULL). */
HJMC_API const char* hjmc_last_error(const hjmc_handle* h);

/* Host-side Picard residual partial sums (a12; R11). For each (j, k):
 *   num[j][k] = Σ_m (v^(k+1)_m − v^(k)_m)²,  den[j][k] = Σ_m (v^(k)_m)²,
 * with v^(0) = g0 (Algorithm 1 init v^(0) = g) and v^(k+1) = vhist[j][k].
 * Host pointers: vhist [K][Kp][M], g0 [M], out [K][Kp][2] (num, den) in double.
 * ε_j(k) = sqrt(num/den) after summing partials over shards. */
HJMC_API int hjmc_residual_partials(const float* vhist, const float* g0, int32_t K, int32_t Kp, int64_t M,
                           double* out);

/* Library version as MAJOR*1000 + MINOR. */
HJMC_API int hjmc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HJMC_H_ */
