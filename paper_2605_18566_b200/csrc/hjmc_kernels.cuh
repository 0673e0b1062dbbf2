// hjmc_kernels.cuh — internal interface between the C-ABI layer and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "hjmc_rng.cuh"
#include "hjmc_systems.cuh"
#include "hjmc_targets.cuh"

namespace hjmc {

struct SolveParams {
  const float* x;          // [M][n]
  const float* drift;      // [M][n] or null
  const uint32_t* qid;     // [M] or null
  uint32_t qid_base;
  int64_t M;
  int K, Kp;
  double T;
  int mode;                // kModeSolve / kModeValueGrad
  const float* c_in;       // value_grad: [M]
  double tau_vg;           // value_grad: τ
  uint32_t jtag, ktag;     // value_grad: counter tags
  uint32_t N;
  RoundKeys rk;            // Philox round keys of cfg.seed
  uint32_t tag;
  int crn, antithetic;
  int proposal;            // HJMC_PROPOSAL_* (R28)
  GammaParams gp;
  SystemParams sp;
  TargetParams tp;
  // outputs (nullable)
  float* v;
  float* dv;
  float* c_out;
  float* vhist;
  float* chist;
  float* vfinal;           // [K][M] scratch for the tube epilogue
  float* g0;
  int* err;
  unsigned long long* bad;
  int skip_stationary;             // HJMC_FLAG_SKIP_STATIONARY
  int reuse_passes;                // HJMC_FLAG_REUSE_PASSES
  int speculate;                   // HJMC_FLAG_SPECULATE_CLAMPS
  unsigned long long* passes;      // Φ passes executed (accounting), nullable
  // stepwise Picard (kModePass): one pass per (query, active horizon)
  double* c_state;                 // [K][M] frozen coefficient in, Γ(x, Dv) out
  const int* active_j;             // [n_active] 1-based horizon indices (device)
  int n_active;
  int kiter;                       // Picard iterate index (counter word when crn = 0)
  // device-resident Algorithm 1 (hjmc_picard_solve): per-horizon activity mask [K] and the
  // iterate index read on the device (graph launches cannot change kernel arguments)
  const int* active_mask;
  const int* kiter_dev;
};

enum : int { kModeSolve = 0, kModeValueGrad = 1, kModePass = 2 };

struct PicardInitParams {
  const float* x;
  int64_t M;
  int K;
  double* c_state;                 // [K][M] ← Γ(x, Dg(x))
  float* v_prev;                   // [K][M] ← g(x)  (Algorithm 1: v^(0) = g)
  float* g0;                       // [M] ← g(x) for the tube epilogue (nullable)
  GammaParams gp;
  SystemParams sp;
  TargetParams tp;
};

struct EvalParams {
  const float* x;
  const float* p;
  int64_t M;
  float* g;
  float* dg;
  float* H;
  float* c;
  GammaParams gp;
  SystemParams sp;
  TargetParams tp;
};

using SolveLauncher = cudaError_t (*)(const SolveParams&, int64_t units, cudaStream_t);
using EvalLauncher = cudaError_t (*)(const EvalParams&, cudaStream_t);
using PicardInitLauncher = cudaError_t (*)(const PicardInitParams&, cudaStream_t);

struct KernelSet {
  SolveLauncher solve = nullptr;
  EvalLauncher eval_target = nullptr;
  PicardInitLauncher picard_init = nullptr;
  int threads = 0;
};

// (target id, n) → compiled kernels; false if not instantiated.
bool lookup_kernels(int target, int n, KernelSet* out);

// BRAT avoid set: type 0 none, 1 disk {c0, c1, r}: ℓ(x) = r − ‖(x0 − c0, x1 − c1)‖.
struct AvoidParams {
  int type;
  float p[3];
};

// tube[m] = max(min(g0[m], min_j vfinal[j][m]), ℓ(x_m))  (running-min BRT; BRAT clamp)
cudaError_t launch_tube(const float* g0, const float* vfinal, int K, int64_t M, float* tube,
                        const float* x, int n, AvoidParams avoid, cudaStream_t s);
cudaError_t launch_hamiltonian(const EvalParams& p, cudaStream_t s);
// Per active horizon a (grid y) and block b (grid x): partial[a][b] = (Σ (v−v_prev)², Σ v_prev²,
// max |v−v_prev|) over that block's queries; then v_prev ← v. Deterministic (fixed order).
cudaError_t launch_picard_residual(const float* v, float* v_prev, int64_t M, const int* active_j,
                                   int n_active, double* partial, int blocks, cudaStream_t s);
// Algorithm 1's stopping test on the device (hjmc_picard_solve): per active horizon j sum the
// residual partials in fixed block order, ε_j(k) = sqrt(num / max(den, 1e-300)) (R11),
// record ε, the sup-norm difference and the iterate count, retire j when ε < tol, advance k,
// and set the graph's while-condition to (any horizon active && k < max_iter).
cudaError_t launch_picard_decide(const double* partial, int K, int blocks, double tol,
                                 int max_iter, int* mask, int* kiter, int* iters, double* eps,
                                 double* dsup, cudaGraphConditionalHandle cond, cudaStream_t s);
// Sharded device-resident Algorithm 1: per-horizon block sums → reduced [3][K] (zeros for retired
// horizons), and the stopping test on (all-reduced) reduced partials (no conditional node).
cudaError_t launch_picard_blocksum(const double* partial, int K, int blocks, const int* mask,
                                   double* reduced, cudaStream_t s);
cudaError_t launch_picard_decide_reduced(const double* reduced, int K, double tol, int max_iter,
                                         int* mask, int* kiter, int* iters, double* eps,
                                         double* dsup, cudaStream_t s);
// Loop state for hjmc_picard_solve: horizons 1..K, all active, k = 0, iters = 0, NaN histories.
cudaError_t launch_picard_solve_init(int* state, int K, int32_t* iters, double* eps,
                                     double* dsup, int max_iter, cudaStream_t s);
cudaError_t launch_debug_normals(int n, uint32_t qid, uint32_t jw, uint32_t kw, uint32_t i0,
                                 uint32_t count, const RoundKeys& rk, uint32_t tag, int antithetic, float* z,
                                 uint32_t* raw, cudaStream_t s);

}  // namespace hjmc
