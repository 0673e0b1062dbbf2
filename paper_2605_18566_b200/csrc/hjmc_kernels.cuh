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
};

enum : int { kModeSolve = 0, kModeValueGrad = 1 };

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

struct KernelSet {
  SolveLauncher solve = nullptr;
  EvalLauncher eval_target = nullptr;
  int threads = 0;
};

// (target id, n) → compiled kernels; false if not instantiated.
bool lookup_kernels(int target, int n, KernelSet* out);

cudaError_t launch_tube(const float* g0, const float* vfinal, int K, int64_t M, float* tube,
                        cudaStream_t s);
cudaError_t launch_hamiltonian(const EvalParams& p, cudaStream_t s);
cudaError_t launch_debug_normals(int n, uint32_t qid, uint32_t jw, uint32_t kw, uint32_t i0,
                                 uint32_t count, const RoundKeys& rk, uint32_t tag, int antithetic, float* z,
                                 uint32_t* raw, cudaStream_t s);

}  // namespace hjmc
