// hjmc_api.cu — the C-ABI of libhjmc (include/hjmc.h): validation, handle-owned scratch,
// launch orchestration and error reporting. No C++ exception crosses the boundary.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <algorithm>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hjmc.h"
#include "hjmc_kernels.cuh"

using namespace hjmc;

namespace {
// NVTX range over one C-ABI call (header-only NVTX v3: a no-op unless a profiler injects it), so
// nsys / ncu --nvtx timelines attribute kernels to the library entry point that launched them.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct hjmc_handle {
  hjmc_config cfg{};
  bool sys_set = false;
  bool tgt_set = false;
  SystemParams sp{};
  TargetParams tp{};
  int tgt_id = -1;
  AvoidParams avoid{};
  KernelSet ks{};
  int* d_err = nullptr;
  unsigned long long* d_bad = nullptr;
  unsigned long long* d_passes = nullptr;
  float* d_g0 = nullptr;
  size_t g0_cap = 0;
  float* d_vfinal = nullptr;
  size_t vfinal_cap = 0;
  // host-path staging
  float* d_stage = nullptr;
  size_t stage_cap = 0;
  cudaStream_t host_stream = nullptr;
  // stepwise Picard state (hjmc_picard_begin / hjmc_picard_pass)
  const float* pic_x = nullptr;
  const uint32_t* pic_qid = nullptr;
  const float* pic_drift = nullptr;
  uint32_t pic_qid_base = 0;
  int64_t pic_M = -1;
  double* d_cstate = nullptr;
  size_t cstate_cap = 0;
  float* d_vprev = nullptr;
  size_t vprev_cap = 0;
  float* d_vtmp = nullptr;
  size_t vtmp_cap = 0;
  int* d_active = nullptr;
  double* d_partial = nullptr;
  size_t partial_cap = 0;
  int64_t last_bad = -1;
  std::string err;
  // device-resident Algorithm 1 (hjmc_picard_solve): the instantiated graph, reused while the
  // call's arguments and the handle's problem (generation) are unchanged
  unsigned generation = 0;
  int* d_pstate = nullptr;          // [K] horizons 1..K, [K] activity mask, [1] iterate counter
  cudaGraph_t pic_graph = nullptr;
  cudaGraphExec_t pic_exec = nullptr;
  std::vector<uintptr_t> pic_key;
  // sharded device-resident Algorithm 1 (hjmc_picard_dev_*)
  int pic_dev_max_iter = 0;
  int pic_dev_blocks = 0;
};

namespace {

thread_local std::string g_create_error;

int fail(hjmc_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg; else g_create_error = msg;
  return code;
}

int cuda_fail(hjmc_handle* h, cudaError_t e, const char* where) {
  return fail(h, HJMC_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int ensure(hjmc_handle* h, float** buf, size_t* cap, size_t elems) {
  if (elems <= *cap && *buf) return HJMC_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc((void**)buf, elems * sizeof(float));
  if (e != cudaSuccess) {
    *buf = nullptr;
    return fail(h, HJMC_ENOMEM, std::string("scratch allocation failed: ") + cudaGetErrorString(e));
  }
  *cap = elems;
  return HJMC_OK;
}

int set_device(hjmc_handle* h) {
  cudaError_t e = cudaSetDevice(h->cfg.device);
  return e == cudaSuccess ? HJMC_OK : cuda_fail(h, e, "cudaSetDevice");
}

double delta_eff(const hjmc_config& c) {
  return c.visc == HJMC_VISC_FULL_LAPLACIAN ? 2.0 * (double)c.delta : (double)c.delta;
}

void fill_common(const hjmc_handle* h, SolveParams* p) {
  std::memset(p, 0, sizeof(*p));
  p->N = h->cfg.N;
  make_round_keys(h->cfg.seed, &p->rk);
  p->tag = h->cfg.tag;
  p->crn = h->cfg.crn;
  p->antithetic = h->cfg.antithetic;
  p->proposal = h->cfg.proposal;
  p->gp.delta_eff = delta_eff(h->cfg);
  p->gp.m0 = h->cfg.m0;
  p->gp.c_min = h->cfg.c_min;
  p->gp.c_max = h->cfg.c_max;
  p->sp = h->sp;
  p->tp = h->tp;
  p->err = h->d_err;
  p->bad = h->d_bad;
  p->skip_stationary = (h->cfg.flags & HJMC_FLAG_SKIP_STATIONARY) ? 1 : 0;
  p->reuse_passes = (h->cfg.flags & HJMC_FLAG_REUSE_PASSES) ? 1 : 0;
  p->speculate = (h->cfg.flags & HJMC_FLAG_SPECULATE_CLAMPS) ? 1 : 0;
  p->passes = h->d_passes;
}

int ready(hjmc_handle* h) {
  if (!h) return HJMC_EINVAL;
  if (!h->sys_set) return fail(h, HJMC_EINVAL, "hjmc_set_dynamics has not been called");
  if (!h->tgt_set) return fail(h, HJMC_EINVAL, "hjmc_set_target has not been called");
  return HJMC_OK;
}

int sync_check_if_requested(hjmc_handle* h, cudaStream_t s) {
  if (h->cfg.flags & HJMC_FLAG_SYNC_CHECK) return hjmc_check(h, (void*)s);
  return HJMC_OK;
}

}  // namespace

extern "C" {

void hjmc_config_defaults(hjmc_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->n = 2;
  c->delta = 0.05f;
  c->T = 0.5f;
  c->K = 1;
  c->Kp = 1;
  c->N = 4096;
  c->seed = 0x5EED000000000001ull;
  c->visc = HJMC_VISC_PAPER_HALF_LAPLACIAN;
  c->crn = 1;
  c->antithetic = 0;
  c->m0 = 1e-3f;
  c->c_min = 0.05f;
  c->c_max = 20.0f;
  c->tag = 0;
  c->device = 0;
  c->flags = 0;
  c->proposal = HJMC_PROPOSAL_PLAIN;
}

int hjmc_version(void) { return HJMC_VERSION_MAJOR * 1000 + HJMC_VERSION_MINOR; }

int hjmc_create(const hjmc_config* cfg, hjmc_handle** out) {
  if (!out) return fail(nullptr, HJMC_EINVAL, "out is NULL");
  *out = nullptr;
  if (!cfg) return fail(nullptr, HJMC_EINVAL, "cfg is NULL");
  const hjmc_config& c = *cfg;
  if (c.n < 1 || c.n > HJMC_MAX_N) return fail(nullptr, HJMC_EINVAL, "n must be in 1..64");
  if (!(c.delta > 0.f) || !std::isfinite(c.delta)) return fail(nullptr, HJMC_EINVAL, "delta must be > 0");
  if (!(c.T > 0.f) || !std::isfinite(c.T)) return fail(nullptr, HJMC_EINVAL, "T must be > 0");
  if (c.K < 1 || c.K > 65535) return fail(nullptr, HJMC_EINVAL, "K must be in 1..65535");
  if (c.Kp < 1) return fail(nullptr, HJMC_EINVAL, "Kp must be >= 1");
  if (!c.crn && c.Kp > 256) return fail(nullptr, HJMC_EINVAL, "Kp must be <= 256 without crn");
  if (c.N < 1) return fail(nullptr, HJMC_EINVAL, "N must be >= 1");
  if (!(c.m0 >= 0.f)) return fail(nullptr, HJMC_EINVAL, "m0 must be >= 0");
  if (!(c.c_min > 0.f) || !(c.c_min <= c.c_max) || !std::isfinite(c.c_max))
    return fail(nullptr, HJMC_EINVAL, "need 0 < c_min <= c_max");
  if (c.visc != HJMC_VISC_PAPER_HALF_LAPLACIAN && c.visc != HJMC_VISC_FULL_LAPLACIAN)
    return fail(nullptr, HJMC_EINVAL, "visc must be 0 or 1");
  if (c.crn != 0 && c.crn != 1) return fail(nullptr, HJMC_EINVAL, "crn must be 0 or 1");
  if (c.antithetic != 0 && c.antithetic != 1) return fail(nullptr, HJMC_EINVAL, "antithetic must be 0 or 1");
  if (c.proposal != HJMC_PROPOSAL_PLAIN && c.proposal != HJMC_PROPOSAL_LAPLACE)
    return fail(nullptr, HJMC_EINVAL, "proposal must be PLAIN or LAPLACE");
  if (c.flags & ~(HJMC_FLAG_SYNC_CHECK | HJMC_FLAG_SKIP_STATIONARY | HJMC_FLAG_REUSE_PASSES |
                  HJMC_FLAG_SPECULATE_CLAMPS))
    return fail(nullptr, HJMC_EINVAL, "unknown flag bits");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return fail(nullptr, HJMC_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (c.device < 0 || c.device >= ndev) return fail(nullptr, HJMC_EINVAL, "device ordinal out of range");
  hjmc_handle* h = new (std::nothrow) hjmc_handle();
  if (!h) return fail(nullptr, HJMC_ENOMEM, "host allocation failed");
  h->cfg = c;
  if ((e = cudaSetDevice(c.device)) != cudaSuccess ||
      (e = cudaMalloc((void**)&h->d_err, sizeof(int))) != cudaSuccess ||
      (e = cudaMalloc((void**)&h->d_bad, sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaMemset(h->d_err, 0, sizeof(int))) != cudaSuccess ||
      (e = cudaMemset(h->d_bad, 0xFF, sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaMalloc((void**)&h->d_passes, sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaMemset(h->d_passes, 0, sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&h->host_stream, cudaStreamNonBlocking)) != cudaSuccess) {
    std::string msg = std::string("device setup failed: ") + cudaGetErrorString(e);
    hjmc_destroy(h);
    return fail(nullptr, HJMC_ECUDA, msg);
  }
  *out = h;
  return HJMC_OK;
}

void hjmc_destroy(hjmc_handle* h) {
  if (!h) return;
  cudaSetDevice(h->cfg.device);
  cudaDeviceSynchronize();
  if (h->d_err) cudaFree(h->d_err);
  if (h->d_bad) cudaFree(h->d_bad);
  if (h->d_passes) cudaFree(h->d_passes);
  if (h->d_g0) cudaFree(h->d_g0);
  if (h->d_vfinal) cudaFree(h->d_vfinal);
  if (h->d_stage) cudaFree(h->d_stage);
  if (h->d_cstate) cudaFree(h->d_cstate);
  if (h->d_vprev) cudaFree(h->d_vprev);
  if (h->d_vtmp) cudaFree(h->d_vtmp);
  if (h->d_active) cudaFree(h->d_active);
  if (h->d_partial) cudaFree(h->d_partial);
  if (h->pic_exec) cudaGraphExecDestroy(h->pic_exec);
  if (h->pic_graph) cudaGraphDestroy(h->pic_graph);
  if (h->d_pstate) cudaFree(h->d_pstate);
  if (h->host_stream) cudaStreamDestroy(h->host_stream);
  delete h;
}

int hjmc_set_dynamics(hjmc_handle* h, int32_t id, const float* params, int32_t np) {
  if (!h) return HJMC_EINVAL;
  const int n = h->cfg.n;
  int want = 0;
  switch (id) {
    case HJMC_SYS_QUADRATIC: want = 0; break;
    case HJMC_SYS_DUBINS_REL:
      if (n != 3) return fail(h, HJMC_EINVAL, "DUBINS_REL needs n == 3");
      want = 3;
      break;
    case HJMC_SYS_ROCKET6:
      if (n != 6) return fail(h, HJMC_EINVAL, "ROCKET6 needs n == 6");
      want = 3;
      break;
    case HJMC_SYS_DUBINS_PAIRS:
      if (n % 3 != 0) return fail(h, HJMC_EINVAL, "DUBINS_PAIRS needs n = 3K");
      want = 3;
      break;
    case HJMC_SYS_ROCKET3:
      if (n != 3) return fail(h, HJMC_EINVAL, "ROCKET3 needs n == 3");
      want = 2;
      break;
    case HJMC_SYS_DOUBLE_INTEGRATOR:
      if (n != 2) return fail(h, HJMC_EINVAL, "DOUBLE_INTEGRATOR needs n == 2");
      want = 0;
      break;
    case HJMC_SYS_MULTIAGENT:
      if (n % 3 != 0 || n < 6) return fail(h, HJMC_EINVAL, "MULTIAGENT needs n = 3A, A >= 2");
      want = 2;
      break;
    default: return fail(h, HJMC_EINVAL, "unknown system id");
  }
  if (np != 0 && np != want) return fail(h, HJMC_EINVAL, "wrong number of system parameters");
  if (np > 0 && !params) return fail(h, HJMC_EINVAL, "params is NULL");
  SystemParams sp{};
  sp.id = id;
  sp.n = n;
  sp.np = np;
  for (int i = 0; i < np; ++i) {
    if (!std::isfinite(params[i])) return fail(h, HJMC_EINVAL, "non-finite system parameter");
    sp.p[i] = params[i];
  }
  h->sp = sp;
  h->sys_set = true;
  ++h->generation;
  return HJMC_OK;
}

int hjmc_set_avoid(hjmc_handle* h, int32_t id, const float* params, int32_t np) {
  if (!h) return HJMC_EINVAL;
  AvoidParams a{};
  if (id == HJMC_AVOID_NONE) {
    if (np != 0) return fail(h, HJMC_EINVAL, "AVOID_NONE takes no parameters");
  } else if (id == HJMC_AVOID_DISK) {
    if (np != 3 || !params) return fail(h, HJMC_EINVAL, "AVOID_DISK needs {c0, c1, r}");
    if (h->cfg.n < 2) return fail(h, HJMC_EINVAL, "AVOID_DISK needs n >= 2");
    for (int i = 0; i < 3; ++i) {
      if (!std::isfinite(params[i])) return fail(h, HJMC_EINVAL, "non-finite avoid parameter");
      a.p[i] = params[i];
    }
  } else {
    return fail(h, HJMC_EINVAL, "unknown avoid id");
  }
  a.type = id;
  h->avoid = a;
  ++h->generation;
  return HJMC_OK;
}

int hjmc_supported(int32_t target_id, int32_t n) {
  KernelSet ks;
  return lookup_kernels(target_id, n, &ks) ? 1 : 0;
}

int hjmc_set_target(hjmc_handle* h, int32_t id, const float* params, int32_t np) {
  if (!h) return HJMC_EINVAL;
  const int n = h->cfg.n;
  int want_max = 1, want_min = 0;
  switch (id) {
    case HJMC_TGT_QUAD_BOWL: break;
    case HJMC_TGT_DISK:
      if (n < 2) return fail(h, HJMC_EINVAL, "DISK needs n >= 2");
      break;
    case HJMC_TGT_REL_DISK6:
      if (n != 6) return fail(h, HJMC_EINVAL, "REL_DISK6 needs n == 6");
      break;
    case HJMC_TGT_PAIR_UNION:
      if (n % 3 != 0) return fail(h, HJMC_EINVAL, "PAIR_UNION needs n = 3K");
      break;
    case HJMC_TGT_LINEAR:
      want_min = want_max = n + 1;
      break;
    case HJMC_TGT_PURSUIT_MIN:
      if (n % 3 != 0 || n < 6) return fail(h, HJMC_EINVAL, "PURSUIT_MIN needs n = 3A, A >= 2");
      break;
    case HJMC_TGT_CONST: break;
    default: return fail(h, HJMC_EINVAL, "unknown target id");
  }
  if (np < want_min || np > want_max) return fail(h, HJMC_EINVAL, "wrong number of target parameters");
  if (np > 0 && !params) return fail(h, HJMC_EINVAL, "params is NULL");
  KernelSet ks;
  if (!lookup_kernels(id, n, &ks))
    return fail(h, HJMC_EUNSUPPORTED, "no kernel compiled for this (target, n)");
  TargetParams tp{};
  tp.np = np;
  for (int i = 0; i < np; ++i) {
    if (!std::isfinite(params[i])) return fail(h, HJMC_EINVAL, "non-finite target parameter");
    tp.p[i] = params[i];
  }
  h->tp = tp;
  h->tgt_id = id;
  h->ks = ks;
  h->tgt_set = true;
  ++h->generation;
  return HJMC_OK;
}

int hjmc_value_grad(hjmc_handle* h, const float* x, const float* c, const uint32_t* qid,
                    uint32_t qid_base, int64_t M, float tau, uint32_t j_tag, uint32_t k_tag,
                    const float* drift, float* v, float* dv, void* stream) {
  NvtxRange nvtx_range("hjmc_value_grad");
  int rc = ready(h);
  if (rc) return rc;
  if (M < 0) return fail(h, HJMC_EINVAL, "M < 0");
  if (M == 0) return HJMC_OK;
  if (!x || !v) return fail(h, HJMC_EINVAL, "x and v are required");
  if (!(tau >= 0.f) || !std::isfinite(tau)) return fail(h, HJMC_EINVAL, "tau must be >= 0");
  if (tau > 0.f && !c) return fail(h, HJMC_EINVAL, "c is required for tau > 0");
  if (j_tag > 65535u || k_tag > 255u) return fail(h, HJMC_EINVAL, "j_tag <= 65535, k_tag <= 255");
  if ((rc = set_device(h))) return rc;
  SolveParams p;
  fill_common(h, &p);
  p.x = x;
  p.drift = drift;
  p.qid = qid;
  p.qid_base = qid_base;
  p.M = M;
  p.K = 1;
  p.Kp = 1;
  p.T = tau;
  p.mode = kModeValueGrad;
  p.c_in = c;
  p.tau_vg = (double)tau;
  p.jtag = j_tag;
  p.ktag = k_tag;
  p.v = v;
  p.dv = dv;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = h->ks.solve(p, M, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "value_grad launch");
  return sync_check_if_requested(h, s);
}

int hjmc_solve_slice(hjmc_handle* h, const float* x, const uint32_t* qid, uint32_t qid_base,
                     int64_t M, const float* drift, const hjmc_result* out, void* stream) {
  NvtxRange nvtx_range("hjmc_solve_slice");
  int rc = ready(h);
  if (rc) return rc;
  if (M < 0) return fail(h, HJMC_EINVAL, "M < 0");
  if (M == 0) return HJMC_OK;
  if (!x) return fail(h, HJMC_EINVAL, "x is required");
  if (!out) return fail(h, HJMC_EINVAL, "out is required");
  const int64_t units = M * (int64_t)h->cfg.K;
  if (units > 0x7FFFFFFFLL) return fail(h, HJMC_EINVAL, "M*K exceeds the grid limit 2^31-1");
  if ((rc = set_device(h))) return rc;
  const bool want_tube = out->tube != nullptr;
  float* g0 = out->g0;
  if (want_tube && !g0) {
    if ((rc = ensure(h, &h->d_g0, &h->g0_cap, (size_t)M))) return rc;
    g0 = h->d_g0;
  }
  float* vfinal = nullptr;
  if (want_tube) {
    if ((rc = ensure(h, &h->d_vfinal, &h->vfinal_cap, (size_t)M * (size_t)h->cfg.K))) return rc;
    vfinal = h->d_vfinal;
  }
  SolveParams p;
  fill_common(h, &p);
  p.x = x;
  p.drift = drift;
  p.qid = qid;
  p.qid_base = qid_base;
  p.M = M;
  p.K = h->cfg.K;
  p.Kp = h->cfg.Kp;
  p.T = (double)h->cfg.T;
  p.mode = kModeSolve;
  p.v = out->v;
  p.dv = out->dv;
  p.c_out = out->c;
  p.vhist = out->vhist;
  p.chist = out->chist;
  p.vfinal = vfinal;
  p.g0 = g0;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = h->ks.solve(p, units, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "solve launch");
  if (want_tube) {
    e = launch_tube(g0, vfinal, h->cfg.K, M, out->tube, x, h->cfg.n, h->avoid, s);
    if (e != cudaSuccess) return cuda_fail(h, e, "tube launch");
  }
  return sync_check_if_requested(h, s);
}

int hjmc_solve_slice_host(hjmc_handle* h, const float* x_host, const uint32_t* qid_host,
                          uint32_t qid_base, int64_t M, const float* drift_host,
                          const hjmc_result* out_host) {
  NvtxRange nvtx_range("hjmc_solve_slice_host");
  int rc = ready(h);
  if (rc) return rc;
  if (M < 0) return fail(h, HJMC_EINVAL, "M < 0");
  if (M == 0) return HJMC_OK;
  if (!x_host || !out_host) return fail(h, HJMC_EINVAL, "x_host and out_host are required");
  if ((rc = set_device(h))) return rc;
  const size_t n = (size_t)h->cfg.n, K = (size_t)h->cfg.K, Kp = (size_t)h->cfg.Kp, m = (size_t)M;
  // staging layout (4-byte words): x | drift | v | dv | c | tube | vhist | chist | g0 | qid
  const size_t sizes[10] = {m * n, drift_host ? m * n : 0, out_host->v ? m : 0,
                            out_host->dv ? m * n : 0, out_host->c ? m : 0, out_host->tube ? m : 0,
                            out_host->vhist ? K * Kp * m : 0, out_host->chist ? K * Kp * m : 0,
                            out_host->g0 ? m : 0, qid_host ? m : 0};
  size_t total = 0, off[10];
  for (int i = 0; i < 10; ++i) {
    off[i] = total;
    total += (sizes[i] + 63) & ~size_t(63);  // 256-byte aligned sub-buffers
  }
  if ((rc = ensure(h, &h->d_stage, &h->stage_cap, total))) return rc;
  float* base = h->d_stage;
  cudaStream_t s = h->host_stream;
  cudaError_t e = cudaMemcpyAsync(base + off[0], x_host, sizes[0] * sizeof(float),
                                  cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && drift_host)
    e = cudaMemcpyAsync(base + off[1], drift_host, sizes[1] * sizeof(float), cudaMemcpyHostToDevice, s);
  uint32_t* dqid = qid_host ? reinterpret_cast<uint32_t*>(base + off[9]) : nullptr;
  if (e == cudaSuccess && qid_host)
    e = cudaMemcpyAsync(dqid, qid_host, sizes[9] * sizeof(uint32_t), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "H2D copy");
  hjmc_result dres{};
  float** dptr[7] = {&dres.v, &dres.dv, &dres.c, &dres.tube, &dres.vhist, &dres.chist, &dres.g0};
  for (int i = 0; i < 7; ++i) *dptr[i] = sizes[2 + i] ? base + off[2 + i] : nullptr;
  rc = hjmc_solve_slice(h, base + off[0], dqid, qid_base, M, drift_host ? base + off[1] : nullptr,
                        &dres, (void*)s);
  if (rc) return rc;
  float* hptr[7] = {out_host->v, out_host->dv, out_host->c, out_host->tube, out_host->vhist,
                    out_host->chist, out_host->g0};
  for (int i = 0; i < 7; ++i) {
    if (!sizes[2 + i]) continue;
    e = cudaMemcpyAsync(hptr[i], base + off[2 + i], sizes[2 + i] * sizeof(float),
                        cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(h, e, "D2H copy");
  }
  return hjmc_check(h, (void*)s);
}

int hjmc_picard_begin(hjmc_handle* h, const float* x, const uint32_t* qid, uint32_t qid_base,
                      int64_t M, const float* drift, void* stream) {
  NvtxRange nvtx_range("hjmc_picard_begin");
  int rc = ready(h);
  if (rc) return rc;
  if (M < 1 || !x) return fail(h, HJMC_EINVAL, "need M >= 1 and x");
  if (M * (int64_t)h->cfg.K > 0x7FFFFFFFLL) return fail(h, HJMC_EINVAL, "M*K exceeds 2^31-1");
  if ((rc = set_device(h))) return rc;
  const size_t KM = (size_t)M * (size_t)h->cfg.K;
  if (KM > h->cstate_cap) {
    if (h->d_cstate) cudaFree(h->d_cstate);
    h->d_cstate = nullptr;
    h->cstate_cap = 0;
    cudaError_t e = cudaMalloc((void**)&h->d_cstate, KM * sizeof(double));
    if (e != cudaSuccess) return fail(h, HJMC_ENOMEM, "picard state allocation failed");
    h->cstate_cap = KM;
  }
  if ((rc = ensure(h, &h->d_vprev, &h->vprev_cap, KM))) return rc;
  if (!h->d_active) {
    cudaError_t e = cudaMalloc((void**)&h->d_active, 65536 * sizeof(int));
    if (e != cudaSuccess) return fail(h, HJMC_ENOMEM, "picard active-list allocation failed");
  }
  h->pic_x = x;
  h->pic_qid = qid;
  h->pic_qid_base = qid_base;
  h->pic_M = M;
  h->pic_drift = drift;
  PicardInitParams ip{};
  ip.x = x;
  ip.M = M;
  ip.K = h->cfg.K;
  ip.c_state = h->d_cstate;
  ip.v_prev = h->d_vprev;
  ip.gp.delta_eff = delta_eff(h->cfg);
  ip.gp.m0 = h->cfg.m0;
  ip.gp.c_min = h->cfg.c_min;
  ip.gp.c_max = h->cfg.c_max;
  ip.sp = h->sp;
  ip.tp = h->tp;
  cudaError_t e = h->ks.picard_init(ip, (cudaStream_t)stream);
  return e == cudaSuccess ? HJMC_OK : cuda_fail(h, e, "picard init launch");
}

// Device-resident Algorithm 1: the same init / pass / residual kernels as hjmc_picard_begin and
// hjmc_picard_pass, ordered in one CUDA graph — init, then a conditional 'while' node looping
// {pass, residual, decision} whose condition the decision kernel sets — so no Picard iterate
// returns to the host. Results are bit-identical to the host-driven loop (same kernels, same
// reduction orders, the same double-precision test). The instantiated graph is cached in the
// handle and relaunched while the arguments and the problem are unchanged.
int hjmc_picard_solve(hjmc_handle* h, const float* x, const uint32_t* qid, uint32_t qid_base,
                      int64_t M, const float* drift, double tol, int32_t max_iter, float* v,
                      float* dv, float* c, int32_t* iters, double* eps, double* dsup, float* tube,
                      void* stream) {
  NvtxRange nvtx_range("hjmc_picard_solve");
  int rc = ready(h);
  if (rc) return rc;
  if (M < 1 || !x) return fail(h, HJMC_EINVAL, "need M >= 1 and x");
  if (M * (int64_t)h->cfg.K > 0x7FFFFFFFLL) return fail(h, HJMC_EINVAL, "M*K exceeds 2^31-1");
  if (max_iter < 1 || !(tol >= 0.0)) return fail(h, HJMC_EINVAL, "need max_iter >= 1, tol >= 0");
  if (!v || !iters || !eps || !dsup) return fail(h, HJMC_EINVAL, "v, iters, eps, dsup required");
  if (!h->cfg.crn && max_iter > 256) return fail(h, HJMC_EINVAL, "max_iter must be <= 256 without crn");
  if ((rc = set_device(h))) return rc;
  const int K = h->cfg.K;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t KM = (size_t)M * (size_t)K;
  const int blocks = (int)std::min<int64_t>(148, (M + 255) / 256);
  const size_t need = (size_t)K * (size_t)blocks * 3;
  // handle scratch (sizes only grow; a reallocation invalidates the cached graph)
  bool realloc = false;
  if (KM > h->cstate_cap) {
    if (h->d_cstate) cudaFree(h->d_cstate);
    h->d_cstate = nullptr;
    h->cstate_cap = 0;
    if (cudaMalloc((void**)&h->d_cstate, KM * sizeof(double)) != cudaSuccess)
      return fail(h, HJMC_ENOMEM, "picard state allocation failed");
    h->cstate_cap = KM;
    realloc = true;
  }
  const float* old_vprev = h->d_vprev;
  if ((rc = ensure(h, &h->d_vprev, &h->vprev_cap, KM))) return rc;
  realloc = realloc || h->d_vprev != old_vprev;
  if (need > h->partial_cap) {
    if (h->d_partial) cudaFree(h->d_partial);
    h->d_partial = nullptr;
    h->partial_cap = 0;
    if (cudaMalloc((void**)&h->d_partial, need * sizeof(double)) != cudaSuccess)
      return fail(h, HJMC_ENOMEM, "picard partials allocation failed");
    h->partial_cap = need;
    realloc = true;
  }
  if (!h->d_pstate) {
    if (cudaMalloc((void**)&h->d_pstate, (2 * 65536 + 1) * sizeof(int)) != cudaSuccess)
      return fail(h, HJMC_ENOMEM, "picard state allocation failed");
    realloc = true;
  }
  float* g0 = nullptr;  // g(x) for the tube epilogue (written by the init kernel)
  if (tube) {
    const float* old_g0 = h->d_g0;
    if ((rc = ensure(h, &h->d_g0, &h->g0_cap, (size_t)M))) return rc;
    realloc = realloc || h->d_g0 != old_g0;
    g0 = h->d_g0;
  }
  h->pic_x = x;
  h->pic_qid = qid;
  h->pic_qid_base = qid_base;
  h->pic_M = M;
  h->pic_drift = drift;
  double tol_bits = tol;
  uintptr_t tol_key;
  std::memcpy(&tol_key, &tol_bits, sizeof(tol_key));
  const std::vector<uintptr_t> key = {
      (uintptr_t)x, (uintptr_t)qid, qid_base, (uintptr_t)M, (uintptr_t)drift, tol_key,
      (uintptr_t)max_iter, (uintptr_t)v, (uintptr_t)dv, (uintptr_t)c, (uintptr_t)iters,
      (uintptr_t)eps, (uintptr_t)dsup, (uintptr_t)tube, (uintptr_t)g0, h->generation,
      // handle scratch the graph reads: another entry point may have reallocated it since
      (uintptr_t)h->d_cstate, (uintptr_t)h->d_vprev, (uintptr_t)h->d_partial,
      (uintptr_t)h->d_pstate};
  cudaError_t e;
  if (realloc || !h->pic_exec || key != h->pic_key) {
    if (h->pic_exec) cudaGraphExecDestroy(h->pic_exec);
    if (h->pic_graph) cudaGraphDestroy(h->pic_graph);
    h->pic_exec = nullptr;
    h->pic_graph = nullptr;
    h->pic_key.clear();
    int* st = h->d_pstate;
    PicardInitParams ip{};
    ip.x = x;
    ip.M = M;
    ip.K = K;
    ip.c_state = h->d_cstate;
    ip.v_prev = h->d_vprev;
    ip.g0 = g0;
    ip.gp.delta_eff = delta_eff(h->cfg);
    ip.gp.m0 = h->cfg.m0;
    ip.gp.c_min = h->cfg.c_min;
    ip.gp.c_max = h->cfg.c_max;
    ip.sp = h->sp;
    ip.tp = h->tp;
    SolveParams p;
    fill_common(h, &p);
    p.x = x;
    p.drift = drift;
    p.qid = qid;
    p.qid_base = qid_base;
    p.M = M;
    p.K = K;
    p.Kp = 1;
    p.T = (double)h->cfg.T;
    p.mode = kModePass;
    p.v = v;
    p.dv = dv;
    p.c_out = c;
    p.c_state = h->d_cstate;
    p.active_j = st;
    p.n_active = K;
    p.active_mask = st + K;
    p.kiter_dev = st + 2 * K;
    p.kiter = 0;
    p.skip_stationary = 0;
    p.reuse_passes = 0;

    cudaGraph_t graph = nullptr;
    cudaGraphConditionalHandle cond;
    auto bail = [&](cudaError_t err, const char* where) {
      if (graph) cudaGraphDestroy(graph);
      return cuda_fail(h, err, where);
    };
    if ((e = cudaGraphCreate(&graph, 0)) != cudaSuccess) return bail(e, "graph create");
    if ((e = cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault)) !=
        cudaSuccess)
      return bail(e, "conditional handle");
    cudaStream_t cap = h->host_stream;
    // 1. init: v^(0) = g, c^(0) = Γ(x, Dg) per horizon; loop state, iteration counts, NaN histories
    if ((e = cudaStreamBeginCaptureToGraph(cap, graph, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed)) != cudaSuccess)
      return bail(e, "init capture");
    cudaError_t le = h->ks.picard_init(ip, cap);
    if (le == cudaSuccess) le = launch_picard_solve_init(st, K, iters, eps, dsup, max_iter, cap);
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaStreamCaptureStatus cs;
    std::vector<cudaGraphNode_t> tail;
    if (le == cudaSuccess &&
        (le = cudaStreamGetCaptureInfo(cap, &cs, nullptr, nullptr, &deps, &ndeps)) == cudaSuccess)
      tail.assign(deps, deps + ndeps);
    cudaGraph_t captured = nullptr;
    e = cudaStreamEndCapture(cap, &captured);
    if (le != cudaSuccess) return bail(le, "init launches");
    if (e != cudaSuccess) return bail(e, "init capture end");
    // 2. the loop
    cudaGraphNode_t node;
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    if ((e = cudaGraphAddNode(&node, graph, tail.data(), tail.size(), &np)) != cudaSuccess)
      return bail(e, "conditional node");
    cudaGraph_t body = np.conditional.phGraph_out[0];
    if ((e = cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed)) != cudaSuccess)
      return bail(e, "body capture");
    le = h->ks.solve(p, M * (int64_t)K, cap);
    if (le == cudaSuccess)
      le = launch_picard_residual(v, h->d_vprev, M, st, K, h->d_partial, blocks, cap);
    if (le == cudaSuccess)
      le = launch_picard_decide(h->d_partial, K, blocks, tol, max_iter, st + K, st + 2 * K, iters,
                                eps, dsup, cond, cap);
    e = cudaStreamEndCapture(cap, &captured);
    if (le != cudaSuccess) return bail(le, "body launches");
    if (e != cudaSuccess) return bail(e, "body capture end");
    // 3. after the loop: the running-min tube with the BRAT clamp over each
    //    horizon's final iterate v[j][·]
    if (tube) {
      if ((e = cudaStreamBeginCaptureToGraph(cap, graph, &node, nullptr, 1,
                                             cudaStreamCaptureModeRelaxed)) != cudaSuccess)
        return bail(e, "tube capture");
      le = launch_tube(g0, v, K, M, tube, x, h->cfg.n, h->avoid, cap);
      e = cudaStreamEndCapture(cap, &captured);
      if (le != cudaSuccess) return bail(le, "tube launch");
      if (e != cudaSuccess) return bail(e, "tube capture end");
    }
    cudaGraphExec_t exec = nullptr;
    if ((e = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess) return bail(e, "graph instantiate");
    h->pic_graph = graph;
    h->pic_exec = exec;
    h->pic_key = key;
  }
  if ((e = cudaGraphLaunch(h->pic_exec, s)) != cudaSuccess) return cuda_fail(h, e, "graph launch");
  return sync_check_if_requested(h, s);
}

int hjmc_picard_pass(hjmc_handle* h, int32_t k, const uint8_t* active, float* v, float* dv,
                     float* c, double* partials, void* stream) {
  NvtxRange nvtx_range("hjmc_picard_pass");
  int rc = ready(h);
  if (rc) return rc;
  if (h->pic_M < 1) return fail(h, HJMC_EINVAL, "hjmc_picard_begin has not been called");
  if (k < 0 || (!h->cfg.crn && k > 255)) return fail(h, HJMC_EINVAL, "bad iterate index k");
  if (!partials) return fail(h, HJMC_EINVAL, "partials is required");
  if ((rc = set_device(h))) return rc;
  const int K = h->cfg.K;
  const int64_t M = h->pic_M;
  std::vector<int> act;
  for (int j = 0; j < K; ++j)
    if (!active || active[j]) act.push_back(j + 1);
  for (int i = 0; i < 3 * K; ++i) partials[i] = 0.0;
  if (act.empty()) return HJMC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  float* vout = v;
  if (!vout) {
    if ((rc = ensure(h, &h->d_vtmp, &h->vtmp_cap, (size_t)M * (size_t)K))) return rc;
    vout = h->d_vtmp;
  }
  const int blocks = (int)std::min<int64_t>(148, (M + 255) / 256);
  const size_t need = act.size() * (size_t)blocks * 3;
  if (need > h->partial_cap) {
    if (h->d_partial) cudaFree(h->d_partial);
    h->d_partial = nullptr;
    h->partial_cap = 0;
    if (cudaMalloc((void**)&h->d_partial, need * sizeof(double)) != cudaSuccess)
      return fail(h, HJMC_ENOMEM, "picard partials allocation failed");
    h->partial_cap = need;
  }
  cudaError_t e = cudaMemcpyAsync(h->d_active, act.data(), act.size() * sizeof(int),
                                  cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "active list copy");
  SolveParams p;
  fill_common(h, &p);
  p.x = h->pic_x;
  p.drift = h->pic_drift;
  p.qid = h->pic_qid;
  p.qid_base = h->pic_qid_base;
  p.M = M;
  p.K = K;
  p.Kp = 1;
  p.T = (double)h->cfg.T;
  p.mode = kModePass;
  p.v = vout;
  p.dv = dv;
  p.c_out = c;
  p.c_state = h->d_cstate;
  p.active_j = h->d_active;
  p.n_active = (int)act.size();
  p.kiter = k;
  p.skip_stationary = 0;
  p.reuse_passes = 0;
  e = h->ks.solve(p, M * (int64_t)act.size(), s);
  if (e != cudaSuccess) return cuda_fail(h, e, "picard pass launch");
  e = launch_picard_residual(vout, h->d_vprev, M, h->d_active, (int)act.size(), h->d_partial,
                             blocks, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "picard residual launch");
  std::vector<double> host(need);
  e = cudaMemcpyAsync(host.data(), h->d_partial, need * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(h, e, "picard partials read");
  for (size_t a = 0; a < act.size(); ++a) {
    double num = 0.0, den = 0.0, mx = 0.0;
    for (int b = 0; b < blocks; ++b) {  // fixed order: deterministic
      const double* q = host.data() + (a * (size_t)blocks + b) * 3;
      num += q[0];
      den += q[1];
      mx = std::max(mx, q[2]);
    }
    double* o = partials + (size_t)(act[a] - 1) * 3;
    o[0] = num;
    o[1] = den;
    o[2] = mx;
  }
  return sync_check_if_requested(h, s);
}

// Sharded device-resident Algorithm 1: the graph mode's kernels without the conditional node,
// driven by the caller so a collective can sit between the residual and the decision.
int hjmc_picard_dev_begin(hjmc_handle* h, const float* x, const uint32_t* qid, uint32_t qid_base,
                          int64_t M, const float* drift, int32_t max_iter, int32_t* iters,
                          double* eps, double* dsup, void* stream) {
  NvtxRange nvtx_range("hjmc_picard_dev_begin");
  int rc = ready(h);
  if (rc) return rc;
  if (M < 1 || !x) return fail(h, HJMC_EINVAL, "need M >= 1 and x");
  if (M * (int64_t)h->cfg.K > 0x7FFFFFFFLL) return fail(h, HJMC_EINVAL, "M*K exceeds 2^31-1");
  if (max_iter < 1 || !iters || !eps || !dsup)
    return fail(h, HJMC_EINVAL, "need max_iter >= 1 and iters, eps, dsup");
  if (!h->cfg.crn && max_iter > 256) return fail(h, HJMC_EINVAL, "max_iter must be <= 256 without crn");
  if ((rc = set_device(h))) return rc;
  const int K = h->cfg.K;
  const size_t KM = (size_t)M * (size_t)K;
  const int blocks = (int)std::min<int64_t>(148, (M + 255) / 256);
  const size_t need = (size_t)K * (size_t)blocks * 3;
  if (KM > h->cstate_cap) {
    if (h->d_cstate) cudaFree(h->d_cstate);
    h->d_cstate = nullptr;
    h->cstate_cap = 0;
    if (cudaMalloc((void**)&h->d_cstate, KM * sizeof(double)) != cudaSuccess)
      return fail(h, HJMC_ENOMEM, "picard state allocation failed");
    h->cstate_cap = KM;
  }
  if ((rc = ensure(h, &h->d_vprev, &h->vprev_cap, KM))) return rc;
  if (need > h->partial_cap) {
    if (h->d_partial) cudaFree(h->d_partial);
    h->d_partial = nullptr;
    h->partial_cap = 0;
    if (cudaMalloc((void**)&h->d_partial, need * sizeof(double)) != cudaSuccess)
      return fail(h, HJMC_ENOMEM, "picard partials allocation failed");
    h->partial_cap = need;
  }
  if (!h->d_pstate && cudaMalloc((void**)&h->d_pstate, (2 * 65536 + 1) * sizeof(int)) != cudaSuccess)
    return fail(h, HJMC_ENOMEM, "picard state allocation failed");
  h->pic_x = x;
  h->pic_qid = qid;
  h->pic_qid_base = qid_base;
  h->pic_M = M;
  h->pic_drift = drift;
  h->pic_dev_max_iter = max_iter;
  h->pic_dev_blocks = blocks;
  PicardInitParams ip{};
  ip.x = x;
  ip.M = M;
  ip.K = K;
  ip.c_state = h->d_cstate;
  ip.v_prev = h->d_vprev;
  ip.gp.delta_eff = delta_eff(h->cfg);
  ip.gp.m0 = h->cfg.m0;
  ip.gp.c_min = h->cfg.c_min;
  ip.gp.c_max = h->cfg.c_max;
  ip.sp = h->sp;
  ip.tp = h->tp;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = h->ks.picard_init(ip, s);
  if (e == cudaSuccess) e = launch_picard_solve_init(h->d_pstate, K, iters, eps, dsup, max_iter, s);
  return e == cudaSuccess ? HJMC_OK : cuda_fail(h, e, "picard dev init launch");
}

int hjmc_picard_dev_pass(hjmc_handle* h, float* v, float* dv, float* c, double* reduced,
                         void* stream) {
  NvtxRange nvtx_range("hjmc_picard_dev_pass");
  int rc = ready(h);
  if (rc) return rc;
  if (h->pic_M < 1 || h->pic_dev_max_iter < 1)
    return fail(h, HJMC_EINVAL, "hjmc_picard_dev_begin has not been called");
  if (!v || !reduced) return fail(h, HJMC_EINVAL, "v and reduced are required");
  if ((rc = set_device(h))) return rc;
  const int K = h->cfg.K;
  const int64_t M = h->pic_M;
  int* st = h->d_pstate;
  SolveParams p;
  fill_common(h, &p);
  p.x = h->pic_x;
  p.drift = h->pic_drift;
  p.qid = h->pic_qid;
  p.qid_base = h->pic_qid_base;
  p.M = M;
  p.K = K;
  p.Kp = 1;
  p.T = (double)h->cfg.T;
  p.mode = kModePass;
  p.v = v;
  p.dv = dv;
  p.c_out = c;
  p.c_state = h->d_cstate;
  p.active_j = st;
  p.n_active = K;
  p.active_mask = st + K;
  p.kiter_dev = st + 2 * K;
  p.kiter = 0;
  p.skip_stationary = 0;
  p.reuse_passes = 0;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = h->ks.solve(p, M * (int64_t)K, s);
  if (e == cudaSuccess)
    e = launch_picard_residual(v, h->d_vprev, M, st, K, h->d_partial, h->pic_dev_blocks, s);
  if (e == cudaSuccess)
    e = launch_picard_blocksum(h->d_partial, K, h->pic_dev_blocks, st + K, reduced, s);
  return e == cudaSuccess ? HJMC_OK : cuda_fail(h, e, "picard dev pass launch");
}

int hjmc_picard_dev_decide(hjmc_handle* h, const double* reduced, double tol, int32_t* iters,
                           double* eps, double* dsup, void* stream) {
  NvtxRange nvtx_range("hjmc_picard_dev_decide");
  int rc = ready(h);
  if (rc) return rc;
  if (h->pic_dev_max_iter < 1) return fail(h, HJMC_EINVAL, "hjmc_picard_dev_begin has not been called");
  if (!reduced || !iters || !eps || !dsup || !(tol >= 0.0))
    return fail(h, HJMC_EINVAL, "need reduced, iters, eps, dsup and tol >= 0");
  if ((rc = set_device(h))) return rc;
  const int K = h->cfg.K;
  int* st = h->d_pstate;
  cudaError_t e = launch_picard_decide_reduced(reduced, K, tol, h->pic_dev_max_iter, st + K,
                                               st + 2 * K, iters, eps, dsup, (cudaStream_t)stream);
  return e == cudaSuccess ? HJMC_OK : cuda_fail(h, e, "picard dev decide launch");
}

int hjmc_eval_target(hjmc_handle* h, const float* x, int64_t M, float* g, float* dg, void* stream) {
  if (!h) return HJMC_EINVAL;
  if (!h->tgt_set) return fail(h, HJMC_EINVAL, "hjmc_set_target has not been called");
  if (M < 0 || (M > 0 && !x)) return fail(h, HJMC_EINVAL, "bad x / M");
  if (M == 0) return HJMC_OK;
  int rc = set_device(h);
  if (rc) return rc;
  EvalParams p{};
  p.x = x;
  p.M = M;
  p.g = g;
  p.dg = dg;
  p.tp = h->tp;
  cudaError_t e = h->ks.eval_target(p, (cudaStream_t)stream);
  return e == cudaSuccess ? HJMC_OK : cuda_fail(h, e, "eval_target launch");
}

int hjmc_eval_hamiltonian(hjmc_handle* h, const float* x, const float* p_in, int64_t M, float* H,
                          float* c, void* stream) {
  if (!h) return HJMC_EINVAL;
  if (!h->sys_set) return fail(h, HJMC_EINVAL, "hjmc_set_dynamics has not been called");
  if (M < 0 || (M > 0 && (!x || !p_in))) return fail(h, HJMC_EINVAL, "bad x / p / M");
  if (M == 0) return HJMC_OK;
  int rc = set_device(h);
  if (rc) return rc;
  EvalParams p{};
  p.x = x;
  p.p = p_in;
  p.M = M;
  p.H = H;
  p.c = c;
  p.sp = h->sp;
  p.gp.delta_eff = delta_eff(h->cfg);
  p.gp.m0 = h->cfg.m0;
  p.gp.c_min = h->cfg.c_min;
  p.gp.c_max = h->cfg.c_max;
  cudaError_t e = launch_hamiltonian(p, (cudaStream_t)stream);
  return e == cudaSuccess ? HJMC_OK : cuda_fail(h, e, "hamiltonian launch");
}

int hjmc_debug_normals(hjmc_handle* h, uint32_t qid, uint32_t jw, uint32_t kw, uint32_t i0,
                       uint32_t count, float* z, uint32_t* raw, void* stream) {
  if (!h) return HJMC_EINVAL;
  if (count > 0 && !z) return fail(h, HJMC_EINVAL, "z is NULL");
  if (jw > 65535u || kw > 255u) return fail(h, HJMC_EINVAL, "jw <= 65535, kw <= 255");
  int rc = set_device(h);
  if (rc) return rc;
  RoundKeys rk;
  make_round_keys(h->cfg.seed, &rk);
  cudaError_t e = launch_debug_normals(h->cfg.n, qid, jw, kw, i0, count, rk, h->cfg.tag,
                                       h->cfg.antithetic, z, raw, (cudaStream_t)stream);
  return e == cudaSuccess ? HJMC_OK : cuda_fail(h, e, "debug_normals launch");
}

int hjmc_check(hjmc_handle* h, void* stream) {
  if (!h) return HJMC_EINVAL;
  int rc = set_device(h);
  if (rc) return rc;
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "stream synchronize");
  int flag = 0;
  unsigned long long bad = 0;
  if ((e = cudaMemcpy(&flag, h->d_err, sizeof(int), cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(&bad, h->d_bad, sizeof(bad), cudaMemcpyDeviceToHost)) != cudaSuccess)
    return cuda_fail(h, e, "error-word read");
  if (!flag) return HJMC_OK;
  h->last_bad = (int64_t)bad;
  cudaMemset(h->d_err, 0, sizeof(int));
  cudaMemset(h->d_bad, 0xFF, sizeof(unsigned long long));
  char buf[128];
  std::snprintf(buf, sizeof(buf), "non-finite v or Dv at global query id %lld", (long long)bad);
  return fail(h, HJMC_ENUMERIC, buf);
}

int64_t hjmc_last_bad_query(const hjmc_handle* h) { return h ? h->last_bad : -1; }

int hjmc_pass_count(hjmc_handle* h, void* stream, uint64_t* passes) {
  if (!h || !passes) return HJMC_EINVAL;
  int rc = set_device(h);
  if (rc) return rc;
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  unsigned long long v = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&v, h->d_passes, sizeof(v), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(h->d_passes, 0, sizeof(v));
  if (e != cudaSuccess) return cuda_fail(h, e, "pass counter read");
  *passes = (uint64_t)v;
  return HJMC_OK;
}

const char* hjmc_last_error(const hjmc_handle* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

int hjmc_tube(hjmc_handle* h, const float* x, int64_t M, const float* vfinal, float* tube,
              void* stream) {
  NvtxRange nvtx_range("hjmc_tube");
  int rc = ready(h);
  if (rc) return rc;
  if (M < 0 || (M > 0 && (!x || !vfinal || !tube))) return fail(h, HJMC_EINVAL, "bad x / vfinal / tube / M");
  if (M == 0) return HJMC_OK;
  if ((rc = set_device(h))) return rc;
  if ((rc = ensure(h, &h->d_g0, &h->g0_cap, (size_t)M))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  EvalParams p{};
  p.x = x;
  p.M = M;
  p.g = h->d_g0;
  p.tp = h->tp;
  cudaError_t e = h->ks.eval_target(p, s);
  if (e == cudaSuccess) e = launch_tube(h->d_g0, vfinal, h->cfg.K, M, tube, x, h->cfg.n, h->avoid, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "tube launch");
  return sync_check_if_requested(h, s);
}

int hjmc_picard_decide(const double* partials, int32_t K, double tol, uint8_t* active,
                       double* eps, double* dsup, int32_t* n_active) {
  if (!partials || !active || K < 1 || !(tol >= 0.0)) return HJMC_EINVAL;
  int32_t left = 0;
  for (int j = 0; j < K; ++j) {
    if (eps) eps[j] = NAN;
    if (dsup) dsup[j] = NAN;
    if (!active[j]) continue;
    const double* q = partials + (size_t)j * 3;
    // the same double-precision expression as the device-resident decision kernel
    const double e = std::sqrt(q[0] / std::fmax(q[1], 1e-300));
    if (eps) eps[j] = e;
    if (dsup) dsup[j] = q[2];
    if (e < tol) active[j] = 0;
    else ++left;
  }
  if (n_active) *n_active = left;
  return HJMC_OK;
}

double hjmc_contraction_constant(double G, double c_min, double L_D, double delta, double L_H,
                                 double m0, double H_star, double P_star) {
  return (2.0 * G / c_min) * (2.0 * L_D / delta) *
         (L_H / (m0 * m0) + 2.0 * H_star * P_star / (m0 * m0 * m0 * m0));
}

int hjmc_contraction_report(const double* d, int64_t count, double q, double* q_hat,
                            double* apost) {
  if (count < 0 || (count > 0 && !d)) return -1;
  if (q_hat)
    for (int64_t k = 0; k + 1 < count; ++k) q_hat[k] = d[k + 1] / d[k];
  const bool certified = q >= 0.0 && q < 1.0;
  if (certified && apost)
    for (int64_t k = 0; k < count; ++k) apost[k] = q / (1.0 - q) * d[k];
  return certified ? 1 : 0;
}

int hjmc_residual_eps(const double* partials, int64_t count, double* eps) {
  if (count < 0 || (count > 0 && (!partials || !eps))) return HJMC_EINVAL;
  for (int64_t i = 0; i < count; ++i)
    eps[i] = std::sqrt(partials[2 * i] / std::fmax(partials[2 * i + 1], 1e-300));
  return HJMC_OK;
}

int hjmc_residual_partials(const float* vhist, const float* g0, int32_t K, int32_t Kp, int64_t M,
                           double* out) {
  if (!vhist || !g0 || !out || K < 1 || Kp < 1 || M < 0) return HJMC_EINVAL;
  for (int j = 0; j < K; ++j) {
    for (int k = 0; k < Kp; ++k) {
      double num = 0.0, den = 0.0;
      const float* cur = vhist + ((size_t)j * Kp + k) * (size_t)M;
      const float* prev = (k == 0) ? g0 : vhist + ((size_t)j * Kp + (k - 1)) * (size_t)M;
      for (int64_t m = 0; m < M; ++m) {
        const double a = (double)cur[m], b = (double)prev[m];
        num += (a - b) * (a - b);
        den += b * b;
      }
      out[((size_t)j * Kp + k) * 2 + 0] = num;
      out[((size_t)j * Kp + k) * 2 + 1] = den;
    }
  }
  return HJMC_OK;
}

}  // extern "C"
