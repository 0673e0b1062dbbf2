// hjmc_aux.cu — small non-templated kernels: tube epilogue, H/Γ evaluator, RNG debug dump.
#include <cuda_runtime.h>

#include <algorithm>

#include <cstdint>

#include "hjmc_kernels.cuh"

namespace hjmc {

namespace {

__global__ void tube_kernel(const float* __restrict__ g0, const float* __restrict__ vfinal, int K,
                            int64_t M, float* __restrict__ tube, const float* __restrict__ x,
                            int n, AvoidParams avoid) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float t = g0[m];  // running min including g
  for (int j = 0; j < K; ++j) t = fminf(t, vfinal[(size_t)j * (size_t)M + (size_t)m]);
  if (avoid.type == 1) {  // BRAT clamp: exclude the obstacle
    const double dx = (double)x[m * n] - avoid.p[0], dy = (double)x[m * n + 1] - avoid.p[1];
    t = fmaxf(t, (float)((double)avoid.p[2] - sqrt(dx * dx + dy * dy)));
  }
  tube[m] = t;
}

__global__ void hamiltonian_kernel(const EvalParams P) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= P.M) return;
  const int n = P.sp.n;
  double x[64], p[64];
  for (int d = 0; d < n; ++d) {
    x[d] = (double)P.x[m * n + d];
    p[d] = (double)P.p[m * n + d];
  }
  if (P.H) P.H[m] = (float)hamiltonian(P.sp, x, p);
  if (P.c) P.c[m] = (float)gamma_update(P.sp, P.gp, x, p);
}

// The sampler's normals exactly as the solve kernels draw them (R19 layout, runtime n): for
// sample i its draw's group g, position r in the group, and the Philox blocks its n normals
// come from; raw receives the words of every block the sample touches, in order.
__global__ void debug_normals_kernel(int n, uint32_t qid, uint32_t jw, uint32_t kw, uint32_t i0,
                                     uint32_t count, const __grid_constant__ RoundKeys rk,
                                     uint32_t tag, int antithetic, float* z, uint32_t* raw) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  const uint32_t i = i0 + s;
  const uint32_t draw = antithetic ? (i >> 1) : i;
  const float sign = (antithetic && (i & 1u)) ? -1.f : 1.f;
  const int g0 = (n % 4 == 0) ? 1 : ((n % 2 == 0) ? 2 : 4);
  const int G = (g0 * n <= 16) ? g0 : 1;
  const uint32_t grp = draw / (uint32_t)G;
  const int first = (G == 1) ? 0 : (int)(draw % (uint32_t)G) * n;
  const int rawmax = 4 * ((n + 3) / 4 + 1);
  int cur = -1, nraw = 0;
  float t[4];
  for (int d = 0; d < n; ++d) {
    const int l = first + d;
    if (l / 4 != cur) {
      cur = l / 4;
      const uint4 w = philox4x32_10(grp, ctr_word1((uint32_t)cur, kw, jw), qid, tag, rk);
      if (raw) {
        uint32_t* r = raw + (size_t)s * rawmax + 4 * nraw;
        r[0] = w.x; r[1] = w.y; r[2] = w.z; r[3] = w.w;
      }
      ++nraw;
      box_muller_hat<true>(w.x, w.y, t[0], t[1]);
      box_muller_hat<true>(w.z, w.w, t[2], t[3]);
    }
    z[(size_t)s * n + d] = sign * kBMScale * t[l % 4];
  }
}

__global__ void picard_residual_kernel(const float* __restrict__ v, float* __restrict__ v_prev,
                                       int64_t M, const int* __restrict__ active_j,
                                       double* __restrict__ partial) {
  __shared__ double s_num[256], s_den[256], s_max[256];
  const int a = blockIdx.y;
  const size_t base = (size_t)(active_j[a] - 1) * (size_t)M;
  double num = 0.0, den = 0.0, mx = 0.0;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < M;
       m += (int64_t)gridDim.x * blockDim.x) {
    const double cur = (double)v[base + m], prev = (double)v_prev[base + m];
    const double d = cur - prev;
    num += d * d;
    den += prev * prev;
    mx = fmax(mx, fabs(d));
    v_prev[base + m] = v[base + m];
  }
  s_num[threadIdx.x] = num;
  s_den[threadIdx.x] = den;
  s_max[threadIdx.x] = mx;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s_num[threadIdx.x] += s_num[threadIdx.x + o];
      s_den[threadIdx.x] += s_den[threadIdx.x + o];
      s_max[threadIdx.x] = fmax(s_max[threadIdx.x], s_max[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* out = partial + ((size_t)a * gridDim.x + blockIdx.x) * 3;
    out[0] = s_num[0];
    out[1] = s_den[0];
    out[2] = s_max[0];
  }
}

__global__ void picard_decide_kernel(const double* __restrict__ partial, int K, int blocks,
                                     double tol, int max_iter, int* mask, int* kiter, int* iters,
                                     double* eps, double* dsup, cudaGraphConditionalHandle cond) {
  if (threadIdx.x != 0) return;  // K is small; one thread keeps the host driver's order
  const int k = *kiter;
  int any = 0;
  for (int j = 0; j < K; ++j) {
    if (!mask[j]) continue;
    double num = 0.0, den = 0.0, mx = 0.0;
    for (int b = 0; b < blocks; ++b) {
      const double* q = partial + ((size_t)j * blocks + b) * 3;
      num += q[0];
      den += q[1];
      mx = fmax(mx, q[2]);
    }
    const double e = sqrt(num / fmax(den, 1e-300));
    eps[(size_t)j * max_iter + k] = e;
    dsup[(size_t)j * max_iter + k] = mx;
    iters[j] = k + 1;
    if (e < tol) mask[j] = 0;
    else any = 1;
  }
  *kiter = k + 1;
  cudaGraphSetConditional(cond, (any && k + 1 < max_iter) ? 1u : 0u);
}

// Sharded device-resident Algorithm 1 (hjmc_picard_dev_pass / _decide): the per-rank block
// partials summed per horizon in the decision kernel's fixed block order, laid out [3][K]
// (Σ(v^(k+1)−v^(k))², Σ(v^(k))², max|v^(k+1)−v^(k)|) so a caller can all-reduce rows 0–1 (sum)
// and row 2 (max) in place; zeros for retired horizons.
__global__ void picard_blocksum_kernel(const double* __restrict__ partial, int K, int blocks,
                                       const int* __restrict__ mask, double* __restrict__ red) {
  if (threadIdx.x != 0) return;
  for (int j = 0; j < K; ++j) {
    double num = 0.0, den = 0.0, mx = 0.0;
    if (mask[j]) {
      for (int b = 0; b < blocks; ++b) {
        const double* q = partial + ((size_t)j * blocks + b) * 3;
        num += q[0];
        den += q[1];
        mx = fmax(mx, q[2]);
      }
    }
    red[j] = num;
    red[K + j] = den;
    red[2 * K + j] = mx;
  }
}

// Algorithm 1's stopping test on reduced [3][K] partials: the same double expression as
// picard_decide_kernel; records ε, the sup-norm difference and the iterate count of every
// active horizon, retires it when ε < tol, advances k. Without a conditional node the caller
// runs max_iter of these; once nothing is active the passes early-exit and this only counts.
__global__ void picard_decide_reduced_kernel(const double* __restrict__ red, int K, double tol,
                                             int max_iter, int* mask, int* kiter, int* iters,
                                             double* eps, double* dsup) {
  if (threadIdx.x != 0) return;
  const int k = *kiter;
  if (k >= max_iter) return;
  for (int j = 0; j < K; ++j) {
    if (!mask[j]) continue;
    const double e = sqrt(red[j] / fmax(red[K + j], 1e-300));
    eps[(size_t)j * max_iter + k] = e;
    dsup[(size_t)j * max_iter + k] = red[2 * K + j];
    iters[j] = k + 1;
    if (e < tol) mask[j] = 0;
  }
  *kiter = k + 1;
}

__global__ void picard_solve_init_kernel(int* state, int K, int32_t* iters, double* eps,
                                         double* dsup, int max_iter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < K) {
    state[i] = i + 1;
    state[K + i] = 1;
    iters[i] = 0;
  }
  if (i == 0) state[2 * K] = 0;
  for (int t = i; t < K * max_iter; t += gridDim.x * blockDim.x) {
    eps[t] = __longlong_as_double(0x7FF8000000000000LL);   // quiet NaN past each stop
    dsup[t] = __longlong_as_double(0x7FF8000000000000LL);
  }
}

}  // namespace

cudaError_t launch_picard_solve_init(int* state, int K, int32_t* iters, double* eps,
                                     double* dsup, int max_iter, cudaStream_t s) {
  const int n = std::max(K, K * max_iter);
  picard_solve_init_kernel<<<(n + 255) / 256, 256, 0, s>>>(state, K, iters, eps, dsup, max_iter);
  return cudaGetLastError();
}

cudaError_t launch_picard_blocksum(const double* partial, int K, int blocks, const int* mask,
                                   double* reduced, cudaStream_t s) {
  picard_blocksum_kernel<<<1, 32, 0, s>>>(partial, K, blocks, mask, reduced);
  return cudaGetLastError();
}

cudaError_t launch_picard_decide_reduced(const double* reduced, int K, double tol, int max_iter,
                                         int* mask, int* kiter, int* iters, double* eps,
                                         double* dsup, cudaStream_t s) {
  picard_decide_reduced_kernel<<<1, 32, 0, s>>>(reduced, K, tol, max_iter, mask, kiter, iters,
                                                eps, dsup);
  return cudaGetLastError();
}

cudaError_t launch_picard_decide(const double* partial, int K, int blocks, double tol,
                                 int max_iter, int* mask, int* kiter, int* iters, double* eps,
                                 double* dsup, cudaGraphConditionalHandle cond, cudaStream_t s) {
  picard_decide_kernel<<<1, 32, 0, s>>>(partial, K, blocks, tol, max_iter, mask, kiter, iters, eps,
                                        dsup, cond);
  return cudaGetLastError();
}

cudaError_t launch_picard_residual(const float* v, float* v_prev, int64_t M, const int* active_j,
                                   int n_active, double* partial, int blocks, cudaStream_t s) {
  if (M <= 0 || n_active <= 0) return cudaSuccess;
  picard_residual_kernel<<<dim3(blocks, n_active), 256, 0, s>>>(v, v_prev, M, active_j, partial);
  return cudaGetLastError();
}

cudaError_t launch_tube(const float* g0, const float* vfinal, int K, int64_t M, float* tube,
                        const float* x, int n, AvoidParams avoid, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  tube_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(g0, vfinal, K, M, tube, x, n, avoid);
  return cudaGetLastError();
}

cudaError_t launch_hamiltonian(const EvalParams& p, cudaStream_t s) {
  if (p.M <= 0) return cudaSuccess;
  hamiltonian_kernel<<<(unsigned)((p.M + 127) / 128), 128, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_debug_normals(int n, uint32_t qid, uint32_t jw, uint32_t kw, uint32_t i0,
                                 uint32_t count, const RoundKeys& rk, uint32_t tag, int antithetic,
                                 float* z, uint32_t* raw, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  debug_normals_kernel<<<(count + 127) / 128, 128, 0, s>>>(n, qid, jw, kw, i0, count, rk, tag,
                                                           antithetic, z, raw);
  return cudaGetLastError();
}

}  // namespace hjmc
