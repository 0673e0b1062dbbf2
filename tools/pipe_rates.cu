// pipe_rates.cu — sm_100a per-pipe throughput microbenchmark (lane-ops per SM clock).
// Each thread runs 8 independent dependency chains of one instruction class; 4 CTAs × 256
// threads per SM keep every SMSP saturated; each CTA times itself with clock64(). The result
// (JSON on stdout) supplies the measured roofline denominators (profiles/pipe_rates.json).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

#define DEFINE_BENCH(NAME, TYPE, INIT, BODY, OPS_PER_BODY)                                  \
  __global__ void NAME(TYPE* out, long long* cyc, TYPE p0, TYPE p1, TYPE p2) {              \
    TYPE v[kChains];                                                                        \
    for (int c = 0; c < kChains; ++c) v[c] = INIT;                                          \
    __syncthreads();                                                                        \
    long long t0 = clock64();                                                               \
    for (int it = 0; it < kIters; ++it) {                                                   \
      _Pragma("unroll") for (int c = 0; c < kChains; ++c) { BODY; }                         \
    }                                                                                       \
    __syncthreads();                                                                        \
    long long t1 = clock64();                                                               \
    TYPE acc = v[0];                                                                        \
    for (int c = 1; c < kChains; ++c) acc = acc + v[c];                                     \
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                                       \
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                        \
  }

__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2a(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sqrta(float x) { float y; asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sina(float x) { float y; asm volatile("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

DEFINE_BENCH(b_ffma, float, p0 + threadIdx.x * 1e-7f + c, v[c] = fmaf(v[c], p1, p2), 1)
DEFINE_BENCH(b_fmul, float, p0 + threadIdx.x * 1e-7f + c, v[c] = v[c] * p1, 1)
DEFINE_BENCH(b_lop3, uint32_t, p0 + threadIdx.x + c, v[c] = v[c] ^ p1 ^ (v[c] >> 3), 2)

DEFINE_BENCH(b_imulwide, uint32_t, p0 + threadIdx.x + c,
             { uint32_t hi = __umulhi(v[c], 0xD2511F53u); v[c] = (v[c] * 0xD2511F53u) ^ hi; }, 1)
DEFINE_BENCH(b_ex2, float, p0 + threadIdx.x * 1e-6f + c * 1e-3f, v[c] = ex2a(-v[c]), 1)
DEFINE_BENCH(b_sqrt, float, p0 + 2.0f + threadIdx.x * 1e-3f + c, v[c] = sqrta(v[c]), 1)
DEFINE_BENCH(b_sin, float, p0 + threadIdx.x * 1e-6f + c * 1e-3f, v[c] = sina(v[c]), 1)
DEFINE_BENCH(b_lg2, float, p0 + 2.0f + threadIdx.x * 1e-3f + c, v[c] = lg2a(v[c]) + p1, 1)

template <typename T>
double run(void (*k)(T*, long long*, T, T, T), T p0, T p1, T p2, int nsm, const char* name,
           double ops_per_body, cudaEvent_t e0, cudaEvent_t e1, float* ms_out) {
  const int ctas_per_sm = 4, threads = 256;
  const int grid = nsm * ctas_per_sm;
  T* out; long long* cyc;
  cudaMalloc(&out, sizeof(T) * grid * threads);
  cudaMalloc(&cyc, sizeof(long long) * grid);
  k<<<grid, threads>>>(out, cyc, p0, p1, p2);  // warm
  cudaEventRecord(e0);
  k<<<grid, threads>>>(out, cyc, p0, p1, p2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms_out, e0, e1);
  std::vector<long long> h(grid);
  cudaMemcpy(h.data(), cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  const double med = (double)h[grid / 2];
  // ops per SM during one CTA's lifetime: 4 concurrent CTAs × threads × iters × chains × ops
  const double ops = (double)ctas_per_sm * threads * kIters * kChains * ops_per_body;
  cudaFree(out); cudaFree(cyc);
  return ops / med;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  printf("{\n  \"device_sms\": %d, \"clock_rate_khz\": %d,\n  \"raw\": {\n", nsm, clk);
  struct R { const char* n; double r; float ms; };
  std::vector<R> rs;
  rs.push_back({"ffma", run<float>(b_ffma, 1.0f, 0.999f, 1e-6f, nsm, "ffma", 1, e0, e1, &ms), ms});
  rs.push_back({"fmul", run<float>(b_fmul, 1.0f, 0.99999f, 0.f, nsm, "fmul", 1, e0, e1, &ms), ms});
  rs.push_back({"lop3_shift", run<uint32_t>(b_lop3, 1u, 0x9E3779B9u, 0u, nsm, "lop3", 2, e0, e1, &ms), ms});

  rs.push_back({"imul_wide_plus_xor", run<uint32_t>(b_imulwide, 1u, 0u, 0u, nsm, "imulwide", 1, e0, e1, &ms), ms});
  rs.push_back({"mufu_ex2", run<float>(b_ex2, 0.5f, 0.f, 0.f, nsm, "ex2", 1, e0, e1, &ms), ms});
  rs.push_back({"mufu_sqrt", run<float>(b_sqrt, 0.f, 0.f, 0.f, nsm, "sqrt", 1, e0, e1, &ms), ms});
  rs.push_back({"mufu_sin", run<float>(b_sin, 0.5f, 0.f, 0.f, nsm, "sin", 1, e0, e1, &ms), ms});
  rs.push_back({"mufu_lg2_plus_fadd", run<float>(b_lg2, 0.f, 2.0f, 0.f, nsm, "lg2", 1, e0, e1, &ms), ms});
  for (size_t i = 0; i < rs.size(); ++i)
    printf("    \"%s\": {\"lane_ops_per_clk_per_sm\": %.3f, \"ms\": %.4f}%s\n", rs[i].n, rs[i].r,
           rs[i].ms, i + 1 < rs.size() ? "," : "");
  printf("  }\n}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
