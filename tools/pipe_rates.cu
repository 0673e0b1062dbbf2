// pipe_rates.cu — sm_100a per-pipe throughput microbenchmark (lane-ops per SM clock).
//
// Each thread runs 8 independent dependency chains of one instruction form; 4 CTAs × 256
// threads per SM saturate every SMSP. Every CTA records its SM id and clock64() at start and
// end; per SM, rate = (lane-ops of all CTAs that ran there) / (last end − first start), and the
// median over SMs is reported. The SASS of each loop body is listed in profiles/pipe_rates.md.
// Output: JSON on stdout (the measured roofline denominators, profiles/pipe_rates.json).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <map>
#include <vector>

constexpr int kIters = 2048;
constexpr int kChains = 8;

struct Stamp {
  long long t0, t1;
  unsigned smid;
};

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

#define DEFINE_BENCH(NAME, TYPE, INIT, BODY)                                              \
  __global__ void NAME(TYPE* out, Stamp* st, TYPE p0, TYPE p1, TYPE p2) {                 \
    TYPE v[kChains];                                                                      \
    for (int c = 0; c < kChains; ++c) v[c] = INIT;                                        \
    __syncthreads();                                                                      \
    long long t0 = clock64();                                                             \
    for (int it = 0; it < kIters; ++it) {                                                 \
      _Pragma("unroll") for (int c = 0; c < kChains; ++c) { BODY; }                       \
    }                                                                                     \
    __syncthreads();                                                                      \
    long long t1 = clock64();                                                             \
    TYPE acc = v[0];                                                                      \
    for (int c = 1; c < kChains; ++c) acc = acc ^ v[c];                                   \
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                                     \
    if (threadIdx.x == 0) st[blockIdx.x] = Stamp{t0, t1, smid()};                         \
  }

#define DEFINE_FBENCH(NAME, INIT, BODY)                                                   \
  __global__ void NAME(float* out, Stamp* st, float p0, float p1, float p2) {             \
    float v[kChains];                                                                     \
    for (int c = 0; c < kChains; ++c) v[c] = INIT;                                        \
    __syncthreads();                                                                      \
    long long t0 = clock64();                                                             \
    for (int it = 0; it < kIters; ++it) {                                                 \
      _Pragma("unroll") for (int c = 0; c < kChains; ++c) { BODY; }                       \
    }                                                                                     \
    __syncthreads();                                                                      \
    long long t1 = clock64();                                                             \
    float acc = v[0];                                                                     \
    for (int c = 1; c < kChains; ++c) acc = acc + v[c];                                   \
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                                     \
    if (threadIdx.x == 0) st[blockIdx.x] = Stamp{t0, t1, smid()};                         \
  }

__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2a(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sqrta(float x) { float y; asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float cosa(float x) { float y; asm volatile("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

// FP32
DEFINE_FBENCH(b_ffma, p0 + threadIdx.x * 1e-7f + c, v[c] = fmaf(v[c], p1, p2))
DEFINE_FBENCH(b_fadd, p0 + threadIdx.x * 1e-7f + c, v[c] = v[c] + p1)
// integer multiply forms (each body: the multiply + one LOP3 on the ALU pipe to keep values moving)
DEFINE_BENCH(b_imad_wide, uint32_t, (uint32_t)p0 + threadIdx.x + c,
             { uint32_t hi = __umulhi(v[c], 0xD2511F53u); v[c] = (v[c] * 0xD2511F53u) ^ hi; })
DEFINE_BENCH(b_imad_lo, uint32_t, (uint32_t)p0 + threadIdx.x + c, v[c] = v[c] * 0xD2511F53u + p1)
DEFINE_BENCH(b_imad_hi, uint32_t, (uint32_t)p0 + threadIdx.x + c,
             v[c] = __umulhi(v[c], 0xD2511F53u) ^ (p1 + c))
// logic (ALU pipe): 3-input XOR chains across neighbouring chains
DEFINE_BENCH(b_lop3, uint32_t, (uint32_t)p0 + threadIdx.x * 7u + c,
             v[c] = v[c] ^ v[(c + 3) % kChains] ^ (p1 + c))
// FP64 (DFMA) and the exact Philox high word on the FP64 pipe (hjmc_rng.cuh mulhi_dfma):
// {c, 0x43300000} = 2^52 + c; fma.rm(2^52 + c, M·2^-32, 2^52 − 2^20·M) = 2^52 + mulhi(c, M)
#define DEFINE_DBENCH(NAME, INIT, BODY)                                                   \
  __global__ void NAME(double* out, Stamp* st, double p0, double p1, double p2) {         \
    double v[kChains];                                                                    \
    for (int c = 0; c < kChains; ++c) v[c] = INIT;                                        \
    __syncthreads();                                                                      \
    long long t0 = clock64();                                                             \
    for (int it = 0; it < kIters; ++it) {                                                 \
      _Pragma("unroll") for (int c = 0; c < kChains; ++c) { BODY; }                       \
    }                                                                                     \
    __syncthreads();                                                                      \
    long long t1 = clock64();                                                             \
    double acc = v[0];                                                                    \
    for (int c = 1; c < kChains; ++c) acc = acc + v[c];                                   \
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                                     \
    if (threadIdx.x == 0) st[blockIdx.x] = Stamp{t0, t1, smid()};                         \
  }
DEFINE_DBENCH(b_dfma, p0 + threadIdx.x * 1e-9 + c, v[c] = fma(v[c], p1, p2))
__device__ __forceinline__ uint32_t mulhi_dfma_pr(uint32_t c) {
  constexpr uint32_t kM = 0xD2511F53u;
  const double b = (double)kM * (1.0 / 4294967296.0), k = 4503599627370496.0 - 1048576.0 * (double)kM;
  double a = __hiloint2double(0x43300000, (int)c), r;
  asm volatile("fma.rm.f64 %0, %1, %2, %3;" : "=d"(r) : "d"(a), "d"(b), "d"(k));
  return (uint32_t)__double2loint(r);
}
// body: mulhi on the FP64 pipe + the low word by IMAD + one LOP3 (the IMAD.WIDE body's work)
DEFINE_BENCH(b_dfma_mulhi, uint32_t, (uint32_t)p0 + threadIdx.x + c,
             { uint32_t hi = mulhi_dfma_pr(v[c]); v[c] = (v[c] * 0xD2511F53u) ^ hi; })
// body: mulhi on the FP64 pipe + one LOP3 (no low word): the FP64 pipe's own rate for the trick
DEFINE_BENCH(b_dfma_mulhi_only, uint32_t, (uint32_t)p0 + threadIdx.x + c,
             v[c] = mulhi_dfma_pr(v[c]) ^ (p1 + c))
__global__ void check_dfma_mulhi(const uint32_t* in, unsigned* bad, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && mulhi_dfma_pr(in[i]) != __umulhi(in[i], 0xD2511F53u)) atomicAdd(bad, 1u);
}

// MUFU (XU pipe)
DEFINE_FBENCH(b_ex2, p0 + threadIdx.x * 1e-6f + c * 1e-3f, v[c] = ex2a(-v[c]))
DEFINE_FBENCH(b_sqrt, p0 + 2.0f + threadIdx.x * 1e-3f + c, v[c] = sqrta(v[c]))
DEFINE_FBENCH(b_lg2, p0 + 2.0f + threadIdx.x * 1e-3f + c, v[c] = lg2a(v[c]) + p1)
DEFINE_FBENCH(b_cos, p0 + threadIdx.x * 1e-6f + c * 1e-3f, v[c] = cosa(v[c]))

struct Result {
  const char* name;
  const char* pipe;
  double lane_ops_per_clk;
};

template <typename T>
double run(void (*k)(T*, Stamp*, T, T, T), T p0, T p1, T p2, int nsm) {
  const int ctas = nsm * 4, threads = 256;
  T* out;
  Stamp* st;
  cudaMalloc(&out, sizeof(T) * ctas * threads);
  cudaMalloc(&st, sizeof(Stamp) * ctas);
  k<<<ctas, threads>>>(out, st, p0, p1, p2);  // warm-up
  k<<<ctas, threads>>>(out, st, p0, p1, p2);
  cudaDeviceSynchronize();
  std::vector<Stamp> h(ctas);
  cudaMemcpy(h.data(), st, sizeof(Stamp) * ctas, cudaMemcpyDeviceToHost);
  std::map<unsigned, std::vector<Stamp>> by;
  for (auto& s : h) by[s.smid].push_back(s);
  std::vector<double> rates;
  const double ops_per_cta = (double)threads * kIters * kChains;  // one op per body
  for (auto& kv : by) {
    long long lo = kv.second[0].t0, hi = kv.second[0].t1;
    for (auto& s : kv.second) { lo = std::min(lo, s.t0); hi = std::max(hi, s.t1); }
    rates.push_back(ops_per_cta * kv.second.size() / (double)(hi - lo));
  }
  std::sort(rates.begin(), rates.end());
  cudaFree(out);
  cudaFree(st);
  return rates[rates.size() / 2];
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::vector<Result> r;
  r.push_back({"ffma", "fp32", run<float>(b_ffma, 1.0f, 0.999f, 1e-6f, nsm)});
  r.push_back({"fadd", "fp32", run<float>(b_fadd, 1.0f, 1e-7f, 0.f, nsm)});
  r.push_back({"imad_wide_u32 (+lop3)", "imul", run<uint32_t>(b_imad_wide, 1u, 0u, 0u, nsm)});
  r.push_back({"imad_lo", "imad_lo", run<uint32_t>(b_imad_lo, 1u, 0x9E3779B9u, 0u, nsm)});
  r.push_back({"imad_hi (+lop3)", "imad_hi", run<uint32_t>(b_imad_hi, 1u, 0x9E3779B9u, 0u, nsm)});
  r.push_back({"lop3", "alu", run<uint32_t>(b_lop3, 1u, 0x9E3779B9u, 0u, nsm)});
  r.push_back({"dfma", "fp64", run<double>(b_dfma, 1.0, 0.999999, 1e-9, nsm)});
  r.push_back({"dfma_mulhi + imad_lo (+lop3)", "fp64+imad", run<uint32_t>(b_dfma_mulhi, 1u, 0u, 0u, nsm)});
  r.push_back({"dfma_mulhi (+lop3)", "fp64", run<uint32_t>(b_dfma_mulhi_only, 1u, 0x9E3779B9u, 0u, nsm)});
  r.push_back({"mufu_ex2", "mufu", run<float>(b_ex2, 0.5f, 0.f, 0.f, nsm)});
  r.push_back({"mufu_sqrt", "mufu_sqrt", run<float>(b_sqrt, 0.f, 0.f, 0.f, nsm)});
  r.push_back({"mufu_lg2 (+fadd)", "mufu_lg2", run<float>(b_lg2, 0.f, 2.0f, 0.f, nsm)});
  r.push_back({"mufu_cos (+fmul.rz)", "mufu_cos", run<float>(b_cos, 0.5f, 0.f, 0.f, nsm)});
  // exactness of the FP64 high word on 2^24 inputs (edge words + a multiplicative sweep)
  unsigned long long bad_total = 0;
  {
    const int n = 1 << 24;
    std::vector<uint32_t> h(n);
    uint32_t x = 0x12345678u;
    for (int i = 0; i < n; ++i) { x = x * 1664525u + 1013904223u; h[i] = x; }
    const uint32_t edges[] = {0u, 1u, 2u, 0x7FFFFFFFu, 0x80000000u, 0xFFFFFFFEu, 0xFFFFFFFFu};
    for (int i = 0; i < 7; ++i) h[i] = edges[i];
    uint32_t* d; unsigned* b;
    cudaMalloc(&d, sizeof(uint32_t) * n); cudaMalloc(&b, sizeof(unsigned));
    cudaMemcpy(d, h.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice);
    cudaMemset(b, 0, sizeof(unsigned));
    check_dfma_mulhi<<<(n + 255) / 256, 256>>>(d, b, n);
    unsigned hb = 0;
    cudaMemcpy(&hb, b, sizeof(unsigned), cudaMemcpyDeviceToHost);
    bad_total = hb;
    cudaFree(d); cudaFree(b);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  printf("{\n  \"device_sms\": %d, \"clock_rate_khz\": %d,\n", nsm, clk);
  printf("  \"dfma_mulhi_mismatches_of_2^24\": %llu,\n", bad_total);
  printf("  \"method\": \"per-SM clock64 window over 4 CTAs x 256 threads x 8 chains; median over SMs\",\n");
  printf("  \"raw\": {\n");
  for (size_t i = 0; i < r.size(); ++i)
    printf("    \"%s\": {\"pipe\": \"%s\", \"lane_ops_per_clk_per_sm\": %.3f}%s\n", r[i].name,
           r[i].pipe, r[i].lane_ops_per_clk, i + 1 < r.size() ? "," : "");
  printf("  }\n}\n");
  return 0;
}
