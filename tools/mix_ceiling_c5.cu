// mix_ceiling_c5.cu — the throughput ceiling of the C5 lane-group kernel's instruction mix
// (DESIGN.md §6), measured with a synthetic kernel that has the same per-lane-sample mix but no
// memory, shuffles or reductions: 48 IMAD.WIDE.U32 + 53 LOP3 (Philox of 3 blocks and the shared
// rounds), 6 Box–Muller pairs (LEA-built floats, FADD, LG2, SQRT, FMUL 2π, COS + SIN with their
// FMUL.RZ, 2 FMUL) = 24 MUFU, one SQRT + EX2 every other sample, and ~37 FFMA of target and
// moments; 2 independent samples per thread (the kernel's two-sample trips) at its occupancy
// (2 CTAs × 256 threads, 128 registers), and 1 sample at 4 CTAs × 64 registers. Output: JSON
// with lane-samples per SM clock (median over SMs) — the real kernel's figure is 4 × evals/s ÷
// (148 SMs × clock).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <map>
#include <vector>

constexpr int kIters = 256;

struct Stamp {
  long long t0, t1;
  unsigned smid;
};
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2a(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sqrta(float x) { float y; asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float cosa(float x) { float y; asm volatile("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sina(float x) { float y; asm volatile("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ void mulw(uint32_t a, uint32_t m, uint32_t& hi, uint32_t& lo) {
  asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}"
               : "=r"(lo), "=r"(hi) : "r"(a), "r"(m));
}
__device__ __forceinline__ float mant(uint32_t w) { return __uint_as_float((w >> 9) + 0x3F800000u); }

// one lane-sample; kInt / kMufu / kFp switch the parts (the weight SQRT + EX2 on odd samples)
template <bool kInt, bool kMufu, bool kFp>
__device__ __forceinline__ void lane_sample(uint32_t& u, uint32_t& w, float& acc, float x0,
                                            uint32_t k0, int odd) {
  uint32_t q[12];
#pragma unroll
  for (int b = 0; b < 3; ++b) {           // 3 Philox blocks: 16 wide multiplies + 17 XOR each
    uint32_t c0 = u + (b << 20), c1 = w ^ (b << 21), c2 = (u ^ 0x5bd1e995u) + (b << 22),
             c3 = w + 0x9E3779B9u + (b << 23);
    if (kInt) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        uint32_t h0, l0, h1, l1;
        mulw(c0, 0xD2511F53u, h0, l0);
        mulw(c2, 0xCD9E8D57u, h1, l1);
        c0 = h1 ^ c1 ^ (k0 + r);
        c2 = h0 ^ c3 ^ (k0 * 3u + r);
        c1 = l1;
        c3 = l0;
      }
      c1 ^= c0 ^ k0;
    }
    q[4 * b] = c0; q[4 * b + 1] = c1; q[4 * b + 2] = c2; q[4 * b + 3] = c3;
  }
  float z[12];
#pragma unroll
  for (int p = 0; p < 6; ++p) {           // 6 Box–Muller pairs
    const float uu = mant(q[2 * p]) - 0.99999994f;
    const float th = 6.2831853f * mant(q[2 * p + 1]);
    if (kMufu) {
      const float r = sqrta(fabsf(lg2a(uu)));
      z[2 * p] = r * cosa(th);
      z[2 * p + 1] = r * sina(th);
    } else {
      z[2 * p] = uu * th;
      z[2 * p + 1] = uu + th;
    }
  }
  float best = 3.0e38f;
  if (kFp) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float a = fmaf(0.1f, z[3 * t], x0), bb = fmaf(0.1f, z[3 * t + 1], x0);
      best = fminf(best, fmaf(a, a, bb * bb));
    }
  } else {
    best = z[0] + z[5];
  }
  float wt = best;
  if (kMufu && odd) wt = ex2a(-sqrta(best));
  if (kFp) {
#pragma unroll
    for (int c = 0; c < 12; ++c) acc = fmaf(wt, z[c], acc);
  } else {
    acc += wt;
  }
  u = q[0] ^ q[5];
  w = q[2] + q[7];
}

template <bool kInt, bool kMufu, bool kFp, int kChains, int kMinB>
__global__ void __launch_bounds__(256, kMinB) lane_mix(float* out, Stamp* st, uint32_t k0) {
  uint32_t u[kChains], w[kChains];
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    u[c] = threadIdx.x * 2654435761u + c * 977u;
    w[c] = u[c] ^ 0x5bd1e995u;
    acc[c] = 0.f;
  }
  const float x0 = 0.5f + threadIdx.x * 1e-3f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      lane_sample<kInt, kMufu, kFp>(u[c], w[c], acc[c], x0, k0, (it + c) & 1);
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c] + (float)(u[c] & 1u);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) st[blockIdx.x] = Stamp{t0, t1, smid()};
}

using Kern = void (*)(float*, Stamp*, uint32_t);
double run(Kern k, int nsm, int ctas_per_sm, int chains) {
  const int ctas = nsm * ctas_per_sm, threads = 256;
  float* out;
  Stamp* st;
  cudaMalloc(&out, sizeof(float) * ctas * threads);
  cudaMalloc(&st, sizeof(Stamp) * ctas);
  k<<<ctas, threads>>>(out, st, 0x9E3779B9u);
  k<<<ctas, threads>>>(out, st, 0x9E3779B9u);
  cudaDeviceSynchronize();
  std::vector<Stamp> h(ctas);
  cudaMemcpy(h.data(), st, sizeof(Stamp) * ctas, cudaMemcpyDeviceToHost);
  std::map<unsigned, std::vector<Stamp>> by;
  for (auto& s : h) by[s.smid].push_back(s);
  std::vector<double> rates;
  for (auto& kv : by) {
    long long lo = kv.second[0].t0, hi = kv.second[0].t1;
    for (auto& s : kv.second) { lo = std::min(lo, s.t0); hi = std::max(hi, s.t1); }
    rates.push_back((double)threads * kIters * chains * kv.second.size() / (double)(hi - lo));
  }
  std::sort(rates.begin(), rates.end());
  cudaFree(out);
  cudaFree(st);
  return rates[rates.size() / 2];
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  struct R { const char* name; double v; };
  std::vector<R> r;
  r.push_back({"full_mix_2samples_2cta", run(lane_mix<true, true, true, 2, 2>, nsm, 2, 2)});
  r.push_back({"full_mix_1sample_4cta", run(lane_mix<true, true, true, 1, 4>, nsm, 4, 1)});
  // the mix without the Philox integer work / without the MUFU ops (everything consumed)
  r.push_back({"no_int_2samples_2cta", run(lane_mix<false, true, true, 2, 2>, nsm, 2, 2)});
  r.push_back({"no_mufu_2samples_2cta", run(lane_mix<true, false, true, 2, 2>, nsm, 2, 2)});
  if (cudaGetLastError() != cudaSuccess) return 1;
  printf("{\n  \"what\": \"synthetic C5 lane-group mix per lane-sample (48 IMAD.WIDE, ~53 LOP3, 25 MUFU, "
         "~50 FP32): lane-samples per SM clock, median over SMs; the real kernel runs 4 x evals/s / "
         "(148 x clock) lane-samples per SM clock\",\n  \"mixes\": {\n");
  for (size_t i = 0; i < r.size(); ++i)
    printf("    \"%s\": {\"lane_samples_per_clk_per_sm\": %.4f}%s\n", r[i].name, r[i].v,
           i + 1 < r.size() ? "," : "");
  printf("  }\n}\n");
  return 0;
}
