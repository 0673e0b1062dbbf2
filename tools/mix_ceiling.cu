// mix_ceiling.cu — how busy can the sm_100a XU (MUFU) pipe be kept when its instructions are
// interleaved with the other work of one C2 query·sample evaluation?
//
// A synthetic "eval" with C2's per-sample instruction mix but no memory, no reductions and no
// loop-carried latency problem (4 independent chains per thread, 4 CTAs × 256 threads per SM,
// the kernel's own occupancy): 8 MUFU (2 LG2, 2 SQRT… in the Box–Muller/target proportions),
// 12 IMAD.WIDE.U32 + 16 LOP3 (Philox share), ~14 FP32. Variants drop parts of the mix, so the
// result separates "MUFU alone" from "MUFU sharing issue/dispatch with IMAD.WIDE + LOP3". The
// achieved MUFU lane-ops/clk/SM of the full mix is the practical ceiling the real kernel's XU
// utilisation should be compared with. Output: JSON on stdout.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <map>
#include <vector>

constexpr int kIters = 512;
constexpr int kChains = 4;

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

// kInt: Philox-like integer work (12 IMAD.WIDE + 12 three-input XOR + 4 extra XOR per eval)
// kFp:  the FP32 share (≈14 per eval); kMufu: the 8 MUFU per eval
template <bool kInt, bool kFp, bool kMufu>
__global__ void __launch_bounds__(256, 4) mix(float* out, Stamp* st, uint32_t k0, float p1) {
  uint32_t u[kChains], w[kChains];
  float f[kChains], acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    u[c] = threadIdx.x * 2654435761u + c;
    w[c] = u[c] ^ 0x5bd1e995u;
    f[c] = 0.25f + threadIdx.x * 1e-4f + c * 1e-2f;
    acc[c] = 0.f;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (kInt) {
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          uint32_t h0, l0, h1, l1;
          mulw(u[c], 0xD2511F53u, h0, l0);
          mulw(w[c], 0xCD9E8D57u, h1, l1);
          u[c] = h1 ^ l0 ^ (k0 + r);
          w[c] = h0 ^ l1 ^ (k0 * 3u + r);
        }
        u[c] ^= w[c] ^ k0;
        w[c] ^= u[c] ^ 0x9E3779B9u;
        u[c] ^= w[c] ^ 0x7F4A7C15u;
        w[c] ^= u[c] ^ k0;
      }
      float x = f[c];
      if (kInt) x = __uint_as_float((u[c] >> 9) | 0x3F800000u) * x;  // consume the ints
      if (kMufu) {
        // 1.5 Box–Muller pairs (LG2, SQRT, COS, SIN ×1.5 → 6) + target SQRT + EX2 = 8
        const float r1 = sqrta(fabsf(lg2a(x)));
        const float a1 = cosa(x * 6.2831853f), b1 = sina(x * 6.2831853f);
        const float r2 = fabsf(lg2a(x + 0.5f));
        const float a2 = cosa(r2);
        const float g = sqrta(fmaf(a1, r1, x) * fmaf(b1, r1, x) + a2 * a2);
        x = ex2a(-g);
      }
      if (kFp) {
        x = fmaf(x, p1, 0.125f);
        float t = x;
#pragma unroll
        for (int q = 0; q < 6; ++q) t = fmaf(t, p1, x);
        acc[c] = fmaf(t, x, acc[c]);
        x = t * 0.5f + 0.25f;
      }
      f[c] = x;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += f[c] + acc[c] + (float)(u[c] & 1u);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) st[blockIdx.x] = Stamp{t0, t1, smid()};
}

// Parametric variant for pricing alternatives: the Philox integer share as above, kM MUFU
// (cycling LG2, SQRT, COS, EX2) and kF dependent FFMAs per eval — e.g. (8, 14) ≈ today's C2
// mix, (7, 24) ≈ one MUFU traded for a 10-FFMA polynomial, (6, 34), (5, 44).
__device__ __forceinline__ void mulsplit(uint32_t a, uint32_t m, uint32_t& hi, uint32_t& lo) {
  asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a), "r"(m));
  asm volatile("mad.lo.u32 %0, %1, %2, 0x9E3779B9;" : "=r"(lo) : "r"(a), "r"(m));
}

template <int kM, int kF, bool kSplit = false>
__global__ void __launch_bounds__(256, 4) pmix(float* out, Stamp* st, uint32_t k0, float p1) {
  uint32_t u[kChains], w[kChains];
  float f[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    u[c] = threadIdx.x * 2654435761u + c;
    w[c] = u[c] ^ 0x5bd1e995u;
    f[c] = 0.25f + threadIdx.x * 1e-4f + c * 1e-2f;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        uint32_t h0, l0, h1, l1;
        if (kSplit) {
          mulsplit(u[c], 0xD2511F53u, h0, l0);
          mulsplit(w[c], 0xCD9E8D57u, h1, l1);
        } else {
          mulw(u[c], 0xD2511F53u, h0, l0);
          mulw(w[c], 0xCD9E8D57u, h1, l1);
        }
        u[c] = h1 ^ l0 ^ (k0 + r);
        w[c] = h0 ^ l1 ^ (k0 * 3u + r);
      }
      u[c] ^= w[c] ^ k0;
      w[c] ^= u[c] ^ 0x9E3779B9u;
      u[c] ^= w[c] ^ 0x7F4A7C15u;
      w[c] ^= u[c] ^ k0;
      float x = __uint_as_float((u[c] >> 9) | 0x3F800000u) * f[c];
      float y = x;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const float a = (m & 1) ? y : x;
        float r;
        switch (m & 3) {
          case 0: r = lg2a(a); break;
          case 1: r = sqrta(fabsf(a)); break;
          case 2: r = cosa(a); break;
          default: r = ex2a(-fabsf(a)); break;
        }
        if (m & 1) y = r; else x = r;
      }
      float t = x + y;
#pragma unroll
      for (int q = 0; q < kF; ++q) t = fmaf(t, p1, (q & 1) ? x : y);
      f[c] = t * 0.5f + 0.25f;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += f[c] + (float)(u[c] & 1u);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) st[blockIdx.x] = Stamp{t0, t1, smid()};
}

// evals per SM clock: median over SMs of (evals of all CTAs on the SM) / (their clock window)
using Kern = void (*)(float*, Stamp*, uint32_t, float);
double run(Kern k, int nsm) {
  const int ctas = nsm * 4, threads = 256;
  float* out;
  Stamp* st;
  cudaMalloc(&out, sizeof(float) * ctas * threads);
  cudaMalloc(&st, sizeof(Stamp) * ctas);
  k<<<ctas, threads>>>(out, st, 0x9E3779B9u, 0.999f);
  k<<<ctas, threads>>>(out, st, 0x9E3779B9u, 0.999f);
  cudaDeviceSynchronize();
  std::vector<Stamp> h(ctas);
  cudaMemcpy(h.data(), st, sizeof(Stamp) * ctas, cudaMemcpyDeviceToHost);
  std::map<unsigned, std::vector<Stamp>> by;
  for (auto& s : h) by[s.smid].push_back(s);
  std::vector<double> rates;
  for (auto& kv : by) {
    long long lo = kv.second[0].t0, hi = kv.second[0].t1;
    for (auto& s : kv.second) { lo = std::min(lo, s.t0); hi = std::max(hi, s.t1); }
    rates.push_back((double)threads * kIters * kChains * kv.second.size() / (double)(hi - lo));
  }
  std::sort(rates.begin(), rates.end());
  cudaFree(out);
  cudaFree(st);
  return rates[rates.size() / 2];
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  struct R { const char* name; double evals_per_clk; int mufu; };
  std::vector<R> r;
  r.push_back({"mufu_only", run(mix<false, false, true>, nsm), 8});
  r.push_back({"mufu+fp32", run(mix<false, true, true>, nsm), 8});
  r.push_back({"int_only", run(mix<true, false, false>, nsm), 0});
  r.push_back({"mufu+int", run(mix<true, false, true>, nsm), 8});
  r.push_back({"full_c2_mix", run(mix<true, true, true>, nsm), 8});
  r.push_back({"p_int+8mufu+14ffma", run(pmix<8, 14>, nsm), 8});
  r.push_back({"p_int+7mufu+24ffma", run(pmix<7, 24>, nsm), 7});
  r.push_back({"p_int+6mufu+34ffma", run(pmix<6, 34>, nsm), 6});
  r.push_back({"p_int+5mufu+44ffma", run(pmix<5, 44>, nsm), 5});
  r.push_back({"p_int+8mufu+30ffma", run(pmix<8, 30>, nsm), 8});
  r.push_back({"p_splitmul+8mufu+14ffma", run(pmix<8, 14, true>, nsm), 8});
  r.push_back({"p_int+0mufu+14ffma", run(pmix<0, 14>, nsm), 0});
  r.push_back({"p_splitmul+0mufu+14ffma", run(pmix<0, 14, true>, nsm), 0});
  if (cudaGetLastError() != cudaSuccess) return 1;
  printf("{\n  \"what\": \"synthetic C2 instruction mix per eval: 8 MUFU, 12 IMAD.WIDE + 16 LOP3, ~14 FP32; "
         "evals per SM clock (median over SMs) and MUFU lane-ops/clk/SM (peak 16)\",\n  \"mixes\": {\n");
  for (size_t i = 0; i < r.size(); ++i)
    printf("    \"%s\": {\"evals_per_clk_per_sm\": %.4f, \"mufu_lane_ops_per_clk\": %.3f}%s\n", r[i].name,
           r[i].evals_per_clk, r[i].evals_per_clk * r[i].mufu, i + 1 < r.size() ? "," : "");
  printf("  }\n}\n");
  return 0;
}
