/* c_api_demo.c — using libhjmc from plain C (no Python, no torch): the C-ABI is the product
 * boundary. Solves a small Dubins slice (config-2 physics, reduced N) twice — once through the
 * device-pointer entry point with explicit cudaMalloc'd buffers, once through the host-buffer
 * convenience call — and checks the two agree bit for bit, then prints a JSON line.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_2605_18566_b200 -lhjmc \
 *       -I /usr/local/cuda/include -L /usr/local/cuda/lib64 -lcudart -lm -o c_api_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hjmc.h"

#define CHECK(call)                                                                        \
  do {                                                                                     \
    int rc_ = (call);                                                                      \
    if (rc_ != HJMC_OK) {                                                                  \
      fprintf(stderr, "%s failed: %d (%s)\n", #call, rc_, hjmc_last_error(h));             \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

int main(void) {
  const int side = 21, n = 3;
  const int64_t M = (int64_t)side * side;
  hjmc_config cfg;
  hjmc_config_defaults(&cfg);
  cfg.n = n;
  cfg.delta = 0.01f;
  cfg.T = 1.0f;
  cfg.K = 4;
  cfg.Kp = 3;
  cfg.N = 8192;
  hjmc_handle* h = NULL;
  if (hjmc_create(&cfg, &h) != HJMC_OK) {
    fprintf(stderr, "hjmc_create: %s\n", hjmc_last_error(NULL));
    return 1;
  }
  const float dubins[3] = {5.f, 5.f, 1.f}, disk[1] = {5.f};
  CHECK(hjmc_set_dynamics(h, HJMC_SYS_DUBINS_REL, dubins, 3));
  CHECK(hjmc_set_target(h, HJMC_TGT_DISK, disk, 1));

  float* x = (float*)malloc(sizeof(float) * M * n);
  for (int a = 0; a < side; ++a)
    for (int b = 0; b < side; ++b) {
      float* q = x + ((int64_t)a * side + b) * n;
      q[0] = -20.f + 40.f * a / (side - 1);
      q[1] = -20.f + 40.f * b / (side - 1);
      q[2] = 1.5707964f;
    }

  /* device path */
  float *dx, *dv, *dtube;
  cudaMalloc((void**)&dx, sizeof(float) * M * n);
  cudaMalloc((void**)&dv, sizeof(float) * M);
  cudaMalloc((void**)&dtube, sizeof(float) * M);
  cudaMemcpy(dx, x, sizeof(float) * M * n, cudaMemcpyHostToDevice);
  hjmc_result dres;
  memset(&dres, 0, sizeof(dres));
  dres.v = dv;
  dres.tube = dtube;
  CHECK(hjmc_solve_slice(h, dx, NULL, 0, M, NULL, &dres, NULL));
  CHECK(hjmc_check(h, NULL));
  float* v1 = (float*)malloc(sizeof(float) * M);
  float* t1 = (float*)malloc(sizeof(float) * M);
  cudaMemcpy(v1, dv, sizeof(float) * M, cudaMemcpyDeviceToHost);
  cudaMemcpy(t1, dtube, sizeof(float) * M, cudaMemcpyDeviceToHost);

  /* host path */
  float* v2 = (float*)malloc(sizeof(float) * M);
  float* t2 = (float*)malloc(sizeof(float) * M);
  hjmc_result hres;
  memset(&hres, 0, sizeof(hres));
  hres.v = v2;
  hres.tube = t2;
  CHECK(hjmc_solve_slice_host(h, x, NULL, 0, M, NULL, &hres));

  int same = memcmp(v1, v2, sizeof(float) * M) == 0 && memcmp(t1, t2, sizeof(float) * M) == 0;
  int inside = 0;
  double vmin = 1e30, vmax = -1e30;
  for (int64_t m = 0; m < M; ++m) {
    inside += t1[m] <= 0.f;
    vmin = fmin(vmin, v1[m]);
    vmax = fmax(vmax, v1[m]);
  }
  uint64_t passes = 0;
  CHECK(hjmc_pass_count(h, NULL, &passes));

  /* Algorithm 1 on the device: Kp passes, tol = 0 → the last horizon's v equals the fixed
   * schedule's v (same counters, same kernels) */
  const int K = cfg.K, Kp = cfg.Kp;
  float *pv, *pc;
  int32_t* piters;
  double *peps, *pdsup;
  cudaMalloc((void**)&pv, sizeof(float) * K * M);
  cudaMalloc((void**)&pc, sizeof(float) * K * M);
  cudaMalloc((void**)&piters, sizeof(int32_t) * K);
  cudaMalloc((void**)&peps, sizeof(double) * K * Kp);
  cudaMalloc((void**)&pdsup, sizeof(double) * K * Kp);
  CHECK(hjmc_picard_solve(h, dx, NULL, 0, M, NULL, 0.0, Kp, pv, NULL, pc, piters, peps, pdsup, NULL,
                          NULL));
  cudaDeviceSynchronize();
  float* v3 = (float*)malloc(sizeof(float) * M);
  int32_t iters[64];
  double eps_last = 0.0;
  cudaMemcpy(v3, pv + (size_t)(K - 1) * M, sizeof(float) * M, cudaMemcpyDeviceToHost);
  cudaMemcpy(iters, piters, sizeof(int32_t) * K, cudaMemcpyDeviceToHost);
  cudaMemcpy(&eps_last, peps + (size_t)(K - 1) * Kp + (Kp - 1), sizeof(double), cudaMemcpyDeviceToHost);
  int picard_same = memcmp(v1, v3, sizeof(float) * M) == 0 && iters[K - 1] == Kp;
  printf("{\"version\": %d, \"M\": %lld, \"identical_device_host\": %s, \"brt_points\": %d, "
         "\"v_min\": %.6f, \"v_max\": %.6f, \"passes\": %llu, "
         "\"picard_graph_matches_fixed_schedule\": %s, \"eps_last\": %.6g}\n",
         hjmc_version(), (long long)M, same ? "true" : "false", inside, vmin, vmax,
         (unsigned long long)passes, picard_same ? "true" : "false", eps_last);
  hjmc_destroy(h);
  cudaFree(dx);
  cudaFree(dv);
  cudaFree(dtube);
  cudaFree(pv); cudaFree(pc); cudaFree(piters); cudaFree(peps); cudaFree(pdsup);
  free(x); free(v1); free(t1); free(v2); free(t2); free(v3);
  return (same && picard_same) ? 0 : 2;
}
