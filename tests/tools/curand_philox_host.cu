// Host-side evaluation of the CUDA toolkit's own Philox4x32-10 (curand_Philox4x32_10 in
// curand_philox4x32_x.h is __host__-capable via NV_IF_ELSE_TARGET). Used ONLY as the library
// pin for the oracle's independent Philox (tests/test_oracle_rng.py). Reads lines
// "c0 c1 c2 c3 k0 k1" (decimal) on stdin and prints the four output words.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>

int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = make_uint4(c0, c1, c2, c3);
    uint2 k = make_uint2(k0, k1);
    uint4 r = curand_Philox4x32_10(c, k);
    std::printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
