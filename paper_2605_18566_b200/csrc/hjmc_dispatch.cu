// hjmc_dispatch.cu — (target id, n) → compiled kernel set (ids as in include/hjmc.h).
#include "hjmc_kernels.cuh"

namespace hjmc {
bool lookup_basic(int target, int n, KernelSet* out);
bool lookup_games(int target, int n, KernelSet* out);
bool lookup_highdim(int target, int n, KernelSet* out);
bool lookup_pairs45(int target, int n, KernelSet* out);
bool lookup_pursuit45(int target, int n, KernelSet* out);

bool lookup_kernels(int target, int n, KernelSet* out) {
  return lookup_basic(target, n, out) || lookup_games(target, n, out) ||
         lookup_highdim(target, n, out) || lookup_pairs45(target, n, out) ||
         lookup_pursuit45(target, n, out);
}
}  // namespace hjmc
