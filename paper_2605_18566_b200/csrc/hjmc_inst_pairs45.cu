// hjmc_inst_pairs45.cu — kernel instantiations: the 15-pair union at n = 45 (config 5; lane
// groups) in its own translation unit so the build parallelises.
#include "hjmc_solve_impl.cuh"

namespace hjmc {
bool lookup_pairs45(int target, int n, KernelSet* out) {
  HJMC_CASE(3, PairUnion, 45)
  return false;
}
}  // namespace hjmc
