// hjmc_inst_highdim.cu — kernel instantiations: K-pair union (config 4 and smaller) and the
// paper's 14-pursuer game target at small n.
#include "hjmc_solve_impl.cuh"

namespace hjmc {
bool lookup_highdim(int target, int n, KernelSet* out) {
  HJMC_CASE(3, PairUnion, 3)
  HJMC_CASE(3, PairUnion, 6)
  HJMC_CASE(3, PairUnion, 9)
  HJMC_CASE(3, PairUnion, 15)
  HJMC_CASE(6, PursuitMin, 6)
  HJMC_CASE(6, PursuitMin, 9)
  return false;
}
}  // namespace hjmc
