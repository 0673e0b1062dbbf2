// hjmc_inst_pursuit45.cu — kernel instantiations: the paper's 45-D pursuit-min game (
// lane groups) and the n = 15 / 45 bowls (closed-form pins).
#include "hjmc_solve_impl.cuh"

namespace hjmc {
bool lookup_pursuit45(int target, int n, KernelSet* out) {
  HJMC_CASE(6, PursuitMin, 45)
  HJMC_CASE(0, QuadBowl, 15)
  HJMC_CASE(0, QuadBowl, 45)
  return false;
}
}  // namespace hjmc
