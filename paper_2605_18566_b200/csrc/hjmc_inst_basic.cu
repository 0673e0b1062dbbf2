// hjmc_inst_basic.cu — kernel instantiations: quadratic bowl (config 1) and the test targets.
#include "hjmc_solve_impl.cuh"

namespace hjmc {
bool lookup_basic(int target, int n, KernelSet* out) {
  HJMC_CASE(0, QuadBowl, 1)
  HJMC_CASE(0, QuadBowl, 2)
  HJMC_CASE(0, QuadBowl, 3)
  HJMC_CASE(0, QuadBowl, 4)
  HJMC_CASE(0, QuadBowl, 6)
  HJMC_CASE(0, QuadBowl, 8)
  HJMC_CASE(4, Linear, 1)
  HJMC_CASE(4, Linear, 2)
  HJMC_CASE(4, Linear, 3)
  HJMC_CASE(4, Linear, 4)
  HJMC_CASE(4, Linear, 6)
  HJMC_CASE(5, Const, 1)
  HJMC_CASE(5, Const, 2)
  HJMC_CASE(5, Const, 3)
  HJMC_CASE(5, Const, 4)
  HJMC_CASE(5, Const, 6)
  return false;
}
}  // namespace hjmc
