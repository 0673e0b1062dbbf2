// hjmc_inst_games.cu — kernel instantiations: Dubins disk (config 2), rocket-6 (config 3).
#include "hjmc_solve_impl.cuh"

namespace hjmc {
bool lookup_games(int target, int n, KernelSet* out) {
  HJMC_CASE(1, Disk, 2)
  HJMC_CASE(1, Disk, 3)
  HJMC_CASE(1, Disk, 4)
  HJMC_CASE(1, Disk, 6)
  HJMC_CASE(2, RelDisk6, 6)
  return false;
}
}  // namespace hjmc
