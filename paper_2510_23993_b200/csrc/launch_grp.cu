// Explicit instantiation of the lane-group integration launchers (lanes_per_cell = 4, 8).
#include "chem_launch_impl.cuh"
namespace chem {
#define CHEM_INST(M) template struct LaunchGrp<M, Rodas4, 4>; template struct LaunchGrp<M, Rodas4, 8>; \
    template struct LaunchGrp<M, Rodas3, 4>; template struct LaunchGrp<M, Rodas3, 8>;
CHEM_FOR_EACH_MECH(CHEM_INST)
#undef CHEM_INST
}  // namespace chem
