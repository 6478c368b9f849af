// Explicit instantiation of the launchers of the paper's explicit scheme for every
// compiled mechanism.
#include "chem_launch_impl.cuh"
namespace chem {
#define CHEM_INST(M) template struct Launch<M, Explicit>;
CHEM_FOR_EACH_MECH(CHEM_INST)
#undef CHEM_INST
}  // namespace chem
