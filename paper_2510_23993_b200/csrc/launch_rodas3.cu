// Explicit instantiation of the Rodas3 integration launchers for every compiled mechanism.
#include "chem_launch_impl.cuh"
namespace chem {
#define CHEM_INST(M) template struct Launch<M, Rodas3>;
CHEM_FOR_EACH_MECH(CHEM_INST)
#undef CHEM_INST
}  // namespace chem
