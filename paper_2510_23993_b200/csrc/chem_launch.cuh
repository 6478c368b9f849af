// chem_launch.cuh — host launchers of the integration kernels, declared here and defined in
// chem_launch_impl.cuh.  Each integrator (RODAS4, RODAS3, explicit) is explicitly
// instantiated in its own translation unit (launch_*.cu) so the sm_100a build compiles them in
// parallel; chem_api.cu sees only these declarations.
#pragma once
#include <cuda_runtime.h>

#include "chem_kernels.cuh"

namespace chem {

constexpr int kIntegrateBS = 32;   // threads per block of the free-running k_integrate
#ifdef CHEM_SMEM_PAD
constexpr size_t kSmemPad = CHEM_SMEM_PAD;
#else
constexpr size_t kSmemPad = 0;
#endif

template <class M, class Meth>
struct Launch {
    // bulk (refill = 0) or sparse (refill = 1) launch of k_integrate<M, Meth, kIntegrateBS>
    static cudaError_t run(const Params<M>& p, const LaunchCtx& L, const uint32_t* ids, int64_t n, int kmax,
                           int refill, int fin, int grid, cudaStream_t s);
    // lockstep bulk launch: persistent blocks, one per SM (chem_opts.lockstep)
    static cudaError_t lock(const Params<M>& p, const LaunchCtx& L, const uint32_t* ids, int64_t n, int kmax,
                            int refill, int fin, int nsm, cudaStream_t s);
    static int blocks_per_sm();
    // CHEM_SMEM_PAD (experiment builds only): extra bytes per block, to lower the resident blocks per SM
    static constexpr size_t smem() { return (size_t)SmemLayout<M, Meth>::bytes_per_thread * kIntegrateBS + kSmemPad; }
};

}  // namespace chem
