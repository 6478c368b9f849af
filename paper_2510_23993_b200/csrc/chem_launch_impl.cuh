// chem_launch_impl.cuh — definitions of the launchers declared in chem_launch.cuh (included only by
// the launch_*.cu translation units, which instantiate them explicitly).
#pragma once
#include <algorithm>

#include "chem_group.cuh"
#include "chem_launch.cuh"

namespace chem {

// cudaFuncSetAttribute / occupancy queries are host API calls of ~10 us each: do them once per kernel
// and device (one process drives one GPU) instead of per launch.  `done_dev` must be a static of the
// caller's own instantiation (one per kernel): a static keyed on the kernel's function-pointer TYPE
// would be shared by every k_integrate variant with the same signature.
template <class K>
inline cudaError_t set_smem_once(int& done_dev, K kern, size_t bytes)
{
    int d = 0;
    cudaGetDevice(&d);
    if (d == done_dev) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done_dev = d;
    return e;
}

template <class M, class Meth, bool DAE>
cudaError_t Launch<M, Meth, DAE>::run(const Params<M>& p, const LaunchCtx& L, const uint32_t* ids, int64_t n,
                                      int kmax, int refill, int fin, int grid, cudaStream_t s)
{
    auto kern = k_integrate<M, Meth, kIntegrateBS, DAE>;
    cudaError_t e = cudaSuccess;
    static int done_dev = -1;   // this instantiation's kernel
    if (smem() > 0) e = set_smem_once(done_dev, kern, smem());
    if (e != cudaSuccess) return e;
    kern<<<grid, kIntegrateBS, smem(), s>>>(p, L, ids, n, kmax, refill, fin);
    return cudaGetLastError();
}

template <class M, class Meth, bool DAE>
cudaError_t Launch<M, Meth, DAE>::lock(const Params<M>& p, const LaunchCtx& L, const uint32_t* ids, int64_t n,
                                       int kmax, int refill, int fin, int nsm, cudaStream_t s)
{
    // persistent: one block per SM walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...
    constexpr size_t b = SmemLayout<M, Meth, DAE>::bytes_per_thread;
    constexpr int BS = b == 0 ? 256 : (int)std::min<size_t>(256, (227 * 1024 / (b == 0 ? 1 : b)) / 32 * 32);
    constexpr size_t sm = b * BS;
    auto kern = k_integrate<M, Meth, BS, DAE, true>;
    static int done_dev = -1;   // this instantiation's (lockstep) kernel
    cudaError_t e = set_smem_once(done_dev, kern, sm);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<int64_t>((n + BS - 1) / BS, nsm);
    kern<<<grid, BS, sm, s>>>(p, L, ids, n, kmax, refill, fin);
    return cudaGetLastError();
}

template <class M, class Meth, bool DAE>
int Launch<M, Meth, DAE>::blocks_per_sm()
{
    static int dev = -1, nb = 0;
    int d = 0;
    cudaGetDevice(&d);
    if (d != dev) {
        auto kern = k_integrate<M, Meth, kIntegrateBS, DAE>;
        if (smem() > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem());
        nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kIntegrateBS, smem());
        dev = d;
    }
    return std::max(nb, 1);
}

template <class M, class Meth, int G>
cudaError_t LaunchGrp<M, Meth, G>::run(const void* gt, const LaunchCtx& L, const uint32_t* ids, int64_t n, int kmax,
                                       int refill, int fin, int grid, cudaStream_t s)
{
    auto kern = k_integrate_grp<M, Meth, G, kGrpBS>;
    const size_t sm = grp_smem_bytes<M, G>(kGrpBS);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    kern<<<grid, kGrpBS, sm, s>>>(static_cast<const GTable<M>*>(gt), L, ids, n, kmax, refill, fin);
    return cudaGetLastError();
}

template <class M, class Meth, int G>
int LaunchGrp<M, Meth, G>::blocks_per_sm()
{
    int nb = 0;
    auto kern = k_integrate_grp<M, Meth, G, kGrpBS>;
    const size_t sm = grp_smem_bytes<M, G>(kGrpBS);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kGrpBS, sm);
    return std::max(nb, 1);
}

}  // namespace chem
