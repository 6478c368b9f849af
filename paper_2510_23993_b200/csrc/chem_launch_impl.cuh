// chem_launch_impl.cuh — definitions of the launchers declared in chem_launch.cuh (included only by
// the launch_*.cu translation units, which instantiate them explicitly).
#pragma once
#include <algorithm>

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

template <class M, class Meth>
cudaError_t Launch<M, Meth>::run(const Params<M>& p, const LaunchCtx& L, const uint32_t* ids, int64_t n,
                                      int kmax, int refill, int fin, int grid, cudaStream_t s)
{
    auto kern = k_integrate<M, Meth, kIntegrateBS>;
    cudaError_t e = cudaSuccess;
    static int done_dev = -1;   // this instantiation's kernel
    if (smem() > 0) e = set_smem_once(done_dev, kern, smem());
    if (e != cudaSuccess) return e;
    kern<<<grid, kIntegrateBS, smem(), s>>>(p, L, ids, n, kmax, refill, fin);
    return cudaGetLastError();
}

template <class M, class Meth>
cudaError_t Launch<M, Meth>::lock(const Params<M>& p, const LaunchCtx& L, const uint32_t* ids, int64_t n,
                                       int kmax, int refill, int fin, int nsm, cudaStream_t s)
{
    // persistent: one block per SM walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...
    constexpr size_t b = SmemLayout<M, Meth>::bytes_per_thread;
    constexpr int BS = b == 0 ? 256 : (int)std::min<size_t>(256, (227 * 1024 / (b == 0 ? 1 : b)) / 32 * 32);
    constexpr size_t sm = b * BS;
    auto kern = k_integrate<M, Meth, BS, true>;
    static int done_dev = -1;   // this instantiation's (lockstep) kernel
    cudaError_t e = set_smem_once(done_dev, kern, sm);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<int64_t>((n + BS - 1) / BS, nsm);
    kern<<<grid, BS, sm, s>>>(p, L, ids, n, kmax, refill, fin);
    return cudaGetLastError();
}

template <class M, class Meth>
int Launch<M, Meth>::blocks_per_sm()
{
    static int dev = -1, nb = 0;
    int d = 0;
    cudaGetDevice(&d);
    if (d != dev) {
        auto kern = k_integrate<M, Meth, kIntegrateBS>;
        if (smem() > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem());
        nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kIntegrateBS, smem());
        dev = d;
    }
    return std::max(nb, 1);
}

}  // namespace chem
