// dmma_probe.cu — NEXT-3 DMMA re-test (SURVEY.md §8(a) A4 "DMMA decision", §8(f) NEXT-3; PAPER.md
// the GEMM form of the rates pays only for big grids and mechanisms).
//
// The contraction timed: X[cell, r] = sum_k nu'[k, r] ln c[cell, k]  ([cells x Ns] . [Ns x Nr]), the
// forward half of the matrix-form rates, for three shapes (dmma_shapes.cuh): the 9x21 H2-air and
// 14x41 GRI H/O/N mechanisms of this repo and a 53x325 GRI-Mech-3.0-shaped pattern.  Three kernels
// do the same algorithmic work (2 nnz(nu') flops per cell), each consuming every X[cell, r] into a
// checksum and updating its inputs every repetition (ln c += 1e-3, Ns DADDs per cell):
//   sparse : FP64 CUDA cores, compile-time sparse pattern (what k_integrate does)
//   dense  : FP64 CUDA cores, all Ns x Nr products with nu' read from memory (no zero skipping)
//   dmma   : FP64 tensor cores, mma.sync.aligned.m8n8k4.row.col.f64 per 8 cells x 8 rows x 4 species,
//            nu' fragments from shared memory, ln c fragments in registers (K, N padded to 4, 8)
// Prints one JSON line per (shape, kernel): ms, cells/s, algorithmic GFLOP/s.
// Build: nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -o dmma_probe dmma_probe.cu
#include <cstdint>
#include <utility>
#include <cstdio>
#include <cuda_runtime.h>

#include "dmma_shapes.cuh"

template <class F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>)
{
    (f(std::integral_constant<int, I>{}), ...);
}
template <int B, int E, class F>
__device__ __forceinline__ void sfor(F&& f)   // B = 0 only: a fold over 0..E-1 (no recursion depth)
{
    static_assert(B == 0, "sfor starts at 0");
    sfor_impl(f, std::make_integer_sequence<int, E>{});
}

__device__ __forceinline__ double lnc_of(uint32_t cell, int k)
{
    uint32_t x = cell * 0x9E3779B1u ^ ((uint32_t)k * 0x85EBCA77u);
    x ^= x >> 15;
    x *= 0x2C1B3C6Du;
    x ^= x >> 12;
    return -30.0 + 35.0 * (double)(x & 0xFFFFFFu) * (1.0 / 16777216.0);
}

template <class S>
__global__ void __launch_bounds__(256) k_sparse(double* out, int reps)
{
    const uint32_t cell = blockIdx.x * blockDim.x + threadIdx.x;
    double l[S::NS];
#pragma unroll
    for (int k = 0; k < S::NS; ++k) l[k] = lnc_of(cell, k);
    double cs = 0.0;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
        for (int k = 0; k < S::NS; ++k) l[k] += 1e-3;
        sfor<0, S::NR>([&](auto r_) {
            constexpr int r = decltype(r_)::value;
            double a = 0.0;
            sfor<0, S::nreac(r)>([&](auto i_) { a += l[S::reac(r, decltype(i_)::value)]; });
            cs += a;
        });
    }
    out[cell] = cs;
}

// nu' of the shape being run, in global memory read through the read-only cache (uniform addresses
// across the warp; the 53 x 325 table exceeds the 64 KB constant bank)
__device__ double gNu[53 * 325];
template <class S>
struct CNu {
    static __device__ __forceinline__ double v(int k, int r) { return __ldg(&gNu[k * S::NR + r]); }
};

template <class S>
__global__ void __launch_bounds__(256) k_dense(double* out, int reps)
{
    const uint32_t cell = blockIdx.x * blockDim.x + threadIdx.x;
    double l[S::NS];
#pragma unroll
    for (int k = 0; k < S::NS; ++k) l[k] = lnc_of(cell, k);
    double cs = 0.0;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
        for (int k = 0; k < S::NS; ++k) l[k] += 1e-3;
#pragma unroll 4
        for (int r = 0; r < S::NR; ++r) {
            double a = 0.0;
#pragma unroll
            for (int k = 0; k < S::NS; ++k) a = fma(CNu<S>::v(k, r), l[k], a);
            cs += a;
        }
    }
    out[cell] = cs;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// one warp = 32 cells = 4 m-tiles of 8; lane: A[m = lane/4][k = lane%4], B[k = lane%4][n = lane/4],
// D[m = lane/4][n = 2(lane%4) + {0, 1}]
template <class S>
__global__ void __launch_bounds__(256) k_dmma(double* out, int reps)
{
    constexpr int KQ = (S::NS + 3) / 4, NJ = (S::NR + 7) / 8;
    extern __shared__ double sB[];            // [KQ][NJ][32] fragments
    for (int i = threadIdx.x; i < KQ * NJ * 32; i += blockDim.x) {
        const int lane = i & 31, j = (i >> 5) % NJ, q = (i >> 5) / NJ;
        const int k = 4 * q + (lane & 3), n = 8 * j + (lane >> 2);
        sB[i] = (k < S::NS && n < S::NR) ? CNu<S>::v(k, n) : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t wbase = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u;
    double a[4][KQ];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int q = 0; q < KQ; ++q) {
            const int k = 4 * q + (lane & 3);
            a[t][q] = k < S::NS ? lnc_of(wbase + 8 * t + (lane >> 2), k) : 0.0;
        }
    double cs = 0.0;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int q = 0; q < KQ; ++q)
                if (4 * q + (lane & 3) < S::NS) a[t][q] += 1e-3;
#pragma unroll 1
        for (int j = 0; j < NJ; ++j) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int q = 0; q < KQ; ++q) dmma(d0, d1, a[t][q], sB[(q * NJ + j) * 32 + lane]);
                cs += d0 + d1;
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = cs;
}

template <class S>
void run(const char* name, double* out, int cells, int reps)
{
    cudaMemcpyToSymbol(gNu, S::nu, sizeof(S::nu));
    constexpr int KQ = (S::NS + 3) / 4, NJ = (S::NR + 7) / 8;
    const size_t smem = (size_t)KQ * NJ * 32 * 8;
    cudaFuncSetAttribute(k_dmma<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = cells / 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double alg = 2.0 * S::NNZ;        // algorithmic flops per cell per repetition
    for (int v = 0; v < 3; ++v) {
        auto launch = [&] {
            if (v == 0) k_sparse<S><<<grid, 256>>>(out, reps);
            else if (v == 1) k_dense<S><<<grid, 256>>>(out, reps);
            else k_dmma<S><<<grid, 256, smem>>>(out, reps);
        };
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int i = 0; i < 3; ++i) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const char* kn[3] = {"sparse_fp64", "dense_fp64", "dmma_m8n8k4"};
        const double padded = v == 2 ? 2.0 * (4 * KQ) * (8 * NJ) : v == 1 ? 2.0 * S::NS * S::NR : alg;
        printf("{\"shape\": \"%s\", \"Ns\": %d, \"Nr\": %d, \"nnz\": %d, \"kernel\": \"%s\", \"ms\": %.4f, "
               "\"cells_per_s\": %.4e, \"alg_gflops\": %.1f, \"executed_gflops\": %.1f, \"smem_bytes\": %zu, "
               "\"err\": \"%s\"}\n",
               name, S::NS, S::NR, S::NNZ, kn[v], best, (double)cells * reps / (best * 1e-3),
               alg * cells * reps / (best * 1e-3) / 1e9, padded * cells * reps / (best * 1e-3) / 1e9,
               v == 2 ? smem : (size_t)0, cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
    }
}

int main()
{
    const int cells = 148 * 8 * 256 * 4;       // 4 waves of 8 x 256-thread blocks per SM
    double* out;
    cudaMalloc(&out, sizeof(double) * cells);
    run<Shape_h2air>("h2air_9x21", out, cells, 200);
    run<Shape_gri14>("gri30_hon_14x41", out, cells, 100);
    run<Shape_gri53>("gri53_shape_53x325", out, cells / 4, 10);
    return 0;
}
