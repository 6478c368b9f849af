// fp64_probe.cu — B200 FP64 micro-probes for the roofline denominators.
//   dfma_peak: 148*k blocks of 256 threads, each thread runs 8 independent DFMA chains for `iters`
//              rounds (2 flops per DFMA), timed with CUDA events -> measured FP64 TFLOP/s.
//   k_exp / k_log: one libdevice exp / log per element over typical arguments; ncu's
//              sm__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum / n gives the executed
//              FP64 op count per call (the w_t of SURVEY §8(d)).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_peak(double* out, int iters, double a, double b)
{
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[blockIdx.x] = s;   // never true: keeps the chains live
}

__global__ void k_exp(const double* x, double* y, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = exp(x[i]);
}
__global__ void k_log(const double* x, double* y, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = log(x[i]);
}

int main(int argc, char** argv)
{
    int dev = 0, sms = 0;
    cudaSetDevice(dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, sizeof(double) * 1 << 20);
    const int iters = argc > 1 ? atoi(argv[1]) : 4000;
    const int blocks = sms * 8;           // 8 x 256 threads = 64 warps per SM
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_peak<<<blocks, 256>>>(out, 10, 0.999999, 1e-7);    // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dfma_peak<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * 256;
    // libdevice exp/log over typical arguments of the rate code (exp: [-60, 5]; log: [1e-20, 1e4])
    const int n = 1 << 20;
    double *x, *y;
    cudaMalloc(&x, sizeof(double) * n);
    cudaMalloc(&y, sizeof(double) * n);
    double* h = (double*)malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) h[i] = -60.0 + 65.0 * (i / (double)n);
    cudaMemcpy(x, h, sizeof(double) * n, cudaMemcpyHostToDevice);
    k_exp<<<n / 256, 256>>>(x, y, n);
    for (int i = 0; i < n; ++i) h[i] = 1e-20 * __builtin_pow(1e24, i / (double)n);
    cudaMemcpy(x, h, sizeof(double) * n, cudaMemcpyHostToDevice);
    k_log<<<n / 256, 256>>>(x, y, n);
    cudaError_t err = cudaDeviceSynchronize();
    printf("{\"probe\": \"dfma_peak\", \"sms\": %d, \"blocks\": %d, \"threads_per_block\": 256, \"iters\": %d, "
           "\"best_ms\": %.4f, \"tflops\": %.3f, \"elements_exp_log\": %d, \"cuda\": \"%s\"}\n",
           sms, blocks, iters, best, flops / (best * 1e-3) / 1e12, n, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
