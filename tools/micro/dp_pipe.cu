// FP64 pipe microbenchmark: DFMA latency (1 chain, 1 warp) and throughput
// (ILP chains x warps) on the B200.  nvcc -arch=sm_100a -O3 dp_pipe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void chains(double *out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    if (s == 1.2345) out[0] = s;
}
static double best_per_sm = 0, best_lat = 1e30;
template <int ILP>
void run(int blocks, int threads, int iters) {
    double *d; cudaMalloc(&d, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    chains<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    chains<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = (double)blocks * threads * iters * ILP;
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("ILP %d blocks %d threads %d: %.3f ms, %.1f DFMA/clk/SM, %.2f cyc per dependent DFMA per warp\n",
           ILP, blocks, threads, ms, ops / cyc / 148.0 , cyc / iters);
    if (blocks == 148 && ops / cyc / 148.0 > best_per_sm) best_per_sm = ops / cyc / 148.0;
    if (blocks == 1 && ILP == 1) best_lat = cyc / iters;
    cudaFree(d);
}
int main() {
    run<1>(1, 32, 100000);
    run<2>(1, 32, 100000);
    run<4>(1, 32, 100000);
    run<8>(1, 32, 100000);
    run<1>(148, 128, 20000);
    run<2>(148, 128, 20000);
    run<4>(148, 128, 20000);
    run<1>(148, 256, 20000);
    run<2>(148, 256, 20000);
    run<4>(148, 256, 20000);
    run<1>(148, 512, 20000);
    run<1>(148, 1024, 20000);
    run<4>(148, 1024, 10000);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"dfma_per_clk_per_sm\": %.2f, \"dfma_latency_cyc\": %.2f, \"clock_mhz\": %.0f, "
           "\"fp64_tflops\": %.2f, \"dp_inst_per_s\": %.4e}\n", best_per_sm, best_lat, clk / 1e3,
           2.0 * best_per_sm * 148 * clk * 1e3 / 1e12, best_per_sm * 148 * clk * 1e3);
    return 0;
}
