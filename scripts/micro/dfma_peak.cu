// FP64 pipe peak on this GPU (SURVEY §8d asks for a measured DFMA peak; it is
// not in MEASURED_PEAKS.json).  Each thread runs 8 independent DFMA chains
// (enough to cover the pipe latency at full occupancy); one DADD variant
// checks that DADD issues at the same rate.  Prints one JSON line.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dfma_peak dfma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;
constexpr int ITERS = 4096;

template <bool ADD>
__global__ void __launch_bounds__(256) k_fp64(double *out, double a, double b) {
    double v[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) v[c] = ADD ? v[c] + a : fma(v[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += v[c];
    if (s == 12345.678) out[0] = s;   // keeps the chains live
}

template <bool ADD>
static double run(int sms, double *out) {
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fp64<ADD><<<blocks, threads>>>(out, 0.999999, 1e-7);   // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fp64<ADD><<<blocks, threads>>>(out, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = (double)blocks * threads * ITERS * CH;   // instructions (thread level)
    return ops / (best * 1e-3);
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double *out;
    cudaMalloc(&out, sizeof(double));
    const double fma_ops = run<false>(sms, out), add_ops = run<true>(sms, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "%s\n", cudaGetErrorString(e));
        return 1;
    }
    const double clk_hz = clk * 1e3;
    printf("{\"dfma_per_s\": %.4e, \"dadd_per_s\": %.4e, \"fp64_tflops\": %.3f, \"dfma_per_sm_per_clk\": %.2f, "
           "\"sms\": %d, \"clock_mhz_attr\": %.0f, \"how\": \"8 independent DFMA (DADD) chains per thread, "
           "%d CTAs x 256 threads, best of 5, CUDA events; TFLOP/s counts an FMA as 2\"}\n",
           fma_ops, add_ops, 2.0 * fma_ops / 1e12, fma_ops / sms / clk_hz, sms, clk_hz / 1e6, sms * 8);
    return 0;
}
