// FP64 DFMA throughput probe (register-resident independent chains, all SMs).
// Used to pin the FP64 ceiling for the "alu" roofline of the fused apply.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_chains(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  double* out;
  cudaMalloc(&out, sizeof(double) * threads * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 8; ++rep) {
    cudaEventRecord(e0);
    dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double fma = (double)threads * blocks * iters * 16 * 8;
  const double tflops = 2.0 * fma / (best * 1e-3) / 1e12;
  printf("{\"fp64_dfma_tflops\": %.3f, \"dfma_per_clk_per_sm_at_reported_clock\": %.2f, \"sms\": %d, \"clock_mhz\": %.0f, \"ms\": %.4f}\n",
         tflops, fma / (best * 1e-3) / sms / (clk * 1e3), sms, clk / 1e3, best);
  return 0;
}
