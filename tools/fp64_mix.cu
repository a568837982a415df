// Are the DMMA (tensor) and DFMA (fp64) pipes independent? Warps [0, nt) run DMMA chains,
// warps [nt, 8) DFMA chains, concurrently; prints the combined FP64 TFLOPS per split.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void mix(double* out, int iters, int nt, double a, double b) {
  const int warp = threadIdx.x >> 5;
  double r = 0.0;
  if (warp < nt) {
    double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        dmma(c[0], c[1], a, b); dmma(c[2], c[3], a, b); dmma(c[4], c[5], a, b); dmma(c[6], c[7], a, b);
      }
    }
    for (int k = 0; k < 8; ++k) r += c[k];
  } else {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
      }
    }
    r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 4, iters = 2048;
  double* out;
  cudaMalloc(&out, sizeof(double) * threads * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int nt = 0; nt <= 8; ++nt) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      mix<<<blocks, threads>>>(out, iters, nt, 0.999999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    // per DMMA warp: iters * 32 DMMA * 512 flop; per DFMA warp: iters * 128 * 32 lanes * 2
    const double fl = (double)blocks * iters * (nt * 32.0 * 512.0 + (8 - nt) * 128.0 * 32.0 * 2.0);
    printf("dmma warps %d / dfma warps %d: %.2f TFLOPS (%.3f ms)\n", nt, 8 - nt, fl / (best * 1e-3) / 1e12, best);
  }
  return 0;
}
