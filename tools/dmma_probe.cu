// FP64 tensor-core probe: (1) fragment-layout check of mma.sync.m8n8k4.f64 against a
// host GEMM, (2) DMMA throughput (register-resident, all SMs).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void layout_check(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x;
  // A 8x4 row-major, B 4x8 (B[k][n] at B[k*8+n])
  double a = A[(lane >> 2) * 4 + (lane & 3)];
  double b = B[(lane & 3) * 8 + (lane >> 2)];
  double d0 = 0, d1 = 0;
  dmma(d0, d1, a, b);
  C[(lane >> 2) * 8 + (lane & 3) * 2 + 0] = d0;
  C[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = d1;
}

__global__ void dmma_tput(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(d[i][0], d[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i; hB[i] = 0.5 * i - 3.0; }
  for (int m = 0; m < 8; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += hA[m * 4 + k] * hB[k * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  layout_check<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("{\"layout_max_err\": %.3e", err);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 256);
  const int iters = 20000, blocks = sms * 4, threads = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dmma_tput<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best) best = ms;
  }
  const double flops = 2.0 * 256.0 * 8 * iters * (blocks * threads / 32);
  printf(", \"dmma_tflops\": %.2f, \"err\": \"%s\"}\n", flops / (best * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
