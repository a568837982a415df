// DMMA (mma.sync.m8n8k4.f64) latency / throughput characterisation on B200:
// TFLOPS vs independent accumulator chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NC>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[NC][2];
#pragma unroll
  for (int i = 0; i < NC; ++i) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NC; ++i) dmma(d[i][0], d[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NC>
void run(int warps_per_sm, double* out) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 32 * (warps_per_sm < 8 ? warps_per_sm : 8);
  const int blocks = sms * (warps_per_sm < 8 ? 1 : warps_per_sm / 8);
  const int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(e0);
    k<NC><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best) best = ms;
  }
  const double n_dmma = (double)NC * iters * (blocks * threads / 32);
  const double tf = 512.0 * n_dmma / (best * 1e-3) / 1e12;
  // cycles per DMMA per warp (latency when NC=1 and few warps)
  const double clk = 1.965e9;
  const double cyc_per_iter = best * 1e-3 * clk / iters;
  printf("chains=%d warps/SM=%2d: %6.2f TFLOPS  %7.1f cyc/iter/warp\n", NC, warps_per_sm, tf, cyc_per_iter);
}

int main() {
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 64 * 32 * 8);
  for (int w : {1, 4, 8, 16, 32}) { run<1>(w, out); run<2>(w, out); run<4>(w, out); run<8>(w, out); }
  return 0;
}
