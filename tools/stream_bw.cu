// Streaming microbenchmark for the access pattern of the lockstep CG loop's phases B / C:
// S vectors of N doubles, every CTA owns a row range (N / grid), each warp step loads a run of
// RUNB bytes of every stream (lanes split into RUNB / 16 lanes per stream, 16-byte loads).
// layout 0: each warp its own contiguous sub-range (the loop's current layout);
// layout 1: the CTA's warps interleaved step by step (8 warps x RUNB contiguous per stream).
// Usage: stream_bw N S   (prints GB/s per (RUNB, layout, unroll, write fraction))
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int RUNB, int U>
__global__ void __launch_bounds__(256, 2) kstream(const double* __restrict__ base, double* out, long N, int S,
                                                  int layout, int wr, double* wbase) {
  constexpr int LPS = RUNB / 16;        // lanes per stream
  constexpr int SPI = 32 / LPS;         // streams per instruction
  constexpr int ROWS = RUNB / 8;        // rows per step
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long rpc = ((N / gridDim.x) + 63) / 64 * 64;
  const long cbeg = (long)blockIdx.x * rpc, cend = min(N, cbeg + rpc);
  long wbeg, wend, wstep;
  if (layout == 0) {
    const long rpw = rpc / 8;
    wbeg = cbeg + warp * rpw;
    wend = min(cend, wbeg + rpw);
    wstep = ROWS;
  } else {
    wbeg = cbeg + warp * ROWS;
    wend = cend;
    wstep = 8 * ROWS;
  }
  const int sl = lane / LPS, sub = lane % LPS;
  double acc = 0.0;
  for (long r0 = wbeg; r0 < wend; r0 += U * wstep) {
    double2 v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long row = r0 + u * wstep + 2 * sub;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int s = i * SPI + sl;
        v[u][i] = make_double2(0.0, 0.0);
        if (s < S && row < wend) v[u][i] = __ldcg(reinterpret_cast<const double2*>(base + (long)s * N + row));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long row = r0 + u * wstep + 2 * sub;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc += v[u][i].x + v[u][i].y;
        const int s = i * SPI + sl;
        if (wr && s < wr && row < wend)
          *reinterpret_cast<double2*>(wbase + (long)s * N + row) = make_double2(v[u][i].x * 0.5, v[u][i].y);
      }
    }
  }
  if (acc == 12345.678) out[threadIdx.x] = acc;
}

template <int RUNB, int U>
void run(const double* d, double* o, double* w, long N, int S, int layout, int wr, int grid) {
  // S <= 8 * SPI streams per pass; more streams run as several passes over the range
  constexpr int SPI = 32 / (RUNB / 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto once = [&]() {
    for (int s0 = 0; s0 < S; s0 += 8 * SPI) {
      const int sn = S - s0 < 8 * SPI ? S - s0 : 8 * SPI;
      const int wn = wr - s0 > 0 ? (wr - s0 < sn ? wr - s0 : sn) : 0;
      kstream<RUNB, U><<<grid, 256>>>(d + (long)s0 * N, o, N, sn, layout, wn, w + (long)s0 * N);
    }
  };
  once();
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) once();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)N * 8 * (S + wr) * reps;
  printf("RUNB %3d U %d layout %d S %3d wr %3d: %7.1f GB/s\n", RUNB, U, layout, S, wr, bytes / (ms * 1e-3) / 1e9);
}


__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void ld256nc(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
// 32-byte lanes: RUNB / 32 lanes per stream (128: the DMMA fragment mapping, 4 lanes per shift)
template <int RUNB, int U, int CG>
__global__ void __launch_bounds__(256, 2) kstream32(const double* __restrict__ base, double* out, long N, int S,
                                                    int layout, int wr, double* wbase) {
  constexpr int LPS = RUNB / 32, SPI = 32 / LPS, ROWS = RUNB / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long rpc = ((N / gridDim.x) + 63) / 64 * 64;
  const long cbeg = (long)blockIdx.x * rpc, cend = min(N, cbeg + rpc);
  const long rpw = rpc / 8;
  const long wbeg = cbeg + warp * rpw, wend = min(cend, wbeg + rpw);
  const int sl = lane / LPS, sub = lane % LPS;
  double acc = 0.0;
  for (long r0 = wbeg; r0 < wend; r0 += U * ROWS) {
    double v[U][4][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long row = r0 + u * ROWS + 4 * sub;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int s = i * SPI + sl;
        v[u][i][0] = v[u][i][1] = v[u][i][2] = v[u][i][3] = 0.0;
        if (s < S && row < wend) {
          if (CG) ld256(base + (long)s * N + row, v[u][i][0], v[u][i][1], v[u][i][2], v[u][i][3]);
          else ld256nc(base + (long)s * N + row, v[u][i][0], v[u][i][1], v[u][i][2], v[u][i][3]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc += (v[u][i][0] + v[u][i][1]) + (v[u][i][2] + v[u][i][3]);
  }
  if (acc == 12345.678) out[threadIdx.x] = acc;
}
template <int RUNB, int U, int CG>
void run32(const double* d, double* o, long N, int S, int grid) {
  constexpr int SPI = 32 / (RUNB / 32);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto once = [&]() {
    for (int s0 = 0; s0 < S; s0 += 4 * SPI) {
      const int sn = S - s0 < 4 * SPI ? S - s0 : 4 * SPI;
      kstream32<RUNB, U, CG><<<grid, 256>>>(d + (long)s0 * N, o, N, sn, 0, 0, nullptr);
    }
  };
  once();
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) once();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("32B-lanes RUNB %3d U %d cg %d S %3d: %7.1f GB/s\n", RUNB, U, CG, S, (double)N * 8 * S * reps / (ms * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
  const long N = argc > 1 ? atol(argv[1]) : (1l << 20);
  const int S = argc > 2 ? atoi(argv[2]) : 48;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = 2 * nsm;
  double *d, *o, *w;
  cudaMalloc(&d, sizeof(double) * N * S);
  cudaMalloc(&w, sizeof(double) * N * S);
  cudaMalloc(&o, 4096);
  cudaMemset(d, 0, sizeof(double) * N * S);
  run32<128, 1, 1>(d, o, N, S, grid); run32<128, 2, 1>(d, o, N, S, grid); run32<128, 1, 0>(d, o, N, S, grid);
  run32<128, 2, 0>(d, o, N, S, grid); run32<256, 1, 1>(d, o, N, S, grid); run32<256, 2, 0>(d, o, N, S, grid);
  for (int wr : {0}) {
    for (int layout = 0; layout < 2; ++layout) {
      run<64, 1>(d, o, w, N, S, layout, wr, grid);
      run<64, 2>(d, o, w, N, S, layout, wr, grid);
      run<128, 1>(d, o, w, N, S, layout, wr, grid);
      run<128, 2>(d, o, w, N, S, layout, wr, grid);
      run<256, 1>(d, o, w, N, S, layout, wr, grid);
      run<256, 2>(d, o, w, N, S, layout, wr, grid);
      run<512, 1>(d, o, w, N, S, layout, wr, grid);
      run<512, 2>(d, o, w, N, S, layout, wr, grid);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
