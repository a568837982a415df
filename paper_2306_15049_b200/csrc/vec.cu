// Streaming kernels of librsk: tall-skinny recycle projections (U^T V, V +- U C),
// batched dots / axpby, the IRN weight update, L-curve norms, and the two CG
// vector kernels (update + dots, combine). All fp64, all reductions deterministic
// (fixed per-thread order, fixed shuffle tree, fixed-order sum of CTA partials).
#include <cstdlib>

#include <cuda_runtime.h>

#include "rsk_internal.h"

namespace rsk {

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ============================================================== projections
// U^T V partials: CTA (chunk, k-tile, nv-tile) computes a 32 x 32 block of
// U[rows of chunk]^T V[rows of chunk]; part[chunk][k][nv] (column-major k x nv).
__global__ void __launch_bounds__(256) gemm_tn_part(int64_t n, int k, const double* __restrict__ U,
                                                    int64_t ldu, int nv, const double* __restrict__ V,
                                                    int64_t ldv, double* __restrict__ part,
                                                    int64_t rows_per_chunk) {
  __shared__ double sU[32][33];
  __shared__ double sV[32][33];
  const int chunk = blockIdx.x;
  const int kt = blockIdx.y * 32, vt = blockIdx.z * 32;
  const int64_t rbeg = (int64_t)chunk * rows_per_chunk;
  const int64_t rend = min(n, rbeg + rows_per_chunk);
  const int tid = threadIdx.x;
  const int i0 = (tid >> 4) * 2, j0 = (tid & 15) * 2;
  double acc00 = 0, acc01 = 0, acc10 = 0, acc11 = 0;
  for (int64_t r0 = rbeg; r0 < rend; r0 += 32) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      const int row = idx & 31, col = idx >> 5;
      const int64_t gr = r0 + row;
      const bool rin = gr < rend;
      sU[col][row] = (rin && kt + col < k) ? __ldg(U + gr + (int64_t)(kt + col) * ldu) : 0.0;
      sV[col][row] = (rin && vt + col < nv) ? __ldg(V + gr + (int64_t)(vt + col) * ldv) : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const double u0 = sU[i0][rr], u1 = sU[i0 + 1][rr];
      const double v0 = sV[j0][rr], v1 = sV[j0 + 1][rr];
      acc00 = fma(u0, v0, acc00);
      acc01 = fma(u0, v1, acc01);
      acc10 = fma(u1, v0, acc10);
      acc11 = fma(u1, v1, acc11);
    }
    __syncthreads();
  }
  double* pc = part + (int64_t)chunk * k * nv;
  const int gi = kt + i0, gj = vt + j0;
  if (gi < k && gj < nv) pc[gi + (int64_t)gj * k] = acc00;
  if (gi < k && gj + 1 < nv) pc[gi + (int64_t)(gj + 1) * k] = acc01;
  if (gi + 1 < k && gj < nv) pc[gi + 1 + (int64_t)gj * k] = acc10;
  if (gi + 1 < k && gj + 1 < nv) pc[gi + 1 + (int64_t)(gj + 1) * k] = acc11;
}

// C = sum over the chunk partials: a warp per output element when there are many chunks
// (lanes stride the chunks, fixed shuffle tree), a thread per element otherwise
__global__ void gemm_tn_reduce(int k, int nv, int nchunk, const double* __restrict__ part,
                               double* __restrict__ C, int64_t ldc) {
  const int64_t tot = (int64_t)k * nv;
  if (nchunk >= 32) {
    const int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (idx >= tot) return;
    double t = 0.0;
    for (int c = lane; c < nchunk; c += 32) t += part[(int64_t)c * tot + idx];
    t = wsum(t);
    if (lane == 0) C[(idx % k) + (int64_t)(idx / k) * ldc] = t;
    return;
  }
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= tot) return;
  double t = 0.0;
  for (int c = 0; c < nchunk; ++c) t += part[(int64_t)c * tot + idx];
  const int i = (int)(idx % k), j = (int)(idx / k);
  C[i + (int64_t)j * ldc] = t;
}

static inline unsigned reduce_blocks(int64_t tot, int nchunk) {
  const int64_t threads = nchunk >= 32 ? tot * 32 : tot;
  return (unsigned)((threads + 255) / 256);
}

// U^T V partials on the FP64 tensor cores (mma.sync.m8n8k4.f64 -> DMMA): CTA (chunk,
// k-tile, nv-tile) computes a 32 x 32 block; warp w takes the 4-row groups w, w + 8, ... of
// the chunk and holds 4 x 4 accumulator fragments (A = U^T: a = U[row q][col g], B = V:
// b = V[row q][col g], D[g][2q..2q+1]); the 8 warp partials are summed in warp order
// through shared memory. Same part[chunk][k][nv] layout as gemm_tn_part.
__device__ __forceinline__ void dmma_tn(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) gemm_tn_part_tc(int64_t n, int k, const double* __restrict__ U, int64_t ldu,
                                                       int nv, const double* __restrict__ V, int64_t ldv,
                                                       double* __restrict__ part, int64_t rows_per_chunk) {
  extern __shared__ double red[];   // [8 warps][32][33]
  const int chunk = blockIdx.x;
  const int kt = blockIdx.y * 32, vt = blockIdx.z * 32;
  const int64_t rbeg = (int64_t)chunk * rows_per_chunk;
  const int64_t rend = min(n, rbeg + rows_per_chunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const double* up[4];
  const double* vp[4];
  bool uk[4], vk[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int cu = kt + 8 * i + g, cv = vt + 8 * i + g;
    uk[i] = cu < k;
    vk[i] = cv < nv;
    up[i] = U + (int64_t)(uk[i] ? cu : 0) * ldu;
    vp[i] = V + (int64_t)(vk[i] ? cv : 0) * ldv;
  }
#pragma unroll 2
  for (int64_t r0 = rbeg + 4 * warp; r0 < rend; r0 += 32) {
    const int64_t row = r0 + q;
    const bool vr = row < rend;
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[i] = (vr && uk[i]) ? __ldg(up[i] + row) : 0.0;
      b[i] = (vr && vk[i]) ? __ldg(vp[i] + row) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_tn(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double* rw = red + (size_t)warp * 32 * 33;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      rw[(8 * i + g) * 33 + 8 * j + 2 * q] = acc[i][j][0];
      rw[(8 * i + g) * 33 + 8 * j + 2 * q + 1] = acc[i][j][1];
    }
  __syncthreads();
  double* pc = part + (int64_t)chunk * k * nv;
  for (int e = threadIdx.x; e < 32 * 32; e += 256) {
    const int m = e >> 5, c = e & 31;
    const int gi = kt + m, gj = vt + c;
    if (gi >= k || gj >= nv) continue;
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[(size_t)w * 32 * 33 + m * 33 + c];
    pc[gi + (int64_t)gj * k] = t;
  }
}

// U^T V with a summation order per element that depends only on n, k and the SM count --
// not on nv: the row chunks are fixed by n, the tensor-core / scalar choice by k, and a V
// wider than the partial buffer runs as column blocks. So a column of V gives the same
// bits whatever other columns share the call (batch-composition invariance of the
// per-shift setup: 1-rank and N-rank shift-sharded runs do identical work).
cudaError_t launch_gemm_tn(Handle* h, int64_t n, int k, const double* U, int64_t ldu, int nv,
                           const double* V, int64_t ldv, double* C, int64_t ldc, cudaStream_t st) {
  const bool tc = k >= 16 && getenv("RSK_GEMM_NOTC") == nullptr;   // tensor-core path for the wide Grams
  int64_t nchunk = 2 * h->sm_count;
  const int64_t maxchunk = (n + 255) / 256;
  if (nchunk > maxchunk) nchunk = maxchunk;
  if (nchunk < 1) nchunk = 1;
  int64_t rpc = (n + nchunk - 1) / nchunk;
  rpc = (rpc + 31) / 32 * 32;
  nchunk = (n + rpc - 1) / rpc;
  // columns of V per launch: the partials [nchunk][k][nvb] must fit the scratch
  const size_t cap = h->scratch_bytes / (sizeof(double) * (size_t)k * (size_t)nchunk);
  if (cap < 1) return cudaErrorMemoryAllocation;
  const int nvb = (int)((size_t)nv < cap ? (size_t)nv : cap);
  const int tk = (k + 31) / 32;
  if (tc) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_tn_part_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(double) * 8 * 32 * 33));
      attr = true;
    }
  }
  for (int v0 = 0; v0 < nv; v0 += nvb) {
    const int nvc = nv - v0 < nvb ? nv - v0 : nvb;
    const int tv = (nvc + 31) / 32;
    dim3 grid((unsigned)nchunk, tk, tv);
    const double* Vb = V + (int64_t)v0 * ldv;
    if (tc) {
      count_launch();
      gemm_tn_part_tc<<<grid, 256, sizeof(double) * 8 * 32 * 33, st>>>(n, k, U, ldu, nvc, Vb, ldv, h->scratch, rpc);
    } else {
      count_launch(); gemm_tn_part<<<grid, 256, 0, st>>>(n, k, U, ldu, nvc, Vb, ldv, h->scratch, rpc);
    }
    const int64_t tot = (int64_t)k * nvc;
    count_launch();
    gemm_tn_reduce<<<reduce_blocks(tot, (int)nchunk), 256, 0, st>>>(k, nvc, (int)nchunk, h->scratch,
                                                                     C + (int64_t)v0 * ldc, ldc);
  }
  return cudaGetLastError();
}

// V (n x nv) += sign * U (n x k) C (k x nv). CTA: 64 rows x 32 cols of V.
__global__ void __launch_bounds__(256) gemm_nn_kernel(int64_t n, int k, const double* __restrict__ U,
                                                      int64_t ldu, int nv, double* __restrict__ V,
                                                      int64_t ldv, const double* __restrict__ C,
                                                      int64_t ldc, double sign) {
  __shared__ double sU[16][65];
  __shared__ double sC[16][33];
  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * 64;
  const int col0 = blockIdx.y * 32;
  const int r = tid & 63;
  const int jb = (tid >> 6) * 8;
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = 0.0;
  for (int k0 = 0; k0 < k; k0 += 16) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      const int rr = idx & 63, kk = idx >> 6;
      const int64_t gr = row0 + rr;
      sU[kk][rr] = (gr < n && k0 + kk < k) ? __ldg(U + gr + (int64_t)(k0 + kk) * ldu) : 0.0;
    }
    for (int idx = tid; idx < 16 * 32; idx += 256) {
      const int kk = idx & 15, cc = idx >> 4;
      sC[kk][cc] = (k0 + kk < k && col0 + cc < nv) ? __ldg(C + (k0 + kk) + (int64_t)(col0 + cc) * ldc) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const double u = sU[kk][r];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(u, sC[kk][jb + c], acc[c]);
    }
    __syncthreads();
  }
  const int64_t gr = row0 + r;
  if (gr >= n) return;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int gc = col0 + jb + c;
    if (gc < nv) {
      double* pv = V + gr + (int64_t)gc * ldv;
      *pv = fma(sign, acc[c], *pv);
    }
  }
}

cudaError_t launch_gemm_nn(Handle* h, int64_t n, int k, const double* U, int64_t ldu, int nv,
                           double* V, int64_t ldv, const double* C, int64_t ldc, double sign,
                           cudaStream_t st) {
  (void)h;
  dim3 grid((unsigned)((n + 63) / 64), (nv + 31) / 32);
  count_launch(); gemm_nn_kernel<<<grid, 256, 0, st>>>(n, k, U, ldu, nv, V, ldv, C, ldc, sign);
  return cudaGetLastError();
}

// ============================================================== batched BLAS-1
constexpr int kChunk = 2048;   // pixels per CTA for the streaming reductions

__global__ void reduce_partials(const double* __restrict__ part, int nchunk, double* out,
                                int do_sqrt) {
  const int s = blockIdx.x;
  double t = 0.0;
  for (int j = threadIdx.x; j < nchunk; j += 32) t += part[(int64_t)s * nchunk + j];
  t = wsum(t);
  if (threadIdx.x == 0) out[s] = do_sqrt ? sqrt(t) : t;
}

__device__ __forceinline__ void block_partial(double v, double* red, double* dst) {
  v = wsum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    t = wsum(t);
    if (lane == 0) *dst = t;
  }
}

__global__ void __launch_bounds__(256) dot_part(int64_t n, const double* __restrict__ X, int64_t ldx,
                                                const double* __restrict__ Y, int64_t ldy,
                                                double* __restrict__ part, int nchunk) {
  __shared__ double red[8];
  const int s = blockIdx.y;
  const double* x = X + (int64_t)s * ldx;
  const double* y = Y + (int64_t)s * ldy;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  double t = 0.0;
#pragma unroll
  for (int e = 0; e < kChunk / 256; ++e) {
    const int64_t i = base + e * 256 + threadIdx.x;
    if (i < n) t = fma(__ldg(x + i), __ldg(y + i), t);
  }
  block_partial(t, red, part + (int64_t)s * nchunk + blockIdx.x);
}

cudaError_t launch_batch_dot(Handle* h, int64_t n, int nv, const double* X, int64_t ldx,
                             const double* Y, int64_t ldy, double* out, cudaStream_t st) {
  const int nchunk = (int)((n + kChunk - 1) / kChunk);
  if (sizeof(double) * (size_t)nchunk * nv > h->scratch_bytes) return cudaErrorMemoryAllocation;
  count_launch(); dot_part<<<dim3(nchunk, nv), 256, 0, st>>>(n, X, ldx, Y, ldy, h->scratch, nchunk);
  count_launch(); reduce_partials<<<nv, 32, 0, st>>>(h->scratch, nchunk, out, 0);
  return cudaGetLastError();
}

__global__ void axpby_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ X,
                             int64_t ldx, const double* __restrict__ b, double* __restrict__ Y,
                             int64_t ldy) {
  const int s = blockIdx.y;
  const double as = a ? a[s] : 0.0;
  const double bs = b ? b[s] : 1.0;
  double* y = Y + (int64_t)s * ldy;
  const double* x = X ? X + (int64_t)s * ldx : nullptr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xv = x ? x[i] : 0.0;
    y[i] = fma(as, xv, bs * y[i]);
  }
}

cudaError_t launch_batch_axpby(int64_t n, int nv, const double* a, const double* X, int64_t ldx,
                               const double* b, double* Y, int64_t ldy, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  count_launch(); axpby_kernel<<<dim3((unsigned)blocks, nv), 256, 0, st>>>(n, a, X, ldx, b, Y, ldy);
  return cudaGetLastError();
}

// ============================================================== IRN weights
// wx = ((Dx x)^2 + tau^2)^(-1/2), wy likewise; eta2 partials under the handle weights.
__global__ void __launch_bounds__(256) irn_kernel(int ny, int nx, const double* __restrict__ x,
                                                  double tau, int iso, double* __restrict__ wx,
                                                  double* __restrict__ wy,
                                                  const double* __restrict__ hwx,
                                                  const double* __restrict__ hwy,
                                                  double* __restrict__ part) {
  __shared__ double red[8];
  const int64_t N = (int64_t)ny * nx;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  const double t2 = __dmul_rn(tau, tau);
  double acc = 0.0;
  for (int e = 0; e < kChunk / 256; ++e) {
    const int64_t p = base + e * 256 + threadIdx.x;
    if (p >= N) break;
    const int i = (int)(p / nx), j = (int)(p - (int64_t)i * nx);
    const double xc = x[p];
    double dx = 0.0, dy = 0.0;
    const bool hx = j < nx - 1, hy = i < ny - 1;
    if (hx) dx = x[p + 1] - xc;
    if (hy) dy = x[p + nx] - xc;
    if (wx && iso) {
      // isotropic (reading G32): one weight per pixel, a missing difference is 0;
      // unfused, in the order ((dx dx + dy dy) + tau tau)
      const double g2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), t2);
      const double w = 1.0 / sqrt(g2);
      wx[p] = hx ? w : 0.0;
      wy[p] = hy ? w : 0.0;
    } else if (wx) {
      wx[p] = hx ? 1.0 / sqrt(fma(dx, dx, t2)) : 0.0;
      wy[p] = hy ? 1.0 / sqrt(fma(dy, dy, t2)) : 0.0;
    }
    if (part) acc += hwx[p] * dx * dx + hwy[p] * dy * dy;
  }
  if (part) block_partial(acc, red, part + blockIdx.x);
}

cudaError_t launch_irn(Handle* h, const double* x, double tau, int iso, double* wx, double* wy,
                       double* eta2, cudaStream_t st) {
  const int64_t N = h->ny * h->nx;
  const int nchunk = (int)((N + kChunk - 1) / kChunk);
  count_launch(); irn_kernel<<<nchunk, 256, 0, st>>>((int)h->ny, (int)h->nx, x, tau, iso, wx, wy, h->wx,
                                                     h->wy, eta2 ? h->scratch : nullptr);
  if (eta2) { count_launch(); reduce_partials<<<1, 32, 0, st>>>(h->scratch, nchunk, eta2, 0); }
  return cudaGetLastError();
}

// ============================================================== Gazzola's weight update
// q = L x, w = |D_k q| / ||D_k q||_inf, w <- 1 - w^p, D_{k+1} = diag(w) D_k,
// W_{k+1} = D_{k+1}^2. Three launches: per-chunk max, final max, elementwise update.
// max is order-independent, so the whole update is deterministic; every other step is
// one correctly rounded operation in the oracle's order.
__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
  return t;
}

__global__ void __launch_bounds__(256) gz_max_part(int ny, int nx, const double* __restrict__ x,
                                                   const double* __restrict__ dx,
                                                   const double* __restrict__ dy,
                                                   double* __restrict__ part) {
  __shared__ double red[8];
  const int64_t N = (int64_t)ny * nx;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  double m = 0.0;
  for (int e = 0; e < kChunk / 256; ++e) {
    const int64_t p = base + e * 256 + threadIdx.x;
    if (p >= N) break;
    const int i = (int)(p / nx), j = (int)(p - (int64_t)i * nx);
    const double xc = x[p];
    if (j < nx - 1) m = fmax(m, fabs(__dmul_rn(dx[p], x[p + 1] - xc)));
    if (i < ny - 1) m = fmax(m, fabs(__dmul_rn(dy[p], x[p + nx] - xc)));
  }
  m = block_max(m, red);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

__global__ void __launch_bounds__(256) gz_max_final(const double* __restrict__ part, int nchunk,
                                                    double* __restrict__ out) {
  __shared__ double red[8];
  double m = 0.0;
  for (int j = threadIdx.x; j < nchunk; j += 256) m = fmax(m, part[j]);
  m = block_max(m, red);
  if (threadIdx.x == 0) *out = m;
}

__device__ __forceinline__ double gz_factor(double t, double m, double pw) {
  const double w = m > 0.0 ? t / m : 0.0;
  double wp;
  if (pw == 2.0) wp = __dmul_rn(w, w);
  else if (pw == 1.0) wp = w;
  else if (pw == 0.5) wp = sqrt(w);
  else wp = pow(w, pw);
  return 1.0 - wp;
}

__global__ void __launch_bounds__(256) gz_update(int ny, int nx, const double* __restrict__ x, double pw,
                                                 const double* __restrict__ mptr, double* __restrict__ dx,
                                                 double* __restrict__ dy, double* __restrict__ wx,
                                                 double* __restrict__ wy) {
  const int64_t N = (int64_t)ny * nx;
  const double m = *mptr;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(p / nx), j = (int)(p - (int64_t)i * nx);
    const double xc = x[p];
    double ndx = 0.0, ndy = 0.0;
    if (j < nx - 1) {
      const double d = dx[p];
      ndx = __dmul_rn(gz_factor(fabs(__dmul_rn(d, x[p + 1] - xc)), m, pw), d);
    }
    if (i < ny - 1) {
      const double d = dy[p];
      ndy = __dmul_rn(gz_factor(fabs(__dmul_rn(d, x[p + nx] - xc)), m, pw), d);
    }
    dx[p] = ndx;
    dy[p] = ndy;
    wx[p] = __dmul_rn(ndx, ndx);
    wy[p] = __dmul_rn(ndy, ndy);
  }
}

cudaError_t launch_gazzola_max(Handle* h, const double* x, const double* dx, const double* dy, double* m,
                               cudaStream_t st) {
  const int64_t N = h->ny * h->nx;
  const int nchunk = (int)((N + kChunk - 1) / kChunk);
  if (sizeof(double) * (size_t)nchunk > h->scratch_bytes) return cudaErrorMemoryAllocation;
  count_launch(); gz_max_part<<<nchunk, 256, 0, st>>>((int)h->ny, (int)h->nx, x, dx, dy, h->scratch);
  count_launch(); gz_max_final<<<1, 256, 0, st>>>(h->scratch, nchunk, m);
  return cudaGetLastError();
}

cudaError_t launch_gazzola_update(Handle* h, const double* x, double pw, const double* m, double* dx,
                                  double* dy, double* wx, double* wy, cudaStream_t st) {
  const int64_t N = h->ny * h->nx;
  int64_t blocks = (N + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  count_launch(); gz_update<<<(unsigned)blocks, 256, 0, st>>>((int)h->ny, (int)h->nx, x, pw, m, dx, dy, wx, wy);
  return cudaGetLastError();
}

// sum over rows [row0, row1) of the image of wx (Dx x)^2 + wy (Dy x)^2 (Dy of the last
// row of the range reads the next image row, when there is one)
__global__ void __launch_bounds__(256) seminorm_part(int ny, int nx, const double* __restrict__ X,
                                                     int64_t ldx, const double* __restrict__ hwx,
                                                     const double* __restrict__ hwy,
                                                     double* __restrict__ part, int nchunk, int row0,
                                                     int row1) {
  __shared__ double red[8];
  const int s = blockIdx.y;
  const double* x = X + (int64_t)s * ldx;
  const int64_t N = (int64_t)row1 * nx;
  const int64_t base = (int64_t)row0 * nx + (int64_t)blockIdx.x * kChunk;
  double acc = 0.0;
  for (int e = 0; e < kChunk / 256; ++e) {
    const int64_t p = base + e * 256 + threadIdx.x;
    if (p >= N) break;
    const int i = (int)(p / nx), j = (int)(p - (int64_t)i * nx);
    const double xc = x[p];
    const double dx = j < nx - 1 ? x[p + 1] - xc : 0.0;
    const double dy = i < ny - 1 ? x[p + nx] - xc : 0.0;
    acc += hwx[p] * dx * dx + hwy[p] * dy * dy;
  }
  block_partial(acc, red, part + (int64_t)s * nchunk + blockIdx.x);
}

cudaError_t launch_seminorm_batch(Handle* h, int nvec, const double* X, int64_t ldx, double* eta2,
                                  cudaStream_t st, int do_sqrt) {
  const int64_t N = h->ny * h->nx;
  const int nchunk = (int)((N + kChunk - 1) / kChunk);
  if (sizeof(double) * (size_t)nchunk * nvec > h->scratch_bytes) return cudaErrorMemoryAllocation;
  count_launch(); seminorm_part<<<dim3(nchunk, nvec), 256, 0, st>>>((int)h->ny, (int)h->nx, X, ldx, h->wx, h->wy,
                                                    h->scratch, nchunk, 0, (int)h->ny);
  count_launch(); reduce_partials<<<nvec, 32, 0, st>>>(h->scratch, nchunk, eta2, do_sqrt);
  return cudaGetLastError();
}

cudaError_t launch_seminorm_rows(Handle* h, int nvec, const double* X, int64_t ldx, int row0, int row1,
                                 double* eta2, cudaStream_t st) {
  const int64_t n = (int64_t)(row1 - row0) * h->nx;
  const int nchunk = (int)((n + kChunk - 1) / kChunk);
  if (nchunk < 1) return cudaErrorInvalidValue;
  if (sizeof(double) * (size_t)nchunk * nvec > h->scratch_bytes) return cudaErrorMemoryAllocation;
  count_launch(); seminorm_part<<<dim3(nchunk, nvec), 256, 0, st>>>((int)h->ny, (int)h->nx, X, ldx, h->wx, h->wy,
                                                    h->scratch, nchunk, row0, row1);
  count_launch(); reduce_partials<<<nvec, 32, 0, st>>>(h->scratch, nchunk, eta2, 0);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) diffnorm_part(int64_t n, const double* __restrict__ Y,
                                                     int64_t ldy, const double* __restrict__ d,
                                                     double* __restrict__ part, int nchunk) {
  __shared__ double red[8];
  const int s = blockIdx.y;
  const double* y = Y + (int64_t)s * ldy;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  double acc = 0.0;
  for (int e = 0; e < kChunk / 256; ++e) {
    const int64_t i = base + e * 256 + threadIdx.x;
    if (i < n) {
      const double t = y[i] - d[i];
      acc = fma(t, t, acc);
    }
  }
  block_partial(acc, red, part + (int64_t)s * nchunk + blockIdx.x);
}

cudaError_t launch_diffnorm_batch(Handle* h, int nvec, const double* Y, int64_t ldy, const double* d,
                                  double* out, cudaStream_t st) {
  const int64_t N = h->ndata;   // data vectors (= ny * nx for the blur)
  const int nchunk = (int)((N + kChunk - 1) / kChunk);
  if (sizeof(double) * (size_t)nchunk * nvec > h->scratch_bytes) return cudaErrorMemoryAllocation;
  count_launch(); diffnorm_part<<<dim3(nchunk, nvec), 256, 0, st>>>(N, Y, ldy, d, h->scratch, nchunk);
  count_launch(); reduce_partials<<<nvec, 32, 0, st>>>(h->scratch, nchunk, out, 1);
  return cudaGetLastError();
}

// d = cx + nu * sqrt(s2[0]) / sqrt(s2[1]) * xi  (s2 = {||cx||^2, ||xi||^2} on device)
__global__ void scale_noise_kernel(int64_t n, const double* __restrict__ cx,
                                   const double* __restrict__ xi, const double* __restrict__ s2,
                                   double nu, double* __restrict__ d) {
  const double sc = nu * sqrt(s2[0]) / sqrt(s2[1]);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = fma(sc, xi[i], cx[i]);
}

cudaError_t launch_scale_noise(int64_t n, const double* cx, const double* xi, const double* s2,
                               double nu, double* d, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  count_launch(); scale_noise_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, cx, xi, s2, nu, d);
  return cudaGetLastError();
}

// ============================================================== CG vector kernels
constexpr int kCgPPT = 8;                 // pixels per thread
constexpr int kCgChunk = kCgPPT * kNT;    // 2048 pixels per CTA

int cg_nblkB(int64_t N) { return (int)((N + kCgChunk - 1) / kCgChunk); }

// Solve L L^T x = z in place (L lower, column-major m x m, m <= kMaxM).
__device__ void dev_chol_solve(int m, const double* L, double* x) {
  for (int i = 0; i < m; ++i) {
    double t = x[i];
    for (int j = 0; j < i; ++j) t -= L[i + j * kMaxM] * x[j];
    x[i] = t / L[i + i * kMaxM];
  }
  for (int i = m - 1; i >= 0; --i) {
    double t = x[i];
    for (int j = i + 1; j < m; ++j) t -= L[j + i * kMaxM] * x[j];
    x[i] = t / L[i + i * kMaxM];
  }
}

// KB: r -= alpha w (LOOP), then rho' = r.r and z = Z^T r (or U^T r for GALERKIN);
// last CTA of the shift reduces the partials in fixed order and forms the scalars.
__global__ void __launch_bounds__(kNT) cg_update_kernel(CgDev* __restrict__ cg, const int* list,
                                                        int mode) {
  __shared__ double red[8][kMaxM + 1];
  __shared__ double tot[kMaxM + 1];
  __shared__ int s_last;
  const int s = list[blockIdx.y];
  const int st0 = cg->status[s];
  if (mode == UPD_LOOP) {
    if (st0 != ST_ACTIVE) return;
  } else if (st0 == ST_IDLE || st0 == ST_BREAKDOWN || st0 == ST_MAXIT || st0 == ST_DONE) {
    return;
  }
  const int64_t N = cg->N;
  const int m = cg->mloc[s];
  const int hasg = cg->hasg[s];
  const int nw = m - hasg;          // W columns in use
  const int g = cg->group[s];
  const double gam = cg->gam[s];
  const double alpha = (mode == UPD_LOOP) ? cg->alpha[s] : 0.0;
  double* __restrict__ r = cg->R + (int64_t)s * N;
  const double* __restrict__ w = cg->Wv + (int64_t)s * N;
  const double* __restrict__ W = cg->grp.W[g];
  const double* __restrict__ AW = cg->grp.AW[g];
  const double* __restrict__ EW = cg->grp.EW[g];
  const int64_t ldw = cg->grp.ldw;
  const double* __restrict__ gh = hasg ? cg->Ghat + (int64_t)s * cg->ldgh : nullptr;
  const double* __restrict__ zg = hasg ? cg->ZGhat + (int64_t)s * cg->ldgh : nullptr;
  const bool galerkin = (mode == UPD_GALERKIN);

  double acc[kMaxM + 1];
#pragma unroll
  for (int j = 0; j <= kMaxM; ++j) acc[j] = 0.0;
  const int64_t base = (int64_t)blockIdx.x * kCgChunk;
#pragma unroll 2
  for (int e = 0; e < kCgPPT; ++e) {
    const int64_t i = base + e * kNT + threadIdx.x;
    if (i >= N) break;
    double rv = r[i];
    if (mode == UPD_LOOP) {
      rv = fma(-alpha, w[i], rv);
      r[i] = rv;
    }
    acc[0] = fma(rv, rv, acc[0]);
#pragma unroll
    for (int j = 0; j < kMaxM; ++j) {
      if (j < nw) {
        const double col = galerkin ? __ldg(W + i + (int64_t)j * ldw)
                                    : fma(gam, __ldg(EW + i + (int64_t)j * ldw), __ldg(AW + i + (int64_t)j * ldw));
        acc[1 + j] = fma(col, rv, acc[1 + j]);
      } else if (j == nw && hasg) {
        const double col = galerkin ? __ldg(gh + i) : __ldg(zg + i);
        acc[1 + j] = fma(col, rv, acc[1 + j]);
      }
    }
  }
  // block reduction of the m+1 values (fixed tree)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j <= kMaxM; ++j) {
    if (j <= m) {
      const double v = wsum(acc[j]);
      if (lane == 0) red[wid][j] = v;
    }
  }
  __syncthreads();
  const int nblk = gridDim.x;
  double* pb = cg->partB + ((int64_t)s * cg->nblkB + blockIdx.x) * (kMaxM + 1);
  if (threadIdx.x <= m) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kNT / 32; ++q) t += red[q][threadIdx.x];
    pb[threadIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned tk = atomicAdd(cg->cnt + 4 * s + 1, 1u);
    s_last = (tk == (unsigned)(nblk - 1));
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x <= m) {
    const double* p0 = cg->partB + (int64_t)s * cg->nblkB * (kMaxM + 1);
    double t = 0.0;
    for (int bq = 0; bq < nblk; ++bq) t += __ldcg(p0 + (int64_t)bq * (kMaxM + 1) + threadIdx.x);
    tot[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  cg->cnt[4 * s + 1] = 0u;
  double z[kMaxM];
  for (int j = 0; j < m; ++j) z[j] = tot[1 + j];
  if (m > 0) dev_chol_solve(m, cg->Lf + (int64_t)s * kMaxM * kMaxM, z);
  double* cf = cg->coef + (int64_t)s * kMaxM;
  for (int j = 0; j < kMaxM; ++j) cf[j] = j < m ? z[j] : 0.0;
  if (galerkin) return;
  const double rho_new = tot[0];
  const double thr = cg->tol * cg->bnorm;
  const bool conv = sqrt(rho_new) <= thr;
  if (mode == UPD_LOOP) {
    const int it = cg->iters[s] + 1;
    cg->iters[s] = it;
    cg->beta[s] = rho_new / cg->rho[s];
    cg->rho[s] = rho_new;
    if (conv) cg->status[s] = ST_RCONV;
    else if (it >= cg->maxit) cg->status[s] = ST_MAXIT;
  } else {
    cg->beta[s] = 0.0;
    cg->alpha[s] = 0.0;
    cg->rho[s] = rho_new;
    if (mode == UPD_CONFIRM) {
      cg->rho_true[s] = rho_new;
      cg->status[s] = conv ? ST_DONE : (cg->iters[s] >= cg->maxit ? ST_MAXIT : ST_ACTIVE);
    } else {
      cg->status[s] = conv ? ST_RCONV : ST_ACTIVE;
    }
  }
}

cudaError_t launch_cg_update(CgDev* dev, const CgDev& host, const int* list, int nlist, int mode,
                             cudaStream_t st) {
  if (nlist <= 0) return cudaSuccess;
  dim3 grid(host.nblkB, nlist);
  count_launch(); cg_update_kernel<<<grid, kNT, 0, st>>>(dev, list, mode);
  return cudaGetLastError();
}

// KC: LOOP: x += alpha p; p = r + beta p - U mu; store r/||r||.
//     GALERKIN: x += U c; r -= Z c.    RESID: r = b - w.
__global__ void __launch_bounds__(kNT) cg_combine_kernel(CgDev* __restrict__ cg, const int* list,
                                                         int mode) {
  __shared__ int s_last;
  const int s = list[blockIdx.y];
  const int st0 = cg->status[s];
  const int64_t N = cg->N;
  double* __restrict__ x = cg->X + (int64_t)s * cg->ldx;
  double* __restrict__ r = cg->R + (int64_t)s * N;
  const int64_t base = (int64_t)blockIdx.x * kCgChunk;
  if (mode == CMB_RESID) {
    if (st0 == ST_IDLE) return;
    const double* __restrict__ w = cg->Wv + (int64_t)s * N;
    for (int e = 0; e < kCgPPT; ++e) {
      const int64_t i = base + e * kNT + threadIdx.x;
      if (i >= N) break;
      r[i] = __ldg(cg->b + i) - w[i];
    }
    return;
  }
  const int m = cg->mloc[s];
  const int hasg = cg->hasg[s];
  const int nw = m - hasg;
  const int g = cg->group[s];
  const double gam = cg->gam[s];
  const double* __restrict__ W = cg->grp.W[g];
  const double* __restrict__ AW = cg->grp.AW[g];
  const double* __restrict__ EW = cg->grp.EW[g];
  const int64_t ldw = cg->grp.ldw;
  const double* __restrict__ gh = hasg ? cg->Ghat + (int64_t)s * cg->ldgh : nullptr;
  const double* __restrict__ zg = hasg ? cg->ZGhat + (int64_t)s * cg->ldgh : nullptr;
  double cf[kMaxM];
#pragma unroll
  for (int j = 0; j < kMaxM; ++j) cf[j] = cg->coef[(int64_t)s * kMaxM + j];

  if (mode == CMB_GALERKIN) {
    if (m == 0 || st0 == ST_IDLE) return;
    for (int e = 0; e < kCgPPT; ++e) {
      const int64_t i = base + e * kNT + threadIdx.x;
      if (i >= N) break;
      double xv = x[i], rv = r[i];
#pragma unroll
      for (int j = 0; j < kMaxM; ++j) {
        if (j < nw) {
          xv = fma(cf[j], __ldg(W + i + (int64_t)j * ldw), xv);
          const double zc = fma(gam, __ldg(EW + i + (int64_t)j * ldw), __ldg(AW + i + (int64_t)j * ldw));
          rv = fma(-cf[j], zc, rv);
        } else if (j == nw && hasg) {
          xv = fma(cf[j], __ldg(gh + i), xv);
          rv = fma(-cf[j], __ldg(zg + i), rv);
        }
      }
      x[i] = xv;
      r[i] = rv;
    }
    return;
  }
  // CMB_LOOP
  const double alpha = cg->alpha[s];
  if (st0 == ST_RCONV || st0 == ST_MAXIT) {
    if (alpha == 0.0) return;       // the final x update has been applied already
  } else if (st0 != ST_ACTIVE) {
    return;
  }
  const bool upd_p = (st0 == ST_ACTIVE);
  const double beta = cg->beta[s];
  double* __restrict__ p = cg->P + (int64_t)s * N;
  const bool do_store = upd_p && cg->store && cg->store_cnt[s] < cg->store_cap;
  double* __restrict__ sto = do_store
      ? cg->store + ((int64_t)s * cg->store_cap + cg->store_cnt[s]) * cg->lds : nullptr;
  const double rinv = do_store ? 1.0 / sqrt(cg->rho[s]) : 0.0;
  for (int e = 0; e < kCgPPT; ++e) {
    const int64_t i = base + e * kNT + threadIdx.x;
    if (i >= N) break;
    const double pv = p[i];
    x[i] = fma(alpha, pv, x[i]);
    if (upd_p) {
      const double rv = r[i];
      double pn = fma(beta, pv, rv);
#pragma unroll
      for (int j = 0; j < kMaxM; ++j) {
        if (j < nw) pn = fma(-cf[j], __ldg(W + i + (int64_t)j * ldw), pn);
        else if (j == nw && hasg) pn = fma(-cf[j], __ldg(gh + i), pn);
      }
      p[i] = pn;
      if (do_store) sto[i] = rv * rinv;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned tk = atomicAdd(cg->cnt + 4 * s + 2, 1u);
    s_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    cg->cnt[4 * s + 2] = 0u;
    cg->alpha[s] = 0.0;
    if (do_store) cg->store_cnt[s] += 1;
  }
}

cudaError_t launch_cg_combine(CgDev* dev, const CgDev& host, const int* list, int nlist, int mode,
                              cudaStream_t st) {
  if (nlist <= 0) return cudaSuccess;
  dim3 grid(host.nblkB, nlist);
  count_launch(); cg_combine_kernel<<<grid, kNT, 0, st>>>(dev, list, mode);
  return cudaGetLastError();
}

}  // namespace rsk
