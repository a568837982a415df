// The shifted operator for a rank-2 PSF (Example 1, §8.2: C = sum_{i=1,2}
// C_i^(1) (x) C_i^(2), i.e. h = u1 v1^T + u2 v2^T) as a composition of the rank-1 passes
// of the tiled core (apply_core.cuh, C and C^T modes: exact zero-boundary "same"
// convolutions with the term's separable taps) and its E-only form (zero taps):
//   C X = C1 X + C2 X,  A X = C^T (C X) = C1^T (C X) + C2^T (C X),
//   Y = A X + gamma E X  (SHIFTED),  Y = A X, EY = E X  (SPLIT).
// Not fused: the general-PSF path of include/rsk.h (rsk_create), used by the MINRES
// batch; the device CG loops embed the rank-1 fused apply. DESIGN.md §4.1c.
#include <cuda_runtime.h>

#include <algorithm>

#include "apply_core.cuh"

namespace rsk {

// dst_s += a * src_s (+ g_s e_s) for the listed vectors (s = list[li] or li)
__global__ void r2_combine(const int* __restrict__ list, int nl, int64_t N, double* __restrict__ dst, int64_t ldd,
                           const double* __restrict__ src, int64_t lds, const double* __restrict__ e, int64_t lde,
                           const double* __restrict__ gamma) {
  const int li = blockIdx.y;
  if (li >= nl) return;
  const int s = list ? list[li] : li;
  const double gm = (e && gamma) ? gamma[s] : 0.0;
  double* d = dst + (int64_t)s * ldd;
  const double* x = src + (int64_t)s * lds;
  const double* ev = e ? e + (int64_t)s * lde : nullptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    double v = d[i] + x[i];
    if (ev) v = fma(gm, ev[i], v);
    d[i] = v;
  }
}

// xdoty[s] = X_s . Y_s, one CTA per listed vector, fixed-order tree
__global__ void r2_dot(const int* __restrict__ list, int nl, int64_t N, const double* __restrict__ X, int64_t ldx,
                       const double* __restrict__ Y, int64_t ldy, double* __restrict__ out) {
  __shared__ double red[32];
  const int li = blockIdx.x;
  const int s = list ? list[li] : li;
  const double* x = X + (int64_t)s * ldx;
  const double* y = Y + (int64_t)s * ldy;
  double t = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) t = fma(x[i], y[i], t);
  t = block_sum(t, red);
  if (threadIdx.x == 0) out[s] = t;
}

cudaError_t launch_apply_rank2(Handle* h, const ApplyLaunch& a, cudaStream_t st) {
  if (a.cg) return cudaErrorNotSupported;
  if (a.nlist <= 0) return cudaSuccess;
  const int64_t N = h->ny * h->nx;
  const int64_t nv = (a.list || a.nvec_total > 0) ? std::max<int64_t>(a.nvec_total, a.nlist) : a.nlist;
  const size_t need = sizeof(double) * (size_t)N * (size_t)nv * 3;
  if (need > h->r2bytes) {
    if (h->r2buf) cudaFree(h->r2buf);
    h->r2buf = nullptr;
    h->r2bytes = 0;
    cudaError_t e = cudaMalloc(&h->r2buf, need);
    if (e != cudaSuccess) return e;
    h->r2bytes = need;
  }
  double* U = h->r2buf;              // C X
  double* V = U + (size_t)N * nv;    // the second term's pass
  double* Eb = V + (size_t)N * nv;   // E X
  const dim3 cg((unsigned)std::min<int64_t>((N + 255) / 256, 4 * h->sm_count), (unsigned)a.nlist);
  ApplyLaunch b = a;
  b.xdoty = nullptr;
  b.EY = nullptr;
  cudaError_t e;
  auto pass = [&](const double* X, int64_t ldx, double* Y, int64_t ldy, int mode, const double* cx,
                  const double* cy) -> cudaError_t {
    ApplyLaunch c = b;
    c.X = X; c.ldx = ldx; c.Y = Y; c.ldy = ldy; c.mode = mode;
    return launch_apply_taps(h, c, cx, cy, 0, st);
  };
  auto add = [&](double* dst, int64_t ldd, const double* src, const double* ev, const double* gam) -> cudaError_t {
    count_launch();
    r2_combine<<<cg, 256, 0, st>>>(a.list, a.nlist, N, dst, ldd, src, N, ev, N, gam);
    return cudaGetLastError();
  };
  if (a.mode == RSK_APPLY_C_ONLY || a.mode == RSK_APPLY_CT_ONLY) {
    const bool fw = a.mode == RSK_APPLY_C_ONLY;
    if ((e = pass(a.X, a.ldx, a.Y, a.ldy, a.mode, fw ? h->cCx : h->cTx, fw ? h->cCy : h->cTy)) != cudaSuccess) return e;
    if ((e = pass(a.X, a.ldx, V, N, a.mode, fw ? h->cCx2 : h->cTx2, fw ? h->cCy2 : h->cTy2)) != cudaSuccess) return e;
    if ((e = add(a.Y, a.ldy, V, nullptr, nullptr)) != cudaSuccess) return e;
  } else {
    // C X
    if ((e = pass(a.X, a.ldx, U, N, RSK_APPLY_C_ONLY, h->cCx, h->cCy)) != cudaSuccess) return e;
    if ((e = pass(a.X, a.ldx, V, N, RSK_APPLY_C_ONLY, h->cCx2, h->cCy2)) != cudaSuccess) return e;
    if ((e = add(U, N, V, nullptr, nullptr)) != cudaSuccess) return e;
    // C^T (C X)
    if ((e = pass(U, N, a.Y, a.ldy, RSK_APPLY_CT_ONLY, h->cTx, h->cTy)) != cudaSuccess) return e;
    if ((e = pass(U, N, V, N, RSK_APPLY_CT_ONLY, h->cTx2, h->cTy2)) != cudaSuccess) return e;
    // E X: the fused core in SPLIT mode with zero taps (its A part is 0)
    {
      ApplyLaunch c = b;
      c.mode = RSK_APPLY_SPLIT;
      c.Y = U; c.ldy = N;   // A part (zeros) into the spent C X buffer
      c.EY = (a.mode == RSK_APPLY_SPLIT) ? a.EY : Eb;
      c.ldey = (a.mode == RSK_APPLY_SPLIT) ? a.ldey : N;
      if ((e = launch_apply_taps(h, c, nullptr, nullptr, 0, st)) != cudaSuccess) return e;
    }
    if (a.mode == RSK_APPLY_SHIFTED) {
      if ((e = add(a.Y, a.ldy, V, Eb, a.gamma)) != cudaSuccess) return e;
    } else {
      if ((e = add(a.Y, a.ldy, V, nullptr, nullptr)) != cudaSuccess) return e;
    }
  }
  if (a.xdoty) {
    count_launch();
    r2_dot<<<a.nlist, 256, 0, st>>>(a.list, a.nlist, N, a.X, a.ldx, a.Y, a.ldy, a.xdoty);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace rsk
