// Parallel-beam CT operator of Example 2 (reading
// G38): C is the line-integral matrix -- entry (ray, pixel) = length of the ray inside the
// pixel square -- for angles given in degrees and unit-width detector bins centred on the
// rotation axis, scaled to unit Frobenius norm. See include/rsk.h
// (rsk_create_ct) for the geometry and the contract.
//
// C is not a stencil, so the fused Toeplitz apply does not apply: the library builds C
// once on the host (Siddon-style traversal: the ray's crossings of the grid lines, sorted,
// each segment attributed to the pixel holding its midpoint) as CSR over rays plus its
// transpose (CSR over pixels), and the shifted apply is two deterministic kernels:
//   ct_fwd   t = C x           one warp per ray, lane-strided row, fixed shuffle tree
//   ct_adj   y = C^T t + gamma E_k x (or the SPLIT / C^T-only forms), one thread per pixel,
//            its transpose row in ray order, the weighted 5-point E stencil fused, and the
//            x . y partial per CTA (fixed-order reduction by apply_dot_reduce's rule)
// Both serve up to 8 vectors of a batch per pass over the matrix entries (the CSR pair is
// read once per 8 shifts, not once per shift); each vector's sums keep the one-vector
// order, so results do not depend on the batch.
// Every librsk call that goes through launch_apply (rsk_apply_shifted, the recycling
// MINRES batch, the L-curve norms, make_rhs) works on a CT handle; the CG device loops
// embed the stencil apply and reject it.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include <cuda_runtime.h>

#include "rsk_internal.h"

using namespace rsk;

struct rsk_handle_s : public Handle {};   // as in rsk.cu

namespace rsk {
namespace {

constexpr int kCtT = 256;

constexpr int kVB = 8;   // vectors per CTA: one pass over a matrix row serves all of them

// t[li][ray] = sum_k val[k] x[li][col[k]] for the kVB vectors li0 + b of this CTA (warp per
// ray; each vector's sum in the same lane-strided order and shuffle tree as for one vector)
__global__ void __launch_bounds__(kCtT) ct_fwd(int64_t m, const int64_t* __restrict__ rp, const int* __restrict__ col,
                                               const double* __restrict__ val, const double* __restrict__ X,
                                               int64_t ldx, const int* __restrict__ list, int nl,
                                               double* __restrict__ T, int64_t ldt) {
  const int li0 = blockIdx.y * kVB;
  const int nvb = min(kVB, nl - li0);
  const double* x[kVB];
#pragma unroll
  for (int b = 0; b < kVB; ++b) {
    const int li = li0 + (b < nvb ? b : 0);
    x[b] = X + (int64_t)(list ? list[li] : li) * ldx;
  }
  const int lane = threadIdx.x & 31;
  const int64_t ray = (int64_t)blockIdx.x * (kCtT / 32) + (threadIdx.x >> 5);
  if (ray >= m) return;
  double acc[kVB];
#pragma unroll
  for (int b = 0; b < kVB; ++b) acc[b] = 0.0;
  for (int64_t k = rp[ray] + lane; k < rp[ray + 1]; k += 32) {
    const double v = val[k];
    const int c = col[k];
#pragma unroll
    for (int b = 0; b < kVB; ++b)
      if (b < nvb) acc[b] = fma(v, __ldg(x[b] + c), acc[b]);
  }
#pragma unroll
  for (int b = 0; b < kVB; ++b) {
    if (b >= nvb) break;
    double t = acc[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) T[(int64_t)(li0 + b) * ldt + ray] = t;
  }
}

// y = C^T t (+ gamma E x | EY = E x), x . y partials (mode as RSK_APPLY_*): warp per pixel
// (lane-strided transpose row, fixed shuffle tree), kVB vectors per pass over the row; lane b
// finishes vector b (E stencil, gamma combine, store)
__global__ void __launch_bounds__(kCtT) ct_adj(int n, const int64_t* __restrict__ rp, const int* __restrict__ col,
                                               const double* __restrict__ val, const double* __restrict__ T,
                                               int64_t ldt, const int* __restrict__ list, int nl, int t_by_sid,
                                               const double* __restrict__ X, int64_t ldx, double* __restrict__ Y,
                                               int64_t ldy, double* __restrict__ EY, int64_t ldey,
                                               const double* __restrict__ gamma, const double* __restrict__ wx,
                                               const double* __restrict__ wy, int mode, double* __restrict__ part) {
  const int li0 = blockIdx.y * kVB;
  const int nvb = min(kVB, nl - li0);
  const int64_t N = (int64_t)n * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t p = (int64_t)blockIdx.x * (kCtT / 32) + warp;
  const double* t[kVB];
#pragma unroll
  for (int b = 0; b < kVB; ++b) {
    const int li = li0 + (b < nvb ? b : 0);
    t[b] = T + (int64_t)(t_by_sid ? (list ? list[li] : li) : li) * ldt;
  }
  double a[kVB];
#pragma unroll
  for (int b = 0; b < kVB; ++b) a[b] = 0.0;
  if (p < N) {
    for (int64_t k = rp[p] + lane; k < rp[p + 1]; k += 32) {
      const double v = val[k];
      const int c = col[k];
#pragma unroll
      for (int b = 0; b < kVB; ++b)
        if (b < nvb) a[b] = fma(v, t[b][c], a[b]);
    }
  }
  double mine = 0.0;   // lane b keeps vector b's row sum
#pragma unroll
  for (int b = 0; b < kVB; ++b) {
    double v = a[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == b) mine = v;
  }
  const bool withE = (mode == RSK_APPLY_SHIFTED || mode == RSK_APPLY_SPLIT);
  double dotv = 0.0;
  if (p < N && lane < nvb) {
    const int li = li0 + lane;
    const int s = list ? list[li] : li;
    double yv = mine;
    if (withE) {
      const double* x = X + (int64_t)s * ldx;
      const int i = (int)(p / n), j = (int)(p - (int64_t)i * n);
      const double xc = x[p];
      double e = 0.0;   // E x = Dx^T (wx Dx x) + Dy^T (wy Dy x), pads of w are 0
      if (j + 1 < n) e -= wx[p] * (x[p + 1] - xc);
      if (j > 0) e += wx[p - 1] * (xc - x[p - 1]);
      if (i + 1 < n) e -= wy[p] * (x[p + n] - xc);
      if (i > 0) e += wy[p - n] * (xc - x[p - n]);
      if (mode == RSK_APPLY_SHIFTED) yv = fma(gamma[s], e, yv);
      else EY[(int64_t)s * ldey + p] = e;
      dotv = xc * yv;
    }
    Y[(int64_t)s * ldy + p] = yv;
  }
  if (part) {   // x . y partial of this CTA per vector: its 8 pixels (warps) in order
    __shared__ double red[kCtT / 32][kVB];
    if (lane < kVB) red[warp][lane] = dotv;
    __syncthreads();
    if (threadIdx.x < nvb) {
      double tot = 0.0;
      for (int w = 0; w < kCtT / 32; ++w) tot += red[w][threadIdx.x];
      part[(int64_t)(li0 + threadIdx.x) * gridDim.x + blockIdx.x] = tot;
    }
  }
}

__global__ void ct_dot_reduce(const double* __restrict__ part, int nblk, const int* __restrict__ list,
                              double* __restrict__ out) {
  const int li = blockIdx.x;
  double t = 0.0;
  for (int j = threadIdx.x; j < nblk; j += 32) t += part[(int64_t)li * nblk + j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) out[list ? list[li] : li] = t;
}

// Siddon-style traversal of ray (theta, s) through the n x n grid (pixel (i, j) is
// x in [j - n/2, j + 1 - n/2], y in [n/2 - i - 1, n/2 - i]): segment lengths per pixel.
void trace_ray(int n, double theta, double s, std::vector<std::pair<int, double>>& out) {
  out.clear();
  const double c = std::cos(theta), sn = std::sin(theta);
  const double px = s * c, py = s * sn, ux = -sn, uy = c;
  const double h = 0.5 * n;
  const double eps = 1e-15;
  double tlo = -1e300, thi = 1e300;
  // clip against the image box
  if (std::fabs(ux) < eps) {
    if (!(px >= -h && px < h)) return;
  } else {
    const double ta = (-h - px) / ux, tb = (h - px) / ux;
    tlo = std::max(tlo, std::min(ta, tb));
    thi = std::min(thi, std::max(ta, tb));
  }
  if (std::fabs(uy) < eps) {
    if (!(py >= -h && py < h)) return;
  } else {
    const double ta = (-h - py) / uy, tb = (h - py) / uy;
    tlo = std::max(tlo, std::min(ta, tb));
    thi = std::min(thi, std::max(ta, tb));
  }
  if (!(thi > tlo)) return;
  std::vector<double> ts;
  ts.reserve(2 * n + 4);
  ts.push_back(tlo);
  ts.push_back(thi);
  if (std::fabs(ux) >= eps)
    for (int k = 0; k <= n; ++k) {
      const double t = (k - h - px) / ux;
      if (t > tlo && t < thi) ts.push_back(t);
    }
  if (std::fabs(uy) >= eps)
    for (int k = 0; k <= n; ++k) {
      const double t = (k - h - py) / uy;
      if (t > tlo && t < thi) ts.push_back(t);
    }
  std::sort(ts.begin(), ts.end());
  for (size_t q = 0; q + 1 < ts.size(); ++q) {
    const double len = ts[q + 1] - ts[q];
    if (len <= 1e-13) continue;
    const double tm = 0.5 * (ts[q] + ts[q + 1]);
    const double xm = px + tm * ux, ym = py + tm * uy;
    // half-open pixel faces [low, high): a ray on a face belongs to the high-side pixel
    const int j = (int)std::floor(xm + h);
    const int i = (int)std::ceil(h - ym) - 1;
    if (i < 0 || i >= n || j < 0 || j >= n) continue;
    if (!out.empty() && out.back().first == i * n + j) out.back().second += len;
    else out.emplace_back(i * n + j, len);
  }
}

}  // namespace

cudaError_t launch_ct_apply(Handle* h, const ApplyLaunch& a, cudaStream_t st) {
  if (a.cg) return cudaErrorNotSupported;
  if (a.nlist <= 0) return cudaSuccess;
  if (a.mode == RSK_APPLY_C_ONLY && a.list) return cudaErrorNotSupported;
  const int n = (int)h->nx;
  const int64_t N = (int64_t)n * n, m = h->ndata;
  const int mode = a.mode;
  const int nb = (int)((N + kCtT / 32 - 1) / (kCtT / 32));   // ct_adj: a warp per pixel
  for (int l0 = 0; l0 < a.nlist; l0 += h->ct_tmp_vecs) {
    const int nl = std::min(h->ct_tmp_vecs, a.nlist - l0);
    const int* lst = a.list ? a.list + l0 : nullptr;
    // for list == nullptr the batch is X + l0 .. (the kernels index by position then)
    const double* X = a.list ? a.X : a.X + (int64_t)l0 * a.ldx;
    double* Y = a.list ? a.Y : a.Y + (int64_t)l0 * a.ldy;
    double* EY = (a.EY && !a.list) ? a.EY + (int64_t)l0 * a.ldey : a.EY;
    const double* gam = (a.gamma && !a.list) ? a.gamma + l0 : a.gamma;
    double* xd = (a.xdoty && !a.list) ? a.xdoty + l0 : a.xdoty;
    if (mode == RSK_APPLY_C_ONLY) {   // (C_ONLY writes by position: no list, checked above)
      count_launch();
      ct_fwd<<<dim3((unsigned)((m + 7) / 8), (nl + kVB - 1) / kVB), kCtT, 0, st>>>(m, h->ct_rp, h->ct_col, h->ct_val, X,
                                                                                  a.ldx, lst, nl, Y, a.ldy);
      continue;
    }
    const double* T = X;
    int64_t ldt = a.ldx;
    int t_by_sid = 1;
    if (mode != RSK_APPLY_CT_ONLY) {
      count_launch();
      ct_fwd<<<dim3((unsigned)((m + 7) / 8), (nl + kVB - 1) / kVB), kCtT, 0, st>>>(m, h->ct_rp, h->ct_col, h->ct_val, X,
                                                                                  a.ldx, lst, nl, h->ct_tmp, m);
      T = h->ct_tmp;
      ldt = m;
      t_by_sid = 0;
    }
    double* part = nullptr;
    if (xd) {
      if (sizeof(double) * (size_t)nb * nl > h->scratch_bytes) return cudaErrorMemoryAllocation;
      part = h->scratch;
    }
    count_launch();
    ct_adj<<<dim3((unsigned)nb, (nl + kVB - 1) / kVB), kCtT, 0, st>>>(n, h->ctT_rp, h->ctT_col, h->ctT_val, T, ldt, lst,
                                                                      nl, t_by_sid, X, a.ldx, Y, a.ldy, EY, a.ldey, gam,
                                                                      h->wx, h->wy, mode, part);
    if (xd) {
      count_launch();
      ct_dot_reduce<<<nl, 32, 0, st>>>(part, nb, lst, xd);
    }
  }
  return cudaGetLastError();
}

}  // namespace rsk

extern "C" rsk_status rsk_create_ct(rsk_handle* out, int device, int64_t n, int nangles, const double* angles_deg_h,
                                    int ndet, int flags) {
  (void)flags;
  if (!out || !angles_deg_h || n < 2 || n > 4096 || nangles < 1 || ndet < 1) return RSK_EINVAL;
  for (int a = 0; a < nangles; ++a)
    if (!std::isfinite(angles_deg_h[a])) return RSK_EINVAL;
  const int64_t N = n * n, m = (int64_t)nangles * ndet;
  // every ray crosses at most 2n pixels: keep the stored entries addressable and the host
  // build bounded (the explicit matrix is meant for Example 2's sizes, n = 82)
  if ((double)m * 2.0 * (double)n > 1.0e9) return RSK_ENOMEM;
  // ---- C on the host: CSR over rays (angle-major, detector-minor)
  std::vector<int64_t> rp((size_t)m + 1, 0);
  std::vector<int> col;
  std::vector<double> val;
  std::vector<std::pair<int, double>> seg;
  const double pi = 3.14159265358979323846;
  for (int a = 0; a < nangles; ++a) {
    const double th = angles_deg_h[a] * pi / 180.0;
    for (int d = 0; d < ndet; ++d) {
      const double s = d - 0.5 * (ndet - 1);
      trace_ray((int)n, th, s, seg);
      for (auto& e : seg) { col.push_back(e.first); val.push_back(e.second); }
      rp[(size_t)a * ndet + d + 1] = (int64_t)col.size();
    }
  }
  const int64_t nnz = (int64_t)col.size();
  if (nnz == 0) return RSK_EINVAL;
  double fro = 0.0;
  for (double v : val) fro += v * v;
  fro = std::sqrt(fro);
  for (double& v : val) v /= fro;                 // unit Frobenius norm
  // ---- C^T: CSR over pixels, entries in ray order
  std::vector<int64_t> rpT((size_t)N + 1, 0);
  for (int c : col) rpT[(size_t)c + 1] += 1;
  for (int64_t p = 0; p < N; ++p) rpT[(size_t)p + 1] += rpT[(size_t)p];
  std::vector<int> colT((size_t)nnz);
  std::vector<double> valT((size_t)nnz);
  {
    std::vector<int64_t> fill(rpT.begin(), rpT.end() - 1);
    for (int64_t r = 0; r < m; ++r)
      for (int64_t k = rp[(size_t)r]; k < rp[(size_t)r + 1]; ++k) {
        const int64_t at = fill[(size_t)col[(size_t)k]]++;
        colT[(size_t)at] = (int)r;
        valT[(size_t)at] = val[(size_t)k];
      }
  }
  rsk_handle h = new (std::nothrow) rsk_handle_s();
  if (!h) return RSK_ENOMEM;
  h->device = device;
  h->ny = n;
  h->nx = n;
  h->r = 0;
  h->ct = true;
  h->ndata = m;
  h->ct_fro = fro;
  h->ct_nnz = nnz;
  if (cudaSetDevice(device) != cudaSuccess) { delete h; return RSK_ECUDA; }
  int smc = 148;
  cudaDeviceGetAttribute(&smc, cudaDevAttrMultiProcessorCount, device);
  h->sm_count = smc;
  h->ct_tmp_vecs = 128;
  h->scratch_bytes = std::max<size_t>(64u << 20, sizeof(double) * (size_t)std::max(N, m) * 2);
  bool ok = cudaMalloc(&h->wx, sizeof(double) * N) == cudaSuccess &&
            cudaMalloc(&h->wy, sizeof(double) * N) == cudaSuccess &&
            cudaMalloc(&h->scratch, h->scratch_bytes) == cudaSuccess &&
            cudaMalloc(&h->scal, sizeof(double) * 64) == cudaSuccess &&
            cudaMalloc(&h->aux, kAuxBytes) == cudaSuccess &&
            cudaMalloc(&h->ct_rp, sizeof(int64_t) * rp.size()) == cudaSuccess &&
            cudaMalloc(&h->ct_col, sizeof(int) * (size_t)nnz) == cudaSuccess &&
            cudaMalloc(&h->ct_val, sizeof(double) * (size_t)nnz) == cudaSuccess &&
            cudaMalloc(&h->ctT_rp, sizeof(int64_t) * rpT.size()) == cudaSuccess &&
            cudaMalloc(&h->ctT_col, sizeof(int) * (size_t)nnz) == cudaSuccess &&
            cudaMalloc(&h->ctT_val, sizeof(double) * (size_t)nnz) == cudaSuccess &&
            cudaMalloc(&h->ct_tmp, sizeof(double) * (size_t)m * h->ct_tmp_vecs) == cudaSuccess &&
            cudaStreamCreateWithFlags(&h->cg_stream, cudaStreamNonBlocking) == cudaSuccess;
  if (!ok) { rsk_destroy(h); return RSK_ENOMEM; }
  ok = cudaMemcpy(h->ct_rp, rp.data(), sizeof(int64_t) * rp.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(h->ct_col, col.data(), sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(h->ct_val, val.data(), sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(h->ctT_rp, rpT.data(), sizeof(int64_t) * rpT.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(h->ctT_col, colT.data(), sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(h->ctT_val, valT.data(), sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice) == cudaSuccess;
  std::vector<double> w((size_t)N);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) w[(size_t)(i * n + j)] = (j < n - 1) ? 1.0 : 0.0;
  ok = ok && cudaMemcpy(h->wx, w.data(), sizeof(double) * N, cudaMemcpyHostToDevice) == cudaSuccess;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) w[(size_t)(i * n + j)] = (i < n - 1) ? 1.0 : 0.0;
  ok = ok && cudaMemcpy(h->wy, w.data(), sizeof(double) * N, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemset(h->scratch, 0, h->scratch_bytes) == cudaSuccess;
  if (!ok) { rsk_destroy(h); return RSK_ECUDA; }
  *out = h;
  return RSK_OK;
}

extern "C" rsk_status rsk_ct_info(rsk_handle h, int64_t* ndata, int64_t* nnz, double* fro_unscaled) {
  if (!h || !h->ct) return RSK_EINVAL;
  if (ndata) *ndata = h->ndata;
  if (nnz) *nnz = h->ct_nnz;
  if (fro_unscaled) *fro_unscaled = h->ct_fro;
  return RSK_OK;
}
