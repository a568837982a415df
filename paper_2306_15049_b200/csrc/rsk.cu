// librsk C ABI: handle lifecycle, argument validation, and the host driver of the
// batched deflated CG (rsk_cg_recycled_batch). See include/rsk.h for the contract.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <vector>

#include "rsk_internal.h"

using namespace rsk;

struct rsk_handle_s : public Handle {};

namespace {

#define RSK_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      h->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call;    \
      h->sticky = true;                                                                \
      return RSK_ECUDA;                                                                \
    }                                                                                  \
  } while (0)

#define RSK_ARG(cond, msg)       \
  do {                           \
    if (!(cond)) {               \
      h->err = (msg);            \
      return RSK_EINVAL;         \
    }                            \
  } while (0)

inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }

// B = G^T G rows for a 1-D factor f (length 2r+1, tap f[b+r] multiplies y[j-b]).
// Window form: out[c] = sum_{t=0}^{4r} B[c][t] in[c - 2r + t],
// B[c][t] = sum_{j in [0,n)} f[j-c+r] f[j-m+r], m = c-2r+t.
void build_B_row(const double* f, int r, int64_t n, int64_t c, double* row) {
  const int T = 4 * r + 1;
  for (int t = 0; t < T; ++t) {
    const int64_t m = c - 2 * r + t;
    double s = 0.0;
    if (m >= 0 && m < n) {
      for (int64_t j = std::max<int64_t>(0, std::max(c, m) - r); j <= std::min<int64_t>(n - 1, std::min(c, m) + r); ++j) {
        const int64_t a = j - c + r, b = j - m + r;
        if (a >= 0 && a <= 2 * r && b >= 0 && b <= 2 * r) s += f[a] * f[b];
      }
    }
    row[t] = s;
  }
}

}  // namespace

namespace rsk {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace rsk

extern "C" int64_t rsk_launch_count(void) { return (int64_t)rsk::g_launches.load(); }

extern "C" const char* rsk_version(void) {
  return "librsk 0.1 (sm_100a, fp64): fused shifted apply, deflated CG, recycle projections";
}

extern "C" const char* rsk_last_error(rsk_handle h) { return h ? h->err.c_str() : "null handle"; }

extern "C" rsk_status rsk_create(rsk_handle* out, int device, int64_t ny, int64_t nx, const double* psf_h,
                                 int pny, int pnx, int flags) {
  (void)flags;
  if (!out || !psf_h || ny < 2 || nx < 2 || pny != pnx || pny % 2 != 1 || pny < 3 || pny > 2 * kMaxR + 1)
    return RSK_EINVAL;
  if (ny > (1 << 20) || nx > (1 << 20)) return RSK_EINVAL;
  const int r = pny / 2, P = pny;
  // rank-1 factorisation h = u v^T (pivot on the largest entry)
  int pi = 0, pj = 0;
  double hmax = 0.0;
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      const double a = std::fabs(psf_h[i * P + j]);
      if (!std::isfinite(psf_h[i * P + j])) return RSK_EINVAL;
      if (a > hmax) { hmax = a; pi = i; pj = j; }
    }
  if (hmax == 0.0) return RSK_EINVAL;
  double u[2 * kMaxR + 1], v[2 * kMaxR + 1];
  for (int i = 0; i < P; ++i) u[i] = psf_h[i * P + pj];
  for (int j = 0; j < P; ++j) v[j] = psf_h[pi * P + j] / psf_h[pi * P + pj];
  double res = 0.0;
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) res = std::max(res, std::fabs(psf_h[i * P + j] - u[i] * v[j]));
  // rank 2 (Example 1's C = sum_{i=1,2} C_i^(1) (x) C_i^(2)): the two leading
  // singular triplets of the P x P PSF, h = s1 U1 V1^T + s2 U2 V2^T (one-sided Jacobi SVD)
  int rank = 1;
  double u2[2 * kMaxR + 1] = {0}, v2[2 * kMaxR + 1] = {0};
  if (res > 1e-13 * hmax) {
    std::vector<double> Hc((size_t)P * P), Us((size_t)P * P), Vs((size_t)P * P), sv(P);
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < P; ++j) Hc[i + (size_t)j * P] = psf_h[i * P + j];
    jacobi_svd(P, Hc.data(), Us.data(), sv.data(), Vs.data());
    for (int i = 0; i < P; ++i) {
      u[i] = sv[0] * Us[i];
      v[i] = Vs[i];
      u2[i] = sv[1] * Us[i + P];
      v2[i] = Vs[i + P];
    }
    double res2 = 0.0;
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < P; ++j)
        res2 = std::max(res2, std::fabs(psf_h[i * P + j] - u[i] * v[j] - u2[i] * v2[j]));
    if (res2 > 1e-13 * hmax) return RSK_EUNSUPPORTED;   // rank > 2: no general 2-D path
    rank = 2;
  }

  rsk_handle h = new (std::nothrow) rsk_handle_s();
  if (!h) return RSK_ENOMEM;
  h->device = device;
  h->ny = ny;
  h->nx = nx;
  h->ndata = ny * nx;
  h->r = r;
  for (int i = 0; i < P; ++i) { h->u[i] = u[i]; h->v[i] = v[i]; h->u2[i] = u2[i]; h->v2[i] = v2[i]; }
  h->rank = rank;
  const int T = 4 * r + 1;
  for (int t = 0; t < kMaxTaps; ++t) {
    h->cBx[t] = h->cBy[t] = h->cCx[t] = h->cCy[t] = h->cTx[t] = h->cTy[t] = 0.0;
  }
  // interior rows of B (any interior c): autocorrelation
  {
    const int64_t big = 8 * (int64_t)r + 8;
    build_B_row(v, r, big, 4 * r + 4, h->cBx);
    build_B_row(u, r, big, 4 * r + 4, h->cBy);
  }
  // C: out[j] = sum_b f[b+r] in[j-b]  ->  t = 2r - b, tap = f[3r - t]   (t in [r, 3r])
  // C^T: out[m] = sum_b f[b+r] in[m+b] ->  t = b + 2r, tap = f[t - r]
  for (int t = 0; t < kMaxTaps; ++t) h->cCx2[t] = h->cCy2[t] = h->cTx2[t] = h->cTy2[t] = 0.0;
  for (int t = r; t <= 3 * r; ++t) {
    h->cCx[t] = v[3 * r - t];
    h->cCy[t] = u[3 * r - t];
    h->cTx[t] = v[t - r];
    h->cTy[t] = u[t - r];
    h->cCx2[t] = v2[3 * r - t];
    h->cCy2[t] = u2[3 * r - t];
    h->cTx2[t] = v2[t - r];
    h->cTy2[t] = u2[t - r];
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete h; return RSK_ECUDA; }
  int smc = 148;
  cudaDeviceGetAttribute(&smc, cudaDevAttrMultiProcessorCount, device);
  h->sm_count = smc;
  std::vector<double> tx((size_t)nx * T), ty((size_t)ny * T);
  for (int64_t c = 0; c < nx; ++c) build_B_row(v, r, nx, c, &tx[(size_t)c * T]);
  for (int64_t c = 0; c < ny; ++c) build_B_row(u, r, ny, c, &ty[(size_t)c * T]);
  const int64_t N = ny * nx;
  h->scratch_bytes = std::max<size_t>(64u << 20, sizeof(double) * (size_t)N * 2);
  bool ok = cudaMalloc(&h->tabBx, sizeof(double) * tx.size()) == cudaSuccess &&
            cudaMalloc(&h->tabBy, sizeof(double) * ty.size()) == cudaSuccess &&
            cudaMalloc(&h->wx, sizeof(double) * N) == cudaSuccess &&
            cudaMalloc(&h->wy, sizeof(double) * N) == cudaSuccess &&
            cudaMalloc(&h->scratch, h->scratch_bytes) == cudaSuccess &&
            cudaMalloc(&h->scal, sizeof(double) * 64) == cudaSuccess &&
            cudaMalloc(&h->aux, kAuxBytes) == cudaSuccess &&
            cudaStreamCreateWithFlags(&h->cg_stream, cudaStreamNonBlocking) == cudaSuccess;
  if (!ok) { rsk_destroy(h); return RSK_ENOMEM; }
  {
    // B_trunc = Toeplitz(B) - D_lo - D_hi: D_lo(c, m) = sum_{j<0} f[j-c+r] f[j-m+r] for
    // c, m < r; D_hi likewise with j >= n (the C-output rows outside the image)
    std::vector<double> dc((size_t)4 * kMaxR * kMaxR, 0.0);
    auto fill = [&](const double* f, int64_t n, int slot, int which) {
      for (int a = 0; a < r; ++a)
        for (int b = 0; b < r; ++b) {
          double sacc = 0.0;
          const int64_t c = which ? n - r + a : a, m = which ? n - r + b : b;
          const int64_t jlo = which ? n : -r, jhi = which ? n + r : 0;
          for (int64_t j = jlo; j < jhi; ++j) {
            const int64_t ia = j - c + r, ib = j - m + r;
            if (ia >= 0 && ia <= 2 * r && ib >= 0 && ib <= 2 * r) sacc += f[ia] * f[ib];
          }
          dc[((size_t)slot * kMaxR + a) * kMaxR + b] = sacc;
        }
    };
    fill(v, nx, 0, 0);
    fill(v, nx, 1, 1);
    fill(u, ny, 2, 0);
    fill(u, ny, 3, 1);
    ok = cudaMalloc(&h->dcorr, sizeof(double) * dc.size()) == cudaSuccess &&
         cudaMemcpy(h->dcorr, dc.data(), sizeof(double) * dc.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) { rsk_destroy(h); return RSK_ENOMEM; }
  }
  std::vector<double> w((size_t)N);
  ok = cudaMemcpy(h->tabBx, tx.data(), sizeof(double) * tx.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(h->tabBy, ty.data(), sizeof(double) * ty.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  for (int64_t i = 0; i < ny; ++i)
    for (int64_t j = 0; j < nx; ++j) w[(size_t)(i * nx + j)] = (j < nx - 1) ? 1.0 : 0.0;
  ok = ok && cudaMemcpy(h->wx, w.data(), sizeof(double) * N, cudaMemcpyHostToDevice) == cudaSuccess;
  for (int64_t i = 0; i < ny; ++i)
    for (int64_t j = 0; j < nx; ++j) w[(size_t)(i * nx + j)] = (i < ny - 1) ? 1.0 : 0.0;
  ok = ok && cudaMemcpy(h->wy, w.data(), sizeof(double) * N, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemset(h->scratch, 0, h->scratch_bytes) == cudaSuccess;
  if (!ok) { rsk_destroy(h); return RSK_ECUDA; }
  *out = h;
  return RSK_OK;
}

extern "C" rsk_status rsk_create_slab(rsk_handle* out, int device, int64_t ny_global, int64_t nx, int64_t row0,
                                      int64_t nrows, const double* psf_h, int pny, int pnx, int halo, int flags) {
  if (!out || ny_global < 2 || nx < 2 || row0 < 0 || nrows < 1 || row0 + nrows > ny_global) return RSK_EINVAL;
  if (pny != pnx || pny % 2 != 1 || halo < 2 * (pny / 2) || nrows < halo) return RSK_EINVAL;
  const int64_t e0 = std::max<int64_t>(0, row0 - halo), e1 = std::min<int64_t>(ny_global, row0 + nrows + halo);
  rsk_status st = rsk_create(out, device, e1 - e0, nx, psf_h, pny, pnx, flags);
  if (st != RSK_OK) return st;
  rsk_handle h = *out;
  h->ny_global = ny_global;
  h->slab_ext0 = e0;
  h->slab_ext1 = e1;
  h->slab_row0 = row0;
  h->slab_row1 = row0 + nrows;
  h->slab_halo = halo;
  return RSK_OK;
}

extern "C" rsk_status rsk_slab_info(rsk_handle h, int64_t* info6_h) {
  if (!h || !info6_h || h->ny_global == 0) return RSK_EINVAL;
  info6_h[0] = h->ny_global;
  info6_h[1] = h->slab_ext0;
  info6_h[2] = h->slab_ext1;
  info6_h[3] = h->slab_row0;
  info6_h[4] = h->slab_row1;
  info6_h[5] = h->slab_halo;
  return RSK_OK;
}

extern "C" rsk_status rsk_destroy(rsk_handle h) {
  if (!h) return RSK_EINVAL;
  cudaSetDevice(h->device);
  cudaFree(h->r2buf);
  cudaFree(h->tabBx);
  cudaFree(h->tabBy);
  cudaFree(h->dcorr);
  cudaFree(h->wx);
  cudaFree(h->wy);
  cudaFree(h->scratch);
  cudaFree(h->scal);
  cudaFree(h->aux);
  cudaFree(h->ct_rp);
  cudaFree(h->ct_col);
  cudaFree(h->ct_val);
  cudaFree(h->ctT_rp);
  cudaFree(h->ctT_col);
  cudaFree(h->ctT_val);
  cudaFree(h->ct_tmp);
  if (h->cg_stream) cudaStreamDestroy(h->cg_stream);
  delete h;
  return RSK_OK;
}

// validity of a weight pair (rsk_set_weights): bit 0 = a non-finite or negative value,
// bit 1 = a non-zero pad (wx[:, nx-1]; wy[ny-1, :] when this handle holds the last row)
__global__ void weights_check_kernel(const double* __restrict__ wx, const double* __restrict__ wy, int64_t ny,
                                     int64_t nx, int bottom, int* flag) {
  int f = 0;
  const int64_t N = ny * nx;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = wx[i], b = wy[i];
    if (!(a >= 0.0) || !(b >= 0.0) || !isfinite(a) || !isfinite(b)) f |= 1;
    if ((i % nx == nx - 1) && a != 0.0) f |= 2;
    if (bottom && i >= N - nx && b != 0.0) f |= 2;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flag, f);
}

extern "C" rsk_status rsk_set_weights(rsk_handle h, const double* wx, const double* wy, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(wx && wy && aligned8(wx) && aligned8(wy), "rsk_set_weights: null or misaligned pointer");
  const size_t bytes = sizeof(double) * (size_t)(h->ny * h->nx);
  // validate before adopting (weights reach 1/tau, so only >= 0 and finite are required;
  // the pads of L's missing rows must be 0). A host sync point, once per outer step.
  int* flag = reinterpret_cast<int*>(h->scal + 63);   // reserved for this check
  RSK_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), S(stream)));
  const int bottom = (h->ny_global == 0 || h->slab_ext1 == h->ny_global) ? 1 : 0;
  count_launch();
  weights_check_kernel<<<2 * h->sm_count, 256, 0, S(stream)>>>(wx, wy, h->ny, h->nx, bottom, flag);
  RSK_CUDA(cudaGetLastError());
  int hf = 0;
  RSK_CUDA(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, S(stream)));
  RSK_CUDA(cudaStreamSynchronize(S(stream)));
  RSK_ARG(!(hf & 1), "rsk_set_weights: a weight is negative or not finite");
  RSK_ARG(!(hf & 2), "rsk_set_weights: non-zero pad (wx[:, nx-1] and wy[ny-1, :] must be 0)");
  RSK_CUDA(cudaMemcpyAsync(h->wx, wx, bytes, cudaMemcpyDeviceToDevice, S(stream)));
  RSK_CUDA(cudaMemcpyAsync(h->wy, wy, bytes, cudaMemcpyDeviceToDevice, S(stream)));
  return RSK_OK;
}

extern "C" rsk_status rsk_apply_shifted_rows(rsk_handle h, int nvec, const double* X, int64_t ldx,
                                             const double* gamma, double* Y, int64_t ldy, double* EY,
                                             int64_t ldey, double* xdoty, int mode, int64_t row0, int64_t row1,
                                             void* stream) {
  if (!h) return RSK_EINVAL;
  const int64_t N = h->ny * h->nx;
  RSK_ARG(nvec >= 0, "rsk_apply_shifted_rows: nvec < 0");
  RSK_ARG(row0 >= 0 && row0 < row1 && row1 <= h->ny, "rsk_apply_shifted_rows: bad row range");
  if (nvec == 0) return RSK_OK;
  RSK_ARG(mode >= RSK_APPLY_SHIFTED && mode <= RSK_APPLY_CT_ONLY, "rsk_apply_shifted_rows: bad mode");
  if (mode != RSK_APPLY_SHIFTED && mode != RSK_APPLY_SPLIT) {
    h->err = "rsk_apply_shifted_rows: SHIFTED and SPLIT only";
    return RSK_EUNSUPPORTED;
  }
  RSK_ARG(X && Y && aligned8(X) && aligned8(Y), "rsk_apply_shifted_rows: null/misaligned X or Y");
  RSK_ARG(ldx >= N && ldy >= N, "rsk_apply_shifted_rows: ld < N");
  RSK_ARG(mode != RSK_APPLY_SHIFTED || gamma, "rsk_apply_shifted_rows: gamma required");
  RSK_ARG(mode != RSK_APPLY_SPLIT || (EY && ldey >= N), "rsk_apply_shifted_rows: EY required for SPLIT");
  {
    const char* xb = (const char*)X;
    const char* xe = (const char*)(X + (nvec - 1) * ldx + N);
    const char* yb = (const char*)Y;
    const char* ye = (const char*)(Y + (nvec - 1) * ldy + N);
    RSK_ARG(ye <= xb || yb >= xe, "rsk_apply_shifted_rows: X and Y overlap");
  }
  if (N < kStripMinN || h->rank != 1 || h->ct) {
    h->err = "rsk_apply_shifted_rows: only the streaming strip core takes a row range";
    return RSK_EUNSUPPORTED;
  }
  ApplyLaunch a{};
  a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy; a.EY = EY; a.ldey = ldey;
  a.gamma = gamma; a.list = nullptr; a.nlist = nvec; a.mode = mode; a.xdoty = xdoty;
  a.cg = nullptr; a.cg_alpha = false;
  const cudaError_t e = launch_apply_strip(h, a, S(stream), (int)row0, (int)row1);
  if (e == cudaErrorNotSupported) {
    h->err = "rsk_apply_shifted_rows: strip core not applicable (width / alignment)";
    return RSK_EUNSUPPORTED;
  }
  RSK_CUDA(e);
  if (row0 == 0 && row1 == h->ny) {
    h->nA += nvec;
    h->nE += nvec;
  }
  return RSK_OK;
}

extern "C" rsk_status rsk_apply_shifted(rsk_handle h, int nvec, const double* X, int64_t ldx,
                                        const double* gamma, double* Y, int64_t ldy, double* EY,
                                        int64_t ldey, double* xdoty, int mode, void* stream) {
  if (!h) return RSK_EINVAL;
  const int64_t N = h->ny * h->nx;
  RSK_ARG(nvec >= 0, "rsk_apply_shifted: nvec < 0");
  if (nvec == 0) return RSK_OK;
  RSK_ARG(mode >= RSK_APPLY_SHIFTED && mode <= RSK_APPLY_CT_ONLY, "rsk_apply_shifted: bad mode");
  RSK_ARG(X && Y && aligned8(X) && aligned8(Y), "rsk_apply_shifted: null/misaligned X or Y");
  // lengths: images N; data vectors (C X output, C^T X input) ndata (= N for the blur)
  const int64_t nin = (mode == RSK_APPLY_CT_ONLY) ? h->ndata : N;
  const int64_t nout = (mode == RSK_APPLY_C_ONLY) ? h->ndata : N;
  RSK_ARG(ldx >= nin && ldy >= nout, "rsk_apply_shifted: ld < vector length");
  RSK_ARG(mode != RSK_APPLY_SHIFTED || gamma, "rsk_apply_shifted: gamma required");
  RSK_ARG(mode != RSK_APPLY_SPLIT || (EY && ldey >= N), "rsk_apply_shifted: EY required for SPLIT");
  {  // X and Y (and EY) must not overlap
    const char* xb = (const char*)X;
    const char* xe = (const char*)(X + (nvec - 1) * ldx + nin);
    const char* yb = (const char*)Y;
    const char* ye = (const char*)(Y + (nvec - 1) * ldy + nout);
    RSK_ARG(ye <= xb || yb >= xe, "rsk_apply_shifted: X and Y overlap");
    if (mode == RSK_APPLY_SPLIT) {
      const char* eb = (const char*)EY;
      const char* ee = (const char*)(EY + (nvec - 1) * ldey + N);
      RSK_ARG((ee <= xb || eb >= xe) && (ee <= yb || eb >= ye), "rsk_apply_shifted: EY overlaps");
    }
  }
  ApplyLaunch a{};
  a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy; a.EY = EY; a.ldey = ldey;
  a.gamma = gamma; a.list = nullptr; a.nlist = nvec; a.mode = mode; a.xdoty = xdoty;
  a.cg = nullptr; a.cg_alpha = false;
  RSK_CUDA(launch_apply(h, a, S(stream)));
  if (mode == RSK_APPLY_SHIFTED || mode == RSK_APPLY_SPLIT) {
    h->nA += nvec;
    h->nE += nvec;
  } else {
    h->nC += nvec;
  }
  return RSK_OK;
}

extern "C" rsk_status rsk_recycle_project(rsk_handle h, int op, int64_t n, int k, const double* U,
                                          int64_t ldu, int nv, double* V, int64_t ldv, double* Cm,
                                          int64_t ldc, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(op >= RSK_PROJ_UTV && op <= RSK_SUB_UC, "rsk_recycle_project: bad op");
  RSK_ARG(n >= 1 && k >= 1 && k <= 256 && nv >= 1, "rsk_recycle_project: bad sizes");
  RSK_ARG(U && V && Cm && aligned8(U) && aligned8(V) && aligned8(Cm), "rsk_recycle_project: null/misaligned");
  RSK_ARG(ldu >= n && ldv >= n && ldc >= k, "rsk_recycle_project: bad leading dimension");
  if (op == RSK_PROJ_UTV) {
    RSK_CUDA(launch_gemm_tn(h, n, k, U, ldu, nv, V, ldv, Cm, ldc, S(stream)));
  } else {
    const char* ub = (const char*)U;
    const char* ue = (const char*)(U + (k - 1) * ldu + n);
    const char* vb = (const char*)V;
    const char* ve = (const char*)(V + (nv - 1) * ldv + n);
    RSK_ARG(ve <= ub || vb >= ue, "rsk_recycle_project: U and V overlap");
    RSK_CUDA(launch_gemm_nn(h, n, k, U, ldu, nv, V, ldv, Cm, ldc, op == RSK_ADD_UC ? 1.0 : -1.0, S(stream)));
  }
  return RSK_OK;
}

extern "C" rsk_status rsk_irn_weights(rsk_handle h, const double* x, double tau, double* wx, double* wy,
                                      double* eta2, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(x && aligned8(x), "rsk_irn_weights: null x");
  RSK_ARG(std::isfinite(tau) && tau > 0.0, "rsk_irn_weights: tau must be finite and > 0");
  RSK_ARG((wx == nullptr) == (wy == nullptr), "rsk_irn_weights: wx and wy must both be given or both NULL");
  RSK_ARG(wx || eta2, "rsk_irn_weights: nothing to compute");
  RSK_CUDA(launch_irn(h, x, tau, 0, wx, wy, eta2, S(stream)));
  return RSK_OK;
}

extern "C" rsk_status rsk_irn_weights_iso(rsk_handle h, const double* x, double tau, double* wx, double* wy,
                                          double* eta2, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(x && aligned8(x), "rsk_irn_weights_iso: null x");
  RSK_ARG(std::isfinite(tau) && tau > 0.0, "rsk_irn_weights_iso: tau must be finite and > 0");
  RSK_ARG((wx == nullptr) == (wy == nullptr), "rsk_irn_weights_iso: wx and wy must both be given or both NULL");
  RSK_ARG(wx || eta2, "rsk_irn_weights_iso: nothing to compute");
  RSK_CUDA(launch_irn(h, x, tau, 1, wx, wy, eta2, S(stream)));
  return RSK_OK;
}

extern "C" rsk_status rsk_gazzola_max(rsk_handle h, const double* x, const double* dx, const double* dy,
                                      double* m, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(x && dx && dy && m, "rsk_gazzola_max: null pointer");
  RSK_ARG(aligned8(x) && aligned8(dx) && aligned8(dy) && aligned8(m), "rsk_gazzola_max: misaligned pointer");
  RSK_CUDA(launch_gazzola_max(h, x, dx, dy, m, S(stream)));
  return RSK_OK;
}

extern "C" rsk_status rsk_gazzola_update(rsk_handle h, const double* x, double p, const double* m, double* dx,
                                         double* dy, double* wx, double* wy, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(x && m && dx && dy && wx && wy, "rsk_gazzola_update: null pointer");
  RSK_ARG(aligned8(x) && aligned8(m) && aligned8(dx) && aligned8(dy) && aligned8(wx) && aligned8(wy),
          "rsk_gazzola_update: misaligned pointer");
  RSK_ARG(std::isfinite(p) && p > 0.0, "rsk_gazzola_update: p must be finite and > 0");
  RSK_ARG(dx != dy && wx != wy && wx != dx && wx != dy && wy != dx && wy != dy,
          "rsk_gazzola_update: dx, dy, wx, wy must be four distinct arrays");
  RSK_CUDA(launch_gazzola_update(h, x, p, m, dx, dy, wx, wy, S(stream)));
  return RSK_OK;
}

extern "C" rsk_status rsk_gazzola_weights(rsk_handle h, const double* x, double p, double* dx, double* dy,
                                          double* wx, double* wy, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(x && dx && dy && wx && wy, "rsk_gazzola_weights: null pointer");
  RSK_ARG(std::isfinite(p) && p > 0.0, "rsk_gazzola_weights: p must be finite and > 0");
  // the max goes to the last scratch slot (the per-chunk partials fill it from the front)
  double* m = h->scratch + (h->scratch_bytes / sizeof(double) - 1);
  rsk_status s = rsk_gazzola_max(h, x, dx, dy, m, stream);
  if (s != RSK_OK) return s;
  return rsk_gazzola_update(h, x, p, m, dx, dy, wx, wy, stream);
}

extern "C" rsk_status rsk_make_rhs(rsk_handle h, const double* x_true, const double* xi, double nu,
                                   double* d, double* b, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(x_true && xi && d && b, "rsk_make_rhs: null pointer");
  RSK_ARG(std::isfinite(nu) && nu >= 0.0, "rsk_make_rhs: bad noise level");
  const int64_t N = h->ny * h->nx, M = h->ndata;   // image and data lengths
  rsk_status s = rsk_apply_shifted(h, 1, x_true, N, nullptr, d, M, nullptr, N, nullptr, RSK_APPLY_C_ONLY, stream);
  if (s != RSK_OK) return s;
  RSK_CUDA(launch_batch_dot(h, M, 1, d, M, d, M, h->scal + 0, S(stream)));
  RSK_CUDA(launch_batch_dot(h, M, 1, xi, M, xi, M, h->scal + 1, S(stream)));
  RSK_CUDA(launch_scale_noise(M, d, xi, h->scal, nu, d, S(stream)));
  return rsk_apply_shifted(h, 1, d, M, nullptr, b, N, nullptr, N, nullptr, RSK_APPLY_CT_ONLY, stream);
}

extern "C" rsk_status rsk_batch_dot(rsk_handle h, int64_t n, int nv, const double* X, int64_t ldx,
                                    const double* Y, int64_t ldy, double* out, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(n >= 1 && nv >= 1 && X && Y && out && ldx >= n && ldy >= n, "rsk_batch_dot: bad arguments");
  RSK_CUDA(launch_batch_dot(h, n, nv, X, ldx, Y, ldy, out, S(stream)));
  return RSK_OK;
}

extern "C" rsk_status rsk_batch_axpby(rsk_handle h, int64_t n, int nv, const double* a_h, const double* X,
                                      int64_t ldx, const double* b_h, double* Y, int64_t ldy, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(n >= 1 && nv >= 1 && nv <= 1024 && a_h && Y && ldy >= n && (!X || ldx >= n), "rsk_batch_axpby: bad arguments");
  double* dev = h->aux + 2 * 256 * 256;
  RSK_CUDA(cudaMemcpyAsync(dev, a_h, sizeof(double) * nv, cudaMemcpyHostToDevice, S(stream)));
  if (b_h) RSK_CUDA(cudaMemcpyAsync(dev + 1024, b_h, sizeof(double) * nv, cudaMemcpyHostToDevice, S(stream)));
  RSK_CUDA(launch_batch_axpby(n, nv, dev, X, ldx, b_h ? dev + 1024 : nullptr, Y, ldy, S(stream)));
  return RSK_OK;
}

// Shifted Cholesky QR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020):
// backward-stable thin QR of an ill-conditioned tall-skinny block in three
// Gram passes. V (n x k) is overwritten; Q (n x k) receives the orthonormal factor.
// Host step of one shifted-Cholesky-QR pass (Fukaya et al. 2020) from the Gram matrix G =
// V^T V of the pass's input (k x k, column-major): T = R_pass^-1 (upper, column-major) so
// that V T is the pass's output, and Racc <- R_pass Racc. Pass 0 equilibrates with the Gram
// diagonal and adds the shift 11 (n k + k (k+1)) u ||G||; later passes are unshifted unless
// Cholesky needs it. Shared by rsk_qr_tall (one domain) and the row-slab QR (Gram
// all-reduced over slabs).
extern "C" rsk_status rsk_cholqr_pass(int k, int64_t n, int pass, const double* G_h, double* T_h, double* Racc_h) {
  if (k < 1 || k > 256 || n < k || pass < 0 || !G_h || !T_h || !Racc_h) return RSK_EINVAL;
  std::vector<double> G(G_h, G_h + (size_t)k * k), Rn((size_t)k * k);
  std::vector<double> dsc(k, 1.0);
  if (pass == 0)
    for (int j = 0; j < k; ++j) dsc[j] = G[j + j * k] > 0 ? 1.0 / std::sqrt(G[j + j * k]) : 1.0;
  std::vector<double> L((size_t)k * k);
  double shift = 0.0;
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) L[i + j * k] = 0.5 * (G[i + j * k] + G[j + i * k]) * dsc[i] * dsc[j];
  double nrm2 = 0.0;
  for (int j = 0; j < k; ++j) nrm2 += L[j + j * k];
  if (pass == 0) shift = 11.0 * ((double)n * k + (double)k * (k + 1)) * 1.1102230246251565e-16 * nrm2;
  std::vector<double> L0 = L;
  int tries = 0;
  for (;;) {
    L = L0;
    for (int j = 0; j < k; ++j) L[j + j * k] += shift;
    if (rsk::chol_lower(k, L.data())) break;
    shift = shift > 0 ? shift * 10.0 : 1e-15 * std::max(nrm2, 1e-300);
    if (++tries > 40) return RSK_EPARTIAL;
  }
  // R_pass = L^T D^-1 ; T = (R_pass)^-1 = D L^-T (upper)
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) Rn[i + j * k] = (i <= j) ? L[j + i * k] / dsc[j] : 0.0;
  for (size_t e = 0; e < (size_t)k * k; ++e) T_h[e] = 0.0;
  for (int j = 0; j < k; ++j) {
    T_h[j + j * k] = 1.0 / Rn[j + j * k];
    for (int i = j - 1; i >= 0; --i) {
      double t = 0.0;
      for (int q = i + 1; q <= j; ++q) t += Rn[i + q * k] * T_h[q + j * k];
      T_h[i + j * k] = -t / Rn[i + i * k];
    }
  }
  if (pass == 0) {
    for (size_t e = 0; e < (size_t)k * k; ++e) Racc_h[e] = Rn[e];
  } else {
    std::vector<double> tmp((size_t)k * k, 0.0);
    for (int j = 0; j < k; ++j)
      for (int i = 0; i <= j; ++i) {
        double t = 0.0;
        for (int q = i; q <= j; ++q) t += Rn[i + q * k] * Racc_h[q + j * k];
        tmp[i + j * k] = t;
      }
    for (size_t e = 0; e < (size_t)k * k; ++e) Racc_h[e] = tmp[e];
  }
  return RSK_OK;
}

extern "C" rsk_status rsk_qr_tall(rsk_handle h, int64_t n, int k, double* V, int64_t ldv, double* Q,
                                  int64_t ldq, double* R_h, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(n >= 1 && k >= 1 && k <= 256 && n >= k && V && Q && R_h && ldv >= n && ldq >= n,
          "rsk_qr_tall: bad arguments");
  cudaStream_t st = S(stream);
  std::vector<double> G((size_t)k * k), T((size_t)k * k), Racc((size_t)k * k, 0.0);
  double* dG = h->aux;
  double* dT = h->aux + 256 * 256;
  for (int pass = 0; pass < 3; ++pass) {   // passes write Q, V, Q
    double* src = (pass % 2 == 0) ? V : Q;
    const int64_t lds = (pass % 2 == 0) ? ldv : ldq;
    double* dst = (pass % 2 == 0) ? Q : V;
    const int64_t ldd = (pass % 2 == 0) ? ldq : ldv;
    RSK_CUDA(launch_gemm_tn(h, n, k, src, lds, k, src, lds, dG, k, st));
    RSK_CUDA(cudaMemcpyAsync(G.data(), dG, sizeof(double) * k * k, cudaMemcpyDeviceToHost, st));
    RSK_CUDA(cudaStreamSynchronize(st));
    if (rsk_cholqr_pass(k, n, pass, G.data(), T.data(), Racc.data()) != RSK_OK) {
      h->err = "rsk_qr_tall: Cholesky failed";
      return RSK_EPARTIAL;
    }
    RSK_CUDA(cudaMemcpyAsync(dT, T.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, st));
    RSK_CUDA(cudaMemset2DAsync(dst, sizeof(double) * ldd, 0, sizeof(double) * n, k, st));
    RSK_CUDA(launch_gemm_nn(h, n, k, src, lds, k, dst, ldd, dT, k, 1.0, st));
  }
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) R_h[i + j * k] = Racc[i + j * k];
  RSK_CUDA(cudaStreamSynchronize(st));
  return RSK_OK;
}

extern "C" rsk_status rsk_lcurve_norms(rsk_handle h, int nvec, const double* X, int64_t ldx, const double* d,
                                       double* rho, double* eta2, void* scratch, void* stream) {
  if (!h) return RSK_EINVAL;
  const int64_t N = h->ny * h->nx;
  RSK_ARG(nvec >= 1 && X && d && rho && eta2 && scratch && ldx >= N, "rsk_lcurve_norms: bad arguments");
  double* Y = static_cast<double*>(scratch);
  const int64_t M = h->ndata;   // data length (scratch: nvec x ndata)
  rsk_status s = rsk_apply_shifted(h, nvec, X, ldx, nullptr, Y, M, nullptr, N, nullptr, RSK_APPLY_C_ONLY, stream);
  if (s != RSK_OK) return s;
  RSK_CUDA(launch_diffnorm_batch(h, nvec, Y, M, d, rho, S(stream)));
  RSK_CUDA(launch_seminorm_batch(h, nvec, X, ldx, eta2, S(stream), /*do_sqrt=*/1));
  return RSK_OK;
}

extern "C" rsk_status rsk_seminorm_rows(rsk_handle h, int nvec, const double* X, int64_t ldx, int64_t row0,
                                        int64_t row1, double* eta2, void* stream) {
  if (!h) return RSK_EINVAL;
  const int64_t N = h->ny * h->nx;
  RSK_ARG(nvec >= 1 && X && eta2 && ldx >= N && row0 >= 0 && row0 < row1 && row1 <= h->ny,
          "rsk_seminorm_rows: bad arguments");
  RSK_CUDA(launch_seminorm_rows(h, nvec, X, ldx, (int)row0, (int)row1, eta2, S(stream)));
  return RSK_OK;
}

extern "C" rsk_status rsk_get_counters(rsk_handle h, int64_t* a, int64_t* e, int64_t* c, int reset) {
  if (!h) return RSK_EINVAL;
  if (a) *a = h->nA;
  if (e) *e = h->nE;
  if (c) *c = h->nC;
  if (reset) h->nA = h->nE = h->nC = 0;
  return RSK_OK;
}

// ============================================================== batched deflated CG
namespace {

struct WsLayout {
  size_t off_R, off_P, off_W, off_dbl, off_int, off_cnt, off_pA, off_pB, off_list, off_dev, off_gb, total;
  size_t off_glist, off_partG, off_cntG, off_partP, off_pbar, off_zw, off_sA, off_sB;
  int nchunkP;
  int64_t rowsP;
  int nblkA, nblkB;
  int nchunkG, maxtilesG;
  int64_t rowsG;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

WsLayout ws_layout(const Handle* h, int ns) {
  WsLayout L{};
  const int64_t N = h->ny * h->nx;
  L.nblkA = apply_tiles(h);
  L.nblkB = cg_nblkB(N);
  // group kernels: row chunks of a multiple of 32 rows, at most kMaxChunkG chunks
  int64_t rows = (N + kMaxChunkG - 1) / kMaxChunkG;
  if (rows < 256) rows = 256;
  rows = (rows + 255) / 256 * 256;   // whole 256-row sub-slabs (cg_group.cu)
  L.rowsG = rows;
  L.nchunkG = (int)((N + rows - 1) / rows);
  L.maxtilesG = (ns + 31) / 32;
  size_t o = 0;
  L.off_glist = o; o = al(o + sizeof(int) * (size_t)(ns + 16));
  L.off_partG = o;
  o = al(o + sizeof(double) * (size_t)RSK_MAX_GROUPS * L.maxtilesG * (L.nchunkG + 16) * kPartRowsG * 32);
  L.off_cntG = o; o = al(o + sizeof(unsigned) * (size_t)RSK_MAX_GROUPS * L.maxtilesG * kTickStride);
  L.off_R = o; o = al(o + sizeof(double) * (size_t)N * ns);
  L.off_P = o; o = al(o + sizeof(double) * (size_t)N * ns);
  L.off_W = o; o = al(o + sizeof(double) * (size_t)N * ns);
  L.off_dbl = o; o = al(o + sizeof(double) * (size_t)ns * (5 + kMaxM + kMaxM * kMaxM));
  L.off_int = o; o = al(o + sizeof(int) * (size_t)ns * 8);
  L.off_cnt = o; o = al(o + sizeof(unsigned) * (size_t)ns * 4);
  L.off_pA = o; o = al(o + sizeof(double) * (size_t)ns * L.nblkA);
  L.off_pB = o; o = al(o + sizeof(double) * (size_t)ns * L.nblkB * (kMaxM + 1));
  L.off_list = o; o = al(o + sizeof(int) * (size_t)ns * 3);
  L.off_dev = o; o = al(o + sizeof(CgDev));
  L.off_gb = o; o = al(o + sizeof(double) * (size_t)(RSK_MAX_GROUPS * (2 * 16 * 16 + 3 * 16 * ns) + ns));
  // persistent loop: one row chunk (multiple of 256 rows) per CTA of the cooperative grid
  {
    const int pg = persist_grid(h);
    int64_t rp = (N + pg - 1) / pg;
    rp = (rp + 255) / 256 * 256;
    L.rowsP = rp;
    L.nchunkP = (int)((N + rp - 1) / rp);
  }
  L.off_partP = o; o = al(o + sizeof(double) * (size_t)ns * (L.nchunkP * persist_pv() + persist_grid(h)));
  L.off_pbar = o; o = al(o + sizeof(unsigned) * 8);
  // streaming loop (cg_stream.cu): per-item apply partials and per-chunk B partials
  L.off_sA = o; o = al(o + sizeof(double) * (size_t)2 * ns * stream_ipv(h));   // hi, lo (double-double)
  L.off_sB = o; o = al(o + sizeof(double) * (size_t)ns * stream_pv() * stream_nchunk(h));
  // cluster-per-shift loop: per cluster, Z_s = AW + gamma_s EW of its current shift
  L.off_zw = o;
  if (N <= cluster_max_n()) o = al(o + sizeof(double) * (size_t)cluster_slots(h) * 16 * N);
  L.total = o;
  return L;
}

}  // namespace

extern "C" size_t rsk_cg_workspace_bytes(rsk_handle h, int nshift, int flags) {
  (void)flags;
  if (!h || nshift <= 0) return 0;
  if (h->ct) return 256;   // CT handles: rsk_minres_recycled_batch only
  return ws_layout(h, nshift).total;
}

extern "C" rsk_status rsk_cg_recycled_batch(rsk_handle h, const rsk_cg_desc* d, rsk_cg_out* o, void* ws,
                                            size_t ws_bytes, void* stream) {
  if (!h) return RSK_EINVAL;
  RSK_ARG(d && o, "rsk_cg_recycled_batch: null desc/out");
  if (h->ct || h->rank != 1) {
    h->err = "rsk_cg_recycled_batch: the CG device loops embed the rank-1 stencil apply; CT and rank-2 "
             "handles use rsk_minres_recycled_batch";
    return RSK_EUNSUPPORTED;
  }
  const int ns = d->nshift;
  const int64_t N = h->ny * h->nx;
  RSK_ARG(ns >= 1, "rsk_cg_recycled_batch: nshift < 1");
  RSK_ARG(d->gamma_h && d->b && d->X && d->ldx >= N, "rsk_cg_recycled_batch: gamma/b/X");
  RSK_ARG(o->iters && o->applies && o->relres_true && o->status && o->m_used, "rsk_cg_recycled_batch: outputs");
  RSK_ARG(d->tol > 0 && std::isfinite(d->tol) && d->maxit >= 1 && d->check_every >= 1, "rsk_cg_recycled_batch: tol/maxit/check_every");
  const bool defl = !(d->flags & RSK_CG_NO_DEFLATION) && d->ngroups > 0;
  RSK_ARG(d->ngroups >= 0 && d->ngroups <= RSK_MAX_GROUPS, "rsk_cg_recycled_batch: ngroups");
  if (defl) {
    RSK_ARG(d->group_of_shift_h && d->ldw >= N, "rsk_cg_recycled_batch: groups");
    for (int g = 0; g < d->ngroups; ++g)
      RSK_ARG(d->J[g] >= 0 && d->J[g] <= 16 && (d->J[g] == 0 || (d->W[g] && d->AW[g] && d->EW[g])),
              "rsk_cg_recycled_batch: group block");
    for (int s = 0; s < ns; ++s)
      RSK_ARG(d->group_of_shift_h[s] >= 0 && d->group_of_shift_h[s] < d->ngroups, "rsk_cg_recycled_batch: group index");
  }
  const bool anyg = defl && d->has_ghat_h != nullptr;
  if (anyg) RSK_ARG(d->Ghat && d->ZGhat && d->ldgh >= N, "rsk_cg_recycled_batch: Ghat/ZGhat");
  if (d->has_ghat2_h)
    for (int s = 0; s < ns; ++s)
      RSK_ARG(d->has_ghat2_h[s] == 0, "rsk_cg_recycled_batch: a second carried column (Alg. 3) needs rsk_minres_recycled_batch");
  const bool store = (d->flags & RSK_CG_STORE_RES) != 0;
  if (store) RSK_ARG(d->store && d->store_cap >= 1 && d->lds >= N, "rsk_cg_recycled_batch: store");
  for (int s = 0; s < ns; ++s) RSK_ARG(std::isfinite(d->gamma_h[s]) && d->gamma_h[s] >= 0, "rsk_cg_recycled_batch: gamma");
  const WsLayout L = ws_layout(h, ns);
  RSK_ARG(ws && ws_bytes >= L.total, "rsk_cg_recycled_batch: workspace too small");
  // The call is host-blocking: drain the caller's stream, then run on the handle's
  // private non-blocking stream (CUDA-graph capture is not allowed on the legacy
  // default stream), and drain that before returning.
  const auto t_enter = std::chrono::steady_clock::now();
  RSK_CUDA(cudaStreamSynchronize(S(stream)));
  const auto t_drained = std::chrono::steady_clock::now();
  cudaStream_t st = h->cg_stream;
  const bool prof = (d->flags & RSK_CG_PROFILE) != 0 && o->ms_loop;

  char* base = static_cast<char*>(ws);
  CgDev hc{};
  hc.nshift = ns;
  hc.N = N;
  hc.R = reinterpret_cast<double*>(base + L.off_R);
  hc.P = reinterpret_cast<double*>(base + L.off_P);
  hc.Wv = reinterpret_cast<double*>(base + L.off_W);
  hc.X = d->X;
  hc.ldx = d->ldx;
  hc.b = d->b;
  hc.Ghat = anyg ? d->Ghat : nullptr;
  hc.ZGhat = anyg ? d->ZGhat : nullptr;
  hc.ldgh = d->ldgh;
  hc.store = store ? d->store : nullptr;
  hc.lds = d->lds;
  hc.store_cap = store ? d->store_cap : 0;
  double* dbl = reinterpret_cast<double*>(base + L.off_dbl);
  hc.gam = dbl;
  hc.rho = dbl + ns;
  hc.alpha = dbl + 2 * ns;
  hc.beta = dbl + 3 * ns;
  hc.rho_true = dbl + 4 * ns;
  hc.coef = dbl + 5 * ns;
  hc.Lf = hc.coef + (size_t)ns * kMaxM;
  int* in = reinterpret_cast<int*>(base + L.off_int);
  hc.status = in;
  hc.iters = in + ns;
  hc.mloc = in + 2 * ns;
  hc.hasg = in + 3 * ns;
  hc.group = in + 4 * ns;
  hc.store_cnt = in + 5 * ns;
  hc.nconf = in + 6 * ns;
  hc.stslot = in + 7 * ns;
  hc.cnt = reinterpret_cast<unsigned*>(base + L.off_cnt);
  hc.partA = reinterpret_cast<double*>(base + L.off_pA);
  hc.partB = reinterpret_cast<double*>(base + L.off_pB);
  hc.nblkA = L.nblkA;
  hc.nblkB = L.nblkB;
  hc.tol = d->tol;
  hc.maxit = d->maxit;
  hc.glist = reinterpret_cast<int*>(base + L.off_glist);
  hc.gmeta = hc.glist + ns;
  hc.partG = reinterpret_cast<double*>(base + L.off_partG);
  hc.cntG = reinterpret_cast<unsigned*>(base + L.off_cntG);
  hc.nchunkG = L.nchunkG;
  hc.rowsG = L.rowsG;
  hc.maxtilesG = L.maxtilesG;
  for (int g = 0; g < RSK_MAX_GROUPS; ++g) {
    hc.grp.W[g] = (defl && g < d->ngroups) ? d->W[g] : nullptr;
    hc.grp.AW[g] = (defl && g < d->ngroups) ? d->AW[g] : nullptr;
    hc.grp.EW[g] = (defl && g < d->ngroups) ? d->EW[g] : nullptr;
    hc.grp.J[g] = (defl && g < d->ngroups) ? d->J[g] : 0;
  }
  hc.grp.ldw = defl ? d->ldw : N;
  int* dlist = reinterpret_cast<int*>(base + L.off_list);
  int* dlist2 = dlist + ns;
  CgDev* dev = reinterpret_cast<CgDev*>(base + L.off_dev);
  double* gb = reinterpret_cast<double*>(base + L.off_gb);

  // ---- ||b||
  RSK_CUDA(launch_batch_dot(h, N, 1, d->b, N, d->b, N, h->scal + 8, st));
  double nb2 = 0.0;
  RSK_CUDA(cudaMemcpyAsync(&nb2, h->scal + 8, sizeof(double), cudaMemcpyDeviceToHost, st));
  RSK_CUDA(cudaStreamSynchronize(st));
  const double nb = std::sqrt(nb2);
  hc.bnorm = nb;
  std::vector<int> hasxp(ns, 0), hasg(ns, 0), grp(ns, 0), mloc(ns, 0), status(ns, ST_ACTIVE), iters(ns, 0);
  std::vector<int64_t> applies(ns, 0);
  for (int s = 0; s < ns; ++s) {
    hasxp[s] = d->has_xp_h ? (d->has_xp_h[s] != 0) : 0;
    hasg[s] = anyg ? (d->has_ghat_h[s] != 0) : 0;
    grp[s] = defl ? d->group_of_shift_h[s] : 0;
  }
  if (nb == 0.0) {
    for (int s = 0; s < ns; ++s) {
      RSK_CUDA(cudaMemsetAsync(d->X + (size_t)s * d->ldx, 0, sizeof(double) * N, st));
      if (d->Gout) RSK_CUDA(cudaMemsetAsync(d->Gout + (size_t)s * d->ldg, 0, sizeof(double) * N, st));
      o->iters[s] = 0; o->applies[s] = 0; o->relres_true[s] = 0.0; o->status[s] = RSK_CG_ZERO_RHS;
      o->m_used[s] = 0;
      if (o->store_count) o->store_count[s] = 0;
    }
    RSK_CUDA(cudaStreamSynchronize(st));
    return RSK_OK;
  }

  // ---- local Grams G_l = sym(U_l^T Z_l) and their Cholesky factors (host)
  std::vector<double> Lf((size_t)ns * kMaxM * kMaxM, 0.0);
  std::vector<int> dropped(ns, 0);
  if (defl) {
    const int G = d->ngroups;
    std::vector<double> WA(G * 256), WE(G * 256), WZg((size_t)G * 16 * ns), AWg((size_t)G * 16 * ns),
        EWg((size_t)G * 16 * ns), gzg(ns);
    for (int g = 0; g < G; ++g) {
      const int J = d->J[g];
      if (J == 0) continue;
      double* o1 = gb + g * 512;
      RSK_CUDA(launch_gemm_tn(h, N, J, d->W[g], d->ldw, J, d->AW[g], d->ldw, o1, J, st));
      RSK_CUDA(launch_gemm_tn(h, N, J, d->W[g], d->ldw, J, d->EW[g], d->ldw, o1 + 256, J, st));
      RSK_CUDA(cudaMemcpyAsync(&WA[g * 256], o1, sizeof(double) * J * J, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaMemcpyAsync(&WE[g * 256], o1 + 256, sizeof(double) * J * J, cudaMemcpyDeviceToHost, st));
      if (anyg) {
        double* o2 = gb + RSK_MAX_GROUPS * 512 + (size_t)g * 48 * ns;
        RSK_CUDA(launch_gemm_tn(h, N, J, d->W[g], d->ldw, ns, d->ZGhat, d->ldgh, o2, J, st));
        RSK_CUDA(launch_gemm_tn(h, N, J, d->AW[g], d->ldw, ns, d->Ghat, d->ldgh, o2 + 16 * ns, J, st));
        RSK_CUDA(launch_gemm_tn(h, N, J, d->EW[g], d->ldw, ns, d->Ghat, d->ldgh, o2 + 32 * ns, J, st));
        RSK_CUDA(cudaMemcpyAsync(&WZg[(size_t)g * 16 * ns], o2, sizeof(double) * J * ns, cudaMemcpyDeviceToHost, st));
        RSK_CUDA(cudaMemcpyAsync(&AWg[(size_t)g * 16 * ns], o2 + 16 * ns, sizeof(double) * J * ns, cudaMemcpyDeviceToHost, st));
        RSK_CUDA(cudaMemcpyAsync(&EWg[(size_t)g * 16 * ns], o2 + 32 * ns, sizeof(double) * J * ns, cudaMemcpyDeviceToHost, st));
      }
    }
    if (anyg) {
      double* o3 = gb + RSK_MAX_GROUPS * (512 + 48 * ns);
      RSK_CUDA(launch_batch_dot(h, N, ns, d->Ghat, d->ldgh, d->ZGhat, d->ldgh, o3, st));
      RSK_CUDA(cudaMemcpyAsync(gzg.data(), o3, sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
    }
    RSK_CUDA(cudaStreamSynchronize(st));
    std::vector<int> Jh(G);
    for (int g = 0; g < G; ++g) Jh[g] = d->J[g];
    rsk_status gs = rsk_local_gram_factors(ns, G, Jh.data(), grp.data(), d->gamma_h, WA.data(), WE.data(),
                                           WZg.data(), AWg.data(), EWg.data(), gzg.data(), Lf.data(),
                                           mloc.data(), hasg.data(), dropped.data());
    if (gs != RSK_OK) { h->err = "rsk_cg_recycled_batch: local Gram factors"; return gs; }
  }

  // ---- upload per-shift state
  {
    std::vector<double> dh((size_t)ns * (5 + kMaxM + kMaxM * kMaxM), 0.0);
    for (int s = 0; s < ns; ++s) dh[s] = d->gamma_h[s];
    std::memcpy(&dh[(size_t)5 * ns + (size_t)ns * kMaxM], Lf.data(), sizeof(double) * Lf.size());
    RSK_CUDA(cudaMemcpyAsync(dbl, dh.data(), sizeof(double) * dh.size(), cudaMemcpyHostToDevice, st));
    std::vector<int> ih((size_t)ns * 8, 0);
    for (int s = 0; s < ns; ++s) {
      ih[s] = ST_ACTIVE;
      ih[2 * ns + s] = mloc[s];
      ih[3 * ns + s] = hasg[s];
      ih[4 * ns + s] = grp[s];
    }
    RSK_CUDA(cudaMemcpyAsync(in, ih.data(), sizeof(int) * ih.size(), cudaMemcpyHostToDevice, st));
    RSK_CUDA(cudaMemsetAsync(hc.cnt, 0, sizeof(unsigned) * ns * 4, st));
    RSK_CUDA(cudaMemsetAsync(hc.cntG, 0, sizeof(unsigned) * RSK_MAX_GROUPS * L.maxtilesG * kTickStride, st));
    RSK_CUDA(cudaMemsetAsync(hc.P, 0, sizeof(double) * (size_t)N * ns, st));
    RSK_CUDA(cudaMemcpyAsync(dev, &hc, sizeof(CgDev), cudaMemcpyHostToDevice, st));
  }
  auto upload_list = [&](int* dl, const std::vector<int>& v) -> cudaError_t {
    if (v.empty()) return cudaSuccess;
    return cudaMemcpyAsync(dl, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice, st);
  };

  // ---- r_p = b - A_g x_p
  std::vector<int> all(ns), withxp;
  for (int s = 0; s < ns; ++s) {
    all[s] = s;
    if (hasxp[s]) withxp.push_back(s);
    else RSK_CUDA(cudaMemsetAsync(d->X + (size_t)s * d->ldx, 0, sizeof(double) * N, st));
  }
  RSK_CUDA(cudaMemsetAsync(hc.Wv, 0, sizeof(double) * (size_t)N * ns, st));
  RSK_CUDA(upload_list(dlist, all));
  if (!withxp.empty()) {
    RSK_CUDA(upload_list(dlist2, withxp));
    ApplyLaunch a{};
    a.X = d->X; a.ldx = d->ldx; a.Y = hc.Wv; a.ldy = N; a.gamma = hc.gam; a.list = dlist2;
    a.nlist = (int)withxp.size(); a.mode = RSK_APPLY_SHIFTED; a.nvec_total = ns;
    RSK_CUDA(launch_apply(h, a, st));
    for (int s : withxp) applies[s] += 1;
  }
  if (d->Gout)
    RSK_CUDA(cudaMemcpy2DAsync(d->Gout, sizeof(double) * d->ldg, d->X, sizeof(double) * d->ldx,
                               sizeof(double) * N, ns, cudaMemcpyDeviceToDevice, st));
  RSK_CUDA(launch_cg_combine(dev, hc, dlist, ns, CMB_RESID, st));
  // ---- Galerkin start on Range(U_l): c = G^-1 U^T r_p, x += U c, r -= Z c
  if (defl) {
    RSK_CUDA(launch_cg_update(dev, hc, dlist, ns, UPD_GALERKIN, st));
    RSK_CUDA(launch_cg_combine(dev, hc, dlist, ns, CMB_GALERKIN, st));
  }
  // ---- rho_0, mu_0; p_0 = r_0 - U mu_0 (combine with alpha = beta = 0)
  RSK_CUDA(launch_cg_update(dev, hc, dlist, ns, UPD_START, st));
  RSK_CUDA(launch_cg_combine(dev, hc, dlist, ns, CMB_LOOP, st));

  // ---- lockstep loop
  std::vector<int> active = all;
  std::vector<int> confirms(ns, 0);
  const int ce = d->check_every;
  std::vector<cudaEvent_t> evs;
  double ms_apply = 0.0, ms_upd = 0.0, ms_cmb = 0.0;
  int64_t n_ka = 0;
  if (prof) {
    evs.assign(4 * ce, nullptr);
    for (auto& e : evs) RSK_CUDA(cudaEventCreate(&e));
  }
  std::vector<int> stat_h(ns), it_h(ns);
  int64_t guard = 0;
  // Persistent device loop (cg_persist.cu): one cooperative launch runs up to
  // kChunkIters lockstep iterations incl. the true-residual confirmations; the host
  // only polls the number of shifts left. Falls back to the host-polled loop below
  // (also used by the per-kernel profiling mode) if the grid cannot be co-scheduled.
  // Small images (working set in L2): one thread-block cluster per shift, no lockstep
  // (cg_cluster.cu). The whole loop incl. confirmations runs in one launch.
  const bool cluster_mode = !prof && getenv("RSK_CG_LEGACY") == nullptr && getenv("RSK_CG_NOCLUSTER") == nullptr &&
                            N <= cluster_max_n() &&
                            // 16-byte vector access to rows of every per-shift / group vector
                            (N % 2 == 0) && (d->ldx % 2 == 0) && (!defl || d->ldw % 2 == 0) &&
                            (!anyg || d->ldgh % 2 == 0) && (!store || d->lds % 2 == 0) &&
                            ((reinterpret_cast<uintptr_t>(d->X) | reinterpret_cast<uintptr_t>(d->b) |
                              reinterpret_cast<uintptr_t>(anyg ? d->Ghat : d->X) |
                              reinterpret_cast<uintptr_t>(anyg ? d->ZGhat : d->X) |
                              reinterpret_cast<uintptr_t>(store ? d->store : d->X)) & 15) == 0;
  // device-loop kernel time (CUDA events on the launching stream) for the roofline
  cudaEvent_t dl0 = nullptr, dl1 = nullptr;
  struct EvGuard {   // the events (and the profiling ones) are released on every exit path
    cudaEvent_t* a; cudaEvent_t* b; std::vector<cudaEvent_t>* v;
    ~EvGuard() {
      if (*a) cudaEventDestroy(*a);
      if (*b) cudaEventDestroy(*b);
      for (auto& e : *v) if (e) cudaEventDestroy(e);
    }
  } evguard{&dl0, &dl1, &evs};
  double dl_kind = 0.0;
  RSK_CUDA(cudaEventCreate(&dl0));
  RSK_CUDA(cudaEventCreate(&dl1));
  std::vector<int> it0(ns, 0);
  RSK_CUDA(cudaMemcpyAsync(it0.data(), hc.iters, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
  RSK_CUDA(cudaStreamSynchronize(st));
  const auto t_setup = std::chrono::steady_clock::now();
  RSK_CUDA(cudaEventRecord(dl0, st));
  if (cluster_mode) {
    unsigned* pbar = reinterpret_cast<unsigned*>(base + L.off_pbar);
    RSK_CUDA(cudaMemsetAsync(pbar, 0, sizeof(unsigned) * 8, st));
    bool ok = false;
    int* dorder = nullptr;
    if (d->order_h) {
      std::vector<int> seen(ns, 0);
      bool perm = true;
      for (int s = 0; s < ns; ++s) {
        const int v = d->order_h[s];
        if (v < 0 || v >= ns || seen[v]) { perm = false; break; }
        seen[v] = 1;
      }
      RSK_ARG(perm, "rsk_cg_recycled_batch: order_h is not a permutation");
      dorder = dlist + 2 * ns;
      RSK_CUDA(cudaMemcpyAsync(dorder, d->order_h, sizeof(int) * ns, cudaMemcpyHostToDevice, st));
    }
    RSK_CUDA(launch_cg_cluster(h, dev, hc, pbar + 6, dorder, reinterpret_cast<double*>(base + L.off_zw), st, &ok));
    if (ok) dl_kind = 1.0;
    if (ok) {
      std::vector<int> ncf(ns, 0);
      RSK_CUDA(cudaMemcpyAsync(stat_h.data(), hc.status, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaMemcpyAsync(ncf.data(), hc.nconf, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaStreamSynchronize(st));
      for (int s = 0; s < ns; ++s) { applies[s] += ncf[s]; confirms[s] += ncf[s]; }
      active.clear();
    }
  }
  // Streaming persistent loop for images beyond L2 (cg_stream.cu; RSK_CG_STREAM=0/1 forces)
  const char* sev = getenv("RSK_CG_STREAM");
  const int sforce = sev ? atoi(sev) : -1;
  if (!active.empty() && !prof && getenv("RSK_CG_LEGACY") == nullptr &&
      (sforce == 1 || (sforce != 0 && N >= kStripMinN))) {
    constexpr int kChunkIters = 512;
    unsigned* pbar = reinterpret_cast<unsigned*>(base + L.off_pbar);
    int* pna = reinterpret_cast<int*>(pbar + 4);
    RSK_CUDA(cudaMemsetAsync(pbar, 0, sizeof(unsigned) * 8, st));
    bool streamed = false;
    int64_t pguard = 0;
    for (;;) {
      bool ok = false;
      RSK_CUDA(cudaMemsetAsync(pbar, 0, sizeof(unsigned), st));   // the counting grid barrier
      RSK_CUDA(launch_cg_stream(h, dev, hc, reinterpret_cast<double*>(base + L.off_sA),
                                reinterpret_cast<double*>(base + L.off_sB), pbar, pna, pna + 1, kChunkIters, st, &ok));
      if (!ok) break;
      streamed = true;
      int hv[2] = {0, 0};
      RSK_CUDA(cudaMemcpyAsync(hv, pna, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaStreamSynchronize(st));
      n_ka += hv[1];
      if (hv[0] == 0) break;
      if (++pguard > (2 * (int64_t)d->maxit + 64) / kChunkIters + 8) {
        h->err = "rsk_cg_recycled_batch: streaming loop guard";
        return RSK_ECUDA;
      }
    }
    if (streamed) {
      dl_kind = 3.0;
      std::vector<int> ncf(ns, 0);
      RSK_CUDA(cudaMemcpyAsync(stat_h.data(), hc.status, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaMemcpyAsync(ncf.data(), hc.nconf, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaStreamSynchronize(st));
      for (int s = 0; s < ns; ++s) { applies[s] += ncf[s]; confirms[s] += ncf[s]; }
      active.clear();
    }
  }
  if (!active.empty() && !prof && getenv("RSK_CG_LEGACY") == nullptr && ns <= persist_max_shift()) {
    constexpr int kChunkIters = 512;
    unsigned* pbar = reinterpret_cast<unsigned*>(base + L.off_pbar);
    int* pna = reinterpret_cast<int*>(pbar + 4);
    double* partP = reinterpret_cast<double*>(base + L.off_partP);
    RSK_CUDA(cudaMemsetAsync(pbar, 0, sizeof(unsigned) * 8, st));
    bool persisted = false;
    int64_t pguard = 0;
    for (;;) {
      bool ok = false;
      RSK_CUDA(launch_cg_persist(h, dev, hc, partP, pbar, pna, pna + 1, L.nchunkP, L.rowsP, kChunkIters, st, &ok));
      if (!ok) break;
      persisted = true;
      int hv[2] = {0, 0};
      RSK_CUDA(cudaMemcpyAsync(hv, pna, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaStreamSynchronize(st));
      n_ka += hv[1];
      if (hv[0] == 0) break;
      if (++pguard > (2 * (int64_t)d->maxit + 64) / kChunkIters + 8) {
        h->err = "rsk_cg_recycled_batch: persistent loop guard";
        return RSK_ECUDA;
      }
    }
    if (persisted) {
      dl_kind = 2.0;
      std::vector<int> ncf(ns, 0);
      RSK_CUDA(cudaMemcpyAsync(stat_h.data(), hc.status, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaMemcpyAsync(ncf.data(), hc.nconf, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaStreamSynchronize(st));
      for (int s = 0; s < ns; ++s) { applies[s] += ncf[s]; confirms[s] += ncf[s]; }
      active.clear();
    }
  }
  const int ngrp = defl ? d->ngroups : 1;
  std::vector<int> gbuf(ns + 16);
  // The lockstep chunk (check_every x {apply, update, combine}) has a static launch
  // shape: list contents and lengths live in device memory, grids are sized for the
  // whole solve (surplus CTAs exit). It is captured once as a CUDA graph and replayed
  // at every poll, so the host issues one launch per chunk.
  // (the per-kernel profiling mode times each launch with events, outside any graph)
  const bool use_graph = getenv("RSK_NO_GRAPH") == nullptr && !prof;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  auto enqueue_chunk = [&](int na_host) -> cudaError_t {
    for (int i = 0; i < ce; ++i) {
      cudaError_t e;
      if (prof && (e = cudaEventRecord(evs[4 * i], st)) != cudaSuccess) return e;
      ApplyLaunch a{};
      a.X = hc.P; a.ldx = N; a.Y = hc.Wv; a.ldy = N; a.gamma = hc.gam; a.list = hc.glist;
      a.nlist = use_graph ? ns : na_host; a.nvec_total = ns;
      a.nlist_dev = use_graph ? hc.gmeta + 8 : nullptr;
      a.mode = RSK_APPLY_SHIFTED; a.cg = dev; a.cg_alpha = true;
      if ((e = launch_apply(h, a, st)) != cudaSuccess) return e;
      if (prof && (e = cudaEventRecord(evs[4 * i + 1], st)) != cudaSuccess) return e;
      if ((e = launch_cg_update_grp(dev, hc, ngrp, L.maxtilesG, st)) != cudaSuccess) return e;
      if (prof && (e = cudaEventRecord(evs[4 * i + 2], st)) != cudaSuccess) return e;
      if ((e = launch_cg_combine_grp(dev, hc, ngrp, L.maxtilesG, st)) != cudaSuccess) return e;
      if (prof && (e = cudaEventRecord(evs[4 * i + 3], st)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  RSK_CUDA(cudaEventRecord(dl1, st));
  RSK_CUDA(cudaEventSynchronize(dl1));
  float dl_ms = 0.0f;
  cudaEventElapsedTime(&dl_ms, dl0, dl1);
  const auto t_loop = std::chrono::steady_clock::now();
  while (!active.empty()) {
    // active shifts grouped by shift group (group-shared kernels), with offsets/counts
    {
      int o2 = 0;
      for (int g = 0; g < ngrp; ++g) {
        int c = 0;
        gbuf[ns + g] = o2;
        for (int s : active)
          if (grp[s] == g) { gbuf[o2 + c] = s; ++c; }
        gbuf[ns + 4 + g] = c;
        o2 += c;
      }
      for (int g = ngrp; g < 4; ++g) { gbuf[ns + g] = o2; gbuf[ns + 4 + g] = 0; }
      gbuf[ns + 8] = o2;
    }
    RSK_CUDA(cudaMemcpyAsync(hc.glist, gbuf.data(), sizeof(int) * (ns + 9), cudaMemcpyHostToDevice, st));
    const int na = (int)active.size();
    n_ka += ce;
    if (use_graph) {
      if (!gexec) {
        RSK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        cudaError_t ce_err = enqueue_chunk(na);
        cudaError_t ee = cudaStreamEndCapture(st, &graph);
        RSK_CUDA(ce_err);
        RSK_CUDA(ee);
        RSK_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
      } else {
        count_launches(3LL * ce);
      }
      RSK_CUDA(cudaGraphLaunch(gexec, st));
    } else {
      RSK_CUDA(enqueue_chunk(na));
    }
    RSK_CUDA(cudaMemcpyAsync(stat_h.data(), hc.status, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
    RSK_CUDA(cudaStreamSynchronize(st));
    if (prof) {
      for (int i = 0; i < ce; ++i) {
        float t1 = 0, t2 = 0;
        float t3 = 0;
        cudaEventElapsedTime(&t1, evs[4 * i], evs[4 * i + 1]);
        cudaEventElapsedTime(&t2, evs[4 * i + 1], evs[4 * i + 2]);
        cudaEventElapsedTime(&t3, evs[4 * i + 2], evs[4 * i + 3]);
        ms_apply += t1;
        ms_upd += t2;
        ms_cmb += t3;
      }
    }
    // confirm the shifts whose recursive residual converged
    std::vector<int> conf;
    for (int s : active)
      if (stat_h[s] == ST_RCONV) conf.push_back(s);
    if (!conf.empty()) {
      RSK_CUDA(upload_list(dlist2, conf));
      ApplyLaunch a{};
      a.X = d->X; a.ldx = d->ldx; a.Y = hc.Wv; a.ldy = N; a.gamma = hc.gam; a.list = dlist2;
      a.nlist = (int)conf.size(); a.mode = RSK_APPLY_SHIFTED; a.nvec_total = ns;
      RSK_CUDA(launch_apply(h, a, st));
      RSK_CUDA(launch_cg_combine(dev, hc, dlist2, (int)conf.size(), CMB_RESID, st));
      RSK_CUDA(launch_cg_update(dev, hc, dlist2, (int)conf.size(), UPD_CONFIRM, st));
      RSK_CUDA(launch_cg_combine(dev, hc, dlist2, (int)conf.size(), CMB_LOOP, st));
      for (int s : conf) { applies[s] += 1; confirms[s] += 1; }
      RSK_CUDA(cudaMemcpyAsync(stat_h.data(), hc.status, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
      RSK_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<int> next;
    for (int s : active)
      if (stat_h[s] == ST_ACTIVE) next.push_back(s);
    active.swap(next);
    if (++guard > (int64_t)d->maxit * 4 + 100) { h->err = "rsk_cg_recycled_batch: loop guard"; return RSK_ECUDA; }
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  if (graph) cudaGraphDestroy(graph);

  // ---- final true residual for shifts that stopped without a confirm (MAXIT / BREAKDOWN)
  std::vector<double> rt(ns, 0.0);
  RSK_CUDA(cudaMemcpyAsync(rt.data(), hc.rho_true, sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
  RSK_CUDA(cudaMemcpyAsync(it_h.data(), hc.iters, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
  std::vector<int> sc(ns, 0);
  if (store) RSK_CUDA(cudaMemcpyAsync(sc.data(), hc.store_cnt, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
  RSK_CUDA(cudaStreamSynchronize(st));
  std::vector<int> unconf;
  for (int s = 0; s < ns; ++s)
    if (stat_h[s] != ST_DONE) unconf.push_back(s);
  if (!unconf.empty()) {
    RSK_CUDA(upload_list(dlist2, unconf));
    ApplyLaunch a{};
    a.X = d->X; a.ldx = d->ldx; a.Y = hc.Wv; a.ldy = N; a.gamma = hc.gam; a.list = dlist2;
    a.nlist = (int)unconf.size(); a.mode = RSK_APPLY_SHIFTED; a.nvec_total = ns;
    RSK_CUDA(launch_apply(h, a, st));
    RSK_CUDA(launch_cg_combine(dev, hc, dlist2, (int)unconf.size(), CMB_RESID, st));
    double* dd = h->aux + 2 * 256 * 256 + 4096;
    RSK_CUDA(launch_batch_dot(h, N, ns, hc.R, N, hc.R, N, dd, st));
    std::vector<double> rr(ns);
    RSK_CUDA(cudaMemcpyAsync(rr.data(), dd, sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
    RSK_CUDA(cudaStreamSynchronize(st));
    for (int s : unconf) rt[s] = rr[s];
  }
  if (d->Gout) {
    std::vector<double> one(ns, 1.0), mone(ns, -1.0);
    rsk_status s2 = rsk_batch_axpby(h, N, ns, one.data(), d->X, d->ldx, mone.data(), d->Gout, d->ldg, (void*)st);
    if (s2 != RSK_OK) return s2;
  }
  bool all_ok = true;
  for (int s = 0; s < ns; ++s) {
    int stt;
    switch (stat_h[s]) {
      case ST_DONE: stt = dropped[s] ? RSK_CG_DEFL_DROPPED : RSK_CG_CONVERGED; break;
      case ST_BREAKDOWN: stt = RSK_CG_BREAKDOWN; break;
      default: stt = RSK_CG_MAXIT; break;
    }
    if (stt != RSK_CG_CONVERGED && stt != RSK_CG_DEFL_DROPPED) all_ok = false;
    o->status[s] = stt;
    o->iters[s] = it_h[s];
    o->applies[s] = applies[s] + it_h[s];
    o->relres_true[s] = std::sqrt(std::max(rt[s], 0.0)) / nb;
    o->m_used[s] = mloc[s];
    if (o->store_count) o->store_count[s] = store ? sc[s] : 0;
  }
  int64_t tot_it = 0, tot_ap = 0;
  for (int s = 0; s < ns; ++s) { tot_it += it_h[s]; tot_ap += o->applies[s]; }
  if (getenv("RSK_CG_TIMING")) {
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto t_end = std::chrono::steady_clock::now();
    fprintf(stderr, "[rsk_cg] ns=%d drain %.2f setup %.2f loop %.2f (device %.2f) finish %.2f ms\n", ns,
            ms(t_enter, t_drained), ms(t_drained, t_setup), ms(t_setup, t_loop), dl_ms, ms(t_loop, t_end));
  }
  h->nA += tot_ap;
  h->nE += tot_ap;
  if (o->ms_loop && !prof) {
    for (int i = 0; i < 5; ++i) o->ms_loop[i] = 0.0;
    o->ms_loop[2] = (double)n_ka;   // lockstep iterations of the device loop (launches: ceil(/512))
  }
  if (o->ms_loop) {
    int64_t dits = 0;
    for (int s = 0; s < ns; ++s) dits += (int64_t)(it_h[s] - it0[s]) + confirms[s];
    o->ms_loop[5] = dl_kind > 0 ? dl_ms : 0.0;
    o->ms_loop[6] = dl_kind > 0 ? (double)dits : 0.0;
    o->ms_loop[7] = dl_kind;
  }
  if (prof) {
    o->ms_loop[0] = ms_apply;
    o->ms_loop[1] = ms_upd;
    o->ms_loop[2] = (double)n_ka;
    o->ms_loop[3] = (double)tot_it * (double)N;
    o->ms_loop[4] = ms_cmb;
  }
  RSK_CUDA(cudaStreamSynchronize(st));
  return all_ok ? RSK_OK : RSK_EPARTIAL;
}
