// Fused matrix-free shifted operator  Y_s = A X_s + gamma_s E_k X_s  (PAPER.md eq:shift
// P:361-365; A = C^T C P:137, E_k = L^T W_k L P:147 with the IRN weights of north_star).
//
// B200 design:
//  * C is a zero-boundary "same" convolution with a rank-1 PSF h = u v^T, so
//    A = (Gy^T Gy) (x) (Gx^T Gx) = By (x) Bx with banded By, Bx of half-bandwidth 2r.
//    A X = By X Bx: two 1-D passes of 4r+1 taps (x-pass, then y-pass). Interior
//    rows of B are the autocorrelation of the 1-D factor (kernel-parameter taps
//    -> constant-bank operands); the 2r rows next to each edge carry the zero-BC
//    truncation and are read from a per-handle table only in edge tiles.
//  * One CTA = one 32x64 output tile of one shift. The (32+4r) x (64+4r) halo tile
//    is staged in shared memory with an odd pitch so that both passes read it
//    conflict-free: x-pass lanes walk down rows (stride = odd pitch), each thread
//    slides a VX-wide register window along its row; y-pass lanes walk along
//    columns and slide a VY-tall register window down the intermediate.
//  * Epilogue fuses the 5-point weighted E_k stencil (needs halo 1 of the same
//    shared tile), the gamma combine, the split output and the X.Y dot partial.
//  * CG mode: the shift id comes from an active list, the CTA exits if its shift
//    is not ACTIVE, and the last CTA of a shift (atomic ticket, fixed-order sum of
//    the per-tile partials) forms pi = p.w and alpha = rho / pi on the device.
#include <cuda_runtime.h>

#include "rsk_internal.h"

namespace rsk {

struct ApplyParams {
  const double* X;
  int64_t ldx;
  double* Y;
  int64_t ldy;
  double* EY;
  int64_t ldey;
  const double* gamma;
  const int* list;
  const double* wx;
  const double* wy;
  const double* tabx;
  const double* taby;
  double* part;     // [list index][ntiles] (plain) or cg->partA[shift][...]
  CgDev* cg;
  int ny, nx, tiles_x, ntiles;
  int mode;
  int use_tab;      // 1: A (B tables at edges), 0: C / C^T (interior taps everywhere)
  int want_dot;
  int cg_alpha;
  double cx[kMaxTaps];
  double cy[kMaxTaps];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block sum (fixed tree), result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

template <int R>
struct ApplyCfg {
  static constexpr int H = 2 * R;           // halo of A (E needs 1 <= H)
  static constexpr int T = 4 * R + 1;       // taps of B
  static constexpr int HY = kTY + 2 * H;    // staged rows
  static constexpr int WX = kTX + 2 * H;    // staged cols
  static constexpr int PX = WX | 1;         // odd pitch: conflict-free column walks
  static constexpr int PT = kTX + 1;        // odd pitch of the intermediate
  static constexpr int VX = (R <= 5) ? 8 : 4;
  static constexpr int VY = (R <= 5) ? 8 : 4;
  static constexpr int RUNX = kTX / VX;
  static constexpr int RUNY = kTY / VY;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(HY * PX + HY * PT) + 64 * sizeof(double);
};

template <int R>
__global__ void __launch_bounds__(kNT) apply_kernel(const __grid_constant__ ApplyParams p) {
  using C = ApplyCfg<R>;
  extern __shared__ double smem[];
  double* S = smem;                 // HY x PX   input tile (with halo H)
  double* Tm = smem + C::HY * C::PX;  // HY x PT  x-pass output
  double* red = Tm + C::HY * C::PT;   // 32 doubles reduction scratch
  __shared__ int s_last;

  const int li = blockIdx.y;
  const int s = p.list ? p.list[li] : li;
  if (p.cg && p.cg_alpha) {
    if (p.cg->status[s] != ST_ACTIVE) return;   // uniform per CTA
  }
  const int tile = blockIdx.x;
  const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
  const int r0 = tyi * kTY, c0 = txi * kTX;
  const int ny = p.ny, nx = p.nx;
  const double* __restrict__ xs = p.X + (int64_t)s * p.ldx;

  // ---- stage the halo tile (zero outside the image = zero boundary condition)
  for (int idx = threadIdx.x; idx < C::HY * C::WX; idx += kNT) {
    const int rr = idx / C::WX, cc = idx - rr * C::WX;
    const int gi = r0 - C::H + rr, gj = c0 - C::H + cc;
    double val = 0.0;
    if (gi >= 0 && gi < ny && gj >= 0 && gj < nx) val = __ldg(xs + (int64_t)gi * nx + gj);
    S[rr * C::PX + cc] = val;
  }
  __syncthreads();

  // ---- x-pass: Tm[rr][c] = sum_t Bx[c0+c][t] S[rr][c+t]
  const bool xin = !p.use_tab || (c0 >= C::H && c0 + kTX <= nx - C::H);
  for (int it = threadIdx.x; it < C::HY * C::RUNX; it += kNT) {
    const int rr = it % C::HY;
    const int run = it / C::HY;
    const double* srow = S + rr * C::PX + run * C::VX;
    double win[C::VX + C::T - 1];
#pragma unroll
    for (int t = 0; t < C::VX + C::T - 1; ++t) win[t] = srow[t];
    double acc[C::VX];
    if (xin) {
#pragma unroll
      for (int v = 0; v < C::VX; ++v) {
        double a = 0.0;
#pragma unroll
        for (int t = 0; t < C::T; ++t) a = fma(p.cx[t], win[v + t], a);
        acc[v] = a;
      }
    } else {
#pragma unroll
      for (int v = 0; v < C::VX; ++v) {
        int gc = c0 + run * C::VX + v;
        gc = gc < nx ? gc : nx - 1;
        const double* tb = p.tabx + (int64_t)gc * C::T;
        double a = 0.0;
#pragma unroll
        for (int t = 0; t < C::T; ++t) a = fma(__ldg(tb + t), win[v + t], a);
        acc[v] = a;
      }
    }
#pragma unroll
    for (int v = 0; v < C::VX; ++v) Tm[rr * C::PT + run * C::VX + v] = acc[v];
  }
  __syncthreads();

  // ---- y-pass + fused epilogue
  const bool yin = !p.use_tab || (r0 >= C::H && r0 + kTY <= ny - C::H);
  const int mode = p.mode;
  const bool withE = (mode == RSK_APPLY_SHIFTED || mode == RSK_APPLY_SPLIT);
  const double g = (mode == RSK_APPLY_SHIFTED) ? __ldg(p.gamma + s) : 0.0;
  double* __restrict__ ys = p.Y + (int64_t)s * p.ldy;
  double* __restrict__ eys = (mode == RSK_APPLY_SPLIT) ? p.EY + (int64_t)s * p.ldey : nullptr;
  double dot = 0.0;
  for (int it = threadIdx.x; it < kTX * C::RUNY; it += kNT) {
    const int cc = it % kTX;
    const int run = it / kTX;
    const int o0 = run * C::VY;
    double win[C::VY + C::T - 1];
#pragma unroll
    for (int t = 0; t < C::VY + C::T - 1; ++t) win[t] = Tm[(o0 + t) * C::PT + cc];
    const int gj = c0 + cc;
#pragma unroll
    for (int v = 0; v < C::VY; ++v) {
      const int o = o0 + v;
      const int gi = r0 + o;
      double a = 0.0;
      if (yin) {
#pragma unroll
        for (int t = 0; t < C::T; ++t) a = fma(p.cy[t], win[v + t], a);
      } else {
        const int gr = gi < ny ? gi : ny - 1;
        const double* tb = p.taby + (int64_t)gr * C::T;
#pragma unroll
        for (int t = 0; t < C::T; ++t) a = fma(__ldg(tb + t), win[v + t], a);
      }
      if (gi < ny && gj < nx) {
        const int so = (o + C::H) * C::PX + cc + C::H;
        const double xc = S[so];
        double out = a;
        if (withE) {
          const int64_t pix = (int64_t)gi * nx + gj;
          const double wxr = __ldg(p.wx + pix);
          const double wyd = __ldg(p.wy + pix);
          const double wxl = gj > 0 ? __ldg(p.wx + pix - 1) : 0.0;
          const double wyu = gi > 0 ? __ldg(p.wy + pix - nx) : 0.0;
          const double ex = wxl * (xc - S[so - 1]) - wxr * (S[so + 1] - xc) +
                            wyu * (xc - S[so - C::PX]) - wyd * (S[so + C::PX] - xc);
          if (mode == RSK_APPLY_SHIFTED) {
            out = fma(g, ex, a);
          } else {
            eys[pix] = ex;
          }
          ys[pix] = out;
        } else {
          ys[(int64_t)gi * nx + gj] = out;
        }
        dot = fma(xc, out, dot);
      }
    }
  }

  if (!p.want_dot) return;
  const double bs = block_sum(dot, red);
  if (!p.cg) {
    if (threadIdx.x == 0) p.part[(int64_t)li * p.ntiles + tile] = bs;
    return;
  }
  // CG: partial -> last CTA of this shift forms pi and alpha
  CgDev* cg = p.cg;
  if (threadIdx.x == 0) {
    cg->partA[(int64_t)s * cg->nblkA + tile] = bs;
    __threadfence();
    const unsigned tk = atomicAdd(cg->cnt + 4 * s + 0, 1u);
    s_last = (tk == (unsigned)(p.ntiles - 1));
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x < 32) {
    __threadfence();
    const double* pa = cg->partA + (int64_t)s * cg->nblkA;
    double t = 0.0;
    for (int j = threadIdx.x; j < p.ntiles; j += 32) t += __ldcg(pa + j);
    t = warp_sum(t);
    if (threadIdx.x == 0) {
      cg->cnt[4 * s + 0] = 0u;
      const double pi = t;
      if (!(pi > 0.0) || !isfinite(pi)) {
        cg->status[s] = ST_BREAKDOWN;
        cg->alpha[s] = 0.0;
      } else {
        cg->alpha[s] = cg->rho[s] / pi;
      }
    }
  }
}

// plain-mode dot reduction: xdoty[s] = sum_tiles part[li][tile]
__global__ void apply_dot_reduce(const double* part, int ntiles, const int* list, double* xdoty) {
  const int li = blockIdx.x;
  const int s = list ? list[li] : li;
  double t = 0.0;
  for (int j = threadIdx.x; j < ntiles; j += 32) t += part[(int64_t)li * ntiles + j];
  t = warp_sum(t);
  if (threadIdx.x == 0) xdoty[s] = t;
}

int apply_tiles(const Handle* h) {
  const int tx = (int)((h->nx + kTX - 1) / kTX), ty = (int)((h->ny + kTY - 1) / kTY);
  return tx * ty;
}

template <int R>
static cudaError_t launch_r(const ApplyParams& prm, int nlist, cudaStream_t st) {
  using C = ApplyCfg<R>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(apply_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(prm.ntiles, nlist);
  count_launch(); apply_kernel<R><<<grid, kNT, C::SMEM, st>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_apply(Handle* h, const ApplyLaunch& a, cudaStream_t st) {
  if (a.nlist <= 0) return cudaSuccess;
  ApplyParams prm;
  prm.X = a.X; prm.ldx = a.ldx;
  prm.Y = a.Y; prm.ldy = a.ldy;
  prm.EY = a.EY; prm.ldey = a.ldey;
  prm.gamma = a.gamma;
  prm.list = a.list;
  prm.wx = h->wx; prm.wy = h->wy;
  prm.tabx = h->tabBx; prm.taby = h->tabBy;
  prm.cg = a.cg;
  prm.ny = (int)h->ny; prm.nx = (int)h->nx;
  prm.tiles_x = (int)((h->nx + kTX - 1) / kTX);
  prm.ntiles = apply_tiles(h);
  prm.mode = a.mode;
  prm.cg_alpha = a.cg_alpha ? 1 : 0;
  prm.want_dot = (a.xdoty != nullptr || a.cg_alpha) ? 1 : 0;
  prm.part = h->scratch;
  const int T = 4 * h->r + 1;
  for (int t = 0; t < kMaxTaps; ++t) { prm.cx[t] = 0.0; prm.cy[t] = 0.0; }
  if (a.mode == RSK_APPLY_C_ONLY) {
    prm.use_tab = 0;
    for (int t = 0; t < T; ++t) { prm.cx[t] = h->cCx[t]; prm.cy[t] = h->cCy[t]; }
  } else if (a.mode == RSK_APPLY_CT_ONLY) {
    prm.use_tab = 0;
    for (int t = 0; t < T; ++t) { prm.cx[t] = h->cTx[t]; prm.cy[t] = h->cTy[t]; }
  } else {
    prm.use_tab = 1;
    for (int t = 0; t < T; ++t) { prm.cx[t] = h->cBx[t]; prm.cy[t] = h->cBy[t]; }
  }
  if (a.xdoty && !a.cg) {
    const size_t need = sizeof(double) * (size_t)prm.ntiles * (size_t)a.nlist;
    if (need > h->scratch_bytes) return cudaErrorMemoryAllocation;
  }
  cudaError_t e;
  switch (h->r) {
    case 1: e = launch_r<1>(prm, a.nlist, st); break;
    case 2: e = launch_r<2>(prm, a.nlist, st); break;
    case 3: e = launch_r<3>(prm, a.nlist, st); break;
    case 4: e = launch_r<4>(prm, a.nlist, st); break;
    case 5: e = launch_r<5>(prm, a.nlist, st); break;
    case 6: e = launch_r<6>(prm, a.nlist, st); break;
    case 7: e = launch_r<7>(prm, a.nlist, st); break;
    case 8: e = launch_r<8>(prm, a.nlist, st); break;
    case 9: e = launch_r<9>(prm, a.nlist, st); break;
    case 10: e = launch_r<10>(prm, a.nlist, st); break;
    case 11: e = launch_r<11>(prm, a.nlist, st); break;
    case 12: e = launch_r<12>(prm, a.nlist, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  if (a.xdoty && !a.cg) {
    count_launch(); apply_dot_reduce<<<a.nlist, 32, 0, st>>>(h->scratch, prm.ntiles, a.list, a.xdoty);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace rsk
