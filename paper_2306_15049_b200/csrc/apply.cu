// Fused matrix-free shifted operator  Y_s = A X_s + gamma_s E_k X_s  (PAPER.md eq:shift
// P:361-365; A = C^T C P:137, E_k = L^T W_k L P:147 with the IRN weights of north_star).
//
// B200 design:
//  * C is a zero-boundary "same" convolution with a rank-1 PSF h = u v^T, so
//    A = (Gy^T Gy) (x) (Gx^T Gx) = By (x) Bx with banded By, Bx of half-bandwidth 2r.
//    A X = By X Bx: two 1-D passes of 4r+1 taps (x-pass, then y-pass). Interior
//    rows of B are the autocorrelation of the 1-D factor (kernel-parameter taps ->
//    constant-bank operands); only the 2r rows next to each image edge carry the
//    zero-BC truncation and read a per-handle table, decided per register run.
//  * Tile = (64 - 4r) output rows x 64 columns, so the staged halo tile is always
//    64 rows x (64 + 4r) columns: every thread keeps one fixed row (x-pass) and one
//    fixed column (y-pass) for the whole kernel -- no per-item index arithmetic.
//  * Persistent CTAs walk (shift, tile) work items, shift-major. The halo tile of
//    the NEXT item is fetched with cp.async (8-byte copies, src-size 0 outside the
//    image = the zero boundary) into the other of two shared buffers while the
//    current item computes. The shared tile has an odd pitch, so x-pass lanes
//    (one row each, sliding a VX-wide register window along it) and y-pass lanes
//    (one column each, sliding a VY-tall window down it) are conflict-free. FMAs
//    run tap-outer / output-inner: VX (VY) independent chains per thread.
//  * Epilogue fuses the 5-point weighted E_k stencil (halo 1 of the same tile; the
//    weight loads are issued before the y-pass FMAs), the gamma combine, the split
//    output and the X.Y dot partial.
//  * CG mode: shift ids come from the active list, items of non-ACTIVE shifts are
//    skipped, and the CTA that finishes the last tile of a shift (atomic ticket,
//    fixed-order sum of the per-tile partials) forms pi = p.w and alpha = rho / pi.
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
  double* part;     // [list index][ntiles] (plain mode)
  CgDev* cg;
  int ny, nx, tiles_x, ntiles, nlist;
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

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__host__ __device__ constexpr int apply_tile_rows(int r) { return 64 - 4 * r; }

template <int R>
struct ApplyCfg {
  static constexpr int H = 2 * R;           // halo of A (E needs 1 <= H)
  static constexpr int T = 4 * R + 1;       // taps of B
  static constexpr int TY = apply_tile_rows(R);
  static constexpr int HY = 64;             // staged rows = TY + 2H
  static constexpr int WX = kTX + 2 * H;    // staged cols
  static constexpr int PX = WX | 1;         // odd pitch: conflict-free column walks
  static constexpr int PT = kTX + 1;        // odd pitch of the intermediate
  static constexpr int VX = (R <= 5) ? 8 : 4;
  static constexpr int RUNX = kTX / VX;     // 8 or 16 runs per row
  static constexpr int XI = RUNX / 4;       // x-pass runs per thread (256 threads = 64 rows x 4)
  static constexpr int VY = TY / 4;         // 4 runs per column, 64 columns = 256 threads
  static constexpr int SBUF = HY * PX;
  static constexpr int LD = HY * WX;        // staged elements per item
  static constexpr size_t SMEM = sizeof(double) * (size_t)(2 * SBUF + HY * PT + 32);
  static_assert(TY >= 4 && TY % 4 == 0, "tile rows");
};

template <int R>
__global__ void __launch_bounds__(kNT, 1) apply_kernel(const __grid_constant__ ApplyParams p) {
  using C = ApplyCfg<R>;
  extern __shared__ double smem[];
  double* Tm = smem + 2 * C::SBUF;                 // HY x PT  x-pass output
  double* red = Tm + C::HY * C::PT;                // reduction scratch
  __shared__ int s_last;

  const int ny = p.ny, nx = p.nx;
  const int nitems = p.nlist * p.ntiles;
  const bool cgmode = p.cg && p.cg_alpha;
  const int tid = threadIdx.x;
  // fixed roles: x-pass row xr and runs xrun0 + 4k; y-pass column yc and run yrun
  const int xr = tid & 63, xrun0 = tid >> 6;
  const int yc = tid & 63, yrun = tid >> 6;
  // staging: element idx = tid + k*256 -> (row, col) advanced incrementally
  const int st_r0 = tid / C::WX, st_c0 = tid - (tid / C::WX) * C::WX;
  constexpr int STEP_R = kNT / C::WX, STEP_C = kNT - (kNT / C::WX) * C::WX;

  auto next_item = [&](int it) -> int {
    if (!cgmode) return it;
    while (it < nitems && p.cg->status[p.list[it / p.ntiles]] != ST_ACTIVE) it += gridDim.x;
    return it < nitems ? it : nitems;
  };
  auto issue = [&](int it, double* S) {
    const int li = it / p.ntiles, tile = it - li * p.ntiles;
    const int s = p.list ? p.list[li] : li;
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int gr0 = tyi * C::TY - C::H, gc0 = txi * kTX - C::H;
    const double* xs = p.X + (int64_t)s * p.ldx;
    const bool inside = gr0 >= 0 && gr0 + C::HY <= ny && gc0 >= 0 && gc0 + C::WX <= nx;
    int rr = st_r0, cc = st_c0;
    if (inside) {
      const double* base = xs + (int64_t)gr0 * nx + gc0;
      for (int idx = tid; idx < C::LD; idx += kNT) {
        cp_async8(S + rr * C::PX + cc, base + (int64_t)rr * nx + cc, true);
        rr += STEP_R; cc += STEP_C;
        if (cc >= C::WX) { cc -= C::WX; ++rr; }
      }
    } else {
      for (int idx = tid; idx < C::LD; idx += kNT) {
        const int gi = gr0 + rr, gj = gc0 + cc;
        const bool v = (gi >= 0) && (gi < ny) && (gj >= 0) && (gj < nx);
        cp_async8(S + rr * C::PX + cc, v ? xs + (int64_t)gi * nx + gj : xs, v);
        rr += STEP_R; cc += STEP_C;
        if (cc >= C::WX) { cc -= C::WX; ++rr; }
      }
    }
    cp_async_commit();
  };

  const int mode = p.mode;
  const bool withE = (mode == RSK_APPLY_SHIFTED || mode == RSK_APPLY_SPLIT);
  int it = next_item(blockIdx.x);
  if (it < nitems) issue(it, smem);
  int stage = 0;
  while (it < nitems) {
    const int nxt = next_item(it + gridDim.x);
    __syncthreads();                       // everyone is done with buffer stage ^ 1
    if (nxt < nitems) issue(nxt, smem + (stage ^ 1) * C::SBUF); else cp_async_commit();
    cp_async_wait1();                      // the current item's tile has landed
    __syncthreads();
    const double* S = smem + stage * C::SBUF;
    const int li = it / p.ntiles, tile = it - li * p.ntiles;
    const int s = p.list ? p.list[li] : li;
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int r0 = tyi * C::TY, c0 = txi * kTX;

    // ---- x-pass: Tm[rr][c] = sum_t Bx[c0+c][t] S[rr][c+t]   (row xr, runs xrun0 + 4k)
#pragma unroll
    for (int k = 0; k < C::XI; ++k) {
      const int run = xrun0 + 4 * k;
      const int cb = c0 + run * C::VX;
      const bool xin = !p.use_tab || (cb >= C::H && cb + C::VX <= nx - C::H);
      const double* srow = S + xr * C::PX + run * C::VX;
      double win[C::VX + C::T - 1];
#pragma unroll
      for (int t = 0; t < C::VX + C::T - 1; ++t) win[t] = srow[t];
      double acc[C::VX];
#pragma unroll
      for (int v = 0; v < C::VX; ++v) acc[v] = 0.0;
      if (xin) {
#pragma unroll
        for (int t = 0; t < C::T; ++t) {
          const double c = p.cx[t];
#pragma unroll
          for (int v = 0; v < C::VX; ++v) acc[v] = fma(c, win[v + t], acc[v]);
        }
      } else {
#pragma unroll
        for (int v = 0; v < C::VX; ++v) {
          int gc = cb + v;
          gc = gc < nx ? gc : nx - 1;
          const double* tb = p.tabx + (int64_t)gc * C::T;
#pragma unroll
          for (int t = 0; t < C::T; ++t) acc[v] = fma(__ldg(tb + t), win[v + t], acc[v]);
        }
      }
#pragma unroll
      for (int v = 0; v < C::VX; ++v) Tm[xr * C::PT + run * C::VX + v] = acc[v];
    }
    __syncthreads();

    // ---- y-pass + fused epilogue (column yc, rows o0 .. o0 + VY - 1)
    const int o0 = yrun * C::VY;
    const int gj = c0 + yc;
    const int rb = r0 + o0;
    double* __restrict__ ys = p.Y + (int64_t)s * p.ldy;
    // issue the weight loads of the epilogue early (they do not depend on the tile)
    double wxl[C::VY], wxr[C::VY], wyu[C::VY], wyd[C::VY];
    if (withE) {
#pragma unroll
      for (int v = 0; v < C::VY; ++v) {
        const int gi = rb + v;
        const bool in = gi < ny && gj < nx;
        const int64_t pix = (int64_t)(in ? gi : 0) * nx + (in ? gj : 0);
        wxr[v] = in ? __ldg(p.wx + pix) : 0.0;
        wyd[v] = in ? __ldg(p.wy + pix) : 0.0;
        wxl[v] = (in && gj > 0) ? __ldg(p.wx + pix - 1) : 0.0;
        wyu[v] = (in && gi > 0) ? __ldg(p.wy + pix - nx) : 0.0;
      }
    }
    const double g = (mode == RSK_APPLY_SHIFTED) ? __ldg(p.gamma + s) : 0.0;
    double win[C::VY + C::T - 1];
#pragma unroll
    for (int t = 0; t < C::VY + C::T - 1; ++t) win[t] = Tm[(o0 + t) * C::PT + yc];
    double acc[C::VY];
#pragma unroll
    for (int v = 0; v < C::VY; ++v) acc[v] = 0.0;
    const bool yin = !p.use_tab || (rb >= C::H && rb + C::VY <= ny - C::H);
    if (yin) {
#pragma unroll
      for (int t = 0; t < C::T; ++t) {
        const double c = p.cy[t];
#pragma unroll
        for (int v = 0; v < C::VY; ++v) acc[v] = fma(c, win[v + t], acc[v]);
      }
    } else {
#pragma unroll
      for (int v = 0; v < C::VY; ++v) {
        int gr = rb + v;
        gr = gr < ny ? gr : ny - 1;
        const double* tb = p.taby + (int64_t)gr * C::T;
#pragma unroll
        for (int t = 0; t < C::T; ++t) acc[v] = fma(__ldg(tb + t), win[v + t], acc[v]);
      }
    }
    double dot = 0.0;
    double* __restrict__ eys = (mode == RSK_APPLY_SPLIT) ? p.EY + (int64_t)s * p.ldey : nullptr;
#pragma unroll
    for (int v = 0; v < C::VY; ++v) {
      const int gi = rb + v;
      if (gi < ny && gj < nx) {
        const int so = (o0 + v + C::H) * C::PX + yc + C::H;
        const double xc = S[so];
        double out = acc[v];
        const int64_t pix = (int64_t)gi * nx + gj;
        if (withE) {
          const double ex = wxl[v] * (xc - S[so - 1]) - wxr[v] * (S[so + 1] - xc) +
                            wyu[v] * (xc - S[so - C::PX]) - wyd[v] * (S[so + C::PX] - xc);
          if (mode == RSK_APPLY_SHIFTED) out = fma(g, ex, out);
          else eys[pix] = ex;
        }
        ys[pix] = out;
        dot = fma(xc, out, dot);
      }
    }

    if (p.want_dot) {
      const double bs = block_sum(dot, red);
      if (!p.cg) {
        if (tid == 0) p.part[(int64_t)li * p.ntiles + tile] = bs;
      } else {
        CgDev* cg = p.cg;
        if (tid == 0) {
          cg->partA[(int64_t)s * cg->nblkA + tile] = bs;
          __threadfence();
          const unsigned tk = atomicAdd(cg->cnt + 4 * s + 0, 1u);
          s_last = (tk == (unsigned)(p.ntiles - 1));
        }
        __syncthreads();
        if (s_last && tid < 32) {
          __threadfence();
          const double* pa = cg->partA + (int64_t)s * cg->nblkA;
          double t = 0.0;
          for (int j = tid; j < p.ntiles; j += 32) t += __ldcg(pa + j);
          t = warp_sum(t);
          if (tid == 0) {
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
    }
    it = nxt;
    stage ^= 1;
  }
  cp_async_wait0();
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
  const int ty = apply_tile_rows(h->r);
  const int tx = (int)((h->nx + kTX - 1) / kTX), tyc = (int)((h->ny + ty - 1) / ty);
  return tx * tyc;
}

template <int R>
static cudaError_t launch_r(const ApplyParams& prm, int sm_count, cudaStream_t st) {
  using C = ApplyCfg<R>;
  static int blocks_per_sm = 0;
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(apply_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, apply_kernel<R>, kNT, C::SMEM);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int nitems = prm.nlist * prm.ntiles;
  int grid = blocks_per_sm * sm_count;
  if (grid > nitems) grid = nitems;
  count_launch();
  apply_kernel<R><<<grid, kNT, C::SMEM, st>>>(prm);
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
  prm.nlist = a.nlist;
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
  const int smc = h->sm_count;
  switch (h->r) {
    case 1: e = launch_r<1>(prm, smc, st); break;
    case 2: e = launch_r<2>(prm, smc, st); break;
    case 3: e = launch_r<3>(prm, smc, st); break;
    case 4: e = launch_r<4>(prm, smc, st); break;
    case 5: e = launch_r<5>(prm, smc, st); break;
    case 6: e = launch_r<6>(prm, smc, st); break;
    case 7: e = launch_r<7>(prm, smc, st); break;
    case 8: e = launch_r<8>(prm, smc, st); break;
    case 9: e = launch_r<9>(prm, smc, st); break;
    case 10: e = launch_r<10>(prm, smc, st); break;
    case 11: e = launch_r<11>(prm, smc, st); break;
    case 12: e = launch_r<12>(prm, smc, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  if (a.xdoty && !a.cg) {
    count_launch();
    apply_dot_reduce<<<a.nlist, 32, 0, st>>>(h->scratch, prm.ntiles, a.list, a.xdoty);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace rsk
