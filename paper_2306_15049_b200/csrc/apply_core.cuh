// Fused matrix-free shifted operator  Y_s = A X_s + gamma_s E_k X_s  (PAPER.md eq:shift
// P:361-365; A = C^T C P:137, E_k = L^T W_k L P:147 with the IRN weights of north_star).
// Work-item core shared by the standalone apply kernel (apply.cu) and phase A of the
// persistent CG kernel (cg_persist.cu).  DESIGN.md §4.1.
//
//  * C is a zero-boundary "same" convolution with a rank-1 PSF h = u v^T, so
//    A = (Gy^T Gy) (x) (Gx^T Gx) = By (x) Bx with banded By, Bx of half-bandwidth 2r:
//    A X = By X Bx, two banded passes of 4r+1 taps.
//  * Both passes run on the FP64 tensor cores (mma.sync.m8n8k4.f64 -> DMMA): an 8x8
//    output block of the x-pass is  S[8 rows][cb .. cb+8+4r) x Toeplitz(Bx)[(8+4r) x 8]
//    (r+2 DMMA k-steps); the y-pass is Toeplitz(By) x T[(8+4r) x 8]. Interior blocks take
//    the Toeplitz fragments from registers; blocks within 2r of an image edge (where the
//    zero boundary truncates B) take them from a fragment-ordered table (coalesced LDG).
//  * Work item = (tile, shift); tile = TY x 64 outputs; the halo tile HY x PX (HY =
//    roundup8(TY + 4r), PX = 64 + 4r padded to 4 mod 8 doubles: conflict-free A-fragment
//    loads) is fetched by ONE TMA box load (3-D map {nx, ny, vector}); out-of-image
//    elements arrive as zeros = the zero boundary. W_k tiles likewise (2-D maps), once per
//    tile for all shifts of it. Odd widths (no 16-byte row pitch) use cp.async instead.
//  * Double-buffered: the next item's box is in flight while the current one computes.
//  * Epilogue fuses the 5-point weighted E_k stencil, the gamma combine, the split output
//    and the X.Y dot; in CG mode the last CTA of a shift (ticket, fixed-order sum of the
//    per-tile partials) forms pi = p.w and alpha = rho / pi.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "rsk_internal.h"
#include "tma.cuh"

namespace rsk {

struct alignas(64) ApplyParams {
  CUtensorMap mapX;   // 3-D {nx, ny, vectors} over X (TMA path)
  CUtensorMap mapX2;  // second source (CG confirm: the iterate x), same geometry
  const double* X;
  int64_t ldx;
  const double* X2;
  int64_t ldx2;
  double* Y;
  int64_t ldy;
  double* EY;
  int64_t ldey;
  const double* gamma;
  const int* list;
  const double* wx;
  const double* wy;
  const double* fragx;  // [col block][KS][32] B_x fragments (A mode)
  const double* fragy;  // [row block][KS][32] B_y fragments (A mode)
  double* part;         // [list index][ntiles] (plain mode dot partials)
  CgDev* cg;
  int ny, nx, tiles_x, ntiles, nlist;
  const int* nlist_dev;  // if set, the list length is read on the device
  int mode;
  int use_tab;   // 1: A (edge fragments from tables), 0: C / C^T (interior taps everywhere)
  int want_dot;
  int cg_alpha;
  int src2_rconv;  // CG: items whose shift status is ST_RCONV read X2 (true-residual confirm)
  int bx_lo, bx_hi, by_lo, by_hi;  // interior 8-column / 8-row block ranges (inclusive)
  double cx[kMaxTaps];
  double cy[kMaxTaps];
};

// TY = 64 - 4r rounded down to 8 rows, so the staged halo is HY = 64 rows = 8 x-pass row
// blocks x 2 halves = 16 work units: one per warp (balanced x-pass)
__host__ __device__ constexpr int tc_tile_rows(int r) {
  return (8 * ((64 - 4 * r) / 8) > 56) ? 56 : 8 * ((64 - 4 * r) / 8);
}
__host__ __device__ constexpr int pad4mod8(int w) { return w + ((4 - (w & 7)) & 7); }
__host__ __device__ constexpr int al16(int n) { return (n + 15) & ~15; }  // 128-byte multiples

constexpr int kAT = 256;   // threads per apply CTA (8 warps); 2 CTAs per SM
constexpr int kApplyCtasPerSm = 2;

template <int R>
struct TcCfg {
  static constexpr int H = 2 * R;            // halo of A (E needs 1 <= H)
  static constexpr int T = 4 * R + 1;        // taps of B
  static constexpr int KS = R + 2;           // DMMA k-steps per 8x8 block: (8 + 4r) / 4
  static constexpr int TY = tc_tile_rows(R); // output rows per tile (multiple of 8)
  static constexpr int HY = ((TY + 4 * R + 7) / 8) * 8;  // staged rows (64)
  static constexpr int RBX = HY / 8;         // x-pass row blocks
  static constexpr int RBY = TY / 8;         // y-pass row blocks (one warp: all of them)
  static constexpr int WX = kTX + 4 * R;     // staged cols used
  static constexpr int PX = pad4mod8(WX);    // staged pitch = TMA box width
  static constexpr int PT = 72;              // x-pass output pitch (= 8 mod 16)
  static constexpr int KU = 8 + R;           // x-pass A-fragment window (32 + 4r columns)
  static constexpr int KUY = 2 * RBY + R;    // y-pass B-fragment window (8 RBY + 4r rows)
  static constexpr int SBUF = al16(HY * PX);
  static constexpr int TBUF = al16(HY * PT);
  static constexpr int OFF_T = SBUF;
  static constexpr int OFF_RED = OFF_T + TBUF;
  static constexpr int OFF_BAR = OFF_RED + 16;        // 1 mbarrier (8 B)
  static constexpr int DBL = OFF_BAR + 2;
  static constexpr size_t SMEM = sizeof(double) * (size_t)DBL;
  static constexpr unsigned XBYTES = 8u * HY * PX;
  static_assert(TY >= 8 && TY % 8 == 0, "tile rows");
  static_assert(HY <= 64, "staged rows");
  static_assert(2 * RBX == 2 * (kAT / 32), "x-pass: two units per warp");
  static_assert(PX <= 256, "TMA box width");
  static_assert(kApplyCtasPerSm * (SMEM + 1024) <= 227 * 1024, "shared memory");
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

// D(8x8) += A(8x4, row) * B(4x8, col) in fp64 on the tensor cores. Fragments (per lane,
// g = lane / 4, q = lane % 4): a = A[g][q], b = B[q][g], d = {D[g][2q], D[g][2q+1]}.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p));
}

// mbarrier use counter (parity of the next wait); every thread runs the same sequence
struct ApplyPipe {
  unsigned use;
};

template <int R, bool kTma>
struct ApplyCore {
  using C = TcCfg<R>;

  __device__ static void init_bars(double* smem) {
    if (kTma && threadIdx.x == 0) {
      mbar_init(reinterpret_cast<uint64_t*>(smem + C::OFF_BAR), 1);
      mbar_fence_init();
    }
    __syncthreads();
  }

  // stage the halo tile of (tile, shift s)
  __device__ static void issue_x(const ApplyParams& p, double* smem, int tile, int s, bool src2) {
    double* S = smem;
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int gr0 = tyi * C::TY - C::H, gc0 = txi * kTX - C::H;
    if (kTma) {
      if (threadIdx.x == 0) {
        uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
        mbar_expect_tx(bar, C::XBYTES);
        tma_load_3d(S, src2 ? &p.mapX2 : &p.mapX, bar, gc0, gr0, s);
      }
    } else {
      const double* xs = src2 ? p.X2 + (int64_t)s * p.ldx2 : p.X + (int64_t)s * p.ldx;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      for (int rr = warp; rr < C::HY; rr += kAT / 32) {
        const int gi = gr0 + rr;
        const bool rv = (gi >= 0) && (gi < p.ny);
        const double* xrow = xs + (int64_t)gi * p.nx;
        for (int cc = lane; cc < C::WX; cc += 32) {
          const int gj = gc0 + cc;
          const bool v = rv && (gj >= 0) && (gj < p.nx);
          cp_async8(S + rr * C::PX + cc, v ? xrow + gj : xs, v);
        }
      }
      cp_async_commit();
    }
  }

  // pull the weight tile of `tile` (rows r0-1 .. r0+TY, cols c0-1 .. c0+64) into L1
  __device__ static void prefetch_w(const ApplyParams& p, int tile) {
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int r0 = tyi * C::TY, c0 = txi * kTX;
    constexpr int LPR = 5;                       // 128-byte lines per 66-double row segment
    constexpr int NL = 2 * (C::TY + 1) * LPR;    // both planes
    for (int e = threadIdx.x; e < NL; e += kAT) {
      const int pl = e / ((C::TY + 1) * LPR);
      const int rem = e - pl * ((C::TY + 1) * LPR);
      const int rr = rem / LPR, ln = rem - rr * LPR;
      const int gi = r0 - 1 + rr;
      const int gj = min(max(c0 - 1 + 16 * ln, 0), p.nx - 1);
      if (gi >= 0 && gi < p.ny) prefetch_l1((pl ? p.wy : p.wx) + (int64_t)gi * p.nx + gj);
    }
  }

  // Process work items [ibeg, iend) of the tile-major item space item = tile * nl + li.
  __device__ static void run(const ApplyParams& p, double* smem, int ibeg, int iend, int nl, ApplyPipe& pp) {
    const double* S = smem;
    double* Tm = smem + C::OFF_T;
    double* red = smem + C::OFF_RED;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    __shared__ int s_last;

    const int ny = p.ny, nx = p.nx;
    const bool cgmode = p.cg && p.cg_alpha;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int mode = p.mode;
    const bool withE = (mode == RSK_APPLY_SHIFTED || mode == RSK_APPLY_SPLIT);
    if (ibeg >= iend) return;
    // interior Toeplitz fragments: x-pass B[k][n] = cx[k - n], y-pass A[m][k] = cy[k - m]
    double bx[C::KS], ay[C::KS];
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks) {
      const int t = 4 * ks + q - g;
      bx[ks] = (t >= 0 && t < C::T) ? p.cx[t] : 0.0;
      ay[ks] = (t >= 0 && t < C::T) ? p.cy[t] : 0.0;
    }
    auto sid_of = [&](int li) -> int { return p.list ? p.list[li] : li; };
    auto src2_of = [&](int s) -> bool { return p.src2_rconv && p.cg->status[s] == ST_RCONV; };

    int wtile = -1;
    {
      const int tile = ibeg / nl, s = sid_of(ibeg - tile * nl);
      issue_x(p, smem, tile, s, src2_of(s));
    }
    for (int it = ibeg; it < iend; ++it) {
      const int tile = it / nl, li = it - tile * nl;
      const int s = sid_of(li);
      const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
      const int r0 = tyi * C::TY, c0 = txi * kTX;
      if (withE && tile != wtile) {
        prefetch_w(p, tile);
        wtile = tile;
      }
      if (kTma) {
        mbar_wait(bar, pp.use & 1);
        pp.use += 1;
      } else {
        cp_async_wait0();
        __syncthreads();
      }

      // ---- x-pass on the tensor cores: T[rb-rows][cols] = S[rb-rows][cols .. cols+8+4r) x Bx.
      // Work unit = (row block rb, half): 4 adjacent 8-column blocks share one window of
      // A fragments (32 + 4r columns = 8 + r k-steps), block c uses window steps 2c .. 2c+r+1.
#pragma unroll 1
      for (int u = warp; u < 2 * C::RBX; u += kAT / 32) {
        const int rb = u >> 1, half = u & 1;
        const int cl0 = half * 32;
        double a[C::KU];
        const double* sa = S + (rb * 8 + g) * C::PX + cl0 + q;
#pragma unroll
        for (int k = 0; k < C::KU; ++k) a[k] = sa[4 * k];
        double d0[4], d1[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) { d0[c] = 0.0; d1[c] = 0.0; }
        const int blk0 = (c0 + cl0) >> 3;
        if (!p.use_tab || (blk0 >= p.bx_lo && blk0 + 3 <= p.bx_hi)) {
#pragma unroll
          for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
            for (int c = 0; c < 4; ++c) dmma(d0[c], d1[c], a[2 * c + ks], bx[ks]);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double* fb = p.fragx + (int64_t)(blk0 + c) * (C::KS * 32) + lane;
#pragma unroll
            for (int ks = 0; ks < C::KS; ++ks) dmma(d0[c], d1[c], a[2 * c + ks], __ldg(fb + ks * 32));
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double2* tp = reinterpret_cast<double2*>(Tm + (rb * 8 + g) * C::PT + cl0 + 8 * c + 2 * q);
          *tp = make_double2(d0[c], d1[c]);
        }
      }
      __syncthreads();

      // ---- y-pass on the tensor cores + fused epilogue: warp = 8-column block, all RBY
      // row blocks share one window of T rows (B fragments).
      const int cbl = warp * 8;
      const double gm = (mode == RSK_APPLY_SHIFTED) ? __ldg(p.gamma + s) : 0.0;
      double* __restrict__ ys = p.Y + (int64_t)s * p.ldy;
      double* __restrict__ eys = (mode == RSK_APPLY_SPLIT) ? p.EY + (int64_t)s * p.ldey : nullptr;
      double dot = 0.0;
      {
        double bw[C::KUY];
        const double* tb = Tm + q * C::PT + cbl + g;   // B[k][n] = T[k][cbl + n]
#pragma unroll
        for (int k = 0; k < C::KUY; ++k) bw[k] = (4 * k + q < C::HY) ? tb[4 * k * C::PT] : 0.0;
        double e0[C::RBY], e1[C::RBY];
#pragma unroll
        for (int j = 0; j < C::RBY; ++j) { e0[j] = 0.0; e1[j] = 0.0; }
        const int rblk0 = r0 >> 3;
        if (!p.use_tab || (rblk0 >= p.by_lo && rblk0 + C::RBY - 1 <= p.by_hi)) {
#pragma unroll
          for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
            for (int j = 0; j < C::RBY; ++j) dmma(e0[j], e1[j], ay[ks], bw[2 * j + ks]);
        } else {
#pragma unroll
          for (int j = 0; j < C::RBY; ++j) {
            const double* fa = p.fragy + (int64_t)(rblk0 + j) * (C::KS * 32) + lane;
#pragma unroll
            for (int ks = 0; ks < C::KS; ++ks) dmma(e0[j], e1[j], __ldg(fa + ks * 32), bw[2 * j + ks]);
          }
        }
        // epilogue: lane holds rows r0 + 8j + g, columns c0 + cbl + 2q, +1
        const bool vec = ((nx & 1) == 0);
        const int lc = cbl + 2 * q;
        const int gj = c0 + lc;
#pragma unroll
        for (int j = 0; j < C::RBY; ++j) {
          const int lr = j * 8 + g;
          const int gi = r0 + lr;
          const bool v0 = gi < ny && gj < nx, v1 = gi < ny && gj + 1 < nx;
          const int so = (lr + C::H) * C::PX + lc + C::H;
          const double x0 = S[so], x1 = S[so + 1];
          double o0 = e0[j], o1 = e1[j];
          if (withE && v0) {
            // 5-point E_k stencil for the two columns; weights through L1 (prefetched)
            const int64_t o = (int64_t)gi * nx + gj;
            double wl, wm, wr, yu0, yu1, yd0, yd1;
            wl = gj > 0 ? __ldg(p.wx + o - 1) : 0.0;
            if (vec) {
              const double2 wmr = __ldg(reinterpret_cast<const double2*>(p.wx + o));
              wm = wmr.x; wr = wmr.y;
              const double2 yd = __ldg(reinterpret_cast<const double2*>(p.wy + o));
              yd0 = yd.x; yd1 = yd.y;
              if (gi > 0) {
                const double2 yu = __ldg(reinterpret_cast<const double2*>(p.wy + o - nx));
                yu0 = yu.x; yu1 = yu.y;
              } else { yu0 = 0.0; yu1 = 0.0; }
            } else {
              wm = __ldg(p.wx + o);
              wr = v1 ? __ldg(p.wx + o + 1) : 0.0;
              yd0 = __ldg(p.wy + o);
              yd1 = v1 ? __ldg(p.wy + o + 1) : 0.0;
              yu0 = gi > 0 ? __ldg(p.wy + o - nx) : 0.0;
              yu1 = (gi > 0 && v1) ? __ldg(p.wy + o - nx + 1) : 0.0;
            }
            const double xl = S[so - 1], xr = S[so + 2];
            const double u0 = S[so - C::PX], u1 = S[so - C::PX + 1];
            const double d0v = S[so + C::PX], d1v = S[so + C::PX + 1];
            const double ex0 = wl * (x0 - xl) - wm * (x1 - x0) + yu0 * (x0 - u0) - yd0 * (d0v - x0);
            const double ex1 = wm * (x1 - x0) - wr * (xr - x1) + yu1 * (x1 - u1) - yd1 * (d1v - x1);
            if (mode == RSK_APPLY_SHIFTED) {
              o0 = fma(gm, ex0, o0);
              o1 = fma(gm, ex1, o1);
            } else if (v1) {
              double* ep = eys + (int64_t)gi * nx + gj;
              if (vec && (p.ldey % 2 == 0)) *reinterpret_cast<double2*>(ep) = make_double2(ex0, ex1);
              else { ep[0] = ex0; ep[1] = ex1; }
            } else {
              eys[(int64_t)gi * nx + gj] = ex0;
            }
          }
          if (v1) {
            double* yp = ys + (int64_t)gi * nx + gj;
            if (vec && (p.ldy % 2 == 0)) *reinterpret_cast<double2*>(yp) = make_double2(o0, o1);
            else { yp[0] = o0; yp[1] = o1; }
            dot = fma(x0, o0, dot);
            dot = fma(x1, o1, dot);
          } else if (v0) {
            ys[(int64_t)gi * nx + gj] = o0;
            dot = fma(x0, o0, dot);
          }
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
            const bool act = cgmode && cg->status[s] == ST_ACTIVE;
            double t = 0.0;
            if (act) {
              __threadfence();
              const double* pa = cg->partA + (int64_t)s * cg->nblkA;
              for (int j = tid; j < p.ntiles; j += 32) t += __ldcg(pa + j);
              t = warp_sum(t);
            }
            if (tid == 0) {
              cg->cnt[4 * s + 0] = 0u;
              if (act) {
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
      }
      __syncthreads();   // everyone is done with S and T
      if (it + 1 < iend) {
        const int t2 = (it + 1) / nl, s2 = sid_of(it + 1 - t2 * nl);
        issue_x(p, smem, t2, s2, src2_of(s2));
      }
    }
  }
};

}  // namespace rsk
