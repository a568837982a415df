// Fused matrix-free shifted operator  Y_s = A X_s + gamma_s E_k X_s  (PAPER.md eq:shift
// P:361-365; A = C^T C P:137, E_k = L^T W_k L P:147 with the IRN weights of north_star).
//
// B200 design:
//  * C is a zero-boundary "same" convolution with a rank-1 PSF h = u v^T, so
//    A = (Gy^T Gy) (x) (Gx^T Gx) = By (x) Bx with banded By, Bx of half-bandwidth 2r:
//    A X = By X Bx, two banded passes of 4r+1 taps. Interior rows of B are the
//    autocorrelation of the 1-D factor; only the 2r rows next to each image edge
//    carry the zero-BC truncation (per-handle table).
//  * Both passes run on the FP64 tensor cores (mma.sync.m8n8k4.f64 -> DMMA): an 8x8
//    output block of the x-pass is  S[8 rows][cb .. cb+8+4r) x Toeplitz(Bx)[(8+4r) x 8],
//    i.e. r+2 DMMA k-steps, with the Toeplitz B-fragments precomputed in registers
//    (table fragments only for edge blocks); the y-pass is Toeplitz(By) x T[(8+4r) x 8].
//    The band costs (8+4r)/(4r+1) = 1.2-1.4x the useful FMAs but one instruction
//    carries 256 FMAs, so the kernel is no longer issue bound (the DFMA version
//    reached ~21% of the FP64 peak at r = 7).
//  * Tile = TY output rows x 64 columns; the staged halo tile is HY = roundup8(TY+4r)
//    rows x (64+4r) columns, pitch = 4 mod 8 doubles so A-fragment loads (8 rows x 4
//    consecutive doubles) are conflict-free; the intermediate has pitch 72 (8 mod 16)
//    so y-pass B-fragment loads (4 rows x 8 doubles) are conflict-free.
//  * Persistent CTAs walk (shift, tile) work items, shift-major; the NEXT item's halo
//    tile is fetched with cp.async (src-size 0 outside the image = zero boundary) into
//    the other shared buffer while the current item computes.
//  * Epilogue fuses the 5-point weighted E_k stencil (halo 1 of the same tile), the
//    gamma combine, the split output and the X.Y dot partial.
//  * CG mode: shift ids come from the active list (length on the device for graph
//    replay), items of non-ACTIVE shifts are skipped, and the CTA that finishes the
//    last tile of a shift (atomic ticket, fixed-order sum of the per-tile partials)
//    forms pi = p.w and alpha = rho / pi.
#include <cuda_runtime.h>

#include <cstdlib>

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
  const int* nlist_dev;   // if set, the list length is read on the device (graph replay)
  int mode;
  int use_tab;      // 1: A (B tables at edges), 0: C / C^T (interior taps everywhere)
  int want_dot;
  int cg_alpha;
  int dbg;          // profiling ablations (RSK_APPLY_DBG): 1 no x-pass, 2 no y-pass, 4 no epilogue, 8 no W staging
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

// D(8x8) += A(8x4, row) * B(4x8, col) in fp64 on the tensor cores. Fragments (per lane,
// g = lane / 4, q = lane % 4): a = A[g][q], b = B[q][g], d = {D[g][2q], D[g][2q+1]}.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__host__ __device__ constexpr int tc_tile_rows(int r) {
  return (8 * ((72 - 4 * r) / 8) > 56) ? 56 : 8 * ((72 - 4 * r) / 8);
}

constexpr int kAT = 512;   // threads per apply CTA: 16 warps = 8 column blocks x 2 row halves

template <int R>
struct TcCfg {
  static constexpr int H = 2 * R;            // halo of A (E needs 1 <= H)
  static constexpr int T = 4 * R + 1;        // taps of B
  static constexpr int KS = R + 2;           // DMMA k-steps per 8x8 block: (8 + 4r) / 4
  static constexpr int TY = tc_tile_rows(R); // output rows per tile (multiple of 8)
  static constexpr int HY = ((TY + 4 * R + 7) / 8) * 8;  // staged rows
  static constexpr int RBX = HY / 8;         // x-pass row blocks
  static constexpr int RBY = TY / 8;         // y-pass row blocks
  static constexpr int WX = kTX + 4 * R;     // staged cols (even)
  static constexpr int PX = (R & 1) ? WX : WX + 4;  // = 4 mod 8 doubles, rows 16B aligned
  static constexpr int PT = 72;              // = 8 mod 16 doubles
  static constexpr int PW = kTX + 1;         // weight tile pitch
  static constexpr int KU = 8 + R;           // x-pass A-fragment window (32 + 4r columns)
  static constexpr int NYH = (RBY + 1) / 2;  // y-pass row blocks per warp
  static constexpr int KUY = 2 * NYH + R;    // y-pass B-fragment window (8 NYH + 4r rows)
  static constexpr int SBUF = HY * PX;
  static constexpr int WBUF = (TY + 1) * PW; // one weight plane (+1 halo row / column)
  static constexpr size_t SMEM = sizeof(double) * (size_t)(2 * SBUF + HY * PT + 2 * WBUF + 32);
  static_assert(TY >= 8 && TY % 8 == 0, "tile rows");
  static_assert(HY <= 72, "staged rows");
};

__device__ __forceinline__ void cp_async16(double* sdst, const double* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gsrc), "r"(sz) : "memory");
}

template <int R>
__global__ void __launch_bounds__(kAT, 1) apply_kernel(const __grid_constant__ ApplyParams p) {
  using C = TcCfg<R>;
  extern __shared__ __align__(16) double smem[];
  double* Tm = smem + 2 * C::SBUF;                 // HY x PT  x-pass output
  double* sWx = Tm + C::HY * C::PT;                // [TY][PW]: wx rows r0.., cols c0-1..c0+63
  double* sWy = sWx + C::WBUF;                     // [TY+1][PW]: wy rows r0-1.., cols c0..c0+63
  double* red = sWy + C::WBUF;                     // reduction scratch
  __shared__ int s_last;

  const int ny = p.ny, nx = p.nx;
  const int nl = p.nlist_dev ? *p.nlist_dev : p.nlist;
  const int nitems = nl * p.ntiles;
  const bool cgmode = p.cg && p.cg_alpha;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int cw = warp & 7, hh = warp >> 3;         // y-pass: column block cw, row half hh
  const int g = lane >> 2, q = lane & 3;
  const bool vec16 = (nx % 2 == 0) && (p.ldx % 2 == 0);
  // interior Toeplitz fragments: x-pass B[k][n] = cx[k - n], y-pass A[m][k] = cy[k - m]
  double bx[C::KS], ay[C::KS];
#pragma unroll
  for (int ks = 0; ks < C::KS; ++ks) {
    const int t = 4 * ks + q - g;
    bx[ks] = (t >= 0 && t < C::T) ? p.cx[t] : 0.0;
    ay[ks] = (t >= 0 && t < C::T) ? p.cy[t] : 0.0;
  }
  // contiguous, tile-major work range: item = tile * nl + li
  const int per = (nitems + gridDim.x - 1) / gridDim.x;
  const int ibeg = blockIdx.x * per;
  const int iend = min(nitems, ibeg + per);

  auto next_item = [&](int it) -> int {
    if (!cgmode) return it < iend ? it : iend;
    while (it < iend && p.cg->status[p.list[it % nl]] != ST_ACTIVE) ++it;
    return it < iend ? it : iend;
  };
  auto issue = [&](int it, double* S) {
    const int tile = it / nl, li = it - tile * nl;
    const int s = p.list ? p.list[li] : li;
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int gr0 = tyi * C::TY - C::H, gc0 = txi * kTX - C::H;   // gc0 is even
    const double* xs = p.X + (int64_t)s * p.ldx;
    if (vec16) {
      // one warp per staged row: each instruction writes 32 consecutive 16-byte pairs of a
      // single row (512 B, bank-conflict free; rows straddling a warp were 3.4x wavefronts)
      constexpr int WP = C::WX / 2;                  // pairs per row
      for (int rr = warp; rr < C::HY; rr += kAT / 32) {
        const int gi = gr0 + rr;
        const bool rv = (gi >= 0) && (gi < ny);
        for (int cp = lane; cp < WP; cp += 32) {
          const int gj = gc0 + 2 * cp;
          const bool v = rv && (gj >= 0) && (gj < nx);
          cp_async16(S + rr * C::PX + 2 * cp, v ? xs + (int64_t)gi * nx + gj : xs, v);
        }
      }
    } else {
      for (int idx = tid; idx < C::HY * C::WX; idx += kAT) {
        const int rr = idx / C::WX, cc = idx - rr * C::WX;
        const int gi = gr0 + rr, gj = gc0 + cc;
        const bool v = (gi >= 0) && (gi < ny) && (gj >= 0) && (gj < nx);
        cp_async8(S + rr * C::PX + cc, v ? xs + (int64_t)gi * nx + gj : xs, v);
      }
    }
    cp_async_commit();
  };

  const int mode = p.mode;
  const bool withE = (mode == RSK_APPLY_SHIFTED || mode == RSK_APPLY_SPLIT);
  int wtile = -1;                                  // tile whose weights are staged
  int it = next_item(ibeg);
  if (it < iend) issue(it, smem);
  int stage = 0;
  while (it < iend) {
    const int nxt = next_item(it + 1);
    const int tile = it / nl, li = it - tile * nl;
    const int s = p.list ? p.list[li] : li;
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int r0 = tyi * C::TY, c0 = txi * kTX;
    __syncthreads();                       // everyone is done with buffer stage ^ 1 (and sW)
    if (withE && tile != wtile && !(p.dbg & 8)) {          // stage this tile's W_k once for all its shifts
      for (int e = tid; e < C::WBUF; e += kAT) {
        const int rr = e / C::PW, cc = e - rr * C::PW;
        {  // wx: rows r0 + rr (rr < TY), cols c0 - 1 + cc
          const int gi = r0 + rr, gj = c0 - 1 + cc;
          const bool v = rr < C::TY && gi < ny && gj >= 0 && gj < nx;
          cp_async8(sWx + e, v ? p.wx + (int64_t)gi * nx + gj : p.wx, v);
        }
        {  // wy: rows r0 - 1 + rr, cols c0 + cc (cc < 64)
          const int gi = r0 - 1 + rr, gj = c0 + cc;
          const bool v = cc < kTX && gi >= 0 && gi < ny && gj < nx;
          cp_async8(sWy + e, v ? p.wy + (int64_t)gi * nx + gj : p.wy, v);
        }
      }
      cp_async_commit();
      wtile = tile;
    }
    if (nxt < iend) issue(nxt, smem + (stage ^ 1) * C::SBUF); else cp_async_commit();
    cp_async_wait1();                      // the current item's tile (and weights) landed
    __syncthreads();
    const double* S = smem + stage * C::SBUF;
    // ---- x-pass on the tensor cores: T[rb-rows][cols] = S[rb-rows][cols .. cols+8+4r) x Bx.
    // Work unit = (row block rb, half): 4 adjacent 8-column blocks share one window of
    // A fragments (32 + 4r columns = 8 + r k-steps), block c uses window steps 2c .. 2c+r+1.
    for (int u = warp; u < ((p.dbg & 1) ? 0 : 2 * C::RBX); u += kAT / 32) {
      const int rb = u >> 1, half = u & 1;
      const int cl0 = half * 32;                       // tile-local first column of the unit
      double a[C::KU];
      const double* sa = S + (rb * 8 + g) * C::PX + cl0 + q;
#pragma unroll
      for (int k = 0; k < C::KU; ++k) a[k] = sa[4 * k];
      double d0[4], d1[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) { d0[c] = 0.0; d1[c] = 0.0; }
      const int cb0 = c0 + cl0;
      const bool xin = !p.use_tab || (cb0 >= C::H && cb0 + 32 <= nx - C::H);
      if (xin) {
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
          for (int c = 0; c < 4; ++c) dmma(d0[c], d1[c], a[2 * c + ks], bx[ks]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int col = cb0 + 8 * c + g;               // output column n = g of block c
#pragma unroll
          for (int ks = 0; ks < C::KS; ++ks) {
            const int t = 4 * ks + q - g;
            const double b = (t >= 0 && t < C::T && col < nx) ? __ldg(p.tabx + (int64_t)col * C::T + t) : 0.0;
            dmma(d0[c], d1[c], a[2 * c + ks], b);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double2* tp = reinterpret_cast<double2*>(Tm + (rb * 8 + g) * C::PT + cl0 + 8 * c + 2 * q);
        *tp = make_double2(d0[c], d1[c]);
      }
    }
    __syncthreads();

    // ---- y-pass on the tensor cores + fused epilogue. Work unit = (column block cw,
    // half hh): NYH contiguous row blocks share one window of T rows (B fragments).
    const int cbl = cw * 8;                // this warp's column block (tile-local)
    const int cb = c0 + cbl;               // global first output column of the block
    const int rbb = hh * C::NYH;           // first row block of this warp
    const double gm = (mode == RSK_APPLY_SHIFTED) ? __ldg(p.gamma + s) : 0.0;
    double* __restrict__ ys = p.Y + (int64_t)s * p.ldy;
    double* __restrict__ eys = (mode == RSK_APPLY_SPLIT) ? p.EY + (int64_t)s * p.ldey : nullptr;
    double dot = 0.0;
    {
      double bw[C::KUY];
      const double* tb = Tm + (rbb * 8 + q) * C::PT + cbl + g;   // B[k][n] = T[rbb*8 + k][cbl + n]
#pragma unroll
      for (int k = 0; k < C::KUY; ++k) bw[k] = (rbb * 8 + 4 * k + q < C::HY) ? tb[4 * k * C::PT] : 0.0;
      double e0[C::NYH], e1[C::NYH];
#pragma unroll
      for (int j = 0; j < C::NYH; ++j) { e0[j] = 0.0; e1[j] = 0.0; }
      const int rg0 = r0 + rbb * 8;
      const bool yin = !p.use_tab || (rg0 >= C::H && rg0 + 8 * C::NYH <= ny - C::H);
      if (p.dbg & 2) {
      } else if (yin) {
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
          for (int j = 0; j < C::NYH; ++j)
            if (rbb + j < C::RBY) dmma(e0[j], e1[j], ay[ks], bw[2 * j + ks]);
      } else {
#pragma unroll
        for (int j = 0; j < C::NYH; ++j) {
          if (rbb + j >= C::RBY) continue;
          const int row = rg0 + 8 * j + g;                // output row m = g of block j
#pragma unroll
          for (int ks = 0; ks < C::KS; ++ks) {
            const int t = 4 * ks + q - g;
            const double a = (t >= 0 && t < C::T && row < ny) ? __ldg(p.taby + (int64_t)row * C::T + t) : 0.0;
            dmma(e0[j], e1[j], a, bw[2 * j + ks]);
          }
        }
      }
      // epilogue: lane holds rows r0 + (rbb+j)*8 + g, columns cb + 2q, cb + 2q + 1
      const bool full = (r0 + C::TY <= ny) && (c0 + kTX <= nx);
#pragma unroll
      for (int j = 0; j < C::NYH; ++j) {
        const int rb = rbb + j;
        if (rb >= C::RBY) continue;
        const int lr = rb * 8 + g;             // tile-local row
        const int gi = r0 + lr;
        const int lc = cbl + 2 * q;            // tile-local first column
        const int gj = c0 + lc;
        const int so = (lr + C::H) * C::PX + lc + C::H;
        const double x0 = S[so], x1 = S[so + 1];
        double o0 = e0[j], o1 = e1[j];
        if (withE && !(p.dbg & 4)) {
          // 5-point E_k stencil for the two columns (weights from the staged tile)
          const double xl = S[so - 1], xr = S[so + 2];
          const double u0 = S[so - C::PX], u1 = S[so - C::PX + 1];
          const double d0v = S[so + C::PX], d1v = S[so + C::PX + 1];
          const double* wxr = sWx + lr * C::PW + lc;   // [lc] = wx(gj-1), [lc+1] = wx(gj), [lc+2] = wx(gj+1)
          const double* wyr = sWy + lr * C::PW + lc;   // row lr: wy(gi-1); row lr+1: wy(gi)
          const double wl = wxr[0], wm = wxr[1], wr = wxr[2];
          const double yu0 = wyr[0], yu1 = wyr[1];
          const double yd0 = wyr[C::PW], yd1 = wyr[C::PW + 1];
          const double ex0 = wl * (x0 - xl) - wm * (x1 - x0) + yu0 * (x0 - u0) - yd0 * (d0v - x0);
          const double ex1 = wm * (x1 - x0) - wr * (xr - x1) + yu1 * (x1 - u1) - yd1 * (d1v - x1);
          if (mode == RSK_APPLY_SHIFTED) {
            o0 = fma(gm, ex0, o0);
            o1 = fma(gm, ex1, o1);
          } else if (full || (gi < ny && gj + 1 < nx)) {
            double* ep = eys + (int64_t)gi * nx + gj;
            if (vec16 && (p.ldey % 2 == 0)) *reinterpret_cast<double2*>(ep) = make_double2(ex0, ex1);
            else { ep[0] = ex0; ep[1] = ex1; }
          } else if (gi < ny && gj < nx) {
            eys[(int64_t)gi * nx + gj] = ex0;
          }
        }
        if (full || (gi < ny && gj + 1 < nx)) {
          if (vec16 && (p.ldy % 2 == 0)) *reinterpret_cast<double2*>(ys + (int64_t)gi * nx + gj) = make_double2(o0, o1);
          else { ys[(int64_t)gi * nx + gj] = o0; ys[(int64_t)gi * nx + gj + 1] = o1; }
          dot = fma(x0, o0, dot);
          dot = fma(x1, o1, dot);
        } else if (gi < ny && gj < nx) {
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
  const int ty = tc_tile_rows(h->r);
  const int tx = (int)((h->nx + kTX - 1) / kTX), tyc = (int)((h->ny + ty - 1) / ty);
  return tx * tyc;
}

template <int R>
static cudaError_t launch_r(const ApplyParams& prm, int sm_count, cudaStream_t st) {
  using C = TcCfg<R>;
  static int blocks_per_sm = 0;
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(apply_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, apply_kernel<R>, kAT, C::SMEM);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int nitems = prm.nlist * prm.ntiles;
  int grid = blocks_per_sm * sm_count;
  if (grid > nitems && !prm.nlist_dev) grid = nitems;
  count_launch();
  apply_kernel<R><<<grid, kAT, C::SMEM, st>>>(prm);
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
  prm.nlist_dev = a.nlist_dev;
  prm.mode = a.mode;
  prm.cg_alpha = a.cg_alpha ? 1 : 0;
  {
    static int dbg = -1;
    if (dbg < 0) { const char* e = getenv("RSK_APPLY_DBG"); dbg = e ? atoi(e) : 0; }
    prm.dbg = dbg;
  }
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
