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
//    (r+2 DMMA k-steps); the y-pass is Toeplitz(By) x T[(8+4r) x 8], Toeplitz fragments
//    in registers. The zero boundary truncates B = G^T G only in an r x r corner at each
//    end (B = Toeplitz - D_lo - D_hi, D_lo(c,m) = sum_{j<0} f[j-c+r] f[j-m+r]), so outputs
//    within r of an edge get a small register-level correction instead of another path.
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
  const double* dcorr;  // [4][kMaxR][kMaxR] zero-boundary corrections of B (see below)
  double* part;         // [list index][ntiles] (plain mode dot partials)
  CgDev* cg;
  int ny, nx, tiles_x, ntiles, nlist;
  const int* nlist_dev;  // if set, the list length is read on the device
  int mode;
  int edge_fix;  // 1: A (B truncated at the image edges), 0: C / C^T (exact with the zero halo)
  int want_dot;
  int cg_alpha;
  int src2_rconv;  // CG: items whose shift status is ST_RCONV read X2 (true-residual confirm)
  unsigned long long* aprof;       // optional per-phase ns of one block (RSK_APPLY_PROF=<block>)
  int aprof_block;
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
constexpr int kApplyCtasPerSm = 1;   // one CTA per SM: 255 registers, double-buffered stage
constexpr int kStages = 2;

// TY_ = 0: the default tile height tc_tile_rows(R) (64-row halo, 16 balanced x-pass
// units); the cluster-per-shift loop uses taller tiles so one shift has <= 1 tile per CTA.
template <int R, int TY_ = 0>
struct TcCfg {
  static constexpr int H = 2 * R;            // halo of A (E needs 1 <= H)
  static constexpr int T = 4 * R + 1;        // taps of B
  static constexpr int KS = R + 2;           // DMMA k-steps per 8x8 block: (8 + 4r) / 4
  static constexpr int TY = TY_ ? TY_ : tc_tile_rows(R); // output rows per tile (multiple of 8)
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
  static constexpr int OFF_T = kStages * SBUF;
  static constexpr int OFF_RED = OFF_T + TBUF;
  static constexpr int OFF_DC = OFF_RED + 16;         // 4 r x r boundary corrections
  static constexpr int OFF_FR = OFF_DC + al16(4 * R * R);    // Toeplitz fragments [2][KS][32]
  static constexpr int OFF_BAR = OFF_FR + al16(2 * KS * 32);  // kStages mbarriers (8 B each)
  static constexpr int DBL = OFF_BAR + kStages;
  static constexpr size_t SMEM = sizeof(double) * (size_t)DBL;
  static constexpr unsigned XBYTES = 8u * HY * PX;
  static_assert(TY >= 8 && TY % 8 == 0, "tile rows");
  static_assert(HY <= 128, "staged rows");
  static_assert(PX <= 256, "TMA box width");
  static_assert(kApplyCtasPerSm * (SMEM + 1024) <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block sum (fixed tree), result valid in thread 0
// Double-double accumulation (Knuth TwoSum, exact for any operand order): sums of many
// terms kept to ~2^-104 relative, so the rounded total does not depend on how the terms were
// grouped (the streaming CG loop's p.w: batch-composition-independent alpha).
__device__ __forceinline__ void dd_add(double& h, double& l, double bh, double bl) {
  const double s = h + bh;
  const double bb = s - h;
  double e = (h - (s - bb)) + (bh - bb);
  e += l + bl;
  h = s + e;
  l = e - (h - s);
}
__device__ __forceinline__ void warp_sum_dd(double& h, double& l) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oh = __shfl_xor_sync(0xffffffffu, h, o), ol = __shfl_xor_sync(0xffffffffu, l, o);
    dd_add(h, l, oh, ol);
  }
}
// red: >= 2 x (warps) doubles; every thread of warp 0 returns the CTA's sum
__device__ __forceinline__ void block_sum_dd(double& h, double& l, double* red) {
  warp_sum_dd(h, l);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) { red[2 * wid] = h; red[2 * wid + 1] = l; }
  __syncthreads();
  if (wid == 0) {
    const bool in = lane < (int)(blockDim.x >> 5);
    h = in ? red[2 * lane] : 0.0;
    l = in ? red[2 * lane + 1] : 0.0;
    warp_sum_dd(h, l);
  }
}

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
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p));
}

// mbarrier use counter (parity of the next wait); every thread runs the same sequence
struct ApplyPipe {
  unsigned use[kStages];
  int stage;   // stage buffer of the next item
};

template <int R, bool kTma, int TY_ = 0>
struct ApplyCore {
  using C = TcCfg<R, TY_>;

  __device__ static void init_bars(double* smem, const ApplyParams& p) {
    // boundary corrections of B (tiny, read at every edge output)
    // per-lane Toeplitz fragments, once per CTA: x-pass B[k][n] = cx[k - n], y-pass
    // A[m][k] = cy[k - m] (k = 4 ks + q, n = m = g). Lane-indexed parameter reads diverge
    // across the constant cache; the items read them back conflict-free from here.
    for (int e = threadIdx.x; e < 2 * C::KS * 32; e += blockDim.x) {
      const int which = e / (C::KS * 32), rem = e - which * C::KS * 32;
      const int ks = rem >> 5, ln = rem & 31;
      const int t = 4 * ks + (ln & 3) - (ln >> 2);
      smem[C::OFF_FR + e] = (t >= 0 && t < C::T) ? (which ? p.cy[t] : p.cx[t]) : 0.0;
    }
    for (int e = threadIdx.x; e < 4 * R * R; e += blockDim.x) {
      const int sl = e / (R * R), rem = e - sl * R * R, a = rem / R, b = rem - a * R;
      smem[C::OFF_DC + e] = p.dcorr ? p.dcorr[((size_t)sl * kMaxR + a) * kMaxR + b] : 0.0;
    }
    if (kTma && threadIdx.x == 0) {
      for (int b = 0; b < kStages; ++b) mbar_init(reinterpret_cast<uint64_t*>(smem + C::OFF_BAR) + b, 1);
      mbar_fence_init();
    }
    __syncthreads();
  }

  // stage the halo tile of (tile, shift s)
  __device__ static void issue_x(const ApplyParams& p, double* smem, int stage, int tile, int s, bool src2) {
    double* S = smem + stage * C::SBUF;
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int gr0 = tyi * C::TY - C::H, gc0 = txi * kTX - C::H;
    if (kTma) {
      if (threadIdx.x == 0) {
        uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR) + stage;
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
  // list / smode (optional, e.g. shared-memory snapshots) override p.list and the
  // status-based choice of the source vector.
  // dot_acc (optional): thread 0 accumulates the items' X.Y block sums in item order
  __device__ __forceinline__ static void run(const ApplyParams& p, double* smem, int ibeg, int iend, int nl, ApplyPipe& pp,
                             const int* list = nullptr, const int* smode = nullptr, double* dot_acc = nullptr) {
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
    const int* lst = list ? list : p.list;
    auto sid_of = [&](int li) -> int { return lst ? lst[li] : li; };
    auto src2_of = [&](int li, int s) -> bool {
      return smode ? (smode[li] == ST_RCONV) : (p.src2_rconv && p.cg->status[s] == ST_RCONV);
    };

    unsigned long long tp0 = 0;
    auto amark = [&](int ph) {
      if (p.aprof && (int)blockIdx.x == (p.aprof_block < 0 ? (int)gridDim.x / 2 : p.aprof_block) && tid == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
        if (tp0) atomicAdd(p.aprof + ph, t1 - tp0);
        tp0 = t1;
      }
    };
    amark(7);
    {
      const int tile = ibeg / nl, li0 = ibeg - tile * nl, s = sid_of(li0);
      issue_x(p, smem, pp.stage, tile, s, src2_of(li0, s));
    }
    for (int it = ibeg; it < iend; ++it) {
      const int tile = it / nl, li = it - tile * nl;
      const int s = sid_of(li);
      const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
      const int r0 = tyi * C::TY, c0 = txi * kTX;
      const int stage = pp.stage;
      const bool more = it + 1 < iend;
      if (more) {   // the other stage was released by the previous item's final barrier
        const int t2 = (it + 1) / nl, l2 = it + 1 - t2 * nl, s2 = sid_of(l2);
        issue_x(p, smem, stage ^ 1, t2, s2, src2_of(l2, s2));
      }
      amark(0);
      if (kTma) {
        mbar_wait(bar + stage, pp.use[stage] & 1);
        pp.use[stage] += 1;
      } else {
        if (more) cp_async_wait1(); else cp_async_wait0();
        __syncthreads();
      }
      const double* S = smem + stage * C::SBUF;
      amark(1);

      // ---- x-pass on the tensor cores: T[rb-rows][cols] = S[rb-rows][cols .. cols+8+4r) x Bx.
      // Work unit = (row block rb, half): 4 adjacent 8-column blocks share one window of
      // A fragments (32 + 4r columns = 8 + r k-steps), block c uses window steps 2c .. 2c+r+1.
      // interior Toeplitz fragments: x-pass B[k][n] = cx[k - n] (from the parameter bank)
      double bx[C::KS];
#pragma unroll
      for (int ks = 0; ks < C::KS; ++ks) bx[ks] = smem[C::OFF_FR + ks * 32 + lane];
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
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
          for (int c = 0; c < 4; ++c) dmma(d0[c], d1[c], a[2 * c + ks], bx[ks]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double2* tp = reinterpret_cast<double2*>(Tm + (rb * 8 + g) * C::PT + cl0 + 8 * c + 2 * q);
          *tp = make_double2(d0[c], d1[c]);
        }
      }
      __syncthreads();
      // zero-boundary corrections of the x-pass on T (only tiles touching the left or right
      // image edge): T[row][col] -= sum_m D(col, m) x(row, m) for the r columns nearest it
      if (p.edge_fix && (c0 < R || c0 + kTX > nx - R)) {
        for (int e = tid; e < C::HY * 2 * R; e += kAT) {
          const int row = e / (2 * R), k = e - row * (2 * R);
          const bool right = k >= R;
          const int col = right ? nx - R + (k - R) : k;          // global column
          const int lc = col - c0;
          if (lc < 0 || lc >= kTX || col < 0 || col >= nx) continue;
          if (right && col < R) continue;                          // tiny images: the left item does both
          const double* srow = S + row * C::PX - (c0 - C::H);    // srow[m] = x(row, m)
          double corr = 0.0;
          if (!right) {
            const double* dl = smem + C::OFF_DC + col * R;
#pragma unroll
            for (int m = 0; m < R; ++m) corr = fma(dl[m], srow[m], corr);
          }
          if (col >= nx - R) {
            const double* dr = smem + C::OFF_DC + (R + col - (nx - R)) * R;
#pragma unroll
            for (int m = 0; m < R; ++m) corr = fma(dr[m], srow[nx - R + m], corr);
          }
          Tm[row * C::PT + lc] -= corr;
        }
        __syncthreads();
      }
      amark(2);

      // ---- y-pass on the tensor cores + fused epilogue: warp = 8-column block, all RBY
      // row blocks share one window of T rows (B fragments). The weights of the first
      // EJ row blocks are requested before the DMMAs so their latency hides behind them.
      const int cbl = warp * 8;
      const double gm = (mode == RSK_APPLY_SHIFTED) ? __ldg(p.gamma + s) : 0.0;
      double* __restrict__ ys = p.Y + (int64_t)s * p.ldy;
      double* __restrict__ eys = (mode == RSK_APPLY_SPLIT) ? p.EY + (int64_t)s * p.ldey : nullptr;
      double dot = 0.0;
      {
        const bool vec = ((nx & 1) == 0);
        const int lc = cbl + 2 * q;
        const int gj = c0 + lc;
        constexpr int EJ = C::RBY > 4 ? 4 : C::RBY;   // weight loads of the first EJ row blocks go out before the y-pass DMMAs
        double wl[EJ], wm[EJ], wr[EJ], yu0[EJ], yu1[EJ], yd0[EJ], yd1[EJ];
        auto load_w = [&](int j, int jj) {
          const int gi = r0 + j * 8 + g;
          const bool v0 = gi < ny && gj < nx, v1 = gi < ny && gj + 1 < nx;
          wl[jj] = wm[jj] = wr[jj] = yu0[jj] = yu1[jj] = yd0[jj] = yd1[jj] = 0.0;
          if (!v0) return;
          const int64_t o = (int64_t)gi * nx + gj;
          if (gj > 0) wl[jj] = __ldg(p.wx + o - 1);
          if (vec) {
            const double2 a2 = __ldg(reinterpret_cast<const double2*>(p.wx + o));
            wm[jj] = a2.x; wr[jj] = a2.y;
            const double2 d2 = __ldg(reinterpret_cast<const double2*>(p.wy + o));
            yd0[jj] = d2.x; yd1[jj] = d2.y;
            if (gi > 0) {
              const double2 u2 = __ldg(reinterpret_cast<const double2*>(p.wy + o - nx));
              yu0[jj] = u2.x; yu1[jj] = u2.y;
            }
          } else {
            wm[jj] = __ldg(p.wx + o);
            yd0[jj] = __ldg(p.wy + o);
            if (gi > 0) yu0[jj] = __ldg(p.wy + o - nx);
            if (v1) {
              wr[jj] = __ldg(p.wx + o + 1);
              yd1[jj] = __ldg(p.wy + o + 1);
              if (gi > 0) yu1[jj] = __ldg(p.wy + o - nx + 1);
            }
          }
        };
        if (withE) {
#pragma unroll
          for (int jj = 0; jj < EJ; ++jj) load_w(jj, jj);
        }
        double bw[C::KUY];
        const double* tb = Tm + q * C::PT + cbl + g;   // B[k][n] = T[k][cbl + n]
#pragma unroll
        for (int k = 0; k < C::KUY; ++k) bw[k] = (4 * k + q < C::HY) ? tb[4 * k * C::PT] : 0.0;
        double e0[C::RBY], e1[C::RBY];
#pragma unroll
        for (int j = 0; j < C::RBY; ++j) { e0[j] = 0.0; e1[j] = 0.0; }
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks) {
          const double ay = smem[C::OFF_FR + (C::KS + ks) * 32 + lane];   // y-pass A[m][k] = cy[k - m]
#pragma unroll
          for (int j = 0; j < C::RBY; ++j) dmma(e0[j], e1[j], ay, bw[2 * j + ks]);
        }
        if (p.edge_fix && (r0 < R || r0 + C::TY > ny - R)) {
          const double* tcol = Tm - (r0 - C::H) * C::PT + lc;   // tcol[m * PT] = T(row m, col lc)
#pragma unroll
          for (int j = 0; j < C::RBY; ++j) {
            const int gi = r0 + 8 * j + g;
            double c0v = 0.0, c1v = 0.0;
            if (gi < R) {
              const double* dt = smem + C::OFF_DC + (2 * R + gi) * R;
#pragma unroll
              for (int m = 0; m < R; ++m) {
                const double dv = dt[m];
                c0v = fma(dv, tcol[m * C::PT], c0v);
                c1v = fma(dv, tcol[m * C::PT + 1], c1v);
              }
            }
            if (gi >= ny - R && gi < ny) {
              const double* db = smem + C::OFF_DC + (3 * R + gi - (ny - R)) * R;
#pragma unroll
              for (int m = 0; m < R; ++m) {
                const double dv = db[m];
                c0v = fma(dv, tcol[(ny - R + m) * C::PT], c0v);
                c1v = fma(dv, tcol[(ny - R + m) * C::PT + 1], c1v);
              }
            }
            e0[j] -= c0v;
            e1[j] -= c1v;
          }
        }
        // epilogue: lane holds rows r0 + 8j + g, columns c0 + cbl + 2q, +1
#pragma unroll
        for (int jc = 0; jc < C::RBY; jc += EJ) {
          if (withE && jc > 0) {
#pragma unroll
            for (int jj = 0; jj < EJ; ++jj)
              if (jc + jj < C::RBY) load_w(jc + jj, jj);
          }
#pragma unroll
          for (int jj = 0; jj < EJ; ++jj) {
            const int j = jc + jj;
            if (j >= C::RBY) break;
            const int lr = j * 8 + g;
            const int gi = r0 + lr;
            const bool v0 = gi < ny && gj < nx, v1 = gi < ny && gj + 1 < nx;
            const int so = (lr + C::H) * C::PX + lc + C::H;
            const double x0 = S[so], x1 = S[so + 1];
            double o0 = e0[j], o1 = e1[j];
            if (withE && v0) {
              // 5-point E_k stencil for the two columns
              const double xl = S[so - 1], xr = S[so + 2];
              const double u0 = S[so - C::PX], u1 = S[so - C::PX + 1];
              const double d0v = S[so + C::PX], d1v = S[so + C::PX + 1];
              const double ex0 = wl[jj] * (x0 - xl) - wm[jj] * (x1 - x0) + yu0[jj] * (x0 - u0) - yd0[jj] * (d0v - x0);
              const double ex1 = wm[jj] * (x1 - x0) - wr[jj] * (xr - x1) + yu1[jj] * (x1 - u1) - yd1[jj] * (d1v - x1);
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
      }

      amark(3);
      if (p.want_dot) {
        const double bs = block_sum(dot, red);
        if (dot_acc) {          // per list index (the cluster loops pass one shift: [0])
          if (tid == 0) dot_acc[li] += bs;
        } else if (!p.cg) {
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
      amark(4);
      __syncthreads();   // everyone is done with S and T
      amark(5);
      pp.stage ^= 1;
    }
  }
};

}  // namespace rsk
