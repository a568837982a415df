// Streaming ("strip") form of the fused shifted apply  Y_s = A X_s + gamma_s E_k X_s
// (PAPER.md eq:shift P:361-365, A = C^T C P:137, E_k = L^T W_k L P:147) for images
// larger than L2 -- the C3 / C4 / C5 path. DESIGN.md §4.1b.
//
// Same algebra as apply_core.cuh (A = By (x) Bx, B = G^T G banded with 4r+1 taps, both
// passes on the FP64 tensor cores, register-level zero-boundary corrections), different
// data flow. A work item is (vector s, column strip of 64 output columns, row segment);
// the CTA walks DOWN the strip in 8-row blocks:
//
//   step t:  wait for input block t (TMA box {64 + 4r (+pad), 8 rows, 1}, already in
//            flight: the ring keeps D blocks ahead)  ->  x-pass of block t into the
//            T ring (8 warps = the 8 column blocks of the strip)  ->  __syncthreads
//            ->  issue input block t + D  ->  y-pass of output block j = t - LAG from
//            the T ring (window of 8 + 4r rows) + the fused epilogue (E_k stencil from
//            the input ring, gamma combine / split output, X.Y partial).
//
// Every x-pass result is used by 4r + 8 output rows (no recomputed halo rows: the tiled
// core recomputes 4r of every 64 - 4r rows, 1.6x the DMMAs at r = 7), and consecutive
// strips of one vector share their 2r-column halos through L2. Both rings are 8 blocks
// deep (input ring: LAG + D + 1 <= 8).
//
// No CTA barrier per step: a warp's x-pass writes and its y-pass reads only its own 8
// columns of the T ring (__syncwarp), and the input ring is a full / empty mbarrier
// pipeline -- full[slot] completes with the TMA bytes, empty[slot] when all 8 warps have
// made their last read of the block (x-pass at step b, E-stencil rows at steps up to
// b + K, K = LAG - floor((H - 1) / 8)); thread 0 waits on empty before re-filling a slot.
// The warps drift apart by up to 7 - D - K steps, so the DMMA, shared-load and
// epilogue phases of different warps overlap instead of running in lockstep.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "apply_core.cuh"
#include "rsk_internal.h"
#include "tma.cuh"

namespace rsk {

constexpr int kStripW = 64;    // output columns per strip (8 warps x 8-column blocks)
constexpr int kStripCtasPerSm = 2;

// TAIL > 0 places the persistent part of the layout (correction table, reduction scratch,
// mbarriers) at that offset (doubles), after a caller's larger scratch region that
// reuses the rings between apply phases (the CG loop of cg_stream.cu)
template <int R, int TAIL = 0>
struct StripCfg {
  static constexpr int H = 2 * R;                   // halo of A
  static constexpr int KS = R + 2;                  // DMMA k-steps per 8x8 block: (8 + 4r) / 4
  static constexpr int LAG = (7 + 4 * R) / 8;       // output block j needs T blocks <= j + LAG
  static constexpr int D = (7 - LAG) < 3 ? (7 - LAG) : 3;   // input blocks in flight ahead
  static constexpr int PX = pad4mod8(kStripW + 4 * R);      // input ring pitch (TMA box width)
  static constexpr int PT = 68;                     // T ring pitch (4 mod 16 doubles: the y-pass B
                                                    // fragments of a half-warp hit 16 distinct banks)
  static constexpr int OFF_IN = 0;                  // [64][PX] input ring (8 slots x 8 rows)
  static constexpr int OFF_T = OFF_IN + al16(64 * PX);   // [64][PT] x-pass ring
  static constexpr int RING_END = OFF_T + al16(64 * PT);
  static constexpr int OFF_DC = TAIL > 0 ? TAIL : RING_END;   // [4R][R] zero-boundary corrections
  static constexpr int OFF_FR = OFF_DC + al16(4 * R * R);    // [2][KS][32] Toeplitz fragments
  static constexpr int OFF_RED = OFF_FR + al16(2 * KS * 32);  // block-reduction scratch
  static constexpr int OFF_BAR = OFF_RED + 16;      // 8 full mbarriers (8 B each)
  static constexpr int OFF_EBAR = OFF_BAR + 8;      // 8 empty mbarriers (8 warp arrivals)
  static constexpr int DBL = OFF_EBAR + 8;
  static constexpr int K = LAG - (H - 1) / 8;       // block b's last read: step b + K
  static_assert(D + K <= 7, "input ring reuse: the issuer at step t needs block t + D - 8 released");
  static constexpr size_t SMEM = sizeof(double) * (size_t)DBL;
  static constexpr unsigned XBYTES = 8u * 8u * PX;
  static_assert(D >= 1, "input ring too shallow for this r");
  static_assert(PX <= 256, "TMA box width");
  static_assert(kStripCtasPerSm * (SMEM + 2048) <= 227 * 1024, "shared memory");
};

struct alignas(64) StripParams {
  CUtensorMap mapX;    // 3-D {nx, ny, vectors}, box {PX, 8, 1}
  CUtensorMap mapX2;   // CG: true-residual confirm source (the iterate x), same geometry
  double* Y;
  int64_t ldy;
  double* EY;
  int64_t ldey;
  const double* gamma;   // indexed by vector id
  const double* wx;
  const double* wy;
  const double* dcorr;   // [4][kMaxR][kMaxR]
  double* part;          // X.Y partial per (vector id, segment x strip)
  int ny, nx;
  int nstrip, nseg, seg_rows;
  int row0, row1;        // output rows [row0, row1) (segments start at row0; default 0, ny)
  int mode;              // RSK_APPLY_SHIFTED or RSK_APPLY_SPLIT
  int want_dot;
  int prefetch_w;        // L1 prefetch of the weights two blocks ahead (RSK_STRIP_NOPF=1: off)
  double cx[kMaxTaps];
  double cy[kMaxTaps];
};

// per-CTA ring state (identical in every thread)
struct StripRing {
  unsigned pos;      // ring blocks consumed so far (slot = pos & 7)
  unsigned parity;   // bit s: parity of the next wait on slot s
};

template <int R, int TAIL = 0>
struct StripCore {
  using C = StripCfg<R, TAIL>;

  __device__ static void init(double* smem, const StripParams& p) {
    for (int e = threadIdx.x; e < 4 * R * R; e += blockDim.x) {
      const int sl = e / (R * R), rem = e - sl * R * R, a = rem / R, b = rem - a * R;
      smem[C::OFF_DC + e] = p.dcorr ? p.dcorr[((size_t)sl * kMaxR + a) * kMaxR + b] : 0.0;
    }
    // per-lane Toeplitz fragments: x-pass B[k][n] = cx[k - n], y-pass A[m][k] = cy[k - m]
    // (k = 4 ks + q, n = m = g)
    for (int e = threadIdx.x; e < 2 * C::KS * 32; e += blockDim.x) {
      const int which = e / (C::KS * 32), rem = e - which * C::KS * 32;
      const int ks = rem >> 5, ln = rem & 31;
      const int t = 4 * ks + (ln & 3) - (ln >> 2);
      smem[C::OFF_FR + e] = (t >= 0 && t <= 4 * R) ? (which ? p.cy[t] : p.cx[t]) : 0.0;
    }
    if (threadIdx.x == 0) {
      for (int b = 0; b < 8; ++b) mbar_init(reinterpret_cast<uint64_t*>(smem + C::OFF_BAR) + b, 1);
      for (int b = 0; b < 8; ++b) mbar_init(reinterpret_cast<uint64_t*>(smem + C::OFF_EBAR) + b, kAT / 32);
      mbar_fence_init();
    }
    __syncthreads();
  }

  // fill ring position P (slot P & 7) with the input block at image row row0; the slot's
  // previous block (P - 8) must have been released by every warp
  __device__ static void issue(const StripParams& p, double* smem, unsigned P, int c0, int row0, int s,
                               bool src2) {
    const unsigned slot = P & 7u;
    if (P >= 8u) mbar_wait(reinterpret_cast<uint64_t*>(smem + C::OFF_EBAR) + slot, ((P >> 3) - 1u) & 1u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR) + slot;
    mbar_expect_tx(bar, C::XBYTES);
    tma_load_3d(smem + C::OFF_IN + slot * 8 * C::PX, src2 ? &p.mapX2 : &p.mapX, bar, c0 - C::H, row0, s);
  }

  // Returns this thread's X.Y partial as a double-double (return value + *dot_lo; caller
  // reduces): per 8-row block the thread's two products, added by TwoSum, so the item's
  // total does not depend on where items start and end. src2: read the vector from mapX2
  // (CG confirm).
  // One item: vector s, a strip, output rows [ra, rb) (rb - ra a multiple of 8 unless rb = ny).
  __device__ static double item(const StripParams& p, double* smem, StripRing& ring, int s, int strip, int ra, int rb,
                                bool src2, double* dot_lo) {
    double* IN = smem + C::OFF_IN;
    double* T = smem + C::OFF_T;
    const double* DC = smem + C::OFF_DC;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int ny = p.ny, nx = p.nx;
    const int nbo = (rb - ra + 7) >> 3;
    const int nbi = nbo + C::LAG;
    const int c0 = strip * kStripW;
    const int rb0 = ra - C::H;            // image row of ring row u = 0 of this item
    const unsigned base = ring.pos;
    unsigned parity = ring.parity;   // a register copy for the step loop (the caller's ring
                                     // state lives across phases and may sit in local memory)
    const int mode = p.mode;
    const bool withE = true;
    const bool edge_l = c0 < R, edge_r = c0 + kStripW > nx - R;
    const double gm = (mode == RSK_APPLY_SHIFTED) ? __ldg(p.gamma + s) : 0.0;
    double* __restrict__ ys = p.Y + (int64_t)s * p.ldy;
    double* __restrict__ eys = (mode == RSK_APPLY_SPLIT) ? p.EY + (int64_t)s * p.ldey : nullptr;
    const bool vec = ((nx & 1) == 0);
    const int cb = warp * 8;
    double dot = 0.0, dlo = 0.0;
    double bx[C::KS], ay[C::KS];
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks) {
      bx[ks] = smem[C::OFF_FR + ks * 32 + lane];
      ay[ks] = smem[C::OFF_FR + (C::KS + ks) * 32 + lane];
    }

    uint64_t* ebars = reinterpret_cast<uint64_t*>(smem + C::OFF_EBAR);
    if (tid == 0)
      for (int t = 0; t < C::D && t < nbi; ++t) issue(p, smem, base + t, c0, rb0 + 8 * t, s, src2);

#pragma unroll 1
    for (int t = 0; t < nbi; ++t) {
      const unsigned slot = (base + t) & 7u;
      if (tid == 0 && t + C::D < nbi) issue(p, smem, base + t + C::D, c0, rb0 + 8 * (t + C::D), s, src2);
      mbar_wait(bars + slot, (parity >> slot) & 1u);
      parity ^= 1u << slot;
      // ---- x-pass of input block t: T[8 rows][cb .. cb+8) = IN[8 rows][cb .. cb+8+4r) x Bx
      {
        const double* sa = IN + (slot * 8 + g) * C::PX + cb + q;
        double a[C::KS];
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks) a[ks] = sa[4 * ks];
        double d0 = 0.0, d1 = 0.0, f0 = 0.0, f1 = 0.0;   // two accumulator chains
#pragma unroll
        for (int ks = 0; ks < C::KS; ks += 2) dmma(d0, d1, a[ks], bx[ks]);
#pragma unroll
        for (int ks = 1; ks < C::KS; ks += 2) dmma(f0, f1, a[ks], bx[ks]);
        d0 += f0; d1 += f1;
        if (edge_l || edge_r) {
          // zero boundary in x: T(row, col) -= sum_m D(col, m) x(row, m) for the r columns
          // nearest each image edge (x(row, m) = IN[row][m - c0 + 2r])
          const double* srow = IN + (slot * 8 + g) * C::PX - (c0 - C::H);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int col = c0 + cb + 2 * q + hh;
            double corr = 0.0;
            if (col < R) {
              const double* dl = DC + col * R;
#pragma unroll
              for (int m = 0; m < R; ++m) corr = fma(dl[m], srow[m], corr);
            }
            if (col >= nx - R && col < nx) {
              const double* dr = DC + (R + col - (nx - R)) * R;
#pragma unroll
              for (int m = 0; m < R; ++m) corr = fma(dr[m], srow[nx - R + m], corr);
            }
            if (hh == 0) d0 -= corr; else d1 -= corr;
          }
        }
        *reinterpret_cast<double2*>(T + (slot * 8 + g) * C::PT + cb + 2 * q) = make_double2(d0, d1);
      }
      __syncwarp();   // the warp's T columns: x-pass stores before its y-pass loads
      {
        // the weights of output block t - LAG + 2 into L1 (two steps ahead of their use)
        const int gi2 = ra + 8 * (t - C::LAG + 2) + g;
        const int gj2 = c0 + cb + 2 * q;
        if (p.prefetch_w && gi2 >= ra && gi2 < rb && gj2 < nx) {
          const int64_t o = (int64_t)gi2 * nx + gj2;
          prefetch_l1(p.wx + o + (gj2 > 0 ? -1 : 0));
          prefetch_l1(p.wx + o + 1);
          prefetch_l1(p.wy + o);
          if (gi2 > 0) prefetch_l1(p.wy + o - nx);
        }
      }
      const int j = t - C::LAG;
      if (j < 0) {
        release(ebars, base, t - C::K, lane);
        continue;
      }
      // ---- y-pass of output block j: rows ra + 8j .. +7 from T window rows u = 8j .. 8j+4r+7
      const int i0 = ra + 8 * j;
      const int gi = i0 + g;                 // this lane's output row
      const int gj = c0 + cb + 2 * q;        // this lane's first output column
      const bool v0 = gi < rb && gj < nx, v1 = gi < rb && gj + 1 < nx;
      // weights of the E_k stencil first (their latency hides behind the DMMAs)
      double wl = 0.0, wm = 0.0, wr = 0.0, yu0 = 0.0, yu1 = 0.0, yd0 = 0.0, yd1 = 0.0;
      if (withE && v0) {
        const int64_t o = (int64_t)gi * nx + gj;
        if (gj > 0) wl = __ldg(p.wx + o - 1);
        if (vec) {
          const double2 a2 = __ldg(reinterpret_cast<const double2*>(p.wx + o));
          wm = a2.x; wr = a2.y;
          const double2 d2 = __ldg(reinterpret_cast<const double2*>(p.wy + o));
          yd0 = d2.x; yd1 = d2.y;
          if (gi > 0) {
            const double2 u2 = __ldg(reinterpret_cast<const double2*>(p.wy + o - nx));
            yu0 = u2.x; yu1 = u2.y;
          }
        } else {
          wm = __ldg(p.wx + o);
          yd0 = __ldg(p.wy + o);
          if (gi > 0) yu0 = __ldg(p.wy + o - nx);
          if (v1) {
            wr = __ldg(p.wx + o + 1);
            yd1 = __ldg(p.wy + o + 1);
            if (gi > 0) yu1 = __ldg(p.wy + o - nx + 1);
          }
        }
      }
      const unsigned ub = base * 8u + 8u * (unsigned)j;   // ring row of u = 8j is ub & 63
      double e0 = 0.0, e1 = 0.0, h0 = 0.0, h1 = 0.0;
      {
        double bw[C::KS];
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks) bw[ks] = T[((ub + 4 * ks + q) & 63u) * C::PT + cb + g];
#pragma unroll
        for (int ks = 0; ks < C::KS; ks += 2) dmma(e0, e1, ay[ks], bw[ks]);
#pragma unroll
        for (int ks = 1; ks < C::KS; ks += 2) dmma(h0, h1, ay[ks], bw[ks]);
      }
      e0 += h0; e1 += h1;
      if (i0 < R || i0 + 8 > ny - R) {
        // zero boundary in y: out(i) -= sum_m D(i, m) T(m) over the r rows nearest the edge
        const int lc = cb + 2 * q;
        double c0v = 0.0, c1v = 0.0;
        if (gi < R) {
          const double* dt = DC + (2 * R + gi) * R;
#pragma unroll
          for (int m = 0; m < R; ++m) {
            const double* tr = T + ((base * 8u + (unsigned)(m - rb0)) & 63u) * C::PT + lc;
            c0v = fma(dt[m], tr[0], c0v);
            c1v = fma(dt[m], tr[1], c1v);
          }
        }
        if (gi >= ny - R && gi < ny) {
          const double* db = DC + (3 * R + gi - (ny - R)) * R;
#pragma unroll
          for (int m = 0; m < R; ++m) {
            const double* tr = T + ((base * 8u + (unsigned)(ny - R + m - rb0)) & 63u) * C::PT + lc;
            c0v = fma(db[m], tr[0], c0v);
            c1v = fma(db[m], tr[1], c1v);
          }
        }
        e0 -= c0v;
        e1 -= c1v;
      }
      // ---- epilogue: E_k stencil from the input ring, combine, store, X.Y
      const unsigned uc = base * 8u + (unsigned)(gi - rb0);   // ring row of this output row
      const double* xc = IN + ((uc) & 63u) * C::PX + cb + 2 * q + C::H;
      const double* xu = IN + ((uc - 1u) & 63u) * C::PX + cb + 2 * q + C::H;
      const double* xd = IN + ((uc + 1u) & 63u) * C::PX + cb + 2 * q + C::H;
      const double2 xc2 = *reinterpret_cast<const double2*>(xc);   // 16-byte aligned (even offsets)
      const double x0 = xc2.x, x1 = xc2.y;
      double o0 = e0, o1 = e1;
      if (withE && v0) {
        const double xl = xc[-1], xr = xc[2];
        const double2 xu2 = *reinterpret_cast<const double2*>(xu);
        const double2 xd2 = *reinterpret_cast<const double2*>(xd);
        const double u0 = xu2.x, u1 = xu2.y, d0v = xd2.x, d1v = xd2.y;
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
        dd_add(dot, dlo, fma(x1, o1, x0 * o0), 0.0);
      } else if (v0) {
        ys[(int64_t)gi * nx + gj] = o0;
        dd_add(dot, dlo, x0 * o0, 0.0);
      }
      release(ebars, base, t - C::K, lane);
    }
    // the blocks whose last read was in this item's final steps
    for (int b = nbi - C::K; b < nbi; ++b) release(ebars, base, b, lane);
    ring.pos = base + (unsigned)nbi;
    ring.parity = parity;
    *dot_lo = dlo;
    return dot;
  }

  // this warp is done with block b of the item (ring position base + b)
  __device__ static void release(uint64_t* ebars, unsigned base, int b, int lane) {
    if (b < 0) return;
    __syncwarp();
    if (lane == 0) mbar_arrive(ebars + ((base + (unsigned)b) & 7u));
  }
};

}  // namespace rsk
