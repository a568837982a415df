// Streaming persistent lockstep loop of the batched deflated CG (rsk_cg_recycled_batch)
// for images beyond L2 (C3, C4, C5): DESIGN.md §4.2.
//
// Same recurrences as cg_persist.cu and the oracle O4 (oracle/defcg.py, reading D1):
//
//   A  w = A_gamma p (ACTIVE) or w = A_gamma x (RCONV: true-residual confirm): the strip
//      apply (strip_core.cuh) over balanced 8-row-block ranges of all (shift, strip)
//      columns; one double-double p.w partial per (shift, CTA)            -- barrier
//   B  alpha = rho / p.w (double-double sum of the partials); per CTA row range and pass
//      of <= 16 shifts of one group: r = r - alpha w (or b - w), partial sums of
//      rho' = r.r, zeta = ZGhat.r and z = [AW ; EW]^T r (FP64 tensor cores) -- barrier
//   B2 one CTA per shift: chunk sums in fixed order, mu = G^-1 z, beta, status -- barrier
//   C  x += alpha p ; p = r + beta p - W mu_W - ghat mu_g (W mu on the tensor cores);
//      residual store                                                      -- barrier
//
// Data movement: phases B and C stream the per-shift vectors and the group columns
// straight into DMMA fragment registers (wide B: 32-byte lane loads, 128-byte runs per
// shift / column per warp instruction; C: 16-byte pairs, 128-byte runs), every load of a
// super-step issued before its arithmetic; two 8-warp CTAs per SM, <= 128 registers.
// Every sum has a fixed order that depends only on N and the launch geometry (CTA and
// warp row ranges, nchunk): results per shift do not depend on the other shifts of the
// batch (the N-rank shift-sharded run does the 1-rank work bit for bit).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "strip_core.cuh"

namespace rsk {

constexpr int kSMaxShift = 256;
constexpr int kSPV = kMaxM + 1;     // partial slots per (shift, chunk): z_0..z_{m-1}, rho at kMaxM

__device__ unsigned long long g_sprof[8];   // per-phase ns (RSK_PERSIST_PROF), block 0's view
__device__ unsigned long long g_sprof3[8];
__device__ unsigned long long g_cta_t[1024][8];   // RSK_PERSIST_PROF: per-CTA phase ends of one iteration
__device__ unsigned long long g_sprof2[8];  // block 0, warp 1: B wait ns, B steps, C wait ns, C steps, B step ns, C step ns

struct alignas(64) StreamParams {
  StripParams sp;     // apply: mapX over P (ld N), mapX2 over the iterates X (ld ldx), Y = Wv
  CgDev* cg;
  double* partA;      // [shift][ipv]
  double* partB;      // [shift][kSPV][nchunk]
  unsigned* bar;      // grid barrier {count, generation}
  int* nactive;
  int* iters_done;
  int nshift;
  int nchunk;         // partial slots per shift = the grid (one row range per CTA)
  int64_t rpc;        // rows per CTA (multiple of 128)
  int64_t cg_N;
  int ipv;            // apply items per vector (segments x strips)
  int max_iters;
  int prof;
  int wide;           // 1: phase B in the wide form (32-byte lanes, 128-byte runs)
};

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ unsigned s_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void s_st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long s_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// counting grid barrier (cooperative launch: all CTAs co-resident): bar[0] counts the
// arrivals since the launch (the host zeroes it before every launch); barrier i of the
// launch completes when it reaches i x gridDim. Thread 0 arrives with a fire-and-forget
// release reduction and polls with acquire loads -- one L2 round trip less than the
// sense-reversing form (last arriver resets and releases). Generic and async-proxy (TMA)
// accesses on either side are ordered by the proxy fences.
__device__ __forceinline__ void sgrid_sync(unsigned* bar, unsigned& target) {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    while (s_ld_acquire(bar) < target) {
    }
    __threadfence();
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
  }
  __syncthreads();
}

// Streaming loads of phases B / C carry the L2 prefetch-size hint (.L2::256B: a miss fills
// the aligned 256-byte block, i.e. this warp's next 16-row super-step too -- more bytes in
// flight without registers or prefetch instructions). A/B on one box (session 3): per
// lockstep iteration at 1 / 4 / 16 / 32 shifts 140 / 306 / 585 / 1053 -> 133 / 297 / 575 /
// 1030 us, C4 k = 1 step 12.18 -> 11.93 s. -DRSK_NO_L2PF builds the plain loads.
#ifndef RSK_NO_L2PF
#define RSK_L2PF 1
#define RSK_PF ".L2::256B"
#else
#define RSK_PF ""
#endif
#ifdef RSK_L2PF
__device__ __forceinline__ double2 ld2cg(const double* p) {
  double2 v;
  asm volatile("ld.global.cg" RSK_PF ".v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld2nc(const double* p) {
  double2 v;
  asm volatile("ld.global.nc" RSK_PF ".v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
#else
__device__ __forceinline__ double2 ld2cg(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ld2nc(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
#endif
// group-block loads: read once per pass and CTA range -- L2 only (RSK_GRP_L1 kept them in L1)
#ifdef RSK_GRP_L1
__device__ __forceinline__ double2 ldgrp(const double2* p) { return __ldg(p); }
#else
__device__ __forceinline__ double2 ldgrp(const double2* p) { return ld2cg(reinterpret_cast<const double*>(p)); }
#endif

// ---------------------------------------------------------------- active list
// one int per entry: sid | mode << 9 | grp << 12 | m << 14 | hg << 19
struct SList {
  int n;
  int e[kSMaxShift];
};
__device__ __forceinline__ int le_sid(int v) { return v & 511; }
__device__ __forceinline__ int le_mode(int v) { return (v >> 9) & 7; }
__device__ __forceinline__ int le_grp(int v) { return (v >> 12) & 3; }
__device__ __forceinline__ int le_m(int v) { return (v >> 14) & 31; }
__device__ __forceinline__ int le_hg(int v) { return (v >> 19) & 1; }

// ACTIVE / RCONV shifts sorted by group (passes reuse the group columns); warp 0 compacts
__device__ void s_build_list(const CgDev* cg, int ns, SList& L, int* tmp) {
  for (int s = threadIdx.x; s < ns; s += blockDim.x) tmp[s] = cg->status[s] | (cg->group[s] << 8);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int n = 0;
    for (int g = 0; g < RSK_MAX_GROUPS; ++g)
      for (int s0 = 0; s0 < ns; s0 += 32) {
        const int s = s0 + lane;
        const int v = s < ns ? tmp[s] : -1;
        const int st = v & 0xff;
        const bool in = s < ns && (v >> 8) == g && (st == ST_ACTIVE || st == ST_RCONV);
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) {
          const int pos = n + __popc(bal & ((1u << lane) - 1u));
          L.e[pos] = s | (st << 9) | (g << 12) | (cg->mloc[s] << 14) | (cg->hasg[s] << 19);
        }
        n += __popc(bal);
      }
    if (lane == 0) L.n = n;
  }
  __syncthreads();
}

// passes: up to kSPass consecutive entries of one group
constexpr int kSPass = 16;
__device__ __forceinline__ int s_pass_end(const SList& L, int li0) {
  const int g = le_grp(L.e[li0]);
  int li1 = li0;
  while (li1 < L.n && li1 < li0 + kSPass && le_grp(L.e[li1]) == g) ++li1;
  return li1;
}
// ---------------------------------------------------------------- shared memory plan
// [0, SCRATCH): the strip apply's input / x-pass rings (phase A) or the B / C stages,
// pass accumulators, cross-warp reduction and per-pass scalars (phases B, B2, C);
// [SCRATCH, ...): the strip apply's persistent tail (corrections, mbarriers) + 2 stage
// mbarriers -- never touched by another phase
constexpr int kSPS = 8;        // per pass entry: beta, 1/|r|, slot, flags, alpha
constexpr int kSMaxPass = 24;  // passes per phase (<= 256 shifts / 16 + groups)
constexpr int kRW = 34;        // phase B staging per (warp, shift): zA[16], zE[16], rho, zeta
template <int R>
struct SCfg {
  // phases B, B2, C reuse the strip apply's rings: B's per-warp partials [8][32][kRW], B2's
  // sums and Cholesky factor, C's per-pass scalars [32][kSPS] and mu [32][kMaxM]
  static constexpr int B_END = 8 * 32 * kRW;
  static constexpr int B2_END = 32 + kMaxM * kMaxM;
  static constexpr int C_END = 32 * kSPS + 32 * kMaxM;
  static constexpr int BC_END = B_END > B2_END ? (B_END > C_END ? B_END : C_END) : (B2_END > C_END ? B2_END : C_END);
  static constexpr int RING_END = StripCfg<R>::RING_END;
  static constexpr int SCRATCH = al16(BC_END > RING_END ? BC_END : RING_END);
  using Strip = StripCfg<R, SCRATCH>;
  static constexpr int DBL = Strip::DBL;
  static constexpr size_t SMEM = sizeof(double) * (size_t)DBL;
};

// pass boundaries of the list (pst[0..npass]), computed by every CTA identically
__device__ __forceinline__ int s_passes(const SList& L, int* pst) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int np = 0, li = 0;
    pst[0] = 0;
    while (li < L.n) {
      li = s_pass_end(L, li);
      pst[++np] = li;
    }
    pst[kSMaxPass] = np;
  }
  __syncthreads();
  return pst[kSMaxPass];
}

// ---------------------------------------------------------------- phase A
// The 8-row output blocks of all (active shift, strip) columns are split evenly over the
// CTAs: CTA k owns blocks [k B / G, (k+1) B / G) of the sequence (list entry, strip,
// block), B = n x nstrip x ceil(ny / 8); it runs them as strip items (one per strip its
// range touches) and writes one X.Y partial per (shift, CTA). Balanced to one item
// prologue (LAG blocks) whatever the number of active shifts.
__device__ __forceinline__ int64_t s_nblk(const StripParams& sp) { return (sp.ny + 7) / 8; }
// CTAs whose block range touches list entry li: [k0, k1]
__device__ __forceinline__ void s_cta_span(const StripParams& sp, int n, int li, int G, int& k0, int& k1) {
  const int64_t per = (int64_t)sp.nstrip * s_nblk(sp);
  const int64_t B = per * n;
  const int64_t b0 = per * li, b1 = per * (li + 1) - 1;
  k0 = (int)((b0 * G) / B);
  k1 = (int)((b1 * G) / B);
  // k owns [ceil(k B / G), ceil((k+1) B / G)): adjust for the rounding of the start
  while (k0 > 0 && ((int64_t)k0 * B + G - 1) / G > b0) --k0;
  while (((int64_t)(k0 + 1) * B + G - 1) / G <= b0) ++k0;
  while (k1 < G - 1 && ((int64_t)(k1 + 1) * B + G - 1) / G <= b1) ++k1;
}

template <int R>
__device__ __forceinline__ void s_phase_a(const StreamParams& P, const SList& L, double* smem, StripRing& ring) {
  using Core = StripCore<R, SCfg<R>::SCRATCH>;
  const StripParams& sp = P.sp;
  const int n = L.n;
  const int G = gridDim.x;
  const int64_t nbk = s_nblk(sp);
  const int64_t per = (int64_t)sp.nstrip * nbk;
  const int64_t B = per * n;
  const int k = blockIdx.x;
  int64_t b = ((int64_t)k * B + G - 1) / G;
  const int64_t bend = ((int64_t)(k + 1) * B + G - 1) / G;
  int cur_li = -1;
  // the CTA's p.w partial of the current shift as a double-double (hi at partA[s][k], lo at
  // partA[nshift + s][k]): the shift's total is then the same whatever the block ranges
  double acc = 0.0, acl = 0.0;
  double* partL = P.partA + (size_t)P.nshift * P.ipv;
  if (b == bend && b < B && threadIdx.x == 0) {   // empty range inside an entry's span
    const int li = (int)(b / per);
    if (le_mode(L.e[li]) != ST_RCONV) {
      P.partA[(size_t)le_sid(L.e[li]) * P.ipv + k] = 0.0;
      partL[(size_t)le_sid(L.e[li]) * P.ipv + k] = 0.0;
    }
  }
  while (b < bend) {
    const int li = (int)(b / per);
    const int64_t rem = b - (int64_t)li * per;
    const int strip = (int)(rem / nbk);
    const int blk = (int)(rem - (int64_t)strip * nbk);
    const int64_t e = imin64(bend, (int64_t)li * per + (int64_t)(strip + 1) * nbk);
    const int blk1 = (int)(e - (int64_t)li * per - (int64_t)strip * nbk);
    const int v = L.e[li];
    const int s = le_sid(v);
    const bool rconv = le_mode(v) == ST_RCONV;
    if (li != cur_li) {
      if (cur_li >= 0 && le_mode(L.e[cur_li]) != ST_RCONV && threadIdx.x == 0) {
        P.partA[(size_t)le_sid(L.e[cur_li]) * P.ipv + k] = acc;
        partL[(size_t)le_sid(L.e[cur_li]) * P.ipv + k] = acl;
      }
      cur_li = li;
      acc = 0.0;
      acl = 0.0;
    }
    double lo;
    double dot = Core::item(sp, smem, ring, s, strip, 8 * blk, (int)imin64(sp.ny, 8 * (int64_t)blk1), rconv, &lo);
    if (!rconv) {
      block_sum_dd(dot, lo, smem + SCfg<R>::Strip::OFF_RED);
      dd_add(acc, acl, dot, lo);   // thread 0: the CTA's items of this shift
    }
    b = e;
  }
  if (cur_li >= 0 && le_mode(L.e[cur_li]) != ST_RCONV && threadIdx.x == 0) {
    P.partA[(size_t)le_sid(L.e[cur_li]) * P.ipv + k] = acc;
    partL[(size_t)le_sid(L.e[cur_li]) * P.ipv + k] = acl;
  }
}

// ---------------------------------------------------------------- phase B
// ---------------------------------------------------------------- phase B (register form)
// The per-shift vectors stream through registers: lane (g, q) updates r of (row q of a
// 4-row k-step, shift 8 nb + g) -- exactly its DMMA B fragment -- and loads the A
// fragments (group columns 8 mb + g, row q) of AW / EW, shared by the four 8-shift N
// blocks of a pass of <= 32 shifts. Every load of a group of k-steps is issued before
// the arithmetic that consumes it. Partials per (shift, CTA row range), fixed order.
template <int R>
__device__ void s_phase_b_reg(const StreamParams& P, const SList& L, double* smem, double* s_alpha, int* pst,
                              CgDev* cg) {
  const int n = L.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t N = cg->N;
  for (int li = warp; li < n; li += 8) {
    const int v = L.e[li];
    double a = 0.0;
    if (le_mode(v) == ST_ACTIVE) {
      const int s = le_sid(v);
      const double* pa = P.partA + (size_t)s * P.ipv;
      const double* pl = P.partA + (size_t)(P.nshift + s) * P.ipv;
      int k0, k1;
      s_cta_span(P.sp, n, li, gridDim.x, k0, k1);
      double pi = 0.0, pil = 0.0;
      for (int c = k0 + lane; c <= k1; c += 32) dd_add(pi, pil, __ldcg(pa + c), __ldcg(pl + c));
      warp_sum_dd(pi, pil);
      if (!(pi > 0.0) || !isfinite(pi)) {
        if (blockIdx.x == 0 && lane == 0) { cg->status[s] = ST_BREAKDOWN; cg->alpha[s] = 0.0; }
      } else {
        a = cg->rho[s] / pi;
        if (blockIdx.x == 0 && lane == 0) cg->alpha[s] = a;
      }
    }
    if (lane == 0) s_alpha[li] = a;
  }
  const int npass = s_passes(L, pst);
  const int64_t cbeg = (int64_t)blockIdx.x * P.rpc;
  const int64_t cend = imin64(N, cbeg + P.rpc);
  double* red = smem;   // [8 warps][32][kRW]
  const int64_t rpw = P.rpc / 8;   // rows per warp (multiple of 8)
  const int64_t wbeg = cbeg + warp * rpw;
  const int64_t wend = imin64(cend, wbeg + rpw);
  for (int pk = 0; pk < npass; ++pk) {
    const int li0 = pst[pk], li1 = pst[pk + 1];
    const int np = li1 - li0;
    const int grp = le_grp(L.e[li0]);
    const int J = cg->grp.J[grp];
    const double* AWg = cg->grp.AW[grp];
    const double* EWg = cg->grp.EW[grp];
    const int64_t ldw = cg->grp.ldw;
    int sv[2], md[2], hgv[2];
    double al[2];
    bool ok[2];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const int li = li0 + 8 * nb + g;
      ok[nb] = li < li1;
      const int v = ok[nb] ? L.e[li] : 0;
      sv[nb] = le_sid(v);
      md[nb] = ok[nb] ? le_mode(v) : ST_ACTIVE;
      hgv[nb] = ok[nb] ? le_hg(v) : 0;
      al[nb] = ok[nb] ? s_alpha[li] : 0.0;
    }
    double dA[2][2][2], dE[2][2][2], rh[2], zt[2];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      rh[nb] = 0.0; zt[nb] = 0.0;
#pragma unroll
      for (int mb = 0; mb < 2; ++mb) { dA[nb][mb][0] = dA[nb][mb][1] = dE[nb][mb][0] = dE[nb][mb][1] = 0.0; }
    }
    const int nbn = (np + 7) >> 3;
    // 8-row super-steps: lane (g, q) loads rows 2q, 2q+1 as one 16-byte pair (64-byte runs
    // per column / shift across the four q lanes); k-step t of the two uses row 2q + t --
    // the same row permutation on A and B, so D sums over all 8 rows
#pragma unroll 2
    for (int64_t row0 = wbeg; row0 < wend; row0 += 8) {
      const int64_t row = row0 + 2 * q;
      const bool vr = row < wend;           // wend - row0 is a multiple of 8 except at N
      const bool vr1 = row + 1 < wend;
      double2 aA[2], aE[2], wv[2], rv[2], zg[2];
#pragma unroll
      for (int mb = 0; mb < 2; ++mb) {
        const int col = 8 * mb + g;
        const bool va = vr && col < J;
        aA[mb] = va ? ldgrp(reinterpret_cast<const double2*>(AWg + (int64_t)col * ldw + row)) : make_double2(0.0, 0.0);
        aE[mb] = va ? ldgrp(reinterpret_cast<const double2*>(EWg + (int64_t)col * ldw + row)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        wv[nb] = rv[nb] = zg[nb] = make_double2(0.0, 0.0);
        if (nb < nbn && ok[nb] && vr) {
          const int64_t o = (int64_t)sv[nb] * N + row;
          wv[nb] = __ldcg(reinterpret_cast<const double2*>(cg->Wv + o));
          rv[nb] = (md[nb] == ST_ACTIVE) ? __ldcg(reinterpret_cast<const double2*>(cg->R + o))
                                         : __ldg(reinterpret_cast<const double2*>(cg->b + row));
          if (hgv[nb]) zg[nb] = __ldg(reinterpret_cast<const double2*>(cg->ZGhat + (int64_t)sv[nb] * cg->ldgh + row));
        }
      }
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        if (nb >= nbn) break;                  // uniform across the warp
        double2 rn = make_double2(0.0, 0.0);
        if (ok[nb] && vr) {
          if (md[nb] == ST_ACTIVE) {
            rn.x = fma(-al[nb], wv[nb].x, rv[nb].x);
            rn.y = fma(-al[nb], wv[nb].y, rv[nb].y);
          } else {
            rn.x = rv[nb].x - wv[nb].x;
            rn.y = rv[nb].y - wv[nb].y;
          }
          if (!vr1) rn.y = 0.0;
          double* rp = cg->R + (int64_t)sv[nb] * N + row;
          if (vr1) *reinterpret_cast<double2*>(rp) = rn;
          else rp[0] = rn.x;
          rh[nb] = fma(rn.x, rn.x, rh[nb]);
          rh[nb] = fma(rn.y, rn.y, rh[nb]);
          zt[nb] = fma(zg[nb].x, rn.x, zt[nb]);
          zt[nb] = fma(zg[nb].y, rn.y, zt[nb]);
        }
        dmma(dA[nb][0][0], dA[nb][0][1], aA[0].x, rn.x);
        dmma(dE[nb][0][0], dE[nb][0][1], aE[0].x, rn.x);
        dmma(dA[nb][0][0], dA[nb][0][1], aA[0].y, rn.y);
        dmma(dE[nb][0][0], dE[nb][0][1], aE[0].y, rn.y);
        if (J > 8) {
          dmma(dA[nb][1][0], dA[nb][1][1], aA[1].x, rn.x);
          dmma(dE[nb][1][0], dE[nb][1][1], aE[1].x, rn.x);
          dmma(dA[nb][1][0], dA[nb][1][1], aA[1].y, rn.y);
          dmma(dE[nb][1][0], dE[nb][1][1], aE[1].y, rn.y);
        }
      }
    }
    // stage: D[m = 8 mb + g][n = 2q, 2q+1] of N-block nb; rho / zeta summed over the q lanes
    double* rw = red + (size_t)warp * 32 * kRW;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      if (nb >= nbn) break;
      double r1 = rh[nb], z1 = zt[nb];
      r1 += __shfl_xor_sync(0xffffffffu, r1, 1);
      r1 += __shfl_xor_sync(0xffffffffu, r1, 2);
      z1 += __shfl_xor_sync(0xffffffffu, z1, 1);
      z1 += __shfl_xor_sync(0xffffffffu, z1, 2);
      if (q == 0) {
        rw[(8 * nb + g) * kRW + 32] = r1;
        rw[(8 * nb + g) * kRW + 33] = z1;
      }
#pragma unroll
      for (int mb = 0; mb < 2; ++mb) {
        const int m = 8 * mb + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int sh = 8 * nb + 2 * q + h;
          rw[sh * kRW + m] = dA[nb][mb][h];
          rw[sh * kRW + 16 + m] = dE[nb][mb][h];
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < np * kSPV; e += blockDim.x) {
      const int k = e / kSPV, j = e - k * kSPV;
      const int v = L.e[li0 + k];
      const int nw = le_m(v) - le_hg(v);
      const bool isz = j < nw, isg = le_hg(v) && j == nw, isr = j == kMaxM;
      if (!(isz || isg || isr)) continue;
      double ta = 0.0, te = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const double* r = red + ((size_t)w * 32 + k) * kRW;
        if (isz) { ta += r[j]; te += r[16 + j]; }
        else ta += r[isr ? 32 : 33];
      }
      const int s = le_sid(v);
      const double val = isz ? fma(cg->gam[s], te, ta) : ta;
      P.partB[((size_t)s * kSPV + j) * P.nchunk + blockIdx.x] = val;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- phase B (wide form)
// Same sums as s_phase_b_reg with 16-row super-steps and 32-byte lane loads: lane (g, q)
// loads rows 4q..4q+3 of shift 8 nb + g (w, r, zg) and of column 8 mt + g of the
// concatenated group block [AW | EW] (2J columns, NMT = ceil(2J / 8) m-tiles); k-step t of
// the four uses row 4q + t on both operands. Each shift / column then moves as one
// 128-byte run per warp instruction -- the 64-byte runs of the 8-row form cap the phase
// near 3 TB/s (tools/stream_bw.cu: 64-byte runs 2.6-3.1 TB/s, 128-byte 5.4-6.3 TB/s).
// Needs N, ldw, ldgh multiples of 4 and 32-byte aligned vectors (launch_cg_stream).
__device__ __forceinline__ void ld4cg(const double* p, double* v) {
  asm volatile("ld.global.cg" RSK_PF ".v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void ld4nc(const double* p, double* v) {
  asm volatile("ld.global.nc" RSK_PF ".v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double* v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}
// Every warp streams its fixed eighth of the CTA's rows (rpc / 8, a multiple of 16) for
// all NB <= 2 N blocks of the pass, so a shift's sums run over the same rows in the same
// order whatever the pass composition (batch-composition invariance, as every other sum
// of the loop); all loads of a 16-row super-step are issued before its arithmetic.
template <int NMT>
__device__ void s_phase_b_wide_pass(const StreamParams& P, const SList& L, double* red, const double* s_alpha,
                                    int li0, int li1, CgDev* cg, int64_t wbeg, int64_t wend) {
  constexpr int NB = 2;
  const int nbn = (li1 - li0 + 7) >> 3;   // N blocks of this pass (1 or 2)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t N = cg->N;
  const int np = li1 - li0;
  const int grp = le_grp(L.e[li0]);
  const int J = cg->grp.J[grp];
  const int64_t ldw = cg->grp.ldw;
  // column 8 mt + g of [AW | EW]
  const double* colp[NMT];
  bool colv[NMT];
#pragma unroll
  for (int mt = 0; mt < NMT; ++mt) {
    const int c = 8 * mt + g;
    colv[mt] = c < 2 * J;
    colp[mt] = colv[mt] ? (c < J ? cg->grp.AW[grp] + (int64_t)c * ldw : cg->grp.EW[grp] + (int64_t)(c - J) * ldw)
                        : cg->grp.AW[grp];
  }
  // per N block: shift id << 3 | flags (bit 0: in the pass, 1: ACTIVE (else RCONV:
  // r = b - w), 2: has ghat); alpha is re-read from shared memory where it is used
  unsigned sf[NB];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    const int li = li0 + 8 * nb + g;
    const bool ok = li < li1;
    const int v = ok ? L.e[li] : 0;
    sf[nb] = ok ? ((unsigned)le_sid(v) << 3 | 1u | (le_mode(v) == ST_ACTIVE ? 2u : 0u) | (le_hg(v) ? 4u : 0u)) : 2u;
  }
  double dz[NB][NMT][2], rh[NB], zt[NB];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    rh[nb] = 0.0; zt[nb] = 0.0;
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt) dz[nb][mt][0] = dz[nb][mt][1] = 0.0;
  }
#pragma unroll 1
  for (int64_t row0 = wbeg; row0 < wend; row0 += 16) {
    const int64_t row = row0 + 4 * q;
    const bool vr = row < wend;   // N % 4 == 0: the 4 rows are all valid or all beyond
    double a[NMT][4];
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt) {
      if (vr && colv[mt]) ld4cg(colp[mt] + row, a[mt]);
      else a[mt][0] = a[mt][1] = a[mt][2] = a[mt][3] = 0.0;
    }
    // the N blocks one after the other (the asm-volatile loads / DMMAs keep their order):
    // one block's vectors in registers at a time, the group fragments shared
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      if (nb >= nbn) break;   // uniform across the CTA
      double wv[4], rv[4], zg[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) wv[t] = rv[t] = zg[t] = 0.0;
      const bool lv = (sf[nb] & 1u) && vr;
      if (lv) {
        const int64_t sd = (int64_t)(sf[nb] >> 3);
        ld4cg(cg->Wv + sd * N + row, wv);
        if (sf[nb] & 2u) ld4cg(cg->R + sd * N + row, rv);
        else ld4nc(cg->b + row, rv);
        if (sf[nb] & 4u) ld4nc(cg->ZGhat + sd * cg->ldgh + row, zg);
      }
      double rn[4] = {0.0, 0.0, 0.0, 0.0};
      if (lv) {
        const double al = s_alpha[li0 + 8 * nb + g];
#pragma unroll
        for (int t = 0; t < 4; ++t) rn[t] = (sf[nb] & 2u) ? fma(-al, wv[t], rv[t]) : rv[t] - wv[t];
        st4(cg->R + (int64_t)(sf[nb] >> 3) * N + row, rn);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          rh[nb] = fma(rn[t], rn[t], rh[nb]);
          zt[nb] = fma(zg[t], rn[t], zt[nb]);
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt) dmma(dz[nb][mt][0], dz[nb][mt][1], a[mt][t], rn[t]);
    }
  }
  // stage: warp's D[c = 8 mt + g][n = 2q, 2q+1] of N block nb (c < J: zA[c], else zE[c - J])
  double* rw = red + (size_t)warp * 32 * kRW;
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    if (nb >= nbn) break;
    double r1 = rh[nb], z1 = zt[nb];
    r1 += __shfl_xor_sync(0xffffffffu, r1, 1);
    r1 += __shfl_xor_sync(0xffffffffu, r1, 2);
    z1 += __shfl_xor_sync(0xffffffffu, z1, 1);
    z1 += __shfl_xor_sync(0xffffffffu, z1, 2);
    if (q == 0) {
      rw[(8 * nb + g) * kRW + 32] = r1;
      rw[(8 * nb + g) * kRW + 33] = z1;
    }
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt) {
      const int c = 8 * mt + g;
      if (c >= 2 * J) continue;
      const int off = c < J ? c : 16 + (c - J);
#pragma unroll
      for (int h = 0; h < 2; ++h) rw[(8 * nb + 2 * q + h) * kRW + off] = dz[nb][mt][h];
    }
  }
  __syncthreads();
  for (int e = tid; e < np * kSPV; e += blockDim.x) {
    const int k = e / kSPV, j = e - k * kSPV;
    const int v2 = L.e[li0 + k];
    const int nw = le_m(v2) - le_hg(v2);
    const bool isz = j < nw, isg = le_hg(v2) && j == nw, isr = j == kMaxM;
    if (!(isz || isg || isr)) continue;
    double ta = 0.0, te = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const double* r = red + ((size_t)w * 32 + k) * kRW;
      if (isz) { ta += r[j]; te += r[16 + j]; }
      else ta += r[isr ? 32 : 33];
    }
    const int s2 = le_sid(v2);
    const double val = isz ? fma(cg->gam[s2], te, ta) : ta;
    P.partB[((size_t)s2 * kSPV + j) * P.nchunk + blockIdx.x] = val;
  }
  __syncthreads();
}

template <int R>
__device__ void s_phase_b_wide(const StreamParams& P, const SList& L, double* smem, double* s_alpha, int* pst,
                               CgDev* cg) {
  const int n = L.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t N = cg->N;
  for (int li = warp; li < n; li += 8) {
    const int v = L.e[li];
    double a = 0.0;
    if (le_mode(v) == ST_ACTIVE) {
      const int s = le_sid(v);
      const double* pa = P.partA + (size_t)s * P.ipv;
      const double* pl = P.partA + (size_t)(P.nshift + s) * P.ipv;
      int k0, k1;
      s_cta_span(P.sp, n, li, gridDim.x, k0, k1);
      double pi = 0.0, pil = 0.0;
      for (int c = k0 + lane; c <= k1; c += 32) dd_add(pi, pil, __ldcg(pa + c), __ldcg(pl + c));
      warp_sum_dd(pi, pil);
      if (!(pi > 0.0) || !isfinite(pi)) {
        if (blockIdx.x == 0 && lane == 0) { cg->status[s] = ST_BREAKDOWN; cg->alpha[s] = 0.0; }
      } else {
        a = cg->rho[s] / pi;
        if (blockIdx.x == 0 && lane == 0) cg->alpha[s] = a;
      }
    }
    if (lane == 0) s_alpha[li] = a;
  }
  const int npass = s_passes(L, pst);
  const int64_t cbeg = (int64_t)blockIdx.x * P.rpc;
  const int64_t cend = imin64(N, cbeg + P.rpc);
  const int64_t rpw = P.rpc / 8;   // rows per warp (multiple of 16)
  const int64_t wbeg = cbeg + warp * rpw;
  const int64_t wend = imin64(cend, wbeg + rpw);
  for (int pk = 0; pk < npass; ++pk) {
    const int li0 = pst[pk], li1 = pst[pk + 1];
    const int J = cg->grp.J[le_grp(L.e[li0])];
    const int nmt = (2 * J + 7) >> 3;
    if (nmt <= 1) s_phase_b_wide_pass<1>(P, L, smem, s_alpha, li0, li1, cg, wbeg, wend);
    else if (nmt == 2) s_phase_b_wide_pass<2>(P, L, smem, s_alpha, li0, li1, cg, wbeg, wend);
    else if (nmt == 3) s_phase_b_wide_pass<3>(P, L, smem, s_alpha, li0, li1, cg, wbeg, wend);
    else s_phase_b_wide_pass<4>(P, L, smem, s_alpha, li0, li1, cg, wbeg, wend);
  }
}

// ---------------------------------------------------------------- phase C (register form)
// x += alpha p; p = r + beta p - W mu_W - ghat mu_g. W mu of a pass on the tensor cores:
// an 8-row block x 8 shifts is D = W[8 x J] M[J x 8] (B = the shifts' mu); lane (g, q)
// finishes the elements (row g, shifts 2q, 2q+1) of each N-block.
template <int R>
__device__ void s_phase_c_reg(const StreamParams& P, const SList& L, double* smem, const double* s_alpha, int* pst,
                              CgDev* cg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t N = cg->N;
  const int npass = s_passes(L, pst);
  const int64_t cbeg = (int64_t)blockIdx.x * P.rpc;
  const int64_t cend = imin64(N, cbeg + P.rpc);
  const int64_t rpw = P.rpc / 8;
  const int64_t wbeg = cbeg + warp * rpw;
  const int64_t wend = imin64(cend, wbeg + rpw);
  double* PS = smem;   // [32][kSPS]: beta, 1/|r|, slot, flags, alpha, mu_g
  double* MU = smem + 32 * kSPS;   // [32][kMaxM]
  for (int pk = 0; pk < npass; ++pk) {
    const int li0 = pst[pk], li1 = pst[pk + 1];
    const int np = li1 - li0;
    const int grp = le_grp(L.e[li0]);
    const int J = cg->grp.J[grp];
    const double* Wg = cg->grp.W[grp];
    const int64_t ldw = cg->grp.ldw;
    __syncthreads();   // the previous pass's PS / MU readers are done
    if (tid < np) {
      const int li = li0 + tid;
      const int v = L.e[li];
      const int s = le_sid(v);
      const int st = cg->status[s];
      const int slot = (st == ST_ACTIVE) ? cg->stslot[s] : -1;
      int f = 0;
      if (le_mode(v) == ST_ACTIVE && s_alpha[li] != 0.0) f |= 1;
      if (st == ST_ACTIVE) f |= 2;
      double* ps = PS + tid * kSPS;
      ps[0] = cg->beta[s];
      ps[1] = (slot >= 0) ? 1.0 / sqrt(cg->rho[s]) : 0.0;
      ps[2] = (double)slot;
      ps[3] = (double)f;
      ps[4] = s_alpha[li];
      const int m = le_m(v);
      ps[5] = m > 0 ? cg->coef[(int64_t)s * kMaxM + m - 1] : 0.0;
    }
    for (int e = tid; e < np * kMaxM; e += blockDim.x) {
      const int k = e / kMaxM, j = e - k * kMaxM;
      MU[e] = cg->coef[(int64_t)le_sid(L.e[li0 + k]) * kMaxM + j];
    }
    __syncthreads();
    // B fragments: mu of shift 8 nb + g, component 4 kk + q (0 beyond its nw or w/o new p)
    double bm[2][4];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const int k = 8 * nb + g;
      const bool okk = k < np && (((int)PS[k * kSPS + 3]) & 2);
      const int nw = okk ? le_m(L.e[li0 + k]) - le_hg(L.e[li0 + k]) : 0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int j = 4 * kk + q;
        bm[nb][kk] = (okk && j < nw) ? MU[k * kMaxM + j] : 0.0;
      }
    }
    const int nkk = (J + 3) >> 2;
    const int nbn = (np + 7) >> 3;
    int flg[2][2];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 8 * nb + 2 * q + h;
        flg[nb][h] = k < np ? (int)PS[k * kSPS + 3] : 0;
      }
    // 16-row blocks: lane (g, q) owns rows 2g, 2g+1 (one 16-byte pair: 128-byte runs per
    // column / shift across the eight g lanes); two DMMAs per k-step, one per row parity
#pragma unroll 1
    for (int64_t row0 = wbeg; row0 < wend; row0 += 16) {
      const int64_t row = row0 + 2 * g;
      const bool vr = row < wend;            // rows come in pairs (N even)
      double2 a[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int j = 4 * kk + q;
        a[kk] = (vr && kk < nkk && j < J) ? ldgrp(reinterpret_cast<const double2*>(Wg + (int64_t)j * ldw + row))
                                          : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        if (nb >= nbn) break;
        double2 pv[2], rv[2], xv[2], gv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          pv[h] = rv[h] = xv[h] = gv[h] = make_double2(0.0, 0.0);
          const int f = vr ? flg[nb][h] : 0;
          if (f) {
            const int k = 8 * nb + 2 * q + h;
            const int v = L.e[li0 + k];
            const int s = le_sid(v);
            const int64_t o = (int64_t)s * N + row;
            pv[h] = ld2cg(cg->P + o);
            if (f & 1) xv[h] = ld2cg(cg->X + (int64_t)s * cg->ldx + row);
            if (f & 2) {
              rv[h] = ld2cg(cg->R + o);
              if (le_hg(v)) gv[h] = ld2nc(cg->Ghat + (int64_t)s * cg->ldgh + row);
            }
          }
        }
        double de[2] = {0.0, 0.0}, dd[2] = {0.0, 0.0};   // rows 2g (even) and 2g+1 (odd)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (kk < nkk) {
            dmma(de[0], de[1], a[kk].x, bm[nb][kk]);
            dmma(dd[0], dd[1], a[kk].y, bm[nb][kk]);
          }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int f = vr ? flg[nb][h] : 0;
          if (!f) continue;
          const int k = 8 * nb + 2 * q + h;
          const int v = L.e[li0 + k];
          const int s = le_sid(v);
          const double* ps = PS + k * kSPS;
          if (f & 1) {
            double2 xn;
            xn.x = fma(ps[4], pv[h].x, xv[h].x);
            xn.y = fma(ps[4], pv[h].y, xv[h].y);
            *reinterpret_cast<double2*>(cg->X + (int64_t)s * cg->ldx + row) = xn;
          }
          if (f & 2) {
            double2 pn;
            pn.x = fma(ps[0], pv[h].x, rv[h].x) - de[h];
            pn.y = fma(ps[0], pv[h].y, rv[h].y) - dd[h];
            if (le_hg(v)) {
              pn.x = fma(-ps[5], gv[h].x, pn.x);
              pn.y = fma(-ps[5], gv[h].y, pn.y);
            }
            *reinterpret_cast<double2*>(cg->P + (int64_t)s * N + row) = pn;
            const int sl = (int)ps[2];
            if (sl >= 0) {
              double* st = cg->store + ((int64_t)s * cg->store_cap + sl) * cg->lds + row;
              st[0] = rv[h].x * ps[1];
              st[1] = rv[h].y * ps[1];
            }
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- phase B2
__device__ void s_phase_b2(const StreamParams& P, const SList& L, double* smem, CgDev* cg) {
  const int n = L.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* zs = smem;
  double* Ls = smem + 32;
  for (int li = blockIdx.x; li < n; li += gridDim.x) {
    const int v = L.e[li];
    const int s = le_sid(v);
    const int mode0 = le_mode(v);
    const int m = le_m(v);
    const double* Lg = cg->Lf + (int64_t)s * kMaxM * kMaxM;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = e / m, j = e - i * m;
      if (j <= i) Ls[i * kMaxM + j] = Lg[i + j * kMaxM];
    }
    for (int j = warp; j < kSPV; j += 8) {
      if (j < m || j == kMaxM) {
        // all ten loads of a lane in flight at once (one L2 round trip per 320 chunks)
        const double* pj = P.partB + ((size_t)s * kSPV + j) * P.nchunk;
        double t = 0.0;
        for (int c0 = 0; c0 < P.nchunk; c0 += 320) {
          double v[10];
#pragma unroll
          for (int i = 0; i < 10; ++i) {
            const int c = c0 + lane + 32 * i;
            v[i] = c < P.nchunk ? __ldcg(pj + c) : 0.0;
          }
          t += (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) + (v[8] + v[9]);
        }
        t = warp_sum(t);
        if (lane == 0) zs[j] = t;
      }
    }
    __syncthreads();
    if (warp == 0) {
      // status by lane 0; the two triangular solves with G = L L^T by the warp (lane i =
      // row i, column-oriented substitution: no local arrays, no spills)
      int nst = 0, newp = 0;
      if (lane == 0) {
        const double rho_new = zs[kMaxM];
        const int st = cg->status[s];
        const double thr = cg->tol * cg->bnorm;
        const bool conv = sqrt(rho_new) <= thr;
        nst = st;
        if (mode0 == ST_ACTIVE) {
          if (st == ST_ACTIVE) {
            const int itn = cg->iters[s] + 1;
            cg->iters[s] = itn;
            cg->beta[s] = rho_new / cg->rho[s];
            cg->rho[s] = rho_new;
            if (conv) nst = ST_RCONV;
            else if (itn >= cg->maxit) nst = ST_MAXIT;
            else newp = 1;
          }
        } else {
          cg->rho_true[s] = rho_new;
          cg->nconf[s] += 1;
          cg->alpha[s] = 0.0;
          if (conv) nst = ST_DONE;
          else if (cg->iters[s] >= cg->maxit) nst = ST_MAXIT;
          else {
            nst = ST_ACTIVE;
            cg->beta[s] = 0.0;
            cg->rho[s] = rho_new;
            newp = 1;
          }
        }
      }
      newp = __shfl_sync(0xffffffffu, newp, 0);
      if (newp) {
        const int i = lane;
        double t = (i < m) ? zs[i] : 0.0;
        // forward: L y = z
        for (int j = 0; j < m; ++j) {
          const double xj = __shfl_sync(0xffffffffu, t, j) / Ls[j * kMaxM + j];
          if (i == j) t = xj;
          else if (i > j && i < m) t = fma(-Ls[i * kMaxM + j], xj, t);
        }
        // backward: L^T x = y
        for (int j = m - 1; j >= 0; --j) {
          const double xj = __shfl_sync(0xffffffffu, t, j) / Ls[j * kMaxM + j];
          if (i == j) t = xj;
          else if (i < j) t = fma(-Ls[j * kMaxM + i], xj, t);
        }
        if (i < kMaxM) cg->coef[(int64_t)s * kMaxM + i] = i < m ? t : 0.0;
        if (lane == 0) {
          int slot = -1;
          if (cg->store && cg->store_cnt[s] < cg->store_cap) {
            slot = cg->store_cnt[s];
            cg->store_cnt[s] = slot + 1;
          }
          cg->stslot[s] = slot;
        }
      }
      if (lane == 0) cg->status[s] = nst;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- the kernel
template <int R>
__global__ void __launch_bounds__(kAT, kStripCtasPerSm) cg_stream_kernel(const __grid_constant__ StreamParams P) {
  extern __shared__ __align__(128) double smem[];
  using SC = SCfg<R>;
  using Core = StripCore<R, SC::SCRATCH>;
  __shared__ SList lists[2];
  __shared__ int tmp[kSMaxShift];
  __shared__ double s_alpha[kSMaxShift];
  __shared__ int pst[kSMaxPass + 1];
  // the loop state's pointers and sizes in shared memory (the struct itself never changes;
  // the arrays it points to do): no global round trip per field access after the L1
  // invalidations of the grid barriers
  __shared__ CgDev s_cg;
  if (threadIdx.x == 0) s_cg = *P.cg;

  CgDev* cg = &s_cg;
  const int ns = P.nshift;
  const int tid = threadIdx.x;
  Core::init(smem, P.sp);
  StripRing ring{0u, 0u};
  unsigned gen = 0u;   // barrier target (bar[0] is zeroed before the launch)
  int cur = 0;
  s_build_list(cg, ns, lists[0], tmp);
  sgrid_sync(P.bar, gen);

  int it = 0;
  unsigned long long t0 = 0;
  auto mark = [&](int ph) {
    if (P.prof && tid == 0 && it == 30 && ph != 1 && ph != 7) g_cta_t[blockIdx.x][ph] = s_timer();
    if (P.prof && tid == 0 && it == 30 && ph == 1) g_cta_t[blockIdx.x][5 + (g_cta_t[blockIdx.x][6] ? 1 : 0)] = s_timer();
    if (P.prof && blockIdx.x == 0 && tid == 0) {
      const unsigned long long t1 = s_timer();
      if (t0) g_sprof[ph] += t1 - t0;
      t0 = t1;
    }
  };
  mark(7);
  for (; it < P.max_iters; ++it) {
    SList& L = lists[cur];
    if (L.n == 0) break;
    s_phase_a<R>(P, L, smem, ring);
    mark(0);
    sgrid_sync(P.bar, gen);
    mark(1);
    if (P.wide) s_phase_b_wide<R>(P, L, smem, s_alpha, pst, &s_cg);
    else s_phase_b_reg<R>(P, L, smem, s_alpha, pst, &s_cg);
    mark(2);
    sgrid_sync(P.bar, gen);
    mark(1);
    s_phase_b2(P, L, smem, &s_cg);
    mark(3);
    sgrid_sync(P.bar, gen);
    mark(1);
    SList& NL = lists[cur ^ 1];
    s_build_list(cg, ns, NL, tmp);   // statuses are stable until the next phase A
    s_phase_c_reg<R>(P, L, smem, s_alpha, pst, &s_cg);
    mark(4);
    sgrid_sync(P.bar, gen);
    mark(1);
    if (P.prof && blockIdx.x == 0 && tid == 0) g_sprof[5] += 1;
    cur ^= 1;
  }
  if (blockIdx.x == 0 && tid == 0) {
    *P.nactive = lists[cur].n;
    *P.iters_done = it;
  }
}

// ---------------------------------------------------------------- the skewed kernel
// RSK_STREAM_SKEW=1 (session 4). The lockstep loop above runs a compute-bound phase (A: the
// apply on the FP64 tensor cores, 16 B/px of DRAM traffic) and two DRAM-bound phases (B, C)
// one after the other, so the DMMA pipe idles in B / C and HBM idles in A. Here the active
// shifts of a launch are split into two halves H0 / H1 (contiguous in the group-sorted
// list) and H1 runs one slot behind H0:
//     slot 1: B(H0) | A(H1)     slot 2: B2(H0) | B(H1)
//     slot 3: C(H0) | B2(H1)    slot 4: A(H0, next iteration) | C(H1)
// In slots 1 and 4 the CTAs of one SM take the two tasks in opposite order (one streams
// while the other computes). Every per-shift operation, sum order and partial slot is the
// one of the lockstep kernel (the phases are batch-composition invariant), so the results
// are bitwise the same; the price is that a group's blocks are read once per half.
__device__ unsigned g_smslot[512];
constexpr int kSkewDefault = 0;   // RSK_STREAM_SKEW overrides
// between the two tasks of a slot: the next task may reuse the shared scratch through the
// other proxy (TMA ring of phase A vs generic stores of B / B2 / C)
__device__ __forceinline__ void s_task_switch() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
}

__device__ void s_build_list_half(const CgDev* cg, int ns, SList& L, int* tmp, const unsigned char* half, int h) {
  for (int s = threadIdx.x; s < ns; s += blockDim.x) tmp[s] = cg->status[s] | (cg->group[s] << 8);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int n = 0;
    for (int g = 0; g < RSK_MAX_GROUPS; ++g)
      for (int s0 = 0; s0 < ns; s0 += 32) {
        const int s = s0 + lane;
        const int v = s < ns ? tmp[s] : -1;
        const int st = v & 0xff;
        const bool in = s < ns && (v >> 8) == g && (st == ST_ACTIVE || st == ST_RCONV) && half[s] == h;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) {
          const int pos = n + __popc(bal & ((1u << lane) - 1u));
          L.e[pos] = s | (st << 9) | (g << 12) | (cg->mloc[s] << 14) | (cg->hasg[s] << 19);
        }
        n += __popc(bal);
      }
    if (lane == 0) L.n = n;
  }
  __syncthreads();
}

template <int R>
__global__ void __launch_bounds__(kAT, kStripCtasPerSm) cg_stream_skew_kernel(const __grid_constant__ StreamParams P) {
  extern __shared__ __align__(128) double smem[];
  using SC = SCfg<R>;
  using Core = StripCore<R, SC::SCRATCH>;
  __shared__ SList lists[2][2];
  __shared__ int tmp[kSMaxShift];
  __shared__ double s_alpha[2][kSMaxShift];
  __shared__ int pst[kSMaxPass + 1];
  __shared__ unsigned char half[kSMaxShift];
  __shared__ int s_flip;
  __shared__ CgDev s_cg;
  if (threadIdx.x == 0) {
    s_cg = *P.cg;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    s_flip = (int)(atomicAdd(&g_smslot[smid & 511u], 1u) & 1u);
  }
  CgDev* cg = &s_cg;
  const int ns = P.nshift;
  const int tid = threadIdx.x;
  Core::init(smem, P.sp);
  StripRing ring{0u, 0u};
  unsigned gen = 0u;
  // the launch's split: first half of the group-sorted active list -> H0, the rest -> H1
  s_build_list(cg, ns, lists[0][0], tmp);
  {
    const SList& F = lists[0][0];
    const int n0 = (F.n + 1) >> 1;
    for (int li = tid; li < F.n; li += blockDim.x) half[le_sid(F.e[li])] = li < n0 ? 0 : 1;
  }
  __syncthreads();
  const bool flip = s_flip != 0;
  s_build_list_half(cg, ns, lists[1][0], tmp, half, 1);
  s_build_list_half(cg, ns, lists[0][0], tmp, half, 0);
  sgrid_sync(P.bar, gen);

  int it = 0;
  unsigned long long t0 = 0;
  auto mark = [&](int ph) {
    if (P.prof && blockIdx.x == 0 && tid == 0) {
      const unsigned long long t1 = s_timer();
      if (t0) g_sprof[ph] += t1 - t0;
      t0 = t1;
    }
  };
  int cur0 = 0, cur1 = 0;
  mark(7);
  // one call site per phase (a task table per slot): the phases are inlined once, as in
  // the lockstep kernel
  enum { T_NONE = 0, T_A, T_B, T_B2, T_C };
  auto run = [&](int kind, const SList* L, int h) {
    switch (kind) {
      case T_A: s_phase_a<R>(P, *L, smem, ring); break;
      case T_B:
        if (P.wide) s_phase_b_wide<R>(P, *L, smem, s_alpha[h], pst, &s_cg);
        else s_phase_b_reg<R>(P, *L, smem, s_alpha[h], pst, &s_cg);
        break;
      case T_B2: s_phase_b2(P, *L, smem, &s_cg); break;
      case T_C: s_phase_c_reg<R>(P, *L, smem, s_alpha[h], pst, &s_cg); break;
      default: break;
    }
  };
  if (lists[0][0].n + lists[1][0].n > 0 && P.max_iters > 0) {
    // slots -1 (A(H0) alone), then 0..3 per iteration
    int slot = -1;
    bool done = false;
#pragma unroll 1
    while (!done) {
      const SList* L0 = &lists[0][cur0];
      const SList* L1 = &lists[1][cur1];
      int k0 = T_NONE, k1 = T_NONE, h0 = 0, h1 = 1;
      const SList* a0 = L0;
      const SList* a1 = L1;
      bool swap = false;
      if (slot == -1) {
        k0 = T_A;
      } else if (slot == 0) {   // B(H0) | A(H1)
        k0 = T_B; k1 = T_A; swap = flip;
      } else if (slot == 1) {   // B2(H0) | B(H1)
        k0 = T_B2; k1 = T_B;
      } else if (slot == 2) {   // C(H0) | B2(H1); H0's statuses are stable: its next list
        s_build_list_half(cg, ns, lists[0][cur0 ^ 1], tmp, half, 0);
        k0 = T_C; k1 = T_B2;
      } else {                  // A(H0) of the next iteration | C(H1)
        s_build_list_half(cg, ns, lists[1][cur1 ^ 1], tmp, half, 1);
        k0 = (it + 1 < P.max_iters) ? T_A : T_NONE;
        a0 = &lists[0][cur0 ^ 1];
        k1 = T_C; swap = !flip;
      }
      if (swap) {
        const int tk = k0; k0 = k1; k1 = tk;
        const int th = h0; h0 = h1; h1 = th;
        const SList* tl = a0; a0 = a1; a1 = tl;
      }
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        if (q) s_task_switch();
        run(q ? k1 : k0, q ? a1 : a0, q ? h1 : h0);
      }
      mark(slot < 0 ? 7 : (slot == 0 ? 0 : slot + 1));
      sgrid_sync(P.bar, gen);
      mark(1);
      if (slot == 3) {
        if (P.prof && blockIdx.x == 0 && tid == 0) g_sprof[5] += 1;
        cur0 ^= 1;
        cur1 ^= 1;
        ++it;
        if (it >= P.max_iters || lists[0][cur0].n + lists[1][cur1].n == 0) done = true;
        slot = 0;
      } else {
        ++slot;
      }
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    *P.nactive = lists[0][cur0].n + lists[1][cur1].n;
    *P.iters_done = it;
  }
}

// ---------------------------------------------------------------- host side
bool strip_fill_params(Handle* h, StripParams& p, const double* X, int64_t ldx, const double* X2, int64_t ldx2,
                       int64_t nvec_map, double* Y, int64_t ldy, double* EY, int64_t ldey, const double* gamma,
                       int mode, int seg_rows);

int stream_seg_rows(int64_t ny) { return ny > 512 ? 256 : 128; }
// partial slots per shift: the largest item count, 64-row segments (s_seg_rows)
int stream_ipv(const Handle* h) { return kStripCtasPerSm * h->sm_count; }   // >= the grid
int stream_nchunk(const Handle* h) { return kStripCtasPerSm * h->sm_count; }   // >= the grid
int stream_grid(const Handle* h) { return kStripCtasPerSm * h->sm_count; }
int stream_pv() { return kSPV; }

extern "C" int rsk_debug_stream_cta(double* out, int n) {   // n x 8 (ns timestamps)
  static unsigned long long v[1024][8];
  if (cudaMemcpyFromSymbol(v, g_cta_t, sizeof(v)) != cudaSuccess) return -1;
  for (int i = 0; i < n && i < 1024; ++i)
    for (int j = 0; j < 8; ++j) out[i * 8 + j] = (double)v[i][j];
  return 0;
}

extern "C" int rsk_debug_stream_prof3(double* out8, int reset) {
  unsigned long long v[8];
  if (cudaMemcpyFromSymbol(v, g_sprof3, sizeof(v)) != cudaSuccess) return -1;
  for (int i = 0; i < 8; ++i) out8[i] = (double)v[i];
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_sprof3, z, sizeof(z));
  }
  return 0;
}

extern "C" int rsk_debug_stream_prof2(double* out8, int reset) {
  unsigned long long v[8];
  if (cudaMemcpyFromSymbol(v, g_sprof2, sizeof(v)) != cudaSuccess) return -1;
  for (int i = 0; i < 8; ++i) out8[i] = (double)v[i];
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_sprof2, z, sizeof(z));
  }
  return 0;
}

extern "C" int rsk_debug_stream_prof(double* out8, int reset) {
  unsigned long long v[8];
  if (cudaMemcpyFromSymbol(v, g_sprof, sizeof(v)) != cudaSuccess) return -1;
  for (int i = 0; i < 8; ++i) out8[i] = (double)v[i];
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_sprof, z, sizeof(z));
  }
  return 0;
}

template <int R>
static cudaError_t launch_stream_r(StreamParams& prm, int sm_count, cudaStream_t st, bool* ok) {
  using SC = SCfg<R>;
  // two CTAs per SM up to r = 10 (the configs); the occupancy query decides beyond
  // read per launch (a launch is 512 lockstep iterations): tests toggle it in-process
  const char* sk = getenv("RSK_STREAM_SKEW");
  const int skew = sk ? (atoi(sk) != 0) : kSkewDefault;
  auto kfn = skew ? cg_stream_skew_kernel<R> : cg_stream_kernel<R>;
  static int bs[2] = {0, 0};
  int& b = bs[skew];
  if (b == 0) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SC::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kfn, kAT, SC::SMEM);
    if (e != cudaSuccess) return e;
    if (b < 1) b = -1;
  }
  if (b < 1) { *ok = false; return cudaSuccess; }
  const int grid = (b < kStripCtasPerSm ? b : kStripCtasPerSm) * sm_count;
  prm.nchunk = grid;
  // rows per CTA: a multiple of 128 (8 warps x 16-row blocks of phase C, 64-row stages)
  prm.rpc = ((prm.cg_N + grid - 1) / grid + 127) / 128 * 128;
  void* args[] = {&prm};
  count_launch();
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kfn, dim3(grid), dim3(kAT), args, SC::SMEM, st);
  if (e != cudaSuccess) {
    static bool warned = false;
    if (!warned) {
      fprintf(stderr, "librsk: cooperative launch of the streaming CG loop failed (%s)\n", cudaGetErrorString(e));
      warned = true;
    }
    cudaGetLastError();
    *ok = false;
    return cudaSuccess;
  }
  *ok = true;
  return cudaSuccess;
}

// Runs up to max_iters lockstep iterations (device counters report the shifts left).
// *ok = false: not applicable (alignment / sizes / TMA) or the cooperative launch is
// impossible; the caller uses the tiled persistent loop instead.
cudaError_t launch_cg_stream(Handle* h, CgDev* dev, const CgDev& hc, double* partA, double* partB, unsigned* bar,
                             int* nactive, int* iters_done, int max_iters, cudaStream_t st, bool* ok) {
  *ok = false;
  const int64_t N = hc.N;
  if (hc.nshift > kSMaxShift || h->r < 1 || h->r > kMaxR) return cudaSuccess;
  // 16-byte rows of every streamed vector
  auto al16p = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if ((N & 1) || (hc.ldx & 1) || (hc.Ghat && (hc.ldgh & 1)) || (hc.grp.ldw & 1) || !al16p(hc.b) ||
      !al16p(hc.X) || !al16p(hc.R) || !al16p(hc.P) ||
      !al16p(hc.Wv) || (hc.Ghat && (!al16p(hc.Ghat) || !al16p(hc.ZGhat))))
    return cudaSuccess;
  StreamParams prm;
  std::memset(&prm, 0, sizeof(prm));
  const int seg = stream_seg_rows(h->ny);
  if (!strip_fill_params(h, prm.sp, hc.P, N, hc.X, hc.ldx, hc.nshift, hc.Wv, N, nullptr, 0, hc.gam,
                         RSK_APPLY_SHIFTED, seg))
    return cudaSuccess;
  prm.sp.want_dot = 1;
  // group blocks: |J| <= 16 and 16-byte rows (the register-form fragment loads)
  for (int gi = 0; gi < RSK_MAX_GROUPS; ++gi) {
    const int J = hc.grp.J[gi];
    if (J <= 0 || !hc.grp.AW[gi]) continue;
    if (J > 16 || !al16p(hc.grp.AW[gi]) || !al16p(hc.grp.EW[gi]) || !al16p(hc.grp.W[gi])) return cudaSuccess;
  }
  prm.cg = dev;
  prm.partA = partA;
  prm.partB = partB;
  prm.bar = bar;
  prm.nactive = nactive;
  prm.iters_done = iters_done;
  prm.nshift = hc.nshift;
  prm.cg_N = N;
  prm.ipv = stream_ipv(h);   // stride of partA; the items of an iteration: s_ipv()
  prm.max_iters = max_iters;
  {
    // wide phase B: 32-byte rows of every vector it streams
    auto al32p = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; };
    bool w = (N % 4) == 0 && (hc.grp.ldw % 4) == 0 && al32p(hc.b) && al32p(hc.R) && al32p(hc.Wv) &&
             (!hc.Ghat || ((hc.ldgh % 4) == 0 && al32p(hc.ZGhat)));
    for (int gi = 0; gi < RSK_MAX_GROUPS; ++gi)
      if (hc.grp.J[gi] > 0 && hc.grp.AW[gi]) w = w && al32p(hc.grp.AW[gi]) && al32p(hc.grp.EW[gi]);
    prm.wide = (w && !getenv("RSK_STREAM_NARROW")) ? 1 : 0;
  }
  {
    static int pf = -1;
    if (pf < 0) pf = getenv("RSK_PERSIST_PROF") ? 1 : 0;
    prm.prof = pf;
  }
  const int smc = h->sm_count;
  switch (h->r) {
    case 1: return launch_stream_r<1>(prm, smc, st, ok);
    case 2: return launch_stream_r<2>(prm, smc, st, ok);
    case 3: return launch_stream_r<3>(prm, smc, st, ok);
    case 4: return launch_stream_r<4>(prm, smc, st, ok);
    case 5: return launch_stream_r<5>(prm, smc, st, ok);
    case 6: return launch_stream_r<6>(prm, smc, st, ok);
    case 7: return launch_stream_r<7>(prm, smc, st, ok);
    case 8: return launch_stream_r<8>(prm, smc, st, ok);
    case 9: return launch_stream_r<9>(prm, smc, st, ok);
    case 10: return launch_stream_r<10>(prm, smc, st, ok);
    case 11: return launch_stream_r<11>(prm, smc, st, ok);
    case 12: return launch_stream_r<12>(prm, smc, st, ok);
    default: return cudaSuccess;
  }
}

}  // namespace rsk
