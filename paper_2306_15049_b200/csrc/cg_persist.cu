// Persistent lockstep loop of the batched deflated CG (rsk_cg_recycled_batch).
//
// One cooperative launch runs up to `max_iters` lockstep iterations of every active
// shift, with grid-wide barriers between the phases instead of kernel boundaries (the
// host-polled three-kernels-per-iteration loop was launch- and latency-bound: ~85 us
// per lockstep iteration at C2 with a few shifts left).  Recurrences are exactly those
// of the oracle O4 (oracle/defcg.py; reading D1 in DESIGN.md):
//
//   A  w = A_gamma p  (ACTIVE)  or  w = A_gamma x  (RCONV: true-residual confirm)
//      fused apply (apply_core.cuh) + per-tile p.w partials; last CTA of a shift forms
//      alpha = rho / p.w (BREAKDOWN if p.w <= 0)                          -- barrier
//   B  r = r - alpha w  (ACTIVE)  or  r = b - w  (RCONV); per row chunk the partials of
//      rho' = r.r  and  z = Z^T r = [(AW + gamma EW)^T r ; ZGhat^T r]     -- barrier
//   B2 one warp per shift: fixed-order sum over chunks; mu = G^-1 z; beta = rho'/rho;
//      status (RCONV on the recursive residual; DONE / MAXIT / restart after a confirm) -- barrier
//   C  x += alpha p ;  p = r + beta p - W mu_W - ghat mu_g ; residual store  -- barrier
//
// Every sum has a fixed order that depends only on N and the launch geometry, so the
// result of a shift does not depend on which other shifts share the batch (bitwise
// reproducible across shift shardings).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "apply_core.cuh"

namespace rsk {

constexpr int kPMaxShift = 256;   // shifts per persistent solve
constexpr int kPV = kMaxM + 1;    // partial slots per (shift, chunk): z_0..z_{m-1}, rho at kMaxM
constexpr int kPT = 32;           // shifts per phase-B tile
constexpr int kPW = kAT / 32;     // warps per CTA

__device__ unsigned long long g_pprof[8];   // per-phase ns (RSK_PERSIST_PROF), block 0's view

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct alignas(64) PersistParams {
  ApplyParams ap;      // CG-mode apply: X = P, X2 = caller x, Y = Wv
  CgDev* cg;
  double* partP;       // [shift][kPV][chunk]
  double* partA;       // [shift][grid]: each CTA's p.w partial of phase A (its items, in order)
  unsigned* bar;       // grid barrier {count, generation}
  int* nactive;        // out: shifts still ACTIVE / RCONV when the launch returns
  int* iters_done;     // out: lockstep iterations run by this launch
  int nshift;
  int nchunk;
  int64_t rows;        // rows per chunk (multiple of kAT)
  int max_iters;
  int prof;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// sense-reversing grid barrier; all CTAs are co-resident (cooperative launch)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& gen) {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");   // generic writes -> later TMA reads
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u) + 1u;
    if (arrived == gridDim.x) {
      bar[0] = 0u;
      __threadfence();
      st_release(bar + 1, gen + 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) {
      }
    }
    __threadfence();
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
  }
  gen += 1u;
  __syncthreads();
}

__device__ __forceinline__ void chol_solve_p(int m, const double* L, double* x) {
  for (int i = 0; i < m; ++i) {
    double t = x[i];
    for (int j = 0; j < i; ++j) t -= L[i + j * kMaxM] * x[j];
    x[i] = t / L[i + i * kMaxM];
  }
  for (int i = m - 1; i >= 0; --i) {
    double t = x[i];
    for (int j = i + 1; j < m; ++j) t -= L[j + i * kMaxM] * x[j];
    x[i] = t / L[i + i * kMaxM];
  }
}

// per-iteration snapshot of the active list (shared memory)
struct PList {
  int n;
  int sid[kPMaxShift];
  int mode[kPMaxShift];     // status at the start of the iteration: ST_ACTIVE or ST_RCONV
  int grp[kPMaxShift];      // shift group, local dimension m, carried column present
  int m[kPMaxShift];
  int hg[kPMaxShift];
};

// list of ACTIVE / RCONV shifts, sorted by group (phase B/C reuse the group blocks);
// warp 0 compacts with ballots
__device__ void build_list(const CgDev* cg, int ns, PList& L, int* tmp) {
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
          L.sid[pos] = s;
          L.mode[pos] = st;
        }
        n += __popc(bal);
      }
    if (lane == 0) L.n = n;
  }
  __syncthreads();
  for (int li = threadIdx.x; li < L.n; li += blockDim.x) {
    const int s = L.sid[li];
    L.grp[li] = cg->group[s];
    L.m[li] = cg->mloc[s];
    L.hg[li] = cg->hasg[s];
  }
  __syncthreads();
}

// Passes of up to 32 consecutive listed shifts of one group (the list is sorted by group).
__device__ __forceinline__ int pass_end(const PList& L, int li0) {
  const int g = L.grp[li0];
  int li1 = li0;
  while (li1 < L.n && li1 < li0 + 32 && L.grp[li1] == g) ++li1;
  return li1;
}

// ---- phase B: r update and the per-chunk partial sums of rho' and z = Z^T r.
// The skinny products [AW; EW]^T R of a pass run on the FP64 tensor cores: a k-step is 4
// rows; lane (g, q) updates r of (row q, shift 8 nb + g) -- exactly its B fragment -- and
// loads the A fragment (column 8 mb + g, row q) of AW / EW, shared by the 4 N-blocks.
// Each shift's column of D, its rho and zeta are summed in an order fixed by the chunk
// geometry only (rows of a warp, then warps), independent of the other shifts in the pass.
constexpr int kRW = 34;   // per (warp, shift) staging: za[16], ze[16], rho, zeta
__device__ __noinline__ void phase_b(const PersistParams& P, const PList& L, double* smem, double* s_alpha,
                                     const double* s_gam, CgDev* cg) {
  const int n = L.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t N = cg->N;
  // alpha = rho / pi from the grid's phase-A partials (every CTA, same fixed order); CTA 0
  // records it and flags breakdowns for B2 / C
  for (int li = warp; li < n; li += kAT / 32) {   // a warp per shift: strided lanes, fixed tree
    double a = 0.0;
    if (L.mode[li] == ST_ACTIVE) {
      const int s = L.sid[li];
      const double* pa = P.partA + (size_t)s * gridDim.x;
      double pi = 0.0;
      for (int c = lane; c < (int)gridDim.x; c += 32) pi += __ldcg(pa + c);
      pi = warp_sum(pi);
      if (!(pi > 0.0) || !isfinite(pi)) {
        if (blockIdx.x == 0 && lane == 0) { cg->status[s] = ST_BREAKDOWN; cg->alpha[s] = 0.0; }
      } else {
        a = cg->rho[s] / pi;
        if (blockIdx.x == 0 && lane == 0) cg->alpha[s] = a;
      }
    }
    if (lane == 0) s_alpha[li] = a;
  }
  __syncthreads();
  double* red = smem;   // [kPW][32][kRW] (the apply stage buffers are free now)
  const int64_t rpw = P.rows / kPW;   // rows per warp (multiple of 32)
  for (int c = blockIdx.x; c < P.nchunk; c += gridDim.x) {
    const int64_t cbeg = (int64_t)c * P.rows;
    const int64_t cend = min(N, cbeg + P.rows);
    const int64_t wbeg = cbeg + warp * rpw;
    const int64_t wend = min(cend, wbeg + rpw);
    for (int li0 = 0; li0 < n; ) {
      const int li1 = pass_end(L, li0);
      const int np = li1 - li0;
      const int grp = L.grp[li0];
      const int J = cg->grp.J[grp];
      const double* AWg = cg->grp.AW[grp];
      const double* EWg = cg->grp.EW[grp];
      const int64_t ldw = cg->grp.ldw;
      // this lane's shifts (one per N-block)
      int sv[4], md[4], hgv[4];
      double al[4];
      bool ok[4];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        const int li = li0 + 8 * nb + g;
        ok[nb] = li < li1;
        sv[nb] = ok[nb] ? L.sid[li] : 0;
        md[nb] = ok[nb] ? L.mode[li] : ST_ACTIVE;
        hgv[nb] = ok[nb] ? L.hg[li] : 0;
        al[nb] = ok[nb] ? s_alpha[li] : 0.0;
      }
      double dA[4][2][2], dE[4][2][2], rh[4], zt[4];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        rh[nb] = 0.0; zt[nb] = 0.0;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) { dA[nb][mb][0] = dA[nb][mb][1] = dE[nb][mb][0] = dE[nb][mb][1] = 0.0; }
      }
#pragma unroll 2
      for (int64_t row0 = wbeg; row0 < wend; row0 += 4) {
        const int64_t row = row0 + q;
        const bool vr = row < wend;
        double aA[2], aE[2];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
          const int col = 8 * mb + g;
          const bool va = vr && col < J;
          aA[mb] = va ? __ldg(AWg + (int64_t)col * ldw + row) : 0.0;
          aE[mb] = va ? __ldg(EWg + (int64_t)col * ldw + row) : 0.0;
        }
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          if (8 * nb >= np) break;                  // uniform across the warp
          double rn = 0.0;
          if (ok[nb] && vr) {
            const int64_t o = (int64_t)sv[nb] * N + row;
            const double wv = cg->Wv[o];
            rn = (md[nb] == ST_ACTIVE) ? fma(-al[nb], wv, cg->R[o]) : __ldg(cg->b + row) - wv;
            cg->R[o] = rn;
            rh[nb] = fma(rn, rn, rh[nb]);
            if (hgv[nb]) zt[nb] = fma(__ldg(cg->ZGhat + (int64_t)sv[nb] * cg->ldgh + row), rn, zt[nb]);
          }
          dmma(dA[nb][0][0], dA[nb][0][1], aA[0], rn);
          dmma(dE[nb][0][0], dE[nb][0][1], aE[0], rn);
          if (J > 8) {
            dmma(dA[nb][1][0], dA[nb][1][1], aA[1], rn);
            dmma(dE[nb][1][0], dE[nb][1][1], aE[1], rn);
          }
        }
      }
      // stage: D[m = 8 mb + g][n = 2q, 2q+1] of N-block nb; rho / zeta summed over the q lanes
      double* rw = red + (size_t)warp * 32 * kRW;
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        if (8 * nb >= np) break;
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
      for (int e = tid; e < np * kPV; e += kAT) {
        const int k = e / kPV, j = e - k * kPV;
        const int li = li0 + k;
        const int nw = L.m[li] - L.hg[li];
        const bool isz = j < nw, isg = L.hg[li] && j == nw, isr = j == kMaxM;
        if (!(isz || isg || isr)) continue;
        double ta = 0.0, te = 0.0;
#pragma unroll
        for (int w = 0; w < kPW; ++w) {
          const double* r = red + ((size_t)w * 32 + k) * kRW;
          if (isz) { ta += r[j]; te += r[16 + j]; }
          else ta += r[isr ? 32 : 33];
        }
        const double v = isz ? fma(s_gam[L.sid[li]], te, ta) : ta;
        P.partP[((size_t)L.sid[li] * kPV + j) * P.nchunk + c] = v;
      }
      __syncthreads();
      li0 = li1;
    }
  }
}

// ---- phase B2: one CTA per shift. Warp w sums slots j = w, w + 8, ... over the chunks
// (coalesced, fixed order); warp 0 then solves G mu = z with the Cholesky factor staged
// in shared memory and updates the shift's scalars and status.
__device__ __noinline__ void phase_b2(const PersistParams& P, const PList& L, double* smem, CgDev* cg) {
  const int n = L.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* zs = smem;                  // [kPV]
  double* Ls = smem + 32;             // [kMaxM][kMaxM] lower factor, row-major
  for (int li = blockIdx.x; li < n; li += gridDim.x) {
    const int s = L.sid[li];
    const int mode0 = L.mode[li];
    const int m = L.m[li];
    const double* Lg = cg->Lf + (int64_t)s * kMaxM * kMaxM;
    for (int e = tid; e < m * m; e += kAT) {
      const int i = e / m, j = e - i * m;
      if (j <= i) Ls[i * kMaxM + j] = Lg[i + j * kMaxM];
    }
    for (int j = warp; j < kPV; j += kPW) {
      if (j < m || j == kMaxM) {
        const double* pj = P.partP + ((size_t)s * kPV + j) * P.nchunk;
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
        int c = lane;
        for (; c + 96 < P.nchunk; c += 128) {
          t0 += pj[c]; t1 += pj[c + 32]; t2 += pj[c + 64]; t3 += pj[c + 96];
        }
        for (; c < P.nchunk; c += 32) t0 += pj[c];
        const double t = warp_sum((t0 + t1) + (t2 + t3));
        if (lane == 0) zs[j] = t;
      }
    }
    __syncthreads();
    if (tid == 0) {
      const double rho_new = zs[kMaxM];
      const int st = cg->status[s];
      const double thr = cg->tol * cg->bnorm;
      const bool conv = sqrt(rho_new) <= thr;
      int nst = st;
      bool newp = false;
      if (mode0 == ST_ACTIVE) {
        if (st == ST_ACTIVE) {   // not BREAKDOWN in phase A
          const int itn = cg->iters[s] + 1;
          cg->iters[s] = itn;
          cg->beta[s] = rho_new / cg->rho[s];
          cg->rho[s] = rho_new;
          if (conv) nst = ST_RCONV;
          else if (itn >= cg->maxit) nst = ST_MAXIT;
          else newp = true;
        }
      } else {   // confirm on the true residual r = b - A_gamma x
        cg->rho_true[s] = rho_new;
        cg->nconf[s] += 1;
        cg->alpha[s] = 0.0;
        if (conv) nst = ST_DONE;
        else if (cg->iters[s] >= cg->maxit) nst = ST_MAXIT;
        else {
          nst = ST_ACTIVE;   // restart from the true residual
          cg->beta[s] = 0.0;
          cg->rho[s] = rho_new;
          newp = true;
        }
      }
      if (newp) {
        // mu = G^-1 z: forward / backward substitution with L L^T = G (m <= kMaxM)
        double* cf = cg->coef + (int64_t)s * kMaxM;
        double x[kMaxM];
#pragma unroll
        for (int i = 0; i < kMaxM; ++i) {
          if (i < m) {
            double t = zs[i];
#pragma unroll
            for (int j = 0; j < i; ++j) t -= Ls[i * kMaxM + j] * x[j];
            x[i] = t / Ls[i * kMaxM + i];
          }
        }
#pragma unroll
        for (int i = kMaxM - 1; i >= 0; --i) {
          if (i < m) {
            double t = x[i];
#pragma unroll
            for (int j = i + 1; j < kMaxM; ++j)
              if (j < m) t -= Ls[j * kMaxM + i] * x[j];
            x[i] = t / Ls[i * kMaxM + i];
          }
        }
#pragma unroll
        for (int j = 0; j < kMaxM; ++j) cf[j] = j < m ? x[j] : 0.0;
        int slot = -1;
        if (cg->store && cg->store_cnt[s] < cg->store_cap) {
          slot = cg->store_cnt[s];
          cg->store_cnt[s] = slot + 1;
        }
        cg->stslot[s] = slot;
      }
      cg->status[s] = nst;
    }
    __syncthreads();
  }
}

// ---- phase C: x += alpha p; p = r + beta p - W mu_W - ghat mu_g; residual store.
// W mu of a pass on the tensor cores: an 8-row block x 8 shifts is D = W[8 x J] M[J x 8]
// (A = W rows, B = the shifts' mu from shared memory); lane (g, q) then finishes the
// elements (row g, shifts 2q, 2q+1) of each N-block.
__device__ __noinline__ void phase_c(const PersistParams& P, const PList& L, double* smem, const double* s_alpha,
                                     int* s_new, double* s_beta, int* s_slot, double* s_rinv, CgDev* cg) {
  const int n = L.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t N = cg->N;
  double* scoef = smem;          // [n][kMaxM]
  for (int li = tid; li < n; li += kAT) {
    const int s = L.sid[li];
    const int st = cg->status[s];
    s_new[li] = st;
    s_beta[li] = cg->beta[s];
    s_slot[li] = (st == ST_ACTIVE) ? cg->stslot[s] : -1;
    s_rinv[li] = (st == ST_ACTIVE && s_slot[li] >= 0) ? 1.0 / sqrt(cg->rho[s]) : 0.0;
  }
  for (int e = tid; e < n * kMaxM; e += kAT) {
    const int li = e / kMaxM, j = e - li * kMaxM;
    scoef[e] = cg->coef[(int64_t)L.sid[li] * kMaxM + j];
  }
  __syncthreads();
  const int64_t rpw = P.rows / kPW;
  for (int c = blockIdx.x; c < P.nchunk; c += gridDim.x) {
    const int64_t cbeg = (int64_t)c * P.rows;
    const int64_t cend = min(N, cbeg + P.rows);
    const int64_t wbeg = cbeg + warp * rpw;
    const int64_t wend = min(cend, wbeg + rpw);
    for (int li0 = 0; li0 < n; ) {
      const int li1 = pass_end(L, li0);
      const int np = li1 - li0;
      const int grp = L.grp[li0];
      const int J = cg->grp.J[grp];
      const double* Wg = cg->grp.W[grp];
      const int64_t ldw = cg->grp.ldw;
      // B fragments: mu of shift 8 nb + g, component 4 kk + q (0 beyond its nw)
      double bm[4][4];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        const int li = li0 + 8 * nb + g;
        const int nw = (li < li1) ? L.m[li] - L.hg[li] : 0;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int j = 4 * kk + q;
          bm[nb][kk] = (li < li1 && j < nw && s_new[li] == ST_ACTIVE) ? scoef[li * kMaxM + j] : 0.0;
        }
      }
      const int nkk = (J + 3) >> 2;
      // per-element flags of this lane's 8 (N-block, h) pairs
      int flg[4][2];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int li = li0 + 8 * nb + 2 * q + h;
          int f = 0;
          if (li < li1) {
            if ((L.mode[li] == ST_ACTIVE) && (s_alpha[li] != 0.0)) f |= 1;
            if (s_new[li] == ST_ACTIVE) f |= 2;
          }
          flg[nb][h] = f;
        }
#pragma unroll 1
      for (int64_t row0 = wbeg; row0 < wend; row0 += 8) {
        const int64_t row = row0 + g;
        const bool vr = row < wend;
        double a[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int j = 4 * kk + q;
          a[kk] = (vr && kk < nkk && j < J) ? __ldg(Wg + (int64_t)j * ldw + row) : 0.0;
        }
        // every element load of the row block first
        double pv[4][2], rv[4][2], xv[4][2], gv[4][2];
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            pv[nb][h] = rv[nb][h] = xv[nb][h] = gv[nb][h] = 0.0;
            const int f = vr ? flg[nb][h] : 0;
            if (f && 8 * nb < np) {
              const int li = li0 + 8 * nb + 2 * q + h;
              const int s = L.sid[li];
              const int64_t o = (int64_t)s * N + row;
              pv[nb][h] = cg->P[o];
              if (f & 1) xv[nb][h] = cg->X[(int64_t)s * cg->ldx + row];
              if (f & 2) {
                rv[nb][h] = cg->R[o];
                if (L.hg[li]) gv[nb][h] = __ldg(cg->Ghat + (int64_t)s * cg->ldgh + row);
              }
            }
          }
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          if (8 * nb >= np) break;
          double d[2] = {0.0, 0.0};
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            if (kk < nkk) dmma(d[0], d[1], a[kk], bm[nb][kk]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int f = vr ? flg[nb][h] : 0;
            if (!f) continue;
            const int li = li0 + 8 * nb + 2 * q + h;
            const int s = L.sid[li];
            const int64_t o = (int64_t)s * N + row;
            if (f & 1) cg->X[(int64_t)s * cg->ldx + row] = fma(s_alpha[li], pv[nb][h], xv[nb][h]);
            if (f & 2) {
              double pn = fma(s_beta[li], pv[nb][h], rv[nb][h]) - d[h];
              const int hg = L.hg[li];
              if (hg) pn = fma(-scoef[li * kMaxM + L.m[li] - hg], gv[nb][h], pn);
              cg->P[o] = pn;
              if (s_slot[li] >= 0)
                cg->store[((int64_t)s * cg->store_cap + s_slot[li]) * cg->lds + row] = rv[nb][h] * s_rinv[li];
            }
          }
        }
      }
      li0 = li1;
    }
  }
}

// ---- phase A: the fused apply over the (tile, shift) items of the active list
template <int R, bool kTma>
__device__ __forceinline__ void phase_a(const PersistParams& P, const PList& L, double* smem, ApplyPipe& pp,
                                        double* s_pw) {
  const int n = L.n;
  const int nitems = n * P.ap.ntiles;
  const int per = (nitems + gridDim.x - 1) / gridDim.x;
  const int ibeg = blockIdx.x * per;
  const int iend = min(nitems, ibeg + per);
  // p.w: per-CTA partials accumulated in shared memory over its items (fixed order), one
  // store per shift; alpha is formed from them at the start of phase B (no per-item ticket)
  for (int li = threadIdx.x; li < n; li += kAT) s_pw[li] = 0.0;
  __syncthreads();
  ApplyCore<R, kTma>::run(P.ap, smem, ibeg, iend, n, pp, L.sid, L.mode, s_pw);
  __syncthreads();
  for (int li = threadIdx.x; li < n; li += kAT) P.partA[(size_t)L.sid[li] * gridDim.x + blockIdx.x] = s_pw[li];
}

template <int R, bool kTma>
__global__ void __launch_bounds__(kAT, kApplyCtasPerSm) cg_persist_kernel(const __grid_constant__ PersistParams P) {
  extern __shared__ __align__(128) double smem[];
  using Core = ApplyCore<R, kTma>;
  __shared__ PList lists[2];
  __shared__ int tmp[kPMaxShift];
  __shared__ double s_alpha[kPMaxShift], s_beta[kPMaxShift], s_rinv[kPMaxShift], s_gam[kPMaxShift];
  __shared__ int s_new[kPMaxShift], s_slot[kPMaxShift];
  __shared__ double s_pw[kPMaxShift];

  // the loop state's pointers and sizes in shared memory: no global round trip per field
  // access after the L1 invalidations of the grid barriers
  __shared__ CgDev s_cg;
  if (threadIdx.x == 0) s_cg = *P.cg;
  __syncthreads();
  CgDev* cg = &s_cg;
  const int ns = P.nshift;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = cg->N;
  Core::init_bars(smem, P.ap);
  ApplyPipe pp{{0u, 0u}, 0};
  unsigned gen = ld_acquire(P.bar + 1);
  int cur = 0;
  build_list(cg, ns, lists[0], tmp);
  for (int s = tid; s < ns; s += kAT) s_gam[s] = cg->gam[s];
  grid_sync(P.bar, gen);   // nobody changes a status before every CTA has read them

  int it = 0;
  unsigned long long t0 = 0;
  auto mark = [&](int ph) {
    if (P.prof && blockIdx.x == 0 && tid == 0) {
      const unsigned long long t1 = gtimer();
      if (t0) g_pprof[ph] += t1 - t0;
      t0 = t1;
    }
  };
  mark(7);
  for (; it < P.max_iters; ++it) {
    PList& L = lists[cur];
    const int n = L.n;
    if (n == 0) break;

    // ================= A: w = A_gamma p (or A_gamma x for confirms)
    phase_a<R, kTma>(P, L, smem, pp, s_pw);
    mark(0);
    grid_sync(P.bar, gen);
    mark(1);

    phase_b(P, L, smem, s_alpha, s_gam, cg);
    mark(2);
    grid_sync(P.bar, gen);
    mark(1);

    phase_b2(P, L, smem, cg);
    mark(3);
    grid_sync(P.bar, gen);
    mark(1);

    PList& NL = lists[cur ^ 1];
    build_list(cg, ns, NL, tmp);   // statuses are stable until the next phase A
    phase_c(P, L, smem, s_alpha, s_new, s_beta, s_slot, s_rinv, cg);
    mark(4);
    grid_sync(P.bar, gen);
    mark(1);
    if (P.prof && blockIdx.x == 0 && tid == 0) g_pprof[5] += 1;
    cur ^= 1;
  }
  if (blockIdx.x == 0 && tid == 0) {
    *P.nactive = lists[cur].n;
    *P.iters_done = it;
  }
}

// ------------------------------------------------------------------ host side
bool fill_apply_params(Handle* h, const ApplyLaunch& a, ApplyParams& prm, int ty_override);

template <int R>
static cudaError_t launch_persist_r(PersistParams& prm, bool tma, int sm_count, cudaStream_t st, bool* ok) {
  using C = TcCfg<R>;
  // phases B / B2 / C reuse the apply's stage and T buffers below the correction table
  static_assert(C::OFF_DC >= kPW * 32 * kRW && C::OFF_DC >= kPMaxShift * kMaxM + 16 * kAT &&
                    C::OFF_DC >= 32 + kMaxM * kMaxM,
                "persistent-loop scratch overlaps the apply's boundary-correction table");
  auto kfn = tma ? cg_persist_kernel<R, true> : cg_persist_kernel<R, false>;
  size_t smem = C::SMEM;
  const size_t accb = sizeof(double) * (size_t)kPW * 32 * kRW;
  const size_t coefb = sizeof(double) * ((size_t)kPMaxShift * kMaxM + 16 * kAT);
  if (smem < accb) smem = accb;
  if (smem < coefb) smem = coefb;
  static int bps[2] = {0, 0};
  int& b = bps[tma ? 1 : 0];
  if (b == 0) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kfn, kAT, smem);
    if (e != cudaSuccess) return e;
    if (b < 1) b = -1;
  }
  if (b < 1) { *ok = false; return cudaSuccess; }
  const int grid = b * sm_count;
  if (prm.nchunk > grid) { *ok = false; return cudaSuccess; }
  void* args[] = {&prm};
  count_launch();
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kfn, dim3(grid), dim3(kAT), args, smem, st);
  if (e != cudaSuccess) {
    static bool warned = false;
    if (!warned) {
      fprintf(stderr, "librsk: cooperative launch failed (%s); host-polled CG loop\n", cudaGetErrorString(e));
      warned = true;
    }
    cudaGetLastError();
    *ok = false;
    return cudaSuccess;
  }
  *ok = true;
  return cudaSuccess;
}

extern "C" int rsk_debug_persist_prof(double* out8, int reset) {
  unsigned long long v[8];
  if (cudaMemcpyFromSymbol(v, g_pprof, sizeof(v)) != cudaSuccess) return -1;
  for (int i = 0; i < 8; ++i) out8[i] = (double)v[i];
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_pprof, z, sizeof(z));
  }
  return 0;
}

int persist_grid(const Handle* h) { return kApplyCtasPerSm * h->sm_count; }
int persist_max_shift() { return kPMaxShift; }
int persist_pv() { return kPV; }

// Runs up to max_iters lockstep iterations; returns (through the device counters) the
// number of shifts still in the loop. *ok = false if the cooperative launch is impossible
// (caller falls back to the host-polled loop).
cudaError_t launch_cg_persist(Handle* h, CgDev* dev, const CgDev& hc, double* partP, unsigned* bar,
                              int* nactive, int* iters_done, int nchunk, int64_t rows, int max_iters,
                              cudaStream_t st, bool* ok) {
  PersistParams prm;
  ApplyLaunch a{};
  a.X = hc.P; a.ldx = hc.N;
  a.X2 = hc.X; a.ldx2 = hc.ldx;
  a.Y = hc.Wv; a.ldy = hc.N;
  a.gamma = hc.gam;
  a.nlist = hc.nshift;
  a.nvec_total = hc.nshift;
  a.mode = RSK_APPLY_SHIFTED;
  a.cg = dev;
  a.cg_alpha = true;
  a.src2_rconv = true;
  const bool tma = fill_apply_params(h, a, prm.ap, 0);
  prm.cg = dev;
  prm.partP = partP;
  prm.partA = partP + (size_t)hc.nshift * nchunk * kPV;
  prm.bar = bar;
  prm.nactive = nactive;
  prm.iters_done = iters_done;
  prm.nshift = hc.nshift;
  prm.nchunk = nchunk;
  prm.rows = rows;
  prm.max_iters = max_iters;
  {
    static int pf = -1;
    if (pf < 0) pf = getenv("RSK_PERSIST_PROF") ? 1 : 0;
    prm.prof = pf;
  }
  *ok = false;
  if (hc.nshift > kPMaxShift) return cudaSuccess;
  const int smc = h->sm_count;
  switch (h->r) {
    case 1: return launch_persist_r<1>(prm, tma, smc, st, ok);
    case 2: return launch_persist_r<2>(prm, tma, smc, st, ok);
    case 3: return launch_persist_r<3>(prm, tma, smc, st, ok);
    case 4: return launch_persist_r<4>(prm, tma, smc, st, ok);
    case 5: return launch_persist_r<5>(prm, tma, smc, st, ok);
    case 6: return launch_persist_r<6>(prm, tma, smc, st, ok);
    case 7: return launch_persist_r<7>(prm, tma, smc, st, ok);
    case 8: return launch_persist_r<8>(prm, tma, smc, st, ok);
    case 9: return launch_persist_r<9>(prm, tma, smc, st, ok);
    case 10: return launch_persist_r<10>(prm, tma, smc, st, ok);
    case 11: return launch_persist_r<11>(prm, tma, smc, st, ok);
    case 12: return launch_persist_r<12>(prm, tma, smc, st, ok);
    default: return cudaSuccess;
  }
}

}  // namespace rsk
