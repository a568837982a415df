// Group-shared CG vector kernels (the hot loop of rsk_cg_recycled_batch, LOOP mode).
//
// Deflated CG (reading D1; eq:corr_g P:462-468 with the local spaces of Alg. 3/4)
// needs, per active shift s of shift group g, every iteration:
//   KB  r_s -= alpha_s w_s;  rho_s = r_s.r_s;  z_s = Z_s^T r_s with
//       Z_s = [AW_g + gamma_s EW_g, ZGhat_s]  ->  mu_s = G_s^-1 z_s, beta_s
//   KC  x_s += alpha_s p_s;  p_s = r_s + beta_s p_s - W_g mu_s,W - ghat_s mu_s,g
// W_g, AW_g, EW_g are shared by all shifts of a group. One CTA covers a chunk of rows
// (a multiple of 256) x a tile of up to 32 active shifts of ONE group.
//  * Streaming phase: thread <-> pixel row, a fully unrolled loop over the tile's
//    shifts, every load of a 4-shift batch issued before it is used: deep
//    memory-level parallelism, no barriers (the v1/v2 kernels were latency bound).
//  * KB: the updated residuals of a 256-row sub-slab land in shared memory; the
//    Z^T r dots are a skinny GEMM [AW; EW] (2J x 256) x R (256 x S), 4 x 4 register
//    blocked per thread over 32-row groups; rho and ZGhat.r accumulate per thread.
//  * Reductions are deterministic: fixed per-thread order, fixed trees, and a
//    two-level ticket (groups of 16 chunks, then the <= 16 group sums) in fixed order.
#include <cuda_runtime.h>

#include "rsk_internal.h"

namespace rsk {

namespace {

__device__ __forceinline__ double wsum32(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ void chol_solve_dev(int m, const double* L, double* x) {
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

// partial layout per (g, tile, chunk): kPV rows x 32 shifts
//   rows 0..15: z_j = sum (AW_j + gamma EW_j) r   (j < J)
//   row 16: rho = r.r       row 17: ZGhat.r
constexpr int kPV = kPartRowsG;
constexpr int kLvl = 16;        // chunks per level-1 group
constexpr int kSub = 256;       // rows per combine sub-slab (= threads)
constexpr int kHalf = 128;      // rows per update sub-slab (2 threads per row)
constexpr int kHP = kHalf + 1;  // odd pitch

// sum `cnt` partial blocks (kPV x 32 each, stride kPV*32) into dst, fixed order, with
// every thread loading its (value, block) pairs before adding
__device__ __forceinline__ void sum_blocks(const double* src, int cnt, double* dst, int S) {
  for (int e = threadIdx.x; e < kPV * 32; e += kNT) {
    if ((e & 31) >= S) continue;
    double v[kLvl];
#pragma unroll
    for (int c = 0; c < kLvl; ++c) v[c] = c < cnt ? __ldcg(src + (int64_t)c * (kPV * 32) + e) : 0.0;
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < kLvl; ++c) t += v[c];
    dst[e] = t;
  }
}

struct TileInfo {
  int sid[32];
  double al[32];
  double gam[32];
  int act[32];
  int hasg[32];
};

}  // namespace

// ------------------------------------------------------------------ KB (update)
__global__ void __launch_bounds__(kNT, 2) cg_update_grp(CgDev* __restrict__ cg) {
  // dynamic smem: sA [2J][kHP] | sR [32][kHP] | sZ [32][kHP]
  extern __shared__ double dsm[];
  __shared__ TileInfo ti;
  __shared__ double tot[kPV * 32];
  __shared__ int s_flag;
  const int g = blockIdx.y, tile = blockIdx.z, chunk = blockIdx.x;
  const int* gm = cg->gmeta;
  const int S = min(32, gm[4 + g] - tile * 32);
  if (S <= 0) return;
  const int J = cg->grp.J[g];
  const int J2 = 2 * J;
  double* sA = dsm;
  double* sR = dsm + J2 * kHP;
  double* sZ = sR + 32 * kHP;
  const int64_t N = cg->N;
  const int64_t ldw = cg->grp.ldw;
  const double* __restrict__ AW = cg->grp.AW[g];
  const double* __restrict__ EW = cg->grp.EW[g];
  const int tid = threadIdx.x;
  if (tid < 32) {
    const bool v = tid < S;
    const int s = v ? cg->glist[gm[g] + tile * 32 + tid] : 0;
    ti.sid[tid] = s;
    ti.al[tid] = v ? cg->alpha[s] : 0.0;
    ti.gam[tid] = v ? cg->gam[s] : 0.0;
    ti.act[tid] = v && cg->status[s] == ST_ACTIVE;
    ti.hasg[tid] = v ? cg->hasg[s] : 0;
  }
  __syncthreads();
  // streaming role: row sr (of kHalf), shifts k = sh + 2u
  const int sr = tid & (kHalf - 1), sh = tid >> 7;
  // rho / zeta role: shift tk, 16-row segment tseg
  const int tk = tid & 31, tseg = tid >> 5;
  double prho = 0.0, pzet = 0.0;
  // GEMM role: k-block kb (4 shifts), j-block jb (4 rows of [AW;EW]), row group rg
  const int njb = (J2 > 16) ? 8 : 4;
  const int nrg = 32 / njb;
  const int rpg = kHalf / nrg;
  const int kb = tid & 7, jb = (tid >> 3) & (njb - 1), rg = (tid >> 3) / njb;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  const int64_t rbeg = (int64_t)chunk * cg->rowsG;
  const int64_t rend = min(N, rbeg + cg->rowsG);
  for (int64_t r0 = rbeg; r0 < rend; r0 += kHalf) {
    const int64_t i = r0 + sr;
    const bool rin = i < rend;
    // stage the [AW; EW] sub-slab (rows split over the two halves)
    for (int j = sh; j < J2; j += 2)
      sA[j * kHP + sr] = rin ? __ldg((j < J ? AW + (int64_t)j * ldw : EW + (int64_t)(j - J) * ldw) + i) : 0.0;
    // streaming pass: loads -> shared memory only (no global stores: loads can be hoisted)
#pragma unroll
    for (int u0 = 0; u0 < 16; u0 += 4) {
      double rv[4], wv[4], zv[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int k = sh + 2 * (u0 + v);
        rv[v] = wv[v] = zv[v] = 0.0;
        if (k < S && rin) {
          const int64_t off = (int64_t)ti.sid[k] * N + i;
          rv[v] = __ldcg(cg->R + off);
          wv[v] = __ldcg(cg->Wv + off);
          if (ti.hasg[k]) zv[v] = __ldg(cg->ZGhat + (int64_t)ti.sid[k] * cg->ldgh + i);
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int k = sh + 2 * (u0 + v);
        if (k < S) {
          const double rn = fma(-ti.al[k], wv[v], rv[v]);
          sR[k * kHP + sr] = rn;
          sZ[k * kHP + sr] = zv[v] * rn;
        }
      }
    }
    __syncthreads();
    // write the updated residuals back (coalesced)
#pragma unroll 4
    for (int u = 0; u < 16; ++u) {
      const int k = sh + 2 * u;
      if (k < S && ti.act[k] && rin) cg->R[(int64_t)ti.sid[k] * N + i] = sR[k * kHP + sr];
    }
    // rho, zeta partials over this thread's 16-row segment
    if (tk < S) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double rn = sR[tk * kHP + tseg * 16 + q];
        prho = fma(rn, rn, prho);
        pzet += sZ[tk * kHP + tseg * 16 + q];
      }
    }
    // GEMM over this sub-slab: acc[a][b] += sum_rows sA[4jb+a][row] * sR[4kb+b][row]
    if (4 * jb < J2 && 4 * kb < S) {
#pragma unroll 4
      for (int rr = 0; rr < rpg; ++rr) {
        const int row = rg * rpg + rr;
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = sA[min(4 * jb + a, J2 - 1) * kHP + row];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = sR[(4 * kb + b) * kHP + row];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
      }
    }
    __syncthreads();
  }
  // ---- CTA-level reductions (once per chunk), fixed order through shared memory
  double* red = sR;                  // [nrg][4 njb][33] = 4224 doubles (inside sR | sZ)
  double* red2 = sZ + 256;           // [8][64]
  const int RJ = 4 * njb;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) red[(rg * RJ + 4 * jb + a) * 33 + 4 * kb + b] = acc[a][b];
  red2[tseg * 64 + tk] = prho;
  red2[tseg * 64 + 32 + tk] = pzet;
  __syncthreads();
  double* pg = cg->partG + ((int64_t)g * cg->maxtilesG + tile) * (int64_t)(cg->nchunkG + kLvl) * (kPV * 32);
  double* pb = pg + (int64_t)chunk * (kPV * 32);
  for (int e = tid; e < 16 * 32; e += kNT) {
    const int j = e >> 5, k = e & 31;
    if (j < J && k < S) {
      double za = 0.0, ze = 0.0;
      for (int q = 0; q < nrg; ++q) {
        za += red[(q * RJ + j) * 33 + k];
        ze += red[(q * RJ + J + j) * 33 + k];
      }
      pb[j * 32 + k] = fma(ti.gam[k], ze, za);
    }
  }
  if (tid < 64) {
    const int k = tid & 31;
    if (k < S) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) t += red2[q * 64 + tid];
      pb[(16 + (tid >> 5)) * 32 + k] = t;
    }
  }
  // ---- two-level ticket: level 1 = groups of kLvl chunks
  const int nch = gridDim.x;
  const int grp1 = chunk / kLvl;
  const int ngrp1 = (nch + kLvl - 1) / kLvl;
  unsigned* tick = cg->cntG + (size_t)(g * cg->maxtilesG + tile) * kTickStride;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int members = min(kLvl, nch - grp1 * kLvl);
    const unsigned tkt = atomicAdd(tick + 2 + grp1, 1u);
    s_flag = (tkt == (unsigned)(members - 1));
  }
  __syncthreads();
  if (!s_flag) return;
  __threadfence();
  double* lvl2 = pg + (int64_t)cg->nchunkG * (kPV * 32);   // kLvl level-2 slots
  sum_blocks(pg + (int64_t)grp1 * kLvl * (kPV * 32), min(kLvl, nch - grp1 * kLvl), tot, S);
  __syncthreads();
  for (int e = tid; e < kPV * 32; e += kNT) lvl2[(int64_t)grp1 * (kPV * 32) + e] = tot[e];
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    tick[2 + grp1] = 0u;
    const unsigned tkt = atomicAdd(tick + 0, 1u);
    s_flag = (tkt == (unsigned)(ngrp1 - 1));
  }
  __syncthreads();
  if (!s_flag) return;
  __threadfence();
  sum_blocks(lvl2, ngrp1, tot, S);
  __syncthreads();
  if (tid == 0) tick[0] = 0u;
  if (tid >= S) return;
  const int s = ti.sid[tid];
  if (cg->status[s] != ST_ACTIVE) return;
  const int m = cg->mloc[s], hg = cg->hasg[s], nw = m - hg;
  double z[kMaxM];
  for (int j = 0; j < nw; ++j) z[j] = tot[j * 32 + tid];
  if (hg) z[nw] = tot[17 * 32 + tid];
  if (m > 0) chol_solve_dev(m, cg->Lf + (int64_t)s * kMaxM * kMaxM, z);
  double* cf = cg->coef + (int64_t)s * kMaxM;
  for (int j = 0; j < kMaxM; ++j) cf[j] = j < m ? z[j] : 0.0;
  const double rho_new = tot[16 * 32 + tid];
  const int itn = cg->iters[s] + 1;
  cg->iters[s] = itn;
  cg->beta[s] = rho_new / cg->rho[s];
  cg->rho[s] = rho_new;
  if (sqrt(rho_new) <= cg->tol * cg->bnorm) cg->status[s] = ST_RCONV;
  else if (itn >= cg->maxit) cg->status[s] = ST_MAXIT;
}

// ------------------------------------------------------------------ KC (combine)
struct CmbInfo {
  int sid[32];
  int mode[32];       // 0 skip, 1 x only, 2 full
  int nw[32];
  int hasg[32];
  double al[32], be[32], rinv[32];
  int sto[32];        // store slot or -1
};

__global__ void __launch_bounds__(kNT) cg_combine_grp(CgDev* __restrict__ cg) {
  __shared__ double sMu[32][kMaxM + 1];  // mu of the tile's shifts
  __shared__ CmbInfo ci;
  __shared__ int s_last;
  const int g = blockIdx.y, tile = blockIdx.z, chunk = blockIdx.x;
  const int* gm = cg->gmeta;
  const int S = min(32, gm[4 + g] - tile * 32);
  if (S <= 0) return;
  const int J = cg->grp.J[g];
  const int64_t N = cg->N;
  const int64_t ldw = cg->grp.ldw;
  const double* __restrict__ W = cg->grp.W[g];
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int k = tid;
    ci.mode[k] = 0; ci.sto[k] = -1; ci.al[k] = ci.be[k] = ci.rinv[k] = 0.0; ci.nw[k] = 0; ci.hasg[k] = 0;
    ci.sid[k] = 0;
    if (k < S) {
      const int s = cg->glist[gm[g] + tile * 32 + k];
      const int st = cg->status[s];
      ci.sid[k] = s;
      const double a = cg->alpha[s];
      ci.al[k] = a;
      ci.mode[k] = (st == ST_ACTIVE) ? 2 : (((st == ST_RCONV || st == ST_MAXIT) && a != 0.0) ? 1 : 0);
      ci.be[k] = cg->beta[s];
      ci.hasg[k] = cg->hasg[s];
      ci.nw[k] = cg->mloc[s] - cg->hasg[s];
      if (ci.mode[k] == 2 && cg->store && cg->store_cnt[s] < cg->store_cap) {
        ci.sto[k] = cg->store_cnt[s];
        ci.rinv[k] = 1.0 / sqrt(cg->rho[s]);
      }
    }
  }
  for (int e = tid; e < 32 * kMaxM; e += kNT) {
    const int k = e / kMaxM, j = e - k * kMaxM;
    sMu[k][j] = 0.0;
  }
  __syncthreads();
  for (int e = tid; e < 32 * kMaxM; e += kNT) {
    const int k = e / kMaxM, j = e - k * kMaxM;
    if (k < S) sMu[k][j] = cg->coef[(int64_t)ci.sid[k] * kMaxM + j];
  }
  __syncthreads();
  const int64_t rbeg = (int64_t)chunk * cg->rowsG;
  const int64_t rend = min(N, rbeg + cg->rowsG);
  for (int64_t r0 = rbeg; r0 < rend; r0 += kSub) {
    const int64_t i = r0 + tid;
    if (i >= rend) break;
    double wv[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) wv[j] = j < J ? __ldg(W + (int64_t)j * ldw + i) : 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) {
      if (k0 < S) {
        double pv[4], xv[4], rv[4], gv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u;
          pv[u] = xv[u] = rv[u] = gv[u] = 0.0;
          if (k < S && ci.mode[k]) {
            const int s = ci.sid[k];
            pv[u] = cg->P[(int64_t)s * N + i];
            xv[u] = cg->X[(int64_t)s * cg->ldx + i];
            if (ci.mode[k] == 2) {
              rv[u] = cg->R[(int64_t)s * N + i];
              if (ci.hasg[k]) gv[u] = __ldg(cg->Ghat + (int64_t)s * cg->ldgh + i);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u;
          if (k < S && ci.mode[k]) {
            const int s = ci.sid[k];
            cg->X[(int64_t)s * cg->ldx + i] = fma(ci.al[k], pv[u], xv[u]);
            if (ci.mode[k] == 2) {
              double pn = fma(ci.be[k], pv[u], rv[u]);
              const int nw = ci.nw[k];
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (j < nw) pn = fma(-sMu[k][j], wv[j], pn);
              if (ci.hasg[k]) pn = fma(-sMu[k][nw], gv[u], pn);
              cg->P[(int64_t)s * N + i] = pn;
              if (ci.sto[k] >= 0)
                cg->store[((int64_t)s * cg->store_cap + ci.sto[k]) * cg->lds + i] = rv[u] * ci.rinv[k];
            }
          }
        }
      }
    }
  }
  __threadfence();
  __syncthreads();
  unsigned* tick = cg->cntG + (size_t)(g * cg->maxtilesG + tile) * kTickStride;
  if (tid == 0) {
    const unsigned tk = atomicAdd(tick + 1, 1u);
    s_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  if (tid == 0) tick[1] = 0u;
  if (tid < S) {
    const int s = ci.sid[tid];
    const int st = cg->status[s];
    if (st == ST_ACTIVE && ci.sto[tid] >= 0) cg->store_cnt[s] += 1;
    if (st == ST_ACTIVE || st == ST_RCONV || st == ST_MAXIT) cg->alpha[s] = 0.0;
  }
}

static size_t update_smem() { return sizeof(double) * (32 + 32 + 32) * kHP; }

cudaError_t launch_cg_update_grp(CgDev* dev, const CgDev& host, int ngroups, int maxtiles, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(cg_update_grp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)update_smem());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(host.nchunkG, ngroups, maxtiles);
  count_launch();
  cg_update_grp<<<grid, kNT, update_smem(), st>>>(dev);
  return cudaGetLastError();
}

cudaError_t launch_cg_combine_grp(CgDev* dev, const CgDev& host, int ngroups, int maxtiles, cudaStream_t st) {
  dim3 grid(host.nchunkG, ngroups, maxtiles);
  count_launch();
  cg_combine_grp<<<grid, kNT, 0, st>>>(dev);
  return cudaGetLastError();
}

}  // namespace rsk
