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
constexpr int kQ = 64;          // rows per update sub-slab (cp.async staged)
constexpr int kQP = kQ + 1;     // odd pitch

__device__ __forceinline__ void cp_async8g(double* sdst, const double* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gsrc), "r"(sz) : "memory");
}

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
__global__ void __launch_bounds__(kNT, 3) cg_update_grp(CgDev* __restrict__ cg) {
  // dynamic smem: sA [32][kQP] | sR [32][kQP] | sW [32][kQP] | sZ [32][kQP]
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
  double* sR = dsm + 32 * kQP;
  double* sWv = sR + 32 * kQP;
  double* sZ = sWv + 32 * kQP;
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
  bool anyz = false;
  for (int k = 0; k < S; ++k) anyz |= (ti.hasg[k] != 0);
  // update role: row ur (of kQ), shifts k = uq + 4u
  const int ur = tid & (kQ - 1), uq = tid >> 6;
  // rho / zeta role: shift tk, 8-row segment tseg
  const int tk = tid & 31, tseg = tid >> 5;
  double prho = 0.0, pzet = 0.0;
  // GEMM role: k-block kb (4 shifts), j-block jb (4 rows of [AW;EW]), row group rg
  const int njb = (J2 > 16) ? 8 : 4;
  const int nrg = 32 / njb;
  const int rpg = kQ / nrg;
  const int kb = tid & 7, jb = (tid >> 3) & (njb - 1), rg = (tid >> 3) / njb;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  const int64_t rbeg = (int64_t)chunk * cg->rowsG;
  const int64_t rend = min(N, rbeg + cg->rowsG);
  for (int64_t r0 = rbeg; r0 < rend; r0 += kQ) {
    // ---- stage every operand of the sub-slab with cp.async (all loads in flight at once)
    const int nrow = (int)min((int64_t)kQ, rend - r0);
    for (int e = tid; e < J2 * kQ; e += kNT) {
      const int j = e / kQ, rr = e - j * kQ;
      const bool v = rr < nrow;
      const double* src = (j < J ? AW + (int64_t)j * ldw : EW + (int64_t)(j - J) * ldw) + r0 + rr;
      cp_async8g(sA + j * kQP + rr, v ? src : AW, v);
    }
    for (int e = tid; e < S * kQ; e += kNT) {
      const int k = e / kQ, rr = e - k * kQ;
      const bool v = rr < nrow;
      const int64_t off = (int64_t)ti.sid[k] * N + r0 + rr;
      cp_async8g(sR + k * kQP + rr, v ? cg->R + off : cg->R, v);
      cp_async8g(sWv + k * kQP + rr, v ? cg->Wv + off : cg->Wv, v);
      if (anyz) {
        const bool vz = v && ti.hasg[k];
        cp_async8g(sZ + k * kQP + rr, vz ? cg->ZGhat + (int64_t)ti.sid[k] * cg->ldgh + r0 + rr : cg->R, vz);
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    // ---- r' = r - alpha w (in shared memory), write back, zeta products
    const int64_t i = r0 + ur;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = uq + 4 * u;
      if (k < S) {
        const double rn = fma(-ti.al[k], sWv[k * kQP + ur], sR[k * kQP + ur]);
        sR[k * kQP + ur] = rn;
        if (anyz) sZ[k * kQP + ur] *= rn;
        if (ti.act[k] && ur < nrow) cg->R[(int64_t)ti.sid[k] * N + i] = rn;
      }
    }
    __syncthreads();
    // ---- rho, zeta partials over this thread's 8-row segment
    if (tk < S) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double rn = sR[tk * kQP + tseg * 8 + q];
        prho = fma(rn, rn, prho);
        if (anyz) pzet += sZ[tk * kQP + tseg * 8 + q];
      }
    }
    // ---- GEMM over this sub-slab: acc[a][b] += sum_rows sA[4jb+a][row] * sR[4kb+b][row]
    if (4 * jb < J2 && 4 * kb < S) {
#pragma unroll 4
      for (int rr = 0; rr < rpg; ++rr) {
        const int row = rg * rpg + rr;
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = sA[min(4 * jb + a, J2 - 1) * kQP + row];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = sR[(4 * kb + b) * kQP + row];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
      }
    }
    __syncthreads();
  }
  // ---- CTA-level reductions (once per chunk), fixed order through shared memory
  double* red = sR;                  // [nrg][4 njb][33] = 4224 doubles (spans sR | sWv | sZ head)
  double* red2 = sA;                 // [8][64] (sA is free after the last sub-slab)
  static_assert(3 * 32 * kQP >= 4224 && 32 * kQP >= 512, "reduction scratch");
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
    // software-pipelined over 4-shift batches: the loads of batch b+1 are issued before
    // the stores of batch b (program order keeps possibly-aliasing accesses in place)
    double buf[2][4][4];   // [parity][p, x, r, ghat][shift in batch]
    auto ld = [&](int k0, double (*v)[4]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u;
        v[0][u] = v[1][u] = v[2][u] = v[3][u] = 0.0;
        if (k < S && ci.mode[k]) {
          const int s = ci.sid[k];
          v[0][u] = cg->P[(int64_t)s * N + i];
          v[1][u] = cg->X[(int64_t)s * cg->ldx + i];
          if (ci.mode[k] == 2) {
            v[2][u] = cg->R[(int64_t)s * N + i];
            if (ci.hasg[k]) v[3][u] = __ldg(cg->Ghat + (int64_t)s * cg->ldgh + i);
          }
        }
      }
    };
    auto st = [&](int k0, double (*v)[4]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u;
        if (k < S && ci.mode[k]) {
          const int s = ci.sid[k];
          cg->X[(int64_t)s * cg->ldx + i] = fma(ci.al[k], v[0][u], v[1][u]);
          if (ci.mode[k] == 2) {
            double pn = fma(ci.be[k], v[0][u], v[2][u]);
            const int nw = ci.nw[k];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < nw) pn = fma(-sMu[k][j], wv[j], pn);
            if (ci.hasg[k]) pn = fma(-sMu[k][nw], v[3][u], pn);
            cg->P[(int64_t)s * N + i] = pn;
            if (ci.sto[k] >= 0)
              cg->store[((int64_t)s * cg->store_cap + ci.sto[k]) * cg->lds + i] = v[2][u] * ci.rinv[k];
          }
        }
      }
    };
    ld(0, buf[0]);
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) {
      if (k0 >= S) break;
      if (k0 + 4 < S) ld(k0 + 4, buf[((k0 >> 2) + 1) & 1]);
      st(k0, buf[(k0 >> 2) & 1]);
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

static size_t update_smem() { return sizeof(double) * 4 * 32 * kQP; }

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
