// Streaming persistent lockstep loop of the batched deflated CG (rsk_cg_recycled_batch)
// for images beyond L2 (C3, C4, C5): DESIGN.md §4.2b.
//
// Same recurrences as cg_persist.cu and the oracle O4 (oracle/defcg.py, reading D1):
//
//   A  w = A_gamma p (ACTIVE) or w = A_gamma x (RCONV: true-residual confirm): the strip
//      apply (strip_core.cuh), items = (shift, 64-column strip, row segment), one X.Y
//      partial per item                                                     -- barrier
//   B  alpha = rho / p.w from the item partials (fixed order); per 1024-row chunk and
//      pass of <= 32 shifts of one group: r = r - alpha w (or b - w), partial sums of
//      rho' = r.r, zeta = ZGhat.r and z = [AW ; EW]^T r (FP64 tensor cores)   -- barrier
//   B2 one CTA per shift: chunk sums in fixed order, mu = G^-1 z, beta, status -- barrier
//   C  x += alpha p ; p = r + beta p - W mu_W - ghat mu_g (W mu on the tensor cores);
//      residual store                                                         -- barrier
//
// Data movement: the per-shift vectors of phases B and C stream through two shared-
// memory stages of 8 shifts x 128 rows by 1-D bulk copies (cp.async.bulk, mbarrier
// completion) and go back by bulk stores, so the bytes in flight do not depend on
// registers or occupancy (two 8-warp CTAs per SM, <= 128 registers). The group columns
// AW, EW, W are read once per (chunk, pass) from HBM into L1 by the DMMA fragment loads
// and re-read from L1 by the other shift batches of the pass.
// Every sum has a fixed order that depends only on N and the launch geometry (segment
// rows, chunk rows): results per shift do not depend on the other shifts of the batch.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "strip_core.cuh"

namespace rsk {

constexpr int kSMaxShift = 256;
constexpr int kSPV = kMaxM + 1;     // partial slots per (shift, chunk): z_0..z_{m-1}, rho at kMaxM
constexpr int kSRows = 128;         // rows per stage
constexpr int kSChunk = 1024;       // rows per partial chunk (8 stages)
constexpr int kSB = 8;              // shifts per stage batch
constexpr int kSVec = 4;            // vectors per shift in a stage
constexpr int kSAcc = 34;           // per pass shift: zA[16], zE[16], rho, zeta

__device__ unsigned long long g_sprof[8];   // per-phase ns (RSK_PERSIST_PROF), block 0's view

struct alignas(64) StreamParams {
  StripParams sp;     // apply: mapX over P (ld N), mapX2 over the iterates X (ld ldx), Y = Wv
  CgDev* cg;
  double* partA;      // [shift][ipv]
  double* partB;      // [shift][kSPV][nchunk]
  unsigned* bar;      // grid barrier {count, generation}
  int* nactive;
  int* iters_done;
  int nshift;
  int nchunk;
  int ipv;            // apply items per vector (segments x strips)
  int max_iters;
  int prof;
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

// sense-reversing grid barrier (cooperative launch: all CTAs co-resident). Generic and
// async-proxy (TMA, bulk copy) accesses on either side are ordered by the proxy fences.
__device__ __forceinline__ void sgrid_sync(unsigned* bar, unsigned& gen) {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u) + 1u;
    if (arrived == gridDim.x) {
      bar[0] = 0u;
      __threadfence();
      s_st_release(bar + 1, gen + 1u);
    } else {
      while (s_ld_acquire(bar + 1) == gen) {
      }
    }
    __threadfence();
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
  }
  gen += 1u;
  __syncthreads();
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

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

// passes: up to 32 consecutive entries of one group
__device__ __forceinline__ int s_pass_end(const SList& L, int li0) {
  const int g = le_grp(L.e[li0]);
  int li1 = li0;
  while (li1 < L.n && li1 < li0 + 32 && le_grp(L.e[li1]) == g) ++li1;
  return li1;
}
__device__ __forceinline__ int s_npass(const SList& L) {
  int np = 0;
  for (int li = 0; li < L.n; li = s_pass_end(L, li)) ++np;
  return np;
}
__device__ __forceinline__ int s_pass_start(const SList& L, int k) {
  int li = 0;
  for (int i = 0; i < k; ++i) li = s_pass_end(L, li);
  return li;
}

// ---------------------------------------------------------------- shared memory plan
// [0, SCRATCH): the strip apply's input / x-pass rings (phase A) or the B / C stages,
// pass accumulators, cross-warp reduction and per-pass scalars (phases B, B2, C);
// [SCRATCH, ...): the strip apply's persistent tail (corrections, mbarriers) + 2 stage
// mbarriers -- never touched by another phase
constexpr int kSPS = 8;   // per pass entry: beta, 1/|r|, slot, flags, alpha
template <int R>
struct SCfg {
  static constexpr int STAGE = kSB * kSVec * kSRows;      // doubles per stage
  static constexpr int OFF_ST = 0;                        // 2 stages
  static constexpr int OFF_ACC = OFF_ST + 2 * STAGE;      // [32][kSAcc]
  static constexpr int OFF_RED = OFF_ACC + 32 * kSAcc;    // [8 warps][4 acc][64]
  static constexpr int OFF_PS = OFF_RED + 8 * 4 * 64;     // [32][kSPS]
  static constexpr int BC_END = OFF_PS + 32 * kSPS;
  static constexpr int RING_END = StripCfg<R>::RING_END;
  static constexpr int SCRATCH = al16(BC_END > RING_END ? BC_END : RING_END);
  using Strip = StripCfg<R, SCRATCH>;
  static constexpr int OFF_BAR = Strip::DBL;              // 2 stage mbarriers
  static constexpr int DBL = OFF_BAR + 2;
  static constexpr size_t SMEM = sizeof(double) * (size_t)DBL;
};

// ---------------------------------------------------------------- phase A
template <int R>
__device__ __forceinline__ void s_phase_a(const StreamParams& P, const SList& L, double* smem, StripRing& ring,
                                          const double* bx, const double* ay) {
  using Core = StripCore<R, SCfg<R>::SCRATCH>;
  const int n = L.n;
  const int nitems = n * P.ipv;
  CgDev* cg = P.cg;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int li = it % n, ss = it / n;
    const int v = L.e[li];
    const int s = le_sid(v);
    const bool rconv = le_mode(v) == ST_RCONV;
    const int strip = ss % P.sp.nstrip, seg = ss / P.sp.nstrip;
    const double dot = Core::item(P.sp, smem, ring, bx, ay, s, strip, seg, rconv);
    if (!rconv) {
      const double bs = block_sum(dot, smem + SCfg<R>::Strip::OFF_RED);
      if (threadIdx.x == 0) P.partA[(size_t)s * P.ipv + ss] = bs;
    }
  }
  (void)cg;
}

// ---------------------------------------------------------------- phase B
// stage layout: [8 shifts][w | r | zg | -][128]
template <int R>
__device__ void s_phase_b(const StreamParams& P, const SList& L, double* smem, double* s_alpha, unsigned& bpar) {
  using SC = SCfg<R>;
  CgDev* cg = P.cg;
  const int n = L.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t N = cg->N;
  // alpha = rho / pi, pi = the shift's item partials in item order (every CTA, same tree)
  for (int li = warp; li < n; li += 8) {
    const int v = L.e[li];
    double a = 0.0;
    if (le_mode(v) == ST_ACTIVE) {
      const int s = le_sid(v);
      const double* pa = P.partA + (size_t)s * P.ipv;
      double pi = 0.0;
      for (int c = lane; c < P.ipv; c += 32) pi += __ldcg(pa + c);
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
  double* ST = smem + SC::OFF_ST;
  double* ACC = smem + SC::OFF_ACC;
  double* RED = smem + SC::OFF_RED;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SC::OFF_BAR);
  const int npass = s_npass(L);
  const int nunits = P.nchunk * npass;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int c = u % P.nchunk, pk = u / P.nchunk;
    const int li0 = s_pass_start(L, pk), li1 = s_pass_end(L, li0);
    const int np = li1 - li0;
    const int grp = le_grp(L.e[li0]);
    const int J = cg->grp.J[grp];
    const double* AWg = cg->grp.AW[grp];
    const double* EWg = cg->grp.EW[grp];
    const int64_t ldw = cg->grp.ldw;
    const int64_t cbeg = (int64_t)c * kSChunk;
    const int nsub = (int)((imin64(N, cbeg + kSChunk) - cbeg + kSRows - 1) / kSRows);
    const int nb = (np + kSB - 1) / kSB;
    const int nsteps = nsub * nb;
    for (int e = tid; e < np * kSAcc; e += blockDim.x) ACC[e] = 0.0;
    // stage issue: step k = (sub k / nb, batch k % nb)
    auto issue = [&](int k) {
      const int sub = k / nb, b = k % nb;
      const int64_t r0 = cbeg + (int64_t)sub * kSRows;
      const int nr = (int)imin64(kSRows, N - r0);
      const unsigned bytes = 8u * nr;
      double* stg = ST + (k & 1) * SC::STAGE;
      unsigned tot = 0;
      for (int k8 = 0; k8 < kSB; ++k8) {
        const int li = li0 + b * kSB + k8;
        if (li >= li1) break;
        const int v = L.e[li];
        const int s = le_sid(v);
        tot += 2 * bytes + (le_hg(v) ? bytes : 0);
      }
      mbar_expect_tx(bars + (k & 1), tot);
      for (int k8 = 0; k8 < kSB; ++k8) {
        const int li = li0 + b * kSB + k8;
        if (li >= li1) break;
        const int v = L.e[li];
        const int s = le_sid(v);
        double* d = stg + k8 * kSVec * kSRows;
        bulk_load(d, cg->Wv + (int64_t)s * N + r0, bytes, bars + (k & 1));
        bulk_load(d + kSRows, cg->R + (int64_t)s * N + r0, bytes, bars + (k & 1));
        if (le_hg(v)) bulk_load(d + 2 * kSRows, cg->ZGhat + (int64_t)s * cg->ldgh + r0, bytes, bars + (k & 1));
      }
    };
    if (tid == 0) {
      bulk_wait_read0();   // the previous unit's last bulk stores have read their stage
      issue(0);
    }
    __syncthreads();   // ACC zeroed
    for (int k = 0; k < nsteps; ++k) {
      const int sub = k / nb, b = k % nb;
      const int64_t r0 = cbeg + (int64_t)sub * kSRows;
      const int nr = (int)imin64(kSRows, N - r0);
      double* stg = ST + (k & 1) * SC::STAGE;
      if (tid == 0 && k + 1 < nsteps) {
        bulk_wait_read0();   // step k-1's bulk stores have read the other stage
        issue(k + 1);
      }
      // A fragments of this warp's 16 rows (group columns 8 mb + g), before the stage wait
      double aA[4][2], aE[4][2];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int row = warp * 16 + kk * 4 + q;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
          const int col = 8 * mb + g;
          const bool va = row < nr && col < J;
          aA[kk][mb] = va ? __ldg(AWg + (int64_t)col * ldw + r0 + row) : 0.0;
          aE[kk][mb] = va ? __ldg(EWg + (int64_t)col * ldw + r0 + row) : 0.0;
        }
      }
      mbar_wait(bars + (k & 1), (bpar >> (k & 1)) & 1u);
      bpar ^= 1u << (k & 1);
      // (a) r update, rho and zeta: warp = shift of the batch, lane = 4 rows
      {
        const int li = li0 + b * kSB + warp;
        double rh = 0.0, zt = 0.0;
        if (li < li1) {
          const int v = L.e[li];
          const bool act = le_mode(v) == ST_ACTIVE;
          const double al = s_alpha[li];
          double* d = stg + warp * kSVec * kSRows;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int row = lane * 4 + h;
            double rn = 0.0;
            if (row < nr) {
              const double wv = d[row];
              rn = act ? fma(-al, wv, d[kSRows + row]) : __ldg(cg->b + r0 + row) - wv;
              rh = fma(rn, rn, rh);
              if (le_hg(v)) zt = fma(d[2 * kSRows + row], rn, zt);
            }
            d[kSRows + row] = rn;
          }
        } else {
          double* d = stg + warp * kSVec * kSRows;
#pragma unroll
          for (int h = 0; h < 4; ++h) d[kSRows + lane * 4 + h] = 0.0;
        }
        rh = warp_sum(rh);
        zt = warp_sum(zt);
        if (lane == 0 && li < li1) {
          double* a = ACC + (li - li0) * kSAcc;
          a[32] += rh;
          a[33] += zt;
        }
      }
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        for (int k8 = 0; k8 < kSB; ++k8) {
          const int li = li0 + b * kSB + k8;
          if (li >= li1) break;
          const int s = le_sid(L.e[li]);
          bulk_store(cg->R + (int64_t)s * N + r0, stg + k8 * kSVec * kSRows + kSRows, 8u * nr);
        }
        bulk_commit();
      }
      // (b) [AW ; EW]^T R on the tensor cores: warp = 16 rows (4 k-steps), D[j][shift]
      {
        double dA[2][2], dE[2][2];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) dA[mb][0] = dA[mb][1] = dE[mb][0] = dE[mb][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int row = warp * 16 + kk * 4 + q;
          const double bv = stg[g * kSVec * kSRows + kSRows + row];   // r'(shift g, row)
#pragma unroll
          for (int mb = 0; mb < 2; ++mb) {
            if (mb == 1 && J <= 8) break;
            dmma(dA[mb][0], dA[mb][1], aA[kk][mb], bv);
            dmma(dE[mb][0], dE[mb][1], aE[kk][mb], bv);
          }
        }
        // D[m = 8 mb + g][n = 2q + h] of this warp -> RED[warp][acc][m * 8 + n]
        double* rw = RED + warp * 4 * 64;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            rw[(2 * mb + 0) * 64 + g * 8 + 2 * q + h] = dA[mb][h];
            rw[(2 * mb + 1) * 64 + g * 8 + 2 * q + h] = dE[mb][h];
          }
      }
      __syncthreads();
      // fixed-order sum over the 8 warps into the pass accumulators
      for (int e = tid; e < kSB * 32; e += blockDim.x) {
        const int k8 = e >> 5, slot = e & 31;        // slot: 0..15 zA, 16..31 zE
        const int li = li0 + b * kSB + k8;
        const int j = slot & 15, isE = slot >> 4;
        if (li >= li1 || j >= J) continue;
        const int mb = j >> 3, m = j & 7;
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += RED[w * 4 * 64 + (2 * mb + isE) * 64 + m * 8 + k8];
        ACC[(li - li0) * kSAcc + slot] += t;
      }
      __syncthreads();
    }
    // chunk partials: z_j = zA_j + gamma zE_j (W columns), zeta (carried column), rho
    for (int e = tid; e < np * kSPV; e += blockDim.x) {
      const int k = e / kSPV, j = e - k * kSPV;
      const int v = L.e[li0 + k];
      const int s = le_sid(v);
      const int nw = le_m(v) - le_hg(v);
      const double* a = ACC + k * kSAcc;
      double val;
      if (j < nw) val = fma(cg->gam[s], a[16 + j], a[j]);
      else if (le_hg(v) && j == nw) val = a[33];
      else if (j == kMaxM) val = a[32];
      else continue;
      P.partB[((size_t)s * kSPV + j) * P.nchunk + c] = val;
    }
    __syncthreads();
  }
  if (tid == 0) bulk_wait0();   // every bulk store of this phase complete before the barrier
}

// ---------------------------------------------------------------- phase B2
__device__ void s_phase_b2(const StreamParams& P, const SList& L, double* smem) {
  CgDev* cg = P.cg;
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
        const double* pj = P.partB + ((size_t)s * kSPV + j) * P.nchunk;
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
        int c = lane;
        for (; c + 96 < P.nchunk; c += 128) {
          t0 += __ldcg(pj + c); t1 += __ldcg(pj + c + 32); t2 += __ldcg(pj + c + 64); t3 += __ldcg(pj + c + 96);
        }
        for (; c < P.nchunk; c += 32) t0 += __ldcg(pj + c);
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
        if (st == ST_ACTIVE) {
          const int itn = cg->iters[s] + 1;
          cg->iters[s] = itn;
          cg->beta[s] = rho_new / cg->rho[s];
          cg->rho[s] = rho_new;
          if (conv) nst = ST_RCONV;
          else if (itn >= cg->maxit) nst = ST_MAXIT;
          else newp = true;
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
          newp = true;
        }
      }
      if (newp) {
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

// ---------------------------------------------------------------- phase C
// stage layout: [8 shifts][p | r | x | ghat][128]
template <int R>
__device__ void s_phase_c(const StreamParams& P, const SList& L, double* smem, const double* s_alpha, unsigned& bpar) {
  using SC = SCfg<R>;
  CgDev* cg = P.cg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t N = cg->N;
  double* ST = smem + SC::OFF_ST;
  double* PS = smem + SC::OFF_PS;   // per pass entry: beta, 1/|r|, slot, flags, alpha
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SC::OFF_BAR);
  const int npass = s_npass(L);
  const int nunits = P.nchunk * npass;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int c = u % P.nchunk, pk = u / P.nchunk;
    const int li0 = s_pass_start(L, pk), li1 = s_pass_end(L, li0);
    const int np = li1 - li0;
    const int grp = le_grp(L.e[li0]);
    const int J = cg->grp.J[grp];
    const double* Wg = cg->grp.W[grp];
    const int64_t ldw = cg->grp.ldw;
    const int64_t cbeg = (int64_t)c * kSChunk;
    const int nsub = (int)((imin64(N, cbeg + kSChunk) - cbeg + kSRows - 1) / kSRows);
    const int nb = (np + kSB - 1) / kSB;
    const int nsteps = nsub * nb;
    // per entry: flags 1 = x += alpha p, 2 = new p (status after B2 is ACTIVE)
    if (tid < np) {
      const int li = li0 + tid;
      const int s = le_sid(L.e[li]);
      const int st = cg->status[s];
      const int slot = (st == ST_ACTIVE) ? cg->stslot[s] : -1;
      int f = 0;
      if (le_mode(L.e[li]) == ST_ACTIVE && s_alpha[li] != 0.0) f |= 1;
      if (st == ST_ACTIVE) f |= 2;
      double* ps = PS + tid * kSPS;
      ps[0] = cg->beta[s];
      ps[1] = (slot >= 0) ? 1.0 / sqrt(cg->rho[s]) : 0.0;
      ps[2] = (double)slot;
      ps[3] = (double)f;
      ps[4] = s_alpha[li];
    }
    __syncthreads();
    auto issue = [&](int k) {
      const int sub = k / nb, b = k % nb;
      const int64_t r0 = cbeg + (int64_t)sub * kSRows;
      const int nr = (int)imin64(kSRows, N - r0);
      const unsigned bytes = 8u * nr;
      double* stg = ST + (k & 1) * SC::STAGE;
      unsigned tot = 0;
      for (int k8 = 0; k8 < kSB; ++k8) {
        const int li = li0 + b * kSB + k8;
        if (li >= li1) break;
        const int f = (int)PS[(li - li0) * kSPS + 3];
        if (!f) continue;
        tot += bytes;                                              // p
        if (f & 1) tot += bytes;                                   // x
        if (f & 2) tot += bytes + (le_hg(L.e[li]) ? bytes : 0);    // r, ghat
      }
      mbar_expect_tx(bars + (k & 1), tot);
      for (int k8 = 0; k8 < kSB; ++k8) {
        const int li = li0 + b * kSB + k8;
        if (li >= li1) break;
        const int f = (int)PS[(li - li0) * kSPS + 3];
        if (!f) continue;
        const int v = L.e[li];
        const int s = le_sid(v);
        double* d = stg + k8 * kSVec * kSRows;
        bulk_load(d, cg->P + (int64_t)s * N + r0, bytes, bars + (k & 1));
        if (f & 1) bulk_load(d + 2 * kSRows, cg->X + (int64_t)s * cg->ldx + r0, bytes, bars + (k & 1));
        if (f & 2) {
          bulk_load(d + kSRows, cg->R + (int64_t)s * N + r0, bytes, bars + (k & 1));
          if (le_hg(v)) bulk_load(d + 3 * kSRows, cg->Ghat + (int64_t)s * cg->ldgh + r0, bytes, bars + (k & 1));
        }
      }
    };
    if (tid == 0 && nsteps > 0) {
      bulk_wait_read0();
      issue(0);
    }
    const int nkk = (J + 3) >> 2;
    for (int k = 0; k < nsteps; ++k) {
      const int sub = k / nb, b = k % nb;
      const int64_t r0 = cbeg + (int64_t)sub * kSRows;
      const int nr = (int)imin64(kSRows, N - r0);
      double* stg = ST + (k & 1) * SC::STAGE;
      if (tid == 0 && k + 1 < nsteps) {
        bulk_wait_read0();
        issue(k + 1);
      }
      // B fragments: mu of batch shift g, component 4 kk + q (0 unless a new p is formed)
      double bm[4];
      {
        const int li = li0 + b * kSB + g;
        const bool ok = li < li1 && (((int)PS[(li - li0) * kSPS + 3]) & 2);
        const int v = ok ? L.e[li] : 0;
        const int nw = ok ? le_m(v) - le_hg(v) : 0;
        const double* cf = cg->coef + (int64_t)le_sid(v) * kMaxM;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int j = 4 * kk + q;
          bm[kk] = (ok && j < nw) ? cf[j] : 0.0;
        }
      }
      // W fragments of this warp's two 8-row blocks, issued before the stage wait
      double a[2][4];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int row = (2 * warp + rr) * 8 + g;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int j = 4 * kk + q;
          a[rr][kk] = (kk < nkk && j < J && row < nr) ? __ldg(Wg + (int64_t)j * ldw + r0 + row) : 0.0;
        }
      }
      mbar_wait(bars + (k & 1), (bpar >> (k & 1)) & 1u);
      bpar ^= 1u << (k & 1);
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int row = (2 * warp + rr) * 8 + g;
        double d[2] = {0.0, 0.0};
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (kk < nkk) dmma(d[0], d[1], a[rr][kk], bm[kk]);
        if (row < nr) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k8 = 2 * q + h;
            const int li = li0 + b * kSB + k8;
            if (li >= li1) continue;
            const double* ps = PS + (li - li0) * kSPS;
            const int f = (int)ps[3];
            if (!f) continue;
            const int v = L.e[li];
            double* ds = stg + k8 * kSVec * kSRows;
            const double pv = ds[row];
            if (f & 1) ds[2 * kSRows + row] = fma(ps[4], pv, ds[2 * kSRows + row]);
            if (f & 2) {
              const double rv = ds[kSRows + row];
              double pn = fma(ps[0], pv, rv) - d[h];
              if (le_hg(v)) pn = fma(-cg->coef[(int64_t)le_sid(v) * kMaxM + le_m(v) - 1], ds[3 * kSRows + row], pn);
              ds[row] = pn;
              const int slot = (int)ps[2];
              if (slot >= 0) {
                const int s = le_sid(v);
                cg->store[((int64_t)s * cg->store_cap + slot) * cg->lds + r0 + row] = rv * ps[1];
              }
            }
          }
        }
      }
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        for (int k8 = 0; k8 < kSB; ++k8) {
          const int li = li0 + b * kSB + k8;
          if (li >= li1) break;
          const int f = (int)PS[(li - li0) * kSPS + 3];
          const int s = le_sid(L.e[li]);
          const double* ds = stg + k8 * kSVec * kSRows;
          if (f & 2) bulk_store(cg->P + (int64_t)s * N + r0, ds, 8u * nr);
          if (f & 1) bulk_store(cg->X + (int64_t)s * cg->ldx + r0, ds + 2 * kSRows, 8u * nr);
        }
        bulk_commit();
      }
    }
    __syncthreads();
  }
  if (tid == 0) bulk_wait0();
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

  CgDev* cg = P.cg;
  const int ns = P.nshift;
  const int tid = threadIdx.x;
  // strip-apply barriers and the B/C stage barriers are distinct mbarriers
  Core::init(smem, P.sp);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) mbar_init(reinterpret_cast<uint64_t*>(smem + SC::OFF_BAR) + b, 1);
    mbar_fence_init();
  }
  double bx[SC::Strip::KS], ay[SC::Strip::KS];
  Core::frags(P.sp, bx, ay);
  StripRing ring{0u, 0u};
  unsigned bpar = 0u;
  unsigned gen = s_ld_acquire(P.bar + 1);
  int cur = 0;
  s_build_list(cg, ns, lists[0], tmp);
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
  mark(7);
  for (; it < P.max_iters; ++it) {
    SList& L = lists[cur];
    if (L.n == 0) break;
    s_phase_a<R>(P, L, smem, ring, bx, ay);
    mark(0);
    sgrid_sync(P.bar, gen);
    mark(1);
    s_phase_b<R>(P, L, smem, s_alpha, bpar);
    mark(2);
    sgrid_sync(P.bar, gen);
    mark(1);
    s_phase_b2(P, L, smem);
    mark(3);
    sgrid_sync(P.bar, gen);
    mark(1);
    SList& NL = lists[cur ^ 1];
    s_build_list(cg, ns, NL, tmp);   // statuses are stable until the next phase A
    s_phase_c<R>(P, L, smem, s_alpha, bpar);
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

// ---------------------------------------------------------------- host side
bool strip_fill_params(Handle* h, StripParams& p, const double* X, int64_t ldx, const double* X2, int64_t ldx2,
                       int64_t nvec_map, double* Y, int64_t ldy, double* EY, int64_t ldey, const double* gamma,
                       int mode, int seg_rows);

int stream_seg_rows(int64_t ny) { return ny > 512 ? 256 : 128; }
int stream_ipv(const Handle* h) {
  const int seg = stream_seg_rows(h->ny);
  return (int)((h->nx + kStripW - 1) / kStripW) * (int)((h->ny + seg - 1) / seg);
}
int stream_nchunk(int64_t N) { return (int)((N + kSChunk - 1) / kSChunk); }
int stream_grid(const Handle* h) { return kStripCtasPerSm * h->sm_count; }
int stream_pv() { return kSPV; }

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
  static_assert(SC::SMEM <= 110 * 1024, "two CTAs per SM");
  auto kfn = cg_stream_kernel<R>;
  static int b = 0;
  if (b == 0) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SC::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kfn, kAT, SC::SMEM);
    if (e != cudaSuccess) return e;
    if (b < 1) b = -1;
  }
  if (b < 1) { *ok = false; return cudaSuccess; }
  const int grid = (b < kStripCtasPerSm ? b : kStripCtasPerSm) * sm_count;
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
  if ((N & 1) || (hc.ldx & 1) || (hc.Ghat && (hc.ldgh & 1)) || !al16p(hc.X) || !al16p(hc.R) || !al16p(hc.P) ||
      !al16p(hc.Wv) || (hc.Ghat && (!al16p(hc.Ghat) || !al16p(hc.ZGhat))))
    return cudaSuccess;
  StreamParams prm;
  const int seg = stream_seg_rows(h->ny);
  if (!strip_fill_params(h, prm.sp, hc.P, N, hc.X, hc.ldx, hc.nshift, hc.Wv, N, nullptr, 0, hc.gam,
                         RSK_APPLY_SHIFTED, seg))
    return cudaSuccess;
  prm.sp.want_dot = 1;
  prm.cg = dev;
  prm.partA = partA;
  prm.partB = partB;
  prm.bar = bar;
  prm.nactive = nactive;
  prm.iters_done = iters_done;
  prm.nshift = hc.nshift;
  prm.nchunk = stream_nchunk(N);
  prm.ipv = prm.sp.nseg * prm.sp.nstrip;
  prm.max_iters = max_iters;
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
