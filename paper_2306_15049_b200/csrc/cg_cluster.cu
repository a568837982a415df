// Cluster-per-shift deflated CG (rsk_cg_recycled_batch, images whose working set sits
// in L2): a thread-block cluster of kCS CTAs (one per SM) owns ONE shift at a time and
// iterates it to completion; clusters take shifts from a device queue, so shifts with
// 20 iterations and shifts with 2000 never wait on each other (no lockstep tail). All
// reductions cross the cluster through distributed shared memory (DSMEM) in a fixed
// CTA-rank order, and the only synchronisation is the hardware cluster barrier
// (3 per iteration), instead of grid barriers or kernel boundaries.
//
// Recurrences are exactly those of the oracle O4 (oracle/defcg.py; reading D1):
//   A  w = A_gamma p (LOOP) or A_gamma x (CONFIRM); pi = p.w; alpha = rho / pi
//   B  r = r - alpha w (LOOP) or b - w (CONFIRM); rho' = r.r; z = Z^T r
//      -> mu = G^-1 z, beta, status (replicated identically in every CTA)
//   C  x += alpha p; p = r + beta p - W mu_W - ghat mu_g; residual store
// A shift's arithmetic depends only on N and the cluster size: results are bitwise
// independent of the batch composition and of the GPU count under shift sharding.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "apply_core.cuh"

namespace rsk {

namespace cgx = cooperative_groups;

constexpr int kCV = kMaxM + 1;   // partial slots: z_0..z_{m-1}, rho at kMaxM
constexpr int kCW = kAT / 32;

__device__ unsigned long long g_cprof[8];   // per-phase ns of cluster 0 rank 0 (RSK_CLUSTER_PROF)

struct alignas(64) ClusterParams {
  ApplyParams ap;      // X = P, X2 = caller x, Y = Wv, want_dot, cg = null
  CgDev* cg;
  unsigned* queue;     // next shift index (device counter, zeroed by the host)
  const int* order;    // start order of the shifts (or null: 0..nshift-1)
  double* zw;          // [cluster][16][N]: Z = AW + gamma EW of the cluster's shift
  int nshift;
  int64_t rows;        // rows per CTA of a cluster
  int prof;
  int smem_r;          // 1: the CTA's rows of r live in shared memory for the whole shift
};

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// r = r - alpha w (loop) or b - w (confirm) over this CTA's rows; per-warp sums of
// z_j = Z_j . r (j < nw), ZGhat . r (slot nw) and r . r (slot kMaxM) into red[warp][slot].
// Separate function: its own register allocation, not the apply's.
template <int MW, int UNR>
__device__ __noinline__ void cluster_update_rows_t(double* __restrict__ Rv, const double* __restrict__ Wv,
                                                 const double* __restrict__ b, const double* __restrict__ Zs,
                                                 const double* __restrict__ Zg, int64_t N, int64_t rbeg,
                                                 int64_t rend, bool loop, double alpha, int nw, int hg,
                                                 double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double acc[MW], accg = 0.0, accr = 0.0;
#pragma unroll
  for (int j = 0; j < MW; ++j) acc[j] = 0.0;
  // pairs of rows through 16-byte loads (rows rbeg.. are even-aligned; an odd tail row
  // takes the scalar path)
  const int64_t npair = (rend - rbeg) >> 1;
#pragma unroll UNR
  for (int64_t q = tid; q < npair; q += kAT) {
    const int64_t i = rbeg + 2 * q;
    const double2 wv = *reinterpret_cast<const double2*>(Wv + i);
    const double2 r0 = loop ? *reinterpret_cast<const double2*>(Rv + i) : __ldg(reinterpret_cast<const double2*>(b + i));
    double2 rn;
    rn.x = loop ? fma(-alpha, wv.x, r0.x) : r0.x - wv.x;
    rn.y = loop ? fma(-alpha, wv.y, r0.y) : r0.y - wv.y;
    // every load of the row pair is issued before the first FMA that consumes one (the
    // scheduler otherwise serialises them through one register quad: 11 L2 round trips
    // per row pair instead of one)
    double2 zv[MW];
#pragma unroll
    for (int j = 0; j < MW; ++j)
      zv[j] = (j < nw) ? __ldcg(reinterpret_cast<const double2*>(Zs + (int64_t)j * N + i)) : make_double2(0.0, 0.0);
    const double2 zgv = hg ? __ldg(reinterpret_cast<const double2*>(Zg + i)) : make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(Rv + i) = rn;
#pragma unroll
    for (int j = 0; j < MW; ++j)
      if (j < nw) acc[j] = fma(zv[j].y, rn.y, fma(zv[j].x, rn.x, acc[j]));
    if (hg) accg = fma(zgv.y, rn.y, fma(zgv.x, rn.x, accg));
    accr = fma(rn.y, rn.y, fma(rn.x, rn.x, accr));
  }
  if (((rend - rbeg) & 1) && tid == 0) {
    const int64_t i = rend - 1;
    const double wv = Wv[i];
    const double rn = loop ? fma(-alpha, wv, Rv[i]) : __ldg(b + i) - wv;
    Rv[i] = rn;
#pragma unroll
    for (int j = 0; j < MW; ++j)
      if (j < nw) acc[j] = fma(Zs[(int64_t)j * N + i], rn, acc[j]);
    if (hg) accg = fma(__ldg(Zg + i), rn, accg);
    accr = fma(rn, rn, accr);
  }
#pragma unroll
  for (int j = 0; j < MW; ++j) {
    if (j < nw) {
      const double v = warp_sum(acc[j]);
      if (lane == 0) red[warp * kCV + j] = v;
    }
  }
  if (hg) {
    const double v = warp_sum(accg);
    if (lane == 0) red[warp * kCV + nw] = v;
  }
  const double v = warp_sum(accr);
  if (lane == 0) red[warp * kCV + kMaxM] = v;
}

// nw <= 8 (the configs' |J|): half the registers per row pair, four row pairs in flight
__device__ __forceinline__ void cluster_update_rows(double* Rv, const double* Wv, const double* b, const double* Zs,
                                                    const double* Zg, int64_t N, int64_t rbeg, int64_t rend,
                                                    bool loop, double alpha, int nw, int hg, double* red) {
  if (nw <= 8) cluster_update_rows_t<8, 4>(Rv, Wv, b, Zs, Zg, N, rbeg, rend, loop, alpha, nw, hg, red);
  else cluster_update_rows_t<16, 2>(Rv, Wv, b, Zs, Zg, N, rbeg, rend, loop, alpha, nw, hg, red);
}

// x += alpha p (upd_x); p = r + beta p - W mu_W - ghat mu_g; residual store (upd_p)
template <int MW, int UNR>
__device__ __noinline__ void cluster_combine_rows_t(double* __restrict__ Xv, double* __restrict__ Pv,
                                                  const double* __restrict__ Rv, const double* __restrict__ Wg,
                                                  int64_t ldw, const double* __restrict__ Gh, double* sto,
                                                  int64_t rbeg, int64_t rend, bool upd_x, bool upd_p,
                                                  double alpha, double beta, const double* smu, int nw, int hg,
                                                  double rinv) {
  const int tid = threadIdx.x;
  const double* mu = smu;   // shared-memory broadcast reads: registers stay free for the loads
  const double mug = hg ? smu[nw] : 0.0;
  auto row1 = [&](int64_t i) {
    const double pv = Pv[i];
    if (upd_x) Xv[i] = fma(alpha, pv, Xv[i]);
    if (upd_p) {
      const double rv = Rv[i];
      double pn = fma(beta, pv, rv);
#pragma unroll
      for (int j = 0; j < MW; ++j)
        if (j < nw) pn = fma(-mu[j], __ldg(Wg + (int64_t)j * ldw + i), pn);
      if (hg) pn = fma(-mug, __ldg(Gh + i), pn);
      Pv[i] = pn;
      if (sto) sto[i] = rv * rinv;
    }
  };
  const int64_t npair = (rend - rbeg) >> 1;
#pragma unroll UNR
  for (int64_t q = tid; q < npair; q += kAT) {
    const int64_t i = rbeg + 2 * q;
    const double2 pv = *reinterpret_cast<const double2*>(Pv + i);
    if (upd_x) {
      const double2 xv = *reinterpret_cast<const double2*>(Xv + i);
      *reinterpret_cast<double2*>(Xv + i) = make_double2(fma(alpha, pv.x, xv.x), fma(alpha, pv.y, xv.y));
    }
    if (upd_p) {
      const double2 rv = *reinterpret_cast<const double2*>(Rv + i);
      double2 wv[MW];   // all loads first (see cluster_update_rows)
#pragma unroll
      for (int j = 0; j < MW; ++j)
        wv[j] = (j < nw) ? __ldcg(reinterpret_cast<const double2*>(Wg + (int64_t)j * ldw + i)) : make_double2(0.0, 0.0);
      const double2 g = hg ? __ldcg(reinterpret_cast<const double2*>(Gh + i)) : make_double2(0.0, 0.0);
      double ax = fma(beta, pv.x, rv.x), ay = fma(beta, pv.y, rv.y);
      double bx = 0.0, by = 0.0;   // two partial chains (even / odd j) halve the FMA latency chain
#pragma unroll
      for (int j = 0; j < MW; ++j)
        if (j < nw) {
          if (j & 1) { bx = fma(-mu[j], wv[j].x, bx); by = fma(-mu[j], wv[j].y, by); }
          else { ax = fma(-mu[j], wv[j].x, ax); ay = fma(-mu[j], wv[j].y, ay); }
        }
      if (hg) { bx = fma(-mug, g.x, bx); by = fma(-mug, g.y, by); }
      *reinterpret_cast<double2*>(Pv + i) = make_double2(ax + bx, ay + by);
      if (sto) *reinterpret_cast<double2*>(sto + i) = make_double2(rv.x * rinv, rv.y * rinv);
    }
  }
  if (((rend - rbeg) & 1) && tid == 0) row1(rend - 1);
}

__device__ __forceinline__ void cluster_combine_rows(double* Xv, double* Pv, const double* Rv, const double* Wg,
                                                     int64_t ldw, const double* Gh, double* sto, int64_t rbeg,
                                                     int64_t rend, bool upd_x, bool upd_p, double alpha, double beta,
                                                     const double* smu, int nw, int hg, double rinv) {
  if (nw <= 8)
    cluster_combine_rows_t<8, 4>(Xv, Pv, Rv, Wg, ldw, Gh, sto, rbeg, rend, upd_x, upd_p, alpha, beta, smu, nw, hg, rinv);
  else
    cluster_combine_rows_t<16, 2>(Xv, Pv, Rv, Wg, ldw, Gh, sto, rbeg, rend, upd_x, upd_p, alpha, beta, smu, nw, hg, rinv);
}

// taller tiles for the cluster loop: a 256-wide image (C2) is 16 tiles of 64 rows, one per
// CTA of a 16-CTA cluster (the default 48-row tile gives 24 tiles = two rounds)
__host__ __device__ constexpr int cluster_tile_rows(int r) { return r <= 6 ? 64 : (r <= 8 ? 56 : tc_tile_rows(r)); }

template <int R, bool kTma>
__global__ void __launch_bounds__(kAT, 1) cg_cluster_kernel(const __grid_constant__ ClusterParams P) {
  extern __shared__ __align__(128) double smem[];
  using Core = ApplyCore<R, kTma, cluster_tile_rows(R)>;
  cgx::cluster_group cl = cgx::this_cluster();
  const int crank = (int)cl.block_rank();
  const int csz = (int)cl.num_blocks();
  __shared__ double s_part[kCV];       // this CTA's partial sums (pushed to the whole cluster)
  __shared__ double s_dot;
  // every CTA's partials, PUSHED here by their owners before the cluster barrier (remote
  // stores are fire-and-forget; after the barrier the reads are local shared memory)
  __shared__ double s_dots[16];
  __shared__ double s_parts[16][kCV];
  __shared__ int s_next;
  __shared__ double s_z[kCV];
  __shared__ double s_red[kCW][kCV];
  __shared__ double s_L[kMaxM * kMaxM];
  __shared__ double s_mu[kMaxM];
  __shared__ double s_dinv[kMaxM];
  __shared__ double s_alpha, s_beta, s_rinv;
  __shared__ int s_nst, s_slot, s_brk;
  __shared__ int s_list[1], s_lmode[1];

  CgDev* cg = P.cg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = cg->N;
  Core::init_bars(smem, P.ap);
  ApplyPipe pp{{0u, 0u}, 0};
  const int64_t rbeg = (int64_t)crank * P.rows;
  const int64_t rend = min(N, rbeg + P.rows);
  const int ntiles = P.ap.ntiles;
  const int tper = (ntiles + csz - 1) / csz;
  const int ibeg = min(ntiles, crank * tper), iend = min(ntiles, ibeg + tper);

  unsigned long long t0 = 0;
  auto mark = [&](int ph) {
    if (P.prof && blockIdx.x == 0 && tid == 0) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
      if (t0 && ph >= 0) g_cprof[ph] += t1 - t0;
      t0 = t1;
    }
  };
  for (;;) {
    if (crank == 0 && tid == 0) s_next = (int)atomicAdd(P.queue, 1u);
    cl_sync();
    const int idx = *cl.map_shared_rank(&s_next, 0);
    cl_sync();
    if (idx >= P.nshift) break;
    const int s = P.order ? P.order[idx] : idx;
    // ---- per-shift state (replicated in every CTA of the cluster)
    int mode = cg->status[s];
    if (mode != ST_ACTIVE && mode != ST_RCONV) continue;
    const int m = cg->mloc[s], hg = cg->hasg[s], nw = m - hg;
    const int grp = cg->group[s];
    const double gam = cg->gam[s];
    const double thr = cg->tol * cg->bnorm;
    double rho = cg->rho[s];
    int iters = cg->iters[s], nconf = cg->nconf[s], scnt = cg->store_cnt[s];
    double rho_true = cg->rho_true[s];
    const int maxit = cg->maxit, store_cap = cg->store_cap;
    const bool has_store = cg->store != nullptr;
    for (int e = tid; e < kMaxM * kMaxM; e += kAT) s_L[e] = cg->Lf[(int64_t)s * kMaxM * kMaxM + e];
    for (int j = tid; j < kMaxM; j += kAT) s_mu[j] = 0.0;
    if (tid == 0) { s_list[0] = s; }
    const double* AWg = cg->grp.AW[grp];
    const double* EWg = cg->grp.EW[grp];
    const double* Wg = cg->grp.W[grp];
    const int64_t ldw = cg->grp.ldw;
    double* Rg = cg->R + (int64_t)s * N;
    // r is touched only by its owning CTA (update, combine, store): keep the CTA's rows in
    // shared memory behind the apply's buffers for the whole shift (-24 B/px per iteration)
    double* sR = smem + ((Core::C::DBL + 1) & ~1);
    double* Rv = Rg;
    if (P.smem_r) {
      for (int64_t i = rbeg + tid; i < rend; i += kAT) sR[i - rbeg] = Rg[i];
      Rv = sR - rbeg;
    }
    double* __restrict__ Pv = cg->P + (int64_t)s * N;
    double* __restrict__ Wv = cg->Wv + (int64_t)s * N;
    double* __restrict__ Xv = cg->X + (int64_t)s * cg->ldx;
    const double* __restrict__ Gh = hg ? cg->Ghat + (int64_t)s * cg->ldgh : nullptr;
    const double* __restrict__ Zg = hg ? cg->ZGhat + (int64_t)s * cg->ldgh : nullptr;
    int status = mode;
    // Z_j = AW_j + gamma EW_j over this CTA's rows, once per shift (same fma as before:
    // the z partials are bitwise those of forming the column inside the loop)
    double* Zs = P.zw + (size_t)(blockIdx.x / csz) * 16 * N;
    for (int64_t i = rbeg + tid; i < rend; i += kAT) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nw) Zs[(int64_t)j * N + i] = fma(gam, __ldg(EWg + (int64_t)j * ldw + i), __ldg(AWg + (int64_t)j * ldw + i));
    }
    // reciprocal pivots of the Cholesky factor (the solves multiply)
    for (int i = tid; i < kMaxM; i += kAT) s_dinv[i] = (i < m) ? 1.0 / s_L[i + i * kMaxM] : 0.0;
    __syncthreads();

    for (;;) {
      // ================= A: w = A_gamma p (LOOP) or A_gamma x (CONFIRM)
      if (tid == 0) { s_lmode[0] = mode; s_dot = 0.0; }
      __syncthreads();
      mark(-1);
      Core::run(P.ap, smem, ibeg, iend, 1, pp, s_list, s_lmode, &s_dot);
      if (tid < csz) *cl.map_shared_rank(&s_dots[crank], tid) = s_dot;   // push p.w partial
      mark(0);
      cl_sync();
      mark(1);
      double alpha = 0.0;
      if (mode == ST_ACTIVE) {
        if (warp == 0) {   // the 16 CTA partials (pushed), fixed shuffle tree in rank order
          const double v = (lane < csz) ? s_dots[lane] : 0.0;
          const double pi = warp_sum(v);
          if (lane == 0) {
            s_brk = !(pi > 0.0) || !isfinite(pi);
            s_alpha = s_brk ? 0.0 : rho / pi;
          }
        }
        __syncthreads();
        if (s_brk) { status = ST_BREAKDOWN; break; }
        alpha = s_alpha;
      }
      mark(2);
      // ================= B: r update; partials of z = Z^T r and rho' = r.r
      cluster_update_rows(Rv, Wv, cg->b, Zs, Zg, N, rbeg, rend, mode == ST_ACTIVE, alpha, nw, hg, &s_red[0][0]);
      __syncthreads();
      mark(3);
      if (tid < kCV) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kCW; ++w) t += s_red[w][tid];
        s_part[tid] = t;
      }
      __syncthreads();
      for (int e = tid; e < csz * kCV; e += kAT) {   // push slot e % kCV to rank e / kCV
        const int c = e / kCV, slot = e - c * kCV;
        if (slot < m || slot == kMaxM) *cl.map_shared_rank(&s_parts[crank][slot], c) = s_part[slot];
      }
      cl_sync();
      mark(1);
      for (int e = tid; e < 32 * 16; e += kAT) {   // slot j = e / 16 from rank c = e % 16
        const int j = e >> 4, c = e & 15;
        const int slot = (j < kCV) ? j : kMaxM;
        const bool need = (j < m || j == kMaxM) && j < kCV;
        double v = (need && c < csz) ? s_parts[c][slot] : 0.0;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);   // within the 16-lane half
        if (need && c == 0) s_z[j] = v;
      }
      __syncthreads();
      // ---- scalars and status (identical in every CTA; warp 0, lanes redundant)
      if (warp == 0) {
        const double rho_new = s_z[kMaxM];
        const bool conv = sqrt(rho_new) <= thr;
        int nst = mode;
        bool newp = false;
        double beta = 0.0;
        if (mode == ST_ACTIVE) {
          iters += 1;
          beta = rho_new / rho;
          rho = rho_new;
          if (conv) nst = ST_RCONV;
          else if (iters >= maxit) nst = ST_MAXIT;
          else newp = true;
        } else {
          rho_true = rho_new;
          nconf += 1;
          if (conv) nst = ST_DONE;
          else if (iters >= maxit) nst = ST_MAXIT;
          else { nst = ST_ACTIVE; beta = 0.0; rho = rho_new; newp = true; }
        }
        int slot = -1;
        if (newp) {
          // mu = G^-1 z: L y = z then L^T mu = y, lane i holds component i
          double x = (lane < m) ? s_z[lane] : 0.0;
          for (int k = 0; k < m; ++k) {
            if (lane == k) x *= s_dinv[k];
            const double xk = __shfl_sync(0xffffffffu, x, k);
            if (lane > k && lane < m) x = fma(-s_L[lane + k * kMaxM], xk, x);
          }
          for (int k = m - 1; k >= 0; --k) {
            if (lane == k) x *= s_dinv[k];
            const double xk = __shfl_sync(0xffffffffu, x, k);
            if (lane < k) x = fma(-s_L[k + lane * kMaxM], xk, x);
          }
          if (lane < kMaxM) s_mu[lane] = (lane < m) ? x : 0.0;
          if (has_store && scnt < store_cap) slot = scnt++;
        }
        if (lane == 0) {
          s_nst = nst;
          s_beta = beta;
          s_slot = slot;
          s_rinv = (slot >= 0) ? 1.0 / sqrt(rho) : 0.0;
        }
      }
      __syncthreads();
      const int nst = s_nst;
      mark(4);
      // ================= C: x += alpha p (LOOP); p = r + beta p - W mu_W - ghat mu_g
      {
        const bool upd_x = (mode == ST_ACTIVE) && alpha != 0.0;
        const bool upd_p = (nst == ST_ACTIVE);
        const double beta = s_beta;
        const int slot = s_slot;
        const double rinv = s_rinv;
        double* sto = (slot >= 0) ? cg->store + ((int64_t)s * cg->store_cap + slot) * cg->lds : nullptr;
        if (upd_x || upd_p)
          cluster_combine_rows(Xv, Pv, Rv, Wg, ldw, Gh, sto, rbeg, rend, upd_x, upd_p, alpha, beta, s_mu, nw, hg, rinv);
      }
      asm volatile("fence.proxy.async.global;\n" ::: "memory");   // p / x stores -> next TMA reads
      mark(5);
      cl_sync();
      mark(1);
      if (P.prof && blockIdx.x == 0 && tid == 0) g_cprof[6] += 1;
      mode = nst;
      status = nst;
      if (nst != ST_ACTIVE && nst != ST_RCONV) break;
    }
    if (P.smem_r) {   // r back to global memory (the host's confirmation norms read it)
      __syncthreads();
      for (int64_t i = rbeg + tid; i < rend; i += kAT) Rg[i] = sR[i - rbeg];
    }
    // ---- per-shift outputs (leader CTA)
    if (crank == 0 && tid == 0) {
      cg->status[s] = status;
      cg->iters[s] = iters;
      cg->rho[s] = rho;
      cg->rho_true[s] = rho_true;
      cg->nconf[s] = nconf;
      cg->store_cnt[s] = scnt;
      cg->alpha[s] = 0.0;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host side
bool fill_apply_params(Handle* h, const ApplyLaunch& a, ApplyParams& prm, int ty_override);

template <int R>
static cudaError_t launch_cluster_r(ClusterParams& prm, bool tma, int csize, int nclusters, int slots, cudaStream_t st,
                                    bool* ok) {
  using C = TcCfg<R, cluster_tile_rows(R)>;
  auto kfn = tma ? cg_cluster_kernel<R, true> : cg_cluster_kernel<R, false>;
  // r in shared memory if it fits next to the apply's buffers and the static arrays
  const size_t rbytes = sizeof(double) * (size_t)prm.rows;
  const size_t base = sizeof(double) * (size_t)((C::DBL + 1) & ~1);
  prm.smem_r = (getenv("RSK_CLUSTER_RGLOBAL") == nullptr && base + rbytes + 12 * 1024 <= 227 * 1024) ? 1 : 0;
  const size_t smem = prm.smem_r ? base + rbytes : C::SMEM;
  static int inited[2] = {0, 0};
  static int maxcl[2] = {0, 0};
  const int ti = tma ? 1 : 0;
  static size_t attr_smem[2] = {0, 0};
  if (!inited[ti] || smem > attr_smem[ti]) {
    inited[ti] = 1;
    attr_smem[ti] = smem;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && csize > 8) e = cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) { cudaGetLastError(); maxcl[ti] = 0; }
    else {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(csize * 64); cfg.blockDim = dim3(kAT); cfg.dynamicSmemBytes = smem;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (void*)kfn, &cfg) != cudaSuccess) { cudaGetLastError(); n = 0; }
      maxcl[ti] = n;
    }
  }
  int ncl = nclusters < maxcl[ti] ? nclusters : maxcl[ti];
  if (ncl > slots) ncl = slots;
  if (ncl < 1) { *ok = false; return cudaSuccess; }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(csize * ncl); cfg.blockDim = dim3(kAT); cfg.dynamicSmemBytes = smem; cfg.stream = st;
  cfg.attrs = at; cfg.numAttrs = 1;
  count_launch();
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, prm);
  if (e != cudaSuccess) {
    fprintf(stderr, "librsk: cluster launch failed (%s); lockstep CG loop\n", cudaGetErrorString(e));
    cudaGetLastError();
    *ok = false;
    return cudaSuccess;
  }
  *ok = true;
  return cudaSuccess;
}

extern "C" int rsk_debug_cluster_prof(double* out8, int reset) {
  unsigned long long v[8];
  if (cudaMemcpyFromSymbol(v, g_cprof, sizeof(v)) != cudaSuccess) return -1;
  for (int i = 0; i < 8; ++i) out8[i] = (double)v[i];
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_cprof, z, sizeof(z));
  }
  return 0;
}

int64_t cluster_max_n() {
  const char* e = getenv("RSK_CG_CLUSTER_MAXN");
  return e ? atoll(e) : 131072;
}

int cluster_size_for(const Handle* h);
int cluster_slots(const Handle* h) { return h->sm_count / cluster_size_for(h) + 1; }

int cluster_size_for(const Handle* h) {
  (void)h;
  const char* e = getenv("RSK_CG_CLUSTER");
  int cs = e ? atoi(e) : 16;
  if (cs != 2 && cs != 4 && cs != 8 && cs != 16) cs = 16;
  return cs;
}

// Runs every ACTIVE / RCONV shift to completion with one cluster per shift.
cudaError_t launch_cg_cluster(Handle* h, CgDev* dev, const CgDev& hc, unsigned* queue, const int* order,
                              double* zw, cudaStream_t st, bool* ok) {
  ClusterParams prm;
  ApplyLaunch a{};
  a.X = hc.P; a.ldx = hc.N;
  a.X2 = hc.X; a.ldx2 = hc.ldx;
  a.Y = hc.Wv; a.ldy = hc.N;
  a.gamma = hc.gam;
  a.nlist = 1;
  a.nvec_total = hc.nshift;
  a.mode = RSK_APPLY_SHIFTED;
  a.src2_rconv = true;
  a.xdoty = reinterpret_cast<double*>(1);   // want_dot (accumulated through dot_acc)
  const bool tma = fill_apply_params(h, a, prm.ap, cluster_tile_rows(h->r));
  prm.ap.cg = nullptr;
  prm.cg = dev;
  prm.queue = queue;
  prm.order = order;
  prm.zw = zw;
  prm.nshift = hc.nshift;
  int cs = cluster_size_for(h);
  int64_t rows = (hc.N + cs - 1) / cs;
  rows = (rows + 1) / 2 * 2;
  prm.rows = rows;
  prm.prof = getenv("RSK_CLUSTER_PROF") ? 1 : 0;
  *ok = false;
  const int ncl = hc.nshift;
  const int slots = cluster_slots(h);
  cudaError_t e = cudaSuccess;
  switch (h->r) {
    case 1: e = launch_cluster_r<1>(prm, tma, cs, ncl, slots, st, ok); break;
    case 2: e = launch_cluster_r<2>(prm, tma, cs, ncl, slots, st, ok); break;
    case 3: e = launch_cluster_r<3>(prm, tma, cs, ncl, slots, st, ok); break;
    case 4: e = launch_cluster_r<4>(prm, tma, cs, ncl, slots, st, ok); break;
    case 5: e = launch_cluster_r<5>(prm, tma, cs, ncl, slots, st, ok); break;
    case 6: e = launch_cluster_r<6>(prm, tma, cs, ncl, slots, st, ok); break;
    case 7: e = launch_cluster_r<7>(prm, tma, cs, ncl, slots, st, ok); break;
    case 8: e = launch_cluster_r<8>(prm, tma, cs, ncl, slots, st, ok); break;
    case 9: e = launch_cluster_r<9>(prm, tma, cs, ncl, slots, st, ok); break;
    case 10: e = launch_cluster_r<10>(prm, tma, cs, ncl, slots, st, ok); break;
    case 11: e = launch_cluster_r<11>(prm, tma, cs, ncl, slots, st, ok); break;
    case 12: e = launch_cluster_r<12>(prm, tma, cs, ncl, slots, st, ok); break;
    default: break;
  }
  return e;
}

}  // namespace rsk
