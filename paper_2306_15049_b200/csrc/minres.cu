// Recycling MINRES batched over shifts: the paper's own inner solver (SURVEY §8(f)
// f2(ii); PAPER.md §"Shift Specific Recycling" P:454-534). See include/rsk.h
// (rsk_minres_recycled_batch) for the contract.
//
// Per shift l, with U~_l = [W_g, g-hat_l] and Z_l = (A + gamma_l E) U~_l =
// [AW_g + gamma_l EW_g, ZGhat_l] (no applies):
//   eq:localU   Z_l = K_l R_l (shifted Cholesky QR3, K_l^T K_l = I, R_l upper)
//   start       r = b - A_g x_0 ; c0 = K^T r ; v_1 = (I - K K^T) r / xi
//   Lanczos     w = A_g v_j (fused apply, alpha_j = v_j . w from its epilogue);
//               c_j = K^T w ; w <- w - K c_j - alpha_j v_j - beta_j v_{j-1};
//               beta_{j+1} = ||w|| ; v_{j+1} = w / beta_{j+1}
//   eq:minShift the y-block min || xi e_1 - T_m y || by Givens rotations (Paige-Saunders
//               MINRES), the Krylov part y_m = V_m y by short recurrences of the
//               directions d_j; K^T A_g y_m is carried with the same recurrence from
//               the c_j, so the first block row needs no extra apply
//   eq:xFinal   x = x_0 + y_m + U~ R^-1 (c0 - K^T A_g y_m)
//   confirm     true residual b - A_g x (restart from x if it fails; reading G14)
// The iteration count is the number of Lanczos applies, as in the oracle
// (oracle/minres.py). All reductions are fixed-order (CTA partials summed in chunk
// order by the last CTA of a ticket), so a shift's arithmetic depends only on N.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "apply_core.cuh"
#include "rsk_internal.h"

namespace rsk {
bool fill_apply_params(Handle* h, const ApplyLaunch& a, ApplyParams& prm, int ty_override);   // apply.cu
namespace {

constexpr int kMrK = RSK_MAX_LOCAL;   // local columns per shift (|J| + 1 <= 17)
constexpr int kMrRows = 512;          // rows per CTA chunk (independent of the batch)
constexpr int kMrT = 256;
constexpr int kMrP = 2 * kMrK + 1;    // partial slots: K^T w (0..), K^T v (kMrK..), norm^2 (2 kMrK)

struct MrDev {
  int64_t N;
  int ns;
  double* V;    // v_j          N x ns
  double* Vp;   // v_{j-1}
  double* Wv;   // A_g v_j, projected in place
  double* D1;   // d_{j-1}
  double* D2;   // d_{j-2}
  double* Y;    // y_m = V_m y
  double* R0;   // residual of the (re)start point x_0
  double* Kb;   // K_s at Kb + s * kMrK * N (ld N)
  const double* gam;
  const double* alpha;   // v_j . A_g v_j (apply epilogue), per shift
  double* c;     // [ns][kMrK]  K^T A_g v_j
  double* c0;    // [ns][kMrK]  K^T r at the (re)start
  double* kd1;   // [ns][kMrK]  K^T A_g d_{j-1}
  double* kd2;   // [ns][kMrK]
  double* kay;   // [ns][kMrK]  K^T A_g y_m
  double* tt;    // [ns][kMrK]  R^-1 (c0 - kay) for eq:xFinal
  double* sc;    // [ns][16] MINRES scalars
  double* part;  // [ns][nchunk][kMrP]
  double* kv;    // [ns][kMrK]  K^T v_j (the Lanczos vector's drift out of K-perp)
  double* rt2;   // [ns] ||b - A_g x||^2 after a confirm
  int* m;        // [ns] local dimension
  int* status;
  int* iters;
  int* go;       // 1: mr_project took this iteration's Lanczos step (reset by mr_kdots)
  unsigned* cnt; // [ns][4] tickets
  const double* b;
  double* X; int64_t ldx;
  const double* W[RSK_MAX_GROUPS];
  int J[RSK_MAX_GROUPS];
  int64_t ldw;
  const double* Ghat; int64_t ldgh;
  const double* Ghat2;
  int* group;
  int* hasg;
  int* hasg2;
  int nchunk;
  double tolb;   // tol * ||b||
  int maxit;
  double* store; // RSK_CG_STORE_RES: normalised Lanczos vectors, shift s slot c at
  int64_t lds;   //   store + (s * store_cap + c) * lds
  int store_cap;
  int* slot;     // [ns] store slot of the vector v being formed, or -1
  int* scnt;     // [ns] vectors stored
};

// MINRES scalars (index into sc[s*16 + .])
enum { S_BETA = 0, S_EPS, S_DBAR, S_CS, S_SN, S_PHIBAR, S_OLDEPS, S_DELTA, S_DENOM, S_PHI, S_INVB, S_XI };

__device__ __forceinline__ double mr_wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum v over the CTA (fixed tree); result valid in thread 0.
__device__ __forceinline__ double mr_block_sum(double v, double* sh) {
  v = mr_wsum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kMrT / 32; ++w) t += sh[w];
  return t;
}

__device__ __forceinline__ bool last_cta(unsigned* c, int nchunk) {
  __shared__ unsigned ticket;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    ticket = atomicAdd(c, 1u);
  }
  __syncthreads();
  const bool last = ticket == (unsigned)(nchunk - 1);
  if (last) {
    __threadfence();
    if (threadIdx.x == 0) *c = 0u;
  }
  return last;
}

// Fixed-order sum of the chunk partials of column j of shift s (thread t takes chunks
// t, t + kMrT, ... in order, then the fixed CTA tree); valid in thread 0.
__device__ __forceinline__ double chunk_sum(const MrDev* g, int s, int j, double* sh) {
  double t = 0.0;
  for (int c = threadIdx.x; c < g->nchunk; c += kMrT) t += g->part[((int64_t)s * g->nchunk + c) * kMrP + j];
  return mr_block_sum(t, sh);
}

// c[s] = K_s^T src_s (src = Wv in the loop, R0 at a start), fixed-order reduction.
__global__ void __launch_bounds__(kMrT) mr_kdots(MrDev* __restrict__ g, const int* __restrict__ list, int start) {
  const int s = list[blockIdx.y];
  if (blockIdx.x == 0 && threadIdx.x == 0) g->go[s] = 0;   // mr_project sets it when it steps s
  if (!start && g->status[s] != ST_ACTIVE) return;
  const int m = g->m[s];
  if (m == 0) return;
  const int64_t N = g->N;
  const int chunk = blockIdx.x;
  const int64_t r0 = (int64_t)chunk * kMrRows, r1 = min(N, r0 + kMrRows);
  const double* src = (start ? g->R0 : g->Wv) + (int64_t)s * N;
  const double* vv = g->V + (int64_t)s * N;
  const double* K = g->Kb + (int64_t)s * kMrK * N;
  double acc[kMrK], acv[kMrK];
#pragma unroll
  for (int j = 0; j < kMrK; ++j) { acc[j] = 0.0; acv[j] = 0.0; }
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kMrT) {
    const double w = src[i];
    const double v = start ? 0.0 : vv[i];
#pragma unroll
    for (int j = 0; j < kMrK; ++j)
      if (j < m) {
        const double k = K[(int64_t)j * N + i];
        acc[j] = fma(k, w, acc[j]);
        acv[j] = fma(k, v, acv[j]);
      }
  }
  __shared__ double sh[kMrT / 32];
  double* part = g->part + ((int64_t)s * g->nchunk + chunk) * kMrP;
#pragma unroll
  for (int j = 0; j < kMrK; ++j) {
    if (j < m) {
      const double t = mr_block_sum(acc[j], sh);
      if (threadIdx.x == 0) part[j] = t;
      if (!start) {
        const double u = mr_block_sum(acv[j], sh);
        if (threadIdx.x == 0) part[kMrK + j] = u;
      }
    }
  }
  if (!last_cta(&g->cnt[s * 4 + 0], g->nchunk)) return;
  for (int j = 0; j < m; ++j) {
    const double t = chunk_sum(g, s, j, sh);
    if (threadIdx.x == 0) (start ? g->c0 : g->c)[s * kMrK + j] = t;
    if (!start) {
      const double u = chunk_sum(g, s, kMrK + j, sh);
      if (threadIdx.x == 0) g->kv[s * kMrK + j] = u;
    }
  }
}

// Lanczos step: w <- w - K c - alpha v - beta v_prev ; beta' = ||w||; the last CTA of a
// shift updates the Givens QR of T_m (Paige-Saunders) and the status.
__global__ void __launch_bounds__(kMrT) mr_project(MrDev* __restrict__ g, const int* __restrict__ list) {
  const int s = list[blockIdx.y];
  if (g->status[s] != ST_ACTIVE) return;
  const int m = g->m[s];
  const int64_t N = g->N;
  const int chunk = blockIdx.x;
  const int64_t r0 = (int64_t)chunk * kMrRows, r1 = min(N, r0 + kMrRows);
  __shared__ double cs_[kMrK];
  if (threadIdx.x < kMrK) cs_[threadIdx.x] = threadIdx.x < m ? g->c[s * kMrK + threadIdx.x] : 0.0;
  __syncthreads();
  // alpha_j = v_j . (I - K K^T) A_g v_j = v_j . A_g v_j - (K^T v_j) . c_j (as the oracle:
  // the projection before the inner product; the second term is v_j's drift out of K-perp)
  double alpha = g->alpha[s];
  for (int j = 0; j < m; ++j) alpha = fma(-g->kv[s * kMrK + j], cs_[j], alpha);
  const double beta = g->sc[s * 16 + S_BETA];
  const double* K = g->Kb + (int64_t)s * kMrK * N;
  double* w = g->Wv + (int64_t)s * N;
  const double* v = g->V + (int64_t)s * N;
  const double* vp = g->Vp + (int64_t)s * N;
  double nrm = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kMrT) {
    double t = w[i];
#pragma unroll
    for (int j = 0; j < kMrK; ++j)
      if (j < m) t = fma(-cs_[j], K[(int64_t)j * N + i], t);
    t = fma(-alpha, v[i], t);
    t = fma(-beta, vp[i], t);
    w[i] = t;
    nrm = fma(t, t, nrm);
  }
  __shared__ double sh[kMrT / 32];
  const double tot = mr_block_sum(nrm, sh);
  double* part = g->part + ((int64_t)s * g->nchunk + chunk) * kMrP;
  if (threadIdx.x == 0) part[kMrK] = tot;
  if (!last_cta(&g->cnt[s * 4 + 1], g->nchunk)) return;
  const double n2 = chunk_sum(g, s, kMrK, sh);
  if (threadIdx.x != 0) return;
  double* sc = g->sc + s * 16;
  const double bn = sqrt(n2);
  const double oldeps = sc[S_EPS];
  const double cs = sc[S_CS], sn = sc[S_SN], dbar = sc[S_DBAR];
  const double delta = cs * dbar + sn * alpha;
  const double gbar = sn * dbar - cs * alpha;
  const double epsln = sn * bn;
  const double dbar2 = -cs * bn;
  double gm = sqrt(gbar * gbar + bn * bn);
  if (gm < 2.2250738585072014e-308) gm = 2.2250738585072014e-308;
  const double cs2 = gbar / gm, sn2 = bn / gm;
  const double phi = cs2 * sc[S_PHIBAR];
  const double phibar = sn2 * sc[S_PHIBAR];
  const double denom = 1.0 / gm;
  // K^T A_g d_j = (c_j - oldeps K^T A_g d_{j-2} - delta K^T A_g d_{j-1}) / gamma_j
  for (int j = 0; j < m; ++j) {
    const int q = s * kMrK + j;
    const double kd = (g->c[q] - oldeps * g->kd2[q] - delta * g->kd1[q]) * denom;
    g->kay[q] = fma(phi, kd, g->kay[q]);
    g->kd2[q] = g->kd1[q];
    g->kd1[q] = kd;
  }
  sc[S_OLDEPS] = oldeps;
  sc[S_DELTA] = delta;
  sc[S_DENOM] = denom;
  sc[S_PHI] = phi;
  sc[S_INVB] = bn > 0.0 ? 1.0 / bn : 0.0;
  sc[S_EPS] = epsln;
  sc[S_DBAR] = dbar2;
  sc[S_CS] = cs2;
  sc[S_SN] = sn2;
  sc[S_PHIBAR] = phibar;
  sc[S_BETA] = bn;
  const int it = g->iters[s] + 1;
  g->iters[s] = it;
  g->go[s] = 1;
  if (!isfinite(bn) || !isfinite(phibar) || !isfinite(alpha)) g->status[s] = ST_BREAKDOWN;
  else if (fabs(phibar) <= g->tolb || bn == 0.0) g->status[s] = ST_RCONV;
  else if (it >= g->maxit) g->status[s] = ST_MAXIT;
  int sl = -1;   // v_{j+1} is stored while the solve goes on (as CG stores r_j)
  if (g->store && g->status[s] == ST_ACTIVE && g->scnt[s] < g->store_cap) sl = g->scnt[s]++;
  g->slot[s] = sl;
}

// d_j = (v_j - oldeps d_{j-2} - delta d_{j-1}) / gamma_j ; y += phi d_j ;
// v_{j-1} <- v_j ; v_{j+1} = w / beta_{j+1}
__global__ void __launch_bounds__(kMrT) mr_vec(MrDev* __restrict__ g, const int* __restrict__ list) {
  const int s = list[blockIdx.y];
  if (!g->go[s]) return;
  const int64_t N = g->N;
  const int64_t r0 = (int64_t)blockIdx.x * kMrRows, r1 = min(N, r0 + kMrRows);
  const double* sc = g->sc + s * 16;
  const double oldeps = sc[S_OLDEPS], delta = sc[S_DELTA], denom = sc[S_DENOM], phi = sc[S_PHI],
               invb = sc[S_INVB];
  const int64_t o = (int64_t)s * N;
  const int sl = g->slot[s];
  double* sto = (sl >= 0) ? g->store + ((int64_t)s * g->store_cap + sl) * g->lds : nullptr;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kMrT) {
    const double v = g->V[o + i];
    const double d1 = g->D1[o + i], d2 = g->D2[o + i];
    const double dn = (v - oldeps * d2 - delta * d1) * denom;
    g->Y[o + i] = fma(phi, dn, g->Y[o + i]);
    g->D2[o + i] = d1;
    g->D1[o + i] = dn;
    g->Vp[o + i] = v;
    const double vn = g->Wv[o + i] * invb;
    g->V[o + i] = vn;
    if (sto) sto[i] = vn;
  }
}

// start: V = R0 - K c0, xi^2 = ||V||^2; the last CTA initialises the MINRES scalars.
__global__ void __launch_bounds__(kMrT) mr_start_proj(MrDev* __restrict__ g, const int* __restrict__ list) {
  const int s = list[blockIdx.y];
  const int m = g->m[s];
  const int64_t N = g->N;
  const int chunk = blockIdx.x;
  const int64_t r0 = (int64_t)chunk * kMrRows, r1 = min(N, r0 + kMrRows);
  __shared__ double cs_[kMrK];
  if (threadIdx.x < kMrK) cs_[threadIdx.x] = threadIdx.x < m ? g->c0[s * kMrK + threadIdx.x] : 0.0;
  __syncthreads();
  const double* K = g->Kb + (int64_t)s * kMrK * N;
  const double* r = g->R0 + (int64_t)s * N;
  double* v = g->V + (int64_t)s * N;
  double nrm = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kMrT) {
    double t = r[i];
#pragma unroll
    for (int j = 0; j < kMrK; ++j)
      if (j < m) t = fma(-cs_[j], K[(int64_t)j * N + i], t);
    v[i] = t;
    nrm = fma(t, t, nrm);
  }
  __shared__ double sh[kMrT / 32];
  const double tot = mr_block_sum(nrm, sh);
  double* part = g->part + ((int64_t)s * g->nchunk + chunk) * kMrP;
  if (threadIdx.x == 0) part[kMrK] = tot;
  if (!last_cta(&g->cnt[s * 4 + 1], g->nchunk)) return;
  const double n2 = chunk_sum(g, s, kMrK, sh);
  if (threadIdx.x == 0) {
    const double xi = sqrt(n2);
    double* sc = g->sc + s * 16;
    sc[S_BETA] = 0.0;       // beta_1 multiplies v_0 = 0
    sc[S_EPS] = 0.0;
    sc[S_DBAR] = 0.0;
    sc[S_CS] = -1.0;
    sc[S_SN] = 0.0;
    sc[S_PHIBAR] = xi;
    sc[S_XI] = xi;
    sc[S_INVB] = xi > 0.0 ? 1.0 / xi : 0.0;
    g->status[s] = (xi > 0.0 && isfinite(xi)) ? ST_ACTIVE : (isfinite(xi) ? ST_RCONV : ST_BREAKDOWN);
    if (xi <= g->tolb && xi > 0.0) g->status[s] = ST_RCONV;   // x_0 + U K^T r already converged
    int sl = -1;
    if (g->store && g->status[s] == ST_ACTIVE && g->scnt[s] < g->store_cap) sl = g->scnt[s]++;
    g->slot[s] = sl;
  }
  if (threadIdx.x < kMrK) {
    const int q = s * kMrK + threadIdx.x;
    g->kd1[q] = 0.0; g->kd2[q] = 0.0; g->kay[q] = 0.0;
  }
}

// start (after mr_start_proj): v_1 = V / xi ; v_0 = d = y = 0
__global__ void __launch_bounds__(kMrT) mr_start_vec(MrDev* __restrict__ g, const int* __restrict__ list) {
  const int s = list[blockIdx.y];
  const int64_t N = g->N;
  const int64_t r0 = (int64_t)blockIdx.x * kMrRows, r1 = min(N, r0 + kMrRows);
  const double invb = g->sc[s * 16 + S_INVB];
  const int64_t o = (int64_t)s * N;
  const int sl = g->slot[s];
  double* sto = (sl >= 0) ? g->store + ((int64_t)s * g->store_cap + sl) * g->lds : nullptr;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kMrT) {
    const double v = g->V[o + i] * invb;
    g->V[o + i] = v;
    g->Vp[o + i] = 0.0; g->D1[o + i] = 0.0; g->D2[o + i] = 0.0; g->Y[o + i] = 0.0;
    if (sto) sto[i] = v;
  }
}

// eq:xFinal: x += y_m + U~ t, t = R^-1 (c0 - K^T A y_m) (host triangular solve)
__global__ void __launch_bounds__(kMrT) mr_final(MrDev* __restrict__ g, const int* __restrict__ list) {
  const int s = list[blockIdx.y];
  const int m = g->m[s];
  const int64_t N = g->N;
  const int64_t r0 = (int64_t)blockIdx.x * kMrRows, r1 = min(N, r0 + kMrRows);
  const int gi = g->group[s];
  const int J = m > 0 ? min(g->J[gi], m) : 0;
  const bool hg = m > J && g->hasg[s];
  const bool hg2 = m > J && g->hasg2[s];
  const double* W = J > 0 ? g->W[gi] : nullptr;
  const double* gh = hg ? g->Ghat + (int64_t)s * g->ldgh : nullptr;
  const double* gh2 = hg2 ? g->Ghat2 + (int64_t)s * g->ldgh : nullptr;
  const int j2 = J + (hg ? 1 : 0);
  __shared__ double t[kMrK];
  if (threadIdx.x < kMrK) t[threadIdx.x] = threadIdx.x < m ? g->tt[s * kMrK + threadIdx.x] : 0.0;
  __syncthreads();
  double* x = g->X + (int64_t)s * g->ldx;
  const double* y = g->Y + (int64_t)s * N;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kMrT) {
    double a = x[i] + y[i];
    for (int j = 0; j < J; ++j) a = fma(t[j], W[(int64_t)j * g->ldw + i], a);
    if (hg) a = fma(t[J], gh[i], a);
    if (hg2) a = fma(t[j2], gh2[i], a);
    x[i] = a;
  }
}

// R0 = b - R0 (R0 held A_g x) and ||R0||^2 -> rt2[s]
__global__ void __launch_bounds__(kMrT) mr_resid(MrDev* __restrict__ g, const int* __restrict__ list) {
  const int s = list[blockIdx.y];
  const int64_t N = g->N;
  const int chunk = blockIdx.x;
  const int64_t r0 = (int64_t)chunk * kMrRows, r1 = min(N, r0 + kMrRows);
  double* r = g->R0 + (int64_t)s * N;
  double nrm = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kMrT) {
    const double t = g->b[i] - r[i];
    r[i] = t;
    nrm = fma(t, t, nrm);
  }
  __shared__ double sh[kMrT / 32];
  const double tot = mr_block_sum(nrm, sh);
  if (threadIdx.x == 0) g->part[((int64_t)s * g->nchunk + chunk) * kMrP + kMrK] = tot;
  if (!last_cta(&g->cnt[s * 4 + 2], g->nchunk)) return;
  const double n2 = chunk_sum(g, s, kMrK, sh);
  if (threadIdx.x == 0) g->rt2[s] = n2;
}

// Z_s = [AW_g + gamma_s EW_g, ZGhat_s, ZGhat2_s] (m columns, ld N; zg / zg2 nullable)
__global__ void mr_formz(int64_t N, const double* __restrict__ AW, const double* __restrict__ EW, int64_t ldw,
                         int J, double gam, const double* __restrict__ zg, const double* __restrict__ zg2,
                         double* __restrict__ Z) {
  const int j = blockIdx.y;
  const double* zc = (j == J && zg) ? zg : zg2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    Z[(int64_t)j * N + i] = j < J ? fma(gam, EW[(int64_t)j * ldw + i], AW[(int64_t)j * ldw + i]) : zc[i];
}

__global__ void mr_gout(int64_t N, int ns, const double* __restrict__ X, int64_t ldx, double* __restrict__ G,
                        int64_t ldg) {
  const int s = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    G[(int64_t)s * ldg + i] = X[(int64_t)s * ldx + i] - G[(int64_t)s * ldg + i];
}

// ============================================================ cluster-per-shift loop
// For images whose working set sits in L2 (as the CG's cg_cluster.cu): a 16-CTA thread-
// block cluster owns one shift and runs its Lanczos / Givens recurrences to the stopping
// point in one launch; partial sums are pushed into every CTA's shared memory before
// the hardware cluster barrier and summed there in rank order (deterministic). Per
// iteration (4 cluster barriers):
//   A  w = A_g v (fused apply, v . w partial)                  -> alpha0
//   B  c = K^T w, kv = K^T v over the CTA's rows               -> alpha = alpha0 - kv . c
//   C  w <- w - K c - alpha v - beta v_prev; ||w||^2           -> beta', Givens (every CTA)
//   D  d, y, v_prev, v updates (and the Lanczos-vector store)
// The recurrences and stopping rule are those of the lockstep kernels above; finalisation
// (eq:xFinal), confirmation and restarts stay on the host path.
constexpr int kMrCS = 16;     // CTAs per cluster
constexpr int kMrSl = 2 * kMrK + 2;   // pushed slots: c (kMrK), kv (kMrK), norm^2, p.w

struct alignas(64) MrClusterParams {
  ApplyParams ap;     // X = V, Y = Wv, want_dot
  MrDev* g;
  unsigned* queue;
  const int* list;    // shifts to run (device), nl of them
  int nl;
  int64_t rows;       // rows per CTA
  int smem_vp;        // 1: the CTA's rows of v_{j-1} live in shared memory for the whole shift
};

__host__ __device__ constexpr int mr_tile_rows(int r) { return r <= 6 ? 64 : (r <= 8 ? 56 : tc_tile_rows(r)); }

__device__ __forceinline__ void mr_cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// phase B rows: per-warp sums of c_j = K_j . w and kv_j = K_j . v into red[warp][j],
// red[warp][kMrK + j] (MK >= m: register arrays sized for the local dimension)
template <int MK>
__device__ __noinline__ void mr_rows_b_t(const double* __restrict__ K, const double* __restrict__ W,
                                         const double* __restrict__ V, int64_t N, int64_t rbeg, int64_t rend, int m,
                                         double (*red)[kMrSl]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double ac[MK], av[MK];
#pragma unroll
  for (int j = 0; j < MK; ++j) { ac[j] = 0.0; av[j] = 0.0; }
  const int64_t np2 = (rend - rbeg) >> 1;   // row pairs (rbeg even): 16-byte loads
#pragma unroll 2
  for (int64_t q = tid; q < np2; q += kAT) {
    const int64_t i = rbeg + 2 * q;
    double2 kk[MK];
#pragma unroll
    for (int j = 0; j < MK; ++j)
      kk[j] = (j < m) ? __ldcg(reinterpret_cast<const double2*>(K + (int64_t)j * N + i)) : make_double2(0.0, 0.0);
    const double2 w = *reinterpret_cast<const double2*>(W + i), v = *reinterpret_cast<const double2*>(V + i);
#pragma unroll
    for (int j = 0; j < MK; ++j)
      if (j < m) {
        ac[j] = fma(kk[j].y, w.y, fma(kk[j].x, w.x, ac[j]));
        av[j] = fma(kk[j].y, v.y, fma(kk[j].x, v.x, av[j]));
      }
  }
  if (((rend - rbeg) & 1) && tid == 0) {
    const int64_t i = rend - 1;
    const double w = W[i], v = V[i];
#pragma unroll
    for (int j = 0; j < MK; ++j)
      if (j < m) {
        const double k = K[(int64_t)j * N + i];
        ac[j] = fma(k, w, ac[j]);
        av[j] = fma(k, v, av[j]);
      }
  }
#pragma unroll
  for (int j = 0; j < MK; ++j) {
    if (j < m) {
      const double x = mr_wsum(ac[j]), y = mr_wsum(av[j]);
      if (lane == 0) { red[warp][j] = x; red[warp][kMrK + j] = y; }
    }
  }
}

__device__ __forceinline__ void mr_rows_b(const double* K, const double* W, const double* V, int64_t N, int64_t rbeg,
                                          int64_t rend, int m, double (*red)[kMrSl]) {
  if (m <= 10) mr_rows_b_t<10>(K, W, V, N, rbeg, rend, m, red);
  else mr_rows_b_t<kMrK>(K, W, V, N, rbeg, rend, m, red);
}

// phase C rows: w <- w - K c - alpha v - beta_prev v_prev over the CTA's rows; returns this
// thread's part of ||w||^2
template <int MK>
__device__ __noinline__ double mr_rows_c_t(const double* __restrict__ K, double* __restrict__ W,
                                           const double* __restrict__ V, const double* __restrict__ Vp, int64_t N,
                                           int64_t rbeg, int64_t rend, int m, const double* sc, double alpha,
                                           double bprev) {
  const int tid = threadIdx.x;
  double cc[MK];
#pragma unroll
  for (int j = 0; j < MK; ++j) cc[j] = (j < m) ? sc[j] : 0.0;
  double nrm = 0.0;
  const int64_t np2 = (rend - rbeg) >> 1;
#pragma unroll 2
  for (int64_t q = tid; q < np2; q += kAT) {
    const int64_t i = rbeg + 2 * q;
    double2 kk[MK];
#pragma unroll
    for (int j = 0; j < MK; ++j)
      kk[j] = (j < m) ? __ldcg(reinterpret_cast<const double2*>(K + (int64_t)j * N + i)) : make_double2(0.0, 0.0);
    double2 t = *reinterpret_cast<const double2*>(W + i);
    const double2 v = *reinterpret_cast<const double2*>(V + i), vp = *reinterpret_cast<const double2*>(Vp + i);
#pragma unroll
    for (int j = 0; j < MK; ++j)
      if (j < m) { t.x = fma(-cc[j], kk[j].x, t.x); t.y = fma(-cc[j], kk[j].y, t.y); }
    t.x = fma(-bprev, vp.x, fma(-alpha, v.x, t.x));
    t.y = fma(-bprev, vp.y, fma(-alpha, v.y, t.y));
    *reinterpret_cast<double2*>(W + i) = t;
    nrm = fma(t.y, t.y, fma(t.x, t.x, nrm));
  }
  if (((rend - rbeg) & 1) && tid == 0) {
    const int64_t i = rend - 1;
    double t = W[i];
#pragma unroll
    for (int j = 0; j < MK; ++j)
      if (j < m) t = fma(-cc[j], K[(int64_t)j * N + i], t);
    t = fma(-bprev, Vp[i], fma(-alpha, V[i], t));
    W[i] = t;
    nrm = fma(t, t, nrm);
  }
  return nrm;
}

__device__ __forceinline__ double mr_rows_c(const double* K, double* W, const double* V, const double* Vp, int64_t N,
                                            int64_t rbeg, int64_t rend, int m, const double* sc, double alpha,
                                            double bprev) {
  if (m <= 10) return mr_rows_c_t<10>(K, W, V, Vp, N, rbeg, rend, m, sc, alpha, bprev);
  return mr_rows_c_t<kMrK>(K, W, V, Vp, N, rbeg, rend, m, sc, alpha, bprev);
}

template <int R, bool kTma>
__global__ void __launch_bounds__(kAT, 1) mr_cluster_kernel(const __grid_constant__ MrClusterParams P) {
  extern __shared__ __align__(128) double smem[];
  using Core = ApplyCore<R, kTma, mr_tile_rows(R)>;
  unsigned crank_u;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank_u));
  const int crank = (int)crank_u;
  const int csz = kMrCS;
  __shared__ double s_dot;
  __shared__ double s_dots[kMrCS];
  __shared__ double s_part[kMrSl];
  __shared__ double s_parts[kMrCS][kMrSl];
  __shared__ double s_red[kAT / 32][kMrSl];
  __shared__ double s_c[kMrK], s_kv[kMrK], s_kd1[kMrK], s_kd2[kMrK], s_kay[kMrK];
  __shared__ double s_co[8];     // alpha, oldeps, delta, denom, phi, invb
  __shared__ double s_beta;      // beta_j of the current Lanczos step
  __shared__ int s_next, s_st, s_slot;
  __shared__ int s_list[1], s_lmode[1];
  MrDev* g = P.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = g->N;
  Core::init_bars(smem, P.ap);
  ApplyPipe pp{{0u, 0u}, 0};
  const int64_t rbeg = (int64_t)crank * P.rows;
  const int64_t rend = min(N, rbeg + P.rows);
  const int ntiles = P.ap.ntiles;
  const int tper = (ntiles + csz - 1) / csz;
  const int ibeg = min(ntiles, crank * tper), iend = min(ntiles, ibeg + tper);
  auto remote = [&](double* p, int rank) -> double* {
    unsigned long long a;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(a) : "l"(p), "r"(rank));
    return reinterpret_cast<double*>(a);
  };
  auto remote_i = [&](int* p, int rank) -> int* {
    unsigned long long a;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(a) : "l"(p), "r"(rank));
    return reinterpret_cast<int*>(a);
  };
  for (;;) {
    if (crank == 0 && tid == 0) s_next = (int)atomicAdd(P.queue, 1u);
    mr_cl_sync();
    const int idx = *remote_i(&s_next, 0);
    mr_cl_sync();
    if (idx >= P.nl) break;
    const int s = P.list[idx];
    if (g->status[s] != ST_ACTIVE) continue;
    const int m = g->m[s];
    const double* K = g->Kb + (int64_t)s * kMrK * N;
    double* V = g->V + (int64_t)s * N;
    double* Vpg = g->Vp + (int64_t)s * N;
    // v_{j-1} is touched only by its owning CTA (phases C and D): its rows stay in shared
    // memory behind the apply's buffers for the whole shift when they fit
    double* sVp = smem + ((Core::C::DBL + 1) & ~1);
    double* Vp = Vpg;
    if (P.smem_vp) {
      for (int64_t i = rbeg + tid; i < rend; i += kAT) sVp[i - rbeg] = Vpg[i];
      Vp = sVp - rbeg;
    }
    double* W = g->Wv + (int64_t)s * N;
    double* D1 = g->D1 + (int64_t)s * N;
    double* D2 = g->D2 + (int64_t)s * N;
    double* Yv = g->Y + (int64_t)s * N;
    double* sc = g->sc + s * 16;
    double beta = sc[S_BETA], eps = sc[S_EPS], dbar = sc[S_DBAR], cs = sc[S_CS], sn = sc[S_SN], phibar = sc[S_PHIBAR];
    int iters = g->iters[s], scnt = g->scnt[s];
    int slot = g->slot[s];      // store slot of the current v (set at the start)
    const double tolb = g->tolb;
    const int maxit = g->maxit;
    if (tid < kMrK) {
      const int q = s * kMrK + tid;
      s_kd1[tid] = g->kd1[q]; s_kd2[tid] = g->kd2[q]; s_kay[tid] = g->kay[q];
    }
    if (tid == 0) { s_list[0] = s; s_lmode[0] = ST_ACTIVE; s_beta = beta; }
    __syncthreads();
    int status = ST_ACTIVE;
    for (;;) {
      // ================= A: w = A_g v, v . w
      if (tid == 0) s_dot = 0.0;
      __syncthreads();
      Core::run(P.ap, smem, ibeg, iend, 1, pp, s_list, s_lmode, &s_dot);
      if (tid < csz) *remote(&s_dots[crank], tid) = s_dot;
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      mr_cl_sync();
      // ================= B: c = K^T w, kv = K^T v (row partials)
      {
        mr_rows_b(K, W, V, N, rbeg, rend, m, s_red);
        __syncthreads();
        if (tid < 2 * kMrK) {
          const int j = tid < kMrK ? tid : tid - kMrK;
          double t = 0.0;
          if (j < m)
            for (int w = 0; w < kAT / 32; ++w) t += s_red[w][tid];
          s_part[tid] = t;
        }
        __syncthreads();
        for (int e = tid; e < csz * 2 * kMrK; e += kAT) {
          const int c = e / (2 * kMrK), sl = e - c * 2 * kMrK;
          *remote(&s_parts[crank][sl], c) = s_part[sl];
        }
      }
      mr_cl_sync();
      if (tid < 2 * kMrK) {
        double t = 0.0;
        for (int c = 0; c < csz; ++c) t += s_parts[c][tid];
        if (tid < kMrK) s_c[tid] = t; else s_kv[tid - kMrK] = t;
      }
      __syncthreads();
      if (tid == 0) {
        double a0 = 0.0;
        for (int c = 0; c < csz; ++c) a0 += s_dots[c];
        for (int j = 0; j < m; ++j) a0 = fma(-s_kv[j], s_c[j], a0);
        s_co[0] = a0;
      }
      __syncthreads();
      const double alpha = s_co[0];
      // ================= C: w <- w - K c - alpha v - beta v_prev, ||w||^2
      {
        const double bprev = s_beta;
        double nrm = mr_rows_c(K, W, V, Vp, N, rbeg, rend, m, s_c, alpha, bprev);
        nrm = mr_wsum(nrm);
        if (lane == 0) s_red[warp][0] = nrm;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
          for (int w = 0; w < kAT / 32; ++w) t += s_red[w][0];
          s_part[2 * kMrK] = t;
        }
        __syncthreads();
        if (tid < csz) *remote(&s_parts[crank][2 * kMrK], tid) = s_part[2 * kMrK];
      }
      mr_cl_sync();
      // ---- Givens (identical in every CTA)
      if (tid == 0) {
        double n2 = 0.0;
        for (int c = 0; c < csz; ++c) n2 += s_parts[c][2 * kMrK];
        const double bn = sqrt(n2);
        const double oldeps = eps;
        const double delta = cs * dbar + sn * alpha;
        const double gbar = sn * dbar - cs * alpha;
        eps = sn * bn;
        dbar = -cs * bn;
        double gm = sqrt(gbar * gbar + bn * bn);
        if (gm < 2.2250738585072014e-308) gm = 2.2250738585072014e-308;
        cs = gbar / gm; sn = bn / gm;
        const double phi = cs * phibar;
        phibar = sn * phibar;
        s_co[1] = oldeps; s_co[2] = delta; s_co[3] = 1.0 / gm; s_co[4] = phi; s_co[5] = bn > 0.0 ? 1.0 / bn : 0.0;
        beta = bn;
        s_beta = bn;
        iters += 1;
        int st = ST_ACTIVE;
        if (!isfinite(bn) || !isfinite(phibar) || !isfinite(alpha)) st = ST_BREAKDOWN;
        else if (fabs(phibar) <= tolb || bn == 0.0) st = ST_RCONV;
        else if (iters >= maxit) st = ST_MAXIT;
        int sl = -1;
        if (g->store && st == ST_ACTIVE && scnt < g->store_cap) sl = scnt++;
        s_st = st;
        s_slot = sl;
      }
      __syncthreads();
      // every thread keeps the scalars in registers (same values as thread 0)
      {
        const double oldeps = s_co[1], delta = s_co[2], denom = s_co[3], phi = s_co[4], invb = s_co[5];
        if (tid < m) {   // K^T A_g d_j recurrence
          const double kd = (s_c[tid] - oldeps * s_kd2[tid] - delta * s_kd1[tid]) * denom;
          s_kay[tid] = fma(phi, kd, s_kay[tid]);
          s_kd2[tid] = s_kd1[tid];
          s_kd1[tid] = kd;
        }
        const int st = s_st;
        const int sl = s_slot;
        double* sto = (sl >= 0) ? g->store + ((int64_t)s * g->store_cap + sl) * g->lds : nullptr;
        // ================= D: d, y, v_prev, v
        auto upd1 = [&](int64_t i) {
          const double v = V[i];
          const double d1 = D1[i], d2 = D2[i];
          const double dn = (v - oldeps * d2 - delta * d1) * denom;
          Yv[i] = fma(phi, dn, Yv[i]);
          D2[i] = d1;
          D1[i] = dn;
          Vp[i] = v;
          const double vn = W[i] * invb;
          V[i] = vn;
          if (sto) sto[i] = vn;
        };
        const int64_t np2 = (rend - rbeg) >> 1;
        for (int64_t q = tid; q < np2; q += kAT) {
          const int64_t i = rbeg + 2 * q;
          const double2 v = *reinterpret_cast<const double2*>(V + i);
          const double2 d1 = *reinterpret_cast<const double2*>(D1 + i), d2 = *reinterpret_cast<const double2*>(D2 + i);
          const double2 y = *reinterpret_cast<const double2*>(Yv + i), w = *reinterpret_cast<const double2*>(W + i);
          double2 dn;
          dn.x = (v.x - oldeps * d2.x - delta * d1.x) * denom;
          dn.y = (v.y - oldeps * d2.y - delta * d1.y) * denom;
          *reinterpret_cast<double2*>(Yv + i) = make_double2(fma(phi, dn.x, y.x), fma(phi, dn.y, y.y));
          *reinterpret_cast<double2*>(D2 + i) = d1;
          *reinterpret_cast<double2*>(D1 + i) = dn;
          *reinterpret_cast<double2*>(Vp + i) = v;
          const double2 vn = make_double2(w.x * invb, w.y * invb);
          *reinterpret_cast<double2*>(V + i) = vn;
          if (sto) *reinterpret_cast<double2*>(sto + i) = vn;
        }
        if (((rend - rbeg) & 1) && tid == 0) upd1(rend - 1);
        asm volatile("fence.proxy.async.global;\n" ::: "memory");   // v stores -> next TMA reads
        mr_cl_sync();
        status = st;
        slot = sl;
      }
      if (status != ST_ACTIVE) break;
    }
    if (P.smem_vp) {   // v_{j-1} back to global memory (a host restart reinitialises it there)
      __syncthreads();
      for (int64_t i = rbeg + tid; i < rend; i += kAT) Vpg[i] = sVp[i - rbeg];
    }
    if (crank == 0 && tid == 0) {
      sc[S_BETA] = beta; sc[S_EPS] = eps; sc[S_DBAR] = dbar; sc[S_CS] = cs; sc[S_SN] = sn; sc[S_PHIBAR] = phibar;
      g->iters[s] = iters;
      g->scnt[s] = scnt;
      g->slot[s] = slot;
      g->status[s] = status;
    }
    if (crank == 0 && tid < kMrK) {
      const int q = s * kMrK + tid;
      g->kd1[q] = s_kd1[tid]; g->kd2[q] = s_kd2[tid]; g->kay[q] = s_kay[tid];
    }
    __syncthreads();
  }
}

template <int R>
cudaError_t mr_launch_r(const MrClusterParams& prm, bool tma, int ncl_req, cudaStream_t st, bool* ok) {
  using C = TcCfg<R, mr_tile_rows(R)>;
  auto kfn = tma ? mr_cluster_kernel<R, true> : mr_cluster_kernel<R, false>;
  const size_t base = sizeof(double) * (size_t)((C::DBL + 1) & ~1);
  const size_t vpb = sizeof(double) * (size_t)prm.rows;
  const int smem_vp = (getenv("RSK_MR_VPGLOBAL") == nullptr && base + vpb + 16 * 1024 <= 227 * 1024) ? 1 : 0;
  const size_t smem = smem_vp ? base + vpb : C::SMEM;
  static int inited[2] = {0, 0};
  static int maxcl[2] = {0, 0};
  static size_t attr_smem[2] = {0, 0};
  const int ti = tma ? 1 : 0;
  if (!inited[ti] || smem > attr_smem[ti]) {
    inited[ti] = 1;
    attr_smem[ti] = smem;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) { cudaGetLastError(); maxcl[ti] = 0; }
    else {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kMrCS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(kMrCS * 64); cfg.blockDim = dim3(kAT); cfg.dynamicSmemBytes = smem;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (void*)kfn, &cfg) != cudaSuccess) { cudaGetLastError(); n = 0; }
      maxcl[ti] = n;
    }
  }
  int ncl = ncl_req < maxcl[ti] ? ncl_req : maxcl[ti];
  if (ncl < 1) { *ok = false; return cudaSuccess; }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kMrCS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(kMrCS * ncl); cfg.blockDim = dim3(kAT); cfg.dynamicSmemBytes = smem; cfg.stream = st;
  cfg.attrs = at; cfg.numAttrs = 1;
  count_launch();
  MrClusterParams p2 = prm;
  p2.smem_vp = smem_vp;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, p2);
  if (e != cudaSuccess) { cudaGetLastError(); *ok = false; return cudaSuccess; }
  *ok = true;
  return cudaSuccess;
}

cudaError_t mr_launch_cluster(Handle* h, const MrClusterParams& prm, bool tma, int ncl, cudaStream_t st, bool* ok) {
  switch (h->r) {
    case 1: return mr_launch_r<1>(prm, tma, ncl, st, ok);
    case 2: return mr_launch_r<2>(prm, tma, ncl, st, ok);
    case 3: return mr_launch_r<3>(prm, tma, ncl, st, ok);
    case 4: return mr_launch_r<4>(prm, tma, ncl, st, ok);
    case 5: return mr_launch_r<5>(prm, tma, ncl, st, ok);
    case 6: return mr_launch_r<6>(prm, tma, ncl, st, ok);
    case 7: return mr_launch_r<7>(prm, tma, ncl, st, ok);
    case 8: return mr_launch_r<8>(prm, tma, ncl, st, ok);
    case 9: return mr_launch_r<9>(prm, tma, ncl, st, ok);
    case 10: return mr_launch_r<10>(prm, tma, ncl, st, ok);
    case 11: return mr_launch_r<11>(prm, tma, ncl, st, ok);
    case 12: return mr_launch_r<12>(prm, tma, ncl, st, ok);
    default: *ok = false; return cudaSuccess;
  }
}

struct MrLayout {
  size_t vec, kb, zs, dbl, in, cnt, part, list, q, dev, total;
  int nchunk;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

MrLayout mr_layout(const Handle* h, int ns, int kmax) {
  MrLayout L{};
  const int64_t N = h->ny * h->nx;
  L.nchunk = (int)((N + kMrRows - 1) / kMrRows);
  size_t o = 0;
  L.vec = o; o = al(o + sizeof(double) * (size_t)N * ns * 7);
  L.kb = o; o = al(o + sizeof(double) * (size_t)N * ns * (kmax > 0 ? kMrK : 0));
  L.zs = o; o = al(o + sizeof(double) * (size_t)N * (kmax > 0 ? kmax : 0));
  L.dbl = o; o = al(o + sizeof(double) * (size_t)ns * (8 * kMrK + 16 + 2));
  L.in = o; o = al(o + sizeof(int) * (size_t)ns * 10);
  L.cnt = o; o = al(o + sizeof(unsigned) * (size_t)ns * 4);
  L.part = o; o = al(o + sizeof(double) * (size_t)ns * L.nchunk * kMrP);
  L.list = o; o = al(o + sizeof(int) * (size_t)ns * 2);
  L.q = o; o = al(o + 64);
  L.dev = o; o = al(o + sizeof(MrDev));
  L.total = o;
  return L;
}

inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

}  // namespace
}  // namespace rsk

using namespace rsk;

struct rsk_handle_s : public Handle {};   // as in rsk.cu

#define MR_ARG(c, msg)            \
  do {                            \
    if (!(c)) {                   \
      h->err = (msg);             \
      return RSK_EINVAL;          \
    }                             \
  } while (0)
#define MR_CUDA(x)                                                              \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      h->err = std::string("rsk_minres_recycled_batch: ") + cudaGetErrorString(e_); \
      h->sticky = true;                                                         \
      return RSK_ECUDA;                                                         \
    }                                                                           \
  } while (0)

extern "C" size_t rsk_minres_workspace_bytes(rsk_handle h, int nshift, int max_local_dim) {
  if (!h || nshift <= 0 || max_local_dim < 0 || max_local_dim > RSK_MAX_LOCAL) return 0;
  return mr_layout(h, nshift, max_local_dim).total;
}

extern "C" rsk_status rsk_minres_recycled_batch(rsk_handle h, const rsk_cg_desc* d, rsk_cg_out* o, void* ws,
                                                size_t ws_bytes, void* stream) {
  if (!h) return RSK_EINVAL;
  if (h->sticky) return RSK_ECUDA;
  MR_ARG(d && o, "rsk_minres_recycled_batch: null desc/out");
  const int ns = d->nshift;
  const int64_t N = h->ny * h->nx;
  MR_ARG(ns >= 1, "rsk_minres_recycled_batch: nshift < 1");
  MR_ARG(d->gamma_h && d->b && d->X && d->ldx >= N, "rsk_minres_recycled_batch: gamma/b/X");
  MR_ARG(o->iters && o->applies && o->relres_true && o->status && o->m_used, "rsk_minres_recycled_batch: outputs");
  MR_ARG(d->tol > 0 && std::isfinite(d->tol) && d->maxit >= 1 && d->check_every >= 1,
         "rsk_minres_recycled_batch: tol/maxit/check_every");
  const bool store = (d->flags & RSK_CG_STORE_RES) != 0;
  if (store) MR_ARG(d->store && d->store_cap >= 1 && d->lds >= N, "rsk_minres_recycled_batch: store");
  const bool defl = !(d->flags & RSK_CG_NO_DEFLATION) && d->ngroups > 0;
  MR_ARG(d->ngroups >= 0 && d->ngroups <= RSK_MAX_GROUPS, "rsk_minres_recycled_batch: ngroups");
  std::vector<int> grp(ns, 0), hasg(ns, 0), hasg2(ns, 0), m(ns, 0), hasxp(ns, 0);
  int kmax = 0;
  const bool anyg = defl && d->has_ghat_h != nullptr;
  const bool anyg2 = defl && d->has_ghat2_h != nullptr;
  if (defl) {
    MR_ARG(d->group_of_shift_h && d->ldw >= N, "rsk_minres_recycled_batch: groups");
    for (int g = 0; g < d->ngroups; ++g)
      MR_ARG(d->J[g] >= 0 && d->J[g] <= 16 && (d->J[g] == 0 || (d->W[g] && d->AW[g] && d->EW[g])),
             "rsk_minres_recycled_batch: group block");
    if (anyg) MR_ARG(d->Ghat && d->ZGhat && d->ldgh >= N, "rsk_minres_recycled_batch: Ghat/ZGhat");
    if (anyg2) MR_ARG(d->Ghat2 && d->ZGhat2 && d->ldgh >= N, "rsk_minres_recycled_batch: Ghat2/ZGhat2");
    for (int s = 0; s < ns; ++s) {
      MR_ARG(d->group_of_shift_h[s] >= 0 && d->group_of_shift_h[s] < d->ngroups,
             "rsk_minres_recycled_batch: group index");
      grp[s] = d->group_of_shift_h[s];
      hasg[s] = anyg ? (d->has_ghat_h[s] != 0) : 0;
      hasg2[s] = anyg2 ? (d->has_ghat2_h[s] != 0) : 0;
      m[s] = d->J[grp[s]] + hasg[s] + hasg2[s];
      MR_ARG(m[s] <= kMrK, "rsk_minres_recycled_batch: local dimension > RSK_MAX_LOCAL");
      kmax = std::max(kmax, m[s]);
    }
  }
  for (int s = 0; s < ns; ++s) {
    MR_ARG(std::isfinite(d->gamma_h[s]) && d->gamma_h[s] >= 0, "rsk_minres_recycled_batch: gamma");
    hasxp[s] = d->has_xp_h ? (d->has_xp_h[s] != 0) : 0;
  }
  const MrLayout L = mr_layout(h, ns, kmax);
  MR_ARG(ws && ws_bytes >= L.total, "rsk_minres_recycled_batch: workspace too small");
  MR_CUDA(cudaStreamSynchronize(S(stream)));
  cudaStream_t st = h->cg_stream;

  char* base = static_cast<char*>(ws);
  MrDev hc{};
  hc.N = N;
  hc.ns = ns;
  double* vec = reinterpret_cast<double*>(base + L.vec);
  hc.V = vec; hc.Vp = vec + (size_t)N * ns; hc.Wv = vec + 2 * (size_t)N * ns;
  hc.D1 = vec + 3 * (size_t)N * ns; hc.D2 = vec + 4 * (size_t)N * ns; hc.Y = vec + 5 * (size_t)N * ns;
  hc.R0 = vec + 6 * (size_t)N * ns;
  hc.Kb = reinterpret_cast<double*>(base + L.kb);
  double* Zs = reinterpret_cast<double*>(base + L.zs);
  double* dbl = reinterpret_cast<double*>(base + L.dbl);
  double* gam = dbl;
  double* alpha = dbl + ns;
  hc.gam = gam; hc.alpha = alpha;
  hc.c = dbl + 2 * ns;
  hc.c0 = hc.c + (size_t)ns * kMrK;
  hc.kd1 = hc.c0 + (size_t)ns * kMrK;
  hc.kd2 = hc.kd1 + (size_t)ns * kMrK;
  hc.kay = hc.kd2 + (size_t)ns * kMrK;
  hc.tt = hc.kay + (size_t)ns * kMrK;
  hc.sc = hc.tt + (size_t)ns * kMrK;
  hc.rt2 = hc.sc + (size_t)ns * 16;
  hc.kv = hc.rt2 + (size_t)ns * 2;
  int* in = reinterpret_cast<int*>(base + L.in);
  hc.m = in; hc.status = in + ns; hc.iters = in + 2 * ns; hc.go = in + 3 * ns; hc.group = in + 4 * ns;
  hc.hasg = in + 5 * ns;
  hc.hasg2 = in + 6 * ns;
  hc.slot = in + 8 * ns;
  hc.scnt = in + 9 * ns;
  hc.store = store ? d->store : nullptr;
  hc.lds = d->lds;
  hc.store_cap = store ? d->store_cap : 0;
  hc.cnt = reinterpret_cast<unsigned*>(base + L.cnt);
  hc.part = reinterpret_cast<double*>(base + L.part);
  int* dlist = reinterpret_cast<int*>(base + L.list);
  MrDev* dev = reinterpret_cast<MrDev*>(base + L.dev);
  hc.b = d->b;
  hc.X = d->X; hc.ldx = d->ldx;
  for (int g = 0; g < RSK_MAX_GROUPS; ++g) {
    hc.W[g] = (defl && g < d->ngroups) ? d->W[g] : nullptr;
    hc.J[g] = (defl && g < d->ngroups) ? d->J[g] : 0;
  }
  hc.ldw = defl ? d->ldw : N;
  hc.Ghat = anyg ? d->Ghat : nullptr;
  hc.ldgh = (anyg || anyg2) ? d->ldgh : N;
  hc.Ghat2 = anyg2 ? d->Ghat2 : nullptr;
  hc.nchunk = L.nchunk;
  hc.maxit = d->maxit;

  // ---- ||b||
  MR_CUDA(launch_batch_dot(h, N, 1, d->b, N, d->b, N, h->scal + 8, st));
  double nb2 = 0.0;
  MR_CUDA(cudaMemcpyAsync(&nb2, h->scal + 8, sizeof(double), cudaMemcpyDeviceToHost, st));
  MR_CUDA(cudaStreamSynchronize(st));
  const double nb = std::sqrt(nb2);
  if (nb == 0.0) {
    for (int s = 0; s < ns; ++s) {
      MR_CUDA(cudaMemsetAsync(d->X + (size_t)s * d->ldx, 0, sizeof(double) * N, st));
      if (d->Gout) MR_CUDA(cudaMemsetAsync(d->Gout + (size_t)s * d->ldg, 0, sizeof(double) * N, st));
      o->iters[s] = 0; o->applies[s] = 0; o->relres_true[s] = 0.0; o->status[s] = RSK_CG_ZERO_RHS;
      o->m_used[s] = 0;
      if (o->store_count) o->store_count[s] = 0;
    }
    MR_CUDA(cudaStreamSynchronize(st));
    return RSK_OK;
  }
  hc.tolb = d->tol * nb;

  // ---- eq:localU: Z_s = K_s R_s per shift (no applies), rank-deficient -> drop g-hat, then U~
  std::vector<std::vector<double>> Rs(ns);
  std::vector<int> dropped(ns, 0);
  for (int s = 0; s < ns; ++s) {
    while (m[s] > 0) {
      const int g = grp[s];
      const int J = std::min(d->J[g], m[s]);
      dim3 gz((unsigned)std::min<int64_t>((N + 255) / 256, 1184), m[s]);
      count_launch();
      mr_formz<<<gz, 256, 0, st>>>(N, d->AW[g], d->EW[g], d->ldw, J, d->gamma_h[s],
                                   hasg[s] ? d->ZGhat + (size_t)s * d->ldgh : nullptr,
                                   hasg2[s] ? d->ZGhat2 + (size_t)s * d->ldgh : nullptr, Zs);
      MR_CUDA(cudaGetLastError());
      std::vector<double> R((size_t)m[s] * m[s]);
      double* Ks = hc.Kb + (size_t)s * kMrK * N;
      rsk_status qs = rsk_qr_tall(h, N, m[s], Zs, N, Ks, N, R.data(), st);
      if (qs == RSK_ECUDA) return qs;
      bool ok = qs == RSK_OK;
      if (ok) {
        double dmin = 1e300, dmax = 0.0;
        for (int j = 0; j < m[s]; ++j) {
          const double a = std::fabs(R[j + (size_t)j * m[s]]);
          dmin = std::min(dmin, a);
          dmax = std::max(dmax, a);
        }
        ok = std::isfinite(dmax) && dmin > 1e-14 * dmax;
      }
      if (ok) { Rs[s] = R; break; }
      dropped[s] = 1;
      if ((hasg[s] || hasg2[s]) && m[s] > d->J[g]) { hasg[s] = 0; hasg2[s] = 0; m[s] = d->J[g]; }
      else m[s] = 0;   // the carried columns go first (as one block), then all of U~
    }
  }

  // ---- upload per-shift state
  {
    std::vector<double> dh((size_t)ns * (8 * kMrK + 16 + 2), 0.0);
    for (int s = 0; s < ns; ++s) dh[s] = d->gamma_h[s];
    MR_CUDA(cudaMemcpyAsync(dbl, dh.data(), sizeof(double) * dh.size(), cudaMemcpyHostToDevice, st));
    std::vector<int> ih((size_t)ns * 10, 0);
    for (int s = 0; s < ns; ++s) {
      ih[s] = m[s];
      ih[ns + s] = ST_IDLE;
      ih[3 * ns + s] = 0;
      ih[4 * ns + s] = grp[s];
      ih[5 * ns + s] = hasg[s];
      ih[6 * ns + s] = hasg2[s];
    }
    MR_CUDA(cudaMemcpyAsync(in, ih.data(), sizeof(int) * ih.size(), cudaMemcpyHostToDevice, st));
    MR_CUDA(cudaMemsetAsync(hc.cnt, 0, sizeof(unsigned) * ns * 4, st));
    MR_CUDA(cudaMemcpyAsync(dev, &hc, sizeof(MrDev), cudaMemcpyHostToDevice, st));
  }
  std::vector<int64_t> applies(ns, 0);
  std::vector<int> all(ns), withxp;
  for (int s = 0; s < ns; ++s) {
    all[s] = s;
    if (hasxp[s]) withxp.push_back(s);
  }
  int* dloop = dlist + ns;   // active list of the lockstep chunk (kept while its graph lives)
  auto upload_to = [&](int* dst, const std::vector<int>& v) -> cudaError_t {
    return cudaMemcpyAsync(dst, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice, st);
  };
  auto upload = [&](const std::vector<int>& v) -> cudaError_t { return upload_to(dlist, v); };
  auto grid = [&](size_t nl) { return dim3((unsigned)L.nchunk, (unsigned)nl); };
  // apply A_g to the vectors `src` (ld ldsrc) of the shifts in dlist into R0 (or Wv)
  auto apply_list = [&](const double* src, int64_t ldsrc, double* dst, int nl, double* xdoty,
                        const int* lst) -> cudaError_t {
    ApplyLaunch a{};
    a.X = src; a.ldx = ldsrc; a.Y = dst; a.ldy = N; a.gamma = gam; a.list = lst; a.nlist = nl;
    a.mode = RSK_APPLY_SHIFTED; a.nvec_total = ns; a.xdoty = xdoty;
    return launch_apply(h, a, st);
  };

  // ---- x_0 and r = b - A_g x_0
  for (int s = 0; s < ns; ++s)
    if (!hasxp[s]) MR_CUDA(cudaMemsetAsync(d->X + (size_t)s * d->ldx, 0, sizeof(double) * N, st));
  if (d->Gout)
    MR_CUDA(cudaMemcpy2DAsync(d->Gout, sizeof(double) * d->ldg, d->X, sizeof(double) * d->ldx,
                              sizeof(double) * N, ns, cudaMemcpyDeviceToDevice, st));
  MR_CUDA(cudaMemsetAsync(hc.R0, 0, sizeof(double) * (size_t)N * ns, st));
  if (!withxp.empty()) {
    MR_CUDA(upload(withxp));
    MR_CUDA(apply_list(d->X, d->ldx, hc.R0, (int)withxp.size(), nullptr, dlist));
    for (int s : withxp) applies[s] += 1;
  }
  MR_CUDA(upload(all));
  count_launch();
  mr_resid<<<grid(ns), kMrT, 0, st>>>(dev, dlist);
  MR_CUDA(cudaGetLastError());

  auto restart = [&](const std::vector<int>& lst) -> cudaError_t {
    cudaError_t e = upload(lst);
    if (e != cudaSuccess) return e;
    count_launches(3);
    mr_kdots<<<grid(lst.size()), kMrT, 0, st>>>(dev, dlist, 1);
    mr_start_proj<<<grid(lst.size()), kMrT, 0, st>>>(dev, dlist);
    mr_start_vec<<<grid(lst.size()), kMrT, 0, st>>>(dev, dlist);
    return cudaGetLastError();
  };
  MR_CUDA(restart(all));

  std::vector<int> status(ns, ST_ACTIVE), iters(ns, 0), done(ns, 0), final_status(ns, RSK_CG_CONVERGED);
  std::vector<double> relres(ns, 0.0);
  // cluster-per-shift device loop for L2-resident images (as the CG, cg_cluster.cu)
  bool use_cluster = getenv("RSK_MR_NOCLUSTER") == nullptr && N <= 131072 && h->r >= 1 && !h->ct && h->rank == 1 &&
                     (N % 2 == 0) && (!store || d->lds % 2 == 0) &&
                     ((reinterpret_cast<uintptr_t>(ws) | reinterpret_cast<uintptr_t>(store ? d->store : ws)) & 15) == 0;
  ApplyParams capx;
  bool cl_tma = false;
  if (use_cluster) {
    ApplyLaunch a{};
    a.X = hc.V; a.ldx = N; a.Y = hc.Wv; a.ldy = N; a.gamma = gam; a.nlist = 1; a.nvec_total = ns;
    a.mode = RSK_APPLY_SHIFTED;
    a.xdoty = reinterpret_cast<double*>(1);   // want_dot (accumulated through dot_acc)
    cl_tma = fill_apply_params(h, a, capx, mr_tile_rows(h->r));
    capx.cg = nullptr;
  }
  std::vector<int> it_restart(ns, -1);   // iterations at the last restart (stagnation guard)
  std::vector<int> glist;                // active set of the captured chunk graph
  cudaGraphExec_t gexec = nullptr;
  const bool use_graph = getenv("RSK_MR_NOGRAPH") == nullptr;
  struct GraphGuard {
    cudaGraphExec_t* g;
    ~GraphGuard() { if (*g) cudaGraphExecDestroy(*g); }
  } gguard{&gexec};
  int64_t guard = 0;
  for (;;) {
    MR_CUDA(cudaMemcpyAsync(status.data(), hc.status, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
    MR_CUDA(cudaMemcpyAsync(iters.data(), hc.iters, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
    MR_CUDA(cudaStreamSynchronize(st));
    std::vector<int> active, fin;
    for (int s = 0; s < ns; ++s) {
      if (done[s]) continue;
      if (status[s] == ST_ACTIVE) active.push_back(s);
      else fin.push_back(s);
    }
    if (!fin.empty()) {
      // ---- eq:xFinal for the finished shifts, then the true-residual confirmation
      std::vector<double> c0((size_t)ns * kMrK), kay((size_t)ns * kMrK), tt((size_t)ns * kMrK, 0.0);
      MR_CUDA(cudaMemcpyAsync(c0.data(), hc.c0, sizeof(double) * c0.size(), cudaMemcpyDeviceToHost, st));
      MR_CUDA(cudaMemcpyAsync(kay.data(), hc.kay, sizeof(double) * kay.size(), cudaMemcpyDeviceToHost, st));
      MR_CUDA(cudaStreamSynchronize(st));
      for (int s : fin) {
        const int k = m[s];
        if (k == 0) continue;
        const std::vector<double>& R = Rs[s];
        double* t = &tt[(size_t)s * kMrK];
        for (int j = 0; j < k; ++j) t[j] = c0[(size_t)s * kMrK + j] - kay[(size_t)s * kMrK + j];
        for (int i = k - 1; i >= 0; --i) {      // R t = c0 - K^T A y_m (upper triangular)
          double a = t[i];
          for (int q = i + 1; q < k; ++q) a -= R[i + (size_t)q * k] * t[q];
          t[i] = a / R[i + (size_t)i * k];
        }
      }
      MR_CUDA(cudaMemcpyAsync(hc.tt, tt.data(), sizeof(double) * tt.size(), cudaMemcpyHostToDevice, st));
      MR_CUDA(upload(fin));
      count_launch();
      mr_final<<<grid(fin.size()), kMrT, 0, st>>>(dev, dlist);
      MR_CUDA(cudaGetLastError());
      MR_CUDA(apply_list(d->X, d->ldx, hc.R0, (int)fin.size(), nullptr, dlist));
      count_launch();
      mr_resid<<<grid(fin.size()), kMrT, 0, st>>>(dev, dlist);
      MR_CUDA(cudaGetLastError());
      std::vector<double> rt2(ns);
      MR_CUDA(cudaMemcpyAsync(rt2.data(), hc.rt2, sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
      MR_CUDA(cudaStreamSynchronize(st));
      std::vector<int> again;
      for (int s : fin) {
        applies[s] += 1;
        const double rr = std::sqrt(rt2[s]) / nb;
        relres[s] = rr;
        if (rr <= d->tol) {
          done[s] = 1;
          final_status[s] = dropped[s] ? RSK_CG_DEFL_DROPPED : RSK_CG_CONVERGED;
        } else if (status[s] == ST_BREAKDOWN || !std::isfinite(rr)) {
          done[s] = 1;
          final_status[s] = RSK_CG_BREAKDOWN;
        } else if (iters[s] >= d->maxit || it_restart[s] == iters[s]) {
          done[s] = 1;              // maxit, or a restart that made no Lanczos step
          final_status[s] = RSK_CG_MAXIT;
        } else {
          it_restart[s] = iters[s];
          again.push_back(s);      // restart from x (x_0 <- x, r = b - A_g x)
        }
      }
      if (!again.empty()) {
        MR_CUDA(restart(again));
        for (int s : again) active.push_back(s);
      }
    }
    if (active.empty()) {
      bool all_done = true;
      for (int s = 0; s < ns; ++s) all_done = all_done && done[s];
      if (all_done) break;
      continue;    // restarted shifts whose x_0 + U K^T r is already converged
    }
    // ---- check_every lockstep Lanczos steps over the active shifts: the first chunk
    // of an active set runs eagerly, later ones replay it as a CUDA graph (the
    // per-iteration kernels are short; launch overhead would dominate small batches)
    const unsigned nl = (unsigned)active.size();
    if (use_cluster) {
      // one launch runs every active shift to its stopping point (cluster per shift)
      MR_CUDA(upload_to(dloop, active));
      glist.clear();
      if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
      unsigned* dq = reinterpret_cast<unsigned*>(base + L.q);
      MR_CUDA(cudaMemsetAsync(dq, 0, sizeof(unsigned), st));
      MrClusterParams cp;
      cp.ap = capx;
      cp.g = dev;
      cp.queue = dq;
      cp.list = dloop;
      cp.nl = (int)nl;
      cp.rows = ((N + kMrCS - 1) / kMrCS + 1) / 2 * 2;   // even: 16-byte row pairs
      bool ok = false;
      MR_CUDA(mr_launch_cluster(h, cp, cl_tma, (int)nl, st, &ok));
      if (ok) {
        if (++guard > (int64_t)d->maxit * 4 + 100) {
          h->err = "rsk_minres_recycled_batch: loop guard";
          return RSK_ECUDA;
        }
        continue;
      }
      use_cluster = false;   // could not co-schedule the clusters: lockstep kernels
    }
    const bool same = (active == glist);
    if (!same) {
      MR_CUDA(upload_to(dloop, active));
      if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
      glist = active;
    }
    auto chunk = [&]() -> cudaError_t {
      for (int it = 0; it < d->check_every; ++it) {
        cudaError_t e = apply_list(hc.V, N, hc.Wv, (int)nl, alpha, dloop);
        if (e != cudaSuccess) return e;
        count_launches(3);
        mr_kdots<<<grid(nl), kMrT, 0, st>>>(dev, dloop, 0);
        mr_project<<<grid(nl), kMrT, 0, st>>>(dev, dloop);
        mr_vec<<<grid(nl), kMrT, 0, st>>>(dev, dloop);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    };
    if (!same || !use_graph) {
      MR_CUDA(chunk());
    } else {
      if (!gexec) {
        cudaGraph_t graph = nullptr;
        MR_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        cudaError_t ce = chunk();
        cudaError_t ee = cudaStreamEndCapture(st, &graph);
        MR_CUDA(ce);
        MR_CUDA(ee);
        MR_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
        cudaGraphDestroy(graph);
      } else {
        count_launches((long long)d->check_every * 5);
      }
      MR_CUDA(cudaGraphLaunch(gexec, st));
    }
    if (++guard > (int64_t)d->maxit * 4 + 100) {
      h->err = "rsk_minres_recycled_batch: loop guard";
      return RSK_ECUDA;
    }
  }
  if (d->Gout) {
    count_launch();
    mr_gout<<<dim3((unsigned)std::min<int64_t>((N + 255) / 256, 1184), ns), 256, 0, st>>>(N, ns, d->X, d->ldx,
                                                                                         d->Gout, d->ldg);
    MR_CUDA(cudaGetLastError());
  }
  std::vector<int> scnt_h(ns, 0);
  MR_CUDA(cudaMemcpyAsync(iters.data(), hc.iters, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
  MR_CUDA(cudaMemcpyAsync(scnt_h.data(), hc.scnt, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
  MR_CUDA(cudaStreamSynchronize(st));
  bool partial = false;
  for (int s = 0; s < ns; ++s) {
    o->iters[s] = iters[s];
    o->applies[s] = applies[s] + iters[s];
    o->relres_true[s] = relres[s];
    o->status[s] = final_status[s];
    o->m_used[s] = m[s];
    if (o->store_count) o->store_count[s] = scnt_h[s];
    partial = partial || (final_status[s] != RSK_CG_CONVERGED && final_status[s] != RSK_CG_DEFL_DROPPED);
  }
  int64_t tot = 0;
  for (int s = 0; s < ns; ++s) tot += o->applies[s];
  h->nA += tot;   // matvec accounting: each A_g apply = 1 A + 1 E
  h->nE += tot;
  return partial ? RSK_EPARTIAL : RSK_OK;
}
