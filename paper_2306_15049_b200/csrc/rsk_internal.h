// Internal declarations of librsk (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/rsk.h"

namespace rsk {

constexpr int kMaxR = 12;                 // PSF half width supported by the fused apply
constexpr int kMaxTaps = 4 * kMaxR + 1;   // taps of B = G^T G
constexpr int kMaxM = RSK_MAX_LOCAL;      // local recycle dimension
constexpr int kNT = 256;                  // threads per CTA for streaming kernels
constexpr size_t kAuxBytes = sizeof(double) * (2 * 256 * 256 + 8192);

// apply tile: (64 - 4r) x kTX output pixels per work item
constexpr int kTX = 64;
// partial rows of the group update kernel: 2 x 16 GEMM rows + rho + ZGhat.r
constexpr int kGrpStride = 34;
constexpr int kMaxChunkG = 256;
constexpr int kPartRowsG = 18;                     // z (16) + rho + ZGhat.r
constexpr int kTickStride = 2 + kMaxChunkG / 16 + 1; // per (group, tile) tickets

// ---- per-shift CG status on the device
enum DevStatus : int {
  ST_ACTIVE = 0,      // iterating
  ST_RCONV = 1,       // recursive residual below tol: needs the true-residual confirm
  ST_DONE = 2,        // confirmed
  ST_BREAKDOWN = 3,
  ST_MAXIT = 4,
  ST_IDLE = 5         // not in this solve (ZERO_RHS, finished)
};

struct GroupPtrs {
  const double* W[RSK_MAX_GROUPS];
  const double* AW[RSK_MAX_GROUPS];
  const double* EW[RSK_MAX_GROUPS];
  int J[RSK_MAX_GROUPS];
  int64_t ldw;
};

// Device-resident state of one rsk_cg_recycled_batch call (carved from ws).
struct CgDev {
  int nshift;
  int64_t N;
  double* R;        // residuals      N x nshift (ld N)
  double* P;        // directions     N x nshift
  double* Wv;       // A_g p / scratch N x nshift
  double* X;        // caller x       (ldx)
  int64_t ldx;
  const double* b;
  const double* Ghat;   // (ldgh) or null
  const double* ZGhat;
  int64_t ldgh;
  double* store;    // residual store or null
  int64_t lds;
  int store_cap;
  // scalars per shift
  double* gam;      // gamma_s
  double* rho;
  double* alpha;
  double* beta;
  double* coef;     // [nshift][kMaxM]  mu (loop) or c (Galerkin start)
  double* Lf;       // [nshift][kMaxM*kMaxM] Cholesky factor (lower, column-major)
  double* rho_true; // true residual^2 at last confirm
  int* status;
  int* iters;
  int* mloc;        // local dimension (after drops)
  int* hasg;        // carried column present (after drops)
  int* group;
  int* store_cnt;
  int* nconf;       // true-residual confirmations done (persistent loop)
  int* stslot;      // residual-store slot of the current iteration, or -1
  unsigned* cnt;    // [nshift][4] last-CTA counters
  double* partA;    // [nshift][nblkA]
  double* partB;    // [nshift][nblkB][kMaxM+1]
  int nblkA;
  int nblkB;
  double bnorm;     // ||b||
  double tol;
  int maxit;
  GroupPtrs grp;
  // group-shared hot-loop kernels (cg_group.cu)
  int* glist;       // active shift ids, grouped: group g at glist[gmeta[g] .. + gmeta[4+g])
  int* gmeta;       // [0..3] offsets, [4..7] counts
  double* partG;    // [4][maxtilesG][nchunkG][kGrpStride][32]
  unsigned* cntG;   // [4][maxtilesG][2]
  int nchunkG;
  int64_t rowsG;
  int maxtilesG;
};

// ---- handle
struct Handle {
  int device = 0;
  int64_t ny = 0, nx = 0;
  int r = 0;
  double u[2 * kMaxR + 1];    // PSF column factor (rows, y)
  double v[2 * kMaxR + 1];    // PSF row factor (cols, x)
  double cBx[kMaxTaps], cBy[kMaxTaps];      // interior taps of B = G^T G
  double cCx[kMaxTaps], cCy[kMaxTaps];      // taps of C   (window form)
  double cTx[kMaxTaps], cTy[kMaxTaps];      // taps of C^T (window form)
  // rank-2 PSF h = u v^T + u2 v2^T (Example 1's C = sum_i C_i^(1) (x) C_i^(2)):
  // the second term's C / C^T taps; the fused-apply device loops are rank-1 only
  int rank = 1;
  double u2[2 * kMaxR + 1], v2[2 * kMaxR + 1];
  double cCx2[kMaxTaps], cCy2[kMaxTaps], cTx2[kMaxTaps], cTy2[kMaxTaps];
  double* r2buf = nullptr;     // rank-2 apply temporaries (3 x vectors x N), grown on demand
  size_t r2bytes = 0;
  double* tabBx = nullptr;    // [nx][4r+1]
  double* tabBy = nullptr;    // [ny][4r+1]
  double* dcorr = nullptr;    // [4][kMaxR][kMaxR] zero-boundary corner corrections of Bx, By
  double* wx = nullptr;       // weights copy
  double* wy = nullptr;
  double* scratch = nullptr;  // reduction scratch
  size_t scratch_bytes = 0;
  double* scal = nullptr;     // small device scalars
  double* aux = nullptr;      // small device buffers for host-driven helpers (kAuxBytes)
  int64_t nA = 0, nE = 0, nC = 0;
  std::string err;
  int sm_count = 148;
  bool sticky = false;
  cudaStream_t cg_stream = nullptr;  // private capture-capable stream of rsk_cg_recycled_batch
  // row slab (rsk_create_slab): this handle's rows are global rows [slab_ext0, slab_ext1),
  // of which [slab_row0, slab_row1) are owned; ny_global = the whole image
  int64_t ny_global = 0, slab_ext0 = 0, slab_ext1 = 0, slab_row0 = 0, slab_row1 = 0, slab_halo = 0;
  // CT operator (rsk_create_ct, ct.cu): C as CSR over rays and C^T as CSR over pixels
  bool ct = false;
  int64_t ndata = 0;          // length of a data vector d: ny*nx (blur) or rays (CT)
  double ct_fro = 0.0;        // Frobenius norm of the unscaled matrix
  int64_t ct_nnz = 0;
  int ct_tmp_vecs = 0;        // capacity of ct_tmp in data vectors
  int64_t* ct_rp = nullptr;
  int* ct_col = nullptr;
  double* ct_val = nullptr;
  int64_t* ctT_rp = nullptr;
  int* ctT_col = nullptr;
  double* ctT_val = nullptr;
  double* ct_tmp = nullptr;   // C x of an apply batch
};

// ---- launchers (apply.cu)
struct ApplyLaunch {
  const double* X; int64_t ldx;
  double* Y; int64_t ldy;
  double* EY; int64_t ldey;
  const double* gamma;        // indexed by shift id
  const int* list;            // device list of shift ids (nullable => identity)
  int nlist;
  int mode;                   // RSK_APPLY_*
  double* xdoty;              // nullable, indexed by shift id
  CgDev* cg;                  // nullable => plain apply; else CG "w = A p" step
  bool cg_alpha;              // CG: compute alpha = rho / (p.w) in last CTA
  const int* nlist_dev;       // nullable: list length read on the device (graph replay)
  const double* X2; int64_t ldx2;  // CG: source of items whose shift is ST_RCONV (confirm)
  bool src2_rconv;
  int nvec_total;              // vectors addressable in X (and X2): TMA map extent
};
cudaError_t launch_apply(Handle* h, const ApplyLaunch& a, cudaStream_t st);
// the tiled apply kernel with explicit taps (C / C^T passes of one rank-1 term, or E alone
// with zero taps); no dot products, no CG mode (apply.cu)
cudaError_t launch_apply_taps(Handle* h, const ApplyLaunch& a, const double* cx, const double* cy, int edge_fix,
                              cudaStream_t st);
// rank-2 PSF handles: the apply as a composition of rank-1 C / C^T passes (apply_rank2.cu)
cudaError_t launch_apply_rank2(Handle* h, const ApplyLaunch& a, cudaStream_t st);
// streaming strip apply for large images (apply_strip.cu); cudaErrorNotSupported = not applicable
constexpr int64_t kStripMinN = 512 * 512;
cudaError_t launch_apply_strip(Handle* h, const ApplyLaunch& a, cudaStream_t st, int row0 = 0, int row1 = 0);
cudaError_t launch_ct_apply(Handle* h, const ApplyLaunch& a, cudaStream_t st);   // ct.cu
int apply_tiles(const Handle* h);
int apply_tile_rows(int r);


// ---- vector kernels (vec.cu)
cudaError_t launch_gemm_tn(Handle* h, int64_t n, int k, const double* U, int64_t ldu, int nv,
                           const double* V, int64_t ldv, double* C, int64_t ldc, cudaStream_t st);
cudaError_t launch_gemm_nn(Handle* h, int64_t n, int k, const double* U, int64_t ldu, int nv,
                           double* V, int64_t ldv, const double* C, int64_t ldc, double sign,
                           cudaStream_t st);
cudaError_t launch_batch_dot(Handle* h, int64_t n, int nv, const double* X, int64_t ldx,
                             const double* Y, int64_t ldy, double* out, cudaStream_t st);
cudaError_t launch_batch_axpby(int64_t n, int nv, const double* a, const double* X,
                               int64_t ldx, const double* b, double* Y, int64_t ldy,
                               cudaStream_t st);  // a, b DEVICE arrays (b nullable)
cudaError_t launch_irn(Handle* h, const double* x, double tau, int iso, double* wx, double* wy,
                       double* eta2, cudaStream_t st);
cudaError_t launch_gazzola_max(Handle* h, const double* x, const double* dx, const double* dy, double* m,
                               cudaStream_t st);
cudaError_t launch_gazzola_update(Handle* h, const double* x, double pw, const double* m, double* dx,
                                  double* dy, double* wx, double* wy, cudaStream_t st);
cudaError_t launch_seminorm_batch(Handle* h, int nvec, const double* X, int64_t ldx,
                                  double* eta2, cudaStream_t st, int do_sqrt = 0);
cudaError_t launch_seminorm_rows(Handle* h, int nvec, const double* X, int64_t ldx, int row0, int row1,
                                 double* eta2, cudaStream_t st);
cudaError_t launch_diffnorm_batch(Handle* h, int nvec, const double* Y, int64_t ldy,
                                  const double* d, double* out, cudaStream_t st);
cudaError_t launch_scale_noise(int64_t n, const double* cx, const double* xi, const double* s2,
                               double nu, double* d, cudaStream_t st);

// CG kernels (vec.cu)
enum UpdMode { UPD_LOOP = 0, UPD_START = 1, UPD_GALERKIN = 2, UPD_CONFIRM = 3 };
cudaError_t launch_cg_update(CgDev* dev, const CgDev& host, const int* list, int nlist, int mode,
                             cudaStream_t st);
enum CmbMode { CMB_LOOP = 0, CMB_GALERKIN = 1, CMB_RESID = 2, CMB_GOUT = 3 };
cudaError_t launch_cg_combine(CgDev* dev, const CgDev& host, const int* list, int nlist, int mode,
                              cudaStream_t st);
int cg_nblkB(int64_t N);
cudaError_t launch_cg_update_grp(CgDev* dev, const CgDev& host, int ngroups, int maxtiles, cudaStream_t st);
cudaError_t launch_cg_combine_grp(CgDev* dev, const CgDev& host, int ngroups, int maxtiles, cudaStream_t st);
// cluster-per-shift loop (cg_cluster.cu)
cudaError_t launch_cg_cluster(Handle* h, CgDev* dev, const CgDev& hc, unsigned* queue, const int* order,
                              double* zw, cudaStream_t st, bool* ok);
int64_t cluster_max_n();          // largest N run cluster-per-shift (L2-resident working set)
int cluster_slots(const Handle* h);   // upper bound on concurrently running clusters
// persistent lockstep loop (cg_persist.cu)
int persist_grid(const Handle* h);
int persist_max_shift();
int persist_pv();
cudaError_t launch_cg_persist(Handle* h, CgDev* dev, const CgDev& hc, double* partP, unsigned* bar,
                              int* nactive, int* iters_done, int nchunk, int64_t rows, int max_iters,
                              cudaStream_t st, bool* ok);

// streaming persistent loop for images beyond L2 (cg_stream.cu)
int stream_ipv(const Handle* h);
int stream_nchunk(const Handle* h);
int stream_pv();
cudaError_t launch_cg_stream(Handle* h, CgDev* dev, const CgDev& hc, double* partA, double* partB, unsigned* bar,
                             int* nactive, int* iters_done, int max_iters, cudaStream_t st, bool* ok);

// kernel-launch accounting (rsk_launch_count): every librsk kernel launch bumps it
void count_launch();
void count_launches(long long n);

// host dense (host_dense.cpp)
bool chol_lower(int n, double* A);  // in-place, column-major lower; false if not SPD
void chol_solve_lower(int n, const double* L, double* x);
void jacobi_eig(int n, const double* H, double* theta, double* V);
void jacobi_svd(int k, const double* R, double* Ur, double* s, double* Vr);

}  // namespace rsk
