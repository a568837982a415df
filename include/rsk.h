/*
 * rsk.h -- C ABI of librsk, the B200-native (sm_100a, fp64) hot path of the
 * recycled shifted solver of arXiv 2306.15049 ("Krylov subspace recycling for
 * general shifted systems ...", Kilmer, de Sturler, O'Connell).
 *
 * Problem (PAPER.md eq:seqsys P:47, eq:shift P:361-365, eq:blkeqn P:126-128):
 *     (A + gamma_l E_k) x^(k,l) = b,   A = C^T C,  E_k = L^T W_k L,  b = C^T d
 * C is a "same"-size 2-D convolution with zero boundary, L = [Dx; Dy]
 * forward differences, W_k the IRN weights (north_star).
 *
 * Conventions for every call
 *   - fp64 only. Images are row-major ny x nx (pixel (i,j) at i*nx + j),
 *     N = ny*nx. A batch of images / a recycle block is "column-major" N x k:
 *     column c starts at ptr + c*ld, ld >= N (elements).
 *   - Array arguments are DEVICE pointers to caller-owned memory unless the
 *     name ends in _h (HOST). Pointers must be 8-byte aligned.
 *   - Ownership: the caller owns every buffer it passes; the library owns the
 *     handle, its PSF tables, a private copy of W_k and its scratch, and never
 *     keeps a caller pointer after a call returns.
 *   - Streams: `stream` is a cudaStream_t passed as void*. Device calls enqueue
 *     asynchronously on it, except rsk_cg_recycled_batch and the helpers that
 *     return host results (documented below), which synchronise `stream`.
 *   - Errors: every call returns rsk_status. RSK_EINVAL = bad argument, nothing
 *     enqueued, outputs untouched. RSK_ECUDA = a CUDA failure; the handle is
 *     then unusable (destroy it). rsk_last_error() gives the message.
 *     Per-shift numerical outcomes are NOT call errors: they are reported in
 *     per-shift status arrays (RSK_CG_*), and the call returns RSK_OK or
 *     RSK_EPARTIAL (some shift not converged). Nothing throws across the ABI.
 *   - Determinism: no floating-point atomics; every reduction has a fixed
 *     order, so results are bitwise reproducible for a fixed (N, launch shape),
 *     independent of which other shifts share the batch.
 *   - Thread safety: one host thread per handle at a time.
 */
#ifndef RSK_H_
#define RSK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rsk_handle_s* rsk_handle;
typedef int rsk_status;

enum {
  RSK_OK = 0,
  RSK_EINVAL = 1,
  RSK_ECUDA = 2,
  RSK_EUNSUPPORTED = 3,
  RSK_EPARTIAL = 4,
  RSK_ENOMEM = 5
};

/* apply modes (rsk_apply_shifted) */
enum {
  RSK_APPLY_SHIFTED = 0, /* Y = A X + gamma_s E X                    */
  RSK_APPLY_SPLIT = 1,   /* Y = A X, EY = E X   (gamma ignored)      */
  RSK_APPLY_C_ONLY = 2,  /* Y = C X             (L-curve residual)   */
  RSK_APPLY_CT_ONLY = 3  /* Y = C^T X           (b = C^T d)          */
};

/* projection ops (rsk_recycle_project) */
enum { RSK_PROJ_UTV = 0, RSK_ADD_UC = 1, RSK_SUB_UC = 2 };

/* per-shift status of rsk_cg_recycled_batch / rsk_orth_guess */
enum {
  RSK_CG_CONVERGED = 0,    /* ||b - A_g x|| <= tol ||b|| on the TRUE residual   */
  RSK_CG_MAXIT = 1,        /* maxit iterations without convergence              */
  RSK_CG_BREAKDOWN = 2,    /* p.A_g p <= 0 or not finite; x = last iterate       */
  RSK_CG_DEFL_DROPPED = 3, /* converged, but G_l was not SPD and U_l was reduced */
  RSK_CG_ZERO_RHS = 4,     /* ||b|| = 0: x = 0, no iterations                    */
  RSK_NOT_SPD = 5,         /* rsk_orth_guess: Cholesky of G(delta) failed        */
  RSK_SINGULAR = 6         /* rsk_oblique_guess: I + delta K^T E U singular      */
};

/* rsk_cg_desc.flags */
enum { RSK_CG_NO_DEFLATION = 1, RSK_CG_STORE_RES = 2, RSK_CG_PROFILE = 4 };

#define RSK_MAX_GROUPS 4
#define RSK_MAX_LOCAL 17 /* |J| <= 16 Ritz columns + 1 carried correction */

/* ------------------------------------------------------------------ lifecycle */

/* rsk_create: bind a handle to `device` for ny x nx images blurred by the
 * centred PSF psf_h[pny][pnx] (host, row-major, pny = pnx odd, 3 <= pny <= 25), i.e.
 *   (C x)[i,j] = sum_{a,b=-r..r} psf[a+r][b+r] x[i-a, j-b], zero boundary
 * (SURVEY O1). The PSF must be rank-1 separable (h = u v^T, as every
 * Gaussian PSF is; detected to 1e-13 relative) -- otherwise RSK_EUNSUPPORTED.
 * C^T uses the flipped PSF, so symmetry is not required. The weights start at
 * W_0 = I on the n(n-1) rows of each difference (pads 0).
 * flags: reserved, pass 0. Returns RSK_EINVAL on bad sizes / non-finite PSF. */
rsk_status rsk_create(rsk_handle* h, int device, int64_t ny, int64_t nx,
                      const double* psf_h, int pny, int pnx, int flags);
/* rsk_create_ct: a handle whose C is Example 2's parallel-beam CT matrix (
 * SURVEY §8(f) f4; reading G38) on n x n images: the line-integral model, entry
 * (ray, pixel) = length of the ray inside the pixel square, pixel (i, j) = the unit square
 * x in [j - n/2, j + 1 - n/2], y in [n/2 - i - 1, n/2 - i]; ray (a, d) is the line
 * x cos(t_a) + y sin(t_a) = d - (ndet - 1)/2 with t_a = angles_deg_h[a] degrees (host
 * [nangles]); rows ordered angle-major; a ray lying on a pixel face counts for the
 * pixel on its high side; C is scaled to unit Frobenius norm. The data length
 * is ndata = nangles * ndet. Built once on the host (CSR of C and of C^T, device
 * resident). On such a handle: rsk_apply_shifted (RSK_APPLY_C_ONLY maps an image to a
 * data vector (ldy >= ndata), RSK_APPLY_CT_ONLY a data vector (ldx >= ndata) to an
 * image; no shift lists for C_ONLY), rsk_make_rhs (xi and d of length ndata),
 * rsk_lcurve_norms (scratch nvec x ndata), the weight / IRN calls and
 * rsk_minres_recycled_batch work; rsk_cg_recycled_batch returns RSK_EUNSUPPORTED (its
 * device loops embed the stencil apply). n in [2, 4096], nangles, ndet >= 1, finite
 * angles, else RSK_EINVAL; nangles * ndet * 2n > 1e9 stored entries -> RSK_ENOMEM. */
rsk_status rsk_create_ct(rsk_handle* h, int device, int64_t n, int nangles, const double* angles_deg_h,
                         int ndet, int flags);
/* rsk_ct_info: ndata, the number of stored entries of C, and the Frobenius norm of C
 * before scaling (host outputs, each nullable). RSK_EINVAL for a non-CT handle. */
rsk_status rsk_ct_info(rsk_handle h, int64_t* ndata, int64_t* nnz, double* fro_unscaled);
/* rsk_create_slab: the handle of one row slab of an ny_global x nx image (SURVEY §8(e2),
 * configs[4] = C5): owned global rows [row0, row0 + nrows) plus up to `halo` >= 2r
 * halo rows on each side, clipped at the image edges -- the handle's image is global rows
 * [max(0, row0 - halo), min(ny_global, row0 + nrows + halo)) and every librsk call on it
 * works on those extended rows (vectors of ext_rows * nx). With the halo rows refreshed
 * from the neighbours, the fused apply is exact on every owned row: the zero-boundary
 * truncation only acts within r rows of the extended array's edge, i.e. inside the halo
 * or at a true image edge. Communication (the halo exchange, the all-reduce of dots) is
 * the caller's, over torch.distributed / NCCL (paper_2306_15049_b200/slab.py) -- the
 * library holds no communicator, so no kernel ever waits on another rank's kernel.
 * EINVAL: bad geometry, halo < 2r, nrows < halo; otherwise as rsk_create. */
rsk_status rsk_create_slab(rsk_handle* h, int device, int64_t ny_global, int64_t nx, int64_t row0,
                           int64_t nrows, const double* psf_h, int pny, int pnx, int halo, int flags);
/* rsk_slab_info: info6_h = {ny_global, ext0, ext1, row0, row1, halo} (host [6]);
 * RSK_EINVAL for a handle not made by rsk_create_slab. */
rsk_status rsk_slab_info(rsk_handle h, int64_t* info6_h);
rsk_status rsk_destroy(rsk_handle h);
const char* rsk_last_error(rsk_handle h);
/* Library build information (static host string). */
const char* rsk_version(void);
/* Number of librsk kernel launches so far in this process (all handles). */
int64_t rsk_launch_count(void);

/* rsk_set_weights: copy W_k into the handle (E_k = L^T W_k L).
 * wx[i][j] weights (Dx x)[i,j] = x[i,j+1]-x[i,j]; wx[i][nx-1] must be 0.
 * wy[i][j] weights (Dy x)[i,j] = x[i+1,j]-x[i,j]; wy[ny-1][j] must be 0.
 * Device pointers, N doubles each. The weights are validated on the device before they
 * are adopted (a host synchronisation of `stream`): a non-finite or negative value, or a
 * non-zero pad (wx[:, nx-1]; wy[ny-1, :] when the handle holds the image's last row),
 * returns RSK_EINVAL and leaves the handle's weights unchanged. IRN weights reach 1/tau,
 * so SPEC's [0, 1] bound is relaxed to >= 0 (reading D2).
 * Streams: the calls of one handle must be issued to one stream at a time (the host-
 * driven helpers stage small coefficients in per-handle device scratch). */
rsk_status rsk_set_weights(rsk_handle h, const double* wx, const double* wy, void* stream);

/* ------------------------------------------------------- the four hot-path calls */

/* rsk_apply_shifted -- the fused matrix-free operator (eq:shift P:361-365):
 *   for s < nvec:  Y_s = A X_s + gamma[s] * E_k X_s          (RSK_APPLY_SHIFTED)
 *                  Y_s = A X_s,  EY_s = E_k X_s               (RSK_APPLY_SPLIT)
 *                  Y_s = C X_s  /  Y_s = C^T X_s               (C_ONLY / CT_ONLY)
 * X, Y: N x nvec device blocks (ldx, ldy >= N), must not overlap (else EINVAL).
 * gamma: device array [nvec] (SHIFTED only; finite, >= 0 -- not checked on device).
 * EY (required for SPLIT, else ignored), xdoty (nullable, device [nvec]):
 *        xdoty[s] = X_s . Y_s (CG's p.Ap), deterministic.
 * Counts nvec applies (1 A + 1 E each; C_ONLY / CT_ONLY count C applies). */
rsk_status rsk_apply_shifted(rsk_handle h, int nvec, const double* X, int64_t ldx,
                             const double* gamma, double* Y, int64_t ldy, double* EY,
                             int64_t ldey, double* xdoty, int mode, void* stream);

/* rsk_apply_shifted_rows -- rsk_apply_shifted restricted to the output rows
 * [row0, row1) of the handle's image (0 <= row0 < row1 <= ny): Y_s (and EY_s) rows
 * outside the range are left untouched; xdoty[s] = X_s . Y_s over the range's rows. The
 * operator itself is unchanged (each output row reads X rows row -/+ 2r, as the full
 * apply): the row-slab solver computes the interior rows, which need no
 * halo, while the halo rows are still in flight, then the rows next to the halos.
 * SHIFTED and SPLIT modes, streaming strip core only (images of >= 512^2 pixels, even
 * widths): otherwise RSK_EUNSUPPORTED and nothing is enqueued (use rsk_apply_shifted).
 * Counts nvec applies only when the range is the whole image. */
rsk_status rsk_apply_shifted_rows(rsk_handle h, int nvec, const double* X, int64_t ldx,
                                  const double* gamma, double* Y, int64_t ldy, double* EY,
                                  int64_t ldey, double* xdoty, int mode, int64_t row0, int64_t row1,
                                  void* stream);

/* rsk_recycle_project -- tall-skinny recycle-space products (U^T r, U c; the
 * Grams of eq:orthupdate and eq:hq):
 *   RSK_PROJ_UTV : Cm (k x nv, column-major, ldc >= k) = U^T V
 *   RSK_ADD_UC   : V += U Cm        RSK_SUB_UC : V -= U Cm
 * U: n x k (ldu), V: n x nv (ldv), Cm: device. 1 <= k <= 256, nv >= 1 (n = rows,
 * usually N). For UTV, V may alias U (Gram); for ADD/SUB, U and V must not
 * overlap (EINVAL). Deterministic. */
rsk_status rsk_recycle_project(rsk_handle h, int op, int64_t n, int k, const double* U,
                               int64_t ldu, int nv, double* V, int64_t ldv, double* Cm,
                               int64_t ldc, void* stream);

/* rsk_irn_weights -- IRN weight update of the outer loop (Alg. 5 P:812-815;
 * north_star rule, readings G2/G3):
 *   wx[i][j] = ((x[i][j+1]-x[i][j])^2 + tau^2)^(-1/2)  (j <= nx-2; 0 at j = nx-1)
 *   wy[i][j] = ((x[i+1][j]-x[i][j])^2 + tau^2)^(-1/2)  (i <= ny-2; 0 at i = ny-1)
 * x: device image. wx, wy: device outputs (both or neither). The handle's
 * weights are NOT changed (call rsk_set_weights to adopt them).
 * eta2 (nullable, device scalar): sum wx_k (Dx x)^2 + sum wy_k (Dy x)^2 under the
 * handle's CURRENT weights -- the L-curve seminorm^2.
 * tau must be finite and > 0 (else EINVAL). */
rsk_status rsk_irn_weights(rsk_handle h, const double* x, double tau, double* wx, double* wy,
                           double* eta2, void* stream);

/* rsk_irn_weights_iso -- isotropic IRN weights (the isotropic TV
 * term of P:117, beta = tau^2; reading G32): one weight per pixel
 *   w[i][j] = (gx^2 + gy^2 + tau^2)^(-1/2),  gx = x[i][j+1]-x[i][j] (0 at j = nx-1),
 *                                            gy = x[i+1][j]-x[i][j] (0 at i = ny-1)
 * written to wx[i][j] (j <= nx-2; 0 at j = nx-1) and wy[i][j] (i <= ny-2; 0 at
 * i = ny-1), computed unfused in that order. Arguments, eta2, ownership and errors
 * as rsk_irn_weights. */
rsk_status rsk_irn_weights_iso(rsk_handle h, const double* x, double tau, double* wx, double* wy,
                               double* eta2, void* stream);

/* rsk_gazzola_weights -- the paper's own edge-preserving weight update
 * (reading G31):
 *   q = L x,  w = |D_k q| / ||D_k q||_inf,  w <- 1 - w.^p,  D_{k+1} = diag(w) D_k,
 *   E_{k+1} = L^T D_{k+1}^2 L.
 * D_k is diagonal over the rows of L and held in the weights' padded layout:
 * dx[i][j] on the Dx row (i, j) (j <= nx-2), dy[i][j] on the Dy row (i <= ny-2),
 * pads 0 (D_0 = I = the identity weights). x: device image (ny x nx).
 * dx, dy: device, IN/OUT (D_k in, D_{k+1} out, pads written 0).
 * wx, wy: device outputs, W_{k+1} = D_{k+1}^2 (adopt with rsk_set_weights).
 * ||D_k q||_inf = 0 leaves D unchanged. p: finite, > 0 (the paper gives no value;
 * p = 2 and 1 are exact squares/copies, 0.5 a sqrt, other p use pow). Uses the
 * handle's scratch; deterministic (max is order-independent). Errors: EINVAL on NULL
 * or misaligned pointers, aliased outputs, bad p. */
rsk_status rsk_gazzola_weights(rsk_handle h, const double* x, double p, double* dx, double* dy,
                               double* wx, double* wy, void* stream);

/* rsk_gazzola_max / rsk_gazzola_update -- the two halves of rsk_gazzola_weights,
 * for a decomposed image (row slabs): m (device scalar) = ||D_k L x||_inf over the
 * handle's grid (a missing Dy row of the grid's last row does not count); the
 * caller may combine the m of several sub-grids (max) before the update, which
 * applies w = |D_k q| / m, w <- 1 - w.^p, D_{k+1} = diag(w) D_k, W = D^2 with that m.
 * Arguments, ownership and errors as rsk_gazzola_weights. */
rsk_status rsk_gazzola_max(rsk_handle h, const double* x, const double* dx, const double* dy,
                           double* m, void* stream);
rsk_status rsk_gazzola_update(rsk_handle h, const double* x, double p, const double* m, double* dx,
                              double* dy, double* wx, double* wy, void* stream);

/* rsk_cg_recycled_batch -- batched deflated CG (the paper's recycled inner
 * solve in CG form; eq:corr_g P:462-468, local spaces eq:localU P:473, Alg. 3/4;
 * readings D1/D3): for every shift l, in lockstep,
 *   U_l = [W_g(l), ghat_l],  Z_l = A_gl U_l = [AW_g + gamma_l EW_g, ZGhat_l]
 *   G_l = sym(U_l^T Z_l) (Cholesky; not SPD -> drop ghat, then all of U: DEFL_DROPPED)
 *   r_p = b - A_gl x_p;  c = G^-1 U^T r_p;  x_0 = x_p + U c;  r_0 = r_p - Z c
 *   p_0 = r_0 - U G^-1 Z^T r_0
 *   loop: w = A_g p; alpha = rho/(p.w); x += alpha p; r -= alpha w; rho' = r.r;
 *         beta = rho'/rho; p = r + beta p - U G^-1 Z^T r
 *   stop when ||r|| <= tol ||b||, confirmed on the true residual b - A_g x
 *   (restart from it otherwise).
 * Host-blocking: polls convergence every check_every iterations, returns when
 * every shift is finished. Returns RSK_OK, or RSK_EPARTIAL if some shift did
 * not converge. `ws` is a caller-allocated device workspace of at least
 * rsk_cg_workspace_bytes(h, nshift, flags) bytes. */
typedef struct {
  int nshift;
  const double* gamma_h;        /* host [nshift], >= 0 finite                   */
  const double* b;              /* device, N                                     */
  double* X;                    /* device N x nshift: in x_p (if has_xp), out x  */
  int64_t ldx;
  const int* has_xp_h;          /* host [nshift] or NULL (NULL: all x_p = 0)     */
  double* Gout;                 /* device N x nshift or NULL: g = x - x_p*/
  int64_t ldg;
  int ngroups;                  /* 0..RSK_MAX_GROUPS                             */
  const int* group_of_shift_h;  /* host [nshift]                                  */
  const double* W[RSK_MAX_GROUPS];  /* device N x J[g], orthonormal columns      */
  const double* AW[RSK_MAX_GROUPS]; /* A W                                       */
  const double* EW[RSK_MAX_GROUPS]; /* E_k W                                     */
  int64_t ldw;
  int J[RSK_MAX_GROUPS];        /* <= 16                                          */
  const double* Ghat;           /* device N x nshift (ldgh) or NULL              */
  const double* ZGhat;          /* device N x nshift: (A + gamma_l E) ghat_l     */
  int64_t ldgh;
  const int* has_ghat_h;        /* host [nshift] or NULL                         */
  double tol;
  int maxit;
  int check_every;              /* lockstep iterations between host polls (>=1) */
  int flags;                    /* RSK_CG_*                                      */
  double* store;                /* RSK_CG_STORE_RES: device, shift s column c at */
  int64_t lds;                  /*   store + (s*store_cap + c)*lds               */
  int store_cap;
  const int* order_h;           /* host [nshift] permutation or NULL: the order  */
                                /* in which the device loop starts the shifts    */
                                /* (longest first shortens the makespan; results */
                                /* do not depend on it)                          */
  const double* Ghat2;          /* second carried column per shift (Alg. 3's     */
  const double* ZGhat2;         /*   g^(k,l-1); ld ldgh) and its image;   */
  const int* has_ghat2_h;       /*   rsk_minres_recycled_batch only (NULL here)  */
} rsk_cg_desc;

typedef struct {                /* host arrays [nshift], filled on return        */
  int* iters;                   /* w = A_g p applies in the loop                 */
  int64_t* applies;             /* all A_g applies (iters + r_p + confirmations) */
  double* relres_true;          /* ||b - A_g x|| / ||b|| at exit                 */
  int* status;                  /* RSK_CG_*                                      */
  int* m_used;                  /* recycle columns used                           */
  int* store_count;             /* residuals stored (RSK_CG_STORE_RES) or NULL   */
  double* ms_loop;              /* NULL or [8]: RSK_CG_PROFILE (host-polled loop) */
                                /*  [0..4] = {apply ms, update ms, apply launches,*/
                                /*  apply px-vectors, combine ms}; always: [5] ms */
                                /*  of the device-loop kernel (CUDA events on the */
                                /*  launching stream), [6] its shift-iterations  */
                                /*  (loop applies incl. confirms), [7] loop kind  */
                                /*  (1 cluster-per-shift, 2 persistent, 0 host)   */
} rsk_cg_out;

size_t rsk_cg_workspace_bytes(rsk_handle h, int nshift, int flags);
rsk_status rsk_cg_recycled_batch(rsk_handle h, const rsk_cg_desc* d, rsk_cg_out* o, void* ws,
                                 size_t ws_bytes, void* stream);

/* rsk_minres_recycled_batch -- recycling MINRES batched over shifts: the paper's
 * OWN inner solver (PAPER.md §"Shift Specific Recycling" P:454-534; SURVEY §8(f)
 * f2(ii)), an alternative to the deflated CG above on the same descriptor. Per
 * shift l, with U~_l = [W_g, ghat_l] and Z_l = (A + gamma_l E) U~_l =
 * [AW_g + gamma_l EW_g, ZGhat_l] (no applies) -- with has_ghat2_h also
 * the second carried column of Alg. 3 / Alg. 4 (U~_l = [W, g^(k-1,l), g^(k,l-1)],
 * Ghat2 / ZGhat2):
 *   eq:localU    Z_l = K_l R_l, K_l^T K_l = I (shifted Cholesky QR3; R_l singular
 *                to 1e-14 relative -> drop the carried columns, then U~: DEFL_DROPPED)
 *   eq:corr_g    r = b - A_g x_p (one apply when has_xp), solve for g = x - x_p
 *   eq:minShift  Lanczos on (I - K K^T) A_g from (I - K K^T) r, the y-block
 *                least squares by Givens rotations (MINRES), the z-block exactly
 *   eq:xFinal    x = x_p + y_m + U~ R^-1 K^T (r - A_g y_m)
 *   stop when the least-squares residual <= tol ||b||, confirmed on the true
 *   residual b - A_g x (restart from x otherwise; reading G14).
 * Same ownership, stream and error conventions as rsk_cg_recycled_batch: the call
 * is host-blocking, `X` holds x_p in and x out, `Gout` (nullable) receives
 * g = x - x_p; with RSK_CG_STORE_RES the first store_cap normalised Lanczos vectors
 * v_1, v_2, ... (the span of CG's normalised residuals) go to `store` exactly as the
 * CG's residuals do (store_count filled). iters = Lanczos applies;
 * applies = iters + the r_p apply + one per true-residual confirmation. ms_loop is
 * not written. `ws`: at least rsk_minres_workspace_bytes(h, nshift, kmax) bytes,
 * kmax = max_l (J_g(l) + has_ghat_l) <= RSK_MAX_LOCAL (7 N-vectors + kmax
 * N-vectors (K_l) per shift). Returns RSK_OK, or RSK_EPARTIAL if a shift did not
 * converge (status MAXIT / BREAKDOWN). */
size_t rsk_minres_workspace_bytes(rsk_handle h, int nshift, int max_local_dim);
rsk_status rsk_minres_recycled_batch(rsk_handle h, const rsk_cg_desc* d, rsk_cg_out* o, void* ws,
                                     size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ support calls */

/* rsk_make_rhs: d = C x_true + nu ||C x_true|| xi/||xi|| (eq:forward P:107,
 * reading G21), b = C^T d. All device, N each. Enqueued on stream. */
rsk_status rsk_make_rhs(rsk_handle h, const double* x_true, const double* xi, double nu,
                        double* d, double* b, void* stream);

/* rsk_batch_dot: out[j] = X_j . Y_j for j < nv (device out[nv]). */
rsk_status rsk_batch_dot(rsk_handle h, int64_t n, int nv, const double* X, int64_t ldx,
                         const double* Y, int64_t ldy, double* out, void* stream);

/* rsk_batch_axpby: Y_j = a[j] X_j + b[j] Y_j, a_h / b_h HOST arrays [nv <= 1024]
 * (b_h may be NULL meaning 1). X may be NULL meaning 0 (pure scaling). */
rsk_status rsk_batch_axpby(rsk_handle h, int64_t n, int nv, const double* a_h,
                           const double* X, int64_t ldx, const double* b_h, double* Y,
                           int64_t ldy, void* stream);

/* rsk_qr_tall: thin QR of the n x k block V (the "skinny QR" of P:188, P:849 and the
 * orthogonalisations of Alg. 1 / eq:establishU) by shifted Cholesky QR3
 * (Gram + shifted Cholesky, then two Cholesky-QR passes): V = Q R with Q^T Q = I
 * to working precision for cond(V) up to ~1e15, R upper triangular with R_jj > 0.
 * V (device, ldv) is OVERWRITTEN as scratch; Q (device, ldq) receives the
 * orthonormal factor; R_h (host, k x k, column-major) receives R. k <= 256,
 * n >= k. Zero columns are not allowed (drop them first). Synchronises stream. */
rsk_status rsk_qr_tall(rsk_handle h, int64_t n, int k, double* V, int64_t ldv, double* Q,
                       int64_t ldq, double* R_h, void* stream);

/* rsk_lcurve_norms: for s < nvec, rho[s] = ||C X_s - d|| and
 * eta[s] = ||W_k^(1/2) L X_s|| under the handle's weights.
 * Device outputs; scratch: device N x nvec. */
rsk_status rsk_lcurve_norms(rsk_handle h, int nvec, const double* X, int64_t ldx,
                            const double* d, double* rho, double* eta, void* scratch,
                            void* stream);

/* rsk_get_counters: cumulative apply counts (matvec accounting, §6). */
/* eta2[s] = sum over image rows [row0, row1) of wx (Dx x_s)^2 + wy (Dy x_s)^2 under the
 * handle's weights (the L-curve seminorm^2 of P:149 / P:161 restricted to a row range; Dy of
 * the range's last row reads the next image row when there is one). Row slabs (§8(e2)) sum
 * their owned rows and all-reduce. eta2: device [nvec]. */
rsk_status rsk_seminorm_rows(rsk_handle h, int nvec, const double* X, int64_t ldx, int64_t row0, int64_t row1,
                             double* eta2, void* stream);

rsk_status rsk_get_counters(rsk_handle h, int64_t* applies_A_h, int64_t* applies_E_h,
                            int64_t* applies_C_h, int reset);

/* ---------------------------------------------------- host small-dense helpers
 * (no handle, no device; all arrays host, column-major) */

/* rsk_orth_guess: the principal-space initial guesses of eq:orthupdate
 * from the anchoring Grams, for m shifts. With (A + gamma_* E) U~ = K R
 * (eq:establishU; R upper triangular, nc x nc) and U = U~ R^-1 never formed:
 *   P  = K^T E U   = KtZE R^-1          Q2 = (E U)^T (E U) = R^-T ZEtZE R^-1
 *   u  = U^T E b   = R^-T ZEtb           v  = K^T b = Ktb
 *   delta_l = gamma_l - gamma_star
 *   G(delta) = I + delta (P + P^T) + delta^2 Q2;   G q = v + delta u  (Cholesky)
 *   C[:,l] = R^-1 q     (so x_0 = U~ C[:,l])
 * KtZE = K^T Z_E, ZEtZE = Z_E^T Z_E (nc x nc), ZEtb = Z_E^T b, Ktb = K^T b.
 * A failed Cholesky sets status_h[l] = RSK_NOT_SPD and C[:,l] = 0 (x_0 = 0). */
rsk_status rsk_orth_guess(int nc, const double* R_h, const double* KtZE_h, const double* ZEtZE_h,
                          const double* ZEtb_h, const double* Ktb_h, double gamma_star, int m,
                          const double* gamma_h, double* C_h, int* status_h);

/* rsk_oblique_guess -- the oblique-projection initial guesses of §sec:oblique
 * (eq:obliqueupdate P:877-882): with (A + gamma_a E) U~ = K R at
 * an anchor shift gamma_a and U = U~ R^-1 (never formed), x_0 = U q with K^T r_0 = 0:
 *   (I + delta_l K^T E U) q = K^T b,   K^T E U = KtZE R^-1,   delta_l = gamma_l - gamma_a
 *   C[:,l] = R^-1 q     (x_0 = U~ C[:,l])
 * Dense LU with partial pivoting per shift. Two anchors (eq:updates P:1000-1005) are
 * two calls, one per shift group, each with its own R, KtZE, Ktb, gamma_a.
 * All host arrays, column-major: R_h, KtZE_h nc x nc; Ktb_h nc; gamma_h m; C_h nc x m.
 * An exactly singular (or non-finite) system sets status_h[l] = RSK_SINGULAR and
 * C[:,l] = 0. EINVAL on NULL, nc <= 0, m < 0, a zero diagonal of R, non-finite gamma_a. */
rsk_status rsk_oblique_guess(int nc, const double* R_h, const double* KtZE_h, const double* Ktb_h,
                             double gamma_anchor, int m, const double* gamma_h, double* C_h,
                             int* status_h);

/* rsk_pencil_ritz: Alg. 2 on the projected pencil (eq:hq P:677):
 * H = sym(Ahat) + gamma sym(Ehat) (nc x nc); cyclic-Jacobi eigenvectors, ascending;
 * Wt_h (nc x J) = eigenvectors of the J smallest Ritz values theta_h[J]. */
rsk_status rsk_pencil_ritz(int nc, const double* Ahat_h, const double* Ehat_h, double gamma, int J,
                           double* Wt_h, double* theta_h);

/* rsk_stabilize_small: Alg. 1 applied to the R factor of a thin QR of a
 * raw block X = Q R whose columns are to be scaled to unit norm (reading G6):
 * Rs = R diag(1/sqrt(colnorm2)), Rs = Ur S Vr^T (one-sided Jacobi), keep the leading
 * i with s_1/s_i < condcap (strict), at most cap. Zs_h (k x nkeep) = Ur(:,keep),
 * so U~ = Q Zs. */
rsk_status rsk_stabilize_small(int k, const double* R_h, const double* colnorm2_h, double condcap,
                               int cap, double* Zs_h, int* nkeep);

/* rsk_carried_select: the near-duplicate test of the local-space update (footnote P:691,
 * reading G12): keep_h[l] = (gnorm2_h[l] > 0 && sqrt(ghnorm2_h[l] / gnorm2_h[l]) >= thr)
 * and scale_h[l] = 1/sqrt(ghnorm2_h[l]) (0 when dropped). */
rsk_status rsk_carried_select(int m, const double* gnorm2_h, const double* ghnorm2_h, double thr,
                              double* scale_h, int* keep_h);

/* rsk_sym_eig: symmetric eigen-decomposition of sym(H) (n x n) by cyclic Jacobi,
 * eigenvalues ascending in theta_h[n], eigenvectors in V_h. */
rsk_status rsk_sym_eig(int n, const double* H_h, double* theta_h, double* V_h);

/* rsk_svd_small: one-sided Jacobi SVD of the k x k R (host): R = Ur S Vr^T,
 * singular values descending. */
rsk_status rsk_svd_small(int k, const double* R_h, double* Ur_h, double* s_h, double* Vr_h);

/* rsk_chol_solve_small: solve sym(G) x = z by Cholesky, nrhs right-hand sides.
 * Returns RSK_EPARTIAL (x untouched) if G is not SPD. */
rsk_status rsk_chol_solve_small(int n, const double* G_h, int nrhs, const double* Z_h,
                                double* X_h);

/* rsk_lcurve_corner: argmax of the discrete curvature of (log rho, log eta)
 * (reading G25): centred differences on the uniform log-lambda grid,
 * endpoints excluded, ties to the smallest index. Returns the 0-based index in
 * *lstar; kappa_h (nullable, [M]) receives the curvatures (-inf at the ends). */
/* Host step of one shifted-Cholesky-QR pass (rsk_qr_tall runs three): from G = V^T V of
 * the pass input (k x k column-major; n = global rows) returns T = R_pass^-1 (upper) with
 * V T the pass output, and updates Racc <- R_pass Racc (pass 0: Racc = R_pass). Row slabs
 * all-reduce G and apply T to their own rows. RSK_EPARTIAL if Cholesky fails. Host only. */
rsk_status rsk_cholqr_pass(int k, int64_t n, int pass, const double* G_h, double* T_h, double* Racc_h);

/* ---- deflated-CG host steps (row-slab loop; also used by the
 * single-domain setup). Loop states: */
enum { RSK_LOOP_ACTIVE = 0, RSK_LOOP_RCONV = 1, RSK_LOOP_DONE = 2, RSK_LOOP_BREAKDOWN = 3, RSK_LOOP_MAXIT = 4 };

/* Local Gram matrices G_l = sym(U_l^T (A + gamma_l E) U_l) of U_l = [W_g, ghat_l] (Alg. 3/4
 * P:700-746, reading D1) assembled from reduced host pieces, and their Cholesky factors;
 * on failure the carried column is dropped, then all of U (dropped_h[s] = 1). WA/WE:
 * [g][256] J_g x J_g (ld J_g) = W^T A W, W^T E W; WZg/AWg/EWg: [g][16 ns] J_g x ns = W^T Zghat_s,
 * (AW)^T ghat_s, (EW)^T ghat_s; gzg [ns] = ghat_s^T Zghat_s (NULL if no ghat). hasg_h in/out.
 * L_h: [ns][RSK_MAX_LOCAL^2], lower, column-major, ld RSK_MAX_LOCAL. Host only. */
rsk_status rsk_local_gram_factors(int ns, int ngroups, const int* J_h, const int* group_of_shift_h,
                                  const double* gamma_h, const double* WA_h, const double* WE_h,
                                  const double* WZg_h, const double* AWg_h, const double* EWg_h,
                                  const double* gzg_h, double* L_h, int* m_h, int* hasg_h, int* dropped_h);

/* mu_s = G_s^-1 [zA_s + gamma_s zE_s ; zG_s] with the factors of rsk_local_gram_factors
 * (zA: J x ns, ld J; zE, zG nullable = 0; mu: [ns][RSK_MAX_LOCAL]). Host only. */
rsk_status rsk_gram_solve(int ns, int J, const double* L_h, const int* m_h, const int* hasg_h,
                          const double* gamma_h, const double* zA_h, const double* zE_h, const double* zG_h,
                          double* mu_h);

/* alpha_s = rho_s / (p_s . w_s) for shifts in RSK_LOOP_ACTIVE (O4 step 3); a non-positive
 * or non-finite p.w sets RSK_LOOP_BREAKDOWN. Host arrays [ns]. */
rsk_status rsk_cg_alpha(int ns, const double* rho_h, const double* pw_h, double* alpha_h, int* state_h);

/* Scalar half of an iteration from the reduced sums of the new residual (O4 steps 3-4):
 * rho' = r.r, zA = (AW)^T r, zE = (EW)^T r (J x ns, ld J), zG = ZGhat^T r. mode_h = state at
 * the iteration start (ACTIVE: loop step, RCONV: r is the true residual). Updates rho, iters,
 * rho_true, nconf, state; writes beta and mu = G^-1 z ([ns][RSK_MAX_LOCAL]). Host only. */
rsk_status rsk_cg_scalars(int ns, int J, const int* mode_h, const double* gamma_h, const double* rho_new_h,
                          const double* zA_h, const double* zE_h, const double* zG_h, const int* m_h,
                          const int* hasg_h, const double* L_h, double thr, int maxit, double* rho_h,
                          double* beta_h, double* mu_h, int* iters_h, double* rho_true_h, int* nconf_h,
                          int* state_h);

rsk_status rsk_lcurve_corner(int M, const double* rho_h, const double* eta_h, int* lstar,
                             double* kappa_h);

#ifdef __cplusplus
}
#endif
#endif /* RSK_H_ */
