// Small dense linear algebra on the host (n_c x n_c and smaller): Cholesky,
// cyclic Jacobi symmetric eigensolver (Alg. 2), one-sided Jacobi SVD
// (Alg. 1 applied to R), the per-shift initial-guess solves of
// eq:orthupdate and the L-curve corner.
// Written independently of the oracle (which uses numpy.linalg).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "rsk_internal.h"

namespace rsk {

// In-place Cholesky of a column-major n x n SPD matrix: lower triangle <- L.
bool chol_lower(int n, double* A) {
  for (int j = 0; j < n; ++j) {
    double d = A[j + j * n];
    for (int k = 0; k < j; ++k) d -= A[j + k * n] * A[j + k * n];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    d = std::sqrt(d);
    A[j + j * n] = d;
    for (int i = j + 1; i < n; ++i) {
      double t = A[i + j * n];
      for (int k = 0; k < j; ++k) t -= A[i + k * n] * A[j + k * n];
      A[i + j * n] = t / d;
    }
    for (int i = 0; i < j; ++i) A[i + j * n] = 0.0;
  }
  return true;
}

void chol_solve_lower(int n, const double* L, double* x) {
  for (int i = 0; i < n; ++i) {
    double t = x[i];
    for (int j = 0; j < i; ++j) t -= L[i + j * n] * x[j];
    x[i] = t / L[i + i * n];
  }
  for (int i = n - 1; i >= 0; --i) {
    double t = x[i];
    for (int j = i + 1; j < n; ++j) t -= L[j + i * n] * x[j];
    x[i] = t / L[i + i * n];
  }
}

// Symmetric eigendecomposition (Golub & Van Loan, Matrix Computations, 4th ed., §8.3):
// Householder tridiagonalisation Q^T A Q = T, then implicit symmetric QR steps with the
// Wilkinson shift on T (bulge chasing by Givens rotations, accumulated into Q); O(n^3)
// once instead of cyclic Jacobi's O(n^3) per sweep. A: n x n column-major (symmetric).
// On return d = eigenvalues (unsorted), Q = eigenvectors (columns, column-major).
// Returns false if the QR iteration does not converge (the caller falls back to Jacobi).
static bool sym_tridiag_qr(int n, std::vector<double>& A, std::vector<double>& Q, std::vector<double>& d) {
  auto a = [&](int i, int j) -> double& { return A[(size_t)i + (size_t)j * n]; };
  auto qq = [&](int i, int j) -> double& { return Q[(size_t)i + (size_t)j * n]; };
  Q.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) qq(i, i) = 1.0;
  std::vector<double> v(n), p(n), w(n);
  for (int k = 0; k + 2 < n; ++k) {
    // reflector H = I - beta v v^T with H x = alpha e_1, x = A[k+1:, k]
    double xn = 0.0;
    for (int i = k + 1; i < n; ++i) xn += a(i, k) * a(i, k);
    xn = std::sqrt(xn);
    if (xn == 0.0) continue;
    const double x0 = a(k + 1, k);
    const double alpha = x0 >= 0.0 ? -xn : xn;
    for (int i = k + 1; i < n; ++i) v[i] = a(i, k);
    v[k + 1] -= alpha;
    double vv = 0.0;
    for (int i = k + 1; i < n; ++i) vv += v[i] * v[i];
    if (vv == 0.0) continue;
    const double beta = 2.0 / vv;
    // trailing block: A <- H A H = A - v q^T - q v^T, p = beta A v, q = p - (beta v^T p / 2) v
    double vp = 0.0;
    for (int i = k + 1; i < n; ++i) {
      double t = 0.0;
      for (int j2 = k + 1; j2 < n; ++j2) t += a(i, j2) * v[j2];
      p[i] = beta * t;
      vp += v[i] * p[i];
    }
    const double kk = 0.5 * beta * vp;
    for (int i = k + 1; i < n; ++i) w[i] = p[i] - kk * v[i];
    for (int j2 = k + 1; j2 < n; ++j2)
      for (int i = k + 1; i < n; ++i) a(i, j2) -= v[i] * w[j2] + w[i] * v[j2];
    a(k + 1, k) = a(k, k + 1) = alpha;
    for (int i = k + 2; i < n; ++i) a(i, k) = a(k, i) = 0.0;
    // Q <- Q H
    for (int i = 0; i < n; ++i) {
      double t = 0.0;
      for (int j2 = k + 1; j2 < n; ++j2) t += qq(i, j2) * v[j2];
      t *= beta;
      for (int j2 = k + 1; j2 < n; ++j2) qq(i, j2) -= t * v[j2];
    }
  }
  d.assign(n, 0.0);
  std::vector<double> e(n > 1 ? n - 1 : 1, 0.0);
  for (int i = 0; i < n; ++i) d[i] = a(i, i);
  for (int i = 0; i + 1 < n; ++i) e[i] = a(i + 1, i);
  const double eps = 1e-16;
  int m = n - 1, iter = 0;
  while (m > 0) {
    if (std::fabs(e[m - 1]) <= eps * (std::fabs(d[m - 1]) + std::fabs(d[m]))) {
      e[m - 1] = 0.0;
      --m;
      continue;
    }
    int l = m - 1;
    while (l > 0 && std::fabs(e[l - 1]) > eps * (std::fabs(d[l - 1]) + std::fabs(d[l]))) --l;
    if (++iter > 60 * n) return false;
    // Wilkinson shift from the trailing 2 x 2 block of T[l..m]
    const double dd = 0.5 * (d[m - 1] - d[m]);
    const double em = e[m - 1];
    const double mu = d[m] - em * em / (dd + (dd >= 0.0 ? 1.0 : -1.0) * std::hypot(dd, em));
    double x = d[l] - mu, z = e[l], bulge = 0.0;
    for (int k = l; k < m; ++k) {
      const double r = std::hypot(x, z);
      const double c = r == 0.0 ? 1.0 : x / r, s2 = r == 0.0 ? 0.0 : z / r;
      if (k > l) e[k - 1] = r;                       // the bulge at (k-1, k+1) is annihilated
      const double dk = d[k], dk1 = d[k + 1], ek = e[k];
      d[k] = c * c * dk + 2.0 * c * s2 * ek + s2 * s2 * dk1;
      d[k + 1] = s2 * s2 * dk - 2.0 * c * s2 * ek + c * c * dk1;
      e[k] = c * s2 * (dk1 - dk) + (c * c - s2 * s2) * ek;
      if (k + 1 < m) {                               // new bulge at (k, k+2)
        bulge = s2 * e[k + 1];
        e[k + 1] *= c;
      }
      for (int i = 0; i < n; ++i) {                  // Q <- Q G^T on columns k, k+1
        const double qk = qq(i, k), qk1 = qq(i, k + 1);
        qq(i, k) = c * qk + s2 * qk1;
        qq(i, k + 1) = -s2 * qk + c * qk1;
      }
      x = e[k];
      z = bulge;
    }
  }
  return true;
}

void jacobi_eig(int n, const double* H, double* theta, double* V) {
  // fast path: Householder + implicit QR; cyclic Jacobi below only if QR does not converge
  {
    std::vector<double> Az((size_t)n * n), Qz, d;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) Az[(size_t)i + (size_t)j * n] = 0.5 * (H[i + j * n] + H[j + i * n]);
    if (n >= 2 && sym_tridiag_qr(n, Az, Qz, d)) {
      std::vector<int> idx(n);
      std::iota(idx.begin(), idx.end(), 0);
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] < d[b]; });
      for (int j = 0; j < n; ++j) {
        theta[j] = d[idx[j]];
        for (int i = 0; i < n; ++i) V[i + j * n] = Qz[(size_t)i + (size_t)idx[j] * n];
      }
      return;
    }
  }
  std::vector<double> A(n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) A[i + j * n] = 0.5 * (H[i + j * n] + H[j + i * n]);
  std::vector<double> Q(n * n, 0.0);
  for (int i = 0; i < n; ++i) Q[i + i * n] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        tot += A[i + j * n] * A[i + j * n];
        if (i != j) off += A[i + j * n] * A[i + j * n];
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p + q * n];
        if (apq == 0.0) continue;
        const double app = A[p + p * n], aqq = A[q + q * n];
        const double tau = (aqq - app) / (2.0 * apq);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
        // A <- J^T A J using the symmetry: columns p, q rotated (contiguous), rows mirrored,
        // the 2 x 2 block in closed form (a_pp - t a_pq, a_qq + t a_pq, 0)
        double* cp = &A[(size_t)p * n];
        double* cq = &A[(size_t)q * n];
        for (int k = 0; k < n; ++k) {
          if (k == p || k == q) continue;
          const double akp = cp[k], akq = cq[k];
          const double np_ = c * akp - s * akq, nq_ = s * akp + c * akq;
          cp[k] = np_;
          cq[k] = nq_;
          A[p + (size_t)k * n] = np_;
          A[q + (size_t)k * n] = nq_;
        }
        cp[p] = app - t * apq;
        cq[q] = aqq + t * apq;
        cp[q] = cq[p] = 0.0;
        for (int k = 0; k < n; ++k) {
          const double qkp = Q[k + p * n], qkq = Q[k + q * n];
          Q[k + p * n] = c * qkp - s * qkq;
          Q[k + q * n] = s * qkp + c * qkq;
        }
      }
    }
  }
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return A[a + a * n] < A[b + b * n]; });
  for (int j = 0; j < n; ++j) {
    theta[j] = A[idx[j] + idx[j] * n];
    for (int i = 0; i < n; ++i) V[i + j * n] = Q[i + idx[j] * n];
  }
}

static void jacobi_svd_plain(int k, const double* R, double* Ur, double* s, double* Vr);

// One-sided Jacobi SVD of a k x k matrix: R = Ur diag(s) Vr^T, s descending.
// k >= 24: preconditioned by Householder QR with column pivoting (R P = Q1 R1), the Jacobi
// sweeps then run on X = R1^T, whose columns are close to orthogonal (a few sweeps instead
// of many): X V = Ux S, so R = (Q1 V) S (P Ux)^T.
void jacobi_svd(int k, const double* R, double* Ur, double* s, double* Vr) {
  if (k < 24) { jacobi_svd_plain(k, R, Ur, s, Vr); return; }
  std::vector<double> A(R, R + (size_t)k * k);
  std::vector<int> perm(k);
  std::iota(perm.begin(), perm.end(), 0);
  std::vector<double> tau(k, 0.0);
  for (int j = 0; j < k; ++j) {
    // pivot: the remaining column of largest norm (recomputed: k is small)
    int pj = j;
    double best = -1.0;
    for (int c = j; c < k; ++c) {
      double t = 0.0;
      for (int i = j; i < k; ++i) t += A[i + (size_t)c * k] * A[i + (size_t)c * k];
      if (t > best) { best = t; pj = c; }
    }
    if (pj != j) {
      for (int i = 0; i < k; ++i) std::swap(A[i + (size_t)j * k], A[i + (size_t)pj * k]);
      std::swap(perm[j], perm[pj]);
    }
    // Householder reflector for A[j:, j]
    double nrm = 0.0;
    for (int i = j; i < k; ++i) nrm += A[i + (size_t)j * k] * A[i + (size_t)j * k];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) { tau[j] = 0.0; continue; }
    const double a0 = A[j + (size_t)j * k];
    const double beta = a0 >= 0 ? -nrm : nrm;
    const double v0 = a0 - beta;
    for (int i = j + 1; i < k; ++i) A[i + (size_t)j * k] /= v0;   // v = [1, A[j+1:, j]]
    tau[j] = (beta - a0) / beta;
    A[j + (size_t)j * k] = beta;
    for (int c = j + 1; c < k; ++c) {
      double w = A[j + (size_t)c * k];
      for (int i = j + 1; i < k; ++i) w += A[i + (size_t)j * k] * A[i + (size_t)c * k];
      w *= tau[j];
      A[j + (size_t)c * k] -= w;
      for (int i = j + 1; i < k; ++i) A[i + (size_t)c * k] -= w * A[i + (size_t)j * k];
    }
  }
  // Q1 (explicit) from the reflectors, R1 = upper triangle of A
  std::vector<double> Q((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) Q[i + (size_t)i * k] = 1.0;
  for (int j = k - 1; j >= 0; --j) {
    if (tau[j] == 0.0) continue;
    for (int c = 0; c < k; ++c) {
      double w = Q[j + (size_t)c * k];
      for (int i = j + 1; i < k; ++i) w += A[i + (size_t)j * k] * Q[i + (size_t)c * k];
      w *= tau[j];
      Q[j + (size_t)c * k] -= w;
      for (int i = j + 1; i < k; ++i) Q[i + (size_t)c * k] -= w * A[i + (size_t)j * k];
    }
  }
  // X = R1^T (lower triangular)
  std::vector<double> X((size_t)k * k, 0.0);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i <= j; ++i) X[j + (size_t)i * k] = A[i + (size_t)j * k];
  std::vector<double> Ux((size_t)k * k), sx(k), Vx((size_t)k * k);
  jacobi_svd_plain(k, X.data(), Ux.data(), sx.data(), Vx.data());   // X = Ux S Vx^T
  // left vectors of zero singular values are not defined by X V = U S: complete Ux to an
  // orthonormal basis (Gram-Schmidt of unit vectors against the kept columns, twice) so
  // that Vr = P Ux is orthogonal for rank-deficient R too
  {
    std::vector<int> good(k, 0);
    for (int j = 0; j < k; ++j) good[j] = sx[j] > 0.0;
    int cand = 0;
    for (int j = 0; j < k; ++j) {
      if (good[j]) continue;
      std::vector<double> u((size_t)k);
      for (; cand < k; ++cand) {
        for (int i = 0; i < k; ++i) u[i] = (i == cand) ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass)
          for (int c = 0; c < k; ++c) {
            if (!good[c]) continue;
            double t = 0.0;
            for (int i = 0; i < k; ++i) t += Ux[i + (size_t)c * k] * u[i];
            for (int i = 0; i < k; ++i) u[i] -= t * Ux[i + (size_t)c * k];
          }
        double nn = 0.0;
        for (int i = 0; i < k; ++i) nn += u[i] * u[i];
        if (nn > 0.25) {
          nn = std::sqrt(nn);
          for (int i = 0; i < k; ++i) Ux[i + (size_t)j * k] = u[i] / nn;
          good[j] = 1;
          ++cand;
          break;
        }
      }
    }
  }
  // R P = Q1 R1 = Q1 X^T = Q1 Vx S Ux^T  ->  Ur = Q1 Vx, Vr = P Ux
  for (int j = 0; j < k; ++j) {
    s[j] = sx[j];
    for (int i = 0; i < k; ++i) {
      double t = 0.0;
      for (int q = 0; q < k; ++q) t += Q[i + (size_t)q * k] * Vx[q + (size_t)j * k];
      Ur[i + (size_t)j * k] = t;
      Vr[perm[i] + (size_t)j * k] = Ux[i + (size_t)j * k];
    }
  }
}

static void jacobi_svd_plain(int k, const double* R, double* Ur, double* s, double* Vr) {
  std::vector<double> A(R, R + (size_t)k * k);
  std::vector<double> V((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) V[i + i * k] = 1.0;
  std::vector<double> cn(k);   // squared column norms, recomputed each sweep, updated per rotation
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int j = 0; j < k; ++j) {
      double t = 0.0;
      for (int i = 0; i < k; ++i) t += A[i + j * k] * A[i + j * k];
      cn[j] = t;
    }
    for (int p = 0; p < k - 1; ++p) {
      for (int q = p + 1; q < k; ++q) {
        const double alpha = cn[p], beta = cn[q];
        double gamma = 0;
        const double* ap_ = &A[(size_t)p * k];
        const double* aq_ = &A[(size_t)q * k];
        for (int i = 0; i < k; ++i) gamma += ap_[i] * aq_[i];
        if (gamma == 0.0 || std::fabs(gamma) <= 1e-15 * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (int i = 0; i < k; ++i) {
          const double ap = A[i + p * k], aq = A[i + q * k];
          A[i + p * k] = c * ap - sn * aq;
          A[i + q * k] = sn * ap + c * aq;
          const double vp = V[i + p * k], vq = V[i + q * k];
          V[i + p * k] = c * vp - sn * vq;
          V[i + q * k] = sn * vp + c * vq;
        }
        cn[p] = alpha - t * gamma;   // the rotation moves t gamma between the two norms
        cn[q] = beta + t * gamma;
      }
    }
    if (!rotated) break;
  }
  std::vector<double> nrm(k);
  for (int j = 0; j < k; ++j) {
    double t = 0;
    for (int i = 0; i < k; ++i) t += A[i + j * k] * A[i + j * k];
    nrm[j] = std::sqrt(t);
  }
  std::vector<int> idx(k);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return nrm[a] > nrm[b]; });
  for (int j = 0; j < k; ++j) {
    const int src = idx[j];
    s[j] = nrm[src];
    for (int i = 0; i < k; ++i) {
      Ur[i + j * k] = nrm[src] > 0 ? A[i + src * k] / nrm[src] : (i == j ? 1.0 : 0.0);
      Vr[i + j * k] = V[i + src * k];
    }
  }
}

}  // namespace rsk

using namespace rsk;

namespace {
// X <- X R^-1 for upper-triangular R (X is rows x nc, column-major, ld rows)
void right_trsm_upper(int rows, int nc, const double* R, double* X) {
  for (int j = 0; j < nc; ++j) {
    for (int q = 0; q < j; ++q) {
      const double rq = R[q + j * nc];
      if (rq == 0.0) continue;
      for (int i = 0; i < rows; ++i) X[i + j * rows] -= X[i + q * rows] * rq;
    }
    const double d = R[j + j * nc];
    for (int i = 0; i < rows; ++i) X[i + j * rows] /= d;
  }
}
// x <- R^-T x (forward substitution with R^T lower)
void trsv_upper_t(int nc, const double* R, double* x) {
  for (int i = 0; i < nc; ++i) {
    double t = x[i];
    for (int q = 0; q < i; ++q) t -= R[q + i * nc] * x[q];
    x[i] = t / R[i + i * nc];
  }
}
}  // namespace

extern "C" rsk_status rsk_orth_guess(int nc, const double* R_h, const double* KtZE_h,
                                     const double* ZEtZE_h, const double* ZEtb_h,
                                     const double* Ktb_h, double gamma_star, int m,
                                     const double* gamma_h, double* C_h, int* status_h) {
  if (nc <= 0 || m < 0 || !R_h || !KtZE_h || !ZEtZE_h || !ZEtb_h || !Ktb_h ||
      (m > 0 && (!gamma_h || !C_h || !status_h)))
    return RSK_EINVAL;
  for (int i = 0; i < nc; ++i)
    if (!(R_h[i + i * nc] != 0.0)) return RSK_EINVAL;
  // P = KtZE R^-1
  std::vector<double> P_(KtZE_h, KtZE_h + (size_t)nc * nc);
  right_trsm_upper(nc, nc, R_h, P_.data());
  // Q2 = R^-T (ZEtZE R^-1): right solve, then transpose-left solve column by column
  std::vector<double> T(ZEtZE_h, ZEtZE_h + (size_t)nc * nc);
  right_trsm_upper(nc, nc, R_h, T.data());
  for (int j = 0; j < nc; ++j) trsv_upper_t(nc, R_h, &T[(size_t)j * nc]);
  std::vector<double> Q2_((size_t)nc * nc);
  for (int j = 0; j < nc; ++j)
    for (int i = 0; i < nc; ++i) Q2_[i + j * nc] = 0.5 * (T[i + j * nc] + T[j + i * nc]);
  std::vector<double> u_(ZEtb_h, ZEtb_h + nc);
  trsv_upper_t(nc, R_h, u_.data());
  const double* P_h = P_.data();
  const double* Q2_h = Q2_.data();
  const double* u_h = u_.data();
  const double* v_h = Ktb_h;
  std::vector<double> G((size_t)nc * nc), q(nc);
  for (int l = 0; l < m; ++l) {
    const double d = gamma_h[l] - gamma_star;
    for (int j = 0; j < nc; ++j)
      for (int i = 0; i < nc; ++i)
        G[i + j * nc] = (i == j ? 1.0 : 0.0) + d * (P_h[i + j * nc] + P_h[j + i * nc]) +
                        d * d * 0.5 * (Q2_h[i + j * nc] + Q2_h[j + i * nc]);
    double* c = C_h + (size_t)l * nc;
    if (!chol_lower(nc, G.data())) {
      status_h[l] = RSK_NOT_SPD;
      for (int i = 0; i < nc; ++i) c[i] = 0.0;
      continue;
    }
    for (int i = 0; i < nc; ++i) q[i] = v_h[i] + d * u_h[i];
    chol_solve_lower(nc, G.data(), q.data());
    // c = R^-1 q (upper triangular back substitution)
    for (int i = nc - 1; i >= 0; --i) {
      double t = q[i];
      for (int j = i + 1; j < nc; ++j) t -= R_h[i + j * nc] * c[j];
      c[i] = t / R_h[i + i * nc];
    }
    status_h[l] = 0;
  }
  return RSK_OK;
}

// Gaussian elimination with partial pivoting on a column-major n x n A (overwritten),
// solving A q = b in place; false when a pivot is exactly zero or not finite.
static bool lu_solve(int n, double* A, double* b) {
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = std::fabs(A[k + (size_t)k * n]);
    for (int i = k + 1; i < n; ++i) {
      const double v = std::fabs(A[i + (size_t)k * n]);
      if (v > best) { best = v; piv = i; }
    }
    if (!(best > 0.0) || !std::isfinite(best)) return false;
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(A[k + (size_t)j * n], A[piv + (size_t)j * n]);
      std::swap(b[k], b[piv]);
    }
    const double akk = A[k + (size_t)k * n];
    for (int i = k + 1; i < n; ++i) {
      const double f = A[i + (size_t)k * n] / akk;
      A[i + (size_t)k * n] = f;
      for (int j = k + 1; j < n; ++j) A[i + (size_t)j * n] -= f * A[k + (size_t)j * n];
      b[i] -= f * b[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double t = b[i];
    for (int j = i + 1; j < n; ++j) t -= A[i + (size_t)j * n] * b[j];
    b[i] = t / A[i + (size_t)i * n];
  }
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(b[i])) return false;
  return true;
}

extern "C" rsk_status rsk_oblique_guess(int nc, const double* R_h, const double* KtZE_h, const double* Ktb_h,
                                        double gamma_anchor, int m, const double* gamma_h, double* C_h,
                                        int* status_h) {
  if (nc <= 0 || m < 0 || !R_h || !KtZE_h || !Ktb_h || (m > 0 && (!gamma_h || !C_h || !status_h)) ||
      !std::isfinite(gamma_anchor))
    return RSK_EINVAL;
  for (int i = 0; i < nc; ++i)
    if (!(R_h[i + i * nc] != 0.0)) return RSK_EINVAL;
  std::vector<double> P_(KtZE_h, KtZE_h + (size_t)nc * nc);   // K^T E U = KtZE R^-1
  right_trsm_upper(nc, nc, R_h, P_.data());
  std::vector<double> G((size_t)nc * nc), q(nc);
  for (int l = 0; l < m; ++l) {
    const double d = gamma_h[l] - gamma_anchor;
    for (int j = 0; j < nc; ++j)
      for (int i = 0; i < nc; ++i) G[i + (size_t)j * nc] = (i == j ? 1.0 : 0.0) + d * P_[i + (size_t)j * nc];
    for (int i = 0; i < nc; ++i) q[i] = Ktb_h[i];
    double* c = C_h + (size_t)l * nc;
    if (!lu_solve(nc, G.data(), q.data())) {
      status_h[l] = RSK_SINGULAR;
      for (int i = 0; i < nc; ++i) c[i] = 0.0;
      continue;
    }
    for (int i = nc - 1; i >= 0; --i) {   // c = R^-1 q
      double t = q[i];
      for (int j = i + 1; j < nc; ++j) t -= R_h[i + (size_t)j * nc] * c[j];
      c[i] = t / R_h[i + (size_t)i * nc];
    }
    status_h[l] = 0;
  }
  return RSK_OK;
}

extern "C" rsk_status rsk_pencil_ritz(int nc, const double* Ahat_h, const double* Ehat_h, double gamma,
                                      int J, double* Wt_h, double* theta_h) {
  if (nc <= 0 || J < 0 || J > nc || !Ahat_h || !Ehat_h || (J > 0 && (!Wt_h || !theta_h)) ||
      !std::isfinite(gamma))
    return RSK_EINVAL;
  std::vector<double> H((size_t)nc * nc), th(nc), V((size_t)nc * nc);
  for (int j = 0; j < nc; ++j)
    for (int i = 0; i < nc; ++i)
      H[i + j * nc] = 0.5 * (Ahat_h[i + j * nc] + Ahat_h[j + i * nc]) +
                      gamma * 0.5 * (Ehat_h[i + j * nc] + Ehat_h[j + i * nc]);
  jacobi_eig(nc, H.data(), th.data(), V.data());
  for (int j = 0; j < J; ++j) {
    theta_h[j] = th[j];
    for (int i = 0; i < nc; ++i) Wt_h[i + j * nc] = V[i + j * nc];
  }
  return RSK_OK;
}

extern "C" rsk_status rsk_stabilize_small(int k, const double* R_h, const double* colnorm2_h,
                                          double condcap, int cap, double* Zs_h, int* nkeep) {
  if (k <= 0 || !R_h || !colnorm2_h || !Zs_h || !nkeep || !(condcap > 1.0)) return RSK_EINVAL;
  std::vector<double> Rs((size_t)k * k), Ur((size_t)k * k), s(k), Vr((size_t)k * k);
  for (int j = 0; j < k; ++j) {
    if (!(colnorm2_h[j] > 0.0)) return RSK_EINVAL;
    const double sc = 1.0 / std::sqrt(colnorm2_h[j]);
    for (int i = 0; i < k; ++i) Rs[i + j * k] = R_h[i + j * k] * sc;
  }
  jacobi_svd(k, Rs.data(), Ur.data(), s.data(), Vr.data());
  int nk = 0;
  for (int i = 0; i < k; ++i)
    if (s[i] > 0.0 && s[0] / s[i] < condcap) nk = i + 1; else break;
  if (cap > 0 && nk > cap) nk = cap;
  for (int j = 0; j < nk; ++j)
    for (int i = 0; i < k; ++i) Zs_h[i + j * k] = Ur[i + j * k];
  *nkeep = nk;
  return RSK_OK;
}

extern "C" rsk_status rsk_carried_select(int m, const double* g2, const double* gh2, double thr,
                                         double* scale_h, int* keep_h) {
  if (m < 0 || (m > 0 && (!g2 || !gh2 || !scale_h || !keep_h))) return RSK_EINVAL;
  for (int l = 0; l < m; ++l) {
    const bool keep = g2[l] > 0.0 && gh2[l] > 0.0 && std::sqrt(gh2[l] / g2[l]) >= thr;
    keep_h[l] = keep ? 1 : 0;
    scale_h[l] = keep ? 1.0 / std::sqrt(gh2[l]) : 0.0;
  }
  return RSK_OK;
}

extern "C" rsk_status rsk_sym_eig(int n, const double* H_h, double* theta_h, double* V_h) {
  if (n <= 0 || !H_h || !theta_h || !V_h) return RSK_EINVAL;
  jacobi_eig(n, H_h, theta_h, V_h);
  return RSK_OK;
}

extern "C" rsk_status rsk_svd_small(int k, const double* R_h, double* Ur_h, double* s_h, double* Vr_h) {
  if (k <= 0 || !R_h || !Ur_h || !s_h || !Vr_h) return RSK_EINVAL;
  jacobi_svd(k, R_h, Ur_h, s_h, Vr_h);
  return RSK_OK;
}

extern "C" rsk_status rsk_chol_solve_small(int n, const double* G_h, int nrhs, const double* Z_h,
                                           double* X_h) {
  if (n <= 0 || nrhs < 0 || !G_h || !Z_h || !X_h) return RSK_EINVAL;
  std::vector<double> L((size_t)n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) L[i + j * n] = 0.5 * (G_h[i + j * n] + G_h[j + i * n]);
  if (!chol_lower(n, L.data())) return RSK_EPARTIAL;
  for (int c = 0; c < nrhs; ++c) {
    std::memcpy(X_h + (size_t)c * n, Z_h + (size_t)c * n, sizeof(double) * n);
    chol_solve_lower(n, L.data(), X_h + (size_t)c * n);
  }
  return RSK_OK;
}

extern "C" rsk_status rsk_lcurve_corner(int M, const double* rho_h, const double* eta_h, int* lstar,
                                        double* kappa_h) {
  if (M <= 0 || !rho_h || !eta_h || !lstar) return RSK_EINVAL;
  std::vector<double> kap(M, -INFINITY);
  for (int l = 1; l + 1 < M; ++l) {
    const double a0 = std::log(rho_h[l - 1]), a1 = std::log(rho_h[l]), a2 = std::log(rho_h[l + 1]);
    const double b0 = std::log(eta_h[l - 1]), b1 = std::log(eta_h[l]), b2 = std::log(eta_h[l + 1]);
    const double r1 = 0.5 * (a2 - a0), e1 = 0.5 * (b2 - b0);
    const double r2 = a2 - 2.0 * a1 + a0, e2 = b2 - 2.0 * b1 + b0;
    const double den = std::pow(r1 * r1 + e1 * e1, 1.5);
    kap[l] = den > 0 ? (r1 * e2 - r2 * e1) / den : -INFINITY;
  }
  int best = 0;
  if (M >= 3) {
    best = 1;
    for (int l = 2; l + 1 < M; ++l)
      if (kap[l] > kap[best]) best = l;
  }
  *lstar = best;
  if (kappa_h)
    for (int l = 0; l < M; ++l) kappa_h[l] = kap[l];
  return RSK_OK;
}

// ---------------------------------------------------------------- deflated-CG host steps
// Local Gram matrices G_l = sym(U_l^T Z_l), U_l = [W_g(l), ghat_l], Z_l = A_gamma U_l, from
// their reduced pieces, and their Cholesky factors with the drop rule of O4 (first the
// carried column, then all of U). Layout: WA/WE [g][16*16] (J_g x J_g, ld J_g),
// WZg/AWg/EWg [g][16*ns] (J_g x ns, ld J_g), L [ns][RSK_MAX_LOCAL^2] (ld RSK_MAX_LOCAL).
extern "C" rsk_status rsk_local_gram_factors(int ns, int ngroups, const int* J_h, const int* group_of_shift_h,
                                             const double* gamma_h, const double* WA_h, const double* WE_h,
                                             const double* WZg_h, const double* AWg_h, const double* EWg_h,
                                             const double* gzg_h, double* L_h, int* m_h, int* hasg_h,
                                             int* dropped_h) {
  using rsk::kMaxM;
  if (ns < 0 || ngroups < 1 || ngroups > RSK_MAX_GROUPS || !J_h || !group_of_shift_h || !gamma_h || !WA_h ||
      !WE_h || !L_h || !m_h || !hasg_h || !dropped_h)
    return RSK_EINVAL;
  std::vector<double> Gm(kMaxM * kMaxM);
  for (int s = 0; s < ns; ++s) {
    const int g = group_of_shift_h[s];
    if (g < 0 || g >= ngroups) return RSK_EINVAL;
    const int J = J_h[g];
    if (J < 0 || J > 16) return RSK_EINVAL;
    if (hasg_h[s] && (!WZg_h || !AWg_h || !EWg_h || !gzg_h)) return RSK_EINVAL;
    const double gm = gamma_h[s];
    int nwk = J, hg = hasg_h[s] ? 1 : 0;
    int m = nwk + hg;
    dropped_h[s] = 0;
    for (;;) {
      if (m == 0) break;
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
          double v;
          if (i < nwk && j < nwk) {
            const double a = WA_h[g * 256 + i + j * J] + gm * WE_h[g * 256 + i + j * J];
            const double b = WA_h[g * 256 + j + i * J] + gm * WE_h[g * 256 + j + i * J];
            v = 0.5 * (a + b);
          } else if (i < nwk && j == nwk) {   // W_i^T Zg  and  ghat^T Z_i
            const double a = WZg_h[(size_t)g * 16 * ns + i + (size_t)s * J];
            const double b = AWg_h[(size_t)g * 16 * ns + i + (size_t)s * J] + gm * EWg_h[(size_t)g * 16 * ns + i + (size_t)s * J];
            v = 0.5 * (a + b);
          } else if (i == nwk && j < nwk) {
            const double a = WZg_h[(size_t)g * 16 * ns + j + (size_t)s * J];
            const double b = AWg_h[(size_t)g * 16 * ns + j + (size_t)s * J] + gm * EWg_h[(size_t)g * 16 * ns + j + (size_t)s * J];
            v = 0.5 * (a + b);
          } else {
            v = gzg_h[s];
          }
          Gm[i + j * m] = v;
        }
      if (rsk::chol_lower(m, Gm.data())) break;
      dropped_h[s] = 1;
      if (hg) { hg = 0; m = nwk; } else { nwk = 0; m = 0; }
    }
    for (int e = 0; e < kMaxM * kMaxM; ++e) L_h[(size_t)s * kMaxM * kMaxM + e] = 0.0;
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) L_h[(size_t)s * kMaxM * kMaxM + i + j * kMaxM] = Gm[i + j * m];
    m_h[s] = m;
    hasg_h[s] = hg;
  }
  return RSK_OK;
}

// mu_s = G_s^-1 [zA_s + gamma_s zE_s ; zG_s] with the factors of rsk_local_gram_factors
// (zE / zG nullable = 0). Forward then backward substitution, same order as the device loop.
extern "C" rsk_status rsk_gram_solve(int ns, int J, const double* L_h, const int* m_h, const int* hasg_h,
                                     const double* gamma_h, const double* zA_h, const double* zE_h,
                                     const double* zG_h, double* mu_h) {
  using rsk::kMaxM;
  if (ns < 0 || J < 0 || J > 16 || !L_h || !m_h || !hasg_h || !gamma_h || !mu_h || (J > 0 && !zA_h))
    return RSK_EINVAL;
  for (int s = 0; s < ns; ++s) {
    double* mu = mu_h + (size_t)s * kMaxM;
    for (int j = 0; j < kMaxM; ++j) mu[j] = 0.0;
    const int m = m_h[s], hg = hasg_h[s], nw = m - hg;
    if (m < 0 || m > kMaxM || nw > J) return RSK_EINVAL;
    for (int j = 0; j < nw; ++j)
      mu[j] = zE_h ? zA_h[j + (size_t)s * J] + gamma_h[s] * zE_h[j + (size_t)s * J] : zA_h[j + (size_t)s * J];
    if (hg) mu[nw] = zG_h ? zG_h[s] : 0.0;
    const double* L = L_h + (size_t)s * kMaxM * kMaxM;
    for (int i = 0; i < m; ++i) {
      double t = mu[i];
      for (int j = 0; j < i; ++j) t -= L[i + j * kMaxM] * mu[j];
      mu[i] = t / L[i + i * kMaxM];
    }
    for (int i = m - 1; i >= 0; --i) {
      double t = mu[i];
      for (int j = i + 1; j < m; ++j) t -= L[j + i * kMaxM] * mu[j];
      mu[i] = t / L[i + i * kMaxM];
    }
  }
  return RSK_OK;
}

// alpha = rho / (p.w) for the shifts in state RSK_LOOP_ACTIVE (O4 step 3); p.w <= 0 or
// non-finite -> RSK_LOOP_BREAKDOWN with alpha = 0.
extern "C" rsk_status rsk_cg_alpha(int ns, const double* rho_h, const double* pw_h, double* alpha_h, int* state_h) {
  if (ns < 0 || !rho_h || !pw_h || !alpha_h || !state_h) return RSK_EINVAL;
  for (int s = 0; s < ns; ++s) {
    alpha_h[s] = 0.0;
    if (state_h[s] != RSK_LOOP_ACTIVE) continue;
    const double pi = pw_h[s];
    if (!(pi > 0.0) || !std::isfinite(pi)) state_h[s] = RSK_LOOP_BREAKDOWN;
    else alpha_h[s] = rho_h[s] / pi;
  }
  return RSK_OK;
}

// The scalar half of a deflated-CG iteration (O4 steps 3-4) from the reduced sums of the
// updated residual: rho' = r.r and z = [AW^T r + gamma EW^T r ; ZGhat^T r]. mode_h[s] is the
// state at the start of the iteration (RSK_LOOP_ACTIVE: loop step; RSK_LOOP_RCONV: r was
// the true residual b - A_gamma x). Writes beta, mu = G^-1 z (Cholesky factor L from
// rsk_local_gram_factors; ld RSK_MAX_LOCAL per shift) and the new state.
extern "C" rsk_status rsk_cg_scalars(int ns, int J, const int* mode_h, const double* gamma_h,
                                     const double* rho_new_h, const double* zA_h, const double* zE_h,
                                     const double* zG_h, const int* m_h, const int* hasg_h, const double* L_h,
                                     double thr, int maxit, double* rho_h, double* beta_h, double* mu_h,
                                     int* iters_h, double* rho_true_h, int* nconf_h, int* state_h) {
  using rsk::kMaxM;
  if (ns < 0 || J < 0 || J > 16 || !mode_h || !gamma_h || !rho_new_h || !m_h || !hasg_h || !L_h || !rho_h ||
      !beta_h || !mu_h || !iters_h || !rho_true_h || !nconf_h || !state_h)
    return RSK_EINVAL;
  for (int s = 0; s < ns; ++s) {
    const int mode = mode_h[s];
    if (mode != RSK_LOOP_ACTIVE && mode != RSK_LOOP_RCONV) continue;
    if (state_h[s] != mode) continue;   // BREAKDOWN in this iteration
    const double rn = rho_new_h[s];
    const bool conv = std::sqrt(rn) <= thr;
    bool newp = false;
    beta_h[s] = 0.0;
    if (mode == RSK_LOOP_ACTIVE) {
      iters_h[s] += 1;
      beta_h[s] = rn / rho_h[s];
      rho_h[s] = rn;
      if (conv) state_h[s] = RSK_LOOP_RCONV;
      else if (iters_h[s] >= maxit) state_h[s] = RSK_LOOP_MAXIT;
      else newp = true;
    } else {
      rho_true_h[s] = rn;
      nconf_h[s] += 1;
      if (conv) state_h[s] = RSK_LOOP_DONE;
      else if (iters_h[s] >= maxit) state_h[s] = RSK_LOOP_MAXIT;
      else { state_h[s] = RSK_LOOP_ACTIVE; rho_h[s] = rn; newp = true; }
    }
    double* mu = mu_h + (size_t)s * kMaxM;
    for (int j = 0; j < kMaxM; ++j) mu[j] = 0.0;
    if (newp) {
      rsk_status e = rsk_gram_solve(1, J, L_h + (size_t)s * kMaxM * kMaxM, m_h + s, hasg_h + s, gamma_h + s,
                                    zA_h + (size_t)s * J, zE_h ? zE_h + (size_t)s * J : nullptr,
                                    zG_h ? zG_h + s : nullptr, mu);
      if (e != RSK_OK) return e;
    }
  }
  return RSK_OK;
}
