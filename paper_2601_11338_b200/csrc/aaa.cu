// aaa.cu — host: the poles of Alg. 1 line 3 by the AAA algorithm.
//
// "Approximate the spectral radius ρ(𝔏) of 𝔏, and build the poles {ξ_j} of rational approximation of
// exp(−x) on the interval [0, t* ρ(𝔏)]. Use AAA" (alg:trace_estimation line 3).
// AAA (Nakatsukasa, Sète, Trefethen, SISC 2018): r(z) = N(z)/D(z), N = Σ_j w_j f_j/(z − z_j),
// D = Σ_j w_j/(z − z_j); each step adds the sample with the largest error |F − R| as a support point
// and takes w as the right singular vector of the smallest singular value of the Loewner matrix
// L_ik = (F_i − f_k)/(Z_i − z_k) over the remaining samples, until max|F − R| <= tol max|F|.
// Host implementation (m <= 30 support points, 2001 samples):
//   * smallest right singular vector: Householder QR of L, then one-sided Jacobi SVD of R
//     (Golub & Van Loan §8.6.3) — no squaring of the condition number;
//   * poles = roots of D: with y_j = z_j − σ, they are the eigenvalues of the diagonal-plus-rank-one
//     matrix diag(y) − u 1ᵀ, u_j = w_j y_j / Σw (plus one spurious eigenvalue at y = 0), by Householder
//     Hessenberg reduction and the Francis QR of eig.cu, then polished by Newton's method on D;
//   * Froissart doublets |Res r| = |N(ξ)/D'(ξ)| < 1e-13 max|F| and poles on [0, X] of the real axis
//     are dropped; each conjugate pair is returned once (Im ξ > 0).
// The same readings as oracle/aaa.py (R18): samples {0} ∪ X·10^linspace(−10, 0, 2000).
#include "wl_internal.cuh"

#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

namespace wl {
namespace {

using cd = std::complex<double>;

// right singular vector of the smallest singular value of the row-major r x m matrix L (r >= m)
std::vector<double> min_right_singular(std::vector<double> L, int r, int m) {
  // Householder QR: R = upper m x m of Qᵀ L
  for (int k = 0; k < m; ++k) {
    double nrm = 0.0;
    for (int i = k; i < r; ++i) nrm += L[(size_t)i * m + k] * L[(size_t)i * m + k];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = L[(size_t)k * m + k] > 0 ? -nrm : nrm;
    std::vector<double> v(r - k);
    for (int i = k; i < r; ++i) v[i - k] = L[(size_t)i * m + k];
    v[0] -= alpha;
    double vv = 0.0;
    for (double x : v) vv += x * x;
    if (vv == 0.0) continue;
    for (int j = k; j < m; ++j) {
      double s = 0.0;
      for (int i = k; i < r; ++i) s += v[i - k] * L[(size_t)i * m + j];
      s = 2.0 * s / vv;
      for (int i = k; i < r; ++i) L[(size_t)i * m + j] -= s * v[i - k];
    }
  }
  std::vector<double> R((size_t)m * m, 0.0), V((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = i; j < m; ++j) R[(size_t)i * m + j] = L[(size_t)i * m + j];
  for (int i = 0; i < m; ++i) V[(size_t)i * m + i] = 1.0;
  // one-sided Jacobi on the columns of R: R V has orthogonal columns, their norms are the singular values
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = 0; i < m; ++i) {
          a += R[(size_t)i * m + p] * R[(size_t)i * m + p];
          b += R[(size_t)i * m + q] * R[(size_t)i * m + q];
          g += R[(size_t)i * m + p] * R[(size_t)i * m + q];
        }
        if (std::abs(g) <= 1e-300 || std::abs(g) <= 1e-16 * std::sqrt(a * b)) continue;
        off = std::max(off, std::abs(g) / std::sqrt(a * b));
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < m; ++i) {
          const double rp = R[(size_t)i * m + p], rq = R[(size_t)i * m + q];
          R[(size_t)i * m + p] = c * rp - s * rq;
          R[(size_t)i * m + q] = s * rp + c * rq;
          const double vp = V[(size_t)i * m + p], vq = V[(size_t)i * m + q];
          V[(size_t)i * m + p] = c * vp - s * vq;
          V[(size_t)i * m + q] = s * vp + c * vq;
        }
      }
    if (off <= 1e-15) break;
  }
  int best = 0;
  double bn = INFINITY;
  for (int j = 0; j < m; ++j) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += R[(size_t)i * m + j] * R[(size_t)i * m + j];
    if (s < bn) { bn = s; best = j; }
  }
  std::vector<double> w(m);
  for (int i = 0; i < m; ++i) w[i] = V[(size_t)i * m + best];
  return w;
}

// eigenvalues of a general real m x m matrix (row-major): balancing (Parlett & Reinsch: a diagonal
// similarity by powers of 2 equalising row and column norms — the diagonal-plus-rank-one matrix below has
// rows of very different scale), Householder Hessenberg reduction, then the Francis QR of eig.cu
bool eigvals_general(std::vector<double> A, int m, std::vector<cd>& ev) {
  for (bool done = false; !done;) {
    done = true;
    for (int i = 0; i < m; ++i) {
      double c = 0.0, r = 0.0;
      for (int j = 0; j < m; ++j)
        if (j != i) {
          c += std::fabs(A[(size_t)j * m + i]);
          r += std::fabs(A[(size_t)i * m + j]);
        }
      if (c == 0.0 || r == 0.0) continue;
      double f = 1.0;
      const double sum = c + r;
      while (c < r / 2.0) { c *= 2.0; r /= 2.0; f *= 2.0; }
      while (c >= r * 2.0) { c /= 2.0; r *= 2.0; f /= 2.0; }
      if ((c + r) < 0.95 * sum) {
        done = false;
        for (int j = 0; j < m; ++j) A[(size_t)i * m + j] /= f;
        for (int j = 0; j < m; ++j) A[(size_t)j * m + i] *= f;
      }
    }
  }
  for (int k = 0; k + 2 < m; ++k) {
    double nrm = 0.0;
    for (int i = k + 1; i < m; ++i) nrm += A[(size_t)i * m + k] * A[(size_t)i * m + k];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = A[(size_t)(k + 1) * m + k] > 0 ? -nrm : nrm;
    std::vector<double> v(m, 0.0);
    for (int i = k + 1; i < m; ++i) v[i] = A[(size_t)i * m + k];
    v[k + 1] -= alpha;
    double vv = 0.0;
    for (double x : v) vv += x * x;
    if (vv == 0.0) continue;
    for (int j = 0; j < m; ++j) {  // A <- (I - 2vvᵀ/vv) A
      double s = 0.0;
      for (int i = k + 1; i < m; ++i) s += v[i] * A[(size_t)i * m + j];
      s = 2.0 * s / vv;
      for (int i = k + 1; i < m; ++i) A[(size_t)i * m + j] -= s * v[i];
    }
    for (int i = 0; i < m; ++i) {  // A <- A (I - 2vvᵀ/vv)
      double s = 0.0;
      for (int j = k + 1; j < m; ++j) s += A[(size_t)i * m + j] * v[j];
      s = 2.0 * s / vv;
      for (int j = k + 1; j < m; ++j) A[(size_t)i * m + j] -= s * v[j];
    }
  }
  std::vector<double> wr, wi;
  if (!hessenberg_eigvals(A, m, wr, wi)) return false;
  ev.resize(m);
  for (int i = 0; i < m; ++i) ev[i] = cd(wr[i], wi[i]);
  return true;
}

}  // namespace

// AAA poles of exp(−x) on [0, xmax] (see the file comment); representatives of conjugate pairs
bool aaa_exp_poles(double xmax, double tol, std::vector<cd>& poles) {
  const int NS = 2001, mmax = 30;
  std::vector<double> Z(NS), F(NS);
  Z[0] = 0.0;
  for (int i = 1; i < NS; ++i) Z[i] = xmax * std::pow(10.0, -10.0 + 10.0 * (double)(i - 1) / (NS - 2));
  double fmax = 0.0;
  for (int i = 0; i < NS; ++i) {
    F[i] = std::exp(-Z[i]);
    fmax = std::max(fmax, std::abs(F[i]));
  }
  std::vector<char> sup(NS, 0);
  std::vector<double> z, f, w, R(NS);
  double mean = 0.0;
  for (double x : F) mean += x;
  mean /= NS;
  std::fill(R.begin(), R.end(), mean);
  for (int it = 0; it < mmax; ++it) {
    int j = 0;
    double emax = -1.0;
    for (int i = 0; i < NS; ++i)
      if (std::abs(F[i] - R[i]) > emax) { emax = std::abs(F[i] - R[i]); j = i; }
    z.push_back(Z[j]);
    f.push_back(F[j]);
    sup[j] = 1;
    const int m = (int)z.size();
    std::vector<int> rows;
    for (int i = 0; i < NS; ++i)
      if (!sup[i]) rows.push_back(i);
    std::vector<double> L((size_t)rows.size() * m);
    for (size_t r = 0; r < rows.size(); ++r)
      for (int k = 0; k < m; ++k) L[r * m + k] = (F[rows[r]] - f[k]) / (Z[rows[r]] - z[k]);
    w = min_right_singular(L, (int)rows.size(), m);
    double err = 0.0;
    for (int i = 0; i < NS; ++i) {
      if (sup[i]) { R[i] = F[i]; continue; }
      double num = 0.0, den = 0.0;
      for (int k = 0; k < m; ++k) {
        const double c = 1.0 / (Z[i] - z[k]);
        num += c * w[k] * f[k];
        den += c * w[k];
      }
      R[i] = num / den;
      err = std::max(err, std::abs(F[i] - R[i]));
    }
    if (err <= tol * fmax) break;
  }
  const int m = (int)z.size();
  poles.clear();
  if (m < 2) return true;
  // roots of D(λ) = Σ w_j/(λ − z_j): eigenvalues of diag(y) − u 1ᵀ (y = z − σ), minus the one at y = 0
  double W = 0.0;
  for (double x : w) W += x;
  if (W == 0.0) return false;
  // Σ w tiny makes the matrix badly scaled and the QR may stall: retry with other shifts σ (< 0 <= z_j)
  std::vector<cd> ev;
  double sigma = 0.0;
  bool ok = false;
  for (double sg : {-1.0, -2.71828, -0.367879, -7.38906, -0.135335, -20.0855}) {
    sigma = sg;
    std::vector<double> G((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int k = 0; k < m; ++k) G[(size_t)i * m + k] = (i == k ? z[i] - sigma : 0.0) - w[i] * (z[i] - sigma) / W;
    if ((ok = eigvals_general(G, m, ev))) break;
  }
  if (!ok) return false;
  int spurious = 0;
  for (int i = 1; i < m; ++i)
    if (std::abs(ev[i]) < std::abs(ev[spurious])) spurious = i;
  auto Dfun = [&](cd l, cd& d, cd& dp, cd& nn) {
    d = dp = nn = 0.0;
    for (int k = 0; k < m; ++k) {
      const cd c = 1.0 / (l - z[k]);
      d += w[k] * c;
      dp -= w[k] * c * c;
      nn += w[k] * f[k] * c;
    }
  };
  for (int i = 0; i < m; ++i) {
    if (i == spurious) continue;
    cd l = ev[i] + sigma;
    for (int nt = 0; nt < 6; ++nt) {  // Newton on D
      cd d, dp, nn;
      Dfun(l, d, dp, nn);
      if (std::abs(dp) == 0.0) break;
      const cd step = d / dp;
      l -= step;
      if (std::abs(step) <= 1e-15 * std::max(1.0, std::abs(l))) break;
    }
    cd d, dp, nn;
    Dfun(l, d, dp, nn);
    const double res = std::abs(nn / dp);
    if (!(res >= 1e-13 * fmax)) continue;  // Froissart doublet
    const bool real = std::abs(l.imag()) <= 1e-10 * std::max(1.0, std::abs(l));
    if (real) {
      if (l.real() >= 0.0 && l.real() <= xmax) continue;  // on the spectral interval
      poles.push_back(cd(l.real(), 0.0));
    } else if (l.imag() > 0.0) {
      poles.push_back(l);
    }
  }
  std::sort(poles.begin(), poles.end(), [](const cd& a, const cd& b) {
    return std::abs(a.imag()) != std::abs(b.imag()) ? std::abs(a.imag()) < std::abs(b.imag()) : a.real() < b.real();
  });
  return true;
}

}  // namespace wl

extern "C" wl_status wl_aaa_exp_poles(double xmax, double tol, int32_t cap, double* re, double* im, int32_t* npoles) {
  return wl::guarded([&] {
    if (!(xmax > 0.0) || !(tol > 0.0) || cap < 0 || !npoles || (cap > 0 && (!re || !im)))
      throw wl::Error(WL_EINVAL, "bad AAA arguments");
    std::vector<std::complex<double>> p;
    if (!wl::aaa_exp_poles(xmax, tol, p)) throw wl::Error(WL_ENOCONV, "AAA: pole eigenvalue iteration failed");
    *npoles = (int32_t)p.size();
    if ((int32_t)p.size() > cap) throw wl::Error(WL_EINVAL, "AAA: more poles than cap");
    for (size_t i = 0; i < p.size(); ++i) {
      re[i] = p[i].real();
      im[i] = p[i].imag();
    }
  });
}
