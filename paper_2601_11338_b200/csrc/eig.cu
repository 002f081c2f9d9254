// eig.cu — eigenvalues of a small real upper Hessenberg matrix (host), for ρ(Z_θ) by Arnoldi
// (the dominant eigenvalue of Z scales α in §5.3, and bounds the
// resolvent series, Prop. pro:whe-we-converge P:317-322).
//
// Francis double-shift QR iteration (Golub & Van Loan, Matrix Computations, Alg. 7.5.1/7.5.2):
// the active window [lo, hi] shrinks by deflating negligible subdiagonal entries; a 1x1 block
// gives a real eigenvalue, a 2x2 block a real pair or a complex-conjugate pair; otherwise one
// implicit double-shift bulge-chasing sweep (3x3 Householder reflectors) is applied to the
// window, with exceptional shifts after 10 and 20 stagnant sweeps.  k <= 128, so O(k^3) host
// work is negligible next to the k SpMMs that built H.
#include "wl_internal.cuh"

#include <cmath>
#include <vector>

namespace wl {

namespace {
// eigenvalues of the 2x2 block [[a, b], [c, d]]
void eig2(double a, double b, double c, double d, double& r1, double& i1, double& r2, double& i2) {
  const double p = 0.5 * (a - d);
  const double q = p * p + b * c;
  if (q >= 0.0) {
    const double z = std::sqrt(q);
    const double s = p >= 0.0 ? p + z : p - z;  // avoid cancellation
    r1 = d + s;
    r2 = s != 0.0 ? d - b * c / s : d + s;
    i1 = i2 = 0.0;
  } else {
    r1 = r2 = d + p;
    i1 = std::sqrt(-q);
    i2 = -i1;
  }
}
}  // namespace

// H: n x n row-major upper Hessenberg (entries below the subdiagonal are ignored), overwritten.
// Returns false if some eigenvalue failed to converge in 60 sweeps (wr/wi then partial).
bool hessenberg_eigvals(std::vector<double>& H, int n, std::vector<double>& wr, std::vector<double>& wi) {
  auto A = [&](int i, int j) -> double& { return H[(size_t)i * n + j]; };
  wr.assign(n, 0.0);
  wi.assign(n, 0.0);
  double norm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = std::max(0, i - 1); j < n; ++j) norm += std::fabs(A(i, j));
  int hi = n - 1, its = 0;
  while (hi >= 0) {
    // deflation: find the start lo of the unreduced block ending at hi
    int lo = hi;
    while (lo > 0) {
      double s = std::fabs(A(lo - 1, lo - 1)) + std::fabs(A(lo, lo));
      if (s == 0.0) s = norm;
      // local test (unit roundoff relative to the neighbouring diagonal); after 20 stagnant sweeps also the
      // global one (relative to ‖H‖), which trades relative accuracy of tiny eigenvalues for convergence
      if (std::fabs(A(lo, lo - 1)) <= 2.220446049250313e-16 * (its >= 20 ? std::max(s, norm) : s)) {
        A(lo, lo - 1) = 0.0;
        break;
      }
      --lo;
    }
    if (lo == hi) {  // 1x1 block
      wr[hi] = A(hi, hi);
      --hi;
      its = 0;
      continue;
    }
    if (lo == hi - 1) {  // 2x2 block
      eig2(A(hi - 1, hi - 1), A(hi - 1, hi), A(hi, hi - 1), A(hi, hi), wr[hi - 1], wi[hi - 1], wr[hi], wi[hi]);
      hi -= 2;
      its = 0;
      continue;
    }
    if (its >= 60) return false;
    // shifts: eigenvalues of the trailing 2x2 (via trace s and determinant t), exceptional every 10
    double s, t;
    if (its == 10 || its == 20 || its == 40) {
      const double w = std::fabs(A(hi, hi - 1)) + std::fabs(A(hi - 1, hi - 2));
      s = 1.5 * w;
      t = w * w;
    } else {
      s = A(hi - 1, hi - 1) + A(hi, hi);
      t = A(hi - 1, hi - 1) * A(hi, hi) - A(hi - 1, hi) * A(hi, hi - 1);
    }
    ++its;
    // first column of (H - σ1 I)(H - σ2 I) = H² - s H + t I, restricted to rows lo..lo+2
    double x = A(lo, lo) * A(lo, lo) + A(lo, lo + 1) * A(lo + 1, lo) - s * A(lo, lo) + t;
    double y = A(lo + 1, lo) * (A(lo, lo) + A(lo + 1, lo + 1) - s);
    double z = A(lo + 1, lo) * A(lo + 2, lo + 1);
    for (int k = lo; k <= hi - 2; ++k) {
      // Householder reflector P = I - 2 v v^T / v^T v zeroing y, z of (x, y, z)
      const double alpha = -std::copysign(std::sqrt(x * x + y * y + z * z), x);
      double v0 = x - alpha, v1 = y, v2 = z;
      const double vn = v0 * v0 + v1 * v1 + v2 * v2;
      if (vn != 0.0) {
        const double beta = 2.0 / vn;
        const int c0 = std::max(lo, k - 1);
        for (int j = c0; j < n; ++j) {  // rows k..k+2 from the left
          const double d = beta * (v0 * A(k, j) + v1 * A(k + 1, j) + v2 * A(k + 2, j));
          A(k, j) -= d * v0;
          A(k + 1, j) -= d * v1;
          A(k + 2, j) -= d * v2;
        }
        const int r1 = std::min(hi, k + 3);
        for (int i = 0; i <= r1; ++i) {  // columns k..k+2 from the right
          const double d = beta * (v0 * A(i, k) + v1 * A(i, k + 1) + v2 * A(i, k + 2));
          A(i, k) -= d * v0;
          A(i, k + 1) -= d * v1;
          A(i, k + 2) -= d * v2;
        }
      }
      x = A(k + 1, k);
      y = A(k + 2, k);
      if (k < hi - 2) z = A(k + 3, k);
    }
    // last 2-vector reflector for rows hi-1, hi
    {
      const int k = hi - 1;
      const double alpha = -std::copysign(std::sqrt(x * x + y * y), x);
      const double v0 = x - alpha, v1 = y;
      const double vn = v0 * v0 + v1 * v1;
      if (vn != 0.0) {
        const double beta = 2.0 / vn;
        for (int j = std::max(lo, k - 1); j < n; ++j) {
          const double d = beta * (v0 * A(k, j) + v1 * A(k + 1, j));
          A(k, j) -= d * v0;
          A(k + 1, j) -= d * v1;
        }
        for (int i = 0; i <= hi; ++i) {
          const double d = beta * (v0 * A(i, k) + v1 * A(i, k + 1));
          A(i, k) -= d * v0;
          A(i, k + 1) -= d * v1;
        }
      }
    }
    // keep the matrix exactly Hessenberg inside the window (bulge remnants are rounding)
    for (int i = lo + 2; i <= hi; ++i)
      for (int j = lo; j < i - 1; ++j) A(i, j) = 0.0;
  }
  return true;
}

}  // namespace wl
