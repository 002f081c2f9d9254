// trace.cu — host side of XNysTrace-exp (Alg. 1, alg:trace_estimation P:584-597).
//
// The device side (engine.cu, wl_xnystrace_exp) builds the block Krylov basis V_{k+1} of 𝔏 from
// the probe block Ω — poles at ∞ (reading R16) — and hands over the kM x kM projected
// matrix H_k = V_kᵀ 𝔏 V_k and R_0 (Ω = V_1 R_0).  Everything after that lives in the kM-dimensional
// coordinates of V_k, where inner products are those of R^n (V_k orthonormal, Ω in span V_1):
//   * H_k = Q Λ Qᵀ (cyclic Jacobi; 𝔏 symmetric ⇒ H_k symmetric, Prop. pro:still-again-an-mmatrix);
//   * in eigen-coordinates Ω ↦ W = Qᵀ [R_0; 0] and Y(t) = (1/n) V_k exp(-t H_k) V_kᵀ Ω ↦ diag(e^{-tλ}/n) W
//     (P:596);
//   * XNysTrace(Y(t), Ω) (reading R17): shifted leave-one-out Nyström, per probe i
//       C Cᵀ = Ω_{-i}ᵀ Y_ν,_{-i},  B = Y_ν,_{-i} C⁻ᵀ,  b = C⁻¹ Y_ν,_{-i}ᵀ ω_i,
//       est_i = ‖B‖_F² + ω_iᵀ y_ν,i − ‖b‖²,   p̂ = mean est − ν n,   ê = std(est) / √M,
//     with ν = 1e-12 ‖Y‖_F / √M.
// All O((kM)^3 + nt M^2 kM) host work; the n-sized work (k block Laplacian actions and the block
// Gram–Schmidt GEMMs) is on the GPU.
#include "wl_internal.cuh"

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

namespace wl {

// Symmetric eigendecomposition by cyclic Jacobi rotations (Golub & Van Loan Alg. 8.5.3).
// A: d x d row-major symmetric (overwritten); lam (d), Q (d x d row-major, columns = eigenvectors).
bool sym_eig_jacobi(std::vector<double>& A, int d, std::vector<double>& lam, std::vector<double>& Q) {
  auto a = [&](int i, int j) -> double& { return A[(size_t)i * d + j]; };
  Q.assign((size_t)d * d, 0.0);
  for (int i = 0; i < d; ++i) Q[(size_t)i * d + i] = 1.0;
  double fro = 0.0;
  for (double v : A) fro += v * v;
  fro = std::sqrt(fro);
  bool ok = false;
  for (int sweep = 0; sweep < 60 && !ok; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < d; ++i)
      for (int j = i + 1; j < d; ++j) off += a(i, j) * a(i, j);
    if (std::sqrt(2.0 * off) <= 1e-15 * fro) { ok = true; break; }
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) {
        const double apq = a(p, q);
        if (std::abs(apq) <= 1e-300) continue;
        const double th = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (th >= 0.0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < d; ++k) {  // columns p, q
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < d; ++k) {  // rows p, q
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < d; ++k) {
          double* r = &Q[(size_t)k * d];
          const double qp = r[p], qq = r[q];
          r[p] = c * qp - s * qq;
          r[q] = s * qp + c * qq;
        }
      }
  }
  lam.resize(d);
  for (int i = 0; i < d; ++i) lam[i] = a(i, i);
  return ok;
}

// Symmetric eigendecomposition by Householder tridiagonalisation and the implicit QL iteration with
// Wilkinson shifts (Golub & Van Loan §8.3; the EISPACK tred2/tql2 pair).  O(d^3) with a small constant:
// the default behind wl_xnystrace_exp (Jacobi above is the slower cross-check).
// A: d x d row-major symmetric (overwritten by the eigenvectors: column i of A = eigenvector i).
bool sym_eig_tridiag_ql(std::vector<double>& A, int d, std::vector<double>& lam) {
  auto a = [&](int i, int j) -> double& { return A[(size_t)i * d + j]; };
  std::vector<double> e(d, 0.0);
  lam.assign(d, 0.0);
  std::vector<double>& dd = lam;
  for (int i = d - 1; i > 0; --i) {  // Householder: zero row i left of the subdiagonal
    const int l = i - 1;
    double h = 0.0, scale = 0.0;
    if (l > 0) {
      for (int k = 0; k <= l; ++k) scale += std::abs(a(i, k));
      if (scale == 0.0) {
        e[i] = a(i, l);
      } else {
        for (int k = 0; k <= l; ++k) {
          a(i, k) /= scale;
          h += a(i, k) * a(i, k);
        }
        double f = a(i, l);
        double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
        e[i] = scale * g;
        h -= f * g;
        a(i, l) = f - g;
        f = 0.0;
        for (int j = 0; j <= l; ++j) {
          a(j, i) = a(i, j) / h;
          g = 0.0;
          for (int k = 0; k <= j; ++k) g += a(j, k) * a(i, k);
          for (int k = j + 1; k <= l; ++k) g += a(k, j) * a(i, k);
          e[j] = g / h;
          f += e[j] * a(i, j);
        }
        const double hh = f / (h + h);
        for (int j = 0; j <= l; ++j) {
          f = a(i, j);
          e[j] = g = e[j] - hh * f;
          for (int k = 0; k <= j; ++k) a(j, k) -= f * e[k] + g * a(i, k);
        }
      }
    } else {
      e[i] = a(i, l);
    }
    dd[i] = h;
  }
  dd[0] = 0.0;
  e[0] = 0.0;
  for (int i = 0; i < d; ++i) {  // accumulate the transformations
    const int l = i - 1;
    if (dd[i] != 0.0) {
      for (int j = 0; j <= l; ++j) {
        double g = 0.0;
        for (int k = 0; k <= l; ++k) g += a(i, k) * a(k, j);
        for (int k = 0; k <= l; ++k) a(k, j) -= g * a(k, i);
      }
    }
    dd[i] = a(i, i);
    a(i, i) = 1.0;
    for (int j = 0; j <= l; ++j) a(j, i) = a(i, j) = 0.0;
  }
  for (int i = 1; i < d; ++i) e[i - 1] = e[i];
  if (d > 0) e[d - 1] = 0.0;
  for (int l = 0; l < d; ++l) {  // implicit QL on the tridiagonal (dd, e)
    int iter = 0, m;
    do {
      for (m = l; m < d - 1; ++m) {
        const double s2 = std::abs(dd[m]) + std::abs(dd[m + 1]);
        if (std::abs(e[m]) <= 1e-16 * s2) break;
      }
      if (m != l) {
        if (iter++ == 60) return false;
        double g = (dd[l + 1] - dd[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = dd[m] - dd[l] + e[l] / (g + (g >= 0.0 ? std::abs(r) : -std::abs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          e[i + 1] = (r = std::hypot(f, g));
          if (r == 0.0) {
            dd[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = dd[i + 1] - p;
          r = (dd[i] - g) * s + 2.0 * c * b;
          dd[i + 1] = g + (p = s * r);
          g = c * r - b;
          for (int k = 0; k < d; ++k) {
            f = a(k, i + 1);
            a(k, i + 1) = s * a(k, i) + c * f;
            a(k, i) = c * a(k, i) - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        dd[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  return true;
}

namespace {
// lower Cholesky of the m x m row-major SPD S (in place); false if not positive definite
bool chol_lower(std::vector<double>& S, int m) {
  for (int j = 0; j < m; ++j) {
    double dj = S[(size_t)j * m + j];
    for (int k = 0; k < j; ++k) dj -= S[(size_t)j * m + k] * S[(size_t)j * m + k];
    if (!(dj > 0.0)) return false;
    dj = std::sqrt(dj);
    S[(size_t)j * m + j] = dj;
    for (int i = j + 1; i < m; ++i) {
      double v = S[(size_t)i * m + j];
      for (int k = 0; k < j; ++k) v -= S[(size_t)i * m + k] * S[(size_t)j * m + k];
      S[(size_t)i * m + j] = v / dj;
    }
  }
  return true;
}
// x <- C⁻¹ x for lower-triangular C (m x m row-major)
void fwd(const std::vector<double>& C, int m, double* x) {
  for (int i = 0; i < m; ++i) {
    double v = x[i];
    for (int k = 0; k < i; ++k) v -= C[(size_t)i * m + k] * x[k];
    x[i] = v / C[(size_t)i * m + i];
  }
}
}  // namespace

// XNysTrace of Y(t) for every t from the eigen-coordinates (see the file header).
//   lam (d), W (d x M row-major) = Qᵀ [R_0; 0];  n = global dimension.
// Returns false if some leave-one-out Gram matrix is not positive definite.
namespace {
bool curve_range(const std::vector<double>& lam, const std::vector<double>& W, int d, int M, double n,
                 const double* times, int s0, int s1, double* p_out, double* e_out) {
  std::vector<double> g(d), Y((size_t)d * M), G((size_t)M * M), S, est(M), Bcol(M), b(M);
  for (int s = s0; s < s1; ++s) {
    const double t = times[s];
    double ny = 0.0;
    for (int a = 0; a < d; ++a) {
      g[a] = std::exp(-t * lam[a]) / n;
      for (int c = 0; c < M; ++c) ny += (g[a] * W[(size_t)a * M + c]) * (g[a] * W[(size_t)a * M + c]);
    }
    const double nu = 1e-12 * std::sqrt(ny) / std::sqrt((double)M);
    for (int a = 0; a < d; ++a)
      for (int c = 0; c < M; ++c) Y[(size_t)a * M + c] = (g[a] + nu) * W[(size_t)a * M + c];  // Y_ν = Y + νΩ
    // G = Ωᵀ Y_ν (M x M): the Gram entries every leave-one-out problem draws from
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
        for (int a = 0; a < d; ++a) v += W[(size_t)a * M + r] * Y[(size_t)a * M + c];
        G[(size_t)r * M + c] = v;
      }
    for (int i = 0; i < M; ++i) {
      const int m = M - 1;
      double tr = 0.0, ww = 0.0;
      const double wy = G[(size_t)i * M + i];  // ω_iᵀ y_ν,i
      if (m > 0) {
        // S = Ω_{-i}ᵀ Y_ν,_{-i} (symmetrised), b = Y_ν,_{-i}ᵀ ω_i
        S.assign((size_t)m * m, 0.0);
        for (int r = 0, rr = 0; r < M; ++r) {
          if (r == i) continue;
          for (int c = 0, cc = 0; c < M; ++c) {
            if (c == i) continue;
            S[(size_t)rr * m + cc] = 0.5 * (G[(size_t)r * M + c] + G[(size_t)c * M + r]);
            ++cc;
          }
          b[rr] = G[(size_t)i * M + r];
          ++rr;
        }
        if (!chol_lower(S, m)) return false;
        // ‖B‖_F² = Σ_a ‖C⁻¹ (row a of Y_ν,_{-i})‖²
        for (int a = 0; a < d; ++a) {
          for (int c = 0, cc = 0; c < M; ++c)
            if (c != i) Bcol[cc++] = Y[(size_t)a * M + c];
          fwd(S, m, Bcol.data());
          for (int c = 0; c < m; ++c) tr += Bcol[c] * Bcol[c];
        }
        fwd(S, m, b.data());
        for (int c = 0; c < m; ++c) ww += b[c] * b[c];
      }
      est[i] = tr + (wy - ww);
    }
    double mean = 0.0;
    for (int i = 0; i < M; ++i) mean += est[i];
    mean /= M;
    double var = 0.0;
    for (int i = 0; i < M; ++i) var += (est[i] - mean) * (est[i] - mean);
    p_out[s] = mean - nu * n;
    e_out[s] = M > 1 ? std::sqrt(var / (M - 1)) / std::sqrt((double)M) : 0.0;
  }
  return true;
}
}  // namespace

// The t-points are independent ("Can be a parfor", Alg. 1 line 5): split over host threads.
bool xnystrace_curve(const std::vector<double>& lam, const std::vector<double>& W, int d, int M, double n,
                     const double* times, int nt, double* p_out, double* e_out) {
  const int nth = std::max(1, std::min<int>({nt, 16, (int)std::thread::hardware_concurrency()}));
  std::vector<std::thread> th;
  std::vector<char> ok(nth, 1);
  for (int w = 0; w < nth; ++w) {
    const int s0 = (int)((int64_t)nt * w / nth), s1 = (int)((int64_t)nt * (w + 1) / nth);
    th.emplace_back([&, w, s0, s1] { ok[w] = curve_range(lam, W, d, M, n, times, s0, s1, p_out, e_out); });
  }
  for (auto& t : th) t.join();
  return std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; });
}

}  // namespace wl
