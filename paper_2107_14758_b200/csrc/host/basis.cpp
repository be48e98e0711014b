// 1D reference objects and the FDM basis (host, once per degree).
//   gll_nodes / gauss_legendre  <- src/quadrature.cpp:8-95
//   lagrange_eval               <- src/reference_interval.cpp:8-50
//   A_hat, B_hat                <- src/reference_interval.cpp:100-130
//   generalized Jacobi eig      <- src/dense_eig.cpp:11-94
//   S, lambda, A_t, B_t, parity <- src/fdm_basis.cpp:10-87
// The device kernels consume S, A_t/B_t (values + structural pattern), the
// interior eigenvalues and the GL(p+2) tables; computing them here once keeps
// the basis identical for every kernel.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "fdm_host.hpp"

namespace fdmgpu::host {
namespace {

// (P_k(x), P_k'(x)) by the three-term recurrence.
void legendre(int k, double x, double& v, double& dv) {
  double p0 = 1.0, d0 = 0.0;
  if (k == 0) {
    v = p0;
    dv = d0;
    return;
  }
  double p1 = x, d1 = 1.0;
  for (int n = 1; n < k; ++n) {
    const double p2 = ((2 * n + 1) * x * p1 - n * p0) / (n + 1);
    const double d2 = d0 + (2 * n + 1) * p1;
    p0 = p1;
    d0 = d1;
    p1 = p2;
    d1 = d2;
  }
  v = p1;
  dv = d1;
}

void mirror(Vec& x) {
  const int n = int(x.size());
  for (int i = 0; i < n / 2; ++i) {
    const double h = 0.5 * (x[n - 1 - i] - x[i]);
    x[i] = -h;
    x[n - 1 - i] = h;
  }
  if (n & 1) x[n / 2] = 0.0;
}

Dense mul(const Dense& A, const Dense& B, bool At = false) {
  const int m = At ? A.c : A.r, k = At ? A.r : A.c;
  Dense C(m, B.c);
  for (int j = 0; j < B.c; ++j)
    for (int l = 0; l < k; ++l) {
      const double b = B(l, j);
      for (int i = 0; i < m; ++i) C(i, j) += (At ? A(l, i) : A(i, l)) * b;
    }
  return C;
}

// sum_q M(q,i) w_q N(q,j), symmetrised.
Dense gram(const Dense& M, const Vec& w, const Dense& N) {
  Dense G(M.c, N.c);
  for (int i = 0; i < M.c; ++i)
    for (int j = 0; j < N.c; ++j) {
      double s = 0.0;
      for (int q = 0; q < M.r; ++q) s += M(q, i) * w[q] * N(q, j);
      G(i, j) = s;
    }
  Dense S(G.r, G.c);
  for (int i = 0; i < G.r; ++i)
    for (int j = 0; j < G.c; ++j) S(i, j) = 0.5 * (G(i, j) + G(j, i));
  return S;
}

// Cyclic Jacobi for symmetric A (src/dense_eig.cpp:11-65); eigenpairs ascending.
void jacobi(Dense A, Vec& lam, Dense& Vout) {
  const int n = A.r;
  Dense V(n, n);
  for (int i = 0; i < n; ++i) V(i, i) = 1.0;
  if (n > 1) {
    for (int sweep = 0; sweep < 30; ++sweep) {
      double off = 0.0;
      for (int p = 0; p < n - 1; ++p)
        for (int q = p + 1; q < n; ++q) off = std::max(off, std::abs(A(p, q)));
      if (off <= 1e-12) break;
      for (int p = 0; p < n - 1; ++p)
        for (int q = p + 1; q < n; ++q) {
          const double apq = A(p, q);
          if (std::abs(apq) <= 1e-17 * std::sqrt(std::abs(A(p, p) * A(q, q)) + 1e-300)) continue;
          const double th = (A(q, q) - A(p, p)) / (2.0 * apq);
          const double t = (th >= 0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
          const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
          for (int k = 0; k < n; ++k) {
            const double x = A(k, p), y = A(k, q);
            A(k, p) = c * x - s * y;
            A(k, q) = s * x + c * y;
          }
          for (int k = 0; k < n; ++k) {
            const double x = A(p, k), y = A(q, k);
            A(p, k) = c * x - s * y;
            A(q, k) = s * x + c * y;
          }
          for (int k = 0; k < n; ++k) {
            const double x = V(k, p), y = V(k, q);
            V(k, p) = c * x - s * y;
            V(k, q) = s * x + c * y;
          }
        }
    }
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return A(a, a) < A(b, b); });
  lam.resize(n);
  Vout = Dense(n, n);
  for (int j = 0; j < n; ++j) {
    lam[j] = A(ord[j], ord[j]);
    for (int i = 0; i < n; ++i) Vout(i, j) = V(i, ord[j]);
  }
}

// A V = B V diag(lam), V B-orthonormal, largest-magnitude entry positive
// (src/dense_eig.cpp:67-94): Cholesky congruence + Jacobi.
void gen_eig(const Dense& A, const Dense& B, Vec& lam, Dense& V) {
  const int n = A.r;
  Dense L(n, n);
  for (int j = 0; j < n; ++j) {
    double d = B(j, j);
    for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0.0)) throw std::invalid_argument("fdm basis: mass block is not positive definite");
    L(j, j) = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = B(i, j);
      for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / L(j, j);
    }
  }
  auto fwd = [&](Dense X) {  // L^{-1} X
    for (int c = 0; c < X.c; ++c)
      for (int i = 0; i < n; ++i) {
        double s = X(i, c);
        for (int k = 0; k < i; ++k) s -= L(i, k) * X(k, c);
        X(i, c) = s / L(i, i);
      }
    return X;
  };
  Dense C = fwd(A), Ct(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ct(i, j) = C(j, i);
  C = fwd(Ct);
  Dense Cs(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Cs(i, j) = 0.5 * (C(i, j) + C(j, i));
  Dense Q;
  jacobi(Cs, lam, Q);
  V = Q;  // L^{-T} Q
  for (int c = 0; c < n; ++c)
    for (int i = n - 1; i >= 0; --i) {
      double s = V(i, c);
      for (int k = i + 1; k < n; ++k) s -= L(k, i) * V(k, c);
      V(i, c) = s / L(i, i);
    }
  for (int j = 0; j < n; ++j) {
    double nrm2 = 0.0;
    for (int i = 0; i < n; ++i) {
      double bv = 0.0;
      for (int k = 0; k < n; ++k) bv += B(i, k) * V(k, j);
      nrm2 += V(i, j) * bv;
    }
    const double nrm = std::sqrt(nrm2);
    int imax = 0;
    double best = -1.0;
    for (int i = 0; i < n; ++i) {
      V(i, j) /= nrm;
      if (std::abs(V(i, j)) > best) {
        best = std::abs(V(i, j));
        imax = i;
      }
    }
    if (V(imax, j) < 0)
      for (int i = 0; i < n; ++i) V(i, j) = -V(i, j);
  }
}

}  // namespace

Vec gll_nodes(int p) {
  if (p < 1) throw std::invalid_argument("gll_nodes: degree must be >= 1");
  Vec x(p + 1);
  x[0] = -1.0;
  x[p] = 1.0;
  for (int k = 1; k < p; ++k) {
    double xk = -std::cos(M_PI * k / p);
    bool ok = false;
    for (int it = 0; it < 100; ++it) {
      double v, d;
      legendre(p, xk, v, d);
      const double dd = (2.0 * xk * d - p * (p + 1.0) * v) / (1.0 - xk * xk);
      const double dx = d / dd;
      xk -= dx;
      if (std::abs(d) < 1e-14 || std::abs(dx) < 1e-15) {
        ok = true;
        break;
      }
    }
    if (!ok) throw std::runtime_error("gll_nodes: Newton did not converge");
    x[k] = xk;
  }
  mirror(x);
  return x;
}

void gauss_legendre(int n, Vec& pts, Vec& wts) {
  if (n < 1) throw std::invalid_argument("gauss_legendre: need n >= 1");
  pts.assign(n, 0.0);
  wts.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double x = -std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double v, d;
      legendre(n, x, v, d);
      const double dx = v / d;
      x -= dx;
      if (std::abs(v) < 1e-15 || std::abs(dx) < 1e-15) break;
    }
    pts[i] = x;
  }
  mirror(pts);
  for (int i = 0; i < n; ++i) {
    double v, d;
    legendre(n, pts[i], v, d);
    wts[i] = 2.0 / ((1.0 - pts[i] * pts[i]) * d * d);
  }
  for (int i = 0; i < n / 2; ++i) wts[i] = wts[n - 1 - i] = 0.5 * (wts[i] + wts[n - 1 - i]);
}

void lagrange_eval(const Vec& nodes, const Vec& pts, Dense& V, Dense& D) {
  const int n = int(nodes.size()), m = int(pts.size());
  Vec w(n);
  for (int j = 0; j < n; ++j) {
    double prod = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != j) prod *= nodes[j] - nodes[k];
    w[j] = 1.0 / prod;
  }
  V = Dense(m, n);
  D = Dense(m, n);
  for (int q = 0; q < m; ++q) {
    const double x = pts[q];
    int hit = -1;
    for (int j = 0; j < n && hit < 0; ++j)
      if (std::abs(x - nodes[j]) < 8e-15) hit = j;
    if (hit >= 0) {
      V(q, hit) = 1.0;
      double diag = 0.0;
      for (int j = 0; j < n; ++j) {
        if (j == hit) continue;
        const double d = (w[j] / w[hit]) / (nodes[hit] - nodes[j]);
        D(q, j) = d;
        diag -= d;
      }
      D(q, hit) = diag;
      continue;
    }
    double s = 0.0, sp = 0.0;
    for (int j = 0; j < n; ++j) {
      const double g = w[j] / (x - nodes[j]);
      s += g;
      sp -= g / (x - nodes[j]);
    }
    for (int j = 0; j < n; ++j) {
      const double lj = (w[j] / (x - nodes[j])) / s;
      V(q, j) = lj;
      D(q, j) = lj * (-1.0 / (x - nodes[j]) - sp / s);
    }
  }
}

Basis1D make_bundle(int p) {
  Basis1D b;
  b.p = p;
  b.nodes = gll_nodes(p);
  Vec gp, gw;
  gauss_legendre(p + 1, gp, gw);
  Dense V, D;
  lagrange_eval(b.nodes, gp, V, D);
  b.A_hat = gram(D, gw, D);
  b.B_hat = gram(V, gw, V);
  // FDM basis: S_II = generalized eigenvectors of the interior blocks,
  // S_IG = -S_II S_II^T B_IG (src/fdm_basis.cpp:34-43).
  const int n1 = p + 1, ni = p - 1;
  const int ends[2] = {0, p};
  b.S = Dense(n1, n1);
  for (int i = 0; i < n1; ++i) b.S(i, i) = 1.0;
  Dense AII(ni, ni), BII(ni, ni), AIG(ni, 2), BIG(ni, 2);
  for (int i = 0; i < ni; ++i) {
    for (int j = 0; j < ni; ++j) {
      AII(i, j) = b.A_hat(1 + i, 1 + j);
      BII(i, j) = b.B_hat(1 + i, 1 + j);
    }
    for (int g = 0; g < 2; ++g) {
      AIG(i, g) = b.A_hat(1 + i, ends[g]);
      BIG(i, g) = b.B_hat(1 + i, ends[g]);
    }
  }
  Dense SII(ni, ni), SIG(ni, 2), AtIG(ni, 2), AtGG(2, 2), BtGG(2, 2);
  if (ni > 0) {
    gen_eig(AII, BII, b.lambda, SII);
    Dense M = mul(SII, BIG, true);  // S_II^T B_IG
    SIG = mul(SII, M);
    for (auto& v : SIG.a) v = -v;
    for (int i = 0; i < ni; ++i) {
      for (int j = 0; j < ni; ++j) b.S(1 + i, 1 + j) = SII(i, j);
      b.S(1 + i, 0) = SIG(i, 0);
      b.S(1 + i, p) = SIG(i, 1);
    }
    Dense T = mul(AII, SIG);
    for (size_t k = 0; k < T.a.size(); ++k) T.a[k] += AIG.a[k];
    AtIG = mul(SII, T, true);
    Dense t1 = mul(mul(SIG, AII, true), SIG), t2 = mul(SIG, AIG, true), t3 = mul(AIG, SIG, true);
    Dense MtM = mul(M, M, true);
    for (int g = 0; g < 2; ++g)
      for (int h = 0; h < 2; ++h) {
        AtGG(g, h) = t1(g, h) + t2(g, h) + t3(g, h) + b.A_hat(ends[g], ends[h]);
        BtGG(g, h) = b.B_hat(ends[g], ends[h]) - MtM(g, h);
      }
  } else {
    for (int g = 0; g < 2; ++g)
      for (int h = 0; h < 2; ++h) {
        AtGG(g, h) = b.A_hat(ends[g], ends[h]);
        BtGG(g, h) = b.B_hat(ends[g], ends[h]);
      }
  }
  b.A_t = Dense(n1, n1);
  b.B_t = Dense(n1, n1);
  b.A_nz.assign(size_t(n1) * n1, 0);
  b.B_nz.assign(size_t(n1) * n1, 0);
  auto put = [&](Dense& M, std::vector<uint8_t>& nz, int i, int j, double v) {
    M(i, j) += v;
    nz[i + size_t(n1) * j] = 1;
  };
  for (int i = 0; i < ni; ++i) {
    put(b.A_t, b.A_nz, 1 + i, 1 + i, b.lambda[i]);
    put(b.B_t, b.B_nz, 1 + i, 1 + i, 1.0);
    for (int g = 0; g < 2; ++g) {
      put(b.A_t, b.A_nz, 1 + i, ends[g], AtIG(i, g));
      put(b.A_t, b.A_nz, ends[g], 1 + i, AtIG(i, g));
    }
  }
  for (int g = 0; g < 2; ++g)
    for (int h = 0; h < 2; ++h) {
      put(b.A_t, b.A_nz, ends[g], ends[h], AtGG(g, h));
      put(b.B_t, b.B_nz, ends[g], ends[h], BtGG(g, h));
    }
  b.parity.assign(n1, 1.0);
  for (int j = 1; j < p; ++j) {
    double dot = 0.0;
    for (int i = 0; i <= p; ++i) dot += b.S(i, j) * b.S(p - i, j);
    b.parity[j] = dot >= 0.0 ? 1.0 : -1.0;
  }
  // True-form quadrature tables (src/assembly.cpp:198-215 uses GL(p+2)).
  b.q = p + 2;
  gauss_legendre(b.q, b.qp, b.wq);
  lagrange_eval(b.nodes, b.qp, b.Vq, b.Dq);
  return b;
}

}  // namespace fdmgpu::host
