// TEST INFRASTRUCTURE ONLY — oracle restatement, see oracle.hpp header.
// L0/L1: quadrature, reference interval, dense eigen, FDM basis, kron,
// sparse helpers, orderings and the up-looking sparse Cholesky.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>

#include "oracle.hpp"

namespace oracle {

Mat Mat::transpose() const {
  Mat t(c, r);
  for (int j = 0; j < c; ++j)
    for (int i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
  return t;
}

Mat matmul(const Mat& A, const Mat& B) {
  if (A.c != B.r) throw std::invalid_argument("matmul: shape mismatch");
  Mat C(A.r, B.c);
  for (int j = 0; j < B.c; ++j)
    for (int k = 0; k < A.c; ++k) {
      const double b = B(k, j);
      for (int i = 0; i < A.r; ++i) C(i, j) += A(i, k) * b;
    }
  return C;
}

int PatMat::nonzeros() const {
  int n = 0;
  for (char z : nz) n += z != 0;
  return n;
}

Csr csr_from_triplets(int n, int m, const std::vector<Triplet>& t) {
  Csr A;
  A.n = n;
  A.m = m;
  std::vector<int64_t> cnt(n + 1, 0);
  for (const auto& e : t) ++cnt[e.i + 1];
  for (int i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<std::pair<int, double>> tmp(t.size());
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (const auto& e : t) tmp[pos[e.i]++] = {e.j, e.v};
  A.ptr.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    auto b = tmp.begin() + cnt[i], en = tmp.begin() + cnt[i + 1];
    std::stable_sort(b, en, [](const auto& x, const auto& y) { return x.first < y.first; });
    for (auto it = b; it != en;) {
      int c = it->first;
      double s = 0.0;
      for (; it != en && it->first == c; ++it) s += it->second;
      A.col.push_back(c);
      A.val.push_back(s);
    }
    A.ptr[i + 1] = int64_t(A.col.size());
  }
  return A;
}

Vec spmv(const Csr& A, const Vec& x) {
  if (int(x.size()) != A.m) throw std::invalid_argument("spmv: dimension mismatch");
  Vec y(A.n, 0.0);
  for (int i = 0; i < A.n; ++i) {
    double acc = 0.0;
    for (int64_t q = A.ptr[i]; q < A.ptr[i + 1]; ++q) acc += A.val[q] * x[A.col[q]];
    y[i] = acc;
  }
  return y;
}

Vec spmv_transpose(const Csr& A, const Vec& x) {
  Vec y(A.m, 0.0);
  for (int i = 0; i < A.n; ++i)
    for (int64_t q = A.ptr[i]; q < A.ptr[i + 1]; ++q) y[A.col[q]] += A.val[q] * x[i];
  return y;
}

Csr extract_submatrix(const Csr& A, const std::vector<int>& dofs) {
  std::vector<int> where(A.n, -1);
  for (size_t k = 0; k < dofs.size(); ++k) where[dofs[k]] = int(k);
  std::vector<Triplet> t;
  for (size_t k = 0; k < dofs.size(); ++k)
    for (int64_t q = A.ptr[dofs[k]]; q < A.ptr[dofs[k] + 1]; ++q)
      if (where[A.col[q]] >= 0) t.push_back({int(k), where[A.col[q]], A.val[q]});
  return csr_from_triplets(int(dofs.size()), int(dofs.size()), t);
}

// ---- quadrature (src/quadrature.cpp) ----------------------------------------
std::pair<double, double> legendre_value_deriv(int k, double x) {
  double pm1 = 1.0, dm1 = 0.0;
  if (k == 0) return {pm1, dm1};
  double p = x, d = 1.0;
  for (int n = 1; n < k; ++n) {
    const double pn1 = ((2 * n + 1) * x * p - n * pm1) / (n + 1);
    const double dn1 = dm1 + (2 * n + 1) * p;
    pm1 = p;
    dm1 = d;
    p = pn1;
    d = dn1;
  }
  return {p, d};
}

static void symmetrize(Vec& x) {  // src/quadrature.cpp:28-37
  const int n = int(x.size());
  for (int i = 0; i < n / 2; ++i) {
    const double v = 0.5 * (x[n - 1 - i] - x[i]);
    x[i] = -v;
    x[n - 1 - i] = v;
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

Vec gll_nodes(int p) {
  if (p < 1) throw std::invalid_argument("gll_nodes: degree must be >= 1");
  Vec x(p + 1);
  x[0] = -1.0;
  x[p] = 1.0;
  for (int k = 1; k < p; ++k) {
    double xk = -std::cos(M_PI * k / p);
    bool converged = false;
    for (int it = 0; it < 100; ++it) {
      const auto [v, d] = legendre_value_deriv(p, xk);
      const double dd = (2.0 * xk * d - p * (p + 1.0) * v) / (1.0 - xk * xk);
      const double dx = d / dd;
      xk -= dx;
      if (std::abs(d) < 1e-14 || std::abs(dx) < 1e-15) {
        converged = true;
        break;
      }
    }
    if (!converged) throw std::runtime_error("gll_nodes: Newton did not converge");
    x[k] = xk;
  }
  symmetrize(x);
  return x;
}

QuadratureRule gauss_legendre_rule(int n) {
  if (n < 1) throw std::invalid_argument("gauss_legendre_rule: need n >= 1");
  QuadratureRule rule;
  rule.points.resize(n);
  rule.weights.resize(n);
  for (int i = 0; i < n; ++i) {
    double x = -std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      const auto [v, d] = legendre_value_deriv(n, x);
      const double dx = v / d;
      x -= dx;
      if (std::abs(v) < 1e-15 || std::abs(dx) < 1e-15) break;
    }
    rule.points[i] = x;
  }
  symmetrize(rule.points);
  for (int i = 0; i < n; ++i) {
    const auto [v, d] = legendre_value_deriv(n, rule.points[i]);
    (void)v;
    const double x = rule.points[i];
    rule.weights[i] = 2.0 / ((1.0 - x * x) * d * d);
  }
  for (int i = 0; i < n / 2; ++i) {
    const double w = 0.5 * (rule.weights[i] + rule.weights[n - 1 - i]);
    rule.weights[i] = rule.weights[n - 1 - i] = w;
  }
  return rule;
}

// ---- reference interval (src/reference_interval.cpp) ------------------------
void lagrange_eval(const Vec& nodes, const Vec& pts, Mat& values, Mat& derivs) {
  const int n = int(nodes.size()), m = int(pts.size());
  Vec w(n);
  for (int j = 0; j < n; ++j) {
    double prod = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != j) prod *= nodes[j] - nodes[k];
    w[j] = 1.0 / prod;
  }
  values = Mat(m, n);
  derivs = Mat(m, n);
  for (int q = 0; q < m; ++q) {
    const double x = pts[q];
    int hit = -1;
    for (int j = 0; j < n; ++j)
      if (std::abs(x - nodes[j]) < 8e-15) {
        hit = j;
        break;
      }
    if (hit >= 0) {
      values(q, hit) = 1.0;
      double diag = 0.0;
      for (int j = 0; j < n; ++j) {
        if (j == hit) continue;
        const double d = (w[j] / w[hit]) / (nodes[hit] - nodes[j]);
        derivs(q, j) = d;
        diag -= d;
      }
      derivs(q, hit) = diag;
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
      values(q, j) = lj;
      derivs(q, j) = lj * (-1.0 / (x - nodes[j]) - sp / s);
    }
  }
}

static void lobatto_eval(int p, const Vec& pts, Mat& values, Mat& derivs) {  // src/reference_interval.cpp:57-78
  const int m = int(pts.size());
  values = Mat(m, p + 1);
  derivs = Mat(m, p + 1);
  for (int q = 0; q < m; ++q) {
    const double x = pts[q];
    values(q, 0) = 0.5 * (1.0 - x);
    derivs(q, 0) = -0.5;
    values(q, p) = 0.5 * (1.0 + x);
    derivs(q, p) = 0.5;
    Vec P(p + 2);
    P[0] = 1.0;
    P[1] = x;
    for (int k = 1; k <= p; ++k) P[k + 1] = ((2 * k + 1) * x * P[k] - k * P[k - 1]) / (k + 1);
    for (int j = 1; j < p; ++j) {
      values(q, j) = (P[j + 1] - P[j - 1]) / (2 * j + 1);
      derivs(q, j) = P[j];
    }
  }
}

void ReferenceInterval::eval(const Vec& pts, Mat& values, Mat& derivs) const {
  if (kind == BasisKind::LobattoHierarchical)
    lobatto_eval(degree, pts, values, derivs);
  else
    lagrange_eval(nodes, pts, values, derivs);
}

// M^T diag(w) N, i.e. Eigen's `M.transpose() * w.asDiagonal() * N`.
static Mat weighted_gram(const Mat& M, const Vec& w, const Mat& N) {
  Mat out(M.c, N.c);
  for (int i = 0; i < M.c; ++i)
    for (int j = 0; j < N.c; ++j) {
      double s = 0.0;
      for (int q = 0; q < M.r; ++q) s += M(q, i) * w[q] * N(q, j);
      out(i, j) = s;
    }
  return out;
}

static void symmetrize_mat(Mat& A) {
  Mat T = A.transpose();
  for (size_t k = 0; k < A.a.size(); ++k) A.a[k] = 0.5 * (A.a[k] + T.a[k]);
}

ReferenceInterval reference_operators(int p, BasisKind kind) {
  if (p < 1) throw std::invalid_argument("reference_operators: degree must be >= 1");
  ReferenceInterval ref;
  ref.degree = p;
  ref.kind = kind;
  ref.nodes = (kind == BasisKind::GlNodal) ? gauss_legendre_rule(p + 1).points : gll_nodes(p);
  const QuadratureRule quad = gauss_legendre_rule(p + 1);
  Mat V, D;
  ref.eval(quad.points, V, D);
  ref.stiffness = weighted_gram(D, quad.weights, D);
  ref.mass = weighted_gram(V, quad.weights, V);
  symmetrize_mat(ref.stiffness);
  symmetrize_mat(ref.mass);
  Mat tv, td;
  ref.eval({-1.0, 1.0}, tv, td);
  for (int j = 0; j <= p; ++j) td(0, j) *= -1.0;
  ref.trace_values = tv;
  ref.trace_normal_derivs = td;
  return ref;
}

// ---- dense eig (src/dense_eig.cpp) -------------------------------------------
std::pair<Vec, Mat> jacobi_sym_eig(Mat A) {
  const int n = A.r;
  Mat V = Mat::identity(n);
  if (n == 1) return {Vec{A(0, 0)}, V};
  const double tol = 1e-12;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) off = std::max(off, std::abs(A(p, q)));
    if (off <= tol) break;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (std::abs(apq) <= 1e-17 * std::sqrt(std::abs(A(p, p) * A(q, q)) + 1e-300)) continue;
        const double theta = (A(q, q) - A(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V(k, p), vkq = V(k, q);
          V(k, p) = c * vkp - s * vkq;
          V(k, q) = s * vkp + c * vkq;
        }
      }
    }
  }
  Vec lambda(n);
  for (int i = 0; i < n; ++i) lambda[i] = A(i, i);
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return lambda[a] < lambda[b]; });
  Vec ls(n);
  Mat Vs(n, n);
  for (int j = 0; j < n; ++j) {
    ls[j] = lambda[order[j]];
    for (int i = 0; i < n; ++i) Vs(i, j) = V(i, order[j]);
  }
  return {ls, Vs};
}

// Dense LLT (Eigen::LLT stand-in): lower L with B = L L^T; false if not SPD.
static bool dense_llt(const Mat& B, Mat& L) {
  const int n = B.r;
  L = Mat(n, n);
  for (int j = 0; j < n; ++j) {
    double d = B(j, j);
    for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0.0)) return false;
    L(j, j) = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = B(i, j);
      for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / L(j, j);
    }
  }
  return true;
}

// Solve L X = B (L lower) in place of B.
static Mat lower_solve(const Mat& L, Mat B) {
  const int n = L.r;
  for (int c = 0; c < B.c; ++c)
    for (int i = 0; i < n; ++i) {
      double s = B(i, c);
      for (int k = 0; k < i; ++k) s -= L(i, k) * B(k, c);
      B(i, c) = s / L(i, i);
    }
  return B;
}

// Solve L^T X = B (upper solve with L^T).
static Mat upper_t_solve(const Mat& L, Mat B) {
  const int n = L.r;
  for (int c = 0; c < B.c; ++c)
    for (int i = n - 1; i >= 0; --i) {
      double s = B(i, c);
      for (int k = i + 1; k < n; ++k) s -= L(k, i) * B(k, c);
      B(i, c) = s / L(i, i);
    }
  return B;
}

std::pair<Vec, Mat> dense_sym_gen_eig(const Mat& A, const Mat& B) {
  if (A.r != B.r || A.r != A.c || B.r != B.c)
    throw std::invalid_argument("dense_sym_gen_eig: dimension mismatch");
  Mat L;
  if (!dense_llt(B, L)) throw std::invalid_argument("dense_sym_gen_eig: B is not positive definite");
  Mat C = lower_solve(L, A);
  C = lower_solve(L, C.transpose());
  symmetrize_mat(C);
  auto [lambda, Q] = jacobi_sym_eig(C);
  Mat V = upper_t_solve(L, Q);
  const int n = V.r;
  for (int j = 0; j < V.c; ++j) {
    double nrm2 = 0.0;
    for (int i = 0; i < n; ++i) {
      double bv = 0.0;
      for (int k = 0; k < n; ++k) bv += B(i, k) * V(k, j);
      nrm2 += V(i, j) * bv;
    }
    const double nrm = std::sqrt(nrm2);
    int imax = 0;
    double vmax = -1.0;
    for (int i = 0; i < n; ++i) {
      V(i, j) /= nrm;
      if (std::abs(V(i, j)) > vmax) {
        vmax = std::abs(V(i, j));
        imax = i;
      }
    }
    if (V(imax, j) < 0)
      for (int i = 0; i < n; ++i) V(i, j) *= -1.0;
  }
  return {lambda, V};
}

// ---- FDM basis (src/fdm_basis.cpp:10-87) --------------------------------------
FdmBasis fdm_basis(const ReferenceInterval& ref) {
  if (ref.kind != BasisKind::GllNodal) throw std::invalid_argument("fdm_basis: expects the GLL-nodal reference");
  const int p = ref.degree, ni = p - 1;
  FdmBasis fdm;
  fdm.degree = p;
  fdm.S = Mat::identity(p + 1);
  fdm.lambda.assign(ni, 0.0);
  const Mat& A = ref.stiffness;
  const Mat& B = ref.mass;
  Mat A_II(ni, ni), B_II(ni, ni), A_IG(ni, 2), B_IG(ni, 2), A_GG(2, 2), B_GG(2, 2);
  for (int i = 0; i < ni; ++i) {
    for (int j = 0; j < ni; ++j) {
      A_II(i, j) = A(1 + i, 1 + j);
      B_II(i, j) = B(1 + i, 1 + j);
    }
    A_IG(i, 0) = A(1 + i, 0);
    A_IG(i, 1) = A(1 + i, p);
    B_IG(i, 0) = B(1 + i, 0);
    B_IG(i, 1) = B(1 + i, p);
  }
  const int sl[2] = {0, p};
  for (int g = 0; g < 2; ++g)
    for (int h = 0; h < 2; ++h) {
      A_GG(g, h) = A(sl[g], sl[h]);
      B_GG(g, h) = B(sl[g], sl[h]);
    }
  Mat S_II(ni, ni), S_IG(ni, 2);
  if (ni > 0) {
    auto [lambda, V] = dense_sym_gen_eig(A_II, B_II);
    fdm.lambda = lambda;
    S_II = V;
    Mat t = matmul(S_II.transpose(), B_IG);
    S_IG = matmul(S_II, t);
    for (auto& v : S_IG.a) v = -v;
    for (int i = 0; i < ni; ++i) {
      for (int j = 0; j < ni; ++j) fdm.S(1 + i, 1 + j) = S_II(i, j);
      fdm.S(1 + i, 0) = S_IG(i, 0);
      fdm.S(1 + i, p) = S_IG(i, 1);
    }
  }
  Mat At_IG(ni, 2), At_GG(2, 2), Bt_GG(2, 2);
  if (ni > 0) {
    Mat AS = matmul(A_II, S_IG);
    for (size_t k = 0; k < AS.a.size(); ++k) AS.a[k] += A_IG.a[k];
    At_IG = matmul(S_II.transpose(), AS);
    Mat SIGt = S_IG.transpose();
    Mat t1 = matmul(matmul(SIGt, A_II), S_IG), t2 = matmul(SIGt, A_IG), t3 = matmul(A_IG.transpose(), S_IG);
    for (int k = 0; k < 4; ++k) At_GG.a[k] = t1.a[k] + t2.a[k] + t3.a[k] + A_GG.a[k];
    Mat M = matmul(S_II.transpose(), B_IG);
    Mat MtM = matmul(M.transpose(), M);
    for (int k = 0; k < 4; ++k) Bt_GG.a[k] = B_GG.a[k] - MtM.a[k];
  } else {
    At_GG = A_GG;
    Bt_GG = B_GG;
  }
  fdm.A_t.val = Mat(p + 1, p + 1);
  fdm.B_t.val = Mat(p + 1, p + 1);
  fdm.A_t.nz.assign(size_t(p + 1) * (p + 1), 0);
  fdm.B_t.nz.assign(size_t(p + 1) * (p + 1), 0);
  auto put = [&](PatMat& M, int i, int j, double v) {
    M.val(i, j) += v;
    M.nz[i + size_t(p + 1) * j] = 1;
  };
  for (int i = 0; i < ni; ++i) {
    put(fdm.A_t, 1 + i, 1 + i, fdm.lambda[i]);
    put(fdm.B_t, 1 + i, 1 + i, 1.0);
    for (int g = 0; g < 2; ++g) {
      put(fdm.A_t, 1 + i, sl[g], At_IG(i, g));
      put(fdm.A_t, sl[g], 1 + i, At_IG(i, g));
    }
  }
  for (int g = 0; g < 2; ++g)
    for (int h = 0; h < 2; ++h) {
      put(fdm.A_t, sl[g], sl[h], At_GG(g, h));
      put(fdm.B_t, sl[g], sl[h], Bt_GG(g, h));
    }
  fdm.parity.assign(p + 1, 1.0);
  for (int j = 1; j < p; ++j) {
    double dot = 0.0;
    for (int i = 0; i <= p; ++i) dot += fdm.S(i, j) * fdm.S(p - i, j);
    fdm.parity[j] = (dot >= 0.0) ? 1.0 : -1.0;
  }
  // deriv_traces = trace_normal_derivs * S (src/fdm_basis.cpp:78)
  fdm.deriv_traces = Mat(2, p + 1);
  for (int e = 0; e < 2; ++e)
    for (int c = 0; c <= p; ++c) {
      double acc = 0.0;
      for (int k = 0; k <= p; ++k) acc += ref.trace_normal_derivs(e, k) * fdm.S(k, c);
      fdm.deriv_traces(e, c) = acc;
    }
  return fdm;
}

// ---- kron (src/kron.cpp) ------------------------------------------------------
int KronOperator::rows() const {
  if (terms.empty()) return 0;
  int n = 1;
  for (const auto& f : terms[0].factors) n *= f.r;
  return n;
}
int KronOperator::cols() const {
  int n = 1;
  for (int d : dims) n *= d;
  return n;
}

Vec apply_axis(const Mat& M, const Vec& x, const std::vector<int>& dims, int axis) {
  const int d = int(dims.size());
  if (axis < 0 || axis >= d) throw std::invalid_argument("apply_axis: bad axis");
  const int n = dims[axis];
  if (M.c != n) throw std::invalid_argument("apply_axis: shape mismatch");
  const int m = M.r;
  int left = 1, right = 1;
  for (int k = 0; k < axis; ++k) left *= dims[k];
  for (int k = axis + 1; k < d; ++k) right *= dims[k];
  Vec y(size_t(left) * m * right, 0.0);
  for (int r = 0; r < right; ++r) {
    const double* X = x.data() + size_t(r) * left * n;
    double* Y = y.data() + size_t(r) * left * m;
    for (int k = 0; k < m; ++k)
      for (int i = 0; i < left; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += X[i + size_t(left) * j] * M(k, j);
        Y[i + size_t(left) * k] = s;
      }
  }
  return y;
}

Vec kron_apply(const KronOperator& op, const Vec& x) {
  if (int(x.size()) != op.cols()) throw std::invalid_argument("kron_apply: shape mismatch");
  Vec y(op.rows(), 0.0);
  for (const auto& term : op.terms) {
    if (term.factors.size() != op.dims.size()) throw std::invalid_argument("kron_apply: term rank mismatch");
    Vec t = x;
    std::vector<int> cur = op.dims;
    for (size_t a = 0; a < term.factors.size(); ++a) {
      t = apply_axis(term.factors[a], t, cur, int(a));
      cur[a] = term.factors[a].r;
    }
    for (size_t i = 0; i < y.size(); ++i) y[i] += term.coeff * t[i];
  }
  return y;
}

Mat dense_kron(const Mat& A, const Mat& B) {
  Mat K(A.r * B.r, A.c * B.c);
  for (int i = 0; i < A.r; ++i)
    for (int j = 0; j < A.c; ++j)
      for (int bi = 0; bi < B.r; ++bi)
        for (int bj = 0; bj < B.c; ++bj) K(i * B.r + bi, j * B.c + bj) = A(i, j) * B(bi, bj);
  return K;
}

Mat kron_materialize(const KronOperator& op) {
  Mat out(op.rows(), op.cols());
  for (const auto& term : op.terms) {
    Mat K = term.factors.back();
    for (int a = int(term.factors.size()) - 2; a >= 0; --a) K = dense_kron(K, term.factors[a]);
    for (size_t k = 0; k < out.a.size(); ++k) out.a[k] += term.coeff * K.a[k];
  }
  return out;
}

// ---- ordering (src/ordering.cpp) ----------------------------------------------
Ordering natural_ordering(int n) {
  Ordering o;
  o.perm.resize(n);
  std::iota(o.perm.begin(), o.perm.end(), 0);
  o.group_offsets = {0, n};
  return o;
}

Ordering patch_ordering(const std::vector<DofLabel>& labels) {
  const int n = int(labels.size());
  for (const auto& l : labels)
    if (l.entity < 0) throw std::invalid_argument("patch_ordering: unclassified DOF");
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    const auto& la = labels[a];
    const auto& lb = labels[b];
    if (la.cls != lb.cls) return int(la.cls) < int(lb.cls);
    if (la.entity != lb.entity) return la.entity < lb.entity;
    return a < b;
  });
  Ordering o;
  o.perm = idx;
  o.group_offsets.push_back(0);
  for (int k = 1; k < n; ++k) {
    const auto& prev = labels[idx[k - 1]];
    const auto& cur = labels[idx[k]];
    const bool interior_pair = prev.cls == DofClass::Interior && cur.cls == DofClass::Interior;
    if (!interior_pair && (prev.cls != cur.cls || prev.entity != cur.entity)) o.group_offsets.push_back(k);
  }
  o.group_offsets.push_back(n);
  return o;
}

// ---- cholesky (src/cholesky.cpp:9-110) ----------------------------------------
CholFactor cholesky(const Csr& A, const Ordering& ord) {
  const int n = A.n;
  if (A.m != n) throw std::invalid_argument("cholesky: matrix not square");
  if (int(ord.perm.size()) != n) throw std::invalid_argument("cholesky: ordering size mismatch");
  std::vector<int> inv(n);
  for (int k = 0; k < n; ++k) inv[ord.perm[k]] = k;
  std::vector<int> parent(n, -1), flag(n), colcount(n, 1);
  for (int k = 0; k < n; ++k) {
    flag[k] = k;
    const int r = ord.perm[k];
    for (int64_t q = A.ptr[r]; q < A.ptr[r + 1]; ++q) {
      int j = inv[A.col[q]];
      for (; j < k && flag[j] != k; j = parent[j]) {
        if (parent[j] == -1) parent[j] = k;
        ++colcount[j];
        flag[j] = k;
      }
    }
  }
  CholFactor F;
  F.n = n;
  F.perm = ord.perm;
  F.colptr.assign(n + 1, 0);
  for (int j = 0; j < n; ++j) F.colptr[j + 1] = F.colptr[j] + colcount[j];
  F.rowind.assign(F.colptr[n], 0);
  F.values.assign(F.colptr[n], 0.0);
  std::vector<int64_t> cursor(F.colptr.begin(), F.colptr.end() - 1);
  std::vector<int> pattern(n), stack(n);
  Vec y(n, 0.0);
  std::fill(flag.begin(), flag.end(), -1);
  for (int k = 0; k < n; ++k) {
    flag[k] = k;
    double dk = 0.0;
    int top = n;
    const int r = ord.perm[k];
    for (int64_t q = A.ptr[r]; q < A.ptr[r + 1]; ++q) {
      const int j = inv[A.col[q]];
      if (j > k) continue;
      if (j == k) {
        dk = A.val[q];
        continue;
      }
      y[j] += A.val[q];
      int len = 0, i = j;
      for (; flag[i] != k; i = parent[i]) {
        stack[len++] = i;
        flag[i] = k;
      }
      while (len > 0) pattern[--top] = stack[--len];
    }
    for (int t = top; t < n; ++t) {
      const int j = pattern[t];
      const double yj = y[j];
      y[j] = 0.0;
      const double ljj = F.values[F.colptr[j]];
      const double lkj = yj / ljj;
      for (int64_t q = F.colptr[j] + 1; q < cursor[j]; ++q) y[F.rowind[q]] -= F.values[q] * lkj;
      F.flops += cursor[j] - F.colptr[j];
      F.rowind[cursor[j]] = k;
      F.values[cursor[j]] = lkj;
      ++cursor[j];
      dk -= lkj * lkj;
    }
    if (!(dk > 0.0)) throw std::runtime_error("cholesky: matrix not SPD at pivot " + std::to_string(k));
    F.rowind[F.colptr[k]] = k;
    F.values[F.colptr[k]] = std::sqrt(dk);
    cursor[k] = F.colptr[k] + 1;
  }
  return F;
}

Vec CholFactor::solve(const Vec& b) const {
  if (int(b.size()) != n) throw std::invalid_argument("CholFactor::solve: size mismatch");
  Vec y(n);
  for (int k = 0; k < n; ++k) y[k] = b[perm[k]];
  for (int j = 0; j < n; ++j) {
    const double xj = y[j] / values[colptr[j]];
    y[j] = xj;
    for (int64_t q = colptr[j] + 1; q < colptr[j + 1]; ++q) y[rowind[q]] -= values[q] * xj;
  }
  for (int j = n - 1; j >= 0; --j) {
    double acc = y[j];
    for (int64_t q = colptr[j] + 1; q < colptr[j + 1]; ++q) acc -= values[q] * y[rowind[q]];
    y[j] = acc / values[colptr[j]];
  }
  Vec x(n);
  for (int k = 0; k < n; ++k) x[perm[k]] = y[k];
  return x;
}

}  // namespace oracle
