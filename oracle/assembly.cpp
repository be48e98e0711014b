// TEST INFRASTRUCTURE ONLY — oracle restatement, see oracle.hpp header.
// L2: bundles, matrix-free operator, transformed (FDM) system, S / S^T
// transforms and the load vector (src/assembly.cpp), plus the [ext]
// per-cell coefficient and sum-factorised trilinear apply.
#include <cmath>
#include <stdexcept>

#include "oracle.hpp"

namespace oracle {

static Vec gather(const Vec& x, const std::vector<int>& dofs) {
  Vec v(dofs.size());
  for (size_t i = 0; i < dofs.size(); ++i) v[i] = x[dofs[i]];
  return v;
}
static void scatter_add(Vec& y, const std::vector<int>& dofs, const Vec& v) {
  for (size_t i = 0; i < dofs.size(); ++i) y[dofs[i]] += v[i];
}
// concat_dofs (src/assembly.cpp:16-23): cell DOFs of all components, component-major.
static std::vector<int> concat_dofs(const Discretization& d, int c) {
  if (d.ncomp == 1) return d.cell_dofs[c];
  std::vector<int> out;
  for (int ci = 0; ci < d.ncomp; ++ci) {
    const auto v = d.comp_dofs(ci, c);
    out.insert(out.end(), v.begin(), v.end());
  }
  return out;
}

Bundle1D make_bundle(int degree) {  // src/assembly.cpp:37-54, CG family
  Bundle1D b;
  b.degree = degree;
  b.ref = reference_operators(degree, BasisKind::GllNodal);
  b.fdm = fdm_basis(b.ref);
  const QuadratureRule quad = gauss_legendre_rule(degree + 1);
  Mat V, D;
  b.ref.eval(quad.points, V, D);
  b.C = Mat(degree + 1, degree + 1);
  for (int i = 0; i <= degree; ++i)
    for (int j = 0; j <= degree; ++j) {
      double s = 0.0;
      for (int q = 0; q < quad.size(); ++q) s += V(q, i) * quad.weights[q] * D(q, j);
      b.C(i, j) = s;
    }
  return b;
}

Vec GlobalOperator::apply(const Vec& x) const {  // src/assembly.cpp:56-88
  const Discretization& d = *disc;
  Vec xp = x;
  d.project_free(xp);
  Vec y(d.ndof, 0.0);
  for (int c = 0; c < d.mesh->num_cells(); ++c) {
    const CellTerm& term = cells[c];
    const auto dofs = concat_dofs(d, c);
    if (term.sumfact)
      scatter_add(y, dofs, sumfact_cell_apply(*bundle, d.dim(), term.G, gather(xp, dofs)));
    else if (term.dense.r > 0) {
      Vec u = gather(xp, dofs), v(dofs.size(), 0.0);
      for (int j = 0; j < term.dense.c; ++j)
        for (int i = 0; i < term.dense.r; ++i) v[i] += term.dense(i, j) * u[j];
      scatter_add(y, dofs, v);
    }
    if (term.has_kron) scatter_add(y, dofs, kron_apply(term.kron, gather(xp, dofs)));
    for (const auto& b : term.kron_blocks)
      scatter_add(y, d.comp_dofs(b.ci, c), kron_apply(b.op, gather(xp, d.comp_dofs(b.cj, c))));
  }
  for (const auto& ft : facets) {  // src/assembly.cpp:71-83
    const Facet& f = d.mesh->facets[ft.facet];
    for (const auto& b : ft.blocks)
      scatter_add(y, d.cell_dofs[f.cell[b.r]], kron_apply(b.op, gather(xp, d.cell_dofs[f.cell[b.s]])));
  }
  for (int i = 0; i < d.ndof; ++i)
    if (d.constrained[i]) y[i] = x[i];
  return y;
}

Csr GlobalOperator::assemble() const {  // src/assembly.cpp:90-129
  const Discretization& d = *disc;
  std::vector<Triplet> t;
  auto add_block = [&](const std::vector<int>& rows, const std::vector<int>& cols, const Mat& M) {
    for (int i = 0; i < M.r; ++i) {
      if (d.constrained[rows[i]]) continue;
      for (int j = 0; j < M.c; ++j)
        if (!d.constrained[cols[j]]) t.push_back({rows[i], cols[j], M(i, j)});
    }
  };
  for (int c = 0; c < d.mesh->num_cells(); ++c) {
    const CellTerm& term = cells[c];
    if (term.sumfact) throw std::invalid_argument("assemble: sum-factorised cell terms are matrix-free only");
    if (term.dense.r > 0) add_block(concat_dofs(d, c), concat_dofs(d, c), term.dense);
    if (term.has_kron) add_block(d.cell_dofs[c], d.cell_dofs[c], kron_materialize(term.kron));
    for (const auto& b : term.kron_blocks) add_block(d.comp_dofs(b.ci, c), d.comp_dofs(b.cj, c), kron_materialize(b.op));
  }
  for (const auto& ft : facets) {  // src/assembly.cpp:109-124
    const Facet& f = d.mesh->facets[ft.facet];
    for (const auto& b : ft.blocks)
      add_block(d.cell_dofs[f.cell[b.r]], d.cell_dofs[f.cell[b.s]], kron_materialize(b.op));
  }
  for (int i = 0; i < d.ndof; ++i)
    if (d.constrained[i]) t.push_back({i, i, 1.0});
  return csr_from_triplets(d.ndof, d.ndof, t);
}

KronOperator cell_matrix_cartesian(const ReferenceInterval& ref, const Vec& mu) {  // src/assembly.cpp:143-154
  const int d = int(mu.size());
  KronOperator op;
  op.dims.assign(d, ref.degree + 1);
  for (int a = 0; a < d; ++a) {
    KronTerm term;
    term.coeff = mu[a];
    for (int b = 0; b < d; ++b) term.factors.push_back(b == a ? ref.stiffness : ref.mass);
    op.terms.push_back(std::move(term));
  }
  return op;
}

static KronOperator affine_cell_operator(const Bundle1D& bundle, const Mat& G, int d, double kappa) {  // src/assembly.cpp:169-194
  KronOperator op;
  op.dims.assign(d, bundle.degree + 1);
  const Mat& A = bundle.ref.stiffness;
  const Mat& B = bundle.ref.mass;
  const Mat& C = bundle.C;
  const Mat Ct = C.transpose();
  for (int a = 0; a < d; ++a) {
    KronTerm term;
    term.coeff = kappa * G(a, a);
    for (int b = 0; b < d; ++b) term.factors.push_back(b == a ? A : B);
    op.terms.push_back(std::move(term));
  }
  for (int a = 0; a < d; ++a)
    for (int b = a + 1; b < d; ++b) {
      KronTerm t1, t2;
      t1.coeff = t2.coeff = kappa * G(a, b);
      for (int k = 0; k < d; ++k) {
        t1.factors.push_back(k == a ? Ct : (k == b ? C : B));
        t2.factors.push_back(k == a ? C : (k == b ? Ct : B));
      }
      op.terms.push_back(std::move(t1));
      op.terms.push_back(std::move(t2));
    }
  return op;
}

static Mat gradient_matrix(const ReferenceInterval& ref, const QuadratureRule& rule, int d, int axis) {  // src/assembly.cpp:160-167
  Mat V, D;
  ref.eval(rule.points, V, D);
  Mat out = (d - 1 == axis) ? D : V;
  for (int b = d - 2; b >= 0; --b) out = dense_kron(out, b == axis ? D : V);
  return out;
}

Mat cell_matrix_quadrature(const Mesh& mesh, int cell, const ReferenceInterval& ref) {  // src/assembly.cpp:198-215
  const int d = mesh.dim;
  const QuadratureRule rule = gauss_legendre_rule(ref.degree + 2);
  CellGeometry geom = cell_geometry(mesh, cell, rule);
  std::vector<Mat> grads;
  for (int a = 0; a < d; ++a) grads.push_back(gradient_matrix(ref, rule, d, a));
  const int nloc = grads[0].c, nq = grads[0].r;
  Mat A(nloc, nloc);
  Vec w(nq);
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      for (int q = 0; q < nq; ++q) w[q] = geom.quad_weights[q] * geom.metric[q](a, b);
      for (int j = 0; j < nloc; ++j)
        for (int i = 0; i < nloc; ++i) {
          double s = 0.0;
          for (int q = 0; q < nq; ++q) s += grads[a](q, i) * w[q] * grads[b](q, j);
          A(i, j) += s;
        }
    }
  Mat T = A.transpose();
  for (size_t k = 0; k < A.a.size(); ++k) A.a[k] = 0.5 * (A.a[k] + T.a[k]);
  return A;
}

// [ext] y = sum_{a,b} grad_a^T diag(G_ab) grad_b u, sum-factorised on the
// tensor GL(p+2) rule; equal to cell_matrix_quadrature(...) * u to rounding.
Vec sumfact_cell_apply(const Bundle1D& b, int d, const Vec& G, const Vec& u) {
  const int p = b.degree, q = p + 2;
  const QuadratureRule rule = gauss_legendre_rule(q);
  Mat V, D;
  b.ref.eval(rule.points, V, D);
  const Mat Vt = V.transpose(), Dt = D.transpose();
  std::vector<Vec> g(d);
  for (int a = 0; a < d; ++a) {
    Vec t = u;
    std::vector<int> dims(d, p + 1);
    for (int ax = 0; ax < d; ++ax) {
      t = apply_axis(ax == a ? D : V, t, dims, ax);
      dims[ax] = q;
    }
    g[a] = std::move(t);
  }
  int nq = 1;
  for (int a = 0; a < d; ++a) nq *= q;
  Vec y(u.size(), 0.0);
  for (int a = 0; a < d; ++a) {
    Vec f(nq, 0.0);
    for (int k = 0; k < nq; ++k)
      for (int bb = 0; bb < d; ++bb) f[k] += G[size_t(k) * d * d + a * d + bb] * g[bb][k];
    std::vector<int> dims(d, q);
    for (int ax = 0; ax < d; ++ax) {
      f = apply_axis(ax == a ? Dt : Vt, f, dims, ax);
      dims[ax] = p + 1;
    }
    for (size_t i = 0; i < y.size(); ++i) y[i] += f[i];
  }
  return y;
}

GlobalOperator poisson_operator(const Discretization& disc, const Bundle1D& bundle, int sumfact_threshold) {
  GlobalOperator op;  // src/assembly.cpp:230-243 with scalar_cell_term (:217-228)
  op.disc = &disc;
  op.bundle = &bundle;
  const Mesh& mesh = *disc.mesh;
  const QuadratureRule rule = gauss_legendre_rule(bundle.degree + 2);
  op.cells.resize(mesh.num_cells());
  for (int c = 0; c < mesh.num_cells(); ++c) {
    CellGeometry geom = cell_geometry(mesh, c, rule);
    const double kap = mesh.kappa(c);  // [ext] per-cell coefficient
    auto& term = op.cells[c];
    if (geom.kind == MapKind::Cartesian) {
      Vec mu = geom.mu;
      for (auto& m : mu) m *= kap;
      term.has_kron = true;
      term.kron = cell_matrix_cartesian(bundle.ref, mu);
    } else if (geom.kind == MapKind::Affine) {
      term.has_kron = true;
      term.kron = affine_cell_operator(bundle, geom.metric[0], mesh.dim, kap);
    } else if (disc.dofs_per_cell > sumfact_threshold) {
      const int d = mesh.dim;
      term.sumfact = true;
      term.G.resize(geom.dets.size() * d * d);
      for (size_t k = 0; k < geom.dets.size(); ++k)
        for (int a = 0; a < d; ++a)
          for (int b = 0; b < d; ++b) term.G[k * d * d + a * d + b] = kap * geom.quad_weights[k] * geom.metric[k](a, b);
    } else {
      term.dense = cell_matrix_quadrature(mesh, c, bundle.ref);
      if (kap != 1.0)
        for (auto& v : term.dense.a) v *= kap;
    }
  }
  return op;
}

Vec TransformedSystem::mode_signs(int cell) const {  // src/assembly.cpp:293-306
  const Discretization& d = *disc;
  Vec s(d.dofs_per_cell, 1.0);
  const auto& flips = d.cell_mode_flip_axis[cell];
  for (int lat = 0; lat < d.dofs_per_cell; ++lat) {
    if (flips[lat] < 0) continue;
    const int axis = flips[lat];
    int idx = lat;
    for (int a = 0; a < axis; ++a) idx /= d.degree + 1;
    idx %= d.degree + 1;
    s[lat] = parity[idx];
  }
  return s;
}

// Structural value/pattern of one cell block sum_a mu_a (x)_b (b==a ? A_t : B_t)
// at lattice pair (r, c); returns false when no term stores the entry
// (src/assembly.cpp:263-270 with sparse_kron, src/kron.cpp:65-79).
static bool cell_entry(const FdmBasis& f, int d, int p, const Vec& mu, int r, int c, double& val) {
  int ri[3] = {0, 0, 0}, ci[3] = {0, 0, 0};
  for (int a = 0, rr = r, cc = c; a < d; ++a, rr /= p + 1, cc /= p + 1) {
    ri[a] = rr % (p + 1);
    ci[a] = cc % (p + 1);
  }
  bool any = false;
  double sum = 0.0;
  for (int a = 0; a < d; ++a) {
    bool present = true;
    double prod = mu[a];
    // sparse_kron chain builds F_{d-1} (x) ... (x) F_0: multiply from the top axis down.
    for (int b = d - 1; b >= 0; --b) {
      const PatMat& F = (b == a) ? f.A_t : f.B_t;
      if (!F.has(ri[b], ci[b])) {
        present = false;
        break;
      }
    }
    if (!present) continue;
    double kv = 1.0;
    {
      const PatMat& Ftop = (d - 1 == a) ? f.A_t : f.B_t;
      kv = Ftop.val(ri[d - 1], ci[d - 1]);
      for (int b = d - 2; b >= 0; --b) kv *= ((b == a) ? f.A_t : f.B_t).val(ri[b], ci[b]);
    }
    sum = any ? sum + kv * prod : kv * prod;
    any = true;
  }
  val = sum;
  return any;
}

// Column lists of the A_t pattern per 1D index (superset of B_t's pattern).
static std::vector<std::vector<int>> pattern_cols(const PatMat& A) {
  std::vector<std::vector<int>> cols(A.rows());
  for (int i = 0; i < A.rows(); ++i)
    for (int j = 0; j < A.cols(); ++j)
      if (A.has(i, j)) cols[i].push_back(j);
  return cols;
}

template <class Fn>
static void for_each_cell_entry(const FdmBasis& f, int d, int p, const Vec& mu, Fn&& fn) {
  const auto cols = pattern_cols(f.A_t);
  int npc = 1;
  for (int a = 0; a < d; ++a) npc *= p + 1;
  for (int r = 0; r < npc; ++r) {
    int ri[3] = {0, 0, 0};
    for (int a = 0, rr = r; a < d; ++a, rr /= p + 1) ri[a] = rr % (p + 1);
    const auto& c0 = cols[ri[0]];
    const auto& c1 = d > 1 ? cols[ri[1]] : c0;
    const std::vector<int> zero{0};
    const auto& c2 = d > 2 ? cols[ri[2]] : zero;
    for (int k2 : c2)
      for (int k1 : c1)
        for (int k0 : c0) {
          const int c = k0 + (p + 1) * (k1 + (p + 1) * k2);
          double v;
          if (cell_entry(f, d, p, mu, r, c, v)) fn(r, c, v);
        }
  }
}

void cell_transformed_entries(const FdmBasis& f, int d, int p, const Vec& mu,
                              const std::function<void(int, int, double)>& fn) {
  for_each_cell_entry(f, d, p, mu, fn);
}

TransformedSystem transformed_poisson(const Discretization& disc, const Bundle1D& bundle, bool eliminate,
                                      bool build_global) {  // src/assembly.cpp:245-291
  TransformedSystem sys;
  sys.disc = &disc;
  sys.S = bundle.fdm.S;
  sys.parity = bundle.fdm.parity;
  sys.inv_multiplicity.resize(disc.ndof);
  for (int i = 0; i < disc.ndof; ++i) sys.inv_multiplicity[i] = 1.0 / disc.multiplicity[i];
  const Mesh& mesh = *disc.mesh;
  const int d = disc.dim(), p = disc.degree;
  const QuadratureRule rule = gauss_legendre_rule(bundle.degree + 2);
  sys.cell_mu.resize(mesh.num_cells());
  for (int c = 0; c < mesh.num_cells(); ++c) {
    CellGeometry geom = cell_geometry(mesh, c, rule);
    sys.cell_mu[c] = geom.mu;
    for (auto& m : sys.cell_mu[c]) m *= mesh.kappa(c);  // [ext]
  }
  if (!build_global) return sys;
  std::vector<Triplet> trips;
  for (int c = 0; c < mesh.num_cells(); ++c) {
    const auto& modes = disc.cell_modes[c];
    const Vec sgn = sys.mode_signs(c);
    for_each_cell_entry(bundle.fdm, d, p, sys.cell_mu[c], [&](int r, int col, double v) {
      const bool drop = eliminate && (disc.constrained[modes[r]] || disc.constrained[modes[col]]);
      if (!drop) trips.push_back({modes[r], modes[col], sgn[r] * sgn[col] * v});
    });
  }
  if (eliminate)
    for (int i = 0; i < disc.ndof; ++i)
      if (disc.constrained[i]) trips.push_back({i, i, 1.0});
  sys.At = csr_from_triplets(disc.ndof, disc.ndof, trips);
  return sys;
}

Csr patch_matrix(const TransformedSystem& sys, const Bundle1D& bundle, int v, const std::vector<int>& dofs) {
  const Discretization& disc = *sys.disc;
  const int d = disc.dim(), p = disc.degree;
  std::vector<int> where(disc.ndof, -1);
  for (size_t k = 0; k < dofs.size(); ++k) where[dofs[k]] = int(k);
  std::vector<Triplet> trips;
  for (int c : disc.mesh->vertex_cells[v]) {
    const auto& modes = disc.cell_modes[c];
    const Vec sgn = sys.mode_signs(c);
    for_each_cell_entry(bundle.fdm, d, p, sys.cell_mu[c], [&](int r, int col, double val) {
      const int wr = where[modes[r]], wc = where[modes[col]];
      if (wr >= 0 && wc >= 0) trips.push_back({wr, wc, sgn[r] * sgn[col] * val});
    });
  }
  return csr_from_triplets(int(dofs.size()), int(dofs.size()), trips);
}

Vec TransformedSystem::apply_S(const Vec& modes) const {  // src/assembly.cpp:308-324
  const Discretization& d = *disc;
  Vec x = modes;
  d.project_free(x);
  Vec y(d.ndof, 0.0);
  std::vector<int> dims(d.dim(), d.degree + 1);
  for (int ci = 0; ci < d.ncomp; ++ci)
  for (int c = 0; c < d.mesh->num_cells(); ++c) {
    Vec v = gather(x, d.comp_modes(ci, c));
    const Vec s = mode_signs(c);
    for (size_t i = 0; i < v.size(); ++i) v[i] *= s[i];
    for (int a = 0; a < d.dim(); ++a) v = apply_axis(S, v, dims, a);
    scatter_add(y, d.comp_dofs(ci, c), v);
  }
  for (int i = 0; i < d.ndof; ++i) y[i] *= inv_multiplicity[i];
  d.project_free(y);
  return y;
}

Vec TransformedSystem::apply_St(const Vec& nodal) const {  // src/assembly.cpp:326-342
  const Discretization& d = *disc;
  Vec x(d.ndof);
  for (int i = 0; i < d.ndof; ++i) x[i] = nodal[i] * inv_multiplicity[i];
  d.project_free(x);
  Vec y(d.ndof, 0.0);
  std::vector<int> dims(d.dim(), d.degree + 1);
  const Mat St = S.transpose();
  for (int ci = 0; ci < d.ncomp; ++ci)
  for (int c = 0; c < d.mesh->num_cells(); ++c) {
    Vec v = gather(x, d.comp_dofs(ci, c));
    for (int a = 0; a < d.dim(); ++a) v = apply_axis(St, v, dims, a);
    const Vec s = mode_signs(c);
    for (size_t i = 0; i < v.size(); ++i) v[i] *= s[i];
    scatter_add(y, d.comp_modes(ci, c), v);
  }
  d.project_free(y);
  return y;
}

Vec load_vector(const Discretization& disc, const Bundle1D& bundle,
                const std::function<double(const std::array<double, 3>&)>& f) {  // src/assembly.cpp:344-373
  const Mesh& mesh = *disc.mesh;
  const int d = mesh.dim;
  const QuadratureRule rule = gauss_legendre_rule(bundle.degree + 2);
  Mat V, D;
  bundle.ref.eval(rule.points, V, D);
  const Mat Vt = V.transpose();
  const int nq1 = rule.size();
  Vec out(disc.ndof, 0.0);
  for (int c = 0; c < mesh.num_cells(); ++c) {
    CellGeometry geom = cell_geometry(mesh, c, rule);
    const int nq = int(geom.dets.size());
    Vec g(nq), xhat(d);
    for (int q = 0; q < nq; ++q) {
      int qq = q;
      for (int a = 0; a < d; ++a) {
        xhat[a] = rule.points[qq % nq1];
        qq /= nq1;
      }
      g[q] = geom.quad_weights[q] * geom.dets[q] * f(cell_map(mesh, c, xhat));
    }
    std::vector<int> dims(d, nq1);
    for (int a = 0; a < d; ++a) {
      g = apply_axis(Vt, g, dims, a);
      dims[a] = bundle.degree + 1;
    }
    scatter_add(out, disc.cell_dofs[c], g);
  }
  return out;
}

}  // namespace oracle
