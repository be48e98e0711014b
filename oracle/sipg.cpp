// TEST INFRASTRUCTURE ONLY — oracle restatement, see oracle.hpp header.
// Symmetric interior-penalty DG (src/sipg.cpp) on Cartesian meshes: the
// GL-nodal bundle with the FDM basis in GL representation, the facet
// matrices (nodal and transformed), the true-form operator's Kronecker path
// and the transformed system feeding the vertex-star PatchSolver.  Not
// restated: the quadrature facet blocks of general 2D cells and the
// reflected mass of flipped facets (non-Cartesian meshes).
#include <stdexcept>

#include "oracle.hpp"

namespace oracle {

double sipg_default_eta(int p, int d) { return (p + 1.0) * (p + d); }  // src/sipg.cpp:7

FdmBasis to_gl_representation(const FdmBasis& fdm, const ReferenceInterval& gll) {  // src/fdm_basis.cpp:89-101
  FdmBasis out = fdm;
  const QuadratureRule gl = gauss_legendre_rule(fdm.degree + 1);
  Mat V, D;
  gll.eval(gl.points, V, D);
  out.S = matmul(V, fdm.S);
  return out;
}

Bundle1D make_bundle_dg(int degree) {  // src/assembly.cpp:37-54, DG family
  Bundle1D b;
  b.degree = degree;
  const ReferenceInterval gll = reference_operators(degree, BasisKind::GllNodal);
  b.ref = reference_operators(degree, BasisKind::GlNodal);
  b.fdm = to_gl_representation(fdm_basis(gll), gll);
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

Mat sipg_facet_dirichlet(const ReferenceInterval& ref, double mu_e, double eta, int side) {  // src/sipg.cpp:20-25
  const int n = ref.degree + 1, e = side > 0 ? 1 : 0;
  Mat E(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double ti = ref.trace_values(e, i), tj = ref.trace_values(e, j);
      const double di = ref.trace_normal_derivs(e, i), dj = ref.trace_normal_derivs(e, j);
      E(i, j) = mu_e * (eta * ti * tj - ti * dj - di * tj);
    }
  return E;
}

Mat sipg_facet_interior(const ReferenceInterval& ref, double mu0, double mu1, double eta, int side0,
                        int side1) {  // src/sipg.cpp:27-45
  const int n = ref.degree + 1;
  const double mu[2] = {mu0, mu1};
  const int sides[2] = {side0 > 0 ? 1 : 0, side1 > 0 ? 1 : 0};
  Mat E(2 * n, 2 * n);
  for (int r = 0; r < 2; ++r)
    for (int s = 0; s < 2; ++s) {
      const double sign = r == s ? 0.5 : -0.5;
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          const double tr = ref.trace_values(sides[r], i), ts = ref.trace_values(sides[s], j);
          const double dr = ref.trace_normal_derivs(sides[r], i), ds = ref.trace_normal_derivs(sides[s], j);
          E(r * n + i, s * n + j) = sign * (eta * (mu0 + mu1) * tr * ts - mu[s] * tr * ds - mu[r] * dr * ts);
        }
    }
  return E;
}

namespace {
// Eigen setFromTriplets on a (p+1)^2 matrix: duplicates summed, every listed
// position stored (explicit zeros too).
void add_trip(PatMat& M, int i, int j, double v) {
  M.val(i, j) += v;
  M.nz[i + size_t(M.val.r) * j] = 1;
}
PatMat empty_pat(int n) {
  PatMat M;
  M.val = Mat(n, n);
  M.nz.assign(size_t(n) * n, 0);
  return M;
}
}  // namespace

PatMat sipg_facet_dirichlet_t(const FdmBasis& fdm, double mu_e, double eta, int side) {  // src/sipg.cpp:47-62
  const int p = fdm.degree, tau = side > 0 ? p : 0, e = side > 0 ? 1 : 0;
  PatMat E = empty_pat(p + 1);
  add_trip(E, tau, tau, eta * mu_e);
  for (int j = 0; j <= p; ++j) {
    add_trip(E, tau, j, -mu_e * fdm.deriv_traces(e, j));
    add_trip(E, j, tau, -mu_e * fdm.deriv_traces(e, j));
  }
  return E;
}

PatMat sipg_facet_interior_t(const FdmBasis& fdm, double mu0, double mu1, double eta, int side0, int side1,
                             int block_r, int block_s) {  // src/sipg.cpp:64-87
  const int p = fdm.degree;
  const double mu[2] = {mu0, mu1};
  const int sides[2] = {side0, side1};
  const int tau_r = sides[block_r] > 0 ? p : 0, tau_s = sides[block_s] > 0 ? p : 0;
  const int er = sides[block_r] > 0 ? 1 : 0, es = sides[block_s] > 0 ? 1 : 0;
  const double sign = block_r == block_s ? 0.5 : -0.5;
  PatMat E = empty_pat(p + 1);
  add_trip(E, tau_r, tau_s, sign * eta * (mu0 + mu1));
  for (int j = 0; j <= p; ++j) {
    add_trip(E, tau_r, j, -sign * mu[block_s] * fdm.deriv_traces(es, j));
    add_trip(E, j, tau_s, -sign * mu[block_r] * fdm.deriv_traces(er, j));
  }
  return E;
}

namespace {

// Facets of a Cartesian-topology mesh must agree on the normal axis and not flip.
void check_cartesian_facet(const Mesh& mesh, const Facet& f, const std::vector<CellGeometry>& geoms) {
  for (int r = 0; r < f.ncells(); ++r)
    if (geoms[f.cell[r]].kind != MapKind::Cartesian)
      throw std::invalid_argument("oracle SIPG: non-Cartesian facets are not restated");
  if (f.ncells() == 2 && (f.axis[0] != f.axis[1] || f.tangential_flip))
    throw std::invalid_argument("oracle SIPG: flipped / rotated facets are not restated");
  (void)mesh;
}

// Entries of the sparse_kron chain F_{d-1} (x) ... (x) F_0 (src/sipg.cpp:280-284), in lattice
// indices (axis 0 fastest); an entry exists when every factor stores its 1D entry.
template <class Fn>
void kron_entries(const std::vector<const PatMat*>& F, int n1, Fn&& fn) {
  const int d = int(F.size());
  int npc = 1;
  for (int a = 0; a < d; ++a) npc *= n1;
  for (int r = 0; r < npc; ++r)
    for (int c = 0; c < npc; ++c) {
      double v = 1.0;
      bool present = true;
      for (int a = d - 1, rr = r, cc = c; a >= 0 && present; --a) {
        int pa = 1;
        for (int b = 0; b < a; ++b) pa *= n1;
        const int ri = (rr / pa) % n1, ci = (cc / pa) % n1;
        if (!F[a]->has(ri, ci)) present = false;
        else v *= F[a]->val(ri, ci);
      }
      if (present) fn(r, c, v);
    }
}

}  // namespace

GlobalOperator dg_poisson_operator(const Discretization& disc, const Bundle1D& bundle, double eta) {  // src/sipg.cpp:176-250
  GlobalOperator op = poisson_operator(disc, bundle);  // scalar_cell_term per cell (src/sipg.cpp:186-190)
  const Mesh& mesh = *disc.mesh;
  const int d = mesh.dim, n1 = bundle.degree + 1;
  const QuadratureRule rule = gauss_legendre_rule(bundle.degree + 2);
  std::vector<CellGeometry> geoms;
  for (int c = 0; c < mesh.num_cells(); ++c) geoms.push_back(cell_geometry(mesh, c, rule));
  for (int fi = 0; fi < int(mesh.facets.size()); ++fi) {
    const Facet& f = mesh.facets[fi];
    if (f.tag == FacetTag::Neumann) continue;
    check_cartesian_facet(mesh, f, geoms);
    GlobalOperator::FacetTerm term;
    term.facet = fi;
    const int axis = f.axis[0];
    if (f.ncells() == 1) {
      const Mat E = sipg_facet_dirichlet(bundle.ref, geoms[f.cell[0]].mu[axis], eta, f.side[0]);
      KronOperator kop;
      kop.dims.assign(d, n1);
      KronTerm kt;
      for (int a = 0; a < d; ++a) kt.factors.push_back(a == axis ? E : bundle.ref.mass);
      kop.terms.push_back(std::move(kt));
      term.blocks.push_back({0, 0, std::move(kop)});
    } else {
      const Mat E = sipg_facet_interior(bundle.ref, geoms[f.cell[0]].mu[axis], geoms[f.cell[1]].mu[axis], eta,
                                        f.side[0], f.side[1]);
      for (int r = 0; r < 2; ++r)
        for (int s = 0; s < 2; ++s) {
          Mat Ers(n1, n1);
          for (int j = 0; j < n1; ++j)
            for (int i = 0; i < n1; ++i) Ers(i, j) = E(r * n1 + i, s * n1 + j);
          KronOperator kop;
          kop.dims.assign(d, n1);
          KronTerm kt;
          for (int a = 0; a < d; ++a) kt.factors.push_back(a == axis ? Ers : bundle.ref.mass);
          kop.terms.push_back(std::move(kt));
          term.blocks.push_back({r, s, std::move(kop)});
        }
    }
    op.facets.push_back(std::move(term));
  }
  return op;
}

TransformedSystem transformed_dg_poisson(const Discretization& disc, const Bundle1D& bundle,
                                         double eta) {  // src/sipg.cpp:252-364
  TransformedSystem sys;
  sys.disc = &disc;
  sys.S = bundle.fdm.S;
  sys.parity = bundle.fdm.parity;
  sys.inv_multiplicity.resize(disc.ndof);
  for (int i = 0; i < disc.ndof; ++i) sys.inv_multiplicity[i] = 1.0 / disc.multiplicity[i];
  const Mesh& mesh = *disc.mesh;
  const int d = mesh.dim, p = bundle.degree, n1 = p + 1;
  const QuadratureRule rule = gauss_legendre_rule(bundle.degree + 2);
  std::vector<CellGeometry> geoms;
  for (int c = 0; c < mesh.num_cells(); ++c) geoms.push_back(cell_geometry(mesh, c, rule));
  sys.cell_mu.resize(mesh.num_cells());
  std::vector<Triplet> trips;
  for (int c = 0; c < mesh.num_cells(); ++c) {
    sys.cell_mu[c] = geoms[c].mu;
    const auto& dofs = disc.cell_dofs[c];
    cell_transformed_entries(bundle.fdm, d, p, geoms[c].mu,
                             [&](int r, int col, double v) { trips.push_back({dofs[r], dofs[col], v}); });
  }
  const PatMat& Bt = bundle.fdm.B_t;
  for (int fi = 0; fi < int(mesh.facets.size()); ++fi) {
    const Facet& f = mesh.facets[fi];
    if (f.tag == FacetTag::Neumann) continue;
    check_cartesian_facet(mesh, f, geoms);
    const int axis = f.axis[0];
    std::vector<const PatMat*> fac(d, &Bt);
    if (f.ncells() == 1) {
      const PatMat E = sipg_facet_dirichlet_t(bundle.fdm, geoms[f.cell[0]].mu[axis], eta, f.side[0]);
      fac[axis] = &E;
      const auto& dofs = disc.cell_dofs[f.cell[0]];
      kron_entries(fac, n1, [&](int r, int c, double v) { trips.push_back({dofs[r], dofs[c], v}); });
    } else {
      const double mu0 = geoms[f.cell[0]].mu[f.axis[0]], mu1 = geoms[f.cell[1]].mu[f.axis[1]];
      for (int r = 0; r < 2; ++r)
        for (int s = 0; s < 2; ++s) {
          const PatMat E = sipg_facet_interior_t(bundle.fdm, mu0, mu1, eta, f.side[0], f.side[1], r, s);
          fac[axis] = &E;
          const auto& rd = disc.cell_dofs[f.cell[r]];
          const auto& sd = disc.cell_dofs[f.cell[s]];
          kron_entries(fac, n1, [&](int i, int j, double v) { trips.push_back({rd[i], sd[j], v}); });
        }
    }
  }
  sys.At = csr_from_triplets(disc.ndof, disc.ndof, trips);
  return sys;
}

}  // namespace oracle
