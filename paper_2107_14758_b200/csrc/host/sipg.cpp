// Host setup of the symmetric interior-penalty DG variant of the path
// (src/sipg.cpp, include/fdmstar/sipg.hpp): the GL-nodal bundle with the FDM
// modes in GL representation, dq_space maps, the facet list with its
// penalty data, the DG vertex stars ((2p+2)^d DOFs) and the
// continuous Q1 coarse level with the DG prolongation -- the inputs of the
// two-level DG solver of tests/test_sipg.cpp:184-197 -- for the device path
// (fdmgpu_set_sipg).  Cartesian meshes (the reference's Kronecker facet path,
// src/sipg.cpp:200-248).
#include <cmath>
#include <stdexcept>

#include "fdm_host.hpp"

namespace fdmgpu::host {

double sipg_default_eta(int p, int d) { return (p + 1.0) * (p + d); }  // src/sipg.cpp:7

namespace {

// sum_q M(q,i) w_q N(q,j), symmetrised (src/reference_interval.cpp:115-121).
Dense sym_gram(const Dense& M, const Vec& w, const Dense& N) {
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

// Endpoint traces of a nodal basis: values and outward normal derivatives
// (row 0 at x = -1 negated), 2 x (p+1) column-major (src/reference_interval.cpp:124-128).
void traces(const Vec& nodes, Dense& tv, Dense& tnd) {
  Vec ends{-1.0, 1.0};
  lagrange_eval(nodes, ends, tv, tnd);
  for (int j = 0; j < tnd.c; ++j) tnd(0, j) = -tnd(0, j);
}

}  // namespace

// make_bundle(Family1D::DG, p) (src/assembly.cpp:37-54): GL-nodal reference
// interval, the FDM basis of the GLL interval re-expressed at the GL nodes
// (to_gl_representation, src/fdm_basis.cpp:89-101: S replaced, A_t, B_t,
// deriv_traces and parity unchanged).
Basis1D make_bundle_dg(int p) {
  Basis1D b = make_bundle(p);  // GLL FDM modes, A_t / B_t, lambda, parity
  const int n1 = p + 1;
  Dense gtv, gtnd;
  traces(b.nodes, gtv, gtnd);
  b.dtr = Dense(2, n1);  // fdm.deriv_traces = trace_normal_derivs(GLL) * S (src/fdm_basis.cpp:78)
  for (int e = 0; e < 2; ++e)
    for (int j = 0; j < n1; ++j) {
      double s = 0.0;
      for (int i = 0; i < n1; ++i) s += gtnd(e, i) * b.S(i, j);
      b.dtr(e, j) = s;
    }
  Vec gp, gw;
  gauss_legendre(n1, gp, gw);
  Dense Vi, Di;
  lagrange_eval(b.nodes, gp, Vi, Di);  // GLL basis at the GL points
  Dense Sgl(n1, n1);
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      double s = 0.0;
      for (int k = 0; k < n1; ++k) s += Vi(i, k) * b.S(k, j);
      Sgl(i, j) = s;
    }
  b.S = Sgl;
  b.nodes = gp;  // GL collocation nodes (reference_operators(p, GlNodal))
  Dense V, D;
  lagrange_eval(b.nodes, gp, V, D);
  b.A_hat = sym_gram(D, gw, D);
  b.B_hat = sym_gram(V, gw, V);
  traces(b.nodes, b.tv, b.tnd);
  b.dg = true;
  return b;
}

std::unique_ptr<Problem> make_dg_problem(int dim, int n, int p, double eta, bool skip_boundary) {
  if (dim < 2 || dim > 3 || n < 1 || p < 1) throw std::invalid_argument("make_dg_problem: bad dim / n / p");
  auto pb = std::make_unique<Problem>();
  pb->config = 0;
  pb->dim = dim;
  pb->n = n;
  pb->p = p;
  pb->dg = true;
  pb->eta = eta < 0 ? sipg_default_eta(p, dim) : eta;
  pb->mesh = cartesian_mesh(dim, std::vector<int>(dim, n), std::vector<double>(dim, 1.0));
  pb->basis = make_bundle_dg(p);
  pb->space = q_space(pb->mesh, p, /*dg=*/true);
  pb->space.mesh = &pb->mesh;
  const int nc = pb->mesh.num_cells(), ncorner = 1 << dim, npc = pb->space.npc, n1 = p + 1;
  pb->cell_kind.resize(nc);
  pb->cell_mu.resize(size_t(nc) * dim);
  pb->cell_xyz.resize(size_t(nc) * ncorner * 3);
  pb->cell_kappa.assign(nc, 1.0);
  // load_vector with f = 1 (src/assembly.cpp, tests/test_sipg.cpp:184-197):
  // b_i = |det J| prod_a w_{i_a} for the GL-nodal basis (exact at GL(p+1))
  Vec gp, gw;
  gauss_legendre(n1, gp, gw);
  pb->rhs.assign(pb->space.ndof, 0.0);
  for (int c = 0; c < nc; ++c) {
    CellCoeffs cc = cell_coeffs(pb->mesh, c, pb->basis);
    if (cc.kind != MapKind::Cartesian) throw std::invalid_argument("SIPG device path: Cartesian cells only");
    pb->cell_kind[c] = 0;
    double det = 1.0;
    const auto& v0 = pb->mesh.vertices[pb->mesh.cells[c][0]];
    for (int a = 0; a < dim; ++a) {
      pb->cell_mu[size_t(c) * dim + a] = cc.mu[a];
      det *= 0.5 * (pb->mesh.vertices[pb->mesh.cells[c][1 << a]][a] - v0[a]);
    }
    for (int b = 0; b < ncorner; ++b)
      for (int r = 0; r < 3; ++r)
        pb->cell_xyz[(size_t(c) * ncorner + b) * 3 + r] = pb->mesh.vertices[pb->mesh.cells[c][b]][r];
    for (int l = 0; l < npc; ++l) {
      double w = det;
      for (int a = 0, t = l; a < dim; ++a, t /= n1) w *= gw[t % n1];
      pb->rhs[pb->space.cell_dofs[size_t(c) * npc + l]] = w;
    }
  }
  pb->skip_boundary = skip_boundary;
  pb->patches = vertex_patches(pb->space, skip_boundary);
  pb->coarse = build_coarse(pb->mesh, pb->space, pb->basis);  // Q1 hats at the GL nodes
  return pb;
}

}  // namespace fdmgpu::host
