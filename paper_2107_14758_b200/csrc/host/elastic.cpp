// Host setup of the linear-elasticity variant of the path (src/elasticity.cpp):
// the vector Q_p space as dim blocks of the scalar space (vector_q_space,
// src/discretization.cpp:313-318), the vector star lists, the body-force
// load (vector_load), and the vector Q1 coarse level with the true form
// (build_elasticity_twolevel, src/elasticity.cpp:204-229).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "fdm_host.hpp"

namespace fdmgpu::host {

Patches vector_patches(const Space& s, const Patches& sp, int ncomp) {
  const int64_t ns = s.ndof;
  Patches P;
  P.vertex = sp.vertex;
  P.cells = sp.cells;
  P.colour = sp.colour;
  P.ptr.push_back(0);
  std::vector<int32_t> dv;
  for (size_t j = 0; j < sp.vertex.size(); ++j) {
    dv.clear();
    for (int ci = 0; ci < ncomp; ++ci)
      for (int64_t k = sp.ptr[j]; k < sp.ptr[j + 1]; ++k) dv.push_back(int32_t(sp.dofs[k] + ci * ns));
    // patch_ordering (src/ordering.cpp:17-45) on the vector labels: a DOF's
    // label is its scalar entity's, whatever the component.
    std::vector<int32_t> idx(dv.size());
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
      const int ga = int(dv[a] % ns), gb = int(dv[b] % ns);
      const int ca = s.label_cls[ga], cb = s.label_cls[gb];
      if (ca != cb) return ca < cb;
      const int ea = s.label_entity[ga], eb = s.label_entity[gb];
      if (ea != eb) return ea < eb;
      return a < b;
    });
    P.dofs.insert(P.dofs.end(), dv.begin(), dv.end());
    P.perm.insert(P.perm.end(), idx.begin(), idx.end());
    P.ptr.push_back(int64_t(P.dofs.size()));
  }
  return P;
}

void rebuild_patches(Problem& pb, bool skip_boundary) {
  pb.skip_boundary = skip_boundary;
  pb.patches = vertex_patches(pb.space, skip_boundary);
  if (pb.ncomp > 1) pb.patches = vector_patches(pb.space, pb.patches, pb.ncomp);
}

namespace {

// bundle.C = V^T diag(w) D on GL(p+1) (src/assembly.cpp:49-52), column-major.
std::vector<double> bundle_C(const Basis1D& b) {
  const int n1 = b.p + 1;
  Vec pts, wts;
  gauss_legendre(n1, pts, wts);
  Dense V, D;
  lagrange_eval(b.nodes, pts, V, D);
  std::vector<double> C(size_t(n1) * n1);
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      double s = 0.0;
      for (int q = 0; q < n1; ++q) s += V(q, i) * wts[q] * D(q, j);
      C[i + size_t(n1) * j] = s;
    }
  return C;
}

// Cell half-extents of an axis-aligned cell (src/geometry.cpp:91-97 lengths).
std::array<double, 3> half_extents(const Mesh& m, int c) {
  std::array<double, 3> L{1.0, 1.0, 1.0};
  const auto& v0 = m.vertices[m.cells[c][0]];
  for (int a = 0; a < m.dim; ++a) L[a] = 0.5 * (m.vertices[m.cells[c][1 << a]][a] - v0[a]);
  return L;
}

// Vector Q1 coarse level: elasticity_primal_operator at p = 1 (Kronecker
// blocks, Cartesian cells), assembled (constrained rows / columns dropped,
// identity on the diagonal, src/assembly.cpp:90-129) and inverted; the
// prolongation is the scalar one per component block.
Coarse build_coarse_elastic(const Problem& pb) {
  const Mesh& m = pb.mesh;
  const int d = m.dim, nd = pb.ncomp;
  const Coarse sc = build_coarse(m, pb.space, pb.basis);
  const int ncs = sc.ndof, nc = nd * ncs, npc = 1 << d;
  const Basis1D b1 = make_bundle(1);
  const std::vector<double> C1 = bundle_C(b1);
  auto Cx = [&](int i, int j) { return C1[i + 2 * j]; };
  auto Ctx = [&](int i, int j) { return C1[j + 2 * i]; };
  std::vector<double> A(size_t(nc) * nc, 0.0);
  std::vector<uint8_t> con(nc);
  for (int ci = 0; ci < nd; ++ci)
    for (int i = 0; i < ncs; ++i) con[ci * ncs + i] = sc.constrained[i];
  const double lmu = pb.lame_mu, llam = pb.lame_lambda;
  for (int c = 0; c < m.num_cells(); ++c) {
    const auto L = half_extents(m, c);
    double prod = 1.0;
    for (int a = 0; a < d; ++a) prod *= L[a];
    double mu[3];
    for (int a = 0; a < d; ++a) mu[a] = prod / (L[a] * L[a]);
    const int32_t* cd = &sc.cell_dofs[size_t(c) * npc];
    for (int bi = 0; bi < nd; ++bi)
      for (int bj = 0; bj < nd; ++bj) {
        // entry (r, s) of the (bi, bj) block: sum over Kronecker terms of coeff * prod_b F_b(r_b, s_b)
        for (int r = 0; r < npc; ++r) {
          const int gr = bi * ncs + cd[r];
          if (con[gr]) continue;
          for (int s = 0; s < npc; ++s) {
            const int gs = bj * ncs + cd[s];
            if (con[gs]) continue;
            double v = 0.0;
            if (bi == bj) {
              for (int a = 0; a < d; ++a) {
                double t = (lmu + (a == bi ? lmu + llam : 0.0)) * mu[a];
                for (int b = 0; b < d; ++b) {
                  const int rb = (r >> b) & 1, sb = (s >> b) & 1;
                  t *= b == a ? b1.A_hat(rb, sb) : b1.B_hat(rb, sb);
                }
                v += t;
              }
            } else {
              const double scale = prod / (L[bi] * L[bj]);
              double t1 = lmu * scale, t2 = llam * scale;
              for (int b = 0; b < d; ++b) {
                const int rb = (r >> b) & 1, sb = (s >> b) & 1;
                t1 *= b == bi ? Cx(rb, sb) : (b == bj ? Ctx(rb, sb) : b1.B_hat(rb, sb));
                t2 *= b == bi ? Ctx(rb, sb) : (b == bj ? Cx(rb, sb) : b1.B_hat(rb, sb));
              }
              v = t1 + t2;
            }
            A[size_t(gr) * nc + gs] += v;
          }
        }
      }
  }
  for (int i = 0; i < nc; ++i)
    if (con[i]) A[size_t(i) * nc + i] = 1.0;
  Coarse C;
  C.ndof = nc;
  C.inverse = dense_spd_inverse(A, nc);
  const int64_t ns = pb.space.ndof;
  C.P_ptr.assign(1, 0);
  for (int ci = 0; ci < nd; ++ci)
    for (int64_t i = 0; i < ns; ++i) {
      for (int64_t q = sc.P_ptr[i]; q < sc.P_ptr[i + 1]; ++q) {
        C.P_col.push_back(sc.P_col[q] + ci * ncs);
        C.P_val.push_back(sc.P_val[q]);
      }
      C.P_ptr.push_back(int64_t(C.P_col.size()));
    }
  C.cell_dofs = sc.cell_dofs;
  C.constrained = con;
  C.phat = sc.phat;
  return C;
}

}  // namespace

std::unique_ptr<Problem> make_elastic_problem(int dim, int n, int p, double mu, double lambda, bool skip_boundary) {
  if (dim < 2 || dim > 3 || n < 1 || p < 1) throw std::invalid_argument("make_elastic_problem: bad dim / n / p");
  if (!(mu > 0.0) || !(lambda >= 0.0) || std::isinf(lambda))
    throw std::invalid_argument("elasticity_primal_operator: lambda must be finite");
  auto pb = std::make_unique<Problem>();
  pb->config = 0;
  pb->dim = dim;
  pb->n = n;
  pb->p = p;
  pb->mesh = cartesian_mesh(dim, std::vector<int>(dim, n), std::vector<double>(dim, 1.0));
  // tag_boundary (src/mesh.cpp:323-332) on facet vertex centroids: Neumann
  // everywhere, then x = 0 Dirichlet (tests/test_elasticity.cpp:24-30).
  for (auto& f : pb->mesh.facets) {
    if (f.ncells() != 1) continue;
    double cx = 0.0;
    for (int v : f.vertices) cx += pb->mesh.vertices[v][0];
    cx /= double(f.vertices.size());
    f.tag = std::abs(cx) < 1e-12 ? 1 : 2;
  }
  std::mt19937_64 rng(0);
  finish_problem(*pb, rng, false);  // scalar space, cell data
  pb->ncomp = dim;
  pb->lame_mu = mu;
  pb->lame_lambda = lambda;
  pb->Cmat = bundle_C(pb->basis);
  rebuild_patches(*pb, skip_boundary);
  // vector_load with f = -0.02 e_{dim-1} (src/elasticity.cpp:169-202) on
  // Cartesian cells: det * f * prod_a (sum_q w_q V(q, i_a)), then zero_constrained.
  const Space& s = pb->space;
  const int64_t ns = s.ndof;
  const int n1 = p + 1;
  std::vector<double> sv(n1, 0.0);
  for (int l = 0; l < n1; ++l)
    for (int q = 0; q < pb->basis.q; ++q) sv[l] += pb->basis.wq[q] * pb->basis.Vq(q, l);
  pb->rhs.assign(size_t(dim) * ns, 0.0);
  for (int c = 0; c < pb->mesh.num_cells(); ++c) {
    const auto L = half_extents(pb->mesh, c);
    double det = 1.0;
    for (int a = 0; a < dim; ++a) det *= L[a];
    for (int k = 0; k < s.npc; ++k) {
      double g = det * -0.02;
      for (int a = 0, kk = k; a < dim; ++a, kk /= n1) g *= sv[kk % n1];
      pb->rhs[(dim - 1) * ns + s.cell_dofs[size_t(c) * s.npc + k]] += g;
    }
  }
  for (int ci = 0; ci < dim; ++ci)
    for (int64_t i = 0; i < ns; ++i)
      if (s.constrained[i]) pb->rhs[ci * ns + i] = 0.0;
  pb->coarse = build_coarse_elastic(*pb);
  return pb;
}

}  // namespace fdmgpu::host
