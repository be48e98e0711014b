// Mesh, geometry surrogate, Q_p DOF numbering, vertex-star patch lists and
// the coarse Q1 level (host setup, once per problem).
//   Mesh::finalize              <- src/mesh.cpp:33-91
//   cartesian_mesh              <- src/mesh.cpp:102-136
//   cell_coeffs (mu surrogate)  <- src/geometry.cpp:45-104
//   q_space first-touch maps    <- src/discretization.cpp:19-264
//   star_dofs                   <- src/discretization.cpp:266-297
//   patch_ordering              <- src/ordering.cpp:17-45
//   vertex_patches              <- src/schwarz.cpp:62-83
//   build_coarse / prolongation <- src/schwarz.cpp:139-165, 239-243
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <set>
#include <stdexcept>
#include <tuple>

#include "fdm_host.hpp"

namespace fdmgpu::host {

namespace {

std::vector<int> facet_corners(int dim, int axis, int side) {  // src/mesh.cpp:16-31
  std::vector<int> out;
  for (int m = 0; m < (1 << (dim - 1)); ++m) {
    int corner = side > 0 ? (1 << axis) : 0, mm = m;
    for (int a = 0; a < dim; ++a) {
      if (a == axis) continue;
      if (mm & 1) corner |= 1 << a;
      mm >>= 1;
    }
    out.push_back(corner);
  }
  return out;
}

Mesh lattice(int dim, const std::vector<std::vector<double>>& xs) {
  Mesh m;
  m.dim = dim;
  int np[3] = {1, 1, 1};
  for (int a = 0; a < dim; ++a) np[a] = int(xs[a].size());
  for (int k = 0; k < np[2]; ++k)
    for (int j = 0; j < np[1]; ++j)
      for (int i = 0; i < np[0]; ++i)
        m.vertices.push_back({xs[0][i], xs[1][j], dim == 3 ? xs[2][k] : 0.0});
  auto vid = [&](int i, int j, int k) { return i + np[0] * (j + np[1] * k); };
  for (int k = 0; k < (dim == 3 ? np[2] - 1 : 1); ++k)
    for (int j = 0; j < np[1] - 1; ++j)
      for (int i = 0; i < np[0] - 1; ++i) {
        std::vector<int> c;
        for (int b = 0; b < (1 << dim); ++b) c.push_back(vid(i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1)));
        m.cells.push_back(std::move(c));
      }
  m.finalize();
  return m;
}

double det3(const double* J, int d) {  // J row-major d x d
  if (d == 2) return J[0] * J[3] - J[1] * J[2];
  return J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) + J[2] * (J[3] * J[7] - J[4] * J[6]);
}

// Jacobian of the multilinear map at xhat (src/geometry.cpp:33-43), row-major.

// G = det * J^{-1} J^{-T} (row-major d x d), via the adjugate.
void metric(const double* J, int d, double& det, double* G) {
  det = det3(J, d);
  double inv[9];
  if (d == 2) {
    inv[0] = J[3] / det;
    inv[1] = -J[1] / det;
    inv[2] = -J[2] / det;
    inv[3] = J[0] / det;
  } else {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
        inv[i * 3 + j] = (J[i1 * 3 + j1] * J[i2 * 3 + j2] - J[i1 * 3 + j2] * J[i2 * 3 + j1]) / det;
      }
  }
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double s = 0.0;
      for (int k = 0; k < d; ++k) s += inv[a * d + k] * inv[b * d + k];
      G[a * d + b] = det * s;
    }
}

}  // namespace

void jacobian(const Mesh& m, int cell, const double* xh, double* J) {
  const int d = m.dim;
  for (int k = 0; k < d * d; ++k) J[k] = 0.0;
  for (int b = 0; b < (1 << d); ++b) {
    const auto& v = m.vertices[m.cells[cell][b]];
    for (int a = 0; a < d; ++a) {
      double g = 1.0;
      for (int e = 0; e < d; ++e) {
        const bool hi = (b >> e) & 1;
        g *= (e == a) ? (hi ? 0.5 : -0.5) : (hi ? 0.5 * (1.0 + xh[e]) : 0.5 * (1.0 - xh[e]));
      }
      for (int r = 0; r < d; ++r) J[r * d + a] += g * v[r];
    }
  }
}

void Mesh::finalize() {
  facets.clear();
  std::map<std::vector<int>, int> lookup;
  for (int c = 0; c < num_cells(); ++c) {
    if (int(cells[c].size()) != (1 << dim)) throw std::invalid_argument("mesh: cell has wrong corner count");
    for (int axis = 0; axis < dim; ++axis)
      for (int side : {-1, 1}) {
        std::vector<int> corners;
        for (int lc : facet_corners(dim, axis, side)) corners.push_back(cells[c][lc]);
        std::vector<int> key = corners;
        std::sort(key.begin(), key.end());
        auto [it, fresh] = lookup.try_emplace(key, int(facets.size()));
        if (fresh) {
          Facet f;
          f.cell[0] = c;
          f.axis[0] = axis;
          f.side[0] = side;
          f.vertices = corners;
          facets.push_back(std::move(f));
          continue;
        }
        Facet& f = facets[it->second];
        if (f.cell[1] >= 0) throw std::invalid_argument("mesh: facet shared by more than two cells");
        f.cell[1] = c;
        f.axis[1] = axis;
        f.side[1] = side;
        if (dim == 2) {
          if (corners == f.vertices)
            f.flip = false;
          else if (corners[0] == f.vertices[1] && corners[1] == f.vertices[0])
            f.flip = true;
          else
            throw std::invalid_argument("mesh: non-conforming facet");
        } else {
          f.oriented = corners == f.vertices;
        }
      }
  }
  for (auto& f : facets)
    if (f.ncells() == 1 && f.tag == 0) f.tag = 1;  // src/mesh.cpp:82
  vertex_cells.assign(num_vertices(), {});
  for (int c = 0; c < num_cells(); ++c)
    for (int v : cells[c]) vertex_cells[v].push_back(c);
  for (auto& vc : vertex_cells) {
    std::sort(vc.begin(), vc.end());
    vc.erase(std::unique(vc.begin(), vc.end()), vc.end());
  }
}

Mesh cartesian_mesh(int dim, const std::vector<int>& counts, const std::vector<double>& lengths) {
  if (dim < 2 || dim > 3) throw std::invalid_argument("cartesian_mesh: dim must be 2 or 3");
  std::vector<std::vector<double>> xs(dim);
  for (int a = 0; a < dim; ++a) {
    if (counts[a] < 1 || !(lengths[a] > 0)) throw std::invalid_argument("cartesian_mesh: bad counts/extents");
    for (int i = 0; i <= counts[a]; ++i) xs[a].push_back(lengths[a] * i / counts[a]);
  }
  return lattice(dim, xs);
}

Mesh tensor_grid_mesh(int dim, const std::vector<std::vector<double>>& coords) { return lattice(dim, coords); }

std::vector<char> boundary_vertices(const Mesh& m) {
  std::vector<char> onb(m.num_vertices(), 0);
  for (const auto& f : m.facets)
    if (f.ncells() == 1)
      for (int v : f.vertices) onb[v] = 1;
  return onb;
}

CellCoeffs cell_coeffs(const Mesh& m, int cell, const Basis1D& b) {
  const int d = m.dim, q = b.q;
  Vec qp, qw;
  gauss_legendre(q, qp, qw);
  int nq = 1;
  for (int a = 0; a < d; ++a) nq *= q;
  std::vector<double> J0(d * d), J(d * d);
  double xh[3];
  bool constant = true, diagonal = true;
  std::array<double, 3> musum{0, 0, 0};
  double scale = 0.0;
  for (int k = 0; k < nq; ++k) {
    double w = 1.0;
    for (int a = 0, kk = k; a < d; ++a, kk /= q) {
      xh[a] = qp[kk % q];
      w *= qw[kk % q];
    }
    jacobian(m, cell, xh, k == 0 ? J0.data() : J.data());
    const double* Jk = k == 0 ? J0.data() : J.data();
    if (k == 0)
      for (double v : J0) scale = std::max(scale, std::abs(v));
    else
      for (int t = 0; t < d * d; ++t)
        if (std::abs(J[t] - J0[t]) > 1e-13 * scale) constant = false;
    double det, G[9];
    metric(Jk, d, det, G);
    if (det <= 0) throw std::runtime_error("cell_geometry: non-positive Jacobian in cell " + std::to_string(cell));
    for (int a = 0; a < d; ++a) musum[a] += w / std::pow(2.0, d) * G[a * d + a];
  }
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c)
      if (r != c && std::abs(J0[r * d + c]) > 1e-13 * scale) diagonal = false;
  CellCoeffs cc{};
  cc.kind = (constant && diagonal) ? MapKind::Cartesian : constant ? MapKind::Affine : MapKind::Bilinear;
  if (cc.kind == MapKind::Cartesian) {
    double prod = 1.0;
    for (int a = 0; a < d; ++a) prod *= J0[a * d + a];
    for (int a = 0; a < d; ++a) cc.mu[a] = prod / (J0[a * d + a] * J0[a * d + a]);
  } else {
    for (int a = 0; a < d; ++a) cc.mu[a] = musum[a];
  }
  for (int a = 0; a < d; ++a) cc.mu[a] *= m.coeff(cell);
  return cc;
}

int Space::num_free() const {
  int n = 0;
  for (uint8_t c : constrained) n += !c;
  return n;
}

Space q_space(const Mesh& m, int p, bool dg) {
  Space s;
  s.mesh = &m;
  s.p = p;
  const int d = m.dim, n1 = p + 1;
  s.npc = d == 3 ? n1 * n1 * n1 : n1 * n1;
  // Entity tables (src/discretization.cpp:19-45).
  std::vector<std::array<int, 6>> cf(m.num_cells(), {-1, -1, -1, -1, -1, -1});
  for (int f = 0; f < int(m.facets.size()); ++f)
    for (int r = 0; r < m.facets[f].ncells(); ++r)
      cf[m.facets[f].cell[r]][2 * m.facets[f].axis[r] + (m.facets[f].side[r] > 0)] = f;
  std::map<std::array<int, 2>, int> edge_id;
  if (d == 3)
    for (int c = 0; c < m.num_cells(); ++c)
      for (int a = 0; a < 3; ++a)
        for (int bits = 0; bits < 4; ++bits) {
          int base = 0, mm = bits;
          for (int o = 0; o < 3; ++o) {
            if (o == a) continue;
            if (mm & 1) base |= 1 << o;
            mm >>= 1;
          }
          std::array<int, 2> e{m.cells[c][base], m.cells[c][base | (1 << a)]};
          if (e[0] > e[1]) std::swap(e[0], e[1]);
          if (edge_id.try_emplace(e, int(s.edge_vertices.size())).second) s.edge_vertices.push_back(e);
        }
  s.cell_dofs.assign(size_t(m.num_cells()) * s.npc, -1);
  s.cell_modes.assign(size_t(m.num_cells()) * s.npc, -1);
  std::vector<double> sign(size_t(m.num_cells()) * s.npc, 1.0);
  bool any_flip = false;
  std::map<std::tuple<int, int, int>, int> shared;
  auto new_dof = [&](uint8_t okind, int oid) {
    s.multiplicity.push_back(0.0);
    s.constrained.push_back(0);
    s.label_cls.push_back(0);
    s.label_entity.push_back(-1);
    s.owner_kind.push_back(okind);
    s.owner_id.push_back(oid);
    return s.ndof++;
  };
  for (int K = 0; K < m.num_cells(); ++K) {
    int idx[3] = {0, 0, 0};
    for (int lat = 0; lat < s.npc; ++lat) {
      int nif = 0, iax[3], isd[3];
      for (int a = 0; a < d; ++a)
        if (idx[a] == 0 || idx[a] == p) {
          iax[nif] = a;
          isd[nif] = idx[a] == 0 ? -1 : 1;
          ++nif;
        }
      int bits = 0;
      for (int k = 0; k < nif; ++k)
        if (isd[k] > 0) bits |= 1 << iax[k];
      int dof;
      uint8_t cls = 0;
      int entity = K;
      int mode_dof = -1;
      double msign = 1.0;
      if (dg) {
        // dq_space (src/discretization.cpp:306-311): every slot is cell-local
        // (owner the cell), classified like the CG slots for patch_ordering
        dof = new_dof(0, K);
        if (nif == 1) {
          cls = 1;
          entity = cf[K][2 * iax[0] + (isd[0] > 0)];
        } else if (nif == 2 && d == 3) {
          const int afree = 3 - iax[0] - iax[1];
          const int v0 = m.cells[K][bits], v1 = m.cells[K][bits | (1 << afree)];
          cls = 2;
          entity = edge_id.at({std::min(v0, v1), std::max(v0, v1)});
        } else if (nif > 0) {
          cls = 3;
          entity = m.cells[K][bits];
        }
      } else if (nif == 0) {
        dof = new_dof(0, K);
      } else if (nif == 1) {
        const int a = iax[0];
        const int f = cf[K][2 * a + (isd[0] > 0)];
        const Facet& F = m.facets[f];
        int t[2] = {0, 0}, nt = 0, tan_axis = -1;
        for (int b = 0; b < d; ++b)
          if (b != a) {
            t[nt++] = idx[b];
            tan_axis = b;
          }
        const int mode_index = t[0] + n1 * t[1];
        if (F.ncells() == 2 && F.cell[1] == K) {
          if (d == 2 && F.flip) t[0] = p - t[0];
          if (d == 3 && !F.oriented)
            throw std::invalid_argument("discretization: 3D meshes must have consistently oriented facets");
        }
        auto [it, fresh] = shared.try_emplace(std::make_tuple(1, f, t[0] + n1 * t[1]), s.ndof);
        dof = fresh ? new_dof(1, f) : it->second;
        if (d == 2 && F.ncells() == 2 && F.cell[1] == K && F.flip) {
          mode_dof = shared.at(std::make_tuple(1, f, mode_index));
          msign = 0.0;  // resolved below from the parity of the tangential mode
          (void)tan_axis;
        }
        cls = 1;
        entity = f;
      } else if (nif == 2 && d == 3) {
        const int afree = 3 - iax[0] - iax[1];
        const int v0 = m.cells[K][bits], v1 = m.cells[K][bits | (1 << afree)];
        const int e = edge_id.at({std::min(v0, v1), std::max(v0, v1)});
        const int i = v0 < v1 ? idx[afree] : p - idx[afree];
        auto [it, fresh] = shared.try_emplace(std::make_tuple(2, e, i), s.ndof);
        dof = fresh ? new_dof(2, e) : it->second;
        cls = 2;
        entity = e;
      } else {
        const int v = m.cells[K][bits];
        auto [it, fresh] = shared.try_emplace(std::make_tuple(3, v, 0), s.ndof);
        dof = fresh ? new_dof(3, v) : it->second;
        cls = 3;
        entity = v;
      }
      const size_t slot = size_t(K) * s.npc + lat;
      s.cell_dofs[slot] = dof;
      s.cell_modes[slot] = mode_dof >= 0 ? mode_dof : dof;
      if (mode_dof >= 0) {
        any_flip = true;
        sign[slot] = msign;  // placeholder, fixed by the caller with the basis parity
      }
      s.multiplicity[dof] += 1.0;
      for (int k = 0; k < nif && !dg; ++k)
        if (m.facets[cf[K][2 * iax[k] + (isd[k] > 0)]].ncells() == 1 &&
            m.facets[cf[K][2 * iax[k] + (isd[k] > 0)]].tag == 1)
          s.constrained[dof] = 1;  // src/discretization.cpp:221-226 (Dirichlet facets)
      s.label_cls[dof] = cls;
      s.label_entity[dof] = entity;
      for (int a = 0; a < d; ++a) {
        if (++idx[a] <= p) break;
        idx[a] = 0;
      }
    }
  }
  if (any_flip) s.mode_sign = std::move(sign);
  return s;
}

std::vector<int32_t> Space::star_dofs(int v) const {
  const auto& star = mesh->vertex_cells[v];
  std::vector<int32_t> out;
  for (int K : star)
    for (int l = 0; l < npc; ++l) {
      const int dof = cell_dofs[size_t(K) * npc + l];
      if (constrained[dof]) continue;
      bool in = false;
      switch (owner_kind[dof]) {
        case 0: in = std::binary_search(star.begin(), star.end(), owner_id[dof]); break;
        case 1: {
          const auto& fv = mesh->facets[owner_id[dof]].vertices;
          in = std::find(fv.begin(), fv.end(), v) != fv.end();
          break;
        }
        case 2: in = edge_vertices[owner_id[dof]][0] == v || edge_vertices[owner_id[dof]][1] == v; break;
        default: in = owner_id[dof] == v;
      }
      if (in) out.push_back(dof);
    }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

std::vector<int32_t> patch_ordering(const Space& s, const std::vector<int32_t>& dofs) {
  const int n = int(dofs.size());
  std::vector<int32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    const int ca = s.label_cls[dofs[a]], cb = s.label_cls[dofs[b]];
    if (ca != cb) return ca < cb;
    const int ea = s.label_entity[dofs[a]], eb = s.label_entity[dofs[b]];
    if (ea != eb) return ea < eb;
    return a < b;
  });
  return idx;
}

Patches vertex_patches(const Space& s, bool skip_boundary) {
  const Mesh& m = *s.mesh;
  const auto onb = boundary_vertices(m);
  Patches P;
  P.ptr.push_back(0);
  auto add = [&](int v, std::vector<int32_t> dofs) {
    auto perm = patch_ordering(s, dofs);
    P.vertex.push_back(v);
    P.dofs.insert(P.dofs.end(), dofs.begin(), dofs.end());
    P.perm.insert(P.perm.end(), perm.begin(), perm.end());
    P.ptr.push_back(int64_t(P.dofs.size()));
    const auto& vc = m.vertex_cells[v];
    for (int k = 0; k < (1 << m.dim); ++k) P.cells.push_back(k < int(vc.size()) ? vc[k] : -1);
  };
  for (int v = 0; v < m.num_vertices(); ++v) {
    if (skip_boundary && onb[v]) continue;
    auto dofs = s.star_dofs(v);
    if (!dofs.empty()) add(v, std::move(dofs));
  }
  if (P.vertex.empty())
    for (int v = 0; v < m.num_vertices(); ++v) {
      auto dofs = s.star_dofs(v);
      if (!dofs.empty()) add(v, std::move(dofs));
    }
  // Colouring: greedy first-fit over "stars share a cell", ascending patch
  // order. On lattice meshes this is the vertex-parity colouring
  // (i mod 2) + 2 (j mod 2) + 4 (k mod 2) up to a relabelling.
  const int np = int(P.vertex.size());
  std::vector<std::vector<int>> cell_patches(m.num_cells());
  for (int j = 0; j < np; ++j)
    for (int k = 0; k < (1 << m.dim); ++k)
      if (P.cells[size_t(j) * (1 << m.dim) + k] >= 0) cell_patches[P.cells[size_t(j) * (1 << m.dim) + k]].push_back(j);
  P.colour.assign(P.vertex.size(), -1);
  for (int j = 0; j < np; ++j) {
    std::set<int> used;
    for (int k = 0; k < (1 << m.dim); ++k) {
      const int c = P.cells[size_t(j) * (1 << m.dim) + k];
      if (c < 0) continue;
      for (int o : cell_patches[c])
        if (P.colour[o] >= 0) used.insert(P.colour[o]);
    }
    int col = 0;
    while (used.count(col)) ++col;
    P.colour[j] = col;
  }
  return P;
}

// Dense Cholesky (natural ordering, as cholesky(A, natural_ordering) on the
// assembled coarse matrix, src/schwarz.cpp:242-243) and the explicit inverse
// (row-major n x n); the coarse problems are at most a few thousand DOFs.
std::vector<double> dense_spd_inverse(const std::vector<double>& A, int nc) {
  std::vector<double> L(size_t(nc) * nc, 0.0);  // row-major lower factor
  for (int j = 0; j < nc; ++j) {
    const double* Lj = &L[size_t(j) * nc];
    double dd = A[size_t(j) * nc + j];
    for (int k = 0; k < j; ++k) dd -= Lj[k] * Lj[k];
    if (!(dd > 0.0)) throw std::runtime_error("cholesky: coarse matrix not SPD at pivot " + std::to_string(j));
    L[size_t(j) * nc + j] = std::sqrt(dd);
    for (int i = j + 1; i < nc; ++i) {
      const double* Li = &L[size_t(i) * nc];
      double s = A[size_t(i) * nc + j];
      for (int k = 0; k < j; ++k) s -= Li[k] * Lj[k];
      L[size_t(i) * nc + j] = s / Lj[j];
    }
  }
  // W[e][i] = (L^{-1})(i, e): forward substitution per unit vector.
  std::vector<double> W(size_t(nc) * nc, 0.0);
  for (int e = 0; e < nc; ++e) {
    double* x = &W[size_t(e) * nc];
    for (int i = e; i < nc; ++i) {
      const double* Li = &L[size_t(i) * nc];
      double s = i == e ? 1.0 : 0.0;
      for (int k = e; k < i; ++k) s -= Li[k] * x[k];
      x[i] = s / Li[i];
    }
  }
  // A^{-1} = L^{-T} L^{-1}: entry (i, j) = sum_k W[i][k] W[j][k].
  std::vector<double> inv(size_t(nc) * nc, 0.0);
  for (int i = 0; i < nc; ++i)
    for (int j = 0; j <= i; ++j) {
      const double* wi = &W[size_t(i) * nc];
      const double* wj = &W[size_t(j) * nc];
      double s = 0.0;
      for (int k = i; k < nc; ++k) s += wi[k] * wj[k];
      inv[size_t(i) * nc + j] = s;
      inv[size_t(j) * nc + i] = s;
    }
  return inv;
}

Coarse build_coarse(const Mesh& m, const Space& fine, const Basis1D& fb) {
  const int d = m.dim;
  Space cs = q_space(m, 1);
  Coarse C;
  C.ndof = cs.ndof;
  const int nc = cs.ndof, npc = 1 << d;
  // Coarse true-form operator (src/assembly.cpp:230-243 at p = 1), dense.
  Basis1D b1 = make_bundle(1);
  std::vector<double> A(size_t(nc) * nc, 0.0);
  Vec qp, qw;
  gauss_legendre(b1.q, qp, qw);
  for (int c = 0; c < m.num_cells(); ++c) {
    CellCoeffs cc = cell_coeffs(m, c, b1);
    std::vector<double> K(npc * npc, 0.0);
    if (cc.kind == MapKind::Cartesian) {
      for (int i = 0; i < npc; ++i)
        for (int j = 0; j < npc; ++j) {
          double s = 0.0;
          for (int a = 0; a < d; ++a) {
            double prod = cc.mu[a];
            for (int b = 0; b < d; ++b) {
              const int ib = (i >> b) & 1, jb = (j >> b) & 1;
              prod *= (b == a ? b1.A_hat(ib, jb) : b1.B_hat(ib, jb));
            }
            s += prod;
          }
          K[i * npc + j] = s;
        }
    } else {
      // Quadrature form with GL(3) (exact for the p = 1 cell matrices).
      const int q = b1.q;
      int nq = 1;
      for (int a = 0; a < d; ++a) nq *= q;
      for (int k = 0; k < nq; ++k) {
        double xh[3], w = 1.0;
        int qi[3];
        for (int a = 0, kk = k; a < d; ++a, kk /= q) {
          qi[a] = kk % q;
          xh[a] = qp[qi[a]];
          w *= qw[qi[a]];
        }
        double J[9], det, G[9];
        jacobian(m, c, xh, J);
        metric(J, d, det, G);
        double grad[8][3];
        for (int i = 0; i < npc; ++i)
          for (int a = 0; a < d; ++a) {
            double g = 1.0;
            for (int b = 0; b < d; ++b) {
              const int ib = (i >> b) & 1;
              g *= (b == a) ? b1.Dq(qi[b], ib) : b1.Vq(qi[b], ib);
            }
            grad[i][a] = g;
          }
        for (int i = 0; i < npc; ++i)
          for (int j = 0; j < npc; ++j) {
            double s = 0.0;
            for (int a = 0; a < d; ++a)
              for (int b = 0; b < d; ++b) s += grad[i][a] * G[a * d + b] * grad[j][b];
            K[i * npc + j] += w * m.coeff(c) * s;
          }
      }
    }
    for (int i = 0; i < npc; ++i) {
      const int gi = cs.cell_dofs[size_t(c) * npc + i];
      if (cs.constrained[gi]) continue;
      for (int j = 0; j < npc; ++j) {
        const int gj = cs.cell_dofs[size_t(c) * npc + j];
        if (!cs.constrained[gj]) A[size_t(gi) * nc + gj] += 0.5 * (K[i * npc + j] + K[j * npc + i]);
      }
    }
  }
  for (int i = 0; i < nc; ++i)
    if (cs.constrained[i]) A[size_t(i) * nc + i] = 1.0;
  C.inverse = dense_spd_inverse(A, nc);
  // Prolongation: Q1 hats at the fine GLL nodes, summed over cells, divided
  // by the fine multiplicity; constrained rows / columns dropped.
  const int p = fb.p, n1 = p + 1;
  Vec ends{-1.0, 1.0};
  Dense ph, phd;
  lagrange_eval(ends, fb.nodes, ph, phd);  // (p+1) x 2
  std::vector<std::map<int, double>> rows(fine.ndof);
  for (int c = 0; c < m.num_cells(); ++c)
    for (int i = 0; i < fine.npc; ++i) {
      const int fi = fine.cell_dofs[size_t(c) * fine.npc + i];
      if (fine.constrained[fi]) continue;
      int fl[3] = {i % n1, (i / n1) % n1, i / (n1 * n1)};
      for (int j = 0; j < npc; ++j) {
        const int cj = cs.cell_dofs[size_t(c) * npc + j];
        if (cs.constrained[cj]) continue;
        double v = 1.0;
        for (int a = 0; a < d; ++a) v *= ph(fl[a], (j >> a) & 1);
        if (v != 0.0) rows[fi][cj] += v;
      }
    }
  C.cell_dofs.assign(cs.cell_dofs.begin(), cs.cell_dofs.end());
  C.constrained.assign(cs.constrained.begin(), cs.constrained.end());
  C.phat.resize(size_t(n1) * 2);
  for (int l = 0; l < n1; ++l)
    for (int j = 0; j < 2; ++j) C.phat[l + size_t(n1) * j] = ph(l, j);
  C.P_ptr.assign(1, 0);
  for (int i = 0; i < fine.ndof; ++i) {
    for (const auto& [cj, v] : rows[i]) {
      C.P_col.push_back(cj);
      C.P_val.push_back(v / fine.multiplicity[i]);
    }
    C.P_ptr.push_back(int64_t(C.P_col.size()));
  }
  return C;
}

}  // namespace fdmgpu::host
