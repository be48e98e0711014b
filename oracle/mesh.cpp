// TEST INFRASTRUCTURE ONLY — oracle restatement, see oracle.hpp header.
// L2: mesh (src/mesh.cpp), geometry (src/geometry.cpp), discretization
// (src/discretization.cpp) for the scalar continuous Q_p space.
#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <stdexcept>
#include <tuple>

#include "oracle.hpp"

namespace oracle {

std::vector<int> Mesh::local_facet_corners(int dim, int axis, int side) {
  std::vector<int> out;
  const int fixed_bit = (side > 0) ? (1 << axis) : 0;
  const int nrem = 1 << (dim - 1);
  for (int m = 0; m < nrem; ++m) {
    int corner = fixed_bit, mm = m;
    for (int a = 0; a < dim; ++a) {
      if (a == axis) continue;
      if (mm & 1) corner |= 1 << a;
      mm >>= 1;
    }
    out.push_back(corner);
  }
  return out;
}

void Mesh::finalize() {
  facets.clear();
  std::map<std::vector<int>, int> lookup;
  for (int c = 0; c < num_cells(); ++c) {
    if (int(cells[c].size()) != corners_per_cell()) throw std::invalid_argument("mesh: cell has wrong corner count");
    for (int v : cells[c])
      if (v < 0 || v >= num_vertices()) throw std::invalid_argument("mesh: cell references a bad vertex");
    for (int axis = 0; axis < dim; ++axis)
      for (int side : {-1, 1}) {
        std::vector<int> corners;
        for (int lc : local_facet_corners(dim, axis, side)) corners.push_back(cells[c][lc]);
        std::vector<int> key = corners;
        std::sort(key.begin(), key.end());
        auto [it, inserted] = lookup.try_emplace(key, int(facets.size()));
        if (inserted) {
          Facet f;
          f.cell[0] = c;
          f.axis[0] = axis;
          f.side[0] = side;
          f.vertices = corners;
          facets.push_back(std::move(f));
        } else {
          Facet& f = facets[it->second];
          if (f.cell[1] >= 0) throw std::invalid_argument("mesh: facet shared by more than two cells");
          f.cell[1] = c;
          f.axis[1] = axis;
          f.side[1] = side;
          if (dim == 2) {
            if (corners == f.vertices)
              f.tangential_flip = false;
            else if (corners[0] == f.vertices[1] && corners[1] == f.vertices[0])
              f.tangential_flip = true;
            else
              throw std::invalid_argument("mesh: non-conforming facet");
          } else {
            f.oriented = (corners == f.vertices);
          }
        }
      }
  }
  for (auto& f : facets)
    if (f.ncells() == 1 && f.tag == FacetTag::Interior) f.tag = FacetTag::Dirichlet;
  vertex_cells.assign(num_vertices(), {});
  for (int c = 0; c < num_cells(); ++c)
    for (int v : cells[c]) vertex_cells[v].push_back(c);
  for (auto& vc : vertex_cells) {
    std::sort(vc.begin(), vc.end());
    vc.erase(std::unique(vc.begin(), vc.end()), vc.end());
  }
}

static Mesh lattice_mesh(int dim, const std::vector<std::vector<double>>& coords) {
  Mesh mesh;
  mesh.dim = dim;
  std::vector<int> np(3, 1);
  for (int a = 0; a < dim; ++a) np[a] = int(coords[a].size());
  auto vid = [&](int i, int j, int k) { return i + np[0] * (j + np[1] * k); };
  for (int k = 0; k < np[2]; ++k)
    for (int j = 0; j < np[1]; ++j)
      for (int i = 0; i < np[0]; ++i) {
        std::array<double, 3> v{0, 0, 0};
        v[0] = coords[0][i];
        v[1] = coords[1][j];
        if (dim == 3) v[2] = coords[2][k];
        mesh.vertices.push_back(v);
      }
  const int nz = (dim == 3) ? np[2] - 1 : 1;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < np[1] - 1; ++j)
      for (int i = 0; i < np[0] - 1; ++i) {
        std::vector<int> c;
        for (int b = 0; b < (1 << dim); ++b) c.push_back(vid(i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1)));
        mesh.cells.push_back(c);
      }
  mesh.finalize();
  return mesh;
}

Mesh cartesian_mesh(int dim, const std::vector<int>& counts, const std::vector<double>& lengths) {
  if (dim < 2 || dim > 3) throw std::invalid_argument("cartesian_mesh: dim must be 2 or 3");
  if (int(counts.size()) != dim || int(lengths.size()) != dim)
    throw std::invalid_argument("cartesian_mesh: counts/lengths size mismatch");
  std::vector<std::vector<double>> coords(dim);
  for (int a = 0; a < dim; ++a) {
    if (counts[a] < 1) throw std::invalid_argument("cartesian_mesh: counts must be >= 1");
    if (!(lengths[a] > 0)) throw std::invalid_argument("cartesian_mesh: extents must be positive");
    for (int i = 0; i <= counts[a]; ++i) coords[a].push_back(lengths[a] * i / counts[a]);  // src/mesh.cpp:120-122
  }
  return lattice_mesh(dim, coords);
}

Mesh tensor_grid_mesh(int dim, const std::vector<std::vector<double>>& coords) { return lattice_mesh(dim, coords); }

std::vector<char> boundary_vertices(const Mesh& mesh) {
  std::vector<char> onb(mesh.num_vertices(), 0);
  for (const auto& f : mesh.facets)
    if (f.ncells() == 1)
      for (int v : f.vertices) onb[v] = 1;
  return onb;
}

// ---- geometry (src/geometry.cpp) ----------------------------------------------
static double corner_shape(int corner, int axis, const Vec& xhat, int dim, bool derivative_axis) {
  double g = 1.0;
  for (int a = 0; a < dim; ++a) {
    const bool hi = (corner >> a) & 1;
    if (derivative_axis && a == axis)
      g *= hi ? 0.5 : -0.5;
    else
      g *= hi ? 0.5 * (1.0 + xhat[a]) : 0.5 * (1.0 - xhat[a]);
  }
  return g;
}

std::array<double, 3> cell_map(const Mesh& mesh, int cell, const Vec& xhat) {
  std::array<double, 3> x{0, 0, 0};
  for (int b = 0; b < mesh.corners_per_cell(); ++b) {
    const double g = corner_shape(b, -1, xhat, mesh.dim, false);
    for (int r = 0; r < 3; ++r) x[r] += g * mesh.vertices[mesh.cells[cell][b]][r];
  }
  return x;
}

Mat cell_map_jacobian(const Mesh& mesh, int cell, const Vec& xhat) {
  const int d = mesh.dim;
  Mat DF(d, d);
  for (int b = 0; b < mesh.corners_per_cell(); ++b) {
    const auto& v = mesh.vertices[mesh.cells[cell][b]];
    for (int a = 0; a < d; ++a) {
      const double g = corner_shape(b, a, xhat, d, true);
      for (int r = 0; r < d; ++r) DF(r, a) += g * v[r];
    }
  }
  return DF;
}

// Closed-form determinant / inverse for d <= 3 (Eigen's fixed-size paths).
static double det_small(const Mat& A) {
  if (A.r == 1) return A(0, 0);
  if (A.r == 2) return A(0, 0) * A(1, 1) - A(0, 1) * A(1, 0);
  return A(0, 0) * (A(1, 1) * A(2, 2) - A(1, 2) * A(2, 1)) - A(0, 1) * (A(1, 0) * A(2, 2) - A(1, 2) * A(2, 0)) +
         A(0, 2) * (A(1, 0) * A(2, 1) - A(1, 1) * A(2, 0));
}
static Mat inv_small(const Mat& A, double det) {
  Mat I(A.r, A.r);
  if (A.r == 1) {
    I(0, 0) = 1.0 / A(0, 0);
  } else if (A.r == 2) {
    I(0, 0) = A(1, 1) / det;
    I(0, 1) = -A(0, 1) / det;
    I(1, 0) = -A(1, 0) / det;
    I(1, 1) = A(0, 0) / det;
  } else {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
        I(i, j) = (A(i1, j1) * A(i2, j2) - A(i1, j2) * A(i2, j1)) / det;
      }
  }
  return I;
}

CellGeometry cell_geometry(const Mesh& mesh, int cell, const QuadratureRule& rule) {
  const int d = mesh.dim, nq1 = rule.size();
  int nq = 1;
  for (int a = 0; a < d; ++a) nq *= nq1;
  CellGeometry geom;
  geom.cell = cell;
  geom.dets.resize(nq);
  geom.quad_weights.resize(nq);
  Vec xhat(d);
  for (int q = 0; q < nq; ++q) {
    int qq = q;
    double w = 1.0;
    for (int a = 0; a < d; ++a) {
      xhat[a] = rule.points[qq % nq1];
      w *= rule.weights[qq % nq1];
      qq /= nq1;
    }
    Mat DF = cell_map_jacobian(mesh, cell, xhat);
    const double det = det_small(DF);
    if (det <= 0) throw std::runtime_error("cell_geometry: non-positive Jacobian in cell " + std::to_string(cell));
    Mat inv = inv_small(DF, det);
    Mat G = matmul(inv, inv.transpose());
    for (auto& g : G.a) g *= det;
    geom.metric.push_back(G);
    geom.jacobians.push_back(DF);
    geom.dets[q] = det;
    geom.quad_weights[q] = w;
  }
  const Mat& J0 = geom.jacobians[0];
  double scale = 0.0;
  for (double v : J0.a) scale = std::max(scale, std::abs(v));
  bool constant = true, diagonal = true;
  for (const auto& J : geom.jacobians)
    for (size_t k = 0; k < J.a.size(); ++k)
      if (std::abs(J.a[k] - J0.a[k]) > 1e-13 * scale) constant = false;
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c)
      if (r != c && std::abs(J0(r, c)) > 1e-13 * scale) diagonal = false;
  geom.kind = (constant && diagonal) ? MapKind::Cartesian : constant ? MapKind::Affine : MapKind::Bilinear;
  if (geom.kind == MapKind::Cartesian) {
    geom.lengths.resize(d);
    geom.mu.resize(d);
    double prod = 1.0;
    for (int a = 0; a < d; ++a) {
      geom.lengths[a] = J0(a, a);
      prod *= geom.lengths[a];
    }
    for (int a = 0; a < d; ++a) geom.mu[a] = prod / (geom.lengths[a] * geom.lengths[a]);
  } else {
    const double ref_measure = std::pow(2.0, d);
    geom.mu.assign(d, 0.0);
    for (int q = 0; q < nq; ++q)
      for (int a = 0; a < d; ++a) geom.mu[a] += geom.quad_weights[q] / ref_measure * geom.metric[q](a, a);
  }
  return geom;
}

// ---- discretization (src/discretization.cpp) ------------------------------------
namespace {
struct EntityTables {  // src/discretization.cpp:12-45
  std::vector<std::array<int, 6>> cell_facets;
  std::map<std::array<int, 2>, int> edge_lookup;
  std::vector<std::array<int, 2>> edge_vertices;
};
EntityTables build_entities(const Mesh& mesh) {
  EntityTables tab;
  tab.cell_facets.assign(mesh.num_cells(), {-1, -1, -1, -1, -1, -1});
  for (int fi = 0; fi < int(mesh.facets.size()); ++fi) {
    const Facet& f = mesh.facets[fi];
    for (int r = 0; r < f.ncells(); ++r) tab.cell_facets[f.cell[r]][2 * f.axis[r] + (f.side[r] > 0 ? 1 : 0)] = fi;
  }
  if (mesh.dim == 3) {
    for (int c = 0; c < mesh.num_cells(); ++c)
      for (int a = 0; a < 3; ++a)
        for (int bits = 0; bits < 4; ++bits) {
          int base = 0, mm = bits;
          for (int o = 0; o < 3; ++o) {
            if (o == a) continue;
            if (mm & 1) base |= 1 << o;
            mm >>= 1;
          }
          std::array<int, 2> pair{mesh.cells[c][base], mesh.cells[c][base | (1 << a)]};
          if (pair[0] > pair[1]) std::swap(pair[0], pair[1]);
          auto [it, inserted] = tab.edge_lookup.try_emplace(pair, int(tab.edge_vertices.size()));
          if (inserted) tab.edge_vertices.push_back(pair);
        }
  }
  return tab;
}
}  // namespace

int Discretization::num_free() const {
  int n = 0;
  for (char c : constrained) n += !c;
  return n;
}

void Discretization::project_free(Vec& x) const {
  for (int d = 0; d < ndof; ++d)
    if (constrained[d]) x[d] = 0.0;
}

static Discretization q_space_impl(const Mesh& mesh, int p, bool dg);
Discretization q_space(const Mesh& mesh, int p) { return q_space_impl(mesh, p, false); }
// dq_space (src/discretization.cpp:306-311): every axis DG, so no slot is
// shared (cg_count = 0: one new DOF per cell slot, no strong Dirichlet rows);
// labels still classify by interface slots.
Discretization dq_space(const Mesh& mesh, int p) { return q_space_impl(mesh, p, true); }

static Discretization q_space_impl(const Mesh& mesh, int p, bool dg) {
  Discretization disc;
  disc.mesh = &mesh;
  disc.degree = p;
  const int d = mesh.dim;
  EntityTables tab = build_entities(mesh);
  disc.edge_vertices = tab.edge_vertices;
  disc.dofs_per_cell = 1;
  for (int a = 0; a < d; ++a) disc.dofs_per_cell *= p + 1;
  disc.cell_dofs.assign(mesh.num_cells(), std::vector<int>(disc.dofs_per_cell, -1));
  disc.cell_modes.assign(mesh.num_cells(), std::vector<int>(disc.dofs_per_cell, -1));
  disc.cell_mode_flip_axis.assign(mesh.num_cells(), std::vector<signed char>(disc.dofs_per_cell, -1));
  std::map<std::tuple<int, int, int>, int> shared;
  for (int K = 0; K < mesh.num_cells(); ++K) {
    std::array<int, 3> idx{0, 0, 0};
    for (int lat = 0; lat < disc.dofs_per_cell; ++lat) {
      int n_iface = 0;
      std::array<int, 3> iface_axis{-1, -1, -1}, iface_side{0, 0, 0};
      for (int a = 0; a < d; ++a)
        if (idx[a] == 0 || idx[a] == p) {
          iface_axis[n_iface] = a;
          iface_side[n_iface] = (idx[a] == 0) ? -1 : 1;
          ++n_iface;
        }
      // All axes are CG here: the sharing entity equals the interface classification.
      Owner owner = Owner::Cell;
      int owner_id = K;
      std::tuple<int, int, int> key{0, 0, 0};
      bool is_shared = false;
      const int cg_count = dg ? 0 : n_iface;
      const auto& cg_axes = iface_axis;
      const auto& cg_sides = iface_side;
      bool mode_flip = false;
      int mode_tangent_axis = -1;
      std::tuple<int, int, int> mode_key{0, 0, 0};
      if (cg_count == 1) {  // src/discretization.cpp:126-158
        const int a = cg_axes[0], s = cg_sides[0];
        const int f = tab.cell_facets[K][2 * a + (s > 0 ? 1 : 0)];
        const Facet& facet = mesh.facets[f];
        std::array<int, 2> t{0, 0}, tdeg{0, 0};
        int nt = 0, tangent_axis = -1;
        for (int b = 0; b < d; ++b) {
          if (b == a) continue;
          t[nt] = idx[b];
          tdeg[nt] = p;
          tangent_axis = b;
          ++nt;
        }
        mode_key = {1, f, t[0] + (tdeg[0] + 1) * t[1]};
        if (facet.ncells() == 2 && facet.cell[1] == K) {
          if (d == 2) {
            if (facet.tangential_flip) {
              t[0] = tdeg[0] - t[0];
              mode_flip = true;
              mode_tangent_axis = tangent_axis;
            }
          } else if (!facet.oriented) {
            throw std::invalid_argument("discretization: 3D meshes must have consistently oriented facets");
          }
        }
        owner = Owner::Facet;
        owner_id = f;
        key = {1, f, t[0] + (tdeg[0] + 1) * t[1]};
        is_shared = true;
      } else if (cg_count == 2 && d == 3) {  // src/discretization.cpp:159-171
        const int afree = 3 - cg_axes[0] - cg_axes[1];
        int bits = 0;
        for (int k = 0; k < 2; ++k)
          if (cg_sides[k] > 0) bits |= 1 << cg_axes[k];
        const int v0 = mesh.cells[K][bits];
        const int v1 = mesh.cells[K][bits | (1 << afree)];
        std::array<int, 2> pair{std::min(v0, v1), std::max(v0, v1)};
        const int edge = tab.edge_lookup.at(pair);
        const int i = (v0 < v1) ? idx[afree] : p - idx[afree];
        owner = Owner::Edge;
        owner_id = edge;
        key = {2, edge, i};
        is_shared = true;
      } else if (cg_count == d) {  // src/discretization.cpp:172-189
        int bits = 0;
        for (int k = 0; k < d; ++k)
          if (cg_sides[k] > 0) bits |= 1 << cg_axes[k];
        const int v = mesh.cells[K][bits];
        owner = Owner::Vertex;
        owner_id = v;
        key = {3, v, 0};
        is_shared = true;
      }
      int dof = -1;
      if (is_shared) {
        auto [it, inserted] = shared.try_emplace(key, disc.ndof);
        dof = it->second;
        if (inserted) {
          disc.labels.push_back({});
          disc.multiplicity.push_back(0.0);
          disc.constrained.push_back(0);
          disc.owner_kind.push_back(owner);
          disc.owner_id.push_back(owner_id);
          ++disc.ndof;
        }
      } else {
        dof = disc.ndof++;
        disc.labels.push_back({});
        disc.multiplicity.push_back(0.0);
        disc.constrained.push_back(0);
        disc.owner_kind.push_back(Owner::Cell);
        disc.owner_id.push_back(K);
      }
      disc.cell_dofs[K][lat] = dof;
      if (mode_flip) {
        disc.cell_modes[K][lat] = shared.at(mode_key);
        disc.cell_mode_flip_axis[K][lat] = static_cast<signed char>(mode_tangent_axis);
      } else {
        disc.cell_modes[K][lat] = dof;
      }
      disc.multiplicity[dof] += 1.0;
      for (int k = 0; k < cg_count; ++k) {  // src/discretization.cpp:221-226
        const int f = tab.cell_facets[K][2 * cg_axes[k] + (cg_sides[k] > 0 ? 1 : 0)];
        if (mesh.facets[f].ncells() == 1 && mesh.facets[f].tag == FacetTag::Dirichlet) disc.constrained[dof] = 1;
      }
      DofLabel label;  // src/discretization.cpp:231-253
      if (n_iface == 0) {
        label = {DofClass::Interior, K};
      } else if (n_iface == 1) {
        const int f = tab.cell_facets[K][2 * iface_axis[0] + (iface_side[0] > 0 ? 1 : 0)];
        label = {DofClass::Facet, f};
      } else if (n_iface == 2 && d == 3) {
        const int afree = 3 - iface_axis[0] - iface_axis[1];
        int bits = 0;
        for (int k = 0; k < 2; ++k)
          if (iface_side[k] > 0) bits |= 1 << iface_axis[k];
        const int v0 = mesh.cells[K][bits];
        const int v1 = mesh.cells[K][bits | (1 << afree)];
        std::array<int, 2> pair{std::min(v0, v1), std::max(v0, v1)};
        label = {DofClass::Edge, tab.edge_lookup.at(pair)};
      } else {
        int bits = 0;
        for (int k = 0; k < n_iface; ++k)
          if (iface_side[k] > 0) bits |= 1 << iface_axis[k];
        label = {DofClass::Vertex, mesh.cells[K][bits]};
      }
      disc.labels[dof] = label;
      int a = 0;
      for (; a < d; ++a) {
        if (++idx[a] <= p) break;
        idx[a] = 0;
      }
    }
  }
  disc.nsc = disc.ndof;
  return disc;
}

std::vector<int> Discretization::star_dofs(int v) const {
  const auto& star_cells = mesh->vertex_cells[v];
  std::set<int> star(star_cells.begin(), star_cells.end());
  std::vector<int> out;
  for (int ci = 0; ci < ncomp; ++ci)
  for (int K : star_cells)
    for (int dof : comp_dofs(ci, K)) {
      if (constrained[dof]) continue;
      bool in = false;
      switch (owner_kind[dof]) {
        case Owner::Cell:
          in = star.count(owner_id[dof]) > 0;
          break;
        case Owner::Facet: {
          const auto& fv = mesh->facets[owner_id[dof]].vertices;
          in = std::find(fv.begin(), fv.end(), v) != fv.end();
          break;
        }
        case Owner::Edge:
          in = edge_vertices[owner_id[dof]][0] == v || edge_vertices[owner_id[dof]][1] == v;
          break;
        case Owner::Vertex:
          in = owner_id[dof] == v;
          break;
      }
      if (in) out.push_back(dof);
    }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

std::vector<int> Discretization::comp_dofs(int ci, int cell) const {
  std::vector<int> out = cell_dofs[cell];
  if (ci > 0)
    for (auto& v : out) v += ci * nsc;
  return out;
}

std::vector<int> Discretization::comp_modes(int ci, int cell) const {
  std::vector<int> out = cell_modes[cell];
  if (ci > 0)
    for (auto& v : out) v += ci * nsc;
  return out;
}

// vector_q_space (src/discretization.cpp:313-318): mesh.dim identical CG
// components.  build_discretization numbers each component with its own
// first-touch map after the previous ones (src/discretization.cpp:86-258), so
// component ci repeats component 0's numbering shifted by ci * nsc.
Discretization vector_q_space(const Mesh& mesh, int p) {
  Discretization d = q_space(mesh, p);
  const int n = d.ndof, nc = mesh.dim;
  d.ncomp = nc;
  d.nsc = n;
  auto rep = [&](auto& v) {
    auto base = v;
    for (int ci = 1; ci < nc; ++ci) v.insert(v.end(), base.begin(), base.end());
  };
  rep(d.labels);
  rep(d.multiplicity);
  rep(d.constrained);
  rep(d.owner_kind);
  rep(d.owner_id);
  d.ndof = n * nc;
  return d;
}

void tag_boundary(Mesh& mesh, const std::function<bool(const std::array<double, 3>&)>& pred,
                  FacetTag tag) {  // src/mesh.cpp:323-332
  for (auto& f : mesh.facets) {
    if (f.ncells() != 1) continue;
    std::array<double, 3> c{0.0, 0.0, 0.0};
    for (int v : f.vertices)
      for (int r = 0; r < 3; ++r) c[r] += mesh.vertices[v][r];
    for (int r = 0; r < 3; ++r) c[r] /= double(f.vertices.size());
    if (pred(c)) f.tag = tag;
  }
}

}  // namespace oracle
