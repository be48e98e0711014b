// Host-side setup of the B200 vertex-star FDM Schwarz path: the parts of
// the reference that run once per problem on the CPU and produce the index
// maps, 1D FDM basis and patch lists the device path consumes.  They mirror
// the reference entry points (names and semantics) of
//   include/fdmstar/{quadrature,reference_interval,dense_eig,fdm_basis,
//                    mesh,geometry,discretization,ordering,schwarz}.hpp
// for the scalar continuous Q_p space on conforming quad/hex meshes.
// Index maps are bit-exact with the reference's first-touch numbering
// (src/discretization.cpp:70-264), which the tests check against the oracle.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <random>
#include <string>
#include <vector>

namespace fdmgpu::host {

using Vec = std::vector<double>;

// Column-major dense matrix.
struct Dense {
  int r = 0, c = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(int rows, int cols) : r(rows), c(cols), a(size_t(rows) * cols, 0.0) {}
  double& operator()(int i, int j) { return a[i + size_t(r) * j]; }
  double operator()(int i, int j) const { return a[i + size_t(r) * j]; }
};

// ---- 1D: quadrature (src/quadrature.cpp), reference interval
// (src/reference_interval.cpp), FDM basis (src/fdm_basis.cpp) -----------------
Vec gll_nodes(int p);
void gauss_legendre(int n, Vec& pts, Vec& wts);
void lagrange_eval(const Vec& nodes, const Vec& pts, Dense& V, Dense& D);

struct Basis1D {
  int p = 0;
  Vec nodes;          // GLL nodes
  Dense A_hat, B_hat; // reference stiffness / mass, GL(p+1)-exact
  Dense S;            // FDM modes (nodal coefficients), (p+1)^2
  Vec lambda;         // p-1 interior eigenvalues, ascending
  Dense A_t, B_t;     // S^T A S, S^T B S with their structural patterns
  std::vector<uint8_t> A_nz, B_nz;
  Vec parity;
  // GL(p+2) interpolation / derivative tables for the true-form trilinear apply
  int q = 0;
  Dense Vq, Dq;       // q x (p+1)
  Vec wq, qp;
  // DG family (make_bundle_dg): nodes / A_hat / B_hat / S of the GL-nodal
  // interval, the FDM modes' outward derivative traces (fdm.deriv_traces) and
  // the nodal traces (trace_values, trace_normal_derivs), all 2 x (p+1)
  bool dg = false;
  Dense dtr, tv, tnd;
};
Basis1D make_bundle(int p);     // src/assembly.cpp:37-54 (CG family)
Basis1D make_bundle_dg(int p);  // src/assembly.cpp:37-54 (DG family), to_gl_representation (src/fdm_basis.cpp:89-101)
double sipg_default_eta(int p, int d);  // src/sipg.cpp:7

// ---- mesh (src/mesh.cpp), geometry (src/geometry.cpp) ------------------------
struct Facet {
  std::array<int, 2> cell{-1, -1}, axis{-1, -1}, side{0, 0};
  bool flip = false, oriented = true;
  int tag = 0;  // 0 interior, 1 dirichlet, 2 neumann (FacetTag, include/fdmstar/mesh.hpp)
  std::vector<int> vertices;
  int ncells() const { return cell[1] >= 0 ? 2 : 1; }
};
struct Mesh {
  int dim = 3;
  std::vector<std::array<double, 3>> vertices;
  std::vector<std::vector<int>> cells;
  std::vector<Facet> facets;
  std::vector<std::vector<int>> vertex_cells;
  std::vector<double> kappa;  // per-cell coefficient (config C4), empty => 1
  int num_cells() const { return int(cells.size()); }
  int num_vertices() const { return int(vertices.size()); }
  double coeff(int c) const { return kappa.empty() ? 1.0 : kappa[c]; }
  void finalize();  // src/mesh.cpp:33-91 (boundary facets tagged dirichlet)
  int find_facet(int cell, int axis, int side) const;  // -1 if absent
};
void jacobian(const Mesh& m, int cell, const double* xh, double* J);
// Mesh files (src/mesh.cpp:354-434): the reference's JSON document.
Mesh load_mesh(const std::string& path);
void save_mesh(const Mesh& m, const std::string& path);
void apply_facet_tags(Mesh& m, const std::vector<int>& cell, const std::vector<int>& local_facet,
                      const std::vector<int>& tag);
void check_orientation(const Mesh& m);
Mesh cartesian_mesh(int dim, const std::vector<int>& counts, const std::vector<double>& lengths);
Mesh tensor_grid_mesh(int dim, const std::vector<std::vector<double>>& coords);
std::vector<char> boundary_vertices(const Mesh& m);

// Cell classification and surrogate coefficients (src/geometry.cpp:45-104).
enum class MapKind { Cartesian = 0, Affine = 1, Bilinear = 2 };
struct CellCoeffs {
  MapKind kind;
  std::array<double, 3> mu;  // kappa * mu^K (surrogate), per axis
};
CellCoeffs cell_coeffs(const Mesh& m, int cell, const Basis1D& b);

// ---- discretization (src/discretization.cpp) ---------------------------------
enum class DofClass { Interior = 0, Facet = 1, Edge = 2, Vertex = 3 };
struct Space {
  const Mesh* mesh = nullptr;
  int p = 0, npc = 0, ndof = 0;
  std::vector<int32_t> cell_dofs;  // ncells x npc, lattice axis 0 fastest
  std::vector<int32_t> cell_modes; // equal to cell_dofs unless a 2D facet flips
  std::vector<double> mode_sign;   // ncells x npc (+-1), empty when all +1
  std::vector<double> multiplicity;
  std::vector<uint8_t> constrained;
  std::vector<int32_t> label_cls, label_entity;
  std::vector<uint8_t> owner_kind;  // 0 cell, 1 facet, 2 edge, 3 vertex
  std::vector<int32_t> owner_id;
  std::vector<std::array<int, 2>> edge_vertices;
  int num_free() const;
  std::vector<int32_t> star_dofs(int v) const;  // src/discretization.cpp:266-297
};
// dg = true: dq_space (src/discretization.cpp:306-311), all DOFs cell-local,
// no strong Dirichlet marking, labels by interface-slot class as the CG ones.
Space q_space(const Mesh& m, int p, bool dg = false);

// patch_ordering (src/ordering.cpp:17-45): interiors, then facet / edge groups
// by entity id, vertex last; ties on the position in `dofs`.
std::vector<int32_t> patch_ordering(const Space& s, const std::vector<int32_t>& dofs);

// Vertex-star patch lists in the order of build_patch_solver (src/schwarz.cpp:62-83).
struct Patches {
  std::vector<int32_t> vertex;
  std::vector<int64_t> ptr;   // npatch+1
  std::vector<int32_t> dofs;  // ascending star_dofs per patch
  std::vector<int32_t> perm;  // patch_ordering, local indices
  std::vector<int32_t> cells; // npatch x 2^dim star cells (ascending ids)
  std::vector<int32_t> colour;  // vertex-parity colouring
};
Patches vertex_patches(const Space& s, bool skip_boundary);

// ---- coarse level (src/schwarz.cpp:139-165, 239-243) -------------------------
struct Coarse {
  int ndof = 0;
  std::vector<double> inverse;  // dense A_c^{-1} (identity rows on constrained)
  std::vector<int64_t> P_ptr;   // prolongation CSR, fine rows
  std::vector<int32_t> P_col;
  std::vector<double> P_val;
  std::vector<int32_t> cell_dofs;     // coarse (p = 1) cell maps, ncells x 2^d
  std::vector<uint8_t> constrained;   // coarse constrained flags
  std::vector<double> phat;           // (p+1) x 2 Q1 hats at the fine nodes, column-major
};
Coarse build_coarse(const Mesh& m, const Space& fine, const Basis1D& fb);
// Row-major inverse of a dense SPD matrix through its Cholesky factor.
std::vector<double> dense_spd_inverse(const std::vector<double>& A, int n);

// ---- synthetic configurations C1..C5 ------------------------
struct Problem {
  int config = 0, dim = 3, n = 8, p = 15;
  Mesh mesh;
  Basis1D basis;
  Space space;
  std::vector<double> rhs;
  std::vector<uint8_t> cell_kind;   // MapKind per cell
  std::vector<double> cell_mu;      // ncells x dim: kappa * mu^K
  std::vector<double> cell_xyz;     // ncells x 2^dim x 3 corner coordinates
  std::vector<double> cell_kappa;   // ncells
  Patches patches;
  Coarse coarse;
  // Linear elasticity (make_elastic_problem): ncomp = dim identical
  // components of `space` (vector_q_space, src/discretization.cpp:313-318);
  // rhs, patches and coarse are then the vector ones.
  int ncomp = 1;
  double lame_mu = 0.0, lame_lambda = 0.0;
  std::vector<double> Cmat;  // bundle.C = V^T W D on GL(p+1), (p+1)^2 column-major
  bool skip_boundary = true;
  // SIPG DG (make_dg_problem): dq_space, penalty eta
  bool dg = false;
  double eta = 0.0;
};
std::unique_ptr<Problem> make_problem(int config, int n_override, int p_override);
// Space, RHS (U[-1,1], or N(0,1) when `normal`, from `rng`), cell data, patches, coarse level.
void finish_problem(Problem& pb, std::mt19937_64& rng, bool normal);
std::unique_ptr<Problem> make_problem_from_mesh(Mesh mesh, int p, uint64_t seed);

// ---- symmetric interior-penalty DG (src/sipg.cpp) -------------------------------
// SIPG Poisson on dq_space(cartesian_mesh(dim, n^dim, unit), p), every boundary
// facet weak Dirichlet, eta < 0 -> sipg_default_eta; RHS load_vector(f = 1);
// DG vertex stars and the continuous Q1 coarse level (tests/test_sipg.cpp:184-197).
std::unique_ptr<Problem> make_dg_problem(int dim, int n, int p, double eta, bool skip_boundary);

// ---- linear elasticity (src/elasticity.cpp) ------------------------------------
// The reference's Table-2 problem generalised to dim = 2|3
// (tests/test_elasticity.cpp:24-30, 162-185): unit square/cube with n cells per
// axis, every boundary facet Neumann except x = 0 (Dirichlet), vector Q_p,
// body force -0.02 e_{dim-1} (vector_load, src/elasticity.cpp:169-202),
// Lame parameters mu, lambda; vector Q1 coarse level with the true form.
std::unique_ptr<Problem> make_elastic_problem(int dim, int n, int p, double mu, double lambda, bool skip_boundary);
// Vector star lists (star_dofs over all components, src/discretization.cpp:
// 266-297) and their patch_ordering, from the scalar ones.
Patches vector_patches(const Space& s, const Patches& scalar, int ncomp);
// The patch lists of `pb` for skip_boundary (scalar or vector).
void rebuild_patches(Problem& pb, bool skip_boundary);
// write_matrix_market (src/sparse.cpp:33-52) for a CSC matrix (column-major, like SpMat).
void write_matrix_market(const std::string& path, int64_t rows, int64_t cols, const int64_t* colptr,
                         const int32_t* rowidx, const double* val, bool symmetric);

}  // namespace fdmgpu::host
