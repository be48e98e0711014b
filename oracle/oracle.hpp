// ============================================================================
//  TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle") of the reference
//  fdmstar path (arXiv 2107.14758, /root/reference/proj).  It is the parity
//  checker for the B200 product and the CPU baseline of bench.py; it is never
//  linked, imported or executed by the product path (paper_2107_14758_b200/).
//
//  Plain C++20, no Eigen: small owned dense/sparse types stand in for the
//  Eigen containers the reference uses.  Every function cites the reference
//  file:line it restates (paths relative to /root/reference/proj).
//
//  Parity pin: the reference cannot be compiled here (Eigen3, doctest and
//  nlohmann json are absent).  The restatement is pinned by
//  the reference's own in-process known-answer tests (tests/test_*.cpp),
//  re-run against this code in tests/test_oracle_pins.py, plus committed
//  golden fixtures generated from it (tests/golden/).
//
//  Extensions NOT in the reference (marked "[ext]"), needed by configs C4/C5:
//    * per-cell coefficient kappa_K scaling mu^K (C4);
//    * tensor-grid and perturbed-vertex mesh generators in cartesian_mesh order;
//    * a sum-factorised quadrature apply for trilinear cells, equal to the
//      dense cell_matrix_quadrature to rounding (C5).
// ============================================================================
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace oracle {

using Vec = std::vector<double>;

// Dense column-major matrix (Eigen::MatrixXd stand-in).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rows, int cols, double v = 0.0) : r(rows), c(cols), a(size_t(rows) * cols, v) {}
  double& operator()(int i, int j) { return a[i + size_t(r) * j]; }
  double operator()(int i, int j) const { return a[i + size_t(r) * j]; }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  Mat transpose() const;
};
Mat matmul(const Mat& A, const Mat& B);

// Small sparse matrix held densely with a structural mask: the stored pattern
// matters (it drives symbolic Cholesky), the values are tiny.  Stand-in for the
// Eigen::SparseMatrix<double> fields of FdmBasis (include/fdmstar/fdm_basis.hpp:26-27).
struct PatMat {
  Mat val;
  std::vector<char> nz;  // same layout as val.a
  int rows() const { return val.r; }
  int cols() const { return val.c; }
  bool has(int i, int j) const { return nz[i + size_t(val.r) * j] != 0; }
  int nonzeros() const;
};

// Row-major CSR with sorted columns and summed duplicates (SpMat,
// include/fdmstar/sparse.hpp:11).  Explicit zeros are kept, as in Eigen.
struct Csr {
  int n = 0, m = 0;
  std::vector<int64_t> ptr;
  std::vector<int> col;
  std::vector<double> val;
  int64_t nnz() const { return ptr.empty() ? 0 : ptr.back(); }
};
struct Triplet {
  int i, j;
  double v;
};
// Eigen setFromTriplets semantics: duplicates summed in triplet order.
Csr csr_from_triplets(int n, int m, const std::vector<Triplet>& t);
Vec spmv(const Csr& A, const Vec& x);                          // src/sparse.cpp:9-18
Csr extract_submatrix(const Csr& A, const std::vector<int>& dofs);  // src/sparse.cpp:20-31
Vec spmv_transpose(const Csr& A, const Vec& x);                // Eigen P^T * x, row order

// ---- L0: quadrature, reference interval, dense eig, FDM basis ----------------
std::pair<double, double> legendre_value_deriv(int k, double x);  // src/quadrature.cpp:8-21
Vec gll_nodes(int p);                                             // src/quadrature.cpp:40-65
struct QuadratureRule {
  Vec points, weights;
  int size() const { return int(points.size()); }
};
QuadratureRule gauss_legendre_rule(int n);  // src/quadrature.cpp:67-95

enum class BasisKind { GllNodal, LobattoHierarchical, GlNodal };
struct ReferenceInterval {  // include/fdmstar/reference_interval.hpp:15-27
  int degree = 0;
  BasisKind kind = BasisKind::GllNodal;
  Vec nodes;
  Mat stiffness, mass, trace_values, trace_normal_derivs;
  void eval(const Vec& pts, Mat& values, Mat& derivs) const;
};
void lagrange_eval(const Vec& nodes, const Vec& pts, Mat& values, Mat& derivs);  // src/reference_interval.cpp:8-50
ReferenceInterval reference_operators(int p, BasisKind kind);  // src/reference_interval.cpp:100-130

std::pair<Vec, Mat> jacobi_sym_eig(Mat A);                        // src/dense_eig.cpp:11-65
std::pair<Vec, Mat> dense_sym_gen_eig(const Mat& A, const Mat& B);  // src/dense_eig.cpp:67-94

struct FdmBasis {  // include/fdmstar/fdm_basis.hpp:21-32
  int degree = 0;
  Mat S;
  Vec lambda;
  PatMat A_t, B_t;
  Vec parity;
  Mat deriv_traces;  // 2 x (p+1): outward normal derivative of each mode at the ends (src/fdm_basis.cpp:78)
};
FdmBasis fdm_basis(const ReferenceInterval& ref);  // src/fdm_basis.cpp:10-87

// ---- L1: kron, ordering, cholesky -------------------------------------------
Vec apply_axis(const Mat& M, const Vec& x, const std::vector<int>& dims, int axis);  // src/kron.cpp:20-38
struct KronTerm {
  double coeff = 1.0;
  std::vector<Mat> factors;
};
struct KronOperator {
  std::vector<int> dims;
  std::vector<KronTerm> terms;
  int rows() const;
  int cols() const;
};
Vec kron_apply(const KronOperator& op, const Vec& x);  // src/kron.cpp:40-55
Mat dense_kron(const Mat& A, const Mat& B);             // src/kron.cpp:57-63
Mat kron_materialize(const KronOperator& op);           // src/kron.cpp:81-90

enum class DofClass { Interior = 0, Facet = 1, Edge = 2, Vertex = 3 };
struct DofLabel {
  DofClass cls = DofClass::Interior;
  int entity = -1;
};
struct Ordering {
  std::vector<int> perm, group_offsets;
};
Ordering natural_ordering(int n);                          // src/ordering.cpp:9-15
Ordering patch_ordering(const std::vector<DofLabel>& labels);  // src/ordering.cpp:17-45

struct CholFactor {  // include/fdmstar/cholesky.hpp:15-27
  int n = 0;
  std::vector<int> perm;
  std::vector<int64_t> colptr;
  std::vector<int> rowind;
  std::vector<double> values;
  int64_t flops = 0;
  int64_t nnz() const { return int64_t(values.size()); }
  Vec solve(const Vec& b) const;  // src/cholesky.cpp:89-110
};
CholFactor cholesky(const Csr& A, const Ordering& ord);  // src/cholesky.cpp:9-87

// ---- L2: mesh, geometry, discretization, assembly ----------------------------
enum class FacetTag { Interior = 0, Dirichlet = 1, Neumann = 2 };
struct Facet {  // include/fdmstar/mesh.hpp:19-28
  std::array<int, 2> cell{-1, -1}, axis{-1, -1}, side{0, 0};
  bool tangential_flip = false, oriented = true;
  FacetTag tag = FacetTag::Interior;
  std::vector<int> vertices;
  int ncells() const { return cell[1] >= 0 ? 2 : 1; }
};
struct Mesh {  // include/fdmstar/mesh.hpp:37-55
  int dim = 2;
  std::vector<std::array<double, 3>> vertices;
  std::vector<std::vector<int>> cells;
  std::vector<Facet> facets;
  std::vector<std::vector<int>> vertex_cells;
  std::vector<double> cell_coeff;  // [ext] kappa_K per cell (empty => 1)
  int num_cells() const { return int(cells.size()); }
  int num_vertices() const { return int(vertices.size()); }
  int corners_per_cell() const { return 1 << dim; }
  double kappa(int c) const { return cell_coeff.empty() ? 1.0 : cell_coeff[c]; }
  void finalize();  // src/mesh.cpp:33-91
  static std::vector<int> local_facet_corners(int dim, int axis, int side);  // src/mesh.cpp:16-31
};
Mesh cartesian_mesh(int dim, const std::vector<int>& counts, const std::vector<double>& lengths);  // src/mesh.cpp:102-136
// [ext] axis-aligned tensor grid with the vertex/cell order of cartesian_mesh.
Mesh tensor_grid_mesh(int dim, const std::vector<std::vector<double>>& coords);
std::vector<char> boundary_vertices(const Mesh& mesh);  // src/schwarz.cpp:31-37

enum class MapKind { Cartesian, Affine, Bilinear };
struct CellGeometry {  // include/fdmstar/geometry.hpp:16-25
  int cell = -1;
  MapKind kind = MapKind::Bilinear;
  std::vector<Mat> jacobians, metric;
  Vec dets, quad_weights, mu, lengths;
};
Mat cell_map_jacobian(const Mesh& mesh, int cell, const Vec& xhat);  // src/geometry.cpp:33-43
std::array<double, 3> cell_map(const Mesh& mesh, int cell, const Vec& xhat);  // src/geometry.cpp:25-31
CellGeometry cell_geometry(const Mesh& mesh, int cell, const QuadratureRule& rule);  // src/geometry.cpp:45-104

enum class Owner { Cell, Facet, Edge, Vertex };
struct Discretization {  // include/fdmstar/discretization.hpp:20-58 (identical CG components)
  const Mesh* mesh = nullptr;
  // Components (vector_q_space, src/discretization.cpp:313-318): build_discretization
  // numbers component ci after components 0..ci-1 with its own first-touch map
  // (src/discretization.cpp:86-258), so with identical components the DOFs of
  // component ci are those of component 0 shifted by ci * nsc.  cell_dofs /
  // cell_modes hold component 0; the per-DOF arrays below span all ndof.
  int ncomp = 1, nsc = 0;
  std::vector<int> comp_dofs(int ci, int cell) const;
  std::vector<int> comp_modes(int ci, int cell) const;
  int degree = 0;
  int dofs_per_cell = 0;
  std::vector<std::vector<int>> cell_dofs, cell_modes;
  std::vector<std::vector<signed char>> cell_mode_flip_axis;
  int ndof = 0;
  std::vector<DofLabel> labels;
  std::vector<double> multiplicity;
  std::vector<char> constrained;
  std::vector<Owner> owner_kind;
  std::vector<int> owner_id;
  std::vector<std::array<int, 2>> edge_vertices;
  int dim() const { return mesh->dim; }
  int num_free() const;
  std::vector<int> star_dofs(int v) const;  // src/discretization.cpp:266-297
  void project_free(Vec& x) const;
};
Discretization q_space(const Mesh& mesh, int p);  // src/discretization.cpp:70-264,299-304
Discretization vector_q_space(const Mesh& mesh, int p);  // src/discretization.cpp:313-318
Discretization dq_space(const Mesh& mesh, int p);         // src/discretization.cpp:306-311 (discontinuous)

struct Bundle1D {  // include/fdmstar/assembly.hpp:19-25
  int degree = 0;
  ReferenceInterval ref;
  FdmBasis fdm;
  Mat C;
};
Bundle1D make_bundle(int degree);  // src/assembly.cpp:37-54 (CG family)
Bundle1D make_bundle_dg(int degree);  // src/assembly.cpp:37-54 (DG family: GL-nodal, FDM basis in GL representation)
FdmBasis to_gl_representation(const FdmBasis& fdm, const ReferenceInterval& gll);  // src/fdm_basis.cpp:89-101

struct GlobalOperator {  // include/fdmstar/assembly.hpp:31-52 (cell terms only)
  const Discretization* disc = nullptr;
  struct CellTerm {
    bool has_kron = false;
    KronOperator kron;
    Mat dense;
    // [ext] sum-factorised trilinear quadrature apply (replaces `dense` when set)
    bool sumfact = false;
    Vec G;  // per quadrature point: w*kappa*G (d*d, row-major), q^d points
    // vector spaces: (ci, cj, op) blocks, y_ci += op x_cj (include/fdmstar/assembly.hpp:40-44)
    struct KronBlock {
      int ci = 0, cj = 0;
      KronOperator op;
    };
    std::vector<KronBlock> kron_blocks;
  };
  std::vector<CellTerm> cells;
  // facet terms (include/fdmstar/assembly.hpp:40-45): y_{cell r} += op x_{cell s}
  struct FacetTerm {
    int facet = -1;
    struct Block {
      int r = 0, s = 0;
      KronOperator op;
    };
    std::vector<Block> blocks;
  };
  std::vector<FacetTerm> facets;
  const Bundle1D* bundle = nullptr;
  Vec apply(const Vec& x) const;   // src/assembly.cpp:56-88
  Csr assemble() const;            // src/assembly.cpp:90-129
};
KronOperator cell_matrix_cartesian(const ReferenceInterval& ref, const Vec& mu);  // src/assembly.cpp:143-154
Mat cell_matrix_quadrature(const Mesh& mesh, int cell, const ReferenceInterval& ref);  // src/assembly.cpp:198-215
// [ext] sumfact_threshold: Bilinear cells with (p+1)^d > threshold use the sum-factorised apply.
GlobalOperator poisson_operator(const Discretization& disc, const Bundle1D& bundle,
                                int sumfact_threshold = 4096);  // src/assembly.cpp:230-243
Vec sumfact_cell_apply(const Bundle1D& b, int d, const Vec& G, const Vec& u);  // [ext]

struct TransformedSystem {  // include/fdmstar/assembly.hpp:57-70
  const Discretization* disc = nullptr;
  Mat S;
  Vec parity;
  Csr At;
  Vec inv_multiplicity;
  std::vector<Vec> cell_mu;  // mu^K (times kappa_K) per cell, kept for patch-only assembly
  std::vector<std::vector<Vec>> comp_mu;  // vector (SDC) systems: per component, coeff * mu^K per cell
  Vec apply_S(const Vec& modes) const;   // src/assembly.cpp:308-324
  Vec apply_St(const Vec& nodal) const;  // src/assembly.cpp:326-342
  Vec mode_signs(int cell) const;        // src/assembly.cpp:293-306
};
TransformedSystem transformed_poisson(const Discretization& disc, const Bundle1D& bundle,
                                      bool eliminate = true, bool build_global = true);  // src/assembly.cpp:245-291
// Entries (lattice row, lattice col, value) of one cell block sum_a mu_a (x)_b (b==a ? A_t : B_t)
// on its structural pattern (src/assembly.cpp:263-270).
void cell_transformed_entries(const FdmBasis& f, int d, int p, const Vec& mu,
                              const std::function<void(int, int, double)>& fn);
// Patch matrix A~_j assembled from the star cells only (equal to
// extract_submatrix(At, dofs), src/sparse.cpp:20-31, without the global matrix).
Csr patch_matrix(const TransformedSystem& sys, const Bundle1D& bundle, int v, const std::vector<int>& dofs);
Vec load_vector(const Discretization& disc, const Bundle1D& bundle,
                const std::function<double(const std::array<double, 3>&)>& f);  // src/assembly.cpp:344-373

// ---- L3/L4: Schwarz, two-level, Krylov ---------------------------------------
enum class DampingFormula { TwoGrid, Smoother, Paper };
struct SolverConfig {  // include/fdmstar/schwarz.hpp:18-27
  bool damping_auto = true;
  double damping_value = 1.0;
  DampingFormula damping_formula = DampingFormula::TwoGrid;
  int lanczos_steps = 10;
  unsigned seed = 0x5EED;
  bool skip_boundary_patches = false;
  int coarse_degree = 1;
  int threads = 1;
};
using LinOp = std::function<Vec(const Vec&)>;
struct KrylovReport {  // include/fdmstar/krylov.hpp:12-20
  int iterations = 0;
  std::vector<double> residuals;
  double kappa = 0, lambda_min = 0, lambda_max = 0;
  bool converged = false;
  double wall_time = 0;
};
std::pair<double, double> tridiag_extremes(const std::vector<double>& diag, const std::vector<double>& off);  // src/krylov.cpp:18-27
std::pair<Vec, KrylovReport> pcg(const LinOp& A, const LinOp& Pinv, const Vec& b, double rtol, int maxit);  // src/krylov.cpp:29-83

struct PatchSolver {  // include/fdmstar/schwarz.hpp:33-45
  struct Patch {
    int vertex = -1;
    std::vector<int> dofs;
    CholFactor factor;
  };
  int ndof = 0, threads = 1;
  std::vector<Patch> patches;
  Vec apply(const Vec& r) const;  // src/schwarz.cpp:41-54
  int64_t factor_nnz() const;
};
// Patch DOF lists + orderings only (the symbolic half of build_patch_solver).
struct PatchList {
  std::vector<int> vertex;
  std::vector<std::vector<int>> dofs;
  std::vector<Ordering> ord;
};
PatchList patch_list(const Discretization& disc, const SolverConfig& config);  // src/schwarz.cpp:62-83
PatchSolver build_patch_solver(const Discretization& disc, const TransformedSystem& sys,
                               const Bundle1D& bundle, const SolverConfig& config,
                               const std::vector<int>* only = nullptr);  // src/schwarz.cpp:62-95

struct TwoLevel {  // include/fdmstar/schwarz.hpp:52-66
  LinOp A;
  std::shared_ptr<const TransformedSystem> sys;
  PatchSolver patches;
  double omega = 1.0, lambda_min = 0.0, lambda_max = 0.0;
  Csr prolong;
  std::shared_ptr<const CholFactor> coarse;
  Vec smooth(const Vec& r) const;  // src/schwarz.cpp:121-123
  Vec apply(const Vec& r) const;   // src/schwarz.cpp:125-133
  LinOp applier() const;
};
struct DampingEstimate {
  double omega = 1.0, lambda_min = 0.0, lambda_max = 0.0;
};
DampingEstimate estimate_damping(const LinOp& P, const LinOp& A, int n, const SolverConfig& config,
                                 const Discretization* disc);  // src/schwarz.cpp:97-119
void calibrate_damping(TwoLevel& tl, const Discretization& disc, const SolverConfig& config);  // src/schwarz.cpp:167-228
Csr build_prolongation(const Discretization& fine, const Discretization& coarse, const Mat& phat);  // src/schwarz.cpp:139-165 (all components)
TwoLevel build_poisson_twolevel(const Discretization& disc, const Bundle1D& bundle,
                                std::shared_ptr<const GlobalOperator> A, const SolverConfig& config,
                                bool calibrate = true);  // src/schwarz.cpp:230-252

void parallel_for(int n, int threads, const std::function<void(int)>& fn);  // src/schwarz.cpp:16-29

// ---- elasticity (src/elasticity.cpp, include/fdmstar/elasticity.hpp) --------
Vec sdc_axis_coefficients(int comp, int dim, double mu, double lambda);  // src/elasticity.cpp:7-11
Mat elasticity_primal_cell(const Mesh& mesh, int cell, const Bundle1D& bundle, double mu,
                           double lambda);  // src/elasticity.cpp:15-67
GlobalOperator elasticity_primal_operator(const Discretization& disc, const Bundle1D& bundle, double mu,
                                          double lambda);  // src/elasticity.cpp:69-120
TransformedSystem sdc_transformed(const Discretization& disc, const Bundle1D& bundle, double mu,
                                  double lambda);  // src/elasticity.cpp:122-167
Vec vector_load(const Discretization& disc, const Bundle1D& bundle,
                const std::function<std::array<double, 3>(const std::array<double, 3>&)>& f);  // src/elasticity.cpp:169-202
TwoLevel build_elasticity_twolevel(const Discretization& disc, const Bundle1D& bundle,
                                   std::shared_ptr<const GlobalOperator> A, double mu, double lambda,
                                   const SolverConfig& config, bool calibrate = true);  // src/elasticity.cpp:204-229
// ---- SIPG discontinuous Galerkin (src/sipg.cpp), Cartesian facets -----------
double sipg_default_eta(int p, int d);                                                        // src/sipg.cpp:7
Mat sipg_facet_dirichlet(const ReferenceInterval& ref, double mu_e, double eta, int side);     // src/sipg.cpp:20-25
Mat sipg_facet_interior(const ReferenceInterval& ref, double mu0, double mu1, double eta, int side0,
                        int side1);                                                           // src/sipg.cpp:27-45
PatMat sipg_facet_dirichlet_t(const FdmBasis& fdm, double mu_e, double eta, int side);        // src/sipg.cpp:47-62
PatMat sipg_facet_interior_t(const FdmBasis& fdm, double mu0, double mu1, double eta, int side0, int side1,
                             int block_r, int block_s);                                       // src/sipg.cpp:64-87
GlobalOperator dg_poisson_operator(const Discretization& disc, const Bundle1D& bundle,
                                   double eta);  // src/sipg.cpp:176-250 (Kronecker path)
TransformedSystem transformed_dg_poisson(const Discretization& disc, const Bundle1D& bundle,
                                         double eta);  // src/sipg.cpp:252-364 (Cartesian, unflipped)

// tag_boundary (src/mesh.cpp:323-332): boundary facets whose vertex centroid satisfies pred.
void tag_boundary(Mesh& mesh, const std::function<bool(const std::array<double, 3>&)>& pred, FacetTag tag);

// ---- [ext] synthetic configurations C1..C5 -----------------
struct ConfigSpec {
  int id = 0;
  int dim = 3, n = 8, p = 15;
};
struct Problem {
  int config = 0, p = 0;
  Mesh mesh;
  Discretization disc;
  Bundle1D bundle;
  Vec rhs;
};
// Builds mesh + space + RHS for config id (1..5); `n_override`/`p_override`
// (>0) give reduced variants with the same generators.
std::unique_ptr<Problem> make_problem(int config, int n_override = 0, int p_override = 0);
// [ext] Problem on an external mesh (the reference's load_mesh data: vertices,
// cells, facet tags applied as src/mesh.cpp:399-407 does); Q_p space, RHS
// U[-1,1] from std::mt19937_64(seed) over all DOFs, project_free.
std::unique_ptr<Problem> make_problem_from_mesh(Mesh mesh, int p, uint64_t seed);

}  // namespace oracle
