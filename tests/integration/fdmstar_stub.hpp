// Declaration stubs of the reference API surface the GpuTwoLevel adapter
// (gpu_twolevel.hpp) touches, so the adapter compiles in
// this repo without the reference tree or Eigen.  Names, member names and
// signatures follow /root/reference/proj/include/fdmstar/*.hpp (cited per
// item); bodies are absent -- nothing here is linked or run.  A maintainer
// compiles gpu_twolevel.hpp against the real headers instead.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <utility>
#include <vector>

// ---- the few Eigen members the adapter uses (Eigen is column-major) ----------
namespace Eigen {
enum StorageOptions { ColMajor = 0, RowMajor = 1 };
class VectorXd {
 public:
  VectorXd() = default;
  explicit VectorXd(long n);
  long size() const;
  double* data();
  const double* data() const;
  double operator[](long i) const;
};
class Vector3d {
 public:
  double operator[](int i) const;
};
template <class Scalar, int Options = ColMajor>
class SparseMatrix {
 public:
  long rows() const;
  long cols() const;
  long outerSize() const;
  long nonZeros() const;
  const int* outerIndexPtr() const;
  const int* innerIndexPtr() const;
  const Scalar* valuePtr() const;
  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, long outer);
    explicit operator bool() const;
    InnerIterator& operator++();
    long row() const;
    long col() const;
    Scalar value() const;
  };
};
class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(long rows, long cols);
  template <class S, int O>
  MatrixXd(const SparseMatrix<S, O>& sparse);  // dense copy of a sparse matrix
  long rows() const;
  long cols() const;
  double* data();
  const double* data() const;
  double& operator()(long r, long c);
  double operator()(long r, long c) const;
};
}  // namespace Eigen

namespace fdmstar {

// mesh.hpp:18-54
enum class FacetTag { Interior = 0, Dirichlet = 1, Neumann = 2 };
struct Facet {
  std::array<int, 2> cell{-1, -1};
  FacetTag tag = FacetTag::Interior;
  std::vector<int> vertices;
  int ncells() const { return cell[1] >= 0 ? 2 : 1; }
};
struct PatchTopology {
  int vertex = -1;
  std::vector<int> cells;  // ascending
};
struct Mesh {
  int dim = 2;
  std::vector<Eigen::Vector3d> vertices;
  std::vector<std::vector<int>> cells;
  std::vector<Facet> facets;
  int num_cells() const;
  int num_vertices() const;
};
PatchTopology vertex_star(const Mesh& mesh, int v);  // mesh.hpp:72

// ordering.hpp:9-28
struct Ordering {
  std::vector<int> perm;
  std::vector<int> group_offsets;
};
enum class DofClass { Interior = 0, Facet = 1, Edge = 2, Vertex = 3 };
struct DofLabel {
  DofClass cls = DofClass::Interior;
  int entity = -1;
};
Ordering patch_ordering(const std::vector<DofLabel>& labels);

// quadrature.hpp:8-21, reference_interval.hpp:16-30, fdm_basis.hpp:19-31
struct QuadratureRule {
  Eigen::VectorXd points, weights;
  int size() const;
};
QuadratureRule gauss_legendre_rule(int n);
struct ReferenceInterval {
  int degree = 0;
  Eigen::VectorXd nodes;
  Eigen::MatrixXd stiffness, mass;
  Eigen::MatrixXd eval_values(const Eigen::VectorXd& pts) const;
  Eigen::MatrixXd eval_derivs(const Eigen::VectorXd& pts) const;
};
struct FdmBasis {
  int degree = 0;
  Eigen::MatrixXd S;
  Eigen::VectorXd lambda;
  Eigen::SparseMatrix<double> A_t, B_t;
};

// discretization.hpp:14-64
enum class Family1D { CG, DG };
struct Discretization {
  struct Component {
    int dofs_per_cell = 0;
    std::vector<std::vector<int>> cell_dofs, cell_modes;
  };
  const Mesh* mesh = nullptr;
  std::vector<Component> comps;
  int ndof = 0;
  std::vector<DofLabel> labels;
  std::vector<double> multiplicity;
  std::vector<char> constrained;
  std::vector<int> star_dofs(int v) const;
};
Discretization q_space(const Mesh& mesh, int p);

// geometry.hpp:12-32
enum class MapKind { Cartesian, Affine, Bilinear };
struct CellGeometry {
  MapKind kind = MapKind::Bilinear;
  Eigen::VectorXd mu;
};
CellGeometry cell_geometry(const Mesh& mesh, int cell, const QuadratureRule& rule);

// sparse.hpp:11, assembly.hpp:19-56, 89, krylov.hpp:10
using SpMat = Eigen::SparseMatrix<double, Eigen::RowMajor>;
struct Bundle1D {
  Family1D family = Family1D::CG;
  int degree = 0;
  ReferenceInterval ref;
  FdmBasis fdm;
  Eigen::MatrixXd C;
};
Bundle1D make_bundle(Family1D family, int degree);
struct GlobalOperator {
  Eigen::MatrixXd assemble_dense() const;
};
GlobalOperator poisson_operator(const Discretization& disc, const Bundle1D& bundle);
using LinOp = std::function<Eigen::VectorXd(const Eigen::VectorXd&)>;

// schwarz.hpp:12-26, 82-85
enum class DampingFormula { TwoGrid, Smoother, Paper };
struct SolverConfig {
  bool damping_auto = true;
  double damping_value = 1.0;
  DampingFormula damping_formula = DampingFormula::TwoGrid;
  int lanczos_steps = 10;
  unsigned seed = 0x5EED;
  bool skip_boundary_patches = false;
  int coarse_degree = 1;
  int threads = 1;
};
SpMat build_prolongation(const Discretization& fine, const Discretization& coarse,
                         const std::vector<std::array<Eigen::MatrixXd, 3>>& phat);

}  // namespace fdmstar
