// GpuTwoLevel: the reference-side adapter a maintainer adds to fdmstar to run
// the vertex-star Schwarz path on the B200 library.  It
// builds the fdmgpu handle from the reference's own setup objects -- exactly
// the inputs build_poisson_twolevel (src/schwarz.cpp:230-252) computes -- and
// exposes the TwoLevel / GlobalOperator LinOps (include/fdmstar/krylov.hpp:10,
// schwarz.hpp:52-66, src/schwarz.cpp:135-137), so
//   auto [x, rep] = pcg(gpu.operator_A(), gpu.applier(), b, 1e-8, maxit);
// replaces the CPU solve unchanged.  Compiled in this repo against the
// declaration stubs of fdmstar_stub.hpp (gpu_twolevel_adapter.cpp); against
// the real headers include <fdmstar/...> instead.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fdmgpu.h"

namespace fdmstar {

// Status codes back to the reference's exception types and messages.
inline void fdm_check(fdmgpu_handle h, fdmgpu_status st) {
  if (st == FDMGPU_OK) return;
  const std::string msg = h ? fdmgpu_last_error(h) : fdmgpu_status_string(st);
  if (st == FDMGPU_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);  // NOT_SPD / INDEFINITE carry the reference's text
}

// Dense inverse of the SPD coarse matrix (row-major, as fdmgpu_set_coarse
// takes it): Cholesky, then one solve per unit vector.
inline std::vector<double> dense_spd_inverse(const Eigen::MatrixXd& A) {
  const int n = int(A.rows());
  std::vector<double> L(size_t(n) * n, 0.0), inv(size_t(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = A(j, j);
    for (int k = 0; k < j; ++k) d -= L[size_t(j) * n + k] * L[size_t(j) * n + k];
    if (!(d > 0.0)) throw std::runtime_error("cholesky: matrix not SPD at pivot " + std::to_string(j));
    L[size_t(j) * n + j] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = A(i, j);
      for (int k = 0; k < j; ++k) s -= L[size_t(i) * n + k] * L[size_t(j) * n + k];
      L[size_t(i) * n + j] = s / L[size_t(j) * n + j];
    }
  }
  std::vector<double> y(n);
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = i == c ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[size_t(i) * n + k] * y[k];
      y[i] = s / L[size_t(i) * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= L[size_t(k) * n + i] * inv[size_t(k) * n + c];
      inv[size_t(i) * n + c] = s / L[size_t(i) * n + i];
    }
  }
  return inv;
}

// GPU-backed TwoLevel for the scalar continuous Poisson problem.
struct GpuTwoLevel {
  fdmgpu_handle h = nullptr;
  int n = 0;

  GpuTwoLevel(const Discretization& disc, const Bundle1D& b, const SolverConfig& cfg, int device = 0) {
    const Mesh& mesh = *disc.mesh;
    const auto& comp = disc.comps[0];
    const int d = mesh.dim, p = b.degree, n1 = p + 1, ncorner = 1 << d;
    n = disc.ndof;
    fdm_check(h, fdmgpu_create(&h, d, p, mesh.num_cells(), disc.ndof, device));
    try {
      // 1D basis (Eigen storage is column-major, as the ABI expects)
      Eigen::MatrixXd At(b.fdm.A_t), Bt(b.fdm.B_t);
      std::vector<uint8_t> Anz(size_t(n1) * n1, 0), Bnz(size_t(n1) * n1, 0);
      for (long k = 0; k < b.fdm.A_t.outerSize(); ++k)
        for (Eigen::SparseMatrix<double>::InnerIterator it(b.fdm.A_t, k); it; ++it) Anz[it.row() + n1 * it.col()] = 1;
      for (long k = 0; k < b.fdm.B_t.outerSize(); ++k)
        for (Eigen::SparseMatrix<double>::InnerIterator it(b.fdm.B_t, k); it; ++it) Bnz[it.row() + n1 * it.col()] = 1;
      const QuadratureRule gl = gauss_legendre_rule(p + 2);  // the true-form rule (src/assembly.cpp:198-215)
      Eigen::MatrixXd Vq = b.ref.eval_values(gl.points), Dq = b.ref.eval_derivs(gl.points);
      fdm_check(h, fdmgpu_set_basis(h, b.fdm.S.data(), b.fdm.lambda.data(), At.data(), Bt.data(), Anz.data(),
                                    Bnz.data(), b.ref.stiffness.data(), b.ref.mass.data(), p + 2, gl.points.data(),
                                    gl.weights.data(), Vq.data(), Dq.data()));
      // DOF maps (Discretization::Component, include/fdmstar/discretization.hpp:22-34)
      std::vector<int32_t> cd, cm;
      for (int c = 0; c < mesh.num_cells(); ++c) {
        cd.insert(cd.end(), comp.cell_dofs[c].begin(), comp.cell_dofs[c].end());
        cm.insert(cm.end(), comp.cell_modes[c].begin(), comp.cell_modes[c].end());
      }
      std::vector<uint8_t> con(disc.constrained.begin(), disc.constrained.end());
      fdm_check(h, fdmgpu_set_mesh_maps(h, cd.data(), cm.data(), nullptr, disc.multiplicity.data(), con.data()));
      // per-cell geometry: map kind, surrogate mu (src/geometry.cpp:91-102), corners
      std::vector<uint8_t> kind;
      std::vector<double> mu, xyz;
      for (int c = 0; c < mesh.num_cells(); ++c) {
        const CellGeometry g = cell_geometry(mesh, c, gl);
        kind.push_back(uint8_t(g.kind));
        for (int a = 0; a < d; ++a) mu.push_back(g.mu[a]);
        for (int v : mesh.cells[c])
          for (int r = 0; r < 3; ++r) xyz.push_back(mesh.vertices[v][r]);
      }
      fdm_check(h, fdmgpu_set_cell_coeffs(h, kind.data(), mu.data(), xyz.data(), nullptr));
      // patches exactly as build_patch_solver lists them (src/schwarz.cpp:62-83)
      std::vector<char> on_boundary(mesh.num_vertices(), 0);
      for (const Facet& f : mesh.facets)
        if (f.ncells() == 1)
          for (int v : f.vertices) on_boundary[v] = 1;
      std::vector<int32_t> vert, dofs, perm, cells;
      std::vector<int64_t> ptr{0};
      for (int v = 0; v < mesh.num_vertices(); ++v) {
        if (cfg.skip_boundary_patches && on_boundary[v]) continue;
        const std::vector<int> dv = disc.star_dofs(v);
        if (dv.empty()) continue;
        std::vector<DofLabel> lab;
        for (int g : dv) lab.push_back(disc.labels[g]);
        const Ordering ord = patch_ordering(lab);
        vert.push_back(v);
        dofs.insert(dofs.end(), dv.begin(), dv.end());
        perm.insert(perm.end(), ord.perm.begin(), ord.perm.end());
        const PatchTopology star = vertex_star(mesh, v);
        for (int k = 0; k < ncorner; ++k) cells.push_back(k < int(star.cells.size()) ? star.cells[k] : -1);
        ptr.push_back(int64_t(dofs.size()));
      }
      fdm_check(h, fdmgpu_set_patches(h, int32_t(vert.size()), vert.data(), ptr.data(), dofs.data(), perm.data(),
                                      cells.data()));
      // coarse level (src/schwarz.cpp:239-243): the Q1 true form, its inverse, and
      // build_prolongation with the Q1 hats at the fine nodes
      const Discretization coarse = q_space(mesh, cfg.coarse_degree);
      const Bundle1D cb = make_bundle(Family1D::CG, cfg.coarse_degree);
      const std::vector<double> cinv = dense_spd_inverse(poisson_operator(coarse, cb).assemble_dense());
      const Eigen::MatrixXd hat = cb.ref.eval_values(b.ref.nodes);  // (p+1) x 2
      const SpMat P = build_prolongation(disc, coarse, {{hat, hat, hat}});
      std::vector<int64_t> Pptr(P.outerIndexPtr(), P.outerIndexPtr() + P.rows() + 1);
      fdm_check(h, fdmgpu_set_coarse(h, int32_t(coarse.ndof), cinv.data(), Pptr.data(), P.innerIndexPtr(),
                                     P.valuePtr()));
      // the same prolongation cell by cell (sum-factorised kernels instead of the CSR)
      std::vector<int32_t> ccd;
      for (int c = 0; c < mesh.num_cells(); ++c)
        ccd.insert(ccd.end(), coarse.comps[0].cell_dofs[c].begin(), coarse.comps[0].cell_dofs[c].end());
      std::vector<uint8_t> ccon(coarse.constrained.begin(), coarse.constrained.end());
      fdm_check(h, fdmgpu_set_coarse_cells(h, ccd.data(), ccon.data(), hat.data()));
      fdm_check(h, fdmgpu_factor(h));  // cholesky() of every patch, batched
      double omega = 0, lmin = 0, lmax = 0;
      if (cfg.damping_auto)
        fdm_check(h, fdmgpu_calibrate_damping(h, cfg.lanczos_steps, cfg.seed, int(cfg.damping_formula), &omega, &lmin,
                                              &lmax));
      else
        fdm_check(h, fdmgpu_set_omega(h, cfg.damping_value));
    } catch (...) {
      fdmgpu_destroy(h);
      throw;
    }
  }
  GpuTwoLevel(const GpuTwoLevel&) = delete;
  GpuTwoLevel& operator=(const GpuTwoLevel&) = delete;
  ~GpuTwoLevel() { fdmgpu_destroy(h); }

  double omega() const {
    double w = 0;
    fdm_check(h, fdmgpu_get_omega(h, &w));
    return w;
  }
  // LinOp drop-ins on host vectors: one H2D + one D2H per call
  LinOp applier() const {  // TwoLevel::applier (src/schwarz.cpp:135-137)
    return [this](const Eigen::VectorXd& r) {
      Eigen::VectorXd z(n);
      fdm_check(h, fdmgpu_apply(h, FDMGPU_OP_VCYCLE, omega(), r.data(), z.data(), 1));
      return z;
    };
  }
  LinOp smoother() const {  // TwoLevel::smooth (src/schwarz.cpp:121-123)
    return [this](const Eigen::VectorXd& r) {
      Eigen::VectorXd z(n);
      fdm_check(h, fdmgpu_apply(h, FDMGPU_OP_SMOOTH, 0.0, r.data(), z.data(), 1));
      return z;
    };
  }
  LinOp operator_A() const {  // GlobalOperator::applier (src/assembly.cpp:133-135)
    return [this](const Eigen::VectorXd& x) {
      Eigen::VectorXd y(n);
      fdm_check(h, fdmgpu_apply(h, FDMGPU_OP_A, 0.0, x.data(), y.data(), 1));
      return y;
    };
  }
};

}  // namespace fdmstar
