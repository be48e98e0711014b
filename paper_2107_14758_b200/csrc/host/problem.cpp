// Synthetic configurations C1..C5 of BASELINE.json:
// seeded libstdc++ std::mt19937_64 streams, the generator the reference
// tests use (tests/test_schwarz.cpp:13-20).  Seeds 0..4 for C1..C5; the RHS
// is the load-vector entries themselves, drawn over all DOFs in global order
// and then zeroed on constrained DOFs.  C4/C5 draw mesh data first and the
// RHS from the same stream afterwards.
#include <cmath>
#include <random>
#include <stdexcept>

#include "fdm_host.hpp"

namespace fdmgpu::host {

std::unique_ptr<Problem> make_problem(int config, int n_override, int p_override) {
  auto pb = std::make_unique<Problem>();
  pb->config = config;
  switch (config) {
    case 1: pb->dim = 2; pb->n = 8; pb->p = 7; break;
    case 2: pb->dim = 3; pb->n = 4; pb->p = 7; break;
    case 3: case 4: pb->dim = 3; pb->n = 8; pb->p = 15; break;
    case 5: pb->dim = 3; pb->n = 8; pb->p = 31; break;
    default: throw std::invalid_argument("make_problem: config must be 1..5");
  }
  if (n_override > 0) pb->n = n_override;
  if (p_override > 0) pb->p = p_override;
  const int d = pb->dim, n = pb->n;
  std::mt19937_64 rng(uint64_t(config - 1));
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  if (config == 4) {
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    std::vector<std::vector<double>> xs(d);
    for (int a = 0; a < d; ++a) {
      std::vector<double> w(n);
      double s = 0.0;
      for (auto& v : w) {
        v = std::exp(std::log(10.0) * u01(rng));
        s += v;
      }
      double acc = 0.0;
      xs[a].push_back(0.0);
      for (double v : w) xs[a].push_back(acc += v / s);
    }
    pb->mesh = tensor_grid_mesh(d, xs);
    std::lognormal_distribution<double> logn(0.0, 1.0);
    pb->mesh.kappa.resize(pb->mesh.num_cells());
    for (auto& k : pb->mesh.kappa) k = logn(rng);
  } else {
    pb->mesh = cartesian_mesh(d, std::vector<int>(d, n), std::vector<double>(d, 1.0));
    if (config == 5) {
      const double h = 1.0 / n;
      const auto onb = boundary_vertices(pb->mesh);
      for (int v = 0; v < pb->mesh.num_vertices(); ++v)
        if (!onb[v])
          for (int a = 0; a < d; ++a) pb->mesh.vertices[v][a] += 0.1 * h * uni(rng);
    }
  }
  finish_problem(*pb, rng, config == 3);
  return pb;
}

void finish_problem(Problem& pb, std::mt19937_64& rng, bool normal) {
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  pb.basis = make_bundle(pb.p);
  pb.space = q_space(pb.mesh, pb.p);
  pb.space.mesh = &pb.mesh;
  pb.rhs.resize(pb.space.ndof);
  if (normal) {
    std::normal_distribution<double> nd(0.0, 1.0);
    for (auto& v : pb.rhs) v = nd(rng);
  } else {
    for (auto& v : pb.rhs) v = uni(rng);
  }
  for (int i = 0; i < pb.space.ndof; ++i)
    if (pb.space.constrained[i]) pb.rhs[i] = 0.0;
  const int d = pb.dim, nc = pb.mesh.num_cells(), ncorner = 1 << d;
  pb.cell_kind.resize(nc);
  pb.cell_mu.resize(size_t(nc) * d);
  pb.cell_xyz.resize(size_t(nc) * ncorner * 3);
  pb.cell_kappa.resize(nc);
  for (int c = 0; c < nc; ++c) {
    CellCoeffs cc = cell_coeffs(pb.mesh, c, pb.basis);
    pb.cell_kind[c] = uint8_t(cc.kind);
    for (int a = 0; a < d; ++a) pb.cell_mu[size_t(c) * d + a] = cc.mu[a];
    for (int b = 0; b < ncorner; ++b)
      for (int r = 0; r < 3; ++r) pb.cell_xyz[(size_t(c) * ncorner + b) * 3 + r] = pb.mesh.vertices[pb.mesh.cells[c][b]][r];
    pb.cell_kappa[c] = pb.mesh.coeff(c);
  }
  pb.patches = vertex_patches(pb.space, /*skip_boundary=*/true);
  pb.coarse = build_coarse(pb.mesh, pb.space, pb.basis);
}

}  // namespace fdmgpu::host
