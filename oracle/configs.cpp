// TEST INFRASTRUCTURE ONLY — oracle restatement, see oracle.hpp header.
// [ext] Synthetic inputs for BASELINE.json configs C1..C5.
// RNG: libstdc++ std::mt19937_64 with the standard distributions, the same
// generator the reference tests use (tests/test_schwarz.cpp:13-20).
#include <cmath>
#include <random>
#include <stdexcept>

#include "oracle.hpp"

namespace oracle {

std::unique_ptr<Problem> make_problem(int config, int n_override, int p_override) {
  auto pb = std::make_unique<Problem>();
  pb->config = config;
  int dim = 3, n = 8, p = 15;
  switch (config) {
    case 1: dim = 2; n = 8; p = 7; break;
    case 2: dim = 3; n = 4; p = 7; break;
    case 3: case 4: dim = 3; n = 8; p = 15; break;
    case 5: dim = 3; n = 8; p = 31; break;
    default: throw std::invalid_argument("make_problem: config must be 1..5");
  }
  if (n_override > 0) n = n_override;
  if (p_override > 0) p = p_override;
  pb->p = p;
  std::mt19937_64 rng(uint64_t(config - 1));  // seeds 0..4 for C1..C5
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  if (config == 4) {
    // Per-axis widths exp(ln10 U[0,1)), normalised; then kappa_K ~ lognormal(0,1).
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    std::vector<std::vector<double>> coords(dim);
    for (int a = 0; a < dim; ++a) {
      std::vector<double> w(n);
      double s = 0.0;
      for (int i = 0; i < n; ++i) {
        w[i] = std::exp(std::log(10.0) * u01(rng));
        s += w[i];
      }
      coords[a].push_back(0.0);
      double acc = 0.0;
      for (int i = 0; i < n; ++i) {
        acc += w[i] / s;
        coords[a].push_back(acc);
      }
    }
    pb->mesh = tensor_grid_mesh(dim, coords);
    std::lognormal_distribution<double> logn(0.0, 1.0);
    pb->mesh.cell_coeff.resize(pb->mesh.num_cells());
    for (auto& k : pb->mesh.cell_coeff) k = logn(rng);
  } else {
    pb->mesh = cartesian_mesh(dim, std::vector<int>(dim, n), std::vector<double>(dim, 1.0));
    if (config == 5) {
      const double h = 1.0 / n;
      const std::vector<char> onb = boundary_vertices(pb->mesh);
      for (int v = 0; v < pb->mesh.num_vertices(); ++v) {
        if (onb[v]) continue;
        for (int a = 0; a < dim; ++a) pb->mesh.vertices[v][a] += 0.1 * h * uni(rng);
      }
    }
  }
  pb->disc = q_space(pb->mesh, p);
  pb->disc.mesh = &pb->mesh;
  pb->bundle = make_bundle(p);
  pb->rhs.resize(pb->disc.ndof);
  if (config == 3) {
    std::normal_distribution<double> nd(0.0, 1.0);
    for (auto& v : pb->rhs) v = nd(rng);
  } else {
    for (auto& v : pb->rhs) v = uni(rng);
  }
  pb->disc.project_free(pb->rhs);
  return pb;
}

std::unique_ptr<Problem> make_problem_from_mesh(Mesh mesh, int p, uint64_t seed) {
  auto pb = std::make_unique<Problem>();
  pb->config = 0;
  pb->p = p;
  pb->mesh = std::move(mesh);
  pb->disc = q_space(pb->mesh, p);
  pb->disc.mesh = &pb->mesh;
  pb->bundle = make_bundle(p);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  pb->rhs.resize(pb->disc.ndof);
  for (auto& v : pb->rhs) v = uni(rng);
  pb->disc.project_free(pb->rhs);
  return pb;
}

}  // namespace oracle
