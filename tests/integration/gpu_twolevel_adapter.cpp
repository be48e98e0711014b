// Compile check of the INTEGRATION.md adapter against the declaration stubs
// of the reference headers (built by csrc/Makefile; not linked or run here --
// tests/integration/capi_consumer.cpp is the C++ caller that runs on the GPU).
#include "fdmstar_stub.hpp"
#include "gpu_twolevel.hpp"

namespace fdmstar {
// The reference solve with the GPU TwoLevel in place of build_poisson_twolevel.
std::pair<LinOp, LinOp> gpu_solver_linops(const GpuTwoLevel& gpu) { return {gpu.operator_A(), gpu.applier()}; }
GpuTwoLevel* make_gpu_twolevel(const Discretization& disc, const Bundle1D& b, const SolverConfig& cfg) {
  return new GpuTwoLevel(disc, b, cfg);
}
}  // namespace fdmstar
