// A C++ caller of the drop-in boundary, compiled against include/fdmgpu.h and
// include/fdmhost.h only and linked against lib/libfdmgpu.so -- the shape of
// a reference-side integration.  The problem arrays come
// from the host setup mirror's getters (a reference integration takes them
// from its own Discretization / Bundle1D / build_patch_solver instead); every
// device call goes through the fdmgpu.h setters in the order
// build_poisson_twolevel (src/schwarz.cpp:230-252) produces its inputs:
//   create -> set_basis -> set_mesh_maps -> set_cell_coeffs -> set_patches
//   -> set_coarse -> factor -> calibrate_damping -> pcg (device vectors)
//   -> the LinOp form (fdmgpu_apply, host vectors) of one V-cycle.
// Prints one JSON line: omega, Lanczos extremes, PCG iterations, kappa, and a
// checksum of the V-cycle output.  tests/test_capi_consumer.py runs it on the
// GPU and compares with the Python path.
//
//   capi_consumer CONFIG [N P]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "fdmgpu.h"
#include "fdmhost.h"

namespace {

// The reference's error model: status codes back to exceptions with the
// library's message (fdm_check).
void check(fdmgpu_handle h, fdmgpu_status st, const char* what) {
  if (st == FDMGPU_OK) return;
  throw std::runtime_error(std::string(what) + ": " + (h ? fdmgpu_last_error(h) : fdmgpu_status_string(st)));
}
void host_check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + ": " + fdmhost_last_error());
}

struct DeviceVec {
  double* p = nullptr;
  explicit DeviceVec(size_t n) {
    if (cudaMalloc(&p, n * sizeof(double)) != cudaSuccess) throw std::runtime_error("cudaMalloc");
  }
  ~DeviceVec() { cudaFree(p); }
};

}  // namespace

int main(int argc, char** argv) {
  if (argc != 2 && argc != 4) {
    std::fprintf(stderr, "usage: %s CONFIG [N P]\n", argv[0]);
    return 2;
  }
  const int config = std::atoi(argv[1]);
  const int n = argc == 4 ? std::atoi(argv[2]) : 0, p_in = argc == 4 ? std::atoi(argv[3]) : 0;
  fdmgpu_handle h = nullptr;
  void* prob = nullptr;
  try {
    prob = fdmhost_problem_create(config, n, p_in);
    if (!prob) throw std::runtime_error(std::string("problem: ") + fdmhost_last_error());
    int64_t info[16];
    host_check(fdmhost_problem_info(prob, info), "problem_info");
    const int dim = int(info[0]), p = int(info[1]), ncells = int(info[2]), npatch = int(info[5]);
    const int64_t ndof = info[3], sum_nj = info[8], ncoarse = info[9], P_nnz = info[10];
    const int npc = int(info[7]), q = int(info[11]), n1 = p + 1;

    // --- inputs, as the reference's setup produces them ---
    std::vector<double> S(n1 * n1), At(n1 * n1), Bt(n1 * n1), Ah(n1 * n1), Bh(n1 * n1), lam(n1), par(n1), nodes(n1);
    std::vector<uint8_t> Anz(n1 * n1), Bnz(n1 * n1);
    host_check(fdmhost_get_basis(prob, S.data(), At.data(), Bt.data(), Anz.data(), Bnz.data(), lam.data(), par.data(),
                                 Ah.data(), Bh.data(), nodes.data()),
               "get_basis");
    std::vector<int32_t> cell_dofs(size_t(ncells) * npc), cell_modes(size_t(ncells) * npc);
    std::vector<uint8_t> constrained(ndof);
    std::vector<double> mult(ndof);
    host_check(fdmhost_get_maps(prob, cell_dofs.data(), cell_modes.data(), constrained.data(), mult.data(), nullptr,
                                nullptr),
               "get_maps");
    std::vector<double> kappa(ncells), mu(size_t(ncells) * dim), xyz(size_t(ncells) * (1 << dim) * 3);
    std::vector<uint8_t> kind(ncells);
    host_check(fdmhost_get_geometry(prob, nullptr, kappa.data(), mu.data(), kind.data(), xyz.data()), "get_geometry");
    std::vector<int32_t> vertex(npatch), pdofs(sum_nj), perm(sum_nj), cells(size_t(npatch) * (1 << dim)),
        colour(npatch);
    std::vector<int64_t> ptr(npatch + 1);
    host_check(fdmhost_get_patches(prob, vertex.data(), ptr.data(), pdofs.data(), perm.data(), cells.data(),
                                   colour.data()),
               "get_patches");
    std::vector<double> cinv(size_t(ncoarse) * ncoarse), Pval(P_nnz);
    std::vector<int64_t> Pptr(ndof + 1);
    std::vector<int32_t> Pcol(P_nnz);
    host_check(fdmhost_get_coarse(prob, cinv.data(), Pptr.data(), Pcol.data(), Pval.data()), "get_coarse");
    std::vector<double> rhs(ndof);
    host_check(fdmhost_get_rhs(prob, rhs.data()), "get_rhs");
    bool cartesian = true;
    for (uint8_t k : kind) cartesian = cartesian && k == 0;
    (void)q;
    if (!cartesian) throw std::runtime_error("this consumer drives Cartesian configurations (C1-C4)");

    // --- the device half of build_poisson_twolevel through fdmgpu.h ---
    check(h, fdmgpu_create(&h, dim, p, ncells, ndof, 0), "fdmgpu_create");
    check(h, fdmgpu_set_basis(h, S.data(), lam.data(), At.data(), Bt.data(), Anz.data(), Bnz.data(), Ah.data(),
                              Bh.data(), 0, nullptr, nullptr, nullptr, nullptr),
          "fdmgpu_set_basis");
    check(h, fdmgpu_set_mesh_maps(h, cell_dofs.data(), cell_modes.data(), nullptr, mult.data(), constrained.data()),
          "fdmgpu_set_mesh_maps");
    check(h, fdmgpu_set_cell_coeffs(h, kind.data(), mu.data(), nullptr, kappa.data()), "fdmgpu_set_cell_coeffs");
    check(h, fdmgpu_set_patches(h, npatch, vertex.data(), ptr.data(), pdofs.data(), perm.data(), cells.data()),
          "fdmgpu_set_patches");
    check(h, fdmgpu_set_coarse(h, int32_t(ncoarse), cinv.data(), Pptr.data(), Pcol.data(), Pval.data()),
          "fdmgpu_set_coarse");
    check(h, fdmgpu_factor(h), "fdmgpu_factor");
    double omega = 0, lmin = 0, lmax = 0;
    check(h, fdmgpu_calibrate_damping(h, 10, 0x5EED, 0, &omega, &lmin, &lmax), "fdmgpu_calibrate_damping");

    // pcg(A->applier(), tl.applier(), b, 1e-8, 200) with device-resident vectors
    DeviceVec b(ndof), x(ndof);
    if (cudaMemcpy(b.p, rhs.data(), ndof * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      throw std::runtime_error("cudaMemcpy");
    fdmgpu_krylov_report rep{};
    check(h, fdmgpu_pcg(h, b.p, x.p, 1e-8, 200, 2, &rep, nullptr), "fdmgpu_pcg");

    // the LinOp drop-in: one TwoLevel::apply on host vectors
    std::vector<double> z(ndof);
    check(h, fdmgpu_apply(h, FDMGPU_OP_VCYCLE, omega, rhs.data(), z.data(), 1), "fdmgpu_apply");
    double zz = 0;
    for (double v : z) zz += v * v;

    // the reference's NOT_SPD error path: negative coefficients -> cholesky throws
    std::vector<double> neg(mu);
    for (double& v : neg) v = -v;
    check(h, fdmgpu_set_cell_coeffs(h, kind.data(), neg.data(), nullptr, kappa.data()), "fdmgpu_set_cell_coeffs");
    const fdmgpu_status st = fdmgpu_factor(h);
    const std::string msg = fdmgpu_last_error(h);

    std::printf("{\"config\": %d, \"ndof\": %lld, \"npatch\": %d, \"omega\": %.17g, \"lambda_min\": %.17g, "
                "\"lambda_max\": %.17g, \"iterations\": %d, \"converged\": %d, \"kappa\": %.17g, "
                "\"vcycle_norm\": %.17g, \"not_spd_status\": %d, \"not_spd_message\": \"%s\"}\n",
                config, (long long)ndof, npatch, omega, lmin, lmax, rep.iterations, rep.converged, rep.kappa,
                std::sqrt(zz), int(st), msg.c_str());
    fdmgpu_destroy(h);
    fdmhost_problem_destroy(prob);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "capi_consumer: %s\n", e.what());
    if (h) fdmgpu_destroy(h);
    if (prob) fdmhost_problem_destroy(prob);
    return 1;
  }
}
