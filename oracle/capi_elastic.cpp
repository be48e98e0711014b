// TEST INFRASTRUCTURE ONLY — extern "C" surface of the oracle's elasticity
// restatement (oracle/elasticity.cpp) for the Python tests and bench.py's
// CPU legs.  Problem: the reference's Table-2 "table" mesh generalised to
// dim = 2|3 (tests/test_elasticity.cpp:24-30: cartesian_mesh on the unit
// square/cube, every boundary facet Neumann, x = 0 Dirichlet), vector Q_p
// space, body force f = -0.02 e_{dim-1} (tests/test_elasticity.cpp:170-172).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

struct ECtx {
  Mesh mesh;
  Discretization disc;
  Bundle1D bundle;
  double mu = 1.0, lambda = 0.0;
  SolverConfig cfg;
  std::shared_ptr<GlobalOperator> A;
  std::unique_ptr<TwoLevel> tl;
  Vec rhs;
};

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

ECtx* E(void* h) { return static_cast<ECtx*>(h); }
}  // namespace

extern "C" {

const char* oracle_elastic_last_error() { return g_err.c_str(); }

// skip_boundary: SolverConfig::skip_boundary_patches (reference default 0).
void* oracle_elastic_create(int dim, int n, int p, double mu, double lambda, int skip_boundary, int threads) {
  ECtx* out = nullptr;
  guard([&] {
    auto c = std::make_unique<ECtx>();
    c->mesh = cartesian_mesh(dim, std::vector<int>(dim, n), std::vector<double>(dim, 1.0));
    tag_boundary(c->mesh, [](const std::array<double, 3>&) { return true; }, FacetTag::Neumann);
    tag_boundary(c->mesh, [](const std::array<double, 3>& x) { return std::abs(x[0]) < 1e-12; }, FacetTag::Dirichlet);
    c->disc = vector_q_space(c->mesh, p);
    c->disc.mesh = &c->mesh;
    c->bundle = make_bundle(p);
    c->mu = mu;
    c->lambda = lambda;
    c->cfg.skip_boundary_patches = skip_boundary != 0;
    c->cfg.threads = threads;
    c->A = std::make_shared<GlobalOperator>(elasticity_primal_operator(c->disc, c->bundle, mu, lambda));
    const int d = dim;
    c->rhs = vector_load(c->disc, c->bundle, [d](const std::array<double, 3>&) {
      std::array<double, 3> f{0.0, 0.0, 0.0};
      f[d - 1] = -0.02;
      return f;
    });
    c->disc.project_free(c->rhs);  // zero_constrained
    out = c.release();
  });
  return out;
}

void oracle_elastic_destroy(void* h) { delete E(h); }

// out: dim, p, ncells, ndof (all components), scalar block size, nfree, dofs per cell (one component)
int oracle_elastic_info(void* h, int64_t* out) {
  return guard([&] {
    const auto& d = E(h)->disc;
    int64_t v[7] = {d.dim(), d.degree, E(h)->mesh.num_cells(), d.ndof, d.nsc, d.num_free(), d.dofs_per_cell};
    std::memcpy(out, v, sizeof(v));
  });
}

int oracle_elastic_rhs(void* h, double* out) {
  return guard([&] { std::memcpy(out, E(h)->rhs.data(), E(h)->rhs.size() * 8); });
}

// random_free of tests/test_elasticity.cpp:13-20 (U[-1,1] from mt19937_64(seed), project_free)
int oracle_elastic_random_free(void* h, uint64_t seed, double* out) {
  return guard([&] {
    const auto& d = E(h)->disc;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> uni(-1, 1);
    Vec x(d.ndof);
    for (auto& v : x) v = uni(rng);
    d.project_free(x);
    std::memcpy(out, x.data(), x.size() * 8);
  });
}

// Component-0 cell maps (ncells x (p+1)^d), constrained / multiplicity (ndof).
int oracle_elastic_maps(void* h, int32_t* cell_dofs, uint8_t* constrained, double* multiplicity) {
  return guard([&] {
    const auto& d = E(h)->disc;
    for (size_t c = 0; c < d.cell_dofs.size(); ++c)
      for (int l = 0; l < d.dofs_per_cell; ++l) cell_dofs[c * d.dofs_per_cell + l] = d.cell_dofs[c][l];
    for (int i = 0; i < d.ndof; ++i) {
      constrained[i] = uint8_t(d.constrained[i]);
      multiplicity[i] = d.multiplicity[i];
    }
  });
}

int oracle_elastic_apply_A(void* h, const double* in, double* out) {
  return guard([&] {
    Vec x(in, in + E(h)->disc.ndof);
    Vec y = E(h)->A->apply(x);
    std::memcpy(out, y.data(), y.size() * 8);
  });
}

// build_elasticity_twolevel (src/elasticity.cpp:204-229); calibrate = 0 keeps omega = 1.
int oracle_elastic_build(void* h, int calibrate) {
  return guard([&] {
    ECtx* c = E(h);
    c->tl = std::make_unique<TwoLevel>(
        build_elasticity_twolevel(c->disc, c->bundle, c->A, c->mu, c->lambda, c->cfg, calibrate != 0));
  });
}

// out: omega, lambda_min, lambda_max, coarse ndof, patches, sum n_j
int oracle_elastic_twolevel_info(void* h, double* out) {
  return guard([&] {
    const auto& tl = *E(h)->tl;
    out[0] = tl.omega;
    out[1] = tl.lambda_min;
    out[2] = tl.lambda_max;
    out[3] = tl.coarse->n;
    out[4] = double(tl.patches.patches.size());
    double s = 0;
    for (const auto& p : tl.patches.patches) s += double(p.dofs.size());
    out[5] = s;
  });
}

int oracle_elastic_set_omega(void* h, double w) {
  return guard([&] { E(h)->tl->omega = w; });
}

// which: 0 apply_St, 1 apply_S, 2 PatchSolver::apply, 3 smooth, 4 V-cycle
int oracle_elastic_op(void* h, int which, const double* in, double* out) {
  return guard([&] {
    ECtx* c = E(h);
    Vec x(in, in + c->disc.ndof), y;
    const auto& tl = *c->tl;
    switch (which) {
      case 0: y = tl.sys->apply_St(x); break;
      case 1: y = tl.sys->apply_S(x); break;
      case 2: y = tl.patches.apply(x); break;
      case 3: y = tl.smooth(x); break;
      case 4: y = tl.apply(x); break;
      default: throw std::invalid_argument("oracle_elastic_op: which 0..4");
    }
    std::memcpy(out, y.data(), y.size() * 8);
  });
}

// Patch lists: ptr (npatch+1), dofs (sum n_j), vertex (npatch).
int oracle_elastic_patches(void* h, int64_t* ptr, int32_t* dofs, int32_t* vertex) {
  return guard([&] {
    const auto& ps = E(h)->tl->patches.patches;
    ptr[0] = 0;
    for (size_t j = 0; j < ps.size(); ++j) {
      ptr[j + 1] = ptr[j] + int64_t(ps[j].dofs.size());
      std::memcpy(dofs + ptr[j], ps[j].dofs.data(), ps[j].dofs.size() * 4);
      vertex[j] = ps[j].vertex;
    }
  });
}

// Dense assembled operator (row-major ndof^2): which 0 = the true form,
// 1 = its diagonal (ci == cj) Kronecker blocks only, the SDC matrix of
// tests/test_elasticity.cpp:115-121.
int oracle_elastic_assemble_dense(void* h, int which, double* out) {
  return guard([&] {
    ECtx* c = E(h);
    GlobalOperator op = *c->A;
    if (which == 1)
      for (auto& t : op.cells) {
        std::vector<GlobalOperator::CellTerm::KronBlock> keep;
        for (auto& b : t.kron_blocks)
          if (b.ci == b.cj) keep.push_back(b);
        t.kron_blocks = keep;
      }
    const Csr A = op.assemble();
    const int n = c->disc.ndof;
    std::memset(out, 0, size_t(n) * n * 8);
    for (int i = 0; i < n; ++i)
      for (int64_t q = A.ptr[i]; q < A.ptr[i + 1]; ++q) out[size_t(i) * n + A.col[q]] = A.val[q];
  });
}

// Kronecker cell blocks materialised (kron) and the dense quadrature cell
// matrix (quad) of `cell`, both (d nloc)^2 column-major, component-major.
int oracle_elastic_cell_matrices(void* h, int cell, double* kron, double* quad) {
  return guard([&] {
    ECtx* c = E(h);
    const int d = c->disc.dim(), nloc = c->disc.dofs_per_cell, N = d * nloc;
    std::memset(kron, 0, size_t(N) * N * 8);
    for (const auto& b : c->A->cells[cell].kron_blocks) {
      const Mat K = kron_materialize(b.op);
      for (int j = 0; j < nloc; ++j)
        for (int i = 0; i < nloc; ++i) kron[size_t(b.ci * nloc + i) + size_t(N) * (b.cj * nloc + j)] = K(i, j);
    }
    const Mat Q = elasticity_primal_cell(c->mesh, cell, c->bundle, c->mu, c->lambda);
    std::memcpy(quad, Q.a.data(), Q.a.size() * 8);
  });
}

// pcg (src/krylov.cpp:29-83) with A = the true form and precond 0 identity,
// 1 smooth, 2 V-cycle.  report: iterations, converged, kappa, lambda_min, lambda_max.
int oracle_elastic_pcg(void* h, const double* b, double* x, double rtol, int maxit, int precond, double* report,
                       double* residuals) {
  return guard([&] {
    ECtx* c = E(h);
    Vec bb(b, b + c->disc.ndof);
    auto A = c->A;
    LinOp Aop = [A](const Vec& v) { return A->apply(v); };
    LinOp P;
    const TwoLevel* tl = c->tl.get();
    if (precond == 0)
      P = [](const Vec& v) { return v; };
    else if (precond == 1)
      P = [tl](const Vec& v) { return tl->smooth(v); };
    else
      P = tl->applier();
    auto [xx, rep] = pcg(Aop, P, bb, rtol, maxit);
    std::memcpy(x, xx.data(), xx.size() * 8);
    report[0] = rep.iterations;
    report[1] = rep.converged;
    report[2] = rep.kappa;
    report[3] = rep.lambda_min;
    report[4] = rep.lambda_max;
    for (size_t k = 0; k < rep.residuals.size(); ++k) residuals[k] = rep.residuals[k];
  });
}

// sdc_axis_coefficients (src/elasticity.cpp:7-11)
int oracle_sdc_axis_coefficients(int comp, int dim, double mu, double lambda, double* out) {
  return guard([&] {
    const Vec c = sdc_axis_coefficients(comp, dim, mu, lambda);
    std::memcpy(out, c.data(), c.size() * 8);
  });
}

}  // extern "C"

// ---- SIPG DG (oracle/sipg.cpp) -------------------------------------------------
namespace {
struct DCtx {
  Mesh mesh;
  Discretization disc;
  Bundle1D bundle;
  double eta = 0.0;
  SolverConfig cfg;
  std::shared_ptr<GlobalOperator> A;
  std::shared_ptr<TransformedSystem> sys;
  std::unique_ptr<TwoLevel> tl;
  std::shared_ptr<Discretization> coarse_disc;
  Vec rhs;
};
DCtx* D(void* h) { return static_cast<DCtx*>(h); }
}  // namespace

extern "C" {

double oracle_sipg_default_eta(int p, int d) { return sipg_default_eta(p, d); }

// Nodal facet matrices of reference_operators(p, kind): dirichlet (p+1)^2, interior (2p+2)^2, column-major;
// traces: values / normal derivatives (2 x (p+1), column-major).
int oracle_sipg_facet_matrices(int p, int kind, double mu0, double mu1, double eta, int side0, int side1,
                               double* dirichlet, double* interior, double* tvals, double* tders) {
  return guard([&] {
    const ReferenceInterval ref = reference_operators(p, static_cast<BasisKind>(kind));
    const Mat E = sipg_facet_dirichlet(ref, mu0, eta, side0);
    const Mat Ei = sipg_facet_interior(ref, mu0, mu1, eta, side0, side1);
    std::memcpy(dirichlet, E.a.data(), E.a.size() * 8);
    std::memcpy(interior, Ei.a.data(), Ei.a.size() * 8);
    std::memcpy(tvals, ref.trace_values.a.data(), ref.trace_values.a.size() * 8);
    std::memcpy(tders, ref.trace_normal_derivs.a.data(), ref.trace_normal_derivs.a.size() * 8);
  });
}

// dq_space on cartesian_mesh(dim, n^dim, unit), SIPG with eta (< 0: sipg_default_eta),
// all boundary facets Dirichlet; rhs = load_vector(f = 1).
void* oracle_dg_create(int dim, int n, int p, double eta, int skip_boundary, int threads) {
  DCtx* out = nullptr;
  guard([&] {
    auto c = std::make_unique<DCtx>();
    c->mesh = cartesian_mesh(dim, std::vector<int>(dim, n), std::vector<double>(dim, 1.0));
    c->disc = dq_space(c->mesh, p);
    c->disc.mesh = &c->mesh;
    c->bundle = make_bundle_dg(p);
    c->eta = eta < 0 ? sipg_default_eta(p, dim) : eta;
    c->cfg.skip_boundary_patches = skip_boundary != 0;
    c->cfg.threads = threads;
    c->A = std::make_shared<GlobalOperator>(dg_poisson_operator(c->disc, c->bundle, c->eta));
    c->sys = std::make_shared<TransformedSystem>(transformed_dg_poisson(c->disc, c->bundle, c->eta));
    c->rhs = load_vector(c->disc, c->bundle, [](const std::array<double, 3>&) { return 1.0; });
    out = c.release();
  });
  return out;
}

void oracle_dg_destroy(void* h) { delete D(h); }

// out: dim, p, ncells, ndof, dofs per cell
int oracle_dg_info(void* h, int64_t* out) {
  return guard([&] {
    const auto& d = D(h)->disc;
    int64_t v[5] = {d.dim(), d.degree, D(h)->mesh.num_cells(), d.ndof, d.dofs_per_cell};
    std::memcpy(out, v, sizeof(v));
  });
}

int oracle_dg_rhs(void* h, double* out) {
  return guard([&] { std::memcpy(out, D(h)->rhs.data(), D(h)->rhs.size() * 8); });
}

// which 0: true-form operator, 1: transformed matrix At; dense row-major, and the
// stored entries per row of At (explicit zeros count, as Eigen stores them).
int oracle_dg_dense(void* h, int which, double* out, int32_t* at_row_nnz, int32_t* label_cls) {
  return guard([&] {
    DCtx* c = D(h);
    const Csr M = which == 0 ? c->A->assemble() : c->sys->At;
    const int n = c->disc.ndof;
    std::memset(out, 0, size_t(n) * n * 8);
    for (int i = 0; i < n; ++i)
      for (int64_t q = M.ptr[i]; q < M.ptr[i + 1]; ++q) out[size_t(i) * n + M.col[q]] = M.val[q];
    for (int i = 0; i < n; ++i) {
      at_row_nnz[i] = int32_t(c->sys->At.ptr[i + 1] - c->sys->At.ptr[i]);
      label_cls[i] = int32_t(c->disc.labels[i].cls);
    }
  });
}

int oracle_dg_apply(void* h, int which, const double* in, double* out) {  // 0 A, 1 S^T, 2 S
  return guard([&] {
    DCtx* c = D(h);
    Vec x(in, in + c->disc.ndof), y;
    y = which == 0 ? c->A->apply(x) : which == 1 ? c->sys->apply_St(x) : c->sys->apply_S(x);
    std::memcpy(out, y.data(), y.size() * 8);
  });
}

// x = S At^{-1} S^T b with a natural-order Cholesky of At (tests/test_sipg.cpp:139-143).
int oracle_dg_fdm_solve(void* h, const double* b, double* x) {
  return guard([&] {
    DCtx* c = D(h);
    const CholFactor F = cholesky(c->sys->At, natural_ordering(c->disc.ndof));
    Vec bb(b, b + c->disc.ndof);
    const Vec y = c->sys->apply_S(F.solve(c->sys->apply_St(bb)));
    std::memcpy(x, y.data(), y.size() * 8);
  });
}

// Vertex-star patch of vertex v: its size and the nnz of its Cholesky factor under
// patch_ordering (tests/test_sipg.cpp:150-167); v < 0 picks the first interior vertex.
int oracle_dg_patch(void* h, int v, int64_t* out) {
  return guard([&] {
    DCtx* c = D(h);
    if (v < 0)
      for (int u = 0; u < c->mesh.num_vertices() && v < 0; ++u)
        if (int(c->mesh.vertex_cells[u].size()) == (1 << c->mesh.dim)) v = u;
    const std::vector<int> dofs = c->disc.star_dofs(v);
    std::vector<DofLabel> labels;
    for (int d : dofs) labels.push_back(c->disc.labels[d]);
    const CholFactor F = cholesky(extract_submatrix(c->sys->At, dofs), patch_ordering(labels));
    out[0] = int64_t(dofs.size());
    out[1] = F.nnz();
  });
}

// The DG two-level solver of tests/test_sipg.cpp:184-197: PatchSolver on At,
// Q1 continuous Poisson coarse level, build_prolongation from it, damping.
int oracle_dg_build(void* h, int calibrate) {
  return guard([&] {
    DCtx* c = D(h);
    auto tl = std::make_unique<TwoLevel>();
    auto A = c->A;
    tl->A = [A](const Vec& x) { return A->apply(x); };
    tl->sys = c->sys;
    tl->patches = build_patch_solver(c->disc, *c->sys, c->bundle, c->cfg);
    c->coarse_disc = std::make_shared<Discretization>(q_space(c->mesh, 1));
    const Bundle1D cb = make_bundle(1);
    const GlobalOperator cop = poisson_operator(*c->coarse_disc, cb);
    tl->coarse = std::make_shared<CholFactor>(cholesky(cop.assemble(), natural_ordering(c->coarse_disc->ndof)));
    Mat V, Dm;
    cb.ref.eval(c->bundle.ref.nodes, V, Dm);
    tl->prolong = build_prolongation(c->disc, *c->coarse_disc, V);
    if (calibrate) calibrate_damping(*tl, c->disc, c->cfg);
    c->tl = std::move(tl);
  });
}

// After oracle_dg_build: which 0 PatchSolver::apply (modal in, modal out),
// 1 TwoLevel::smooth, 2 TwoLevel::apply (V-cycle at the solver's omega).
int oracle_dg_op(void* h, int which, const double* in, double* out) {
  return guard([&] {
    DCtx* c = D(h);
    if (!c->tl) throw std::invalid_argument("oracle_dg_op: build first");
    Vec x(in, in + c->disc.ndof), y;
    y = which == 0 ? c->tl->patches.apply(x) : which == 1 ? c->tl->smooth(x) : c->tl->apply(x);
    std::memcpy(out, y.data(), y.size() * 8);
  });
}

int oracle_dg_set_omega(void* h, double w) {
  return guard([&] {
    if (!D(h)->tl) throw std::invalid_argument("oracle_dg_set_omega: build first");
    D(h)->tl->omega = w;
  });
}

// Patch lists of the built solver: npatch (count only when ptr is null), then
// vertex, ptr (npatch+1), dofs, factor nnz per patch.
int oracle_dg_patches(void* h, int64_t* count, int32_t* vertex, int64_t* ptr, int32_t* dofs, int64_t* nnz) {
  return guard([&] {
    DCtx* c = D(h);
    if (!c->tl) throw std::invalid_argument("oracle_dg_patches: build first");
    const auto& P = c->tl->patches.patches;
    count[0] = int64_t(P.size());
    int64_t tot = 0;
    for (const auto& q : P) tot += int64_t(q.dofs.size());
    count[1] = tot;
    if (!ptr) return;
    ptr[0] = 0;
    for (size_t j = 0; j < P.size(); ++j) {
      vertex[j] = P[j].vertex;
      ptr[j + 1] = ptr[j] + int64_t(P[j].dofs.size());
      std::memcpy(dofs + ptr[j], P[j].dofs.data(), P[j].dofs.size() * 4);
      nnz[j] = P[j].factor.nnz();
    }
  });
}

// report: iterations, converged, kappa, omega, npatches
int oracle_dg_pcg(void* h, const double* b, double* x, double rtol, int maxit, double* report) {
  return guard([&] {
    DCtx* c = D(h);
    Vec bb(b, b + c->disc.ndof);
    auto A = c->A;
    LinOp Aop = [A](const Vec& v) { return A->apply(v); };
    auto [xx, rep] = pcg(Aop, c->tl->applier(), bb, rtol, maxit);
    std::memcpy(x, xx.data(), xx.size() * 8);
    report[0] = rep.iterations;
    report[1] = rep.converged;
    report[2] = rep.kappa;
    report[3] = c->tl->omega;
    report[4] = double(c->tl->patches.patches.size());
  });
}

}  // extern "C"
