// TEST INFRASTRUCTURE ONLY — extern "C" surface of the oracle for the Python
// tests (ctypes) and bench.py's cpu_baseline / --impl reference legs.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

struct Ctx {
  std::unique_ptr<Problem> pb;
  std::shared_ptr<GlobalOperator> A;
  std::shared_ptr<TransformedSystem> sys;
  PatchList pl;
  PatchSolver ps;
  SolverConfig cfg;
  std::unique_ptr<TwoLevel> tl;
};

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

// build_global: 1 = assemble the global transformed matrix as the reference
// does (src/assembly.cpp:245-291); 0 = patch matrices from star cells only.
void* oracle_create(int config, int n, int p, int build_global, int threads) {
  Ctx* c = nullptr;
  int rc = guard([&] {
    auto ctx = std::make_unique<Ctx>();
    ctx->pb = make_problem(config, n, p);
    ctx->cfg.skip_boundary_patches = true;
    ctx->cfg.threads = threads;
    ctx->A = std::make_shared<GlobalOperator>(poisson_operator(ctx->pb->disc, ctx->pb->bundle));
    ctx->sys = std::make_shared<TransformedSystem>(transformed_poisson(ctx->pb->disc, ctx->pb->bundle, true, build_global != 0));
    ctx->pl = patch_list(ctx->pb->disc, ctx->cfg);
    ctx->ps.ndof = ctx->pb->disc.ndof;
    ctx->ps.threads = threads;
    ctx->ps.patches.resize(ctx->pl.vertex.size());
    for (size_t j = 0; j < ctx->pl.vertex.size(); ++j) {
      ctx->ps.patches[j].vertex = ctx->pl.vertex[j];
      ctx->ps.patches[j].dofs = ctx->pl.dofs[j];
    }
    c = ctx.release();
  });
  return rc ? nullptr : c;
}

// [ext] external mesh: vertices (nv x 3), cells (nc x 2^dim), facet tags
// (cell, local facet 2*axis + (side > 0), 0/1/2 = interior/dirichlet/neumann).
void* oracle_create_mesh(int dim, int nv, const double* vertices, int nc, const int* cells, int ntag,
                         const int* tag_cell, const int* tag_lf, const int* tag_kind, int p, uint64_t seed,
                         int build_global, int threads) {
  Ctx* c = nullptr;
  int rc = guard([&] {
    Mesh m;
    m.dim = dim;
    for (int v = 0; v < nv; ++v) m.vertices.push_back({vertices[3 * v], vertices[3 * v + 1], vertices[3 * v + 2]});
    const int ncorner = 1 << dim;
    for (int k = 0; k < nc; ++k) m.cells.emplace_back(cells + size_t(k) * ncorner, cells + size_t(k + 1) * ncorner);
    m.finalize();
    for (int k = 0; k < ntag; ++k) {  // src/mesh.cpp:399-407
      const int lf = tag_lf[k], axis = lf / 2, side = (lf % 2) ? 1 : -1;
      int fi = -1;
      for (int f = 0; f < int(m.facets.size()) && fi < 0; ++f)
        for (int r = 0; r < m.facets[f].ncells(); ++r)
          if (m.facets[f].cell[r] == tag_cell[k] && m.facets[f].axis[r] == axis && m.facets[f].side[r] == side) fi = f;
      if (fi < 0) throw std::runtime_error("load_mesh: facet_tags entry names a missing facet");
      m.facets[fi].tag = static_cast<FacetTag>(tag_kind[k]);
    }
    auto ctx = std::make_unique<Ctx>();
    ctx->pb = make_problem_from_mesh(std::move(m), p, seed);
    ctx->cfg.skip_boundary_patches = true;
    ctx->cfg.threads = threads;
    ctx->A = std::make_shared<GlobalOperator>(poisson_operator(ctx->pb->disc, ctx->pb->bundle));
    ctx->sys = std::make_shared<TransformedSystem>(transformed_poisson(ctx->pb->disc, ctx->pb->bundle, true, build_global != 0));
    ctx->pl = patch_list(ctx->pb->disc, ctx->cfg);
    ctx->ps.ndof = ctx->pb->disc.ndof;
    ctx->ps.threads = threads;
    ctx->ps.patches.resize(ctx->pl.vertex.size());
    for (size_t j = 0; j < ctx->pl.vertex.size(); ++j) {
      ctx->ps.patches[j].vertex = ctx->pl.vertex[j];
      ctx->ps.patches[j].dofs = ctx->pl.dofs[j];
    }
    c = ctx.release();
  });
  return rc ? nullptr : c;
}

// [ext] SolverConfig::skip_boundary_patches (include/fdmstar/schwarz.hpp:24);
// the handles start with true (the configs); false = the reference default.
int oracle_set_skip_boundary_patches(void* h, int skip) {
  return guard([&] {
    Ctx* ctx = static_cast<Ctx*>(h);
    ctx->cfg.skip_boundary_patches = skip != 0;
    ctx->pl = patch_list(ctx->pb->disc, ctx->cfg);
    ctx->ps = PatchSolver();
    ctx->tl.reset();
    ctx->ps.ndof = ctx->pb->disc.ndof;
    ctx->ps.threads = ctx->cfg.threads;
    ctx->ps.patches.resize(ctx->pl.vertex.size());
    for (size_t j = 0; j < ctx->pl.vertex.size(); ++j) {
      ctx->ps.patches[j].vertex = ctx->pl.vertex[j];
      ctx->ps.patches[j].dofs = ctx->pl.dofs[j];
    }
  });
}

void oracle_destroy(void* h) { delete static_cast<Ctx*>(h); }

// out[0..9] = dim, p, ncells, ndof, nfree, npatches, nvertices, dofs_per_cell, sum n_j, config
int oracle_info(void* h, int64_t* out) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    const auto& d = c->pb->disc;
    int64_t s = 0;
    for (const auto& v : c->pl.dofs) s += int64_t(v.size());
    int64_t vals[10] = {d.dim(), d.degree, c->pb->mesh.num_cells(), d.ndof, d.num_free(), int64_t(c->pl.vertex.size()),
                        c->pb->mesh.num_vertices(), d.dofs_per_cell, s, c->pb->config};
    std::memcpy(out, vals, sizeof(vals));
  });
}

int oracle_get_rhs(void* h, double* out) {
  return guard([&] {
    const auto& r = static_cast<Ctx*>(h)->pb->rhs;
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int oracle_get_maps(void* h, int32_t* cell_dofs, int32_t* cell_modes, uint8_t* constrained, double* multiplicity,
                    int32_t* label_cls, int32_t* label_entity) {
  return guard([&] {
    const auto& d = static_cast<Ctx*>(h)->pb->disc;
    for (size_t c = 0; c < d.cell_dofs.size(); ++c)
      for (int l = 0; l < d.dofs_per_cell; ++l) {
        cell_dofs[c * d.dofs_per_cell + l] = d.cell_dofs[c][l];
        cell_modes[c * d.dofs_per_cell + l] = d.cell_modes[c][l];
      }
    for (int i = 0; i < d.ndof; ++i) {
      constrained[i] = uint8_t(d.constrained[i]);
      multiplicity[i] = d.multiplicity[i];
      label_cls[i] = int32_t(d.labels[i].cls);
      label_entity[i] = d.labels[i].entity;
    }
  });
}

// vertices: nvertices*3; cell_coeff: ncells (kappa); cell_mu: ncells*dim
int oracle_get_geometry(void* h, double* vertices, double* cell_coeff, double* cell_mu) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    const auto& m = c->pb->mesh;
    for (int v = 0; v < m.num_vertices(); ++v)
      for (int a = 0; a < 3; ++a) vertices[3 * v + a] = m.vertices[v][a];
    for (int k = 0; k < m.num_cells(); ++k) {
      cell_coeff[k] = m.kappa(k);
      for (int a = 0; a < m.dim; ++a) cell_mu[k * m.dim + a] = c->sys->cell_mu[k][a];
    }
  });
}

// S, A_t, B_t: (p+1)^2 column-major; nz masks likewise; lambda: p-1; parity: p+1
int oracle_get_basis(void* h, double* S, double* At, double* Bt, uint8_t* Atnz, uint8_t* Btnz, double* lambda,
                     double* parity) {
  return guard([&] {
    const auto& f = static_cast<Ctx*>(h)->pb->bundle.fdm;
    const size_t n = f.S.a.size();
    std::memcpy(S, f.S.a.data(), n * 8);
    std::memcpy(At, f.A_t.val.a.data(), n * 8);
    std::memcpy(Bt, f.B_t.val.a.data(), n * 8);
    for (size_t k = 0; k < n; ++k) {
      Atnz[k] = uint8_t(f.A_t.nz[k]);
      Btnz[k] = uint8_t(f.B_t.nz[k]);
    }
    std::memcpy(lambda, f.lambda.data(), f.lambda.size() * 8);
    std::memcpy(parity, f.parity.data(), f.parity.size() * 8);
  });
}

// Patch lists: vertex[np], ptr[np+1], dofs[sum] (ascending star_dofs),
// perm[sum] (patch_ordering, local indices), ngroups[np], groups (concat offsets)
int oracle_get_patches(void* h, int32_t* vertex, int64_t* ptr, int32_t* dofs, int32_t* perm) {
  return guard([&] {
    const auto& pl = static_cast<Ctx*>(h)->pl;
    ptr[0] = 0;
    for (size_t j = 0; j < pl.vertex.size(); ++j) {
      vertex[j] = pl.vertex[j];
      const int64_t o = ptr[j];
      for (size_t k = 0; k < pl.dofs[j].size(); ++k) {
        dofs[o + k] = pl.dofs[j][k];
        perm[o + k] = pl.ord[j].perm[k];
      }
      ptr[j + 1] = o + int64_t(pl.dofs[j].size());
    }
  });
}

int oracle_patch_group_offsets(void* h, int j, int32_t* out, int* count) {
  return guard([&] {
    const auto& g = static_cast<Ctx*>(h)->pl.ord.at(j).group_offsets;
    *count = int(g.size());
    if (out) std::memcpy(out, g.data(), g.size() * 4);
  });
}

int oracle_apply_St(void* h, const double* in, double* out) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Vec x(in, in + c->pb->disc.ndof);
    Vec y = c->sys->apply_St(x);
    std::memcpy(out, y.data(), y.size() * 8);
  });
}

int oracle_apply_S(void* h, const double* in, double* out) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Vec x(in, in + c->pb->disc.ndof);
    Vec y = c->sys->apply_S(x);
    std::memcpy(out, y.data(), y.size() * 8);
  });
}

int oracle_apply_A(void* h, const double* in, double* out) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Vec x(in, in + c->pb->disc.ndof);
    Vec y = c->A->apply(x);
    std::memcpy(out, y.data(), y.size() * 8);
  });
}

// Factor patches idx[0..n) (all when idx == nullptr) with `threads` workers.
int oracle_factor_patches(void* h, const int32_t* idx, int n, int threads) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    std::vector<int> todo;
    if (idx)
      todo.assign(idx, idx + n);
    else
      for (size_t j = 0; j < c->pl.vertex.size(); ++j) todo.push_back(int(j));
    parallel_for(int(todo.size()), threads, [&](int t) {
      const int j = todo[t];
      const Csr Aj = c->sys->At.n > 0 ? extract_submatrix(c->sys->At, c->pl.dofs[j])
                                      : patch_matrix(*c->sys, c->pb->bundle, c->pl.vertex[j], c->pl.dofs[j]);
      c->ps.patches[j].factor = cholesky(Aj, c->pl.ord[j]);
    });
  });
}

// Timing harness only (bench.py cpu legs): patch dst gets a copy of patch
// src's factor.  All interior stars share one structure and size, so a solve
// with the copy streams the same bytes as a solve with dst's own factor would
// (the values are src's); used where factoring every timed patch is too slow
// (C5: 143 s per patch).
int oracle_copy_factor(void* h, int src, int dst) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    auto& P = c->ps.patches;
    if (P.at(src).factor.n != int(P.at(dst).dofs.size()))
      throw std::invalid_argument("copy_factor: patch sizes differ or source not factored");
    P.at(dst).factor = P.at(src).factor;
  });
}

// out: nnz(L_j), flops (reference counter), n_j
int oracle_patch_factor_info(void* h, int j, int64_t* out) {
  return guard([&] {
    const auto& F = static_cast<Ctx*>(h)->ps.patches.at(j).factor;
    out[0] = F.nnz();
    out[1] = F.flops;
    out[2] = F.n;
  });
}

// CSC factor of patch j (colptr n+1, rowind nnz, values nnz)
int oracle_patch_factor_get(void* h, int j, int64_t* colptr, int32_t* rowind, double* values) {
  return guard([&] {
    const auto& F = static_cast<Ctx*>(h)->ps.patches.at(j).factor;
    std::memcpy(colptr, F.colptr.data(), F.colptr.size() * 8);
    std::memcpy(rowind, F.rowind.data(), F.rowind.size() * 4);
    std::memcpy(values, F.values.data(), F.values.size() * 8);
  });
}

// Patch matrix (CSR) of patch j: ptr n+1, col nnz, val nnz; returns sizes if buffers null.
int oracle_patch_matrix(void* h, int j, int64_t* nnz_out, int64_t* ptr, int32_t* col, double* val) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    const Csr A = c->sys->At.n > 0 ? extract_submatrix(c->sys->At, c->pl.dofs.at(j))
                                   : patch_matrix(*c->sys, c->pb->bundle, c->pl.vertex.at(j), c->pl.dofs.at(j));
    *nnz_out = A.nnz();
    if (ptr) {
      std::memcpy(ptr, A.ptr.data(), A.ptr.size() * 8);
      std::memcpy(col, A.col.data(), A.col.size() * 4);
      std::memcpy(val, A.val.data(), A.val.size() * 8);
    }
  });
}

int oracle_patch_solve_one(void* h, int j, const double* rj, double* xj) {
  return guard([&] {
    const auto& F = static_cast<Ctx*>(h)->ps.patches.at(j).factor;
    Vec b(rj, rj + F.n);
    Vec x = F.solve(b);
    std::memcpy(xj, x.data(), x.size() * 8);
  });
}

int oracle_patch_apply(void* h, const double* r, double* z) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Vec x(r, r + c->pb->disc.ndof);
    Vec y = c->ps.apply(x);
    std::memcpy(z, y.data(), y.size() * 8);
  });
}

int oracle_smooth(void* h, const double* r, double* z) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Vec x(r, r + c->pb->disc.ndof);
    Vec y = c->sys->apply_S(c->ps.apply(c->sys->apply_St(x)));
    std::memcpy(z, y.data(), y.size() * 8);
  });
}

// Builds the two-level tree around the already factored patches
// (src/schwarz.cpp:230-252); calibrate=1 runs calibrate_damping.
int oracle_build_twolevel(void* h, int calibrate) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    auto tl = std::make_unique<TwoLevel>();
    auto A = c->A;
    tl->A = [A](const Vec& x) { return A->apply(x); };
    tl->sys = c->sys;
    tl->patches = c->ps;
    static thread_local int dummy;
    (void)dummy;
    auto coarse_disc = std::make_shared<Discretization>(q_space(c->pb->mesh, c->cfg.coarse_degree));
    auto coarse_bundle = std::make_shared<Bundle1D>(make_bundle(c->cfg.coarse_degree));
    GlobalOperator cop = poisson_operator(*coarse_disc, *coarse_bundle);
    tl->coarse = std::make_shared<CholFactor>(cholesky(cop.assemble(), natural_ordering(coarse_disc->ndof)));
    Mat V, D;
    coarse_bundle->ref.eval(c->pb->bundle.ref.nodes, V, D);
    tl->prolong = build_prolongation(c->pb->disc, *coarse_disc, V);
    if (calibrate) calibrate_damping(*tl, c->pb->disc, c->cfg);
    c->tl = std::move(tl);
  });
}

// out: omega, lambda_min, lambda_max, coarse ndof, prolong nnz
int oracle_twolevel_info(void* h, double* out) {
  return guard([&] {
    const auto& tl = *static_cast<Ctx*>(h)->tl;
    out[0] = tl.omega;
    out[1] = tl.lambda_min;
    out[2] = tl.lambda_max;
    out[3] = tl.coarse->n;
    out[4] = double(tl.prolong.nnz());
  });
}

int oracle_set_omega(void* h, double omega) {
  return guard([&] { static_cast<Ctx*>(h)->tl->omega = omega; });
}

// Prolongation CSR (fine x coarse): ptr ndof+1, col, val; sizes when null.
int oracle_prolongation(void* h, int64_t* nnz_out, int64_t* ptr, int32_t* col, double* val) {
  return guard([&] {
    const auto& P = static_cast<Ctx*>(h)->tl->prolong;
    *nnz_out = P.nnz();
    if (ptr) {
      std::memcpy(ptr, P.ptr.data(), P.ptr.size() * 8);
      std::memcpy(col, P.col.data(), P.col.size() * 4);
      std::memcpy(val, P.val.data(), P.val.size() * 8);
    }
  });
}

int oracle_vcycle(void* h, const double* r, double* z) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Vec x(r, r + c->pb->disc.ndof);
    Vec y = c->tl->apply(x);
    std::memcpy(z, y.data(), y.size() * 8);
  });
}

// report: iterations, converged, kappa, lambda_min, lambda_max, wall_time;
// residuals: maxit entries (relative residual history).
int oracle_pcg(void* h, const double* b, double* x, double rtol, int maxit, double* report, double* residuals,
               int precond) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Vec bb(b, b + c->pb->disc.ndof);
    auto A = c->A;
    LinOp Aop = [A](const Vec& v) { return A->apply(v); };
    LinOp P;
    if (precond == 0)
      P = [](const Vec& v) { return v; };
    else if (precond == 1)
      P = [c](const Vec& v) { return c->sys->apply_S(c->ps.apply(c->sys->apply_St(v))); };
    else
      P = c->tl->applier();
    auto [xx, rep] = pcg(Aop, P, bb, rtol, maxit);
    std::memcpy(x, xx.data(), xx.size() * 8);
    report[0] = rep.iterations;
    report[1] = rep.converged;
    report[2] = rep.kappa;
    report[3] = rep.lambda_min;
    report[4] = rep.lambda_max;
    report[5] = rep.wall_time;
    for (size_t k = 0; k < rep.residuals.size(); ++k) residuals[k] = rep.residuals[k];
  });
}

// Load vector of f = 1 with homogeneous Dirichlet rows zeroed (src/assembly.cpp:344-373).
int oracle_load_vector_one(void* h, double* out) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Vec f = load_vector(c->pb->disc, c->pb->bundle, [](const std::array<double, 3>&) { return 1.0; });
    c->pb->disc.project_free(f);
    std::memcpy(out, f.data(), f.size() * 8);
  });
}

// Dense true-form cell matrix (src/assembly.cpp:198-215) of cell `cell`.
int oracle_cell_matrix_quadrature(void* h, int cell, double* out) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    Mat A = cell_matrix_quadrature(c->pb->mesh, cell, c->pb->bundle.ref);
    std::memcpy(out, A.a.data(), A.a.size() * 8);
  });
}

// Sum-factorised apply of cell `cell`'s true-form operator ([ext]).
int oracle_cell_sumfact_apply(void* h, int cell, const double* u, double* y) {
  return guard([&] {
    Ctx* c = static_cast<Ctx*>(h);
    const int d = c->pb->mesh.dim, p = c->pb->p;
    const QuadratureRule rule = gauss_legendre_rule(p + 2);
    CellGeometry geom = cell_geometry(c->pb->mesh, cell, rule);
    Vec G(geom.dets.size() * d * d);
    const double kap = c->pb->mesh.kappa(cell);
    for (size_t k = 0; k < geom.dets.size(); ++k)
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) G[k * d * d + a * d + b] = kap * geom.quad_weights[k] * geom.metric[k](a, b);
    const int npc = c->pb->disc.dofs_per_cell;
    Vec uu(u, u + npc);
    Vec yy = sumfact_cell_apply(c->pb->bundle, d, G, uu);
    std::memcpy(y, yy.data(), yy.size() * 8);
  });
}

// ---- stateless pins of the 1D / LA layer (reference tests) ----------------------
int oracle_gll_nodes(int p, double* out) {
  return guard([&] {
    Vec x = gll_nodes(p);
    std::memcpy(out, x.data(), x.size() * 8);
  });
}

int oracle_gauss_legendre(int n, double* pts, double* wts) {
  return guard([&] {
    QuadratureRule r = gauss_legendre_rule(n);
    std::memcpy(pts, r.points.data(), n * 8);
    std::memcpy(wts, r.weights.data(), n * 8);
  });
}

int oracle_legendre(int k, double x, double* out) {
  return guard([&] {
    auto [v, d] = legendre_value_deriv(k, x);
    out[0] = v;
    out[1] = d;
  });
}

// kind: 0 GLL nodal, 1 Lobatto hierarchical, 2 GL nodal. Outputs (p+1)^2 col-major.
int oracle_reference_operators(int p, int kind, double* stiffness, double* mass, double* nodes, double* trace_values) {
  return guard([&] {
    ReferenceInterval r = reference_operators(p, BasisKind(kind));
    std::memcpy(stiffness, r.stiffness.a.data(), r.stiffness.a.size() * 8);
    std::memcpy(mass, r.mass.a.data(), r.mass.a.size() * 8);
    std::memcpy(nodes, r.nodes.data(), r.nodes.size() * 8);
    std::memcpy(trace_values, r.trace_values.a.data(), r.trace_values.a.size() * 8);
  });
}

int oracle_fdm_basis(int p, int kind, double* S, double* lambda, double* At, double* Bt, uint8_t* Atnz,
                     uint8_t* Btnz, double* parity) {
  return guard([&] {
    FdmBasis f = fdm_basis(reference_operators(p, BasisKind(kind)));
    const size_t n = f.S.a.size();
    std::memcpy(S, f.S.a.data(), n * 8);
    std::memcpy(At, f.A_t.val.a.data(), n * 8);
    std::memcpy(Bt, f.B_t.val.a.data(), n * 8);
    for (size_t k = 0; k < n; ++k) {
      Atnz[k] = uint8_t(f.A_t.nz[k]);
      Btnz[k] = uint8_t(f.B_t.nz[k]);
    }
    std::memcpy(lambda, f.lambda.data(), f.lambda.size() * 8);
    std::memcpy(parity, f.parity.data(), f.parity.size() * 8);
  });
}

int oracle_dense_sym_gen_eig(int n, const double* A, const double* B, double* lambda, double* V) {
  return guard([&] {
    Mat a(n, n), b(n, n);
    std::memcpy(a.a.data(), A, size_t(n) * n * 8);
    std::memcpy(b.a.data(), B, size_t(n) * n * 8);
    auto [l, v] = dense_sym_gen_eig(a, b);
    std::memcpy(lambda, l.data(), n * 8);
    std::memcpy(V, v.a.data(), size_t(n) * n * 8);
  });
}

// Sparse Cholesky of a dense-given SPD matrix (zeros dropped, as the reference
// tests' to_sparse) under ordering `perm`; L returned dense (column-major).
int oracle_cholesky_dense(int n, const double* A, const int32_t* perm, double* L, int64_t* info, const double* b,
                          double* x) {
  return guard([&] {
    std::vector<Triplet> t;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        if (A[i + size_t(n) * j] != 0.0) t.push_back({i, j, A[i + size_t(n) * j]});
    Csr S = csr_from_triplets(n, n, t);
    Ordering ord;
    ord.perm.assign(perm, perm + n);
    ord.group_offsets = {0, n};
    CholFactor F = cholesky(S, ord);
    if (L) {
      std::fill(L, L + size_t(n) * n, 0.0);
      for (int j = 0; j < n; ++j)
        for (int64_t q = F.colptr[j]; q < F.colptr[j + 1]; ++q) L[F.rowind[q] + size_t(n) * j] = F.values[q];
    }
    info[0] = F.nnz();
    info[1] = F.flops;
    if (b && x) {
      Vec bb(b, b + n);
      Vec xx = F.solve(bb);
      std::memcpy(x, xx.data(), n * 8);
    }
  });
}

int oracle_patch_ordering(int n, const int32_t* cls, const int32_t* ent, int32_t* perm, int32_t* offsets,
                          int* noffsets) {
  return guard([&] {
    std::vector<DofLabel> labels(n);
    for (int i = 0; i < n; ++i) labels[i] = {DofClass(cls[i]), ent[i]};
    Ordering o = patch_ordering(labels);
    std::memcpy(perm, o.perm.data(), n * 4);
    *noffsets = int(o.group_offsets.size());
    std::memcpy(offsets, o.group_offsets.data(), o.group_offsets.size() * 4);
  });
}

int oracle_tridiag_extremes(int n, const double* diag, const double* off, double* out) {
  return guard([&] {
    std::vector<double> d(diag, diag + n), o(off, off + (n > 0 ? n - 1 : 0));
    auto [lo, hi] = tridiag_extremes(d, o);
    out[0] = lo;
    out[1] = hi;
  });
}

// PCG on a dense SPD matrix with a dense (or identity when P == nullptr)
// preconditioner matrix; report as oracle_pcg.
int oracle_pcg_dense(int n, const double* A, const double* P, const double* b, double rtol, int maxit, double* x,
                     double* report) {
  return guard([&] {
    auto mv = [n](const double* M) {
      return [n, M](const Vec& v) {
        Vec y(n, 0.0);
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) y[i] += M[i + size_t(n) * j] * v[j];
        return y;
      };
    };
    LinOp Aop = mv(A);
    LinOp Pop = P ? LinOp(mv(P)) : LinOp([](const Vec& v) { return v; });
    Vec bb(b, b + n);
    auto [xx, rep] = pcg(Aop, Pop, bb, rtol, maxit);
    std::memcpy(x, xx.data(), n * 8);
    report[0] = rep.iterations;
    report[1] = rep.converged;
    report[2] = rep.kappa;
    report[3] = rep.lambda_min;
    report[4] = rep.lambda_max;
    report[5] = rep.wall_time;
  });
}

// estimate_damping on dense operators (src/schwarz.cpp:97-119); out omega,lmin,lmax
int oracle_estimate_damping_dense(int n, const double* A, const double* P, double* out) {
  return guard([&] {
    auto mv = [n](const double* M) {
      return [n, M](const Vec& v) {
        Vec y(n, 0.0);
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) y[i] += M[i + size_t(n) * j] * v[j];
        return y;
      };
    };
    SolverConfig cfg;
    DampingEstimate e = estimate_damping(mv(P), mv(A), n, cfg, nullptr);
    out[0] = e.omega;
    out[1] = e.lambda_min;
    out[2] = e.lambda_max;
  });
}

}  // extern "C"
