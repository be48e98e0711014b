// extern "C" surface of the host setup (the mirror of the reference's
// cartesian_mesh / q_space / make_bundle / build_patch_solver inputs) and
// fdmhost_attach, which feeds a problem into an fdmgpu handle through the
// public C ABI only (include/fdmgpu.h) — the same calls a reference-side
// integration makes.
#include <cstring>
#include <exception>
#include <string>

#include "../../../include/fdmhost.h"
#include "fdm_host.hpp"

using namespace fdmgpu::host;

namespace {
thread_local std::string g_err;
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
template <class T>
void put(T* dst, const std::vector<T>& v) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T));
}
}  // namespace

extern "C" {

const char* fdmhost_last_error() { return g_err.c_str(); }

void* fdmhost_problem_create(int config, int n, int p) {
  Problem* out = nullptr;
  if (guard([&] { out = make_problem(config, n, p).release(); })) return nullptr;
  return out;
}

// Linear elasticity (make_elastic_problem): the reference's Table-2 problem
// in dim = 2|3 with n cells per axis, vector Q_p, Lame mu / lambda.
void* fdmhost_elastic_create(int dim, int n, int p, double mu, double lambda, int skip_boundary_patches) {
  Problem* out = nullptr;
  if (guard([&] { out = make_elastic_problem(dim, n, p, mu, lambda, skip_boundary_patches != 0).release(); }))
    return nullptr;
  return out;
}

// Symmetric interior-penalty DG (make_dg_problem): dq_space on the unit
// square / cube with n cells per axis, weak Dirichlet, penalty eta.
void* fdmhost_dg_create(int dim, int n, int p, double eta, int skip_boundary_patches) {
  Problem* out = nullptr;
  if (guard([&] { out = make_dg_problem(dim, n, p, eta, skip_boundary_patches != 0).release(); })) return nullptr;
  return out;
}

// Problem on a mesh file in the reference's JSON format (load_mesh,
// src/mesh.cpp:375-434); Q_p space, unit coefficient, RHS U[-1,1] from seed.
void* fdmhost_problem_from_mesh_file(const char* path, int p, uint64_t seed) {
  Problem* out = nullptr;
  if (guard([&] { out = make_problem_from_mesh(load_mesh(path), p, seed).release(); })) return nullptr;
  return out;
}

// Same from arrays: vertices (nv x 3), cells (nc x 2^dim), facet tags
// (cell, local facet 2*axis + (side > 0), tag 0/1/2 = interior/dirichlet/neumann).
void* fdmhost_problem_from_mesh(int dim, int nv, const double* vertices, int nc, const int32_t* cells, int ntag,
                                const int32_t* tag_cell, const int32_t* tag_local_facet, const int32_t* tag_kind,
                                int p, uint64_t seed) {
  Problem* out = nullptr;
  if (guard([&] {
        if (dim < 2 || dim > 3 || nv < 1 || nc < 1 || !vertices || !cells)
          throw std::invalid_argument("problem_from_mesh: bad mesh arrays");
        Mesh m;
        m.dim = dim;
        for (int v = 0; v < nv; ++v) m.vertices.push_back({vertices[3 * v], vertices[3 * v + 1], vertices[3 * v + 2]});
        const int ncorner = 1 << dim;
        for (int c = 0; c < nc; ++c) {
          m.cells.emplace_back(cells + size_t(c) * ncorner, cells + size_t(c + 1) * ncorner);
          for (int v : m.cells.back())
            if (v < 0 || v >= nv) throw std::invalid_argument("problem_from_mesh: cell vertex out of range");
        }
        m.finalize();
        if (ntag > 0) {
          for (int k = 0; k < ntag; ++k)
            if (tag_kind[k] < 0 || tag_kind[k] > 2) throw std::invalid_argument("problem_from_mesh: bad facet tag");
          apply_facet_tags(m, std::vector<int>(tag_cell, tag_cell + ntag),
                           std::vector<int>(tag_local_facet, tag_local_facet + ntag),
                           std::vector<int>(tag_kind, tag_kind + ntag));
        }
        check_orientation(m);
        out = make_problem_from_mesh(std::move(m), p, seed).release();
      }))
    return nullptr;
  return out;
}

int fdmhost_save_mesh(void* ph, const char* path) {
  return guard([&] { save_mesh(static_cast<Problem*>(ph)->mesh, path); });
}

// SolverConfig::skip_boundary_patches (include/fdmstar/schwarz.hpp:24): the
// problems are built with true (the configs' setting); false adds the
// boundary-vertex stars as the reference default does (src/schwarz.cpp:71-81).
int fdmhost_problem_set_skip_boundary_patches(void* ph, int skip) {
  return guard([&] {
    Problem& P = *static_cast<Problem*>(ph);
    rebuild_patches(P, skip != 0);
  });
}

// write_matrix_market (src/sparse.cpp:33-52): CSC input, `symmetric` keeps row >= col.
int fdmhost_write_matrix_market(const char* path, int64_t rows, int64_t cols, const int64_t* colptr,
                                const int32_t* rowidx, const double* val, int symmetric) {
  return guard([&] {
    if (!path || rows < 0 || cols < 0 || !colptr || (colptr[cols] > 0 && (!rowidx || !val)))
      throw std::invalid_argument("write_matrix_market: bad arguments");
    write_matrix_market(path, rows, cols, colptr, rowidx, val, symmetric != 0);
  });
}

void fdmhost_problem_destroy(void* ph) { delete static_cast<Problem*>(ph); }

// out: dim, p, ncells, ndof, nfree, npatch, nvertices, npc, sum n_j, ncoarse,
//      P nnz, q, config, n (cells per axis), all_cartesian, ncomp
int fdmhost_problem_info(void* ph, int64_t* out) {
  return guard([&] {
    const Problem& P = *static_cast<Problem*>(ph);
    bool cart = true;
    for (auto k : P.cell_kind) cart = cart && k == 0;
    const int64_t v[16] = {P.dim, P.p, P.mesh.num_cells(), int64_t(P.ncomp) * P.space.ndof,
                           int64_t(P.ncomp) * P.space.num_free(),
                           int64_t(P.patches.vertex.size()), P.mesh.num_vertices(), P.space.npc,
                           P.patches.ptr.back(), P.coarse.ndof, int64_t(P.coarse.P_col.size()), P.basis.q,
                           P.config, P.n, cart ? 1 : 0, P.ncomp};
    std::memcpy(out, v, sizeof(v));
  });
}

int fdmhost_get_rhs(void* ph, double* out) {
  return guard([&] { put(out, static_cast<Problem*>(ph)->rhs); });
}

int fdmhost_get_maps(void* ph, int32_t* cell_dofs, int32_t* cell_modes, uint8_t* constrained, double* multiplicity,
                     int32_t* label_cls, int32_t* label_entity) {
  return guard([&] {
    const Problem& P = *static_cast<Problem*>(ph);
    const Space& s = P.space;
    put(cell_dofs, s.cell_dofs);  // component 0 for vector problems
    put(cell_modes, s.cell_modes);
    for (int ci = 0; ci < P.ncomp; ++ci) {  // per-DOF arrays over all components
      const size_t o = size_t(ci) * s.ndof;
      if (constrained) put(constrained + o, s.constrained);
      if (multiplicity) put(multiplicity + o, s.multiplicity);
      if (label_cls) put(label_cls + o, s.label_cls);
      if (label_entity) put(label_entity + o, s.label_entity);
    }
  });
}

int fdmhost_get_geometry(void* ph, double* vertices, double* kappa, double* mu, uint8_t* kind, double* corner_xyz) {
  return guard([&] {
    const Problem& P = *static_cast<Problem*>(ph);
    if (vertices)
      for (int v = 0; v < P.mesh.num_vertices(); ++v)
        for (int a = 0; a < 3; ++a) vertices[3 * v + a] = P.mesh.vertices[v][a];
    put(kappa, P.cell_kappa);
    put(mu, P.cell_mu);
    put(kind, P.cell_kind);
    put(corner_xyz, P.cell_xyz);
  });
}

int fdmhost_get_basis(void* ph, double* S, double* At, double* Bt, uint8_t* Anz, uint8_t* Bnz, double* lambda,
                      double* parity, double* Ahat, double* Bhat, double* nodes) {
  return guard([&] {
    const Basis1D& b = static_cast<Problem*>(ph)->basis;
    put(S, b.S.a);
    put(At, b.A_t.a);
    put(Bt, b.B_t.a);
    put(Anz, b.A_nz);
    put(Bnz, b.B_nz);
    put(lambda, b.lambda);
    put(parity, b.parity);
    put(Ahat, b.A_hat.a);
    put(Bhat, b.B_hat.a);
    put(nodes, b.nodes);
  });
}

int fdmhost_get_patches(void* ph, int32_t* vertex, int64_t* ptr, int32_t* dofs, int32_t* perm, int32_t* cells,
                        int32_t* colour) {
  return guard([&] {
    const Patches& P = static_cast<Problem*>(ph)->patches;
    put(vertex, P.vertex);
    put(ptr, P.ptr);
    put(dofs, P.dofs);
    put(perm, P.perm);
    put(cells, P.cells);
    put(colour, P.colour);
  });
}

int fdmhost_get_coarse(void* ph, double* inverse, int64_t* P_ptr, int32_t* P_col, double* P_val) {
  return guard([&] {
    const Coarse& C = static_cast<Problem*>(ph)->coarse;
    put(inverse, C.inverse);
    put(P_ptr, C.P_ptr);
    put(P_col, C.P_col);
    put(P_val, C.P_val);
  });
}

// Creates an fdmgpu handle for the problem and uploads every input through
// the public C ABI (does not factor).  Returns the fdmgpu status.
// sep_order: 0 plane-by-plane separator (default), 1 reference patch_ordering, -1 keep.
int fdmhost_attach(void* ph, int device, int sep_order, fdmgpu_handle* out) {
  Problem& P = *static_cast<Problem*>(ph);
  fdmgpu_handle h = nullptr;
  const int64_t ndof = int64_t(P.ncomp) * P.space.ndof;
  fdmgpu_status st = fdmgpu_create(&h, P.dim, P.p, P.mesh.num_cells(), ndof, device);
  if (st != FDMGPU_OK) {
    g_err = h ? fdmgpu_last_error(h) : "fdmgpu_create failed (no CUDA device?)";
    return st;
  }
  auto fail = [&](fdmgpu_status s) {
    g_err = fdmgpu_last_error(h);
    fdmgpu_destroy(h);
    return int(s);
  };
  if (sep_order >= 0 && (st = fdmgpu_set_separator_order(h, sep_order)) != FDMGPU_OK) return fail(st);
  if (P.ncomp > 1 && (st = fdmgpu_set_elasticity(h, P.lame_mu, P.lame_lambda, P.Cmat.data())) != FDMGPU_OK)
    return fail(st);
  const Basis1D& b = P.basis;
  if (P.dg) {  // SIPG: penalty, traces, facet list, cell corners (fdmgpu_set_sipg)
    const auto& F = P.mesh.facets;
    const int nf = int(F.size());
    std::vector<int32_t> fc(2 * size_t(nf)), fa(nf), fs(2 * size_t(nf)), cv;
    std::vector<uint8_t> ft(nf);
    for (int f = 0; f < nf; ++f) {
      for (int r = 0; r < 2; ++r) {
        fc[2 * f + r] = F[f].cell[r];
        fs[2 * f + r] = F[f].side[r];
      }
      fa[f] = F[f].axis[0];
      ft[f] = uint8_t(F[f].tag);
    }
    for (const auto& cell : P.mesh.cells) cv.insert(cv.end(), cell.begin(), cell.end());
    if ((st = fdmgpu_set_sipg(h, P.eta, b.dtr.a.data(), b.tv.a.data(), b.tnd.a.data(), nf, fc.data(), fa.data(),
                              fs.data(), ft.data(), cv.data())) != FDMGPU_OK)
      return fail(st);
  }
  if ((st = fdmgpu_set_basis(h, b.S.a.data(), b.lambda.data(), b.A_t.a.data(), b.B_t.a.data(), b.A_nz.data(),
                             b.B_nz.data(), b.A_hat.a.data(), b.B_hat.a.data(), b.q, b.qp.data(), b.wq.data(),
                             b.Vq.a.data(), b.Dq.a.data())) != FDMGPU_OK)
    return fail(st);
  const Space& s = P.space;
  std::vector<double> mult(s.multiplicity);
  std::vector<uint8_t> con(s.constrained);
  for (int ci = 1; ci < P.ncomp; ++ci) {  // vector_q_space: identical component blocks
    mult.insert(mult.end(), s.multiplicity.begin(), s.multiplicity.end());
    con.insert(con.end(), s.constrained.begin(), s.constrained.end());
  }
  if ((st = fdmgpu_set_mesh_maps(h, s.cell_dofs.data(), s.cell_modes.data(),
                                 s.mode_sign.empty() ? nullptr : s.mode_sign.data(), mult.data(), con.data())) !=
      FDMGPU_OK)
    return fail(st);
  if ((st = fdmgpu_set_cell_coeffs(h, P.cell_kind.data(), P.cell_mu.data(), P.cell_xyz.data(),
                                   P.ncomp > 1 ? nullptr : P.cell_kappa.data())) != FDMGPU_OK)
    return fail(st);
  const Patches& pt = P.patches;
  if ((st = fdmgpu_set_patches(h, int32_t(pt.vertex.size()), pt.vertex.data(), pt.ptr.data(), pt.dofs.data(),
                               pt.perm.data(), pt.cells.data())) != FDMGPU_OK)
    return fail(st);
  const Coarse& C = P.coarse;
  if ((st = fdmgpu_set_coarse(h, C.ndof, C.inverse.data(), C.P_ptr.data(), C.P_col.data(), C.P_val.data())) !=
      FDMGPU_OK)
    return fail(st);
  if ((st = fdmgpu_set_coarse_cells(h, C.cell_dofs.data(), C.constrained.data(), C.phat.data())) != FDMGPU_OK)
    return fail(st);
  *out = h;
  return FDMGPU_OK;
}

}  // extern "C"
