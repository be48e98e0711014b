/* fdmhost.h -- C ABI of the host setup mirror (csrc/host/), built into the same
 * libfdmgpu.so.  It restates, in C++, the reference's setup for the hot path --
 * meshes and mesh files (src/mesh.cpp), Q_p maps and star_dofs
 * (src/discretization.cpp), patch_ordering (src/ordering.cpp), the FDM basis
 * (src/fdm_basis.cpp) and the Q1 coarse level (src/schwarz.cpp:139-165,
 * 239-243) -- and hands the arrays to fdmgpu.h (fdmhost_attach).  A reference
 * integration keeps its own setup and calls fdmgpu.h directly;
 * this mirror serves the tests, the bench and Python users.
 *
 * Problem handles are opaque.  Functions returning int return 0 on success and
 * 1 on failure with the message in fdmhost_last_error() (the reference's
 * exception text where one exists). */
#ifndef FDMHOST_H
#define FDMHOST_H

#include <stdint.h>

#include "fdmgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* fdmhost_last_error(void);

/* One of the BASELINE.json configurations 1..5, optionally reduced to n cells
 * per axis / degree p (0 = the config's value). */
void* fdmhost_problem_create(int config, int n, int p);
/* Linear elasticity (src/elasticity.cpp): the reference's Table-2 problem
 * (tests/test_elasticity.cpp:24-30, 162-185) in dim = 2|3 -- unit square /
 * cube, n cells per axis, x = 0 Dirichlet, other boundary facets Neumann --
 * with vector Q_p, Lame mu / lambda, body force -0.02 e_{dim-1}, the SDC
 * relaxation and a vector Q1 coarse level.  skip_boundary_patches: the
 * reference default is 0. */
void* fdmhost_elastic_create(int dim, int n, int p, double mu, double lambda, int skip_boundary_patches);
/* Symmetric interior-penalty DG (src/sipg.cpp): dq_space(cartesian_mesh(dim,
 * n^dim, unit), p), every boundary facet weak Dirichlet, penalty eta (< 0:
 * sipg_default_eta), RHS load_vector(f = 1), DG vertex stars
 * (skip_boundary_patches: the reference default is 0), Q1 coarse level. */
void* fdmhost_dg_create(int dim, int n, int p, double eta, int skip_boundary_patches);
/* Q_p problem on a mesh file in the reference's JSON format (load_mesh,
 * src/mesh.cpp:375-434), RHS U[-1,1] from std::mt19937_64(seed). */
void* fdmhost_problem_from_mesh_file(const char* path, int p, uint64_t seed);
/* Same from arrays: vertices nv x 3, cells nc x 2^dim (tensor corner order),
 * facet tags (cell, local facet 2*axis + (side > 0), 0/1/2 =
 * interior/dirichlet/neumann). */
void* fdmhost_problem_from_mesh(int dim, int nv, const double* vertices, int nc, const int32_t* cells, int ntag,
                                const int32_t* tag_cell, const int32_t* tag_local_facet, const int32_t* tag_kind,
                                int p, uint64_t seed);
/* save_mesh (src/mesh.cpp:354-373). */
int fdmhost_save_mesh(void* problem, const char* path);
/* SolverConfig::skip_boundary_patches (include/fdmstar/schwarz.hpp:24):
 * problems start with 1 (the configs); 0 adds the boundary-vertex stars. */
int fdmhost_problem_set_skip_boundary_patches(void* problem, int skip);
/* write_matrix_market (src/sparse.cpp:33-52) for a CSC matrix (colptr has
 * cols + 1 entries, row indices ascending per column); symmetric != 0 writes
 * the lower triangle under a "symmetric" header. */
int fdmhost_write_matrix_market(const char* path, int64_t rows, int64_t cols, const int64_t* colptr,
                                const int32_t* rowidx, const double* val, int symmetric);
void fdmhost_problem_destroy(void* problem);

/* out[16]: dim, p, ncells, ndof, nfree, npatch, nvertices, dofs per cell,
 * sum n_j, coarse ndof, P nnz, quadrature points, config, n, all Cartesian,
 * components (1 scalar, dim elasticity; ndof / nfree / sum n_j / coarse ndof
 * count all components, cell maps are component 0's). */
int fdmhost_problem_info(void* problem, int64_t* out);
int fdmhost_get_rhs(void* problem, double* out);
int fdmhost_get_maps(void* problem, int32_t* cell_dofs, int32_t* cell_modes, uint8_t* constrained,
                     double* multiplicity, int32_t* label_cls, int32_t* label_entity);
int fdmhost_get_geometry(void* problem, double* vertices, double* kappa, double* mu, uint8_t* kind,
                         double* corner_xyz);
int fdmhost_get_basis(void* problem, double* S, double* At, double* Bt, uint8_t* Anz, uint8_t* Bnz, double* lambda,
                      double* parity, double* Ahat, double* Bhat, double* nodes);
int fdmhost_get_patches(void* problem, int32_t* vertex, int64_t* ptr, int32_t* dofs, int32_t* perm, int32_t* cells,
                        int32_t* colour);
int fdmhost_get_coarse(void* problem, double* inverse, int64_t* P_ptr, int32_t* P_col, double* P_val);
/* Creates an fdmgpu handle on `device` and uploads the problem through the
 * fdmgpu.h setters (sep_order: 0 plane-by-plane separator order, 1 the
 * reference's patch_ordering). */
int fdmhost_attach(void* problem, int device, int sep_order, fdmgpu_handle* out);

#ifdef __cplusplus
}
#endif

#endif /* FDMHOST_H */
