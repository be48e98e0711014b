/*
 * fdmgpu.h — C ABI of the B200 (sm_100a, FP64) vertex-star FDM Schwarz path.
 *
 * Drop-in boundary for the reference's Poisson/PCG hot path
 * (/root/reference/proj).  Every entry point names the reference interface it
 * replaces; the reference-side binding a maintainer would add is shown in
 * INTEGRATION.md.  Conventions:
 *   - plain pointers and sizes only; no torch / Eigen types;
 *   - every call returns fdmgpu_status; fdmgpu_last_error(h) gives the message
 *     (same text as the reference's exception where one exists);
 *   - one CUDA stream per handle (fdmgpu_set_stream to share a caller's
 *     stream); calls on one handle are not thread-safe, distinct handles are;
 *   - vectors are global DOF vectors of length ndof in the reference's
 *     first-touch numbering (src/discretization.cpp:70-264); "device" calls
 *     take device pointers, "_host" calls take host pointers and copy.
 *   - there is no CPU fallback: without a CUDA device every call that needs
 *     one fails with FDMGPU_CUDA_ERROR.
 */
#ifndef FDMGPU_H
#define FDMGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fdmgpu_context* fdmgpu_handle;

typedef enum {
  FDMGPU_OK = 0,
  FDMGPU_INVALID_ARGUMENT = 1, /* std::invalid_argument (e.g. src/kron.cpp:23-25)            */
  FDMGPU_NOT_SPD = 2,          /* "cholesky: matrix not SPD at pivot k" (src/cholesky.cpp:80) */
  FDMGPU_INDEFINITE = 3,       /* "pcg: indefinite operator at iteration k" (src/krylov.cpp:50) */
  FDMGPU_OUT_OF_MEMORY = 4,
  FDMGPU_CUDA_ERROR = 5,
  FDMGPU_UNSUPPORTED = 6 /* patch topology outside the shared-lattice pattern, 2D facet flips */
} fdmgpu_status;

/* KrylovReport (include/fdmstar/krylov.hpp:12-20). */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double kappa;
  double lambda_min;
  double lambda_max;
  double final_residual;
  double wall_time;
} fdmgpu_krylov_report;

/* Shared patch layout and factor statistics (PatchSolver::factor_nnz,
 * CholFactor::flops: include/fdmstar/schwarz.hpp:44, cholesky.hpp:21-24). */
typedef struct {
  int32_t npatch;        /* vertex-star patches                                   */
  int32_t n;             /* DOFs per patch, (2p-1)^d                              */
  int32_t n_interior;    /* cell-interior DOFs per patch, 2^d (p-1)^d             */
  int32_t n_interface;   /* separator DOFs per patch                              */
  int32_t tile;          /* dense tile edge of the interface factor               */
  int32_t tile_cols;     /* interface tile rows/columns                           */
  int32_t tiles;         /* stored (non-zero) lower tiles per patch               */
  int32_t pad_;
  int64_t nnz_L;         /* nnz(L_j) under the separator order in use, per patch  */
  int64_t flops_ref;     /* CholFactor::flops per patch (multiply-adds), same     */
  int64_t factor_bytes;  /* device bytes of the stored factor, all patches        */
  int64_t tile_gemms;    /* tile updates per patch (factorisation work units)     */
  int64_t nnz_L_reference;   /* nnz(L_j) under the reference patch_ordering       */
  int64_t flops_reference;   /* CholFactor::flops under the reference ordering    */
  int32_t separator_order;   /* 0 plane, 1 reference                              */
  int32_t top_direct;        /* 1: the Schur split forms S~_RR = S_RR - S_RF S_FF^{-1} S_FR from S's sparse
                                couplings and factors it densely (no full separator factor); else 0   */
  int64_t stream_bytes;      /* packed factor bytes streamed per sweep, all patches */
  int64_t dmma_flops;        /* FP64 tensor-pipe flops the batched factorisation issues per patch
                                (dense 64x64 tile GEMMs minus the skipped zero 16-wide panels) */
  int32_t schur_split;       /* Schur split: 1 the solve streams the top-separator factor L_RR, 2 its
                                symmetric inverse S~_RR^{-1} (default); 0 the full separator factor */
  int32_t n_top;             /* |R|: top-separator DOFs per patch (Schur split), else 0              */
  int64_t solve_values;      /* matrix values one relaxation solve reads per patch (fwd + bwd):
                                split: 2 nnz(L_RR) + 2 x S_FF components + S_RF + S_FR; else 2 nnz(L_G) */
} fdmgpu_layout;

/* Operator ids for fdmgpu_apply. */
enum {
  FDMGPU_OP_APPLY_ST = 0,   /* TransformedSystem::apply_St (src/assembly.cpp:326-342)  */
  FDMGPU_OP_APPLY_S = 1,    /* TransformedSystem::apply_S  (src/assembly.cpp:308-324)  */
  FDMGPU_OP_PATCH = 2,      /* PatchSolver::apply          (src/schwarz.cpp:41-54)     */
  FDMGPU_OP_SMOOTH = 3,     /* TwoLevel::smooth            (src/schwarz.cpp:121-123)   */
  FDMGPU_OP_A = 4,          /* GlobalOperator::apply       (src/assembly.cpp:56-88)    */
  FDMGPU_OP_VCYCLE = 5      /* TwoLevel::apply             (src/schwarz.cpp:125-133)   */
};

const char* fdmgpu_last_error(fdmgpu_handle h);
const char* fdmgpu_status_string(fdmgpu_status s);

/* ---- construction ---------------------------------------------------------- */
/* Replaces the device-side half of build_poisson_twolevel
 * (src/schwarz.cpp:230-252): a handle for a scalar Q_p space of dimension
 * dim (2|3) and degree p on ncells cells with ndof global DOFs. */
fdmgpu_status fdmgpu_create(fdmgpu_handle* out, int32_t dim, int32_t p, int32_t ncells, int64_t ndof,
                            int32_t device);
fdmgpu_status fdmgpu_destroy(fdmgpu_handle h);
fdmgpu_status fdmgpu_set_stream(fdmgpu_handle h, void* cuda_stream);
fdmgpu_status fdmgpu_synchronize(fdmgpu_handle h);

/* Linear elasticity, the SDC variant of the path (src/elasticity.cpp,
 * include/fdmstar/elasticity.hpp): turns a handle created for the vector Q_p
 * space (ndof = dim x scalar DOFs, vector_q_space's component-major
 * numbering, src/discretization.cpp:313-318) into the device half of
 * build_elasticity_twolevel (src/elasticity.cpp:204-229).  Call right after
 * fdmgpu_create.  The setters then take: set_mesh_maps -- component 0's cell
 * maps with multiplicity / constrained over all ndof; set_cell_coeffs -- the
 * geometric mu^K (Cartesian cells only, kappa NULL); set_patches -- the
 * vector star lists of build_patch_solver (all components) and their
 * patch_ordering; set_coarse -- the vector Q1 coarse inverse and
 * prolongation; set_coarse_cells -- component 0's coarse cell maps and the
 * vector coarse constrained flags.  FDMGPU_OP_A applies the true form
 * elasticity_primal_operator (src/elasticity.cpp:69-120), the relaxation the
 * SDC surrogate sdc_transformed (src/elasticity.cpp:122-167): per component
 * the scalar path with coefficients sdc_axis_coefficients(ci) * mu^K.
 * C = bundle.C (V^T W D on GL(p+1), src/assembly.cpp:49-52), (p+1)^2
 * column-major.  mu, lambda: the Lame parameters. */
fdmgpu_status fdmgpu_set_elasticity(fdmgpu_handle h, double mu, double lambda, const double* C);

/* Symmetric interior-penalty DG, the SIPG variant of the path (src/sipg.cpp,
 * include/fdmstar/sipg.hpp; the two-level DG solver of
 * tests/test_sipg.cpp:184-197).  Turns a fresh scalar handle for
 * dq_space(mesh, p) (all DOFs cell-local: cell_dofs per cell, multiplicity 1,
 * nothing constrained) into the device half of that solver; call before
 * fdmgpu_set_patches.  Cartesian cells.  Inputs:
 *   eta                 the penalty (sipg_default_eta = (p+1)(p+d), src/sipg.cpp:7);
 *   deriv_traces        FdmBasis::deriv_traces of the DG bundle (2 x (p+1), col-major);
 *   trace_values,       the GL-nodal reference interval's endpoint traces
 *   trace_normal_derivs (reference_interval.hpp:22-23, 2 x (p+1), col-major);
 *   facets              mesh.facets: cells (nf x 2, -1 = none), normal axis,
 *                       sides (nf x 2, -1/+1), tag (0 interior, 1 Dirichlet, 2 Neumann);
 *   cell_vertices       mesh.cells (ncells x 2^dim corner vertex ids, tensor order).
 * The setters then take: set_basis -- the DG bundle (S in GL representation,
 * A_t / B_t, A_hat / B_hat the GL-nodal stiffness / mass); set_patches -- the
 * DG vertex stars of build_patch_solver ((2p+2)^d DOFs each, whole cells) and
 * their patch_ordering; set_coarse -- the Q1 coarse inverse and
 * build_prolongation(dq_space, q_space(mesh, 1)).  FDMGPU_OP_A is then
 * dg_poisson_operator (src/sipg.cpp:176-250), the relaxation the patches of
 * transformed_dg_poisson (src/sipg.cpp:252-364), whose factors keep every
 * patch DOF (no interior elimination). */
fdmgpu_status fdmgpu_set_sipg(fdmgpu_handle h, double eta, const double* deriv_traces, const double* trace_values,
                              const double* trace_normal_derivs, int32_t nfacets, const int32_t* facet_cells,
                              const int32_t* facet_axis, const int32_t* facet_sides, const uint8_t* facet_tags,
                              const int32_t* cell_vertices);

/* FdmBasis (include/fdmstar/fdm_basis.hpp:21-32) and the reference interval
 * (reference_interval.hpp:15-27).  All (p+1)^2 arrays column-major:
 * S, A_t = S^T A S, B_t = S^T B S (values + structural 0/1 patterns), lambda
 * (p-1 interior eigenvalues), A_hat / B_hat (reference stiffness / mass),
 * and the GL(q) rule (points, weights) with its tables Vq, Dq (q x (p+1),
 * column-major) used by the true-form trilinear operator
 * (src/assembly.cpp:198-215, q = p+2). */
fdmgpu_status fdmgpu_set_basis(fdmgpu_handle h, const double* S, const double* lambda, const double* A_t,
                               const double* B_t, const uint8_t* A_t_pattern, const uint8_t* B_t_pattern,
                               const double* A_hat, const double* B_hat, int32_t q, const double* q_points,
                               const double* wq, const double* Vq, const double* Dq);

/* Discretization::Component maps (include/fdmstar/discretization.hpp:22-34):
 * cell_dofs / cell_modes ncells x (p+1)^d (axis 0 fastest), optional
 * mode_signs (+-1, same shape; NULL = all +1), multiplicity and the strong
 * Dirichlet mask (ndof). */
fdmgpu_status fdmgpu_set_mesh_maps(fdmgpu_handle h, const int32_t* cell_dofs, const int32_t* cell_modes,
                                   const double* mode_signs, const double* multiplicity,
                                   const uint8_t* constrained);

/* Per-cell data of cell_geometry (src/geometry.cpp:45-104): kind (0
 * Cartesian, 1 affine, 2 bilinear/trilinear), mu = kappa_K * mu^K (ncells x
 * dim; the separable surrogate of the patch solver and the exact Cartesian
 * coefficients), corner coordinates (ncells x 2^dim x 3, tensor corner order;
 * may be NULL when every cell is Cartesian) and kappa (ncells; NULL = 1). */
fdmgpu_status fdmgpu_set_cell_coeffs(fdmgpu_handle h, const uint8_t* kind, const double* mu,
                                     const double* corner_xyz, const double* kappa);

/* PatchSolver::Patch lists (src/schwarz.cpp:62-83): for patch j, the vertex,
 * its ascending star_dofs dofs[ptr[j]..ptr[j+1]) (src/discretization.cpp:
 * 266-297), the patch_ordering permutation perm (local indices,
 * src/ordering.cpp:17-45) and its 2^dim star cells (ascending ids; a
 * boundary-vertex star -- SolverConfig::skip_boundary_patches = false, the
 * reference default -- has fewer cells and pads with -1). */
fdmgpu_status fdmgpu_set_patches(fdmgpu_handle h, int32_t npatch, const int32_t* vertex, const int64_t* ptr,
                                 const int32_t* dofs, const int32_t* perm, const int32_t* star_cells);

/* Coarse level of TwoLevel (include/fdmstar/schwarz.hpp:52-66): dense
 * inverse of the assembled coarse matrix (ndof_c^2, row-major) and the
 * prolongation CSR (ndof rows, src/schwarz.cpp:139-165). */
fdmgpu_status fdmgpu_set_coarse(fdmgpu_handle h, int32_t ndof_c, const double* coarse_inverse,
                                const int64_t* P_ptr, const int32_t* P_col, const double* P_val);

/* Optional: the cell structure of the same prolongation, so P and P^T run as
 * cell-wise sum-factorised kernels instead of the CSR:
 * coarse_cell_dofs (ncells x 2^d, corner bit a = side along axis a, as the
 * reference's q_space(p = 1) cell_dofs), the coarse constrained flags, and the
 * Q1 hats at the fine GLL nodes, phat[(p+1) x 2] column-major -- the entries
 * build_prolongation (src/schwarz.cpp:139-165) sums.  Same operator; sums in
 * a different order (results equal to rounding). */
fdmgpu_status fdmgpu_set_coarse_cells(fdmgpu_handle h, const int32_t* coarse_cell_dofs,
                                      const uint8_t* coarse_constrained, const double* phat);

/* Batched numeric factorisation of every patch matrix A~_j under its
 * patch ordering (replaces cholesky(), src/cholesky.cpp:9-87, inside
 * build_patch_solver, src/schwarz.cpp:84-93).  Returns FDMGPU_NOT_SPD with
 * "cholesky: matrix not SPD at pivot k (patch j)" on a non-positive pivot.
 * With the plane-by-plane separator order (3D scalar CG layouts) it also
 * prepares the Schur-split solve the relaxation then uses (fdmgpu_layout.
 * schur_split): the first two facet planes are applied from the Schur
 * complement's own entries and only the top separator block is streamed, as
 * its explicit symmetric inverse (default) or its Cholesky factor (env
 * FDMGPU_TOP=chol); env FDMGPU_SCHUR=0 at fdmgpu_set_patches keeps the full
 * separator factor.  Patch solutions agree to rounding in every form. */
fdmgpu_status fdmgpu_factor(fdmgpu_handle h);
fdmgpu_status fdmgpu_get_layout(fdmgpu_handle h, fdmgpu_layout* out);
/* The separator Schur complement S_G = A_BB - A_BI A_II^{-1} A_IB of patch j
 * -- the matrix the batched factorisation factors (extract_submatrix of the
 * transformed matrix, src/sparse.cpp:17-31, with the closed-form interior
 * elimination applied) -- as a dense m x m column-major array in this
 * handle's separator order (fdmgpu_get_patch_elimination_dofs positions
 * n_I..n-1; absent positions of boundary stars hold identity rows). */
fdmgpu_status fdmgpu_patch_schur(fdmgpu_handle h, int32_t j, double* out);
/* Debug / parity entry, the twin of fdmgpu_patch_schur: x_j = A~_j^{-1} r_j
 * for patch j alone -- CholFactor::solve of patches[j].factor
 * (src/cholesky.cpp:89-110) as PatchSolver::apply calls it
 * (src/schwarz.cpp:41-54) -- with r_j / x_j host arrays in the order of
 * patches[j].dofs (ascending star_dofs ids, src/discretization.cpp:266-297),
 * length n_j.  Runs the batched device solve and keeps patch j's
 * correction only (cost of one relaxation's patch stage). */
fdmgpu_status fdmgpu_patch_solve_one(fdmgpu_handle h, int32_t j, const double* rhs, double* out);
/* Debug / parity entry: the separator Cholesky factor L of patch j (dense m x m,
 * column-major, lower triangle; S_G = L L^T with fdmgpu_patch_schur's S_G) -- the
 * factor cholesky() computes (src/cholesky.cpp:9-87) for the separator block.
 * Needs the dense factor tiles, i.e. a factor whose solve records were packed
 * into their own buffer (FDMGPU_UNSUPPORTED for factors packed in place). */
fdmgpu_status fdmgpu_patch_factor(fdmgpu_handle h, int32_t j, double* out);
/* Per-patch global DOFs in elimination order (npatch x n): dofs[perm[k]]. */
fdmgpu_status fdmgpu_get_patch_elimination_dofs(fdmgpu_handle h, int32_t* out);

/* ---- operators ----------------------------------------------------------------- */
/* Generic entry: op = FDMGPU_OP_*, omega used by FDMGPU_OP_VCYCLE, host != 0
 * means `in` / `out` are host pointers (copied inside, synchronous). */
fdmgpu_status fdmgpu_apply(fdmgpu_handle h, int32_t op, double omega, const double* in, double* out,
                           int32_t host);
/* Asynchronous host-buffer form of fdmgpu_apply for a stream of independent
 * vectors (many right-hand sides, serving): copies host_in (pinned) in on a
 * copy stream, runs op on the handle stream, copies the result out to
 * host_out (pinned) on a second copy stream, and returns at once, so the
 * copies of one call overlap the compute of its neighbours.  Two staging
 * slots: a call waits (on the device) for the slot used two calls earlier.
 * Host buffers must stay untouched until fdmgpu_synchronize returns, which
 * waits for every call in flight.  Same results as fdmgpu_apply. */
fdmgpu_status fdmgpu_apply_async(fdmgpu_handle h, int32_t op, double omega, const double* host_in, double* host_out);
/* Device-side join: the handle stream waits for every fdmgpu_apply_async copy-out in flight
 * (work enqueued on it afterwards -- e.g. a timing event -- runs after them). */
fdmgpu_status fdmgpu_async_join(fdmgpu_handle h);
fdmgpu_status fdmgpu_transform(fdmgpu_handle h, int32_t dir, const double* in, double* out); /* 0 S^T, 1 S */
fdmgpu_status fdmgpu_patch_solve(fdmgpu_handle h, const double* r_modal, double* z_modal);
fdmgpu_status fdmgpu_smooth(fdmgpu_handle h, const double* r, double* z);
fdmgpu_status fdmgpu_apply_A(fdmgpu_handle h, const double* x, double* y);
fdmgpu_status fdmgpu_vcycle(fdmgpu_handle h, double omega, const double* r, double* z);

/* pcg (src/krylov.cpp:29-83) with A = GlobalOperator::apply and
 * precond 0 = identity, 1 = smooth, 2 = V(1,1) cycle at the handle's omega.
 * b, x device vectors; residuals (optional, host, maxit entries) receives the
 * relative residual history. */
fdmgpu_status fdmgpu_pcg(fdmgpu_handle h, const double* b, double* x, double rtol, int32_t maxit,
                         int32_t precond, fdmgpu_krylov_report* report, double* residuals);

/* calibrate_damping (src/schwarz.cpp:97-119, 167-228): formula 0 TwoGrid,
 * 1 Smoother, 2 Paper; sets and returns omega with the Lanczos extremes. */
fdmgpu_status fdmgpu_calibrate_damping(fdmgpu_handle h, int32_t lanczos_steps, uint32_t seed, int32_t formula,
                                       double* omega, double* lambda_min, double* lambda_max);
fdmgpu_status fdmgpu_set_omega(fdmgpu_handle h, double omega);
fdmgpu_status fdmgpu_get_omega(fdmgpu_handle h, double* omega);

/* Internal elimination order of the separator DOFs, applied by the next
 * fdmgpu_set_patches: 0 = facet groups plane by plane (default; ~45 % fewer
 * factor nonzeros), 1 = the reference patch_ordering (src/ordering.cpp:17-45).
 * Patch solutions agree to rounding either way.  Env FDMGPU_SEP_ORDER=reference
 * selects 1 at fdmgpu_create. */
fdmgpu_status fdmgpu_set_separator_order(fdmgpu_handle h, int32_t order);

/* Number of kernels this handle has launched so far (evidence for bench.py). */
int64_t fdmgpu_launch_count(fdmgpu_handle h);

/* Per-kernel CUDA-event timing on the handle stream (bench.py roofline):
 * enable != 0 starts recording (and clears earlier records); which = 0 patch
 * solve, 1 factorisation kernels, 2 cell transforms, 3 stiffness apply, 4 the
 * top-block stage of the patch solve (Schur split: S~_RR^{-1} product or L_RR
 * solves; part of class 0). */
fdmgpu_status fdmgpu_kernel_timing(fdmgpu_handle h, int32_t enable);
fdmgpu_status fdmgpu_kernel_time(fdmgpu_handle h, int32_t which, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* FDMGPU_H */
