// Internal state of an fdmgpu handle (see include/fdmgpu.h) and the launch
// interface between the host orchestration (capi.cpp) and the sm_100a
// kernels (kernels/*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fdmgpu.h"

namespace fdmgpu {

constexpr int kTile = 64;  // dense tile edge of the interface factor
constexpr int kHdrBytes = 144;  // solve-record header: 2 x 64 sub-block indices + full / compact counts
constexpr int kCompact = 10;    // doubles per compact 8x8 sub-block (8 row values + 8 column bytes + pad)
constexpr int kHdrHost = kHdrBytes + 128;  // host tile_hdr stride: record header + compact index table
constexpr int kFormG = 6;      // column tiles per CTA of the direct top-block assembly (k_schur_form)
constexpr int kFormG2 = 12;    // column tiles per CTA of its half-row-tile form (k_schur_form2)
constexpr int kSpmvRows = 16;   // rows per block of the Schur split's coupling products

struct Error : std::runtime_error {
  fdmgpu_status status;
  Error(fdmgpu_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define FDM_CUDA(call)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw ::fdmgpu::Error(e_ == cudaErrorMemoryAllocation ? FDMGPU_OUT_OF_MEMORY : FDMGPU_CUDA_ERROR, \
                            std::string(#call) + ": " + cudaGetErrorString(e_));              \
  } while (0)

// Owning device allocation.
template <class T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  DevArray() = default;
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  ~DevArray() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    reset();
    if (count == 0) return;
    FDM_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void upload(const T* host, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) FDM_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
  size_t bytes() const { return n * sizeof(T); }
};

// Shared symbolic structure of all interior vertex-star patches (one
// canonical lattice pattern).
struct PatchLayout {
  int n = 0, nI = 0, m = 0, mpad = 0, nT = 0, ntiles = 0;
  int span = 0;                      // 2p+1 lattice points per axis
  int ragged = 0;                    // boundary stars embedded in the template (absent positions)
  std::vector<int32_t> lat;          // n: packed patch-lattice coords P (elimination order)
  std::vector<int32_t> pos_of_lat;   // span^d: elimination position or -1
  std::vector<int32_t> tile_row, tile_col, col_start;  // tile pattern, column-major order
  std::vector<int32_t> pair_ptr, pair_a, pair_b;       // left-looking update pairs per tile
  std::vector<int32_t> entries;      // structural nonzeros of S_G: tile << 12 | col << 6 | row
  std::vector<int32_t> tile_mask;             // 16x16 sub-blocks the factorisation touches per tile (GEMM panel skips)
  std::vector<int64_t> tile_mask8;            // 8x8 sub-blocks per tile kept in the solve stream
  std::vector<int32_t> tile_poff8;            // stream record offset (doubles): header + sub-blocks
  int lead_cols = 0;                          // leading tile columns without updates (batched)
  std::vector<int32_t> lead_diag, lead_trsm;  // their diagonal tiles; (tile, diagonal tile) pairs
  std::vector<uint8_t> tile_hdr;              // kHdrBytes record header per tile
  std::vector<int32_t> tile_bptr, tile_blk;   // per tile: its record's sub-blocks (bit bi*8 + bj), in record order
  std::vector<int64_t> tile_ccol;             // per record sub-block: compact column bytes (0 for full blocks)
  std::vector<int32_t> active, active_ptr;    // per column: tiles the update kernel must visit
  int64_t nnz_L = 0, flops_ref = 0, tile_gemms = 0;          // order in use
  int64_t dmma_flops = 0;                                   // tensor-pipe flops the factor kernels issue
  std::vector<int> colcount;                                // nnz per factor column (elimination order; diagnostics)
  int64_t nnz_L_reference = 0, flops_reference = 0;         // reference patch_ordering
};

// Two-level Schur split of the separator solve (schur_split.cpp).  With the
// plane-by-plane separator order the first two facet planes F = P0 | P1 have
// diagonal self-couplings, and P0 couples P1 only inside small components
// (3D: the facets sharing one tangential index, 2(p-1) + 2(p-1) DOFs), so
// S_FF^{-1} is applied exactly from S_FF's own entries (component-wise: a
// dense coupling block, the Cholesky inverse of its P1 Schur complement and
// the P0 diagonal), S_RF / S_FR stay unfactored, and only the dense Cholesky
// factor of S~_RR = S_RR - S_RF S_FF^{-1} S_FR (the top separator: the last
// plane, the edges and the vertex) is streamed:
//   x_R = S~_RR^{-1} (b_R - S_RF S_FF^{-1} b_F),  x_F = S_FF^{-1} (b_F - S_FR x_R).
// The fill block L_RF (a dense |R| x |P1| block, 62 % of the separator
// factor's nonzeros at p = 31) is never read by the solve.
struct SchurSplit {
  bool on = false;
  int nF = 0, n0 = 0, n1 = 0, nR = 0;
  int ncomp = 0, c0 = 0, c1 = 0;          // components; max P0 / P1 members (padded storage)
  std::vector<int32_t> comp0, comp1;      // ncomp x c0 / c1 separator positions (-1 = pad)
  std::vector<int32_t> rf_ptr, rf_col;    // S_RF, CSR over R rows (R-local), F columns (separator positions)
  std::vector<int32_t> fr_ptr, fr_col;    // S_FR, CSR over the F rows in component order, R-local columns
  std::vector<int32_t> fr_row;            // F row (separator position) of each S_FR row
  std::vector<int32_t> comp_fr;           // ncomp + 1: component k's S_FR rows (its P0 members, then P1)
  std::vector<int32_t> rf_blk, fr_blk;    // entry offset of every kSpmvRows-row block (4-aligned; + end)
  int rf_bmax = 0, fr_bmax = 0;           // largest block (entries, padding included)
  int64_t rf_nnz = 0, fr_nnz = 0;         // structural entries (without the block padding)
  int64_t comp_stride = 0;                // doubles per component: M (c1 x c0), Linv (c1 x c1), d0 (c0)
  int64_t vstride = 0;                    // doubles per patch: components, S_RF values, S_FR values
  int64_t rf_off = 0, fr_off = 0;         // value offsets inside a patch's block
  PatchLayout R;                          // dense tile layout of L_RR / S~_RR^{-1} (rows / columns nF..m-1)
  bool inv = true;                        // stream S~_RR^{-1} (symmetric, one pass) instead of L_RR (two passes)
  int nchunk = 1;                         // inverse: CTAs per patch of the symmetric product
  std::vector<int32_t> chunk_start;       // nchunk + 1 tile offsets
  // Direct top block (default with inv; FDMGPU_DIRECT=0 keeps the full tile factorisation):
  // S~_RR = S_RR - S_RF S_FF^{-1} S_FR is formed from S's sparse couplings and the explicit
  // component inverses, then factored as a dense nR x nR matrix -- the dense |R| x |P1| fill
  // block of the full factor is never computed.
  bool direct = false;
  int nl = 0;                             // c0 + c1: local indices of a component (P0 members, then P1)
  int nRp = 0;                            // R.mpad
  std::vector<int32_t> kr;                // ncomp x nRp: (first entry << 8 | count) of row r's S_RF entries in component k
  std::vector<int32_t> rk_ent;            // entries sorted by (component, row): local index | rf entry << 8
  std::vector<int32_t> e2;                // ncomp x nRp: the first two entries' local indices | min(count, 2) << 16 | (count > 2) << 18
  std::vector<int32_t> rr_entries;        // structural S_RR entries + padding diagonal: tile << 12 | col << 6 | row (R layout)
  std::vector<int32_t> form_I, form_J0;   // form CTAs: row tile I, first column tile (kFormG column tiles per CTA)
  std::vector<int32_t> form2_I, form2_J0; // k_schur_form2 CTAs: half row tile 2 I + h, first column tile (kFormG2 per CTA)
  std::vector<int32_t> pair_ptr, pair_a, pair_b, tile_mask;  // dense left-looking update lists of the R layout
};

// Device-resident PCG scalars (kernels/pcg.cu).
struct PcgDev {
  double bnorm, rtol, rz, rz_new, pAp, alpha, beta, res;
  int k, maxit, status;  // status: 0 running, 1 converged, 2 indefinite at iteration k+1, 3 maxit
};

struct Context;
void destroy_sub(Context* s);  // capi.cpp: frees a component sub-handle

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int64_t launches = 0;

  int dim = 3, p = 1, n1 = 2, npc = 8, ncells = 0;
  int64_t ndof = 0;

  // Vector (linear-elasticity SDC) handles, fdmgpu_set_elasticity: ncomp = dim
  // identical Q_p components, component ci's DOFs = component 0's + ci * nsc
  // (src/discretization.cpp:86-258).  The SDC relaxation is block diagonal over
  // components (src/elasticity.cpp:122-167), so each component runs on its
  // own scalar sub-context (its own coefficients c_ci * mu^K, factors and
  // buffers, this handle's stream); this context owns the true-form vector
  // operator (kernels/elastic.cu), the vector coarse level and the PCG loop.
  int ncomp = 1;
  int64_t nsc = 0;
  double lame_mu = 0.0, lame_lambda = 0.0;
  DevArray<double> Cm;                 // bundle.C = V^T W D on GL(p+1) (src/assembly.cpp:49-52)
  std::vector<Context*> comp;          // owned sub-contexts (ncomp > 1)
  int ncs = 0;                         // scalar coarse block size

  // Symmetric interior-penalty DG (fdmgpu_set_sipg, src/sipg.cpp): dq_space
  // DOFs (all cell-local), the SIPG true form (cell Kronecker terms + facet
  // penalty terms, dg_poisson_operator :176-250) as FDMGPU_OP_A, the
  // transformed DG matrix (transformed_dg_poisson :252-364) in the patches,
  // which keep every DOF of their 2^d cells (no interior elimination).
  bool dg = false;
  double eta = 0.0;
  DevArray<double> dtr, tv, tnd;          // 2 x (p+1): FDM-mode derivative traces, GL nodal traces / normal derivs
  DevArray<int32_t> fnbr;                 // ncells x 2d: neighbour across local facet (axis, side), -1 none
  DevArray<uint8_t> ftag;                 // ncells x 2d: 0 interior, 1 dirichlet, 2 neumann
  std::vector<int32_t> h_cell_vertices;   // ncells x 2^d mesh corners (tensor order)

  // basis
  DevArray<double> S, St, Ahat, Bhat, At, Bt, Vq, Dq, wq, qpts, Qbuf;
  std::vector<double> h_At, h_Bt;
  std::vector<uint8_t> h_Anz, h_Bnz;
  int q = 0;
  bool have_basis = false;

  // maps
  DevArray<int32_t> cell_dofs, cell_modes, g_ptr, g_idx, gm_ptr, gm_idx;
  DevArray<double> mode_sign, inv_mult, E, E2;
  // modal DOFs on cell boundaries (ascending): the only entries of the patch-summed
  // correction the interior-rebuilding S transform reads (op_smooth's compact patch gather)
  DevArray<int32_t> bnd_list;
  DevArray<uint8_t> constrained;
  std::vector<int32_t> h_cell_dofs, h_cell_modes;
  std::vector<uint8_t> h_constrained;
  bool modes_alias = true, have_maps = false;

  // cell coefficients
  DevArray<uint8_t> kind;
  DevArray<double> mu, xyz, kappa;
  std::vector<double> h_mu;
  bool all_cartesian = true, have_coeffs = false;

  // patches
  int npatch = 0;
  PatchLayout L;
  DevArray<int32_t> pdofs, lat, pos_of_lat, pcells, pg_ptr, pg_idx;
  DevArray<int32_t> tile_row, tile_col, col_start, pair_ptr, pair_a, pair_b, entries, tile_mask, active, tile_poff8, lead_diag, lead_trsm;
  DevArray<int64_t> tile_mask8, tile_ccol;
  DevArray<int32_t> tile_bptr, tile_blk;
  DevArray<uint8_t> tile_hdr;
  DevArray<double> corr, tiles, nK;
  // packed solve records in their own buffer when memory allows (packing then
  // overlaps the factorisation on pack_stream); empty -> packed in place
  DevArray<double> packed;
  cudaStream_t pack_stream = nullptr;
  cudaEvent_t pack_ev = nullptr;
  std::vector<int32_t> h_pdofs, h_pcells;
  // Schur-split solve (SchurSplit above; FDMGPU_SCHUR=0 keeps the full-factor stream)
  SchurSplit sx;
  bool schur_enabled = true;
  DevArray<int32_t> sx_comp0, sx_comp1, sx_comp_fr, sx_rf_blk, sx_fr_blk, sx_rf_ptr, sx_rf_col, sx_fr_ptr, sx_fr_col, sx_fr_row, sx_pdofs, sx_pairs, sx_tidx;
  DevArray<int32_t> sx_tile_row, sx_tile_col, sx_col_start, sx_poff8, sx_bptr, sx_blk;
  DevArray<int64_t> sx_ccol;
  DevArray<uint8_t> sx_hdr;
  DevArray<int32_t> sx_chunk;
  DevArray<int32_t> sx_form2_I, sx_form2_J0;
  DevArray<int32_t> sx_kr, sx_rk_ent, sx_rr_entries, sx_form_I, sx_form_J0, sx_pair_ptr, sx_pair_a, sx_pair_b, sx_tile_mask;
  DevArray<int32_t> sx_e2;         // direct top block: SchurSplit::e2
  DevArray<double> sx_fv2;         // direct top block: the first two S_RF values of (component, row), npatch x ncomp x nRp x 2
  DevArray<double> sx_inv, sx_fv;  // direct top block: component inverses (npatch x ncomp x nl x nl), S_RF values in rk_ent order
  DevArray<double> sx_vals, sx_tR, sx_F, diagL, sx_UT, sx_part;  // per-patch values; R right-hand sides; F work; L_KK of R tiles
  int sx_K0 = 0;                                 // first full-factor tile column overlapping R
  int solve_cs = 0;                     // CTAs per split patch (FDMGPU_SOLVE_CS; 0 = auto, 1 = no split)
  bool solve_tail = true;                // cluster-split only the last partial wave (FDMGPU_SOLVE_TAIL)
  int cl_cs = 0;                         // cluster size cl_list / cl_col were built for
  DevArray<int32_t> cl_list, cl_col;     // per-rank tile lists of the cluster solve
  int cl_fit[5] = {-1, -1, -1, -1, -1};  // co-resident clusters per cluster size (memo)
  DevArray<unsigned> tail_sync;          // finished split-tail CTAs, completed calls
  DevArray<unsigned> fac_flag;           // npatch x nT: epoch at which L_KK^{-1} was published (k_patch_column)
  unsigned fac_epoch = 0;                // factorisation count (flags never need a reset)
  bool fused_columns = true;             // FDMGPU_FUSED=0: separate update / trsm launches
  bool have_patches = false, factored = false;
  DevArray<unsigned long long> d_err;

  // coarse level
  int nc = 0;
  DevArray<double> cinv, P_val, PT_val, rc, zc;
  DevArray<int32_t> P_ptr, P_col, PT_ptr, PT_col;
  bool have_coarse = false;
  // cell-wise transfer (fdmgpu_set_coarse_cells): coarse cell maps, coarse
  // gather CSR over (cell, corner) slots, prolongation owner flags, Q1 hats
  DevArray<int32_t> ccd, cg_ptr, cg_idx;
  DevArray<uint8_t> powner;
  DevArray<double> phat, cellsum;
  bool have_coarse_cells = false;

  // work vectors (ndof)
  DevArray<double> w[12];
  DevArray<double> red;   // reduction partials
  std::vector<double> h_red;
  double omega = 1.0, lambda_min = 0.0, lambda_max = 0.0;

  // device PCG: one CUDA graph with a WHILE node (rebuilt when the
  // preconditioner, omega or the coefficient capacity changes)
  DevArray<PcgDev> pcg_state;
  DevArray<double> pcg_alphas, pcg_betas, pcg_res;
  cudaGraphExec_t pcg_exec = nullptr;
  cudaStream_t cap_stream = nullptr;  // private stream for graph captures
  int pcg_precond = -1, pcg_cap = 0;
  double pcg_omega = 0.0;

  // asynchronous host-buffer applies (fdmgpu_apply_async): copy-in / copy-out
  // streams, two staging slots, per-slot events
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  DevArray<double> stage_in[2], stage_out[2];
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  int async_slot = 0;
  bool async_ready = false;  // streams, events and both staging slots all created

  // optional per-kernel CUDA-event timing (fdmgpu_kernel_timing)
  bool timing = false;
  bool capturing = false;  // inside a CUDA-graph capture: launches are recorded, not counted
  bool force_staged = false;  // FDMGPU_FORCE_STAGED=1: staged cell kernels for every p (tests)
  bool pdl = true;            // programmatic dependent launch in the relaxation chain (FDMGPU_PDL=0 disables)
  int sep_order = 0;  // 0 plane-by-plane facets (default), 1 reference patch_ordering (FDMGPU_SEP_ORDER)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev[5];

  void check_ready(bool need_patches, bool need_factor, bool need_coarse) const;
  // Component sub-context ci, synchronised with this handle's launch state
  // (stream -- swapped during graph capture --, capture / timing / PDL flags).
  Context& sub(int ci) {
    Context& s = *comp[ci];
    s.stream = stream;
    s.capturing = capturing;
    s.timing = timing;
    s.pdl = pdl;
    return s;
  }
  ~Context() {
    for (Context* s : comp) destroy_sub(s);
    if (pcg_exec) cudaGraphExecDestroy(pcg_exec);
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t e : {ev_in[k], ev_comp[k], ev_out[k]})
        if (e) cudaEventDestroy(e);
    if (h2d_stream) cudaStreamDestroy(h2d_stream);
    if (pack_ev) cudaEventDestroy(pack_ev);
    if (pack_stream) cudaStreamDestroy(pack_stream);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (auto& v : tev)
      for (auto& [a, b] : v) {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
  }
};

// Records CUDA events around one launch on the handle stream when timing is on.
// Timed kernel classes: 0 patch solve, 1 factor (assemble/update/trsm),
// 2 cell transforms, 3 stiffness apply, 4 the Schur split's top-block stage
// of the patch solve (inside class 0).
struct KernelTimer {
  Context& c;
  int slot;
  cudaEvent_t a = nullptr, b = nullptr;
  KernelTimer(Context& ctx, int s) : c(ctx), slot(s) {
    if (!c.timing) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, c.stream);
  }
  ~KernelTimer() {
    if (!c.timing) return;
    cudaEventRecord(b, c.stream);
    c.tev[slot].emplace_back(a, b);
  }
};

// ---- kernel launchers (kernels/*.cu) -------------------------------------------
void launch_cells_transform(Context& c, int dir, const double* in, int flags, const double* aux);  // writes c.E
void launch_cells_schur(Context& c, const double* in);              // writes c.E
void launch_cells_recon(Context& c, double* z, const double* rb);
void launch_gather(Context& c, int mode, const double* E, const double* x, double* out);
void launch_gather_bnd(Context& c, const double* E, double* out);  // mode 0 over the cell-boundary DOFs only
bool cells_slab32(const Context& c);  // the p = 31 slab transform path is the one launch_cells_transform takes
void launch_gather_vec(Context& c, int mode, const double* E, const double* x, double* out);  // all components
void launch_cells_stiffness(Context& c, const double* x);            // writes c.E
void launch_cells_quadrature(Context& c, const double* x);           // writes c.E (true form)
void launch_cells_elastic(Context& c, const double* x);              // writes c.E (ncomp blocks, elasticity)
size_t elastic_smem_bytes(const Context& c);
void launch_patch_assemble(Context& c);
void launch_dg_patch_assemble(Context& c);                            // kernels/sipg.cu
void launch_dg_facets(Context& c, const double* x);                    // adds the SIPG facet terms to c.E
void launch_patch_assemble_one(Context& c, int j, double* out);  // S_G of patch j, tile layout
void launch_patch_update(Context& c, int K);
void launch_patch_trsm(Context& c, int K);
void launch_patch_column(Context& c, int K);  // fused update + diagonal factor + trsm of tile column K
void launch_patch_lead(Context& c);
void launch_patch_pack(Context& c);
void launch_patch_pack_col(Context& c, int K);   // separate record buffer, side stream
void launch_patch_pack_join(Context& c);
void launch_schur_setup(Context& c);   // Schur split: S_FF components, S_RF / S_FR values (any time after set_cell_coeffs)
void launch_schur_retile(Context& c);  // Schur split: L_RR records from the factored tiles
void launch_schur_direct(Context& c);  // Schur split, direct top block: S~_RR formed and factored without the full factor
void launch_patch_solve(Context& c, const double* r_modal);          // writes c.corr
void launch_patch_gather(Context& c, double* z_modal);
void launch_patch_gather_bnd(Context& c, double* z_modal);  // cell-boundary DOFs only (op_smooth)
void launch_axpby(Context& c, int64_t n, double a, const double* x, double b, const double* y, double* out);
void launch_dot_partials(Context& c, int64_t n, const double* x, const double* y, int k);
void launch_restrict(Context& c, const double* fine, double* coarse);
void launch_coarse_solve(Context& c, const double* rc, double* zc);
void launch_prolong_add(Context& c, const double* coarse, double* fine);
constexpr int kRedBlocks = 296;  // fixed reduction grid: deterministic partial sums
void launch_dot_finish(Context& c, int k, double* dst);
void pcg_state_init(Context& c, void* st, double bnorm, double rtol, double rz, int maxit);
void pcg_state_read(Context& c, const void* st, int* k, int* status);
void launch_pcg_alpha(Context& c, void* st, double* alphas, cudaGraphConditionalHandle hw);
void launch_pcg_update_xr(Context& c, const void* st, const double* p, const double* Ap, double* x, double* r);
void launch_pcg_residual(Context& c, void* st, double* residuals, cudaGraphConditionalHandle hw,
                         cudaGraphConditionalHandle hi);
void launch_pcg_beta(Context& c, void* st, double* betas);
void launch_pcg_update_p(Context& c, const void* st, const double* z, double* p);
void prepare_buffers(Context& c);

}  // namespace fdmgpu
