// extern "C" implementation of include/fdmgpu.h: uploads, the batched
// factorisation schedule, and the host-driven V-cycle / PCG / damping
// calibration around the device operators.  All arithmetic on vectors of
// length ndof runs on the GPU; the host only sees scalars (dot products) and
// the Lanczos tridiagonal, as in src/krylov.cpp:29-83.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "context.hpp"

namespace fdmgpu {
void analyze_schur_split(Context& c);

// Schur-split solve state (SchurSplit, context.hpp): host analysis, index
// uploads and the split's buffers -- the L_RR records (c.packed), the diagonal
// L_KK side copies, per-patch values, right-hand side / work vectors.  Left
// off (full-factor stream) when the layout does not split or memory is short.
void setup_schur_split(Context& c) {
  c.sx = SchurSplit();
  for (auto* a : {&c.sx_comp0, &c.sx_comp1, &c.sx_comp_fr, &c.sx_rf_blk, &c.sx_fr_blk, &c.sx_rf_ptr, &c.sx_rf_col, &c.sx_fr_ptr, &c.sx_fr_col,
                  &c.sx_fr_row, &c.sx_pdofs, &c.sx_pairs, &c.sx_tidx, &c.sx_tile_row, &c.sx_tile_col, &c.sx_col_start,
                  &c.sx_poff8, &c.sx_bptr, &c.sx_blk})
    a->reset();
  c.sx_ccol.reset();
  c.sx_hdr.reset();
  for (auto* a : {&c.sx_vals, &c.sx_tR, &c.sx_F, &c.diagL, &c.sx_UT, &c.sx_part, &c.sx_inv, &c.sx_fv, &c.sx_fv2}) a->reset();
  for (auto* a : {&c.sx_kr, &c.sx_rk_ent, &c.sx_rr_entries, &c.sx_form_I, &c.sx_form_J0, &c.sx_form2_I, &c.sx_form2_J0, &c.sx_e2, &c.sx_pair_ptr, &c.sx_pair_a,
                  &c.sx_pair_b, &c.sx_tile_mask})
    a->reset();
  c.sx_chunk.reset();
  if (c.dg) return;
  analyze_schur_split(c);
  SchurSplit& S = c.sx;
  if (!S.on) return;
  const auto& L = c.L;
  const int K0 = S.nF / kTile;
  const size_t np = size_t(c.npatch);
  const size_t tt = size_t(kTile) * kTile, rtiles = size_t(S.R.ntiles) * tt;
  const size_t rec = S.inv ? std::max(size_t(S.R.tile_poff8.back()), rtiles) : size_t(S.R.tile_poff8.back());
  if (S.inv) {  // symmetric product: chunks per patch so that npatch x nchunk CTAs fill whole waves
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device);
    int best = 1;
    double best_eff = 0.0;
    for (int g = 1; g <= 16; ++g) {
      if (g > S.R.ntiles) break;
      const double waves = double(c.npatch) * g / nsm, eff = waves / std::ceil(waves);
      if (eff > best_eff + 0.01 || (g >= 4 && best < 4 && eff > best_eff - 0.05)) {
        best = g;
        best_eff = eff;
      }
    }
    const char* ch = std::getenv("FDMGPU_SYMV_CHUNKS");  // override (tests / tuning)
    S.nchunk = ch ? std::max(1, std::min(64, std::atoi(ch))) : best;
    S.chunk_start.assign(1, 0);
    const int64_t total = S.R.tile_poff8.back();
    for (int g = 1; g < S.nchunk; ++g) {
      const int64_t target = total * g / S.nchunk;
      int t = S.chunk_start.back();
      while (t < S.R.ntiles && S.R.tile_poff8[t] < target) ++t;
      S.chunk_start.push_back(t);
    }
    S.chunk_start.push_back(S.R.ntiles);
  }
  // (the full factor tiles are allocated after this analysis, unless the top block is formed directly)
  const size_t need = sizeof(double) * (np * rec + np * size_t(S.vstride) + np * size_t(S.nR + S.nF) +
                                        (S.inv ? np * rtiles + np * S.nchunk * size_t(S.R.mpad) : 0) +
                                        (S.direct ? np * size_t(S.ncomp) * S.nl * S.nl + np * S.rk_ent.size() + np * size_t(S.ncomp) * S.nRp * 2
                                                  : np * size_t(L.nT - K0) * tt + np * size_t(L.ntiles) * tt));
  size_t fb = 0, tb = 0;
  FDM_CUDA(cudaMemGetInfo(&fb, &tb));
  if (need + (size_t(1) << 30) > fb) {  // keep 1 GiB of headroom for work vectors
    S = SchurSplit();
    return;
  }
  // every R x R tile of the full factor must exist (L_RR is dense)
  std::vector<int32_t> tidx(size_t(L.nT) * L.nT, -1);
  for (int t = 0; t < L.ntiles; ++t) tidx[size_t(L.tile_row[t]) * L.nT + L.tile_col[t]] = t;
  for (int I = K0; I < L.nT; ++I)
    for (int J = K0; J <= I; ++J)
      if (tidx[size_t(I) * L.nT + J] < 0) {
        S = SchurSplit();
        return;
      }
  // (r | c << 16) of every stored coupling value (S_RF then S_FR, block padding -1 = zero)
  std::vector<int32_t> pairs(S.rf_col.size() + S.fr_col.size(), -1);
  for (int r = 0; r < S.nR; ++r)
    for (int e = S.rf_ptr[r]; e < S.rf_ptr[r + 1]; ++e) pairs[e] = (S.nF + r) | (S.rf_col[e] << 16);
  for (size_t f = 0; f < S.fr_row.size(); ++f)
    for (int e = S.fr_ptr[f]; e < S.fr_ptr[f + 1]; ++e)
      pairs[S.rf_col.size() + e] = S.fr_row[f] | ((S.nF + S.fr_col[e]) << 16);
  std::vector<int32_t> rp(np * S.nR);
  for (size_t i = 0; i < rp.size(); ++i) rp[i] = int32_t(i);
  c.sx_K0 = K0;
  c.sx_comp0.upload(S.comp0, c.stream);
  c.sx_comp1.upload(S.comp1, c.stream);
  c.sx_comp_fr.upload(S.comp_fr, c.stream);
  c.sx_rf_blk.upload(S.rf_blk, c.stream);
  c.sx_fr_blk.upload(S.fr_blk, c.stream);
  c.sx_rf_ptr.upload(S.rf_ptr, c.stream);
  c.sx_rf_col.upload(S.rf_col.empty() ? std::vector<int32_t>{0} : S.rf_col, c.stream);
  c.sx_fr_ptr.upload(S.fr_ptr, c.stream);
  c.sx_fr_col.upload(S.fr_col.empty() ? std::vector<int32_t>{0} : S.fr_col, c.stream);
  c.sx_fr_row.upload(S.fr_row, c.stream);
  c.sx_pairs.upload(pairs.empty() ? std::vector<int32_t>{0} : pairs, c.stream);
  c.sx_pdofs.upload(rp, c.stream);
  c.sx_tidx.upload(tidx, c.stream);
  c.sx_tile_row.upload(S.R.tile_row, c.stream);
  c.sx_tile_col.upload(S.R.tile_col, c.stream);
  c.sx_col_start.upload(S.R.col_start, c.stream);
  c.sx_poff8.upload(S.R.tile_poff8, c.stream);
  c.sx_bptr.upload(S.R.tile_bptr, c.stream);
  c.sx_blk.upload(S.R.tile_blk, c.stream);
  c.sx_ccol.upload(S.R.tile_ccol, c.stream);
  c.sx_hdr.upload(S.R.tile_hdr, c.stream);
  c.packed.alloc(np * rec);
  if (S.inv) {
    c.sx_UT.alloc(np * rtiles);
    c.sx_part.alloc(np * S.nchunk * size_t(S.R.mpad));
    c.sx_chunk.upload(S.chunk_start, c.stream);
  }
  if (S.direct) {
    c.sx_kr.upload(S.kr, c.stream);
    c.sx_rk_ent.upload(S.rk_ent, c.stream);
    c.sx_rr_entries.upload(S.rr_entries, c.stream);
    c.sx_form_I.upload(S.form_I, c.stream);
    c.sx_form_J0.upload(S.form_J0, c.stream);
    c.sx_form2_I.upload(S.form2_I, c.stream);
    c.sx_form2_J0.upload(S.form2_J0, c.stream);
    c.sx_pair_ptr.upload(S.pair_ptr, c.stream);
    c.sx_pair_a.upload(S.pair_a, c.stream);
    c.sx_pair_b.upload(S.pair_b, c.stream);
    c.sx_tile_mask.upload(S.tile_mask, c.stream);
    c.sx_inv.alloc(np * size_t(S.ncomp) * S.nl * S.nl);
    c.sx_fv.alloc(np * S.rk_ent.size());
    c.sx_e2.upload(S.e2, c.stream);
    c.sx_fv2.alloc(np * size_t(S.ncomp) * S.nRp * 2);
  } else {
    c.diagL.alloc(np * size_t(L.nT - K0) * kTile * kTile);
  }
  c.sx_vals.alloc(np * size_t(S.vstride));
  c.sx_tR.alloc(np * size_t(S.nR));
  c.sx_F.alloc(np * size_t(S.nF));
}

void analyze_patches(Context& c, int npatch, const int32_t* vertex, const int64_t* ptr, const int32_t* dofs,
                     const int32_t* perm, const int32_t* star_cells);
void analyze_dg_patches(Context& c, int npatch, const int32_t* vertex, const int64_t* ptr, const int32_t* dofs,
                        const int32_t* perm, const int32_t* star_cells);

void Context::check_ready(bool need_patches, bool need_factor, bool need_coarse) const {
  if (!have_basis || !have_maps || !have_coeffs)
    throw Error(FDMGPU_INVALID_ARGUMENT, "fdmgpu: basis, mesh maps and cell coefficients must be set first");
  if (need_patches && !have_patches) throw Error(FDMGPU_INVALID_ARGUMENT, "fdmgpu: patches not set");
  if (need_factor && !factored) throw Error(FDMGPU_INVALID_ARGUMENT, "fdmgpu: patches not factored");
  if (need_coarse && !have_coarse) throw Error(FDMGPU_INVALID_ARGUMENT, "fdmgpu: coarse level not set");
}

namespace {

// Gather CSR: for each DOF, its (cell, lattice) slots in ascending cell order.
// skip_absent: entries -1 (absent positions of boundary stars) are left out.
void build_gather(const std::vector<int32_t>& map, int64_t ndof, std::vector<int32_t>& ptr,
                  std::vector<int32_t>& idx, bool skip_absent = false) {
  ptr.assign(ndof + 1, 0);
  for (int32_t g : map) {
    if (skip_absent && g == -1) continue;
    if (g < 0 || g >= ndof) throw Error(FDMGPU_INVALID_ARGUMENT, "cell map entry out of range");
    ++ptr[g + 1];
  }
  for (int64_t i = 0; i < ndof; ++i) ptr[i + 1] += ptr[i];
  idx.assign(ptr[ndof], 0);
  std::vector<int32_t> pos(ptr.begin(), ptr.end() - 1);
  for (size_t e = 0; e < map.size(); ++e)
    if (map[e] >= 0) idx[pos[map[e]]++] = int32_t(e);
}

double host_dot(Context& c, const double* x, const double* y) {
  launch_dot_partials(c, c.ndof, x, y, 0);
  c.h_red.resize(kRedBlocks);
  FDM_CUDA(cudaMemcpyAsync(c.h_red.data(), c.red.p, kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  FDM_CUDA(cudaStreamSynchronize(c.stream));
  double s = 0.0;
  for (int b = 0; b < kRedBlocks; ++b) s += c.h_red[b];
  return s;
}

// Drops the captured PCG graph: it holds the device pointers and the kernel
// path of the state it was captured on, so every setter that reallocates or
// re-selects device state must call this (the next pcg re-captures).
void invalidate_graph(Context& c) {
  if (c.pcg_exec) {
    cudaGraphExecDestroy(c.pcg_exec);
    c.pcg_exec = nullptr;
  }
  c.pcg_precond = -1;
}

void copy_dev(Context& c, double* dst, const double* src) {
  FDM_CUDA(cudaMemcpyAsync(dst, src, c.ndof * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
}

// ---- device operators ----------------------------------------------------------
// Vector (elasticity SDC) handles run the block-diagonal operators component
// by component on their scalar sub-contexts (contiguous component blocks).
template <class Fn>
void per_component(Context& c, const double* in, double* out, Fn&& fn) {
  for (int ci = 0; ci < c.ncomp; ++ci) fn(c.sub(ci), in + ci * c.nsc, out + ci * c.nsc);
}

void op_transform(Context& c, int dir, const double* in, double* out) {
  if (c.ncomp > 1)
    return per_component(c, in, out, [&](Context& s, const double* i, double* o) { op_transform(s, dir, i, o); });
  launch_cells_transform(c, dir, in, 0, nullptr);
  launch_gather(c, dir, c.E.p, nullptr, out);
}

// PatchSolver::apply on a modal vector (src/schwarz.cpp:41-54): Schur-reduced
// separator RHS, batched separator solves, patch sum, interior rebuild.
void op_patch(Context& c, const double* in, double* out) {
  if (c.ncomp > 1) return per_component(c, in, out, [](Context& s, const double* i, double* o) { op_patch(s, i, o); });
  if (c.dg) {  // SIPG: the patches hold every DOF of their cells, no interior elimination
    launch_patch_solve(c, in);
    launch_patch_gather(c, out);
    return;
  }
  launch_cells_schur(c, in);
  launch_gather(c, 3, c.E.p, in, c.w[6].p);
  launch_patch_solve(c, c.w[6].p);
  launch_patch_gather(c, out);
  launch_cells_recon(c, out, in);
}

// TwoLevel::smooth (src/schwarz.cpp:121-123) = S * PatchSolver(S^T r), with
// the interior elimination fused into the two cell transforms.
void op_smooth(Context& c, const double* r, double* z) {
  if (c.ncomp > 1) return per_component(c, r, z, [](Context& s, const double* i, double* o) { op_smooth(s, i, o); });
  if (c.dg) {  // S * PatchSolver(S^T r) on the transformed DG system
    launch_cells_transform(c, 0, r, 0, nullptr);
    launch_gather(c, 0, c.E.p, nullptr, c.w[6].p);
    launch_patch_solve(c, c.w[6].p);
    launch_patch_gather(c, c.w[7].p);
    launch_cells_transform(c, 1, c.w[7].p, 0, nullptr);
    launch_gather(c, 1, c.E.p, nullptr, z);
    return;
  }
  launch_cells_transform(c, 0, r, 1, nullptr);  // S^T r, minus each cell's interior-elimination share
  // p = 31 slab path: only the cell-boundary entries of S^T r are summed over the cells (the
  // separator solves read nothing else); the cell-interior entries have one owner and stay where
  // the S^T pass left them, in the E-vector, for the S pass's interior rebuild (FDMGPU_SMOOTH_LOCAL=0:
  // the full gather and the rebuild through the global vector)
  const char* lenv = std::getenv("FDMGPU_SMOOTH_LOCAL");
  const bool local = !(lenv && lenv[0] == '0') && cells_slab32(c) && c.bnd_list.p;
  if (local) {
    launch_gather_bnd(c, c.E.p, c.w[6].p);
    launch_patch_solve(c, c.w[6].p);
    launch_patch_gather_bnd(c, c.w[7].p);
    launch_cells_transform(c, 1, c.w[7].p, 2 | 4, c.E.p);  // rebuild interiors from E, S
    launch_gather(c, 1, c.E.p, nullptr, z);
    return;
  }
  launch_gather(c, 0, c.E.p, nullptr, c.w[6].p);
  launch_patch_solve(c, c.w[6].p);               // separator solves
  // patch-summed separator corrections: only the cell-boundary entries -- the S
  // transform rebuilds every cell-interior value from the faces and never reads them
  launch_patch_gather_bnd(c, c.w[7].p);
  launch_cells_transform(c, 1, c.w[7].p, 2, c.w[6].p);  // rebuild interiors, S
  launch_gather(c, 1, c.E.p, nullptr, z);
}

void op_A(Context& c, const double* x, double* y) {  // src/assembly.cpp:56-88
  if (c.ncomp > 1) {  // elasticity_primal_operator (src/elasticity.cpp:69-120): all blocks in one cell pass
    launch_cells_elastic(c, x);
    launch_gather_vec(c, 2, c.E.p, x, y);
    return;
  }
  launch_cells_stiffness(c, x);
  if (c.dg) launch_dg_facets(c, x);  // dg_poisson_operator's facet terms (src/sipg.cpp:192-248)
  launch_gather(c, 2, c.E.p, x, y);
}

// Coarse transfer: component-wise cell kernels on vector handles with cell
// transfer data, else the handle's own (CSR or cell) path.
void transfer_restrict(Context& c, const double* fine, double* coarse) {
  if (c.ncomp > 1 && c.have_coarse_cells) {
    for (int ci = 0; ci < c.ncomp; ++ci) launch_restrict(c.sub(ci), fine + ci * c.nsc, coarse + ci * c.ncs);
    return;
  }
  launch_restrict(c, fine, coarse);
}
void transfer_prolong_add(Context& c, const double* coarse, double* fine) {
  if (c.ncomp > 1 && c.have_coarse_cells) {
    for (int ci = 0; ci < c.ncomp; ++ci) launch_prolong_add(c.sub(ci), coarse + ci * c.ncs, fine + ci * c.nsc);
    return;
  }
  launch_prolong_add(c, coarse, fine);
}

void op_vcycle(Context& c, double omega, const double* r, double* z) {  // src/schwarz.cpp:125-133
  double* t1 = c.w[3].p;
  double* t2 = c.w[4].p;
  double* t3 = c.w[5].p;
  op_smooth(c, r, t1);
  launch_axpby(c, c.ndof, omega, t1, 0.0, t1, z);  // z = omega * smooth(r)
  op_A(c, z, t2);
  launch_axpby(c, c.ndof, 1.0, r, -1.0, t2, t3);  // r1 = r - A z
  transfer_restrict(c, t3, c.rc.p);
  launch_coarse_solve(c, c.rc.p, c.zc.p);
  transfer_prolong_add(c, c.zc.p, z);  // z += P A_c^{-1} P^T r1
  op_A(c, z, t2);
  launch_axpby(c, c.ndof, 1.0, r, -1.0, t2, t3);  // r2 = r - A z
  op_smooth(c, t3, t1);
  launch_axpby(c, c.ndof, omega, t1, 1.0, z, z);  // z += omega * smooth(r2)
}

void op_precond(Context& c, int precond, double omega, const double* r, double* z) {
  if (precond == 0)
    copy_dev(c, z, r);
  else if (precond == 1)
    op_smooth(c, r, z);
  else
    op_vcycle(c, omega, r, z);
}

// Extremal eigenvalues of a symmetric tridiagonal (Sturm bisection); the
// reference uses Eigen::SelfAdjointEigenSolver (src/krylov.cpp:18-27).
std::pair<double, double> tridiag_extremes(const std::vector<double>& dg, const std::vector<double>& off) {
  const int n = int(dg.size());
  if (n == 0) return {0.0, 0.0};
  double lo = dg[0], hi = dg[0];
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? std::abs(off[i - 1]) : 0.0) + (i + 1 < n ? std::abs(off[i]) : 0.0);
    lo = std::min(lo, dg[i] - r);
    hi = std::max(hi, dg[i] + r);
  }
  auto count = [&](double x) {
    int cnt = 0;
    double q = 1.0;
    for (int i = 0; i < n; ++i) {
      q = dg[i] - x - (i > 0 ? off[i - 1] * off[i - 1] / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0) ++cnt;
    }
    return cnt;
  };
  auto kth = [&](int k) {
    double a = lo, b = hi;
    for (int it = 0; it < 200; ++it) {
      const double m = 0.5 * (a + b);
      if (m <= a || m >= b) break;
      if (count(m) > k)
        b = m;
      else
        a = m;
    }
    return 0.5 * (a + b);
  };
  return {kth(0), kth(n - 1)};
}

// Builds the device-resident PCG loop (kernels/pcg.cu) as one CUDA graph:
// WHILE(cont){ A p, p.Ap, alpha, x/r update, |r|, IF(continue){ z = Pinv r,
// r.z, beta, p update } }.  Vectors: r = w0, z = w1, p = w2, Ap = w8, x = w9.
void build_pcg_graph(Context& c, int precond, double omega) {
  if (c.pcg_exec) {
    cudaGraphExecDestroy(c.pcg_exec);
    c.pcg_exec = nullptr;
  }
  prepare_buffers(c);
  for (Context* s : c.comp) prepare_buffers(*s);
  const bool timing = c.timing;
  c.timing = false;  // no event records inside the captured graph
  c.capturing = true;
  // Capture on a private stream (the handle's stream may be the legacy default
  // stream, which cannot be captured); the graph is launched on c.stream.
  if (!c.cap_stream) FDM_CUDA(cudaStreamCreateWithFlags(&c.cap_stream, cudaStreamNonBlocking));
  FDM_CUDA(cudaStreamSynchronize(c.stream));
  cudaStream_t user_stream = c.stream;
  c.stream = c.cap_stream;
  double* r = c.w[0].p;
  double* z = c.w[1].p;
  double* p = c.w[2].p;
  double* Ap = c.w[8].p;
  double* x = c.w[9].p;
  PcgDev* st = c.pcg_state.p;
  cudaGraph_t g = nullptr, tmp = nullptr;
  FDM_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw, hi;
  FDM_CUDA(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  FDM_CUDA(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  FDM_CUDA(cudaGraphConditionalHandleCreate(&hi, body, 0, 0));
  FDM_CUDA(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  op_A(c, p, Ap);
  launch_dot_partials(c, c.ndof, p, Ap, 0);
  launch_dot_finish(c, 0, &st->pAp);
  launch_pcg_alpha(c, st, c.pcg_alphas.p, hw);
  launch_pcg_update_xr(c, st, p, Ap, x, r);
  launch_dot_partials(c, c.ndof, r, r, 0);
  launch_dot_finish(c, 0, &st->res);
  launch_pcg_residual(c, st, c.pcg_res.p, hw, hi);
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  FDM_CUDA(cudaStreamGetCaptureInfo(c.stream, &cs, nullptr, nullptr, &deps, &nd));
  std::vector<cudaGraphNode_t> dv(deps, deps + nd);
  FDM_CUDA(cudaStreamEndCapture(c.stream, &tmp));
  cudaGraphNodeParams ip = {};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = hi;
  ip.conditional.type = cudaGraphCondTypeIf;
  ip.conditional.size = 1;
  cudaGraphNode_t in;
  FDM_CUDA(cudaGraphAddNode(&in, body, dv.data(), dv.size(), &ip));
  cudaGraph_t ibody = ip.conditional.phGraph_out[0];
  FDM_CUDA(cudaStreamBeginCaptureToGraph(c.stream, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  op_precond(c, precond, omega, r, z);
  launch_dot_partials(c, c.ndof, r, z, 0);
  launch_dot_finish(c, 0, &st->rz_new);
  launch_pcg_beta(c, st, c.pcg_betas.p);
  launch_pcg_update_p(c, st, z, p);
  FDM_CUDA(cudaStreamEndCapture(c.stream, &tmp));
  FDM_CUDA(cudaGraphInstantiate(&c.pcg_exec, g, 0));
  FDM_CUDA(cudaGraphDestroy(g));
  c.timing = timing;
  c.capturing = false;
  c.stream = user_stream;
  c.pcg_precond = precond;
  c.pcg_omega = omega;
}

// pcg (src/krylov.cpp:29-83), device resident: x must not alias b.
void run_pcg(Context& c, const double* b, double* x, double rtol, int maxit, int precond, double omega,
             fdmgpu_krylov_report* rep, std::vector<double>* residuals) {
  const auto t0 = std::chrono::steady_clock::now();
  fdmgpu_krylov_report R{};
  double* r = c.w[0].p;
  double* z = c.w[1].p;
  double* p = c.w[2].p;
  double* xi = c.w[9].p;
  const double bnorm = std::sqrt(host_dot(c, b, b));
  if (residuals) residuals->clear();
  FDM_CUDA(cudaMemsetAsync(xi, 0, c.ndof * sizeof(double), c.stream));
  if (bnorm == 0.0 || maxit <= 0) {
    if (x != xi) FDM_CUDA(cudaMemcpyAsync(x, xi, c.ndof * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    R.converged = bnorm == 0.0;
    R.kappa = bnorm == 0.0 ? 1.0 : 0.0;
    *rep = R;
    return;
  }
  copy_dev(c, r, b);
  op_precond(c, precond, omega, r, z);
  copy_dev(c, p, z);
  const double rz = host_dot(c, r, z);
  if (!c.pcg_state.p) c.pcg_state.alloc(1);
  if (c.pcg_cap < maxit) {
    c.pcg_cap = std::max(maxit, 256);
    c.pcg_alphas.alloc(c.pcg_cap);
    c.pcg_betas.alloc(c.pcg_cap);
    c.pcg_res.alloc(c.pcg_cap);
    c.pcg_precond = -1;  // buffers moved: rebuild
  }
  if (!c.pcg_exec || c.pcg_precond != precond || c.pcg_omega != omega) build_pcg_graph(c, precond, omega);
  pcg_state_init(c, c.pcg_state.p, bnorm, rtol, rz, maxit);
  FDM_CUDA(cudaGraphLaunch(c.pcg_exec, c.stream));
  c.launches += 1;
  int k = 0, status = 0;
  pcg_state_read(c, c.pcg_state.p, &k, &status);
  const int na = status == 2 ? k : k;  // alphas written for iterations 0..k-1 (k on indefinite: none at k)
  std::vector<double> alphas(na), betas(std::max(na - 1, 0)), res(k);
  if (na) FDM_CUDA(cudaMemcpy(alphas.data(), c.pcg_alphas.p, na * sizeof(double), cudaMemcpyDeviceToHost));
  if (na > 1) FDM_CUDA(cudaMemcpy(betas.data(), c.pcg_betas.p, (na - 1) * sizeof(double), cudaMemcpyDeviceToHost));
  if (k) FDM_CUDA(cudaMemcpy(res.data(), c.pcg_res.p, k * sizeof(double), cudaMemcpyDeviceToHost));
  if (status == 2) throw Error(FDMGPU_INDEFINITE, "pcg: indefinite operator at iteration " + std::to_string(k + 1));
  if (x != xi) FDM_CUDA(cudaMemcpyAsync(x, xi, c.ndof * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  FDM_CUDA(cudaStreamSynchronize(c.stream));
  if (residuals) *residuals = res;
  R.iterations = k;
  R.converged = status == 1;
  R.final_residual = k ? res[k - 1] : 0.0;
  std::vector<double> td, to;
  for (size_t i = 0; i < alphas.size(); ++i) {
    double dk = 1.0 / alphas[i];
    if (i > 0) dk += betas[i - 1] / alphas[i - 1];
    td.push_back(dk);
    if (i + 1 < alphas.size()) to.push_back(std::sqrt(betas[i]) / alphas[i]);
  }
  auto [lmin, lmax] = tridiag_extremes(td, to);
  R.lambda_min = lmin;
  R.lambda_max = lmax;
  R.kappa = lmin > 0 ? lmax / lmin : 0.0;
  R.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *rep = R;
}

std::vector<double> random_free(Context& c, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  std::vector<double> b(c.ndof);
  for (auto& v : b) v = uni(rng);
  for (int64_t i = 0; i < c.ndof; ++i)
    if (c.h_constrained[i]) b[i] = 0.0;
  return b;
}

// NVTX range around one public call (visible to ncu --nvtx / nsys when a tool
// is attached; a no-op otherwise).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <class Fn>
fdmgpu_status guarded(fdmgpu_handle h, Fn&& fn) {
  Context* c = reinterpret_cast<Context*>(h);
  if (!c) return FDMGPU_INVALID_ARGUMENT;
  try {
    if (c->device >= 0) cudaSetDevice(c->device);
    fn(*c);
    return FDMGPU_OK;
  } catch (const Error& e) {
    c->err = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    c->err = "host allocation failed";
    return FDMGPU_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    c->err = e.what();
    return FDMGPU_INVALID_ARGUMENT;
  }
}

// Forwards a public call to every component sub-handle; a failure is
// re-thrown with the sub-handle's status and message.
template <class Fn>
void forward(Context& c, Fn&& fn) {
  for (int ci = 0; ci < int(c.comp.size()); ++ci) {
    Context& s = c.sub(ci);
    const fdmgpu_status st = fn(reinterpret_cast<fdmgpu_handle>(&s), ci);
    if (st != FDMGPU_OK) throw Error(st, s.err);
  }
}

}  // namespace
}  // namespace fdmgpu

using fdmgpu::Context;

using fdmgpu::Error;

struct fdmgpu_context : fdmgpu::Context {};

namespace fdmgpu {
void destroy_sub(Context* s) {
  s->stream = nullptr;  // the parent's stream
  s->own_stream = false;
  delete reinterpret_cast<fdmgpu_context*>(s);
}
}  // namespace fdmgpu

extern "C" {

const char* fdmgpu_last_error(fdmgpu_handle h) { return h ? h->err.c_str() : "null handle"; }

const char* fdmgpu_status_string(fdmgpu_status s) {
  switch (s) {
    case FDMGPU_OK: return "ok";
    case FDMGPU_INVALID_ARGUMENT: return "invalid argument";
    case FDMGPU_NOT_SPD: return "matrix not SPD";
    case FDMGPU_INDEFINITE: return "indefinite operator";
    case FDMGPU_OUT_OF_MEMORY: return "out of memory";
    case FDMGPU_CUDA_ERROR: return "CUDA error";
    case FDMGPU_UNSUPPORTED: return "unsupported";
  }
  return "unknown";
}

fdmgpu_status fdmgpu_create(fdmgpu_handle* out, int32_t dim, int32_t p, int32_t ncells, int64_t ndof, int32_t device) {
  if (!out) return FDMGPU_INVALID_ARGUMENT;
  *out = nullptr;
  if ((dim != 2 && dim != 3) || p < 1 || ncells < 1 || ndof < 1) return FDMGPU_INVALID_ARGUMENT;
  auto* c = new fdmgpu_context();
  c->device = device;
  c->dim = dim;
  c->p = p;
  c->n1 = p + 1;
  c->npc = dim == 3 ? c->n1 * c->n1 * c->n1 : c->n1 * c->n1;
  c->ncells = ncells;
  c->ndof = ndof;
  fdmgpu_status st = fdmgpu::guarded(c, [](Context& cc) {
    int n = 0;
    FDM_CUDA(cudaGetDeviceCount(&n));
    if (cc.device < 0 || cc.device >= n) throw Error(FDMGPU_CUDA_ERROR, "no such CUDA device");
    FDM_CUDA(cudaSetDevice(cc.device));
    FDM_CUDA(cudaStreamCreateWithFlags(&cc.stream, cudaStreamNonBlocking));
    cc.own_stream = true;
    const char* pd = std::getenv("FDMGPU_PDL");
    cc.pdl = !(pd && pd[0] == '0');
    const char* fs = std::getenv("FDMGPU_FORCE_STAGED");
    cc.force_staged = fs && fs[0] == '1';
    const char* so = std::getenv("FDMGPU_SEP_ORDER");
    cc.sep_order = (so && std::string(so) == "reference") ? 1 : 0;
    // Separator solve split: the last partial wave of patches runs on clusters
    // of CTAs (FDMGPU_SOLVE_CS=2..4 fixes the size, 1 keeps one CTA per patch;
    // FDMGPU_SOLVE_TAIL=0 splits every patch).
    const char* cs = std::getenv("FDMGPU_SOLVE_CS");
    if (cs && cs[0] >= '1' && cs[0] <= '4' && cs[1] == 0) cc.solve_cs = cs[0] - '0';
    const char* st = std::getenv("FDMGPU_SOLVE_TAIL");
    cc.solve_tail = !(st && st[0] == '0');
    const char* fu = std::getenv("FDMGPU_FUSED");
    cc.fused_columns = !(fu && fu[0] == '0');
    cc.E.alloc(size_t(cc.ncells) * cc.npc);
    for (auto& v : cc.w) {
      v.alloc(cc.ndof);
      FDM_CUDA(cudaMemsetAsync(v.p, 0, v.bytes(), cc.stream));  // finite from the start (see bnd_list)
    }
    cc.red.alloc(4 * fdmgpu::kRedBlocks);
    cc.d_err.alloc(1);
  });
  if (st != FDMGPU_OK) {
    *out = nullptr;
    delete c;
    return st;
  }
  *out = c;
  return FDMGPU_OK;
}

fdmgpu_status fdmgpu_destroy(fdmgpu_handle h) {
  if (!h) return FDMGPU_INVALID_ARGUMENT;
  if (h->device >= 0) cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  cudaStream_t s = h->own_stream ? h->stream : nullptr;
  delete h;
  if (s) cudaStreamDestroy(s);
  return FDMGPU_OK;
}

fdmgpu_status fdmgpu_set_stream(fdmgpu_handle h, void* stream) {
  return fdmgpu::guarded(h, [&](Context& c) {
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    if (c.own_stream) cudaStreamDestroy(c.stream);
    c.stream = static_cast<cudaStream_t>(stream);
    c.own_stream = false;
    for (Context* sc : c.comp) sc->stream = c.stream;
  });
}

/* Linear elasticity (src/elasticity.cpp): turns a fresh handle into a vector
 * handle with dim identical components and the SDC relaxation. */
fdmgpu_status fdmgpu_set_elasticity(fdmgpu_handle h, double mu, double lambda, const double* C) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::invalidate_graph(c);
    if (c.have_maps || !c.comp.empty()) throw Error(FDMGPU_INVALID_ARGUMENT, "set_elasticity: call right after fdmgpu_create");
    if (!C) throw Error(FDMGPU_INVALID_ARGUMENT, "set_elasticity: null C");
    if (!(mu > 0.0) || !(lambda >= 0.0) || std::isinf(lambda))
      throw Error(FDMGPU_INVALID_ARGUMENT, "elasticity_primal_operator: lambda must be finite");
    if (c.ndof % c.dim != 0) throw Error(FDMGPU_INVALID_ARGUMENT, "set_elasticity: ndof must be dim x scalar DOFs");
    c.ncomp = c.dim;
    c.nsc = c.ndof / c.dim;
    c.lame_mu = mu;
    c.lame_lambda = lambda;
    c.Cm.upload(C, size_t(c.n1) * c.n1, c.stream);
    c.E.alloc(size_t(c.ncomp) * c.ncells * c.npc);
    for (int ci = 0; ci < c.ncomp; ++ci) {
      fdmgpu_handle sh = nullptr;
      const fdmgpu_status st = fdmgpu_create(&sh, c.dim, c.p, c.ncells, c.nsc, c.device);
      if (st != FDMGPU_OK) throw Error(st, "set_elasticity: component handle");
      FDM_CUDA(cudaStreamSynchronize(sh->stream));
      cudaStreamDestroy(sh->stream);
      sh->own_stream = false;
      sh->stream = c.stream;
      sh->sep_order = c.sep_order;
      c.comp.push_back(sh);
    }
    FDM_CUDA(cudaStreamSynchronize(c.stream));
  });
}

/* Symmetric interior-penalty DG (src/sipg.cpp): marks a fresh scalar handle
 * as the dq_space SIPG problem -- penalty eta, the FDM modes' derivative
 * traces, the GL nodal traces, the facet list -- before set_patches. */
fdmgpu_status fdmgpu_set_sipg(fdmgpu_handle h, double eta, const double* deriv_traces, const double* trace_values,
                              const double* trace_normal_derivs, int32_t nfacets, const int32_t* facet_cells,
                              const int32_t* facet_axis, const int32_t* facet_sides, const uint8_t* facet_tags,
                              const int32_t* cell_vertices) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::invalidate_graph(c);
    if (c.ncomp > 1 || c.have_patches) throw Error(FDMGPU_INVALID_ARGUMENT, "set_sipg: call on a scalar handle before set_patches");
    if (!deriv_traces || !trace_values || !trace_normal_derivs || nfacets < 0 || (nfacets > 0 && (!facet_cells || !facet_axis || !facet_sides || !facet_tags)) || !cell_vertices)
      throw Error(FDMGPU_INVALID_ARGUMENT, "set_sipg: null array");
    if (!(eta > 0.0)) throw Error(FDMGPU_INVALID_ARGUMENT, "sipg: penalty eta must be positive");
    const int twod = 2 * c.dim, ncorner = 1 << c.dim;
    std::vector<int32_t> nbr(size_t(c.ncells) * twod, -1);
    std::vector<uint8_t> tag(size_t(c.ncells) * twod, 2);  // a facet slot no facet claims: no term
    for (int f = 0; f < nfacets; ++f) {
      const int ax = facet_axis[f];
      if (ax < 0 || ax >= c.dim || facet_tags[f] > 2) throw Error(FDMGPU_INVALID_ARGUMENT, "set_sipg: bad facet");
      if ((facet_cells[2 * f] < 0 || facet_cells[2 * f + 1] < 0) && facet_tags[f] == 0)
        throw Error(FDMGPU_INVALID_ARGUMENT, "set_sipg: boundary facet tagged interior (Mesh::finalize tags them)");
      for (int r = 0; r < 2; ++r) {
        const int K = facet_cells[2 * f + r];
        if (K < 0) continue;
        if (K >= c.ncells) throw Error(FDMGPU_INVALID_ARGUMENT, "set_sipg: facet cell out of range");
        const int slot = 2 * ax + (facet_sides[2 * f + r] > 0 ? 1 : 0);
        nbr[size_t(K) * twod + slot] = facet_cells[2 * f + 1 - r];
        tag[size_t(K) * twod + slot] = facet_cells[2 * f + 1 - r] >= 0 ? 0 : facet_tags[f];
      }
    }
    c.dg = true;
    c.eta = eta;
    const size_t nt = size_t(2) * c.n1;
    c.dtr.upload(deriv_traces, nt, c.stream);
    c.tv.upload(trace_values, nt, c.stream);
    c.tnd.upload(trace_normal_derivs, nt, c.stream);
    c.fnbr.upload(nbr, c.stream);
    c.ftag.upload(tag, c.stream);
    c.h_cell_vertices.assign(cell_vertices, cell_vertices + size_t(c.ncells) * ncorner);
    FDM_CUDA(cudaStreamSynchronize(c.stream));
  });
}

fdmgpu_status fdmgpu_synchronize(fdmgpu_handle h) {
  return fdmgpu::guarded(h, [](Context& c) {
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    if (c.h2d_stream) FDM_CUDA(cudaStreamSynchronize(c.h2d_stream));
    if (c.d2h_stream) FDM_CUDA(cudaStreamSynchronize(c.d2h_stream));
  });
}

fdmgpu_status fdmgpu_set_basis(fdmgpu_handle h, const double* S, const double* lambda, const double* A_t,
                               const double* B_t, const uint8_t* A_t_pattern, const uint8_t* B_t_pattern,
                               const double* A_hat, const double* B_hat, int32_t q, const double* q_points,
                               const double* wq, const double* Vq, const double* Dq) {
  (void)lambda;
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::invalidate_graph(c);
    if (!S || !A_t || !B_t || !A_t_pattern || !B_t_pattern || !A_hat || !B_hat)
      throw Error(FDMGPU_INVALID_ARGUMENT, "set_basis: null array");
    const int n1 = c.n1, nn = n1 * n1;
    std::vector<double> St(nn), At(nn), Bt(nn);
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) St[i + n1 * j] = S[j + n1 * i];
    c.h_Anz.assign(A_t_pattern, A_t_pattern + nn);
    c.h_Bnz.assign(B_t_pattern, B_t_pattern + nn);
    for (int k = 0; k < nn; ++k) {  // values outside the stored pattern are structural zeros
      At[k] = c.h_Anz[k] ? A_t[k] : 0.0;
      Bt[k] = c.h_Bnz[k] ? B_t[k] : 0.0;
    }
    c.h_At = At;
    c.h_Bt = Bt;
    c.S.upload(S, nn, c.stream);
    c.St.upload(St, c.stream);
    c.At.upload(At, c.stream);
    c.Bt.upload(Bt, c.stream);
    c.Ahat.upload(A_hat, nn, c.stream);
    c.Bhat.upload(B_hat, nn, c.stream);
    c.q = q;
    if (q > 0 && Vq && Dq && wq && q_points) {
      c.qpts.upload(q_points, q, c.stream);
      c.Vq.upload(Vq, size_t(q) * n1, c.stream);
      c.Dq.upload(Dq, size_t(q) * n1, c.stream);
      c.wq.upload(wq, q, c.stream);
    }
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    fdmgpu::forward(c, [&](fdmgpu_handle sh, int) {
      return fdmgpu_set_basis(sh, S, lambda, A_t, B_t, A_t_pattern, B_t_pattern, A_hat, B_hat, q, q_points, wq, Vq, Dq);
    });
    c.have_basis = true;
  });
}

fdmgpu_status fdmgpu_set_mesh_maps(fdmgpu_handle h, const int32_t* cell_dofs, const int32_t* cell_modes,
                                   const double* mode_signs, const double* multiplicity, const uint8_t* constrained) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::invalidate_graph(c);
    if (!cell_dofs || !multiplicity || !constrained) throw Error(FDMGPU_INVALID_ARGUMENT, "set_mesh_maps: null array");
    const size_t nm = size_t(c.ncells) * c.npc;
    if (c.ncomp > 1) {
      // Vector handle: component-0 cell maps, per-DOF arrays over all components
      // (identical blocks); each component handle gets the scalar maps.
      if (mode_signs || (cell_modes && !std::equal(cell_dofs, cell_dofs + nm, cell_modes)))
        throw Error(FDMGPU_UNSUPPORTED, "set_mesh_maps: elasticity needs unflipped lattice meshes");
      for (int ci = 1; ci < c.ncomp; ++ci)
        for (int64_t i = 0; i < c.nsc; ++i)
          if (constrained[ci * c.nsc + i] != constrained[i] || multiplicity[ci * c.nsc + i] != multiplicity[i])
            throw Error(FDMGPU_INVALID_ARGUMENT, "set_mesh_maps: components must share one scalar space");
      for (size_t k = 0; k < nm; ++k)
        if (cell_dofs[k] < 0 || cell_dofs[k] >= c.nsc) throw Error(FDMGPU_INVALID_ARGUMENT, "set_mesh_maps: DOF out of range");
      c.h_cell_dofs.assign(cell_dofs, cell_dofs + nm);
      c.h_cell_modes = c.h_cell_dofs;
      c.h_constrained.assign(constrained, constrained + c.ndof);
      std::vector<double> inv(c.ndof);
      for (int64_t i = 0; i < c.ndof; ++i) {
        if (!(multiplicity[i] > 0)) throw Error(FDMGPU_INVALID_ARGUMENT, "set_mesh_maps: multiplicity must be > 0");
        inv[i] = 1.0 / multiplicity[i];
      }
      c.cell_dofs.upload(c.h_cell_dofs, c.stream);
      c.cell_modes.upload(c.h_cell_dofs, c.stream);
      c.inv_mult.upload(inv, c.stream);
      c.constrained.upload(c.h_constrained, c.stream);
      FDM_CUDA(cudaStreamSynchronize(c.stream));
      fdmgpu::forward(c, [&](fdmgpu_handle sh, int) {
        return fdmgpu_set_mesh_maps(sh, cell_dofs, nullptr, nullptr, multiplicity, constrained);
      });
      c.have_maps = true;
      return;
    }
    c.h_cell_dofs.assign(cell_dofs, cell_dofs + nm);
    c.h_cell_modes.assign(cell_modes ? cell_modes : cell_dofs, (cell_modes ? cell_modes : cell_dofs) + nm);
    c.modes_alias = c.h_cell_modes == c.h_cell_dofs;
    c.h_constrained.assign(constrained, constrained + c.ndof);
    std::vector<double> inv(c.ndof);
    for (int64_t i = 0; i < c.ndof; ++i) {
      if (!(multiplicity[i] > 0)) throw Error(FDMGPU_INVALID_ARGUMENT, "set_mesh_maps: multiplicity must be > 0");
      inv[i] = 1.0 / multiplicity[i];
    }
    std::vector<int32_t> ptr, idx;
    fdmgpu::build_gather(c.h_cell_dofs, c.ndof, ptr, idx);
    c.cell_dofs.upload(c.h_cell_dofs, c.stream);
    c.g_ptr.upload(ptr, c.stream);
    c.g_idx.upload(idx, c.stream);
    if (!c.modes_alias) {
      fdmgpu::build_gather(c.h_cell_modes, c.ndof, ptr, idx);
      c.cell_modes.upload(c.h_cell_modes, c.stream);
      c.gm_ptr.upload(ptr, c.stream);
      c.gm_idx.upload(idx, c.stream);
    } else {
      c.cell_modes.upload(c.h_cell_dofs, c.stream);
    }
    bool unit = true;
    if (mode_signs)
      for (size_t k = 0; k < nm; ++k) unit = unit && mode_signs[k] == 1.0;
    if (!unit)
      c.mode_sign.upload(mode_signs, nm, c.stream);
    else
      c.mode_sign.reset();
    c.inv_mult.upload(inv, c.stream);
    c.constrained.upload(c.h_constrained, c.stream);
    {  // cell-boundary modal DOFs: positions with a lattice coordinate 0 or p in some cell
      std::vector<uint8_t> on(c.ndof, 0);
      const int n1 = c.n1;
      for (int k = 0; k < c.ncells; ++k)
        for (int l = 0; l < c.npc; ++l) {
          bool bnd = false;
          for (int a = 0, r = l; a < c.dim; ++a, r /= n1) bnd = bnd || r % n1 == 0 || r % n1 == n1 - 1;
          if (bnd) on[c.h_cell_modes[size_t(k) * c.npc + l]] = 1;
        }
      std::vector<int32_t> list;
      for (int64_t g = 0; g < c.ndof; ++g)
        if (on[g]) list.push_back(int32_t(g));
      c.bnd_list.upload(list, c.stream);
    }
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    c.have_maps = true;
  });
}

fdmgpu_status fdmgpu_set_cell_coeffs(fdmgpu_handle h, const uint8_t* kind, const double* mu, const double* xyz,
                                     const double* kappa) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::invalidate_graph(c);
    if (!kind || !mu) throw Error(FDMGPU_INVALID_ARGUMENT, "set_cell_coeffs: null array");
    if (c.ncomp > 1) {
      // elasticity_primal_operator's Kronecker path (src/elasticity.cpp:83-119):
      // Cartesian cells, no kappa; component ci's SDC coefficients are
      // sdc_axis_coefficients(ci) * mu^K (src/elasticity.cpp:141-151).
      for (int k = 0; k < c.ncells; ++k)
        if (kind[k] != 0) throw Error(FDMGPU_UNSUPPORTED, "elasticity: non-Cartesian cells need the dense quadrature form");
      if (kappa)
        for (int k = 0; k < c.ncells; ++k)
          if (kappa[k] != 1.0) throw Error(FDMGPU_INVALID_ARGUMENT, "elasticity: per-cell kappa is not part of the operator");
      c.all_cartesian = true;
      c.kind.upload(kind, c.ncells, c.stream);
      c.h_mu.assign(mu, mu + size_t(c.ncells) * c.dim);
      c.mu.upload(c.h_mu, c.stream);
      FDM_CUDA(cudaStreamSynchronize(c.stream));
      fdmgpu::forward(c, [&](fdmgpu_handle sh, int ci) {
        std::vector<double> m(c.h_mu.size());
        for (int k = 0; k < c.ncells; ++k)
          for (int a = 0; a < c.dim; ++a) {
            const double coeff = c.lame_mu + (a == ci ? c.lame_mu + c.lame_lambda : 0.0);
            m[size_t(k) * c.dim + a] = coeff * c.h_mu[size_t(k) * c.dim + a];
          }
        return fdmgpu_set_cell_coeffs(sh, kind, m.data(), xyz, nullptr);
      });
      c.have_coeffs = true;
      c.factored = false;
      return;
    }
    c.all_cartesian = true;
    for (int k = 0; k < c.ncells; ++k) c.all_cartesian = c.all_cartesian && kind[k] == 0;
    if (!c.all_cartesian && !xyz)
      throw Error(FDMGPU_INVALID_ARGUMENT, "set_cell_coeffs: non-Cartesian cells need corner coordinates");
    c.kind.upload(kind, c.ncells, c.stream);
    c.h_mu.assign(mu, mu + size_t(c.ncells) * c.dim);
    c.mu.upload(c.h_mu, c.stream);
    if (xyz) c.xyz.upload(xyz, size_t(c.ncells) * (1 << c.dim) * 3, c.stream);
    std::vector<double> kap(c.ncells, 1.0);
    if (kappa) kap.assign(kappa, kappa + c.ncells);
    c.kappa.upload(kap, c.stream);
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    c.have_coeffs = true;
    c.factored = false;
  });
}

fdmgpu_status fdmgpu_set_patches(fdmgpu_handle h, int32_t npatch, const int32_t* vertex, const int64_t* ptr,
                                 const int32_t* dofs, const int32_t* perm, const int32_t* star_cells) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::invalidate_graph(c);
    fdmgpu::NvtxRange nvtx_("fdmgpu_set_patches");
    c.check_ready(false, false, false);
    if (npatch < 1 || !vertex || !ptr || !dofs || !perm || !star_cells)
      throw Error(FDMGPU_INVALID_ARGUMENT, "set_patches: bad arguments");
    if (c.ncomp > 1) {
      // Vector stars (star_dofs over all components, src/discretization.cpp:
      // 266-297): the SDC patch matrix is block diagonal over components, so
      // component ci solves its own star with the order patch_ordering gives
      // its DOFs inside the vector order.
      std::vector<std::vector<int64_t>> cptr(c.ncomp, std::vector<int64_t>(1, 0));
      std::vector<std::vector<int32_t>> cdofs(c.ncomp), cperm(c.ncomp);
      std::vector<int32_t> local;
      for (int j = 0; j < npatch; ++j) {
        const int64_t b = ptr[j], e = ptr[j + 1];
        local.assign(size_t(e - b), -1);
        std::vector<int32_t> cnt(c.ncomp, 0);
        for (int64_t k = b; k < e; ++k) {
          const int32_t g = dofs[k];
          if (g < 0 || g >= c.ndof) throw Error(FDMGPU_INVALID_ARGUMENT, "set_patches: DOF out of range");
          const int ci = int(g / c.nsc);
          local[k - b] = cnt[ci]++;
          cdofs[ci].push_back(int32_t(g - ci * c.nsc));
        }
        for (int64_t k = b; k < e; ++k) {
          const int32_t q = perm[k];
          if (q < 0 || q >= e - b) throw Error(FDMGPU_INVALID_ARGUMENT, "set_patches: bad permutation");
          cperm[int(dofs[b + q] / c.nsc)].push_back(local[q]);
        }
        for (int ci = 0; ci < c.ncomp; ++ci) cptr[ci].push_back(int64_t(cdofs[ci].size()));
      }
      fdmgpu::forward(c, [&](fdmgpu_handle sh, int ci) {
        sh->sep_order = c.sep_order;
        return fdmgpu_set_patches(sh, npatch, vertex, cptr[ci].data(), cdofs[ci].data(), cperm[ci].data(), star_cells);
      });
      c.npatch = npatch;
      c.have_patches = true;
      c.factored = false;
      return;
    }
    if (c.mode_sign.p || !c.modes_alias)
      throw Error(FDMGPU_UNSUPPORTED, "set_patches: facet mode flips (2D non-lattice meshes) are not supported");
    if (c.dg)
      fdmgpu::analyze_dg_patches(c, npatch, vertex, ptr, dofs, perm, star_cells);
    else
      fdmgpu::analyze_patches(c, npatch, vertex, ptr, dofs, perm, star_cells);
    c.npatch = npatch;
    // split-tail solve state belongs to the previous tile pattern / patch count
    c.cl_cs = 0;
    for (int& f : c.cl_fit) f = -1;
    c.tail_sync.reset();
    const auto& L = c.L;
    const size_t tile_bytes = size_t(npatch) * L.ntiles * fdmgpu::kTile * fdmgpu::kTile * sizeof(double);
    size_t free_b = 0, total_b = 0;
    FDM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (tile_bytes + size_t(npatch) * L.n * 12 > free_b)
      throw Error(FDMGPU_OUT_OF_MEMORY, "set_patches: factor needs " + std::to_string(tile_bytes >> 20) +
                                            " MiB, free " + std::to_string(free_b >> 20) + " MiB");
    // separator DOFs per patch (elimination positions n_I..n-1) and n_K per cell
    const int m = L.m;
    std::vector<int32_t> sep(size_t(npatch) * m);
    std::vector<double> nK(c.ncells, 0.0);
    for (int j = 0; j < npatch; ++j) {
      std::copy(c.h_pdofs.begin() + size_t(j) * L.n + L.nI, c.h_pdofs.begin() + size_t(j + 1) * L.n,
                sep.begin() + size_t(j) * m);
      for (int k = 0; k < (1 << c.dim); ++k) {
        const int K = c.h_pcells[size_t(j) * (1 << c.dim) + k];
        if (K >= 0) nK[K] += 1.0;
      }
    }
    c.pdofs.upload(sep, c.stream);
    c.nK.upload(nK, c.stream);
    c.lat.upload(L.lat, c.stream);
    c.pos_of_lat.upload(L.pos_of_lat, c.stream);
    c.pcells.upload(c.h_pcells, c.stream);
    c.tile_row.upload(L.tile_row, c.stream);
    c.tile_col.upload(L.tile_col, c.stream);
    c.col_start.upload(L.col_start, c.stream);
    c.pair_ptr.upload(L.pair_ptr, c.stream);
    c.entries.upload(L.entries, c.stream);
    c.tile_mask.upload(L.tile_mask, c.stream);
    c.tile_mask8.upload(L.tile_mask8, c.stream);
    c.tile_poff8.upload(L.tile_poff8, c.stream);
    c.tile_hdr.upload(L.tile_hdr, c.stream);
    c.tile_bptr.upload(L.tile_bptr, c.stream);
    c.tile_blk.upload(L.tile_blk, c.stream);
    c.tile_ccol.upload(L.tile_ccol, c.stream);
    c.lead_diag.upload(L.lead_diag, c.stream);
    c.lead_trsm.upload(L.lead_trsm, c.stream);
    c.active.upload(L.active, c.stream);
    if (L.pair_a.empty()) {
      c.pair_a.alloc(1);
      c.pair_b.alloc(1);
    } else {
      c.pair_a.upload(L.pair_a, c.stream);
      c.pair_b.upload(L.pair_b, c.stream);
    }
    std::vector<int32_t> pptr, pidx;
    fdmgpu::build_gather(sep, c.ndof, pptr, pidx, true);  // ascending (patch, position) per separator DOF
    c.pg_ptr.upload(pptr, c.stream);
    c.pg_idx.upload(pidx, c.stream);
    c.corr.alloc(size_t(npatch) * m);
    c.fac_flag.alloc(size_t(npatch) * L.nT);
    FDM_CUDA(cudaMemsetAsync(c.fac_flag.p, 0, c.fac_flag.bytes(), c.stream));
    c.fac_epoch = 0;
    // Separate solve-record buffer when it takes under a quarter of the free
    // memory (C3: 3.7 GB; packing then overlaps the factorisation, 24.3 -> 23.8 ms);
    // else (C5: 63.5 GB) the records are packed in place after the factorisation.
    // FDMGPU_PACK=inplace forces the latter.
    c.packed.reset();
    c.tiles.reset();
    fdmgpu::setup_schur_split(c);
    // the full separator factor tiles; not needed when the split forms its top block directly
    if (!(c.sx.on && c.sx.direct)) c.tiles.alloc(size_t(npatch) * L.ntiles * fdmgpu::kTile * fdmgpu::kTile);
    if (!c.sx.on) {
      const char* pk = std::getenv("FDMGPU_PACK");
      const size_t rec_bytes = size_t(npatch) * size_t(L.tile_poff8.back()) * sizeof(double);
      size_t fb = 0, tb = 0;
      FDM_CUDA(cudaMemGetInfo(&fb, &tb));
      if (!(pk && std::string(pk) == "inplace") && 4 * rec_bytes < fb) c.packed.alloc(rec_bytes / sizeof(double));
    }
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    c.have_patches = true;
    c.factored = false;
  });
}

fdmgpu_status fdmgpu_set_coarse(fdmgpu_handle h, int32_t ndof_c, const double* cinv, const int64_t* P_ptr,
                                const int32_t* P_col, const double* P_val) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::invalidate_graph(c);
    if (ndof_c < 1 || !cinv || !P_ptr) throw Error(FDMGPU_INVALID_ARGUMENT, "set_coarse: bad args");
    const int64_t nnz = P_ptr[c.ndof];  // 0 when every coarse DOF is constrained
    if (nnz > 0 && (!P_col || !P_val)) throw Error(FDMGPU_INVALID_ARGUMENT, "set_coarse: bad args");
    c.nc = ndof_c;
    c.cinv.upload(cinv, size_t(ndof_c) * ndof_c, c.stream);
    std::vector<int32_t> ptr(c.ndof + 1), tptr(ndof_c + 1, 0), tcol(nnz);
    std::vector<double> tval(nnz);
    for (int64_t i = 0; i <= c.ndof; ++i) ptr[i] = int32_t(P_ptr[i]);
    for (int64_t qq = 0; qq < nnz; ++qq) ++tptr[P_col[qq] + 1];
    for (int i = 0; i < ndof_c; ++i) tptr[i + 1] += tptr[i];
    std::vector<int32_t> pos(tptr.begin(), tptr.end() - 1);
    for (int64_t i = 0; i < c.ndof; ++i)
      for (int64_t qq = P_ptr[i]; qq < P_ptr[i + 1]; ++qq) {
        tcol[pos[P_col[qq]]] = int32_t(i);
        tval[pos[P_col[qq]]++] = P_val[qq];
      }
    c.P_ptr.upload(ptr, c.stream);
    c.P_col.upload(P_col, nnz, c.stream);
    c.P_val.upload(P_val, nnz, c.stream);
    c.PT_ptr.upload(tptr, c.stream);
    c.PT_col.upload(tcol, c.stream);
    c.PT_val.upload(tval, c.stream);
    c.rc.alloc(ndof_c);
    c.zc.alloc(ndof_c);
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    c.have_coarse = true;
  });
}

fdmgpu_status fdmgpu_set_coarse_cells(fdmgpu_handle h, const int32_t* coarse_cell_dofs,
                                      const uint8_t* coarse_constrained, const double* phat) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::invalidate_graph(c);
    if (!c.have_coarse || !c.have_maps) throw Error(FDMGPU_INVALID_ARGUMENT, "set_coarse_cells: set maps and coarse first");
    if (!coarse_cell_dofs || !coarse_constrained || !phat)
      throw Error(FDMGPU_INVALID_ARGUMENT, "set_coarse_cells: null array");
    if (c.ncomp > 1) {
      // Vector Q1 coarse space: component blocks of nc / ncomp coarse DOFs,
      // prolongation per component (build_prolongation, src/schwarz.cpp:145-158).
      if (c.nc % c.ncomp) throw Error(FDMGPU_INVALID_ARGUMENT, "set_coarse_cells: coarse ndof must be ncomp x scalar");
      c.ncs = c.nc / c.ncomp;
      fdmgpu::forward(c, [&](fdmgpu_handle sh, int) {
        sh->nc = c.ncs;
        sh->have_coarse = true;  // transfer data only: the coarse solve stays on the vector handle
        return fdmgpu_set_coarse_cells(sh, coarse_cell_dofs, coarse_constrained, phat);
      });
      const char* tr = std::getenv("FDMGPU_TRANSFER");
      c.have_coarse_cells = !(tr && std::string(tr) == "csr");
      return;
    }
    const int ncorner = 1 << c.dim;
    const size_t nslots = size_t(c.ncells) * ncorner;
    // coarse gather: per free coarse DOF its (cell, corner) slots, ascending
    std::vector<int32_t> cptr(c.nc + 1, 0), cidx;
    for (size_t e = 0; e < nslots; ++e) {
      const int j = coarse_cell_dofs[e];
      if (j < 0 || j >= c.nc) throw Error(FDMGPU_INVALID_ARGUMENT, "set_coarse_cells: coarse DOF out of range");
      if (!coarse_constrained[j]) ++cptr[j + 1];
    }
    for (int j = 0; j < c.nc; ++j) cptr[j + 1] += cptr[j];
    cidx.resize(cptr[c.nc]);
    std::vector<int32_t> pos(cptr.begin(), cptr.end() - 1);
    for (size_t e = 0; e < nslots; ++e) {
      const int j = coarse_cell_dofs[e];
      if (!coarse_constrained[j]) cidx[pos[j]++] = int32_t(e);
    }
    // prolongation owner: the first (lowest) cell holding a free fine DOF writes it
    std::vector<uint8_t> owner(size_t(c.ncells) * c.npc, 0), seen(size_t(c.ndof), 0);
    for (size_t e = 0; e < owner.size(); ++e) {
      const int g = c.h_cell_dofs[e];
      if (!c.h_constrained[g] && !seen[g]) {
        seen[g] = 1;
        owner[e] = 1;
      }
    }
    std::vector<int32_t> ccd(coarse_cell_dofs, coarse_cell_dofs + nslots);
    for (size_t e = 0; e < nslots; ++e)
      if (coarse_constrained[ccd[e]]) ccd[e] = -1;  // constrained coarse DOFs carry no prolongation
    c.ccd.upload(ccd, c.stream);
    c.cg_ptr.upload(cptr, c.stream);
    c.cg_idx.upload(cidx, c.stream);
    c.powner.upload(owner, c.stream);
    c.phat.upload(phat, size_t(c.n1) * 2, c.stream);
    c.cellsum.alloc(nslots);
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    const char* tr = std::getenv("FDMGPU_TRANSFER");  // "csr": keep the CSR transfer (tests)
    c.have_coarse_cells = !(tr && std::string(tr) == "csr");
  });
}

fdmgpu_status fdmgpu_factor(fdmgpu_handle h) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::NvtxRange nvtx_("fdmgpu_factor");
    c.check_ready(true, false, false);
    if (c.ncomp > 1) {
      c.factored = false;
      fdmgpu::forward(c, [](fdmgpu_handle sh, int) { return fdmgpu_factor(sh); });
      c.factored = true;
      return;
    }
    const unsigned long long none = ~0ULL;
    FDM_CUDA(cudaMemcpyAsync(c.d_err.p, &none, sizeof(none), cudaMemcpyHostToDevice, c.stream));
    const bool direct = c.sx.on && c.sx.direct;  // top block formed directly: no full separator factor
    if (direct) {
      fdmgpu::launch_schur_setup(c);
      ++c.fac_epoch;
      fdmgpu::launch_schur_direct(c);
    } else {
    if (c.dg)
      fdmgpu::launch_dg_patch_assemble(c);
    else
      fdmgpu::launch_patch_assemble(c);
    fdmgpu::launch_schur_setup(c);  // no-op without the Schur split
    fdmgpu::launch_patch_lead(c);
    for (int K = 0; K < c.L.lead_cols; ++K) fdmgpu::launch_patch_pack_col(c, K);
    ++c.fac_epoch;
    for (int K = c.L.lead_cols; K < c.L.nT; ++K) {
      if (c.fused_columns) {
        fdmgpu::launch_patch_column(c, K);
      } else {
        fdmgpu::launch_patch_update(c, K);
        fdmgpu::launch_patch_trsm(c, K);
      }
      fdmgpu::launch_patch_pack_col(c, K);  // no-op when packing in place
    }
    if (c.sx.on)
      fdmgpu::launch_schur_retile(c);  // L_RR -> dense records; the full tiles stay intact
    else if (c.packed.p)
      fdmgpu::launch_patch_pack_join(c);
    else
      fdmgpu::launch_patch_pack(c);  // dense tiles -> packed 8x8 sub-block records, in place
    }
    unsigned long long e = 0;
    FDM_CUDA(cudaMemcpyAsync(&e, c.d_err.p, sizeof(e), cudaMemcpyDeviceToHost, c.stream));
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    c.factored = false;
    if (e != none)
      throw Error(FDMGPU_NOT_SPD, "cholesky: matrix not SPD at pivot " + std::to_string(e & 0xffffffffULL) +
                                      " (patch " + std::to_string(e >> 32) + ")");
    c.factored = true;
  });
}

fdmgpu_status fdmgpu_get_layout(fdmgpu_handle h, fdmgpu_layout* out) {
  return fdmgpu::guarded(h, [&](Context& c) {
    c.check_ready(true, false, false);
    if (c.ncomp > 1) {  // per-component layout; byte totals over all components
      fdmgpu_layout L{};
      fdmgpu::forward(c, [&](fdmgpu_handle sh, int ci) {
        fdmgpu_layout Li{};
        const fdmgpu_status st = fdmgpu_get_layout(sh, &Li);
        if (ci == 0)
          L = Li;
        else {
          L.factor_bytes += Li.factor_bytes;
          L.stream_bytes += Li.stream_bytes;
        }
        return st;
      });
      *out = L;
      return;
    }
    fdmgpu_layout L{};
    L.npatch = c.npatch;
    L.n = c.L.n;
    L.n_interior = c.L.nI;
    L.n_interface = c.L.m;
    L.tile = fdmgpu::kTile;
    L.tile_cols = c.L.nT;
    L.tiles = c.L.ntiles;
    L.nnz_L = c.L.nnz_L;
    L.flops_ref = c.L.flops_ref;
    L.factor_bytes = int64_t(c.tiles.bytes());
    L.top_direct = (c.sx.on && c.sx.direct) ? 1 : 0;
    if (L.top_direct) L.factor_bytes = int64_t(c.packed.bytes() + c.sx_UT.bytes() + c.sx_inv.bytes() + c.sx_fv.bytes());
    L.tile_gemms = c.L.tile_gemms;
    L.nnz_L_reference = c.L.nnz_L_reference;
    L.flops_reference = c.L.flops_reference;
    L.separator_order = c.sep_order;
    L.dmma_flops = c.L.dmma_flops;
    const auto& S = c.sx;
    if (S.on) {
      L.stream_bytes = int64_t(S.R.tile_poff8.back()) * 8 * c.npatch;
      L.schur_split = S.inv ? 2 : 1;
      L.n_top = S.nR;
      int64_t comp = 0;
      for (int k = 0; k < S.ncomp; ++k) {
        int64_t a0 = 0, a1 = 0;
        for (int i = 0; i < S.c0; ++i) a0 += S.comp0[size_t(k) * S.c0 + i] >= 0;
        for (int i = 0; i < S.c1; ++i) a1 += S.comp1[size_t(k) * S.c1 + i] >= 0;
        comp += a1 * a0 + a1 * (a1 + 1) / 2 + a0;
      }
      L.solve_values = (S.inv ? 1 : 2) * S.R.nnz_L + 2 * comp + S.rf_nnz + S.fr_nnz;
    } else {
      L.stream_bytes = int64_t(c.L.tile_poff8.back()) * 8 * c.npatch;
      L.schur_split = 0;
      L.n_top = 0;
      L.solve_values = 2 * (c.L.nnz_L - int64_t(c.dim + 1) * c.L.nI);
    }
    *out = L;
  });
}

fdmgpu_status fdmgpu_patch_schur(fdmgpu_handle h, int32_t j, double* out) {
  return fdmgpu::guarded(h, [&](Context& c) {
    c.check_ready(true, false, false);
    if (c.ncomp > 1 || c.dg) throw Error(FDMGPU_UNSUPPORTED, "patch_schur: scalar CG handles only");
    if (j < 0 || j >= c.npatch || !out) throw Error(FDMGPU_INVALID_ARGUMENT, "patch_schur: bad patch index");
    const auto& L = c.L;
    const size_t tt = size_t(fdmgpu::kTile) * fdmgpu::kTile;
    fdmgpu::DevArray<double> scratch;
    scratch.alloc(size_t(L.ntiles) * tt);
    fdmgpu::launch_patch_assemble_one(c, j, scratch.p);
    std::vector<double> h_t(scratch.n);
    FDM_CUDA(cudaMemcpyAsync(h_t.data(), scratch.p, scratch.bytes(), cudaMemcpyDeviceToHost, c.stream));
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    const int m = L.m, T = fdmgpu::kTile;
    std::fill(out, out + size_t(m) * m, 0.0);
    for (int t = 0; t < L.ntiles; ++t)
      for (int cc = 0; cc < T; ++cc)
        for (int rr = 0; rr < T; ++rr) {
          const int r = L.tile_row[t] * T + rr, col = L.tile_col[t] * T + cc;
          if (r >= m || col >= m || col > r) continue;
          const int swz = ((cc & 3) << 2) | ((cc >> 2) & 3);  // tile swizzle (kernels/common.cuh tsw)
          const double v = h_t[size_t(t) * tt + size_t(cc) * T + (rr ^ swz)];
          out[size_t(col) * m + r] = v;
          out[size_t(r) * m + col] = v;
        }
  });
}

fdmgpu_status fdmgpu_patch_solve_one(fdmgpu_handle h, int32_t j, const double* rhs, double* out) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::NvtxRange nvtx_("fdmgpu_patch_solve_one");
    c.check_ready(true, true, false);
    if (c.ncomp > 1 || c.dg) throw Error(FDMGPU_UNSUPPORTED, "patch_solve_one: scalar CG handles only");
    if (j < 0 || j >= c.npatch || !rhs || !out) throw Error(FDMGPU_INVALID_ARGUMENT, "patch_solve_one: bad arguments");
    const int n = c.L.n, ncorner = 1 << c.dim;
    std::vector<int32_t> dofs;
    for (int k = 0; k < n; ++k)
      if (c.h_pdofs[size_t(j) * n + k] >= 0) dofs.push_back(c.h_pdofs[size_t(j) * n + k]);
    std::sort(dofs.begin(), dofs.end());  // star_dofs order (ascending global ids)
    std::vector<double> r(c.ndof, 0.0);
    for (size_t k = 0; k < dofs.size(); ++k) r[dofs[k]] = rhs[k];
    // only patch j's cells carry its interior block
    std::vector<double> ind(c.ncells, 0.0);
    for (int k = 0; k < ncorner; ++k) {
      const int K = c.h_pcells[size_t(j) * ncorner + k];
      if (K >= 0) ind[K] = 1.0;
    }
    fdmgpu::DevArray<double> nk1;
    nk1.upload(ind, c.stream);
    double* rin = c.w[9].p;
    double* zout = c.w[10].p;
    FDM_CUDA(cudaMemcpyAsync(rin, r.data(), c.ndof * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    // PatchSolver::apply restricted to patch j: every patch solves, then all
    // corrections but patch j's are dropped before the patch sum
    fdmgpu::launch_cells_schur(c, rin);
    fdmgpu::launch_gather(c, 3, c.E.p, rin, c.w[6].p);
    fdmgpu::launch_patch_solve(c, c.w[6].p);
    const size_t m = size_t(c.L.m);
    if (j > 0) FDM_CUDA(cudaMemsetAsync(c.corr.p, 0, size_t(j) * m * sizeof(double), c.stream));
    if (j + 1 < c.npatch)
      FDM_CUDA(cudaMemsetAsync(c.corr.p + size_t(j + 1) * m, 0, size_t(c.npatch - j - 1) * m * sizeof(double), c.stream));
    fdmgpu::launch_patch_gather(c, zout);
    std::swap(c.nK.p, nk1.p);
    std::swap(c.nK.n, nk1.n);
    try {
      fdmgpu::launch_cells_recon(c, zout, rin);
      FDM_CUDA(cudaStreamSynchronize(c.stream));
    } catch (...) {
      std::swap(c.nK.p, nk1.p);
      std::swap(c.nK.n, nk1.n);
      throw;
    }
    std::swap(c.nK.p, nk1.p);
    std::swap(c.nK.n, nk1.n);
    std::vector<double> z(c.ndof);
    FDM_CUDA(cudaMemcpy(z.data(), zout, c.ndof * sizeof(double), cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < dofs.size(); ++k) out[k] = z[dofs[k]];
  });
}

fdmgpu_status fdmgpu_patch_factor(fdmgpu_handle h, int32_t j, double* out) {
  return fdmgpu::guarded(h, [&](Context& c) {
    c.check_ready(true, true, false);
    if (c.ncomp > 1) throw Error(FDMGPU_UNSUPPORTED, "patch_factor: scalar handles only");
    if (j < 0 || j >= c.npatch || !out) throw Error(FDMGPU_INVALID_ARGUMENT, "patch_factor: bad patch index");
    if (!c.packed.p)
      throw Error(FDMGPU_UNSUPPORTED, "patch_factor: the dense factor tiles were packed in place (large factor)");
    if (!c.tiles.p)
      throw Error(FDMGPU_UNSUPPORTED, "patch_factor: the top block is formed directly, the full separator factor does "
                                      "not exist (FDMGPU_DIRECT=0 keeps it)");
    const auto& L = c.L;
    const int T = fdmgpu::kTile, m = L.m;
    const size_t tt = size_t(T) * T;
    std::vector<double> h_t(size_t(L.ntiles) * tt);
    FDM_CUDA(cudaMemcpyAsync(h_t.data(), c.tiles.p + size_t(j) * L.ntiles * tt, h_t.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, c.stream));
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    std::fill(out, out + size_t(m) * m, 0.0);
    std::vector<double> W(tt), Ld(tt);
    for (int t = 0; t < L.ntiles; ++t) {
      for (int cc = 0; cc < T; ++cc)
        for (int rr = 0; rr < T; ++rr) {
          const int swz = ((cc & 3) << 2) | ((cc >> 2) & 3);  // tile swizzle (kernels/common.cuh tsw)
          W[size_t(cc) * T + rr] = h_t[size_t(t) * tt + size_t(cc) * T + (rr ^ swz)];
        }
      if (L.tile_row[t] == L.tile_col[t]) {  // stored L_KK^{-1} (lower): invert back to L_KK
        std::fill(Ld.begin(), Ld.end(), 0.0);
        for (int col = 0; col < T; ++col) {
          // solve W x = e_col (W lower triangular), x = column col of L_KK
          for (int r = col; r < T; ++r) {
            double v = r == col ? 1.0 : 0.0;
            for (int k = col; k < r; ++k) v -= W[size_t(k) * T + r] * Ld[size_t(col) * T + k];
            Ld[size_t(col) * T + r] = v / W[size_t(r) * T + r];
          }
        }
        W = Ld;
      }
      for (int cc = 0; cc < T; ++cc)
        for (int rr = 0; rr < T; ++rr) {
          const int r = L.tile_row[t] * T + rr, col = L.tile_col[t] * T + cc;
          if (r < m && col < m && r >= col) out[size_t(col) * m + r] = W[size_t(cc) * T + rr];
        }
    }
  });
}

fdmgpu_status fdmgpu_get_patch_elimination_dofs(fdmgpu_handle h, int32_t* out) {
  return fdmgpu::guarded(h, [&](Context& c) {
    c.check_ready(true, false, false);
    if (c.ncomp > 1) throw Error(FDMGPU_UNSUPPORTED, "patch elimination dofs: scalar handles only");
    std::memcpy(out, c.h_pdofs.data(), c.h_pdofs.size() * sizeof(int32_t));
  });
}

fdmgpu_status fdmgpu_apply(fdmgpu_handle h, int32_t op, double omega, const double* in, double* out, int32_t host) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::NvtxRange nvtx_("fdmgpu_apply");
    if (!in || !out) throw Error(FDMGPU_INVALID_ARGUMENT, "apply: null vector");
    const bool needs_factor = op == FDMGPU_OP_PATCH || op == FDMGPU_OP_SMOOTH || op == FDMGPU_OP_VCYCLE;
    c.check_ready(needs_factor, needs_factor, op == FDMGPU_OP_VCYCLE);
    const double* din = in;
    double* dout = out;
    const size_t bytes = c.ndof * sizeof(double);
    if (host) {
      FDM_CUDA(cudaMemcpyAsync(c.w[9].p, in, bytes, cudaMemcpyHostToDevice, c.stream));
      din = c.w[9].p;
      dout = c.w[10].p;
    } else if (in == out) {
      throw Error(FDMGPU_INVALID_ARGUMENT, "apply: in and out must not alias");
    }
    switch (op) {
      case FDMGPU_OP_APPLY_ST: fdmgpu::op_transform(c, 0, din, dout); break;
      case FDMGPU_OP_APPLY_S: fdmgpu::op_transform(c, 1, din, dout); break;
      case FDMGPU_OP_PATCH: fdmgpu::op_patch(c, din, dout); break;
      case FDMGPU_OP_SMOOTH: fdmgpu::op_smooth(c, din, dout); break;
      case FDMGPU_OP_A: fdmgpu::op_A(c, din, dout); break;
      case FDMGPU_OP_VCYCLE: fdmgpu::op_vcycle(c, omega, din, dout); break;
      default: throw Error(FDMGPU_INVALID_ARGUMENT, "apply: unknown operator id");
    }
    if (host) {
      FDM_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, c.stream));
      FDM_CUDA(cudaStreamSynchronize(c.stream));
    }
  });
}

fdmgpu_status fdmgpu_apply_async(fdmgpu_handle h, int32_t op, double omega, const double* host_in, double* host_out) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::NvtxRange nvtx_("fdmgpu_apply_async");
    if (!host_in || !host_out) throw Error(FDMGPU_INVALID_ARGUMENT, "apply_async: null vector");
    const bool needs_factor = op == FDMGPU_OP_PATCH || op == FDMGPU_OP_SMOOTH || op == FDMGPU_OP_VCYCLE;
    c.check_ready(needs_factor, needs_factor, op == FDMGPU_OP_VCYCLE);
    if (op < FDMGPU_OP_APPLY_ST || op > FDMGPU_OP_VCYCLE) throw Error(FDMGPU_INVALID_ARGUMENT, "apply: unknown operator id");
    if (!c.async_ready) {
      // all-or-nothing setup: a failure part way leaves nothing half-initialised
      try {
        if (!c.h2d_stream) FDM_CUDA(cudaStreamCreateWithFlags(&c.h2d_stream, cudaStreamNonBlocking));
        if (!c.d2h_stream) FDM_CUDA(cudaStreamCreateWithFlags(&c.d2h_stream, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
          for (cudaEvent_t* e : {&c.ev_in[k], &c.ev_comp[k], &c.ev_out[k]})
            if (!*e) FDM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
          if (c.stage_in[k].n != size_t(c.ndof)) c.stage_in[k].alloc(c.ndof);
          if (c.stage_out[k].n != size_t(c.ndof)) c.stage_out[k].alloc(c.ndof);
        }
      } catch (...) {
        for (int k = 0; k < 2; ++k) {
          c.stage_in[k].reset();
          c.stage_out[k].reset();
        }
        throw;
      }
      c.async_ready = true;
    }
    const int s = c.async_slot;
    c.async_slot ^= 1;
    const size_t bytes = c.ndof * sizeof(double);
    // copy-in once this slot's previous input has been consumed
    FDM_CUDA(cudaStreamWaitEvent(c.h2d_stream, c.ev_comp[s], 0));
    FDM_CUDA(cudaMemcpyAsync(c.stage_in[s].p, host_in, bytes, cudaMemcpyHostToDevice, c.h2d_stream));
    FDM_CUDA(cudaEventRecord(c.ev_in[s], c.h2d_stream));
    // compute once the input is in and this slot's previous output has been copied out
    FDM_CUDA(cudaStreamWaitEvent(c.stream, c.ev_in[s], 0));
    FDM_CUDA(cudaStreamWaitEvent(c.stream, c.ev_out[s], 0));
    const double* din = c.stage_in[s].p;
    double* dout = c.stage_out[s].p;
    switch (op) {
      case FDMGPU_OP_APPLY_ST: fdmgpu::op_transform(c, 0, din, dout); break;
      case FDMGPU_OP_APPLY_S: fdmgpu::op_transform(c, 1, din, dout); break;
      case FDMGPU_OP_PATCH: fdmgpu::op_patch(c, din, dout); break;
      case FDMGPU_OP_SMOOTH: fdmgpu::op_smooth(c, din, dout); break;
      case FDMGPU_OP_A: fdmgpu::op_A(c, din, dout); break;
      default: fdmgpu::op_vcycle(c, omega, din, dout); break;
    }
    FDM_CUDA(cudaEventRecord(c.ev_comp[s], c.stream));
    FDM_CUDA(cudaStreamWaitEvent(c.d2h_stream, c.ev_comp[s], 0));
    FDM_CUDA(cudaMemcpyAsync(host_out, dout, bytes, cudaMemcpyDeviceToHost, c.d2h_stream));
    FDM_CUDA(cudaEventRecord(c.ev_out[s], c.d2h_stream));
  });
}

fdmgpu_status fdmgpu_async_join(fdmgpu_handle h) {
  return fdmgpu::guarded(h, [&](Context& c) {
    for (int k = 0; k < 2; ++k)
      if (c.ev_out[k]) FDM_CUDA(cudaStreamWaitEvent(c.stream, c.ev_out[k], 0));
  });
}

fdmgpu_status fdmgpu_transform(fdmgpu_handle h, int32_t dir, const double* in, double* out) {
  return fdmgpu_apply(h, dir == 0 ? FDMGPU_OP_APPLY_ST : FDMGPU_OP_APPLY_S, 0.0, in, out, 0);
}
fdmgpu_status fdmgpu_patch_solve(fdmgpu_handle h, const double* r, double* z) {
  return fdmgpu_apply(h, FDMGPU_OP_PATCH, 0.0, r, z, 0);
}
fdmgpu_status fdmgpu_smooth(fdmgpu_handle h, const double* r, double* z) {
  return fdmgpu_apply(h, FDMGPU_OP_SMOOTH, 0.0, r, z, 0);
}
fdmgpu_status fdmgpu_apply_A(fdmgpu_handle h, const double* x, double* y) {
  return fdmgpu_apply(h, FDMGPU_OP_A, 0.0, x, y, 0);
}
fdmgpu_status fdmgpu_vcycle(fdmgpu_handle h, double omega, const double* r, double* z) {
  return fdmgpu_apply(h, FDMGPU_OP_VCYCLE, omega, r, z, 0);
}

fdmgpu_status fdmgpu_pcg(fdmgpu_handle h, const double* b, double* x, double rtol, int32_t maxit, int32_t precond,
                         fdmgpu_krylov_report* report, double* residuals) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::NvtxRange nvtx_("fdmgpu_pcg");
    if (!b || !x || !report || maxit < 0 || b == x) throw Error(FDMGPU_INVALID_ARGUMENT, "pcg: bad arguments");
    c.check_ready(precond > 0, precond > 0, precond == 2);
    std::vector<double> res;
    fdmgpu::run_pcg(c, b, x, rtol, maxit, precond, c.omega, report, residuals ? &res : nullptr);
    if (residuals) std::copy(res.begin(), res.end(), residuals);
  });
}

fdmgpu_status fdmgpu_calibrate_damping(fdmgpu_handle h, int32_t lanczos_steps, uint32_t seed, int32_t formula,
                                       double* omega, double* lambda_min, double* lambda_max) {
  return fdmgpu::guarded(h, [&](Context& c) {
    fdmgpu::NvtxRange nvtx_("fdmgpu_calibrate_damping");
    c.check_ready(true, true, true);
    double* b = c.w[11].p;
    double* x = c.w[10].p;
    fdmgpu_krylov_report rep{};
    // estimate_damping (src/schwarz.cpp:97-119): CG-Lanczos of the smoother.
    auto hb = fdmgpu::random_free(c, seed);
    FDM_CUDA(cudaMemcpyAsync(b, hb.data(), c.ndof * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    double est_omega = 1.0, est_lmin = 0.0, est_lmax = 0.0;
    try {
      fdmgpu::run_pcg(c, b, x, 1e-12, lanczos_steps, 1, 1.0, &rep, nullptr);
      if (rep.lambda_min > 0.0 && rep.lambda_max > 0.0) {
        est_lmin = rep.lambda_min;
        est_lmax = rep.lambda_max;
        est_omega = formula == 2 ? 0.5 * (est_lmax + est_lmin) : 2.0 / (est_lmax + est_lmin);
      }
    } catch (const Error& e) {
      if (e.status != FDMGPU_INDEFINITE) throw;
    }
    c.lambda_min = est_lmin;
    c.lambda_max = est_lmax;
    if (est_lmax <= 0.0) {
      c.omega = 1.0;
    } else if (formula != 0) {
      c.omega = est_omega;
    } else {
      // Two-grid calibration (src/schwarz.cpp:184-227).
      const double omega0 = 1.0 / est_lmax;
      auto hb2 = fdmgpu::random_free(c, uint64_t(seed) + 1);
      FDM_CUDA(cudaMemcpyAsync(b, hb2.data(), c.ndof * sizeof(double), cudaMemcpyHostToDevice, c.stream));
      auto cycle_kappa = [&](double w) {
        try {
          fdmgpu::run_pcg(c, b, x, 1e-12, lanczos_steps, 2, w, &rep, nullptr);
          if (rep.lambda_min <= 0.0) return std::numeric_limits<double>::infinity();
          return rep.lambda_max / rep.lambda_min;
        } catch (const Error& e) {
          if (e.status != FDMGPU_INDEFINITE) throw;
          return std::numeric_limits<double>::infinity();
        }
      };
      double mu_c = est_lmin;
      try {
        fdmgpu::run_pcg(c, b, x, 1e-12, lanczos_steps, 2, omega0, &rep, nullptr);
        if (rep.lambda_min > 0.0 && rep.lambda_min < 1.0) mu_c = (1.0 - std::sqrt(1.0 - rep.lambda_min)) / omega0;
      } catch (const Error& e) {
        if (e.status != FDMGPU_INDEFINITE) throw;
      }
      mu_c = std::min(std::max(mu_c, est_lmin), est_lmax);
      double best_omega = 2.0 / (mu_c + est_lmax);
      double best_kappa = cycle_kappa(best_omega);
      for (double f : {0.8, 1.2, 1.4}) {
        const double w = f * omega0;
        if (w >= 2.0 * omega0 || std::abs(w - best_omega) < 1e-3) continue;
        const double k = cycle_kappa(w);
        if (k < best_kappa) {
          best_kappa = k;
          best_omega = w;
        }
      }
      c.omega = best_omega;
    }
    if (omega) *omega = c.omega;
    if (lambda_min) *lambda_min = c.lambda_min;
    if (lambda_max) *lambda_max = c.lambda_max;
  });
}

fdmgpu_status fdmgpu_set_omega(fdmgpu_handle h, double omega) {
  return fdmgpu::guarded(h, [&](Context& c) { c.omega = omega; });
}

fdmgpu_status fdmgpu_get_omega(fdmgpu_handle h, double* omega) {
  return fdmgpu::guarded(h, [&](Context& c) { *omega = c.omega; });
}

int64_t fdmgpu_launch_count(fdmgpu_handle h) {
  if (!h) return -1;
  int64_t n = h->launches;
  for (Context* s : h->comp) n += s->launches;
  return n;
}

fdmgpu_status fdmgpu_set_separator_order(fdmgpu_handle h, int32_t order) {
  return fdmgpu::guarded(h, [&](Context& c) {
    if (order != 0 && order != 1) throw Error(FDMGPU_INVALID_ARGUMENT, "separator order: 0 plane, 1 reference");
    c.sep_order = order;
    for (Context* s : c.comp) s->sep_order = order;
  });
}

fdmgpu_status fdmgpu_kernel_timing(fdmgpu_handle h, int32_t enable) {
  return fdmgpu::guarded(h, [&](Context& c) {
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    for (auto& v : c.tev) {
      for (auto& [a, b] : v) {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
      v.clear();
    }
    c.timing = enable != 0;
    fdmgpu::forward(c, [&](fdmgpu_handle sh, int) { return fdmgpu_kernel_timing(sh, enable); });
  });
}

fdmgpu_status fdmgpu_kernel_time(fdmgpu_handle h, int32_t which, double* total_ms, int64_t* launches) {
  return fdmgpu::guarded(h, [&](Context& c) {
    if (which < 0 || which > 4) throw Error(FDMGPU_INVALID_ARGUMENT, "kernel_time: class 0..4");
    FDM_CUDA(cudaStreamSynchronize(c.stream));
    double t = 0.0;
    int64_t n = 0;
    auto add = [&](Context& cc) {
      for (auto& [a, b] : cc.tev[which]) {
        float ms = 0.f;
        FDM_CUDA(cudaEventElapsedTime(&ms, a, b));
        t += ms;
      }
      n += int64_t(cc.tev[which].size());
    };
    add(c);
    for (Context* s : c.comp) add(*s);
    *total_ms = t;
    *launches = n;
  });
}

}  // extern "C"
