// Vector kernels of the V-cycle and PCG (src/schwarz.cpp:125-133,
// src/krylov.cpp:29-83): axpby, deterministic two-stage dot products, Q1
// restriction / prolongation (src/schwarz.cpp:128-129) and the dense coarse
// solve.  Reductions use a fixed grid and fixed per-thread order, so every
// result is bitwise reproducible run to run.
#include "common.cuh"

namespace fdmgpu {

namespace {

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                        double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = (b == 0.0 ? 0.0 : b * y[i]) + a * x[i];
}

template <int BS>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[BS / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) ws[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < BS / 32 ? ws[threadIdx.x] : 0.0;
    s = warp_sum(s);
  }
  __syncthreads();
  return s;
}

__global__ void k_dot_partials(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                               double* __restrict__ partial) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    s = fma(x[i], y[i], s);
  s = block_sum<256>(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// rc[i] = sum_q PT_val[q] * fine[PT_col[q]]  (one CTA per coarse row)
__global__ void k_restrict(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                           const double* __restrict__ val, const double* __restrict__ fine, double* __restrict__ rc) {
  const int i = blockIdx.x;
  // four independent chains: the fine[col[q]] gathers of a thread overlap
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const int q1 = ptr[i + 1], st = blockDim.x;
  int q = ptr[i] + threadIdx.x;
  for (; q + 3 * st < q1; q += 4 * st) {
    s0 = fma(val[q], fine[col[q]], s0);
    s1 = fma(val[q + st], fine[col[q + st]], s1);
    s2 = fma(val[q + 2 * st], fine[col[q + 2 * st]], s2);
    s3 = fma(val[q + 3 * st], fine[col[q + 3 * st]], s3);
  }
  for (; q < q1; q += st) s0 = fma(val[q], fine[col[q]], s0);
  double s = (s0 + s1) + (s2 + s3);
  s = block_sum<256>(s);
  if (threadIdx.x == 0) rc[i] = s;
}

__global__ void k_coarse_gemv(int nc, const double* __restrict__ inv, const double* __restrict__ rc,
                              double* __restrict__ zc) {
  const int i = blockIdx.x;
  double s = 0.0;
  for (int jj = threadIdx.x; jj < nc; jj += blockDim.x) s = fma(inv[size_t(i) * nc + jj], rc[jj], s);
  s = block_sum<256>(s);
  if (threadIdx.x == 0) zc[i] = s;
}

__global__ void k_prolong_add(int64_t n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                              const double* __restrict__ val, const double* __restrict__ zc,
                              double* __restrict__ fine) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int q = ptr[i]; q < ptr[i + 1]; ++q) s = fma(val[q], zc[col[q]], s);
  fine[i] += s;
}

// Cell-wise restriction P^T r (src/schwarz.cpp:139-165 summed per cell): each
// fine node contributes r_i / mult_i to the 2^d corner sums of every cell
// holding it, weighted by the separable Q1 hats; the corner sums are then
// gathered per coarse DOF in ascending (cell, corner) order.  Thread per x-line
// of the cell: the line's map and value loads are issued together.
template <int N1C>
__global__ void k_restrict_cells(int dim, int n1_rt, int npc, const double* __restrict__ r,
                                 const int32_t* __restrict__ cdofs, const double* __restrict__ inv_mult,
                                 const uint8_t* __restrict__ cons, const double* __restrict__ phat,
                                 double* __restrict__ cellsum) {
  constexpr int NB = N1C > 0 ? N1C : 32;
  const int n1 = N1C > 0 ? N1C : n1_rt;
  extern __shared__ double sm[];
  const int rows = dim == 3 ? n1 * n1 : n1;
  double* rs = sm;             // [rows][2]  x-reduced
  double* ys = rs + 2 * rows;  // [n1][4]    y-reduced (3D)
  const int c = blockIdx.x;
  const int32_t* cd = cdofs + size_t(c) * npc;
  for (int row = threadIdx.x; row < rows; row += blockDim.x) {
    int g[NB];
#pragma unroll
    for (int l0 = 0; l0 < NB; ++l0) g[l0] = l0 < n1 ? cd[l0 + n1 * row] : 0;
    double v[NB];
#pragma unroll
    for (int l0 = 0; l0 < NB; ++l0) {
      const double rv = r[g[l0]], w = inv_mult[g[l0]];
      v[l0] = (l0 < n1 && !cons[g[l0]]) ? rv * w : 0.0;
    }
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int l0 = 0; l0 < NB; ++l0) {
      if (l0 < n1) {
        s0 = fma(phat[l0], v[l0], s0);
        s1 = fma(phat[l0 + n1], v[l0], s1);
      }
    }
    rs[2 * row] = s0;
    rs[2 * row + 1] = s1;
  }
  __syncthreads();
  if (dim == 2) {
    if (threadIdx.x < 4) {
      const int a0 = threadIdx.x & 1, a1 = threadIdx.x >> 1;
      double s = 0.0;
      for (int l1 = 0; l1 < n1; ++l1) s = fma(phat[l1 + n1 * a1], rs[2 * l1 + a0], s);
      cellsum[size_t(c) * 4 + threadIdx.x] = s;
    }
    return;
  }
  for (int e = threadIdx.x; e < 4 * n1; e += blockDim.x) {  // (l2, a0, a1)
    const int l2 = e >> 2, a0 = e & 1, a1 = (e >> 1) & 1;
    double s = 0.0;
    for (int l1 = 0; l1 < n1; ++l1) s = fma(phat[l1 + n1 * a1], rs[2 * (l1 + n1 * l2) + a0], s);
    ys[e] = s;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int a01 = threadIdx.x & 3, a2 = threadIdx.x >> 2;
    double s = 0.0;
    for (int l2 = 0; l2 < n1; ++l2) s = fma(phat[l2 + n1 * a2], ys[4 * l2 + a01], s);
    cellsum[size_t(c) * 8 + threadIdx.x] = s;
  }
}

__global__ void k_restrict_gather(int nc, const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                  const double* __restrict__ cellsum, double* __restrict__ rc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  double s = 0.0;
  for (int q = ptr[j]; q < ptr[j + 1]; ++q) s += cellsum[idx[q]];
  rc[j] = s;  // constrained coarse DOFs have no slots: 0
}

// Cell-wise prolongation fine += P zc: every free fine node is written once, by
// the lowest cell holding it, with its trilinear interpolant of the cell's
// free coarse corner values (separable: thread per x-line, the 2^d corners
// folded to the line's two end values first).
template <int N1C>
__global__ void k_prolong_cells(int dim, int n1_rt, int npc, const double* __restrict__ zc,
                                const int32_t* __restrict__ ccd, const int32_t* __restrict__ cdofs,
                                const uint8_t* __restrict__ owner, const double* __restrict__ phat,
                                double* __restrict__ fine) {
  constexpr int NB = N1C > 0 ? N1C : 32;
  const int n1 = N1C > 0 ? N1C : n1_rt;
  __shared__ double zv[8];
  const int c = blockIdx.x, ncorner = 1 << dim;
  if (threadIdx.x < ncorner) {
    const int j = ccd[size_t(c) * ncorner + threadIdx.x];
    zv[threadIdx.x] = j >= 0 ? zc[j] : 0.0;
  }
  __syncthreads();
  const int rows = dim == 3 ? n1 * n1 : n1;
  const int32_t* cd = cdofs + size_t(c) * npc;
  const uint8_t* ow = owner + size_t(c) * npc;
  for (int row = threadIdx.x; row < rows; row += blockDim.x) {
    const int l1 = row % n1, l2 = dim == 3 ? row / n1 : 0;
    double e0 = 0.0, e1 = 0.0;  // the line's values at x = -1 / +1
    for (int j = 0; j < ncorner; j += 2) {
      double w = phat[l1 + n1 * ((j >> 1) & 1)];
      if (dim == 3) w *= phat[l2 + n1 * (j >> 2)];
      e0 = fma(w, zv[j], e0);
      e1 = fma(w, zv[j + 1], e1);
    }
    int g[NB];
    bool on[NB];
#pragma unroll
    for (int l0 = 0; l0 < NB; ++l0) {
      const int l = l0 + n1 * row;
      on[l0] = l0 < n1 && ow[l];
      g[l0] = on[l0] ? cd[l] : 0;
    }
    double f[NB];
#pragma unroll
    for (int l0 = 0; l0 < NB; ++l0) f[l0] = on[l0] ? fine[g[l0]] : 0.0;
#pragma unroll
    for (int l0 = 0; l0 < NB; ++l0)
      if (on[l0]) fine[g[l0]] = f[l0] + fma(phat[l0], e0, phat[l0 + n1] * e1);
  }
}

}  // namespace

void launch_axpby(Context& c, int64_t n, double a, const double* x, double b, const double* y, double* out) {
  k_axpby<<<4 * 148, 256, 0, c.stream>>>(n, a, x, b, y, out);
  FDM_LAUNCH_CHECK(c);
}

void launch_dot_partials(Context& c, int64_t n, const double* x, const double* y, int k) {
  k_dot_partials<<<kRedBlocks, 256, 0, c.stream>>>(n, x, y, c.red.p + size_t(k) * kRedBlocks);
  FDM_LAUNCH_CHECK(c);
}

void launch_restrict(Context& c, const double* fine, double* coarse) {
  if (c.have_coarse_cells && c.n1 <= 32) {  // (generic kernels unroll to 32 points per line)
    const int rows = c.dim == 3 ? c.n1 * c.n1 : c.n1;
    const size_t sm = sizeof(double) * (2 * rows + 4 * c.n1);
    auto go = [&](auto kern) {
      kern<<<c.ncells, 256, sm, c.stream>>>(c.dim, c.n1, c.npc, fine, c.cell_dofs.p, c.inv_mult.p, c.constrained.p,
                                            c.phat.p, c.cellsum.p);
    };
    if (c.n1 == 16)
      go(k_restrict_cells<16>);
    else if (c.n1 == 8)
      go(k_restrict_cells<8>);
    else
      go(k_restrict_cells<0>);
    FDM_LAUNCH_CHECK(c);
    k_restrict_gather<<<(c.nc + 255) / 256, 256, 0, c.stream>>>(c.nc, c.cg_ptr.p, c.cg_idx.p, c.cellsum.p, coarse);
    FDM_LAUNCH_CHECK(c);
    return;
  }
  k_restrict<<<c.nc, 256, 0, c.stream>>>(c.PT_ptr.p, c.PT_col.p, c.PT_val.p, fine, coarse);
  FDM_LAUNCH_CHECK(c);
}

void launch_coarse_solve(Context& c, const double* rc, double* zc) {
  k_coarse_gemv<<<c.nc, 256, 0, c.stream>>>(c.nc, c.cinv.p, rc, zc);
  FDM_LAUNCH_CHECK(c);
}

void launch_prolong_add(Context& c, const double* coarse, double* fine) {
  const int threads = 256;
  if (c.have_coarse_cells && c.n1 <= 32) {
    auto go = [&](auto kern) {
      kern<<<c.ncells, threads, 0, c.stream>>>(c.dim, c.n1, c.npc, coarse, c.ccd.p, c.cell_dofs.p, c.powner.p, c.phat.p,
                                               fine);
    };
    if (c.n1 == 16)
      go(k_prolong_cells<16>);
    else if (c.n1 == 8)
      go(k_prolong_cells<8>);
    else
      go(k_prolong_cells<0>);
    FDM_LAUNCH_CHECK(c);
    return;
  }
  k_prolong_add<<<unsigned((c.ndof + threads - 1) / threads), threads, 0, c.stream>>>(c.ndof, c.P_ptr.p, c.P_col.p,
                                                                                       c.P_val.p, coarse, fine);
  FDM_LAUNCH_CHECK(c);
}

}  // namespace fdmgpu
