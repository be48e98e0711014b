// Staged cell kernels for tiles that do not fit in shared memory (3D p >= 16,
// e.g. config C5 at p = 31: a (p+1)^3 tile is 256 KB) and the true-form
// operator of non-Cartesian cells.
//
//   * S / S^T transform: gather into the cell-local E-vector, then one
//     launch per axis contracting E in place through L2 (src/kron.cpp:20-38),
//     with the FDM interior elimination / rebuild (see cells.cu) as separate
//     per-cell passes on the modal tile.
//   * Trilinear true-form operator (src/assembly.cpp:198-228, symmetrised
//     dense matrix on the GL(p+2) tensor rule): the
//     (p+1)^3 x (p+1)^3 cell matrix (8.6 GB per cell at p = 31) is never
//     formed; it is applied sum-factorised as G^T diag(w kappa G) G in three
//     stages: x/y interpolation per z-slab, z-interpolation + pointwise
//     metric (recomputed from the 8 cell corners) + z-projection per
//     quadrature column, x/y projection per z-slab.
#include "common.cuh"

namespace fdmgpu {

namespace {

__global__ void k_cell_load(int npc, int dir, const double* __restrict__ in, double* __restrict__ E,
                            const int32_t* __restrict__ cdofs, const double* __restrict__ inv_mult,
                            const uint8_t* __restrict__ cons, const double* __restrict__ sign, int64_t total) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int g = cdofs[e];
    double v = cons[g] ? 0.0 : in[g];
    if (dir == 0)
      v *= inv_mult[g];
    else if (sign)
      v *= sign[e];
    E[e] = v;
  }
}

// out[c][.., k, ..] = sum_j M[k + n1 j] in[c][.., j, ..] along the axis with `stride`.
__global__ void k_axis_contract(int n1, int npc, int stride, const double* __restrict__ M, const double* __restrict__ in,
                                double* __restrict__ out, int64_t total) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = e / npc;
    const int o = int(e - c * npc);
    const int k = (o / stride) % n1;
    const double* src = in + c * npc + (o - k * stride);
    double s = 0.0;
    for (int j = 0; j < n1; ++j) s = fma(__ldg(M + k + n1 * j), src[j * stride], s);
    out[e] = s;
  }
}

__global__ void k_cell_sign(int64_t total, const double* __restrict__ sign, double* __restrict__ E) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x)
    E[e] *= sign[e];
}

__device__ __forceinline__ double diag_at(int dim, int n1, const double* mu, const double* At, const double* Bt,
                                          const int* x) {
  double s = 0.0;
  for (int q = 0; q < dim; ++q) {
    double prod = mu[q];
    for (int b = dim - 1; b >= 0; --b) prod *= (b == q ? At : Bt)[x[b] * (n1 + 1)];
    s += prod;
  }
  return s;
}

// E[c][facet point] -= sum_x A~_{f,x} E[c][x] / D_x   (one thread per face point)
__global__ void k_cell_schur_g(int dim, int n1, int npc, int ncells, double* __restrict__ E,
                               const double* __restrict__ mu, const double* __restrict__ At,
                               const double* __restrict__ Bt) {
  const int p = n1 - 1, pm = p - 1;
  int nt = 1;
  for (int a = 1; a < dim; ++a) nt *= pm;
  const int64_t per_cell = int64_t(2 * dim) * nt;
  const int64_t total = per_cell * ncells;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(e / per_cell);
    const int idx = int(e - int64_t(c) * per_cell);
    const int face = idx / nt, a = face >> 1, ee = (face & 1) ? p : 0;
    int t = idx % nt;
    int x[3] = {0, 0, 0};
    double mus[3] = {0, 0, 0};
    for (int q = 0; q < dim; ++q) mus[q] = mu[size_t(c) * dim + q];
    double coef = mus[a];
    int lin0 = 0, stride_a = 1;
    for (int b = 0, s = 1; b < dim; ++b, s *= n1) {
      if (b == a) {
        stride_a = s;
        continue;
      }
      x[b] = 1 + t % pm;
      t /= pm;
      coef *= Bt[x[b] * (n1 + 1)];
      lin0 += x[b] * s;
    }
    double* u = E + size_t(c) * npc;
    double acc = 0.0;
    for (int xa = 1; xa < p; ++xa) {
      x[a] = xa;
      acc = fma(At[ee + n1 * xa] * u[lin0 + xa * stride_a], 1.0 / diag_at(dim, n1, mus, At, Bt, x), acc);
    }
    u[lin0 + ee * stride_a] -= coef * acc;
  }
}

// E[c][x] = (nK b[x] - sum_{a,e} A~_{x,f} E[c][f]) / D_x for every interior x.
__global__ void k_cell_recon_g(int dim, int n1, int npc, int ncells, double* __restrict__ E,
                               const double* __restrict__ rb, const int32_t* __restrict__ cdofs,
                               const double* __restrict__ mu, const double* __restrict__ At,
                               const double* __restrict__ Bt, const double* __restrict__ nK) {
  const int p = n1 - 1, pm = p - 1;
  int ni = 1;
  for (int a = 0; a < dim; ++a) ni *= pm;
  const int64_t total = int64_t(ni) * ncells;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(e / ni);
    int ii = int(e - int64_t(c) * ni);
    int x[3] = {0, 0, 0}, lin = 0;
    for (int a = 0, s = 1; a < dim; ++a, s *= n1) {
      x[a] = 1 + ii % pm;
      ii /= pm;
      lin += x[a] * s;
    }
    double mus[3] = {0, 0, 0};
    for (int q = 0; q < dim; ++q) mus[q] = mu[size_t(c) * dim + q];
    double* u = E + size_t(c) * npc;
    double v = nK[c] * rb[cdofs[size_t(c) * npc + lin]];
    for (int a = 0, s = 1; a < dim; ++a, s *= n1) {
      double coef = mus[a];
      for (int b = 0; b < dim; ++b)
        if (b != a) coef *= Bt[x[b] * (n1 + 1)];
      const int base = lin - x[a] * s;
      v -= coef * (At[x[a]] * u[base] + At[x[a] + n1 * p] * u[base + p * s]);
    }
    u[lin] = v / diag_at(dim, n1, mus, At, Bt, x);
  }
}

// ---- trilinear true-form operator, 3D -----------------------------------------
// Stage 1: per (cell, z-level kz): t0 = V_x u, t1 = D_x u, then
// T[c][0] = V_y t0 (-> d/dz path), T[c][1] = D_y t0 (d/dy), T[c][2] = V_y t1 (d/dx);
// layout T[c][f][kz][qy][qx].
__global__ void k_quad_stage1(int n1, int q, const double* __restrict__ x, const int32_t* __restrict__ cdofs,
                              const uint8_t* __restrict__ cons, const double* __restrict__ Vq,
                              const double* __restrict__ Dq, double* __restrict__ T) {
  extern __shared__ double sm[];
  double* V = sm;              // q x n1, V[qi + q j]
  double* D = V + q * n1;
  double* u = D + q * n1;      // n1 x n1 slab, u[i + n1 j]
  double* t0 = u + n1 * n1;    // q x n1, t0[qx + q j]
  double* t1 = t0 + q * n1;
  const int c = blockIdx.x / n1, kz = blockIdx.x % n1;
  const int npc = n1 * n1 * n1, q2 = q * q;
  for (int i = threadIdx.x; i < q * n1; i += blockDim.x) {
    V[i] = Vq[i];
    D[i] = Dq[i];
  }
  const int32_t* cd = cdofs + size_t(c) * npc + size_t(kz) * n1 * n1;
  for (int l = threadIdx.x; l < n1 * n1; l += blockDim.x) {
    const int g = cd[l];
    u[l] = cons[g] ? 0.0 : x[g];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < q * n1; o += blockDim.x) {
    const int qx = o % q, j = o / q;
    double s0 = 0.0, s1 = 0.0;
    for (int i = 0; i < n1; ++i) {
      const double ui = u[i + n1 * j];
      s0 = fma(V[qx + q * i], ui, s0);
      s1 = fma(D[qx + q * i], ui, s1);
    }
    t0[o] = s0;
    t1[o] = s1;
  }
  __syncthreads();
  double* out = T + size_t(c) * 3 * n1 * q2 + size_t(kz) * q2;
  for (int o = threadIdx.x; o < q2; o += blockDim.x) {
    const int qx = o % q, qy = o / q;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int j = 0; j < n1; ++j) {
      const double v = V[qy + q * j], d = D[qy + q * j];
      a0 = fma(v, t0[qx + q * j], a0);
      a1 = fma(d, t0[qx + q * j], a1);
      a2 = fma(v, t1[qx + q * j], a2);
    }
    out[o] = a0;
    out[size_t(n1) * q2 + o] = a1;
    out[2 * size_t(n1) * q2 + o] = a2;
  }
}

constexpr int kQuadCols = 64;

// Stage 2: per quadrature column (qx, qy): gradients g = (V_z T2, V_z T1, D_z T0),
// f = w kappa G g with G = det J^{-1} J^{-T} of the trilinear map, then the
// z-projection back into T in place: T0 <- V_z^T f_x, T1 <- V_z^T f_y, T2 <- D_z^T f_z.
__global__ void k_quad_stage2(int n1, int q, double* __restrict__ T, const double* __restrict__ Vq,
                              const double* __restrict__ Dq, const double* __restrict__ wq,
                              const double* __restrict__ xyz, const double* __restrict__ kappa,
                              const double* __restrict__ qpts) {
  extern __shared__ double sm[];
  double* V = sm;
  double* D = V + q * n1;
  double* W = D + q * n1;           // q weights, q points
  double* X = W + 2 * q;            // 24 corner coordinates
  double* col = X + 24;             // [3 * n1][kQuadCols]
  double* fs = col + 3 * n1 * kQuadCols;  // [3 * q][kQuadCols]
  const int q2 = q * q;
  const int chunks = (q2 + kQuadCols - 1) / kQuadCols;
  const int c = blockIdx.x / chunks;
  const int cc = (blockIdx.x % chunks) * kQuadCols + threadIdx.x;
  for (int i = threadIdx.x; i < q * n1; i += blockDim.x) {
    V[i] = Vq[i];
    D[i] = Dq[i];
  }
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    W[i] = wq[i];
    W[q + i] = qpts[i];
  }
  for (int i = threadIdx.x; i < 24; i += blockDim.x) X[i] = xyz[size_t(c) * 24 + i];
  __syncthreads();
  if (cc >= q2) return;
  const int tid = threadIdx.x;
  const int qx = cc % q, qy = cc / q;
  double* base = T + size_t(c) * 3 * n1 * q2 + cc;
  for (int f = 0; f < 3; ++f)
    for (int k = 0; k < n1; ++k) col[(f * n1 + k) * kQuadCols + tid] = base[(size_t(f) * n1 + k) * q2];
  const double kap = kappa[c];
  const double xh0 = W[q + qx], xh1 = W[q + qy];
  for (int qz = 0; qz < q; ++qz) {
    double g0 = 0.0, g1 = 0.0, g2 = 0.0;
    for (int k = 0; k < n1; ++k) {
      const double v = V[qz + q * k], d = D[qz + q * k];
      g0 = fma(v, col[(2 * n1 + k) * kQuadCols + tid], g0);
      g1 = fma(v, col[(1 * n1 + k) * kQuadCols + tid], g1);
      g2 = fma(d, col[(0 * n1 + k) * kQuadCols + tid], g2);
    }
    // Jacobian of the trilinear map (src/geometry.cpp:33-43), J[r][a]
    const double xh[3] = {xh0, xh1, W[q + qz]};
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int b = 0; b < 8; ++b) {
      double dphi[3];
      for (int a = 0; a < 3; ++a) {
        double gg = 1.0;
        for (int e = 0; e < 3; ++e) {
          const bool hi = (b >> e) & 1;
          gg *= (e == a) ? (hi ? 0.5 : -0.5) : (hi ? 0.5 * (1.0 + xh[e]) : 0.5 * (1.0 - xh[e]));
        }
        dphi[a] = gg;
      }
      for (int r = 0; r < 3; ++r)
        for (int a = 0; a < 3; ++a) J[r][a] += dphi[a] * X[3 * b + r];
    }
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    double inv[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
        inv[i][j] = (J[i1][j1] * J[i2][j2] - J[i1][j2] * J[i2][j1]) / det;
      }
    double G[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) G[a][b] = det * (inv[a][0] * inv[b][0] + inv[a][1] * inv[b][1] + inv[a][2] * inv[b][2]);
    const double w = W[qx] * W[qy] * W[qz] * kap;
    const double g[3] = {g0, g1, g2};
    for (int a = 0; a < 3; ++a) fs[(a * q + qz) * kQuadCols + tid] = w * (G[a][0] * g[0] + G[a][1] * g[1] + G[a][2] * g[2]);
  }
  for (int k = 0; k < n1; ++k) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int qz = 0; qz < q; ++qz) {
      const double v = V[qz + q * k], d = D[qz + q * k];
      a0 = fma(v, fs[(0 * q + qz) * kQuadCols + tid], a0);
      a1 = fma(v, fs[(1 * q + qz) * kQuadCols + tid], a1);
      a2 = fma(d, fs[(2 * q + qz) * kQuadCols + tid], a2);
    }
    base[(size_t(0) * n1 + k) * q2] = a0;  // x-gradient path
    base[(size_t(1) * n1 + k) * q2] = a1;  // y
    base[(size_t(2) * n1 + k) * q2] = a2;  // z
  }
}

// Stage 3: per (cell, kz): b0 = V_y^T T0, b12 = D_y^T T1 + V_y^T T2,
// E = D_x^T b0 + V_x^T b12.
__global__ void k_quad_stage3(int n1, int q, const double* __restrict__ T, const double* __restrict__ Vq,
                              const double* __restrict__ Dq, double* __restrict__ E) {
  extern __shared__ double sm[];
  double* V = sm;
  double* D = V + q * n1;
  double* b0 = D + q * n1;   // q x n1: b0[qx + q j]
  double* b12 = b0 + q * n1;
  const int c = blockIdx.x / n1, kz = blockIdx.x % n1;
  const int q2 = q * q;
  for (int i = threadIdx.x; i < q * n1; i += blockDim.x) {
    V[i] = Vq[i];
    D[i] = Dq[i];
  }
  __syncthreads();
  const double* in = T + size_t(c) * 3 * n1 * q2 + size_t(kz) * q2;
  for (int o = threadIdx.x; o < q * n1; o += blockDim.x) {
    const int qx = o % q, j = o / q;
    double s0 = 0.0, s12 = 0.0;
    for (int qy = 0; qy < q; ++qy) {
      const double v = V[qy + q * j], d = D[qy + q * j];
      s0 = fma(v, in[qx + q * qy], s0);
      s12 = fma(d, in[size_t(n1) * q2 + qx + q * qy], s12);
      s12 = fma(v, in[2 * size_t(n1) * q2 + qx + q * qy], s12);
    }
    b0[o] = s0;
    b12[o] = s12;
  }
  __syncthreads();
  double* out = E + size_t(c) * n1 * n1 * n1 + size_t(kz) * n1 * n1;
  for (int o = threadIdx.x; o < n1 * n1; o += blockDim.x) {
    const int i = o % n1, j = o / n1;
    double s = 0.0;
    for (int qx = 0; qx < q; ++qx) s = fma(D[qx + q * i], b0[qx + q * j], fma(V[qx + q * i], b12[qx + q * j], s));
    out[o] = s;
  }
}

unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  return unsigned(b > 148 * 64 ? 148 * 64 : b);
}

// OP_PATCH helpers for staged tiles: keep interior modal values only.
__global__ void k_cell_mask_interior(int dim, int n1, int npc, int64_t total, double* __restrict__ E, int keep_interior) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    int l = int(e % npc);
    bool interior = true;
    for (int a = 0; a < dim; ++a, l /= n1) interior = interior && (l % n1 != 0) && (l % n1 != n1 - 1);
    if (interior != (keep_interior != 0)) E[e] = 0.0;
  }
}

__global__ void k_cell_store_interior(int dim, int n1, int npc, int64_t total, const double* __restrict__ E,
                                      const int32_t* __restrict__ cdofs, double* __restrict__ z) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    int l = int(e % npc);
    bool interior = true;
    for (int a = 0; a < dim; ++a, l /= n1) interior = interior && (l % n1 != 0) && (l % n1 != n1 - 1);
    if (interior) z[cdofs[e]] = E[e];
  }
}

}  // namespace

void launch_cells_transform_fused(Context& c, int dir, const double* in, int flags, const double* aux);
void launch_cells_schur_fused(Context& c, const double* in);
void launch_cells_recon_fused(Context& c, double* z, const double* rb);
void launch_cells_stiffness_kron(Context& c, const double* x);

bool cells_fit_smem(const Context& c) {
  if (c.force_staged) return false;
  int ni = 1;
  for (int a = 0; a < c.dim; ++a) ni *= c.p - 1;
  const size_t need = sizeof(double) * (3 * size_t(c.n1) * c.n1 + 2 * size_t(c.npc) + ni);
  const size_t need_k = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 4 * size_t(c.npc));
  return need <= 227 * 1024 && need_k <= 227 * 1024;
}

// Staged transform (any tile size): E <- S^T-or-S contractions of the gathered
// cell values, with the optional FDM interior elimination / rebuild passes.
void launch_cells_transform_staged(Context& c, int dir, const double* in, int flags, const double* aux) {
  const int64_t total = int64_t(c.ncells) * c.npc;
  if (c.E2.n < size_t(total)) c.E2.alloc(total);
  {
    KernelTimer timer(c, 2);
    k_cell_load<<<grid_for(total), 256, 0, c.stream>>>(c.npc, dir, in, c.E.p, dir == 0 ? c.cell_dofs.p : c.cell_modes.p,
                                                       c.inv_mult.p, c.constrained.p, c.mode_sign.p, total);
    FDM_LAUNCH_CHECK(c);
  }
  if (flags & 2) {  // rebuild interior modes before S
    const int64_t t = int64_t(c.ncells) * (c.L.nI / (1 << c.dim));
    k_cell_recon_g<<<grid_for(t), 256, 0, c.stream>>>(c.dim, c.n1, c.npc, c.ncells, c.E.p, aux, c.cell_modes.p,
                                                      c.mu.p, c.At.p, c.Bt.p, c.nK.p);
    FDM_LAUNCH_CHECK(c);
  }
  const double* M = dir == 0 ? c.St.p : c.S.p;
  double* src = c.E.p;
  double* dst = c.E2.p;
  for (int a = 0, stride = 1; a < c.dim; ++a, stride *= c.n1) {
    KernelTimer timer(c, 2);
    k_axis_contract<<<grid_for(total), 256, 0, c.stream>>>(c.n1, c.npc, stride, M, src, dst, total);
    FDM_LAUNCH_CHECK(c);
    std::swap(src, dst);
  }
  if (src != c.E.p) {
    FDM_CUDA(cudaMemcpyAsync(c.E.p, src, total * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  }
  if (dir == 0 && c.mode_sign.p) {
    k_cell_sign<<<grid_for(total), 256, 0, c.stream>>>(total, c.mode_sign.p, c.E.p);
    FDM_LAUNCH_CHECK(c);
  }
  if (flags & 1) {
    int nt = 1;
    for (int a = 1; a < c.dim; ++a) nt *= c.p - 1;
    const int64_t t = int64_t(c.ncells) * 2 * c.dim * nt;
    k_cell_schur_g<<<grid_for(t), 256, 0, c.stream>>>(c.dim, c.n1, c.npc, c.ncells, c.E.p, c.mu.p, c.At.p, c.Bt.p);
    FDM_LAUNCH_CHECK(c);
  }
}

void launch_cells_quadrature(Context& c, const double* x) {
  if (c.dim != 3) throw Error(FDMGPU_UNSUPPORTED, "true-form quadrature operator: 3D only");
  if (!c.Vq.p || !c.xyz.p || !c.qpts.p) throw Error(FDMGPU_INVALID_ARGUMENT, "quadrature tables / corners not set");
  const int n1 = c.n1, q = c.q;
  const size_t need = size_t(c.ncells) * 3 * n1 * q * q;
  if (c.Qbuf.n < need) c.Qbuf.alloc(need);
  KernelTimer timer(c, 3);
  const size_t s1 = sizeof(double) * (2 * q * n1 + n1 * n1 + 2 * q * n1);
  FDM_CUDA(cudaFuncSetAttribute(k_quad_stage1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s1)));
  k_quad_stage1<<<c.ncells * n1, 256, s1, c.stream>>>(n1, q, x, c.cell_dofs.p, c.constrained.p, c.Vq.p, c.Dq.p,
                                                       c.Qbuf.p);
  FDM_LAUNCH_CHECK(c);
  const int chunks = (q * q + kQuadCols - 1) / kQuadCols;
  const size_t s2 = sizeof(double) * (2 * q * n1 + 2 * q + 24 + 3 * size_t(n1) * kQuadCols + 3 * size_t(q) * kQuadCols);
  FDM_CUDA(cudaFuncSetAttribute(k_quad_stage2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s2)));
  k_quad_stage2<<<c.ncells * chunks, kQuadCols, s2, c.stream>>>(n1, q, c.Qbuf.p, c.Vq.p, c.Dq.p, c.wq.p, c.xyz.p,
                                                                c.kappa.p, c.qpts.p);
  FDM_LAUNCH_CHECK(c);
  const size_t s3 = sizeof(double) * (4 * q * n1);
  FDM_CUDA(cudaFuncSetAttribute(k_quad_stage3, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s3)));
  k_quad_stage3<<<c.ncells * n1, 256, s3, c.stream>>>(n1, q, c.Qbuf.p, c.Vq.p, c.Dq.p, c.E.p);
  FDM_LAUNCH_CHECK(c);
}

}  // namespace fdmgpu

namespace fdmgpu {

// Allocate lazily-sized scratch before a CUDA-graph capture.
void prepare_buffers(Context& c) {
  if (!cells_fit_smem(c)) {
    const size_t total = size_t(c.ncells) * c.npc;
    if (c.E2.n < total) c.E2.alloc(total);
  }
  const bool kron_fits = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 4 * size_t(c.npc)) <= 227 * 1024;
  if (!(c.all_cartesian && kron_fits) && c.dim == 3 && c.q > 0) {
    const size_t need = size_t(c.ncells) * 3 * c.n1 * c.q * c.q;
    if (c.Qbuf.n < need) c.Qbuf.alloc(need);
  }
}

void launch_cells_transform(Context& c, int dir, const double* in, int flags, const double* aux) {
  if (cells_fit_smem(c))
    launch_cells_transform_fused(c, dir, in, flags, aux);
  else
    launch_cells_transform_staged(c, dir, in, flags, aux);
}

void launch_cells_stiffness(Context& c, const double* x) {
  const bool kron_fits = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 4 * size_t(c.npc)) <= 227 * 1024;
  if (c.all_cartesian && kron_fits)
    launch_cells_stiffness_kron(c, x);
  else
    launch_cells_quadrature(c, x);
}

void launch_cells_schur(Context& c, const double* in) {
  if (cells_fit_smem(c)) return launch_cells_schur_fused(c, in);
  const int64_t total = int64_t(c.ncells) * c.npc;
  k_cell_load<<<grid_for(total), 256, 0, c.stream>>>(c.npc, 1, in, c.E.p, c.cell_modes.p, c.inv_mult.p,
                                                     c.constrained.p, nullptr, total);
  FDM_LAUNCH_CHECK(c);
  k_cell_mask_interior<<<grid_for(total), 256, 0, c.stream>>>(c.dim, c.n1, c.npc, total, c.E.p, 1);
  FDM_LAUNCH_CHECK(c);
  int nt = 1;
  for (int a = 1; a < c.dim; ++a) nt *= c.p - 1;
  const int64_t t = int64_t(c.ncells) * 2 * c.dim * nt;
  k_cell_schur_g<<<grid_for(t), 256, 0, c.stream>>>(c.dim, c.n1, c.npc, c.ncells, c.E.p, c.mu.p, c.At.p, c.Bt.p);
  FDM_LAUNCH_CHECK(c);
  k_cell_mask_interior<<<grid_for(total), 256, 0, c.stream>>>(c.dim, c.n1, c.npc, total, c.E.p, 0);
  FDM_LAUNCH_CHECK(c);
}

void launch_cells_recon(Context& c, double* z, const double* rb) {
  if (cells_fit_smem(c)) return launch_cells_recon_fused(c, z, rb);
  const int64_t total = int64_t(c.ncells) * c.npc;
  k_cell_load<<<grid_for(total), 256, 0, c.stream>>>(c.npc, 1, z, c.E.p, c.cell_modes.p, c.inv_mult.p,
                                                     c.constrained.p, nullptr, total);
  FDM_LAUNCH_CHECK(c);
  const int64_t t = int64_t(c.ncells) * (c.L.nI / (1 << c.dim));
  k_cell_recon_g<<<grid_for(t), 256, 0, c.stream>>>(c.dim, c.n1, c.npc, c.ncells, c.E.p, rb, c.cell_modes.p, c.mu.p,
                                                    c.At.p, c.Bt.p, c.nK.p);
  FDM_LAUNCH_CHECK(c);
  k_cell_store_interior<<<grid_for(total), 256, 0, c.stream>>>(c.dim, c.n1, c.npc, total, c.E.p, c.cell_modes.p, z);
  FDM_LAUNCH_CHECK(c);
}

}  // namespace fdmgpu
