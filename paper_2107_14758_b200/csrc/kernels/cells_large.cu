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
// Every contraction is a small GEMM on shared-memory operands, run on the FP64
// tensor pipe (mma.sync m8n8k4 f64 -> DMMA): dims padded to multiples of 8
// (q = 33 -> 40) with zero rows/columns, each warp task an 8 x 16 output block
// (one A fragment, two B fragments per k-step).  Operand strides are chosen
// so fragment loads touch every bank pair exactly twice (two wavefronts).
constexpr int kQP = 40;  // padded quadrature count (q <= 40)

template <class FA, class FB, class FO>
__device__ __forceinline__ void dgemm_tc(int M, int N, int K, FA A, FB B, FO O) {
  // M, N multiples of 8, K multiple of 4
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int tm = M >> 3, tn = (N + 15) >> 4;
  const int ar = lane >> 2, ak = lane & 3;
  for (int task = warp; task < tm * tn; task += nw) {
    const int m0 = 8 * (task / tn), n0 = 16 * (task % tn);
    const bool two = n0 + 8 < N;
    double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
    for (int k0 = 0; k0 < K; k0 += 4) {
      const double a = A(m0 + ar, k0 + ak);
      const double b0 = B(k0 + ak, n0 + ar);
      const double b1 = two ? B(k0 + ak, n0 + 8 + ar) : 0.0;
      dmma884(d[0][0], d[0][1], a, b0);
      dmma884(d[1][0], d[1][1], a, b1);
    }
    const int r = m0 + ar, c = n0 + 2 * ak;
    O(r, c, d[0][0]);
    O(r, c + 1, d[0][1]);
    if (two) {
      O(r, c + 8, d[1][0]);
      O(r, c + 9, d[1][1]);
    }
  }
}

// Row-strip form: a warp task is an 8 x (8 NF) output block -- one A fragment and NF B
// fragments per k-step, NF independent accumulator chains (the 8 x 16 form above keeps two,
// and its short dependent DMMA chains were the stall ncu showed in these kernels).  `rot`
// rotates the task -> warp assignment so back-to-back calls fill the warps evenly.  Each
// output's sum runs over k in the same order as dgemm_tc (bitwise the same result).
template <int NF, int U, class FA, class FB, class FO>
__device__ __forceinline__ void dgemm_tc_s(int M, int N, int K, int rot, FA A, FB B, FO O) {
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int warp = int((threadIdx.x >> 5) + nw - rot % nw) % nw;
  const int tm = M >> 3, tn = (N + 8 * NF - 1) / (8 * NF);
  const int ar = lane >> 2, ak = lane & 3;
  for (int task = warp; task < tm * tn; task += nw) {
    const int m0 = 8 * (task / tn), n0 = 8 * NF * (task % tn);
    double d[NF][2];
#pragma unroll
    for (int f = 0; f < NF; ++f) d[f][0] = d[f][1] = 0.0;
#pragma unroll(U)
    for (int k0 = 0; k0 < K; k0 += 4) {
      const double a = A(m0 + ar, k0 + ak);
      double b[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) b[f] = n0 + 8 * f < N ? B(k0 + ak, n0 + 8 * f + ar) : 0.0;
#pragma unroll
      for (int f = 0; f < NF; ++f)
        if (n0 + 8 * f < N) dmma884(d[f][0], d[f][1], a, b[f]);
    }
    const int r = m0 + ar;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int c = n0 + 8 * f + 2 * ak;
      if (n0 + 8 * f < N) {
        O(r, c, d[f][0]);
        O(r, c + 1, d[f][1]);
      }
    }
  }
}

// One row strip (rows m0 .. m0 + 7, all 8 NF columns) into registers / from registers to O:
// the two halves of dgemm_tc_s, for outputs that overwrite an operand (stored after a barrier).
template <int NF, int U, class FA, class FB>
__device__ __forceinline__ void strip_compute(int m0, int K, FA A, FB B, double (&d)[NF][2]) {
  const int lane = threadIdx.x & 31, ar = lane >> 2, ak = lane & 3;
#pragma unroll
  for (int f = 0; f < NF; ++f) d[f][0] = d[f][1] = 0.0;
#pragma unroll(U)
  for (int k0 = 0; k0 < K; k0 += 4) {
    const double a = A(m0 + ar, k0 + ak);
    double b[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) b[f] = B(k0 + ak, 8 * f + ar);
#pragma unroll
    for (int f = 0; f < NF; ++f) dmma884(d[f][0], d[f][1], a, b[f]);
  }
}
template <int NF, class FO>
__device__ __forceinline__ void strip_store(int m0, const double (&d)[NF][2], FO O) {
  const int lane = threadIdx.x & 31, r = m0 + (lane >> 2), c0 = 2 * (lane & 3);
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    O(r, 8 * f + c0, d[f][0]);
    O(r, 8 * f + c0 + 1, d[f][1]);
  }
}

template <int S, int NF, class FA, class FB, class FO>
__device__ __forceinline__ void qgemm(int M, int N, int K, int rot, FA A, FB B, FO O) {
  if constexpr (S > 0)
    dgemm_tc_s<NF, (S >= 2 ? 4 : 2)>(M, N, K, rot, A, B, O);
  else
    dgemm_tc(M, N, K, A, B, O);
}

// V, D padded: Vp[qx + kQP i] (zero for qx >= q)
__device__ __forceinline__ void load_vd_padded(double* Vp, double* Dp, const double* __restrict__ Vq,
                                               const double* __restrict__ Dq, int q, int n1, int n1p) {
  for (int i = threadIdx.x; i < kQP * n1p; i += blockDim.x) {
    const int qx = i % kQP, j = i / kQP;
    const bool in = qx < q && j < n1;
    Vp[i] = in ? Vq[qx + q * j] : 0.0;
    Dp[i] = in ? Dq[qx + q * j] : 0.0;
  }
}

__host__ __device__ __forceinline__ int pad8(int n) { return (n + 7) & ~7; }
__host__ __device__ __forceinline__ int pad4(int n) { return (n + 3) & ~3; }

// Stage 1: per (cell, z-level kz): t0 = V_x u, t1 = D_x u, then
// T[c][0] = V_y t0 (-> d/dz path), T[c][1] = D_y t0 (d/dy), T[c][2] = V_y t1 (d/dx);
// layout T[c][f][kz][qy][qx].
template <int STRIP>
__global__ void __launch_bounds__(256) k_quad_stage1(int n1, int q, const double* __restrict__ x,
                                                      const int32_t* __restrict__ cdofs,
                                                      const uint8_t* __restrict__ cons, const double* __restrict__ Vq,
                                                      const double* __restrict__ Dq, double* __restrict__ T) {
  extern __shared__ __align__(16) double sm[];
  const int n1p = pad8(n1), n1k = pad4(n1), su = n1k + 4;
  double* Vp = sm;                  // kQP x n1p
  double* Dp = Vp + kQP * n1p;
  double* u = Dp + kQP * n1p;       // u[j * su + i], zero padded to n1p x n1k
  double* t0 = u + su * n1p;        // t0[j * kQP + qx]
  double* t1 = t0 + kQP * n1p;
  const int c = blockIdx.x / n1, kz = blockIdx.x % n1;
  const int npc = n1 * n1 * n1, q2 = q * q;
  load_vd_padded(Vp, Dp, Vq, Dq, q, n1, n1p);
  for (int i = threadIdx.x; i < su * n1p; i += blockDim.x) u[i] = 0.0;
  __syncthreads();
  const int32_t* cd = cdofs + size_t(c) * npc + size_t(kz) * n1 * n1;
#pragma unroll 4
  for (int l = threadIdx.x; l < n1 * n1; l += blockDim.x) {
    const int g = cd[l];
    const double xv = x[g];
    u[(l / n1) * su + l % n1] = cons[g] ? 0.0 : xv;
  }
  __syncthreads();
  auto Au = [&](int j, int i) { return u[j * su + i]; };
  qgemm<STRIP, 5>(n1p, kQP, n1k, 0, Au, [&](int i, int qx) { return Vp[qx + kQP * i]; },
           [&](int j, int qx, double v) { t0[j * kQP + qx] = v; });
  qgemm<STRIP, 5>(n1p, kQP, n1k, n1p >> 3, Au, [&](int i, int qx) { return Dp[qx + kQP * i]; },
           [&](int j, int qx, double v) { t1[j * kQP + qx] = v; });
  __syncthreads();
  double* out = T + size_t(c) * 3 * n1 * q2 + size_t(kz) * q2;
  auto AV = [&](int qy, int j) { return Vp[qy + kQP * j]; };
  auto B0 = [&](int j, int qx) { return t0[j * kQP + qx]; };
  qgemm<STRIP, 5>(kQP, kQP, n1k, 0, AV, B0, [&](int qy, int qx, double v) {
    if (qy < q && qx < q) out[qx + q * qy] = v;
  });
  qgemm<STRIP, 5>(kQP, kQP, n1k, kQP >> 3, [&](int qy, int j) { return Dp[qy + kQP * j]; }, B0, [&](int qy, int qx, double v) {
    if (qy < q && qx < q) out[size_t(n1) * q2 + qx + q * qy] = v;
  });
  qgemm<STRIP, 5>(kQP, kQP, n1k, 2 * (kQP >> 3), AV, [&](int j, int qx) { return t1[j * kQP + qx]; }, [&](int qy, int qx, double v) {
    if (qy < q && qx < q) out[2 * size_t(n1) * q2 + qx + q * qy] = v;
  });
}

// Stage 2: per (cell, qy): interpolate the three fields to the quadrature
// points along z, g = (V_z T2, V_z T1, D_z T0) = (du/dxi, du/deta, du/dzeta);
// f = w kappa G g with G = det J^{-1} J^{-T} of the trilinear map (Jacobian
// from the 8 cell corners, src/geometry.cpp:33-43); project back in place:
// T0 <- V_z^T f_x, T1 <- V_z^T f_y, T2 <- D_z^T f_z.
template <int STRIP>
__global__ void __launch_bounds__(256) k_quad_stage2(int n1, int q, double* __restrict__ T,
                                                      const double* __restrict__ Vq, const double* __restrict__ Dq,
                                                      const double* __restrict__ wq, const double* __restrict__ xyz,
                                                      const double* __restrict__ kappa,
                                                      const double* __restrict__ qpts) {
  extern __shared__ __align__(16) double sm[];
  const int n1p = pad8(n1), n1k = pad4(n1);
  double* Vp = sm;
  double* Dp = Vp + kQP * n1p;
  double* C = Dp + kQP * n1p;         // C[f][kz < n1k][qx] (stride kQP, zero padded)
  // g / f [field][qz][qx] (kQP x kQP, zero padded); STRIP == 3: over C (the z interpolation keeps its
  // outputs in registers until every warp has read C) -- 63 KB instead of 91 KB, three CTAs per SM
  double* G = STRIP == 3 ? C : C + 3 * n1k * kQP;
  double* W = STRIP == 3 ? C + max(3 * n1k * kQP, 3 * kQP * kQP) : G + 3 * kQP * kQP;  // q weights, q points
  double* X = W + 2 * q;              // 24 corner coordinates, X[3 b + r]
  double* J0 = X + 24;                // Jacobian tables [q][3] x 4
  double* J2 = J0 + 3 * q;
  double* AL = J2 + 3 * q;
  double* BE = AL + 3 * q;
  const int c = blockIdx.x / q, qy = blockIdx.x % q;
  const int q2 = q * q;
  load_vd_padded(Vp, Dp, Vq, Dq, q, n1, n1p);
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    W[i] = wq[i];
    W[q + i] = qpts[i];
  }
  for (int i = threadIdx.x; i < 24; i += blockDim.x) X[i] = xyz[size_t(c) * 24 + i];
  double* base = T + size_t(c) * 3 * n1 * q2 + size_t(qy) * q;
  staged_copy<8>(
      3 * n1k * kQP,
      [&](int i) {
        const int fk = i / kQP, qx = i - fk * kQP, f = fk / n1k, k = fk - f * n1k;
        return (qx < q && k < n1) ? base[size_t(f * n1 + k) * q2 + qx] : 0.0;
      },
      [&](int i, double v) { C[i] = v; });
  __syncthreads();
  // Jacobian columns of x = sum_b N_b(xi) X_b:  col0 depends on (xi_y, xi_z),
  // col2 on (xi_x, xi_y), col1 = h0(xi_z) al(xi_x) + h1(xi_z) be(xi_x).
  {
    const double ey = W[q + qy];
    const double hy[2] = {0.5 * (1.0 - ey), 0.5 * (1.0 + ey)};
    for (int i = threadIdx.x; i < q; i += blockDim.x) {
      const double t = W[q + i];
      const double h[2] = {0.5 * (1.0 - t), 0.5 * (1.0 + t)};
      for (int r = 0; r < 3; ++r) {
        double j0 = 0.0, j2 = 0.0, al = 0.0, be = 0.0;
        for (int u = 0; u < 2; ++u)
          for (int v = 0; v < 2; ++v) {
            j0 += hy[u] * h[v] * 0.5 * (X[3 * (1 + 2 * u + 4 * v) + r] - X[3 * (2 * u + 4 * v) + r]);
            j2 += h[u] * hy[v] * 0.5 * (X[3 * (u + 2 * v + 4) + r] - X[3 * (u + 2 * v) + r]);
          }
        for (int u = 0; u < 2; ++u) {
          al += h[u] * 0.5 * (X[3 * (u + 2) + r] - X[3 * u + r]);
          be += h[u] * 0.5 * (X[3 * (u + 6) + r] - X[3 * (u + 4) + r]);
        }
        J0[3 * i + r] = j0;
        J2[3 * i + r] = j2;
        AL[3 * i + r] = al;
        BE[3 * i + r] = be;
      }
    }
  }
  const int kq2 = kQP * kQP;
  auto AVz = [&](int qz, int k) { return Vp[qz + kQP * k]; };
  auto ADz = [&](int qz, int k) { return Dp[qz + kQP * k]; };
  auto BC2 = [&](int k, int qx) { return C[(2 * n1k + k) * kQP + qx]; };
  auto BC1 = [&](int k, int qx) { return C[(n1k + k) * kQP + qx]; };
  auto BC0 = [&](int k, int qx) { return C[k * kQP + qx]; };
  if constexpr (STRIP == 3) {
    // 3 x 5 strip tasks over the 8 warps (t = warp, warp + 8), results held in registers
    constexpr int NS = kQP / 8;
    const int warp = threadIdx.x >> 5;
    double dA[NS][2], dB[NS][2];
    auto run = [&](int t, double (&d)[NS][2]) {
      const int gm = t / NS, m0 = 8 * (t % NS);
      if (gm == 0)
        strip_compute<NS, 4>(m0, n1k, AVz, BC2, d);
      else if (gm == 1)
        strip_compute<NS, 4>(m0, n1k, AVz, BC1, d);
      else
        strip_compute<NS, 4>(m0, n1k, ADz, BC0, d);
    };
    auto put = [&](int t, const double (&d)[NS][2]) {
      const int gm = t / NS;
      strip_store<NS>(8 * (t % NS), d, [&](int qz, int qx, double v) { G[gm * kq2 + qz * kQP + qx] = v; });
    };
    for (int w0 = 0; w0 < 3 * NS; w0 += 16) {  // (blockDim.x = 256: one round)
      const int t0 = w0 + warp, t1 = w0 + warp + 8;
      if (t0 < 3 * NS) run(t0, dA);
      if (t1 < 3 * NS) run(t1, dB);
      __syncthreads();  // every warp has read C
      if (t0 < 3 * NS) put(t0, dA);
      if (t1 < 3 * NS) put(t1, dB);
    }
  } else {
    qgemm<STRIP, 5>(kQP, kQP, n1k, 0, AVz, BC2, [&](int qz, int qx, double v) { G[qz * kQP + qx] = v; });
    qgemm<STRIP, 5>(kQP, kQP, n1k, kQP >> 3, AVz, BC1, [&](int qz, int qx, double v) { G[kq2 + qz * kQP + qx] = v; });
    qgemm<STRIP, 5>(kQP, kQP, n1k, 2 * (kQP >> 3), ADz, BC0,
                    [&](int qz, int qx, double v) { G[2 * kq2 + qz * kQP + qx] = v; });
  }
  __syncthreads();
  const double kap = kappa[c], wy = W[qy];
  for (int pnt = threadIdx.x; pnt < kq2; pnt += blockDim.x) {
    const int qz = pnt / kQP, qx = pnt - qz * kQP;
    if (qz >= q || qx >= q) {
      G[pnt] = G[kq2 + pnt] = G[2 * kq2 + pnt] = 0.0;
      continue;
    }
    const double tz = W[q + qz];
    const double hz0 = 0.5 * (1.0 - tz), hz1 = 0.5 * (1.0 + tz);
    double J[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      J[r][0] = J0[3 * qz + r];
      J[r][1] = hz0 * AL[3 * qx + r] + hz1 * BE[3 * qx + r];
      J[r][2] = J2[3 * qx + r];
    }
    double adj[3][3];  // det * J^{-1}
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
        adj[i][j] = J[i1][j1] * J[i2][j2] - J[i1][j2] * J[i2][j1];
      }
    const double det = J[0][0] * adj[0][0] + J[0][1] * adj[1][0] + J[0][2] * adj[2][0];
    const double g[3] = {G[pnt], G[kq2 + pnt], G[2 * kq2 + pnt]};
    double hv[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) hv[r] = adj[0][r] * g[0] + adj[1][r] * g[1] + adj[2][r] * g[2];
    const double sc = W[qx] * wy * W[qz] * kap / det;
#pragma unroll
    for (int a2 = 0; a2 < 3; ++a2) G[a2 * kq2 + pnt] = sc * (adj[a2][0] * hv[0] + adj[a2][1] * hv[1] + adj[a2][2] * hv[2]);
  }
  __syncthreads();
  const int Kq = (q + 3) & ~3;  // projection over qz (rows >= q are zero)
  auto BVk = [&](int k, int qz) { return Vp[qz + kQP * k]; };
  qgemm<STRIP, 5>(n1p, kQP, Kq, 0, BVk, [&](int qz, int qx) { return G[qz * kQP + qx]; }, [&](int k, int qx, double v) {
    if (qx < q && k < n1) base[size_t(k) * q2 + qx] = v;
  });
  qgemm<STRIP, 5>(n1p, kQP, Kq, n1p >> 3, BVk, [&](int qz, int qx) { return G[kq2 + qz * kQP + qx]; }, [&](int k, int qx, double v) {
    if (qx < q && k < n1) base[size_t(n1 + k) * q2 + qx] = v;
  });
  qgemm<STRIP, 5>(n1p, kQP, Kq, 2 * (n1p >> 3), [&](int k, int qz) { return Dp[qz + kQP * k]; },
           [&](int qz, int qx) { return G[2 * kq2 + qz * kQP + qx]; }, [&](int k, int qx, double v) {
             if (qx < q && k < n1) base[size_t(2 * n1 + k) * q2 + qx] = v;
           });
}

// Stage 3: per (cell, kz): b0 = V_y^T T0, b12 = D_y^T T1 + V_y^T T2,
// E = D_x^T b0 + V_x^T b12.
template <int STRIP>
__global__ void __launch_bounds__(256) k_quad_stage3(int n1, int q, const double* __restrict__ T,
                                                      const double* __restrict__ Vq, const double* __restrict__ Dq,
                                                      double* __restrict__ E) {
  extern __shared__ __align__(16) double sm[];
  const int Kq = (q + 3) & ~3, n1p = pad8(n1);
  double* Vp = sm;
  double* Dp = Vp + kQP * n1p;
  double* P = Dp + kQP * n1p;        // 3 planes [f][qy < Kq][qx < kQP], zero padded
  // b0[j * kQP + qx], b12: STRIP == 3 keeps the y projections in registers until every warp has read
  // P and stores them over it (55 KB instead of 75 KB: more CTAs per SM)
  double* b0 = STRIP == 3 ? P : P + 3 * Kq * kQP;
  double* b12 = b0 + kQP * n1p;
  const int c = blockIdx.x / n1, kz = blockIdx.x % n1;
  const int q2 = q * q, pl = Kq * kQP;
  load_vd_padded(Vp, Dp, Vq, Dq, q, n1, n1p);
  const double* in = T + size_t(c) * 3 * n1 * q2 + size_t(kz) * q2;
  staged_copy<8>(
      3 * pl,
      [&](int i) {
        const int f = i / pl, e = i - f * pl, qy = e / kQP, qx = e - qy * kQP;
        return (qy < q && qx < q) ? in[size_t(f) * n1 * q2 + qy * q + qx] : 0.0;
      },
      [&](int i, double v) { P[i] = v; });
  __syncthreads();
  auto AV = [&](int j, int qy) { return Vp[qy + kQP * j]; };
  auto ADV = [&](int j, int k) { return k < Kq ? Dp[k + kQP * j] : Vp[k - Kq + kQP * j]; };
  auto BP0 = [&](int qy, int qx) { return P[qy * kQP + qx]; };
  auto BP12 = [&](int k, int qx) { return P[pl + k * kQP + qx]; };  // T1 rows then T2 rows (contiguous)
  if constexpr (STRIP == 3) {
    constexpr int NS = kQP / 8;
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, ns = n1p >> 3;
    for (int w0 = 0; w0 < 2 * ns; w0 += nw) {
      const int t = w0 + warp;
      double d[NS][2];
      if (t < ns)
        strip_compute<NS, 4>(8 * t, Kq, AV, BP0, d);
      else if (t < 2 * ns)
        strip_compute<NS, 4>(8 * (t - ns), 2 * Kq, ADV, BP12, d);
      __syncthreads();  // every warp has read P (one round at n1p = 32, 8 warps)
      if (t < ns)
        strip_store<NS>(8 * t, d, [&](int j, int qx, double v) { b0[j * kQP + qx] = v; });
      else if (t < 2 * ns)
        strip_store<NS>(8 * (t - ns), d, [&](int j, int qx, double v) { b12[j * kQP + qx] = v; });
    }
  } else {
    qgemm<STRIP, 5>(n1p, kQP, Kq, 0, AV, BP0, [&](int j, int qx, double v) { b0[j * kQP + qx] = v; });
    qgemm<STRIP, 5>(n1p, kQP, 2 * Kq, n1p >> 3, ADV, BP12, [&](int j, int qx, double v) { b12[j * kQP + qx] = v; });
  }
  __syncthreads();
  double* out = E + size_t(c) * n1 * n1 * n1 + size_t(kz) * n1 * n1;
  dgemm_tc(n1p, n1p, 2 * Kq, [&](int j, int k) { return k < Kq ? b0[j * kQP + k] : b12[j * kQP + k - Kq]; },
           [&](int k, int i) { return k < Kq ? Dp[k + kQP * i] : Vp[k - Kq + kQP * i]; },
           [&](int j, int i, double v) {
             if (i < n1 && j < n1) out[i + n1 * j] = v;
           });
}

// ---- p = 31 (n1 = 32), 3D: slab-blocked transform ------------------------------
// A 32^3 tile (256 KB) does not fit in shared memory, so the transform runs as
//   T1  per (cell, 8 z-slabs): gather (+ FDM interior rebuild for S), contract
//       x and y in shared memory (line passes as in the p = 15 kernels: thread
//       per 32-point line in registers, contracted index written slowest, two
//       passes cycle back), store the slabs to the E-vector;
//   T2  per (cell, 8 y-planes): thread per z-line straight from E into
//       registers, contract z, mode signs, interior elimination at the z- and
//       x-faces (x-face sums are warp reductions: lanes run along x), store;
//   T3  (S^T only) interior elimination at the y-faces, thread per y-line.
// Interior-mode diagonal D = sum_q mu_q prod_b (A~ | B~)_{x_b x_b} is formed
// from the 1D diagonals (separable), in the order of compute_invD.
constexpr int kL32 = 32, kSlab32 = 1024, kNpc32 = 32768;

__device__ __forceinline__ int pos32(int o) {
  return (o & ~31) | ((((o >> 1) & 15) ^ ((o >> 5) & 7)) << 1) | (o & 1);
}

__device__ __forceinline__ void load_line32(const double* __restrict__ b, int r, double (&x)[32]) {
  const double2* row = reinterpret_cast<const double2*>(b + 32 * r);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const double2 t = row[c ^ (r & 7)];
    x[2 * c] = t.x;
    x[2 * c + 1] = t.y;
  }
}

__device__ __forceinline__ double dot32(const double* __restrict__ Mrow, const double (&x)[32]) {
  const double2* m = reinterpret_cast<const double2*>(Mrow);
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const double2 mm = m[c];
    a0 = fma(mm.x, x[2 * c], a0);
    a1 = fma(mm.y, x[2 * c + 1], a1);
  }
  return a0 + a1;
}

// 1D tables of the FDM interior algebra: diagonals of A~ / B~, the face rows
// and columns of A~ (element (i, j) of the n1 x n1 column-major A~ is At[i + n1 j]).
struct Fdm32 {
  double ad[kL32], bd[kL32];  // A~_ii, B~_ii
  double ac0[kL32], acp[kL32];  // A~_{i,0}, A~_{i,p}   (rebuild)
  double ar0[kL32], arp[kL32];  // A~_{0,j}, A~_{p,j}   (elimination)
};

__device__ __forceinline__ void load_fdm32(Fdm32* t, const double* __restrict__ At, const double* __restrict__ Bt) {
  for (int i = threadIdx.x; i < kL32; i += blockDim.x) {
    t->ad[i] = At[i * (kL32 + 1)];
    t->bd[i] = Bt[i * (kL32 + 1)];
    t->ac0[i] = At[i];
    t->acp[i] = At[i + kL32 * (kL32 - 1)];
    t->ar0[i] = At[kL32 * i];
    t->arp[i] = At[kL32 - 1 + kL32 * i];
  }
}

__device__ __forceinline__ double diag32(const Fdm32& t, const double* mu, int x, int y, int z) {
  double s = 0.0;
  s += mu[0] * t.bd[z] * t.bd[y] * t.ad[x];
  s += mu[1] * t.bd[z] * t.ad[y] * t.bd[x];
  s += mu[2] * t.ad[z] * t.bd[y] * t.bd[x];
  return s;
}

__device__ __forceinline__ void load_rows32(double* __restrict__ Mt, const double* __restrict__ M) {
  for (int i = threadIdx.x; i < kL32 * kL32; i += blockDim.x) Mt[(i >> 5) + 32 * (i & 31)] = M[i];
}

template <int GB>  // gather batch: map loads, then value loads, GB per thread in flight
__global__ void __launch_bounds__(256, 2) k_cells_t1_32(int dir, int flags, const double* __restrict__ in,
                                                      const double* __restrict__ aux, const double* eaux,
                                                      double* __restrict__ E,
                                                      const int32_t* __restrict__ cdofs,
                                                      const double* __restrict__ inv_mult,
                                                      const uint8_t* __restrict__ cons,
                                                      const double* __restrict__ sign, const double* __restrict__ M,
                                                      const double* __restrict__ mu, const double* __restrict__ At,
                                                      const double* __restrict__ Bt, const double* __restrict__ nK) {
  extern __shared__ __align__(16) double sm[];
  double* Mt = sm;                    // 1024
  double* slab = Mt + kL32 * kL32;    // 8 x 1024, pos32 layout
  double* zf = slab + 8 * kSlab32;    // 2 x 1024 (z = 0, z = p face planes; rebuild only)
  Fdm32* t = reinterpret_cast<Fdm32*>(zf + 2 * kSlab32);
  const int c = blockIdx.x >> 2, z0 = 8 * (blockIdx.x & 3);
  const int tid = threadIdx.x;
  const bool recon = dir == 1 && (flags & 2);
  load_rows32(Mt, M);
  if (recon) load_fdm32(t, At, Bt);
  const int32_t* cd = cdofs + size_t(c) * kNpc32;
  // gather in batches of 8 per thread: all map loads first, then the independent
  // value loads (8 DRAM round trips in flight per thread instead of a chain)
#pragma unroll 1
  for (int h = 0; h < 32 / GB; ++h) {
    int gi[GB];
#pragma unroll
    for (int u = 0; u < GB; ++u) gi[u] = cd[z0 * kSlab32 + tid + 256 * (GB * h + u)];
    double v[GB];
#pragma unroll
    for (int u = 0; u < GB; ++u) {
      const int l = z0 * kSlab32 + tid + 256 * (GB * h + u), g = gi[u];
      const double xv = in[g];
      const double w = dir == 0 ? inv_mult[g] : (sign ? sign[size_t(c) * kNpc32 + l] : 1.0);
      v[u] = cons[g] ? 0.0 : xv * w;
    }
#pragma unroll
    for (int u = 0; u < GB; ++u) {
      const int i = tid + 256 * (GB * h + u);
      slab[(i & ~1023) + pos32(i & 1023)] = v[u];
    }
  }
  if (recon) {  // the z = 0 / z = p face planes, gathered 8 per thread with the loads in flight together
    int gi[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = tid + 256 * u;
      gi[u] = cd[(i >> 10) * (kL32 - 1) * kSlab32 + (i & 1023)];
    }
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = tid + 256 * u, l = (i >> 10) * (kL32 - 1) * kSlab32 + (i & 1023), g = gi[u];
      const double xv = in[g];
      const double w = sign ? sign[size_t(c) * kNpc32 + l] : 1.0;
      v[u] = cons[g] ? 0.0 : xv * w;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) zf[tid + 256 * u] = v[u];
  }
  __syncthreads();
  if (recon) {
    const double m[3] = {mu[size_t(c) * 3], mu[size_t(c) * 3 + 1], mu[size_t(c) * 3 + 2]};
    const double nk = nK[c];
    constexpr int pm = kL32 - 2, npts = 8 * pm * pm;
    // interior rebuild, 8 points per thread per batch: the aux gathers of a batch are
    // issued together (one dependent round trip per batch, not per point)
#pragma unroll 1
    for (int b0 = tid; b0 < npts; b0 += 256 * 8) {
      double av[8];
      {
        int ga[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = b0 + 256 * u, s = i / (pm * pm), z = z0 + s;
          const int y = 1 + (i / pm) % pm, x = 1 + i % pm;
          const bool in = i < npts && z > 0 && z < kL32 - 1;
          // flags & 4: aux is the cell-local E-vector of the S^T pass (the interior right-hand
          // side where that pass left it: no map load, contiguous reads; this CTA's slabs of E
          // are read here, before its own stores)
          ga[u] = !in ? -1 : (flags & 4) ? z * kSlab32 + x + 32 * y : cd[size_t(z) * kSlab32 + x + 32 * y];
        }
        const double* asrc = (flags & 4) ? eaux + size_t(c) * kNpc32 : aux;
#pragma unroll
        for (int u = 0; u < 8; ++u) av[u] = ga[u] >= 0 ? asrc[ga[u]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = b0 + 256 * u, s = i / (pm * pm), z = z0 + s;
        if (i >= npts || z == 0 || z == kL32 - 1) continue;
        const int y = 1 + (i / pm) % pm, x = 1 + i % pm;
        double* sl = slab + s * kSlab32;
        const int o = x + 32 * y;
        double v = nk * av[u];
        // faces along x, y (this slab) and z (the face planes), as recon_interior
        const double cx = m[0] * t->bd[y] * t->bd[z];
        v -= cx * (t->ac0[x] * sl[pos32(0 + 32 * y)] + t->acp[x] * sl[pos32(kL32 - 1 + 32 * y)]);
        const double cy = m[1] * t->bd[x] * t->bd[z];
        v -= cy * (t->ac0[y] * sl[pos32(x)] + t->acp[y] * sl[pos32(x + 32 * (kL32 - 1))]);
        const double cz = m[2] * t->bd[x] * t->bd[y];
        v -= cz * (t->ac0[z] * zf[o] + t->acp[z] * zf[kSlab32 + o]);
        sl[pos32(o)] = v * (1.0 / diag32(*t, m, x, y, z));
      }
    }
    __syncthreads();
  }
  // x and y line passes, warp w on slab w: OUT(k, line) = sum_j M(k, j) X(j, line) as a
  // 32 x 32 x 32 GEMM on the FP64 tensor pipe (DMMA m8n8k4; the 16 accumulator tiles in
  // registers, A fragments of M and B fragments of the slab read from shared memory once
  // per pass, OUT stored with the contracted index slowest so the second pass contracts y
  // and restores the order)
  double* sl = slab + (tid >> 5) * kSlab32;
  const int lane = tid & 31, lq = lane >> 2, lr = lane & 3;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    double d[4][4][2];  // [mt][nt] accumulators
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      double xb[4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) xb[nt] = sl[pos32(32 * (8 * nt + lq) + 4 * kt + lr)];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const double fa = Mt[32 * (8 * mt + lq) + 4 * kt + lr];  // A fragment M(8 mt + lq, 4 kt + lr)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(d[mt][nt][0], d[mt][nt][1], fa, xb[nt]);
      }
    }
    __syncwarp();  // the whole slab is read before it is overwritten
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        *reinterpret_cast<double2*>(sl + pos32(8 * nt + 2 * lr + 32 * (8 * mt + lq))) =
            make_double2(d[mt][nt][0], d[mt][nt][1]);
    __syncwarp();
  }
  __syncthreads();
  double* e = E + size_t(c) * kNpc32 + size_t(z0) * kSlab32;
  for (int i = tid; i < 8 * kSlab32; i += 256) e[i] = slab[(i & ~1023) + pos32(i & 1023)];
}

// z contraction, warp per y-plane of the cell: OUT(z', x) = sum_z M(z', z) U(z, x)
// as a 32 x 32 x 32 GEMM on the FP64 tensor pipe (DMMA m8n8k4): B fragments
// straight from the E-vector (lane: z = 4 kt + lane % 4, x = 8 nt + lane / 4),
// A fragments of M from shared memory, the 16 accumulator tiles in registers.
// Lane (lq, lr) then holds OUT(8 mt + lq, 8 nt + 2 lr + {0, 1}); the interior
// elimination sums run on these fragments: the x-face sums (over x, per z')
// reduce over the 4 lanes sharing lq, the z-face sums (over z', per x) over the
// 8 lanes sharing lr.  Mode signs and the z-face corrections are applied
// before the pairs are stored.
__global__ void __launch_bounds__(256, 2) k_cells_t2_32(int dir, int flags, double* __restrict__ E,
                                                         const double* __restrict__ sign, const double* __restrict__ M,
                                                         const double* __restrict__ mu, const double* __restrict__ At,
                                                         const double* __restrict__ Bt) {
  extern __shared__ __align__(16) double sm[];
  double* Mt = sm;  // 1024
  Fdm32* t = reinterpret_cast<Fdm32*>(Mt + kL32 * kL32);
  const int c = blockIdx.x >> 2;
  const int tid = threadIdx.x, lane = tid & 31, lq = lane >> 2, lr = lane & 3;
  const int y = 8 * (blockIdx.x & 3) + (tid >> 5);
  const bool schur = dir == 0 && (flags & 1);
  load_rows32(Mt, M);
  if (schur) load_fdm32(t, At, Bt);
  double* pl = E + size_t(c) * kNpc32 + 32 * y;  // plane y: element (z, x) at z * kSlab32 + x
  double d[4][4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
  __syncthreads();
#pragma unroll
  for (int kt = 0; kt < 8; ++kt) {
    double xb[4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) xb[nt] = pl[size_t(4 * kt + lr) * kSlab32 + 8 * nt + lq];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const double fa = Mt[32 * (8 * mt + lq) + 4 * kt + lr];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma884(d[mt][nt][0], d[mt][nt][1], fa, xb[nt]);
    }
  }
  __syncwarp();  // the plane is read before it is overwritten
  if (dir == 0 && sign) {
    const double* sg = sign + size_t(c) * kNpc32 + 32 * y;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) d[mt][nt][e] *= sg[size_t(8 * mt + lq) * kSlab32 + 8 * nt + 2 * lr + e];
  }
  if (schur) {
    const double m[3] = {mu[size_t(c) * 3], mu[size_t(c) * 3 + 1], mu[size_t(c) * 3 + 2]};
    const bool yi = y > 0 && y < kL32 - 1;
    double s0z[4][2], spz[4][2];  // z-face partial sums per (nt, e) column x
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) s0z[nt][0] = s0z[nt][1] = spz[nt][0] = spz[nt][1] = 0.0;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int z = 8 * mt + lq;
      const bool zi = z > 0 && z < kL32 - 1;
      double s0 = 0.0, sp = 0.0;  // x-face partial sums of this lane's 8 x values at z
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int x = 8 * nt + 2 * lr + e;
          const bool xi = x > 0 && x < kL32 - 1;
          const double w = (xi && yi && zi) ? d[mt][nt][e] * (1.0 / diag32(*t, m, x, y, z)) : 0.0;
          s0 = fma(t->ar0[x], w, s0);
          sp = fma(t->arp[x], w, sp);
          s0z[nt][e] = fma(t->ar0[z], w, s0z[nt][e]);
          spz[nt][e] = fma(t->arp[z], w, spz[nt][e]);
        }
      // x faces (e, y, z): over the 4 lanes sharing lq
      s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
      sp += __shfl_xor_sync(0xffffffffu, sp, 1);
      s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
      sp += __shfl_xor_sync(0xffffffffu, sp, 2);
      if (yi && zi) {
        const double cx = m[0] * t->bd[y] * t->bd[z];
        if (lr == 0) d[mt][0][0] -= cx * s0;   // x = 0
        if (lr == 3) d[mt][3][1] -= cx * sp;   // x = 31
      }
    }
    // z faces (x, y, e): over the 8 lanes sharing lr
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double a0 = s0z[nt][e], ap = spz[nt][e];
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          a0 += __shfl_xor_sync(0xffffffffu, a0, o);
          ap += __shfl_xor_sync(0xffffffffu, ap, o);
        }
        const int x = 8 * nt + 2 * lr + e;
        if (yi && x > 0 && x < kL32 - 1) {
          const double cz = m[2] * t->bd[x] * t->bd[y];
          if (lq == 0) d[0][nt][e] -= cz * a0;  // z = 0
          if (lq == 7) d[3][nt][e] -= cz * ap;  // z = 31
        }
      }
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
      *reinterpret_cast<double2*>(pl + size_t(8 * mt + lq) * kSlab32 + 8 * nt + 2 * lr) =
          make_double2(d[mt][nt][0], d[mt][nt][1]);
}

// y faces (x, e, z) for x, z interior: thread per y-line.
__global__ void __launch_bounds__(256) k_cells_t3_32(double* __restrict__ E, const double* __restrict__ mu,
                                                      const double* __restrict__ At, const double* __restrict__ Bt) {
  __shared__ Fdm32 t;
  const int c = blockIdx.x >> 2;
  const int tid = threadIdx.x, x = tid & 31, z = 8 * (blockIdx.x & 3) + (tid >> 5);
  load_fdm32(&t, At, Bt);
  __syncthreads();
  if (x == 0 || x == kL32 - 1 || z == 0 || z == kL32 - 1) return;
  const double m[3] = {mu[size_t(c) * 3], mu[size_t(c) * 3 + 1], mu[size_t(c) * 3 + 2]};
  double* row = E + size_t(c) * kNpc32 + size_t(z) * kSlab32 + x;
  double s0 = 0.0, sp = 0.0;
#pragma unroll 6
  for (int y = 1; y < kL32 - 1; ++y) {
    const double w = row[32 * y] * (1.0 / diag32(t, m, x, y, z));
    s0 = fma(t.ar0[y], w, s0);
    sp = fma(t.arp[y], w, sp);
  }
  const double cy = m[1] * t.bd[x] * t.bd[z];
  row[0] -= cy * s0;
  row[32 * (kL32 - 1)] -= cy * sp;
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
  const int Kq = (q + 3) & ~3, n1p = pad8(n1), n1k = pad4(n1);
  const size_t s1 = sizeof(double) * (4 * size_t(kQP) * n1p + size_t(n1k + 4) * n1p);
  const size_t s2 = sizeof(double) * (2 * size_t(kQP) * n1p + 3 * size_t(n1k) * kQP + 3 * size_t(kQP) * kQP + 2 * q + 24 +
                                      12 * size_t(q));
  const size_t s3 = sizeof(double) * (4 * size_t(kQP) * n1p + 3 * size_t(Kq) * kQP);
  if (q > kQP || s1 > 227 * 1024 || s2 > 227 * 1024 || s3 > 227 * 1024)
    throw Error(FDMGPU_UNSUPPORTED, "true-form quadrature operator: p too large");
  // FDMGPU_QUAD_STRIP (A/B switch; same sums, bitwise equal results):
  const char* senv = std::getenv("FDMGPU_QUAD_STRIP");
  // 0: 8 x 16 tasks (2.02 ms at C5) | 1, 2: row strips, k-loop unrolled by 2, 4 (1.81, 1.77 ms) | 3 (default): strips, and
  // stages 2 / 3 keep their intermediate over its input (63 / 55 KB: three CTAs per SM; 1.60 ms)
  const int strip = senv ? std::atoi(senv) : 3;
   // 1 | 2: k-loop unrolled by 2 | 4 (C5 residual 2.02 -> 1.81 | 1.77 ms)
  auto k1 = strip == 0 ? k_quad_stage1<0> : strip >= 2 ? k_quad_stage1<2> : k_quad_stage1<1>;
  auto k2 = strip == 0 ? k_quad_stage2<0> : strip == 3 ? k_quad_stage2<3> : strip == 2 ? k_quad_stage2<2> : k_quad_stage2<1>;
  auto k3 = strip == 0 ? k_quad_stage3<0> : strip == 3 ? k_quad_stage3<3> : strip == 2 ? k_quad_stage3<2> : k_quad_stage3<1>;
  FDM_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s1)));
  k1<<<c.ncells * n1, 256, s1, c.stream>>>(n1, q, x, c.cell_dofs.p, c.constrained.p, c.Vq.p, c.Dq.p, c.Qbuf.p);
  FDM_LAUNCH_CHECK(c);
  const size_t s2a = sizeof(double) * (2 * size_t(kQP) * n1p + std::max(3 * size_t(n1k) * kQP, 3 * size_t(kQP) * kQP) +
                                       2 * q + 24 + 12 * size_t(q));
  const size_t s2u = strip == 3 ? s2a : s2;
  FDM_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s2u)));
  k2<<<c.ncells * q, 256, s2u, c.stream>>>(n1, q, c.Qbuf.p, c.Vq.p, c.Dq.p, c.wq.p, c.xyz.p, c.kappa.p, c.qpts.p);
  FDM_LAUNCH_CHECK(c);
  const size_t s3a = sizeof(double) * (2 * size_t(kQP) * n1p + std::max(3 * size_t(Kq) * kQP, 2 * size_t(kQP) * n1p));
  const size_t s3u = strip == 3 ? s3a : s3;
  FDM_CUDA(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s3u)));
  k3<<<c.ncells * n1, 256, s3u, c.stream>>>(n1, q, c.Qbuf.p, c.Vq.p, c.Dq.p, c.E.p);
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

// p = 31 slab path (T1, T2, T3 above)
static void launch_cells_transform_32(Context& c, int dir, const double* in, int flags, const double* aux) {
  const double* M = dir == 0 ? c.St.p : c.S.p;
  const int32_t* cd = dir == 0 ? c.cell_dofs.p : c.cell_modes.p;
  // the face planes and FDM tables only for the interior rebuild (S with recon):
  // S^T fits three CTAs per SM
  const bool recon = dir == 1 && (flags & 2);
  const size_t s1 = sizeof(double) * (kL32 * kL32 + (recon ? 10 : 8) * kSlab32) + (recon ? sizeof(Fdm32) : 0);
  const size_t s2 = sizeof(double) * kL32 * kL32 + sizeof(Fdm32);
  const char* benv = std::getenv("FDMGPU_T1_BATCH");  // gathers in flight per thread: 8 | 16 (A/B)
  auto kt1 = benv && std::atoi(benv) == 16 ? k_cells_t1_32<16> : k_cells_t1_32<8>;
  FDM_CUDA(cudaFuncSetAttribute(kt1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s1)));
  KernelTimer timer(c, 2);
  kt1<<<c.ncells * 4, 256, s1, c.stream>>>(dir, flags, in, (flags & 4) ? nullptr : aux, (flags & 4) ? aux : nullptr, c.E.p, cd, c.inv_mult.p, c.constrained.p,
                                                     c.mode_sign.p, M, c.mu.p, c.At.p, c.Bt.p, c.nK.p);
  FDM_LAUNCH_CHECK(c);
  k_cells_t2_32<<<c.ncells * 4, 256, s2, c.stream>>>(dir, flags, c.E.p, c.mode_sign.p, M, c.mu.p, c.At.p, c.Bt.p);
  FDM_LAUNCH_CHECK(c);
  if (dir == 0 && (flags & 1)) {
    k_cells_t3_32<<<c.ncells * 4, 256, 0, c.stream>>>(c.E.p, c.mu.p, c.At.p, c.Bt.p);
    FDM_LAUNCH_CHECK(c);
  }
}

bool cells_slab32(const Context& c) { return !cells_fit_smem(c) && c.n1 == kL32 && c.dim == 3 && !c.force_staged; }

void launch_cells_transform(Context& c, int dir, const double* in, int flags, const double* aux) {
  if (cells_fit_smem(c))
    launch_cells_transform_fused(c, dir, in, flags, aux);
  else if (c.n1 == kL32 && c.dim == 3 && !c.force_staged)
    launch_cells_transform_32(c, dir, in, flags, aux);
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
