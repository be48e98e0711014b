// Cell-local sum-factorised kernels (K1 basis transform, K4 stiffness apply)
// and the deterministic owner-gather that assembles cell contributions into
// global DOF vectors.
//
//   K1  apply_St / apply_S   <- src/assembly.cpp:308-342 (+ apply_axis, src/kron.cpp:20-38)
//   K4  GlobalOperator::apply, Cartesian Kronecker cells
//                            <- src/assembly.cpp:56-88, 143-154, src/kron.cpp:40-55
//
// One CTA per cell; the (p+1)^d tile lives in shared memory and each 1D
// contraction is one pass "thread per output" whose lane mapping is
// bank-conflict free for every axis (axis 0: lanes share the line and read
// it by broadcast; axes >= 1: lanes read consecutive doubles).  Results go
// to a cell-local E-vector; k_gather then sums each global DOF's cell
// contributions in ascending cell order (the reference's scatter_add order),
// so there are no FP64 atomics and results are run-to-run deterministic.
//
// FDM-interior fusion (used inside the relaxation).  In the FDM basis a
// cell-interior mode x of cell K couples only to itself (D^K_x = A~_xx) and
// to the facet modes of K that share its tangential indices.  Every vertex
// star containing a facet mode contains both cells adjacent to it, so
//   * the interior-elimination part of each patch's right-hand side,
//     b_f - sum_{K ∋ f} sum_x A~^K_fx b_x / D^K_x, is the same for every patch:
//     the S^T kernel subtracts its cell's share at the facet points (SCHUR);
//   * the patch-summed interior correction is
//     z_x = (n_K b_x - sum_{faces (a,e) of K} A~^K_{x,f(a,e,x)} z_f) / D^K_x,
//     with z_f the patch-summed facet correction and n_K the number of stars
//     containing K: the S kernel rebuilds it before contracting (RECON).
// The patch kernel is then left with the separator solve only.
#include "common.cuh"

namespace fdmgpu {

namespace {

enum : int { kSchur = 1, kRecon = 2 };

// out[.., k, ..] = alpha * sum_j M1[k + n1 j] in1[.., j, ..] (+ beta * same with M2/in2).
// N1C > 0 makes the tile edge a compile-time constant (index math becomes
// shifts / multiplies and the j loop unrolls); N1C = 0 is the generic path.
template <int N1C>
__device__ __forceinline__ void contract(int n1_rt, int npc, int axis, const double* __restrict__ M1,
                                         const double* __restrict__ in1, double alpha, const double* __restrict__ M2,
                                         const double* __restrict__ in2, double beta, double* __restrict__ out) {
  const int n1 = N1C > 0 ? N1C : n1_rt;
  const int stride = axis == 0 ? 1 : (axis == 1 ? n1 : n1 * n1);
  for (int o = threadIdx.x; o < npc; o += blockDim.x) {
    const int k = (o / stride) % n1;
    const int base = o - k * stride;
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int j = 0; j < (N1C > 0 ? N1C : 64); ++j) {
      if (N1C == 0 && j >= n1) break;
      s1 = fma(M1[k + n1 * j], in1[base + j * stride], s1);
      if (M2) s2 = fma(M2[k + n1 * j], in2[base + j * stride], s2);
    }
    out[o] = M2 ? alpha * s1 + beta * s2 : alpha * s1;
  }
}

struct PosId {
  __device__ __forceinline__ int operator()(int o) const { return o; }
};

// Shared-memory layout of the line-blocked n1 = 16 kernels: 16-double rows
// with their 16-byte chunks XOR-swizzled by the row index, so a thread
// reading a whole row (4 x double2 per 8 lanes) and 16 threads writing one
// element each of a row are both bank-conflict free.
// Element o of a 16^3 tile (axis 0 fastest) -> shared-memory slot: the
// double pair (o >> 1) & 7 within each 16-double row is XORed with
// (row ^ row >> 4) & 7, so both DMMA fragment accesses of the line passes are
// conflict-free: reading 8 consecutive rows x 4 columns, and writing double
// pairs of 8 rows 16 apart (the contracted index becomes the slowest).
struct Pos16 {
  __device__ __forceinline__ int operator()(int o) const {
    return (o & ~15) | ((((o >> 1) & 7) ^ (((o >> 4) ^ (o >> 8)) & 7)) << 1) | (o & 1);
  }
};

struct CellFdm {
  int dim, n1, p, ni;     // ni = (p-1)^dim interior points
  const double* At;       // shared-memory copies, (p+1)^2 column-major
  const double* Bt;
  double mu[3];
  double* invD;           // ni
};

// lattice index of interior point number ii (each coordinate in 1..p-1)
template <int N1C>
__device__ __forceinline__ int interior_lat(const CellFdm& f, int ii, int* x) {
  const int n1 = N1C > 0 ? N1C : f.n1;
  const int pm = n1 - 2;
  int lin = 0, stride = 1;
  for (int a = 0; a < f.dim; ++a, stride *= n1) {
    x[a] = 1 + ii % pm;
    ii /= pm;
    lin += x[a] * stride;
  }
  return lin;
}

template <int N1C>
__device__ void compute_invD(const CellFdm& f) {
  for (int ii = threadIdx.x; ii < f.ni; ii += blockDim.x) {
    int x[3];
    interior_lat<N1C>(f, ii, x);
    double s = 0.0;
    for (int q = 0; q < f.dim; ++q) {
      double prod = f.mu[q];
      for (int b = f.dim - 1; b >= 0; --b) prod *= (b == q ? f.At : f.Bt)[x[b] * (f.n1 + 1)];
      s += prod;
    }
    f.invD[ii] = 1.0 / s;
  }
}

// 1 / D_x from the interior point's coordinates (same product order as compute_invD);
// used when f.invD is null (the p = 15 kernels keep the table out of shared memory).
__device__ __forceinline__ double inv_diag(const CellFdm& f, const int* x) {
  double s = 0.0;
  for (int q = 0; q < f.dim; ++q) {
    double prod = f.mu[q];
    for (int b = f.dim - 1; b >= 0; --b) prod *= (b == q ? f.At : f.Bt)[x[b] * (f.n1 + 1)];
    s += prod;
  }
  return 1.0 / s;
}

// u[facet point] -= sum_x A~_{f x} u[x] / D_x for the 2 dim faces of the cell.
template <int N1C, class Pos = PosId>
__device__ void schur_faces(const CellFdm& f, double* u, Pos P = Pos()) {
  const int n1c = N1C > 0 ? N1C : f.n1;
  const int pm = n1c - 2;
  int nt = 1;
  for (int a = 1; a < f.dim; ++a) nt *= pm;
  for (int idx = threadIdx.x; idx < 2 * f.dim * nt; idx += blockDim.x) {
    const int face = idx / nt, a = face >> 1, e = (face & 1) ? f.p : 0;
    int t = idx % nt;
    int x[3] = {0, 0, 0};
    double coef = f.mu[a];
    for (int b = 0; b < f.dim; ++b) {
      if (b == a) continue;
      x[b] = 1 + t % pm;
      t /= pm;
      coef *= f.Bt[x[b] * (f.n1 + 1)];
    }
    int stride_a = 1, lin0 = 0, ii0 = 0, istride_a = 1;
    for (int b = 0, s = 1, is = 1; b < f.dim; ++b, s *= n1c, is *= pm) {
      if (b == a) {
        stride_a = s;
        istride_a = is;
      } else {
        lin0 += x[b] * s;
        ii0 += (x[b] - 1) * is;
      }
    }
    double acc = 0.0;
#pragma unroll
    for (int xa = 1; xa < (N1C > 0 ? N1C - 1 : 64); ++xa) {
      if (N1C == 0 && xa >= f.p) break;
      double id;
      if (f.invD) {
        id = f.invD[ii0 + (xa - 1) * istride_a];
      } else {
        x[a] = xa;
        id = inv_diag(f, x);
      }
      acc = fma(f.At[e + n1c * xa] * u[P(lin0 + xa * stride_a)], id, acc);
    }
    u[P(lin0 + e * stride_a)] -= coef * acc;
  }
}

// u[x] = (nK * b[x] - sum_{a, e} A~_{x, f(a,e)} u[f(a,e)]) / D_x for every interior x.
template <int N1C, class Pos = PosId>
__device__ void recon_interior(const CellFdm& f, double* u, const double* __restrict__ rb,
                               const int32_t* __restrict__ cd, double nK, Pos P = Pos()) {
  for (int ii = threadIdx.x; ii < f.ni; ii += blockDim.x) {
    int x[3];
    const int lin = interior_lat<N1C>(f, ii, x);
    double v = nK * rb[cd[lin]];
    for (int a = 0, s = 1; a < f.dim; ++a, s *= f.n1) {
      double coef = f.mu[a];
      for (int b = 0; b < f.dim; ++b)
        if (b != a) coef *= f.Bt[x[b] * (f.n1 + 1)];
      const int base = lin - x[a] * s;
      const double fsum = f.At[x[a] + f.n1 * 0] * u[P(base)] + f.At[x[a] + f.n1 * f.p] * u[P(base + f.p * s)];
      v -= coef * fsum;
    }
    u[P(lin)] = v * (f.invD ? f.invD[ii] : inv_diag(f, x));
  }
}

__device__ void load_cell_fdm(CellFdm& f, double* smem_tables, int dim, int n1, int c, const double* __restrict__ mu,
                              const double* __restrict__ At, const double* __restrict__ Bt) {
  f.dim = dim;
  f.n1 = n1;
  f.p = n1 - 1;
  f.ni = 1;
  for (int a = 0; a < dim; ++a) f.ni *= f.p - 1;
  double* at = smem_tables;
  double* bt = at + n1 * n1;
  for (int i = threadIdx.x; i < n1 * n1; i += blockDim.x) {
    at[i] = At[i];
    bt[i] = Bt[i];
  }
  f.At = at;
  f.Bt = bt;
  for (int a = 0; a < 3; ++a) f.mu[a] = a < dim ? mu[size_t(c) * dim + a] : 0.0;
  f.invD = bt + n1 * n1;
}

template <int N1C>
__global__ void k_cells_transform(int dim, int n1, int npc, int dir, int flags, const double* __restrict__ in,
                                  const double* __restrict__ aux, double* __restrict__ E,
                                  const int32_t* __restrict__ cdofs, const double* __restrict__ inv_mult,
                                  const uint8_t* __restrict__ cons, const double* __restrict__ sign,
                                  const double* __restrict__ M, const double* __restrict__ mu,
                                  const double* __restrict__ At, const double* __restrict__ Bt,
                                  const double* __restrict__ nK) {
  extern __shared__ double sm[];
  double* Ms = sm;
  double* b0 = Ms + n1 * n1;
  double* b1 = b0 + npc;
  double* tables = b1 + npc;  // At, Bt, invD (only with flags)
  const int c = blockIdx.x;
  for (int i = threadIdx.x; i < n1 * n1; i += blockDim.x) Ms[i] = M[i];
  CellFdm f;
  if (flags) load_cell_fdm(f, tables, dim, n1, c, mu, At, Bt);
  const int32_t* cd = cdofs + size_t(c) * npc;
  for (int l = threadIdx.x; l < npc; l += blockDim.x) {
    const int g = cd[l];
    double v = cons[g] ? 0.0 : in[g];
    if (dir == 0)
      v *= inv_mult[g];
    else if (sign)
      v *= sign[size_t(c) * npc + l];
    b0[l] = v;
  }
  __syncthreads();
  if (flags) {
    compute_invD<N1C>(f);
    __syncthreads();
  }
  if (flags & kRecon) {
    recon_interior<N1C>(f, b0, aux, cd, nK[c]);
    __syncthreads();
  }
  double* src = b0;
  double* dst = b1;
  for (int a = 0; a < dim; ++a) {
    contract<N1C>(n1, npc, a, Ms, src, 1.0, nullptr, nullptr, 0.0, dst);
    __syncthreads();
    double* t = src;
    src = dst;
    dst = t;
  }
  if (dir == 0 && sign) {
    for (int l = threadIdx.x; l < npc; l += blockDim.x) src[l] *= sign[size_t(c) * npc + l];
    __syncthreads();
  }
  if (flags & kSchur) {
    schur_faces<N1C>(f, src);
    __syncthreads();
  }
  double* e = E + size_t(c) * npc;
  for (int l = threadIdx.x; l < npc; l += blockDim.x) e[l] = src[l];
}

// PatchSolver-only helpers on modal vectors (FDMGPU_OP_PATCH):
// E = -(cell share of the interior elimination) at facet points, 0 elsewhere.
__global__ void k_cells_schur(int dim, int n1, int npc, const double* __restrict__ in, double* __restrict__ E,
                              const int32_t* __restrict__ cdofs, const uint8_t* __restrict__ cons,
                              const double* __restrict__ mu, const double* __restrict__ At,
                              const double* __restrict__ Bt) {
  extern __shared__ double sm[];
  double* u = sm;
  double* tables = u + npc;
  const int c = blockIdx.x;
  CellFdm f;
  load_cell_fdm(f, tables, dim, n1, c, mu, At, Bt);
  const int32_t* cd = cdofs + size_t(c) * npc;
  for (int l = threadIdx.x; l < npc; l += blockDim.x) {
    const int g = cd[l];
    u[l] = cons[g] ? 0.0 : in[g];
  }
  __syncthreads();
  compute_invD<0>(f);
  __syncthreads();
  // keep the interior values, zero everything else, then subtract at facets
  for (int l = threadIdx.x; l < npc; l += blockDim.x) {
    bool interior = true;
    for (int a = 0, r = l; a < dim; ++a, r /= n1) interior = interior && (r % n1 != 0) && (r % n1 != n1 - 1);
    if (!interior) u[l] = 0.0;
  }
  __syncthreads();
  schur_faces<0>(f, u);
  __syncthreads();
  double* e = E + size_t(c) * npc;
  for (int l = threadIdx.x; l < npc; l += blockDim.x) {
    bool interior = true;
    for (int a = 0, r = l; a < dim; ++a, r /= n1) interior = interior && (r % n1 != 0) && (r % n1 != n1 - 1);
    e[l] = interior ? 0.0 : u[l];
  }
}

// Writes the reconstructed interior modes of every cell into z (in place).
__global__ void k_cells_recon(int dim, int n1, int npc, double* __restrict__ z, const double* __restrict__ rb,
                              const int32_t* __restrict__ cdofs, const double* __restrict__ mu,
                              const double* __restrict__ At, const double* __restrict__ Bt,
                              const double* __restrict__ nK) {
  extern __shared__ double sm[];
  double* u = sm;
  double* tables = u + npc;
  const int c = blockIdx.x;
  CellFdm f;
  load_cell_fdm(f, tables, dim, n1, c, mu, At, Bt);
  const int32_t* cd = cdofs + size_t(c) * npc;
  for (int l = threadIdx.x; l < npc; l += blockDim.x) u[l] = z[cd[l]];
  __syncthreads();
  compute_invD<0>(f);
  __syncthreads();
  recon_interior<0>(f, u, rb, cd, nK[c]);
  __syncthreads();
  for (int ii = threadIdx.x; ii < f.ni; ii += blockDim.x) {
    int x[3];
    const int lin = interior_lat<0>(f, ii, x);
    z[cd[lin]] = u[lin];
  }
}

// Cartesian stiffness: y_K = sum_a mu_a (A on axis a, B elsewhere) u_K.
template <int N1C>
__global__ void k_cells_stiffness(int dim, int n1, int npc, const double* __restrict__ x, double* __restrict__ E,
                                  const int32_t* __restrict__ cdofs, const uint8_t* __restrict__ cons,
                                  const double* __restrict__ mu, const double* __restrict__ Ahat,
                                  const double* __restrict__ Bhat) {
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = As + n1 * n1;
  double* u = Bs + n1 * n1;
  double* t0 = u + npc;
  double* t1 = t0 + npc;
  double* q = t1 + npc;
  const int c = blockIdx.x;
  for (int i = threadIdx.x; i < n1 * n1; i += blockDim.x) {
    As[i] = Ahat[i];
    Bs[i] = Bhat[i];
  }
  const int32_t* cd = cdofs + size_t(c) * npc;
  for (int l = threadIdx.x; l < npc; l += blockDim.x) {
    const int g = cd[l];
    u[l] = cons[g] ? 0.0 : x[g];
  }
  const double m0 = mu[size_t(c) * dim], m1 = mu[size_t(c) * dim + 1], m2 = dim == 3 ? mu[size_t(c) * dim + 2] : 0.0;
  __syncthreads();
  contract<N1C>(n1, npc, 0, Bs, u, 1.0, nullptr, nullptr, 0.0, t0);  // B_x u
  contract<N1C>(n1, npc, 0, As, u, 1.0, nullptr, nullptr, 0.0, t1);  // A_x u
  __syncthreads();
  double* e = E + size_t(c) * npc;
  if (dim == 2) {
    // mu0 B_y A_x u + mu1 A_y B_x u
    contract<N1C>(n1, npc, 1, Bs, t1, m0, As, t0, m1, u);
    __syncthreads();
    for (int l = threadIdx.x; l < npc; l += blockDim.x) e[l] = u[l];
    return;
  }
  // P = mu0 B_y A_x u + mu1 A_y B_x u  (into u),  Q = B_y B_x u
  contract<N1C>(n1, npc, 1, Bs, t1, m0, As, t0, m1, u);
  contract<N1C>(n1, npc, 1, Bs, t0, 1.0, nullptr, nullptr, 0.0, q);
  __syncthreads();
  // y = B_z P + mu2 A_z Q
  contract<N1C>(n1, npc, 2, Bs, u, 1.0, As, q, m2, t0);
  __syncthreads();
  for (int l = threadIdx.x; l < npc; l += blockDim.x) e[l] = t0[l];
}

// ---- n1 = 16, dim = 3 kernels (p = 15: C3, C4) -----------------------------------
// Every 1D contraction is a pass over the 256 lines of the current fastest
// axis, run as the GEMM OUT(16 x 256) = M(16 x 16) X(16 x 256) on the FP64
// tensor pipe (DMMA m8n8k4): warp w owns lines 32w .. 32w+31 (4 n-tiles), M
// is held as A fragments in registers for the whole kernel, the warp's X
// fragments are read once per pass, and OUT(k, r) is written to element
// r + 256 k, i.e. the contracted index becomes the slowest one, so three
// passes cycle the axes back to the original order, in place (one 32 KB
// buffer per field).
constexpr int kL16 = 16, kNpc16 = 4096, kLines16 = 256;

// Mt[j + 16 k] = M[k + 16 j]: row k of M contiguous
__device__ __forceinline__ void load_rows16(double* __restrict__ Mt, const double* __restrict__ M) {
  for (int i = threadIdx.x; i < kL16 * kL16; i += blockDim.x) Mt[(i >> 4) + 16 * (i & 15)] = M[i];
}

struct MFrag16 {
  double a[2][4];  // [m-tile][k-tile]: M(8 mt + lane / 4, 4 kt + lane % 4)
};
__device__ __forceinline__ void mfrag16(MFrag16& f, const double* __restrict__ Mt) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) f.a[mt][kt] = Mt[16 * (8 * mt + (lane >> 2)) + 4 * kt + (lane & 3)];
}
// X fragments of the warp's 32 lines: X(4 kt + lane % 4, line 8 nt + lane / 4)
__device__ __forceinline__ void xfrag16(const double* __restrict__ b, double (&x)[4][4]) {
  const Pos16 P;
  const int lane = threadIdx.x & 31, r0 = 32 * (threadIdx.x >> 5) + (lane >> 2);
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) x[kt][nt] = b[P(16 * (r0 + 8 * nt) + 4 * kt + (lane & 3))];
}
// OUT(8 mt + lane / 4, lines 8 nt + 2 (lane % 4) + {0, 1}) -> elements r + 256 k
__device__ __forceinline__ void store16(double* __restrict__ b, int mt, int nt, double d0, double d1) {
  const Pos16 P;
  const int lane = threadIdx.x & 31;
  const int k = 8 * mt + (lane >> 2), r = 32 * (threadIdx.x >> 5) + 8 * nt + 2 * (lane & 3);
  *reinterpret_cast<double2*>(b + P(r + kLines16 * k)) = make_double2(d0, d1);
}

__global__ void __launch_bounds__(kLines16, 4) k_cells_transform16(int dir, int flags, const double* __restrict__ in,
                                                                 const double* __restrict__ aux, double* __restrict__ E,
                                                                 const int32_t* __restrict__ cdofs,
                                                                 const double* __restrict__ inv_mult,
                                                                 const uint8_t* __restrict__ cons,
                                                                 const double* __restrict__ sign,
                                                                 const double* __restrict__ M, const double* __restrict__ mu,
                                                                 const double* __restrict__ At,
                                                                 const double* __restrict__ Bt,
                                                                 const double* __restrict__ nK) {
  extern __shared__ __align__(16) double sm[];
  double* Mt = sm;               // 256
  double* b = Mt + kL16 * kL16;  // 4096, Pos16 layout
  double* tables = b + kNpc16;   // At, Bt (only with flags; 1/D computed on the fly)
  const Pos16 P;
  const int c = blockIdx.x, r = threadIdx.x;
  pdl_trigger();
  load_rows16(Mt, M);
  CellFdm f;
  if (flags) {
    load_cell_fdm(f, tables, 3, kL16, c, mu, At, Bt);
    f.invD = nullptr;
  }
  const int32_t* cd = cdofs + size_t(c) * kNpc16;
  pdl_wait();  // `in` / `aux` come from the previous kernel
  // gather: all map loads first, then the independent value loads (no branch on
  // the constraint flag, so in[g], cons[g] and the weight load in parallel)
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    int gi[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) gi[u] = cd[r + kLines16 * (8 * h + u)];
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int l = r + kLines16 * (8 * h + u), g = gi[u];
      const double xv = in[g];
      const double w = dir == 0 ? inv_mult[g] : (sign ? sign[size_t(c) * kNpc16 + l] : 1.0);
      v[u] = cons[g] ? 0.0 : xv * w;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) b[P(r + kLines16 * (8 * h + u))] = v[u];
  }
  __syncthreads();
  if (flags & kRecon) {
    recon_interior<kL16>(f, b, aux, cd, nK[c], P);
    __syncthreads();
  }
  MFrag16 fm;
  mfrag16(fm, Mt);
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    double x[4][4];
    xfrag16(b, x);
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) dmma884(d0, d1, fm.a[mt][kt], x[kt][nt]);
        store16(b, mt, nt, d0, d1);
      }
    __syncthreads();
  }
  if (dir == 0 && sign) {
    for (int l = r; l < kNpc16; l += kLines16) b[P(l)] *= sign[size_t(c) * kNpc16 + l];
    __syncthreads();
  }
  if (flags & kSchur) {
    schur_faces<kL16>(f, b, P);
    __syncthreads();
  }
  double* e = E + size_t(c) * kNpc16;
  for (int l = r; l < kNpc16; l += kLines16) e[l] = b[P(l)];
}

// Cartesian stiffness y_K = mu0 Bz By Ax u + mu1 Bz Ay Bx u + mu2 Az By Bx u in
// three line passes over two in-place buffers:
//   (Bx u, Ax u) -> (P = mu0 By Ax u + mu1 Ay Bx u, Q = By Bx u) -> y = Bz P + mu2 Az Q.
__global__ void __launch_bounds__(kLines16, 2) k_cells_stiffness16(const double* __restrict__ x, double* __restrict__ E,
                                                                 const int32_t* __restrict__ cdofs,
                                                                 const uint8_t* __restrict__ cons,
                                                                 const double* __restrict__ mu,
                                                                 const double* __restrict__ Ahat,
                                                                 const double* __restrict__ Bhat) {
  extern __shared__ __align__(16) double sm[];
  double* As = sm;              // rows of A
  double* Bs = As + kL16 * kL16;
  double* b0 = Bs + kL16 * kL16;
  double* b1 = b0 + kNpc16;
  const Pos16 P;
  const int c = blockIdx.x, r = threadIdx.x;
  pdl_trigger();
  // static data (1D matrices, the cell map, mu) before the wait for x: with
  // programmatic dependent launch this overlaps the previous kernel's tail
  load_rows16(As, Ahat);
  load_rows16(Bs, Bhat);
  const int32_t* cd = cdofs + size_t(c) * kNpc16;
  int gi[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) gi[u] = cd[r + kLines16 * u];
  pdl_wait();  // x comes from the previous kernel
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    if (h)
#pragma unroll
      for (int u = 0; u < 8; ++u) gi[u] = cd[r + kLines16 * (8 + u)];
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double xv = x[gi[u]];
      v[u] = cons[gi[u]] ? 0.0 : xv;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) b0[P(r + kLines16 * (8 * h + u))] = v[u];
  }
  const double m0 = mu[size_t(c) * 3], m1 = mu[size_t(c) * 3 + 1], m2 = mu[size_t(c) * 3 + 2];
  __syncthreads();
  MFrag16 fa, fb;
  mfrag16(fa, As);
  mfrag16(fb, Bs);
  {  // (Bx u, Ax u)
    double x[4][4];
    xfrag16(b0, x);
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) {
          dmma884(p0, p1, fb.a[mt][kt], x[kt][nt]);
          dmma884(q0, q1, fa.a[mt][kt], x[kt][nt]);
        }
        store16(b0, mt, nt, p0, p1);
        store16(b1, mt, nt, q0, q1);
      }
    __syncthreads();
  }
  {  // (P = mu0 By Ax u + mu1 Ay Bx u, Q = By Bx u)
    double t0[4][4], t1[4][4];
    xfrag16(b0, t0);
    xfrag16(b1, t1);
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) {
          dmma884(p0, p1, m0 * fb.a[mt][kt], t1[kt][nt]);
          dmma884(p0, p1, m1 * fa.a[mt][kt], t0[kt][nt]);
          dmma884(q0, q1, fb.a[mt][kt], t0[kt][nt]);
        }
        store16(b0, mt, nt, p0, p1);
        store16(b1, mt, nt, q0, q1);
      }
    __syncthreads();
  }
  {  // y = Bz P + mu2 Az Q
    double pp[4][4], qq[4][4];
    xfrag16(b0, pp);
    xfrag16(b1, qq);
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double y0 = 0.0, y1 = 0.0;
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) {
          dmma884(y0, y1, fb.a[mt][kt], pp[kt][nt]);
          dmma884(y0, y1, m2 * fa.a[mt][kt], qq[kt][nt]);
        }
        store16(b0, mt, nt, y0, y1);
      }
    __syncthreads();
  }
  double* e = E + size_t(c) * kNpc16;
  for (int l = r; l < kNpc16; l += kLines16) e[l] = b0[P(l)];
}

// ---- vector elasticity, n1 = 16, dim = 3 (kernels/elastic.cu has the generic path) ----
// elasticity_primal_operator's Kronecker blocks (src/elasticity.cpp:83-119) on
// the FP64 tensor pipe with the line-pass scheme above.  Output component i
// accumulates in registers: every third pass leaves its result in the same
// fragment positions (element r + 256 k of the original lattice order), so
// y_i never touches shared memory and is stored once.  Per (i, j) block the
// input tile x_j is gathered into b0 and run through three passes over two
// buffers: the diagonal block as k_cells_stiffness16 with mu'_a = c_ia mu_a;
// a cross block's two terms (C on i, C^T on j | C^T on i, C on j; B on the
// third axis k) share the B pass when it comes first (k = 0) or combine before
// the last pass when it comes last (k = 2).
__device__ __forceinline__ void gather16(double* __restrict__ b, const double* __restrict__ x,
                                         const int32_t* __restrict__ cd, const uint8_t* __restrict__ cons,
                                         int64_t off) {
  const Pos16 P;
  const int r = threadIdx.x;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    int64_t gi[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) gi[u] = cd[r + kLines16 * (8 * h + u)] + off;
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double xv = x[gi[u]];
      v[u] = cons[gi[u]] ? 0.0 : xv;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) b[P(r + kLines16 * (8 * h + u))] = v[u];
  }
}

// Rows of a 16 x 16 matrix at a padded stride of 20 doubles: the A-fragment
// loads (8 rows x 4 columns per warp) of the per-pass fragment reloads are
// then conflict-free (row starts 20 words apart cover all 16 bank pairs).
constexpr int kRow20 = 20, kMat20 = 16 * kRow20;
__device__ __forceinline__ void load_rows20(double* __restrict__ Mt, const double* __restrict__ M, bool transpose) {
  for (int i = threadIdx.x; i < kL16 * kL16; i += blockDim.x) {
    const int r = i & 15, c = i >> 4;  // M column-major: M(r, c) = M[r + 16 c]
    Mt[(transpose ? c : r) * kRow20 + (transpose ? r : c)] = M[i];
  }
}
__device__ __forceinline__ void mfrag20(MFrag16& f, const double* __restrict__ Mt) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) f.a[mt][kt] = Mt[kRow20 * (8 * mt + (lane >> 2)) + 4 * kt + (lane & 3)];
}

// OUT = a * M . T (one product per output tile)
__device__ __forceinline__ void mm16(double& d0, double& d1, const MFrag16& f, double a, const double (&t)[4][4],
                                     int mt, int nt) {
#pragma unroll
  for (int kt = 0; kt < 4; ++kt) dmma884(d0, d1, a * f.a[mt][kt], t[kt][nt]);
}

// Cross block (i, j) with B on axis K, accumulated into acc: three passes
// (axis 0, 1, 2) over b0 / b1; Ms holds the rows of A, B, C, C^T.
template <int K>
__device__ __forceinline__ void elastic_cross16(const double* __restrict__ Ms, double* __restrict__ b0,
                                                double* __restrict__ b1, int i, int j, double al, double be,
                                                double (&acc)[2][4][2]) {
  // factor of term 1 (C on i, C^T on j) / term 2 (C^T on i, C on j) on axis a; B = 1, C = 2, C^T = 3
  auto f1 = [&](int a) { return a == i ? 2 : (a == j ? 3 : 1); };
  auto f2 = [&](int a) { return a == i ? 3 : (a == j ? 2 : 1); };
  {  // pass 1 (axis 0): K = 0 -> B x once, else (F1_0 x, F2_0 x)
    double t[4][4];
    xfrag16(b0, t);
    __syncthreads();
    MFrag16 g;
    mfrag20(g, Ms + kMat20 * f1(0));
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double p0 = 0.0, p1 = 0.0;
        mm16(p0, p1, g, 1.0, t, mt, nt);
        store16(b0, mt, nt, p0, p1);
      }
    if (K != 0) {
      mfrag20(g, Ms + kMat20 * f2(0));
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          double q0 = 0.0, q1 = 0.0;
          mm16(q0, q1, g, 1.0, t, mt, nt);
          store16(b1, mt, nt, q0, q1);
        }
    }
    __syncthreads();
  }
  {  // pass 2 (axis 1)
    double t0[4][4], t1[4][4];
    xfrag16(b0, t0);
    if (K != 0) xfrag16(b1, t1);
    __syncthreads();
    MFrag16 g1, g2;
    mfrag20(g1, Ms + kMat20 * f1(1));
    mfrag20(g2, Ms + kMat20 * f2(1));
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
        if (K == 0) {  // shared B x: two outputs
          mm16(p0, p1, g1, al, t0, mt, nt);
          mm16(q0, q1, g2, be, t0, mt, nt);
          store16(b0, mt, nt, p0, p1);
          store16(b1, mt, nt, q0, q1);
        } else if (K == 2) {  // both end with B: combine now
          mm16(p0, p1, g1, al, t0, mt, nt);
          mm16(p0, p1, g2, be, t1, mt, nt);
          store16(b0, mt, nt, p0, p1);
        } else {
          mm16(p0, p1, g1, al, t0, mt, nt);
          mm16(q0, q1, g2, be, t1, mt, nt);
          store16(b0, mt, nt, p0, p1);
          store16(b1, mt, nt, q0, q1);
        }
      }
    __syncthreads();
  }
  {  // pass 3 (axis 2) into the accumulator
    double t0[4][4];
    xfrag16(b0, t0);
    MFrag16 g;
    mfrag20(g, Ms + kMat20 * f1(2));
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) mm16(acc[mt][nt][0], acc[mt][nt][1], g, 1.0, t0, mt, nt);
    if (K != 2) {
      xfrag16(b1, t0);
      mfrag20(g, Ms + kMat20 * f2(2));
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) mm16(acc[mt][nt][0], acc[mt][nt][1], g, 1.0, t0, mt, nt);
    }
  }
}

__global__ void __launch_bounds__(kLines16, 1) k_cells_elastic16(const double* __restrict__ x, double* __restrict__ E,
                                                               int ncells, int64_t nsc,
                                                               const int32_t* __restrict__ cdofs,
                                                               const uint8_t* __restrict__ cons,
                                                               const double* __restrict__ mu, double lmu, double llam,
                                                               const double* __restrict__ Ahat,
                                                               const double* __restrict__ Bhat,
                                                               const double* __restrict__ Cm) {
  extern __shared__ __align__(16) double sm[];
  double* Ms = sm;               // rows of A, B, C, C^T (stride kRow20)
  double* b0 = Ms + 4 * kMat20;  // 4096, Pos16 layout
  double* b1 = b0 + kNpc16;
  const int c = blockIdx.x, lane = threadIdx.x & 31;
  load_rows20(Ms, Ahat, false);
  load_rows20(Ms + kMat20, Bhat, false);
  load_rows20(Ms + 2 * kMat20, Cm, false);
  load_rows20(Ms + 3 * kMat20, Cm, true);  // C^T
  const int32_t* cd = cdofs + size_t(c) * kNpc16;
  double m[3];
  for (int a = 0; a < 3; ++a) m[a] = mu[size_t(c) * 3 + a];
  pdl_wait();
#pragma unroll 1
  for (int i = 0; i < 3; ++i) {
    double acc[2][4][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll 1
    for (int j = 0; j < 3; ++j) {
      __syncthreads();  // previous block's last fragment reads of b0 / b1 are done
      gather16(b0, x, cd, cons, j * nsc);
      __syncthreads();
      if (j == i) {  // diagonal block: sum_a mu'_a A_a (x) B (x) B, mu'_a = (mu + (mu + lambda) [a == i]) mu_a
        const double m0 = (llam * (i == 0) + lmu * (1 + (i == 0))) * m[0];
        const double m1 = (llam * (i == 1) + lmu * (1 + (i == 1))) * m[1];
        const double m2 = (llam * (i == 2) + lmu * (1 + (i == 2))) * m[2];
        MFrag16 fa, fb;
        mfrag20(fa, Ms);
        mfrag20(fb, Ms + kMat20);
        {
          double t[4][4];
          xfrag16(b0, t);
          __syncthreads();
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
              mm16(p0, p1, fb, 1.0, t, mt, nt);
              mm16(q0, q1, fa, 1.0, t, mt, nt);
              store16(b0, mt, nt, p0, p1);
              store16(b1, mt, nt, q0, q1);
            }
          __syncthreads();
        }
        {
          double t0[4][4], t1[4][4];
          xfrag16(b0, t0);
          xfrag16(b1, t1);
          __syncthreads();
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
              mm16(p0, p1, fb, m0, t1, mt, nt);
              mm16(p0, p1, fa, m1, t0, mt, nt);
              mm16(q0, q1, fb, 1.0, t0, mt, nt);
              store16(b0, mt, nt, p0, p1);
              store16(b1, mt, nt, q0, q1);
            }
          __syncthreads();
        }
        {
          double t0[4][4], t1[4][4];
          xfrag16(b0, t0);
          xfrag16(b1, t1);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              mm16(acc[mt][nt][0], acc[mt][nt][1], fb, 1.0, t0, mt, nt);
              mm16(acc[mt][nt][0], acc[mt][nt][1], fa, m2, t1, mt, nt);
            }
        }
        continue;
      }
      // cross block (i, j): alpha (C on i, C^T on j) + beta (C^T on i, C on j), B on the third axis
      const double s = sqrt(m[i] * m[j]);
      switch (3 - i - j) {
        case 0: elastic_cross16<0>(Ms, b0, b1, i, j, lmu * s, llam * s, acc); break;
        case 1: elastic_cross16<1>(Ms, b0, b1, i, j, lmu * s, llam * s, acc); break;
        default: elastic_cross16<2>(Ms, b0, b1, i, j, lmu * s, llam * s, acc); break;
      }
    }
    // y_i: element r + 256 k of the lattice order, straight from the accumulator
    double* e = E + (size_t(i) * ncells + c) * kNpc16;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int kk = 8 * mt + (lane >> 2), r = 32 * (threadIdx.x >> 5) + 8 * nt + 2 * (lane & 3);
        *reinterpret_cast<double2*>(e + r + kLines16 * kk) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      }
  }
  pdl_trigger();
}

// mode 0: apply_St (sum, project); 1: apply_S (sum * inv_mult, project);
// 2: operator (sum; constrained rows y_i = x_i); 3: x + sum (project).
// VEC: vector (elasticity) handles, all components in one grid -- DOF g is
// scalar DOF g mod nsc of component g / nsc, whose E block starts at
// (g / nsc) * eoff; the gather maps are the (shared) scalar ones.
template <bool VEC>
__global__ void k_gather(int64_t ndof, int mode, const double* __restrict__ E, const int32_t* __restrict__ ptr,
                         const int32_t* __restrict__ idx, const double* __restrict__ inv_mult,
                         const uint8_t* __restrict__ cons, const double* __restrict__ x, double* __restrict__ out,
                         int64_t nsc, int64_t eoff) {
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  pdl_trigger();
  // The maps are static: load them (and the first two entry indices -- one
  // for cell-interior DOFs, two on facets) while the predecessor finishes.
  int q0 = 0, q1 = 0, i0 = 0, i1 = 0;
  bool c = false;
  double w = 1.0;
  if (g < ndof) {
    int64_t gl = g;
    if (VEC) {
      const int64_t comp = g / nsc;
      gl = g - comp * nsc;
      E += comp * eoff;
    }
    q0 = ptr[gl];
    q1 = ptr[gl + 1];
    c = cons[g];
    if (mode == 1) w = inv_mult[g];
    if (q1 > q0) i0 = idx[q0];
    if (q1 > q0 + 1) i1 = idx[q0 + 1];
  }
  pdl_wait();
  if (g >= ndof) return;
  double s = q1 > q0 ? E[i0] : 0.0;
  if (q1 > q0 + 1) s += E[i1];
  for (int q = q0 + 2; q < q1; ++q) s += E[idx[q]];
  s *= w;
  if (mode == 3) s += x[g];
  if (c) s = (mode == 2) ? x[g] : 0.0;
  out[g] = s;
}

// k_gather (mode 0: plain sums, constrained DOFs zero) over a list of DOFs: the same sums in
// the same order; entries of `out` outside the list are left alone.
__global__ void k_gather_list(int64_t n, const int32_t* __restrict__ list, const double* __restrict__ E,
                              const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                              const uint8_t* __restrict__ cons, double* __restrict__ out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  pdl_trigger();
  int g = 0, q0 = 0, q1 = 0, i0 = 0, i1 = 0;
  bool c = false;
  if (i < n) {
    g = list[i];
    q0 = ptr[g];
    q1 = ptr[g + 1];
    c = cons[g];
    if (q1 > q0) i0 = idx[q0];
    if (q1 > q0 + 1) i1 = idx[q0 + 1];
  }
  pdl_wait();
  if (i >= n) return;
  double s = q1 > q0 ? E[i0] : 0.0;
  if (q1 > q0 + 1) s += E[i1];
  for (int q = q0 + 2; q < q1; ++q) s += E[idx[q]];
  out[g] = c ? 0.0 : s;
}

size_t fdm_tables_bytes(const Context& c) {
  int ni = 1;
  for (int a = 0; a < c.dim; ++a) ni *= c.p - 1;
  return sizeof(double) * (2 * size_t(c.n1) * c.n1 + size_t(ni));
}

template <class K>
void set_smem(K kernel, size_t smem) {
  if (smem > 227 * 1024) throw Error(FDMGPU_UNSUPPORTED, "cell tile exceeds shared memory (p too large for dim)");
  FDM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
}

int cell_threads(const Context& c) { return c.npc >= 1024 ? 512 : 256; }

}  // namespace

void launch_cells_transform_fused(Context& c, int dir, const double* in, int flags, const double* aux) {
  if (c.n1 == kL16 && c.dim == 3) {
    const size_t smem16 = sizeof(double) * (kL16 * kL16 + size_t(kNpc16) + (flags ? 2 * kL16 * kL16 : 0));
    set_smem(k_cells_transform16, smem16);
    KernelTimer timer(c, 2);
    launch_pdl(c.pdl && !c.timing, k_cells_transform16, dim3(c.ncells), dim3(kLines16), smem16, c.stream, dir, flags, in,
               aux, c.E.p, dir == 0 ? c.cell_dofs.p : c.cell_modes.p, c.inv_mult.p, c.constrained.p, c.mode_sign.p,
               dir == 0 ? c.St.p : c.S.p, c.mu.p, c.At.p, c.Bt.p, c.nK.p);
    FDM_LAUNCH_CHECK(c);
    return;
  }
  const size_t smem = sizeof(double) * (size_t(c.n1) * c.n1 + 2 * size_t(c.npc)) + (flags ? fdm_tables_bytes(c) : 0);
  auto go = [&](auto kernel) {
    set_smem(kernel, smem);
    KernelTimer timer(c, 2);
    kernel<<<c.ncells, cell_threads(c), smem, c.stream>>>(
        c.dim, c.n1, c.npc, dir, flags, in, aux, c.E.p, dir == 0 ? c.cell_dofs.p : c.cell_modes.p, c.inv_mult.p,
        c.constrained.p, c.mode_sign.p, dir == 0 ? c.St.p : c.S.p, c.mu.p, c.At.p, c.Bt.p, c.nK.p);
    FDM_LAUNCH_CHECK(c);
  };
  switch (c.n1) {
    case 4: go(k_cells_transform<4>); break;
    case 6: go(k_cells_transform<6>); break;
    case 8: go(k_cells_transform<8>); break;
    case 16: go(k_cells_transform<16>); break;
    default: go(k_cells_transform<0>);
  }
}

void launch_cells_schur_fused(Context& c, const double* in) {
  const size_t smem = sizeof(double) * size_t(c.npc) + fdm_tables_bytes(c);
  set_smem(k_cells_schur, smem);
  k_cells_schur<<<c.ncells, cell_threads(c), smem, c.stream>>>(c.dim, c.n1, c.npc, in, c.E.p, c.cell_modes.p,
                                                               c.constrained.p, c.mu.p, c.At.p, c.Bt.p);
  FDM_LAUNCH_CHECK(c);
}

void launch_cells_recon_fused(Context& c, double* z, const double* rb) {
  const size_t smem = sizeof(double) * size_t(c.npc) + fdm_tables_bytes(c);
  set_smem(k_cells_recon, smem);
  k_cells_recon<<<c.ncells, cell_threads(c), smem, c.stream>>>(c.dim, c.n1, c.npc, z, rb, c.cell_modes.p, c.mu.p,
                                                               c.At.p, c.Bt.p, c.nK.p);
  FDM_LAUNCH_CHECK(c);
}

void launch_gather(Context& c, int mode, const double* E, const double* x, double* out) {
  const bool modes = (mode == 0 || mode == 3) && !c.modes_alias;
  const int threads = 256;
  const int64_t blocks = (c.ndof + threads - 1) / threads;
  launch_pdl(c.pdl && !c.timing, k_gather<false>, dim3(unsigned(blocks)), dim3(threads), 0, c.stream, c.ndof, mode, E,
             modes ? c.gm_ptr.p : c.g_ptr.p, modes ? c.gm_idx.p : c.g_idx.p, c.inv_mult.p, c.constrained.p, x, out,
             c.ndof, int64_t(0));
  FDM_LAUNCH_CHECK(c);
}

// S^T gather (mode 0) of the cell-boundary DOFs only (Context::bnd_list); the others keep their old values.
void launch_gather_bnd(Context& c, const double* E, double* out) {
  if (!c.bnd_list.p) return launch_gather(c, 0, E, nullptr, out);
  const bool modes = !c.modes_alias;
  const int threads = 256;
  const int64_t n = int64_t(c.bnd_list.n), blocks = (n + threads - 1) / threads;
  launch_pdl(c.pdl && !c.timing, k_gather_list, dim3(unsigned(blocks)), dim3(threads), 0, c.stream, n,
             (const int32_t*)c.bnd_list.p, E, (const int32_t*)(modes ? c.gm_ptr.p : c.g_ptr.p),
             (const int32_t*)(modes ? c.gm_idx.p : c.g_idx.p), (const uint8_t*)c.constrained.p, out);
  FDM_LAUNCH_CHECK(c);
}

void launch_gather_vec(Context& c, int mode, const double* E, const double* x, double* out) {
  const Context& s = *c.comp[0];  // the components share the scalar gather maps
  const int threads = 256;
  const int64_t blocks = (c.ndof + threads - 1) / threads;
  launch_pdl(c.pdl && !c.timing, k_gather<true>, dim3(unsigned(blocks)), dim3(threads), 0, c.stream, c.ndof, mode, E,
             s.g_ptr.p, s.g_idx.p, c.inv_mult.p, c.constrained.p, x, out, c.nsc, int64_t(c.ncells) * c.npc);
  FDM_LAUNCH_CHECK(c);
}

bool launch_cells_elastic16(Context& c, const double* x) {
  if (c.n1 != kL16 || c.dim != 3) return false;
  const size_t smem = sizeof(double) * (4 * kMat20 + 2 * size_t(kNpc16));
  set_smem(k_cells_elastic16, smem);
  KernelTimer timer(c, 3);
  launch_pdl(c.pdl && !c.timing, k_cells_elastic16, dim3(c.ncells), dim3(kLines16), smem, c.stream, x, c.E.p,
             c.ncells, c.nsc, c.cell_dofs.p, c.constrained.p, c.mu.p, c.lame_mu, c.lame_lambda, c.Ahat.p, c.Bhat.p,
             c.Cm.p);
  FDM_LAUNCH_CHECK(c);
  return true;
}

void launch_cells_stiffness_kron(Context& c, const double* x) {
  if (c.n1 == kL16 && c.dim == 3) {
    const size_t smem16 = sizeof(double) * (2 * kL16 * kL16 + 2 * size_t(kNpc16));
    set_smem(k_cells_stiffness16, smem16);
    KernelTimer timer(c, 3);
    launch_pdl(c.pdl && !c.timing, k_cells_stiffness16, dim3(c.ncells), dim3(kLines16), smem16, c.stream, x,
               c.E.p, (const int32_t*)c.cell_dofs.p, (const uint8_t*)c.constrained.p, (const double*)c.mu.p,
               (const double*)c.Ahat.p, (const double*)c.Bhat.p);
    FDM_LAUNCH_CHECK(c);
    return;
  }
  const size_t smem = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 4 * size_t(c.npc));
  auto go = [&](auto kernel) {
    set_smem(kernel, smem);
    KernelTimer timer(c, 3);
    kernel<<<c.ncells, cell_threads(c), smem, c.stream>>>(c.dim, c.n1, c.npc, x, c.E.p, c.cell_dofs.p,
                                                          c.constrained.p, c.mu.p, c.Ahat.p, c.Bhat.p);
    FDM_LAUNCH_CHECK(c);
  };
  switch (c.n1) {
    case 4: go(k_cells_stiffness<4>); break;
    case 6: go(k_cells_stiffness<6>); break;
    case 8: go(k_cells_stiffness<8>); break;
    case 16: go(k_cells_stiffness<16>); break;
    default: go(k_cells_stiffness<0>);
  }
}

}  // namespace fdmgpu
