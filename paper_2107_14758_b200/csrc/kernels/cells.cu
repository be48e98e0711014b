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
#include "common.cuh"

namespace fdmgpu {

namespace {

// out[.., k, ..] = alpha * sum_j M1[k + n1 j] in1[.., j, ..] (+ beta * same with M2/in2)
__device__ __forceinline__ void contract(int n1, int npc, int stride, const double* __restrict__ M1,
                                         const double* __restrict__ in1, double alpha, const double* __restrict__ M2,
                                         const double* __restrict__ in2, double beta, double* __restrict__ out) {
  for (int o = threadIdx.x; o < npc; o += blockDim.x) {
    const int k = (o / stride) % n1;
    const int base = o - k * stride;
    double s1 = 0.0, s2 = 0.0;
    for (int j = 0; j < n1; ++j) {
      s1 = fma(M1[k + n1 * j], in1[base + j * stride], s1);
      if (M2) s2 = fma(M2[k + n1 * j], in2[base + j * stride], s2);
    }
    out[o] = M2 ? alpha * s1 + beta * s2 : alpha * s1;
  }
}

__global__ void k_cells_transform(int dim, int n1, int npc, int dir, const double* __restrict__ in,
                                  double* __restrict__ E, const int32_t* __restrict__ cdofs,
                                  const double* __restrict__ inv_mult, const uint8_t* __restrict__ cons,
                                  const double* __restrict__ sign, const double* __restrict__ M) {
  extern __shared__ double sm[];
  double* Ms = sm;
  double* b0 = Ms + n1 * n1;
  double* b1 = b0 + npc;
  const int c = blockIdx.x;
  for (int i = threadIdx.x; i < n1 * n1; i += blockDim.x) Ms[i] = M[i];
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
  double* src = b0;
  double* dst = b1;
  int stride = 1;
  for (int a = 0; a < dim; ++a, stride *= n1) {
    contract(n1, npc, stride, Ms, src, 1.0, nullptr, nullptr, 0.0, dst);
    __syncthreads();
    double* t = src;
    src = dst;
    dst = t;
  }
  double* e = E + size_t(c) * npc;
  for (int l = threadIdx.x; l < npc; l += blockDim.x) {
    double v = src[l];
    if (dir == 0 && sign) v *= sign[size_t(c) * npc + l];
    e[l] = v;
  }
}

// Cartesian stiffness: y_K = sum_a mu_a (A on axis a, B elsewhere) u_K.
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
  contract(n1, npc, 1, Bs, u, 1.0, nullptr, nullptr, 0.0, t0);  // B_x u
  contract(n1, npc, 1, As, u, 1.0, nullptr, nullptr, 0.0, t1);  // A_x u
  __syncthreads();
  double* e = E + size_t(c) * npc;
  if (dim == 2) {
    // mu0 B_y A_x u + mu1 A_y B_x u
    contract(n1, npc, n1, Bs, t1, m0, As, t0, m1, u);
    __syncthreads();
    for (int l = threadIdx.x; l < npc; l += blockDim.x) e[l] = u[l];
    return;
  }
  // P = mu0 B_y A_x u + mu1 A_y B_x u  (into u),  Q = B_y B_x u
  contract(n1, npc, n1, Bs, t1, m0, As, t0, m1, u);
  contract(n1, npc, n1, Bs, t0, 1.0, nullptr, nullptr, 0.0, q);
  __syncthreads();
  // y = B_z P + mu2 A_z Q
  contract(n1, npc, n1 * n1, Bs, u, 1.0, As, q, m2, t0);
  __syncthreads();
  for (int l = threadIdx.x; l < npc; l += blockDim.x) e[l] = t0[l];
}

// mode 0: apply_St (sum, project); 1: apply_S (sum * inv_mult, project);
// 2: operator (sum; constrained rows y_i = x_i).
__global__ void k_gather(int64_t ndof, int mode, const double* __restrict__ E, const int32_t* __restrict__ ptr,
                         const int32_t* __restrict__ idx, const double* __restrict__ inv_mult,
                         const uint8_t* __restrict__ cons, const double* __restrict__ x, double* __restrict__ out) {
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (g >= ndof) return;
  double s = 0.0;
  for (int q = ptr[g]; q < ptr[g + 1]; ++q) s += E[idx[q]];
  if (mode == 1) s *= inv_mult[g];
  if (cons[g]) s = (mode == 2) ? x[g] : 0.0;
  out[g] = s;
}

}  // namespace

void launch_cells_transform(Context& c, int dir, const double* in) {
  const size_t smem = sizeof(double) * (size_t(c.n1) * c.n1 + 2 * size_t(c.npc));
  if (smem > 227 * 1024) throw Error(FDMGPU_UNSUPPORTED, "cell tile exceeds shared memory (p too large for dim)");
  static bool attr_set = false;
  if (!attr_set) {
    FDM_CUDA(cudaFuncSetAttribute(k_cells_transform, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set = true;
  }
  const int threads = c.npc >= 1024 ? 512 : 256;
  k_cells_transform<<<c.ncells, threads, smem, c.stream>>>(
      c.dim, c.n1, c.npc, dir, in, c.E.p, dir == 0 ? c.cell_dofs.p : c.cell_modes.p, c.inv_mult.p, c.constrained.p,
      c.mode_sign.p, dir == 0 ? c.St.p : c.S.p);
  FDM_LAUNCH_CHECK(c);
}

void launch_gather(Context& c, int mode, const double* E, const double* x, double* out) {
  const bool modes = (mode == 0) && !c.modes_alias;
  const int threads = 256;
  const int64_t blocks = (c.ndof + threads - 1) / threads;
  k_gather<<<unsigned(blocks), threads, 0, c.stream>>>(c.ndof, mode, E, modes ? c.gm_ptr.p : c.g_ptr.p,
                                                       modes ? c.gm_idx.p : c.g_idx.p, c.inv_mult.p, c.constrained.p,
                                                       x, out);
  FDM_LAUNCH_CHECK(c);
}

void launch_cells_stiffness(Context& c, const double* x) {
  if (!c.all_cartesian) throw Error(FDMGPU_UNSUPPORTED, "non-Cartesian cells need the quadrature operator");
  const size_t smem = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 4 * size_t(c.npc));
  if (smem > 227 * 1024) throw Error(FDMGPU_UNSUPPORTED, "cell tile exceeds shared memory (p too large for dim)");
  static bool attr_set = false;
  if (!attr_set) {
    FDM_CUDA(cudaFuncSetAttribute(k_cells_stiffness, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set = true;
  }
  const int threads = c.npc >= 1024 ? 512 : 256;
  k_cells_stiffness<<<c.ncells, threads, smem, c.stream>>>(c.dim, c.n1, c.npc, x, c.E.p, c.cell_dofs.p,
                                                           c.constrained.p, c.mu.p, c.Ahat.p, c.Bhat.p);
  FDM_LAUNCH_CHECK(c);
}

}  // namespace fdmgpu
