// Matrix-free vector Q_p linear-elasticity operator on Cartesian cells
// (GlobalOperator::apply over elasticity_primal_operator's Kronecker blocks,
// src/assembly.cpp:56-88 with src/elasticity.cpp:69-120):
//
//   y_i += sum_a c_i[a] mu_a (A on axis a, B elsewhere) x_i                (diagonal block)
//        + sum_{j != i} s_ij [ mu_L (C on i, C^T on j, B elsewhere)
//                              + lambda_L (C^T on i, C on j, B elsewhere) ] x_j   (cross blocks)
//
// with c_i = sdc_axis_coefficients(i) = mu_L + (mu_L + lambda_L) delta_ia,
// mu_a the cell's Cartesian coefficients prod(L)/L_a^2 and
// s_ij = prod(L)/(L_i L_j) = sqrt(mu_i mu_j).  One CTA per cell: the d
// component tiles are gathered once into shared memory (constrained entries
// zeroed: project_free), every Kronecker term is d sum-factorised 1D
// contractions through two ping-pong tiles, and the last contraction of each
// term accumulates into the output tile, which is stored to the cell-local
// E-vector of its component.  The owner gather (k_gather, mode 2) then sums
// cells in ascending order per component, so results are deterministic and
// need no FP64 atomics.
#include "common.cuh"

namespace fdmgpu {

namespace {

// out[o] (+)= coeff * sum_l M[k + n1 l] in[base + l stride], k = o's index on `axis`.
template <int N1C>
__device__ __forceinline__ void contract_axis(int n1_rt, int npc, int axis, const double* __restrict__ M,
                                              const double* __restrict__ in, double* __restrict__ out, double coeff,
                                              bool accumulate) {
  if constexpr (N1C > 0) {
    // Thread t owns output index k = t mod n1 on the contracted axis for the whole
    // pass (blockDim is a multiple of n1), so row k of M sits in registers and
    // every output costs n1 loads of `in` (lanes sharing a line broadcast).
    static_assert(256 % N1C == 0, "block size must be a multiple of n1");
    const int stride = axis == 0 ? 1 : (axis == 1 ? N1C : N1C * N1C);
    const int k = threadIdx.x % N1C;
    double mk[N1C];
#pragma unroll
    for (int l = 0; l < N1C; ++l) mk[l] = M[k + N1C * l];
    for (int mm = threadIdx.x / N1C; mm < npc / N1C; mm += blockDim.x / N1C) {
      const int lo = mm % stride, hi = mm / stride;
      const int base = lo + hi * stride * N1C;
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < N1C; ++l) s = fma(mk[l], in[base + l * stride], s);
      const int o = base + k * stride;
      out[o] = accumulate ? fma(coeff, s, out[o]) : coeff * s;
    }
    __syncthreads();
    return;
  }
  const int n1 = N1C > 0 ? N1C : n1_rt;
  const int stride = axis == 0 ? 1 : (axis == 1 ? n1 : n1 * n1);
  for (int o = threadIdx.x; o < npc; o += blockDim.x) {
    const int k = (o / stride) % n1;
    const int base = o - k * stride;
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < (N1C > 0 ? N1C : 32); ++l) {
      if (N1C == 0 && l >= n1) break;
      s = fma(M[k + n1 * l], in[base + l * stride], s);
    }
    out[o] = accumulate ? fma(coeff, s, out[o]) : coeff * s;
  }
  __syncthreads();
}

// One Kronecker term: Y (+)= coeff * (F_{d-1} (x) ... (x) F_0) X.  Passes run
// axis 0 first (the order of kron_apply, src/kron.cpp:40-55).  The final
// accumulate into Y is race free: each pass ends with a barrier, and within a
// pass every Y entry has exactly one writer.
template <int N1C>
__device__ __forceinline__ void kron_term(int dim, int n1, int npc, const double* const* F, const double* X, double* T1,
                                          double* T2, double* Y, double coeff, bool& first) {
  const double* in = X;
  double* bufs[2] = {T1, T2};
  for (int a = 0; a < dim; ++a) {
    const bool last = a == dim - 1;
    double* out = last ? Y : bufs[a & 1];
    contract_axis<N1C>(n1, npc, a, F[a], in, out, last ? coeff : 1.0, last && !first);
    in = out;
  }
  first = false;
}

template <int N1C>
__global__ void __launch_bounds__(256) k_cells_elastic(int dim, int n1_rt, int npc, int ncells, int64_t nsc,
                                                       const double* __restrict__ x, double* __restrict__ E,
                                                       const int32_t* __restrict__ cell_dofs,
                                                       const uint8_t* __restrict__ cons, const double* __restrict__ mu,
                                                       double lmu, double llam, const double* __restrict__ Ah,
                                                       const double* __restrict__ Bh, const double* __restrict__ Cm) {
  const int n1 = N1C > 0 ? N1C : n1_rt;
  extern __shared__ double sm[];
  double* sA = sm;
  double* sB = sA + n1 * n1;
  double* sC = sB + n1 * n1;
  double* sCt = sC + n1 * n1;
  double* X = sCt + n1 * n1;  // dim component tiles
  double* T1 = X + size_t(dim) * npc;
  double* T2 = T1 + npc;
  double* Y = T2 + npc;
  const int cell = blockIdx.x;
  for (int k = threadIdx.x; k < n1 * n1; k += blockDim.x) {
    sA[k] = Ah[k];
    sB[k] = Bh[k];
    sC[k] = Cm[k];
    const int r = k % n1, l = k / n1;
    sCt[k] = Cm[l + n1 * r];
  }
  pdl_wait();
  const int32_t* cd = cell_dofs + size_t(cell) * npc;
  for (int ci = 0; ci < dim; ++ci)
    staged_copy<4>(
        npc,
        [&](int k) {
          const int64_t g = cd[k] + ci * nsc;
          return cons[g] ? 0.0 : x[g];
        },
        [&](int k, double v) { X[size_t(ci) * npc + k] = v; });
  double m[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < dim; ++a) m[a] = mu[size_t(cell) * dim + a];
  __syncthreads();
  for (int i = 0; i < dim; ++i) {
    bool first = true;
    const double* F[3];
    // diagonal block: sum_a c_i[a] mu_a A_a (x) B (x) B
    for (int a = 0; a < dim; ++a) {
      for (int b = 0; b < dim; ++b) F[b] = b == a ? sA : sB;
      const double c = a == i ? lmu + (lmu + llam) : lmu;
      kron_term<N1C>(dim, n1, npc, F, X + size_t(i) * npc, T1, T2, Y, c * m[a], first);
    }
    // cross blocks (i, j): mu_L s (C on i, C^T on j) + lambda_L s (C^T on i, C on j), B elsewhere
    for (int j = 0; j < dim; ++j) {
      if (j == i) continue;
      const double s = sqrt(m[i] * m[j]);
      for (int b = 0; b < dim; ++b) F[b] = b == i ? sC : (b == j ? sCt : sB);
      kron_term<N1C>(dim, n1, npc, F, X + size_t(j) * npc, T1, T2, Y, lmu * s, first);
      for (int b = 0; b < dim; ++b) F[b] = b == i ? sCt : (b == j ? sC : sB);
      kron_term<N1C>(dim, n1, npc, F, X + size_t(j) * npc, T1, T2, Y, llam * s, first);
    }
    double* e = E + (size_t(i) * ncells + cell) * npc;
    for (int k = threadIdx.x; k < npc; k += blockDim.x) e[k] = Y[k];
    __syncthreads();
  }
  pdl_trigger();
}

template <class K>
void set_smem(K kernel, size_t smem) {
  if (smem > 227 * 1024) throw Error(FDMGPU_UNSUPPORTED, "elasticity: component tiles exceed shared memory (p too large)");
  FDM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
}

}  // namespace

size_t elastic_smem_bytes(const Context& c) {
  return sizeof(double) * (4 * size_t(c.n1) * c.n1 + size_t(c.dim + 3) * c.npc);
}

bool launch_cells_elastic16(Context& c, const double* x);  // cells.cu: n1 = 16, dim = 3 on the DMMA pipe

void launch_cells_elastic(Context& c, const double* x) {
  if (!c.force_staged && launch_cells_elastic16(c, x)) return;
  const size_t smem = elastic_smem_bytes(c);
  auto go = [&](auto kernel) {
    set_smem(kernel, smem);
    KernelTimer timer(c, 3);
    launch_pdl(c.pdl && !c.timing, kernel, dim3(c.ncells), dim3(256), smem, c.stream, c.dim, c.n1, c.npc, c.ncells,
               c.nsc, x, c.E.p, c.cell_dofs.p, c.constrained.p, c.mu.p, c.lame_mu, c.lame_lambda, c.Ahat.p, c.Bhat.p,
               c.Cm.p);
    FDM_LAUNCH_CHECK(c);
  };
  switch (c.n1) {
    case 4: go(k_cells_elastic<4>); break;
    case 8: go(k_cells_elastic<8>); break;
    case 16: go(k_cells_elastic<16>); break;
    default: go(k_cells_elastic<0>); break;
  }
}

}  // namespace fdmgpu
