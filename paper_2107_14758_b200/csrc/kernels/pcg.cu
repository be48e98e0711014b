// Device-resident PCG (src/krylov.cpp:29-83) as one CUDA graph:
//   WHILE(cont) {  Ap = A p;  pAp = p.Ap;  alpha = rz / pAp (indefinite -> stop);
//                  x += alpha p;  r -= alpha Ap;  res = |r| / |b|;
//                  IF(not converged and k < maxit) { z = Pinv r;  rz' = r.z;
//                                                     beta = rz'/rz;  p = z + beta p } }
// Scalars live in device memory; dot products use fixed-grid partials
// finished by one thread in a fixed order (deterministic run to run).  The
// host reads the CG coefficients back once, after the loop, for the Lanczos
// estimate (src/krylov.cpp:69-80): no host round trip inside the loop.
#include "common.cuh"

namespace fdmgpu {

namespace {

__global__ void k_dot_finish(const double* __restrict__ partials, int n, double* __restrict__ dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < n; ++b) s += partials[b];
    *dst = s;
  }
}

__global__ void k_pcg_alpha(PcgDev* st, double* alphas, cudaGraphConditionalHandle h_while) {
  if (threadIdx.x || blockIdx.x) return;
  if (!(st->pAp > 0.0)) {
    st->status = 2;
    cudaGraphSetConditional(h_while, 0);
    return;
  }
  st->alpha = st->rz / st->pAp;
  alphas[st->k] = st->alpha;
}

// x += alpha p; r -= alpha Ap  (skipped once the operator was found indefinite)
__global__ void k_pcg_update_xr(int64_t n, const PcgDev* __restrict__ st, const double* __restrict__ p,
                                const double* __restrict__ Ap, double* __restrict__ x, double* __restrict__ r) {
  if (st->status == 2) return;
  const double a = st->alpha;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    x[i] = x[i] + a * p[i];
    r[i] = r[i] + (-a) * Ap[i];
  }
}

__global__ void k_pcg_residual(PcgDev* st, double* residuals, cudaGraphConditionalHandle h_while,
                               cudaGraphConditionalHandle h_if) {
  if (threadIdx.x || blockIdx.x) return;
  if (st->status == 2) {
    cudaGraphSetConditional(h_if, 0);
    cudaGraphSetConditional(h_while, 0);
    return;
  }
  const double res = sqrt(st->res) / st->bnorm;  // st->res holds r.r on entry
  st->res = res;
  residuals[st->k] = res;
  st->k += 1;
  unsigned go = 1;
  if (res <= st->rtol) {
    st->status = 1;
    go = 0;
  } else if (st->k >= st->maxit) {
    st->status = 3;
    go = 0;
  }
  cudaGraphSetConditional(h_if, go);
  cudaGraphSetConditional(h_while, go);
}

__global__ void k_pcg_beta(PcgDev* st, double* betas) {
  if (threadIdx.x || blockIdx.x) return;
  st->beta = st->rz_new / st->rz;
  betas[st->k - 1] = st->beta;
  st->rz = st->rz_new;
}

// p = z + beta p
__global__ void k_pcg_update_p(int64_t n, const PcgDev* __restrict__ st, const double* __restrict__ z,
                               double* __restrict__ p) {
  const double b = st->beta;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = b * p[i] + z[i];
}

}  // namespace

// Device-side scalar helpers used by the graph builder in capi.cpp.
void launch_dot_finish(Context& c, int k, double* dst) {
  k_dot_finish<<<1, 32, 0, c.stream>>>(c.red.p + size_t(k) * kRedBlocks, kRedBlocks, dst);
  FDM_LAUNCH_CHECK(c);
}

size_t pcg_state_bytes() { return sizeof(PcgDev); }

void pcg_state_init(Context& c, void* st, double bnorm, double rtol, double rz, int maxit) {
  PcgDev h{};
  h.bnorm = bnorm;
  h.rtol = rtol;
  h.rz = rz;
  h.maxit = maxit;
  h.k = 0;
  h.status = 0;
  FDM_CUDA(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, c.stream));
}

void pcg_state_read(Context& c, const void* st, int* k, int* status) {
  PcgDev h{};
  FDM_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  FDM_CUDA(cudaStreamSynchronize(c.stream));
  *k = h.k;
  *status = h.status;
}

// Capture-time launchers (recorded into the loop body graph).
void launch_pcg_alpha(Context& c, void* st, double* alphas, cudaGraphConditionalHandle hw) {
  k_pcg_alpha<<<1, 32, 0, c.stream>>>(static_cast<PcgDev*>(st), alphas, hw);
  FDM_LAUNCH_CHECK(c);
}
void launch_pcg_update_xr(Context& c, const void* st, const double* p, const double* Ap, double* x, double* r) {
  k_pcg_update_xr<<<4 * 148, 256, 0, c.stream>>>(c.ndof, static_cast<const PcgDev*>(st), p, Ap, x, r);
  FDM_LAUNCH_CHECK(c);
}
void launch_pcg_residual(Context& c, void* st, double* residuals, cudaGraphConditionalHandle hw,
                         cudaGraphConditionalHandle hi) {
  k_pcg_residual<<<1, 32, 0, c.stream>>>(static_cast<PcgDev*>(st), residuals, hw, hi);
  FDM_LAUNCH_CHECK(c);
}
void launch_pcg_beta(Context& c, void* st, double* betas) {
  k_pcg_beta<<<1, 32, 0, c.stream>>>(static_cast<PcgDev*>(st), betas);
  FDM_LAUNCH_CHECK(c);
}
void launch_pcg_update_p(Context& c, const void* st, const double* z, double* p) {
  k_pcg_update_p<<<4 * 148, 256, 0, c.stream>>>(c.ndof, static_cast<const PcgDev*>(st), z, p);
  FDM_LAUNCH_CHECK(c);
}

}  // namespace fdmgpu
