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
  k_restrict<<<c.nc, 256, 0, c.stream>>>(c.PT_ptr.p, c.PT_col.p, c.PT_val.p, fine, coarse);
  FDM_LAUNCH_CHECK(c);
}

void launch_coarse_solve(Context& c, const double* rc, double* zc) {
  k_coarse_gemv<<<c.nc, 256, 0, c.stream>>>(c.nc, c.cinv.p, rc, zc);
  FDM_LAUNCH_CHECK(c);
}

void launch_prolong_add(Context& c, const double* coarse, double* fine) {
  const int threads = 256;
  k_prolong_add<<<unsigned((c.ndof + threads - 1) / threads), threads, 0, c.stream>>>(c.ndof, c.P_ptr.p, c.P_col.p,
                                                                                       c.P_val.p, coarse, fine);
  FDM_LAUNCH_CHECK(c);
}

}  // namespace fdmgpu
