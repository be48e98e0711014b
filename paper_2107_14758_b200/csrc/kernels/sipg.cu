// Symmetric interior-penalty DG kernels (src/sipg.cpp) on Cartesian cells:
//   k_dg_patch_assemble  entries of the transformed DG patch matrices
//                        (transformed_dg_poisson, src/sipg.cpp:252-364) into
//                        the shared dense-tile layout (layout_dg.cpp), from
//                        per-cell mu, eta and the 1D FDM tables -- the DG
//                        counterpart of k_patch_assemble;
//   k_dg_facets          the facet penalty terms of the true form
//                        (dg_poisson_operator, src/sipg.cpp:176-250) added to
//                        the cell terms of k_cells_stiffness: per cell, its
//                        2d facets as rank-3 (in the facet axis) x mass
//                        (tangential) Kronecker blocks; every CTA writes only
//                        its own cell's rows (deterministic, no atomics).
#include "common.cuh"

namespace fdmgpu {

namespace {

constexpr int T = kTile;
constexpr int TT = T * T;

struct DgArgs {
  int dim, p, n1, npc, m, ntiles;
  double eta;
  const int32_t* lat;     // canonical position codes slot * npc + l
  const int32_t* pcells;  // npatch x 2^d cells by slot
  const int32_t* psep;    // npatch x m DOFs, -1 absent
  const double* mu;       // ncells x d
  const double* At;       // (p+1)^2 column-major, structural zeros applied
  const double* Bt;
  const double* dtr;      // 2 x (p+1) column-major: outward derivative traces of the FDM modes
  const int32_t* fnbr;    // ncells x 2d
  const uint8_t* ftag;    // ncells x 2d
};

// Transformed 1D facet matrix entry (src/sipg.cpp:47-87):
//   E(i, j) = [i = tau_r][j = tau_s] alpha - [i = tau_r] beta dtr(e_s, j) - [j = tau_s] gamma dtr(e_r, i)
__device__ __forceinline__ double facet_t(const DgArgs& a, int i, int j, int tr, int ts, double alpha, double beta,
                                          double gamma) {
  const int er = tr ? 1 : 0, es = ts ? 1 : 0;
  double v = 0.0;
  if (i == tr && j == ts) v += alpha;
  if (i == tr) v -= beta * a.dtr[es + 2 * j];
  if (j == ts) v -= gamma * a.dtr[er + 2 * i];
  return v;
}

__device__ double dg_entry(const DgArgs& a, int j, int r, int c) {
  const int ncorner = 1 << a.dim, twod = 2 * a.dim;
  const int sr = a.lat[r] / a.npc, sc = a.lat[c] / a.npc;
  int lr[3] = {0, 0, 0}, lc[3] = {0, 0, 0};
  for (int b = 0, tr = a.lat[r] % a.npc, tc = a.lat[c] % a.npc; b < a.dim; ++b, tr /= a.n1, tc /= a.n1) {
    lr[b] = tr % a.n1;
    lc[b] = tc % a.n1;
  }
  const int Kr = a.pcells[size_t(j) * ncorner + sr], Kc = a.pcells[size_t(j) * ncorner + sc];
  auto bprod = [&](int skip) {
    double v = 1.0;
    for (int b = 0; b < a.dim; ++b)
      if (b != skip) v *= a.Bt[lr[b] + a.n1 * lc[b]];
    return v;
  };
  if (sr == sc) {
    const double* mu = a.mu + size_t(Kr) * a.dim;
    double v = 0.0;
    for (int q = 0; q < a.dim; ++q) v += mu[q] * a.At[lr[q] + a.n1 * lc[q]] * bprod(q);  // cell block
    for (int q = 0; q < a.dim; ++q) {
      const double bp = bprod(q);
      if (bp == 0.0) continue;
      for (int side = 0; side < 2; ++side) {
        const int f = 2 * q + side;
        const int tag = a.ftag[size_t(Kr) * twod + f];
        if (tag == 2) continue;  // Neumann: no facet term
        const int tau = side ? a.p : 0;
        double alpha, beta;
        if (tag == 1) {  // Dirichlet (sipg_facet_dirichlet_t)
          alpha = a.eta * mu[q];
          beta = mu[q];
        } else {         // own block of an interior facet (sign 1/2)
          const int N = a.fnbr[size_t(Kr) * twod + f];
          alpha = 0.5 * a.eta * (mu[q] + a.mu[size_t(N) * a.dim + q]);
          beta = 0.5 * mu[q];
        }
        v += facet_t(a, lr[q], lc[q], tau, tau, alpha, beta, beta) * bp;
      }
    }
    return v;
  }
  const int x = sr ^ sc;
  if (x & (x - 1)) return 0.0;  // not facet neighbours
  const int q = __ffs(x) - 1;
  const double bp = bprod(q);
  if (bp == 0.0) return 0.0;
  // the row cell's facet toward the vertex: its - side when it lies on the + side
  const int tr = ((sr >> q) & 1) ? 0 : a.p, ts = a.p - tr;
  const double mr = a.mu[size_t(Kr) * a.dim + q], mc = a.mu[size_t(Kc) * a.dim + q];
  return facet_t(a, lr[q], lc[q], tr, ts, -0.5 * a.eta * (mr + mc), -0.5 * mc, -0.5 * mr) * bp;
}

__global__ void k_dg_patch_assemble(DgArgs a, int nentries, const int32_t* __restrict__ entries,
                                    const int32_t* __restrict__ tile_row, const int32_t* __restrict__ tile_col,
                                    double* __restrict__ tiles) {
  const int j = blockIdx.y;
  double* base = tiles + size_t(j) * a.ntiles * TT;
  const int32_t* sep = a.psep + size_t(j) * a.m;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nentries; e += gridDim.x * blockDim.x) {
    const int code = entries[e];
    const int t = code >> 12, cc = (code >> 6) & 63, rr = code & 63;
    const int r = tile_row[t] * T + rr, c = tile_col[t] * T + cc;
    const double v = (sep[r] < 0 || sep[c] < 0) ? (r == c ? 1.0 : 0.0) : dg_entry(a, j, r, c);
    base[size_t(t) * TT + tsw(rr, cc)] = v;
  }
}

// Identity on the padded positions m..mpad-1 of the last diagonal tile.
__global__ void k_dg_pad(int m, int mpad, int ntiles, int last_diag, double* __restrict__ tiles) {
  double* dt = tiles + (size_t(blockIdx.x) * ntiles + last_diag) * TT;
  for (int r = m + threadIdx.x; r < mpad; r += blockDim.x) dt[tsw(r % T, r % T)] = 1.0;
}

// True-form SIPG facet terms of cell r (src/sipg.cpp:20-45, 200-248): for each
// non-Neumann local facet (axis q, side) and each cell s of its blocks,
//   E_rs(i, j) = sign (eta (mu_0 + mu_1) tv_r(i) tv_s(j) - mu_s tv_r(i) tnd_s(j) - mu_r tnd_r(i) tv_s(j))
// (Dirichlet: mu_e (eta tv tv^T - tv tnd^T - tnd tv^T)) on axis q, the GL mass
// on the others; E[r] += tv_r (M (x) M)(G1) - tnd_r (M (x) M)(G2) with the
// trace sums G1 = sum_s (alpha_s T1_s - beta_s T2_s), G2 = sum_s gamma_s T1_s,
// T1_s / T2_s the value / normal-derivative traces of u_s across axis q.
__global__ void k_dg_facets(int dim, int p, int npc, double eta, const double* __restrict__ x,
                            const int32_t* __restrict__ cell_dofs, const double* __restrict__ mu,
                            const double* __restrict__ tv, const double* __restrict__ tnd,
                            const double* __restrict__ M, const int32_t* __restrict__ fnbr,
                            const uint8_t* __restrict__ ftag, double* __restrict__ E) {
  extern __shared__ double sm[];
  const int n1 = p + 1, twod = 2 * dim;
  int nt = 1;
  for (int b = 1; b < dim; ++b) nt *= n1;
  double* G1 = sm;
  double* G2 = G1 + nt;
  double* H1 = G2 + nt;
  double* H2 = H1 + nt;
  const int r = blockIdx.x;
  for (int q = 0; q < dim; ++q) {
    int st[3], ns = 0;  // lattice strides of the tangential axes
    int stride_q = 1;
    for (int b = 0, s = 1; b < dim; ++b, s *= n1) {
      if (b == q)
        stride_q = s;
      else
        st[ns++] = s;
    }
    for (int side = 0; side < 2; ++side) {
      const int f = 2 * q + side;
      const int tag = ftag[size_t(r) * twod + f];
      if (tag == 2) continue;
      const double mr = mu[size_t(r) * dim + q];
      const int N = tag == 0 ? fnbr[size_t(r) * twod + f] : -1;
      const double mn = N >= 0 ? mu[size_t(N) * dim + q] : 0.0;
      // trace sums over the blocks (r, r) and (r, N)
      for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        const int off = ns == 0 ? 0 : ns == 1 ? t * st[0] : (t % n1) * st[0] + (t / n1) * st[1];
        double g1 = 0.0, g2 = 0.0;
        for (int blk = 0; blk < (N >= 0 ? 2 : 1); ++blk) {
          const int s = blk ? N : r;
          const int es = blk ? 1 - side : side;  // the neighbour sees the facet on its other side
          double t1 = 0.0, t2 = 0.0;
          const int32_t* cd = cell_dofs + size_t(s) * npc;
          for (int jj = 0; jj < n1; ++jj) {
            const double u = x[cd[off + jj * stride_q]];
            t1 += tv[es + 2 * jj] * u;
            t2 += tnd[es + 2 * jj] * u;
          }
          double alpha, beta, gamma;
          if (tag == 1) {
            alpha = eta * mr;
            beta = gamma = mr;
          } else {
            const double sign = blk ? -0.5 : 0.5;
            alpha = sign * eta * (mr + mn);
            beta = sign * (blk ? mn : mr);
            gamma = sign * mr;
          }
          g1 += alpha * t1 - beta * t2;
          g2 += gamma * t1;
        }
        G1[t] = g1;
        G2[t] = g2;
      }
      __syncthreads();
      // tangential mass (x) mass
      if (ns == 1) {
        for (int t = threadIdx.x; t < nt; t += blockDim.x) {
          double h1 = 0.0, h2 = 0.0;
          for (int k = 0; k < n1; ++k) {
            h1 += M[t + n1 * k] * G1[k];
            h2 += M[t + n1 * k] * G2[k];
          }
          H1[t] = h1;
          H2[t] = h2;
        }
      } else {
        for (int t = threadIdx.x; t < nt; t += blockDim.x) {  // first tangential axis
          const int t0 = t % n1, t1 = t / n1;
          double h1 = 0.0, h2 = 0.0;
          for (int k = 0; k < n1; ++k) {
            h1 += M[t0 + n1 * k] * G1[k + n1 * t1];
            h2 += M[t0 + n1 * k] * G2[k + n1 * t1];
          }
          H1[t] = h1;
          H2[t] = h2;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nt; t += blockDim.x) {  // second
          const int t0 = t % n1, t1 = t / n1;
          double h1 = 0.0, h2 = 0.0;
          for (int k = 0; k < n1; ++k) {
            h1 += M[t1 + n1 * k] * H1[t0 + n1 * k];
            h2 += M[t1 + n1 * k] * H2[t0 + n1 * k];
          }
          G1[t] = h1;
          G2[t] = h2;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nt; t += blockDim.x) {
          H1[t] = G1[t];
          H2[t] = G2[t];
        }
      }
      __syncthreads();
      double* Er = E + size_t(r) * npc;
      for (int lin = threadIdx.x; lin < npc; lin += blockDim.x) {
        const int i = (lin / stride_q) % n1;
        int t = 0;
        for (int k = ns - 1; k >= 0; --k) t = t * n1 + (lin / st[k]) % n1;
        Er[lin] += tv[side + 2 * i] * H1[t] - tnd[side + 2 * i] * H2[t];
      }
      __syncthreads();
    }
  }
}

}  // namespace

void launch_dg_patch_assemble(Context& c) {
  DgArgs a;
  a.dim = c.dim;
  a.p = c.p;
  a.n1 = c.n1;
  a.npc = c.npc;
  a.m = c.L.m;
  a.ntiles = c.L.ntiles;
  a.eta = c.eta;
  a.lat = c.lat.p;
  a.pcells = c.pcells.p;
  a.psep = c.pdofs.p;
  a.mu = c.mu.p;
  a.At = c.At.p;
  a.Bt = c.Bt.p;
  a.dtr = c.dtr.p;
  a.fnbr = c.fnbr.p;
  a.ftag = c.ftag.p;
  KernelTimer timer(c, 1);
  FDM_CUDA(cudaMemsetAsync(c.tiles.p, 0, c.tiles.bytes(), c.stream));
  const int ne = int(c.L.entries.size());
  dim3 grid(unsigned((ne + 255) / 256 < 64 ? (ne + 255) / 256 : 64), c.npatch);
  k_dg_patch_assemble<<<grid, 256, 0, c.stream>>>(a, ne, c.entries.p, c.tile_row.p, c.tile_col.p, c.tiles.p);
  FDM_LAUNCH_CHECK(c);
  if (c.L.mpad > c.L.m) {
    k_dg_pad<<<c.npatch, 64, 0, c.stream>>>(c.L.m, c.L.mpad, c.L.ntiles, c.L.col_start[c.L.nT - 1], c.tiles.p);
    FDM_LAUNCH_CHECK(c);
  }
}

void launch_dg_facets(Context& c, const double* x) {
  int nt = 1;
  for (int b = 1; b < c.dim; ++b) nt *= c.n1;
  const size_t smem = sizeof(double) * 4 * size_t(nt);
  KernelTimer timer(c, 3);
  k_dg_facets<<<c.ncells, 256, smem, c.stream>>>(c.dim, c.p, c.npc, c.eta, x, c.cell_dofs.p, c.mu.p, c.tv.p, c.tnd.p,
                                                 c.Bhat.p, c.fnbr.p, c.ftag.p, c.E.p);
  FDM_LAUNCH_CHECK(c);
}

}  // namespace fdmgpu
