#include <algorithm>
#include <cstdlib>
// Vertex-star patch kernels: batched numeric factorisation (K2), the
// patch relaxation solve (K3) and the deterministic patch owner-gather.
//
// Reference path replaced (src/schwarz.cpp:41-54, 84-93; src/cholesky.cpp:9-110):
//   for each patch j: A~_j = R_j A~ R_j^T, P A~_j P^T = L L^T (up-looking),
//   c_j = L^{-T} L^{-1} P r_j, then z += R_j^T c_j in ascending j.
//
// B200 layout.  All interior patches share one elimination order on the
// (2p-1)^d patch lattice (layout.cpp).  Interior DOFs are eliminated first
// and couple only to their cell's d near facets (zero fill),
// so their factor columns are never stored: the kernels rebuild
// D_k = A~_kk and A~_{f,k} from the per-cell mu and the 1D tables A_t / B_t.
// What is stored is the Cholesky factor of the separator Schur complement
// S_G = A~_GG - A~_GI D^{-1} A~_IG as dense 64x64 tiles on one shared tile
// pattern (diagonal tiles hold L_KK^{-1}, so the solves are pure GEMVs),
// streamed by the solve kernel through a TMA-bulk-copy / mbarrier ring.
#include "common.cuh"

namespace fdmgpu {

namespace {

constexpr int T = kTile;
constexpr int TT = kTile * kTile;

struct PatchArgs {
  int dim, p, n1, n, nI, m, mpad, nT, ntiles, span;
  const int32_t* lat;
  const int32_t* pos_of_lat;
  const int32_t* pcells;
  const int32_t* psep;  // npatch x m separator DOFs, -1 = absent (boundary star)
  const double* mu;
  const double* At;
  const double* Bt;
  unsigned long long* err;
  int64_t rec_stride;  // doubles per patch in the solve-record buffer
  int64_t out_stride;  // solve output: corr + j * out_stride + out_off (the separator solution)
  int out_off;
  double* diagL;       // Schur split: L_KK of the diagonal tiles K >= diagK0 (npatch x diagNT tiles), or null
  int diagK0, diagNT;
  const int32_t* err_map;  // pivot position of a failing row (component factorisations), or null: K T + row
};

PatchArgs make_args(Context& c) {
  PatchArgs a;
  a.dim = c.dim;
  a.p = c.p;
  a.n1 = c.n1;
  a.n = c.L.n;
  a.nI = c.L.nI;
  a.m = c.L.m;
  a.mpad = c.L.mpad;
  a.nT = c.L.nT;
  a.ntiles = c.L.ntiles;
  a.span = c.L.span;
  a.lat = c.lat.p;
  a.pos_of_lat = c.pos_of_lat.p;
  a.pcells = c.pcells.p;
  a.psep = c.pdofs.p;
  a.rec_stride = c.packed.p ? int64_t(c.L.tile_poff8.back()) : int64_t(c.L.ntiles) * TT;
  a.mu = c.mu.p;
  a.At = c.At.p;
  a.Bt = c.Bt.p;
  a.err = c.d_err.p;
  a.out_stride = c.L.m;
  a.out_off = 0;
  a.diagL = c.sx.on ? c.diagL.p : nullptr;
  a.diagK0 = c.sx_K0;
  a.diagNT = c.L.nT - c.sx_K0;
  a.err_map = nullptr;
  return a;
}

__device__ __forceinline__ void unpack(int32_t v, int* P) {
  P[0] = v & 255;
  P[1] = (v >> 8) & 255;
  P[2] = (v >> 16) & 255;
}

__device__ __forceinline__ int lin_of(const PatchArgs& a, const int* P) {
  int v = P[a.dim - 1];
  for (int b = a.dim - 2; b >= 0; --b) v = v * a.span + P[b];
  return v;
}

// The single axis on which lattice point P lies on a separator plane through
// the vertex (P_a == p), or -1 when it is interior (none) or edge/vertex (>1).
__device__ __forceinline__ int facet_axis(const PatchArgs& a, const int* P) {
  int fa = -1, cnt = 0;
  for (int b = 0; b < a.dim; ++b)
    if (P[b] == a.p) {
      fa = b;
      ++cnt;
    }
  return cnt == 1 ? fa : -1;
}

// A~^K_kk for a cell-interior lattice point l of cell with coefficients mus.
__device__ __forceinline__ double diag_interior(const PatchArgs& a, const double* mus, const int* l,
                                                const double* At, const double* Bt) {
  double s = 0.0;
  for (int q = 0; q < a.dim; ++q) {
    double prod = mus[q];
    for (int b = a.dim - 1; b >= 0; --b) prod *= (b == q ? At : Bt)[l[b] + a.n1 * l[b]];
    s += prod;
  }
  return s;
}

// A~^K(f, x) for facet point f (endpoint e on axis fa) and the interior point x
// that shares f's tangential indices; x_fa is the interior index.
__device__ __forceinline__ double facet_coupling(const PatchArgs& a, const double* mus, int fa, int e, int xa,
                                                 const int* l, const double* At, const double* Bt) {
  double prod = mus[fa] * At[e + a.n1 * xa];
  for (int b = 0; b < a.dim; ++b)
    if (b != fa) prod *= Bt[l[b] + a.n1 * l[b]];
  return prod;
}

// Entry (r, c) of the separator Schur complement S_G, r,c in [0, m).
// smask: star slots holding a cell (boundary stars miss some).
__device__ double schur_entry(const PatchArgs& a, const double* __restrict__ mu_patch, int smask, int r, int c,
                              const double* At, const double* Bt) {
  int P[3] = {0, 0, 0}, Q[3] = {0, 0, 0};
  unpack(a.lat[a.nI + r], P);
  unpack(a.lat[a.nI + c], Q);
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int b = 0; b < a.dim; ++b) {
    const int plo = P[b] > a.p ? 1 : 0, phi = P[b] < a.p ? 0 : 1;
    const int qlo = Q[b] > a.p ? 1 : 0, qhi = Q[b] < a.p ? 0 : 1;
    lo[b] = max(plo, qlo);
    hi[b] = min(phi, qhi);
    if (lo[b] > hi[b]) return 0.0;  // no common cell
  }
  const int fr = facet_axis(a, P), fc = facet_axis(a, Q);
  double v = 0.0;
  for (int s2 = lo[2]; s2 <= hi[2]; ++s2)
    for (int s1 = lo[1]; s1 <= hi[1]; ++s1)
      for (int s0 = lo[0]; s0 <= hi[0]; ++s0) {
        const int s[3] = {s0, s1, s2};
        const int slot = s0 | (s1 << 1) | (s2 << 2);
        if (!((smask >> slot) & 1)) continue;
        const double* mus = mu_patch + slot * a.dim;
        int lr[3] = {0, 0, 0}, lc[3] = {0, 0, 0};
        for (int b = 0; b < a.dim; ++b) {
          lr[b] = P[b] - s[b] * a.p;
          lc[b] = Q[b] - s[b] * a.p;
        }
        // cell block sum_q mu_q (x)_b (b == q ? A_t : B_t)  (src/assembly.cpp:263-270)
        double cv = 0.0;
        for (int q = 0; q < a.dim; ++q) {
          double prod = 1.0;
          for (int b = a.dim - 1; b >= 0; --b) prod *= (b == q ? At : Bt)[lr[b] + a.n1 * lc[b]];
          cv += prod * mus[q];
        }
        // minus the elimination of this cell's interior block
        double sc = 0.0;
        if (fr >= 0 && fc >= 0) {
          bool same_tan = true;
          for (int b = 0; b < a.dim; ++b)
            if (b != fr && b != fc && lr[b] != lc[b]) same_tan = false;
          if (same_tan) {
            if (fr == fc) {
              int x[3] = {lr[0], lr[1], lr[2]};
              for (int xi = 1; xi < a.p; ++xi) {
                x[fr] = xi;
                const double cp = facet_coupling(a, mus, fr, lr[fr], xi, x, At, Bt);
                sc += cp * cp / diag_interior(a, mus, x, At, Bt);
              }
            } else {
              int x[3] = {lr[0], lr[1], lr[2]};
              x[fr] = lc[fr];
              x[fc] = lr[fc];
              const double cr = facet_coupling(a, mus, fr, lr[fr], x[fr], x, At, Bt);
              const double cc = facet_coupling(a, mus, fc, lc[fc], x[fc], x, At, Bt);
              sc = cr * cc / diag_interior(a, mus, x, At, Bt);
            }
          }
        }
        v += cv - sc;
      }
  return v;
}

__device__ __forceinline__ void record_pivot_error(unsigned long long* err, int patch, int pivot) {
  if (err) atomicMin(err, (static_cast<unsigned long long>(patch) << 32) | static_cast<unsigned>(pivot));
}

// Separator Schur complement S_G on the structural nonzeros only (`entries`,
// shared by all patches); all other stored tile entries were zeroed first.
// (patches j0 + blockIdx.y; tiles indexed by blockIdx.y)
__global__ void k_patch_assemble(PatchArgs a, int nentries, const int32_t* __restrict__ entries,
                                 const int32_t* __restrict__ tile_row, const int32_t* __restrict__ tile_col,
                                 double* __restrict__ tiles, int j0) {
  extern __shared__ double sm[];
  double* At = sm;
  double* Bt = At + a.n1 * a.n1;
  double* mup = Bt + a.n1 * a.n1;  // 2^d x d
  const int j = j0 + blockIdx.y;
  const int ncorner = 1 << a.dim;
  for (int i = threadIdx.x; i < a.n1 * a.n1; i += blockDim.x) {
    At[i] = a.At[i];
    Bt[i] = a.Bt[i];
  }
  int smask = 0;
  for (int s = 0; s < ncorner; ++s) smask |= (a.pcells[size_t(j) * ncorner + s] >= 0) << s;
  for (int i = threadIdx.x; i < ncorner * a.dim; i += blockDim.x) {
    const int s = i / a.dim, q = i % a.dim, K = a.pcells[size_t(j) * ncorner + s];
    mup[i] = K >= 0 ? a.mu[size_t(K) * a.dim + q] : 0.0;
  }
  __syncthreads();
  double* base = tiles + size_t(blockIdx.y) * a.ntiles * TT;
  const int32_t* sep = a.psep + size_t(j) * a.m;
  const bool whole = smask == (1 << ncorner) - 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nentries; e += gridDim.x * blockDim.x) {
    const int code = entries[e];
    const int t = code >> 12, cc = (code >> 6) & 63, rr = code & 63;
    const int r = tile_row[t] * T + rr, c = tile_col[t] * T + cc;
    double v;
    if (!whole && (sep[r] < 0 || sep[c] < 0))
      v = r == c ? 1.0 : 0.0;  // absent position of a boundary star: decoupled identity row
    else
      v = schur_entry(a, mup, smask, r, c, At, Bt);
    base[size_t(t) * TT + tsw(rr, cc)] = v;
  }
}

// Identity on the padded separator positions m..mpad-1 (last diagonal tile)
// and the interior pivots D_k > 0 (the first n_I pivots of the reference order).
__global__ void k_patch_pad_check(PatchArgs a, double* __restrict__ tiles, int last_diag) {
  const int j = blockIdx.x;
  double* dt = tiles + (size_t(j) * a.ntiles + last_diag) * TT;
  if (tiles)
    for (int r = a.m + threadIdx.x; r < a.mpad; r += blockDim.x) dt[tsw(r % T, r % T)] = 1.0;
  const int ncorner = 1 << a.dim;
  double mup[24];
  for (int i = 0; i < ncorner * a.dim; ++i) {
    const int K = a.pcells[size_t(j) * ncorner + i / a.dim];
    mup[i] = K >= 0 ? a.mu[size_t(K) * a.dim + i % a.dim] : 0.0;
  }
  for (int k = threadIdx.x; k < a.nI; k += blockDim.x) {
    int P[3] = {0, 0, 0}, s[3] = {0, 0, 0}, l[3] = {0, 0, 0};
    unpack(a.lat[k], P);
    for (int b = 0; b < a.dim; ++b) {
      s[b] = P[b] > a.p ? 1 : 0;
      l[b] = P[b] - s[b] * a.p;
    }
    const int slot = s[0] | (s[1] << 1) | (s[2] << 2);
    if (a.pcells[size_t(j) * ncorner + slot] < 0) continue;  // missing cell of a boundary star
    if (!(diag_interior(a, mup + slot * a.dim, l, a.At, a.Bt) > 0.0)) record_pivot_error(a.err, j, k);
  }
}

// Warp-tiled FP64 tensor-core GEMM on swizzled 64x64 tiles: acc += A B^T.
// 8 warps; warp w owns rows 32 (w >> 2) .. +31 and columns 16 (w & 3) .. +15
// as 4 x 2 DMMA m8n8k4 accumulators (16 doubles per thread).  Fragment loads
// are conflict-free on the tile swizzle (common.cuh).
struct TileAcc {
  double v[4][2][2];
  __device__ __forceinline__ int row(int i) const { return 32 * ((threadIdx.x >> 5) >> 2) + 8 * i + ((threadIdx.x & 31) >> 2); }
  __device__ __forceinline__ int col(int j, int e) const {
    return 16 * ((threadIdx.x >> 5) & 3) + 8 * j + 2 * (threadIdx.x & 3) + e;
  }
};

__device__ __forceinline__ void tile_gemm_abt(const double* __restrict__ A, const double* __restrict__ B, TileAcc& acc,
                                              int maskA = 0xffff, int maskB = 0xffff) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = w >> 2, wc = w & 3;
  const int r0 = 32 * wr + (lane >> 2), c0 = 16 * wc + (lane >> 2), kl = lane & 3;
  // 16-wide k panels q where this warp's A rows (sub-block rows 2wr, 2wr+1)
  // and B rows (sub-block row wc) hold structural nonzeros (warp uniform).
  int qmask = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool a_on = ((maskA >> ((2 * wr) * 4 + q)) | (maskA >> ((2 * wr + 1) * 4 + q))) & 1;
    const bool b_on = (maskB >> (wc * 4 + q)) & 1;
    if (a_on && b_on) qmask |= 1 << q;
  }
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    if (!((qmask >> q) & 1)) continue;
#pragma unroll
    for (int k0 = 16 * q; k0 < 16 * q + 16; k0 += 4) {
      const int k = k0 + kl;
      double av[4], bv[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = A[tsw(r0 + 8 * i, k)];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) bv[jj] = B[tsw(c0 + 8 * jj, k)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) dmma884(acc.v[i][jj][0], acc.v[i][jj][1], av[i], bv[jj]);
    }
  }
}

// POTRF + triangular inverse of the 64x64 SPD tile in Dm (column-major, ld 65),
// 256 threads; writes L^{-1} (lower, diag included) swizzled into `out`.
// Rank-4 blocked and register resident: thread t owns column c = t / 4, rows
// r = 4 i + t % 4 (i < 16).  Per 4-column panel the owner warp factors the
// panel in shared memory (Lp keeps all 16 panels, row-major by 4), one
// barrier, then every thread applies the rank-4 update to its registers.
// The inverse W = L^{-1} runs 4 rows at a time per column, warp local: the
// column's 4 lanes finalise one row each (shuffles), then fold the block into
// their running sums of the rows below (rotated so indices stay static).
__device__ void diag_factor_invert(double* Dm, double* Wm, double* out, const PatchArgs& a, int K, int patch) {
  constexpr int LD = T + 1;
  double* Lp = Wm;                 // [16][T][4]
  double* rdiag = Lp + 16 * T * 4;  // [T]
  const int tid = threadIdx.x, lane = tid & 31, c = tid >> 2, rq = tid & 3, warp = tid >> 5;
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = Dm[c * LD + 4 * i + rq];
#pragma unroll 1
  for (int jb = 0; jb < 16; ++jb) {
    const int j0 = 4 * jb;
    double* P = Lp + size_t(jb) * T * 4;
    if (warp == (jb >> 1)) {  // owner warp: columns j0..j0+3 are lanes 16 (jb & 1) .. + 15
      if ((c >> 2) == jb) {
#pragma unroll
        for (int i = 0; i < 16; ++i) P[(4 * i + rq) * 4 + (c - j0)] = v[i];
      }
      __syncwarp();
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = j0 + jj;
        double d = P[j * 4 + jj];
        if (lane == 0 && !(d > 0.0)) {
          const int pos = a.err_map ? a.err_map[j] : K * T + j;
          if (pos >= 0 && pos < a.m) record_pivot_error(a.err, patch, a.nI + pos);
        }
        if (!(d > 0.0)) d = 1.0;
        const double s = rsqrt(d);
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = lane + 32 * h;
          if (r > j) P[r * 4 + jj] *= s;
          if (r == j) P[r * 4 + jj] = d * s;
        }
        if (lane == 0) rdiag[j] = s;
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = lane + 32 * h;
#pragma unroll
          for (int j2 = jj + 1; j2 < 4; ++j2)
            if (r >= j0 + j2) P[r * 4 + j2] -= P[r * 4 + jj] * P[(j0 + j2) * 4 + jj];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (c >= j0 + 4) {  // rank-4 update of the thread's column (all rows; the upper part is unused)
      const double4 lc = *reinterpret_cast<const double4*>(P + c * 4);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double4 lr = *reinterpret_cast<const double4*>(P + (4 * i + rq) * 4);
        v[i] = fma(-lr.x, lc.x, fma(-lr.y, lc.y, fma(-lr.z, lc.z, fma(-lr.w, lc.w, v[i]))));
      }
    }
  }
  // inverse: W(k, c) = (delta_kc - sum_{c <= m < k} L(k, m) W(m, c)) / L(k, k)
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = 0.0;  // running sums of rows 4 (kb + i) + rq
#pragma unroll 1
  for (int kb = 0; kb < 16; ++kb) {
    const double* P = Lp + size_t(kb) * T * 4;
    double wv[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int k = 4 * kb + m;
      double sum = v[0];
#pragma unroll
      for (int m2 = 0; m2 < m; ++m2) sum = fma(P[k * 4 + m2], wv[m2], sum);
      const double my = ((k == c ? 1.0 : 0.0) - sum) * rdiag[k];
      wv[m] = __shfl_sync(0xffffffffu, my, (lane & ~3) | m);
    }
    double mine = wv[0];
#pragma unroll
    for (int m = 1; m < 4; ++m) mine = rq == m ? wv[m] : mine;
    Dm[c * LD + 4 * kb + rq] = mine;  // Dm is free: L lives in Lp
#pragma unroll
    for (int i = 1; i < 16; ++i) {
      const int r = 4 * (kb + i) + rq;
      if (r < T) {
        const double4 l = *reinterpret_cast<const double4*>(P + r * 4);
        v[i] = fma(l.x, wv[0], fma(l.y, wv[1], fma(l.z, wv[2], fma(l.w, wv[3], v[i]))));
      }
    }
#pragma unroll
    for (int i = 0; i < 15; ++i) v[i] = v[i + 1];
    v[15] = 0.0;
  }
  __syncthreads();
  for (int e = tid; e < TT; e += blockDim.x) {
    const int r = e % T, cc = e / T;
    out[tsw(r, cc)] = r >= cc ? Dm[cc * LD + r] : 0.0;
  }
  if (a.diagL && K >= a.diagK0 && patch >= 0) {  // the Schur split re-tiles L_RR from L itself
    double* o = a.diagL + (size_t(patch) * a.diagNT + (K - a.diagK0)) * TT;
    for (int e = tid; e < TT; e += blockDim.x) {
      const int r = e % T, cc = e / T;
      o[tsw(r, cc)] = r >= cc ? Lp[size_t(cc >> 2) * T * 4 + r * 4 + (cc & 3)] : 0.0;
    }
  }
}

constexpr int kUpdThreads = 256;
constexpr int kUpdStages = 3;  // TMA pipeline depth (2 operand tiles per stage, 64 KB)

// Left-looking update of tile column K: C(I,K) = A(I,K) - sum_J L(I,J) L(K,J)^T
// for every stored tile (I,K); the CTA owning the diagonal tile then factors
// and inverts it.  Operand tiles arrive by TMA bulk copy, double-buffered.
__global__ void __launch_bounds__(kUpdThreads, 3) k_patch_update(PatchArgs a, int K, const int32_t* __restrict__ active,
                                                                const int32_t* __restrict__ tile_row,
                                                                const int32_t* __restrict__ pair_ptr,
                                                                const int32_t* __restrict__ pair_a,
                                                                const int32_t* __restrict__ pair_b,
                                                                const int32_t* __restrict__ tile_mask,
                                                                double* __restrict__ tiles, int nst) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);  // nst (<= 3) barriers
  double* buf = sm + 16;                              // [stages][A,B][TT] (128-byte aligned)
  const int t = active[blockIdx.x], j = blockIdx.y;  // tiles of column K with work
  const int I = tile_row[t];
  if (K < 0) K = I;  // batched leading columns: diagonal tiles without updates
  double* base = tiles + size_t(j) * a.ntiles * TT;
  const int p0 = pair_ptr[t], np = pair_ptr[t + 1] - p0;
  const int tid = threadIdx.x;
  pdl_trigger();
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();  // operands of column K-1 come from the previous launch
  // Whole operand tiles (one 32 KB bulk copy each).  Copying only the 16-column
  // panels the GEMM reads moved fewer bytes but was slower (C5 factor 917 -> 959 ms,
  // C3 unchanged: the light columns are not operand-bandwidth bound).
  auto issue = [&](int s, int i) {
    mbar_arrive_expect_tx(&full[s], 2 * TT * sizeof(double));
    bulk_g2s(buf + (2 * s) * TT, base + size_t(pair_a[p0 + i]) * TT, TT * sizeof(double), &full[s]);
    bulk_g2s(buf + (2 * s + 1) * TT, base + size_t(pair_b[p0 + i]) * TT, TT * sizeof(double), &full[s]);
  };
  if (tid == 0)
    for (int s = 0; s < nst && s < np; ++s) issue(s, s);
  TileAcc acc = {};
  for (int i = 0; i < np; ++i) {
    const int s = i % nst;
    mbar_wait(&full[s], (i / nst) & 1);
    tile_gemm_abt(buf + (2 * s) * TT, buf + (2 * s + 1) * TT, acc, tile_mask[pair_a[p0 + i]], tile_mask[pair_b[p0 + i]]);
    __syncthreads();
    if (tid == 0 && i + nst < np) issue(s, i + nst);
  }
  double* ct = base + size_t(t) * TT;
  if (I != K) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) ct[tsw(acc.row(i), acc.col(jj, e))] -= acc.v[i][jj][e];
    return;
  }
  constexpr int LD = T + 1;
  double* Dm = buf;           // reuse the operand buffers (all copies consumed)
  double* Wm = buf + T * LD;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = acc.row(i), cc = acc.col(jj, e);
        Dm[cc * LD + r] = ct[tsw(r, cc)] - acc.v[i][jj][e];
      }
  __syncthreads();
  diag_factor_invert(Dm, Wm, ct, a, K, j);
}

// Fused tile column K: for every stored tile (I, K) of every patch,
// C(I,K) = A(I,K) - sum_J L(I,J) L(K,J)^T (left-looking, as k_patch_update);
// the diagonal CTA factors and inverts its tile and publishes L_KK^{-1} through
// a device-scope flag; each off-diagonal CTA then finishes
// L(I,K) = C(I,K) L_KK^{-T} itself (k_patch_trsm's GEMM) -- one launch per
// column instead of two, and C(I,K) never leaves the SM.  1D grid: blocks
// [0, npatch) are the diagonal tiles of every patch, the rest the off-diagonal
// tiles patch by patch (consecutive CTAs share their patch's L(K,J) operands in
// L2).  Every diagonal CTA has a lower block index than any off-diagonal CTA,
// so it is dispatched first and the waits cannot starve it.
__global__ void __launch_bounds__(kUpdThreads, 3) k_patch_column(PatchArgs a, int K, const int32_t* __restrict__ col_start,
                                                                const int32_t* __restrict__ pair_ptr,
                                                                const int32_t* __restrict__ pair_a,
                                                                const int32_t* __restrict__ pair_b,
                                                                const int32_t* __restrict__ tile_mask,
                                                                double* __restrict__ tiles,
                                                                unsigned* __restrict__ diag_flag, unsigned epoch) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  double* buf = sm + 16;  // [A, B][TT] operand stage, then Dm / Wm or C / L_KK^{-1}
  const int t0 = col_start[K], noff = col_start[K + 1] - t0 - 1;
  const int npatch = int(gridDim.x) / (noff + 1), b = blockIdx.x;
  const int j = b < npatch ? b : (b - npatch) / noff;
  const int t = b < npatch ? t0 : t0 + 1 + (b - npatch) % noff;
  double* base = tiles + size_t(j) * a.ntiles * TT;
  const int p0 = pair_ptr[t], np = pair_ptr[t + 1] - p0;
  const int tid = threadIdx.x;
  pdl_trigger();
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();  // operands of column K-1 come from the previous launch
  auto issue = [&](int i) {
    mbar_arrive_expect_tx(&full[0], 2 * TT * sizeof(double));
    bulk_g2s(buf, base + size_t(pair_a[p0 + i]) * TT, TT * sizeof(double), &full[0]);
    bulk_g2s(buf + TT, base + size_t(pair_b[p0 + i]) * TT, TT * sizeof(double), &full[0]);
  };
  if (tid == 0 && np > 0) issue(0);
  TileAcc acc = {};
  for (int i = 0; i < np; ++i) {
    mbar_wait(&full[0], i & 1);
    tile_gemm_abt(buf, buf + TT, acc, tile_mask[pair_a[p0 + i]], tile_mask[pair_b[p0 + i]]);
    __syncthreads();
    if (tid == 0 && i + 1 < np) issue(i + 1);
  }
  double* ct = base + size_t(t) * TT;
  if (t == t0) {  // diagonal tile: factor, invert, publish
    constexpr int LD = T + 1;
    double* Dm = buf;
    double* Wm = buf + T * LD;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = acc.row(i), cc = acc.col(jj, e);
          Dm[cc * LD + r] = ct[tsw(r, cc)] - acc.v[i][jj][e];
        }
    __syncthreads();
    diag_factor_invert(Dm, Wm, ct, a, K, j);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(diag_flag + size_t(j) * a.nT + K), "r"(epoch) : "memory");
    }
    return;
  }
  double* Cs = buf;
  double* Ls = buf + TT;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int idx = tsw(acc.row(i), acc.col(jj, e));
        Cs[idx] = ct[idx] - acc.v[i][jj][e];
      }
  if (tid == 0) wait_geq(diag_flag + size_t(j) * a.nT + K, epoch);
  __syncthreads();
  const double2* dt = reinterpret_cast<const double2*>(base + size_t(t0) * TT);
  for (int i = tid; i < TT / 2; i += kUpdThreads) reinterpret_cast<double2*>(Ls)[i] = __ldcg(dt + i);
  __syncthreads();
  TileAcc lk = {};
  tile_gemm_abt(Cs, Ls, lk, tile_mask[t], tile_mask[t0]);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
      for (int e = 0; e < 2; ++e) ct[tsw(lk.row(i), lk.col(jj, e))] = lk.v[i][jj][e];
}

// L(I,K) = C(I,K) L_KK^{-T} for the off-diagonal tiles of column K.
__global__ void __launch_bounds__(kUpdThreads) k_patch_trsm(PatchArgs a, int K, const int32_t* __restrict__ col_start,
                                                              const int32_t* __restrict__ lead,
                                                              const int32_t* __restrict__ tile_mask,
                                                              double* __restrict__ tiles) {
  extern __shared__ __align__(128) double sm[];
  double* Cs = sm;
  double* Ls = sm + TT;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + 2 * TT);
  // K < 0: batched leading columns, (tile, diagonal tile) pairs in `lead`
  const int t0 = K >= 0 ? col_start[K] : lead[2 * blockIdx.x + 1];
  const int t = K >= 0 ? t0 + 1 + blockIdx.x : lead[2 * blockIdx.x], j = blockIdx.y;
  double* base = tiles + size_t(j) * a.ntiles * TT;
  const int tid = threadIdx.x;
  pdl_trigger();
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();
  if (tid == 0) {
    mbar_arrive_expect_tx(&full[0], 2 * TT * sizeof(double));
    bulk_g2s(Cs, base + size_t(t) * TT, TT * sizeof(double), &full[0]);
    bulk_g2s(Ls, base + size_t(t0) * TT, TT * sizeof(double), &full[0]);
  }
  mbar_wait(&full[0], 0);
  TileAcc acc = {};
  tile_gemm_abt(Cs, Ls, acc, tile_mask[t], tile_mask[t0]);
  double* out = base + size_t(t) * TT;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
      for (int e = 0; e < 2; ++e) out[tsw(acc.row(i), acc.col(jj, e))] = acc.v[i][jj][e];
}


// ---- K3: patch relaxation solve -------------------------------------------------
constexpr int kSolveConsumers = 8;                         // consumer warps
constexpr int kSolveThreads = 32 * (kSolveConsumers + 1);  // + 1 TMA producer warp
constexpr int SB8 = 64;   // doubles per packed 8x8 sub-block (solve stream)
constexpr int kHdr = kHdrBytes / 8;  // doubles of the per-tile stream header (context.hpp)
constexpr int kSlot = TT + kHdr;  // ring slot: the densest possible record

// Packed solve stream.  After factorisation every 64x64 tile is compacted
// into one record (layout.cpp): the kHdrBytes header (tile_hdr: record index
// of each sub-block, row- and column-major, and the full / compact block
// counts), the structurally nonzero full 8x8 sub-blocks (layout below), then
// the compact sub-blocks (at most one structural entry per row: the 8 row
// values and the 8 column bytes).  Exact: the dropped entries are structural
// zeros of the factor.  `cur` is the dense swizzled tile, `blk` / `ccol` the
// tile's record sub-blocks (bit bi*8 + bj) and compact column bytes.
__device__ __forceinline__ void write_record(const double* __restrict__ cur, double* __restrict__ dst,
                                             const uint8_t* __restrict__ hdr_t, const int32_t* __restrict__ blk,
                                             const int64_t* __restrict__ ccol) {
  if (threadIdx.x < kHdr) dst[threadIdx.x] = reinterpret_cast<const double*>(hdr_t)[threadIdx.x];
  const int nf = reinterpret_cast<const int32_t*>(hdr_t + 128)[0], nc = reinterpret_cast<const int32_t*>(hdr_t + 128)[1];
  dst += kHdr;
  for (int d = threadIdx.x; d < nf * SB8; d += blockDim.x) {
    const int bit = blk[d >> 6], w = d & 63;
    const int bi = bit >> 3, bj = bit & 7, rr = w >> 3, cc = 2 * (((w >> 1) & 3) ^ ((rr >> 1) & 3)) + (w & 1);
    dst[d] = cur[tsw(8 * bi + rr, 8 * bj + cc)];
  }
  dst += nf * SB8;
  for (int d = threadIdx.x; d < nc * kCompact; d += blockDim.x) {
    const int cb = d / kCompact, w = d - cb * kCompact;
    const int bit = blk[nf + cb];
    const long long cc = ccol[nf + cb];
    double v = 0.0;
    if (w < 8)
      v = cur[tsw(8 * (bit >> 3) + w, 8 * (bit & 7) + int((cc >> (8 * w)) & 0xff))];
    else if (w == 8)
      v = __longlong_as_double(cc);
    else
      v = __longlong_as_double(static_cast<long long>(bit));
    dst[d] = v;
  }
  if (nc > 0 && threadIdx.x < 16)  // compact index table
    dst[nc * kCompact + threadIdx.x] = reinterpret_cast<const double*>(hdr_t + kHdrBytes)[threadIdx.x];
}

__global__ void k_patch_pack(int ntiles, const int32_t* __restrict__ bptr, const int32_t* __restrict__ blk,
                             const int64_t* __restrict__ ccol, const int32_t* __restrict__ poff8,
                             const uint8_t* __restrict__ hdr, double* __restrict__ tiles) {
  extern __shared__ __align__(128) double tile[];  // 2 x TT (double buffer, filled by TMA)
  __shared__ __align__(8) uint64_t bar[2];
  double* base = tiles + size_t(blockIdx.x) * ntiles * TT;
  auto load = [&](int t) {  // one thread
    mbar_arrive_expect_tx(&bar[t & 1], TT * sizeof(double));
    bulk_g2s(tile + (t & 1) * TT, base + size_t(t) * TT, TT * sizeof(double), &bar[t & 1]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) load(0);
  for (int t = 0; t < ntiles; ++t) {
    // Prefetch t+1 (its buffer was released by the barrier ending t-1).  Its
    // source region starts at (t+1)*TT >= the end of tile t's packed
    // destination, so the in-place compaction never overwrites unread data.
    if (threadIdx.x == 0 && t + 1 < ntiles) load(t + 1);
    mbar_wait(&bar[t & 1], (t >> 1) & 1);
    write_record(tile + (t & 1) * TT, base + size_t(poff8[t]), hdr + size_t(t) * kHdrHost, blk + bptr[t],
                 ccol + bptr[t]);
    __syncthreads();
  }
}

// Same records into a separate buffer, for the tiles [t0, t0 + gridDim.x) of
// every patch (blockIdx.y): launched per tile column on a side stream while
// the factorisation continues, so the packing hides under the compute-bound
// updates (the dense tiles stay intact as update operands).
__global__ void __launch_bounds__(256) k_patch_pack_cols(int t0, int ntiles, const int32_t* __restrict__ bptr,
                                                        const int32_t* __restrict__ blk,
                                                        const int64_t* __restrict__ ccol,
                                                        const int32_t* __restrict__ poff8,
                                                        const uint8_t* __restrict__ hdr,
                                                        const double* __restrict__ tiles, double* __restrict__ packed,
                                                        int64_t pstride) {
  __shared__ __align__(16) double cur[TT];
  const int t = t0 + blockIdx.x, j = blockIdx.y;
  const double2* src = reinterpret_cast<const double2*>(tiles + (size_t(j) * ntiles + t) * TT);
  for (int i = threadIdx.x; i < TT / 2; i += blockDim.x) reinterpret_cast<double2*>(cur)[i] = __ldcs(src + i);
  __syncthreads();
  write_record(cur, packed + size_t(j) * pstride + poff8[t], hdr + size_t(t) * kHdrHost, blk + bptr[t],
               ccol + bptr[t]);
}

// Packed 8x8 sub-block layout: row-major, element (r, c) at
// r*8 + 2*((c >> 1) ^ ((r >> 1) & 3)) + (c & 1).  Lane (r = lane & 7,
// g = lane >> 3) owns block-columns g and 7 - g (balanced on the triangular
// diagonal tiles) and reads row r of a sub-block as four 16-byte loads,
// conflict free per quarter-warp.  Both solve directions use this lane map:
//   forward  (y_I -= L_IK y_K): 8 row sums per lane, closed by two shuffles;
//   backward (u_K -= L_IK^T y_I): 16 column partials per lane accumulated over
//            the tiles of a column, reduced across the 8 row lanes once.
// Absent sub-blocks read a shared zero block instead of branching, so every
// tile is one straight-line sequence of independent loads and FMA chains.
__device__ __forceinline__ void ld_row8(const double* __restrict__ B, int r, double v[8]) {
  const double2* row = reinterpret_cast<const double2*>(B + r * 8);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double2 t = row[j ^ ((r >> 1) & 3)];
    v[2 * j] = t.x;
    v[2 * j + 1] = t.y;
  }
}

// Sub-block (bi, bj) of a stream record: header byte -> full block (absent
// and compact sub-blocks read the shared zero block; compact ones are added
// by compact_fwd / compact_bwd after the branch-free full-block pass).
__device__ __forceinline__ const double* rec_block(const double* rec, const double* zblk, unsigned long long hw,
                                                   int e) {
  const unsigned idx = unsigned(hw >> (8 * e)) & 0xffu;
  return idx == 0xffu ? zblk : rec + kHdr + idx * SB8;
}

// Compact sub-blocks of a record (at most one entry per row): slot = 8 row
// values, the 8 column bytes, the sub-block bit.  After the compact blocks the
// record holds the compact index table (row-major then column-major bytes,
// 0xff = not compact), read exactly like the header: the compact pass runs
// the full-block loop structure with one value per lane row, absent positions
// reading a zero slot, so it stays branch-free (only records with compact
// blocks take it; warp-uniform).
__device__ __forceinline__ int rec_ncompact(const double* rec) { return reinterpret_cast<const int*>(rec)[33]; }
__device__ __forceinline__ const double* rec_compact(const double* rec) {
  return rec + kHdr + reinterpret_cast<const int*>(rec)[32] * SB8;
}
__device__ __forceinline__ const double* cmp_slot(const double* cbase, const double* czero, unsigned long long hw, int e) {
  const unsigned idx = unsigned(hw >> (8 * e)) & 0xffu;
  return idx == 0xffu ? czero : cbase + idx * kCompact;
}

// Forward: o0 / o1 (rows 8g + r, 8(7-g) + r) += L(row, 8 bj + col_r) x(8 bj + col_r).
__device__ __forceinline__ void compact_fwd(const double* __restrict__ rec, const double* __restrict__ czero, int r,
                                            int g, const double (&x)[64], double& o0, double& o1) {
  const int nc = rec_ncompact(rec);
  if (nc == 0) return;
  const double* cbase = rec_compact(rec);
  const unsigned long long* crow = reinterpret_cast<const unsigned long long*>(cbase + nc * kCompact);
  const unsigned long long hw0 = crow[g], hw1 = crow[7 - g];
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int bj = 0; bj < 8; ++bj) {
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const double* cb = cmp_slot(cbase, czero, jj ? hw1 : hw0, bj);
      const double val = cb[r];
      const int col = reinterpret_cast<const unsigned char*>(cb + 8)[r];
      double xs = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) xs = k == col ? x[8 * bj + k] : xs;
      if (jj)
        a1 = fma(val, xs, a1);
      else
        a0 = fma(val, xs, a0);
    }
  }
  o0 += a0;
  o1 += a1;
}

// Backward: acc[jj][col_r] += L(8 bi + r, 8 bj + col_r) y(8 bi + r) for bj = g (jj 0) / 7 - g (jj 1).
__device__ __forceinline__ void compact_bwd(const double* __restrict__ rec, const double* __restrict__ czero, int r,
                                            int g, const double yv[8], double (&acc)[2][8]) {
  const int nc = rec_ncompact(rec);
  if (nc == 0) return;
  const double* cbase = rec_compact(rec);
  const unsigned long long* ccolt = reinterpret_cast<const unsigned long long*>(cbase + nc * kCompact) + 8;
#pragma unroll
  for (int jj = 0; jj < 2; ++jj) {
    const unsigned long long hw = ccolt[jj ? 7 - g : g];
#pragma unroll
    for (int bi = 0; bi < 8; ++bi) {
      const double* cb = cmp_slot(cbase, czero, hw, bi);
      const double t = cb[r] * yv[bi];
      const int col = reinterpret_cast<const unsigned char*>(cb + 8)[r];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[jj][k] += k == col ? t : 0.0;
    }
  }
}

// Forward, rows map: lane (r, g) owns block-rows g and 7 - g (two sub-block
// rows of 8 doubles each per block-column) and the whole x = y_K in
// registers, so its two output rows need no cross-lane reduction.
__device__ __forceinline__ void tile_fwd(const double* __restrict__ rec, const double* __restrict__ zblk, int r, int g,
                                         const double (&x)[64], double& o0, double& o1, const double* __restrict__ xs) {
  const unsigned long long* hrow = reinterpret_cast<const unsigned long long*>(rec);  // [bi][bj] bytes
  const unsigned long long hw0 = hrow[g], hw1 = hrow[7 - g];
  double a[2][4];  // 4 independent chains per output row (both rows interleaved)
#pragma unroll
  for (int jj = 0; jj < 2; ++jj)
#pragma unroll
    for (int k = 0; k < 4; ++k) a[jj][k] = 0.0;
#pragma unroll
  for (int bj = 0; bj < 8; ++bj) {
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      double v[8];
      ld_row8(rec_block(rec, zblk, jj ? hw1 : hw0, bj), r, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[jj][k & 3] = fma(v[k], x[8 * bj + k], a[jj][k & 3]);
    }
  }
  o0 = (a[0][0] + a[0][1]) + (a[0][2] + a[0][3]);
  o1 = (a[1][0] + a[1][1]) + (a[1][2] + a[1][3]);
  compact_fwd(rec, zblk, r, g, x, o0, o1);
}

// Backward, columns map: acc[jj][k] += sum_bi L_tile(8 bi + r, 8 bj + k) * yv[bi]
// for the lane's block-columns bj = g, 7 - g;  yv[bi] = x[8 bi + r].
__device__ __forceinline__ void tile_bwd(const double* __restrict__ rec, const double* __restrict__ zblk, int r, int g,
                                         const double yv[8], double (&acc)[2][8], const double* __restrict__ ys) {
  const unsigned long long* hcol = reinterpret_cast<const unsigned long long*>(rec) + 8;  // [bj][bi] bytes
#pragma unroll
  for (int jj = 0; jj < 2; ++jj) {
    const unsigned long long hw = hcol[jj ? 7 - g : g];
#pragma unroll
    for (int bi = 0; bi < 8; ++bi) {
      double v[8];
      ld_row8(rec_block(rec, zblk, hw, bi), r, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[jj][k] = fma(v[k], yv[bi], acc[jj][k]);
    }
  }
  compact_bwd(rec, zblk, r, g, yv, acc);
}

// Sum acc over the 8 row lanes sharing g (recursive halving, 14 shuffles).
// The lane ends with columns c and c + 1 of the 64-column tile.
__device__ __forceinline__ void reduce_cols(const double (&acc)[2][8], int lane, double& s0, double& s1, int& c) {
  double w8[8], w4[4];
  {
    const bool up = lane & 4;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double lo = acc[0][i], hi = acc[1][i];
      w8[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, 4);
    }
  }
  {
    const bool up = lane & 2;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      w4[i] = (up ? w8[i + 4] : w8[i]) + __shfl_xor_sync(0xffffffffu, up ? w8[i] : w8[i + 4], 2);
  }
  const bool up = lane & 1;
  s0 = (up ? w4[2] : w4[0]) + __shfl_xor_sync(0xffffffffu, up ? w4[0] : w4[2], 1);
  s1 = (up ? w4[3] : w4[1]) + __shfl_xor_sync(0xffffffffu, up ? w4[1] : w4[3], 1);
  const int g = lane >> 3, jj = (lane >> 2) & 1, k = 4 * ((lane >> 1) & 1) + 2 * (lane & 1);
  c = 8 * (jj ? 7 - g : g) + k;
}

__device__ __forceinline__ void load_x(const double* __restrict__ x, double (&xr)[64]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double2 t = reinterpret_cast<const double2*>(x)[j];
    xr[2 * j] = t.x;
    xr[2 * j + 1] = t.y;
  }
}

// One CTA per patch.  A producer warp streams the patch's packed separator
// factor records (forward order, then backward by column) into a byte ring
// of shared memory with cp.async.bulk; kRingEntries mbarrier pairs track the
// records in flight, so the prefetch depth is set by bytes (~9 average
// records in ~200 KB), not by the largest record.  Stream position q goes to
// consumer warp q % 8 and ring entry q % 16: each entry is only ever waited
// on by one warp, in order, so an mbarrier can never be two phases ahead of
// its waiter.  The producer frees ring bytes in stream order (the oldest
// record first).  Output: the separator solution.
constexpr int kRingEntries = 16;

__global__ void __launch_bounds__(kSolveThreads)
    k_patch_solve(PatchArgs a, int ring_len, const double* __restrict__ rt, double* __restrict__ corr,
                  const double* __restrict__ tiles, const int32_t* __restrict__ pdofs,
                  const int32_t* __restrict__ col_start, const int32_t* __restrict__ tile_row,
                  const int32_t* __restrict__ rec_off, int j0, unsigned* __restrict__ tail_sync,
                  unsigned tail_ctas) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                          // ring_len doubles
  double* y = ring + ring_len;                // mpad
  double* part = y + a.mpad;                  // kSolveConsumers x T
  double* zblk = part + kSolveConsumers * T;  // SB8 zeros (absent sub-blocks)
  uint64_t* full = reinterpret_cast<uint64_t*>(zblk + SB8);
  uint64_t* empty = full + kRingEntries;
  int* slot_off = reinterpret_cast<int*>(empty + kRingEntries);  // ring offset of entry e's record
  const int j = j0 + blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* tb = tiles + size_t(j) * a.rec_stride;
  pdl_trigger();
  if (tid == 0) {
    for (int e = 0; e < kRingEntries; ++e) {
      mbar_init(&full[e], 1);
      mbar_init(&empty[e], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kSolveConsumers) {
    if (lane == 0) {
      int q = 0, qt = 0, head = 0;  // next position, oldest unreleased position, ring head
      // L2 policy: forward-sweep records evict_last, backward-sweep records
      // (read once more, last) evict_first, so the most recently streamed
      // forward records -- the first ones the backward sweep reads -- stay in L2
      // (measured: solve 1.284 -> 1.261 ms at C3).
      const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
      auto release_oldest = [&]() {
        mbar_wait(&empty[qt & (kRingEntries - 1)], (qt / kRingEntries) & 1);
        ++qt;
      };
      auto issue = [&](int t) {
        const int len = rec_off[t + 1] - rec_off[t];
        while (q - qt >= kRingEntries) release_oldest();
        for (;;) {  // find room at head (or at 0 after a wrap) by freeing the oldest records
          if (qt == q) {
            if (head + len > ring_len) head = 0;
            break;
          }
          const int tail = slot_off[qt & (kRingEntries - 1)];
          if (tail < head) {  // in flight: [tail, head)
            if (head + len <= ring_len) break;
            if (len <= tail) {
              head = 0;
              break;
            }
          } else if (tail > head && head + len <= tail) {  // in flight: [tail, end) + [0, head)
            break;
          }
          release_oldest();
        }
        const int e = q & (kRingEntries - 1);
        slot_off[e] = head;
        const uint32_t bytes = uint32_t(len) * sizeof(double);
        mbar_arrive_expect_tx(&full[e], bytes);
        bulk_g2s_hint(ring + head, tb + rec_off[t], bytes, &full[e],
                      q < a.ntiles ? pol_keep : pol_stream);
        head += len;
        ++q;
      };
      for (int t = 0; t < a.ntiles; ++t) issue(t);
      for (int K = a.nT - 1; K >= 0; --K) {
        const int t0 = col_start[K], t1 = col_start[K + 1];
        for (int t = t0 + 1; t < t1; ++t) issue(t);
        issue(t0);
      }
    }
    return;
  }

  constexpr int NC = 32 * kSolveConsumers;
  const int rl = lane & 7, g = lane >> 3;
  // The separator RHS comes from the kernel before.  With a split tail
  // (tail_ctas > 0) that kernel is the tail solve, which already waited for
  // the RHS producer before triggering this launch: no wait here, so both run
  // side by side; instead CTA 0 holds this grid open until the tail is done.
  if (tail_ctas == 0) pdl_wait();
  // record of stream position q, after its bytes landed
  auto acquire = [&](int q) {
    const int e = q & (kRingEntries - 1);
    mbar_wait(&full[e], (q / kRingEntries) & 1);
    return ring + slot_off[e];
  };
  auto release = [&](int q) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[q & (kRingEntries - 1)]);
  };
  // ---- phase A: gather the Schur-reduced separator RHS (the interior elimination
  // was folded into the S^T cell kernel: bhat is patch independent) ----------------
  const int32_t* pdI = pdofs + size_t(j) * a.m;
  for (int r = tid; r < a.mpad; r += NC) y[r] = (r < a.m && pdI[r] >= 0) ? rt[pdI[r]] : 0.0;
  for (int r = tid; r < SB8; r += NC) zblk[r] = 0.0;
  named_sync(1, NC);

  // ---- phase B: forward substitution over tile columns (y <- L_G^{-1} y) ----------------
  int q = 0;  // stream position, mirrors the producer
  double o0, o1;
  double xr[64];
  for (int K = 0; K < a.nT; ++K) {
    const int t0 = col_start[K], cnt = col_start[K + 1] - t0;
    double* yK = y + K * T;
    if (warp == (q & 7)) {
      load_x(yK, xr);
      const double* rec = acquire(q);
      tile_fwd(rec, zblk, rl, g, xr, o0, o1, yK);  // L_KK^{-1} y_K
      release(q);
      yK[8 * g + rl] = o0;
      yK[8 * (7 - g) + rl] = o1;
    }
    ++q;
    named_sync(1, NC);
    int i = 1 + ((warp - q) & 7);  // this warp's first tile of the column
    if (i < cnt) load_x(yK, xr);
    for (; i < cnt; i += 8) {
      const int qi = q + i - 1;
      const double* rec = acquire(qi);
      tile_fwd(rec, zblk, rl, g, xr, o0, o1, yK);
      release(qi);
      double* yI = y + tile_row[t0 + i] * T;
      yI[8 * g + rl] -= o0;
      yI[8 * (7 - g) + rl] -= o1;
    }
    q += cnt - 1;
    named_sync(1, NC);
  }

  // ---- phase C: backward substitution (x <- L_G^{-T} y), columns descending ---------------
  double acc[2][8];
  for (int K = a.nT - 1; K >= 0; --K) {
    const int t0 = col_start[K], cnt = col_start[K + 1] - t0;
    int i = 1 + ((warp - q) & 7);
    if (i < cnt) {
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[jj][k] = 0.0;
      for (; i < cnt; i += 8) {
        const int qi = q + i - 1;
        const double* yI = y + tile_row[t0 + i] * T;
        double yv[8];
#pragma unroll
        for (int bi = 0; bi < 8; ++bi) yv[bi] = yI[8 * bi + rl];
        const double* rec = acquire(qi);
        tile_bwd(rec, zblk, rl, g, yv, acc, yI);
        release(qi);
      }
      double s0, s1;
      int c;
      reduce_cols(acc, lane, s0, s1, c);
      part[warp * T + c] = s0;
      part[warp * T + c + 1] = s1;
    } else {
      part[warp * T + lane] = 0.0;
      part[warp * T + lane + 32] = 0.0;
    }
    q += cnt - 1;
    named_sync(1, NC);
    if (warp == (q & 7)) {
      double* yK = y + K * T;
      double u0 = yK[lane], u1 = yK[lane + 32];
      for (int w = 0; w < kSolveConsumers; ++w) {
        u0 -= part[w * T + lane];
        u1 -= part[w * T + lane + 32];
      }
      yK[lane] = u0;
      yK[lane + 32] = u1;
      __syncwarp();
      double yv[8];
#pragma unroll
      for (int bi = 0; bi < 8; ++bi) yv[bi] = yK[8 * bi + rl];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[jj][k] = 0.0;
      const double* rec = acquire(q);
      tile_bwd(rec, zblk, rl, g, yv, acc, y + K * T);  // x_K = L_KK^{-T} y_K (no compact blocks)
      release(q);
      double s0, s1;
      int c;
      reduce_cols(acc, lane, s0, s1, c);
      yK[c] = s0;
      yK[c + 1] = s1;
    }
    ++q;
    named_sync(1, NC);
  }

  // ---- phase D: write the separator solution x_G (interiors are rebuilt per cell)
  double* cj = corr + size_t(j) * a.out_stride + a.out_off;
  for (int r = tid; r < a.m; r += NC) cj[r] = y[r];
  if (tail_ctas > 0 && blockIdx.x == 0 && tid == 0) {
    // tail_sync[0]: finished tail CTAs (cumulative), [1]: calls completed
    const unsigned E1 = __ldcg(tail_sync + 1) + 1u;
    wait_geq(tail_sync, tail_ctas * E1);
    atomicAdd(tail_sync + 1, 1u);
  }
}

// Cluster variant: one patch per cluster of CS CTAs (SMs).  Tile row I of
// the separator factor belongs to CTA I % CS, which streams exactly the
// records of its rows (forward, then backward by column) through its own
// ring, keeps y_I, and solves the diagonal tiles of its rows.
//   forward  column K: the owner of K solves y_K = L_KK^{-1} y_K and
//            broadcasts it with st.async into every CTA's y (completing
//            fbar[K] there); each CTA then applies its tiles (I, K).
//   backward column K: each CTA sums L_IK^T x_I over its tiles into one
//            64-vector and st.asyncs it into slot `rank` of the owner's psum
//            (completing pbar[K]); the owner subtracts the CS partials in
//            rank order, solves x_K = L_KK^{-T} u and broadcasts x_K (bbar[K]).
// Every barrier is used for exactly one phase; a partial for column K is
// sent only after x_{K+1} arrived, i.e. after every owner consumed the psum
// slot's previous use.  Same arithmetic per tile as k_patch_solve; only the
// order of the backward partial sums differs (rounding level).  This spreads
// one patch's dependency chain over CS SMs: a lone patch is latency bound
// (0.38 ms at C3), so the last partial wave of single-CTA patches wastes HBM
// bandwidth that CS-way patches recover.
template <int CS>
__global__ void __launch_bounds__(kSolveThreads)
    k_patch_solve_cl(PatchArgs a, int ring_len, const double* __restrict__ rt, double* __restrict__ corr,
                     const double* __restrict__ tiles, const int32_t* __restrict__ pdofs,
                     const int32_t* __restrict__ tile_row, const int32_t* __restrict__ rec_off,
                     const int32_t* __restrict__ cl_list, const int32_t* __restrict__ cl_col, int j0,
                     unsigned* __restrict__ tail_done) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                              // ring_len doubles
  double* y = ring + ring_len;                    // mpad (owned rows; broadcast y_K / x_K)
  double* part = y + a.mpad;                      // 2 x kSolveConsumers x T
  double* psum = part + 2 * kSolveConsumers * T;  // CS x T backward partials (owner side)
  double* zblk = psum + CS * T;                   // SB8 zeros
  uint64_t* full = reinterpret_cast<uint64_t*>(zblk + SB8);
  uint64_t* empty = full + kRingEntries;
  uint64_t* fbar = empty + kRingEntries;  // nT
  uint64_t* bbar = fbar + a.nT;           // nT
  uint64_t* pbar = bbar + a.nT;           // nT
  int* slot_off = reinterpret_cast<int*>(pbar + a.nT);
  const int rank = int(cluster_ctarank());
  const int j = j0 + blockIdx.x / CS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* tb = tiles + size_t(j) * a.rec_stride;
  const int32_t* col = cl_col + rank * (a.nT + 1);
  // Wait for the predecessor before letting the single-CTA solve launch: that
  // launch then runs beside this one without waiting for it (see launch_patch_solve).
  pdl_wait();
  pdl_trigger();
  if (tid < kRingEntries) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], 1);
  }
  for (int K = tid; K < a.nT; K += blockDim.x) {
    mbar_init(&fbar[K], 1);
    mbar_init(&bbar[K], 1);
    mbar_init(&pbar[K], 1);
    mbar_arrive_expect_tx(&fbar[K], T * sizeof(double));
    mbar_arrive_expect_tx(&bbar[K], T * sizeof(double));
    if (K % CS == rank) mbar_arrive_expect_tx(&pbar[K], CS * T * sizeof(double));
  }
  mbar_fence_init();
  cluster_sync_all();

  if (warp == kSolveConsumers) {
    if (lane == 0) {
      int q = 0, qt = 0, head = 0;
      const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
      auto release_oldest = [&]() {
        mbar_wait(&empty[qt & (kRingEntries - 1)], (qt / kRingEntries) & 1);
        ++qt;
      };
      auto issue = [&](int t, uint64_t pol) {
        const int len = rec_off[t + 1] - rec_off[t];
        while (q - qt >= kRingEntries) release_oldest();
        for (;;) {
          if (qt == q) {
            if (head + len > ring_len) head = 0;
            break;
          }
          const int tail = slot_off[qt & (kRingEntries - 1)];
          if (tail < head) {
            if (head + len <= ring_len) break;
            if (len <= tail) {
              head = 0;
              break;
            }
          } else if (tail > head && head + len <= tail) {
            break;
          }
          release_oldest();
        }
        const int e = q & (kRingEntries - 1);
        slot_off[e] = head;
        const uint32_t bytes = uint32_t(len) * sizeof(double);
        mbar_arrive_expect_tx(&full[e], bytes);
        bulk_g2s_hint(ring + head, tb + rec_off[t], bytes, &full[e], pol);
        head += len;
        ++q;
      };
      for (int i = col[0]; i < col[a.nT]; ++i) issue(cl_list[i], pol_keep);
      for (int K = a.nT - 1; K >= 0; --K) {
        const int s0 = col[K], s1 = col[K + 1], own = (K % CS == rank) ? 1 : 0;
        for (int i = s0 + own; i < s1; ++i) issue(cl_list[i], pol_stream);
        if (own) issue(cl_list[s0], pol_stream);
      }
    }
  } else {
    constexpr int NC = 32 * kSolveConsumers;
    const int rl = lane & 7, g = lane >> 3;
    auto acquire = [&](int q) {
      const int e = q & (kRingEntries - 1);
      mbar_wait(&full[e], (q / kRingEntries) & 1);
      return ring + slot_off[e];
    };
    auto release = [&](int q) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[q & (kRingEntries - 1)]);
    };
    pdl_wait();
    // ---- phase A: this CTA's rows of the Schur-reduced separator RHS
    const int32_t* pdI = pdofs + size_t(j) * a.m;
    for (int r = tid; r < a.mpad; r += NC)
      if ((r / T) % CS == rank) y[r] = (r < a.m && pdI[r] >= 0) ? rt[pdI[r]] : 0.0;
    for (int r = tid; r < SB8; r += NC) zblk[r] = 0.0;
    named_sync(1, NC);

    // ---- phase B: forward substitution
    int q = 0;
    double o0, o1;
    double xr[64];
    for (int K = 0; K < a.nT; ++K) {
      const int s0 = col[K], own = (K % CS == rank) ? 1 : 0, noff = col[K + 1] - s0 - own;
      double* yK = y + K * T;
      if (own) {
        if (warp == (q & 7)) {
          load_x(yK, xr);
          const double* rec = acquire(q);
          tile_fwd(rec, zblk, rl, g, xr, o0, o1, yK);
          release(q);
#pragma unroll
          for (int d = 0; d < CS; ++d) {
            const uint32_t bar = dsmem_addr(&fbar[K], d);
            st_async_f64(dsmem_addr(yK + 8 * g + rl, d), o0, bar);
            st_async_f64(dsmem_addr(yK + 8 * (7 - g) + rl, d), o1, bar);
          }
        }
        ++q;
      }
      int i = (warp - q) & 7;
      if (i < noff) {
        mbar_wait(&fbar[K], 0);
        load_x(yK, xr);
      }
      for (; i < noff; i += 8) {
        const int qi = q + i;
        const double* rec = acquire(qi);
        tile_fwd(rec, zblk, rl, g, xr, o0, o1, yK);
        release(qi);
        double* yI = y + tile_row[cl_list[s0 + own + i]] * T;
        yI[8 * g + rl] -= o0;
        yI[8 * (7 - g) + rl] -= o1;
      }
      q += noff;
      named_sync(1, NC);
    }

    // ---- phase C: backward substitution, columns descending
    double acc[2][8];
    for (int K = a.nT - 1; K >= 0; --K) {
      const int s0 = col[K], own = (K % CS == rank) ? 1 : 0, noff = col[K + 1] - s0 - own;
      double* pw = part + ((K & 1) * kSolveConsumers + warp) * T;
      int i = (warp - q) & 7;
      if (i < noff) {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[jj][k] = 0.0;
        for (; i < noff; i += 8) {
          const int qi = q + i, I = tile_row[cl_list[s0 + own + i]];
          mbar_wait(&bbar[I], 0);
          const double* yI = y + I * T;
          double yv[8];
#pragma unroll
          for (int bi = 0; bi < 8; ++bi) yv[bi] = yI[8 * bi + rl];
          const double* rec = acquire(qi);
          tile_bwd(rec, zblk, rl, g, yv, acc, yI);
          release(qi);
        }
        double s0v, s1v;
        int c;
        reduce_cols(acc, lane, s0v, s1v, c);
        pw[c] = s0v;
        pw[c + 1] = s1v;
      } else {
        pw[lane] = 0.0;
        pw[lane + 32] = 0.0;
      }
      q += noff;
      named_sync(1, NC);
      if (warp == (q & 7)) {
        const double* pk = part + (K & 1) * kSolveConsumers * T;
        double u0 = 0.0, u1 = 0.0;
#pragma unroll
        for (int w = 0; w < kSolveConsumers; ++w) {
          u0 += pk[w * T + lane];
          u1 += pk[w * T + lane + 32];
        }
        if (K + 1 < a.nT) mbar_wait(&bbar[K + 1], 0);  // the owner's psum slot is free again
        const int dst = K % CS;
        const uint32_t pb = dsmem_addr(&pbar[K], dst);
        st_async_f64(dsmem_addr(psum + rank * T + lane, dst), u0, pb);
        st_async_f64(dsmem_addr(psum + rank * T + lane + 32, dst), u1, pb);
        if (own) {
          mbar_wait(&pbar[K], 0);
          const double* yK = y + K * T;
          double v0 = yK[lane], v1 = yK[lane + 32];
#pragma unroll
          for (int cc = 0; cc < CS; ++cc) {
            v0 -= psum[cc * T + lane];
            v1 -= psum[cc * T + lane + 32];
          }
          double yv[8];
#pragma unroll
          for (int bi = 0; bi < 8; ++bi) {
            const double t0 = __shfl_sync(0xffffffffu, v0, 8 * (bi & 3) + rl);
            const double t1 = __shfl_sync(0xffffffffu, v1, 8 * (bi & 3) + rl);
            yv[bi] = bi < 4 ? t0 : t1;
          }
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[jj][k] = 0.0;
          const double* rec = acquire(q);
          tile_bwd(rec, zblk, rl, g, yv, acc, yK);  // diagonal tile: no compact blocks
          release(q);
          double s0v, s1v;
          int c;
          reduce_cols(acc, lane, s0v, s1v, c);
#pragma unroll
          for (int d = 0; d < CS; ++d)
            st_async_f64x2(dsmem_addr(y + K * T + c, d), s0v, s1v, dsmem_addr(&bbar[K], d));
        }
      }
      q += own;
    }

    // ---- phase D: every broadcast landed; write this CTA's rows of x_G
    for (int K = tid; K < a.nT; K += NC) {
      mbar_wait(&fbar[K], 0);
      mbar_wait(&bbar[K], 0);
    }
    named_sync(1, NC);
    double* cj = corr + size_t(j) * a.out_stride + a.out_off;
    for (int r = tid; r < a.m; r += NC)
      if ((r / T) % CS == rank) cj[r] = y[r];
  }
  cluster_sync_all();  // no CTA leaves while a peer may still write into it
  if (tid == 0) {      // this CTA's rows of corr are written
    __threadfence();
    atomicAdd(tail_done, 1u);
  }
}

// z[g] = sum of patch corrections of DOF g in ascending patch order
// (src/schwarz.cpp:49-53 order, no atomics).
__global__ void k_patch_gather(int64_t ndof, const double* __restrict__ corr, const int32_t* __restrict__ ptr,
                               const int32_t* __restrict__ idx, double* __restrict__ z) {
  pdl_trigger();
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  int q0 = 0, q1 = 0, i0 = 0;  // static map, loaded before the wait
  if (g < ndof) {
    q0 = ptr[g];
    q1 = ptr[g + 1];
    if (q1 > q0) i0 = idx[q0];
  }
  pdl_wait();
  if (g >= ndof) return;
  double s = q1 > q0 ? corr[i0] : 0.0;
  for (int q = q0 + 1; q < q1; ++q) s += corr[idx[q]];
  z[g] = s;
}


// ---- Schur split of the separator solve (SchurSplit, context.hpp; schur_split.cpp) --------
// Block elimination with F = P0 | P1 (the first two facet planes) and R (the
// last plane, edges, vertex):
//   x_R = S~_RR^{-1} (b_R - S_RF S_FF^{-1} b_F),  x_F = S_FF^{-1} (b_F - S_FR x_R),
// S~_RR's Cholesky factor L_RR is the R block of the full separator factor
// (re-tiled from it after the factorisation), S_FF^{-1} is applied per
// component: with M = S_{P1,P0} of the component, D0 = diag S_{P0,P0} and
// W = chol(diag S_{P1,P1} - M D0^{-1} M^T)^{-1},
//   x1 = W^T W (b1 - M D0^{-1} b0),  x0 = D0^{-1} (b0 - M^T x1).
struct SchurArgs {
  int nF, nR, m, ncomp, c0, c1;
  int64_t vstride, comp_stride, rf_off, fr_off;
  const int32_t* comp0;
  const int32_t* comp1;
  const int32_t* comp_fr;
  const int32_t* rf_blk;
  const int32_t* fr_blk;
  const int32_t* rf_ptr;
  const int32_t* rf_col;
  const int32_t* fr_ptr;
  const int32_t* fr_col;
  const int32_t* fr_row;
  double* vals;
};

SchurArgs make_schur_args(Context& c) {
  const SchurSplit& S = c.sx;
  SchurArgs s;
  s.nF = S.nF;
  s.nR = S.nR;
  s.m = c.L.m;
  s.ncomp = S.ncomp;
  s.c0 = S.c0;
  s.c1 = S.c1;
  s.vstride = S.vstride;
  s.comp_stride = S.comp_stride;
  s.rf_off = S.rf_off;
  s.fr_off = S.fr_off;
  s.comp0 = c.sx_comp0.p;
  s.comp1 = c.sx_comp1.p;
  s.comp_fr = c.sx_comp_fr.p;
  s.rf_blk = c.sx_rf_blk.p;
  s.fr_blk = c.sx_fr_blk.p;
  s.rf_ptr = c.sx_rf_ptr.p;
  s.rf_col = c.sx_rf_col.p;
  s.fr_ptr = c.sx_fr_ptr.p;
  s.fr_col = c.sx_fr_col.p;
  s.fr_row = c.sx_fr_row.p;
  s.vals = c.sx_vals.p;
  return s;
}

// Patch-star coefficients and the 1D tables in shared memory (as k_patch_assemble).
__device__ __forceinline__ int load_patch_coeffs(const PatchArgs& a, int j, double* At, double* Bt, double* mup) {
  const int ncorner = 1 << a.dim;
  for (int i = threadIdx.x; i < a.n1 * a.n1; i += blockDim.x) {
    At[i] = a.At[i];
    Bt[i] = a.Bt[i];
  }
  int smask = 0;
  for (int s = 0; s < ncorner; ++s) smask |= (a.pcells[size_t(j) * ncorner + s] >= 0) << s;
  for (int i = threadIdx.x; i < ncorner * a.dim; i += blockDim.x) {
    const int s = i / a.dim, q = i % a.dim, K = a.pcells[size_t(j) * ncorner + s];
    mup[i] = K >= 0 ? a.mu[size_t(K) * a.dim + q] : 0.0;
  }
  return smask;
}

// S_G(r, c) of patch j as the assembly writes it (absent positions of a
// boundary star: decoupled identity rows).
__device__ __forceinline__ double sg_entry(const PatchArgs& a, const int32_t* sep, bool whole, const double* mup,
                                           int smask, int r, int c, const double* At, const double* Bt) {
  if (!whole && (sep[r] < 0 || sep[c] < 0)) return r == c ? 1.0 : 0.0;
  return schur_entry(a, mup, smask, r, c, At, Bt);
}

// S_RF and S_FR values (`pairs`: r | c << 16, S_RF's entries then S_FR's).
__global__ void k_schur_couplings(PatchArgs a, SchurArgs s, int npairs, const int32_t* __restrict__ pairs) {
  extern __shared__ double sm[];
  double* At = sm;
  double* Bt = At + a.n1 * a.n1;
  double* mup = Bt + a.n1 * a.n1;
  const int j = blockIdx.y;
  const int smask = load_patch_coeffs(a, j, At, Bt, mup);
  __syncthreads();
  const int32_t* sep = a.psep + size_t(j) * a.m;
  const bool whole = smask == (1 << (1 << a.dim)) - 1;
  double* out = s.vals + size_t(j) * s.vstride + s.rf_off;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < npairs; e += gridDim.x * blockDim.x) {
    const int32_t pv = pairs[e];
    const unsigned pc = unsigned(pv);
    out[e] = pv < 0 ? 0.0 : sg_entry(a, sep, whole, mup, smask, int(pc & 0xffffu), int(pc >> 16), At, Bt);
  }
}

// Per (component, patch): M, D0 and W = chol(S'_11)^{-1} (diag_factor_invert
// on the 64x64 identity-padded matrix).  256 threads.
__global__ void __launch_bounds__(256) k_schur_comps(PatchArgs a, SchurArgs s, int report) {
  extern __shared__ __align__(16) double sm[];
  constexpr int LD = T + 1;
  double* Dm = sm;                   // 64 x 65
  double* Wm = Dm + T * LD;          // 16 x 64 x 4 + 64
  double* MW = Wm + 16 * T * 4 + T;  // M (64 x 65), then the swizzled L^{-1}
  double* d0 = MW + T * LD;          // 64
  double* d1 = d0 + T;               // 64
  double* mup = d1 + T;              // 24
  const int k = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  // the 1D tables stay in global memory (L1-resident): two CTAs per SM at p = 31
  int smask = 0;
  const int ncorner = 1 << a.dim;
  for (int sl = 0; sl < ncorner; ++sl) smask |= (a.pcells[size_t(j) * ncorner + sl] >= 0) << sl;
  for (int i = tid; i < ncorner * a.dim; i += blockDim.x) {
    const int sl = i / a.dim, q = i % a.dim, K = a.pcells[size_t(j) * ncorner + sl];
    mup[i] = K >= 0 ? a.mu[size_t(K) * a.dim + q] : 0.0;
  }
  __syncthreads();
  const double* At = a.At;
  const double* Bt = a.Bt;
  const int32_t* sep = a.psep + size_t(j) * a.m;
  const bool whole = smask == (1 << ncorner) - 1;
  const int32_t* m0 = s.comp0 + size_t(k) * s.c0;
  const int32_t* m1 = s.comp1 + size_t(k) * s.c1;
  double* M = MW;
  for (int idx = tid; idx < s.c1 * s.c0; idx += blockDim.x) {
    const int i = idx / s.c0, jj = idx % s.c0, r = m1[i], c = m0[jj];
    M[i * LD + jj] = (r < 0 || c < 0) ? 0.0 : sg_entry(a, sep, whole, mup, smask, r, c, At, Bt);
  }
  for (int jj = tid; jj < s.c0; jj += blockDim.x) {
    const int c = m0[jj];
    d0[jj] = c < 0 ? 1.0 : sg_entry(a, sep, whole, mup, smask, c, c, At, Bt);
    if (report && !(d0[jj] > 0.0)) record_pivot_error(a.err, j, a.nI + c);
  }
  for (int i = tid; i < s.c1; i += blockDim.x) {
    const int r = m1[i];
    d1[i] = r < 0 ? 1.0 : sg_entry(a, sep, whole, mup, smask, r, r, At, Bt);
  }
  __syncthreads();
  double* out = s.vals + size_t(j) * s.vstride + size_t(k) * s.comp_stride;
  const int ldm = s.c0 | 1;
  for (int idx = tid; idx < s.c1 * ldm; idx += blockDim.x) {
    const int i = idx / ldm, jj = idx % ldm;
    out[idx] = jj < s.c0 ? M[i * LD + jj] : 0.0;
  }
  // M D0^{-1} once (in the factor's work area, free until diag_factor_invert), then
  // S'_11 = D1 - (M D0^{-1}) M^T: one division per entry of M, not per product term
  double* Ms = Wm;
  for (int idx = tid; idx < s.c1 * s.c0; idx += blockDim.x) {
    const int i = idx / s.c0, jj = idx % s.c0;
    Ms[i * LD + jj] = M[i * LD + jj] / d0[jj];
  }
  __syncthreads();
  for (int idx = tid; idx < TT; idx += blockDim.x) {
    const int cc = idx / T, r = idx % T;
    double v = r == cc ? 1.0 : 0.0;
    if (r < s.c1 && cc < s.c1) {
      v = r == cc ? d1[r] : 0.0;
      for (int jj = 0; jj < s.c0; ++jj) v -= M[r * LD + jj] * Ms[cc * LD + jj];
    }
    Dm[cc * LD + r] = v;
  }
  __syncthreads();  // M and its scaled copy are dead: their space takes the factor's work area and the inverse
  PatchArgs an = a;
  if (!report) an.err = nullptr;  // the full factorisation reports non-SPD pivots
  an.err_map = m1;
  an.diagL = nullptr;
  double* Wo = MW;
  diag_factor_invert(Dm, Wm, Wo, an, 0, j);
  __syncthreads();
  out += s.c1 * ldm;
  for (int i = tid >> 5; i < s.c1; i += blockDim.x >> 5)  // W lower triangle, row i at i(i+1)/2
    for (int q = tid & 31; q <= i; q += 32) out[i * (i + 1) / 2 + q] = Wo[tsw(i, q)];
  out += s.c1 * (s.c1 + 1) / 2;
  for (int jj = tid; jj < s.c0; jj += blockDim.x) out[jj] = d0[jj];
}

// R block of the full separator factor, re-tiled from row / column nF on:
// tile (I, J) of L_RR; diagonal tiles are inverted (the solve reads
// L_KK^{-1}), then packed as stream records of the dense R layout.
__global__ void __launch_bounds__(256) k_schur_retile(PatchArgs a, int nF, int K0, const int32_t* __restrict__ tidx,
                                                      const int32_t* __restrict__ rrow,
                                                      const int32_t* __restrict__ rcol,
                                                      const int32_t* __restrict__ bptr, const int32_t* __restrict__ blk,
                                                      const int64_t* __restrict__ ccol,
                                                      const int32_t* __restrict__ poff8,
                                                      const uint8_t* __restrict__ hdr, const double* __restrict__ tiles,
                                                      const double* __restrict__ diagL, double* __restrict__ packed,
                                                      int64_t pstride, int dense_out) {
  extern __shared__ __align__(128) double sm[];
  double* cur = sm;      // TT
  double* Lm = sm + TT;  // T x (T + 1)
  const int t = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  const int I = rrow[t], J = rcol[t];
  const bool diag = I == J;
  const double* tb = tiles + size_t(j) * a.ntiles * TT;
  const double* db = diagL + size_t(j) * a.diagNT * TT;
  for (int e = tid; e < TT; e += blockDim.x) {
    const int r = e % T, cc = e / T;
    const int R0 = nF + I * T + r, C0 = nF + J * T + cc;
    double v = 0.0;
    if (R0 >= a.m || C0 >= a.m)
      v = (diag && r == cc) ? 1.0 : 0.0;  // padding: identity
    else if (C0 <= R0) {
      const int oI = R0 / T, oJ = C0 / T;
      const int idx = tsw(R0 % T, C0 % T);
      v = oI == oJ ? db[size_t(oI - K0) * TT + idx] : tb[size_t(tidx[oI * a.nT + oJ]) * TT + idx];
    }
    if (diag)
      Lm[cc * (T + 1) + r] = v;
    else
      cur[tsw(r, cc)] = v;
  }
  __syncthreads();
  if (diag) {
    // W = L^{-1} by columns: W(k, c) = (delta_kc - sum_{c <= q < k} L(k, q) W(q, c)) / L(k, k)
    double* Wc = cur;  // column-major scratch, then swizzled
    if (tid < T) {
      const int c = tid;
      for (int kk = 0; kk < c; ++kk) Wc[c * T + kk] = 0.0;
      for (int kk = c; kk < T; ++kk) {
        double sum = kk == c ? 1.0 : 0.0;
        for (int q = c; q < kk; ++q) sum -= Lm[q * (T + 1) + kk] * Wc[c * T + q];
        Wc[c * T + kk] = sum / Lm[kk * (T + 1) + kk];
      }
    }
    __syncthreads();
    for (int e = tid; e < TT; e += blockDim.x) Lm[(e / T) * (T + 1) + e % T] = Wc[e];
    __syncthreads();
    for (int e = tid; e < TT; e += blockDim.x) {
      const int r = e % T, cc = e / T;
      cur[tsw(r, cc)] = Lm[cc * (T + 1) + r];
    }
    __syncthreads();
  }
  if (dense_out) {  // dense swizzled tile t (the inverse-top path inverts L_RR next)
    double* o = packed + size_t(j) * pstride + size_t(t) * TT;
    for (int e = tid; e < TT; e += blockDim.x) o[e] = cur[e];
    return;
  }
  write_record(cur, packed + size_t(j) * pstride + poff8[t], hdr + size_t(t) * kHdrHost, blk + bptr[t], ccol + bptr[t]);
}

// Inverse top block, step 1: U = W^T for W = L_RR^{-1}, tile (I, J) of the
// dense R layout (index col_start[J] + I - J) holding W_IJ^T:
//   W_JJ = L_JJ^{-1} (the re-tiled diagonal),  W_IJ = -W_II sum_{K=J}^{I-1} L_IK W_KJ  (I > J).
// CTA per (column J, patch), rows I in order; C^T = sum_K U(K,J) L(I,K)^T and
// U(I,J) = -C^T W_II^T run on the FP64 tensor pipe (tile_gemm_abt), operands
// by TMA bulk copy (one stage; three CTAs per SM overlap each other).
__global__ void __launch_bounds__(kUpdThreads, 3) k_schur_uinv(int nT, const int32_t* __restrict__ col_start,
                                                              const double* __restrict__ RT, double* __restrict__ UT,
                                                              int64_t stride) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  double* buf = sm + 16;  // [A, B][TT]
  const int J = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  const double* rt = RT + size_t(j) * stride;
  double* ut = UT + size_t(j) * stride;
  auto tix = [&](int I, int K) { return col_start[K] + (I - K); };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_fence_init();
  }
  {  // U(J,J) = W_JJ^T
    const double* d = rt + size_t(tix(J, J)) * TT;
    double* o = ut + size_t(tix(J, J)) * TT;
    for (int e = tid; e < TT; e += blockDim.x) {
      const int r = e % T, c = e / T;
      o[tsw(r, c)] = d[tsw(c, r)];
    }
  }
  fence_proxy_async_global();
  __syncthreads();
  unsigned phase = 0;
  for (int I = J + 1; I < nT; ++I) {
    TileAcc acc = {};
    for (int K = J; K < I; ++K) {
      if (tid == 0) {
        mbar_arrive_expect_tx(&full[0], 2 * TT * sizeof(double));
        bulk_g2s(buf, ut + size_t(tix(K, J)) * TT, TT * sizeof(double), &full[0]);
        bulk_g2s(buf + TT, rt + size_t(tix(I, K)) * TT, TT * sizeof(double), &full[0]);
      }
      mbar_wait(&full[0], phase);
      phase ^= 1;
      tile_gemm_abt(buf, buf + TT, acc);
      __syncthreads();
    }
    if (tid == 0) {
      mbar_arrive_expect_tx(&full[0], TT * sizeof(double));
      bulk_g2s(buf + TT, rt + size_t(tix(I, I)) * TT, TT * sizeof(double), &full[0]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) buf[tsw(acc.row(i), acc.col(jj, e))] = acc.v[i][jj][e];
    __syncthreads();
    mbar_wait(&full[0], phase);
    phase ^= 1;
    TileAcc u = {};
    tile_gemm_abt(buf, buf + TT, u);
    double* o = ut + size_t(tix(I, J)) * TT;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) o[tsw(u.row(i), u.col(jj, e))] = -u.v[i][jj][e];
    fence_proxy_async_global();
    __syncthreads();
  }
}

// Inverse top block, step 2: A = S~_RR^{-1} = W^T W, A_IJ = sum_{K>=I} U(K,I) U(K,J)^T
// for every lower tile (I >= J; diagonal tiles full), packed into the stream
// records of the symmetric dense layout.  CTA per (tile, patch).
__global__ void __launch_bounds__(kUpdThreads, 3) k_schur_ainv(int nT, const int32_t* __restrict__ col_start,
                                                              const int32_t* __restrict__ rrow,
                                                              const int32_t* __restrict__ rcol,
                                                              const double* __restrict__ UT, int64_t ustride,
                                                              const int32_t* __restrict__ bptr,
                                                              const int32_t* __restrict__ blk,
                                                              const int64_t* __restrict__ ccol,
                                                              const int32_t* __restrict__ poff8,
                                                              const uint8_t* __restrict__ hdr,
                                                              double* __restrict__ packed, int64_t pstride) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  double* buf = sm + 16;
  const int t = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  const int I = rrow[t], J = rcol[t];
  const double* ut = UT + size_t(j) * ustride;
  auto tix = [&](int R, int K) { return col_start[K] + (R - K); };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_fence_init();
  }
  __syncthreads();
  TileAcc acc = {};
  for (int K = I; K < nT; ++K) {
    if (tid == 0) {
      mbar_arrive_expect_tx(&full[0], 2 * TT * sizeof(double));
      bulk_g2s(buf, ut + size_t(tix(K, I)) * TT, TT * sizeof(double), &full[0]);
      bulk_g2s(buf + TT, ut + size_t(tix(K, J)) * TT, TT * sizeof(double), &full[0]);
    }
    mbar_wait(&full[0], (K - I) & 1);
    tile_gemm_abt(buf, buf + TT, acc);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
      for (int e = 0; e < 2; ++e) buf[tsw(acc.row(i), acc.col(jj, e))] = acc.v[i][jj][e];
  __syncthreads();
  write_record(buf, packed + size_t(j) * pstride + poff8[t], hdr + size_t(t) * kHdrHost, blk + bptr[t], ccol + bptr[t]);
}


// ---- Direct top block: S~_RR = S_RR - S_RF S_FF^{-1} S_FR without the full factor ----
// The full separator factor spends most of its flops on the dense |R| x |P1|
// fill block and its update of the R x R block (C5: 51 of 69 GFLOP per patch).
// S_FF^{-1} is block diagonal over the components and every R row holds only a
// few S_RF entries per component (facet rows: one P0 and one P1 mode), so
//   S~(r, c) = S(r, c) - sum_k sum_{a in row r, comp k} sum_{b in row c, comp k} S(r,a) Inv_k(a,b) S(c,b)
// costs ~4 multiply-adds per (r, c, k).  k_schur_inv forms the explicit
// component inverses, k_schur_form the correction tile by tile, k_schur_rr adds
// S_RR's own structural entries; the dense Cholesky of the R layout follows
// (k_patch_column on the dense pair lists).

// Inv_k = S_{Fk,Fk}^{-1} (nl x nl, P0 members then P1) from M, W, D0:
//   X = W^T W, Z = X M D0^{-1}:  [D0^{-1} + D0^{-1} M^T Z, -Z^T; -Z, X].
__global__ void __launch_bounds__(256) k_schur_inv(SchurArgs s, int nl, double* __restrict__ inv) {
  extern __shared__ __align__(16) double sm[];
  const int k = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  const int c0 = s.c0, c1 = s.c1, ldm = c0 | 1, ldx = c1 | 1, ldz = c0 | 1;
  double* M = sm;
  double* W = M + c1 * ldm;
  double* d0 = W + c1 * (c1 + 1) / 2;
  double* X = d0 + c0;
  double* Z = X + c1 * ldx;
  const double* src = s.vals + size_t(j) * s.vstride + size_t(k) * s.comp_stride;
  const int nin = c1 * ldm + c1 * (c1 + 1) / 2 + c0;
  for (int i = tid; i < nin; i += blockDim.x) sm[i] = src[i];
  __syncthreads();
  for (int idx = tid; idx < c1 * c1; idx += blockDim.x) {
    const int a = idx / c1, b = idx % c1;
    if (b > a) continue;
    double acc = 0.0;
    for (int q = a; q < c1; ++q) acc = fma(W[q * (q + 1) / 2 + a], W[q * (q + 1) / 2 + b], acc);
    X[a * ldx + b] = acc;
    X[b * ldx + a] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < c1 * c0; idx += blockDim.x) {
    const int a = idx / c0, jj = idx % c0;
    double acc = 0.0;
    for (int i = 0; i < c1; ++i) acc = fma(X[a * ldx + i], M[i * ldm + jj], acc);
    Z[a * ldz + jj] = acc / d0[jj];
  }
  __syncthreads();
  double* out = inv + (size_t(j) * s.ncomp + k) * nl * nl;
  for (int idx = tid; idx < c1 * c1; idx += blockDim.x) {
    const int a = idx / c1, b = idx % c1;
    out[size_t(c0 + a) * nl + c0 + b] = X[a * ldx + b];
  }
  for (int idx = tid; idx < c1 * c0; idx += blockDim.x) {
    const int a = idx / c0, jj = idx % c0;
    const double v = -Z[a * ldz + jj];
    out[size_t(c0 + a) * nl + jj] = v;
    out[size_t(jj) * nl + c0 + a] = v;
  }
  for (int idx = tid; idx < c0 * c0; idx += blockDim.x) {
    const int jj = idx / c0, j2 = idx % c0;
    if (j2 > jj) continue;
    double acc = 0.0;
    for (int i = 0; i < c1; ++i) acc = fma(M[i * ldm + jj], Z[i * ldz + j2], acc);
    const double v = (jj == j2 ? 1.0 : 0.0) / d0[jj] + acc / d0[jj];
    out[size_t(jj) * nl + j2] = v;
    out[size_t(j2) * nl + jj] = v;
  }
}

// S_RF values in (component, row) entry order: fv[patch][e] = S_RF value of rk_ent[e].
__global__ void k_schur_fv(SchurArgs s, int nent, const int32_t* __restrict__ rk_ent, double* __restrict__ fv) {
  const int j = blockIdx.y;
  const double* v = s.vals + size_t(j) * s.vstride + s.rf_off;
  double* o = fv + size_t(j) * nent;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nent; e += gridDim.x * blockDim.x) o[e] = v[rk_ent[e] >> 8];
}

// The first two S_RF values of every (component, row): fv2[patch][k][r] = (v0, v1), zero where absent
// (and on the padding rows); the local indices are in SchurSplit::e2.
__global__ void k_schur_fv2(SchurArgs s, int nRp, const int32_t* __restrict__ kr, const int32_t* __restrict__ rk_ent,
                            double* __restrict__ fv2) {
  const int j = blockIdx.y;
  const double* v = s.vals + size_t(j) * s.vstride + s.rf_off;
  const int n = s.ncomp * nRp;
  double2* o = reinterpret_cast<double2*>(fv2) + size_t(j) * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int pk = kr[i], e0 = pk >> 8, cnt = pk & 255;
    double2 w;
    w.x = cnt > 0 ? v[rk_ent[e0] >> 8] : 0.0;
    w.y = cnt > 1 ? v[rk_ent[e0 + 1] >> 8] : 0.0;
    o[i] = w;
  }
}

// -(S_RF S_FF^{-1} S_FR) on row tile I and up to G column tiles J0.. of one patch
// (512 threads).  Per component k, phase A: Y[rr][lb] = sum_a S(r, a) Inv_k(a, lb)
// for the tile's 64 rows (warp per row, lanes along lb); phase B: thread
// (column cl, 8 rows) adds Y[rr][lb] S(c, b) over column c's entries of
// component k.  Everything phase A and B read arrives in shared memory by TMA
// bulk copies issued ahead: Inv_k (nl x nl, single buffer: fetched while phase
// B of the previous component runs -- with Inv_k read from global memory every
// warp sat in the same L2 round trips at the same time, ncu: 36 % of stall
// samples at the barrier, 23 % on those loads) and the direct-indexed tables
// e2 / fv2 of the first two entries of every (component, row) (the tile's 64
// rows for phase A, the CTA's nG x 64 columns for phase B, double buffered).
// Rows with more entries (edge modes) continue through kr / rk_ent / fv.
// Sums run in entry order.
constexpr int kFormThreads = 512;
template <int G>
__global__ void __launch_bounds__(kFormThreads, 1)
    k_schur_form(int nR, int nRp, int ncomp, int nl, const int32_t* __restrict__ form_I,
                 const int32_t* __restrict__ form_J0, const int32_t* __restrict__ kr,
                 const int32_t* __restrict__ rk_ent, int nent, const double* __restrict__ fv,
                 const int32_t* __restrict__ e2, const double* __restrict__ fv2, const double* __restrict__ inv,
                 const int32_t* __restrict__ col_start, double* __restrict__ RT, int64_t rstride) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2], barA[2], barI;
  __shared__ __align__(16) double2 rowV[2 * T];  // phase A's table rows (the tile's 64 rows), two components in flight
  __shared__ __align__(16) int32_t rowE[2 * T];
  const int pitch = nl | 1;
  double* Ism = sm;                                              // Inv_k, nl x nl
  double2* tabV = reinterpret_cast<double2*>(Ism + nl * nl);     // [2][G T] first two values
  int32_t* tabE = reinterpret_cast<int32_t*>(tabV + 2 * G * T);  // [2][G T] their local indices | flags
  double* Y = reinterpret_cast<double*>(tabE + 2 * G * T);       // [T][pitch]
  const int f = blockIdx.x, j = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int I = form_I[f], J0 = form_J0[f];
  const int nG = min(G, I - J0 + 1);
  const double* fvj = fv + size_t(j) * nent;
  const double2* f2j = reinterpret_cast<const double2*>(fv2) + size_t(j) * ncomp * nRp;
  const double* invj = inv + size_t(j) * ncomp * nl * nl;
  const int cl = tid & 63, rg = tid >> 6;
  double acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[g][i] = 0.0;
  const uint32_t nb = uint32_t(nG) * T, ibytes = uint32_t(nl) * nl * 8u;
  auto fetchB = [&](int k) {
    const int b = k & 1;
    mbar_arrive_expect_tx(&bar[b], nb * 20u);
    bulk_g2s(tabV + b * G * T, f2j + size_t(k) * nRp + J0 * T, nb * 16u, &bar[b]);
    bulk_g2s(tabE + b * G * T, e2 + size_t(k) * nRp + J0 * T, nb * 4u, &bar[b]);
  };
  auto fetchA = [&](int k) {
    const int b = k & 1;
    mbar_arrive_expect_tx(&barA[b], uint32_t(T) * 20u);
    bulk_g2s(rowV + b * T, f2j + size_t(k) * nRp + I * T, uint32_t(T) * 16u, &barA[b]);
    bulk_g2s(rowE + b * T, e2 + size_t(k) * nRp + I * T, uint32_t(T) * 4u, &barA[b]);
  };
  auto fetchI = [&](int k) {
    mbar_arrive_expect_tx(&barI, ibytes);
    bulk_g2s(Ism, invj + size_t(k) * nl * nl, ibytes, &barI);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&barA[0], 1);
    mbar_init(&barA[1], 1);
    mbar_init(&barI, 1);
    mbar_fence_init();
    fetchI(0);
    fetchA(0);
    if (ncomp > 1) fetchA(1);
    fetchB(0);
  }
  __syncthreads();  // the barriers are initialised before anyone waits on them
#pragma unroll 1
  for (int k = 0; k < ncomp; ++k) {
    // ---- phase A: Y = S_RF(rows of tile I, component k) Inv_k
    mbar_wait(&barA[k & 1], (k >> 1) & 1);
    mbar_wait(&barI, k & 1);
    {
      const int32_t* pk = rowE + (k & 1) * T;
      const double2* v = rowV + (k & 1) * T;
#pragma unroll
      for (int ii = 0; ii < T / 16; ++ii) {
        const int rr = warp + 16 * ii;
        const int pr = pk[rr];
        const double2 vr = v[rr];
        const double* row0 = Ism + (pr & 255) * nl;
        const double* row1 = Ism + ((pr >> 8) & 255) * nl;
        double y[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int lb = lane + 32 * q;
          y[q] = lb < nl ? fma(vr.y, row1[lb], vr.x * row0[lb]) : 0.0;
        }
        if (pr >> 18) {  // more than two entries
          const int kk = kr[size_t(k) * nRp + I * T + rr];
          const int e0 = kk >> 8, cnt = kk & 255;
          for (int e = e0 + 2; e < e0 + cnt; ++e) {
            const double va = fvj[e];
            const double* row = Ism + (rk_ent[e] & 255) * nl;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int lb = lane + 32 * q;
              if (lb < nl) y[q] = fma(va, row[lb], y[q]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int lb = lane + 32 * q;
          if (lb < nl) Y[rr * pitch + lb] = y[q];
        }
      }
    }
    __syncthreads();
    // Inv_{k+1} streams in under phase B; the table buffers refilled here were last read before this barrier
    if (tid == 0) {
      if (k + 1 < ncomp) {
        fetchI(k + 1);
        fetchB(k + 1);
      }
      if (k + 2 < ncomp) fetchA(k + 2);
    }
    // ---- phase B: acc(rows, column cl of tile J0 + g) += Y(rows, lb) S(c, b)
    mbar_wait(&bar[k & 1], (k >> 1) & 1);
    const int32_t* pk = tabE + (k & 1) * G * T + cl;
    const double2* v = tabV + (k & 1) * G * T + cl;
    const double* yr = Y + rg * 8 * pitch;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (g < nG) {
        const int pg = pk[g * T];
        const double2 vg = v[g * T];
        const double* y0 = yr + (pg & 255);
        const double* y1 = yr + ((pg >> 8) & 255);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[g][i] = fma(y0[i * pitch], vg.x, acc[g][i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[g][i] = fma(y1[i * pitch], vg.y, acc[g][i]);
        if (pg >> 18) {
          const int kk = kr[size_t(k) * nRp + (J0 + g) * T + cl];
          const int e0 = kk >> 8, cnt = kk & 255;
          for (int e = e0 + 2; e < e0 + cnt; ++e) {
            const int lb = rk_ent[e] & 255;
            const double vb = fvj[e];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[g][i] = fma(yr[i * pitch + lb], vb, acc[g][i]);
          }
        }
      }
    }
    __syncthreads();  // Y is free for the next component
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (g < nG) {
      const int J = J0 + g;
      double* o = RT + size_t(j) * rstride + size_t(col_start[J] + I - J) * TT;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[tsw(rg * 8 + i, cl)] = -acc[g][i];
    }
  }
}

// k_schur_form on half row tiles (32 rows x up to G column tiles per CTA, thread = column x 4
// rows): phase A of a CTA halves (the rows' products with Inv_k are recomputed by every CTA of the
// row tile), and Y is double buffered, so a warp goes from phase B of component k straight to
// phase A of k + 1 -- one barrier per component, the two phases of different warps overlap.
// Inv_{k+2} is fetched after that barrier and lands under phase B of k + 1.  Same sums, same order.
template <int G>
__global__ void __launch_bounds__(kFormThreads, 1)
    k_schur_form2(int nR, int nRp, int ncomp, int nl, const int32_t* __restrict__ form_Ih,
                  const int32_t* __restrict__ form_J0, const int32_t* __restrict__ kr,
                  const int32_t* __restrict__ rk_ent, int nent, const double* __restrict__ fv,
                  const int32_t* __restrict__ e2, const double* __restrict__ fv2, const double* __restrict__ inv,
                  const int32_t* __restrict__ col_start, double* __restrict__ RT, int64_t rstride) {
  constexpr int HR = T / 2;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2], barA[2], barI;
  __shared__ __align__(16) double2 rowV[2 * HR];
  __shared__ __align__(16) int32_t rowE[2 * HR];
  const int pitch = nl | 1;
  double* Ism = sm;                                              // Inv_k, nl x nl
  double2* tabV = reinterpret_cast<double2*>(Ism + nl * nl);     // [2][G T]
  int32_t* tabE = reinterpret_cast<int32_t*>(tabV + 2 * G * T);  // [2][G T]
  double* Y0 = reinterpret_cast<double*>(tabE + 2 * G * T);      // [2][HR][pitch]
  const int f = blockIdx.x, j = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Ih = form_Ih[f], I = Ih >> 1, r0 = (Ih & 1) * HR, J0 = form_J0[f];
  const int nG = min(G, I - J0 + 1);
  const double* fvj = fv + size_t(j) * nent;
  const double2* f2j = reinterpret_cast<const double2*>(fv2) + size_t(j) * ncomp * nRp;
  const double* invj = inv + size_t(j) * ncomp * nl * nl;
  const int cl = tid & 63, rg = tid >> 6;
  double acc[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[g][i] = 0.0;
  const uint32_t nb = uint32_t(nG) * T, ibytes = uint32_t(nl) * nl * 8u;
  auto fetchB = [&](int k) {
    const int b = k & 1;
    mbar_arrive_expect_tx(&bar[b], nb * 20u);
    bulk_g2s(tabV + b * G * T, f2j + size_t(k) * nRp + J0 * T, nb * 16u, &bar[b]);
    bulk_g2s(tabE + b * G * T, e2 + size_t(k) * nRp + J0 * T, nb * 4u, &bar[b]);
  };
  auto fetchA = [&](int k) {
    const int b = k & 1;
    mbar_arrive_expect_tx(&barA[b], uint32_t(HR) * 20u);
    bulk_g2s(rowV + b * HR, f2j + size_t(k) * nRp + I * T + r0, uint32_t(HR) * 16u, &barA[b]);
    bulk_g2s(rowE + b * HR, e2 + size_t(k) * nRp + I * T + r0, uint32_t(HR) * 4u, &barA[b]);
  };
  auto fetchI = [&](int k) {
    mbar_arrive_expect_tx(&barI, ibytes);
    bulk_g2s(Ism, invj + size_t(k) * nl * nl, ibytes, &barI);
  };
  auto phaseA = [&](int k) {
    double* Y = Y0 + (k & 1) * HR * pitch;
    mbar_wait(&barA[k & 1], (k >> 1) & 1);
    mbar_wait(&barI, k & 1);
    const int32_t* pk = rowE + (k & 1) * HR;
    const double2* v = rowV + (k & 1) * HR;
#pragma unroll
    for (int ii = 0; ii < HR / 16; ++ii) {
      const int rr = warp + 16 * ii;
      const int pr = pk[rr];
      const double2 vr = v[rr];
      const double* row0 = Ism + (pr & 255) * nl;
      const double* row1 = Ism + ((pr >> 8) & 255) * nl;
      double y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int lb = lane + 32 * q;
        y[q] = lb < nl ? fma(vr.y, row1[lb], vr.x * row0[lb]) : 0.0;
      }
      if (pr >> 18) {  // more than two entries
        const int kk = kr[size_t(k) * nRp + I * T + r0 + rr];
        const int e0 = kk >> 8, cnt = kk & 255;
        for (int e = e0 + 2; e < e0 + cnt; ++e) {
          const double va = fvj[e];
          const double* row = Ism + (rk_ent[e] & 255) * nl;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int lb = lane + 32 * q;
            if (lb < nl) y[q] = fma(va, row[lb], y[q]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int lb = lane + 32 * q;
        if (lb < nl) Y[rr * pitch + lb] = y[q];
      }
    }
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&barA[0], 1);
    mbar_init(&barA[1], 1);
    mbar_init(&barI, 1);
    mbar_fence_init();
    fetchI(0);
    fetchA(0);
    if (ncomp > 1) fetchA(1);
    fetchB(0);
    if (ncomp > 1) fetchB(1);
  }
  __syncthreads();  // the barriers are initialised before anyone waits on them
  phaseA(0);
  __syncthreads();
  if (tid == 0) {
    if (ncomp > 1) fetchI(1);
    if (ncomp > 2) fetchA(2);
  }
#pragma unroll 1
  for (int k = 0; k < ncomp; ++k) {
    // ---- phase B(k)
    mbar_wait(&bar[k & 1], (k >> 1) & 1);
    {
      const int32_t* pk = tabE + (k & 1) * G * T + cl;
      const double2* v = tabV + (k & 1) * G * T + cl;
      const double* yr = Y0 + (k & 1) * HR * pitch + rg * 4 * pitch;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (g < nG) {
          const int pg = pk[g * T];
          const double2 vg = v[g * T];
          const double* y0 = yr + (pg & 255);
          const double* y1 = yr + ((pg >> 8) & 255);
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[g][i] = fma(y0[i * pitch], vg.x, acc[g][i]);
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[g][i] = fma(y1[i * pitch], vg.y, acc[g][i]);
          if (pg >> 18) {
            const int kk = kr[size_t(k) * nRp + (J0 + g) * T + cl];
            const int e0 = kk >> 8, cnt = kk & 255;
            for (int e = e0 + 2; e < e0 + cnt; ++e) {
              const int lb = rk_ent[e] & 255;
              const double vb = fvj[e];
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[g][i] = fma(yr[i * pitch + lb], vb, acc[g][i]);
            }
          }
        }
      }
    }
    // ---- phase A(k + 1) into the other Y buffer
    if (k + 1 < ncomp) phaseA(k + 1);
    __syncthreads();
    // Inv's buffer, table buffer k & 1 and row-table buffer (k + 1) & 1 were last read before this barrier
    if (tid == 0) {
      if (k + 2 < ncomp) {
        fetchI(k + 2);
        fetchB(k + 2);
      }
      if (k + 3 < ncomp) fetchA(k + 3);
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (g < nG) {
      const int J = J0 + g;
      double* o = RT + size_t(j) * rstride + size_t(col_start[J] + I - J) * TT;
#pragma unroll
      for (int i = 0; i < 4; ++i) o[tsw(r0 + rg * 4 + i, cl)] = -acc[g][i];
    }
  }
}

// += S_RR's own structural entries (and the identity on the padding rows).
__global__ void k_schur_rr(PatchArgs a, int nF, int nentries, const int32_t* __restrict__ entries,
                           const int32_t* __restrict__ rrow, const int32_t* __restrict__ rcol,
                           double* __restrict__ RT, int64_t rstride) {
  extern __shared__ double sm[];
  double* At = sm;
  double* Bt = At + a.n1 * a.n1;
  double* mup = Bt + a.n1 * a.n1;
  const int j = blockIdx.y;
  const int smask = load_patch_coeffs(a, j, At, Bt, mup);
  __syncthreads();
  const int32_t* sep = a.psep + size_t(j) * a.m;
  const bool whole = smask == (1 << (1 << a.dim)) - 1;
  double* base = RT + size_t(j) * rstride;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nentries; e += gridDim.x * blockDim.x) {
    const int code = entries[e];
    const int t = code >> 12, cc = (code >> 6) & 63, rr = code & 63;
    const int r = nF + rrow[t] * T + rr, c = nF + rcol[t] * T + cc;
    double v;
    if (r >= a.m || c >= a.m)
      v = r == c ? 1.0 : 0.0;
    else
      v = sg_entry(a, sep, whole, mup, smask, r, c, At, Bt);
    base[size_t(t) * TT + tsw(rr, cc)] += v;
  }
}

// Inverse top block, solve: x_R = A t_R with A symmetric, each lower tile
// streamed once: x_I += A_IJ t_J and, off the diagonal, x_J += A_IJ^T t_I.
// No dependency chain, so each patch's tile stream is split into `nchunk`
// contiguous chunks, one CTA each (grid: patch-major).  Warp roles:
//   producer (1 warp): streams the chunk's records through the byte ring (as k_patch_solve);
//   consumers (NCONS warps): stream position q goes to warp q mod NCONS: tile_fwd (row part)
//     and tile_bwd + reduce_cols (column part) on the record, the two 64-vectors
//     into stage slot q mod kSymvSlots, the record released at once;
//   committer (1 warp): adds the stage slots to the CTA accumulator in stream
//     order (deterministic sums, no CTA-wide barrier per tile).
// Slots and ring entries hand over through mbarriers.  The accumulator goes
// to partial[patch][chunk] (summed in chunk order by k_schur_xsum).
constexpr int kSymvSlots = 16;
template <int NCONS>
__global__ void __launch_bounds__(32 * (NCONS + 2))
    k_schur_symv(PatchArgs a, int ring_len, int nchunk, const int32_t* __restrict__ chunk_start,
                 const double* __restrict__ tR, const double* __restrict__ recs, const int32_t* __restrict__ tile_row,
                 const int32_t* __restrict__ tile_col, const int32_t* __restrict__ rec_off,
                 double* __restrict__ partial) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                       // ring_len doubles
  double* tv = ring + ring_len;            // mpad: t_R
  double* xa = tv + a.mpad;                // mpad: accumulator
  double* stage = xa + a.mpad;             // kSymvSlots x 2T
  double* zblk = stage + kSymvSlots * 2 * T;  // SB8 zeros
  uint64_t* full = reinterpret_cast<uint64_t*>(zblk + SB8);
  uint64_t* empty = full + kRingEntries;
  uint64_t* sfull = empty + kRingEntries;
  uint64_t* sempty = sfull + kSymvSlots;
  int* slot_off = reinterpret_cast<int*>(sempty + kSymvSlots);
  const int j = blockIdx.x / nchunk, ch = blockIdx.x % nchunk;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t0 = chunk_start[ch], nt = chunk_start[ch + 1] - t0;
  const double* tb = recs + size_t(j) * a.rec_stride;
  constexpr int kProducer = NCONS, kCommitter = NCONS + 1;
  constexpr int NW = 32 * (NCONS + 1);  // consumers + committer
  pdl_trigger();
  if (tid == 0) {
    for (int e = 0; e < kRingEntries; ++e) {
      mbar_init(&full[e], 1);
      mbar_init(&empty[e], 1);
    }
    for (int e = 0; e < kSymvSlots; ++e) {
      mbar_init(&sfull[e], 1);
      mbar_init(&sempty[e], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kProducer) {
    if (lane == 0) {
      int q = 0, qt = 0, head = 0;
      const uint64_t pol = policy_evict_first();  // every record is read once per sweep
      auto release_oldest = [&]() {
        mbar_wait(&empty[qt & (kRingEntries - 1)], (qt / kRingEntries) & 1);
        ++qt;
      };
      for (int i = 0; i < nt; ++i) {
        const int t = t0 + i;
        const int len = rec_off[t + 1] - rec_off[t];
        while (q - qt >= kRingEntries) release_oldest();
        for (;;) {
          if (qt == q) {
            if (head + len > ring_len) head = 0;
            break;
          }
          const int tail = slot_off[qt & (kRingEntries - 1)];
          if (tail < head) {
            if (head + len <= ring_len) break;
            if (len <= tail) {
              head = 0;
              break;
            }
          } else if (tail > head && head + len <= tail) {
            break;
          }
          release_oldest();
        }
        const int e = q & (kRingEntries - 1);
        slot_off[e] = head;
        const uint32_t bytes = uint32_t(len) * sizeof(double);
        mbar_arrive_expect_tx(&full[e], bytes);
        bulk_g2s_hint(ring + head, tb + rec_off[t], bytes, &full[e], pol);
        head += len;
        ++q;
      }
    }
    return;
  }
  pdl_wait();
  const int ct = warp == kCommitter ? tid - 32 : tid;  // 0 .. NW-1 over consumers + committer
  for (int r = ct; r < a.mpad; r += NW) {
    tv[r] = r < a.m ? tR[size_t(j) * a.m + r] : 0.0;
    xa[r] = 0.0;
  }
  for (int r = ct; r < SB8; r += NW) zblk[r] = 0.0;
  named_sync(1, NW);
  if (warp == kCommitter) {
    for (int q = 0; q < nt; ++q) {
      const int sl = q & (kSymvSlots - 1);
      const int t = t0 + q, I = tile_row[t], J = tile_col[t];
      mbar_wait(&sfull[sl], (q / kSymvSlots) & 1);
      const double* st = stage + sl * 2 * T;
      const double r0 = st[lane], r1 = st[lane + 32];
      double c0 = 0.0, c1 = 0.0;
      if (I != J) {
        c0 = st[T + lane];
        c1 = st[T + lane + 32];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[sl]);
      xa[I * T + lane] += r0;
      xa[I * T + lane + 32] += r1;
      if (I != J) {
        xa[J * T + lane] += c0;
        xa[J * T + lane + 32] += c1;
      }
      __syncwarp();
    }
  } else {
    const int rl = lane & 7, g = lane >> 3;
    double xr[64];
    for (int q = warp; q < nt; q += NCONS) {
      const int t = t0 + q, I = tile_row[t], J = tile_col[t];
      const int e = q & (kRingEntries - 1), sl = q & (kSymvSlots - 1);
      load_x(tv + J * T, xr);
      double yv[8];
#pragma unroll
      for (int bi = 0; bi < 8; ++bi) yv[bi] = tv[I * T + 8 * bi + rl];
      mbar_wait(&full[e], (q / kRingEntries) & 1);
      const double* rec = ring + slot_off[e];
      double o0, o1;
      tile_fwd(rec, zblk, rl, g, xr, o0, o1, nullptr);
      double s0 = 0.0, s1 = 0.0;
      int c = 0;
      if (I != J) {
        double acc[2][8];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[jj][k] = 0.0;
        tile_bwd(rec, zblk, rl, g, yv, acc, nullptr);
        reduce_cols(acc, lane, s0, s1, c);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[e]);
      mbar_wait(&sempty[sl], ((q / kSymvSlots) & 1) ^ 1);
      double* st = stage + sl * 2 * T;
      st[8 * g + rl] = o0;
      st[8 * (7 - g) + rl] = o1;
      if (I != J) {
        st[T + c] = s0;
        st[T + c + 1] = s1;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[sl]);
    }
  }
  named_sync(1, NW);
  double* pj = partial + (size_t(j) * nchunk + ch) * a.mpad;
  for (int r = ct; r < a.mpad; r += NW) pj[r] = xa[r];
}

// x_R = sum of the chunk partials in chunk order -> corr[patch][nF + r].
__global__ void k_schur_xsum(int nR, int mpadR, int nchunk, int m, int nF, const double* __restrict__ partial,
                             double* __restrict__ corr) {
  const int j = blockIdx.y;
  pdl_trigger();
  pdl_wait();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nR; r += gridDim.x * blockDim.x) {
    const double* p = partial + size_t(j) * nchunk * mpadR + r;
    double s = p[0];
    for (int c = 1; c < nchunk; ++c) s += p[size_t(c) * mpadR];
    corr[size_t(j) * m + nF + r] = s;
  }
}

// S_FF^{-1} of one component (128 threads): the component's value block --
// M (c1 x c0, row stride c0|1), W = chol(S'_11)^{-1} (c1 x c1 lower triangle,
// packed by rows), D0 (c0) -- arrives in shared memory by one TMA bulk copy
// issued at entry; b from the S^T output (mode 0, forward half) or from
// c_F = b_F - S_FR x_R (mode 1, backward half).  Every product runs two
// threads per output (row or column halves, combined by one shuffle); M's odd
// row stride makes both its row-wise and column-wise reads conflict free.
// Output: mode 0 -> Fw (npatch x nF), mode 1 -> corr (F part of the separator solution).
constexpr int kCompThreads = 128;
// STAGED: the block is bulk-copied into shared memory (44 KB at p = 31: 5 CTAs per
// SM); otherwise the products read it straight from global memory through L1
// (2.5 KB of shared memory: up to 16 CTAs per SM).
template <bool STAGED>
__global__ void __launch_bounds__(kCompThreads) k_schur_comp(PatchArgs a, SchurArgs s, const double* __restrict__ rt,
                                                             const double* __restrict__ cF, double* __restrict__ out,
                                                             int mode) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double b0[64], b1[64], t0[64], t1[64];
  const int k = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  const int c0 = s.c0, c1 = s.c1, ldm = c0 | 1;
  const double* src = s.vals + size_t(j) * s.vstride + size_t(k) * s.comp_stride;
  if (STAGED) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      mbar_fence_init();
      const uint32_t bytes = uint32_t(s.comp_stride * sizeof(double));
      mbar_arrive_expect_tx(&bar, bytes);
      bulk_g2s(sm, src, bytes, &bar);  // values do not depend on the predecessor
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
  }
  const int32_t* m0 = s.comp0 + size_t(k) * c0;
  const int32_t* m1 = s.comp1 + size_t(k) * c1;
  const int32_t* sep = a.psep + size_t(j) * a.m;
  int p0 = -1, p1 = -1, g0 = -1, g1 = -1;
  if (tid < c0) {
    p0 = m0[tid];
    g0 = p0 >= 0 ? (mode == 0 ? sep[p0] : p0) : -1;
  }
  if (tid < c1) {
    p1 = m1[tid];
    g1 = p1 >= 0 ? (mode == 0 ? sep[p1] : p1) : -1;
  }
  pdl_trigger();
  pdl_wait();
  const double* bsrc = mode == 0 ? rt : cF + size_t(j) * s.nF;
  if (tid < 64) {
    b0[tid] = g0 >= 0 ? bsrc[g0] : 0.0;
    b1[tid] = g1 >= 0 ? bsrc[g1] : 0.0;
  }
  if (STAGED) mbar_wait(&bar, 0);
  const double* M = STAGED ? sm : src;
  const double* W = M + c1 * ldm;  // lower triangle packed by rows: W(i, q) at i(i+1)/2 + q
  const double* d0 = W + c1 * (c1 + 1) / 2;
  __syncthreads();
  if (tid < c0) t0[tid] = b0[tid] / d0[tid];  // u0 = D0^{-1} b0
  __syncthreads();
  // thread pair (2 o, 2 o + 1) computes output o; h = half
  const int o = tid >> 1, h = tid & 1;
  {  // r1 = b1 - M u0 (rows)
    double acc = 0.0;
    if (o < c1) {
      const double* row = M + o * ldm;
      for (int q = h; q < c0; q += 2) acc = fma(row[q], t0[q], acc);
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (o < c1 && h == 0) t1[o] = b1[o] - acc;
  }
  __syncthreads();
  {  // y = W r1 (rows, lower)
    double acc = 0.0;
    if (o < c1) {
      const double* row = W + o * (o + 1) / 2;
      for (int q = h; q <= o; q += 2) acc = fma(row[q], t1[q], acc);
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (o < c1 && h == 0) b1[o] = acc;
  }
  __syncthreads();
  {  // x1 = W^T y (columns)
    double acc = 0.0;
    if (o < c1)
      for (int q = o + h; q < c1; q += 2) acc = fma(W[q * (q + 1) / 2 + o], b1[q], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (o < c1 && h == 0) t1[o] = acc;
  }
  __syncthreads();
  {  // x0 = D0^{-1} (b0 - M^T x1) (columns)
    double acc = 0.0;
    if (o < c0)
      for (int i = h; i < c1; i += 2) acc = fma(M[i * ldm + o], t1[i], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (o < c0 && h == 0) t0[o] = (b0[o] - acc) / d0[o];
  }
  __syncthreads();
  double* op = out + size_t(j) * (mode == 0 ? s.nF : s.m);
  if (p0 >= 0) op[p0] = t0[tid];
  if (p1 >= 0) op[p1] = t1[tid];
}

// Unfilled couplings, one CTA per block of kSpmvRows rows of one patch:
//   mode 0: t_R = b_R - S_RF w   (rows R, x = Fw, out = tR)
//   mode 1: c_F = b_F - S_FR x_R (rows F in component order, x = x_R in corr, out = cF)
// The block's values and column indices (contiguous, 16-byte aligned) arrive
// in shared memory by two TMA bulk copies issued at entry; 8 threads per row.
constexpr int kSpmvThreads = 8 * kSpmvRows;  // TPR = 8 (16 threads per row: 2 x kSpmvThreads)
// STAGED: the block's values / columns bulk-copied into shared memory; otherwise
// read straight from global memory (coalesced: a row's entries are contiguous).
template <bool STAGED, int TPR>
__global__ void __launch_bounds__(TPR * kSpmvRows) k_schur_spmv(PatchArgs a, SchurArgs s, const double* __restrict__ rt,
                                                             const double* __restrict__ xin, double* __restrict__ out,
                                                             int mode) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  const int b = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  const int32_t* blk = mode == 0 ? s.rf_blk : s.fr_blk;
  const int32_t* ptr = mode == 0 ? s.rf_ptr : s.fr_ptr;
  const int32_t* col = mode == 0 ? s.rf_col : s.fr_col;
  const double* v = s.vals + size_t(j) * s.vstride + (mode == 0 ? s.rf_off : s.fr_off);
  const int e0 = blk[b], ne = blk[b + 1] - e0;
  const double* vs = STAGED ? sm : v + e0;
  const int32_t* cs = STAGED ? reinterpret_cast<const int32_t*>(sm + ne) : col + e0;
  if (STAGED) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      mbar_fence_init();
      if (ne > 0) {
        mbar_arrive_expect_tx(&bar, uint32_t(ne) * 12u);
        bulk_g2s(sm, v + e0, uint32_t(ne) * 8u, &bar);
        bulk_g2s(sm + ne, col + e0, uint32_t(ne) * 4u, &bar);
      } else {
        mbar_arrive(&bar);
      }
    }
    __syncthreads();
  }
  const int nrows = mode == 0 ? s.nR : s.nF;
  const int rl = tid / TPR, sub = tid % TPR, r = b * kSpmvRows + rl;
  const bool live = r < nrows;
  int r0 = 0, r1 = 0, pos = -1, g = -1;
  if (live) {
    r0 = ptr[r] - e0;
    r1 = ptr[r + 1] - e0;
    pos = mode == 0 ? s.nF + r : s.fr_row[r];
    g = a.psep[size_t(j) * a.m + pos];
  }
  const double* x = mode == 0 ? xin + size_t(j) * s.nF : xin + size_t(j) * s.m + s.nF;
  pdl_trigger();
  pdl_wait();
  const double bv = (sub == 0 && g >= 0) ? rt[g] : 0.0;
  if (STAGED) mbar_wait(&bar, 0);
  // four independent gathers in flight per thread (the x reads are L1/L2 latency)
  double a4[4] = {0.0, 0.0, 0.0, 0.0};
  int e = r0 + sub;
  for (; e + 3 * TPR < r1; e += 4 * TPR) {
    double xv[4], vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      vv[u] = vs[e + TPR * u];
      xv[u] = x[cs[e + TPR * u]];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) a4[u] = fma(vv[u], xv[u], a4[u]);
  }
  if (TPR == 16) {  // the tail's gathers in flight together as well (a row is ~ 7 entries per thread)
    double xv[3], vv[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const bool in = e + TPR * u < r1;
      vv[u] = in ? vs[e + TPR * u] : 0.0;
      xv[u] = in ? x[cs[e + TPR * u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 3; ++u) a4[u] = fma(vv[u], xv[u], a4[u]);
  } else {
    for (; e < r1; e += TPR) a4[0] = fma(vs[e], x[cs[e]], a4[0]);
  }
  double acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  if (TPR == 16) acc += __shfl_xor_sync(0xffffffffu, acc, 8);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  if (live && sub == 0) {
    if (mode == 0)
      out[size_t(j) * s.nR + r] = bv - acc;
    else
      out[size_t(j) * s.nF + pos] = bv - acc;
  }
}

// k_patch_gather over a list of DOFs (the cell-boundary ones): same sums, same order.
__global__ void k_patch_gather_list(int64_t n, const int32_t* __restrict__ list, const double* __restrict__ corr,
                                    const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                    double* __restrict__ z) {
  pdl_trigger();
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  int g = 0, q0 = 0, q1 = 0, i0 = 0;
  if (i < n) {
    g = list[i];
    q0 = ptr[g];
    q1 = ptr[g + 1];
    if (q1 > q0) i0 = idx[q0];
  }
  pdl_wait();
  if (i >= n) return;
  double s = q1 > q0 ? corr[i0] : 0.0;
  for (int q = q0 + 1; q < q1; ++q) s += corr[idx[q]];
  z[g] = s;
}

}  // namespace

// Solve records: the separate packed buffer when it exists, else the tiles (packed in place).
static const double* rec_base(const Context& c) { return c.packed.p ? c.packed.p : c.tiles.p; }

void launch_patch_assemble(Context& c) {
  PatchArgs a = make_args(c);
  KernelTimer timer(c, 1);
  FDM_CUDA(cudaMemsetAsync(c.tiles.p, 0, c.tiles.bytes(), c.stream));
  const size_t smem = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 24);
  const int ne = int(c.L.entries.size());
  dim3 grid(unsigned((ne + 255) / 256 < 64 ? (ne + 255) / 256 : 64), c.npatch);
  k_patch_assemble<<<grid, 256, smem, c.stream>>>(a, ne, c.entries.p, c.tile_row.p, c.tile_col.p, c.tiles.p, 0);
  FDM_LAUNCH_CHECK(c);
  k_patch_pad_check<<<c.npatch, 256, 0, c.stream>>>(a, c.tiles.p, c.L.col_start[c.L.nT - 1]);
  FDM_LAUNCH_CHECK(c);
}

// Separator Schur complement of one patch into `out` (ntiles x TT, zeroed here).
void launch_patch_assemble_one(Context& c, int j, double* out) {
  PatchArgs a = make_args(c);
  FDM_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * size_t(c.L.ntiles) * TT, c.stream));
  const size_t smem = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 24);
  const int ne = int(c.L.entries.size());
  dim3 grid(unsigned((ne + 255) / 256 < 148 ? (ne + 255) / 256 : 148), 1);
  k_patch_assemble<<<grid, 256, smem, c.stream>>>(a, ne, c.entries.p, c.tile_row.p, c.tile_col.p, out, j);
  FDM_LAUNCH_CHECK(c);
}

void launch_patch_update(Context& c, int K) {
  PatchArgs a = make_args(c);
  FDM_CUDA(cudaFuncSetAttribute(k_patch_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(double) * (16 + 2 * kUpdStages * TT))));
  const int na = c.L.active_ptr[K + 1] - c.L.active_ptr[K];
  // One operand stage: with the 65 KB diagonal work area three CTAs fit per SM
  // and overlap each other's TMA latency, which measured faster than one CTA
  // with a kUpdStages-deep pipeline in every tile column (C3 31.9 -> 24.8 ms).
  const int nst = 1;
  const size_t diag_area = size_t(T + 1) * T + 16 * T * 4 + T;  // Dm, Lp, rdiag
  const size_t smem = sizeof(double) * (16 + std::max(size_t(2 * nst * TT), diag_area));
  dim3 grid(na, c.npatch);
  KernelTimer timer(c, 1);
  launch_pdl(c.pdl && !c.timing, k_patch_update, grid, dim3(kUpdThreads), smem, c.stream, a, K,
             (const int32_t*)(c.active.p + c.L.active_ptr[K]), (const int32_t*)c.tile_row.p,
             (const int32_t*)c.pair_ptr.p, (const int32_t*)c.pair_a.p, (const int32_t*)c.pair_b.p,
             (const int32_t*)c.tile_mask.p, c.tiles.p, nst);
  FDM_LAUNCH_CHECK(c);
}

// Leading tile columns whose tiles receive no updates (the first separator
// plane: its facets share no cell) are independent: factor all their diagonal
// tiles in one launch (only the diagonal work area: 2 CTAs per SM), then all
// their off-diagonal tiles in one triangular-solve launch.
void launch_patch_lead(Context& c) {
  if (c.L.lead_cols == 0) return;
  PatchArgs a = make_args(c);
  const size_t smem_d = sizeof(double) * (16 + size_t(T + 1) * T + 16 * T * 4 + T);
  const size_t smem_t = sizeof(double) * 2 * TT + 64;
  FDM_CUDA(cudaFuncSetAttribute(k_patch_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(double) * (16 + 2 * kUpdStages * TT))));
  FDM_CUDA(cudaFuncSetAttribute(k_patch_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_t)));
  KernelTimer timer(c, 1);
  k_patch_update<<<dim3(c.L.lead_cols, c.npatch), kUpdThreads, smem_d, c.stream>>>(
      a, -1, c.lead_diag.p, c.tile_row.p, c.pair_ptr.p, c.pair_a.p, c.pair_b.p, c.tile_mask.p, c.tiles.p, 1);
  FDM_LAUNCH_CHECK(c);
  const int nt = int(c.L.lead_trsm.size() / 2);
  if (nt > 0) {
    k_patch_trsm<<<dim3(nt, c.npatch), kUpdThreads, smem_t, c.stream>>>(a, -1, c.col_start.p, c.lead_trsm.p,
                                                                         c.tile_mask.p, c.tiles.p);
    FDM_LAUNCH_CHECK(c);
  }
}

void launch_patch_column(Context& c, int K) {
  PatchArgs a = make_args(c);
  const size_t diag_area = size_t(T + 1) * T + 16 * T * 4 + T;  // Dm, Lp, rdiag
  const size_t smem = sizeof(double) * (16 + std::max(size_t(2 * TT), diag_area));
  FDM_CUDA(cudaFuncSetAttribute(k_patch_column, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int cnt = c.L.col_start[K + 1] - c.L.col_start[K];
  dim3 grid(unsigned(c.npatch * cnt));
  KernelTimer timer(c, 1);
  launch_pdl(c.pdl && !c.timing, k_patch_column, grid, dim3(kUpdThreads), smem, c.stream, a, K,
             (const int32_t*)c.col_start.p, (const int32_t*)c.pair_ptr.p, (const int32_t*)c.pair_a.p,
             (const int32_t*)c.pair_b.p, (const int32_t*)c.tile_mask.p, c.tiles.p, c.fac_flag.p, c.fac_epoch);
  FDM_LAUNCH_CHECK(c);
}

void launch_patch_trsm(Context& c, int K) {
  const int cnt = c.L.col_start[K + 1] - c.L.col_start[K] - 1;
  if (cnt <= 0) return;
  PatchArgs a = make_args(c);
  const size_t smem = sizeof(double) * 2 * TT + 64;
  FDM_CUDA(cudaFuncSetAttribute(k_patch_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  dim3 grid(cnt, c.npatch);
  KernelTimer timer(c, 1);
  launch_pdl(c.pdl && !c.timing, k_patch_trsm, grid, dim3(kUpdThreads), smem, c.stream, a, K,
             (const int32_t*)c.col_start.p, (const int32_t*)nullptr, (const int32_t*)c.tile_mask.p, c.tiles.p);
  FDM_LAUNCH_CHECK(c);
}

// What the separator solve streams: the full factor's records, or (Schur
// split) the dense L_RR records with right-hand sides from the split's tR.
struct SolveView {
  const PatchLayout* L;
  const int32_t* col_start;
  const int32_t* tile_row;
  const int32_t* poff8;
  const int32_t* pdofs;
};
static SolveView solve_view(const Context& c) {
  if (c.sx.on) return {&c.sx.R, c.sx_col_start.p, c.sx_tile_row.p, c.sx_poff8.p, c.sx_pdofs.p};
  return {&c.L, c.col_start.p, c.tile_row.p, c.tile_poff8.p, c.pdofs.p};
}

// Cluster solve (k_patch_solve_cl): per-rank tile lists, built once per CS.
static void build_cluster_lists(Context& c, int cs) {
  if (c.cl_cs == cs) return;
  const auto& L = *solve_view(c).L;
  std::vector<int32_t> list, colp(size_t(cs) * (L.nT + 1));
  for (int r = 0; r < cs; ++r) {
    colp[size_t(r) * (L.nT + 1)] = int32_t(list.size());
    for (int K = 0; K < L.nT; ++K) {
      for (int t = L.col_start[K]; t < L.col_start[K + 1]; ++t)
        if (L.tile_row[t] % cs == r) list.push_back(t);  // the diagonal tile (row K) comes first
      colp[size_t(r) * (L.nT + 1) + K + 1] = int32_t(list.size());
    }
  }
  c.cl_list.upload(list, c.stream);
  c.cl_col.upload(colp, c.stream);
  c.cl_cs = cs;
}

template <int CS>
static size_t solve_cl_smem(const Context& c, int* ring_out) {
  const PatchLayout& L = *solve_view(c).L;
  const size_t budget = 227 * 1024;
  const size_t fixed = sizeof(double) * (size_t(L.mpad) + 2 * kSolveConsumers * T + CS * T + SB8) +
                       2 * kRingEntries * sizeof(uint64_t) + 3 * size_t(L.nT) * sizeof(uint64_t) +
                       kRingEntries * sizeof(int);
  int max_rec = 0;
  for (int t = 0; t < L.ntiles; ++t) max_rec = std::max(max_rec, L.tile_poff8[t + 1] - L.tile_poff8[t]);
  const int ring = fixed < budget ? int(((budget - fixed) / sizeof(double)) & ~size_t(15)) : 0;
  if (ring < max_rec) throw Error(FDMGPU_UNSUPPORTED, "separator too large for the shared-memory cluster solve");
  *ring_out = ring;
  return fixed + size_t(ring) * sizeof(double);
}

// Clusters of cs CTAs of the split solve that can be resident at once.
static int max_active_clusters(Context& c, int cs) {
  auto& memo = c.cl_fit[cs];
  if (memo >= 0) return memo;
  int ring = 0, n = 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kSolveThreads);
  cfg.gridDim = dim3(cs);
  cfg.attrs = at;
  cfg.numAttrs = 1;
  switch (cs) {
    case 3:
      cfg.dynamicSmemBytes = solve_cl_smem<3>(c, &ring);
      FDM_CUDA(cudaFuncSetAttribute(k_patch_solve_cl<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      FDM_CUDA(cudaOccupancyMaxActiveClusters(&n, k_patch_solve_cl<3>, &cfg));
      break;
    case 4:
      cfg.dynamicSmemBytes = solve_cl_smem<4>(c, &ring);
      FDM_CUDA(cudaFuncSetAttribute(k_patch_solve_cl<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      FDM_CUDA(cudaOccupancyMaxActiveClusters(&n, k_patch_solve_cl<4>, &cfg));
      break;
    default:
      cfg.dynamicSmemBytes = solve_cl_smem<2>(c, &ring);
      FDM_CUDA(cudaFuncSetAttribute(k_patch_solve_cl<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      FDM_CUDA(cudaOccupancyMaxActiveClusters(&n, k_patch_solve_cl<2>, &cfg));
  }
  return memo = n;
}

template <int CS>
static void launch_solve_cl(Context& c, const PatchArgs& a, const double* r_modal, int j0) {
  int ring = 0;
  const size_t smem = solve_cl_smem<CS>(c, &ring);
  const SolveView v = solve_view(c);
  FDM_CUDA(cudaFuncSetAttribute(k_patch_solve_cl<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  launch_cluster(c.pdl && !c.timing, CS, k_patch_solve_cl<CS>, dim3((c.npatch - j0) * CS), dim3(kSolveThreads),
                 smem, c.stream, a, ring, r_modal, c.corr.p, rec_base(c), v.pdofs, v.tile_row, v.poff8,
                 (const int32_t*)c.cl_list.p, (const int32_t*)c.cl_col.p, j0, c.tail_sync.p);
}

// Ring size (doubles) of the separator solve: all shared memory left after
// the separator vector, the backward partials, the zero block and the barriers.
static int solve_ring(const Context& c, size_t* smem_out) {
  const PatchLayout& L = *solve_view(c).L;
  const size_t budget = 227 * 1024;
  const size_t fixed = sizeof(double) * (size_t(L.mpad) + kSolveConsumers * T + SB8) +
                       2 * kRingEntries * sizeof(uint64_t) + kRingEntries * sizeof(int);
  int max_rec = 0;
  for (int t = 0; t < L.ntiles; ++t) max_rec = std::max(max_rec, L.tile_poff8[t + 1] - L.tile_poff8[t]);
  const int ring = fixed < budget ? int(((budget - fixed) / sizeof(double)) & ~size_t(15)) : 0;
  if (ring < max_rec) throw Error(FDMGPU_UNSUPPORTED, "separator too large for the shared-memory solve");
  *smem_out = fixed + size_t(ring) * sizeof(double);
  return ring;
}

static void launch_dense_solve(Context& c, const PatchArgs& a, const double* r_modal);

void launch_patch_solve(Context& c, const double* r_modal) {
  KernelTimer timer(c, 0);  // one interval for the whole separator solve (all launches)
  PatchArgs a = make_args(c);
  if (!c.sx.on) {
    launch_dense_solve(c, a, r_modal);
    return;
  }
  const SchurSplit& S = c.sx;
  const SchurArgs s = make_schur_args(c);
  const bool pdl = c.pdl && !c.timing;
  const char* cenv = std::getenv("FDMGPU_COMP_STAGED");
  const bool staged = !(cenv && cenv[0] == '0');
  auto kcomp = staged ? k_schur_comp<true> : k_schur_comp<false>;
  const size_t csm = staged ? sizeof(double) * size_t(S.comp_stride) : 0;
  FDM_CUDA(cudaFuncSetAttribute(kcomp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(csm)));
  const dim3 cgrid(S.ncomp, c.npatch);
  // w = S_FF^{-1} b_F;  t_R = b_R - S_RF w
  launch_pdl(pdl, kcomp, cgrid, dim3(kCompThreads), csm, c.stream, a, s, r_modal, (const double*)nullptr,
             c.sx_F.p, 0);
  FDM_LAUNCH_CHECK(c);
  const char* senv = std::getenv("FDMGPU_SPMV_STAGED");
  const bool sstaged = !(senv && senv[0] == '0');
  const char* tenv = std::getenv("FDMGPU_SPMV_TPR");  // threads per row: 8 | 16 (A/B)
  const int tpr = tenv && std::atoi(tenv) == 16 ? 16 : 8;
  auto kspmv = tpr == 16 ? (sstaged ? k_schur_spmv<true, 16> : k_schur_spmv<false, 16>)
                         : (sstaged ? k_schur_spmv<true, 8> : k_schur_spmv<false, 8>);
  const int spmv_threads = tpr * kSpmvRows;
  const size_t smem_rf = sstaged ? size_t(S.rf_bmax) * 12 : 0, smem_fr = sstaged ? size_t(S.fr_bmax) * 12 : 0;
  FDM_CUDA(cudaFuncSetAttribute(kspmv, cudaFuncAttributeMaxDynamicSharedMemorySize, int(std::max(smem_rf, smem_fr))));
  launch_pdl(pdl, kspmv, dim3(int(S.rf_blk.size()) - 1, c.npatch), dim3(spmv_threads), smem_rf, c.stream, a, s,
             r_modal, (const double*)c.sx_F.p, c.sx_tR.p, 0);
  FDM_LAUNCH_CHECK(c);
  // x_R = S~_RR^{-1} t_R (dense stream) -> corr[nF..m)
  PatchArgs aR = a;
  aR.m = S.R.m;
  aR.mpad = S.R.mpad;
  aR.nT = S.R.nT;
  aR.ntiles = S.R.ntiles;
  aR.rec_stride = int64_t(S.R.tile_poff8.back());
  aR.out_stride = c.L.m;
  aR.out_off = S.nF;
  {
  KernelTimer top_timer(c, 4);  // the top-block stage alone
  if (S.inv) {
    const size_t budget = 227 * 1024;
    const size_t fixed = sizeof(double) * (2 * size_t(S.R.mpad) + 2 * kSymvSlots * T + SB8) +
                         2 * (kRingEntries + kSymvSlots) * sizeof(uint64_t) + kRingEntries * sizeof(int);
    int max_rec = 0;
    for (int t = 0; t < S.R.ntiles; ++t) max_rec = std::max(max_rec, S.R.tile_poff8[t + 1] - S.R.tile_poff8[t]);
    const int ring = fixed < budget ? int(((budget - fixed) / sizeof(double)) & ~size_t(15)) : 0;
    if (ring < max_rec) throw Error(FDMGPU_UNSUPPORTED, "top separator too large for the shared-memory product");
    const size_t smem = fixed + size_t(ring) * sizeof(double);
    // consumer warps: each holds its record while it computes, so fewer warps leave
    // more of the ring in flight (FDMGPU_SYMV_WARPS: 4 | 8, tuning)
    const char* wenv = std::getenv("FDMGPU_SYMV_WARPS");
    const int ncons = wenv && std::atoi(wenv) == 8 ? 8 : 4;
    auto kern = ncons == 8 ? k_schur_symv<8> : k_schur_symv<4>;
    FDM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    launch_pdl(pdl, kern, dim3(c.npatch * S.nchunk), dim3(32 * (ncons + 2)), smem, c.stream, aR, ring, S.nchunk,
               (const int32_t*)c.sx_chunk.p, (const double*)c.sx_tR.p, rec_base(c), (const int32_t*)c.sx_tile_row.p,
               (const int32_t*)c.sx_tile_col.p, (const int32_t*)c.sx_poff8.p, c.sx_part.p);
    FDM_LAUNCH_CHECK(c);
    launch_pdl(pdl, k_schur_xsum, dim3((S.nR + 255) / 256, c.npatch), dim3(256), size_t(0), c.stream, S.nR, S.R.mpad,
               S.nchunk, c.L.m, S.nF, (const double*)c.sx_part.p, c.corr.p);
    FDM_LAUNCH_CHECK(c);
  } else {
    launch_dense_solve(c, aR, c.sx_tR.p);
  }
  }
  // c_F = b_F - S_FR x_R;  x_F = S_FF^{-1} c_F -> corr[0..nF)
  launch_pdl(pdl, kspmv, dim3(int(S.fr_blk.size()) - 1, c.npatch), dim3(spmv_threads), smem_fr, c.stream, a, s,
             r_modal, (const double*)c.corr.p, c.sx_F.p, 1);
  FDM_LAUNCH_CHECK(c);
  launch_pdl(pdl, kcomp, cgrid, dim3(kCompThreads), csm, c.stream, a, s, r_modal, (const double*)c.sx_F.p,
             c.corr.p, 1);
  FDM_LAUNCH_CHECK(c);
}

static void launch_dense_solve(Context& c, const PatchArgs& a, const double* r_modal) {
  const SolveView v = solve_view(c);
  const PatchLayout& L = *v.L;
  // Patches [0, nsolo): one CTA each (full waves); [nsolo, npatch): the last
  // partial wave, each patch split over several SMs (all patches when
  // solve_tail is off).  The split launch goes first and triggers the
  // single-CTA launch once all its CTAs run, so the two overlap; CTA 0 of the
  // single-CTA grid waits for the split CTAs' completion count, so whatever
  // waits for that grid sees both.
  int nsolo = 0;
  unsigned tail_ctas = 0;
  // Split only separators of >= 16 tile columns: below that the per-column
  // exchange costs more than the chain it shortens (C2, 8 columns: 41 us
  // split vs 35 us whole).
  if (c.solve_cs != 1 && L.nT >= 16) {
    int nsm = 0;
    FDM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device));
    nsolo = c.solve_tail ? (c.npatch / nsm) * nsm : 0;
    const int ntail = c.npatch - nsolo;
    if (c.tail_sync.n == 0) {
      c.tail_sync.alloc(2);
      FDM_CUDA(cudaMemsetAsync(c.tail_sync.p, 0, c.tail_sync.bytes(), c.stream));
    }
    // Cluster size: 2 when the single-CTA launch runs beside the split one
    // (the 94 split CTAs leave 54 SMs to it); with no full wave, the largest
    // size whose clusters all fit at once (3-CTA clusters: 45, 4-CTA: 33 at
    // 220 KB per CTA), since a lone patch speeds up with every SM it gets.
    int cs = c.solve_cs;
    if (cs == 0) {
      cs = 2;
      if (nsolo == 0)
        for (int cand : {4, 3})
          if (max_active_clusters(c, cand) >= ntail) {
            cs = cand;
            break;
          }
    }
    if (ntail > 0 && cs >= 2) {
      build_cluster_lists(c, cs);
      switch (cs) {
        case 2: launch_solve_cl<2>(c, a, r_modal, nsolo); break;
        case 3: launch_solve_cl<3>(c, a, r_modal, nsolo); break;
        case 4: launch_solve_cl<4>(c, a, r_modal, nsolo); break;
        default: throw Error(FDMGPU_INVALID_ARGUMENT, "solve cluster size must be 1..4");
      }
      FDM_LAUNCH_CHECK(c);
      tail_ctas = unsigned(ntail * cs);
    }
    if (nsolo == 0) return;
  } else {
    nsolo = c.npatch;
  }
  size_t smem = 0;
  const int ring = solve_ring(c, &smem);
  FDM_CUDA(cudaFuncSetAttribute(k_patch_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  // (PDL after a split tail even when timing: the overlap is part of the solve)
  launch_pdl(c.pdl && (!c.timing || tail_ctas > 0), k_patch_solve, dim3(nsolo), dim3(kSolveThreads), smem, c.stream, a, ring, r_modal,
             c.corr.p, rec_base(c), v.pdofs, v.col_start, v.tile_row, v.poff8, 0, c.tail_sync.p, tail_ctas);
  FDM_LAUNCH_CHECK(c);
}

// Schur split, factor side: S_FF components and the S_RF / S_FR values from mu
// (independent of the factorisation; the same S_G entries as k_patch_assemble).
void launch_schur_setup(Context& c) {
  if (!c.sx.on) return;
  PatchArgs a = make_args(c);
  const SchurArgs s = make_schur_args(c);
  KernelTimer timer(c, 1);
  const size_t smem_c = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 24);
  const int np = int(c.sx.rf_col.size() + c.sx.fr_col.size());  // stored entries (block padding included)
  if (np > 0) {
    dim3 grid(unsigned(std::min(64, (np + 255) / 256)), c.npatch);
    k_schur_couplings<<<grid, 256, smem_c, c.stream>>>(a, s, np, c.sx_pairs.p);
    FDM_LAUNCH_CHECK(c);
  }
  const size_t smem = sizeof(double) * (size_t(T) * (T + 1) * 2 + 16 * T * 4 + T + 2 * T + 24);
  FDM_CUDA(cudaFuncSetAttribute(k_schur_comps, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  k_schur_comps<<<dim3(c.sx.ncomp, c.npatch), 256, smem, c.stream>>>(a, s, c.sx.direct ? 1 : 0);
  FDM_LAUNCH_CHECK(c);
}

static void launch_top_inverse(Context& c);

// Schur split with the top block formed directly (SchurSplit::direct): interior
// pivot check, component inverses, S~_RR into the dense R tiles, its dense tile
// Cholesky (k_patch_column on the R layout's pair lists), then the inverse.
void launch_schur_direct(Context& c) {
  PatchArgs a = make_args(c);
  const SchurArgs s = make_schur_args(c);
  const auto& S = c.sx;
  const auto& R = S.R;
  KernelTimer timer(c, 1);
  k_patch_pad_check<<<c.npatch, 256, 0, c.stream>>>(a, nullptr, 0);
  FDM_LAUNCH_CHECK(c);
  const int c0 = S.c0, c1 = S.c1;
  const size_t smem_i = sizeof(double) * (size_t(c1) * (c0 | 1) + size_t(c1) * (c1 + 1) / 2 + c0 + size_t(c1) * (c1 | 1) +
                                          size_t(c1) * (c0 | 1) + 2);
  FDM_CUDA(cudaFuncSetAttribute(k_schur_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_i)));
  k_schur_inv<<<dim3(S.ncomp, c.npatch), 256, smem_i, c.stream>>>(s, S.nl, c.sx_inv.p);
  FDM_LAUNCH_CHECK(c);
  const int nent = int(S.rk_ent.size());
  k_schur_fv<<<dim3(unsigned(std::min(64, (nent + 255) / 256)), c.npatch), 256, 0, c.stream>>>(s, nent, c.sx_rk_ent.p,
                                                                                                c.sx_fv.p);
  FDM_LAUNCH_CHECK(c);
  const int64_t rstride = int64_t(R.ntiles) * TT;
  const size_t smem_f = sizeof(double) * (size_t(S.nl) * S.nl + T * size_t(S.nl | 1)) + size_t(2) * kFormG * T * 20;
  k_schur_fv2<<<dim3(unsigned(std::min(64, (S.ncomp * S.nRp + 255) / 256)), c.npatch), 256, 0, c.stream>>>(
      s, S.nRp, c.sx_kr.p, c.sx_rk_ent.p, c.sx_fv2.p);
  FDM_LAUNCH_CHECK(c);
  // half-row-tile form (double-buffered Y, one barrier per component) when it fits; FDMGPU_FORM=1 keeps the
  // whole-row-tile kernel
  const size_t smem_f2 = sizeof(double) * (size_t(S.nl) * S.nl + T * size_t(S.nl | 1)) + size_t(2) * kFormG2 * T * 20;
  const char* fenv = std::getenv("FDMGPU_FORM");
  if (!(fenv && fenv[0] == '1') && smem_f2 + 4096 <= 227 * 1024) {
    FDM_CUDA(cudaFuncSetAttribute(k_schur_form2<kFormG2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_f2)));
    k_schur_form2<kFormG2><<<dim3(unsigned(S.form2_I.size()), c.npatch), kFormThreads, smem_f2, c.stream>>>(
        S.nR, S.nRp, S.ncomp, S.nl, c.sx_form2_I.p, c.sx_form2_J0.p, c.sx_kr.p, c.sx_rk_ent.p, nent, c.sx_fv.p,
        c.sx_e2.p, c.sx_fv2.p, c.sx_inv.p, c.sx_col_start.p, c.packed.p, rstride);
  } else {
    FDM_CUDA(cudaFuncSetAttribute(k_schur_form<kFormG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_f)));
    k_schur_form<kFormG><<<dim3(unsigned(S.form_I.size()), c.npatch), kFormThreads, smem_f, c.stream>>>(
        S.nR, S.nRp, S.ncomp, S.nl, c.sx_form_I.p, c.sx_form_J0.p, c.sx_kr.p, c.sx_rk_ent.p, nent, c.sx_fv.p, c.sx_e2.p,
        c.sx_fv2.p, c.sx_inv.p, c.sx_col_start.p, c.packed.p, rstride);
  }
  FDM_LAUNCH_CHECK(c);
  const size_t smem_c = sizeof(double) * (2 * size_t(c.n1) * c.n1 + 24);
  const int nrr = int(S.rr_entries.size());
  k_schur_rr<<<dim3(unsigned(std::min(64, (nrr + 255) / 256)), c.npatch), 256, smem_c, c.stream>>>(
      a, S.nF, nrr, c.sx_rr_entries.p, c.sx_tile_row.p, c.sx_tile_col.p, c.packed.p, rstride);
  FDM_LAUNCH_CHECK(c);
  // dense left-looking tile Cholesky of S~_RR in place (diagonal tiles end as L_KK^{-1})
  PatchArgs ar = a;
  ar.m = S.nR;
  ar.mpad = R.mpad;
  ar.nT = R.nT;
  ar.ntiles = R.ntiles;
  ar.nI = c.L.nI + S.nF;  // pivot positions reported in the patch numbering
  ar.diagL = nullptr;
  const size_t diag_area = size_t(T + 1) * T + 16 * T * 4 + T;
  const size_t smem_k = sizeof(double) * (16 + std::max(size_t(2 * TT), diag_area));
  FDM_CUDA(cudaFuncSetAttribute(k_patch_column, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_k)));
  for (int K = 0; K < R.nT; ++K) {
    const int cnt = R.col_start[K + 1] - R.col_start[K];
    launch_pdl(c.pdl && !c.timing && K > 0, k_patch_column, dim3(unsigned(c.npatch * cnt)), dim3(kUpdThreads), smem_k,
               c.stream, ar, K, (const int32_t*)c.sx_col_start.p, (const int32_t*)c.sx_pair_ptr.p,
               (const int32_t*)c.sx_pair_a.p, (const int32_t*)c.sx_pair_b.p, (const int32_t*)c.sx_tile_mask.p,
               c.packed.p, c.fac_flag.p, c.fac_epoch);
    FDM_LAUNCH_CHECK(c);
  }
  launch_top_inverse(c);
}

// Schur split: the R block of the factored tiles -> dense L_RR stream records.
void launch_schur_retile(Context& c) {
  if (!c.sx.on) return;
  PatchArgs a = make_args(c);
  KernelTimer timer(c, 1);
  const auto& R = c.sx.R;
  const size_t smem = sizeof(double) * (TT + size_t(T) * (T + 1));
  FDM_CUDA(cudaFuncSetAttribute(k_schur_retile, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const bool inv = c.sx.inv;
  const int64_t rstride = int64_t(R.ntiles) * TT;
  k_schur_retile<<<dim3(R.ntiles, c.npatch), 256, smem, c.stream>>>(
      a, c.sx.nF, c.sx_K0, c.sx_tidx.p, c.sx_tile_row.p, c.sx_tile_col.p, c.sx_bptr.p, c.sx_blk.p, c.sx_ccol.p,
      c.sx_poff8.p, c.sx_hdr.p, c.tiles.p, c.diagL.p, c.packed.p, inv ? rstride : int64_t(R.tile_poff8.back()),
      inv ? 1 : 0);
  FDM_LAUNCH_CHECK(c);
  if (!inv) return;
  launch_top_inverse(c);
}

// S~_RR^{-1} = W^T W, W = L_RR^{-1}: U = W^T from the dense L_RR tiles, then A
// into the stream records (over the dense tiles, which U no longer needs)
static void launch_top_inverse(Context& c) {
  const auto& R = c.sx.R;
  const int64_t rstride = int64_t(R.ntiles) * TT;
  const size_t gsm = sizeof(double) * (16 + 2 * TT);
  FDM_CUDA(cudaFuncSetAttribute(k_schur_uinv, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gsm)));
  FDM_CUDA(cudaFuncSetAttribute(k_schur_ainv, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gsm)));
  k_schur_uinv<<<dim3(R.nT, c.npatch), kUpdThreads, gsm, c.stream>>>(R.nT, c.sx_col_start.p, c.packed.p, c.sx_UT.p,
                                                                     rstride);
  FDM_LAUNCH_CHECK(c);
  k_schur_ainv<<<dim3(R.ntiles, c.npatch), kUpdThreads, gsm, c.stream>>>(
      R.nT, c.sx_col_start.p, c.sx_tile_row.p, c.sx_tile_col.p, c.sx_UT.p, rstride, c.sx_bptr.p, c.sx_blk.p,
      c.sx_ccol.p, c.sx_poff8.p, c.sx_hdr.p, c.packed.p, int64_t(R.tile_poff8.back()));
  FDM_LAUNCH_CHECK(c);
}

// Column-wise packing into the separate record buffer (side stream): call
// after column K's tiles are final (after its trsm).
void launch_patch_pack_col(Context& c, int K) {
  if (!c.packed.p || c.sx.on) return;
  if (!c.pack_stream) {
    FDM_CUDA(cudaStreamCreateWithFlags(&c.pack_stream, cudaStreamNonBlocking));
    FDM_CUDA(cudaEventCreateWithFlags(&c.pack_ev, cudaEventDisableTiming));
  }
  const int t0 = c.L.col_start[K], n = c.L.col_start[K + 1] - t0;
  FDM_CUDA(cudaEventRecord(c.pack_ev, c.stream));
  FDM_CUDA(cudaStreamWaitEvent(c.pack_stream, c.pack_ev, 0));
  k_patch_pack_cols<<<dim3(n, c.npatch), 256, 0, c.pack_stream>>>(t0, c.L.ntiles, c.tile_bptr.p, c.tile_blk.p,
                                                                  c.tile_ccol.p, c.tile_poff8.p, c.tile_hdr.p,
                                                                  c.tiles.p, c.packed.p, int64_t(c.L.tile_poff8.back()));
  FDM_LAUNCH_CHECK(c);
}

// Joins the side stream (the records are complete when the handle stream passes this).
void launch_patch_pack_join(Context& c) {
  if (!c.packed.p || !c.pack_stream || c.sx.on) return;
  FDM_CUDA(cudaEventRecord(c.pack_ev, c.pack_stream));
  FDM_CUDA(cudaStreamWaitEvent(c.stream, c.pack_ev, 0));
}

void launch_patch_pack(Context& c) {
  KernelTimer timer(c, 1);
  FDM_CUDA(cudaFuncSetAttribute(k_patch_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, int(2 * TT * sizeof(double))));
  k_patch_pack<<<c.npatch, 512, 2 * TT * sizeof(double), c.stream>>>(c.L.ntiles, c.tile_bptr.p, c.tile_blk.p,
                                                                     c.tile_ccol.p, c.tile_poff8.p, c.tile_hdr.p,
                                                                     c.tiles.p);
  FDM_LAUNCH_CHECK(c);
}

void launch_patch_gather_bnd(Context& c, double* z_modal) {
  if (!c.bnd_list.p) return launch_patch_gather(c, z_modal);
  const int threads = 256;
  const int64_t n = int64_t(c.bnd_list.n), blocks = (n + threads - 1) / threads;
  launch_pdl(c.pdl && !c.timing, k_patch_gather_list, dim3(unsigned(blocks)), dim3(threads), 0, c.stream, n,
             (const int32_t*)c.bnd_list.p, (const double*)c.corr.p, (const int32_t*)c.pg_ptr.p,
             (const int32_t*)c.pg_idx.p, z_modal);
  FDM_LAUNCH_CHECK(c);
}

void launch_patch_gather(Context& c, double* z_modal) {
  const int threads = 256;
  const int64_t blocks = (c.ndof + threads - 1) / threads;
  launch_pdl(c.pdl && !c.timing, k_patch_gather, dim3(unsigned(blocks)), dim3(threads), 0, c.stream, c.ndof,
             (const double*)c.corr.p, (const int32_t*)c.pg_ptr.p, (const int32_t*)c.pg_idx.p, z_modal);
  FDM_LAUNCH_CHECK(c);
}

}  // namespace fdmgpu
