// Two-level Schur split of the separator solve: host analysis (see
// SchurSplit in context.hpp for the algebra).
//
// Reference path: CholFactor::solve (src/cholesky.cpp:89-110) applied to the
// patch matrix of PatchSolver::apply (src/schwarz.cpp:41-54).  The device
// factorisation is unchanged (the full separator Cholesky, kernels/patch.cu);
// only what the relaxation streams changes.  With the separator ordered
// P0 | P1 | R (facet planes 0 and 1 first, layout.cpp "plane" order), block
// elimination gives the same solution as the full triangular solves up to
// rounding, while the solve reads the dense factor of the last block
// (|R| = (2p-1)^2 ... at p = 31: 3781 of 10981 separator DOFs; 7.15 M of the
// 21.0 M separator-factor nonzeros) and S's own unfilled couplings.
//
// Everything here is derived from the canonical symbolic pattern of S_G
// (L.entries) and checked; when a check fails (reference separator order,
// DG layouts, 2D with a large P1 block, ...) the split stays off and the
// full-factor stream is used.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <string>

#include "context.hpp"

namespace fdmgpu {

namespace {

int find(std::vector<int>& par, int x) {
  while (par[x] != x) x = par[x] = par[par[x]];
  return x;
}

// Dense lower tile layout of an nR x nR block with full-block records: 8x8
// sub-blocks inside the block (diagonal tiles: bi >= bj, or all of them for the
// symmetric inverse, sym), a header like symbolic_tiles' (no compact blocks).
void dense_layout(PatchLayout& R, int nR, bool sym) {
  const int T = kTile;
  R = PatchLayout();
  R.m = nR;
  R.nT = (nR + T - 1) / T;
  R.mpad = R.nT * T;
  for (int K = 0; K < R.nT; ++K) {
    R.col_start.push_back(int32_t(R.tile_row.size()));
    for (int I = K; I < R.nT; ++I) {
      R.tile_row.push_back(I);
      R.tile_col.push_back(K);
    }
  }
  R.col_start.push_back(int32_t(R.tile_row.size()));
  R.ntiles = int(R.tile_row.size());
  R.tile_mask8.assign(R.ntiles, 0);
  R.tile_poff8.assign(R.ntiles + 1, 0);
  R.tile_hdr.assign(size_t(R.ntiles) * kHdrHost, 0);
  R.tile_bptr.assign(R.ntiles + 1, 0);
  const int nb = (nR + 7) / 8;  // 8-row blocks holding a row of the block
  for (int t = 0; t < R.ntiles; ++t) {
    const int I = R.tile_row[t], K = R.tile_col[t];
    uint64_t mask = 0;
    for (int bi = 0; bi < 8; ++bi)
      for (int bj = 0; bj < 8; ++bj)
        if (8 * I + bi < nb && 8 * K + bj < nb && (sym || I != K || bi >= bj)) mask |= uint64_t(1) << (bi * 8 + bj);
    R.tile_mask8[t] = int64_t(mask);
    uint8_t* hr = &R.tile_hdr[size_t(t) * kHdrHost];
    std::fill(hr + kHdrBytes, hr + kHdrHost, uint8_t(0xff));
    int nf = 0;
    for (int b = 0; b < 64; ++b) {
      const uint8_t v = ((mask >> b) & 1) ? uint8_t(nf) : uint8_t(0xff);
      hr[b] = v;
      hr[64 + (b & 7) * 8 + (b >> 3)] = v;
      if ((mask >> b) & 1) {
        ++nf;
        R.tile_blk.push_back(b);
        R.tile_ccol.push_back(0);
      }
    }
    reinterpret_cast<int32_t*>(hr + 128)[0] = nf;
    reinterpret_cast<int32_t*>(hr + 128)[1] = 0;
    R.tile_bptr[t + 1] = int32_t(R.tile_blk.size());
    R.tile_poff8[t + 1] = R.tile_poff8[t] + kHdrBytes / 8 + 64 * nf;
  }
  R.nnz_L = int64_t(nR) * (nR + 1) / 2;
}

}  // namespace

void analyze_schur_split(Context& c) {
  SchurSplit& S = c.sx;
  S = SchurSplit();
  const PatchLayout& L = c.L;
  const char* env = std::getenv("FDMGPU_SCHUR");
  if (!c.schur_enabled || (env && env[0] == '0') || c.dg || L.m < 2) return;
  const int d = c.dim, p = c.p, m = L.m;
  auto group = [&](int r) {
    const int32_t v = L.lat[L.nI + r];
    const int P[3] = {v & 255, (v >> 8) & 255, (v >> 16) & 255};
    int cnt = 0, ax = 0;
    for (int a = 0; a < d; ++a)
      if (P[a] == p) {
        ++cnt;
        ax = a;
      }
    return cnt == 1 ? ax : d + cnt;  // facet axis, else edge / vertex
  };
  // P0 = [0, n0), P1 = [n0, nF) must be the leading contiguous groups 0 and 1
  int n0 = 0;
  while (n0 < m && group(n0) == 0) ++n0;
  int nF = n0;
  while (nF < m && group(nF) == 1) ++nF;
  if (n0 == 0 || nF == n0 || nF >= m) return;
  for (int r = nF; r < m; ++r)
    if (group(r) <= 1) return;
  // structural nonzeros (r > c) of S_G
  std::vector<std::pair<int, int>> pr;
  pr.reserve(L.entries.size());
  for (int32_t code : L.entries) {
    const int t = code >> 12, cc = (code >> 6) & 63, rr = code & 63;
    const int r = L.tile_row[t] * kTile + rr, col = L.tile_col[t] * kTile + cc;
    if (r != col) pr.emplace_back(r, col);
  }
  std::vector<int> par(nF);
  std::iota(par.begin(), par.end(), 0);
  for (auto [r, col] : pr) {
    if (r < nF && col < nF) {
      const bool r0 = r < n0, c0 = col < n0;
      if (r0 == c0) return;  // a coupling inside P0 or inside P1: S_FF is not of the split form
      par[find(par, r)] = find(par, col);
    }
  }
  // components in order of their smallest position
  std::vector<int> cid(nF, -1);
  std::vector<std::vector<int>> m0, m1;
  for (int r = 0; r < nF; ++r) {
    const int root = find(par, r);
    if (cid[root] < 0) {
      cid[root] = int(m0.size());
      m0.emplace_back();
      m1.emplace_back();
    }
    (r < n0 ? m0 : m1)[cid[root]].push_back(r);
  }
  const int ncomp = int(m0.size());
  int c0 = 1, c1 = 1;
  for (int k = 0; k < ncomp; ++k) {
    c0 = std::max(c0, int(m0[k].size()));
    c1 = std::max(c1, int(m1[k].size()));
  }
  if (c0 > 64 || c1 > 64) return;  // the component kernel holds one component per CTA in registers / smem
  S.n0 = n0;
  S.n1 = nF - n0;
  S.nF = nF;
  S.nR = m - nF;
  S.ncomp = ncomp;
  S.c0 = c0;
  S.c1 = c1;
  S.comp0.assign(size_t(ncomp) * c0, -1);
  S.comp1.assign(size_t(ncomp) * c1, -1);
  for (int k = 0; k < ncomp; ++k) {
    std::copy(m0[k].begin(), m0[k].end(), S.comp0.begin() + size_t(k) * c0);
    std::copy(m1[k].begin(), m1[k].end(), S.comp1.begin() + size_t(k) * c1);
  }
  // S_RF (R rows, F columns) and its transpose S_FR (F rows in component order)
  std::vector<std::vector<int>> rf(S.nR), fr(nF);
  for (auto [r, col] : pr)
    if (r >= nF && col < nF) {
      rf[r - nF].push_back(col);
      fr[col].push_back(r - nF);
    }
  // Row blocks of kSpmvRows rows, each block's entries starting on a 4-entry
  // boundary (padding: column 0, value 0) so the solve stages a block's values
  // and columns with one 16-byte-aligned bulk copy each.
  auto blocked = [&](int nrows, auto&& row_of, std::vector<int32_t>& ptr, std::vector<int32_t>& col,
                     std::vector<int32_t>& blk, int& bmax, int64_t& nnz) {
    ptr.assign(nrows + 1, 0);
    col.clear();
    blk.clear();
    bmax = 0;
    nnz = 0;
    for (int r = 0; r < nrows; ++r) {
      if (r % kSpmvRows == 0) {
        while (col.size() % 4) col.push_back(0);
        if (!blk.empty()) bmax = std::max(bmax, int(col.size()) - blk.back());
        blk.push_back(int32_t(col.size()));
      }
      auto& row = row_of(r);
      std::sort(row.begin(), row.end());
      ptr[r] = int32_t(col.size());
      col.insert(col.end(), row.begin(), row.end());
      nnz += int64_t(row.size());
    }
    ptr[nrows] = int32_t(col.size());
    while (col.size() % 4) col.push_back(0);
    if (!blk.empty()) bmax = std::max(bmax, int(col.size()) - blk.back());
    blk.push_back(int32_t(col.size()));
  };
  blocked(S.nR, [&](int r) -> std::vector<int>& { return rf[r]; }, S.rf_ptr, S.rf_col, S.rf_blk, S.rf_bmax, S.rf_nnz);
  S.comp_fr.assign(1, 0);
  for (int k = 0; k < ncomp; ++k) {
    for (const auto* mem : {&m0[k], &m1[k]})
      for (int f : *mem) S.fr_row.push_back(f);
    S.comp_fr.push_back(int32_t(S.fr_row.size()));
  }
  blocked(nF, [&](int i) -> std::vector<int>& { return fr[S.fr_row[i]]; }, S.fr_ptr, S.fr_col, S.fr_blk, S.fr_bmax,
          S.fr_nnz);
  // component block: M (c1 rows, stride c0 | 1: the odd stride keeps row-per-thread and
  // column-per-thread reads bank-conflict free), W lower triangle packed by rows (row i at
  // i(i+1)/2), D0 (c0); 16-byte aligned for the bulk copy
  S.comp_stride = (int64_t(c1) * (c0 | 1) + int64_t(c1) * (c1 + 1) / 2 + c0 + 1) & ~int64_t(1);
  S.rf_off = S.comp_stride * ncomp;
  S.fr_off = S.rf_off + int64_t(S.rf_col.size());
  S.vstride = (S.fr_off + int64_t(S.fr_col.size()) + 3) & ~int64_t(3);  // 32-byte aligned patch blocks
  // top block: the symmetric inverse S~_RR^{-1} (default; one streamed pass per
  // solve) or its Cholesky factor L_RR (FDMGPU_TOP=chol: forward + backward passes)
  const char* top = std::getenv("FDMGPU_TOP");
  S.inv = !(top && std::string(top) == "chol");
  dense_layout(S.R, S.nR, S.inv);
  // worth it only when the split reads clearly fewer values than the full
  // stream (3D: ~0.35 of them; 2D: R is the vertex alone, no gain)
  int64_t comp = 0;
  for (int k = 0; k < ncomp; ++k) {
    const int64_t a0 = int64_t(m0[k].size()), a1 = int64_t(m1[k].size());
    comp += a1 * a0 + a1 * (a1 + 1) / 2 + a0;
  }
  const int64_t split_vals = 2 * S.R.nnz_L + 2 * comp + S.rf_nnz + S.fr_nnz;
  const int64_t full_vals = 2 * (L.nnz_L - int64_t(d + 1) * L.nI);
  if (4 * split_vals > 3 * full_vals && !(env && env[0] == '1')) {
    S = SchurSplit();
    return;
  }
  S.on = true;
  // Direct top block: per-component views of S_RF, the structural entries of
  // S_RR in the R tile layout and the dense left-looking update lists.
  const char* dir = std::getenv("FDMGPU_DIRECT");
  S.direct = S.inv && !(dir && dir[0] == '0') && c0 + c1 <= 128 && (c0 + c1) % 2 == 0 && S.rf_col.size() < (size_t(1) << 23);  // (even: Inv_k moves by 16-byte bulk copies)
  if (!S.direct) return;
  S.nl = c0 + c1;
  S.nRp = S.R.mpad;
  std::vector<int> fcomp(nF, 0), floc(nF, 0);
  for (int k = 0; k < ncomp; ++k) {
    for (size_t i = 0; i < m0[k].size(); ++i) {
      fcomp[m0[k][i]] = k;
      floc[m0[k][i]] = int(i);
    }
    for (size_t i = 0; i < m1[k].size(); ++i) {
      fcomp[m1[k][i]] = k;
      floc[m1[k][i]] = c0 + int(i);
    }
  }
  std::vector<std::vector<int32_t>> bucket(size_t(ncomp) * S.nR);  // (component, row) -> entries
  for (int r = 0; r < S.nR; ++r)
    for (int e = S.rf_ptr[r]; e < S.rf_ptr[r + 1]; ++e) {
      const int f = S.rf_col[e];
      bucket[size_t(fcomp[f]) * S.nR + r].push_back(int32_t(floc[f] | (e << 8)));
    }
  S.kr.assign(size_t(ncomp) * S.nRp, 0);
  S.rk_ent.clear();
  for (int k = 0; k < ncomp; ++k)
    for (int r = 0; r < S.nR; ++r) {
      const auto& b = bucket[size_t(k) * S.nR + r];
      if (b.size() > 255 || S.rk_ent.size() >= (size_t(1) << 23)) {
        S.direct = false;
        return;
      }
      S.kr[size_t(k) * S.nRp + r] = int32_t((S.rk_ent.size() << 8) | b.size());
      S.rk_ent.insert(S.rk_ent.end(), b.begin(), b.end());
    }
  if (S.rk_ent.empty()) S.rk_ent.push_back(0);
  // direct-indexed view of the first two entries (the common case: one P0 and one P1 mode)
  S.e2.assign(size_t(ncomp) * S.nRp, 0);
  for (int k = 0; k < ncomp; ++k)
    for (int r = 0; r < S.nR; ++r) {
      const auto& b = bucket[size_t(k) * S.nR + r];
      const int n = int(b.size());
      const int l0 = n > 0 ? (b[0] & 255) : 0, l1 = n > 1 ? (b[1] & 255) : 0;
      S.e2[size_t(k) * S.nRp + r] = int32_t(l0 | (l1 << 8) | (std::min(n, 2) << 16) | ((n > 2 ? 1 : 0) << 18));
    }
  // S_RR: structural entries of S_G inside R x R (both triangles inside diagonal tiles),
  // the diagonal, and the identity on the padding rows
  std::vector<int32_t> tix(size_t(S.R.nT) * S.R.nT, -1);
  for (int t = 0; t < S.R.ntiles; ++t) tix[size_t(S.R.tile_row[t]) * S.R.nT + S.R.tile_col[t]] = t;
  auto add_rr = [&](int r, int col) {
    const int I = r / kTile, J = col / kTile;
    if (I < J) return;
    S.rr_entries.push_back(int32_t((tix[size_t(I) * S.R.nT + J] << 12) | ((col % kTile) << 6) | (r % kTile)));
  };
  for (auto [r, col] : pr)
    if (r >= nF && col >= nF) {
      add_rr(r - nF, col - nF);
      add_rr(col - nF, r - nF);
    }
  for (int r = 0; r < S.nRp; ++r) add_rr(r, r);
  std::sort(S.rr_entries.begin(), S.rr_entries.end());
  S.rr_entries.erase(std::unique(S.rr_entries.begin(), S.rr_entries.end()), S.rr_entries.end());
  for (int I = 0; I < S.R.nT; ++I)
    for (int J0 = 0; J0 <= I; J0 += kFormG) {
      S.form_I.push_back(I);
      S.form_J0.push_back(J0);
    }
  for (int Ih = 0; Ih < 2 * S.R.nT; ++Ih)
    for (int J0 = 0; J0 <= Ih / 2; J0 += kFormG2) {
      S.form2_I.push_back(Ih);
      S.form2_J0.push_back(J0);
    }
  // dense left-looking updates: tile (I, K) -= sum_{J < K} L(I, J) L(K, J)^T
  S.pair_ptr.assign(1, 0);
  for (int t = 0; t < S.R.ntiles; ++t) {
    const int I = S.R.tile_row[t], K = S.R.tile_col[t];
    for (int J = 0; J < K; ++J) {
      S.pair_a.push_back(tix[size_t(I) * S.R.nT + J]);
      S.pair_b.push_back(tix[size_t(K) * S.R.nT + J]);
    }
    S.pair_ptr.push_back(int32_t(S.pair_a.size()));
  }
  if (S.pair_a.empty()) {
    S.pair_a.push_back(0);
    S.pair_b.push_back(0);
  }
  S.tile_mask.assign(S.R.ntiles, 0xffff);
}

}  // namespace fdmgpu
