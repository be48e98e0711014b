// Shared symbolic analysis of the vertex-star patches (host, once per handle).
//
// Every interior vertex star of a conforming hex/quad mesh is a (2p-1)^d
// lattice of DOFs; with the reference's patch_ordering (src/ordering.cpp:
// 17-45) all interior stars of a lattice-topology mesh induce the same
// elimination order on that lattice.  This file
//   1. maps each patch's elimination order onto patch-lattice coordinates
//      P in [1, 2p-1]^d and verifies that every patch uses one canonical
//      order (otherwise FDMGPU_UNSUPPORTED: no silent per-patch fallback);
//   2. runs the reference's symbolic pass (etree + column counts,
//      src/cholesky.cpp:18-31) on the canonical patch pattern, generated
//      from the structural Kronecker pattern of A_t / B_t
//      (src/fdm_basis.cpp:58-76, src/assembly.cpp:263-283);
//   3. derives the dense-tile pattern of the interface (separator) factor and
//      the left-looking tile-update pairs used by the batched factorisation.
// Interior columns have exactly d+1 entries (zero fill)
// and are never stored: the kernels rebuild them from mu and the 1D tables.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <functional>
#include <unordered_map>

#include "context.hpp"

namespace fdmgpu {

namespace {

inline int32_t pack(const int* P) { return P[0] | (P[1] << 8) | (P[2] << 16); }
inline void unpack(int32_t v, int* P) {
  P[0] = v & 255;
  P[1] = (v >> 8) & 255;
  P[2] = (v >> 16) & 255;
}

}  // namespace

// Symbolic factorisation (etree + column counts, src/cholesky.cpp:18-31) of
// the canonical patch pattern `neigh` (all structural neighbours of an
// elimination position) and everything the batched kernels derive from it:
// the dense-tile pattern of the columns from L.nI on (the factor the device
// stores), 16x16 / 8x8 sub-block masks, the packed solve-record offsets and
// headers, the left-looking tile-update pairs, the update-free leading
// columns, and the structural nonzeros of the stored block after eliminating
// positions [0, L.nI) (the entries the assembly kernels evaluate).
void symbolic_tiles(PatchLayout& L, const std::function<void(int, std::vector<int>&)>& neigh) {
  const int T = kTile;
  L.nT = (L.m + T - 1) / T;
  L.mpad = L.nT * T;
  std::vector<int> parent(L.n, -1), flag(L.n, -1), colcount(L.n, 1), row;
  std::vector<uint8_t> tmark(size_t(L.nT) * L.nT, 0);
  const char* dbg_env = std::getenv("FDMGPU_DEBUG");
  const bool dbg = dbg_env && dbg_env[0] == '1';
  std::vector<uint8_t> m32(dbg ? size_t(L.mpad / 32) * (L.mpad / 32) : 0), m16(size_t(L.mpad / 16) * (L.mpad / 16), 0);
  std::vector<uint8_t> m8(size_t(L.mpad / 8) * (L.mpad / 8), 0);
  const bool dbg3 = dbg_env && dbg_env[0] == '3';
  std::vector<uint64_t> bits8(m8.size(), 0);  // strictly-lower element mask per 8x8 block
  int64_t nnz_sep = 0;
  std::vector<int> nb;
  for (int k = 0; k < L.n; ++k) {
    neigh(k, nb);
    row.clear();
    for (int pos : nb)
      if (pos < k) row.push_back(pos);
    flag[k] = k;
    for (int j0 : row) {
      for (int jj = j0; jj < k && flag[jj] != k; jj = parent[jj]) {
        if (parent[jj] == -1) parent[jj] = k;
        ++colcount[jj];
        flag[jj] = k;
        if (k >= L.nI && jj >= L.nI) {
          tmark[size_t((k - L.nI) / T) * L.nT + (jj - L.nI) / T] = 1;
          ++nnz_sep;
          m16[size_t((k - L.nI) / 16) * (L.mpad / 16) + (jj - L.nI) / 16] = 1;
          ++m8[size_t((k - L.nI) / 8) * (L.mpad / 8) + (jj - L.nI) / 8];  // strictly-lower entries per 8x8 block
          bits8[size_t((k - L.nI) / 8) * (L.mpad / 8) + (jj - L.nI) / 8] |= uint64_t(1)
                                                                          << (((k - L.nI) % 8) * 8 + (jj - L.nI) % 8);
          if (dbg) m32[size_t((k - L.nI) / 32) * (L.mpad / 32) + (jj - L.nI) / 32] = 1;
        }
      }
    }
  }
  for (int k = 0; k < L.n; ++k) {
    L.nnz_L += colcount[k];
    L.flops_ref += int64_t(colcount[k]) * (colcount[k] - 1) / 2;
  }
  L.colcount = colcount;
  L.nnz_L_reference = L.nnz_L;
  L.flops_reference = L.flops_ref;
  for (int K = 0; K < L.nT; ++K) tmark[size_t(K) * L.nT + K] = 1;
  if (dbg3) {
    // pattern classes of the partially filled off-diagonal 8x8 blocks
    const int nb8 = L.mpad / 8;
    int64_t onerow = 0, onecol = 0, perrow1 = 0, percol1 = 0, other = 0, full = 0, otherslots = 0;
    for (int bi = 0; bi < nb8; ++bi)
      for (int bj = 0; bj < bi; ++bj) {
        const uint64_t b = bits8[size_t(bi) * nb8 + bj];
        if (!b) continue;
        if (b == ~uint64_t(0)) {
          ++full;
          continue;
        }
        int rows = 0, cols = 0, maxr = 0, maxc = 0;
        for (int r = 0; r < 8; ++r) {
          const int n = __builtin_popcountll((b >> (8 * r)) & 0xff);
          rows += n > 0;
          maxr = std::max(maxr, n);
        }
        for (int c = 0; c < 8; ++c) {
          int n = 0;
          for (int r = 0; r < 8; ++r) n += (b >> (8 * r + c)) & 1;
          cols += n > 0;
          maxc = std::max(maxc, n);
        }
        if (rows == 1) ++onerow;
        else if (cols == 1) ++onecol;
        else if (maxr == 1) ++perrow1;
        else if (maxc == 1) ++percol1;
        else {
          ++other;
          otherslots += 64 - __builtin_popcountll(b);
        }
      }
    std::fprintf(stderr, "[fdmgpu] 8x8 blocks: full %lld, one row %lld, one column %lld, <=1 per row %lld, <=1 per column %lld, other %lld (%lld padded slots)\n",
                 (long long)full, (long long)onerow, (long long)onecol, (long long)perrow1, (long long)percol1,
                 (long long)other, (long long)otherslots);
  }
  if (dbg_env && dbg_env[0] == '2') {
    // fill of the off-diagonal 8x8 blocks of the solve records, by tile column
    std::vector<int64_t> hist(65, 0), pad_col(L.nT, 0), blk_col(L.nT, 0);
    const int nb8 = L.mpad / 8;
    for (int bi = 0; bi < nb8; ++bi)
      for (int bj = 0; bj < bi; ++bj) {
        const int v = m8[size_t(bi) * nb8 + bj];
        if (!v) continue;
        ++hist[v];
        pad_col[bj / 8] += 64 - v;
        ++blk_col[bj / 8];
      }
    int64_t pad = 0, blocks = 0;
    for (int v = 1; v <= 64; ++v) {
      pad += hist[v] * (64 - v);
      blocks += hist[v];
    }
    std::fprintf(stderr, "[fdmgpu] off-diagonal 8x8 blocks %lld, padded slots %lld (%.2f %%)\n", (long long)blocks,
                 (long long)pad, 100.0 * pad / (64.0 * blocks));
    for (int v = 1; v <= 64; ++v)
      if (hist[v]) std::fprintf(stderr, "[fdmgpu]   fill %2d: %lld blocks\n", v, (long long)hist[v]);
    for (int K = 0; K < L.nT; ++K)
      std::fprintf(stderr, "[fdmgpu]   tile column %d: %lld blocks, %lld padded slots\n", K, (long long)blk_col[K],
                   (long long)pad_col[K]);
  }
  if (dbg) {
    int64_t t64 = 0, t32 = 0, t16 = 0, t8 = 0;
    for (auto v : m8) t8 += v != 0;
    std::fprintf(stderr, "[fdmgpu] blocks8 %lld (%.3f)\n", (long long)t8, double(nnz_sep + L.m) / (t8 * 64.0));
    for (auto v : tmark) t64 += v;
    for (auto v : m32) t32 += v;
    for (auto v : m16) t16 += v;
    std::fprintf(stderr, "[fdmgpu] sep nnz %lld (+diag %d) | tiles64 %lld (%.3f) | blocks32 %lld (%.3f) | blocks16 %lld (%.3f)\n",
                 (long long)nnz_sep, L.m, (long long)t64, double(nnz_sep + L.m) / (t64 * 4096.0), (long long)t32,
                 double(nnz_sep + L.m) / (t32 * 1024.0), (long long)t16, double(nnz_sep + L.m) / (t16 * 256.0));
  }
  std::vector<int32_t> tidx(size_t(L.nT) * L.nT, -1);
  for (int K = 0; K < L.nT; ++K) {
    L.col_start.push_back(int32_t(L.tile_row.size()));
    for (int I = K; I < L.nT; ++I)
      if (tmark[size_t(I) * L.nT + K]) {
        tidx[size_t(I) * L.nT + K] = int32_t(L.tile_row.size());
        L.tile_row.push_back(I);
        L.tile_col.push_back(K);
      }
  }
  L.col_start.push_back(int32_t(L.tile_row.size()));
  L.ntiles = int(L.tile_row.size());
  // 16x16 sub-block masks (bit bi*4 + bj) used by the factor GEMMs to skip
  // structurally zero k panels: off-diagonal tiles mark the sub-blocks the
  // symbolic factor touches, diagonal tiles (L_KK^{-1}) their lower triangle.
  const int nb16 = L.mpad / 16;
  L.tile_mask.assign(L.ntiles, 0);
  for (int t = 0; t < L.ntiles; ++t) {
    const int I = L.tile_row[t], K = L.tile_col[t];
    int mask = 0;
    for (int bi = 0; bi < 4; ++bi)
      for (int bj = 0; bj < 4; ++bj) {
        const bool on = I == K ? bi >= bj : m16[size_t(4 * I + bi) * nb16 + (4 * K + bj)] != 0;
        if (on) mask |= 1 << (bi * 4 + bj);
      }
    L.tile_mask[t] = mask;
  }
  // 8x8 sub-block masks (bit bi*8 + bj) of the packed solve stream, same rule.
  // Stream record of a tile: a 144-byte header -- the record index of every
  // full sub-block, row-major then column-major (0xff = absent or compact),
  // then the full-block count F and compact count C -- followed by F full
  // blocks (64 doubles), C compact blocks (10 doubles: one value per row, the 8
  // column bytes, the sub-block bit bi*8 + bj) and, when C > 0, the 128-byte
  // compact index table (row-major, column-major; 0xff = not compact).
  // Compact blocks are the off-diagonal sub-blocks with at most one structural
  // entry per row (facet couplings across a shared axis that runs fast in one
  // facet's numbering: one column, or a shifted diagonal): 8 values instead of
  // 64.  Opt-in (FDMGPU_COMPACT=1): 6.5 % (C5) / 12 % (C3) fewer streamed bytes,
  // but the solve's consumers then bound it (C5 19.29 -> 19.42 ms, C3 1.13 ->
  // 1.32 ms, profiles/r2_solve_records.md), so the default keeps every
  // present sub-block full.
  const char* cenv = std::getenv("FDMGPU_COMPACT");
  const bool compact = cenv && cenv[0] == '1';
  const int nb8 = L.mpad / 8;
  L.tile_mask8.assign(L.ntiles, 0);
  L.tile_poff8.assign(L.ntiles + 1, 0);
  L.tile_hdr.assign(size_t(L.ntiles) * kHdrHost, 0);
  L.tile_bptr.assign(L.ntiles + 1, 0);
  L.tile_blk.clear();
  L.tile_ccol.clear();
  for (int t = 0; t < L.ntiles; ++t) {
    const int I = L.tile_row[t], K = L.tile_col[t];
    uint64_t mask = 0, cmask = 0;
    for (int bi = 0; bi < 8; ++bi)
      for (int bj = 0; bj < 8; ++bj) {
        const size_t b8 = size_t(8 * I + bi) * nb8 + (8 * K + bj);
        const bool on = I == K ? bi >= bj : m8[b8] != 0;
        if (!on) continue;
        mask |= uint64_t(1) << (bi * 8 + bj);
        if (compact && I != K) {
          bool sparse_rows = true;
          for (int r = 0; r < 8; ++r) sparse_rows = sparse_rows && __builtin_popcountll((bits8[b8] >> (8 * r)) & 0xff) <= 1;
          if (sparse_rows) cmask |= uint64_t(1) << (bi * 8 + bj);
        }
      }
    L.tile_mask8[t] = int64_t(mask);
    uint8_t* hr = &L.tile_hdr[size_t(t) * kHdrHost];
    uint8_t* ct = hr + kHdrBytes;  // compact index table (stored after the compact blocks when C > 0)
    std::fill(ct, ct + 128, uint8_t(0xff));
    int nf = 0, nc = 0;
    for (int pass = 0; pass < 2; ++pass)  // full blocks first, then compact ones
      for (int b = 0; b < 64; ++b) {
        if (!((mask >> b) & 1) || ((cmask >> b) & 1) != uint64_t(pass)) continue;
        // compact sub-blocks read as absent in the full-block pass (0xff) and
        // through the compact table in the compact pass
        const uint8_t v = pass ? uint8_t(0xff) : uint8_t(nf++);
        hr[b] = v;                            // [bi*8 + bj]
        hr[64 + (b & 7) * 8 + (b >> 3)] = v;  // [bj*8 + bi]
        if (pass) {
          ct[b] = uint8_t(nc);
          ct[64 + (b & 7) * 8 + (b >> 3)] = uint8_t(nc);
          ++nc;
        }
        int64_t cc = 0;
        if (pass) {  // column of each row's entry (0 for an empty row: its values are zero)
          const uint64_t e = bits8[size_t(8 * I + (b >> 3)) * nb8 + (8 * K + (b & 7))];
          for (int r = 0; r < 8; ++r) {
            const unsigned row = unsigned(e >> (8 * r)) & 0xffu;
            cc |= int64_t(row ? __builtin_ctz(row) : 0) << (8 * r);
          }
        }
        L.tile_blk.push_back(b);
        L.tile_ccol.push_back(cc);
      }
    for (int b = 0; b < 64; ++b)
      if (!((mask >> b) & 1)) {
        hr[b] = 0xff;
        hr[64 + (b & 7) * 8 + (b >> 3)] = 0xff;
      }
    reinterpret_cast<int32_t*>(hr + 128)[0] = nf;
    reinterpret_cast<int32_t*>(hr + 128)[1] = nc;
    L.tile_bptr[t + 1] = int32_t(L.tile_blk.size());
    L.tile_poff8[t + 1] = L.tile_poff8[t] + kHdrBytes / 8 + 64 * nf + kCompact * nc + (nc ? 16 : 0);
    // the in-place compaction (k_patch_pack) needs every packed prefix to end
    // before the next unpacked tile starts
    if (int64_t(L.tile_poff8[t + 1]) > int64_t(t + 1) * T * T)
      throw Error(FDMGPU_UNSUPPORTED, "separator factor too dense for the packed solve stream");
  }
  L.pair_ptr.push_back(0);
  for (int t = 0; t < L.ntiles; ++t) {
    const int I = L.tile_row[t], K = L.tile_col[t];
    for (int J = 0; J < K; ++J) {
      const int a = tidx[size_t(I) * L.nT + J], bb = tidx[size_t(K) * L.nT + J];
      // a pair contributes only through the 16-column panels both tiles occupy
      auto panels = [&](int m) {
        int pm = 0;
        for (int q = 0; q < 4; ++q)
          if (m & (0x1111 << q)) pm |= 1 << q;
        return pm;
      };
      if (a >= 0 && bb >= 0 && (panels(L.tile_mask[a]) & panels(L.tile_mask[bb]))) {
        L.pair_a.push_back(a);
        L.pair_b.push_back(bb);
      }
    }
    L.pair_ptr.push_back(int32_t(L.pair_a.size()));
    if (I != K) ++L.tile_gemms;  // TRSM against the diagonal inverse
  }
  L.tile_gemms += int64_t(L.pair_a.size());
  // FP64 tensor-pipe work the factor kernels issue per patch: tile_gemm_abt
  // (kernels/patch.cu) skips the 16-wide k panels where a warp's A rows (two
  // 16-row sub-blocks) or its B rows hold no structural nonzero.
  auto gemm_flops = [&](int ma, int mb) {
    int64_t f = 0;
    for (int w = 0; w < 8; ++w) {
      const int wr = w >> 2, wc = w & 3;
      for (int q = 0; q < 4; ++q) {
        const bool a_on = (((ma >> ((2 * wr) * 4 + q)) | (ma >> ((2 * wr + 1) * 4 + q))) & 1) != 0;
        const bool b_on = ((mb >> (wc * 4 + q)) & 1) != 0;
        if (a_on && b_on) f += 2 * 32 * 16 * 16;
      }
    }
    return f;
  };
  L.dmma_flops = 0;
  for (int t = 0; t < L.ntiles; ++t) {
    for (int q = L.pair_ptr[t]; q < L.pair_ptr[t + 1]; ++q)
      L.dmma_flops += gemm_flops(L.tile_mask[L.pair_a[q]], L.tile_mask[L.pair_b[q]]);
    const int K = L.tile_col[t];
    if (L.tile_row[t] != K) L.dmma_flops += gemm_flops(L.tile_mask[t], L.tile_mask[L.col_start[K]]);  // trsm
  }
  // Update launches only visit tiles with work: the diagonal tile (factor +
  // invert) and off-diagonal tiles with at least one update pair.
  L.active_ptr.assign(1, 0);
  for (int K = 0; K < L.nT; ++K) {
    for (int t = L.col_start[K]; t < L.col_start[K + 1]; ++t)
      if (L.tile_row[t] == K || L.pair_ptr[t + 1] > L.pair_ptr[t]) L.active.push_back(t);
    L.active_ptr.push_back(int32_t(L.active.size()));
  }
  // leading columns with no updates at all (factorised in one batch, launch_patch_lead)
  L.lead_cols = 0;
  while (L.lead_cols < L.nT) {
    const int K = L.lead_cols, t0 = L.col_start[K];
    if (L.active_ptr[K + 1] - L.active_ptr[K] != 1 || L.pair_ptr[t0 + 1] > L.pair_ptr[t0]) break;
    ++L.lead_cols;
  }
  L.lead_diag.clear();
  L.lead_trsm.clear();
  for (int K = 0; K < L.lead_cols; ++K) {
    L.lead_diag.push_back(L.col_start[K]);
    for (int t = L.col_start[K] + 1; t < L.col_start[K + 1]; ++t) {
      L.lead_trsm.push_back(t);
      L.lead_trsm.push_back(L.col_start[K]);
    }
  }

  // Structural nonzeros of the separator Schur complement S_G = A~_GG -
  // A~_GI D^-1 A~_IG (lower triangle), packed (tile << 12 | col << 6 | row):
  // the assembly kernel evaluates only these; every other stored entry
  // starts at zero (fill).
  std::vector<int> nb2, cols;
  std::vector<int> seen(L.n, -1);
  for (int k = L.nI; k < L.n; ++k) {
    neigh(k, nb);
    cols.clear();
    auto add = [&](int cpos) {
      if (cpos >= L.nI && cpos <= k && seen[cpos] != k) {
        seen[cpos] = k;
        cols.push_back(cpos);
      }
    };
    for (int q : nb) {
      if (q >= L.nI) {
        add(q);
      } else {
        neigh(q, nb2);
        for (int q2 : nb2) add(q2);
      }
    }
    const int r = k - L.nI;
    for (int cpos : cols) {
      const int cc = cpos - L.nI;
      const int t = tidx[size_t(r / T) * L.nT + cc / T];
      if (t < 0) throw Error(FDMGPU_UNSUPPORTED, "separator entry outside the tile pattern");
      L.entries.push_back((t << 12) | ((cc % T) << 6) | (r % T));
    }
  }
  std::sort(L.entries.begin(), L.entries.end());
}

// Builds c.L, c.h_pdofs, c.h_pcells from the patch lists.
//
// Boundary stars (SolverConfig::skip_boundary_patches = false, the reference
// default, src/schwarz.cpp:71-81) have fewer than 2^d cells and lose their
// constrained DOFs; they are embedded in the same (2p-1)^d template: missing
// cells leave their slot empty (-1), absent positions get pdofs = -1 and an
// identity row in the separator factor, so every patch shares one symbolic
// layout.  The reference eliminates only the DOFs a star has; a decoupled
// identity row changes no other entry of the factor, so the solution is the
// same up to rounding.
void analyze_patches(Context& c, int npatch, const int32_t* vertex, const int64_t* ptr, const int32_t* dofs,
                     const int32_t* perm, const int32_t* star_cells) {
  const int d = c.dim, p = c.p, n1 = p + 1, ncorner = 1 << d;
  if (p < 2 || p > 31) throw Error(FDMGPU_UNSUPPORTED, "patch layout needs 2 <= p <= 31");
  PatchLayout& L = c.L;
  L = PatchLayout();
  L.span = 2 * p + 1;
  int expect_n = 1, expect_nI = ncorner;
  for (int a = 0; a < d; ++a) {
    expect_n *= 2 * p - 1;
    expect_nI *= p - 1;
  }
  L.n = expect_n;
  L.nI = expect_nI;
  L.m = L.n - L.nI;
  c.h_pdofs.assign(size_t(npatch) * L.n, -1);
  c.h_pcells.assign(size_t(npatch) * ncorner, -1);
  std::vector<int32_t> where(c.ndof, -1), touched, inpatch(c.ndof, -1);
  auto corner_lin = [&](int cb) {
    int l = 0, stride = 1;
    for (int a = 0; a < d; ++a, stride *= n1) l += ((cb >> a) & 1) * p * stride;
    return l;
  };
  auto is_full = [&](int j) {
    if (ptr[j + 1] - ptr[j] != L.n) return false;
    for (int k = 0; k < ncorner; ++k)
      if (star_cells[size_t(j) * ncorner + k] < 0) return false;
    return true;
  };
  // Lattice code of every DOF of patch j, in its own elimination order, and
  // the slot of each star cell.  The corner of cell K at the patch vertex:
  // for a full star, the corner holding the vertex DOF (eliminated last);
  // otherwise the corner that maps all of K's patch DOFs into [1, 2p-1]^d,
  // axes the present DOFs leave free taking side 0 (a star cell adjacent to
  // another across axis a always holds free DOFs of their shared facet, so
  // such a choice never puts two cells in one slot).
  auto map_patch = [&](int j, std::vector<int32_t>& latj) {
    const int64_t b = ptr[j], nj = ptr[j + 1] - ptr[j];
    if (nj < 1 || nj > L.n)
      throw Error(FDMGPU_UNSUPPORTED, "patch " + std::to_string(j) + " (vertex " + std::to_string(vertex[j]) +
                                          ") has " + std::to_string(nj) + " DOFs, at most (2p-1)^d = " +
                                          std::to_string(L.n) + " fit the star lattice");
    const bool full = is_full(j);
    for (int64_t k = 0; k < nj; ++k) {
      const int g = dofs[b + k];
      if (g < 0 || g >= c.ndof) throw Error(FDMGPU_INVALID_ARGUMENT, "set_patches: DOF out of range");
      inpatch[g] = j;
    }
    const int gv = dofs[b + perm[b + nj - 1]];
    for (int k = 0; k < ncorner; ++k) {
      const int K = star_cells[size_t(j) * ncorner + k];
      if (K < 0) continue;
      if (K >= c.ncells) throw Error(FDMGPU_UNSUPPORTED, "patch star cell out of range");
      const int32_t* cd = c.h_cell_dofs.data() + size_t(K) * c.npc;
      int bits = -1;
      if (full) {
        for (int cb = 0; cb < ncorner && bits < 0; ++cb)
          if (cd[corner_lin(cb)] == gv) bits = cb;
      } else {
        int need0 = 0, need1 = 0;  // axes on which K's patch DOFs force the corner side
        int l[3] = {0, 0, 0};
        for (int lin = 0; lin < c.npc; ++lin) {
          if (inpatch[cd[lin]] == j)
            for (int a = 0; a < d; ++a) {
              if (l[a] == 0) need0 |= 1 << a;
              if (l[a] == p) need1 |= 1 << a;
            }
          for (int a = 0; a < d; ++a) {
            if (++l[a] <= p) break;
            l[a] = 0;
          }
        }
        if (!(need0 & need1)) bits = need1;
      }
      if (bits < 0) throw Error(FDMGPU_UNSUPPORTED, "star cell does not contain the patch vertex");
      const int slot = (~bits) & (ncorner - 1);
      if (c.h_pcells[size_t(j) * ncorner + slot] >= 0) throw Error(FDMGPU_UNSUPPORTED, "star cells overlap a slot");
      c.h_pcells[size_t(j) * ncorner + slot] = K;
      int l[3] = {0, 0, 0};
      for (int lin = 0; lin < c.npc; ++lin) {
        int P[3] = {0, 0, 0};
        bool in = true;
        for (int a = 0; a < d; ++a) {
          P[a] = ((slot >> a) & 1) * p + l[a];
          in = in && P[a] >= 1 && P[a] <= 2 * p - 1;
        }
        if (in) {
          const int g = cd[lin];
          const int32_t code = pack(P);
          if (where[g] == -1) {
            where[g] = code;
            touched.push_back(g);
          } else if (where[g] != code) {
            throw Error(FDMGPU_UNSUPPORTED, "inconsistent lattice position of a shared DOF");
          }
        }
        for (int a = 0; a < d; ++a) {
          if (++l[a] <= p) break;
          l[a] = 0;
        }
      }
    }
    latj.assign(nj, -1);
    for (int64_t k = 0; k < nj; ++k) {
      latj[k] = where[dofs[b + perm[b + k]]];
      if (latj[k] < 0) throw Error(FDMGPU_UNSUPPORTED, "patch DOF outside its star lattice");
    }
    for (int g : touched) where[g] = -1;
    touched.clear();
    return full;
  };
  // Canonical template: the elimination order of the first full star (all
  // full stars must share it); with no full star, a synthetic order with the
  // interiors first, then facets, edges and the vertex, each lexicographic.
  std::vector<int32_t> lat0, latj;
  int j0 = -1;
  for (int j = 0; j < npatch && j0 < 0; ++j)
    if (is_full(j)) j0 = j;
  if (j0 >= 0) {
    map_patch(j0, lat0);
    std::fill(c.h_pcells.begin() + size_t(j0) * ncorner, c.h_pcells.begin() + size_t(j0 + 1) * ncorner, -1);
  } else {
    for (int cls = 0; cls <= d; ++cls) {  // number of coordinates at the vertex plane P_a = p
      int P[3] = {0, 0, 0};
      for (int lin = 0; lin < L.n; ++lin) {
        int t = lin, cnt = 0;
        for (int a = 0; a < d; ++a) {
          P[a] = 1 + t % (2 * p - 1);
          t /= 2 * p - 1;
          cnt += P[a] == p;
        }
        if (cnt == cls) lat0.push_back(pack(P));
      }
    }
  }
  auto key = [](int32_t code) { return (code & 63) | (((code >> 8) & 63) << 6) | (((code >> 16) & 63) << 12); };
  std::vector<int32_t> pos0(size_t(1) << 18, -1);  // 2p - 1 <= 63
  for (int k = 0; k < L.n; ++k) pos0[key(lat0[k])] = k;
  L.ragged = 0;
  for (int j = 0; j < npatch; ++j) {
    const int64_t b = ptr[j];
    const bool full = map_patch(j, latj);
    if (full && latj != lat0)
      throw Error(FDMGPU_UNSUPPORTED, "patch " + std::to_string(j) +
                                          " does not share the canonical elimination order (non-lattice mesh)");
    if (!full) ++L.ragged;
    for (size_t k = 0; k < latj.size(); ++k) {
      const int t = pos0[key(latj[k])];
      if (t < 0) throw Error(FDMGPU_UNSUPPORTED, "patch DOF outside its star lattice");
      c.h_pdofs[size_t(j) * L.n + t] = dofs[b + perm[b + k]];
    }
  }
  // Internal separator elimination order.  Default (sep_order 0, "plane"):
  // the facet groups plane by plane -- the facets of one plane never share a
  // cell, so they eliminate without mutual fill (the "one group per facet
  // separator plane" of include/fdmstar/ordering.hpp:25-27) -- then edges,
  // then the vertex; within a group the reference order is kept.  This cuts
  // the separator factor from 1.87M to 1.08M nonzeros at p = 15 (37.6M ->
  // 21.0M at p = 31).  sep_order 1 ("reference") keeps the patch_ordering
  // perm itself (facet groups by global facet id, src/ordering.cpp:17-45).
  // The patch solution is order independent up to rounding.
  const std::vector<int32_t> lat_ref = lat0;
  if (c.sep_order == 0) {
    const int nI0 = expect_nI, m0 = expect_n - expect_nI;
    std::vector<int> idx(m0);
    for (int r = 0; r < m0; ++r) idx[r] = r;
    auto key = [&](int r) {
      int P[3];
      unpack(lat0[nI0 + r], P);
      int cnt = 0, ax = 0;
      for (int a = 0; a < d; ++a)
        if (P[a] == p) {
          ++cnt;
          ax = a;
        }
      return cnt == 1 ? ax : (cnt == 2 ? d : d + 1);
    };
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return key(x) < key(y); });
    std::vector<int32_t> lat1(lat0);
    for (int r = 0; r < m0; ++r) lat1[nI0 + r] = lat0[nI0 + idx[r]];
    for (int j = 0; j < npatch; ++j) {
      std::vector<int32_t> tmp(c.h_pdofs.begin() + size_t(j) * L.n + nI0, c.h_pdofs.begin() + size_t(j + 1) * L.n);
      for (int r = 0; r < m0; ++r) c.h_pdofs[size_t(j) * L.n + nI0 + r] = tmp[idx[r]];
    }
    lat0 = lat1;
  }
  L.lat = lat0;
  int span_d = 1;
  for (int a = 0; a < d; ++a) span_d *= L.span;
  L.pos_of_lat.assign(span_d, -1);
  auto lin_of = [&](const int* P) {
    int v = 0, s = 1;
    for (int a = 0; a < d; ++a, s *= L.span) v += P[a] * s;
    return v;
  };
  for (int k = 0; k < L.n; ++k) {
    int P[3];
    unpack(L.lat[k], P);
    L.pos_of_lat[lin_of(P)] = k;
    bool interior = true;
    for (int a = 0; a < d; ++a) interior = interior && P[a] != p;
    if (interior != (k < L.nI)) throw Error(FDMGPU_UNSUPPORTED, "patch ordering does not eliminate interiors first");
  }

  // ---- symbolic factorisation of the canonical patch (src/cholesky.cpp:18-31)
  std::vector<std::vector<int>> Acols(n1);
  for (int i = 0; i < n1; ++i)
    for (int jj = 0; jj < n1; ++jj)
      if (c.h_Anz[i + size_t(n1) * jj] || c.h_Bnz[i + size_t(n1) * jj]) Acols[i].push_back(jj);
  auto has = [&](const std::vector<uint8_t>& nz, int i, int jj) { return nz[i + size_t(n1) * jj] != 0; };
  std::vector<int> mark(L.n, -1);
  int stamp = 0;
  // All structural neighbours (any position) of position k in the canonical
  // patch matrix: union of the Kronecker patterns of the cells containing it.
  auto neigh = [&](int k, std::vector<int>& out) {
    out.clear();
    ++stamp;
    int P[3];
    unpack(L.lat[k], P);
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
      lo[a] = a < d ? (P[a] > p ? 1 : 0) : 0;
      hi[a] = a < d ? (P[a] < p ? 0 : 1) : 0;
    }
    for (int s2 = lo[2]; s2 <= hi[2]; ++s2)
      for (int s1 = lo[1]; s1 <= hi[1]; ++s1)
        for (int s0 = lo[0]; s0 <= hi[0]; ++s0) {
          const int s[3] = {s0, s1, s2};
          int l[3] = {0, 0, 0};
          for (int a = 0; a < d; ++a) l[a] = P[a] - s[a] * p;
          const auto& c0 = Acols[l[0]];
          const auto& c1 = Acols[l[1]];
          static const std::vector<int> zero{0};
          const auto& c2 = d == 3 ? Acols[l[2]] : zero;
          for (int x2 : c2)
            for (int x1 : c1)
              for (int x0 : c0) {
                const int x[3] = {x0, x1, x2};
                bool any = false;
                for (int a = 0; a < d && !any; ++a) {
                  bool all = true;
                  for (int bb = 0; bb < d && all; ++bb) all = has(bb == a ? c.h_Anz : c.h_Bnz, l[bb], x[bb]);
                  any = all;
                }
                if (!any) continue;
                int Q[3] = {0, 0, 0};
                bool in = true;
                for (int a = 0; a < d; ++a) {
                  Q[a] = s[a] * p + x[a];
                  in = in && Q[a] >= 1 && Q[a] <= 2 * p - 1;
                }
                if (!in) continue;
                const int pos = L.pos_of_lat[lin_of(Q)];
                if (pos >= 0 && mark[pos] != stamp) {
                  mark[pos] = stamp;
                  out.push_back(pos);
                }
              }
        }
  };
  symbolic_tiles(L, neigh);
  std::vector<int> nb;
  if (lat_ref != L.lat) {
    // Column counts under the reference patch_ordering (SURVEY.md Appendix A
    // figures, reported beside the ones of the order in use).
    const std::vector<int32_t> lat_use = L.lat;
    auto set_lat = [&](const std::vector<int32_t>& lt) {
      L.lat = lt;
      std::fill(L.pos_of_lat.begin(), L.pos_of_lat.end(), -1);
      for (int k = 0; k < L.n; ++k) {
        int P[3];
        unpack(L.lat[k], P);
        L.pos_of_lat[lin_of(P)] = k;
      }
    };
    set_lat(lat_ref);
    std::vector<int> par2(L.n, -1), flag2(L.n, -1), cc2(L.n, 1);
    for (int k = 0; k < L.n; ++k) {
      neigh(k, nb);
      flag2[k] = k;
      for (int j0 : nb) {
        if (j0 >= k) continue;
        for (int jj = j0; jj < k && flag2[jj] != k; jj = par2[jj]) {
          if (par2[jj] == -1) par2[jj] = k;
          ++cc2[jj];
          flag2[jj] = k;
        }
      }
    }
    L.nnz_L_reference = 0;
    L.flops_reference = 0;
    for (int k = 0; k < L.n; ++k) {
      L.nnz_L_reference += cc2[k];
      L.flops_reference += int64_t(cc2[k]) * (cc2[k] - 1) / 2;
    }
    set_lat(lat_use);
  }
}

}  // namespace fdmgpu
