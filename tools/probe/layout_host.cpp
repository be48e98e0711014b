// Host-only layout statistics (no GPU): runs the library's shared symbolic
// analysis (fdmgpu::analyze_patches / symbolic_tiles) on a configuration and
// prints the separator factor structure: tiles, nnz, stored solve-record
// bytes, tile GEMM pairs, and the padding of the 8x8 sub-block records.
//   g++ -O2 -std=c++20 -I include -I paper_2107_14758_b200/csrc tools/probe/layout_host.cpp \
//       -L paper_2107_14758_b200/lib -lfdmgpu -Wl,-rpath,$PWD/paper_2107_14758_b200/lib -o /tmp/layout_host
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "context.hpp"
#include "fdmhost.h"

namespace fdmgpu {
void analyze_patches(Context& c, int npatch, const int32_t* vertex, const int64_t* ptr, const int32_t* dofs,
                     const int32_t* perm, const int32_t* star_cells);
void analyze_schur_split(Context& c);
}

int main(int argc, char** argv) {
  const int config = argc > 1 ? std::atoi(argv[1]) : 3, n = argc > 2 ? std::atoi(argv[2]) : 0,
            p = argc > 3 ? std::atoi(argv[3]) : 0, order = argc > 4 ? std::atoi(argv[4]) : 0;
  void* pb = fdmhost_problem_create(config, n, p);
  if (!pb) {
    std::fprintf(stderr, "%s\n", fdmhost_last_error());
    return 1;
  }
  int64_t info[16];
  fdmhost_problem_info(pb, info);
  const int dim = int(info[0]), pp = int(info[1]), nc = int(info[2]), npatch = int(info[5]), npc = int(info[7]);
  const int64_t ndof = info[3], sum_nj = info[8];
  fdmgpu::Context c;
  c.dim = dim;
  c.p = pp;
  c.n1 = pp + 1;
  c.npc = npc;
  c.ncells = nc;
  c.ndof = ndof;
  c.sep_order = order;
  const int n1 = pp + 1;
  std::vector<double> S(n1 * n1), At(n1 * n1), Bt(n1 * n1), Ah(n1 * n1), Bh(n1 * n1), lam(n1), par(n1), nodes(n1);
  c.h_Anz.resize(n1 * n1);
  c.h_Bnz.resize(n1 * n1);
  fdmhost_get_basis(pb, S.data(), At.data(), Bt.data(), c.h_Anz.data(), c.h_Bnz.data(), lam.data(), par.data(),
                    Ah.data(), Bh.data(), nodes.data());
  c.h_cell_dofs.resize(size_t(nc) * npc);
  std::vector<int32_t> cm(size_t(nc) * npc);
  fdmhost_get_maps(pb, c.h_cell_dofs.data(), cm.data(), nullptr, nullptr, nullptr, nullptr);
  std::vector<int32_t> vert(npatch), dofs(sum_nj), perm(sum_nj), cells(size_t(npatch) << dim), col(npatch);
  std::vector<int64_t> ptr(npatch + 1);
  fdmhost_get_patches(pb, vert.data(), ptr.data(), dofs.data(), perm.data(), cells.data(), col.data());
  fdmgpu::analyze_patches(c, npatch, vert.data(), ptr.data(), dofs.data(), perm.data(), cells.data());
  const auto& L = c.L;
  fdmgpu::analyze_schur_split(c);
  {
    const auto& S = c.sx;
    const double dense = double(S.R.tile_poff8.empty() ? 0 : S.R.tile_poff8.back()) * 8;
    const double vals = double(S.vstride) * 8;
    std::printf("schur split %d: n0 %d n1 %d nR %d comps %d (c0 %d c1 %d) rf nnz %zu fr nnz %zu; R tiles %d records %.0f B, "
                "values %.0f B (components %.0f B); per sweep (fwd+bwd records, comps x2, rf, fr) %.0f B\n",
                int(S.on), S.n0, S.n1, S.nR, S.ncomp, S.c0, S.c1, S.rf_col.size(), S.fr_col.size(), S.R.ntiles, dense,
                vals, 8.0 * S.rf_off, 2 * dense + 2 * 8.0 * S.rf_off + 8.0 * (S.rf_col.size() + S.fr_col.size()));
  }
  int64_t blocks8 = 0, diag_blocks = 0;
  for (int t = 0; t < L.ntiles; ++t) {
    const int b = __builtin_popcountll(uint64_t(L.tile_mask8[t]));
    blocks8 += b;
    if (L.tile_row[t] == L.tile_col[t]) diag_blocks += b;
  }
  const int64_t nnz_sep = L.nnz_L - int64_t(dim + 1) * L.nI;
  std::printf("config %d p %d: n %d nI %d m %d nT %d tiles %d lead_cols %d\n", config, pp, L.n, L.nI, L.m, L.nT,
              L.ntiles, L.lead_cols);
  std::printf("nnz_L %lld (reference order %lld), separator nnz %lld, flops %lld (ref %lld), tile gemms %lld, pairs %zu\n",
              (long long)L.nnz_L, (long long)L.nnz_L_reference, (long long)nnz_sep, (long long)L.flops_ref,
              (long long)L.flops_reference, (long long)L.tile_gemms, L.pair_a.size());
  const double rec = double(L.tile_poff8.back()) * 8;
  std::printf("stored record bytes / patch %.0f (headers %.0f, 8x8 blocks %lld = %.0f B), nnz bytes %.0f: ratio %.4f\n",
              rec, 128.0 * L.ntiles, (long long)blocks8, 512.0 * blocks8, 8.0 * nnz_sep, rec / (8.0 * nnz_sep));
  std::printf("diag-tile blocks %lld; dense tile flops %.4e vs in-use %.4e (x%.2f)\n", (long long)diag_blocks,
              2.0 * 64 * 64 * 64 * double(L.tile_gemms), 2.0 * double(L.flops_ref),
              2.0 * 64 * 64 * 64 * double(L.tile_gemms) / (2.0 * double(L.flops_ref)));
  // DMMA work the factor kernels execute: tile_gemm_abt skips the 16-wide k
  // panels where a warp's A rows (two 16-row sub-blocks) or B rows hold no
  // structural nonzero (kernels/patch.cu); warp w: A sub-rows 2(w>>2), 2(w>>2)+1, B sub-row w&3.
  auto gemm_flops = [&](int ma, int mb) {
    double f = 0.0;
    for (int w = 0; w < 8; ++w) {
      const int wr = w >> 2, wc = w & 3;
      for (int q = 0; q < 4; ++q) {
        const bool a_on = (((ma >> ((2 * wr) * 4 + q)) | (ma >> ((2 * wr + 1) * 4 + q))) & 1) != 0;
        const bool b_on = ((mb >> (wc * 4 + q)) & 1) != 0;
        if (a_on && b_on) f += 2.0 * 32 * 16 * 16;
      }
    }
    return f;
  };
  double exec = 0.0;
  for (int t = 0; t < L.ntiles; ++t) {
    for (int q = L.pair_ptr[t]; q < L.pair_ptr[t + 1]; ++q) exec += gemm_flops(L.tile_mask[L.pair_a[q]], L.tile_mask[L.pair_b[q]]);
    const int K = L.tile_col[t];
    if (L.tile_row[t] != K) exec += gemm_flops(L.tile_mask[t], L.tile_mask[L.col_start[K]]);  // trsm
  }
  if (std::getenv("PER_COLUMN")) {
    for (int K = 0; K < L.nT; ++K) {
      double f = 0.0;
      int np = 0;
      for (int t = L.col_start[K]; t < L.col_start[K + 1]; ++t) {
        for (int q = L.pair_ptr[t]; q < L.pair_ptr[t + 1]; ++q, ++np) f += gemm_flops(L.tile_mask[L.pair_a[q]], L.tile_mask[L.pair_b[q]]);
        if (L.tile_row[t] != K) f += gemm_flops(L.tile_mask[t], L.tile_mask[L.col_start[K]]);
      }
      // operand bytes: full tiles vs only the 16-column panels both operands hold nonzeros in
      double full = 0, panel = 0;
      auto colmask = [&](int m) { int cm = 0; for (int q = 0; q < 4; ++q) for (int b = 0; b < 4; ++b) if ((m >> (b * 4 + q)) & 1) cm |= 1 << q; return cm; };
      for (int t = L.col_start[K]; t < L.col_start[K + 1]; ++t)
        for (int q = L.pair_ptr[t]; q < L.pair_ptr[t + 1]; ++q) {
          full += 65536;
          panel += 16384.0 * __builtin_popcount(colmask(L.tile_mask[L.pair_a[q]]) & colmask(L.tile_mask[L.pair_b[q]]));
        }
      std::printf("col %d tiles %d pairs %d exec_flops %.4e operand MB/patch full %.2f panels %.2f\n", K,
                  L.col_start[K + 1] - L.col_start[K], np, f, full / 1e6, panel / 1e6);
    }
  }
  std::printf("executed DMMA flops / patch %.4e (x%.2f of in-use), diagonal POTRF+inverse tiles %d\n", exec,
              exec / (2.0 * double(L.flops_ref)), L.nT);
  if (std::getenv("GROUP_STATS")) {  // nnz(L) and flops by separator group (CG layouts)
    const char* names[6] = {"interior", "plane0 facets", "plane1 facets", "plane2 facets", "edges", "vertex"};
    int64_t nnz[6] = {0}, fl[6] = {0}, cnt[6] = {0};
    for (int k = 0; k < L.n; ++k) {
      const int code = L.lat[k];
      int P[3] = {code & 255, (code >> 8) & 255, (code >> 16) & 255}, at = 0, ax = 0;
      for (int a = 0; a < dim; ++a)
        if (P[a] == pp) {
          ++at;
          ax = a;
        }
      const int gidx = at == 0 ? 0 : at == 1 ? 1 + ax : at == 2 ? 4 : 5;
      nnz[gidx] += L.colcount[k];
      fl[gidx] += int64_t(L.colcount[k]) * (L.colcount[k] - 1) / 2;
      ++cnt[gidx];
    }
    for (int g = 0; g < 6; ++g)
      std::printf("%-14s %7lld columns  nnz %12lld  madds %14lld\n", names[g], (long long)cnt[g], (long long)nnz[g],
                  (long long)fl[g]);
  }
  if (std::getenv("COMPACT_STATS")) {  // compact sub-blocks per tile (FDMGPU_COMPACT=1 layouts)
    std::vector<int> hist(65, 0);
    int tiles_with = 0, maxrow = 0;
    for (int t = 0; t < L.ntiles; ++t) {
      const uint8_t* hr = &L.tile_hdr[size_t(t) * fdmgpu::kHdrHost];
      const int nc = reinterpret_cast<const int32_t*>(hr + 128)[1];
      ++hist[nc];
      tiles_with += nc > 0;
      int rows[8] = {0};
      for (int q = L.tile_bptr[t]; q < L.tile_bptr[t + 1]; ++q)
        if (L.tile_ccol[q] != 0 || (q - L.tile_bptr[t]) >= reinterpret_cast<const int32_t*>(hr + 128)[0]) ++rows[L.tile_blk[q] >> 3];
      for (int r = 0; r < 8; ++r) maxrow = std::max(maxrow, rows[r]);
    }
    std::printf("tiles with compact blocks %d of %d; max per block-row %d; nc histogram:", tiles_with, L.ntiles, maxrow);
    for (int v = 1; v <= 64; ++v)
      if (hist[v]) std::printf(" %d:%d", v, hist[v]);
    std::printf("\n");
  }
  fdmhost_problem_destroy(pb);
  return 0;
}
