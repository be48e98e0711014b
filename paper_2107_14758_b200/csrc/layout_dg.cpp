// Shared symbolic analysis of the SIPG-DG vertex-star patches (host, once per
// handle).  A DG star is every DOF of the 2^d cells around the vertex,
// (2p+2)^d of them (dq_space DOFs are all cell-local, so
// star_dofs returns whole cells, src/discretization.cpp:266-297).  A patch
// position is (slot, l): the star cell's slot relative to the vertex (bit a
// set when the cell lies on the + side along axis a, the CG convention of
// layout.cpp) and the cell-local lattice index.  With the reference's
// patch_ordering (src/ordering.cpp:17-45) every interior star of a Cartesian
// mesh induces one elimination order on those positions up to the order of
// its facet groups; this file embeds every star in the first full star's
// order (absent cells of boundary stars -> identity rows), and runs the
// shared symbolic / tile analysis (symbolic_tiles) on the pattern of the
// transformed DG matrix (transformed_dg_poisson, src/sipg.cpp:252-364):
//   cell blocks      sum_a (A_t on a, B_t elsewhere)                (:262-270)
//   own facet block  (row tau full + column tau full on a) (x) B_t   (:47-87)
//   neighbour block  across the shared facet, same pattern rule      (:64-87)
// No interior elimination here: the factor keeps every position (n_I = 0).
#include <algorithm>
#include <functional>
#include <string>

#include "context.hpp"

namespace fdmgpu {

void symbolic_tiles(PatchLayout& L, const std::function<void(int, std::vector<int>&)>& neigh);

void analyze_dg_patches(Context& c, int npatch, const int32_t* vertex, const int64_t* ptr, const int32_t* dofs,
                        const int32_t* perm, const int32_t* star_cells) {
  const int d = c.dim, p = c.p, n1 = p + 1, ncorner = 1 << d, npc = c.npc;
  PatchLayout& L = c.L;
  L = PatchLayout();
  L.n = ncorner * npc;
  L.nI = 0;
  L.m = L.n;
  L.span = 0;
  if (L.n > 8192) throw Error(FDMGPU_UNSUPPORTED, "DG star of " + std::to_string(L.n) + " DOFs: at most 8192 supported");
  c.h_pdofs.assign(size_t(npatch) * L.n, -1);
  c.h_pcells.assign(size_t(npatch) * ncorner, -1);
  // owner cell and local lattice index of every DOF
  std::vector<int32_t> own_cell(c.ndof, -1), own_lat(c.ndof, -1);
  for (int K = 0; K < c.ncells; ++K)
    for (int l = 0; l < npc; ++l) {
      const int g = c.h_cell_dofs[size_t(K) * npc + l];
      if (own_cell[g] >= 0) throw Error(FDMGPU_INVALID_ARGUMENT, "SIPG: DG DOFs must be cell-local");
      own_cell[g] = K;
      own_lat[g] = l;
    }
  auto slot_of = [&](int j, int K) {
    const int v = vertex[j];
    for (int bits = 0; bits < ncorner; ++bits)
      if (c.h_cell_vertices[size_t(K) * ncorner + bits] == v) return (~bits) & (ncorner - 1);
    throw Error(FDMGPU_UNSUPPORTED, "star cell does not contain the patch vertex");
  };
  std::vector<int32_t> code;  // patch j's positions in its own elimination order
  auto map_patch = [&](int j) {
    const int64_t b = ptr[j], nj = ptr[j + 1] - ptr[j];
    if (nj < 1 || nj > L.n) throw Error(FDMGPU_UNSUPPORTED, "DG patch " + std::to_string(j) + " has too many DOFs");
    std::vector<int> slot_cell(ncorner, -1);
    for (int k = 0; k < ncorner; ++k) {
      const int K = star_cells[size_t(j) * ncorner + k];
      if (K < 0) continue;
      if (K >= c.ncells) throw Error(FDMGPU_INVALID_ARGUMENT, "patch star cell out of range");
      const int s = slot_of(j, K);
      if (slot_cell[s] >= 0) throw Error(FDMGPU_UNSUPPORTED, "star cells overlap a slot");
      slot_cell[s] = K;
    }
    for (int s = 0; s < ncorner; ++s) c.h_pcells[size_t(j) * ncorner + s] = slot_cell[s];
    code.assign(nj, -1);
    for (int64_t k = 0; k < nj; ++k) {
      const int g = dofs[b + perm[b + k]];
      if (g < 0 || g >= c.ndof) throw Error(FDMGPU_INVALID_ARGUMENT, "set_patches: DOF out of range");
      const int K = own_cell[g];
      int s = -1;
      for (int q = 0; q < ncorner; ++q)
        if (slot_cell[q] == K) s = q;
      if (s < 0) throw Error(FDMGPU_UNSUPPORTED, "DG patch DOF outside its star cells");
      code[k] = s * npc + own_lat[g];
    }
    return nj == L.n;
  };
  // canonical order: the first full star's (all full stars must share it)
  std::vector<int32_t> canon;
  for (int j = 0; j < npatch && canon.empty(); ++j)
    if (map_patch(j)) canon = code;
  if (canon.empty()) throw Error(FDMGPU_UNSUPPORTED, "SIPG patches: no full vertex star to take the order from");
  std::vector<int32_t> pos(L.n, -1);
  for (int k = 0; k < L.n; ++k) pos[canon[k]] = k;
  // Every star is embedded in the template by position.  patch_ordering sorts
  // the facet / edge / vertex groups by global entity id, and the outer
  // facets of a DG star (unlike a CG star's) carry patch DOFs, so stars next
  // to the boundary can order their groups differently; they are factored in
  // the template's order (the patch solution is order independent up to
  // rounding, as for the CG boundary stars in layout.cpp).
  L.ragged = 0;
  for (int j = 0; j < npatch; ++j) {
    const bool full = map_patch(j);
    if (!full) ++L.ragged;
    const int64_t b = ptr[j];
    for (size_t k = 0; k < code.size(); ++k) c.h_pdofs[size_t(j) * L.n + pos[code[k]]] = dofs[b + perm[b + k]];
  }
  L.lat = canon;
  L.pos_of_lat = pos;

  // structural neighbours of elimination position k in the transformed DG patch matrix
  std::vector<std::vector<int>> Apat(n1), Bpat(n1), all(n1);
  for (int i = 0; i < n1; ++i)
    for (int jj = 0; jj < n1; ++jj) {
      if (c.h_Anz[i + size_t(n1) * jj]) Apat[i].push_back(jj);
      if (c.h_Bnz[i + size_t(n1) * jj]) Bpat[i].push_back(jj);
      all[i].push_back(jj);
    }
  std::vector<int> mark(L.n, -1), one(1);
  int stamp = 0;
  auto neigh = [&](int k, std::vector<int>& out) {
    out.clear();
    ++stamp;
    const int s = canon[k] / npc, lk = canon[k] % npc;
    int l[3] = {0, 0, 0};
    for (int a = 0, t = lk; a < d; ++a, t /= n1) l[a] = t % n1;
    // candidates per axis; `ts` = target slot
    auto emit = [&](int ts, const std::vector<int>* cand[3]) {
      static const std::vector<int> zero{0};
      const std::vector<int>& c2 = d == 3 ? *cand[2] : zero;
      for (int x2 : c2)
        for (int x1 : *cand[1])
          for (int x0 : *cand[0]) {
            const int q = pos[ts * npc + x0 + n1 * (x1 + n1 * x2)];
            if (mark[q] != stamp) {
              mark[q] = stamp;
              out.push_back(q);
            }
          }
    };
    const std::vector<int>* cand[3];
    for (int a = 0; a < d; ++a) {
      // cell block, axis a carries A_t
      for (int b = 0; b < d; ++b) cand[b] = b == a ? &Apat[l[b]] : &Bpat[l[b]];
      emit(s, cand);
      // facet blocks on axis a: own cell (both facets) and the neighbour slot
      for (int side = 0; side < 2; ++side) {
        const int tau = side ? p : 0;
        for (int b = 0; b < d; ++b) cand[b] = &Bpat[l[b]];
        one[0] = tau;
        cand[a] = l[a] == tau ? &all[l[a]] : &one;
        emit(s, cand);
        // the neighbour across this facet is in the star when the facet holds the vertex
        const bool toward_vertex = ((s >> a) & 1) ? side == 0 : side == 1;
        if (toward_vertex) {
          const int ts = s ^ (1 << a);
          std::vector<int> tau_s(1, side ? 0 : p);
          cand[a] = l[a] == tau ? &all[l[a]] : &tau_s;
          emit(ts, cand);
        }
      }
    }
  };
  symbolic_tiles(L, neigh);
}

}  // namespace fdmgpu
