// Row partition + halo plan for the distributed solve (SURVEY.md §8(e),
// configs[4]). Host-only C++ (no CUDA), exposed through the C ABI so the
// multi-rank protocol can be exercised on CPU (tests/test_dist_plan.py).
//
// A part owns a contiguous range of mesh nodes [n0, n1) — with the reference
// node numbering (i*(ny+1)+j)*(nz+1)+k (test_meshes.hpp:18) that is a slab of
// i-planes — i.e. the A-rows 3n0..3n1-1 and the V-rows of its conductor nodes.
// Ghost nodes are neighbours owned by other parts. Local vector layout per
// part (k right-hand sides interleaved):
//   [ A of owned nodes (3L) | A of ghost nodes (3G) | V owned (Vo) | V ghost (Vg) ]
// so the SpMV addresses A by local node id (3 l) and V by local V index
// (3(L+G) + v), and the owned rows are two contiguous segments.
#include "dist_plan.h"

#include <algorithm>
#include <stdexcept>

namespace ect {

HaloPlan build_halo_plan(int64_t n_nodes, const int* nbr_off, const int* nbr,
                         const int* cond_fwd, const int64_t* splits, int n_parts, int part) {
  if (part < 0 || part >= n_parts) throw std::invalid_argument("halo plan: bad part index");
  HaloPlan P;
  P.n_parts = n_parts;
  P.part = part;
  P.n0 = splits[part];
  P.n1 = splits[part + 1];
  if (!(0 <= P.n0 && P.n0 <= P.n1 && P.n1 <= n_nodes)) {
    throw std::invalid_argument("halo plan: splits must be non-decreasing within [0, n_nodes]");
  }
  P.L = P.n1 - P.n0;
  auto owner_of = [&](int64_t g) {
    // parts are contiguous node ranges: upper_bound on the split points
    return static_cast<int>(std::upper_bound(splits, splits + n_parts + 1, g) - splits) - 1;
  };
  // ghosts: neighbour nodes outside [n0, n1), sorted by global id
  std::vector<int> ghosts;
  for (int64_t i = P.n0; i < P.n1; ++i)
    for (int p = nbr_off[i]; p < nbr_off[i + 1]; ++p)
      if (nbr[p] < P.n0 || nbr[p] >= P.n1) ghosts.push_back(nbr[p]);
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  P.ghost_nodes = ghosts;
  P.G = static_cast<int64_t>(ghosts.size());
  // owned conductor V-dofs are the contiguous global range [c0, c1)
  P.c0 = -1;
  int64_t vo = 0;
  for (int64_t i = P.n0; i < P.n1; ++i)
    if (cond_fwd[i] >= 0) {
      if (P.c0 < 0) P.c0 = cond_fwd[i];
      ++vo;
    }
  if (P.c0 < 0) P.c0 = 0;
  P.Vo = vo;
  int64_t vg = 0;
  for (int g : ghosts) vg += cond_fwd[g] >= 0;
  P.Vg = vg;
  // local V index of every local node (owned then ghosts), -1 if not conductor
  P.local_vdof.assign(P.L + P.G, -1);
  for (int64_t i = P.n0; i < P.n1; ++i)
    if (cond_fwd[i] >= 0) P.local_vdof[i - P.n0] = static_cast<int>(cond_fwd[i] - P.c0);
  int64_t v = P.Vo;
  for (int64_t q = 0; q < P.G; ++q)
    if (cond_fwd[ghosts[q]] >= 0) P.local_vdof[P.L + q] = static_cast<int>(v++);
  // receive ranges per neighbour part (ghosts of one owner are contiguous)
  for (int64_t q = 0; q < P.G;) {
    const int owner = owner_of(ghosts[q]);
    int64_t e = q;
    int64_t vcount = 0;
    const int64_t vstart = P.local_vdof[P.L + q] >= 0 ? P.local_vdof[P.L + q] : -1;
    int64_t vfirst = -1;
    while (e < P.G && owner_of(ghosts[e]) == owner) {
      if (cond_fwd[ghosts[e]] >= 0) {
        if (vfirst < 0) vfirst = P.local_vdof[P.L + e];
        ++vcount;
      }
      ++e;
    }
    (void)vstart;
    HaloPeer peer;
    peer.part = owner;
    peer.recv_node_begin = q;        // ghost index
    peer.recv_node_count = e - q;
    peer.recv_v_begin = vfirst < 0 ? 0 : vfirst - P.Vo;  // index within V ghosts
    peer.recv_v_count = vcount;
    P.peers.push_back(peer);
    q = e;
  }
  // send lists: owned nodes that are neighbours of each other part's nodes.
  // Part q's ghosts from us are exactly our owned nodes adjacent to q's range;
  // with a symmetric neighbour relation these are the owned nodes having a
  // neighbour owned by q. Sorted by global id, as q's ghost numbering.
  for (auto& peer : P.peers) {
    const int q = peer.part;
    for (int64_t i = P.n0; i < P.n1; ++i) {
      bool need = false;
      for (int p = nbr_off[i]; p < nbr_off[i + 1] && !need; ++p)
        need = owner_of(nbr[p]) == q;
      if (need) {
        peer.send_nodes.push_back(static_cast<int>(i - P.n0));
        if (cond_fwd[i] >= 0) peer.send_cond_nodes.push_back(static_cast<int>(i - P.n0));
      }
    }
  }
  return P;
}

}  // namespace ect
