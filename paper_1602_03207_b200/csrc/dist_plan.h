// Row partition + halo plan for the distributed solve (see dist_plan.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace ect {

struct HaloPeer {
  int part = -1;
  // receive side: ghost nodes [recv_node_begin, +count) in ghost numbering, and
  // their conductor V-dofs [recv_v_begin, +count) within the V-ghost block
  int64_t recv_node_begin = 0, recv_node_count = 0;
  int64_t recv_v_begin = 0, recv_v_count = 0;
  // send side: owned local node ids the peer needs (ascending global id), and
  // the conductor subset (their V values follow the A values in the message)
  std::vector<int> send_nodes;
  std::vector<int> send_cond_nodes;
};

struct HaloPlan {
  int n_parts = 1, part = 0;
  int64_t n0 = 0, n1 = 0;  // owned node range
  int64_t L = 0, G = 0;    // owned / ghost node counts
  int64_t c0 = 0;          // global V-dof of the first owned conductor node
  int64_t Vo = 0, Vg = 0;  // owned / ghost V-dof counts
  std::vector<int> ghost_nodes;   // global ids, ascending
  std::vector<int> local_vdof;    // local node -> local V index (or -1)
  std::vector<HaloPeer> peers;    // ascending part id
  int64_t local_nodes() const { return L + G; }
  int64_t na_local() const { return 3 * (L + G); }
  int64_t n_local() const { return 3 * (L + G) + Vo + Vg; }
};

HaloPlan build_halo_plan(int64_t n_nodes, const int* nbr_off, const int* nbr,
                         const int* cond_fwd, const int64_t* splits, int n_parts, int part);

}  // namespace ect
