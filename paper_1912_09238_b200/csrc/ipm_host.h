// ipm_host.h — host-side mesh tables and domain decomposition of libipm (no CUDA).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ipm.h"

namespace ipm {

// Face tables of a mesh (global or a rank's local part).
//   nbr  [cells][F]: >= 0 neighbour cell (local index, or cells + halo slot), < 0 boundary -1-tag
//   nrm  [cells][F][2] outward unit normals (triangles; empty otherwise)
//   coef [cells][F]  |e| / |Omega_j|
//   area [cells], rgeo [cells] (triangles: perimeter / area), cx, cy [cells] centroids
struct MeshTables {
  int F = 0;
  int64_t cells = 0;
  std::vector<int32_t> nbr;
  std::vector<double> nrm, coef, area, rgeo, cx, cy;
  double inv_dx = 0.0, inv_dy = 0.0;
};

// Owned cells, halo cells and exchange lists of one rank.
//   local_gid  owned cells (ascending global id)
//   halo_gid   face neighbours owned by other ranks; grouped by peer (ascending rank),
//              ascending global id within a peer; halo slot h is node-state row cells + h
//   send_gid   per peer (same grouping), the owned cells adjacent to that peer, ascending gid:
//              rank r's send list to s equals rank s's halo list from r, element by element
struct Partition {
  std::vector<int64_t> local_gid, halo_gid, send_gid;
  std::vector<int32_t> send_local;
  std::vector<int32_t> peers, send_count, recv_count;
};

bool build_mesh(const ipm_config& C, MeshTables& M, std::string& err);
// cells in Morton order of their centroids (a processing order, not a renumbering)
void morton_order(const std::vector<double>& cx, const std::vector<double>& cy, std::vector<int32_t>& order);
bool build_partition(const ipm_config& C, const MeshTables& G, int rank, int nranks, Partition& P, std::string& err);
// local face tables of a partition (neighbours remapped to local / halo indices)
void local_tables(const MeshTables& G, const Partition& P, MeshTables& L);

}  // namespace ipm
