// ipm_mesh.cpp — host-side mesh face tables and the 2D domain decomposition:
//   1D:        contiguous slabs
//   cartesian: px x py blocks (rank r = ry px + rx)
//   triangles: Morton-ordered centroids cut into contiguous ranges
// The flux needs only face neighbours, so the halo is one layer of face neighbours; dual problems
// need no communication.
#include <algorithm>
#include <cmath>
#include <map>
#include <unordered_map>

#include "ipm_host.h"

namespace ipm {

static int64_t split(int64_t n, int parts, int r) { return (n * (int64_t)r) / parts; }

bool build_mesh(const ipm_config& C, MeshTables& M, std::string& err) {
  if (C.mesh_kind == IPM_MESH_1D) {
    if (C.nx < 1) return err = "nx >= 1", false;
    M.F = 2;
    M.cells = C.nx;
    const double dx = (C.x1 - C.x0) / C.nx;
    M.inv_dx = 1.0 / dx;
    M.nbr.resize(M.cells * 2);
    M.coef.assign(M.cells * 2, M.inv_dx);
    M.area.assign(M.cells, dx);
    M.cx.resize(M.cells);
    M.cy.assign(M.cells, 0.0);
    for (int64_t j = 0; j < M.cells; ++j) {
      M.nbr[j * 2 + 0] = j > 0 ? (int32_t)(j - 1) : (C.periodic ? (int32_t)(M.cells - 1) : -1);
      M.nbr[j * 2 + 1] = j < M.cells - 1 ? (int32_t)(j + 1) : (C.periodic ? 0 : -2);
      M.cx[j] = C.x0 + (j + 0.5) * dx;
    }
    return true;
  }
  if (C.mesh_kind == IPM_MESH_CART2D) {
    if (C.nx < 1 || C.ny < 1) return err = "nx, ny >= 1", false;
    M.F = 4;
    const int64_t nx = C.nx, ny = C.ny;
    M.cells = nx * ny;
    const double dx = (C.x1 - C.x0) / nx, dy = (C.y1 - C.y0) / ny;
    M.inv_dx = 1.0 / dx;
    M.inv_dy = 1.0 / dy;
    M.nbr.resize(M.cells * 4);
    M.coef.resize(M.cells * 4);
    M.area.assign(M.cells, dx * dy);
    M.cx.resize(M.cells);
    M.cy.resize(M.cells);
    for (int64_t iy = 0; iy < ny; ++iy)
      for (int64_t ix = 0; ix < nx; ++ix) {
        const int64_t j = iy * nx + ix;
        M.nbr[j * 4 + 0] = (int32_t)(ix > 0 ? j - 1 : (C.periodic ? iy * nx + nx - 1 : -1));
        M.nbr[j * 4 + 1] = (int32_t)(ix < nx - 1 ? j + 1 : (C.periodic ? iy * nx : -2));
        M.nbr[j * 4 + 2] = (int32_t)(iy > 0 ? j - nx : (C.periodic ? (ny - 1) * nx + ix : -3));
        M.nbr[j * 4 + 3] = (int32_t)(iy < ny - 1 ? j + nx : (C.periodic ? ix : -4));
        M.coef[j * 4 + 0] = M.coef[j * 4 + 1] = M.inv_dx;
        M.coef[j * 4 + 2] = M.coef[j * 4 + 3] = M.inv_dy;
        M.cx[j] = C.x0 + (ix + 0.5) * dx;
        M.cy[j] = C.y0 + (iy + 0.5) * dy;
      }
    return true;
  }
  if (C.mesh_kind == IPM_MESH_TRI) {
    if (C.n_tri < 1 || !C.h_vert || !C.h_tri || !C.h_tri_tag) return err = "triangle mesh arrays required", false;
    M.F = 3;
    M.cells = C.n_tri;
    const int64_t n = M.cells;
    M.nbr.assign(n * 3, 0);
    M.nrm.assign(n * 6, 0.0);
    M.coef.assign(n * 3, 0.0);
    M.area.assign(n, 0.0);
    M.rgeo.assign(n, 0.0);
    M.cx.assign(n, 0.0);
    M.cy.assign(n, 0.0);
    std::unordered_map<int64_t, int64_t> edge_owner;
    edge_owner.reserve((size_t)n * 3);
    for (int64_t t = 0; t < n; ++t)
      for (int e = 0; e < 3; ++e) {
        const int a = C.h_tri[t * 3 + e], b = C.h_tri[t * 3 + (e + 1) % 3];
        const int64_t key = (int64_t)std::min(a, b) * C.n_vert + std::max(a, b);
        const int tag = C.h_tri_tag[t * 3 + e];
        M.nbr[t * 3 + e] = -1 - (tag < 0 ? 0 : tag);
        auto it = edge_owner.find(key);
        if (it == edge_owner.end()) {
          edge_owner.emplace(key, t * 3 + e);
        } else {
          const int64_t o = it->second;
          M.nbr[t * 3 + e] = (int32_t)(o / 3);
          M.nbr[o] = (int32_t)t;
        }
      }
    for (int64_t t = 0; t < n; ++t) {
      const double* A = C.h_vert + 2 * C.h_tri[t * 3 + 0];
      const double* B = C.h_vert + 2 * C.h_tri[t * 3 + 1];
      const double* Cc = C.h_vert + 2 * C.h_tri[t * 3 + 2];
      const double ar = 0.5 * ((B[0] - A[0]) * (Cc[1] - A[1]) - (Cc[0] - A[0]) * (B[1] - A[1]));
      if (!(ar > 0.0)) return err = "triangles must be counter-clockwise with positive area", false;
      M.area[t] = ar;
      M.cx[t] = (A[0] + B[0] + Cc[0]) / 3.0;
      M.cy[t] = (A[1] + B[1] + Cc[1]) / 3.0;
      double per = 0.0;
      for (int e = 0; e < 3; ++e) {
        const double* V0 = C.h_vert + 2 * C.h_tri[t * 3 + e];
        const double* V1 = C.h_vert + 2 * C.h_tri[t * 3 + (e + 1) % 3];
        const double ex = V1[0] - V0[0], ey = V1[1] - V0[1];
        const double len = std::sqrt(ex * ex + ey * ey);
        M.nrm[(t * 3 + e) * 2 + 0] = ey / len;
        M.nrm[(t * 3 + e) * 2 + 1] = -ex / len;
        M.coef[t * 3 + e] = len / ar;
        per += len;
      }
      M.rgeo[t] = per / ar;
    }
    return true;
  }
  return err = "mesh_kind", false;
}

static uint64_t morton2(uint32_t x, uint32_t y) {
  auto spread = [](uint64_t v) {
    v &= 0xffffffffull;
    v = (v | (v << 16)) & 0x0000ffff0000ffffull;
    v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
    v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
  };
  return spread(x) | (spread(y) << 1);
}

// processing order of cells by the Morton code of their centroids (neighbours close in time: their node
// states are reused from L2 by the flux kernel)
void morton_order(const std::vector<double>& cx, const std::vector<double>& cy, std::vector<int32_t>& order) {
  const int64_t n = (int64_t)cx.size();
  order.resize(n);
  if (n == 0) return;
  double x0 = cx[0], x1 = cx[0], y0 = cy[0], y1 = cy[0];
  for (int64_t j = 0; j < n; ++j) {
    x0 = std::min(x0, cx[j]);
    x1 = std::max(x1, cx[j]);
    y0 = std::min(y0, cy[j]);
    y1 = std::max(y1, cy[j]);
  }
  std::vector<std::pair<uint64_t, int64_t>> key(n);
  for (int64_t j = 0; j < n; ++j) {
    const uint32_t qx = (uint32_t)std::lround((cx[j] - x0) / std::max(x1 - x0, 1e-300) * 65535.0);
    const uint32_t qy = (uint32_t)std::lround((cy[j] - y0) / std::max(y1 - y0, 1e-300) * 65535.0);
    key[j] = {morton2(qx, qy), j};
  }
  std::sort(key.begin(), key.end());
  for (int64_t s = 0; s < n; ++s) order[s] = (int32_t)key[s].second;
}

bool build_partition(const ipm_config& C, const MeshTables& G, int rank, int nranks, Partition& P,
                     std::string& err) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return err = "rank / nranks", false;
  const int64_t n = G.cells;
  std::vector<int32_t> owner(n, 0);
  if (C.mesh_kind == IPM_MESH_1D) {
    for (int r = 0; r < nranks; ++r)
      for (int64_t j = split(n, nranks, r); j < split(n, nranks, r + 1); ++j) owner[j] = r;
  } else if (C.mesh_kind == IPM_MESH_CART2D) {
    const int px = C.px > 0 ? C.px : nranks, py = C.py > 0 ? C.py : 1;
    if (px * py != nranks) return err = "px * py must equal nranks", false;
    for (int ry = 0; ry < py; ++ry)
      for (int rx = 0; rx < px; ++rx)
        for (int64_t iy = split(C.ny, py, ry); iy < split(C.ny, py, ry + 1); ++iy)
          for (int64_t ix = split(C.nx, px, rx); ix < split(C.nx, px, rx + 1); ++ix)
            owner[iy * C.nx + ix] = ry * px + rx;
  } else {
    double x0 = G.cx[0], x1 = G.cx[0], y0 = G.cy[0], y1 = G.cy[0];
    for (int64_t j = 0; j < n; ++j) {
      x0 = std::min(x0, G.cx[j]);
      x1 = std::max(x1, G.cx[j]);
      y0 = std::min(y0, G.cy[j]);
      y1 = std::max(y1, G.cy[j]);
    }
    std::vector<std::pair<uint64_t, int64_t>> key(n);
    for (int64_t j = 0; j < n; ++j) {
      const uint32_t qx = (uint32_t)std::lround((G.cx[j] - x0) / std::max(x1 - x0, 1e-300) * 65535.0);
      const uint32_t qy = (uint32_t)std::lround((G.cy[j] - y0) / std::max(y1 - y0, 1e-300) * 65535.0);
      key[j] = {morton2(qx, qy), j};
    }
    std::sort(key.begin(), key.end());
    for (int r = 0; r < nranks; ++r)
      for (int64_t s = split(n, nranks, r); s < split(n, nranks, r + 1); ++s) owner[key[s].second] = r;
  }
  P = Partition();
  for (int64_t j = 0; j < n; ++j)
    if (owner[j] == rank) P.local_gid.push_back(j);
  std::map<int, std::vector<int64_t>> halo, send;
  for (int64_t j : P.local_gid)
    for (int f = 0; f < G.F; ++f) {
      const int nb = G.nbr[j * G.F + f];
      if (nb < 0 || owner[nb] == rank) continue;
      halo[owner[nb]].push_back(nb);
      send[owner[nb]].push_back(j);
    }
  std::unordered_map<int64_t, int32_t> local_index;
  local_index.reserve(P.local_gid.size() * 2);
  for (size_t i = 0; i < P.local_gid.size(); ++i) local_index[P.local_gid[i]] = (int32_t)i;
  for (auto& kv : halo) {
    auto& h = kv.second;
    std::sort(h.begin(), h.end());
    h.erase(std::unique(h.begin(), h.end()), h.end());
    auto& s = send[kv.first];
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    P.peers.push_back(kv.first);
    P.recv_count.push_back((int32_t)h.size());
    P.send_count.push_back((int32_t)s.size());
    P.halo_gid.insert(P.halo_gid.end(), h.begin(), h.end());
    P.send_gid.insert(P.send_gid.end(), s.begin(), s.end());
  }
  for (int64_t g : P.send_gid) P.send_local.push_back(local_index[g]);
  return true;
}

void local_tables(const MeshTables& G, const Partition& P, MeshTables& L) {
  const int F = G.F;
  const int64_t n = (int64_t)P.local_gid.size();
  std::unordered_map<int64_t, int32_t> slot;
  slot.reserve((P.local_gid.size() + P.halo_gid.size()) * 2);
  for (int64_t i = 0; i < n; ++i) slot[P.local_gid[i]] = (int32_t)i;
  for (size_t h = 0; h < P.halo_gid.size(); ++h) slot[P.halo_gid[h]] = (int32_t)(n + (int64_t)h);
  L = MeshTables();
  L.F = F;
  L.cells = n;
  L.inv_dx = G.inv_dx;
  L.inv_dy = G.inv_dy;
  L.nbr.resize(n * F);
  L.coef.resize(n * F);
  L.area.resize(n);
  L.cx.resize(n);
  L.cy.resize(n);
  if (!G.nrm.empty()) L.nrm.resize(n * F * 2);
  if (!G.rgeo.empty()) L.rgeo.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t g = P.local_gid[i];
    for (int f = 0; f < F; ++f) {
      const int nb = G.nbr[g * F + f];
      L.nbr[i * F + f] = nb < 0 ? nb : slot.at(nb);
      L.coef[i * F + f] = G.coef[g * F + f];
      if (!G.nrm.empty()) {
        L.nrm[(i * F + f) * 2] = G.nrm[(g * F + f) * 2];
        L.nrm[(i * F + f) * 2 + 1] = G.nrm[(g * F + f) * 2 + 1];
      }
    }
    L.area[i] = G.area[g];
    L.cx[i] = G.cx[g];
    L.cy[i] = G.cy[g];
    if (!G.rgeo.empty()) L.rgeo[i] = G.rgeo[g];
  }
}

}  // namespace ipm
