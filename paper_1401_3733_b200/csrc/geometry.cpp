// Decomposition checks and the even-odd face schedule (host logic).
//
// build_geometry restates the checks of proj/src/geometry.cpp:70-95 (even,
// divisible extents; optional 8x4x4x4 floor) and adds the even-odd layout's
// own requirement (even LOCAL extents, so every rank holds exactly half of
// each parity and global parity equals local parity).
//
// The face schedule replaces build_exchange_plan (proj/src/transport.cpp:
// 142-171): only decomposed directions exchange (the reference also packs
// self-faces, geometry.cpp:119-121), and each message carries half-spinor
// records for one parity only.
#include <string>

#include "lbcu_internal.hpp"

namespace lbcu {

int rep_dim(int rep, int n) {  // group.cpp:29-38
  if (n < 2) throw Error(LBCU_CONFIG_ERROR, "group rank must be >= 2, got " + std::to_string(n));
  switch (rep) {
    case LBCU_REP_FUNDAMENTAL: return n;
    case LBCU_REP_ADJOINT: return n * n - 1;
    case LBCU_REP_ANTISYMMETRIC: return n * (n - 1) / 2;
    case LBCU_REP_SYMMETRIC: return n * (n + 1) / 2;
  }
  throw Error(LBCU_CONFIG_ERROR, "unknown representation");
}

Geometry build_geometry(const int global[4], const int grid[4], int rank, bool enforce_floor) {
  Geometry g;
  g.nranks = 1;
  for (int d = 0; d < 4; ++d) {
    g.global[d] = global[d];
    g.grid[d] = grid[d];
    if (global[d] <= 0 || grid[d] <= 0)
      throw Error(LBCU_CONFIG_ERROR, "lattice extents and grid entries must be positive");
    if (global[d] % 2 != 0)
      throw Error(LBCU_CONFIG_ERROR, "lattice extent " + std::to_string(global[d]) + " is odd");
    if (global[d] % grid[d] != 0)
      throw Error(LBCU_CONFIG_ERROR, "extent " + std::to_string(global[d]) +
                                         " not divisible by grid " + std::to_string(grid[d]) +
                                         " in direction " + std::to_string(d));
    g.local[d] = global[d] / grid[d];
    g.nranks *= grid[d];
  }
  if (enforce_floor) {
    const int floor[4] = {8, 4, 4, 4};
    for (int d = 0; d < 4; ++d)
      if (g.local[d] < floor[d])
        throw Error(LBCU_CONFIG_ERROR, "local lattice " + std::to_string(g.local[0]) + "x" +
                                           std::to_string(g.local[1]) + "x" +
                                           std::to_string(g.local[2]) + "x" +
                                           std::to_string(g.local[3]) +
                                           " is below the 8x4x4x4 floor");
  }
  for (int d = 0; d < 4; ++d)
    if (g.local[d] % 2 != 0)
      throw Error(LBCU_CONFIG_ERROR, "even-odd layout needs even local extents, got " +
                                         std::to_string(g.local[d]) + " in direction " +
                                         std::to_string(d));
  if (rank < 0 || rank >= g.nranks) throw Error(LBCU_CONTRACT_VIOLATION, "rank outside worker grid");
  g.rank = rank;
  int r = rank;  // proc_coords, geometry.cpp:15-22 (row-major, z fastest)
  for (int d = 3; d >= 0; --d) {
    g.coords[d] = r % grid[d];
    r /= grid[d];
  }
  g.volume = static_cast<int64_t>(g.local[0]) * g.local[1] * g.local[2] * g.local[3];
  g.vh = g.volume / 2;
  g.stride = (g.vh + 63) / 64 * 64;
  for (int d = 0; d < 4; ++d) {
    g.decomposed[d] = grid[d] > 1;
    g.any_decomposed = g.any_decomposed || g.decomposed[d];
  }
  return g;
}

static int proc_rank(const int c[4], const int grid[4]) {
  return ((c[0] * grid[1] + c[1]) * grid[2] + c[2]) * grid[3] + c[3];
}

FacePlan plan_faces(const Geometry& geo) {
  FacePlan p;
  for (int mu = 0; mu < 4; ++mu)
    for (int dir = 0; dir < 2; ++dir) {
      const int f = 2 * mu + dir;
      if (!geo.decomposed[mu]) {
        p.partner[f] = -1;
        p.count[f] = 0;
        continue;
      }
      int nc[4] = {geo.coords[0], geo.coords[1], geo.coords[2], geo.coords[3]};
      nc[mu] = (nc[mu] + (dir ? 1 : -1) + geo.grid[mu]) % geo.grid[mu];
      p.partner[f] = proc_rank(nc, geo.grid);
      p.count[f] = geo.volume / geo.local[mu] / 2;
    }
  return p;
}

// Record j of face f: the site on the x_mu = edge slab whose in-face
// lexicographic position (other coordinates in t,x,y,z order) is 2j or 2j+1,
// whichever has the requested parity. Mirrors the device pack/unpack index
// (dslash.cu: face_record / face_index).
int64_t face_site(const Geometry& geo, int f, int input_parity, int64_t j) {
  const int mu = f / 2, dir = f % 2;
  const int edge = dir ? geo.local[mu] - 1 : 0;
  int others[3], k = 0;
  for (int d = 0; d < 4; ++d)
    if (d != mu) others[k++] = d;
  int c[4];
  int64_t fp = 2 * j;
  for (int q = 2; q >= 0; --q) {
    c[others[q]] = static_cast<int>(fp % geo.local[others[q]]);
    fp /= geo.local[others[q]];
  }
  c[mu] = edge;
  const int sum = c[0] + c[1] + c[2] + c[3];
  c[others[2]] += (sum + input_parity) & 1;
  return ((static_cast<int64_t>(c[0]) * geo.local[1] + c[1]) * geo.local[2] + c[2]) * geo.local[3] +
         c[3];
}

}  // namespace lbcu
