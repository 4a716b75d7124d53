// Synthetic mesh generators and the host CSR builder (C ABI).
//
// Vertex numbering defines every tie-break downstream, so each generator
// fixes it explicitly:
//   grid      : make_grid_mesh semantics (reference pipeline.cpp:38-55)
//   random    : random_mesh(rows, cols, seed) semantics, std::mt19937_64
//               diagonal flips (reference tests/test_support.hpp:66-86)
//   torus     : R x C wraparound grid, cells split like make_grid_mesh
//   icosphere : frequency-f geodesic sphere, numbering of SURVEY.md App. C
// The CSR builder restates graph_from_edges / mesh_to_graph
// (reference graph.cpp:14-75): sorted, deduplicated, symmetric, no loops.
// CSR construction sits before the timed path.
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "mp_internal.h"

namespace {

int64_t grid_tris(int32_t rows, int32_t cols) { return 2LL * (rows - 1) * (cols - 1); }

}  // namespace

extern "C" {

int64_t mp_grid_mesh_triangles(int32_t rows, int32_t cols) {
  return rows < 2 || cols < 2 ? 0 : grid_tris(rows, cols);
}

// pipeline.cpp:38-55: cell (r,c) -> (a,b,d), (b,e,d) with a=r*C+c, b=a+1, d=a+C, e=d+1.
int mp_make_grid_mesh(int32_t rows, int32_t cols, int32_t* tris) {
  if (rows < 2 || cols < 2) return mp::set_error(MP_EINVAL, "grid needs at least two rows and columns");
  int64_t t = 0;
  for (int32_t r = 0; r + 1 < rows; ++r)
    for (int32_t c = 0; c + 1 < cols; ++c) {
      int32_t a = r * cols + c, b = a + 1, d = a + cols, e = d + 1;
      int32_t* o = tris + 6 * t;
      o[0] = a, o[1] = b, o[2] = d, o[3] = b, o[4] = e, o[5] = d;
      ++t;
    }
  return MP_OK;
}

// tests/test_support.hpp:66-86: one mt19937_64 draw per cell, low bit picks the diagonal.
int mp_make_random_mesh(int32_t rows, int32_t cols, uint64_t seed, int32_t* tris) {
  if (rows < 2 || cols < 2) return mp::set_error(MP_EINVAL, "grid needs at least two rows and columns");
  std::mt19937_64 rng(seed);
  int64_t t = 0;
  for (int32_t r = 0; r + 1 < rows; ++r)
    for (int32_t c = 0; c + 1 < cols; ++c) {
      int32_t a = r * cols + c, b = a + 1, d = a + cols, e = d + 1;
      int32_t* o = tris + 6 * t;
      if (rng() & 1) {
        o[0] = a, o[1] = b, o[2] = d, o[3] = b, o[4] = e, o[5] = d;
      } else {
        o[0] = a, o[1] = b, o[2] = e, o[3] = a, o[4] = e, o[5] = d;
      }
      ++t;
    }
  return MP_OK;
}

int64_t mp_torus_mesh_triangles(int32_t rows, int32_t cols) {
  return rows < 3 || cols < 3 ? 0 : 2LL * rows * cols;
}

// Wraparound grid: id = r*C + c; every cell split like make_grid_mesh, indices mod R / mod C.
int mp_make_torus_mesh(int32_t rows, int32_t cols, int32_t* tris) {
  if (rows < 3 || cols < 3) return mp::set_error(MP_EINVAL, "torus needs at least three rows and columns");
  int64_t t = 0;
  for (int32_t r = 0; r < rows; ++r)
    for (int32_t c = 0; c < cols; ++c) {
      int32_t r1 = (r + 1) % rows, c1 = (c + 1) % cols;
      int32_t a = r * cols + c, b = r * cols + c1, d = r1 * cols + c, e = r1 * cols + c1;
      int32_t* o = tris + 6 * t;
      o[0] = a, o[1] = b, o[2] = d, o[3] = b, o[4] = e, o[5] = d;
      ++t;
    }
  return MP_OK;
}

int64_t mp_icosphere_vertices(int32_t f) { return f < 1 ? 0 : 10LL * f * f + 2; }
int64_t mp_icosphere_triangles(int32_t f) { return f < 1 ? 0 : 20LL * f * f; }

// Frequency-f geodesic icosphere (SURVEY.md Appendix C numbering):
// corners 0..11; edge-interior points 12 + e*(f-1) + (s-1), s steps from the
// smaller corner of the e-th (min,max)-sorted edge; face-interior points
// consecutive from 12+30(f-1), face-major, then i, then j.
int mp_make_icosphere_mesh(int32_t f, int32_t* tris) {
  if (f < 1) return mp::set_error(MP_EINVAL, "icosphere frequency must be positive");
  static const int kFaces[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                    {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                    {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                    {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
  std::vector<std::pair<int, int>> edges;
  for (auto& fc : kFaces)
    for (int k = 0; k < 3; ++k) {
      int a = fc[k], b = fc[(k + 1) % 3];
      edges.emplace_back(std::min(a, b), std::max(a, b));
    }
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  if (edges.size() != 30) return mp::set_error(MP_EINVAL, "icosahedron edge table broken");
  auto edge_point = [&](int a, int b, int steps_from_a) -> int32_t {
    if (steps_from_a == 0) return a;
    if (steps_from_a == f) return b;
    int lo = std::min(a, b), hi = std::max(a, b);
    int e = static_cast<int>(std::lower_bound(edges.begin(), edges.end(), std::make_pair(lo, hi)) -
                             edges.begin());
    int s = (a == lo) ? steps_from_a : f - steps_from_a;
    return 12 + e * (f - 1) + (s - 1);
  };
  int32_t next_face_id = 12 + 30 * (f - 1);
  std::vector<int32_t> G(static_cast<size_t>(f + 1) * (f + 1), -1);
  auto at = [&](int i, int j) -> int32_t& { return G[static_cast<size_t>(i) * (f + 1) + j]; };
  int64_t t = 0;
  for (auto& fc : kFaces) {
    int a = fc[0], b = fc[1], c = fc[2];
    for (int i = 0; i <= f; ++i)
      for (int j = 0; i + j <= f; ++j) {
        if (j == 0) at(i, j) = edge_point(a, b, i);
        else if (i == 0) at(i, j) = edge_point(a, c, j);
        else if (i + j == f) at(i, j) = edge_point(c, b, i);
        else at(i, j) = next_face_id++;
      }
    for (int i = 0; i < f; ++i)
      for (int j = 0; i + j < f; ++j) {
        int32_t* o = tris + 3 * t++;
        o[0] = at(i, j), o[1] = at(i + 1, j), o[2] = at(i, j + 1);
        if (i + j + 1 < f) {
          o = tris + 3 * t++;
          o[0] = at(i + 1, j), o[1] = at(i + 1, j + 1), o[2] = at(i, j + 1);
        }
      }
  }
  if (next_face_id != mp_icosphere_vertices(f) || t != mp_icosphere_triangles(f))
    return mp::set_error(MP_EINVAL, "icosphere numbering broken");
  return MP_OK;
}

// graph.cpp:14-75 restated: validate, count, scatter, per-list sort + dedup.
// Two-call: nbr == nullptr only computes off[] and *nnz.
int mp_mesh_to_graph(int32_t nv, int64_t ntri, const int32_t* tris, int32_t* off, int32_t* nbr,
                     int64_t* nnz) {
  for (int64_t t = 0; t < ntri; ++t) {
    const int32_t* c = tris + 3 * t;
    for (int k = 0; k < 3; ++k)
      if (c[k] < 0 || c[k] >= nv)
        return mp::set_error(MP_EINVAL, "triangle " + std::to_string(t) + " references vertex " +
                                            std::to_string(c[k]) + " outside [0, " +
                                            std::to_string(nv) + ")");
    if (c[0] == c[1] || c[1] == c[2] || c[0] == c[2])
      return mp::set_error(MP_EINVAL, "triangle " + std::to_string(t) + " has repeated corners");
  }
  std::vector<int64_t> start(static_cast<size_t>(nv) + 1, 0);
  for (int64_t t = 0; t < 3 * ntri; ++t) start[tris[t] + 1] += 2;
  for (int32_t v = 0; v < nv; ++v) start[v + 1] += start[v];
  std::vector<int32_t> raw(static_cast<size_t>(start[nv]));
  std::vector<int64_t> cur(start.begin(), start.end() - 1);
  static const int kPairs[3][2] = {{0, 1}, {1, 2}, {0, 2}};
  for (int64_t t = 0; t < ntri; ++t) {
    const int32_t* c = tris + 3 * t;
    for (auto& pr : kPairs) {
      int32_t u = c[pr[0]], w = c[pr[1]];
      raw[cur[u]++] = w;
      raw[cur[w]++] = u;
    }
  }
  int64_t write = 0;
  for (int32_t v = 0; v < nv; ++v) {
    auto b = raw.begin() + start[v], e = raw.begin() + start[v + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    off[v] = static_cast<int32_t>(write);
    if (nbr) std::copy(b, u, nbr + write);
    write += u - b;
  }
  off[nv] = static_cast<int32_t>(write);
  *nnz = write;
  return MP_OK;
}

}  // extern "C"
