// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference meshperm core, compiled from the
// sources where they lie under /root/reference/proj/core (see oracle/Makefile).
// The resulting oracle/_ref/libmeshperm_ref.so is the "reference" oracle:
// tests/ use it to pin the C restatement (oracle/mp_oracle.c) and the CUDA
// path, and bench.py's reference arm / cpu_baseline leg time it on the GPU
// box's host cores.  Every entry point forwards to the reference stage
// function named in its comment; nothing here re-implements an algorithm.
#include <algorithm>
#include <bit>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "meshperm/assemble.hpp"
#include "meshperm/etree.hpp"
#include "meshperm/graph.hpp"
#include <fstream>
#include "meshperm/io.hpp"
#include "meshperm/local_order.hpp"
#include "meshperm/patching.hpp"
#include "meshperm/pipeline.hpp"
#include "meshperm/quotient.hpp"
#include "meshperm/symbolic.hpp"
#include "test_support.hpp"  // the reference test suite's generators (tests/)

using namespace meshperm;

namespace {
thread_local std::string g_err;

AdjacencyGraph make_graph(int32_t n, const int32_t* off, const int32_t* nbr) {
  AdjacencyGraph g;
  g.n = n;
  g.offsets.assign(off, off + n + 1);
  g.neighbors.assign(nbr, nbr + off[n]);
  return g;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = std::string("error: ") + e.what();
    return 2;
  }
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
      .count();
}

OrderMode mode_of(int m) {
  return m == 0 ? OrderMode::approx_md : m == 1 ? OrderMode::exact_md : OrderMode::natural;
}

void flatten_tree(const EliminationTree& tree, int32_t* node_offsets, int32_t* node_vertices,
                  int32_t* local_perm) {
  int32_t pos = 0;
  for (index_t i = 0; i < tree.node_count(); ++i) {
    node_offsets[i] = pos;
    const auto& nd = tree.nodes[i];
    for (std::size_t k = 0; k < nd.vertices.size(); ++k) {
      if (node_vertices) node_vertices[pos + k] = nd.vertices[k];
      if (local_perm) local_perm[pos + k] = k < nd.local_perm.size() ? nd.local_perm[k] : -1;
    }
    pos += static_cast<int32_t>(nd.vertices.size());
  }
  node_offsets[tree.node_count()] = pos;
}

EliminationTree unflatten_tree(int32_t n, int32_t nd_level, const int32_t* node_offsets,
                               const int32_t* node_vertices, const int32_t* local_perm) {
  EliminationTree tree;
  tree.n = n;
  tree.nd_level = nd_level;
  tree.nodes.resize((std::size_t{1} << (nd_level + 1)) - 1);
  for (std::size_t i = 0; i < tree.nodes.size(); ++i) {
    auto& nd = tree.nodes[i];
    nd.level = static_cast<index_t>(std::bit_width(static_cast<unsigned>(i + 1)) - 1);
    nd.vertices.assign(node_vertices + node_offsets[i], node_vertices + node_offsets[i + 1]);
    if (local_perm)
      nd.local_perm.assign(local_perm + node_offsets[i], local_perm + node_offsets[i + 1]);
  }
  return tree;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// graph.cpp:63-75 mesh_to_graph (validates, builds sorted dedup CSR).
// Two-call: pass nbr_out == nullptr to learn the neighbor count.
int ref_mesh_to_graph(int32_t nv, int64_t ntri, const int32_t* tris, int32_t* off_out,
                      int32_t* nbr_out, int64_t* nnz_out) {
  return guarded([&] {
    TriangleMesh mesh;
    mesh.vertex_count = nv;
    mesh.triangles.resize(ntri);
    for (int64_t t = 0; t < ntri; ++t)
      mesh.triangles[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    AdjacencyGraph g = mesh_to_graph(mesh);
    *nnz_out = static_cast<int64_t>(g.neighbors.size());
    if (off_out) std::memcpy(off_out, g.offsets.data(), sizeof(int32_t) * (nv + 1));
    if (nbr_out) std::memcpy(nbr_out, g.neighbors.data(), sizeof(int32_t) * g.neighbors.size());
  });
}

// graph.cpp:53-61 build_graph (block_size 1) / graph.cpp:77-94 compress_blocks
// (block_size > 1) of a SparsePattern{n, entries (rows[k], cols[k])}.
// Two-call like ref_mesh_to_graph; off_out holds n / block_size + 1 ints.
int ref_pattern_to_graph(int32_t n, int64_t nnz, const int32_t* rows, const int32_t* cols, int32_t block_size,
                         int32_t* off_out, int32_t* nbr_out, int64_t* nnz_out) {
  return guarded([&] {
    SparsePattern pattern;
    pattern.n = n;
    pattern.entries.resize(nnz);
    for (int64_t k = 0; k < nnz; ++k) pattern.entries[k] = {rows[k], cols[k]};
    AdjacencyGraph g = block_size == 1 ? build_graph(pattern) : compress_blocks(pattern, block_size);
    *nnz_out = static_cast<int64_t>(g.neighbors.size());
    if (off_out) std::memcpy(off_out, g.offsets.data(), sizeof(int32_t) * (g.n + 1));
    if (nbr_out) std::memcpy(nbr_out, g.neighbors.data(), sizeof(int32_t) * g.neighbors.size());
  });
}

// pipeline.cpp:38-55 make_grid_mesh.  tris_out holds 2*(r-1)*(c-1)*3 ints.
int ref_make_grid_mesh(int32_t rows, int32_t cols, int32_t* tris_out) {
  return guarded([&] {
    TriangleMesh m = make_grid_mesh(rows, cols);
    for (std::size_t t = 0; t < m.triangles.size(); ++t)
      for (int c = 0; c < 3; ++c) tris_out[3 * t + c] = m.triangles[t][c];
  });
}

// tests/test_support.hpp:66-86 mtest::random_mesh (the reference's own
// generator: std::mt19937_64 picks each cell's diagonal).
int ref_random_mesh(int32_t rows, int32_t cols, uint64_t seed, int32_t* tris_out) {
  return guarded([&] {
    TriangleMesh m = mtest::random_mesh(rows, cols, seed);
    for (std::size_t t = 0; t < m.triangles.size(); ++t)
      for (int c = 0; c < 3; ++c) tris_out[3 * t + c] = m.triangles[t][c];
  });
}

// etree.cpp:42-46
int32_t ref_default_nd_level(int32_t n) { return default_nd_level(n); }

// patching.cpp:295-345 compute_patches
int ref_compute_patches(int32_t n, const int32_t* off, const int32_t* nbr, int32_t target,
                        uint64_t seed, int32_t* assignment, int32_t* patch_count) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    PatchPartition p = compute_patches(g, target, seed);
    std::memcpy(assignment, p.assignment.data(), sizeof(int32_t) * n);
    *patch_count = p.patch_count;
  });
}

// patching.cpp:347-384 enforce_connectivity
int ref_enforce_connectivity(int32_t n, const int32_t* off, const int32_t* nbr,
                             const int32_t* assignment, int32_t patch_count, int32_t* out,
                             int32_t* out_count) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    PatchPartition p;
    p.assignment.assign(assignment, assignment + n);
    p.patch_count = patch_count;
    PatchPartition r = enforce_connectivity(p, g);
    std::memcpy(out, r.assignment.data(), sizeof(int32_t) * n);
    *out_count = r.patch_count;
  });
}

// quotient.cpp:47-80 build_quotient -> node weights + sorted positive edges.
// Two-call on the edge arrays (pass edge_p == nullptr to get the count).
int ref_build_quotient(int32_t n, const int32_t* off, const int32_t* nbr,
                       const int32_t* assignment, int32_t patch_count, int64_t* node_weight,
                       int32_t* edge_p, int32_t* edge_q, int64_t* edge_w, int64_t* n_edges) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    GroupMap gm{std::vector<index_t>(assignment, assignment + n), patch_count};
    QuotientGraph q = build_quotient(g, gm);
    auto edges = q.positive_edges();
    *n_edges = static_cast<int64_t>(edges.size());
    if (node_weight) std::memcpy(node_weight, q.node_weight.data(), sizeof(int64_t) * patch_count);
    if (edge_p)
      for (std::size_t i = 0; i < edges.size(); ++i) {
        edge_p[i] = std::get<0>(edges[i]);
        edge_q[i] = std::get<1>(edges[i]);
        edge_w[i] = std::get<2>(edges[i]);
      }
  });
}

// etree.cpp:86-147 build_etree (root quotient built inside, as in
// pipeline.cpp:118-125).  node_offsets has 2^(L+1) entries, node_vertices n.
int ref_build_etree(int32_t n, const int32_t* off, const int32_t* nbr, const int32_t* assignment,
                    int32_t patch_count, int32_t nd_level, uint64_t seed, int32_t* node_offsets,
                    int32_t* node_vertices) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    GroupMap gm{std::vector<index_t>(assignment, assignment + n), patch_count};
    EliminationTree t = build_etree(g, gm, nd_level, seed);
    flatten_tree(t, node_offsets, node_vertices, nullptr);
  });
}

// local_order.cpp:57-87 order_tree_nodes.  mode 0 approx, 1 exact, 2 natural.
int ref_order_tree_nodes(int32_t n, const int32_t* off, const int32_t* nbr, int32_t nd_level,
                         const int32_t* node_offsets, const int32_t* node_vertices, int32_t mode,
                         int32_t threads, int32_t* local_perm) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    EliminationTree t = unflatten_tree(n, nd_level, node_offsets, node_vertices, nullptr);
    order_tree_nodes(t, g, mode_of(mode), threads);
    std::vector<int32_t> tmp(t.node_count() + 1);
    flatten_tree(t, tmp.data(), nullptr, local_perm);
  });
}

// local_order.cpp:10-42 minimum_degree on a whole graph.
int ref_minimum_degree(int32_t n, const int32_t* off, const int32_t* nbr, int32_t mode,
                       int32_t* order) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    LocalPermutation lp = minimum_degree(g, mode_of(mode));
    std::memcpy(order, lp.order.data(), sizeof(int32_t) * n);
  });
}

// assemble.cpp:24-85 schedule_postorder|levelorder + compute_perm.
int ref_compute_perm(int32_t n, const int32_t* off, const int32_t* nbr, int32_t nd_level,
                     const int32_t* node_offsets, const int32_t* node_vertices,
                     const int32_t* local_perm, int32_t levelorder, int32_t* perm,
                     int32_t* inverse) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    EliminationTree t = unflatten_tree(n, nd_level, node_offsets, node_vertices, local_perm);
    Schedule s = levelorder ? schedule_levelorder(t) : schedule_postorder(t);
    Permutation p = compute_perm(t, g, s);
    std::memcpy(perm, p.perm.data(), sizeof(int32_t) * n);
    std::memcpy(inverse, p.inverse.data(), sizeof(int32_t) * n);
  });
}

// assemble.cpp:65-85 compute_perm with a caller schedule (any node sequence;
// invalid ones throw from validate_schedule).
int ref_compute_perm_schedule(int32_t n, const int32_t* off, const int32_t* nbr, int32_t nd_level,
                              const int32_t* node_offsets, const int32_t* node_vertices,
                              const int32_t* local_perm, const int32_t* sched, int64_t len, int32_t* perm,
                              int32_t* inverse) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    EliminationTree t = unflatten_tree(n, nd_level, node_offsets, node_vertices, local_perm);
    Schedule s(sched, sched + len);
    Permutation p = compute_perm(t, g, s);
    std::memcpy(perm, p.perm.data(), sizeof(int32_t) * n);
    std::memcpy(inverse, p.inverse.data(), sizeof(int32_t) * n);
  });
}

// assemble.cpp:48-63 validate_schedule: *bad = first violation or -1.
int ref_validate_schedule(int32_t nd_level, const int32_t* seq, int64_t len, int64_t* bad) {
  return guarded([&] {
    EliminationTree t;
    t.nd_level = nd_level;
    t.nodes.resize((std::size_t{1} << (nd_level + 1)) - 1);
    auto r = validate_schedule(t, std::span<const index_t>(seq, static_cast<std::size_t>(len)));
    *bad = r ? static_cast<int64_t>(*r) : -1;
  });
}

// symbolic.cpp:33-45 elimination_fill
int ref_elimination_fill(int32_t n, const int32_t* off, const int32_t* nbr, const int32_t* perm,
                         int64_t* column_counts, int64_t* nnz_A, int64_t* nnz_L, int64_t* cost,
                         double* fill_ratio) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    Permutation p = Permutation::from_order(std::vector<index_t>(perm, perm + n));
    FillReport r = elimination_fill(g, p);
    if (column_counts) std::memcpy(column_counts, r.column_counts.data(), sizeof(int64_t) * n);
    *nnz_A = r.nnz_A;
    *nnz_L = r.nnz_L;
    *cost = r.cost;
    *fill_ratio = r.fill_ratio;
  });
}

// symbolic.cpp:82-96 factor_etree_parents
int ref_factor_etree_parents(int32_t n, const int32_t* off, const int32_t* nbr,
                             const int32_t* perm, int32_t* parents) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    Permutation p = Permutation::from_order(std::vector<index_t>(perm, perm + n));
    auto par = factor_etree_parents(g, p);
    std::memcpy(parents, par.data(), sizeof(int32_t) * n);
  });
}

// symbolic.cpp:98-119 cross_block_fill
int ref_cross_block_fill(int32_t n, const int32_t* off, const int32_t* nbr, const int32_t* perm,
                         int32_t nd_level, const int32_t* node_offsets,
                         const int32_t* node_vertices, int64_t* crossing) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    Permutation p = Permutation::from_order(std::vector<index_t>(perm, perm + n));
    EliminationTree t = unflatten_tree(n, nd_level, node_offsets, node_vertices, nullptr);
    *crossing = cross_block_fill(g, p, t);
  });
}

// The ordering stages of run_pipeline (pipeline.cpp:100-138) on an in-memory
// graph, timed per stage exactly like time_stage (pipeline.cpp:16-21).
// stage_ms[0..4] = patch, quotient, etree, local, assemble.
int ref_order(int32_t n, const int32_t* off, const int32_t* nbr, int32_t patch_size,
              int32_t nd_level, uint64_t seed, int32_t mode, int32_t levelorder, int32_t threads,
              int32_t* assignment, int32_t* patch_count, int32_t* nd_level_out,
              int32_t* node_offsets, int32_t* node_vertices, int32_t* local_perm, int32_t* perm,
              int32_t* inverse, double* stage_ms) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    index_t L = nd_level >= 0 ? nd_level : default_nd_level(n);
    *nd_level_out = L;
    auto t0 = std::chrono::steady_clock::now();
    GroupMap gm = compute_patches(g, patch_size, seed).to_group_map();
    stage_ms[0] = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    QuotientGraph q = build_quotient(g, gm);
    stage_ms[1] = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    EliminationTree tree = build_etree(g, gm, std::move(q), L, seed);
    stage_ms[2] = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    order_tree_nodes(tree, g, mode_of(mode), threads < 1 ? 1 : threads);
    stage_ms[3] = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    Schedule s = levelorder ? schedule_levelorder(tree) : schedule_postorder(tree);
    Permutation p = compute_perm(tree, g, s);
    stage_ms[4] = ms_since(t0);
    if (assignment) std::memcpy(assignment, gm.assignment.data(), sizeof(int32_t) * n);
    *patch_count = gm.patch_count;
    if (node_offsets) flatten_tree(tree, node_offsets, node_vertices, local_perm);
    if (perm) std::memcpy(perm, p.perm.data(), sizeof(int32_t) * n);
    if (inverse) std::memcpy(inverse, p.inverse.data(), sizeof(int32_t) * n);
  });
}

// io.cpp:88-184 parse_off / parse_obj / parse_mesh.  format 0 by extension,
// 1 OFF, 2 OBJ; tris_out NULL = counts only.
int ref_parse_mesh(const char* path, int32_t format, int32_t* nv, int64_t* ntri, int32_t* tris_out) {
  return guarded([&] {
    TriangleMesh m = format == 1 ? parse_off(path) : format == 2 ? parse_obj(path) : parse_mesh(path);
    *nv = m.vertex_count;
    *ntri = static_cast<int64_t>(m.triangles.size());
    if (tris_out)
      for (std::size_t t = 0; t < m.triangles.size(); ++t)
        for (int k = 0; k < 3; ++k) tris_out[3 * t + k] = m.triangles[t][k];
  });
}

// io.cpp:186-240 parse_matrix_market (symmetrized pattern).
int ref_parse_matrix_market(const char* path, int32_t* n, int64_t* nnz, int32_t* rows, int32_t* cols) {
  return guarded([&] {
    SparsePattern p = parse_matrix_market(path);
    *n = p.n;
    *nnz = static_cast<int64_t>(p.entries.size());
    if (rows && cols)
      for (std::size_t k = 0; k < p.entries.size(); ++k) rows[k] = p.entries[k].first, cols[k] = p.entries[k].second;
  });
}

// io.cpp:242-262 read_patch_file.
int ref_read_patch_file(const char* path, int32_t n, int32_t* assignment, int32_t* patch_count) {
  return guarded([&] {
    GroupMap g = read_patch_file(path, n);
    std::copy(g.assignment.begin(), g.assignment.end(), assignment);
    *patch_count = g.patch_count;
  });
}

// io.cpp:264-268 write_permutation (inverse filled for completeness).
int ref_write_permutation(const char* path, int32_t n, const int32_t* perm) {
  return guarded([&] {
    Permutation p;
    p.perm.assign(perm, perm + n);
    p.inverse.assign(n, 0);
    for (int32_t k = 0; k < n; ++k)
      if (perm[k] >= 0 && perm[k] < n) p.inverse[perm[k]] = k;
    write_permutation(p, path);
  });
}

// io.cpp:270-281 read_permutation; perm NULL = count only.
int ref_read_permutation(const char* path, int32_t* n, int32_t* perm) {
  return guarded([&] {
    std::vector<index_t> p = read_permutation(path);
    *n = static_cast<int32_t>(p.size());
    if (perm) std::copy(p.begin(), p.end(), perm);
  });
}

// io.cpp:283-293 write_etree of a flattened tree.
int ref_write_etree(const char* path, int32_t n, int32_t nd_level, const int32_t* node_offsets,
                    const int32_t* node_vertices) {
  return guarded([&] {
    write_etree(unflatten_tree(n, nd_level, node_offsets, node_vertices, nullptr), path);
  });
}

// pipeline.cpp:193-205 write_csv of rows given field by field (strings as
// '\n'-free C strings; doubles as given).
int ref_write_csv(const char* path, int32_t count, const char* const* input, const char* const* method,
                  const int64_t* ints /* n, nnz_A, patch_size, nd_level, nnz_L, cost per row */,
                  const double* dbl /* t_patch .. t_assemble, fill_ratio per row */) {
  return guarded([&] {
    std::vector<BenchRow> rows(count);
    for (int32_t i = 0; i < count; ++i) {
      BenchRow& r = rows[i];
      r.input = input[i];
      r.method = method[i];
      r.n = ints[6 * i], r.nnz_A = ints[6 * i + 1];
      r.patch_size = static_cast<index_t>(ints[6 * i + 2]), r.nd_level = static_cast<index_t>(ints[6 * i + 3]);
      r.nnz_L = ints[6 * i + 4], r.cost = ints[6 * i + 5];
      r.t_patch_ms = dbl[6 * i], r.t_quotient_ms = dbl[6 * i + 1], r.t_etree_ms = dbl[6 * i + 2];
      r.t_local_ms = dbl[6 * i + 3], r.t_assemble_ms = dbl[6 * i + 4], r.fill_ratio = dbl[6 * i + 5];
    }
    std::ofstream out(path);
    write_csv(out, rows);
  });
}

// patching.cpp:386-433 validate_user_patches.  sizes / disconnected / unused
// hold patch_count entries each.
int ref_validate_user_patches(int32_t n, const int32_t* off, const int32_t* nbr, const int32_t* assignment,
                              int32_t assignment_len, int32_t patch_count, int64_t* sizes, int32_t* disconnected,
                              int32_t* n_disconnected, int32_t* unused, int32_t* n_unused) {
  return guarded([&] {
    AdjacencyGraph g = make_graph(n, off, nbr);
    GroupMap gm{std::vector<index_t>(assignment, assignment + assignment_len), patch_count};
    PatchReport r = validate_user_patches(gm, g);
    std::copy(r.patch_sizes.begin(), r.patch_sizes.end(), sizes);
    std::copy(r.disconnected_patches.begin(), r.disconnected_patches.end(), disconnected);
    std::copy(r.unused_patches.begin(), r.unused_patches.end(), unused);
    *n_disconnected = static_cast<int32_t>(r.disconnected_patches.size());
    *n_unused = static_cast<int32_t>(r.unused_patches.size());
  });
}

// pipeline.cpp:57-160 run_pipeline itself (mesh file, matrix file or grid;
// optional patch file and output files): perm (rows out), nnz_L, cost, the
// CSV method label.
int ref_run_pipeline(const char* mesh_path, const char* matrix_path, int32_t rows, int32_t cols,
                     const char* patch_file, int32_t patch_size, int32_t nd_level, uint64_t seed,
                     int32_t block_size, const char* out_perm, const char* out_etree, int32_t* perm_out,
                     int64_t* nnz_L, int64_t* cost, char* method_out /* 64 bytes */) {
  return guarded([&] {
    RunConfig c;
    if (mesh_path && *mesh_path) c.mesh_path = mesh_path;
    if (matrix_path && *matrix_path) c.matrix_path = matrix_path;
    c.grid_rows = rows, c.grid_cols = cols;
    if (patch_file && *patch_file) c.patch_file = patch_file;
    if (out_perm && *out_perm) c.out_perm = out_perm;
    if (out_etree && *out_etree) c.out_etree = out_etree;
    c.patch_size = patch_size, c.nd_level = nd_level, c.seed = seed, c.block_size = block_size;
    c.collect_timing = false;
    PipelineResult r = run_pipeline(c);
    std::copy(r.perm.perm.begin(), r.perm.perm.end(), perm_out);
    *nnz_L = r.row.nnz_L;
    *cost = r.row.cost;
    std::snprintf(method_out, 64, "%s", r.row.method.c_str());
  });
}

}  // extern "C"
