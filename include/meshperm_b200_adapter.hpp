// Header-only C++ adapter from the reference's meshperm types to the C ABI in
// meshperm_b200.h.  A maintainer compiles it with the
// reference's headers on the include path (-I proj/core/include); every
// existing caller of the reference (write_etree, cross_block_fill,
// elimination_fill, the acceptance checks) consumes its results unchanged.
// tests/cpp/adapter_main.cpp builds it against the reference core and checks
// exactly that.
#pragma once
#include <bit>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "meshperm/assemble.hpp"
#include "meshperm/etree.hpp"
#include "meshperm/graph.hpp"
#include "meshperm/local_order.hpp"
#include "meshperm/pipeline.hpp"
#include "meshperm/symbolic.hpp"
#include "meshperm/types.hpp"
#include "meshperm_b200.h"

namespace meshperm::b200 {

// MP_* codes back to the reference's exception types (pipeline.cpp:141-142,
// quotient.cpp:48-51, io.cpp:12-14).
inline void check(int rc) {
  if (rc == MP_OK) return;
  if (rc == MP_EINVAL) throw std::invalid_argument(mp_last_error());
  if (rc == MP_ELOGIC) throw std::logic_error(mp_last_error());
  throw std::runtime_error(mp_last_error());
}

class Context {
 public:
  explicit Context(int device = 0) { check(mp_context_create(&h_, device)); }
  ~Context() { mp_context_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  mp_context* get() const { return h_; }

 private:
  mp_context* h_ = nullptr;
};

struct Ordered {
  GroupMap patches;
  EliminationTree tree;
  Permutation perm;
  FillReport fill;
  std::vector<index_t> etree_parent;  // factor_etree_parents (symbolic.hpp:31)
};

// run_pipeline's ordering stages + elimination_fill (pipeline.cpp:100-146)
// for a mesh / pattern graph, on the GPU.
inline Ordered order(Context& ctx, const AdjacencyGraph& g, index_t patch_size = 256, index_t nd_level = -1,
                     std::uint64_t seed = 0, OrderMode mode = OrderMode::approx_md,
                     ScheduleKind schedule = ScheduleKind::postorder) {
  const index_t L = nd_level >= 0 ? nd_level : mp_default_nd_level(g.n);
  const std::size_t nn = (std::size_t{1} << (L + 1)) - 1;
  const std::size_t n = static_cast<std::size_t>(g.n);
  std::vector<int32_t> off(nn + 1), verts(n), lperm(n), perm(n), inv(n), parent(n);
  std::vector<int64_t> counts(n);
  Ordered o;
  o.patches.assignment.resize(n);
  mp_csr csr{g.n, g.offsets.data(), g.neighbors.data(), 0};
  const int32_t lm = mode == OrderMode::approx_md ? MP_LOCAL_APPROX
                     : mode == OrderMode::exact_md ? MP_LOCAL_EXACT : MP_LOCAL_NATURAL;
  const int32_t sc = schedule == ScheduleKind::postorder ? MP_SCHEDULE_POSTORDER : MP_SCHEDULE_LEVELORDER;
  mp_config cfg{patch_size, L, seed, lm, sc, 1, 1, nullptr, 0};
  mp_result r{};
  r.patch_of = o.patches.assignment.data();
  r.tree_node_offsets = off.data();
  r.tree_vertices = verts.data();
  r.tree_local_perm = lperm.data();
  r.perm = perm.data();
  r.inverse = inv.data();
  r.etree_parent = parent.data();
  r.column_counts = counts.data();
  check(mp_order(ctx.get(), &csr, &cfg, &r));
  o.patches.patch_count = r.patch_count;
  o.tree.n = g.n;
  o.tree.nd_level = L;
  o.tree.nodes.resize(nn);
  for (std::size_t i = 0; i < nn; ++i) {  // EtreeNode{vertices, local_perm, level}
    auto& nd = o.tree.nodes[i];
    nd.vertices.assign(verts.begin() + off[i], verts.begin() + off[i + 1]);
    nd.local_perm.assign(lperm.begin() + off[i], lperm.begin() + off[i + 1]);
    nd.level = static_cast<index_t>(std::bit_width(i + 1) - 1);
  }
  o.perm.perm = std::move(perm);
  o.perm.inverse = std::move(inv);
  o.fill.nnz_A = r.nnz_A;
  o.fill.nnz_L = r.nnz_L;
  o.fill.fill_ratio = r.fill_ratio;
  o.fill.column_counts = std::move(counts);
  o.fill.cost = r.cost;
  o.etree_parent = std::move(parent);
  return o;
}

namespace detail {

// A CSR graph returned by one of the device graph builds (host copy).
struct Csr {
  int32_t n = 0;
  std::vector<int32_t> off, nbr;
  mp_csr view() const { return mp_csr{n, off.data(), nbr.data(), 0}; }
  AdjacencyGraph graph() const {
    AdjacencyGraph g;
    g.n = n;
    g.offsets.assign(off.begin(), off.end());
    g.neighbors.assign(nbr.begin(), nbr.end());
    return g;
  }
};

inline Csr mesh_graph(Context& ctx, int32_t nv, const std::vector<int32_t>& tris) {
  Csr c;
  c.n = nv;
  c.off.resize(static_cast<std::size_t>(nv) + 1);
  const int64_t ntri = static_cast<int64_t>(tris.size() / 3);
  int64_t nnz = 0;
  check(mp_mesh_to_graph_device(ctx.get(), nv, ntri, tris.data(), 0, c.off.data(), nullptr, 0, &nnz));
  c.nbr.resize(static_cast<std::size_t>(nnz));
  check(mp_mesh_to_graph_device(ctx.get(), nv, ntri, tris.data(), 0, c.off.data(), c.nbr.data(), 0, &nnz));
  return c;
}

inline Csr pattern_graph(Context& ctx, int32_t n, const std::vector<int32_t>& rows, const std::vector<int32_t>& cols,
                         int32_t b) {
  Csr c;
  c.n = n / b;
  c.off.resize(static_cast<std::size_t>(c.n) + 1);
  const int64_t nnz_in = static_cast<int64_t>(rows.size());
  int64_t nnz = 0;
  check(mp_pattern_to_graph_device(ctx.get(), n, nnz_in, rows.data(), cols.data(), 0, b, c.off.data(), nullptr, 0,
                                   &nnz));
  c.nbr.resize(static_cast<std::size_t>(nnz));
  check(mp_pattern_to_graph_device(ctx.get(), n, nnz_in, rows.data(), cols.data(), 0, b, c.off.data(), c.nbr.data(),
                                   0, &nnz));
  return c;
}

inline std::string basename_of(const std::string& path) {  // pipeline.cpp:23-26
  const auto slash = path.find_last_of("/\\");
  return slash == std::string::npos ? path : path.substr(slash + 1);
}

}  // namespace detail

// run_pipeline (pipeline.hpp:71, pipeline.cpp:57-160) on the GPU: the same
// RunConfig checks and messages, the file / grid / MatrixMarket inputs read
// by the library's readers, the CSR built on the device, the patches (or the
// validated user patch file), ND tree, local orders, permutation (expanded
// for block_size > 1) and the fill from mp_order; for a blocked matrix the
// fill and the separation self-check run on the row graph with the expanded
// tree, as the reference does.  BenchRow stage times are device-timed (CUDA
// events).  Returns the reference's PipelineResult; writes out_perm /
// out_etree with the reference's formats.
inline PipelineResult run_pipeline(Context& ctx, const RunConfig& c) {
  int sources = !c.mesh_path.empty();
  sources += !c.matrix_path.empty();
  sources += c.grid_rows > 0 || c.grid_cols > 0;
  if (sources != 1) throw std::invalid_argument("exactly one input source must be given");
  const index_t b = c.block_size;
  if (b < 1) throw std::invalid_argument("block size must be positive");
  if (c.patch_size < 1) throw std::invalid_argument("patch size must be positive");

  // ordering graph (one node per block) and, for a blocked matrix, the row graph
  detail::Csr ord, meas;
  const bool blocked_matrix = !c.matrix_path.empty() && b > 1;
  if (!c.matrix_path.empty()) {
    int32_t n = 0;
    int64_t nnz = 0;
    check(mp_read_matrix_market(c.matrix_path.c_str(), &n, &nnz, nullptr, nullptr));
    std::vector<int32_t> rows(static_cast<std::size_t>(nnz)), cols(static_cast<std::size_t>(nnz));
    check(mp_read_matrix_market(c.matrix_path.c_str(), &n, &nnz, rows.data(), cols.data()));
    meas = detail::pattern_graph(ctx, n, rows, cols, 1);
    ord = blocked_matrix ? detail::pattern_graph(ctx, n, rows, cols, b) : meas;
  } else {
    int32_t nv = 0;
    std::vector<int32_t> tris;
    if (!c.mesh_path.empty()) {
      int64_t nt = 0;
      check(mp_read_mesh(c.mesh_path.c_str(), 0, &nv, &nt, nullptr));
      tris.resize(static_cast<std::size_t>(3 * nt));
      check(mp_read_mesh(c.mesh_path.c_str(), 0, &nv, &nt, tris.data()));
    } else {
      const int64_t nt = mp_grid_mesh_triangles(c.grid_rows, c.grid_cols);
      tris.resize(static_cast<std::size_t>(3 * std::max<int64_t>(nt, 0)));
      check(mp_make_grid_mesh(c.grid_rows, c.grid_cols, tris.data()));
      nv = c.grid_rows * c.grid_cols;
    }
    ord = detail::mesh_graph(ctx, nv, tris);
  }
  const index_t L = c.nd_level >= 0 ? c.nd_level : mp_default_nd_level(ord.n);
  std::vector<int32_t> user;
  int32_t user_count = 0;
  if (!c.patch_file.empty()) {
    user.resize(static_cast<std::size_t>(ord.n));
    check(mp_read_patch_file(c.patch_file.c_str(), ord.n, user.data(), &user_count));
  }

  const std::size_t nn = (std::size_t{1} << (L + 1)) - 1;
  const std::size_t N = static_cast<std::size_t>(ord.n) * static_cast<std::size_t>(b);
  std::vector<int32_t> off(nn + 1), verts(N), lperm(N), perm(N), inv(N), parent(N);
  std::vector<int64_t> counts(N);
  const int32_t lm = c.local_mode == OrderMode::approx_md ? MP_LOCAL_APPROX
                     : c.local_mode == OrderMode::exact_md ? MP_LOCAL_EXACT : MP_LOCAL_NATURAL;
  const int32_t sc = c.schedule == ScheduleKind::postorder ? MP_SCHEDULE_POSTORDER : MP_SCHEDULE_LEVELORDER;
  mp_config cfg{static_cast<int32_t>(c.patch_size), static_cast<int32_t>(L), c.seed, lm, sc,
                static_cast<int32_t>(b), blocked_matrix ? 0 : 1, user.empty() ? nullptr : user.data(), user_count,
                nullptr, 0};
  mp_result r{};
  r.tree_node_offsets = off.data();
  r.tree_vertices = verts.data();
  r.tree_local_perm = lperm.data();
  r.perm = perm.data();
  r.inverse = inv.data();
  if (!blocked_matrix) r.etree_parent = parent.data(), r.column_counts = counts.data();
  const mp_csr og = ord.view();
  check(mp_order(ctx.get(), &og, &cfg, &r));

  PipelineResult out;
  FillReport& fill = out.fill;
  count_t row_n = static_cast<count_t>(N);
  if (blocked_matrix) {
    // the expanded tree on the row graph: self-check, then the fill
    const mp_csr mg = meas.view();
    int64_t viol = 0;
    check(mp_tree_separation_check(ctx.get(), &mg, static_cast<int32_t>(L), off.data(), verts.data(), 0, &viol));
    if (viol != 0) throw std::logic_error("separator failed to disconnect its sides");
    check(mp_tree_fill(ctx.get(), &mg, static_cast<int32_t>(L), off.data(), verts.data(), lperm.data(), sc,
                       counts.data(), nullptr, 0, &fill.nnz_A, &fill.nnz_L, &fill.cost, &fill.fill_ratio));
    row_n = meas.n;
  } else {
    fill.nnz_A = r.nnz_A;
    fill.nnz_L = r.nnz_L;
    fill.cost = r.cost;
    fill.fill_ratio = r.fill_ratio;
  }
  fill.column_counts = std::move(counts);

  BenchRow& row = out.row;
  row.input = !c.input_id.empty()      ? c.input_id
              : !c.mesh_path.empty()   ? detail::basename_of(c.mesh_path)
              : !c.matrix_path.empty() ? detail::basename_of(c.matrix_path)
                                       : "grid-" + std::to_string(c.grid_rows) + "x" + std::to_string(c.grid_cols);
  row.n = row_n;
  row.nnz_A = fill.nnz_A;
  row.method = c.patch_file.empty() ? "ours-" + std::to_string(c.patch_size) : "user-patches";
  row.patch_size = c.patch_size;
  row.nd_level = L;
  if (c.collect_timing) {
    row.t_patch_ms = r.stage_ms[0];
    row.t_quotient_ms = r.stage_ms[1];
    row.t_etree_ms = r.stage_ms[2];
    row.t_local_ms = r.stage_ms[3];
    row.t_assemble_ms = r.stage_ms[4];
  }
  row.nnz_L = fill.nnz_L;
  row.fill_ratio = fill.fill_ratio;
  row.cost = fill.cost;

  if (!c.out_perm.empty()) check(mp_write_permutation(c.out_perm.c_str(), static_cast<int32_t>(N), perm.data()));
  if (!c.out_etree.empty())
    check(mp_write_etree(c.out_etree.c_str(), static_cast<int32_t>(L), off.data(), verts.data()));

  out.tree.n = static_cast<index_t>(N);
  out.tree.nd_level = L;
  out.tree.nodes.resize(nn);
  for (std::size_t i = 0; i < nn; ++i) {
    auto& nd = out.tree.nodes[i];
    nd.vertices.assign(verts.begin() + off[i], verts.begin() + off[i + 1]);
    nd.local_perm.assign(lperm.begin() + off[i], lperm.begin() + off[i + 1]);
    nd.level = static_cast<index_t>(std::bit_width(i + 1) - 1);
  }
  out.perm.perm = std::move(perm);
  out.perm.inverse = std::move(inv);
  return out;
}

// run_baselines (pipeline.hpp:75-76, pipeline.cpp:162-186): "natural",
// "md" and "nd-vertex" configurations of run_pipeline on the GPU.
inline std::vector<BenchRow> run_baselines(Context& ctx, const RunConfig& config,
                                           std::span<const std::string> names) {
  std::vector<BenchRow> rows;
  for (const std::string& name : names) {
    RunConfig base = config;
    base.out_perm.clear();
    base.out_etree.clear();
    base.patch_file.clear();
    if (name == "natural") {
      base.nd_level = 0;
      base.local_mode = OrderMode::natural;
    } else if (name == "md") {
      base.nd_level = 0;
      base.local_mode = OrderMode::approx_md;
    } else if (name == "nd-vertex") {
      base.patch_size = 1;
    } else {
      throw std::invalid_argument("unknown baseline: " + name);
    }
    BenchRow row = run_pipeline(ctx, base).row;
    row.method = name == "md" ? "md-only" : name;
    rows.push_back(std::move(row));
  }
  return rows;
}

}  // namespace meshperm::b200
