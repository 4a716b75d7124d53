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

}  // namespace meshperm::b200
