// TEST INFRASTRUCTURE (built by oracle/Makefile into oracle/_ref/adapter_test,
// run by tests/test_gpu_parity.py on a GPU): the reference's own code consumes
// the GPU path through include/meshperm_b200_adapter.hpp.  For each mesh the
// adapter's order() must equal the reference stages (compute_patches ->
// build_etree -> order_tree_nodes -> compute_perm), and the reference's
// elimination_fill / factor_etree_parents / cross_block_fill / write_etree
// must accept its outputs unchanged.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "meshperm/io.hpp"
#include "meshperm/patching.hpp"
#include "meshperm/pipeline.hpp"
#include "meshperm_b200_adapter.hpp"

using namespace meshperm;

static int failures = 0;
#define EXPECT(cond)                                                  \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static void check_mesh(b200::Context& ctx, const TriangleMesh& mesh, index_t patch, index_t L, OrderMode mode,
                       ScheduleKind sched, const std::string& etree_path) {
  const AdjacencyGraph g = mesh_to_graph(mesh);
  const b200::Ordered o = b200::order(ctx, g, patch, L, 0, mode, sched);
  // the reference stages on the same input
  const index_t lv = L >= 0 ? L : default_nd_level(g.n);
  GroupMap gm = compute_patches(g, patch, 0).to_group_map();
  EXPECT(gm.patch_count == o.patches.patch_count && gm.assignment == o.patches.assignment);
  EliminationTree t = build_etree(g, gm, lv, 0);
  order_tree_nodes(t, g, mode, 1);
  EXPECT(t.node_count() == o.tree.node_count());
  for (index_t i = 0; i < t.node_count() && i < o.tree.node_count(); ++i) {
    EXPECT(t.nodes[i].vertices == o.tree.nodes[i].vertices);
    EXPECT(t.nodes[i].local_perm == o.tree.nodes[i].local_perm);
    EXPECT(t.nodes[i].level == o.tree.nodes[i].level);
  }
  const Schedule s = sched == ScheduleKind::postorder ? schedule_postorder(t) : schedule_levelorder(t);
  const Permutation p = compute_perm(t, g, s);
  EXPECT(p.perm == o.perm.perm && p.inverse == o.perm.inverse);
  // reference consumers of the GPU outputs
  const FillReport f = elimination_fill(g, o.perm);
  EXPECT(f.nnz_L == o.fill.nnz_L && f.cost == o.fill.cost && f.nnz_A == o.fill.nnz_A);
  EXPECT(f.column_counts == o.fill.column_counts);
  EXPECT(factor_etree_parents(g, o.perm) == o.etree_parent);
  EXPECT(cross_block_fill(g, o.perm, o.tree) == 0);
  write_etree(o.tree, etree_path);
}

int main(int argc, char** argv) {
  const std::string scratch = argc > 1 ? argv[1] : "/tmp";
  b200::Context ctx(0);
  check_mesh(ctx, make_grid_mesh(64, 64), 256, -1, OrderMode::approx_md, ScheduleKind::postorder,
             scratch + "/adapter_etree_1.txt");
  check_mesh(ctx, make_grid_mesh(150, 211), 64, 5, OrderMode::approx_md, ScheduleKind::levelorder,
             scratch + "/adapter_etree_2.txt");
  check_mesh(ctx, make_grid_mesh(40, 33), 16, 3, OrderMode::exact_md, ScheduleKind::postorder,
             scratch + "/adapter_etree_3.txt");
  // error mapping: the reference's exception types
  bool threw = false;
  try {
    b200::order(ctx, mesh_to_graph(make_grid_mesh(8, 8)), 4, 30);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  if (failures) return 1;
  std::printf("adapter ok\n");
  return 0;
}
