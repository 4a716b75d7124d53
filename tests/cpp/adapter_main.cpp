// TEST INFRASTRUCTURE (built by oracle/Makefile into oracle/_ref/adapter_test,
// run by tests/test_gpu_parity.py on a GPU): the reference's own code consumes
// the GPU path through include/meshperm_b200_adapter.hpp.  For each mesh the
// adapter's order() must equal the reference stages (compute_patches ->
// build_etree -> order_tree_nodes -> compute_perm), and the reference's
// elimination_fill / factor_etree_parents / cross_block_fill / write_etree
// must accept its outputs unchanged.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

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

static std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// run_pipeline: the reference's (pipeline.cpp:57-160) and the adapter's on
// the same RunConfig must agree on every output but the stage times, and the
// files they write must be byte-identical.
static void check_pipeline(b200::Context& ctx, RunConfig c, const std::string& tag, const std::string& scratch) {
  RunConfig ours = c;
  c.out_perm = scratch + "/ref_" + tag + ".perm";
  c.out_etree = scratch + "/ref_" + tag + ".etree";
  ours.out_perm = scratch + "/gpu_" + tag + ".perm";
  ours.out_etree = scratch + "/gpu_" + tag + ".etree";
  const PipelineResult want = run_pipeline(c);
  const PipelineResult got = b200::run_pipeline(ctx, ours);
  const BenchRow &a = want.row, &b = got.row;
  EXPECT(a.input == b.input && a.n == b.n && a.nnz_A == b.nnz_A && a.method == b.method);
  EXPECT(a.patch_size == b.patch_size && a.nd_level == b.nd_level);
  EXPECT(a.nnz_L == b.nnz_L && a.cost == b.cost && a.fill_ratio == b.fill_ratio);
  EXPECT(want.perm.perm == got.perm.perm && want.perm.inverse == got.perm.inverse);
  EXPECT(want.fill.column_counts == got.fill.column_counts);
  EXPECT(want.tree.node_count() == got.tree.node_count());
  for (index_t i = 0; i < want.tree.node_count() && i < got.tree.node_count(); ++i) {
    EXPECT(want.tree.nodes[i].vertices == got.tree.nodes[i].vertices);
    EXPECT(want.tree.nodes[i].local_perm == got.tree.nodes[i].local_perm);
  }
  EXPECT(slurp(c.out_perm) == slurp(ours.out_perm));
  EXPECT(slurp(c.out_etree) == slurp(ours.out_etree));
  if (failures) std::fprintf(stderr, "pipeline case %s failed\n", tag.c_str());
}

static void write_off(const TriangleMesh& m, const std::string& path) {
  std::ofstream out(path);
  out << "OFF\n" << m.vertex_count << ' ' << m.triangles.size() << " 0\n";
  for (index_t v = 0; v < m.vertex_count; ++v) out << v << " 0 0\n";
  for (const auto& t : m.triangles) out << "3 " << t[0] << ' ' << t[1] << ' ' << t[2] << '\n';
}

// lower triangle (with the diagonal) of a graph's pattern, MatrixMarket symmetric
static void write_mm(const AdjacencyGraph& g, const std::string& path) {
  std::vector<std::pair<index_t, index_t>> e;
  for (index_t u = 0; u < g.n; ++u) {
    e.push_back({u, u});
    for (auto j = g.offsets[u]; j < g.offsets[u + 1]; ++j)
      if (g.neighbors[j] < u) e.push_back({u, g.neighbors[j]});
  }
  std::ofstream out(path);
  out << "%%MatrixMarket matrix coordinate pattern symmetric\n" << g.n << ' ' << g.n << ' ' << e.size() << '\n';
  for (const auto& [r, c] : e) out << r + 1 << ' ' << c + 1 << '\n';
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

  // ---- run_pipeline / run_baselines (pipeline.hpp:71-76) through the adapter
  {
    RunConfig c;
    c.grid_rows = 64, c.grid_cols = 64;  // BASELINE configs[0]
    check_pipeline(ctx, c, "grid", scratch);
    c.block_size = 3, c.schedule = ScheduleKind::levelorder;  // expand_blocks on a mesh
    check_pipeline(ctx, c, "grid_b3", scratch);
  }
  {
    const std::string off = scratch + "/adapter_mesh.off";
    write_off(make_grid_mesh(37, 53), off);
    RunConfig c;
    c.mesh_path = off, c.patch_size = 64, c.nd_level = 4, c.local_mode = OrderMode::exact_md;
    check_pipeline(ctx, c, "off", scratch);
    // user patches: the reference's own compute_patches with two patches
    // merged into one disconnected id (enforce_connectivity splits it)
    const AdjacencyGraph g = mesh_to_graph(make_grid_mesh(37, 53));
    GroupMap gm = compute_patches(g, 64, 0).to_group_map();
    const std::string pf = scratch + "/adapter_patches.txt";
    {
      std::ofstream out(pf);
      for (index_t v = 0; v < g.n; ++v) {
        const index_t p = gm.assignment[v];
        out << (p == gm.patch_count - 1 ? 0 : p) << '\n';
      }
    }
    c.patch_file = pf, c.local_mode = OrderMode::approx_md;
    check_pipeline(ctx, c, "user", scratch);
  }
  {
    const std::string mm = scratch + "/adapter_matrix.mtx";
    write_mm(expand_graph(mesh_to_graph(make_grid_mesh(24, 31)), 2), mm);
    RunConfig c;
    c.matrix_path = mm, c.patch_size = 32;
    check_pipeline(ctx, c, "mtx", scratch);
    c.block_size = 2;  // compress_blocks ordering graph, fill on the row graph
    check_pipeline(ctx, c, "mtx_b2", scratch);
  }
  {
    RunConfig c;
    c.grid_rows = 40, c.grid_cols = 40, c.collect_timing = false;
    const std::vector<std::string> names{"natural", "md", "nd-vertex"};
    const auto want = run_baselines(c, names);
    const auto got = b200::run_baselines(ctx, c, names);
    EXPECT(want.size() == got.size());
    for (std::size_t i = 0; i < want.size() && i < got.size(); ++i) {
      EXPECT(want[i].method == got[i].method && want[i].nd_level == got[i].nd_level);
      EXPECT(want[i].nnz_L == got[i].nnz_L && want[i].cost == got[i].cost && want[i].nnz_A == got[i].nnz_A);
      EXPECT(got[i].t_patch_ms == 0.0 && got[i].t_local_ms == 0.0);
    }
    bool bad = false;
    try {
      RunConfig two;
      two.grid_rows = 8, two.grid_cols = 8, two.mesh_path = "x.off";
      b200::run_pipeline(ctx, two);
    } catch (const std::invalid_argument& e) {
      bad = std::string(e.what()) == "exactly one input source must be given";
    }
    EXPECT(bad);
  }
  if (failures) return 1;
  std::printf("adapter ok\n");
  return 0;
}
