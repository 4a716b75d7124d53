/* meshperm_b200 — B200-native patch-based nested-dissection permutation.
 *
 * The C ABI the reference's symbolic-analysis callers bind to.  The
 * reference (meshperm, /root/reference/proj) exposes free C++ functions in
 * namespace meshperm; each entry point below names the reference interface
 * it replaces (core/include/meshperm/<file>:<line>).  Plain pointers and
 * sizes only: no C++ or torch types cross this boundary.
 *
 * Conventions (reference types.hpp:10-11): vertex/patch ids are int32,
 * counts and weights int64.  A CSR graph (graph.hpp:10-24) has
 * offsets[n+1] and neighbors[offsets[n]] with sorted, duplicate-free,
 * symmetric lists and no self loops.
 *
 * Memory: every array argument is either host memory or device memory of
 * the context's GPU, selected per call by the `on_device` flag of the struct
 * it belongs to (mp_csr.on_device for inputs, mp_result.on_device for
 * outputs).  Host arrays are staged through pinned buffers owned by the
 * context.  Outputs are caller-allocated; sizes follow from n and nd_level.
 *
 * Errors: every function returns MP_OK (0) or an MP_E* code; the message of
 * the last failure on the calling thread is mp_last_error().  Contract
 * violations the reference reports with std::invalid_argument return
 * MP_EINVAL with the same message text.
 *
 * Threading: a context is used by one host thread at a time; independent
 * contexts (one per GPU, or several per GPU) run concurrently.  Results are
 * independent of the stream, the context and the GPU count.
 */
#ifndef MESHPERM_B200_H
#define MESHPERM_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MP_OK = 0,
  MP_EINVAL = 1,  /* std::invalid_argument in the reference */
  MP_ECUDA = 2,   /* CUDA runtime / launch failure */
  MP_ENOMEM = 3,  /* device or pinned allocation failed */
  MP_ELOGIC = 4,  /* std::logic_error in the reference (self-check) */
  MP_EIO = 5      /* std::runtime_error from the reference's file I/O (io.cpp) */
};

enum { MP_LOCAL_APPROX = 0, MP_LOCAL_EXACT = 1, MP_LOCAL_NATURAL = 2 }; /* local_order.hpp:10 OrderMode */
enum { MP_SCHEDULE_POSTORDER = 0, MP_SCHEDULE_LEVELORDER = 1 };          /* pipeline.hpp:15 ScheduleKind */

typedef struct mp_context mp_context;

typedef struct {
  int32_t n;
  const int32_t* offsets;   /* n + 1 */
  const int32_t* neighbors; /* offsets[n] */
  int32_t on_device;        /* 1: both arrays live on the context's GPU */
} mp_csr;

/* RunConfig (pipeline.hpp:17-37), the fields the ordering path reads. */
typedef struct {
  int32_t patch_size;   /* 256 */
  int32_t nd_level;     /* -1: default_nd_level(n) */
  uint64_t seed;        /* 0 */
  int32_t local_mode;   /* MP_LOCAL_* (approx_md) */
  int32_t schedule;     /* MP_SCHEDULE_* (postorder) */
  int32_t block_size;   /* 1; >1 expands perm/tree by b (assemble.hpp:43) */
  int32_t want_fill;    /* 1: factor etree + column counts + nnz(L) (symbolic.hpp:23-31) */
  /* RunConfig.patch_file path (pipeline.cpp:101-111): NULL = compute_patches;
   * else a user GroupMap (n ids in [0, user_patch_count), host or device as
   * the csr) that is validated and, if a patch is disconnected, split by
   * enforce_connectivity before the ND tree. */
  const int32_t* user_patches;
  int32_t user_patch_count;
  /* compute_perm(tree, g, schedule) with an arbitrary node sequence
   * (assemble.hpp:37): NULL = the `schedule` enum; else schedule_len host
   * ints, validated like validate_schedule (MP_EINVAL "invalid schedule at
   * position N", assemble.cpp:71-72). */
  const int32_t* schedule_nodes;
  int64_t schedule_len;
} mp_config;

/* PipelineResult (pipeline.hpp:56-61) flattened.  Array pointers may be
 * NULL when not wanted.  Sizes: nn = 2^(nd_level+1) - 1 tree nodes,
 * N = block_size * n rows. */
typedef struct {
  int32_t on_device;           /* 1: array outputs are device pointers */
  int32_t* patch_of;           /* n      GroupMap.assignment */
  int32_t* tree_node_offsets;  /* nn+1   EliminationTree node i holds   */
  int32_t* tree_vertices;      /* N        tree_vertices[off[i]..off[i+1]) */
  int32_t* tree_local_perm;    /* N      EtreeNode.local_perm, same layout */
  int32_t* perm;               /* N      Permutation.perm (new -> old) */
  int32_t* inverse;            /* N      Permutation.inverse */
  int32_t* etree_parent;       /* N      factor_etree_parents (positions) */
  int64_t* column_counts;      /* N      FillReport.column_counts */
  /* scalars, always written to host */
  int32_t patch_count;
  int32_t nd_level;
  int64_t nnz_A, nnz_L, cost;
  double fill_ratio;
  /* device-timed stage times (CUDA events), ms:
     0 patch, 1 quotient, 2 etree, 3 local, 4 assemble, 5 symbolic */
  float stage_ms[6];
  int64_t kernel_launches;     /* kernels launched by this call */
  /* device time (CUDA events) of the dominant kernels, ms, summed over launches:
     0 farthest-point seeds, 1 Lloyd rounds, 2 FM bipartition, 3 separator
     refinement, 4 minimum degree, 5 symbolic game */
  float kernel_ms[6];
  /* work counters of this call: 0 FPS adjacency scans (R_fps), 1 FM moves,
     2 refine moves, 3 Lloyd BFS levels, 4 FPS batches, 5 FPS grid-mode BFS
     levels, 6 FPS candidates evaluated, 7 FPS worker-region BFS levels,
     8..15 FPS phase timers (ns, CTA 0: grid-mode, regions, walk+commit,
     refresh, candidate selection) */
  int64_t work[16];
} mp_result;

const char* mp_last_error(void);
const char* mp_version(void);

/* Context: owns the device workspace (grown on demand, reused across calls),
 * pinned staging buffers, a stream and the timing events. */
int mp_context_create(mp_context** ctx, int32_t device);
void mp_context_destroy(mp_context* ctx);
/* Number of contexts the caller runs concurrently on this device (default 1):
 * the persistent grid-wide kernels (farthest-point seeding, Lloyd rounds)
 * size their grids to 1/share of the SMs so that concurrent contexts overlap
 * instead of queueing behind each other's whole-GPU launches.  Results do not
 * depend on it. */
int mp_context_set_sm_share(mp_context* ctx, int32_t share);
/* How mp_order / mp_tree_fill compute column counts, parents and nnz(L):
 * 0 (default) the factor's elimination tree + Gilbert-Ng-Peyton column counts
 * split by the ND tree; 1 the elimination game of symbolic.cpp:33-45 played
 * node by node.  Both give identical outputs; 1 is kept as a cross-check.
 * cross_block_fill, elimination_fill of an arbitrary permutation and trees
 * whose separators leak always use the game. */
int mp_context_set_fill_algorithm(mp_context* ctx, int32_t algo);
/* Internal tuning / fallback selection of one context (defaults: 0 = the
 * library's own choice).  Results never depend on these; they exist so that
 * tests can force the fallback paths and so that the sizing can be studied.
 *   MP_TUNE_FPS_CLUSTER      farthest-point cluster phase: 8 or 16 CTAs, -1 off
 *   MP_TUNE_FPS_QCAP         cluster-phase queue slots (small: forces overflow)
 *   MP_TUNE_FPS_GRID_RADIUS  cluster / grid mode while the radius exceeds it
 *   MP_TUNE_FPS_GRID_CANDS   grid-mode candidates per batch
 *   MP_TUNE_FPS_SUB_REGION   largest region of the four-group worker mode
 *   MP_TUNE_LLOYD_BLOCKS     CTAs of the Lloyd kernel
 *   MP_TUNE_LLOYD_CLUSTER_N  meshes up to this many vertices run Lloyd on one
 *                            thread-block cluster (default 12288; -1 never)
 *   MP_TUNE_MD_THREADS       threads of the shared-memory minimum-degree CTAs
 * MP_EINVAL for an unknown key. */
enum {
  MP_TUNE_FPS_CLUSTER = 0,
  MP_TUNE_FPS_QCAP = 1,
  MP_TUNE_FPS_GRID_RADIUS = 2,
  MP_TUNE_FPS_GRID_CANDS = 3,
  MP_TUNE_FPS_SUB_REGION = 4,
  MP_TUNE_LLOYD_BLOCKS = 5,
  MP_TUNE_LLOYD_CLUSTER_N = 6,
  MP_TUNE_MD_THREADS = 7,
  MP_TUNE_COUNT = 8
};
int mp_context_set_tuning(mp_context* ctx, int32_t key, int64_t value);
/* cudaStream_t to run on; NULL restores the context's own stream. */
int mp_context_set_stream(mp_context* ctx, void* stream);

/* ---- whole path: run_pipeline's ordering stages (pipeline.cpp:100-140) ---- */
int mp_order(mp_context* ctx, const mp_csr* g, const mp_config* cfg, mp_result* out);
/* Batch of independent graphs (C4): frame f is
 * mp_order(ctx, &graphs[f], &cfgs[f], &results[f]) on one of the nctx contexts
 * (one host thread each, all on their own streams, sm_share = nctx for the
 * call).  status[f] (optional) gets each frame's code; the return value is the
 * code of the lowest failing frame, its message prefixed "frame f: ".  The
 * contexts must be distinct (MP_EINVAL otherwise): a context is never used by
 * two host threads at once. */
int mp_order_batch(mp_context* const* ctxs, int32_t nctx, int32_t count, const mp_csr* graphs,
                   const mp_config* cfgs, mp_result* results, int32_t* status);

/* ---- multi-GPU: one very large mesh sharded over ranks (C3) ----
 * One process (or host thread) per GPU, each with its own context, calls
 * mp_order_sharded with the same graph and config.  Every rank computes the
 * patches and the top k = ceil(log2 world) ND levels (sequential chains:
 * replicated, not shipped); the level-k subtrees are then dealt to ranks by
 * size (largest first, least-loaded rank), each rank splits and orders (MD)
 * its own subtrees only, and two all-gathers exchange (1) node sizes and
 * (2) the owned nodes' vertex lists + local orders.  The fill (etree +
 * column counts, a few percent of the path) then runs on every rank over the
 * assembled tree.  With mp_context_set_fill_algorithm(ctx, 1) each rank plays
 * the elimination game on its own subtrees and a third all-gather exchanges
 * the subtree roots' live elements and the owned column counts / parents.
 * Every rank returns the complete, rank-count-independent mp_result --
 * bit-identical to mp_order.
 *
 * The all-gather is the caller's or the library's NCCL one: recv receives
 * world * bytes, rank r's contribution at r * bytes.  device_buffers = 1:
 * send / recv are device memory of the context's GPU and the collective is
 * enqueued on `stream` (NCCL); 0: host memory (e.g. an MPI or gloo
 * all-gather), stream unused. */
typedef struct {
  int32_t rank, world;
  int32_t device_buffers;
  int (*allgather)(void* user, const void* send, void* recv, int64_t bytes, void* stream);
  void* user;
} mp_comm;

int mp_order_sharded(mp_context* ctx, const mp_csr* g, const mp_config* cfg, const mp_comm* comm, mp_result* out);

/* NCCL plumbing for mp_comm (libnccl.so.2 is loaded on first use, so the
 * library has no link-time NCCL dependency).  Rank 0 creates the unique id
 * and ships its 128 bytes to the other ranks out of band; every rank then
 * creates its communicator on its GPU.  mp_nccl_comm_init fills comm with
 * the library's ncclAllGather (device_buffers = 1). */
int mp_nccl_get_unique_id(uint8_t id[128]);
int mp_nccl_comm_init(mp_comm* comm, const uint8_t id[128], int32_t world, int32_t rank, int32_t device);
void mp_nccl_comm_destroy(mp_comm* comm);

/* ---- stage entry points (reference free functions) ---- */
/* etree.hpp:35-36 default_nd_level */
int32_t mp_default_nd_level(int32_t n);

/* patching.hpp:26-27 compute_patches(g, target_size, seed).to_group_map() */
int mp_compute_patches(mp_context* ctx, const mp_csr* g, int32_t target_size, uint64_t seed,
                       int32_t* assignment, int32_t on_device, int32_t* patch_count);

/* patching.hpp:31-32 enforce_connectivity(partition, g) */
int mp_enforce_connectivity(mp_context* ctx, const mp_csr* g, const int32_t* assignment,
                            int32_t patch_count, int32_t* out, int32_t on_device,
                            int32_t* out_count);
/* patching.hpp:44-45 validate_user_patches: PatchReport of a user
 * assignment (on_device as the csr).  patch_sizes (patch_count int64),
 * disconnected / unused (patch_count ints each, ascending ids) may be NULL;
 * the counts are always written.  MP_EINVAL "patch id P out of range at
 * vertex v" for the first bad vertex, as the reference throws. */
int mp_validate_user_patches(mp_context* ctx, const mp_csr* g, const int32_t* assignment, int32_t patch_count,
                             int64_t* patch_sizes, int32_t* disconnected, int32_t* n_disconnected,
                             int32_t* unused, int32_t* n_unused);

/* quotient.hpp:41 build_quotient + QuotientGraph::positive_edges (quotient.hpp:36).
 * Two-call: edge arrays NULL returns only *n_edges. Host outputs. */
int mp_build_quotient(mp_context* ctx, const mp_csr* g, const int32_t* assignment,
                      int32_t patch_count, int64_t* node_weight, int32_t* edge_p,
                      int32_t* edge_q, int64_t* edge_w, int64_t* n_edges);

/* etree.hpp:52-53 build_etree(g, gmap, nd_level, seed).  Host or device
 * outputs per on_device; assignment follows g->on_device. */
int mp_build_etree(mp_context* ctx, const mp_csr* g, const int32_t* assignment,
                   int32_t patch_count, int32_t nd_level, uint64_t seed,
                   int32_t* node_offsets, int32_t* node_vertices, int32_t on_device);

/* local_order.hpp:36 order_tree_nodes(tree, g, mode) -> local_perm per node */
int mp_order_tree_nodes(mp_context* ctx, const mp_csr* g, int32_t nd_level,
                        const int32_t* node_offsets, const int32_t* node_vertices,
                        int32_t mode, int32_t* local_perm, int32_t on_device);

/* Sharded local orderings: order_tree_nodes for the nodes
 * with node_mask[i] != 0 only, then compute_perm's scatter for those nodes:
 * local_perm and perm entries of masked nodes are written, all others are
 * left untouched (another rank owns them).  local_order.hpp:36 +
 * assemble.hpp:25-38 restricted to a node subset.  node_mask has nn entries. */
int mp_order_subtrees(mp_context* ctx, const mp_csr* g, int32_t nd_level, const int32_t* node_offsets,
                      const int32_t* node_vertices, int32_t mode, int32_t schedule, const uint8_t* node_mask,
                      int32_t* local_perm, int32_t* perm, int32_t on_device);

/* assemble.hpp:25-38 schedule_* + compute_perm */
int mp_compute_perm(mp_context* ctx, int32_t n, int32_t nd_level, const int32_t* node_offsets,
                    const int32_t* node_vertices, const int32_t* local_perm, int32_t schedule,
                    int32_t* perm, int32_t* inverse, int32_t on_device);

/* assemble.hpp:35 validate_schedule: *first_violation = the first position
 * that lists a node out of range, twice, or before one of its children (a
 * short sequence reports `length`), or -1 when the sequence is valid. */
int mp_validate_schedule(int32_t nd_level, const int32_t* sequence, int64_t length, int64_t* first_violation);
/* assemble.hpp:37 compute_perm(tree, g, schedule) with any valid node
 * sequence (schedule_nodes: schedule_len host ints). */
int mp_compute_perm_schedule(mp_context* ctx, int32_t n, int32_t nd_level, const int32_t* node_offsets,
                             const int32_t* node_vertices, const int32_t* local_perm, const int32_t* schedule_nodes,
                             int64_t schedule_len, int32_t* perm, int32_t* inverse, int32_t on_device);

/* symbolic.hpp:23 elimination_fill + :31 factor_etree_parents for a
 * permutation produced from an ND tree (perm = compute_perm(tree, ...)):
 * the factor's elimination tree built subtree by subtree (Liu's algorithm,
 * one CTA per tree node and level) and Gilbert-Ng-Peyton column counts.  A
 * tree whose separators do not separate (edges between unrelated nodes) is
 * handled as an arbitrary permutation (mp_elimination_fill). */
int mp_tree_fill(mp_context* ctx, const mp_csr* g, int32_t nd_level, const int32_t* node_offsets,
                 const int32_t* node_vertices, const int32_t* local_perm, int32_t schedule,
                 int64_t* column_counts, int32_t* etree_parent, int32_t on_device,
                 int64_t* nnz_A, int64_t* nnz_L, int64_t* cost, double* fill_ratio);
/* The same for compute_perm(tree, g, schedule) with any valid node sequence. */
int mp_tree_fill_schedule(mp_context* ctx, const mp_csr* g, int32_t nd_level, const int32_t* node_offsets,
                          const int32_t* node_vertices, const int32_t* local_perm, const int32_t* schedule_nodes,
                          int64_t schedule_len, int64_t* column_counts, int32_t* etree_parent, int32_t on_device,
                          int64_t* nnz_A, int64_t* nnz_L, int64_t* cost, double* fill_ratio);

/* symbolic.hpp:23 elimination_fill + :31 factor_etree_parents for ANY
 * permutation perm[n] (new position -> old index; host or device per
 * on_device): the same etree + column-count computation on a one-node tree
 * (the etree is then one CTA's serial pass; the ND-structured mp_tree_fill
 * splits it over tree nodes).  With fill algorithm 1 the elimination game.
 * MP_EINVAL "permutation is not a bijection" as symbolic.cpp:16-18. */
int mp_elimination_fill(mp_context* ctx, const mp_csr* g, const int32_t* perm, int64_t* column_counts,
                        int32_t* etree_parent, int32_t on_device, int64_t* nnz_A, int64_t* nnz_L, int64_t* cost,
                        double* fill_ratio);
/* symbolic.hpp:37 cross_block_fill(g, perm, tree): the number of factor
 * entries joining vertices whose tree nodes are neither equal nor ancestor-
 * related, for any permutation and tree (the exact value; the pipeline's
 * self-check only needs zero / non-zero, see mp_tree_separation_check). */
int mp_cross_block_fill(mp_context* ctx, const mp_csr* g, const int32_t* perm, int32_t nd_level,
                        const int32_t* node_offsets, const int32_t* node_vertices, int32_t on_device,
                        int64_t* crossing);

/* ---- synthetic inputs and host CSR build (outside the timed path) ---- */
int64_t mp_grid_mesh_triangles(int32_t rows, int32_t cols);
int mp_make_grid_mesh(int32_t rows, int32_t cols, int32_t* tris);          /* pipeline.hpp:65 */
int mp_make_random_mesh(int32_t rows, int32_t cols, uint64_t seed, int32_t* tris);
int64_t mp_torus_mesh_triangles(int32_t rows, int32_t cols);
int mp_make_torus_mesh(int32_t rows, int32_t cols, int32_t* tris);
int64_t mp_icosphere_vertices(int32_t f);
int64_t mp_icosphere_triangles(int32_t f);
int mp_make_icosphere_mesh(int32_t f, int32_t* tris);
/* the pipeline's separation self-check (pipeline.cpp:141-142;
 * cross_block_fill, symbolic.hpp:37) in edge-locality form: *violations =
 * number of edges whose endpoints lie in tree nodes that are neither equal
 * nor ancestor-related (tests/etree_test.cpp:171-179).  Zero implies
 * cross_block_fill == 0 for the postorder and levelorder schedules.  The
 * tree arrays are host or device memory per on_device; g per g->on_device.
 * mp_order runs this check after its timed stages and fails with MP_ELOGIC
 * ("separator failed to disconnect its sides") like run_pipeline. */
int mp_tree_separation_check(mp_context* ctx, const mp_csr* g, int32_t nd_level,
                             const int32_t* node_offsets, const int32_t* node_vertices,
                             int32_t on_device, int64_t* violations);
/* graph.hpp:51 mesh_to_graph on the device (graph.cpp:14-75,
 * validate_mesh types.cpp:20-33).  tris (3 * ntri corners) in host or device
 * memory per tris_on_device; off (nv + 1) and nbr (capacity >= nnz = 2|E|;
 * NULL = offsets and *nnz only) in host or device memory per out_on_device.
 * MP_EINVAL with the reference's message for a bad triangle. */
int mp_mesh_to_graph_device(mp_context* ctx, int32_t nv, int64_t ntri, const int32_t* tris,
                            int32_t tris_on_device, int32_t* off, int32_t* nbr, int32_t out_on_device,
                            int64_t* nnz);
/* the matrix input path on the device.  A SparsePattern
 * {n, entries (rows[k], cols[k])} becomes the ordering graph: build_graph
 * (graph.hpp:48, graph.cpp:53-61) for block_size 1, compress_blocks
 * (graph.hpp:59, graph.cpp:77-94) for block_size > 1 (n / block_size nodes,
 * an edge between blocks joined by any entry).  Array placement and the
 * nbr == NULL count-only call as in mp_mesh_to_graph_device; MP_EINVAL with
 * the reference's messages ("pattern entry out of range", "matrix size N is
 * not a multiple of block size B", "block size must be positive"). */
int mp_pattern_to_graph_device(mp_context* ctx, int32_t n, int64_t nnz, const int32_t* rows,
                               const int32_t* cols, int32_t in_on_device, int32_t block_size,
                               int32_t* off, int32_t* nbr, int32_t out_on_device, int64_t* nnz_out);
/* graph.hpp:62 lift_patches: out[v * b + t] = assignment[v] (n * b entries). */
int mp_lift_patches(mp_context* ctx, int32_t n, const int32_t* assignment, int32_t block_size,
                    int32_t* out, int32_t on_device);
/* graph.hpp:56 mesh_to_graph on the host (input generation); nbr NULL = count only */
int mp_mesh_to_graph(int32_t nv, int64_t ntri, const int32_t* tris, int32_t* off, int32_t* nbr,
                     int64_t* nnz);

/* ---- On-disk formats (io.hpp / io.cpp): host-only text I/O.
 * Accepted syntax, error texts ("path:line: msg") and written bytes follow the
 * reference; its std::runtime_error becomes MP_EIO, validate_mesh's
 * std::invalid_argument stays MP_EINVAL.  Two-call convention: a NULL output
 * array returns only the counts. */
/* io.cpp:178 parse_mesh (.off / .obj by extension, polygons fan-triangulated) */
int mp_read_mesh(const char* path, int32_t format /* 0 by extension, 1 OFF, 2 OBJ */, int32_t* vertex_count,
                 int64_t* triangle_count, int32_t* tris);
/* io.cpp:186 parse_matrix_market + types.cpp:9 symmetrize: 0-based, sorted, unique */
int mp_read_matrix_market(const char* path, int32_t* n, int64_t* nnz, int32_t* rows, int32_t* cols);
/* io.cpp:242 read_patch_file: exactly n nonnegative ids; patch_count = max + 1 */
int mp_read_patch_file(const char* path, int32_t n, int32_t* assignment, int32_t* patch_count);
/* io.cpp:264 write_permutation / io.cpp:270 read_permutation: one index per line */
int mp_write_permutation(const char* path, int32_t n, const int32_t* perm);
int mp_read_permutation(const char* path, int32_t* n, int32_t* perm);
/* io.cpp:283 write_etree: "idx level count v..." per node of the 2^(L+1)-1 tree */
int mp_write_etree(const char* path, int32_t nd_level, const int32_t* node_offsets,
                   const int32_t* node_vertices);

/* pipeline.hpp:39-54 BenchRow and pipeline.cpp:188-205 csv_header / write_csv
 * (the reference writes to a stream; here to a file path). */
typedef struct {
  const char* input;
  int64_t n, nnz_A;
  const char* method;
  int32_t patch_size, nd_level;
  double t_patch_ms, t_quotient_ms, t_etree_ms, t_local_ms, t_assemble_ms;
  int64_t nnz_L;
  double fill_ratio;
  int64_t cost;
} mp_bench_row;
const char* mp_csv_header(void);
int mp_write_csv(const char* path, const mp_bench_row* rows, int32_t count);

#ifdef __cplusplus
}
#endif
#endif
