// The library context and the internal stage interfaces (device pointers).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <vector>

#include "mp_internal.h"

struct mp_context {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // second stream for work that overlaps the main one inside a stage (forked
  // from and joined back into `stream` with fork_ev)
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t fork_ev[2] = {};
  int num_sms = 148;
  int smem_optin = 232448;  // cudaDevAttrMaxSharedMemoryPerBlockOptin
  int64_t launches = 0;  // kernels launched through this context (cumulative)
  cudaEvent_t ev[8] = {};
  // pinned staging for host-memory arguments
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // symbolic boundary-pool size learnt from earlier calls (ints per vertex)
  double sym_pool_ratio = 0.0;
  // per-kernel event pairs of the current call (mp_result.kernel_ms)
  std::vector<cudaEvent_t> kev;
  std::vector<std::pair<int, int>> kev_used;  // (kernel slot, first event index)
  void ktime_reset() {
    kev_used.clear();
    for (auto& w : work) w = 0;
  }
  // device work counters of the current call (mp_result.work), device memory
  unsigned long long* dwork = nullptr;
  int64_t work[16] = {};
  int ktime_begin(int slot);
  void ktime_end(int first);
  // Persistent device slabs (cudaMalloc, grown on demand, kept across calls)
  // for the large per-call scratch, so repeated calls do no pool traffic.
  std::vector<std::pair<void*, size_t>> slabs;
  void* slab(int id, size_t bytes);
  int fps_workers = 0;  // worker CTAs of the batched FPS (decided once)
  int sm_share = 1;     // contexts expected to run concurrently on the device (grid sizing)
  int fill_algo = 0;    // 0: etree + column counts (colcount.cu), 1: the elimination game (symbolic.cu)
  int64_t tune[8] = {};  // mp_context_set_tuning (MP_TUNE_*), 0 = default
  // private stream-ordered pool for the per-call scratch (release threshold
  // raised on this pool only, never on the device's default pool)
  cudaMemPool_t pool = nullptr;
};

namespace mp {

// The pool DevBuf allocates from on this thread (set by ContextScope).
extern thread_local cudaMemPool_t tl_pool;

// Entry-point scope: the context's device is current and its private pool
// serves DevBuf allocations; both are restored on exit.
struct ContextScope {
  int prev = 0;
  int dev = 0;
  cudaMemPool_t prev_pool = nullptr;
  explicit ContextScope(const mp_context& ctx) : dev(ctx.device), prev_pool(tl_pool) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
    tl_pool = ctx.pool;
  }
  ~ContextScope() {
    tl_pool = prev_pool;
    if (prev != dev) cudaSetDevice(prev);
  }
  ContextScope(const ContextScope&) = delete;
  ContextScope& operator=(const ContextScope&) = delete;
};

// Debug section timer: with MP_PROFILE=1 in the environment, synchronises the
// stream at every mark and prints host wall time between marks to stderr.
struct SectionTimer {
  cudaStream_t s;
  const char* scope;
  bool on;
  double t0;
  SectionTimer(cudaStream_t st, const char* sc);
  void mark(const char* what);
};

struct DGraph {
  int32_t n;
  const int32_t* off;
  const int32_t* nbr;
};

// Persistent context slab ids (mp_context::slab): 0-4 farthest-point seeding.
enum SlabId { kSlabMd = 5, kSlabFill = 6 };

// Kernel-time slots reported in mp_result.kernel_ms.
enum KernelSlot { kKFps = 0, kKLloyd = 1, kKFm = 2, kKRefine = 3, kKMd = 4, kKSym = 5, kKSlots = 6 };

// Count a launch and check it.
#define MP_KERNEL(ctx, ...)        \
  do {                             \
    __VA_ARGS__;                   \
    ++(ctx).launches;              \
    MP_CUDA(cudaGetLastError());   \
  } while (0)

// Stage 1 (patching.cu): compute_patches -> assignment (device, n), returns patch count.
int32_t compute_patches_dev(mp_context& ctx, const DGraph& g, int32_t target, uint64_t seed,
                            int32_t* assignment);
// patching.cu: enforce_connectivity on a device assignment; returns the new patch count.
int32_t enforce_connectivity_dev(mp_context& ctx, const DGraph& g, const int32_t* in,
                                 int32_t patch_count, int32_t* out);
// patching.cu: validate_user_patches (patching.cpp:386-433); throws MP_EINVAL
// with the reference's message for an out-of-range id.
struct UserPatchReport {
  std::vector<int64_t> sizes;
  std::vector<int32_t> disconnected, unused;
};
UserPatchReport validate_user_patches_dev(mp_context& ctx, const DGraph& g, const int32_t* in, int32_t patch_count);

// Sharded ND (mp_order_sharded): every rank splits the top k
// levels; at level k the subtrees are dealt to ranks (owner[i] = rank for
// nodes of level >= k, -1 above) and a rank splits only its own subtrees
// further -- the others stay whole in their level-k root in its local tree.
struct ShardSpec {
  int32_t rank = 0, world = 1, k = 0;
  std::vector<int32_t> owner;  // out: nn entries
};
std::vector<int32_t> deal_subtrees(const std::vector<int64_t>& root_size, int32_t k, int32_t L, int32_t world);

// ND tree (ndtree.cu).  node_of[v] receives the tree node of every vertex;
// node_offsets (nn+1) / node_vertices (n) the flattened EliminationTree.
void build_etree_dev(mp_context& ctx, const DGraph& g, const int32_t* assignment,
                     int32_t patch_count, int32_t nd_level, int32_t* node_of,
                     int32_t* node_offsets, int32_t* node_vertices, ShardSpec* shard = nullptr);

// Quotient (ndtree.cu): node weights (P) + positive edges, device outputs; returns #edges.
int64_t build_quotient_dev(mp_context& ctx, const DGraph& g, const int32_t* assignment,
                           int32_t patch_count, int64_t* node_weight, int32_t** edge_p,
                           int32_t** edge_q, int64_t** edge_w);

// Local ordering (md.cu): local_perm per node, layout of node_vertices.
void order_tree_nodes_dev(mp_context& ctx, const DGraph& g, int32_t nd_level,
                          const int32_t* node_of, const int32_t* node_offsets,
                          const int32_t* node_vertices, int32_t mode, int32_t* local_perm,
                          const uint8_t* node_mask = nullptr);

// Node schedules (assemble.cu): schedule_postorder / schedule_levelorder
// (assemble.cpp:24-46), or a caller sequence checked like validate_schedule
// (assemble.cpp:48-63; MP_EINVAL "invalid schedule at position N").
using Schedule = std::vector<int32_t>;
Schedule make_schedule(int32_t L, int32_t kind);
int64_t validate_schedule_host(int32_t L, const int32_t* seq, int64_t len);
Schedule resolve_schedule(int32_t L, int32_t kind, const int32_t* nodes, int64_t len);
std::vector<int32_t> node_positions(const std::vector<int32_t>& node_offsets, int32_t L, const Schedule& sched);

// Assembly (assemble.cu): schedule + perm/inverse.  node_pos (nn+1) receives
// the first permutation position of every node.
void compute_perm_dev(mp_context& ctx, int32_t n, int32_t nd_level, const int32_t* node_offsets,
                      const int32_t* node_vertices, const int32_t* local_perm, const Schedule& schedule,
                      int32_t* perm, int32_t* inverse, int32_t* node_pos);
void compute_perm_blocks_dev(mp_context& ctx, int32_t n, int32_t L, const int32_t* node_offsets,
                             const int32_t* node_vertices, const int32_t* local_perm, const Schedule& schedule,
                             int32_t b, int32_t* perm, int32_t* inverse, int32_t* node_pos_dev);
// Sharded assembly: perm entries of the masked nodes only (no inverse, no
// bijection check -- the other ranks own the remaining positions).
void compute_perm_partial_dev(mp_context& ctx, int32_t n, int32_t nd_level, const int32_t* node_offsets,
                              const int32_t* node_vertices, const int32_t* local_perm, const Schedule& schedule,
                              const uint8_t* node_mask, int32_t* perm);

// Sharded game (mp_order_sharded): this rank plays the nodes of its own
// subtrees below level k (owner[i] == rank), hands their level-k roots' live
// elements to `exchange` (an all-gather returning every rank's buffer,
// concatenated), imports the others', then plays levels k-1..0 itself.
// Column counts / parents are then valid at the positions of its own nodes
// and of the top nodes; nnz_L / cost are left to the caller's gather.
struct FillShard {
  int32_t rank = 0, k = 0;
  std::vector<int32_t> owner;
  std::function<std::vector<int32_t>(const std::vector<int32_t>&)> exchange;
};
// Symbolic (symbolic.cu): column counts (by position) and factor etree parents.
void tree_fill_dev(mp_context& ctx, const DGraph& g, int32_t nd_level, const int32_t* node_of,
                   const int32_t* node_offsets, const int32_t* node_vertices,
                   const int32_t* local_perm, const int32_t* node_pos, const int32_t* inverse,
                   int64_t* column_counts, int32_t* etree_parent, int64_t* nnz_L, int64_t* cost,
                   const int32_t* cross_owner = nullptr, int64_t* crossing = nullptr,
                   const FillShard* shard = nullptr);
// The same outputs from the factor's elimination tree (colcount.cu): Liu's
// etree split by the ND tree, a postorder, Gilbert-Ng-Peyton column counts.
// Needs a tree whose separators separate (no edge between unrelated nodes).
void tree_fill_fast_dev(mp_context& ctx, const DGraph& g, int32_t nd_level, const int32_t* node_of,
                        const int32_t* node_offsets, const int32_t* node_vertices, const int32_t* local_perm,
                        const int32_t* node_pos, const int32_t* inverse, int64_t* column_counts,
                        int32_t* etree_parent, int64_t* nnz_L, int64_t* cost);
void sum_counts_dev(mp_context& ctx, int64_t n, const int64_t* column_counts, int64_t* nnz_L, int64_t* cost);
// The same game for any permutation (one-node tree): elimination_fill,
// factor_etree_parents and, with cross_owner, cross_block_fill's count.
void elimination_game_dev(mp_context& ctx, const DGraph& g, const int32_t* perm, int64_t* column_counts,
                          int32_t* etree_parent, int64_t* nnz_L, int64_t* cost, const int32_t* cross_owner,
                          int64_t* crossing);

// node_of[v] from the flattened tree (assemble.cu).
void node_of_from_tree_dev(mp_context& ctx, int32_t n, int32_t nn, const int32_t* node_offsets,
                           const int32_t* node_vertices, int32_t* node_of);

}  // namespace mp
