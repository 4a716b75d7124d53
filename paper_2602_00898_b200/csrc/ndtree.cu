// Stages 2+4 — separator extraction and the patch-guided ND tree
// (reference core/src/{quotient,partition,etree}.cpp).
//
// The reference recurses depth first, keeping one master quotient updated
// incrementally (quotient_remove, quotient.cpp:82-103) and restricting it per
// node (restrict_quotient, :105-127).  Sibling subtrees touch disjoint patch
// sets and no edge joins two alive vertices of different subtrees, so the
// restricted quotient of a node equals the quotient of the node's alive
// vertices.  The device version therefore runs level by level: every level
// rebuilds the per-node quotients from the alive vertices (one sort of the
// crossing-edge keys), then one CTA per node runs bipartition_quotient
// (partition.cpp:25-163) and one CTA per node refine_separator
// (:187-283); the super separator (:165-185) is a grid pass.  Results are
// identical to the depth-first recursion.
#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kFmPasses = 10;        // partition.cpp:13
constexpr double kBalanceTol = 1.2;  // partition.hpp:34
constexpr int kMaxNdLevel = 24;      // etree.cpp:16
constexpr int kNodeThreads = 1024;
constexpr int32_t kGainBias = 0x40000000;

int grid_for(const mp_context& ctx, int64_t n, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), ctx.num_sms * 16LL)));
}

__global__ void iota32(int32_t n, int32_t* a) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}
__global__ void fill32(int64_t n, int32_t* a, int32_t v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    a[i] = v;
}

// ---------------------------------------------------------------- per level
struct LevelArgs {
  DGraph g;
  const int32_t* assign;
  int32_t P;
  int32_t first;           // first node id of the level
  int32_t width;           // nodes at the level
  const int32_t* vlist;    // vertices grouped by node, ascending inside a node
  const int32_t* seg_start;// per level node (local index)
  const int32_t* seg_cnt;
  int32_t* node_of;
  int32_t* pw;             // patch weights at this level (P)
  int32_t* pnode;          // node (local index) of each weighted patch
  int32_t* np_node;        // alive patches per level node
  int32_t* active;         // per level node
  int32_t* lidx;           // patch -> index inside its node's patch list
  const int32_t* plist;    // alive patches grouped by node, ascending
  const int32_t* poff;     // per level node (width+1)
  const int32_t* qoff;     // per patch (P+1), quotient adjacency at this level
  const int32_t* qnbr;
  const int32_t* qw;
  uint8_t* side;           // per patch
  int8_t* region;          // per vertex
  uint8_t* in_super;       // per vertex
  uint8_t* in_list;        // per vertex
  int32_t* bcount;         // per level node: [2*i] left boundary, [2*i+1] right
  int32_t* sep_list;       // scratch, vlist layout
  int32_t* next_vlist;
  int32_t* next_start;     // per next-level node
  int32_t* next_cnt;
  unsigned long long* stats;  // [0] moves FM, [1] moves refine (work counters)
  // FM scratch (per patch, in plist layout)
  int32_t* fm_gain;
  int32_t* fm_w;           // global state for nodes whose state does not fit shared memory
  int32_t* fm_ab;          // (ab, ae) pairs, 2 * P
  int32_t* fm_ae;
  uint8_t* fm_side;        // 4 * P bytes: status words (fm_st)
  const int32_t* qloc;     // quotient adjacency as node-local patch indices
  int32_t* fm_fifo;        // capacity per node: poff span + edges -> allocated 2*P + E
  const int64_t* fm_fifo_off;  // per level node
  int32_t* slot_of;        // refine: vertex -> candidate-list slot
  int32_t* ref_pull;       // refine: global fallback lists (vlist layout)
  uint8_t* ref_own;
  uint8_t* ref_in;
  int32_t* ref_pulled;
  uint8_t* vside;          // per vertex: side of its patch (this level)
  const int32_t* ell;      // n * 8 ELL adjacency
  int64_t fm_smem_bytes;   // dynamic shared memory of the FM launch
  int32_t fm_w16;          // every patch weight of the level is below 65536 (fm_node<SMC, W16>)
  int32_t* fm_moves;
  const uint8_t* own_mask; // sharded build (mp_order_sharded): nodes this rank splits; NULL = all
  int32_t* ref_cnt;        // per level node: initial separator size (ref_init)
  int32_t* ref_rw;         // per level node: [2*i] / [2*i+1] remaining vertices per side
};

__global__ void level_weights(LevelArgs a) {
  for (int32_t li = blockIdx.y; li < a.width; li += gridDim.y) {
    const int32_t s0 = a.seg_start[li], cnt = a.seg_cnt[li];
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
      int32_t p = a.assign[a.vlist[s0 + i]];
      if (atomicAdd(&a.pw[p], 1) == 0) a.pnode[p] = li;
    }
  }
}
__global__ void level_patch_counts(LevelArgs a) {
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < a.P; p += gridDim.x * blockDim.x)
    if (a.pw[p] > 0) atomicAdd(&a.np_node[a.pnode[p]], 1);
}
__global__ void level_activity(LevelArgs a, int32_t nd_level, int32_t level, int32_t* n_active) {
  for (int32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < a.width; li += gridDim.x * blockDim.x) {
    // etree.cpp:123-131: leaf at nd_level, below 2 vertices, or <= 1 alive patch
    bool act = level < nd_level && a.seg_cnt[li] >= 2 && a.np_node[li] >= 2;
    // sharded build: subtrees below the shard level that another rank owns
    // stay whole in their level-k root here (that rank splits them)
    if (a.own_mask && !a.own_mask[a.first + li]) act = false;
    a.active[li] = act ? 1 : 0;
    if (act) atomicAdd(n_active, 1);
  }
}
__global__ void flag_alive_patches(int32_t P, const int32_t* pw, const int32_t* pnode,
                                   const int32_t* active, int32_t* flag, int32_t* key) {
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    bool ok = pw[p] > 0 && active[pnode[p]];
    flag[p] = ok ? 1 : 0;
    key[p] = ok ? pnode[p] : 0;
  }
}
__global__ void build_ell_nd(DGraph g, int32_t* ell) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
    const int32_t o = g.off[v], deg = g.off[v + 1] - o;
    int32_t* e = ell + static_cast<int64_t>(v) * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) e[k] = k < deg ? g.nbr[o + k] : -1;
    if (deg > 8) e[7] = -(o + 7) - 2;
  }
}
__global__ void masked_counts(int32_t width, const int32_t* active, const int32_t* np_node, int32_t* out) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= width; i += gridDim.x * blockDim.x)
    out[i] = (i < width && active[i]) ? np_node[i] : 0;
}
__global__ void node_edge_count(int32_t na, const int32_t* plist, const int32_t* pnode, const int32_t* qoff,
                                int64_t* ecnt) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
    const int32_t p = plist[i];
    atomicAdd(reinterpret_cast<unsigned long long*>(&ecnt[pnode[p]]),
              static_cast<unsigned long long>(qoff[p + 1] - qoff[p] + 1));
  }
}
__global__ void set_lidx(int32_t total, const int32_t* plist, const int32_t* pnode, const int32_t* poff,
                         int32_t* lidx) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    int32_t p = plist[i];
    lidx[p] = i - poff[pnode[p]];
  }
}
// Small quotients (P <= kSmallP): the alive patches of the active nodes,
// grouped by node and ascending inside it (the stable radix sort of the
// general path), with the per-node offsets and the node-local indices -- in
// ONE CTA: a bitonic sort of (node << 13 | patch) keys in shared memory and a
// block scan of the node counts, instead of a dozen small launches per level.
constexpr int32_t kSmallP = 8192;
__global__ void __launch_bounds__(1024) level_lists_small(int32_t P, int32_t width, const int32_t* pw,
                                                          const int32_t* pnode, const int32_t* np_node,
                                                          const int32_t* active, int32_t* plist, int32_t* poff,
                                                          int32_t* lidx, int32_t* cnt) {
  __shared__ uint32_t key[kSmallP];
  __shared__ int32_t sh[32], s_na;
  int32_t N = 1;
  while (N < P) N <<= 1;
  if (threadIdx.x == 0) s_na = 0;
  __syncthreads();
  int32_t mine = 0;
  for (int32_t q = threadIdx.x; q < N; q += blockDim.x) {
    const bool ok = q < P && pw[q] > 0 && active[pnode[q]];
    key[q] = ok ? (static_cast<uint32_t>(pnode[q]) << 13) | static_cast<uint32_t>(q) : 0xffffffffu;
    mine += ok;
  }
  atomicAdd(&s_na, mine);
  for (int32_t k = 2; k <= N; k <<= 1)
    for (int32_t j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int32_t i = threadIdx.x; i < N; i += blockDim.x) {
        const int32_t l = i ^ j;
        if (l > i) {
          const uint32_t x = key[i], y = key[l];
          if (((i & k) == 0) == (x > y)) key[i] = y, key[l] = x;
        }
      }
    }
  __syncthreads();
  // per-node offsets: exclusive scan of the active nodes' patch counts
  int32_t run = 0;
  for (int32_t b0 = 0; b0 <= width; b0 += blockDim.x) {
    const int32_t i = b0 + threadIdx.x;
    const int32_t c = (i < width && active[i]) ? np_node[i] : 0;
    int32_t tot;
    const int32_t ex = block_excl_scan(c, sh, &tot);
    if (i <= width) poff[i] = run + ex;
    run += tot;
  }
  __syncthreads();
  const int32_t na = s_na;
  for (int32_t i = threadIdx.x; i < na; i += blockDim.x) {
    const uint32_t kk = key[i];
    const int32_t q = static_cast<int32_t>(kk & 0x1fffu), node = static_cast<int32_t>(kk >> 13);
    plist[i] = q;
    lidx[q] = i - poff[node];
  }
  if (threadIdx.x == 0) cnt[1] = na, cnt[2] = na;
}
// Small levels (nkeys <= kSmallKeys, P <= kSmallP, width <= 1024): the
// quotient CSR of the alive vertices (sort + run-length encoding of the
// crossing keys), the per-node fifo offsets and the node-local adjacency in
// ONE CTA -- the general path's CUB sort, run-length encoding, scans and four
// small kernels, and its read-back of the run count, become one launch.
constexpr int32_t kSmallKeys = 8192;
__global__ void __launch_bounds__(1024) quotient_small(int32_t nk, const uint64_t* keys, int32_t P, int32_t width,
                                                       int32_t na, const int32_t* plist, const int32_t* pnode,
                                                       const int32_t* lidx, int32_t* qoff, int32_t* qnbr, int32_t* qw,
                                                       int32_t* qloc, int64_t* fifo_off) {
  extern __shared__ uint64_t qsm[];
  uint64_t* k64 = qsm;                                           // N sorted keys
  int32_t* rstart = reinterpret_cast<int32_t*>(k64 + kSmallKeys);  // run starts (U + 1)
  int32_t* qdeg = rstart + kSmallKeys + 1;                       // P + 1
  int32_t* ecnt = qdeg + kSmallP + 1;                            // width + 1
  __shared__ int32_t sh[32], s_u;
  int32_t N = 1;
  while (N < nk) N <<= 1;
  for (int32_t i = threadIdx.x; i < N; i += blockDim.x) k64[i] = i < nk ? keys[i] : ~0ull;
  for (int32_t i = threadIdx.x; i <= P; i += blockDim.x) qdeg[i] = 0;
  for (int32_t i = threadIdx.x; i <= width; i += blockDim.x) ecnt[i] = 0;
  for (int32_t k = 2; k <= N; k <<= 1)
    for (int32_t j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int32_t i = threadIdx.x; i < N; i += blockDim.x) {
        const int32_t l = i ^ j;
        if (l > i) {
          const uint64_t x = k64[i], y = k64[l];
          if (((i & k) == 0) == (x > y)) k64[i] = y, k64[l] = x;
        }
      }
    }
  __syncthreads();
  // run-length encoding: run r starts at rstart[r]
  int32_t run = 0;
  for (int32_t b0 = 0; b0 < nk; b0 += blockDim.x) {
    const int32_t i = b0 + threadIdx.x;
    const int32_t f = (i < nk && (i == 0 || k64[i] != k64[i - 1])) ? 1 : 0;
    int32_t tot;
    const int32_t ex = block_excl_scan(f, sh, &tot);
    if (f) {
      const int32_t r = run + ex;
      rstart[r] = i;
      qnbr[r] = static_cast<int32_t>(k64[i] & 0xffffffffu);
      atomicAdd(&qdeg[static_cast<int32_t>(k64[i] >> 32)], 1);
    }
    run += tot;
  }
  if (threadIdx.x == 0) s_u = run, rstart[run] = nk;
  __syncthreads();
  const int32_t U = s_u;
  for (int32_t r = threadIdx.x; r < U; r += blockDim.x) {
    qw[r] = rstart[r + 1] - rstart[r];
    qloc[r] = lidx[qnbr[r]];
  }
  // qoff: exclusive scan of the patch degrees
  run = 0;
  for (int32_t b0 = 0; b0 <= P; b0 += blockDim.x) {
    const int32_t i = b0 + threadIdx.x;
    const int32_t c = i < P ? qdeg[i] : 0;
    int32_t tot;
    const int32_t ex = block_excl_scan(c, sh, &tot);
    if (i <= P) qoff[i] = run + ex;
    run += tot;
  }
  __syncthreads();
  // fifo slabs: a node's quotient entries + 1 per alive patch (partition.cpp:76-77)
  for (int32_t i = threadIdx.x; i < na; i += blockDim.x) {
    const int32_t q = plist[i];
    atomicAdd(&ecnt[pnode[q]], qoff[q + 1] - qoff[q] + 1);
  }
  __syncthreads();
  int64_t run64 = 0;
  for (int32_t b0 = 0; b0 <= width; b0 += blockDim.x) {
    const int32_t i = b0 + threadIdx.x;
    const int32_t c = i < width ? ecnt[i] : 0;
    int32_t tot;
    const int32_t ex = block_excl_scan(c, sh, &tot);
    if (i <= width) fifo_off[i] = run64 + ex;
    run64 += tot;
  }
}
// Crossing-edge keys among alive vertices of active nodes; both directions.
__global__ void emit_crossing(LevelArgs a, uint64_t* keys, int32_t* count) {
  for (int32_t li = blockIdx.y; li < a.width; li += gridDim.y) {
    if (!a.active[li]) continue;
    const int32_t s0 = a.seg_start[li], cnt = a.seg_cnt[li], node = a.first + li;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
      const int32_t u = a.vlist[s0 + i];
      const int32_t pu = a.assign[u];
      for (int32_t j = a.g.off[u]; j < a.g.off[u + 1]; ++j) {
        const int32_t v = a.g.nbr[j];
        if (v <= u || a.node_of[v] != node) continue;
        const int32_t pv = a.assign[v];
        if (pv == pu) continue;
        int32_t slot = atomicAdd(count, 2);
        keys[slot] = (static_cast<uint64_t>(pu) << 32) | static_cast<uint32_t>(pv);
        keys[slot + 1] = (static_cast<uint64_t>(pv) << 32) | static_cast<uint32_t>(pu);
      }
    }
  }
}
__global__ void quotient_csr(int32_t U, const uint64_t* ukeys, const int32_t* ucnt, int32_t* qdeg,
                             int32_t* qnbr, int32_t* qw) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < U; i += gridDim.x * blockDim.x) {
    qnbr[i] = static_cast<int32_t>(ukeys[i] & 0xffffffffu);
    qw[i] = ucnt[i];
    atomicAdd(&qdeg[static_cast<int32_t>(ukeys[i] >> 32)], 1);
  }
}

// ---------------------------------------------------------------- FM (one CTA per node)
// bipartition_quotient, partition.cpp:25-163.  The node's patch state
// (weight, gain, side, lock, adjacency bounds, cache slot) lives in shared
// memory when it fits (global scratch otherwise); the adjacency carries
// node-local indices (qloc).
//
// Move selection.  The reference takes the first feasible entry of its
// std::set<(-gain, id)>: the max key (gain desc, id asc) over the feasible
// unlocked patches.  The move loop runs in warp 0 alone over a per-side
// candidate cache: lane l holds entry l of side 0 and entry l of side 1
// (key, patch, weight), and a bound B_s says every unlocked side-s patch
// outside the cache has key <= B_s.  The best feasible cached key f_s is the
// side's answer when f_s > B_s (or nothing is outside); the move is the larger
// answer provided no side with an unknown answer could beat it (B_s < best).
// A move changes only its neighbours' keys: cached ones are re-read, raised
// uncached ones above B_s are inserted (a full cache evicts its minimum into
// B_s).  When a side's answer is unknown the whole CTA refills that side with
// its top 32 keys (radix select); if it is still unknown right after a
// refill, the CTA takes the exact argmax over all patches for one move.  The
// chosen move is always the reference's; on the C2 root (3,901 patches,
// 23,406 moves) the cache needs 35 refills.
// Per-patch status word: side (byte 0), lock / visited flag (byte 1), cache
// slot (byte 2: side << 5 | lane, or kNoSlot).
__device__ __forceinline__ uint32_t fm_st(uint32_t side, uint32_t flag, uint32_t slot) {
  return side | (flag << 8) | (slot << 16);
}
constexpr int kFmThreads = 256;
constexpr uint8_t kNoSlot = 0xff;
constexpr int kFmDone = 8, kFmExact = 4;  // segment exit reasons (1, 2: refill side 0 / 1)

// FM move keys (gain desc, id asc): 32-bit when the node has < 65536 patches
// and |gain| < 32768, 64-bit otherwise.  0 is never a key.
template <class K> struct FmKey;
template <> struct FmKey<uint32_t> {
  static __device__ __forceinline__ uint32_t make(int32_t gain, int32_t i) {
    return (static_cast<uint32_t>(gain + 32768) << 16) | (0xffffu - static_cast<uint32_t>(i));
  }
  static __device__ __forceinline__ int32_t id(uint32_t k) { return static_cast<int32_t>(0xffffu - (k & 0xffffu)); }
  static __device__ __forceinline__ int32_t gain(uint32_t k) { return static_cast<int32_t>(k >> 16) - 32768; }
  static __device__ __forceinline__ uint32_t wmax(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }
  static __device__ __forceinline__ uint32_t wmin(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
};
template <> struct FmKey<uint64_t> {
  static __device__ __forceinline__ uint64_t make(int32_t gain, int32_t i) {
    return key_max(static_cast<uint32_t>(gain + kGainBias), static_cast<uint32_t>(i));
  }
  static __device__ __forceinline__ int32_t id(uint64_t k) { return static_cast<int32_t>(key_max_id(k)); }
  static __device__ __forceinline__ int32_t gain(uint64_t k) {
    return static_cast<int32_t>(static_cast<uint32_t>(k >> 32) - static_cast<uint32_t>(kGainBias));
  }
  static __device__ __forceinline__ uint64_t wmax(uint64_t v) { return warp_max_u64(v); }
  static __device__ __forceinline__ uint64_t wmin(uint64_t v) { return warp_min_u64(v); }
};

// imbalance_of(ns, nt) > max(tol, imbalance_of(H, L)) with tol = 1.2, the
// reference's double test (partition.cpp:114-124).  EXACT: integer form, valid
// for node weights below 2^26 (the host checks n):
//  * fl(h/l) > fl(1.2) <=> 5h > 6l: a ratio h/l != 6/5 lies at least 1/(5l)
//    from 6/5, far beyond the rounding of either double;
//  * fl(h/l) > fl(H/L) <=> hL > Hl: distinct ratios with hL, Hl < 2^52 are
//    more than one rounding apart, so the rounded doubles keep their order.
// Infinite ratios (l = 0 or L = 0) come out right: 0 > ... is false.
static_assert(kBalanceTol == 1.2, "fm_infeasible encodes tol = 6/5");
constexpr int64_t kFmExactWeights = int64_t(1) << 26;
template <bool EXACT>
__device__ __forceinline__ bool fm_infeasible(int32_t ns, int32_t nt, int32_t H, int32_t L) {
  const int32_t h = max(ns, nt), l = min(ns, nt);
  if constexpr (EXACT) {
    return (5 * h > 6 * l) & (static_cast<int64_t>(h) * L > static_cast<int64_t>(H) * l);  // 5h < 2^29
  } else {
    const double cur = imbalance_of(H, L);
    return imbalance_of(ns, nt) > (kBalanceTol > cur ? kBalanceTol : cur);
  }
}
// imbalance_of(a0, a1) < imbalance_of(b0, b1) (the best-prefix tie test)
template <bool EXACT>
__device__ __forceinline__ bool fm_imb_less(int32_t a0, int32_t a1, int32_t b0, int32_t b1) {
  if constexpr (EXACT) {
    return static_cast<int64_t>(max(a0, a1)) * min(b0, b1) < static_cast<int64_t>(max(b0, b1)) * min(a0, a1);
  } else {
    return imbalance_of(a0, a1) < imbalance_of(b0, b1);
  }
}

// Patch status views.  get() / set() speak the wide format of fm_st (side |
// flag << 8 | slot << 16) whatever the storage.  Wide: one u32 per patch
// (bytes side, lock / visited flag, cache slot).  Compact: one u16 (byte 0 =
// side | flag << 1, byte 1 = slot) -- with 16-bit gains, 4 B of shared state
// per patch, so nodes up to ~54K patches (C3's root) keep the state on chip.
struct FmStWide {
  uint32_t* p;
  __device__ __forceinline__ uint32_t get(int32_t i) const { return p[i]; }
  __device__ __forceinline__ void set(int32_t i, uint32_t v) const { p[i] = v; }
  __device__ __forceinline__ uint32_t side(int32_t i) const { return reinterpret_cast<const uint8_t*>(p)[4 * i]; }
  __device__ __forceinline__ uint32_t flag(int32_t i) const { return reinterpret_cast<const uint8_t*>(p)[4 * i + 1]; }
  __device__ __forceinline__ void set_slot(int32_t i, uint32_t sl) const {
    reinterpret_cast<uint8_t*>(p)[4 * i + 2] = static_cast<uint8_t>(sl);
  }
  __device__ __forceinline__ void flip(int32_t i) const { reinterpret_cast<uint8_t*>(p)[4 * i] ^= 1; }
};
struct FmStCompact {
  uint16_t* p;
  __device__ __forceinline__ uint32_t get(int32_t i) const {
    const uint32_t v = p[i];
    return (v & 1u) | (((v >> 1) & 1u) << 8) | ((v >> 8) << 16);
  }
  __device__ __forceinline__ void set(int32_t i, uint32_t v) const {
    p[i] = static_cast<uint16_t>((v & 1u) | (((v >> 8) & 1u) << 1) | (((v >> 16) & 0xffu) << 8));
  }
  __device__ __forceinline__ uint32_t side(int32_t i) const { return reinterpret_cast<const uint8_t*>(p)[2 * i] & 1u; }
  __device__ __forceinline__ uint32_t flag(int32_t i) const {
    return (reinterpret_cast<const uint8_t*>(p)[2 * i] >> 1) & 1u;
  }
  __device__ __forceinline__ void set_slot(int32_t i, uint32_t sl) const {
    reinterpret_cast<uint8_t*>(p)[2 * i + 1] = static_cast<uint8_t>(sl);
  }
  __device__ __forceinline__ void flip(int32_t i) const { reinterpret_cast<uint8_t*>(p)[2 * i] ^= 1; }
};

// Byte status (compact layout with shared-memory weights): side (bit 0),
// flag (bit 1), cache-slot valid (bit 2), slot lane (bits 3-7).  A valid
// slot's side is always the patch's own side (side-t caches hold side-t
// patches; a move locks its patch and drops its slot first), so the wide
// slot side << 5 | lane is rebuilt from the side bit.
struct FmStByte {
  uint8_t* p;
  __device__ __forceinline__ uint32_t get(int32_t i) const {
    const uint32_t v = p[i];
    const uint32_t sl = (v & 4u) ? (((v & 1u) << 5) | (v >> 3)) : 0xffu;
    return (v & 1u) | (((v >> 1) & 1u) << 8) | (sl << 16);
  }
  __device__ __forceinline__ void set(int32_t i, uint32_t v) const {
    const uint32_t sl = (v >> 16) & 0xffu;
    p[i] = static_cast<uint8_t>((v & 1u) | (((v >> 8) & 1u) << 1) | (sl == 0xffu ? 0u : (4u | ((sl & 31u) << 3))));
  }
  __device__ __forceinline__ uint32_t side(int32_t i) const { return p[i] & 1u; }
  __device__ __forceinline__ uint32_t flag(int32_t i) const { return (p[i] >> 1) & 1u; }
  __device__ __forceinline__ void set_slot(int32_t i, uint32_t sl) const {
    p[i] = static_cast<uint8_t>((p[i] & 3u) | (sl == 0xffu ? 0u : (4u | ((sl & 31u) << 3))));
  }
  __device__ __forceinline__ void flip(int32_t i) const { p[i] ^= 1u; }
};

// CTA-wide: refill the side-t cache with the 32 largest keys of the unlocked
// side-t patches; B[t] = the 33rd largest (0 when there are at most 32).
// The threshold is an MSD radix select over the bits below the common prefix
// of the largest and smallest candidate key.
template <class K, class G, class SV>
__device__ __forceinline__ void fm_refill(int32_t t, int32_t np, G gain, SV st, K (*ck)[32], int32_t (*cp)[32], K* B, int32_t* hist, uint64_t* red,
                          int32_t* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x < 32) {
    const int32_t p = cp[t][threadIdx.x];
    if (p >= 0) st.set_slot(p, kNoSlot);
    cp[t][threadIdx.x] = -1;
    ck[t][threadIdx.x] = 0;
  }
  int64_t c = 0;
  uint64_t mx = 0, mn = ~0ull;
  for (int32_t i = threadIdx.x; i < np; i += blockDim.x)
    if ((st.get(i) & 0xffffu) == static_cast<uint32_t>(t)) {  // unlocked, side t
      const uint64_t k = FmKey<K>::make(gain[i], i);
      ++c, mx = k > mx ? k : mx, mn = k < mn ? k : mn;
    }
  c = block_sum_i64(c, reinterpret_cast<int64_t*>(red));
  mx = block_max_u64(mx, red);
  mn = block_min_u64(mn, red);
  uint64_t T = 0;
  if (c > 32) {
    const int hb = 63 - __clzll(static_cast<long long>(mx ^ mn));  // keys are distinct: mx != mn
    const uint64_t low = hb == 63 ? ~0ull : ((1ull << (hb + 1)) - 1);
    uint64_t prefix = mx & ~low, pmask = ~low;
    int32_t rank = 33;
    for (int lo = hb + 1; lo > 0;) {
      const int dbits = lo < 8 ? lo : 8;
      lo -= dbits;
      const int32_t nbins = 1 << dbits;
      for (int32_t b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
      __syncthreads();
      for (int32_t i0 = wid * 32; i0 < np; i0 += nw * 32) {
        const int32_t i = i0 + lane;
        int32_t d = -1;
        if (i < np && (st.get(i) & 0xffffu) == static_cast<uint32_t>(t)) {
          const uint64_t k = FmKey<K>::make(gain[i], i);
          if ((k & pmask) == prefix) d = static_cast<int32_t>((k >> lo) & static_cast<uint64_t>(nbins - 1));
        }
        const uint32_t m = __match_any_sync(0xffffffffu, d);
        if (d >= 0 && lane == __ffs(m) - 1) atomicAdd(&hist[d], __popc(m));
      }
      __syncthreads();
      if (wid == 0) {  // digit holding the rank-th largest: bins from the top
        int32_t loc = 0;
        for (int q = 0; q < 8; ++q) {
          const int32_t b = nbins - 1 - (lane * 8 + q);
          if (b >= 0) loc += hist[b];
        }
        int32_t inc = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        int32_t run = inc - loc;
        if (run < rank && rank <= inc) {
          for (int q = 0; q < 8; ++q) {
            const int32_t b = nbins - 1 - (lane * 8 + q);
            if (run + hist[b] >= rank) {
              sh[0] = b, sh[1] = rank - run;
              break;
            }
            run += hist[b];
          }
        }
      }
      __syncthreads();
      prefix |= static_cast<uint64_t>(sh[0]) << lo;
      pmask |= static_cast<uint64_t>(nbins - 1) << lo;
      rank = sh[1];
      __syncthreads();
    }
    T = prefix;  // the 33rd largest key itself
  }
  if (threadIdx.x == 0) sh[2] = 0;
  __syncthreads();
  for (int32_t i = threadIdx.x; i < np; i += blockDim.x)
    if ((st.get(i) & 0xffffu) == static_cast<uint32_t>(t)) {
      const K k = FmKey<K>::make(gain[i], i);
      if (k > T) {
        const int32_t slot = atomicAdd(&sh[2], 1);
        ck[t][slot] = k, cp[t][slot] = i;
        st.set_slot(i, (t << 5) | slot);
      }
    }
  if (threadIdx.x == 0) B[t] = static_cast<K>(T);
  __syncthreads();
}

// Prefetch helper for the layouts whose adjacency (and, SMC / global, the
// weights) stay in global memory: warp 0 appends every patch that enters a
// candidate cache to a shared ring; while warp 0 runs its move segment, warp 1
// loads each such patch's adjacency bounds and prefetches its adjacency rows
// and its neighbours' weights into L1 (the SM's L1 serves warp 0's later
// loads: a cached candidate is usually moved within a few moves, and its move
// then reads these lines).  Pure hints: a stale or overwritten ring entry is
// still a valid patch index, and the loop leaves as soon as warp 0 posts the
// segment's end (s_done == iter) -- or after a bounded idle spin.
constexpr int32_t kFmPfRing = 256;
__device__ __forceinline__ void prefetch_l1(const int32_t* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
template <bool WGLOBAL>
__device__ __forceinline__ void fm_prefetch_helper(const int2* abe, const int32_t* qloc, const int32_t* qw,
                                                   const int32_t* w, const int32_t* ring, const volatile int32_t* tailp,
                                                   const volatile int32_t* donep, int32_t iter, int32_t& head) {
  const int lane = threadIdx.x & 31;
  for (int32_t spins = 0; spins < (1 << 26);) {  // idle polls: shared-memory loads on the helper's own SMSP
    const int32_t tail = *tailp;
    if (tail == head) {
      if (*donep == iter) break;
      ++spins;
      continue;
    }
    const int32_t h = max(head, tail - kFmPfRing);
    const int32_t cnt = min(tail - h, 32);
    if (lane < cnt) {
      const int32_t p = ring[(h + lane) & (kFmPfRing - 1)];
      const int2 e = abe[p];
      if (e.y > e.x) {
        prefetch_l1(qloc + e.x), prefetch_l1(qloc + e.y - 1);
        prefetch_l1(qw + e.x), prefetch_l1(qw + e.y - 1);
        if constexpr (WGLOBAL)
          for (int32_t j = e.x; j < e.y; ++j) prefetch_l1(w + __ldg(&qloc[j]));
      }
    }
    head = h + cnt;
  }
}

// One node's bipartition.  SM: the patch state (20 B per patch) lives in
// shared memory, else in global scratch (plist layout).  SMA: the packed
// adjacency (local id << 16 | weight) is in shared memory too, else it is
// read from qloc / qw (read-only, L2) -- the middle case keeps nodes whose
// adjacency does not fit (C5 root) on shared-memory state.
// SMC: compact state -- 16-bit gains and status in shared memory, weights and
// adjacency bounds in global scratch, adjacency from L2; with W16, 16-bit
// weights join them and the status shrinks to one byte (5 B per patch: C3's
// 39K-patch root keeps its weights on chip; the host checks they fit 16 bits).
// adjacency bounds in global scratch, adjacency from L2 (C3's root and level
// 1: 39K / 19K patches, whose 20-byte state does not fit).
template <class K, bool EXACT, bool SM, bool SMA = SM, bool SMC = false, bool W16 = false>
__device__ __forceinline__ void fm_node(const LevelArgs& a, int32_t li, int32_t pbeg, int32_t np) {
  static_assert(SM || !SMA, "packed adjacency in shared memory needs the shared state layout");
  static_assert(!(SM && SMC), "one state layout");
  static_assert(SMC || !W16, "16-bit shared weights are a compact-layout variant");
  using G = typename std::conditional<SMC, int16_t, int32_t>::type;
  using SV = typename std::conditional<W16, FmStByte, typename std::conditional<SMC, FmStCompact, FmStWide>::type>::type;
  using WT = typename std::conditional<W16, uint16_t, int32_t>::type;
  const int32_t* pl = a.plist + pbeg;
  int32_t* fifo = a.fm_fifo + a.fm_fifo_off[li];
  int32_t* moves = a.fm_moves + pbeg;
  extern __shared__ uint64_t fm_sm64_[];
  WT* w;
  G* gain;
  int2* abe;
  SV stv;  // status (fm_st)
  uint32_t* packed = nullptr;
  if constexpr (SM) {  // byte offsets from the shared base (keeps the address space visible)
    char* base = reinterpret_cast<char*>(fm_sm64_);
    w = reinterpret_cast<int32_t*>(base);
    gain = reinterpret_cast<G*>(w + np);
    abe = reinterpret_cast<int2*>(base + 8LL * np);
    stv.p = reinterpret_cast<uint32_t*>(base + 16LL * np);
    if constexpr (SMA) packed = reinterpret_cast<uint32_t*>(base + ((20LL * np + 15) & ~15LL));
  } else if constexpr (SMC) {
    char* base = reinterpret_cast<char*>(fm_sm64_);
    abe = reinterpret_cast<int2*>(a.fm_ab) + pbeg;
    gain = reinterpret_cast<G*>(base);
    const int64_t a1 = (2LL * np + 15) & ~15LL;
    if constexpr (W16) {  // gains | byte status | 16-bit weights
      stv.p = reinterpret_cast<uint8_t*>(base + a1);
      w = reinterpret_cast<WT*>(base + a1 + ((np + 15LL) & ~15LL));
    } else {
      w = a.fm_w + pbeg;
      stv.p = reinterpret_cast<uint16_t*>(base + a1);
    }
  } else {
    w = a.fm_w + pbeg;
    gain = a.fm_gain + pbeg;
    abe = reinterpret_cast<int2*>(a.fm_ab) + pbeg;
    stv.p = reinterpret_cast<uint32_t*>(a.fm_side) + pbeg;
  }
  auto side = [&](int32_t i) -> uint32_t { return stv.side(i); };
  auto flag = [&](int32_t i) -> uint32_t { return stv.flag(i); };
  auto A_nb = [&](int32_t j) -> int32_t {
    if constexpr (SMA) return static_cast<int32_t>(packed[j] >> 16);
    else return __ldg(&a.qloc[j]);
  };
  auto A_w = [&](int32_t j) -> int32_t {
    if constexpr (SMA) return static_cast<int32_t>(packed[j] & 0xffffu);
    else return __ldg(&a.qw[j]);
  };

  __shared__ uint64_t red[32];
  __shared__ int32_t hist[256], sh[4];
  __shared__ K s_ck[2][32], s_B[2], s_exact;
  __shared__ int32_t s_cp[2][32];
  __shared__ int32_t s_left, s_cut, s_sw[2], s_best_cut, s_pass_cut, s_best_s[2], s_pass_s[2];
  __shared__ int32_t s_nm, s_best_len, s_need, s_stop;
  constexpr bool PF = !SMA;  // adjacency from global memory: prefetch the candidates' rows
  __shared__ int32_t s_pf_ring[PF ? kFmPfRing : 1];
  __shared__ volatile int32_t s_pf_tail, s_pf_done;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t pf_head = 0, seg_iter = 0;  // helper warp's ring position; segment counter (every thread)
  if constexpr (PF) {
    for (int32_t i = threadIdx.x; i < kFmPfRing; i += blockDim.x) s_pf_ring[i] = 0;
    if (threadIdx.x == 0) s_pf_tail = 0, s_pf_done = -1;
  }

  int64_t tot = 0;
  for (int32_t i = threadIdx.x; i < np; i += blockDim.x) {
    const int32_t p = pl[i];
    w[i] = static_cast<WT>(a.pw[p]);
    abe[i] = make_int2(a.qoff[p], a.qoff[p + 1]);
    stv.set(i, fm_st(1, 0, kNoSlot));  // right (partition.cpp:34)
    tot += w[i];
  }
  tot = block_sum_i64(tot, reinterpret_cast<int64_t*>(red));
  if constexpr (SMA) {  // node-local packed adjacency
    int32_t run = 0;
    for (int32_t i0 = 0; i0 < np; i0 += blockDim.x) {
      const int32_t i = i0 + threadIdx.x;
      const int2 e = i < np ? abe[i] : make_int2(0, 0);
      const int32_t d = e.y - e.x;
      int32_t tt;
      const int32_t off = block_excl_scan(d, reinterpret_cast<int32_t*>(red), &tt);
      if (i < np) {
        for (int32_t q = 0; q < d; ++q)
          packed[run + off + q] = (static_cast<uint32_t>(__ldg(&a.qloc[e.x + q])) << 16) | __ldg(&a.qw[e.x + q]);
        abe[i] = make_int2(run + off, run + off + d);
      }
      run += tt;
    }
    __syncthreads();
  }

  // ---- greedy growing from the heaviest patch (partition.cpp:53-79), warp 0
  if (wid == 0) {
    int64_t left = 0;
    int32_t head = 0, tail = 0;
    while (left * 2 < tot) {
      int32_t u = -1;
      while (head < tail) {  // first unvisited fifo entry
        const int32_t h = head + lane;
        const int32_t x = h < tail ? fifo[h] : 0;
        const uint32_t m = __ballot_sync(0xffffffffu, h < tail && !flag(x));
        if (m) {
          const int l = __ffs(m) - 1;
          u = __shfl_sync(0xffffffffu, x, l);
          head += l + 1;
          break;
        }
        head = min(head + 32, tail);
      }
      if (u < 0) {  // fifo empty: heaviest unvisited patch (weight desc, id asc)
        uint64_t best = 0;
        for (int32_t i = lane; i < np; i += 32)
          if (!flag(i)) {
            const uint64_t k = key_max(static_cast<uint32_t>(w[i]), static_cast<uint32_t>(i));
            best = k > best ? k : best;
          }
        u = static_cast<int32_t>(key_max_id(warp_max_u64(best)));
      }
      if (lane == 0) stv.set(u, fm_st(0, 1, kNoSlot));
      left += w[u];
      __syncwarp();
      const int2 e = abe[u];
      for (int32_t j0 = e.x; j0 < e.y; j0 += 32) {
        const int32_t j = j0 + lane;
        const int32_t nb = j < e.y ? A_nb(j) : 0;
        const bool push = j < e.y && !flag(nb);
        const uint32_t m = __ballot_sync(0xffffffffu, push);
        if (push) fifo[tail + __popc(m & ((1u << lane) - 1))] = nb;
        tail += __popc(m);
      }
      __syncwarp();
    }
    if (lane == 0) s_left = static_cast<int32_t>(left);
  }
  __syncthreads();
  // cut of the grown split (partition.cpp:81-84)
  int64_t cut = 0;
  for (int32_t i = threadIdx.x; i < np; i += blockDim.x) {
    const int2 e = abe[i];
    for (int32_t j = e.x; j < e.y; ++j) {
      const int32_t nb = A_nb(j);
      if (nb > i && side(i) != side(nb)) cut += A_w(j);  // local order == patch id order
    }
  }
  cut = block_sum_i64(cut, reinterpret_cast<int64_t*>(red));
  if (threadIdx.x == 0) {
    s_cut = static_cast<int32_t>(cut);  // node weights and cut fit int32 (n < 2^31, 2m < 2^31)
    s_sw[0] = s_left;
    s_sw[1] = static_cast<int32_t>(tot) - s_left;
  }
  __syncthreads();

  // ---- FM passes with rollback to the best prefix (partition.cpp:95-159)
  int64_t total_moves = 0;
  for (int pass = 0; pass < kFmPasses; ++pass) {
    for (int32_t i = threadIdx.x; i < np; i += blockDim.x) {
      int32_t val = 0;
      const uint32_t si = side(i);
      const int2 e = abe[i];
      for (int32_t j = e.x; j < e.y; ++j) {
        const int32_t wj = A_w(j);
        val += side(A_nb(j)) != si ? wj : -wj;
      }
      gain[i] = val;
    }
    __syncthreads();
    for (int32_t i = threadIdx.x; i < np; i += blockDim.x) {
      stv.set(i, fm_st(side(i), 0, kNoSlot));  // unlocked
    }
    if (threadIdx.x < 64) s_cp[threadIdx.x >> 5][threadIdx.x & 31] = -1;
    if (threadIdx.x == 0) {
      s_pass_cut = s_best_cut = s_cut;
      s_pass_s[0] = s_best_s[0] = s_sw[0];
      s_pass_s[1] = s_best_s[1] = s_sw[1];
      s_nm = 0, s_best_len = 0;
      s_need = 3;
    }
    __syncthreads();
    for (;;) {
      const int32_t need = s_need;
      if (need & 1) fm_refill<K>(0, np, gain, stv, s_ck, s_cp, s_B, hist, red, sh);
      if (need & 2) fm_refill<K>(1, np, gain, stv, s_ck, s_cp, s_B, hist, red, sh);
      if constexpr (PF) {  // warps 2-3: the refilled caches' adjacency rows (warp 0 starts its segment at once)
        if ((need & 3) && wid >= 2 && wid < 4) {
          const int32_t p = s_cp[wid - 2][lane];
          if (p >= 0) {
            const int2 e = abe[p];
            if (e.y > e.x) prefetch_l1(a.qloc + e.x), prefetch_l1(a.qloc + e.y - 1), prefetch_l1(a.qw + e.x), prefetch_l1(a.qw + e.y - 1);
          }
        }
      }
      if (need & kFmExact) {  // the reference's own scan: max key over every feasible unlocked patch
        const int32_t sw0 = s_sw[0], sw1 = s_sw[1], H = max(sw0, sw1), L = min(sw0, sw1);
        uint64_t best = 0;
        for (int32_t i = threadIdx.x; i < np; i += blockDim.x) {
          if (flag(i)) continue;
          const int32_t wi = w[i], S = side(i) ? sw1 : sw0, T = side(i) ? sw0 : sw1;
          if (S - wi > 0 && !fm_infeasible<EXACT>(S - wi, T + wi, H, L)) {
            const uint64_t k = FmKey<K>::make(gain[i], i);
            best = k > best ? k : best;
          }
        }
        best = block_max_u64(best, red);
        if (threadIdx.x == 0) s_exact = static_cast<K>(best);
        __syncthreads();
      }
      if (wid == 0) {
        int32_t sw0 = s_sw[0], sw1 = s_sw[1], cut = s_cut, best_cut = s_best_cut;
        int32_t best_s0 = s_best_s[0], best_s1 = s_best_s[1];
        int32_t nm = s_nm, best_len = s_best_len;
        K B0 = s_B[0], B1 = s_B[1];
        int32_t cp0 = s_cp[0][lane], cp1 = s_cp[1][lane];
        K ck0 = cp0 >= 0 ? FmKey<K>::make(gain[cp0], cp0) : K(0);
        K ck1 = cp1 >= 0 ? FmKey<K>::make(gain[cp1], cp1) : K(0);
        int32_t cw0 = cp0 >= 0 ? w[cp0] : 0, cw1 = cp1 >= 0 ? w[cp1] : 0;
        __syncwarp();  // every lane has read the shared state before lane 0 rewrites it
        uint32_t refilled = static_cast<uint32_t>(need & 3);
        int32_t pf_tail = PF ? s_pf_tail : 0;
        // one move: lock ch, flip it, update the neighbours' gains and the caches
        auto apply = [&](K kbest, int32_t sd) {
          const int32_t ch = FmKey<K>::id(kbest);
          const int2 e = abe[ch];
          const uint32_t own = __ballot_sync(0xffffffffu, (sd ? cp1 : cp0) == ch);
          int32_t wc;
          if constexpr (SM) {
            wc = w[ch];
          } else {  // global weights: the cached copy of the lane holding ch
            const int32_t cwl = __shfl_sync(0xffffffffu, sd ? cw1 : cw0, own ? __ffs(own) - 1 : 0);
            wc = own ? cwl : w[ch];
          }
          if (own && lane == __ffs(own) - 1) {
            if (sd) cp1 = -1, ck1 = 0, cw1 = 0;
            else cp0 = -1, ck0 = 0, cw0 = 0;
          }
          if (lane == 0) {
            stv.set(ch, fm_st(1 - sd, 1, kNoSlot));
            moves[nm] = ch;
          }
          ++nm;
          sw0 += sd ? wc : -wc;
          sw1 += sd ? -wc : wc;
          cut -= FmKey<K>::gain(kbest);
          __syncwarp();
          // neighbours' gains (partition.cpp:137-142)
          const int32_t sc = 1 - sd;
          for (int32_t j0 = e.x; j0 < e.y; j0 += 32) {
            const int32_t j = j0 + lane;
            bool upd = false, ins = false;
            int32_t nb = 0, sn = 0;
            K nk = 0;
            if (j < e.y) {
              nb = A_nb(j);
              const int32_t wj = A_w(j);
              const uint32_t sw = stv.get(nb);
              if (!(sw & 0xff00u)) {  // unlocked
                sn = static_cast<int32_t>(sw & 1u);
                const int32_t g = gain[nb] + (sn == sc ? -2 * wj : 2 * wj);
                gain[nb] = g;
                nk = FmKey<K>::make(g, nb);
                upd = (sw >> 16) != kNoSlot;
                ins = !upd && nk > (sn ? B1 : B0);
              }
            }
            __syncwarp();
            if (__any_sync(0xffffffffu, upd)) {  // re-read the cached keys
              if (cp0 >= 0) ck0 = FmKey<K>::make(gain[cp0], cp0);
              if (cp1 >= 0) ck1 = FmKey<K>::make(gain[cp1], cp1);
            }
            uint32_t im = __ballot_sync(0xffffffffu, ins);
            while (im) {  // raised uncached keys above the bound join the cache
              const int l = __ffs(im) - 1;
              im &= im - 1;
              const K nbk = __shfl_sync(0xffffffffu, nk, l);
              const int32_t nbp = __shfl_sync(0xffffffffu, nb, l);
              const int32_t t = __shfl_sync(0xffffffffu, sn, l);
              const K ct = t ? ck1 : ck0;
              const uint32_t fr = __ballot_sync(0xffffffffu, ct == 0);
              int o;
              if (fr) {
                o = __ffs(fr) - 1;
              } else {
                const K mn = FmKey<K>::wmin(ct);
                if (nbk < mn) {  // below the whole cache: it only raises the bound
                  if (t) B1 = max(B1, nbk);
                  else B0 = max(B0, nbk);
                  continue;
                }
                o = __ffs(__ballot_sync(0xffffffffu, ct == mn)) - 1;
                if (t) B1 = max(B1, mn);
                else B0 = max(B0, mn);
                if (lane == o) stv.set_slot(t ? cp1 : cp0, kNoSlot);
              }
              if (lane == o) {
                const int32_t wq = w[nbp];
                if (t) ck1 = nbk, cp1 = nbp, cw1 = wq;
                else ck0 = nbk, cp0 = nbp, cw0 = wq;
                stv.set_slot(nbp, (t << 5) | o);
                if constexpr (PF) {
                  s_pf_ring[pf_tail & (kFmPfRing - 1)] = nbp;
                  s_pf_tail = pf_tail + 1;
                }
              }
              if constexpr (PF) ++pf_tail;
            }
            __syncwarp();
          }
          if (cut < best_cut || (cut == best_cut && fm_imb_less<EXACT>(sw0, sw1, best_s0, best_s1))) {
            best_cut = cut;
            best_len = nm;
            best_s0 = sw0, best_s1 = sw1;
          }
        };
        int32_t reason = 0;
        if (need & kFmExact) {
          const K e = s_exact;
          if (e == 0) reason = kFmDone;
          else apply(e, static_cast<int32_t>(side(FmKey<K>::id(e)))), refilled = 0;
        }
        while (!reason) {
          // feasibility of the cached entries
          const int32_t H = max(sw0, sw1), L = min(sw0, sw1);
          const bool f0 = (ck0 != 0) & (sw0 - cw0 > 0) & !fm_infeasible<EXACT>(sw0 - cw0, sw1 + cw0, H, L);
          const bool f1 = (ck1 != 0) & (sw1 - cw1 > 0) & !fm_infeasible<EXACT>(sw1 - cw1, sw0 + cw1, H, L);
          const K fk0 = FmKey<K>::wmax(f0 ? ck0 : K(0)), fk1 = FmKey<K>::wmax(f1 ? ck1 : K(0));
          const K best = max(fk0, fk1);
          const bool u0 = B0 != 0 && !(fk0 > B0) && B0 > best;
          const bool u1 = B1 != 0 && !(fk1 > B1) && B1 > best;
          if (u0 || u1) {  // a side's answer may lie outside its cache
            reason = ((u0 && (refilled & 1)) || (u1 && (refilled & 2))) ? kFmExact : (u0 ? 1 : 0) | (u1 ? 2 : 0);
            break;
          }
          if (best == 0) {
            reason = kFmDone;
            break;
          }
          refilled = 0;
          apply(best, fk1 == best ? 1 : 0);
        }
        s_cp[0][lane] = cp0, s_cp[1][lane] = cp1;
        if (lane == 0) {
          s_sw[0] = sw0, s_sw[1] = sw1, s_cut = cut, s_best_cut = best_cut;
          s_best_s[0] = best_s0, s_best_s[1] = best_s1;
          s_nm = nm, s_best_len = best_len;
          s_B[0] = B0, s_B[1] = B1;
          s_need = reason;
          if constexpr (PF) s_pf_done = seg_iter;
        }
      } else if (PF && wid == 1) {
        if constexpr (W16) fm_prefetch_helper<false>(abe, a.qloc, a.qw, nullptr, s_pf_ring, &s_pf_tail, &s_pf_done, seg_iter, pf_head);
        else fm_prefetch_helper<!SM>(abe, a.qloc, a.qw, w, s_pf_ring, &s_pf_tail, &s_pf_done, seg_iter, pf_head);
      }
      ++seg_iter;
      __syncthreads();
      if (s_need == kFmDone) break;
    }
    const int32_t nm = s_nm, bl = s_best_len;
    total_moves += nm;
    for (int32_t m = bl + threadIdx.x; m < nm; m += blockDim.x) stv.flip(moves[m]);
    __syncthreads();
    if (threadIdx.x == 0) {  // the state after the best prefix (partition.cpp:150-156)
      s_cut = s_best_cut;
      s_sw[0] = s_best_s[0];
      s_sw[1] = s_best_s[1];
      const bool improved = s_best_cut < s_pass_cut ||
                            (s_best_cut == s_pass_cut &&
                             fm_imb_less<EXACT>(s_best_s[0], s_best_s[1], s_pass_s[0], s_pass_s[1]));
      s_stop = improved ? 0 : 1;
    }
    __syncthreads();
    if (s_stop) break;
  }
  for (int32_t i = threadIdx.x; i < np; i += blockDim.x) a.side[pl[i]] = static_cast<uint8_t>(side(i));
  if (threadIdx.x == 0) atomicAdd(&a.stats[0], static_cast<unsigned long long>(total_moves));
}

// Shared-memory bytes of a node's FM state + packed adjacency (fm_node<SM>).
__host__ __device__ inline int64_t fm_node_smem(int64_t np, int64_t entries) {
  return ((20 * np + 15) & ~int64_t(15)) + 4 * entries + 16;
}
// Shared-memory bytes of a node's compact state (fm_node<SMC>).
__host__ __device__ inline int64_t fm_node_smem_compact(int64_t np) {
  return 2 * ((2 * np + 15) & ~int64_t(15)) + 16;
}
// ... and of the 5-byte compact state with 16-bit weights (fm_node<SMC, W16>).
__host__ __device__ inline int64_t fm_node_smem_compact_w16(int64_t np) {
  return 2 * ((2 * np + 15) & ~int64_t(15)) + ((np + 15) & ~int64_t(15)) + 16;
}

// EXACT: integer feasibility (n < 2^26).  32-bit keys imply < 65536 patches
// and edge weights < 32768, so a node whose state fits uses the packed
// shared-memory layout; 64-bit-key nodes always use the global layout.
// HYB: the level has a node whose adjacency does not fit but whose state
// does, or whose wide state does not fit but whose compact state does (a
// separate instantiation, so levels without one keep the smaller kernel).
template <class K, bool EXACT, bool HYB = false>
__global__ void __launch_bounds__(kFmThreads, 1) fm_kernel(LevelArgs a) {
  const int32_t li = blockIdx.x;
  if (!a.active[li]) return;
  const int32_t pbeg = a.poff[li], np = a.poff[li + 1] - pbeg;
  if constexpr (sizeof(K) == 4) {
    const int64_t e_node = (a.fm_fifo_off[li + 1] - a.fm_fifo_off[li]) - np;
    if (fm_node_smem(np, e_node) <= a.fm_smem_bytes) {
      fm_node<K, EXACT, true>(a, li, pbeg, np);
      return;
    }
    if constexpr (HYB) {
      if (fm_node_smem(np, 0) <= a.fm_smem_bytes) {  // state only; adjacency from L2
        fm_node<K, EXACT, true, false>(a, li, pbeg, np);
        return;
      }
      if (a.fm_w16 && fm_node_smem_compact_w16(np) <= a.fm_smem_bytes) {  // + 16-bit weights, byte status
        fm_node<K, EXACT, false, false, true, true>(a, li, pbeg, np);
        return;
      }
      if (fm_node_smem_compact(np) <= a.fm_smem_bytes) {  // 16-bit gains (32-bit keys: |gain| < 32768)
        fm_node<K, EXACT, false, false, true>(a, li, pbeg, np);
        return;
      }
    }
  }
  fm_node<K, EXACT, false>(a, li, pbeg, np);
}

// largest total quotient edge weight of a patch: bounds |gain| for the key width
// Largest weight of the level's alive patches (fm_node<SMC, W16> needs < 65536).
__global__ void max_alive_weight(int32_t na, const int32_t* plist, const int32_t* pw, int32_t* out) {
  int32_t m = 0;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) m = max(m, pw[plist[i]]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void fm_gain_bound(int32_t na, const int32_t* plist, const int32_t* qoff, const int32_t* qw, int32_t* out) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
    const int32_t p = plist[i];
    int64_t sum = 0;
    for (int32_t j = qoff[p]; j < qoff[p + 1]; ++j) sum += qw[j];
    atomicMax(out, static_cast<int32_t>(sum < 0x7fffffff ? sum : 0x7fffffff));
  }
}
__global__ void local_adjacency(int32_t U, const int32_t* qnbr, const int32_t* lidx, int32_t* qloc) {
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < U; j += gridDim.x * blockDim.x) qloc[j] = lidx[qnbr[j]];
}

// ---------------------------------------------------------------- super separator
// partition.cpp:165-185 plus refine's boundary counts (:212-214).
__global__ void super_pass(LevelArgs a) {
  for (int32_t li = blockIdx.y; li < a.width; li += gridDim.y) {
    if (!a.active[li]) continue;
    const int32_t s0 = a.seg_start[li], cnt = a.seg_cnt[li], node = a.first + li;
    int32_t nl = 0, nr = 0;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
      const int32_t u = a.vlist[s0 + i];
      const uint8_t su = a.side[a.assign[u]];
      uint8_t sup = 0;
      for (int32_t j = a.g.off[u]; j < a.g.off[u + 1] && !sup; ++j) {
        const int32_t v = a.g.nbr[j];
        if (a.node_of[v] == node && a.side[a.assign[v]] != su) sup = 1;
      }
      a.region[u] = static_cast<int8_t>(su);
      a.vside[u] = su;
      a.in_super[u] = sup;
      if (sup) (su == 0 ? nl : nr)++;
    }
    if (nl) atomicAdd(&a.bcount[2 * li], nl);
    if (nr) atomicAdd(&a.bcount[2 * li + 1], nr);
  }
}

// ---------------------------------------------------------------- refine (one CTA per node)
struct RefKey {
  uint64_t hi, lo;  // (new_size, new_imb bits, vertex) lexicographic
};
__device__ __forceinline__ bool ref_less(const RefKey& x, const RefKey& y) {
  return x.hi < y.hi || (x.hi == y.hi && x.lo < y.lo);
}
// refine_separator (partition.cpp:187-283).  The candidate list (every
// vertex that has been in the separator) lives in shared memory with, per
// entry, the vertex, its patch side, an in-separator flag and its pull count
// (neighbours in the opposite region), maintained incrementally: a move only
// changes the regions of the moved vertex and the vertices it pulls, so only
// their neighbours' counts change.  A candidate's new imbalance depends only on
// (side, pull), so the divisions are a per-move table (warp 0), and a move is
// a block argmin of (new size, new imbalance, vertex) over the entries.
// Per-vertex state is one byte of region (0/1 sides, 2 separator, 3 gone --
// dead vertices never count as neighbours) plus the vertex's patch side, so
// no node-membership lookups are needed; adjacency comes from the ELL copy.
constexpr int32_t kRefSmemList = 12 * 1024;  // candidate entries kept in shared memory (10 B each)
constexpr int32_t kRefSmemN = 4096;          // graphs up to this size refine with their state in shared memory

// Ordered compaction of [0, cnt) by the whole block: warp w owns the
// contiguous range [w * per, (w + 1) * per); pass 1 counts, pass 2 emits with
// ballot ranks.  One block-wide exchange instead of a block scan per 1024
// items (a 1M-vertex node is 1,000 scans).  classify(i) returns -1 (skip), 0
// or 1; emit(i, cls, rank within its class).  Returns the two class counts.
template <class Cls, class Emit>
__device__ __forceinline__ int2 block_ordered_split(int32_t cnt, int32_t* sh64, Cls classify, Emit emit) {
  constexpr int U = 8;  // 32-element groups per step: their loads are in flight together
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t per = (cnt + nw - 1) / nw;
  const int32_t lo = min(cnt, wid * per), hi = min(cnt, lo + per);
  int32_t c0 = 0, c1 = 0;
  for (int32_t i0 = lo; i0 < hi; i0 += 32 * U) {
    int c[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int32_t i = i0 + 32 * q + lane;
      c[q] = i < hi ? classify(i) : -1;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      c0 += __popc(__ballot_sync(0xffffffffu, c[q] == 0));
      c1 += __popc(__ballot_sync(0xffffffffu, c[q] == 1));
    }
  }
  if (lane == 0) sh64[wid] = c0, sh64[32 + wid] = c1;
  __syncthreads();
  int32_t b0 = 0, b1 = 0, t0 = 0, t1 = 0;
  for (int32_t w = 0; w < nw; ++w) {
    const int32_t x0 = sh64[w], x1 = sh64[32 + w];
    if (w < wid) b0 += x0, b1 += x1;
    t0 += x0, t1 += x1;
  }
  const uint32_t below = (1u << lane) - 1;
  for (int32_t i0 = lo; i0 < hi; i0 += 32 * U) {
    int c[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int32_t i = i0 + 32 * q + lane;
      c[q] = i < hi ? classify(i) : -1;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int32_t i = i0 + 32 * q + lane;
      const uint32_t m0 = __ballot_sync(0xffffffffu, c[q] == 0), m1 = __ballot_sync(0xffffffffu, c[q] == 1);
      if (c[q] == 0) emit(i, 0, b0 + __popc(m0 & below));
      if (c[q] == 1) emit(i, 1, b1 + __popc(m1 & below));
      b0 += __popc(m0), b1 += __popc(m1);
    }
  }
  __syncthreads();
  return make_int2(t0, t1);
}
constexpr int kRefTab = 16;  // pulls tabulated per side

__device__ __forceinline__ RefKey warp_min_ref(RefKey k) {
  // lexicographic (hi, lo) minimum in four 32-bit redux steps
  const uint32_t h1 = static_cast<uint32_t>(k.hi >> 32), h0 = static_cast<uint32_t>(k.hi);
  const uint32_t l1 = static_cast<uint32_t>(k.lo >> 32), l0 = static_cast<uint32_t>(k.lo);
  const uint32_t m1 = __reduce_min_sync(0xffffffffu, h1);
  const uint32_t m0 = __reduce_min_sync(0xffffffffu, h1 == m1 ? h0 : 0xffffffffu);
  const bool e1 = h1 == m1 && h0 == m0;
  const uint32_t n1 = __reduce_min_sync(0xffffffffu, e1 ? l1 : 0xffffffffu);
  const uint32_t n0 = __reduce_min_sync(0xffffffffu, e1 && l1 == n1 ? l0 : 0xffffffffu);
  return RefKey{(static_cast<uint64_t>(m1) << 32) | m0, (static_cast<uint64_t>(n1) << 32) | n0};
}

// Initial separator of every active node (partition.cpp:212-222: the smaller
// boundary, ties to the left), grid-wide over the level's vertices: members
// join the node's candidate list (global, slot order arbitrary -- the moves
// pick by key) and leave their region; the rest is counted per side.
__global__ void ref_init(LevelArgs a) {
  __shared__ int64_t red[32];
  const int lane = threadIdx.x & 31;
  for (int32_t li = blockIdx.y; li < a.width; li += gridDim.y) {
    if (!a.active[li]) continue;
    const int32_t s0 = a.seg_start[li], cnt = a.seg_cnt[li];
    const int8_t take = a.bcount[2 * li] <= a.bcount[2 * li + 1] ? 0 : 1;
    int32_t c0 = 0, c1 = 0;
    const int32_t w0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    for (int32_t i0 = w0; i0 < cnt; i0 += gridDim.x * blockDim.x) {
      const int32_t i = i0 + lane;
      const int32_t v = i < cnt ? a.vlist[s0 + i] : -1;
      const int8_t r = v >= 0 ? a.region[v] : int8_t(-1);
      const bool mem = v >= 0 && a.in_super[v] && r == take;
      const int32_t slot = warp_append(&a.ref_cnt[li], mem);
      if (mem) {
        a.sep_list[s0 + slot] = v;
        a.ref_own[s0 + slot] = static_cast<uint8_t>(take);
        a.ref_in[s0 + slot] = 1;
        a.slot_of[v] = slot;
        a.region[v] = 2;
      } else if (v >= 0) {
        (r == 0 ? c0 : c1)++;
      }
    }
    const int64_t t0 = block_sum_i64(c0, red), t1 = block_sum_i64(c1, red);
    if (threadIdx.x == 0) {
      if (t0) atomicAdd(&a.ref_rw[2 * li], static_cast<int32_t>(t0));
      if (t1) atomicAdd(&a.ref_rw[2 * li + 1], static_cast<int32_t>(t1));
    }
  }
}

// Split after refine: every vertex of an active node left in region 0 / 1
// moves to the left / right child (node_of, child counts); the stable radix
// sort that follows on key (node << 1 | side) packs the children's vertex
// lists in node order, ascending inside each (separator and leaf vertices
// get the drop key and sort past the end).
__global__ void split_classify(LevelArgs a, uint32_t* keys, uint32_t drop_key, int32_t* next_cnt) {
  __shared__ int64_t red[32];
  for (int32_t li = blockIdx.y; li < a.width; li += gridDim.y) {
    const int32_t s0 = a.seg_start[li], cnt = a.seg_cnt[li];
    const bool act = a.active[li] != 0;
    const int32_t node = a.first + li;
    int32_t c0 = 0, c1 = 0;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
      const int32_t v = a.vlist[s0 + i];
      const int8_t r = act ? a.region[v] : int8_t(3);
      if (r == 0 || r == 1) {
        keys[s0 + i] = (static_cast<uint32_t>(li) << 1) | static_cast<uint32_t>(r);
        a.node_of[v] = 2 * node + 1 + r;
        (r ? c1 : c0)++;
      } else {
        keys[s0 + i] = drop_key;
      }
    }
    if (act) {
      const int64_t t0 = block_sum_i64(c0, red), t1 = block_sum_i64(c1, red);
      if (threadIdx.x == 0) {
        if (t0) atomicAdd(&next_cnt[2 * li], static_cast<int32_t>(t0));
        if (t1) atomicAdd(&next_cnt[2 * li + 1], static_cast<int32_t>(t1));
      }
    }
  }
}

// SM: small graphs (n <= kRefSmemN) copy the per-vertex state the moves read
// -- ELL rows, list slots, regions, patch sides -- into shared memory, so a
// move's dependent loads are shared-memory round trips instead of L2 ones;
// the regions and slots of the list entries (every vertex a move touches)
// are written back at the end.
template <bool SM>
__global__ void __launch_bounds__(kNodeThreads) refine_kernel(LevelArgs a) {
  constexpr int32_t kCap = SM ? kRefSmemN : kRefSmemList;  // candidate entries kept in shared memory
  const int32_t li = blockIdx.x;
  const int32_t s0 = a.seg_start[li], cnt = a.seg_cnt[li];
  __shared__ int32_t shi[32];
  __shared__ RefKey sred[32];
  __shared__ int64_t s_rw[2], s_size;
  __shared__ double s_imb, s_ni[2][kRefTab];
  __shared__ int32_t s_list, s_mv, s_moves, s_pw[32];
  extern __shared__ int32_t ref_sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (!a.active[li]) return;  // no split (split_classify drops its vertices)
  // candidate list: shared memory while it fits (checked before every move;
  // a move adds at most one entry), the global scratch of the node otherwise
  bool in_smem;
  int32_t *lv, *lpull;
  uint8_t *lown, *lin;
  auto use_lists = [&](bool sm) {
    in_smem = sm;
    lv = sm ? ref_sm : a.sep_list + s0;
    lpull = sm ? ref_sm + kCap : a.ref_pull + s0;
    lown = sm ? reinterpret_cast<uint8_t*>(ref_sm + 2 * kCap) : a.ref_own + s0;
    lin = sm ? reinterpret_cast<uint8_t*>(ref_sm + 2 * kCap) + kCap : a.ref_in + s0;
  };
  int8_t* region = a.region;
  const int32_t* ell = a.ell;
  int32_t* slot_of = a.slot_of;
  const uint8_t* vside = a.vside;
  if constexpr (SM) {
    const int32_t n = a.g.n;
    int32_t* sell = ref_sm + (10 * kCap) / 4;  // after the candidate lists
    int32_t* sslot = sell + 8 * n;
    int8_t* sreg = reinterpret_cast<int8_t*>(sslot + n);
    uint8_t* sside = reinterpret_cast<uint8_t*>(sreg + n);
    for (int32_t i = threadIdx.x; i < 8 * n; i += blockDim.x) sell[i] = a.ell[i];
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
      sslot[i] = a.slot_of[i];
      sreg[i] = a.region[i];
      sside[i] = a.vside[i];
    }
    ell = sell, slot_of = sslot, region = sreg, vside = sside;
    __syncthreads();
  }

  // neighbour w of v through the ELL copy, slot k of a warp-uniform walk;
  // returns -1 past the end (the CSR tail serves vertices of degree > 8)
  auto nbr_at = [&](int32_t v, int32_t k) -> int32_t {
    if (k < 7) return ell[static_cast<int64_t>(v) * 8 + k];
    const int32_t x7 = ell[static_cast<int64_t>(v) * 8 + 7];
    if (x7 >= -1) return k == 7 ? x7 : -1;
    const int32_t j = -x7 - 2 + (k - 7);
    return j < a.g.off[v + 1] ? a.g.nbr[j] : -1;
  };
  auto degree = [&](int32_t v) { return a.g.off[v + 1] - a.g.off[v]; };

  // initial separator (ref_init): the list in the node's global scratch,
  // moved into shared memory when it fits
  {
    const int32_t run = a.ref_cnt[li];
    const int64_t r0 = a.ref_rw[2 * li], r1 = a.ref_rw[2 * li + 1];
    use_lists(run < kCap / 2);
    if (in_smem)
      for (int32_t k = threadIdx.x; k < run; k += blockDim.x) {
        lv[k] = a.sep_list[s0 + k];
        lown[k] = a.ref_own[s0 + k];
        lin[k] = 1;
      }
    if (threadIdx.x == 0) {
      s_list = run;
      s_size = run;
      s_rw[0] = r0, s_rw[1] = r1;
      s_imb = imbalance_of(r0, r1);
      s_moves = 0;
    }
    if (wid == 0) {  // imbalance table for the first move
      const int32_t own = lane >> 4, pull = lane & 15;
      const int64_t ro = own ? r1 : r0, rp = own ? r0 : r1;
      s_ni[own][pull] = imbalance_of(ro + 1, rp - pull);
    }
    __syncthreads();
    for (int32_t k = threadIdx.x; k < run; k += blockDim.x) {
      const int32_t v = lv[k];
      const int8_t opp = 1 - static_cast<int8_t>(lown[k]);
      int32_t pull = 0;
      for (int32_t j = a.g.off[v]; j < a.g.off[v + 1]; ++j) pull += region[a.g.nbr[j]] == opp;
      lpull[k] = pull;
    }
    __syncthreads();
  }
  // greedy moves (partition.cpp:235-274)
  for (;;) {
    if (in_smem && s_list >= kCap) {  // the list outgrew shared memory: move it to global
      int32_t* gv = a.sep_list + s0;
      int32_t* gp = a.ref_pull + s0;
      uint8_t* go = a.ref_own + s0;
      uint8_t* gi = a.ref_in + s0;
      for (int32_t i = threadIdx.x; i < s_list; i += blockDim.x) gv[i] = lv[i], gp[i] = lpull[i], go[i] = lown[i], gi[i] = lin[i];
      use_lists(false);
      __syncthreads();
    }
    const int64_t cur = s_size;
    const double cimb = s_imb;
    const double thr = kBalanceTol > cimb ? kBalanceTol : cimb;
    const int64_t rw0 = s_rw[0], rw1 = s_rw[1];
    const int32_t nl = s_list;
    RefKey best{~0ull, ~0ull};
    for (int32_t i = threadIdx.x; i < nl; i += blockDim.x) {
      if (lin[i] != 1) continue;
      const int32_t pull = lpull[i];
      const int64_t ns = cur - 1 + pull;
      if (ns > cur) continue;
      const uint8_t own = lown[i];
      const double ni = pull < kRefTab ? s_ni[own][pull]
                                       : imbalance_of((own ? rw1 : rw0) + 1, (own ? rw0 : rw1) - pull);
      if (ni > thr) continue;
      if (!(ns < cur || ni < cimb)) continue;
      const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(ni));
      const RefKey k{(static_cast<uint64_t>(ns) << 32) | (bits >> 32),
                     ((bits & 0xffffffffull) << 32) | static_cast<uint32_t>(lv[i])};
      if (ref_less(k, best)) best = k;
    }
    best = warp_min_ref(best);
    if (lane == 0) sred[wid] = best;
    __syncthreads();
    if (wid == 0) {
      RefKey k = lane < nwarps ? sred[lane] : RefKey{~0ull, ~0ull};
      k = warp_min_ref(k);
      const int32_t mv = k.hi == ~0ull ? -1 : static_cast<int32_t>(k.lo & 0xffffffffu);
      if (lane == 0) s_mv = mv;
      if (mv >= 0) {
        // mv's slot, its ELL row and its degree are independent loads
        const int32_t e_mv = lane < 8 ? ell[static_cast<int64_t>(mv) * 8 + lane] : -1;
        const int32_t im = slot_of[mv];
        const int32_t e7 = __shfl_sync(0xffffffffu, e_mv, 7);
        const int32_t dmv = e7 < -1 ? degree(mv) : 0;  // CSR tail: exact degree needed
        const int8_t own = static_cast<int8_t>(lown[im]), opp = 1 - own;
        int32_t np = 0;
        int32_t* pulled = a.ref_pulled + s0;
        if (e7 >= -1 || dmv <= 32) {
          // ---- fast path (degree <= 32): one neighbour per lane, three
          // dependent L2 round trips in all (mv's row; the neighbours' region /
          // slot / side / rows; the pulled vertices' neighbours' region / slot)
          int32_t w = -1;
          if (e7 >= -1) w = lane < 8 ? e_mv : -1;
          else if (lane < 7) w = e_mv;
          else {
            const int32_t j = -e7 - 2 + (lane - 7);
            w = j < a.g.off[mv + 1] ? a.g.nbr[j] : -1;
          }
          int32_t rw = 3, sw = -1;
          uint8_t vs = 0;
          int4 r0 = make_int4(-1, -1, -1, -1), r1 = r0;  // w's ELL row (used if w is pulled)
          if (w >= 0) {
            rw = region[w], sw = slot_of[w], vs = vside[w];
            const int4* row = reinterpret_cast<const int4*>(ell + static_cast<int64_t>(w) * 8);
            r0 = row[0], r1 = row[1];
          }
          const bool pull = rw == opp;
          const uint32_t m = __ballot_sync(0xffffffffu, pull);
          const bool fresh = pull && sw < 0;
          const uint32_t mf = __ballot_sync(0xffffffffu, fresh);
          np = __popc(m);
          // mv: 2 -> own raises the pull of separator neighbours whose opposite is own
          if (rw == 2 && lin[sw] == 1 && lown[sw] == opp) atomicAdd(&lpull[sw], 1);
          const int32_t tail = s_list;
          int32_t ws = sw;
          if (pull) s_pw[__popc(m & ((1u << lane) - 1))] = w;
          __syncwarp();
          if (pull) {
            region[w] = 2;
            if (fresh) {
              ws = tail + __popc(mf & ((1u << lane) - 1));
              lv[ws] = w;
              lown[ws] = vs;
              slot_of[w] = ws;
            }
            lin[ws] = 2;  // 2 = pulled by this move
          }
          // pulled w (opp -> 2): its own pull count and the separator neighbours
          // on side `own` it no longer pulls.  Region values are as after this
          // move: mv is `own`, every pulled vertex is 2 (corrected in registers).
          int32_t cntp = 0;
          if (pull) {
            const int8_t wopp = static_cast<int8_t>(1 - vs);
            const int32_t xs[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            int8_t rx[8];
            int32_t ix[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int32_t x = xs[k];
              rx[k] = x >= 0 ? region[x] : int8_t(3);
              ix[k] = x >= 0 ? slot_of[x] : -1;
            }
            auto visit = [&](int32_t x, int8_t r, int32_t slot) {
              if (x == mv) r = own;
              else if (r == opp)  // was it pulled by this move? (then it is 2 now)
                for (int32_t t = 0; t < np; ++t)
                  if (s_pw[t] == x) r = 2, slot = -1;
              cntp += r == wopp;
              if (r == 2 && slot >= 0 && lin[slot] == 1 && lown[slot] == own) atomicSub(&lpull[slot], 1);
            };
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (k < 7 || xs[7] >= -1)
                if (xs[k] >= 0) visit(xs[k], rx[k], ix[k]);
            if (xs[7] < -1)  // CSR tail of a pulled vertex with more than 8 neighbours
              for (int32_t j = -xs[7] - 2; j < a.g.off[w + 1]; ++j) {
                const int32_t x = a.g.nbr[j];
                visit(x, region[x], slot_of[x]);
              }
            lpull[ws] = cntp;
          }
          __syncwarp();
          if (pull) lin[ws] = 1;
          if (lane == 0) {
            region[mv] = own;
            lin[im] = 0;
            s_list = tail + __popc(mf);
          }
        } else {
        // ---- general path (degree > 32)
        // 1. pull mv's opposite-region neighbours into the separator
        int32_t tail = s_list;
        for (int32_t k0 = 0; k0 < dmv; k0 += 32) {
          const int32_t w = k0 + lane < dmv ? nbr_at(mv, k0 + lane) : -1;
          const bool pull = w >= 0 && region[w] == opp;
          const uint32_t m = __ballot_sync(0xffffffffu, pull);
          const bool fresh = pull && slot_of[w] < 0;
          const uint32_t mf = __ballot_sync(0xffffffffu, fresh);
          if (pull) {
            region[w] = 2;
            pulled[np + __popc(m & ((1u << lane) - 1))] = w;
          }
          if (fresh) {
            const int32_t k2 = tail + __popc(mf & ((1u << lane) - 1));
            lv[k2] = w;
            lown[k2] = vside[w];
            slot_of[w] = k2;
          }
          tail += __popc(mf);
          np += __popc(m);
        }
        __syncwarp();
        for (int32_t t = lane; t < np; t += 32) lin[slot_of[pulled[t]]] = 2;  // 2 = pulled by this move
        if (lane == 0) {
          region[mv] = own;
          lin[im] = 0;
          s_list = tail;
        }
        __syncwarp();
        // 2a. mv: 2 -> own raises the pull of separator neighbours whose opposite is own
        for (int32_t k0 = 0; k0 < dmv; k0 += 32) {
          const int32_t x = k0 + lane < dmv ? nbr_at(mv, k0 + lane) : -1;
          if (x >= 0 && region[x] == 2) {
            const int32_t ix = slot_of[x];
            if (lin[ix] == 1 && lown[ix] == opp) atomicAdd(&lpull[ix], 1);
          }
        }
        // 2b/3. every pulled w (opp -> 2): (w, slot) pairs across the warp
        for (int32_t t0 = 0; t0 < np; t0 += 4) {
          const int32_t t = t0 + (lane >> 3);
          const int32_t wv = t < np ? pulled[t] : -1;
          const int32_t dw = wv >= 0 ? degree(wv) : 0;
          const uint8_t wopp = wv >= 0 ? static_cast<uint8_t>(1 - vside[wv]) : 0;
          int32_t cntp = 0;
          for (int32_t k = (lane & 7); k < dw; k += 8) {
            const int32_t x = nbr_at(wv, k);
            if (x < 0) continue;
            const int8_t rx = region[x];
            cntp += rx == wopp;
            if (rx == 2) {
              const int32_t ix = slot_of[x];
              if (lin[ix] == 1 && lown[ix] == own) atomicSub(&lpull[ix], 1);
            }
          }
          // fresh pull count of wv: sum over its 8-lane group
          cntp += __shfl_xor_sync(0xffffffffu, cntp, 1);
          cntp += __shfl_xor_sync(0xffffffffu, cntp, 2);
          cntp += __shfl_xor_sync(0xffffffffu, cntp, 4);
          if (wv >= 0 && (lane & 7) == 0) lpull[slot_of[wv]] = cntp;
        }
        __syncwarp();
        for (int32_t t = lane; t < np; t += 32) lin[slot_of[pulled[t]]] = 1;
        }
        const int64_t nrw0 = s_rw[0] + (own == 0 ? 1 : -np), nrw1 = s_rw[1] + (own == 1 ? 1 : -np);
        // imbalance table of the next move
        {
          const int32_t o2 = lane >> 4, pull = lane & 15;
          const int64_t ro = o2 ? nrw1 : nrw0, rp = o2 ? nrw0 : nrw1;
          s_ni[o2][pull] = imbalance_of(ro + 1, rp - pull);
        }
        __syncwarp();  // every lane has read s_rw / s_size
        if (lane == 0) {
          s_rw[0] = nrw0, s_rw[1] = nrw1;
          s_size = s_size - 1 + np;
          s_imb = imbalance_of(nrw0, nrw1);
          ++s_moves;
        }
      }
    }
    __syncthreads();
    if (s_mv < 0) break;
  }
  // the separator stays at `node` and leaves play (region 3); split_classify
  // moves the sides to the children
  for (int32_t i = threadIdx.x; i < s_list; i += blockDim.x) {
    const int32_t v = lv[i];
    slot_of[v] = -1;
    if (region[v] == 2) region[v] = 3;  // the separator leaves the game
    if constexpr (SM) a.slot_of[v] = -1, a.region[v] = region[v];
  }
  if (threadIdx.x == 0) atomicAdd(&a.stats[1], static_cast<unsigned long long>(s_moves));
}

template <class T>
void cub_sort_keys(const T* in, T* out, int64_t n, int end_bit, cudaStream_t s) {
  size_t tmp = 0;
  MP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, in, out, n, 0, end_bit, s));
  DevBuf<char> t(tmp, s);
  MP_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, in, out, n, 0, end_bit, s));
}

int bits_for(int64_t x) {
  int b = 1;
  while ((1LL << b) <= x) ++b;
  return b;
}

// Per-patch quotient CSR of the crossing-edge keys (sorted, run-length
// encoded): qoff (P+1), qnbr, qw.  Returns the number of directed entries.
int64_t quotient_from_keys(mp_context& ctx, uint64_t* keys, int64_t nkeys, int32_t P, DevBuf<int32_t>& qoff,
                           DevBuf<int32_t>& qnbr, DevBuf<int32_t>& qw) {
  cudaStream_t s = ctx.stream;
  DevBuf<uint64_t> sorted(std::max<int64_t>(nkeys, 1), s), ukeys(std::max<int64_t>(nkeys, 1), s);
  DevBuf<int32_t> ucnt(std::max<int64_t>(nkeys, 1), s), nruns(1, s), qdeg(P + 1, s);
  MP_CUDA(cudaMemsetAsync(qdeg, 0, sizeof(int32_t) * (P + 1), s));
  int32_t U = 0;
  if (nkeys > 0) {
    const int pb = bits_for(P);
    cub_sort_keys(keys, sorted.get(), nkeys, 32 + pb, s);
    size_t tmp = 0;
    MP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp, sorted.get(), ukeys.get(), ucnt.get(), nruns.get(),
                                               nkeys, s));
    DevBuf<char> t(tmp, s);
    MP_CUDA(cub::DeviceRunLengthEncode::Encode(t.get(), tmp, sorted.get(), ukeys.get(), ucnt.get(), nruns.get(),
                                               nkeys, s));
    MP_CUDA(cudaMemcpyAsync(&U, nruns.get(), 4, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
  }
  qoff.alloc(P + 1, s);
  qnbr.alloc(std::max(U, 1), s);
  qw.alloc(std::max(U, 1), s);
  if (U > 0)
    MP_KERNEL(ctx, quotient_csr<<<grid_for(ctx, U), 256, 0, s>>>(U, ukeys, ucnt, qdeg, qnbr, qw));
  size_t tmp = 0;
  MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, qdeg.get(), qoff.get(), P + 1, s));
  DevBuf<char> t(tmp, s);
  MP_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, qdeg.get(), qoff.get(), P + 1, s));
  return U;
}

// node_offsets from the node-sorted keys: the run boundary between keys
// kout[i-1] < kout[i] starts every node in (kout[i-1], kout[i]] at i (empty
// nodes included); the ends of the key range fill the rest.
__global__ void node_bounds(int32_t n, int64_t nn, const int32_t* kout, int32_t* node_offsets) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
    const int64_t lo = i == 0 ? 0 : static_cast<int64_t>(kout[i - 1]) + 1;
    const int64_t hi = i == n ? nn : static_cast<int64_t>(kout[i]);
    for (int64_t x = lo; x <= hi; ++x) node_offsets[x] = i;
  }
}

__global__ void count_weights_all(int32_t n, const int32_t* assign, int32_t* pw) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    atomicAdd(&pw[assign[v]], 1);
}
__global__ void emit_crossing_all(DGraph g, const int32_t* assign, uint64_t* keys, int32_t* count) {
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < g.n; u += gridDim.x * blockDim.x) {
    const int32_t pu = assign[u];
    for (int32_t j = g.off[u]; j < g.off[u + 1]; ++j) {
      const int32_t v = g.nbr[j];
      if (v <= u) continue;
      const int32_t pv = assign[v];
      if (pv == pu) continue;
      int32_t lo = min(pu, pv), hi = max(pu, pv);
      keys[atomicAdd(count, 1)] = (static_cast<uint64_t>(lo) << 32) | static_cast<uint32_t>(hi);
    }
  }
}
__global__ void check_assign(int32_t n, const int32_t* assign, int32_t P, int32_t* bad) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (assign[v] < 0 || assign[v] >= P) atomicMin(bad, v);
}
__global__ void split_keys(int32_t U, const uint64_t* k, const int32_t* c, int32_t* ep, int32_t* eq,
                           int64_t* ew) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < U; i += gridDim.x * blockDim.x) {
    ep[i] = static_cast<int32_t>(k[i] >> 32);
    eq[i] = static_cast<int32_t>(k[i] & 0xffffffffu);
    ew[i] = c[i];
  }
}
__global__ void widen(int32_t P, const int32_t* a, int64_t* b) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) b[i] = a[i];
}

void validate_assignment(mp_context& ctx, int32_t n, const int32_t* assign, int32_t P) {
  cudaStream_t s = ctx.stream;
  DevBuf<int32_t> bad(1, s);
  MP_KERNEL(ctx, fill32<<<1, 32, 0, s>>>(1, bad, 0x7fffffff));
  MP_KERNEL(ctx, check_assign<<<grid_for(ctx, n), 256, 0, s>>>(n, assign, P, bad));
  int32_t h;
  MP_CUDA(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (h != 0x7fffffff) {
    int32_t pv = 0;
    MP_CUDA(cudaMemcpy(&pv, assign + h, 4, cudaMemcpyDeviceToHost));
    throw Error(MP_EINVAL, "patch id " + std::to_string(pv) + " out of range for vertex " + std::to_string(h));
  }
}

}  // namespace

int64_t build_quotient_dev(mp_context& ctx, const DGraph& g, const int32_t* assign, int32_t P,
                           int64_t* node_weight, int32_t** edge_p, int32_t** edge_q, int64_t** edge_w) {
  cudaStream_t s = ctx.stream;
  validate_assignment(ctx, g.n, assign, P);
  DevBuf<int32_t> pw(std::max(P, 1), s), cnt(1, s);
  MP_CUDA(cudaMemsetAsync(pw, 0, sizeof(int32_t) * std::max(P, 1), s));
  MP_KERNEL(ctx, count_weights_all<<<grid_for(ctx, g.n), 256, 0, s>>>(g.n, assign, pw));
  if (P > 0) MP_KERNEL(ctx, widen<<<grid_for(ctx, P), 256, 0, s>>>(P, pw, node_weight));
  int32_t m2 = 0;
  MP_CUDA(cudaMemcpyAsync(&m2, g.off + g.n, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  DevBuf<uint64_t> keys(std::max(m2 / 2, 1), s), sorted(std::max(m2 / 2, 1), s), uk(std::max(m2 / 2, 1), s);
  DevBuf<int32_t> uc(std::max(m2 / 2, 1), s), nr(1, s);
  MP_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
  MP_KERNEL(ctx, emit_crossing_all<<<grid_for(ctx, g.n), 256, 0, s>>>(g, assign, keys, cnt));
  int32_t nk = 0;
  MP_CUDA(cudaMemcpyAsync(&nk, cnt, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  int32_t U = 0;
  if (nk > 0) {
    cub_sort_keys(keys.get(), sorted.get(), nk, 32 + bits_for(P), s);
    size_t tmp = 0;
    MP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp, sorted.get(), uk.get(), uc.get(), nr.get(), nk, s));
    DevBuf<char> t(tmp, s);
    MP_CUDA(cub::DeviceRunLengthEncode::Encode(t.get(), tmp, sorted.get(), uk.get(), uc.get(), nr.get(), nk, s));
    MP_CUDA(cudaMemcpyAsync(&U, nr.get(), 4, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
  }
  if (edge_p) {
    MP_CUDA(dev_malloc_async(reinterpret_cast<void**>(edge_p), sizeof(int32_t) * std::max(U, 1), s));
    MP_CUDA(dev_malloc_async(reinterpret_cast<void**>(edge_q), sizeof(int32_t) * std::max(U, 1), s));
    MP_CUDA(dev_malloc_async(reinterpret_cast<void**>(edge_w), sizeof(int64_t) * std::max(U, 1), s));
    if (U > 0) MP_KERNEL(ctx, split_keys<<<grid_for(ctx, U), 256, 0, s>>>(U, uk, uc, *edge_p, *edge_q, *edge_w));
  }
  return U;
}

// Level-k subtrees dealt to ranks: largest first (vertex count of the
// level-k node = the whole subtree), each to the least-loaded rank (ties:
// lower rank, then lower node id).  Deterministic from the tree alone.
std::vector<int32_t> deal_subtrees(const std::vector<int64_t>& root_size, int32_t k, int32_t L, int32_t world) {
  const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
  const int32_t first = (1 << k) - 1, width = 1 << k;
  std::vector<int32_t> owner(nn, -1), order(width);
  for (int32_t j = 0; j < width; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return root_size[x] > root_size[y]; });
  std::vector<int64_t> load(world, 0);
  for (int32_t j : order) {
    const int32_t dst = static_cast<int32_t>(std::min_element(load.begin(), load.end()) - load.begin());
    load[dst] += root_size[j];
    // the whole subtree of root first+j
    std::vector<int32_t> st{first + j};
    while (!st.empty()) {
      const int32_t i = st.back();
      st.pop_back();
      if (i >= nn) continue;
      owner[i] = dst;
      st.push_back(2 * i + 1), st.push_back(2 * i + 2);
    }
  }
  return owner;
}

void build_etree_dev(mp_context& ctx, const DGraph& g, const int32_t* assign, int32_t P, int32_t L,
                     int32_t* node_of, int32_t* node_offsets, int32_t* node_vertices, ShardSpec* shard) {
  if (L < 0 || L > kMaxNdLevel) throw Error(MP_EINVAL, "nd_level out of range");
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  const int64_t nn = (1LL << (L + 1)) - 1;
  validate_assignment(ctx, n, assign, P);
  int32_t m2 = 0;
  if (n > 0) {
    MP_CUDA(cudaMemcpyAsync(&m2, g.off + n, 4, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
  }
  const int32_t Pm = std::max(P, 1);
  DevBuf<int32_t> vl_a(std::max(n, 1), s), vl_b(std::max(n, 1), s), seplist(std::max(n, 1), s);
  DevBuf<int32_t> pw(Pm, s), pnode(Pm, s), lidx(Pm, s), flag(Pm, s), pkey(Pm, s), pkey_out(Pm, s);
  DevBuf<int32_t> alive_p(Pm, s), plist(Pm, s), fm_gain(Pm, s), fm_moves(Pm, s), cnt(4, s);
  DevBuf<unsigned long long> stats(2, s);
  DevBuf<int32_t> fm_w(Pm, s), fm_ab(2LL * Pm, s), fm_ae(1, s);
  DevBuf<uint8_t> fm_side(4LL * Pm, s);
  DevBuf<int32_t> slot_of(std::max(n, 1), s), ref_pull(std::max(n, 1), s), ref_pulled(std::max(n, 1), s);
  DevBuf<uint8_t> ref_own(std::max(n, 1), s), ref_in(std::max(n, 1), s);
  DevBuf<int8_t> region(std::max(n, 1), s);
  DevBuf<uint8_t> in_super(std::max(n, 1), s), in_list(std::max(n, 1), s), side(Pm, s);
  DevBuf<uint64_t> keys(std::max(m2, 1), s);
  MP_CUDA(cudaMemsetAsync(in_list, 0, std::max(n, 1), s));
  MP_CUDA(cudaMemsetAsync(region, 3, std::max(n, 1), s));  // 3 = not in play
  DevBuf<uint8_t> vside(std::max(n, 1), s);
  DevBuf<uint32_t> split_keys(std::max(n, 1), s), split_keys_out(std::max(n, 1), s);
  DevBuf<int32_t> ell(8LL * std::max(n, 1), s);
  if (n > 0) MP_KERNEL(ctx, build_ell_nd<<<grid_for(ctx, n), 256, 0, s>>>(g, ell));
  MP_CUDA(cudaMemsetAsync(stats, 0, 16, s));
  MP_KERNEL(ctx, fill32<<<grid_for(ctx, n), 256, 0, s>>>(n, node_of, 0));
  MP_KERNEL(ctx, fill32<<<grid_for(ctx, n), 256, 0, s>>>(n, slot_of, -1));
  MP_KERNEL(ctx, iota32<<<grid_for(ctx, n), 256, 0, s>>>(n, vl_a));

  // level-node segment tables (host-built for the root, device afterwards)
  int32_t width = 1;
  DevBuf<int32_t> seg_start(1, s), seg_cnt(1, s);
  MP_CUDA(cudaMemsetAsync(seg_start, 0, 4, s));
  MP_CUDA(cudaMemcpyAsync(seg_cnt.get(), &n, 4, cudaMemcpyHostToDevice, s));
  int32_t* cur_list = vl_a.get();
  int32_t* nxt_list = vl_b.get();
  DevBuf<uint8_t> own_mask;  // sharded build: set at the shard level
  if (shard) shard->owner.assign(nn, -1);

  SectionTimer st(s, "etree");
  st.mark("setup");
  for (int32_t level = 0; level < L && n > 0; ++level) {
    const int32_t first = (1 << level) - 1;
    int32_t na_level = 0;
    DevBuf<int32_t> np_node(width, s), active(width, s), poff(width + 1, s), bcount(2 * width, s),
        next_start(2 * width, s), next_cnt(2 * width, s);
    DevBuf<int64_t> fifo_off(width + 1, s);
    MP_CUDA(cudaMemsetAsync(pw, 0, sizeof(int32_t) * Pm, s));
    MP_CUDA(cudaMemsetAsync(np_node, 0, sizeof(int32_t) * width, s));
    MP_CUDA(cudaMemsetAsync(bcount, 0, sizeof(int32_t) * 2 * width, s));
    MP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * 4, s));
    LevelArgs a{};
    a.g = g, a.assign = assign, a.P = P, a.first = first, a.width = width;
    a.vlist = cur_list, a.seg_start = seg_start, a.seg_cnt = seg_cnt, a.node_of = node_of;
    a.pw = pw, a.pnode = pnode, a.np_node = np_node, a.active = active, a.lidx = lidx;
    a.side = side, a.region = region, a.in_super = in_super, a.in_list = in_list, a.bcount = bcount;
    a.sep_list = seplist, a.next_vlist = nxt_list, a.next_start = next_start, a.next_cnt = next_cnt;
    a.fm_w = fm_w, a.fm_ab = fm_ab, a.fm_ae = fm_ae, a.fm_side = fm_side;
    a.slot_of = slot_of, a.ref_pull = ref_pull, a.ref_own = ref_own, a.ref_in = ref_in, a.ref_pulled = ref_pulled;
    a.vside = vside, a.ell = ell;
    a.stats = ctx.dwork ? ctx.dwork + 1 : stats.get(), a.fm_gain = fm_gain, a.fm_moves = fm_moves;
    const dim3 lgrid(std::max(1, grid_for(ctx, n) / std::max(1, width)), std::min(width, 65535));
    if (shard && level == shard->k && shard->world > 1) {
      // the shard level: deal the level-k subtrees by their vertex counts
      std::vector<int32_t> hc(width);
      MP_CUDA(cudaMemcpyAsync(hc.data(), seg_cnt.get(), sizeof(int32_t) * width, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
      shard->owner = deal_subtrees(std::vector<int64_t>(hc.begin(), hc.end()), level, L, shard->world);
      std::vector<uint8_t> hm(nn);
      for (int64_t i = 0; i < nn; ++i) hm[i] = shard->owner[i] < 0 || shard->owner[i] == shard->rank;
      own_mask.alloc(nn, s);
      MP_CUDA(cudaMemcpyAsync(own_mask.get(), hm.data(), nn, cudaMemcpyHostToDevice, s));
      MP_CUDA(cudaStreamSynchronize(s));
    }
    a.own_mask = own_mask.get();
    MP_KERNEL(ctx, level_weights<<<lgrid, 256, 0, s>>>(a));
    MP_KERNEL(ctx, level_patch_counts<<<grid_for(ctx, P), 256, 0, s>>>(a));
    MP_KERNEL(ctx, level_activity<<<grid_for(ctx, width), 256, 0, s>>>(a, L, level, cnt.get()));
    // alive patches of active nodes, grouped by node, ascending
    if (P <= kSmallP) {
      MP_KERNEL(ctx, level_lists_small<<<1, 1024, 0, s>>>(P, width, pw, pnode, np_node, active, plist, poff, lidx,
                                                           cnt));
      int32_t hc[2];
      MP_CUDA(cudaMemcpyAsync(hc, cnt.get(), 8, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
      if (hc[0] == 0) break;  // no active node at this level: the tree is complete
      na_level = hc[1];
    } else {
    MP_KERNEL(ctx, flag_alive_patches<<<grid_for(ctx, P), 256, 0, s>>>(P, pw, pnode, active, flag, pkey));
    {
      DevBuf<int32_t> ids(Pm, s), sel(Pm, s), selkey(Pm, s);
      MP_KERNEL(ctx, iota32<<<grid_for(ctx, P), 256, 0, s>>>(P, ids));
      size_t tmp = 0;
      MP_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, ids.get(), flag.get(), sel.get(), cnt.get() + 1, P, s));
      DevBuf<char> t(tmp, s);
      MP_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, ids.get(), flag.get(), sel.get(), cnt.get() + 1, P, s));
      MP_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, pkey.get(), flag.get(), selkey.get(), cnt.get() + 2, P, s));
      DevBuf<char> t2(tmp, s);
      MP_CUDA(cub::DeviceSelect::Flagged(t2.get(), tmp, pkey.get(), flag.get(), selkey.get(), cnt.get() + 2, P, s));
      int32_t hc[2];
      MP_CUDA(cudaMemcpyAsync(hc, cnt.get(), 8, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
      if (hc[0] == 0) break;  // no active node at this level: the tree is complete
      const int32_t na = hc[1];
      // stable radix sort by node keeps ascending patch ids inside each node
      size_t tmp2 = 0;
      const int nb = bits_for(width);
      MP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, selkey.get(), pkey_out.get(), sel.get(), plist.get(),
                                              na, 0, nb, s));
      DevBuf<char> t3(tmp2, s);
      MP_CUDA(cub::DeviceRadixSort::SortPairs(t3.get(), tmp2, selkey.get(), pkey_out.get(), sel.get(), plist.get(),
                                              na, 0, nb, s));
      // poff: exclusive scan of np_node masked by activity
      DevBuf<int32_t> npm(width + 1, s);
      MP_KERNEL(ctx, masked_counts<<<grid_for(ctx, width + 1), 256, 0, s>>>(width, active, np_node, npm));
      size_t tmp3 = 0;
      MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp3, npm.get(), poff.get(), width + 1, s));
      DevBuf<char> t4(tmp3, s);
      MP_CUDA(cub::DeviceScan::ExclusiveSum(t4.get(), tmp3, npm.get(), poff.get(), width + 1, s));
      na_level = na;
      MP_KERNEL(ctx, set_lidx<<<grid_for(ctx, na), 256, 0, s>>>(na, plist, pnode, poff, lidx));
    }
    }
    a.plist = plist, a.poff = poff;
    st.mark("level/patches");
    // quotient of the alive vertices, per node
    MP_CUDA(cudaMemsetAsync(cnt.get() + 3, 0, 4, s));
    MP_KERNEL(ctx, emit_crossing<<<lgrid, 256, 0, s>>>(a, keys, cnt.get() + 3));
    int32_t nkeys = 0;
    MP_CUDA(cudaMemcpyAsync(&nkeys, cnt.get() + 3, 4, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    DevBuf<int32_t> qoff, qnbr, qw, qloc;
    int64_t U = 0;  // quotient entries (an upper bound on the small path: the key count)
    const bool small_q = nkeys <= kSmallKeys && P <= kSmallP && width <= 1024;
    if (small_q) {
      U = nkeys;
      qoff.alloc(P + 1, s);
      qnbr.alloc(std::max<int64_t>(U, 1), s);
      qw.alloc(std::max<int64_t>(U, 1), s);
      qloc.alloc(std::max<int64_t>(U, 1), s);
      const size_t qs = sizeof(uint64_t) * kSmallKeys + sizeof(int32_t) * (kSmallKeys + 1 + kSmallP + 1 + 1025);
      allow_max_smem(quotient_small, ctx.device);
      MP_KERNEL(ctx, quotient_small<<<1, 1024, qs, s>>>(nkeys, keys, P, width, na_level, plist, pnode, lidx, qoff, qnbr,
                                                        qw, qloc, fifo_off));
    } else {
      U = quotient_from_keys(ctx, keys, nkeys, P, qoff, qnbr, qw);
    }
    a.qoff = qoff, a.qnbr = qnbr, a.qw = qw;
    // fifo slab per node: every push follows a directed quotient entry of the
    // node, so its entries + 1 bound the pushes (partition.cpp:76-77)
    if (!small_q) {
      DevBuf<int64_t> ecnt(width + 1, s);
      MP_CUDA(cudaMemsetAsync(ecnt, 0, sizeof(int64_t) * (width + 1), s));
      if (na_level > 0)
        MP_KERNEL(ctx, node_edge_count<<<grid_for(ctx, na_level), 256, 0, s>>>(na_level, plist, pnode, qoff, ecnt));
      size_t tmp = 0;
      MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, ecnt.get(), fifo_off.get(), width + 1, s));
      DevBuf<char> t(tmp, s);
      MP_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, ecnt.get(), fifo_off.get(), width + 1, s));
    }
    DevBuf<int32_t> fifo(U + na_level + 1, s);
    a.fm_fifo = fifo, a.fm_fifo_off = fifo_off;
    st.mark("level/quotient");
    // bipartition per node
    const int32_t maxnp = na_level;
    if (!small_q) {
      qloc.alloc(std::max<int64_t>(U, 1), s);
      if (U > 0)
        MP_KERNEL(ctx, local_adjacency<<<grid_for(ctx, U), 256, 0, s>>>(static_cast<int32_t>(U), qnbr, lidx, qloc));
    }
    a.qloc = qloc;
    size_t fm_smem = 1024;
    bool fm_hybrid = false;  // a node whose state fits shared memory but whose adjacency does not
    bool fm_w16 = false;     // every alive patch weight fits 16 bits
    {
      // opt-in limit minus the kernels' static shared memory
      cudaFuncAttributes fa32{}, fa64{}, fah{};
      MP_CUDA(cudaFuncGetAttributes(&fa32, fm_kernel<uint32_t, true>));
      MP_CUDA(cudaFuncGetAttributes(&fa64, fm_kernel<uint64_t, false>));
      MP_CUDA(cudaFuncGetAttributes(&fah, fm_kernel<uint32_t, true, true>));
      const size_t cap = static_cast<size_t>(ctx.smem_optin) -
                         std::max({fa32.sharedSizeBytes, fa64.sharedSizeBytes, fah.sharedSizeBytes});
      // every node holds at most the level's alive patches and quotient
      // entries: when that bound fits, no per-node sizes are read back
      const size_t bound = static_cast<size_t>(fm_node_smem(na_level, U));
      if (bound <= cap) {
        fm_smem = std::max(fm_smem, bound);
      } else {
        // room for the packed adjacency of the largest node that fits
        std::vector<int64_t> hfo(width + 1);
        std::vector<int32_t> hpo(width + 1);
        DevBuf<int32_t> dmaxw(1, s);
        int32_t hmaxw = 0;
        MP_CUDA(cudaMemsetAsync(dmaxw, 0, 4, s));
        if (na_level > 0)
          MP_KERNEL(ctx, max_alive_weight<<<grid_for(ctx, na_level), 256, 0, s>>>(na_level, plist, a.pw, dmaxw));
        MP_CUDA(cudaMemcpyAsync(hfo.data(), fifo_off.get(), sizeof(int64_t) * (width + 1), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaMemcpyAsync(hpo.data(), poff.get(), sizeof(int32_t) * (width + 1), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaMemcpyAsync(&hmaxw, dmaxw.get(), 4, cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        fm_w16 = hmaxw < 65536;
        size_t need = 0;
        bool partial = false;  // some node fits only as state or compact state
        for (int32_t i = 0; i < width; ++i) {
          const int64_t np_i = hpo[i + 1] - hpo[i];
          if (np_i == 0) continue;
          const size_t full = static_cast<size_t>(fm_node_smem(np_i, (hfo[i + 1] - hfo[i]) - np_i));
          need = std::max(need, full);
          partial |= full > cap && static_cast<size_t>(fm_node_smem_compact(np_i)) <= cap;
        }
        fm_smem = partial ? cap : std::min<size_t>(std::max(fm_smem, need), cap);
        fm_hybrid = partial;
      }
    }
    a.fm_smem_bytes = static_cast<int64_t>(fm_smem);
    a.fm_w16 = fm_w16 ? 1 : 0;
    // 32-bit move keys when every node fits (patch count and gain range)
    // (a patch's quotient weight is at most the level's crossing entries)
    int32_t hgb = nkeys;
    if (nkeys >= 32768) {
      DevBuf<int32_t> gb(1, s);
      MP_CUDA(cudaMemsetAsync(gb, 0, 4, s));
      if (na_level > 0) MP_KERNEL(ctx, fm_gain_bound<<<grid_for(ctx, na_level), 256, 0, s>>>(na_level, plist, qoff, qw, gb));
      MP_CUDA(cudaMemcpyAsync(&hgb, gb.get(), 4, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
    }
    const bool k32 = maxnp < 65536 && hgb < 32768;
    const bool exact = n < kFmExactWeights;  // node weights < 2^26: integer feasibility
    auto launch_fm = [&](auto kernel) {
      allow_max_smem(kernel, ctx.device);
      const int kt__ = ctx.ktime_begin(kKFm);
      MP_KERNEL(ctx, kernel<<<width, kFmThreads, fm_smem, s>>>(a));
      ctx.ktime_end(kt__);
    };
    if (k32 && fm_hybrid) exact ? launch_fm(fm_kernel<uint32_t, true, true>) : launch_fm(fm_kernel<uint32_t, false, true>);
    else if (k32) exact ? launch_fm(fm_kernel<uint32_t, true>) : launch_fm(fm_kernel<uint32_t, false>);
    else exact ? launch_fm(fm_kernel<uint64_t, true>) : launch_fm(fm_kernel<uint64_t, false>);
    st.mark("level/fm");
    MP_KERNEL(ctx, super_pass<<<lgrid, 256, 0, s>>>(a));
    DevBuf<int32_t> ref_cnt(width, s), ref_rw(2 * width, s);
    MP_CUDA(cudaMemsetAsync(ref_cnt, 0, sizeof(int32_t) * width, s));
    MP_CUDA(cudaMemsetAsync(ref_rw, 0, sizeof(int32_t) * 2 * width, s));
    a.ref_cnt = ref_cnt, a.ref_rw = ref_rw;
    const size_t ref_smem = static_cast<size_t>(kRefSmemList) * 10;  // 120 KB
    const bool ref_sm_state = n <= kRefSmemN;
    allow_max_smem(refine_kernel<false>, ctx.device);
    allow_max_smem(refine_kernel<true>, ctx.device);
    {
      const int kt__ = ctx.ktime_begin(kKRefine);
      MP_KERNEL(ctx, ref_init<<<lgrid, 256, 0, s>>>(a));
      if (ref_sm_state)  // lists of kRefSmemN entries + 38 B of state per vertex
        MP_KERNEL(ctx, refine_kernel<true><<<width, kNodeThreads, 10 * kRefSmemN + 38 * static_cast<size_t>(n), s>>>(a));
      else
        MP_KERNEL(ctx, refine_kernel<false><<<width, kNodeThreads, ref_smem, s>>>(a));
      ctx.ktime_end(kt__);
    }
    st.mark("level/super+refine");
    // split: children's vertex lists packed in node order by a stable radix
    // sort on (node << 1 | side); the rest gets drop_key and sorts past the end
    {
      const uint32_t drop_key = static_cast<uint32_t>(2 * width);
      MP_KERNEL(ctx, fill32<<<grid_for(ctx, n), 256, 0, s>>>(n, reinterpret_cast<int32_t*>(split_keys.get()),
                                                               static_cast<int32_t>(drop_key)));
      MP_CUDA(cudaMemsetAsync(next_cnt, 0, sizeof(int32_t) * 2 * width, s));
      MP_KERNEL(ctx, split_classify<<<lgrid, 256, 0, s>>>(a, split_keys, drop_key, next_cnt));
      const int nb = bits_for(drop_key);
      size_t tmp = 0;
      MP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, split_keys.get(), split_keys_out.get(), cur_list, nxt_list,
                                              n, 0, nb, s));
      DevBuf<char> t(tmp, s);
      MP_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, split_keys.get(), split_keys_out.get(), cur_list, nxt_list,
                                              n, 0, nb, s));
      size_t tmp2 = 0;
      MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, next_cnt.get(), next_start.get(), 2 * width, s));
      DevBuf<char> t2(tmp2, s);
      MP_CUDA(cub::DeviceScan::ExclusiveSum(t2.get(), tmp2, next_cnt.get(), next_start.get(), 2 * width, s));
    }
    st.mark("level/split");
    // next level
    seg_start = std::move(next_start);
    seg_cnt = std::move(next_cnt);
    std::swap(cur_list, nxt_list);
    width *= 2;
  }
  // flatten: stable sort of vertices by node id (ascending vertex inside a node)
  if (n > 0) {
    DevBuf<int32_t> ids(n, s), kout(n, s);
    MP_KERNEL(ctx, iota32<<<grid_for(ctx, n), 256, 0, s>>>(n, ids));
    size_t tmp = 0;
    const int nb = bits_for(nn);
    MP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, node_of, kout.get(), ids.get(), node_vertices, n, 0, nb, s));
    DevBuf<char> t(tmp, s);
    MP_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, node_of, kout.get(), ids.get(), node_vertices, n, 0, nb, s));
    MP_KERNEL(ctx, node_bounds<<<grid_for(ctx, n + 1), 256, 0, s>>>(n, nn, kout, node_offsets));
  } else {
    MP_CUDA(cudaMemsetAsync(node_offsets, 0, sizeof(int32_t) * (nn + 1), s));
  }
}

}  // namespace mp
