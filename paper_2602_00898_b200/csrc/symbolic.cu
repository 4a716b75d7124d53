// Stage 5b — factor elimination tree and column counts, nnz(L)
// (reference core/src/symbolic.cpp:33-45 elimination_fill, :82-96
// factor_etree_parents, on the EliminationState game of elimination.cpp).
//
// The reference plays one sequential elimination game over the whole graph
// in permutation order.  The ND tree splits that game exactly: once the
// vertices of a subtree are eliminated, what the rest of the game sees of
// them is one live element per connected piece, with a boundary inside the
// ancestor separators.  So the device plays the game node by node, bottom-up
// one tree level per launch, one CTA per node:
//   * variables of a node vertex = its neighbours in the node or in an
//     ancestor (neighbours below are represented by the children's leftover
//     elements, which keep exactly the same reach sets);
//   * inherited elements = the children's live elements, attached to the node
//     vertices in their boundary (or passed up when none is in the node);
//   * pivots in local_perm order; |reach| + 1 is the column count, the
//     smallest permutation position in the reach is the etree parent.
// Reach sets are identical to the sequential game, so column counts, nnz(L),
// Σ counts² and parents are bit-exact for any schedule.
#include <cub/cub.cuh>

#include <algorithm>
#include <functional>
#include <utility>
#include <vector>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kSymThreads = 512;
constexpr int kSymWide = 1024;  // block size for levels narrower than half the SMs
constexpr int kU = 4;  // reach entries per thread per sweep step

int grid_for(const mp_context& ctx, int64_t n, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), ctx.num_sms * 16LL)));
}

struct SymArgs {
  DGraph g;
  int32_t nn;
  int32_t level;
  const int32_t* node_of;
  const int32_t* node_offsets;
  const int32_t* node_vertices;
  const int32_t* local_perm;
  const int32_t* local_of;
  const int32_t* node_pos;   // first permutation position per node
  const int32_t* inverse;    // vertex -> permutation position
  int32_t* adj;              // CSR slots
  int32_t* el;               // CSR slots
  int32_t* nadj;
  int32_t* nel;
  int64_t* bptr;             // per element
  int32_t* bsz;              // per element
  int32_t* emark;            // per element, token = pivot + 1
  int32_t* pool;
  int64_t pool_cap;
  unsigned long long* pool_cursor;
  const int64_t* ws_off;     // per level-local node: private mark + scratch workspace
  int32_t* ws;
  const int64_t* left_off;   // per node: leftover-element list slab
  int32_t* left_cnt;         // per node
  int32_t* left_list;
  int64_t* column_counts;    // by position
  int32_t* parent;           // by position
  int32_t* overflow;
  int32_t smem_path;         // path sizes up to this use shared-memory marks
  // cross_block_fill (symbolic.cpp:98-119): tree node of every vertex in the
  // caller's tree, and the count of reach members whose node is unrelated to
  // the pivot's (NULL: not counted)
  const int32_t* cross_owner;
  unsigned long long* cross_count;
  const uint8_t* play_mask;  // sharded game: nodes this rank plays (NULL = all)
};

// private index of w (in node A, an ancestor-or-self of the CTA's node)
__device__ __forceinline__ int32_t priv_idx(const SymArgs& a, const int32_t* abase, int32_t w) {
  return abase[tree_level(a.node_of[w])] + a.local_of[w];
}

// Pool space is taken from the global cursor in per-CTA chunks that double
// from kChunk0 to kChunkMax ints (the unused tail of a CTA's last chunk is at
// most what it used); every thread tracks the chunk identically (all inputs
// to the bookkeeping are block-uniform), so only a refill needs a broadcast.
constexpr unsigned long long kChunk0 = 2048, kChunkMax = 1 << 20;

extern __shared__ int32_t sym_dyn[];

__global__ void __launch_bounds__(kSymWide) sym_kernel(SymArgs a) {
  const int32_t first = (1 << a.level) - 1;
  const int32_t X = first + blockIdx.x;
  if (X >= a.nn) return;
  if (a.play_mask && !a.play_mask[X]) return;  // another rank plays this node
  if (*static_cast<volatile int32_t*>(a.overflow)) return;  // an earlier node ran out of pool
  const int32_t xb = a.node_offsets[X], nx = a.node_offsets[X + 1] - xb;
  const int32_t lc = 2 * X + 1, rc = 2 * X + 2;
  const bool has_children = lc < a.nn;
  const int64_t lslab = a.left_off[X];
  int32_t* myleft = a.left_list + lslab;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ int32_t abase[32];
  __shared__ int32_t s_cnt[2], s_nleft;
  __shared__ unsigned long long s_chunk;
  __shared__ uint64_t red[32];
  if (threadIdx.x == 0) {
    s_nleft = 0;
    s_cnt[0] = s_cnt[1] = 0;
    // ancestor sizes along the path: abase[level] = sum of the sizes above
    int32_t path[32];
    int32_t depth = 0;
    for (int32_t t = X;; t = (t - 1) / 2) {
      path[depth++] = t;
      if (t == 0) break;
    }
    int32_t run = 0;
    for (int32_t l = 0; l < depth; ++l) {
      const int32_t A = path[depth - 1 - l];
      abase[l] = run;
      run += a.node_offsets[A + 1] - a.node_offsets[A];
    }
    abase[depth] = run;
  }
  __syncthreads();
  const int32_t path_size = abase[a.level + 1];
  // marks + scratch: shared memory when the launch provided room for this
  // level's longest path, else this node's global workspace.  A reach lies
  // inside the path (node + ancestors), so scratch needs path_size entries.
  int32_t* marks = a.smem_path >= path_size ? sym_dyn : a.ws + a.ws_off[blockIdx.x];
  int32_t* scratch = marks + path_size;
  for (int32_t i = threadIdx.x; i < path_size; i += blockDim.x) marks[i] = 0;
  const int32_t* verts = a.node_vertices + xb;

  // ---- variables: neighbours in X or an ancestor
  for (int32_t k = threadIdx.x; k < nx; k += blockDim.x) {
    const int32_t v = verts[k];
    const int32_t o = a.g.off[v];
    int32_t c = 0;
    for (int32_t j = o; j < a.g.off[v + 1]; ++j) {
      const int32_t w = a.g.nbr[j];
      if (is_ancestor_or_self(a.node_of[w], X)) a.adj[o + c++] = w;
    }
    a.nadj[v] = c;
    a.nel[v] = 0;
  }
  __syncthreads();
  // ---- inherited elements (warp per element)
  if (has_children) {
    for (int side = 0; side < 2; ++side) {
      const int32_t c = side ? rc : lc;
      const int32_t* cl = a.left_list + a.left_off[c];
      const int32_t ncl = a.left_cnt[c];
      for (int32_t i = wid; i < ncl; i += nw) {
        const int32_t e = cl[i];
        const int32_t* bd = a.pool + a.bptr[e];
        const int32_t sz = a.bsz[e];
        bool any = false;
        for (int32_t j = lane; j < sz; j += 32) {
          const int32_t w = bd[j];
          const bool mine = a.node_of[w] == X;
          if (mine) a.el[a.g.off[w] + atomicAdd(&a.nel[w], 1)] = e;
          any |= mine;
        }
        any = __any_sync(0xffffffffu, any);
        if (!any && lane == 0) myleft[atomicAdd(&s_nleft, 1)] = e;
      }
    }
  }
  __syncthreads();
  // ---- the game on X, pivots in local_perm order; two barriers per pivot
  const int32_t pos0 = a.node_pos[X];
  unsigned long long cur = 0, cend = 0, chunk = kChunk0;  // this CTA's pool chunk (block-uniform)
  // the pivot sequence and CSR offsets are static: the next pivot's are
  // loaded while this one runs
  int32_t p_next = nx ? verts[a.local_perm[xb]] : 0;
  int32_t o_next = nx ? a.g.off[p_next] : 0;
  for (int32_t k = 0; k < nx; ++k) {
    const int32_t p = p_next, po = o_next;
    if (k + 1 < nx) {
      p_next = verts[a.local_perm[xb + k + 1]];
      o_next = a.g.off[p_next];
    }
    const int32_t tok = k + 1;
    int32_t* cnt = &s_cnt[k & 1];
    const int32_t np_adj = a.nadj[p], np_el = a.nel[p];
    const int32_t* padj = a.adj + po;
    const int32_t* pel = a.el + po;
    // reach = adj(p) + the boundaries of p's elements, minus p; the smallest
    // permutation position in it is folded in on the way.  Each thread takes
    // kU entries at a time so their dependent loads are in flight together.
    uint64_t mn = ~0ull;
    const int32_t powner = a.cross_owner ? a.cross_owner[p] : 0;
    uint32_t ncross = 0;
    auto sweep = [&](const int32_t* list, int32_t len) {
      for (int32_t i0 = threadIdx.x; i0 < len; i0 += kU * blockDim.x) {
        int32_t w[kU], pi[kU];
        uint32_t inv[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
          const int32_t i = i0 + q * blockDim.x;
          w[q] = i < len ? list[i] : p;
        }
#pragma unroll
        for (int q = 0; q < kU; ++q)
          if (w[q] != p) pi[q] = priv_idx(a, abase, w[q]), inv[q] = static_cast<uint32_t>(a.inverse[w[q]]);
#pragma unroll
        for (int q = 0; q < kU; ++q)
          if (w[q] != p && atomicExch(&marks[pi[q]], tok) != tok) {
            scratch[atomicAdd(cnt, 1)] = w[q];
            mn = min(mn, static_cast<uint64_t>(inv[q]));
            if (a.cross_owner) {
              const int32_t wo = a.cross_owner[w[q]];
              ncross += wo != powner && !is_ancestor_or_self(wo, powner) && !is_ancestor_or_self(powner, wo);
            }
          }
      }
    };
    sweep(padj, np_adj);
    // elements: each warp loads up to 32 (boundary, size) pairs at once, then
    // the whole block sweeps each boundary (a root-separator element can hold
    // thousands of vertices)
    for (int32_t e0 = 0; e0 < np_el; e0 += 32) {
      const int32_t ne = min(32, np_el - e0);
      int32_t my_e = -1, my_sz = 0;
      int64_t my_bp = 0;
      if (lane < ne) {
        my_e = pel[e0 + lane];
        my_bp = a.bptr[my_e];
        my_sz = a.bsz[my_e];
        if (wid == 0) a.emark[my_e] = p + 1;
      }
      for (int32_t j = 0; j < ne; ++j) {
        const int32_t sz = __shfl_sync(0xffffffffu, my_sz, j);
        sweep(a.pool + __shfl_sync(0xffffffffu, my_bp, j), sz);
      }
    }
    if (a.cross_owner) {
      ncross = __reduce_add_sync(0xffffffffu, ncross);
      if (lane == 0 && ncross) atomicAdd(a.cross_count, static_cast<unsigned long long>(ncross));
    }
    mn = warp_min_u64(mn);
    if (lane == 0) red[wid] = mn;
    __syncthreads();
    const int32_t nb = *cnt;
    mn = lane < nw ? red[lane] : ~0ull;
    mn = warp_min_u64(mn);
    if (cur + nb > cend) {  // block-uniform: refill the chunk
      const unsigned long long take = max(static_cast<unsigned long long>(nb), chunk);
      chunk = min(2 * chunk, kChunkMax);
      if (threadIdx.x == 0) {
        const unsigned long long at = atomicAdd(a.pool_cursor, take);
        if (static_cast<int64_t>(at + take) > a.pool_cap) {
          atomicExch(a.overflow, 1);
          s_chunk = ~0ull;
        } else {
          s_chunk = at;
        }
      }
      __syncthreads();
      cur = s_chunk;
      if (cur == ~0ull) return;  // host retries with a larger pool
      cend = cur + take;
    }
    const unsigned long long at = cur;
    cur += nb;
    if (threadIdx.x == 0) {
      // column count and etree parent (symbolic.cpp:40-43, :86-93)
      a.column_counts[pos0 + k] = static_cast<int64_t>(nb) + 1;
      a.parent[pos0 + k] = nb ? static_cast<int32_t>(mn) : -1;
      a.bptr[p] = static_cast<int64_t>(at);
      a.bsz[p] = nb;
      a.nadj[p] = 0;
      a.nel[p] = 0;
      s_cnt[(k + 1) & 1] = 0;
    }
    int32_t* dst = a.pool + at;
    for (int32_t i = threadIdx.x; i < nb; i += blockDim.x) dst[i] = scratch[i];
    for (int32_t ei = threadIdx.x; ei < np_el; ei += blockDim.x) a.bsz[pel[ei]] = 0;
    // update the node's own boundary members (elimination.cpp:75-83): drop
    // reach members and p from adj, absorbed elements from el, append p.
    // Lists are read ahead in chunks of 8 before the in-place compaction
    // writes (the aliasing would otherwise serialise every load).
    for (int32_t i = threadIdx.x; i < nb; i += blockDim.x) {
      const int32_t w = scratch[i];
      // membership and the list heads are loaded together
      const int32_t xw = a.node_of[w], o = a.g.off[w], na = a.nadj[w], ne = a.nel[w];
      if (xw != X) continue;
      int32_t* wa = a.adj + o;
      int32_t c = 0;
      for (int32_t j0 = 0; j0 < na; j0 += 8) {
        int32_t x[8];
        bool keep[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = j0 + q < na ? wa[j0 + q] : p;
#pragma unroll
        for (int q = 0; q < 8; ++q) keep[q] = x[q] != p && marks[priv_idx(a, abase, x[q])] != tok;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (keep[q]) wa[c++] = x[q];
      }
      a.nadj[w] = c;
      int32_t* we = a.el + o;
      int32_t ce = 0;
      for (int32_t j0 = 0; j0 < ne; j0 += 8) {
        int32_t e[8];
        bool keep[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) e[q] = j0 + q < ne ? we[j0 + q] : -1;
#pragma unroll
        for (int q = 0; q < 8; ++q) keep[q] = e[q] >= 0 && a.emark[e[q]] != p + 1;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (keep[q]) we[ce++] = e[q];
      }
      we[ce++] = p;
      a.nel[w] = ce;
    }
    __syncthreads();
  }
  // ---- leftover: live elements created here, plus the pass-through ones
  for (int32_t k = threadIdx.x; k < nx; k += blockDim.x) {
    const int32_t v = verts[k];
    if (a.bsz[v] > 0) myleft[atomicAdd(&s_nleft, 1)] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) a.left_cnt[X] = s_nleft;
}

__global__ void local_of_kernel(int32_t n, const int32_t* node_of, const int32_t* node_offsets,
                                const int32_t* node_vertices, int32_t* local_of) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t v = node_vertices[i];
    local_of[v] = i - node_offsets[node_of[v]];
  }
}
__global__ void sum_counts(int32_t n, const int64_t* cc, unsigned long long* out) {
  __shared__ int64_t red[32];
  int64_t s = 0, q = 0;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    s += cc[i];
    q += cc[i] * cc[i];
  }
  s = block_sum_i64(s, red);
  q = block_sum_i64(q, red);
  if (threadIdx.x == 0) {
    atomicAdd(&out[0], static_cast<unsigned long long>(s));
    atomicAdd(&out[1], static_cast<unsigned long long>(q));
  }
}
// element records [e, |boundary|, boundary...] at rec_off[i] (export of a
// subtree root's live elements, mp_order_sharded)
__global__ void pack_elements(int32_t ne, const int32_t* elems, const int64_t* rec_off, const int64_t* bptr,
                              const int32_t* bsz, const int32_t* pool, int32_t* out) {
  const int lane = threadIdx.x & 31;
  for (int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < ne; i += (gridDim.x * blockDim.x) >> 5) {
    const int32_t e = elems[i], sz = bsz[e];
    int32_t* o = out + rec_off[i];
    if (lane == 0) o[0] = e, o[1] = sz;
    const int32_t* src = pool + bptr[e];
    for (int32_t j = lane; j < sz; j += 32) o[2 + j] = src[j];
  }
}
__global__ void gather_bsz(int32_t ne, const int32_t* elems, const int32_t* bsz, int32_t* out) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += gridDim.x * blockDim.x) out[i] = bsz[elems[i]];
}
// import: element i gets boundary pool[base + off[i] ..) of size sz[i]
__global__ void set_elements(int32_t ne, const int32_t* elems, const int32_t* sz, const int64_t* off, int64_t base,
                             int64_t* bptr, int32_t* bsz) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += gridDim.x * blockDim.x) {
    bptr[elems[i]] = base + off[i];
    bsz[elems[i]] = sz[i];
  }
}
__global__ void clear_bsz(int32_t n, int32_t* bsz) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) bsz[i] = 0;
}

}  // namespace

void sum_counts_dev(mp_context& ctx, int64_t n, const int64_t* column_counts, int64_t* nnz_L, int64_t* cost) {
  cudaStream_t s = ctx.stream;
  *nnz_L = 0, *cost = 0;
  if (n == 0) return;
  DevBuf<unsigned long long> sums(2, s);
  MP_CUDA(cudaMemsetAsync(sums, 0, 16, s));
  MP_KERNEL(ctx, sum_counts<<<grid_for(ctx, n), 256, 0, s>>>(static_cast<int32_t>(n), column_counts, sums));
  unsigned long long h[2];
  MP_CUDA(cudaMemcpyAsync(h, sums, 16, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  *nnz_L = static_cast<int64_t>(h[0]);
  *cost = static_cast<int64_t>(h[1]);
}

void tree_fill_dev(mp_context& ctx, const DGraph& g, int32_t L, const int32_t* node_of,
                   const int32_t* node_offsets, const int32_t* node_vertices, const int32_t* local_perm,
                   const int32_t* node_pos, const int32_t* inverse, int64_t* column_counts,
                   int32_t* etree_parent, int64_t* nnz_L, int64_t* cost, const int32_t* cross_owner,
                   int64_t* crossing, const FillShard* shard) {
  const bool sharded_game = shard && shard->k > 0 && shard->k <= L;
  if (!cross_owner && !crossing && !sharded_game && ctx.fill_algo == 0) {
    tree_fill_fast_dev(ctx, g, L, node_of, node_offsets, node_vertices, local_perm, node_pos, inverse, column_counts,
                       etree_parent, nnz_L, cost);
    return;
  }
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
  *nnz_L = 0;
  *cost = 0;
  if (n == 0) return;
  // host view of the tree shape (nn+1 ints)
  std::vector<int32_t> hoff(nn + 1);
  MP_CUDA(cudaMemcpyAsync(hoff.data(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
  int32_t m2 = 0;
  MP_CUDA(cudaMemcpyAsync(&m2, g.off + n, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  auto size_of = [&](int32_t i) -> int64_t { return hoff[i + 1] - hoff[i]; };
  // leftover slabs: subtree sizes
  std::vector<int64_t> sub(nn, 0), left_off(nn + 1, 0);
  for (int32_t i = nn - 1; i >= 0; --i) {
    sub[i] = size_of(i);
    if (2 * i + 1 < nn) sub[i] += sub[2 * i + 1] + sub[2 * i + 2];
  }
  for (int32_t i = 0; i < nn; ++i) left_off[i + 1] = left_off[i] + sub[i];
  // path sizes (node + ancestors), per level workspace offsets
  std::vector<int64_t> path(nn, 0);
  for (int32_t i = 0; i < nn; ++i) path[i] = size_of(i) + (i ? path[(i - 1) / 2] : 0);
  // marks + scratch (8 B per path vertex) live in shared
  // memory for nodes whose path fits kSymSmem (keeps 2 CTAs per SM); longer
  // paths use a per-node global workspace
  constexpr int64_t kSymSmem = 100 * 1024;
  allow_max_smem(sym_kernel, ctx.device);
  int64_t ws_max = 0;
  std::vector<std::vector<int64_t>> ws_offs(L + 1);
  std::vector<int32_t> smem_path(L + 1, 0);
  for (int32_t l = 0; l <= L; ++l) {
    const int32_t first = (1 << l) - 1, width = 1 << l;
    auto& wo = ws_offs[l];
    wo.assign(width + 1, 0);
    int64_t longest = 0;
    for (int32_t j = 0; j < width; ++j) longest = std::max(longest, path[first + j]);
    smem_path[l] = static_cast<int32_t>(std::min<int64_t>(longest, kSymSmem / 8));
    for (int32_t j = 0; j < width; ++j)
      wo[j + 1] = wo[j] + (path[first + j] > smem_path[l] ? 2 * path[first + j] + 2 : 0);
    ws_max = std::max(ws_max, wo[width]);
  }
  DevBuf<int32_t> local_of(n, s), nadj(n, s), nel(n, s), bsz(n, s), emark(n, s), ws(std::max<int64_t>(ws_max, 1), s),
      left_cnt(nn, s), left_list(std::max<int64_t>(left_off[nn], 1), s), overflow(1, s);
  DevBuf<int64_t> bptr(n, s), d_left_off(nn + 1, s), d_ws_off((static_cast<size_t>(1) << L) + 1, s);
  DevBuf<int32_t> adj(std::max(m2, 1), s), el(std::max(m2, 1), s);
  DevBuf<unsigned long long> cursor(1, s), cross(1, s);
  DevBuf<uint8_t> play_mask;
  MP_KERNEL(ctx, local_of_kernel<<<grid_for(ctx, n), 256, 0, s>>>(n, node_of, node_offsets, node_vertices, local_of));
  MP_CUDA(cudaMemcpyAsync(d_left_off, left_off.data(), sizeof(int64_t) * (nn + 1), cudaMemcpyHostToDevice, s));
  // sharded game (mp_order_sharded): this rank plays its own subtrees below
  // the shard level, exchanges their roots' live elements, then every rank
  // plays the top levels
  const bool sharded = shard && shard->k > 0 && shard->k <= L;
  const int32_t k = sharded ? shard->k : 0;
  if (sharded) {
    std::vector<uint8_t> hm(nn);
    for (int32_t i = 0; i < nn; ++i) hm[i] = shard->owner[i] < 0 || shard->owner[i] == shard->rank;
    play_mask.alloc(nn, s);
    MP_CUDA(cudaMemcpyAsync(play_mask.get(), hm.data(), nn, cudaMemcpyHostToDevice, s));
  }
  std::vector<int32_t> received;  // all ranks' exported roots (the collective runs once)
  bool exchanged = false;
  // boundary pool: sum of reach sizes = nnz(L) - n; start from the ratio seen
  // on earlier calls of this context, grow and replay on overflow
  int64_t cap = std::max<int64_t>(48LL * n, static_cast<int64_t>(ctx.sym_pool_ratio * 1.25 * n)) + 4096;
  for (int attempt = 0; attempt < 8; ++attempt) {
    DevBuf<int32_t> pool(cap, s);
    MP_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));
    MP_CUDA(cudaMemsetAsync(overflow, 0, 4, s));
    MP_CUDA(cudaMemsetAsync(emark, 0, sizeof(int32_t) * n, s));
    MP_KERNEL(ctx, clear_bsz<<<grid_for(ctx, n), 256, 0, s>>>(n, bsz));
    SymArgs a{};
    a.g = g, a.nn = nn, a.node_of = node_of, a.node_offsets = node_offsets, a.node_vertices = node_vertices;
    a.local_perm = local_perm, a.local_of = local_of, a.node_pos = node_pos, a.inverse = inverse;
    a.adj = adj, a.el = el, a.nadj = nadj, a.nel = nel, a.bptr = bptr, a.bsz = bsz, a.emark = emark;
    a.pool = pool, a.pool_cap = cap, a.pool_cursor = cursor, a.ws = ws, a.left_off = d_left_off;
    a.left_cnt = left_cnt, a.left_list = left_list, a.column_counts = column_counts, a.parent = etree_parent;
    a.overflow = overflow;
    a.cross_owner = cross_owner, a.cross_count = cross;
    MP_CUDA(cudaMemsetAsync(cross, 0, sizeof(unsigned long long), s));
    auto play = [&](int32_t hi, int32_t lo, const uint8_t* mask) {
      a.play_mask = mask;
      for (int32_t l = hi; l >= lo; --l) {
        const int32_t width = 1 << l;
        MP_CUDA(cudaMemcpyAsync(d_ws_off, ws_offs[l].data(), sizeof(int64_t) * (width + 1), cudaMemcpyHostToDevice, s));
        a.level = l;
        a.ws_off = d_ws_off;
        a.smem_path = smem_path[l];
        const size_t dyn = 8 * static_cast<size_t>(smem_path[l]);
        const int kt = ctx.ktime_begin(kKSym);
        MP_KERNEL(ctx, sym_kernel<<<width, 2 * width <= ctx.num_sms ? kSymWide : kSymThreads, dyn, s>>>(a));
        ctx.ktime_end(kt);
      }
    };
    auto overflowed = [&](unsigned long long* used) {
      int32_t h_over = 0;
      MP_CUDA(cudaMemcpyAsync(&h_over, overflow, 4, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaMemcpyAsync(used, cursor, 8, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
      return h_over != 0;
    };
    unsigned long long used = 0;
    play(L, k, sharded ? play_mask.get() : nullptr);
    bool over = overflowed(&used);
    if (sharded && !over) {
      // ---- export: [root, count, (element, |boundary|, boundary...)...] per own level-k root
      const int32_t first = (1 << k) - 1, width = 1 << k;
      std::vector<int32_t> hcnt(nn);
      MP_CUDA(cudaMemcpyAsync(hcnt.data(), left_cnt.get(), sizeof(int32_t) * nn, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
      std::vector<int32_t> roots, elems;
      for (int32_t j = 0; j < width; ++j)
        if (shard->owner[first + j] == shard->rank) roots.push_back(first + j);
      std::vector<size_t> root_at;
      for (int32_t X : roots) {
        root_at.push_back(elems.size());
        const size_t at = elems.size();
        elems.resize(at + hcnt[X]);
        if (hcnt[X])
          MP_CUDA(cudaMemcpyAsync(elems.data() + at, left_list.get() + left_off[X], sizeof(int32_t) * hcnt[X],
                                  cudaMemcpyDeviceToHost, s));
      }
      MP_CUDA(cudaStreamSynchronize(s));
      const int32_t ne = static_cast<int32_t>(elems.size());
      std::vector<int32_t> esz(ne);
      std::vector<int64_t> rec_off(ne);
      DevBuf<int32_t> d_elems(std::max(ne, 1), s), d_esz(std::max(ne, 1), s);
      if (ne) {
        MP_CUDA(cudaMemcpyAsync(d_elems, elems.data(), sizeof(int32_t) * ne, cudaMemcpyHostToDevice, s));
        MP_KERNEL(ctx, gather_bsz<<<grid_for(ctx, ne), 256, 0, s>>>(ne, d_elems, bsz, d_esz));
        MP_CUDA(cudaMemcpyAsync(esz.data(), d_esz.get(), sizeof(int32_t) * ne, cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
      }
      // layout: [nroots] then per root [X, cnt, records...]
      std::vector<int32_t> buf(1, static_cast<int32_t>(roots.size()));
      int64_t total = 1;
      for (size_t r = 0; r < roots.size(); ++r) {
        total += 2;
        const size_t e0 = root_at[r], e1 = r + 1 < roots.size() ? root_at[r + 1] : elems.size();
        for (size_t i = e0; i < e1; ++i) rec_off[i] = total, total += 2 + esz[i];
      }
      buf.resize(total);
      if (ne) {
        DevBuf<int64_t> d_off(ne, s);
        DevBuf<int32_t> d_buf(total, s);
        MP_CUDA(cudaMemcpyAsync(d_off, rec_off.data(), sizeof(int64_t) * ne, cudaMemcpyHostToDevice, s));
        MP_KERNEL(ctx, pack_elements<<<grid_for(ctx, 32LL * ne), 256, 0, s>>>(ne, d_elems, d_off, bptr, bsz, pool,
                                                                             d_buf));
        MP_CUDA(cudaMemcpyAsync(buf.data(), d_buf.get(), sizeof(int32_t) * total, cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
      }
      {
        int64_t at = 1;
        for (size_t r = 0; r < roots.size(); ++r) {
          buf[at] = roots[r], buf[at + 1] = hcnt[roots[r]];
          at += 2;
          const size_t e0 = root_at[r], e1 = r + 1 < roots.size() ? root_at[r + 1] : elems.size();
          for (size_t i = e0; i < e1; ++i) at += 2 + esz[i];
        }
        buf[0] = static_cast<int32_t>(roots.size());
      }
      if (!exchanged) {
        received = shard->exchange(buf);
        exchanged = true;
      }
      // ---- import the other ranks' roots: their live elements join this pool
      std::vector<int32_t> ie, isz, blob;
      std::vector<int64_t> ioff;
      std::vector<std::pair<int32_t, std::vector<int32_t>>> lists;
      for (size_t at = 0; at < received.size();) {
        const int32_t nr = received[at++];
        for (int32_t r = 0; r < nr; ++r) {
          const int32_t X = received[at], cnt = received[at + 1];
          at += 2;
          const bool mine = shard->owner[X] == shard->rank;
          std::vector<int32_t> lst;
          for (int32_t i = 0; i < cnt; ++i) {
            const int32_t e = received[at], sz = received[at + 1];
            if (!mine) {
              ie.push_back(e), isz.push_back(sz), ioff.push_back(static_cast<int64_t>(blob.size()));
              blob.insert(blob.end(), received.begin() + at + 2, received.begin() + at + 2 + sz);
              lst.push_back(e);
            }
            at += 2 + sz;
          }
          if (!mine) lists.emplace_back(X, std::move(lst));
        }
      }
      const int64_t base = static_cast<int64_t>(used);
      if (base + static_cast<int64_t>(blob.size()) > cap) {
        over = true;  // no room for the imported boundaries: grow and replay
        used += blob.size();
      } else {
        const int32_t ni = static_cast<int32_t>(ie.size());
        if (!blob.empty())
          MP_CUDA(cudaMemcpyAsync(pool.get() + base, blob.data(), sizeof(int32_t) * blob.size(),
                                  cudaMemcpyHostToDevice, s));
        DevBuf<int32_t> d_ie(std::max(ni, 1), s), d_isz(std::max(ni, 1), s);
        DevBuf<int64_t> d_ioff(std::max(ni, 1), s);
        if (ni) {
          MP_CUDA(cudaMemcpyAsync(d_ie, ie.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, s));
          MP_CUDA(cudaMemcpyAsync(d_isz, isz.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, s));
          MP_CUDA(cudaMemcpyAsync(d_ioff, ioff.data(), sizeof(int64_t) * ni, cudaMemcpyHostToDevice, s));
          MP_KERNEL(ctx, set_elements<<<grid_for(ctx, ni), 256, 0, s>>>(ni, d_ie, d_isz, d_ioff, base, bptr, bsz));
        }
        for (auto& [X, lst] : lists) {
          const int32_t c = static_cast<int32_t>(lst.size());
          if (c)
            MP_CUDA(cudaMemcpyAsync(left_list.get() + left_off[X], lst.data(), sizeof(int32_t) * c,
                                    cudaMemcpyHostToDevice, s));
          MP_CUDA(cudaMemcpyAsync(left_cnt.get() + X, &c, 4,
                                  cudaMemcpyHostToDevice, s));
          MP_CUDA(cudaStreamSynchronize(s));  // the host copies live in this loop iteration
        }
        const unsigned long long nc = static_cast<unsigned long long>(base + blob.size());
        MP_CUDA(cudaMemcpyAsync(cursor, &nc, 8, cudaMemcpyHostToDevice, s));
        MP_CUDA(cudaStreamSynchronize(s));
        // ---- the top levels, replicated on every rank
        play(k - 1, 0, nullptr);
        over = overflowed(&used);
      }
    }
    if (!over) {
      ctx.sym_pool_ratio = std::max(ctx.sym_pool_ratio, static_cast<double>(used) / std::max(n, 1));
      break;
    }
    cap = std::max<int64_t>(2 * cap, static_cast<int64_t>(used) * 2);
    if (attempt == 7) throw Error(MP_ENOMEM, "symbolic: element pool exhausted");
  }
  if (!sharded) sum_counts_dev(ctx, n, column_counts, nnz_L, cost);  // sharded: the caller sums after its gather
  if (crossing) {
    unsigned long long hc = 0;
    MP_CUDA(cudaMemcpyAsync(&hc, cross, 8, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    *crossing = static_cast<int64_t>(hc);
  }
}

namespace {
__global__ void game_tree(int32_t n, const int32_t* perm, int32_t* verts, int32_t* inverse, int32_t* node_of,
                          int32_t* bad) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    verts[i] = i;
    node_of[i] = 0;
    const int32_t v = perm[i];
    if (v < 0 || v >= n) {
      atomicExch(bad, 1);
      continue;
    }
    if (atomicExch(&inverse[v], i) != -1) atomicExch(bad, 1);
  }
}
}  // namespace

// elimination_fill / factor_etree_parents / cross_block_fill for an arbitrary
// permutation (symbolic.cpp:33-45, :82-96, :98-119): the game on a one-node
// tree whose local order is the permutation itself (one CTA plays every pivot).
void elimination_game_dev(mp_context& ctx, const DGraph& g, const int32_t* perm, int64_t* column_counts,
                          int32_t* etree_parent, int64_t* nnz_L, int64_t* cost, const int32_t* cross_owner,
                          int64_t* crossing) {
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  *nnz_L = 0, *cost = 0;
  if (crossing) *crossing = 0;
  if (n == 0) return;
  DevBuf<int32_t> off(2, s), verts(n, s), inv(n, s), node_of(n, s), pos(2, s), bad(1, s);
  const int32_t hoff[2] = {0, n};
  MP_CUDA(cudaMemcpyAsync(off, hoff, sizeof hoff, cudaMemcpyHostToDevice, s));
  MP_CUDA(cudaMemcpyAsync(pos, hoff, sizeof hoff, cudaMemcpyHostToDevice, s));
  MP_CUDA(cudaMemsetAsync(inv, 0xff, sizeof(int32_t) * n, s));
  MP_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  MP_KERNEL(ctx, game_tree<<<grid_for(ctx, n), 256, 0, s>>>(n, perm, verts, inv, node_of, bad));
  int32_t hb = 0;
  MP_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (hb) throw Error(MP_EINVAL, "permutation is not a bijection");  // symbolic.cpp:16-18
  // local_perm of the single node = positions into its iota vertex list = perm
  tree_fill_dev(ctx, g, 0, node_of, off, verts, perm, pos, inv, column_counts, etree_parent, nnz_L, cost,
                cross_owner, crossing);
}

}  // namespace mp
