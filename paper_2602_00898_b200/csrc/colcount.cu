// Stage 5b, fast path — factor elimination tree, column counts and nnz(L)
// without playing the elimination game (reference core/src/symbolic.cpp:33-45
// elimination_fill, :82-96 factor_etree_parents).
//
// The reference plays the quotient-graph game and reads |reach| + 1 and the
// smallest reach position off every pivot.  Both are functions of the factor's
// elimination tree alone, so this path computes the tree and the counts
// directly, in O(|A| log n) work, never materialising a reach set:
//
//  1. etree (Liu's ancestor algorithm), split by the ND tree.  Lower neighbours
//     of a node's vertices lie in the node or below it (separator property), so
//     the nodes of one level are independent: bottom-up one level per launch,
//     one CTA per node.  Everything below the node is seen through the roots of
//     the children's forests (one per connected piece), found by a short
//     remap chain; the node's own ancestor array lives in shared memory.
//       E1 (all threads)  lower-neighbour targets of every column, compacted in
//                         column order; child roots get local slot ids;
//       E2 (warp 0)       Liu over the target stream, 32 targets per load, the
//                         lanes of one column resolving their roots together;
//       E3 (all threads)  roots of the node's forest -> croot / remap, then
//                         subtree sizes (one serial shared-memory pass).
//  2. postorder of the etree, top-down one level per launch: every vertex
//     claims its subtree's range from its parent's cursor (any postorder gives
//     the same counts).
//  3. Gilbert-Ng-Peyton column counts: per row i, its lower neighbours sorted
//     by postorder; the row subtree's leaves are those not above the previous
//     neighbour, consecutive leaves cancel at their LCA (first postorder index
//     >= b whose subtree starts at or before a: sparse-table descent).  Column
//     count = subtree sum of the deltas = a prefix-sum difference.
// Outputs are identical to the game's (bit-exact, tests/test_gpu_parity.py).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kCcThreads = 256;

int grid_for(const mp_context& ctx, int64_t n, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), ctx.num_sms * 16LL)));
}

struct CcArgs {
  DGraph g;
  int32_t n, nn, level;
  const int32_t* node_offsets;
  const int32_t* node_pos;
  const int32_t* inv;       // vertex -> position
  const int32_t* vert;      // position -> vertex
  const int32_t* D;         // exclusive prefix of degrees in position order (stream / slot segments)
  int32_t* parent;          // by position (output)
  int32_t* croot;           // by position: root of its piece after its own node
  int32_t* remap;           // by position: a piece root's root one attachment later (-1 = still a root)
  int32_t* size;            // by position: etree subtree size
  int32_t* slot_of;         // by position: local slot of a child root (-1 unclaimed, -2 being claimed)
  int2* stream;             // per node segment [D[P0], ...): (column, target)
  int32_t* rootlist;        // per node segment: child roots by slot
  int32_t* gpars;           // per node segment: slot -> local parent column
  int32_t* ganc;            // per node segment [P0 + D[P0], ...): ancestor array when shared memory is short
  int32_t* start;           // by position: first postorder index of the subtree
  int32_t* cursor;          // by position: next free postorder index for a child
  unsigned int* super;      // cursor of the forest roots
  int32_t anc_cap, sz_cap;  // shared-memory capacities (elements)
};

extern __shared__ int32_t cc_dyn[];

__device__ __forceinline__ int32_t resolve_root(const CcArgs& a, int32_t q) {
  int32_t r = a.croot[q];
  int32_t t = a.remap[r];
  if (t < 0) return r;
  while (t >= 0) r = t, t = a.remap[r];
  a.croot[q] = r;  // compress (benign race: every writer stores the same root)
  return r;
}

// Slot id of child root r in this CTA's node (claimed once; racing claimers wait).
__device__ __forceinline__ int32_t claim_slot(const CcArgs& a, int32_t r, int32_t seg, int32_t* s_nroots) {
  volatile int32_t* so = a.slot_of;
  int32_t s = so[r];
  if (s >= 0) return s;
  if (s == -1) {
    const int32_t old = atomicCAS(&a.slot_of[r], -1, -2);
    if (old == -1) {
      const int32_t id = atomicAdd(s_nroots, 1);
      a.rootlist[seg + id] = r;
      __threadfence_block();
      atomicExch(&a.slot_of[r], id);
      return id;
    }
  }
  while ((s = so[r]) < 0) {
  }
  return s;
}

__global__ void __launch_bounds__(kCcThreads) cc_etree_level(CcArgs a) {
  const int32_t X = (1 << a.level) - 1 + blockIdx.x;
  if (X >= a.nn) return;
  const int32_t xb = a.node_offsets[X], nx = a.node_offsets[X + 1] - xb;
  if (nx == 0) return;
  const int32_t P0 = a.node_pos[X];
  const int32_t seg = a.D[P0];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __shared__ int32_t s_nroots, sh[32];
  if (threadIdx.x == 0) s_nroots = 0;
  __syncthreads();
  // ---- E1: lower-neighbour targets, compacted in column order
  int32_t run = 0;
  for (int32_t base = 0; base < nx; base += blockDim.x) {
    const int32_t k = base + threadIdx.x;
    int32_t cnt = 0, e0 = 0, e1 = 0;
    if (k < nx) {
      const int32_t v = a.vert[P0 + k];
      e0 = a.g.off[v], e1 = a.g.off[v + 1];
      for (int32_t e = e0; e < e1; ++e) cnt += a.inv[a.g.nbr[e]] < P0 + k;
    }
    int32_t tot = 0;
    const int32_t ex = block_excl_scan(cnt, sh, &tot);
    if (cnt) {
      int32_t w = seg + run + ex;
      for (int32_t e = e0; e < e1; ++e) {
        const int32_t q = a.inv[a.g.nbr[e]];
        if (q >= P0 + k) continue;
        const int32_t t = q >= P0 ? q - P0 : nx + claim_slot(a, resolve_root(a, q), seg, &s_nroots);
        a.stream[w++] = make_int2(k, t);
      }
    }
    run += tot;
  }
  __syncthreads();
  const int32_t nroots = s_nroots, ne = nx + nroots, len = run;
  const bool anc_sm = ne <= a.anc_cap, sz_sm = nx <= a.sz_cap;
  int32_t* anc = anc_sm ? cc_dyn : a.ganc + static_cast<int64_t>(P0) + seg;
  int32_t* sz = sz_sm ? cc_dyn + a.anc_cap : a.size + P0;
  for (int32_t e = threadIdx.x; e < ne; e += blockDim.x) anc[e] = -1;
  __syncthreads();
  // ---- E2: Liu's algorithm over the target stream (warp 0)
  if (wid == 0) {
    volatile int32_t* va = anc;
    const int2 none = make_int2(0x7fffffff, 0);
    int2 cur = lane < len ? a.stream[seg + lane] : none;
    for (int32_t c0 = 0; c0 < len; c0 += 32) {
      const int2 nxt = c0 + 32 + lane < len ? a.stream[seg + c0 + 32 + lane] : none;
      uint32_t pending = __ballot_sync(0xffffffffu, cur.x != 0x7fffffff);
      while (pending) {
        const int32_t col = __shfl_sync(0xffffffffu, cur.x, __ffs(pending) - 1);
        const bool act = cur.x == col;
        const uint32_t am = __ballot_sync(0xffffffffu, act);
        if (act) {
          int32_t r = cur.y;
          for (;;) {
            const int32_t up = va[r];
            if (up == col) break;
            va[r] = col;
            if (up < 0) {
              if (r < nx) a.parent[P0 + r] = P0 + col;
              else a.gpars[seg + r - nx] = col;
              break;
            }
            r = up;
          }
        }
        __syncwarp();
        pending &= ~am;
      }
      cur = nxt;
    }
  }
  __syncthreads();
  for (int32_t k = threadIdx.x; k < nx; k += blockDim.x) sz[k] = 1;
  __syncthreads();
  // ---- E3: roots of the node's forest; child subtrees hang under their parents
  for (int32_t e = threadIdx.x; e < ne; e += blockDim.x) {
    int32_t r = e;
    for (int32_t up = anc[r]; up >= 0; up = anc[r]) r = up;
    if (e < nx) {
      a.croot[P0 + e] = P0 + r;
    } else {
      const int32_t R = a.rootlist[seg + e - nx], pc = a.gpars[seg + e - nx];
      a.remap[R] = P0 + r;
      a.parent[R] = P0 + pc;
      atomicAdd(&sz[pc], a.size[R]);
    }
  }
  __syncthreads();
  // subtree sizes of the node's own vertices: children precede parents
  if (wid == 0) {
    for (int32_t kb = 0; kb < nx; kb += 32) {
      const int32_t p = kb + lane < nx ? a.parent[P0 + kb + lane] - P0 : -1;
      const int32_t m = min(32, nx - kb);
      for (int32_t i = 0; i < m; ++i) {
        const int32_t pk = __shfl_sync(0xffffffffu, p, i);
        if (lane == 0 && pk >= 0 && pk < nx) sz[pk] += sz[kb + i];
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (sz_sm)
    for (int32_t k = threadIdx.x; k < nx; k += blockDim.x) a.size[P0 + k] = sz[k];
}

// Postorder ranges, top-down: a vertex's subtree occupies [start, start+size),
// the vertex itself last; children claim their ranges from the parent's cursor.
__global__ void __launch_bounds__(kCcThreads) cc_post_level(CcArgs a) {
  const int32_t X = (1 << a.level) - 1 + blockIdx.x;
  if (X >= a.nn) return;
  const int32_t xb = a.node_offsets[X], nx = a.node_offsets[X + 1] - xb;
  if (nx == 0) return;
  const int32_t P0 = a.node_pos[X];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool sm = nx <= a.sz_cap;
  int32_t* cur = sm ? cc_dyn : a.cursor + P0;
  if (wid == 0) {
    for (int32_t kb = ((nx - 1) >> 5) << 5; kb >= 0; kb -= 32) {
      const int32_t k = kb + lane;
      const int32_t p = k < nx ? a.parent[P0 + k] : -1, s = k < nx ? a.size[P0 + k] : 0;
      const int32_t m = min(32, nx - kb);
      int32_t mine = 0;
      for (int32_t i = m - 1; i >= 0; --i) {
        const int32_t pk = __shfl_sync(0xffffffffu, p, i), sk = __shfl_sync(0xffffffffu, s, i);
        int32_t st = 0;
        if (lane == 0) {
          if (pk < 0) {
            st = static_cast<int32_t>(atomicAdd(a.super, static_cast<unsigned>(sk)));
          } else if (pk >= P0 && pk < P0 + nx) {
            st = cur[pk - P0];
            cur[pk - P0] = st + sk;
          } else {
            st = atomicAdd(&a.cursor[pk], sk);
          }
          cur[kb + i] = st;
        }
        st = __shfl_sync(0xffffffffu, st, 0);
        if (lane == i) mine = st;
      }
      if (k < nx) a.start[P0 + k] = mine;
      __syncwarp();
    }
  }
  __syncthreads();
  if (sm)
    for (int32_t k = threadIdx.x; k < nx; k += blockDim.x) a.cursor[P0 + k] = cur[k];
}

__global__ void cc_vert(int32_t n, const int32_t* node_of, const int32_t* node_offsets, const int32_t* node_vertices,
                        const int32_t* local_perm, const int32_t* node_pos, const int32_t* off, int32_t* vert,
                        int32_t* deg) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t X = node_of[node_vertices[i]];
    const int32_t xb = node_offsets[X];
    const int32_t v = node_vertices[xb + local_perm[i]];
    const int32_t p = node_pos[X] + (i - xb);
    vert[p] = v;
    deg[p] = off[v + 1] - off[v];
  }
}

__global__ void cc_post_index(int32_t n, const int32_t* start, const int32_t* size, int32_t* post, int32_t* F) {
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int32_t q = start[p] + size[p] - 1;
    post[p] = q;
    F[q] = start[p];
  }
}

__global__ void cc_sparse_level(int32_t n, int32_t half, const int32_t* prev, int32_t* out) {
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c + 2 * half <= n; c += gridDim.x * blockDim.x)
    out[c] = min(prev[c], prev[c + half]);
}

// first postorder index c' >= c whose subtree starts at or before pa: the LCA
// of the nodes at postorder pa < c (sparse table ST[l][c] = min F[c, c+2^l))
__device__ __forceinline__ int32_t lca_post(const int32_t* ST, int64_t n, int32_t LOG, int32_t pa, int32_t c) {
  for (int32_t l = LOG; l >= 0; --l)
    if (c + (1LL << l) <= n && __ldg(ST + l * n + c) > pa) c += 1 << l;
  return c;
}

constexpr int kRowCap = 32;

__global__ void __launch_bounds__(256) cc_rows(int32_t n, DGraph g, const int32_t* vert, const int32_t* inv,
                                               const int32_t* parent, const int32_t* post, const int32_t* start,
                                               const int32_t* ST, int32_t LOG, unsigned long long* delta) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t v = vert[i];
    const int32_t e0 = g.off[v], e1 = g.off[v + 1];
    int32_t pb[kRowCap], sb[kRowCap];
    int32_t d = 0;
    for (int32_t e = e0; e < e1; ++e) {
      const int32_t q = inv[g.nbr[e]];
      if (q >= i) continue;
      if (d < kRowCap) {
        // insertion by postorder index
        const int32_t pq = post[q], sq = start[q];
        int32_t j = d;
        while (j > 0 && pb[j - 1] > pq) pb[j] = pb[j - 1], sb[j] = sb[j - 1], --j;
        pb[j] = pq, sb[j] = sq;
      }
      ++d;
    }
    const unsigned long long one = 1ull, minus = ~0ull;
    if (d == 0) {
      atomicAdd(&delta[post[i]], one);
    } else if (d <= kRowCap) {
      atomicAdd(&delta[pb[0]], one);
      for (int32_t k = 1; k < d; ++k)
        if (sb[k] > pb[k - 1]) {
          atomicAdd(&delta[pb[k]], one);
          atomicAdd(&delta[lca_post(ST, n, LOG, pb[k - 1], pb[k])], minus);
        }
    } else {
      // wide row: the previous neighbour of each by a scan (O(d^2), rare)
      for (int32_t e = e0; e < e1; ++e) {
        const int32_t q = inv[g.nbr[e]];
        if (q >= i) continue;
        const int32_t pq = post[q];
        int32_t prev = -1;
        for (int32_t f = e0; f < e1; ++f) {
          const int32_t r = inv[g.nbr[f]];
          if (r >= i) continue;
          const int32_t pr = post[r];
          if (pr < pq && pr > prev) prev = pr;
        }
        if (prev < 0) {
          atomicAdd(&delta[pq], one);
        } else if (start[q] > prev) {
          atomicAdd(&delta[pq], one);
          atomicAdd(&delta[lca_post(ST, n, LOG, prev, pq)], minus);
        }
      }
    }
    if (parent[i] >= 0) atomicAdd(&delta[post[parent[i]]], minus);
  }
}

__global__ void cc_counts(int32_t n, const int64_t* S, const int32_t* post, const int32_t* start, int64_t* cc) {
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    cc[p] = S[post[p]] - (start[p] > 0 ? S[start[p] - 1] : 0);
}

}  // namespace

void tree_fill_fast_dev(mp_context& ctx, const DGraph& g, int32_t L, const int32_t* node_of,
                        const int32_t* node_offsets, const int32_t* node_vertices, const int32_t* local_perm,
                        const int32_t* node_pos, const int32_t* inverse, int64_t* column_counts,
                        int32_t* etree_parent, int64_t* nnz_L, int64_t* cost) {
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
  *nnz_L = 0, *cost = 0;
  if (n == 0) return;
  std::vector<int32_t> hoff(nn + 1);
  int32_t m2 = 0;
  MP_CUDA(cudaMemcpyAsync(hoff.data(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaMemcpyAsync(&m2, g.off + n, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  const int kt = ctx.ktime_begin(kKSym);
  int32_t LOG = 0;
  while ((2LL << LOG) <= n) ++LOG;
  DevBuf<int32_t> vert(n, s), deg(n + 1, s), D(n + 1, s), croot(n, s), remap(n, s), size(n, s), slot_of(n, s),
      start(n, s), cursor(n, s), post(n, s);
  DevBuf<unsigned int> super(1, s);
  // the large scratch: one persistent context slab
  const size_t M = std::max(m2, 1);
  SlabCarve sc;
  const size_t o_stream = sc.add(sizeof(int2) * M), o_root = sc.add(sizeof(int32_t) * M),
               o_pars = sc.add(sizeof(int32_t) * M), o_anc = sc.add(sizeof(int32_t) * (static_cast<size_t>(n) + M)),
               o_delta = sc.add(sizeof(unsigned long long) * n), o_S = sc.add(sizeof(int64_t) * n),
               o_ST = sc.add(sizeof(int32_t) * static_cast<size_t>(LOG + 1) * n);
  void* slab = ctx.slab(kSlabFill, sc.total);
  int2* stream = SlabCarve::at<int2>(slab, o_stream);
  int32_t* rootlist = SlabCarve::at<int32_t>(slab, o_root);
  int32_t* gpars = SlabCarve::at<int32_t>(slab, o_pars);
  int32_t* ganc = SlabCarve::at<int32_t>(slab, o_anc);
  unsigned long long* delta = SlabCarve::at<unsigned long long>(slab, o_delta);
  int64_t* S = SlabCarve::at<int64_t>(slab, o_S);
  int32_t* ST = SlabCarve::at<int32_t>(slab, o_ST);
  MP_CUDA(cudaMemsetAsync(etree_parent, 0xff, sizeof(int32_t) * n, s));
  MP_CUDA(cudaMemsetAsync(remap, 0xff, sizeof(int32_t) * n, s));
  MP_CUDA(cudaMemsetAsync(slot_of, 0xff, sizeof(int32_t) * n, s));
  MP_CUDA(cudaMemsetAsync(super, 0, sizeof(unsigned int), s));
  MP_CUDA(cudaMemsetAsync(delta, 0, sizeof(unsigned long long) * n, s));
  MP_CUDA(cudaMemsetAsync(deg.get() + n, 0, sizeof(int32_t), s));
  MP_KERNEL(ctx, cc_vert<<<grid_for(ctx, n), 256, 0, s>>>(n, node_of, node_offsets, node_vertices, local_perm,
                                                          node_pos, g.off, vert, deg));
  size_t tmp = 0;
  MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg.get(), D.get(), n + 1, s));
  {
    DevBuf<uint8_t> t(std::max<size_t>(tmp, 1), s);
    MP_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, deg.get(), D.get(), n + 1, s));
  }
  allow_max_smem(cc_etree_level, ctx.device);
  allow_max_smem(cc_post_level, ctx.device);
  CcArgs a{};
  a.g = g, a.n = n, a.nn = nn, a.node_offsets = node_offsets, a.node_pos = node_pos, a.inv = inverse;
  a.vert = vert, a.D = D, a.parent = etree_parent, a.croot = croot, a.remap = remap, a.size = size;
  a.slot_of = slot_of, a.stream = stream, a.rootlist = rootlist, a.gpars = gpars, a.ganc = ganc;
  a.start = start, a.cursor = cursor, a.super = super;
  const int64_t smem_elems = (std::min(ctx.smem_optin, 227 * 1024) - 2048) / 4;
  auto level_max = [&](int32_t l) {
    int32_t mx = 0;
    for (int32_t j = (1 << l) - 1; j < std::min(nn, (2 << l) - 1); ++j) mx = std::max(mx, hoff[j + 1] - hoff[j]);
    return mx;
  };
  for (int32_t l = L; l >= 0; --l) {
    const int32_t mx = level_max(l);
    if (mx == 0) continue;
    const int64_t want_anc = mx + std::min<int64_t>(mx, 4096) + 32;
    a.anc_cap = static_cast<int32_t>(std::min<int64_t>(want_anc, smem_elems));
    a.sz_cap = static_cast<int32_t>(std::min<int64_t>(mx, smem_elems - a.anc_cap));
    if (a.sz_cap < mx) a.sz_cap = 0;
    a.level = l;
    const size_t dyn = 4 * (static_cast<size_t>(a.anc_cap) + a.sz_cap);
    MP_KERNEL(ctx, cc_etree_level<<<1 << l, kCcThreads, dyn, s>>>(a));
  }
  for (int32_t l = 0; l <= L; ++l) {
    const int32_t mx = level_max(l);
    if (mx == 0) continue;
    a.anc_cap = 0;
    a.sz_cap = static_cast<int32_t>(std::min<int64_t>(mx, smem_elems));
    if (a.sz_cap < mx) a.sz_cap = 0;
    a.level = l;
    MP_KERNEL(ctx, cc_post_level<<<1 << l, kCcThreads, 4 * static_cast<size_t>(a.sz_cap), s>>>(a));
  }
  MP_KERNEL(ctx, cc_post_index<<<grid_for(ctx, n), 256, 0, s>>>(n, start, size, post, ST));
  for (int32_t l = 1; l <= LOG; ++l)
    MP_KERNEL(ctx, cc_sparse_level<<<grid_for(ctx, n), 256, 0, s>>>(n, 1 << (l - 1), ST + (l - 1) * static_cast<int64_t>(n),
                                                                    ST + l * static_cast<int64_t>(n)));
  MP_KERNEL(ctx, cc_rows<<<grid_for(ctx, n), 256, 0, s>>>(n, g, vert, inverse, etree_parent, post, start, ST, LOG,
                                                          delta));
  tmp = 0;
  const int64_t* din = reinterpret_cast<const int64_t*>(delta);
  MP_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, din, S, n, s));
  {
    DevBuf<uint8_t> t(std::max<size_t>(tmp, 1), s);
    MP_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, din, S, n, s));
  }
  MP_KERNEL(ctx, cc_counts<<<grid_for(ctx, n), 256, 0, s>>>(n, S, post, start, column_counts));
  ctx.ktime_end(kt);
  sum_counts_dev(ctx, n, column_counts, nnz_L, cost);
}

}  // namespace mp
