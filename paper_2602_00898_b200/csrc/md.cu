// Stage 3 — per-node minimum-degree orderings (reference
// core/src/local_order.cpp:10-87 on core/src/elimination.cpp:8-98).
//
// One CTA per non-empty ND-tree node (order_tree_nodes, local_order.cpp:57-87).
// The CTA keeps the quotient-graph elimination state of the node's induced
// subgraph: variable lists and element lists live in slots of the vertex's
// CSR range (|adj|+|elems| never grows, see below), element boundaries in a
// per-node ping-pong pool with compaction, approximate degrees in shared
// memory.  Each pivot is the block-wide argmin of (degree, local id), which is
// the std::set<(deg,id)> order of the reference (local_order.cpp:24-40).
//
// Slot bound: when pivot p is eliminated every boundary member w either had
// p in its variable list (p is removed) or an element of p in its element
// list (absorbed and removed), and gains exactly one element (p); so
// |adj(w)|+|elems(w)| never exceeds the initial degree.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kMdThreads = 512;
constexpr int32_t kSmemDegCap = 12 * 1024;  // nodes up to this size keep degrees in smem
constexpr uint32_t kInfDeg = 0xffffffffu;

int grid_for(const mp_context& ctx, int64_t n, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), ctx.num_sms * 16LL)));
}

struct MdArgs {
  DGraph g;
  int32_t nn;
  const int32_t* node_of;
  const int32_t* node_offsets;
  const int32_t* node_vertices;
  const int32_t* local_of;   // position of v inside its node
  int32_t mode;              // 0 approx, 1 exact
  int32_t* adj;              // slot storage, CSR layout (global ids)
  int32_t* el;               // slot storage, CSR layout (element = pivot global id)
  int32_t* nadj;             // per vertex
  int32_t* nel;              // per vertex
  int32_t* bptr;             // per element (global id) -> pool offset (relative to node pool)
  int32_t* bsz;              // per element
  int32_t* vmark;            // per vertex, token = pivot + 1
  int32_t* emark;            // per element
  uint32_t* gdeg;            // per vertex (used when the node exceeds kSmemDegCap)
  int32_t* pool;             // all node pools
  const int64_t* pool_off;   // per node: [pool_off[i], pool_off[i+1]) = two halves
  int32_t* order_ws;         // per vertex scratch: pivots in order (node_vertices layout)
  int32_t* local_perm;       // output, node_vertices layout
  int32_t* overflow;         // set on pool exhaustion
  int32_t min_nv;            // md_kernel: only nodes with at least this many vertices
  const uint8_t* node_mask;  // non-null: order only nodes with mask != 0 (sharded C3 path)
};

__device__ __forceinline__ uint32_t md_key_deg(int64_t d) {
  return d >= static_cast<int64_t>(kInfDeg) ? kInfDeg - 1 : static_cast<uint32_t>(d);
}

__global__ void __launch_bounds__(kMdThreads) md_kernel(MdArgs a) {
  const int32_t node = blockIdx.x;
  const int32_t vb = a.node_offsets[node], nv = a.node_offsets[node + 1] - vb;
  if (nv == 0 || nv < a.min_nv || (a.node_mask && !a.node_mask[node])) return;
  const int32_t* verts = a.node_vertices + vb;
  int32_t* lperm = a.local_perm + vb;
  int32_t* order = a.order_ws + vb;
  if (a.mode == 2) {  // natural: identity (local_order.cpp:253-256)
    for (int32_t k = threadIdx.x; k < nv; k += blockDim.x) lperm[k] = k;
    return;
  }
  extern __shared__ uint32_t sdeg_dyn[];
  const bool smem_deg = nv <= kSmemDegCap;
  uint32_t* deg = smem_deg ? sdeg_dyn : a.gdeg + vb;  // indexed by local id

  __shared__ uint64_t red[32];
  __shared__ int32_t s_nb, s_cursor, s_half, s_need_compact;
  const int64_t pbase = a.pool_off[node];
  const int64_t pcap = (a.pool_off[node + 1] - pbase) / 2;

  // ---- induced subgraph: variable lists = neighbours inside the node
  for (int32_t k = threadIdx.x; k < nv; k += blockDim.x) {
    const int32_t v = verts[k];
    int32_t c = 0;
    const int32_t o = a.g.off[v];
    for (int32_t j = o; j < a.g.off[v + 1]; ++j) {
      const int32_t w = a.g.nbr[j];
      if (a.node_of[w] == node) a.adj[o + c++] = w;
    }
    a.nadj[v] = c;
    a.nel[v] = 0;
    a.bsz[v] = 0;
    a.vmark[v] = 0;
    a.emark[v] = 0;
    deg[k] = static_cast<uint32_t>(c);  // approx degree with no elements = |adj|
  }
  if (threadIdx.x == 0) s_cursor = 0, s_half = 0;
  __syncthreads();
  int32_t xcount = 0;  // exact mode: running token counter (same in every thread)

  for (int32_t k = 0; k < nv; ++k) {
    // ---- pivot: min (degree, local id)
    uint64_t best = ~0ull;
    for (int32_t i = threadIdx.x; i < nv; i += blockDim.x) {
      const uint32_t d = deg[i];
      if (d != kInfDeg) {
        const uint64_t kk = key_min(d, static_cast<uint32_t>(i));
        best = kk < best ? kk : best;
      }
    }
    best = block_min_u64(best, red);
    const int32_t kp = static_cast<int32_t>(best & 0xffffffffu);
    const int32_t p = verts[kp];
    const int32_t tok = p + 1;
    const int32_t np_adj = a.nadj[p], np_el = a.nel[p];
    const int32_t* padj = a.adj + a.g.off[p];
    const int32_t* pel = a.el + a.g.off[p];

    // ---- room for the new boundary (at most nv - k - 1 members)
    if (threadIdx.x == 0) {
      s_need_compact = (s_cursor + (nv - k)) > pcap;
      s_nb = 0;
      a.vmark[p] = tok;
    }
    __syncthreads();
    if (s_need_compact) {
      // copy live boundaries (bsz > 0) of the elements created so far into the
      // other half, element by element in pivot order
      int32_t* src = a.pool + pbase + (s_half ? pcap : 0);
      int32_t* dst = a.pool + pbase + (s_half ? 0 : pcap);
      int32_t run = 0;
      for (int32_t i0 = 0; i0 < k; i0 += blockDim.x) {
        const int32_t i = i0 + threadIdx.x;
        const int32_t e = i < k ? order[i] : -1;
        const int32_t sz = e >= 0 ? a.bsz[e] : 0;
        int32_t tot;
        __shared__ int32_t shs[32];
        const int32_t off = block_excl_scan(sz, shs, &tot);
        if (sz > 0) {
          const int32_t from = a.bptr[e];
          for (int32_t t = 0; t < sz; ++t) dst[run + off + t] = src[from + t];
          a.bptr[e] = run + off;
        }
        run += tot;
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        s_half ^= 1;
        s_cursor = run;
        if (run + (nv - k) > pcap) atomicExch(a.overflow, 1);
      }
      __syncthreads();
    }
    int32_t* half = a.pool + pbase + (s_half ? pcap : 0);
    int32_t* out = half + s_cursor;
    // ---- reach set: variables of p plus boundaries of p's elements
    for (int32_t i = threadIdx.x; i < np_adj; i += blockDim.x) {
      const int32_t w = padj[i];
      if (atomicExch(&a.vmark[w], tok) != tok) out[atomicAdd(&s_nb, 1)] = w;
    }
    for (int32_t ei = 0; ei < np_el; ++ei) {
      const int32_t e = pel[ei];
      const int32_t* bd = half + a.bptr[e];
      const int32_t sz = a.bsz[e];
      for (int32_t i = threadIdx.x; i < sz; i += blockDim.x) {
        const int32_t w = bd[i];
        if (atomicExch(&a.vmark[w], tok) != tok) out[atomicAdd(&s_nb, 1)] = w;
      }
    }
    for (int32_t ei = threadIdx.x; ei < np_el; ei += blockDim.x) a.emark[pel[ei]] = tok;
    __syncthreads();
    const int32_t nb = s_nb;
    if (threadIdx.x == 0) {
      a.bptr[p] = s_cursor;
      a.bsz[p] = nb;
      order[k] = p;
      lperm[k] = kp;
      deg[kp] = kInfDeg;
    }
    // absorbed elements' boundaries are dropped after the member updates
    __syncthreads();
    // ---- update every boundary member (elimination.cpp:75-83)
    for (int32_t i = threadIdx.x; i < nb; i += blockDim.x) {
      const int32_t w = out[i];
      const int32_t o = a.g.off[w];
      int32_t* wa = a.adj + o;
      int32_t c = 0;
      const int32_t na = a.nadj[w];
      // in-place compaction with 8 reads in flight ahead of the writes
      for (int32_t j0 = 0; j0 < na; j0 += 8) {
        int32_t xs[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) xs[q] = j0 + q < na ? wa[j0 + q] : -1;
        int32_t mk[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mk[q] = xs[q] >= 0 ? a.vmark[xs[q]] : tok;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (mk[q] != tok) wa[c++] = xs[q];
      }
      a.nadj[w] = c;
      int32_t* we = a.el + o;
      int32_t ce = 0;
      const int32_t ne = a.nel[w];
      int64_t d = c;
      for (int32_t j0 = 0; j0 < ne; j0 += 8) {
        int32_t es[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) es[q] = j0 + q < ne ? we[j0 + q] : -1;
        int32_t mk[8], bs[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mk[q] = es[q] >= 0 ? a.emark[es[q]] : tok, bs[q] = es[q] >= 0 ? a.bsz[es[q]] : 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (mk[q] != tok) {
            we[ce++] = es[q];
            d += bs[q];
          }
      }
      we[ce++] = p;
      d += nb;
      a.nel[w] = ce;
      if (a.mode == 0) deg[a.local_of[w]] = md_key_deg(d);
    }
    __syncthreads();
    for (int32_t ei = threadIdx.x; ei < np_el; ei += blockDim.x) a.bsz[pel[ei]] = 0;
    if (threadIdx.x == 0) {
      a.nadj[p] = 0;
      a.nel[p] = 0;
      s_cursor += nb;
    }
    if (a.mode == 1) {
      // exact degree (elimination.cpp:23-44): one block-wide marked union per member
      __shared__ int32_t s_cnt;
      for (int32_t i = 0; i < nb; ++i) {
        const int32_t w = out[i];
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        // negative tokens, unique per exact count; pivot tokens are positive
        const int32_t xt = -2 - (xcount++ & 0x3fffffff);
        if (threadIdx.x == 0) a.vmark[w] = xt;
        __syncthreads();
        const int32_t o = a.g.off[w];
        for (int32_t j = threadIdx.x; j < a.nadj[w]; j += blockDim.x) {
          const int32_t x = a.adj[o + j];
          if (atomicExch(&a.vmark[x], xt) != xt) atomicAdd(&s_cnt, 1);
        }
        for (int32_t ei = 0; ei < a.nel[w]; ++ei) {
          const int32_t e = a.el[o + ei];
          const int32_t* bd = half + a.bptr[e];
          for (int32_t j = threadIdx.x; j < a.bsz[e]; j += blockDim.x) {
            const int32_t x = bd[j];
            if (atomicExch(&a.vmark[x], xt) != xt) atomicAdd(&s_cnt, 1);
          }
        }
        __syncthreads();
        if (threadIdx.x == 0) deg[a.local_of[w]] = static_cast<uint32_t>(s_cnt);
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// Fast approximate-MD kernel (the default mode).  Node-local ids throughout:
// variable and element lists hold local ids (an element is named by its
// pivot's local id), and the per-vertex state lives in shared memory:
//   st[v]   = |adj| | |elems| << 16    deg[v] = approx degree (INF once gone)
//   mark[v] = token: a vertex mark while v is alive, the absorption mark of
//             element v once v is eliminated (the two uses never overlap)
//   bsz[e]  = boundary size of element e (0 = absorbed / empty)
//   blk[b]  = min (degree, id) key of the 32 vertices of block b
// Per pivot: argmin over blk (every warp, redundantly), reach collection,
// member updates, dirty-block refresh: three barriers (B2, B3, B4).
constexpr int32_t kMdFastCap = 6 * 1024;  // nodes up to this size use the fast kernel

__global__ void __launch_bounds__(kMdThreads) md_fast_kernel(MdArgs a) {
  const int32_t node = a.nn - 1 - static_cast<int32_t>(blockIdx.x);  // leaves (the big nodes) first
  const int32_t vb = a.node_offsets[node], nv = a.node_offsets[node + 1] - vb;
  if (nv == 0 || nv > kMdFastCap || (a.node_mask && !a.node_mask[node])) return;
  const int32_t* verts = a.node_vertices + vb;
  int32_t* lperm = a.local_perm + vb;
  int32_t* order = a.order_ws + vb;
  int32_t* bp = a.bptr + vb;  // element boundary offsets, local ids (node slab)
  extern __shared__ uint64_t md_sm[];
  const int32_t nb = (nv + 31) / 32;
  uint64_t* blk = md_sm;
  uint32_t* deg = reinterpret_cast<uint32_t*>(blk + nb);
  int32_t* mark = reinterpret_cast<int32_t*>(deg + nv);
  int32_t* bsz = mark + nv;
  int32_t* st = bsz + nv;
  int32_t* loff = st + nv;  // CSR offset of each local vertex (its list slots)
  uint32_t* dirty = reinterpret_cast<uint32_t*>(loff + nv);  // nb bits
  // this pivot's reach (local ids < kMdFastCap fit 16 bits), read back by the
  // member updates without a trip through the global pool
  int16_t* sreach = reinterpret_cast<int16_t*>(dirty + (nb + 31) / 32 + 1);
  __shared__ int32_t s_nbc[2], s_cursor, s_half, s_dcnt;
  __shared__ int32_t s_dlist[kMdThreads];  // dirty blocks of this pivot (<= reach + 1 distinct)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int64_t pbase = a.pool_off[node];
  const int64_t pcap = (a.pool_off[node + 1] - pbase) / 2;

  // induced subgraph in local ids; list slots at the vertex's CSR range
  for (int32_t k = threadIdx.x; k < nv; k += blockDim.x) {
    const int32_t v = verts[k];
    const int32_t o = a.g.off[v];
    int32_t c = 0;
    for (int32_t j = o; j < a.g.off[v + 1]; ++j) {
      const int32_t w = a.g.nbr[j];
      if (a.node_of[w] == node) a.adj[o + c++] = a.local_of[w];
    }
    if (c > 0x7fff) atomicExch(a.overflow, 2);  // packed list lengths: the general kernel redoes it
    st[k] = c;
    loff[k] = o;
    deg[k] = static_cast<uint32_t>(c);
    mark[k] = 0;
    bsz[k] = 0;
  }
  for (int32_t b = threadIdx.x; b < (nb + 31) / 32; b += blockDim.x) dirty[b] = 0;
  if (threadIdx.x == 0) s_cursor = 0, s_half = 0, s_dcnt = 0, s_nbc[0] = s_nbc[1] = 0;
  __syncthreads();
  for (int32_t b = wid; b < nb; b += nwarp) {
    const int32_t i = b * 32 + lane;
    const uint64_t m = warp_min_u64(i < nv ? key_min(deg[i], static_cast<uint32_t>(i)) : ~0ull);
    if (lane == 0) blk[b] = m;
  }
  __syncthreads();

  for (int32_t k = 0; k < nv; ++k) {
    // ---- pivot: min (degree, local id), computed by every warp (no barrier
    // to broadcast it; blk is stable since the previous B4)
    uint64_t best = ~0ull;
    for (int32_t b = lane; b < nb; b += 32) best = min(best, blk[b]);
    best = warp_min_u64(best);
    const int32_t p = static_cast<int32_t>(best & 0xffffffffu);
    const int32_t tok = k + 1;
    int32_t* cnt = &s_nbc[k & 1];
    const int32_t po = loff[p];
    const int32_t pst = st[p];
    const int32_t np_adj = pst & 0xffff, np_el = pst >> 16;
    if (s_cursor + (nv - k) > pcap) {  // block-uniform: compact live boundaries into the other half
      int32_t* src = a.pool + pbase + (s_half ? pcap : 0);
      int32_t* dst = a.pool + pbase + (s_half ? 0 : pcap);
      int32_t run = 0;
      for (int32_t i0 = 0; i0 < k; i0 += blockDim.x) {
        const int32_t i = i0 + threadIdx.x;
        const int32_t e = i < k ? order[i] : -1;
        const int32_t sz = e >= 0 ? bsz[e] : 0;
        int32_t tot;
        __shared__ int32_t shs[32];
        const int32_t off = block_excl_scan(sz, shs, &tot);
        if (sz > 0) {
          const int32_t from = bp[e];
          for (int32_t t = 0; t < sz; ++t) dst[run + off + t] = src[from + t];
          bp[e] = run + off;
        }
        run += tot;
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        s_half ^= 1;
        s_cursor = run;
        if (run + (nv - k) > pcap) atomicExch(a.overflow, 1);
      }
      __syncthreads();
    }
    int32_t* half = a.pool + pbase + (s_half ? pcap : 0);
    const int32_t cur0 = s_cursor;
    int32_t* out = half + cur0;
    // ---- reach set: variables of p plus boundaries of p's elements (p itself
    // is skipped explicitly; its mark is set for the member updates below)
    const int32_t* padj = a.adj + po;
    const int32_t* pel = a.el + po;
    for (int32_t i = threadIdx.x; i < np_adj; i += blockDim.x) {
      const int32_t w = padj[i];
      if (atomicExch(&mark[w], tok) != tok) {
        const int32_t at = atomicAdd(cnt, 1);
        out[at] = w;
        sreach[at] = static_cast<int16_t>(w);
      }
    }
    for (int32_t ei = 0; ei < np_el; ++ei) {
      const int32_t e = pel[ei];
      const int32_t* bd = half + bp[e];
      const int32_t sz = bsz[e];
      for (int32_t i = threadIdx.x; i < sz; i += blockDim.x) {
        const int32_t w = bd[i];
        if (w != p && atomicExch(&mark[w], tok) != tok) {
          const int32_t at = atomicAdd(cnt, 1);
          out[at] = w;
          sreach[at] = static_cast<int16_t>(w);
        }
      }
    }
    // absorbed elements get the pivot's token (element ids are dead vertices,
    // disjoint from the live vertices marked above)
    for (int32_t ei = threadIdx.x; ei < np_el; ei += blockDim.x) mark[pel[ei]] = tok;
    if (threadIdx.x == 0) {
      mark[p] = tok;
      bp[p] = cur0;
      order[k] = p;
      lperm[k] = p;
      deg[p] = 0xffffffffu;
      if (!(atomicOr(&dirty[(p >> 5) >> 5], 1u << ((p >> 5) & 31)) & (1u << ((p >> 5) & 31))))
        s_dlist[atomicAdd(&s_dcnt, 1)] = p >> 5;
    }
    __syncthreads();  // B2: reach, marks and absorption marks visible
    const int32_t nbd = *cnt;
    // ---- member updates (elimination.cpp:75-83) and their approx degrees
    for (int32_t i = threadIdx.x; i < nbd; i += blockDim.x) {
      const int32_t w = sreach[i];
      const int32_t o = loff[w];
      const int32_t wst = st[w];
      int32_t* wa = a.adj + o;
      int32_t c = 0;
      const int32_t na = wst & 0xffff, ne = wst >> 16;
      // lists are compacted in place: read 8 entries ahead of the writes so the
      // loads are in flight together (the compiler cannot reorder across the
      // possibly-aliasing stores)
      for (int32_t j0 = 0; j0 < na; j0 += 8) {
        int32_t xs[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) xs[q] = j0 + q < na ? wa[j0 + q] : -1;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (xs[q] >= 0 && mark[xs[q]] != tok) wa[c++] = xs[q];
      }
      int32_t* we = a.el + o;
      int32_t ce = 0;
      int64_t d = c + nbd;
      for (int32_t j0 = 0; j0 < ne; j0 += 8) {
        int32_t es[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) es[q] = j0 + q < ne ? we[j0 + q] : -1;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (es[q] >= 0 && mark[es[q]] != tok) {
            we[ce++] = es[q];
            d += bsz[es[q]];
          }
      }
      we[ce++] = p;
      st[w] = c | (ce << 16);
      deg[w] = md_key_deg(d);
      const uint32_t bit = 1u << ((w >> 5) & 31);
      if (!(atomicOr(&dirty[(w >> 5) >> 5], bit) & bit)) s_dlist[atomicAdd(&s_dcnt, 1)] = w >> 5;
    }
    __syncthreads();  // B3
    for (int32_t ei = threadIdx.x; ei < np_el; ei += blockDim.x) bsz[pel[ei]] = 0;
    if (threadIdx.x == 0) {
      bsz[p] = nbd;
      st[p] = 0;
      s_cursor += nbd;
      s_nbc[(k + 1) & 1] = 0;  // its last reader was the previous pivot, before this B2
    }
    // ---- refresh dirty blocks
    const int32_t ndirty = s_dcnt;
    for (int32_t q = wid; q < ndirty; q += nwarp) {
      const int32_t b = s_dlist[q];
      const int32_t i = b * 32 + lane;
      const uint64_t m = warp_min_u64(i < nv ? key_min(deg[i], static_cast<uint32_t>(i)) : ~0ull);
      if (lane == 0) {
        blk[b] = m;
        dirty[b >> 5] = 0;  // every set bit of the word is in the list
      }
    }
    __syncthreads();  // B4
    if (threadIdx.x == 0) s_dcnt = 0;
  }
}

__global__ void local_of_kernel(int32_t n, const int32_t* node_of, const int32_t* node_offsets,
                                const int32_t* node_vertices, int32_t* local_of) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t v = node_vertices[i];
    local_of[v] = i - node_offsets[node_of[v]];
  }
}
// per node pool capacity: 2 halves of (4 * degree sum + 2 * size + 64)
__global__ void node_pool_need(int32_t nn, const int32_t* node_offsets, const int32_t* node_vertices,
                               const int32_t* off, const uint8_t* node_mask, int64_t* need) {
  for (int32_t node = blockIdx.x; node < nn; node += gridDim.x) {
    const int32_t b = node_offsets[node], e = (node_mask && !node_mask[node]) ? b : node_offsets[node + 1];
    int64_t d = 0;
    for (int32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      const int32_t v = node_vertices[i];
      d += off[v + 1] - off[v];
    }
    __shared__ int64_t red[32];
    d = block_sum_i64(d, red);
    if (threadIdx.x == 0) need[node] = e > b ? 2 * (4 * d + 2LL * (e - b) + 64) : 0;
  }
}

}  // namespace

void order_tree_nodes_dev(mp_context& ctx, const DGraph& g, int32_t L, const int32_t* node_of,
                          const int32_t* node_offsets, const int32_t* node_vertices, int32_t mode,
                          int32_t* local_perm, const uint8_t* node_mask) {
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
  if (n == 0) return;
  DevBuf<int32_t> local_of(n, s), nadj(n, s), nel(n, s), bptr(n, s), bsz(n, s), vmark(n, s), emark(n, s),
      order(n, s), overflow(1, s);
  DevBuf<uint32_t> gdeg(n, s);
  DevBuf<int64_t> need(nn + 1, s), pool_off(nn + 1, s);
  int32_t m2 = 0;
  MP_CUDA(cudaMemcpyAsync(&m2, g.off + n, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  MP_KERNEL(ctx, local_of_kernel<<<grid_for(ctx, n), 256, 0, s>>>(n, node_of, node_offsets, node_vertices, local_of));
  MP_CUDA(cudaMemsetAsync(need, 0, sizeof(int64_t) * (nn + 1), s));
  MP_KERNEL(ctx, node_pool_need<<<std::min(nn, 4096), 256, 0, s>>>(nn, node_offsets, node_vertices, g.off, node_mask, need));
  {
    size_t tmp = 0;
    MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, need.get(), pool_off.get(), nn + 1, s));
    DevBuf<char> t(tmp, s);
    MP_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, need.get(), pool_off.get(), nn + 1, s));
  }
  int64_t pool_total = 0;
  MP_CUDA(cudaMemcpyAsync(&pool_total, pool_off.get() + nn, 8, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaMemsetAsync(overflow, 0, 4, s));
  MP_CUDA(cudaStreamSynchronize(s));
  // slot lists and the element-boundary pool: one persistent context slab
  SlabCarve sc;
  const size_t o_adj = sc.add(sizeof(int32_t) * std::max(m2, 1)), o_el = sc.add(sizeof(int32_t) * std::max(m2, 1)),
               o_pool = sc.add(sizeof(int32_t) * std::max<int64_t>(pool_total, 1));
  void* slab = ctx.slab(kSlabMd, sc.total);
  int32_t* adj = SlabCarve::at<int32_t>(slab, o_adj);
  int32_t* el = SlabCarve::at<int32_t>(slab, o_el);
  int32_t* pool = SlabCarve::at<int32_t>(slab, o_pool);
  MdArgs a{};
  a.g = g, a.nn = nn, a.node_of = node_of, a.node_offsets = node_offsets, a.node_vertices = node_vertices;
  a.local_of = local_of, a.mode = mode, a.adj = adj, a.el = el, a.nadj = nadj, a.nel = nel;
  a.bptr = bptr, a.bsz = bsz, a.vmark = vmark, a.emark = emark, a.gdeg = gdeg, a.pool = pool;
  a.pool_off = pool_off, a.order_ws = order, a.local_perm = local_perm, a.overflow = overflow;
  a.node_mask = node_mask;
  const size_t smem = sizeof(uint32_t) * kSmemDegCap;
  allow_max_smem(md_kernel, ctx.device);
  const int kt__ = ctx.ktime_begin(kKMd);
  if (mode == 0) {
    // largest node decides the shared-memory footprint of the fast kernel
    std::vector<int32_t> hoff(nn + 1);
    MP_CUDA(cudaMemcpyAsync(hoff.data(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    int32_t maxnv = 0;
    for (int32_t i = 0; i < nn; ++i) maxnv = std::max(maxnv, hoff[i + 1] - hoff[i]);
    const int32_t fast_nv = std::min(maxnv, kMdFastCap);
    const int32_t fnb = (fast_nv + 31) / 32;
    const size_t fsmem = sizeof(uint64_t) * fnb + sizeof(int32_t) * 5 * fast_nv + sizeof(uint32_t) * ((fnb + 31) / 32 + 1) +
                         sizeof(int16_t) * (fast_nv + 2);
    allow_max_smem(md_fast_kernel, ctx.device);
    MP_KERNEL(ctx, md_fast_kernel<<<nn, kMdThreads, fsmem, s>>>(a));
    int32_t h_flag = 0;
    MP_CUDA(cudaMemcpyAsync(&h_flag, overflow.get(), 4, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (h_flag == 2) {  // a vertex of degree > 32767: the general kernel orders every node
      MP_CUDA(cudaMemsetAsync(overflow, 0, 4, s));
      MP_KERNEL(ctx, md_kernel<<<nn, kMdThreads, smem, s>>>(a));
    } else if (maxnv > kMdFastCap) {
      a.min_nv = kMdFastCap + 1;  // the general kernel takes the remaining (large) nodes
      MP_KERNEL(ctx, md_kernel<<<nn, kMdThreads, smem, s>>>(a));
    }
  } else {
    MP_KERNEL(ctx, md_kernel<<<nn, kMdThreads, smem, s>>>(a));
  }
  ctx.ktime_end(kt__);
  int32_t h_over = 0;
  MP_CUDA(cudaMemcpyAsync(&h_over, overflow, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (h_over) throw Error(MP_ENOMEM, "minimum_degree: element pool exhausted");
}

}  // namespace mp
