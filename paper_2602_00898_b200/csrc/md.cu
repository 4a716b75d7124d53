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
constexpr int32_t kSmemDegCap = 48 * 1024;  // nodes up to this size keep degrees in smem (C3's 39K-vertex leaves)
constexpr uint32_t kInfDeg = 0xffffffffu;
constexpr int32_t kMdDirtyCap = 1024;  // dirty blocks listed per pivot (more: recompute all)

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
  const int32_t* sched;      // md_smem_kernel: node per CTA, largest first
  uint64_t* gblk;            // md_node_global: block minima when shared memory is short
  uint32_t* gdbits;          // md_node_global: dirty-block bits when shared memory is short
  int64_t gsmem_bytes;       // md_node_global: dynamic shared memory of the launch
  int64_t smem_bytes;        // md_smem_kernel: dynamic shared memory per CTA
  const uint8_t* node_mask;  // non-null: order only nodes with mask != 0 (sharded C3 path)
};

__device__ __forceinline__ uint32_t md_key_deg(int64_t d) {
  return d >= static_cast<int64_t>(kInfDeg) ? kInfDeg - 1 : static_cast<uint32_t>(d);
}

// One node with its lists, pool and (above kSmemDegCap) degrees in global
// memory: exact mode, natural mode, and approximate-mode nodes too large for
// md_smem_kernel.
// DT = uint16_t: degrees in shared memory as 16 bits (0xffff = eliminated),
// for nodes below 65,535 vertices -- half the shared memory, so two 256-thread
// CTAs share an SM (C3's 256 leaves of ~39K vertices run in one wave).  The
// pivot loop is SM-throughput bound, not latency bound: two co-resident
// leaves each run at about half speed, so the gain over two waves of one
// 512-thread CTA per SM comes from the 256-thread CTA (C3 MD 370 -> 335 ms;
// 256 threads one per SM: 334; 128 threads two per SM: 394).
template <class DT = uint32_t>
__device__ __forceinline__ void md_node_global(const MdArgs& a, int32_t node) {
  const int32_t vb = a.node_offsets[node], nv = a.node_offsets[node + 1] - vb;
  if (nv == 0 || (a.node_mask && !a.node_mask[node])) return;
  const int32_t* verts = a.node_vertices + vb;
  int32_t* lperm = a.local_perm + vb;
  int32_t* order = a.order_ws + vb;
  if (a.mode == 2) {  // natural: identity (local_order.cpp:253-256)
    for (int32_t k = threadIdx.x; k < nv; k += blockDim.x) lperm[k] = k;
    return;
  }
  extern __shared__ uint32_t sdeg_dyn[];
  constexpr bool kDeg16 = sizeof(DT) == 2;
  const bool smem_deg = kDeg16 || nv <= kSmemDegCap;
  DT* deg;  // indexed by local id
  if constexpr (kDeg16) deg = reinterpret_cast<DT*>(sdeg_dyn);
  else deg = smem_deg ? sdeg_dyn : a.gdeg + vb;
  // stored degree <-> 32-bit degree (kInfDeg once eliminated)
  auto dget = [&](int32_t i) -> uint32_t {
    const uint32_t d = deg[i];
    if constexpr (kDeg16) return d == 0xffffu ? kInfDeg : d;
    else return d;
  };
  auto dput = [&](int32_t i, uint32_t d) {
    if constexpr (kDeg16) deg[i] = static_cast<DT>(d == kInfDeg ? 0xffffu : d);
    else deg[i] = d;
  };

  __shared__ uint64_t red[32];
  __shared__ int32_t s_nb, s_cursor, s_half, s_need_compact, s_ndirty, s_ip, s_dlist[kMdDirtyCap];
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
    dput(k, static_cast<uint32_t>(c));  // approx degree with no elements = |adj|
  }
  if (threadIdx.x == 0) s_cursor = 0, s_half = 0, s_ndirty = 0;
  __syncthreads();
  int32_t xcount = 0;  // exact mode: running token counter (same in every thread)
  // (degree, id) block minima: the argmin reads nbk entries, not nv; a lowered
  // key lowers its block's minimum at once, a block whose minimum rose is
  // recomputed at the end of the pivot (blk / dirty bits in shared memory
  // after the degrees when they fit, else in the node's global slab)
  const int32_t nbk = (nv + 31) / 32, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int64_t deg_bytes = smem_deg ? ((static_cast<int64_t>(sizeof(DT)) * nv + 7) & ~7LL) : 0;
  const bool blk_sm = deg_bytes + 8LL * nbk + 4LL * (nbk / 32 + 1) <= a.gsmem_bytes;
  uint64_t* blk = blk_sm ? reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(sdeg_dyn) + deg_bytes)
                         : a.gblk + (vb >> 5) + node;
  uint32_t* dbits = blk_sm ? reinterpret_cast<uint32_t*>(blk + nbk) : a.gdbits + (vb >> 10) + 2 * node;
  auto key_of = [&](int32_t i) -> uint64_t {
    const uint32_t d = i < nv ? dget(i) : kInfDeg;
    return d != kInfDeg ? key_min(d, static_cast<uint32_t>(i)) : ~0ull;
  };
  auto mark_dirty = [&](int32_t b) {
    const uint32_t bit = 1u << (b & 31);
    if (!(atomicOr(&dbits[b >> 5], bit) & bit)) {
      const int32_t at = atomicAdd(&s_ndirty, 1);
      if (at < kMdDirtyCap) s_dlist[at] = b;
    }
  };
  // a member's degree changed from od to nd
  auto rekey = [&](int32_t lw, uint32_t od, uint32_t nd) {
    const uint64_t ok = key_min(od, static_cast<uint32_t>(lw)), nk = key_min(nd, static_cast<uint32_t>(lw));
    if (nk < ok) atomicMin(reinterpret_cast<unsigned long long*>(&blk[lw >> 5]), nk);
    else if (nk > ok && ok == blk[lw >> 5]) mark_dirty(lw >> 5);
  };
  for (int32_t b = threadIdx.x; b <= nbk / 32; b += blockDim.x) dbits[b] = 0;
  for (int32_t b = wid; b < nbk; b += nwarp) {
    const uint64_t m = warp_min_u64(key_of(b * 32 + lane));
    if (lane == 0) blk[b] = m;
  }
  __syncthreads();

  for (int32_t k = 0; k < nv; ++k) {
    // ---- pivot: min (degree, local id) over the block minima
    uint64_t best = ~0ull;
    for (int32_t b = threadIdx.x; b < nbk; b += blockDim.x) best = min(best, blk[b]);
    best = block_min_u64(best, red);
    if (threadIdx.x == 0) s_ndirty = 0;  // every reader of the last pivot's count is past its barrier
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
    // ---- reach set: variables of p plus boundaries of p's elements.  With
    // at most one element the parts are disjoint and duplicate-free (adj(p)
    // lost that element's boundary when it formed; p appears in it once), so
    // they are copied with plain stores and p is swapped out after the
    // member updates; several elements deduplicate through the marks.
    const bool simple = np_el <= 1;
    int32_t ptotal = 0;
    if (simple) {
      const int32_t e1 = np_el ? pel[0] : 0;
      const int32_t* bd = half + (np_el ? a.bptr[e1] : 0);
      const int32_t sz = np_el ? a.bsz[e1] : 0;
      ptotal = np_adj + sz;
      for (int32_t i = threadIdx.x; i < ptotal; i += blockDim.x) {
        const int32_t w = i < np_adj ? padj[i] : bd[i - np_adj];
        out[i] = w;
        if (w == p) s_ip = i;
        else a.vmark[w] = tok;
      }
      if (threadIdx.x == 0) s_nb = ptotal - np_el;
    } else {
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
    }
    for (int32_t ei = threadIdx.x; ei < np_el; ei += blockDim.x) a.emark[pel[ei]] = tok;
    __syncthreads();
    const int32_t nb = s_nb;
    const int32_t nscan = simple ? ptotal : nb;  // out entries to visit (p among them when simple)
    if (threadIdx.x == 0) {
      a.bptr[p] = s_cursor;
      a.bsz[p] = nb;
      order[k] = p;
      lperm[k] = kp;
      dput(kp, kInfDeg);
      mark_dirty(kp >> 5);  // the pivot was its block's minimum
    }
    // absorbed elements' boundaries are dropped after the member updates
    __syncthreads();
    // ---- update every boundary member (elimination.cpp:75-83).  The
    // member's scalars, then the first eight slots of BOTH its lists, then
    // their marks and element sizes are loaded as three waves of independent
    // L2 requests (the stores of the in-place compactions come after them);
    // longer lists continue eight slots at a time.
    for (int32_t i = threadIdx.x; i < nscan; i += blockDim.x) {
      const int32_t w = out[i];
      if (w == p) continue;
      const int32_t o = a.g.off[w];
      const int32_t na = a.nadj[w], ne = a.nel[w];
      const int32_t lw = a.mode == 0 ? a.local_of[w] : 0;
      int32_t* wa = a.adj + o;
      int32_t* we = a.el + o;
      int32_t xs[8], es[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) xs[q] = q < na ? wa[q] : -1, es[q] = q < ne ? we[q] : -1;
      int32_t mx[8], me[8], bs[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        mx[q] = xs[q] >= 0 ? a.vmark[xs[q]] : tok;
        me[q] = es[q] >= 0 ? a.emark[es[q]] : tok;
        bs[q] = es[q] >= 0 ? a.bsz[es[q]] : 0;
      }
      int32_t c = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (mx[q] != tok) wa[c++] = xs[q];
      for (int32_t j0 = 8; j0 < na; j0 += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) xs[q] = j0 + q < na ? wa[j0 + q] : -1;
#pragma unroll
        for (int q = 0; q < 8; ++q) mx[q] = xs[q] >= 0 ? a.vmark[xs[q]] : tok;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (mx[q] != tok) wa[c++] = xs[q];
      }
      a.nadj[w] = c;
      int32_t ce = 0;
      int64_t d = c;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (me[q] != tok) {
          we[ce++] = es[q];
          d += bs[q];
        }
      for (int32_t j0 = 8; j0 < ne; j0 += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) es[q] = j0 + q < ne ? we[j0 + q] : -1;
#pragma unroll
        for (int q = 0; q < 8; ++q) me[q] = es[q] >= 0 ? a.emark[es[q]] : tok, bs[q] = es[q] >= 0 ? a.bsz[es[q]] : 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (me[q] != tok) {
            we[ce++] = es[q];
            d += bs[q];
          }
      }
      we[ce++] = p;
      d += nb;
      a.nel[w] = ce;
      if (a.mode == 0) {
        const uint32_t od = dget(lw), nd = md_key_deg(d);
        dput(lw, nd);
        rekey(lw, od, nd);
      }
    }
    __syncthreads();
    if (simple && np_el && threadIdx.x == 0 && s_ip != ptotal - 1) out[s_ip] = out[ptotal - 1];  // p's boundary without p
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
        if (threadIdx.x == 0) {
          const int32_t lw = a.local_of[w];
          const uint32_t od = dget(lw), nd = static_cast<uint32_t>(s_cnt);
          dput(lw, nd);
          rekey(lw, od, nd);
        }
        __syncthreads();
      }
    }
    __syncthreads();
    const int32_t ndirty = s_ndirty;
    if (ndirty > kMdDirtyCap) {  // list overflow: every block
      for (int32_t b = wid; b < nbk; b += nwarp) {
        const uint64_t m = warp_min_u64(key_of(b * 32 + lane));
        if (lane == 0) blk[b] = m;
      }
      for (int32_t b = threadIdx.x; b <= nbk / 32; b += blockDim.x) dbits[b] = 0;
    } else {
      for (int32_t q = wid; q < ndirty; q += nwarp) {
        const int32_t b = s_dlist[q];
        const uint64_t m = warp_min_u64(key_of(b * 32 + lane));
        if (lane == 0) {
          blk[b] = m;
          atomicAnd(&dbits[b >> 5], ~(1u << (b & 31)));
        }
      }
    }
    __syncthreads();
  }
}

// md_kernel's dynamic shared memory for nodes up to nv vertices: their
// degrees (when nv <= kSmemDegCap) plus room for the block minima and
// dirty bits (16 KB covers 2K blocks = 64K vertices).
inline size_t md_global_smem(int64_t nv) {
  return sizeof(uint32_t) * static_cast<size_t>(std::min<int64_t>(std::max<int64_t>(nv, 1), kSmemDegCap)) + 16384 + 512;
}

__global__ void __launch_bounds__(kMdThreads) md_kernel(MdArgs a) {
  md_node_global(a, a.sched ? a.sched[blockIdx.x] : static_cast<int32_t>(blockIdx.x));
}
constexpr int kMd16Threads = 256;
constexpr int64_t kMd16MaxNv = 65534;  // 16-bit degrees: every degree < nv <= 0xfffe
inline size_t md_global_smem16(int64_t nv) {
  return ((2 * static_cast<size_t>(std::max<int64_t>(nv, 1)) + 7) & ~size_t(7)) + 16384 + 512;
}
__global__ void __launch_bounds__(kMd16Threads, 2) md_kernel16(MdArgs a) {
  md_node_global<uint16_t>(a, a.sched[blockIdx.x]);
}

// Shared-memory approximate-MD kernel (the default mode).  The whole
// elimination state of a node lives in one CTA's shared memory, in node-local
// ids, so a pivot's dependent chain never leaves the SM; four warps run it
// (cheap barriers, one reach member per thread):
//   kd[v]   32-bit key (approx degree << 13 | v), ~0 once eliminated
//   blk[b]  min key of the 32 vertices of block b (the argmin is a min over
//           blk); a lowered key lowers it at once (atomicMin), a block whose
//           minimum rose (the pivot's, a member that was its block minimum)
//           is recomputed after the member updates
//   st[v]   live: |adj| | |elems| << 16; element: |boundary| (0 = absorbed)
//   ebp[e]  boundary offset of element e in the current pool half
//   L[loff[v] .. loff[v+1])  v's list slots: variables from the front, elements
//           from the back (|adj| + |elems| never exceeds the initial degree)
//   pool    element boundaries, two halves (compaction copies the live ones)
//   inr / absb  bit sets: this pivot's reach, the elements it absorbs
// The approx degree of a member is |adj| + sum of its elements' boundaries <=
// deg0 * nv, so keys are exact while max local degree * nv < 2^19.  A node
// whose boundaries outgrow the shared halves continues with halves in its
// global pool slab; a node whose lists or keys do not fit is ordered by
// md_node_global in the same CTA.
constexpr int32_t kMdSmemMaxNv = 8192;  // local ids in 13 bits
constexpr int32_t kMdMinHalf = 1024;    // smallest shared pool half worth running with
constexpr uint32_t kKeyInf = 0xffffffffu;
constexpr int kMdSmemThreads = 128;  // four warps: cheap barriers, one member per thread

// Two layouts of the per-vertex state.  Wide: u32 list state / offsets and
// u16 stamps (k + 1, unique for the whole node).  Compact (nodes that do not
// fit wide, C5's 8K-vertex leaves): u16 state / offsets (degree < 256, degree
// sum < 2^16) and u8 stamps unique inside windows of 255 pivots.
struct MdWide {
  using S = uint32_t;
  using T = uint16_t;
  static constexpr int kShift = 16;
  static constexpr uint32_t kMask = 0xffffu;
  static constexpr int32_t kWindow = 1 << 30;
};
struct MdCompact {
  using S = uint16_t;
  using T = uint8_t;
  static constexpr int kShift = 8;
  static constexpr uint32_t kMask = 0xffu;
  static constexpr int32_t kWindow = 255;
};

template <class Lay>
__host__ __device__ inline int64_t md_smem_fixed(int32_t nv) {
  const int64_t nb = (nv + 31) / 32;
  const int64_t sw = sizeof(typename Lay::S), tw = sizeof(typename Lay::T);
  // u32: block minima, keys, boundary offsets, dedup bits, dirty stamps; then
  // list state, list offsets (S) and the reach / absorbed stamps (T), 4-byte padded
  return 4 * nb + 8LL * nv + 8 * nb + ((sw * nv + 3) & ~3) + ((sw * (nv + 1) + 3) & ~3) + 2 * ((tw * nv + 3) & ~3) + 16;
}

template <class Lay>
__global__ void __launch_bounds__(kMdSmemThreads) md_smem_kernel(MdArgs a) {
  using S = typename Lay::S;
  using T = typename Lay::T;
  const int32_t node = a.sched[blockIdx.x];  // largest nodes first
  const int32_t vb = a.node_offsets[node], nv = a.node_offsets[node + 1] - vb;
  if (nv == 0 || (a.node_mask && !a.node_mask[node])) return;
  const int32_t* verts = a.node_vertices + vb;
  int32_t* lperm = a.local_perm + vb;
  extern __shared__ uint64_t md_sm[];
  const int32_t nb = (nv + 31) / 32;
  uint32_t* blk = reinterpret_cast<uint32_t*>(md_sm);
  uint32_t* kd = blk + nb;
  uint32_t* ebp = kd + nv;
  uint32_t* inr = ebp + nv;
  uint32_t* dstp = inr + nb;  // dirty-block stamp: k + 1 = listed for refresh after pivot k
  char* cb = reinterpret_cast<char*>(dstp + nb);
  S* st = reinterpret_cast<S*>(cb);  // live: |adj| | |elems| << kShift; element: |boundary|
  cb += (sizeof(S) * nv + 3) & ~3;
  S* loff = reinterpret_cast<S*>(cb);  // nv + 1 list offsets
  cb += (sizeof(S) * (nv + 1) + 3) & ~3;
  T* mk = reinterpret_cast<T*>(cb);  // reach stamp
  cb += (sizeof(T) * nv + 3) & ~3;
  T* ea = reinterpret_cast<T*>(cb);  // absorbed stamp
  cb += (sizeof(T) * nv + 3) & ~3;
  uint16_t* L = reinterpret_cast<uint16_t*>(cb);
  __shared__ int32_t s_cursor, s_cap, s_inglobal, s_maxdeg, s_nbd[2], s_ndirty, s_ip, sh[32];
  __shared__ int32_t s_dlist[kMdSmemMaxNv / 32];
  __shared__ int64_t s_red64[32];
  __shared__ uint16_t* s_cur;
  __shared__ uint16_t* s_other;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;

  // ---- local degrees -> list slot offsets
  if (threadIdx.x == 0) s_maxdeg = 0;
  __syncthreads();
  int32_t mymax = 0;
  for (int32_t k = threadIdx.x; k < nv; k += blockDim.x) {
    const int32_t v = verts[k];
    int32_t c = 0;
    for (int32_t j = a.g.off[v]; j < a.g.off[v + 1]; ++j) c += a.node_of[a.g.nbr[j]] == node;
    st[k] = c;
    mymax = max(mymax, c);
  }
  atomicMax(&s_maxdeg, mymax);
  __syncthreads();
  int32_t run = 0;
  for (int32_t b0 = 0; b0 < nv; b0 += blockDim.x) {
    const int32_t k = b0 + threadIdx.x;
    int32_t tot;
    const int32_t ex = block_excl_scan(k < nv ? static_cast<int32_t>(st[k]) : 0, sh, &tot);
    if (k < nv) loff[k] = static_cast<S>(run + ex);
    run += tot;
  }
  const int64_t D = run;
  const int64_t half = (a.smem_bytes - md_smem_fixed<Lay>(nv) - 2 * D) / 4;  // u16 entries per pool half
  if (half < kMdMinHalf || static_cast<int64_t>(s_maxdeg) * nv >= (1LL << 19) ||
      static_cast<uint32_t>(s_maxdeg) > Lay::kMask || static_cast<uint64_t>(D) > static_cast<uint64_t>(S(~S(0)))) {
    __syncthreads();
    md_node_global(a, node);  // lists or keys do not fit: global state
    return;
  }
  if (threadIdx.x == 0) {
    loff[nv] = static_cast<S>(D);
    s_cursor = 0, s_inglobal = 0;
    s_cap = static_cast<int32_t>(half);
    s_cur = L + D;
    s_other = L + D + half;
  }
  for (int32_t b = threadIdx.x; b < nb; b += blockDim.x) inr[b] = 0, dstp[b] = 0;
  for (int32_t i = threadIdx.x; i < nv; i += blockDim.x) mk[i] = 0, ea[i] = 0;
  if (threadIdx.x == 0) s_nbd[0] = s_nbd[1] = 0, s_ndirty = 0;
  // induced subgraph in local ids
  for (int32_t k = threadIdx.x; k < nv; k += blockDim.x) {
    const int32_t v = verts[k];
    const uint32_t o = loff[k];
    int32_t c = 0;
    for (int32_t j = a.g.off[v]; j < a.g.off[v + 1]; ++j) {
      const int32_t w = a.g.nbr[j];
      if (a.node_of[w] == node) L[o + c++] = static_cast<uint16_t>(a.local_of[w]);
    }
    st[k] = static_cast<S>(c);
    kd[k] = (static_cast<uint32_t>(c) << 13) | static_cast<uint32_t>(k);
  }
  __syncthreads();
  for (int32_t b = wid; b < nb; b += nwarp) {
    const int32_t i = b * 32 + lane;
    const uint32_t m = __reduce_min_sync(0xffffffffu, i < nv ? kd[i] : kKeyInf);
    if (lane == 0) blk[b] = m;
  }
  __syncthreads();

  // ---- the pivots
  const uint32_t below = (1u << lane) - 1;
  // a block whose minimum may have risen is recomputed after the member updates
  auto mark_dirty = [&](int32_t b, uint32_t sp) {
    if (atomicExch(&dstp[b], sp) != sp) s_dlist[atomicAdd(&s_ndirty, 1)] = b;
  };
  for (int32_t k = 0; k < nv; ++k) {
    // 8-bit stamps: unique inside a window of 255 pivots; the arrays are
    // cleared when a window starts (every user of the old stamps is behind B4)
    if (Lay::kWindow < kMdSmemMaxNv && k > 0 && k % Lay::kWindow == 0) {
      for (int32_t i = threadIdx.x; i < nv; i += blockDim.x) mk[i] = 0, ea[i] = 0;
      __syncthreads();
    }
    const T stamp = static_cast<T>(k % Lay::kWindow + 1);
    const uint32_t dstamp = static_cast<uint32_t>(k + 1);
    // pivot: min key over the block minima (every warp; blk is stable since B4)
    uint32_t best = kKeyInf;
#pragma unroll 4
    for (int32_t b = lane; b < nb; b += 32) best = min(best, blk[b]);
    best = __reduce_min_sync(0xffffffffu, best);
    const int32_t p = static_cast<int32_t>(best & 0x1fffu);
    int32_t* cnt = &s_nbd[k & 1];
    if (s_cursor + (nv - k) > s_cap) {  // block-uniform: compact the live boundaries
      int64_t live = 0;
      for (int32_t e = threadIdx.x; e < nv; e += blockDim.x)
        if (kd[e] == kKeyInf) live += st[e];
      live = block_sum_i64(live, s_red64);
      uint16_t* src = s_cur;
      uint16_t* dst;
      int64_t cap;
      bool to_global = false;
      if (!s_inglobal && live + (nv - k) <= half) {
        dst = s_other, cap = half;
      } else {
        // global halves: the node's slab of the int32 pool, as u16 entries
        const int64_t pb = a.pool_off[node], gcap = a.pool_off[node + 1] - pb;  // u16 entries per half
        uint16_t* g0 = reinterpret_cast<uint16_t*>(a.pool + pb);
        dst = (s_inglobal && src == g0) ? g0 + gcap : g0;
        cap = gcap;
        to_global = true;
      }
      int32_t crun = 0;
      for (int32_t b0 = 0; b0 < nv; b0 += blockDim.x) {
        const int32_t e = b0 + threadIdx.x;
        const int32_t sz = (e < nv && kd[e] == kKeyInf) ? static_cast<int32_t>(st[e]) : 0;
        int32_t tot;
        const int32_t ex = block_excl_scan(sz, sh, &tot);
        const uint32_t from = sz > 0 ? ebp[e] : 0;
        if (sz > 0) ebp[e] = static_cast<uint32_t>(crun + ex);
        // each warp copies its live boundaries one element at a time
        uint32_t live_m = __ballot_sync(0xffffffffu, sz > 0);
        while (live_m) {
          const int l = __ffs(live_m) - 1;
          live_m &= live_m - 1;
          const int32_t szl = __shfl_sync(0xffffffffu, sz, l);
          const uint32_t fl = __shfl_sync(0xffffffffu, from, l);
          const int32_t tl = crun + __shfl_sync(0xffffffffu, ex, l);
          for (int32_t t = lane; t < szl; t += 32) dst[tl + t] = src[fl + t];
        }
        crun += tot;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (!to_global) s_other = src;
        s_cur = dst;
        s_cap = static_cast<int32_t>(cap);
        s_inglobal = to_global ? 1 : 0;
        s_cursor = crun;
        if (crun + (nv - k) > cap) atomicExch(a.overflow, 1);
      }
      __syncthreads();
    }
    uint16_t* cur = s_cur;
    const int32_t cur0 = s_cursor;
    uint16_t* out = cur + cur0;
    const uint32_t pst = st[p];
    const int32_t np_adj = pst & Lay::kMask, np_el = pst >> Lay::kShift;
    const uint32_t po = loff[p], pe = loff[p + 1];
    // ---- reach: variables of p plus the boundaries of p's elements.  With at
    // most one element the parts need no deduplication: adj(p) lost every
    // member of that element's boundary when the element formed (and lists
    // only shrink), the boundary holds distinct live vertices, p among them
    // once.  So they are copied as they are (p's entry is swapped out after
    // the member updates) and the count is known without a barrier.
    int32_t nbd = 0, ptotal = 0;
    const bool simple = np_el <= 1;
    if (simple) {
      const int32_t e1 = np_el ? L[pe - 1] : 0;
      const uint16_t* bd = cur + (np_el ? ebp[e1] : 0);
      const int32_t sz = np_el ? static_cast<int32_t>(st[e1]) : 0;
      ptotal = np_adj + sz;
      nbd = ptotal - np_el;
      if (np_el && threadIdx.x == 0) ea[e1] = stamp;
      for (int32_t i = threadIdx.x; i < ptotal; i += blockDim.x) {
        const int32_t w = i < np_adj ? L[po + i] : bd[i - np_adj];
        out[i] = static_cast<uint16_t>(w);
        if (w == p) s_ip = i;
        else mk[w] = stamp;
      }
    } else {  // several elements: deduplicate (warp-aggregated appends)
      for (int32_t i0 = 0; i0 < np_adj; i0 += blockDim.x) {
        const int32_t i = i0 + threadIdx.x;
        bool fresh = false;
        int32_t w = 0;
        if (i < np_adj) {
          w = L[po + i];
          const uint32_t bit = 1u << (w & 31);
          fresh = !(atomicOr(&inr[w >> 5], bit) & bit);
        }
        const int32_t at = warp_append(cnt, fresh);
        if (fresh) out[at] = static_cast<uint16_t>(w), mk[w] = stamp;
      }
      for (int32_t ei = 0; ei < np_el; ++ei) {
        const int32_t e = L[pe - 1 - ei];
        const uint16_t* bd = cur + ebp[e];
        const int32_t sz = static_cast<int32_t>(st[e]);
        if (threadIdx.x == 0) ea[e] = stamp;
        for (int32_t i0 = 0; i0 < sz; i0 += blockDim.x) {
          const int32_t i = i0 + threadIdx.x;
          bool fresh = false;
          int32_t w = 0;
          if (i < sz) {
            w = bd[i];
            const uint32_t bit = 1u << (w & 31);
            fresh = w != p && !(atomicOr(&inr[w >> 5], bit) & bit);
          }
          const int32_t at = warp_append(cnt, fresh);
          if (fresh) out[at] = static_cast<uint16_t>(w), mk[w] = stamp;
        }
      }
    }
    // the pivot's own bookkeeping on the last thread (thread 0 leads the
    // reach copy); its block, whose minimum p was, is refreshed after the
    // member updates by the last warp without going through the dirty list
    if (threadIdx.x == blockDim.x - 1) {
      ebp[p] = static_cast<uint32_t>(cur0);
      lperm[k] = p;
      kd[p] = kKeyInf;
    }
    __syncthreads();  // B2
    if (!simple) nbd = ptotal = *cnt;
    // ---- member updates (elimination.cpp:75-83), one member per thread; a
    // lowered key lowers its block's minimum at once, a raised block minimum
    // is recomputed below
    for (int32_t i = threadIdx.x; i < ptotal; i += blockDim.x) {
      const int32_t w = out[i];
      if (w == p) continue;
      const uint32_t o = loff[w], oe = loff[w + 1];
      const uint32_t wst = st[w];
      const int32_t na = wst & Lay::kMask, ne = wst >> Lay::kShift;
      // both lists in chunks of four: the chunk's slots, then their bit-set
      // words and sizes, are independent loads in flight together (a chunk's
      // compacting writes land at or below its reads)
      int32_t c = 0;
      for (int32_t j0 = 0; j0 < na; j0 += 4) {
        int32_t x[4];
        T iw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = j0 + q < na ? L[o + j0 + q] : p;
#pragma unroll
        for (int q = 0; q < 4; ++q) iw[q] = mk[x[q]];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (x[q] != p && iw[q] != stamp) L[o + c++] = static_cast<uint16_t>(x[q]);
      }
      int32_t ce = 0;
      uint32_t d = static_cast<uint32_t>(c + nbd);
      for (int32_t j0 = 0; j0 < ne; j0 += 4) {
        int32_t e[4];
        T ab[4];
        uint32_t sz[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) e[q] = j0 + q < ne ? L[oe - 1 - (j0 + q)] : -1;
#pragma unroll
        for (int q = 0; q < 4; ++q) ab[q] = e[q] >= 0 ? ea[e[q]] : stamp;
#pragma unroll
        for (int q = 0; q < 4; ++q) sz[q] = e[q] >= 0 ? st[e[q]] : 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (ab[q] != stamp) {
            L[oe - 1 - ce++] = static_cast<uint16_t>(e[q]);
            d += sz[q];
          }
      }
      L[oe - 1 - ce++] = static_cast<uint16_t>(p);
      st[w] = static_cast<S>(c | (ce << Lay::kShift));
      const uint32_t nk = (d << 13) | static_cast<uint32_t>(w), ok = kd[w];
      kd[w] = nk;
      const int32_t b = w >> 5;
      if (nk < ok) atomicMin(&blk[b], nk);
      else if (nk > ok && ok == blk[b]) mark_dirty(b, dstamp);
    }
    __syncthreads();  // B3
    if (!simple)  // the deduplication bits (simple reaches only stamp)
      for (int32_t i = threadIdx.x; i < ptotal; i += blockDim.x) {
        const int32_t w = out[i];
        if (w != p) atomicAnd(&inr[w >> 5], ~(1u << (w & 31)));
      }
    for (int32_t ei = threadIdx.x; ei < np_el; ei += blockDim.x) {
      const int32_t e = L[pe - 1 - ei];
      st[e] = 0;  // absorbed
    }
    const int32_t ndirty = s_ndirty;
    for (int32_t q = wid; q < ndirty; q += nwarp) {
      const int32_t b = s_dlist[q];
      const int32_t v = b * 32 + lane;
      const uint32_t m = __reduce_min_sync(0xffffffffu, v < nv ? kd[v] : kKeyInf);
      if (lane == 0) {
        blk[b] = m;
      }
    }
    if (wid == nwarp - 1) {  // the pivot's block (a second refresh of it via the list is identical)
      const int32_t v = (p & ~31) + lane;
      const uint32_t m = __reduce_min_sync(0xffffffffu, v < nv ? kd[v] : kKeyInf);
      if (lane == 0) blk[p >> 5] = m;
    }
    if (threadIdx.x == 0) {
      if (simple && np_el && s_ip != ptotal - 1) out[s_ip] = out[ptotal - 1];  // the boundary without p
      st[p] = static_cast<S>(nbd);
      s_cursor = cur0 + nbd;
      s_nbd[(k + 1) & 1] = 0;  // its last reader was the previous pivot, before this B2
    }
    __syncthreads();  // B4
    if (threadIdx.x == 0) s_ndirty = 0;
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
  std::vector<int64_t> hneed(mode == 0 ? nn : 0);  // per node: 2 (4 deg sum + 2 nv + 64)
  if (mode == 0) MP_CUDA(cudaMemcpyAsync(hneed.data(), need.get(), sizeof(int64_t) * nn, cudaMemcpyDeviceToHost, s));
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
  // md_kernel: degrees (kSmemDegCap) + block minima / dirty bits of nodes up to 64K vertices
  const size_t smem = md_global_smem(kMdSmemMaxNv);
  DevBuf<uint64_t> gblk(static_cast<size_t>(n >> 5) + nn + 1, s);
  DevBuf<uint32_t> gdbits(static_cast<size_t>(n >> 10) + 2LL * nn + 2, s);
  a.gblk = gblk, a.gdbits = gdbits;
  a.gsmem_bytes = static_cast<int64_t>(smem);
  allow_max_smem(md_kernel, ctx.device);
  const int kt__ = ctx.ktime_begin(kKMd);
  if (mode == 0) {
    // one CTA per non-empty node, largest first: shared-memory state where it
    // fits, global lists (md_node_global) for the rest, in the same launch
    std::vector<int32_t> hoff(nn + 1);
    std::vector<uint8_t> hmask(node_mask ? nn : 0);
    MP_CUDA(cudaMemcpyAsync(hoff.data(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
    if (node_mask) MP_CUDA(cudaMemcpyAsync(hmask.data(), node_mask, nn, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> sched;
    for (int32_t i = 0; i < nn; ++i)
      if (hoff[i + 1] > hoff[i] && (!node_mask || hmask[i])) sched.push_back(i);
    std::stable_sort(sched.begin(), sched.end(), [&](int32_t x, int32_t y) {
      return hoff[x + 1] - hoff[x] > hoff[y + 1] - hoff[y];
    });
    const int32_t ns = static_cast<int32_t>(sched.size());
    int32_t big = 0;
    while (big < ns && hoff[sched[big] + 1] - hoff[sched[big]] > kMdSmemMaxNv) ++big;
    DevBuf<int32_t> dsched(std::max(ns, 1), s);
    if (ns > 0) MP_CUDA(cudaMemcpyAsync(dsched, sched.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
    if (big > 0) {
      // nodes above kMdSmemMaxNv: 512-thread CTAs with global lists, on the
      // auxiliary stream so they overlap the shared-memory kernel
      MP_CUDA(cudaEventRecord(ctx.fork_ev[0], s));
      MP_CUDA(cudaStreamWaitEvent(ctx.aux_stream, ctx.fork_ev[0], 0));
      MdArgs ab = a;
      ab.sched = dsched;
      // degrees of the largest such node in shared memory, plus block minima
      int64_t maxnv = 0;
      for (int32_t i = 0; i < big; ++i) maxnv = std::max<int64_t>(maxnv, hoff[sched[i] + 1] - hoff[sched[i]]);
      if (maxnv <= kMd16MaxNv) {
        // 16-bit degrees, 256-thread CTAs: two per SM (one wave) when the big
        // nodes outnumber the SMs, else one per SM (the shared memory is padded
        // past half an SM so the scheduler cannot pair two leaves on one SM)
        size_t bsmem = md_global_smem16(maxnv);
        if (big <= ctx.num_sms) bsmem = std::max<size_t>(bsmem, 120 * 1024);
        ab.gsmem_bytes = static_cast<int64_t>(bsmem);
        allow_max_smem(md_kernel16, ctx.device);
        MP_KERNEL(ctx, md_kernel16<<<big, kMd16Threads, bsmem, ctx.aux_stream>>>(ab));
      } else {
        const size_t bsmem = md_global_smem(maxnv);
        ab.gsmem_bytes = static_cast<int64_t>(bsmem);
        MP_KERNEL(ctx, md_kernel<<<big, kMdThreads, bsmem, ctx.aux_stream>>>(ab));
      }
      MP_CUDA(cudaEventRecord(ctx.fork_ev[1], ctx.aux_stream));
    }
    if (ns > big) {
      a.sched = dsched.get() + big;
      allow_max_smem(md_smem_kernel<MdWide>, ctx.device);
      allow_max_smem(md_smem_kernel<MdCompact>, ctx.device);
      cudaFuncAttributes fw{}, fc{};
      MP_CUDA(cudaFuncGetAttributes(&fw, md_smem_kernel<MdWide>));
      MP_CUDA(cudaFuncGetAttributes(&fc, md_smem_kernel<MdCompact>));
      // dynamic shared memory: what the largest shared-memory node needs
      // (state + lists from its degree sum + pool halves of 4 nv entries), so
      // small nodes (C4 frames) keep several CTAs per SM and leave room for
      // the other contexts' kernels.  The compact layout when some node fits
      // only that way (its lists plus the smallest pool halves).
      const int64_t cap = static_cast<int64_t>(ctx.smem_optin) -
                          static_cast<int64_t>(std::max(fw.sharedSizeBytes, fc.sharedSizeBytes));
      int64_t want_w = 0, want_c = 0;
      bool compact = false;
      for (int32_t i = big; i < ns; ++i) {
        const int32_t node = sched[i];
        const int64_t nv = hoff[node + 1] - hoff[node];
        const int64_t dsum = (hneed[node] / 2 - 64 - 2 * nv) / 4;
        const int64_t fw_n = md_smem_fixed<MdWide>(static_cast<int32_t>(nv)) + 2 * dsum;
        const int64_t fc_n = md_smem_fixed<MdCompact>(static_cast<int32_t>(nv)) + 2 * dsum;
        want_w = std::max(want_w, fw_n + 4 * std::max<int64_t>(kMdMinHalf, 4 * nv));
        want_c = std::max(want_c, fc_n + 4 * std::max<int64_t>(kMdMinHalf, 4 * nv));
        if (fw_n + 4 * kMdMinHalf > cap && fc_n + 4 * kMdMinHalf <= cap) compact = true;
      }
      a.smem_bytes = std::min(cap, ((compact ? want_c : want_w) + 1023) & ~int64_t(1023));
      a.gsmem_bytes = a.smem_bytes;
      const int threads = ctx.tune[MP_TUNE_MD_THREADS] > 0
                              ? static_cast<int>(std::min<int64_t>(kMdSmemThreads, ctx.tune[MP_TUNE_MD_THREADS]) & ~31)
                              : kMdSmemThreads;
      if (compact)
        MP_KERNEL(ctx, md_smem_kernel<MdCompact><<<ns - big, std::max(threads, 32), static_cast<size_t>(a.smem_bytes), s>>>(a));
      else
        MP_KERNEL(ctx, md_smem_kernel<MdWide><<<ns - big, std::max(threads, 32), static_cast<size_t>(a.smem_bytes), s>>>(a));
    }
    if (big > 0) MP_CUDA(cudaStreamWaitEvent(s, ctx.fork_ev[1], 0));
  } else {
    std::vector<int32_t> hoff(nn + 1);
    MP_CUDA(cudaMemcpyAsync(hoff.data(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    int64_t maxnv = 0;
    for (int32_t i = 0; i < nn; ++i) maxnv = std::max<int64_t>(maxnv, hoff[i + 1] - hoff[i]);
    a.gsmem_bytes = static_cast<int64_t>(md_global_smem(maxnv));
    MP_KERNEL(ctx, md_kernel<<<nn, kMdThreads, static_cast<size_t>(a.gsmem_bytes), s>>>(a));
  }
  ctx.ktime_end(kt__);
  int32_t h_over = 0;
  MP_CUDA(cudaMemcpyAsync(&h_over, overflow, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (h_over) throw Error(MP_ENOMEM, "minimum_degree: element pool exhausted");
}

}  // namespace mp
