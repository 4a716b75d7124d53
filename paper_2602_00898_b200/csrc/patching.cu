// Stage 1 — mesh patch partitioning (reference core/src/patching.cpp).
//
//   connected components   graph.cpp:183-205   union-find hooking to the min id
//   farthest-point seeds   patching.cpp:26-65  one CTA per component, tile-max tree
//   Lloyd assign/recenter  patching.cpp:69-139 one cooperative persistent kernel,
//                                              level-synchronous BFS, atomicMin ties
//   enforce_connectivity   patching.cpp:347-384 same-patch union-find + fresh ids
//   repair_sizes           patching.cpp:149-291 one CTA, member chains
//
// Every tie-break of the reference is reproduced exactly:
// FPS argmax = (dist desc, id asc); assign = lower label on equal distance;
// recenter = deepest, then lowest id; repair = (size, id) orders.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kLloydRounds = 10;  // patching.cpp:15
constexpr int kTile = 256;        // FPS argmax tile (positions in the component list)
constexpr int kFpsThreads = 1024;
constexpr int kTouchCap = 2048;   // touched-tile list capacity per round (overflow = full rescan)
constexpr int32_t kBatchedFpsMin = 1 << 15;  // single components from this size use fps_batched_dev

enum CompMode : int32_t { kModeSingletons = 0, kModeOne = 1, kModeFps = 2 };

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {  // patching.cpp:17-22
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d649bb133111ebULL;
  return x ^ (x >> 31);
}

// ------------------------------------------------------------ union-find CC
__device__ __forceinline__ int32_t uf_find(int32_t* par, int32_t x) {
  volatile int32_t* vp = par;
  for (;;) {
    int32_t p = vp[x];
    if (p == x) return x;
    int32_t gp = vp[p];
    if (gp == p) return p;
    vp[x] = gp;  // path halving; gp is an ancestor, benign race
    x = gp;
  }
}

// Start every vertex at its smallest neighbour in the same label class (or
// itself): chains strictly decrease, so they end at set roots, and most hooks
// below find their endpoints already joined.
__global__ void uf_init(DGraph g, int32_t* par, const int32_t* label) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
    const int32_t lv = label ? label[v] : 0;
    int32_t m = v;
    for (int32_t j = g.off[v]; j < g.off[v + 1]; ++j) {
      const int32_t w = g.nbr[j];
      if (w < m && (!label || label[w] == lv)) m = w;
    }
    par[v] = m;
  }
}

// Hook the larger root under the smaller one, so every root is the minimum
// vertex of its set.  label != nullptr restricts to edges inside a label class.
__global__ void uf_hook(DGraph g, int32_t* par, const int32_t* label) {
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < g.n; u += gridDim.x * blockDim.x) {
    const int32_t lu = label ? label[u] : 0;
    for (int32_t j = g.off[u]; j < g.off[u + 1]; ++j) {
      int32_t v = g.nbr[j];
      if (v <= u) continue;
      if (label && label[v] != lu) continue;
      int32_t ru = uf_find(par, u), rv = uf_find(par, v);
      while (ru != rv) {
        if (ru < rv) {
          int32_t t = ru;
          ru = rv;
          rv = t;
        }
        int32_t old = atomicCAS(&par[ru], ru, rv);
        if (old == ru) break;
        ru = uf_find(par, old);
        rv = uf_find(par, rv);
      }
    }
  }
}

// Read-only root lookup into a second array: a path-halving find racing with
// the final writes could leave a non-root pointer behind.
__global__ void uf_roots(int32_t n, const int32_t* par, int32_t* root) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int32_t x = v, p = par[x];
    while (p != x) x = p, p = par[x];
    root[v] = x;
  }
}

// par receives, for every vertex, the smallest vertex of its set.
void union_find(mp_context& ctx, const DGraph& g, const int32_t* label, int32_t* par) {
  const int blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(g.n, 256), ctx.num_sms * 8));
  DevBuf<int32_t> work(std::max(g.n, 1), ctx.stream);
  MP_KERNEL(ctx, uf_init<<<blocks, 256, 0, ctx.stream>>>(g, work, label));
  MP_KERNEL(ctx, uf_hook<<<blocks, 256, 0, ctx.stream>>>(g, work, label));
  MP_KERNEL(ctx, uf_roots<<<blocks, 256, 0, ctx.stream>>>(g.n, work, par));
}

// ------------------------------------------------------------ components
__global__ void root_flags(int32_t n, const int32_t* par, int32_t* flag) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    flag[v] = par[v] == v ? 1 : 0;
}
__global__ void comp_of_kernel(int32_t n, const int32_t* par, const int32_t* rank, int32_t* comp_of,
                               int32_t* comp_size) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int32_t c = rank[par[v]];
    comp_of[v] = c;
    atomicAdd(&comp_size[c], 1);
  }
}
__global__ void iota_kernel(int32_t n, int32_t* a) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    a[v] = v;
}
__global__ void scatter_pos(int32_t n, const int32_t* list, int32_t* pos_of) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    pos_of[list[i]] = i;
}

// Per-component plan (patching.cpp:307-322): k = max(1, llround(|comp|/target)),
// mode, patch base, FPS tile bases.  One CTA, chunked block scans.
__global__ void plan_components(int32_t C, const int32_t* comp_size, int32_t target,
                                int32_t* comp_start, int32_t* comp_k, int32_t* comp_mode,
                                int32_t* comp_base, int32_t* tile_base, int32_t* super_base,
                                int32_t* totals /* [0]=patches [1]=tiles [2]=supers [3]=largest FPS component */) {
  __shared__ int32_t sh[32];
  __shared__ int32_t s_max;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  int32_t run_start = 0, run_base = 0, run_tile = 0, run_super = 0;
  for (int32_t c0 = 0; c0 < C; c0 += blockDim.x) {
    int32_t c = c0 + threadIdx.x;
    int32_t sz = 0, k = 0, np = 0, nt = 0, ns = 0, mode = 0;
    if (c < C) {
      sz = comp_size[c];
      long long kk = llround(static_cast<double>(sz) / static_cast<double>(target));
      k = kk < 1 ? 1 : static_cast<int32_t>(kk);
      if (k >= sz) mode = kModeSingletons, np = sz;
      else if (k == 1) mode = kModeOne, np = 1;
      else {
        mode = kModeFps, np = k;
        nt = static_cast<int32_t>(ceil_div(sz, kTile));
        ns = static_cast<int32_t>(ceil_div(nt, kTile));
      }
    }
    if (mode == kModeFps) atomicMax(&s_max, sz);
    int32_t tot;
    int32_t es = block_excl_scan(sz, sh, &tot);
    int32_t add_s = tot;
    int32_t eb = block_excl_scan(np, sh, &tot);
    int32_t add_b = tot;
    int32_t et = block_excl_scan(nt, sh, &tot);
    int32_t add_t = tot;
    int32_t eu = block_excl_scan(ns, sh, &tot);
    int32_t add_u = tot;
    if (c < C) {
      comp_start[c] = run_start + es;
      comp_k[c] = k;
      comp_mode[c] = mode;
      comp_base[c] = run_base + eb;
      tile_base[c] = run_tile + et;
      super_base[c] = run_super + eu;
    }
    run_start += add_s, run_base += add_b, run_tile += add_t, run_super += add_u;
  }
  __syncthreads();
  if (threadIdx.x == 0) totals[0] = run_base, totals[1] = run_tile, totals[2] = run_super, totals[3] = s_max;
}

// Assignments of singleton / one-patch components (patching.cpp:313-322).
__global__ void assign_trivial(int32_t n, const int32_t* comp_list, const int32_t* comp_of,
                               const int32_t* comp_start, const int32_t* comp_mode,
                               const int32_t* comp_base, int32_t* assignment) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int32_t v = comp_list ? comp_list[i] : i;
    int32_t c = comp_of ? comp_of[v] : 0;
    int32_t mode = comp_mode[c];
    if (mode == kModeSingletons) assignment[v] = comp_base[c] + (i - comp_start[c]);
    else if (mode == kModeOne) assignment[v] = comp_base[c];
  }
}

// ------------------------------------------------------------ farthest-point seeds
// One CTA per FPS component (patching.cpp:26-65).  dist lives in HBM/L2; the
// argmax over the component is a two-level tile-max tree of packed
// (dist desc, id asc) keys, refreshed only over tiles a relaxation touched.
// A relaxation is a single-source BFS with strict decrease; it runs edge
// parallel (one thread per (frontier vertex, neighbour slot) of an 8-wide ELL
// copy of the adjacency), with the frontier and the touched-tile bitmap in
// shared memory and one barrier per level (rotating frontier counters).
constexpr int kEll = 8;
constexpr int kFrontCap = 4096;          // smem frontier entries per buffer (overflow -> global)
constexpr int kSmemTileWords = 2048;     // smem touched bitmap: components up to 16.7M vertices

struct FpsArgs {
  DGraph g;
  const int32_t* ell;        // n * kEll: neighbours, -1 padded; slot 7 < -1 encodes a CSR tail
  const int32_t* comp_list;  // nullptr: identity (single component)
  const int32_t* pos_of;     // nullptr: identity
  const int32_t* comp_start;
  const int32_t* comp_size;
  const int32_t* comp_k;
  const int32_t* comp_mode;
  const int32_t* comp_base;
  const int32_t* tile_base;
  const int32_t* super_base;
  int32_t* dist;
  uint64_t* tile_key;
  uint64_t* super_key;
  uint32_t* tile_bits;   // global touched bitmap for components too large for smem
  int32_t* frontier;     // 2 * n scratch; component c uses [2*start, 2*start + 2*size)
  int32_t* seeds;        // by global patch id
  uint64_t seed;
  unsigned long long* work;  // [0] += adjacency scans of the relaxations (R_fps)
  int32_t smem_n;            // components up to this size keep dist + ELL in shared memory
};

__device__ __forceinline__ int32_t vtx_at(const FpsArgs& a, int32_t pos) {
  return a.comp_list ? a.comp_list[pos] : pos;
}
__device__ __forceinline__ int32_t pos_in(const FpsArgs& a, int32_t v) {
  return a.pos_of ? a.pos_of[v] : v;
}

__global__ void build_ell(DGraph g, int32_t* ell) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
    const int32_t o = g.off[v], deg = g.off[v + 1] - o;
    int32_t* e = ell + static_cast<int64_t>(v) * kEll;
#pragma unroll
    for (int k = 0; k < kEll; ++k) e[k] = k < deg ? g.nbr[o + k] : -1;
    if (deg > kEll) e[kEll - 1] = -(o + kEll - 1) - 2;  // CSR tail from index o+7
  }
}

__global__ void __launch_bounds__(kFpsThreads) fps_kernel(FpsArgs a) {
  const int32_t c = blockIdx.x;
  if (a.comp_mode[c] != kModeFps) return;
  const int32_t start = a.comp_start[c], size = a.comp_size[c], k = a.comp_k[c];
  const int32_t ntile = static_cast<int32_t>(ceil_div(size, kTile));
  const int32_t nsuper = static_cast<int32_t>(ceil_div(ntile, kTile));
  uint64_t* tkey = a.tile_key + a.tile_base[c];
  uint64_t* skey = a.super_key + a.super_base[c];
  int32_t* gfront0 = a.frontier + 2LL * start;  // overflow parts of the two frontier buffers
  int32_t* gfront1 = gfront0 + size;

  extern __shared__ int32_t fsm[];
  int32_t* sfront0 = fsm;
  int32_t* sfront1 = fsm + kFrontCap;
  uint32_t* sbits = reinterpret_cast<uint32_t*>(fsm + 2 * kFrontCap);
  const int32_t nwords = (ntile + 31) / 32;
  uint32_t* tbits = nwords <= kSmemTileWords ? sbits : a.tile_bits + (a.tile_base[c] + 31) / 32 + c;
  // Small components (a.smem_n): the distances and the adjacency (ELL rows in
  // component-local 16-bit ids) live in shared memory, so a BFS level is
  // shared-memory work between two barriers instead of L2 round trips;
  // frontiers then hold local ids.  A vertex of degree > 8 keeps the
  // component on the global path.
  int32_t* sdist = fsm + 2 * kFrontCap + kSmemTileWords;
  uint16_t* sell = reinterpret_cast<uint16_t*>(sdist + a.smem_n);

  __shared__ int32_t touched[kTouchCap];
  __shared__ int32_t n_touched, overflow, cnt[3], s_cur;
  __shared__ uint32_t super_bits[64];  // up to 2048 supertiles (524M vertices)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;

  bool sm = size <= a.smem_n;
  if (sm) {
    bool tail = false;
    for (int32_t i = threadIdx.x; i < size; i += blockDim.x) {
      const int32_t v = vtx_at(a, start + i);
#pragma unroll
      for (int k = 0; k < kEll; ++k) {
        const int32_t x = a.ell[static_cast<int64_t>(v) * kEll + k];
        tail |= x < -1;
        sell[i * kEll + k] = x >= 0 ? static_cast<uint16_t>(pos_in(a, x) - start) : uint16_t(0xffff);
      }
      sdist[i] = kUnreached;
    }
    sm = !__syncthreads_or(tail);
  }
  for (int32_t i = threadIdx.x; i < size; i += blockDim.x) a.dist[vtx_at(a, start + i)] = kUnreached;
  for (int32_t i = threadIdx.x; i < 64; i += blockDim.x) super_bits[i] = 0;
  for (int32_t i = threadIdx.x; i < nwords; i += blockDim.x) tbits[i] = 0;
  if (threadIdx.x == 0) {
    n_touched = 0, overflow = 0;
    s_cur = vtx_at(a, start + static_cast<int32_t>(splitmix64(a.seed) % static_cast<uint64_t>(size)));
  }
  __syncthreads();

  auto mark_tile_pos = [&](int32_t p) {  // p: position in the component
    const int32_t t = p / kTile;
    const uint32_t bit = 1u << (t & 31);
    if (!(atomicOr(&tbits[t >> 5], bit) & bit)) {
      const int32_t slot = atomicAdd(&n_touched, 1);
      if (slot < kTouchCap) touched[slot] = t;
      else overflow = 1;
    }
  };
  auto mark_tile = [&](int32_t v) {
    const int32_t t = (pos_in(a, v) - start) / kTile;
    const uint32_t bit = 1u << (t & 31);
    if (!(atomicOr(&tbits[t >> 5], bit) & bit)) {
      const int32_t slot = atomicAdd(&n_touched, 1);
      if (slot < kTouchCap) touched[slot] = t;
      else overflow = 1;
    }
  };
  auto tile_max = [&](int32_t t) -> uint64_t {  // warp-cooperative
    uint64_t best = 0;
    const int32_t lo = t * kTile, hi = min(size, lo + kTile);
    for (int32_t p = lo + lane; p < hi; p += 32) {
      const int32_t v = vtx_at(a, start + p);
      const int32_t dv = sm ? sdist[p] : __ldcg(&a.dist[v]);
      const uint64_t kk = key_max(static_cast<uint32_t>(dv), static_cast<uint32_t>(v));
      best = kk > best ? kk : best;
    }
    return warp_max_u64(best);
  };
  auto super_max = [&](int32_t sidx) -> uint64_t {
    uint64_t best = 0;
    const int32_t lo = sidx * kTile, hi = min(ntile, lo + kTile);
    for (int32_t t = lo + lane; t < hi; t += 32) {
      const uint64_t kk = __ldcg(&tkey[t]);
      best = kk > best ? kk : best;
    }
    return warp_max_u64(best);
  };

  unsigned long long scans = 0;
  for (int32_t s = 0; s < k; ++s) {
    const int32_t cur = s_cur;
    if (threadIdx.x == 0) {
      a.seeds[a.comp_base[c] + s] = cur;
      if (sm) {
        const int32_t lc = pos_in(a, cur) - start;
        sdist[lc] = 0;
        sfront0[0] = lc;
        mark_tile_pos(lc);
      } else {
        a.dist[cur] = 0;
        sfront0[0] = cur;
        mark_tile(cur);
      }
      cnt[0] = 1, cnt[1] = 0, cnt[2] = 0;
    }
    __syncthreads();
    if (sm) {  // relax_from (patching.cpp:35-49) on the shared-memory field
      for (int32_t d = 0;; ++d) {
        const int32_t nf = cnt[d % 3];
        if (nf == 0) break;
        if (threadIdx.x == 0) cnt[(d + 2) % 3] = 0;
        const int32_t* sin = (d & 1) ? sfront1 : sfront0;
        int32_t* sout = (d & 1) ? sfront0 : sfront1;
        int32_t* cout = &cnt[(d + 1) % 3];
        const int32_t items = nf * kEll;
        for (int32_t it = threadIdx.x; it < items; it += blockDim.x) {
          const int32_t u = sin[it >> 3];
          const uint16_t x = sell[u * kEll + (it & (kEll - 1))];
          if (x == 0xffff) continue;
          ++scans;
          if (d + 1 < sdist[x] && atomicMin(&sdist[x], d + 1) > d + 1) {
            sout[atomicAdd(cout, 1)] = x;  // a vertex enters a frontier once: nf <= size <= kFrontCap
            mark_tile_pos(x);
          }
        }
        __syncthreads();
      }
    } else {
    // relax_from (patching.cpp:35-49)
    for (int32_t d = 0;; ++d) {
      const int32_t nf = cnt[d % 3];
      if (nf == 0) break;
      if (threadIdx.x == 0) cnt[(d + 2) % 3] = 0;
      const int32_t* sin = (d & 1) ? sfront1 : sfront0;
      const int32_t* gin = (d & 1) ? gfront1 : gfront0;
      int32_t* sout = (d & 1) ? sfront0 : sfront1;
      int32_t* gout = (d & 1) ? gfront0 : gfront1;
      int32_t* cout = &cnt[(d + 1) % 3];
      auto relax = [&](int32_t w) {
        if (d + 1 < __ldcg(&a.dist[w])) {
          if (atomicMin(&a.dist[w], d + 1) > d + 1) {
            const int32_t slot = atomicAdd(cout, 1);
            if (slot < kFrontCap) sout[slot] = w;
            else gout[slot - kFrontCap] = w;
            mark_tile(w);
          }
        }
      };
      const int32_t items = nf * kEll;
      for (int32_t it = threadIdx.x; it < items; it += blockDim.x) {
        const int32_t i = it >> 3, slot = it & (kEll - 1);
        const int32_t u = i < kFrontCap ? sin[i] : __ldcg(&gin[i - kFrontCap]);
        const int32_t x = a.ell[static_cast<int64_t>(u) * kEll + slot];
        if (x >= 0) {
          ++scans;
          relax(x);
        } else if (x < -1) {  // degree > 8: this slot walks the CSR tail
          const int32_t e = a.g.off[u + 1];
          for (int32_t j = -x - 2; j < e; ++j) {
            ++scans;
            relax(a.g.nbr[j]);
          }
        }
      }
      __syncthreads();
    }
    }  // sm / global
    // refresh touched tiles, then touched supertiles, then the top
    if (overflow) {
      for (int32_t t = wid; t < ntile; t += nwarp) {
        const uint64_t m = tile_max(t);
        if (lane == 0) tkey[t] = m;
      }
      for (int32_t i = threadIdx.x; i < nwords; i += blockDim.x) tbits[i] = 0;
      __syncthreads();
      for (int32_t sidx = wid; sidx < nsuper; sidx += nwarp) {
        const uint64_t m = super_max(sidx);
        if (lane == 0) skey[sidx] = m;
      }
    } else {
      const int32_t nt = n_touched;
      for (int32_t i = wid; i < nt; i += nwarp) {
        const int32_t t = touched[i];
        const uint64_t m = tile_max(t);
        if (lane == 0) {
          tkey[t] = m;
          atomicAnd(&tbits[t >> 5], ~(1u << (t & 31)));
          const int32_t su = t / kTile;
          atomicOr(&super_bits[su >> 5], 1u << (su & 31));
        }
      }
      __syncthreads();
      const int32_t swords = (nsuper + 31) / 32;
      int32_t rank = 0;
      for (int32_t wi = 0; wi < swords; ++wi) {
        uint32_t bits = super_bits[wi];
        while (bits) {
          const int32_t b = __ffs(bits) - 1;
          bits &= bits - 1;
          if (rank % nwarp == wid) {
            const uint64_t m = super_max(wi * 32 + b);
            if (lane == 0) skey[wi * 32 + b] = m;
          }
          ++rank;
        }
      }
    }
    __syncthreads();
    // argmax over the component (patching.cpp:52-60): (dist desc, id asc)
    if (wid == 0) {
      uint64_t best = 0;
      for (int32_t i = lane; i < nsuper; i += 32) {
        const uint64_t kk = __ldcg(&skey[i]);
        best = kk > best ? kk : best;
      }
      best = warp_max_u64(best);
      if (lane == 0) {
        s_cur = static_cast<int32_t>(key_max_id(best));
        n_touched = 0;
        overflow = 0;
      }
      for (int32_t i = lane; i < 64; i += 32) super_bits[i] = 0;
    }
    __syncthreads();
  }
  if (sm)
    for (int32_t i = threadIdx.x; i < size; i += blockDim.x) a.dist[vtx_at(a, start + i)] = sdist[i];
  if (a.work && scans) atomicAdd(&a.work[0], scans);
}

// ------------------------------------------------------------ Lloyd rounds
struct LloydArgs {
  DGraph g;
  const int32_t* ell;        // n * 8 ELL adjacency (build_ell)
  const int32_t* comp_of;    // nullptr: single component 0
  const int32_t* comp_mode;
  int32_t* comp_active;      // per component
  int32_t* changed;          // [kLloydRounds][C], zero-initialised
  int32_t C;
  const int32_t* patch_comp; // per global patch id: its component (nullptr: 0)
  int32_t P;                 // global patch ids [0, P)
  int32_t* seeds;
  int32_t* dist;
  int32_t* label;
  int32_t* prev;
  uint64_t* best;            // per patch, recenter argmax
  int32_t* fa;
  int32_t* fb;
  int32_t* counters;         // [3] rotating frontier counters + [3] = any-active
  unsigned long long* work;  // [3] += BFS levels
};

__device__ __forceinline__ bool lloyd_active(const LloydArgs& a, int32_t v) {
  // one component: active for as long as the rounds run (they end when it settles)
  if (!a.comp_of) return true;
  int32_t c = a.comp_of[v];
  return a.comp_mode[c] == kModeFps && __ldcg(&a.comp_active[c]) != 0;
}

// One BFS level over `items` (frontier vertex, ELL slot) pairs in CTA-sized
// chunks: a chunk's pushes gather in shared memory and reserve their range of
// the next frontier with ONE global atomic (a per-warp atomic on the shared
// counter serialises ~15K warps per level at C2).  item(it, push) handles one
// pair and calls push(w) for every newly reached vertex.
constexpr int kLvlPer = 4;                 // items per thread per chunk
constexpr int kLvlBuf = 256 * kLvlPer * 2; // shared push buffer (pairs + CSR tails)
template <class F>
__device__ __forceinline__ void chunked_level(int64_t items, int32_t* gcount, int32_t* next, int32_t* sbuf,
                                              int32_t* sh, F&& item) {
  const int64_t chunk = static_cast<int64_t>(blockDim.x) * kLvlPer;
  for (int64_t c0 = static_cast<int64_t>(blockIdx.x) * chunk; c0 < items; c0 += static_cast<int64_t>(gridDim.x) * chunk) {
    if (threadIdx.x == 0) sh[0] = 0;
    __syncthreads();
    auto push = [&](int32_t w) {
      const int32_t slot = atomicAdd(&sh[0], 1);
      if (slot < kLvlBuf) sbuf[slot] = w;
      else next[atomicAdd(gcount, 1)] = w;  // overflow (high-degree tails): direct
    };
#pragma unroll
    for (int q = 0; q < kLvlPer; ++q) item(c0 + q * static_cast<int64_t>(blockDim.x) + threadIdx.x, push);
    __syncthreads();
    const int32_t cnt = min(sh[0], kLvlBuf);
    if (threadIdx.x == 0 && cnt) sh[1] = atomicAdd(gcount, cnt);
    __syncthreads();
    for (int32_t i = threadIdx.x; i < cnt; i += blockDim.x) next[sh[1] + i] = sbuf[i];
  }
}

// Small levels (few items): grid-stride over items with one warp-aggregated
// global append per warp -- cheaper than chunked_level's three barriers when
// only a handful of CTAs have work.
constexpr int64_t kChunkMinItems = 65536;
template <class F>
__device__ __forceinline__ void warp_level(int64_t items, int32_t* gcount, int32_t* next, F&& item) {
  const int lane = threadIdx.x & 31;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = tid - lane; base < items; base += nthreads) {
    int32_t pw = -1;  // the ELL item's push; CSR-tail extras go straight out
    item(base + lane, [&](int32_t w) {
      if (pw < 0) pw = w;
      else next[atomicAdd(gcount, 1)] = w;
    });
    const bool push = pw >= 0;
    const int32_t slot = warp_append(gcount, push);
    if (push) next[slot] = pw;
  }
}

// The rounds' barriers: the whole cooperative grid, or -- for small meshes,
// whose BFS levels hold a few hundred vertices -- one thread-block cluster
// that IS the grid (barrier.cluster ~ 400 cycles instead of a grid barrier's
// several microseconds over 148 CTAs; C1's 300 barriers dominate Lloyd).
struct GridBarrier {
  cg::grid_group g = cg::this_grid();
  __device__ void sync() { g.sync(); }
};
struct ClusterBarrier {
  __device__ void sync() { cg::this_cluster().sync(); }
};

constexpr int32_t kLloydSmemBest = 512;  // patches whose recenter keys the shared-memory Lloyd keeps on chip

struct BlockBarrier {
  __device__ void sync() { __syncthreads(); }
};

// SM variant's BFS level: one frontier vertex per thread, its eight ELL slots'
// loads and claims in flight together, warp-aggregated appends (shared-memory
// counter).  visit(w, label(u)) claims w; a CSR tail (degree > 8) is walked
// by the owning thread.
template <class V>
__device__ __forceinline__ void vertex_level(int32_t nf, const int32_t* front, const int32_t* ell, const int32_t* label,
                                             const DGraph& g, int32_t* gcount, int32_t* next, V&& visit) {
  const int lane = threadIdx.x & 31;
  for (int32_t i0 = 0; i0 < nf; i0 += blockDim.x) {
    const int32_t i = i0 + threadIdx.x;
    uint32_t got = 0;
    int32_t xs[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) xs[k] = -1;
    int32_t u = -1, lu = 0;
    if (i < nf) {
      u = front[i];
      lu = label[u];
      const int4 r0 = reinterpret_cast<const int4*>(ell)[2 * u], r1 = reinterpret_cast<const int4*>(ell)[2 * u + 1];
      xs[0] = r0.x, xs[1] = r0.y, xs[2] = r0.z, xs[3] = r0.w, xs[4] = r1.x, xs[5] = r1.y, xs[6] = r1.z, xs[7] = r1.w;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (xs[k] >= 0 && visit(xs[k], lu)) got |= 1u << k;
    }
    const int32_t np = __popc(got);
    int32_t inc = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    int32_t base = 0;
    if (lane == 31 && tot) base = atomicAdd(gcount, tot);
    base = __shfl_sync(0xffffffffu, base, 31);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if ((got >> k) & 1u) next[base + inc - np + __popc(got & ((1u << k) - 1))] = xs[k];
    if (u >= 0 && xs[7] < -1)  // CSR tail of a vertex with more than 8 neighbours
      for (int32_t j = -xs[7] - 2; j < g.off[u + 1]; ++j) {
        const int32_t w = g.nbr[j];
        if (visit(w, lu)) next[atomicAdd(gcount, 1)] = w;
      }
  }
}

// SM: one CTA with the per-vertex state (distances, labels, previous labels,
// both frontiers, the ELL rows) in shared memory -- small meshes (C1), whose
// BFS levels are then shared-memory work between two CTA barriers.
template <class Barrier, bool SM = false>
__global__ void __launch_bounds__(512) lloyd_kernel(LloydArgs a_in) {
  Barrier grid;
  __shared__ int32_t s_lbuf[kLvlBuf], s_lsh[2], s_cnt[4];
  __shared__ LloydArgs a_sm;  // SM: the arguments with the per-vertex arrays rebound to shared memory
  __shared__ uint64_t s_best[SM ? kLloydSmemBest : 1];
  if constexpr (SM) {
    extern __shared__ int32_t lsm[];
    const int32_t n0 = a_in.g.n;
    int32_t* ell = lsm;
    for (int32_t i = threadIdx.x; i < 8 * n0; i += blockDim.x) ell[i] = a_in.ell[i];
    if (threadIdx.x == 0) {
      a_sm = a_in;
      a_sm.ell = ell;
      a_sm.dist = ell + 8 * n0;
      a_sm.label = a_sm.dist + n0;
      a_sm.prev = a_sm.label + n0;
      a_sm.fa = a_sm.prev + n0;
      a_sm.fb = a_sm.fa + n0;
      a_sm.counters = s_cnt;
      if (a_in.P <= kLloydSmemBest) a_sm.best = s_best;  // the recenter argmax keys in shared memory
    }
    int32_t* prev = ell + 10 * n0;
    for (int32_t i = threadIdx.x; i < n0; i += blockDim.x) prev[i] = a_in.prev[i];
    __syncthreads();
  }
  const LloydArgs& a = SM ? a_sm : a_in;
  // per-vertex state loads: shared memory, or L2 (__ldcg) on the grid
  auto ld = [](const int32_t* p) -> int32_t {
    if constexpr (SM) return *p;
    else return __ldcg(p);
  };
  const int lane = threadIdx.x & 31;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int32_t n = a.g.n;

  for (int round = 0; round < kLloydRounds; ++round) {
    // ---- assign_to_seeds (patching.cpp:69-99)
    if (tid == 0) a.counters[0] = 0, a.counters[1] = 0, a.counters[2] = 0;
    for (int64_t v = tid; v < n; v += nthreads)
      if (lloyd_active(a, v)) a.dist[v] = kUnreached, a.label[v] = 0x7fffffff;
    grid.sync();
    for (int64_t p = tid; p < a.P; p += nthreads) {
      int32_t c = a.patch_comp ? a.patch_comp[p] : 0;
      if (c < 0 || a.comp_mode[c] != kModeFps || !__ldcg(&a.comp_active[c])) continue;
      int32_t s = a.seeds[p];
      a.dist[s] = 0;
      a.label[s] = static_cast<int32_t>(p);
      a.fa[atomicAdd(&a.counters[0], 1)] = s;
    }
    grid.sync();
    {
      int32_t* front = a.fa;
      int32_t* next = a.fb;
      for (int32_t d = 0;; ++d) {
        const int32_t cin = d % 3, cout = (d + 1) % 3, cclr = (d + 2) % 3;
        const int32_t nf = ld(&a.counters[cin]);
        if (nf == 0) break;
        if (tid == 0) a.counters[cclr] = 0;
        // edge parallel over (frontier vertex, ELL slot), CTA-aggregated appends
        const int64_t items = static_cast<int64_t>(nf) * 8;
        auto visit = [&](int32_t w, int32_t lu) -> bool {
          int32_t dw = ld(&a.dist[w]);
          bool fresh = false;
          if (dw == kUnreached) {
            dw = atomicCAS(&a.dist[w], kUnreached, d + 1);
            if (dw == kUnreached) fresh = true, dw = d + 1;
          }
          if (dw == d + 1) atomicMin(&a.label[w], lu);
          return fresh;
        };
        auto body = [&](int64_t it, auto&& push) {
          if (it >= items) return;
          const int32_t u = front[it >> 3];
          const int32_t x = a.ell[static_cast<int64_t>(u) * 8 + (it & 7)];
          if (x >= 0) {
            if (visit(x, ld(&a.label[u]))) push(x);
          } else if (x < -1) {  // degree > 8: CSR tail
            const int32_t lu = ld(&a.label[u]);
            for (int32_t j = -x - 2; j < a.g.off[u + 1]; ++j) {
              const int32_t w = a.g.nbr[j];
              if (visit(w, lu)) push(w);
            }
          }
        };
        if constexpr (SM) vertex_level(nf, front, a.ell, a.label, a.g, &a.counters[cout], next, visit);
        else if (items >= kChunkMinItems) chunked_level(items, &a.counters[cout], next, s_lbuf, s_lsh, body);
        else warp_level(items, &a.counters[cout], next, body);
        grid.sync();
        if (tid == 0 && a.work) atomicAdd(&a.work[3], 1ull);
        int32_t* t = front;
        front = next;
        next = t;
      }
    }
    // ---- stability test (patching.cpp:327-334) per component
    int32_t* chg = a.changed + static_cast<int64_t>(round) * a.C;
    for (int64_t v = tid; v < n; v += nthreads)
      if (lloyd_active(a, v) && ld(&a.label[v]) != a.prev[v]) chg[a.comp_of ? a.comp_of[v] : 0] = 1;
    grid.sync();
    if (tid == 0) a.counters[3] = 0;
    for (int64_t v = tid; v < n; v += nthreads) {
      if (!lloyd_active(a, v)) continue;
      int32_t c = a.comp_of ? a.comp_of[v] : 0;
      if (__ldcg(&chg[c])) a.prev[v] = ld(&a.label[v]);
    }
    grid.sync();
    for (int64_t c = tid; c < a.C; c += nthreads) {
      if (a.comp_mode[c] != kModeFps || !a.comp_active[c]) continue;
      if (!__ldcg(&chg[c])) a.comp_active[c] = 0;
      else atomicAdd(&a.counters[3], 1);
    }
    grid.sync();
    if (ld(&a.counters[3]) == 0 || round == kLloydRounds - 1) break;

    // ---- recenter_seeds (patching.cpp:103-139); dist is reused as depth
    if (tid == 0) a.counters[0] = 0, a.counters[1] = 0, a.counters[2] = 0;
    for (int64_t p = tid; p < a.P; p += nthreads) a.best[p] = 0;
    grid.sync();
    for (int64_t v = tid; v < n; v += nthreads) {
      if (!lloyd_active(a, v)) continue;
      const int32_t lv = ld(&a.label[v]);
      bool boundary = false;
      if constexpr (SM) {  // the neighbours from the shared-memory ELL rows (a CSR tail from global)
        const int4 r0 = reinterpret_cast<const int4*>(a.ell)[2 * v], r1 = reinterpret_cast<const int4*>(a.ell)[2 * v + 1];
        const int32_t xs[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) boundary |= xs[k] >= 0 && a.label[xs[k]] != lv;
        if (xs[7] < -1)
          for (int32_t j = -xs[7] - 2; j < a.g.off[v + 1] && !boundary; ++j) boundary = a.label[a.g.nbr[j]] != lv;
      } else {
        for (int32_t j = a.g.off[v]; j < a.g.off[v + 1] && !boundary; ++j)
          boundary = ld(&a.label[a.g.nbr[j]]) != lv;
      }
      a.dist[v] = boundary ? 0 : kUnreached;
      if (boundary) a.fa[atomicAdd(&a.counters[0], 1)] = static_cast<int32_t>(v);
    }
    grid.sync();
    {
      int32_t* front = a.fa;
      int32_t* next = a.fb;
      for (int32_t d = 0;; ++d) {
        const int32_t cin = d % 3, cout = (d + 1) % 3, cclr = (d + 2) % 3;
        const int32_t nf = ld(&a.counters[cin]);
        if (nf == 0) break;
        if (tid == 0) a.counters[cclr] = 0;
        const int64_t items = static_cast<int64_t>(nf) * 8;
        auto visit = [&](int32_t w, int32_t lu) -> bool {
          if (ld(&a.label[w]) != lu || ld(&a.dist[w]) != kUnreached) return false;
          return atomicCAS(&a.dist[w], kUnreached, d + 1) == kUnreached;
        };
        auto body = [&](int64_t it, auto&& push) {
          if (it >= items) return;
          const int32_t u = front[it >> 3];
          const int32_t x = a.ell[static_cast<int64_t>(u) * 8 + (it & 7)];
          if (x >= 0) {
            if (visit(x, ld(&a.label[u]))) push(x);
          } else if (x < -1) {
            const int32_t lu = ld(&a.label[u]);
            for (int32_t j = -x - 2; j < a.g.off[u + 1]; ++j) {
              const int32_t w = a.g.nbr[j];
              if (visit(w, lu)) push(w);
            }
          }
        };
        if constexpr (SM) vertex_level(nf, front, a.ell, a.label, a.g, &a.counters[cout], next, visit);
        else if (items >= kChunkMinItems) chunked_level(items, &a.counters[cout], next, s_lbuf, s_lsh, body);
        else warp_level(items, &a.counters[cout], next, body);
        grid.sync();
        int32_t* t = front;
        front = next;
        next = t;
      }
    }
    for (int64_t v = tid; v < n; v += nthreads) {
      if (!lloyd_active(a, v)) continue;
      const int32_t dv = ld(&a.dist[v]);
      if (dv == kUnreached) continue;
      atomicMax(reinterpret_cast<unsigned long long*>(&a.best[ld(&a.label[v])]),
                static_cast<unsigned long long>(key_max(static_cast<uint32_t>(dv) + 1u, static_cast<uint32_t>(v))));
    }
    grid.sync();
    for (int64_t p = tid; p < a.P; p += nthreads) {
      int32_t c = a.patch_comp ? a.patch_comp[p] : 0;
      if (c < 0 || a.comp_mode[c] != kModeFps || !__ldcg(&a.comp_active[c])) continue;
      uint64_t b = (SM && a.P <= kLloydSmemBest) ? a.best[p] : __ldcg(&a.best[p]);
      if (b != 0) a.seeds[p] = static_cast<int32_t>(key_max_id(b));
    }
    grid.sync();
  }
  if constexpr (SM) {
    __syncthreads();
    for (int32_t i = threadIdx.x; i < a.g.n; i += blockDim.x) a_in.prev[i] = a.prev[i];
  }
}

// Meshes up to this many vertices run the Lloyd rounds on one cluster.
constexpr int64_t kLloydClusterN = 12288;
constexpr int64_t kLloydSmemN = 4096;  // ... and up to this many on one CTA with the state in shared memory
constexpr int kLloydClusterThreads = 512;

// Cluster size for the one-cluster Lloyd: 16 CTAs where the device allows a
// non-portable cluster, else 8; probed once per device.
int lloyd_cluster_ctas(int device) {
  static std::mutex mu;
  static std::map<int, int> cached;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cached.find(device);
  if (it != cached.end()) return it->second;
  const bool nonportable = cudaFuncSetAttribute(lloyd_kernel<ClusterBarrier>,
                                                cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
  cudaGetLastError();
  int found = 0;
  for (int cs : {16, 8}) {
    if (cs > 8 && !nonportable) continue;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs), cfg.blockDim = dim3(kLloydClusterThreads), cfg.attrs = at, cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, lloyd_kernel<ClusterBarrier>, &cfg) == cudaSuccess && ncl > 0) {
      found = cs;
      break;
    }
    cudaGetLastError();
  }
  cached[device] = found;
  return found;
}

__global__ void lloyd_finish(int32_t n, const int32_t* comp_of, const int32_t* comp_mode,
                             const int32_t* prev, int32_t* assignment) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int32_t c = comp_of ? comp_of[v] : 0;
    if (comp_mode[c] == kModeFps) assignment[v] = prev[v];
  }
}

__global__ void patch_comp_kernel(int32_t C, const int32_t* comp_mode, const int32_t* comp_base,
                                  const int32_t* comp_k, int32_t* patch_comp) {
  for (int32_t c = blockIdx.x; c < C; c += gridDim.x) {
    if (comp_mode[c] != kModeFps) continue;
    for (int32_t p = threadIdx.x; p < comp_k[c]; p += blockDim.x) patch_comp[comp_base[c] + p] = c;
  }
}

__global__ void fill_i32(int64_t n, int32_t* a, int32_t v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    a[i] = v;
}

// ------------------------------------------------------------ enforce_connectivity
__global__ void patch_min_vertex(int32_t n, const int32_t* assignment, int32_t* minv) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    atomicMin(&minv[assignment[v]], v);
}
__global__ void collect_extra_roots(int32_t n, const int32_t* par, const int32_t* assignment,
                                    const int32_t* minv, uint64_t* keys, int32_t* count) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (par[v] != v) continue;
    int32_t p = assignment[v];
    if (minv[p] == v) continue;
    keys[atomicAdd(count, 1)] = (static_cast<uint64_t>(p) << 32) | static_cast<uint32_t>(v);
  }
}
__global__ void fresh_ids(int32_t E, const uint64_t* keys, int32_t P, int32_t* root_id) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x)
    root_id[static_cast<int32_t>(keys[i] & 0xffffffffu)] = P + i;
}
__global__ void relabel_components(int32_t n, const int32_t* par, const int32_t* assignment,
                                   const int32_t* root_id, int32_t* out) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int32_t r = root_id[par[v]];
    out[v] = r >= 0 ? r : assignment[v];
  }
}
__global__ void check_range(int32_t n, const int32_t* assignment, int32_t P, int32_t* bad) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int32_t p = assignment[v];
    if (p < 0 || p >= P) atomicMin(bad, v);
  }
}

// ------------------------------------------------------------ repair_sizes
// One CTA (patching.cpp:149-291).  Members of a patch are a chain of
// segments in `pool`; merges splice chains, splits write two new segments.
struct RepairArgs {
  DGraph g;
  int32_t* assignment;
  int32_t P0;
  int32_t cap_p;       // capacity for patch ids (P0 + splits)
  int32_t cap_seg;
  int64_t cap_pool;
  int32_t target;
  int32_t* size;       // cap_p
  int32_t* exempt;     // cap_p
  int32_t* head;       // cap_p (segment id, -1 = none)
  int32_t* tail;       // cap_p
  int32_t* seg_start;  // cap_seg
  int32_t* seg_len;
  int32_t* seg_next;
  int32_t* pool;       // cap_pool
  int32_t* pool2;      // cap_pool: compaction target (the two pools swap)
  int32_t* dist;       // n, kUnreached outside the current patch work
  int32_t* lab;        // n
  int32_t* fa;         // n
  int32_t* fb;         // n
  int32_t* remap;      // cap_p
  int32_t* out;        // [0] patch count, [1] error
  int32_t smem_words;  // dynamic shared memory of the split's local graph (32-bit words)
};

__global__ void __launch_bounds__(1024) repair_kernel(RepairArgs a) {
  extern __shared__ uint32_t rsm[];
  __shared__ uint64_t red[32];
  __shared__ int32_t shi[32];
  __shared__ int32_t s_P, s_nseg, s_cnt, s_err;
  __shared__ int64_t s_pool;
  const int32_t low = (a.target + 1) / 2;
  const int64_t high = 2LL * a.target;
  if (threadIdx.x == 0) {
    s_P = a.P0;
    s_nseg = a.P0;
    s_pool = a.g.n;
    s_err = 0;
  }
  __syncthreads();
  const int64_t max_iter = 4LL * a.P0 + 64;

  int32_t* pool = a.pool;  // member storage; splits append to it, compaction swaps it
  int32_t* spare = a.pool2;
  // iterate the member chain of patch p: f(v) for every member, block-parallel
  auto for_members = [&](int32_t p, auto&& f) {
    for (int32_t sgi = a.head[p]; sgi >= 0; sgi = a.seg_next[sgi]) {
      const int32_t st = a.seg_start[sgi], len = a.seg_len[sgi];
      for (int32_t i = threadIdx.x; i < len; i += blockDim.x) f(pool[st + i]);
    }
  };
  // Splits append 2 x |patch| ints to the pool and 2 segments; when either
  // runs out, every live patch's chain is copied into one contiguous segment
  // of the spare pool (a warp per patch, bases from a block scan of the
  // sizes) and the pools swap.  Member order inside a patch never affects a
  // result (every choice is a min / max by id), so this is invisible.
  auto compact = [&](int32_t P) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __shared__ int32_t s_base[1024];
    int64_t run = 0;
    for (int32_t p0 = 0; p0 < P; p0 += blockDim.x) {
      const int32_t p = p0 + threadIdx.x;
      const int32_t sz = p < P ? max(a.size[p], 0) : 0;
      int32_t tot;
      const int32_t e = block_excl_scan(sz, shi, &tot);
      s_base[threadIdx.x] = static_cast<int32_t>(run) + e;
      __syncthreads();
      for (int32_t k = wid; k < static_cast<int32_t>(blockDim.x) && p0 + k < P; k += nw) {
        const int32_t q = p0 + k;
        if (a.size[q] <= 0) continue;
        int32_t at = s_base[k];
        for (int32_t sgi = a.head[q]; sgi >= 0; sgi = a.seg_next[sgi]) {
          const int32_t st = a.seg_start[sgi], len = a.seg_len[sgi];
          for (int32_t i = lane; i < len; i += 32) spare[at + i] = pool[st + i];
          at += len;
        }
      }
      __syncthreads();
      for (int32_t q = p0 + threadIdx.x; q < P && q < p0 + static_cast<int32_t>(blockDim.x); q += blockDim.x) {
        if (a.size[q] > 0) {
          a.seg_start[q] = s_base[q - p0];
          a.seg_len[q] = a.size[q];
          a.seg_next[q] = -1;
          a.head[q] = a.tail[q] = q;
        } else {
          a.head[q] = a.tail[q] = -1;
        }
      }
      run += tot;
      __syncthreads();
    }
    int32_t* t = pool;
    pool = spare;
    spare = t;
    if (threadIdx.x == 0) {
      s_nseg = P;
      s_pool = run;
    }
    __syncthreads();
  };

  for (int64_t iter = 0; iter < max_iter; ++iter) {
    const int32_t P = s_P;
    // smallest mergeable patch (size, id)
    uint64_t best = ~0ull;
    for (int32_t p = threadIdx.x; p < P; p += blockDim.x) {
      int32_t sz = a.size[p];
      if (sz <= 0 || sz >= low || a.exempt[p]) continue;
      uint64_t kk = key_min(static_cast<uint32_t>(sz), static_cast<uint32_t>(p));
      best = kk < best ? kk : best;
    }
    best = block_min_u64(best, red);
    if (best != ~0ull) {
      const int32_t mp = static_cast<int32_t>(best & 0xffffffffu);
      uint64_t tb = ~0ull;
      for_members(mp, [&](int32_t v) {
        for (int32_t j = a.g.off[v]; j < a.g.off[v + 1]; ++j) {
          int32_t q = a.assignment[a.g.nbr[j]];
          if (q == mp) continue;
          uint64_t kk = key_min(static_cast<uint32_t>(a.size[q]), static_cast<uint32_t>(q));
          tb = kk < tb ? kk : tb;
        }
      });
      tb = block_min_u64(tb, red);
      if (tb == ~0ull) {
        if (threadIdx.x == 0) a.exempt[mp] = 1;
        __syncthreads();
        continue;
      }
      const int32_t tgt = static_cast<int32_t>(tb & 0xffffffffu);
      for_members(mp, [&](int32_t v) { a.assignment[v] = tgt; });
      __syncthreads();
      if (threadIdx.x == 0) {
        a.seg_next[a.tail[tgt]] = a.head[mp];
        a.tail[tgt] = a.tail[mp];
        a.head[mp] = a.tail[mp] = -1;
        a.size[tgt] += a.size[mp];
        a.size[mp] = 0;
      }
      __syncthreads();
      continue;
    }
    // largest oversized patch (size desc, id asc)
    uint64_t big = 0;
    for (int32_t p = threadIdx.x; p < P; p += blockDim.x) {
      int32_t sz = a.size[p];
      if (sz <= high) continue;
      uint64_t kk = key_max(static_cast<uint32_t>(sz), static_cast<uint32_t>(p));
      big = kk > big ? kk : big;
    }
    big = block_max_u64(big, red);
    if (big == 0) break;
    const int32_t sp = static_cast<int32_t>(key_max_id(big));
    const int32_t spsize = a.size[sp];
    if (s_nseg + 2 > a.cap_seg || s_pool + 2LL * spsize > a.cap_pool) compact(P);
    if (P >= a.cap_p || s_nseg + 2 > a.cap_seg || s_pool + 2LL * spsize > a.cap_pool) {
      if (threadIdx.x == 0) s_err = 1;
      __syncthreads();
      break;
    }
    // gather members contiguously into the pool (new segment region)
    const int64_t gbase = s_pool;
    __syncthreads();
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for_members(sp, [&](int32_t v) { pool[gbase + atomicAdd(&s_cnt, 1)] = v; });
    __syncthreads();
    const int32_t* mem = pool + gbase;
    // The split's three BFS runs (two farthest-vertex sweeps, the two-source
    // competition) on the patch's induced subgraph staged in shared memory
    // (local ids; dist and label packed in one word so the competition is one
    // atomicMin): each level is shared-memory work between two barriers
    // instead of a chain of L2 round trips.  Patches whose subgraph does not
    // fit take the global-memory BFS below.
    bool local = false;
    if (a.smem_words > 0) {
      for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x) a.dist[mem[i]] = i;  // global -> local id
      __syncthreads();
      int64_t dsum = 0;
      for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x) {
        const int32_t u = mem[i];
        for (int32_t j = a.g.off[u]; j < a.g.off[u + 1]; ++j) dsum += a.assignment[a.g.nbr[j]] == sp;
      }
      dsum = block_sum_i64(dsum, reinterpret_cast<int64_t*>(red));
      // sd, lm, off (spsize + 1), two u16 frontiers, u16 adjacency
      local = spsize < 65536 && 3LL * spsize + 1 + spsize + (dsum + 1) / 2 <= a.smem_words;
    }
    if (local) {
      uint32_t* sd = rsm;                      // spsize: dist << 1 | label, ~0 unreached
      int32_t* lm = reinterpret_cast<int32_t*>(sd + spsize);  // local -> global id
      int32_t* lo = lm + spsize;               // spsize + 1 adjacency offsets
      uint16_t* fr0 = reinterpret_cast<uint16_t*>(lo + spsize + 1);
      uint16_t* fr1 = fr0 + spsize;
      uint16_t* la = fr1 + spsize;             // local adjacency
      int32_t run = 0;
      for (int32_t i0 = 0; i0 < spsize; i0 += blockDim.x) {
        const int32_t i = i0 + threadIdx.x;
        int32_t c = 0;
        if (i < spsize) {
          const int32_t u = mem[i];
          lm[i] = u;
          for (int32_t j = a.g.off[u]; j < a.g.off[u + 1]; ++j) c += a.assignment[a.g.nbr[j]] == sp;
        }
        int32_t tot;
        const int32_t e = block_excl_scan(c, shi, &tot);
        if (i < spsize) lo[i] = run + e;
        run += tot;
      }
      if (threadIdx.x == 0) lo[spsize] = run;
      __syncthreads();
      for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x) {
        const int32_t u = lm[i];
        int32_t o = lo[i];
        for (int32_t j = a.g.off[u]; j < a.g.off[u + 1]; ++j) {
          const int32_t w = a.g.nbr[j];
          if (a.assignment[w] == sp) la[o++] = static_cast<uint16_t>(__ldcg(&a.dist[w]));
        }
      }
      __syncthreads();
      // level-synchronous BFS from the given local sources; packed values
      // (d << 1 | label) with atomicMin keep the smallest label among a
      // vertex's same-level predecessors (patching.cpp:246-252); returns the
      // farthest vertex (dist desc, global id asc) (patching.cpp:165-185)
      auto bfs = [&](int32_t ns, const int32_t* src, const uint32_t* lab) -> int32_t {
        for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x) sd[i] = ~0u;
        __syncthreads();
        uint64_t far = 0;
        if (threadIdx.x == 0) {
          for (int32_t q = 0; q < ns; ++q) sd[src[q]] = lab[q], fr0[q] = static_cast<uint16_t>(src[q]);
          s_cnt = 0;
        }
        if (threadIdx.x == 0) far = key_max(0u, static_cast<uint32_t>(lm[src[0]]));
        __syncthreads();
        int32_t nf = ns;
        uint16_t *front = fr0, *next = fr1;
        for (uint32_t d = 1; nf > 0; ++d) {
          for (int32_t i = threadIdx.x; i < nf; i += blockDim.x) {
            const int32_t u = front[i];
            const uint32_t lu = sd[u] & 1u;
            for (int32_t j = lo[u]; j < lo[u + 1]; ++j) {
              const int32_t w = la[j];
              if (sd[w] <= (d << 1)) continue;  // settled at an earlier level (or this one with label 0)
              if (atomicMin(&sd[w], (d << 1) | lu) == ~0u) {
                next[atomicAdd(&s_cnt, 1)] = static_cast<uint16_t>(w);
                far = max(far, key_max(d, static_cast<uint32_t>(lm[w])));
              }
            }
          }
          __syncthreads();
          nf = s_cnt;
          __syncthreads();
          if (threadIdx.x == 0) s_cnt = 0;
          uint16_t* t = front;
          front = next;
          next = t;
        }
        __syncthreads();
        far = block_max_u64(far, red);
        return static_cast<int32_t>(key_max_id(far));
      };
      uint64_t mn = ~0ull;
      for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x) mn = min(mn, static_cast<uint64_t>(lm[i]));
      mn = block_min_u64(mn, red);
      const uint32_t zero[2] = {0u, 1u};
      int32_t src[2];
      src[0] = __ldcg(&a.dist[static_cast<int32_t>(mn)]);
      const int32_t b_g = bfs(1, src, zero);
      src[0] = __ldcg(&a.dist[b_g]);
      const int32_t c_g = bfs(1, src, zero);
      src[0] = __ldcg(&a.dist[b_g]), src[1] = __ldcg(&a.dist[c_g]);
      bfs(2, src, zero);  // labels 0 (b) and 1 (c)
      for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x)
        a.lab[lm[i]] = (sd[i] != ~0u && (sd[i] & 1u)) ? 1 : 0;
      __syncthreads();
    } else {
      // farthest-vertex sweeps (patching.cpp:165-185, 231-233)
      uint64_t mn = ~0ull;
      for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x)
        mn = min(mn, static_cast<uint64_t>(mem[i]));
      mn = block_min_u64(mn, red);
      int32_t ends[3];
      ends[0] = static_cast<int32_t>(mn);
      for (int sweep = 1; sweep <= 2; ++sweep) {
        for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x) a.dist[mem[i]] = kUnreached;
        __syncthreads();
        const int32_t from = ends[sweep - 1];
        if (threadIdx.x == 0) {
          a.dist[from] = 0;
          a.fa[0] = from;
          s_cnt = 0;
        }
        __syncthreads();
        int32_t nf = 1, d = 0;
        int32_t *front = a.fa, *next = a.fb;
        uint64_t far = key_max(0u, static_cast<uint32_t>(from));
        while (nf > 0) {
          for (int32_t i = threadIdx.x; i < nf; i += blockDim.x) {
            const int32_t u = front[i];
            for (int32_t j = a.g.off[u]; j < a.g.off[u + 1]; ++j) {
              const int32_t w = a.g.nbr[j];
              if (a.assignment[w] != sp) continue;
              if (atomicCAS(&a.dist[w], kUnreached, d + 1) == kUnreached) {
                next[atomicAdd(&s_cnt, 1)] = w;
                uint64_t kk = key_max(static_cast<uint32_t>(d + 1), static_cast<uint32_t>(w));
                far = kk > far ? kk : far;
              }
            }
          }
          __syncthreads();
          nf = s_cnt;
          __syncthreads();
          if (threadIdx.x == 0) s_cnt = 0;
          int32_t* t = front;
          front = next;
          next = t;
          ++d;
          __syncthreads();
        }
        far = block_max_u64(far, red);
        ends[sweep] = static_cast<int32_t>(key_max_id(far));
      }
      // two-source competition, ties to b's half (patching.cpp:234-261)
      const int32_t b = ends[1], cc = ends[2];
      for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x) {
        a.dist[mem[i]] = kUnreached;
        a.lab[mem[i]] = 0x7fffffff;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        a.dist[b] = 0, a.lab[b] = 0;
        a.dist[cc] = 0, a.lab[cc] = 1;
        a.fa[0] = b, a.fa[1] = cc;
        s_cnt = 0;
      }
      __syncthreads();
      {
        int32_t nf = 2, d = 0;
        int32_t *front = a.fa, *next = a.fb;
        while (nf > 0) {
          for (int32_t i = threadIdx.x; i < nf; i += blockDim.x) {
            const int32_t u = front[i];
            const int32_t lu = a.lab[u];
            for (int32_t j = a.g.off[u]; j < a.g.off[u + 1]; ++j) {
              const int32_t w = a.g.nbr[j];
              if (a.assignment[w] != sp) continue;
              int32_t dw = atomicCAS(&a.dist[w], kUnreached, d + 1);
              if (dw == kUnreached) {
                next[atomicAdd(&s_cnt, 1)] = w;
                dw = d + 1;
              }
              if (dw == d + 1) atomicMin(&a.lab[w], lu);
            }
          }
          __syncthreads();
          nf = s_cnt;
          __syncthreads();
          if (threadIdx.x == 0) s_cnt = 0;
          int32_t* t = front;
          front = next;
          next = t;
          ++d;
          __syncthreads();
        }
      }
    }
    // split members stably: keep (label != 1) then fresh (label == 1)
    const int32_t fresh = P;
    const int64_t kbase = gbase + spsize;  // keep list, then fresh list after it
    int32_t nkeep_total = 0;
    {
      int32_t run_keep = 0, run_fresh = 0;
      // first pass: count keep
      int32_t cnt = 0;
      for (int32_t i = threadIdx.x; i < spsize; i += blockDim.x) cnt += (a.lab[mem[i]] != 1);
      int64_t ck = block_sum_i64(cnt, reinterpret_cast<int64_t*>(red));
      nkeep_total = static_cast<int32_t>(ck);
      for (int32_t i0 = 0; i0 < spsize; i0 += blockDim.x) {
        int32_t i = i0 + threadIdx.x;
        int32_t v = i < spsize ? mem[i] : -1;
        int32_t isf = (i < spsize && a.lab[v] == 1) ? 1 : 0;
        int32_t isk = (i < spsize && !isf) ? 1 : 0;
        int32_t tk, tf;
        int32_t ek = block_excl_scan(isk, shi, &tk);
        int32_t ef = block_excl_scan(isf, shi, &tf);
        if (isk) pool[kbase + run_keep + ek] = v;
        if (isf) {
          pool[kbase + nkeep_total + run_fresh + ef] = v;
          a.assignment[v] = fresh;
        }
        run_keep += tk, run_fresh += tf;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t sk = s_nseg, sf = s_nseg + 1;
      a.seg_start[sk] = static_cast<int32_t>(kbase);
      a.seg_len[sk] = nkeep_total;
      a.seg_next[sk] = -1;
      a.seg_start[sf] = static_cast<int32_t>(kbase + nkeep_total);
      a.seg_len[sf] = spsize - nkeep_total;
      a.seg_next[sf] = -1;
      a.head[sp] = a.tail[sp] = sk;
      a.head[fresh] = a.tail[fresh] = sf;
      a.size[sp] = nkeep_total;
      a.size[fresh] = spsize - nkeep_total;
      a.exempt[fresh] = 0;
      s_nseg += 2;
      s_pool = kbase + spsize;
      s_P = P + 1;
    }
    __syncthreads();
  }
  __syncthreads();
  // compact ids ascending (patching.cpp:282-290)
  const int32_t P = s_P;
  int32_t run = 0;
  for (int32_t p0 = 0; p0 < P; p0 += blockDim.x) {
    int32_t p = p0 + threadIdx.x;
    int32_t live = (p < P && a.size[p] > 0) ? 1 : 0;
    int32_t tot;
    int32_t e = block_excl_scan(live, shi, &tot);
    if (p < P) a.remap[p] = live ? run + e : -1;
    run += tot;
  }
  if (threadIdx.x == 0) a.out[0] = run, a.out[1] = s_err;
}

__global__ void seg_init(int32_t P, const int32_t* start, const int32_t* count, int32_t* head,
                         int32_t* tail, int32_t* seg_start, int32_t* seg_len, int32_t* seg_next,
                         int32_t* size, int32_t* exempt) {
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    head[p] = tail[p] = p;
    seg_start[p] = start[p];
    seg_len[p] = count[p];
    seg_next[p] = -1;
    size[p] = count[p];
    exempt[p] = 0;
  }
}
__global__ void count_patches(int32_t n, const int32_t* assignment, int32_t* cnt) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    atomicAdd(&cnt[assignment[v]], 1);
}
__global__ void apply_remap(int32_t n, const int32_t* remap, int32_t* assignment) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    assignment[v] = remap[assignment[v]];
}

int grid_for(const mp_context& ctx, int64_t n, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), ctx.num_sms * 16LL)));
}

// Stable counting sort of vertices by patch id (ascending id within a patch).
void bucket_by_patch(mp_context& ctx, int32_t n, const int32_t* assignment, int32_t P,
                     int32_t* start, int32_t* count, int32_t* list) {
  cudaStream_t s = ctx.stream;
  MP_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t) * P, s));
  MP_KERNEL(ctx, count_patches<<<grid_for(ctx, n), 256, 0, s>>>(n, assignment, count));
  size_t tmp = 0;
  MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, count, start, P, s));
  DevBuf<char> t(tmp, s);
  MP_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, count, start, P, s));
  DevBuf<int32_t> keys_out(n, s), vals_in(n, s);
  MP_KERNEL(ctx, iota_kernel<<<grid_for(ctx, n), 256, 0, s>>>(n, vals_in));
  int end_bit = 1;
  while ((1LL << end_bit) < P) ++end_bit;
  size_t tmp2 = 0;
  MP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, assignment, keys_out.get(), vals_in.get(),
                                          list, n, 0, end_bit, s));
  DevBuf<char> t2(tmp2, s);
  MP_CUDA(cub::DeviceRadixSort::SortPairs(t2.get(), tmp2, assignment, keys_out.get(), vals_in.get(),
                                          list, n, 0, end_bit, s));
}

constexpr int kRepairSmemBytes = 96 * 1024;  // the split's local graph (patches up to ~3.5K vertices)

int32_t repair_sizes_dev(mp_context& ctx, const DGraph& g, int32_t* assignment, int32_t P,
                         int32_t target) {
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  RepairArgs a{};
  a.g = g;
  a.assignment = assignment;
  a.P0 = P;
  // every split takes one of the 4P+64 iterations (patching.cpp:187): ids
  // are never reused, so P0 + 4P0 + 64 bounds them; segments and pool space
  // are recycled by the in-kernel compaction
  a.cap_p = 5 * P + 65;
  a.cap_seg = 2 * a.cap_p + 16;
  a.cap_pool = 3LL * n + 1024;
  a.target = target;
  DevBuf<int32_t> size(a.cap_p, s), exempt(a.cap_p, s), head(a.cap_p, s), tail(a.cap_p, s),
      seg_start(a.cap_seg, s), seg_len(a.cap_seg, s), seg_next(a.cap_seg, s), pool(a.cap_pool, s),
      pool2(a.cap_pool, s),
      dist(n, s), lab(n, s), fa(n, s), fb(n, s), remap(a.cap_p, s), out(2, s), cnt(P, s), st(P, s);
  bucket_by_patch(ctx, n, assignment, P, st, cnt, pool);
  MP_KERNEL(ctx, seg_init<<<grid_for(ctx, P), 256, 0, s>>>(P, st, cnt, head, tail, seg_start, seg_len,
                                                          seg_next, size, exempt));
  a.size = size, a.exempt = exempt, a.head = head, a.tail = tail, a.seg_start = seg_start;
  a.seg_len = seg_len, a.seg_next = seg_next, a.pool = pool, a.pool2 = pool2, a.dist = dist, a.lab = lab;
  a.fa = fa, a.fb = fb, a.remap = remap, a.out = out;
  allow_max_smem(repair_kernel, ctx.device);
  a.smem_words = kRepairSmemBytes / 4;
  MP_KERNEL(ctx, repair_kernel<<<1, 1024, kRepairSmemBytes, s>>>(a));
  int32_t h_out[2];
  MP_CUDA(cudaMemcpyAsync(h_out, out, sizeof h_out, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (h_out[1]) throw Error(MP_ENOMEM, "repair_sizes: split workspace exhausted");
  MP_KERNEL(ctx, apply_remap<<<grid_for(ctx, n), 256, 0, s>>>(n, remap, assignment));
  return h_out[0];
}

}  // namespace

void fps_batched_dev(mp_context& ctx, const DGraph& g, const int32_t* ell, int32_t k, uint64_t seed, int32_t* seeds,
                     int32_t* dist);

int32_t enforce_connectivity_dev(mp_context& ctx, const DGraph& g, const int32_t* in,
                                 int32_t P, int32_t* out) {
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  if (n == 0) return P;
  DevBuf<int32_t> bad(1, s);
  MP_KERNEL(ctx, fill_i32<<<1, 32, 0, s>>>(1, bad, 0x7fffffff));
  MP_KERNEL(ctx, check_range<<<grid_for(ctx, n), 256, 0, s>>>(n, in, P, bad));
  int32_t h_bad;
  MP_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (h_bad != 0x7fffffff)
    throw Error(MP_EINVAL, "patch id out of range at vertex " + std::to_string(h_bad));
  DevBuf<int32_t> par(n, s), minv(std::max(P, 1), s), root_id(n, s), cnt(1, s);
  DevBuf<uint64_t> keys(n, s);
  union_find(ctx, g, in, par);
  MP_KERNEL(ctx, fill_i32<<<grid_for(ctx, P), 256, 0, s>>>(P, minv, 0x7fffffff));
  MP_KERNEL(ctx, patch_min_vertex<<<grid_for(ctx, n), 256, 0, s>>>(n, in, minv));
  MP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t), s));
  MP_KERNEL(ctx, collect_extra_roots<<<grid_for(ctx, n), 256, 0, s>>>(n, par, in, minv, keys, cnt));
  int32_t E = 0;
  MP_CUDA(cudaMemcpyAsync(&E, cnt, sizeof E, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  MP_KERNEL(ctx, fill_i32<<<grid_for(ctx, n), 256, 0, s>>>(n, root_id, -1));
  if (E > 0) {
    DevBuf<uint64_t> sorted(E, s);
    size_t tmp = 0;
    MP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.get(), sorted.get(), E, 0, 64, s));
    DevBuf<char> t(tmp, s);
    MP_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, keys.get(), sorted.get(), E, 0, 64, s));
    MP_KERNEL(ctx, fresh_ids<<<grid_for(ctx, E), 256, 0, s>>>(E, sorted, P, root_id));
  }
  MP_KERNEL(ctx, relabel_components<<<grid_for(ctx, n), 256, 0, s>>>(n, par, in, root_id, out));
  return P + E;
}

// ------------------------------------------------------------ validate_user_patches
// patching.cpp:386-433: sizes, patches with more than one component (union-
// find restricted to same-patch edges, one root per component), unused ids.
__global__ void patch_stats(int32_t n, const int32_t* assignment, const int32_t* par,
                            unsigned long long* size, int32_t* ncomp) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int32_t p = assignment[v];
    atomicAdd(&size[p], 1ull);
    if (par[v] == v) atomicAdd(&ncomp[p], 1);
  }
}

UserPatchReport validate_user_patches_dev(mp_context& ctx, const DGraph& g, const int32_t* in, int32_t P) {
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  if (P < 0) throw Error(MP_EINVAL, "patch count must be nonnegative");
  UserPatchReport r;
  r.sizes.assign(P, 0);
  if (n > 0) {
    DevBuf<int32_t> bad(1, s);
    MP_KERNEL(ctx, fill_i32<<<1, 32, 0, s>>>(1, bad, 0x7fffffff));
    MP_KERNEL(ctx, check_range<<<grid_for(ctx, n), 256, 0, s>>>(n, in, P, bad));
    int32_t h_bad;
    MP_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (h_bad != 0x7fffffff) {  // the first offending vertex, as the sequential scan reports it
      int32_t p = 0;
      MP_CUDA(cudaMemcpyAsync(&p, in + h_bad, sizeof p, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
      throw Error(MP_EINVAL, "patch id " + std::to_string(p) + " out of range at vertex " + std::to_string(h_bad));
    }
  }
  std::vector<int32_t> ncomp(P, 0);
  if (n > 0 && P > 0) {
    DevBuf<int32_t> par(n, s), d_ncomp(P, s);
    DevBuf<unsigned long long> d_size(P, s);
    union_find(ctx, g, in, par);
    MP_CUDA(cudaMemsetAsync(d_size, 0, sizeof(unsigned long long) * P, s));
    MP_CUDA(cudaMemsetAsync(d_ncomp, 0, sizeof(int32_t) * P, s));
    MP_KERNEL(ctx, patch_stats<<<grid_for(ctx, n), 256, 0, s>>>(n, in, par, d_size, d_ncomp));
    MP_CUDA(cudaMemcpyAsync(r.sizes.data(), d_size, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(ncomp.data(), d_ncomp, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
  }
  for (int32_t p = 0; p < P; ++p) {
    if (ncomp[p] > 1) r.disconnected.push_back(p);
    if (r.sizes[p] == 0) r.unused.push_back(p);
  }
  return r;
}

int32_t compute_patches_dev(mp_context& ctx, const DGraph& g, int32_t target, uint64_t seed,
                            int32_t* assignment) {
  if (target < 1) throw Error(MP_EINVAL, "target patch size must be positive");
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  if (n == 0) return 0;
  SectionTimer st(s, "patch");

  // connected components, ordered by smallest member (graph.cpp:183-205)
  DevBuf<int32_t> par(n, s), flag(n, s), rank(n, s);
  union_find(ctx, g, nullptr, par);
  MP_KERNEL(ctx, root_flags<<<grid_for(ctx, n), 256, 0, s>>>(n, par, flag));
  {
    size_t tmp = 0;
    MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag.get(), rank.get(), n, s));
    DevBuf<char> t(tmp, s);
    MP_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, flag.get(), rank.get(), n, s));
  }
  int32_t last[2];
  MP_CUDA(cudaMemcpyAsync(&last[0], rank.get() + n - 1, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaMemcpyAsync(&last[1], flag.get() + n - 1, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  const int32_t C = last[0] + last[1];

  DevBuf<int32_t> comp_of, comp_list, pos_of;
  DevBuf<int32_t> comp_size(C, s), comp_start(C, s), comp_k(C, s), comp_mode(C, s), comp_base(C, s),
      tile_base(C, s), super_base(C, s), totals(4, s);
  if (C == 1) {
    int32_t hn = n;
    MP_CUDA(cudaMemcpyAsync(comp_size.get(), &hn, 4, cudaMemcpyHostToDevice, s));
  } else {
    comp_of.alloc(n, s);
    comp_list.alloc(n, s);
    pos_of.alloc(n, s);
    MP_CUDA(cudaMemsetAsync(comp_size, 0, sizeof(int32_t) * C, s));
    MP_KERNEL(ctx, comp_of_kernel<<<grid_for(ctx, n), 256, 0, s>>>(n, par, rank, comp_of, comp_size));
    DevBuf<int32_t> vals(n, s), keys_out(n, s);
    MP_KERNEL(ctx, iota_kernel<<<grid_for(ctx, n), 256, 0, s>>>(n, vals));
    int end_bit = 1;
    while ((1LL << end_bit) < C) ++end_bit;
    size_t tmp = 0;
    MP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, comp_of.get(), keys_out.get(), vals.get(),
                                            comp_list.get(), n, 0, end_bit, s));
    DevBuf<char> t(tmp, s);
    MP_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, comp_of.get(), keys_out.get(), vals.get(),
                                            comp_list.get(), n, 0, end_bit, s));
    MP_KERNEL(ctx, scatter_pos<<<grid_for(ctx, n), 256, 0, s>>>(n, comp_list, pos_of));
  }
  st.mark("components");
  MP_KERNEL(ctx, plan_components<<<1, 1024, 0, s>>>(C, comp_size, target, comp_start, comp_k, comp_mode,
                                                   comp_base, tile_base, super_base, totals));
  int32_t h_tot[4];
  MP_CUDA(cudaMemcpyAsync(h_tot, totals, sizeof h_tot, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  const int32_t P0 = h_tot[0];

  MP_KERNEL(ctx, assign_trivial<<<grid_for(ctx, n), 256, 0, s>>>(n, comp_list, comp_of, comp_start,
                                                                comp_mode, comp_base, assignment));
  if (h_tot[1] > 0) {  // at least one FPS component
    DevBuf<int32_t> dist(n, s), fr(2LL * n, s), seeds(P0, s), ell(static_cast<int64_t>(n) * kEll, s);
    MP_KERNEL(ctx, build_ell<<<grid_for(ctx, n), 256, 0, s>>>(g, ell));
    DevBuf<uint64_t> tkey(h_tot[1], s), skey(h_tot[2], s);
    DevBuf<uint32_t> tbits(h_tot[1] / 32 + 2LL * C + 2, s);
    MP_CUDA(cudaMemsetAsync(tbits, 0, sizeof(uint32_t) * tbits.n, s));
    FpsArgs fa{};
    fa.g = g;
    fa.comp_list = comp_list.get();
    fa.pos_of = pos_of.get();
    fa.comp_start = comp_start, fa.comp_size = comp_size, fa.comp_k = comp_k;
    fa.comp_mode = comp_mode, fa.comp_base = comp_base, fa.tile_base = tile_base;
    fa.super_base = super_base, fa.dist = dist, fa.tile_key = tkey, fa.super_key = skey;
    fa.tile_bits = tbits, fa.frontier = fr, fa.seeds = seeds, fa.seed = seed, fa.work = ctx.dwork;
    st.mark("plan+ell");
    if (C == 1 && n >= kBatchedFpsMin) {
      // one large component: exact speculative batches over the whole GPU
      fps_batched_dev(ctx, g, ell, P0, seed, seeds, dist);
    } else {
      fa.ell = ell;
      // shared-memory components: 4 B distance + 16 B local ELL row per vertex
      const int32_t max_size = h_tot[3];
      const int64_t base_b = sizeof(int32_t) * (2 * kFrontCap + kSmemTileWords);
      const int64_t room = (static_cast<int64_t>(ctx.smem_optin) - 16 * 1024 - base_b) / 20;
      fa.smem_n = static_cast<int32_t>(std::min<int64_t>({room, kFrontCap, 65535, max_size}));
      const size_t fps_smem = static_cast<size_t>(base_b + 20LL * fa.smem_n);
      allow_max_smem(fps_kernel, ctx.device);
      { const int kt__ = ctx.ktime_begin(kKFps); MP_KERNEL(ctx, fps_kernel<<<C, kFpsThreads, fps_smem, s>>>(fa)); ctx.ktime_end(kt__); }
    }

    st.mark("fps");
    // Lloyd rounds: one cooperative kernel
    DevBuf<int32_t> label(n, s), prev(n, s), active(C, s), changed(static_cast<int64_t>(kLloydRounds) * C, s),
        counters(4, s), patch_comp;
    DevBuf<uint64_t> best(P0, s);
    MP_KERNEL(ctx, fill_i32<<<grid_for(ctx, n), 256, 0, s>>>(n, prev, kNone));
    MP_KERNEL(ctx, fill_i32<<<grid_for(ctx, C), 256, 0, s>>>(C, active, 1));
    MP_CUDA(cudaMemsetAsync(changed, 0, sizeof(int32_t) * changed.n, s));
    if (C > 1) {
      patch_comp.alloc(P0, s);
      MP_KERNEL(ctx, fill_i32<<<grid_for(ctx, P0), 256, 0, s>>>(P0, patch_comp, -1));
      MP_KERNEL(ctx, patch_comp_kernel<<<std::min(C, 4096), 256, 0, s>>>(C, comp_mode, comp_base, comp_k,
                                                                        patch_comp));
    }
    LloydArgs la{};
    la.g = g;
    la.comp_of = comp_of.get();
    la.comp_mode = comp_mode;
    la.comp_active = active;
    la.changed = changed;
    la.C = C;
    la.patch_comp = patch_comp.get();
    la.P = P0;
    la.seeds = seeds;
    la.dist = dist;
    la.label = label;
    la.prev = prev;
    la.best = best;
    la.fa = fr.get();
    la.fb = fr.get() + n;
    la.counters = counters;
    la.ell = ell;
    la.work = ctx.dwork;
    void* args[] = {&la};
    const int64_t cl_max = ctx.tune[MP_TUNE_LLOYD_CLUSTER_N] != 0 ? ctx.tune[MP_TUNE_LLOYD_CLUSTER_N] : kLloydClusterN;
    const int cl = n <= cl_max ? lloyd_cluster_ctas(ctx.device) : 0;
    const size_t lsm_bytes = sizeof(int32_t) * 13 * static_cast<size_t>(n);  // ELL (8) + dist, label, prev, two frontiers
    cudaFuncAttributes lfa{};
    MP_CUDA(cudaFuncGetAttributes(&lfa, lloyd_kernel<BlockBarrier, true>));
    if (n <= kLloydSmemN && ctx.tune[MP_TUNE_LLOYD_CLUSTER_N] >= 0 &&
        lsm_bytes + lfa.sharedSizeBytes <= static_cast<size_t>(ctx.smem_optin)) {
      allow_max_smem(lloyd_kernel<BlockBarrier, true>, ctx.device);
      const int kt__ = ctx.ktime_begin(kKLloyd);
      MP_KERNEL(ctx, lloyd_kernel<BlockBarrier, true><<<1, kLloydClusterThreads, lsm_bytes, s>>>(la));
      ctx.ktime_end(kt__);
    } else if (cl > 0) {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cl), cfg.blockDim = dim3(kLloydClusterThreads), cfg.dynamicSmemBytes = 0;
      cfg.stream = s, cfg.attrs = at, cfg.numAttrs = 1;
      const int kt__ = ctx.ktime_begin(kKLloyd);
      MP_KERNEL(ctx, MP_CUDA(cudaLaunchKernelEx(&cfg, lloyd_kernel<ClusterBarrier>, la)));
      ctx.ktime_end(kt__);
    } else {
    int bpsm = 0;
    MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, lloyd_kernel<GridBarrier>, 256, 0));
    int blocks = std::max(1, std::min(bpsm, 4)) * std::max(ctx.num_sms / std::max(ctx.sm_share, 1), 1);
    // small meshes: one CTA per SM is enough and makes the grid barriers cheaper
    blocks = static_cast<int>(std::min<int64_t>(blocks, std::max<int64_t>(ctx.num_sms / std::max(ctx.sm_share, 1), ceil_div(n, 512))));
    if (ctx.tune[MP_TUNE_LLOYD_BLOCKS] > 0)
      blocks = std::max(1, std::min<int>(blocks, static_cast<int>(ctx.tune[MP_TUNE_LLOYD_BLOCKS])));
    { const int kt__ = ctx.ktime_begin(kKLloyd); MP_KERNEL(ctx, MP_CUDA(cudaLaunchCooperativeKernel((void*)lloyd_kernel<GridBarrier>, blocks, 256, args, 0, s))); ctx.ktime_end(kt__); }
    }
    MP_KERNEL(ctx, lloyd_finish<<<grid_for(ctx, n), 256, 0, s>>>(n, comp_of.get(), comp_mode, prev, assignment));
  }
  st.mark("lloyd");
  DevBuf<int32_t> conn(n, s);
  int32_t P1 = enforce_connectivity_dev(ctx, g, assignment, P0, conn);
  MP_CUDA(cudaMemcpyAsync(assignment, conn, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  st.mark("connectivity");
  const int32_t P2 = repair_sizes_dev(ctx, g, assignment, P1, target);
  st.mark("repair");
  return P2;
}

}  // namespace mp
