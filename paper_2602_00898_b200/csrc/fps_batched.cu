// Farthest-point seeding, exact speculative batches (reference
// core/src/patching.cpp:26-65), for one large connected component.
//
// The reference picks seeds one at a time: argmax over the component of the
// packed key (dist desc, id asc), then relaxes dist from the new seed.  A
// relaxation from c only lowers dist inside R(c) = {v : d(c,v) < dist(v)},
// and min() makes relaxations commute.  A batch therefore:
//   1. takes a candidate list S sorted by key desc that is downward closed
//      (every vertex with key >= min key(S) is in S): a dist threshold picked
//      from a histogram of the tile maxima, then the vertices of the tiles at
//      or above it (tiles are id ranges, so ties truncate by ascending id);
//   2. computes R(c_j) and d(c_j, .) for the first W candidates in parallel,
//      one worker CTA each, against the committed dist;
//   3. walks S in order (every CTA, redundantly): a candidate inside an
//      accepted region is skipped -- its key fell to <= M, the largest key an
//      accepted region can leave; the first candidate outside the accepted
//      regions whose key beats M is the true next seed; a candidate whose key
//      does not beat M ends the batch;
//   4. commits min(dist, d(c_j, .)) over the accepted regions and refreshes
//      the touched tile maxima.
// The accepted sequence is exactly the sequential FPS sequence.  Batch 0 is
// the seed-derived start vertex alone (patching.cpp:32).
#include <cub/cub.cuh>

#include <algorithm>
#include <map>
#include <mutex>
#include <cstdlib>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kThreads = 1024;
constexpr int kBins = 4096;       // tile-max dist histogram (distances binned by >> shift)
constexpr int kSCap = 4096;       // candidate list capacity
constexpr int kFront = 4096;      // smem frontier per buffer in a worker
constexpr int kMaxWorkers = 640;  // candidates per batch (bit-matrix width)
constexpr int kMaxSub = 4;        // worker groups per CTA when regions are small
constexpr int kSubRegion = 4096;  // ... i.e. when the last batch's largest region was below this
constexpr int kMaskWords = kMaxWorkers / 32;
constexpr int kGridCands = 64;    // candidates per grid-mode batch
constexpr int kQHead = 0, kQTail = 32, kQPend = 64;  // cluster-queue control words, 128 B apart
constexpr int kMaxDepth = 250;    // worker BFS depth bound (< the grid radius, clamped to it)

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {  // patching.cpp:17-22
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d649bb133111ebULL;
  return x ^ (x >> 31);
}

struct BatchArgs {
  DGraph g;
  const int32_t* ell;      // n * 8 ELL adjacency (slot 7 < -1 encodes a CSR tail)
  int32_t n, k, tile_shift, ntile;
  uint64_t seed;
  int32_t* dist;
  uint64_t* tkey;          // ntile tile maxima
  int32_t* smax;           // n/32 subtile maximum distances (refreshed with the tiles)
  uint32_t* tbits;         // touched tiles
  int32_t* tlist;          // ntile
  uint32_t* vm;            // visit bits, one plane of vwords words per worker: bit v of plane j = v in region j
  int64_t vwords;
  int32_t* dw;             // grid-mode distances, grid_cands * n
  int32_t* reg;            // W * n worker region lists (level-ordered)
  int32_t* cand;           // kSCap
  uint64_t* ckey;          // kSCap
  uint64_t* mkey;          // kMaxWorkers: largest key a region leaves
  uint32_t* inm;           // kMaxWorkers * kMaskWords membership bits
  int32_t* regn;           // kMaxWorkers region sizes
  int32_t* ctl;            // [0] seeds done [1] ncand [2] touched count [3] grid mode [4..6] level counters [8] glist size
                           // [9] worker groups per CTA [10] list overflow [11] largest region
  uint64_t* glist;         // grid-mode region entries (cand << 32 | vertex)
  int32_t* tscratch;       // ntile: tiles at the tied maximum distance
  unsigned int* bar;       // grid barrier counter (zeroed before the launch)
  int32_t grid_radius;     // candidates farther than this use the grid-mode regions
  int32_t grid_cands;      // candidates per grid-mode batch
  int32_t sub_region;      // largest region (last batch) that still runs kMaxSub groups per CTA
  int32_t resume;          // 1: fps_cluster_phase ran the large-radius seeds; continue from its state
  int32_t* queue;          // cluster phase work queue (qcap slots, -1 = empty)
  int32_t* qctl;           // [0] head [1] tail [2] pending
  int64_t qcap;
  int32_t* seeds;          // output, k
  unsigned long long* work;
};

// Grid barrier for a co-resident (cooperatively launched) grid: one arrival
// atomic per CTA on a monotone counter, spin on it with acquire loads.
struct GridBar {
  unsigned int* count;
  unsigned int target = 0;
  __device__ void sync() {
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(count, 1u);
      unsigned int seen;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(count));
      } while (static_cast<int>(seen - target) < 0);
    }
    __syncthreads();
  }
};

__device__ __forceinline__ uint64_t vkey(int32_t d, int32_t v) {
  return key_max(static_cast<uint32_t>(d), static_cast<uint32_t>(v));
}

// Block-wide bitonic sort (descending) of m = power-of-two keys in smem.
// Compare-exchange stages with a partner less than 64 elements away run in
// registers: a warp owns 64 consecutive keys (two per lane; partners at
// distance 1 in the same thread, 2..32 one shuffle away), so only the stages
// with stride >= 64 go through shared memory and a block barrier (15 of the
// 66 stages at m = 2048).
__device__ __forceinline__ void bitonic_reg_stages(uint64_t& x0, uint64_t& x1, int32_t base, int32_t size,
                                                   int32_t top_stride) {
  const int lane = threadIdx.x & 31;
  for (int32_t stride = top_stride; stride > 0; stride >>= 1) {
    if (stride == 1) {
      const bool desc = ((base + 2 * lane) & size) == 0;
      const uint64_t hi = max(x0, x1), lo = min(x0, x1);
      x0 = desc ? hi : lo;
      x1 = desc ? lo : hi;
    } else {
      const int32_t pl = stride >> 1;  // partner lane distance
      const bool lower = ((2 * lane) & stride) == 0;
      const bool desc = ((base + 2 * lane) & size) == 0;
      const bool keep_max = lower == desc;
      const uint64_t y0 = __shfl_xor_sync(0xffffffffu, x0, pl), y1 = __shfl_xor_sync(0xffffffffu, x1, pl);
      x0 = keep_max ? max(x0, y0) : min(x0, y0);
      x1 = keep_max ? max(x1, y1) : min(x1, y1);
    }
  }
}

__device__ void bitonic_desc(uint64_t* s, int32_t m) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (m < 64) {  // tiny lists: plain shared-memory network
    for (int32_t size = 2; size <= m; size <<= 1) {
      for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (int32_t t = threadIdx.x; t < m / 2; t += blockDim.x) {
          const int32_t i = 2 * t - (t & (stride - 1));
          const int32_t j = i + stride;
          const bool up = (i & size) == 0;
          const uint64_t x = s[i], y = s[j];
          if ((x < y) == up) s[i] = y, s[j] = x;
        }
        __syncthreads();
      }
    }
    return;
  }
  const int32_t nchunk = m >> 6;
  // sizes 2..64: every 64-key chunk sorted in registers (alternating directions)
  for (int32_t c = wid; c < nchunk; c += nw) {
    const int32_t base = c << 6;
    uint64_t x0 = s[base + 2 * lane], x1 = s[base + 2 * lane + 1];
    for (int32_t size = 2; size <= 64; size <<= 1) bitonic_reg_stages(x0, x1, base, size, size >> 1);
    s[base + 2 * lane] = x0, s[base + 2 * lane + 1] = x1;
  }
  __syncthreads();
  for (int32_t size = 128; size <= m; size <<= 1) {
    for (int32_t stride = size >> 1; stride >= 64; stride >>= 1) {
      for (int32_t t = threadIdx.x; t < m / 2; t += blockDim.x) {
        const int32_t i = 2 * t - (t & (stride - 1));
        const int32_t j = i + stride;
        const bool up = (i & size) == 0;
        const uint64_t x = s[i], y = s[j];
        if ((x < y) == up) s[i] = y, s[j] = x;
      }
      __syncthreads();
    }
    for (int32_t c = wid; c < nchunk; c += nw) {
      const int32_t base = c << 6;
      uint64_t x0 = s[base + 2 * lane], x1 = s[base + 2 * lane + 1];
      bitonic_reg_stages(x0, x1, base, size, 32);
      s[base + 2 * lane] = x0, s[base + 2 * lane + 1] = x1;
    }
    __syncthreads();
  }
}

// Leader: the downward-closed candidate list of this batch.
__device__ void select_candidates(const BatchArgs& a, int32_t W, uint64_t* sS, int32_t* hist, int32_t* shi) {
  __shared__ int32_t s_n, s_thr, s_gq, s_gs;
  int32_t* ssub = hist;                   // subtile list (reuses the histogram, kBins >= kSCap)
  __shared__ int32_t scnt[kMaxWorkers];   // exact mode: per-subtile counts / offsets
  __shared__ uint64_t red[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int32_t tsize = 1 << a.tile_shift;
  // histogram of tile-max distances, binned so the largest fits
  // (the tile scans keep kU loads in flight per thread: C3 has 39K tiles,
  // ~38 per thread, and one dependent L2 round trip each cost ~30 us a batch)
  constexpr int kU = 8;
  uint64_t mx = 0;
  for (int32_t t0 = threadIdx.x; t0 < a.ntile; t0 += kU * blockDim.x) {
    uint64_t v[kU];
#pragma unroll
    for (int g = 0; g < kU; ++g) {
      const int32_t t = t0 + g * static_cast<int32_t>(blockDim.x);
      v[g] = t < a.ntile ? __ldcg(&a.tkey[t]) : 0;
    }
#pragma unroll
    for (int g = 0; g < kU; ++g) mx = max(mx, v[g] >> 32);
  }
  mx = block_max_u64(mx, red);
  int32_t shift = 0;
  while ((mx >> shift) >= static_cast<uint64_t>(kBins)) ++shift;
  for (int32_t b = threadIdx.x; b < kBins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  // late batches put most tiles in a few bins: one shared atomic per distinct
  // bin per warp instead of one per tile
  for (int32_t t0 = 0; t0 < a.ntile; t0 += kU * blockDim.x) {
    int32_t bs[kU];
#pragma unroll
    for (int g = 0; g < kU; ++g) {
      const int32_t t = t0 + g * static_cast<int32_t>(blockDim.x) + static_cast<int32_t>(threadIdx.x);
      bs[g] = t < a.ntile ? static_cast<int32_t>((__ldcg(&a.tkey[t]) >> 32) >> shift) : -1;
    }
#pragma unroll
    for (int g = 0; g < kU; ++g) {
      const int32_t b = bs[g];
      const uint32_t m = __match_any_sync(0xffffffffu, b);
      if (b >= 0 && lane == __ffs(m) - 1) atomicAdd(&hist[b], __popc(m));
    }
  }
  __syncthreads();
  // the highest bin b where the suffix count reaches W: tiles in bins > b are
  // fewer than W and form the threshold; if there are none, the top bin's
  // exact maximum distance with ties truncated by id
  const int32_t per = kBins / static_cast<int32_t>(blockDim.x);
  int32_t mine = 0;
  for (int32_t q = 0; q < per; ++q) mine += hist[kBins - 1 - (static_cast<int32_t>(threadIdx.x) * per + q)];
  int32_t tot;
  const int32_t before = block_excl_scan(mine, shi, &tot);
  if (threadIdx.x == 0) s_thr = -1;
  __syncthreads();
  if (before < W && before + mine >= W) {
    int32_t run = before;
    for (int32_t q = 0; q < per; ++q) {
      const int32_t b = kBins - 1 - (static_cast<int32_t>(threadIdx.x) * per + q);
      if (run + hist[b] >= W) {
        s_thr = b + 1;
        break;
      }
      run += hist[b];
    }
  }
  __syncthreads();
  int64_t thr_d;  // candidates: all vertices with dist >= thr_d
  bool exact = false;
  if (s_thr < 0) {
    thr_d = 0;  // fewer than W tiles overall
  } else if ((static_cast<int64_t>(s_thr) << shift) > static_cast<int64_t>(mx)) {
    thr_d = static_cast<int64_t>(mx);
    exact = true;
  } else {
    thr_d = static_cast<int64_t>(s_thr) << shift;
  }
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  // Candidates: every vertex with dist >= thr_d (or, in exact mode, the first
  // W vertices in id order with dist == thr_d).  Tiles at or above the
  // threshold are compacted in order, then their 32-vertex subtiles whose
  // maximum qualifies, then those subtiles are swept one warp each.
  for (int pass = 0; pass < 2; ++pass) {
    const bool ex = exact;
    int32_t* tl = a.tscratch;
    const int32_t spt = tsize >> 5;  // subtiles per tile
    const int32_t cap_sub = ex ? min(W, kSCap) : kSCap;
    int32_t nq = 0, nsub = 0;
    if (!ex) {
      // every vertex above the threshold is taken and the list is sorted by
      // key afterwards, so tiles and subtiles are gathered unordered: shared
      // counters, kG items per thread with their loads in flight together
      constexpr int kG = 4;
      if (threadIdx.x == 0) s_gq = 0, s_gs = 0;
      __syncthreads();
      for (int32_t t0 = threadIdx.x; t0 < a.ntile; t0 += kG * blockDim.x) {
        uint64_t tk[kG];
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const int32_t t = t0 + g * blockDim.x;
          tk[g] = t < a.ntile ? __ldcg(&a.tkey[t]) : 0;
        }
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const int32_t t = t0 + g * blockDim.x;
          if (t < a.ntile && static_cast<int64_t>(tk[g] >> 32) >= thr_d) tl[atomicAdd(&s_gq, 1)] = t;
        }
      }
      __syncthreads();
      nq = s_gq;
      const int64_t total = static_cast<int64_t>(nq) * spt;
      for (int64_t q0 = threadIdx.x; q0 < total; q0 += kG * blockDim.x) {
        int32_t sub[kG];
        int64_t sd[kG];
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const int64_t q = q0 + static_cast<int64_t>(g) * blockDim.x;
          sub[g] = q < total ? __ldcg(&tl[q / spt]) * spt + static_cast<int32_t>(q % spt) : -1;
        }
#pragma unroll
        for (int g = 0; g < kG; ++g)
          sd[g] = sub[g] >= 0 && (static_cast<int64_t>(sub[g]) << 5) < a.n ? static_cast<int64_t>(__ldcg(&a.smax[sub[g]])) : -1;
#pragma unroll
        for (int g = 0; g < kG; ++g)
          if (sd[g] >= thr_d && sd[g] >= 0) {
            const int32_t at = atomicAdd(&s_gs, 1);
            if (at < cap_sub) ssub[at] = sub[g];
          }
      }
      __syncthreads();
      nsub = s_gs;
    } else {
      for (int32_t t0 = 0; t0 < a.ntile; t0 += blockDim.x) {
        const int32_t t = t0 + threadIdx.x;
        int32_t f = 0;
        if (t < a.ntile) f = static_cast<int64_t>(__ldcg(&a.tkey[t]) >> 32) == thr_d;
        int32_t tt;
        const int32_t e = block_excl_scan(f, shi, &tt);
        if (f) tl[nq + e] = t;
        nq += tt;
      }
      __syncthreads();
      // qualifying subtiles, in id order (exact mode truncates ties by id)
      for (int64_t q0 = 0; q0 < static_cast<int64_t>(nq) * spt && nsub < cap_sub; q0 += blockDim.x) {
        const int64_t q = q0 + threadIdx.x;
        int32_t f = 0, sub = 0;
        if (q < static_cast<int64_t>(nq) * spt) {
          sub = __ldcg(&tl[q / spt]) * spt + static_cast<int32_t>(q % spt);
          if ((static_cast<int64_t>(sub) << 5) < a.n) f = static_cast<int64_t>(__ldcg(&a.smax[sub])) == thr_d;
        }
        int32_t tt;
        const int32_t e = block_excl_scan(f, shi, &tt);
        if (f && nsub + e < cap_sub) ssub[nsub + e] = sub;
        nsub += tt;
      }
    }
    if (!ex && nsub > cap_sub) {  // more than kSCap candidates: the exact-max rule instead
      __syncthreads();
      thr_d = static_cast<int64_t>(mx);
      exact = true;
      continue;
    }
    nsub = min(nsub, cap_sub);
    __syncthreads();
    if (!ex) {
      for (int32_t k = wid; k < nsub; k += nwarp) {
        const int32_t v = (ssub[k] << 5) + lane;
        const int32_t dv = v < a.n ? __ldcg(&a.dist[v]) : -1;
        const bool take = dv >= thr_d;
        const int32_t slot = warp_append(&s_n, take);
        if (take && slot < kSCap) sS[slot] = vkey(dv, v);
      }
      __syncthreads();
      if (s_n > kSCap) {  // a non-tie set cannot be truncated: the exact-max rule instead
        thr_d = static_cast<int64_t>(mx);
        exact = true;
        __syncthreads();
        if (threadIdx.x == 0) s_n = 0;
        __syncthreads();
        continue;
      }
    } else {
      // ties at the maximum, truncated in ascending id order: per-subtile
      // counts, one block scan (<= W subtiles), then ordered writes
      int32_t cnt = 0;
      for (int32_t k = wid; k < nsub; k += nwarp) {
        const int32_t v = (ssub[k] << 5) + lane;
        const int32_t c = __popc(__ballot_sync(0xffffffffu, v < a.n && __ldcg(&a.dist[v]) == thr_d));
        if (lane == 0) scnt[k] = c;
      }
      __syncthreads();
      if (threadIdx.x < nsub) cnt = scnt[threadIdx.x];
      int32_t tt;
      const int32_t base = block_excl_scan(cnt, shi, &tt);
      if (threadIdx.x < nsub) scnt[threadIdx.x] = base;
      __syncthreads();
      const int32_t capv = min(W, kSCap);
      for (int32_t k = wid; k < nsub; k += nwarp) {
        const int32_t v = (ssub[k] << 5) + lane;
        const int32_t dv = v < a.n ? __ldcg(&a.dist[v]) : -1;
        const bool take = dv == thr_d;
        const uint32_t m = __ballot_sync(0xffffffffu, take);
        const int32_t pos = scnt[k] + __popc(m & ((1u << lane) - 1));
        if (take && pos < capv) sS[pos] = vkey(dv, v);
      }
      if (threadIdx.x == 0) s_n = min(tt, capv);
      if (threadIdx.x == 0 && a.work) atomicAdd(&a.work[15], 1ull);
    }
    break;
  }
  __syncthreads();
  const int32_t ns = min(s_n, kSCap);
  int32_t m2 = 1;
  while (m2 < ns) m2 <<= 1;
  for (int32_t i = ns + threadIdx.x; i < m2; i += blockDim.x) sS[i] = 0;
  __syncthreads();
  bitonic_desc(sS, m2);
  const int32_t nc = min(ns, W);
  for (int32_t i = threadIdx.x; i < nc; i += blockDim.x) {
    a.ckey[i] = sS[i];
    a.cand[i] = static_cast<int32_t>(key_max_id(sS[i]));
  }
  if (threadIdx.x == 0) {
    a.ctl[1] = nc;
    if (a.work) {
      atomicAdd(&a.work[4], 1ull), atomicAdd(&a.work[6], static_cast<unsigned long long>(nc));
      atomicAdd(&a.work[13], exact ? 1ull : 0ull);
      atomicAdd(&a.work[14], static_cast<unsigned long long>(ns));
    }
  }
}

__global__ void __launch_bounds__(kThreads) fps_batched_kernel(BatchArgs a) {
  GridBar grid{a.bar};
  extern __shared__ uint64_t bsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  __shared__ int32_t s_cnt[3], s_n, s_done, shi[32];
  __shared__ uint64_t s_red[32];
  __shared__ int32_t s_acc[kMaxWorkers];
  unsigned long long scans = 0;
  // worker groups (per batch): nsub groups of G threads per CTA, one candidate each
  __shared__ int32_t s_wcnt[kMaxSub][3], s_wn[kMaxSub], s_wnlev[kMaxSub];
  __shared__ int32_t s_wlstart[kMaxSub][kMaxDepth + 2];  // region-list offset of each BFS level

  if (a.resume && __ldcg(&a.ctl[12]) == 0) {  // seeds, dist, tiles and the next candidates from fps_cluster_phase
    if (__ldcg(&a.ctl[0]) >= a.k) return;
  } else {  // (no cluster phase, or its queue overflowed: start over here)
    if (a.resume) {
      const int32_t nt = a.ntile / 32 + 1;
      for (int64_t i = gtid; i < nt; i += gthreads) a.tbits[i] = 0;
    }
    for (int64_t v = gtid; v < a.n; v += gthreads) a.dist[v] = kUnreached;
    if (gtid == 0) {
      a.ctl[0] = 0, a.ctl[2] = 0, a.ctl[1] = 1, a.ctl[3] = 1;  // batch 0: the start vertex, grid mode
      a.ctl[9] = 1, a.ctl[10] = 0, a.ctl[11] = 0;
      a.cand[0] = static_cast<int32_t>(splitmix64(a.seed) % static_cast<uint64_t>(a.n));  // patching.cpp:32
      a.ckey[0] = ~0ull;
    }
    grid.sync();
  }
  for (int32_t batch = 0;; ++batch) {
    // ---- 2. regions.  Large radii: all candidates advance together over the
    // whole grid (one grid barrier per level, entries (cand, vertex) appended
    // to one list).  Small radii: one worker CTA per candidate.
    const bool gridmode = __ldcg(&a.ctl[3]) != 0;
    int32_t nc, nsub, G, sub, gt, wk, my_word;
    uint32_t my_bit;
    int64_t reg_cap, my_plane;
    int32_t* my_reg;
    long long t_reg0 = clock64();
    for (;;) {  // a worker whose region outgrows its list share: redo with one group per CTA
    nc = __ldcg(&a.ctl[1]);
    nsub = __ldcg(&a.ctl[9]);  // worker groups per CTA (1 or kMaxSub)
    G = static_cast<int32_t>(blockDim.x) / nsub;
    sub = static_cast<int32_t>(threadIdx.x) / G, gt = static_cast<int32_t>(threadIdx.x) - sub * G;
    wk = static_cast<int32_t>(blockIdx.x) * nsub + sub;  // candidate of this group
    my_word = wk >> 5;
    my_bit = 1u << (wk & 31);
    my_plane = static_cast<int64_t>(wk) * a.vwords;
    reg_cap = a.n / nsub;
    my_reg = a.reg + static_cast<int64_t>(blockIdx.x) * a.n + static_cast<int64_t>(sub) * reg_cap;
    auto gsync = [&]() {
      if (nsub == 1) __syncthreads();
      else asm volatile("bar.sync %0, %1;" ::"r"(1 + sub), "r"(G) : "memory");
    };
    if (gridmode) {
      for (int32_t j = static_cast<int32_t>(gtid); j < nc; j += static_cast<int32_t>(gthreads)) {
        const int32_t c = __ldcg(&a.cand[j]);
        atomicOr(&a.vm[static_cast<int64_t>(j) * a.vwords + (c >> 5)], 1u << (c & 31));
        a.dw[static_cast<int64_t>(j) * a.n + c] = 0;
        a.glist[j] = (static_cast<uint64_t>(j) << 32) | static_cast<uint32_t>(c);
        a.mkey[j] = vkey(0, c);
      }
      if (gtid == 0) a.ctl[4] = nc, a.ctl[5] = 0, a.ctl[6] = 0, a.ctl[8] = 0;
      grid.sync();
      int32_t lbeg = 0;  // current level = glist[lbeg, lbeg + nf)
      for (int32_t d = 0;; ++d) {
        const int32_t nf = __ldcg(&a.ctl[4 + d % 3]);
        if (nf == 0) break;
        if (gtid == 0) a.ctl[4 + (d + 2) % 3] = 0;
        int32_t* cout = &a.ctl[4 + (d + 1) % 3];
        const int32_t lnext = lbeg + nf;
        const int64_t items = static_cast<int64_t>(nf) * 8;
        for (int64_t base = gtid - lane; base < items; base += gthreads) {
          const int64_t it = base + lane;
          uint64_t e = 0;
          int32_t x = -1;
          if (it < items) {
            e = __ldcg(&a.glist[lbeg + (it >> 3)]);
            x = a.ell[static_cast<int64_t>(static_cast<uint32_t>(e)) * 8 + (it & 7)];
          }
          const int32_t j = static_cast<int32_t>(e >> 32);
          int32_t* jdw = a.dw + static_cast<int64_t>(j) * a.n;
          const int32_t jword = j >> 5;
          const uint32_t jbit = 1u << (j & 31);
          uint64_t mk = 0;  // largest key this lane claims (the region's max key, mkey)
          auto claim = [&](int32_t w) -> bool {
            const uint32_t wb = 1u << (w & 31);
            if (d + 1 < __ldcg(&a.dist[w]) && !(atomicOr(&a.vm[static_cast<int64_t>(j) * a.vwords + (w >> 5)], wb) & wb)) {
              jdw[w] = d + 1;
              mk = max(mk, vkey(d + 1, w));
              return true;
            }
            return false;
          };
          const bool push = x >= 0 && claim(x);
          const int32_t slot = warp_append(cout, push);
          if (push) a.glist[lnext + slot] = (static_cast<uint64_t>(j) << 32) | static_cast<uint32_t>(x);
          if (x < -1) {
            const int32_t u = static_cast<int32_t>(static_cast<uint32_t>(e));
            for (int32_t q = -x - 2; q < a.g.off[u + 1]; ++q) {
              const int32_t w = a.g.nbr[q];
              if (claim(w)) a.glist[lnext + atomicAdd(cout, 1)] = (static_cast<uint64_t>(j) << 32) | static_cast<uint32_t>(w);
            }
          }
          // one atomic per warp when its lanes share the candidate (always with one)
          if (__match_any_sync(0xffffffffu, j) == 0xffffffffu) {
            const uint64_t gm = warp_max_u64(mk);
            if (lane == 0 && gm) atomicMax(reinterpret_cast<unsigned long long*>(&a.mkey[j]), static_cast<unsigned long long>(gm));
          } else if (mk) {
            atomicMax(reinterpret_cast<unsigned long long*>(&a.mkey[j]), static_cast<unsigned long long>(mk));
          }
        }
        grid.sync();
        if (gtid == 0 && a.work) atomicAdd(&a.work[5], 1ull);
        lbeg = lnext;
      }
      if (gtid == 0) a.ctl[8] = lbeg;  // entries in glist
      for (int32_t q = static_cast<int32_t>(gtid); q < nc * nc; q += static_cast<int32_t>(gthreads)) {
        const int32_t i = q / nc, j = q % nc;
        const int32_t cj = __ldcg(&a.cand[j]);
        if ((__ldcg(&a.vm[static_cast<int64_t>(i) * a.vwords + (cj >> 5)]) >> (cj & 31)) & 1u)
          atomicOr(&a.inm[i * kMaskWords + (j >> 5)], 1u << (j & 31));
      }
    } else if (wk < nc) {
      // worker group `sub` of this CTA (G threads) grows the region of candidate wk
      const int32_t c = __ldcg(&a.cand[wk]);
      const int32_t fcap = kFront / nsub;
      int32_t* sf0 = reinterpret_cast<int32_t*>(bsm) + 2 * fcap * sub;
      int32_t* sf1 = sf0 + fcap;
      int32_t* cnt3 = s_wcnt[sub];
      int32_t* lstart = s_wlstart[sub];
      if (gt == 0) {
        atomicOr(&a.vm[my_plane + (c >> 5)], 1u << (c & 31));
        my_reg[0] = c;
        lstart[0] = 0;
        sf0[0] = c;
        cnt3[0] = 1, cnt3[1] = 0, cnt3[2] = 0;
        s_wn[sub] = 1;  // region size
      }
      gsync();
      uint64_t mk = vkey(0, c);
      // region size, tracked identically by every thread of the group (all
      // inputs are group-uniform), so one barrier per level suffices: the
      // level counters rotate over three slots (read / written / cleared)
      int32_t wn = 1;
      for (int32_t d = 0;; ++d) {
        const int32_t nf = cnt3[d % 3];
        if (nf == 0) {
          if (gt == 0) s_wnlev[sub] = d;
          break;
        }
        if (gt == 0) cnt3[(d + 2) % 3] = 0;
        const int32_t* fin = (d & 1) ? sf1 : sf0;
        int32_t* fout = (d & 1) ? sf0 : sf1;
        const int32_t rbase = wn - nf;  // this level's vertices end the region list
        const int32_t rtop = wn;
        if (gt == 0) lstart[d + 1] = rtop;  // depth d+1 entries start here
        int32_t* cout = &cnt3[(d + 1) % 3];
        const int32_t items = nf * 8;
        auto relax = [&](int32_t w) {
          if (d + 1 < __ldcg(&a.dist[w]) &&
              !(atomicOr(&a.vm[my_plane + (w >> 5)], 1u << (w & 31)) & (1u << (w & 31)))) {
            const int32_t slot = atomicAdd(cout, 1);
            if (slot < fcap) fout[slot] = w;
            if (rtop + slot < reg_cap) my_reg[rtop + slot] = w;
            mk = max(mk, vkey(d + 1, w));
          }
        };
        // kUnroll items per thread with their loads and claims in flight together
        constexpr int kUnroll = 4;
        for (int32_t it0 = 0; it0 < items; it0 += kUnroll * G) {
          int32_t us[kUnroll], xs[kUnroll], ds[kUnroll];
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const int32_t it = it0 + q * G + gt;
            us[q] = -1, xs[q] = -1;
            if (it < items) {
              const int32_t i = it >> 3;
              us[q] = i < fcap ? fin[i] : __ldcg(&my_reg[rbase + i]);
              xs[q] = a.ell[static_cast<int64_t>(us[q]) * 8 + (it & 7)];
            }
          }
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) ds[q] = xs[q] >= 0 ? __ldcg(&a.dist[xs[q]]) : 0;
          uint32_t old[kUnroll];  // the claimed vertex's previous visit bit (1: already ours)
#pragma unroll
          for (int q = 0; q < kUnroll; ++q)
            old[q] = (xs[q] >= 0 && d + 1 < ds[q])
                         ? atomicOr(&a.vm[my_plane + (xs[q] >> 5)], 1u << (xs[q] & 31)) >> (xs[q] & 31) & 1u
                         : 1u;
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            if (!old[q]) {
              const int32_t w = xs[q];
              const int32_t slot = atomicAdd(cout, 1);
              if (slot < fcap) fout[slot] = w;
              if (rtop + slot < reg_cap) my_reg[rtop + slot] = w;
              mk = max(mk, vkey(d + 1, w));
            }
            if (xs[q] < -1)  // CSR tail of a vertex with more than 8 neighbours
              for (int32_t j = -xs[q] - 2; j < a.g.off[us[q] + 1]; ++j) relax(a.g.nbr[j]);
          }
        }
        gsync();
        if (wn + *cout > reg_cap) {  // the region outgrew this group's list share
          if (gt == 0) s_wnlev[sub] = 0, atomicExch(&a.ctl[10], 1);
          break;
        }
        wn += *cout;
        if (gt == 0 && a.work && wk == 0) atomicAdd(&a.work[7], 1ull);
      }
      if (gt == 0) s_wn[sub] = wn;
      // group max of mk
      mk = warp_max_u64(mk);
      if (lane == 0) s_red[wid] = mk;
      gsync();
      if (gt < 32) {
        const int32_t w0 = sub * (G >> 5);
        uint64_t r = gt < (G >> 5) ? s_red[w0 + gt] : 0;
        r = warp_max_u64(r);
        if (gt == 0) {
          a.mkey[wk] = r;
          a.regn[wk] = s_wn[sub];
          atomicMax(&a.ctl[11], s_wn[sub]);
        }
      }
      for (int32_t j0 = 0; j0 < nc; j0 += G) {  // which candidates lie in this region
        const int32_t j = j0 + gt;
        int32_t cj = 0;
        if (j < nc) cj = __ldcg(&a.cand[j]);
        const bool in = j < nc && ((__ldcg(&a.vm[my_plane + (cj >> 5)]) >> (cj & 31)) & 1u);
        const uint32_t bits = __ballot_sync(0xffffffffu, in);
        if (lane == 0 && j < kMaxWorkers) a.inm[wk * kMaskWords + (j >> 5)] = bits;
      }
    }
    grid.sync();
    if (__ldcg(&a.ctl[10]) == 0) break;
    for (int64_t q = gtid; q < static_cast<int64_t>(kMaxWorkers) * a.vwords; q += gthreads) a.vm[q] = 0;
    grid.sync();
    if (gtid == 0) a.ctl[10] = 0, a.ctl[9] = 1, a.ctl[1] = min(nc, static_cast<int32_t>(gridDim.x));
    grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.work) atomicAdd(&a.work[9], static_cast<unsigned long long>(clock64() - t_reg0));
    // ---- 3. the walk, every CTA redundantly (exact sequential argmax semantics).
    // The candidates' keys, region maxima and in-region masks are staged in
    // shared memory by the whole CTA first (one parallel L2 round), so each
    // accepted candidate costs shared-memory reads instead of dependent L2 loads.
    {
      uint64_t* s_ck = bsm;                                                   // nc keys
      uint64_t* s_mk = bsm + kMaxWorkers;                                     // nc region maxima
      uint32_t* s_in = reinterpret_cast<uint32_t*>(bsm + 2 * kMaxWorkers);    // nc x kMaskWords
      for (int32_t j = threadIdx.x; j < nc; j += blockDim.x) s_ck[j] = __ldcg(&a.ckey[j]), s_mk[j] = __ldcg(&a.mkey[j]);
      for (int32_t q = threadIdx.x; q < nc * kMaskWords; q += blockDim.x) s_in[q] = __ldcg(&a.inm[q]);
      __syncthreads();
      if (wid == 0) {
        uint32_t U = 0;  // lane w: bits [32w, 32w+32) of the accepted-region union
        uint64_t Mx = 0;
        int32_t done = __ldcg(&a.ctl[0]);
        for (int32_t j = lane; j < kMaxWorkers; j += 32) s_acc[j] = 0;
        __syncwarp();
        for (int32_t j = 0; j < nc; ++j) {
          const uint32_t uw = __shfl_sync(0xffffffffu, U, j >> 5);
          if ((uw >> (j & 31)) & 1u) continue;  // inside an accepted region: not a seed
          if (done >= a.k || !(s_ck[j] > Mx)) break;
          if (lane == 0) s_acc[j] = 1;
          if (lane < kMaskWords) U |= s_in[j * kMaskWords + lane];
          Mx = max(Mx, s_mk[j]);
          if (blockIdx.x == 0 && lane == 0) a.seeds[done] = __ldcg(&a.cand[j]);
          ++done;
        }
        if (lane == 0) s_done = done;
      }
      __syncthreads();
    }
    // ---- 4. commit the accepted regions
    long long t_c0 = clock64();
    if (gridmode) {
      const int32_t ne = __ldcg(&a.ctl[8]);
      for (int32_t q = static_cast<int32_t>(gtid); q < ne; q += static_cast<int32_t>(gthreads)) {
        const uint64_t e = __ldcg(&a.glist[q]);
        const int32_t j = static_cast<int32_t>(e >> 32), w = static_cast<int32_t>(static_cast<uint32_t>(e));
        a.vm[static_cast<int64_t>(j) * a.vwords + (w >> 5)] = 0;  // every region is finished: clear its bits
        if (!s_acc[j]) continue;
        atomicMin(&a.dist[w], __ldcg(&a.dw[static_cast<int64_t>(j) * a.n + w]));
        const int32_t t = w >> a.tile_shift;
        const uint32_t bit = 1u << (t & 31);
        if (!(atomicOr(&a.tbits[t >> 5], bit) & bit)) a.tlist[atomicAdd(&a.ctl[2], 1)] = t;
        scans += a.g.off[w + 1] - a.g.off[w];
      }
    } else if (wk < nc) {
      const int32_t rn = __ldcg(&a.regn[wk]);
      const bool acc = s_acc[wk] != 0;
      const int32_t nlev = s_wnlev[sub];
      const int32_t* lstart = s_wlstart[sub];
      for (int32_t i = gt; i < rn; i += G) {
        const int32_t w = __ldcg(&my_reg[i]);
        a.vm[my_plane + (w >> 5)] = 0;  // clear (every worker's region is finished)
        if (!acc) continue;
        int32_t lo = 0, hi = nlev - 1;  // depth of entry i: last level starting at or before i
        while (lo < hi) {
          const int32_t mid = (lo + hi + 1) >> 1;
          if (lstart[mid] <= i) lo = mid;
          else hi = mid - 1;
        }
        atomicMin(&a.dist[w], lo);
        const int32_t t = w >> a.tile_shift;
        const uint32_t bit = 1u << (t & 31);
        if (!(atomicOr(&a.tbits[t >> 5], bit) & bit)) a.tlist[atomicAdd(&a.ctl[2], 1)] = t;
        scans += a.g.off[w + 1] - a.g.off[w];
      }
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.work) atomicAdd(&a.work[10], static_cast<unsigned long long>(clock64() - t_c0));
    if (s_done >= a.k) break;
    // ---- refresh the touched tile maxima (distributed), clear the marks
    long long t_r0 = clock64();
    // every walk has read the membership matrix: clear it for the next batch
    for (int32_t q = static_cast<int32_t>(gtid); q < kMaxWorkers * kMaskWords; q += static_cast<int32_t>(gthreads)) a.inm[q] = 0;
    {
      const int64_t gw = gtid >> 5, nwarps = gthreads >> 5;
      const int32_t tsize = 1 << a.tile_shift;
      const int32_t nt = __ldcg(&a.ctl[2]);
      for (int64_t i = gw; i < nt; i += nwarps) {
        const int32_t t = __ldcg(&a.tlist[i]);
        uint64_t best = 0;
        const int32_t lo = t * tsize, hi = min(a.n, lo + tsize);
        // eight 32-vertex subtiles per step, their loads in flight together
        for (int32_t b0 = lo; b0 < hi; b0 += 8 * 32) {
          int32_t dv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int32_t v = b0 + 32 * q + lane;
            dv[q] = v < hi ? __ldcg(&a.dist[v]) : -1;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int32_t v0 = b0 + 32 * q;
            if (v0 >= hi) break;
            if (v0 + lane < hi) best = max(best, vkey(dv[q], v0 + lane));
            const int32_t sm = __reduce_max_sync(0xffffffffu, dv[q]);
            if (lane == 0) a.smax[v0 >> 5] = sm;
          }
        }
        best = warp_max_u64(best);
        if (lane == 0) {
          a.tkey[t] = best;
          a.tbits[t >> 5] = 0;  // every set bit of the word belongs to a listed tile
        }
      }
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.work) atomicAdd(&a.work[11], static_cast<unsigned long long>(clock64() - t_r0));
    // ---- 1. next candidates (leader); grid mode while the radius is large
    if (blockIdx.x == 0) {
      long long t_s0 = clock64();
      // small regions last batch: kMaxSub worker groups per CTA (more candidates)
      const int32_t nsub_next = (!gridmode && __ldcg(&a.ctl[11]) < a.sub_region) ? kMaxSub : 1;
      const int32_t W = min(static_cast<int32_t>(gridDim.x) * nsub_next, kMaxWorkers);
      __syncthreads();
      if (threadIdx.x == 0) a.ctl[0] = s_done, a.ctl[2] = 0, a.ctl[9] = nsub_next, a.ctl[11] = 0;
      select_candidates(a, W, bsm, reinterpret_cast<int32_t*>(bsm + kSCap), shi);
      if (threadIdx.x == 0) {
        const int32_t top = static_cast<int32_t>(__ldcg(&a.ckey[0]) >> 32);
        const bool gm = top > a.grid_radius;
        a.ctl[3] = gm ? 1 : 0;
        if (gm && a.ctl[1] > a.grid_cands) a.ctl[1] = a.grid_cands;
        if (a.work) atomicAdd(&a.work[12], static_cast<unsigned long long>(clock64() - t_s0));
      }
    }
    grid.sync();
  }
  if (a.work) {
    const uint64_t tot = block_sum_i64(static_cast<int64_t>(scans), reinterpret_cast<int64_t*>(s_red));
    if (threadIdx.x == 0 && tot) atomicAdd(&a.work[0], static_cast<unsigned long long>(tot));
  }
}

// Large-radius seeds, one at a time, on one thread-block cluster.  While the
// farthest vertex is farther than grid_radius the candidate list is the single
// argmax (a batch of one is always accepted), so its BFS writes dist directly:
// a claim is atomicMin(dist[w], d + 1) returning a larger value (the region
// R(c) = {v : d(c, v) < dist(v)}, patching.cpp:35-49).  Levels are separated by
// the hardware cluster barrier instead of a grid-wide one.  At the end the
// cluster's CTA 0 selects the first candidate batch for fps_batched_kernel.
constexpr int32_t kBackoffNs = 2048;  // longest idle-poll back-off (64 ns steps)
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(kThreads, 1) fps_cluster_phase(BatchArgs a, int32_t w_main) {
  extern __shared__ uint64_t bsm[];
  __shared__ int32_t shi[32];
  __shared__ uint64_t s_red[32];
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int64_t ctid = static_cast<int64_t>(rank) * blockDim.x + threadIdx.x;
  const int64_t cthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;  // the grid is one cluster
  // Asynchronous label-correcting BFS (no level barriers).  Every lane holds
  // at most one work item (vertex, dist); a warp relaxes its items' neighbours
  // with atomicMin(dist, d + 1), keeps the vertices it lowered as its next items
  // (one per free lane: the front stays with the warp that reached it, so a hop
  // costs an ELL row load and the atomics) and spills the rest to a global
  // queue that idle lanes poll.  The fixed point is the exact BFS distance
  // min'd with the previous dist (relaxations commute): the level-synchronous
  // result.  `pending` counts existing unprocessed items (raised before a new
  // item is published, lowered after an item is done), so pending == 0 means
  // no work is left anywhere.  Each CTA appends the vertices it lowers to its
  // region list for the tile refresh.
  int32_t* const myl = a.reg + static_cast<int64_t>(rank) * a.n;
  __shared__ int32_t s_len;
  unsigned long long scans = 0, levels = 0;
  const int32_t tsize = 1 << a.tile_shift;
  uint64_t* q = reinterpret_cast<uint64_t*>(a.queue);  // items dist << 32 | vertex, ~0 = empty
  int32_t* qc = a.qctl;  // head, tail, pending: one 128-byte line each (no shared hot spot)
  const int64_t qcap = a.qcap;
  const int wid = threadIdx.x >> 5;
  uint64_t* stage = bsm + 256 * wid;  // per warp: this step's lowered (dist, vertex) (dynamic smem)

  for (int64_t v = ctid; v < a.n; v += cthreads) a.dist[v] = kUnreached;
  if (ctid == 0) a.ctl[2] = 0, a.ctl[12] = 0;  // touched tiles, overflow
  cluster_barrier();
  int32_t c = static_cast<int32_t>(splitmix64(a.seed) % static_cast<uint64_t>(a.n));  // patching.cpp:32
  int32_t done = 0;
  for (;;) {
    if (threadIdx.x == 0) s_len = 0;
    if (ctid == 0) {
      const int32_t t = *reinterpret_cast<volatile int32_t*>(&qc[kQTail]);
      a.seeds[done] = c;
      a.dist[c] = 0;
      myl[0] = c;
      s_len = 1;
      q[t] = static_cast<uint32_t>(c);  // dist 0
      qc[kQHead] = t, qc[kQTail] = t + 1, qc[kQPend] = 1;
    }
    ++done;
    cluster_barrier();
    int64_t my_slot = -1;  // this lane's reserved queue slot (kept until its item arrives)
    int32_t u = -1, du = 0;  // this lane's item
    for (int idle = 0;;) {
      // Lanes holding a queue reservation poll it; the load is issued here and
      // consumed after this step's relaxations (a working warp does not wait
      // for it).  Only a warp without any item reserves new slots, so a
      // working warp keeps the vertices it lowers in its own lanes (its front
      // grows locally; the excess is spilled) and its step is one ELL row
      // load plus the atomicMin round trip -- no queue round trips.
      uint64_t pv = ~0ull;
      if (u < 0 && my_slot >= 0) pv = *reinterpret_cast<volatile uint64_t*>(&q[my_slot]);
      bool have = u >= 0;
      if (!__any_sync(0xffffffffu, have)) {
        if (pv != ~0ull) u = static_cast<int32_t>(static_cast<uint32_t>(pv)), du = static_cast<int32_t>(pv >> 32), my_slot = -1;
        pv = ~0ull;
        const uint32_t needy = __ballot_sync(0xffffffffu, u < 0 && my_slot < 0);
        if (needy) {
          int32_t h0 = 0;
          if (lane == 0) h0 = atomicAdd(&qc[kQHead], __popc(needy));
          h0 = __shfl_sync(0xffffffffu, h0, 0);
          if (u < 0 && my_slot < 0) my_slot = static_cast<int64_t>(h0) + __popc(needy & ((1u << lane) - 1));
        }
        if (__any_sync(0xffffffffu, my_slot >= qcap)) {
          if (lane == 0) atomicExch(&a.ctl[12], 1), atomicExch(&qc[kQPend], 0);  // abort: the main kernel redoes FPS
          break;
        }
        have = u >= 0;
        if (!__any_sync(0xffffffffu, have)) {
          int32_t pend = lane == 0 ? *reinterpret_cast<volatile int32_t*>(&qc[kQPend]) : 0;
          pend = __shfl_sync(0xffffffffu, pend, 0);  // one verdict per warp
          if (pend == 0) break;                       // no work anywhere: region complete
          if (++idle > (1 << 22)) {                   // watchdog (never expected): fall back
            if (lane == 0) atomicExch(&a.ctl[12], 1), atomicExch(&qc[kQPend], 0);
            break;
          }
          if (idle > 2) __nanosleep(min(64 * idle, kBackoffNs));  // back off: idle polls must not starve the atomics
          continue;
        }
      }
      idle = 0;
      // relax the items' neighbours (the lowered ones as a slot mask: the
      // candidates stay in registers, no local-memory array)
      uint32_t lmask = 0;
      int32_t cand[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) cand[k] = -1;
      const uint64_t hi = static_cast<uint64_t>(du + 1) << 32;
      if (have) {
        const int32_t nd = du + 1;
        const int4* row = reinterpret_cast<const int4*>(a.ell + static_cast<int64_t>(u) * 8);
        const int4 r0 = row[0], r1 = row[1];
        cand[0] = r0.x, cand[1] = r0.y, cand[2] = r0.z, cand[3] = r0.w;
        cand[4] = r1.x, cand[5] = r1.y, cand[6] = r1.z, cand[7] = r1.w;
        int32_t old[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) old[k] = cand[k] >= 0 ? atomicMin(&a.dist[cand[k]], nd) : 0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (cand[k] >= 0 && old[k] > nd) lmask |= 1u << k;
        scans += a.g.off[u + 1] - a.g.off[u];
        if (cand[7] < -1)  // CSR tail of a vertex with more than 8 neighbours: straight to the queue
          for (int32_t j = -cand[7] - 2; j < a.g.off[u + 1]; ++j) {
            const int32_t w = a.g.nbr[j];
            if (atomicMin(&a.dist[w], nd) > nd) {
              atomicAdd(&qc[kQPend], 1);
              const int32_t t = atomicAdd(&qc[kQTail], 1);
              if (t < qcap) q[t] = hi | static_cast<uint32_t>(w);
              else atomicExch(&a.ctl[12], 1);
              const int32_t li = atomicAdd(&s_len, 1);
              if (li < a.n) myl[li] = w;
              else atomicExch(&a.ctl[12], 1);
            }
          }
      }
      // stage the lowered vertices warp-wide
      const int32_t np = __popc(lmask);
      int32_t inc = np;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int32_t tot = __shfl_sync(0xffffffffu, inc, 31);
      const int32_t nproc = __popc(__ballot_sync(0xffffffffu, have));
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if ((lmask >> k) & 1u) stage[inc - np + __popc(lmask & ((1u << k) - 1))] = hi | static_cast<uint32_t>(cand[k]);
      u = -1;
      // lanes without a reservation take the first items; the rest is spilled
      const uint32_t freel = __ballot_sync(0xffffffffu, my_slot < 0);
      const int32_t nfree = __popc(freel);
      const int32_t keep = min(tot, nfree), spill = tot - keep;
      int32_t base = 0, lbase = 0;
      if (lane == 0 && tot) {
        atomicAdd(&qc[kQPend], tot);  // before any of them can be retired
        if (spill) base = atomicAdd(&qc[kQTail], spill);
        lbase = atomicAdd(&s_len, tot);
      }
      base = __shfl_sync(0xffffffffu, base, 0);
      lbase = __shfl_sync(0xffffffffu, lbase, 0);
      __syncwarp();
      if (my_slot < 0) {
        const int32_t r = __popc(freel & ((1u << lane) - 1));
        if (r < keep) {
          const uint64_t it = stage[r];
          u = static_cast<int32_t>(static_cast<uint32_t>(it)), du = static_cast<int32_t>(it >> 32);
        }
      }
      for (int32_t i = lane; i < tot; i += 32) {
        const uint64_t it = stage[i];
        if (lbase + i < a.n) myl[lbase + i] = static_cast<int32_t>(static_cast<uint32_t>(it));
        else atomicExch(&a.ctl[12], 1);
        if (i >= keep) {
          const int64_t t = static_cast<int64_t>(base) + (i - keep);
          if (t < qcap) q[t] = it;
          else atomicExch(&a.ctl[12], 1);
        }
      }
      // a reserved slot that was filled: its item is this lane's next one
      if (pv != ~0ull) u = static_cast<int32_t>(static_cast<uint32_t>(pv)), du = static_cast<int32_t>(pv >> 32), my_slot = -1;
      // (same-address atomics of one thread are ordered: the increment above
      //  lands before this decrement, so pending never reads 0 early)
      if (lane == 0 && nproc) atomicSub(&qc[kQPend], nproc);
      __syncwarp();
      ++levels;
    }
    cluster_barrier();
    if (__ldcg(&a.ctl[12])) break;  // queue or list overflow: fps_batched_kernel starts over
    // mark the tiles of this CTA's region vertices
    for (int32_t i = threadIdx.x; i < min(s_len, a.n); i += blockDim.x) {
      const int32_t w = myl[i];
      const int32_t t = w >> a.tile_shift;
      const uint32_t bit = 1u << (t & 31);
      if (!(atomicOr(&a.tbits[t >> 5], bit) & bit)) a.tlist[atomicAdd(&a.ctl[2], 1)] = t;
    }
    cluster_barrier();
    // refresh the touched tile and subtile maxima
    {
      const int64_t gw = ctid >> 5, nwarps = cthreads >> 5;
      const int32_t nt = __ldcg(&a.ctl[2]);
      for (int64_t i = gw; i < nt; i += nwarps) {
        const int32_t t = __ldcg(&a.tlist[i]);
        uint64_t best = 0;
        const int32_t lo = t * tsize, hi = min(a.n, lo + tsize);
        // eight 32-vertex subtiles per step, their loads in flight together
        for (int32_t b0 = lo; b0 < hi; b0 += 8 * 32) {
          int32_t dv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int32_t v = b0 + 32 * q + lane;
            dv[q] = v < hi ? __ldcg(&a.dist[v]) : -1;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int32_t v0 = b0 + 32 * q;
            if (v0 >= hi) break;
            if (v0 + lane < hi) best = max(best, vkey(dv[q], v0 + lane));
            const int32_t sm = __reduce_max_sync(0xffffffffu, dv[q]);
            if (lane == 0) a.smax[v0 >> 5] = sm;
          }
        }
        best = warp_max_u64(best);
        if (lane == 0) {
          a.tkey[t] = best;
          a.tbits[t >> 5] = 0;
        }
      }
    }
    cluster_barrier();
    if (done >= a.k) break;
    // the next seed: argmax (dist desc, id asc) over the tile maxima (every CTA)
    uint64_t best = 0;
    for (int32_t t0 = threadIdx.x; t0 < a.ntile; t0 += 8 * blockDim.x) {
      uint64_t v[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const int32_t t = t0 + g * static_cast<int32_t>(blockDim.x);
        v[g] = t < a.ntile ? __ldcg(&a.tkey[t]) : 0;
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) best = max(best, v[g]);
    }
    best = block_max_u64(best, s_red);
    if (static_cast<int32_t>(best >> 32) <= a.grid_radius) break;
    c = static_cast<int32_t>(key_max_id(best));
    if (ctid == 0) a.ctl[2] = 0;  // every CTA has read the touched count (refresh, barrier above)
    cluster_barrier();
  }
  // hand over: seeds done, no touched tiles, the first candidate batch
  if (rank == 0) {
    if (threadIdx.x == 0) {
      a.ctl[0] = done, a.ctl[2] = 0, a.ctl[3] = 0, a.ctl[9] = 1, a.ctl[10] = 0, a.ctl[11] = 0;
      if (a.work) {
        atomicAdd(&a.work[4], static_cast<unsigned long long>(done));
        atomicAdd(&a.work[5], levels);
      }
    }
    __syncthreads();
    if (done < a.k && !__ldcg(&a.ctl[12])) select_candidates(a, w_main, bsm, reinterpret_cast<int32_t*>(bsm + kSCap), shi);
  }
  if (a.work) {
    const uint64_t tot = block_sum_i64(static_cast<int64_t>(scans), reinterpret_cast<int64_t*>(s_red));
    if (threadIdx.x == 0 && tot) atomicAdd(&a.work[0], static_cast<unsigned long long>(tot));
  }
}

}  // namespace

// Seeds of one component spanning the whole graph (positions = vertex ids).
void fps_batched_dev(mp_context& ctx, const DGraph& g, const int32_t* ell, int32_t k, uint64_t seed, int32_t* seeds,
                     int32_t* dist) {
  // worker-mode regions are shallower than the grid radius (their depth is
  // below the candidate's distance): kMaxDepth bounds the per-level offsets
  const int64_t gr = ctx.tune[MP_TUNE_FPS_GRID_RADIUS], gc = ctx.tune[MP_TUNE_FPS_GRID_CANDS];
  const int32_t grid_radius = static_cast<int32_t>(std::min<int64_t>(gr > 0 ? gr : 200, kMaxDepth));
  const int32_t grid_cands = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(gc > 0 ? gc : 1, kGridCands)));
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  int tile_shift = 8;
  while ((static_cast<int64_t>(n) + (1 << tile_shift) - 1) >> tile_shift > 65536) ++tile_shift;
  const int32_t ntile = static_cast<int32_t>((static_cast<int64_t>(n) + (1 << tile_shift) - 1) >> tile_shift);
  int bpsm = 0;
  // candidate selection (kSCap keys + kBins histogram) or the walk's staging
  // (keys, region maxima, in-region masks of kMaxWorkers candidates)
  const size_t smem = std::max(sizeof(uint64_t) * kSCap + sizeof(int32_t) * kBins,
                               sizeof(uint64_t) * 2 * kMaxWorkers + sizeof(uint32_t) * kMaxWorkers * kMaskWords);
  allow_max_smem(fps_batched_kernel, ctx.device);
  MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, fps_batched_kernel, kThreads, smem));
  if (bpsm < 1) throw Error(MP_ECUDA, "fps_batched_kernel does not fit on an SM");
  // workers: one per SM, bounded by the bit-matrix width and by memory
  // (a 4-byte region list per vertex each); decided once per context
  if (ctx.fps_workers == 0) {
    int W0 = std::min(std::max(ctx.num_sms / std::max(ctx.sm_share, 1), 4), kMaxWorkers);
    size_t free_b = 0, total_b = 0;
    MP_CUDA(cudaMemGetInfo(&free_b, &total_b));
    while (W0 > 1 && 4ull * n * W0 > free_b / 2) W0 /= 2;
    ctx.fps_workers = W0;
  }
  const int W = ctx.fps_workers;
  const int64_t wn = static_cast<int64_t>(W) * n;
  // visit bits: 32 bytes per vertex, shared by all regions (L2-resident at 1M)
  const int64_t vwords = (static_cast<int64_t>(n) + 31) / 32;  // one bit plane of n bits per worker
  uint32_t* vm = static_cast<uint32_t*>(ctx.slab(0, sizeof(uint32_t) * kMaxWorkers * vwords));
  int32_t* dw = static_cast<int32_t*>(ctx.slab(1, sizeof(int32_t) * static_cast<int64_t>(grid_cands) * n));
  // region lists: one row of n per worker CTA, and per cluster CTA of fps_cluster_phase (up to 16)
  int32_t* reg = static_cast<int32_t*>(ctx.slab(2, sizeof(int32_t) * std::max<int64_t>(W, 16) * n));
  uint64_t* glist = static_cast<uint64_t*>(ctx.slab(3, sizeof(uint64_t) * (static_cast<int64_t>(grid_cands) * n + 64)));
  DevBuf<int32_t> tlist(ntile, s), cand(kSCap, s), regn(kMaxWorkers, s), ctl(16, s);
  DevBuf<uint64_t> tkey(ntile, s), ckey(kSCap, s), mkey(kMaxWorkers, s);
  DevBuf<uint32_t> tbits(ntile / 32 + 1, s), inm(kMaxWorkers * kMaskWords, s);
  DevBuf<int32_t> tscratch(ntile, s), bar(1, s), smax(n / 32 + 1, s);
  MP_CUDA(cudaMemsetAsync(bar, 0, sizeof(int32_t), s));
  MP_CUDA(cudaMemsetAsync(inm, 0, sizeof(uint32_t) * inm.n, s));
  MP_CUDA(cudaMemsetAsync(vm, 0, sizeof(uint32_t) * kMaxWorkers * vwords, s));
  MP_CUDA(cudaMemsetAsync(tbits, 0, sizeof(uint32_t) * tbits.n, s));
  BatchArgs a{};
  a.g = g, a.ell = ell, a.n = n, a.k = k, a.tile_shift = tile_shift, a.ntile = ntile, a.seed = seed;
  a.dist = dist, a.tkey = tkey, a.tbits = tbits, a.tlist = tlist, a.vm = vm, a.vwords = vwords, a.dw = dw, a.reg = reg;
  a.cand = cand, a.ckey = ckey, a.mkey = mkey, a.inm = inm, a.regn = regn, a.ctl = ctl, a.seeds = seeds;
  a.work = ctx.dwork;
  a.glist = glist;
  a.tscratch = tscratch;
  a.smax = smax;
  a.bar = reinterpret_cast<unsigned int*>(bar.get());
  a.grid_radius = grid_radius;
  a.grid_cands = grid_cands;
  a.sub_region = ctx.tune[MP_TUNE_FPS_SUB_REGION] > 0 ? static_cast<int32_t>(ctx.tune[MP_TUNE_FPS_SUB_REGION]) : kSubRegion;
  const int kt = ctx.ktime_begin(kKFps);
  // large-radius seeds on one cluster (16 CTAs where the device allows, else 8)
  a.resume = 0;
  // the cluster kernel's dynamic smem: the select scratch, or 256 staged items per warp
  const size_t cl_smem = std::max(smem, sizeof(uint64_t) * 256 * (kThreads / 32));
  a.qcap = 8LL * n + 1024;  // uint64 items
  if (ctx.tune[MP_TUNE_FPS_QCAP] > 0) a.qcap = std::max<int64_t>(64, std::min<int64_t>(a.qcap, ctx.tune[MP_TUNE_FPS_QCAP]));
  a.queue = static_cast<int32_t*>(ctx.slab(4, sizeof(uint64_t) * a.qcap));
  DevBuf<int32_t> qctl(96, s);
  a.qctl = qctl;
  MP_CUDA(cudaMemsetAsync(a.queue, 0xff, sizeof(uint64_t) * a.qcap, s));
  MP_CUDA(cudaMemsetAsync(qctl, 0, sizeof(int32_t) * 96, s));
  if (ctx.tune[MP_TUNE_FPS_CLUSTER] >= 0) {
    // cluster size: 16 CTAs (non-portable) where the device allows, else 8;
    // probed once per device (MP_TUNE_FPS_CLUSTER overrides and is re-probed).
    // The function attributes are per device too, so they are set for every
    // device this process launches on, not only the first one probed.
    static std::mutex mu;
    static std::map<int, int> cached;  // device -> cluster CTAs (0: no cluster launch)
    const bool ce = ctx.tune[MP_TUNE_FPS_CLUSTER] > 0;
    int cluster_ctas = 0;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = cached.find(ctx.device);
      if (ce || it == cached.end()) {
        allow_max_smem(fps_cluster_phase, ctx.device);
        const bool nonportable =
            cudaFuncSetAttribute(fps_cluster_phase, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
        cudaGetLastError();
        const int first = ce ? static_cast<int>(ctx.tune[MP_TUNE_FPS_CLUSTER]) : 16;
        for (int cs : {first, 16, 8}) {
          if (cs < 1 || cs > 16 || (cs > 8 && !nonportable)) continue;
          cudaLaunchConfig_t cfg{};
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cs, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
          cfg.gridDim = dim3(cs), cfg.blockDim = dim3(kThreads), cfg.dynamicSmemBytes = cl_smem;
          cfg.attrs = at, cfg.numAttrs = 1;
          int ncl = 0;
          if (cudaOccupancyMaxActiveClusters(&ncl, fps_cluster_phase, &cfg) == cudaSuccess && ncl > 0) {
            cluster_ctas = cs;
            break;
          }
          cudaGetLastError();
        }
        if (!ce) cached[ctx.device] = cluster_ctas;
      } else {
        cluster_ctas = it->second;
      }
    }
    if (cluster_ctas > 0) {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cluster_ctas, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cluster_ctas), cfg.blockDim = dim3(kThreads), cfg.dynamicSmemBytes = cl_smem;
      cfg.stream = s, cfg.attrs = at, cfg.numAttrs = 1;
      MP_KERNEL(ctx, MP_CUDA(cudaLaunchKernelEx(&cfg, fps_cluster_phase, a, static_cast<int32_t>(W))));
      a.resume = 1;
    }
  }
  void* args[] = {&a};
  MP_KERNEL(ctx, MP_CUDA(cudaLaunchCooperativeKernel((void*)fps_batched_kernel, W, kThreads, args, smem, s)));
  ctx.ktime_end(kt);
}

}  // namespace mp
