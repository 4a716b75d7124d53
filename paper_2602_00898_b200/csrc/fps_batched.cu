// Farthest-point seeding, exact speculative batches (reference
// core/src/patching.cpp:26-65), for one large connected component.
//
// The reference picks seeds one at a time: argmax over the component of the
// packed key (dist desc, id asc), then relaxes dist from the new seed.  A
// relaxation from c only lowers dist inside R(c) = {v : d(c,v) < dist(v)},
// and min() makes relaxations commute.  A batch therefore:
//   1. takes a candidate list S, sorted by key desc, that is downward closed
//      (every vertex with key >= min key(S) is in S): all vertices of the
//      top-B tiles of the tile-max tree with key >= the B-th largest tile max;
//   2. computes R(c_j) and d(c_j, .) for the first W candidates in parallel,
//      one worker CTA each, against the committed dist;
//   3. walks S in order: a candidate inside an accepted region is skipped (its
//      key fell to <= M, the largest key any accepted region can leave); the
//      first candidate outside the accepted regions whose key beats M is the
//      true next seed; a candidate whose key does not beat M ends the batch;
//   4. commits min(dist, d(c_j, .)) over the accepted regions and refreshes
//      the touched tiles.
// The accepted sequence is exactly the sequential FPS sequence.  The first
// seeds (regions spanning most of the mesh) are relaxed by the whole grid,
// level-synchronously.
#include <cub/cub.cuh>

#include <algorithm>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kThreads = 1024;
constexpr int kMaxTiles = 8192;   // tile-key sort in shared memory
constexpr int kSCap = 4096;       // candidate list capacity
constexpr int kFront = 4096;      // smem frontier per buffer in a worker
constexpr int kMaxWorkers = 256;  // candidates per batch (bit-matrix width)
constexpr int kMaskWords = kMaxWorkers / 32;
constexpr int kGridSeeds = 6;     // seeds relaxed by the whole grid

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {  // patching.cpp:17-22
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d649bb133111ebULL;
  return x ^ (x >> 31);
}

struct BatchArgs {
  DGraph g;
  const int32_t* ell;      // n * 8 ELL adjacency (slot 7 < -1 encodes a CSR tail)
  int32_t n, k, tile_shift, ntile, nsuper;
  uint64_t seed;
  int32_t* dist;
  uint64_t* tkey;          // ntile
  uint64_t* skey;          // nsuper (256 tiles each)
  uint32_t* tbits;         // touched tiles
  int32_t* tlist;          // ntile
  uint32_t* sbits;         // touched supertiles
  int32_t* slist;          // nsuper
  int32_t* fa;             // grid-mode frontiers (n each)
  int32_t* fb;
  int32_t* vis;            // W * n private visit tokens
  int32_t* dw;             // W * n private distances
  int32_t* reg;            // W * n region lists
  int32_t* cand;           // kSCap
  uint64_t* ckey;          // kSCap
  uint64_t* mkey;          // kMaxWorkers: largest key a region leaves
  uint32_t* inm;           // kMaxWorkers * kMaskWords membership bits
  int32_t* regn;           // kMaxWorkers region sizes
  int32_t* acc;            // kMaxWorkers accepted flags
  int32_t* ctl;            // [0] seeds done [1] ncand [2] tcount [3] scount [4..6] frontier counters [7] cur
  int32_t* seeds;          // output, k
  unsigned long long* work;
};

__device__ __forceinline__ uint64_t vkey(int32_t d, int32_t v) {
  return key_max(static_cast<uint32_t>(d), static_cast<uint32_t>(v));
}

__device__ void mark_tile(const BatchArgs& a, int32_t v) {
  const int32_t t = v >> a.tile_shift;
  const uint32_t bit = 1u << (t & 31);
  if (!(atomicOr(&a.tbits[t >> 5], bit) & bit)) a.tlist[atomicAdd(&a.ctl[2], 1)] = t;
}

// Distributed refresh of the touched tiles, then of the touched supertiles.
__device__ void refresh(cg::grid_group& grid, const BatchArgs& a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int32_t tsize = 1 << a.tile_shift;
  const int32_t nt = __ldcg(&a.ctl[2]);
  for (int64_t i = gw; i < nt; i += nwarps) {
    const int32_t t = __ldcg(&a.tlist[i]);
    uint64_t best = 0;
    const int32_t lo = t * tsize, hi = min(a.n, lo + tsize);
    for (int32_t v = lo + lane; v < hi; v += 32) best = max(best, vkey(__ldcg(&a.dist[v]), v));
    best = warp_max_u64(best);
    if (lane == 0) {
      a.tkey[t] = best;
      a.tbits[t >> 5] = 0;  // whole word: every bit of the word belongs to listed tiles
      const int32_t su = t >> 8;
      const uint32_t bit = 1u << (su & 31);
      if (!(atomicOr(&a.sbits[su >> 5], bit) & bit)) a.slist[atomicAdd(&a.ctl[3], 1)] = su;
    }
  }
  grid.sync();
  const int32_t ns = __ldcg(&a.ctl[3]);
  for (int64_t i = gw; i < ns; i += nwarps) {
    const int32_t su = __ldcg(&a.slist[i]);
    uint64_t best = 0;
    const int32_t lo = su << 8, hi = min(a.ntile, lo + 256);
    for (int32_t t = lo + lane; t < hi; t += 32) best = max(best, __ldcg(&a.tkey[t]));
    best = warp_max_u64(best);
    if (lane == 0) {
      a.skey[su] = best;
      a.sbits[su >> 5] = 0;
    }
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl[2] = 0, a.ctl[3] = 0;
}

// Block-wide bitonic sort (descending) of m = power-of-two keys in smem.
__device__ void bitonic_desc(uint64_t* s, int32_t m) {
  for (int32_t size = 2; size <= m; size <<= 1) {
    for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (int32_t t = threadIdx.x; t < m / 2; t += blockDim.x) {
        const int32_t i = 2 * t - (t & (stride - 1));
        const int32_t j = i + stride;
        const bool up = (i & size) == 0;  // descending run
        const uint64_t x = s[i], y = s[j];
        if ((x < y) == up) s[i] = y, s[j] = x;
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kThreads) fps_batched_kernel(BatchArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint64_t bsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  __shared__ int32_t s_cnt[3], s_n;
  __shared__ uint64_t s_red[32];
  __shared__ uint32_t s_mask[kMaskWords];
  unsigned long long scans = 0;

  for (int64_t v = gtid; v < a.n; v += gthreads) a.dist[v] = kUnreached;
  if (gtid == 0) {
    a.ctl[0] = 0, a.ctl[2] = 0, a.ctl[3] = 0;
    a.ctl[7] = static_cast<int32_t>(splitmix64(a.seed) % static_cast<uint64_t>(a.n));
  }
  grid.sync();

  // ---------------- phase 0: the first seeds, relaxed by the whole grid
  const int32_t k0 = min(a.k, kGridSeeds);
  for (int32_t s = 0; s < k0; ++s) {
    const int32_t cur = __ldcg(&a.ctl[7]);
    if (gtid == 0) {
      a.seeds[s] = cur;
      a.dist[cur] = 0;
      a.fa[0] = cur;
      a.ctl[4] = 1, a.ctl[5] = 0, a.ctl[6] = 0;
      mark_tile(a, cur);
    }
    grid.sync();
    int32_t* front = a.fa;
    int32_t* next = a.fb;
    for (int32_t d = 0;; ++d) {
      const int32_t nf = __ldcg(&a.ctl[4 + d % 3]);
      if (nf == 0) break;
      if (gtid == 0) a.ctl[4 + (d + 2) % 3] = 0;
      int32_t* cout = &a.ctl[4 + (d + 1) % 3];
      const int64_t items = static_cast<int64_t>(nf) * 8;
      for (int64_t it = gtid; it < items; it += gthreads) {
        const int32_t u = __ldcg(&front[it >> 3]);
        const int32_t x = a.ell[static_cast<int64_t>(u) * 8 + (it & 7)];
        auto relax = [&](int32_t w) {
          ++scans;
          if (d + 1 < __ldcg(&a.dist[w]) && atomicMin(&a.dist[w], d + 1) > d + 1) {
            next[atomicAdd(cout, 1)] = w;
            mark_tile(a, w);
          }
        };
        if (x >= 0) relax(x);
        else if (x < -1)
          for (int32_t j = -x - 2; j < a.g.off[u + 1]; ++j) relax(a.g.nbr[j]);
      }
      grid.sync();
      int32_t* t = front;
      front = next;
      next = t;
    }
    refresh(grid, a);
    if (blockIdx.x == 0) {  // argmax (patching.cpp:52-60)
      uint64_t best = 0;
      for (int32_t i = threadIdx.x; i < a.nsuper; i += blockDim.x) best = max(best, __ldcg(&a.skey[i]));
      best = block_max_u64(best, s_red);
      if (threadIdx.x == 0) {
        a.ctl[7] = static_cast<int32_t>(key_max_id(best));
        a.ctl[0] = s + 1;
      }
    }
    grid.sync();
  }

  // ---------------- phase 1: speculative batches
  const int32_t W = min(static_cast<int32_t>(gridDim.x), kMaxWorkers);
  int32_t* my_vis = a.vis + static_cast<int64_t>(blockIdx.x) * a.n;
  int32_t* my_dw = a.dw + static_cast<int64_t>(blockIdx.x) * a.n;
  int32_t* my_reg = a.reg + static_cast<int64_t>(blockIdx.x) * a.n;
  for (int32_t batch = 0;; ++batch) {
    if (__ldcg(&a.ctl[0]) >= a.k) break;
    // 1. candidates (leader CTA)
    if (blockIdx.x == 0) {
      uint64_t* sk = bsm;                 // tile keys, sorted
      uint64_t* sS = bsm + kMaxTiles;     // candidate keys
      int32_t m = 1;
      while (m < a.ntile) m <<= 1;
      for (int32_t t = threadIdx.x; t < m; t += blockDim.x) sk[t] = t < a.ntile ? __ldcg(&a.tkey[t]) : 0;
      __syncthreads();
      bitonic_desc(sk, m);
      int32_t B = min(W, a.ntile);
      for (;;) {
        const uint64_t K = sk[B - 1];
        if (threadIdx.x == 0) s_n = 0;
        __syncthreads();
        const int32_t tsize = 1 << a.tile_shift;
        for (int32_t i = wid; i < B; i += nwarp) {
          const int32_t t = static_cast<int32_t>(key_max_id(sk[i])) >> a.tile_shift;
          const int32_t lo = t * tsize, hi = min(a.n, lo + tsize);
          for (int32_t v = lo + lane; v < hi; v += 32) {
            const uint64_t kv = vkey(__ldcg(&a.dist[v]), v);
            if (kv >= K) {
              const int32_t slot = atomicAdd(&s_n, 1);
              if (slot < kSCap) sS[slot] = kv;
            }
          }
        }
        __syncthreads();
        if (s_n <= kSCap || B == 1) break;
        B = max(1, B / 2);
        __syncthreads();
      }
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
      if (threadIdx.x == 0) a.ctl[1] = nc;
    }
    grid.sync();
    // 2. regions, one worker CTA per candidate
    const int32_t nc = __ldcg(&a.ctl[1]);
    const int32_t token = batch + 1;
    if (static_cast<int32_t>(blockIdx.x) < nc) {
      const int32_t c = __ldcg(&a.cand[blockIdx.x]);
      int32_t* sf0 = reinterpret_cast<int32_t*>(bsm);
      int32_t* sf1 = sf0 + kFront;
      if (threadIdx.x == 0) {
        my_vis[c] = token;
        my_dw[c] = 0;
        my_reg[0] = c;
        sf0[0] = c;
        s_cnt[0] = 1, s_cnt[1] = 0, s_cnt[2] = 0;
        s_n = 1;  // region size
      }
      __syncthreads();
      uint64_t mk = vkey(0, c);
      for (int32_t d = 0;; ++d) {
        const int32_t nf = s_cnt[d % 3];
        if (nf == 0) break;
        if (threadIdx.x == 0) s_cnt[(d + 2) % 3] = 0;
        const int32_t* fin = (d & 1) ? sf1 : sf0;
        int32_t* fout = (d & 1) ? sf0 : sf1;
        const int32_t rbase = s_n - nf;  // this level's vertices sit at the end of the region list
        int32_t* cout = &s_cnt[(d + 1) % 3];
        const int32_t items = nf * 8;
        for (int32_t it = threadIdx.x; it < items; it += blockDim.x) {
          const int32_t i = it >> 3;
          const int32_t u = i < kFront ? fin[i] : __ldcg(&my_reg[rbase + i]);
          const int32_t x = a.ell[static_cast<int64_t>(u) * 8 + (it & 7)];
          auto relax = [&](int32_t w) {
            if (d + 1 < __ldcg(&a.dist[w]) && atomicExch(&my_vis[w], token) != token) {
              my_dw[w] = d + 1;
              const int32_t slot = atomicAdd(cout, 1);
              if (slot < kFront) fout[slot] = w;
              my_reg[s_n + slot] = w;
              mk = max(mk, vkey(d + 1, w));
            }
          };
          if (x >= 0) relax(x);
          else if (x < -1)
            for (int32_t j = -x - 2; j < a.g.off[u + 1]; ++j) relax(a.g.nbr[j]);
        }
        __syncthreads();
        if (threadIdx.x == 0) s_n += *cout;
        __syncthreads();
      }
      mk = block_max_u64(mk, s_red);
      // membership of the other candidates in this region
      for (int32_t j = threadIdx.x; j < kMaxWorkers; j += blockDim.x) {
        const bool in = j < nc && __ldcg(&my_vis[__ldcg(&a.cand[j])]) == token;
        const uint32_t bits = __ballot_sync(0xffffffffu, in);
        if (lane == 0) a.inm[blockIdx.x * kMaskWords + (j >> 5)] = bits;
      }
      if (threadIdx.x == 0) {
        a.mkey[blockIdx.x] = mk;
        a.regn[blockIdx.x] = s_n;
      }
    }
    grid.sync();
    // 3. the walk (leader): exact sequential argmax semantics
    if (blockIdx.x == 0) {
      if (wid == 0) {
        uint32_t U = 0;  // lane w holds bits [32w, 32w+32) of the accepted-region union
        uint64_t Mx = 0;
        int32_t done = __ldcg(&a.ctl[0]);
        for (int32_t j = 0; j < nc; ++j) {
          const uint32_t uw = __shfl_sync(0xffffffffu, U, j >> 5);
          int32_t accept = 0;
          if (!((uw >> (j & 31)) & 1u)) {
            if (done < a.k && __ldcg(&a.ckey[j]) > Mx) accept = 1;
            else accept = -1;  // stop
          }
          if (accept < 0) break;
          if (lane == 0) a.acc[j] = accept;
          if (accept) {
            if (lane < kMaskWords) U |= __ldcg(&a.inm[j * kMaskWords + lane]);
            Mx = max(Mx, __ldcg(&a.mkey[j]));
            if (lane == 0) a.seeds[done] = __ldcg(&a.cand[j]);
            ++done;
          }
        }
        if (lane == 0) a.ctl[0] = done;
      }
    }
    // candidates after the stop point are rejected
    grid.sync();
    // 4. commit the accepted regions
    if (static_cast<int32_t>(blockIdx.x) < nc) {
      const int32_t j = blockIdx.x;
      if (__ldcg(&a.acc[j]) == 1) {
        const int32_t rn = __ldcg(&a.regn[j]);
        for (int32_t i = threadIdx.x; i < rn; i += blockDim.x) {
          const int32_t w = __ldcg(&my_reg[i]);
          atomicMin(&a.dist[w], __ldcg(&my_dw[w]));
          mark_tile(a, w);
          scans += a.g.off[w + 1] - a.g.off[w];
        }
      }
    }
    grid.sync();
    // reset the acceptance flags of this batch
    for (int32_t j = static_cast<int32_t>(gtid); j < nc; j += static_cast<int32_t>(gthreads)) a.acc[j] = 0;
    refresh(grid, a);
  }
  if (a.work) {
    const uint64_t tot = block_sum_i64(static_cast<int64_t>(scans), reinterpret_cast<int64_t*>(s_red));
    if (threadIdx.x == 0 && tot) atomicAdd(&a.work[0], static_cast<unsigned long long>(tot));
  }
}

}  // namespace

__global__ void build_ell_batched(DGraph g, int32_t* ell) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
    const int32_t o = g.off[v], deg = g.off[v + 1] - o;
    int32_t* e = ell + static_cast<int64_t>(v) * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) e[k] = k < deg ? g.nbr[o + k] : -1;
    if (deg > 8) e[7] = -(o + 7) - 2;
  }
}

// Seeds of one component spanning the whole graph (positions = vertex ids).
void fps_batched_dev(mp_context& ctx, const DGraph& g, int32_t k, uint64_t seed, int32_t* seeds, int32_t* dist) {
  cudaStream_t s = ctx.stream;
  const int32_t n = g.n;
  int tile_shift = 8;
  while ((static_cast<int64_t>(n) + (1 << tile_shift) - 1) >> tile_shift > kMaxTiles) ++tile_shift;
  const int32_t ntile = static_cast<int32_t>((static_cast<int64_t>(n) + (1 << tile_shift) - 1) >> tile_shift);
  const int32_t nsuper = (ntile + 255) / 256;
  int bpsm = 0;
  const size_t smem = sizeof(uint64_t) * (kMaxTiles + kSCap);
  MP_CUDA(cudaFuncSetAttribute(fps_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, fps_batched_kernel, kThreads, smem));
  if (bpsm < 1) throw Error(MP_ECUDA, "fps_batched_kernel does not fit on an SM");
  // workers: one per SM, bounded by the bit-matrix width and by memory (12 bytes/vertex each)
  int W = std::min(ctx.num_sms, kMaxWorkers);
  size_t free_b = 0, total_b = 0;
  MP_CUDA(cudaMemGetInfo(&free_b, &total_b));
  while (W > 1 && 12ull * n * W > free_b / 2) W /= 2;
  DevBuf<int32_t> ell(8LL * n, s), fa(n, s), fb(n, s), vis(static_cast<int64_t>(W) * n, s),
      dw(static_cast<int64_t>(W) * n, s), reg(static_cast<int64_t>(W) * n, s), tlist(ntile, s), slist(nsuper, s),
      cand(kSCap, s), regn(kMaxWorkers, s), acc(kMaxWorkers, s), ctl(8, s);
  DevBuf<uint64_t> tkey(ntile, s), skey(nsuper, s), ckey(kSCap, s), mkey(kMaxWorkers, s);
  DevBuf<uint32_t> tbits(ntile / 32 + 1, s), sbits(nsuper / 32 + 1, s), inm(kMaxWorkers * kMaskWords, s);
  MP_CUDA(cudaMemsetAsync(vis, 0, sizeof(int32_t) * vis.n, s));
  MP_CUDA(cudaMemsetAsync(tbits, 0, sizeof(uint32_t) * tbits.n, s));
  MP_CUDA(cudaMemsetAsync(sbits, 0, sizeof(uint32_t) * sbits.n, s));
  MP_CUDA(cudaMemsetAsync(acc, 0, sizeof(int32_t) * kMaxWorkers, s));
  MP_CUDA(cudaMemsetAsync(tkey, 0, sizeof(uint64_t) * ntile, s));
  MP_KERNEL(ctx, build_ell_batched<<<std::max(1, std::min((n + 255) / 256, ctx.num_sms * 16)), 256, 0, s>>>(g, ell));
  BatchArgs a{};
  a.g = g, a.ell = ell, a.n = n, a.k = k, a.tile_shift = tile_shift, a.ntile = ntile, a.nsuper = nsuper;
  a.seed = seed, a.dist = dist, a.tkey = tkey, a.skey = skey, a.tbits = tbits, a.tlist = tlist, a.sbits = sbits;
  a.slist = slist, a.fa = fa, a.fb = fb, a.vis = vis, a.dw = dw, a.reg = reg, a.cand = cand, a.ckey = ckey;
  a.mkey = mkey, a.inm = inm, a.regn = regn, a.acc = acc, a.ctl = ctl, a.seeds = seeds, a.work = ctx.dwork;
  void* args[] = {&a};
  const int kt = ctx.ktime_begin(kKFps);
  MP_KERNEL(ctx, MP_CUDA(cudaLaunchCooperativeKernel((void*)fps_batched_kernel, W, kThreads, args, smem, s)));
  ctx.ktime_end(kt);
}

}  // namespace mp
