// Device CSR construction from triangles: mesh_to_graph / graph_from_edges
// (reference core/src/graph.cpp:14-75, validate_mesh types.cpp:20-33),
// SURVEY §8 row f1.  The output is the reference's AdjacencyGraph exactly:
// per-vertex neighbour lists sorted ascending, duplicates (edges shared by two
// triangles) removed, no self loops.
//
// HBM-bound integer work, no sort of the whole edge set:
//   1. tri_count:   validate every triangle, 2 raw entries per corner (atomics)
//   2. scan         raw list offsets
//   3. tri_scatter: each corner appends its two opposite corners
//   4. list_mark / list_sort_long: lists longer than kSortCap (a vertex in
//                   more than kSortCap / 2 triangles; block patterns) are
//                   sorted + deduplicated in place, one warp each
//   5. list_finish: one thread per vertex sorts + dedups its raw list in
//                   shared memory, a block scan of the unique lengths plus a
//                   decoupled look-back across tiles gives the CSR offsets, and
//                   the thread writes its offset and neighbours directly (no
//                   separate scan or compaction pass)
// Algorithmic bytes: 12 per triangle read + 4 (n + 1) + 4 nnz written.
#include <cub/cub.cuh>

#include <string>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortCap = 48;  // raw entries per vertex sorted in shared memory

__global__ void tri_count(int64_t ntri, int32_t nv, const int32_t* __restrict__ tris, int32_t* cnt,
                          unsigned long long* bad) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ntri;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t a = __ldg(&tris[3 * t]), b = __ldg(&tris[3 * t + 1]), c = __ldg(&tris[3 * t + 2]);
    const bool range = a < 0 || a >= nv || b < 0 || b >= nv || c < 0 || c >= nv;
    if (range || a == b || b == c || a == c) {  // first bad triangle wins (reference order)
      atomicMin(bad, (static_cast<unsigned long long>(t) << 1) | (range ? 0ull : 1ull));
      continue;
    }
    atomicAdd(&cnt[a], 2), atomicAdd(&cnt[b], 2), atomicAdd(&cnt[c], 2);
  }
}

__global__ void tri_scatter(int64_t ntri, int32_t nv, const int32_t* __restrict__ tris, int32_t* cur, int32_t* raw) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ntri;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t a = __ldg(&tris[3 * t]), b = __ldg(&tris[3 * t + 1]), c = __ldg(&tris[3 * t + 2]);
    if (a < 0 || a >= nv || b < 0 || b >= nv || c < 0 || c >= nv || a == b || b == c || a == c) continue;
    int32_t p = atomicAdd(&cur[a], 2);
    raw[p] = b, raw[p + 1] = c;
    p = atomicAdd(&cur[b], 2);
    raw[p] = a, raw[p + 1] = c;
    p = atomicAdd(&cur[c], 2);
    raw[p] = a, raw[p + 1] = b;
  }
}

// SparsePattern entries (rows[k], cols[k]) -> edges between blocks
// (i / b, j / b), diagonal blocks dropped: build_graph (b = 1, graph.cpp:53-61)
// and compress_blocks (graph.cpp:77-94).  The first out-of-range entry wins.
__global__ void pair_count(int64_t nnz, int32_t n, int32_t b, const int32_t* __restrict__ rows,
                           const int32_t* __restrict__ cols, int32_t* cnt, unsigned long long* bad) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = __ldg(&rows[k]), j = __ldg(&cols[k]);
    if (i < 0 || i >= n || j < 0 || j >= n) {
      atomicMin(bad, static_cast<unsigned long long>(k));
      continue;
    }
    const int32_t u = i / b, v = j / b;
    if (u != v) atomicAdd(&cnt[u], 1), atomicAdd(&cnt[v], 1);
  }
}
__global__ void pair_scatter(int64_t nnz, int32_t n, int32_t b, const int32_t* __restrict__ rows,
                             const int32_t* __restrict__ cols, int32_t* cur, int32_t* raw) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = __ldg(&rows[k]), j = __ldg(&cols[k]);
    if (i < 0 || i >= n || j < 0 || j >= n) continue;
    const int32_t u = i / b, v = j / b;
    if (u == v) continue;
    raw[atomicAdd(&cur[u], 1)] = v;
    raw[atomicAdd(&cur[v], 1)] = u;
  }
}

// Lists longer than kSortCap, for list_sort_long.
__global__ void list_mark(int32_t nv, const int32_t* ro, int32_t* nlong, int32_t* longv) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x)
    if (ro[v + 1] - ro[v] > kSortCap) longv[atomicAdd(nlong, 1)] = v;
}

// One warp per long list: odd-even transposition in global memory (rare: a
// vertex in more than kSortCap / 2 triangles).
__global__ void list_sort_long(const int32_t* nlong, const int32_t* longv, const int32_t* ro, int32_t* raw,
                               int32_t* deg) {
  const int lane = threadIdx.x & 31;
  const int32_t nl = *nlong;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < nl;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int32_t v = longv[w];
    const int32_t b = ro[v], len = ro[v + 1] - b;
    for (int32_t r = 0; r < len; ++r) {
      for (int32_t i = 2 * lane + (r & 1); i + 1 < len; i += 64) {
        const int32_t x = raw[b + i], y = raw[b + i + 1];
        if (x > y) raw[b + i] = y, raw[b + i + 1] = x;
      }
      __syncwarp();
    }
    if (lane == 0) {
      int32_t u = 0;
      for (int32_t k = 0; k < len; ++k)
        if (u == 0 || raw[b + u - 1] != raw[b + k]) raw[b + u++] = raw[b + k];
      deg[v] = u;
    }
  }
}

// 1D bulk copy global -> shared (TMA, cp.async.bulk) completing on an mbarrier.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

constexpr int32_t kStage = kSortThreads * 16;  // staged raw entries per tile (16 KB; larger tiles read global)

// Tiles of kSortThreads vertices, taken in order from a counter.  The tile's
// raw lists are one contiguous range of raw: a bulk copy (TMA) stages it in
// shared memory, each thread sorts + dedups its list there (long lists are
// already sorted in place, their unique length in deg), the block scans the
// unique lengths, thread 0 resolves the tile's offset by decoupled look-back
// over the earlier tiles' published sums (tstate[t] = flag << 32 | value,
// 1 aggregate, 2 inclusive), the lists are packed into an output stage and
// the CTA writes offsets and neighbours with coalesced stores.  A tile whose
// range does not fit the stage sorts from global memory.
__global__ void __launch_bounds__(kSortThreads) list_finish(int32_t nv, const int32_t* ro, const int32_t* raw,
                                                           const int32_t* deg, int32_t* off, int32_t* nbr,
                                                           unsigned long long* tstate, int32_t* tcounter) {
  extern __shared__ __align__(128) int32_t lf_stage[];  // in[kStage] | outs[kStage]
  int32_t* in = lf_stage;
  int32_t* outs = lf_stage + kStage;
  __shared__ uint64_t bar;
  __shared__ int32_t sh[32], s_tile, s_prefix, s_a0, s_staged;
  volatile unsigned long long* vs = tstate;
  if (threadIdx.x == 0) mbar_init(&bar);
  __syncthreads();  // the barrier is initialised before any thread can observe it
  uint32_t phase = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      const int32_t tile = atomicAdd(tcounter, 1);
      s_tile = tile;
      s_staged = 0;
      const int64_t v0 = static_cast<int64_t>(tile) * kSortThreads;
      if (v0 < nv) {
        const int32_t v1 = static_cast<int32_t>(v0 + kSortThreads < nv ? v0 + kSortThreads : nv);
        const int32_t a0 = ro[v0] & ~3, a1 = (ro[v1] + 3) & ~3;  // 16-byte aligned superset
        s_a0 = a0;
        if (a1 - a0 <= kStage && a1 > a0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic use of `in`
          bulk_load(in, raw + a0, static_cast<uint32_t>(a1 - a0) * 4u, &bar);
          s_staged = 1;
        }
      }
    }
    __syncthreads();
    const int32_t tile = s_tile;
    if (static_cast<int64_t>(tile) * kSortThreads >= nv) break;
    const bool staged = s_staged;
    if (staged) {
      mbar_wait(&bar, phase);
      phase ^= 1;
    }
    const int32_t v = tile * kSortThreads + threadIdx.x;
    int32_t u = 0, b = 0, len = 0;
    int32_t* my = nullptr;
    int32_t loc[kSortCap];  // unstaged tiles only
    if (v < nv) {
      b = ro[v], len = ro[v + 1] - b;
      if (len > kSortCap) {
        u = deg[v];  // sorted in place by list_sort_long
      } else {
        if (staged) {
          my = in + (b - s_a0);
        } else {
          my = loc;
          for (int32_t k = 0; k < len; ++k) loc[k] = raw[b + k];
        }
        for (int32_t k = 1; k < len; ++k) {  // insertion sort
          const int32_t x = my[k];
          int32_t j = k;
          while (j > 0 && my[j - 1] > x) my[j] = my[j - 1], --j;
          my[j] = x;
        }
        for (int32_t k = 0; k < len; ++k)
          if (u == 0 || my[u - 1] != my[k]) my[u++] = my[k];
      }
    }
    int32_t tot = 0;
    const int32_t ex = block_excl_scan(u, sh, &tot);
    // decoupled look-back, one warp: 32 predecessors per step, stop at the
    // nearest published inclusive prefix
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      if (tile == 0) {
        if (lane == 0) vs[0] = (2ull << 32) | static_cast<uint32_t>(tot), s_prefix = 0;
      } else {
        if (lane == 0) vs[tile] = (1ull << 32) | static_cast<uint32_t>(tot);
        int32_t prefix = 0;
        for (int32_t hi = tile - 1;;) {
          const int32_t t = hi - lane;  // lane 0 nearest
          unsigned long long x = 0;
          uint32_t fl = 2;
          if (t >= 0) {
            do {
              x = vs[t];
              fl = static_cast<uint32_t>(x >> 32);
            } while (fl == 0);
          }
          const uint32_t incl = __ballot_sync(0xffffffffu, t >= 0 && fl == 2);
          const int stop = incl ? __ffs(incl) - 1 : 32;  // nearest inclusive (or none in the window)
          int32_t val = (t >= 0 && lane <= stop) ? static_cast<int32_t>(static_cast<uint32_t>(x)) : 0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
          prefix += val;
          if (incl || hi - 32 < 0) break;
          hi -= 32;
        }
        if (lane == 0) {
          vs[tile] = (2ull << 32) | static_cast<uint32_t>(prefix + tot);
          s_prefix = prefix;
        }
      }
    }
    // pack the deduplicated lists (never more than the staged input)
    const int32_t* src = len > kSortCap ? (staged ? in + (b - s_a0) : raw + b) : my;
    if (staged && v < nv)
      for (int32_t k = 0; k < u; ++k) outs[ex + k] = src[k];
    __syncthreads();
    const int32_t P = s_prefix;
    if (v < nv) {
      off[v] = P + ex;
      if (v == nv - 1) off[nv] = P + ex + u;
      if (nbr && !staged)
        for (int32_t k = 0; k < u; ++k) nbr[P + ex + k] = src[k];
    }
    if (nbr && staged)
      for (int32_t i = threadIdx.x; i < tot; i += blockDim.x) nbr[P + i] = outs[i];
    __syncthreads();  // the stages are consumed before the next tile
  }
}

}  // namespace

int grid_for_items(const mp_context& ctx, int64_t items) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), ctx.num_sms * 16LL)));
}

// Shared back half: raw lists (counted in cnt, appended by scatter(cursors,
// raw)) -> sorted, deduplicated CSR.  check_bad(verdict) throws for invalid
// input after the one host synchronisation.
template <class Count, class Scatter, class Check>
int64_t csr_from_raw(mp_context& ctx, int32_t nv, int64_t nraw, int32_t* off, int32_t* nbr, DevBuf<int32_t>* alloc,
                     Count count, Scatter scatter, unsigned long long* bad, Check check_bad) {
  cudaStream_t s = ctx.stream;
  if (nraw > 0x7fffffffLL) throw Error(MP_EINVAL, "input too large for int32 offsets");
  DevBuf<int32_t> cnt(static_cast<size_t>(nv) + 1, s), ro(static_cast<size_t>(nv) + 1, s), raw(std::max<int64_t>(nraw, 1) + 4, s);  // +4: bulk copies read whole 16-byte groups
  MP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nv + 1), s));
  MP_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
  count(cnt.get());
  size_t tmp = 0;
  MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.get(), ro.get(), nv + 1, s));
  DevBuf<char> t1(tmp, s);
  MP_CUDA(cub::DeviceScan::ExclusiveSum(t1.get(), tmp, cnt.get(), ro.get(), nv + 1, s));
  MP_CUDA(cudaMemcpyAsync(cnt.get(), ro.get(), sizeof(int32_t) * nv, cudaMemcpyDeviceToDevice, s));  // cursors
  scatter(cnt.get(), raw.get());
  DevBuf<int32_t> deg(static_cast<size_t>(nv) + 1, s), longv(static_cast<size_t>(nv) + 1, s);
  MP_CUDA(cudaMemsetAsync(longv.get() + nv, 0, sizeof(int32_t), s));  // long-list count
  // neighbours: the caller's array, or one sized by the raw count (an upper
  // bound of nnz, so no host round trip before the finish)
  if (!nbr && alloc) {
    alloc->alloc(std::max<int64_t>(nraw, 1), s);
    nbr = alloc->get();
  }
  const int64_t tiles = ceil_div(std::max(nv, 1), kSortThreads);
  DevBuf<unsigned long long> tstate(tiles, s);
  DevBuf<int32_t> tcounter(1, s);
  MP_CUDA(cudaMemsetAsync(tstate, 0, sizeof(unsigned long long) * tiles, s));
  MP_CUDA(cudaMemsetAsync(tcounter, 0, sizeof(int32_t), s));
  if (nv > 0) {
    MP_KERNEL(ctx, list_mark<<<grid_for_items(ctx, nv), 256, 0, s>>>(nv, ro, longv.get() + nv, longv));
    MP_KERNEL(ctx, list_sort_long<<<ctx.num_sms, 256, 0, s>>>(longv.get() + nv, longv, ro, raw, deg));
    const int fg = static_cast<int>(std::min<int64_t>(tiles, ctx.num_sms * 8LL));
    allow_max_smem(list_finish, ctx.device);
    MP_KERNEL(ctx, list_finish<<<fg, kSortThreads, 2 * kStage * sizeof(int32_t), s>>>(nv, ro, raw, deg, off, nbr, tstate,
                                                                                      tcounter));
  } else {
    MP_CUDA(cudaMemsetAsync(off, 0, sizeof(int32_t), s));
  }
  int32_t nnz = 0;
  unsigned long long hbad = 0;
  MP_CUDA(cudaMemcpyAsync(&nnz, off + nv, sizeof nnz, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  check_bad(hbad);
  return nnz;
}

// Builds off (nv + 1) and the neighbours (device pointers): into nbr when it
// is non-null, else into *alloc (sized here) when that is non-null, else
// offsets only.  Returns nnz = 2|E|.  Throws MP_EINVAL with the reference's
// messages.
int64_t mesh_to_graph_dev(mp_context& ctx, int32_t nv, int64_t ntri, const int32_t* tris, int32_t* off,
                          int32_t* nbr, DevBuf<int32_t>* alloc) {
  cudaStream_t s = ctx.stream;
  if (nv < 0) throw Error(MP_EINVAL, "negative vertex count");
  const int grid = grid_for_items(ctx, std::max<int64_t>(ntri, nv));
  DevBuf<unsigned long long> bad(1, s);
  return csr_from_raw(
      ctx, nv, 6 * ntri, off, nbr, alloc,
      [&](int32_t* cnt) { if (ntri > 0) MP_KERNEL(ctx, tri_count<<<grid, 256, 0, s>>>(ntri, nv, tris, cnt, bad)); },
      [&](int32_t* cur, int32_t* raw) { if (ntri > 0) MP_KERNEL(ctx, tri_scatter<<<grid, 256, 0, s>>>(ntri, nv, tris, cur, raw)); },
      bad.get(),
      [&](unsigned long long hbad) {  // validate_mesh's message for the first bad triangle (types.cpp:20-33)
        if (hbad == ~0ull) return;
        const int64_t t = static_cast<int64_t>(hbad >> 1);
        int32_t c[3];
        MP_CUDA(cudaMemcpy(c, tris + 3 * t, sizeof c, cudaMemcpyDeviceToHost));
        if (!(hbad & 1ull)) {
          for (int k = 0; k < 3; ++k)
            if (c[k] < 0 || c[k] >= nv)
              throw Error(MP_EINVAL, "triangle " + std::to_string(t) + " references vertex " + std::to_string(c[k]) +
                                         " outside [0, " + std::to_string(nv) + ")");
        }
        throw Error(MP_EINVAL, "triangle " + std::to_string(t) + " has repeated corners");
      });
}

// build_graph (b = 1) / compress_blocks (b > 1) of a SparsePattern on the device.
int64_t pattern_to_graph_dev(mp_context& ctx, int32_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                             int32_t b, int32_t* off, int32_t* nbr, DevBuf<int32_t>* alloc) {
  cudaStream_t s = ctx.stream;
  if (b < 1) throw Error(MP_EINVAL, "block size must be positive");
  if (n < 0) throw Error(MP_EINVAL, "negative matrix size");
  if (n % b != 0)
    throw Error(MP_EINVAL, "matrix size " + std::to_string(n) + " is not a multiple of block size " + std::to_string(b));
  const int32_t nodes = n / b;
  const int grid = grid_for_items(ctx, std::max<int64_t>(nnz, nodes));
  DevBuf<unsigned long long> bad(1, s);
  return csr_from_raw(
      ctx, nodes, 2 * nnz, off, nbr, alloc,
      [&](int32_t* cnt) { if (nnz > 0) MP_KERNEL(ctx, pair_count<<<grid, 256, 0, s>>>(nnz, n, b, rows, cols, cnt, bad)); },
      [&](int32_t* cur, int32_t* raw) { if (nnz > 0) MP_KERNEL(ctx, pair_scatter<<<grid, 256, 0, s>>>(nnz, n, b, rows, cols, cur, raw)); },
      bad.get(),
      [&](unsigned long long hbad) {
        if (hbad != ~0ull) throw Error(MP_EINVAL, "pattern entry out of range");
      });
}

__global__ void lift_kernel(int64_t n, int32_t b, const int32_t* in, int32_t* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * b;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i / b];
}

}  // namespace mp

using namespace mp;

extern "C" int mp_mesh_to_graph_device(mp_context* ctx, int32_t nv, int64_t ntri, const int32_t* tris,
                                       int32_t tris_on_device, int32_t* off, int32_t* nbr, int32_t out_on_device,
                                       int64_t* nnz) {
  return guarded([&] {
    if (!ctx || (!tris && ntri > 0) || !off) throw Error(MP_EINVAL, "null argument");
    if (ntri < 0) throw Error(MP_EINVAL, "negative triangle count");
    ContextScope scope(*ctx);
    cudaStream_t s = ctx->stream;
    DevBuf<int32_t> dtris, doff, dnbr;
    const int32_t* t = tris;
    if (!tris_on_device && ntri > 0) {
      dtris.alloc(3 * ntri, s);
      MP_CUDA(cudaMemcpyAsync(dtris.get(), tris, sizeof(int32_t) * 3 * ntri, cudaMemcpyHostToDevice, s));
      t = dtris.get();
    }
    int32_t* o = off;
    if (!out_on_device) {
      doff.alloc(static_cast<size_t>(nv) + 1, s);
      o = doff.get();
    }
    const bool want = nbr != nullptr;
    const int64_t m = mesh_to_graph_dev(*ctx, nv, ntri, t, o, out_on_device ? nbr : nullptr,
                                        (!out_on_device && want) ? &dnbr : nullptr);
    if (!out_on_device) {
      MP_CUDA(cudaMemcpyAsync(off, o, sizeof(int32_t) * (static_cast<size_t>(nv) + 1), cudaMemcpyDeviceToHost, s));
      if (want && m > 0) MP_CUDA(cudaMemcpyAsync(nbr, dnbr.get(), sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
    }
    if (nnz) *nnz = m;
  });
}

extern "C" int mp_pattern_to_graph_device(mp_context* ctx, int32_t n, int64_t nnz, const int32_t* rows,
                                         const int32_t* cols, int32_t in_on_device, int32_t block_size, int32_t* off,
                                         int32_t* nbr, int32_t out_on_device, int64_t* nnz_out) {
  return guarded([&] {
    if (!ctx || (nnz > 0 && (!rows || !cols)) || !off) throw Error(MP_EINVAL, "null argument");
    if (nnz < 0) throw Error(MP_EINVAL, "negative entry count");
    if (block_size < 1) throw Error(MP_EINVAL, "block size must be positive");
    ContextScope scope(*ctx);
    cudaStream_t s = ctx->stream;
    DevBuf<int32_t> dr, dc, doff, dnbr;
    const int32_t *r = rows, *c = cols;
    if (!in_on_device && nnz > 0) {
      dr.alloc(nnz, s), dc.alloc(nnz, s);
      MP_CUDA(cudaMemcpyAsync(dr.get(), rows, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
      MP_CUDA(cudaMemcpyAsync(dc.get(), cols, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
      r = dr.get(), c = dc.get();
    }
    const int32_t nodes = n >= 0 && n % block_size == 0 ? n / block_size : 0;
    int32_t* o = off;
    if (!out_on_device) {
      doff.alloc(static_cast<size_t>(nodes) + 1, s);
      o = doff.get();
    }
    const bool want = nbr != nullptr;
    const int64_t m = pattern_to_graph_dev(*ctx, n, nnz, r, c, block_size, o, out_on_device ? nbr : nullptr,
                                           (!out_on_device && want) ? &dnbr : nullptr);
    if (!out_on_device) {
      MP_CUDA(cudaMemcpyAsync(off, o, sizeof(int32_t) * (static_cast<size_t>(nodes) + 1), cudaMemcpyDeviceToHost, s));
      if (want && m > 0) MP_CUDA(cudaMemcpyAsync(nbr, dnbr.get(), sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaStreamSynchronize(s));
    }
    if (nnz_out) *nnz_out = m;
  });
}

extern "C" int mp_lift_patches(mp_context* ctx, int32_t n, const int32_t* assignment, int32_t block_size,
                               int32_t* out, int32_t on_device) {
  return guarded([&] {
    if (!ctx || (n > 0 && (!assignment || !out))) throw Error(MP_EINVAL, "null argument");
    if (block_size < 1) throw Error(MP_EINVAL, "block size must be positive");
    if (!on_device) {  // host arrays: nothing to gain from a device round trip
      for (int64_t v = 0; v < n; ++v)
        for (int32_t t = 0; t < block_size; ++t) out[v * block_size + t] = assignment[v];
      return;
    }
    ContextScope scope(*ctx);
    if (n > 0)
      MP_KERNEL(*ctx, lift_kernel<<<grid_for_items(*ctx, static_cast<int64_t>(n) * block_size), 256, 0, ctx->stream>>>(
                          n, block_size, assignment, out));
    MP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

