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
//   4. list_sort:   one thread per vertex sorts + dedups its raw list in shared
//                   memory (lists longer than kSortCap: listed, one warp each)
//   5. scan         CSR offsets of the deduplicated lengths
//   6. list_copy:   compact the sorted lists into neighbors[]
// Algorithmic bytes: 12 per triangle read + 4 (n + 1) + 4 nnz written.
#include <cub/cub.cuh>

#include <string>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

constexpr int kSortThreads = 128;
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

// Sort + dedup each raw list in place; deg[v] = unique length.  Long lists are
// left for list_sort_long (appended to `longv`, counted in longv[-1]).
__global__ void __launch_bounds__(kSortThreads) list_sort(int32_t nv, const int32_t* ro, int32_t* raw, int32_t* deg,
                                                         int32_t* nlong, int32_t* longv) {
  __shared__ int32_t sm[kSortThreads * kSortCap];
  int32_t* my = sm + threadIdx.x;  // strided: entry k at my[k * kSortThreads] (bank-conflict free)
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const int32_t b = ro[v], len = ro[v + 1] - b;
    if (len > kSortCap) {
      longv[atomicAdd(nlong, 1)] = v;
      continue;
    }
    for (int32_t k = 0; k < len; ++k) {  // insertion sort while loading
      const int32_t x = raw[b + k];
      int32_t j = k;
      while (j > 0 && my[(j - 1) * kSortThreads] > x) {
        my[j * kSortThreads] = my[(j - 1) * kSortThreads];
        --j;
      }
      my[j * kSortThreads] = x;
    }
    int32_t u = 0;
    for (int32_t k = 0; k < len; ++k) {
      const int32_t x = my[k * kSortThreads];
      if (k == 0 || my[(k - 1) * kSortThreads] != x) raw[b + u++] = x;
    }
    deg[v] = u;
  }
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

__global__ void list_copy(int32_t nv, const int32_t* ro, const int32_t* raw, const int32_t* off, int32_t* nbr) {
  // one warp per vertex: lists are short, lanes copy consecutive entries
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < nv;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int32_t v = static_cast<int32_t>(w);
    const int32_t b = ro[v], o = off[v], d = off[v + 1] - o;
    for (int32_t k = lane; k < d; k += 32) nbr[o + k] = raw[b + k];
  }
}

}  // namespace

// Builds off (nv + 1) and the neighbours (device pointers): into nbr when it
// is non-null, else into *alloc (sized here) when that is non-null, else
// offsets only.  Returns nnz = 2|E|.  Throws MP_EINVAL with the reference's
// messages.
// Shared back half: raw lists (counted in cnt, appended by scatter(cursors,
// raw)) -> sorted, deduplicated CSR.  check_bad(verdict) throws for invalid
// input after the one host synchronisation.
template <class Count, class Scatter, class Check>
int64_t csr_from_raw(mp_context& ctx, int32_t nv, int64_t nraw, int32_t* off, int32_t* nbr, DevBuf<int32_t>* alloc,
                     Count count, Scatter scatter, unsigned long long* bad, Check check_bad) {
  cudaStream_t s = ctx.stream;
  if (nraw > 0x7fffffffLL) throw Error(MP_EINVAL, "input too large for int32 offsets");
  DevBuf<int32_t> cnt(static_cast<size_t>(nv) + 1, s), ro(static_cast<size_t>(nv) + 1, s), raw(std::max<int64_t>(nraw, 1), s);
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
  MP_CUDA(cudaMemsetAsync(deg.get() + nv, 0, sizeof(int32_t), s));
  MP_CUDA(cudaMemsetAsync(longv.get() + nv, 0, sizeof(int32_t), s));  // long-list count
  if (nv > 0) {
    const int sg = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nv, kSortThreads), ctx.num_sms * 8LL)));
    MP_KERNEL(ctx, list_sort<<<sg, kSortThreads, 0, s>>>(nv, ro, raw, deg, longv.get() + nv, longv));
    MP_KERNEL(ctx, list_sort_long<<<ctx.num_sms, 256, 0, s>>>(longv.get() + nv, longv, ro, raw, deg));
  }
  MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg.get(), off, nv + 1, s));
  DevBuf<char> t2(tmp, s);
  MP_CUDA(cub::DeviceScan::ExclusiveSum(t2.get(), tmp, deg.get(), off, nv + 1, s));
  int32_t nnz = 0;
  unsigned long long hbad = 0;
  MP_CUDA(cudaMemcpyAsync(&nnz, off + nv, sizeof nnz, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, s));
  if (!nbr && alloc) {
    MP_CUDA(cudaStreamSynchronize(s));
    check_bad(hbad);
    alloc->alloc(std::max(nnz, 1), s);
    nbr = alloc->get();
  }
  if (nbr && nv > 0) {
    const int cg = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(static_cast<int64_t>(nv) * 32, 256),
                                                                            ctx.num_sms * 16LL)));
    MP_KERNEL(ctx, list_copy<<<cg, 256, 0, s>>>(nv, ro, raw, off, nbr));
  }
  MP_CUDA(cudaStreamSynchronize(s));
  check_bad(hbad);
  return nnz;
}

int grid_for_items(const mp_context& ctx, int64_t items) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), ctx.num_sms * 16LL)));
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

