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
int64_t mesh_to_graph_dev(mp_context& ctx, int32_t nv, int64_t ntri, const int32_t* tris, int32_t* off,
                          int32_t* nbr, DevBuf<int32_t>* alloc) {
  cudaStream_t s = ctx.stream;
  if (nv < 0) throw Error(MP_EINVAL, "negative vertex count");
  const int64_t nraw = 6 * ntri;
  if (nraw > 0x7fffffffLL) throw Error(MP_EINVAL, "mesh too large for int32 offsets");
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(ntri, nv), 256),
                                                                          ctx.num_sms * 16LL)));
  DevBuf<int32_t> cnt(static_cast<size_t>(nv) + 1, s), ro(static_cast<size_t>(nv) + 1, s), raw(std::max<int64_t>(nraw, 1), s);
  DevBuf<unsigned long long> bad(1, s);
  MP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nv + 1), s));
  MP_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
  if (ntri > 0) MP_KERNEL(ctx, tri_count<<<grid, 256, 0, s>>>(ntri, nv, tris, cnt, bad));
  // (bad triangles are skipped by the scatter; the verdict is read with nnz)
  auto check_bad = [&](unsigned long long hbad) {
  if (hbad != ~0ull) {  // validate_mesh's message for the first bad triangle (types.cpp:20-33)
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
  }
  };
  size_t tmp = 0;
  MP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.get(), ro.get(), nv + 1, s));
  DevBuf<char> t1(tmp, s);
  MP_CUDA(cub::DeviceScan::ExclusiveSum(t1.get(), tmp, cnt.get(), ro.get(), nv + 1, s));
  MP_CUDA(cudaMemcpyAsync(cnt.get(), ro.get(), sizeof(int32_t) * nv, cudaMemcpyDeviceToDevice, s));  // cursors
  if (ntri > 0) MP_KERNEL(ctx, tri_scatter<<<grid, 256, 0, s>>>(ntri, nv, tris, cnt, raw));
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
  MP_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof hbad, cudaMemcpyDeviceToHost, s));
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

}  // namespace mp

using namespace mp;

extern "C" int mp_mesh_to_graph_device(mp_context* ctx, int32_t nv, int64_t ntri, const int32_t* tris,
                                       int32_t tris_on_device, int32_t* off, int32_t* nbr, int32_t out_on_device,
                                       int64_t* nnz) {
  return guarded([&] {
    if (!ctx || (!tris && ntri > 0) || !off) throw Error(MP_EINVAL, "null argument");
    if (ntri < 0) throw Error(MP_EINVAL, "negative triangle count");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
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
    if (prev != ctx->device) cudaSetDevice(prev);
  });
}
