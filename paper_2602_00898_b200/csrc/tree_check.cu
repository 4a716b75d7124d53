// The pipeline's separation self-check (reference pipeline.cpp:141-142,
// cross_block_fill symbolic.cpp:98-119), in its
// edge-locality form (tests/etree_test.cpp:171-179): count the edges whose
// endpoints lie in tree nodes that are neither equal nor ancestor-related.
// With no such edge, elimination in any descendants-first schedule
// (postorder, levelorder) never creates a factor entry between unrelated
// nodes, i.e. cross_block_fill == 0; a nonzero count means a separator failed
// to disconnect its sides.  One CSR pass instead of an elimination game.
#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

// node of every vertex from the flattened tree (offsets ascending)
__global__ void node_of_from_tree(int32_t n, int32_t nn, const int32_t* off, const int32_t* verts, int32_t* node_of,
                                  int32_t* bad) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int32_t lo = 0, hi = nn - 1;  // last node whose offset is <= i
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (off[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const int32_t v = verts[i];
    if (v < 0 || v >= n) {
      atomicExch(bad, 1);
      continue;
    }
    node_of[v] = lo;
  }
}

__global__ void unrelated_edges(DGraph g, const int32_t* node_of, unsigned long long* count) {
  __shared__ int64_t red[32];
  int64_t c = 0;
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < g.n; u += gridDim.x * blockDim.x) {
    const int32_t a = node_of[u];
    for (int32_t j = g.off[u]; j < g.off[u + 1]; ++j) {
      const int32_t v = g.nbr[j];
      if (v <= u) continue;
      const int32_t b = node_of[v];
      if (a != b && !is_ancestor_or_self(a, b) && !is_ancestor_or_self(b, a)) ++c;
    }
  }
  c = block_sum_i64(c, red);
  if (threadIdx.x == 0 && c) atomicAdd(count, static_cast<unsigned long long>(c));
}

}  // namespace

int64_t unrelated_edges_dev(mp_context& ctx, const DGraph& g, const int32_t* node_of) {
  cudaStream_t s = ctx.stream;
  DevBuf<unsigned long long> cnt(1, s);
  MP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(g.n, 256), ctx.num_sms * 8LL)));
  if (g.n > 0) MP_KERNEL(ctx, unrelated_edges<<<grid, 256, 0, s>>>(g, node_of, cnt));
  unsigned long long h = 0;
  MP_CUDA(cudaMemcpyAsync(&h, cnt.get(), sizeof h, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  return static_cast<int64_t>(h);
}

}  // namespace mp

using namespace mp;

extern "C" int mp_tree_separation_check(mp_context* ctx, const mp_csr* g, int32_t nd_level,
                                        const int32_t* node_offsets, const int32_t* node_vertices,
                                        int32_t on_device, int64_t* violations) {
  return guarded([&] {
    if (!ctx || !g || !node_offsets || !node_vertices || !violations) throw Error(MP_EINVAL, "null argument");
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    ContextScope scope(*ctx);
    cudaStream_t s = ctx->stream;
    const int32_t n = g->n, nn = (1 << (nd_level + 1)) - 1;
    DevBuf<int32_t> doff, dnbr, toff, tv, node_of(std::max(n, 1), s), bad(1, s);
    const int32_t *off = g->offsets, *nbr = g->neighbors, *to = node_offsets, *tvv = node_vertices;
    if (!g->on_device) {
      const int32_t m2 = g->offsets[n];
      doff.alloc(n + 1, s), dnbr.alloc(std::max(m2, 1), s);
      MP_CUDA(cudaMemcpyAsync(doff.get(), g->offsets, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, s));
      if (m2) MP_CUDA(cudaMemcpyAsync(dnbr.get(), g->neighbors, sizeof(int32_t) * m2, cudaMemcpyHostToDevice, s));
      off = doff.get(), nbr = dnbr.get();
    }
    if (!on_device) {
      toff.alloc(nn + 1, s), tv.alloc(std::max(n, 1), s);
      MP_CUDA(cudaMemcpyAsync(toff.get(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyHostToDevice, s));
      if (n) MP_CUDA(cudaMemcpyAsync(tv.get(), node_vertices, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
      to = toff.get(), tvv = tv.get();
    }
    MP_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), s));
    MP_CUDA(cudaMemsetAsync(node_of, 0xff, sizeof(int32_t) * std::max(n, 1), s));
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), ctx->num_sms * 8LL)));
    if (n > 0) MP_KERNEL(*ctx, node_of_from_tree<<<grid, 256, 0, s>>>(n, nn, to, tvv, node_of, bad));
    int32_t hb = 0;
    MP_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof hb, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (hb) throw Error(MP_EINVAL, "tree vertex out of range");
    *violations = unrelated_edges_dev(*ctx, DGraph{n, off, nbr}, node_of);
  });
}
