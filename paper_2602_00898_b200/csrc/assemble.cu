// Stage 5a — permutation assembly (reference core/src/assemble.cpp).
//
// schedule_postorder / schedule_levelorder (assemble.cpp:24-46) are computed
// on the host over the 2^(L+1)-1 node ids (tiny), the per-node start
// positions are an exclusive scan of node sizes in schedule order, and one
// CTA per node scatters perm[pos + j] = vertices[local_perm[j]] plus the
// inverse (compute_perm :65-85, Permutation::from_order :8-22).  Block
// expansion (expand_blocks :87-114) is fused into the same scatter.
#include <algorithm>
#include <string>
#include <vector>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {
namespace {

// node_of[v] = node for every listed vertex; a vertex out of range or listed
// twice flags *bad (node_of must be -1 on entry).
__global__ void node_of_kernel(int32_t nn, int32_t n, const int32_t* node_offsets, const int32_t* node_vertices,
                               int32_t* node_of, int32_t* bad) {
  for (int32_t node = blockIdx.x; node < nn; node += gridDim.x)
    for (int32_t i = node_offsets[node] + threadIdx.x; i < node_offsets[node + 1]; i += blockDim.x) {
      const int32_t v = node_vertices[i];
      if (v < 0 || v >= n) {
        atomicExch(bad, 1);
        continue;
      }
      if (atomicExch(&node_of[v], node) != -1) atomicExch(bad, 2);
    }
}

__global__ void fill_neg(int64_t n, int32_t* a) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    a[i] = -1;
}

// perm[b*(pos+j)+t] = b*vertices[local_perm[j]] + t ; inverse likewise.
__global__ void scatter_perm(int32_t nn, const int32_t* node_offsets, const int32_t* node_vertices,
                             const int32_t* local_perm, const int32_t* node_pos, int32_t n, int32_t b,
                             const uint8_t* node_mask, int32_t* perm, int32_t* inverse, int32_t* bad) {
  for (int32_t node = blockIdx.x; node < nn; node += gridDim.x) {
    if (node_mask && !node_mask[node]) continue;
    const int32_t o = node_offsets[node], sz = node_offsets[node + 1] - o, pos = node_pos[node];
    for (int32_t j = threadIdx.x; j < sz; j += blockDim.x) {
      const int32_t lp = local_perm[o + j];
      if (lp < 0 || lp >= sz) {
        atomicExch(bad, 1);
        continue;
      }
      const int32_t v = node_vertices[o + lp];
      if (v < 0 || v >= n) {
        atomicExch(bad, 1);
        continue;
      }
      for (int32_t t = 0; t < b; ++t) {
        const int32_t newpos = b * (pos + j) + t, old = b * v + t;
        perm[newpos] = old;
        if (inverse && atomicExch(&inverse[old], newpos) != -1) atomicExch(bad, 2);
      }
    }
  }
}

}  // namespace

// Validates a caller tree before anything is scattered by it: offsets start
// at 0, are monotone and end at n (host check of nn+1 ints), and every vertex
// is in range and listed exactly once (device check).
void node_of_from_tree_dev(mp_context& ctx, int32_t n, int32_t nn, const int32_t* node_offsets,
                           const int32_t* node_vertices, int32_t* node_of) {
  cudaStream_t s = ctx.stream;
  std::vector<int32_t> hoff(nn + 1);
  MP_CUDA(cudaMemcpyAsync(hoff.data(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  for (int32_t i = 0; i < nn; ++i)
    if (hoff[i + 1] < hoff[i]) throw Error(MP_EINVAL, "tree node offsets are not monotone");
  if (hoff[0] != 0 || hoff[nn] != n) throw Error(MP_EINVAL, "tree vertex lists do not cover the graph");
  if (n == 0) return;
  DevBuf<int32_t> bad(1, s);
  MP_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  MP_CUDA(cudaMemsetAsync(node_of, 0xff, sizeof(int32_t) * n, s));
  MP_KERNEL(ctx, node_of_kernel<<<std::min(nn, 8192), 256, 0, s>>>(nn, n, node_offsets, node_vertices, node_of, bad));
  int32_t h_bad = 0;
  MP_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (h_bad == 1) throw Error(MP_EINVAL, "tree vertex out of range");
  if (h_bad == 2) throw Error(MP_EINVAL, "tree lists a vertex twice");
}

// Host schedules (assemble.cpp:24-46).
Schedule make_schedule(int32_t L, int32_t kind) {
  const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
  Schedule out;
  out.reserve(nn);
  if (kind == MP_SCHEDULE_LEVELORDER) {
    for (int32_t l = L; l >= 0; --l)
      for (int32_t i = (1 << l) - 1; i < (1 << (l + 1)) - 1; ++i) out.push_back(i);
  } else {
    // iterative postorder: left subtree, right subtree, node
    std::vector<std::pair<int32_t, int>> st{{0, 0}};
    while (!st.empty()) {
      auto& [idx, state] = st.back();
      if (idx >= nn) {
        st.pop_back();
        continue;
      }
      if (state == 0) {
        state = 1;
        st.push_back({2 * idx + 1, 0});
      } else if (state == 1) {
        state = 2;
        st.push_back({2 * idx + 2, 0});
      } else {
        out.push_back(idx);
        st.pop_back();
      }
    }
  }
  return out;
}

// validate_schedule (assemble.cpp:48-63): the first position that lists a
// node out of range, twice, or before one of its children; a short sequence
// reports its length; -1 when valid.
int64_t validate_schedule_host(int32_t L, const int32_t* seq, int64_t len) {
  const int64_t nn = (1LL << (L + 1)) - 1;
  std::vector<char> done(nn, 0);
  for (int64_t pos = 0; pos < len; ++pos) {
    const int64_t idx = seq[pos];
    if (idx < 0 || idx >= nn || done[idx]) return pos;
    const int64_t l = 2 * idx + 1, r = 2 * idx + 2;
    if (l < nn && !done[l]) return pos;
    if (r < nn && !done[r]) return pos;
    done[idx] = 1;
  }
  return len != nn ? len : -1;
}

Schedule resolve_schedule(int32_t L, int32_t kind, const int32_t* nodes, int64_t len) {
  if (!nodes) {
    if (kind != MP_SCHEDULE_POSTORDER && kind != MP_SCHEDULE_LEVELORDER) throw Error(MP_EINVAL, "unknown schedule");
    return make_schedule(L, kind);
  }
  if (len < 0) throw Error(MP_EINVAL, "negative schedule length");
  const int64_t bad = validate_schedule_host(L, nodes, len);
  if (bad >= 0) throw Error(MP_EINVAL, "invalid schedule at position " + std::to_string(bad));  // assemble.cpp:71-72
  return Schedule(nodes, nodes + len);
}

// Per-node first position (host, from node sizes), shared by assembly and symbolic.
std::vector<int32_t> node_positions(const std::vector<int32_t>& node_offsets, int32_t L, const Schedule& sched) {
  const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
  std::vector<int32_t> pos(nn + 1, 0);
  int32_t run = 0;
  for (int32_t idx : sched) {
    pos[idx] = run;
    run += node_offsets[idx + 1] - node_offsets[idx];
  }
  pos[nn] = run;
  return pos;
}

void compute_perm_blocks_dev(mp_context& ctx, int32_t n, int32_t L, const int32_t* node_offsets,
                             const int32_t* node_vertices, const int32_t* local_perm, const Schedule& schedule,
                             int32_t b, int32_t* perm, int32_t* inverse, int32_t* node_pos_dev) {
  cudaStream_t s = ctx.stream;
  const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
  std::vector<int32_t> hoff(nn + 1);
  MP_CUDA(cudaMemcpyAsync(hoff.data(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  for (int32_t i = 0; i < nn; ++i)
    if (hoff[i + 1] < hoff[i]) throw Error(MP_EINVAL, "tree node offsets are not monotone");
  if (hoff[nn] - hoff[0] != n || hoff[0] != 0)
    throw Error(MP_EINVAL, "tree vertex lists do not cover the graph");
  std::vector<int32_t> pos = node_positions(hoff, L, schedule);
  MP_CUDA(cudaMemcpyAsync(node_pos_dev, pos.data(), sizeof(int32_t) * (nn + 1), cudaMemcpyHostToDevice, s));
  DevBuf<int32_t> bad(1, s);
  MP_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  const int64_t N = static_cast<int64_t>(b) * n;
  MP_KERNEL(ctx, fill_neg<<<static_cast<int>(std::min<int64_t>(ceil_div(std::max<int64_t>(N, 1), 256), ctx.num_sms * 16LL)),
                           256, 0, s>>>(N, inverse));
  MP_KERNEL(ctx, scatter_perm<<<std::min(nn, 8192), 256, 0, s>>>(nn, node_offsets, node_vertices, local_perm,
                                                                 node_pos_dev, n, b, nullptr, perm, inverse, bad));
  int32_t h_bad = 0;
  MP_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (h_bad == 1) throw Error(MP_EINVAL, "permutation entry out of range");
  if (h_bad == 2) throw Error(MP_EINVAL, "permutation repeats an index");
}

void compute_perm_dev(mp_context& ctx, int32_t n, int32_t L, const int32_t* node_offsets,
                      const int32_t* node_vertices, const int32_t* local_perm, const Schedule& schedule, int32_t* perm,
                      int32_t* inverse, int32_t* node_pos) {
  compute_perm_blocks_dev(ctx, n, L, node_offsets, node_vertices, local_perm, schedule, 1, perm, inverse, node_pos);
}

void compute_perm_partial_dev(mp_context& ctx, int32_t n, int32_t L, const int32_t* node_offsets,
                              const int32_t* node_vertices, const int32_t* local_perm, const Schedule& schedule,
                              const uint8_t* node_mask, int32_t* perm) {
  cudaStream_t s = ctx.stream;
  const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
  std::vector<int32_t> hoff(nn + 1);
  MP_CUDA(cudaMemcpyAsync(hoff.data(), node_offsets, sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  for (int32_t i = 0; i < nn; ++i)
    if (hoff[i + 1] < hoff[i]) throw Error(MP_EINVAL, "tree node offsets are not monotone");
  if (hoff[nn] - hoff[0] != n || hoff[0] != 0)
    throw Error(MP_EINVAL, "tree vertex lists do not cover the graph");
  std::vector<int32_t> pos = node_positions(hoff, L, schedule);
  DevBuf<int32_t> pos_dev(nn + 1, s), bad(1, s);
  MP_CUDA(cudaMemcpyAsync(pos_dev, pos.data(), sizeof(int32_t) * (nn + 1), cudaMemcpyHostToDevice, s));
  MP_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  MP_KERNEL(ctx, scatter_perm<<<std::min(nn, 8192), 256, 0, s>>>(nn, node_offsets, node_vertices, local_perm, pos_dev,
                                                                 n, 1, node_mask, perm, nullptr, bad));
  int32_t h_bad = 0;
  MP_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (h_bad) throw Error(MP_EINVAL, "permutation entry out of range");
}

}  // namespace mp
