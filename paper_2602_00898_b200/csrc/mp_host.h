// Host-side helpers shared by the C-ABI translation units (api.cu, shard.cu):
// caller graph / array views and output copies.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "mp_context.h"
#include "mp_device.cuh"

namespace mp {

inline int32_t default_nd_level_host(int32_t n) {  // etree.cpp:42-46
  int32_t level = 0;
  for (int32_t x = n / 512; x > 1; x >>= 1) ++level;
  return std::min<int32_t>(8, level);
}

// Device view of a caller CSR (copied when it is host memory).
struct GraphView {
  DevBuf<int32_t> off, nbr;
  DGraph g{};
  int64_t m2 = 0;
};

inline void make_view(mp_context& ctx, const mp_csr* c, GraphView& gv) {
  if (!c) throw Error(MP_EINVAL, "null graph");
  if (c->n < 0) throw Error(MP_EINVAL, "negative vertex count");
  cudaStream_t s = ctx.stream;
  const int32_t n = c->n;
  if (c->on_device) {
    int32_t m2 = 0;
    MP_CUDA(cudaMemcpyAsync(&m2, c->offsets + n, 4, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    gv.g = {n, c->offsets, c->neighbors};
    gv.m2 = m2;
  } else {
    gv.m2 = c->offsets[n];
    gv.off.alloc(n + 1, s);
    gv.nbr.alloc(std::max<int64_t>(gv.m2, 1), s);
    MP_CUDA(cudaMemcpyAsync(gv.off.get(), c->offsets, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, s));
    if (gv.m2)
      MP_CUDA(cudaMemcpyAsync(gv.nbr.get(), c->neighbors, sizeof(int32_t) * gv.m2, cudaMemcpyHostToDevice, s));
    gv.g = {n, gv.off.get(), gv.nbr.get()};
  }
}

// Input array: device pointer as-is, or a device copy of host memory.
template <class T>
inline const T* input_ptr(mp_context& ctx, const T* p, int64_t count, bool on_device, DevBuf<T>& hold) {
  if (on_device || !p) return p;
  hold.alloc(std::max<int64_t>(count, 1), ctx.stream);
  if (count) MP_CUDA(cudaMemcpyAsync(hold.get(), p, sizeof(T) * count, cudaMemcpyHostToDevice, ctx.stream));
  return hold.get();
}

template <class T>
inline void output_copy(mp_context& ctx, T* dst, const T* src, int64_t count, bool on_device) {
  if (!dst || count == 0) return;
  MP_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * count,
                          on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx.stream));
}

// run_pipeline's patch stage (pipeline.cpp:101-114): compute_patches, or a
// user GroupMap validated and, when a patch is disconnected, split by
// enforce_connectivity.  Returns the patch count; asg (device, n) receives ids.
inline int32_t patch_stage(mp_context& ctx, const GraphView& gv, const mp_config* cfg, bool csr_on_device,
                           int32_t* asg) {
  const int32_t n = gv.g.n;
  if (!cfg->user_patches) return compute_patches_dev(ctx, gv.g, cfg->patch_size, cfg->seed, asg);
  DevBuf<int32_t> hold;
  const int32_t* user = input_ptr(ctx, cfg->user_patches, n, csr_on_device, hold);
  const UserPatchReport rep = validate_user_patches_dev(ctx, gv.g, user, cfg->user_patch_count);
  if (!rep.disconnected.empty()) return enforce_connectivity_dev(ctx, gv.g, user, cfg->user_patch_count, asg);
  if (n > 0) MP_CUDA(cudaMemcpyAsync(asg, user, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, ctx.stream));
  return cfg->user_patch_count;
}

}  // namespace mp
