// Device-side helpers shared by the kernels: error checks, packed keys,
// warp/block reductions, stream-ordered scratch allocation.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_set>

#include "mp_internal.h"

namespace cg = cooperative_groups;

#define MP_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t err__ = (call);                                                           \
    if (err__ != cudaSuccess)                                                             \
      throw mp::Error(err__ == cudaErrorMemoryAllocation ? MP_ENOMEM : MP_ECUDA,          \
                      std::string(#call) + ": " + cudaGetErrorString(err__));             \
  } while (0)

#define MP_LAUNCH_CHECK() MP_CUDA(cudaGetLastError())

namespace mp {

constexpr int32_t kUnreached = 0x7fffffff;
constexpr int32_t kNone = -1;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// (value asc, id asc) packed so that the numeric MIN is the wanted element.
__device__ __forceinline__ uint64_t key_min(uint32_t value, uint32_t id) {
  return (static_cast<uint64_t>(value) << 32) | id;
}
// (value desc, id asc) packed so that the numeric MAX is the wanted element.
__device__ __forceinline__ uint64_t key_max(uint32_t value, uint32_t id) {
  return (static_cast<uint64_t>(value) << 32) | (0xffffffffu - id);
}
__device__ __forceinline__ uint32_t key_max_id(uint64_t k) {
  return 0xffffffffu - static_cast<uint32_t>(k & 0xffffffffu);
}

// 64-bit warp max/min as two 32-bit redux.sync steps (high word, then the
// low word among the lanes holding the winning high word); full warp only.
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return (static_cast<uint64_t>(mh) << 32) | ml;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  const uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
  const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
  return (static_cast<uint64_t>(mh) << 32) | ml;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide reductions; `red` is >= 32 u64 of shared scratch.  All threads
// receive the result.  Two barriers.
__device__ __forceinline__ uint64_t block_max_u64(uint64_t v, uint64_t* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max_u64(v);
  if (lane == 0) red[wid] = v;
  __syncthreads();
  uint64_t r = lane < nw ? red[lane] : 0;
  r = warp_max_u64(r);
  __syncthreads();
  return r;
}
__device__ __forceinline__ uint64_t block_min_u64(uint64_t v, uint64_t* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_min_u64(v);
  if (lane == 0) red[wid] = v;
  __syncthreads();
  uint64_t r = lane < nw ? red[lane] : ~0ull;
  r = warp_min_u64(r);
  __syncthreads();
  return r;
}
__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum_i64(v);
  if (lane == 0) red[wid] = v;
  __syncthreads();
  int64_t r = lane < nw ? red[lane] : 0;
  r = warp_sum_i64(r);
  __syncthreads();
  return r;
}

// Exclusive block scan of int32 (returns this thread's exclusive prefix, and
// the block total through *total).  `sh` holds >= 32 ints.
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* sh, int32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int32_t s = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh[lane] = s;
  }
  __syncthreads();
  int32_t base = wid > 0 ? sh[wid - 1] : 0;
  *total = sh[nw - 1];
  __syncthreads();
  return base + x - v;
}

// Warp-aggregated append: one atomic per warp; every lane of the warp must
// call it (pred may differ).  Returns the slot for predicated lanes, else -1.
__device__ __forceinline__ int32_t warp_append(int32_t* counter, bool pred) {
  const uint32_t mask = __ballot_sync(0xffffffffu, pred);
  if (!mask) return -1;
  const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
  int32_t base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  return pred ? base + __popc(mask & ((1u << lane) - 1)) : -1;
}

// IEEE double imbalance ratio, partition.cpp:15-21.  Division is the
// correctly rounded __ddiv_rn regardless of compiler flags.
__device__ __forceinline__ double imbalance_of(int64_t a, int64_t b) {
  if (a == 0 && b == 0) return 1.0;
  if (a == 0 || b == 0) return __longlong_as_double(0x7ff0000000000000ll);
  int64_t hi = a > b ? a : b, lo = a < b ? a : b;
  return __ddiv_rn(static_cast<double>(hi), static_cast<double>(lo));
}

// Is tree node a an ancestor of (or equal to) b?  etree.cpp:27 semantics.
__host__ __device__ inline bool is_ancestor_or_self(int32_t a, int32_t b) {
  while (b > a) b = (b - 1) / 2;
  return b == a;
}
__host__ __device__ inline int32_t tree_level(int32_t idx) {
  int32_t l = 0;
  for (uint32_t x = static_cast<uint32_t>(idx) + 1; x > 1; x >>= 1) ++l;
  return l;
}

// Raise a kernel's dynamic shared memory limit to the device maximum, once
// per kernel.  The attribute is process-wide, so it is never sized per call:
// concurrent contexts (FramePool threads) launching the same kernel with
// different dynamic sizes would otherwise race on it.
template <class K>
inline void allow_max_smem(K* kernel, int device) {
  static std::mutex mu;
  static std::unordered_set<uint64_t> done;
  const uint64_t key = reinterpret_cast<uint64_t>(reinterpret_cast<const void*>(kernel)) ^ (uint64_t(device) << 56);
  std::lock_guard<std::mutex> g(mu);
  if (done.count(key)) return;
  int optin = 0;
  MP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  cudaFuncAttributes fa{};
  MP_CUDA(cudaFuncGetAttributes(&fa, kernel));
  MP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               optin - static_cast<int>(fa.sharedSizeBytes)));
  done.insert(key);
}

// Stream-ordered allocation from the calling entry point's context pool
// (ContextScope), else from the device's current pool.
cudaError_t dev_malloc_async(void** p, size_t bytes, cudaStream_t s);

// Stream-ordered scratch buffer (cudaMallocAsync from the context pool).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) MP_CUDA(dev_malloc_async(reinterpret_cast<void**>(&p), sizeof(T) * count, st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr, o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p, n = o.n, s = o.s;
    o.p = nullptr, o.n = 0;
    return *this;
  }
  T* get() const { return p; }
  operator T*() const { return p; }
};

// Several arrays carved out of one persistent context slab (mp_context::slab):
// the large per-call scratch of a stage lives there, so repeated calls neither
// allocate nor fragment the stream-ordered pool.
struct SlabCarve {
  size_t total = 0;
  size_t add(size_t bytes) {
    const size_t at = total;
    total += (bytes + 255) & ~size_t(255);
    return at;
  }
  template <class T>
  static T* at(void* base, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(base) + off);
  }
};

}  // namespace mp
