// C ABI (include/meshperm_b200.h): context management, host<->device
// marshalling and the mp_order pipeline (reference run_pipeline ordering
// stages, core/src/pipeline.cpp:100-140).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "mp_context.h"
#include "mp_device.cuh"
#include "mp_host.h"

namespace mp {

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
SectionTimer::SectionTimer(cudaStream_t st, const char* sc) : s(st), scope(sc) {
  const char* e = getenv("MP_PROFILE");
  on = e && e[0] == '1';
  if (on) cudaStreamSynchronize(s);
  t0 = now_ms();
}
void SectionTimer::mark(const char* what) {
  if (!on) return;
  cudaStreamSynchronize(s);
  const double t = now_ms();
  fprintf(stderr, "[mp] %s/%s %.3f ms\n", scope, what, t - t0);
  t0 = t;
}

thread_local std::string g_last_error;
thread_local cudaMemPool_t tl_pool = nullptr;

cudaError_t dev_malloc_async(void** p, size_t bytes, cudaStream_t s) {
  return tl_pool ? cudaMallocFromPoolAsync(p, bytes, tl_pool, s) : cudaMallocAsync(p, bytes, s);
}

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int64_t unrelated_edges_dev(mp_context& ctx, const DGraph& g, const int32_t* node_of);

namespace {

// NVTX ranges (SURVEY §5 tracing): one per mp_order call plus one per stage,
// visible in Nsight Systems / ncu --nvtx; no-ops when no tool is attached.
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
// Consecutive stage ranges inside a call; balanced on every exit path.
struct NvtxStages {
  bool open = false;
  void next(const char* name) {
    end();
    nvtxRangePushA(name);
    open = true;
  }
  void end() {
    if (open) nvtxRangePop();
    open = false;
  }
  ~NvtxStages() { end(); }
};

// expand_blocks (assemble.cpp:87-114) for the tree, and the closed-form
// expansion of column counts / parents.
__global__ void expand_tree(int32_t n, int32_t b, const int32_t* verts, const int32_t* lperm, int32_t* verts_b,
                            int32_t* lperm_b) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int32_t t = 0; t < b; ++t) {
      if (verts_b) verts_b[static_cast<int64_t>(b) * i + t] = b * verts[i] + t;
      if (lperm_b) lperm_b[static_cast<int64_t>(b) * i + t] = b * lperm[i] + t;
    }
}
__global__ void scale_offsets(int32_t nn1, int32_t b, const int32_t* off, int32_t* out) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nn1; i += gridDim.x * blockDim.x) out[i] = b * off[i];
}
__global__ void expand_counts(int32_t n, int32_t b, const int64_t* cc, const int32_t* par, int64_t* cc_b,
                              int32_t* par_b, unsigned long long* sums) {
  __shared__ int64_t red[32];
  int64_t s = 0, q = 0;
  for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int64_t c = cc[k];
    for (int32_t t = 0; t < b; ++t) {
      const int64_t d = static_cast<int64_t>(b) * (c - 1) + (b - t);
      const int64_t pos = static_cast<int64_t>(b) * k + t;
      if (cc_b) cc_b[pos] = d;
      if (par_b) par_b[pos] = t + 1 < b ? static_cast<int32_t>(pos + 1) : (par[k] < 0 ? -1 : b * par[k]);
      s += d;
      q += d * d;
    }
  }
  s = block_sum_i64(s, red);
  q = block_sum_i64(q, red);
  if (threadIdx.x == 0) {
    atomicAdd(&sums[0], static_cast<unsigned long long>(s));
    atomicAdd(&sums[1], static_cast<unsigned long long>(q));
  }
}

int grid_for(const mp_context& ctx, int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), ctx.num_sms * 16LL)));
}


}  // namespace
}  // namespace mp

int mp_context::ktime_begin(int slot) {
  const size_t first = 2 * kev_used.size();
  while (kev.size() < first + 2) {
    cudaEvent_t e;
    MP_CUDA(cudaEventCreate(&e));
    kev.push_back(e);
  }
  MP_CUDA(cudaEventRecord(kev[first], stream));
  kev_used.push_back({slot, static_cast<int>(first)});
  return static_cast<int>(first);
}
void mp_context::ktime_end(int first) { MP_CUDA(cudaEventRecord(kev[first + 1], stream)); }

void* mp_context::slab(int id, size_t bytes) {
  if (static_cast<int>(slabs.size()) <= id) slabs.resize(id + 1, {nullptr, 0});
  auto& sl = slabs[id];
  if (sl.second < bytes) {
    if (sl.first) {
      MP_CUDA(cudaStreamSynchronize(stream));
      MP_CUDA(cudaFree(sl.first));
      sl = {nullptr, 0};
    }
    const size_t grow = bytes + bytes / 8;
    MP_CUDA(cudaMalloc(&sl.first, grow));
    sl.second = grow;
  }
  return sl.first;
}

using namespace mp;

extern "C" {

const char* mp_last_error(void) { return g_last_error.c_str(); }
const char* mp_version(void) { return "meshperm_b200 0.1 (sm_100a)"; }
int32_t mp_default_nd_level(int32_t n) { return default_nd_level_host(n); }

int mp_context_create(mp_context** out, int32_t device) {
  return guarded([&] {
    if (!out) throw Error(MP_EINVAL, "null context pointer");
    int count = 0;
    MP_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw Error(MP_EINVAL, "no CUDA device " + std::to_string(device));
    auto* ctx = new mp_context();
    ctx->device = device;
    ContextScope sd(*ctx);
    MP_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    MP_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    MP_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    MP_CUDA(cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    for (auto& e : ctx->ev) MP_CUDA(cudaEventCreate(&e));
    for (auto& e : ctx->fork_ev) MP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    MP_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->dwork), 16 * sizeof(unsigned long long)));
    MP_CUDA(cudaMemset(ctx->dwork, 0, 16 * sizeof(unsigned long long)));
    // a private stream-ordered pool that keeps freed scratch between calls;
    // the device's default pool (shared with the host application) is untouched
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    MP_CUDA(cudaMemPoolCreate(&ctx->pool, &props));
    uint64_t thr = UINT64_MAX;
    MP_CUDA(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = ctx;
  });
}

void mp_context_destroy(mp_context* ctx) {
  if (!ctx) return;
  ContextScope sd(*ctx);
  cudaStreamSynchronize(ctx->stream);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->kev) cudaEventDestroy(e);
  for (auto& e : ctx->fork_ev)
    if (e) cudaEventDestroy(e);
  for (auto& sl : ctx->slabs)
    if (sl.first) cudaFree(sl.first);
  if (ctx->dwork) cudaFree(ctx->dwork);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  delete ctx;
}

int mp_context_set_sm_share(mp_context* ctx, int32_t share) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    if (share < 1) throw Error(MP_EINVAL, "share must be positive");
    if (ctx->sm_share == share) return;  // keep the sizing decided for it
    ctx->sm_share = share;
    ctx->fps_workers = 0;  // re-decided on the next call
  });
}

int mp_context_set_fill_algorithm(mp_context* ctx, int32_t algo) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    if (algo != 0 && algo != 1) throw Error(MP_EINVAL, "fill algorithm must be 0 or 1");
    ctx->fill_algo = algo;
  });
}

int mp_context_set_tuning(mp_context* ctx, int32_t key, int64_t value) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    if (key < 0 || key >= MP_TUNE_COUNT) throw Error(MP_EINVAL, "unknown tuning key");
    ctx->tune[key] = value;
  });
}

int mp_context_set_stream(mp_context* ctx, void* stream) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  });
}

int mp_compute_patches(mp_context* ctx, const mp_csr* g, int32_t target, uint64_t seed, int32_t* assignment,
                       int32_t on_device, int32_t* patch_count) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    ContextScope sd(*ctx);
    GraphView gv;
    make_view(*ctx, g, gv);
    DevBuf<int32_t> asg(std::max(g->n, 1), ctx->stream);
    int32_t pc = compute_patches_dev(*ctx, gv.g, target, seed, asg);
    output_copy(*ctx, assignment, asg.get(), g->n, on_device);
    MP_CUDA(cudaStreamSynchronize(ctx->stream));
    *patch_count = pc;
  });
}

int mp_enforce_connectivity(mp_context* ctx, const mp_csr* g, const int32_t* assignment, int32_t patch_count,
                            int32_t* out, int32_t on_device, int32_t* out_count) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    ContextScope sd(*ctx);
    GraphView gv;
    make_view(*ctx, g, gv);
    DevBuf<int32_t> hold, res(std::max(g->n, 1), ctx->stream);
    const int32_t* in = input_ptr(*ctx, assignment, g->n, on_device != 0, hold);
    int32_t pc = enforce_connectivity_dev(*ctx, gv.g, in, patch_count, res);
    output_copy(*ctx, out, res.get(), g->n, on_device);
    MP_CUDA(cudaStreamSynchronize(ctx->stream));
    *out_count = pc;
  });
}

int mp_validate_user_patches(mp_context* ctx, const mp_csr* g, const int32_t* assignment, int32_t patch_count,
                             int64_t* patch_sizes, int32_t* disconnected, int32_t* n_disconnected,
                             int32_t* unused, int32_t* n_unused) {
  return guarded([&] {
    if (!ctx || !g || !n_disconnected || !n_unused || (g->n > 0 && !assignment)) throw Error(MP_EINVAL, "null argument");
    ContextScope sd(*ctx);
    GraphView gv;
    make_view(*ctx, g, gv);
    DevBuf<int32_t> hold;
    const int32_t* in = input_ptr(*ctx, assignment, g->n, g->on_device != 0, hold);
    const UserPatchReport r = validate_user_patches_dev(*ctx, gv.g, in, patch_count);
    if (patch_sizes) std::copy(r.sizes.begin(), r.sizes.end(), patch_sizes);
    if (disconnected) std::copy(r.disconnected.begin(), r.disconnected.end(), disconnected);
    if (unused) std::copy(r.unused.begin(), r.unused.end(), unused);
    *n_disconnected = static_cast<int32_t>(r.disconnected.size());
    *n_unused = static_cast<int32_t>(r.unused.size());
  });
}

int mp_build_quotient(mp_context* ctx, const mp_csr* g, const int32_t* assignment, int32_t patch_count,
                      int64_t* node_weight, int32_t* edge_p, int32_t* edge_q, int64_t* edge_w, int64_t* n_edges) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    ContextScope sd(*ctx);
    cudaStream_t s = ctx->stream;
    GraphView gv;
    make_view(*ctx, g, gv);
    DevBuf<int32_t> hold;
    const int32_t* in = input_ptr(*ctx, assignment, g->n, g->on_device != 0, hold);
    DevBuf<int64_t> nw(std::max(patch_count, 1), s);
    int32_t *ep = nullptr, *eq = nullptr;
    int64_t* ew = nullptr;
    int64_t U = build_quotient_dev(*ctx, gv.g, in, patch_count, nw, &ep, &eq, &ew);
    if (node_weight) output_copy(*ctx, node_weight, nw.get(), patch_count, false);
    if (edge_p) {
      output_copy(*ctx, edge_p, ep, U, false);
      output_copy(*ctx, edge_q, eq, U, false);
      output_copy(*ctx, edge_w, ew, U, false);
    }
    MP_CUDA(cudaStreamSynchronize(s));
    cudaFreeAsync(ep, s), cudaFreeAsync(eq, s), cudaFreeAsync(ew, s);
    *n_edges = U;
  });
}

int mp_build_etree(mp_context* ctx, const mp_csr* g, const int32_t* assignment, int32_t patch_count,
                   int32_t nd_level, uint64_t seed, int32_t* node_offsets, int32_t* node_vertices, int32_t on_device) {
  (void)seed;  // bipartition_quotient ignores it (partition.cpp:27)
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    ContextScope sd(*ctx);
    cudaStream_t s = ctx->stream;
    GraphView gv;
    make_view(*ctx, g, gv);
    DevBuf<int32_t> hold;
    const int32_t* in = input_ptr(*ctx, assignment, g->n, g->on_device != 0, hold);
    const int64_t nn = (1LL << (nd_level + 1)) - 1;
    DevBuf<int32_t> node_of(std::max(g->n, 1), s), off(nn + 1, s), verts(std::max(g->n, 1), s);
    build_etree_dev(*ctx, gv.g, in, patch_count, nd_level, node_of, off, verts);
    output_copy(*ctx, node_offsets, off.get(), nn + 1, on_device);
    output_copy(*ctx, node_vertices, verts.get(), g->n, on_device);
    MP_CUDA(cudaStreamSynchronize(s));
  });
}

int mp_order_tree_nodes(mp_context* ctx, const mp_csr* g, int32_t nd_level, const int32_t* node_offsets,
                        const int32_t* node_vertices, int32_t mode, int32_t* local_perm, int32_t on_device) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    if (mode < 0 || mode > 2) throw Error(MP_EINVAL, "unknown local ordering mode");
    ContextScope sd(*ctx);
    cudaStream_t s = ctx->stream;
    GraphView gv;
    make_view(*ctx, g, gv);
    const int32_t nn = static_cast<int32_t>((1LL << (nd_level + 1)) - 1);
    DevBuf<int32_t> h1, h2, node_of(std::max(g->n, 1), s), lp(std::max(g->n, 1), s);
    const int32_t* off = input_ptr(*ctx, node_offsets, nn + 1, on_device != 0, h1);
    const int32_t* verts = input_ptr(*ctx, node_vertices, g->n, on_device != 0, h2);
    node_of_from_tree_dev(*ctx, g->n, nn, off, verts, node_of);
    order_tree_nodes_dev(*ctx, gv.g, nd_level, node_of, off, verts, mode, lp);
    output_copy(*ctx, local_perm, lp.get(), g->n, on_device);
    MP_CUDA(cudaStreamSynchronize(s));
  });
}

int mp_order_subtrees(mp_context* ctx, const mp_csr* g, int32_t nd_level, const int32_t* node_offsets,
                      const int32_t* node_vertices, int32_t mode, int32_t schedule, const uint8_t* node_mask,
                      int32_t* local_perm, int32_t* perm, int32_t on_device) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    if (mode < 0 || mode > 2) throw Error(MP_EINVAL, "unknown local ordering mode");
    if (!node_mask || !local_perm || !perm) throw Error(MP_EINVAL, "null node_mask / local_perm / perm");
    ContextScope sd(*ctx);
    cudaStream_t s = ctx->stream;
    GraphView gv;
    make_view(*ctx, g, gv);
    const int32_t n = g->n;
    const int32_t nn = static_cast<int32_t>((1LL << (nd_level + 1)) - 1);
    DevBuf<int32_t> h1, h2, node_of(std::max(n, 1), s);
    DevBuf<uint8_t> h3;
    const int32_t* off = input_ptr(*ctx, node_offsets, nn + 1, on_device != 0, h1);
    const int32_t* verts = input_ptr(*ctx, node_vertices, n, on_device != 0, h2);
    const uint8_t* mask = input_ptr(*ctx, node_mask, nn, on_device != 0, h3);
    // outputs: entries of unmasked nodes are left as the caller had them
    DevBuf<int32_t> lp_h, pm_h;
    int32_t* lp = local_perm;
    int32_t* pm = perm;
    if (!on_device) {
      lp_h.alloc(std::max(n, 1), s);
      pm_h.alloc(std::max(n, 1), s);
      MP_CUDA(cudaMemcpyAsync(lp_h.get(), local_perm, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
      MP_CUDA(cudaMemcpyAsync(pm_h.get(), perm, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
      lp = lp_h, pm = pm_h;
    }
    node_of_from_tree_dev(*ctx, n, nn, off, verts, node_of);
    order_tree_nodes_dev(*ctx, gv.g, nd_level, node_of, off, verts, mode, lp, mask);
    compute_perm_partial_dev(*ctx, n, nd_level, off, verts, lp, resolve_schedule(nd_level, schedule, nullptr, 0), mask, pm);
    if (!on_device) {
      MP_CUDA(cudaMemcpyAsync(local_perm, lp, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaMemcpyAsync(perm, pm, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    }
    MP_CUDA(cudaStreamSynchronize(s));
  });
}

int mp_compute_perm_schedule(mp_context* ctx, int32_t n, int32_t nd_level, const int32_t* node_offsets,
                             const int32_t* node_vertices, const int32_t* local_perm, const int32_t* schedule_nodes,
                             int64_t schedule_len, int32_t* perm, int32_t* inverse, int32_t on_device) {
  return guarded([&] {
    if (!ctx) throw Error(MP_EINVAL, "null context");
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    if (!schedule_nodes) throw Error(MP_EINVAL, "null schedule");
    ContextScope sd(*ctx);
    const Schedule sched = resolve_schedule(nd_level, 0, schedule_nodes, schedule_len);
    cudaStream_t s = ctx->stream;
    const int32_t nn = static_cast<int32_t>((1LL << (nd_level + 1)) - 1);
    DevBuf<int32_t> h1, h2, h3, pm(std::max(n, 1), s), inv(std::max(n, 1), s), pos(nn + 1, s);
    const int32_t* off = input_ptr(*ctx, node_offsets, nn + 1, on_device != 0, h1);
    const int32_t* verts = input_ptr(*ctx, node_vertices, n, on_device != 0, h2);
    const int32_t* lp = input_ptr(*ctx, local_perm, n, on_device != 0, h3);
    compute_perm_dev(*ctx, n, nd_level, off, verts, lp, sched, pm, inv, pos);
    output_copy(*ctx, perm, pm.get(), n, on_device);
    output_copy(*ctx, inverse, inv.get(), n, on_device);
    MP_CUDA(cudaStreamSynchronize(s));
  });
}

int mp_compute_perm(mp_context* ctx, int32_t n, int32_t nd_level, const int32_t* node_offsets,
                    const int32_t* node_vertices, const int32_t* local_perm, int32_t schedule, int32_t* perm,
                    int32_t* inverse, int32_t on_device) {
  if (nd_level < 0 || nd_level > 24) return set_error(MP_EINVAL, "nd_level out of range");
  if (schedule != MP_SCHEDULE_POSTORDER && schedule != MP_SCHEDULE_LEVELORDER)
    return set_error(MP_EINVAL, "unknown schedule");
  const Schedule sched = make_schedule(nd_level, schedule);
  return mp_compute_perm_schedule(ctx, n, nd_level, node_offsets, node_vertices, local_perm, sched.data(),
                                  static_cast<int64_t>(sched.size()), perm, inverse, on_device);
}

int mp_validate_schedule(int32_t nd_level, const int32_t* sequence, int64_t length, int64_t* first_violation) {
  return guarded([&] {
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    if (!first_violation || (length > 0 && !sequence) || length < 0) throw Error(MP_EINVAL, "null argument");
    *first_violation = validate_schedule_host(nd_level, sequence, length);
  });
}

int mp_tree_fill_schedule(mp_context* ctx, const mp_csr* g, int32_t nd_level, const int32_t* node_offsets,
                          const int32_t* node_vertices, const int32_t* local_perm, const int32_t* schedule_nodes,
                          int64_t schedule_len, int64_t* column_counts, int32_t* etree_parent, int32_t on_device,
                          int64_t* nnz_A, int64_t* nnz_L, int64_t* cost, double* fill_ratio) {
  return guarded([&] {
    if (!ctx || !g) throw Error(MP_EINVAL, "null argument");
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    if (!schedule_nodes) throw Error(MP_EINVAL, "null schedule");
    ContextScope sd(*ctx);
    const Schedule sched = resolve_schedule(nd_level, 0, schedule_nodes, schedule_len);
    cudaStream_t s = ctx->stream;
    GraphView gv;
    make_view(*ctx, g, gv);
    const int32_t n = g->n;
    const int32_t nn = static_cast<int32_t>((1LL << (nd_level + 1)) - 1);
    DevBuf<int32_t> h1, h2, h3, node_of(std::max(n, 1), s), pm(std::max(n, 1), s), inv(std::max(n, 1), s),
        pos(nn + 1, s), par(std::max(n, 1), s);
    DevBuf<int64_t> cc(std::max(n, 1), s);
    const int32_t* off = input_ptr(*ctx, node_offsets, nn + 1, on_device != 0, h1);
    const int32_t* verts = input_ptr(*ctx, node_vertices, n, on_device != 0, h2);
    const int32_t* lp = input_ptr(*ctx, local_perm, n, on_device != 0, h3);
    compute_perm_dev(*ctx, n, nd_level, off, verts, lp, sched, pm, inv, pos);
    node_of_from_tree_dev(*ctx, n, nn, off, verts, node_of);
    int64_t L = 0, C = 0;
    // a caller's tree whose separators leak: the game on the permutation itself
    // (the node-by-node split needs separated subtrees)
    if (unrelated_edges_dev(*ctx, gv.g, node_of) == 0)
      tree_fill_dev(*ctx, gv.g, nd_level, node_of, off, verts, lp, pos, inv, cc, par, &L, &C);
    else
      elimination_game_dev(*ctx, gv.g, pm, cc, par, &L, &C, nullptr, nullptr);
    output_copy(*ctx, column_counts, cc.get(), n, on_device);
    output_copy(*ctx, etree_parent, par.get(), n, on_device);
    MP_CUDA(cudaStreamSynchronize(s));
    const int64_t A = static_cast<int64_t>(n) + gv.m2;
    if (nnz_A) *nnz_A = A;
    if (nnz_L) *nnz_L = L;
    if (cost) *cost = C;
    if (fill_ratio) *fill_ratio = A > 0 ? static_cast<double>(L) / static_cast<double>(A) : 0.0;
  });
}

int mp_tree_fill(mp_context* ctx, const mp_csr* g, int32_t nd_level, const int32_t* node_offsets,
                 const int32_t* node_vertices, const int32_t* local_perm, int32_t schedule, int64_t* column_counts,
                 int32_t* etree_parent, int32_t on_device, int64_t* nnz_A, int64_t* nnz_L, int64_t* cost,
                 double* fill_ratio) {
  if (nd_level < 0 || nd_level > 24) return set_error(MP_EINVAL, "nd_level out of range");
  if (schedule != MP_SCHEDULE_POSTORDER && schedule != MP_SCHEDULE_LEVELORDER)
    return set_error(MP_EINVAL, "unknown schedule");
  const Schedule sched = make_schedule(nd_level, schedule);
  return mp_tree_fill_schedule(ctx, g, nd_level, node_offsets, node_vertices, local_perm, sched.data(),
                               static_cast<int64_t>(sched.size()), column_counts, etree_parent, on_device, nnz_A,
                               nnz_L, cost, fill_ratio);
}

int mp_elimination_fill(mp_context* ctx, const mp_csr* g, const int32_t* perm, int64_t* column_counts,
                        int32_t* etree_parent, int32_t on_device, int64_t* nnz_A, int64_t* nnz_L, int64_t* cost,
                        double* fill_ratio) {
  return guarded([&] {
    if (!ctx || !g || (g->n > 0 && !perm)) throw Error(MP_EINVAL, "null argument");
    ContextScope sd(*ctx);
    cudaStream_t s = ctx->stream;
    GraphView gv;
    make_view(*ctx, g, gv);
    const int32_t n = g->n;
    DevBuf<int32_t> hp, par(std::max(n, 1), s);
    DevBuf<int64_t> cc(std::max(n, 1), s);
    const int32_t* pm = input_ptr(*ctx, perm, n, on_device != 0, hp);
    int64_t L = 0, C = 0;
    elimination_game_dev(*ctx, gv.g, pm, cc, par, &L, &C, nullptr, nullptr);
    output_copy(*ctx, column_counts, cc.get(), n, on_device);
    output_copy(*ctx, etree_parent, par.get(), n, on_device);
    MP_CUDA(cudaStreamSynchronize(s));
    const int64_t A = static_cast<int64_t>(n) + gv.m2;  // symbolic.cpp:22-29 finish
    if (nnz_A) *nnz_A = A;
    if (nnz_L) *nnz_L = L;
    if (cost) *cost = C;
    if (fill_ratio) *fill_ratio = A > 0 ? static_cast<double>(L) / static_cast<double>(A) : 0.0;
  });
}

int mp_cross_block_fill(mp_context* ctx, const mp_csr* g, const int32_t* perm, int32_t nd_level,
                        const int32_t* node_offsets, const int32_t* node_vertices, int32_t on_device,
                        int64_t* crossing) {
  return guarded([&] {
    if (!ctx || !g || !crossing || (g->n > 0 && !perm) || !node_offsets) throw Error(MP_EINVAL, "null argument");
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    ContextScope sd(*ctx);
    cudaStream_t s = ctx->stream;
    GraphView gv;
    make_view(*ctx, g, gv);
    const int32_t n = g->n;
    const int32_t nn = static_cast<int32_t>((1LL << (nd_level + 1)) - 1);
    DevBuf<int32_t> hp, h1, h2, owner(std::max(n, 1), s), par(std::max(n, 1), s);
    DevBuf<int64_t> cc(std::max(n, 1), s);
    const int32_t* pm = input_ptr(*ctx, perm, n, on_device != 0, hp);
    const int32_t* off = input_ptr(*ctx, node_offsets, nn + 1, on_device != 0, h1);
    const int32_t* verts = input_ptr(*ctx, node_vertices, n, on_device != 0, h2);
    // tree.n != g.n (symbolic.cpp:102-103) shows up as offsets not covering n
    node_of_from_tree_dev(*ctx, n, nn, off, verts, owner);
    int64_t L = 0, C = 0, X = 0;
    elimination_game_dev(*ctx, gv.g, pm, cc, par, &L, &C, owner, &X);
    *crossing = X;
  });
}

// run_pipeline's ordering stages (pipeline.cpp:100-140) on a device CSR.
int mp_order(mp_context* ctx, const mp_csr* g, const mp_config* cfg, mp_result* out) {
  return guarded([&] {
    if (!ctx || !g || !cfg || !out) throw Error(MP_EINVAL, "null argument");
    if (cfg->block_size < 1) throw Error(MP_EINVAL, "block size must be positive");
    if (cfg->patch_size < 1) throw Error(MP_EINVAL, "patch size must be positive");
    if (cfg->local_mode < 0 || cfg->local_mode > 2) throw Error(MP_EINVAL, "unknown local ordering mode");
    if (!cfg->schedule_nodes && (cfg->schedule < 0 || cfg->schedule > 1)) throw Error(MP_EINVAL, "unknown schedule");
    ContextScope sd(*ctx);
    cudaStream_t s = ctx->stream;
    const int64_t launches0 = ctx->launches;
    const int32_t n = g->n, b = cfg->block_size;
    const int32_t L = cfg->nd_level >= 0 ? cfg->nd_level : default_nd_level_host(n);
    if (L > 24) throw Error(MP_EINVAL, "nd_level out of range");
    const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
    const int64_t N = static_cast<int64_t>(b) * n;
    // schedule_postorder / schedule_levelorder, or the caller's node sequence
    // validated up front like compute_perm does (assemble.cpp:71-72)
    const Schedule sched = resolve_schedule(L, cfg->schedule, cfg->schedule_nodes, cfg->schedule_len);

    ctx->ktime_reset();
    MP_CUDA(cudaMemsetAsync(ctx->dwork, 0, 16 * sizeof(unsigned long long), s));
    NvtxScope call_range("mp_order");
    NvtxStages stage;
    MP_CUDA(cudaEventRecord(ctx->ev[0], s));
    GraphView gv;
    make_view(*ctx, g, gv);
    DevBuf<int32_t> asg(std::max(n, 1), s), node_of(std::max(n, 1), s), off(nn + 1, s), verts(std::max(n, 1), s),
        lp(std::max(n, 1), s), pm(std::max<int64_t>(N, 1), s), inv(std::max<int64_t>(N, 1), s), pos(nn + 1, s);
    MP_CUDA(cudaEventRecord(ctx->ev[1], s));
    stage.next("mp_order/patch");
    const int32_t pc = patch_stage(*ctx, gv, cfg, g->on_device != 0, asg);
    MP_CUDA(cudaEventRecord(ctx->ev[2], s));
    stage.next("mp_order/quotient");
    // the per-level quotient is rebuilt inside the level loop (ndtree.cu), so
    // the quotient stage has no separate launch; its time is part of etree
    MP_CUDA(cudaEventRecord(ctx->ev[3], s));
    stage.next("mp_order/etree");
    build_etree_dev(*ctx, gv.g, asg, pc, L, node_of, off, verts);
    MP_CUDA(cudaEventRecord(ctx->ev[4], s));
    stage.next("mp_order/local");
    order_tree_nodes_dev(*ctx, gv.g, L, node_of, off, verts, cfg->local_mode, lp);
    MP_CUDA(cudaEventRecord(ctx->ev[5], s));
    stage.next("mp_order/assemble");
    DevBuf<int32_t> pm1, inv1;
    if (b == 1) {
      compute_perm_blocks_dev(*ctx, n, L, off, verts, lp, sched, 1, pm, inv, pos);
    } else {
      pm1.alloc(std::max(n, 1), s);
      inv1.alloc(std::max(n, 1), s);
      compute_perm_blocks_dev(*ctx, n, L, off, verts, lp, sched, 1, pm1, inv1, pos);
      compute_perm_blocks_dev(*ctx, n, L, off, verts, lp, sched, b, pm, inv, pos);
    }
    MP_CUDA(cudaEventRecord(ctx->ev[6], s));
    stage.next("mp_order/symbolic");
    int64_t nnzL = 0, cost = 0;
    DevBuf<int64_t> cc;
    DevBuf<int32_t> par;
    if (cfg->want_fill) {
      cc.alloc(std::max<int64_t>(N, 1), s);
      par.alloc(std::max<int64_t>(N, 1), s);
      if (b == 1) {
        tree_fill_dev(*ctx, gv.g, L, node_of, off, verts, lp, pos, inv, cc, par, &nnzL, &cost);
      } else {
        DevBuf<int64_t> cc1(std::max(n, 1), s);
        DevBuf<int32_t> par1(std::max(n, 1), s);
        DevBuf<unsigned long long> sums(2, s);
        int64_t l1 = 0, c1 = 0;
        tree_fill_dev(*ctx, gv.g, L, node_of, off, verts, lp, pos, inv1, cc1, par1, &l1, &c1);
        MP_CUDA(cudaMemsetAsync(sums, 0, 16, s));
        MP_KERNEL(*ctx, expand_counts<<<grid_for(*ctx, n), 256, 0, s>>>(n, b, cc1, par1, cc, par, sums));
        unsigned long long h[2];
        MP_CUDA(cudaMemcpyAsync(h, sums, 16, cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        nnzL = static_cast<int64_t>(h[0]);
        cost = static_cast<int64_t>(h[1]);
      }
    }
    MP_CUDA(cudaEventRecord(ctx->ev[7], s));
    stage.end();
    // the pipeline's self-check (pipeline.cpp:141-142), untimed like the reference's
    if (unrelated_edges_dev(*ctx, gv.g, node_of) != 0)
      throw Error(MP_ELOGIC, "separator failed to disconnect its sides");
    // outputs
    const bool od = out->on_device != 0;
    output_copy(*ctx, out->patch_of, asg.get(), n, od);
    if (b == 1) {
      output_copy(*ctx, out->tree_node_offsets, off.get(), nn + 1, od);
      output_copy(*ctx, out->tree_vertices, verts.get(), n, od);
      output_copy(*ctx, out->tree_local_perm, lp.get(), n, od);
    } else {
      DevBuf<int32_t> offb(nn + 1, s), vb(N, s), lpb(N, s);
      MP_KERNEL(*ctx, scale_offsets<<<grid_for(*ctx, nn + 1), 256, 0, s>>>(nn + 1, b, off, offb));
      MP_KERNEL(*ctx, expand_tree<<<grid_for(*ctx, n), 256, 0, s>>>(n, b, verts, lp, vb, lpb));
      output_copy(*ctx, out->tree_node_offsets, offb.get(), nn + 1, od);
      output_copy(*ctx, out->tree_vertices, vb.get(), N, od);
      output_copy(*ctx, out->tree_local_perm, lpb.get(), N, od);
      MP_CUDA(cudaStreamSynchronize(s));
    }
    output_copy(*ctx, out->perm, pm.get(), N, od);
    output_copy(*ctx, out->inverse, inv.get(), N, od);
    if (cfg->want_fill) {
      output_copy(*ctx, out->column_counts, cc.get(), N, od);
      output_copy(*ctx, out->etree_parent, par.get(), N, od);
    }
    MP_CUDA(cudaStreamSynchronize(s));
    out->patch_count = pc;
    out->nd_level = L;
    // nnz_A of the measured system: b^2 (n + 2m) (pipeline.cpp:174-175 on expand_graph)
    out->nnz_A = static_cast<int64_t>(b) * b * (n + gv.m2);
    out->nnz_L = nnzL;
    out->cost = cost;
    out->fill_ratio = out->nnz_A > 0 ? static_cast<double>(nnzL) / static_cast<double>(out->nnz_A) : 0.0;
    float ms = 0;
    const int pairs[6][2] = {{1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 7}};
    for (int i = 0; i < 6; ++i) {
      MP_CUDA(cudaEventElapsedTime(&ms, ctx->ev[pairs[i][0]], ctx->ev[pairs[i][1]]));
      out->stage_ms[i] = ms;
    }
    if (!cfg->want_fill) out->stage_ms[5] = 0;
    for (int i = 0; i < kKSlots; ++i) out->kernel_ms[i] = 0;
    for (auto& [slot, first] : ctx->kev_used) {
      MP_CUDA(cudaEventElapsedTime(&ms, ctx->kev[first], ctx->kev[first + 1]));
      out->kernel_ms[slot] += ms;
    }
    out->kernel_launches = ctx->launches - launches0;
    unsigned long long hw[16];
    MP_CUDA(cudaMemcpy(hw, ctx->dwork, sizeof hw, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 16; ++i) out->work[i] = static_cast<int64_t>(hw[i]);
  });
}

}  // extern "C"
