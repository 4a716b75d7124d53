// Multi-GPU ordering of one very large mesh (BASELINE configs[2] "C3",
// SURVEY §8e): mp_order_sharded and the NCCL plumbing of mp_comm.
//
// The reference orders one mesh on one host (run_pipeline, pipeline.cpp:
// 100-140); its only parallel stage is order_tree_nodes' thread fan-out over
// independent tree nodes (local_order.cpp:77-86).  Subtrees of the ND tree are
// independent beyond that: sibling subtrees own disjoint patches, no edge
// joins two of them (the separator property), quotient updates stay inside a
// subtree (quotient.cpp:94), and in the elimination game a finished subtree
// is visible to the rest only through its live elements.  So, per rank:
//
//   patches + top k = ceil(log2 world) ND levels   replicated (sequential chains)
//   level-k subtrees dealt by size                  deal_subtrees (ndtree.cu)
//   own subtrees: ND levels k..L-1, MD, fill game   this rank only
//   all-gather 1: node sizes                        -> global tree offsets
//   all-gather 2: own nodes' vertices + local order -> global tree, perm, inverse
//   all-gather 3: own level-k roots' live elements  -> every rank plays the top
//   all-gather 4: own positions' column counts / parents -> nnz(L)
//
// Every output equals mp_order's bit for bit, at any world size.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "mp_context.h"
#include "mp_device.cuh"
#include "mp_host.h"

namespace mp {

int64_t unrelated_edges_dev(mp_context& ctx, const DGraph& g, const int32_t* node_of);

namespace {

// ---------------------------------------------------------------- NCCL (dlopen)
using ncclResult_t = int;
using ncclComm_t = void*;
struct ncclUniqueId {
  char internal[128];
};
constexpr int kNcclInt8 = 0;

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_gather)
      err = "libnccl.so.2 lacks the expected entry points";
  });
  if (!err.empty()) throw Error(MP_ECUDA, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* m = nccl().error_string ? nccl().error_string(r) : "error";
    throw Error(MP_ECUDA, std::string(what) + ": " + m);
  }
}

// mp_comm.allgather of the library's NCCL communicator (device buffers)
int nccl_allgather(void* user, const void* send, void* recv, int64_t bytes, void* stream) {
  const ncclResult_t r = nccl().all_gather(send, recv, static_cast<size_t>(bytes), kNcclInt8,
                                           static_cast<ncclComm_t>(user), static_cast<cudaStream_t>(stream));
  if (r != 0) return set_error(MP_ECUDA, std::string("ncclAllGather: ") +
                                             (nccl().error_string ? nccl().error_string(r) : "error"));
  return MP_OK;
}

// ---------------------------------------------------------------- all-gathers
class Exchange {
 public:
  Exchange(mp_context& ctx, const mp_comm& c) : ctx_(ctx), c_(c) {}
  int32_t world() const { return c_.world; }

  // fixed-size all-gather of host data (world * mine.size() back)
  template <class T>
  std::vector<T> host(const std::vector<T>& mine) {
    const int64_t bytes = static_cast<int64_t>(sizeof(T) * mine.size());
    std::vector<T> all(mine.size() * c_.world);
    if (c_.world == 1) return mine;
    if (!c_.device_buffers) {
      call(mine.data(), all.data(), bytes);
      return all;
    }
    cudaStream_t s = ctx_.stream;
    DevBuf<char> ds(std::max<int64_t>(bytes, 1), s), dr(std::max<int64_t>(bytes * c_.world, 1), s);
    if (bytes) MP_CUDA(cudaMemcpyAsync(ds.get(), mine.data(), bytes, cudaMemcpyHostToDevice, s));
    call(ds.get(), dr.get(), bytes);
    if (bytes) MP_CUDA(cudaMemcpyAsync(all.data(), dr.get(), bytes * c_.world, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    return all;
  }

  // variable-size all-gather of host int32 data: rank r's vector, in rank order
  std::vector<std::vector<int32_t>> hostv(const std::vector<int32_t>& mine) {
    const std::vector<int64_t> len = host(std::vector<int64_t>{static_cast<int64_t>(mine.size())});
    const int64_t width = *std::max_element(len.begin(), len.end());
    std::vector<int32_t> pad(mine);
    pad.resize(width, 0);
    const std::vector<int32_t> all = host(pad);
    std::vector<std::vector<int32_t>> out(c_.world);
    for (int32_t r = 0; r < c_.world; ++r) out[r].assign(all.begin() + r * width, all.begin() + r * width + len[r]);
    return out;
  }

  // fixed-size all-gather of device data: recv (world * bytes) on the device
  void device(const void* send, void* recv, int64_t bytes) {
    cudaStream_t s = ctx_.stream;
    if (c_.world == 1) {
      if (bytes) MP_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
      return;
    }
    if (c_.device_buffers) {
      call(send, recv, bytes);
      return;
    }
    std::vector<char> hs(bytes), hr(bytes * c_.world);
    if (bytes) MP_CUDA(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    call(hs.data(), hr.data(), bytes);
    if (bytes) MP_CUDA(cudaMemcpyAsync(recv, hr.data(), bytes * c_.world, cudaMemcpyHostToDevice, s));
    MP_CUDA(cudaStreamSynchronize(s));
  }

 private:
  void call(const void* send, void* recv, int64_t bytes) {
    if (c_.device_buffers) MP_CUDA(cudaStreamSynchronize(ctx_.stream));  // inputs complete (foreign streams)
    const int rc = c_.allgather(c_.user, send, recv, bytes, ctx_.stream);
    if (rc != MP_OK) throw Error(rc, std::string("all-gather failed: ") + mp_last_error());
    if (c_.device_buffers) MP_CUDA(cudaStreamSynchronize(ctx_.stream));
  }
  mp_context& ctx_;
  const mp_comm& c_;
};

// ---------------------------------------------------------------- segment copies
struct Seg {
  int64_t src, dst, len;
};

template <class T>
__global__ void copy_segments(int32_t nseg, const Seg* seg, const T* src, T* dst) {
  for (int32_t i = blockIdx.x; i < nseg; i += gridDim.x) {
    const Seg sg = seg[i];
    for (int64_t j = threadIdx.x; j < sg.len; j += blockDim.x) dst[sg.dst + j] = src[sg.src + j];
  }
}

template <class T>
void copy_segs(mp_context& ctx, const std::vector<Seg>& segs, const T* src, T* dst) {
  if (segs.empty()) return;
  cudaStream_t s = ctx.stream;
  DevBuf<Seg> d(segs.size(), s);
  MP_CUDA(cudaMemcpyAsync(d.get(), segs.data(), sizeof(Seg) * segs.size(), cudaMemcpyHostToDevice, s));
  const int32_t ns = static_cast<int32_t>(segs.size());
  MP_KERNEL(ctx, copy_segments<T><<<std::min(ns, 4096), 256, 0, s>>>(ns, d.get(), src, dst));
  MP_CUDA(cudaStreamSynchronize(s));  // the host table is released on return
}

int32_t ceil_log2(int32_t w) {
  int32_t k = 0;
  while ((1 << k) < w) ++k;
  return k;
}

}  // namespace
}  // namespace mp

using namespace mp;

extern "C" {

int mp_nccl_get_unique_id(uint8_t id[128]) {
  return guarded([&] {
    if (!id) throw Error(MP_EINVAL, "null id");
    ncclUniqueId u{};
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
  });
}

int mp_nccl_comm_init(mp_comm* comm, const uint8_t id[128], int32_t world, int32_t rank, int32_t device) {
  return guarded([&] {
    if (!comm || !id) throw Error(MP_EINVAL, "null argument");
    if (world < 1 || rank < 0 || rank >= world) throw Error(MP_EINVAL, "rank out of range");
    int prev = 0;
    MP_CUDA(cudaGetDevice(&prev));
    MP_CUDA(cudaSetDevice(device));
    ncclUniqueId u{};
    std::memcpy(u.internal, id, 128);
    ncclComm_t c = nullptr;
    const ncclResult_t r = nccl().comm_init_rank(&c, world, u, rank);
    cudaSetDevice(prev);
    nccl_check(r, "ncclCommInitRank");
    comm->rank = rank, comm->world = world, comm->device_buffers = 1;
    comm->allgather = nccl_allgather;
    comm->user = c;
  });
}

void mp_nccl_comm_destroy(mp_comm* comm) {
  if (!comm || !comm->user || comm->allgather != nccl_allgather) return;
  try {
    nccl().comm_destroy(static_cast<ncclComm_t>(comm->user));
  } catch (...) {
  }
  comm->user = nullptr;
}

int mp_order_sharded(mp_context* ctx, const mp_csr* g, const mp_config* cfg, const mp_comm* comm, mp_result* out) {
  return guarded([&] {
    if (!ctx || !g || !cfg || !out || !comm) throw Error(MP_EINVAL, "null argument");
    if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world) throw Error(MP_EINVAL, "rank out of range");
    if (comm->world > 1 && !comm->allgather) throw Error(MP_EINVAL, "null all-gather");
    if (cfg->block_size != 1) throw Error(MP_EINVAL, "the sharded path orders scalar graphs (block size 1)");
    if (cfg->patch_size < 1) throw Error(MP_EINVAL, "patch size must be positive");
    if (cfg->local_mode < 0 || cfg->local_mode > 2) throw Error(MP_EINVAL, "unknown local ordering mode");
    if (!cfg->schedule_nodes && (cfg->schedule < 0 || cfg->schedule > 1)) throw Error(MP_EINVAL, "unknown schedule");
    ContextScope sd(*ctx);
    cudaStream_t s = ctx->stream;
    const int64_t launches0 = ctx->launches;
    const int32_t n = g->n, rank = comm->rank, world = comm->world;
    const int32_t L = cfg->nd_level >= 0 ? cfg->nd_level : default_nd_level_host(n);
    if (L > 24) throw Error(MP_EINVAL, "nd_level out of range");
    const int32_t nn = static_cast<int32_t>((1LL << (L + 1)) - 1);
    const Schedule sched = resolve_schedule(L, cfg->schedule, cfg->schedule_nodes, cfg->schedule_len);
    Exchange ex(*ctx, *comm);

    ctx->ktime_reset();
    MP_CUDA(cudaMemsetAsync(ctx->dwork, 0, 16 * sizeof(unsigned long long), s));
    MP_CUDA(cudaEventRecord(ctx->ev[0], s));
    GraphView gv;
    make_view(*ctx, g, gv);
    const int32_t n1 = std::max(n, 1);
    DevBuf<int32_t> asg(n1, s), node_of_l(n1, s), off_l(nn + 1, s), verts_l(n1, s), lp_l(n1, s);
    DevBuf<int32_t> off_g(nn + 1, s), verts_g(n1, s), lp_g(n1, s), node_of_g(n1, s), pm(n1, s), inv(n1, s),
        pos(nn + 1, s);
    MP_CUDA(cudaEventRecord(ctx->ev[1], s));
    // ---- patches: replicated (FPS is one sequential chain)
    const int32_t pc = patch_stage(*ctx, gv, cfg, g->on_device != 0, asg);
    MP_CUDA(cudaEventRecord(ctx->ev[2], s));
    MP_CUDA(cudaEventRecord(ctx->ev[3], s));
    // ---- ND: top k levels on every rank, own subtrees below
    ShardSpec spec;
    spec.rank = rank, spec.world = world, spec.k = std::min(L, ceil_log2(world));
    build_etree_dev(*ctx, gv.g, asg, pc, L, node_of_l, off_l, verts_l, world > 1 ? &spec : nullptr);
    std::vector<int32_t> owner = world > 1 ? spec.owner : std::vector<int32_t>(nn, -1);
    const bool sharded = std::any_of(owner.begin(), owner.end(), [](int32_t o) { return o >= 0; });
    MP_CUDA(cudaEventRecord(ctx->ev[4], s));
    // ---- MD on the nodes this rank orders (own subtrees + the replicated top)
    std::vector<uint8_t> mine(nn);
    for (int32_t i = 0; i < nn; ++i) mine[i] = owner[i] < 0 || owner[i] == rank;
    DevBuf<uint8_t> d_mine(nn, s);
    MP_CUDA(cudaMemcpyAsync(d_mine, mine.data(), nn, cudaMemcpyHostToDevice, s));
    order_tree_nodes_dev(*ctx, gv.g, L, node_of_l, off_l, verts_l, cfg->local_mode, lp_l, d_mine);
    // ---- all-gather 1: node sizes -> global offsets
    std::vector<int32_t> hoff_l(nn + 1);
    MP_CUDA(cudaMemcpyAsync(hoff_l.data(), off_l.get(), sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> size_mine(nn, 0), size_g(nn), hoff_g(nn + 1, 0);
    for (int32_t i = 0; i < nn; ++i) size_mine[i] = owner[i] == rank ? hoff_l[i + 1] - hoff_l[i] : 0;
    const std::vector<int32_t> sizes_all = sharded ? ex.host(size_mine) : std::vector<int32_t>();
    for (int32_t i = 0; i < nn; ++i) {
      size_g[i] = owner[i] < 0 ? hoff_l[i + 1] - hoff_l[i] : sizes_all[static_cast<size_t>(owner[i]) * nn + i];
      hoff_g[i + 1] = hoff_g[i] + size_g[i];
    }
    if (hoff_g[nn] != n) throw Error(MP_ELOGIC, "sharded tree does not cover the graph");
    MP_CUDA(cudaMemcpyAsync(off_g.get(), hoff_g.data(), sizeof(int32_t) * (nn + 1), cudaMemcpyHostToDevice, s));
    // ---- all-gather 2: own nodes' vertex lists and local orders -> global tree
    {
      std::vector<int64_t> cnt(world, 0);
      for (int32_t i = 0; i < nn; ++i)
        if (owner[i] >= 0) cnt[owner[i]] += size_g[i];
      const int64_t width = *std::max_element(cnt.begin(), cnt.end());
      std::vector<Seg> pack, local, remote;
      std::vector<int64_t> at(world, 0);
      for (int32_t i = 0; i < nn; ++i) {
        const int64_t len = size_g[i];
        if (owner[i] < 0) {
          local.push_back({hoff_l[i], hoff_g[i], len});
        } else {
          const int32_t r = owner[i];
          if (r == rank) pack.push_back({hoff_l[i], at[r], len});
          remote.push_back({2 * width * r + at[r], hoff_g[i], len});
          at[r] += len;
        }
      }
      copy_segs(*ctx, local, verts_l.get(), verts_g.get());
      copy_segs(*ctx, local, lp_l.get(), lp_g.get());
      if (sharded) {
        DevBuf<int32_t> send(std::max<int64_t>(2 * width, 1), s), recv(std::max<int64_t>(2 * width * world, 1), s);
        copy_segs(*ctx, pack, verts_l.get(), send.get());
        copy_segs(*ctx, pack, lp_l.get(), send.get() + width);
        ex.device(send.get(), recv.get(), 2 * width * static_cast<int64_t>(sizeof(int32_t)));
        copy_segs(*ctx, remote, recv.get(), verts_g.get());
        for (auto& sg : remote) sg.src += width;
        copy_segs(*ctx, remote, recv.get(), lp_g.get());
      }
    }
    MP_CUDA(cudaEventRecord(ctx->ev[5], s));
    // ---- assembly on the global tree (every rank)
    node_of_from_tree_dev(*ctx, n, nn, off_g, verts_g, node_of_g);
    compute_perm_blocks_dev(*ctx, n, L, off_g, verts_g, lp_g, sched, 1, pm, inv, pos);
    MP_CUDA(cudaEventRecord(ctx->ev[6], s));
    // ---- fill: own subtrees, the roots' live elements exchanged, the top replicated
    int64_t nnzL = 0, cost = 0;
    DevBuf<int64_t> cc;
    DevBuf<int32_t> par;
    if (cfg->want_fill) {
      cc.alloc(n1, s);
      par.alloc(n1, s);
      FillShard fs;
      fs.rank = rank, fs.k = spec.k, fs.owner = owner;
      fs.exchange = [&](const std::vector<int32_t>& buf) {
        std::vector<int32_t> cat;
        for (auto& part : ex.hostv(buf)) cat.insert(cat.end(), part.begin(), part.end());
        return cat;
      };
      // the etree / column-count fill (colcount.cu) is replicated on every
      // rank; the game (fill_algo 1) plays its own subtrees and exchanges
      const bool shard_game = sharded && ctx->fill_algo == 1;
      tree_fill_dev(*ctx, gv.g, L, node_of_g, off_g, verts_g, lp_g, pos, inv, cc, par, &nnzL, &cost, nullptr,
                    nullptr, shard_game ? &fs : nullptr);
      if (shard_game) {
        // all-gather 4: column counts and parents at the own nodes' positions
        std::vector<int32_t> hpos(nn + 1);
        MP_CUDA(cudaMemcpyAsync(hpos.data(), pos.get(), sizeof(int32_t) * (nn + 1), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> cnt(world, 0);
        for (int32_t i = 0; i < nn; ++i)
          if (owner[i] >= 0) cnt[owner[i]] += size_g[i];
        const int64_t width = *std::max_element(cnt.begin(), cnt.end());
        std::vector<Seg> pack, remote;
        std::vector<int64_t> at(world, 0);
        for (int32_t i = 0; i < nn; ++i) {
          if (owner[i] < 0 || size_g[i] == 0) continue;
          const int32_t r = owner[i];
          if (r == rank) pack.push_back({hpos[i], at[r], size_g[i]});
          else remote.push_back({width * r + at[r], hpos[i], size_g[i]});
          at[r] += size_g[i];
        }
        DevBuf<int64_t> sc(std::max<int64_t>(width, 1), s), rc(std::max<int64_t>(width * world, 1), s);
        DevBuf<int32_t> sp(std::max<int64_t>(width, 1), s), rp(std::max<int64_t>(width * world, 1), s);
        copy_segs(*ctx, pack, cc.get(), sc.get());
        copy_segs(*ctx, pack, par.get(), sp.get());
        ex.device(sc.get(), rc.get(), width * static_cast<int64_t>(sizeof(int64_t)));
        ex.device(sp.get(), rp.get(), width * static_cast<int64_t>(sizeof(int32_t)));
        copy_segs(*ctx, remote, rc.get(), cc.get());
        copy_segs(*ctx, remote, rp.get(), par.get());
        sum_counts_dev(*ctx, n, cc, &nnzL, &cost);
      }
    }
    MP_CUDA(cudaEventRecord(ctx->ev[7], s));
    // the pipeline's self-check (pipeline.cpp:141-142) on the global tree
    if (unrelated_edges_dev(*ctx, gv.g, node_of_g) != 0)
      throw Error(MP_ELOGIC, "separator failed to disconnect its sides");
    // outputs (every rank holds the complete result)
    const bool od = out->on_device != 0;
    output_copy(*ctx, out->patch_of, asg.get(), n, od);
    output_copy(*ctx, out->tree_node_offsets, off_g.get(), nn + 1, od);
    output_copy(*ctx, out->tree_vertices, verts_g.get(), n, od);
    output_copy(*ctx, out->tree_local_perm, lp_g.get(), n, od);
    output_copy(*ctx, out->perm, pm.get(), n, od);
    output_copy(*ctx, out->inverse, inv.get(), n, od);
    if (cfg->want_fill) {
      output_copy(*ctx, out->column_counts, cc.get(), n, od);
      output_copy(*ctx, out->etree_parent, par.get(), n, od);
    }
    MP_CUDA(cudaStreamSynchronize(s));
    out->patch_count = pc;
    out->nd_level = L;
    out->nnz_A = static_cast<int64_t>(n) + gv.m2;
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
    // work[15]: vertices this rank ordered (its subtrees + the top)
    int64_t own_v = 0;
    for (int32_t i = 0; i < nn; ++i)
      if (mine[i]) own_v += size_g[i];
    out->work[15] = own_v;
  });
}

}  // extern "C"
