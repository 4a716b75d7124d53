// Batches of independent meshes (SURVEY §8b "mp_order_batch for C4", §8e).
//
// The reference orders a batch frame by frame (one run_pipeline per frame,
// pipeline.cpp:100-140).  On one B200 a single frame leaves most SMs idle
// (the FM / refine / MD chains run one CTA per tree node), so the batch is
// spread over `nctx` contexts, each driven by its own host thread and
// stream: a worker takes the next frame index from a shared counter and runs
// mp_order on it.  Every context's grid-wide kernels are sized to 1/nctx of
// the SMs for the duration of the call (mp_context_set_sm_share), so the
// frames overlap instead of queueing behind each other's whole-GPU launches.
// Results are per frame and identical to sequential mp_order calls.
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "mp_context.h"
#include "mp_internal.h"

using namespace mp;

extern "C" int mp_order_batch(mp_context* const* ctxs, int32_t nctx, int32_t count, const mp_csr* graphs,
                              const mp_config* cfgs, mp_result* results, int32_t* status) {
  if (!ctxs || nctx < 1 || count < 0 || (count > 0 && (!graphs || !cfgs || !results)))
    return set_error(MP_EINVAL, "null or empty batch argument");
  for (int32_t c = 0; c < nctx; ++c) {
    if (!ctxs[c]) return set_error(MP_EINVAL, "null context");
    // a context (stream, scratch, timers) serves one host thread at a time
    for (int32_t d = 0; d < c; ++d)
      if (ctxs[d] == ctxs[c]) return set_error(MP_EINVAL, "context listed twice in the batch");
  }
  std::vector<int32_t> share(nctx);
  for (int32_t c = 0; c < nctx; ++c) {
    share[c] = ctxs[c]->sm_share;
    mp_context_set_sm_share(ctxs[c], nctx);
  }
  std::atomic<int32_t> next{0};
  std::mutex mu;
  int first_code = MP_OK;
  int32_t first_frame = count;
  std::string first_msg;
  auto worker = [&](int32_t c) {
    for (int32_t f; (f = next.fetch_add(1)) < count;) {
      const int rc = mp_order(ctxs[c], &graphs[f], &cfgs[f], &results[f]);
      if (status) status[f] = rc;
      if (rc != MP_OK) {
        std::lock_guard<std::mutex> g(mu);
        if (f < first_frame) first_frame = f, first_code = rc, first_msg = mp_last_error();
      }
    }
  };
  const int32_t nthreads = std::min(nctx, std::max(count, 1));
  std::vector<std::thread> pool;
  pool.reserve(nthreads - 1);
  for (int32_t c = 1; c < nthreads; ++c) pool.emplace_back(worker, c);
  worker(0);
  for (auto& t : pool) t.join();
  for (int32_t c = 0; c < nctx; ++c) mp_context_set_sm_share(ctxs[c], share[c]);
  if (first_code != MP_OK) return set_error(first_code, "frame " + std::to_string(first_frame) + ": " + first_msg);
  return MP_OK;
}
