// Native trace runner (include/aqua_cfs.h, aqua_trace_run): the engine loop
// of BASELINE configs[2] -- admission by the virtual clock, the native CFS
// scheduler, libaqua paging, and the synthetic decode -- without a host
// interpreter in the loop.  Same semantics and call log as the Python
// driver (paper_2407_21255_b200/driver.py) and the oracle (oracle/sim.py).
//
// Streams (R7, A8): the swap stream waits for the decode stream before a
// preemption (the blocks' last writer); decode waits for a resume ticket
// before the iteration that needs those prompts.
#include <cuda_runtime.h>

#include <algorithm>
#include <unordered_map>
#include <vector>

#include "aqua_cfs.h"

namespace {

enum : int64_t { kPlan = 1, kSwapOut = 2, kSwapIn = 3, kAlloc = 4, kIter = 5, kFree = 6 };

struct Log {
  int64_t* buf;
  int64_t cap;
  int64_t n = 0;
  bool on;
  void put(int64_t v) {
    if (on && n < cap) buf[n] = v;
    n += on ? 1 : 0;
  }
};

}  // namespace

extern "C" {

aqua_status aqua_trace_run(aqua_ctx* ctx, aqua_cfs* sched, int32_t n, const aqua_trace_req* reqs,
                           const aqua_trace_opts* o, aqua_trace_stats* stats, int64_t* log_buf, int64_t log_cap,
                           int64_t* log_len) {
  if (!ctx || !sched || (n > 0 && !reqs) || !o || !stats) return AQUA_E_INVAL;
  *stats = aqua_trace_stats{};
  Log log{log_buf, log_buf ? log_cap : 0, 0, log_buf != nullptr};
  std::vector<aqua_trace_req> pending(reqs, reqs + n);
  std::stable_sort(pending.begin(), pending.end(), [](const aqua_trace_req& a, const aqua_trace_req& b) {
    return a.arrival != b.arrival ? a.arrival < b.arrival : a.pid < b.pid;
  });
  const int32_t cap = 1 << 16;
  std::vector<uint64_t> outs(cap), ins(cap), dec(cap), pre(cap), fin(cap);
  std::vector<int32_t> pre_tok(cap);
  std::vector<aqua_cfs_work> work(cap);
  std::vector<int32_t> ids, counts, q;
  std::unordered_map<uint64_t, int32_t> written;
  cudaEvent_t dec_done = nullptr;
  const bool gpu = o->decode_stream != o->swap_stream;
  if (gpu && cudaEventCreateWithFlags(&dec_done, cudaEventDisableTiming) != cudaSuccess) return AQUA_E_CUDA;
  auto cleanup = [&](aqua_status s) {
    if (dec_done) cudaEventDestroy(dec_done);
    if (log_len) *log_len = log.n;
    return s;
  };
  auto query_ids = [&](uint64_t pid, int32_t* loc, int32_t* k) -> aqua_status {
    int32_t st = 0;
    if (aqua_status s = aqua_query(ctx, pid, &st, loc, k, nullptr, 0)) return s;
    q.resize(std::max(*k, 1));
    return aqua_query(ctx, pid, nullptr, nullptr, nullptr, q.data(), *k);
  };
  auto log_out = [&](int32_t no) -> aqua_status {
    log.put(kSwapOut);
    log.put(no);
    for (int32_t i = 0; i < no; ++i) log.put(static_cast<int64_t>(outs[i]));
    int64_t blocks = 0;
    for (int32_t i = 0; i < no; ++i) {
      int32_t loc = 0, k = 0;
      if (aqua_status s = query_ids(outs[i], &loc, &k)) return s;
      log.put(loc);
      log.put(k);
      for (int32_t x = 0; x < k; ++x) log.put(q[x]);
      blocks += k;
    }
    stats->blocks_out += blocks;
    stats->swap_out_calls += 1;
    return AQUA_OK;
  };
  auto log_in = [&](int32_t ni) {
    log.put(kSwapIn);
    log.put(ni);
    for (int32_t i = 0; i < ni; ++i) log.put(static_cast<int64_t>(ins[i]));
    int64_t k = 0;
    for (int32_t i = 0; i < ni; ++i) {
      log.put(counts[i]);
      for (int32_t x = 0; x < counts[i]; ++x) log.put(ids[k + x]);
      k += counts[i];
    }
    stats->blocks_in += k;
    stats->swap_in_calls += 1;
  };
  auto verify = [&](int32_t ni) -> aqua_status {
    if (!o->d_mismatches) return AQUA_OK;
    for (int32_t i = 0; i < ni; ++i) {
      auto w = written.find(ins[i]);
      if (aqua_status s = aqua_kv_verify_pattern(ctx, ins[i], w == written.end() ? 0 : w->second, o->fill_seed,
                                                 o->decode_stream, o->d_mismatches))
        return s;
    }
    return AQUA_OK;
  };

  size_t pi = 0;
  int64_t it = 0;
  for (;;) {
    double t = 0;
    aqua_cfs_vclock(sched, &t);
    while (pi < pending.size() && pending[pi].arrival <= t) {
      const aqua_trace_req& r = pending[pi++];
      if (aqua_status s = aqua_cfs_add(sched, r.pid, r.arrival, r.prompt_tokens, r.output_tokens)) return cleanup(s);
    }
    int32_t res = 0, no = 0, ni = 0, nw = 0;
    if (aqua_status s = aqua_cfs_next(sched, &res, outs.data(), &no, ins.data(), &ni, work.data(), &nw, cap))
      return cleanup(s);
    if (nw == 0) {
      if (pi >= pending.size()) break;
      aqua_cfs_advance_to(sched, pending[pi].arrival);
      continue;
    }
    if (res && log.on) {
      int32_t nd = 0, np = 0;
      if (aqua_status s = aqua_cfs_partition(sched, dec.data(), &nd, pre.data(), pre_tok.data(), &np, cap))
        return cleanup(s);
      log.put(kPlan);
      log.put(it);
      log.put(nd);
      for (int32_t i = 0; i < nd; ++i) log.put(static_cast<int64_t>(dec[i]));
      log.put(np);
      for (int32_t i = 0; i < np; ++i) {
        log.put(static_cast<int64_t>(pre[i]));
        log.put(pre_tok[i]);
      }
    }
    if (no && gpu) {     // the blocks' last writer is the decode stream
      cudaEventRecord(dec_done, reinterpret_cast<cudaStream_t>(o->decode_stream));
      cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(o->swap_stream), dec_done, 0);
    }
    int64_t need = 0;
    for (int32_t i = 0; i < ni; ++i) {
      int32_t st = 0, loc = 0, k = 0;
      if (aqua_status s = aqua_query(ctx, ins[i], &st, &loc, &k, nullptr, 0)) return cleanup(s);
      need += k;
    }
    ids.assign(std::max<int64_t>(need, 1), 0);
    counts.assign(std::max(ni, 1), 0);
    uint64_t t_in = 0;
    if (no && ni && o->swap_stream2) {
      uint64_t t_out = 0;
      if (aqua_status s = aqua_swap_exchange(ctx, no, outs.data(), ni, ins.data(), o->swap_stream, o->swap_stream2,
                                             std::max(1, o->exchange_pieces), ids.data(), need, counts.data(),
                                             &t_out, &t_in))
        return cleanup(s);
      if (aqua_status s = log_out(no)) return cleanup(s);
      log_in(ni);
    } else {
      if (no) {
        uint64_t t_out = 0;
        if (aqua_status s = aqua_swap_out(ctx, no, outs.data(), o->swap_stream, &t_out)) return cleanup(s);
        if (aqua_status s = log_out(no)) return cleanup(s);
      }
      if (ni) {
        if (aqua_status s = aqua_swap_in(ctx, ni, ins.data(), o->swap_stream, ids.data(), need, counts.data(), &t_in))
          return cleanup(s);
        log_in(ni);
      }
    }
    if (ni) {
      if (aqua_status s = aqua_wait(ctx, t_in, o->decode_stream)) return cleanup(s);   // decode needs them next
      if (aqua_status s = verify(ni)) return cleanup(s);
    }
    for (int32_t w = 0; w < nw; ++w) {
      if (work[w].grow > 0) {
        ids.resize(std::max<size_t>(ids.size(), work[w].grow));
        if (aqua_status s = aqua_alloc_blocks(ctx, work[w].pid, work[w].grow, o->decode_stream, ids.data()))
          return cleanup(s);
        log.put(kAlloc);
        log.put(static_cast<int64_t>(work[w].pid));
        log.put(work[w].grow);
        for (int32_t x = 0; x < work[w].grow; ++x) log.put(ids[x]);
      }
    }
    log.put(kIter);
    log.put(it);
    log.put(nw);
    for (int32_t w = 0; w < nw; ++w) {
      log.put(static_cast<int64_t>(work[w].pid));
      log.put(work[w].ctx0);
      log.put(work[w].tokens);
      written[work[w].pid] = work[w].ctx0 + work[w].tokens;
    }
    if (o->fill) {
      std::vector<uint64_t> p(nw);
      std::vector<int32_t> a(nw), b(nw);
      for (int32_t w = 0; w < nw; ++w) {
        p[w] = work[w].pid;
        a[w] = work[w].ctx0;
        b[w] = work[w].ctx0 + work[w].tokens;
      }
      if (aqua_status s = aqua_kv_fill_pattern_batch(ctx, nw, p.data(), a.data(), b.data(), o->fill_seed,
                                                     o->decode_stream))
        return cleanup(s);
    }
    int32_t nf = 0;
    double vc = 0;
    if (aqua_status s = aqua_cfs_commit(sched, fin.data(), &nf, cap, &vc)) return cleanup(s);
    for (int32_t f = 0; f < nf; ++f) {
      written.erase(fin[f]);
      if (aqua_status s = aqua_free(ctx, fin[f], o->decode_stream)) return cleanup(s);
      log.put(kFree);
      log.put(static_cast<int64_t>(fin[f]));
    }
    ++it;
  }
  stats->iterations = it;
  aqua_cfs_vclock(sched, &stats->vclock);
  if (log.on && log.n > log.cap) return cleanup(AQUA_E_INVAL);   // *log_len = the size needed
  return cleanup(AQUA_OK);
}

}  // extern "C"
