// libaqua host library: C ABI (include/aqua.h), bookkeeping of the paged
// KV pool, block tables, lender / host swap arenas and tickets, descriptor
// staging, and dispatch of the sm_100a copy kernels (aqua_kernels.cu).
//
// Paper anchors (arXiv 2407.21255): Sec. 6 "Allocating AquaTensors"
// P:737-756 (producer first, DRAM fallback), Sec. 5 P:529-534 (one producer
// per consumer), Sec. 7 P:836-853 (page out / page in, gather / scatter),
// P:855-857 (location query), Sec. 8 P:864-866 (library surface, CUDA
// gather kernel in vLLM v0.5.3, safe transfers).  Readings R1..R18:
// DESIGN.md.  This file never does data movement on the CPU: with no usable
// GPU every data call fails (only AQUA_DRYRUN contexts run without one).
#include "aqua.h"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "aqua_idset.h"
#include "aqua_internal.h"

using aqua::Desc;
using aqua::kArenaBit;

namespace {

struct Arena {
  bool present = false;
  int device = 0;              // lender ordinal, AQUA_HOST or AQUA_MAPPED
  uint8_t* base = nullptr;     // device-visible base
  void* host_ptr = nullptr;    // host arena: pointer for cudaFreeHost
  uint64_t bytes = 0;
  int32_t nslots = 0;
  bool owned = false;
  bool peer = false;           // memory of another GPU (P2P / NVLink)
  int mem_device = -1;         // the GPU holding a GPU arena's memory (MAPPED: from the pointer)
  int probe = -1;              // lend-time probe bits (aqua_arena_info), -1 = not probed
  aqua::IdSet free;            // lowest-first (R4)
  std::vector<uint64_t> tick;  // last library ticket that touched each slot
};

struct Prompt {
  int32_t state = AQUA_ST_RESIDENT;
  int32_t loc = AQUA_LOC_LOCAL;
  std::vector<int32_t> ids;    // block table (RESIDENT) or slots (SWAPPED)
};

struct TicketRec {
  cudaEvent_t ev;
  cudaStream_t st;
  cudaEvent_t start = nullptr;   // AQUA_OPT_TIMING: recorded before the copy
};

struct StageRegion {
  size_t off, len;
  uint64_t ticket;
};

}  // namespace

struct aqua_ctx {
  int device = 0;
  bool dry = false;
  int32_t L = 0, bs = 0, H = 0, D = 0, e = 0, NB = 0;
  int64_t S = 0, U = 0, P_kv = 0, P_b = 0;
  std::vector<uint64_t> layer_base;
  aqua::IdSet free_blocks;
  std::vector<uint64_t> btick;  // last library ticket that touched each block
  std::unordered_map<uint64_t, Prompt> prompts;
  std::unordered_map<uint64_t, Prompt> prefixes;  // NEXT-2 cached-prefix images (ids: own namespace)
  Arena gpu, host;              // AQUA_LOC_PEER, AQUA_LOC_HOST
  int kernel = AQUA_KERNEL_AUTO;
  int max_ctas = 0;
  int tma_piece = 0;
  int tma_stages = 0;
  int ldst_variant = 2;
  int tma_variant = 0;
  int inline_max = aqua::kInlineDescBig;
  int tma_sched = AQUA_TMA_SCHED_AUTO;   // AQUA_OPT_TMA_SCHED: 0 static, n > 0 claimed n-unit batches
  int pack_vec = 64;            // register movers pack chunks of <= pack_vec x 16 B (AQUA_LDST_PACK env)
  int hybrid_ldst_units = 0;    // hybrid register warps' batch in units (0: AUTO / the ring's; AQUA_HYBRID_LDST_UNITS env)
  int rate_gbps = 0;            // AQUA_OPT_RATE_GBPS: paging budget -> CTA cap (0 = off)
  int peer_ctas = 32;           // AQUA_OPT_PEER_CTAS: CTA cap for launches touching a peer arena
  int peer_test = 0;            // AQUA_OPT_PEER_TEST
  uint32_t* d_ctr = nullptr;    // kCtrSlots {next, done} pairs (inside the d_layer_base allocation)
  uint32_t ctr_next = 0;
  std::vector<uint64_t> ctr_tick;   // ticket of the last launch that used each pair
  std::vector<int> ctr_pending;     // pairs used since the last record()
  int num_sms = 148;
  uint64_t* d_layer_base = nullptr;
  // pinned -> device descriptor staging ring
  uint8_t* h_stage = nullptr;
  uint8_t* d_stage = nullptr;
  size_t stage_cap = 0, stage_head = 0;
  // smallest staging ring (AQUA_STAGE_MIN_BYTES: a test hook).  16 MiB holds
  // the descriptors of 64 calls of 32K blocks, so the host can queue that far
  // ahead of the GPU: with 1 MiB (4 such calls) back-to-back 512 B-chunk calls
  // ran at 5.1-5.6 TB/s instead of their 6.07 (profiles/r02_block_order_ring*.jsonl)
  size_t stage_min = size_t(16) << 20;
  std::deque<StageRegion> stage_live;
  // tickets
  uint64_t next_ticket = 1;
  std::map<uint64_t, TicketRec> live;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<cudaEvent_t> tev_pool;          // timing-enabled events
  bool timing = false;
  std::unordered_map<uint64_t, float> elapsed;  // retired timed tickets -> ms
  std::deque<uint64_t> elapsed_order;
  // reclaimed library-owned lender arenas, freed once their ticket completes
  struct Zombie {
    int device;
    uint8_t* ptr;
    uint64_t ticket;
  };
  std::vector<Zombie> zombies;
  // gather-temp baseline buffer
  uint8_t* d_temp = nullptr;
  size_t temp_cap = 0;
  // AQUA_KERNEL_CE_HOST staging buffers, one per direction (out, in), and
  // the ticket of their last use
  uint8_t* ce_temp[2] = {nullptr, nullptr};
  size_t ce_cap[2] = {0, 0};
  uint64_t ce_tick[2] = {0, 0};
  bool poisoned = false;
  std::string err;
  std::vector<Desc> last_ds;    // the last call's descriptors (aqua_last_descriptors decodes them)
  int32_t last_mig_dst = -1;    // >= 0: they were a migration to this location
  uint64_t launches = 0;
  // shape of the last copy-kernel launch (aqua_last_launch)
  int32_t last_grid = 0, last_threads = 0, last_stages = 0, last_engine = 0, last_variant = 0;
  int64_t last_batch = 0, last_inline = 0;
};

namespace {

// NVTX ranges around the public calls (host-side tracing: nsys / ncu NVTX
// filters).  Header-only NVTX v3; without an attached tool a push/pop costs
// a few nanoseconds.
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};
#define AQUA_NVTX(name) NvtxScope aqua_nvtx_scope_(name)

thread_local std::string g_err;
constexpr int kHostCtas = 8;   // CTA cap for host-only swaps (PCIe-bound)
constexpr int kSwapGBpsPerSm = 50;   // swap GB/s one SM sustains (per direction) on the HBM path

// Makes `d` the current device for the scope of a call (no-op for dry runs).
struct DevGuard {
  int prev = -1, want;
  bool skip;
  explicit DevGuard(int d, bool skip_ = false) : want(d), skip(skip_) {
    if (skip) return;
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != want) cudaSetDevice(want);
  }
  ~DevGuard() {
    if (!skip && prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

aqua_status fail(aqua_ctx* c, aqua_status s, const std::string& m) {
  if (c) c->err = m;
  g_err = m;
  return s;
}

aqua_status cuda_fail(aqua_ctx* c, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  if (c) c->poisoned = true;
  return fail(c, AQUA_E_CUDA, m);
}

#define CK(ctx, expr)                                     \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr); \
  } while (0)

// ------------------------------------------------------------ tickets
void retire(aqua_ctx* c) {
  // Tickets mostly complete in issue order: retire from the oldest and stop
  // at the first one still pending (a full scan only when many pile up, so a
  // call costs O(completed) cudaEventQuery calls, not O(live)).
  const bool full = c->live.size() > 4096;
  int scanned = 0;
  for (auto it = c->live.begin(); it != c->live.end() && (full || scanned < 64); ++scanned) {
    cudaError_t q = cudaEventQuery(it->second.ev);
    if (q == cudaSuccess) {
      if (it->second.start) {
        float ms = -1.f;
        if (cudaEventElapsedTime(&ms, it->second.start, it->second.ev) != cudaSuccess) cudaGetLastError();
        c->elapsed[it->first] = ms;
        c->elapsed_order.push_back(it->first);
        if (c->elapsed_order.size() > 65536) {
          c->elapsed.erase(c->elapsed_order.front());
          c->elapsed_order.pop_front();
        }
        c->tev_pool.push_back(it->second.start);
        c->tev_pool.push_back(it->second.ev);
      } else {
        c->ev_pool.push_back(it->second.ev);
      }
      it = c->live.erase(it);
    } else {
      if (q != cudaErrorNotReady) cudaGetLastError();
      if (!full) break;
      ++it;
    }
  }
  while (!c->stage_live.empty() && !c->live.count(c->stage_live.front().ticket))
    c->stage_live.pop_front();
  for (auto it = c->zombies.begin(); it != c->zombies.end();) {
    if (c->live.count(it->ticket)) {
      ++it;
      continue;
    }
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(it->device);
    cudaFree(it->ptr);
    if (prev >= 0) cudaSetDevice(prev);
    it = c->zombies.erase(it);
  }
}

aqua_status get_event(aqua_ctx* c, bool timing, cudaEvent_t* ev) {
  auto& pool = timing ? c->tev_pool : c->ev_pool;
  if (!pool.empty()) {
    *ev = pool.back();
    pool.pop_back();
    return AQUA_OK;
  }
  CK(c, cudaEventCreateWithFlags(ev, timing ? cudaEventDefault : cudaEventDisableTiming));
  return AQUA_OK;
}

// Records the ticket event on `st`.  `start` (nullable) is a timing event
// recorded before the copy; the ticket then measures the copy's device time.
aqua_status record(aqua_ctx* c, cudaStream_t st, uint64_t* t, cudaEvent_t start = nullptr) {
  const uint64_t id = c->next_ticket++;
  for (int s : c->ctr_pending) c->ctr_tick[s] = id;
  c->ctr_pending.clear();
  if (c->dry) {
    *t = id;
    return AQUA_OK;
  }
  cudaEvent_t ev;
  if (aqua_status s = get_event(c, start != nullptr, &ev)) return s;
  CK(c, cudaEventRecord(ev, st));
  c->live[id] = TicketRec{ev, st, start};
  *t = id;
  return AQUA_OK;
}

aqua_status timing_start(aqua_ctx* c, cudaStream_t st, cudaEvent_t* start) {
  *start = nullptr;
  if (!c->timing || c->dry) return AQUA_OK;
  if (aqua_status s = get_event(c, true, start)) return s;
  CK(c, cudaEventRecord(*start, st));
  return AQUA_OK;
}

// Make `st` wait for every live ticket in `ts` recorded on another stream.
aqua_status wait_all(aqua_ctx* c, const std::vector<uint64_t>& ts, cudaStream_t st) {
  if (c->dry) return AQUA_OK;
  // few distinct tickets per call: dedupe linearly instead of sorting
  std::vector<uint64_t> u;
  uint64_t prev = 0;
  for (uint64_t t : ts) {
    if (t == 0 || t == prev) continue;
    prev = t;
    if (std::find(u.begin(), u.end(), t) == u.end()) u.push_back(t);
  }
  for (uint64_t t : u) {
    auto it = c->live.find(t);
    if (it == c->live.end() || it->second.st == st) continue;
    CK(c, cudaStreamWaitEvent(st, it->second.ev, 0));
  }
  return AQUA_OK;
}

// ------------------------------------------------------------ staging ring
// Copies `len` bytes from host `src` to a device region through pinned
// memory, on stream `st`.  The region stays reserved until the ticket that
// the caller stores in stage_live.back() completes.
aqua_status stage_upload(aqua_ctx* c, const void* src, size_t nbytes, cudaStream_t st, void** dptr) {
  const size_t len = (nbytes + 255) & ~size_t(255);
  if (len > c->stage_cap) {
    // grow: drain every user of the old ring, then reallocate
    for (auto& r : c->stage_live) {
      auto it = c->live.find(r.ticket);
      if (it != c->live.end()) CK(c, cudaEventSynchronize(it->second.ev));
    }
    c->stage_live.clear();
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->d_stage) cudaFree(c->d_stage);
    c->h_stage = nullptr;
    c->d_stage = nullptr;
    size_t cap = std::max<size_t>(len * 2, c->stage_min);
    CK(c, cudaHostAlloc(reinterpret_cast<void**>(&c->h_stage), cap, cudaHostAllocDefault));
    CK(c, cudaMalloc(reinterpret_cast<void**>(&c->d_stage), cap));
    c->stage_cap = cap;
    c->stage_head = 0;
  }
  if (c->stage_head + len > c->stage_cap) c->stage_head = 0;
  const size_t off = c->stage_head;
  // wait (host) for any live region overlapping [off, off+len)
  for (auto it = c->stage_live.begin(); it != c->stage_live.end();) {
    const bool overlap = it->off < off + len && off < it->off + it->len;
    if (overlap) {
      auto lt = c->live.find(it->ticket);
      if (lt != c->live.end()) CK(c, cudaEventSynchronize(lt->second.ev));
      it = c->stage_live.erase(it);
    } else {
      ++it;
    }
  }
  std::memcpy(c->h_stage + off, src, nbytes);
  CK(c, cudaMemcpyAsync(c->d_stage + off, c->h_stage + off, nbytes, cudaMemcpyHostToDevice, st));
  c->stage_head = off + len;
  c->stage_live.push_back(StageRegion{off, len, 0});
  *dptr = c->d_stage + off;
  return AQUA_OK;
}

void stage_seal(aqua_ctx* c, size_t nregions, uint64_t ticket) {
  for (size_t i = 0; i < nregions && i < c->stage_live.size(); ++i)
    c->stage_live[c->stage_live.size() - 1 - i].ticket = ticket;
}

// ------------------------------------------------------------ copy engines
// AQUA_KERNEL_CE_HOST: host images through the DMA copy engines.  Per chunk
// of descriptors (<= kCeChunk bytes) the TMA kernel gathers the blocks into a
// device staging buffer laid out [j][chunk range] (swap_out) and one 2-D
// cudaMemcpyAsync per run of consecutive slots moves it to pinned DRAM -- or
// the reverse for swap_in.  The copy engines keep PCIe busy in both
// directions at once (aqua_swap_exchange), where SM-issued zero-copy
// accesses reach less (profiles/r01_duplex.jsonl).
constexpr size_t kCeChunk = size_t(256) << 20;

aqua_status run_copy(aqua_ctx* c, const std::vector<Desc>& ds, aqua::Dir dir, cudaStream_t st,
                     int* regions, int32_t c0 = 0, int32_t nc = -1, const Desc* dev_desc = nullptr);

aqua_status run_copy_ce_host(aqua_ctx* c, const std::vector<Desc>& ds, aqua::Dir dir, cudaStream_t st,
                             int32_t c0, int32_t nc) {
  const int di = dir == aqua::kOut ? 0 : 1;
  const size_t per = static_cast<size_t>(nc) * c->S;           // bytes of one descriptor's range
  if (c->ce_cap[di] < per) {
    // first use, or a range larger than the buffer: (re)allocate once the
    // buffer's last user has finished
    if (c->ce_temp[di]) {
      auto it = c->live.find(c->ce_tick[di]);
      if (it != c->live.end()) CK(c, cudaEventSynchronize(it->second.ev));
      CK(c, cudaFree(c->ce_temp[di]));
      c->ce_temp[di] = nullptr;
      c->ce_cap[di] = 0;
    }
    const size_t cap = std::max(kCeChunk, per);
    CK(c, cudaMalloc(reinterpret_cast<void**>(&c->ce_temp[di]), cap));
    c->ce_cap[di] = cap;
  }
  const size_t chunk = c->ce_cap[di] / per;                      // descriptors per chunk (>= 1)
  if (aqua_status s = wait_all(c, {c->ce_tick[di]}, st)) return s;   // the buffer's last user
  uint8_t* tmp = c->ce_temp[di];
  const int kernel_engine = AQUA_KERNEL_TMA;
  for (size_t j0 = 0; j0 < ds.size(); j0 += chunk) {
    const size_t j1 = std::min(ds.size(), j0 + chunk);
    std::vector<Desc> td;
    td.reserve(j1 - j0);
    for (size_t j = j0; j < j1; ++j) td.push_back(Desc{ds[j].block, static_cast<uint32_t>(j - j0)});
    auto dma = [&](bool to_host) -> aqua_status {
      size_t j = j0;
      while (j < j1) {
        size_t r = 1;
        while (j + r < j1 && ds[j + r].slot_arena == ds[j].slot_arena + r) ++r;
        uint8_t* img = c->host.base + int64_t(ds[j].slot_arena & ~kArenaBit) * c->U + int64_t(c0) * c->S;
        uint8_t* t = tmp + (j - j0) * per;
        if (to_host)
          CK(c, cudaMemcpy2DAsync(img, c->U, t, per, per, r, cudaMemcpyDefault, st));
        else
          CK(c, cudaMemcpy2DAsync(t, per, img, c->U, per, r, cudaMemcpyDefault, st));
        j += r;
      }
      return AQUA_OK;
    };
    // the staging buffer acts as a GPU "arena" of slots of `per` bytes whose
    // chunk c sits at (c - c0)*S: base shifted by -c0*S, U = per
    // (the staging buffer is the borrower's own memory, never a peer's)
    const int saved_kernel = c->kernel;
    uint8_t* saved_base = c->gpu.base;
    const int64_t saved_U = c->U;
    const bool saved_peer = c->gpu.peer;
    c->kernel = kernel_engine;
    c->gpu.base = tmp - int64_t(c0) * c->S;
    c->U = static_cast<int64_t>(per);
    c->gpu.peer = false;
    int regions = 0;
    aqua_status s = AQUA_OK;
    if (dir == aqua::kOut) {
      s = run_copy(c, td, aqua::kOut, st, &regions, c0, nc, nullptr);
      c->kernel = saved_kernel, c->gpu.base = saved_base, c->U = saved_U, c->gpu.peer = saved_peer;
      if (!s) s = dma(true);
    } else {
      c->kernel = saved_kernel, c->gpu.base = saved_base, c->U = saved_U, c->gpu.peer = saved_peer;
      s = dma(false);
      if (!s) {
        c->kernel = kernel_engine, c->gpu.base = tmp - int64_t(c0) * c->S, c->U = static_cast<int64_t>(per);
        c->gpu.peer = false;
        s = run_copy(c, td, aqua::kIn, st, &regions, c0, nc, nullptr);
        c->kernel = saved_kernel, c->gpu.base = saved_base, c->U = saved_U, c->gpu.peer = saved_peer;
      }
    }
    if (s) return s;
    if (regions) {      // a staged descriptor upload: keep it until this stream passes here
      uint64_t t;
      if (aqua_status s2 = record(c, st, &t)) return s2;
      stage_seal(c, regions, t);
    }
  }
  return record(c, st, &c->ce_tick[di]);
}

// The TMA engine's AUTO work distribution for one launch (profiles/
// r01_tma_sched*.jsonl, r01_hybrid*.jsonl, r02_small_chunks_*.jsonl,
// r02_hybrid_split_batches.jsonl; a unit = one stage = p.group chunks;
// p.piece = the chunk size when p.group > 1):
// * one CTA per SM: claimed batches with a 4-stage ring -- 2-unit batches for
//   chunks of >= 8 KiB (6.80 / 6.71 TB/s on C2 / C4 vs 6.52 / 6.37 static).
//   Chunks below a stage are grouped per unit and the warp's lanes issue the
//   unit's pool-side copies (round 2); by chunk size: 4 KiB and 2 KiB 4-unit
//   batches (6.43 / 6.35 TB/s), 1 KiB 32-unit batches (6.04; 8: 5.78, 2: 4.96).
//   Below 1 KiB the TMA unit's per-request cost (~60 cycles) caps the ring
//   alone (512 B: 3.73 TB/s), so the hybrid ring + LDST warps runs, the ring
//   claiming 32-unit batches and the register warps 2-unit ones (5.22 vs 4.82
//   with one batch size for both).  Fewer than 8 batches per CTA halve the
//   ring's batch, down to 2 units, then static ranges.  A caller-set small
//   stage (AQUA_OPT_TMA_PIECE) keeps >= 64 KiB per batch (16 KiB pieces in
//   2-unit batches ran at 5.85 vs 6.62 TB/s);
// * under an SM cap, sub-stage chunks: the hybrid, ring 32-unit / register
//   warps 2-unit batches (32 CTAs: 1.39 / 1.75 / 2.46 TB/s at 512 B / 1 KiB /
//   2 KiB vs 1.32 / 1.63 / 2.19 with 4-unit batches for both); stage-sized
//   chunks: static ranges, already at the ~100 GB/s per-SM limit;
// * host-only launches (PCIe-bound, capped): static ranges, no hybrid.
// *sched: 0 static, n > 0 claimed batches of n units; *variant: 0 ring, 3
// hybrid; *ldst_units: the hybrid register warps' batch (units; 0 = *sched).
void auto_schedule(const aqua_ctx* c, const aqua::SwapHeader& p, int cap, bool all_host, int* sched,
                   int* variant, int* ldst_units) {
  const bool all_sms = cap == 0 || cap >= c->num_sms;
  const int64_t units = p.nitems / p.group;
  const int grid = static_cast<int>(std::min<int64_t>(all_sms ? c->num_sms : cap, p.nitems));
  const bool hybrid_ok = !all_host && *variant == 0;
  const int64_t unit_bytes = int64_t(p.piece) * p.group;
  const int min_sched = static_cast<int>(std::max<int64_t>(2, (65536 + unit_bytes - 1) / unit_bytes));
  bool hybrid = false;
  if (all_sms) {
    if (p.group == 1 || p.piece >= 8192) {
      *sched = 2;
    } else if (p.piece >= 2048) {
      *sched = 4;
    } else {
      *sched = 32;
      hybrid = p.piece < 1024 && hybrid_ok;
    }
  } else if (p.group > 1 && hybrid_ok) {
    *sched = 32;
    hybrid = true;
  } else {
    *sched = 0;
    return;
  }
  *sched = std::max(*sched, min_sched);
  while (*sched > min_sched && units < int64_t(grid) * *sched * 8) *sched /= 2;
  if (units < int64_t(grid) * *sched * 8) {
    *sched = 0;                          // too small a call for claims: static ranges, the plain ring
    return;
  }
  if (hybrid) {
    *variant = 3;
    if (*ldst_units <= 0) *ldst_units = 2;
  }
}

// Moves chunks [c0, c0 + nc) (c = 2l + kv; default: all 2L) of every
// descriptor with the configured engine.
aqua_status run_copy(aqua_ctx* c, const std::vector<Desc>& ds, aqua::Dir dir, cudaStream_t st,
                     int* regions, int32_t c0, int32_t nc, const Desc* dev_desc) {
  *regions = 0;
  if (ds.empty()) return AQUA_OK;
  if (nc < 0) nc = 2 * c->L;
  aqua::SwapHeader p{};
  const Desc* inl = nullptr;
  p.pack_vec = c->pack_vec;
  p.layer_base = c->d_layer_base;
  p.arena_base[0] = reinterpret_cast<uint64_t>(c->gpu.base);
  p.arena_base[1] = reinterpret_cast<uint64_t>(c->host.base);
  p.ndesc = static_cast<int64_t>(ds.size());
  p.L = c->L;
  p.S = c->S;
  p.U = c->U;
  p.P_kv = c->P_kv;
  p.P_b = c->P_b;
  p.c0 = c0;
  p.nc = nc;
  // AUTO: images in host DRAM go through the copy engines (full-duplex PCIe,
  // no SMs held for the transfer: profiles/r01_duplex2.jsonl); everything
  // else through the fused TMA kernel
  // one pass over the descriptors: which arenas the call touches
  // (for kMig the descriptor's `block` is the source slot, bit 31 = its arena)
  bool img_all_host = true, img_any_host = false, src_any_gpu = false, each_touches_host = true;
  for (const Desc& d : ds) {
    const bool h = d.slot_arena & kArenaBit;
    const bool src_host = static_cast<uint32_t>(d.block) & kArenaBit;
    img_all_host = img_all_host && h;
    img_any_host = img_any_host || h;
    src_any_gpu = src_any_gpu || !src_host;
    each_touches_host = each_touches_host && (h || (dir == aqua::kMig && src_host));
  }
  int engine = c->kernel;
  if (engine == AQUA_KERNEL_AUTO && dir == aqua::kMig && !dev_desc) {
    // Lender <-> host migration (NEXT-1): both images are slot-contiguous, so
    // the copy engines move each run of consecutive source and destination
    // slots as one DMA and hold no SMs (the zero-copy kernel needed 8 for the
    // PCIe time; profiles/r02_migrate_ce.jsonl).
    const int64_t off = int64_t(c0) * c->S, width = int64_t(nc) * c->S;
    auto addr = [&](uint32_t sa) {
      return ((sa & kArenaBit) ? c->host.base : c->gpu.base) + int64_t(sa & ~kArenaBit) * c->U + off;
    };
    size_t j = 0;
    while (j < ds.size()) {
      const uint32_t s0 = static_cast<uint32_t>(ds[j].block), d0 = ds[j].slot_arena;
      size_t r = 1;
      while (j + r < ds.size() && static_cast<uint32_t>(ds[j + r].block) == s0 + r && ds[j + r].slot_arena == d0 + r)
        ++r;
      if (width == c->U)
        CK(c, cudaMemcpyAsync(addr(d0), addr(s0), r * c->U, cudaMemcpyDefault, st));
      else
        CK(c, cudaMemcpy2DAsync(addr(d0), c->U, addr(s0), c->U, width, r, cudaMemcpyDefault, st));
      j += r;
    }
    return AQUA_OK;
  }
  if (engine == AQUA_KERNEL_AUTO) {
    const bool host_only = dir != aqua::kMig && !dev_desc && img_all_host;
    if (!host_only && img_any_host && dir != aqua::kMig && !dev_desc) {
      // A call with images in both arenas (the lender filled up, R5): one
      // fused launch would hold every SM for as long as PCIe takes.  Split it:
      // the GPU-arena images on the TMA kernel (HBM/NVLink speed), then the
      // host images through the copy engines, which hold no SMs
      // (profiles/r02_mixed_split.jsonl).  Same stream, disjoint destinations.
      std::vector<Desc> dg, dh;
      for (const Desc& d : ds) ((d.slot_arena & kArenaBit) ? dh : dg).push_back(d);
      int rg = 0;
      if (aqua_status s = run_copy(c, dg, dir, st, &rg, c0, nc, nullptr)) return s;
      if (rg) {   // seal this part's staged descriptors before the copy engines stage theirs
        uint64_t t;
        if (aqua_status s = record(c, st, &t)) return s;
        stage_seal(c, rg, t);
      }
      return run_copy_ce_host(c, dh, dir, st, c0, nc);
    }
    engine = host_only ? AQUA_KERNEL_CE_HOST : AQUA_KERNEL_TMA;
  }
  if (dir == aqua::kMig && engine != AQUA_KERNEL_LDST) engine = AQUA_KERNEL_TMA;  // baselines do not migrate
  if (nc != 2 * c->L && engine == AQUA_BASE_GATHER_TEMP) engine = AQUA_KERNEL_TMA;  // whole blocks only

  auto chunk_ptrs = [&](const Desc& d, int cc, uint8_t** pool, uint8_t** img) {
    const int l = cc >> 1, kv = cc & 1;
    *pool = reinterpret_cast<uint8_t*>(c->layer_base[l]) + kv * c->P_kv + int64_t(d.block) * c->P_b;
    uint8_t* ab = (d.slot_arena & kArenaBit) ? c->host.base : c->gpu.base;
    *img = ab + int64_t(d.slot_arena & ~kArenaBit) * c->U + int64_t(cc) * c->S;
  };

  if (engine == AQUA_KERNEL_CE_HOST) {
    if (dir != aqua::kMig && img_all_host && !dev_desc) return run_copy_ce_host(c, ds, dir, st, c0, nc);
    engine = AQUA_KERNEL_TMA;   // only host images go through the copy engines
  }
  if (engine == AQUA_KERNEL_TMA || engine == AQUA_KERNEL_LDST) {
    // Block-major layout: kv_plane_stride == S puts a block's K and V chunks
    // of a layer side by side in the pool, and they are side by side in the
    // image (chunk 2l + kv): move them as one chunk of 2S (whole layers only).
    int64_t S_eff = c->S;
    if (c->P_kv == c->S && (c0 % 2) == 0 && (nc % 2) == 0) {
      S_eff = 2 * c->S;
      p.S = S_eff;
      p.c0 = c0 / 2;
      p.nc = nc / 2;
      p.kv_merged = 1;
    }
    if (dev_desc) {
      p.desc = dev_desc;                      // already uploaded by the caller
    } else if (ds.size() <= static_cast<size_t>(c->inline_max)) {
      p.desc = nullptr;                       // descriptors ride in the kernel parameters
      inl = ds.data();
    } else {
      void* dd;
      aqua_status s = stage_upload(c, ds.data(), ds.size() * sizeof(Desc), st, &dd);
      if (s) return s;
      *regions = 1;
      p.desc = static_cast<const Desc*>(dd);
    }
    int ctas = 0;
    cudaError_t e;
    // A counter pair for a launch with claimed batches of `batch` items; the
    // pair's previous launch must be done with it (stream order or its
    // ticket).  Claims count items in 32 bits, each worker claiming at most
    // one batch past the end: a launch with more items (far beyond any real
    // call) falls back to static work.
    auto take_counter = [&](int64_t batch) -> aqua_status {
      if (!c->d_ctr || p.nitems + int64_t(c->num_sms) * 9 * 2 * batch >= (int64_t(1) << 31)) return AQUA_OK;
      const int slot = static_cast<int>(c->ctr_next++ % aqua::kCtrSlots);
      if (aqua_status s = wait_all(c, {c->ctr_tick[slot]}, st)) return s;
      c->ctr_pending.push_back(slot);
      p.work_ctr = c->d_ctr + 2 * slot;
      p.batch = static_cast<int32_t>(batch);
      return AQUA_OK;
    };
    // A call whose images all live in host DRAM is PCIe-bound: 4 SMs already
    // saturate it (profiles/r01_host_ctas.jsonl), so cap it at 8 and leave
    // the other SMs to decode (unless the caller set a smaller cap).
    int cap = c->max_ctas;
    // A paging budget (GB/s of swap per direction) becomes an SM cap: one SM
    // moves ~50 GB/s of swap through HBM (profiles/r01_hbm_probe2.jsonl,
    // r01_hybrid*.jsonl: ~100 GB/s of read + write), so leave the rest to decode.
    if (c->rate_gbps > 0) {
      const int want = std::max(1, (c->rate_gbps + kSwapGBpsPerSm - 1) / kSwapGBpsPerSm);
      if (cap == 0 || want < cap) cap = std::min(want, c->num_sms);
    }
    const bool all_host = each_touches_host;
    if (all_host && (cap == 0 || cap > kHostCtas)) cap = kHostCtas;
    // A launch that touches a peer lender's arena is NVLink-bound: cap it at
    // peer_ctas (the rest of the SMs stay with decode), and serve it with
    // plain loads/stores if the lend-time probe saw bulk copies misbehave.
    const bool touches_peer = c->gpu.present && c->gpu.peer && (!img_all_host || (dir == aqua::kMig && src_any_gpu));
    if (touches_peer) {
      if (c->peer_ctas > 0 && (cap == 0 || cap > c->peer_ctas)) cap = c->peer_ctas;
      if ((c->gpu.probe & 6) != 6 && engine == AQUA_KERNEL_TMA) engine = AQUA_KERNEL_LDST;
    }
    // AUTO, plane-major chunks of 512 B and 1 KiB on the whole GPU: every bulk
    // copy costs the SM's TMA unit ~90 cycles (profiles/r02_scatter_probe.jsonl),
    // so the small-chunk register kernel moves them (device time per call,
    // r02_small_device.jsonl: 512 B 5.81 / 5.80 TB/s vs 4.61 / 5.11 for the
    // hybrid, 1 KiB 5.99 / 5.98 vs 5.80 / 5.85 for the ring).  Merged K+V
    // chunks of block-major layouts stay on the ring (1 KiB merged: 4.93 vs
    // 5.31, r02_small_chunks_bm2.jsonl); host images (zero-copy over PCIe)
    // never take it.  Under an SM cap it runs 16-warp CTAs
    // (r02_small_caps.jsonl, per 1 GiB call: 512 B 52 vs 42 GB/s of read +
    // write per SM for the hybrid, 1 KiB 63-66 vs 54-57; from 2 KiB the ring
    // / hybrid stay ahead) -- except on a peer lender's arena, whose capped
    // launches keep the ring / hybrid.
    bool small_auto = false;
    if (c->kernel == AQUA_KERNEL_AUTO && engine == AQUA_KERNEL_TMA && (cap == 0 || cap >= c->num_sms || !touches_peer) &&
        !p.kv_merged && (S_eff == 512 || S_eff == 1024) && dir != aqua::kMig) {
      if (!img_any_host) engine = AQUA_KERNEL_LDST, small_auto = true;
    }
    if (engine == AQUA_KERNEL_TMA) {
      // stage = 32 KiB (or the option): one piece of a large chunk, or a
      // group of whole small chunks that are contiguous in the image
      const int stage = c->tma_piece > 0 ? c->tma_piece : 32768;
      int piece = stage;
      if (piece >= S_eff) {
        piece = static_cast<int>(S_eff);
        p.group = std::max(1, std::min(stage / piece, p.nc));
      } else {
        p.group = 1;
      }
      p.piece = piece;
      p.npieces = static_cast<int32_t>((S_eff + piece - 1) / piece);
      p.nitems = p.ndesc * p.nc * p.npieces;
      int sched = c->tma_sched, variant = c->tma_variant;
      int ldst_units = c->hybrid_ldst_units;   // the hybrid's register warps: batches of this many units
      if (sched == AQUA_TMA_SCHED_AUTO) auto_schedule(c, p, cap, all_host, &sched, &variant, &ldst_units);
      if (ldst_units <= 0) ldst_units = sched;
      const bool hybrid = variant == 3;          // TMA ring + LDST warps: always claimed batches
      if (hybrid && sched <= 0) sched = 2;
      if (sched > 0) {
        if (aqua_status s = take_counter(int64_t(sched) * p.group)) return s;
        if (hybrid && p.work_ctr) p.batch_ldst = static_cast<int32_t>(int64_t(ldst_units) * p.group);
      }
      aqua::LaunchInfo li;
      const int v_used = hybrid && !p.work_ctr ? 0 : variant;   // no counter: the plain ring
      e = aqua::launch_swap_tma(p, inl, dir, c->num_sms, cap, c->tma_stages, st, &ctas, v_used, &li);
      c->last_grid = li.grid, c->last_threads = li.threads, c->last_stages = li.stages;
      c->last_engine = AQUA_KERNEL_TMA, c->last_variant = v_used, c->last_batch = p.batch;
      c->last_inline = p.desc ? 0 : p.ndesc;
    } else {
      // variant 2: grid-stride 4 KiB items, software pipelined; variant 3
      // (small chunks of 512 B .. 4 KiB): rounds of whole chunks
      const int64_t nvec = S_eff / 16;
      const bool small = (small_auto || c->ldst_variant == 3) && S_eff % 16 == 0 && nvec >= 32 && nvec <= 256 &&
                         256 % nvec == 0;
      p.piece = small ? static_cast<int>(S_eff) : 4096;
      p.group = 1;
      p.npieces = static_cast<int32_t>((S_eff + p.piece - 1) / p.piece);
      p.nitems = p.ndesc * p.nc * p.npieces;
      aqua::LaunchInfo li;
      e = aqua::launch_swap_ldst(p, inl, dir, c->num_sms, all_host && cap == kHostCtas ? 2 * kHostCtas : cap, st, &ctas,
                                 small ? 3 : 2, &li);
      c->last_grid = li.grid, c->last_threads = li.threads, c->last_stages = 0;
      c->last_engine = AQUA_KERNEL_LDST, c->last_variant = small ? 3 : 2, c->last_batch = 0;
      c->last_inline = p.desc ? 0 : p.ndesc;
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "swap kernel launch");
    c->launches++;
    return AQUA_OK;
  }
  if (engine == AQUA_BASE_PER_CHUNK) {
    for (const Desc& d : ds)
      for (int cc = c0; cc < c0 + nc; ++cc) {
        uint8_t *pool, *img;
        chunk_ptrs(d, cc, &pool, &img);
        if (dir == aqua::kOut)
          CK(c, cudaMemcpyAsync(img, pool, c->S, cudaMemcpyDefault, st));
        else
          CK(c, cudaMemcpyAsync(pool, img, c->S, cudaMemcpyDefault, st));
      }
    return AQUA_OK;
  }
  if (engine == AQUA_BASE_GATHER_TEMP) {
    // The paper's two-step path: gather into a temporary tensor
    // on this GPU, then one large copy per contiguous run of slots.
    const size_t need = ds.size() * static_cast<size_t>(c->U);
    if (need > c->temp_cap) {
      CK(c, cudaDeviceSynchronize());
      if (c->d_temp) cudaFree(c->d_temp);
      c->d_temp = nullptr;
      CK(c, cudaMalloc(reinterpret_cast<void**>(&c->d_temp), need));
      c->temp_cap = need;
    }
    std::vector<Desc> td(ds.size());
    for (size_t j = 0; j < ds.size(); ++j) td[j] = Desc{ds[j].block, static_cast<uint32_t>(j)};
    void* dd;
    aqua_status s = stage_upload(c, td.data(), td.size() * sizeof(Desc), st, &dd);
    if (s) return s;
    *regions = 1;
    p.desc = static_cast<const Desc*>(dd);
    p.arena_base[0] = reinterpret_cast<uint64_t>(c->d_temp);
    p.piece = 4096;
    p.group = 1;
    p.npieces = static_cast<int32_t>((c->S + 4095) / 4096);
    p.nitems = p.ndesc * nc * p.npieces;
    auto runs = [&](bool to_arena) -> aqua_status {
      size_t j = 0;
      while (j < ds.size()) {
        size_t r = 1;
        while (j + r < ds.size() && ds[j + r].slot_arena == ds[j].slot_arena + r) ++r;
        uint8_t* ab = (ds[j].slot_arena & kArenaBit) ? c->host.base : c->gpu.base;
        uint8_t* img = ab + int64_t(ds[j].slot_arena & ~kArenaBit) * c->U;
        uint8_t* tmp = c->d_temp + j * static_cast<size_t>(c->U);
        if (to_arena)
          CK(c, cudaMemcpyAsync(img, tmp, r * c->U, cudaMemcpyDefault, st));
        else
          CK(c, cudaMemcpyAsync(tmp, img, r * c->U, cudaMemcpyDefault, st));
        j += r;
      }
      return AQUA_OK;
    };
    int ctas = 0;
    if (dir == aqua::kOut) {
      cudaError_t e = aqua::launch_swap_ldst(p, nullptr, aqua::kOut, c->num_sms, c->max_ctas, st, &ctas);
      if (e != cudaSuccess) return cuda_fail(c, e, "gather kernel launch");
      c->launches++;
      return runs(true);
    }
    aqua_status rs = runs(false);
    if (rs) return rs;
    cudaError_t e = aqua::launch_swap_ldst(p, nullptr, aqua::kIn, c->num_sms, c->max_ctas, st, &ctas);
    if (e != cudaSuccess) return cuda_fail(c, e, "scatter kernel launch");
    c->launches++;
    return AQUA_OK;
  }
  return fail(c, AQUA_E_INVAL, "unknown copy engine");
}

// Enqueue the copy of `ds` on `st`: one launch (layer_group <= 0 or >= L),
// or one launch per group of layer_group layers in layer order, each with its
// own ticket in group_tickets[] (layer-wise streaming, NEXT-3), so a consumer
// can start on layer group g as soon as its ticket completes.  *ticket = the
// last one, which covers the whole copy.
aqua_status enqueue_copy(aqua_ctx* c, const std::vector<Desc>& ds, aqua::Dir dir, cudaStream_t st,
                         int32_t layer_group, uint64_t* group_tickets, uint64_t* ticket) {
  if (layer_group <= 0 || layer_group >= c->L) {
    cudaEvent_t t_start;
    if (aqua_status s = timing_start(c, st, &t_start)) return s;
    int regions = 0;
    if (aqua_status s = run_copy(c, ds, dir, st, &regions)) return s;
    if (aqua_status s = record(c, st, ticket, t_start)) return s;
    stage_seal(c, regions, *ticket);
    if (group_tickets) group_tickets[0] = *ticket;
    return AQUA_OK;
  }
  const Desc* dd = nullptr;
  int up = 0;
  bool fused = c->kernel == AQUA_KERNEL_AUTO || c->kernel == AQUA_KERNEL_TMA || c->kernel == AQUA_KERNEL_LDST;
  if (c->kernel == AQUA_KERNEL_AUTO && dir != aqua::kMig) {
    // images in both arenas: each group's run_copy splits the call (lender
    // part on the TMA kernel, host part on the copy engines), so no shared upload
    bool any_host = false, any_gpu = false;
    for (const Desc& d : ds) ((d.slot_arena & kArenaBit) ? any_host : any_gpu) = true;
    if (any_host && any_gpu) fused = false;
  }
  if (fused && ds.size() > static_cast<size_t>(c->inline_max)) {
    void* d;
    if (aqua_status s = stage_upload(c, ds.data(), ds.size() * sizeof(Desc), st, &d)) return s;
    dd = static_cast<const Desc*>(d);
    up = 1;
  }
  const int32_t ng = (c->L + layer_group - 1) / layer_group;
  for (int32_t g = 0; g < ng; ++g) {
    const int32_t l0 = g * layer_group, l1 = std::min(c->L, l0 + layer_group);
    cudaEvent_t t_start;
    if (aqua_status s = timing_start(c, st, &t_start)) return s;
    int regions = 0;
    if (aqua_status s = run_copy(c, ds, dir, st, &regions, 2 * l0, 2 * (l1 - l0), dd)) return s;
    if (aqua_status s = record(c, st, ticket, t_start)) return s;
    stage_seal(c, regions, *ticket);
    if (group_tickets) group_tickets[g] = *ticket;
  }
  if (up) {   // the shared descriptor upload lives until the last group is done
    for (auto& r : c->stage_live)
      if (r.ticket == 0) r.ticket = *ticket;
  }
  return AQUA_OK;
}

aqua_status precheck(aqua_ctx* c) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  if (c->poisoned) return fail(c, AQUA_E_CUDA, "ctx poisoned by an earlier CUDA error: " + c->err);
  if (!c->dry) retire(c);
  return AQUA_OK;
}

void set_last(aqua_ctx* c, const std::vector<Desc>& ds) {
  c->last_ds.assign(ds.begin(), ds.end());
  c->last_mig_dst = -1;
}
// The same for a caller that no longer needs its descriptors: no copy.
void set_last(aqua_ctx* c, std::vector<Desc>&& ds) {
  c->last_ds.swap(ds);
  c->last_mig_dst = -1;
}

Arena* arena_of(aqua_ctx* c, int loc) { return loc == AQUA_LOC_HOST ? &c->host : &c->gpu; }

// Orders `st` after the last library use of every block and slot the
// descriptors touch (R7), then enqueues the copy; a dry context only draws a
// ticket.  For kMig the descriptor's `block` field is the source slot.
aqua_status launch(aqua_ctx* c, const std::vector<Desc>& ds, aqua::Dir dir, cudaStream_t st, uint64_t* ticket,
                   int32_t layer_group = 0, uint64_t* group_tickets = nullptr) {
  *ticket = 0;
  if (ds.empty()) return AQUA_OK;
  if (c->dry) return record(c, st, ticket);
  DevGuard g(c->device);
  // the distinct tickets of the sources and destinations, collected in one
  // pass (a call's blocks and slots mostly share one or two)
  std::vector<uint64_t> ts;
  uint64_t last = 0;
  auto note = [&](uint64_t t) {
    if (t == 0 || t == last) return;
    last = t;
    if (std::find(ts.begin(), ts.end(), t) == ts.end()) ts.push_back(t);
  };
  const uint64_t* gt = c->gpu.tick.data();
  const uint64_t* ht = c->host.tick.data();
  for (const Desc& d : ds) {
    if (dir == aqua::kMig) {
      const uint32_t sb = static_cast<uint32_t>(d.block);
      note(((sb & kArenaBit) ? ht : gt)[sb & ~kArenaBit]);
    } else {
      note(c->btick[d.block]);
    }
    note(((d.slot_arena & kArenaBit) ? ht : gt)[d.slot_arena & ~kArenaBit]);
  }
  if (aqua_status s = wait_all(c, ts, st)) return s;
  return enqueue_copy(c, ds, dir, st, layer_group, group_tickets, ticket);
}

}  // namespace

extern "C" {

const char* aqua_version(void) { return "aqua-b200 0.1 (sm_100a)"; }

const char* aqua_strerror(aqua_status s) {
  switch (s) {
    case AQUA_OK: return "ok";
    case AQUA_E_INVAL: return "invalid argument";
    case AQUA_E_NOBLOCKS: return "not enough free blocks in the pool";
    case AQUA_E_NOSPACE: return "no swap space (lender and host full)";
    case AQUA_E_STATE: return "unknown prompt or wrong state";
    case AQUA_E_CUDA: return "CUDA error (context poisoned)";
    case AQUA_E_PEER: return "lender unreachable by P2P";
  }
  return "unknown status";
}

const char* aqua_last_error(aqua_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

aqua_status aqua_create(int device, const aqua_kv_layout* lay, aqua_ctx** out) {
  AQUA_NVTX("aqua_create");
  if (!out || !lay) return fail(nullptr, AQUA_E_INVAL, "null argument");
  *out = nullptr;
  if (device < 0 && device != AQUA_DRYRUN) return fail(nullptr, AQUA_E_INVAL, "bad device");
  if (lay->num_layers <= 0 || lay->block_tokens <= 0 || lay->num_kv_heads <= 0 || lay->head_dim <= 0 ||
      lay->elem_bytes <= 0 || lay->num_blocks <= 0 || !lay->layer_base)
    return fail(nullptr, AQUA_E_INVAL, "layout sizes must be > 0 and layer_base non-null");
  const int64_t S = int64_t(lay->block_tokens) * lay->num_kv_heads * lay->head_dim * lay->elem_bytes;
  const int64_t NB = lay->num_blocks;
  const int64_t P_kv = lay->kv_plane_stride ? lay->kv_plane_stride : NB * S;
  const int64_t P_b = lay->block_stride ? lay->block_stride : S;
  if (S % 16 || P_kv % 16 || P_b % 16 || P_kv < 0 || P_b < 0)
    return fail(nullptr, AQUA_E_INVAL, "S and strides must be multiples of 16 bytes");
  if (S > (int64_t(1) << 30) || int64_t(2) * lay->num_layers * S > (int64_t(1) << 40))
    return fail(nullptr, AQUA_E_INVAL, "chunk too large");
  // chunks of distinct (kv, b) must not overlap: plane-major (flash) or block-major
  const bool plane_major = P_b >= S && P_kv >= (NB - 1) * P_b + S;
  const bool block_major = P_b >= 2 * S && P_kv >= S && P_kv + S <= P_b;
  if (!plane_major && !block_major) return fail(nullptr, AQUA_E_INVAL, "overlapping chunk layout");
  for (int l = 0; l < lay->num_layers; ++l)
    if (reinterpret_cast<uintptr_t>(lay->layer_base[l]) % 16)
      return fail(nullptr, AQUA_E_INVAL, "layer_base must be 16-byte aligned");

  aqua_ctx* c = new aqua_ctx();
  if (const char* pk = std::getenv("AQUA_LDST_PACK")) c->pack_vec = std::atoi(pk);   // tuning experiments
  if (const char* hu = std::getenv("AQUA_HYBRID_LDST_UNITS")) c->hybrid_ldst_units = std::atoi(hu);
  // a tiny staging ring makes tests wrap and regrow it within a few calls
  if (const char* sm = std::getenv("AQUA_STAGE_MIN_BYTES")) c->stage_min = std::max<size_t>(256, std::strtoull(sm, nullptr, 10));
  // AQUA_KERNEL=auto|tma|ldst|ce_host overrides the default copy engine
  // (operational escape hatch; aqua_set_option still wins afterwards)
  if (const char* k = std::getenv("AQUA_KERNEL")) {
    const std::string v(k);
    if (v == "tma") c->kernel = AQUA_KERNEL_TMA;
    else if (v == "ldst") c->kernel = AQUA_KERNEL_LDST;
    else if (v == "ce_host") c->kernel = AQUA_KERNEL_CE_HOST;
  }
  c->device = device;
  c->dry = device == AQUA_DRYRUN;
  c->L = lay->num_layers;
  c->bs = lay->block_tokens;
  c->H = lay->num_kv_heads;
  c->D = lay->head_dim;
  c->e = lay->elem_bytes;
  c->NB = lay->num_blocks;
  c->S = S;
  c->U = 2 * c->L * S;
  c->P_kv = P_kv;
  c->P_b = P_b;
  c->layer_base.resize(c->L);
  for (int l = 0; l < c->L; ++l) c->layer_base[l] = reinterpret_cast<uint64_t>(lay->layer_base[l]);
  c->free_blocks.init(c->NB, true);
  c->btick.assign(c->NB, 0);
  if (!c->dry) {
    DevGuard g(device);
    cudaError_t e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    // layer bases, then the counter pairs of dynamically scheduled launches
    if (e == cudaSuccess)
      e = cudaMalloc(reinterpret_cast<void**>(&c->d_layer_base),
                     c->L * sizeof(uint64_t) + aqua::kCtrSlots * 2 * sizeof(uint32_t));
    if (e == cudaSuccess)
      e = cudaMemcpy(c->d_layer_base, c->layer_base.data(), c->L * sizeof(uint64_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      c->d_ctr = reinterpret_cast<uint32_t*>(c->d_layer_base + c->L);
      e = cudaMemset(c->d_ctr, 0, aqua::kCtrSlots * 2 * sizeof(uint32_t));
    }
    c->ctr_tick.assign(aqua::kCtrSlots, 0);
    if (e != cudaSuccess) {
      std::string m = std::string("aqua_create: ") + cudaGetErrorString(e);
      cudaGetLastError();
      delete c;
      return fail(nullptr, AQUA_E_CUDA, m);
    }
  }
  *out = c;
  return AQUA_OK;
}

aqua_status aqua_destroy(aqua_ctx* c) {
  AQUA_NVTX("aqua_destroy");
  if (!c) return AQUA_E_INVAL;
  if (!c->dry) {
    DevGuard g(c->device);
    for (auto& kv : c->live) {
      cudaEventSynchronize(kv.second.ev);
      cudaEventDestroy(kv.second.ev);
      if (kv.second.start) cudaEventDestroy(kv.second.start);
    }
    for (auto ev : c->ev_pool) cudaEventDestroy(ev);
    for (auto ev : c->tev_pool) cudaEventDestroy(ev);
    if (c->gpu.present && c->gpu.owned) {
      DevGuard g2(c->gpu.device);
      cudaFree(c->gpu.base);
    }
    for (auto& z : c->zombies) {
      DevGuard g2(z.device);
      cudaFree(z.ptr);
    }
    if (c->host.present && c->host.owned) cudaFreeHost(c->host.host_ptr);
    if (c->d_layer_base) cudaFree(c->d_layer_base);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->d_stage) cudaFree(c->d_stage);
    if (c->d_temp) cudaFree(c->d_temp);
    for (uint8_t* t : c->ce_temp)
      if (t) cudaFree(t);
    cudaGetLastError();
  }
  delete c;
  return AQUA_OK;
}

aqua_status aqua_lend(aqua_ctx* c, int lender, void* base, uint64_t bytes, int32_t* out_nslots) {
  AQUA_NVTX("aqua_lend");
  if (aqua_status s = precheck(c)) return s;
  const bool is_host = lender == AQUA_HOST;
  Arena& a = is_host ? c->host : c->gpu;
  if (a.present) return fail(c, AQUA_E_INVAL, is_host ? "host arena already lent" : "one GPU lender per borrower (P:529-534)");
  if (lender < 0 && lender != AQUA_HOST && lender != AQUA_MAPPED) return fail(c, AQUA_E_INVAL, "bad lender");
  if (lender == AQUA_MAPPED && !base) return fail(c, AQUA_E_INVAL, "AQUA_MAPPED needs a base");
  if (base && reinterpret_cast<uintptr_t>(base) % 16) return fail(c, AQUA_E_INVAL, "base must be 16-byte aligned");
  const int64_t ns = static_cast<int64_t>(bytes / static_cast<uint64_t>(c->U));
  if (ns > 0x7fffffff) return fail(c, AQUA_E_INVAL, "too many slots");
  Arena na;
  na.present = true;
  na.device = lender;
  na.bytes = bytes;
  na.nslots = static_cast<int32_t>(ns);
  if (c->dry) {
    na.base = static_cast<uint8_t*>(base);
  } else {
    DevGuard g(c->device);
    if (is_host) {
      if (base) {
        void* dp = nullptr;
        cudaError_t e = cudaHostGetDevicePointer(&dp, base, 0);
        if (e != cudaSuccess) {
          cudaGetLastError();
          return fail(c, AQUA_E_INVAL, "host base is not pinned/mapped memory");
        }
        na.base = static_cast<uint8_t*>(dp);
      } else if (bytes) {
        void* hp = nullptr;
        CK(c, cudaHostAlloc(&hp, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        void* dp = nullptr;
        CK(c, cudaHostGetDevicePointer(&dp, hp, 0));
        na.host_ptr = hp;
        na.base = static_cast<uint8_t*>(dp);
        na.owned = true;
      }
    } else if (lender == AQUA_MAPPED) {
      na.base = static_cast<uint8_t*>(base);
    } else {
      int ndev = 0;
      CK(c, cudaGetDeviceCount(&ndev));
      if (lender >= ndev) return fail(c, AQUA_E_INVAL, "lender device out of range");
      if (lender != c->device) {
        int can = 0;
        CK(c, cudaDeviceCanAccessPeer(&can, c->device, lender));
        if (!can) return fail(c, AQUA_E_PEER, "borrower cannot access lender by P2P");
        cudaError_t e = cudaDeviceEnablePeerAccess(lender, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        } else if (e != cudaSuccess) {
          cudaGetLastError();
          return fail(c, AQUA_E_PEER, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        }
      }
      if (base) {
        na.base = static_cast<uint8_t*>(base);
      } else if (bytes) {
        DevGuard g2(lender);
        CK(c, cudaMalloc(reinterpret_cast<void**>(&na.base), bytes));
        na.owned = true;
      }
    }
  }
  if (!c->dry && !is_host && na.base) {
    DevGuard g(c->device);
    int mem_dev = lender;
    if (lender == AQUA_MAPPED) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, base) == cudaSuccess && at.type == cudaMemoryTypeDevice)
        mem_dev = at.device;
      else
        cudaGetLastError();
    }
    na.mem_device = mem_dev;
    na.peer = (mem_dev >= 0 && mem_dev != c->device) || c->peer_test > 0;
    if (na.peer && bytes >= 16) {   // (an arena too small to hold a 16-byte vector has no slots to probe)
      // once per lent arena: do plain, bulk-store and bulk-load accesses
      // reach it correctly? (restores the bytes it touches)
      int* d_res = nullptr;
      int res = 0;
      cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&d_res), sizeof(int));
      if (e == cudaSuccess) e = cudaMemset(d_res, 0, sizeof(int));
      if (e == cudaSuccess) e = aqua::launch_peer_probe(na.base, static_cast<int64_t>(bytes), d_res, nullptr);
      if (e == cudaSuccess) e = cudaMemcpy(&res, d_res, sizeof(int), cudaMemcpyDeviceToHost);
      if (d_res) cudaFree(d_res);
      if (e != cudaSuccess) {
        if (na.owned) {
          DevGuard g2(lender);
          cudaFree(na.base);
        }
        return cuda_fail(c, e, "lender probe");
      }
      if (c->peer_test == 2) res &= 1;
      na.probe = res;
      if (!(res & 1)) {
        if (na.owned) {
          DevGuard g2(lender);
          cudaFree(na.base);
        }
        return fail(c, AQUA_E_PEER, "lender arena: plain loads/stores do not round-trip");
      }
    }
    c->peer_test = 0;   // the hook applies to one lend
  }
  na.free.init(na.nslots, true);
  na.tick.assign(na.nslots, 0);
  a = std::move(na);
  if (out_nslots) *out_nslots = a.nslots;
  return AQUA_OK;
}

aqua_status aqua_alloc_blocks(aqua_ctx* c, uint64_t pid, int32_t n, aqua_stream_t stream, int32_t* out_ids) {
  AQUA_NVTX("aqua_alloc_blocks");
  if (aqua_status s = precheck(c)) return s;
  if (n < 0 || (n > 0 && !out_ids)) return fail(c, AQUA_E_INVAL, "n < 0 or null out_ids");
  auto it = c->prompts.find(pid);
  if (it != c->prompts.end() && it->second.state != AQUA_ST_RESIDENT)
    return fail(c, AQUA_E_STATE, "pid is swapped out");
  if (static_cast<int64_t>(c->free_blocks.size()) < n) return fail(c, AQUA_E_NOBLOCKS, "pool exhausted");
  DevGuard g(c->device, c->dry);
  std::vector<int32_t> ids;
  ids.reserve(n);
  auto fb = c->free_blocks.begin();
  for (int32_t i = 0; i < n; ++i) ids.push_back(*fb++);
  std::vector<uint64_t> ts;
  for (int32_t b : ids) ts.push_back(c->btick[b]);
  if (aqua_status s = wait_all(c, ts, reinterpret_cast<cudaStream_t>(stream))) return s;
  c->free_blocks.erase_lowest(n);
  Prompt& p = c->prompts[pid];
  for (int32_t b : ids) c->btick[b] = 0;
  p.ids.insert(p.ids.end(), ids.begin(), ids.end());
  std::copy(ids.begin(), ids.end(), out_ids);
  return AQUA_OK;
}

aqua_status aqua_adopt_blocks(aqua_ctx* c, uint64_t pid, int32_t n, const int32_t* ids, aqua_stream_t stream) {
  AQUA_NVTX("aqua_adopt_blocks");
  if (aqua_status s = precheck(c)) return s;
  if (n < 0 || (n > 0 && !ids)) return fail(c, AQUA_E_INVAL, "n < 0 or null ids");
  std::unordered_set<int32_t> seen;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t b = ids[i];
    if (b < 0 || b >= c->NB || !seen.insert(b).second || !c->free_blocks.count(b))
      return fail(c, AQUA_E_INVAL, "ids must be in range, free and distinct");
  }
  auto it = c->prompts.find(pid);
  if (it != c->prompts.end() && it->second.state != AQUA_ST_RESIDENT)
    return fail(c, AQUA_E_STATE, "pid is swapped out");
  DevGuard g(c->device, c->dry);
  std::vector<uint64_t> ts;
  for (int32_t i = 0; i < n; ++i) ts.push_back(c->btick[ids[i]]);
  if (aqua_status s = wait_all(c, ts, reinterpret_cast<cudaStream_t>(stream))) return s;
  Prompt& p = c->prompts[pid];
  for (int32_t i = 0; i < n; ++i) {
    c->free_blocks.erase(ids[i]);
    c->btick[ids[i]] = 0;
    p.ids.push_back(ids[i]);
  }
  return AQUA_OK;
}

// Validation + placement of a preemption (R5: whole prompt on the GPU
// lender if it fits, else the host arena; slots lowest-first per arena in
// call order).  No state change.
static aqua_status plan_out(aqua_ctx* c, int32_t n, const uint64_t* pids, std::vector<Prompt*>* ps,
                            std::vector<int>* loc, std::vector<std::vector<int32_t>>* slots,
                            std::vector<Desc>* ds) {
  if (n < 0 || (n > 0 && !pids)) return fail(c, AQUA_E_INVAL, "n < 0 or null pids");
  std::unordered_set<uint64_t> seen;
  for (int32_t i = 0; i < n; ++i)
    if (!seen.insert(pids[i]).second) return fail(c, AQUA_E_INVAL, "duplicate pid");
  for (int32_t i = 0; i < n; ++i) {
    auto it = c->prompts.find(pids[i]);
    if (it == c->prompts.end() || it->second.state != AQUA_ST_RESIDENT)
      return fail(c, AQUA_E_STATE, "pid not resident");
    ps->push_back(&it->second);
  }
  int64_t gpu_left = c->gpu.present ? static_cast<int64_t>(c->gpu.free.size()) : -1;
  int64_t host_left = c->host.present ? static_cast<int64_t>(c->host.free.size()) : -1;
  loc->assign(n, AQUA_LOC_PEER);
  for (int32_t i = 0; i < n; ++i) {
    const int64_t np = static_cast<int64_t>((*ps)[i]->ids.size());
    if (gpu_left >= np) {
      (*loc)[i] = AQUA_LOC_PEER;
      gpu_left -= np;
    } else if (host_left >= np) {
      (*loc)[i] = AQUA_LOC_HOST;
      host_left -= np;
    } else {
      return fail(c, AQUA_E_NOSPACE, "no swap space for a prompt");
    }
  }
  slots->assign(n, {});
  size_t total = 0;
  for (int32_t i = 0; i < n; ++i) total += (*ps)[i]->ids.size();
  ds->resize(total);
  Desc* dp = ds->data();
  aqua::IdSet::Scan gs = c->gpu.free.scan(), hs = c->host.free.scan();
  for (int32_t i = 0; i < n; ++i) {
    const std::vector<int32_t>& ids = (*ps)[i]->ids;
    const int32_t np = static_cast<int32_t>(ids.size());
    std::vector<int32_t>& sv = (*slots)[i];
    sv.resize(np);
    aqua::IdSet::fill((*loc)[i] == AQUA_LOC_PEER ? gs : hs, np, sv.data());   // lowest free slots (R4)
    const uint32_t bit = (*loc)[i] == AQUA_LOC_HOST ? kArenaBit : 0u;
    for (int32_t k = 0; k < np; ++k) dp[k] = Desc{ids[k], static_cast<uint32_t>(sv[k]) | bit};
    dp += np;
  }
  return AQUA_OK;
}

static aqua_status swap_out_impl(aqua_ctx* c, int32_t n, const uint64_t* pids, aqua_stream_t stream,
                                 uint64_t* out_ticket, int32_t layer_group, uint64_t* group_tickets) {
  if (aqua_status s = precheck(c)) return s;
  if (out_ticket) *out_ticket = 0;
  std::vector<Prompt*> ps;
  std::vector<int> loc;
  std::vector<std::vector<int32_t>> slots;
  std::vector<Desc> ds;
  if (aqua_status s = plan_out(c, n, pids, &ps, &loc, &slots, &ds)) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint64_t ticket = 0;
  if (aqua_status s = launch(c, ds, aqua::kOut, st, &ticket, layer_group, group_tickets)) return s;
  set_last(c, std::move(ds));   // ds is not read below
  // commit bookkeeping
  for (int32_t i = 0; i < n; ++i) {
    Arena* a = arena_of(c, loc[i]);
    a->free.erase_all(slots[i].data(), slots[i].size());
    uint64_t* st_tick = a->tick.data();
    for (int32_t s : slots[i]) st_tick[s] = ticket;
    c->free_blocks.insert_all(ps[i]->ids.data(), ps[i]->ids.size());
    uint64_t* bt_tick = c->btick.data();
    for (int32_t b : ps[i]->ids) bt_tick[b] = ticket;
    ps[i]->state = AQUA_ST_SWAPPED;
    ps[i]->loc = loc[i];
    ps[i]->ids = std::move(slots[i]);
  }
  if (out_ticket) *out_ticket = ticket;
  return AQUA_OK;
}

static aqua_status swap_in_impl(aqua_ctx* c, int32_t n, const uint64_t* pids, aqua_stream_t stream,
                                int32_t* out_ids, int64_t out_ids_cap, int32_t* out_counts, uint64_t* out_ticket,
                                int32_t layer_group, uint64_t* group_tickets) {
  if (aqua_status s = precheck(c)) return s;
  if (out_ticket) *out_ticket = 0;
  if (n < 0 || (n > 0 && !pids)) return fail(c, AQUA_E_INVAL, "n < 0 or null pids");
  std::unordered_set<uint64_t> seen;
  for (int32_t i = 0; i < n; ++i)
    if (!seen.insert(pids[i]).second) return fail(c, AQUA_E_INVAL, "duplicate pid");
  std::vector<Prompt*> ps;
  int64_t need = 0;
  for (int32_t i = 0; i < n; ++i) {
    auto it = c->prompts.find(pids[i]);
    if (it == c->prompts.end() || it->second.state != AQUA_ST_SWAPPED)
      return fail(c, AQUA_E_STATE, "pid not swapped");
    ps.push_back(&it->second);
    need += static_cast<int64_t>(it->second.ids.size());
  }
  if (need > 0 && (!out_ids || out_ids_cap < need)) return fail(c, AQUA_E_INVAL, "out_ids too small");
  if (n > 0 && !out_counts) return fail(c, AQUA_E_INVAL, "null out_counts");
  if (need > static_cast<int64_t>(c->free_blocks.size())) return fail(c, AQUA_E_NOBLOCKS, "pool exhausted");
  std::vector<Desc> ds;
  ds.resize(static_cast<size_t>(need));
  Desc* dp = ds.data();
  std::vector<std::vector<int32_t>> fresh(n);
  aqua::IdSet::Scan fs = c->free_blocks.scan();
  for (int32_t i = 0; i < n; ++i) {
    const std::vector<int32_t>& sl = ps[i]->ids;
    const int32_t np = static_cast<int32_t>(sl.size());
    fresh[i].resize(np);
    aqua::IdSet::fill(fs, np, fresh[i].data());                               // lowest free blocks (R4)
    const uint32_t bit = ps[i]->loc == AQUA_LOC_HOST ? kArenaBit : 0u;
    for (int32_t k = 0; k < np; ++k) dp[k] = Desc{fresh[i][k], static_cast<uint32_t>(sl[k]) | bit};
    dp += np;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint64_t ticket = 0;
  if (aqua_status s = launch(c, ds, aqua::kIn, st, &ticket, layer_group, group_tickets)) return s;
  set_last(c, std::move(ds));   // ds is not read below
  c->free_blocks.erase_lowest(static_cast<int32_t>(need));
  int64_t k = 0;
  for (int32_t i = 0; i < n; ++i) {
    Arena* a = arena_of(c, ps[i]->loc);
    a->free.insert_all(ps[i]->ids.data(), ps[i]->ids.size());
    uint64_t* st_tick = a->tick.data();
    for (int32_t s : ps[i]->ids) st_tick[s] = ticket;
    uint64_t* bt_tick = c->btick.data();
    for (int32_t b : fresh[i]) {
      bt_tick[b] = ticket;
      out_ids[k++] = b;
    }
    out_counts[i] = static_cast<int32_t>(fresh[i].size());
    ps[i]->state = AQUA_ST_RESIDENT;
    ps[i]->loc = AQUA_LOC_LOCAL;
    ps[i]->ids = std::move(fresh[i]);
  }
  if (out_ticket) *out_ticket = ticket;
  return AQUA_OK;
}

aqua_status aqua_swap_out(aqua_ctx* c, int32_t n, const uint64_t* pids, aqua_stream_t stream, uint64_t* out_ticket) {
  AQUA_NVTX("aqua_swap_out");
  return swap_out_impl(c, n, pids, stream, out_ticket, 0, nullptr);
}

aqua_status aqua_swap_in(aqua_ctx* c, int32_t n, const uint64_t* pids, aqua_stream_t stream, int32_t* out_ids,
                         int64_t out_ids_cap, int32_t* out_counts, uint64_t* out_ticket) {
  AQUA_NVTX("aqua_swap_in");
  return swap_in_impl(c, n, pids, stream, out_ids, out_ids_cap, out_counts, out_ticket, 0, nullptr);
}

aqua_status aqua_swap_out_layers(aqua_ctx* c, int32_t n, const uint64_t* pids, aqua_stream_t stream,
                                 int32_t layer_group, uint64_t* out_tickets) {
  AQUA_NVTX("aqua_swap_out_layers");
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  if (layer_group < 1 || !out_tickets) return fail(c, AQUA_E_INVAL, "layer_group >= 1 and out_tickets needed");
  const int32_t ng = (c->L + layer_group - 1) / layer_group;
  for (int32_t g = 0; g < ng; ++g) out_tickets[g] = 0;
  uint64_t last = 0;
  aqua_status s = swap_out_impl(c, n, pids, stream, &last, layer_group, out_tickets);
  if (s == AQUA_OK && c->dry)
    for (int32_t g = 0; g < ng; ++g) out_tickets[g] = last;
  return s;
}

aqua_status aqua_swap_in_layers(aqua_ctx* c, int32_t n, const uint64_t* pids, aqua_stream_t stream,
                                int32_t layer_group, int32_t* out_ids, int64_t out_ids_cap, int32_t* out_counts,
                                uint64_t* out_tickets) {
  AQUA_NVTX("aqua_swap_in_layers");
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  if (layer_group < 1 || !out_tickets) return fail(c, AQUA_E_INVAL, "layer_group >= 1 and out_tickets needed");
  const int32_t ng = (c->L + layer_group - 1) / layer_group;
  for (int32_t g = 0; g < ng; ++g) out_tickets[g] = 0;
  uint64_t last = 0;
  aqua_status s = swap_in_impl(c, n, pids, stream, out_ids, out_ids_cap, out_counts, &last, layer_group, out_tickets);
  if (s == AQUA_OK && c->dry)
    for (int32_t g = 0; g < ng; ++g) out_tickets[g] = last;
  return s;
}

// Preempt + resume in one call (reschedule with both lists): the SAME
// bookkeeping and bytes as aqua_swap_out(out) followed by aqua_swap_in(in),
// but the copies run on two streams, pipelined in `pieces` pieces: resume
// piece k waits only for the preemption piece that freed its blocks.  The two
// directions of a full-duplex link (NVLink egress / ingress, PCIe D2H / H2D)
// are then busy at the same time instead of one after the other.
aqua_status aqua_swap_exchange(aqua_ctx* c, int32_t n_out, const uint64_t* out_pids, int32_t n_in,
                               const uint64_t* in_pids, aqua_stream_t out_stream, aqua_stream_t in_stream,
                               int32_t pieces, int32_t* out_ids, int64_t out_ids_cap, int32_t* out_counts,
                               uint64_t* out_ticket, uint64_t* in_ticket) {
  AQUA_NVTX("aqua_swap_exchange");
  if (aqua_status s = precheck(c)) return s;
  if (out_ticket) *out_ticket = 0;
  if (in_ticket) *in_ticket = 0;
  if (n_out < 0 || n_in < 0 || (n_out > 0 && !out_pids) || (n_in > 0 && !in_pids) || pieces < 1)
    return fail(c, AQUA_E_INVAL, "bad counts, pointers or pieces");
  // ---- validate everything first (all-or-nothing, as the two calls would)
  std::vector<Prompt*> po;
  std::vector<int> loc;
  std::vector<std::vector<int32_t>> slots;
  std::vector<Desc> dso;
  if (aqua_status s = plan_out(c, n_out, out_pids, &po, &loc, &slots, &dso)) return s;
  const int64_t freed = static_cast<int64_t>(dso.size());
  std::unordered_set<uint64_t> seen_in;
  std::vector<Prompt*> pi;
  int64_t need = 0;
  for (int32_t i = 0; i < n_in; ++i) {
    if (!seen_in.insert(in_pids[i]).second) return fail(c, AQUA_E_INVAL, "duplicate pid");
    auto it = c->prompts.find(in_pids[i]);
    if (it == c->prompts.end() || it->second.state != AQUA_ST_SWAPPED)
      return fail(c, AQUA_E_STATE, "pid not swapped");
    pi.push_back(&it->second);
    need += static_cast<int64_t>(it->second.ids.size());
  }
  if (need > 0 && (!out_ids || out_ids_cap < need)) return fail(c, AQUA_E_INVAL, "out_ids too small");
  if (n_in > 0 && !out_counts) return fail(c, AQUA_E_INVAL, "null out_counts");
  if (need > static_cast<int64_t>(c->free_blocks.size()) + freed)
    return fail(c, AQUA_E_NOBLOCKS, "pool exhausted");

  // piece of the preemption that reads each block (its end event frees it)
  const int32_t npo = std::max<int32_t>(1, std::min<int32_t>(pieces, static_cast<int32_t>(dso.size())));
  std::unordered_map<int32_t, int32_t> freed_by;
  for (int32_t k = 0; k < npo; ++k) {
    const size_t j0 = dso.size() * k / npo, j1 = dso.size() * (k + 1) / npo;   // the launch ranges below
    for (size_t j = j0; j < j1; ++j) freed_by[dso[j].block] = k;
  }
  // old tickets, read before any bookkeeping changes them
  std::vector<uint64_t> wait_out, wait_in;
  for (const Desc& d : dso) {
    wait_out.push_back(c->btick[d.block]);
    wait_out.push_back(arena_of(c, (d.slot_arena & kArenaBit) ? AQUA_LOC_HOST : AQUA_LOC_PEER)
                           ->tick[d.slot_arena & ~kArenaBit]);
  }
  // ---- preemption bookkeeping
  for (int32_t i = 0; i < n_out; ++i) {
    Arena* a = arena_of(c, loc[i]);
    for (int32_t sl : slots[i]) a->free.erase(sl);
    for (int32_t b : po[i]->ids) c->free_blocks.insert(b);
  }
  // ---- plan the resume on the updated free set (lowest-first)
  std::vector<Desc> dsi;
  std::vector<std::vector<int32_t>> fresh(n_in);
  {
    auto fb = c->free_blocks.begin();
    for (int32_t i = 0; i < n_in; ++i) {
      const uint32_t bit = pi[i]->loc == AQUA_LOC_HOST ? kArenaBit : 0u;
      for (int32_t sl : pi[i]->ids) {
        const int32_t b = *fb++;
        fresh[i].push_back(b);
        dsi.push_back(Desc{b, static_cast<uint32_t>(sl) | bit});
      }
    }
  }
  for (const Desc& d : dsi) {
    wait_in.push_back(arena_of(c, (d.slot_arena & kArenaBit) ? AQUA_LOC_HOST : AQUA_LOC_PEER)
                          ->tick[d.slot_arena & ~kArenaBit]);
    if (!freed_by.count(d.block)) wait_in.push_back(c->btick[d.block]);
  }
  set_last(c, dsi);
  // resume pieces: descriptors grouped by the preemption piece they wait for
  std::vector<std::vector<Desc>> parts(npo);
  for (const Desc& d : dsi) {
    auto f = freed_by.find(d.block);
    parts[f == freed_by.end() ? 0 : f->second].push_back(d);
  }
  // ---- launches
  uint64_t t_out = 0, t_in = 0, first_in = 0;
  if (!c->dry) {
    DevGuard g(c->device);
    cudaStream_t so = reinterpret_cast<cudaStream_t>(out_stream);
    cudaStream_t si = reinterpret_cast<cudaStream_t>(in_stream);
    std::vector<uint64_t> piece_ticket(npo, 0);
    if (!dso.empty()) {
      if (aqua_status s = wait_all(c, wait_out, so)) return s;
      for (int32_t k = 0; k < npo; ++k) {
        const size_t j0 = dso.size() * k / npo, j1 = dso.size() * (k + 1) / npo;
        std::vector<Desc> part(dso.begin() + j0, dso.begin() + j1);
        if (aqua_status s = enqueue_copy(c, part, aqua::kOut, so, 0, nullptr, &piece_ticket[k])) return s;
      }
      t_out = piece_ticket[npo - 1];
    }
    if (!dsi.empty()) {
      if (aqua_status s = wait_all(c, wait_in, si)) return s;
      for (int32_t k = 0; k < npo; ++k) {
        if (piece_ticket[k]) {
          auto it = c->live.find(piece_ticket[k]);
          if (it != c->live.end() && si != so) CK(c, cudaStreamWaitEvent(si, it->second.ev, 0));
        }
        if (parts[k].empty()) continue;
        if (aqua_status s = enqueue_copy(c, parts[k], aqua::kIn, si, 0, nullptr, &t_in)) return s;
        if (!first_in) first_in = t_in;
      }
      if (!t_in) record(c, si, &t_in);
    }
    // AQUA_OPT_TIMING: the call tickets span all their pieces -- move the
    // first piece's start event onto the last ticket of each direction
    auto span = [c](uint64_t first, uint64_t last) {
      if (!first || !last || first == last) return;
      auto a = c->live.find(first), b = c->live.find(last);
      if (a == c->live.end() || b == c->live.end() || !a->second.start || !b->second.start) return;
      c->tev_pool.push_back(b->second.start);
      b->second.start = a->second.start;
      a->second.start = nullptr;   // its end event stays a live ticket (retired into the plain pool)
    };
    if (!dso.empty()) span(piece_ticket[0], t_out);
    if (!dsi.empty()) span(first_in, t_in);
  } else {
    if (!dso.empty()) record(c, nullptr, &t_out);
    if (!dsi.empty()) record(c, nullptr, &t_in);
  }
  // ---- final bookkeeping and tickets
  for (int32_t i = 0; i < n_out; ++i) {
    Arena* a = arena_of(c, loc[i]);
    for (int32_t sl : slots[i]) a->tick[sl] = t_out;
    for (int32_t b : po[i]->ids) c->btick[b] = t_out;
    po[i]->state = AQUA_ST_SWAPPED;
    po[i]->loc = loc[i];
    po[i]->ids = std::move(slots[i]);
  }
  c->free_blocks.erase_lowest(static_cast<int32_t>(need));
  int64_t k = 0;
  for (int32_t i = 0; i < n_in; ++i) {
    Arena* a = arena_of(c, pi[i]->loc);
    for (int32_t sl : pi[i]->ids) {
      a->free.insert(sl);
      a->tick[sl] = t_in;
    }
    for (int32_t b : fresh[i]) {
      c->btick[b] = t_in;
      out_ids[k++] = b;
    }
    out_counts[i] = static_cast<int32_t>(fresh[i].size());
    pi[i]->state = AQUA_ST_RESIDENT;
    pi[i]->loc = AQUA_LOC_LOCAL;
    pi[i]->ids = std::move(fresh[i]);
  }
  if (out_ticket) *out_ticket = t_out;
  if (in_ticket) *in_ticket = t_in;
  return AQUA_OK;
}

// Move the images `ps` (prompts or cached prefixes, capacity already checked)
// to the lowest free slots of arena `dst`, in order, with one fused launch.
static aqua_status move_images(aqua_ctx* c, const std::vector<Prompt*>& ps, int32_t dst, cudaStream_t st,
                               uint64_t* out_ticket) {
  Arena* ad = arena_of(c, dst);
  std::vector<Desc> ds;
  std::vector<std::vector<int32_t>> fresh(ps.size());
  const uint32_t dbit = dst == AQUA_LOC_HOST ? kArenaBit : 0u;
  auto it = ad->free.begin();
  for (size_t i = 0; i < ps.size(); ++i) {
    const uint32_t sbit = ps[i]->loc == AQUA_LOC_HOST ? kArenaBit : 0u;
    for (int32_t so : ps[i]->ids) {
      const int32_t sn = *it++;
      fresh[i].push_back(sn);
      ds.push_back(Desc{static_cast<int32_t>(static_cast<uint32_t>(so) | sbit), static_cast<uint32_t>(sn) | dbit});
    }
  }
  c->last_ds.assign(ds.begin(), ds.end());
  c->last_mig_dst = dst;
  uint64_t ticket = 0;
  if (aqua_status s = launch(c, ds, aqua::kMig, st, &ticket)) return s;
  for (size_t i = 0; i < ps.size(); ++i) {
    Arena* as = arena_of(c, ps[i]->loc);
    for (int32_t so : ps[i]->ids) {
      as->free.insert(so);
      as->tick[so] = ticket;
    }
    for (int32_t sn : fresh[i]) {
      ad->free.erase(sn);
      ad->tick[sn] = ticket;
    }
    ps[i]->loc = dst;
    ps[i]->ids = std::move(fresh[i]);
  }
  if (out_ticket) *out_ticket = ticket;
  return AQUA_OK;
}

static aqua_status migrate_impl(aqua_ctx* c, const std::vector<uint64_t>& pids, int32_t dst, cudaStream_t st,
                                uint64_t* out_ticket) {
  if (dst != AQUA_LOC_PEER && dst != AQUA_LOC_HOST) return fail(c, AQUA_E_INVAL, "dst must be PEER or HOST");
  std::unordered_set<uint64_t> seen;
  for (uint64_t pid : pids)
    if (!seen.insert(pid).second) return fail(c, AQUA_E_INVAL, "duplicate pid");
  std::vector<Prompt*> ps;
  int64_t need = 0;
  for (uint64_t pid : pids) {
    auto it = c->prompts.find(pid);
    if (it == c->prompts.end() || it->second.state != AQUA_ST_SWAPPED || it->second.loc == dst)
      return fail(c, AQUA_E_STATE, "pid has no image outside dst");
    ps.push_back(&it->second);
    need += static_cast<int64_t>(it->second.ids.size());
  }
  Arena* ad = arena_of(c, dst);
  if (!ad->present || need > ad->free.size()) return fail(c, AQUA_E_NOSPACE, "dst arena missing or full");
  return move_images(c, ps, dst, st, out_ticket);
}

aqua_status aqua_migrate(aqua_ctx* c, int32_t n, const uint64_t* pids, int32_t dst_loc, aqua_stream_t stream,
                         uint64_t* out_ticket) {
  AQUA_NVTX("aqua_migrate");
  if (aqua_status s = precheck(c)) return s;
  if (out_ticket) *out_ticket = 0;
  if (n < 0 || (n > 0 && !pids)) return fail(c, AQUA_E_INVAL, "n < 0 or null pids");
  std::vector<uint64_t> v(pids, pids + n);
  return migrate_impl(c, v, dst_loc, reinterpret_cast<cudaStream_t>(stream), out_ticket);
}

aqua_status aqua_reclaim(aqua_ctx* c, aqua_stream_t stream, uint64_t* out_ticket) {
  AQUA_NVTX("aqua_reclaim");
  if (aqua_status s = precheck(c)) return s;
  if (out_ticket) *out_ticket = 0;
  if (!c->gpu.present) return AQUA_OK;                 // idempotent
  // prompts in ascending pid, then cached prefixes in ascending id
  std::vector<uint64_t> pids, fids;
  for (const auto& kv : c->prompts)
    if (kv.second.state == AQUA_ST_SWAPPED && kv.second.loc == AQUA_LOC_PEER) pids.push_back(kv.first);
  for (const auto& kv : c->prefixes)
    if (kv.second.loc == AQUA_LOC_PEER) fids.push_back(kv.first);
  std::sort(pids.begin(), pids.end());
  std::sort(fids.begin(), fids.end());
  std::vector<Prompt*> ps;
  int64_t need = 0;
  for (uint64_t p : pids) ps.push_back(&c->prompts[p]);
  for (uint64_t f : fids) ps.push_back(&c->prefixes[f]);
  for (Prompt* p : ps) need += static_cast<int64_t>(p->ids.size());
  if (need > 0 && (!c->host.present || need > c->host.free.size()))
    return fail(c, AQUA_E_NOSPACE, "host cannot hold the lender's images");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint64_t ticket = 0;
  // the ticket must cover every library access to the lender: order the
  // stream after all of them first, then move the images (or just record)
  if (!c->dry) {
    DevGuard g(c->device);
    if (aqua_status s = wait_all(c, c->gpu.tick, st)) return s;
  }
  // every image moves -- zero-block ones too (only their location changes)
  if (!ps.empty())
    if (aqua_status s = move_images(c, ps, AQUA_LOC_HOST, st, &ticket)) return s;
  if (ticket == 0 && !c->dry) {
    DevGuard g(c->device);
    if (aqua_status s = record(c, st, &ticket)) return s;
  }
  if (!c->dry && c->gpu.owned) c->zombies.push_back(aqua_ctx::Zombie{c->gpu.device, c->gpu.base, ticket});
  c->gpu = Arena();
  if (out_ticket) *out_ticket = ticket;
  return AQUA_OK;
}

// ---------------------------------------------------------------- NEXT-2
aqua_status aqua_prefix_store(aqua_ctx* c, uint64_t fid, uint64_t src_pid, int32_t n, aqua_stream_t stream,
                              uint64_t* out_ticket) {
  AQUA_NVTX("aqua_prefix_store");
  if (aqua_status s = precheck(c)) return s;
  if (out_ticket) *out_ticket = 0;
  if (c->prefixes.count(fid)) return fail(c, AQUA_E_INVAL, "prefix id in use");
  auto it = c->prompts.find(src_pid);
  if (it == c->prompts.end() || it->second.state != AQUA_ST_RESIDENT) return fail(c, AQUA_E_STATE, "src not resident");
  Prompt& src = it->second;
  if (n < 0 || n > static_cast<int32_t>(src.ids.size())) return fail(c, AQUA_E_INVAL, "bad block count");
  int loc;
  if (c->gpu.present && c->gpu.free.size() >= n)
    loc = AQUA_LOC_PEER;
  else if (c->host.present && c->host.free.size() >= n)
    loc = AQUA_LOC_HOST;
  else
    return fail(c, AQUA_E_NOSPACE, "no swap space for the prefix");
  Arena* a = arena_of(c, loc);
  const uint32_t bit = loc == AQUA_LOC_HOST ? kArenaBit : 0u;
  std::vector<Desc> ds;
  std::vector<int32_t> slots;
  auto fit = a->free.begin();
  for (int32_t j = 0; j < n; ++j) {
    const int32_t sl = *fit++;
    slots.push_back(sl);
    ds.push_back(Desc{src.ids[j], static_cast<uint32_t>(sl) | bit});
  }
  set_last(c, ds);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint64_t ticket = 0;
  if (aqua_status s = launch(c, ds, aqua::kOut, st, &ticket)) return s;
  for (size_t j = 0; j < slots.size(); ++j) {
    a->free.erase(slots[j]);
    a->tick[slots[j]] = ticket;
    c->btick[src.ids[j]] = ticket;     // last reader of the prompt's blocks
  }
  Prompt img;
  img.state = AQUA_ST_SWAPPED;
  img.loc = loc;
  img.ids = std::move(slots);
  c->prefixes[fid] = std::move(img);
  if (out_ticket) *out_ticket = ticket;
  return AQUA_OK;
}

aqua_status aqua_prefix_load(aqua_ctx* c, uint64_t fid, uint64_t dst_pid, aqua_stream_t stream, int32_t* out_ids,
                             int32_t cap, uint64_t* out_ticket) {
  AQUA_NVTX("aqua_prefix_load");
  if (aqua_status s = precheck(c)) return s;
  if (out_ticket) *out_ticket = 0;
  auto fi = c->prefixes.find(fid);
  if (fi == c->prefixes.end()) return fail(c, AQUA_E_STATE, "unknown prefix");
  const Prompt& img = fi->second;
  auto pi = c->prompts.find(dst_pid);
  if (pi != c->prompts.end() && pi->second.state != AQUA_ST_RESIDENT) return fail(c, AQUA_E_STATE, "dst swapped");
  const int32_t n = static_cast<int32_t>(img.ids.size());
  if (n > 0 && (!out_ids || cap < n)) return fail(c, AQUA_E_INVAL, "out_ids too small");
  if (n > c->free_blocks.size()) return fail(c, AQUA_E_NOBLOCKS, "pool exhausted");
  Arena* a = arena_of(c, img.loc);
  const uint32_t bit = img.loc == AQUA_LOC_HOST ? kArenaBit : 0u;
  std::vector<Desc> ds;
  std::vector<int32_t> fresh;
  auto fb = c->free_blocks.begin();
  for (int32_t j = 0; j < n; ++j) {
    const int32_t b = *fb++;
    fresh.push_back(b);
    ds.push_back(Desc{b, static_cast<uint32_t>(img.ids[j]) | bit});
  }
  set_last(c, ds);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint64_t ticket = 0;
  if (aqua_status s = launch(c, ds, aqua::kIn, st, &ticket)) return s;
  c->free_blocks.erase_lowest(n);
  Prompt& p = c->prompts[dst_pid];
  for (int32_t j = 0; j < n; ++j) {
    c->btick[fresh[j]] = ticket;
    a->tick[img.ids[j]] = ticket;      // last reader of the image
    p.ids.push_back(fresh[j]);
    out_ids[j] = fresh[j];
  }
  if (out_ticket) *out_ticket = ticket;
  return AQUA_OK;
}

aqua_status aqua_prefix_drop(aqua_ctx* c, uint64_t fid) {
  if (aqua_status s = precheck(c)) return s;
  auto fi = c->prefixes.find(fid);
  if (fi == c->prefixes.end()) return fail(c, AQUA_E_STATE, "unknown prefix");
  Arena* a = arena_of(c, fi->second.loc);
  for (int32_t sl : fi->second.ids) a->free.insert(sl);   // slot ticks keep the last reader
  c->prefixes.erase(fi);
  return AQUA_OK;
}

aqua_status aqua_prefix_query(aqua_ctx* c, uint64_t fid, int32_t* location, int32_t* n, int32_t* slots, int32_t cap) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  auto fi = c->prefixes.find(fid);
  if (fi == c->prefixes.end()) return fail(c, AQUA_E_STATE, "unknown prefix");
  if (location) *location = fi->second.loc;
  if (n) *n = static_cast<int32_t>(fi->second.ids.size());
  if (slots) {
    if (cap < static_cast<int32_t>(fi->second.ids.size())) return fail(c, AQUA_E_INVAL, "capacity too small");
    std::copy(fi->second.ids.begin(), fi->second.ids.end(), slots);
  }
  return AQUA_OK;
}

aqua_status aqua_free(aqua_ctx* c, uint64_t pid, aqua_stream_t stream) {
  AQUA_NVTX("aqua_free");
  if (aqua_status s = precheck(c)) return s;
  auto it = c->prompts.find(pid);
  if (it == c->prompts.end()) return fail(c, AQUA_E_STATE, "unknown pid");
  Prompt& p = it->second;
  if (p.state == AQUA_ST_RESIDENT) {
    uint64_t t = 0;
    if (!c->dry && !p.ids.empty()) {
      DevGuard g(c->device);
      cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
      std::vector<uint64_t> ts;
      for (int32_t b : p.ids) ts.push_back(c->btick[b]);
      if (aqua_status s = wait_all(c, ts, st)) return s;
      if (aqua_status s = record(c, st, &t)) return s;
    }
    for (int32_t b : p.ids) {
      c->free_blocks.insert(b);
      c->btick[b] = t;
    }
  } else {
    Arena* a = arena_of(c, p.loc);
    for (int32_t s : p.ids) a->free.insert(s);
  }
  c->prompts.erase(it);
  return AQUA_OK;
}

aqua_status aqua_wait(aqua_ctx* c, uint64_t ticket, aqua_stream_t stream) {
  AQUA_NVTX("aqua_wait");
  if (aqua_status s = precheck(c)) return s;
  if (c->dry) return AQUA_OK;
  DevGuard g(c->device);
  auto it = c->live.find(ticket);
  if (it == c->live.end()) return AQUA_OK;
  CK(c, cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), it->second.ev, 0));
  return AQUA_OK;
}

aqua_status aqua_sync(aqua_ctx* c, uint64_t ticket) {
  AQUA_NVTX("aqua_sync");
  if (aqua_status s = precheck(c)) return s;
  if (c->dry) return AQUA_OK;
  auto it = c->live.find(ticket);
  if (it == c->live.end()) return AQUA_OK;
  CK(c, cudaEventSynchronize(it->second.ev));
  return AQUA_OK;
}

aqua_status aqua_ticket_done(aqua_ctx* c, uint64_t ticket, int32_t* done) {
  if (aqua_status s = precheck(c)) return s;
  if (!done) return fail(c, AQUA_E_INVAL, "null done");
  *done = 1;
  if (c->dry) return AQUA_OK;
  auto it = c->live.find(ticket);
  if (it == c->live.end()) return AQUA_OK;
  cudaError_t q = cudaEventQuery(it->second.ev);
  if (q == cudaErrorNotReady) {
    *done = 0;
    return AQUA_OK;
  }
  if (q != cudaSuccess) return cuda_fail(c, q, "cudaEventQuery");
  return AQUA_OK;
}

aqua_status aqua_ticket_elapsed(aqua_ctx* c, uint64_t ticket, float* ms) {
  if (aqua_status s = precheck(c)) return s;
  if (!ms) return fail(c, AQUA_E_INVAL, "null ms");
  auto it = c->live.find(ticket);
  if (it != c->live.end()) {
    if (!it->second.start) return fail(c, AQUA_E_STATE, "ticket was not timed (AQUA_OPT_TIMING off)");
    cudaError_t q = cudaEventQuery(it->second.ev);
    if (q == cudaErrorNotReady) return fail(c, AQUA_E_STATE, "ticket not complete");
    if (q != cudaSuccess) return cuda_fail(c, q, "cudaEventQuery");
    CK(c, cudaEventElapsedTime(ms, it->second.start, it->second.ev));
    return AQUA_OK;
  }
  auto e = c->elapsed.find(ticket);
  if (e == c->elapsed.end()) return fail(c, AQUA_E_STATE, "no timing recorded for this ticket");
  *ms = e->second;
  return AQUA_OK;
}

aqua_status aqua_query(aqua_ctx* c, uint64_t pid, int32_t* state, int32_t* location, int32_t* n,
                       int32_t* ids, int32_t cap) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  auto it = c->prompts.find(pid);
  if (it == c->prompts.end()) return fail(c, AQUA_E_STATE, "unknown pid");
  const Prompt& p = it->second;
  if (state) *state = p.state;
  if (location) *location = p.loc;
  if (n) *n = static_cast<int32_t>(p.ids.size());
  if (ids) {
    if (cap < static_cast<int32_t>(p.ids.size())) return fail(c, AQUA_E_INVAL, "ids capacity too small");
    std::copy(p.ids.begin(), p.ids.end(), ids);
  }
  return AQUA_OK;
}

aqua_status aqua_counts(aqua_ctx* c, int32_t* fb, int32_t* pf, int32_t* hf) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  if (fb) *fb = static_cast<int32_t>(c->free_blocks.size());
  if (pf) *pf = c->gpu.present ? static_cast<int32_t>(c->gpu.free.size()) : -1;
  if (hf) *hf = c->host.present ? static_cast<int32_t>(c->host.free.size()) : -1;
  return AQUA_OK;
}

aqua_status aqua_arena_base(aqua_ctx* c, int32_t loc, void** base, int32_t* nslots) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  if (loc != AQUA_LOC_PEER && loc != AQUA_LOC_HOST) return fail(c, AQUA_E_INVAL, "loc");
  Arena* a = arena_of(c, loc);
  if (!a->present) return fail(c, AQUA_E_STATE, "no such arena");
  if (base) *base = a->base;
  if (nslots) *nslots = a->nslots;
  return AQUA_OK;
}

aqua_status aqua_arena_info(aqua_ctx* c, int32_t which, int32_t* device, int32_t* peer, int32_t* probe,
                            int32_t* nslots) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  if (which != AQUA_LOC_PEER && which != AQUA_LOC_HOST) return fail(c, AQUA_E_INVAL, "which");
  const Arena& a = which == AQUA_LOC_HOST ? c->host : c->gpu;
  if (!a.present) return fail(c, AQUA_E_STATE, "arena not lent");
  if (device) *device = which == AQUA_LOC_HOST ? AQUA_HOST : (a.mem_device >= 0 ? a.mem_device : a.device);
  if (peer) *peer = a.peer ? 1 : 0;
  if (probe) *probe = a.probe;
  if (nslots) *nslots = a.nslots;
  return AQUA_OK;
}

aqua_status aqua_set_option(aqua_ctx* c, int32_t opt, int64_t v) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  switch (opt) {
    case AQUA_OPT_KERNEL:
      if (v < AQUA_KERNEL_AUTO || v > AQUA_KERNEL_CE_HOST || v == 5) return fail(c, AQUA_E_INVAL, "kernel");
      c->kernel = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_MAX_CTAS:
      if (v < 0 || v > (1 << 20)) return fail(c, AQUA_E_INVAL, "max_ctas");
      c->max_ctas = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_TMA_PIECE:
      if (v < 0 || v > 65536 || v % 16) return fail(c, AQUA_E_INVAL, "tma piece");
      c->tma_piece = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_TMA_STAGES:
      if (v < 0 || v > 32 || v == 1) return fail(c, AQUA_E_INVAL, "tma stages");
      c->tma_stages = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_TIMING:
      if (v != 0 && v != 1) return fail(c, AQUA_E_INVAL, "timing");
      c->timing = v != 0;
      return AQUA_OK;
    case AQUA_OPT_LDST_VARIANT:
      if (v != 2 && v != 3) return fail(c, AQUA_E_INVAL, "ldst variant (2 pipelined, 3 small chunks; 0, 1 retired)");
      c->ldst_variant = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_TMA_VARIANT:
      if (v != 0 && v != 3) return fail(c, AQUA_E_INVAL, "tma variant (0 ring, 3 hybrid; 1, 2 retired in round 2)");
      c->tma_variant = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_INLINE_MAX:
      if (v < 0 || v > aqua::kInlineDescBig) return fail(c, AQUA_E_INVAL, "inline max");
      c->inline_max = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_TMA_SCHED:
      if ((v < 0 || v > (1 << 20)) && v != AQUA_TMA_SCHED_AUTO)
        return fail(c, AQUA_E_INVAL, "tma sched (0 static, n > 0 claimed batches, AUTO; round robin retired)");
      c->tma_sched = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_TMA_STATIC_PCT:
      if (v != 0) return fail(c, AQUA_E_INVAL, "tma static pct (retired in round 2: only 0)");
      return AQUA_OK;
    case AQUA_OPT_RATE_GBPS:
      if (v < 0 || v > (1 << 20)) return fail(c, AQUA_E_INVAL, "rate");
      c->rate_gbps = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_PEER_CTAS:
      if (v < 0 || v > (1 << 20)) return fail(c, AQUA_E_INVAL, "peer ctas");
      c->peer_ctas = static_cast<int>(v);
      return AQUA_OK;
    case AQUA_OPT_PEER_TEST:
      if (v < 0 || v > 2) return fail(c, AQUA_E_INVAL, "peer test");
      c->peer_test = static_cast<int>(v);
      return AQUA_OK;
  }
  return fail(c, AQUA_E_INVAL, "unknown option");
}

aqua_status aqua_get_option(aqua_ctx* c, int32_t opt, int64_t* v) {
  if (!c || !v) return fail(c, AQUA_E_INVAL, "null argument");
  switch (opt) {
    case AQUA_OPT_KERNEL: *v = c->kernel; return AQUA_OK;
    case AQUA_OPT_MAX_CTAS: *v = c->max_ctas; return AQUA_OK;
    case AQUA_OPT_TMA_PIECE: *v = c->tma_piece; return AQUA_OK;
    case AQUA_OPT_TMA_STAGES: *v = c->tma_stages; return AQUA_OK;
    case AQUA_OPT_TIMING: *v = c->timing; return AQUA_OK;
    case AQUA_OPT_LDST_VARIANT: *v = c->ldst_variant; return AQUA_OK;
    case AQUA_OPT_TMA_VARIANT: *v = c->tma_variant; return AQUA_OK;
    case AQUA_OPT_INLINE_MAX: *v = c->inline_max; return AQUA_OK;
    case AQUA_OPT_TMA_SCHED: *v = c->tma_sched; return AQUA_OK;
    case AQUA_OPT_TMA_STATIC_PCT: *v = 0; return AQUA_OK;
    case AQUA_OPT_RATE_GBPS: *v = c->rate_gbps; return AQUA_OK;
    case AQUA_OPT_PEER_CTAS: *v = c->peer_ctas; return AQUA_OK;
    case AQUA_OPT_PEER_TEST: *v = c->peer_test; return AQUA_OK;
  }
  return fail(c, AQUA_E_INVAL, "unknown option");
}

aqua_status aqua_last_descriptors(aqua_ctx* c, int32_t* blocks, int32_t* slots, int32_t* locs, int64_t cap,
                                  int64_t* n_out) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  const int64_t n = static_cast<int64_t>(c->last_ds.size());
  if (n_out) *n_out = n;
  const int64_t m = std::min(n, cap);
  const bool mig = c->last_mig_dst >= 0;
  for (int64_t i = 0; i < m; ++i) {
    const Desc& d = c->last_ds[i];
    // a migration's `block` is the source slot (bit 31 = its arena)
    if (blocks) blocks[i] = mig ? static_cast<int32_t>(static_cast<uint32_t>(d.block) & ~kArenaBit) : d.block;
    if (slots) slots[i] = static_cast<int32_t>(d.slot_arena & ~kArenaBit);
    if (locs) locs[i] = mig ? c->last_mig_dst : ((d.slot_arena & kArenaBit) ? AQUA_LOC_HOST : AQUA_LOC_PEER);
  }
  return AQUA_OK;
}

aqua_status aqua_last_launch(aqua_ctx* c, int32_t* grid, int32_t* threads, int32_t* stages, int32_t* engine,
                             int32_t* variant, int64_t* batch_items, int64_t* inline_desc) {
  if (!c) return fail(nullptr, AQUA_E_INVAL, "null ctx");
  if (!c->last_grid) return fail(c, AQUA_E_STATE, "no copy kernel launched yet");
  if (grid) *grid = c->last_grid;
  if (threads) *threads = c->last_threads;
  if (stages) *stages = c->last_stages;
  if (engine) *engine = c->last_engine;
  if (variant) *variant = c->last_variant;
  if (batch_items) *batch_items = c->last_batch;
  if (inline_desc) *inline_desc = c->last_inline;
  return AQUA_OK;
}

aqua_status aqua_launch_count(aqua_ctx* c, uint64_t* n) {
  if (!c || !n) return fail(c, AQUA_E_INVAL, "null argument");
  *n = c->launches;
  return AQUA_OK;
}

aqua_status aqua_ipc_export(void* dev_ptr, uint8_t handle[64]) {
  if (!dev_ptr || !handle) return fail(nullptr, AQUA_E_INVAL, "null argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, AQUA_E_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
  std::memcpy(handle, &h, 64);
  return AQUA_OK;
}

aqua_status aqua_ipc_import(int device, const uint8_t handle[64], void** out) {
  if (!handle || !out) return fail(nullptr, AQUA_E_INVAL, "null argument");
  DevGuard g(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  cudaError_t e = cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, AQUA_E_PEER, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  }
  return AQUA_OK;
}

aqua_status aqua_ipc_close(int device, void* ptr) {
  DevGuard g(device);
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, AQUA_E_CUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
  }
  return AQUA_OK;
}

aqua_status aqua_ipc_alloc(int device, uint64_t bytes, void** out) {
  if (!out || !bytes) return fail(nullptr, AQUA_E_INVAL, "null out or zero bytes");
  DevGuard g(device);
  cudaError_t e = cudaMalloc(out, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, AQUA_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return AQUA_OK;
}

aqua_status aqua_ipc_free(int device, void* ptr) {
  DevGuard g(device);
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, AQUA_E_CUDA, std::string("cudaFree: ") + cudaGetErrorString(e));
  }
  return AQUA_OK;
}

aqua_status aqua_can_access_peer(int device, int peer, int32_t* can) {
  if (!can) return fail(nullptr, AQUA_E_INVAL, "null argument");
  int v = 0;
  cudaError_t e = device == peer ? cudaSuccess : cudaDeviceCanAccessPeer(&v, device, peer);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, AQUA_E_CUDA, std::string("cudaDeviceCanAccessPeer: ") + cudaGetErrorString(e));
  }
  *can = device == peer ? 1 : v;
  return AQUA_OK;
}

static aqua_status pattern_call(aqua_ctx* c, uint64_t pid, int32_t t0, int32_t t1, uint64_t seed,
                                aqua_stream_t stream, uint64_t* d_mism, bool verify) {
  if (aqua_status s = precheck(c)) return s;
  auto it = c->prompts.find(pid);
  if (it == c->prompts.end() || it->second.state != AQUA_ST_RESIDENT)
    return fail(c, AQUA_E_STATE, "pid not resident");
  if (c->e != 2 || c->D % 8) return fail(c, AQUA_E_INVAL, "pattern needs elem_bytes 2 and head_dim % 8 == 0");
  const Prompt& p = it->second;
  if (t0 < 0 || t1 < t0 || static_cast<int64_t>(t1) > static_cast<int64_t>(p.ids.size()) * c->bs)
    return fail(c, AQUA_E_INVAL, "token range outside the prompt's blocks");
  if (verify && !d_mism) return fail(c, AQUA_E_INVAL, "null mismatch counter");
  if (c->dry) return fail(c, AQUA_E_INVAL, "pattern kernels need a GPU ctx");
  if (t1 == t0 || p.ids.empty()) return AQUA_OK;
  DevGuard g(c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<uint64_t> ts;
  for (int32_t b : p.ids) ts.push_back(c->btick[b]);
  if (aqua_status s = wait_all(c, ts, st)) return s;
  void* dbt;
  if (aqua_status s = stage_upload(c, p.ids.data(), p.ids.size() * sizeof(int32_t), st, &dbt)) return s;
  aqua::PatternParams pp{};
  pp.bt = static_cast<const int32_t*>(dbt);
  pp.layer_base = c->d_layer_base;
  pp.P_kv = c->P_kv;
  pp.P_b = c->P_b;
  pp.L = c->L;
  pp.bs = c->bs;
  pp.H = c->H;
  pp.D = c->D;
  pp.t0 = t0;
  pp.t1 = t1;
  pp.pid = pid;
  pp.seed = seed;
  pp.mismatches = reinterpret_cast<unsigned long long*>(d_mism);
  cudaError_t e = verify ? aqua::launch_pattern_verify(pp, c->num_sms, st) : aqua::launch_pattern_fill(pp, c->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "pattern kernel launch");
  c->launches++;
  uint64_t t = 0;
  if (aqua_status s = record(c, st, &t)) return s;
  stage_seal(c, 1, t);
  for (int32_t b : p.ids) c->btick[b] = t;
  return AQUA_OK;
}

aqua_status aqua_kv_fill_pattern_batch(aqua_ctx* c, int32_t n, const uint64_t* pids, const int32_t* t0s,
                                       const int32_t* t1s, uint64_t seed, aqua_stream_t stream) {
  if (aqua_status s = precheck(c)) return s;
  if (n < 0 || (n > 0 && (!pids || !t0s || !t1s))) return fail(c, AQUA_E_INVAL, "bad arguments");
  if (c->e != 2 || c->D % 8) return fail(c, AQUA_E_INVAL, "pattern needs elem_bytes 2 and head_dim % 8 == 0");
  if (c->dry) return fail(c, AQUA_E_INVAL, "pattern kernels need a GPU ctx");
  std::vector<aqua::FillItem> items;
  std::vector<int32_t> bt_all;
  std::vector<uint64_t> ts;
  std::vector<const Prompt*> ps;
  int64_t units = 0;
  const int64_t per_tok = int64_t(2) * c->L * c->H * (c->D / 8);
  for (int32_t i = 0; i < n; ++i) {
    auto it = c->prompts.find(pids[i]);
    if (it == c->prompts.end() || it->second.state != AQUA_ST_RESIDENT)
      return fail(c, AQUA_E_STATE, "pid not resident");
    const Prompt& p = it->second;
    if (t0s[i] < 0 || t1s[i] < t0s[i] || static_cast<int64_t>(t1s[i]) > static_cast<int64_t>(p.ids.size()) * c->bs)
      return fail(c, AQUA_E_INVAL, "token range outside the prompt's blocks");
    if (t1s[i] == t0s[i]) continue;
    items.push_back(aqua::FillItem{pids[i], units, static_cast<int32_t>(bt_all.size()), t0s[i], t1s[i]});
    units += per_tok * (t1s[i] - t0s[i]);
    bt_all.insert(bt_all.end(), p.ids.begin(), p.ids.end());
    for (int32_t b : p.ids) ts.push_back(c->btick[b]);
    ps.push_back(&p);
  }
  if (items.empty()) return AQUA_OK;
  DevGuard g(c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (aqua_status s = wait_all(c, ts, st)) return s;
  // one upload: [items][block tables]
  const size_t ib = items.size() * sizeof(aqua::FillItem);
  std::vector<uint8_t> buf(ib + bt_all.size() * sizeof(int32_t));
  std::memcpy(buf.data(), items.data(), ib);
  std::memcpy(buf.data() + ib, bt_all.data(), bt_all.size() * sizeof(int32_t));
  void* d;
  if (aqua_status s = stage_upload(c, buf.data(), buf.size(), st, &d)) return s;
  aqua::FillBatchParams fp{};
  fp.items = static_cast<const aqua::FillItem*>(d);
  fp.bt_all = reinterpret_cast<const int32_t*>(static_cast<uint8_t*>(d) + ib);
  fp.layer_base = c->d_layer_base;
  fp.P_kv = c->P_kv;
  fp.P_b = c->P_b;
  fp.total_units = units;
  fp.n = static_cast<int32_t>(items.size());
  fp.L = c->L;
  fp.bs = c->bs;
  fp.H = c->H;
  fp.D = c->D;
  fp.seed = seed;
  cudaError_t e = aqua::launch_pattern_fill_batch(fp, c->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "pattern batch launch");
  c->launches++;
  uint64_t t = 0;
  if (aqua_status s = record(c, st, &t)) return s;
  stage_seal(c, 1, t);
  for (const Prompt* p : ps)
    for (int32_t b : p->ids) c->btick[b] = t;
  return AQUA_OK;
}

aqua_status aqua_kv_fill_pattern(aqua_ctx* c, uint64_t pid, int32_t t0, int32_t t1, uint64_t seed,
                                 aqua_stream_t stream) {
  return pattern_call(c, pid, t0, t1, seed, stream, nullptr, false);
}

aqua_status aqua_kv_verify_pattern(aqua_ctx* c, uint64_t pid, int32_t ntok, uint64_t seed, aqua_stream_t stream,
                                   uint64_t* d_mismatches) {
  return pattern_call(c, pid, 0, ntok, seed, stream, d_mismatches, true);
}

}  // extern "C"
