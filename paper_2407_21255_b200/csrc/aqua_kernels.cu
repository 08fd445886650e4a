// sm_100a kernels of libaqua: the fused block-table gather/scatter that
// pages a prompt's KV blocks between the borrower's pool and a swap arena
// (peer HBM over NVLink 5 / NVSwitch, the same HBM, or mapped pinned host
// memory), plus the harness pattern kernels.
//
// Paper: Sec. 7 "Efficient context switching" gathers the
// per-layer pieces into a temporary GPU tensor and then copies it to the
// AquaTensor; the reverse for swap-in.  Here the temporary tensor is gone:
// every (block, layer, K|V) chunk is moved straight from its pool address to
// its final place in the lender's slot (and back), in one launch for all the
// prompts of a call.  Pure byte movement: no arithmetic on values, no tensor
// cores.
//
// Work item = one piece (<= `piece` bytes) of one chunk (l, kv) of one
// descriptor j.  Items are numbered j-major, then c = 2l + kv, then piece,
// so consecutive items are consecutive bytes of the slot-major image.
//
// Engines (the host picks one per launch):
//   swap_tma_kernel<D, P, 0>   product: one warp per SM drives a ring of TMA
//                              bulk copies (lane 0 the whole-stage copies,
//                              the lanes together a unit's scattered pool-
//                              side chunks); work in static ranges or
//                              claimed batches (AUTO)
//   swap_tma_kernel<D, P, 8>   hybrid: the same ring + 8 warps moving
//                              claimed batches through registers (capped
//                              launches of sub-stage chunks)
//   swap_ldst_kernel           16-byte LDG/STG, grid-stride, software
//                              pipelined (second engine; peer fallback)
// Round 1's tuning experiments (warp-specialised ring, two rings per CTA,
// round-robin batches, a static head, unpipelined / claimed LDST flavours)
// were retired in round 2: AUTO never chose them.
// P = SwapParamsT<256 or 4064>: the descriptors ride in the launch
// parameters when they fit (else SwapHeader::desc points at a staged copy).
#include "aqua_internal.h"

#include <algorithm>
#include <cstdlib>

namespace aqua {
namespace {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "AQUA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra AQUA_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// TMA bulk copy shared -> global (local HBM, a P2P-mapped peer address or
// mapped host memory), tracked by bulk groups.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int4 ld_stream(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(void* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// ------------------------------------------------------------ addressing
struct Cursor {
  int64_t j;
  int32_t c, q;
  __device__ __forceinline__ void init(int64_t item, const SwapHeader& p) {
    const int64_t per_desc = int64_t(p.nc) * p.npieces;
    uint32_t r;
    if (item < (int64_t(1) << 32) && per_desc < (int64_t(1) << 32)) {   // 32-bit divides (64-bit: a long subroutine)
      const uint32_t it = static_cast<uint32_t>(item), pd = static_cast<uint32_t>(per_desc);
      const uint32_t jj = it / pd;
      j = jj;
      r = it - jj * pd;
    } else {
      j = item / per_desc;
      r = static_cast<uint32_t>(item - j * per_desc);
    }
    const uint32_t cl = r / static_cast<uint32_t>(p.npieces);
    q = static_cast<int32_t>(r - cl * static_cast<uint32_t>(p.npieces));
    c = p.c0 + static_cast<int32_t>(cl);
  }
};

template <class P>
__device__ __forceinline__ Desc desc_at(const P& p, int64_t j) {
  return p.desc ? p.desc[j] : p.inl[j];
}

// chunk(l, kv, b) = layer_base[l] + kv*P_kv + b*P_b            (R1)
// image chunk    = arena + slot*U + (2l+kv)*S                   (R3)
template <Dir D>
__device__ __forceinline__ void item_addrs(const SwapHeader& p, const Desc d, int c, int q,
                                           const uint8_t*& src, uint8_t*& dst, uint32_t& bytes) {
  const int l = p.kv_merged ? c : c >> 1, kv = p.kv_merged ? 0 : c & 1;
  const int64_t off = int64_t(q) * p.piece;
  const uint32_t a = d.slot_arena >> 31;
  const int64_t slot = d.slot_arena & ~kArenaBit;
  const uint64_t base = a ? p.arena_base[1] : p.arena_base[0];   // no dynamic param indexing
  uint8_t* img = reinterpret_cast<uint8_t*>(base) + slot * p.U + int64_t(c) * p.S + off;
  const int64_t rem = p.S - off;
  bytes = static_cast<uint32_t>(rem < p.piece ? rem : p.piece);
  if (D == kMig) {
    // image -> image: the source slot rides in `block` (bit 31 = its arena)
    const uint32_t sb = static_cast<uint32_t>(d.block);
    const uint64_t sbase = (sb >> 31) ? p.arena_base[1] : p.arena_base[0];
    src = reinterpret_cast<const uint8_t*>(sbase) + int64_t(sb & ~kArenaBit) * p.U + int64_t(c) * p.S + off;
    dst = img;
    return;
  }
  uint8_t* pool = reinterpret_cast<uint8_t*>(__ldg(p.layer_base + l)) + kv * p.P_kv +
                  int64_t(d.block) * p.P_b + off;
  if (D == kOut) {
    src = pool;
    dst = img;
  } else {
    src = img;
    dst = pool;
  }
}

// ------------------------------------------------------------ TMA ring kernel
// One CTA = one warp; lane 0 drives a `stages`-deep ring of shared-memory
// stages: cp.async.bulk loads (mbarrier complete_tx) run stages-1 units
// ahead of the cp.async.bulk stores.  Work distribution: see below.
//
// A unit is `group` consecutive chunks of one descriptor when a chunk fits a
// piece (S <= piece): they are contiguous in the image, so the image side is
// ONE bulk op of k*S bytes and the pool side k bulk ops of S bytes.  With
// larger chunks a unit is one piece of one chunk (group == 1).
struct Unit {
  int64_t j;
  int32_t c, q;
  int64_t left;     // items of this CTA not yet covered
};

__device__ __forceinline__ int unit_len(const SwapHeader& p, const Unit& u) {
  if (p.group == 1) return 1;
  int64_t k = p.c0 + p.nc - u.c;
  if (k > p.group) k = p.group;
  if (k > u.left) k = u.left;
  return static_cast<int>(k);
}

__device__ __forceinline__ void unit_next(const SwapHeader& p, Unit& u, int k) {
  u.left -= k;
  if (p.group == 1) {
    if (++u.q == p.npieces) {
      u.q = 0;
      if (++u.c == p.c0 + p.nc) {
        u.c = p.c0;
        ++u.j;
      }
    }
  } else {
    u.c += k;
    if (u.c == p.c0 + p.nc) {
      u.c = p.c0;
      ++u.j;
    }
  }
}

// Work distribution.  Static (p.batch == 0): each CTA owns one contiguous
// item range.  Claimed batches (p.batch > 0, p.work_ctr set; the default
// with one CTA per SM): CTA b starts on batch b, then claims batches of
// p.batch items from the launch's counter, fetched one batch ahead so its
// latency hides behind the ring.  Per-SM copy rates differ by a few percent
// (ncu sm__cycles_active min..max 4.4 % with static ranges, 0.6 % claimed),
// and consecutive claims keep the pieces in flight chip-wide in a narrow
// window of the image: 6.80 vs 6.52 TB/s on C2.  The loader
// runs ahead of the storer, so the batches it has entered wait in a small
// queue.
//
// Claim n items (a batch): the counter counts items claimed beyond the
// CTAs' first batches.  Inline atom.add, not atomicAdd: for a uniform-address
// atomicAdd the compiler emits a warp-aggregated atomic whose SHFL of the
// result waits for the atomic at once; this one is issued by one lane and its
// result is only waited for where it is used, one batch later (round 1 used
// atom.inc on batch ids for the same reason; item counts let the hybrid's
// ring and register warps claim batches of different sizes).
__device__ __forceinline__ uint32_t claim_items(uint32_t* ctr, uint32_t n) {
  uint32_t v;
  asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(v) : "l"(ctr), "r"(n) : "memory");
  return v;
}

// Called once by every claiming worker (`total` of them) after its last
// claim; the last one resets the counter pair for the next launch.
__device__ __forceinline__ void dyn_finish(uint32_t* ctr, uint32_t total) {
  __threadfence();
  if (atomicAdd(ctr + 1, 1u) == total - 1) {       // last worker: every claim is done
    ctr[0] = 0;
    ctr[1] = 0;
    __threadfence();
  }
}

// Hybrid variant (LW > 0 LDST warps, AQUA_OPT_TMA_VARIANT 3): besides the
// TMA ring of warp 0, warps 1..LW claim batches of the same launch and copy
// them item by item with 16-byte loads and stores through registers, two
// rounds in flight per warp.  A CTA's TMA engine moves at most ~100 GB/s of
// read + write (profiles/r01_tma_rings.jsonl: the same at 4 and 6 stages), so
// under an SM cap the register path adds a second mover on the same SM.
// `base` = the items the rings' first (static) batches cover; the register
// warps claim batches of p.batch_ldst items.
template <Dir D, class P>
__device__ __forceinline__ void ldst_worker(const P& p, int64_t base, uint32_t total) {
  const int lane = threadIdx.x & 31;
  const uint32_t bw = static_cast<uint32_t>(p.batch_ldst > 0 ? p.batch_ldst : p.batch);
  uint32_t raw = lane == 0 ? claim_items(p.work_ctr, bw) : 0u;
  int64_t a = int64_t(__shfl_sync(0xffffffffu, raw, 0)) + base;
  while (a < p.nitems) {
    raw = lane == 0 ? claim_items(p.work_ctr, bw) : 0u;  // the next batch, used after this one
    const int64_t e = a + bw < p.nitems ? a + bw : p.nitems;
    Cursor cu;
    cu.init(a, p);
    int64_t j = cu.j;
    int32_t c = cu.c, q = cu.q;
    int4 va[8], vb[8];
    // Whole chunks of 512 B .. 2 KiB (npieces == 1): pack 256 / nvec chunks
    // into each 4 KiB round.  Unroll slot u of every lane belongs to chunk
    // (u * 32) / nvec of the round (uniform across the warp), so the
    // descriptor reads stay warp-uniform.
    const int nvec_s = static_cast<int>(p.S >> 4);
    if (p.npieces == 1 && nvec_s >= 32 && nvec_s <= p.pack_vec && nvec_s < 256 && (256 % nvec_s) == 0) {
      const int k = 256 / nvec_s;            // chunks per round
      const int32_t rel0 = c - p.c0;         // position of item a within its descriptor
      // loads of a round also compute the stores' addresses (kept per unroll
      // slot in registers); 32-bit index math (rel < nc + batch)
      auto load_round = [&](int4* v, uint8_t** dp, int64_t o0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int32_t o = static_cast<int32_t>(o0) + (u * 32) / nvec_s;
          dp[u] = nullptr;
          if (a + o < e) {
            const uint32_t rel = static_cast<uint32_t>(rel0 + o);
            const uint32_t dj = rel / static_cast<uint32_t>(p.nc);
            const int32_t cc = p.c0 + static_cast<int32_t>(rel - dj * static_cast<uint32_t>(p.nc));
            const uint8_t* src;
            uint32_t bytes;
            item_addrs<D>(p, desc_at(p, j + dj), cc, 0, src, dp[u], bytes);
            const size_t vo = size_t((u * 32) % nvec_s + lane) * 16;
            v[u] = ld_stream(src + vo);
            dp[u] += vo;
          }
        }
      };
      auto store_round = [&](const int4* v, uint8_t* const* dp) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (dp[u]) st_stream(dp[u], v[u]);
      };
      uint8_t *da[8], *db[8];
      const int64_t n = e - a;
      load_round(va, da, 0);
      for (int64_t o = 0; o < n; o += 2 * k) {
        if (o + k < n) load_round(vb, db, o + k);
        store_round(va, da);
        if (o + k >= n) break;
        if (o + 2 * k < n) load_round(va, da, o + 2 * k);
        store_round(vb, db);
      }
      a = int64_t(__shfl_sync(0xffffffffu, raw, 0)) + base;
      continue;
    }
    for (int64_t it = a; it < e; ++it) {
      const uint8_t* src;
      uint8_t* dst;
      uint32_t bytes;
      item_addrs<D>(p, desc_at(p, j), c, q, src, dst, bytes);
      const int nvec = static_cast<int>(bytes >> 4);
      // rounds of 32 lanes x 8 vectors (4 KiB), ping-ponging between two
      // register sets: round r + 1's loads are issued before round r's stores
      auto load = [&](int4* v, int base) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + u * 32 + lane;
          if (idx < nvec) v[u] = ld_stream(src + size_t(idx) * 16);
        }
      };
      auto store = [&](const int4* v, int base) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + u * 32 + lane;
          if (idx < nvec) st_stream(dst + size_t(idx) * 16, v[u]);
        }
      };
      load(va, 0);
      for (int base = 0; base < nvec; base += 512) {
        if (base + 256 < nvec) load(vb, base + 256);
        store(va, base);
        if (base + 256 >= nvec) break;
        if (base + 512 < nvec) load(va, base + 512);
        store(vb, base + 256);
      }
      if (++q == p.npieces) {
        q = 0;
        if (++c == p.c0 + p.nc) {
          c = p.c0;
          ++j;
        }
      }
    }
    a = int64_t(__shfl_sync(0xffffffffu, raw, 0)) + base;
  }
  if (lane == 0) dyn_finish(p.work_ctr, total);
}

// The ring is driven by all 32 lanes of warp 0 in lockstep: they keep the
// same cursors and wait on the same mbarriers.  Whole-stage bulk copies
// (a piece of a large chunk, or the image side of a grouped unit: k chunks
// contiguous in the image) are issued by lane 0; the pool side of a grouped
// unit -- k separate chunks at scattered block addresses -- is spread over
// the lanes, lane t issuing chunk t (t + 32, ... when k > 32).  With small
// chunks (S <= 2 KiB: 16+ pool-side copies per 32 KiB stage) one issuing
// thread was the limit; the lanes compute their chunk
// addresses and issue their copies in parallel.  Each lane commits its own
// bulk-store groups and waits for them before the warp refills a stage.
template <Dir D, class P, int LW>
__global__ void __launch_bounds__(LW > 0 ? 32 * (1 + LW) : 32) swap_tma_kernel(const __grid_constant__ P p,
                                                                               const int stages) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t workers = gridDim.x * (1 + LW);   // claiming workers (LW > 0: every warp claims)
  if (LW > 0 && threadIdx.x >= 32) {
    ldst_worker<D>(p, int64_t(gridDim.x) * p.batch, workers);
    return;
  }
  const int lane = threadIdx.x;
  const int64_t stage_bytes = int64_t(p.piece) * p.group;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(stages) * stage_bytes);
  const int64_t G = gridDim.x, b = blockIdx.x;
  const bool dyn = p.batch > 0;          // claimed batches (a counter pair is always set then)
  // The next batch starts at G * batch + shfl(raw): `raw` is lane 0's claim
  // result, kept untouched until the switch that needs it so the atomic's
  // latency hides.
  int64_t i0, i1;
  uint32_t raw = 0;
  if (!dyn) {
    i0 = p.nitems * b / G;
    i1 = p.nitems * (b + 1) / G;
  } else {
    i0 = b * p.batch;
    i1 = i0 + p.batch < p.nitems ? i0 + p.batch : p.nitems;
    if (lane == 0) raw = claim_items(p.work_ctr, p.batch);
  }
  auto next_start = [&]() {
    const int64_t a = int64_t(__shfl_sync(0xffffffffu, raw, 0)) + G * p.batch;
    if (lane == 0) raw = claim_items(p.work_ctr, p.batch);
    return a;
  };
  if (i1 <= i0) {                        // fewer batches than CTAs: nothing of our own
    if (dyn && lane == 0) dyn_finish(p.work_ctr, workers);
    return;
  }
  if (lane == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = policy_evict_first();

  Unit lu, su;
  {
    Cursor cu;
    cu.init(i0, p);
    lu = Unit{cu.j, cu.c, cu.q, i1 - i0};
    su = lu;
  }
  // the first items of the batches the loader has entered but the storer
  // has not (the loader runs up to stages - 1 units ahead)
  int64_t queue[32];
  int qh = 0, qt = 0;
  auto open_batch = [&](int64_t a, Unit& u) {
    Cursor cu;
    cu.init(a, p);
    u = Unit{cu.j, cu.c, cu.q, (a + p.batch < p.nitems ? a + p.batch : p.nitems) - a};
  };
  int lstage = 0, issued = 0;
  auto issue_load = [&]() {
    const int k = unit_len(p, lu);
    const Desc d = desc_at(p, lu.j);
    uint8_t* buf = smem + size_t(lstage) * stage_bytes;
    const uint8_t* src;
    uint8_t* dst;
    uint32_t bytes;
    if (k == 1 || D != kOut) {             // one copy: a piece, or the image side of k chunks
      if (lane == 0) {
        item_addrs<D>(p, d, lu.c, lu.q, src, dst, bytes);
        mbar_expect_tx(&bars[lstage], bytes * k);
        bulk_g2s(buf, src, bytes * k, &bars[lstage], pol);
      }
    } else {                               // pool side: k scattered chunk loads over the lanes
      if (lane == 0) mbar_expect_tx(&bars[lstage], static_cast<uint32_t>(p.S) * k);
      __syncwarp();
      for (int t = lane; t < k; t += 32) {
        item_addrs<D>(p, d, lu.c + t, 0, src, dst, bytes);
        bulk_g2s(buf + size_t(t) * bytes, src, bytes, &bars[lstage], pol);
      }
    }
    unit_next(p, lu, k);
    if (dyn && lu.left == 0) {             // enter the next claimed batch, if any
      const int64_t a = next_start();
      if (a < p.nitems) {
        queue[qt++ & 31] = a;
        open_batch(a, lu);
      }
    }
    ++issued;
    if (++lstage == stages) lstage = 0;
  };
  while (lu.left > 0 && issued < stages - 1) issue_load();

  int sstage = 0;
  uint32_t parity = 0;
  while (su.left > 0) {
    mbar_wait(&bars[sstage], parity);
    const int k = unit_len(p, su);
    const Desc d = desc_at(p, su.j);
    uint8_t* buf = smem + size_t(sstage) * stage_bytes;
    const uint8_t* src;
    uint8_t* dst;
    uint32_t bytes;
    if (k == 1 || D != kIn) {              // one copy: a piece, or the image side of k chunks
      if (lane == 0) {
        item_addrs<D>(p, d, su.c, su.q, src, dst, bytes);
        bulk_s2g(dst, buf, bytes * k, pol);
      }
    } else {                               // pool side: k scattered chunk stores over the lanes
      for (int t = lane; t < k; t += 32) {
        item_addrs<D>(p, d, su.c + t, 0, src, dst, bytes);
        bulk_s2g(dst, buf + size_t(t) * bytes, bytes, pol);
      }
    }
    bulk_commit();
    unit_next(p, su, k);
    if (dyn && su.left == 0 && qh != qt) open_batch(queue[qh++ & 31], su);
    if (++sstage == stages) {
      sstage = 0;
      parity ^= 1u;
    }
    if (lu.left > 0) {
      bulk_wait_read<1>();  // this lane's stores of the previous unit have read its stage
      __syncwarp();         // ... and every other lane's
      issue_load();         // -> the stage of the previous unit
    }
  }
  bulk_wait<0>();
  if (dyn && lane == 0) dyn_finish(p.work_ctr, workers);
}

// ------------------------------------------------------------ LDG/STG kernel
// Grid-stride over items of up to 512*UNROLL bytes; a warp moves one item
// with UNROLL independent 16-byte loads per lane in flight.
// Streaming hints (ld.nc.L1::no_allocate.L2::256B / st.L1::no_allocate) and
// the next item's loads issued before the current item's stores (software
// pipelined; the plain and unpipelined flavours measured in round 1 were
// slower, profiles/r01_ldst_variants.jsonl).
template <Dir D, int UNROLL, class P>
__global__ void __launch_bounds__(256) swap_ldst_kernel(const __grid_constant__ P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  auto load = [&](int64_t it, int4* v, uint8_t** dst, int* nvec) {
    Cursor cu;
    cu.init(it, p);
    const uint8_t* src;
    uint32_t bytes;
    item_addrs<D>(p, desc_at(p, cu.j), cu.c, cu.q, src, *dst, bytes);
    *nvec = static_cast<int>(bytes >> 4);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int idx = u * 32 + lane;
      if (idx < *nvec) v[u] = ld_stream(src + size_t(idx) * 16);
    }
  };
  auto store = [&](const int4* v, uint8_t* dst, int nvec) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int idx = u * 32 + lane;
      if (idx < nvec) st_stream(dst + size_t(idx) * 16, v[u]);
    }
  };
  int4 a[UNROLL], b[UNROLL];
  uint8_t *da = nullptr, *db = nullptr;
  int na = 0, nb = 0;
  int64_t it = warp;
  if (it < p.nitems) load(it, a, &da, &na);
  while (it < p.nitems) {
    const int64_t nx = it + nwarps;
    if (nx < p.nitems) load(nx, b, &db, &nb);
    store(a, da, na);
    it = nx;
    if (it >= p.nitems) break;
    const int64_t ny = it + nwarps;
    if (ny < p.nitems) load(ny, a, &da, &na);
    store(b, db, nb);
    it = ny;
  }
}

// ------------------------------------------------------------ pattern (C-11)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t word(uint64_t seed, uint64_t pid, uint64_t t, uint64_t l, uint64_t kv,
                                         uint64_t h, uint64_t d) {
  const uint64_t pk = (pid << 46) | (t << 26) | (l << 18) | (kv << 17) | (h << 10) | d;
  return static_cast<uint32_t>(splitmix64(seed ^ pk) & 0xFFFFu);
}

// Thread = 8 consecutive 16-bit words (16 bytes) of one token row.  Index
// order d8, h, t, kv, l so that neighbouring threads write neighbouring bytes.
template <bool VERIFY>
__global__ void __launch_bounds__(256) pattern_kernel(const PatternParams p) {
  const int D8 = p.D >> 3;
  const int t_lo = VERIFY ? 0 : p.t0;
  const int64_t nt = p.t1 - t_lo;
  const int64_t total = int64_t(D8) * p.H * nt * 2 * p.L;
  unsigned long long bad = 0;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t r = idx;
    const int d8 = static_cast<int>(r % D8);
    r /= D8;
    const int h = static_cast<int>(r % p.H);
    r /= p.H;
    const int t = t_lo + static_cast<int>(r % nt);
    r /= nt;
    const int kv = static_cast<int>(r & 1);
    const int l = static_cast<int>(r >> 1);
    const int blk = __ldg(p.bt + t / p.bs);
    const int row = t % p.bs;
    uint8_t* a = reinterpret_cast<uint8_t*>(__ldg(p.layer_base + l)) + kv * p.P_kv + int64_t(blk) * p.P_b +
                 (int64_t(row * p.H + h) * p.D + d8 * 8) * 2;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t d = uint64_t(d8) * 8 + 2 * e;
      w[e] = word(p.seed, p.pid, t, l, kv, h, d) | (word(p.seed, p.pid, t, l, kv, h, d + 1) << 16);
    }
    if (VERIFY) {
      const uint4 got = *reinterpret_cast<const uint4*>(a);
      const uint32_t g[4] = {got.x, got.y, got.z, got.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        bad += ((g[e] & 0xFFFFu) != (w[e] & 0xFFFFu));
        bad += ((g[e] >> 16) != (w[e] >> 16));
      }
    } else {
      *reinterpret_cast<uint4*>(a) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  if (VERIFY) {
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(p.mismatches, bad);
  }
}

// Unit = 8 words of one token row, as in pattern_kernel; the item is found
// by binary search over the items' unit prefix sums.
__global__ void __launch_bounds__(256) pattern_fill_batch_kernel(const FillBatchParams p) {
  const int D8 = p.D >> 3;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < p.total_units;
       u += int64_t(gridDim.x) * blockDim.x) {
    int lo = 0, hi = p.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (p.items[mid].unit0 <= u) lo = mid; else hi = mid - 1;
    }
    const FillItem it = p.items[lo];
    int64_t r = u - it.unit0;
    const int d8 = static_cast<int>(r % D8);
    r /= D8;
    const int h = static_cast<int>(r % p.H);
    r /= p.H;
    const int64_t nt = it.t1 - it.t0;
    const int t = it.t0 + static_cast<int>(r % nt);
    r /= nt;
    const int kv = static_cast<int>(r & 1);
    const int l = static_cast<int>(r >> 1);
    const int blk = __ldg(p.bt_all + it.bt_off + t / p.bs);
    const int row = t % p.bs;
    uint8_t* a = reinterpret_cast<uint8_t*>(__ldg(p.layer_base + l)) + kv * p.P_kv + int64_t(blk) * p.P_b +
                 (int64_t(row * p.H + h) * p.D + d8 * 8) * 2;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t d = uint64_t(d8) * 8 + 2 * e;
      w[e] = word(p.seed, it.pid, t, l, kv, h, d) | (word(p.seed, it.pid, t, l, kv, h, d + 1) << 16);
    }
    *reinterpret_cast<uint4*>(a) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <typename K>
int grid_for(int64_t work_units, int per_cta, int num_sms, int ctas_per_sm, int grid_cap) {
  int64_t g = (work_units + per_cta - 1) / per_cta;
  int64_t cap = int64_t(num_sms) * ctas_per_sm;
  if (grid_cap > 0 && grid_cap < cap) cap = grid_cap;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}


// ------------------------------------------------------------ lender probe
// Checks, once per lent GPU arena, that the three kinds of access the copy
// engines make reach it correctly: plain 16-byte loads/stores (LDST engine),
// TMA bulk stores (swap_out) and TMA bulk loads (swap_in pull).  The first
// n bytes of the arena are saved in shared memory and restored at the end,
// so the probe leaves the arena's bytes as it found them (invariant I2).
// result bits: 1 plain ok, 2 bulk store ok, 4 bulk load ok.
constexpr int kProbeBytes = 4096;

__device__ __forceinline__ uint4 probe_word(int i, uint32_t salt) {
  const uint32_t x = 0x9E3779B9u * static_cast<uint32_t>(i + 1) ^ salt;
  return make_uint4(x, ~x, x * 3u, x ^ 0xA5A5A5A5u);
}
__device__ __forceinline__ bool same(const uint4& a, const uint4& b) {
  return a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w;
}

__global__ void __launch_bounds__(32) peer_probe_kernel(uint8_t* remote, int n, int* result) {
  __shared__ alignas(128) uint4 saved[kProbeBytes / 16];
  __shared__ alignas(128) uint4 buf[kProbeBytes / 16];
  __shared__ alignas(8) uint64_t bar;
  const int lane = threadIdx.x, nv = n / 16;
  volatile uint4* r = reinterpret_cast<volatile uint4*>(remote);
  bool plain = true, bstore = true, bload = true;
  for (int i = lane; i < nv; i += 32) {
    const uint4 v = const_cast<const uint4&>(r[i]);
    saved[i] = v;
  }
  // plain stores, read back
  for (int i = lane; i < nv; i += 32) const_cast<uint4&>(r[i]) = probe_word(i, 0x1234u);
  __threadfence_system();
  __syncwarp();
  for (int i = lane; i < nv; i += 32) plain = plain && same(const_cast<const uint4&>(r[i]), probe_word(i, 0x1234u));
  // a TMA bulk store of another pattern, read back with plain loads
  for (int i = lane; i < nv; i += 32) buf[i] = probe_word(i, 0xBEEFu);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(remote),
                 "r"(smem_u32(buf)), "r"(nv * 16)
                 : "memory");
    bulk_commit();
    bulk_wait<0>();
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncwarp();
  __threadfence_system();
  for (int i = lane; i < nv; i += 32) bstore = bstore && same(const_cast<const uint4&>(r[i]), probe_word(i, 0xBEEFu));
  // plain stores of a third pattern, fetched with a TMA bulk load
  for (int i = lane; i < nv; i += 32) {
    const_cast<uint4&>(r[i]) = probe_word(i, 0x5151u);
    buf[i] = make_uint4(0, 0, 0, 0);
  }
  __threadfence_system();
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    mbar_expect_tx(&bar, nv * 16);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(buf)),
        "l"(remote), "r"(nv * 16), "r"(smem_u32(&bar))
        : "memory");
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  for (int i = lane; i < nv; i += 32) bload = bload && same(buf[i], probe_word(i, 0x5151u));
  // restore the arena's bytes
  for (int i = lane; i < nv; i += 32) const_cast<uint4&>(r[i]) = saved[i];
  __threadfence_system();
  const unsigned ok_plain = __all_sync(0xffffffffu, plain), ok_bs = __all_sync(0xffffffffu, bstore),
                 ok_bl = __all_sync(0xffffffffu, bload);
  if (lane == 0) *result = (ok_plain ? 1 : 0) | (ok_bs ? 2 : 0) | (ok_bl ? 4 : 0);
}

}  // namespace

cudaError_t launch_peer_probe(uint8_t* remote, int64_t bytes, int* d_result, cudaStream_t s) {
  const int n = static_cast<int>(std::min<int64_t>(bytes, kProbeBytes)) & ~15;
  if (n <= 0) return cudaSuccess;
  peer_probe_kernel<<<1, 32, 0, s>>>(remote, n, d_result);
  return cudaGetLastError();
}

namespace {

}  // namespace

int tma_smem_bytes(int piece, int stages) { return piece * stages + 8 * stages; }

namespace {

// One ring kernel instantiation (LW register warps); the opt-in shared
// memory attribute is per device and per instantiation: set once.
template <int LW, class P>
cudaError_t launch_ring(const P& p, Dir dir, int grid, int smem, int stages, cudaStream_t s, int dev) {
  static thread_local bool set_smem[3][64] = {};
  bool& have = set_smem[dir][dev & 63];
  if (!have) {
    const cudaError_t e = cudaFuncSetAttribute(dir == kOut  ? swap_tma_kernel<kOut, P, LW>
                                               : dir == kIn ? swap_tma_kernel<kIn, P, LW>
                                                            : swap_tma_kernel<kMig, P, LW>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    have = true;
  }
  constexpr int nt = 32 * (1 + LW);
  if (dir == kOut)
    swap_tma_kernel<kOut, P, LW><<<grid, nt, smem, s>>>(p, stages);
  else if (dir == kIn)
    swap_tma_kernel<kIn, P, LW><<<grid, nt, smem, s>>>(p, stages);
  else
    swap_tma_kernel<kMig, P, LW><<<grid, nt, smem, s>>>(p, stages);
  return cudaGetLastError();
}

template <class P>
cudaError_t launch_tma_t(const P& p, Dir dir, int num_sms, int grid_cap, int stages_opt, cudaStream_t s,
                         int* ctas_used, int variant, LaunchInfo* info) {
  // One CTA per SM and a shallow ring: 3 x 32 KiB or 64 KiB of loads in
  // flight per SM measured best for HBM on B200 (profiles/r01_stages.jsonl);
  // deeper rings lose 3-4 %.
  const int stage_bytes = p.piece * p.group;
  const int grid = grid_for<void>(p.nitems, 1, num_sms, 1, grid_cap);
  // Ring depth: keep ~9 MiB of loads in flight chip-wide.  With all 148 SMs
  // that is 3 x 32 KiB stages (2 in flight), measured best; with an SM cap
  // each CTA needs a deeper ring: 64 CTAs x 6 stages still reach 6.26 TB/s
  // (profiles/r01_stages*.jsonl, r01_ctas_stages.jsonl).  At most ~200 KiB.
  int stages = stages_opt;
  if (stages <= 0) {
    const int64_t want_inflight = int64_t(9) << 20;
    const int64_t per_cta = (want_inflight + int64_t(grid) * stage_bytes - 1) / (int64_t(grid) * stage_bytes);
    stages = static_cast<int>(std::min<int64_t>(per_cta + 1, std::max(3, (200 * 1024) / stage_bytes)));
    stages = std::max(stages, 3);
    // claimed batches run best one stage deeper: 4 x 32 KiB at 148 CTAs
    // (profiles/r01_tma_sched6.jsonl: C2 6.79 vs 6.74 TB/s, C4 6.72 vs 6.54)
    if (p.work_ctr) stages = std::max(stages, 4);
  }
  stages = std::max(2, std::min(stages, 32));
  while (stages > 2 && tma_smem_bytes(stage_bytes, stages) > 227 * 1024) --stages;
  if (tma_smem_bytes(stage_bytes, stages) > 227 * 1024) return cudaErrorInvalidConfiguration;
  const int smem = tma_smem_bytes(stage_bytes, stages);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const bool hybrid = variant == 3;
  // variant 3: TMA ring + 8 register warps per CTA (4 and 16 measured worse,
  // profiles/r02_hybrid_warps.jsonl)
  constexpr int kLdstWarps = 8;
  int nt = 32;
  if (hybrid) {
    if (!p.work_ctr) return cudaErrorInvalidValue;    // the LDST warps only claim batches
    e = launch_ring<kLdstWarps>(p, dir, grid, smem, stages, s, dev);
    nt = 32 * (1 + kLdstWarps);
  } else {
    e = launch_ring<0>(p, dir, grid, smem, stages, s, dev);
  }
  if (e != cudaSuccess) return e;
  if (ctas_used) *ctas_used = grid;
  if (info) *info = LaunchInfo{grid, nt, stages};
  return cudaGetLastError();
}

// Small chunks through registers (AQUA_OPT_LDST_VARIANT 3; AUTO for chunks
// below 2 KiB).  A bulk copy costs the SM's TMA unit ~90 cycles whatever its
// size (profiles/r02_scatter_probe.jsonl: TMA reads of 512 B runs top out at
// 1.67 TB/s, of 1 KiB runs at 3.08), while 16-byte loads of scattered 512 B
// runs reach 6.9 TB/s -- DRAM does not mind the scatter.  So for chunks of
// 512 B .. 4 KiB (nvec = S/16 vectors, nvec | 256) each warp moves rounds of
// 4 KiB = 256 / nvec whole chunks: slot u of every lane belongs to chunk
// (32 u) / nvec of the round (warp-uniform: one descriptor, one layer base,
// one address per slot for the whole warp), vector (32 u + lane) % nvec of
// it; all 8 loads of a round are in flight before its 8 stores.  Rounds are
// dealt grid-stride (static, like the probe's scattered copy that reaches
// 6.3 / 6.4 TB/s at 512 B / 1 KiB).  The (descriptor, chunk) of slot 0 is
// divided out once per round; the other slots step from it.
template <Dir D, class P, int NT>
__global__ void __launch_bounds__(NT) swap_small_kernel(const __grid_constant__ P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int nvec = static_cast<int>(p.S >> 4);
  const int k = 256 / nvec;                             // chunks per round
  const int64_t nrounds = (p.nitems + k - 1) / k;
  for (int64_t r = warp; r < nrounds; r += nwarps) {
    const int64_t i0 = r * k;
    int64_t j = i0 / p.nc;
    int32_t c = p.c0 + static_cast<int32_t>(i0 - j * p.nc);
    // pointers of chunk (j, c); the next chunk of the same descriptor is
    // one S further in the image and, in the pool, the V plane of the same
    // layer (+ P_kv) or the next layer's K plane (layer base + block offset)
    const uint8_t* src;
    uint8_t* dst;
    uint32_t bytes;
    int64_t boff = 0;
    auto locate = [&]() {
      const Desc d = desc_at(p, j);
      item_addrs<D>(p, d, c, 0, src, dst, bytes);
      boff = int64_t(d.block) * p.P_b;
    };
    auto step = [&]() {
      if (++c == p.c0 + p.nc) {
        c = p.c0;
        ++j;
        if (j < p.ndesc) locate();
        return;
      }
      if (D == kMig) {
        src += p.S;
        dst += p.S;
        return;
      }
      uint8_t* pool;
      if (!p.kv_merged && (c & 1))                      // K -> V of the same layer
        pool = const_cast<uint8_t*>(D == kOut ? src : dst) + p.P_kv;
      else                                              // next layer's K plane
        pool = reinterpret_cast<uint8_t*>(__ldg(p.layer_base + (p.kv_merged ? c : c >> 1))) + boff;
      if (D == kOut) {
        src = pool;
        dst += p.S;
      } else {
        src += p.S;
        dst = pool;
      }
    };
    locate();
    int4 v[8];
    uint8_t* dp[8];
    int t_prev = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = (u * 32) / nvec;                    // chunk of the round (uniform)
      if (t != t_prev) {
        step();
        t_prev = t;
      }
      dp[u] = nullptr;
      if (i0 + t < p.nitems) {
        const size_t vo = size_t((u * 32) % nvec + lane) * 16;
        v[u] = ld_stream(src + vo);
        dp[u] = dst + vo;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (dp[u]) st_stream(dp[u], v[u]);
  }
}

template <class P>
cudaError_t launch_ldst_t(const P& p, Dir dir, int num_sms, int grid_cap, cudaStream_t s, int* ctas_used,
                          int variant, LaunchInfo* info) {
  // small-chunk kernel: 2 CTAs of 8 warps per SM (1 .. 8 measured,
  // profiles/r02_small_ldst*.jsonl: 2 is the best or within 2 % of it)
  constexpr int small_cps = 2;
  if (variant == 3) {                    // small chunks: rounds of whole chunks through registers
    const int k = 256 / static_cast<int>(p.S >> 4);
    const int64_t rounds = (p.nitems + k - 1) / k;
    // Under an SM cap (fewer CTAs than 2 per SM) each CTA gets the SM's
    // whole register budget for warps: 16 warps (512 threads at 108
    // registers) instead of 8, twice the 4 KiB rounds in flight per SM
    const bool capped = grid_cap > 0 && grid_cap < num_sms * small_cps;
    const int nt = capped ? 512 : 256;
    const int grid = grid_for<void>(rounds, nt / 32, num_sms, capped ? 1 : small_cps, grid_cap);
    if (capped) {
      if (dir == kOut)
        swap_small_kernel<kOut, P, 512><<<grid, 512, 0, s>>>(p);
      else if (dir == kIn)
        swap_small_kernel<kIn, P, 512><<<grid, 512, 0, s>>>(p);
      else
        swap_small_kernel<kMig, P, 512><<<grid, 512, 0, s>>>(p);
    } else if (dir == kOut) {
      swap_small_kernel<kOut, P, 256><<<grid, 256, 0, s>>>(p);
    } else if (dir == kIn) {
      swap_small_kernel<kIn, P, 256><<<grid, 256, 0, s>>>(p);
    } else {
      swap_small_kernel<kMig, P, 256><<<grid, 256, 0, s>>>(p);
    }
    if (ctas_used) *ctas_used = grid;
    if (info) *info = LaunchInfo{grid, nt, 0};
    return cudaGetLastError();
  }
  // software pipelined, one 256-thread CTA per SM: 6,624 / 6,572 GB/s on C2
  // (profiles/r01_ldst_variants.jsonl)
  const int grid = grid_for<void>(p.nitems, 8, num_sms, 1, grid_cap);
  if (dir == kOut)
    swap_ldst_kernel<kOut, 8, P><<<grid, 256, 0, s>>>(p);
  else if (dir == kIn)
    swap_ldst_kernel<kIn, 8, P><<<grid, 256, 0, s>>>(p);
  else
    swap_ldst_kernel<kMig, 8, P><<<grid, 256, 0, s>>>(p);
  if (ctas_used) *ctas_used = grid;
  if (info) *info = LaunchInfo{grid, 256, 0};
  return cudaGetLastError();
}

// Builds the parameter block of the smallest size class that holds the
// call's inline descriptors and hands it to `f`.
template <class F>
cudaError_t with_params(const SwapHeader& h, const Desc* inl, F&& f) {
  if (h.desc || h.ndesc <= kInlineDesc) {
    SwapParamsT<kInlineDesc> p;
    static_cast<SwapHeader&>(p) = h;
    if (!h.desc) std::copy(inl, inl + h.ndesc, p.inl);
    return f(p);
  }
  if (h.ndesc > kInlineDescBig || !inl) return cudaErrorInvalidValue;
  static thread_local SwapParamsT<kInlineDescBig> p;   // 32 KiB: off the stack
  static_cast<SwapHeader&>(p) = h;
  std::copy(inl, inl + h.ndesc, p.inl);
  return f(p);
}

}  // namespace

cudaError_t launch_swap_tma(const SwapHeader& h, const Desc* inl, Dir dir, int num_sms, int grid_cap,
                            int stages_opt, cudaStream_t s, int* ctas_used, int variant, LaunchInfo* info) {
  if (h.nitems == 0) return cudaSuccess;
  return with_params(h, inl, [&](const auto& p) {
    return launch_tma_t(p, dir, num_sms, grid_cap, stages_opt, s, ctas_used, variant, info);
  });
}

cudaError_t launch_swap_ldst(const SwapHeader& h, const Desc* inl, Dir dir, int num_sms, int grid_cap,
                             cudaStream_t s, int* ctas_used, int variant, LaunchInfo* info) {
  if (h.nitems == 0) return cudaSuccess;
  return with_params(h, inl, [&](const auto& p) {
    return launch_ldst_t(p, dir, num_sms, grid_cap, s, ctas_used, variant, info);
  });
}

cudaError_t launch_pattern_fill(const PatternParams& p, int num_sms, cudaStream_t s) {
  const int64_t total = int64_t(p.D / 8) * p.H * (p.t1 - p.t0) * 2 * p.L;
  if (total <= 0) return cudaSuccess;
  const int grid = grid_for<void>(total, 256, num_sms, 8, 0);
  pattern_kernel<false><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_pattern_fill_batch(const FillBatchParams& p, int num_sms, cudaStream_t s) {
  if (p.total_units <= 0) return cudaSuccess;
  const int grid = grid_for<void>(p.total_units, 256, num_sms, 8, 0);
  pattern_fill_batch_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_pattern_verify(const PatternParams& p, int num_sms, cudaStream_t s) {
  const int64_t total = int64_t(p.D / 8) * p.H * p.t1 * 2 * p.L;
  if (total <= 0) return cudaSuccess;
  const int grid = grid_for<void>(total, 256, num_sms, 8, 0);
  pattern_kernel<true><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace aqua
