// Internal interface between the host library (aqua_host.cpp) and the
// sm_100a kernels (aqua_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace aqua {

// One swap descriptor: a pool block and an arena slot.  The arena index
// (0 = GPU lender / self-lender, 1 = pinned host) rides in bit 31 of slot.
struct Desc {
  int32_t block;
  uint32_t slot_arena;
};
constexpr uint32_t kArenaBit = 0x80000000u;

// swap_out: pool -> arena; swap_in: arena -> pool; migrate: arena -> arena
// (for kMig the descriptor's `block` field holds the SOURCE slot, with the
// source arena in bit 31, reinterpreted as uint32).
enum Dir : int { kOut = 0, kIn = 1, kMig = 2 };

// Calls with at most kInlineDesc descriptors pass them inside the kernel
// parameters (__grid_constant__): no staging copy on the critical path.
// Two parameter sizes: 2 KiB of descriptors (small calls keep a small launch)
// and, up to kInlineDescBig, the large-parameter launch of CUDA 12.1+ (32,764
// bytes of parameters on sm_70+), which covers e.g. a 32K-token Llama-3-8B
// prompt (2,048 blocks) in one launch without a descriptor upload.  Larger
// calls go through the pinned staging ring + one H2D copy.
constexpr int kInlineDesc = 256;
constexpr int kInlineDescBig = 4064;

struct SwapHeader {
  const Desc* desc;            // device array [ndesc], or nullptr -> use the inline array
  const uint64_t* layer_base;  // device array [L]
  uint64_t arena_base[2];      // device-visible bases: [0] GPU lender, [1] host
  int64_t ndesc;
  int32_t L;
  int32_t piece;               // bytes per work item (multiple of 16, divides nothing in particular)
  int32_t npieces;             // ceil(S / piece)
  int32_t group;               // TMA: chunks per stage when npieces == 1 (else 1)
  int32_t c0, nc;              // chunk range [c0, c0+nc) of each block (layer-wise: c = 2l + kv)
  int64_t S, U, P_kv, P_b;
  int64_t nitems;              // ndesc * nc * npieces
  // TMA engine work distribution.  batch == 0: each CTA one contiguous item
  // range.  batch > 0: batches of `batch` items, CTA b starting on batch b,
  // then claims through this {items claimed, workers done} counter pair,
  // which the last claiming worker resets to {0, 0}.  The hybrid's register
  // warps claim batches of batch_ldst items (0: batch).
  uint32_t* work_ctr;
  int32_t batch;
  int32_t batch_ldst;
  int32_t pack_vec;            // register movers pack whole chunks of <= pack_vec 16-byte vectors per round
  int32_t kv_merged;           // 1: a "chunk" is a layer's adjacent K+V pair (c = l, S = 2 x chunk bytes)
};
// Counter pairs per context for dynamically scheduled launches; a pair is
// reused only after the ticket of its last launch (stream-ordered, like R7).
constexpr int kCtrSlots = 256;

// The kernel parameter block: header + N inline descriptors.
template <int N>
struct SwapParamsT : SwapHeader {
  Desc inl[N];                 // inline descriptors when desc == nullptr
};
static_assert(sizeof(SwapParamsT<kInlineDescBig>) + 16 <= 32764, "kernel parameter limit");

struct PatternParams {
  const int32_t* bt;           // device block table of the prompt
  const uint64_t* layer_base;
  int64_t P_kv, P_b;
  int32_t L, bs, H, D;
  int32_t t0, t1;              // fill: tokens [t0, t1); verify: [0, t1)
  uint64_t pid, seed;
  unsigned long long* mismatches;  // verify only
};

// Batched fill: one launch writes token ranges of many prompts.
struct FillItem {
  uint64_t pid;
  int64_t unit0;               // first work unit of this item (prefix sum)
  int32_t bt_off;              // offset of its block table in the shared array
  int32_t t0, t1;
};
struct FillBatchParams {
  const FillItem* items;       // device [n]
  const int32_t* bt_all;       // device concatenated block tables
  const uint64_t* layer_base;
  int64_t P_kv, P_b;
  int64_t total_units;
  int32_t n, L, bs, H, D;
  uint64_t seed;
};
cudaError_t launch_pattern_fill_batch(const FillBatchParams& p, int num_sms, cudaStream_t s);

// Launchers: return the CUDA error of the launch (cudaSuccess on success).
// grid_cap = max CTAs (0 = derived from the SM count).
// What a launcher launched (reported by aqua_last_launch).
struct LaunchInfo {
  int grid = 0, threads = 0, stages = 0;
};

// h.desc == nullptr: the h.ndesc descriptors at `inl` (host memory, at most
// kInlineDescBig) are copied into the kernel parameters.
cudaError_t launch_swap_tma(const SwapHeader& h, const Desc* inl, Dir dir, int num_sms, int grid_cap, int stages,
                            cudaStream_t s, int* ctas_used, int variant = 0, LaunchInfo* info = nullptr);
// variant 3: the small-chunk kernel (h.S = 512 B .. 4 KiB, S/16 | 256, h.piece = h.S); else 2.
cudaError_t launch_swap_ldst(const SwapHeader& h, const Desc* inl, Dir dir, int num_sms, int grid_cap,
                             cudaStream_t s, int* ctas_used, int variant = 2, LaunchInfo* info = nullptr);
cudaError_t launch_pattern_fill(const PatternParams& p, int num_sms, cudaStream_t s);
cudaError_t launch_pattern_verify(const PatternParams& p, int num_sms, cudaStream_t s);

// One-warp probe of a lent GPU arena (aqua_lend): plain, TMA bulk-store and
// TMA bulk-load round trips over its first <= 4 KiB, which it restores.
// *d_result bits: 1 plain ok, 2 bulk store ok, 4 bulk load ok.
cudaError_t launch_peer_probe(uint8_t* arena, int64_t bytes, int* d_result, cudaStream_t s);

// Max dynamic shared memory the TMA kernel will request (for attribute setup).
int tma_smem_bytes(int piece, int stages);

}  // namespace aqua
