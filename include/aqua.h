/*
 * aqua.h -- C ABI of libaqua: B200-native preempt/resume paging of a
 * prompt's paged KV cache into HBM lent by a peer GPU (NVLink 5 / NVSwitch),
 * with pinned host DRAM as the fallback.  From-scratch implementation of the
 * data path of arXiv 2407.21255 ("Aqua").
 *
 * Citations: P:n = line n of the paper text, S:n = line n of
 * SPEC.md; the section is named beside each.  Readings R1..R18 are listed
 * in DESIGN.md.
 *
 * The operations (paper):
 *   - AquaTensor swap space on a producer GPU, DRAM fallback: Sec. 6
 *     "Allocating AquaTensors" P:737-756 and fig:aqua_design P:668-676
 *     ("If GPU 0 only has enough memory to offload one tensor, AquaLib falls
 *     back to the host DRAM"); one producer per consumer, Sec. 5 P:529-534.
 *   - preemption = paging out the prompts not in the next batch, resumption
 *     = paging in the prompts not on the GPU: Sec. 7 P:836-837.
 *   - gather the per-layer KV pieces and copy them to the AquaTensor;
 *     copy back and scatter: Sec. 7 "Efficient context switching" P:840-853.
 *   - location query: P:855-857.  Library surface: Sec. 8 P:864.
 * The paged block pool / block table is the vLLM v0.5.3 substrate the paper
 * modifies; its layout is reading R1.
 *
 * Sizes.  S = block_tokens * num_kv_heads * head_dim * elem_bytes is one
 * (layer, K|V, block) chunk; U = 2 * num_layers * S is one block across all
 * layers and K/V, the unit of work and the size of one swap slot.
 *
 * Byte definitions (exact; tolerance 0):
 *   chunk(l, kv, b) = bytes [kv*kv_plane_stride + b*block_stride, +S) of
 *                     layer_base[l]                                   (R1)
 *   slot s of an arena = bytes [s*U, (s+1)*U); chunk (l, kv) of a block's
 *                     image at offset (2*l + kv)*S inside its slot      (R3)
 *   swap_out: arena[slot_j*U + (2l+kv)*S + x] = chunk(l, kv, bt[j])[x]
 *   swap_in:  chunk(l, kv, new_j)[x] = arena[slot_j*U + (2l+kv)*S + x]
 * Whole blocks are copied, the unused tail of a last block included (R6).
 *
 * Allocation policy (R4): blocks and slots are taken lowest-id-first,
 * ascending, in call order.  Placement (R5): each prompt's whole image goes
 * to the peer lender if it has enough free slots, else to the host arena,
 * else the call fails with AQUA_E_NOSPACE.
 *
 * Ownership.  The KV pool belongs to the caller (e.g. torch tensors); the
 * library stores its pointers only.  An arena is owned by the library iff
 * aqua_lend was called with base == NULL.  All out-arrays are
 * caller-allocated host memory.
 *
 * Errors.  Negative status codes.  Every call validates completely before
 * changing any state: a failing call changes nothing (all-or-nothing, as
 * SPEC S:376).  AQUA_E_CUDA is sticky: the ctx is poisoned and every later
 * call on it returns AQUA_E_CUDA.  aqua_last_error(ctx) gives a message.
 *
 * Streams and tickets.  Copies are enqueued on the caller's stream after the
 * work already queued there.  Each swap returns a ticket (an event recorded
 * after its copy).  The library itself orders every reuse of a block or slot
 * after the last library operation that touched it (R7: stream-ordered
 * deferred reuse instead of the paper's "transfers at loop boundaries",
 * P:866), and makes swap_in wait for the swap_out that wrote the image.
 * The caller orders its own work: the swap stream must wait for the decode
 * that wrote the blocks being swapped out (cudaStreamWaitEvent), and decode
 * must wait for a swap_in ticket (aqua_wait) before reading the blocks.
 *
 * Thread safety: a ctx is not thread-safe; distinct ctxs are independent.
 * No CPU fallback: without a GPU only AQUA_DRYRUN contexts work (bookkeeping
 * and descriptors, no data movement) -- every data call on a real context
 * fails with AQUA_E_CUDA if the device is unusable.
 */
#ifndef AQUA_H_
#define AQUA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define AQUA_API __attribute__((visibility("default")))
#else
#define AQUA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* aqua_stream_t;  /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  AQUA_OK = 0,
  AQUA_E_INVAL = -1,    /* bad argument; nothing changed */
  AQUA_E_NOBLOCKS = -2, /* the local pool cannot satisfy the call; preempt first */
  AQUA_E_NOSPACE = -3,  /* neither the lender nor the host arena can hold an image */
  AQUA_E_STATE = -4,    /* unknown pid or wrong state (e.g. swap_out of a SWAPPED prompt) */
  AQUA_E_CUDA = -5,     /* CUDA error; the ctx is poisoned */
  AQUA_E_PEER = -6      /* lender unreachable (no P2P access / IPC handle will not open) */
} aqua_status;

enum { AQUA_HOST = -1,     /* aqua_lend lender_device: pinned host DRAM (the paper's baseline) */
       AQUA_MAPPED = -3 }; /* aqua_lend lender_device: caller-mapped peer memory (IPC import) */
enum { AQUA_DRYRUN = -2 }; /* aqua_create device: bookkeeping + descriptors only, no CUDA */

enum { AQUA_ST_RESIDENT = 1, AQUA_ST_SWAPPED = 2 };
enum { AQUA_LOC_LOCAL = 0, AQUA_LOC_PEER = 1, AQUA_LOC_HOST = 2 };

/* Copy engines for aqua_set_option(AQUA_OPT_KERNEL).  AUTO, TMA, LDST and
 * CE_HOST are the product; PER_CHUNK and GATHER_TEMP are baselines kept for
 * measurement only.  Value 5 (a batched-memcpy baseline in round 1) is
 * retired and rejected with AQUA_E_INVAL.  The environment variable AQUA_KERNEL
 * (auto | tma | ldst | ce_host) sets a context's initial engine. */
enum {
  AQUA_KERNEL_AUTO = 0,       /* product default: CE_HOST when every image of the call is in host DRAM; a call with
                                 images in both arenas is split (GPU-arena images as below, host images CE_HOST);
                                 migrations on the copy engines (one DMA per run of consecutive slots); the LDST
                                 small-chunk kernel for plane-major 512 B and 1 KiB chunks (capped launches on a peer arena
                                 excepted); else TMA (picked from measurements) */
  AQUA_KERNEL_TMA = 1,        /* fused gather/scatter, cp.async.bulk smem ring (UBLKCP) */
  AQUA_KERNEL_LDST = 2,       /* fused gather/scatter, 16-byte LDG/STG register path */
  AQUA_BASE_PER_CHUNK = 3,    /* baseline: one cudaMemcpyAsync per chunk (vLLM-style) */
  AQUA_BASE_GATHER_TEMP = 4,  /* baseline: the paper's gather-to-temp + one copy */
  AQUA_KERNEL_CE_HOST = 6     /* host images via a GPU staging buffer + DMA copy engines (full-duplex PCIe);
                                 GPU-lender images still use the TMA kernel */
};
enum {
  AQUA_OPT_KERNEL = 1,        /* one of AQUA_KERNEL_* / AQUA_BASE_* */
  AQUA_OPT_MAX_CTAS = 2,      /* cap on CTAs per swap launch (0 = all SMs); SMs left for decode */
  AQUA_OPT_TMA_PIECE = 3,     /* bytes per TMA stage (multiple of 16, <= 65536; 0 = auto: 32 KiB) */
  AQUA_OPT_TMA_STAGES = 4,    /* TMA ring depth (2..32; 0 = auto: ~9 MiB of loads in flight chip-wide, 3..~200 KiB) */
  AQUA_OPT_TIMING = 5,        /* 1: each swap also records a start event; aqua_ticket_elapsed gives its device time */
  AQUA_OPT_LDST_VARIANT = 6,  /* LDST engine flavour: 2 (default) grid-stride 4 KiB items, software-pipelined;
                                 3 the small-chunk kernel (chunks of 512 B .. 4 KiB moved whole, several per 4 KiB
                                 register round, 2 CTAs of 8 warps per SM, or 16-warp CTAs under a CTA cap; AUTO picks it for
                                 plane-major 512 B / 1 KiB chunks; other chunk sizes fall back to 2).  0 and 1 (round-1 experiments) were retired: E_INVAL */
  AQUA_OPT_TMA_VARIANT = 7,   /* TMA engine: 0 (default) one ring per CTA driven by one warp; 3 hybrid: the ring
                                 plus 8 warps copying claimed batches through registers.  1 and 2 (warp-specialised,
                                 two rings) reached the same HBM rate in round 1 and were retired: AQUA_E_INVAL */
  AQUA_OPT_INLINE_MAX = 8,    /* largest call (in blocks, per launch) whose descriptors ride in the kernel
                                 parameters instead of a pinned-ring upload + H2D copy: 0..4064 (default 4064,
                                 the 32,764-byte parameter limit of CUDA 12.1+; 256 = the small parameter block) */
  AQUA_OPT_TMA_SCHED = 9,     /* TMA engine work distribution: 0 = each CTA one contiguous item range;
                                 n > 0 = batches of n ring units claimed dynamically (atomic counter per launch);
                                 AQUA_TMA_SCHED_AUTO (default) = the AUTO policy.  Round-robin
                                 batches (-n) were retired in round 2: AQUA_E_INVAL */
  AQUA_OPT_TMA_STATIC_PCT = 10, /* retired in round 2 (a static head before the claimed batches): only 0 */
  AQUA_OPT_RATE_GBPS = 11,    /* paging budget in GB/s of swap per direction (0 = off): the copy kernels run on
                                 ceil(rate / 50) SMs (one SM moves ~50 GB/s of swap on the HBM path), leaving the other
                                 SMs and HBM bandwidth to decode; combines with AQUA_OPT_MAX_CTAS (the smaller cap wins) */
  AQUA_OPT_PEER_CTAS = 12,    /* CTA cap for launches that touch a PEER lender's arena (another GPU's HBM over
                                 NVLink; 0 = all SMs).  Default 32: one SM issues ~63 GB/s of HBM writes and keeps
                                 ~200 KiB of copies in flight under a cap, so ~15 SMs could carry
                                 900 GB/s per direction; 32 leaves 2x margin for NVLink latency and the other 116
                                 SMs to decode.  A placeholder until the per-SM NVLink rate is measured
                                 (scripts/nvlink_peer.py); the smallest of this, MAX_CTAS and RATE_GBPS wins */
  AQUA_OPT_PEER_TEST = 13     /* test hook, set before aqua_lend: 1 treats the next GPU arena as a peer (probe +
                                 peer cap) even on the borrower's own device; 2 also makes its bulk-copy probe fail
                                 (the LDST fallback); 0 (default) detects peers from the arena's device */
};

enum { AQUA_TMA_SCHED_AUTO = 1 << 30 };

typedef struct aqua_ctx aqua_ctx;   /* one per borrower device (per TP rank) */

typedef struct {
  int32_t num_layers;        /* L */
  int32_t block_tokens;      /* bs */
  int32_t num_kv_heads;      /* H (per TP shard) */
  int32_t head_dim;          /* D */
  int32_t elem_bytes;        /* e (2 for fp16/bf16; opaque: no arithmetic on values) */
  int32_t num_blocks;        /* NB */
  void* const* layer_base;   /* L device pointers, 16-byte aligned, caller-owned; copied at create */
  int64_t kv_plane_stride;   /* bytes from the K plane to the V plane of a layer (flash: NB*S); 0 = NB*S */
  int64_t block_stride;      /* bytes between consecutive blocks (flash: S); 0 = S */
} aqua_kv_layout;

/* Create a context for borrower `device` (a CUDA device ordinal, or
 * AQUA_DRYRUN).  Validates the layout: all sizes > 0, S and both strides
 * multiples of 16, chunks of distinct (kv, b) do not overlap, pointers
 * 16-byte aligned.  *out = NULL on failure. */
AQUA_API aqua_status aqua_create(int device, const aqua_kv_layout* layout, aqua_ctx** out);
/* Waits for outstanding tickets, frees library-owned arenas, then the ctx. */
AQUA_API aqua_status aqua_destroy(aqua_ctx* ctx);

/* Register swap space lent to this borrower (AquaTensor backing store).
 * lender_device: a device ordinal (a peer, or this device = "self-lender"),
 * AQUA_HOST (pinned host DRAM), or AQUA_MAPPED (base is peer memory already
 * mapped into this process, e.g. from aqua_ipc_import).
 * base == NULL: the library allocates `bytes` (cudaMalloc on the lender /
 * cudaHostAlloc mapped) and owns it.  base != NULL: caller-owned, must
 * outlive the ctx, 16-byte aligned.  Capacity = floor(bytes / U) slots.
 * At most one GPU lender (device or mapped) per ctx plus one
 * host arena: a second one is AQUA_E_INVAL.  A device lender that cannot be
 * reached by P2P gives AQUA_E_PEER (the caller may fall back to AQUA_HOST,
 * as the paper does).  out_nslots may be NULL. */
AQUA_API aqua_status aqua_lend(aqua_ctx* ctx, int lender_device, void* base, uint64_t bytes,
                      int32_t* out_nslots);

/* Append n fresh blocks (lowest free ids, ascending) to prompt pid, creating
 * it RESIDENT if new; the ids are written to out_ids[n].  `stream` is where
 * the caller will write the blocks: it is made to wait for any in-flight
 * library copy that last touched them.  AQUA_E_NOBLOCKS if fewer than n are
 * free; AQUA_E_STATE if pid is SWAPPED. */
AQUA_API aqua_status aqua_alloc_blocks(aqua_ctx* ctx, uint64_t pid, int32_t n, aqua_stream_t stream,
                              int32_t* out_ids);
/* Append caller-chosen block ids in the given order (an engine keeping its
 * own block list).  Every id must be in [0, NB), free and distinct, else
 * AQUA_E_INVAL.  Same stream rule as aqua_alloc_blocks. */
AQUA_API aqua_status aqua_adopt_blocks(aqua_ctx* ctx, uint64_t pid, int32_t n, const int32_t* ids,
                              aqua_stream_t stream);

/* Preempt: for each pid (RESIDENT, listed once) in
 * call order, place its image (R5), enqueue ONE batched fused gather->store
 * launch for all of them on `stream`, release their blocks (reusable after
 * the ticket, R7) and mark them SWAPPED.  *out_ticket (nullable) gets the
 * completion ticket (0 if nothing was copied). */
AQUA_API aqua_status aqua_swap_out(aqua_ctx* ctx, int32_t n, const uint64_t* pids, aqua_stream_t stream,
                          uint64_t* out_ticket);
/* Resume: for each pid (SWAPPED, listed once) in call
 * order, allocate fresh blocks (R4), enqueue one batched load->scatter launch
 * on `stream`, release the slots and mark the prompts RESIDENT.  out_ids gets
 * the concatenated new block tables in pid order (capacity out_ids_cap
 * entries; too small -> AQUA_E_INVAL), out_counts[n] the per-prompt counts.
 * AQUA_E_NOBLOCKS if the pool cannot hold them all. */
AQUA_API aqua_status aqua_swap_in(aqua_ctx* ctx, int32_t n, const uint64_t* pids, aqua_stream_t stream,
                         int32_t* out_ids, int64_t out_ids_cap, int32_t* out_counts,
                         uint64_t* out_ticket);

/* A reschedule with both lists ("paging out prompts that are not
 * a part of the next batch and paging in prompts that were not on the GPU")
 * in one call: exactly aqua_swap_out(out_pids) followed by
 * aqua_swap_in(in_pids) -- same validation (all-or-nothing over both), ids,
 * slots and bytes -- but the preemption runs on out_stream and the resume on
 * in_stream, pipelined in `pieces` pieces: resume piece k waits only for the
 * preemption piece that freed its blocks, so both directions of a
 * full-duplex link (NVLink, PCIe) carry data at the same time.
 * out_ticket / in_ticket cover the preemption / the resume. */
AQUA_API aqua_status aqua_swap_exchange(aqua_ctx* ctx, int32_t n_out, const uint64_t* out_pids, int32_t n_in,
                                        const uint64_t* in_pids, aqua_stream_t out_stream,
                                        aqua_stream_t in_stream, int32_t pieces, int32_t* out_ids,
                                        int64_t out_ids_cap, int32_t* out_counts, uint64_t* out_ticket,
                                        uint64_t* in_ticket);

/* NEXT-3, layer-wise streaming (Sec. 9: FlexGen "pages the
 * previous layer's context out and the next layer's in"): exactly
 * aqua_swap_out / aqua_swap_in (same bookkeeping, same bytes), but the copy
 * is issued as ceil(L / layer_group) launches in layer order, and
 * out_tickets[g] completes when layers [g*layer_group, (g+1)*layer_group) are
 * done -- decode can start on layer group 0 of a resumed prompt while the
 * rest is still in flight.  The last ticket covers the whole copy.
 * out_tickets has ceil(L / layer_group) entries; layer_group >= 1. */
AQUA_API aqua_status aqua_swap_out_layers(aqua_ctx* ctx, int32_t n, const uint64_t* pids, aqua_stream_t stream,
                                          int32_t layer_group, uint64_t* out_tickets);
AQUA_API aqua_status aqua_swap_in_layers(aqua_ctx* ctx, int32_t n, const uint64_t* pids, aqua_stream_t stream,
                                         int32_t layer_group, int32_t* out_ids, int64_t out_ids_cap,
                                         int32_t* out_counts, uint64_t* out_tickets);

/* Forget pid: RESIDENT -> its blocks are freed (their last use
 * is taken to be the work already queued on `stream`); SWAPPED -> its slots
 * are freed. */
AQUA_API aqua_status aqua_free(aqua_ctx* ctx, uint64_t pid, aqua_stream_t stream);

/* NEXT-1, elastic lending (Sec. 6 "Reclaiming AquaTensors" P:758-768;
 * fig:elastic_result P:1073-1099).  Move the swap images of SWAPPED prompts
 * (listed once, none already in dst) to arena dst_loc (AQUA_LOC_PEER or
 * AQUA_LOC_HOST), lowest free slots in call order (R4):
 *   dst[new_j*U : +U] = src[old_j*U : +U];  the old slots are freed.
 * All-or-nothing: AQUA_E_NOSPACE if dst is missing or too small.  On
 * `stream`: under AQUA_KERNEL_AUTO the copy engines (one DMA per run of slots
 * consecutive on both sides, no SM held); with an explicit TMA / LDST engine
 * one fused kernel launch (arena -> arena). */
AQUA_API aqua_status aqua_migrate(aqua_ctx* ctx, int32_t n, const uint64_t* pids, int32_t dst_loc,
                                  aqua_stream_t stream, uint64_t* out_ticket);
/* The GPU lender takes its memory back: every image on it moves to the host
 * arena (ascending pid), then the lender is detached, so later swap_outs go
 * to the host until aqua_lend is called again (a re-offer).  The
 * ticket covers every library access to the lender: after it completes the
 * lender's memory is unused (a library-owned arena is freed then).
 * All-or-nothing (AQUA_E_NOSPACE if the host cannot hold the images);
 * without a GPU lender it is a no-op with ticket 0. */
AQUA_API aqua_status aqua_reclaim(aqua_ctx* ctx, aqua_stream_t stream, uint64_t* out_ticket);

/* NEXT-2, prefix caching (Sec. 8: "a new prefill caching API with
 * unique IDs, and both CFS and prefill caching share the same swap space";
 * Sec. 9).  Cached-prefix ids are their own
 * namespace.
 * aqua_prefix_store: persist the first n blocks of a RESIDENT prompt as
 *   image `prefix_id` in swap space (placement as swap_out, R5).  Copy, not
 *   move: the prompt keeps its blocks (its later writers must wait for the
 *   ticket).  AQUA_E_INVAL if the id is in use or n is out of range.
 * aqua_prefix_load: a cache hit -- append n fresh blocks (lowest first) to
 *   dst_pid (created RESIDENT if new) and copy the image into them; the
 *   image stays.  out_ids[cap] gets the new block ids.
 * aqua_prefix_drop: free the image's slots.
 * aqua_reclaim moves cached prefixes off the lender as well (after the
 * prompts, ascending id). */
AQUA_API aqua_status aqua_prefix_store(aqua_ctx* ctx, uint64_t prefix_id, uint64_t src_pid, int32_t n,
                                       aqua_stream_t stream, uint64_t* out_ticket);
AQUA_API aqua_status aqua_prefix_load(aqua_ctx* ctx, uint64_t prefix_id, uint64_t dst_pid, aqua_stream_t stream,
                                      int32_t* out_ids, int32_t cap, uint64_t* out_ticket);
AQUA_API aqua_status aqua_prefix_drop(aqua_ctx* ctx, uint64_t prefix_id);
AQUA_API aqua_status aqua_prefix_query(aqua_ctx* ctx, uint64_t prefix_id, int32_t* location, int32_t* n,
                                       int32_t* slots, int32_t cap);

/* Make `stream` wait for a ticket (cudaStreamWaitEvent; no-op if done). */
AQUA_API aqua_status aqua_wait(aqua_ctx* ctx, uint64_t ticket, aqua_stream_t stream);
/* Block the host until the ticket completes. */
AQUA_API aqua_status aqua_sync(aqua_ctx* ctx, uint64_t ticket);
/* Device time (ms) of the copy behind a swap ticket, from just before its
 * descriptor upload / copy to its completion event.  Needs AQUA_OPT_TIMING = 1
 * at swap time; AQUA_E_STATE if not timed or not complete yet.  The last
 * 65536 retired timed tickets are remembered. */
AQUA_API aqua_status aqua_ticket_elapsed(aqua_ctx* ctx, uint64_t ticket, float* ms);
/* *done = 1 if the ticket has completed, else 0. */
AQUA_API aqua_status aqua_ticket_done(aqua_ctx* ctx, uint64_t ticket, int32_t* done);

/* Where is pid?  state = AQUA_ST_*, location = AQUA_LOC_*,
 * n = number of blocks (RESIDENT) or slots (SWAPPED); ids_or_slots (nullable,
 * capacity cap) receives the block table or the slot list. */
AQUA_API aqua_status aqua_query(aqua_ctx* ctx, uint64_t pid, int32_t* state, int32_t* location,
                       int32_t* n, int32_t* ids_or_slots, int32_t cap);
/* Free counts: blocks, peer-lender slots, host slots (-1 if no such arena). */
AQUA_API aqua_status aqua_counts(aqua_ctx* ctx, int32_t* free_blocks, int32_t* peer_free_slots,
                        int32_t* host_free_slots);
/* Device-visible base address of an arena (loc = AQUA_LOC_PEER / _HOST). */
AQUA_API aqua_status aqua_arena_base(aqua_ctx* ctx, int32_t loc, void** base, int32_t* nslots);

AQUA_API aqua_status aqua_set_option(aqua_ctx* ctx, int32_t option, int64_t value);
AQUA_API aqua_status aqua_get_option(aqua_ctx* ctx, int32_t option, int64_t* value);

/* The descriptors of the most recent swap call, as executed (also in
 * AQUA_DRYRUN): per block, in call order, src block / dst slot (swap_out)
 * or src slot / dst block (swap_in), and the arena (AQUA_LOC_PEER/_HOST).
 * *n_out = total count; at most cap entries are written. */
AQUA_API aqua_status aqua_last_descriptors(aqua_ctx* ctx, int32_t* blocks, int32_t* slots, int32_t* locs,
                                  int64_t cap, int64_t* n_out);
/* Kernel launches issued by this ctx so far (swap + harness kernels). */
AQUA_API aqua_status aqua_launch_count(aqua_ctx* ctx, uint64_t* launches);
/* Shape of the most recent swap / migrate kernel launch (what AUTO chose), for reporting: CTAs, threads per CTA,
 * TMA ring stages (0 for the LDST engine), engine (AQUA_KERNEL_TMA / AQUA_KERNEL_LDST), variant, items per claimed
 * batch (0 = static ranges; < 0 never), descriptors passed in the kernel parameters (0 = staged upload).  Any out
 * pointer may be NULL.  AQUA_E_STATE before the first launch (and for copy-engine-only calls, which launch none). */
AQUA_API aqua_status aqua_last_launch(aqua_ctx* ctx, int32_t* grid, int32_t* threads, int32_t* stages,
                                      int32_t* engine, int32_t* variant, int64_t* batch_items, int64_t* inline_desc);

/* What aqua_lend found about an arena (which = AQUA_LOC_PEER for the GPU lender, AQUA_LOC_HOST for host DRAM):
 * the device holding its memory (AQUA_HOST for host DRAM), whether it is a peer GPU (NVLink / P2P), and the
 * result of the lend-time probe (bit 1 plain 16-byte loads/stores, 2 TMA bulk stores, 4 TMA bulk loads round-trip
 * correctly; 7 = all; -1 = not probed: host arenas and the borrower's own HBM).  A peer arena whose bulk copies
 * fail the probe is served by the LDST engine (plain loads and stores over NVLink) instead of TMA; one whose plain
 * accesses fail is refused by aqua_lend with AQUA_E_PEER.  AQUA_E_STATE if that arena is not lent. */
AQUA_API aqua_status aqua_arena_info(aqua_ctx* ctx, int32_t which, int32_t* device, int32_t* peer, int32_t* probe,
                                     int32_t* nslots);

/* Cross-process lending (setup only).  The lender process
 * exports a 64-byte handle for a device allocation; the borrower process
 * imports it on `device` (peer access enabled lazily) and passes the pointer
 * to aqua_lend(ctx, AQUA_MAPPED, ptr, bytes, ...). */
AQUA_API aqua_status aqua_ipc_export(void* dev_ptr, uint8_t handle[64]);
AQUA_API aqua_status aqua_ipc_import(int device, const uint8_t handle[64], void** out_ptr);
AQUA_API aqua_status aqua_ipc_close(int device, void* ptr);
/* A dedicated cudaMalloc on `device` (its own allocation, so an exported
 * handle maps to offset 0) for memory a producer offers to a consumer
 * process; freed with aqua_ipc_free after every importer has closed it. */
AQUA_API aqua_status aqua_ipc_alloc(int device, uint64_t bytes, void** out_ptr);
AQUA_API aqua_status aqua_ipc_free(int device, void* ptr);
/* 1 if `device` can access `peer` by P2P (cudaDeviceCanAccessPeer). */
AQUA_API aqua_status aqua_can_access_peer(int device, int peer, int32_t* can);

/* Harness kernels (tests / bench / C3 driver), C-11: write the
 * closed-form KV pattern of tokens [t0, t1) of pid into its blocks
 * (synthetic decode; elem_bytes must be 2), and count the words of tokens
 * [0, ntok) that differ from the pattern into *d_mismatches (a device
 * uint64, accumulated with atomicAdd).  Both are stream-ordered. */
AQUA_API aqua_status aqua_kv_fill_pattern(aqua_ctx* ctx, uint64_t pid, int32_t t0, int32_t t1,
                                 uint64_t seed, aqua_stream_t stream);
/* The same fill for many prompts in ONE launch (synthetic decode of a whole
 * iteration): tokens [t0s[i], t1s[i]) of pids[i]. */
AQUA_API aqua_status aqua_kv_fill_pattern_batch(aqua_ctx* ctx, int32_t n, const uint64_t* pids, const int32_t* t0s,
                                                const int32_t* t1s, uint64_t seed, aqua_stream_t stream);
AQUA_API aqua_status aqua_kv_verify_pattern(aqua_ctx* ctx, uint64_t pid, int32_t ntok, uint64_t seed,
                                   aqua_stream_t stream, uint64_t* d_mismatches);

AQUA_API const char* aqua_strerror(aqua_status s);
AQUA_API const char* aqua_last_error(aqua_ctx* ctx);
/* Library version string. */
AQUA_API const char* aqua_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AQUA_H_ */
