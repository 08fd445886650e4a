/*
 * aqua_cfs.h -- native time-slice scheduler that drives libaqua's paging
 * (hot-path row A0: CFS reschedule -> ordered page_out / page_in lists).
 *
 * Paper, Sec. 7: batch partitioning into p prefill and d
 * decode tokens, d set to its upper bound (the number of prompts that fit
 * in memory), prefill prompts with the least prefill done first, decode
 * prompts with the least tokens generated, leftover d slots to the prefill
 * prompts, stop when memory is exhausted; reschedule every k iterations or
 * when a request completes, paging out the prompts not in the next batch and
 * paging in the prompts not on the GPU.  Readings R8-R18 and R21:
 * ties (arrival, id); memory test ceil((ctx + t) / bs) blocks per prompt
 * summed <= num_blocks; prefill filled before decode; a non-fitting prompt
 * stops its walk; extra reschedule when the plan's next iteration no longer
 * fits or has no work; literal eviction of every resident prompt not in the
 * plan; a preempted prefill keeps its partial KV; with no prefill prompt
 * chosen (p = 0) the spare decode slots walk the prefill prompts (R21).
 * FCFS is the no-preemption baseline.
 *
 * Iteration protocol (the caller owns the KV pool, via libaqua):
 *   aqua_cfs_add() every request whose arrival <= aqua_cfs_vclock();
 *   aqua_cfs_next()  -> page_out, page_in (call aqua_swap_out / aqua_swap_in
 *                       in that order), and the work list: per prompt, the
 *                       KV length before the iteration (ctx0), the tokens
 *                       it runs (t) and the blocks to append (grow) with
 *                       aqua_alloc_blocks, in list order;
 *   run the iteration (write the KV of tokens [ctx0, ctx0 + t));
 *   aqua_cfs_commit() -> finished pids (free them with aqua_free, in order)
 *                       and the virtual clock advanced by
 *                       t_base + t_token * tokens.
 * If aqua_cfs_next() returns no work the runnable set is empty: advance the
 * clock to the next arrival with aqua_cfs_advance_to().
 */
#ifndef AQUA_CFS_H_
#define AQUA_CFS_H_

#include "aqua.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aqua_cfs aqua_cfs;

enum { AQUA_POLICY_CFS = 0, AQUA_POLICY_FCFS = 1 };
enum { AQUA_PHASE_PREFILL = 0, AQUA_PHASE_DECODE = 1 };

typedef struct {
  int32_t policy;        /* AQUA_POLICY_* */
  int32_t batch_tokens;  /* b (chunk size, 512 in the paper's setup P:485) */
  int32_t k;             /* reschedule interval in iterations (R8: 8) */
  int32_t block_tokens;  /* bs */
  int32_t num_blocks;    /* NB of the borrower pool */
  int32_t pad_;
  double t_base;         /* virtual iteration cost t_base + t_token * tokens */
  double t_token;
} aqua_cfs_config;

typedef struct {
  uint64_t pid;
  int32_t ctx0;          /* KV tokens stored before this iteration */
  int32_t tokens;        /* tokens this iteration (prefill chunk or 1 decode) */
  int32_t grow;          /* blocks to append before the iteration */
  int32_t phase;         /* AQUA_PHASE_* at plan time */
} aqua_cfs_work;

AQUA_API aqua_status aqua_cfs_create(const aqua_cfs_config* cfg, aqua_cfs** out);
AQUA_API aqua_status aqua_cfs_destroy(aqua_cfs* s);
/* Make a request runnable (arrival in virtual seconds). */
AQUA_API aqua_status aqua_cfs_add(aqua_cfs* s, uint64_t pid, double arrival, int32_t prompt_tokens,
                                  int32_t output_tokens);
/* Overwrite a runnable request's service counters (tests / restarts).  A
 * request added without KV that is given ctx > 0 here is a restart whose KV
 * the caller holds as a swapped image (aqua_swap_out): the scheduler counts
 * ceil(ctx / bs) blocks for it and pages it in when a plan includes it. */
AQUA_API aqua_status aqua_cfs_set_state(aqua_cfs* s, uint64_t pid, int32_t phase, int32_t prefill_done,
                                        int32_t generated, int32_t ctx);
/* Plan one iteration.  Arrays have capacity `cap`; *rescheduled = 1 when a
 * new plan was made (then page_out / page_in may be non-empty).  On any
 * error (AQUA_E_INVAL: a list would exceed cap; AQUA_E_NOBLOCKS: nothing
 * fits) the scheduler's state is unchanged. */
AQUA_API aqua_status aqua_cfs_next(aqua_cfs* s, int32_t* rescheduled, uint64_t* page_out, int32_t* n_out,
                                   uint64_t* page_in, int32_t* n_in, aqua_cfs_work* work, int32_t* n_work,
                                   int32_t cap);
/* Apply the planned iteration; finished pids (capacity cap) in work order.
 * AQUA_E_INVAL (more finishes than cap) changes nothing. */
AQUA_API aqua_status aqua_cfs_commit(aqua_cfs* s, uint64_t* finished, int32_t* n_fin, int32_t cap,
                                     double* vclock);
/* The partition of the current runnable set (no side effects): decode ids in
 * selection order, then prefill (id, tokens) in selection order. */
AQUA_API aqua_status aqua_cfs_partition(aqua_cfs* s, uint64_t* decode, int32_t* n_decode, uint64_t* prefill,
                                        int32_t* prefill_tokens, int32_t* n_prefill, int32_t cap);
/* Switch policy between iterations ("fall back to FCFS from CFS
 * when tensors are on DRAM").  Entering FCFS admits the resident prompts (in
 * arrival order); swapped prompts are paged in when FCFS admits them; if the
 * inherited residents outgrow the pool the latest-arrived one is paged out
 * (R18).  Returning to CFS replans at the next iteration. */
AQUA_API aqua_status aqua_cfs_set_policy(aqua_cfs* s, int32_t policy);
AQUA_API aqua_status aqua_cfs_vclock(aqua_cfs* s, double* vclock);
AQUA_API aqua_status aqua_cfs_advance_to(aqua_cfs* s, double vclock);
/* Runnable prompts, prompts with KV resident in the pool, iterations run. */
AQUA_API aqua_status aqua_cfs_stats(aqua_cfs* s, int32_t* runnable, int32_t* resident, int64_t* iterations);

/* ---- Native trace runner (the engine loop of BASELINE configs[2]) --------
 * Runs a whole request trace through the scheduler and libaqua: admission by
 * the virtual clock, aqua_cfs_next, swap_out / swap_in (or aqua_swap_exchange
 * when swap_stream2 is set), block growth, the synthetic decode (pattern
 * fill of each iteration's tokens, one launch) and frees -- with the same
 * semantics and call log as the Python driver and the oracle.  Streams: the
 * swap stream waits for the decode stream before a preemption; the decode
 * stream waits for each resume's ticket.  With d_mismatches every resumed
 * prompt is checked against its pattern (restore invariant at full scale). */
typedef struct {
  uint64_t pid;
  double arrival;             /* virtual seconds */
  int32_t prompt_tokens, output_tokens;
} aqua_trace_req;

typedef struct {
  aqua_stream_t decode_stream, swap_stream;
  aqua_stream_t swap_stream2;  /* non-NULL: reschedules with both lists use aqua_swap_exchange */
  int32_t exchange_pieces;
  int32_t fill;                /* 1: write each iteration's KV pattern (needs a GPU ctx) */
  uint64_t fill_seed;
  uint64_t* d_mismatches;      /* device counter, or NULL: no verification */
} aqua_trace_opts;

typedef struct {
  int64_t iterations, swap_out_calls, swap_in_calls, blocks_out, blocks_in;
  double vclock;
} aqua_trace_stats;

/* Call log (optional): int64 records, in order --
 *   1 plan:     it, nD, D..., nP, (pid, tokens)...
 *   2 swap_out: n, pids..., then per pid: location, nslots, slots...
 *   3 swap_in:  n, pids..., then per pid: nblocks, blocks...
 *   4 alloc:    pid, n, ids...        5 iter: it, n, (pid, ctx0, tokens)...
 *   6 free:     pid
 * *log_len = records' total length; AQUA_E_INVAL if log_cap was too small
 * (the run itself completed). */
AQUA_API aqua_status aqua_trace_run(aqua_ctx* ctx, aqua_cfs* sched, int32_t n, const aqua_trace_req* reqs,
                                    const aqua_trace_opts* opts, aqua_trace_stats* stats, int64_t* log_buf,
                                    int64_t log_cap, int64_t* log_len);

#ifdef __cplusplus
}
#endif
#endif /* AQUA_CFS_H_ */
