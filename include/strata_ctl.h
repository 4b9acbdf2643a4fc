/*
 * strata_ctl.h — the control plane that drives strata_load / strata_offload.
 *
 * "The Scheduler ... references a HiRadixTree, which is an extension to SGLang's RadixTree,
 *  effectively serving as a page table and stores metadata about each KV cache page".
 * "When a request is submitted, it enters a request waiting queue ... the Scheduler ... selects a
 *  subset to form the next batch ... then sends this batch to GPU executor and initiates a KV cache
 *  loading request to the Cache Controller".
 *
 * One strata_ctl holds, for one GPU's KV pool and its host tier:
 *   - the HiRadixTree: a radix tree over token ids.  A committed node maps each of its tokens to a
 *     device slot (page*P + offset in the paged pool) and/or a host slot (chunk*C + offset in the
 *     page-first host tier).  A transient node carries a mark instead, IN_QUEUE ("a request is
 *     referencing a new context") or IN_FLIGHT ("the cache for the corresponding tokens is under
 *     computation");
 *   - the waiting queue and the scheduler: deferral on delay hit, Algorithm 1
 *     balanced batch formation with bundle hits;
 *   - the cache controller's page allocators (device pages, host chunks), LRU eviction with
 *     write-back to the host tier, and the per-round LOAD and WRITE-BACK plans, in
 *     exactly the strata_xfer shape (include/strata.h), that move the batch's host-resident prefix
 *     onto the device and the evicted device-only nodes onto the host.
 *
 * Every reading of the paper taken where it is silent is DESIGN.md R17-R26 (cited at each call).
 * Pure host code: no CUDA call is made, so all of it runs (and is tested) without a GPU.
 * A handle is NOT thread-safe (one scheduler thread, as in SGLang).  Errors as in strata.h
 * (negative codes, strata_last_error()).
 */
#ifndef STRATA_CTL_H
#define STRATA_CTL_H

#include "strata.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct strata_ctl* strata_ctl_t;

enum strata_ctl_flags {       /* ablations: each switches one mechanism of §4.3 off */
  STRATA_CTL_NO_DEFER = 1,    /* no transient marks, no deferral (SGLang's default) */
  STRATA_CTL_NO_BALANCE = 2,  /* no loading_bound test: Algorithm 1 without the D list = FIFO */
  STRATA_CTL_NO_BUNDLE = 4    /* no AddBundleHit */
};
enum strata_ctl_tier { STRATA_TIER_DEVICE = 0, STRATA_TIER_HOST = 1 };
enum strata_ctl_list { STRATA_CTL_BATCH = 0, STRATA_CTL_DEFERRED = 1, STRATA_CTL_FORMED = 2,
                       STRATA_CTL_QUEUE = 3 };
enum strata_ctl_plan_kind { STRATA_CTL_LOAD = 0, STRATA_CTL_WRITEBACK = 1 };

typedef struct {
  int32_t page_size;           /* P: device page size in tokens (>= 1), as strata_pool_desc */
  int32_t chunk_tokens;        /* C: host chunk size in tokens (>= 1), as strata_pool_desc */
  int64_t num_pages;           /* device pages this ctl allocates: indices [0, num_pages) */
  int64_t num_chunks;          /* host chunks this ctl allocates: indices [0, num_chunks) */
  int64_t deferral_threshold;  /* delay hit iff transient-matched tokens > this (100);
                                  also the bundle-hit overlap threshold (R20) */
  double loading_bound_ratio;  /* loading-bound iff load / max(compute, 1) > this (100) */
  int64_t max_batch_tokens;    /* compute tokens per prefill batch; <= 0: unlimited (R21) */
  int32_t max_batch_reqs;      /* requests per prefill batch; <= 0: unlimited (R21) */
  int32_t flags;               /* strata_ctl_flags */
} strata_ctl_desc;

typedef struct {               /* longest stored prefix of a token list, by kind of node */
  int64_t total, device, host, transient;   /* device+host counted as device */
} strata_ctl_match_t;

typedef struct {               /* what one strata_ctl_schedule round did */
  int64_t num_batch;           /* requests dispatched (the prefill batch) */
  int64_t num_deferred;        /* requests deferred on a delay hit (now at the queue front) */
  int64_t num_formed;          /* requests Algorithm 1 chose (>= num_batch: dispatch stops at the
                                  first request the device pool cannot hold) */
  int64_t formed_load;         /* Algorithm 1's aggregated load of the formed batch, tokens */
  int64_t formed_compute;      /* and its compute, tokens */
  int64_t new_tokens;          /* tokens the dispatched batch prefills */
  int64_t load_tokens;         /* tokens in the LOAD plan */
  int64_t writeback_tokens;    /* tokens in the WRITE-BACK plan */
} strata_ctl_round;

typedef struct {               /* a plan in strata_xfer's shape (include/strata.h:25-27) */
  int64_t num_reqs;
  const int64_t* num_tokens;   /* [num_reqs] */
  const int64_t* chunk_start;  /* [num_reqs] */
  const int32_t* chunk_offset; /* [num_reqs] */
  const int32_t* host_chunks;  /* [host_chunks_len] host arrays: copy to the device for strata_xfer */
  int64_t host_chunks_len;
  const int64_t* page_start;   /* [num_reqs] */
  const int32_t* page_offset;  /* [num_reqs] */
  const int32_t* dev_pages;    /* [dev_pages_len] */
  int64_t dev_pages_len;
} strata_ctl_plan;

typedef struct {
  int64_t nodes, transient_nodes;
  int64_t free_pages, free_chunks;
  int64_t device_tokens, host_tokens;   /* tokens resident in committed nodes */
  int64_t queued, dispatched;
} strata_ctl_stats;

/* Create / destroy.  Capacities must fit int32 page / chunk indices. */
int strata_ctl_create(const strata_ctl_desc* d, strata_ctl_t* out);
int strata_ctl_destroy(strata_ctl_t c);

/* Make tokens[0..n) resident on `tier` (committed nodes; transient nodes on the path are
 * converted), allocating slots for the tokens not yet resident there, evicting LRU nodes if the tier
 * is full (R23).  slots_out (n entries, may be NULL) receives every token's slot on that tier; the
 * caller then owns writing those slots' KV (e.g. the host tier bytes of a context offloaded before).
 * STRATA_ERR_OOM if the tier cannot make room.  Like strata_ctl_schedule, it replaces both plans:
 * the WRITE-BACK plan then holds the write-backs its evictions need (run it before writing the new
 * slots) and the LOAD plan is empty. */
int strata_ctl_insert(strata_ctl_t c, const int32_t* tokens, int64_t n, int32_t tier, double now,
                      int64_t* slots_out);

/* Longest stored prefix of tokens[0..n) with its breakdown (no mutation). */
int strata_ctl_match(strata_ctl_t c, const int32_t* tokens, int64_t n, strata_ctl_match_t* out);

/* Enqueue a request (n >= 1 tokens; the ctl copies them).  STRATA_ERR_DUPLICATE if req_id exists. */
int strata_ctl_submit(strata_ctl_t c, int64_t req_id, const int32_t* tokens, int64_t n);

/* One scheduling round at time `now`: clear last round's in-queue marks (R18); defer delay hits
 * (PAPER.md:317); Algorithm 1 over the rest; dispatch the batch: pin each
 * member's cached prefix, load its host-only part, allocate its new tokens, mark its transient
 * nodes in-flight.  Replaces the LOAD and WRITE-BACK plans: run WRITE-BACK
 * (strata_offload) before LOAD (strata_load) on the same stream, before the batch's prefill. */
int strata_ctl_schedule(strata_ctl_t c, double now, strata_ctl_round* out);

/* Copy a request-id list of the last round (BATCH, DEFERRED, FORMED) or the current QUEUE into
 * ids_out (may be NULL); *n_out = its length. */
int strata_ctl_ids(strata_ctl_t c, int32_t which, int64_t* ids_out, int64_t* n_out);

/* The last round's plan (arrays owned by the ctl, valid until the next schedule / insert / destroy). */
int strata_ctl_plan_get(strata_ctl_t c, int32_t which, strata_ctl_plan* out);

/* A dispatched request's device slot for each of its tokens (its page table for the prefill).
 * slots_out may be NULL; *n_out = token count.  STRATA_ERR_INVALID_ARG if not dispatched. */
int strata_ctl_req_slots(strata_ctl_t c, int64_t req_id, int64_t* slots_out, int64_t* n_out);

/* The request's prefill finished: its tokens become committed device nodes ("converted into
 * standard nodes"), its prefix is unpinned; slots another request committed first are
 * released (R26). */
int strata_ctl_complete(strata_ctl_t c, int64_t req_id, double now);

/* Drop a queued or dispatched request: unpin, release its new slots, remove in-flight nodes nobody
 * else covers. */
int strata_ctl_abort(strata_ctl_t c, int64_t req_id);

int strata_ctl_get_stats(strata_ctl_t c, strata_ctl_stats* out);

/* Canonical dump for tests: one line per node, sorted by path:
 * "path;dev;host;mark;tref;ref;last_access" with comma-separated integer lists.  Owned by the ctl,
 * valid until the next call on it. */
const char* strata_ctl_dump(strata_ctl_t c);

/* Bubble filling: decode steps that fit in a loading stall,
 * floor((t_load - t_comp) / decode_step) when t_load > t_comp and decode_reqs > 0, else 0. */
int64_t strata_ctl_bubble_steps(double t_load_ms, double t_comp_ms, double decode_step_ms,
                                int64_t decode_reqs);

#ifdef __cplusplus
}
#endif
#endif
