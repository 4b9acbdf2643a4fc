/*
 * strata_disk.h — the disk tier below the host tier.
 *
 * "the cache controller opportunistically prefetches data from storage to host memory when a cache
 *  hit is detected at the storage layer ... Once the scheduler dispatches the request for execution,
 *  the cache controller terminates any in-flight prefetch and leverages the available cache already
 *  in host or GPU memory" (§4.2.1).  The same page-first layout that makes host <->
 * GPU transfers large makes disk transfers large: "other media, such as host memory and external
 * storage, can adopt a page-first layout that maximizes transfer efficiency with larger, contiguous
 * data blocks", up to 4x lower latency than layer-first at 8192 tokens, page size 32
 * (fig:disk).
 *
 * A disk tier is a file of `num_chunks` disk chunks, each holding exactly the bytes of one host chunk
 * (chunk_bytes = L*2*C*H*D*e, include/strata.h LAYOUTS), in one of two layouts:
 *   STRATA_DISK_PAGE_FIRST   disk chunk k at file offset k*chunk_bytes (one contiguous read per chunk)
 *   STRATA_DISK_LAYER_FIRST  layer l of disk chunk k at offset (l*num_chunks + k)*layer_bytes with
 *                            layer_bytes = chunk_bytes/L (L reads per chunk; the comparison layout)
 * Either way a prefetch leaves the host chunk byte-identical to what a writeback stored.
 *
 * Jobs are asynchronous (a pool of I/O threads, one chunk per work item), cancellable between chunks,
 * and report per-chunk completion so a cancelled prefetch still credits the chunks it finished.
 * Only host memory is touched: no CUDA call is made, so this part runs without a GPU.
 * Handles are thread-safe.  Errors as in strata.h (negative codes, strata_last_error()).
 */
#ifndef STRATA_DISK_H
#define STRATA_DISK_H

#include "strata.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct strata_disk* strata_disk_t;

enum strata_disk_layout { STRATA_DISK_PAGE_FIRST = 0, STRATA_DISK_LAYER_FIRST = 1 };
enum strata_disk_flags {
  STRATA_DISK_O_DIRECT = 1, /* bypass the page cache (needs 4096-byte aligned chunk/layer bytes and
                               host buffers; otherwise STRATA_ERR_ALIGNMENT at open / submit) */
  STRATA_DISK_CREATE = 2    /* create / extend the file to num_chunks*chunk_bytes */
};
enum strata_disk_status {   /* per-chunk status reported by strata_disk_wait */
  STRATA_DISK_PENDING = 0, STRATA_DISK_DONE = 1, STRATA_DISK_CANCELLED = 2, STRATA_DISK_FAILED = 3
};

typedef struct {
  const char* path;       /* file backing the tier */
  int64_t chunk_bytes;    /* bytes per chunk (= the host tier's chunk_bytes) */
  int32_t num_layers;     /* L: chunk_bytes must be a multiple of L */
  int32_t layout;         /* strata_disk_layout */
  int64_t num_chunks;     /* capacity in disk chunks */
  int32_t flags;          /* strata_disk_flags */
  int32_t io_threads;     /* worker threads, 0 = 8 */
} strata_disk_desc;

int strata_disk_open(const strata_disk_desc* d, strata_disk_t* out);

/* Cancels every unfinished job, waits for in-flight reads/writes, closes the file. NULL: no-op. */
int strata_disk_close(strata_disk_t d);

/* Asynchronous prefetch: disk chunk disk_chunks[i] -> host chunk host_chunks[i] of the host tier at
 * host_base (same chunk_bytes), i < n.  Index arrays are copied; host_base must stay valid until the
 * job completes or is cancelled and waited for.  *job receives the job id. */
int strata_disk_prefetch(strata_disk_t d, void* host_base, const int32_t* disk_chunks, const int32_t* host_chunks,
                         int64_t n, uint64_t* job);

/* Asynchronous writeback ("backup ... to lower memory hierarchies"): host chunk
 * host_chunks[i] -> disk chunk disk_chunks[i]. */
int strata_disk_writeback(strata_disk_t d, const void* host_base, const int32_t* host_chunks,
                          const int32_t* disk_chunks, int64_t n, uint64_t* job);

/* Stop a job: chunks not yet started are never transferred; chunks in flight complete.
 * Returns immediately; use strata_disk_wait to collect the final state. */
int strata_disk_cancel(strata_disk_t d, uint64_t job);

/* Wait up to timeout_ms (< 0: forever) for a job to settle (every chunk done, cancelled or failed).
 * *ndone (nullable) = chunks fully transferred; status (nullable, [n]) = per-chunk strata_disk_status.
 * Returns STRATA_OK when settled, STRATA_ERR_TIMEOUT if not settled in time, STRATA_ERR_IO if any
 * chunk failed.  A settled job is forgotten after a successful wait (its id becomes invalid). */
int strata_disk_wait(strata_disk_t d, uint64_t job, int64_t timeout_ms, int64_t* ndone, int32_t* status);

#ifdef __cplusplus
}
#endif

#endif /* STRATA_DISK_H */
