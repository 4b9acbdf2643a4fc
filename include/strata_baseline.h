/*
 * strata_baseline.h — copy-engine baselines and the link roofline, exported by libstrata next to
 * the product calls so every method moves bytes from the SAME registered host tier
 * (SURVEY.md §8d "Same memory type").  None of these is on the product path.
 *
 * They produce exactly the result strata_load / strata_offload define (include/strata.h LAYOUTS),
 * so the GPU parity tests also pin them against the CPU oracle.
 */
#ifndef STRATA_BASELINE_H
#define STRATA_BASELINE_H

#include "strata.h"

#ifdef __cplusplus
extern "C" {
#endif

enum strata_dir { STRATA_H2D = 0, STRATA_D2H = 1 };

/* The fragmentation baseline: "invoking standard cudaMemcpyAsync API repetitively with small data
 * transfers" (PAPER.md:236 §4.2; per-page DMA, PAPER.md:166-169 §3.1, :182; SGLang-HiCache
 * "layer-wise ... using cudaMemcpyAsync", §5.1).
 * One cudaMemcpyAsync per (layer, kv, device page) — split further where the page's tokens cross a
 * host chunk boundary, and per head when the device rows are not head-contiguous.
 * x->host_chunks and x->dev_pages must be HOST pointers here (the CPU issues the copies).
 * x->engine / num_ctas / threads are ignored.  No events are recorded.
 * *ncopies (nullable) receives the number of cudaMemcpyAsync calls issued. */
int strata_baseline_memcpy_pages(strata_pool_t p, const strata_xfer* x, int32_t dir,
                                 strata_stream_t stream, int64_t* ncopies);

/* The link roofline: ONE contiguous cudaMemcpyAsync of `bytes` between the registered host tier
 * (starting `host_offset` bytes in) and device memory `dev` (the denominator). */
int strata_baseline_contiguous(strata_pool_t p, int32_t dir, void* dev, int64_t host_offset,
                               int64_t bytes, strata_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* STRATA_BASELINE_H */
