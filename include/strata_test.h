/*
 * strata_test.h — pure host-side planning functions of libstrata exported for tests (no GPU, no
 * CUDA calls).  Not part of the data path's contract; the values they return are the ones
 * strata_load / strata_offload use (csrc/transfer.cpp ring_geometry).
 */
#ifndef STRATA_TEST_H
#define STRATA_TEST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The ring engine's per-CTA geometry for token rows of `tok_bytes` bytes, host
 * chunks of `chunk_tokens` tokens and access granularity `gran` (16, or 8 for narrow rows), with
 * `smem_budget` bytes of shared memory per CTA, `inflight_bytes` host bytes in flight over `ctas`
 * CTAs, `warps` requested device-side warps per CTA and a piece-size target of `stage_target`
 * bytes.  out[0] = rows per piece R, out[1] = ring depth S, out[2] = device-side warps W (W divides
 * S), out[3] = bytes per stage.  Returns 0, or STRATA_ERR_UNSUPPORTED (-7) when not even a 2-stage
 * ring of one-row pieces fits (the caller then uses another engine), STRATA_ERR_INVALID_ARG (-1)
 * for a non-positive size or a NULL `out`. */
int strata_test_ring_geometry(int32_t tok_bytes, int32_t chunk_tokens, int32_t gran, int32_t smem_budget,
                              int64_t inflight_bytes, int32_t ctas, int32_t warps, int32_t stage_target,
                              int32_t out[4]);

#ifdef __cplusplus
}
#endif

#endif /* STRATA_TEST_H */
