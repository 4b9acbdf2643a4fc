/*
 * strata.h — C ABI of libstrata, the B200-native GPU-assisted KV-cache I/O path of
 * "Strata: Hierarchical Context Caching for Long Context Language Model Serving" (arXiv 2508.18572).
 *
 * The library moves cached KV between a pinned, GPU-mapped host tier and the GPU's paged KV pool:
 *
 *   strata_load     host tier -> device pool   page-table-indexed gather + layout transform
 *   strata_offload  device pool -> host tier   the matching scatter ("backup")
 *
 * Both are sm_100a kernels that read/write host memory through zero-copy UVA mappings instead of
 * one cudaMemcpyAsync per page ("GPU-assisted I/O": a kernel with thousands of threads, each moving
 * a small chunk through registers or shared memory, §4.2), and both record one
 * CUDA event per layer so a consumer can start layer l while later layers still stream in
 * (PAPER.md:227 §4.1, :281 §4.2.1).
 *
 * LAYOUTS (DESIGN.md §3 readings R1-R5)
 *   Host tier, page-first ("arranges layers of a page contiguously"):
 *     num_chunks chunks of C tokens; chunk = [L][K,V][C][Ht][D] elements of e bytes,
 *     chunk_bytes = L*KV*C*Ht*D*e.  This GPU moves heads [h0, h0+H) of the tier's Ht heads
 *     (host_heads, head_begin; default Ht = H, h0 = 0: a per-GPU tier).  Token ho of chunk hc,
 *     layer l, kv, this GPU's head h starts at
 *       host_base + hc*chunk_bytes + ((l*KV + kv)*C + ho)*Ht*D*e + (h0 + h)*D*e         (token-major)
 *       host_base + hc*chunk_bytes + ((((h0 + h)*L + l)*KV + kv)*C + ho)*D*e           (head-major)
 *     KV = 2 (a K and a V buffer per layer), or KV = 1 with STRATA_POOL_SINGLE_KV (R27).
 *     STRATA_HOST_HEAD_MAJOR stores each chunk as [Ht][L][K,V][C][D] (R28): every head's part is a
 *     one-head page-first chunk, so a single tier holding every KV head serves any tensor-parallel
 *     degree with the same long runs (K and V of C tokens per layer and head) as a per-GPU tier.
 *   Device pool, layer-first, paged: one K and one V buffer per layer,
 *     caller-owned; token slot (page pg, offset po < P), head h starts at
 *       {k,v}_ptrs[l] + pg*page_stride + po*token_stride + h*head_stride.
 *     With STRATA_POOL_SINGLE_KV a layer has one buffer (k_ptrs; v_ptrs unused, may be NULL):
 *     MLA's latent cache (DeepSeek-V2/V3: one compressed vector per token from which K and V are
 *     both derived, e.g. H = 1, D = 576, bf16 -> 1152 B per token and layer).
 *     Default strides (0) are NHD: token_stride = H*D*e, head_stride = D*e, page_stride = P*H*D*e.
 *   Request r moves num_tokens[r] tokens; token i (0-based in this call) lives at
 *       host:   ci = chunk_offset[r] + i, chunk host_chunks[chunk_start[r] + ci / C], position ci % C
 *       device: pi = page_offset[r]  + i, page  dev_pages [page_start[r]  + pi / P], offset   pi % P
 *
 * DATA IS OPAQUE BYTES: no conversion, no rounding; NaN payloads and -0.0 survive (R9).
 * Rows (H*D*e), strides and bases need not be multiples of 16 bytes (R29): pools where they all are
 * take the vectorised engines; others take a narrow LDG kernel with the widest access dividing them.
 *
 * ERRORS: every call returns int, STRATA_OK (0) on success, a negative STRATA_ERR_* otherwise;
 * strata_last_error() gives a thread-local message for the last failure.  No C++ exception crosses
 * the ABI.  Argument, alignment and range checks of host-side values are synchronous.  Index-range
 * and duplicate-destination checks of the device index lists run only when the pool has
 * STRATA_VALIDATE (or env STRATA_VALIDATE=1): a device check kernel plus a stream synchronisation.
 * Asynchronous kernel faults surface as STRATA_ERR_CUDA on a later call.
 *
 * ENVIRONMENT (defaults are the measured choices of DESIGN.md §6; the knobs exist for A/B runs):
 *   STRATA_VALIDATE=1          as the STRATA_VALIDATE pool flag, for every pool
 *   STRATA_RING_INFLIGHT_KB=n  ring: host bytes in flight over all CTAs, KiB (default 224; 320 for rows < 2 KiB)
 *   STRATA_RING_STAGE_KB=n     ring: piece size (default 16)
 *   STRATA_RING_WARPS=n        ring: scatter warps per load CTA (default 8; STRATA_RING_GATHER_WARPS for offloads, 8)
 *   STRATA_RING_SMEM_KB=n      ring: cap on a CTA's shared memory
 *   STRATA_RING_EXCLUSIVE=1    ring: a CTA reserves its SM's shared memory (no co-resident CTAs)
 *   STRATA_RING_BULK_STORE=1   ring loads: page writes as cp.async.bulk stores instead of st.global
 *   STRATA_RING_STAGES=n       ring: cap on the stages per CTA
 *   STRATA_RING_DEBUG=bits     A/B only: 1 = ring loads skip the page writes, 2 = evict-first L2
 *                              policy on the ring's host reads
 *   STRATA_OFFLOAD_SHARE_GBS=n ring offloads pace their host stores to n GB/s in total while ring
 *                              loads run on the device (default 16; 0 = unpaced)
 *   STRATA_LDG_FUSED=0|force   per-layer launches only (LDG and ring) | fuse even 1-CTA LDG grids
 *   STRATA_COPY_STREAMS=n      copy streams of the DMA engine per direction (default 1)
 *   STRATA_STAGE_MB=n          DMA staging slot size (default 128)
 *   STRATA_DMA_EDGE_SPLIT=n    first / last layer in n times smaller pieces (default 4; 1 = off)
 *   STRATA_DMA_ORDERED=0       drop the per-piece barrier between copy streams (default on)
 *   STRATA_DMA_STRIDED=0       one copy per chunk instead of strided runs of consecutive chunks
 *
 * THREADING: a pool handle is single-writer (one thread at a time); distinct handles are
 * independent.  Operations of one handle may be in flight at once on different streams (e.g. a
 * load and an offload: both directions of the link); the library orders their use of its internal
 * staging buffers, the caller keeps their destinations disjoint (tests/test_gpu_concurrent.py).
 * Exception: a STRATA_ENGINE_DMA operation captured into a CUDA graph is ordered only by the graph;
 * do not replay it while another DMA operation of the same pool and direction is in flight.
 */
#ifndef STRATA_H
#define STRATA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same types as cudaStream_t / cudaEvent_t (CUDA runtime), declared here so consumers of this
 * header need no CUDA headers. */
struct CUstream_st;
struct CUevent_st;
typedef struct CUstream_st* strata_stream_t;
typedef struct CUevent_st* strata_event_t;

typedef struct strata_pool* strata_pool_t; /* opaque, library-owned */

enum strata_status {
  STRATA_OK = 0,
  STRATA_ERR_INVALID_ARG = -1,  /* null pointer, bad size or range in a host-side value */
  STRATA_ERR_ALIGNMENT = -2,    /* a base or stride not a multiple of the element size e (R12) */
  STRATA_ERR_INDEX_RANGE = -3,  /* (validate) chunk/page index outside the pool or list */
  STRATA_ERR_DUPLICATE = -4,    /* (validate) two tokens of one call target the same destination */
  STRATA_ERR_CUDA = -5,         /* a CUDA runtime call failed (incl. an earlier async fault) */
  STRATA_ERR_OOM = -6,          /* host allocation / registration failed */
  STRATA_ERR_UNSUPPORTED = -7,  /* feature not available on this device / build */
  STRATA_ERR_STALE_TICKET = -8, /* ticket older than the event ring, or not issued yet */
  STRATA_ERR_TIMEOUT = -9,      /* (strata_disk.h) job not settled within the timeout */
  STRATA_ERR_IO = -10           /* (strata_disk.h) a file read / write failed */
};

enum strata_pool_flags {
  STRATA_HOST_HUGEPAGES = 1,     /* library-allocated host tier: MAP_HUGETLB, else THP madvise */
  STRATA_HOST_WRITECOMBINED = 2, /* library-allocated host tier via cudaHostAllocWriteCombined */
  STRATA_VALIDATE = 4,           /* check index lists on the device before every transfer */
  STRATA_HOST_NO_NUMA_BIND = 8,  /* do not bind library-allocated host memory to the GPU's node */
  STRATA_HOST_CUDA_ALLOC = 16,   /* library-allocated host tier via cudaHostAlloc(Mapped|Portable)
                                    instead of mmap + cudaHostRegister */
  STRATA_POOL_SINGLE_KV = 32,    /* one KV buffer per layer (MLA latent cache, KV = 1 in LAYOUTS);
                                    v_ptrs is ignored */
  STRATA_HOST_HEAD_MAJOR = 64    /* host chunks are [Ht][L][K,V][C][D] (LAYOUTS, R28) */
};

/* Transfer engines (strata_xfer.engine). Both are bit-identical; they differ in how bytes move. */
enum strata_engine {
  STRATA_ENGINE_DEFAULT = 0,  /* library choice, always a zero-copy kernel: loads of >= 16 MiB of
                                 16-byte-granular rows take STRATA_ENGINE_LDG at the paper's 2 x 1024
                                 threads (the same ~51 GB/s as the ring, less interference with
                                 co-running decode: DESIGN.md §6.1); otherwise STRATA_ENGINE_TMA (the
                                 ring) wherever the tier has whole host rows in 16-byte units (and for
                                 loads of 8- / 4-byte-granular narrow rows), else STRATA_ENGINE_LDG.
                                 The copy engines (DMA) run only when asked for. */
  STRATA_ENGINE_LDG = 1,      /* warps, 16-byte LDG/STG register staging, warp index broadcast; >= 2
                                 CTAs run every layer in one launch */
  STRATA_ENGINE_TMA = 2,      /* the ring engine: one persistent launch per operation; per CTA a TMA
                                 warp moves each page-first host run (<= 16 KiB piece) with one
                                 cp.async.bulk through a shared-memory ring, LSU warps scatter the
                                 rows to their pages (offload: cp.async gather, bulk host store) */
  STRATA_ENGINE_TMA_BULK = 3, /* one warp per CTA, cp.async.bulk on both sides of the ring */
  STRATA_ENGINE_DMA = 4       /* copy-engine gather of whole page-first host runs (one cudaMemcpyAsync
                                 per run, one in-order copy stream) into a double-buffered HBM staging ring + the LDG
                                 kernel scattering staged rows to their pages (offload: the mirror).
                                 Needs strata_xfer.host_chunks_host. */
};

typedef struct {
  int32_t device;                 /* CUDA device ordinal the pool lives on */
  int32_t num_layers;             /* L >= 1 */
  int32_t num_heads;              /* H >= 1: this GPU's KV-head slice (TP shard) */
  int32_t head_dim;               /* D >= 1 */
  int32_t elem_bytes;             /* e >= 1 (2 for fp16/bf16) */
  int32_t page_size;              /* P >= 1: device tokens per page */
  int32_t chunk_tokens;           /* C >= 1: host tokens per chunk */
  int32_t flags;                  /* strata_pool_flags */
  void* const* k_ptrs;            /* [num_layers] device base of each layer's K buffer (copied) */
  void* const* v_ptrs;            /* [num_layers] device base of each layer's V buffer (copied);
                                     NULL allowed with STRATA_POOL_SINGLE_KV */
  int64_t page_stride;            /* device bytes between pages   (0 = P*H*D*e) */
  int64_t token_stride;           /* device bytes between tokens  (0 = H*D*e) */
  int64_t head_stride;            /* device bytes between heads   (0 = D*e) */
  int64_t num_pages;              /* device capacity in pages (>= 1) */
  void* host_base;                /* caller host memory to register, or NULL: library allocates */
  int64_t num_chunks;             /* host capacity in chunks (>= 1) */
  int32_t host_heads;             /* Ht: heads per token in the host tier (0 = num_heads) */
  int32_t head_begin;             /* h0: first host head this GPU moves; h0 + num_heads <= Ht */
} strata_pool_desc;

typedef struct {
  int32_t num_reqs;               /* R >= 0 */
  int32_t layer_begin;            /* l0, half-open layer range [l0, l1) (R11) */
  int32_t layer_end;              /* l1, 0 <= l0 <= l1 <= L */
  int32_t engine;                 /* strata_engine */
  int32_t num_ctas;               /* SM quota; 0 = library default (ring loads:
                                     2 CTAs, 4 for rows < 1 KiB; ring offloads: 4; operations below
                                     16 MiB: up to 16, every piece in flight; LDG: 2 for loads, 1
                                     for offloads) */
  int32_t threads;                /* threads per CTA for STRATA_ENGINE_LDG; 0 = default */
  const int64_t* num_tokens;      /* [R] host: tokens to move per request (>= 0) */
  const int32_t* host_chunks;     /* device int32: all requests' chunk lists concatenated */
  const int64_t* chunk_start;     /* [R] host: start of request r's list in host_chunks */
  const int32_t* dev_pages;       /* device int32: all requests' page lists concatenated */
  const int64_t* page_start;      /* [R] host: start of request r's list in dev_pages */
  const int32_t* chunk_offset;    /* [R] host or NULL (= 0): token offset inside the first chunk */
  const int32_t* page_offset;     /* [R] host or NULL (= 0): token offset inside the first page */
  int64_t host_chunks_len;        /* entries in host_chunks (0 = unknown: list bounds unchecked) */
  int64_t dev_pages_len;          /* entries in dev_pages   (0 = unknown) */
  const int32_t* host_chunks_host;/* host mirror of host_chunks (same content), or NULL.  Required by
                                     STRATA_ENGINE_DMA (the CPU issues the copy-engine gathers);
                                     ignored by the kernel engines. */
  int32_t layer_group;            /* STRATA_ENGINE_DMA: copy G consecutive layers of a chunk as one
                                     run (page-first chunks keep them contiguous).  Layer l's event
                                     then completes with its group [l0 + G*k, l0 + G*(k+1)), i.e.
                                     coarser overlap for larger copies.  0 or 1 = per layer. */
  int32_t inflight_kib;           /* ring engine: host bytes kept in flight over all CTAs, in KiB
                                     (0 = library default: 224, 320 for rows < 2 KiB).  The
                                     interference knob of
                                     PAPER.md:257-262 beside num_ctas: co-running HBM-bound work slows
                                     with the host reads queued, not with the SMs used.
                                     Ignored by the other engines. */
} strata_xfer;

/* Register the host tier and bind it to the device pool described by *d ("CPU registered pinned
 * memory" the I/O kernels read directly, §4.2; a node-sized pinned tier).
 * Host memory: if d->host_base != NULL it must hold num_chunks*chunk_bytes bytes, aligned to the
 * element size; the library page-locks and maps it (cudaHostRegisterMapped|Portable) and
 * unregisters it when the LAST pool whose tier lies inside that registration closes (several pools
 * — e.g. the TP ranks of one process — may share one caller tier); memory the caller registered
 * itself is never unregistered by the library; the caller keeps ownership.  A range that overlaps an
 * open pool's caller tier without lying inside it is rejected (INVALID_ARG): register the enclosing
 * range first.  If NULL, the library allocates it
 * (NUMA-local to the GPU, pre-touched, optionally huge pages / write-combined), owns and frees it.
 * Device buffers stay caller-owned and must outlive the handle.
 * Errors: INVALID_ARG, ALIGNMENT, OOM, CUDA.  On error *out is set to NULL. */
int strata_register_host_pool(const strata_pool_desc* d, strata_pool_t* out);

/* Wait for the pool's outstanding operations, unregister (and free if library-owned) the host
 * tier, destroy the events.  NULL is a no-op. */
int strata_unregister_host_pool(strata_pool_t p);

/* Host address and size of the registered host tier (for filling / reading it on the CPU). */
int strata_host_pool_ptr(strata_pool_t p, void** host_base, size_t* bytes);

/* LOAD (§4.2 GPU-assisted I/O; the page-first -> layer-first transform of
 * PAPER.md:284-290 §4.2.1; page-table indirection PAPER.md:653-655 §2.2): for every request r,
 * token i < num_tokens[r], layer l in [l0,l1), kv, head: copy D*e bytes
 * from the host tier to the device pool (addresses in the LAYOUTS block).  Enqueued on `stream`;
 * layers are processed in increasing order and event (ticket, l) completes once every byte of
 * layer l of this call is in the device pool.  n = 0 or l0 = l1 is a successful no-op that still
 * records the events of the covered layers.  Index lists must stay valid until the stream passes
 * the operation (same contract as cudaMemcpyAsync).  Duplicate destinations are a caller error
 * (rejected under STRATA_VALIDATE, unspecified otherwise); duplicate sources are legal.
 * *ticket (nullable) receives the operation's ticket for strata_layer_event. */
int strata_load(strata_pool_t p, const strata_xfer* x, strata_stream_t stream, uint64_t* ticket);

/* OFFLOAD ("backup"): the inverse scatter, device pool -> host tier, same
 * arguments and event semantics.  Host bytes are CPU-visible once the layer's event (or the
 * stream) has completed. */
int strata_offload(strata_pool_t p, const strata_xfer* x, strata_stream_t stream, uint64_t* ticket);

/* Per-layer completion (§4.1): the library-owned event recorded after layer `layer`
 * of operation `ticket` (0 = the latest operation).  The event stays valid until the ring slot is
 * reused 8 operations later; an older ticket returns STRATA_ERR_STALE_TICKET.  A layer outside the
 * operation's range returns STRATA_ERR_INVALID_ARG.  Use with cudaStreamWaitEvent /
 * cudaEventSynchronize; never destroy it.  An operation issued while its stream was being captured
 * into a CUDA graph (CAPTURED ticket) has its own events, recorded as external event nodes of the
 * graph: every replay signals them, so this returns the event of the LATEST replay's layer, and a
 * captured ticket never goes stale while the pool lives (its events are destroyed with the pool).
 * strata_wait_layer on a captured ticket from a consumer stream captured into the same graph waits
 * on the capture-internal event instead (a graph edge; needs the ticket's ring slot not yet reused,
 * else STRATA_ERR_STALE_TICKET).  A new operation that
 * reuses a ring slot is ordered after the slot's previous one-launch operation (whose device-side
 * layer flags it shares), so a layer event never fires before that layer's bytes landed. */
int strata_layer_event(strata_pool_t p, uint64_t ticket, int32_t layer, strata_event_t* out);

/* Decode-aware SM quota (NEXT-1; "a small number of large CUDA blocks", DESIGN.md
 * §6.1): a stream-ordered cap on the CTAs that take new work in this pool's running and later
 * one-launch LDG loads (the default engine for loads >= 16 MiB of 16-byte rows).  Enqueues on
 * `stream` a device write of `max_ctas` to the pool's quota word (cuStreamWriteValue32); 0 lifts
 * the cap.  Loads launched after the FIRST call assign row groups dynamically: while the cap is
 * q > 0, CTAs q, q+1, ... take no new rows (their SMs keep no host reads in flight) and CTAs
 * 0..q-1 move the rest, so every result stays bit-exact and every layer event still fires.  Typical
 * use: strata_set_load_quota(pool, 1, decode_stream) before a decode step, (pool, 0, decode_stream)
 * after it.  Loads launched before the first call, ring / per-layer launches and offloads ignore
 * it.  The word is library-owned device memory, zeroed at registration; calls may be captured
 * into CUDA graphs.  Errors: STRATA_ERR_INVALID_ARG (max_ctas < 0), STRATA_ERR_UNSUPPORTED (no
 * stream memory operations), STRATA_ERR_CUDA. */
int strata_set_load_quota(strata_pool_t p, int32_t max_ctas, strata_stream_t stream);

/* Consumer-side wait: make stream `consumer` wait until layer `layer` of operation
 * `ticket` (0 = latest) is complete — cudaStreamWaitEvent on the layer's event.  Errors as
 * strata_layer_event, plus STRATA_ERR_CUDA. */
int strata_wait_layer(strata_pool_t p, uint64_t ticket, int32_t layer, strata_stream_t consumer);

/* Milliseconds from the start of operation `ticket` (0 = latest) on its stream to the completion of
 * layer `layer` (CUDA event timing).  Blocks until that layer is complete.  Errors as
 * strata_layer_event, plus STRATA_ERR_CUDA (also: a captured ticket whose graph has not been
 * replayed yet; after a replay it times that replay). */
int strata_layer_elapsed_ms(strata_pool_t p, uint64_t ticket, int32_t layer, float* ms);

/* Cumulative per-pool counters since registration (observability; no synchronisation). */
typedef struct {
  int64_t operations;       /* strata_load + strata_offload calls that returned STRATA_OK */
  int64_t kernel_launches;  /* libstrata kernels launched (transfer, scatter/gather, validate) */
  int64_t dma_copies;       /* copy-engine copies submitted by STRATA_ENGINE_DMA */
  int64_t bytes;            /* algorithmic KV bytes moved (2*H*D*e per token per layer) */
  int32_t last_engine;      /* strata_engine that executed the most recent operation */
  int32_t reserved;
} strata_counters;

int strata_get_counters(strata_pool_t p, strata_counters* out);

/* Thread-local message describing the last non-OK return on this thread ("" if none). */
const char* strata_last_error(void);

/* Library version as 10000*major + 100*minor + patch. */
int strata_version(void);

#ifdef __cplusplus
}
#endif

#endif /* STRATA_H */
