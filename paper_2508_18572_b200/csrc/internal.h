// internal.h — libstrata internals shared by the host side (api.cpp, transfer.cpp, dma.cpp,
// baselines.cpp, disk.cpp) and the sm_100a kernels (kernels.cu).  Not part of the ABI; see
// include/strata.h for the contract.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/strata.h"

namespace strata {

// Requests per kernel launch: their tables travel in the kernel parameters (no staging copy, so a
// call is graph-capturable).  Calls with more requests are split into several launches per layer.
constexpr int kMaxReqsPerLaunch = 128;
constexpr int kEventRing = 8;          // operations whose per-layer events stay valid

// Per-launch request table (struct of arrays).  Flat token index g in [0, ntok) enumerates the
// tokens of the launch's requests in order; request r owns [tok_end[r-1], tok_end[r]).
struct ReqTable {
  int32_t n;
  int32_t tok_end[kMaxReqsPerLaunch];
  int32_t chunk_base[kMaxReqsPerLaunch];   // chunk_start[r]: first entry of r's chunk list
  int32_t page_base[kMaxReqsPerLaunch];    // page_start[r]
  int32_t off_c[kMaxReqsPerLaunch];        // token offset inside the first host chunk
  int32_t off_p[kMaxReqsPerLaunch];        // token offset inside the first device page
};

// Everything one per-layer launch needs; passed by value as a __grid_constant__ parameter.
struct XferParams {
  // geometry (bytes unless noted)
  int32_t C, P;                 // host chunk tokens, device page tokens
  int32_t H;                    // heads of this GPU's slice
  int32_t tok_bytes;            // S_tok = H*D*e (one token, one of K/V, one layer)
  int32_t head_bytes;           // D*e
  int32_t vpt;                  // 16-byte vectors per token row = tok_bytes/16
  int32_t vpt_shift;            // log2(vpt) if vpt is a power of two, else -1
  uint32_t vpt_magic;           // else: row = umulhi(idx, vpt_magic) exactly for idx < 32*vpt (0 = divide)
  int32_t vph;                  // 16-byte vectors per head = head_bytes/16
  int32_t vph_shift;            // log2(vph) if a power of two, else -1
  int32_t rows_per_group;       // LDG engine: token rows handled by one warp iteration (<= 32)
  int32_t tma_rows;             // TMA engine: token rows per pipeline stage (<= 32)
  int32_t tma_stages;           // TMA engine: pipeline depth
  int32_t tma_stage_bytes;      // TMA engine: bytes per stage (>= tma_rows * tok_bytes)
  int32_t c_shift, p_shift;     // log2(C), log2(P) when powers of two, else -1
  int64_t chunk_bytes;          // L*KV*C*S_tok
  int64_t layer_off;            // byte offset of (layer, K) inside a host chunk: l*KV*C*S_tok
  int64_t kv_off;               // K -> V offset in the host tier: C*Ht*D*e (token-major), C*D*e (head-major)
  int64_t page_stride, token_stride, head_stride;
  // host side of a row (R28): token cr, head h of a chunk-layer-kv block starts at
  //   block + cr*host_tok_stride + host_head_off + h*host_head_stride
  // token-major: (Ht*D*e, h0*D*e, D*e); head-major: (D*e, h0*L*KV*C*D*e, L*KV*C*D*e)
  int64_t host_tok_stride, host_head_off, host_head_stride;
  // data
  char* host;                   // device-visible address of the host tier (UVA)
  char* kbase;                  // this layer's K buffer
  char* vbase;                  // this layer's V buffer
  const int32_t* host_chunks;   // device index lists
  const int32_t* dev_pages;
  int32_t ntok;                 // tokens in this launch
  int32_t nkv;                  // KV buffers per layer: 2 (K, V) or 1 (MLA latent); rows = nkv*ntok
  int32_t gran;                 // 16: vectorised kernels; 8/4/2/1: the narrow LDG kernel (R29)
  int32_t wpr, wph;             // narrow kernel: gran-byte words per row / per head
  uint32_t wpr_magic, wph_magic;   // their multiply-high divisors (0 = divide)
  ReqTable rt;
};

struct ValidateParams {
  int32_t C, P;
  int32_t ntok;
  int32_t dir;                  // 0 load (destinations = device slots), 1 offload (host slots)
  int64_t num_pages, num_chunks;
  int64_t chunks_len, pages_len;   // list lengths (0 = unknown)
  const int32_t* host_chunks;
  const int32_t* dev_pages;
  uint32_t* bitmap;             // one bit per destination slot, zeroed by the caller
  int32_t* err;                 // bit 0: index range, bit 1: duplicate
  ReqTable rt;
};

// One launch for every layer of an LDG operation (kernels.cu ldg_fused_kernel).
constexpr int kMaxFusedLayers = 128;
struct FusedParams {
  XferParams x;                 // geometry, index lists, request table (kbase/vbase/layer_off unused)
  int32_t l0, l1;               // layer range
  uint32_t epoch;               // published to flags[l] when layer l is complete
  int32_t total_warps;          // warps in the grid (each arrives once per layer)
  uint32_t* counters;           // [L] arrival counters of this op slot (0 on entry, reset by the kernel)
  uint32_t* flags;              // [L] completion flags of this op slot
  uint32_t* loads_active;       // load: the device-wide running-load counter ring offloads pace beside
                                // (ring_loads_active()); NULL for offloads
  uint32_t* next;               // [L] row-group counters of this op slot (dynamic assignment, quota path)
  const int32_t* quota;         // load: the pool's quota word (strata_set_load_quota), or NULL: static
                                // group assignment (ldg_fused_kernel); else ldg_quota_kernel
  char* kb[kMaxFusedLayers];    // per-layer K / V bases
  char* vb[kMaxFusedLayers];
};

// The ring engine (ring.cu, STRATA_ENGINE_TMA): a persistent kernel over every layer of an operation
// whose unit of work is a PIECE — up to `rows` consecutive tokens of one (request, host chunk, K|V)
// segment, i.e. one contiguous run of the page-first host chunk.  A piece crosses
// the host link as ONE cp.async.bulk (TMA) through a `stages`-deep shared-memory ring; its rows are
// scattered to / gathered from their pages on the device side.
//   piece k of a layer: segment k / pps, sub-piece k % pps; segment -> (pair = chunk position of a
//   request, kv); pair -> request by binary search over pair_end.
constexpr int kRingMaxStages = 16;
constexpr int kRingMaxWarps = 16;   // LSU scatter warps of a load CTA
constexpr int kRingMaxRows = 64;    // rows per piece (2 per lane of the piece's warp)
struct RingParams {
  XferParams x;                 // geometry, index lists, request table (kbase/vbase/layer_off unused)
  int32_t l0, l1;               // layer range
  uint32_t epoch;               // published to flags[l] when layer l is complete
  int32_t arrivals;             // arrivals per layer: load = CTAs * warps, offload = CTAs
  uint32_t* counters;           // [L] arrival counters of the op slot, or NULL: no per-layer flags
  uint32_t* flags;              // [L] completion flags of the op slot
  int32_t rows;                 // R: rows per piece (<= kRingMaxRows)
  int32_t stages;               // S: ring depth (<= kRingMaxStages)
  int32_t stage_bytes;          // bytes per stage (R * tok rounded up to 128)
  int32_t pps;                  // pieces per segment = ceil(C / R)
  int32_t npieces;              // pieces per layer
  int32_t host_run;             // 1: a piece's host rows are one contiguous run (host_tok_stride == tok)
  int32_t warps;                // device-side LSU warps per CTA: load scatter / offload gather (+1 TMA warp)
  int32_t bulk_store;           // load: the device side as cp.async.bulk stores instead of st.global
  int32_t smem_reserve;         // > 0: dynamic shared memory to request (>= the ring's): keeps the SM exclusive
  uint32_t word_magic;          // narrow rows: row of word v < R*tok/gran = umulhi(v, magic) (0: divide)
  int32_t debug;                // A/B experiments only (env STRATA_RING_DEBUG): bit 0 = skip the page writes
  int32_t pace_ps_per_byte;     // offload: while ring loads run on the device, this CTA issues its host
                                // stores at most one byte per pace_ps_per_byte ps (0 = unpaced)
  int32_t pair_end[kMaxReqsPerLaunch];   // inclusive prefix sums of chunk positions per request
  char* kb[kMaxFusedLayers];    // per-layer K / V bases
  char* vb[kMaxFusedLayers];
};
// Shared-memory bytes in front of the ring's stages (mbarriers).
int ring_header_bytes();
// Device address of the running-load counter of the current device (ring.cu's g_loads_active): every
// running load CTA (ring, fused LDG) counts itself in it; ring offloads pace their host stores while
// it is non-zero.
uint32_t* ring_loads_active();
cudaError_t launch_ring(const RingParams& p, int dir, int ctas, cudaStream_t s);
cudaError_t ring_prepare(int smem);

// Kernel launchers (kernels.cu).  dir: 0 = load (host -> device), 1 = offload (device -> host).
cudaError_t launch_ldg(const XferParams& p, int dir, int ctas, int threads, int unroll, cudaStream_t s);
cudaError_t launch_ldg_fused(const FusedParams& p, int dir, int ctas, int threads, cudaStream_t s);
// STRATA_ENGINE_TMA_BULK: one warp per CTA, cp.async.bulk on both sides of a shared-memory ring.
cudaError_t launch_tma(const XferParams& p, int dir, int ctas, cudaStream_t s);
cudaError_t launch_validate(const ValidateParams& v, cudaStream_t s);
// Largest dynamic shared memory the TMA engine may use per CTA on this device.
int tma_smem_limit();
// Shared-memory bytes in front of the TMA ring (mbarriers + per-stage address tables).
int tma_header_bytes(int stages);
// Opt the TMA kernels in to `smem` bytes of dynamic shared memory on the current device.
cudaError_t tma_prepare(int smem);
constexpr int kTmaMaxStages = 32;

// Records `msg` as this thread's strata_last_error() and returns `code` (api.cpp).
int set_last_error(int code, const char* msg);

}  // namespace strata

struct strata_pool {
  strata_pool_desc d;                 // copy; k_ptrs/v_ptrs re-pointed at the vectors below
  std::vector<void*> k, v;
  int64_t tok_bytes, head_bytes, chunk_bytes;
  int32_t nkv = 2;                    // KV buffers per layer (1: STRATA_POOL_SINGLE_KV)
  int32_t gran = 16;                  // widest access dividing every row, stride and base (R29)
  int32_t host_heads = 0, head_begin = 0;   // Ht, h0 (R28)
  bool head_major = false;
  int64_t host_kv_off = 0, host_tok_stride = 0, host_head_off = 0, host_head_stride = 0;
  // a host row (this GPU's heads of one token) is tok_bytes contiguous: what the TMA rings need
  bool host_row_contig() const { return host_head_stride == head_bytes || d.num_heads == 1; }
  int64_t page_stride, token_stride, head_stride;
  // host tier
  char* host = nullptr;               // host address
  char* host_dev = nullptr;           // device-visible address (UVA: usually == host)
  size_t host_bytes = 0;
  int host_kind = 0;                  // 0 caller memory, 1 mmap (library), 2 cudaHostAlloc (library)
  bool registered_by_us = false;
  size_t map_bytes = 0;               // mmap length
  // per-layer completion events: ring of kEventRing operations x L layers
  std::vector<cudaEvent_t> events;
  // fused: the op ran as one fused LDG launch; its layer l is complete once flags[slot][l] >= epoch
  // captured: recorded into a CUDA graph capture; its events exist only inside that graph
  struct Op { uint64_t ticket; int32_t l0, l1; bool fused = false; bool captured = false; };
  Op ops[strata::kEventRing];
  // captured operations: their own L+1 events (start, layers), recorded as EXTERNAL event nodes so
  // every replay of the graph signals them; kept while the pool lives (a captured ticket never goes
  // stale), keyed by ticket.  The ring slot's events are recorded too (capture-internal: a consumer
  // captured into the same graph waits on those, which become graph edges).
  struct CapturedOp { int32_t l0, l1; std::vector<cudaEvent_t> ev; };
  std::map<uint64_t, CapturedOp> captured_ops;
  uint64_t next_ticket = 1;
  // validate scratch (device)
  uint32_t* bitmap = nullptr;
  size_t bitmap_words = 0;
  int32_t* err_dev = nullptr;
  int32_t* err_host = nullptr;        // pinned
  int tma_smem = 0;
  uint32_t* loads_active = nullptr;   // device address of the running-load counter (ring_loads_active())
  strata_counters counters = {};
  // STRATA_ENGINE_DMA, one state per direction (0 load, 1 offload; lazy): a double-buffered HBM
  // staging ring, copy streams and their events.  Separate per direction so a load and an offload
  // of one pool can be in flight at once on different streams (both directions of the link);
  // `seq` numbers the pieces of a direction across operations, so an operation on another stream
  // waits for the previous one's last use of a staging slot (tests/test_gpu_concurrent.py).
  // Copy streams: capacity kCopyStreams, `ncs` used (env STRATA_COPY_STREAMS).  Default 1: one
  // in-order copy stream beats 2-8 on every config and in both directions
  // (profiles/r01/copy_streams: Llama-8B 55.36 vs 54.37 GB/s at 1 vs 4; bidirectional 101 vs 91)
  static constexpr int kCopyStreams = 8;
  struct DmaDir {
    int ncs = 1;
    char* stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;           // bytes per staging slot
    cudaStream_t cs[kCopyStreams] = {};
    cudaEvent_t ev_fork = nullptr;
    cudaEvent_t ev_slot[2] = {nullptr, nullptr};   // staging slot reusable
    cudaEvent_t ev_copy[2][kCopyStreams] = {};     // a slot's copies done, per stream
    // a second set of the three above, swapped in while an operation is being captured: records
    // made inside a capture must not become the 'latest record' a later live operation waits on
    cudaEvent_t cap_fork = nullptr;
    cudaEvent_t cap_slot[2] = {nullptr, nullptr};
    cudaEvent_t cap_copy[2][kCopyStreams] = {};
    uint64_t seq = 0;                 // pieces issued in this direction so far
    bool captured = false;            // a graph captured this direction: its buffers must not move
  } dma[2];
  int32_t* slot_ids = nullptr;        // device iota [0, slot_cap): chunk index of each staging slot
  int64_t slot_cap = 0;
  // fused LDG operations (lazy): per op slot, L arrival counters + L layer flags (device), and a side
  // stream that turns each flag into the layer's event (cuStreamWaitValue32 + cudaEventRecord)
  uint32_t* fused_sync = nullptr;     // [kEventRing][3][L]: arrival counters, layer flags, group counters
  int32_t* quota = nullptr;           // decode-aware load quota word (in fused_sync) once strata_set_load_quota ran, else NULL
  cudaStream_t side[strata::kEventRing] = {};
  int fused_state = 0;                // 0 untried, 1 ready, -1 unavailable (stream memory ops missing)
};

// ------------------------------------------------------------------------------------------------
// Shared between api.cpp (ABI surface), transfer.cpp (validation, planning, kernel engines) and
// dma.cpp (copy-engine engine).
namespace strata {

// Records a formatted message as strata_last_error() and returns `code` (api.cpp).
int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int cuda_fail(cudaError_t e, const char* what);

// Makes `dev` current for the scope, restoring the caller's device afterwards.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// Per-call plan: the non-empty requests, split into launches (batches) of <= kMaxReqsPerLaunch.
struct Batch {
  int32_t first, count;     // requests [first, first+count) among the non-empty ones
  int32_t ntok;
};

struct Plan {
  std::vector<int32_t> reqs;   // indices of requests with tokens
  std::vector<Batch> batches;
  int64_t total_tokens = 0;
};

// Defaults chosen on B200 measurements.
// The paper's quota: 2 CTAs x 1024 threads.  On B200 that moves 50.3 GB/s (90.7 % of
// the link) with 0.8 % prefill-GEMM and 10.8 % decode slowdown (profiles/r01/interference2.jsonl).
constexpr int kDefaultCtasLdg = 2;
// The paper's backup quota: "one block for backing up data from GPU to CPU (a non-critical path),
// where the bandwidth is already sufficient and overhead must be minimized".  On B200
// one 1024-thread CTA offloads 39-40 GB/s and costs a co-running decode ~5 % instead of ~12 %.
constexpr int kDefaultCtasLdgOffload = 1;
// The narrow kernel (R29) streams 8-byte or smaller words (half the bytes in flight per warp of the
// 16-byte LDG engine): it saturates from 16 CTAs (72 / 100 / 120-byte rows: 46.4 / 46.6 / 48.2 GB/s;
// profiles/r01/final/narrow_probe.jsonl).
constexpr int kDefaultCtasNarrow = 16;
constexpr int kDefaultThreadsLdg = 1024;   // host-read throughput of an SM scales with its warps
constexpr int64_t kDmaMinLayerBytes = int64_t(4) << 20;
constexpr int64_t kDmaMinOffloadRun = int64_t(128) << 10;
constexpr int64_t kDmaMinLoadRun = int64_t(24) << 10;   // default engine: DMA loads need >= 24 KiB runs
constexpr int kDefaultUnroll = 8;
constexpr int kDefaultCtasTma = 2;   // STRATA_ENGINE_TMA_BULK (scaled up for small rows, transfer.cpp)
// The ring engine (ring.cu), the default.  Loads: CTAs of 1 producer + kDefaultRingWarps scatter
// warps; offloads: CTAs of 1 gather + 1 store warp; 32 KiB pieces, as many stages as fit.
// Quotas (profiles/r02/ring_sweep6_bulkstore_70b.jsonl, ring_sweep5_warp_pieces.jsonl): rows of >= 1 KiB
// reach the SM zero-copy plateau (51.4 GB/s load, 52.6 offload) from 2 CTAs, 256-byte rows (70B TP=8)
// need 4 (2 CTAs: 43.8 / 40.1).  One CTA tops out at ~36-39 GB/s: the SM's L1->XBAR request path
// (profiles/r02/ncu_ring_load_1cta_v4.txt).
constexpr int kDefaultCtasRingLoad = 2;
// Offloads: 4 CTAs.  The cp.async gathers of a large, randomly paged pool keep 2 CTAs below the link
// (Qwen-14B batch, 70 GiB pool: 49.8 GB/s from 2 CTAs, 52.7 from 3 or 4; 1152-byte MLA rows 48.0 vs
// 52.1; Llama-8B 52.2-52.6 either way: profiles/r02/probe2/sweep_qwen_off.jsonl, sweep70/, probe4/).
// The paper gives backups one block as a non-critical path; on B200 the SM count of
// the I/O kernel does not move the co-runners' slowdown, the bytes in flight do.
constexpr int kDefaultCtasRingOffload = 4;
// While ring loads run on the device, offloads pace themselves to this many GB/s in total
// (RingParams::pace_ps_per_byte; 0 = unpaced).  A load and an unpaced offload in flight together
// leave the load 15 GB/s (the offload's posted writes crowd out its read requests; waiting for store
// completion does not help); paced to 16 GB/s the load keeps 48.7 of its 51.2 GB/s while the backup
// continues — the backup is the non-critical path.  Offloads alone are not paced.
// (profiles/r02/bidir/pacing/)
constexpr int kDefaultOffloadShareGBs = 16;
constexpr int kRingSmallRowBytes = 1024;   // rows below this take twice the quota
constexpr int64_t kSmallOpBytes = int64_t(16) << 20;   // ring operations below this: all pieces in flight
constexpr int kSmallOpCtas = 16;
constexpr int kDefaultRingWarps = 8;         // load: scatter warps
constexpr int kDefaultRingGatherWarps = 8;   // offload: cp.async gather warps
constexpr int kDefaultRingStageKB = 16;
constexpr int kDefaultRingInflightKB = 224;  // host bytes in flight over all CTAs (2 CTAs: 7 x 16 KiB each)
// Rows shorter than 2 KiB keep their stages longer on the device side (more rows, more page-table
// entries, and for 1152-byte MLA rows a non-power-of-two vector count per piece), so fewer of the
// ring's bytes are on the link at any moment: 224 KiB moves 44.7 GB/s for 256-byte rows (70B TP=8, 4
// CTAs) and 45.7 for 1152-byte rows (2 CTAs), 320 KiB 50.4 / 51.0 (profiles/r02/sweep70/).
constexpr int kRingShortRowBytes = 2048;
constexpr int kDefaultRingInflightShortKB = 320;
constexpr int kDefaultRingExclusive = 0;     // 1: a ring CTA reserves its SM's shared memory
constexpr int kTmaStageTarget = 32 << 10;

int check_xfer(const strata_pool* p, const strata_xfer* x, Plan& plan);                     // transfer.cpp
void fill_table(const strata_xfer* x, const Plan& plan, const Batch& b, ReqTable& rt);        // transfer.cpp
int ilog2_exact(int v);                                                                       // transfer.cpp
bool dma_runs_ok(const strata_pool* p);                                                       // transfer.cpp
uint32_t div_magic(int d, int n_max);   // m with umulhi(n, m) == n / d for n < n_max, or 0  transfer.cpp
int transfer(strata_pool* p, const strata_xfer* x, cudaStream_t s, uint64_t* ticket, int dir); // transfer.cpp
// Records event `idx` (0 = start, 1 + l = layer l) of the operation in ring slot `slot` on `s`; for a
// captured operation also its dedicated event as an external node (transfer.cpp).
cudaError_t op_record(strata_pool* p, int slot, int idx, cudaStream_t s);
int transfer_dma(strata_pool* p, const strata_xfer* x, const Plan& plan, XferParams xp, cudaStream_t s,
                 int dir, int slot_ev);                                                       // dma.cpp
void free_dma(strata_pool* p);
void free_fused(strata_pool* p);
cudaError_t set_load_quota(strata_pool* p, int32_t max_ctas, cudaStream_t s);   // transfer.cpp
bool ensure_fused(strata_pool* p);   // fused-LDG resources; false: unavailable (per-layer path) transfer.cpp
// Consumer-side wait on a fused operation's layer flag (stream memory op), transfer.cpp.
cudaError_t wait_fused_layer(strata_pool* p, int slot, int32_t layer, cudaStream_t consumer);                                                              // transfer.cpp                                                                // dma.cpp

}  // namespace strata
