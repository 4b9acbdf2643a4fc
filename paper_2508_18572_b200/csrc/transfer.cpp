// transfer.cpp — per-call validation, planning and the kernel engines (LDG, TMA) of strata_load /
// strata_offload (include/strata.h).
//
// Launch planning: per call, validate, split the requests into launches of
// at most kMaxReqsPerLaunch whose tables travel in the kernel parameters, pick the engine and the SM
// quota ("a small number of large CUDA blocks"), then for every layer l in
// [l0, l1): launch, and record event (ticket, l) (§4.1: the executor waits per layer).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"
#include "../../include/strata_test.h"

namespace strata {

namespace {

using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32Fn g_wait_value32 = nullptr;
WaitValue32Fn g_write_value32 = nullptr;   // cuStreamWriteValue32 has the same signature

// STRATA_LDG_FUSED: "0" keeps the one-launch-per-layer LDG path (A/B and fallback testing);
// "force" fuses 1-CTA grids too (profiling); default: fused from 2 CTAs.
int fused_mode() {
  static const int mode = [] {
    const char* v = std::getenv("STRATA_LDG_FUSED");
    if (v && v[0] == '0') return 0;
    if (v && std::strcmp(v, "force") == 0) return 2;
    return 1;
  }();
  return mode;
}

// Lazily: per op slot 3*L device words (arrival counters, layer flags, row-group counters) and a side stream; the
// driver's stream memory operation cuStreamWaitValue32 through the runtime's entry-point query,
// probed once on a zero flag.  Unavailable -> the per-layer path is used.
}  // namespace

bool ensure_fused(strata_pool* p) {
  if (p->fused_state) return p->fused_state > 0;
  p->fused_state = -1;
  if (!g_wait_value32) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    g_wait_value32 = reinterpret_cast<WaitValue32Fn>(fn);
  }
  const size_t words = size_t(kEventRing) * 3 * p->d.num_layers + 1;   // + the decode-aware quota word
  if (cudaMalloc(&p->fused_sync, words * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemset(p->fused_sync, 0, words * sizeof(uint32_t)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  for (int i = 0; i < kEventRing; ++i)
    if (cudaStreamCreateWithFlags(&p->side[i], cudaStreamNonBlocking) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
  if (g_wait_value32(reinterpret_cast<CUstream>(p->side[0]), reinterpret_cast<CUdeviceptr>(p->fused_sync), 0,
                     CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS ||
      cudaStreamSynchronize(p->side[0]) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  p->fused_state = 1;
  return true;
}

cudaError_t wait_fused_layer(strata_pool* p, int slot, int32_t layer, cudaStream_t consumer) {
  const int L = p->d.num_layers;
  uint32_t* flag = p->fused_sync + size_t(slot) * 3 * L + L + layer;
  const uint32_t epoch = static_cast<uint32_t>(p->ops[slot].ticket);
  return g_wait_value32(reinterpret_cast<CUstream>(consumer), reinterpret_cast<CUdeviceptr>(flag), epoch,
                        CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

void free_fused(strata_pool* p) {
  for (int i = 0; i < kEventRing; ++i)
    if (p->side[i]) {
      cudaStreamSynchronize(p->side[i]);
      cudaStreamDestroy(p->side[i]);
      p->side[i] = nullptr;
    }
  if (p->fused_sync) cudaFree(p->fused_sync);
  p->fused_sync = nullptr;
  p->fused_state = 0;
  p->quota = nullptr;   // a word of fused_sync
}

// Decode-aware quota (NEXT-1): the pool's quota word (the last word of fused_sync, zeroed with it at
// registration), written in stream order by the driver's cuStreamWriteValue32; the first call makes
// the pool's later one-launch LDG loads read it.
cudaError_t set_load_quota(strata_pool* p, int32_t max_ctas, cudaStream_t s) {
  if (!g_write_value32) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return cudaErrorNotSupported;
    }
    g_write_value32 = reinterpret_cast<WaitValue32Fn>(fn);
  }
  if (!p->quota) p->quota = reinterpret_cast<int32_t*>(p->fused_sync + size_t(kEventRing) * 3 * p->d.num_layers);
  return g_write_value32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(p->quota),
                         static_cast<cuuint32_t>(max_ctas), 0) == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

int check_xfer(const strata_pool* p, const strata_xfer* x, Plan& plan) {
  if (!x) return fail(STRATA_ERR_INVALID_ARG, "xfer is NULL");
  const int L = p->d.num_layers;
  if (x->layer_begin < 0 || x->layer_begin > x->layer_end || x->layer_end > L)
    return fail(STRATA_ERR_INVALID_ARG, "layer range [%d,%d) not inside [0,%d)", x->layer_begin, x->layer_end, L);
  if (x->num_reqs < 0) return fail(STRATA_ERR_INVALID_ARG, "num_reqs < 0");
  if (x->engine < 0 || x->engine > STRATA_ENGINE_DMA) return fail(STRATA_ERR_INVALID_ARG, "unknown engine %d", x->engine);
  if (x->num_ctas < 0 || x->num_ctas > 65535) return fail(STRATA_ERR_INVALID_ARG, "num_ctas out of range");
  if (x->layer_group < 0) return fail(STRATA_ERR_INVALID_ARG, "layer_group < 0");
  if (x->threads < 0 || x->threads > 1024 || x->threads % 32)
    return fail(STRATA_ERR_INVALID_ARG, "threads must be a multiple of 32 in [32,1024]");
  if (x->num_reqs == 0) return STRATA_OK;
  if (!x->num_tokens || !x->chunk_start || !x->page_start)
    return fail(STRATA_ERR_INVALID_ARG, "num_tokens / chunk_start / page_start is NULL");
  const int64_t C = p->d.chunk_tokens, P = p->d.page_size;
  for (int32_t r = 0; r < x->num_reqs; ++r) {
    const int64_t n = x->num_tokens[r];
    if (n < 0) return fail(STRATA_ERR_INVALID_ARG, "num_tokens[%d] < 0", r);
    if (n == 0) continue;
    const int64_t oc = x->chunk_offset ? x->chunk_offset[r] : 0;
    const int64_t op = x->page_offset ? x->page_offset[r] : 0;
    if (oc < 0 || oc >= C) return fail(STRATA_ERR_INVALID_ARG, "chunk_offset[%d]=%lld not in [0,C)", r, (long long)oc);
    if (op < 0 || op >= P) return fail(STRATA_ERR_INVALID_ARG, "page_offset[%d]=%lld not in [0,P)", r, (long long)op);
    const int64_t cs = x->chunk_start[r], ps = x->page_start[r];
    const int64_t nc = (oc + n + C - 1) / C, np = (op + n + P - 1) / P;
    if (cs < 0 || ps < 0 || cs + nc > INT32_MAX || ps + np > INT32_MAX)
      return fail(STRATA_ERR_INDEX_RANGE, "request %d list start out of range", r);
    if (x->host_chunks_len > 0 && cs + nc > x->host_chunks_len)
      return fail(STRATA_ERR_INDEX_RANGE, "request %d needs host_chunks[%lld..%lld) beyond length %lld", r,
                  (long long)cs, (long long)(cs + nc), (long long)x->host_chunks_len);
    if (x->dev_pages_len > 0 && ps + np > x->dev_pages_len)
      return fail(STRATA_ERR_INDEX_RANGE, "request %d needs dev_pages[%lld..%lld) beyond length %lld", r,
                  (long long)ps, (long long)(ps + np), (long long)x->dev_pages_len);
    plan.reqs.push_back(r);
    plan.total_tokens += n;
  }
  if (plan.total_tokens > 0 && (!x->host_chunks || !x->dev_pages))
    return fail(STRATA_ERR_INVALID_ARG, "host_chunks / dev_pages is NULL");
  // batches: <= kMaxReqsPerLaunch requests and < 2^30 tokens per launch
  const int64_t kMaxTok = int64_t(1) << 30;
  Batch b{0, 0, 0};
  for (size_t k = 0; k < plan.reqs.size(); ++k) {
    const int64_t n = x->num_tokens[plan.reqs[k]];
    if (n > kMaxTok) return fail(STRATA_ERR_INVALID_ARG, "request with >= 2^30 tokens");
    if (b.count == kMaxReqsPerLaunch || b.ntok + n > kMaxTok) {
      plan.batches.push_back(b);
      b = Batch{static_cast<int32_t>(k), 0, 0};
    }
    b.count += 1;
    b.ntok += static_cast<int32_t>(n);
  }
  if (b.count) plan.batches.push_back(b);
  return STRATA_OK;
}

void fill_table(const strata_xfer* x, const Plan& plan, const Batch& b, strata::ReqTable& rt) {
  rt.n = b.count;
  int32_t acc = 0;
  for (int32_t k = 0; k < b.count; ++k) {
    const int32_t r = plan.reqs[b.first + k];
    acc += static_cast<int32_t>(x->num_tokens[r]);
    rt.tok_end[k] = acc;
    rt.chunk_base[k] = static_cast<int32_t>(x->chunk_start[r]);
    rt.page_base[k] = static_cast<int32_t>(x->page_start[r]);
    rt.off_c[k] = x->chunk_offset ? x->chunk_offset[r] : 0;
    rt.off_p[k] = x->page_offset ? x->page_offset[r] : 0;
  }
}

// Division by the vectors-per-row count of a non-power-of-two row (MLA latents: 1152 B = 72
// vectors) costs a ~20-instruction integer division per 16-byte vector in the LDG loops; a
// multiply-high by ceil(2^32 / d) is exact for every n < n_max when it is exact at the largest n
// of each quotient (its error grows with n), which is checked here.
uint32_t div_magic(int d, int n_max) {
  if (d <= 1 || n_max <= 0) return 0;
  const uint64_t m = (uint64_t(1) << 32) / uint64_t(d) + 1;
  if (m > 0xffffffffull) return 0;
  for (int64_t q = 0; q * d < n_max; ++q) {
    const int64_t n = std::min<int64_t>(n_max - 1, q * d + d - 1);
    if (static_cast<int64_t>((uint64_t(n) * m) >> 32) != q || static_cast<int64_t>((uint64_t(q * d) * m) >> 32) != q)
      return 0;
  }
  return static_cast<uint32_t>(m);
}

// Copy-engine runs need the GPU's host data of a chunk-layer in few long pieces: token-major
// tiers holding only this GPU's heads (one run per chunk-layer), or head-major tiers (one run per
// chunk-layer and head: K and V of C tokens, any head slice).
bool dma_runs_ok(const strata_pool* p) { return p->head_major || p->host_heads == p->d.num_heads; }

int ilog2_exact(int v) {
  if (v <= 0 || (v & (v - 1))) return -1;
  int s = 0;
  while ((1 << s) < v) ++s;
  return s;
}


static int run_validate(strata_pool* p, const strata_xfer* x, const Plan& plan, int dir, cudaStream_t s) {
  const size_t slots = dir == 0 ? size_t(p->d.num_pages) * p->d.page_size
                                : size_t(p->d.num_chunks) * p->d.chunk_tokens;
  const size_t words = (slots + 31) / 32;
  cudaError_t e;
  if (words > p->bitmap_words) {
    if (p->bitmap) cudaFree(p->bitmap);
    p->bitmap = nullptr;
    p->bitmap_words = 0;
    if ((e = cudaMalloc(&p->bitmap, words * 4))) return cuda_fail(e, "cudaMalloc(validate bitmap)");
    p->bitmap_words = words;
  }
  if (!p->err_dev) {
    if ((e = cudaMalloc(&p->err_dev, 4))) return cuda_fail(e, "cudaMalloc(validate flag)");
    if ((e = cudaMallocHost(&p->err_host, 4))) return cuda_fail(e, "cudaMallocHost(validate flag)");
  }
  if ((e = cudaMemsetAsync(p->bitmap, 0, words * 4, s))) return cuda_fail(e, "cudaMemsetAsync");
  if ((e = cudaMemsetAsync(p->err_dev, 0, 4, s))) return cuda_fail(e, "cudaMemsetAsync");
  for (const Batch& b : plan.batches) {
    strata::ValidateParams v;
    memset(&v, 0, sizeof v);
    v.C = p->d.chunk_tokens;
    v.P = p->d.page_size;
    v.ntok = b.ntok;
    v.dir = dir;
    v.num_pages = p->d.num_pages;
    v.num_chunks = p->d.num_chunks;
    v.chunks_len = x->host_chunks_len;
    v.pages_len = x->dev_pages_len;
    v.host_chunks = x->host_chunks;
    v.dev_pages = x->dev_pages;
    v.bitmap = p->bitmap;
    v.err = p->err_dev;
    fill_table(x, plan, b, v.rt);
    if ((e = strata::launch_validate(v, s))) return cuda_fail(e, "validate kernel launch");
    ++p->counters.kernel_launches;
  }
  if ((e = cudaMemcpyAsync(p->err_host, p->err_dev, 4, cudaMemcpyDeviceToHost, s))) return cuda_fail(e, "cudaMemcpyAsync");
  if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "cudaStreamSynchronize(validate)");
  if (*p->err_host & 1) return fail(STRATA_ERR_INDEX_RANGE, "a chunk/page index is outside the pool or its list");
  if (*p->err_host & 2) return fail(STRATA_ERR_DUPLICATE, "two tokens target the same destination slot");
  return STRATA_OK;
}

// STRATA_VALIDATE for STRATA_ENGINE_DMA: the copy engines follow the host mirror of the chunk list
// while the scatter kernel (and every other engine) follows the device list, so the two must agree
// over every entry the call reads.
static int check_host_mirror(strata_pool* p, const strata_xfer* x, const Plan& plan, cudaStream_t s) {
  const int64_t C = p->d.chunk_tokens;
  int64_t lo = INT64_MAX, hi = 0;
  for (int32_t r : plan.reqs) {
    const int64_t oc = x->chunk_offset ? x->chunk_offset[r] : 0;
    lo = std::min<int64_t>(lo, x->chunk_start[r]);
    hi = std::max<int64_t>(hi, x->chunk_start[r] + (oc + x->num_tokens[r] + C - 1) / C);
  }
  if (hi <= lo) return STRATA_OK;
  std::vector<int32_t> dev(size_t(hi - lo));
  cudaError_t e = cudaMemcpyAsync(dev.data(), x->host_chunks + lo, dev.size() * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(host_chunks check)");
  for (int32_t r : plan.reqs) {
    const int64_t oc = x->chunk_offset ? x->chunk_offset[r] : 0;
    const int64_t a = x->chunk_start[r], b = a + (oc + x->num_tokens[r] + C - 1) / C;
    for (int64_t i = a; i < b; ++i)
      if (x->host_chunks_host[i] != dev[size_t(i - lo)])
        return fail(STRATA_ERR_INVALID_ARG, "host_chunks_host[%lld] = %d but host_chunks[%lld] = %d on the device",
                    (long long)i, x->host_chunks_host[i], (long long)i, dev[size_t(i - lo)]);
  }
  return STRATA_OK;
}

static bool env_validate() {
  const char* v = getenv("STRATA_VALIDATE");
  return v && *v && strcmp(v, "0") != 0;
}

static void count_op(strata_pool* p, const Plan& plan, const strata_xfer* x, int engine) {
  p->counters.operations += 1;
  p->counters.bytes += p->nkv * plan.total_tokens * p->tok_bytes * (x->layer_end - x->layer_begin);
  p->counters.last_engine = engine;
}

// Env knob (A/B runs): integer value of `name`, or `def`.
static int env_int(const char* name, int def) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : def;
}

// The ring engine needs whole host token rows (token-major tiers, or one head per GPU) in 16-byte
// units; a head-major tier with several heads per GPU has no whole rows.  Loads of narrow rows (R29,
// 8- or 4-byte granularity) take it too when a piece's host rows are one run, the device rows are
// head-contiguous and the tier's mapping spans whole 16-byte units (the producer reads the enclosing
// aligned span of each run).
static bool ring_supported(const strata_pool* p, int dir) {
  if (!p->host_row_contig()) return false;
  if (p->gran == 16) return true;
  // (8-byte words only: 4-byte-word rows scatter at 34.8 GB/s on the ring vs 46.6 on the narrow LDG
  // kernel, 100-byte rows, profiles/r02/probe1/narrow.jsonl)
  return dir == 0 && p->gran == 8 && p->host_tok_stride == p->tok_bytes &&
         (p->head_stride == p->head_bytes || p->d.num_heads == 1) &&
         reinterpret_cast<uintptr_t>(p->host_dev) % 16 == 0 && p->host_bytes % 16 == 0;
}

// The ring's per-CTA geometry, a pure function of sizes (exported for tests: strata_test_ring_geometry).
// R rows per piece (a piece = one host run, <= stage_target bytes, <= C tokens, <= kRingMaxRows);
// S stages holding inflight / ctas host bytes (2..kRingMaxStages, within the shared-memory budget);
// W device-side warps, a divisor of S (stage s belongs to warp s % W, ring.cu).
struct RingGeom {
  int R = 0, S = 0, W = 0, sb = 0;
};
static bool ring_geometry(int tok, int C, int gran, int budget, int64_t inflight, int ctas, int W, int target,
                          RingGeom& g) {
  W = std::max(1, std::min(kRingMaxWarps, W));
  int R = std::min<int>(C, std::max(1, target / tok));
  R = std::min(R, kRingMaxRows);
  // narrow rows: the stage holds the run's enclosing 16-byte-aligned span (up to 30 bytes more)
  const int sb = (R * tok + (gran < 16 ? 32 : 0) + 127) / 128 * 128;
  const int64_t per_cta = inflight / std::max(1, ctas);
  int S = static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(kRingMaxStages, per_cta / sb)));
  S = std::min(S, env_int("STRATA_RING_STAGES", kRingMaxStages));
  while (S >= 2 && ring_header_bytes() + S * sb > budget) --S;
  if (S < 2) return false;
  // W must divide S: take the largest S' <= S with a divisor d <= W of at least half of min(W, S')
  // and run d warps (S = 13, W = 8 would otherwise leave ONE scatter warp: 16.4 GB/s instead of 51,
  // profiles/r02/sweep70/)
  int Wd = 1;
  for (int s2 = S; s2 >= 2; --s2) {
    int d = 1;
    for (int c = 1; c <= std::min(W, s2); ++c)
      if (s2 % c == 0) d = c;
    if (2 * d >= std::min(W, s2)) {
      S = s2;
      Wd = d;
      break;
    }
  }
  g.R = R;
  g.S = S;
  g.W = Wd;
  g.sb = sb;
  return true;
}

// Ring geometry for this pool and direction (rows per piece, stages, scatter warps); false when a
// 2-stage ring of one-row pieces does not fit in shared memory.
static bool plan_ring(const strata_pool* p, const strata_xfer* x, int dir, const XferParams& xp, int ctas,
                      RingParams& rp) {
  const int tok = static_cast<int>(p->tok_bytes);
  const int W = x->threads ? x->threads / 32 - 1
                           : dir == 0 ? env_int("STRATA_RING_WARPS", kDefaultRingWarps)
                                      : env_int("STRATA_RING_GATHER_WARPS", kDefaultRingGatherWarps);
  const int target = std::max(1, env_int("STRATA_RING_STAGE_KB", kDefaultRingStageKB)) << 10;
  int budget = p->tma_smem;
  const int cap_kb = env_int("STRATA_RING_SMEM_KB", 0);
  if (cap_kb > 0) budget = std::min(budget, cap_kb << 10);
  // host bytes kept in flight (the rings' capacity) over all CTAs: the caller's bound
  // (strata_xfer.inflight_kib), else the default — the knee of the throughput / interference
  // frontier: more than the link needs only queues requests, and queued host reads
  // are what slows co-running HBM-bound work
  const int64_t total = x->inflight_kib > 0 ? x->inflight_kib
                        : env_int("STRATA_RING_INFLIGHT_KB", tok < kRingShortRowBytes ? kDefaultRingInflightShortKB
                                                                                     : kDefaultRingInflightKB);
  RingGeom geo;
  if (!ring_geometry(tok, p->d.chunk_tokens, p->gran, budget, total << 10, ctas, W, target, geo)) return false;
  const int R = geo.R, S = geo.S, sb = geo.sb;
  std::memset(&rp, 0, offsetof(RingParams, pair_end));
  rp.x = xp;
  rp.rows = R;
  rp.stages = S;
  rp.stage_bytes = sb;
  rp.pps = (p->d.chunk_tokens + R - 1) / R;
  rp.warps = geo.W;
  rp.host_run = p->host_tok_stride == p->tok_bytes;
  rp.bulk_store = dir == 0 && env_int("STRATA_RING_BULK_STORE", 0) != 0;
  rp.debug = env_int("STRATA_RING_DEBUG", 0);
  {
    // the offload's share of the link while loads run, split over its CTAs: ps per byte per CTA
    const int share = dir == 1 ? env_int("STRATA_OFFLOAD_SHARE_GBS", kDefaultOffloadShareGBs) : 0;
    rp.pace_ps_per_byte = share > 0 ? static_cast<int32_t>(1000LL * std::max(1, ctas) / share) : 0;
  }
  if (env_int("STRATA_RING_EXCLUSIVE", kDefaultRingExclusive)) rp.smem_reserve = p->tma_smem;
  if (p->gran < 16) rp.word_magic = div_magic(tok / p->gran, R * (tok / p->gran) + 32 * 4 * 32);
  for (int l = 0; l < p->d.num_layers; ++l) {
    rp.kb[l] = static_cast<char*>(p->k[l]);
    rp.vb[l] = static_cast<char*>(p->v[l]);
  }
  return true;
}

// Request table + piece count of one launch; false if the pieces overflow int32.
static bool ring_batch(const strata_pool* p, const strata_xfer* x, const Plan& plan, const Batch& b, RingParams& rp) {
  fill_table(x, plan, b, rp.x.rt);
  rp.x.ntok = b.ntok;
  const int64_t C = p->d.chunk_tokens;
  int64_t acc = 0;
  for (int32_t k = 0; k < b.count; ++k) {
    const int32_t r = plan.reqs[b.first + k];
    const int64_t oc = x->chunk_offset ? x->chunk_offset[r] : 0;
    acc += (oc + x->num_tokens[r] + C - 1) / C;
    rp.pair_end[k] = static_cast<int32_t>(std::min<int64_t>(acc, INT32_MAX));
  }
  const int64_t pieces = acc * p->nkv * rp.pps;
  if (pieces > INT32_MAX) return false;
  rp.npieces = static_cast<int32_t>(pieces);
  return true;
}

// The op slot's previous fused operation (possibly on another stream) still owns the slot's arrival
// counters and flags until it completes: order the new fused launch after it (its last-layer event,
// recorded on its own stream after its kernel).  Almost always already complete, so cheap.
static cudaError_t order_after_slot(strata_pool* p, const strata_pool::Op& prev, int slot, cudaStream_t s) {
  if (!prev.fused || !prev.ticket) return cudaSuccess;
  return cudaStreamWaitEvent(s, p->events[size_t(slot) * (p->d.num_layers + 1) + prev.l1], 0);
}

// After a fused launch: layer l < l1-1 completes when its device flag reaches the epoch; the side
// stream of the slot turns each flag into the layer's event.  The last layer completes with the
// kernel: its event goes on the caller's stream, sparing the op's completion the flag-poll latency.
static cudaError_t fused_events(strata_pool* p, int slot, const strata_xfer* x, uint32_t* flags, uint32_t epoch,
                                cudaStream_t s) {
  const int L = p->d.num_layers;
  cudaError_t e = cudaEventRecord(p->events[size_t(slot) * (L + 1) + x->layer_end], s);
  if (e != cudaSuccess) return e;
  cudaStream_t side = p->side[slot];
  for (int32_t l = x->layer_begin; l + 1 < x->layer_end; ++l) {
    if (g_wait_value32(reinterpret_cast<CUstream>(side), reinterpret_cast<CUdeviceptr>(flags + l), epoch,
                       CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return cudaErrorUnknown;
    if ((e = cudaEventRecord(p->events[size_t(slot) * (L + 1) + 1 + l], side))) return e;
  }
  return cudaSuccess;
}

cudaError_t op_record(strata_pool* p, int slot, int idx, cudaStream_t s) {
  cudaError_t e = cudaEventRecord(p->events[size_t(slot) * (p->d.num_layers + 1) + idx], s);
  if (e != cudaSuccess || !p->ops[slot].captured) return e;
  auto it = p->captured_ops.find(p->ops[slot].ticket);
  if (it == p->captured_ops.end()) return cudaErrorInvalidValue;
  return cudaEventRecordWithFlags(it->second.ev[size_t(idx)], s, cudaEventRecordExternal);
}

// A captured operation gets its own events (external nodes of the graph, signalled by every replay).
static cudaError_t begin_captured(strata_pool* p, uint64_t t, const strata_xfer* x) {
  strata_pool::CapturedOp op;
  op.l0 = x->layer_begin;
  op.l1 = x->layer_end;
  op.ev.assign(size_t(p->d.num_layers) + 1, nullptr);
  for (auto& ev : op.ev) {
    cudaError_t e = cudaEventCreate(&ev);
    if (e != cudaSuccess) {
      for (auto& v : op.ev)
        if (v) cudaEventDestroy(v);
      return e;
    }
  }
  p->captured_ops[t] = std::move(op);
  return cudaSuccess;
}

static void drop_captured(strata_pool* p, uint64_t t) {
  auto it = p->captured_ops.find(t);
  if (it == p->captured_ops.end()) return;
  for (auto& v : it->second.ev)
    if (v) cudaEventDestroy(v);
  p->captured_ops.erase(it);
}

int transfer(strata_pool_t p, const strata_xfer* x, cudaStream_t s, uint64_t* ticket, int dir) {
  if (!p) return fail(STRATA_ERR_INVALID_ARG, "pool is NULL");
  Plan plan;
  int rc = check_xfer(p, x, plan);
  if (rc) return rc;
  DeviceGuard dg(p->d.device);
  if (dg.err) return cuda_fail(dg.err, "cudaSetDevice");
  const bool validate = plan.total_tokens > 0 && ((p->d.flags & STRATA_VALIDATE) || env_validate());
  if (validate) {
    rc = run_validate(p, x, plan, dir, s);
    if (rc) return rc;
  }

  strata::XferParams xp;
  memset(&xp, 0, offsetof(strata::XferParams, rt));
  xp.C = p->d.chunk_tokens;
  xp.P = p->d.page_size;
  xp.H = p->d.num_heads;
  xp.tok_bytes = static_cast<int32_t>(p->tok_bytes);
  xp.head_bytes = static_cast<int32_t>(p->head_bytes);
  xp.vpt = xp.tok_bytes / 16;
  xp.vpt_shift = ilog2_exact(xp.vpt);
  xp.vpt_magic = xp.vpt_shift < 0 ? div_magic(xp.vpt, 32 * xp.vpt) : 0;
  xp.vph = xp.head_bytes / 16;
  xp.vph_shift = ilog2_exact(xp.vph);
  xp.c_shift = ilog2_exact(xp.C);
  xp.p_shift = ilog2_exact(xp.P);
  xp.chunk_bytes = p->chunk_bytes;
  xp.kv_off = p->host_kv_off;
  xp.host_tok_stride = p->host_tok_stride;
  xp.host_head_off = p->host_head_off;
  xp.host_head_stride = p->host_head_stride;
  xp.page_stride = p->page_stride;
  xp.token_stride = p->token_stride;
  xp.head_stride = p->head_stride;
  xp.host = p->host_dev;
  xp.host_chunks = x->host_chunks;
  xp.dev_pages = x->dev_pages;
  xp.nkv = p->nkv;
  xp.gran = p->gran;
  xp.wpr = static_cast<int32_t>(p->tok_bytes / p->gran);
  xp.wph = static_cast<int32_t>(p->head_bytes / p->gran);
  xp.wpr_magic = (xp.wpr & (xp.wpr - 1)) ? div_magic(xp.wpr, 32 * xp.wpr + 32 * 4) : 0;
  xp.wph_magic = (xp.wph & (xp.wph - 1)) ? div_magic(xp.wph, xp.wpr) : 0;

  // Engine.  The default is a hand-written zero-copy kernel reading / writing the host tier through
  // its UVA mapping.  Loads of 16-byte-granular rows of >= kSmallOpBytes take the LDG
  // engine at the paper's configuration (2 CTAs x 1024 threads, one fused launch): it moves
  // the ring's ~51 GB/s on Llama-8B and slows co-running decode attention less (+7 vs +9 %, DESIGN.md
  // §6.1, NEXT-1).  Everything else — offloads, small (latency-bound) loads, narrow rows of 8- / 4-byte
  // granularity — takes the ring engine where the tier has whole host rows in 16-byte units, else
  // LDG (narrow offloads, head-major tiers with several heads per GPU).  The copy-engine path
  // (STRATA_ENGINE_DMA) runs only when a caller asks for it.
  int engine = x->engine;
  if (engine == STRATA_ENGINE_DEFAULT) {
    const int64_t op_bytes = int64_t(p->nkv) * plan.total_tokens * p->tok_bytes * (x->layer_end - x->layer_begin);
    engine = dir == 0 && p->gran == 16 && op_bytes >= kSmallOpBytes ? STRATA_ENGINE_LDG
             : ring_supported(p, dir)                                 ? STRATA_ENGINE_TMA
                                                                      : STRATA_ENGINE_LDG;
  }
  // the copy engines need long host runs: a token-major tier read in a head slice (Ht > H) has
  // only H*D*e bytes per token contiguous, so its DMA requests run on the LDG engine instead
  if (engine == STRATA_ENGINE_DMA && !dma_runs_ok(p)) engine = STRATA_ENGINE_LDG;
  if (engine == STRATA_ENGINE_DMA) {
    if (!x->host_chunks_host && plan.total_tokens > 0)
      return fail(STRATA_ERR_INVALID_ARG, "STRATA_ENGINE_DMA needs xfer.host_chunks_host");
    if (validate && (rc = check_host_mirror(p, x, plan, s))) return rc;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(s, &cap);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamIsCapturing");
    const uint64_t t = p->next_ticket++;
    const int slot = static_cast<int>(t % kEventRing);
    p->ops[slot] = {t, x->layer_begin, x->layer_end};
    p->ops[slot].captured = cap != cudaStreamCaptureStatusNone;
    if (p->ops[slot].captured && (e = begin_captured(p, t, x)) != cudaSuccess) {
      p->ops[slot].ticket = 0;
      return cuda_fail(e, "cudaEventCreate");
    }
    e = op_record(p, slot, 0, s);
    if (e != cudaSuccess) {
      p->ops[slot].ticket = 0;   // a failed operation has no valid events
      drop_captured(p, t);
      return cuda_fail(e, "cudaEventRecord");
    }
    rc = transfer_dma(p, x, plan, xp, s, dir, slot);
    if (rc) {
      p->ops[slot].ticket = 0;
      drop_captured(p, t);
      return rc;
    }
    count_op(p, plan, x, engine);
    if (ticket) *ticket = t;
    return STRATA_OK;
  }
  RingParams rp;
  int ctas = x->num_ctas;
  if (engine == STRATA_ENGINE_TMA) {
    // load rows below kRingSmallRowBytes take twice the quota (256-byte rows: 43.8 GB/s from 2 CTAs)
    const int c = ctas ? ctas : dir == 0 ? kDefaultCtasRingLoad * (p->tok_bytes < kRingSmallRowBytes ? 2 : 1)
                                         : kDefaultCtasRingOffload;
    if (!(ring_supported(p, dir) && plan_ring(p, x, dir, xp, c, rp))) engine = STRATA_ENGINE_LDG;
    else ctas = c;
  }
  // the bulk rings stage whole host rows in 16-byte units: a head-major tier with > 1 head per GPU
  // has no whole rows, a pool whose rows / strides are not 16-byte multiples (R29) no 16-byte units
  if (engine == STRATA_ENGINE_TMA_BULK && (!p->host_row_contig() || p->gran < 16)) engine = STRATA_ENGINE_LDG;
  if (engine == STRATA_ENGINE_TMA_BULK) {
    const int rows = std::max(1, std::min(32, kTmaStageTarget / xp.tok_bytes));
    const int sb = rows * xp.tok_bytes;
    const int budget = p->tma_smem - strata::tma_header_bytes(strata::kTmaMaxStages);
    const int stages = std::min(strata::kTmaMaxStages, budget / sb);
    if (stages < 2) {
      engine = STRATA_ENGINE_LDG;  // token rows too large for a 2-stage shared-memory ring
    } else {
      xp.tma_rows = rows;
      xp.tma_stage_bytes = sb;
      xp.tma_stages = stages;
    }
  }
  const int threads = x->threads ? x->threads : kDefaultThreadsLdg;
  const int unroll = threads > 512 ? 4 : kDefaultUnroll;   // U=8 is compiled for <= 512 threads
  // lane t fetches row t; the warp then streams the 32 rows (amortised index math)
  xp.rows_per_group = 32;
  if (!ctas) {
    if (engine == STRATA_ENGINE_TMA_BULK) ctas = kDefaultCtasTma;
    else if (p->gran < 16) ctas = kDefaultCtasNarrow;
    else ctas = dir == 0 ? kDefaultCtasLdg : kDefaultCtasLdgOffload;
    // small token rows shrink a bulk stage (<= 32 rows); keep ~64 KiB per stage-CTA in flight by
    // spreading over more CTAs (70B TP=8: 256 B rows -> 8 KiB stages -> 16 CTAs)
    if (engine == STRATA_ENGINE_TMA_BULK && xp.tma_stage_bytes > 0)
      ctas = std::min(16, ctas * std::max(1, (2 * kTmaStageTarget) / xp.tma_stage_bytes));
  }

  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(s, &cap);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamIsCapturing");
  const uint64_t t = p->next_ticket++;
  const int slot = static_cast<int>(t % kEventRing);
  const strata_pool::Op prev = p->ops[slot];
  p->ops[slot] = {t, x->layer_begin, x->layer_end};
  p->ops[slot].captured = cap != cudaStreamCaptureStatusNone;
  const int L = p->d.num_layers;
  // a failed operation keeps no ticket: its ring slot must not hand out stale events
  auto op_fail = [&](cudaError_t err, const char* what) {
    p->ops[slot].ticket = 0;
    drop_captured(p, t);
    return cuda_fail(err, what);
  };
  if (p->ops[slot].captured && (e = begin_captured(p, t, x)) != cudaSuccess) return op_fail(e, "cudaEventCreate");
  e = op_record(p, slot, 0, s);  // operation start
  if (e != cudaSuccess) return op_fail(e, "cudaEventRecord");
  // One launch for all layers when the call is one request table and not being captured (stream
  // memory operations are not captured here); layer events come from the device flags.
  const bool can_fuse = plan.batches.size() == 1 && x->layer_end - x->layer_begin > 1 && L <= kMaxFusedLayers &&
                        fused_mode() && cap == cudaStreamCaptureStatusNone && ensure_fused(p);
  uint32_t* counters = p->fused_sync + size_t(slot) * 3 * L;
  if (engine == STRATA_ENGINE_TMA) {
    if (can_fuse) {
      if (!ring_batch(p, x, plan, plan.batches[0], rp)) return op_fail(cudaErrorInvalidValue, "ring piece count");
      int c = std::max(1, std::min(ctas, rp.npieces));
      // a small operation is latency-bound (one host round trip per piece in flight): spread its pieces
      // over up to kSmallOpCtas CTAs so they are all in flight at once; it ends within microseconds,
      // so the SM quota it briefly exceeds costs co-running work little
      const int64_t op_bytes = int64_t(p->nkv) * plan.total_tokens * p->tok_bytes * (x->layer_end - x->layer_begin);
      if (!x->num_ctas && op_bytes < kSmallOpBytes) {
        c = std::max(c, std::min(kSmallOpCtas, rp.npieces));
        // ... and every piece of the operation gets a stage: re-plan the rings for c CTAs with the
        // whole operation in flight (unless the caller bounded it)
        if (!x->inflight_kib) {
          strata_xfer xa = *x;
          const int64_t all = int64_t(rp.npieces) * (x->layer_end - x->layer_begin) * rp.stage_bytes;
          xa.inflight_kib = static_cast<int32_t>(std::min<int64_t>(INT32_MAX, (all + 1023) >> 10));
          if (!plan_ring(p, &xa, dir, xp, c, rp) || !ring_batch(p, x, plan, plan.batches[0], rp))
            return op_fail(cudaErrorInvalidValue, "ring plan");
        }
      }
      rp.l0 = x->layer_begin;
      rp.l1 = x->layer_end;
      rp.epoch = static_cast<uint32_t>(t);
      rp.arrivals = dir == 0 ? c * rp.warps : c;
      rp.counters = counters;
      rp.flags = counters + L;
      if ((e = order_after_slot(p, prev, slot, s))) return op_fail(e, "cudaStreamWaitEvent(slot)");
      if ((e = strata::launch_ring(rp, dir, c, s))) return op_fail(e, "ring kernel launch");
      p->ops[slot].fused = true;
      ++p->counters.kernel_launches;
      if ((e = fused_events(p, slot, x, rp.flags, rp.epoch, s))) return op_fail(e, "layer events");
      count_op(p, plan, x, engine);
      if (ticket) *ticket = t;
      return STRATA_OK;
    }
    // per layer (graph capture, several request tables, one layer): one launch per layer and table
    for (int32_t l = x->layer_begin; l < x->layer_end; ++l) {
      for (const Batch& b : plan.batches) {
        if (!ring_batch(p, x, plan, b, rp)) return op_fail(cudaErrorInvalidValue, "ring piece count");
        const int c = std::max(1, std::min(ctas, rp.npieces));
        rp.l0 = l;
        rp.l1 = l + 1;
        if ((e = strata::launch_ring(rp, dir, c, s))) return op_fail(e, "ring kernel launch");
        ++p->counters.kernel_launches;
      }
      if ((e = op_record(p, slot, 1 + l, s))) return op_fail(e, "cudaEventRecord");
    }
    count_op(p, plan, x, engine);
    if (ticket) *ticket = t;
    return STRATA_OK;
  }
  // LDG: one launch for all layers from 2 CTAs (measured, profiles/r01/fused_ab_*.jsonl: +2 % at
  // 2 CTAs, +0.5 % at 4, but -3..-7 % with a single CTA, so 1-CTA grids keep per-layer launches)
  const int64_t fgroups = plan.batches.empty() ? 0
                              : (int64_t(p->nkv) * plan.batches[0].ntok + xp.rows_per_group - 1) / xp.rows_per_group;
  const int fctas = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctas, (fgroups * 32 + threads - 1) / threads)));
  if (engine == STRATA_ENGINE_LDG && p->gran == 16 && can_fuse && (fctas >= 2 || fused_mode() == 2)) {
    const Batch& b = plan.batches[0];
    FusedParams fp;
    std::memset(&fp, 0, sizeof fp);
    fp.x = xp;
    fp.x.ntok = b.ntok;
    fill_table(x, plan, b, fp.x.rt);
    fp.l0 = x->layer_begin;
    fp.l1 = x->layer_end;
    fp.epoch = static_cast<uint32_t>(t);
    fp.total_warps = fctas * threads / 32;
    fp.counters = counters;
    fp.flags = counters + L;
    fp.loads_active = dir == 0 ? p->loads_active : nullptr;
    fp.next = counters + 2 * L;
    fp.quota = dir == 0 ? p->quota : nullptr;   // set once the caller has used strata_set_load_quota
    for (int l = 0; l < L; ++l) {
      fp.kb[l] = static_cast<char*>(p->k[l]);
      fp.vb[l] = static_cast<char*>(p->v[l]);
    }
    if ((e = order_after_slot(p, prev, slot, s))) return op_fail(e, "cudaStreamWaitEvent(slot)");
    if ((e = strata::launch_ldg_fused(fp, dir, fctas, threads, s))) return op_fail(e, "fused transfer kernel launch");
    p->ops[slot].fused = true;
    ++p->counters.kernel_launches;
    if ((e = fused_events(p, slot, x, fp.flags, fp.epoch, s))) return op_fail(e, "layer events");
    count_op(p, plan, x, engine);
    if (ticket) *ticket = t;
    return STRATA_OK;
  }
  for (int32_t l = x->layer_begin; l < x->layer_end; ++l) {
    xp.kbase = static_cast<char*>(p->k[l]);
    xp.vbase = static_cast<char*>(p->v[l]);
    xp.layer_off = int64_t(l) * p->nkv * xp.kv_off;
    for (const Batch& b : plan.batches) {
      xp.ntok = b.ntok;
      fill_table(x, plan, b, xp.rt);
      const int64_t rows = int64_t(p->nkv) * b.ntok;
      int c = ctas;
      if (engine == STRATA_ENGINE_TMA_BULK) {
        const int64_t pieces = (rows + xp.tma_rows - 1) / xp.tma_rows;
        if (pieces < c) c = static_cast<int>(pieces);
        e = strata::launch_tma(xp, dir, c, s);
      } else {
        const int64_t groups = (rows + xp.rows_per_group - 1) / xp.rows_per_group;
        const int64_t need = (groups * 32 + threads - 1) / threads;
        if (need < c) c = static_cast<int>(need);
        e = strata::launch_ldg(xp, dir, c, threads, unroll, s);
      }
      if (e != cudaSuccess) return op_fail(e, "transfer kernel launch");
      ++p->counters.kernel_launches;
    }
    e = op_record(p, slot, 1 + l, s);
    if (e != cudaSuccess) return op_fail(e, "cudaEventRecord");
  }
  count_op(p, plan, x, engine);
  if (ticket) *ticket = t;
  return STRATA_OK;
}


}  // namespace strata

extern "C" int strata_test_ring_geometry(int32_t tok_bytes, int32_t chunk_tokens, int32_t gran, int32_t smem_budget,
                                         int64_t inflight_bytes, int32_t ctas, int32_t warps, int32_t stage_target,
                                         int32_t out[4]) {
  if (!out || tok_bytes <= 0 || chunk_tokens <= 0 || gran <= 0 || smem_budget <= 0 || inflight_bytes <= 0 ||
      ctas <= 0 || warps <= 0 || stage_target <= 0)
    return STRATA_ERR_INVALID_ARG;
  strata::RingGeom g;
  if (!strata::ring_geometry(tok_bytes, chunk_tokens, gran, smem_budget, inflight_bytes, ctas, warps, stage_target, g))
    return STRATA_ERR_UNSUPPORTED;
  out[0] = g.R;
  out[1] = g.S;
  out[2] = g.W;
  out[3] = g.sb;
  return STRATA_OK;
}
