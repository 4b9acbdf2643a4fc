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

namespace strata {

namespace {

using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32Fn g_wait_value32 = nullptr;

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

// Lazily: per op slot 2*L device words (arrival counters, layer flags) and a side stream; the
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
  const size_t words = size_t(kEventRing) * 2 * p->d.num_layers;
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
  uint32_t* flag = p->fused_sync + size_t(slot) * 2 * L + L + layer;
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

static bool env_validate() {
  const char* v = getenv("STRATA_VALIDATE");
  return v && *v && strcmp(v, "0") != 0;
}

static void count_op(strata_pool* p, const Plan& plan, const strata_xfer* x, int engine) {
  p->counters.operations += 1;
  p->counters.bytes += p->nkv * plan.total_tokens * p->tok_bytes * (x->layer_end - x->layer_begin);
  p->counters.last_engine = engine;
}

int transfer(strata_pool_t p, const strata_xfer* x, cudaStream_t s, uint64_t* ticket, int dir) {
  if (!p) return fail(STRATA_ERR_INVALID_ARG, "pool is NULL");
  Plan plan;
  int rc = check_xfer(p, x, plan);
  if (rc) return rc;
  DeviceGuard dg(p->d.device);
  if (dg.err) return cuda_fail(dg.err, "cudaSetDevice");
  cudaError_t e = cudaGetLastError();  // surface an earlier asynchronous fault
  if (e != cudaSuccess) return cuda_fail(e, "earlier CUDA error");
  if (plan.total_tokens > 0 && ((p->d.flags & STRATA_VALIDATE) || env_validate())) {
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

  int engine = x->engine;
  if (engine == STRATA_ENGINE_DEFAULT) {
    // Measured on B200: the copy-engine gather + SM scatter moves 98 % of the link
    // for layer-sized transfers; below a few MiB per layer its per-piece submission latency is not
    // amortised and the zero-copy LDG kernel wins.  Without a host mirror of the chunk list only
    // the kernel engines can run.
    // (Offloads group layers into >= 128 KiB runs inside the DMA engine, see transfer_dma.)
    // Loads copy one chunk-layer per run (per head for head-major tiers); below ~24 KiB a run the
    // copy engines fall behind the SM path (72-byte rows at C = 64: 9 KiB runs, DMA 24 vs LDG 33.5
    // GB/s; tools/narrow_probe.py).  Offloads group layers into >= 128 KiB runs anyway.
    const int64_t layer_bytes = p->nkv * plan.total_tokens * p->tok_bytes;
    const int64_t run = int64_t(p->nkv) * p->d.chunk_tokens * (p->head_major ? p->head_bytes : p->tok_bytes);
    const bool dma = x->host_chunks_host && layer_bytes >= kDmaMinLayerBytes && dma_runs_ok(p) &&
                     (dir == 1 || run >= kDmaMinLoadRun);
    engine = dma ? STRATA_ENGINE_DMA : STRATA_ENGINE_LDG;
  }
  // the copy engines need long host runs: a token-major tier read in a head slice (Ht > H) has
  // only H*D*e bytes per token contiguous, so its DMA requests run on the LDG engine instead
  if (engine == STRATA_ENGINE_DMA && !dma_runs_ok(p)) engine = STRATA_ENGINE_LDG;
  if (engine == STRATA_ENGINE_DMA) {
    if (!x->host_chunks_host && plan.total_tokens > 0)
      return fail(STRATA_ERR_INVALID_ARG, "STRATA_ENGINE_DMA needs xfer.host_chunks_host");
    const uint64_t t = p->next_ticket++;
    const int slot = static_cast<int>(t % kEventRing);
    p->ops[slot] = {t, x->layer_begin, x->layer_end};
    e = cudaEventRecord(p->events[size_t(slot) * (p->d.num_layers + 1)], s);
    if (e != cudaSuccess) {
      p->ops[slot].ticket = 0;   // a failed operation has no valid events
      return cuda_fail(e, "cudaEventRecord");
    }
    rc = transfer_dma(p, x, plan, xp, s, dir, slot);
    if (rc) {
      p->ops[slot].ticket = 0;
      return rc;
    }
    count_op(p, plan, x, engine);
    if (ticket) *ticket = t;
    return STRATA_OK;
  }
  // the TMA rings stage whole host rows in 16-byte units: a head-major tier with > 1 head per GPU
  // has no whole rows, a pool whose rows / strides are not 16-byte multiples (R29) no 16-byte units
  if ((engine == STRATA_ENGINE_TMA || engine == STRATA_ENGINE_TMA_BULK) && (!p->host_row_contig() || p->gran < 16))
    engine = STRATA_ENGINE_LDG;
  const bool tma = engine == STRATA_ENGINE_TMA || engine == STRATA_ENGINE_TMA_BULK;
  // TMA engine geometry: rows per stage (<= 32 lanes), stage bytes, depth
  if (tma) {
    // the warp-specialised ring is producer-bound per stage: larger stages (64 KiB) amortise it
    const int target = engine == STRATA_ENGINE_TMA ? 2 * kTmaStageTarget : kTmaStageTarget;
    int rows = std::max(1, std::min(32, target / xp.tok_bytes));
    const int sb = rows * xp.tok_bytes;
    const int budget = p->tma_smem - strata::tma_header_bytes(strata::kTmaMaxStages);
    int stages = std::min(strata::kTmaMaxStages, budget / sb);
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
  // lane t fetches row t; the warp then streams the 32 rows (amortised index math).  The narrow
  // kernel (R29) takes one row per warp, so its grid is sized per row.
  xp.rows_per_group = 32;
  int ctas = x->num_ctas ? x->num_ctas
             : engine != STRATA_ENGINE_LDG ? kDefaultCtasTma
             : p->gran < 16                ? kDefaultCtasNarrow
             : dir == 0                    ? kDefaultCtasLdg
                                           : kDefaultCtasLdgOffload;
  // small token rows shrink a TMA stage (<= 32 rows); keep ~64 KiB per stage-CTA in flight by
  // spreading over more CTAs (70B TP=8: 256 B rows -> 8 KiB stages -> 16 CTAs)
  if (!x->num_ctas && engine != STRATA_ENGINE_LDG && xp.tma_stage_bytes > 0)
    ctas = std::min(16, ctas * std::max(1, (2 * kTmaStageTarget) / xp.tma_stage_bytes));

  const uint64_t t = p->next_ticket++;
  const int slot = static_cast<int>(t % kEventRing);
  p->ops[slot] = {t, x->layer_begin, x->layer_end};
  const int L = p->d.num_layers;
  // a failed operation keeps no ticket: its ring slot must not hand out stale events
  auto op_fail = [&](cudaError_t err, const char* what) {
    p->ops[slot].ticket = 0;
    return cuda_fail(err, what);
  };
  e = cudaEventRecord(p->events[size_t(slot) * (L + 1)], s);  // operation start
  if (e != cudaSuccess) return op_fail(e, "cudaEventRecord");
  // One launch for all layers when the call is one request table and not being captured (stream
  // memory operations are not captured here); layer events come from the device flags.  Measured
  // (profiles/r01/fused_ab_*.jsonl): +2 % at the default 2 CTAs (51.2 GB/s, 99.4 % of the SM
  // zero-copy ceiling), +0.5 % at 4, but -3..-7 % with a single CTA, so 1-CTA grids keep the
  // per-layer launches.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const int64_t fgroups = plan.batches.empty() ? 0
                              : (int64_t(p->nkv) * plan.batches[0].ntok + xp.rows_per_group - 1) / xp.rows_per_group;
  const int fctas = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctas, (fgroups * 32 + threads - 1) / threads)));
  if (engine == STRATA_ENGINE_LDG && p->gran == 16 && plan.batches.size() == 1 && x->layer_end - x->layer_begin > 1 &&
      (fctas >= 2 || fused_mode() == 2) && L <= kMaxFusedLayers && fused_mode() && cudaStreamIsCapturing(s, &cap) == cudaSuccess &&
      cap == cudaStreamCaptureStatusNone && ensure_fused(p)) {
    const Batch& b = plan.batches[0];
    FusedParams fp;
    std::memset(&fp, 0, sizeof fp);
    fp.x = xp;
    fp.x.ntok = b.ntok;
    fill_table(x, plan, b, fp.x.rt);
    const int c = fctas;
    fp.l0 = x->layer_begin;
    fp.l1 = x->layer_end;
    fp.epoch = static_cast<uint32_t>(t);
    fp.total_warps = c * threads / 32;
    fp.counters = p->fused_sync + size_t(slot) * 2 * L;
    fp.flags = fp.counters + L;
    for (int l = 0; l < L; ++l) {
      fp.kb[l] = static_cast<char*>(p->k[l]);
      fp.vb[l] = static_cast<char*>(p->v[l]);
    }
    e = strata::launch_ldg_fused(fp, dir, c, threads, s);
    if (e != cudaSuccess) return op_fail(e, "fused transfer kernel launch");
    p->ops[slot].fused = true;
    ++p->counters.kernel_launches;
    cudaStream_t side = p->side[slot];
    // the last layer completes with the kernel: its event goes on the caller's stream, sparing the
    // op's completion the side stream's flag-poll latency
    e = cudaEventRecord(p->events[size_t(slot) * (L + 1) + x->layer_end], s);
    if (e != cudaSuccess) return op_fail(e, "cudaEventRecord");
    for (int32_t l = x->layer_begin; l + 1 < x->layer_end; ++l) {
      if (g_wait_value32(reinterpret_cast<CUstream>(side), reinterpret_cast<CUdeviceptr>(fp.flags + l), fp.epoch,
                         CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return op_fail(cudaErrorUnknown, "cuStreamWaitValue32");
      e = cudaEventRecord(p->events[size_t(slot) * (L + 1) + 1 + l], side);
      if (e != cudaSuccess) return op_fail(e, "cudaEventRecord");
    }
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
      if (engine != STRATA_ENGINE_LDG) {
        const int64_t pieces = (rows + xp.tma_rows - 1) / xp.tma_rows;
        if (pieces < c) c = static_cast<int>(pieces);
        e = strata::launch_tma(xp, dir, c, engine == STRATA_ENGINE_TMA, s);
      } else {
        const int64_t groups = (rows + xp.rows_per_group - 1) / xp.rows_per_group;
        const int64_t need = (groups * 32 + threads - 1) / threads;
        if (need < c) c = static_cast<int>(need);
        e = strata::launch_ldg(xp, dir, c, threads, unroll, s);
      }
      if (e != cudaSuccess) return op_fail(e, "transfer kernel launch");
      ++p->counters.kernel_launches;
    }
    e = cudaEventRecord(p->events[size_t(slot) * (L + 1) + 1 + l], s);
    if (e != cudaSuccess) return op_fail(e, "cudaEventRecord");
  }
  count_op(p, plan, x, engine);
  if (ticket) *ticket = t;
  return STRATA_OK;
}


}  // namespace strata
