// api.cpp — the libstrata C ABI (include/strata.h): host-tier registration, argument validation,
// launch planning and per-layer completion events.  Kernels live in kernels.cu.
//
// Host tier registration follows "CPU registered pinned memory" (§4.2): the tier is
// page-locked and mapped into the GPU's address space (UVA), so the kernels read and write it
// directly — no staging copies.  Library-allocated tiers are bound to the GPU's NUMA node and
// pre-touched (SURVEY.md §7 hard part 3).
//
// Launch planning: per call, validate, split the requests into launches of
// at most kMaxReqsPerLaunch whose tables travel in the kernel parameters, pick the SM quota
// ("a small number of large CUDA blocks"), then for every layer l in [l0, l1):
// launch, and record event (ticket, l) (§4.1: the executor waits per layer).
#include <cuda_runtime.h>

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

using strata::kEventRing;
using strata::kMaxReqsPerLaunch;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(STRATA_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

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

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// NUMA node of the GPU's PCIe function (sysfs), -1 if unknown.
int gpu_numa_node(int dev) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) return -1;
  for (char* c = bus; *c; ++c) *c = static_cast<char>(tolower(*c));
  std::ifstream f(std::string("/sys/bus/pci/devices/") + bus + "/numa_node");
  int node = -1;
  if (!(f >> node)) return -1;
  return node;
}

void bind_to_node(void* addr, size_t len, int node) {
  if (node < 0 || node >= 64) return;
  unsigned long mask = 1ul << node;
  const int MPOL_BIND_ = 2;
  // best effort: a failure (e.g. no NUMA support in the kernel) leaves the default policy
  syscall(SYS_mbind, addr, len, MPOL_BIND_, &mask, 64ul, 0u);
}

void pretouch(char* p, size_t bytes) {
  unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (bytes < (64u << 20)) nt = 1;
  std::vector<std::thread> th;
  const size_t per = (bytes / nt + 4095) & ~size_t(4095);
  for (unsigned t = 0; t < nt; ++t) {
    const size_t lo = std::min(bytes, t * per), hi = std::min(bytes, lo + per);
    if (hi > lo) th.emplace_back([=] { memset(p + lo, 0, hi - lo); });
  }
  for (auto& t : th) t.join();
}

int check_desc(const strata_pool_desc* d) {
  if (!d) return fail(STRATA_ERR_INVALID_ARG, "desc is NULL");
  if (d->num_layers < 1 || d->num_heads < 1 || d->head_dim < 1 || d->elem_bytes < 1 ||
      d->page_size < 1 || d->chunk_tokens < 1)
    return fail(STRATA_ERR_INVALID_ARG, "geometry fields must be >= 1 (L=%d H=%d D=%d e=%d P=%d C=%d)",
                d->num_layers, d->num_heads, d->head_dim, d->elem_bytes, d->page_size, d->chunk_tokens);
  if (d->num_pages < 1 || d->num_chunks < 1)
    return fail(STRATA_ERR_INVALID_ARG, "num_pages and num_chunks must be >= 1");
  if (d->num_pages > INT32_MAX || d->num_chunks > INT32_MAX)
    return fail(STRATA_ERR_INVALID_ARG, "pool indices are int32 (R10): num_pages/num_chunks < 2^31");
  if (!d->k_ptrs || !d->v_ptrs) return fail(STRATA_ERR_INVALID_ARG, "k_ptrs / v_ptrs is NULL");
  const int64_t head_bytes = int64_t(d->head_dim) * d->elem_bytes;
  const int64_t tok = head_bytes * d->num_heads;
  if (tok % 16) return fail(STRATA_ERR_ALIGNMENT, "H*D*e = %lld is not a multiple of 16 (R12)", (long long)tok);
  if (tok > INT32_MAX / 64) return fail(STRATA_ERR_INVALID_ARG, "token row too large");
  const int64_t ts = d->token_stride ? d->token_stride : tok;
  const int64_t hs = d->head_stride ? d->head_stride : head_bytes;
  const int64_t ps = d->page_stride ? d->page_stride : d->page_size * ts;
  if (ts < 0 || hs < 0 || ps < 0) return fail(STRATA_ERR_INVALID_ARG, "negative stride");
  if (ts % 16 || hs % 16 || ps % 16)
    return fail(STRATA_ERR_ALIGNMENT, "device strides must be multiples of 16 (page %lld token %lld head %lld)",
                (long long)ps, (long long)ts, (long long)hs);
  if (hs != head_bytes && head_bytes % 16)
    return fail(STRATA_ERR_ALIGNMENT, "non-contiguous heads need D*e %% 16 == 0");
  for (int l = 0; l < d->num_layers; ++l) {
    if (!d->k_ptrs[l] || !d->v_ptrs[l]) return fail(STRATA_ERR_INVALID_ARG, "layer %d K/V pointer is NULL", l);
    if (!aligned16(d->k_ptrs[l]) || !aligned16(d->v_ptrs[l]))
      return fail(STRATA_ERR_ALIGNMENT, "layer %d K/V pointer not 16-byte aligned", l);
  }
  if (d->host_base && !aligned16(d->host_base)) return fail(STRATA_ERR_ALIGNMENT, "host_base not 16-byte aligned");
  const int64_t chunk = int64_t(d->num_layers) * 2 * d->chunk_tokens * tok;
  if (chunk / tok / 2 / d->chunk_tokens != d->num_layers || d->num_chunks > INT64_MAX / chunk)
    return fail(STRATA_ERR_INVALID_ARG, "host tier size overflows");
  return STRATA_OK;
}

void free_host(strata_pool* p) {
  if (p->registered_by_us && p->host) cudaHostUnregister(p->host);
  if (p->host_kind == 1 && p->host) munmap(p->host, p->map_bytes);
  if (p->host_kind == 2 && p->host) cudaFreeHost(p->host);
  p->host = nullptr;
}

void free_dma(strata_pool* p);

void destroy(strata_pool* p) {
  free_dma(p);
  for (cudaEvent_t e : p->events)
    if (e) cudaEventDestroy(e);
  if (p->bitmap) cudaFree(p->bitmap);
  if (p->err_dev) cudaFree(p->err_dev);
  if (p->err_host) cudaFreeHost(p->err_host);
  free_host(p);
  delete p;
}

// -------------------------------------------------------------------------------------------------
// Per-call planning.
struct Batch {
  int32_t first, count;     // requests [first, first+count) among the non-empty ones
  int32_t ntok;
};

struct Plan {
  std::vector<int32_t> reqs;   // indices of requests with tokens
  std::vector<Batch> batches;
  int64_t total_tokens = 0;
};

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

int ilog2_exact(int v) {
  if (v <= 0 || (v & (v - 1))) return -1;
  int s = 0;
  while ((1 << s) < v) ++s;
  return s;
}

// Defaults chosen on B200 measurements: both engines saturate the PCIe Gen5 link
// with a small SM quota.
// The paper's quota: 2 CTAs x 1024 threads.  On B200 that moves 50.3 GB/s (90.7 % of
// the link) with 0.8 % prefill-GEMM and 10.8 % decode slowdown (profiles/r01/interference2.jsonl).
constexpr int kDefaultCtasLdg = 2;
constexpr int kDefaultThreadsLdg = 1024;   // host-read throughput of an SM scales with its warps
constexpr int64_t kDmaMinLayerBytes = int64_t(4) << 20;
constexpr int64_t kDmaMinOffloadRun = int64_t(128) << 10;
constexpr int kDefaultUnroll = 8;
constexpr int kDefaultCtasTma = 2;   // warp-specialised ring: 51.0 GB/s at 2 CTAs (sweep_tma_ws15.jsonl)
constexpr int kTmaStageTarget = 32 << 10;

int run_validate(strata_pool* p, const strata_xfer* x, const Plan& plan, int dir, cudaStream_t s) {
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

bool env_validate() {
  const char* v = getenv("STRATA_VALIDATE");
  return v && *v && strcmp(v, "0") != 0;
}

// -------------------------------------------------------------------------------------------------
// STRATA_ENGINE_DMA: copy engines move whole page-first runs, an SM kernel does the scatter.
//
// The page-first host tier keeps, for one layer, the K rows and then the V rows of a chunk's C
// tokens back to back (R1), so a layer of a fully covered chunk is ONE contiguous 2*C*S_tok run
// (256 KiB for Llama-8B at C=64).  The copy engines read such runs at up to 98 % of the link
// (cudaMemcpyBatchAsync of 256 KiB copies over 4 streams, profiles/r01/ce_probe.jsonl) where
// SM-issued reads top out at 92.6 %.  Each run lands in an HBM staging slot laid out exactly like
// a compact host tier with one layer (slot j = [K rows][V rows] of C tokens), so the unchanged LDG
// kernel scatters it to the pages with chunk index = slot index.  Two slots alternate so the copy
// engines fill one while the SMs scatter the other.
struct ChunkPos {
  int32_t req;      // request index
  int32_t cq;       // position in the request's chunk list
  int32_t lo, cnt;  // tokens [lo, lo+cnt) of the chunk
  int32_t i0;       // index of the first of them within the request
};

struct Piece {
  size_t first, count;  // chunk positions [first, first+count) -> staging slots 0..count-1
};

constexpr size_t kStageTarget = size_t(64) << 20;   // bytes per staging slot
constexpr int kDefaultCtasScatter = 4;   // 2: 53.6-54.0, 4: 54.1-54.2, 8: 54.2-54.4 GB/s

int ensure_dma(strata_pool* p, size_t slot_bytes, int64_t slots) {
  cudaError_t e;
  if (!p->cs[0]) {
    if (const char* v = getenv("STRATA_COPY_STREAMS"))
      p->ncs = std::max(1, std::min(strata_pool::kCopyStreams, atoi(v)));
    for (auto& c : p->cs)
      if ((e = cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking))) return cuda_fail(e, "cudaStreamCreate");
    if ((e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming))) return cuda_fail(e, "cudaEventCreate");
    for (int s = 0; s < 2; ++s) {
      if ((e = cudaEventCreateWithFlags(&p->ev_slot[s], cudaEventDisableTiming))) return cuda_fail(e, "cudaEventCreate");
      for (auto& ev : p->ev_copy[s])
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming))) return cuda_fail(e, "cudaEventCreate");
    }
  }
  if (p->stage_bytes < slot_bytes) {
    for (auto& b : p->stage) {
      if (b) cudaFree(b);
      b = nullptr;
    }
    p->stage_bytes = 0;
    for (auto& b : p->stage)
      if ((e = cudaMalloc(&b, slot_bytes))) return fail(STRATA_ERR_OOM, "cudaMalloc(staging %zu): %s", slot_bytes,
                                                        cudaGetErrorString(e));
    p->stage_bytes = slot_bytes;
  }
  if (p->slot_cap < slots) {
    if (p->slot_ids) cudaFree(p->slot_ids);
    p->slot_ids = nullptr;
    p->slot_cap = 0;
    std::vector<int32_t> iota(static_cast<size_t>(slots));
    for (int64_t i = 0; i < slots; ++i) iota[i] = static_cast<int32_t>(i);
    if ((e = cudaMalloc(&p->slot_ids, iota.size() * 4))) return cuda_fail(e, "cudaMalloc(slot ids)");
    if ((e = cudaMemcpy(p->slot_ids, iota.data(), iota.size() * 4, cudaMemcpyHostToDevice)))
      return cuda_fail(e, "cudaMemcpy(slot ids)");
    p->slot_cap = slots;
  }
  return STRATA_OK;
}

void free_dma(strata_pool* p) {
  for (auto& b : p->stage)
    if (b) cudaFree(b);
  if (p->slot_ids) cudaFree(p->slot_ids);
  for (auto& c : p->cs)
    if (c) cudaStreamDestroy(c);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  for (int s = 0; s < 2; ++s) {
    if (p->ev_slot[s]) cudaEventDestroy(p->ev_slot[s]);
    for (auto& ev : p->ev_copy[s])
      if (ev) cudaEventDestroy(ev);
  }
}

// Submit a copy list over the pool's copy streams (contiguous shares, one batch call each).
cudaError_t submit_copies(strata_pool* p, std::vector<void*>& dst, std::vector<void*>& src, std::vector<size_t>& sz,
                          int dir, int slot) {
  cudaMemcpyAttributes attr;
  memset(&attr, 0, sizeof attr);
  attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  attr.srcLocHint.type = dir == 0 ? cudaMemLocationTypeHost : cudaMemLocationTypeDevice;
  attr.srcLocHint.id = dir == 0 ? 0 : p->d.device;
  attr.dstLocHint.type = dir == 0 ? cudaMemLocationTypeDevice : cudaMemLocationTypeHost;
  attr.dstLocHint.id = dir == 0 ? p->d.device : 0;
  const size_t n = dst.size();
  const int ns = p->ncs;
  // cudaMemcpyBatchAsync refuses stream capture; under capture the copies become plain memcpy nodes
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaError_t e0 = cudaStreamIsCapturing(p->cs[0], &cap);
  if (e0 != cudaSuccess) return e0;
  const cudaMemcpyKind kind = dir == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  for (int c = 0; c < ns; ++c) {
    const size_t lo = n * c / ns, hi = n * (c + 1) / ns;
    if (hi > lo && cap == cudaStreamCaptureStatusActive) {
      for (size_t i = lo; i < hi; ++i) {
        cudaError_t e = cudaMemcpyAsync(dst[i], src[i], sz[i], kind, p->cs[c]);
        if (e != cudaSuccess) return e;
      }
    } else if (hi > lo) {
      size_t idx = 0, fail_idx = 0;
      cudaError_t e = cudaMemcpyBatchAsync(dst.data() + lo, src.data() + lo, sz.data() + lo, hi - lo, &attr, &idx, 1,
                                           &fail_idx, p->cs[c]);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(p->ev_copy[slot][c], p->cs[c]);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int transfer_dma(strata_pool* p, const strata_xfer* x, const Plan& plan, strata::XferParams xp, cudaStream_t s,
                 int dir, int slot_ev) {
  if (!x->host_chunks_host && plan.total_tokens > 0)
    return fail(STRATA_ERR_INVALID_ARG, "STRATA_ENGINE_DMA needs xfer.host_chunks_host");
  const int64_t C = p->d.chunk_tokens, P = p->d.page_size, tok = p->tok_bytes;
  const int L = p->d.num_layers;
  // chunk positions of the call, request by request
  std::vector<ChunkPos> pos;
  for (int32_t r : plan.reqs) {
    const int64_t n = x->num_tokens[r];
    const int64_t oc = x->chunk_offset ? x->chunk_offset[r] : 0;
    int64_t i = 0;
    for (int32_t cq = 0; i < n; ++cq) {
      const int64_t lo = cq == 0 ? oc : 0;
      const int64_t cnt = std::min(C - lo, n - i);
      const int64_t hc = x->host_chunks_host[x->chunk_start[r] + cq];
      if (hc < 0 || hc >= p->d.num_chunks) return fail(STRATA_ERR_INDEX_RANGE, "host chunk %lld out of range", (long long)hc);
      pos.push_back({r, cq, static_cast<int32_t>(lo), static_cast<int32_t>(cnt), static_cast<int32_t>(i)});
      i += cnt;
    }
  }
  const size_t unit = static_cast<size_t>(2 * C * tok);             // one chunk-layer: K rows, V rows
  // layers per copy run.  Loads keep per-layer granularity (grouping does not raise H2D throughput,
  // profiles/r01/sweep_groups*.jsonl); offloads ("backup", a non-critical path) group
  // layers until a run is >= 128 KiB, which D2H copies need (70B TP=8 rank: 44.6 -> 55.8 GB/s).
  int G = x->layer_group;
  if (G <= 0)
    G = dir == 0 ? 1 : static_cast<int>(std::min<int64_t>(8, (kDmaMinOffloadRun + 2 * C * tok - 1) / (2 * C * tok)));
  G = std::max(1, std::min(G, std::max(1, x->layer_end - x->layer_begin)));
  const size_t gunit = unit * static_cast<size_t>(G);                 // staging bytes per chunk
  const size_t per_piece = std::max<size_t>(1, std::min(pos.size(), kStageTarget / gunit));
  // pieces: <= per_piece chunk positions and <= kMaxReqsPerLaunch requests each
  std::vector<Piece> pieces;
  for (size_t k = 0; k < pos.size();) {
    Piece pc{k, 0};
    int nreq = 0;
    int32_t last = -1;
    while (k < pos.size() && pc.count < per_piece) {
      if (pos[k].req != last) {
        if (nreq == kMaxReqsPerLaunch) break;
        ++nreq;
        last = pos[k].req;
      }
      ++pc.count;
      ++k;
    }
    pieces.push_back(pc);
  }
  int rc = ensure_dma(p, per_piece * gunit, static_cast<int64_t>(per_piece));
  if (rc) return rc;

  cudaError_t e;
  const int threads = x->threads ? x->threads : kDefaultThreadsLdg;
  const int unroll = threads > 512 ? 4 : kDefaultUnroll;
  xp.rows_per_group = 32;   // lane t fetches row t; the warp then streams the 32 rows
  const int ctas = x->num_ctas ? x->num_ctas : kDefaultCtasScatter;
  // staging slot j holds chunk position j's G layers: [G][K,V][C][H][D], a compact host tier
  xp.chunk_bytes = static_cast<int64_t>(gunit);
  xp.kv_off = C * tok;
  xp.host_chunks = p->slot_ids;

  if ((e = cudaEventRecord(p->ev_fork, s))) return cuda_fail(e, "cudaEventRecord");
  for (int ci = 0; ci < p->ncs; ++ci)
    if ((e = cudaStreamWaitEvent(p->cs[ci], p->ev_fork, 0))) return cuda_fail(e, "cudaStreamWaitEvent");
  std::vector<void*> dst, src;
  std::vector<size_t> sz;
  int64_t i = 0;
  int last_slot = 0;
  auto layer_event = [&](int32_t l) { return p->events[size_t(slot_ev) * (L + 1) + 1 + l]; };
  for (int32_t lg = x->layer_begin; lg < x->layer_end; lg += G) {
    const int gl = std::min<int>(G, x->layer_end - lg);   // layers in this group
    for (const Piece& pc : pieces) {
      const bool last_piece = &pc == &pieces.back();
      const int slot = static_cast<int>(i & 1);
      char* stage = p->stage[slot];
      // copy list of this piece for layers [lg, lg+gl) (host <-> staging slot)
      dst.clear();
      src.clear();
      sz.clear();
      for (size_t j = 0; j < pc.count; ++j) {
        const ChunkPos& cp = pos[pc.first + j];
        const int64_t hc = x->host_chunks_host[x->chunk_start[cp.req] + cp.cq];
        char* h = p->host + hc * p->chunk_bytes + int64_t(lg) * 2 * C * tok;
        char* d = stage + j * gunit;
        auto add = [&](int64_t off, int64_t bytes) {
          dst.push_back(dir == 0 ? d + off : h + off);
          src.push_back(dir == 0 ? h + off : d + off);
          sz.push_back(static_cast<size_t>(bytes));
        };
        if (cp.lo == 0 && cp.cnt == C) {
          add(0, gl * 2 * C * tok);                    // the group's K,V runs are adjacent: one copy
        } else {
          for (int g = 0; g < gl; ++g) {
            add(g * 2 * C * tok + cp.lo * tok, cp.cnt * tok);        // K rows of layer lg+g
            add(g * 2 * C * tok + (C + cp.lo) * tok, cp.cnt * tok);  // V rows
          }
        }
      }
      // request table of the piece: sub-requests addressing staging slots
      strata::ReqTable& rt = xp.rt;
      rt.n = 0;
      int32_t acc = 0;
      for (size_t j = 0; j < pc.count; ++j) {
        const ChunkPos& cp = pos[pc.first + j];
        if (j == 0 || cp.req != pos[pc.first + j - 1].req) {
          const int k = rt.n++;
          const int64_t op = x->page_offset ? x->page_offset[cp.req] : 0;
          const int64_t pi0 = op + cp.i0;
          rt.tok_end[k] = acc;
          rt.chunk_base[k] = static_cast<int32_t>(j);
          rt.off_c[k] = cp.lo;
          rt.page_base[k] = static_cast<int32_t>(x->page_start[cp.req] + pi0 / P);
          rt.off_p[k] = static_cast<int32_t>(pi0 % P);
        }
        acc += cp.cnt;
        rt.tok_end[rt.n - 1] = acc;
      }
      xp.ntok = acc;
      xp.host = stage;
      const int64_t groups = (2LL * acc + xp.rows_per_group - 1) / xp.rows_per_group;
      const int c = static_cast<int>(std::min<int64_t>(ctas, (groups * 32 + threads - 1) / threads));
      // one scatter / gather launch per layer of the group over the slot's layer sub-blocks
      auto launch_group = [&](int kdir) -> cudaError_t {
        for (int g = 0; g < gl; ++g) {
          xp.kbase = static_cast<char*>(p->k[lg + g]);
          xp.vbase = static_cast<char*>(p->v[lg + g]);
          xp.layer_off = int64_t(g) * 2 * C * tok;
          cudaError_t le = strata::launch_ldg(xp, kdir, c, threads, unroll, s);
          if (le != cudaSuccess) return le;
          ++p->counters.kernel_launches;
          // loads: layer lg+g is complete once its scatter of the group's last piece has run
          if (kdir == 0 && last_piece && (le = cudaEventRecord(layer_event(lg + g), s))) return le;
        }
        return cudaSuccess;
      };
      const int ncs = p->ncs;
      if (dir == 0) {
        // copies into the slot (after its previous scatter), then the scatters on the caller's stream
        if (i >= 2)
          for (int ci = 0; ci < ncs; ++ci)
            if ((e = cudaStreamWaitEvent(p->cs[ci], p->ev_slot[slot], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = submit_copies(p, dst, src, sz, dir, slot))) return cuda_fail(e, "cudaMemcpyBatchAsync");
        for (int ci = 0; ci < ncs; ++ci)
          if ((e = cudaStreamWaitEvent(s, p->ev_copy[slot][ci], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = launch_group(0))) return cuda_fail(e, "scatter kernel launch");
        if ((e = cudaEventRecord(p->ev_slot[slot], s))) return cuda_fail(e, "cudaEventRecord");
      } else {
        // gathers into the slot (after its previous copies drained), then copies to the host tier
        if (i >= 2)
          for (int ci = 0; ci < ncs; ++ci)
            if ((e = cudaStreamWaitEvent(s, p->ev_copy[slot][ci], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = launch_group(1))) return cuda_fail(e, "gather kernel launch");
        if ((e = cudaEventRecord(p->ev_slot[slot], s))) return cuda_fail(e, "cudaEventRecord");
        for (int ci = 0; ci < ncs; ++ci)
          if ((e = cudaStreamWaitEvent(p->cs[ci], p->ev_slot[slot], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = submit_copies(p, dst, src, sz, dir, slot))) return cuda_fail(e, "cudaMemcpyBatchAsync");
      }
      p->counters.dma_copies += static_cast<int64_t>(dst.size());
      last_slot = slot;
      ++i;
    }
    if (dir == 0 && pieces.empty()) {
      for (int g = 0; g < gl; ++g)
        if ((e = cudaEventRecord(layer_event(lg + g), s))) return cuda_fail(e, "cudaEventRecord");
    } else if (dir == 1) {
      // host bytes of the group are written once every copy stream has passed its last piece
      if (!pieces.empty())
        for (int c = 1; c < p->ncs; ++c)
          if ((e = cudaStreamWaitEvent(p->cs[0], p->ev_copy[last_slot][c], 0)))
            return cuda_fail(e, "cudaStreamWaitEvent");
      for (int g = 0; g < gl; ++g)
        if ((e = cudaEventRecord(layer_event(lg + g), p->cs[0]))) return cuda_fail(e, "cudaEventRecord");
    }
  }
  if (dir == 1 && i > 0)  // join: the caller's stream is ordered after every copy
    for (int ci = 0; ci < p->ncs; ++ci)
      if ((e = cudaStreamWaitEvent(s, p->ev_copy[last_slot][ci], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
  return STRATA_OK;
}

void count_op(strata_pool* p, const Plan& plan, const strata_xfer* x, int engine) {
  p->counters.operations += 1;
  p->counters.bytes += 2 * plan.total_tokens * p->tok_bytes * (x->layer_end - x->layer_begin);
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
  xp.vph = xp.head_bytes / 16;
  xp.c_shift = ilog2_exact(xp.C);
  xp.p_shift = ilog2_exact(xp.P);
  xp.chunk_bytes = p->chunk_bytes;
  xp.kv_off = int64_t(p->d.chunk_tokens) * p->tok_bytes;
  xp.page_stride = p->page_stride;
  xp.token_stride = p->token_stride;
  xp.head_stride = p->head_stride;
  xp.host = p->host_dev;
  xp.host_chunks = x->host_chunks;
  xp.dev_pages = x->dev_pages;

  int engine = x->engine;
  if (engine == STRATA_ENGINE_DEFAULT) {
    // Measured on B200: the copy-engine gather + SM scatter moves 98 % of the link
    // for layer-sized transfers; below a few MiB per layer its per-piece submission latency is not
    // amortised and the zero-copy LDG kernel wins.  Without a host mirror of the chunk list only
    // the kernel engines can run.
    // (Offloads group layers into >= 128 KiB runs inside the DMA engine, see transfer_dma.)
    const int64_t layer_bytes = 2 * plan.total_tokens * p->tok_bytes;
    const bool dma = x->host_chunks_host && layer_bytes >= kDmaMinLayerBytes;
    engine = dma ? STRATA_ENGINE_DMA : STRATA_ENGINE_LDG;
  }
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
  xp.rows_per_group = 32;   // lane t fetches row t; the warp then streams the 32 rows (amortised index math)
  int ctas = x->num_ctas ? x->num_ctas : (engine == STRATA_ENGINE_LDG ? kDefaultCtasLdg : kDefaultCtasTma);
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
  for (int32_t l = x->layer_begin; l < x->layer_end; ++l) {
    xp.kbase = static_cast<char*>(p->k[l]);
    xp.vbase = static_cast<char*>(p->v[l]);
    xp.layer_off = int64_t(l) * 2 * p->d.chunk_tokens * p->tok_bytes;
    for (const Batch& b : plan.batches) {
      xp.ntok = b.ntok;
      fill_table(x, plan, b, xp.rt);
      const int64_t rows = 2LL * b.ntok;
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

}  // namespace

int strata::set_last_error(int code, const char* msg) {
  g_err = msg;
  return code;
}

extern "C" {

int strata_version(void) { return 100; }

const char* strata_last_error(void) { return g_err.c_str(); }

int strata_register_host_pool(const strata_pool_desc* d, strata_pool_t* out) {
  if (!out) return fail(STRATA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  int rc = check_desc(d);
  if (rc) return rc;
  strata_pool* p = new (std::nothrow) strata_pool();
  if (!p) return fail(STRATA_ERR_OOM, "out of host memory");
  p->d = *d;
  p->k.assign(d->k_ptrs, d->k_ptrs + d->num_layers);
  p->v.assign(d->v_ptrs, d->v_ptrs + d->num_layers);
  p->d.k_ptrs = p->k.data();
  p->d.v_ptrs = p->v.data();
  p->head_bytes = int64_t(d->head_dim) * d->elem_bytes;
  p->tok_bytes = p->head_bytes * d->num_heads;
  p->chunk_bytes = int64_t(d->num_layers) * 2 * d->chunk_tokens * p->tok_bytes;
  p->token_stride = d->token_stride ? d->token_stride : p->tok_bytes;
  p->head_stride = d->head_stride ? d->head_stride : p->head_bytes;
  p->page_stride = d->page_stride ? d->page_stride : d->page_size * p->token_stride;
  p->host_bytes = size_t(d->num_chunks) * size_t(p->chunk_bytes);

  DeviceGuard dg(d->device);
  if (dg.err) {
    delete p;
    return cuda_fail(dg.err, "cudaSetDevice");
  }
  cudaError_t e;
  int can_map = 0;
  if ((e = cudaDeviceGetAttribute(&can_map, cudaDevAttrCanMapHostMemory, d->device))) {
    delete p;
    return cuda_fail(e, "cudaDeviceGetAttribute");
  }
  if (!can_map) {
    delete p;
    return fail(STRATA_ERR_UNSUPPORTED, "device cannot map host memory");
  }

  if (d->host_base) {
    p->host = static_cast<char*>(d->host_base);
    p->host_kind = 0;
    e = cudaHostRegister(p->host, p->host_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      cudaGetLastError();
    } else if (e != cudaSuccess) {
      p->host = nullptr;
      delete p;
      return cuda_fail(e, "cudaHostRegister(host_base)");
    } else {
      p->registered_by_us = true;
    }
  } else if (d->flags & (STRATA_HOST_WRITECOMBINED | STRATA_HOST_CUDA_ALLOC)) {
    void* h = nullptr;
    unsigned fl = cudaHostAllocMapped | cudaHostAllocPortable;
    if (d->flags & STRATA_HOST_WRITECOMBINED) fl |= cudaHostAllocWriteCombined;
    e = cudaHostAlloc(&h, p->host_bytes, fl);
    if (e != cudaSuccess) {
      const size_t want = p->host_bytes;
      delete p;
      return fail(STRATA_ERR_OOM, "cudaHostAlloc(%zu, flags %u): %s", want, fl, cudaGetErrorString(e));
    }
    p->host = static_cast<char*>(h);
    p->host_kind = 2;
  } else {
    const size_t huge = size_t(2) << 20;
    p->map_bytes = (p->host_bytes + huge - 1) / huge * huge;
    void* h = MAP_FAILED;
    if (d->flags & STRATA_HOST_HUGEPAGES)
      h = mmap(nullptr, p->map_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB, -1, 0);
    if (h == MAP_FAILED) h = mmap(nullptr, p->map_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (h == MAP_FAILED) {
      const size_t want = p->map_bytes;
      const int err = errno;
      delete p;
      return fail(STRATA_ERR_OOM, "mmap(%zu): %s", want, strerror(err));
    }
    p->host = static_cast<char*>(h);
    p->host_kind = 1;
    if (d->flags & STRATA_HOST_HUGEPAGES) madvise(h, p->map_bytes, MADV_HUGEPAGE);
    if (!(d->flags & STRATA_HOST_NO_NUMA_BIND)) bind_to_node(h, p->map_bytes, gpu_numa_node(d->device));
    pretouch(p->host, p->map_bytes);
    e = cudaHostRegister(p->host, p->map_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      destroy(p);
      return fail(STRATA_ERR_OOM, "cudaHostRegister(%zu): %s", p->map_bytes, cudaGetErrorString(e));
    }
    p->registered_by_us = true;
  }
  void* dptr = nullptr;
  if ((e = cudaHostGetDevicePointer(&dptr, p->host, 0))) {
    destroy(p);
    return cuda_fail(e, "cudaHostGetDevicePointer");
  }
  p->host_dev = static_cast<char*>(dptr);

  p->events.assign(size_t(kEventRing) * (d->num_layers + 1), nullptr);
  for (auto& ev : p->events) {
    if ((e = cudaEventCreate(&ev))) {
      destroy(p);
      return cuda_fail(e, "cudaEventCreate");
    }
  }
  for (auto& op : p->ops) op = {0, 0, 0};
  p->tma_smem = strata::tma_smem_limit();
  if (p->tma_smem > 0 && (e = strata::tma_prepare(p->tma_smem))) {
    destroy(p);
    return cuda_fail(e, "cudaFuncSetAttribute(TMA smem)");
  }
  *out = p;
  return STRATA_OK;
}

int strata_unregister_host_pool(strata_pool_t p) {
  if (!p) return STRATA_OK;
  DeviceGuard dg(p->d.device);
  // wait for every operation whose events are still live
  for (const auto& op : p->ops) {
    if (op.ticket && op.l1 > op.l0) {
      const int slot = static_cast<int>(op.ticket % kEventRing);
      cudaEventSynchronize(p->events[size_t(slot) * (p->d.num_layers + 1) + op.l1]);
    }
  }
  destroy(p);
  return STRATA_OK;
}

int strata_host_pool_ptr(strata_pool_t p, void** host_base, size_t* bytes) {
  if (!p) return fail(STRATA_ERR_INVALID_ARG, "pool is NULL");
  if (host_base) *host_base = p->host;
  if (bytes) *bytes = p->host_bytes;
  return STRATA_OK;
}

int strata_load(strata_pool_t p, const strata_xfer* x, strata_stream_t stream, uint64_t* ticket) {
  return transfer(p, x, reinterpret_cast<cudaStream_t>(stream), ticket, 0);
}

int strata_offload(strata_pool_t p, const strata_xfer* x, strata_stream_t stream, uint64_t* ticket) {
  return transfer(p, x, reinterpret_cast<cudaStream_t>(stream), ticket, 1);
}

namespace {
// Resolves (ticket, layer) to the ring slot; 0 on success.
int find_op(strata_pool_t p, uint64_t& ticket, int32_t layer, int& slot) {
  if (!p) return fail(STRATA_ERR_INVALID_ARG, "pool is NULL");
  const uint64_t last = p->next_ticket - 1;
  if (ticket == 0) ticket = last;
  if (ticket == 0 || ticket > last || ticket + kEventRing <= last)
    return fail(STRATA_ERR_STALE_TICKET, "ticket %llu not live (latest %llu, ring %d)",
                (unsigned long long)ticket, (unsigned long long)last, kEventRing);
  slot = static_cast<int>(ticket % kEventRing);
  const auto& op = p->ops[slot];
  if (op.ticket != ticket) return fail(STRATA_ERR_STALE_TICKET, "ticket %llu overwritten", (unsigned long long)ticket);
  if (layer < op.l0 || layer >= op.l1)
    return fail(STRATA_ERR_INVALID_ARG, "layer %d outside the operation's range [%d,%d)", layer, op.l0, op.l1);
  return STRATA_OK;
}
}  // namespace

int strata_layer_event(strata_pool_t p, uint64_t ticket, int32_t layer, strata_event_t* out) {
  if (!out) return fail(STRATA_ERR_INVALID_ARG, "out is NULL");
  int slot = 0;
  int rc = find_op(p, ticket, layer, slot);
  if (rc) return rc;
  *out = reinterpret_cast<strata_event_t>(p->events[size_t(slot) * (p->d.num_layers + 1) + 1 + layer]);
  return STRATA_OK;
}

int strata_get_counters(strata_pool_t p, strata_counters* out) {
  if (!p || !out) return fail(STRATA_ERR_INVALID_ARG, "pool / out is NULL");
  *out = p->counters;
  return STRATA_OK;
}

int strata_wait_layer(strata_pool_t p, uint64_t ticket, int32_t layer, strata_stream_t consumer) {
  int slot = 0;
  int rc = find_op(p, ticket, layer, slot);
  if (rc) return rc;
  cudaError_t e = cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(consumer),
                                      p->events[size_t(slot) * (p->d.num_layers + 1) + 1 + layer], 0);
  return e == cudaSuccess ? STRATA_OK : cuda_fail(e, "cudaStreamWaitEvent");
}

int strata_layer_elapsed_ms(strata_pool_t p, uint64_t ticket, int32_t layer, float* ms) {
  if (!ms) return fail(STRATA_ERR_INVALID_ARG, "ms is NULL");
  int slot = 0;
  int rc = find_op(p, ticket, layer, slot);
  if (rc) return rc;
  const size_t base = size_t(slot) * (p->d.num_layers + 1);
  cudaError_t e = cudaEventSynchronize(p->events[base + 1 + layer]);
  if (e == cudaSuccess) e = cudaEventElapsedTime(ms, p->events[base], p->events[base + 1 + layer]);
  return e == cudaSuccess ? STRATA_OK : cuda_fail(e, "cudaEventElapsedTime");
}

}  // extern "C"
