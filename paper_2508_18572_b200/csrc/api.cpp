// api.cpp — the libstrata C ABI surface (include/strata.h): host-tier registration, the per-layer
// completion events and counters, error reporting.  Validation, planning and the kernel engines live
// in transfer.cpp, the copy-engine engine in dma.cpp, the kernels in kernels.cu.
//
// Host tier registration follows "CPU registered pinned memory" (§4.2): the tier is
// page-locked and mapped into the GPU's address space (UVA), so the kernels read and write it
// directly — no staging copies.  Library-allocated tiers are bound to the GPU's NUMA node and
// pre-touched (SURVEY.md §7 hard part 3).
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
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
using strata::cuda_fail;
using strata::DeviceGuard;
using strata::fail;
using strata::kEventRing;

namespace {

thread_local std::string g_err;

}  // namespace

int strata::fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int strata::cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();   // the failing call just set it: leave no stale error for the caller's next launch
  return fail(STRATA_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

namespace {

// Widest access (16, 8, 4, 2 or 1 bytes) that divides every row size, stride, offset and base of
// the pool: 16 selects the vectorised engines, anything else the narrow LDG kernel (R29).
int access_granularity(const strata_pool* p) {
  int g = 16;
  auto fit = [&](uint64_t v) {
    while (g > 1 && v % uint64_t(g)) g >>= 1;
  };
  fit(uint64_t(p->tok_bytes));
  fit(uint64_t(p->head_bytes));
  fit(uint64_t(p->token_stride));
  fit(uint64_t(p->head_stride));
  fit(uint64_t(p->page_stride));
  fit(uint64_t(p->host_tok_stride));
  fit(uint64_t(p->host_head_stride));
  fit(uint64_t(p->host_head_off));
  fit(uint64_t(p->host_kv_off));
  fit(uint64_t(p->chunk_bytes));
  fit(reinterpret_cast<uintptr_t>(p->host_dev));
  for (int l = 0; l < p->d.num_layers; ++l) {
    fit(reinterpret_cast<uintptr_t>(p->k[l]));
    fit(reinterpret_cast<uintptr_t>(p->v[l]));
  }
  return g;
}

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
  const bool single = d->flags & STRATA_POOL_SINGLE_KV;
  const int64_t nkv = single ? 1 : 2;
  if (!d->k_ptrs || (!single && !d->v_ptrs)) return fail(STRATA_ERR_INVALID_ARG, "k_ptrs / v_ptrs is NULL");
  const int64_t head_bytes = int64_t(d->head_dim) * d->elem_bytes;
  const int64_t tok = head_bytes * d->num_heads;
  if (tok > INT32_MAX / 64) return fail(STRATA_ERR_INVALID_ARG, "token row too large");
  const int64_t ts = d->token_stride ? d->token_stride : tok;
  const int64_t hs = d->head_stride ? d->head_stride : head_bytes;
  const int64_t ps = d->page_stride ? d->page_stride : d->page_size * ts;
  if (ts < 0 || hs < 0 || ps < 0) return fail(STRATA_ERR_INVALID_ARG, "negative stride");
  // Rows need not be multiples of 16 bytes (R29: 16-byte-aligned pools take the vectorised engines,
  // others the narrow LDG kernel), but every base and stride must be a multiple of the element size.
  const int64_t e = d->elem_bytes;
  if (ts % e || hs % e || ps % e)
    return fail(STRATA_ERR_ALIGNMENT, "device strides must be multiples of the element size %lld (page %lld token "
                "%lld head %lld)", (long long)e, (long long)ps, (long long)ts, (long long)hs);
  const int64_t Ht = d->host_heads ? d->host_heads : d->num_heads;
  if (d->host_heads < 0 || d->head_begin < 0 || d->head_begin + int64_t(d->num_heads) > Ht)
    return fail(STRATA_ERR_INVALID_ARG, "head slice [%d,%d) not inside the host tier's %lld heads", d->head_begin,
                d->head_begin + d->num_heads, (long long)Ht);
  auto aligned_e = [&](const void* q) { return (reinterpret_cast<uintptr_t>(q) % uintptr_t(e)) == 0; };
  for (int l = 0; l < d->num_layers; ++l) {
    void* const vp = single ? d->k_ptrs[l] : d->v_ptrs[l];
    if (!d->k_ptrs[l] || !vp) return fail(STRATA_ERR_INVALID_ARG, "layer %d K/V pointer is NULL", l);
    if (!aligned_e(d->k_ptrs[l]) || !aligned_e(vp))
      return fail(STRATA_ERR_ALIGNMENT, "layer %d K/V pointer not aligned to the element size", l);
  }
  if (d->host_base && !aligned_e(d->host_base))
    return fail(STRATA_ERR_ALIGNMENT, "host_base not aligned to the element size");
  const int64_t htok = head_bytes * Ht;   // one token of one chunk-layer-kv block, all host heads
  const int64_t chunk = int64_t(d->num_layers) * nkv * d->chunk_tokens * htok;
  if (chunk / htok / nkv / d->chunk_tokens != d->num_layers || d->num_chunks > INT64_MAX / chunk)
    return fail(STRATA_ERR_INVALID_ARG, "host tier size overflows");
  return STRATA_OK;
}

// MemAvailable from /proc/meminfo in MiB (-1 if unknown): context for an allocation failure.
long mem_available_mb() {
  FILE* f = fopen("/proc/meminfo", "r");
  if (!f) return -1;
  char line[256];
  long kb = -1;
  while (fgets(line, sizeof line, f))
    if (sscanf(line, "MemAvailable: %ld kB", &kb) == 1) break;
  fclose(f);
  return kb < 0 ? -1 : kb / 1024;
}

// Caller memory registered by this library, shared by every pool whose tier lies inside it (e.g. one
// host tier holding every KV head, read by the pools of several TP ranks, R28): the registration is
// undone only when the last of those pools closes, never while another still reads it through UVA.
struct HostReg {
  char* base;
  size_t bytes;
  int refs;
};
std::mutex g_reg_mu;
std::vector<HostReg> g_regs;

// 0: registered (or shared) by the library, 1: registered by someone else (not ours to undo).
cudaError_t register_caller(char* base, size_t bytes, bool& ours) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  for (auto& r : g_regs)
    if (base >= r.base && base + bytes <= r.base + r.bytes) {
      ++r.refs;
      ours = true;
      return cudaSuccess;
    }
  // a range that overlaps one of the library's registrations without lying inside it cannot share
  // it (the registration would be undone under this pool when the other pools close)
  for (const auto& r : g_regs)
    if (base < r.base + r.bytes && r.base < base + bytes) return cudaErrorHostMemoryAlreadyRegistered;
  cudaError_t e = cudaHostRegister(base, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    ours = false;
    return cudaSuccess;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e;
  }
  g_regs.push_back({base, bytes, 1});
  ours = true;
  return cudaSuccess;
}

void unregister_caller(char* base, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  for (size_t i = 0; i < g_regs.size(); ++i) {
    HostReg& r = g_regs[i];
    if (base >= r.base && base + bytes <= r.base + r.bytes) {
      if (--r.refs == 0) {
        cudaHostUnregister(r.base);
        g_regs.erase(g_regs.begin() + static_cast<std::ptrdiff_t>(i));
      }
      return;
    }
  }
}

void free_host(strata_pool* p) {
  if (p->registered_by_us && p->host) {
    if (p->host_kind == 0) unregister_caller(p->host, p->host_bytes);
    else cudaHostUnregister(p->host);
  }
  if (p->host_kind == 1 && p->host) munmap(p->host, p->map_bytes);
  if (p->host_kind == 2 && p->host) cudaFreeHost(p->host);
  p->host = nullptr;
}

void destroy(strata_pool* p) {
  strata::free_dma(p);
  strata::free_fused(p);
  for (cudaEvent_t e : p->events)
    if (e) cudaEventDestroy(e);
  for (auto& kv : p->captured_ops)
    for (cudaEvent_t e : kv.second.ev)
      if (e) cudaEventDestroy(e);
  if (p->bitmap) cudaFree(p->bitmap);
  if (p->err_dev) cudaFree(p->err_dev);
  if (p->err_host) cudaFreeHost(p->err_host);
  free_host(p);
  delete p;
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
  p->nkv = (d->flags & STRATA_POOL_SINGLE_KV) ? 1 : 2;
  p->k.assign(d->k_ptrs, d->k_ptrs + d->num_layers);
  // a single-buffer pool never touches its V bases; they alias K so no path sees a null pointer
  if (p->nkv == 2) p->v.assign(d->v_ptrs, d->v_ptrs + d->num_layers);
  else p->v = p->k;
  p->d.k_ptrs = p->k.data();
  p->d.v_ptrs = p->v.data();
  p->head_bytes = int64_t(d->head_dim) * d->elem_bytes;
  p->tok_bytes = p->head_bytes * d->num_heads;
  p->host_heads = d->host_heads ? d->host_heads : d->num_heads;
  p->head_begin = d->head_begin;
  p->head_major = d->flags & STRATA_HOST_HEAD_MAJOR;
  p->chunk_bytes = int64_t(d->num_layers) * p->nkv * d->chunk_tokens * p->host_heads * p->head_bytes;
  if (p->head_major) {   // chunk = [Ht][L][KV][C][D]
    p->host_kv_off = int64_t(d->chunk_tokens) * p->head_bytes;
    p->host_tok_stride = p->head_bytes;
    p->host_head_stride = int64_t(d->num_layers) * p->nkv * p->host_kv_off;
    p->host_head_off = int64_t(p->head_begin) * p->host_head_stride;
  } else {               // chunk = [L][KV][C][Ht][D]
    p->host_kv_off = int64_t(d->chunk_tokens) * p->host_heads * p->head_bytes;
    p->host_tok_stride = int64_t(p->host_heads) * p->head_bytes;
    p->host_head_off = int64_t(p->head_begin) * p->head_bytes;
    p->host_head_stride = p->head_bytes;
  }
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
    bool ours = false;
    e = register_caller(p->host, p->host_bytes, ours);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      p->host = nullptr;
      delete p;
      return fail(STRATA_ERR_INVALID_ARG, "host_base range overlaps the host tier of another open pool without "
                  "lying inside it (pools may share a tier only when one range contains the other's)");
    }
    if (e != cudaSuccess) {
      p->host = nullptr;
      delete p;
      return cuda_fail(e, "cudaHostRegister(host_base)");
    }
    p->registered_by_us = ours;
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
      // page-locking the mapping failed (memory pressure / locked-memory limits): fall back to the
      // driver's own pinned allocator before giving up
      cudaGetLastError();
      munmap(p->host, p->map_bytes);
      p->host = nullptr;
      p->host_kind = 0;
      void* h2 = nullptr;
      const cudaError_t e2 = cudaHostAlloc(&h2, p->host_bytes, cudaHostAllocMapped | cudaHostAllocPortable);
      if (e2 != cudaSuccess) {
        cudaGetLastError();
        const size_t want = p->map_bytes;
        const long avail_mb = mem_available_mb();
        destroy(p);
        return fail(STRATA_ERR_OOM, "cudaHostRegister(%zu): %s; cudaHostAlloc: %s (MemAvailable %ld MiB)", want,
                    cudaGetErrorString(e), cudaGetErrorString(e2), avail_mb);
      }
      p->host = static_cast<char*>(h2);
      p->host_kind = 2;
    } else {
      p->registered_by_us = true;
    }
  }
  void* dptr = nullptr;
  if ((e = cudaHostGetDevicePointer(&dptr, p->host, 0))) {
    destroy(p);
    return cuda_fail(e, "cudaHostGetDevicePointer");
  }
  p->host_dev = static_cast<char*>(dptr);
  p->gran = access_granularity(p);

  p->events.assign(size_t(kEventRing) * (d->num_layers + 1), nullptr);
  for (auto& ev : p->events) {
    if ((e = cudaEventCreate(&ev))) {
      destroy(p);
      return cuda_fail(e, "cudaEventCreate");
    }
  }
  for (auto& op : p->ops) op = {0, 0, 0};
  p->tma_smem = strata::tma_smem_limit();
  p->loads_active = strata::ring_loads_active();   // resolved here, never under stream capture
  if (p->tma_smem > 0 && ((e = strata::tma_prepare(p->tma_smem)) || (e = strata::ring_prepare(p->tma_smem)))) {
    destroy(p);
    return cuda_fail(e, "cudaFuncSetAttribute(TMA smem)");
  }
  strata::ensure_fused(p);   // setup only: keeps allocation and stream creation out of timed calls
  *out = p;
  return STRATA_OK;
}

int strata_unregister_host_pool(strata_pool_t p) {
  if (!p) return STRATA_OK;
  DeviceGuard dg(p->d.device);
  // wait for every operation whose events are still live
  for (const auto& op : p->ops) {
    if (op.ticket && op.l1 > op.l0 && !op.captured) {
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
  return strata::transfer(p, x, reinterpret_cast<cudaStream_t>(stream), ticket, 0);
}

int strata_offload(strata_pool_t p, const strata_xfer* x, strata_stream_t stream, uint64_t* ticket) {
  return strata::transfer(p, x, reinterpret_cast<cudaStream_t>(stream), ticket, 1);
}

namespace {
// A captured operation (its own events, signalled by every replay of its graph); NULL otherwise.
const strata_pool::CapturedOp* captured_op(strata_pool_t p, uint64_t ticket) {
  auto it = p->captured_ops.find(ticket);
  return it == p->captured_ops.end() ? nullptr : &it->second;
}

// Resolves (ticket, layer) to the ring slot; 0 on success.  A captured ticket resolves to slot -1
// once its ring slot has been reused (it never goes stale: its events are its own).
int find_op(strata_pool_t p, uint64_t& ticket, int32_t layer, int& slot) {
  if (!p) return fail(STRATA_ERR_INVALID_ARG, "pool is NULL");
  const uint64_t last = p->next_ticket - 1;
  if (ticket == 0) ticket = last;
  if (const auto* c = ticket ? captured_op(p, ticket) : nullptr) {
    if (layer < c->l0 || layer >= c->l1)
      return fail(STRATA_ERR_INVALID_ARG, "layer %d outside the operation's range [%d,%d)", layer, c->l0, c->l1);
    slot = static_cast<int>(ticket % kEventRing);
    if (p->ops[slot].ticket != ticket) slot = -1;
    return STRATA_OK;
  }
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
  if (const auto* c = captured_op(p, ticket)) {   // the external event every replay records
    *out = reinterpret_cast<strata_event_t>(c->ev[size_t(1 + layer)]);
    return STRATA_OK;
  }
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
  cudaError_t e;
  if (const auto* c = captured_op(p, ticket)) {
    // a consumer captured into the graph waits on the slot's capture-internal event (a graph edge);
    // one outside any capture on the external event the latest replay recorded
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if ((e = cudaStreamIsCapturing(reinterpret_cast<cudaStream_t>(consumer), &cs))) return cuda_fail(e, "cudaStreamIsCapturing");
    if (cs == cudaStreamCaptureStatusNone)
      e = cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(consumer), c->ev[size_t(1 + layer)], 0);
    else if (slot >= 0)
      e = cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(consumer),
                              p->events[size_t(slot) * (p->d.num_layers + 1) + 1 + layer], 0);
    else
      return fail(STRATA_ERR_STALE_TICKET, "captured ticket %llu: its ring slot was reused, so a consumer inside a "
                  "capture can no longer depend on it (wait from outside the capture)", (unsigned long long)ticket);
    return e == cudaSuccess ? STRATA_OK : cuda_fail(e, "cudaStreamWaitEvent");
  }
  // a fused operation's layers (except the last, whose event the caller's stream records) are
  // waited on at their device flag directly, without the side stream's event hop
  if (p->ops[slot].fused && layer + 1 < p->ops[slot].l1) {
    e = strata::wait_fused_layer(p, slot, layer, reinterpret_cast<cudaStream_t>(consumer));
    return e == cudaSuccess ? STRATA_OK : cuda_fail(e, "cuStreamWaitValue32");
  }
  e = cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(consumer),
                          p->events[size_t(slot) * (p->d.num_layers + 1) + 1 + layer], 0);
  return e == cudaSuccess ? STRATA_OK : cuda_fail(e, "cudaStreamWaitEvent");
}

int strata_set_load_quota(strata_pool_t p, int32_t max_ctas, strata_stream_t stream) {
  if (!p) return fail(STRATA_ERR_INVALID_ARG, "pool is NULL");
  if (max_ctas < 0) return fail(STRATA_ERR_INVALID_ARG, "max_ctas = %d < 0", max_ctas);
  strata::DeviceGuard dg(p->d.device);
  if (!strata::ensure_fused(p)) return fail(STRATA_ERR_UNSUPPORTED, "one-launch operations are unavailable on this device");
  const cudaError_t e = strata::set_load_quota(p, max_ctas, reinterpret_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported) return fail(STRATA_ERR_UNSUPPORTED, "cuStreamWriteValue32 is unavailable");
  return e == cudaSuccess ? STRATA_OK : cuda_fail(e, "cuStreamWriteValue32");
}

int strata_layer_elapsed_ms(strata_pool_t p, uint64_t ticket, int32_t layer, float* ms) {
  if (!ms) return fail(STRATA_ERR_INVALID_ARG, "ms is NULL");
  int slot = 0;
  int rc = find_op(p, ticket, layer, slot);
  if (rc) return rc;
  if (const auto* c = captured_op(p, ticket)) {   // the latest replay's external events
    cudaError_t e = cudaEventSynchronize(c->ev[size_t(1 + layer)]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms, c->ev[0], c->ev[size_t(1 + layer)]);
    if (e == cudaSuccess) return STRATA_OK;
    cudaGetLastError();   // the library's own failed call: not left pending on the caller's thread
    return fail(STRATA_ERR_CUDA, "captured ticket %llu: %s (has its graph been replayed?)",
                (unsigned long long)ticket, cudaGetErrorString(e));
  }
  const size_t base = size_t(slot) * (p->d.num_layers + 1);
  cudaError_t e = cudaEventSynchronize(p->events[base + 1 + layer]);
  if (e == cudaSuccess) e = cudaEventElapsedTime(ms, p->events[base], p->events[base + 1 + layer]);
  return e == cudaSuccess ? STRATA_OK : cuda_fail(e, "cudaEventElapsedTime");
}

}  // extern "C"
