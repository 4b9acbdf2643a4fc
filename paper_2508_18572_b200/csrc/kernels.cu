// kernels.cu — sm_100a kernels of libstrata: the GPU-assisted KV load (host tier -> paged device
// pool) and offload (the inverse scatter), plus the STRATA_VALIDATE index checker.
//
// "instead of invoking standard cudaMemcpyAsync API repetitively with small data transfers, a
//  GPU-assisted I/O job operates by launching a CUDA kernel ... Each thread is responsible for
//  loading a small chunk of data from a source (either GPU global memory or CPU registered pinned
//  memory) into its local register files and then streaming this data to a destination"
//                                                           (§4.2)
// The layout transform (page-first host chunk <-> layer-first paged pool) is address arithmetic on
// each token row (§4.2.1) — row_addr() below.
//
// Kernels of the engines (bit-identical, chosen per call by strata_xfer.engine; api.cpp):
//   ldg_kernel          zero-copy register staging: a warp owns a group of 32 token rows, lane t
//                       fetches row t's indices (one group ahead) and the warp streams the rows
//                       with U independent 16-byte LDG/STG per lane, addresses broadcast by
//                       __shfl_sync.  Also the scatter / gather of the DMA engine (HBM staging).
//   tma_kernel          zero-copy TMA, single warp, bulk copies on both sides of the ring
//                       (STRATA_ENGINE_TMA_BULK).  The ring engine (STRATA_ENGINE_TMA) is ring.cu.
//   ldg_fused_kernel    the LDG engine over every layer of an operation in one launch, per-layer
//                       completion published as device flags.
//   ldg_narrow_kernel   the LDG engine's shape over 8/4/2/1-byte words, for pools whose rows,
//                       strides or bases are not 16-byte multiples (R29).
// Measured on the B200 box (profiles/r01): SM-issued host reads top out at 51.4 GB/s (92.6 % of the
// 55.5 GB/s pinned memcpy) whatever the instruction or cache hint; per SM they scale with resident
// warps (~1 KiB in flight per warp), so the LDG engine uses 1024-thread CTAs and reaches 50.3 GB/s
// with the paper's 2-CTA quota.  HBM sees < 1 % of its bandwidth.
#include <cuda_runtime.h>
#include <cstdint>

#include "device.cuh"
#include "internal.h"

namespace strata {
namespace {

using namespace dev;

// ---------------------------------------------------------------------------------------------
// Index fetch + layout transform for one token row.  Row = (kv, g): kv-major over the launch's
// flat tokens (rows [0,N) are K, [N,2N) are V; a single-buffer pool has only [0,N)), so
// consecutive rows of one chunk are consecutive host bytes.  Returns the host address and the device address of the row's first byte.
__device__ __forceinline__ int find_req(const ReqTable& rt, int32_t g) {
  int lo = 0, hi = rt.n - 1;  // first r with tok_end[r] > g
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (rt.tok_end[mid] > g) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// The index fetch is split in two so kernels can software-pipeline it: row_fetch issues the two
// int32 index loads (page table, chunk list) for a row and returns at once; row_finish, called an
// iteration later when the loads have landed, applies the layout transform.  This keeps the
// index-load latency (~0.5-1 us from L2/HBM) off the critical path of each pipeline iteration.
struct RowIdx {
  int32_t hc, pg;     // host chunk index, device page index (loaded)
  int32_t cr, pr;     // token position inside the chunk / page
  int32_t kv;         // 0 = K row, 1 = V row; -1 = no row
};

__device__ __forceinline__ RowIdx row_fetch(const XferParams& p, int64_t row) {
  RowIdx x;
  x.kv = row >= p.ntok;
  const int32_t g = static_cast<int32_t>(row - (x.kv ? p.ntok : 0));
  const int r = find_req(p.rt, g);
  const int32_t i = g - (r ? p.rt.tok_end[r - 1] : 0);
  const int32_t ci = p.rt.off_c[r] + i;         // position in the request's host chunk list
  const int32_t pi = p.rt.off_p[r] + i;         // position in the request's device page list
  const int32_t cq = p.c_shift >= 0 ? (ci >> p.c_shift) : ci / p.C;
  const int32_t pq = p.p_shift >= 0 ? (pi >> p.p_shift) : pi / p.P;
  x.cr = ci - cq * p.C;
  x.pr = pi - pq * p.P;
  x.hc = __ldg(p.host_chunks + p.rt.chunk_base[r] + cq);
  x.pg = __ldg(p.dev_pages + p.rt.page_base[r] + pq);
  return x;
}

// Row of 16-byte vector idx inside a group of rows (idx < 32 * vpt).
__device__ __forceinline__ int vec_row(const XferParams& p, int idx) {
  if (p.vpt_shift >= 0) return idx >> p.vpt_shift;
  if (p.vpt_magic) return static_cast<int>(__umulhi(static_cast<unsigned>(idx), p.vpt_magic));
  return idx / p.vpt;
}

__device__ __forceinline__ RowIdx row_none() {
  RowIdx x;
  x.hc = x.pg = x.cr = x.pr = 0;
  x.kv = -1;
  return x;
}

__device__ __forceinline__ void row_finish(const XferParams& p, const RowIdx& x, char* kbase, char* vbase,
                                           int64_t layer_off, char*& hp, char*& dp) {
  // host: chunk hc, layer l, kv, token cr, this GPU's first head   (page-first; R28)
  hp = p.host + static_cast<int64_t>(x.hc) * p.chunk_bytes + layer_off + x.kv * p.kv_off +
       static_cast<int64_t>(x.cr) * p.host_tok_stride + p.host_head_off;
  // device: page pg, offset pr of this layer's K/V  (layer-first paged pool)
  dp = (x.kv ? vbase : kbase) + static_cast<int64_t>(x.pg) * p.page_stride +
       static_cast<int64_t>(x.pr) * p.token_stride;
}
__device__ __forceinline__ void row_finish(const XferParams& p, const RowIdx& x, char*& hp, char*& dp) {
  row_finish(p, x, p.kbase, p.vbase, p.layer_off, hp, dp);
}

// ---------------------------------------------------------------------------------------------
// LDG engine.  DIR 0: host -> device, DIR 1: device -> host.  CONTIG: device rows head-contiguous
// (head_stride == D*e), so a device row is tok_bytes contiguous like the host row.
// One row group (rows row0 .. row0 + RG - 1 of this layer's K|V rows) by one warp: lane t holds the
// fetched indices of row t (`cur`); its host and device addresses go to the other lanes by shuffle.
// (ldg_quota_kernel's body; ldg_layer keeps its own inline copy.)
template <int U, bool CONTIG, bool HCONTIG, int DIR>
__device__ __forceinline__ void ldg_group(const XferParams& p, const RowIdx& cur, char* kbase, char* vbase,
                                          int64_t layer_off, int64_t row0, int64_t nrows, int lane) {
  const int nr = static_cast<int>(min(static_cast<int64_t>(p.rows_per_group), nrows - row0));
  char* hp = nullptr;
  char* dp = nullptr;
  if (cur.kv >= 0) row_finish(p, cur, kbase, vbase, layer_off, hp, dp);   // by lane, broadcast below
  const uint64_t my_src = reinterpret_cast<uint64_t>(DIR == 0 ? hp : dp);
  const uint64_t my_dst = reinterpret_cast<uint64_t>(DIR == 0 ? dp : hp);
  const int nvec = nr * p.vpt;
  for (int base = 0; base < nvec; base += 32 * U) {
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int idx = base + j * 32 + lane;
      const int rl = vec_row(p, idx);
      const int w = idx - rl * p.vpt;
      const uint64_t s = __shfl_sync(kFull, my_src, rl & 31);
      if (idx < nvec) {
        const uint64_t a = DIR == 0 ? row_vec<HCONTIG>(s, w, p, p.host_head_stride)
                                    : row_vec<CONTIG>(s, w, p, p.head_stride);
        v[j] = ld_stream(reinterpret_cast<const void*>(a));
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int idx = base + j * 32 + lane;
      const int rl = vec_row(p, idx);
      const int w = idx - rl * p.vpt;
      const uint64_t d = __shfl_sync(kFull, my_dst, rl & 31);
      if (idx < nvec) {
        const uint64_t a = DIR == 0 ? row_vec<CONTIG>(d, w, p, p.head_stride)
                                    : row_vec<HCONTIG>(d, w, p, p.host_head_stride);
        st_vec(reinterpret_cast<void*>(a), v[j]);
      }
    }
  }
}

// Indices of row `lane` of group gi (row_none past the end).
__device__ __forceinline__ RowIdx ldg_fetch(const XferParams& p, int64_t gi, int64_t ngroups, int64_t nrows, int lane) {
  const int64_t row = gi * p.rows_per_group + lane;
  return (gi < ngroups && lane < p.rows_per_group && row < nrows) ? row_fetch(p, row) : row_none();
}

// One layer of the LDG engine for this warp: groups warp, warp + nwarps, ...  `nx` holds the
// already-fetched indices of the warp's first group (identical for every layer).
template <int U, bool CONTIG, bool HCONTIG, int DIR>
__device__ __forceinline__ void ldg_layer(const XferParams& p, char* kbase, char* vbase, int64_t layer_off,
                                          RowIdx nx, int64_t warp, int64_t nwarps, int lane) {
  const int64_t nrows = static_cast<int64_t>(p.nkv) * p.ntok;
  const int RG = p.rows_per_group;
  const int64_t ngroups = (nrows + RG - 1) / RG;
  // lane t fetches row t of the group; the next group's fetch is issued before this group's data
  // loads so its latency hides under them.  (The body is ldg_group's, kept inline here: the measured
  // default kernel — folding it into the shared helper cost 1.6 % of its rate, profiles/r02/final5.)
  auto fetch = [&](int64_t gi) {
    const int64_t row = gi * RG + lane;
    return (gi < ngroups && lane < RG && row < nrows) ? row_fetch(p, row) : row_none();
  };
  for (int64_t gi = warp; gi < ngroups; gi += nwarps) {
    const int64_t row0 = gi * RG;
    const int nr = static_cast<int>(min(static_cast<int64_t>(RG), nrows - row0));
    const RowIdx cur = nx;
    nx = fetch(gi + nwarps);
    char* hp = nullptr;
    char* dp = nullptr;
    if (cur.kv >= 0) row_finish(p, cur, kbase, vbase, layer_off, hp, dp);   // by lane, broadcast below
    const uint64_t my_src = reinterpret_cast<uint64_t>(DIR == 0 ? hp : dp);
    const uint64_t my_dst = reinterpret_cast<uint64_t>(DIR == 0 ? dp : hp);
    const int nvec = nr * p.vpt;
    for (int base = 0; base < nvec; base += 32 * U) {
      int4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int idx = base + j * 32 + lane;
        const int rl = vec_row(p, idx);
        const int w = idx - rl * p.vpt;
        const uint64_t s = __shfl_sync(kFull, my_src, rl & 31);
        if (idx < nvec) {
          const uint64_t a = DIR == 0 ? row_vec<HCONTIG>(s, w, p, p.host_head_stride)
                                      : row_vec<CONTIG>(s, w, p, p.head_stride);
          v[j] = ld_stream(reinterpret_cast<const void*>(a));
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int idx = base + j * 32 + lane;
        const int rl = vec_row(p, idx);
        const int w = idx - rl * p.vpt;
        const uint64_t d = __shfl_sync(kFull, my_dst, rl & 31);
        if (idx < nvec) {
          const uint64_t a = DIR == 0 ? row_vec<CONTIG>(d, w, p, p.head_stride)
                                      : row_vec<HCONTIG>(d, w, p, p.host_head_stride);
          st_vec(reinterpret_cast<void*>(a), v[j]);
        }
      }
    }
  }
}

__device__ __forceinline__ RowIdx ldg_first(const XferParams& p, int64_t warp, int lane) {
  const int64_t nrows = static_cast<int64_t>(p.nkv) * p.ntok;
  const int64_t ngroups = (nrows + p.rows_per_group - 1) / p.rows_per_group;
  const int64_t row = warp * p.rows_per_group + lane;
  return (warp < ngroups && lane < p.rows_per_group && row < nrows) ? row_fetch(p, row) : row_none();
}

// LDG engine, one layer per launch.  DIR 0: host -> device, DIR 1: device -> host.  CONTIG: device
// rows head-contiguous (head_stride == D*e), so a device row is tok_bytes contiguous like the host row.
template <int U, bool CONTIG, bool HCONTIG, int DIR>
__global__ void __launch_bounds__(U >= 8 ? 512 : 1024, 1) ldg_kernel(const __grid_constant__ XferParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  ldg_layer<U, CONTIG, HCONTIG, DIR>(p, p.kbase, p.vbase, p.layer_off, ldg_first(p, warp, lane), warp, nwarps, lane);
}

// LDG engine, every layer of the operation in ONE launch (the persistent variant):
// warps flow from layer l into layer l+1 without a kernel boundary, and layer l's completion is a
// device flag.  Each warp, after its share of layer l, fences its stores (system scope: offload
// rows land in host memory) and arrives on counters[l]; the last arriver resets the counter for the
// slot's next operation and publishes `epoch` to flags[l].  The host side turns each flag into the
// layer's CUDA event with cuStreamWaitValue32 + cudaEventRecord on the op slot's side stream.
// Loads land in HBM and are consumed by GPU work: GPU-scope fences.  Offloads land in host memory,
// which the host may read after the event: system scope.
template <int U, bool CONTIG, bool HCONTIG, int DIR>
__global__ void __launch_bounds__(U >= 8 ? 512 : 1024, 1) ldg_fused_kernel(const __grid_constant__ FusedParams fp) {
  const XferParams& p = fp.x;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const RowIdx first = ldg_first(p, warp, lane);
  const int64_t layer_step = static_cast<int64_t>(p.nkv) * p.kv_off;
  if (DIR == 0 && fp.loads_active && threadIdx.x == 0) atomicAdd(fp.loads_active, 1u);   // ring offloads yield
  for (int l = fp.l0; l < fp.l1; ++l) {
    ldg_layer<U, CONTIG, HCONTIG, DIR>(p, fp.kb[l], fp.vb[l], int64_t(l) * layer_step, first, warp, nwarps, lane);
    __syncwarp();
    if (lane == 0) {
      layer_fence<DIR>();
      const uint32_t prev = atomicAdd(fp.counters + l, 1u);
      if (prev == static_cast<uint32_t>(fp.total_warps - 1)) {
        fp.counters[l] = 0;
        layer_fence<DIR>();
        st_release<DIR>(fp.flags + l, fp.epoch);
      }
    }
  }
  if (DIR == 0 && fp.loads_active) {
    __syncthreads();
    if (threadIdx.x == 0) atomicSub(fp.loads_active, 1u);
  }
}

// Decode-aware quota (NEXT-1, strata_set_load_quota): the fused LDG load with DYNAMIC row-group
// assignment.  Warps take the groups of layer l from next[l] (one atomicAdd per group, taken one
// group ahead so its index fetch hides under the current group's host loads).  While the pool's
// quota word q is > 0, CTAs with blockIdx.x >= q take no new group: their warps wait — no host reads
// in flight from their SMs, the lever that lowers co-running decode's slowdown —
// until the cap is lifted or every group of the layer is taken; the other CTAs move those rows.
// Layer completion counts warps as in ldg_fused_kernel; the last arriver also resets next[l].
__device__ __forceinline__ int32_t ld_relaxed_sys(const int32_t* a) {
  int32_t v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ int64_t quota_grab(uint32_t* next, const int32_t* quota, int64_t ngroups, int lane) {
  uint32_t g = 0;
  if (lane == 0) {
    for (;;) {
      const int32_t q = ld_relaxed_sys(quota);
      if (q <= 0 || static_cast<int32_t>(blockIdx.x) < q) {
        g = atomicAdd(next, 1u);
        break;
      }
      if (static_cast<int64_t>(ld_relaxed_gpu(next)) >= ngroups) {   // nothing left to take this layer
        g = static_cast<uint32_t>(ngroups);
        break;
      }
      __nanosleep(2000);
    }
  }
  return static_cast<int64_t>(__shfl_sync(kFull, g, 0));
}

template <int U, bool CONTIG, bool HCONTIG>
__global__ void __launch_bounds__(U >= 8 ? 512 : 1024, 1) ldg_quota_kernel(const __grid_constant__ FusedParams fp) {
  const XferParams& p = fp.x;
  const int lane = threadIdx.x & 31;
  const int64_t nrows = static_cast<int64_t>(p.nkv) * p.ntok;
  const int RG = p.rows_per_group;
  const int64_t ngroups = (nrows + RG - 1) / RG;
  const int64_t layer_step = static_cast<int64_t>(p.nkv) * p.kv_off;
  const int total_warps = fp.total_warps;
  if (fp.loads_active && threadIdx.x == 0) atomicAdd(fp.loads_active, 1u);   // ring offloads yield
  for (int l = fp.l0; l < fp.l1; ++l) {
    int64_t gi = quota_grab(fp.next + l, fp.quota, ngroups, lane);
    RowIdx nx = ldg_fetch(p, gi, ngroups, nrows, lane);
    while (gi < ngroups) {
      const int64_t gn = quota_grab(fp.next + l, fp.quota, ngroups, lane);
      const RowIdx cur = nx;
      nx = ldg_fetch(p, gn, ngroups, nrows, lane);
      ldg_group<U, CONTIG, HCONTIG, 0>(p, cur, fp.kb[l], fp.vb[l], int64_t(l) * layer_step, gi * RG, nrows, lane);
      gi = gn;
    }
    __syncwarp();
    if (lane == 0) {
      layer_fence<0>();
      const uint32_t prev = atomicAdd(fp.counters + l, 1u);
      if (prev == static_cast<uint32_t>(total_warps - 1)) {
        fp.counters[l] = 0;
        fp.next[l] = 0;   // every warp has taken its last group of layer l
        layer_fence<0>();
        st_release<0>(fp.flags + l, fp.epoch);
      }
    }
  }
  if (fp.loads_active) {
    __syncthreads();
    if (threadIdx.x == 0) atomicSub(fp.loads_active, 1u);
  }
}

constexpr int kTmaHeader = 16 * kTmaMaxStages;           // mbarriers: full[32], empty[32]

__host__ __device__ constexpr int tma_table_bytes(int stages) { return stages * 32 * 12; }
__host__ __device__ constexpr int tma_buf_offset(int stages) {
  return (kTmaHeader + tma_table_bytes(stages) + 127) / 128 * 128;
}

// One warp per CTA.  Pieces of `tma_rows` consecutive token rows are distributed round-robin over
// CTAs; piece k of this CTA uses stage k % S.
template <int DIR, bool CONTIG>
__global__ void __launch_bounds__(32, 1) tma_kernel(const __grid_constant__ XferParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.tma_stages;
  const int T = p.tma_rows;
  const int SB = p.tma_stage_bytes;
  const int tok = p.tok_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* tab_addr = reinterpret_cast<uint64_t*>(smem + kTmaHeader);              // [S][32]
  int32_t* tab_len = reinterpret_cast<int32_t*>(smem + kTmaHeader + S * 32 * 8);   // [S][32]
  unsigned char* buf = smem + tma_buf_offset(S);
  const int lane = threadIdx.x;

  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    mbar_init_fence();
  }
  __syncwarp();

  const int64_t nrows = static_cast<int64_t>(p.nkv) * p.ntok;
  const int64_t npieces = (nrows + T - 1) / T;
  const int64_t my = npieces > blockIdx.x ? (npieces - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  // index fetch for piece k (issued one pipeline step ahead of its use, see row_fetch)
  auto fetch = [&](int64_t k) {
    const int64_t row = (blockIdx.x + k * gridDim.x) * T + lane;
    return (k < my && lane < T && row < nrows) ? row_fetch(p, row) : row_none();
  };

  auto issue = [&](int64_t k, const RowIdx& x) {
    const int s = static_cast<int>(k % S);
    const bool valid = x.kv >= 0;
    char* hp = nullptr;
    char* dp = nullptr;
    if (valid) row_finish(p, x, hp, dp);
    // host-side runs: a lane starts a run unless its row directly follows the previous lane's
    const uint64_t hprev = __shfl_up_sync(kFull, reinterpret_cast<uint64_t>(hp), 1);
    const int vprev = __shfl_up_sync(kFull, static_cast<int>(valid), 1);
    const bool head = valid && !(lane > 0 && vprev && hprev + tok == reinterpret_cast<uint64_t>(hp));
    const unsigned heads = __ballot_sync(kFull, head);
    const int nvalid = __popc(__ballot_sync(kFull, valid));
    const unsigned later = lane == 31 ? 0u : (heads & ~((2u << lane) - 1u));
    const int run = (later ? __ffs(later) - 1 : nvalid) - lane;
    unsigned char* st = buf + static_cast<size_t>(s) * SB;
    if (DIR == 0) {
      tab_addr[s * 32 + lane] = reinterpret_cast<uint64_t>(dp);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nvalid * tok));
      __syncwarp();
      if (head) bulk_g2s(st + lane * tok, hp, static_cast<uint32_t>(run * tok), &full[s]);
    } else {
      tab_addr[s * 32 + lane] = reinterpret_cast<uint64_t>(hp);
      tab_len[s * 32 + lane] = head ? run : 0;
      if (lane == 0) mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nvalid * tok));
      __syncwarp();
      if (valid) {
        if (CONTIG) {
          bulk_g2s(st + lane * tok, dp, static_cast<uint32_t>(tok), &full[s]);
        } else {
          for (int h = 0; h < p.H; ++h)
            bulk_g2s(st + lane * tok + h * p.head_bytes, dp + h * p.head_stride,
                     static_cast<uint32_t>(p.head_bytes), &full[s]);
        }
      }
    }
  };

  auto consume = [&](int64_t k) {
    const int s = static_cast<int>(k % S);
    mbar_wait(&full[s], static_cast<uint32_t>((k / S) & 1));
    unsigned char* st = buf + static_cast<size_t>(s) * SB;
    if (DIR == 0) {
      char* dp = reinterpret_cast<char*>(tab_addr[s * 32 + lane]);
      if (dp) {
        if (CONTIG) {
          bulk_s2g(dp, st + lane * tok, static_cast<uint32_t>(tok));
        } else {
          for (int h = 0; h < p.H; ++h)
            bulk_s2g(dp + h * p.head_stride, st + lane * tok + h * p.head_bytes,
                     static_cast<uint32_t>(p.head_bytes));
        }
      }
    } else {
      const int run = tab_len[s * 32 + lane];
      if (run) bulk_s2g(reinterpret_cast<char*>(tab_addr[s * 32 + lane]), st + lane * tok,
                        static_cast<uint32_t>(run * tok));
    }
    bulk_commit();
  };

  const int64_t pro = my < S ? my : S;
  RowIdx nx = fetch(0);
  for (int64_t k = 0; k < pro; ++k) {
    const RowIdx cur = nx;
    nx = fetch(k + 1);
    issue(k, cur);
  }
  for (int64_t k = 0; k < my; ++k) {
    consume(k);
    // refill the stage piece k-1 used once its stores have read shared memory
    if (k >= 1 && k - 1 + S < my) {
      const RowIdx cur = nx;          // fetched one step ago: piece k-1+S
      nx = fetch(k + S);
      bulk_wait_read<1>();
      __syncwarp();
      issue(k - 1 + S, cur);
    }
  }
  bulk_wait_all();
}

// ---------------------------------------------------------------------------------------------
// Narrow LDG kernel (R29): pools whose rows, strides or bases are not 16-byte multiples.  Same
// shape as the LDG engine: a warp owns a group of 32 rows, lane t fetches row t's indices one group
// ahead, and the warp streams the group's W-byte words (W = the pool's access granularity: 8, 4, 2
// or 1) with 4 independent loads per lane, row addresses broadcast by __shfl_sync; word -> (row,
// head, offset) by multiply-high when the divisors allow it.
template <int W>
struct Word;
template <> struct Word<8> { using T = unsigned long long; };
template <> struct Word<4> { using T = unsigned int; };
template <> struct Word<2> { using T = unsigned short; };
template <> struct Word<1> { using T = unsigned char; };

__device__ __forceinline__ int div_by(int n, int d, uint32_t magic) {
  return magic ? static_cast<int>(__umulhi(static_cast<unsigned>(n), magic)) : n / d;
}

template <int W, int DIR>
__global__ void __launch_bounds__(1024) ldg_narrow_kernel(const __grid_constant__ XferParams p) {
  using T = typename Word<W>::T;
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t nrows = static_cast<int64_t>(p.nkv) * p.ntok;
  const int64_t ngroups = (nrows + 31) / 32;
  const int wpr = p.wpr, wph = p.wph;
  const bool dcont = p.head_stride == p.head_bytes || p.H == 1;
  const bool hcont = p.host_head_stride == p.head_bytes || p.H == 1;
  const bool scont = DIR == 0 ? hcont : dcont, tcont = DIR == 0 ? dcont : hcont;
  const int64_t sstride = DIR == 0 ? p.host_head_stride : p.head_stride;
  const int64_t tstride = DIR == 0 ? p.head_stride : p.host_head_stride;
  auto word_addr = [&](uint64_t base, int w, bool cont, int64_t stride) {
    if (cont) return base + static_cast<uint64_t>(w) * W;
    const int h = div_by(w, wph, p.wph_magic);
    return base + h * stride + static_cast<uint64_t>(w - h * wph) * W;
  };
  auto fetch = [&](int64_t gi) {
    const int64_t row = gi * 32 + lane;
    return (gi < ngroups && row < nrows) ? row_fetch(p, row) : row_none();
  };
  RowIdx nx = fetch(warp);
  for (int64_t gi = warp; gi < ngroups; gi += nwarps) {
    const RowIdx cur = nx;
    nx = fetch(gi + nwarps);
    char* hp = nullptr;
    char* dp = nullptr;
    if (cur.kv >= 0) row_finish(p, cur, hp, dp);
    const uint64_t my_src = reinterpret_cast<uint64_t>(DIR == 0 ? hp : dp);
    const uint64_t my_dst = reinterpret_cast<uint64_t>(DIR == 0 ? dp : hp);
    const int nr = static_cast<int>(min(static_cast<int64_t>(32), nrows - gi * 32));
    const int total = nr * wpr;
    for (int base = 0; base < total; base += 32 * U) {
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * 32 + lane;
        const int r = div_by(idx, wpr, p.wpr_magic);
        const uint64_t sb = __shfl_sync(kFull, my_src, r & 31);
        if (idx < total) v[u] = __ldg(reinterpret_cast<const T*>(word_addr(sb, idx - r * wpr, scont, sstride)));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * 32 + lane;
        const int r = div_by(idx, wpr, p.wpr_magic);
        const uint64_t db = __shfl_sync(kFull, my_dst, r & 31);
        if (idx < total) *reinterpret_cast<T*>(word_addr(db, idx - r * wpr, tcont, tstride)) = v[u];
      }
    }
  }
}

template <int DIR>
cudaError_t ldg_narrow_launch(const XferParams& p, int ctas, int threads, cudaStream_t s) {
  switch (p.gran) {
    case 8: return launch_k(ldg_narrow_kernel<8, DIR>, ctas, threads, 0, s, p);
    case 4: return launch_k(ldg_narrow_kernel<4, DIR>, ctas, threads, 0, s, p);
    case 2: return launch_k(ldg_narrow_kernel<2, DIR>, ctas, threads, 0, s, p);
    default: return launch_k(ldg_narrow_kernel<1, DIR>, ctas, threads, 0, s, p);
  }
}

// ---------------------------------------------------------------------------------------------
__global__ void validate_kernel(const __grid_constant__ ValidateParams v) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < v.ntok; g += stride) {
    const int32_t gg = static_cast<int32_t>(g);
    int lo = 0, hi = v.rt.n - 1;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (v.rt.tok_end[mid] > gg) hi = mid; else lo = mid + 1;
    }
    const int r = lo;
    const int32_t i = gg - (r ? v.rt.tok_end[r - 1] : 0);
    const int64_t ci = static_cast<int64_t>(v.rt.off_c[r]) + i;
    const int64_t pi = static_cast<int64_t>(v.rt.off_p[r]) + i;
    const int64_t cidx = v.rt.chunk_base[r] + ci / v.C;
    const int64_t pidx = v.rt.page_base[r] + pi / v.P;
    if ((v.chunks_len > 0 && cidx >= v.chunks_len) || (v.pages_len > 0 && pidx >= v.pages_len)) {
      atomicOr(v.err, 1);
      continue;
    }
    const int64_t hc = v.host_chunks[cidx];
    const int64_t pg = v.dev_pages[pidx];
    if (hc < 0 || hc >= v.num_chunks || pg < 0 || pg >= v.num_pages) {
      atomicOr(v.err, 1);
      continue;
    }
    const int64_t key = v.dir == 0 ? pg * v.P + pi % v.P : hc * v.C + ci % v.C;
    const uint32_t bit = 1u << (key & 31);
    const uint32_t old = atomicOr(v.bitmap + (key >> 5), bit);
    if (old & bit) atomicOr(v.err, 2);
  }
}

template <int U, int DIR>
cudaError_t ldg_launch(const XferParams& p, bool contig, bool hcontig, int ctas, int threads, cudaStream_t s) {
  if (contig && hcontig) return launch_k(ldg_kernel<U, true, true, DIR>, ctas, threads, 0, s, p);
  else if (contig) return launch_k(ldg_kernel<U, true, false, DIR>, ctas, threads, 0, s, p);
  else if (hcontig) return launch_k(ldg_kernel<U, false, true, DIR>, ctas, threads, 0, s, p);
  else return launch_k(ldg_kernel<U, false, false, DIR>, ctas, threads, 0, s, p);
}

template <int U, int DIR>
cudaError_t ldg_fused_launch(const FusedParams& p, bool contig, bool hcontig, int ctas, int threads, cudaStream_t s) {
  if (DIR == 0 && p.quota) {
    if (contig && hcontig) return launch_k(ldg_quota_kernel<U, true, true>, ctas, threads, 0, s, p);
    else if (contig) return launch_k(ldg_quota_kernel<U, true, false>, ctas, threads, 0, s, p);
    else if (hcontig) return launch_k(ldg_quota_kernel<U, false, true>, ctas, threads, 0, s, p);
    else return launch_k(ldg_quota_kernel<U, false, false>, ctas, threads, 0, s, p);
  }
  if (contig && hcontig) return launch_k(ldg_fused_kernel<U, true, true, DIR>, ctas, threads, 0, s, p);
  else if (contig) return launch_k(ldg_fused_kernel<U, true, false, DIR>, ctas, threads, 0, s, p);
  else if (hcontig) return launch_k(ldg_fused_kernel<U, false, true, DIR>, ctas, threads, 0, s, p);
  else return launch_k(ldg_fused_kernel<U, false, false, DIR>, ctas, threads, 0, s, p);
}

template <int DIR, bool CONTIG>
cudaError_t tma_launch(const XferParams& p, int ctas, cudaStream_t s) {
  const int smem = tma_buf_offset(p.tma_stages) + p.tma_stages * p.tma_stage_bytes;
  return launch_k(tma_kernel<DIR, CONTIG>, ctas, 32, smem, s, p);
}

}  // namespace

// device / host rows contiguous: heads adjacent (or a single head) on that side
static bool dev_contig(const XferParams& p) { return p.head_stride == p.head_bytes || p.H == 1; }
static bool host_contig(const XferParams& p) { return p.host_head_stride == p.head_bytes || p.H == 1; }

cudaError_t launch_ldg(const XferParams& p, int dir, int ctas, int threads, int unroll, cudaStream_t s) {
  if (p.gran < 16) return dir == 0 ? ldg_narrow_launch<0>(p, ctas, threads, s) : ldg_narrow_launch<1>(p, ctas, threads, s);
  const bool contig = dev_contig(p), hcontig = host_contig(p);
  if (threads > 512) unroll = 4;  // U=8 needs > 64 registers per thread
  if (unroll == 4) return dir == 0 ? ldg_launch<4, 0>(p, contig, hcontig, ctas, threads, s)
                                   : ldg_launch<4, 1>(p, contig, hcontig, ctas, threads, s);
  if (unroll == 8) return dir == 0 ? ldg_launch<8, 0>(p, contig, hcontig, ctas, threads, s)
                                   : ldg_launch<8, 1>(p, contig, hcontig, ctas, threads, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_ldg_fused(const FusedParams& p, int dir, int ctas, int threads, cudaStream_t s) {
  const bool contig = dev_contig(p.x), hcontig = host_contig(p.x);
  if (threads > 512) return dir == 0 ? ldg_fused_launch<4, 0>(p, contig, hcontig, ctas, threads, s)
                                     : ldg_fused_launch<4, 1>(p, contig, hcontig, ctas, threads, s);
  return dir == 0 ? ldg_fused_launch<8, 0>(p, contig, hcontig, ctas, threads, s)
                  : ldg_fused_launch<8, 1>(p, contig, hcontig, ctas, threads, s);
}

cudaError_t launch_tma(const XferParams& p, int dir, int ctas, cudaStream_t s) {
  const bool contig = dev_contig(p);
  if (dir == 0) return contig ? tma_launch<0, true>(p, ctas, s) : tma_launch<0, false>(p, ctas, s);
  return contig ? tma_launch<1, true>(p, ctas, s) : tma_launch<1, false>(p, ctas, s);
}

cudaError_t launch_validate(const ValidateParams& v, cudaStream_t s) {
  const int threads = 256;
  int64_t blocks = (v.ntok + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  if (blocks > 1184) blocks = 1184;
  return launch_k(validate_kernel, static_cast<int>(blocks), threads, 0, s, v);
}

int tma_smem_limit() {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
  return optin;
}

int tma_header_bytes(int stages) { return tma_buf_offset(stages); }

cudaError_t tma_prepare(int smem) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(tma_kernel<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(tma_kernel<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(tma_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  return cudaFuncSetAttribute(tma_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

}  // namespace strata
