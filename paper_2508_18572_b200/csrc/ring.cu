// ring.cu — the ring engine (STRATA_ENGINE_TMA): zero-copy KV load / offload built for a small SM
// quota ("a small number of large CUDA blocks", 2 for loads, 1 for backups).
//
// The host link is crossed by the TMA engine in long runs instead of by LSU requests: the page-first
// host tier keeps a (chunk, layer, K|V) block of C tokens contiguous (§4.2.1), so a
// PIECE — up to R consecutive tokens of one such block — is ONE cp.async.bulk between mapped host
// memory and a shared-memory stage.  The device side of a piece is R token rows at their pages
// (page table): the layout transform is the address arithmetic of that side
// (PAPER.md:289).  One persistent launch covers every layer of the operation; layer l's completion is
// a device flag, published once every CTA has finished its pieces of layer l.
//
//   load    warp 0       producer: one bulk host -> stage copy per piece (or one per row when the
//                        host rows of a piece are strided: a head slice of a wider token-major tier)
//           warps 1..W   scatter: ld.shared.v4 -> st.global.v4 to the rows' pages (16-byte vectors,
//                        U in flight per lane), row addresses from a per-stage table they fill one
//                        piece ahead (page-table index loads issued a piece early)
//   offload warp 0       store: one bulk stage -> host copy per piece; a stage is released when its
//                        store has read shared memory (cp.async.bulk.wait_group.read)
//           warps 1..W   gather: 16-byte cp.async from the rows' pages into the stage, completion
//                        counted on the stage's mbarrier (cp.async.mbarrier.arrive.noinc)
//
// Why on B200 (profiles/r01/tma_probe.jsonl): one TMA warp alone reads mapped host memory at the
// SM zero-copy plateau (51.4 GB/s from ONE SM), while LSU reads need ~1 KiB in flight per warp and
// 1024 threads per SM to reach 42 GB/s.  The stores to the pages stay on the LSU (scattered 2 KiB
// rows; bulk stores would share the TMA unit with the host reads).
#include <cuda_runtime.h>
#include <cstdint>

#include "device.cuh"
#include "internal.h"

namespace strata {
namespace {

using namespace dev;

constexpr int kRingBarBytes = 2 * kRingMaxStages * 8;   // full[16], empty[16]
constexpr int kU = 4;                                   // 16-byte vectors in flight per scatter lane

// [full[16] | empty[16] | row-address table [S][R] | pad to 128 | S stages]
__host__ __device__ constexpr int ring_buf_offset(int stages, int rows) {
  return (kRingBarBytes + stages * rows * 8 + 127) / 128 * 128;
}

struct Piece {
  int32_t r;    // request in the launch table
  int32_t kv;   // 0 K, 1 V
  int32_t j;    // chunk position in the request's chunk list
  int32_t i0;   // first token of the piece (0-based within the request's tokens of this call)
  int32_t n;    // rows (0: an empty tail piece of a partial chunk)
};

__device__ __forceinline__ Piece piece_of(const RingParams& p, int32_t k) {
  const XferParams& x = p.x;
  Piece pc;
  const int32_t seg = k / p.pps;
  const int32_t sub = k - seg * p.pps;
  const int32_t pair = x.nkv == 2 ? (seg >> 1) : seg;
  pc.kv = seg - pair * x.nkv;
  int lo = 0, hi = x.rt.n - 1;   // first request whose chunk positions end after `pair`
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (p.pair_end[mid] > pair) hi = mid; else lo = mid + 1;
  }
  pc.r = lo;
  pc.j = pair - (lo ? p.pair_end[lo - 1] : 0);
  const int32_t oc = x.rt.off_c[lo];
  const int32_t nr = x.rt.tok_end[lo] - (lo ? x.rt.tok_end[lo - 1] : 0);
  const int32_t a = max(0, pc.j * x.C - oc);          // the chunk's first token of this request
  const int32_t b = min(nr, (pc.j + 1) * x.C - oc);   // one past its last
  pc.i0 = a + sub * p.rows;
  pc.n = max(0, min(b - pc.i0, p.rows));
  return pc;
}

// Host address of row 0 of a piece in layer l (page-first chunk; R28 head offset).
__device__ __forceinline__ const char* piece_host(const RingParams& p, const Piece& pc, int32_t hc, int l) {
  const XferParams& x = p.x;
  return x.host + int64_t(hc) * x.chunk_bytes + int64_t(l) * x.nkv * x.kv_off + pc.kv * x.kv_off +
         int64_t(x.rt.off_c[pc.r] + pc.i0 - pc.j * x.C) * x.host_tok_stride + x.host_head_off;
}

// Device row of token i of a piece, split so the page-index load is consumed late: `pg` is the
// loaded page (issued here), `base` the rest of the address (layer-first pool).
struct RowPre {
  int32_t pg;      // -1: no row
  uint64_t base;   // K/V base of the layer + offset in page * token_stride
};
__device__ __forceinline__ RowPre row_pre(const RingParams& p, const Piece& pc, int32_t t, char* kb, char* vb) {
  const XferParams& x = p.x;
  RowPre rp;
  rp.pg = -1;
  rp.base = 0;
  if (t < pc.n) {
    const int32_t pi = x.rt.off_p[pc.r] + pc.i0 + t;
    const int32_t pq = x.p_shift >= 0 ? (pi >> x.p_shift) : pi / x.P;
    rp.pg = __ldg(x.dev_pages + x.rt.page_base[pc.r] + pq);
    rp.base = reinterpret_cast<uint64_t>(pc.kv ? vb : kb) + uint64_t(int64_t(pi - pq * x.P) * x.token_stride);
  }
  return rp;
}
__device__ __forceinline__ uint64_t row_addr(const RingParams& p, const RowPre& rp) {
  return rp.pg < 0 ? 0 : rp.base + uint64_t(int64_t(rp.pg) * p.x.page_stride);
}

__device__ __forceinline__ int piece_row(const RingParams& p, int v) {
  if (p.x.vpt_shift >= 0) return v >> p.x.vpt_shift;
  if (p.piece_magic) return static_cast<int>(__umulhi(static_cast<unsigned>(v), p.piece_magic));
  return v / p.x.vpt;
}

__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(threads) : "memory");
}

// Layer l complete for this arriver: the last of p.arrivals resets the counter (for the op slot's
// next operation, which the host orders after this one) and publishes the epoch.
template <int DIR>
__device__ __forceinline__ void arrive_layer(const RingParams& p, int l) {
  layer_fence<DIR>();
  const uint32_t prev = atomicAdd(p.counters + l, 1u);
  if (prev == static_cast<uint32_t>(p.arrivals - 1)) {
    p.counters[l] = 0;
    layer_fence<DIR>();
    st_release<DIR>(p.flags + l, p.epoch);
  }
}

// Page-index lookahead of the device-side warps: every thread keeps the (page, base) of its row for
// the next kLook pieces in registers, so a piece's page-table loads were issued kLook pieces earlier
// (one piece of lookahead left ~0.6-0.9 us of index latency on each piece's critical path:
// profiles/r02/ring_sweep1.jsonl, 1-CTA rate proportional to the piece size).
constexpr int kLook = 4;

struct RowQueue {
  RowPre r[kLook];
  int32_t n[kLook];
};

__device__ __forceinline__ void rowq_set(const RingParams& p, RowQueue& q, int i, int32_t m, int32_t mine, int t,
                                         char* kb, char* vb) {
  const int G = gridDim.x;
  const Piece pc = m < mine ? piece_of(p, blockIdx.x + m * G) : Piece{0, 0, 0, 0, 0};
  q.r[i] = row_pre(p, pc, t, kb, vb);
  q.n[i] = pc.n;
}
__device__ __forceinline__ void rowq_init(const RingParams& p, RowQueue& q, int32_t mine, int t, char* kb, char* vb) {
#pragma unroll
  for (int i = 0; i < kLook; ++i) rowq_set(p, q, i, i, mine, t, kb, vb);
}
// pops the head (piece m) and issues the index loads of piece m + kLook
__device__ __forceinline__ RowPre rowq_pop(const RingParams& p, RowQueue& q, int32_t m, int32_t mine, int t,
                                           char* kb, char* vb, int& n) {
  const RowPre head = q.r[0];
  n = q.n[0];
#pragma unroll
  for (int i = 0; i + 1 < kLook; ++i) {
    q.r[i] = q.r[i + 1];
    q.n[i] = q.n[i + 1];
  }
  rowq_set(p, q, kLook - 1, m + kLook, mine, t, kb, vb);
  return head;
}

// ---------------------------------------------------------------------------------------------
template <bool CONTIG>
__global__ void __launch_bounds__(32 * (1 + kRingMaxWarps), 1) ring_load_kernel(const __grid_constant__ RingParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XferParams& x = p.x;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kRingMaxStages;
  uint64_t* table = reinterpret_cast<uint64_t*>(smem + kRingBarBytes);   // [S][R] device row addresses
  unsigned char* buf = smem + ring_buf_offset(p.stages, p.rows);
  const int S = p.stages, R = p.rows, SB = p.stage_bytes, tok = x.tok_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, b = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.warps);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const int32_t mine = p.npieces > b ? (p.npieces - 1 - b) / G + 1 : 0;   // this CTA's pieces per layer

  if (warp == 0) {
    // ---------------- producer: host -> stage ----------------
    uint32_t q = 0;
    for (int l = p.l0; l < p.l1; ++l) {
      for (int32_t m0 = 0; m0 < mine; m0 += 32) {
        // lane t decodes piece m0 + t and fetches its host chunk index; the loop below issues them
        const int32_t m = m0 + lane;
        const char* src = nullptr;
        int n = 0;
        if (m < mine) {
          const Piece pc = piece_of(p, b + m * G);
          const int32_t hc = __ldg(x.host_chunks + x.rt.chunk_base[pc.r] + pc.j);
          src = piece_host(p, pc, hc, l);
          n = pc.n;
        }
        const int cnt = min(32, mine - m0);
        for (int t = 0; t < cnt; ++t, ++q) {
          const int s = static_cast<int>(q % S);
          const uint64_t a = __shfl_sync(kFull, reinterpret_cast<uint64_t>(src), t);
          const int nt = __shfl_sync(kFull, n, t);
          if (q >= static_cast<uint32_t>(S)) mbar_wait(&empty[s], ((q / S) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nt * tok));
          __syncwarp();
          unsigned char* st = buf + static_cast<size_t>(s) * SB;
          if (p.host_run) {
            if (lane == 0 && nt) bulk_g2s(st, reinterpret_cast<const void*>(a), static_cast<uint32_t>(nt * tok), &full[s]);
          } else {
            for (int i = lane; i < nt; i += 32)
              bulk_g2s(st + i * tok, reinterpret_cast<const char*>(a) + int64_t(i) * x.host_tok_stride,
                       static_cast<uint32_t>(tok), &full[s]);
          }
        }
      }
    }
  } else {
    // ---------------- scatter warps: stage -> pages ----------------
    const int ct = threadIdx.x - 32, nct = p.warps * 32;
    uint32_t q = 0;
    for (int l = p.l0; l < p.l1; ++l) {
      char* kb = p.kb[l];
      char* vb = p.vb[l];
      RowQueue rq;
      rowq_init(p, rq, mine, ct, kb, vb);
      for (int32_t m = 0; m < mine; ++m, ++q) {
        const int s = static_cast<int>(q % S);
        int n;
        const RowPre cur = rowq_pop(p, rq, m, mine, ct, kb, vb, n);
        if (ct < R) table[s * R + ct] = row_addr(p, cur);
        named_sync(1, nct);
        mbar_wait(&full[s], (q / S) & 1);
        const unsigned char* st = buf + static_cast<size_t>(s) * SB;
        const uint64_t* tab = table + s * R;
        const int nvec = n * x.vpt;
        for (int v0 = ct; v0 < nvec; v0 += nct * kU) {
          int4 val[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int v = v0 + u * nct;
            if (v < nvec) val[u] = ld_shared_v4(st + v * 16);
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int v = v0 + u * nct;
            if (v < nvec) {
              const int row = piece_row(p, v);
              const int w = v - row * x.vpt;
              st_vec(reinterpret_cast<void*>(row_vec<CONTIG>(tab[row], w, x, x.head_stride)), val[u]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (p.counters) {
        __syncwarp();
        if (lane == 0) arrive_layer<0>(p, l);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Offload.  Gather warps copy a piece's rows from their pages into the stage with cp.async (16-byte
// LSU copies that complete asynchronously, no register staging: the bytes in flight are bounded by
// the ring, not by registers) and arrive on full[s] when their copies have landed; warp 0 writes the
// stage to the host run with one cp.async.bulk.  (Gathering with one cp.async.bulk per row as well
// put every small copy on the SM's single TMA unit next to the host stores: 5.6 GB/s at 256-byte
// rows, profiles/r02/ring_sweep1.jsonl.)
template <bool CONTIG>
__global__ void __launch_bounds__(32 * (1 + kRingMaxWarps), 1) ring_offload_kernel(const __grid_constant__ RingParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XferParams& x = p.x;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kRingMaxStages;
  uint64_t* table = reinterpret_cast<uint64_t*>(smem + kRingBarBytes);   // [S][R] device row addresses
  unsigned char* buf = smem + ring_buf_offset(p.stages, p.rows);
  const int S = p.stages, R = p.rows, SB = p.stage_bytes, tok = x.tok_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, b = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 32 * p.warps);   // one cp.async arrive (.noinc) per gather thread
      mbar_init(&empty[s], 1);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const int32_t mine = p.npieces > b ? (p.npieces - 1 - b) / G + 1 : 0;

  if (warp == 0) {
    // ---------------- store: stage -> host run ----------------
    uint32_t q = 0, released = 0;
    for (int l = p.l0; l < p.l1; ++l) {
      for (int32_t m0 = 0; m0 < mine; m0 += 32) {
        const int32_t m = m0 + lane;
        char* dst = nullptr;
        int n = 0;
        if (m < mine) {
          const Piece pc = piece_of(p, b + m * G);
          const int32_t hc = __ldg(x.host_chunks + x.rt.chunk_base[pc.r] + pc.j);
          dst = const_cast<char*>(piece_host(p, pc, hc, l));
          n = pc.n;
        }
        const int cnt = min(32, mine - m0);
        for (int t = 0; t < cnt; ++t, ++q) {
          const int s = static_cast<int>(q % S);
          const uint64_t a = __shfl_sync(kFull, reinterpret_cast<uint64_t>(dst), t);
          const int nt = __shfl_sync(kFull, n, t);
          mbar_wait(&full[s], (q / S) & 1);
          fence_proxy_async_smem();   // the gather's cp.async (generic proxy) writes -> the bulk store
          const unsigned char* st = buf + static_cast<size_t>(s) * SB;
          if (p.host_run) {
            if (lane == 0 && nt) bulk_s2g(reinterpret_cast<void*>(a), st, static_cast<uint32_t>(nt * tok));
          } else {
            for (int i = lane; i < nt; i += 32)
              bulk_s2g(reinterpret_cast<char*>(a) + int64_t(i) * x.host_tok_stride, st + i * tok,
                       static_cast<uint32_t>(tok));
          }
          bulk_commit();
          bulk_wait_read<1>();   // every store but this piece's has read its stage
          __syncwarp();
          for (; released < q; ++released)
            if (lane == 0) mbar_arrive(&empty[released % S]);
        }
      }
      bulk_wait_all();   // layer l's host bytes are written
      __syncwarp();
      for (; released < q; ++released)
        if (lane == 0) mbar_arrive(&empty[released % S]);
      if (p.counters && lane == 0) arrive_layer<1>(p, l);
    }
  } else {
    // ---------------- gather warps: pages -> stage ----------------
    const int gt = threadIdx.x - 32, ngt = p.warps * 32;
    uint32_t q = 0;
    for (int l = p.l0; l < p.l1; ++l) {
      char* kb = p.kb[l];
      char* vb = p.vb[l];
      RowQueue rq;
      rowq_init(p, rq, mine, gt, kb, vb);
      for (int32_t m = 0; m < mine; ++m, ++q) {
        const int s = static_cast<int>(q % S);
        int n;
        const RowPre cur = rowq_pop(p, rq, m, mine, gt, kb, vb, n);
        if (q >= static_cast<uint32_t>(S)) mbar_wait(&empty[s], ((q / S) - 1) & 1);
        if (gt < R) table[s * R + gt] = row_addr(p, cur);
        named_sync(1, ngt);
        unsigned char* st = buf + static_cast<size_t>(s) * SB;
        const uint64_t* tab = table + s * R;
        const int nvec = n * x.vpt;
        for (int v = gt; v < nvec; v += ngt) {
          const int row = piece_row(p, v);
          const int w = v - row * x.vpt;
          cp_async16(st + v * 16, reinterpret_cast<const void*>(row_vec<CONTIG>(tab[row], w, x, x.head_stride)));
        }
        cp_async_arrive_noinc(&full[s]);
      }
    }
  }
}

}  // namespace

int ring_header_bytes(int stages, int rows) { return ring_buf_offset(stages, rows); }

cudaError_t launch_ring(const RingParams& p, int dir, int ctas, cudaStream_t s) {
  const int smem = ring_buf_offset(p.stages, p.rows) + p.stages * p.stage_bytes;
  const bool contig = p.x.head_stride == p.x.head_bytes || p.x.H == 1;
  const int threads = 32 * (1 + p.warps);
  if (dir == 0)
    return contig ? launch_k(ring_load_kernel<true>, ctas, threads, smem, s, p)
                  : launch_k(ring_load_kernel<false>, ctas, threads, smem, s, p);
  return contig ? launch_k(ring_offload_kernel<true>, ctas, threads, smem, s, p)
                : launch_k(ring_offload_kernel<false>, ctas, threads, smem, s, p);
}

cudaError_t ring_prepare(int smem) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(ring_load_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(ring_load_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(ring_offload_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  return cudaFuncSetAttribute(ring_offload_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

}  // namespace strata
