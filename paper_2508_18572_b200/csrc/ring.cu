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
//                        U in flight per lane); warp w owns pieces w, w+W, ... and loads their
//                        page-table entries two of its pieces ahead
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

constexpr int kRingBarBytes = 2 * kRingMaxStages * 8 + kRingMaxStages * 4;   // full[16], empty[16], pad[16]
constexpr int kU = 4;                                   // 16-byte vectors in flight per scatter lane

// Load CTAs running on this device (ring loads and fused LDG loads of all pools of the process): ring
// offloads pace their host stores while it is non-zero (RingParams::pace_ps_per_byte).
__device__ unsigned int g_loads_active;

// [full[16] | empty[16] | pad[16] (narrow rows: host-run offset in its 16-byte unit) | pad to 128 | S stages]
__host__ __device__ constexpr int ring_buf_offset() { return (kRingBarBytes + 127) / 128 * 128; }

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

// Device-side warps own whole PIECES: the CTA's piece q (its sequence number over the operation) goes
// to warp q % W, which moves all of its rows (lane j holds the (page, base) of rows j and j + 32;
// R <= 64).  The host side makes W divide the ring depth S, so stage s is always drained (load) or
// filled (offload) by warp s % W: a warp then waits on each of its stages' barriers one phase at a
// time, never two phases ahead (mbarrier parity waits cannot tell phase k from phase k + 2).  Every warp runs its
// own pieces' latency chains (page-table loads issued kLook of its pieces early, the stage wait, the
// row loop), so W pieces drain at once.  (All warps on every piece, with a shared row-address table
// and a named barrier per piece, left the 1-CTA kernel issue-latency bound at ~27-37 GB/s:
// profiles/r02/ncu_ring_load_1cta_v1.txt, ring_sweep4.jsonl.)
constexpr int kLook = 2;
constexpr int kRowsPerLane = kRingMaxRows / 32;

struct RowQueue {
  RowPre r[kLook][kRowsPerLane];
  int32_t n[kLook];
};

__device__ __forceinline__ void rowq_set(const RingParams& p, RowQueue& q, int i, int32_t m, int32_t mine, int lane,
                                         char* kb, char* vb) {
  const int G = gridDim.x;
  const Piece pc = m < mine ? piece_of(p, blockIdx.x + m * G) : Piece{0, 0, 0, 0, 0};
#pragma unroll
  for (int c = 0; c < kRowsPerLane; ++c) q.r[i][c] = row_pre(p, pc, lane + 32 * c, kb, vb);
  q.n[i] = pc.n;
}
// warp wi's pieces of a layer: m = wi, wi + W, ...; queue slot i holds the warp's i-th next piece
__device__ __forceinline__ void rowq_init(const RingParams& p, RowQueue& q, int32_t m0, int32_t mine, int lane,
                                          char* kb, char* vb) {
#pragma unroll
  for (int i = 0; i < kLook; ++i) rowq_set(p, q, i, m0 + i * p.warps, mine, lane, kb, vb);
}
// pops the head (piece m) and issues the index loads of the warp's piece kLook ahead
__device__ __forceinline__ void rowq_pop(const RingParams& p, RowQueue& q, int32_t m, int32_t mine, int lane,
                                         char* kb, char* vb, uint64_t (&addr)[kRowsPerLane], int& n) {
#pragma unroll
  for (int c = 0; c < kRowsPerLane; ++c) addr[c] = row_addr(p, q.r[0][c]);
  n = q.n[0];
#pragma unroll
  for (int i = 0; i + 1 < kLook; ++i) {
#pragma unroll
    for (int c = 0; c < kRowsPerLane; ++c) q.r[i][c] = q.r[i + 1][c];
    q.n[i] = q.n[i + 1];
  }
  rowq_set(p, q, kLook - 1, m + kLook * p.warps, mine, lane, kb, vb);
}

// Row j's device address, held by lane j % 32 in slot j / 32.  Lanes may ask for rows of different
// slots in one instruction (narrow rows whose vector count is not a power of two: a group of 32 / vpt
// rows can straddle row 32), so every slot is shuffled and the lane keeps its own.
__device__ __forceinline__ uint64_t row_base(const uint64_t (&addr)[kRowsPerLane], int j) {
  uint64_t v = 0;
#pragma unroll
  for (int c = 0; c < kRowsPerLane; ++c) {
    const uint64_t t = __shfl_sync(kFull, addr[c], j & 31);
    if ((j >> 5) == c) v = t;
  }
  return v;
}

// Every (row, 16-byte vector) of one piece by one warp.  Wide rows (vpt >= 32): one row at a time,
// lane c covers vectors c, c+32, ...; narrow rows: 32 / vpt rows per instruction, lane = (row slot,
// vector).  kU vectors per lane are batched so their shared / global accesses overlap.
//   DIR 0 (load):    stage -> registers -> page rows (ld.shared.v4 / st.global.v4)
//   DIR 1 (offload): page rows -> stage (cp.async, completion counted on the stage's barrier)
template <bool CONTIG, int DIR>
__device__ __forceinline__ void piece_rows(const RingParams& p, int lane, int n, const uint64_t (&addr)[kRowsPerLane],
                                           unsigned char* st) {
  const XferParams& x = p.x;
  const int vpt = x.vpt, tok = x.tok_bytes;
  if (vpt >= 32) {
    for (int j = 0; j < n; ++j) {
      const uint64_t base = row_base(addr, j);
      unsigned char* srow = st + j * tok;
      for (int c0 = 0; c0 < vpt; c0 += 32 * kU) {
        if (DIR == 0) {
          int4 val[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int c = c0 + u * 32 + lane;
            if (c < vpt) val[u] = ld_shared_v4(srow + c * 16);
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int c = c0 + u * 32 + lane;
            if (c < vpt) st_vec(reinterpret_cast<void*>(row_vec<CONTIG>(base, c, x, x.head_stride)), val[u]);
          }
        } else {
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int c = c0 + u * 32 + lane;
            if (c < vpt) cp_async16(srow + c * 16, reinterpret_cast<const void*>(row_vec<CONTIG>(base, c, x, x.head_stride)));
          }
        }
      }
    }
  } else {
    const int rpi = 32 / vpt;             // rows per warp instruction
    const int lr = lane / vpt, lc = lane - lr * vpt;
    const bool on = lr < rpi;
    for (int j0 = 0; j0 < n; j0 += rpi * kU) {
      int4 val[kU];
      uint64_t dst[kU];
      bool ok[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = j0 + u * rpi + lr;
        const uint64_t base = row_base(addr, j & (kRingMaxRows - 1));
        ok[u] = on && j < n;
        dst[u] = row_vec<CONTIG>(base, lc, x, x.head_stride);
        unsigned char* sv = st + j * tok + lc * 16;
        if (DIR == 0) {
          if (ok[u]) val[u] = ld_shared_v4(sv);
        } else {
          if (ok[u]) cp_async16(sv, reinterpret_cast<const void*>(dst[u]));
        }
      }
      if (DIR == 0) {
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (ok[u]) st_vec(reinterpret_cast<void*>(dst[u]), val[u]);
      }
    }
  }
}

// Load variant (p.bulk_store): the piece's rows leave the stage as cp.async.bulk stores, one per run of
// rows that are adjacent on the device (a page of P >= 2 tokens) — fewer, larger requests on the SM's
// path to L2 than 16-byte st.global (which the 1-CTA load saturates: profiles/r02/ncu_ring_load_1cta_v4.txt).
template <bool CONTIG>
__device__ __forceinline__ void piece_rows_bulk(const RingParams& p, int lane, int n, const uint64_t (&addr)[kRowsPerLane],
                                                unsigned char* st) {
  const XferParams& x = p.x;
  const int tok = x.tok_bytes;
#pragma unroll
  for (int c = 0; c < kRowsPerLane; ++c) {
    if (32 * c >= n) break;
    const int j = lane + 32 * c;
    const uint64_t a = addr[c];
    if (CONTIG) {
      const uint64_t prev = __shfl_up_sync(kFull, a, 1);
      const bool head = j < n && !(lane > 0 && prev && prev + tok == a);
      const unsigned heads = __ballot_sync(kFull, head);
      const int lim = min(32, n - 32 * c);
      const unsigned later = lane == 31 ? 0u : (heads & ~((2u << lane) - 1u));
      const int run = (later ? __ffs(later) - 1 : lim) - lane;
      if (head) bulk_s2g(reinterpret_cast<void*>(a), st + j * tok, static_cast<uint32_t>(run * tok));
    } else if (j < n) {
      for (int h = 0; h < x.H; ++h)
        bulk_s2g(reinterpret_cast<char*>(a) + int64_t(h) * x.head_stride, st + j * tok + h * x.head_bytes,
                 static_cast<uint32_t>(x.head_bytes));
    }
  }
  bulk_commit();
}

// ---------------------------------------------------------------------------------------------
// Narrow rows (R29: a pool whose rows, strides or bases are multiples of 8 or 4 bytes but not 16):
// the host run of a piece starts `pad` = src % 16 bytes into a 16-byte unit, so the producer copies
// the enclosing 16-byte-aligned span (a few bytes of the neighbouring rows of the same tier ride
// along, never written anywhere) and records `pad` for the stage; the scatter moves WORD-byte words.
template <int WORD>
struct WordT;
template <> struct WordT<8> { using T = unsigned long long; };
template <> struct WordT<4> { using T = unsigned int; };

template <int WORD>
__device__ __forceinline__ void piece_rows_narrow(const RingParams& p, int lane, int n,
                                                  const uint64_t (&addr)[kRowsPerLane], const unsigned char* st) {
  using T = typename WordT<WORD>::T;
  const int tok = p.x.tok_bytes, wpr = tok / WORD;
  const int total = n * wpr;
  for (int v0 = 0; v0 < total; v0 += 32 * kU) {
    T val[kU];
    uint64_t dst[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int v = v0 + u * 32 + lane;
      const int j = p.word_magic ? static_cast<int>(__umulhi(static_cast<unsigned>(v), p.word_magic)) : v / wpr;
      const int w = v - j * wpr;
      const uint64_t base = row_base(addr, j & (kRingMaxRows - 1));   // every lane shuffles (convergent)
      dst[u] = base + static_cast<uint64_t>(w) * WORD;
      if (v < total) val[u] = *reinterpret_cast<const T*>(st + j * tok + w * WORD);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (v0 + u * 32 + lane < total) *reinterpret_cast<T*>(dst[u]) = val[u];
  }
}

template <bool CONTIG, int WORD>
__global__ void __launch_bounds__(32 * (1 + kRingMaxWarps), 1) ring_load_kernel(const __grid_constant__ RingParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XferParams& x = p.x;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kRingMaxStages;
  int* pads = reinterpret_cast<int*>(empty + kRingMaxStages);
  unsigned char* buf = smem + ring_buf_offset();
  const int S = p.stages, SB = p.stage_bytes, tok = x.tok_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, b = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);   // the piece's scatter warp
    }
    mbar_init_fence();
  }
  if (threadIdx.x == 0) atomicAdd(&g_loads_active, 1u);
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
          unsigned char* st = buf + static_cast<size_t>(s) * SB;
          if (WORD < 16) {
            // the enclosing 16-byte-aligned span of the run; the stage's rows start `pad` bytes in
            const uint64_t a0 = a & ~uint64_t(15);
            const uint32_t pad = static_cast<uint32_t>(a - a0);
            const uint32_t span = nt ? (pad + static_cast<uint32_t>(nt * tok) + 15u) & ~15u : 0u;
            if (lane == 0) {
              pads[s] = static_cast<int>(pad);
              mbar_arrive_expect_tx(&full[s], span);   // releases the pad write to the stage's scatter warp
              if (span) bulk_g2s(st, reinterpret_cast<const void*>(a0), span, &full[s]);
            }
            __syncwarp();
            continue;
          }
          if (lane == 0) mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nt * tok));
          __syncwarp();
          if (p.host_run) {
            if (lane == 0 && nt) {
              if (p.debug & 2)
                bulk_g2s_hint(st, reinterpret_cast<const void*>(a), static_cast<uint32_t>(nt * tok), &full[s],
                              l2_policy_evict_first());
              else
                bulk_g2s(st, reinterpret_cast<const void*>(a), static_cast<uint32_t>(nt * tok), &full[s]);
            }
          } else {
            for (int i = lane; i < nt; i += 32)
              bulk_g2s(st + i * tok, reinterpret_cast<const char*>(a) + int64_t(i) * x.host_tok_stride,
                       static_cast<uint32_t>(tok), &full[s]);
          }
        }
      }
    }
  } else {
    // ---------------- scatter warps: stage -> pages (warp wi: pieces q == wi mod W) ----------------
    const int wi = warp - 1, W = p.warps;
    for (int l = p.l0; l < p.l1; ++l) {
      char* kb = p.kb[l];
      char* vb = p.vb[l];
      const uint32_t q0 = static_cast<uint32_t>(l - p.l0) * static_cast<uint32_t>(mine);
      const int32_t mfirst = static_cast<int32_t>((static_cast<uint32_t>(wi) + W - q0 % W) % W);   // q = q0 + m == wi (mod W)
      RowQueue rq;
      rowq_init(p, rq, mfirst, mine, lane, kb, vb);
      for (int32_t m = mfirst; m < mine; m += W) {
        const uint32_t q = q0 + m;
        const int s = static_cast<int>(q % S);
        int n;
        uint64_t addr[kRowsPerLane];
        rowq_pop(p, rq, m, mine, lane, kb, vb, addr, n);
        mbar_wait(&full[s], (q / S) & 1);
        if (WORD < 16) {
          piece_rows_narrow<WORD < 16 ? WORD : 8>(p, lane, n, addr, buf + static_cast<size_t>(s) * SB + pads[s]);
        } else if (p.debug & 1) {
          // A/B only (STRATA_RING_DEBUG=1): the host reads without the page writes
        } else if (p.bulk_store) {
          piece_rows_bulk<CONTIG>(p, lane, n, addr, buf + static_cast<size_t>(s) * SB);
          bulk_wait_read<0>();   // the TMA has read this stage
        } else {
          piece_rows<CONTIG, 0>(p, lane, n, addr, buf + static_cast<size_t>(s) * SB);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (p.bulk_store) {
        bulk_wait_all();         // the layer's bulk stores are performed
        fence_proxy_async_global();
      }
      if (p.counters) {
        __syncwarp();
        if (lane == 0) arrive_layer<0>(p, l);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicSub(&g_loads_active, 1u);
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
  unsigned char* buf = smem + ring_buf_offset();
  const int S = p.stages, SB = p.stage_bytes, tok = x.tok_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, b = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 32);   // one cp.async arrive (.noinc) per thread of the piece's gather warp
      mbar_init(&empty[s], 1);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const int32_t mine = p.npieces > b ? (p.npieces - 1 - b) / G + 1 : 0;

  if (warp == 0) {
    // ---------------- store: stage -> host run ----------------
    uint32_t q = 0, released = 0;
    uint64_t next_ns = 0;   // pacing: earliest issue time of the next store while a load runs
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
          if (p.pace_ps_per_byte > 0) {
            // while a ring load runs on this device the backup (a non-critical path)
            // paces its host stores to its share of the link instead of crowding out the load;
            // lane 0 decides and waits, the warp follows
            if (lane == 0 && *reinterpret_cast<volatile unsigned int*>(&g_loads_active) > 0) {
              uint64_t now = globaltimer_ns();
              while (now < next_ns) {
                __nanosleep(256);
                now = globaltimer_ns();
              }
              next_ns = now + (static_cast<uint64_t>(nt) * tok * p.pace_ps_per_byte) / 1000;
            }
            __syncwarp();
          }
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
    // ---------------- gather warps: pages -> stage (warp wi: pieces q == wi mod W) ----------------
    const int wi = warp - 1, W = p.warps;
    for (int l = p.l0; l < p.l1; ++l) {
      char* kb = p.kb[l];
      char* vb = p.vb[l];
      const uint32_t q0 = static_cast<uint32_t>(l - p.l0) * static_cast<uint32_t>(mine);
      const int32_t mfirst = static_cast<int32_t>((static_cast<uint32_t>(wi) + W - q0 % W) % W);   // q = q0 + m == wi (mod W)
      RowQueue rq;
      rowq_init(p, rq, mfirst, mine, lane, kb, vb);
      for (int32_t m = mfirst; m < mine; m += W) {
        const uint32_t q = q0 + m;
        const int s = static_cast<int>(q % S);
        int n;
        uint64_t addr[kRowsPerLane];
        rowq_pop(p, rq, m, mine, lane, kb, vb, addr, n);
        if (q >= static_cast<uint32_t>(S)) mbar_wait(&empty[s], ((q / S) - 1) & 1);
        piece_rows<CONTIG, 1>(p, lane, n, addr, buf + static_cast<size_t>(s) * SB);
        cp_async_arrive_noinc(&full[s]);
      }
    }
  }
}

}  // namespace

int ring_header_bytes() { return ring_buf_offset(); }

uint32_t* ring_loads_active() {
  void* a = nullptr;
  if (cudaGetSymbolAddress(&a, g_loads_active) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;   // the LDG load then runs uncounted (offloads beside it unpaced)
  }
  return static_cast<uint32_t*>(a);
}

cudaError_t launch_ring(const RingParams& p, int dir, int ctas, cudaStream_t s) {
  // exclusive: reserve the SM's shared memory so no other kernel's CTA shares the SM
  const int smem = p.smem_reserve > 0 ? p.smem_reserve : ring_buf_offset() + p.stages * p.stage_bytes;
  const bool contig = p.x.head_stride == p.x.head_bytes || p.x.H == 1;
  const int threads = 32 * (1 + p.warps);
  if (dir == 0) {
    if (p.x.gran == 8) return launch_k(ring_load_kernel<true, 8>, ctas, threads, smem, s, p);
    return contig ? launch_k(ring_load_kernel<true, 16>, ctas, threads, smem, s, p)
                  : launch_k(ring_load_kernel<false, 16>, ctas, threads, smem, s, p);
  }
  return contig ? launch_k(ring_offload_kernel<true>, ctas, threads, smem, s, p)
                : launch_k(ring_offload_kernel<false>, ctas, threads, smem, s, p);
}

cudaError_t ring_prepare(int smem) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(ring_load_kernel<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(ring_load_kernel<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(ring_load_kernel<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(ring_offload_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  return cudaFuncSetAttribute(ring_offload_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

}  // namespace strata
