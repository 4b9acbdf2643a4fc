// dma.cpp — STRATA_ENGINE_DMA (include/strata.h): copy engines gather whole page-first runs into an
// HBM staging ring, the LDG kernel scatters them to the pages (offload: the mirror).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"

namespace strata {

// -------------------------------------------------------------------------------------------------
// STRATA_ENGINE_DMA: copy engines move whole page-first runs, an SM kernel does the scatter.
//
// The page-first host tier keeps, for one layer, the K rows and then the V rows of a chunk's C
// tokens back to back (R1), so a layer of a fully covered chunk is ONE contiguous 2*C*S_tok run
// (256 KiB for Llama-8B at C=64).  The copy engines read such runs at up to 98 % of the link
// (256 KiB copies, profiles/r01/ce_probe.jsonl) where SM-issued reads top out at 92.6 %.  Each run
// is one cudaMemcpyAsync (the batched submission API of round 1 is closed on the GPU pool after
// unexplained Xid 32 faults).  Each run lands in an HBM staging slot laid out exactly like
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

// bytes per staging slot (2 slots) and scatter quota: 64 MiB / 4 CTAs 54.2, 64 / 8 54.4,
// 128 / 8 54.7, 256 / 8 54.7 GB/s (profiles/r01/stage.jsonl): fewer, larger pieces leave fewer
// inter-piece event waits on the copy streams and a shorter scatter tail.
constexpr size_t kStageTarget = size_t(128) << 20;
constexpr int kDefaultCtasScatter = 8;
constexpr size_t kDmaMinEdgePiece = size_t(16) << 20;   // edge pieces are not cut below this

// Staging buffers are allocated once, at the first DMA operation of a direction, at their full size
// (the stage target, or one group of chunk-layers if that is larger) so that they never move: a CUDA
// graph that captured a DMA operation keeps pointing at them.  A later operation that would need
// more (only with STRATA_STAGE_MB raised, or a group larger than the target) is refused once this
// direction has been captured, and reallocates otherwise.
static int ensure_dma(strata_pool* p, strata_pool::DmaDir& D, size_t slot_bytes, int64_t slots, size_t full_bytes,
                      int64_t full_slots, bool capturing) {
  cudaError_t e;
  if (capturing) D.captured = true;
  if (!D.cs[0]) {
    if (capturing) return fail(STRATA_ERR_UNSUPPORTED, "the first STRATA_ENGINE_DMA operation of a pool and "
                                                       "direction must run outside stream capture (it allocates)");
    if (const char* v = getenv("STRATA_COPY_STREAMS"))
      D.ncs = std::max(1, std::min(strata_pool::kCopyStreams, atoi(v)));
    for (auto& c : D.cs)
      if ((e = cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking))) return cuda_fail(e, "cudaStreamCreate");
    for (cudaEvent_t* f : {&D.ev_fork, &D.cap_fork})
      if ((e = cudaEventCreateWithFlags(f, cudaEventDisableTiming))) return cuda_fail(e, "cudaEventCreate");
    for (int s = 0; s < 2; ++s) {
      for (cudaEvent_t* f : {&D.ev_slot[s], &D.cap_slot[s]})
        if ((e = cudaEventCreateWithFlags(f, cudaEventDisableTiming))) return cuda_fail(e, "cudaEventCreate");
      for (int c = 0; c < strata_pool::kCopyStreams; ++c)
        for (cudaEvent_t* f : {&D.ev_copy[s][c], &D.cap_copy[s][c]})
          if ((e = cudaEventCreateWithFlags(f, cudaEventDisableTiming))) return cuda_fail(e, "cudaEventCreate");
    }
  }
  const bool grow_stage = D.stage_bytes < slot_bytes, grow_ids = p->slot_cap < slots;
  if (grow_stage || grow_ids) {
    if ((grow_stage && D.captured) || (grow_ids && (p->dma[0].captured || p->dma[1].captured)))
      return fail(STRATA_ERR_UNSUPPORTED, "STRATA_ENGINE_DMA staging would have to grow (%zu -> %zu bytes) after a "
                  "graph captured it", D.stage_bytes, slot_bytes);
    cudaDeviceSynchronize();   // earlier operations may still use the old buffers
  }
  if (D.stage_bytes < slot_bytes) {
    for (auto& b : D.stage) {
      if (b) cudaFree(b);
      b = nullptr;
    }
    D.stage_bytes = 0;
    const size_t want = std::max(slot_bytes, full_bytes);
    for (auto& b : D.stage)
      if ((e = cudaMalloc(&b, want))) return fail(STRATA_ERR_OOM, "cudaMalloc(staging %zu): %s", want,
                                                  cudaGetErrorString(e));
    D.stage_bytes = want;
  }
  if (p->slot_cap < slots) {
    if (p->slot_ids) cudaFree(p->slot_ids);
    p->slot_ids = nullptr;
    p->slot_cap = 0;
    const int64_t n = std::max(slots, full_slots);
    std::vector<int32_t> iota(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) iota[i] = static_cast<int32_t>(i);
    if ((e = cudaMalloc(&p->slot_ids, iota.size() * 4))) return cuda_fail(e, "cudaMalloc(slot ids)");
    if ((e = cudaMemcpy(p->slot_ids, iota.data(), iota.size() * 4, cudaMemcpyHostToDevice)))
      return cuda_fail(e, "cudaMemcpy(slot ids)");
    p->slot_cap = n;
  }
  return STRATA_OK;
}

void free_dma(strata_pool* p) {
  if (p->slot_ids) cudaFree(p->slot_ids);
  for (auto& D : p->dma) {
    for (auto& b : D.stage)
      if (b) cudaFree(b);
    for (auto& c : D.cs)
      if (c) cudaStreamDestroy(c);
    for (cudaEvent_t ev : {D.ev_fork, D.cap_fork})
      if (ev) cudaEventDestroy(ev);
    for (int s = 0; s < 2; ++s) {
      for (cudaEvent_t ev : {D.ev_slot[s], D.cap_slot[s]})
        if (ev) cudaEventDestroy(ev);
      for (int c = 0; c < strata_pool::kCopyStreams; ++c)
        for (cudaEvent_t ev : {D.ev_copy[s][c], D.cap_copy[s][c]})
          if (ev) cudaEventDestroy(ev);
    }
  }
}

// A run of k chunks with consecutive host ids: layer block j of each sits chunk_bytes after the
// previous one on the host and one staging slot after it on the device, so the run is ONE strided
// copy (cudaMemcpy2DAsync) instead of k.  Host allocators that hand out chunks in order (the
// control plane's free lists, a fresh tier) make such runs the common case.
struct Copy2D {
  void* dst;
  size_t dpitch;
  const void* src;
  size_t spitch, width, height;
};

// Submit a copy list over the pool's copy streams (contiguous shares, one cudaMemcpyAsync per run);
// the strided runs go to the first stream.
static cudaError_t submit_copies(strata_pool* p, strata_pool::DmaDir& D, std::vector<void*>& dst, std::vector<void*>& src, std::vector<size_t>& sz,
                          const std::vector<Copy2D>& c2d, int dir, int slot) {
  (void)p;
  const size_t n = dst.size();
  const int ns = D.ncs;
  const cudaMemcpyKind kind = dir == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  for (const Copy2D& r : c2d) {
    cudaError_t e = cudaMemcpy2DAsync(r.dst, r.dpitch, r.src, r.spitch, r.width, r.height, kind, D.cs[0]);
    if (e != cudaSuccess) return e;
  }
  for (int c = 0; c < ns; ++c) {
    const size_t lo = n * c / ns, hi = n * (c + 1) / ns;
    for (size_t i = lo; i < hi; ++i) {
      cudaError_t e = cudaMemcpyAsync(dst[i], src[i], sz[i], kind, D.cs[c]);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(D.ev_copy[slot][c], D.cs[c]);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Geometry of one DMA operation: what a chunk position contributes to the host <-> staging copies.
struct DmaGeom {
  int64_t C, P, tok, nkv, hb, Hl, h0;
  size_t unit;    // one chunk-layer of this GPU's heads: nkv*C*H*D*e
  int G;          // layers per copy run (layer group)
  size_t gunit;   // staging bytes per chunk position: G*unit
  bool hm;        // head-major host chunks (R28)
  int64_t lay() const { return nkv * C * hb; }   // head-major: one layer of one head
};

// The call's chunk positions, request by request (a position = the tokens of one host chunk).
static int collect_positions(const strata_pool* p, const strata_xfer* x, const Plan& plan, std::vector<ChunkPos>& pos) {
  const int64_t C = p->d.chunk_tokens;
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
  return STRATA_OK;
}

// Pieces: <= cap chunk positions and <= kMaxReqsPerLaunch requests each.
static std::vector<Piece> make_pieces(const std::vector<ChunkPos>& pos, size_t cap) {
  std::vector<Piece> v;
  for (size_t k = 0; k < pos.size();) {
    Piece pc{k, 0};
    int nreq = 0;
    int32_t last = -1;
    while (k < pos.size() && pc.count < cap) {
      if (pos[k].req != last) {
        if (nreq == kMaxReqsPerLaunch) break;
        ++nreq;
        last = pos[k].req;
      }
      ++pc.count;
      ++k;
    }
    v.push_back(pc);
  }
  return v;
}

struct CopyList {
  std::vector<void*> dst, src;
  std::vector<size_t> sz;
  std::vector<Copy2D> c2d;
  void clear() {
    dst.clear();
    src.clear();
    sz.clear();
    c2d.clear();
  }
  void add(char* host, char* staged, int64_t bytes, int dir) {   // one run: host <-> staging
    dst.push_back(dir == 0 ? staged : host);
    src.push_back(dir == 0 ? host : staged);
    sz.push_back(static_cast<size_t>(bytes));
  }
};

// Host <-> staging copies of one piece for layers [lg, lg+gl): staging slot j holds chunk position
// j's G layers in the host tier's own order for this GPU's heads — token-major [G][KV][C][H][D], or
// head-major [H][G][KV][C][D] (R28).  Runs of full chunks with consecutive host ids become one
// strided copy (per head for head-major); the rest is one copy per contiguous run.
static void build_copies(strata_pool* p, const strata_xfer* x, const std::vector<ChunkPos>& pos, const Piece& pc,
                         const DmaGeom& m, int32_t lg, int gl, char* stage, int dir, bool strided, CopyList& out) {
  auto host_chunk = [&](size_t j) {
    const ChunkPos& c = pos[pc.first + j];
    return int64_t(x->host_chunks_host[x->chunk_start[c.req] + c.cq]);
  };
  auto full = [&](size_t j) { return pos[pc.first + j].lo == 0 && pos[pc.first + j].cnt == m.C; };
  const int64_t lay = m.lay();
  for (size_t j = 0; j < pc.count; ++j) {
    const ChunkPos& cp = pos[pc.first + j];
    const int64_t hc = host_chunk(j);
    char* const hbase = p->host + hc * p->chunk_bytes;
    char* const d = stage + j * m.gunit;
    if (strided && full(j)) {   // full chunks: extend over consecutive host ids
      size_t k = 1;
      while (j + k < pc.count && full(j + k) && host_chunk(j + k) == hc + int64_t(k)) ++k;
      if (k >= 2) {
        // token-major: the group's layers of a chunk are one block; head-major: one block per head
        // of this GPU (the layers of head h0+b, [L][KV][C][D] inside the chunk)
        const int nblk = m.hm ? int(m.Hl) : 1;
        for (int b = 0; b < nblk; ++b) {
          char* h0p = hbase + (m.hm ? (m.h0 + b) * p->host_head_stride + int64_t(lg) * lay : int64_t(lg) * int64_t(m.unit));
          char* d0p = d + (m.hm ? size_t(b) * m.G * lay : 0);
          const size_t width = m.hm ? size_t(gl) * lay : size_t(gl) * m.unit;
          if (dir == 0) out.c2d.push_back({d0p, m.gunit, h0p, size_t(p->chunk_bytes), width, k});
          else out.c2d.push_back({h0p, size_t(p->chunk_bytes), d0p, m.gunit, width, k});
          p->counters.dma_copies += 1;
        }
        j += k - 1;
        continue;
      }
    }
    if (m.hm) {
      // head-major: head h0+hh of the chunk is a one-head page-first chunk [L][KV][C][D]
      auto hoff = [&](int64_t hh, int g, int kv) {
        return (m.h0 + hh) * p->host_head_stride + int64_t(lg + g) * lay + kv * m.C * m.hb;
      };
      auto soff = [&](int64_t hh, int g, int kv) { return (hh * m.G + g) * lay + kv * m.C * m.hb; };
      for (int64_t hh = 0; hh < m.Hl; ++hh) {
        if (full(j)) {
          out.add(hbase + hoff(hh, 0, 0), d + soff(hh, 0, 0), gl * lay, dir);   // the group's layers of the head
        } else {
          for (int g = 0; g < gl; ++g)
            for (int kv = 0; kv < m.nkv; ++kv)
              out.add(hbase + hoff(hh, g, kv) + cp.lo * m.hb, d + soff(hh, g, kv) + cp.lo * m.hb, cp.cnt * m.hb, dir);
        }
      }
    } else {
      char* const h = hbase + int64_t(lg) * int64_t(m.unit);
      if (full(j)) {
        out.add(h, d, gl * int64_t(m.unit), dir);   // the group's K,V runs are adjacent: one copy
      } else {
        for (int g = 0; g < gl; ++g) {
          const int64_t o = g * int64_t(m.unit);
          out.add(h + o + cp.lo * m.tok, d + o + cp.lo * m.tok, cp.cnt * m.tok, dir);   // K rows of layer lg+g
          if (m.nkv == 2)                                                                // V rows
            out.add(h + o + (m.C + cp.lo) * m.tok, d + o + (m.C + cp.lo) * m.tok, cp.cnt * m.tok, dir);
        }
      }
    }
  }
}

// Request table of a piece: sub-requests whose "chunks" are staging slots 0..count-1.  Returns the
// piece's token count.
static int32_t piece_table(const strata_xfer* x, const std::vector<ChunkPos>& pos, const Piece& pc, int64_t P,
                           strata::ReqTable& rt) {
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
  return acc;
}

int transfer_dma(strata_pool* p, const strata_xfer* x, const Plan& plan, strata::XferParams xp, cudaStream_t s,
                 int dir, int slot_ev) {
  if (!x->host_chunks_host && plan.total_tokens > 0)
    return fail(STRATA_ERR_INVALID_ARG, "STRATA_ENGINE_DMA needs xfer.host_chunks_host");
  std::vector<ChunkPos> pos;
  int rc = collect_positions(p, x, plan, pos);
  if (rc) return rc;
  DmaGeom m;
  m.C = p->d.chunk_tokens;
  m.P = p->d.page_size;
  m.tok = p->tok_bytes;
  m.nkv = p->nkv;
  m.hb = p->head_bytes;
  m.Hl = p->d.num_heads;
  m.h0 = p->head_begin;
  m.hm = p->head_major;
  m.unit = static_cast<size_t>(m.nkv * m.C * m.tok);
  // layers per copy run.  Loads keep per-layer granularity (grouping does not raise H2D throughput,
  // profiles/r01/sweep_groups*.jsonl); offloads ("backup", a non-critical path) group
  // layers until a run is >= 128 KiB, which D2H copies need (70B TP=8 rank: 44.6 -> 55.8 GB/s).
  int G = x->layer_group;
  if (G <= 0)
    G = dir == 0 ? 1 : static_cast<int>(std::min<int64_t>(8, (kDmaMinOffloadRun + int64_t(m.unit) - 1) / int64_t(m.unit)));
  m.G = std::max(1, std::min(G, std::max(1, x->layer_end - x->layer_begin)));
  m.gunit = m.unit * static_cast<size_t>(m.G);
  size_t stage_target = kStageTarget;
  if (const char* v = getenv("STRATA_STAGE_MB")) stage_target = std::max<size_t>(1, strtoull(v, nullptr, 10)) << 20;
  const size_t per_piece = std::max<size_t>(1, std::min(pos.size(), stage_target / m.gunit));
  bool ordered = true;   // env STRATA_DMA_ORDERED=0 drops the piece barrier (A/B only)
  if (const char* v = getenv("STRATA_DMA_ORDERED")) ordered = atoi(v) != 0;
  bool strided = true;   // env STRATA_DMA_STRIDED=0: one copy per chunk (A/B only)
  if (const char* v = getenv("STRATA_DMA_STRIDED")) strided = atoi(v) != 0;
  const std::vector<Piece> pieces = make_pieces(pos, per_piece);
  // The first and the last layer group are cut into `edge` times smaller pieces: the first layer's
  // event then waits for one small scatter instead of a whole-layer one (earlier start of layer-wise
  // prefill), and the op's tail, the last scatter with no copy left to hide it, shrinks the same way.
  int edge = 4;   // env STRATA_DMA_EDGE_SPLIT (1 = off)
  if (const char* v = getenv("STRATA_DMA_EDGE_SPLIT")) edge = std::max(1, atoi(v));
  const size_t edge_cap = std::min(per_piece, std::max<size_t>({1, per_piece / size_t(edge), kDmaMinEdgePiece / m.gunit}));
  const std::vector<Piece> edge_pieces = edge_cap < per_piece ? make_pieces(pos, edge_cap) : pieces;
  strata_pool::DmaDir& D = p->dma[dir];
  cudaStreamCaptureStatus capst = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &capst) != cudaSuccess) return cuda_fail(cudaErrorUnknown, "cudaStreamIsCapturing");
  // full size: the stage target over the smallest run unit (one chunk-layer), at least this call's
  rc = ensure_dma(p, D, per_piece * m.gunit, static_cast<int64_t>(per_piece), stage_target,
                  static_cast<int64_t>(std::max<size_t>(1, stage_target / m.unit)),
                  capst == cudaStreamCaptureStatusActive);
  if (rc) return rc;
  // a captured operation records into the capture set of events (swapped back on every exit)
  struct CaptureEvents {
    strata_pool::DmaDir& D;
    bool on;
    void swap() {
      std::swap(D.ev_fork, D.cap_fork);
      for (int s = 0; s < 2; ++s) {
        std::swap(D.ev_slot[s], D.cap_slot[s]);
        for (int c = 0; c < strata_pool::kCopyStreams; ++c) std::swap(D.ev_copy[s][c], D.cap_copy[s][c]);
      }
    }
    CaptureEvents(strata_pool::DmaDir& d, bool capturing) : D(d), on(capturing) { if (on) swap(); }
    ~CaptureEvents() { if (on) swap(); }
  } capture_events(D, capst == cudaStreamCaptureStatusActive);

  cudaError_t e;
  const int threads = x->threads ? x->threads : kDefaultThreadsLdg;
  const int unroll = threads > 512 ? 4 : kDefaultUnroll;
  xp.rows_per_group = 32;   // lane t fetches row t; the warp then streams the 32 rows
  const int ctas = x->num_ctas ? x->num_ctas : p->gran < 16 ? kDefaultCtasNarrow : kDefaultCtasScatter;
  // the scatter / gather kernel sees the staging slots as a compact host tier (chunk = slot)
  xp.chunk_bytes = static_cast<int64_t>(m.gunit);
  xp.kv_off = m.hm ? m.C * m.hb : m.C * m.tok;
  xp.host_chunks = p->slot_ids;
  xp.host_tok_stride = m.hm ? m.hb : m.tok;
  xp.host_head_off = 0;
  xp.host_head_stride = m.hm ? int64_t(m.G) * m.lay() : m.hb;

  if ((e = cudaEventRecord(D.ev_fork, s))) return cuda_fail(e, "cudaEventRecord");
  for (int ci = 0; ci < D.ncs; ++ci)
    if ((e = cudaStreamWaitEvent(D.cs[ci], D.ev_fork, 0))) return cuda_fail(e, "cudaStreamWaitEvent");
  CopyList cl;
  int64_t i = 0;                 // pieces of this operation
  // pieces of this direction, across operations; a graph capture starts its own sequence (its
  // nodes may not depend on uncaptured work, and a replay is ordered by the graph's own edges)
  uint64_t capture_seq = 0;
  uint64_t& seq = capst == cudaStreamCaptureStatusActive ? capture_seq : D.seq;
  int last_slot = 0;
  for (int32_t lg = x->layer_begin; lg < x->layer_end; lg += m.G) {
    const int gl = std::min<int>(m.G, x->layer_end - lg);   // layers in this group
    const std::vector<Piece>& gp = (lg == x->layer_begin || lg + m.G >= x->layer_end) ? edge_pieces : pieces;
    for (const Piece& pc : gp) {
      const bool last_piece = &pc == &gp.back();
      const int slot = static_cast<int>(seq & 1);
      char* stage = D.stage[slot];
      cl.clear();
      build_copies(p, x, pos, pc, m, lg, gl, stage, dir, strided, cl);
      xp.ntok = piece_table(x, pos, pc, m.P, xp.rt);
      xp.host = stage;
      const int64_t groups = (m.nkv * xp.ntok + xp.rows_per_group - 1) / xp.rows_per_group;
      const int c = static_cast<int>(std::min<int64_t>(ctas, (groups * 32 + threads - 1) / threads));
      // one scatter / gather launch per layer of the group over the slot's layer sub-blocks
      auto launch_group = [&](int kdir) -> cudaError_t {
        for (int g = 0; g < gl; ++g) {
          xp.kbase = static_cast<char*>(p->k[lg + g]);
          xp.vbase = static_cast<char*>(p->v[lg + g]);
          xp.layer_off = m.hm ? int64_t(g) * m.lay() : int64_t(g) * int64_t(m.unit);
          cudaError_t le = strata::launch_ldg(xp, kdir, c, threads, unroll, s);
          if (le != cudaSuccess) return le;
          ++p->counters.kernel_launches;
          // loads: layer lg+g is complete once its scatter of the group's last piece has run
          if (kdir == 0 && last_piece && (le = op_record(p, slot_ev, 1 + lg + g, s))) return le;
        }
        return cudaSuccess;
      };
      const int ncs = D.ncs;
      if (dir == 0) {
        // copies into the slot (after its previous scatter), then the scatters on the caller's stream
        if (seq >= 2)
          for (int ci = 0; ci < ncs; ++ci)
            if ((e = cudaStreamWaitEvent(D.cs[ci], D.ev_slot[slot], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
        // piece barrier: no copy stream starts piece i before every stream has finished piece i-1.
        // Without it the copy engines are not served fairly, a lagging stream's share of layer l
        // completes together with layer l+1 and the layer events arrive in pairs (4.6 / 0.6 ms
        // instead of 2.4 / 2.4 ms for Llama-8B), which halves the granularity of layer-wise overlap.
        if (i >= 1 && ordered)
          for (int ci = 0; ci < ncs; ++ci)
            for (int cj = 0; cj < ncs; ++cj)
              if (cj != ci && (e = cudaStreamWaitEvent(D.cs[ci], D.ev_copy[slot ^ 1][cj], 0)))
                return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = submit_copies(p, D, cl.dst, cl.src, cl.sz, cl.c2d, dir, slot))) return cuda_fail(e, "cudaMemcpyAsync (DMA runs)");
        for (int ci = 0; ci < ncs; ++ci)
          if ((e = cudaStreamWaitEvent(s, D.ev_copy[slot][ci], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = launch_group(0))) return cuda_fail(e, "scatter kernel launch");
        if ((e = cudaEventRecord(D.ev_slot[slot], s))) return cuda_fail(e, "cudaEventRecord");
      } else {
        // gathers into the slot (after its previous copies drained), then copies to the host tier
        if (seq >= 2)
          for (int ci = 0; ci < ncs; ++ci)
            if ((e = cudaStreamWaitEvent(s, D.ev_copy[slot][ci], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = launch_group(1))) return cuda_fail(e, "gather kernel launch");
        if ((e = cudaEventRecord(D.ev_slot[slot], s))) return cuda_fail(e, "cudaEventRecord");
        for (int ci = 0; ci < ncs; ++ci)
          if ((e = cudaStreamWaitEvent(D.cs[ci], D.ev_slot[slot], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = submit_copies(p, D, cl.dst, cl.src, cl.sz, cl.c2d, dir, slot))) return cuda_fail(e, "cudaMemcpyAsync (DMA runs)");
      }
      p->counters.dma_copies += static_cast<int64_t>(cl.dst.size());
      last_slot = slot;
      ++i;
      ++seq;
    }
    if (dir == 0 && pieces.empty()) {
      for (int g = 0; g < gl; ++g)
        if ((e = op_record(p, slot_ev, 1 + lg + g, s))) return cuda_fail(e, "cudaEventRecord");
    } else if (dir == 1) {
      // host bytes of the group are written once every copy stream has passed its last piece
      if (!pieces.empty())
        for (int c = 1; c < D.ncs; ++c)
          if ((e = cudaStreamWaitEvent(D.cs[0], D.ev_copy[last_slot][c], 0)))
            return cuda_fail(e, "cudaStreamWaitEvent");
      for (int g = 0; g < gl; ++g)
        if ((e = op_record(p, slot_ev, 1 + lg + g, D.cs[0]))) return cuda_fail(e, "cudaEventRecord");
    }
  }
  if (dir == 1 && i > 0)  // join: the caller's stream is ordered after every copy
    for (int ci = 0; ci < D.ncs; ++ci)
      if ((e = cudaStreamWaitEvent(s, D.ev_copy[last_slot][ci], 0))) return cuda_fail(e, "cudaStreamWaitEvent");
  return STRATA_OK;
}

}  // namespace strata
