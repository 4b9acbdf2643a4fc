// baselines.cpp — copy-engine baselines and the link roofline (include/strata_baseline.h).
//
// Not on the product path.  They move the same bytes as strata_load / strata_offload from the same
// registered host tier, so the comparison isolates the transfer mechanism:
//   * per-page cudaMemcpyAsync loop — the paper's fragmentation baseline (PAPER.md:166-169, :182
//     ~22 % of PCIe 5.0 at P=32; SGLang-HiCache),
//   * one contiguous cudaMemcpyAsync (the measured link roofline).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/strata_baseline.h"
#include "internal.h"

namespace {

int bfail(int code, const char* what, cudaError_t e = cudaSuccess) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s%s%s", what, e != cudaSuccess ? ": " : "", e != cudaSuccess ? cudaGetErrorString(e) : "");
  return strata::set_last_error(code, buf);
}

struct Copy {
  void* dst;
  const void* src;
  size_t bytes;
};

// Enumerate the copy list: layer-wise (the order a layer-wise loader issues them), then K/V, then
// requests, then maximal runs that are contiguous on both sides: tokens of one device page that
// also sit in one host chunk (and one head at a time when device rows are not head-contiguous).
template <class F>
int for_each_copy(strata_pool_t p, const strata_xfer* x, int dir, F&& emit) {
  if (!p || !x) return bfail(STRATA_ERR_INVALID_ARG, "pool / xfer is NULL");
  const int L = p->d.num_layers;
  if (x->layer_begin < 0 || x->layer_begin > x->layer_end || x->layer_end > L)
    return bfail(STRATA_ERR_INVALID_ARG, "bad layer range");
  if (x->num_reqs < 0) return bfail(STRATA_ERR_INVALID_ARG, "num_reqs < 0");
  if (x->num_reqs > 0 && (!x->num_tokens || !x->chunk_start || !x->page_start))
    return bfail(STRATA_ERR_INVALID_ARG, "NULL request table");
  const int64_t C = p->d.chunk_tokens, P = p->d.page_size, tok = p->tok_bytes;
  // one copy per token row when the row's heads are adjacent on both sides; runs of tokens when
  // consecutive tokens are adjacent on both sides too
  const bool one_head = p->d.num_heads == 1;
  const bool rows_contig = (p->head_stride == p->head_bytes || one_head) &&
                           (p->host_head_stride == p->head_bytes || one_head);
  const bool pages_contig = rows_contig && p->token_stride == tok && p->host_tok_stride == tok;
  const int64_t kv_blk = p->host_kv_off;   // K -> V (and, times KV, layer) step in a chunk (R28)
  for (int32_t l = x->layer_begin; l < x->layer_end; ++l) {
    for (int kv = 0; kv < p->nkv; ++kv) {
      char* base = static_cast<char*>(kv ? p->v[l] : p->k[l]);
      for (int32_t r = 0; r < x->num_reqs; ++r) {
        const int64_t n = x->num_tokens[r];
        const int64_t oc = x->chunk_offset ? x->chunk_offset[r] : 0;
        const int64_t op = x->page_offset ? x->page_offset[r] : 0;
        int64_t i = 0;
        while (i < n) {
          const int64_t ci = oc + i, pi = op + i;
          const int64_t hc = x->host_chunks[x->chunk_start[r] + ci / C];
          const int64_t pg = x->dev_pages[x->page_start[r] + pi / P];
          if (hc < 0 || hc >= p->d.num_chunks || pg < 0 || pg >= p->d.num_pages)
            return bfail(STRATA_ERR_INDEX_RANGE, "index out of range");
          int64_t run = 1;
          if (pages_contig) run = std::min({n - i, C - ci % C, P - pi % P});
          char* h = p->host + hc * p->chunk_bytes + (int64_t(l) * p->nkv + kv) * kv_blk +
                    (ci % C) * p->host_tok_stride + p->host_head_off;
          char* d = base + pg * p->page_stride + (pi % P) * p->token_stride;
          if (rows_contig) {
            if (dir == 0) emit(Copy{d, h, size_t(run * tok)});
            else emit(Copy{h, d, size_t(run * tok)});
          } else {
            for (int hh = 0; hh < p->d.num_heads; ++hh) {
              char* hp = h + hh * p->host_head_stride;
              char* dp = d + hh * p->head_stride;
              if (dir == 0) emit(Copy{dp, hp, size_t(p->head_bytes)});
              else emit(Copy{hp, dp, size_t(p->head_bytes)});
            }
          }
          i += run;
        }
      }
    }
  }
  return STRATA_OK;
}

}  // namespace

extern "C" {

int strata_baseline_memcpy_pages(strata_pool_t p, const strata_xfer* x, int32_t dir, strata_stream_t stream,
                                 int64_t* ncopies) {
  if (dir != STRATA_H2D && dir != STRATA_D2H) return bfail(STRATA_ERR_INVALID_ARG, "bad dir");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t count = 0;
  cudaError_t err = cudaSuccess;
  const cudaMemcpyKind kind = dir == STRATA_H2D ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  int rc = for_each_copy(p, x, dir, [&](const Copy& c) {
    if (err != cudaSuccess) return;
    err = cudaMemcpyAsync(c.dst, c.src, c.bytes, kind, s);
    ++count;
  });
  if (rc) return rc;
  if (err != cudaSuccess) return bfail(STRATA_ERR_CUDA, "cudaMemcpyAsync", err);
  if (ncopies) *ncopies = count;
  return STRATA_OK;
}

int strata_baseline_contiguous(strata_pool_t p, int32_t dir, void* dev, int64_t host_offset, int64_t bytes,
                               strata_stream_t stream) {
  if (!p || !dev) return bfail(STRATA_ERR_INVALID_ARG, "pool / dev is NULL");
  if (host_offset < 0 || bytes < 0 || size_t(host_offset + bytes) > p->host_bytes)
    return bfail(STRATA_ERR_INVALID_ARG, "range outside the host tier");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = dir == STRATA_H2D
                      ? cudaMemcpyAsync(dev, p->host + host_offset, size_t(bytes), cudaMemcpyHostToDevice, s)
                      : cudaMemcpyAsync(p->host + host_offset, dev, size_t(bytes), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return bfail(STRATA_ERR_CUDA, "cudaMemcpyAsync", e);
  return STRATA_OK;
}

}  // extern "C"
