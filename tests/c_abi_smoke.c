/*
 * c_abi_smoke.c — a plain C99 consumer of include/strata.h (no Python, no torch, no CUDA headers):
 * proves the boundary is a C ABI.  Built and run by tests/test_c_abi.py.
 *
 *   without a GPU: every argument check returns its documented code before touching CUDA, and a valid
 *                  descriptor reports STRATA_ERR_CUDA;
 *   with a GPU (argv[1] == "gpu"): registers a tiny pool over cudaMalloc'd buffers (the CUDA runtime is
 *                  reached through dlopen'd symbols, so this file still includes no CUDA header), loads
 *                  two layers with every engine, and checks one token row against the host tier.
 */
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "strata.h"
#include "strata_disk.h"
#include "strata_ctl.h"

static int failures = 0;
#define EXPECT(cond, ...)                      \
  do {                                         \
    if (!(cond)) {                             \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);            \
      fprintf(stderr, "\n");                   \
      ++failures;                              \
    }                                          \
  } while (0)

static void cpu_checks(void) {
  strata_pool_t p = (strata_pool_t)0x1;
  void* k[2] = {(void*)0x10000, (void*)0x20000};
  void* v[2] = {(void*)0x30000, (void*)0x40000};
  strata_pool_desc d;
  memset(&d, 0, sizeof d);
  d.num_layers = 2; d.num_heads = 2; d.head_dim = 64; d.elem_bytes = 2; d.page_size = 16;
  d.chunk_tokens = 64; d.k_ptrs = k; d.v_ptrs = v; d.num_pages = 256; d.num_chunks = 64;
  EXPECT(strata_register_host_pool(NULL, &p) == STRATA_ERR_INVALID_ARG, "NULL desc");
  EXPECT(p == NULL, "out not cleared");
  d.token_stride = 257;   /* not a multiple of the 2-byte element (R29) */
  EXPECT(strata_register_host_pool(&d, &p) == STRATA_ERR_ALIGNMENT, "token stride");
  EXPECT(strlen(strata_last_error()) > 0, "no error message");
  d.token_stride = 0;
  d.host_heads = 2; d.head_begin = 1;   /* heads [1,3) of a 2-head host tier (R28) */
  EXPECT(strata_register_host_pool(&d, &p) == STRATA_ERR_INVALID_ARG, "head slice outside the host tier");
  d.host_heads = 0; d.head_begin = 0;
  strata_xfer x;
  memset(&x, 0, sizeof x);
  EXPECT(strata_load(NULL, &x, NULL, NULL) == STRATA_ERR_INVALID_ARG, "NULL pool");
  EXPECT(strata_unregister_host_pool(NULL) == STRATA_OK, "unregister NULL");
  strata_disk_t disk = (strata_disk_t)0x1;
  EXPECT(strata_disk_open(NULL, &disk) == STRATA_ERR_INVALID_ARG && disk == NULL, "disk NULL desc");
  EXPECT(strata_version() >= 100, "version");
}

/* The control plane (strata_ctl.h) is host code: a context offloaded earlier hits in the host tier,
 * the scheduler dispatches the request, and its LOAD plan, decoded with strata.h's token formula,
 * moves exactly the context's host slots to the request's device slots. */
static void ctl_checks(void) {
  strata_ctl_desc cd;
  memset(&cd, 0, sizeof cd);
  cd.page_size = 4; cd.chunk_tokens = 8; cd.num_pages = 64; cd.num_chunks = 16;
  cd.deferral_threshold = 100; cd.loading_bound_ratio = 100.0;
  strata_ctl_t c = NULL;
  EXPECT(strata_ctl_create(NULL, &c) == STRATA_ERR_INVALID_ARG, "ctl NULL desc");
  EXPECT(strata_ctl_create(&cd, &c) == STRATA_OK && c, "ctl create: %s", strata_last_error());
  if (!c) return;
  int32_t ctx[20], req[23];
  int64_t hslots[20], dslots[23], n = 0;
  for (int i = 0; i < 20; ++i) ctx[i] = req[i] = 1000 + i;
  req[20] = 7; req[21] = 8; req[22] = 9;
  EXPECT(strata_ctl_insert(c, ctx, 20, STRATA_TIER_HOST, 0.0, hslots) == STRATA_OK, "insert");
  EXPECT(strata_ctl_submit(c, 42, req, 23) == STRATA_OK, "submit");
  EXPECT(strata_ctl_submit(c, 42, req, 23) == STRATA_ERR_DUPLICATE, "duplicate id");
  strata_ctl_round r;
  EXPECT(strata_ctl_schedule(c, 1.0, &r) == STRATA_OK && r.num_batch == 1 && r.load_tokens == 20 &&
         r.new_tokens == 3, "schedule: batch %lld load %lld new %lld", (long long)r.num_batch,
         (long long)r.load_tokens, (long long)r.new_tokens);
  EXPECT(strata_ctl_req_slots(c, 42, dslots, &n) == STRATA_OK && n == 23, "req slots");
  strata_ctl_plan pl;
  EXPECT(strata_ctl_plan_get(c, STRATA_CTL_LOAD, &pl) == STRATA_OK, "plan");
  int64_t t = 0;
  for (int64_t q = 0; q < pl.num_reqs; ++q)
    for (int64_t i = 0; i < pl.num_tokens[q]; ++i, ++t) {
      const int64_t ci = pl.chunk_offset[q] + i, pi = pl.page_offset[q] + i;
      const int64_t h = (int64_t)pl.host_chunks[pl.chunk_start[q] + ci / 8] * 8 + ci % 8;
      const int64_t dv = (int64_t)pl.dev_pages[pl.page_start[q] + pi / 4] * 4 + pi % 4;
      EXPECT(t < 20 && h == hslots[t] && dv == dslots[t], "plan token %lld", (long long)t);
    }
  EXPECT(t == 20, "plan covers %lld tokens", (long long)t);
  EXPECT(strata_ctl_complete(c, 42, 2.0) == STRATA_OK, "complete");
  strata_ctl_match_t m;
  EXPECT(strata_ctl_match(c, req, 23, &m) == STRATA_OK && m.device == 23 && m.total == 23, "match");
  EXPECT(strata_ctl_bubble_steps(20.0, 5.0, 3.0, 8) == 5, "bubble steps");
  EXPECT(strata_ctl_destroy(c) == STRATA_OK, "destroy");
}

typedef int (*malloc_fn)(void**, size_t);
typedef int (*memset_fn)(void*, int, size_t);
typedef int (*memcpy_fn)(void*, const void*, size_t, int);
typedef int (*sync_fn)(void);

static int gpu_checks(void) {
  void* rt = dlopen("libcudart.so.12", RTLD_NOW | RTLD_GLOBAL);
  if (!rt) rt = dlopen("/usr/local/cuda/lib64/libcudart.so.12", RTLD_NOW | RTLD_GLOBAL);
  if (!rt) rt = dlopen("/usr/local/cuda/lib64/libcudart.so", RTLD_NOW | RTLD_GLOBAL);
  if (!rt) { fprintf(stderr, "no libcudart: %s\n", dlerror()); return 1; }
  malloc_fn cmalloc = (malloc_fn)dlsym(rt, "cudaMalloc");
  memset_fn cmemset = (memset_fn)dlsym(rt, "cudaMemset");
  memcpy_fn cmemcpy = (memcpy_fn)dlsym(rt, "cudaMemcpy");
  sync_fn csync = (sync_fn)dlsym(rt, "cudaDeviceSynchronize");
  const int L = 2, H = 2, D = 64, e = 2, P = 1, C = 16, pages = 64, chunks = 8, n = 40;
  const size_t tok = (size_t)H * D * e, layer_bytes = (size_t)pages * P * tok;
  void *k[2], *v[2];
  for (int l = 0; l < L; ++l) {
    cmalloc(&k[l], layer_bytes); cmalloc(&v[l], layer_bytes);
    cmemset(k[l], 0xA5, layer_bytes); cmemset(v[l], 0xA5, layer_bytes);
  }
  strata_pool_desc d;
  memset(&d, 0, sizeof d);
  d.num_layers = L; d.num_heads = H; d.head_dim = D; d.elem_bytes = e; d.page_size = P; d.chunk_tokens = C;
  d.k_ptrs = k; d.v_ptrs = v; d.num_pages = pages; d.num_chunks = chunks;
  strata_pool_t pool = NULL;
  int rc = strata_register_host_pool(&d, &pool);
  EXPECT(rc == STRATA_OK, "register: %d %s", rc, strata_last_error());
  if (rc) return 1;
  void* host = NULL; size_t hb = 0;
  strata_host_pool_ptr(pool, &host, &hb);
  for (size_t i = 0; i < hb; ++i) ((unsigned char*)host)[i] = (unsigned char)(i * 131 + 7);
  /* token i -> host chunk (i / C) of list {5, 2, 7}, device page 63 - i */
  int32_t hchunks_h[3] = {5, 2, 7}, pages_h[64];
  for (int i = 0; i < n; ++i) pages_h[i] = 63 - i;
  int32_t *hchunks_d, *pages_d;
  cmalloc((void**)&hchunks_d, sizeof hchunks_h); cmalloc((void**)&pages_d, sizeof pages_h);
  cmemcpy(hchunks_d, hchunks_h, sizeof hchunks_h, 1); cmemcpy(pages_d, pages_h, sizeof pages_h, 1);
  int64_t ntok = n, cstart = 0, pstart = 0;
  for (int engine = 1; engine <= 4; ++engine) {
    strata_xfer x;
    memset(&x, 0, sizeof x);
    x.num_reqs = 1; x.layer_begin = 0; x.layer_end = L; x.engine = engine;
    x.num_tokens = &ntok; x.host_chunks = hchunks_d; x.chunk_start = &cstart; x.dev_pages = pages_d;
    x.page_start = &pstart; x.host_chunks_len = 3; x.dev_pages_len = n; x.host_chunks_host = hchunks_h;
    uint64_t ticket = 0;
    rc = strata_load(pool, &x, NULL, &ticket);
    EXPECT(rc == STRATA_OK, "load engine %d: %d %s", engine, rc, strata_last_error());
    csync();
    float ms = -1;
    EXPECT(strata_layer_elapsed_ms(pool, ticket, L - 1, &ms) == STRATA_OK && ms >= 0, "elapsed");
    /* token 33 (chunk list pos 2 -> host chunk 7, row 1), layer 1, V, lands in page 63-33 = 30 */
    unsigned char got[256], *want = (unsigned char*)host + 7 * (size_t)L * 2 * C * tok + ((1 * 2 + 1) * C + 1) * tok;
    cmemcpy(got, (char*)v[1] + 30 * tok, tok, 2);
    EXPECT(memcmp(got, want, tok) == 0, "engine %d: V row of token 33, layer 1 differs", engine);
  }
  strata_counters cnt;
  EXPECT(strata_get_counters(pool, &cnt) == STRATA_OK && cnt.operations == 4, "counters");
  EXPECT(strata_unregister_host_pool(pool) == STRATA_OK, "unregister");
  return 0;
}

int main(int argc, char** argv) {
  cpu_checks();
  ctl_checks();
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) gpu_checks();
  if (failures) {
    fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  printf("c_abi_smoke ok (%s)\n", argc > 1 ? argv[1] : "cpu");
  return 0;
}
