/*
 * oracle.c — CPU oracle for the Strata KV-cache I/O path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load
 * this library.  The product path (libstrata) never links, loads or calls it, and this file shares
 * no code, header, table or helper with paper_2508_18572_b200/csrc/.
 *
 * What it computes (the plain definition; a copy, not an approximation — DESIGN.md §3):
 *
 *   LOAD:    for r, for i in [0,n_r), for l in [l0,l1), for kv in [0,KV), for h in [0,H):
 *              dev'[dst(r,i,l,kv,h) : +D*e] = host[src(r,i,l,kv,h) : +D*e]
 *            every other device byte is unchanged.
 *   OFFLOAD: the same loops with source and destination swapped; every other host byte unchanged.
 *
 *   ci = off_c[r] + i;  hc = host_chunks[chunk_start[r] + ci / C];  ho = ci % C
 *   pi = off_p[r] + i;  pg = dev_pages [page_start [r] + pi / P];  po = pi % P
 *   src(l,kv,h) = host + hc*chunk_bytes + ((l*KV + kv)*C + ho)*Ht*D*e + (h0 + h)*D*e   (token-major)
 *   src(l,kv,h) = host + hc*chunk_bytes + (((h0 + h)*L + l)*KV + kv)*C*D*e + ho*D*e   (head-major)
 *   chunk_bytes = L*KV*C*Ht*D*e
 *   dst(l,kv,h) = pool[l][kv] + pg*page_stride + po*token_stride + h*head_stride
 *
 *   The host tier holds Ht >= H heads per token; this GPU moves heads [h0, h0+H) (R28:
 *   Ht = H, h0 = 0 is the per-GPU tier of R13; a shared tier read by every TP rank has Ht = all
 *   KV heads).  Token-major is R1's [L][KV][C][Ht][D] chunk; head-major keeps [Ht][L][KV][C][D]:
 *   every head's part of a chunk is itself a one-head page-first chunk.
 *
 *   KV = 2 (a K and a V buffer per layer, MHA/GQA) or KV = 1 (one buffer per layer: MLA's latent
 *   cache, where K and V are both derived from one compressed vector per token — DESIGN.md R27).
 *
 * Passages followed:
 *   - GPU-assisted I/O moves KV between "CPU registered pinned memory" and GPU global memory
 *     (§4.2 "Efficient KV Cache I/O").
 *   - Host tier is page-first: "arranges layers of a page contiguously" (PAPER.md:286, :290,
 *     §4.2.1, fig:layout) -> host chunk = [L][K,V][C tokens][H][D] (reading R1).
 *   - Device pool is layer-first, "computation-friendly", paged: tokens map
 *     to non-contiguous pages (§2.2 "Memory Management of KV Cache").
 *   - The layout transform is address arithmetic (§4.2.1).
 *   - Chunk size arithmetic as in SPEC.md:171-179 (tier_store transfer_chunk_size).
 *
 * Index bounds are checked (returns -1 and touches nothing further); duplicates are not detected
 * (the last writer in loop order wins — callers never pass them, reading R8).
 *
 * nthreads > 1 parallelises the i loop with OpenMP; it is used only to time the oracle on the box's
 * host cores (SURVEY.md §8d "Oracle timing").  The loop body is identical.
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t L, H, D, e;        /* layers, KV heads on this GPU, head_dim, bytes per element */
    int64_t P, C;              /* device page size, host chunk size (tokens) */
    int64_t page_stride;       /* device bytes between pages */
    int64_t token_stride;      /* device bytes between tokens of a page */
    int64_t head_stride;       /* device bytes between heads of a token */
    int64_t num_pages;         /* device capacity in pages */
    int64_t num_chunks;        /* host capacity in chunks */
    int64_t KV;                /* buffers per layer: 2 (K, V) or 1 (MLA latent) */
    int64_t Ht, h0;            /* host heads per token (>= H) and this GPU's first head */
    int64_t head_major;        /* 0: chunk = [L][KV][C][Ht][D]; 1: [Ht][L][KV][C][D] */
} oracle_geom;

typedef struct {
    int64_t R;
    const int64_t* num_tokens;   /* [R] */
    const int32_t* host_chunks;  /* concatenated chunk lists */
    const int64_t* chunk_start;  /* [R] */
    const int32_t* dev_pages;    /* concatenated page lists */
    const int64_t* page_start;   /* [R] */
    const int32_t* chunk_offset; /* [R] or NULL (= 0) */
    const int32_t* page_offset;  /* [R] or NULL (= 0) */
    int64_t layer_begin, layer_end;
} oracle_reqs;

/* dir = 0: LOAD (host -> device image); dir = 1: OFFLOAD (device image -> host). */
static int oracle_move(const oracle_geom* g, uint8_t* host, uint8_t* const* k_img,
                       uint8_t* const* v_img, const oracle_reqs* q, int dir, int nthreads) {
    const int64_t row_bytes = g->D * g->e;            /* one head of one token */
    const int64_t chunk_bytes = g->L * g->KV * g->C * g->Ht * row_bytes;
    int bad = 0;
    (void)nthreads;
    for (int64_t r = 0; r < q->R; ++r) {
        const int64_t n = q->num_tokens[r];
        const int64_t oc = q->chunk_offset ? q->chunk_offset[r] : 0;
        const int64_t op = q->page_offset ? q->page_offset[r] : 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) if (nthreads > 1) reduction(|: bad)
#endif
        for (int64_t i = 0; i < n; ++i) {
            const int64_t ci = oc + i;
            const int64_t hc = q->host_chunks[q->chunk_start[r] + ci / g->C];
            const int64_t ho = ci % g->C;
            const int64_t pi = op + i;
            const int64_t pg = q->dev_pages[q->page_start[r] + pi / g->P];
            const int64_t po = pi % g->P;
            if (hc < 0 || hc >= g->num_chunks || pg < 0 || pg >= g->num_pages) {
                bad = 1;
                continue;
            }
            for (int64_t l = q->layer_begin; l < q->layer_end; ++l) {
                for (int64_t kv = 0; kv < g->KV; ++kv) {
                    uint8_t* pool = kv == 0 ? k_img[l] : v_img[l];
                    for (int64_t h = 0; h < g->H; ++h) {
                        const int64_t lkv = l * g->KV + kv;
                        uint8_t* hp = host + hc * chunk_bytes +
                                      (g->head_major ? (((g->h0 + h) * g->L * g->KV + lkv) * g->C + ho) * row_bytes
                                                     : (lkv * g->C + ho) * g->Ht * row_bytes + (g->h0 + h) * row_bytes);
                        uint8_t* dp = pool + pg * g->page_stride + po * g->token_stride +
                                      h * g->head_stride;
                        if (dir == 0) memcpy(dp, hp, (size_t)row_bytes);
                        else memcpy(hp, dp, (size_t)row_bytes);
                    }
                }
            }
        }
        if (bad) return -1;
    }
    return 0;
}

int oracle_load(const oracle_geom* g, const uint8_t* host, uint8_t* const* k_img, uint8_t* const* v_img,
                const oracle_reqs* q, int nthreads) {
    return oracle_move(g, (uint8_t*)host, k_img, v_img, q, 0, nthreads);
}

int oracle_offload(const oracle_geom* g, uint8_t* host, uint8_t* const* k_img, uint8_t* const* v_img,
                   const oracle_reqs* q, int nthreads) {
    return oracle_move(g, host, k_img, v_img, q, 1, nthreads);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
