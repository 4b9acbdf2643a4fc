"""Test helpers: device-image construction and the tagged-coordinate host pattern.

The tag pattern restates the host layout reading R1 by numpy
broadcasting, independently of both oracles and of the CUDA path.
"""
from __future__ import annotations

import numpy as np

CANARY = 0xA5


def nhd_strides(g):
    tok = g.H * g.D * g.e
    return (g.P * tok, tok, g.D * g.e)


def hnd_strides(g):
    """Head-major pages: [page][head][token][dim]."""
    return (g.H * g.P * g.D * g.e, g.D * g.e, g.P * g.D * g.e)


def layer_bytes(g, strides=None):
    ps, ts, hs = strides or nhd_strides(g)
    return g.num_pages * ps


def dev_images(g, fill=CANARY, rng=None, strides=None):
    """Host images of the device pool: (k_imgs, v_imgs), one uint8 buffer per layer."""
    nb = layer_bytes(g, strides)
    if rng is None:
        k = [np.full(nb, fill, np.uint8) for _ in range(g.L)]
        v = [np.full(nb, fill, np.uint8) for _ in range(g.L)]
    else:
        k = [rng.integers(0, 256, nb, dtype=np.uint8) for _ in range(g.L)]
        v = [rng.integers(0, 256, nb, dtype=np.uint8) for _ in range(g.L)]
    return k, v


def tagged_host(g) -> np.ndarray:
    """Host pool where every 16-byte vector encodes its own coordinates as 4 x u32:
    (chunk, (layer<<1)|kv, token_in_chunk, (head<<16)|vec)  with vec < D*e/16.
    Layout: [num_chunks][L][KV][C][H][D*e/16] vectors (reading R1; KV = g.kv, 2 or 1 for MLA)."""
    vph = g.D * g.e // 16
    assert vph >= 1 and g.D * g.e % 16 == 0
    shape = (g.num_chunks, g.L, getattr(g, "kv", 2), g.C, g.H, vph)
    c, l, kv, t, h, v = np.meshgrid(*[np.arange(s, dtype=np.uint32) for s in shape], indexing="ij")
    tags = np.stack([c, (l << 1) | kv, t, (h << 16) | v], axis=-1)
    return np.ascontiguousarray(tags).view(np.uint8).reshape(-1)


def slots_of(q, r, g):
    """Device slot (page*P + offset) and host (chunk, pos) of every token of request r — the
    page-table semantics restated for checks."""
    out = []
    n = int(q.num_tokens[r])
    for i in range(n):
        pi = int(q.page_offset[r]) + i
        ci = int(q.chunk_offset[r]) + i
        pg = int(q.dev_pages[int(q.page_start[r]) + pi // g.P])
        hc = int(q.host_chunks[int(q.chunk_start[r]) + ci // g.C])
        out.append((pg, pi % g.P, hc, ci % g.C))
    return out
