"""Second, independent oracle: numpy fancy indexing over reshaped views.  TEST INFRASTRUCTURE ONLY.

It computes the same plain definition as ``oracle.c`` but by a different route:
instead of a per-(token, layer, kv, head) memcpy loop it views

    host  as  [num_chunks, L, KV, C, H, D*e]              (page-first host chunk, PAPER.md:286, :290;
                                                            KV = 2 for K,V or 1 for an MLA latent)
    pool  as  [num_pages, P, H, D*e] with the byte strides  (layer-first paged pool, PAPER.md:284,
                                                            :653-655)

and moves all tokens of a request with one fancy-indexed assignment per (layer, kv).  It shares no
code with ``oracle.c`` or with the CUDA path.  Meant for tiny pools (it materialises index arrays).
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np
from numpy.lib.stride_tricks import as_strided


def _host_view(host: np.ndarray, g) -> np.ndarray:
    """[num_chunks][L][KV][C][H][D*e] view of this GPU's heads [h0, h0+H) of the host tier.

    Token-major chunk: [L][K,V][C][Ht][D*e] ("arranges layers of a page contiguously");
    head-major chunk: [Ht][L][K,V][C][D*e], exposed token-major by moving the head axis (R28).
    """
    Ht = getattr(g, "Ht", 0) or g.H
    h0 = getattr(g, "h0", 0)
    if getattr(g, "head_major", False):
        v = host.reshape(g.num_chunks, Ht, g.L, _kv(g), g.C, g.D * g.e)[:, h0:h0 + g.H]
        return np.moveaxis(v, 1, 4)
    return host.reshape(g.num_chunks, g.L, _kv(g), g.C, Ht, g.D * g.e)[:, :, :, :, h0:h0 + g.H]


def _kv(g) -> int:
    return getattr(g, "kv", 2)


def _pool_view(buf: np.ndarray, g, strides) -> np.ndarray:
    page_stride, token_stride, head_stride = strides
    return as_strided(buf, shape=(g.num_pages, g.P, g.H, g.D * g.e),
                      strides=(page_stride, token_stride, head_stride, 1), writeable=True)


def _token_coords(q, r: int, g):
    """Per-token (hc, ho, pg, po) of request r: page-table indirection."""
    n = int(q.num_tokens[r])
    i = np.arange(n, dtype=np.int64)
    ci = int(q.chunk_offset[r]) + i
    pi = int(q.page_offset[r]) + i
    cs, ps = int(q.chunk_start[r]), int(q.page_start[r])
    hc = q.host_chunks[cs + ci // g.C].astype(np.int64)
    pg = q.dev_pages[ps + pi // g.P].astype(np.int64)
    return hc, ci % g.C, pg, pi % g.P


def _check(g, hc, pg):
    if hc.size and (hc.min() < 0 or hc.max() >= g.num_chunks):
        raise IndexError("host chunk index out of range")
    if pg.size and (pg.min() < 0 or pg.max() >= g.num_pages):
        raise IndexError("device page index out of range")


def load(g, host: np.ndarray, k_imgs: Sequence[np.ndarray], v_imgs: Sequence[np.ndarray], q,
         layer_begin: int, layer_end: int, strides=None) -> None:
    """LOAD in place into the device images k_imgs[l] / v_imgs[l] (uint8, one per layer)."""
    strides = strides or _nhd(g)
    hv = _host_view(host, g)
    for r in range(q.R):
        hc, ho, pg, po = _token_coords(q, r, g)
        _check(g, hc, pg)
        for l in range(layer_begin, layer_end):
            for kv, imgs in ((0, k_imgs), (1, v_imgs))[:_kv(g)]:
                dev = _pool_view(imgs[l], g, strides)
                dev[pg, po] = hv[hc, l, kv, ho]


def offload(g, host: np.ndarray, k_imgs: Sequence[np.ndarray], v_imgs: Sequence[np.ndarray], q,
            layer_begin: int, layer_end: int, strides=None) -> None:
    """OFFLOAD in place into the host pool image ``host`` (uint8)."""
    strides = strides or _nhd(g)
    hv = _host_view(host, g)
    for r in range(q.R):
        hc, ho, pg, po = _token_coords(q, r, g)
        _check(g, hc, pg)
        for l in range(layer_begin, layer_end):
            for kv, imgs in ((0, k_imgs), (1, v_imgs))[:_kv(g)]:
                dev = _pool_view(imgs[l], g, strides)
                hv[hc, l, kv, ho] = dev[pg, po]


def _nhd(g):
    """Default NHD device rows: token_stride = H*D*e, head_stride = D*e, page_stride = P*H*D*e."""
    tok = g.H * g.D * g.e
    return (g.P * tok, tok, g.D * g.e)
