"""kvgen — seeded synthetic inputs for the Strata I/O path.

This module is shared by the oracle tests, the GPU parity tests and ``bench.py``. It holds NONE of
the method's arithmetic: no address transform, no page-table gather/scatter, no copy. It only draws
the inputs the paper's workloads are shaped like:

* KV geometries of the paper's models (§5.1 "Models"),
* cached-prefix lengths shaped like LooGLE / NarrativeQA (Table 1, avg. 21,613 and
  54,797 input tokens),
* fragmented device page allocations (§1 "paging causes data fragmentation";
  the distribution is not given — DESIGN.md reading R14),
* host chunk lists over a host pool, and uniform random payload bytes (every bit pattern, incl. NaN
  payloads and -0.0 for fp16/bf16).

Every randomized draw uses ``numpy.random.Generator(PCG64(seed))`` with ``seed`` passed explicitly.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence

import numpy as np

__all__ = [
    "Geometry", "Requests", "CONFIGS", "geometry", "rng_for", "pages_needed", "chunks_needed",
    "make_requests", "fill_random", "random_bytes", "churn_free_list", "head_slice",
]


@dataclasses.dataclass(frozen=True)
class Geometry:
    """KV geometry of one GPU's share of a model (DESIGN.md §2 notation).

    L layers, H KV heads held by this GPU, D head_dim, e bytes per element, P device page size in
    tokens, C host chunk size in tokens, pool capacities in pages / chunks.
    """
    L: int
    H: int
    D: int
    e: int
    P: int
    C: int
    num_pages: int
    num_chunks: int
    kv: int = 2   # KV buffers per layer: 2 (K and V: MHA/GQA), 1 (MLA's shared latent, R27)
    # Host tier heads (R28): the tier holds Ht >= H heads per token (0 = H) and this GPU
    # moves heads [h0, h0+H) of them; head_major stores a chunk as [Ht][L][KV][C][D] instead of the
    # token-major [L][KV][C][Ht][D]: each head's part is a one-head page-first chunk.
    Ht: int = 0
    h0: int = 0
    head_major: bool = False

    @property
    def host_heads(self) -> int:
        return self.Ht or self.H

    @property
    def token_bytes(self) -> int:
        """S_tok = H*D*e: bytes of one token's K (or V) in one layer."""
        return self.H * self.D * self.e

    @property
    def chunk_bytes(self) -> int:
        """One host chunk holds C tokens of every layer's K and V for all Ht host heads:
        L*kv*C*Ht*D*e bytes."""
        return self.L * self.kv * self.C * self.host_heads * self.D * self.e

    @property
    def host_bytes(self) -> int:
        return self.num_chunks * self.chunk_bytes

    @property
    def layer_buffer_bytes(self) -> int:
        """Bytes of one layer's K (or V) device buffer with dense NHD rows."""
        return self.num_pages * self.P * self.token_bytes


# The five BASELINE.json configs (SURVEY.md §8d "Concrete synthetic inputs").
# n: cached-prefix tokens per request; tp: KV-head shards (H below is the per-GPU slice).
CONFIGS: Dict[str, dict] = {
    "tiny": dict(L=2, H=2, D=64, e=2, P=16, C=64, n=[1024], num_pages=256, num_chunks=64, tp=1),
    "llama8b_32k": dict(L=32, H=8, D=128, e=2, P=1, C=64, n=[32768], num_pages=40960,
                        num_chunks=640, tp=1),
    # LooGLE-like lengths in 16K-64K, deliberately not page aligned.
    "qwen14b_batch8": dict(L=48, H=8, D=128, e=2, P=1, C=64,
                           n=[16397, 20483, 24593, 32771, 40973, 49157, 57349, 65521],
                           num_pages=384064, num_chunks=6010, tp=1),
    # Llama-3.1-70B: 8 KV heads, TP=8 -> 1 head per GPU (per-rank geometry).
    "llama70b_tp8": dict(L=80, H=1, D=128, e=2, P=1, C=64, n=[131072], num_pages=163840,
                         num_chunks=2560, tp=8),
    # DeepSeek-V3 MLA latent cache (one buffer per layer: kv_lora_rank 512 + rope 64 = 576 bf16 per
    # token; 61 layers), 32K-token prefix.  A variant beyond BASELINE.json's configs;
    # the latent is replicated, not head-sharded, under TP, so multi-GPU runs are replicas.
    # Llama-3.1-70B TP=8 from ONE host tier holding all 8 KV heads in head-major chunks (R28): each
    # rank moves its head h0 = rank of it; 32K-token prefix (a 12.5 GiB shared tier).
    "llama70b_tp8_shared": dict(L=80, H=1, D=128, e=2, P=1, C=64, n=[32768], num_pages=40960,
                                num_chunks=640, tp=8, Ht=8, head_major=True),
    "deepseek_v3_mla": dict(L=61, H=1, D=576, e=2, P=1, C=64, n=[32768], num_pages=40960,
                            num_chunks=640, tp=1, kv=1),
}


def geometry(name: str, P: Optional[int] = None, **over) -> Geometry:
    """Geometry of a named config; ``P`` overrides the page size keeping the slot capacity."""
    c = dict(CONFIGS[name])
    c.update(over)
    slots = c["num_pages"] * c["P"]
    if P is not None and P != c["P"]:
        c["num_pages"] = -(-slots // P)
        c["P"] = P
    return Geometry(L=c["L"], H=c["H"], D=c["D"], e=c["e"], P=c["P"], C=c["C"],
                    num_pages=c["num_pages"], num_chunks=c["num_chunks"], kv=c.get("kv", 2), Ht=c.get("Ht", 0),
                    h0=c.get("h0", 0), head_major=c.get("head_major", False))


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def pages_needed(offset: int, n: int, P: int) -> int:
    """Pages a request of n tokens starting at in-page offset ``offset`` occupies (capacity
    accounting rounds up: S:159-160, 33 tokens at P=32 occupy 2 pages)."""
    return -(-(offset + n) // P) if n > 0 else 0


def chunks_needed(offset: int, n: int, C: int) -> int:
    return -(-(offset + n) // C) if n > 0 else 0


@dataclasses.dataclass
class Requests:
    """One strata_xfer worth of request tables (all host numpy arrays).

    ``host_chunks`` / ``dev_pages`` are the concatenated per-request lists; ``chunk_start`` /
    ``page_start`` index into them; offsets are the token offsets inside the first chunk / page.
    """
    num_tokens: np.ndarray    # int64 [R]
    host_chunks: np.ndarray   # int32 [sum chunks]
    chunk_start: np.ndarray   # int64 [R]
    dev_pages: np.ndarray     # int32 [sum pages]
    page_start: np.ndarray    # int64 [R]
    chunk_offset: np.ndarray  # int32 [R]
    page_offset: np.ndarray   # int32 [R]

    @property
    def R(self) -> int:
        return int(self.num_tokens.shape[0])

    @property
    def total_tokens(self) -> int:
        return int(self.num_tokens.sum())


def churn_free_list(rng: np.random.Generator, num_pages: int, P: int, rounds: int = 1000,
                    lo: int = 1024, hi: int = 65536, occupancy: float = 0.7) -> np.ndarray:
    """Allocator-churn free list (SURVEY.md §8c generator spec, fragmentation mode ii).

    Start from a sorted free list; each round allocates a request of U[lo,hi] tokens from the
    front and, while more than ``occupancy`` of the pool is in use, frees a uniformly random live
    request by appending its pages at the back. Returns the final free list (int64 page ids).
    """
    from collections import deque
    free = deque(range(num_pages))
    live: List[List[int]] = []
    in_use = 0
    for _ in range(rounds):
        need = -(-int(rng.integers(lo, hi + 1)) // P)
        while in_use > occupancy * num_pages and live:
            victim = live.pop(int(rng.integers(0, len(live))))
            free.extend(victim)
            in_use -= len(victim)
        if need > len(free):
            continue
        got = [free.popleft() for _ in range(need)]
        live.append(got)
        in_use += need
    for v in live:  # return everything: the benchmark allocates from the churned order
        free.extend(v)
    return np.fromiter(free, dtype=np.int64, count=len(free))


def mean_run_length(pages: np.ndarray) -> float:
    """Mean length of runs of adjacent page ids (reported with churn mode)."""
    if pages.size == 0:
        return 0.0
    breaks = np.count_nonzero(np.diff(pages) != 1)
    return pages.size / (breaks + 1)


def make_requests(rng: np.random.Generator, n: Sequence[int], P: int, C: int, num_pages: int,
                  num_chunks: int, frag: str = "perm", offsets: bool = False,
                  chunk_frag: str = "perm") -> Requests:
    """Draw request tables for the token counts ``n``.

    frag: "perm" (uniform random permutation of pool pages, mode i), "churn" (allocator churn,
    mode ii) or "identity" (pages 0,1,2,... in order). chunk_frag: "perm" or "identity" for host
    chunks. offsets: draw off_p ~ U[0,P) and off_c ~ U[0,C) (fuzz tests); else 0.
    Destinations never repeat (reading R8: duplicates are a caller error).
    """
    R = len(n)
    n_arr = np.asarray(n, dtype=np.int64)
    off_p = rng.integers(0, P, size=R).astype(np.int32) if offsets else np.zeros(R, np.int32)
    off_c = rng.integers(0, C, size=R).astype(np.int32) if offsets else np.zeros(R, np.int32)
    npg = [pages_needed(int(off_p[r]), int(n_arr[r]), P) for r in range(R)]
    nch = [chunks_needed(int(off_c[r]), int(n_arr[r]), C) for r in range(R)]
    tot_p, tot_c = sum(npg), sum(nch)
    if tot_p > num_pages or tot_c > num_chunks:
        raise ValueError(f"pool too small: need {tot_p} pages / {tot_c} chunks, "
                         f"have {num_pages} / {num_chunks}")
    if frag == "perm":
        pages = rng.permutation(num_pages)[:tot_p]
    elif frag == "churn":
        pages = churn_free_list(rng, num_pages, P)[:tot_p]
    elif frag == "identity":
        pages = np.arange(tot_p)
    else:
        raise ValueError(frag)
    if chunk_frag == "perm":
        chunks = rng.permutation(num_chunks)[:tot_c]
    elif chunk_frag == "identity":
        chunks = np.arange(tot_c)
    else:
        raise ValueError(chunk_frag)
    page_start = np.zeros(R, np.int64)
    chunk_start = np.zeros(R, np.int64)
    if R:
        page_start[1:] = np.cumsum(npg)[:-1]
        chunk_start[1:] = np.cumsum(nch)[:-1]
    return Requests(num_tokens=n_arr, host_chunks=chunks.astype(np.int32), chunk_start=chunk_start,
                    dev_pages=pages.astype(np.int32), page_start=page_start,
                    chunk_offset=off_c, page_offset=off_p)


def random_bytes(rng: np.random.Generator, size: int) -> np.ndarray:
    """Uniform random bytes (every bit pattern occurs)."""
    return rng.integers(0, 256, size=size, dtype=np.uint8)


def fill_random(buf: np.ndarray, seed: int, block: int = 1 << 26) -> None:
    """Fill a large uint8 buffer in place with seeded pseudo-random bytes, fast.

    One 64 MiB block is drawn from PCG64(seed); block b of the buffer is that block XOR a per-block
    64-bit constant drawn from the same generator, so every block differs. Used for multi-GiB pools
    where drawing every byte from PCG64 would take minutes.
    """
    assert buf.dtype == np.uint8 and buf.ndim == 1
    rng = rng_for(seed)
    nbytes = buf.shape[0]
    base = rng.bit_generator.random_raw(block // 8).astype(np.uint64)
    nblocks = -(-nbytes // block)
    keys = rng.bit_generator.random_raw(nblocks).astype(np.uint64)
    for b in range(nblocks):
        lo = b * block
        hi = min(nbytes, lo + block)
        m = (hi - lo) // 8
        if m:
            dst = buf[lo:lo + m * 8].view(np.uint64)
            np.bitwise_xor(base[:m], keys[b], out=dst)
        if lo + m * 8 < hi:
            tail = hi - (lo + m * 8)
            buf[lo + m * 8:hi] = base[:1].view(np.uint8)[:tail] ^ np.uint8(b & 0xFF)


def head_slice(rank: int, world: int, H_total: int) -> range:
    """KV heads owned by ``rank`` of ``world`` tensor-parallel ranks (contiguous blocks, the way TP
    shards KV heads; §5.1). Requires world | H_total."""
    if H_total % world:
        raise ValueError(f"{H_total} KV heads do not shard over {world} ranks")
    h = H_total // world
    return range(rank * h, (rank + 1) * h)
