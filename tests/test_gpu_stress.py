"""Randomised stress parity (slow): 1500 cases drawn over EVERY axis at once — engine, SM quota,
row width (16-byte multiples and narrow rows, R29),
direction, page / chunk size, ragged counts and offsets, fragmentation, device row layout (NHD, HND,
padded), one or two KV buffers (R27), host head slices and head-major chunks (R28), consecutive or
permuted host chunks (strided copy runs), layer groups, layer ranges — each bit-exact against the
CPU oracle over whole buffers.  The per-feature suites pin each axis; this one looks for bad
interactions between them."""
import os

import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.gpu_helpers import GpuCase

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402

ENGINES = [st.STRATA_ENGINE_DEFAULT, st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_TMA_BULK,
           st.STRATA_ENGINE_DMA]


def _case(i):
    # STRESS_SEED_BASE shifts the whole draw (soak runs over fresh cases)
    rng = kvgen.rng_for(90000 + int(os.environ.get("STRESS_SEED_BASE", "0")) + i)
    kv = int(rng.choice([1, 2]))
    Ht = int(rng.choice([1, 2, 4, 8]))
    H = int(rng.choice([h for h in (1, 2, 4, 8) if h <= Ht]))
    h0 = int(rng.integers(0, Ht - H + 1))
    head_major = bool(rng.integers(0, 2)) and Ht > 1
    # 16-byte rows mostly; a fifth of the cases take narrow rows (R29: 3..72-byte heads)
    D = int(rng.choice([3, 10, 36, 72])) if rng.random() < 0.2 else int(rng.choice([64, 128, 576] if H == 1 else [64, 128]))
    if rng.random() < 0.15:   # rows of a non-power-of-two count of 16-byte vectors (ring: groups straddling row 32)
        D = int(rng.choice([24, 40, 48, 88, 200]))
    e = int(rng.choice([1, 2]))
    P = int(rng.choice([1, 2, 8, 16, 64]))
    C = int(rng.choice([1, 8, 64, 128]))
    L = int(rng.choice([1, 2, 4]))
    ns = [int(rng.integers(0, 3 * C + 9)) for _ in range(int(rng.choice([1, 2, 5])))]
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + int(rng.integers(1, 6))
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + int(rng.integers(1, 4))
    g = Geometry(L=L, H=H, D=D, e=e, P=P, C=C, num_pages=num_pages, num_chunks=num_chunks, kv=kv, Ht=Ht, h0=h0,
                 head_major=head_major)
    tok = g.token_bytes
    layout = rng.choice(["nhd", "hnd", "padded"])
    if layout == "hnd" and H > 1 and (D * e) % e == 0:
        strides = (H * P * D * e, D * e, P * D * e)
    elif layout == "padded":
        strides = (P * (tok + 2 * e) + 4 * e, tok + 2 * e, D * e)
    else:
        strides = None
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True,
                            chunk_frag=str(rng.choice(["perm", "identity"])))
    l0 = int(rng.integers(0, L))
    l1 = int(rng.integers(l0, L + 1))
    return dict(g=g, q=q, strides=strides, engine=ENGINES[i % len(ENGINES)], ctas=int(rng.choice([0, 1, 2, 4])),
                group=int(rng.choice([0, 1, 2, 3])), l0=l0, l1=l1, offload=bool(i % 2))


@pytest.mark.parametrize("i", range(1500))
def test_stress(i):
    f = _case(i)
    g, q = f["g"], f["q"]
    c = GpuCase(g, q, strides=f["strides"], seed=i, dev_fill="random" if f["offload"] else "canary")
    try:
        kw = dict(engine=f["engine"], num_ctas=f["ctas"], layer_group=f["group"])
        if f["offload"]:
            before = c.pool.host.copy()
            c.pool.offload(c.reqs, f["l0"], f["l1"], **kw)
            torch.cuda.synchronize()
            exp = c.expected_offload(before, f["l0"], f["l1"])
            assert np.array_equal(c.pool.host, exp), f
        else:
            c.pool.load(c.reqs, f["l0"], f["l1"], **kw)
            torch.cuda.synchronize()
            c.check_load(f["l0"], f["l1"])
    finally:
        c.close()
