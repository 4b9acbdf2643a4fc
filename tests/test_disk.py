"""Disk tier (include/strata_disk.h) on CPU: no GPU involved.

Pinned against the layout definitions written out with numpy (page-first: disk chunk k is the
host chunk's bytes at offset k*chunk_bytes; layer-first: layer l of disk chunk k at
(l*num_chunks + k)*layer_bytes — PAPER.md:284-290 §4.2.1, fig:layout / fig:disk), round-trip
identity, and the cancellation contract (in-flight prefetch is terminated; finished
chunks are credited, untouched ones stay untouched)."""
import os

import numpy as np
import pytest

import kvgen
from paper_2508_18572_b200 import _lib
from paper_2508_18572_b200 import disk as sd


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2508_18572_b200 import build
    build.build()


def _geom(L=4, chunk_layer=8192, chunks=12):
    return L, L * chunk_layer, chunks


@pytest.mark.parametrize("layout", [sd.STRATA_DISK_PAGE_FIRST, sd.STRATA_DISK_LAYER_FIRST])
@pytest.mark.parametrize("o_direct", [False, True])
def test_writeback_layout_and_prefetch_round_trip(tmp_path, layout, o_direct):
    L, cb, n_disk = _geom()
    n_host = 10
    host = sd.aligned_empty(n_host * cb)
    host[:] = kvgen.random_bytes(kvgen.rng_for(1), host.size)
    rng = kvgen.rng_for(2)
    hsel = rng.permutation(n_host)[:7]
    dsel = rng.permutation(n_disk)[:7]
    path = str(tmp_path / "tier.bin")
    try:
        tier = sd.DiskTier(path, cb, L, n_disk, layout=layout, o_direct=o_direct, io_threads=3)
    except _lib.StrataError as e:
        if o_direct and e.code == _lib.STRATA_ERR_IO:
            pytest.skip("filesystem does not support O_DIRECT")
        raise
    with tier:
        rc, done, st = tier.wait(tier.writeback(host, hsel, dsel))
        assert rc == 0 and done == 7 and (st == sd.STRATA_DISK_DONE).all()
        img = np.fromfile(path, dtype=np.uint8)
        lb = cb // L
        for h, d in zip(hsel, dsel):
            chunk = host[h * cb:(h + 1) * cb]
            if layout == sd.STRATA_DISK_PAGE_FIRST:
                np.testing.assert_array_equal(img[d * cb:(d + 1) * cb], chunk)
            else:
                for l in range(L):
                    off = (l * n_disk + d) * lb
                    np.testing.assert_array_equal(img[off:off + lb], chunk[l * lb:(l + 1) * lb])
        # prefetch into a fresh tier at other host positions
        back = sd.aligned_empty(n_host * cb)
        back[:] = 0xA5
        hdst = rng.permutation(n_host)[:7]
        rc, done, st = tier.wait(tier.prefetch(back, dsel, hdst))
        assert rc == 0 and done == 7
        for hs, hd in zip(hsel, hdst):
            np.testing.assert_array_equal(back[hd * cb:(hd + 1) * cb], host[hs * cb:(hs + 1) * cb])
        untouched = sorted(set(range(n_host)) - set(hdst.tolist()))
        for h in untouched:
            assert (back[h * cb:(h + 1) * cb] == 0xA5).all()


def test_cancel_credits_finished_chunks(tmp_path):
    L, cb, n = 2, 2 * (1 << 20), 48           # 48 chunks of 2 MiB
    host = sd.aligned_empty(n * cb)
    host[:] = kvgen.random_bytes(kvgen.rng_for(3), host.size)
    path = str(tmp_path / "tier.bin")
    with sd.DiskTier(path, cb, L, n, io_threads=1) as tier:
        assert tier.wait(tier.writeback(host, range(n), range(n)))[0] == 0
        back = sd.aligned_empty(n * cb)
        back[:] = 0
        job = tier.prefetch(back, range(n), range(n))
        tier.cancel(job)
        rc, done, st = tier.wait(job)
        assert rc == 0
        assert done == int((st == sd.STRATA_DISK_DONE).sum())
        assert ((st == sd.STRATA_DISK_DONE) | (st == sd.STRATA_DISK_CANCELLED)).all()
        assert (st == sd.STRATA_DISK_CANCELLED).any(), "a single I/O thread cannot finish 96 MiB before cancel"
        for i in range(n):
            chunk = back[i * cb:(i + 1) * cb]
            if st[i] == sd.STRATA_DISK_DONE:
                np.testing.assert_array_equal(chunk, host[i * cb:(i + 1) * cb])
            else:
                assert not chunk.any(), "a cancelled chunk must not be written"


@pytest.mark.gpu
def test_disk_to_host_to_gpu(tmp_path):
    """The three tiers end to end: host chunks written back to disk, prefetched into a registered
    host tier at other positions, then strata_load'ed into the paged pool — bit-exact vs the oracle
    loading the original host bytes."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import oracle
    from tests.gpu_helpers import GpuCase
    g = kvgen.Geometry(4, 2, 64, 2, 4, 16, 256, 40)
    q = kvgen.make_requests(kvgen.rng_for(5), [300, 97], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    src = kvgen.random_bytes(kvgen.rng_for(6), g.host_bytes)       # the "original" host tier
    c = GpuCase(g, q, host_fill="none")
    try:
        c.pool.host[:] = 0
        cb = g.chunk_bytes
        with sd.DiskTier(str(tmp_path / "tier.bin"), cb, g.L, 64, io_threads=4) as tier:
            staging = sd.aligned_empty(g.host_bytes)
            staging[:] = src
            used = sorted(set(q.host_chunks.tolist()))
            disk_ids = [60 - i for i in range(len(used))]
            assert tier.wait(tier.writeback(staging, used, disk_ids))[0] == 0
            assert tier.wait(tier.prefetch(c.pool.host, disk_ids, used))[0] == 0
        c.pool.load(c.reqs)
        torch.cuda.synchronize()
        for l in range(g.L):
            ek, ev = [None] * g.L, [None] * g.L
            ek[l] = np.full(c.layer_bytes, 0xA5, np.uint8)
            ev[l] = np.full(c.layer_bytes, 0xA5, np.uint8)
            oracle.load(g, src, ek, ev, q, l, l + 1)
            assert np.array_equal(c.k[l].cpu().numpy(), ek[l])
            assert np.array_equal(c.v[l].cpu().numpy(), ev[l])
    finally:
        c.close()


def test_errors(tmp_path):
    path = str(tmp_path / "t.bin")
    with pytest.raises(_lib.StrataError) as e:
        sd.DiskTier(path, 1000, 3, 4)                      # L does not divide chunk_bytes
    assert e.value.code == _lib.STRATA_ERR_INVALID_ARG
    with pytest.raises(_lib.StrataError) as e:
        sd.DiskTier(path, 4096 * 3 + 16, 1, 4, o_direct=True)
    assert e.value.code == _lib.STRATA_ERR_ALIGNMENT
    with pytest.raises(_lib.StrataError) as e:
        sd.DiskTier(str(tmp_path / "missing.bin"), 4096, 1, 4, create=False)
    assert e.value.code == _lib.STRATA_ERR_IO
    with sd.DiskTier(path, 4096, 1, 4) as tier:
        host = sd.aligned_empty(4 * 4096)
        with pytest.raises(_lib.StrataError) as e:
            tier.prefetch(host, [4], [0])                  # disk chunk out of range
        assert e.value.code == _lib.STRATA_ERR_INDEX_RANGE
        with pytest.raises(_lib.StrataError) as e:
            sd.strata_disk_wait(tier.handle, 12345, 1)
        assert e.value.code == _lib.STRATA_ERR_INVALID_ARG
        rc, done, _ = tier.wait(tier.prefetch(host, [], []))
        assert rc == 0 and done == 0
