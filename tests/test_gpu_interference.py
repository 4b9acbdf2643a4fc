"""NEXT-1: interference of the zero-copy load with co-running prefill and decode.

The paper's claim for its I/O kernel: "nearly 50 GB/s" with "less than 5 % and 10 % slowdown on
prefill and decode" (§4.2, fig:interference), from as few as one or two CTAs
(PAPER.md:258).  On this B200 box the decode half of that joint claim does not reproduce for any
engine: HBM-bound decode slows with the host reads kept in flight (no-store and exclusive-SM variants
cost the same), and the link needs ~200 KiB in flight to run near its ceiling — measured frontier
(profiles/r02/interference_*.jsonl): ~29 GB/s +5.6 %, ~44 +11 %, ~48.6 +12.5 %,
~51.2 +15.6 % (LDG at 2 CTAs: 50.9 +12.1 %).  The decode slowdown splits into a memory-side part and a per-kernel-boundary part: the same 8 GiB HBM
read issued as 4 / 32 / 128 / 512 reduction kernels slows +6 / +17 / +103 / +163 % beside the default
load (each kernel boundary ~20 us longer; a contiguous copy-engine memcpy: ~14 us), graph-replayed or
not (profiles/r02/interference/decode_split_kernels.jsonl).  The memory-side part — `decode_long`,
the read as 4 kernels — meets the paper's < 10 % at the default point.  With the paper's decode pass run by a real
decode kernel (`attn`: FlashInfer paged decode attention, 16 requests x 4K, 32 layers) the default
slows it +6.6 ... +7.4 % beside the paper's own configuration (the LDG engine, 2 CTAs x 1024
threads) and +8.4 ... +10.2 % beside the ring engine at the same ~51 GB/s (profiles/r02/interf_real/,
pace/, s3a/); the library default for large loads follows that result.  Three operating points are
asserted:

  default        the library default (LDG, 2 CTAs x 1024 threads): >= 85 % of the link
                 with the paper's budget on its decode pass — prefill <= +5 %, attention decode
                 <= +10 % — and the read proxies (<= +10 % long kernels, <= +16 % 32 kernels);
  ring           the ring engine (2 CTAs, 224 KiB in flight): >= 85 % of the link, prefill <= +5 %,
                 decode <= +20 % (the frontier at that rate), attention decode <= +12 %;
  budget         one ring CTA: the paper's budget, prefill <= +5 % and decode <= +10 %,
                 at >= 50 % of the link.

Method (round 1's settled "cool-down" protocol, tools/interference.py): the proxy alone and the
proxy beside a continuous load alternate for 3 rounds, 1 s idle before every block; medians.

  prefill proxy  bf16 GEMMs of a Llama-3.1-8B layer for 2 x 4K tokens (tensor-core bound)
  decode proxy   a read of 16 x 4K tokens of Llama-8B KV per layer for 32 layers (HBM bound)
  decode_long    the same 8 GiB read as 4 kernels (the memory-side interference alone)
  attn           FlashInfer paged decode attention, 16 requests x 4K tokens, 32 layers (the real kernel)
"""
import statistics
import time

import pytest

import kvgen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402

POINTS = {   # operating point: (engine, num_ctas, min fraction of the link, {proxy: max slowdown})
    "default": (0, 0, 0.85, {"prefill": 0.05, "decode": 0.16, "decode_long": 0.10, "attn": 0.10}),
    "ring": (st.STRATA_ENGINE_TMA, 0, 0.85, {"prefill": 0.05, "decode": 0.20, "decode_long": 0.10, "attn": 0.12}),
    "budget": (st.STRATA_ENGINE_TMA, 1, 0.50, {"prefill": 0.05, "decode": 0.10, "decode_long": 0.10, "attn": 0.05}),
}


def _prefill():
    M = 8192
    shapes = [(4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096)]
    xs = {k: torch.randn(M, k, dtype=torch.bfloat16, device="cuda") for k, _ in shapes}
    ws = [torch.randn(k, n, dtype=torch.bfloat16, device="cuda") for k, n in shapes]
    return lambda: [torch.matmul(xs[k], w) for (k, _), w in zip(shapes, ws)]


def _decode(kernels=32):
    kv = [torch.randn(32 // kernels * 16 * 4096 * 8 * 128 * 2, dtype=torch.bfloat16, device="cuda")
          for _ in range(kernels)]
    return lambda: [t.sum(dtype=torch.float32) for t in kv]


def _attn():
    """The paper's decode pass (16 requests x 4K) with a real decode kernel: FlashInfer
    paged decode attention over Llama-3.1-8B heads (32 query / 8 KV heads, d = 128, bf16, page 16,
    scattered pages), one kernel per layer, 32 layers of 256 MiB of KV each."""
    w, q, out, caches = _attn_parts()
    return lambda: [w.run(q, c, out=out) for c in caches]


def _attn_parts():
    flashinfer = pytest.importorskip("flashinfer")
    batch, ctx, page = 16, 4096, 16
    npg = batch * ctx // page
    gen = torch.Generator(device="cuda").manual_seed(7)
    caches = [(torch.randn(npg, page, 8, 128, dtype=torch.bfloat16, device="cuda", generator=gen),
               torch.randn(npg, page, 8, 128, dtype=torch.bfloat16, device="cuda", generator=gen)) for _ in range(32)]
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(torch.empty(256 << 20, dtype=torch.uint8, device="cuda"), "NHD")
    w.plan(torch.arange(0, npg + 1, ctx // page, dtype=torch.int32, device="cuda"),
           torch.randperm(npg, device="cuda", generator=gen).to(torch.int32),
           torch.full((batch,), page, dtype=torch.int32, device="cuda"), 32, 8, 128, page,
           q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
    q = torch.randn(batch, 32, 128, dtype=torch.bfloat16, device="cuda", generator=gen)
    out = torch.empty_like(q)
    return w, q, out, caches


def _time(fn, stream, reps=15):
    evs = []
    with torch.cuda.stream(stream):
        fn()
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            evs.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


@pytest.mark.parametrize("point", ["default", "ring", "budget"])
@pytest.mark.parametrize("proxy", ["prefill", "decode", "decode_long", "attn"])
def test_interference_operating_points(proxy, point):
    engine, ctas, min_frac, budget = POINTS[point]
    g = kvgen.geometry("llama8b_32k")
    q = kvgen.make_requests(kvgen.rng_for(1), [32768], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    try:
        reqs = st.Requests.from_kvgen(q)
        lo, hi = torch.cuda.Stream.priority_range()
        io, comp = torch.cuda.Stream(priority=hi), torch.cuda.Stream(priority=lo)
        bytes_load = 2 * g.L * 32768 * g.token_bytes
        scratch = torch.empty(bytes_load // g.L, dtype=torch.uint8, device="cuda")
        ts = []
        for _ in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(io)
            st.strata_baseline_contiguous(pool.handle, st.STRATA_H2D, scratch.data_ptr(), 0, scratch.numel(), io)
            b.record(io)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        link = scratch.numel() / (statistics.median(ts[2:]) / 1e3) / 1e9
        fn = {"prefill": _prefill, "decode": _decode, "decode_long": lambda: _decode(4), "attn": _attn}[proxy]()
        load = lambda: pool.load(reqs, stream=io, engine=engine, num_ctas=ctas)  # noqa: E731
        load()
        torch.cuda.synchronize()
        alone, co, io_gbs = [], [], []
        for _ in range(3):
            time.sleep(1.0)
            alone.append(_time(fn, comp))
            n_loads = max(2, int(alone[-1] * 16 / (bytes_load / (min_frac * link) / 1e6)) + 2)
            time.sleep(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(io)
            for _ in range(n_loads):
                load()
            b.record(io)
            co.append(_time(fn, comp))
            b.synchronize()
            io_gbs.append(n_loads * bytes_load / (a.elapsed_time(b) / 1e3) / 1e9)
        slow = statistics.median(c / a_ - 1 for c, a_ in zip(co, alone))
        rate = statistics.median(io_gbs)
        print(f"{point} {proxy}: slowdown {slow:+.3f} (rounds {[round(c / a_ - 1, 3) for c, a_ in zip(co, alone)]}), "
              f"load beside it {rate:.1f} GB/s of a {link:.1f} GB/s link")
        assert slow <= budget[proxy], f"{point}: {proxy} slowdown {slow:.3f} > {budget[proxy]}"
        assert rate >= min_frac * link, f"{point}: co-run load {rate:.1f} GB/s < {min_frac:.0%} of the {link:.1f} GB/s link"
    finally:
        pool.close()


def _decode_step():
    """A whole Llama-3.1-8B decode step at batch 16 x 4K context (~290 kernels): per layer RMSNorm,
    QKV GEMM, FlashInfer paged decode attention, O GEMM, RMSNorm, gate/up GEMM, SiLU x up, down GEMM
    (random bf16 weights; KV as in _attn)."""
    attn_layers = _attn_parts()
    w, q, out, caches = attn_layers
    B, Hd = 16, 4096
    gen = torch.Generator(device="cuda").manual_seed(8)
    mk = lambda *s: torch.randn(*s, dtype=torch.bfloat16, device="cuda", generator=gen) * 0.02  # noqa: E731
    layers = [(mk(Hd, 6144), mk(Hd, Hd), mk(Hd, 2 * 14336), mk(14336, Hd), mk(Hd), mk(Hd)) for _ in caches]
    x = torch.randn(B, Hd, dtype=torch.bfloat16, device="cuda", generator=gen)

    def run():
        h = x
        for (wqkv, wo, wgu, wd, n1, n2), c in zip(layers, caches):
            a = torch.nn.functional.rms_norm(h, (Hd,), n1)
            qkv = a @ wqkv
            w.run(qkv[:, :Hd].reshape(B, 32, 128), c, out=out)
            h = h + out.reshape(B, Hd) @ wo
            a = torch.nn.functional.rms_norm(h, (Hd,), n2)
            gu = a @ wgu
            h = h + (torch.nn.functional.silu(gu[:, :14336]) * gu[:, 14336:]) @ wd
        return h
    return run


@pytest.mark.parametrize("proxy,budget", [("attn", 0.05), ("decode_step", 0.12)])
def test_decode_aware_quota(proxy, budget):
    """strata_set_load_quota around the co-runner (the serving engine's decode step) beside default
    loads: measured +2.3 % (attention decode) and +8.5 % (a whole decode step, +23.4 % without the
    quota) with the load at 47 / 42 GB/s (profiles/r02/quota/).  Asserted: the budgets here and the
    load >= 70 % of the link while the co-runner loops."""
    g = kvgen.geometry("llama8b_32k")
    q = kvgen.make_requests(kvgen.rng_for(1), [32768], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    try:
        reqs = st.Requests.from_kvgen(q)
        lo, hi = torch.cuda.Stream.priority_range()
        io, comp = torch.cuda.Stream(priority=hi), torch.cuda.Stream(priority=lo)
        pool.set_load_quota(0, stream=comp)
        bytes_load = 2 * g.L * 32768 * g.token_bytes
        scratch = torch.empty(bytes_load // g.L, dtype=torch.uint8, device="cuda")
        ts = []
        for _ in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(io)
            st.strata_baseline_contiguous(pool.handle, st.STRATA_H2D, scratch.data_ptr(), 0, scratch.numel(), io)
            b.record(io)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        link = scratch.numel() / (statistics.median(ts[2:]) / 1e3) / 1e9
        inner = {"attn": _attn, "decode_step": _decode_step}[proxy]()

        def fn():
            pool.set_load_quota(1, stream=comp)
            inner()
            pool.set_load_quota(0, stream=comp)
        load = lambda: pool.load(reqs, stream=io)  # noqa: E731
        load()
        torch.cuda.synchronize()
        alone, co, io_gbs = [], [], []
        for _ in range(3):
            time.sleep(1.0)
            alone.append(_time(fn, comp))
            n_loads = max(2, int(alone[-1] * 16 / (bytes_load / (0.7 * link) / 1e6)) + 2)
            time.sleep(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(io)
            for _ in range(n_loads):
                load()
            b.record(io)
            co.append(_time(fn, comp))
            b.synchronize()
            io_gbs.append(n_loads * bytes_load / (a.elapsed_time(b) / 1e3) / 1e9)
        slow = statistics.median(c / a_ - 1 for c, a_ in zip(co, alone))
        rate = statistics.median(io_gbs)
        print(f"quota-bracketed {proxy}: slowdown {slow:+.3f} (rounds {[round(c / a_ - 1, 3) for c, a_ in zip(co, alone)]}), "
              f"load beside it {rate:.1f} GB/s of a {link:.1f} GB/s link")
        assert slow <= budget, f"{proxy} slowdown {slow:.3f} > {budget}"
        assert rate >= 0.7 * link, f"co-run load {rate:.1f} GB/s < 70 % of the {link:.1f} GB/s link"
    finally:
        pool.close()

