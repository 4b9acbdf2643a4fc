"""Host logic of the ring engine's launch planning, no GPU: the per-CTA geometry
strata_load / strata_offload use (csrc/transfer.cpp ring_geometry, exported as
strata_test_ring_geometry).  Pins the measured defaults and the invariants the
kernel relies on: W divides S (stage s belongs to warp s % W, ring.cu), the ring fits the shared
memory budget, a piece is one host run of at most C tokens and 64 rows."""
import itertools

import pytest

import paper_2508_18572_b200 as st

SMEM = 232448 - 1024   # the 227 KB opt-in limit of sm_100 less some headroom, as the library requests
KIB = 1024


def geo(tok, C=64, gran=16, smem=SMEM, inflight=224 * KIB, ctas=2, warps=8, target=16 * KIB):
    return st.strata_test_ring_geometry(tok, C, gran, smem, inflight, ctas, warps, target)


def test_llama8b_default():
    # 2 KiB rows, 224 KiB over 2 CTAs, 16 KiB pieces: 8-row pieces, 7 stages, 7 scatter warps
    assert geo(2048) == (8, 7, 7, 16384)


def test_short_rows_default():
    # 70B TP=8 rank rows (256 B) at their default 320 KiB over 4 CTAs: 64-row pieces, 5 stages
    R, S, W, sb = geo(256, inflight=320 * KIB, ctas=4)
    assert (R, sb) == (64, 16384) and S == 5 and W == 5


def test_prime_depth_never_leaves_one_warp():
    # 13 stages requested with 8 warps: 13 has no divisor in 2..8, so the ring drops to 12 stages / 6
    # warps instead of running ONE scatter warp (16.4 GB/s measured, profiles/r02/sweep70/)
    R, S, W, sb = geo(2048, inflight=13 * 16 * KIB, ctas=1)
    assert (S, W) == (12, 6)


def test_mla_rows_round_to_128_bytes():
    # 1152-byte latent rows: 14 rows per 16 KiB piece, stage padded to a 128-byte multiple
    R, S, W, sb = geo(1152, inflight=320 * KIB)
    assert R == 14 and sb == (14 * 1152 + 127) // 128 * 128


def test_narrow_rows_stage_holds_the_aligned_span():
    R, S, W, sb = geo(72, gran=8)
    assert sb >= R * 72 + 30 and sb % 128 == 0


def test_no_ring_when_two_stages_do_not_fit():
    assert geo(2048, smem=2 * 16384) is None          # header + 2 stages > budget
    assert geo(2048, smem=2 * 16384 + 4096) is not None


def test_bad_arguments():
    with pytest.raises(st.StrataError):
        geo(0)
    with pytest.raises(st.StrataError):
        geo(2048, ctas=0)


@pytest.mark.parametrize("tok,C,gran", [(2048, 64, 16), (256, 64, 16), (1152, 64, 16), (4096, 16, 16),
                                         (16, 256, 16), (72, 64, 8), (64 * 1024, 64, 16)])
def test_invariants_over_a_grid(tok, C, gran):
    for inflight, ctas, warps, target, smem in itertools.product(
            [16 * KIB, 96 * KIB, 224 * KIB, 448 * KIB, 4 * 1024 * KIB], [1, 2, 3, 4, 16],
            [1, 2, 3, 7, 8, 16], [4 * KIB, 16 * KIB, 64 * KIB], [48 * KIB, 100 * KIB, SMEM]):
        g = geo(tok, C, gran, smem, inflight, ctas, warps, target)
        if g is None:
            continue
        R, S, W, sb = g
        assert 1 <= R <= min(C, 64)
        assert R == 1 or R * tok <= target                # a piece is at most the target (or one row)
        assert sb >= R * tok and sb % 128 == 0
        assert 2 <= S <= 16 and S % W == 0                 # W divides S
        assert 2 * W >= min(min(warps, 16), S)             # at least half the warps asked for
        assert S * sb <= smem                              # the stages fit (the header is < 1 KiB)
