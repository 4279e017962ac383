"""Host logic of the tensor-core GEMM (csrc/prefill_gemm.cu plan_gemm, through adamk_prefill_gemm_plan): how a problem
is cut into tiles, last-wave column slices and K splits on a 148-SM B200.  No GPU: pure arithmetic in the library."""

import pytest

from paper_2605_11581_b200 import prefill as P
from paper_2605_11581_b200.plugin import AdamkError


def test_prefill_shapes_pick_the_fuller_last_wave():
    # Qwen2.5-7B, 4096 tokens.  gate/up: 16 x 148 pair tiles = exactly 32 waves of 74 pairs -> CTA pairs, no slicing
    p = P.gemm_plan(1, 4096, 3584, 2 * 18944, P.EPI_SWIGLU)
    assert p["tile"] == P.TILE_PAIR and p["tiles"] == 16 * 148 and p["tail_split"] == 1 and p["n_items"] == p["tiles"] and p["grid"] == 148
    # O projection: 448 one-CTA tiles = 3 waves + 4 tiles, cut into 4 slices of 64 columns each -> 3.25 waves (pairs: 3.5)
    p = P.gemm_plan(1, 4096, 3584, 3584, P.EPI_RESID)
    assert p["tile"] == P.TILE_256 and p["tiles"] == 448 and p["main_items"] == 444 and p["tail_split"] == 4 and p["n_items"] == 460
    # narrow outputs use 128-wide tiles; a forced pair tile slices its last wave in two
    assert P.gemm_plan(2, 300, 512, 328, P.EPI_STORE)["tile"] == P.TILE_128
    p = P.gemm_plan(1, 4096, 3584, 3584, P.EPI_RESID, tile_n=P.TILE_PAIR)
    assert p["tiles"] == 224 and p["main_items"] == 222 and p["tail_split"] == 2 and p["n_items"] == 226 and p["grid"] == 148
    # a single 128-token tile never goes to a pair
    assert P.gemm_plan(1, 128, 1536, 2048, P.EPI_STORE)["tile"] == P.TILE_256


def test_decode_shapes_split_k_and_stack_planes():
    # batch 8, two planes: 16 rows of one token tile; short weights take 128-wide tiles (half the one-warp epilogue):
    # 16 tiles x 8 K ranges of 3 k blocks = 128 CTAs
    p = P.gemm_plan(2, 8, 1536, 2048, P.EPI_ATOMIC)
    assert (p["tile"], p["tiles"], p["ksplit"], p["kb_per_split"], p["stacked"], p["grid"]) == (P.TILE_128, 16, 8, 3, 1, 128)
    p = P.gemm_plan(2, 8, 1536, 2048, P.EPI_ATOMIC, tile_n=P.TILE_256)
    assert (p["tiles"], p["ksplit"], p["kb_per_split"], p["grid"]) == (8, 12, 2, 96)
    # down projection: 12 tiles x 12 ranges; the 55 MB gate/up matrix stays on 256-wide tiles: 70 tiles x 2 ranges
    p = P.gemm_plan(2, 8, 8960, 1536, P.EPI_ATOMIC)
    assert (p["tile"], p["tiles"], p["ksplit"], p["grid"]) == (P.TILE_128, 12, 12, 144)
    p = P.gemm_plan(2, 8, 1536, 17920, P.EPI_ATOMIC)
    assert p["tile"] == P.TILE_256 and p["tiles"] == 70 and p["ksplit"] == 2 and p["grid"] == 140
    # LM head: more tiles than SMs -> no K split; batch 128 x 2 planes does not fit one tile -> two passes over K
    assert P.gemm_plan(2, 8, 1536, 151936, P.EPI_ATOMIC)["ksplit"] == 1
    assert P.gemm_plan(2, 128, 1536, 2048, P.EPI_ATOMIC)["stacked"] == 0 and P.gemm_plan(2, 64, 1536, 2048, P.EPI_ATOMIC)["stacked"] == 1
    assert P.gemm_plan(3, 42, 1536, 2048, P.EPI_ATOMIC)["stacked"] == 1 and P.gemm_plan(3, 43, 1536, 2048, P.EPI_ATOMIC)["stacked"] == 0
    # every split count the planner can produce covers K exactly
    for K in (64, 192, 1536, 3584, 8960, 18944):
        for N in (256, 1536, 4608):
            p = P.gemm_plan(1, 4, K, N, P.EPI_ATOMIC)
            kb = -(-K // 64)
            assert (p["ksplit"] - 1) * p["kb_per_split"] < kb <= p["ksplit"] * p["kb_per_split"]
            assert p["n_items"] * p["ksplit"] >= p["grid"] >= 1


def test_plan_rejects_what_the_launcher_rejects():
    for args in ((1, 16, 60, 64, P.EPI_STORE, 0), (4, 16, 64, 64, P.EPI_STORE, 0), (1, 16, 64, 64, 7, 0), (1, 16, 64, 64, P.EPI_STORE, 192),
                 (1, 16, 64, 2048, P.EPI_ATOMIC, P.TILE_PAIR), (1, 16, 64, 200, P.EPI_SWIGLU, P.TILE_256)):
        with pytest.raises(AdamkError):
            P.gemm_plan(*args)
