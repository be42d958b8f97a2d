"""CPU checks of the host-side launch configuration (api.cu choose_config):
the rules the measurements chose, asserted as invariants over the BASELINE shapes.  No kernel
is launched; without a device the library assumes 148 SMs and ideal cluster packing."""

import pytest

from paper_2508_15601_b200 import api

SHAPES_8B = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
SHAPES_70B = [(10240, 8192), (8192, 8192), (57344, 8192), (8192, 28672)]
MIXTRAL = [(14336, 4096)]
SMS = 148


@pytest.mark.parametrize("M", [1, 8, 16, 17, 32, 33, 64])
@pytest.mark.parametrize("N,K", SHAPES_8B + SHAPES_70B + MIXTRAL)
def test_decode_configs_fit_one_wave(M, N, K):
    c = api.query_gemm_config(M, N, K)
    tiles = (N // 128) * ((M + c["tile_m"] - 1) // c["tile_m"])
    assert c["tile_m"] == (16 if M <= 16 else 32 if M <= 32 else 64)
    assert c["kind"] in (1, 2)
    assert c["grid_ctas"] <= SMS  # persistent / single wave
    if c["kind"] == 2 and c["split_k"] == 1:  # one CTA per tile: 70-100 % of the SMs busy
        assert 0.7 * SMS <= tiles <= SMS and c["grid_ctas"] == tiles
    elif c["kind"] == 2:  # cluster split-K: CS CTAs per tile, >= 8 chunks of 256 k each
        cs = c["split_k"]
        assert 2 <= cs <= 8 and c["grid_ctas"] == tiles * cs
        assert (K // 256) // cs >= 8
    else:  # stream-K over every SM (or fewer when there is less work)
        assert c["split_k"] == -c["grid_ctas"]


@pytest.mark.parametrize("M", [65, 100, 128, 200, 256, 300, 512])
@pytest.mark.parametrize("N,K", SHAPES_8B + SHAPES_70B + [(384, 4096), (640, 2048)])
def test_mid_m_configs(M, N, K):
    """65 <= M <= 512 with N % 256 == 0: CTA pairs (kind 5) with split-K over S pairs of one
    cluster -- the largest S in 4..2 whose clusters of 2 S CTAs are co-resident for every pair
    tile and leave >= 4 stages per split; with no such S the tiled kernel's configuration stays
    (N % 256 != 0 too)."""
    c = api.query_gemm_config(M, N, K)
    if N % 256 == 0:
        # (the CPU-side query has no device: co-resident clusters of 2 S = SMS // (2 S))
        ntile = 128 if M <= 128 else 256  # M <= 128: 128-token pair tiles
        pairs = (N // 256) * ((M + ntile - 1) // ntile)
        want = next((k for k in (4, 3, 2) if pairs <= SMS // (2 * k) and K // 64 >= 4 * k), 1)
        if want > 1:
            assert (c["kind"], c["tile_m"], c["split_k"]) == (5, ntile, want), c
            assert c["grid_ctas"] == (N // 128) * want * ((M + ntile - 1) // ntile)
            return
        if c["kind"] == 5:  # the tiled chooser's own unsplit 256-token tiles run on pairs
            assert c["split_k"] == 1 and c["tile_m"] == 256
            return
    assert c["kind"] == 0 and c["split_k"] >= 1  # the tiled kernel's cluster split (its caps apply)


def test_mid_m_pair_toggle_restores_tiled_split():
    api.set_prefill_pair(False)
    try:
        c = api.query_gemm_config(256, 4096, 4096)
    finally:
        api.set_prefill_pair(True)
    assert c["kind"] == 0 and c["tile_m"] == 128


@pytest.mark.parametrize("M", [1024, 2048, 4096, 8192])
@pytest.mark.parametrize("N,K", SHAPES_8B + SHAPES_70B)
def test_prefill_full_tiles(M, N, K):
    c = api.query_gemm_config(M, N, K)
    assert c["tile_m"] == 256
    assert c["kind"] == (5 if c["split_k"] == 1 and N % 256 == 0 else 0)
    tiles = (N // 128) * ((M + 255) // 256)
    assert c["split_k"] == (1 if tiles > 64 else c["split_k"])
    assert c["grid_ctas"] == tiles * c["split_k"]


@pytest.mark.parametrize("M", [1, 8, 9, 16])
@pytest.mark.parametrize("N,K", SHAPES_8B + SHAPES_70B + MIXTRAL + [(8192, 29568)])
def test_register_fed_configs(M, N, K):
    """Opt-in register-fed decode kernel (kind 3): cluster split for few tiles (S <= 8 CTAs per
    tile, >= 2 chunks each, one wave at two CTAs per SM), stream-K over 2 x SMs CTAs otherwise;
    32-bit range math (tiles x chunks x CTAs < 2^32)."""
    api.set_decode_path(2, 0)
    try:
        c = api.query_gemm_config(M, N, K)
    finally:
        api.set_decode_path(0, 0)
    tiles, kc = N // 128, (K + 255) // 256
    assert c["kind"] == 3 and c["tile_m"] == (8 if M <= 8 else 16)
    if c["split_k"] > 0:
        S = c["split_k"]
        assert tiles <= SMS and 1 <= S <= 8 and c["grid_ctas"] == tiles * S <= 2 * SMS
        assert S == 1 or kc >= 2 * S
    else:
        P = -c["split_k"]
        assert tiles > SMS and P == c["grid_ctas"] == min(2 * SMS, tiles * kc)
        assert tiles * kc * P < 2 ** 32
    assert api.query_gemm_config(M, N, K)["kind"] in (1, 2)  # the default path is the TMEM kernel


@pytest.mark.parametrize("M", [1024, 2048, 8192])
@pytest.mark.parametrize("N,K", SHAPES_8B)
def test_persistent_prefill_opt_in(M, N, K):
    assert api.query_gemm_config(M, N, K)["kind"] == 5  # default: the CTA-pair kernel
    api.set_prefill_persistent(True)
    try:
        c = api.query_gemm_config(M, N, K)
    finally:
        api.set_prefill_persistent(False)
    tiles = (N // 128) * ((M + 191) // 192)
    assert c["kind"] == 4 and c["tile_m"] == 192 and c["grid_ctas"] == min(SMS, tiles)


@pytest.mark.parametrize("M", [1024, 4096])
@pytest.mark.parametrize("N,K", SHAPES_8B + SHAPES_70B + [(384, 4096), (640, 2048)])
def test_pair_prefill_dispatch(M, N, K):
    """Kind 5 (CTA pairs) exactly where the tiled chooser picks unsplit 256-token tiles and
    N % 256 == 0; tm_set_prefill_pair(0) restores the tiled kernel with the same grid."""
    c = api.query_gemm_config(M, N, K)
    assert c["kind"] == (5 if N % 256 == 0 and c["split_k"] == 1 else 0)
    api.set_prefill_pair(False)
    try:
        t = api.query_gemm_config(M, N, K)
    finally:
        api.set_prefill_pair(True)
    assert t["kind"] == 0 and (t["tile_m"], t["split_k"], t["grid_ctas"]) == (c["tile_m"], c["split_k"], c["grid_ctas"])


def test_tp_allreduce_finalize_rejects_bad_arguments_without_a_device():
    """Argument validation happens before any CUDA call (runs on the CPU box)."""
    import ctypes
    lib = api.lib()
    P = (ctypes.c_void_p * 2)(16, 32)
    S = (ctypes.c_void_p * 2)(64, 128)
    for rank, world in ((0, 0), (2, 2), (0, 9), (-1, 2)):
        assert lib.tm_tp_allreduce_finalize(P, S, None, rank, world, 8, ctypes.c_void_p(256), None) != 0
    P1 = (ctypes.c_void_p * 1)(20)  # misaligned partial
    assert lib.tm_tp_allreduce_finalize(P1, S, None, 0, 1, 8, ctypes.c_void_p(256), None) != 0
