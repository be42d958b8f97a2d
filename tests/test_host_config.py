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
@pytest.mark.parametrize("N,K", SHAPES_8B + SHAPES_70B)
def test_mid_m_cluster_split(M, N, K):
    c = api.query_gemm_config(M, N, K)
    assert c["kind"] == 0
    nt = c["tile_m"]
    if M <= 128:
        assert nt == 128
    elif M <= 256:
        assert nt == (128 if 2 * (N // 128) <= SMS else 256)
    else:
        assert nt == 256
    tiles = (N // 128) * ((M + nt - 1) // nt)
    s = c["split_k"]
    # the largest split in 2..4 that keeps tiles * split <= 128 CTAs, else no split
    want = next((k for k in (4, 3, 2) if tiles * k <= 128), 1)
    assert s == want, (tiles, s, want)


@pytest.mark.parametrize("M", [1024, 2048, 4096, 8192])
@pytest.mark.parametrize("N,K", SHAPES_8B + SHAPES_70B)
def test_prefill_full_tiles(M, N, K):
    c = api.query_gemm_config(M, N, K)
    assert (c["kind"], c["tile_m"]) == (0, 256)
    tiles = (N // 128) * ((M + 255) // 256)
    assert c["split_k"] == (1 if tiles > 64 else c["split_k"])
    assert c["grid_ctas"] == tiles * c["split_k"]
