"""CPU-only checks of the C-ABI boundary: the library loads and exports every symbol
include/tm_w4a16.h declares, with the declared shape/size helpers behaving as documented.
No kernel is launched (no GPU here)."""

import ctypes
import os
import re

from paper_2508_15601_b200 import api, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(tm_[a-z0-9_]+)\s*\(", src))
    return names


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    assert {"tm_pack_w4", "tm_gemm_w4a16"} <= names
    assert len(names) >= 10


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(build.build())
    missing = [n for n in _declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_symbol():
    assert _declared_functions() <= set(api._SIGS)


def test_host_only_entry_points():
    lib = api.lib()
    assert api.pack_w4_bytes(4096, 28672, 128) == 4096 * 28672 // 2
    assert lib.tm_pack_w4_bytes(100, 128, 128) == -2   # TM_ERR_UNSUPPORTED_SHAPE
    assert lib.tm_pack_w4_bytes(128, 100, 128) == -2
    assert lib.tm_pack_w4_bytes(128, 128, 32) == -2
    assert lib.tm_pack_w4_bytes(0, 128, 128) == -1
    assert api.lib().tm_status_string(-3) == b"TM_ERR_MISALIGNED"
    assert "LAYOUT v1" in api.version()
    # null pointers are rejected before any CUDA call
    assert lib.tm_pack_w4(None, None, None, 128, 128, 128, None, None) == -1
    assert lib.tm_gemm_w4a16(None, None, None, None, None, 1, 128, 128, None) == -1


def test_config_selection_host_logic():
    api.set_gemm_override(0, 0)
    c = api.query_gemm_config(16, 28672, 4096)  # decode, many tiles: persistent stream-K
    assert c["tile_m"] == 16 and c["split_k"] < 0 and c["grid_ctas"] == -c["split_k"] and c["kind"] == 1
    assert c["grid_ctas"] <= 224 * 16  # never more CTAs than 256-k chunks
    c = api.query_gemm_config(16, 4096, 4096)  # decode, 32 tiles x 16 chunks: 2 CTAs per tile
    assert c == dict(tile_m=16, split_k=2, grid_ctas=64, kind=2)
    c = api.query_gemm_config(16, 4096, 14336)  # 32 tiles x 56 chunks: 4 CTAs per tile
    assert c == dict(tile_m=16, split_k=4, grid_ctas=128, kind=2)
    api.set_decode_cluster(1)  # never: stream-K
    assert api.query_gemm_config(16, 4096, 4096)["kind"] == 1
    api.set_decode_cluster(3)
    assert api.query_gemm_config(16, 4096, 4096) == dict(tile_m=16, split_k=3, grid_ctas=96, kind=2)
    api.set_decode_cluster(0)
    c = api.query_gemm_config(1, 128, 256)
    assert c["grid_ctas"] == 1  # one tile of one chunk
    c = api.query_gemm_config(4096, 4096, 4096)
    assert c["tile_m"] == 256 and c["split_k"] == 1 and c["grid_ctas"] == 32 * 16
    api.set_gemm_override(64, 3)
    assert api.query_gemm_config(5, 256, 1024) == dict(tile_m=64, split_k=3, grid_ctas=6, kind=0)
    api.set_gemm_override(0, 0)
    try:
        api.set_gemm_override(48, 0)
        raise AssertionError("tile 48 must be rejected")
    except api.TMError:
        pass


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2508_15601_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f
                assert "oracle/" not in src.replace("oracle/ ", ""), f
