"""CPU checks of the C ABI boundary: the sm_100a library builds, loads without a
GPU, exports every symbol include/dm_moe.h declares, and rejects bad shapes with
the documented negative status codes before touching the device."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2605_11005_b200 import _lib, build

HEADER = Path(__file__).resolve().parents[1] / "include" / "dm_moe.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"DM_API\s+[\w\s\*]+?\b(dm_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert len(syms) >= 20
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table and header drifted"


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_and_sizes(lib):
    assert lib.dm_version() == 1
    assert lib.dm_capacity_rows_fn(4096, 8, 2) == _lib.capacity_rows(4096, 8, 2)
    assert lib.dm_route_workspace_size_fn(4096, 4096, 8, 2) == _lib.route_workspace_size(4096, 4096, 8, 2)
    assert lib.dm_router_wgrad_workspace_size_fn(4096, 4096, 8) == _lib.router_wgrad_workspace_size(4096, 4096, 8)


@pytest.mark.parametrize("T,E,k", [(1, 1, 1), (4096, 8, 2), (4096, 256, 8), (32768, 8, 2), (5, 300, 16)])
def test_capacity_bounds_any_routing(T, E, k):
    cap = _lib.capacity_rows(T, E, k)
    assert cap % _lib.DM_ROW_ALIGN == 0
    # worst case: every expert gets a count that is 1 mod 128
    worst = sum(((c + 127) // 128) * 128 for c in [T * k // E] * E)
    assert worst <= cap


def test_shape_errors_are_negative_codes_without_gpu(lib):
    # H not a multiple of 8 -> DM_ERR_ALIGN, topk too large -> DM_ERR_SHAPE; both checked on the host
    rc = lib.dm_router_logits(None, None, None, 16, 12, 4, None)
    assert rc == -3 and "multiple of 8" in _lib.last_error()
    rc = lib.dm_router_topk(None, 16, 8, 17, None, None, None, None, None)
    assert rc == -1
    rc = lib.dm_grouped_w13_swiglu_fwd(None, None, None, 8, 8, 100, 4096, 14336, None, None, None)
    assert rc == -1 and "cap_rows" in _lib.last_error()
    rc = lib.dm_grouped_wgrad(None, 100, None, 256, None, 1, 8, 1024, 1024, None, ctypes.c_float(0.0), None)
    assert rc == -1
    with pytest.raises(_lib.DMShapeError):
        _lib.call("dm_combine_fwd", None, None, None, 4, 10, 2, None, None, None)
    # attention: head_dim 128 only; seq_len a multiple of 128 dividing T; nh a multiple of nkv
    rc = lib.dm_attention_bwd(None, None, None, None, 256, 256, 4, 2, 64, None, None, None)
    assert rc == -1 and "head_dim" in _lib.last_error()
    rc = lib.dm_attention_bwd(None, None, None, None, 300, 200, 4, 2, 128, None, None, None)
    assert rc == -1 and "seq_len" in _lib.last_error()
    rc = lib.dm_attention_bwd(None, None, None, None, 256, 256, 6, 4, 128, None, None, None)
    assert rc == -1
    rc = lib.dm_attention_fwd(None, 256, 256, 4, 2, 64, None, None, None)
    assert rc == -1
    # batched GEMM ranges: cap must be 128-aligned; b_div must divide G
    rc = lib.dm_batch_group_ranges(None, 4, 8, 100, 1, None, None, None)
    assert rc == -1 and "batch_group_ranges" in _lib.last_error()
    rc = lib.dm_grouped_w2_fwd_ranges(None, None, None, None, 10, 5, 3, 1024, 4096, 1024, None, None)
    assert rc == -4 and "b_div" in _lib.last_error()


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(_lib.DMLibraryMissing):
        _lib.load(tmp_path / "nope.so")


def test_sass_is_blackwell_native(lib):
    import shutil
    import subprocess

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump unavailable")
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "grouped GEMMs must issue tcgen05.mma"
    assert "UTMALDG" in sass, "operands must be staged by TMA"
    assert "LDTM" in sass, "epilogue must read accumulators from TMEM"
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass), "no legacy mma.sync path"
