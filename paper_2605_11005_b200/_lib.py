"""ctypes binding of libdm_moe.so (include/dm_moe.h).

There is deliberately no fallback: if the sm_100a library is missing or a call
fails, this raises. Status codes map to exceptions the way the reference maps
its failure modes to typed errors (config.py:17-35, taskgraph.py:35, sim.py:34-39).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libdm_moe.so"

DM_CHUNK_TOKENS = 32
DM_ROW_ALIGN = 128
DM_GLU_BLOCK = 64      # gate/up interleave block of W13 / h13 / dh13 (dm_moe.h)
DM_MAX_TOPK = 16
DM_MAX_EXPERTS = 1024


class DMError(RuntimeError):
    """A dm_* entry point returned a non-zero status."""

    def __init__(self, fn: str, code: int, msg: str):
        self.fn, self.code, self.msg = fn, code, msg
        super().__init__(f"{fn} failed with status {code}: {msg}")


class DMShapeError(DMError, ValueError):
    pass


class DMLibraryMissing(RuntimeError):
    pass


_vp, _i32p, _f32p = C.c_void_p, C.c_void_p, C.c_void_p
_i, _f, _sz = C.c_int, C.c_float, C.c_size_t

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "dm_version": (_i, []),
    "dm_last_error_string": (C.c_char_p, []),
    "dm_num_sms": (_i, [_i]),
    "dm_launch_count": (C.c_longlong, []),
    "dm_capacity_rows_fn": (_i, [_i, _i, _i]),
    "dm_route_workspace_size_fn": (_sz, [_i, _i, _i, _i]),
    "dm_router_wgrad_workspace_size_fn": (_sz, [_i, _i, _i]),
    "dm_router_logits": (_i, [_vp, _f32p, _f32p, _i, _i, _i, _vp]),
    "dm_router_topk": (_i, [_f32p, _i, _i, _i, _i32p, _f32p, _i32p, _i32p, _vp]),
    "dm_expert_scan": (_i, [_i32p, _i, _i, _i32p, _i32p, _i32p, _vp]),
    "dm_permute": (_i, [_vp, _i32p, _i32p, _i32p, _i32p, _i32p, _i, _i, _i, _i, _i32p, _i32p, _vp, _vp]),
    "dm_route_and_dispatch": (_i, [_vp, _f32p, _i, _i, _i, _i, _vp, _i32p, _f32p, _i32p, _i32p,
                                   _i32p, _i32p, _vp, _vp]),
    "dm_grouped_w13_swiglu_fwd": (_i, [_vp, _vp, _i32p, _i, _i, _i, _i, _i, _vp, _vp, _vp]),
    "dm_grouped_w2_fwd": (_i, [_vp, _vp, _i32p, _i, _i, _i, _i, _i, _vp, _vp]),
    "dm_grouped_w2_dgrad_swiglu_bwd": (_i, [_vp, _vp, _vp, _i32p, _i, _i, _i, _i, _i, _vp, _vp]),
    "dm_grouped_w13_dgrad": (_i, [_vp, _vp, _i32p, _i, _i, _i, _i, _i, _vp, _vp]),
    "dm_grouped_wgrad": (_i, [_vp, _i, _vp, _i, _i32p, _i, _i, _i, _i, _f32p, _f, _vp]),
    "dm_grouped_w13_swiglu_fwd_ranges": (_i, [_vp, _vp, _i32p, _i32p, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp]),
    "dm_grouped_w2_fwd_ranges": (_i, [_vp, _vp, _i32p, _i32p, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    "dm_grouped_w2_dgrad_swiglu_bwd_ranges": (_i, [_vp, _vp, _vp, _i32p, _i32p, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    "dm_grouped_w13_dgrad_ranges": (_i, [_vp, _vp, _i32p, _i32p, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    "dm_batch_group_ranges": (_i, [_i32p, _i, _i, _i, _i, _i32p, _i32p, _vp]),
    "dm_debug_gemm_profile": (_i, [_vp]),
    "dm_debug_route_profile": (_i, [_vp]),
    "dm_combine_fwd": (_i, [_vp, _i32p, _f32p, _i, _i, _i, _vp, _vp, _vp]),
    "dm_combine_bwd": (_i, [_vp, _vp, _i32p, _f32p, _i32p, _i32p, _i, _i, _i, _i, _vp, _f32p,
                            _f32p, _f32p, _vp]),
    "dm_router_wgrad_sorted": (_i, [_vp, _i32p, _f32p, _i32p, _i32p, _i, _i, _i, _f32p, _f32p, _f, _vp]),
    "dm_permute_bwd": (_i, [_vp, _i32p, _i32p, _f32p, _f32p, _i, _i, _i, _i, _vp, _vp, _vp]),
    "dm_router_wgrad": (_i, [_vp, _i32p, _f32p, _i, _i, _i, _i, _f32p, _f32p, _f, _vp]),
    # fp32 mode (bytes_per_element 4)
    "dm_route_and_dispatch_f32": (_i, [_f32p, _f32p, _i, _i, _i, _i, _vp, _i32p, _f32p, _i32p, _i32p,
                                       _i32p, _i32p, _vp, _vp]),
    "dm_grouped_gemm_f32": (_i, [_vp, _vp, _i, _i32p, _i, _i, _i, _i, _i, _f32p, _vp]),
    "dm_combine_fwd_f32": (_i, [_f32p, _i32p, _f32p, _i, _i, _i, _f32p, _f32p, _vp]),
    "dm_combine_bwd_f32": (_i, [_f32p, _f32p, _i32p, _f32p, _i32p, _i32p, _i, _i, _i, _i, _vp, _f32p,
                                _f32p, _f32p, _vp]),
    "dm_permute_bwd_f32": (_i, [_f32p, _i32p, _i32p, _f32p, _f32p, _i, _i, _i, _i, _f32p, _f32p, _vp]),
    "dm_router_wgrad_sorted_f32": (_i, [_f32p, _i32p, _f32p, _i32p, _i32p, _i, _i, _i, _f32p, _f32p, _f, _vp]),
    "dm_swiglu_fwd_split": (_i, [_f32p, _i, _i, _vp, _vp]),
    "dm_swiglu_bwd_split": (_i, [_f32p, _f32p, _i, _i, _vp, _vp]),
    "dm_split3": (_i, [_f32p, _i, _i, _i, _i, _vp, _vp]),
    "dm_grouped_wgrad_strided": (_i, [_vp, _i, _i, _vp, _i, _i, _i32p, _i, _i, _i, _i, _f32p, _f, _vp]),
    "dm_attention_fwd": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _f32p, _vp]),
    "dm_attention_bwd": (_i, [_vp, _vp, _vp, _f32p, _i, _i, _i, _i, _i, _f32p, _vp, _vp]),
}

_lib = None


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load (once) and type the library. Raises DMLibraryMissing if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise DMLibraryMissing(
            f"{p} not found: build it with `python -m paper_2605_11005_b200.build` "
            "(there is no CPU fallback for the MoE hot path)"
        )
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    return load().dm_last_error_string().decode(errors="replace")


def call(name: str, *args) -> None:
    """Invoke a status-returning dm_* entry point; raise on failure."""
    rc = getattr(load(), name)(*args)
    if rc != 0:
        msg = last_error()
        if rc < 0:
            raise DMShapeError(name, rc, msg)
        raise DMError(name, rc, msg)


def launch_count() -> int:
    return int(load().dm_launch_count())


def capacity_rows(T: int, E: int, k: int) -> int:
    r = T * k + E * (DM_ROW_ALIGN - 1)
    return (r + DM_ROW_ALIGN - 1) // DM_ROW_ALIGN * DM_ROW_ALIGN


def num_chunks(T: int) -> int:
    return (T + DM_CHUNK_TOKENS - 1) // DM_CHUNK_TOKENS


DM_ROUTE_UNIT_TOKENS = 4


def route_workspace_size(T: int, H: int, E: int, k: int) -> int:
    """Mirror of dm_route_workspace_size (include/dm_moe.h); the last 4 KB hold the
    streaming router's completion counters, which must be zero on first use."""
    a = lambda v: (v + 255) & ~255  # noqa: E731
    nunit = (T + DM_ROUTE_UNIT_TOKENS - 1) // DM_ROUTE_UNIT_TOKENS
    return a(T * E * 4) + 2 * a(nunit * E * 4) + a(T * k * 4) + 4096


def router_wgrad_token_block(E: int) -> int:
    return 128 if E <= 16 else 512


def router_wgrad_workspace_size(T: int, H: int, E: int) -> int:
    """Mirror of dm_router_wgrad_workspace_size: partial blocks, then the sorted kernel's
    segment-completion counters (zero on first use)."""
    tb = router_wgrad_token_block(E)
    ntb = (T + tb - 1) // tb
    ctr = ((H + 1023) // 1024 * E + (H + 255) // 256) * 4
    return ntb * E * H * 4 + ((ctr + 255) & ~255)
