"""CPU ORACLE for the DisagMoE MoE layer — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module, and only as the checker or as the timed CPU
baseline. The product path (paper_2605_11005_b200) never imports it and has no
CPU fallback.

PARITY UNPINNED by the reference: arxiv/paper_2605_11005 ships no MoE
arithmetic, no golden vectors and no known-answer tests (the
package is a cost model + simulator, pkg/pyproject.toml:8). What this file
restates is the paper's layer semantics — top-k gating and a gate-weighted sum
of expert outputs, experts as SwiGLU FFNs (the "up- and
down-projection" GroupGEMMs of PAPER.md:291 extended to SwiGLU's three
matrices) — under the conventions of DESIGN.md §3. Routing (logits, top-k,
permutation) is delegated to oracle/moe_oracle.c, which reproduces the GPU's
fixed fp32 reduction order exactly; everything else is float64 numpy on the
exact bf16 input values. The regression KATs in tests/golden/ were generated
from this file by tests/golden/make_golden.py.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
ROW_ALIGN = 128  # include/dm_moe.h DM_ROW_ALIGN

# ------------------------------------------------------------------ bf16 helpers


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (uint16)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    return ((u + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def round_bf16(a: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(f32_to_bf16_bits(a))


# ------------------------------------------------------------------ C routing


def build_lib() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "moe_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_clib = None


def clib() -> C.CDLL:
    global _clib
    if _clib is None:
        _clib = C.CDLL(str(build_lib()))
        p = C.c_void_p
        _clib.dm_oracle_router.argtypes = [p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p]
        _clib.dm_oracle_router_logits.argtypes = [p, p, C.c_int, C.c_int, C.c_int, p]
        _clib.dm_oracle_router_logits_f32.argtypes = [p, p, C.c_int, C.c_int, C.c_int, p]
        _clib.dm_oracle_topk.argtypes = [p, C.c_int, C.c_int, C.c_int, p, p]
        _clib.dm_oracle_dispatch.argtypes = [p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, p]
        _clib.dm_oracle_dispatch.restype = C.c_int
    return _clib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def router(x_bits: np.ndarray, wg: np.ndarray, k: int):
    """Canonical-order logits, top-k ids (ties -> lower id) and softmax weights."""
    T, H = x_bits.shape
    E = wg.shape[0]
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    wg = np.ascontiguousarray(wg, dtype=np.float32)
    logits = np.empty((T, E), np.float32)
    idx = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float32)
    clib().dm_oracle_router(_ptr(x_bits), _ptr(wg), T, H, E, k, _ptr(logits), _ptr(idx), _ptr(w))
    return logits, idx, w


def router_f32(x: np.ndarray, wg: np.ndarray, k: int):
    """fp32 mode: canonical-order logits of fp32 activations, top-k, softmax weights."""
    T, H = x.shape
    E = wg.shape[0]
    x = np.ascontiguousarray(x, dtype=np.float32)
    wg = np.ascontiguousarray(wg, dtype=np.float32)
    logits = np.empty((T, E), np.float32)
    clib().dm_oracle_router_logits_f32(_ptr(x), _ptr(wg), T, H, E, _ptr(logits))
    idx, w = topk(logits, k)
    return logits, idx, w


def topk(logits: np.ndarray, k: int):
    T, E = logits.shape
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    idx = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float32)
    clib().dm_oracle_topk(_ptr(logits), T, E, k, _ptr(idx), _ptr(w))
    return idx, w


def capacity_rows(T: int, E: int, k: int, align: int = ROW_ALIGN) -> int:
    r = T * k + E * (align - 1)
    return (r + align - 1) // align * align


def dispatch(idx: np.ndarray, E: int, align: int = ROW_ALIGN, cap: int | None = None):
    """Stable counting sort by expert over token-major (t, j), padded blocks."""
    T, k = idx.shape
    cap = capacity_rows(T, E, k, align) if cap is None else cap
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    counts = np.empty(E, np.int32)
    pad_off = np.empty(E + 1, np.int32)
    row_map = np.empty((T, k), np.int32)
    src = np.empty(cap, np.int32)
    rc = clib().dm_oracle_dispatch(_ptr(idx), T, k, E, align, cap, _ptr(counts), _ptr(pad_off),
                                   _ptr(row_map), _ptr(src))
    if rc != 0:
        raise ValueError(f"oracle dispatch failed ({rc})")
    return counts, pad_off, row_map, src


def dispatch_numpy(idx: np.ndarray, E: int, align: int = ROW_ALIGN):
    """Independent numpy restatement of dispatch() (stable argsort), for cross-checks."""
    T, k = idx.shape
    flat = idx.reshape(-1).astype(np.int64)
    counts = np.bincount(flat, minlength=E).astype(np.int32)
    padded = (counts + align - 1) // align * align
    pad_off = np.concatenate([[0], np.cumsum(padded)]).astype(np.int32)
    order = np.argsort(flat, kind="stable")
    rank = np.empty_like(order)
    starts = np.concatenate([[0], np.cumsum(counts)])[:-1]
    sorted_e = flat[order]
    rank[order] = np.arange(flat.size) - starts[sorted_e]
    row_map = (pad_off[flat] + rank).reshape(T, k).astype(np.int32)
    return counts, pad_off, row_map


# ------------------------------------------------------------------ layer math


GLU_BLOCK = 64   # include/dm_moe.h DM_GLU_BLOCK


def interleave_w13(w1: np.ndarray, w3: np.ndarray, block: int = GLU_BLOCK) -> np.ndarray:
    """[E, D_e, H] gate/up -> the kernels' [E, 2*D_e, H] DM_GLU_BLOCK-row block interleave."""
    E, De, H = w1.shape
    out = np.empty((E, 2 * De, H), w1.dtype)
    v = out.reshape(E, De // block, 2, block, H)
    v[:, :, 0] = w1.reshape(E, De // block, block, H)
    v[:, :, 1] = w3.reshape(E, De // block, block, H)
    return out


def deinterleave_cols(h: np.ndarray, block: int = GLU_BLOCK):
    """[R, 2*D_e] interleaved columns -> (gate [R, D_e], up [R, D_e])."""
    R, two = h.shape
    De = two // 2
    v = h.reshape(R, De // block, 2, block)
    return v[:, :, 0].reshape(R, De), v[:, :, 1].reshape(R, De)


def _silu(g):
    return g / (1.0 + np.exp(-g))


@dataclass
class Forward:
    logits: np.ndarray
    idx: np.ndarray
    w: np.ndarray
    counts: np.ndarray
    pad_off: np.ndarray
    row_map: np.ndarray
    src: np.ndarray
    g: np.ndarray = field(repr=False)        # [R_total_padded, D_e] gate pre-activation
    u: np.ndarray = field(repr=False)
    act: np.ndarray = field(repr=False)
    y_perm: np.ndarray = field(repr=False)   # [cap, H]
    y: np.ndarray = field(repr=False)        # [T, H]


def _values(x) -> np.ndarray:
    """uint16 arrays are bf16 bit patterns (bf16 mode); float arrays are values (fp32 mode)."""
    return bf16_bits_to_f32(x) if x.dtype == np.uint16 else np.asarray(x, np.float32)


def moe_forward(x_bits, wg, w1, w3, w2, k, dtype=np.float64) -> Forward:
    """Full layer forward. x_bits: uint16 bf16 [T,H] (bf16 mode) or float32 [T,H]
    (fp32 mode, bytes_per_element 4); w1/w3 [E,D_e,H], w2 [E,H,D_e] as float arrays
    (bf16 values in bf16 mode); wg fp32 [E,H]."""
    T, H = x_bits.shape
    E = wg.shape[0]
    De = w1.shape[1]
    logits, idx, w = router(x_bits, wg, k) if x_bits.dtype == np.uint16 else router_f32(x_bits, wg, k)
    counts, pad_off, row_map, src = dispatch(idx, E)
    x = _values(x_bits).astype(dtype)
    cap = src.shape[0]
    g = np.zeros((cap, De), dtype)
    u = np.zeros((cap, De), dtype)
    y_perm = np.zeros((cap, H), dtype)
    for e in range(E):
        a, n = pad_off[e], counts[e]
        if n == 0:
            continue
        xe = x[src[a:a + n]]
        g[a:a + n] = xe @ w1[e].astype(dtype, copy=False).T
        u[a:a + n] = xe @ w3[e].astype(dtype, copy=False).T
    act = _silu(g) * u
    for e in range(E):
        a, n = pad_off[e], counts[e]
        if n:
            y_perm[a:a + n] = act[a:a + n] @ w2[e].astype(dtype, copy=False).T
    y = np.einsum("tk,tkh->th", w.astype(dtype), y_perm[row_map])
    return Forward(logits, idx, w, counts, pad_off, row_map, src, g, u, act, y_perm, y)


@dataclass
class Backward:
    dx: np.ndarray
    dwg: np.ndarray
    dw1: np.ndarray
    dw3: np.ndarray
    dw2: np.ndarray
    dw: np.ndarray        # d loss / d gate weight [T, k]
    dlogit: np.ndarray    # d loss / d selected logit [T, k]
    dy_perm: np.ndarray = field(repr=False)
    dx_perm: np.ndarray = field(repr=False)


def moe_backward(fwd: Forward, x_bits, wg, w1, w3, w2, dy, dtype=np.float64) -> Backward:
    """Gradients of <y, dy> w.r.t. x, W_g, W1, W3, W2 (dy given as float values)."""
    T, H = x_bits.shape
    E, De, _ = w1.shape
    x = _values(x_bits).astype(dtype)
    dy = np.asarray(dy, dtype)
    w = fwd.w.astype(dtype)
    rm = fwd.row_map
    cap = fwd.src.shape[0]
    dw = np.einsum("th,tkh->tk", dy, fwd.y_perm[rm])
    s = (w * dw).sum(axis=1, keepdims=True)
    dlogit = w * (dw - s)
    dy_perm = np.zeros((cap, H), dtype)
    dy_perm[rm.reshape(-1)] = (w[:, :, None] * dy[:, None, :]).reshape(-1, H)
    dx_perm = np.zeros((cap, H), dtype)
    dw1 = np.zeros((E, De, H), dtype)
    dw3 = np.zeros((E, De, H), dtype)
    dw2 = np.zeros((E, H, De), dtype)
    for e in range(E):
        a, n = fwd.pad_off[e], fwd.counts[e]
        if n == 0:
            continue
        sl = slice(a, a + n)
        g, u, act = fwd.g[sl], fwd.u[sl], fwd.act[sl]
        d_act = dy_perm[sl] @ w2[e].astype(dtype, copy=False)
        sg = 1.0 / (1.0 + np.exp(-g))
        dg = d_act * u * sg * (1.0 + g * (1.0 - sg))
        du = d_act * g * sg
        dx_perm[sl] = dg @ w1[e].astype(dtype, copy=False) + du @ w3[e].astype(dtype, copy=False)
        xe = x[fwd.src[sl]]
        dw1[e] = dg.T @ xe
        dw3[e] = du.T @ xe
        dw2[e] = dy_perm[sl].T @ act
    dx = dx_perm[rm].sum(axis=1) + np.einsum("tk,tkh->th", dlogit, wg.astype(dtype)[fwd.idx])
    dwg = np.zeros((E, H), dtype)
    np.add.at(dwg, fwd.idx.reshape(-1), (dlogit[:, :, None] * x[:, None, :]).reshape(-1, H))
    return Backward(dx, dwg, dw1, dw3, dw2, dw, dlogit, dy_perm, dx_perm)


def moe_stack(x_bits, layers, k, dy, inputs=None):
    """Stack of residual MoE blocks x_{l+1} = bf16(x_l + MoE_l(x_l)) (the runtime's
    layers > 1 model; the reference's tiny config has 2 layers, BASELINE configs[0]).
    layers: [(wg, w1, w3, w2)] per layer. Returns (y [T,H] float, dx, forwards,
    backwards, xs); the gradient entering layer l is bf16-rounded like the GPU's dx.

    inputs: optional bf16 bits of the layer inputs x_1..x_{L-1} as produced by the
    device under test. Routing is discontinuous, so a one-ulp difference in x_l can
    legitimately flip a near-tied expert; feeding the device's own x_l checks every
    layer bit-exactly on identical inputs (the chain itself is checked by comparing
    xs[l] with inputs[l-1] within tolerance)."""
    xs, fs = [x_bits], []
    for l, (wg, w1, w3, w2) in enumerate(layers):
        f = moe_forward(xs[-1] if l == 0 or inputs is None else inputs[l - 1], wg, w1, w3, w2, k)
        fs.append(f)
        base = xs[-1] if l == 0 or inputs is None else inputs[l - 1]
        xs.append(f32_to_bf16_bits((bf16_bits_to_f32(base) + f.y).astype(np.float32)))
    g = round_bf16(np.asarray(dy, np.float32))
    bs = [None] * len(layers)
    for l in reversed(range(len(layers))):
        xl = xs[l] if l == 0 or inputs is None else inputs[l - 1]
        b = moe_backward(fs[l], xl, *layers[l], g)
        bs[l] = b
        g = round_bf16((g + b.dx).astype(np.float32))
    return bf16_bits_to_f32(xs[-1]), g, fs, bs, xs


def normwise_rel_err(got, ref) -> float:
    """max|got - ref| / max|ref| (DESIGN.md §3 error metric)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max()
    if den == 0:
        return float(np.abs(got).max())
    return float(np.abs(got - ref).max() / den)


# ------------------------------------------------------------------ inputs


def make_inputs(T, H, E, k, De, seed=0, skew=0.0, tie_rows=()):
    """Seeded synthetic inputs: x~N(0,1) bf16, W_g~N(0,.02^2) fp32,
    W1/W3/W2~N(0,.02^2) bf16, dy~N(0,1) bf16.
    skew > 0: every token gets a shared component mu (0.5 per element) and the first
    k experts' gate rows gain skew * mu/|mu|^2, i.e. a +skew logit bias — large skew
    routes (nearly) all tokens to experts 0..k-1 and leaves the rest empty.
    tie_rows: W_g row pairs (a, b) made identical, forcing bit-exact logit ties."""
    rng = np.random.default_rng(seed)
    xf = rng.standard_normal((T, H), dtype=np.float32)
    wg = (rng.standard_normal((E, H), dtype=np.float32) * 0.02).astype(np.float32)
    if skew:
        mu = np.full(H, 0.5, np.float32)
        xf = xf + mu
        wg[:k] += (np.float32(skew) * mu / np.float32(mu @ mu)).astype(np.float32)
    for a, b in tie_rows:
        wg[b] = wg[a]
    x_bits = f32_to_bf16_bits(xf)
    w1 = round_bf16(rng.standard_normal((E, De, H), dtype=np.float32) * 0.02)
    w3 = round_bf16(rng.standard_normal((E, De, H), dtype=np.float32) * 0.02)
    w2 = round_bf16(rng.standard_normal((E, H, De), dtype=np.float32) * 0.02)
    dy = round_bf16(rng.standard_normal((T, H), dtype=np.float32))
    return x_bits, wg, w1, w3, w2, dy


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
