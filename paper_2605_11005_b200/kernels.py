"""Thin torch-tensor wrappers over the dm_* C ABI (one function per entry point).

Tensors must already live on the current CUDA device; the calls are
stream-ordered on torch's current stream and never synchronise. Shapes and
dtypes are checked here so misuse fails loudly before reaching the ABI.
"""

from __future__ import annotations

import torch

from . import _lib

BF16 = torch.bfloat16
F32 = torch.float32


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("dm kernels need CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("dm kernels need contiguous tensors")
    return t.data_ptr()


def _stream(stream: torch.cuda.Stream | None = None) -> int:
    """cudaStream_t of `stream`, or of the current stream of the current device. The
    raw-handle query avoids torch.cuda.current_stream()'s Python overhead (~10 us), which
    dominated the host side of small-shape AF-Pipe iterations."""
    if stream is not None:
        return stream.cuda_stream
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def _check(t: torch.Tensor, dtype: torch.dtype, shape: tuple, name: str) -> None:
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")


# ------------------------------------------------------------------ dispatch
def router_logits(x, wg, logits, stream=None):
    T, H = x.shape
    E = wg.shape[0]
    _check(x, BF16, (T, H), "x"); _check(wg, torch.float32, (E, H), "wg")
    _check(logits, torch.float32, (T, E), "logits")
    _lib.call("dm_router_logits", _ptr(x), _ptr(wg), _ptr(logits), T, H, E, _stream(stream))


def router_topk(logits, k, idx, w, rank, chunk_hist, stream=None):
    T, E = logits.shape
    _check(idx, torch.int32, (T, k), "idx"); _check(w, torch.float32, (T, k), "w")
    _check(rank, torch.int32, (T, k), "rank")
    _check(chunk_hist, torch.int32, (_lib.num_chunks(T), E), "chunk_hist")
    _lib.call("dm_router_topk", _ptr(logits), T, E, k, _ptr(idx), _ptr(w), _ptr(rank), _ptr(chunk_hist),
              _stream(stream))


def expert_scan(chunk_hist, T, counts, pad_off, chunk_base, stream=None):
    nch, E = chunk_hist.shape
    _check(counts, torch.int32, (E,), "counts"); _check(pad_off, torch.int32, (E + 1,), "pad_off")
    _check(chunk_base, torch.int32, (nch, E), "chunk_base")
    _lib.call("dm_expert_scan", _ptr(chunk_hist), T, E, _ptr(counts), _ptr(pad_off), _ptr(chunk_base),
              _stream(stream))


def permute(x, idx, rank, chunk_base, counts, pad_off, row_map, src_token, x_perm, stream=None):
    T, H = x.shape
    k = idx.shape[1]
    E = counts.shape[0]
    _check(row_map, torch.int32, (T, k), "row_map")
    if x_perm.dtype != BF16 or x_perm.shape[1] != H:
        raise ValueError("x_perm must be bf16 [cap, H]")
    _lib.call("dm_permute", _ptr(x), _ptr(idx), _ptr(rank), _ptr(chunk_base), _ptr(counts), _ptr(pad_off), T,
              H, E, k, _ptr(row_map), _ptr(src_token), _ptr(x_perm), _stream(stream))


def route_and_dispatch(x, wg, k, workspace, idx, w, counts, pad_off, row_map, src_token, x_perm, stream=None):
    T, H = x.shape
    E = wg.shape[0]
    _check(x, BF16, (T, H), "x"); _check(wg, torch.float32, (E, H), "wg")
    need = _lib.route_workspace_size(T, H, E, k)
    if workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"route workspace too small ({need} bytes needed)")
    _lib.call("dm_route_and_dispatch", _ptr(x), _ptr(wg), T, H, E, k, _ptr(workspace), _ptr(idx), _ptr(w),
              _ptr(counts), _ptr(pad_off), _ptr(row_map), _ptr(src_token), _ptr(x_perm), _stream(stream))


# --------------------------------------------------------------- expert FFN
# group_off: int32 [G+1] row offsets (128-aligned); group g uses weight matrix g % E.
def _groups(group_off, E):
    G = group_off.numel() - 1
    if group_off.dtype != torch.int32 or G < E:
        raise ValueError("group_off must be int32 [G+1] with G >= number of experts")
    return G


def w13_swiglu_fwd(x_perm, w13, group_off, h13, act, stream=None):
    cap, H = x_perm.shape
    E, two_de, _ = w13.shape
    De = two_de // 2
    _check(h13, BF16, (cap, 2 * De), "h13"); _check(act, BF16, (cap, De), "act")
    _lib.call("dm_grouped_w13_swiglu_fwd", _ptr(x_perm), _ptr(w13), _ptr(group_off), _groups(group_off, E), E,
              cap, H, De, _ptr(h13), _ptr(act), _stream(stream))


def w2_fwd(act, w2, group_off, y_perm, stream=None):
    cap, De = act.shape
    E, H, _ = w2.shape
    _check(y_perm, BF16, (cap, H), "y_perm")
    _lib.call("dm_grouped_w2_fwd", _ptr(act), _ptr(w2), _ptr(group_off), _groups(group_off, E), E, cap, H, De,
              _ptr(y_perm), _stream(stream))


def w2_dgrad_swiglu_bwd(dy_perm, w2, h13, group_off, dh13, stream=None):
    cap, H = dy_perm.shape
    E, _, De = w2.shape
    _check(dh13, BF16, (cap, 2 * De), "dh13")
    _lib.call("dm_grouped_w2_dgrad_swiglu_bwd", _ptr(dy_perm), _ptr(w2), _ptr(h13), _ptr(group_off),
              _groups(group_off, E), E, cap, H, De, _ptr(dh13), _stream(stream))


def w13_dgrad(dh13, w13, group_off, dx_perm, stream=None):
    cap, two_de = dh13.shape
    E, _, H = w13.shape
    _check(dx_perm, BF16, (cap, H), "dx_perm")
    _lib.call("dm_grouped_w13_dgrad", _ptr(dh13), _ptr(w13), _ptr(group_off), _groups(group_off, E), E, cap,
              H, two_de // 2, _ptr(dx_perm), _stream(stream))


# -------------------------------------------- the same GEMMs over explicit group ranges
def batch_group_ranges(pad_off, cap, group_start, group_end, expert_major=True, stream=None):
    """Row ranges of n micro-batches stacked cap rows apart, from their [n, E+1] padded
    offsets: expert-major (g = e * n + i) or micro-batch-major (g = i * E + e)."""
    n, e1 = pad_off.shape
    _check(group_start, torch.int32, (n * (e1 - 1),), "group_start")
    _check(group_end, torch.int32, (n * (e1 - 1),), "group_end")
    _lib.call("dm_batch_group_ranges", _ptr(pad_off), n, e1 - 1, cap, int(bool(expert_major)), _ptr(group_start),
              _ptr(group_end), _stream(stream))


def _ranges(gs, ge, E, b_div):
    if gs.dtype != torch.int32 or ge.dtype != torch.int32 or gs.numel() != ge.numel() or gs.numel() < E:
        raise ValueError("group_start / group_end must be int32 [G] with G >= number of experts")
    if b_div < 1:
        raise ValueError("b_div must be >= 1")
    return gs.numel()


def w13_swiglu_fwd_ranges(x_perm, w13, gs, ge, b_div, h13, act, stream=None):
    cap, H = x_perm.shape
    E, two_de, _ = w13.shape
    De = two_de // 2
    _check(h13, BF16, (cap, 2 * De), "h13"); _check(act, BF16, (cap, De), "act")
    _lib.call("dm_grouped_w13_swiglu_fwd_ranges", _ptr(x_perm), _ptr(w13), _ptr(gs), _ptr(ge),
              _ranges(gs, ge, E, b_div), E, b_div, cap, H, De, _ptr(h13), _ptr(act), _stream(stream))


def w2_fwd_ranges(act, w2, gs, ge, b_div, y_perm, stream=None):
    cap, De = act.shape
    E, H, _ = w2.shape
    _check(y_perm, BF16, (cap, H), "y_perm")
    _lib.call("dm_grouped_w2_fwd_ranges", _ptr(act), _ptr(w2), _ptr(gs), _ptr(ge), _ranges(gs, ge, E, b_div), E,
              b_div, cap, H, De, _ptr(y_perm), _stream(stream))


def w2_dgrad_swiglu_bwd_ranges(dy_perm, w2, h13, gs, ge, b_div, dh13, stream=None):
    cap, H = dy_perm.shape
    E, _, De = w2.shape
    _check(dh13, BF16, (cap, 2 * De), "dh13")
    _lib.call("dm_grouped_w2_dgrad_swiglu_bwd_ranges", _ptr(dy_perm), _ptr(w2), _ptr(h13), _ptr(gs), _ptr(ge),
              _ranges(gs, ge, E, b_div), E, b_div, cap, H, De, _ptr(dh13), _stream(stream))


def w13_dgrad_ranges(dh13, w13, gs, ge, b_div, dx_perm, stream=None):
    cap, two_de = dh13.shape
    E, _, H = w13.shape
    _check(dx_perm, BF16, (cap, H), "dx_perm")
    _lib.call("dm_grouped_w13_dgrad_ranges", _ptr(dh13), _ptr(w13), _ptr(gs), _ptr(ge), _ranges(gs, ge, E, b_div),
              E, b_div, cap, H, two_de // 2, _ptr(dx_perm), _stream(stream))


def wgrad(a_tok, b_tok, seg_off, dW, beta=0.0, stream=None, seg_stride_rows=None):
    """dW[e] = sum over segments of a_tok[rows]^T b_tok[rows]. seg_off is [E+1] (one
    segment) or [nseg, E+1]; by default segment i starts at row i * rows/nseg (stacked
    equal blocks); seg_stride_rows=0 means seg_off holds absolute row offsets."""
    rows, M = a_tok.shape
    _, N = b_tok.shape
    so = seg_off if seg_off.dim() == 2 else seg_off.view(1, -1)
    nseg, E1 = so.shape
    E = E1 - 1
    if seg_stride_rows is None:
        if rows % nseg:
            raise ValueError("token buffers must stack nseg equal blocks")
        seg_stride_rows = rows // nseg
    if not so.is_contiguous():
        raise ValueError("seg_off must be contiguous")
    _check(dW, torch.float32, (E, M, N), "dW")
    _lib.call("dm_grouped_wgrad", _ptr(a_tok), M, _ptr(b_tok), N, _ptr(so), nseg, E, rows, seg_stride_rows,
              _ptr(dW), float(beta), _stream(stream))


# ------------------------------------------------------------------ combine
def combine_fwd(y_perm, row_map, w, y, stream=None, resid=None):
    """y = resid + sum_j w_j * y_perm[row_map[:, j]] (resid: optional residual input)."""
    T, k = row_map.shape
    H = y_perm.shape[1]
    _check(y, BF16, (T, H), "y")
    if resid is not None:
        _check(resid, BF16, (T, H), "resid")
    _lib.call("dm_combine_fwd", _ptr(y_perm), _ptr(row_map), _ptr(w), T, H, k, _ptr(resid), _ptr(y),
              _stream(stream))


def combine_bwd(dy, y_perm, row_map, w, counts, pad_off, dy_perm, dw, dlogit, stream=None, dl_perm=None):
    T, H = dy.shape
    k = row_map.shape[1]
    E = counts.shape[0]
    _lib.call("dm_combine_bwd", _ptr(dy), _ptr(y_perm), _ptr(row_map), _ptr(w), _ptr(counts), _ptr(pad_off),
              T, H, E, k, _ptr(dy_perm), _ptr(dw), _ptr(dlogit), _ptr(dl_perm), _stream(stream))


def router_wgrad_sorted(x, src_token, dl_perm, counts, pad_off, dwg, beta=0.0, stream=None, partial_ws=None):
    T, H = x.shape
    E = dwg.shape[0]
    _lib.call("dm_router_wgrad_sorted", _ptr(x), _ptr(src_token), _ptr(dl_perm), _ptr(counts), _ptr(pad_off),
              T, H, E, _ptr(partial_ws), _ptr(dwg), float(beta), _stream(stream))


def permute_bwd(dx_perm, row_map, idx, dlogit, wg, dx, stream=None, resid=None):
    """dx = resid + sum_j dx_perm[row_map[:, j]] + sum_j dlogit_j * W_g[idx_j] (resid optional)."""
    T, k = row_map.shape
    H = dx.shape[1]
    E = wg.shape[0]
    if resid is not None:
        _check(resid, BF16, (T, H), "resid")
    _lib.call("dm_permute_bwd", _ptr(dx_perm), _ptr(row_map), _ptr(idx), _ptr(dlogit), _ptr(wg), T, H, E, k,
              _ptr(resid), _ptr(dx), _stream(stream))


def router_wgrad(x, idx, dlogit, partial_ws, dwg, beta=0.0, stream=None):
    T, H = x.shape
    k = idx.shape[1]
    E = dwg.shape[0]
    need = _lib.router_wgrad_workspace_size(T, H, E)
    if partial_ws.numel() * partial_ws.element_size() < need:
        raise ValueError(f"router wgrad workspace too small ({need} bytes needed)")
    _lib.call("dm_router_wgrad", _ptr(x), _ptr(idx), _ptr(dlogit), T, H, E, k, _ptr(partial_ws), _ptr(dwg),
              float(beta), _stream(stream))


# ------------------------------------------------------------------ fp32 mode
# (bytes_per_element 4): fp32 activations, split-3 bf16 GEMM operands (dm_moe.h).
SPLIT_ACT, SPLIT_WK, SPLIT_WMN = 0, 1, 2


def split3(src, dst, layout, groups=1, stream=None):
    """fp32 [groups*rows, cols] -> split-3 bf16 (layout SPLIT_ACT / SPLIT_WK / SPLIT_WMN)."""
    rows_total, cols = src.reshape(-1, src.shape[-1]).shape
    _lib.call("dm_split3", _ptr(src), groups, rows_total // groups, cols, layout, _ptr(dst), _stream(stream))


def route_and_dispatch_f32(x, wg, k, workspace, idx, w, counts, pad_off, row_map, src_token, x3, stream=None):
    T, H = x.shape
    E = wg.shape[0]
    _check(x, F32, (T, H), "x")
    _lib.call("dm_route_and_dispatch_f32", _ptr(x), _ptr(wg), T, H, E, k, _ptr(workspace), _ptr(idx), _ptr(w),
              _ptr(counts), _ptr(pad_off), _ptr(row_map), _ptr(src_token), _ptr(x3), _stream(stream))


def gemm_f32(a3, b3, b_mn_major, group_off, c, num_weights, stream=None):
    """c[cap, N] fp32 = a3[cap, K3] . B3_(g % E); B3 K-major [E*N, K3] or MN-major [E*K3, N]."""
    cap, K3 = a3.shape
    N = c.shape[1]
    G = group_off.shape[-1] - 1
    _check(c, F32, (cap, N), "c")
    _lib.call("dm_grouped_gemm_f32", _ptr(a3), _ptr(b3), int(b_mn_major), _ptr(group_off), G, num_weights, cap,
              N, K3, _ptr(c), _stream(stream))


def combine_fwd_f32(y_perm, row_map, w, y, stream=None, resid=None):
    T, k = row_map.shape
    H = y_perm.shape[1]
    _check(y, F32, (T, H), "y")
    _lib.call("dm_combine_fwd_f32", _ptr(y_perm), _ptr(row_map), _ptr(w), T, H, k, _ptr(resid), _ptr(y),
              _stream(stream))


def combine_bwd_f32(dy, y_perm, row_map, w, counts, pad_off, dy3, dw, dlogit, dl_perm, stream=None):
    T, H = dy.shape
    k = row_map.shape[1]
    E = counts.shape[0]
    _lib.call("dm_combine_bwd_f32", _ptr(dy), _ptr(y_perm), _ptr(row_map), _ptr(w), _ptr(counts), _ptr(pad_off),
              T, H, E, k, _ptr(dy3), _ptr(dw), _ptr(dlogit), _ptr(dl_perm), _stream(stream))


def permute_bwd_f32(dx_perm, row_map, idx, dlogit, wg, dx, stream=None, resid=None):
    T, k = row_map.shape
    H = dx.shape[1]
    E = wg.shape[0]
    _lib.call("dm_permute_bwd_f32", _ptr(dx_perm), _ptr(row_map), _ptr(idx), _ptr(dlogit), _ptr(wg), T, H, E, k,
              _ptr(resid), _ptr(dx), _stream(stream))


def router_wgrad_sorted_f32(x, src_token, dl_perm, counts, pad_off, dwg, beta=0.0, stream=None, partial_ws=None):
    T, H = x.shape
    E = dwg.shape[0]
    _lib.call("dm_router_wgrad_sorted_f32", _ptr(x), _ptr(src_token), _ptr(dl_perm), _ptr(counts), _ptr(pad_off),
              T, H, E, _ptr(partial_ws), _ptr(dwg), float(beta), _stream(stream))


def swiglu_fwd_split(h13, act3, stream=None):
    rows, two_de = h13.shape
    _lib.call("dm_swiglu_fwd_split", _ptr(h13), rows, two_de // 2, _ptr(act3), _stream(stream))


def swiglu_bwd_split(d_act, h13, dh13_3, stream=None):
    rows, De = d_act.shape
    _lib.call("dm_swiglu_bwd_split", _ptr(d_act), _ptr(h13), rows, De, _ptr(dh13_3), _stream(stream))


def wgrad_split3(a3, M, b3, N, seg_off, dW, beta=0.0, stream=None, seg_stride_rows=None):
    """dW[g] (+)= A^T B over each group's rows from split-3 operands a3 [R, 3M], b3 [R, 3N]:
    three strided ragged-K GEMMs a_hi.b_hi + a_hi.b_lo + a_lo.b_hi (fp32 reduce-add)."""
    total_rows = a3.shape[0]
    so = seg_off.reshape(-1, seg_off.shape[-1])
    nseg, E = so.shape[0], so.shape[1] - 1
    stride = total_rows // nseg if seg_stride_rows is None else seg_stride_rows
    if not (a3.is_contiguous() and b3.is_contiguous()):
        raise ValueError("split-3 operands must be contiguous")
    base_a, base_b = a3.data_ptr(), b3.data_ptr()
    hi_a, lo_a = base_a, base_a + 2 * M * a3.element_size()
    hi_b, lo_b = base_b, base_b + 2 * N * b3.element_size()
    for i, (pa, pb) in enumerate(((hi_a, hi_b), (hi_a, lo_b), (lo_a, hi_b))):
        _lib.call("dm_grouped_wgrad_strided", pa, M, 3 * M, pb, N, 3 * N, _ptr(so), nseg, E, total_rows, stride,
                  _ptr(dW), float(beta) if i == 0 else 1.0, _stream(stream))


# ---------------------------------------------------------------- attention
def attention_fwd(qkv, seq_len, nh, nkv, out, lse, stream=None):
    """Causal GQA flash-attention forward (head_dim 128) on the packed projection
    qkv [T, (nh + 2 nkv) * 128]: out [T, nh * 128] bf16, lse [T / seq_len, nh, seq_len]
    fp32 (natural log, logits scaled by 1/sqrt(128))."""
    T = qkv.shape[0]
    _check(qkv, BF16, (T, (nh + 2 * nkv) * 128), "qkv")
    _check(out, BF16, (T, nh * 128), "out")
    _check(lse, F32, (T // seq_len, nh, seq_len), "lse")
    _lib.call("dm_attention_fwd", _ptr(qkv), T, seq_len, nh, nkv, 128, _ptr(out), _ptr(lse), _stream(stream))


def attention_bwd(qkv, out, dout, lse, seq_len, nh, nkv, dqkv, dl_ws=None, stream=None):
    """Backward of attention_fwd: dqkv [T, (nh + 2 nkv) * 128] bf16 (dQ | dK | dV) from the
    packed projection, the forward's out / lse and dout [T, nh * 128]."""
    T = qkv.shape[0]
    _check(qkv, BF16, (T, (nh + 2 * nkv) * 128), "qkv")
    _check(out, BF16, (T, nh * 128), "out")
    _check(dout, BF16, (T, nh * 128), "dout")
    _check(lse, F32, (T // seq_len, nh, seq_len), "lse")
    _check(dqkv, BF16, (T, (nh + 2 * nkv) * 128), "dqkv")
    if dl_ws is None:
        dl_ws = torch.empty(2, T // seq_len, nh, seq_len, dtype=F32, device=qkv.device)
    _check(dl_ws, F32, (2, T // seq_len, nh, seq_len), "dl_ws")
    _lib.call("dm_attention_bwd", _ptr(qkv), _ptr(out), _ptr(dout), _ptr(lse), T, seq_len, nh, nkv, 128,
              _ptr(dl_ws), _ptr(dqkv), _stream(stream))
