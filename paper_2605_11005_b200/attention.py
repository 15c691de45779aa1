"""A-side causal self-attention of a transformer layer.

The reference models attention only as a cost, C_a = b·(s·H²·(2+2/g) + 4·s²·H)
(`pkg/src/afpipe/costs.py:84-87`), placed on the attention (A) GPU groups of the
AF-Pipe schedule. This module gives the A ranks that work for real so the
long-context (configs[3]) and A:F allocation (configs[4]) sweeps measure the
overlap the paper is about. It is not part of the MoE hot path itself.

Block: h = x + W_o · attn(x W_q, x W_k, x W_v), causal, GQA with g query heads per
KV head (ModelConfig.gqa_group), head_dim 128, no normalisation / RoPE (shape and
FLOPs are what the schedule needs). Parameter gradients accumulate in fp32
`.grad`-style buffers (`dw_qkv`, `dw_o`).

Own path (CUDA, seq_len a multiple of 128 — 256 for an odd GQA group —, H % 256 == 0 and an
even head count, `own_path_supported`): every FLOP runs in this repo's sm_100a kernels, no
autograd graph —
  forward   qkv = x·W_qkvᵀ and y = o·W_oᵀ on the grouped tcgen05 GEMM (`dm_grouped_w2_fwd`, one
            group), o / LSE on `dm_attention_fwd`, h = x + y;
  backward  dO = dh·W_o and dx_attn = dqkv·W_qkv on `dm_grouped_w13_dgrad`, dQ/dK/dV on
            `dm_attention_bwd` (fed the forward's O / LSE), dW_o += dhᵀ·o and
            dW_qkv += dqkvᵀ·x on the ragged-K wgrad (`dm_grouped_wgrad`, fp32 TMA reduce-add).
Other shapes (and CPU, for the gloo tests) run the library block: torch projections and
scaled_dot_product_attention (cuDNN / flash) under autograd, labelled "library".
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

BF16, F32 = torch.bfloat16, torch.float32
HEAD_DIM = 128
_BACKENDS = [SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION]


def attention_flops(hidden: int, gqa_group: int, seq_len: int, micro_batch: int,
                    head_dim: int = HEAD_DIM) -> tuple[int, int]:
    """(fwd, bwd) FLOPs of one micro-batch: projections 2·T·H·(H + 2H/g) + 2·T·H²,
    causal attention 2·s²·H per sequence (QKᵀ and PV, half masked); bwd = 2x / 2.5x.
    (The reference's C_a, costs.py:84-87, counts the same terms as multiply-adds.)"""
    T, H = seq_len * micro_batch, hidden
    nh = hidden // head_dim
    nkv = nh // gqa_group
    proj = 2 * T * H * (nh + 2 * nkv) * head_dim + 2 * T * H * H
    attn = 2 * seq_len * seq_len * H * micro_batch
    return proj + attn, 2 * proj + int(2.5 * attn)


def own_attention_supported(x: torch.Tensor, seq_len: int, head_dim: int = HEAD_DIM, gqa_group: int = 1) -> bool:
    """dm_attention_fwd / _bwd's shape contract: head_dim 128, whole sequences, seq_len a multiple
    of 128 (pairs of query heads share a tile pair) or 256 (odd GQA group: adjacent row tiles)."""
    row_tile = 128 if gqa_group % 2 == 0 else 256
    return x.is_cuda and head_dim == HEAD_DIM and seq_len % row_tile == 0 and x.shape[0] % seq_len == 0


def own_path_supported(x: torch.Tensor, seq_len: int, nh: int, nkv: int, head_dim: int = HEAD_DIM) -> bool:
    """The whole block on own kernels: the attention contract plus the grouped GEMM's
    (output and reduction widths multiples of 128: the dgrads contract over (nh + 2 nkv)·128
    and H columns viewed as 2·D_e, so H % 256 == 0 and nh even)."""
    H = x.shape[1]
    return (own_attention_supported(x, seq_len, head_dim, nh // nkv) and H % 256 == 0 and nh % 2 == 0
            and x.shape[0] % 128 == 0)


class AttentionBlock:
    def __init__(self, hidden: int, gqa_group: int = 1, device="cuda", seed: int = 0,
                 head_dim: int = HEAD_DIM, own_kernel: bool = True):
        if hidden % head_dim:
            raise ValueError(f"hidden {hidden} not a multiple of head_dim {head_dim}")
        self.H, self.d = hidden, head_dim
        self.own_kernel = own_kernel   # the own-kernel block where supported
        self.nh = hidden // head_dim
        if self.nh % gqa_group:
            raise ValueError(f"{self.nh} heads not divisible by gqa_group {gqa_group}")
        self.nkv = self.nh // gqa_group
        dev = torch.device(device)
        g = torch.Generator(device=dev).manual_seed(seed)
        rows = (self.nh + 2 * self.nkv) * head_dim
        self.w_qkv = torch.empty(rows, hidden, dtype=BF16, device=dev).normal_(0, 0.02, generator=g)
        self.w_o = torch.empty(hidden, hidden, dtype=BF16, device=dev).normal_(0, 0.02, generator=g)
        self.w_qkv.requires_grad_(True)
        self.w_o.requires_grad_(True)
        self.dw_qkv = torch.zeros(rows, hidden, dtype=F32, device=dev)
        self.dw_o = torch.zeros(hidden, hidden, dtype=F32, device=dev)
        self._saved: dict = {}
        self._goff: dict = {}
        self.last_path = None   # "own" / "library": which path the last forward took

    def flops(self, seq_len: int, micro_batch: int) -> tuple[int, int]:
        return attention_flops(self.H, self.nh // self.nkv, seq_len, micro_batch, self.d)

    def _group_off(self, T: int, device) -> torch.Tensor:
        key = (T, str(device))
        if key not in self._goff:
            self._goff[key] = torch.tensor([0, T], dtype=torch.int32, device=device)
        return self._goff[key]

    # ---------------------------------------------------------------- own kernels
    def _forward_own(self, slot, x: torch.Tensor, out: torch.Tensor, seq_len: int) -> None:
        from . import kernels as K

        T, H = x.shape
        go = self._group_off(T, x.device)
        wq = self.w_qkv.detach().view(1, -1, H)
        wo = self.w_o.detach().view(1, H, H)
        qkv = torch.empty(T, wq.shape[1], dtype=BF16, device=x.device)
        K.w2_fwd(x, wq, go, qkv)                                   # qkv = x W_qkv^T
        o = torch.empty(T, self.nh * self.d, dtype=BF16, device=x.device)
        lse = torch.empty(T // seq_len, self.nh, seq_len, dtype=F32, device=x.device)
        K.attention_fwd(qkv, seq_len, self.nh, self.nkv, o, lse)
        y = torch.empty(T, H, dtype=BF16, device=x.device)
        K.w2_fwd(o, wo, go, y)                                     # y = o W_o^T
        torch.add(x, y, out=out)
        self._saved[slot] = ("own", x, qkv, o, lse, seq_len)

    def _backward_own(self, saved, grad_h: torch.Tensor, dx_out: torch.Tensor, accumulate: bool) -> None:
        from . import kernels as K

        _, x, qkv, o, lse, seq_len = saved
        T, H = x.shape
        go = self._group_off(T, x.device)
        seg = go.view(1, 2)
        dh = grad_h.contiguous()
        w13_o = self.w_o.detach().view(1, H, H)                    # dgrad: dO = dh W_o
        do = torch.empty(T, H, dtype=BF16, device=x.device)
        K.w13_dgrad(dh, w13_o, go, do)
        K.wgrad(dh, o, seg, self.dw_o.view(1, H, H), beta=1.0 if accumulate else 0.0)   # dW_o (+)= dh^T o
        dqkv = torch.empty_like(qkv)
        K.attention_bwd(qkv, o, do, lse, seq_len, self.nh, self.nkv, dqkv)
        R = qkv.shape[1]
        K.wgrad(dqkv, x, seg, self.dw_qkv.view(1, R, H), beta=1.0 if accumulate else 0.0)
        dxa = torch.empty(T, H, dtype=BF16, device=x.device)
        K.w13_dgrad(dqkv, self.w_qkv.detach().view(1, R, H), go, dxa)   # dx_attn = dqkv W_qkv
        torch.add(dh, dxa, out=dx_out)

    # ----------------------------------------------------------- library block
    def _attend(self, x: torch.Tensor, seq_len: int) -> torch.Tensor:
        T, H = x.shape
        b = T // seq_len
        qkv = x @ self.w_qkv.t()
        q, k, v = qkv.split([self.nh * self.d, self.nkv * self.d, self.nkv * self.d], dim=1)
        q = q.view(b, seq_len, self.nh, self.d).transpose(1, 2)
        k = k.view(b, seq_len, self.nkv, self.d).transpose(1, 2)
        v = v.view(b, seq_len, self.nkv, self.d).transpose(1, 2)
        with sdpa_kernel(_BACKENDS if x.is_cuda else [SDPBackend.MATH]):
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=self.nkv != self.nh)
        o = o.transpose(1, 2).reshape(T, H)
        return o @ self.w_o.t()

    def forward(self, slot, x: torch.Tensor, out: torch.Tensor, seq_len: int) -> None:
        """out = x + attn(x) (bf16 [T, H]); keeps what the backward needs under `slot`."""
        if self.own_kernel and own_path_supported(x, seq_len, self.nh, self.nkv, self.d):
            self.last_path = "own"
            self._forward_own(slot, x.detach(), out, seq_len)
            return
        self.last_path = "library"
        with torch.enable_grad():
            xi = x.detach().requires_grad_(True)
            h = xi + self._attend(xi, seq_len)
        out.copy_(h.detach())
        self._saved[slot] = ("library", xi, h)

    def backward(self, slot, grad_h: torch.Tensor, dx_out: torch.Tensor, accumulate: bool) -> None:
        """dx_out = dL/dx given dL/dh; parameter grads (+)= into dw_qkv / dw_o (fp32)."""
        saved = self._saved.pop(slot)
        if saved[0] == "own":
            self._backward_own(saved, grad_h, dx_out, accumulate)
            return
        _, xi, h = saved
        gx, gq, go = torch.autograd.grad(h, (xi, self.w_qkv, self.w_o), grad_outputs=grad_h)
        dx_out.copy_(gx)
        if accumulate:
            self.dw_qkv.add_(gq)
            self.dw_o.add_(go)
        else:
            self.dw_qkv.copy_(gq)
            self.dw_o.copy_(go)

    def grads(self) -> list[torch.Tensor]:
        return [self.dw_qkv, self.dw_o]
