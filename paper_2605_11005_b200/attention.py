"""A-side causal self-attention of a transformer layer.

The reference models attention only as a cost, C_a = b·(s·H²·(2+2/g) + 4·s²·H)
(`pkg/src/afpipe/costs.py:84-87`), placed on the attention (A) GPU groups of the
AF-Pipe schedule. This module gives the A ranks that work for real so the
long-context (configs[3]) and A:F allocation (configs[4]) sweeps measure the
overlap the paper is about. It is NOT part of the MoE hot path this repo
rebuilds: it is the stopgap SURVEY.md §8f names — cuBLAS projections and torch's
scaled_dot_product_attention restricted to the cuDNN / flash backends (cuDNN's
Blackwell attention kernels, measured 1.3 PFLOP/s fwd+bwd at s = 16K on B200,
scripts/probe_sdpa.py) — and is labelled as library code wherever it is timed.

Block: h = x + W_o · attn(x W_q, x W_k, x W_v), causal, GQA with g query heads per
KV head (ModelConfig.gqa_group), head_dim 128, no normalisation / RoPE (shape and
FLOPs are what the schedule needs). Gradients come from torch autograd on the
per-micro-batch graph saved by `forward`; parameter gradients accumulate in fp32
`.grad`-style buffers (`dw_qkv`, `dw_o`).

On CUDA with seq_len a multiple of 128 (256 for an odd GQA group) the attention forward is this repo's own sm_100a
kernel (`dm_attention_fwd`: tcgen05/TMEM/TMA flash attention, csrc/attention_fwd.cu); its
(O, LSE) feed cuDNN's SDPA backward (the LSE matches cuDNN's to 5e-5), so only the
backward and the projections remain library code.
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


class _OwnCausalAttention(torch.autograd.Function):
    """o [T, nh·D] = causal GQA attention of the packed projection qkv [T, (nh + 2 nkv)·D]:
    forward on dm_attention_fwd, backward on cuDNN's SDPA backward with our (O, LSE)."""

    @staticmethod
    def forward(ctx, qkv, seq_len, nh, nkv):
        from . import kernels as K

        T = qkv.shape[0]
        out = torch.empty(T, nh * HEAD_DIM, dtype=BF16, device=qkv.device)
        lse = torch.empty(T // seq_len, nh, seq_len, dtype=F32, device=qkv.device)
        K.attention_fwd(qkv, seq_len, nh, nkv, out, lse)
        ctx.save_for_backward(qkv, out, lse)
        ctx.shape = (seq_len, nh, nkv)
        return out

    @staticmethod
    def backward(ctx, grad_out):
        qkv, out, lse = ctx.saved_tensors
        s, nh, nkv = ctx.shape
        T = qkv.shape[0]
        b = T // s
        x = qkv.view(b, s, nh + 2 * nkv, HEAD_DIM).transpose(1, 2)        # [b, heads, s, D] views
        q, k, v = x[:, :nh], x[:, nh:nh + nkv], x[:, nh + nkv:]            # GQA handled by cuDNN
        o = out.view(b, s, nh, HEAD_DIM).transpose(1, 2)
        do = grad_out.contiguous().view(b, s, nh, HEAD_DIM).transpose(1, 2)
        zero = torch.zeros((), dtype=torch.int64, device=qkv.device)   # philox seed / offset (no dropout)
        dq, dk, dv = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
            do, q, k, v, o, lse.unsqueeze(-1), zero, zero, None, None, None, s, s, 0.0, True)
        dqkv = torch.empty_like(qkv)
        d = dqkv.view(b, s, nh + 2 * nkv, HEAD_DIM)
        d[:, :, :nh].copy_(dq.transpose(1, 2))
        d[:, :, nh:nh + nkv].copy_(dk.transpose(1, 2))
        d[:, :, nh + nkv:].copy_(dv.transpose(1, 2))
        return dqkv, None, None, None


def own_attention_supported(x: torch.Tensor, seq_len: int, head_dim: int = HEAD_DIM, gqa_group: int = 1) -> bool:
    """dm_attention_fwd's shape contract: head_dim 128, whole sequences, seq_len a multiple of
    128 (pairs of query heads share a tile pair) or 256 (odd GQA group: adjacent row tiles)."""
    row_tile = 128 if gqa_group % 2 == 0 else 256
    return x.is_cuda and head_dim == HEAD_DIM and seq_len % row_tile == 0 and x.shape[0] % seq_len == 0


class AttentionBlock:
    def __init__(self, hidden: int, gqa_group: int = 1, device="cuda", seed: int = 0,
                 head_dim: int = HEAD_DIM, own_kernel: bool = True):
        if hidden % head_dim:
            raise ValueError(f"hidden {hidden} not a multiple of head_dim {head_dim}")
        self.H, self.d = hidden, head_dim
        self.own_kernel = own_kernel   # dm_attention_fwd for the forward where supported
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
        self.last_path = None   # "own" / "library": which attention path the last forward took

    def flops(self, seq_len: int, micro_batch: int) -> tuple[int, int]:
        return attention_flops(self.H, self.nh // self.nkv, seq_len, micro_batch, self.d)

    def _attend(self, x: torch.Tensor, seq_len: int) -> torch.Tensor:
        T, H = x.shape
        b = T // seq_len
        qkv = x @ self.w_qkv.t()
        if self.own_kernel and own_attention_supported(x, seq_len, self.d, self.nh // self.nkv):
            self.last_path = "own"
            o = _OwnCausalAttention.apply(qkv.contiguous(), seq_len, self.nh, self.nkv)
            return o @ self.w_o.t()
        self.last_path = "library"
        q, k, v = qkv.split([self.nh * self.d, self.nkv * self.d, self.nkv * self.d], dim=1)
        q = q.view(b, seq_len, self.nh, self.d).transpose(1, 2)
        k = k.view(b, seq_len, self.nkv, self.d).transpose(1, 2)
        v = v.view(b, seq_len, self.nkv, self.d).transpose(1, 2)
        with sdpa_kernel(_BACKENDS if x.is_cuda else [SDPBackend.MATH]):
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=self.nkv != self.nh)
        o = o.transpose(1, 2).reshape(T, H)
        return o @ self.w_o.t()

    def forward(self, slot, x: torch.Tensor, out: torch.Tensor, seq_len: int) -> None:
        """out = x + attn(x) (bf16 [T, H]); keeps the autograd graph under `slot`."""
        with torch.enable_grad():
            xi = x.detach().requires_grad_(True)
            h = xi + self._attend(xi, seq_len)
        out.copy_(h.detach())
        self._saved[slot] = (xi, h)

    def backward(self, slot, grad_h: torch.Tensor, dx_out: torch.Tensor, accumulate: bool) -> None:
        """dx_out = dL/dx given dL/dh; parameter grads (+)= into dw_qkv / dw_o (fp32)."""
        xi, h = self._saved.pop(slot)
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
