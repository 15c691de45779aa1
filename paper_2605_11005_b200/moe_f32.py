"""fp32 mode of the MoE hot path (experiment `bytes_per_element: 4`, reference
pkg/src/afpipe/config.py ModelConfig; 1e-4 parity in fp32 mode).

Activations, gradients and master weights are fp32. The expert GEMMs still run on
the tcgen05 tensor cores: every fp32 operand is split into two bf16 terms and the
three significant cross products are summed inside ONE bf16 GEMM over a 3x longer
reduction ("split-3", include/dm_moe.h): activations are stored as rows
[hi | hi | lo], weights as [hi | lo | hi] (K-major) or stacked [hi; lo; hi] per
expert (MN-major), so the fp32 TMEM accumulator receives a_hi.b_hi + a_hi.b_lo +
a_lo.b_hi (error ~2^-16 relative, vs 2^-8 for plain bf16). The SwiGLU epilogues
become separate fp32 elementwise kernels that emit the next GEMM's split-3 operand.

Same stage split, device-side group offsets and deferred wgrad as moe.py; the
router runs on fp32 x in the same canonical order (bit-exact routing).
"""

from __future__ import annotations

import torch

from . import _lib
from . import kernels as K
from .moe import MoEShape

BF16, F32, I32 = torch.bfloat16, torch.float32, torch.int32


class ExpertParamsF32:
    """fp32 master weights W13 [E, 2D_e, H] (DM_GLU_BLOCK-row gate/up blocks) and W2 [E, H, D_e],
    their fp32 gradients, and the split-3 bf16 copies the GEMMs read (refreshed by
    `prepare()` after every weight update)."""

    def __init__(self, w13: torch.Tensor, w2: torch.Tensor):
        self.w13 = w13.to(F32).contiguous()
        self.w2 = w2.to(F32).contiguous()
        E, two_de, H = self.w13.shape
        De = two_de // 2
        dev = self.w13.device
        self.dw13 = torch.zeros_like(self.w13)
        self.dw2 = torch.zeros_like(self.w2)
        self.w13_k = torch.empty(E * two_de, 3 * H, dtype=BF16, device=dev)     # fwd B (K = H)
        self.w13_mn = torch.empty(E * 3 * two_de, H, dtype=BF16, device=dev)    # dgrad B (K = 2D_e)
        self.w2_k = torch.empty(E * H, 3 * De, dtype=BF16, device=dev)          # fwd B (K = D_e)
        self.w2_mn = torch.empty(E * 3 * H, De, dtype=BF16, device=dev)         # dgrad B (K = H)
        self.prepare()

    @property
    def num_experts(self) -> int:
        return self.w13.shape[0]

    def prepare(self, stream=None) -> None:
        E = self.num_experts
        K.split3(self.w13, self.w13_k, K.SPLIT_WK, stream=stream)
        K.split3(self.w13, self.w13_mn, K.SPLIT_WMN, groups=E, stream=stream)
        K.split3(self.w2, self.w2_k, K.SPLIT_WK, stream=stream)
        K.split3(self.w2, self.w2_mn, K.SPLIT_WMN, groups=E, stream=stream)


class SlabF32:
    """F-side tensors of `n` micro-batches stacked in [n*cap, .] slabs (moe.ActivationSlab)."""

    def __init__(self, shape: MoEShape, n: int, device):
        s, dev = shape, torch.device(device)
        self.n, self.cap = n, s.cap
        R = n * self.cap
        e = lambda *sh, dt=BF16: torch.empty(*sh, dtype=dt, device=dev)  # noqa: E731
        self.pad_off = torch.zeros(n, s.E + 1, dtype=I32, device=dev)
        self.x3 = e(R, 3 * s.H)
        self.h13 = e(R, 2 * s.De, dt=F32)
        self.act3 = e(R, 3 * s.De)
        self.y_perm = e(R, s.H, dt=F32)
        self.dy3 = e(R, 3 * s.H)
        self.d_act = e(R, s.De, dt=F32)
        self.dh13_3 = e(R, 6 * s.De)
        self.dx_perm = e(R, s.H, dt=F32)

    def rows(self, i: int) -> slice:
        return slice(i * self.cap, (i + 1) * self.cap)


class BuffersF32:
    """One micro-batch: fp32 token tensors (x, y, dy, dx) + views into the slab."""

    def __init__(self, shape: MoEShape, device, slab: SlabF32, index: int, residual: bool = False):
        s, dev = shape, torch.device(device)
        z = lambda *sh, dt=F32: torch.empty(*sh, dtype=dt, device=dev)  # noqa: E731
        self.shape, self.residual, self.cap = s, residual, slab.cap
        self.x, self.y, self.dy, self.dx = z(s.T, s.H), z(s.T, s.H), z(s.T, s.H), z(s.T, s.H)
        self.idx, self.row_map = z(s.T, s.k, dt=I32), z(s.T, s.k, dt=I32)
        self.w, self.dw, self.dlogit = z(s.T, s.k), z(s.T, s.k), z(s.T, s.k)
        self.counts = z(s.E, dt=I32)
        self.src = z(slab.cap, dt=I32)
        self.dl_perm = z(slab.cap)
        self.route_ws = torch.zeros(_lib.route_workspace_size(s.T, s.H, s.E, s.k), dtype=torch.uint8, device=dev)
        self.wgrad_ws = torch.zeros(_lib.router_wgrad_workspace_size(s.T, s.H, s.E) // 4, dtype=F32, device=dev)
        self.pad_off = slab.pad_off[index]
        r = slab.rows(index)
        for name in ("x3", "h13", "act3", "y_perm", "dy3", "d_act", "dh13_3", "dx_perm"):
            setattr(self, name, getattr(slab, name)[r])


class MoELayerF32:
    """Fused single-device MoE layer in fp32 mode (moe.MoELayer's fp32 counterpart)."""

    def __init__(self, shape: MoEShape, wg: torch.Tensor, w13: torch.Tensor, w2: torch.Tensor, device="cuda",
                 num_buffers: int = 1, residual: bool = False):
        shape.validate()
        _lib.load()
        self.shape, self.device = shape, torch.device(device)
        self.wg = wg.to(self.device, F32).contiguous()
        self.dwg = torch.zeros_like(self.wg)
        self.experts = ExpertParamsF32(w13.to(self.device), w2.to(self.device))
        self.slab = SlabF32(shape, num_buffers, self.device)
        self.buffers = [BuffersF32(shape, self.device, self.slab, i, residual) for i in range(num_buffers)]

    @classmethod
    def random(cls, shape: MoEShape, device="cuda", seed: int = 0, num_buffers: int = 1,
               residual: bool = False) -> "MoELayerF32":
        g = torch.Generator(device="cpu").manual_seed(seed)
        wg = torch.randn(shape.E, shape.H, generator=g) * 0.02
        w13 = torch.randn(shape.E, 2 * shape.De, shape.H, generator=g) * 0.02
        w2 = torch.randn(shape.E, shape.H, shape.De, generator=g) * 0.02
        return cls(shape, wg, w13, w2, device, num_buffers, residual)

    dtype = F32

    # ---- stages (same split as moe.py; bench / profiling call these)
    def stage_dispatch(self, b: BuffersF32, stream=None) -> None:
        s = self.shape
        K.route_and_dispatch_f32(b.x, self.wg, s.k, b.route_ws, b.idx, b.w, b.counts, b.pad_off, b.row_map, b.src,
                                 b.x3, stream)

    def stage_f_forward(self, b: BuffersF32, stream=None) -> None:
        ex, E = self.experts, self.shape.E
        K.gemm_f32(b.x3, ex.w13_k, False, b.pad_off, b.h13, E, stream)
        K.swiglu_fwd_split(b.h13, b.act3, stream)
        K.gemm_f32(b.act3, ex.w2_k, False, b.pad_off, b.y_perm, E, stream)

    def stage_combine(self, b: BuffersF32, stream=None) -> None:
        K.combine_fwd_f32(b.y_perm, b.row_map, b.w, b.y, stream, resid=b.x if b.residual else None)

    def stage_combine_bwd(self, b: BuffersF32, stream=None) -> None:
        K.combine_bwd_f32(b.dy, b.y_perm, b.row_map, b.w, b.counts, b.pad_off, b.dy3, b.dw, b.dlogit, b.dl_perm,
                          stream)

    def stage_f_backward(self, b: BuffersF32, accumulate: bool = False, stream=None, defer_wgrad: bool = True):
        s, ex = self.shape, self.experts
        K.gemm_f32(b.dy3, ex.w2_mn, True, b.pad_off, b.d_act, s.E, stream)
        K.swiglu_bwd_split(b.d_act, b.h13, b.dh13_3, stream)
        K.gemm_f32(b.dh13_3, ex.w13_mn, True, b.pad_off, b.dx_perm, s.E, stream)
        if not defer_wgrad:
            beta = 1.0 if accumulate else 0.0
            K.wgrad_split3(b.dy3, s.H, b.act3, s.De, b.pad_off, ex.dw2, beta, stream)
            K.wgrad_split3(b.dh13_3, 2 * s.De, b.x3, s.H, b.pad_off, ex.dw13, beta, stream)

    def stage_permute_bwd(self, b: BuffersF32, stream=None) -> None:
        K.permute_bwd_f32(b.dx_perm, b.row_map, b.idx, b.dlogit, self.wg, b.dx, stream,
                          resid=b.dy if b.residual else None)

    def stage_router_wgrad(self, b: BuffersF32, accumulate: bool, stream=None) -> None:
        K.router_wgrad_sorted_f32(b.x, b.src, b.dl_perm, b.counts, b.pad_off, self.dwg,
                                  1.0 if accumulate else 0.0, stream, partial_ws=b.wgrad_ws)

    def forward(self, b: BuffersF32, stream=None) -> None:
        self.stage_dispatch(b, stream)
        self.stage_f_forward(b, stream)
        self.stage_combine(b, stream)

    def backward(self, b: BuffersF32, accumulate: bool, stream=None, defer_wgrad: bool = False) -> None:
        self.stage_combine_bwd(b, stream)
        self.stage_f_backward(b, accumulate, stream, defer_wgrad)
        self.stage_permute_bwd(b, stream)
        self.stage_router_wgrad(b, accumulate, stream)

    def forward_backward(self, b: BuffersF32, accumulate: bool = False, stream=None,
                         defer_wgrad: bool = False) -> None:
        self.forward(b, stream)
        self.backward(b, accumulate, stream, defer_wgrad)

    def wgrad(self, n: int | None = None, accumulate: bool = False, stream=None) -> None:
        """Deferred weight gradients over micro-batches 0..n-1 of the slab."""
        s, sl, ex = self.shape, self.slab, self.experts
        n = len(self.buffers) if n is None else n
        rows = slice(0, n * sl.cap)
        so = sl.pad_off[:n]
        beta = 1.0 if accumulate else 0.0
        K.wgrad_split3(sl.dy3[rows], s.H, sl.act3[rows], s.De, so, ex.dw2, beta, stream)
        K.wgrad_split3(sl.dh13_3[rows], 2 * s.De, sl.x3[rows], s.H, so, ex.dw13, beta, stream)

    def iteration(self, n: int | None = None, accumulate: bool = False, stream=None) -> None:
        n = len(self.buffers) if n is None else n
        for i in range(n):
            self.forward_backward(self.buffers[i], accumulate or i > 0, stream, defer_wgrad=True)
        self.wgrad(n, accumulate, stream)

    def zero_grad(self) -> None:
        self.dwg.zero_()
        self.experts.dw13.zero_()
        self.experts.dw2.zero_()


class MoEFunctionF32(torch.autograd.Function):
    """autograd entry point in fp32 mode: y = MoE(x; W_g, W13, W2), all fp32."""

    @staticmethod
    def forward(ctx, x, wg, w13, w2, k: int):
        T, H = x.shape
        E, two_de, _ = w13.shape
        shape = MoEShape(T=T, H=H, E=E, k=k, De=two_de // 2)
        layer = MoELayerF32(shape, wg.detach(), w13.detach(), w2.detach(), x.device)
        buf = layer.buffers[0]
        buf.x.copy_(x)
        layer.forward(buf)
        ctx.layer = layer
        return buf.y.clone()

    @staticmethod
    def backward(ctx, dy):
        layer = ctx.layer
        buf = layer.buffers[0]
        buf.dy.copy_(dy.float())
        layer.backward(buf, accumulate=False)
        ex = layer.experts
        return buf.dx.clone(), layer.dwg, ex.dw13, ex.dw2, None
