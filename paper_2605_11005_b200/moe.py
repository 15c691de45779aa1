"""The MoE layer hot path on B200: dispatch -> SwiGLU experts -> combine, fwd + bwd.

Stage split follows the AF-Pipe task boundaries of the reference DAG
(/root/reference/pkg/src/afpipe/taskgraph.py:307-356):

    A side (attention ranks)           F side (FFN ranks)
    a_dispatch      (A FwdCompute tail) f_forward   (F FwdCompute, :333-334)
    a_combine       (A FwdCompute head of the next visit, fed by the N2M recv :335-339)
    a_combine_bwd   (A BwdCompute)      f_backward  (F BwdCompute, :346-347)
    a_dispatch_bwd  (A BwdCompute, after the recv of :348-349)

Every stage is a fixed sequence of dm_* kernel launches on one CUDA stream
with no host synchronisation: per-expert sizes stay on the device (pad_off),
buffers are pre-sized to dm_capacity_rows(). There is no CPU fallback — a
missing libdm_moe.so raises at construction.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from . import kernels as K

BF16 = torch.bfloat16
F32 = torch.float32
I32 = torch.int32


@dataclass(frozen=True)
class MoEShape:
    """T tokens per micro-batch, hidden H, E experts, top-k, expert hidden D_e."""

    T: int
    H: int
    E: int
    k: int
    De: int

    @property
    def R(self) -> int:
        return self.T * self.k

    @property
    def cap(self) -> int:
        return _lib.capacity_rows(self.T, self.E, self.k)

    def validate(self) -> None:
        # 128-column tiles: the expert GEMMs run 256-wide tiles and clip a 128-wide tail
        # (deepseek_moe.yaml: moe_hidden 1408 = 11 x 128)
        if self.H % 128 or self.De % 128 or self.H < 128 or self.De < 128:
            raise ValueError(f"hidden ({self.H}) and moe_hidden ({self.De}) must be multiples of 128")
        if not (1 <= self.k <= min(self.E, _lib.DM_MAX_TOPK)):
            raise ValueError(f"topk {self.k} out of range for E={self.E}")
        if self.E > _lib.DM_MAX_EXPERTS:
            raise ValueError(f"experts {self.E} > {_lib.DM_MAX_EXPERTS}")

    # Algorithmic work: GEMM FLOPs and HBM bytes per micro-batch.
    def gemm_flops_fwd(self) -> int:
        return 6 * self.R * self.H * self.De

    def gemm_flops_bwd(self) -> int:
        return 12 * self.R * self.H * self.De

    def gemm_hbm_bytes(self, microbatches: int, e: int = 2, batched: bool = False) -> int:
        """Algorithmic HBM bytes of one iteration's expert GEMMs (unpadded rows): the
        forward and dgrad passes stream W13 + W2 (once per micro-batch, or once per
        iteration when the micro-batches run as one batched GEMM) and their activation
        operands/outputs; the deferred W pass reads every micro-batch's operands once and
        writes dW13 + dW2 in fp32. Fine-grained MoE (DeepSeek-V3: ~128 rows per expert) is
        bound by this, not by tensor FLOPs."""
        T, H, E, De, R = self.T, self.H, self.E, self.De, self.R
        w = E * 3 * H * De * e
        fwd = R * (H + 2 * De + De + De + H) * e          # x_perm, h13, act (w+r), y_perm
        dgrad = R * (H + 2 * De + 2 * De + 2 * De + H) * e  # dy_perm, h13, dh13 (w+r), dx_perm
        wgrad = microbatches * R * (H + De + 2 * De + H) * e + E * 3 * H * De * 4
        weights = 2 * w * (1 if batched else microbatches)
        return microbatches * (fwd + dgrad) + weights + wgrad

    def hbm_bytes(self, e: int = 2) -> dict[str, int]:
        T, H, R = self.T, self.H, self.R
        return {
            "dispatch": T * H * e + R * H * e + 8 * R,
            "combine_fwd": R * H * e + 4 * R + T * H * e,
            "combine_bwd": T * H * e + 2 * R * H * e + 4 * R,
            "permute_bwd": R * H * e + T * H * e,
        }

    @classmethod
    def from_experiment(cls, exp) -> "MoEShape":
        m = exp.model
        return cls(T=exp.workload.seq_len * exp.workload.micro_batch, H=m.hidden, E=m.experts,
                   k=m.topk, De=m.moe_hidden)


def interleave_w13(w1: torch.Tensor, w3: torch.Tensor, block: int = _lib.DM_GLU_BLOCK) -> torch.Tensor:
    """[E, D_e, H] gate + up -> [E, 2*D_e, H] with DM_GLU_BLOCK-row gate/up blocks (dm_moe.h)."""
    E, De, H = w1.shape
    out = torch.empty(E, 2 * De, H, dtype=w1.dtype, device=w1.device)
    v = out.view(E, De // block, 2, block, H)
    v[:, :, 0] = w1.view(E, De // block, block, H)
    v[:, :, 1] = w3.view(E, De // block, block, H)
    return out


def split_w13(w13: torch.Tensor, block: int = _lib.DM_GLU_BLOCK) -> tuple[torch.Tensor, torch.Tensor]:
    E, two_de, H = w13.shape
    v = w13.view(E, two_de // (2 * block), 2, block, H)
    return v[:, :, 0].reshape(E, two_de // 2, H), v[:, :, 1].reshape(E, two_de // 2, H)


class RouterParams:
    """A-side parameters: W_g fp32 [E, H] and its gradient."""

    def __init__(self, wg: torch.Tensor):
        self.wg = wg.contiguous()
        self.dwg = torch.zeros_like(self.wg)


class ExpertParams:
    """F-side parameters for a block of experts: W13 [E,2D_e,H], W2 [E,H,D_e] bf16,
    fp32 gradients dW13 / dW2 (accumulated across micro-batches with beta=1)."""

    def __init__(self, w13: torch.Tensor, w2: torch.Tensor):
        self.w13 = w13.contiguous()
        self.w2 = w2.contiguous()
        self.dw13 = torch.zeros(self.w13.shape, dtype=F32, device=w13.device)
        self.dw2 = torch.zeros(self.w2.shape, dtype=F32, device=w2.device)

    @property
    def num_experts(self) -> int:
        return self.w13.shape[0]


GEMM_MAX_GROUPS = 1024   # grouped_gemm_sm100.cu: groups per launch


class ActivationSlab:
    """F-side activations of `n` micro-batches stacked in contiguous [n*cap, .] slabs.

    Micro-batch i owns rows [i*cap, (i+1)*cap) of every slab, and row i of the
    [n, E+1] offset slab. Keeping a whole iteration resident (HBM is 180 GB) lets
    the weight-gradient GEMM run once per iteration with K = all of its tokens
    (dm_grouped_wgrad with nseg = n), instead of a fp32 read-modify-write of
    dW per micro-batch.
    """

    def __init__(self, shape: MoEShape, n: int, device, rows: int | None = None, f_side: bool = True):
        s = shape
        dev = torch.device(device)
        self.n = n
        self.cap = s.cap if rows is None else rows
        R = n * self.cap
        e = lambda *sh, dt=BF16: torch.empty(*sh, dtype=dt, device=dev)  # noqa: E731
        self.pad_off = torch.zeros(n, s.E + 1, dtype=I32, device=dev)
        self.x_perm = e(R, s.H)
        self.y_perm = e(R, s.H)
        self.dy_perm = e(R, s.H)
        self.dx_perm = e(R, s.H)
        if f_side:
            self.h13 = e(R, 2 * s.De)
            self.act = e(R, s.De)
            self.dh13 = e(R, 2 * s.De)

    def rows(self, i: int) -> slice:
        return slice(i * self.cap, (i + 1) * self.cap)


class MicroBatchBuffers:
    """Device buffers of one in-flight micro-batch; permuted/F-side tensors are
    views into an ActivationSlab (both sides live on one device on the fused path).

    residual=True makes the layer a residual block, y = x + MoE(x) and
    dx = dy + J^T dy, fused into combine_fwd / permute_bwd (layer stacks)."""

    def __init__(self, shape: MoEShape, device, slab: ActivationSlab, index: int, a_side: bool = True,
                 residual: bool = False):
        s = shape
        self.residual = residual
        dev = torch.device(device)
        z = lambda *sh, dt=BF16: torch.empty(*sh, dtype=dt, device=dev)  # noqa: E731
        self.shape = s
        self.slab = slab
        self.index = index
        self.cap = slab.cap
        rows = slab.rows(index)
        self.counts = z(s.E, dt=I32)
        self.pad_off = slab.pad_off[index]
        if a_side:
            self.x = z(s.T, s.H)
            self.idx = z(s.T, s.k, dt=I32)
            self.w = z(s.T, s.k, dt=F32)
            self.row_map = z(s.T, s.k, dt=I32)
            self.src = z(slab.cap, dt=I32)
            # zeroed: the streaming router's completion counters live in its last 4 KB
            self.route_ws = torch.zeros(_lib.route_workspace_size(s.T, s.H, s.E, s.k), dtype=torch.uint8, device=dev)
            self.wgrad_ws = torch.zeros(_lib.router_wgrad_workspace_size(s.T, s.H, s.E) // 4, dtype=F32, device=dev)
            self.y = z(s.T, s.H)
            self.dy = z(s.T, s.H)
            self.dw = z(s.T, s.k, dt=F32)
            self.dlogit = z(s.T, s.k, dt=F32)
            self.dl_perm = z(slab.cap, dt=F32)
            self.dx = z(s.T, s.H)
        self.x_perm = slab.x_perm[rows]
        self.y_perm = slab.y_perm[rows]
        self.dy_perm = slab.dy_perm[rows]
        self.dx_perm = slab.dx_perm[rows]
        if hasattr(slab, "h13"):
            self.h13 = slab.h13[rows]
            self.act = slab.act[rows]
            self.dh13 = slab.dh13[rows]


# ---------------------------------------------------------------- stages
def a_dispatch(buf: MicroBatchBuffers, router: RouterParams, stream=None) -> None:
    s = buf.shape
    K.route_and_dispatch(buf.x, router.wg, s.k, buf.route_ws, buf.idx, buf.w, buf.counts, buf.pad_off,
                         buf.row_map, buf.src, buf.x_perm, stream)


def f_forward(buf: MicroBatchBuffers, experts: ExpertParams, pad_off=None, stream=None) -> None:
    po = buf.pad_off if pad_off is None else pad_off
    K.w13_swiglu_fwd(buf.x_perm, experts.w13, po, buf.h13, buf.act, stream)
    K.w2_fwd(buf.act, experts.w2, po, buf.y_perm, stream)


def a_combine(buf: MicroBatchBuffers, stream=None) -> None:
    K.combine_fwd(buf.y_perm, buf.row_map, buf.w, buf.y, stream, resid=buf.x if buf.residual else None)


def a_combine_bwd(buf: MicroBatchBuffers, stream=None) -> None:
    K.combine_bwd(buf.dy, buf.y_perm, buf.row_map, buf.w, buf.counts, buf.pad_off, buf.dy_perm, buf.dw,
                  buf.dlogit, stream, dl_perm=buf.dl_perm)


def f_backward(buf: MicroBatchBuffers, experts: ExpertParams, accumulate: bool, pad_off=None,
               stream=None, defer_wgrad: bool = False) -> None:
    """dgrad (always) and, unless deferred to f_wgrad, this micro-batch's wgrad."""
    po = buf.pad_off if pad_off is None else pad_off
    K.w2_dgrad_swiglu_bwd(buf.dy_perm, experts.w2, buf.h13, po, buf.dh13, stream)
    K.w13_dgrad(buf.dh13, experts.w13, po, buf.dx_perm, stream)
    if not defer_wgrad:
        beta = 1.0 if accumulate else 0.0
        K.wgrad(buf.dy_perm, buf.act, po, experts.dw2, beta, stream)
        K.wgrad(buf.dh13, buf.x_perm, po, experts.dw13, beta, stream)


def f_wgrad(slab: ActivationSlab, n: int, experts: ExpertParams, accumulate: bool, stream=None) -> None:
    """Deferred weight-gradient pass over micro-batches 0..n-1 of the slab."""
    beta = 1.0 if accumulate else 0.0
    rows = slice(0, n * slab.cap)
    so = slab.pad_off[:n]
    K.wgrad(slab.dy_perm[rows], slab.act[rows], so, experts.dw2, beta, stream)
    K.wgrad(slab.dh13[rows], slab.x_perm[rows], so, experts.dw13, beta, stream)


def a_dispatch_bwd(buf: MicroBatchBuffers, router: RouterParams, accumulate: bool, stream=None) -> None:
    a_permute_bwd(buf, router, stream)
    a_router_wgrad(buf, router, accumulate, stream)


def a_permute_bwd(buf: MicroBatchBuffers, router: RouterParams, stream=None) -> None:
    K.permute_bwd(buf.dx_perm, buf.row_map, buf.idx, buf.dlogit, router.wg, buf.dx, stream,
                  resid=buf.dy if buf.residual else None)


def a_router_wgrad(buf: MicroBatchBuffers, router: RouterParams, accumulate: bool, stream=None) -> None:
    """dW_g (+)= dlogit^T x, deterministic. Few experts (E <= 16): token blocks, every x
    row read once, acc[E][8] per lane, partials reduced in token-block order by the last
    CTA of each column chunk. Many experts: over the expert-sorted rows (dlogit scattered
    to them by combine_bwd), R*H FMAs instead of T*E*H."""
    beta = 1.0 if accumulate else 0.0
    if buf.shape.E <= 16:
        K.router_wgrad(buf.x, buf.idx, buf.dlogit, buf.wgrad_ws, router.dwg, beta, stream)
    else:
        K.router_wgrad_sorted(buf.x, buf.src, buf.dl_perm, buf.counts, buf.pad_off, router.dwg, beta, stream,
                              partial_ws=buf.wgrad_ws)


class MoELayer:
    """Fused single-device MoE layer (1 GPU: A and F stages on one device).

    `iteration(n)` runs micro-batches 0..n-1 fwd + bwd (dgrad) and then one
    deferred weight-gradient pass; `forward_backward(buf)` is the one-micro-batch
    form with the wgrad inline.
    """

    def __init__(self, shape: MoEShape, wg: torch.Tensor, w13: torch.Tensor, w2: torch.Tensor,
                 device="cuda", num_buffers: int = 1, residual: bool = False):
        shape.validate()
        _lib.load()  # fail loudly if the sm_100a library is absent
        self.shape = shape
        self.device = torch.device(device)
        self.router = RouterParams(wg.to(self.device, F32))
        self.experts = ExpertParams(w13.to(self.device, BF16), w2.to(self.device, BF16))
        self.slab = ActivationSlab(shape, num_buffers, self.device)
        self.buffers = [MicroBatchBuffers(shape, self.device, self.slab, i, residual=residual)
                        for i in range(num_buffers)]

    @classmethod
    def random(cls, shape: MoEShape, device="cuda", seed: int = 0, num_buffers: int = 1,
               residual: bool = False) -> "MoELayer":
        g = torch.Generator(device="cpu").manual_seed(seed)
        wg = torch.randn(shape.E, shape.H, generator=g) * 0.02
        dev = torch.device(device)
        w13 = torch.empty(shape.E, 2 * shape.De, shape.H, dtype=BF16, device=dev)
        w2 = torch.empty(shape.E, shape.H, shape.De, dtype=BF16, device=dev)
        gd = torch.Generator(device=dev).manual_seed(seed + 1)
        w13.normal_(0.0, 0.02, generator=gd)
        w2.normal_(0.0, 0.02, generator=gd)
        return cls(shape, wg, w13, w2, device, num_buffers, residual)

    # stage entry points shared with moe_f32.MoELayerF32 (bench / profiling use these)
    def stage_dispatch(self, buf, stream=None):
        a_dispatch(buf, self.router, stream)

    def stage_f_forward(self, buf, stream=None):
        f_forward(buf, self.experts, stream=stream)

    def stage_combine(self, buf, stream=None):
        a_combine(buf, stream)

    def stage_combine_bwd(self, buf, stream=None):
        a_combine_bwd(buf, stream)

    def stage_f_backward(self, buf, accumulate: bool, stream=None):
        f_backward(buf, self.experts, accumulate, stream=stream, defer_wgrad=True)

    def stage_permute_bwd(self, buf, stream=None):
        a_permute_bwd(buf, self.router, stream)

    def stage_router_wgrad(self, buf, accumulate: bool, stream=None):
        a_router_wgrad(buf, self.router, accumulate, stream)

    dtype = BF16

    def forward(self, buf: MicroBatchBuffers, stream=None) -> None:
        a_dispatch(buf, self.router, stream)
        f_forward(buf, self.experts, stream=stream)
        a_combine(buf, stream)

    def backward(self, buf: MicroBatchBuffers, accumulate: bool, stream=None, defer_wgrad: bool = False) -> None:
        a_combine_bwd(buf, stream)
        f_backward(buf, self.experts, accumulate, stream=stream, defer_wgrad=defer_wgrad)
        a_dispatch_bwd(buf, self.router, accumulate, stream)

    def forward_backward(self, buf: MicroBatchBuffers, accumulate: bool = False, stream=None,
                         defer_wgrad: bool = False) -> None:
        self.forward(buf, stream)
        self.backward(buf, accumulate, stream, defer_wgrad)

    def wgrad(self, n: int | None = None, accumulate: bool = False, stream=None) -> None:
        f_wgrad(self.slab, len(self.buffers) if n is None else n, self.experts, accumulate, stream)

    # ---- batched F side: the n micro-batches' expert GEMMs as ONE launch each, groups
    # ordered expert-major (dm_batch_group_ranges), so each expert's W13 / W2 stream once per
    # iteration instead of once per micro-batch; per-row results are bit-identical.
    def batched_supported(self, n: int) -> bool:
        """Batched F side: by default (DM_BATCHED unset / "auto") for fine-grained experts, where
        the shared weight pass and pair tiles pay (DeepSeek-V3 +13-19%, the tiny config +40%);
        coarse experts (Mixtral) measured 1% slower batched on the same box, so they stay per
        micro-batch unless DM_BATCHED=1. DM_BATCHED=0 disables it."""
        import os

        mode = os.environ.get("DM_BATCHED", "auto")
        if mode == "0" or n < 2 or self.shape.E * n > GEMM_MAX_GROUPS or os.environ.get("DM_GEMM_1SM") == "1":
            return False
        return mode == "1" or self.merged_groups()

    def merged_groups(self) -> bool:
        """Expert-major groups (one weight pass for all micro-batches, chunks of different
        micro-batches sharing pair tiles) when experts are fine-grained (< 512 rows per expert
        and micro-batch: weight streaming and half tiles dominate, e.g. DeepSeek-V3); coarse
        experts (Mixtral: ~1024 rows) keep the per-micro-batch tile order in one launch — the
        expert-major order re-reads their large A panels from DRAM (ncu: w13 dgrad 26 GB)."""
        return self.shape.R < 512 * self.shape.E

    def _group_ranges(self, n: int, stream=None):
        key = ("ranges", n)
        if getattr(self, "_rng_key", None) != key:
            self._rng = (torch.empty(n * self.shape.E, dtype=I32, device=self.device),
                         torch.empty(n * self.shape.E, dtype=I32, device=self.device))
            self._rng_key = key
        gs, ge = self._rng
        K.batch_group_ranges(self.slab.pad_off[:n], self.slab.cap, gs, ge, self.merged_groups(), stream)
        return gs, ge

    def f_forward_all(self, n: int, stream=None) -> None:
        sl, ex = self.slab, self.experts
        rows = slice(0, n * sl.cap)
        gs, ge = self._group_ranges(n, stream)
        bd = n if self.merged_groups() else 1
        K.w13_swiglu_fwd_ranges(sl.x_perm[rows], ex.w13, gs, ge, bd, sl.h13[rows], sl.act[rows], stream)
        K.w2_fwd_ranges(sl.act[rows], ex.w2, gs, ge, bd, sl.y_perm[rows], stream)

    def f_backward_all(self, n: int, stream=None) -> None:
        sl, ex = self.slab, self.experts
        rows = slice(0, n * sl.cap)
        gs, ge = self._rng   # from this iteration's forward
        bd = n if self.merged_groups() else 1
        K.w2_dgrad_swiglu_bwd_ranges(sl.dy_perm[rows], ex.w2, sl.h13[rows], gs, ge, bd, sl.dh13[rows], stream)
        K.w13_dgrad_ranges(sl.dh13[rows], ex.w13, gs, ge, bd, sl.dx_perm[rows], stream)

    def forward_all(self, n: int, stream=None) -> None:
        for i in range(n):
            a_dispatch(self.buffers[i], self.router, stream)
        self.f_forward_all(n, stream)
        for i in range(n):
            a_combine(self.buffers[i], stream)

    def backward_all(self, n: int, accumulate: bool, stream=None) -> None:
        for i in range(n):
            a_combine_bwd(self.buffers[i], stream)
        self.f_backward_all(n, stream)
        for i in range(n):
            a_dispatch_bwd(self.buffers[i], self.router, accumulate or i > 0, stream)

    def iteration(self, n: int | None = None, accumulate: bool = False, stream=None) -> None:
        """Micro-batches 0..n-1 (inputs already in buffers[i].x / .dy), then the W pass:
        batched (all forwards, all backwards, one GEMM launch per stage) when supported,
        else micro-batch by micro-batch. Same results either way."""
        n = len(self.buffers) if n is None else n
        if self.batched_supported(n):
            self.forward_all(n, stream)
            self.backward_all(n, accumulate, stream)
        else:
            for i in range(n):
                self.forward_backward(self.buffers[i], accumulate=accumulate or i > 0, stream=stream,
                                      defer_wgrad=True)
        self.wgrad(n, accumulate, stream)

    def zero_grad(self) -> None:
        self.router.dwg.zero_()
        self.experts.dw13.zero_()
        self.experts.dw2.zero_()

    launches_per_wgrad_pass = 2

    def launches_per_microbatch(self, deferred_wgrad: bool = False) -> int:
        """dm kernel launches of one micro-batch: dispatch (one cooperative streaming
        launch when E <= 16, H % 256 == 0, k <= 8 and W_g fits in smem; else the
        32-token fused router + scan + permute = 3 when W_g fits in 160 KB; else
        logits + top-k + scan + permute = 4), expert fwd 2, combine 1, combine bwd 1,
        dgrad 2, permute bwd 1, router wgrad 1 (segments reduced in-kernel), plus 2 wgrad
        GEMMs unless deferred to the iteration's W pass."""
        s = self.shape
        return dispatch_launches(s) + 7 + 1 + (0 if deferred_wgrad else 2)


def dispatch_launches(s: MoEShape) -> int:
    """Kernel launches of dm_route_and_dispatch (mirrors dispatch.cu's path choice)."""
    ni = (s.H // 8 + 31) // 32
    em = 8 if s.E <= 8 else 16
    nunit = -(-s.T // _lib.DM_ROUTE_UNIT_TOKENS)
    sms = _lib.load().dm_num_sms(torch.cuda.current_device())
    grid = min(nunit, sms)
    upc = -(-nunit // grid)
    grid = -(-nunit // upc)
    scratch = ((grid * s.E + upc * _lib.DM_ROUTE_UNIT_TOKENS * s.k) * 4 + 1023) // 1024 * 1024
    import os

    if (os.environ.get("DM_DISPATCH_LEGACY", "0") != "1" and s.E <= 16 and s.H % 256 == 0 and _lib.DM_ROUTE_UNIT_TOKENS * s.k <= 32
            and 1024 + em * s.H * 4 + 4096 <= 227 * 1024 and upc <= 64 and scratch + 4 * s.H <= em * s.H * 4):
        return 1   # one cooperative launch: route, grid barrier, scan, permute
    if s.E <= 16 and em * ni * 64 * 16 <= 160 * 1024:
        return 3
    return 4


def _router_wgrad_segments(s: MoEShape) -> int:
    """Row segments dm_router_wgrad_sorted uses (mirrors combine.cu's launcher)."""
    import math

    sms = _lib.load().dm_num_sms(torch.cuda.current_device())
    gx = math.ceil(s.H / 8 / 128)
    cap_seg = math.ceil(s.T / _lib.router_wgrad_token_block(s.E))
    return max(1, min(math.ceil(4 * sms / (gx * s.E)), cap_seg))


def link_residual_stack(stack_bufs: list[list[MicroBatchBuffers]]) -> None:
    """Chain per-layer buffers of a residual layer stack in place: layer l+1 reads its
    input from layer l's output (x_{l+1} is y_l) and layer l's upstream gradient is
    layer l+1's input gradient (dy_l is dx_{l+1}), so no copies sit between layers."""
    for lo, hi in zip(stack_bufs[:-1], stack_bufs[1:]):
        for a, b in zip(lo, hi):
            b.x = a.y
            a.dy = b.dx


class MoEStack:
    """Fused single-device stack of residual MoE blocks, x_{l+1} = x_l + MoE_l(x_l)
    (the tiny config's 2-layer model), optionally preceded per layer by the A-side
    attention block (attention.AttentionBlock: h_l = x_l + attn(x_l), then
    x_{l+1} = h_l + MoE_l(h_l)). A 1-layer stack without attention is the plain layer.

    I/O per micro-batch i: `input(i)`, `output_grad(i)` in; `output(i)`, `input_grad(i)` out.
    """

    def __init__(self, layers: list, attention: list | None = None, seq_len: int | None = None):
        if not layers:
            raise ValueError("empty stack")
        if attention is not None and len(attention) != len(layers):
            raise ValueError("one attention block per layer")
        self.layers = layers
        self.attn = attention
        self.buffers = layers[0].buffers
        self.out_buffers = layers[-1].buffers
        if attention is None:
            link_residual_stack([l.buffers for l in layers])
        else:
            s = layers[0].shape
            self.seq_len = seq_len or s.T
            dt, dev = layers[0].dtype, layers[0].device
            n = len(self.buffers)
            self.inp = [torch.empty(s.T, s.H, dtype=dt, device=dev) for _ in range(n)]
            self.dinp = [torch.empty(s.T, s.H, dtype=dt, device=dev) for _ in range(n)]

    def input(self, i: int) -> torch.Tensor:
        return self.buffers[i].x if self.attn is None else self.inp[i]

    def input_grad(self, i: int) -> torch.Tensor:
        return self.buffers[i].dx if self.attn is None else self.dinp[i]

    def output(self, i: int) -> torch.Tensor:
        return self.out_buffers[i].y

    def output_grad(self, i: int) -> torch.Tensor:
        return self.out_buffers[i].dy

    @classmethod
    def random(cls, shape: MoEShape, num_layers: int, device="cuda", seed: int = 0,
               num_buffers: int = 1) -> "MoEStack":
        return cls([MoELayer.random(shape, device, seed + 1000 * l, num_buffers, residual=True)
                    for l in range(num_layers)])

    def forward(self, i: int, stream=None) -> None:
        for l, layer in enumerate(self.layers):
            if self.attn is not None:
                x_in = self.inp[i] if l == 0 else self.layers[l - 1].buffers[i].y
                self.attn[l].forward(i, x_in, layer.buffers[i].x, self.seq_len)
            layer.forward(layer.buffers[i], stream)

    def backward(self, i: int, accumulate: bool = False, stream=None, defer_wgrad: bool = False) -> None:
        for l in reversed(range(len(self.layers))):
            layer = self.layers[l]
            layer.backward(layer.buffers[i], accumulate, stream, defer_wgrad)
            if self.attn is not None:
                dst = self.dinp[i] if l == 0 else self.layers[l - 1].buffers[i].dy
                self.attn[l].backward(i, layer.buffers[i].dx, dst, accumulate)

    def forward_backward(self, i: int, accumulate: bool = False, stream=None, defer_wgrad: bool = False) -> None:
        self.forward(i, stream)
        self.backward(i, accumulate, stream, defer_wgrad)

    def batched_supported(self, n: int) -> bool:
        return all(getattr(l, "batched_supported", lambda n: False)(n) for l in self.layers)

    def forward_all(self, n: int, stream=None) -> None:
        """Layer by layer, every micro-batch (the batched form of forward(i) for all i)."""
        for l, layer in enumerate(self.layers):
            if self.attn is not None:
                for i in range(n):
                    x_in = self.inp[i] if l == 0 else self.layers[l - 1].buffers[i].y
                    self.attn[l].forward(i, x_in, layer.buffers[i].x, self.seq_len)
            layer.forward_all(n, stream)

    def backward_all(self, n: int, accumulate: bool = False, stream=None) -> None:
        for l in reversed(range(len(self.layers))):
            layer = self.layers[l]
            layer.backward_all(n, accumulate, stream)
            if self.attn is not None:
                for i in range(n):
                    dst = self.dinp[i] if l == 0 else self.layers[l - 1].buffers[i].dy
                    self.attn[l].backward(i, layer.buffers[i].dx, dst, accumulate or i > 0)

    def iteration(self, n: int | None = None, accumulate: bool = False, stream=None) -> None:
        n = len(self.buffers) if n is None else n
        if self.batched_supported(n):
            self.forward_all(n, stream)
            self.backward_all(n, accumulate, stream)
        else:
            for i in range(n):
                self.forward_backward(i, accumulate or i > 0, stream, defer_wgrad=True)
        for layer in self.layers:
            layer.wgrad(n, accumulate, stream)

    def zero_grad(self) -> None:
        for layer in self.layers:
            layer.zero_grad()

    def capture(self, n: int | None = None, accumulate: bool = False) -> "StackGraphs":
        """Record the iteration as CUDA graphs: one per micro-batch (fwd + bwd of every
        layer, wgrad deferred) and one for the W pass. Every launch is stream-ordered
        with device-side sizes and fixed buffers, so the graphs replay with new data
        written in place; the host then issues n + 1 graph launches per iteration
        instead of ~13 kernel launches per layer and micro-batch."""
        n = len(self.buffers) if n is None else n
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):          # warm-up: lazy kernel attributes, TMA paths
            self.iteration(n, accumulate)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graphs, launches = [], 0
        batched = self.batched_supported(n)
        if batched:   # two graphs: every micro-batch's forward, then every backward (batched GEMMs)
            for part in (lambda: self.forward_all(n), lambda: self.backward_all(n, accumulate)):
                g = torch.cuda.CUDAGraph()
                c0 = _lib.launch_count()
                with torch.cuda.graph(g):
                    part()
                launches += _lib.launch_count() - c0
                graphs.append(g)
        for i in range(0 if batched else n):
            g = torch.cuda.CUDAGraph()
            c0 = _lib.launch_count()
            with torch.cuda.graph(g):
                self.forward_backward(i, accumulate or i > 0, defer_wgrad=True)
            launches += _lib.launch_count() - c0
            graphs.append(g)
        gw = torch.cuda.CUDAGraph()
        c0 = _lib.launch_count()
        with torch.cuda.graph(gw):
            for layer in self.layers:
                layer.wgrad(n, accumulate)
        launches += _lib.launch_count() - c0
        return StackGraphs(graphs, gw, launches, batched)


@dataclass
class StackGraphs:
    """Captured iteration of a MoEStack (MoEStack.capture): `microbatch[i]` (fwd + bwd of
    micro-batch i) then `wgrad`; batched: `microbatch` = [all forwards, all backwards]."""

    microbatch: list
    wgrad: object
    launches_per_iteration: int
    batched: bool = False

    def replay(self) -> None:
        for g in self.microbatch:
            g.replay()
        self.wgrad.replay()


class MoEFunction(torch.autograd.Function):
    """autograd entry point: y = MoE(x; W_g, W13, W2) on one device.

    Gradients: dx (bf16), dW_g / dW13 / dW2 (fp32, same shapes as the weights).
    """

    @staticmethod
    def forward(ctx, x, wg, w13, w2, k: int):
        T, H = x.shape
        E, two_de, _ = w13.shape
        shape = MoEShape(T=T, H=H, E=E, k=k, De=two_de // 2)
        shape.validate()
        buf = MicroBatchBuffers(shape, x.device, ActivationSlab(shape, 1, x.device), 0)
        buf.x.copy_(x)
        router = RouterParams(wg.detach().float().contiguous())
        experts = ExpertParams.__new__(ExpertParams)
        experts.w13, experts.w2 = w13.detach().contiguous(), w2.detach().contiguous()
        a_dispatch(buf, router)
        f_forward(buf, experts)
        a_combine(buf)
        ctx.buf, ctx.router, ctx.experts = buf, router, experts
        return buf.y.clone()

    @staticmethod
    def backward(ctx, dy):
        buf, router, experts = ctx.buf, ctx.router, ctx.experts
        experts.dw13 = torch.empty(experts.w13.shape, dtype=F32, device=dy.device)
        experts.dw2 = torch.empty(experts.w2.shape, dtype=F32, device=dy.device)
        buf.dy.copy_(dy.to(BF16))
        a_combine_bwd(buf)
        f_backward(buf, experts, accumulate=False)
        a_dispatch_bwd(buf, router, accumulate=False)
        return buf.dx.clone(), router.dwg, experts.dw13, experts.dw2, None


def moe(x: torch.Tensor, wg: torch.Tensor, w13: torch.Tensor, w2: torch.Tensor, k: int) -> torch.Tensor:
    """y = MoE(x); bf16 x -> the bf16 path, fp32 x -> fp32 mode (moe_f32)."""
    if x.dtype == F32:
        from .moe_f32 import MoEFunctionF32

        return MoEFunctionF32.apply(x, wg, w13, w2, k)
    return MoEFunction.apply(x, wg, w13, w2, k)
