"""AF-Pipe runtime: attention (A) ranks and FFN (F) ranks of one node exchanging
micro-batches of a stack of MoE layers over NCCL (NVLink 5 / NVSwitch).

One process per GPU (torchrun). Ranks [0, n_attn) are A ranks — data parallel,
each routes its own micro-batches with a replicated router W_g; ranks
[n_attn, world) are F ranks — expert parallel, F rank f owns the contiguous
expert block of reference taskgraph._balanced_blocks (taskgraph.py:257-259).
Per micro-batch i (afpipe.build_layer_dag):

    A_f   route + permute x -> x_perm (expert blocks grouped by owning F rank)
    M2N   A -> F: header pad_off[lo_f..hi_f] (E_loc+1 ints, fixed size) then the
          contiguous x_perm slice [pad_off[lo_f], pad_off[hi_f]) (reference
          M2NSend/M2NRecv twins, taskgraph.py:204-242, volume costs.py:95-103)
    F_f   grouped SwiGLU GEMMs over (A rank, expert) groups
    N2M   F -> A: y_perm rows back into the same slice (taskgraph.py:335-339)
    A_t   combine (weighted sum), loss turnaround, combine bwd -> dy_perm
    M2N_b A -> F: dy_perm slices;   F_b: dgrad GEMMs (wgrad deferred)
    N2M_b F -> A: dx_perm slices;   A_b: permute bwd + router grads
    end:  F: one wgrad pass per layer over all (micro-batch, A rank) segments;
          A: all-reduce of dW_g over the A group (the only DP collective).

With `layers` = L > 1 (pipeline_depth 1, virtual_stages L: BASELINE configs[0]) the
layers are residual blocks x_{l+1} = x_l + MoE_l(x_l): A_f of layer l > 0 is layer
l-1's combine (residual fused) followed by layer l's dispatch, A_t turns around the
last layer, and A_b of layer l > 0 also runs layer l-1's combine backward
(afpipe.build_layer_dag). Layer l+1's input buffer IS layer l's output buffer.

Message sizes are data dependent; the only host synchronisation is reading the
128-aligned offsets once per micro-batch (A: its own pad_off after dispatch;
F: the received headers) on a side copy stream, so the compute stream never
drains. Every rank issues its tasks in the planned order of afpipe.plan_layer,
which makes the per-pair send/recv sequences identical on both ends.

Stage arithmetic comes from a `Stages` object: `GpuStages` (the sm_100a
kernels through the C ABI) is the product. Tests inject a CPU restatement to
exercise this file's protocol under gloo; there is no automatic fallback.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import torch

from . import _lib
from .afpipe import COMPUTE, SEND, LayerDurations, issue_order, plan_layer
from .moe import ActivationSlab, ExpertParams, MicroBatchBuffers, MoEShape, RouterParams, link_residual_stack
from .transport import AF, NcclTransport, direction_of

BF16, F32, I32 = torch.bfloat16, torch.float32, torch.int32


# ------------------------------------------------------------------ topology
def balanced_blocks(total: int, parts: int) -> list[int]:
    """Sizes of `parts` contiguous blocks of `total` (reference taskgraph.py:257-259)."""
    base, extra = divmod(total, parts)
    return [base + (1 if i < extra else 0) for i in range(parts)]


@dataclass(frozen=True)
class Topology:
    """A:F split of `world` ranks, optionally into `depth` = p pipeline groups
    (reference pipeline_depth; placement.assign_layers, placement.py:42-55): ranks
    [0, n_attn) are A ranks, A group g = ranks [g*a_p, (g+1)*a_p) with a_p = n_attn/p;
    the rest are F ranks, F group g = the g-th block of f_p = n_ffn/p ranks. Layer l runs
    on A group and F group l mod p; stream j (a DP replica of the micro-batch chain) uses
    member j of every A group."""

    world: int
    n_attn: int
    experts: int
    depth: int = 1

    def __post_init__(self):
        if not (1 <= self.n_attn < self.world):
            raise ValueError(f"need 1 <= n_attn < world (n_attn={self.n_attn}, world={self.world})")
        if self.depth < 1 or self.n_attn % self.depth or self.n_ffn % self.depth:
            raise ValueError(f"pipeline depth {self.depth} must divide n_attn={self.n_attn} and n_ffn={self.n_ffn}")
        if self.f_per_group > self.experts:
            raise ValueError(f"{self.f_per_group} FFN ranks per group for {self.experts} experts")

    @property
    def n_ffn(self) -> int:
        return self.world - self.n_attn

    @property
    def a_per_group(self) -> int:
        return self.n_attn // self.depth

    @property
    def f_per_group(self) -> int:
        return self.n_ffn // self.depth

    @property
    def streams(self) -> int:
        """Independent micro-batch chains (tokens per step = streams * mb * T)."""
        return self.a_per_group

    def role(self, rank: int) -> tuple[str, int]:
        return ("A", rank) if rank < self.n_attn else ("F", rank - self.n_attn)

    def group_of(self, rank: int) -> tuple[int, int]:
        """(pipeline group, member index within the group) of a rank."""
        role, i = self.role(rank)
        per = self.a_per_group if role == "A" else self.f_per_group
        return i // per, i % per

    def a_rank(self, a: int, group: int = 0) -> int:
        return group * self.a_per_group + a

    def f_rank(self, f: int, group: int = 0) -> int:
        return self.n_attn + group * self.f_per_group + f

    def expert_block(self, f: int) -> tuple[int, int]:
        """Expert range of member f of an F group (every group holds all experts of its layers)."""
        sizes = balanced_blocks(self.experts, self.f_per_group)
        lo = sum(sizes[:f])
        return lo, lo + sizes[f]

    def layers_of(self, group: int, layers: int) -> list[int]:
        return list(range(group, layers, self.depth))

    @classmethod
    def default(cls, world: int, experts: int, n_attn: int | None = None, depth: int = 1) -> "Topology":
        """A:F = n_attn : world-n_attn; default half/half (BASELINE configs[1]: 4 + 4)."""
        if n_attn is None:
            n_attn = max(1, world // 2)
        return cls(world, n_attn, experts, depth)


# ------------------------------------------------------------------ streams
class _Streams:
    """compute / send / recv / copy streams on CUDA; no-ops on CPU (gloo tests). `copy`
    carries the small count reads the exchange waits on, `h2d` / `d2h` the e2e mode's
    activation copies, so a 32 MB input copy never delays a count read."""

    def __init__(self, device: torch.device):
        self.cuda = device.type == "cuda"
        if self.cuda:
            self.compute = torch.cuda.current_stream(device)
            self.send = torch.cuda.Stream(device)
            self.recv = torch.cuda.Stream(device)
            self.copy = torch.cuda.Stream(device)
            self.h2d = torch.cuda.Stream(device)
            self.d2h = torch.cuda.Stream(device)

    def ctx(self, which: str):
        """Make stream `which` current; leaving returns to the compute stream (contexts are
        never nested). Lighter than torch.cuda.stream(), whose per-call device/stream
        queries dominated the host side of small-shape iterations."""
        if not self.cuda:
            return _Null()
        return _StreamCtx(getattr(self, which), self.compute)

    def event(self, which: str = "compute", timing: bool = False):
        if not self.cuda:
            return None
        ev = torch.cuda.Event(enable_timing=timing)
        ev.record(getattr(self, which))
        return ev

    def wait(self, which: str, ev) -> None:
        if self.cuda and ev is not None:
            getattr(self, which).wait_event(ev)


class _StreamCtx:
    __slots__ = ("s", "back")

    def __init__(self, s, back):
        self.s, self.back = s, back

    def __enter__(self):
        torch.cuda.set_stream(self.s)
        return self

    def __exit__(self, *a):
        torch.cuda.set_stream(self.back)
        return False


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _exchange(ops: list[tuple[str, torch.Tensor, int]], direction: str = AF):
    """One coalesced group of P2P ops on the default NCCL/gloo transport (kept for callers
    outside AFPipeRank; the runtime itself goes through its `transport`)."""
    return _default_transport().exchange(ops, direction)


_DEFAULT_TX = []


def _default_transport() -> NcclTransport:
    if not _DEFAULT_TX:
        _DEFAULT_TX.append(NcclTransport())
    return _DEFAULT_TX[0]


# ------------------------------------------------------------------ stages
class GpuStages:
    """The product stage implementations: sm_100a kernels via the C ABI."""

    def __init__(self):
        _lib.load()

    def a_dispatch(self, buf: MicroBatchBuffers, router: RouterParams):
        from .moe import a_dispatch

        a_dispatch(buf, router)

    def a_combine(self, buf: MicroBatchBuffers):
        from .moe import a_combine

        a_combine(buf)

    def a_combine_bwd(self, buf: MicroBatchBuffers):
        from .moe import a_combine_bwd

        a_combine_bwd(buf)

    def a_backward(self, buf: MicroBatchBuffers, router: RouterParams, accumulate: bool):
        from .moe import a_dispatch_bwd

        a_dispatch_bwd(buf, router, accumulate)

    def f_forward(self, fb, experts: ExpertParams, group_off: torch.Tensor, ranges=None):
        """ranges = (start, end, b_div): expert-major row ranges over the A ranks' slices (one
        weight pass for all of them, 128-row chunks of different A ranks sharing pair tiles)."""
        from . import kernels as K

        if ranges is not None:
            gs, ge, bd = ranges
            K.w13_swiglu_fwd_ranges(fb.x_perm, experts.w13, gs, ge, bd, fb.h13, fb.act)
            K.w2_fwd_ranges(fb.act, experts.w2, gs, ge, bd, fb.y_perm)
            return
        K.w13_swiglu_fwd(fb.x_perm, experts.w13, group_off, fb.h13, fb.act)
        K.w2_fwd(fb.act, experts.w2, group_off, fb.y_perm)

    def f_backward(self, fb, experts: ExpertParams, group_off: torch.Tensor, ranges=None):
        from . import kernels as K

        if ranges is not None:
            gs, ge, bd = ranges
            K.w2_dgrad_swiglu_bwd_ranges(fb.dy_perm, experts.w2, fb.h13, gs, ge, bd, fb.dh13)
            K.w13_dgrad_ranges(fb.dh13, experts.w13, gs, ge, bd, fb.dx_perm)
            return
        K.w2_dgrad_swiglu_bwd(fb.dy_perm, experts.w2, fb.h13, group_off, fb.dh13)
        K.w13_dgrad(fb.dh13, experts.w13, group_off, fb.dx_perm)

    def f_wgrad(self, slab: ActivationSlab, experts: ExpertParams, seg_off: torch.Tensor, accumulate: bool,
                seg_stride_rows: int = 0):
        """seg_stride_rows 0: absolute segment rows; > 0: segment i's rows are relative
        to i * seg_stride_rows (the fixed-size 1:1 exchange)."""
        from . import kernels as K

        beta = 1.0 if accumulate else 0.0
        K.wgrad(slab.dy_perm, slab.act, seg_off, experts.dw2, beta, seg_stride_rows=seg_stride_rows)
        K.wgrad(slab.dh13, slab.x_perm, seg_off, experts.dw13, beta, seg_stride_rows=seg_stride_rows)


@dataclass
class _FMicroBatch:
    """F-side view of micro-batch i: a region of the F slab holding the n_attn
    received slices back to back (rows [base, base + rows))."""

    x_perm: torch.Tensor
    y_perm: torch.Tensor
    dy_perm: torch.Tensor
    dx_perm: torch.Tensor
    h13: torch.Tensor
    act: torch.Tensor
    dh13: torch.Tensor
    headers: list[torch.Tensor] = field(default_factory=list)   # per A rank, [E_loc+1] int32
    slices: list[tuple[int, int]] = field(default_factory=list)  # per A rank (row begin, rows) in region
    group_off: torch.Tensor | None = None                        # [n_attn*E_loc + 1] (region-relative)
    works: dict = field(default_factory=dict)


@dataclass
class IterationStats:
    ms: float
    events: list = field(default_factory=list)   # (task name, mb, lane, start_ms, end_ms) relative to t0


class AFPipeRank:
    """One rank of the AF-Pipe runtime for a stack of `layers` MoE layers over
    `topo.depth` pipeline groups (layer l on A group / F group l mod depth).

    A ranks: `lbufs[l][i]` (layer l, micro-batch i) and `routers[l]` for the layers of
    their group; `input(i)` / `input_grad(i)` on group 0, `out_bufs[i]` (y, dy) on the
    group of the last layer. F ranks: `expert_layers[l]`, one activation slab per layer
    of their group. Per-layer state is keyed by layer index; `router` / `experts` /
    `bufs` alias the group's first layer (the single-layer API)."""

    def __init__(self, shape: MoEShape, topo: Topology, rank: int, microbatches: int, device,
                 stages=None, seed: int = 0, weights=None, durations: LayerDurations | None = None,
                 record_events: bool = False, layers: int = 1, residual: bool | None = None,
                 attention: bool = False, seq_len: int | None = None, gqa_group: int = 1, transport=None):
        shape.validate() if device.type == "cuda" else None
        # NcclTransport (one process per GPU) or transport.LoopbackTransport (ranks as
        # threads of one process on one device)
        self.tx = transport if transport is not None else _default_transport()
        if layers < 1:
            raise ValueError(f"layers must be >= 1, got {layers}")
        if topo.depth > layers:
            raise ValueError(f"pipeline depth {topo.depth} > layers {layers}")
        self.shape, self.topo, self.rank, self.mb, self.L = shape, topo, rank, microbatches, layers
        self.p = topo.depth
        self.attention = attention
        self.seq_len = seq_len or shape.T
        self.residual = (layers > 1 or attention) if residual is None else residual
        self.device = torch.device(device)
        self.role, self.idx = topo.role(rank)
        self.group, self.member = topo.group_of(rank)
        # One A and one F rank per pipeline group: the F rank owns every expert, so the
        # A rank's whole capacity buffer is the slice; exchanges are fixed-size (cap rows)
        # and the received padded offsets are used on the device as the F-side group
        # offsets directly — no host synchronisation anywhere in the iteration.
        self.fixed = (topo.a_per_group == 1 and topo.f_per_group == 1
                      and os.environ.get("DM_AFPIPE_FIXED", "1") != "0")
        self.my_layers = topo.layers_of(self.group, layers)
        self.stages = stages if stages is not None else GpuStages()
        self.st = _Streams(self.device)
        self.record_events = record_events and self.st.cuda
        self._attn_flops = None
        if attention:
            from .attention import attention_flops

            self._attn_flops = attention_flops(shape.H, gqa_group, self.seq_len, shape.T // self.seq_len)
        d = durations or self._default_durations()
        self.plan = plan_layer(microbatches, d, layers=layers, depth=self.p)
        self.order = issue_order(self.plan, f"{self.role}{self.group}")
        if isinstance(weights, dict):
            weights = [weights]
        if weights is not None and len(weights) != layers:
            raise ValueError(f"{len(weights)} weight sets for {layers} layers")
        s = shape
        mbr = range(microbatches)
        if self.role == "A":
            self.routers, self.lbufs = {}, {}
            for l in self.my_layers:
                if weights:
                    wg = weights[l]["wg"]
                else:
                    wg = torch.randn(s.E, s.H, generator=torch.Generator().manual_seed(seed + 1000 * l)) * 0.02
                self.routers[l] = RouterParams(wg.to(self.device, F32))
                slab = ActivationSlab(s, microbatches, self.device, f_side=False)
                self.lbufs[l] = [MicroBatchBuffers(s, self.device, slab, i, residual=self.residual) for i in mbr]
            self.attn = None
            e = lambda: torch.empty(s.T, s.H, dtype=BF16, device=self.device)  # noqa: E731
            if attention:   # A-side attention per layer (library stopgap, attention.py)
                from .attention import AttentionBlock

                self.attn = {l: AttentionBlock(s.H, gqa_group, self.device, seed=seed + 77 + l) for l in self.my_layers}
                # attention input x_l and its gradient: the stream input/grad on layer 0,
                # received from / sent to the previous layer's A group otherwise
                self.xin = {l: [e() for _ in mbr] for l in self.my_layers}
                self.gin = {l: [e() for _ in mbr] for l in self.my_layers}
                if self.p == 1:
                    for l in self.my_layers[1:]:
                        self.xin[l] = [b.y for b in self.lbufs[l - 1]]
                        self.gin[l] = [b.dy for b in self.lbufs[l - 1]]
            elif self.p == 1:
                link_residual_stack([self.lbufs[l] for l in self.my_layers])
            first = self.my_layers[0]
            self.router, self.bufs = self.routers[first], self.lbufs[first]
            if layers - 1 in self.lbufs:
                self.out_bufs = self.lbufs[layers - 1]
            self.pad_host = {l: [torch.empty(s.E + 1, dtype=I32, pin_memory=self.st.cuda) for _ in mbr]
                             for l in self.my_layers}
            self.pad_ready = {l: [None] * microbatches for l in self.my_layers}
            self.a_group = None
        else:
            lo, hi = topo.expert_block(self.member)
            self.lo, self.hi, self.E_loc = lo, hi, hi - lo
            self.n_src = topo.a_per_group   # A ranks feeding this F group
            # worst case: every routed row of every A rank of the group lands on this F rank
            self.cap_f = self.n_src * s.cap
            self.expert_layers, self.slabs, self.lfmb, self.seg_offs = {}, {}, {}, {}
            for l in self.my_layers:
                if weights:
                    w13, w2 = weights[l]["w13"][lo:hi], weights[l]["w2"][lo:hi]
                else:
                    g = torch.Generator(device=self.device).manual_seed(seed + 1 + self.member + 1000 * l)
                    w13 = torch.empty(self.E_loc, 2 * s.De, s.H, dtype=BF16, device=self.device).normal_(0, 0.02, generator=g)
                    w2 = torch.empty(self.E_loc, s.H, s.De, dtype=BF16, device=self.device).normal_(0, 0.02, generator=g)
                self.expert_layers[l] = ExpertParams(w13.to(self.device), w2.to(self.device))
                sl = ActivationSlab(s, microbatches, self.device, rows=self.cap_f)
                fmb = []
                for i in mbr:
                    r = sl.rows(i)
                    fmb.append(_FMicroBatch(sl.x_perm[r], sl.y_perm[r], sl.dy_perm[r], sl.dx_perm[r],
                                            sl.h13[r], sl.act[r], sl.dh13[r]))
                    fmb[-1].headers = [torch.zeros(self.E_loc + 1, dtype=I32, device=self.device)
                                       for _ in range(self.n_src)]
                self.slabs[l] = sl
                self.lfmb[l] = fmb
                self.seg_offs[l] = torch.zeros(microbatches * self.n_src, self.E_loc + 1, dtype=I32, device=self.device)
            first = self.my_layers[0]
            self.experts, self.slab, self.fmb, self.seg_off = (self.expert_layers[first], self.slabs[first],
                                                               self.lfmb[first], self.seg_offs[first])
        self.trace: list = []
        self.t0 = None
        self.host_io = None
        self.x_free, self.dy_free = [], []   # per micro-batch: last reader of x / dy done (e2e)
        self._start_override = None          # tracing: compute-interval start after a task's waits

    # ----------------------------------------------------------------- plan
    def _default_durations(self) -> LayerDurations:
        """Rough per-stage estimates (ns) to derive the issue order; only the order matters."""
        s = self.shape
        tflops = 1.0e15
        per_f = max(1, self.topo.f_per_group)
        n_src = self.topo.a_per_group
        f_fwd = int(6 * s.R * s.H * s.De * n_src / per_f / tflops * 1e9)
        m2n = int(2 * s.R * s.H / max(1, min(n_src, per_f)) / 7.0e11 * 1e9)
        a = int(sum(s.hbm_bytes().values()) / 4 / 5.0e12 * 1e9)
        af = ab = 0
        if self._attn_flops is not None:
            af, ab = (int(f / tflops * 1e9) for f in self._attn_flops)
        return LayerDurations(a_fwd=a + af, a_turn=2 * a, a_bwd=2 * a + ab, f_fwd=f_fwd, f_bwd=2 * f_fwd,
                              m2n=max(1, m2n))

    # ------------------------------------------------------------ tracing
    def _xchg(self, ops, name: str, i: int):
        """Issue one P2P group on the current stream; when tracing, bracket sends with
        events on the send stream ([data ready, transfer complete])."""
        sending = any(k == "send" for k, _, _ in ops)
        ev0 = self.st.event("send", True) if (self.record_events and sending) else None
        works = self.tx.exchange(ops, direction_of(name))
        if ev0 is not None:
            for w in works:
                w.wait()
            nbytes = sum(t.numel() * t.element_size() for k, t, _ in ops if k == "send")
            self.trace.append((name, i, SEND, ev0, self.st.event("send", True), nbytes))
        return works

    def _compute(self, name: str, i: int, fn):
        """Run a compute task; with tracing, its interval starts after the task's stream waits on
        incoming data (`_mark_waited`), so time the compute engine spends waiting for a transfer
        is not counted as compute (it would hide exposed communication)."""
        ev0 = self.st.event("compute", True) if self.record_events else None
        self._start_override = None
        fn()
        if ev0 is not None:
            self.trace.append((name, i, COMPUTE, self._start_override or ev0, self.st.event("compute", True), 0))

    def _mark_waited(self):
        if self.record_events:
            self._start_override = self.st.event("compute", True)

    # ------------------------------------------------------------- A side
    def _a_pad(self, layer: int, i: int) -> list[int]:
        ev = self.pad_ready[layer][i]
        if ev is not None:
            ev.synchronize()
        return self.pad_host[layer][i].tolist()

    def _a_slices(self, pad: list[int]):
        out = []
        for f in range(self.topo.f_per_group):
            lo, hi = self.topo.expert_block(f)
            out.append((f, pad[lo], pad[hi], lo, hi))
        return out

    def set_host_io(self, xs, dys, ys, dxs) -> None:
        """Pinned host tensors per micro-batch: inputs copied in on the copy stream at
        iteration start, y / dx copied back as each micro-batch finishes (e2e mode).
        Group 0 ranks use x / dx, the last layer's group y / dy."""
        self.host_io = (xs, dys, ys, dxs)
        if len(self.x_free) != len(xs):   # first e2e iteration: wait for all earlier work
            now = self.st.event("compute")
            self.x_free, self.dy_free = [now] * len(xs), [now] * len(xs)

    @property
    def has_input(self) -> bool:
        return self.role == "A" and 0 in self.my_layers

    @property
    def has_output(self) -> bool:
        return self.role == "A" and (self.L - 1) in self.my_layers

    def _h2d_inputs(self):
        """Queue this iteration's input copies on the h2d stream. Micro-batch i's x (dy)
        overwrites its buffer as soon as the previous iteration's last reader of it, A_b of
        layer 0 (of the last layer), is done — not at the iteration boundary — so the copies
        overlap the previous iteration's tail; A_f waits on x only, the turnaround on dy."""
        xs, dys, _, _ = self.host_io
        n = len(xs)
        self.x_ready, self.dy_ready = [None] * n, [None] * n
        with self.st.ctx("h2d"):
            for i in range(n):
                if self.has_input:
                    self.st.wait("h2d", self.x_free[i])
                    self.input(i).copy_(xs[i], non_blocking=True)
                    self.x_ready[i] = self.st.event("h2d")
            for i in range(n):
                if self.has_output:
                    self.st.wait("h2d", self.dy_free[i])
                    self.out_bufs[i].dy.copy_(dys[i], non_blocking=True)
                    self.dy_ready[i] = self.st.event("h2d")

    def input(self, i: int) -> torch.Tensor:
        """A rank of group 0: micro-batch i's input activations (before attention if any)."""
        return self.xin[0][i] if self.attn is not None else self.lbufs[0][i].x

    def input_grad(self, i: int) -> torch.Tensor:
        return self.gin[0][i] if self.attn is not None else self.lbufs[0][i].dx

    def _layer_input(self, layer: int, i: int) -> torch.Tensor:
        """Where layer l's residual-stream input x_l lives on this rank."""
        return self.xin[layer][i] if self.attn is not None else self.lbufs[layer][i].x

    def _layer_input_grad(self, layer: int, i: int) -> torch.Tensor:
        return self.gin[layer][i] if self.attn is not None else self.lbufs[layer][i].dx

    def a_task(self, name: str, i: int, layer: int, accumulate: bool):
        b = self.lbufs[layer][i]
        if name == "A_f":
            if layer == 0:
                if self.host_io is not None:
                    self.st.wait("compute", self.x_ready[i])
                    self._mark_waited()
            elif self.p == 1:   # previous layer's combine writes this layer's input (residual fused)
                prev = self.lbufs[layer - 1][i]
                self._wait_works(prev, "N2M")
                self.stages.a_combine(prev)
            else:               # x_l arrived from the previous layer's A group
                self._wait_works(b, "A2A")
            if self.attn is not None:
                self.attn[layer].forward(i, self._layer_input(layer, i), b.x, self.seq_len)
            self.stages.a_dispatch(b, self.routers[layer])
            done = self.st.event("compute")
            if not self.fixed:
                with self.st.ctx("copy"):
                    self.st.wait("copy", done)
                    self.pad_host[layer][i].copy_(b.pad_off, non_blocking=self.st.cuda)
                    self.pad_ready[layer][i] = self.st.event("copy")
            b.fwd_done = done
        elif name == "A_c":     # depth > 1: this layer's combine, then x_{l+1} leaves (A2A)
            self._wait_works(b, "N2M")
            self.stages.a_combine(b)
            b.comb_done = self.st.event("compute")
        elif name == "A_t":
            self._wait_works(b, "N2M")
            if layer == self.L - 1 and self.host_io is not None:
                self.st.wait("compute", self.dy_ready[i])
                self._mark_waited()
            self.stages.a_combine(b)
            self.stages.a_combine_bwd(b)
            b.turn_done = self.st.event("compute")
        elif name == "A_cb":    # depth > 1: dy_l arrived (A2A_b); this layer's combine backward
            self._wait_works(b, "A2A_b")
            if layer == self.L - 1 and self.host_io is not None:
                self.st.wait("compute", self.dy_ready[i])
                self._mark_waited()
            self.stages.a_combine_bwd(b)
            b.turn_done = self.st.event("compute")
        elif name == "A_b":
            self._wait_works(b, "N2M_b")
            self.stages.a_backward(b, self.routers[layer], accumulate)
            if self.attn is not None:
                self.attn[layer].backward(i, b.dx, self._layer_input_grad(layer, i), accumulate)
            if layer > 0 and self.p == 1:   # this layer's dx is the previous layer's upstream gradient
                prev = self.lbufs[layer - 1][i]
                self.stages.a_combine_bwd(prev)
                prev.turn_done = self.st.event("compute")
            else:
                b.bwd_done = self.st.event("compute")
            if self.host_io is not None and layer in (0, self.L - 1):
                done = self.st.event("compute")
                if layer == self.L - 1:   # y_i was final at the turnaround
                    self.dy_free[i] = done
                    with self.st.ctx("d2h"):
                        self.st.wait("d2h", b.turn_done)
                        self.host_io[2][i].copy_(self.out_bufs[i].y, non_blocking=True)
                if layer == 0:            # x_i has no reader left this iteration; dx_i is final
                    self.x_free[i] = done
                    with self.st.ctx("d2h"):
                        self.st.wait("d2h", done)
                        self.host_io[3][i].copy_(self.input_grad(i), non_blocking=True)

    def a_comm(self, name: str, i: int, layer: int, lane: str):
        if name in ("A2A", "A2A_b"):
            return self._a2a(name, i, layer, lane)
        b = self.lbufs[layer][i]
        g = self.group
        if self.fixed:
            return self._a_comm_fixed(name, i, b, self.topo.f_rank(0, g))
        pad = self._a_pad(layer, i)
        ops = []
        if name == "M2N":
            with self.st.ctx("send"):
                self.st.wait("send", b.fwd_done)
                for f, r0, r1, lo, hi in self._a_slices(pad):
                    peer = self.topo.f_rank(f, g)
                    hdr = b.pad_off[lo:hi + 1]
                    ops += [("send", hdr, peer), ("send", b.x_perm[r0:r1], peer)]
                b.works_M2N = self._xchg(ops, name, i)
        elif name == "M2N_b":
            with self.st.ctx("send"):
                self.st.wait("send", b.turn_done)
                for f, r0, r1, lo, hi in self._a_slices(pad):
                    ops.append(("send", b.dy_perm[r0:r1], self.topo.f_rank(f, g)))
                b.works_M2N_b = self._xchg(ops, name, i)
        elif name in ("N2M", "N2M_b"):
            dst = b.y_perm if name == "N2M" else b.dx_perm
            with self.st.ctx("recv"):
                for f, r0, r1, lo, hi in self._a_slices(pad):
                    ops.append(("recv", dst[r0:r1], self.topo.f_rank(f, g)))
                setattr(b, "works_" + name, self.tx.exchange(ops, direction_of(name)))

    def _a_comm_fixed(self, name: str, i: int, b, peer: int):
        """1:1 group: whole-capacity messages (the used rows are ~all of it when one F rank
        holds every expert), header = the full padded offsets."""
        if name == "M2N":
            with self.st.ctx("send"):
                self.st.wait("send", b.fwd_done)
                b.works_M2N = self._xchg([("send", b.pad_off, peer), ("send", b.x_perm, peer)], name, i)
        elif name == "M2N_b":
            with self.st.ctx("send"):
                self.st.wait("send", b.turn_done)
                b.works_M2N_b = self._xchg([("send", b.dy_perm, peer)], name, i)
        else:
            dst = b.y_perm if name == "N2M" else b.dx_perm
            with self.st.ctx("recv"):
                setattr(b, "works_" + name, self.tx.exchange([("recv", dst, peer)], direction_of(name)))

    def _a2a(self, name: str, i: int, layer: int, lane: str):
        """depth > 1: the residual stream between consecutive layers' A groups (same
        stream member). Forward x_{l+1} = layer l's combine output; backward its gradient."""
        p, j = self.p, self.member
        if name == "A2A":       # task layer = l (the producer); consumer layer l + 1
            if lane == SEND:
                b = self.lbufs[layer][i]
                peer = self.topo.a_rank(j, (layer + 1) % p)
                with self.st.ctx("send"):
                    self.st.wait("send", b.comb_done)
                    b.works_A2A_send = self._xchg([("send", b.y, peer)], name, i)
            else:
                nb = self.lbufs[layer + 1][i]
                peer = self.topo.a_rank(j, layer % p)
                with self.st.ctx("recv"):
                    nb.works_A2A = self.tx.exchange([("recv", self._layer_input(layer + 1, i), peer)], direction_of(name))
        else:                   # "A2A_b": task layer = l - 1 (the consumer); producer layer l
            if lane == SEND:
                src = self.lbufs[layer + 1][i]
                peer = self.topo.a_rank(j, layer % p)
                with self.st.ctx("send"):
                    self.st.wait("send", src.bwd_done)
                    src.works_A2A_b_send = self._xchg([("send", self._layer_input_grad(layer + 1, i), peer)],
                                                      name, i)
            else:
                b = self.lbufs[layer][i]
                peer = self.topo.a_rank(j, (layer + 1) % p)
                with self.st.ctx("recv"):
                    b.works_A2A_b = self.tx.exchange([("recv", b.dy, peer)], direction_of(name))

    def _wait_works(self, obj, name):
        works = getattr(obj, "works_" + name, []) or []
        for w in works:
            w.wait()  # CUDA: the current (compute) stream waits on the NCCL stream
        if works:
            self._mark_waited()

    # ------------------------------------------------------------- F side
    def f_comm(self, name: str, i: int, layer: int):
        fm = self.lfmb[layer][i]
        n_a = self.n_src
        src_rank = lambda a: self.topo.a_rank(a, self.group)  # noqa: E731
        if self.fixed:
            return self._f_comm_fixed(name, i, layer, fm, src_rank(0))
        if name == "M2N":
            with self.st.ctx("recv"):
                hw = self.tx.exchange([("recv", fm.headers[a], src_rank(a)) for a in range(n_a)], AF)
                for w in hw:
                    w.wait()
            with self.st.ctx("copy"):
                self.st.wait("copy", self.st.event("recv"))
                host = torch.stack(fm.headers).to("cpu", non_blocking=False) if not self.st.cuda else None
                if self.st.cuda:
                    pinned = torch.empty(n_a, self.E_loc + 1, dtype=I32, pin_memory=True)
                    pinned.copy_(torch.stack(fm.headers), non_blocking=True)
                    ev = self.st.event("copy")
                    ev.synchronize()
                    host = pinned
            hdr = host.tolist()
            # region layout: A rank a's slice at rows [base_a, base_a + n_a_rows), back to back
            fm.slices, base, offs = [], 0, [0]
            for a in range(n_a):
                rows = hdr[a][-1] - hdr[a][0]
                fm.slices.append((base, rows))
                for e in range(self.E_loc):
                    offs.append(base + hdr[a][e + 1] - hdr[a][0])
                base += rows
            if base > self.cap_f:
                raise RuntimeError(f"F rank {self.rank}: {base} rows exceed capacity {self.cap_f}")
            go = torch.tensor(offs, dtype=I32)
            seg = torch.tensor([[i * self.cap_f + fm.slices[a][0] + hdr[a][e] - hdr[a][0]
                                 for e in range(self.E_loc + 1)] for a in range(n_a)], dtype=I32)
            if self.st.cuda:
                go, seg = go.pin_memory(), seg.pin_memory()
            fm.group_off = torch.empty(len(offs), dtype=I32, device=self.device)
            fm.group_off.copy_(go, non_blocking=self.st.cuda)
            fm.ranges = None
            if n_a > 1 and self.st.cuda and base < 512 * self.E_loc * n_a and self.E_loc * n_a <= 1024:
                # fine-grained experts (< 512 rows per expert): expert-major ranges over the A
                # ranks' slices, so one weight pass serves all of them (moe.MoELayer.merged_groups)
                st_ = [fm.slices[a][0] + hdr[a][e] - hdr[a][0] for e in range(self.E_loc) for a in range(n_a)]
                en_ = [fm.slices[a][0] + hdr[a][e + 1] - hdr[a][0] for e in range(self.E_loc) for a in range(n_a)]
                if getattr(fm, "_rg_host", None) is None:   # pinned / device staging, allocated once
                    fm._rg_host = torch.empty(2, len(st_), dtype=I32).pin_memory()
                    fm._rg_dev = torch.empty(2, len(st_), dtype=I32, device=self.device)
                # the previous iteration's copy out of the pinned buffer must be done before it
                # is rewritten (the host already synchronised on this micro-batch's header)
                if getattr(fm, "_rg_copied", None) is not None:
                    fm._rg_copied.synchronize()
                fm._rg_host[0] = torch.tensor(st_, dtype=I32)
                fm._rg_host[1] = torch.tensor(en_, dtype=I32)
                fm._rg_dev.copy_(fm._rg_host, non_blocking=True)
                fm._rg_copied = self.st.event("compute")
                fm.ranges = (fm._rg_dev[0], fm._rg_dev[1], n_a)
            self.seg_offs[layer][i * n_a:(i + 1) * n_a].copy_(seg, non_blocking=self.st.cuda)
            with self.st.ctx("recv"):
                ops = [("recv", fm.x_perm[b0:b0 + r], src_rank(a)) for a, (b0, r) in enumerate(fm.slices)]
                fm.works["M2N"] = self.tx.exchange(ops, AF)
        elif name == "M2N_b":
            with self.st.ctx("recv"):
                ops = [("recv", fm.dy_perm[b0:b0 + r], src_rank(a)) for a, (b0, r) in enumerate(fm.slices)]
                fm.works["M2N_b"] = self.tx.exchange(ops, AF)
        elif name in ("N2M", "N2M_b"):
            src = fm.y_perm if name == "N2M" else fm.dx_perm
            ready = fm.works.get(name + "_ready")
            with self.st.ctx("send"):
                self.st.wait("send", ready)
                ops = [("send", src[b0:b0 + r], src_rank(a)) for a, (b0, r) in enumerate(fm.slices)]
                fm.works[name] = self._xchg(ops, name, i)

    def _f_comm_fixed(self, name: str, i: int, layer: int, fm, peer: int):
        """1:1 group: the header lands in this micro-batch's wgrad segment row, which is
        also the GEMM group-offset array (relative rows; wgrad strides by cap_f)."""
        if name == "M2N":
            seg = self.seg_offs[layer][i]
            fm.group_off = seg
            fm.slices = [(0, self.cap_f)]
            with self.st.ctx("recv"):
                fm.works["M2N"] = self.tx.exchange([("recv", seg, peer), ("recv", fm.x_perm, peer)], AF)
        elif name == "M2N_b":
            with self.st.ctx("recv"):
                fm.works["M2N_b"] = self.tx.exchange([("recv", fm.dy_perm, peer)], AF)
        else:
            src = fm.y_perm if name == "N2M" else fm.dx_perm
            with self.st.ctx("send"):
                self.st.wait("send", fm.works.get(name + "_ready"))
                fm.works[name] = self._xchg([("send", src, peer)], name, i)

    def f_task(self, name: str, i: int, layer: int):
        fm = self.lfmb[layer][i]
        experts = self.expert_layers[layer]
        if name == "F_f":
            for w in fm.works.get("M2N", []):
                w.wait()
            self._mark_waited()
            self.stages.f_forward(fm, experts, fm.group_off, getattr(fm, "ranges", None))
            fm.works["N2M_ready"] = self.st.event("compute")
        elif name == "F_b":
            for w in fm.works.get("M2N_b", []):
                w.wait()
            self._mark_waited()
            self.stages.f_backward(fm, experts, fm.group_off, getattr(fm, "ranges", None))
            fm.works["N2M_b_ready"] = self.st.event("compute")

    # ------------------------------------------------------------ iteration
    @property
    def capturable(self) -> bool:
        """The iteration has no host synchronisation (1 A + 1 F rank per pipeline group:
        fixed-size messages, device-side offsets) and no host I/O or tracing."""
        return self.st.cuda and self.fixed and self.host_io is None and not self.record_events

    def capture(self, accumulate: bool = False):
        """Record one iteration — kernels, the NCCL sends/receives on their streams, the W
        pass and the dW_g all-reduce — as a CUDA graph (PAPER.md:266's non-blocking streams
        with the host out of the loop); `graph.replay()` on the caller's stream runs it.
        Every rank of the job captures once, in the same order, after the process groups
        exist (one eager warm-up iteration initialises NCCL and the kernels). Drop the
        graph before destroying the process group: a live graph holding NCCL work makes
        the teardown hang."""
        if not self.capturable:
            raise RuntimeError("AF-Pipe iteration capture needs the fixed-size (1A:1F per group) exchange, "
                               "no host I/O and no event tracing")
        self.run_iteration(accumulate)
        torch.cuda.synchronize(self.device)
        outer = self.st.compute
        side = torch.cuda.Stream(self.device)   # the legacy default stream cannot be captured
        side.wait_stream(outer)
        g = torch.cuda.CUDAGraph()
        self.st.compute = side
        c0 = _lib.launch_count() if self.st.cuda else 0
        try:
            with torch.cuda.graph(g, stream=side):
                self.run_iteration(accumulate)
        finally:
            self.st.compute = outer
        self.graph_launches = _lib.launch_count() - c0   # dm kernels per replay
        outer.wait_stream(side)
        return g

    def run_iteration(self, accumulate: bool = False) -> None:
        # comm/copy streams must not touch this iteration's buffers before the
        # compute stream is done with the previous iteration's uses of them
        start = self.st.event("compute")
        for which in ("send", "recv", "copy", "d2h"):
            self.st.wait(which, start)
        self.trace = []
        self.t0 = self.st.event("compute", self.record_events)
        if self.host_io is not None and self.role == "A":
            self._h2d_inputs()
        for t in self.order:
            name, i, layer = t.name, t.microbatch, t.layer
            if self.role == "A":
                if t.lane == COMPUTE:
                    self._compute(name, i, lambda: self.a_task(name, i, layer, accumulate or i > 0))
                else:
                    self.a_comm(name, i, layer, t.lane)
            else:
                if t.lane == COMPUTE:
                    self._compute(name, i, lambda: self.f_task(name, i, layer))
                else:
                    self.f_comm(name, i, layer)
        if self.role == "F":
            def w_pass():
                for l in self.my_layers:
                    self.stages.f_wgrad(self.slabs[l], self.expert_layers[l], self.seg_offs[l], accumulate,
                                        self.cap_f if self.fixed else 0)
            self._compute("W", -1, w_pass)
            for l in self.my_layers:
                for fm in self.lfmb[l]:
                    for k in ("N2M", "N2M_b"):
                        for w in fm.works.get(k, []):
                            w.wait()
        else:
            for l in self.my_layers:
                for b in self.lbufs[l]:
                    for k in ("M2N", "M2N_b", "A2A_send", "A2A_b_send"):
                        self._wait_works(b, k)
            if self.host_io is not None and self.st.cuda:   # the iteration ends with y / dx on the host
                self.st.compute.wait_stream(self.st.d2h)
            if self.a_group is not None and self.topo.a_per_group > 1:
                for l in self.my_layers:
                    self.tx.all_reduce(self.routers[l].dwg, self.a_group)
                for blk in (self.attn or {}).values():
                    for g in blk.grads():
                        self.tx.all_reduce(g, self.a_group)

    def init_groups(self):
        """Set up the transport and create the per-pipeline-group
        A communicators (collective: every rank calls new_group for every group, in the
        same order)."""
        self.tx.setup(self.topo.world)
        for g in range(self.topo.depth):
            ranks = [self.topo.a_rank(j, g) for j in range(self.topo.a_per_group)]
            pg = self.tx.new_group(ranks)
            if self.role == "A" and self.group == g:
                self.a_group = pg


def trace_intervals(rank: "AFPipeRank") -> list[tuple[str, int, str, float, float, int]]:
    """(task, micro-batch, lane, start_ms, end_ms, bytes) relative to the iteration's t0
    event (call after the iteration's work has completed)."""
    out = []
    for name, i, lane, e0, e1, nbytes in rank.trace:
        out.append((name, i, lane, rank.t0.elapsed_time(e0), rank.t0.elapsed_time(e1), nbytes))
    return out


def env_rank() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))
