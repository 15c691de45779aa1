"""Inter-group transport of the AF-Pipe runtime: the M2N / N2M exchanges between
attention (A) and FFN (F) ranks, the A-group gradient all-reduce, and group creation.

Reference semantics: every transfer is a send/recv twin occupying both endpoints
(`_Builder.add_transfer`, /root/reference/pkg/src/afpipe/taskgraph.py:204-242) on
full-duplex lanes — one send and one receive lane per worker (sim.py:3-7,
SPEC.md:362) — and the paper runs them on dedicated send/recv process groups
(PAPER.md:266). Two implementations share one interface:

* `NcclTransport` (the product, one process per GPU): NCCL point-to-point over
  NVLink 5 / NVSwitch through torch.distributed, both directions on one communicator.
  (One communicator per direction was tried: it deadlocked the Mixtral-size 1:1
  exchange, eager and graph-captured alike, and slowed the 2:2 / 1:3 F ranks by
  ~15%; `scripts/diag_n2.sh`. NCCL progresses one communicator's operations in issue
  order, which is the order both ends agree on.)
* `LoopbackTransport` (one process, one GPU): every rank is a host thread with its
  own CUDA streams; a send and its matching receive meet in a `LoopbackHub`, which
  issues the device-to-device copy on a per-(src, dst, direction) lane stream once
  both sides have posted, ordered after the sender's data-ready event and the
  receiver's buffer-free event. Works complete when that copy does. This runs the
  whole multi-rank AF-Pipe runtime — real kernels, streams and events — on a
  single B200 (SURVEY.md §4 implication 4), and on CPU tensors for the CPU tests.

Message matching is FIFO per (src, dst, direction), the NCCL rule, so both
transports need the same thing from the runtime: identical per-pair issue order
on both ends (AFPipeRank issues in the planned order of afpipe.plan_layer).
"""

from __future__ import annotations

import threading
from collections import defaultdict, deque
from concurrent.futures import ThreadPoolExecutor

import torch
import torch.distributed as dist

AF, FA = "af", "fa"   # A -> F and F -> A lanes


def direction_of(task: str) -> str:
    """Lane of a transfer task: N2M / N2M_b and the backward residual hop go F->A
    (resp. A_{g+1} -> A_g), everything else A->F."""
    return FA if task.startswith("N2M") or task == "A2A_b" else AF


# ------------------------------------------------------------------- NCCL
class NcclTransport:
    """torch.distributed P2P (NCCL on CUDA tensors, gloo in the CPU tests)."""

    def __init__(self):
        self._fast: dict[int, object] = {}

    def setup(self, world: int) -> None:
        """Nothing to create: every exchange runs on the default process group."""

    def new_group(self, ranks):
        return dist.new_group(list(ranks))

    def all_reduce(self, t: torch.Tensor, group) -> None:
        dist.all_reduce(t, group=group)

    def _coalescing_pg(self, pg, dev):
        key = id(pg)
        if key not in self._fast:
            ok = hasattr(pg, "_start_coalescing") and pg._get_backend(dev).supports_coalescing
            self._fast[key] = pg if ok else False
        return self._fast[key]

    def exchange(self, ops: list[tuple[str, torch.Tensor, int]], direction: str = AF):
        """One coalesced group of P2P ops on the current stream; returns the works.

        On CUDA tensors the group is issued straight on the default ProcessGroup
        (_start_coalescing / send / recv / _end_coalescing — what batch_isend_irecv does,
        without its per-op Python validation, which dominated small-shape iterations);
        other backends use the public batch_isend_irecv."""
        ops = [o for o in ops if o[1].numel() > 0]
        if not ops:
            return []
        group = None
        dev = ops[0][1].device
        if dev.type == "cuda":
            pg = dist.distributed_c10d._get_default_group()
            fast = self._coalescing_pg(pg, dev)
            if fast:
                fast._start_coalescing(dev)
                for k, t, peer in ops:   # groups span all ranks: group rank == global rank
                    if k == "send":
                        fast.send([t], peer, 0)
                    else:
                        fast.recv([t], peer, 0)
                return [fast._end_coalescing(dev)]
        p2p = [dist.P2POp(dist.isend if k == "send" else dist.irecv, t, peer, group) for k, t, peer in ops]
        return dist.batch_isend_irecv(p2p)


# ---------------------------------------------------------------- loopback
class LoopbackTimeout(RuntimeError):
    """A loopback work waited longer than the hub's timeout: a send/recv pair never met
    (mismatched issue orders — what would hang NCCL)."""


class _Post:
    __slots__ = ("t", "ev", "done", "stream")

    def __init__(self, t: torch.Tensor, ev, stream):
        self.t, self.ev, self.stream, self.done = t, ev, stream, None


class _Work:
    __slots__ = ("hub", "post")

    def __init__(self, hub: "LoopbackHub", post: _Post):
        self.hub, self.post = hub, post

    def wait(self) -> bool:
        """Host-block until the transfer has been issued, then order the current stream
        after its completion (NCCL's work.wait() is the same stream wait)."""
        self.hub._await(self.post)
        if self.post.done is not True:
            torch.cuda.current_stream(self.post.t.device).wait_event(self.post.done)
        return True

    def is_completed(self) -> bool:
        return self.post.done is not None


class LoopbackHub:
    """Meeting point of the ranks of one LoopbackWorld (one device)."""

    def __init__(self, device, timeout_s: float = 300.0):
        self.device = torch.device(device)
        self.cuda = self.device.type == "cuda"
        self.cv = threading.Condition()
        self.timeout_s = timeout_s
        self.sends: dict[tuple, deque] = defaultdict(deque)
        self.recvs: dict[tuple, deque] = defaultdict(deque)
        self.lanes: dict[tuple, object] = {}
        self.reductions: dict[tuple, list] = {}
        self.bytes_moved = 0

    def _lane(self, key):
        if key not in self.lanes:
            self.lanes[key] = torch.cuda.Stream(self.device) if self.cuda else None
        return self.lanes[key]

    def _await(self, post: _Post) -> None:
        with self.cv:
            if not self.cv.wait_for(lambda: post.done is not None, timeout=self.timeout_s):
                raise LoopbackTimeout(f"loopback transfer of {tuple(post.t.shape)} never matched")

    def _transfer(self, key, src: _Post, dst: _Post) -> None:
        """Both ends posted (called under the lock): copy src -> dst on the lane stream."""
        if src.t.numel() != dst.t.numel() or src.t.dtype != dst.t.dtype:
            err = RuntimeError(f"loopback {key}: send {tuple(src.t.shape)}/{src.t.dtype} does not match "
                               f"recv {tuple(dst.t.shape)}/{dst.t.dtype}")
            src.done = dst.done = True
            raise err
        if self.cuda:
            lane = self._lane(key)
            lane.wait_event(src.ev)
            lane.wait_event(dst.ev)
            with torch.cuda.stream(lane):
                dst.t.view(-1).copy_(src.t.reshape(-1), non_blocking=True)
            src.t.record_stream(lane)
            dst.t.record_stream(lane)
            done = torch.cuda.Event()
            done.record(lane)
        else:
            dst.t.view(-1).copy_(src.t.reshape(-1))
            done = True
        self.bytes_moved += src.t.numel() * src.t.element_size()
        src.done = dst.done = done
        self.cv.notify_all()

    def post(self, kind: str, t: torch.Tensor, me: int, peer: int, direction: str) -> _Work:
        ev = None
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
        p = _Post(t, ev, None)
        key = (me, peer, direction) if kind == "send" else (peer, me, direction)
        with self.cv:
            mine, other = (self.sends, self.recvs) if kind == "send" else (self.recvs, self.sends)
            if other[key]:
                q = other[key].popleft()
                src, dst = (p, q) if kind == "send" else (q, p)
                self._transfer(key, src, dst)
            else:
                mine[key].append(p)
        return _Work(self, p)

    def all_reduce(self, t: torch.Tensor, group: tuple, me: int, seq: int) -> _Work:
        """Sum over the group in a fixed (rank) order — deterministic — written back to
        every member's tensor by the last member to arrive."""
        ev = None
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
        p = _Post(t, ev, None)
        key = ("all_reduce", group, seq)
        with self.cv:
            parts = self.reductions.setdefault(key, [])
            parts.append((me, p))
            if len(parts) == len(group):
                del self.reductions[key]
                parts.sort(key=lambda mp: mp[0])
                posts = [q for _, q in parts]
                if self.cuda:
                    lane = self._lane(("all_reduce", group))
                    for q in posts:
                        lane.wait_event(q.ev)
                    with torch.cuda.stream(lane):
                        acc = posts[0].t.clone()
                        for q in posts[1:]:
                            acc += q.t
                        for q in posts:
                            q.t.copy_(acc)
                    done = torch.cuda.Event()
                    done.record(lane)
                else:
                    acc = posts[0].t.clone()
                    for q in posts[1:]:
                        acc += q.t
                    for q in posts:
                        q.t.copy_(acc)
                    done = True
                for q in posts:
                    q.done = done
                self.cv.notify_all()
        return _Work(self, p)


class LoopbackTransport:
    """The transport of one rank of a LoopbackWorld."""

    def __init__(self, hub: LoopbackHub, rank: int):
        self.hub, self.rank = hub, rank
        self._seq: dict[tuple, int] = defaultdict(int)

    def setup(self, world: int) -> None:
        pass

    def new_group(self, ranks):
        return tuple(sorted(ranks))

    def exchange(self, ops, direction: str = AF):
        return [self.hub.post(k, t, self.rank, peer, direction) for k, t, peer in ops if t.numel() > 0]

    def all_reduce(self, t: torch.Tensor, group) -> None:
        group = tuple(group)
        seq = self._seq[group]
        self._seq[group] += 1
        self.hub.all_reduce(t, group, self.rank, seq).wait()


class LoopbackWorld:
    """`world` ranks in one process on one device: rank r runs in its own host thread
    (a persistent single-worker pool) whose current CUDA stream is a fresh stream, so
    ranks get independent compute/send/recv streams exactly as separate processes
    would, and talk through one LoopbackHub.

        world = LoopbackWorld(4, "cuda:0")
        ranks = world.run(lambda r, tx: AFPipeRank(..., rank=r, transport=tx))
        world.run(lambda r, tx: (ranks[r].init_groups(), ranks[r].run_iteration()))
    """

    def __init__(self, world: int, device, timeout_s: float = 300.0):
        self.world = world
        self.device = torch.device(device)
        self.hub = LoopbackHub(self.device, timeout_s)
        self.transports = [LoopbackTransport(self.hub, r) for r in range(world)]
        self._pools = [ThreadPoolExecutor(max_workers=1, initializer=self._init_thread) for _ in range(world)]

    def _init_thread(self):
        if self.device.type == "cuda":
            torch.cuda.set_device(self.device)
            torch.cuda.set_stream(torch.cuda.Stream(self.device))

    def run(self, fn) -> list:
        """fn(rank, transport) on every rank concurrently; returns the per-rank results
        (re-raising the first failure after every rank has finished or timed out)."""
        futs = [p.submit(fn, r, self.transports[r]) for r, p in enumerate(self._pools)]
        out, err = [], None
        for f in futs:
            try:
                out.append(f.result())
            except BaseException as e:  # noqa: BLE001 - re-raised below
                out.append(None)
                err = err or e
        if err is not None:
            raise err
        return out

    def synchronize(self) -> None:
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)

    def close(self) -> None:
        for p in self._pools:
            p.shutdown(wait=True)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
        return False
