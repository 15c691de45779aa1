"""AF-Pipe issue-order planner and the measured-trace metrics.

The runtime executes the AF-Pipe DAG of the reference on CUDA streams; this
module decides *the order* in which each rank issues its work and evaluates
measured timelines with the reference's metric definitions.

DAG (reference _build_afpipe, /root/reference/pkg/src/afpipe/taskgraph.py:307-356):
per micro-batch the chain A_{l mod p} fwd -> M2N -> F_{l mod p} fwd -> N2M ->
A_{(l+1) mod p} ... then the reversed chain with gradients; exchanges are
send/recv twins that occupy both endpoints' comm lanes over the same interval
(taskgraph.py:204-242). 1F1B credits: A_g = 2L-2g, F_g = 2L-2g-1 (:316-321).

Policy (reference simulate, sim.py:101-216): repeatedly commit the ready unit
with the smallest (earliest feasible start, 1F1B preference, micro-batch,
virtual index, A-before-F, owner, lane, id). Integer nanoseconds throughout.
The resulting per-(owner, lane) order is what each rank issues to its
compute / send / recv streams; tests/golden/afpipe_orders.json pins it
against the reference simulator.
"""

from __future__ import annotations

from dataclasses import dataclass, field

COMPUTE, SEND, RECV = "compute", "comm.send", "comm.recv"
FWD, BWD = "fwd", "bwd"


@dataclass
class PlanTask:
    id: int
    kind: str               # FwdCompute | BwdCompute | M2NSend | M2NRecv
    owner: str              # "A{g}" / "F{g}"
    lane: str               # compute | comm.send | comm.recv
    duration_ns: int
    deps: tuple[int, ...]
    microbatch: int
    layer: int
    virtual_index: int
    component: str | None   # "A" / "F" for compute tasks
    direction: str          # fwd | bwd
    twin: int | None = None
    start_ns: int = -1

    @property
    def end_ns(self) -> int:
        return self.start_ns + self.duration_ns

    @property
    def is_compute(self) -> bool:
        return self.lane == COMPUTE

    @property
    def tag(self) -> str:
        """Short label: F/B (compute fwd/bwd), s/r (send/recv) + mb.layer."""
        if self.is_compute:
            return f"{'F' if self.direction == FWD else 'B'}{self.microbatch}.L{self.layer}"
        return f"{'s' if self.lane == SEND else 'r'}{self.microbatch}.L{self.layer}{'b' if self.direction == BWD else ''}"


@dataclass
class Plan:
    tasks: list[PlanTask]
    credits: dict[str, int]
    iteration_ns: int = 0
    lanes: dict[tuple[str, str], list[int]] = field(default_factory=dict)

    def order(self, owner: str, lane: str) -> list[PlanTask]:
        return [self.tasks[i] for i in self.lanes.get((owner, lane), [])]


@dataclass(frozen=True)
class StageDurations:
    """Per-visit durations in ns (bwd defaults to 2x fwd, reference visit_times)."""

    attn_fwd: int
    ffn_fwd: int
    m2n: int
    attn_bwd: int | None = None
    ffn_bwd: int | None = None

    def a_bwd(self) -> int:
        return self.attn_bwd if self.attn_bwd is not None else 2 * self.attn_fwd

    def f_bwd(self) -> int:
        return self.ffn_bwd if self.ffn_bwd is not None else 2 * self.ffn_fwd


def build_dag(layers: int, depth: int, microbatches: int, d: StageDurations) -> Plan:
    tasks: list[PlanTask] = []

    def new(kind, owner, lane, dur, deps, mb, layer, comp, direction, twin=None):
        t = PlanTask(len(tasks), kind, owner, lane, dur, tuple(deps), mb, layer, layer // depth, comp,
                     direction, twin)
        tasks.append(t)
        return t.id

    def exchange(src, dst, dep, mb, layer, direction):
        s = new("M2NSend", src, SEND, d.m2n, (dep,), mb, layer, None, direction)
        r = new("M2NRecv", dst, RECV, d.m2n, (dep,), mb, layer, None, direction)
        tasks[s].twin, tasks[r].twin = r, s
        return r

    credits = {}
    for g in range(depth):
        credits[f"A{g}"] = max(1, 2 * layers - 2 * g)
        credits[f"F{g}"] = max(1, 2 * layers - 2 * g - 1)

    for mb in range(microbatches):
        upstream = None
        for layer in range(layers):
            g = layer % depth
            a = new("FwdCompute", f"A{g}", COMPUTE, d.attn_fwd, () if upstream is None else (upstream,),
                    mb, layer, "A", FWD)
            r = exchange(f"A{g}", f"F{g}", a, mb, layer, FWD)
            f = new("FwdCompute", f"F{g}", COMPUTE, d.ffn_fwd, (r,), mb, layer, "F", FWD)
            upstream = exchange(f"F{g}", f"A{(layer + 1) % depth}", f, mb, layer, FWD) if layer + 1 < layers else f
        for layer in reversed(range(layers)):
            g = layer % depth
            fb = new("BwdCompute", f"F{g}", COMPUTE, d.f_bwd(), (upstream,), mb, layer, "F", BWD)
            r = exchange(f"F{g}", f"A{g}", fb, mb, layer, BWD)
            ab = new("BwdCompute", f"A{g}", COMPUTE, d.a_bwd(), (r,), mb, layer, "A", BWD)
            if layer > 0:
                upstream = exchange(f"A{g}", f"F{(layer - 1) % depth}", ab, mb, layer, BWD)
    return Plan(tasks, credits)


_COMP_RANK = {"A": 0, "F": 1, None: 2}


def schedule(plan: Plan) -> Plan:
    """Greedy list schedule; fills start_ns, per-lane orders and iteration_ns."""
    tasks = plan.tasks
    if not tasks:
        return plan
    # schedulable units: lone tasks and send/recv pairs (keyed by the send side)
    unit_of = {}
    unit_deps: dict[int, set[int]] = {}
    for t in tasks:
        if t.twin is not None and t.lane == RECV:
            unit_of[t.id] = t.twin
            continue
        unit_of[t.id] = t.id
        deps = set(t.deps)
        if t.twin is not None:
            deps |= set(tasks[t.twin].deps)
        unit_deps[t.id] = deps
    waiting = {u: len(ds) for u, ds in unit_deps.items()}
    children: dict[int, list[int]] = {t.id: [] for t in tasks}
    for u, ds in unit_deps.items():
        for dep in ds:
            children[dep].append(u)
    ready = sorted(u for u, n in waiting.items() if n == 0)
    busy_until: dict[tuple[str, str], int] = {}
    started = {"fwd": {}, "bwd": {}}
    done_at: dict[int, int] = {}
    lanes: dict[tuple[str, str], list[int]] = {}

    def members(u):
        t = tasks[u]
        return (t,) if t.twin is None else (t, tasks[t.twin])

    def feasible_start(u):
        at = max((done_at[dep] for dep in unit_deps[u]), default=0)
        for m in members(u):
            at = max(at, busy_until.get((m.owner, m.lane), 0))
        return at

    def preference(t: PlanTask):
        if not t.is_compute:
            return 0
        inflight = started["fwd"].get(t.owner, 0) - started["bwd"].get(t.owner, 0)
        want_bwd = inflight >= plan.credits.get(t.owner, 1)
        return 0 if (t.direction == BWD) == want_bwd else 1

    while ready:
        scored = [((feasible_start(u), preference(tasks[u]), tasks[u].microbatch, tasks[u].virtual_index,
                    _COMP_RANK[tasks[u].component], tasks[u].owner, tasks[u].lane, u), u) for u in ready]
        key, u = min(scored)
        ready.remove(u)
        for m in members(u):
            m.start_ns = key[0]
            busy_until[(m.owner, m.lane)] = m.end_ns
            done_at[m.id] = m.end_ns
            lanes.setdefault((m.owner, m.lane), []).append(m.id)
            if m.is_compute:
                bucket = started["bwd" if m.direction == BWD else "fwd"]
                bucket[m.owner] = bucket.get(m.owner, 0) + 1
            for c in children[m.id]:
                waiting[c] -= 1
                if waiting[c] == 0:
                    ready.append(c)
    plan.lanes = lanes
    plan.iteration_ns = max(t.end_ns for t in tasks)
    return plan


def plan_afpipe(layers: int, depth: int, microbatches: int, d: StageDurations) -> Plan:
    return schedule(build_dag(layers, depth, microbatches, d))


# Task names of the single-MoE-layer runtime chain: with the
# expert block sharded over several F ranks a token's k outputs live on different
# ranks, so the combine (and the loss turnaround) runs on the A side. Per micro-batch:
#   A_f -> M2N -> F_f -> N2M -> A_t -> M2N_b -> F_b -> N2M_b -> A_b
# i.e. the reference's interior-layer pattern (taskgraph.py:335-339, :352-356)
# with the A visit split in dispatch (A_f), turnaround (A_t) and dispatch-bwd (A_b).
@dataclass(frozen=True)
class LayerDurations:
    a_fwd: int       # dispatch (routing + permute)
    a_turn: int      # combine fwd + loss turnaround + combine bwd
    a_bwd: int       # permute bwd + router grads
    f_fwd: int       # expert GEMMs fwd
    f_bwd: int       # expert dgrad GEMMs
    m2n: int         # one exchange in either direction


def build_layer_dag(microbatches: int, d: LayerDurations, a_credit: int = 2, f_credit: int = 2,
                    layers: int = 1, depth: int = 1) -> Plan:
    """Runtime chain of a stack of `layers` residual MoE blocks, layer l on A group and
    F group l mod `depth` (reference taskgraph.py:307-356 with the loss turnaround on the
    A side; virtual_stages = ceil(layers / depth)). Per micro-batch, depth 1:

        A_f[0] M2N[0] F_f[0] N2M[0] A_f[1] ... F_f[L-1] N2M[L-1] A_t
        M2N_b[L-1] F_b[L-1] N2M_b[L-1] A_b[L-1] M2N_b[L-2] ... A_b[0]

    where A_f[l>0] is layer l-1's combine fused with layer l's dispatch and A_b[l>0]
    includes layer l-1's combine backward (same rank). With depth > 1 consecutive layers
    live on different A groups: layer l's combine (A_c) stays on the rank holding its
    routing, the residual stream x_{l+1} moves A_g -> A_g' (A2A), and backward the
    gradient of x_l returns A_g' -> A_g (A2A_b) ahead of layer l-1's combine backward
    (A_cb). layers=1 is the single-layer chain."""
    tasks: list[PlanTask] = []
    p = depth

    def new(kind, owner, lane, dur, deps, mb, layer, comp, direction, name):
        t = PlanTask(len(tasks), kind, owner, lane, dur, tuple(deps), mb, layer, layer // p, comp, direction)
        t.name = name  # type: ignore[attr-defined]
        tasks.append(t)
        return t.id

    def exchange(src, dst, dep, mb, layer, direction, name, dur=None):
        s = new("M2NSend", src, SEND, d.m2n if dur is None else dur, (dep,), mb, layer, None, direction, name)
        r = new("M2NRecv", dst, RECV, d.m2n if dur is None else dur, (dep,), mb, layer, None, direction, name)
        tasks[s].twin, tasks[r].twin = r, s
        return r

    A = lambda l: f"A{l % p}"  # noqa: E731
    F = lambda l: f"F{l % p}"  # noqa: E731
    a2a = max(1, d.m2n // 2)   # T x H residual stream vs T x k x H routed rows
    for mb in range(microbatches):
        r = None
        for layer in range(layers):
            fused = layer > 0 and p == 1
            dur = d.a_fwd + (d.a_turn // 2 if fused else 0)
            af = new("FwdCompute", A(layer), COMPUTE, dur, () if r is None else (r,), mb, layer, "A", FWD, "A_f")
            r = exchange(A(layer), F(layer), af, mb, layer, FWD, "M2N")
            ff = new("FwdCompute", F(layer), COMPUTE, d.f_fwd, (r,), mb, layer, "F", FWD, "F_f")
            r = exchange(F(layer), A(layer), ff, mb, layer, FWD, "N2M")
            if p > 1 and layer < layers - 1:
                ac = new("FwdCompute", A(layer), COMPUTE, d.a_turn // 2, (r,), mb, layer, "A", FWD, "A_c")
                r = exchange(A(layer), A(layer + 1), ac, mb, layer, FWD, "A2A", a2a)
        top = layers - 1
        at = new("BwdCompute", A(top), COMPUTE, d.a_turn, (r,), mb, top, "A", BWD, "A_t")
        r = exchange(A(top), F(top), at, mb, top, BWD, "M2N_b")
        for layer in reversed(range(layers)):
            fb = new("BwdCompute", F(layer), COMPUTE, d.f_bwd, (r,), mb, layer, "F", BWD, "F_b")
            r = exchange(F(layer), A(layer), fb, mb, layer, BWD, "N2M_b")
            fused = layer > 0 and p == 1
            dur = d.a_bwd + (d.a_turn // 2 if fused else 0)
            ab = new("BwdCompute", A(layer), COMPUTE, dur, (r,), mb, layer, "A", BWD, "A_b")
            if layer > 0:
                if p == 1:
                    r = exchange(A(layer), F(layer - 1), ab, mb, layer - 1, BWD, "M2N_b")
                else:
                    r = exchange(A(layer), A(layer - 1), ab, mb, layer - 1, BWD, "A2A_b", a2a)
                    acb = new("BwdCompute", A(layer - 1), COMPUTE, d.a_turn // 2, (r,), mb, layer - 1, "A", BWD,
                              "A_cb")
                    r = exchange(A(layer - 1), F(layer - 1), acb, mb, layer - 1, BWD, "M2N_b")
    credits = {}
    for g in range(p):
        credits[f"A{g}"] = a_credit
        credits[f"F{g}"] = f_credit
    return Plan(tasks, credits)


def plan_layer(microbatches: int, d: LayerDurations, a_credit: int = 2, f_credit: int = 2,
               layers: int = 1, depth: int = 1) -> Plan:
    """Scheduled runtime chain; every rank issues its tasks in planned-start order,
    which keeps the per-pair send/recv order identical on both ends (twins share a start).
    Credits scale with the virtual stages as in the reference (taskgraph.py:316-321)."""
    v = -(-layers // depth)
    return schedule(build_layer_dag(microbatches, d, a_credit * v, f_credit * v, layers, depth))


def issue_order(plan: Plan, owner: str) -> list[PlanTask]:
    """The owner's tasks across all its lanes, by planned start (then compute < send < recv, id)."""
    lane_rank = {COMPUTE: 0, SEND: 1, RECV: 2}
    mine = [t for t in plan.tasks if t.owner == owner]
    return sorted(mine, key=lambda t: (t.start_ns, lane_rank[t.lane], t.id))


# ----------------------------------------------------------- trace metrics
def _union(intervals):
    out: list[list[int]] = []
    for s, e in sorted(intervals):
        if out and s <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([s, e])
    return out


def _uncovered(a, b) -> int:
    """Length of union(a) not covered by union(b)."""
    a, b = _union(a), _union(b)
    total, j = 0, 0
    for s, e in a:
        cur = s
        while cur < e:
            while j < len(b) and b[j][1] <= cur:
                j += 1
            if j == len(b) or b[j][0] >= e:
                total += e - cur
                break
            if b[j][0] > cur:
                total += b[j][0] - cur
            cur = min(b[j][1], e)
    return total


def exposed_comm_global(events) -> int:
    """Reference definition (sim.py:273-299): ns during which communication runs
    while every compute engine idles. events: iterable of (start, end, is_compute)."""
    ev = [e for e in events if e[1] > e[0]]
    return _uncovered([(s, e) for s, e, c in ev if not c], [(s, e) for s, e, c in ev if c])


def exposed_comm_per_rank(events_by_rank: dict) -> dict:
    """Strict definition: per rank, comm time not covered by that rank's own compute."""
    return {r: exposed_comm_global(ev) for r, ev in events_by_rank.items()}
