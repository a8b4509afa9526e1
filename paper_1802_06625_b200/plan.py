"""Admission and launch planning for the device executor.

The threaded reference executor (runtime.py:118-193) resolves every dynamic
port's rate per firing on the host (Eq. 1, runtime.py:107-116).  Here the
same information is computed once per graph as *conditions*: every
(control output port, element) pair of the control table (model.py:137-163)
is one boolean sequence over iterations, and every actor and FIFO is gated by
exactly one condition or by none ("always").  Propagation goes

    DRP of a dynamic actor  ->  its control-table entry
    static actor            <-  the condition of any FIFO touching it
    FIFO                    =   condition of its producer port
                            =   condition of its consumer port   (Eq. 1)

Admission first runs the reference's decidability analysis (admission.py:
the five design rules, DPG identification and validation, period schedules
and bounds, analysis.py:414-460) and raises InconsistentGraph exactly when the
reference does.  A graph the analysis accepts but whose FIFO ends carry
different conditions (an always-active actor feeding a gated subchain, as in
fixtures.encapsulated_pass) is outside the executor's class and raises
UnsupportedGraph.  The executor covers acyclic graphs whose dynamic regions
are not nested, with configuration actors that have no data inputs and
initial delay tokens only on aligned, always-active channels between device
actors (every shipped app: the motion app's one-frame delay is such a
channel); anything else raises UnsupportedGraph rather than running
incorrectly.

Per iteration n every "always" actor fires once and every gated actor fires
iff its condition is true at n, which is the firing sequence both reference
engines produce (interp.py:126-148 is the oracle's version of the rule).
Buffer bounds are the analysis' beta = delay + r + (C-1)*r for a rate-r FIFO
at the caller's c_factor (compute_bounds, analysis.py:398-411).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import admission
from .admission import AnalysisReport
from .behaviors import ActorBehavior, DeviceBehavior
from .errors import InconsistentGraph, InvalidParams, UnsupportedGraph
from .graph import (CONFIG, CONTROL_IN, CONTROL_OUT, DRP, DYNAMIC, Graph, PortRef)

ALWAYS = -1


@dataclass(frozen=True)
class Condition:
    ctl: PortRef        # control output port of a configuration actor
    element: int        # 1-based element of the control value


@dataclass
class FilterBankGroup:
    """route -> K x fir_branch -> branch_sum region fired as one kernel."""

    router: str
    combiner: str
    branches: list[str]          # fir_branch actors in the combiner's sorted port order
    internal_fifos: set[str]


@dataclass
class ExecPlan:
    graph: Graph
    conds: list[Condition]
    actor_cond: dict[str, int]
    fifo_cond: dict[str, int]
    order: list[str]                       # topological order over data FIFOs
    roles: dict[str, str]                  # source | config | dynamic | device | sink
    control_fifos: list[str]
    data_fifos: list[str]
    eq1_ports: list[tuple[str, str, int, int]]   # (actor, port, own_cond, moved_cond)
    admission: AnalysisReport
    epoch_cap: int | None = None           # max iterations per epoch (delayed cycles)
    extra: dict[str, int | None] = field(default_factory=dict)   # drain firings per actor
    loose: set[str] = field(default_factory=set)   # delayed channels inside cycles


def admit(g: Graph, c_factor: int = 3) -> ExecPlan:
    """Build the condition plan or raise InconsistentGraph (the reference's
    analysis rejects the graph) / UnsupportedGraph (consistent, but outside
    the executor's class) / InvalidParams (c_factor < 2, fifos.py:80-81)."""
    if c_factor < 2:
        raise InvalidParams(f"buffering factor must be >= 2, got {c_factor}")
    report = admission.analyze(g, c_factor)
    if not report.consistent:
        raise InconsistentGraph(report)
    unsupported: list[str] = []

    # every dynamic port needs a table entry (analysis.py:420-427)
    conds: list[Condition] = []
    cond_index: dict[Condition, int] = {}

    def cond_of(ctl: PortRef, element: int) -> int:
        c = Condition(ctl, element)
        if c not in cond_index:
            cond_index[c] = len(conds)
            conds.append(c)
        return cond_index[c]

    port_cond: dict[PortRef, int] = {}
    for a in g.actors:
        if a.kind == DYNAMIC:
            for p in a.drps:
                ref = PortRef(a.id, p.id)
                port_cond[ref] = cond_of(*g.control_lookup(ref))

    roles: dict[str, str] = {}
    actor_cond: dict[str, int | None] = {}
    for a in g.actors:
        data_in = [p for p in a.input_ports if p.kind != CONTROL_IN]
        data_out = [p for p in a.output_ports if p.kind != CONTROL_OUT]
        if a.kind == CONFIG:
            if data_in:
                unsupported.append(f"configuration actor {a.id} reads data ports; control "
                                   "tokens must be computable ahead of the data")
            roles[a.id] = "config"
            actor_cond[a.id] = ALWAYS
        elif a.kind == DYNAMIC:
            roles[a.id] = "dynamic"
            actor_cond[a.id] = ALWAYS
        elif not data_in:
            roles[a.id] = "source"
            actor_cond[a.id] = ALWAYS
        elif not data_out:
            roles[a.id] = "sink"
            actor_cond[a.id] = None
        else:
            roles[a.id] = "device"
            actor_cond[a.id] = None

    control_fifos = [f.id for f in g.fifos if g.actor(f.src.actor).port(f.src.port).kind
                     == CONTROL_OUT]
    data_fifos = [f.id for f in g.fifos if f.id not in set(control_fifos)]

    # control channels: rule 2 (checked by the analysis) leaves one delay per
    # control port; initial control tokens are outside the executor's class
    for fid in control_fifos:
        f = g.fifo(fid)
        if f.delay:
            unsupported.append(f"control channel {fid} carries initial delay tokens")

    # propagate conditions through static actors
    def pc(ref: PortRef) -> int | None:
        if ref in port_cond:
            return port_cond[ref]
        return actor_cond[ref.actor]

    changed = True
    while changed:
        changed = False
        for fid in data_fifos:
            f = g.fifo(fid)
            cs, cd = pc(f.src), pc(f.dst)
            if cs is None and cd is not None and f.src not in port_cond:
                actor_cond[f.src.actor] = cd
                changed = True
            elif cd is None and cs is not None and f.dst not in port_cond:
                actor_cond[f.dst.actor] = cs
                changed = True
    for aid, c in actor_cond.items():
        if c is None:
            actor_cond[aid] = ALWAYS

    fifo_cond: dict[str, int] = {}
    for fid in data_fifos:
        f = g.fifo(fid)
        cs, cd = pc(f.src), pc(f.dst)
        if cs != cd:
            def name(c):
                if c == ALWAYS:
                    return "always"
                return f"{conds[c].ctl}[{conds[c].element}]"
            # the analysis accepted the graph, so this is a layout the
            # per-iteration condition schedule does not cover (a nested
            # region, or an always-active actor feeding a gated subchain)
            unsupported.append(f"fifo {fid}: producer {f.src} is gated by {name(cs)} but "
                               f"consumer {f.dst} by {name(cd)}")
        fifo_cond[fid] = cs
    for fid in control_fifos:
        fifo_cond[fid] = ALWAYS
    # initial delay tokens on data FIFOs: supported on aligned channels
    # (fifos.py:87-92): the producer side writes delay/rate chunks ahead of the
    # consumer side, which first reads the delay payload -- on a gated channel
    # both sides index by the condition's firing count, so the consumer's k-th
    # firing reads the producer's (k - delay/rate)-th
    for fid in data_fifos:
        f = g.fifo(fid)
        if not f.delay:
            continue
        if f.delay % f.rate:
            unsupported.append(f"fifo {fid}: {f.delay} delay tokens are not a multiple of its "
                               f"rate {f.rate}")

    # Cycles (the analysis has rejected delay-free ones): an epoch of E
    # iterations fires every actor's iterations in one launch, which is
    # correct across a channel whose consumer at iteration n reads tokens the
    # producer wrote at n - delay/rate when that lies in an earlier epoch.  So
    # inside a strongly connected component every delayed channel caps the
    # epoch at delay/rate iterations and drops out of the intra-epoch order.
    comp = _components(g, data_fifos)
    epoch_cap = None
    loose: set[str] = set()       # channels not ordering the actors within an epoch
    for fid in data_fifos:
        f = g.fifo(fid)
        if comp[f.src.actor] == comp[f.dst.actor] and f.delay and not f.delay % f.rate:
            d = f.delay // f.rate
            epoch_cap = d if epoch_cap is None else min(epoch_cap, d)
            loose.add(fid)

    # topological order over the ordering channels
    indeg = {a.id: 0 for a in g.actors}
    succ: dict[str, list[str]] = {a.id: [] for a in g.actors}
    for fid in data_fifos:
        if fid in loose:
            continue
        f = g.fifo(fid)
        succ[f.src.actor].append(f.dst.actor)
        indeg[f.dst.actor] += 1
    ready = sorted(a for a, d in indeg.items() if d == 0)
    order: list[str] = []
    while ready:
        a = ready.pop(0)
        order.append(a)
        for b in succ[a]:
            indeg[b] -= 1
            if indeg[b] == 0:
                ready.append(b)
        ready.sort()
    if len(order) != len(g.actors):
        stuck = sorted(a for a, d in indeg.items() if d > 0)
        unsupported.append(f"cycle through {stuck} without delay tokens on every loop")

    # Drain phase (runtime.py:118-124, interp.py:150-205): after the sources
    # stop, an actor keeps firing while every input holds a firing's tokens,
    # i.e. extra(a) = min over its inputs of extra(producer) + delay/rate
    # (sources and configuration actors: 0) -- the shortest-path fixed point;
    # None where no source bounds it (a sourceless cycle spins until the
    # timeout, test_runtime.py:224-235).
    extra = _drain_extra(g, data_fifos, control_fifos, roles)
    for aid, e in extra.items():
        if e and actor_cond[aid] != ALWAYS:
            # a gated actor left with tokens after the sources stop; the
            # reference engines disagree on it (the interpreter reports
            # stranded tokens, the threaded runtime fires it once more)
            unsupported.append(f"actor {aid} is dynamically gated and would fire on delay "
                               "tokens after the sources stop")

    if unsupported:
        raise UnsupportedGraph("; ".join(unsupported))

    eq1 = []
    for a in g.actors:
        if a.kind != DYNAMIC:
            continue
        for p in a.drps:
            ref = PortRef(a.id, p.id)
            fid = g.fifo_into(ref).id if p.direction == "in" else g.fifos_from(ref)[0].id
            eq1.append((a.id, p.id, port_cond[ref], fifo_cond[fid]))

    return ExecPlan(g, conds, {k: v for k, v in actor_cond.items()}, fifo_cond, order, roles,
                    control_fifos, data_fifos, eq1, report, epoch_cap, extra, loose)


def _components(g: Graph, data_fifos: list[str]) -> dict[str, int]:
    """Strongly connected components over the data channels (Tarjan)."""
    succ: dict[str, list[str]] = {a.id: [] for a in g.actors}
    for fid in data_fifos:
        f = g.fifo(fid)
        succ[f.src.actor].append(f.dst.actor)
    index: dict[str, int] = {}
    low: dict[str, int] = {}
    comp: dict[str, int] = {}
    stack: list[str] = []
    on: set[str] = set()
    counter = [0, 0]

    def visit(v: str) -> None:
        work = [(v, iter(succ[v]))]
        index[v] = low[v] = counter[0]
        counter[0] += 1
        stack.append(v)
        on.add(v)
        while work:
            u, it = work[-1]
            nxt = next(it, None)
            if nxt is not None:
                if nxt not in index:
                    index[nxt] = low[nxt] = counter[0]
                    counter[0] += 1
                    stack.append(nxt)
                    on.add(nxt)
                    work.append((nxt, iter(succ[nxt])))
                elif nxt in on:
                    low[u] = min(low[u], index[nxt])
                continue
            work.pop()
            if work:
                low[work[-1][0]] = min(low[work[-1][0]], low[u])
            if low[u] == index[u]:
                while True:
                    w = stack.pop()
                    on.discard(w)
                    comp[w] = counter[1]
                    if w == u:
                        break
                counter[1] += 1

    for a in g.actors:
        if a.id not in index:
            visit(a.id)
    return comp


def _drain_extra(g: Graph, data_fifos: list[str], control_fifos: list[str],
                 roles: dict[str, str]) -> dict[str, int | None]:
    """Firings after the sources stop, per actor (None: unbounded)."""
    INF = float("inf")
    extra = {a.id: (0 if roles[a.id] in ("source", "config") else INF) for a in g.actors}
    ins: dict[str, list[tuple[str, int]]] = {a.id: [] for a in g.actors}
    for fid in data_fifos + control_fifos:
        f = g.fifo(fid)
        ins[f.dst.actor].append((f.src.actor, f.delay // f.rate))
    for _ in range(len(g.actors) + 1):
        changed = False
        for a in g.actors:
            if not ins[a.id]:
                continue
            v = min(extra[p] + d for p, d in ins[a.id])
            if v < extra[a.id]:
                extra[a.id] = v
                changed = True
        if not changed:
            break
    return {k: (None if v == INF else int(v)) for k, v in extra.items()}


def find_filter_banks(plan: ExecPlan, behaviors: dict[str, ActorBehavior]) -> list[FilterBankGroup]:
    """Regions route -> {fir_branch} -> branch_sum that can fire fused.

    Conditions: the router has one data input and only DRP outputs, each DRP
    feeds exactly one fir_branch whose single output feeds a DRP of the same
    branch_sum combiner, and the combiner's data inputs are all such branches
    with one data output.  The branch channels then never leave registers.
    """
    g = plan.graph
    groups = []
    for x in g.actors:
        bx = behaviors.get(x.id)
        if plan.roles[x.id] != "dynamic" or getattr(bx, "kernel", None) != "route":
            continue
        if len(x.data_inputs) != 1:
            continue
        outs = [p for p in x.output_ports]
        if not outs or any(p.kind != DRP for p in outs):
            continue
        branches: dict[str, str] = {}   # combiner port -> fir actor
        internal: set[str] = set()
        combiner = None
        ok = True
        for p in outs:
            fs = g.fifos_from(PortRef(x.id, p.id))
            if len(fs) != 1:
                ok = False
                break
            b = g.actor(fs[0].dst.actor)
            if getattr(behaviors.get(b.id), "kernel", None) != "fir" or \
                    len(b.input_ports) != 1 or len(b.output_ports) != 1:
                ok = False
                break
            fo = g.fifos_from(PortRef(b.id, b.output_ports[0].id))
            if len(fo) != 1:
                ok = False
                break
            y = g.actor(fo[0].dst.actor)
            if combiner is None:
                combiner = y.id
            if y.id != combiner or y.port(fo[0].dst.port).kind != DRP:
                ok = False
                break
            branches[fo[0].dst.port] = b.id
            internal.update({fs[0].id, fo[0].id})
        if not ok or combiner is None:
            continue
        y = g.actor(combiner)
        if getattr(behaviors.get(y.id), "kernel", None) != "branch_sum":
            continue
        if sorted(p.id for p in y.data_inputs) != sorted(branches):
            continue
        if len([p for p in y.output_ports]) != 1:
            continue
        if any(g.fifo(fid).delay for fid in internal):
            continue            # a delayed branch channel stays materialised
        spans = {g.fifo(fid).rate * g.fifo(fid).token_bytes for fid in internal}
        src = g.fifo_into(PortRef(x.id, x.data_inputs[0].id))
        if spans != {src.rate * src.token_bytes}:
            continue
        groups.append(FilterBankGroup(x.id, combiner, [branches[p] for p in sorted(branches)],
                                      internal))
    return groups


@dataclass
class MatmulChain:
    """Consecutive matmul actors fired as one kernel (pb_fire_matmul_chain)."""

    actors: list[str]            # in data order
    internal_fifos: set[str]     # the link channels (not materialised)


def find_matmul_chains(plan: ExecPlan, behaviors: dict[str, ActorBehavior]) -> list[MatmulChain]:
    """Maximal chains a_1 -> ... -> a_k (k >= 2) of 8x8 matmul actors
    (bypass.py:36-49) under one condition whose link channels are exclusive
    (the producer's only output, the consumer's only input), undelayed and one
    token per firing, and whose members fire no extra drain firings.  Such a
    chain's tokens between members never need to leave registers."""
    g = plan.graph

    def is_mm(aid):
        b = behaviors.get(aid)
        if getattr(b, "kernel", None) != "matmul":
            return False
        a = g.actor(aid)
        if len(a.data_inputs) != 1 or len(a.output_ports) != 1:
            return False
        n2 = len(g.actor(aid).params.get("w", []))
        return n2 == 64 and plan.extra.get(aid, 0) == 0

    def link(aid):   # the channel to the next member, or None
        a = g.actor(aid)
        fs = g.fifos_from(PortRef(aid, a.output_ports[0].id))
        if len(fs) != 1:
            return None
        f = fs[0]
        nxt = f.dst.actor
        if not is_mm(nxt) or f.delay or f.rate != 1 or f.token_bytes != 256 or \
                plan.actor_cond[nxt] != plan.actor_cond[aid] or \
                plan.fifo_cond[f.id] != plan.actor_cond[aid]:
            return None
        return f
    chains = []
    heads = [a.id for a in g.actors if is_mm(a.id)]
    has_pred = set()
    for aid in heads:
        f = link(aid)
        if f is not None:
            has_pred.add(f.dst.actor)
    for aid in heads:
        if aid in has_pred:
            continue
        members, internal = [aid], set()
        cur = aid
        while True:
            f = link(cur)
            if f is None or len(members) == 8:
                break
            members.append(f.dst.actor)
            internal.add(f.id)
            cur = f.dst.actor
        if len(members) >= 2:
            chains.append(MatmulChain(members, internal))
    return chains


@dataclass
class BypassRegion:
    """route -> matmul chain -> path_merge, the route's other output straight
    into the merge's bypass port (bypass.py:69-132), fired as one kernel."""

    chain: MatmulChain
    route: str
    merge: str
    chain_out: str       # the chain's output channel into the merge (not materialised)
    bypass_fifo: str     # route -> merge bypass channel
    out_fifo: str        # the merge's output channel


def find_bypass_regions(plan: ExecPlan, behaviors: dict[str, ActorBehavior],
                        chains: list[MatmulChain]) -> list[BypassRegion]:
    g = plan.graph
    kern = lambda aid: getattr(behaviors.get(aid), "kernel", None)
    out = []
    for c in chains:
        head, tail = g.actor(c.actors[0]), g.actor(c.actors[-1])
        f_in = g.fifo_into(PortRef(head.id, head.data_inputs[0].id))
        r = g.actor(f_in.src.actor)
        if kern(r.id) != "route" or len(r.data_inputs) != 1 or len(r.output_ports) != 2 or \
                any(p.kind != DRP for p in r.output_ports) or f_in.delay:
            continue
        fo = g.fifos_from(PortRef(tail.id, tail.output_ports[0].id))
        if len(fo) != 1 or fo[0].delay:
            continue
        m = g.actor(fo[0].dst.actor)
        bport = m.params.get("bypass_port", "")
        if kern(m.id) != "path_merge" or len(m.data_inputs) != 2 or fo[0].dst.port == bport \
                or len(m.output_ports) != 1:
            continue
        other = [p for p in r.output_ports if p.id != f_in.src.port]
        fb = g.fifos_from(PortRef(r.id, other[0].id))
        if len(fb) != 1 or fb[0].dst != PortRef(m.id, bport) or fb[0].delay:
            continue
        fm = g.fifos_from(PortRef(m.id, m.output_ports[0].id))
        if len(fm) != 1 or fm[0].delay:
            continue
        src = g.fifo_into(PortRef(r.id, r.data_inputs[0].id))
        span = src.rate * src.token_bytes
        if any(f.rate * f.token_bytes != span for f in (f_in, fo[0], fb[0], fm[0])) or span != 256:
            continue
        if plan.extra.get(m.id, 0) != 0 or plan.extra.get(r.id, 0) != 0:
            continue
        out.append(BypassRegion(c, r.id, m.id, fo[0].id, fb[0].id, fm[0].id))
    return out


@dataclass
class MotionRegion:
    """blur -> frame_diff_threshold (cur, prev delayed one frame) -> plus_median
    fired as one kernel (pb_fire_motion_region)."""

    blur: str
    detect: str
    clean: str
    cur_fifo: str
    prev_fifo: str
    mask_fifo: str
    out_fifo: str
    side: int


def find_motion_regions(plan: ExecPlan, behaviors: dict[str, ActorBehavior]) -> list[MotionRegion]:
    """The motion app's chain (apps/motion.py:74-108): a gauss_blur whose one
    output port feeds exactly a frame_diff_threshold's "cur" (undelayed) and
    "prev" (one token of delay), whose one output feeds only a plus_median with
    one output channel; every actor and channel always active, one frame per
    firing, a power-of-two side, no drain firings."""
    g = plan.graph
    op = lambda aid: getattr(behaviors.get(aid), "op", None) \
        if getattr(behaviors.get(aid), "kernel", None) == "image" else None
    out = []
    for a in g.actors:
        if op(a.id) != 0 or len(a.data_inputs) != 1 or len(a.output_ports) != 1:
            continue
        fs = g.fifos_from(PortRef(a.id, a.output_ports[0].id))
        if len(fs) != 2:
            continue
        d = fs[0].dst.actor
        if fs[1].dst.actor != d or op(d) != 1:
            continue
        by_port = {f.dst.port: f for f in fs}
        if set(by_port) != {"cur", "prev"}:
            continue
        fc, fp = by_port["cur"], by_port["prev"]
        tb = fc.token_bytes
        side = int(round(tb ** 0.5))
        if fc.delay or fp.delay != 1 or fc.rate != 1 or fp.rate != 1 or fp.token_bytes != tb \
                or side * side != tb or side < 8 or side > 128 or side & (side - 1):
            continue
        da = g.actor(d)
        if len(da.output_ports) != 1:
            continue
        fm = g.fifos_from(PortRef(d, da.output_ports[0].id))
        if len(fm) != 1 or fm[0].delay or fm[0].rate != 1 or fm[0].token_bytes != tb:
            continue
        m = fm[0].dst.actor
        ma = g.actor(m)
        if op(m) != 2 or len(ma.output_ports) != 1:
            continue
        fo = g.fifos_from(PortRef(m, ma.output_ports[0].id))
        if len(fo) != 1 or fo[0].delay or fo[0].rate != 1 or fo[0].token_bytes != tb:
            continue
        members = (a.id, d, m)
        fifos = (fc.id, fp.id, fm[0].id, fo[0].id)
        if any(plan.actor_cond[x] != ALWAYS or plan.extra.get(x, 0) != 0 for x in members) or \
                any(plan.fifo_cond[f] != ALWAYS for f in fifos):
            continue
        out.append(MotionRegion(a.id, d, m, fc.id, fp.id, fm[0].id, fo[0].id, side))
    return out


def is_device(b: ActorBehavior) -> bool:
    return isinstance(b, DeviceBehavior) or bool(getattr(b, "kernel", ""))
