"""Decidability analysis of PRUNE graphs: the admission gate of the engine.

The reference admits a graph through `analysis.analyze(graph, c_factor)`
(analysis.py:414-460), which runs the five design rules (rules.py:162-291),
identifies the dynamic processing graphs (analysis.py:139-184), decomposes
and validates them (:194-319), schedules the fully-active graph and every
dynamic component (:322-395) and derives the buffer bounds (:398-411).
`runtime.instantiate` raises InconsistentGraph for any graph it reports as
inconsistent (runtime.py:327-336).  This module re-derives the same verdict,
the same violation/diagnostic codes and subjects and the same bounds, so the
device engine admits exactly the graphs the reference admits; the engine's
own executor-class checks (plan.py) come after and raise UnsupportedGraph.

The formulation differs from the reference's where graph theory gives a
direct answer:

* linked ports: the members of all simple directed chains from the output
  port's consumers to the input port's feeder are the vertices that lie on
  some simple path; on an acyclic remainder that is "reachable from a head
  and reaching the feeder", otherwise a pruned path search decides it;
* rule 5's "lies on a chain connecting x and y" is the union of the
  biconnected blocks on the block-cut-tree path from x to y;
* a period schedule deadlocks exactly on the actors that sit on, or
  downstream of, a cycle of channels holding fewer initial tokens than their
  rate, which a Kahn pass over those channels finds without simulation.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .graph import (CONTROL_IN, CONTROL_OUT, DRP, SRP, STATIC, ControlTableError, Graph,
                    PortRef)

RULE_NAMES = {1: "linked port control rule", 2: "balanced delay rule",
              3: "connecting subchain rule", 4: "single-sided dynamism rule",
              5: "encapsulation rule"}


@dataclass(frozen=True)
class Violation:
    """A design-rule violation (rules.py:31-42): rule number and subjects."""

    rule: int
    subjects: tuple[str, ...]
    message: str

    @property
    def name(self) -> str:
        return RULE_NAMES[self.rule]

    def render(self) -> str:
        return f"rule {self.rule} ({self.name}): {', '.join(self.subjects)}: {self.message}"


@dataclass(frozen=True)
class Diagnostic:
    """An analysis finding (analysis.py:80-87): code and subjects."""

    code: str
    subjects: tuple[str, ...]
    message: str

    def render(self) -> str:
        return f"{self.code}: {', '.join(self.subjects)}: {self.message}"


@dataclass(frozen=True)
class LinkedPair:
    """An output dynamic port linked to an input one (rules.py:45-61)."""

    out_port: PortRef
    in_port: PortRef
    direct: bool
    members: frozenset[str]      # actors on the connecting subchains

    @property
    def parents(self) -> tuple[str, str]:
        return self.out_port.actor, self.in_port.actor


@dataclass(frozen=True)
class Component:
    """One dynamic component of a DPG (analysis.py:53-64)."""

    index: int
    members: tuple[str, ...]
    in_drps: tuple[PortRef, ...]
    out_drps: tuple[PortRef, ...]
    elements: tuple[int, ...]
    direct_fifo: str | None = None


@dataclass(frozen=True)
class Dpg:
    """q configures the dynamic pair (x, y) (analysis.py:67-77)."""

    q: str
    x: str
    y: str
    control_port: PortRef
    declared_len: int
    members: tuple[str, ...]
    dcs: tuple[Component, ...] = ()


class BufferBounds:
    """analysis.py:115-118 (the per-region split is not kept)."""

    def __init__(self, beta: dict[str, int], c_factor: int):
        self.beta = dict(beta)
        self.c_factor = c_factor


@dataclass
class AnalysisReport:
    """Verdict, findings, regions and the per-FIFO bound beta(f) for the
    chosen buffering factor (analysis.ConsistencyReport, :121-132)."""

    verdict: str = "consistent"
    violations: tuple[Violation, ...] = ()
    diagnostics: tuple[Diagnostic, ...] = ()
    dpgs: tuple[Dpg, ...] = ()
    regions: tuple[str, ...] = ()
    beta: dict[str, int] = field(default_factory=dict)
    c_factor: int = 3

    @property
    def consistent(self) -> bool:
        return self.verdict == "consistent"

    @property
    def bounds(self) -> "BufferBounds | None":
        """analysis.BufferBounds (:115-118): the per-FIFO bound beta at c_factor."""
        if not self.consistent:
            return None
        return BufferBounds(self.beta, self.c_factor)

    @property
    def problems(self) -> list[str]:
        return [v.render() for v in self.violations] + [d.render() for d in self.diagnostics]


# ------------------------------------------------------------ graph helpers

def _succ(g: Graph, skip: frozenset[str] = frozenset()) -> dict[str, list[str]]:
    out: dict[str, list[str]] = {a.id: [] for a in g.actors}
    for f in g.fifos:
        if f.src.actor not in skip and f.dst.actor not in skip:
            out[f.src.actor].append(f.dst.actor)
    return out


def _reach(adj: dict[str, list[str]], starts) -> set[str]:
    seen = set(starts)
    todo = list(seen)
    while todo:
        for b in adj[todo.pop()]:
            if b not in seen:
                seen.add(b)
                todo.append(b)
    return seen


def _acyclic(adj: dict[str, list[str]], nodes: set[str]) -> bool:
    indeg = {v: 0 for v in nodes}
    for v in nodes:
        for w in adj[v]:
            if w in indeg:
                indeg[w] += 1
    ready = [v for v, d in indeg.items() if d == 0]
    n = 0
    while ready:
        v = ready.pop()
        n += 1
        for w in adj[v]:
            if w in indeg:
                indeg[w] -= 1
                if indeg[w] == 0:
                    ready.append(w)
    return n == len(nodes)


def _path_members(adj: dict[str, list[str]], heads: list[str], goal: str) -> set[str]:
    """Actors on some simple directed path from one of `heads` to `goal`
    (adj already excludes the forbidden actors)."""
    back: dict[str, list[str]] = {v: [] for v in adj}
    for v, ws in adj.items():
        for w in ws:
            back[w].append(v)
    to_goal = _reach(back, [goal])
    live = [h for h in heads if h in to_goal]
    if not live:
        return set()
    fwd = _reach(adj, live)
    core = fwd & to_goal
    if _acyclic(adj, core):
        return core
    # cyclic remainder: simple-path membership needs a search (pruned to core)
    members: set[str] = set()
    for h in set(live):
        stack = [(h, (h,))]
        while stack:
            v, path = stack.pop()
            if v == goal:
                members.update(path)
                continue
            for w in adj[v]:
                if w in core and w not in path:
                    stack.append((w, path + (w,)))
    return members


def linked_pairs(g: Graph) -> list[LinkedPair]:
    """Every linked dynamic-port pair (rules.py:91-129): the ports share a
    FIFO, or a simple chain of other actors carries data from the output
    port's consumers to the input port's feeder."""
    outs, ins = [], []
    for a in g.actors:
        for p in a.drps:
            (outs if p.direction == "out" else ins).append(PortRef(a.id, p.id))
    pairs = []
    cache: dict[frozenset[str], dict[str, list[str]]] = {}
    for px in outs:
        from_px = g.fifos_from(px)
        for py in ins:
            if px.actor == py.actor:
                continue
            direct = any(f.dst == py for f in from_px)
            last = g.fifo_into(py).src.actor
            members: set[str] = set()
            if last not in (px.actor, py.actor):
                skip = frozenset((px.actor, py.actor))
                if skip not in cache:
                    cache[skip] = _succ(g, skip)
                heads = [f.dst.actor for f in from_px if f.dst.actor not in skip]
                members = _path_members(cache[skip], heads, last)
            if direct or members:
                pairs.append(LinkedPair(px, py, direct, frozenset(members)))
    pairs.sort(key=lambda p: (str(p.out_port), str(p.in_port)))
    return pairs


def _blocks_between(g: Graph, x: str, y: str) -> set[str]:
    """Actors on at least one simple undirected x..y chain: the union of the
    biconnected blocks on the block-cut-tree path from x to y."""
    nbr: dict[str, set[str]] = {a.id: set() for a in g.actors}
    for f in g.fifos:
        if f.src.actor != f.dst.actor:
            nbr[f.src.actor].add(f.dst.actor)
            nbr[f.dst.actor].add(f.src.actor)
    # Hopcroft-Tarjan biconnected components from x (iterative)
    disc: dict[str, int] = {x: 0}
    low: dict[str, int] = {x: 0}
    blocks: list[set[str]] = []
    estack: list[tuple[str, str]] = []
    stack = [(x, None, iter(sorted(nbr[x])))]
    while stack:
        v, parent, it = stack[-1]
        w = next(it, None)
        if w is None:
            stack.pop()
            if parent is not None:
                low[parent] = min(low[parent], low[v])
                if low[v] >= disc[parent]:
                    blk = set()
                    while True:
                        e = estack.pop()
                        blk.update(e)
                        if e == (parent, v):
                            break
                    blocks.append(blk)
            continue
        if w == parent:
            continue
        if w not in disc:
            disc[w] = low[w] = len(disc)
            estack.append((v, w))
            stack.append((w, v, iter(sorted(nbr[w]))))
        elif disc[w] < disc[v]:
            low[v] = min(low[v], disc[w])
            estack.append((v, w))
    if y not in disc:
        return set()
    # block-cut tree: block nodes b<k>, vertex nodes for x, y and cut vertices
    owners: dict[str, list[int]] = {}
    for k, blk in enumerate(blocks):
        for v in blk:
            owners.setdefault(v, []).append(k)
    tree: dict[object, set] = {}
    for v, ks in owners.items():
        if len(ks) > 1 or v in (x, y):
            for k in ks:
                tree.setdefault(("v", v), set()).add(("b", k))
                tree.setdefault(("b", k), set()).add(("v", v))
    prev = {("v", x): None}
    todo = [("v", x)]
    while todo:
        node = todo.pop()
        for nxt in tree.get(node, ()):
            if nxt not in prev:
                prev[nxt] = node
                todo.append(nxt)
    out: set[str] = set()
    node = ("v", y)
    while node is not None:
        if node[0] == "b":
            out |= blocks[node[1]]
        node = prev[node]
    return out


# -------------------------------------------------------------------- rules

def design_rules(g: Graph, pairs: list[LinkedPair]) -> list[Violation]:
    """Rules 1-5 (rules.py:162-291), sorted by rule then subjects."""
    found: list[Violation] = []
    # rule 1: linked ports share one controlling port and element
    for pr in pairs:
        a, b = g.control_lookup(pr.out_port), g.control_lookup(pr.in_port)
        if a != b:
            found.append(Violation(1, (str(pr.out_port), str(pr.in_port)),
                                   f"linked ports controlled by {a[0]}[{a[1]}] vs "
                                   f"{b[0]}[{b[1]}]"))
    # rule 2: every fan-out of a control port carries the same delay
    fan: dict[PortRef, list] = {}
    for f in g.fifos:
        if g.actor(f.src.actor).port(f.src.port).kind == CONTROL_OUT:
            fan.setdefault(f.src, []).append(f)
    for src in sorted(fan, key=str):
        first, *rest = sorted(fan[src], key=lambda f: str(f.dst))
        for f in rest:
            if f.delay != first.delay:
                found.append(Violation(2, (str(src), str(first.dst), str(f.dst)),
                                       f"control delays differ: {first.dst} has {first.delay}, "
                                       f"{f.dst} has {f.delay}"))
    # rule 3: subchain members are static and serve one dynamic pair
    owners: dict[str, set[tuple[str, str]]] = {}
    flagged: set[str] = set()
    for pr in pairs:
        key = tuple(sorted(pr.parents))
        for m in sorted(pr.members):
            owners.setdefault(m, set()).add(key)
            if g.actor(m).kind != STATIC and m not in flagged:
                flagged.add(m)
                found.append(Violation(3, (m,), "connecting subchain member is not a static "
                                                 "actor"))
    for m in sorted(owners):
        if len(owners[m]) > 1:
            names = "; ".join("{" + ", ".join(o) + "}" for o in sorted(owners[m]))
            found.append(Violation(3, (m,), f"subchain actor serves several dynamic actor "
                                            f"pairs: {names}"))
    # rule 4: no actor owns dynamic ports in both directions
    for a in g.actors:
        if len({p.direction for p in a.drps}) > 1:
            found.append(Violation(4, (a.id,), "actor has both input and output dynamic ports"))
    # rule 5: actors touching a subchain through a static port sit on an x..y chain
    between: dict[tuple[str, str], set[str]] = {}
    marks: set[tuple[str, str, str, str]] = set()
    for pr in pairs:
        if not pr.members:
            continue
        x, y = pr.parents
        for ai in sorted(pr.members):
            for f in g.fifos:
                for near, far in ((f.src, f.dst), (f.dst, f.src)):
                    b = far.actor
                    if near.actor != ai or b in pr.members or b in (x, y):
                        continue
                    if g.actor(b).port(far.port).kind != SRP:
                        continue
                    if (x, y) not in between:
                        between[(x, y)] = _blocks_between(g, x, y)
                    if b not in between[(x, y)] and (b, ai, x, y) not in marks:
                        marks.add((b, ai, x, y))
                        found.append(Violation(5, (b, ai),
                                               f"{b} touches subchain actor {ai} through a "
                                               f"static port but lies on no chain connecting "
                                               f"{x} and {y}"))
    found.sort(key=lambda v: (v.rule, v.subjects))
    return found


# ------------------------------------------------------------ DPG analysis

class _Reject(Exception):
    def __init__(self, code: str, actor: str, detail: str):
        self.diag = Diagnostic(code, (actor,), detail)


def dynamic_processing_graphs(g: Graph, pairs: list[LinkedPair]) -> list[Dpg]:
    """Group dynamic/configuration actors into DPGs (analysis.py:139-184);
    raises _Reject(OrphanDynamicActor | SharedMembership)."""
    keys: dict[str, set[frozenset[str]]] = {}
    for pr in pairs:
        for a in pr.parents:
            keys.setdefault(a, set()).add(frozenset(pr.parents))
    for a in g.actors:
        if a.kind != "dynamic":
            continue
        ks = keys.get(a.id, set())
        if not ks:
            raise _Reject("OrphanDynamicActor", a.id,
                          f"dynamic actor {a.id} is linked to no partner")
        if len(ks) > 1:
            raise _Reject("SharedMembership", a.id, f"actor {a.id} is claimed by two dynamic "
                          "processing graphs (linked into two dynamic actor pairs)")
    dpgs = []
    q_of: dict[str, frozenset[str]] = {}
    member_of: dict[str, frozenset[str]] = {}
    for key in sorted({k for ks in keys.values() for k in ks}, key=sorted):
        x, y = next(pr.parents for pr in pairs if frozenset(pr.parents) == key)
        group = [pr for pr in pairs if pr.parents == (x, y)]
        ctl = g.control_lookup(group[0].out_port)[0]
        if ctl.actor in q_of and q_of[ctl.actor] != key:
            raise _Reject("SharedMembership", ctl.actor,
                          f"actor {ctl.actor} is claimed by two dynamic processing graphs "
                          "(configuration actor controls two dynamic pairs)")
        q_of[ctl.actor] = key
        sub = sorted(set().union(*(pr.members for pr in group)))
        for m in sub:
            if member_of.setdefault(m, key) != key:
                raise _Reject("SharedMembership", m, f"actor {m} is claimed by two dynamic "
                              "processing graphs (subchain actor shared between regions)")
        dpgs.append(Dpg(ctl.actor, x, y, ctl, g.value_length(ctl),
                        tuple([ctl.actor, x, y] + sub)))
    return dpgs


def components(g: Graph, d: Dpg, pairs: list[LinkedPair]) -> Dpg:
    """Dynamic components of a DPG (analysis.py:194-261): connected pieces
    of its subchain actors, plus one placeholder per direct x->y FIFO."""
    group = [pr for pr in pairs if pr.parents == (d.x, d.y)]
    sub = set().union(*(pr.members for pr in group)) if group else set()
    parent = {m: m for m in sub}

    def root(v):
        while parent[v] != v:
            parent[v] = parent[parent[v]]
            v = parent[v]
        return v
    for f in g.fifos:
        if f.src.actor in sub and f.dst.actor in sub:
            parent[root(f.src.actor)] = root(f.dst.actor)
    comps: dict[str, list[str]] = {}
    for m in sub:
        comps.setdefault(root(m), []).append(m)
    ordered = sorted(tuple(sorted(c)) for c in comps.values())
    xs = [PortRef(d.x, p.id) for p in g.actor(d.x).drps if p.direction == "out"]
    ys = [PortRef(d.y, p.id) for p in g.actor(d.y).drps if p.direction == "in"]
    dcs = []
    for k, comp in enumerate(ordered, start=1):
        cs = set(comp)
        din = tuple(p for p in xs if any(f.dst.actor in cs for f in g.fifos_from(p)))
        dout = tuple(p for p in ys if g.fifo_into(p).src.actor in cs)
        els = tuple(sorted({g.control_lookup(p)[1] for p in din + dout}))
        dcs.append(Component(k, comp, din, dout, els))
    for pr in sorted((pr for pr in group if pr.direct),
                     key=lambda pr: g.fifo_into(pr.in_port).id):
        fid = g.fifo_into(pr.in_port).id
        els = tuple(sorted({g.control_lookup(pr.out_port)[1], g.control_lookup(pr.in_port)[1]}))
        dcs.append(Component(len(dcs) + 1, (f"dummy:{fid}",), (pr.out_port,), (pr.in_port,),
                             els, fid))
    return Dpg(d.q, d.x, d.y, d.control_port, d.declared_len, d.members, tuple(dcs))


def check_components(g: Graph, d: Dpg) -> list[Diagnostic]:
    """Component <-> control element mapping checks (analysis.py:264-319)."""
    name = f"dpg {d.q}"
    out: list[Diagnostic] = []
    if not d.dcs:
        return [Diagnostic("SurjectivityFailure", (name,),
                           "no dynamic component between the dynamic actors")]
    for dc in d.dcs:
        label = f"dc {dc.index}"
        if not dc.in_drps:
            out.append(Diagnostic("SurjectivityFailure", (name, label),
                                  f"component not fed by any dynamic port of {d.x}"))
        if not dc.out_drps:
            out.append(Diagnostic("SurjectivityFailure", (name, label),
                                  f"component feeds no dynamic port of {d.y}"))
        if len(dc.elements) != 1:
            out.append(Diagnostic("ControlElementFailure", (name, label),
                                  f"ports of one component use control elements "
                                  f"{list(dc.elements)}"))
    touched: dict[PortRef, list[int]] = {}
    for dc in d.dcs:
        for p in dc.in_drps + dc.out_drps:
            touched.setdefault(p, []).append(dc.index)
    ports = [PortRef(d.x, p.id) for p in g.actor(d.x).drps if p.direction == "out"] + \
            [PortRef(d.y, p.id) for p in g.actor(d.y).drps if p.direction == "in"]
    for p in ports:
        t = touched.get(p, [])
        if not t:
            out.append(Diagnostic("SurjectivityFailure", (name, str(p)),
                                  "dynamic port reaches no component"))
        elif len(t) > 1:
            out.append(Diagnostic("DrpFanoutFailure", (name, str(p)),
                                  f"dynamic port reaches components {t}"))
    m = len(d.dcs)
    if d.declared_len != m:
        out.append(Diagnostic("BijectionFailure", (name,),
                              f"declared control-value length {d.declared_len} != component "
                              f"count {m}"))
    else:
        single = [dc.elements[0] for dc in d.dcs if len(dc.elements) == 1]
        if len(single) == m and len(set(single)) != m:
            out.append(Diagnostic("BijectionFailure", (name,),
                                  f"control elements {sorted(single)} do not map components "
                                  "one-to-one"))
    return out


def _regions(g: Graph, dpgs: list[Dpg]) -> list[tuple[str, set[str], list]]:
    """The fully-active graph and one activation round per component
    (analysis.py:322-346): (id, actors, fifos)."""
    out = [("static", {a.id for a in g.actors}, list(g.fifos))]
    for d in dpgs:
        for dc in d.dcs:
            rid = f"{d.q}.dc{dc.index}"
            if dc.direct_fifo is not None:
                out.append((rid, {d.x, d.y}, [g.fifo(dc.direct_fifo)]))
                continue
            ms = set(dc.members)
            fs = [f for f in g.fifos if (f.src.actor in ms and f.dst.actor in ms) or
                  f.src in dc.in_drps or f.dst in dc.out_drps]
            out.append((rid, ms | {d.x, d.y}, fs))
    return out


def stuck_actors(actors: set[str], fifos: list) -> list[str]:
    """Actors that cannot fire in one period where every actor fires once
    (analysis.py:349-395): a FIFO with fewer initial tokens than its rate
    makes its consumer wait for its producer, so the stuck actors are those
    a Kahn pass over such FIFOs never releases."""
    indeg = {a: 0 for a in actors}
    nxt: dict[str, list[str]] = {a: [] for a in actors}
    for f in fifos:
        # a FIFO leaving the region (a component port that also feeds an
        # outside actor) fails like the reference's lookup (KeyError)
        src, dst = nxt[f.src.actor], indeg[f.dst.actor]
        if f.delay < f.rate:
            indeg[f.dst.actor] = dst + 1
            src.append(f.dst.actor)
    ready = [a for a, k in indeg.items() if k == 0]
    while ready:
        for b in nxt[ready.pop()]:
            indeg[b] -= 1
            if indeg[b] == 0:
                ready.append(b)
    return sorted(a for a, k in indeg.items() if k > 0)


def analyze(g: Graph, c_factor: int = 3) -> AnalysisReport:
    """The reference's admission analysis (analysis.py:414-460): never raises
    for graph-level problems; the report carries the verdict."""
    rep = AnalysisReport(c_factor=c_factor)
    uncontrolled = []
    for a in g.actors:
        if a.kind != "dynamic":
            continue
        for p in a.drps:
            try:
                g.control_lookup(PortRef(a.id, p.id))
            except ControlTableError as e:
                uncontrolled.append(Diagnostic("Uncontrolled", (f"{a.id}.{p.id}",), str(e)))
    if uncontrolled:
        rep.verdict, rep.diagnostics = "inconsistent", tuple(uncontrolled)
        return rep
    pairs = linked_pairs(g)
    violations = design_rules(g, pairs)
    if violations:
        rep.verdict, rep.violations = "inconsistent", tuple(violations)
        return rep
    try:
        dpgs = [components(g, d, pairs) for d in dynamic_processing_graphs(g, pairs)]
    except _Reject as e:
        rep.verdict, rep.diagnostics = "inconsistent", (e.diag,)
        return rep
    rep.dpgs = tuple(dpgs)
    diags = [x for d in dpgs for x in check_components(g, d)]
    if diags:
        rep.verdict, rep.diagnostics = "inconsistent", tuple(diags)
        return rep
    regions = _regions(g, dpgs)
    rep.regions = tuple(r for r, _, _ in regions)
    for rid, actors, fifos in regions:
        stuck = stuck_actors(actors, fifos)
        if stuck:
            diags.append(Diagnostic("DeadlockError", tuple(stuck),
                                    f"region {rid}: no fireable actor; stuck cycle through "
                                    f"{', '.join(stuck)}"))
    if diags:
        rep.verdict, rep.diagnostics = "inconsistent", tuple(diags)
        return rep
    # beta(f) = worst single-period occupancy (delay + rate) plus C-1 extra
    # chunks (analysis.py:387, :398-411); the same in every region holding f
    for _, _, fifos in regions:
        for f in fifos:
            rep.beta[f.id] = max(rep.beta.get(f.id, 0), f.delay + f.rate + (c_factor - 1) * f.rate)
    return rep


def layout_slots(rate: int, delay: int, factor: int) -> int:
    """Slots of a reference channel (fifos.py:87-98 layout_plan): aligned
    when delay % rate == 0."""
    if delay % rate == 0:
        return max(rate * factor, delay)
    return rate * factor + delay


__all__ = ["AnalysisReport", "Component", "Diagnostic", "Dpg", "LinkedPair", "Violation",
           "analyze", "check_components", "components", "design_rules",
           "dynamic_processing_graphs", "layout_slots", "linked_pairs", "stuck_actors",
           "CONTROL_IN", "DRP"]
