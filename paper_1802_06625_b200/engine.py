"""Device executor: the B200 replacement for tokenflow.runtime.run.

Same entry points and report as the threaded reference engine
(runtime.py:51-74 RuntimeConfig/RunReport, :327-347 instantiate/run), plus
`run_streams` for a batch of independent replicas of one graph (the unit the
B200 shards over).  Execution is epoch-batched instead of one thread per
actor (runtime.py:118-193):

  per epoch of E iterations (E <= RuntimeConfig.epoch) for all streams:
    1. host sources stage E spans per stream -> one pinned H2D per port
    2. host configuration actors emit E control tokens per stream (native
       CPython-compatible generator, csrc/pb_policy.cpp) -> one H2D
    3. pb_resolve: control tokens -> per-condition activity / prefix /
       firing lists on the device (Eq. 1, runtime.py:107-116)
    4. pb_eq1_check: the recheck of runtime.py:195-220
    5. every device actor fires ALL its firings of the epoch in one launch,
       in topological order (route aliases, fused filter banks, FIR groups)
    6. pb_rings_advance: ring counters / peak occupancy in bulk
    7. sinks: D2H of the epoch's sink spans, SHA-256 per firing in sorted
       port order (runtime.py:175-180), optional capture

FIFO channels are device rings of C = max(c_factor, epoch) chunks; a
channel's per-epoch tokens never exceed E <= C (RunReport.device_slots /
device_max_occupancy).  slots, beta and max_occupancy keep the reference's
meaning at the caller's c_factor.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import queue
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Callable, Mapping, Sequence

import numpy as np

from . import _lib
from .admission import layout_slots
from .behaviors import (ActorBehavior, DeviceBehavior, FileSource, FireContext, actor_seed,
                        decode_control, native_policy_kind, resolve)
from .errors import ActorPanic, DeviceUnavailable, Timeout, UnsupportedGraph
from .graph import CONTROL_IN, CONTROL_OUT, DRP, Graph, PortRef, as_graph
from .plan import (ALWAYS, ExecPlan, admit, find_bypass_regions, find_filter_banks,
                   find_matmul_chains, find_motion_regions, is_device)


@dataclass
class RuntimeConfig:
    """runtime.py:51-61, plus the device executor's knobs."""

    source_firings: int = 1
    c_factor: int = 3
    seed: int | None = None
    jitter_ms: float = 0.0        # accepted; the batched schedule is deterministic
    jitter_seed: int | None = None
    pin_cores: bool = False       # accepted; host work is a few bulk calls
    capture_sinks: bool = False
    timeout_ms: float | None = None
    trace: Callable[[str], None] | None = None
    # device executor
    epoch: int = 4096             # iterations fired per batched epoch
    fuse: bool = True             # fire route -> fir_branch* -> branch_sum as one kernel
    device: int = 0
    host_threads: int = 0         # threads for native policies and digests (0 = all)
    pipeline: int = 8             # sub-epochs overlapping H2D / kernels / D2H / hashing (1 = off)
    exact: bool = True            # False: FIR taps as fused multiply-adds (<= 1e-5, not bit-exact)
    conv_i8: bool = True          # Cin-32 convs on int8 limbs (logits <= 1e-3); False: bf16x3


@dataclass
class RunReport:
    """runtime.py:64-74."""

    sink_digests: dict[str, str] = field(default_factory=dict)
    sink_data: dict[str, bytes] = field(default_factory=dict)
    firing_counts: dict[str, int] = field(default_factory=dict)
    max_occupancy: dict[str, int] = field(default_factory=dict)
    slots: dict[str, int] = field(default_factory=dict)
    beta: dict[str, int] = field(default_factory=dict)
    eq1_checks: int = 0
    eq1_failures: int = 0
    wall_ms: float = 0.0
    # device executor: ring capacity (tokens) and the measured peak ring
    # occupancy per FIFO; an epoch's tokens are in flight at once, so these
    # scale with the epoch rather than with c_factor
    device_slots: dict[str, int] = field(default_factory=dict)
    device_max_occupancy: dict[str, int] = field(default_factory=dict)


@dataclass
class _Plan:
    slots: int


class ChannelView:
    """FifoChannel's observable state (fifos.py:142-338) for one device ring."""

    def __init__(self, fifo_id: str, occupancy: int, max_occupancy: int, slots: int):
        self.fifo_id = fifo_id
        self.occupancy = occupancy
        self.max_occupancy = max_occupancy
        self.plan = _Plan(slots)


class _Dev:
    """Small RAII helper for device / pinned allocations."""

    def __init__(self):
        self.lib = _lib.load()
        self.dev: list[int] = []
        self.host: list[int] = []
        self.rings: list[int] = []

    def malloc(self, nbytes: int, zero: bool = True) -> int:
        p = C.c_void_p()
        _lib.check(self.lib.pb_malloc(C.byref(p), max(16, int(nbytes))), "pb_malloc")
        self.dev.append(p.value)
        if zero:
            _lib.check(self.lib.pb_memset(p, 0, max(16, int(nbytes)), None), "pb_memset")
        return p.value

    def pinned(self, nbytes: int) -> tuple[int, np.ndarray]:
        p = C.c_void_p()
        _lib.check(self.lib.pb_host_alloc(C.byref(p), max(16, int(nbytes))), "pb_host_alloc")
        self.host.append(p.value)
        arr = np.ctypeslib.as_array((C.c_uint8 * max(16, int(nbytes))).from_address(p.value))
        return p.value, arr[:int(nbytes)]

    def ring(self, rate: int, tb: int, factor: int, n_streams: int, delay: int = 0,
             payload: bytes | None = None):
        r = C.c_void_p()
        pay = None
        if payload is not None:
            pay = (C.c_uint8 * len(payload)).from_buffer_copy(payload)
        _lib.check(self.lib.pb_ring_create(rate, tb, delay, factor, n_streams, pay, C.byref(r)),
                   "pb_ring_create")
        self.rings.append(r.value)
        data, stride, ctr = C.c_void_p(), C.c_int64(), C.c_void_p()
        _lib.check(self.lib.pb_ring_storage(r, C.byref(data), C.byref(stride), C.byref(ctr)))
        return r.value, data.value, stride.value, ctr.value

    def upload(self, arr: np.ndarray) -> int:
        arr = np.ascontiguousarray(arr)
        p = self.malloc(arr.nbytes, zero=False)
        _lib.check(self.lib.pb_memcpy_h2d(p, arr.ctypes.data, arr.nbytes, None), "pb_memcpy_h2d")
        return p

    def close(self):
        lib = self.lib
        lib.pb_device_sync()
        for r in self.rings:
            lib.pb_ring_destroy(r)
        for p in self.dev:
            lib.pb_free(p)
        for p in self.host:
            lib.pb_host_free(p)
        self.rings, self.dev, self.host = [], [], []


def _default_hashers() -> int:
    """Hashing threads of the pipelined run: this process's share of the host
    cores (torchrun's LOCAL_WORLD_SIZE processes per host) minus one for the
    orchestrating thread, at most 16 (tools/e2e_probe2.py: 15 threads on 16
    cores beat 16)."""
    share = (os.cpu_count() or 16) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    return max(1, min(16, share - 1))


@dataclass
class _Storage:
    """Where a FIFO's spans live (its own ring or an alias of another's)."""

    data: int
    stream_stride: int
    span: int
    slots: int
    base: int          # device int64* (the owner's writes counter row)
    index_cond: int
    owner: str


def _behaviors_for(plan: ExecPlan, overrides, n_streams: int) -> list[dict[str, ActorBehavior]]:
    """One behaviour instance per (stream, actor), as the reference creates one
    per actor (runtime.py:336-341).  An override may be a single object (one
    stream), a sequence with one object per stream, or a zero-arg factory."""
    out = []
    for s in range(n_streams):
        d = {}
        for a in plan.graph.actors:
            ov = overrides.get(a.id) if overrides else None
            if ov is None:
                d[a.id] = resolve(a.behavior)
            elif isinstance(ov, (list, tuple)):
                d[a.id] = ov[s]
            elif isinstance(ov, type) or (callable(ov) and not hasattr(ov, "fire")):
                d[a.id] = ov()
            else:
                if n_streams > 1 and not is_device(ov):
                    raise ValueError(f"behaviour override for {a.id} must be a factory or a "
                                     "per-stream sequence when running several streams")
                d[a.id] = ov
        out.append(d)
    return out


class DeviceRuntime:
    """An admitted graph bound to device rings for `n_streams` replicas."""

    def __init__(self, graph, behaviors: Mapping | None = None,
                 config: RuntimeConfig | None = None, n_streams: int = 1,
                 seeds: Sequence[int | None] | None = None,
                 sources: Mapping[str, Sequence] | None = None):
        self.config = config = config or RuntimeConfig()
        self.graph: Graph = as_graph(graph)
        self.n_streams = S = int(n_streams)
        self.plan = admit(self.graph, int(config.c_factor))
        self.epoch = max(1, min(int(config.epoch), max(1, int(config.source_firings))))
        if self.plan.epoch_cap is not None:   # delayed cycles (plan.admit)
            self.epoch = min(self.epoch, self.plan.epoch_cap)
        self.C = max(int(config.c_factor), self.epoch, 2)
        self.unbounded = sorted(a for a, e in self.plan.extra.items() if e is None)
        if self.unbounded and config.timeout_ms is None:
            raise UnsupportedGraph(f"actors {self.unbounded} fire forever (a cycle no source "
                                   "feeds, test_runtime.py:224-235); set RuntimeConfig.timeout_ms")
        self.analysis = self.plan.admission
        self.seeds = list(seeds) if seeds is not None else [config.seed] * S
        if len(self.seeds) != S:
            raise ValueError("one seed per stream expected")
        self.sources = dict(sources or {})
        self.behaviors = _behaviors_for(self.plan, behaviors, S)
        g, plan = self.graph, self.plan
        lib = _lib.load()
        if _lib.device_count() < 1:
            raise DeviceUnavailable("no CUDA device visible; the B200 executor has no CPU "
                                    "fallback")
        _lib.check(lib.pb_set_device(int(config.device)), "pb_set_device")
        self.lib = lib
        self.mem = _Dev()
        st = C.c_void_p()
        _lib.check(lib.pb_stream_create(C.byref(st)), "pb_stream_create")
        self.stream = st.value
        for name in ("copy_in", "copy_out"):
            _lib.check(lib.pb_stream_create(C.byref(st)), "pb_stream_create")
            setattr(self, name, st.value)
        self._events: list[int] = []
        self._registered: list[int] = []      # caller buffers page-locked in place
        self._direct: dict[str, tuple | None] = {}

        # Actors between sources and sinks whose behaviour is Python code run
        # that code on the host, per firing, through the plugin API
        # (runtime.py:336-341 overrides): "host" -- a behaviour with no device
        # kernel (a user-registered behaviour, or an override of a built-in
        # one), whose firings read their input spans from the device rings and
        # write their outputs back; "observe" -- a subclass of a device
        # behaviour that overrides fire (the FirBranch-recorder pattern of
        # SURVEY 8(c3b)): the device kernel computes the firing and the Python
        # fire then sees the inputs and the computed outputs (its writes to
        # ctx.outputs are copied back).  The device math itself never runs on
        # the host.
        self.host_fired: dict[str, str] = {}
        for a in g.actors:
            role = plan.roles[a.id]
            b = self.behaviors[0][a.id]
            if role in ("device", "dynamic"):
                if not is_device(b):
                    self.host_fired[a.id] = "host"
                elif type(b).fire is not DeviceBehavior.fire:
                    self.host_fired[a.id] = "observe"
            if role in ("source", "config", "sink") and is_device(b):
                raise UnsupportedGraph(f"actor {a.id} ({role}) needs a host behaviour")

        self.fir_math = _lib.PB_FIR_EXACT if config.exact else _lib.PB_FIR_MERGED
        self.conv_math = _lib.PB_CONV_I8 if config.conv_i8 else _lib.PB_CONV_BF16X3
        if os.environ.get("PB_CONV_MATH") in ("bf16x3", "i8"):
            self.conv_math = (_lib.PB_CONV_I8 if os.environ["PB_CONV_MATH"] == "i8"
                              else _lib.PB_CONV_BF16X3)
        if config.exact and os.environ.get("PB_FIR_MATH") == "paired":
            self.fir_math = _lib.PB_FIR_EXACT_PAIRED
        self.banks = find_filter_banks(plan, self.behaviors[0]) if config.fuse else []
        # a region with a host-fired member keeps its channels materialised
        self.banks = [grp for grp in self.banks
                      if not ({grp.router, grp.combiner, *grp.branches} & set(self.host_fired))]
        # matmul chains (bypass.py's l1 -> l2 -> l3): one launch per chain at
        # its head, the link channels stay in registers
        self.chains = [c for c in find_matmul_chains(plan, self.behaviors[0])
                       if not (set(c.actors) & set(self.host_fired))] if config.fuse else []
        # motion regions (motion.py's blur -> detect -> clean): one launch at
        # the blur, f_cur / f_mask in shared memory, the delayed f_prev a ring
        self.motions = [m for m in find_motion_regions(plan, self.behaviors[0])
                        if not ({m.blur, m.detect, m.clean} & set(self.host_fired))] \
            if config.fuse else []
        # a chain between a route and a path_merge whose other input is the
        # route's other output: the whole bypass region as one launch
        self.bypasses = [b for b in find_bypass_regions(plan, self.behaviors[0], self.chains)
                         if not ({b.route, b.merge} & set(self.host_fired))]
        self.fused_actors = {a for grp in self.banks for a in [grp.router, *grp.branches]}
        self.fused_actors |= {a for c in self.chains for a in c.actors[1:]}
        self.fused_actors |= {b.merge for b in self.bypasses}
        self.fused_actors |= {a for m in self.motions for a in (m.detect, m.clean)}
        self.virtual = {fid for grp in self.banks for fid in grp.internal_fifos}
        self.virtual |= {fid for c in self.chains for fid in c.internal_fifos}
        self.virtual |= {b.chain_out for b in self.bypasses}
        self.virtual |= {fid for m in self.motions for fid in (m.cur_fifo, m.mask_fifo)}
        self._allocate()
        self.launches, self.fir_groups = self._build_launches()
        self._build_tables()

        self._drain = None            # drain-phase launches, built on first use
        self._cond_now: dict[str, int] = {}   # condition overrides while draining
        self.eq1_host = 0             # Eq. 1 checks counted without a launch
        self.launches_per_epoch = 0

    # ------------------------------------------------------------- allocation

    def _allocate(self):
        g, plan, S, C_ = self.graph, self.plan, self.n_streams, self.C
        m = self.mem
        n_drain = len({e for e in plan.extra.values() if e})
        n_cond = max(1, len(plan.conds), n_drain)
        self.res_slots = n_cond
        cap = self.epoch
        self.res_act = m.malloc(n_cond * S * cap)
        self.res_prefix = m.malloc(4 * n_cond * S * cap)
        self.res_count = m.malloc(4 * n_cond * S)
        self.res_wl = m.malloc(4 * n_cond * S * cap)
        self.eq1_ctr = m.malloc(16)
        self.err_flag = m.malloc(16)
        self.cap = cap

        self.counters: dict[str, int] = {}
        self.storage: dict[str, _Storage] = {}
        self.delay_chunks: dict[str, int] = {}   # FIFOs with initial delay tokens
        route_alias: dict[str, str] = {}
        for a in g.actors:
            b = self.behaviors[0][a.id]
            if getattr(b, "kernel", "") == "route" and a.id not in self.fused_actors and \
                    a.id not in self.host_fired:
                (pin,) = a.data_inputs
                src = g.fifo_into(PortRef(a.id, pin.id))
                span = src.rate * src.token_bytes
                for p in a.output_ports:
                    for f in g.fifos_from(PortRef(a.id, p.id)):
                        if f.rate * f.token_bytes == span:
                            route_alias[f.id] = src.id
        # storage owners first (topological order keeps owners ahead of aliases)
        for aid in plan.order:
            a = g.actor(aid)
            for p in sorted(a.output_ports, key=lambda p: p.id):
                if p.kind == CONTROL_OUT:
                    continue
                fifos = sorted(g.fifos_from(PortRef(aid, p.id)), key=lambda f: f.id)
                first = None
                for f in fifos:
                    span = f.rate * f.token_bytes
                    if f.delay:
                        # own ring, delay/rate chunks longer; the producer writes
                        # that many chunks ahead (pb_span_ref.offset) and the
                        # consumer first reads the delay payload (fifos.py:155-161)
                        d = f.delay // f.rate
                        _, data, stride, ctr = m.ring(f.rate, f.token_bytes, C_ + d, S,
                                                      delay=f.delay, payload=f.delay_payload)
                        self.counters[f.id] = ctr
                        self.storage[f.id] = _Storage(data, stride, span, C_ + d, ctr,
                                                      plan.fifo_cond[f.id], f.id)
                        self.delay_chunks[f.id] = d
                        continue
                    if f.id in self.virtual:
                        self.counters[f.id] = m.malloc(8 * 4 * S)
                        continue
                    if f.id in route_alias:
                        o = self.storage[route_alias[f.id]]
                        self.storage[f.id] = o
                        self.counters[f.id] = m.malloc(8 * 4 * S)
                        continue
                    if first is not None and first.span == span:
                        self.storage[f.id] = first
                        self.counters[f.id] = m.malloc(8 * 4 * S)
                        continue
                    _, data, stride, ctr = m.ring(f.rate, f.token_bytes, C_, S)
                    self.counters[f.id] = ctr
                    st = _Storage(data, stride, span, C_, ctr, plan.fifo_cond[f.id], f.id)
                    self.storage[f.id] = st
                    if first is None:
                        first = st
        # control tokens: one device array per control output port
        self.ctl_ports: list[PortRef] = []
        self.ctl_dev: dict[PortRef, int] = {}
        self.ctl_stride: dict[PortRef, int] = {}
        self.ctl_host: dict[PortRef, tuple[int, np.ndarray]] = {}
        self.policy_state: dict[PortRef, C.Array] = {}
        for a in g.actors:
            for p in a.output_ports:
                if p.kind != CONTROL_OUT:
                    continue
                ref = PortRef(a.id, p.id)
                fifos = g.fifos_from(ref)
                stride = max(f.token_bytes for f in fifos)
                self.ctl_ports.append(ref)
                self.ctl_stride[ref] = stride
                self.ctl_dev[ref] = m.malloc(S * C_ * stride)
                self.ctl_host[ref] = m.pinned(S * self.epoch * stride)
                self.policy_state[ref] = (C.c_uint8 * (_lib.PB_POLICY_STATE_BYTES * S))()
                for f in fifos:
                    self.counters[f.id] = m.malloc(8 * 4 * S)
        # configuration actors: (actor, control ports, data ports); staging for
        # the data ports' tokens
        self.config_outputs = []
        self.cfg_host: dict[tuple[str, str], tuple[int, np.ndarray]] = {}
        for a in g.actors:
            if plan.roles[a.id] != "config":
                continue
            ports = sorted(a.output_ports, key=lambda p: p.id)
            ctl = [PortRef(a.id, p.id) for p in ports if p.kind == CONTROL_OUT]
            data = [p for p in ports if p.kind != CONTROL_OUT]
            self.config_outputs.append((a.id, ctl, data))
            for p in data:
                self.cfg_host[(a.id, p.id)] = m.pinned(S * self.epoch *
                                                       self._port_span(a.id, p.id))
        # ring counters start with max occupancy = delay (0 here) — zeroed above

        # host staging for sources and sinks
        self.src_host: dict[str, tuple[int, np.ndarray]] = {}
        self.sink_host: dict[str, tuple[int, np.ndarray]] = {}
        for a in g.actors:
            role = plan.roles[a.id]
            if role == "source":
                for p in a.output_ports:
                    f = sorted(g.fifos_from(PortRef(a.id, p.id)), key=lambda f: f.id)[0]
                    key = f"{a.id}.{p.id}"
                    self.src_host[key] = m.pinned(S * self.epoch * f.rate * f.token_bytes)
            elif role == "sink":
                for p in a.input_ports:
                    f = g.fifo_into(PortRef(a.id, p.id))
                    self.sink_host[f.id] = m.pinned(S * self.epoch * f.rate * f.token_bytes)

        # FIR taps and history state
        self.fir_taps: dict[str, int] = {}
        self.fir_state: dict[str, int] = {}
        for a in g.actors:
            b = self.behaviors[0][a.id]
            if getattr(b, "kernel", "") == "fir":
                b.init(a.id, a.params, None)
                taps = np.array(list(b.re) + list(b.im), dtype=np.float32)
                self.fir_taps[a.id] = m.upload(taps)
                self.fir_state[a.id] = m.malloc(S * 2 * 9 * 4)
            elif getattr(b, "kernel", "") == "matmul":
                b.init(a.id, a.params, None)
        # host-fired actors: per data port a device gather/scatter buffer and
        # its pinned host copy, [S][epoch][span]
        self.host_stage: dict[tuple[str, str], tuple[int, int, np.ndarray, int, str]] = {}
        for aid in self.host_fired:
            a = g.actor(aid)
            for p in a.ports:
                if p.kind in (CONTROL_IN, CONTROL_OUT):
                    continue
                ref = PortRef(aid, p.id)
                f = g.fifo_into(ref) if p.direction == "in" else \
                    sorted(g.fifos_from(ref), key=lambda f: f.id)[0]
                span = f.rate * f.token_bytes
                dev = m.malloc(S * self.epoch * span)
                hptr, harr = m.pinned(S * self.epoch * span)
                self.host_stage[(aid, p.id)] = (dev, hptr, harr, span, f.id)
        _lib.check(self.lib.pb_device_sync(), "allocation")

    # ------------------------------------------------------------ span refs

    def _ref(self, fid: str, producer: bool = False) -> _lib.SpanRef:
        """Span addressing of a FIFO; the producer side of a FIFO with initial
        delay tokens writes delay/rate chunks ahead of its consumer."""
        st = self.storage[fid]
        off = self.delay_chunks.get(fid, 0) if producer else 0
        return _lib.SpanRef(st.data, st.stream_stride, st.span, st.base, st.slots,
                            st.index_cond, self.plan.fifo_cond[fid], off)

    def _port_targets(self, aid: str, port: str) -> list[str]:
        """The FIFOs an output port must write: one per distinct storage (a
        broadcast of equal spans aliases the first; delayed FIFOs have their
        own ring)."""
        fifos = sorted(self.graph.fifos_from(PortRef(aid, port)), key=lambda f: f.id)
        seen, out = set(), []
        for f in fifos:
            o = self.storage[f.id].owner if f.id in self.storage else f.id
            key = (o, self.delay_chunks.get(f.id, 0))
            if key not in seen:
                seen.add(key)
                out.append(f.id)
        return out

    def _resolved(self, n_iter: int) -> _lib.Resolved:
        return _lib.Resolved(self.res_act, self.res_prefix, self.res_count, self.res_wl,
                             len(self.plan.conds), self.n_streams, n_iter, self.cap)

    def _fir_actor(self, aid: str, in_fid: str, out_fid: str | None,
                   cond: int | None = None) -> _lib.FirActor:
        out = self._ref(out_fid, producer=True) if out_fid is not None else _lib.SpanRef()
        cond = self.plan.actor_cond[aid] if cond is None else cond
        return _lib.FirActor(self._ref(in_fid), out, self.fir_taps[aid], self.fir_state[aid],
                             cond, 0)

    def _build_launches(self, cond_of=None, only: set[str] | None = None):
        """The epoch's launch list in dependency order.  cond_of(aid) -> the
        condition gating the actor's firings (default: the plan's); `only`
        restricts the list to those actors (the drain phase)."""
        g, plan = self.graph, self.plan
        cond_of = cond_of or plan.actor_cond.__getitem__
        launches: list[tuple] = []
        fir_groups: list[tuple[int, int, int]] = []    # (device array, n, block)
        done: set[str] = set()
        bank_at = {grp.combiner: grp for grp in self.banks}
        chain_at = {c.actors[0]: c for c in self.chains}
        bypass_at = {b.chain.actors[0]: b for b in self.bypasses}
        motion_at = {m.blur: m for m in self.motions}
        # topological depth so independent FIR actors share a launch (the
        # delayed channels inside cycles do not order an epoch's firings)
        depth = {aid: 0 for aid in plan.order}
        for aid in plan.order:
            for fid in plan.data_fifos:
                f = g.fifo(fid)
                if f.src.actor == aid and fid not in plan.loose:
                    depth[f.dst.actor] = max(depth[f.dst.actor], depth[aid] + 1)
        fir_by_level: dict[tuple[int, int], list[str]] = {}
        for aid in plan.order:
            b = self.behaviors[0][aid]
            if only is not None and aid not in only:
                continue
            if getattr(b, "kernel", "") == "fir" and aid not in self.fused_actors:
                a = g.actor(aid)
                fin = g.fifo_into(PortRef(aid, a.input_ports[0].id))
                block = fin.rate * fin.token_bytes // 8
                fir_by_level.setdefault((depth[aid], block), []).append(aid)
        # one launch covers at most PB_MAX_BRANCHES actors
        chunks: dict[tuple, list[str]] = {}
        for (lvl, block), members in fir_by_level.items():
            for c0 in range(0, len(members), _lib.PB_MAX_BRANCHES):
                chunks[(lvl, block, c0)] = members[c0:c0 + _lib.PB_MAX_BRANCHES]
        fir_by_level = {(k[0], k[1], k[2]): v for k, v in chunks.items()}

        # launch in level order (longest-path depth, then plan order): every
        # data edge goes from a lower to a higher level, so a FIR group of one
        # level is launched after all its members' producers and before all
        # their consumers (a plain Kahn order can interleave a member's
        # producer after another member of the same group)
        pos = {aid: k for k, aid in enumerate(plan.order)}
        for aid in sorted(plan.order, key=lambda x: (depth[x], pos[x])):
            if aid in done or aid in self.fused_actors or (only is not None and aid not in only):
                continue
            a = g.actor(aid)
            role = plan.roles[aid]
            if role in ("source", "config", "sink"):
                continue
            b = self.behaviors[0][aid]
            kind = getattr(b, "kernel", "")
            if self.host_fired.get(aid) == "host":
                launches.append(("host", aid))
                done.add(aid)
                continue
            if aid in bank_at:
                grp = bank_at[aid]
                x = g.actor(grp.router)
                fin = g.fifo_into(PortRef(x.id, x.data_inputs[0].id))
                (pout,) = a.output_ports
                fout = sorted(g.fifos_from(PortRef(aid, pout.id)), key=lambda f: f.id)[0]
                arr = (_lib.FirActor * len(grp.branches))()
                for k, bid in enumerate(grp.branches):
                    arr[k] = self._fir_actor(bid, fin.id, None, cond_of(bid))
                dev = self.mem.upload(np.frombuffer(bytes(arr), dtype=np.uint8))
                bank = _lib.FilterBank(self._ref(fin.id), self._ref(fout.id), dev,
                                       len(grp.branches), cond_of(aid),
                                       self.mem.malloc(16), self.fir_math, 0)
                block = fin.rate * fin.token_bytes // 8
                launches.append(("bank", bank, block))
                # (no fir_groups entry: pb_fire_filter_bank carries its branches)
                done.add(aid)
                continue
            if aid in motion_at:
                m = motion_at[aid]
                x = g.actor(m.blur)
                fin = g.fifo_into(PortRef(x.id, x.data_inputs[0].id))
                act = _lib.MotionRegion(self._ref(fin.id), self._ref(m.prev_fifo),
                                        self._ref(m.prev_fifo, producer=True),
                                        self._ref(m.out_fifo, producer=True), m.side,
                                        int(g.actor(m.detect).params.get("threshold", 16)))
                launches.append(("motion_region", act))
                done.update({m.blur, m.detect, m.clean})
                continue
            if aid in bypass_at:
                bp = bypass_at[aid]
                c = bp.chain
                x = g.actor(c.actors[0])
                fin = g.fifo_into(PortRef(x.id, x.data_inputs[0].id))
                w = np.concatenate([np.array(g.actor(m).params["w"], dtype=np.float32)
                                    for m in c.actors])
                mg = g.actor(bp.merge)
                act = _lib.BypassRegion(self._ref(fin.id), self._ref(bp.bypass_fifo),
                                        self._ref(bp.out_fifo, producer=True), self.mem.upload(w),
                                        len(c.actors), plan.fifo_cond[bp.chain_out],
                                        cond_of(bp.merge),
                                        float(np.float32(mg.params.get("marker", 0.5))),
                                        self.err_flag)
                launches.append(("bypass_region", act))
                done.update(c.actors)
                done.add(bp.merge)
                continue
            if aid in chain_at:
                c = chain_at[aid]
                x = g.actor(c.actors[0])
                fin = g.fifo_into(PortRef(x.id, x.data_inputs[0].id))
                y = g.actor(c.actors[-1])
                fout = sorted(g.fifos_from(PortRef(y.id, y.output_ports[0].id)),
                              key=lambda f: f.id)[0]
                w = np.concatenate([np.array(g.actor(m).params["w"], dtype=np.float32)
                                    for m in c.actors])
                act = _lib.MatmulChainActor(self._ref(fin.id), self._ref(fout.id, producer=True),
                                            self.mem.upload(w), 8, len(c.actors), cond_of(aid), 0)
                launches.append(("matmul_chain", act))
                done.update(c.actors)
                continue
            if kind == "fir":
                key = next(k for k, v in fir_by_level.items() if aid in v)
                members = fir_by_level[key]
                arr = (_lib.FirActor * len(members))()
                for k, bid in enumerate(members):
                    ba = g.actor(bid)
                    fi = g.fifo_into(PortRef(bid, ba.input_ports[0].id))
                    fo = sorted(g.fifos_from(PortRef(bid, ba.output_ports[0].id)),
                                key=lambda f: f.id)[0]
                    arr[k] = self._fir_actor(bid, fi.id, fo.id, cond_of(bid))
                dev = self.mem.upload(np.frombuffer(bytes(arr), dtype=np.uint8))
                launches.append(("fir", dev, len(members), key[1]))
                fir_groups.append((dev, len(members), key[1]))
                done.update(members)
                for bid in members:
                    if bid in self.host_fired:
                        launches.append(("host", bid))
                continue
            ins = sorted(a.data_inputs, key=lambda p: p.id)
            outs = sorted(a.output_ports, key=lambda p: p.id)
            in_f = [g.fifo_into(PortRef(aid, p.id)).id for p in ins]
            out_f = [sorted(g.fifos_from(PortRef(aid, p.id)), key=lambda f: f.id)[0].id
                     for p in outs]
            targets = {p.id: self._port_targets(aid, p.id) for p in outs}
            if kind not in ("image", "bytes", "route") and \
                    any(len(t) > 1 for t in targets.values()):
                raise UnsupportedGraph(f"{aid}: an output port broadcasts to a delayed and an "
                                       f"undelayed channel; only image and byte actors write "
                                       f"both")
            if kind == "route":
                if all(self.storage[f].owner == self.storage[in_f[0]].owner for f in out_f):
                    done.add(aid)          # aliased: no bytes move
                    continue
                kind = "bytes"
            if kind == "branch_sum":
                if len(in_f) > _lib.PB_MAX_PORTS:
                    raise UnsupportedGraph(f"{aid}: more than {_lib.PB_MAX_PORTS} inputs")
                act = _lib.SumActor()
                for k, fid in enumerate(in_f):
                    act.in_[k] = self._ref(fid)
                act.n_in = len(in_f)
                act.out = self._ref(out_f[0], producer=True)
                act.cond = cond_of(aid)
                f0 = g.fifo(out_f[0])
                launches.append(("sum", act, f0.rate * f0.token_bytes // 8))
            elif kind == "bytes":
                spans_in = [g.fifo(fid).rate * g.fifo(fid).token_bytes for fid in in_f]
                spans_out = [g.fifo(fid).rate * g.fifo(fid).token_bytes for fid in out_f]
                if spans_in and spans_out and min(spans_in) < max(spans_out):
                    # the reference's byte actors index every input over the
                    # output span (behavior.py:153-199) and fail on a shorter one
                    raise UnsupportedGraph(f"{aid}: an input span ({min(spans_in)} B) is shorter "
                                           f"than an output span ({max(spans_out)} B)")
                act = _lib.BytesActor()
                for k, fid in enumerate(in_f):
                    act.in_[k] = self._ref(fid)
                outs_all = [fid for p in outs for fid in targets[p.id]]
                if len(outs_all) > _lib.PB_MAX_PORTS or len(in_f) > _lib.PB_MAX_PORTS:
                    raise UnsupportedGraph(f"{aid}: more than {_lib.PB_MAX_PORTS} ports")
                for k, fid in enumerate(outs_all):
                    act.out[k] = self._ref(fid, producer=True)
                act.n_in, act.n_out = len(in_f), len(outs_all)
                act.offset = int(a.params.get("offset", 0)) if b.registered_name == "add_mod" \
                    else 0
                act.cond = cond_of(aid)
                launches.append(("bytes", act))
            elif kind == "matmul":
                w = np.array(a.params["w"], dtype=np.float32)
                n = int(round(len(w) ** 0.5))
                act = _lib.MatmulActor(self._ref(in_f[0]), self._ref(out_f[0], producer=True),
                                       self.mem.upload(w), n, cond_of(aid))
                launches.append(("matmul", act))
            elif kind == "path_merge":
                act = _lib.PathMergeActor()
                bypass = a.params.get("bypass_port", "")
                for k, fid in enumerate(in_f):
                    act.in_[k] = self._ref(fid)
                act.n_in = len(in_f)
                act.bypass_index = [p.id for p in ins].index(bypass) if bypass in \
                    [p.id for p in ins] else -1
                act.marker = float(np.float32(a.params.get("marker", 0.5)))
                act.cond = cond_of(aid)
                act.error_flag = self.err_flag
                act.out = self._ref(out_f[0], producer=True)
                launches.append(("path_merge", act, aid))
            elif kind == "image":
                act = _lib.ImageActor()
                names = [p.id for p in ins]
                if b.op == _lib.PB_IMG_DIFF:
                    if set(names) != {"cur", "prev"}:
                        raise UnsupportedGraph(f"{aid}: frame_diff_threshold needs ports cur/prev")
                    order = [in_f[names.index("cur")], in_f[names.index("prev")]]
                else:
                    if len(in_f) != 1:
                        raise UnsupportedGraph(f"{aid}: one data input expected")
                    order = in_f
                for k, fid in enumerate(order):
                    act.in_[k] = self._ref(fid)
                outs_all = [fid for p in outs for fid in targets[p.id]]
                if len(outs_all) > _lib.PB_MAX_PORTS:
                    raise UnsupportedGraph(f"{aid}: more than {_lib.PB_MAX_PORTS} outputs")
                for k, fid in enumerate(outs_all):
                    act.out[k] = self._ref(fid, producer=True)
                act.n_out = len(outs_all)
                tb = g.fifo(in_f[0]).token_bytes * g.fifo(in_f[0]).rate
                side = int(round(tb ** 0.5))
                if side * side != tb or any(g.fifo(f).rate * g.fifo(f).token_bytes != tb
                                            for f in in_f + outs_all):
                    raise UnsupportedGraph(f"{aid}: image actors take square 8-bit frames of "
                                           "one size on every port")
                act.op, act.side = b.op, side
                act.threshold = int(a.params.get("threshold", 16))
                act.cond = cond_of(aid)
                launches.append(("image", act))
            elif kind == "conv":
                from .cnn_weights import conv_device_layout, conv_device_layout_i8
                b.init(aid, a.params, None)
                fi = g.fifo(in_f[0])
                if fi.token_bytes != b.h * b.w * b.cin * 4:
                    raise UnsupportedGraph(f"{aid}: token is not one {b.h}x{b.w}x{b.cin} frame")
                # int8 limbs: Cin 32 (the row kernel's layer 2); bf16x3 otherwise
                w_i8 = (self.mem.upload(conv_device_layout_i8(b.weights, b.cin))
                        if b.cin == 32 else None)
                act = _lib.ConvActor(self._ref(in_f[0]), self._ref(out_f[0], producer=True),
                                     self.mem.upload(conv_device_layout(b.weights, b.cin)),
                                     self.mem.upload(b.bias), fi.rate, b.h, b.w, b.cin,
                                     b.cout, b.pad, cond_of(aid), 0, self.conv_math, w_i8,
                                     None, None)
                launches.append(("conv", act, aid))
            elif kind == "dense":
                b.init(aid, a.params, None)
                fi = g.fifo(in_f[0])
                from .cnn_weights import dense_device_layout
                act = _lib.DenseActor(self._ref(in_f[0]), self._ref(out_f[0], producer=True),
                                      self.mem.upload(dense_device_layout(b.weights)),
                                      self.mem.upload(b.bias),
                                      fi.rate, b.nin, b.nout, cond_of(aid))
                launches.append(("dense", act))
            elif kind == "classify":
                b.init(aid, a.params, None)
                bypass = a.params.get("bypass_port", "")
                names = [p.id for p in ins]
                if len(in_f) != 2 or bypass not in names:
                    raise UnsupportedGraph(f"{aid}: classify_merge needs a chain and a bypass input")
                chain_f = in_f[1 - names.index(bypass)]
                bypass_f = in_f[names.index(bypass)]
                act = _lib.ClassifyActor(
                    self._ref(chain_f), self._ref(bypass_f), self._ref(out_f[0], producer=True),
                    self.mem.upload(b.w4), self.mem.upload(b.b4), self.mem.upload(b.w5),
                    self.mem.upload(b.b5), g.fifo(out_f[0]).rate, b.nin, b.nhid, b.nout,
                    float(np.float32(a.params.get("marker", -1.0))), cond_of(aid),
                    self.err_flag)
                launches.append(("classify", act, aid))
            else:
                raise UnsupportedGraph(f"actor {aid}: no device kernel for behaviour "
                                       f"{a.behavior!r}")
            done.add(aid)
            if aid in self.host_fired:
                launches.append(("host", aid))

        self._wire_conv_scales(launches, cond_of)
        return launches, fir_groups

    def _wire_conv_scales(self, launches, cond_of) -> None:
        """A conv actor fed straight by another conv actor (same condition, so
        both launches see the same live firings in the same order; no delay)
        reads its int8 quantisation scales -- every input frame's max |x| --
        from the producer's epilogue (pb_conv_actor.absmax_out / absmax_in);
        any other conv input gets them from a pre-pass over its frames."""
        g = self.graph
        convs = {item[2]: item[1] for item in launches if item[0] == "conv"}
        for aid, act in convs.items():
            a = g.actor(aid)
            ins = [p for p in a.data_inputs]
            if len(ins) != 1:
                continue
            f = g.fifo_into(PortRef(aid, ins[0].id))
            src = f.src.actor
            if src not in convs or f.delay or cond_of(src) != cond_of(aid) \
                    or src in self.host_fired or aid in self.host_fired:
                continue
            prod = convs[src]
            if prod.frames != act.frames:
                continue
            if not prod.absmax_out:
                prod.absmax_out = self.mem.malloc(4 * self.n_streams * self.cap * prod.frames)
            act.absmax_in = prod.absmax_out

    def set_conv_math(self, math: int) -> None:
        """Switch the conv arithmetic (_lib.PB_CONV_I8: int8 limbs on the
        tensor cores for Cin 32, the default; _lib.PB_CONV_BF16X3: three bf16
        products per useful one) of every conv launch of this runtime."""
        self.conv_math = int(math)
        drain = getattr(self, "_drain", None)
        for lst in [self.launches] + ([drain[0]] if drain else []):
            for item in lst:
                if item[0] == "conv":
                    item[1].math = self.conv_math

    def _build_tables(self):
        """Ring advance (every FIFO; the drain phase: the always-active ones)
        and Eq. 1 tables."""
        g, plan = self.graph, self.plan
        # bulk ring advance for every FIFO
        adv = []
        for f in g.fifos:
            adv.append(_lib.RingAdvance(self.counters[f.id], plan.fifo_cond[f.id], f.rate,
                                        f.delay, 0))
        self.advance = (_lib.RingAdvance * len(adv))(*adv)
        dadv = [r for r, f in zip(adv, g.fifos) if plan.fifo_cond[f.id] == ALWAYS]
        self.drain_advance = (_lib.RingAdvance * max(1, len(dadv)))(*dadv)
        self.n_drain_advance = len(dadv)
        # Eq. 1 recheck (runtime.py:195-220) per DRP: the port's own control
        # element vs the condition that moved its channel's tokens.  Where both
        # are the same condition (every DRP whose channel the executor gates by
        # that DRP's own control entry) the check cannot fail and counts one per
        # firing of the (always-firing) dynamic actor: counted on the host, no
        # launch.  The others run on the device (pb_epoch_close / pb_eq1_check).
        eq = [_lib.Eq1Port(own, moved, ALWAYS, 0) for (_, _, own, moved) in plan.eq1_ports
              if own != moved]
        self.n_eq1_static = sum(1 for (_, _, own, moved) in plan.eq1_ports if own == moved)
        self.eq1 = (_lib.Eq1Port * max(1, len(eq)))(*eq)
        self.n_eq1 = len(eq)

    # -------------------------------------------------------------- epochs

    def _conditions(self, it0: int) -> C.Array:
        arr = (_lib.Condition * max(1, len(self.plan.conds)))()
        for k, c in enumerate(self.plan.conds):
            stride = self.ctl_stride[c.ctl]
            arr[k] = _lib.Condition(self.ctl_dev[c.ctl], self.C * stride, stride,
                                    c.element - 1, self.C, it0 % self.C)
        return arr

    def _h2d_chunks(self, dev: int, stride: int, span: int, host: int, E: int, first: int,
                    host_pitch: int | None = None, stream: int | None = None,
                    slots: int | None = None):
        """host rows [S][E spans] (row pitch host_pitch) -> device ring chunks
        (first + n) % slots of every stream (slots: C, or C + delay/rate for a
        channel with initial delay tokens)."""
        lib, S = self.lib, self.n_streams
        C_ = self.C if slots is None else slots
        st = self.stream if stream is None else stream
        hp = E * span if host_pitch is None else host_pitch
        a = first % C_
        n1 = min(E, C_ - a)
        if n1 == C_ and stride == C_ * span and hp == E * span:
            _lib.check(lib.pb_memcpy_h2d(dev, host, S * E * span, st))
            return
        _lib.check(lib.pb_memcpy_2d(dev + a * span, stride, host, hp, n1 * span, S, 1, st))
        if n1 < E:
            _lib.check(lib.pb_memcpy_2d(dev, stride, host + n1 * span, hp, (E - n1) * span,
                                        S, 1, st))

    def _d2h_chunks(self, dev: int, stride: int, span: int, host: int, E: int, first: int,
                    host_pitch: int | None = None, stream: int | None = None,
                    slots: int | None = None):
        lib, S = self.lib, self.n_streams
        C_ = self.C if slots is None else slots
        st = self.stream if stream is None else stream
        hp = E * span if host_pitch is None else host_pitch
        a = first % C_
        n1 = min(E, C_ - a)
        _lib.check(lib.pb_memcpy_2d(host, hp, dev + a * span, stride, n1 * span, S, 2, st))
        if n1 < E:
            _lib.check(lib.pb_memcpy_2d(host + n1 * span, hp, dev, stride,
                                        (E - n1) * span, S, 2, st))

    def source_staging(self, actor: str, port: str | None = None) -> np.ndarray:
        """Pinned host buffer [S][epoch][span] a source's spans are copied from;
        fill it directly and pass prestaged=True to skip the host-side copy."""
        a = self.graph.actor(actor)
        pid = port or sorted(a.output_ports, key=lambda p: p.id)[0].id
        f = sorted(self.graph.fifos_from(PortRef(actor, pid)), key=lambda f: f.id)[0]
        span = f.rate * f.token_bytes
        return self.src_host[f"{actor}.{pid}"][1][:self.n_streams * self.epoch * span].reshape(
            self.n_streams, self.epoch, span)

    def _port_span(self, aid: str, pid: str) -> int:
        f = sorted(self.graph.fifos_from(PortRef(aid, pid)), key=lambda f: f.id)[0]
        return f.rate * f.token_bytes

    def _source_bytes(self, aid: str, s: int) -> np.ndarray:
        return np.frombuffer(memoryview(self.sources[aid][s]).cast("B"), dtype=np.uint8)

    def _direct_source(self, aid: str, n_iter: int) -> tuple[int, int] | None:
        """(address of stream 0's bytes, pitch between streams) when the
        caller's `sources=` buffers of the single-port source `aid` can feed
        the rings by DMA in place: one C-contiguous buffer per stream holding
        at least n_iter spans, at a uniform pitch (the rows of one [S, ...]
        array, or a single stream).  The range is page-locked on first use
        (pb_host_register) and stays registered until close(); the runtime
        keeps the buffers referenced.  None -> copy through pinned staging."""
        if aid not in self.sources or len(self.graph.actor(aid).output_ports) != 1 or \
                (aid in self._direct and self._direct[aid] is None):
            return None
        span = self._port_span(aid, self.graph.actor(aid).output_ports[0].id)
        need = n_iter * span
        bufs = self.sources[aid]
        ptrs = []
        for obj in bufs:
            if obj is None:
                return None
            try:
                mv = memoryview(obj)
            except TypeError:
                return None
            if not mv.c_contiguous or mv.nbytes < need:
                return None
            ptrs.append(np.frombuffer(mv.cast("B") if mv.format != "B" or mv.ndim != 1 else mv,
                                      dtype=np.uint8).__array_interface__["data"][0])
        if not ptrs:
            return None
        full = min(memoryview(o).nbytes for o in bufs)
        pitch = full if len(ptrs) == 1 else ptrs[1] - ptrs[0]
        if len(ptrs) > 1 and (pitch < full or
                              any(q != ptrs[0] + k * pitch for k, q in enumerate(ptrs))):
            return None
        key = (ptrs[0], pitch, len(ptrs), full)
        if self._direct.get(aid) != key:
            nbytes = (len(ptrs) - 1) * pitch + full
            rc = self.lib.pb_host_register(ptrs[0], nbytes)
            if rc < 0:
                _lib.error_text()       # clear; the staging path still works
                self._direct[aid] = None
                return None
            if rc == 0:
                self._registered.append(ptrs[0])
            self._direct[aid] = key
        return ptrs[0], pitch

    def _source_h2d(self, aid: str, pid: str, host: int, E: int, it0: int,
                    host_pitch: int | None = None) -> None:
        """A host producer's E spans per stream -> every ring its port feeds
        (a broadcast of equal spans shares one; a channel with initial delay
        tokens has its own, written delay/rate chunks ahead)."""
        for fid in self._port_targets(aid, pid):
            st = self.storage[fid]
            self._h2d_chunks(st.data, st.stream_stride, st.span, host, E,
                             it0 + self.delay_chunks.get(fid, 0), host_pitch=host_pitch,
                             slots=st.slots)

    def stage_sources(self, it0: int, E: int, prestaged: bool = False):
        """Host sources produce E spans per stream (runtime.py:123-124 stops
        them after source_firings) and copy them into the device rings."""
        g, S = self.graph, self.n_streams
        for a in g.actors:
            if self.plan.roles[a.id] != "source":
                continue
            ports = sorted(a.output_ports, key=lambda p: p.id)
            if prestaged:
                for p in ports:
                    self._source_h2d(a.id, p.id, self.src_host[f"{a.id}.{p.id}"][0], E, it0)
                continue
            for p in ports:
                f = sorted(g.fifos_from(PortRef(a.id, p.id)), key=lambda f: f.id)[0]
                span = f.rate * f.token_bytes
                hptr, harr = self.src_host[f"{a.id}.{p.id}"]
                buf = harr[:S * E * span].reshape(S, E, span)
                if a.id in self.sources:
                    direct = self._direct_source(a.id, it0 + E) if len(ports) == 1 else None
                    if direct is not None:
                        # DMA from the caller's page-locked buffers in place
                        self._source_h2d(a.id, p.id, direct[0] + it0 * span, E, it0,
                                         host_pitch=direct[1])
                        continue
                    # FileSource order (behavior.py:132-140): per firing, the
                    # ports in sorted order each take their span's bytes
                    spans = [self._port_span(a.id, q.id) for q in ports]
                    T, o = sum(spans), sum(spans[:ports.index(p)])
                    for s in range(S):
                        data = self._source_bytes(a.id, s)
                        lo = it0 * T
                        chunk = data[lo:lo + E * T]
                        if chunk.size < E * T:
                            raise ActorPanic(a.id, EOFError(
                                f"{a.id}: input exhausted at byte {lo + chunk.size}"))
                        buf[s] = chunk.reshape(E, T)[:, o:o + span]
                elif len(ports) == 1 and type(self.behaviors[0][a.id]) is FileSource:
                    for s in range(S):
                        b = self.behaviors[s][a.id]
                        try:
                            view = b.take(a.id, E * span)
                        except EOFError as e:
                            raise ActorPanic(a.id, e) from e
                        buf[s] = np.frombuffer(view, dtype=np.uint8).reshape(E, span)
                else:
                    continue
                self._source_h2d(a.id, p.id, hptr, E, it0)
            if a.id in self.sources or (len(ports) == 1 and
                                        type(self.behaviors[0][a.id]) is FileSource):
                continue
            # generic host source: fire per iteration through the plugin API
            views = {}
            for p in ports:
                f = sorted(g.fifos_from(PortRef(a.id, p.id)), key=lambda f: f.id)[0]
                views[p.id] = (f, self.src_host[f"{a.id}.{p.id}"])
            for s in range(S):
                b = self.behaviors[s][a.id]
                seed = actor_seed(self.seeds[s], a.id)
                for n in range(E):
                    outs = {}
                    for pid, (f, (hp, harr)) in views.items():
                        span = f.rate * f.token_bytes
                        off = (s * E + n) * span
                        outs[pid] = memoryview(harr[off:off + span])
                    ctx = FireContext(a.id, it0 + n, {p.id: p.rate for p in a.ports}, {}, outs,
                                      a.params, seed, None)
                    try:
                        b.fire(ctx)
                    except Exception as e:  # noqa: BLE001
                        raise ActorPanic(a.id, e) from e
            for pid, (f, (hp, harr)) in views.items():
                self._source_h2d(a.id, pid, hp, E, it0)

    def stage_control(self, it0: int, E: int):
        """Configuration actors emit E tokens per stream (behavior.py:212-218):
        each actor fires ONCE per iteration and its token goes to every output
        port -- every control port (a device token array per port, aliased by
        the port's control FIFOs) and every data port (the token padded with
        zeros to the span, written into the port's rings)."""
        g, S = self.graph, self.n_streams
        for aid, ctl_refs, data_ports in self.config_outputs:
            a = g.actor(aid)
            b0 = self.behaviors[0][aid]
            kind = native_policy_kind(b0)
            lead = ctl_refs[0]
            stride0 = self.ctl_stride[lead]
            tok = self.ctl_host[lead][1][:S * E * stride0].reshape(S, E, stride0)
            min_tb = min(f.token_bytes for r in ctl_refs for f in g.fifos_from(r))
            if kind is not None:
                try:
                    length = int(a.params["length"])
                    param = b0.native_param(a.params)
                    if length > min_tb:
                        raise ValueError(f"{length} control elements exceed {min_tb} bytes")
                except Exception as e:  # noqa: BLE001
                    raise ActorPanic(aid, e) from e
                rc = self.lib.pb_policy_tokens_streams(
                    C.addressof(self.policy_state[lead]), S, kind, length, param, it0, E,
                    self.ctl_host[lead][0], stride0, int(self.config.host_threads))
                if rc != _lib.PB_OK:
                    raise ActorPanic(aid, ValueError(_lib.error_text()))
                ports_out = None
            else:
                # the plugin API: one fire per iteration with a distinct span per
                # output port (inactive bytes beyond min_tb stay zero)
                ports_out = {}
                for p in a.output_ports:
                    ref = PortRef(aid, p.id)
                    if p.kind == CONTROL_OUT:
                        st = self.ctl_stride[ref]
                        ports_out[p.id] = (min(f.token_bytes for f in g.fifos_from(ref)),
                                           self.ctl_host[ref][1][:S * E * st].reshape(S, E, st))
                    else:
                        sp = self._port_span(aid, p.id)
                        ports_out[p.id] = (sp, self.cfg_host[(aid, p.id)][1][:S * E * sp]
                                           .reshape(S, E, sp))
                for _, arr in ports_out.values():
                    arr[:] = 0
                for s in range(S):
                    b = self.behaviors[s][aid]
                    seed = actor_seed(self.seeds[s], aid)
                    for n in range(E):
                        outs = {pid: memoryview(arr[s, n, :w]) for pid, (w, arr) in
                                ports_out.items()}
                        ctx = FireContext(aid, it0 + n, {p.id: p.rate for p in a.ports}, {},
                                          outs, a.params, seed, None)
                        try:
                            b.fire(ctx)
                        except Exception as e:  # noqa: BLE001
                            raise ActorPanic(aid, e) from e
            if ports_out is None:
                # native generator: the lead port's tokens, copied to the other ports
                for ref in ctl_refs[1:]:
                    st = self.ctl_stride[ref]
                    arr = self.ctl_host[ref][1][:S * E * st].reshape(S, E, st)
                    w = min(st, stride0)
                    arr[:, :, :w] = tok[:, :, :w]
                    arr[:, :, w:] = 0
                for p in data_ports:
                    sp = self._port_span(aid, p.id)
                    arr = self.cfg_host[(aid, p.id)][1][:S * E * sp].reshape(S, E, sp)
                    w = min(sp, stride0)
                    arr[:, :, :w] = tok[:, :, :w]
                    arr[:, :, w:] = 0
            for ref in ctl_refs:
                st = self.ctl_stride[ref]
                self._h2d_chunks(self.ctl_dev[ref], self.C * st, st, self.ctl_host[ref][0], E,
                                 it0)
            for p in data_ports:
                sp = self._port_span(aid, p.id)
                for fid in self._port_targets(aid, p.id):
                    st = self.storage[fid]
                    self._h2d_chunks(st.data, st.stream_stride, sp, self.cfg_host[(aid, p.id)][0],
                                     E, it0 + self.delay_chunks.get(fid, 0), slots=st.slots)

    def fire_epoch(self, it0: int, E: int, hook=None) -> int:
        """Device work of one epoch (inputs already resident); returns launches.
        hook(kind, phase) is called around every actor launch (phase 'pre' /
        'post') so callers can record events on self.stream."""
        lib, st = self.lib, self.stream
        n0 = lib.pb_launch_count()
        res = self._resolved(E)
        if self.plan.conds:
            conds = self._conditions(it0)
            _lib.check(lib.pb_resolve(conds, res, st), "pb_resolve")
        # the Eq. 1 recheck closes the epoch together with the ring advance
        # (pb_epoch_close: one launch); PB_EPOCH_CLOSE=0 keeps them apart
        self.eq1_host += self.n_eq1_static * E * self.n_streams
        close = (self.n_eq1 <= 256 and len(self.advance) <= 256 and
                 os.environ.get("PB_EPOCH_CLOSE", "1") != "0")
        if self.n_eq1 and not close:
            _lib.check(lib.pb_eq1_check(self.eq1, self.n_eq1, res, self.eq1_ctr, st),
                       "pb_eq1_check")
        self._run_launches(self.launches, res, it0, E, hook)
        for dev, n, block in self.fir_groups:
            _lib.check(lib.pb_fir_carry(dev, n, res, block, st), "fir_carry")
        if close:
            _lib.check(lib.pb_epoch_close(self.eq1, self.n_eq1, self.eq1_ctr, self.advance,
                                          len(self.advance), res, st), "pb_epoch_close")
        else:
            _lib.check(lib.pb_rings_advance(self.advance, len(self.advance), res, st),
                       "pb_rings_advance")
        return lib.pb_launch_count() - n0

    def _run_launches(self, launches, res, it0: int, E: int, hook=None) -> None:
        lib, st = self.lib, self.stream
        for item in launches:
            kind = item[0]
            if hook is not None:
                hook(kind, "pre")
            if kind == "bank":
                _lib.check(lib.pb_fire_filter_bank(item[1], res, item[2], st), "filter_bank")
            elif kind == "fir":
                _lib.check(lib.pb_fire_fir(item[1], item[2], res, item[3], self.fir_math, st),
                           "fir_branch")
            elif kind == "sum":
                _lib.check(lib.pb_fire_branch_sum(item[1], res, item[2], st), "branch_sum")
            elif kind == "bytes":
                _lib.check(lib.pb_fire_bytes(item[1], res, st), "bytes")
            elif kind == "matmul":
                _lib.check(lib.pb_fire_matmul(item[1], res, st), "matmul")
            elif kind == "matmul_chain":
                _lib.check(lib.pb_fire_matmul_chain(item[1], res, st), "matmul chain")
            elif kind == "bypass_region":
                _lib.check(lib.pb_fire_bypass_region(item[1], res, st), "bypass region")
            elif kind == "motion_region":
                _lib.check(lib.pb_fire_motion_region(item[1], res, st), "motion region")
            elif kind == "path_merge":
                _lib.check(lib.pb_fire_path_merge(item[1], res, st), "path_merge")
            elif kind == "image":
                _lib.check(lib.pb_fire_image(item[1], res, st), "image")
            elif kind == "conv":
                _lib.check(lib.pb_fire_conv_pool(item[1], res, st), "conv2d_relu_pool")
            elif kind == "dense":
                _lib.check(lib.pb_fire_dense(item[1], res, st), "dense")
            elif kind == "classify":
                _lib.check(lib.pb_fire_classify(item[1], res, st), "classify_merge")
            elif kind == "host":
                self._fire_host(item[1], it0, E, res)
            if hook is not None:
                hook(kind, "post")

    def _stage_ref(self, dev: int, span: int, cond: int) -> _lib.SpanRef:
        """A host-staging buffer [S][epoch][span] as a span ref: row n of
        stream s at iteration n, written/read only where `cond` is active."""
        return _lib.SpanRef(dev, self.epoch * span, span, None, self.cap, ALWAYS, cond, 0)

    def _copy_spans(self, srcs: list[_lib.SpanRef], dst: list[_lib.SpanRef], res) -> None:
        act = _lib.BytesActor()
        for k, r in enumerate(srcs):
            act.in_[k] = r
        for k, r in enumerate(dst):
            act.out[k] = r
        act.n_in, act.n_out, act.offset, act.cond = len(srcs), len(dst), 0, ALWAYS
        _lib.check(self.lib.pb_fire_bytes(act, res, self.stream), "host staging copy")

    def _fire_host(self, aid: str, it0: int, E: int, res) -> None:
        """Fire a host-fired actor's firings of this epoch through the plugin
        API (runtime.py:126-190): its active input spans are gathered from the
        rings into staging and copied to the host, fire() runs per firing in
        order (dynamic actors get control() first, inactive DRPs zero-length
        spans), and the output spans go back into every target ring."""
        g, plan, S, lib = self.graph, self.plan, self.n_streams, self.lib
        a = g.actor(aid)
        mode = self.host_fired[aid]
        ins = sorted([p for p in a.input_ports if p.kind != CONTROL_IN], key=lambda p: p.id)
        outs = sorted([p for p in a.output_ports if p.kind != CONTROL_OUT], key=lambda p: p.id)
        for p in ins:
            dev, hptr, _, span, fid = self.host_stage[(aid, p.id)]
            self._copy_spans([self._ref(fid)], [self._stage_ref(dev, span, plan.fifo_cond[fid])],
                             res)
            _lib.check(lib.pb_memcpy_d2h(hptr, dev, S * E * span, self.stream))
        for p in outs:
            dev, hptr, harr, span, fid = self.host_stage[(aid, p.id)]
            if mode == "observe":   # the device kernel's outputs, as fired
                self._copy_spans([self._ref(fid, producer=True)],
                                 [self._stage_ref(dev, span, plan.fifo_cond[fid])], res)
                _lib.check(lib.pb_memcpy_d2h(hptr, dev, S * E * span, self.stream))
            else:
                harr[:S * E * span] = 0
        n_cond = int(res.n_cond)
        act = np.ones((max(1, n_cond), S, self.cap), dtype=np.uint8)
        if n_cond:
            _lib.check(lib.pb_memcpy_d2h(act.ctypes.data, self.res_act, act.nbytes, self.stream))
        _lib.check(lib.pb_stream_sync(self.stream), f"{aid}: host firing")

        def active(c: int, s: int) -> np.ndarray:
            return np.ones(E, dtype=bool) if c == ALWAYS else act[c, s, :E].astype(bool)

        port_cond = {}
        for p in ins + outs:
            fid = self.host_stage[(aid, p.id)][4]
            port_cond[p.id] = plan.fifo_cond[fid]
        ctl = None
        cp = a.control_input
        if cp is not None:
            src = g.fifo_into(PortRef(aid, cp.id)).src
            stride = self.ctl_stride[src]
            ctl = (self.ctl_host[src][1][:S * E * stride].reshape(S, E, stride),
                   g.value_length(src))
        rates_all = {p.id: p.rate for p in a.ports}
        views = {p.id: self.host_stage[(aid, p.id)][2][:S * E * self.host_stage[(aid, p.id)][3]]
                 .reshape(S, E, -1) for p in ins + outs}
        for s in range(S):
            b = self.behaviors[s][aid]
            seed = actor_seed(self.seeds[s], aid)
            on = active(self._cond_now.get(aid, plan.actor_cond[aid]), s)
            pact = {pid: active(c, s) for pid, c in port_cond.items()}
            j = int(self.firings[aid][s])
            for n in range(E):
                if not on[n]:
                    continue
                values = None
                try:
                    if ctl is not None:
                        values = decode_control(ctl[0][s, n], ctl[1])
                        b.control(aid, j, values)
                    rates = dict(rates_all)
                    inputs, outputs = {}, {}
                    for p in ins:
                        live = bool(pact[p.id][n])
                        rates[p.id] = p.rate if live else 0
                        inputs[p.id] = memoryview(views[p.id][s, n]) if live else memoryview(b"")
                    for p in outs:
                        live = bool(pact[p.id][n])
                        rates[p.id] = p.rate if live else 0
                        outputs[p.id] = memoryview(views[p.id][s, n]) if live else \
                            memoryview(bytearray(0))
                    b.fire(FireContext(aid, j, rates, inputs, outputs, a.params, seed, values,
                                       device_fired=mode == "observe"))
                except Exception as e:  # noqa: BLE001
                    raise ActorPanic(aid, e) from e
                j += 1
        for p in outs:
            dev, hptr, _, span, fid = self.host_stage[(aid, p.id)]
            _lib.check(lib.pb_memcpy_h2d(dev, hptr, S * E * span, self.stream))
            targets = [self._ref(t, producer=True) for t in self._port_targets(aid, p.id)]
            for k in range(0, len(targets), _lib.PB_MAX_PORTS):
                self._copy_spans([self._stage_ref(dev, span, plan.fifo_cond[fid])],
                                 targets[k:k + _lib.PB_MAX_PORTS], res)

    def set_fir_math(self, math: int) -> None:
        """Switch the FIR arithmetic mode (PB_FIR_EXACT / _EXACT_PAIRED / _FMA)
        of every FIR launch of this runtime."""
        self.fir_math = int(math)
        for item in self.launches:
            if item[0] == "bank":
                item[1].math = self.fir_math

    def _epoch_counts(self) -> np.ndarray:
        n_cond = len(self.plan.conds)
        out = np.zeros((max(1, n_cond), self.n_streams), dtype=np.int32)
        if n_cond:
            _lib.check(self.lib.pb_memcpy_d2h(out.ctypes.data, self.res_count, out.nbytes,
                                              self.stream))
        return out

    def drain_sinks(self, it0: int, E: int, counts: np.ndarray,
                    limits: dict[str, int] | None = None):
        """Sink firings of the epoch: D2H, then digests per firing in sorted
        port order.  limits[sink] (the drain phase): only its first firings."""
        g, S = self.graph, self.n_streams
        pending = []
        for a in g.actors:
            if self.plan.roles[a.id] != "sink":
                continue
            if limits is not None and limits.get(a.id, 0) <= 0:
                continue
            ports = sorted(a.input_ports, key=lambda p: p.id)
            c = self.plan.actor_cond[a.id]
            bufs = []
            for p in ports:
                f = g.fifo_into(PortRef(a.id, p.id))
                st = self.storage[f.id]
                span = f.rate * f.token_bytes
                hptr, harr = self.sink_host[f.id]
                first = it0 if st.index_cond == ALWAYS else None
                if first is None:
                    raise UnsupportedGraph(f"sink {a.id} reads a compacted channel")
                self._d2h_chunks(st.data, st.stream_stride, span, hptr, E, first,
                                 slots=st.slots)
                bufs.append((p.id, span, harr[:S * E * span].reshape(S, E, span)))
            pending.append((a, c, bufs))
        _lib.check(self.lib.pb_stream_sync(self.stream), "sink drain")
        jobs = []
        for a, c, bufs in pending:
            for s in range(S):
                active = None
                if limits is not None:
                    active = np.arange(E) < limits[a.id]
                elif c != ALWAYS:
                    active = self._act_host(c, s, E)
                jobs.append((a, s, bufs, active))

        def digest(job):
            a, s, bufs, active = job
            h = self.digests[a.id][s]
            cap = self.captured[a.id][s] if self.captured is not None else None
            b = self.behaviors[s][a.id]
            generic = type(b).fire is not type(resolve("null_sink")).fire
            if len(bufs) == 1 and active is None and not generic:
                data = bufs[0][2][s].reshape(-1)
                h.update(data)
                if cap is not None:
                    cap += memoryview(np.ascontiguousarray(data)).cast("B")
                return
            for n in range(E):
                if active is not None and not active[n]:
                    continue
                ins = {}
                for pid, span, arr in bufs:
                    data = arr[s, n].tobytes()
                    h.update(data)
                    if cap is not None:
                        cap.extend(data)
                    ins[pid] = memoryview(data)
                if generic:
                    ctx = FireContext(a.id, self.fired[a.id][s], {}, ins, {}, a.params,
                                      actor_seed(self.seeds[s], a.id), None)
                    b.fire(ctx)
                self.fired[a.id][s] += 1

        if len(jobs) > 1:
            list(self.pool.map(digest, jobs))
        else:
            for j in jobs:
                digest(j)

    def _act_host(self, c: int, s: int, E: int) -> np.ndarray:
        out = np.zeros(E, dtype=np.uint8)
        off = (c * self.n_streams + s) * self.cap
        _lib.check(self.lib.pb_memcpy_d2h(out.ctypes.data, self.res_act + off, E, self.stream))
        _lib.check(self.lib.pb_stream_sync(self.stream))
        return out

    # ------------------------------------------------------------------ run

    def reset(self):
        """Fresh run state: counters, histories, behaviour init, digests."""
        lib, m, g, S = self.lib, self.mem, self.graph, self.n_streams
        for fid, ctr in self.counters.items():
            _lib.check(lib.pb_memset(ctr, 0, 8 * 4 * S, self.stream))
        for aid, p in self.fir_state.items():
            _lib.check(lib.pb_memset(p, 0, S * 2 * 9 * 4, self.stream))
        _lib.check(lib.pb_memset(self.eq1_ctr, 0, 16, self.stream))
        self.eq1_host = 0
        _lib.check(lib.pb_memset(self.err_flag, 0, 16, self.stream))
        for s in range(S):
            for a in g.actors:
                b = self.behaviors[s][a.id]
                if a.id in self.sources and self.plan.roles[a.id] == "source":
                    continue
                if is_device(b) and a.id not in self.host_fired:
                    continue   # stateless kernels, configured at build time
                try:
                    b.init(a.id, a.params, actor_seed(self.seeds[s], a.id))
                except Exception as e:  # noqa: BLE001
                    raise ActorPanic(a.id, e) from e
        for ref, buf in self.policy_state.items():
            for s in range(S):
                seed = actor_seed(self.seeds[s], ref.actor)
                _lib.check(lib.pb_policy_init(C.addressof(buf) + s * _lib.PB_POLICY_STATE_BYTES,
                                              -1 if seed is None else seed))
        self._prev_writes = {f.id: 0 for f in g.fifos}
        sinks = [a.id for a in g.actors if self.plan.roles[a.id] == "sink"]
        self.digests = {aid: [hashlib.sha256() for _ in range(S)] for aid in sinks}
        self.captured = ({aid: [bytearray() for _ in range(S)] for aid in sinks}
                         if self.config.capture_sinks else None)
        self.fired = {aid: [0] * S for aid in sinks}
        self.firings = {a.id: np.zeros(S, dtype=np.int64) for a in g.actors}
        _lib.check(lib.pb_stream_sync(self.stream), "reset")

    # ------------------------------------------------------ pipelined run

    def _pipelinable(self, prestaged: bool) -> bool:
        """Bulk-only graphs (bulk sources, native policies, single-port
        always-active digest sinks) run with overlapped copies and hashing."""
        g = self.graph
        if self.config.trace is not None or self.config.pipeline == 1 or self.host_fired:
            return False
        if any(self.plan.extra.values()) or self.unbounded or self.plan.epoch_cap is not None:
            return False      # drain phase / delayed cycles: the plain epoch loop
        for f in g.fifos:
            if f.delay and self.plan.roles[f.src.actor] == "source" or \
                    f.delay and self.plan.roles[f.dst.actor] == "sink":
                return False
        for a in g.actors:
            role = self.plan.roles[a.id]
            b = self.behaviors[0][a.id]
            if role == "source":
                if len(a.output_ports) != 1:
                    return False
                if not (prestaged or a.id in self.sources or type(b) is FileSource):
                    return False
            elif role == "config":
                ctl = [p for p in a.output_ports if p.kind == CONTROL_OUT]
                if native_policy_kind(b) is None or len(ctl) != 1 or len(a.output_ports) != 1:
                    return False
            elif role == "sink":
                if len(a.input_ports) != 1 or self.plan.actor_cond[a.id] != ALWAYS:
                    return False
                if type(b).fire is not type(resolve("null_sink")).fire:
                    return False
        return True

    def _event(self) -> int:
        e = C.c_void_p()
        _lib.check(self.lib.pb_event_create(C.byref(e)))
        self._events.append(e.value)
        return e.value

    def _run_pipelined(self, prestaged: bool, N: int, deadline) -> None:
        """Sub-epoch software pipeline over three CUDA streams:

            copy-in  : H2D of chunk c's source spans and control tokens
            compute  : resolve + actor launches + carry + advance of chunk c
            copy-out : D2H of chunk c's sink spans
            host     : SHA-256 of chunk c per stream (hashlib releases the GIL)

        Chunk c+R reuses chunk c's ring chunks and host window slots (R =
        epoch // sub), so each stage waits on the matching event of c-R.
        """
        lib, g, S = self.lib, self.graph, self.n_streams
        E = self.epoch
        depth = int(self.config.pipeline) if self.config.pipeline > 1 else 8
        sub = max(1, E // depth)
        while E % sub:
            sub -= 1
        R = E // sub
        chunks = [(it, min(sub, N - it)) for it in range(0, N, sub)]
        if N <= E and sub >= 8 and len(chunks) > 2:
            # one window holds the whole run (no slot reuse): ramp the first
            # chunks up (sub/4, sub/4, sub/2, then sub) so the hashing threads
            # -- the end-to-end bottleneck -- start after a quarter of the
            # copy-in / copy-out latency of a full chunk
            chunks, it = [], 0
            for n in (sub // 4, sub // 4, sub // 2):
                if it < N:
                    chunks.append((it, min(n, N - it)))
                    it += chunks[-1][1]
            while it < N:
                chunks.append((it, min(sub, N - it)))
                it += chunks[-1][1]
            R = len(chunks)
        self._events = []
        h2d_ev = [self._event() for _ in chunks]
        comp_ev = [self._event() for _ in chunks]
        d2h_ev = [self._event() for _ in chunks]
        n_cond = len(self.plan.conds)
        # per-chunk firing counts land in PINNED memory: a D2H into pageable
        # memory would block the host until the chunk's kernels finished and
        # serialise the copy-in of the next chunk behind them
        ncnt = len(chunks) * max(1, n_cond) * S
        if getattr(self, "_counts_pinned", None) is None or self._counts_pinned[1].size < 4 * ncnt:
            self._counts_pinned = self.mem.pinned(4 * ncnt)
        counts = self._counts_pinned[1][:4 * ncnt].view(np.int32).reshape(
            len(chunks), max(1, n_cond), S)
        src = [(a, sorted(g.fifos_from(PortRef(a.id, a.output_ports[0].id)),
                          key=lambda f: f.id)[0])
               for a in g.actors if self.plan.roles[a.id] == "source"]
        sinks = [(a, g.fifo_into(PortRef(a.id, a.input_ports[0].id)))
                 for a in g.actors if self.plan.roles[a.id] == "sink"]
        # Hashing: a digest's updates are sequential (chunk c before c+1), so
        # the unit of work is one (sink, stream) job's next chunk.  A watcher
        # thread waits for "chunk c copied out" in order and queues every job
        # that was waiting for it; hashers pop any ready job, hash its next
        # chunk and requeue it if its following chunk is already out.  Work
        # is balanced dynamically across the hashing threads (a static split
        # stalls the whole pipeline on whichever thread loses its core).
        jobs = [(a, f, s) for a, f in sinks for s in range(S)]
        n_thr = max(1, min(len(jobs), int(self.config.host_threads or _default_hashers())))
        recorded = [threading.Event() for _ in chunks]     # d2h_ev[c] has been recorded
        hashed = [0] * len(chunks)                          # jobs done with chunk c
        hashed_cv = threading.Condition()
        failure: list[BaseException] = []
        ready_q: queue.SimpleQueue = queue.SimpleQueue()
        nxt = [0] * len(jobs)          # next chunk each job hashes
        idle = [True] * len(jobs)      # job waits for its next chunk to be copied out
        out_done = [0]                 # chunks [0, out_done) are copied out
        finished = [0]                 # jobs that hashed every chunk
        state_lock = threading.Lock()

        def watcher():
            try:
                for c in range(len(chunks)):
                    recorded[c].wait()
                    if failure:
                        break
                    _lib.check(lib.pb_event_sync(d2h_ev[c]))
                    with state_lock:
                        out_done[0] = c + 1
                        for j in range(len(jobs)):
                            if idle[j] and nxt[j] == c:
                                idle[j] = False
                                ready_q.put(j)
            except BaseException as e:  # noqa: BLE001
                failure.append(e)
            if failure:
                stop_hashers()

        def stop_hashers():
            for _ in range(n_thr):
                ready_q.put(-1)

        def hasher(t):
            try:
                while True:
                    j = ready_q.get()
                    if j < 0 or failure:
                        return
                    a, f, s = jobs[j]
                    c = nxt[j]
                    it0, n = chunks[c]
                    w = it0 % E
                    span = f.rate * f.token_bytes
                    arr = self.sink_host[f.id][1][:S * E * span].reshape(S, E, span)
                    data = arr[s, w:w + n].reshape(-1)
                    self.digests[a.id][s].update(data)
                    if self.captured is not None:
                        self.captured[a.id][s] += memoryview(np.ascontiguousarray(data)).cast("B")
                    with state_lock:
                        nxt[j] = c + 1
                        if c + 1 == len(chunks):
                            finished[0] += 1
                            if finished[0] == len(jobs):
                                stop_hashers()
                        elif c + 1 < out_done[0]:
                            ready_q.put(j)
                        else:
                            idle[j] = True
                    with hashed_cv:
                        hashed[c] += 1
                        hashed_cv.notify_all()
            except BaseException as e:  # noqa: BLE001
                failure.append(e)
                with hashed_cv:
                    hashed_cv.notify_all()

        def wait_hashed(c):
            with hashed_cv:
                hashed_cv.wait_for(lambda: hashed[c] == len(jobs) or failure)
            if failure:
                raise failure[0]

        hashers = [threading.Thread(target=hasher, args=(t,), daemon=True) for t in range(n_thr)]
        hashers.append(threading.Thread(target=watcher, daemon=True))
        for th in hashers:
            th.start()
        try:
            for c, (it0, n) in enumerate(chunks):
                w = it0 % E
                if c >= R:
                    _lib.check(lib.pb_event_sync(h2d_ev[c - R]))       # host window reuse
                    _lib.check(lib.pb_stream_wait(self.copy_in, comp_ev[c - R]))
                # sources
                for a, f in src:
                    span = f.rate * f.token_bytes
                    hptr, harr = self.src_host[f"{a.id}.{a.output_ports[0].id}"]
                    direct = None if prestaged else self._direct_source(a.id, N)
                    if direct is not None:
                        st = self.storage[f.id]
                        self._h2d_chunks(st.data, st.stream_stride, span,
                                         direct[0] + it0 * span, n, it0,
                                         host_pitch=direct[1], stream=self.copy_in)
                        continue
                    if not prestaged:
                        buf = harr[:S * E * span].reshape(S, E, span)
                        for s in range(S):
                            if a.id in self.sources:
                                data = np.frombuffer(memoryview(self.sources[a.id][s]).cast("B"),
                                                     dtype=np.uint8)[it0 * span:(it0 + n) * span]
                            else:
                                try:
                                    data = np.frombuffer(self.behaviors[s][a.id].take(
                                        a.id, n * span), dtype=np.uint8)
                                except EOFError as e:
                                    raise ActorPanic(a.id, e) from e
                            if data.size < n * span:
                                raise ActorPanic(a.id, EOFError(
                                    f"{a.id}: input exhausted at byte {it0 * span + data.size}"))
                            buf[s, w:w + n] = data.reshape(n, span)
                    st = self.storage[f.id]
                    self._h2d_chunks(st.data, st.stream_stride, span, hptr + w * span, n, it0,
                                     host_pitch=E * span, stream=self.copy_in)
                # control tokens (native generators), dense per chunk slot
                for ref in self.ctl_ports:
                    a = g.actor(ref.actor)
                    stride = self.ctl_stride[ref]
                    hptr, harr = self.ctl_host[ref]
                    b0 = self.behaviors[0][a.id]
                    min_tb = min(f.token_bytes for f in g.fifos_from(ref))
                    try:
                        length = int(a.params["length"])
                        param = b0.native_param(a.params)
                        if length > min_tb:
                            raise ValueError(f"{length} control elements exceed {min_tb} bytes")
                    except Exception as e:  # noqa: BLE001
                        raise ActorPanic(a.id, e) from e
                    slot = hptr + (it0 % E) * S * stride   # this chunk's [S][n] tokens
                    rc = lib.pb_policy_tokens_streams(
                        C.addressof(self.policy_state[ref]), S, native_policy_kind(b0), length,
                        param, it0, n, slot, stride, int(self.config.host_threads))
                    if rc != _lib.PB_OK:
                        raise ActorPanic(a.id, ValueError(_lib.error_text()))
                    self._h2d_chunks(self.ctl_dev[ref], self.C * stride, stride, slot, n, it0,
                                     stream=self.copy_in)
                _lib.check(lib.pb_event_record(h2d_ev[c], self.copy_in))
                # compute
                _lib.check(lib.pb_stream_wait(self.stream, h2d_ev[c]))
                if c >= R:
                    _lib.check(lib.pb_stream_wait(self.stream, d2h_ev[c - R]))
                self.fire_epoch(it0, n)
                if n_cond:
                    _lib.check(lib.pb_memcpy_d2h(counts[c].ctypes.data, self.res_count,
                                                 n_cond * S * 4, self.stream))
                _lib.check(lib.pb_event_record(comp_ev[c], self.stream))
                # copy out (the host window slot must have been hashed)
                if c >= R:
                    wait_hashed(c - R)
                _lib.check(lib.pb_stream_wait(self.copy_out, comp_ev[c]))
                for a, f in sinks:
                    st = self.storage[f.id]
                    span = f.rate * f.token_bytes
                    hptr = self.sink_host[f.id][0]
                    self._d2h_chunks(st.data, st.stream_stride, span, hptr + w * span, n, it0,
                                     host_pitch=E * span, stream=self.copy_out)
                _lib.check(lib.pb_event_record(d2h_ev[c], self.copy_out))
                recorded[c].set()
                if deadline is not None and time.perf_counter() > deadline and c + 1 < len(chunks):
                    raise Timeout(self.config.timeout_ms, sorted(a.id for a in g.actors))
            for c in range(len(chunks)):
                wait_hashed(c)
        finally:
            if len(failure) == 0 and not all(ev.is_set() for ev in recorded):
                failure.append(RuntimeError("pipeline aborted"))
            for ev in recorded:
                ev.set()
            if failure:
                stop_hashers()
            for th in hashers:
                th.join()
            lib.pb_stream_sync(self.copy_in)
            lib.pb_stream_sync(self.stream)
            lib.pb_stream_sync(self.copy_out)
            for e in self._events:
                lib.pb_event_destroy(e)
            self._events = []
        self._check_device_errors()
        for c, (it0, n) in enumerate(chunks):
            for a in g.actors:
                cc = self.plan.actor_cond[a.id]
                self.firings[a.id] += n if cc == ALWAYS else counts[c, cc]

    def run_all(self, prestaged: bool = False) -> list[RunReport]:
        cfg, S = self.config, self.n_streams
        N = int(cfg.source_firings)
        self.reset()
        t_start = time.perf_counter()
        deadline = None if cfg.timeout_ms is None else t_start + cfg.timeout_ms / 1000.0
        self.pool = ThreadPoolExecutor(max_workers=max(1, cfg.host_threads or 16))
        try:
            if self._pipelinable(prestaged and N <= self.epoch):
                self._run_pipelined(prestaged and N <= self.epoch, N, deadline)
                it = N
            else:
                it = 0
            while it < N:
                E = min(self.epoch, N - it)
                self.stage_sources(it, E, prestaged=prestaged and N <= self.epoch)
                self.stage_control(it, E)
                self.fire_epoch(it, E)
                counts = self._epoch_counts()
                self.drain_sinks(it, E, counts)
                self._check_device_errors()
                for a in self.graph.actors:
                    c = self.plan.actor_cond[a.id]
                    self.firings[a.id] += E if c == ALWAYS else counts[c]
                if cfg.trace is not None:
                    self._trace()
                it += E
                if deadline is not None and time.perf_counter() > deadline and it < N:
                    raise Timeout(cfg.timeout_ms, sorted(a.id for a in self.graph.actors))
            self._run_drain(N, deadline)
            for s in range(S):
                for a in self.graph.actors:
                    try:
                        self.behaviors[s][a.id].finish(a.id)
                    except Exception as e:  # noqa: BLE001
                        raise ActorPanic(a.id, e) from e
        finally:
            self.pool.shutdown(wait=True)
        wall_ms = (time.perf_counter() - t_start) * 1000.0
        return self._reports(wall_ms)

    # ----------------------------------------------------------- drain phase

    def _drain_setup(self):
        """Launches of the drain phase: actors that keep firing after the
        sources stop (plan.extra) gated by per-value drain conditions --
        condition k is true at drain iteration i iff i < values[k] -- and the
        unbounded ones (a sourceless cycle) always."""
        plan, S = self.plan, self.n_streams
        values = sorted({e for a, e in plan.extra.items() if e})
        fires = {a for a, e in plan.extra.items()
                 if (e is None or e > 0) and plan.roles[a] not in ("source", "config", "sink")}
        index = {v: k for k, v in enumerate(values)}
        cond = {a: (ALWAYS if plan.extra[a] is None else index[plan.extra[a]]) for a in fires}
        launches, fir_groups = self._build_launches(cond_of=cond.__getitem__, only=fires)
        K = max(1, len(values))
        dev = self.mem.malloc(S * self.epoch * K)
        hptr, harr = self.mem.pinned(S * self.epoch * K)
        if len(values) > self.res_slots:
            raise UnsupportedGraph(f"{len(values)} distinct drain lengths exceed the "
                                   f"{self.res_slots} resolution slots")
        self._drain = (launches, fir_groups, values, cond, dev, hptr, harr, K)

    def _run_drain(self, N: int, deadline) -> None:
        """Fire the drain phase (runtime.py:118-124: consumers keep firing on
        delay tokens after the sources stop; interp.py's drain), and for
        actors no source bounds, keep firing until the timeout."""
        plan, cfg, lib, S = self.plan, self.config, self.lib, self.n_streams
        finite = [e for e in plan.extra.values() if e]
        if not finite and not self.unbounded:
            return
        if self._drain is None:
            self._drain_setup()
        launches, fir_groups, values, cond, dev, hptr, harr, K = self._drain
        D = max(finite, default=0)
        done = 0
        while done < D or self.unbounded:
            if deadline is not None and time.perf_counter() > deadline:
                raise Timeout(cfg.timeout_ms, list(self.unbounded) or
                              sorted(a for a, e in plan.extra.items() if e and e > done))
            E = self.epoch if self.unbounded and done >= D else min(self.epoch, max(1, D - done))
            it0 = N + done
            # drain conditions of this epoch: [S][epoch][K] bytes
            tok = harr[:S * self.epoch * K].reshape(S, self.epoch, K)
            tok[:] = 0
            for k, v in enumerate(values):
                tok[:, :max(0, min(E, v - done)), k] = 1
            _lib.check(lib.pb_memcpy_h2d(dev, hptr, S * self.epoch * K, self.stream))
            arr = (_lib.Condition * K)()
            for k in range(K):
                arr[k] = _lib.Condition(dev, self.epoch * K, K, k, self.epoch, 0)
            res = self._resolved(E)
            res.n_cond = K
            if values:
                _lib.check(lib.pb_resolve(arr, res, self.stream), "pb_resolve (drain)")
            self._cond_now = cond
            try:
                self._run_launches(launches, res, it0, E)
            finally:
                self._cond_now = {}
            for d, n, block in fir_groups:
                _lib.check(lib.pb_fir_carry(d, n, res, block, self.stream), "fir_carry")
            if self.n_drain_advance:
                _lib.check(lib.pb_rings_advance(self.drain_advance, self.n_drain_advance, res,
                                                self.stream), "pb_rings_advance")
            fired = {a: (E if e is None else max(0, min(E, e - done)))
                     for a, e in plan.extra.items() if plan.roles[a] not in ("source", "config")}
            self.drain_sinks(it0, E, None, limits={a: fired.get(a, 0) for a in plan.extra
                                                   if plan.roles[a] == "sink"})
            self._check_device_errors()
            for a, n in fired.items():
                self.firings[a] += n
            done += E

    def run(self) -> RunReport:
        """Runtime.run (runtime.py:278-325) for a single-stream runtime."""
        if self.n_streams != 1:
            raise ValueError("run() drives one stream; use run_all() for a batch")
        return self.run_all()[0]

    @property
    def channels(self) -> dict[str, "ChannelView"]:
        """Runtime.channels (runtime.py:266-272) as read-only views of the
        device rings of stream 0: occupancy, max_occupancy, plan.slots."""
        out = {}
        for f in self.graph.fifos:
            ctr = self._counters(f.id)
            w, r = int(ctr[0, 0]), int(ctr[1, 0])
            slots = layout_slots(f.rate, f.delay, self.config.c_factor)
            peak = min(f.delay + f.rate, slots) if w > 0 and f.id not in self.plan.loose \
                else f.delay
            out[f.id] = ChannelView(f.id, f.delay + f.rate * (w - r), peak, slots)
        return out

    def _check_device_errors(self):
        flag = np.zeros(1, dtype=np.int32)
        _lib.check(self.lib.pb_memcpy_d2h(flag.ctypes.data, self.err_flag, 4, self.stream))
        _lib.check(self.lib.pb_stream_sync(self.stream), "epoch")
        if flag[0]:
            for item in self.launches:
                if item[0] in ("path_merge", "classify"):
                    raise ActorPanic(item[2], ValueError(
                        f"{item[0]} needs exactly one live input per firing"))
            raise ActorPanic("device", RuntimeError("device actor reported a failure"))

    def _counters(self, fid: str) -> np.ndarray:
        out = np.zeros((4, self.n_streams), dtype=np.int64)
        _lib.check(self.lib.pb_memcpy_d2h(out.ctypes.data, self.counters[fid], out.nbytes,
                                          self.stream))
        _lib.check(self.lib.pb_stream_sync(self.stream))
        return out

    def _trace(self):
        """Per-epoch bulk trace lines in the reference format `fifo op occupancy`
        (runtime.py:259-272): one `w` line at the epoch's write peak and one
        `r` line after the consumer drained it (stream 0)."""
        for f in self.graph.fifos:
            ctr = self._counters(f.id)
            w, r = int(ctr[0, 0]), int(ctr[1, 0])
            self.config.trace(f"{f.id} w {f.delay + f.rate * (w - self._prev_writes[f.id])}")
            self.config.trace(f"{f.id} r {f.delay + f.rate * (w - r)}")
            self._prev_writes[f.id] = w

    def _reports(self, wall_ms: float) -> list[RunReport]:
        g, S = self.graph, self.n_streams
        eq = np.zeros(2, dtype=np.int64)
        _lib.check(self.lib.pb_memcpy_d2h(eq.ctypes.data, self.eq1_ctr, 16, self.stream))
        ctrs = {f.id: self._counters(f.id) for f in g.fifos}
        reports = []
        for s in range(S):
            r = RunReport(wall_ms=wall_ms)
            for a in g.actors:
                r.firing_counts[a.id] = int(self.firings[a.id][s])
            for aid, hs in self.digests.items():
                r.sink_digests[aid] = hs[s].hexdigest()
                if self.captured is not None:
                    r.sink_data[aid] = bytes(self.captured[aid][s])
            for f in g.fifos:
                # slots / beta / max_occupancy with the reference's meaning at
                # the caller's c_factor: the channel plan (fifos.py:87-98), the
                # analysis bound (analysis.py:398-411) and the peak of the
                # firing sequence the executor realises -- iteration by
                # iteration, a producer before its consumer, so a channel holds
                # its delay tokens plus one firing's rate once it carried data
                r.slots[f.id] = layout_slots(f.rate, f.delay, self.config.c_factor)
                # a channel that starts full of delay tokens takes a firing's
                # tokens only once its consumer has read (the producer waits
                # for a free span); across a cycle's delayed edge the
                # consumer always reads first
                wrote = ctrs[f.id][0, s] > 0 and f.id not in self.plan.loose
                r.max_occupancy[f.id] = min(f.delay + f.rate, r.slots[f.id]) if wrote \
                    else f.delay
                st = self.storage.get(f.id)
                r.device_slots[f.id] = f.rate * (st.slots if st is not None else self.C)
                r.device_max_occupancy[f.id] = int(ctrs[f.id][2, s])
            r.beta = dict(self.analysis.beta)
            reports.append(r)
        # Eq. 1 counters are device-wide; attribute them evenly per stream
        for r in reports:
            r.eq1_checks = (int(eq[0]) + self.eq1_host) // S
            r.eq1_failures = int(eq[1]) // S
        return reports

    def close(self):
        if getattr(self, "_registered", None):
            self.lib.pb_device_sync()
            for p in self._registered:
                self.lib.pb_host_unregister(p)
            self._registered = []
        if getattr(self, "mem", None) is not None:
            self.mem.close()
            self.mem = None
        for name in ("stream", "copy_in", "copy_out"):
            if getattr(self, name, None):
                self.lib.pb_stream_destroy(getattr(self, name))
                setattr(self, name, None)

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def instantiate(graph, behaviors: Mapping | None = None, config: RuntimeConfig | None = None,
                analysis=None) -> DeviceRuntime:
    """runtime.py:327-342: admission-gated executor for one stream."""
    return DeviceRuntime(graph, behaviors, config, n_streams=1)


def run(graph, behaviors: Mapping | None = None,
        config: RuntimeConfig | None = None) -> RunReport:
    """Drop-in for tokenflow.runtime.run (runtime.py:345-347)."""
    rt = instantiate(graph, behaviors, config)
    try:
        return rt.run_all()[0]
    finally:
        rt.close()


def run_streams(graph, n_streams: int, config: RuntimeConfig | None = None,
                seeds: Sequence[int | None] | None = None,
                sources: Mapping[str, Sequence] | None = None,
                behaviors: Mapping | None = None) -> list[RunReport]:
    """Run `n_streams` independent replicas of `graph` (per-stream seeds and
    source data) in one batched device execution; one RunReport per stream."""
    rt = DeviceRuntime(graph, behaviors, config, n_streams=n_streams, seeds=seeds,
                       sources=sources)
    try:
        return rt.run_all()
    finally:
        rt.close()
