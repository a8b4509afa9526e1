"""B200-native execution path for the data-parallel actors of PRUNE
(arXiv 1802.06625), drop-in for the reference engine `tokenflow.runtime`.

    from paper_1802_06625_b200 import run, RuntimeConfig
    report = run(graph, config=RuntimeConfig(source_firings=160, seed=11))

`graph` is a reference `tokenflow` Graph, a JSON description dict or a path.
Every data-parallel firing runs in libprune_b200.so (sm_100a); there is no
CPU fallback.
"""
from .behaviors import (ActorBehavior, DeviceBehavior, FireContext, actor_seed, available,
                        behavior, decode_control, encode_control, resolve)
from .engine import DeviceRuntime, RunReport, RuntimeConfig, instantiate, run, run_streams
from .errors import (ActorPanic, DeviceUnavailable, EndOfStream, ExecutionError,
                     InconsistentGraph, InvalidParams, Poisoned, ProtocolError, Timeout,
                     UnsupportedGraph)
from .graph import as_graph, from_description
from .plan import admit

__all__ = [
    "ActorBehavior", "DeviceBehavior", "FireContext", "actor_seed", "available", "behavior",
    "decode_control", "encode_control", "resolve", "DeviceRuntime", "RunReport",
    "RuntimeConfig", "instantiate", "run", "run_streams", "ActorPanic", "DeviceUnavailable",
    "EndOfStream", "ExecutionError", "InconsistentGraph", "InvalidParams", "Poisoned",
    "ProtocolError", "Timeout", "UnsupportedGraph", "as_graph", "from_description", "admit",
]
