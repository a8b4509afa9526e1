"""Exception types of the reference engine, kept with the same names and
meaning so callers can switch engines without touching their handlers.

Reference: pkg/src/tokenflow/fifos.py:25-46 (channel errors) and
pkg/src/tokenflow/runtime.py:26-48 (execution errors).
"""
from __future__ import annotations


class FifoError(Exception):
    pass


class InvalidParams(FifoError, ValueError):
    """fifos.py:29 — bad rate / token size / delay / buffering factor."""


class ProtocolError(FifoError):
    """fifos.py:33 — span protocol misuse (here also: a non-blocking ring call
    that the reference would have blocked on)."""


class EndOfStream(FifoError):
    """fifos.py:37 — channel closed with fewer tokens than one firing needs."""


class Poisoned(FifoError):
    """fifos.py:41 — channel force-released after a failure elsewhere."""

    def __init__(self, fifo_id: str, reason: str = ""):
        self.fifo_id = fifo_id
        super().__init__(f"channel {fifo_id} poisoned" + (f": {reason}" if reason else ""))


class ExecutionError(Exception):
    pass


class InconsistentGraph(ExecutionError):
    """runtime.py:30 — the admission analysis rejected the graph."""

    def __init__(self, report):
        self.report = report
        problems = list(getattr(report, "problems", None) or [])
        if not problems:
            problems = [v.render() for v in getattr(report, "violations", ())]
            problems += [d.render() for d in getattr(report, "diagnostics", ())]
        super().__init__("graph failed consistency analysis: " + "; ".join(problems))


class ActorPanic(ExecutionError):
    """runtime.py:38 — an actor's init/fire/finish raised."""

    def __init__(self, actor: str, cause: BaseException):
        self.actor = actor
        self.cause = cause
        super().__init__(f"actor {actor} failed: {cause!r}")


class Timeout(ExecutionError):
    """runtime.py:45 — the run exceeded RuntimeConfig.timeout_ms."""

    def __init__(self, ms: float | None, alive: list[str], message: str | None = None):
        self.alive = alive
        super().__init__(message or f"run exceeded {ms:.0f} ms; still running: "
                                    f"{', '.join(alive)}")


class UnsupportedGraph(ExecutionError):
    """The graph is consistent but outside the class the device executor
    schedules (delay tokens, cycles, nested dynamic regions, ...)."""


class DeviceUnavailable(RuntimeError):
    """The CUDA library or a B200 is missing.  There is no CPU fallback."""
