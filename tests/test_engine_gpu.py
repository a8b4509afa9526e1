"""Engine behaviour on the B200: bypass app, failure modes, rings."""
import hashlib

import numpy as np
import pytest

from paper_1802_06625_b200 import (ActorBehavior, ActorPanic, EndOfStream, InvalidParams,
                                   ProtocolError, RuntimeConfig, UnsupportedGraph, run)
from paper_1802_06625_b200 import _lib

pytestmark = pytest.mark.gpu


def bypass_desc(path):
    """apps/bypass.py:69-132 (the reference's adaptive-bypass graph)."""
    from paper_1802_06625_b200.apps import bypass
    return bypass.build_description(path)


@pytest.mark.parametrize("epoch", [4096, 5])
def test_bypass_app_matches_reference(golden, tmp_path, epoch):
    arr = golden["bypass_small"]
    p = tmp_path / "input.bin"
    p.write_bytes(arr["input"].tobytes())
    rep = run(bypass_desc(str(p)), config=RuntimeConfig(source_firings=32, seed=5,
                                                        capture_sinks=True, epoch=epoch))
    g = golden["bypass"]["default"]
    assert rep.sink_data["sink"] == arr["sink"].tobytes()
    assert rep.sink_digests["sink"] == g["sink_digest"]
    assert rep.firing_counts == g["firing_counts"]


def test_source_exhaustion_is_actor_panic(tmp_path):
    from paper_1802_06625_b200.apps import predistortion as pd
    p = tmp_path / "short.bin"
    p.write_bytes(pd.make_input(11, 3))
    with pytest.raises(ActorPanic) as ei:
        run(pd.build_description(256, 4, str(p)), config=RuntimeConfig(source_firings=5, seed=1))
    assert ei.value.actor == "src" and isinstance(ei.value.cause, EOFError)


class BadInit(ActorBehavior):
    def init(self, actor_id, params, seed):
        raise RuntimeError("init exploded")

    def fire(self, ctx):
        pass


def test_init_failure_is_actor_panic(tmp_path):
    from paper_1802_06625_b200.apps import predistortion as pd
    p = tmp_path / "in.bin"
    p.write_bytes(pd.make_input(11, 2))
    with pytest.raises(ActorPanic) as ei:
        run(pd.build_description(256, 4, str(p)), behaviors={"sink": BadInit()},
            config=RuntimeConfig(source_firings=2))
    assert ei.value.actor == "sink"


class Recorder(ActorBehavior):
    def __init__(self):
        self.seen = []

    def fire(self, ctx):
        self.seen.append((ctx.firing, bytes(next(iter(ctx.inputs.values())))))


def test_custom_host_sink_sees_every_firing(tmp_path, golden):
    arr = golden["dpd_small"]
    from paper_1802_06625_b200.apps import predistortion as pd
    p = tmp_path / "in.bin"
    p.write_bytes(arr["small_input"].tobytes())
    rec = Recorder()
    rep = run(pd.build_description(256, 4, str(p)), behaviors={"sink": rec},
              config=RuntimeConfig(source_firings=6, seed=11))
    assert [f for f, _ in rec.seen] == list(range(6))
    assert b"".join(b for _, b in rec.seen) == arr["small_sink"].tobytes()
    assert rep.sink_digests["sink"] == hashlib.sha256(arr["small_sink"].tobytes()).hexdigest()


def test_host_behaviour_between_device_actors_is_unsupported(tmp_path):
    from paper_1802_06625_b200.apps import predistortion as pd
    with pytest.raises(UnsupportedGraph):
        run(pd.build_description(256, 4, str(tmp_path / "x")), behaviors={"b1": Recorder()},
            config=RuntimeConfig(source_firings=1))


# ---------------------------------------------------------------- rings

def make_ring(rate, tb, delay, factor, payload=None):
    import ctypes as C
    lib = _lib.load()
    r = C.c_void_p()
    buf = None if payload is None else C.create_string_buffer(payload, len(payload))
    _lib.check(lib.pb_ring_create(rate, tb, delay, factor, 1, buf, C.byref(r)))
    return lib, r


def push(lib, r, data):
    import ctypes as C
    b = C.create_string_buffer(data, len(data))
    return lib.pb_ring_push_host(r, 0, b, 1, None)


def pop(lib, r, n):
    import ctypes as C
    b = C.create_string_buffer(n)
    rc = lib.pb_ring_pop_host(r, 0, b, 1, None)
    return rc, b.raw


@pytest.mark.parametrize("rate,delay,factor", [(1, 0, 3), (2, 3, 3), (3, 1, 2), (2, 7, 2),
                                               (1, 5, 2), (4, 4, 3)])
def test_ring_preserves_the_stream(rate, delay, factor):
    """Token stream preservation through device rings (test_fifo.py:335-373):
    the consumer sees delay payload tokens then exactly the produced ones."""
    tb = 3
    payload = bytes((200 + i) % 256 for i in range(delay * tb))
    lib, r = make_ring(rate, tb, delay, factor, payload or None)
    span = rate * tb
    produced = bytes(range(256)) * 4
    chunks = [produced[i:i + span] for i in range(0, span * 20, span)]
    got = b""
    w = 0
    for _ in range(200):
        progressed = False
        if w < len(chunks) and push(lib, r, chunks[w]) == 0:
            w += 1
            progressed = True
        rc, data = pop(lib, r, span)
        if rc == 0:
            got += data
            progressed = True
        if not progressed:
            break
    import ctypes as C
    wr, rd, mx = C.c_int64(), C.c_int64(), C.c_int64()
    lib.pb_ring_counters(r, 0, C.byref(wr), C.byref(rd), C.byref(mx))
    p = _lib.Plan()
    lib.pb_ring_plan(r, C.byref(p))
    expect = (payload + b"".join(chunks))[:len(got)]
    assert got == expect and len(got) >= span * 15
    assert mx.value <= p.slots
    lib.pb_ring_close(r)
    while True:
        rc, data = pop(lib, r, span)
        if rc != 0:
            assert rc == _lib.PB_E_EOS
            break
        got += data
    assert got == (payload + b"".join(chunks[:w]))[:len(got)]
    lib.pb_ring_destroy(r)


def test_ring_protocol_errors():
    lib, r = make_ring(1, 4, 0, 2)
    assert push(lib, r, b"aaaa") == 0 and push(lib, r, b"bbbb") == 0
    assert push(lib, r, b"cccc") == _lib.PB_E_PROTOCOL          # full: would block
    assert pop(lib, r, 4) == (0, b"aaaa")
    lib.pb_ring_close(r)
    assert push(lib, r, b"dddd") == _lib.PB_E_PROTOCOL          # write after close
    assert pop(lib, r, 4) == (0, b"bbbb")
    assert pop(lib, r, 4)[0] == _lib.PB_E_EOS
    lib.pb_ring_poison(r, b"boom")
    assert pop(lib, r, 4)[0] == _lib.PB_E_POISONED
    with pytest.raises(InvalidParams):
        _lib.check(lib.pb_ring_create(0, 4, 0, 2, 1, None, None))
    lib.pb_ring_destroy(r)
