"""CNN (BASELINE config 3) throughput on one B200: frames/s through the
vision graph with every firing processed, plus per-kernel device times."""
import ctypes as C
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1802_06625_b200 import RuntimeConfig, _lib
from paper_1802_06625_b200.apps import vision
from paper_1802_06625_b200.engine import DeviceRuntime


def measure(S=4, firings=64, R=24, steps=20, debug=0):
    desc = vision.build_description(R, policy="fixed_policy")
    rt = DeviceRuntime(desc, config=RuntimeConfig(source_firings=firings, epoch=firings),
                       n_streams=S, seeds=list(range(S)), sources={"src": [None] * S})
    st = rt.source_staging("src")
    for s in range(S):
        st[s] = vision.make_frames(s, firings * R).reshape(firings, -1).view(np.uint8)
    lib = rt.lib
    for item in rt.launches:   # profiling only: skip conv roles (pb_conv_actor.debug)
        if item[0] == "conv":
            item[1].debug = debug
    rt.reset()
    rt.stage_sources(0, firings, prestaged=True)
    rt.stage_control(0, firings)
    for _ in range(3):
        rt.fire_epoch(0, firings)
    lib.pb_stream_sync(rt.stream)

    def ev():
        e = C.c_void_p()
        lib.pb_event_create(C.byref(e))
        return e.value
    marks = {}

    seen = {}

    def hook(kind, phase):
        e = ev()
        lib.pb_event_record(e, rt.stream)
        if phase == "pre":   # conv launches of one epoch are l1 then l2
            seen[kind] = seen.get(kind, 0) + 1
        k = kind if kind != "conv" else f"conv_l{(seen[kind] - 1) % 2 + 1}"
        marks.setdefault(k, []).append(e)
    e0, e1 = ev(), ev()
    lib.pb_event_record(e0, rt.stream)
    for _ in range(steps):
        rt.fire_epoch(0, firings, hook=hook)
    lib.pb_event_record(e1, rt.stream)
    lib.pb_stream_sync(rt.stream)
    ms = C.c_float()
    lib.pb_event_elapsed_ms(e0, e1, C.byref(ms))
    step_ms = ms.value / steps
    per_kernel = {}
    for kind, evs in marks.items():
        ts = []
        for i in range(0, len(evs) - 1, 2):
            lib.pb_event_elapsed_ms(evs[i], evs[i + 1], C.byref(ms))
            ts.append(ms.value)
        per_kernel[kind] = statistics.mean(ts)
    frames = S * firings * R
    rt.close()
    return {"frames_per_step": frames, "step_ms": step_ms,
            "frames_per_s": frames / (step_ms / 1e3), "kernel_ms": per_kernel,
            "tflops_useful": frames * vision.flops_per_frame() / (step_ms / 1e3) / 1e12}


if __name__ == "__main__":
    print(json.dumps(measure(*[int(a) for a in sys.argv[1:]])))
