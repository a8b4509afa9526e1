"""Motion detection (apps/motion.py) on one B200: device-resident
frames/s of the blur -> diff/threshold (one-frame delay) -> median graph over
many independent 64x64 streams, per-kernel device times and HBM roofline, and
the reference interpreter (oracle/_ref, one process per core) beside it."""
import ctypes as C
import json
import os
import statistics
import sys
import tempfile
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np

from paper_1802_06625_b200 import RuntimeConfig
from paper_1802_06625_b200.apps import motion
from paper_1802_06625_b200.engine import DeviceRuntime

SIDE = 64
FB = SIDE * SIDE
# HBM bytes per frame as the graph executes (one launch per actor): blur reads
# the frame and writes f_cur and the delayed f_prev ring; detect reads both
# and writes the mask; median reads the mask and writes the output
BYTES_PER_FRAME = (FB + 2 * FB) + (2 * FB + FB) + (FB + FB)
# the fused region (motion_region_kernel) reads each frame and writes its output;
# the frame before each CTA run is read a second time (kMRF = 16 frames per CTA)
BYTES_PER_FRAME_FUSED = FB + FB + FB / 16


def _ref_stream(args):
    seed, frames = args
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    from tokenflow.interp import interpret
    from tokenflow.model import build_graph
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "input.bin"
        p.write_bytes(motion.make_input(seed, frames))
        g = build_graph(motion.build_description(SIDE, str(p)))
        t0 = time.perf_counter()
        interpret(g, source_firings=frames, seed=seed)
        return time.perf_counter() - t0


def measure(S=256, frames=256, steps=50, fuse=1):
    rt = DeviceRuntime(motion.build_description(), config=RuntimeConfig(
        source_firings=frames, epoch=frames, fuse=bool(fuse)), n_streams=S, seeds=list(range(S)),
        sources={"src": [None] * S})
    st = rt.source_staging("src")
    for s in range(S):
        st[s] = np.frombuffer(motion.make_input(s, frames), np.uint8).reshape(frames, -1)
    lib = rt.lib
    rt.reset()
    rt.stage_sources(0, frames, prestaged=True)
    rt.stage_control(0, frames)
    for _ in range(3):
        rt.fire_epoch(0, frames)
    lib.pb_stream_sync(rt.stream)

    def ev():
        e = C.c_void_p()
        lib.pb_event_create(C.byref(e))
        return e.value
    marks = {}

    def hook(kind, phase):
        e = ev()
        lib.pb_event_record(e, rt.stream)
        marks.setdefault(kind, []).append(e)
    e0, e1 = ev(), ev()
    lib.pb_event_record(e0, rt.stream)
    for _ in range(steps):
        rt.fire_epoch(0, frames, hook=hook)
    lib.pb_event_record(e1, rt.stream)
    lib.pb_stream_sync(rt.stream)
    ms = C.c_float()
    lib.pb_event_elapsed_ms(e0, e1, C.byref(ms))
    step_ms = ms.value / steps
    kern = []
    evs = marks.get("image", []) or marks.get("motion_region", [])
    for i in range(0, len(evs) - 1, 2):
        lib.pb_event_elapsed_ms(evs[i], evs[i + 1], C.byref(ms))
        kern.append(ms.value)
    per_step_kernels = sum(kern) / steps if kern else float("nan")
    if fuse:
        per_op = {"motion_region": statistics.mean(kern)} if kern else {}
    else:
        ops = ["blur", "diff", "median"]   # launch order of one epoch
        per_op = {op: statistics.mean(kern[k::3]) for k, op in enumerate(ops)} if kern else {}
    bpf = BYTES_PER_FRAME_FUSED if fuse else BYTES_PER_FRAME
    n = S * frames
    rt.close()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    achieved = n * bpf / (per_step_kernels / 1e3) / 1e9
    out = {"metric": "motion frames/s (64x64, blur -> diff -> median, device-resident)",
           "streams": S, "frames_per_stream": frames, "frames_per_step": n,
           "step_ms": step_ms, "frames_per_s": n / (step_ms / 1e3),
           "image_kernels_ms_per_step": per_step_kernels, "kernel_ms": per_op,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                        "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                        "bytes_per_frame": bpf,
                        "note": "fused region: the frame in, the output out, the frame "
                                "before each 8-frame run again" if fuse else
                                "bytes as the unfused graph moves them (three launches)"},
           "fused_region": bool(fuse)}
    if (ROOT / "oracle" / "_ref").is_dir():
        cores = os.cpu_count() or 1
        ref_frames = 64
        with ProcessPoolExecutor(cores) as ex:
            ts = list(ex.map(_ref_stream, [(s, ref_frames) for s in range(cores)]))
        out["cpu_baseline"] = {"value": cores * ref_frames / max(ts), "unit": "frames/s",
                               "cores": cores, "kind": "reference",
                               "sample": f"{cores} streams x {ref_frames} frames through "
                                         "tokenflow.interp.interpret, one process per core"}
    return out


if __name__ == "__main__":
    print(json.dumps(measure(*[int(a) for a in sys.argv[1:]])))
