"""CNN e2e phases: H2D bandwidth of the frames and run_all at several depths."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1802_06625_b200 import RuntimeConfig
from paper_1802_06625_b200.apps import vision
from paper_1802_06625_b200.engine import DeviceRuntime

S, F, R = 4, 64, 24
out = {}
for pipe in (4, 8, 16):
    desc = vision.build_description(R, policy="fixed_policy")
    rt = DeviceRuntime(desc, config=RuntimeConfig(source_firings=F, epoch=F, pipeline=pipe),
                       n_streams=S, seeds=list(range(S)), sources={"src": [None] * S})
    st = rt.source_staging("src")
    for s in range(S):
        st[s] = vision.make_frames(s, F * R).reshape(F, -1).view(np.uint8)
    out["pipelinable"] = rt._pipelinable(True)
    rt.run_all(prestaged=True)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        rt.run_all(prestaged=True)
        ts.append(time.perf_counter() - t0)
    out[f"run_all_ms_pipe{pipe}"] = 1e3 * min(ts)
    lib = rt.lib
    t0 = time.perf_counter()
    rt.stage_sources(0, F, prestaged=True)
    lib.pb_stream_sync(rt.stream)
    lib.pb_stream_sync(rt.copy_in)
    out[f"h2d_GBps"] = S * F * R * vision.FRAME_BYTES / (time.perf_counter() - t0) / 1e9
    rt.close()
print(json.dumps(out, indent=1))
