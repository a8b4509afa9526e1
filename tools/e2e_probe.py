"""Break down one end-to-end DPD step (C2) into its host/device phases."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1802_06625_b200 import RuntimeConfig, _lib
from paper_1802_06625_b200.apps import predistortion as pd
from paper_1802_06625_b200.engine import DeviceRuntime

S, blocks, B = 64, 256, 4096
for pipe in (8, 16, 4, 1):
    rt = DeviceRuntime(pd.build_description(B, 4), config=RuntimeConfig(
        source_firings=blocks, epoch=blocks, pipeline=pipe), n_streams=S,
        seeds=[1000 + s for s in range(S)], sources={"src": [None] * S})
    st = rt.source_staging("src")
    for s in range(S):
        st[s] = pd.stream_input(s, blocks, B).reshape(blocks, -1).view(np.uint8)
    rt.run_all(prestaged=True)
    for rep in range(2):
        t0 = time.perf_counter(); rt.reset(); t1 = time.perf_counter()
        reps = rt.run_all(prestaged=True); t2 = time.perf_counter()
    print(f"pipeline={pipe}: reset {1e3*(t1-t0):.1f} ms, run_all {1e3*(t2-t1):.1f} ms", flush=True)
    # pieces
    lib = rt.lib
    rt.reset()
    t0 = time.perf_counter(); rt.stage_sources(0, blocks, prestaged=True); lib.pb_stream_sync(rt.stream); t1 = time.perf_counter()
    rt.stage_control(0, blocks); lib.pb_stream_sync(rt.stream); t2 = time.perf_counter()
    rt.fire_epoch(0, blocks); lib.pb_stream_sync(rt.stream); t3 = time.perf_counter()
    f = rt.graph.fifo_into(pd and rt.graph.actor("sink").input_ports[0] and __import__("paper_1802_06625_b200.graph", fromlist=["PortRef"]).PortRef("sink", "in"))
    stg = rt.storage[f.id]
    rt._d2h_chunks(stg.data, stg.stream_stride, 8 * B, rt.sink_host[f.id][0], blocks, 0); lib.pb_stream_sync(rt.stream); t4 = time.perf_counter()
    print(f"  H2D src {1e3*(t1-t0):.1f} ms ({536870912/(t1-t0)/1e9:.1f} GB/s), control {1e3*(t2-t1):.1f}, fire {1e3*(t3-t2):.1f}, D2H {1e3*(t4-t3):.1f} ms ({536870912/(t4-t3)/1e9:.1f} GB/s)", flush=True)
    rt.close()
    if pipe == 8:
        pass
