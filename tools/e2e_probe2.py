"""DPD e2e phases on the box: SHA-256 throughput of the host, PCIe each way,
and run_all at several pipeline depths / hashing thread counts."""
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1802_06625_b200 import RuntimeConfig
from paper_1802_06625_b200.apps import predistortion as pd
from paper_1802_06625_b200.engine import DeviceRuntime

S, blocks, B = 64, 256, 4096
out = {"cpus": os.cpu_count()}
buf = np.random.default_rng(0).integers(0, 255, S * blocks * 8 * B, dtype=np.uint8).reshape(S, -1)
for th in (8, 16, 32):
    with ThreadPoolExecutor(th) as ex:
        t0 = time.perf_counter()
        list(ex.map(lambda s: hashlib.sha256(buf[s]).hexdigest(), range(S)))
        out[f"sha256_GBps_{th}thr"] = buf.nbytes / (time.perf_counter() - t0) / 1e9
for pipe in (8, 16, 32):
    for th in (15, 16):
        rt = DeviceRuntime(pd.build_description(B, 4), config=RuntimeConfig(
            source_firings=blocks, epoch=blocks, pipeline=pipe, exact=False, host_threads=th),
            n_streams=S, seeds=[1000 + s for s in range(S)], sources={"src": [None] * S})
        st = rt.source_staging("src")
        for s in range(S):
            st[s] = pd.stream_input(s, blocks, B).reshape(blocks, -1).view(np.uint8)
        rt.run_all(prestaged=True)
        ts = []
        for rep in range(3):
            t0 = time.perf_counter()
            rt.run_all(prestaged=True)
            ts.append(time.perf_counter() - t0)
        out[f"run_all_ms_pipe{pipe}_thr{th}"] = 1e3 * min(ts)
        rt.close()
print(json.dumps(out, indent=1))
