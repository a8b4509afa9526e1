"""BASELINE config 1 through the drop-in run(): the reference's default DPD app
(B=256, K=4, 160 blocks, seed 11) end to end, first call (CUDA context, library
load, allocation) and warm calls, next to the reference interpreter (oracle/_ref)."""
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_06625_b200 import RuntimeConfig, run
from paper_1802_06625_b200.apps import predistortion as pd

out = {}
with tempfile.TemporaryDirectory() as d:
    path = Path(d) / "input.bin"
    path.write_bytes(pd.make_input(11, 160, 256))
    desc = pd.build_description(256, 4, input_path=str(path))
    for k in range(4):
        t0 = time.perf_counter()
        rep = run(desc, config=RuntimeConfig(source_firings=160, seed=11))
        out[f"run_ms_{k}"] = 1e3 * (time.perf_counter() - t0)
    out["digest"] = rep.sink_digests
    ref = Path(__file__).resolve().parent.parent / "oracle" / "_ref"
    if ref.is_dir():
        sys.path.insert(0, str(ref))
        from tokenflow.model import build_graph  # noqa: E402
        from tokenflow.interp import interpret  # noqa: E402
        g = build_graph(desc)
        t0 = time.perf_counter()
        r = interpret(g, source_firings=160, seed=11)
        out["ref_interpret_ms"] = 1e3 * (time.perf_counter() - t0)
        out["ref_digest"] = r.sink_digests
print(json.dumps(out, indent=1))
