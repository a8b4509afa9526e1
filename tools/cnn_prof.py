"""Role timing of conv_pool_kernel (needs a -DPB_CONV_PROF=1 build, selected
with PB_LIB_PATH): per layer, the mean per-CTA cycles each role spends in
each phase, summed over the launch (slots: csrc/pb_cnn.cu PROF calls)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_1802_06625_b200 import RuntimeConfig
from paper_1802_06625_b200.apps import vision
from paper_1802_06625_b200.engine import DeviceRuntime

SLOTS = {0: "cvt.wait_sched", 1: "cvt.wait_raw", 2: "cvt.wait_empty", 3: "cvt.fill",
         4: "cvt.fence+arrive", 5: "cvt.bar+release", 6: "cvt.raw_issue", 7: "mma.cursor",
         8: "mma.wait_full", 9: "mma.wait_acc_empty", 10: "mma.issue", 11: "epi.super+cursor",
         12: "epi.wait_acc_full", 13: "epi.tmem", 14: "epi.math+store", 15: "sched.total"}


def main(S=4, F=64, R=24, steps=5, debug=0):
    desc = vision.build_description(R, policy="fixed_policy")
    rt = DeviceRuntime(desc, config=RuntimeConfig(source_firings=F, epoch=F), n_streams=S,
                       seeds=list(range(S)), sources={"src": [None] * S})
    st = rt.source_staging("src")
    for s in range(S):
        st[s] = vision.make_frames(s, F * R).reshape(F, -1).view(np.uint8)
    lib = rt.lib
    for item in rt.launches:
        if item[0] == "conv":
            item[1].debug = debug
    rt.reset()
    rt.stage_sources(0, F, prestaged=True)
    rt.stage_control(0, F)
    buf = np.zeros((160, 16), np.uint64)
    acc = {"l1": np.zeros(16), "l2": np.zeros(16)}
    seen = [0]

    def hook(kind, phase):
        if kind != "conv":
            return
        lib.pb_stream_sync(rt.stream)
        lib.pb_conv_debug_counters(buf.ctypes.data, 1)
        if phase == "post":
            layer = "l1" if seen[0] % 2 == 0 else "l2"
            seen[0] += 1
            acc[layer] += buf[:148].astype(np.float64).mean(axis=0)
    rt.fire_epoch(0, F)
    for _ in range(steps):
        rt.fire_epoch(0, F, hook=hook)
    lib.pb_stream_sync(rt.stream)
    out = {}
    for layer, v in acc.items():
        v = v / steps
        out[layer] = {SLOTS[k]: round(float(v[k])) for k in SLOTS}
    rt.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
