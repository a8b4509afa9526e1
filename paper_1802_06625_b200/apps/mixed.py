"""BASELINE config 5: one heterogeneous graph holding the DPD filter-bank
region (subset_policy control, dynamic rates) and the adaptive CNN vision
graph (alternate_policy bypass), each with its own host configuration actor
and source, side by side in one description.  Actor and FIFO ids get a
"dpd_" / "cnn_" prefix; the two sinks are dpd_sink and cnn_sink.
"""
from __future__ import annotations

from typing import Any

from . import predistortion, vision


def _prefixed(desc: dict[str, Any], p: str) -> dict[str, Any]:
    actors = []
    for a in desc["actors"]:
        a = dict(a, id=p + a["id"])
        actors.append(a)
    fifos = []
    for f in desc["fifos"]:
        fifos.append(dict(f, id=p + f["id"], src=p + f["src"], dst=p + f["dst"]))
    ctl = desc.get("control", {})
    control = {"value_lengths": {p + k: v for k, v in ctl.get("value_lengths", {}).items()},
               "table": [dict(e, port=p + e["port"], drp=p + e["drp"])
                         for e in ctl.get("table", [])]}
    return {"actors": actors, "fifos": fifos, "control": control}


def build_description(block: int = 4096, branches: int = 4, frames_per_firing: int = 24,
                      dpd_input: str = "dpd.bin", cnn_input: str = "frames.bin") -> dict[str, Any]:
    d = _prefixed(predistortion.build_description(block, branches, input_path=dpd_input), "dpd_")
    c = _prefixed(vision.build_description(frames_per_firing, input_path=cnn_input), "cnn_")
    return {"name": "mixed",
            "actors": d["actors"] + c["actors"],
            "fifos": d["fifos"] + c["fifos"],
            "control": {"value_lengths": {**d["control"]["value_lengths"],
                                          **c["control"]["value_lengths"]},
                        "table": d["control"]["table"] + c["control"]["table"]}}
