"""Write tests/golden/apps.json: the reference's own app graph descriptions
(predistortion, bypass, motion; input path "input.bin") and their input
generators' first bytes, by importing the REFERENCE package (tokenflow from
/root/reference/pkg/src).  Run here (the build container) only:

    python tests/golden/make_apps.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

REF = Path(os.environ.get("PRUNE_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))

from tokenflow.apps import bypass as rbp  # noqa: E402
from tokenflow.apps import motion as rmo  # noqa: E402
from tokenflow.apps import predistortion as rpd  # noqa: E402

OUT = Path(__file__).resolve().parent
apps = {
    "predistortion": {"description": rpd.build_description("input.bin"),
                      "input_sha256": hashlib.sha256(rpd.make_input(11, 8)).hexdigest()},
    "bypass": {"description": rbp.build_description("input.bin"),
               "input_sha256": hashlib.sha256(rbp.make_input(5, 8)).hexdigest()},
    "motion": {"description": rmo.build_description("input.bin"),
               "input_sha256": hashlib.sha256(rmo.make_input(7, 4)).hexdigest()},
}
(OUT / "apps.json").write_text(json.dumps(apps, indent=1, sort_keys=True))
print("wrote", OUT / "apps.json")
