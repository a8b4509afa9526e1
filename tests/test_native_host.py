"""libprune_b200 on the host: loads, exports every declared symbol, and its
host-only functions (capacity plan, gates, CPython-compatible policies,
crc32) match the reference.  No device calls."""
import ctypes as C
import json
import random
import re
import zlib
from pathlib import Path

import pytest

from paper_1802_06625_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "prune_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-zA-Z_0-9]+\*?\s+\*?(pb_[a-z0-9_]+)\(",
                                 text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) > 40
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def ref_layout(rate, delay, factor):
    # restated from fifos.py:87-98
    aligned = delay % rate == 0
    if aligned:
        return aligned, max(rate * factor, delay), None
    return aligned, rate * factor + delay, (rate * factor, 0, delay)


def ref_writer_gate(w, rate, delay, factor, aligned):
    if aligned:
        slots = max(rate * factor, delay)
        last = delay + (w + 1) * rate - 1 - slots
        return 0 if last < 0 else last // rate + 1
    n, c = divmod(w, factor)
    if n == 0:
        return 0
    if delay > rate * factor:
        return ref_copy_gate(n - 1, rate, delay, factor)
    return (delay + (n - 1) * rate * factor + (c + 1) * rate - 1) // rate + 1


def ref_reader_gate(i, rate, delay):
    need = (i + 1) * rate - delay
    return 0 if need <= 0 else -(-need // rate)


def ref_copy_gate(n, rate, delay, factor):
    span = min(delay, rate * factor)
    return n * factor + (span - 1) // rate + 1


def test_capacity_plan_and_gates_sweep():
    lib = _lib.load()
    for rate in range(1, 6):
        for delay in range(0, 12):
            for factor in range(2, 5):
                p = _lib.Plan()
                assert lib.pb_layout_plan(rate, delay, factor, 3, C.byref(p)) == 0
                aligned, slots, copy = ref_layout(rate, delay, factor)
                assert bool(p.aligned) == aligned and p.slots == slots
                assert p.nbytes == slots * 3
                if copy:
                    assert (p.copy_src, p.copy_dst, p.copy_count) == copy
                for w in range(0, 3 * factor + 2):
                    assert lib.pb_writer_gate(w, rate, delay, factor, int(aligned)) == \
                        ref_writer_gate(w, rate, delay, factor, aligned)
                    assert lib.pb_reader_gate(w, rate, delay) == ref_reader_gate(w, rate, delay)
                    if not aligned:
                        assert lib.pb_copy_gate(w, rate, delay, factor) == \
                            ref_copy_gate(w, rate, delay, factor)


def test_capacity_frozen_values():
    # pkg/tests/test_fifo.py:36-41 style: rate 2, delay 3, factor 3 is unaligned
    p = _lib.Plan()
    _lib.load().pb_layout_plan(2, 3, 3, 4, C.byref(p))
    assert (p.aligned, p.slots, p.nbytes) == (0, 9, 36)


@pytest.mark.parametrize("args", [(0, 0, 3, 1), (1, -1, 3, 1), (1, 0, 1, 1), (1, 0, 3, 0)])
def test_invalid_params_raise(args):
    rate, delay, factor, tb = args
    with pytest.raises(_lib.InvalidParams):
        _lib.call("pb_layout_plan", rate, delay, factor, tb, None)


KINDS = {"fixed_policy": 0, "alternate_policy": 1, "seeded_policy": 2, "subset_policy": 3}


def native_tokens(kind, length, param, seed, n, first=0, state=None):
    lib = _lib.load()
    if state is None:
        state = (C.c_uint8 * _lib.PB_POLICY_STATE_BYTES)()
        assert lib.pb_policy_init(state, -1 if seed is None else seed) == 0
    out = (C.c_uint8 * (n * length))()
    assert lib.pb_policy_tokens(state, kind, length, param, first, n, out, length) == 0
    return [bytes(out[i * length:(i + 1) * length]).hex() for i in range(n)], state


def test_policies_match_reference_golden(golden):
    for key, vecs in golden["policies"].items():
        name, params, seed = key.split("|")
        params = json.loads(params)
        seed = None if seed == "None" else int(seed)
        param = params.get("element", params.get("min_active", 2))
        got, _ = native_tokens(KINDS[name], params["length"], param, seed, len(vecs))
        assert got == vecs, key


def test_policy_state_continues_across_epochs():
    full, _ = native_tokens(3, 10, 2, 77, 50)
    a, st = native_tokens(3, 10, 2, 77, 20)
    b, _ = native_tokens(3, 10, 2, 77, 30, first=20, state=st)
    assert a + b == full


@pytest.mark.parametrize("seed", [0, 1, 12345, 2**31 - 1, 2**40 + 17])
def test_subset_policy_matches_cpython_random(seed):
    rng = random.Random(seed)
    for length, lo in [(4, 2), (10, 2), (25, 1), (40, 3)]:
        pass
    for length, lo in [(4, 2), (10, 2), (25, 1), (40, 3)]:
        rng = random.Random(seed)
        want = []
        for _ in range(40):
            size = rng.randint(min(lo, length), length)
            chosen = set(rng.sample(range(1, length + 1), size))
            want.append(bytes(1 if k in chosen else 0 for k in range(1, length + 1)).hex())
        got, _ = native_tokens(3, length, lo, seed, 40)
        assert got == want, (length, lo)


def test_streams_entry_point_matches_single():
    lib = _lib.load()
    S, n, L = 5, 33, 4
    states = (C.c_uint8 * (_lib.PB_POLICY_STATE_BYTES * S))()
    for s in range(S):
        lib.pb_policy_init(C.addressof(states) + s * _lib.PB_POLICY_STATE_BYTES, 1000 + s)
    out = (C.c_uint8 * (S * n * L))()
    assert lib.pb_policy_tokens_streams(states, S, 3, L, 2, 0, n, out, L, 3) == 0
    for s in range(S):
        want, _ = native_tokens(3, L, 2, 1000 + s, n)
        got = [bytes(out[(s * n + i) * L:(s * n + i + 1) * L]).hex() for i in range(n)]
        assert got == want


def test_crc32_matches_zlib():
    lib = _lib.load()
    for text in [b"", b"conf", b"src", b"a much longer actor identifier"]:
        buf = C.create_string_buffer(text)
        assert lib.pb_crc32(buf, len(text)) == zlib.crc32(text)


def test_no_fma_in_fir_kernels():
    """Bit-exactness needs every FIR product rounded on its own: the SASS of
    the FIR / filter-bank / sum / matmul kernels must hold no FFMA/FFMA2."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True,
                          check=True).stdout
    fn, bad, seen = None, [], set()
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split("Function :")[1].strip()
            continue
        # fir_persistent<*, 2> / <bank, 3> are the opt-in tolerance modes
        # (PB_FIR_FMA, PB_FIR_MERGED)
        exact = not ("fir_persistent" in fn and ("Li2E" in fn or "Li3E" in fn)) if fn else False
        if fn and exact and any(k in fn for k in ("fir_persistent", "branch_sum", "matmul")):
            seen.add(fn)
            if "FFMA" in line or "HFMA2.MMA" in line:
                bad.append((fn, line.strip()))
    assert len(seen) >= 6 and not bad, bad[:5]
    assert "FMUL2" in sass and "FADD2" in sass


def test_no_cpu_fallback_without_a_device(tmp_path):
    """The product path has no CPU fallback: without a visible CUDA device the
    drop-in run() raises DeviceUnavailable instead of computing anything."""
    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    from paper_1802_06625_b200 import DeviceUnavailable, RuntimeConfig, run
    from paper_1802_06625_b200.apps import predistortion as pd
    p = tmp_path / "input.bin"
    p.write_bytes(pd.make_input(11, 4))
    with pytest.raises(DeviceUnavailable):
        run(pd.build_description(256, 4, str(p)), config=RuntimeConfig(source_firings=4, seed=11))
