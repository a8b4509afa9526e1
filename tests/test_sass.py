"""The built library carries Blackwell-native instructions where DESIGN.md
says it does (cuobjdump of libprune_b200.so, sm_100a): tcgen05 MMAs
(UTCHMMA / UTCQMMA), TMEM loads (LDTM) and TMA tensor loads (UTMALDG) in the
conv kernels, tcgen05 MMAs in the dense layer, bulk-copy TMA (UBLKCP) feeding
the DPD stream kernel, and no FFMA in the bit-exact FIR paths."""
import re
import shutil
import subprocess

import pytest

from paper_1802_06625_b200 import build

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


@pytest.fixture(scope="module")
def sass():
    lib = build.build()
    try:
        out = subprocess.run([CUOBJDUMP, "-sass", str(lib)], capture_output=True, text=True,
                             timeout=300, check=True).stdout
    except (FileNotFoundError, subprocess.CalledProcessError) as e:
        pytest.skip(f"cuobjdump unavailable: {e}")
    funcs = {}
    name = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name is not None:
            funcs[name].append(line)
    return {k: "\n".join(v) for k, v in funcs.items()}


def ops(sass, pattern):
    bodies = [v for k, v in sass.items() if re.search(pattern, k)]
    assert bodies, f"no kernel matching {pattern}"
    return bodies


@pytest.mark.parametrize("kernel", [r"conv_pool_kernelILi0ELi3E", r"conv_pool_kernelILi1ELi32E"])
def test_conv_kernels_use_tcgen05_and_tmem(sass, kernel):
    for body in ops(sass, kernel):
        assert re.search(r"\bUTC[HQ]MMA", body), kernel
        assert re.search(r"\bLDTM\b", body), kernel


def test_layer1_input_tiles_arrive_by_tma(sass):
    for body in ops(sass, r"conv_pool_kernelILi0ELi3E"):
        assert re.search(r"\bUTMALDG\b", body)


def test_layer2_runs_on_cta_pairs(sass):
    (body,) = ops(sass, r"conv_pool_kernelILi1ELi32ELb1E")
    assert "UTCHMMA.2CTA" in body or "2CTA" in body


def test_dense_kernel_uses_tcgen05(sass):
    for body in ops(sass, r"dense_kernel"):
        assert re.search(r"\bUTC[HQ]MMA", body) and re.search(r"\bLDTM\b", body)


def test_dpd_stream_kernel_is_fed_by_bulk_tma(sass):
    for body in ops(sass, r"bank_stream_kernel"):
        assert re.search(r"\bUBLKCP\b", body)


def test_exact_fir_paths_have_no_fma(sass):
    # fir_persistent<bank, EXACT> / <actors, EXACT>: every product and sum is
    # rounded separately (predistortion.py:51-65 under numpy), so no FFMA
    for body in ops(sass, r"fir_persistentILb[01]ELi0E"):
        assert not re.search(r"\bFFMA\b", body)


def test_row_conv_kernels_are_tensor_memory_native(sass):
    """The default conv path (pb_conv_rows.cu): layer 1 bf16 TS MMAs (A in
    TMEM: UTCHMMA with a tmem A operand, tcgen05.st = STTM) fed by bulk copies
    (UBLKCP); layer 2 on the int8 tensor cores (UTCIMMA) with its A operand
    written to TMEM (STTM) and its accumulators read back (LDTM)."""
    (l1,) = ops(sass, r"conv_rows_kernelILi3ELb0E")
    assert re.search(r"\bUTCHMMA\b.*tmem\[", l1) and re.search(r"\bSTTM\b", l1)
    assert re.search(r"\bUBLKCP\b", l1) and re.search(r"\bLDTM\b", l1)
    (l2,) = ops(sass, r"conv_rows_kernelILi32ELb1E")
    assert re.search(r"\bUTCIMMA\b", l2) and re.search(r"\bSTTM\b", l2)
    assert re.search(r"\bLDTM\b", l2)
    assert not re.search(r"\bUTCHMMA\b", l2)   # no bf16 products left in the int8 layer
