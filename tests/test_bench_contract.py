"""bench.py's reference arm (the reference's own CPU path, no GPU needed)
prints the contract's JSON line: one line, impl "reference", the headline
metric/unit, a cpu_baseline describing the run and an e2e block."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_contract_line():
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "1", "--cpu-streams", "2", "--cpu-blocks", "2", "--block", "256"],
        capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    base = json.loads((ROOT / "BASELINE.json").read_text())
    assert d["impl"] == "reference"
    assert d["metric"] == base["metric"] and d["unit"] == "Msamples/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_honours_steps_and_workload_string():
    """--steps/--warmup are the reference arm's own (BENCH r1: same_steps
    false); config.workload is the string our arm reports."""
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "3",
         "--warmup", "2", "--cpu-streams", "2", "--cpu-blocks", "2", "--block", "256"],
        capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["steps"] == 3 and d["warmup"] == 2
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["config"]["workload"] == bench.workload_name(64, 256, 256, 4)


def test_gpus_flag_launches_ranks_without_torchrun():
    """`python bench.py --gpus 2` (the driver's command form, no torchrun)
    starts two ranks itself; --plumbing checks the launch path on CPU (gloo)."""
    import os
    env = dict(os.environ, PB_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--plumbing"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and sorted(r["rank"] for r in d["ranks"]) == [0, 1]
    assert len({r["pid"] for r in d["ranks"]}) == 2
