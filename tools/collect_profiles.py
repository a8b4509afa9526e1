"""Copy the round's GPU evidence from gpurun_out/ into profiles/ (tracked):
launch list (per-launch time + DRAM bytes, cold-cache and serialised under
ncu: compare shares, not absolutes), ncu --set full summaries, the DRAM
traffic per launch of the headline kernels (read by bench.py as
roofline.traffic) and the bench line."""
import csv
import json
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
R = sys.argv[1] if len(sys.argv) > 1 else "r1"
out = ROOT / "gpurun_out"
prof = ROOT / "profiles"


def launches(name=f"{R}_launches.csv"):
    rows = [r for r in csv.reader(open(out / name)) if len(r) > 10]
    h = rows[0]
    iK, iM, iV, iI = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = {}
    for r in rows[1:]:
        e = d.setdefault(int(r[iI]), {"id": int(r[iI]), "kernel": r[iK].split("(")[0]})
        v = float(r[iV].replace(",", ""))
        e[{"gpu__time_duration.sum": "ns", "dram__bytes_read.sum": "dram_read",
           "dram__bytes_write.sum": "dram_write"}.get(r[iM], r[iM])] = v
    return [d[k] for k in sorted(d)]


L = launches()
LC = launches(f"{R}_launches_cnn.csv") if (out / f"{R}_launches_cnn.csv").exists() else []
(prof / f"{R}_launches_cnn.json").write_text(json.dumps({
    "command": "tools/profile_round.sh: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
               "dram__bytes_write.sum --clock-control none -c 60 python tools/cnn_bench.py 4 64 24 2",
    "note": "CNN vision graph, 4 streams x 64 firings x 24 frames per launch; cold-cache and "
            "serialised under ncu: compare shares, not absolutes; units ns and bytes",
    "launches": LC}, indent=1))
(prof / f"{R}_launches.json").write_text(json.dumps({
    "command": "tools/profile_round.sh: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
               "dram__bytes_write.sum --clock-control none -c 80 python bench.py --steps 2 "
               "--warmup 3 --skip-cpu --e2e-steps 0 --cnn-steps 1 --cnn-e2e-steps 0",
    "note": "per-launch device times, cold-cache and serialised under ncu: compare shares, "
            "not absolutes; units ns and bytes",
    "launches": L}, indent=1))
traffic = {}


def last(kname):
    xs = [x for x in L + LC if kname in x["kernel"]]
    return xs[-1] if xs else None


m, p = last("bank_stream_kernel"), last("bank_plan")
if m and p:
    traffic["bank_plan_par_kernel + bank_stream_kernel"] = \
        m["dram_read"] + m["dram_write"] + p["dram_read"] + p["dram_write"]
e = last("fir_persistent<1, 0>")
if e:
    traffic["fir_persistent<bank, EXACT>"] = e["dram_read"] + e["dram_write"]
# both conv layers run as the row-streaming kernel (pb_conv_rows.cu)
for nm, pat in (("conv_rows_kernel<3, false>", "conv_rows_kernel<3, 0>"),
                ("conv_rows_kernel<32, true>", "conv_rows_kernel<32, 1>"),
                ("dense_kernel", "dense_kernel")):
    x = last(pat)
    if x:
        traffic[nm] = x["dram_read"] + x["dram_write"]
(prof / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1))
for r in ("merged", "exact", "cnn", "dense"):
    src = out / f"{R}_ncu_{r}.json"
    if src.exists():
        shutil.copy(src, prof / f"{R}_ncu_{r}.json")
if (out / "bench.json").exists():
    shutil.copy(out / "bench.json", prof / f"{R}_bench.json")
print(json.dumps(traffic, indent=1))
