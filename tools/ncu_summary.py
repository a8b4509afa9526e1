"""Summarise an ncu --set full report: key metrics per kernel (used for profiles/)."""
import csv
import io
import json
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.per_cycle_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'launch__grid_size', 'launch__block_size',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__cycles_elapsed.avg.per_second', 'smsp__inst_executed.sum']
STALLS = ['barrier', 'long_scoreboard', 'short_scoreboard', 'wait', 'math_pipe_throttle',
          'mio_throttle', 'not_selected', 'selected', 'dispatch_stall', 'lg_throttle',
          'no_instruction', 'drain', 'branch_resolving', 'sleeping', 'membar', 'misc']


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        d = {}
        for w in WANT:
            if w in hdr:
                d[w] = vals[hdr.index(w)] + " " + units[hdr.index(w)]
        st = {}
        for s in STALLS:
            key = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if key in hdr:
                st[s] = float(vals[hdr.index(key)] or 0)
        d["stalls_per_issue"] = {k: round(v, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])
                                 if v > 0.01}
        key = name.split("(")[0]
        if key in res:
            key = f"{key} #{sum(k.startswith(key) for k in res) + 1}"
        res[key] = d
    return res


def metric_list():
    """The counters above as an ncu --metrics list: hardware counters only (no
    SASS-patching sections), for kernels whose --set full replay stalls."""
    return ",".join(WANT + [f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
                            for s in STALLS])


if __name__ == "__main__":
    if sys.argv[1] == "--metrics":
        print(metric_list())
        sys.exit(0)
    print(json.dumps(summarise(sys.argv[1]), indent=1))
