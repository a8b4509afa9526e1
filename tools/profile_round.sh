#!/usr/bin/env bash
# Round profiling pass (run under gpurun): launch list of one bench step,
# ncu --set full of the dominant kernel (fused filter bank) and of the
# per-actor FIR kernel; summaries land in gpurun_out/ and are copied to
# profiles/ by hand.
set -x
mkdir -p gpurun_out
R=${ROUND:-r1}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/${R}_launches.csv python bench.py --steps 3 --warmup 3 --skip-cpu --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fir_persistent -s 2 -c 1 \
  -o gpurun_out/${R}_bank python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 > gpurun_out/${R}_ncu_bank.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fir_persistent -s 1 -c 1 \
  -o gpurun_out/${R}_fir python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 --no-fuse > gpurun_out/${R}_ncu_fir.log 2>&1
python tools/ncu_summary.py gpurun_out/${R}_bank.ncu-rep > gpurun_out/${R}_ncu_bank.json
python tools/ncu_summary.py gpurun_out/${R}_fir.ncu-rep > gpurun_out/${R}_ncu_fir.json
