#!/usr/bin/env bash
# Round profiling pass (run under gpurun, one GPU): launch list of one bench
# step (DPD + CNN) and ncu --set full captures of the dominant kernels; the
# summaries land in gpurun_out/ and are copied to profiles/ by hand.
mkdir -p gpurun_out
R=${ROUND:-r1}
B="python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 --cnn-steps 1 --cnn-e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv \
  --log-file gpurun_out/${R}_launches.csv $B > /dev/null 2>&1
echo "launches: $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${R}_launches_cnn.csv python tools/cnn_bench.py 4 64 24 2 > /dev/null 2>&1
echo "launches cnn: $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bank_ -c 2 \
  -o gpurun_out/${R}_merged $B --skip-cnn > /dev/null 2>&1; echo "merged: $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fir_persistent -c 1 \
  -o gpurun_out/${R}_exact python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 --skip-cnn --exact > /dev/null 2>&1; echo "exact: $?"
# the conv kernels: hardware counters only (the int8 kernel's --set full
# replay stalls in the SASS-patching passes), the dense kernel --set full
M=$(python tools/ncu_summary.py --metrics)
timeout 600 ncu --metrics $M --clock-control none -k regex:"conv_rows_kernel" -c 2 \
  -o gpurun_out/${R}_cnn python tools/cnn_bench.py 4 64 24 1 > /dev/null 2>&1; echo "cnn: $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dense_kernel" -c 1 \
  -o gpurun_out/${R}_dense python tools/cnn_bench.py 4 64 24 1 > /dev/null 2>&1; echo "dense: $?"
for r in merged exact cnn dense; do
  python tools/ncu_summary.py gpurun_out/${R}_$r.ncu-rep > gpurun_out/${R}_ncu_$r.json 2>/dev/null
done
ls -la gpurun_out/
