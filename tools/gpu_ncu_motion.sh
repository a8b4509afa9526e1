# ncu hardware counters of the fused motion region and the bypass region
M=$(python tools/ncu_summary.py --metrics)
timeout 300 ncu --metrics $M --clock-control none -k regex:"motion_region|bypass_region" -c 2 -o gpurun_out/r2_apps python tools/motion_bench.py 64 64 2 1 > /dev/null 2>&1; echo "motion: $?"
timeout 300 ncu --metrics $M --clock-control none -k regex:"bypass_region" -c 1 -o gpurun_out/r2_apps_b python tools/bypass_bench.py 256 256 2 1 > /dev/null 2>&1; echo "bypass: $?"
python tools/ncu_summary.py gpurun_out/r2_apps.ncu-rep > gpurun_out/r2_ncu_motion.json; python tools/ncu_summary.py gpurun_out/r2_apps_b.ncu-rep > gpurun_out/r2_ncu_bypass.json
cat gpurun_out/r2_ncu_motion.json | head -60
