B="python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 --skip-cnn"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bank_plan" -c 1 -o gpurun_out/plan_full $B > /dev/null 2>&1; echo "ncu: $?"
timeout 600 ncu --set full --cache-control none --clock-control none -k regex:"bank_plan" -c 3 -o gpurun_out/plan_warm $B > /dev/null 2>&1; echo "ncu warm: $?"
