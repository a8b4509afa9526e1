VARIANTS="copyonly" bash tools/gpu_ms.sh
B="python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 --skip-cnn"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bank_" -c 2 -o gpurun_out/ms_full $B > /dev/null 2>&1; echo "ncu: $?"
python tools/ncu_summary.py gpurun_out/ms_full.ncu-rep > gpurun_out/ms_full.json
