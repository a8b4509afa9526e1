# ncu --set full of both row-streaming conv launches at the bench size (6144 frames)
mkdir -p gpurun_out
R=${ROUND:-r2}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_rows_kernel|dense_kernel" -c 3 \
  -o gpurun_out/${R}_cnn python tools/cnn_bench.py 4 64 24 1 > /dev/null 2>&1; echo "cnn: $?"
python tools/ncu_summary.py gpurun_out/${R}_cnn.ncu-rep > gpurun_out/${R}_ncu_cnn.json 2>/dev/null
ls -la gpurun_out
