# the int8 conv kernel under ncu --set full (kernel replay; it timed out once)
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:conv_rows_kernel -c 2 \
  -o gpurun_out/r2_cnn_i8 python tools/cnn_bench.py 4 64 24 1 > gpurun_out/ncu_i8.log 2>&1; echo "full i8: $?"; grep -v "^==PROF== Profiling" gpurun_out/ncu_i8.log | tail -5; grep -c "Profiling" gpurun_out/ncu_i8.log
python tools/ncu_summary.py gpurun_out/r2_cnn_i8.ncu-rep > gpurun_out/r2_ncu_cnn_i8.json 2>/dev/null; head -c 300 gpurun_out/r2_ncu_cnn_i8.json
