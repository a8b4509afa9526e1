mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_pool|dense_kernel" -c 3 -o gpurun_out/cnn2 python tools/cnn_bench.py 2 16 24 1 > gpurun_out/ncu_cnn2.log 2>&1
tail -3 gpurun_out/ncu_cnn2.log
