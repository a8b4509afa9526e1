mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_pool -c 2 -o gpurun_out/cnn_conv python tools/cnn_bench.py 1 4 24 1 > gpurun_out/ncu_cnn.log 2>&1
tail -5 gpurun_out/ncu_cnn.log
python tools/ncu_summary.py gpurun_out/cnn_conv.ncu-rep > gpurun_out/cnn_conv.json; head -c 3000 gpurun_out/cnn_conv.json
