# layer-1 row-parity MMA split: CNN tests, C3 throughput (repeated), role timing, ncu HW counters
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cnn_gpu.py tests/test_mixed_gpu.py -q -p no:cacheprovider -s --tb=line 2>&1 | grep -E "worst|passed|failed|Error|error|assert" | tail -8
for i in 1 2 3; do timeout 60 python tools/cnn_bench.py 4 64 24 50 2>&1 | tail -1; done
timeout 60 python tools/cnn_bench.py 4 64 24 1 16 2>&1 | grep -E 'conv_rows_prof' | sort | uniq | awk 'NR%4==1' | cut -c1-200
M=$(python tools/ncu_summary.py --metrics)
timeout 300 ncu --metrics $M --clock-control none -k regex:"conv_rows_kernel|dense_kernel" -c 3 \
  -o gpurun_out/r2_cnn_hw python tools/cnn_bench.py 4 64 24 1 > gpurun_out/ncu_hw.log 2>&1; echo "ncu hw: $?"
python tools/ncu_summary.py gpurun_out/r2_cnn_hw.ncu-rep > gpurun_out/r2_ncu_cnn_hw.json 2>/dev/null; head -c 1500 gpurun_out/r2_ncu_cnn_hw.json
