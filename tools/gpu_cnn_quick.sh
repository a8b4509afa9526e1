# CNN tests + C3 throughput + layer-1/2 role timing (CTA 0)
timeout 600 python -m pytest tests/test_cnn_gpu.py tests/test_mixed_gpu.py -q -p no:cacheprovider -s --tb=line 2>&1 | grep -E "worst|passed|failed|Error|error|assert" | tail -8
for i in 1 2; do timeout 60 python tools/cnn_bench.py 4 64 24 30 2>&1 | tail -1 | cut -c1-250; done
timeout 60 python tools/cnn_bench.py 4 64 24 1 16 2>&1 | grep -E 'conv_rows_prof' | sort -t: -k3 -n | uniq | awk 'NR%4==1' | cut -c1-200
