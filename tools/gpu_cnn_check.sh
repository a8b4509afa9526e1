# CNN: GPU tests, timings per layer, role timing
timeout 300 python -m pytest tests/test_cnn_gpu.py tests/test_mixed_gpu.py -q -x --timeout 120 -p no:cacheprovider 2>&1 | tail -4
for d in 0 4; do
  echo -n "debug=$d "; timeout 60 python tools/cnn_bench.py 4 64 24 10 $d | python -c "import json,sys;d=json.load(sys.stdin);print({k:round(v,3) for k,v in d['kernel_ms'].items()}, round(d['frames_per_s']/1e6,3), 'M frames/s')"
done
timeout 60 python tools/cnn_bench.py 4 64 24 1 16 2>&1 | grep conv_rows_prof | sort | uniq | awk 'NR%4==1'
