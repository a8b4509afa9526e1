# row-streaming conv (A in TMEM) vs the round-1 tile kernel: CNN tests + timing
set -x
timeout 60 python tools/cnn_bench.py 1 1 2 1 > gpurun_out/cnn_tiny.json 2>&1; echo tiny rc=$?; cat gpurun_out/cnn_tiny.json | tail -3
timeout 200 python -m pytest tests/test_cnn_gpu.py -q -x --timeout 60 -p no:cacheprovider 2>&1 | tail -15
timeout 60 python tools/cnn_bench.py 4 64 24 10 > gpurun_out/cnn_rows.json 2>&1; echo rc=$?
PB_CONV_IMPL=tiles timeout 120 python tools/cnn_bench.py 4 64 24 10 > gpurun_out/cnn_tiles.json 2>&1; echo rc=$?
cat gpurun_out/cnn_rows.json gpurun_out/cnn_tiles.json | cut -c1-600
